cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_rowpart.py tests/test_cpp_api.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest109.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 1 --steps 5 --warmup 3 --rowpart > gpurun_out/bench109_rowpart.log 2>&1
echo "exit $?" >> gpurun_out/bench109_rowpart.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 1 --steps 5 --warmup 3 --config 3 --rowpart --no-e2e --no-cpu-baseline > gpurun_out/bench109_rowpart_c3.log 2>&1
echo "exit $?" >> gpurun_out/bench109_rowpart_c3.log
echo done
