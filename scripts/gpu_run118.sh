cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_convert.py -m gpu -q -p no:cacheprovider -k "int32 or smallest" > gpurun_out/pytest118.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest118.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 1 --steps 5 --warmup 3 --rowpart --no-cpu-baseline > gpurun_out/bench118_rowpart.log 2>&1
echo "exit $?" >> gpurun_out/bench118_rowpart.log
echo done
