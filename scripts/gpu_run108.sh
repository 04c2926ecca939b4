cd $GRAFT_REPO_ROOT
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 1 --steps 5 --warmup 3 --rowpart > gpurun_out/bench108_rowpart.log 2>&1
echo "exit $?" >> gpurun_out/bench108_rowpart.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 1 --steps 5 --warmup 3 --config 3 --rowpart --no-e2e --no-cpu-baseline > gpurun_out/bench108_rowpart_c3.log 2>&1
echo "exit $?" >> gpurun_out/bench108_rowpart_c3.log
echo done
