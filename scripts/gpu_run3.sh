cd $GRAFT_REPO_ROOT
timeout 300 python scripts/debug_hang.py > gpurun_out/debug3.log 2>&1
echo "exit $?" >> gpurun_out/debug3.log
CUDA_LAUNCH_BLOCKING=1 timeout 300 python scripts/debug_hang.py > gpurun_out/debug3_blocking.log 2>&1
echo "exit $?" >> gpurun_out/debug3_blocking.log
timeout 120 scripts/_bin/gather_bench > gpurun_out/gather_bench.log 2>&1
