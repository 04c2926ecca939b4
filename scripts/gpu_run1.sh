cd $GRAFT_REPO_ROOT
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/pytest1.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest1.log
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 > gpurun_out/bench_c1.log 2>&1
echo "exit $?" >> gpurun_out/bench_c1.log
timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
echo "exit $?" >> gpurun_out/bench_c3.log
