cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_spmm.py -m "gpu" -q --timeout 300 -p no:cacheprovider -x > gpurun_out/pytest62.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest62.log
timeout 1200 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench62_c5.log 2>&1
timeout 600 python bench.py --config 1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench62_c1.log 2>&1
