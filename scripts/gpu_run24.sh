cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_convert.py -m "gpu and not slow" -q --timeout 120 -p no:cacheprovider -x > gpurun_out/pytest24.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest24.log
timeout 600 python bench.py --config 2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench24_c2.log 2>&1
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench24_c4.log 2>&1
