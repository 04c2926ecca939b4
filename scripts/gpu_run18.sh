cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_convert.py -m "gpu and not slow" -q --timeout 120 -p no:cacheprovider > gpurun_out/pytest18.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest18.log
timeout 600 python bench.py --config 2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench18_c2.log 2>&1
SFG_COO_V1=1 timeout 600 python bench.py --config 2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench18_c2_v1.log 2>&1
