cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_spmm.py -m "gpu and not slow" -q --timeout 120 -p no:cacheprovider -x > gpurun_out/pytest29.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest29.log
SKIP_VARIANTS=1 timeout 300 python scripts/coo_exp.py > gpurun_out/coo_exp29.log 2>&1
SKIP_VARIANTS=1 SFG_COO_V1=1 timeout 300 python scripts/coo_exp.py > gpurun_out/coo_exp29_v1.log 2>&1
timeout 600 python bench.py --config 2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench29_c2.log 2>&1
