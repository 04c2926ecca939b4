cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_convert.py tests/test_gpu_spmv.py -m "gpu and not slow" -q --timeout 120 -p no:cacheprovider -x > gpurun_out/pytest27.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest27.log
SFG_ROWPTR_BULK=1 timeout 900 python -m pytest tests/test_gpu_convert.py -m "gpu and not slow" -q --timeout 120 -p no:cacheprovider -x > gpurun_out/pytest27b.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest27b.log
timeout 600 python bench.py --config 2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench27_c2.log 2>&1
SFG_ROWPTR_BULK=1 timeout 600 python bench.py --config 2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench27_c2_bulk.log 2>&1
timeout 600 python bench.py --config 1 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench27_c1.log 2>&1
