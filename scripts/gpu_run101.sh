cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_spmm.py tests/test_gpu_rowpart.py -m "gpu" -q --timeout 300 -p no:cacheprovider -x > gpurun_out/pytest101.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest101.log
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench101_c5.log 2>&1
echo done
