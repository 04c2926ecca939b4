cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_spmm.py -m "gpu" -q --timeout 120 -p no:cacheprovider -x > gpurun_out/pytest75.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest75.log
timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench75_c3.log 2>&1
