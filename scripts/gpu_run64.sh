cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_mm.py -q --timeout 120 -p no:cacheprovider > gpurun_out/pytest64.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest64.log
timeout 900 python scripts/bench_mm.py 1048576 16 > gpurun_out/bench_mm64.log 2>&1
