cd $GRAFT_REPO_ROOT
timeout 300 python scripts/debug_hang.py > gpurun_out/debug5.log 2>&1
echo "exit $?" >> gpurun_out/debug5.log
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -x --timeout 120 -p no:cacheprovider > gpurun_out/pytest5.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest5.log
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 > gpurun_out/bench5_c2.log 2>&1
echo "exit $?" >> gpurun_out/bench5_c2.log
