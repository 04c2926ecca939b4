cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x --timeout 120 -p no:cacheprovider > gpurun_out/pytest12.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest12.log
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench12_c4.log 2>&1
timeout 600 python bench.py --config 2 --steps 20 --warmup 3 > gpurun_out/bench12_c2.log 2>&1
