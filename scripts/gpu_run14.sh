cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x --timeout 120 -p no:cacheprovider > gpurun_out/pytest14.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest14.log
timeout 300 python scripts/prof_bcsr.py 65536 > gpurun_out/prof14_plain.log 2>&1
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench14_c4.log 2>&1
timeout 600 python bench.py --config 2 --steps 20 --warmup 3 > gpurun_out/bench14_c2.log 2>&1
timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench14_c3.log 2>&1
