cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m "gpu and not slow" -q --timeout 120 -p no:cacheprovider > gpurun_out/pytest21.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest21.log
SFG_TRACE_ALLOC=1 timeout 300 python scripts/debug_stall.py > gpurun_out/debug_stall21.log 2>&1
for v in 0 3; do
SFG_COO_PIPE=$v timeout 600 python bench.py --config 2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench21_c2_p$v.log 2>&1
done
SFG_COO_V1=1 timeout 600 python bench.py --config 2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench21_c2_v1.log 2>&1
