cd $GRAFT_REPO_ROOT
SFG_TRACE_ALLOC=1 timeout 300 python scripts/debug_stall.py > gpurun_out/debug_stall.log 2>&1
SFG_TRACE_ALLOC=1 timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench20_c2.log 2>&1
