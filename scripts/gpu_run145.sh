cd $GRAFT_REPO_ROOT
for v in 4 5 6; do SFG_SPMV_VAR=$v timeout 600 python bench.py --config 1 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench145_v$v.log 2>&1; done
echo done
