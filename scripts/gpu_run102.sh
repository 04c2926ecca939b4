cd $GRAFT_REPO_ROOT
for v in 0 1 2; do
SFG_SPMM_VAR=$v timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench102_c5_v$v.log 2>&1
done
echo done
