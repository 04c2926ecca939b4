cd $GRAFT_REPO_ROOT
for v in 0 1 2 3 4; do
SFG_SPMM_VAR=$v timeout 600 python bench.py --config 3 --steps 10 --warmup 3 > gpurun_out/bench99_c3_v$v.log 2>&1
done
echo done
