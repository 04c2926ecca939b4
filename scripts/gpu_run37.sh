cd $GRAFT_REPO_ROOT
for v in 0 2 3; do
echo "variant $v" >> gpurun_out/prof37.log
SFG_TC_PROF=1 SFG_BCSR_TC_VAR=$v timeout 120 python scripts/prof_bcsr.py 65536 >> gpurun_out/prof37.log 2>&1
done
