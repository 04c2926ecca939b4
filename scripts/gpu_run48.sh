cd $GRAFT_REPO_ROOT
for ab in 7 0; do
echo "ablate $ab" >> gpurun_out/prof48.log
SFG_TC_PROF=1 SFG_TC_ABLATE=$ab SFG_BCSR_TC_VAR=3 timeout 120 python scripts/prof_bcsr.py 65536 >> gpurun_out/prof48.log 2>&1
done
