cd $GRAFT_REPO_ROOT
for ab in 7 23 71 87 0 16; do
echo "ablate $ab" >> gpurun_out/prof47.log
SFG_TC_ABLATE=$ab timeout 120 python scripts/prof_bcsr.py 65536 >> gpurun_out/prof47.log 2>&1
done
