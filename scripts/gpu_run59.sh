cd $GRAFT_REPO_ROOT
for v in 0 1 2 3 4; do
echo "var $v" >> gpurun_out/prof59.log
SFG_TC_VAR=$v timeout 120 python scripts/prof_bcsr.py 65536 >> gpurun_out/prof59.log 2>&1
done
