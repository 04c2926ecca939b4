cd $GRAFT_REPO_ROOT
for ab in 2 4 6; do
echo "ablate $ab" >> gpurun_out/prof58.log
SFG_TC_ABLATE=$ab timeout 120 python scripts/prof_bcsr.py 65536 >> gpurun_out/prof58.log 2>&1
SFG_TC_PROF=1 SFG_TC_ABLATE=$ab timeout 120 python scripts/prof_bcsr.py 65536 2>&1 | grep "tc prof" | awk '{key=$4; n[key]++; s[key]+=$6} END{for(k in n) printf "warp %s wait %.1f%%\n", k, s[k]/n[k]}' | sort -k2 -n | tr '\n' ' ' >> gpurun_out/prof58.log
echo >> gpurun_out/prof58.log
done
