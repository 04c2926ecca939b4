cd $GRAFT_REPO_ROOT
SFG_DEBUG=1 timeout 200 python scripts/debug_s20.py > gpurun_out/debug6.log 2>&1
echo "exit $?" >> gpurun_out/debug6.log
