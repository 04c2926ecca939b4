cd $GRAFT_REPO_ROOT
for ab in 0 7; do
echo "ablate $ab" >> gpurun_out/prof41.log
SFG_TC_ABLATE=$ab SFG_BCSR_TC_VAR=4 timeout 120 python scripts/prof_bcsr.py 65536 >> gpurun_out/prof41.log 2>&1
done
echo "var 3" >> gpurun_out/prof41.log
SFG_BCSR_TC_VAR=3 timeout 120 python scripts/prof_bcsr.py 65536 >> gpurun_out/prof41.log 2>&1
SFG_BCSR_TC_VAR=3 timeout 300 python -m pytest tests/test_gpu_spmm.py -m "gpu and not slow" -q --timeout 60 -p no:cacheprovider -x -k "tensor_core" 2>&1 | tail -1 >> gpurun_out/prof41.log
