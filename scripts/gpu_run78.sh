cd $GRAFT_REPO_ROOT
for v in 0 1 2 3; do
echo "var $v" >> gpurun_out/prof78.log
SFG_TC_VAR=$v timeout 120 python scripts/prof_bcsr.py 65536 >> gpurun_out/prof78.log 2>&1
SFG_TC_VAR=$v timeout 300 python -m pytest tests/test_gpu_spmm.py -m "gpu" -q --timeout 60 -p no:cacheprovider -x -k "tensor_core" 2>&1 | tail -1 >> gpurun_out/prof78.log
done
