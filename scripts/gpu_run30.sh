cd $GRAFT_REPO_ROOT
for v in 0 1 2 3 4; do
echo "variant $v" >> gpurun_out/coo_exp30.log
SKIP_VARIANTS=1 SFG_COO_RUN=$v timeout 300 python scripts/coo_exp.py >> gpurun_out/coo_exp30.log 2>&1
SFG_COO_RUN=$v timeout 600 python -m pytest tests/test_gpu_spmv.py -m "gpu and not slow" -q --timeout 120 -p no:cacheprovider -x -k "coo or hyb or COO or HYB" 2>&1 | tail -1 >> gpurun_out/coo_exp30.log
done
