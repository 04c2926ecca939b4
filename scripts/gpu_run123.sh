cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_spmm.py -m gpu -q -p no:cacheprovider -k "tensor_core" > gpurun_out/pytest123.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest123.log
for pf in 0 4 8 16 32; do
  echo "pf $pf" >> gpurun_out/prof123.log
  SFG_TC_PF=$pf timeout 300 python scripts/prof_bcsr.py 524288 >> gpurun_out/prof123.log 2>&1
done
echo done
