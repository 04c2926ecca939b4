cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 120 -p no:cacheprovider -k "bcsr" > gpurun_out/pytest11.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest11.log
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench11_c4.log 2>&1
echo "c4 exit $?" >> gpurun_out/bench11_c4.log
SFG_BCSR_TC_PER_ROW=1 timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench11_c4_perrow.log 2>&1
