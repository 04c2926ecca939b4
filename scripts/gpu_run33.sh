cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_spmm.py -m "gpu and not slow" -q --timeout 120 -p no:cacheprovider -x -k "bcsr or BCSR" > gpurun_out/pytest33.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest33.log
timeout 300 python scripts/prof_bcsr.py 65536 > gpurun_out/prof33_plain.log 2>&1
timeout 300 python scripts/prof_bcsr.py 131072 >> gpurun_out/prof33_plain.log 2>&1
