cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_spmm.py tests/test_gpu_spgemm.py -m "gpu" -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest104.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest104.log
echo done
