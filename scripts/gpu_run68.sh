cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_convert_src.py -q --timeout 120 -p no:cacheprovider -x > gpurun_out/pytest68.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest68.log
