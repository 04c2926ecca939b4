cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_rowpart.py tests/test_cpp_api.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest146.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest146.log
timeout 900 python bench.py --config 1 --steps 20 --warmup 5 > gpurun_out/bench146_c1.log 2>&1
echo done
