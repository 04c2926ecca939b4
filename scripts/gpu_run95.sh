cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_rowpart.py tests/test_gpu_spmv.py -m "gpu" -q --timeout 300 -p no:cacheprovider -x > gpurun_out/pytest95.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest95.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench95_c2.log 2>&1
echo done
