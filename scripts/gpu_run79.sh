cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_spmm.py -m "gpu" -q --timeout 120 -p no:cacheprovider -x > gpurun_out/pytest79.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest79.log
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 > gpurun_out/bench79_c4.log 2>&1
