cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_convert.py tests/test_gpu_spmv.py tests/test_gpu_spmm.py tests/test_gpu_container.py -m "gpu" -q --timeout 300 -p no:cacheprovider -x > gpurun_out/pytest119.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest119.log
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench119_c2_$i.log 2>&1; done
echo done
