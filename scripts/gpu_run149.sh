cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_convert.py tests/test_gpu_spmm.py tests/test_gpu_spmv.py tests/test_gpu_convert_src.py tests/test_gpu_container.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest149.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest149.log
for i in 1 2; do timeout 600 python bench.py --config 3 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench149_c3_$i.log 2>&1; done
echo done
