cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_spmm.py tests/test_gpu_rowpart.py tests/test_gpu_spgemm.py tests/test_cpp_api.py -m "gpu" -q --timeout 300 -p no:cacheprovider -x > gpurun_out/pytest97.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest97.log
timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench97_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_spmm_rows_batch" -s 2 -c 1 -o gpurun_out/full97_c3 python bench.py --config 3 --steps 3 --warmup 3 --profile --no-e2e > gpurun_out/full97.log 2>&1
echo done
