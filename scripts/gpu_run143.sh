cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_csc_bcsr.py tests/test_gpu_convert_src.py tests/test_gpu_spmm.py tests/test_gpu_container.py tests/test_gpu_spgemm.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest143.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest143.log
timeout 600 python scripts/bench_bcsr_convert.py > gpurun_out/bench_bcsr_convert143.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches143_bcsrconv.csv python scripts/bench_bcsr_convert.py > /dev/null 2>&1
echo done
