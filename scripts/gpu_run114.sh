cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_csc_bcsr.py tests/test_gpu_convert_src.py tests/test_gpu_spgemm.py tests/test_gpu_container.py -m "gpu" -q --timeout 300 -p no:cacheprovider -x > gpurun_out/pytest114.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest114.log
timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench114_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches114_c3.csv python bench.py --config 3 --steps 2 --warmup 3 --profile > /dev/null 2>&1
echo done
