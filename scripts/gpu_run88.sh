cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_spmm.py tests/test_gpu_spgemm.py -m "gpu" -q --timeout 300 -p no:cacheprovider -x > gpurun_out/pytest88.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest88.log
timeout 600 python bench.py --config 3 --steps 10 --warmup 3 > gpurun_out/bench88_c3.log 2>&1
SFG_SPMM_MULTI=1 timeout 600 python bench.py --config 3 --steps 10 --warmup 3 > gpurun_out/bench88_c3_multi.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches88_c3.csv python bench.py --config 3 --steps 2 --warmup 3 --profile > /dev/null 2>&1
echo done
