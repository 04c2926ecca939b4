cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x --timeout 120 -p no:cacheprovider > gpurun_out/pytest8.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest8.log
timeout 300 python bench.py --config 2 --steps 5 --warmup 3 --profile > gpurun_out/plain8_c2.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches8_c2.csv \
  python bench.py --config 2 --steps 5 --warmup 3 --profile > gpurun_out/ncu8_c2.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu8_c2.log
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench8_c2.log 2>&1
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench8_c1.log 2>&1
