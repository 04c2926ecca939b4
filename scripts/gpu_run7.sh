cd $GRAFT_REPO_ROOT
timeout 200 python scripts/debug_s20.py > gpurun_out/debug7.log 2>&1
echo "exit $?" >> gpurun_out/debug7.log
timeout 1500 python -m pytest tests -m "gpu and not slow" -q --timeout 120 -p no:cacheprovider > gpurun_out/pytest7.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest7.log
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench7_c2.log 2>&1
echo "exit $?" >> gpurun_out/bench7_c2.log
timeout 300 python bench.py --config 2 --steps 3 --warmup 3 --profile > gpurun_out/plain7_c2.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches7_c2.csv \
  python bench.py --config 2 --steps 3 --warmup 3 --profile > gpurun_out/ncu7_c2.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu7_c2.log
