cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x --timeout 120 -p no:cacheprovider > gpurun_out/pytest9.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest9.log
for c in 2 1 3; do
timeout 300 python bench.py --config $c --steps 5 --warmup 3 --profile > gpurun_out/plain9_c$c.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches9_c$c.csv \
  python bench.py --config $c --steps 5 --warmup 3 --profile > gpurun_out/ncu9_c$c.log 2>&1
done
timeout 600 python bench.py --config 2 --steps 20 --warmup 3 > gpurun_out/bench9_c2.log 2>&1
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench9_c4.log 2>&1
echo "c4 exit $?" >> gpurun_out/bench9_c4.log
