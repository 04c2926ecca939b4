cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m "gpu and not slow" -q --timeout 120 -p no:cacheprovider > gpurun_out/pytest17.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest17.log
timeout 600 python bench.py --config 2 --steps 20 --warmup 3 > gpurun_out/bench17_c2.log 2>&1
timeout 600 python bench.py --config 1 --steps 20 --warmup 3 > gpurun_out/bench17_c1.log 2>&1
for c in 2 1; do
timeout 300 python bench.py --config $c --steps 5 --warmup 3 --profile > gpurun_out/plain17_c$c.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches17_c$c.csv \
  python bench.py --config $c --steps 5 --warmup 3 --profile > gpurun_out/ncu17_c$c.log 2>&1
done
timeout 1200 python -m pytest tests -m "gpu and slow" -q --timeout 900 -p no:cacheprovider --durations=10 > gpurun_out/pytest17_slow.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest17_slow.log
