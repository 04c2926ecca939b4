cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest2.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest2.log
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 > gpurun_out/bench_c2.log 2>&1
echo "exit $?" >> gpurun_out/bench_c2.log
timeout 300 python bench.py --config 2 --steps 3 --warmup 3 --profile > gpurun_out/plain_c2.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
  python bench.py --config 2 --steps 3 --warmup 3 --profile > gpurun_out/ncu_c2.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_c2.log
