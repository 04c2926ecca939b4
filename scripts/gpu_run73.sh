cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_convert.py -m "gpu and not slow" -q --timeout 120 -p no:cacheprovider -x > gpurun_out/pytest73.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest73.log
timeout 600 python bench.py --config 2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench73_c2.log 2>&1
timeout 600 python bench.py --config 1 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench73_c1.log 2>&1
timeout 300 python bench.py --config 2 --steps 5 --warmup 3 --profile > gpurun_out/plain73.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches73_c2.csv python bench.py --config 2 --steps 5 --warmup 3 --profile > gpurun_out/ncu73.log 2>&1
