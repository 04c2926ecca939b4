cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_convert.py tests/test_gpu_convert_src.py -m "gpu" -q --timeout 120 -p no:cacheprovider -x > gpurun_out/pytest86.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest86.log
timeout 300 python scripts/bench_ingest.py > gpurun_out/bench_ingest86.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches86_ingest.csv python scripts/bench_ingest.py > /dev/null 2>&1
echo done
