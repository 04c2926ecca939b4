cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest133.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest133.log
timeout 300 python scripts/bench_ingest.py > gpurun_out/bench_ingest133.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches133_ingest.csv python scripts/bench_ingest.py > /dev/null 2>&1
echo done
