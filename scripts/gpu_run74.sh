cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench74_c3.log 2>&1
timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --profile > gpurun_out/plain74.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches74_c3.csv python bench.py --config 3 --steps 5 --warmup 3 --profile > gpurun_out/ncu74.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmm_rows" -s 3 -c 1 -o gpurun_out/prof74_c3 python bench.py --config 3 --steps 3 --warmup 3 --profile > gpurun_out/prof74_ncu.log 2>&1
