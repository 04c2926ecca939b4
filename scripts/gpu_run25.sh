cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --config 2 --steps 3 --warmup 3 --profile > gpurun_out/plain25_c2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_row_scan|k_row_ptr" -s 4 -c 2 -o gpurun_out/prof25_c2 python bench.py --config 2 --steps 3 --warmup 3 --profile > gpurun_out/prof25_c2_ncu.log 2>&1
