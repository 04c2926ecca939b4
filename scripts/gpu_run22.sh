cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --config 2 --steps 3 --warmup 3 --profile > gpurun_out/plain22_c2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_row_scan|k_row_ptr|k_ell_fill|k_spmv_ell|k_split|k_spmv_coo" -s 12 -c 6 -o gpurun_out/prof22_c2 python bench.py --config 2 --steps 3 --warmup 3 --profile > gpurun_out/prof22_c2_ncu.log 2>&1
timeout 300 python bench.py --config 1 --steps 3 --warmup 3 --profile > gpurun_out/plain22_c1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_coo_to_csr|k_spmv_csr" -s 4 -c 2 -o gpurun_out/prof22_c1 python bench.py --config 1 --steps 3 --warmup 3 --profile > gpurun_out/prof22_c1_ncu.log 2>&1
