cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider --durations=5 > gpurun_out/pytest32.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest32.log
timeout 600 python bench.py > gpurun_out/bench32_default.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench32_ref.log 2>&1
for c in 1 3 4; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench32_c$c.log 2>&1
done
for c in 2 1 3; do
timeout 300 python bench.py --config $c --steps 5 --warmup 3 --profile > gpurun_out/plain32_c$c.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches32_c$c.csv \
  python bench.py --config $c --steps 5 --warmup 3 --profile > gpurun_out/ncu32_c$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_row_scan|k_row_ptr|k_ell_fill|k_spmv_ell|k_split|k_spmv_coo" -s 12 -c 6 -o gpurun_out/prof32_c2 python bench.py --config 2 --steps 3 --warmup 3 --profile > gpurun_out/prof32_c2_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_coo_to_csr|k_spmv_csr" -s 4 -c 2 -o gpurun_out/prof32_c1 python bench.py --config 1 --steps 3 --warmup 3 --profile > gpurun_out/prof32_c1_ncu.log 2>&1
