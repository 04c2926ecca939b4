cd $GRAFT_REPO_ROOT
O=gpurun_out/r96
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
echo "exit $?" >> $O/smoke.log
for c in 2 1 3 4 5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > $O/bench_c$c.log 2>&1
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_c2.log 2>&1
for c in 1 3 4 5; do timeout 900 python bench.py --impl reference --config $c --steps 3 --warmup 3 > $O/bench_ref_c$c.log 2>&1; done
for c in 1 2 3 4 5; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches_c$c.csv python bench.py --config $c --steps 2 --warmup 3 --profile --no-e2e > $O/ncu_launch_c$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_row_scan|k_row_ptr|k_ell_fill|k_spmv_ell|k_split|k_spmv_coo" -s 12 -c 6 -o $O/full_c2 python bench.py --config 2 --steps 3 --warmup 3 --profile --no-e2e > $O/full_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_coo_to_csr|k_spmv_csr" -s 4 -c 2 -o $O/full_c1 python bench.py --config 1 --steps 3 --warmup 3 --profile --no-e2e > $O/full_c1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmm_rows_batch|k_csc_scatter|k_coo_to_dcsr" -s 6 -c 3 -o $O/full_c3 python bench.py --config 3 --steps 3 --warmup 3 --profile --no-e2e > $O/full_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmm_merge|k_coo_to_csr" -s 4 -c 2 -o $O/full_c5 python bench.py --config 5 --steps 2 --warmup 3 --profile --no-e2e > $O/full_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bcsr_tc_panel" -s 2 -c 1 -o $O/full_c4 python bench.py --config 4 --steps 2 --warmup 3 --profile --no-e2e > $O/full_c4.log 2>&1
echo done > $O/done
