cd $GRAFT_REPO_ROOT
O=gpurun_out/r107
mkdir -p $O
for c in 3 5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > $O/bench_c$c.log 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches_c$c.csv python bench.py --config $c --steps 2 --warmup 3 --profile --no-e2e > $O/ncu_launch_c$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmm_rows_batch|k_csc_scatter|k_csc_fix|k_coo_to_dcsr" -s 8 -c 4 -o $O/full_c3 python bench.py --config 3 --steps 3 --warmup 3 --profile --no-e2e > $O/full_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmm_merge|k_coo_to_csr" -s 4 -c 2 -o $O/full_c5 python bench.py --config 5 --steps 2 --warmup 3 --profile --no-e2e > $O/full_c5.log 2>&1
echo done > $O/done
