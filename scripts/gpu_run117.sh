cd $GRAFT_REPO_ROOT
O=gpurun_out/r117
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
echo "exit $?" >> $O/smoke.log
for c in 2 1 3 4 5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > $O/bench_c$c.log 2>&1
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_c2.log 2>&1
timeout 600 python scripts/bench_ingest.py > $O/bench_ingest.log 2>&1
timeout 600 python scripts/bench_mm.py 1048576 16 > $O/bench_mm.log 2>&1
for c in 3; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches_c$c.csv python bench.py --config $c --steps 2 --warmup 3 --profile > $O/ncu_launch_c$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmm_rows_batch|k_blk_scatter|k_blk_sort|k_coo_to_dcsr" -s 8 -c 4 -o $O/full_c3 python bench.py --config 3 --steps 3 --warmup 3 --profile > $O/full_c3.log 2>&1
echo done > $O/done
