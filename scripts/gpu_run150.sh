cd $GRAFT_REPO_ROOT
O=gpurun_out/r150
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
echo "exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.log 2>&1
timeout 900 python bench.py --config 3 --steps 20 --warmup 5 > $O/bench_c3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches_c3.csv python bench.py --config 3 --steps 2 --warmup 3 --profile > $O/ncu_launch_c3.log 2>&1
echo done > $O/done
