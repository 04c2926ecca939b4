cd $GRAFT_REPO_ROOT
O=gpurun_out/r120
mkdir -p $O
timeout 900 python bench.py --config 2 --steps 20 --warmup 5 > $O/bench_c2.log 2>&1
timeout 900 python bench.py > $O/bench_default.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv python bench.py --config 2 --steps 2 --warmup 3 --profile > $O/ncu_launch_c2.log 2>&1
for t in 4 16 32; do timeout 900 python bench.py --threshold $t --no-cpu-baseline --no-e2e > $O/bench_t$t.log 2>&1; done
echo done > $O/done
