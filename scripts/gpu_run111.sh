cd $GRAFT_REPO_ROOT
O=gpurun_out/r111
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
echo "exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.log 2>&1
echo "exit $?" >> $O/bench_default.log
timeout 900 python bench.py --impl reference > $O/bench_ref_default.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 1 --steps 5 --warmup 3 --rowpart --no-cpu-baseline > $O/bench_rowpart.log 2>&1
echo "exit $?" >> $O/bench_rowpart.log
for t in 4 16 32; do timeout 900 python bench.py --threshold $t --no-cpu-baseline --no-e2e > $O/bench_t$t.log 2>&1; done
echo done > $O/done
