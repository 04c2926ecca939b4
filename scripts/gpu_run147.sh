cd $GRAFT_REPO_ROOT
O=gpurun_out/r147
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
echo "exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.log 2>&1
echo done > $O/done
