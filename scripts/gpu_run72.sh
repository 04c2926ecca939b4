cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider --durations=5 > gpurun_out/pytest72.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest72.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke72.log 2>&1
echo "exit $?" >> gpurun_out/smoke72.log
