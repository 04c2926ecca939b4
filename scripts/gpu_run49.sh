cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m "gpu" -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest49.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest49.log
timeout 300 python scripts/prof_bcsr.py 65536 > gpurun_out/prof49.log 2>&1
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 > gpurun_out/bench49_c4.log 2>&1
