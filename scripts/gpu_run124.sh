cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest124.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest124.log
for i in 1 2; do timeout 600 python bench.py --config 3 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench124_c3_$i.log 2>&1; done
echo done
