cd $GRAFT_REPO_ROOT
true
echo "pytest exit $?" >> gpurun_out/pytest94.log
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/bench94_c5.log 2>&1
echo done
