cd $GRAFT_REPO_ROOT
timeout 1200 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/bench61_c5.log 2>&1
echo "exit $?" >> gpurun_out/bench61_c5.log
