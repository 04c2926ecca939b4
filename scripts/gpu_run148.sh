cd $GRAFT_REPO_ROOT
for i in 1 2 3; do timeout 900 python bench.py > gpurun_out/bench148_$i.log 2>&1; done
echo done
