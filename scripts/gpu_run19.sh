cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_spmv.py -m "gpu and not slow" -q --timeout 120 -p no:cacheprovider > gpurun_out/pytest19.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest19.log
for v in 0 1 2 3 4; do
SFG_COO_PIPE=$v timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench19_c2_p$v.log 2>&1
done
SFG_COO_V1=1 timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench19_c2_v1.log 2>&1
