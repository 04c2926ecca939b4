cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_spmm.py -m "gpu" -q --timeout 300 -p no:cacheprovider -x > gpurun_out/pytest103.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest103.log
for v in 0 1 2; do
SFG_SPMM_VAR=$v timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench103_c5_v$v.log 2>&1
done
echo done
