cd $GRAFT_REPO_ROOT
SFG_ROWPTR_BULK=1 timeout 900 python -m pytest tests/test_gpu_convert.py -m "gpu and not slow" -q --timeout 120 -p no:cacheprovider -x > gpurun_out/pytest28.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest28.log
timeout 600 python bench.py --config 2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench28_c2.log 2>&1
for st in 2 3 4; do
SFG_ROWPTR_BULK=1 SFG_ROWPTR_STAGES=$st timeout 600 python bench.py --config 2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench28_c2_bulk$st.log 2>&1
done
