cd $GRAFT_REPO_ROOT
for f in 4 8 0; do
echo "flat $f" >> gpurun_out/bench76.log
SFG_SPMM_FLAT=$f timeout 900 python -m pytest tests/test_gpu_spmm.py -m "gpu" -q --timeout 120 -p no:cacheprovider -x 2>&1 | tail -1 >> gpurun_out/bench76.log
SFG_SPMM_FLAT=$f timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['kernels']['spmm'])" >> gpurun_out/bench76.log
done
