cd $GRAFT_REPO_ROOT
for v in 0 1 2 3 4 5; do
echo "variant $v" >> gpurun_out/csr31.log
SFG_CSR_VAR=$v timeout 600 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['kernels']['spmv'])" >> gpurun_out/csr31.log 2>&1
SFG_CSR_VAR=$v timeout 600 python -m pytest tests/test_gpu_spmv.py -m "gpu and not slow" -q --timeout 120 -p no:cacheprovider -x -k "csr or CSR" 2>&1 | tail -1 >> gpurun_out/csr31.log
done
