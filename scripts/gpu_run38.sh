cd $GRAFT_REPO_ROOT
for v in 9 3; do
echo "variant $v" >> gpurun_out/bench38.log
SFG_BCSR_TC_VAR=$v timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])" >> gpurun_out/bench38.log
done
