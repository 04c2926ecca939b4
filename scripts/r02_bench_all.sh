#!/bin/bash
# The default bench line plus every BASELINE config (same contract), and the
# reference arm of the default config; outputs -> gpurun_out/r02_bench_*.json
python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err
for c in 1 2 3 4; do
  python bench.py --config $c > gpurun_out/r02_bench_config$c.json 2> gpurun_out/r02_bench_config$c.err
done
for v in "16 f32" "4 bf16" "4 f32"; do
  set -- $v
  python bench.py --config 4 --block $1 --bcsr-dtype $2 --no-e2e --no-cpu-baseline \
    > gpurun_out/r02_bench_config4_$1_$2.json 2> gpurun_out/r02_bench_config4_$1_$2.err
done
python bench.py --impl reference > gpurun_out/r02_bench_reference_config5.json 2> gpurun_out/r02_bench_reference.err
for f in gpurun_out/r02_bench_default.json gpurun_out/r02_bench_config?.json gpurun_out/r02_bench_config4_*.json gpurun_out/r02_bench_reference_config5.json; do
  python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', d.get('ms_per_step'), d.get('value'), d.get('unit'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'), d.get('clocks',{}).get('sm_mhz'))
"
done
