#!/bin/bash
# ncu --set full of the tcgen05 BCSR kernels at config 4 (one launch each,
# after the same command has run clean without ncu); summaries -> profiles/
set -e
for v in "16 bf16 k_bcsr_tc_panel" "16 f32 k_bcsr_tc_panel" "4 bf16 k_bcsr4_tc"; do
  set -- $v
  python bench.py --config 4 --block $1 --bcsr-dtype $2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 -o gpurun_out/r02_c4_$1_$2 \
    python bench.py --config 4 --block $1 --bcsr-dtype $2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
    > gpurun_out/r02_c4_$1_$2.ncu.log 2>&1
done
