#!/bin/bash
# ncu launch lists (time + DRAM bytes per kernel) of configs 1-4, for
# profiles/r02_launches_config<N>.csv and profiles/traffic_config<N>.json
for c in 1 2 3 4; do
  python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r02_launches_config$c.csv 2>&1
done
