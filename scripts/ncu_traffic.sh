#!/bin/bash
# DRAM traffic / L2 hit rate of the epoch kernel under environment settings:
#   scripts/ncu_traffic.sh "<bench args>" "ENV=a" "ENV=b" ...
args="$1"; shift
for e in "$@"; do
  echo "== $e"
  env $e ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
    --clock-control none -k regex:hog3tm -s 3 -c 1 python bench.py $args --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-naive 2>&1 \
    | grep -E "dram__bytes|hit_rate|gpu__time" 
done
