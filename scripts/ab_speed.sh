# Speed A/B of library builds on the bench workload (config 2), interleaved:
#   bash scripts/ab_speed.sh libA.so libB.so [rounds]
R=${3:-3}
for r in $(seq $R); do
  for L in "$1" "$2"; do
    CMTF_B200_LIB=$PWD/paper_1708_08640_b200/$L python bench.py --no-cpu-baseline --no-e2e --steps 10 \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['ms_per_step'],4), round(d['breakdown_ms']['tensor'],4))"
  done
done
