# Interleaved A/B of environment settings on bench workloads (same library):
#   bash scripts/ab_env_cfg.sh "CMTF_TM_GATHER_CA=0" "CMTF_TM_GATHER_CA=1" 2 "--config config5 --nnz 1e9" ...
A=$1; B=$2; R=${3:-2}; shift 3
[ $# -eq 0 ] && set -- "--config config5 --nnz 1e9"
for c in "$@"; do
  echo "== $c"
  for r in $(seq $R); do
    for S in "$A" "$B"; do
      env $S python bench.py $c --no-cpu-baseline --no-e2e --no-naive --steps 5 --warmup 3 2>/dev/null \
        | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$S', round(d['ms_per_step'],3), d['quality'])"
    done
  done
done
