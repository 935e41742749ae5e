# Interleaved speed A/B of library builds on the large bench workloads:
#   bash scripts/ab_cfg.sh "libA.so libB.so" [rounds] ["--config config5 --nnz 1e9" "--config config3" ...]
LIBS=$1; R=${2:-2}; shift 2
[ $# -eq 0 ] && set -- "--config config5 --nnz 1e9" "--config config3" "--config config2"
for c in "$@"; do
  echo "== $c"
  for r in $(seq $R); do
    for L in $LIBS; do
      CMTF_B200_LIB=$PWD/paper_1708_08640_b200/$L python bench.py $c --no-cpu-baseline --no-e2e --no-naive --steps 5 --warmup 3 2>/dev/null \
        | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$L', round(d['ms_per_step'],3), round(d['breakdown_ms']['tensor'],3), d['quality'])"
    done
  done
done
