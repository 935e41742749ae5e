#!/bin/bash
# A/B of environment settings on bench.py device epochs:
#   scripts/ab_env.sh "<bench args>" "ENV1=a" "ENV1=b" ...
args="$1"; shift
for e in "$@"; do
  line=$(env $e python bench.py $args --no-cpu-baseline --no-e2e --no-naive 2>&1 | tail -1)
  python - "$e" "$line" <<'PY'
import json, sys
try:
    d = json.loads(sys.argv[2])
    print(f"{sys.argv[1]:24s} ms/step {d['ms_per_step']:.3f}  value {d['value']:.4g}  frac {d['roofline']['frac']:.3f}  rmse {d['quality']['train_rmse']:.5f}")
except Exception:
    print(sys.argv[1], "FAILED", sys.argv[2][-400:])
PY
done
