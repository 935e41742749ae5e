# Hot-row damping constant sweep: order-4 small vs oracle, config 2 (0.1 and
# full) vs the reference's runs, DSGD emulated G = 2, 4, 8.
K=${1:-'0.5 0.25 1.0'}
for k in $K; do
  echo "== kappa $k"
  python scripts/order4_check.py "[{\"kappa\":$k}]" 2>&1 | tail -1
  python scripts/c2_sweep.py 0.1 "[{\"kappa\":$k}]" 2>&1 | tail -1
  python scripts/c2_sweep.py 1.0 "[{\"kappa\":$k}]" 2>&1 | tail -1
  python scripts/dsgd_emulated.py c0.1 2,4,8 $k 2>&1 | tail -3
done
