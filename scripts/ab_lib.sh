# A/B of two builds of the library on the parity workloads (kappa default):
# order-4 small vs oracle, config 2 (0.1, full) vs the reference, DSGD G=2,4,8.
for L in "$@"; do
  echo "== $L"
  export CMTF_B200_LIB=$PWD/paper_1708_08640_b200/$L
  python scripts/order4_check.py '[{"kernel":"opt"},{"kernel":"naive"}]' 2>&1 | tail -2
  python scripts/c2_sweep.py 0.1 '[{}]' 2>&1 | tail -1
  python scripts/c2_sweep.py 1.0 '[{}]' 2>&1 | tail -1
  python scripts/dsgd_emulated.py c0.1 2,4,8 2>&1 | tail -3
done
