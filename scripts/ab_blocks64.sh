for r in 1 2; do for B in 32 64 48; do
CMTF_TM_BLOCKS=$B python bench.py --no-cpu-baseline --no-e2e --no-naive --steps 4 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('B=$B', round(d['ms_per_step'],2), d['quality'])"
done; done
