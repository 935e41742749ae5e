#!/bin/bash
# ncu --set full of the order-4 tcgen05 epoch kernel on config 4 (full size), summarised on the box
mkdir -p gpurun_out/final
O=gpurun_out/final
rep=/tmp/ncu_r2_c4_hog4tm.ncu-rep
cp profiles/ncu_r2_metrics.json $O/ncu_r2_metrics.json
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:hog4tm -s 3 -c 1 -o ${rep%.ncu-rep} -f \
    python bench.py --config config4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-naive > $O/ncu_c4.log 2>&1
echo c4_rc=$?
python scripts/ncu_summary.py $rep > $O/ncu_r2_c4_hog4tm_summary.txt 2>&1
python scripts/ncu_src_lines.py $rep 40 > $O/ncu_r2_c4_hog4tm_lines.txt 2>&1
python scripts/ncu_stall_lines.py $rep stall_long_sb 12 >> $O/ncu_r2_c4_hog4tm_lines.txt 2>&1
python scripts/ncu_stall_lines.py $rep stall_barrier 8 >> $O/ncu_r2_c4_hog4tm_lines.txt 2>&1
python scripts/ncu_metrics_json.py $rep "hog4tm_kernel config4 scale 1 (round 2, final)" $O/ncu_r2_metrics.json >> $O/ncu_c4.log 2>&1
python bench.py --config config4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c4.log 2>&1; tail -1 $O/bench_c4.log | cut -c1-400
