#!/bin/bash
# ncu --set full of the epoch kernel at the round's final library, config 5 @1e9
mkdir -p gpurun_out/final5
O=gpurun_out/final5
cp profiles/ncu_r2_metrics.json $O/ncu_r2_metrics.json
rep=/tmp/ncu_r2_c5_1e9_final2.ncu-rep
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:hog3tm -s 3 -c 1 -o ${rep%.ncu-rep} -f \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-naive > $O/ncu_c5.log 2>&1
echo rc=$?
python scripts/ncu_summary.py $rep > $O/ncu_r2_c5_1e9_final2_summary.txt 2>&1
python scripts/ncu_src_lines.py $rep 40 > $O/ncu_r2_c5_1e9_final2_lines.txt 2>&1
python scripts/ncu_metrics_json.py $rep "hog3tm_kernel<10> config5 nnz 1e+09 rank 10 (round 2, final2: gathers through L1)" $O/ncu_r2_metrics.json >> $O/ncu_c5.log 2>&1
ls -la $O
