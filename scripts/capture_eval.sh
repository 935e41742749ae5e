#!/bin/bash
# ncu --set full of the tcgen05 evaluation kernels (config 5 @1e9, config 4)
# and the launch list of the default bench command at the round's final
# library; summaries into gpurun_out/final2/.
mkdir -p gpurun_out/final2
O=gpurun_out/final2
for cfg in "c5_1e9:eval3tm:config5 1e9" "c4:eval4tm:config4"; do
  tag=${cfg%%:*}; rest=${cfg#*:}; k=${rest%%:*}; a=${rest#*:}
  rep=/tmp/ncu_r2_${tag}_${k}.ncu-rep
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o ${rep%.ncu-rep} -f \
      python scripts/stats_ab.py $a > $O/ncu_${tag}_${k}.log 2>&1
  echo ${tag}_rc=$?
  python scripts/ncu_summary.py $rep > $O/ncu_r2_${tag}_${k}_summary.txt 2>&1
  python scripts/ncu_src_lines.py $rep 25 > $O/ncu_r2_${tag}_${k}_lines.txt 2>&1
done
K="regex:hog3|hog4|eval|pairwise|nonfinite|row_norms|accum_delta|build_rrec|check_entries|delta_kernel|dup_|gather_|hot_|iota_u32|merge_matrix|mode_key|mrec_hot|pack_|part_|pos_from|rebase|reg_kernel|remap_pos|reshuffle|rrec_ids|scatter_affine|DeviceRadix|DeviceSelect|DeviceScan|DeviceCompact|serial_epoch|generic|matrix_sweep"
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 800 --csv \
    --log-file $O/launches_r2_final_config5_1e9.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo launch_rc=$?
python scripts/launch_summary.py $O/launches_r2_final_config5_1e9.csv > $O/launches_r2_final_config5_1e9_summary.txt 2>&1
ls -la $O
