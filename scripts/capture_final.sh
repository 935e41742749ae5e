#!/bin/bash
# Round-end captures on the GPU box: launch list of the default bench command,
# ncu --set full of the epoch kernel for configs 5 (@1e9), 3 and 2; the
# reports are summarised here (they exceed what gpurun copies back) into
# gpurun_out/final/.
mkdir -p gpurun_out/final
O=gpurun_out/final
K="regex:hog3|hog4|eval|nonfinite|row_norms|accum_delta|build_rrec|check_entries|delta_kernel|dup_|gather_|hot_|iota_u32|merge_matrix|mode_key|mrec_hot|pack_|part_|pos_from|rebase|reg_kernel|remap_pos|reshuffle|rrec_ids|scatter_affine|DeviceRadix|DeviceSelect|DeviceScan|DeviceCompact|serial_epoch|generic|matrix_sweep"
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 800 --csv \
    --log-file $O/launches_r2_config5_1e9.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo launch_rc=$?
cp profiles/ncu_r2_metrics.json $O/ncu_r2_metrics.json
for cfg in "c5_1e9:config5 nnz 1e+09 rank 10:" "c3:config3 scale 1:--config config3" "c2:config2:--config config2"; do
  tag=${cfg%%:*}; rest=${cfg#*:}; key=${rest%%:*}; a=${rest#*:}
  rep=/tmp/ncu_r2_${tag}_final.ncu-rep
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:hog3tm -s 3 -c 1 -o ${rep%.ncu-rep} -f \
      python bench.py $a --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-naive > $O/ncu_${tag}.log 2>&1
  echo ${tag}_rc=$?
  python scripts/ncu_summary.py $rep > $O/ncu_r2_${tag}_final_summary.txt 2>&1
  python scripts/ncu_src_lines.py $rep 40 > $O/ncu_r2_${tag}_final_lines.txt 2>&1
  python scripts/ncu_stall_lines.py $rep stall_long_sb 15 >> $O/ncu_r2_${tag}_final_lines.txt 2>&1
  python scripts/ncu_metrics_json.py $rep "hog3tm_kernel<10> ${key} (round 2, final)" $O/ncu_r2_metrics.json >> $O/ncu_${tag}.log 2>&1
done
ls -la $O
