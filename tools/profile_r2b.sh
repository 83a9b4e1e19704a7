#!/bin/bash
# Round-2 (session 3) profile set, each command already ran clean without ncu:
#  * launch list of one C5 pipeline pass (gpu__time_duration, all launches)
#  * DRAM traffic of every walk launch of the pass -> profiles/ncu_traffic_c5.json
#  * ncu --set full of the C5 knn_all launch (row-ring beam_knn_kernel), the largest build search,
#    the largest prune_tc_build / prune_tc_reverse launches (fp16 Gram)
# Text summaries are written next to each report; the reports stay on the box.
set -x
D=gpurun_out/prof3; mkdir -p $D
C=$(cat gpurun_out/.commit 2>/dev/null || echo unknown)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_c5.csv python tools/profile_step.py C5 1 > $D/launch.log 2>&1
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"build_search_kernel|beam_knn_kernel" --csv --log-file $D/traffic_c5.csv python tools/profile_step.py C5 1 > $D/traffic.log 2>&1
python tools/ncu_traffic.py $D/traffic_c5.csv C5 "$1" > $D/traffic_json.log 2>&1; cp profiles/ncu_traffic_c5.json $D/
timeout 900 ncu --set full --clock-control none --import-source on -k regex:beam_knn -c 1 -o $D/beam_c5 python tools/profile_step.py C5 1 > $D/beam.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:build_search -s 19 -c 1 -o $D/bsearch_c5 python tools/profile_step.py C5 1 > $D/bsearch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prune_tc -s 57 -c 2 -o $D/ptc_c5 python tools/profile_step.py C5 1 > $D/ptc.log 2>&1
for r in $D/*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  python tools/ncu_summary.py report $r > $D/$b.summary.txt 2>&1
  python tools/ncu_lines.py $r 30 > $D/$b.lines.txt 2>&1
done
python tools/ncu_summary.py launches $D/launches_c5.csv > $D/launch_table_c5.txt 2>&1
rm -f $D/*.ncu-rep
ls -la $D
