#!/bin/bash
# Round-2 profile set (each command already ran clean without ncu):
#  * launch list of one C5 bench step (gpu__time_duration, all launches)
#  * ncu --set full of the CTA-pair tcgen05 screen over the full C5 exact kNN pass
#  * ncu --set full of the C5 knn_all beam-walk launch and the largest C5 build search
#  * ncu --set full of the largest C5 prune_tc_build / prune_tc_reverse launches
# Text summaries are written next to each report; the reports stay on the box.
set -x
D=gpurun_out/prof2; mkdir -p $D
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_c5.csv python tools/profile_step.py C5 1 > $D/launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tc_screen_kernel -c 1 -o $D/tcscreen_c5 python tools/run_config.py C5 - brute > $D/tc.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:beam_knn -c 1 -o $D/beam_c5 python tools/profile_step.py C5 1 > $D/beam.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:build_search -s 19 -c 1 -o $D/bsearch_c5 python tools/profile_step.py C5 1 > $D/bsearch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prune_tc -s 38 -c 2 -o $D/ptc_c5 python tools/profile_step.py C5 1 > $D/ptc.log 2>&1
for r in $D/*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  python tools/ncu_summary.py report $r > $D/$b.summary.txt 2>&1
  python tools/ncu_lines.py $r 30 > $D/$b.lines.txt 2>&1
done
python tools/ncu_summary.py launches $D/launches_c5.csv > $D/launch_table_c5.txt 2>&1
rm -f $D/*.ncu-rep
ls -la $D
