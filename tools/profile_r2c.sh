#!/bin/bash
# Round-2 final profile set (each command already ran clean without ncu):
#  * launch list of one C5 pipeline pass (gpu__time_duration, all launches)
#  * DRAM traffic of every walk launch of the pass -> profiles/ncu_traffic_c5.json
#  * the C5 knn_all launch of beam_knn_kernel: the summary's counters + source-level stall samples
#    (a --set full replay of this 1.2 s launch does not finish in 15 minutes)
#  * ncu --set full of the largest build search and the largest prune_tc_build / prune_tc_reverse launches
# Text summaries are written next to each report; the reports stay on the box.
set -x
D=gpurun_out/prof4; mkdir -p $D
KEYS=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.per_cycle_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,launch__registers_per_thread,launch__grid_size,launch__block_size,launch__occupancy_limit_shared_mem,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,dram__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__t_sector_hit_rate.pct
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_c5.csv python tools/profile_step.py C5 1 > $D/launch.log 2>&1
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"build_search_kernel|beam_knn_kernel" --csv --log-file $D/traffic_c5.csv python tools/profile_step.py C5 1 > $D/traffic.log 2>&1
python tools/ncu_traffic.py $D/traffic_c5.csv C5 "$1" > $D/traffic_json.log 2>&1; cp profiles/ncu_traffic_c5.json $D/
timeout 1500 ncu --metrics $KEYS --section SourceCounters --clock-control none --import-source on -k regex:beam_knn -c 1 -o $D/beam_c5 python tools/profile_step.py C5 1 > $D/beam.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:build_search -s 19 -c 1 -o $D/bsearch_c5 python tools/profile_step.py C5 1 > $D/bsearch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prune_tc_build -s 19 -c 1 -o $D/ptcb_c5 python tools/profile_step.py C5 1 > $D/ptcb.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prune_tc_reverse -s 38 -c 1 -o $D/ptcr_c5 python tools/profile_step.py C5 1 > $D/ptcr.log 2>&1
for r in $D/*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  python tools/ncu_summary.py report $r > $D/$b.summary.txt 2>&1
  python tools/ncu_lines.py $r 30 > $D/$b.lines.txt 2>&1
done
python tools/ncu_summary.py launches $D/launches_c5.csv > $D/launch_table_c5.txt 2>&1
rm -f $D/*.ncu-rep
ls -la $D
