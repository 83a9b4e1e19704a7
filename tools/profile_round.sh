#!/bin/bash
# Round profile: bench (no profiler), C2 launch list, and ncu --set full captures
# of the top kernels (each command already ran clean without ncu).
set -x
mkdir -p gpurun_out/prof
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_c2.csv python tools/profile_step.py C2 > gpurun_out/prof/launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:beam_knn -s 2 -c 1 -o gpurun_out/prof/beam_c2 python tools/profile_step.py C2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:build_search -s 33 -c 1 -o gpurun_out/prof/bsearch_c2 python tools/profile_step.py C2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"prune_tc" -s 32 -c 2 -o gpurun_out/prof/ptc_c5 python tools/run_config.py C5 200000 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:beam_knn -c 1 -o gpurun_out/prof/beam_c5 python tools/run_config.py C5 200000 > /dev/null 2>&1
ls -la gpurun_out/prof
# text summaries on the box; only the summaries and the launch list come back
for r in gpurun_out/prof/*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  python tools/ncu_summary.py report $r > gpurun_out/prof/$b.summary.txt 2>&1
  python tools/ncu_lines.py $r 25 > gpurun_out/prof/$b.lines.txt 2>&1
  ncu -i $r --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/prof/$b.dram.csv 2>&1
done
python tools/launch_table.py gpurun_out/prof/launches_c2.csv > gpurun_out/prof/launch_table.txt 2>&1
rm -f gpurun_out/prof/*.ncu-rep
du -sh gpurun_out
