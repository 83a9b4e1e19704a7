#!/bin/bash
# ncu --set full captures of the float-build seed pre-screen (tc_screen_kernel in
# dump mode + seed_mask_kernel) and the short-row count decision (tc_screen_kernel
# in counting mode) on a 200k-point C5 sample; the bench line first, without ncu.
set -x
mkdir -p gpurun_out/prof2
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/prof2/bench.json 2> gpurun_out/prof2/bench.err
timeout 600 python tools/run_config.py C5 200000 > gpurun_out/prof2/c5s.log 2>&1
PK_TC_COUNT_MIN=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"tc_screen_kernel|seed_mask_kernel" -c 6 -o gpurun_out/prof2/tcx_c5 \
  python tools/run_config.py C5 200000 > gpurun_out/prof2/ncu.log 2>&1
for r in gpurun_out/prof2/*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  python tools/ncu_summary.py report $r > gpurun_out/prof2/$b.summary.txt 2>&1
  ncu -i $r --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size > gpurun_out/prof2/$b.dram.csv 2>&1
done
rm -f gpurun_out/prof2/*.ncu-rep
du -sh gpurun_out
