D=gpurun_out/spec; mkdir -p $D
for m in 0 2; do
PK_SPEC_ROWS=$m timeout 900 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section WarpStateStats --section Occupancy --clock-control none -k regex:beam_knn -c 1 -o $D/beam_s$m python tools/profile_step.py C5 1 > $D/beam_s$m.log 2>&1
ncu -i $D/beam_s$m.ncu-rep --page raw --csv > $D/beam_s$m.raw.csv 2>&1
done
rm -f $D/*.ncu-rep
