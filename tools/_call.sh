tools/variant.sh Makefile 's/-Xptxas -v$/-Xptxas -v -DPK_PHASE_TIMERS/' python tools/phase_probe.py C5 > gpurun_out/c14_phase.log 2>&1; echo rc=$?; cat gpurun_out/c14_phase.log | tail -5
