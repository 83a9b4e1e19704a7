timeout 1500 python tools/check_full_sampled.py C5 brute > gpurun_out/c12_full_c5.log 2>&1; echo c5_rc=$?; cat gpurun_out/c12_full_c5.log
timeout 1200 python tools/check_full_sampled.py C4 > gpurun_out/c12_full_c4.log 2>&1; echo c4_rc=$?; cat gpurun_out/c12_full_c4.log
