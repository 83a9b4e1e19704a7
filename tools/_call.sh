set -x
for loc in 0 1; do PK_LOCALITY=$loc timeout 600 python tools/run_config.py C5 > gpurun_out/c5_c5_loc$loc.log 2>&1; tail -3 gpurun_out/c5_c5_loc$loc.log; done
for loc in 0 1; do PK_LOCALITY=$loc timeout 600 python tools/run_config.py C4 > gpurun_out/c5_c4_loc$loc.log 2>&1; tail -3 gpurun_out/c5_c4_loc$loc.log; done
timeout 1200 python -m pytest tests/test_parity_scale_gpu.py -q -m gpu -k "config_shaped" > gpurun_out/c5_scale.log 2>&1; echo scale_rc=$?; tail -3 gpurun_out/c5_scale.log
timeout 900 python -m pytest tests/ -q -m gpu -x --ignore=tests/test_parity_scale_gpu.py > gpurun_out/c5_gpu.log 2>&1; echo gpu_rc=$?; tail -3 gpurun_out/c5_gpu.log
