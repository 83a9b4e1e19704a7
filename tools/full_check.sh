# full GPU suite, smoke and a default bench run (one gpurun call)
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_all.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_rc=$?; tail -3 gpurun_out/bench_default.err
