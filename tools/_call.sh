nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/gather_probe tools/gather_probe.cu && /tmp/gather_probe > gpurun_out/c13_gather.log 2>&1; cat gpurun_out/c13_gather.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/c13_bench.json 2> gpurun_out/c13_bench.err; echo bench_rc=$?; tail -3 gpurun_out/c13_bench.err
