timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; grep -E "^E  |passed|failed|^FAILED|Error" gpurun_out/pytest_gpu.log | head -20
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$?; tail -2 gpurun_out/bench.err
python - <<'PY'
import json; d=json.load(open("gpurun_out/bench.json")); print(round(d["value"]), round(d["ms_per_step"],2), round(d["e2e"]["value"]), d["dtype"]); print({k: round(v,2) for k,v in d["stage_ms"].items()}); print(list(d["kernels_ms_per_step"].items())[:6]); print(d["counters_per_step"]); r=d["roofline"]; print(r["kernel"], r["achieved"], r["frac"])
PY
