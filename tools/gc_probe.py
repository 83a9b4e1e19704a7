"""Run bench.py with a gc callback and report collections longer than 5 ms
(and whether they fell inside a timed region: bench.py prints step windows
when PK_BENCH_TRACE=1).

    python tools/gc_probe.py [bench args ...]
"""
import gc
import runpy
import sys
import time

sys.argv = ["bench.py"] + (sys.argv[1:] or ["--steps", "8", "--warmup", "3", "--no-cpu-baseline", "--no-tc-sample"])
ts = []


def cb(phase, info):
    if phase == "start":
        ts.append([time.perf_counter(), info["generation"]])
    else:
        ts[-1].append(time.perf_counter())


gc.callbacks.append(cb)
t0 = time.perf_counter()
runpy.run_path("/root/repo/bench.py", run_name="__main__")
big = [(round(t[0] - t0, 3), round((t[2] - t[0]) * 1e3, 2), t[1]) for t in ts if len(t) == 3 and t[2] - t[0] > 0.005]
print("gc pauses > 5 ms (start s, ms, generation):", big, "collections", len(ts), file=sys.stderr)
