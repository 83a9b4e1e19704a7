import gc, sys, time, runpy
sys.argv = ["bench.py", "--steps", "8", "--warmup", "3", "--no-cpu-baseline", "--no-tc-sample"]
ts = []
def cb(phase, info):
    if phase == "start":
        ts.append([time.perf_counter(), info["generation"]])
    else:
        ts[-1].append(time.perf_counter())
gc.callbacks.append(cb)
runpy.run_path("/root/repo/bench.py", run_name="__main__")
big = [(round((t[2]-t[0])*1e3,2), t[1]) for t in ts if len(t) == 3 and t[2]-t[0] > 0.005]
print("gc pauses > 5ms:", big, "total collections", len(ts), file=sys.stderr)
