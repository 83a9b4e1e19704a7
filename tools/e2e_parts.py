import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2312_03940_b200 as pk
from paper_2312_03940_b200 import workloads, cluster
data, _ = workloads.generate("C2")
kw = workloads.pipeline_args("C2", pk)
pinned = torch.from_numpy(np.array(data, dtype=np.float32, copy=True)).pin_memory()
hv = pinned.numpy()
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); p = pk.PointSet(hv)
    t1 = time.perf_counter(); p.device(); torch.cuda.synchronize()
    t2 = time.perf_counter(); _ = p.mode; p.packed(); torch.cuda.synchronize()
    t3 = time.perf_counter(); out = cluster.run_pipeline_device(p, **kw); torch.cuda.synchronize()
    t4 = time.perf_counter()
    r = cluster._to_host_many([out["rho"], out["lam"], out["delta"], out["ids"], out["dists"], out["labels"], cluster._ids_of_device(out["centers"]), cluster._ids_of_device(out["noise"])])
    t5 = time.perf_counter()
    print(f"pointset {1e3*(t1-t0):.2f} upload {1e3*(t2-t1):.2f} mode+pack {1e3*(t3-t2):.2f} pipeline {1e3*(t4-t3):.2f} d2h {1e3*(t5-t4):.2f}  stages {[round(v*1e3,2) for v in out['timings'].values()]}")

# pieces of the upload
import warnings
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); arr = np.ascontiguousarray(hv, dtype=np.float32)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        host = torch.from_numpy(arr)
    t1 = time.perf_counter(); dev = torch.empty((100000, 128), dtype=torch.float32, device="cuda"); torch.cuda.synchronize()
    t2 = time.perf_counter(); dev.copy_(host); torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"wrap {1e3*(t1-t0):.3f} alloc {1e3*(t2-t1):.3f} copy {1e3*(t3-t2):.3f}")
    del dev
