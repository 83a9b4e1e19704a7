"""Functional check of the multi-GPU split on one device: `world` ranks
sharing cuda:0 with host (gloo) collectives must reproduce the
single-process outputs bit for bit.  Not a measurement.

    python tools/check_shard.py [CONFIG] [N] [WORLD]
"""
import hashlib
import os
import socket
import sys
import time

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def digest(cfg, n, comm):
    import paper_2312_03940_b200 as pk
    from paper_2312_03940_b200 import workloads
    from paper_2312_03940_b200.cluster import run_pipeline_device

    torch.cuda.set_device(0)
    w = workloads.WORKLOADS[cfg]
    comps = max(1, int(round(w.components * n / w.n)))
    data, _ = workloads.generate(cfg, n=n, components=comps)
    kw = workloads.pipeline_args(cfg, pk, n_centers=min(w.n_centers, comps))
    trace = []
    t = time.time()
    out = run_pipeline_device(pk.PointSet(data), **kw, comm=comm, trace=trace)
    el = time.time() - t
    adj, deg = out["index"].graph.device_arrays()[:2]
    h = {}
    for name, x in (("adj", adj), ("deg", deg), ("ids", out["ids"]), ("dists", out["dists"]), ("rho", out["rho"]),
                    ("lam", out["lam"]), ("delta", out["delta"]), ("labels", out["labels"])):
        h[name] = hashlib.sha256(x.detach().cpu().numpy().tobytes()).hexdigest()[:16]
    return h, trace, el


def worker(rank, world, port, cfg, n, q):
    from paper_2312_03940_b200.shard import Comm

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        q.put((rank, digest(cfg, n, Comm())))
    except Exception:  # noqa: BLE001
        import traceback

        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
    world = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    ref, trace, el = digest(cfg, n, None)
    print("single:", ref, trace, f"{el:.2f}s")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=worker, args=(r, world, port, cfg, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    ok = True
    for _ in range(world):
        r, res = q.get(timeout=1200)
        if isinstance(res, str):
            print(f"rank {r} failed:\n{res}")
            ok = False
            continue
        h, tr, el = res
        same = {k: h[k] == ref[k] for k in ref}
        print(f"rank {r}:", same, tr, f"{el:.2f}s")
        ok &= all(same.values())
    for p in procs:
        p.join(timeout=60)
    print("IDENTICAL" if ok else "MISMATCH")
    sys.exit(0 if ok else 1)
