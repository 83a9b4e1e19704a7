#!/usr/bin/env python
"""Benchmark: end-to-end ANN density-peaks clustering (points/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C2] [--n N_POINTS] [--no-cpu-baseline]

A step is one full pass of the hot path over the configuration's synthetic
point set (BASELINE.json configs[1] = C2 by default: n=100,000 d=128
SIFT-shaped, Vamana R=64 L=128 alpha=1.1, kth_normalized k=16, doubling from
2k, 100 product centers): graph build, kNN densities, dependent points,
policies + union-find labels, all on the GPU.  `value` = points/s with the
points already resident in HBM; L2 is flushed (a 256 MiB write) before every
timed step because C2 (51 MB) fits in the 126 MB L2.  `e2e` = the same
through the public API (`run_pipeline(PointSet(host array))`) with the
host->device upload of the points and the device->host read of every result
array inside the timed region.

Multi-GPU (torchrun, one rank per GPU, NCCL): the same n points are split
across the ranks (shard.py: build batches, kNN queries, dependent-point
queries; out-lists / rows / kNN rows all-gathered, lam / delta all-reduced),
so the total work is fixed ("scaling": "strong"); value = n / (max over ranks
of the step time).

--impl reference times the reference algorithm's CPU implementation on the
host cores: the oracle/ C restatement of the reference's numba kernels
(OpenMP over all host threads) driving the same pipeline; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "points/sec end-to-end ANN-DPC at 1/2/4/8 B200; dep-point queries/s; % roofline"
TIMED_KERNELS = ("build_search_kernel", "beam_knn_kernel", "build_prune_block_kernel", "reverse_block_kernel",
                 "reverse_big_kernel", "build_prune_kernel", "reverse_kernel", "scan_denser_kernel")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tc-sample", action="store_true")
    ap.add_argument("--no-hbm-sample", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        pk = json.load(open(path))
        return pk["hbm_gbs"], pk["bf16_tflops"], "measured"
    return 6650.0, 1590.0, "fallback"


# ---------------------------------------------------------------------------- clocks


class ClockSampler:
    """SM clocks / clock-event (throttle) reasons sampled during the timed region
    through NVML in a background thread (25 ms period).  NVML reads are cheap;
    an nvidia-smi process in loop mode takes driver locks that stalled a timed
    step.  Falls back to nvidia-smi when NVML is unavailable."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []  # (host time, sm MHz, max MHz, reason bits)
        self.thread = None
        self.proc = None
        self.stop_flag = threading.Event()
        self.source = None

    def _nvml_handle(self):
        import pynvml
        import torch

        pynvml.nvmlInit()
        try:
            pr = torch.cuda.get_device_properties(self.gpu)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.gpu)

    def start(self):
        if os.environ.get("PK_BENCH_NO_SMI") == "1":  # diagnosis only
            return
        try:
            nv, h = self._nvml_handle()
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.source = "nvml"

            def loop():
                while not self.stop_flag.is_set():
                    try:
                        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                        rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((time.perf_counter(), float(sm), float(mx), int(rs)))
                    except Exception:
                        pass
                    self.stop_flag.wait(0.025)

            self.thread = threading.Thread(target=loop, daemon=True)
            self.thread.start()
            return
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.source = "nvidia-smi"
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read_smi, daemon=True)
        self.thread.start()

    def _read_smi(self):
        names = list(self.REASONS)
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.strip().split(",")]
            if len(parts) < 9:
                continue
            try:
                bits = sum(self.REASONS[nm] for nm, v in zip(names, parts[5:9]) if v.lower() == "active")
                self.samples.append((time.perf_counter(), float(parts[1]), float(parts[2]), bits))
            except ValueError:
                continue

    def wait_first(self, n=2, timeout=3.0):
        """Block until the sampler has produced n samples."""
        t = time.perf_counter()
        while self.thread is not None and len(self.samples) < n and time.perf_counter() - t < timeout:
            time.sleep(0.01)

    def mark(self, t0, t1):
        """The timed region's host-time window (samples inside it are used)."""
        self.window = (t0, t1)

    def stop(self):
        if self.thread is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        self.stop_flag.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        self.thread.join(timeout=2)
        samples = self.samples
        w = getattr(self, "window", None)
        if w is not None:
            inside = [x for x in samples if w[0] <= x[0] <= w[1]]
            samples = inside or sorted(samples, key=lambda x: min(abs(x[0] - w[0]), abs(x[0] - w[1])))[:2]
        sm = [x[1] for x in samples]
        mx = [x[2] for x in samples]
        reasons = sorted(nm for nm, bit in self.REASONS.items() if any(x[3] & bit for x in samples))
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm), "source": self.source}


# ---------------------------------------------------------------------------- tensor-core sample


def brute_tc_sample(n=131_072, k=16, reps=3):
    """Brute-force exact-mode distance tiles (tensor-core bound):
    pk_brute_knn_tc over a C5-generator sample (d=1024), all n queries.  Flops
    = 2 m n d of the screening GEMM; time = tc_screen_kernel's CUDA-event time."""
    import torch

    import paper_2312_03940_b200 as pk
    from paper_2312_03940_b200 import _lib, index, workloads

    data, _ = workloads.generate("C5", n=n, components=max(1, n // 1281))
    p = pk.PointSet(data)
    q = torch.arange(n, dtype=torch.int64, device="cuda")
    index.brute_device(p, q[:4096], k)
    torch.cuda.synchronize()
    _lib.prof_collect(reset=True)
    _lib.prof_only(["tc_screen_kernel", "tc_rescore_kernel"])
    _lib.prof_enable(True)
    index.TC_STATS.update(rows=0, uncertified=0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        index.brute_device(p, q, k)
    e1.record()
    torch.cuda.synchronize()
    _lib.prof_enable(False)
    prof = _lib.prof_collect(reset=True)
    scr_ms = prof["tc_screen_kernel"][1] / reps
    flops = 2.0 * n * n * 1024
    _, tflops, kind = peaks()
    ach = flops / (scr_ms / 1e3) / 1e12
    del p, data
    torch.cuda.empty_cache()
    return {"bound": "tensor", "kernel": "tc_screen_kernel", "achieved": ach, "peak": tflops, "unit": "TFLOP/s",
            "frac": ach / tflops, "traffic": None, "peak_source": kind,
            "sample": f"exact kNN (BruteForceIndex path) of all {n} points, C5 generator d=1024, k={k}, fp16 "
                      f"tcgen05 screening + float64 rescoring",
            "screen_ms": scr_ms, "call_ms": e0.elapsed_time(e1) / reps,
            "rescore_ms": prof.get("tc_rescore_kernel", (0, 0.0))[1] / reps,
            "uncertified_rows": index.TC_STATS["uncertified"] // reps}


def hbm_gather_sample(n=200_000, k=16, reps=2):
    """Beam-search kNN at HBM scale (the gather-bound kernel):
    knn_all over a C5-generator sample (d = 1024 float32, 820 MB >> the 126 MB
    L2) on a graph built with C5's R = 64, L = 200.  One untimed counting pass
    gives the distinct evaluations U and expansions X; bytes = (U - n s) 4 d +
    X 4 R (fp32 rows, seeds excluded); time = beam_knn_kernel's CUDA-event time."""
    import torch

    import paper_2312_03940_b200 as pk
    from paper_2312_03940_b200 import _lib, vamana, workloads

    w = workloads.WORKLOADS["C5"]
    data, _ = workloads.generate("C5", n=n, components=max(1, n // 1281))
    p = pk.PointSet(data)
    del data
    g = pk.build_vamana(p, R=w.R, L_build=w.L, alpha=w.alpha, seed=0, query_beam=w.L)
    q = torch.arange(n, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(3, dtype=torch.int64, device="cuda")
    os.environ["PK_COUNT_UNIQUE"] = "1"
    try:
        vamana.beam_knn_raw(g.graph, q, w.L, k, cnt)
        torch.cuda.synchronize()
    finally:
        os.environ.pop("PK_COUNT_UNIQUE", None)
    evals, expansions, uniq = cnt.tolist()
    _lib.prof_collect(reset=True)
    _lib.prof_only(["beam_knn_kernel"])
    _lib.prof_enable(True)
    for _ in range(reps):
        vamana.beam_knn_raw(g.graph, q, w.L, k)
    torch.cuda.synchronize()
    _lib.prof_enable(False)
    prof = _lib.prof_collect(reset=True)
    ms = prof["beam_knn_kernel"][1] / reps
    s = int(np.ceil(np.sqrt(n)))
    alg = (uniq - n * s) * 4 * w.d + expansions * 4 * w.R
    hbm, _, kind = peaks()
    ach = alg / (ms / 1e3) / 1e9
    del g, p
    torch.cuda.empty_cache()
    return {"bound": "hbm", "kernel": "beam_knn_kernel", "achieved": ach, "peak": hbm, "unit": "GB/s",
            "frac": ach / hbm, "traffic": None, "peak_source": kind,
            "sample": f"knn_all (k={k}, L={w.L}) over a C5-generator sample n={n}, d={w.d} float32 "
                      f"({n * w.d * 4 / 1e6:.0f} MB, larger than L2), graph R={w.R} L={w.L}",
            "kernel_ms": ms, "queries_per_s": n / (ms / 1e3), "unique_evals_per_query": uniq / n,
            "expansions_per_query": expansions / n, "algorithmic_bytes": alg,
            "definition": "(unique evals - seeds) x 4d + expansions x 4R over all queries"}


# ---------------------------------------------------------------------------- counting pass


def unique_evaluations(p, kw, vamana, comm):
    """One untimed pipeline pass in the kernels' counting mode: per-warp global
    bitmaps record every id a search evaluates, giving the exact number of
    distinct evaluations (the roofline's U) next to the expansions (X)."""
    import torch

    from paper_2312_03940_b200.cluster import run_pipeline_device

    bst = torch.zeros(5, dtype=torch.int64, device="cuda")
    bem = torch.zeros(3, dtype=torch.int64, device="cuda")
    vamana.STATS["build"], vamana.STATS["beam"] = bst, bem
    os.environ["PK_COUNT_UNIQUE"] = "1"
    try:
        run_pipeline_device(p, **kw, comm=comm)
        torch.cuda.synchronize()
    finally:
        os.environ.pop("PK_COUNT_UNIQUE", None)
        vamana.STATS["build"] = vamana.STATS["beam"] = None
    b, e = bst.tolist(), bem.tolist()
    return {"build_unique": b[4], "build_evals": b[0], "build_expansions": b[3],
            "beam_unique": e[2], "beam_evals": e[0], "beam_expansions": e[1]}


# ---------------------------------------------------------------------------- CPU baseline


def cpu_pipeline(name, n_override=None):
    """The reference algorithm on the host cores via the oracle C restatement."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    from paper_2312_03940_b200 import workloads

    w = workloads.WORKLOADS[name]
    cores = os.cpu_count() or 1
    if n_override is not None:
        n = n_override
    else:
        # bounded sample: the full configuration when the host has many cores,
        # otherwise a smaller instance of the same generator (~10-30 s)
        n = min(w.n, max(10_000, cores * 3_000))
    comps = max(1, int(round(w.components * n / w.n)))
    data, _ = workloads.generate(name, n=n, components=comps)
    oracle.build()
    oracle.set_num_threads(cores)
    t = time.perf_counter()
    out = oracle.pipeline(data, index="vamana", R=w.R, L_build=w.L, L=w.L, alpha=w.alpha, seed=0, k=w.k,
                          density_kind=w.density, center_policy=("product", max(1, min(w.n_centers, comps))),
                          rho_min=0.0, initial_k=2 * w.k, threshold=300)
    secs = time.perf_counter() - t
    sample = (f"full {name} pipeline" if n == w.n else f"{name}-generator instance n={n} ({comps} comps)") + \
        f" through oracle/ (C restatement of _kernels.py + numpy stages), OpenMP {cores} threads"
    return n / secs, cores, sample, secs, out["timings"]


# ---------------------------------------------------------------------------- reference arm


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2312_03940_b200 import workloads

    w = workloads.WORKLOADS[args.config]
    for _ in range(args.warmup):
        cpu_pipeline(args.config, n_override=min(w.n, 5_000))
    vals, total = [], 0.0
    info = None
    for _ in range(args.steps):
        v, cores, sample, secs, timings = cpu_pipeline(args.config, args.n)
        vals.append(v)
        total += secs
        info = (cores, sample, timings)
    value = float(np.mean(vals))
    cores, sample, timings = info
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(args.config, args.n, 1),
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "stage_seconds": timings,
    }
    print(json.dumps(line), flush=True)


def workload_config(name, n_override, n_gpus):
    par = "single GPU" if n_gpus == 1 else f"sharded x{n_gpus} (queries + build batches split, NCCL all-gather)"
    from paper_2312_03940_b200 import workloads

    w = workloads.WORKLOADS[name]
    n = n_override or w.n
    return {"workload": f"{name}: n={n} d={w.d} Vamana R={w.R} L={w.L} alpha={w.alpha} {w.density} k={w.k} "
                        f"ProductCenter({w.n_centers}) doubling from {2 * w.k}, threshold 300",
            "n": n, "d": w.d, "R": w.R, "L": w.L, "k": w.k, "density": w.density,
            "parallelism": par, "l2": "flushed (256 MiB write) before every timed step",
            "host": "python gc.freeze() after the warm-up steps (start-up heap out of the collector)"}


# ---------------------------------------------------------------------------- our arm


def main_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2312_03940_b200 as pk
    from paper_2312_03940_b200 import _lib, vamana, workloads
    from paper_2312_03940_b200.cluster import run_pipeline_device
    from paper_2312_03940_b200.core import upload_points
    from paper_2312_03940_b200.shard import Comm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # PK_BENCH_BACKEND=gloo PK_BENCH_DEVICE=0: functional check of the multi-rank
    # path with every rank on one device (not a measurement)
    local = int(os.environ.get("PK_BENCH_DEVICE", local))
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        backend = os.environ.get("PK_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        comm = Comm()

    name = args.config
    w = workloads.WORKLOADS[name]
    n = args.n or w.n
    comps = w.components if args.n is None else max(1, int(round(w.components * n / w.n)))
    data, truth = workloads.generate(name, n=n, components=comps)
    kw = workloads.pipeline_args(name, pk, n_centers=min(w.n_centers, comps))

    dev_pts = upload_points(data)
    p = pk.PointSet(data).attach_device(dev_pts)
    _ = p.mode
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()

    # the clock sampler (an nvidia-smi process) starts before the warm-up so its
    # start-up does not land in the timed steps; samples are filtered to the window
    clocks = ClockSampler(local)
    clocks.start()
    # warm-up (untimed), holding the previous result alive as the timed loop does
    # (so the caching allocator already has room for two results' tensors)
    last = None
    for _ in range(args.warmup):
        last = run_pipeline_device(p, **kw, comm=comm)
    torch.cuda.synchronize()
    # a serving process freezes its start-up heap: every object created so far
    # (torch, numpy, the package) leaves the collector's generations, so a
    # gen-2 collection inside a timed step scans only the step's own objects
    # (unfrozen, full collections took 15-27 ms of a 37 ms step)
    import gc

    gc.collect()
    gc.freeze()

    build_stats = torch.zeros(5, dtype=torch.int64, device="cuda")
    beam_stats = torch.zeros(3, dtype=torch.int64, device="cuda")
    vamana.STATS["build"] = build_stats
    vamana.STATS["beam"] = beam_stats
    _lib.prof_collect(reset=True)
    # event timing only for the kernels the roofline and the breakdown need (every
    # launch is still counted); bracketing all ~300 launches per step costs ~1 ms
    _lib.prof_only(TIMED_KERNELS)
    _lib.prof_enable(os.environ.get("PK_BENCH_PROF", "1") == "1")
    clocks.wait_first()
    total_ms = 0.0
    t_win0 = time.perf_counter()
    step_ms = []
    stage = {"index": 0.0, "density": 0.0, "dependent": 0.0, "unionfind": 0.0}
    step_stages = []
    rounds = []
    last = None
    stream = torch.cuda.current_stream()
    for _ in range(args.steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        trace = []
        last = run_pipeline_device(p, **kw, trace=trace, comm=comm)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        step_ms.append(e0.elapsed_time(e1))
        if os.environ.get("PK_BENCH_TRACE") == "1":
            print(f"timed step {len(step_ms) - 1}: host {time.perf_counter():.3f}", file=sys.stderr, flush=True)
        total_ms += step_ms[-1]
        for kk_, v in last["timings"].items():
            stage[kk_] += v
        step_stages.append({kk_: round(v * 1e3, 2) for kk_, v in last["timings"].items()})
        rounds = trace
    clocks.mark(t_win0, time.perf_counter())
    clk = clocks.stop()
    _lib.prof_enable(False)
    prof = _lib.prof_collect(reset=True)
    vamana.STATS["build"] = None
    vamana.STATS["beam"] = None

    t_local = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    ms_step = float(t_local.item()) / args.steps
    value = n / (ms_step / 1e3)  # the n points are split across the ranks

    # quality of the last timed run (ARI vs generator labels)
    labels = _lib.to_host(last["labels"])
    ari_truth = pk.ari(labels, truth)

    # end-to-end through the public API with host buffers
    pinned = torch.from_numpy(np.array(data, dtype=np.float32, copy=True)).pin_memory()
    host_view = pinned.numpy()
    e2e_ms = 0.0
    e2e_steps_ms = []
    e2e_stage_ms = []
    h2d = d2h = 0
    # untimed e2e warm-up: two calls with the first result still alive, as in the
    # timed loop (each result's arrays live in a pinned staging block of torch's
    # caching host allocator, so the loop alternates between two blocks)
    r0 = pk.run_pipeline(pk.PointSet(host_view), **kw, comm=comm)
    r1 = pk.run_pipeline(pk.PointSet(host_view), **kw, comm=comm)
    del r0, r1
    torch.cuda.synchronize()
    for _ in range(args.e2e_steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = pk.run_pipeline(pk.PointSet(host_view), **kw, comm=comm)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        e2e_ms += e0.elapsed_time(e1)
        e2e_steps_ms.append(round(e0.elapsed_time(e1), 3))
        e2e_stage_ms.append({k_: round(v * 1e3, 2) for k_, v in res.timings.items()})
        h2d = n * w.d * 4
        st = res.state
        d2h = sum(a.nbytes for a in (st.rho, st.lam, st.delta, st.neighbors.ids, st.neighbors.dists,
                                     res.clustering.labels, res.clustering.centers, res.clustering.noise))
    t_e2e = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
    e2e_value = n / (float(t_e2e.item()) / args.e2e_steps / 1e3)

    # roofline: the dominant HBM-gather kernel (beam searches)
    hbm, tflops, peak_kind = peaks()
    launches = sum(c for c, _ in prof.values())
    overall = max(prof.items(), key=lambda kv: kv[1][1])
    gather = {k_: v for k_, v in prof.items() if k_.startswith(("build_search", "beam_knn"))}
    dom = max(gather.items(), key=lambda kv: kv[1][1])
    dom_name, (dom_cnt, dom_ms) = dom
    bs = _lib.to_host(build_stats) / args.steps
    be = _lib.to_host(beam_stats) / args.steps
    # untimed counting pass: the exact number of DISTINCT ids each search
    # evaluated (U of SURVEY.md 8(d); the lossy seen table re-evaluates a few)
    uniq = unique_evaluations(p, kw, vamana, comm)
    queries_beam = n + sum(r[0] for r in rounds if isinstance(r[1], int))
    s = int(np.ceil(np.sqrt(n)))
    d4 = w.d * 4
    # both launch wrappers run the same beam-search walk (WarpBeam): build-time
    # searches of the inserted points and query-time kNN searches
    per_kernel = {}
    for kn, (cnt_, ms_) in gather.items():
        if kn.startswith("build_search"):
            # per inserted point: non-seed unique search evaluations + adjacency rows
            ev_ns = uniq["build_unique"] - n * s
            ab = ev_ns * d4 + uniq["build_expansions"] * w.R * 4
        else:
            ev_ns = uniq["beam_unique"] - queries_beam * s
            ab = ev_ns * d4 + uniq["beam_expansions"] * w.R * 4
        per_kernel[kn] = {"algorithmic_bytes_per_step": ab, "ms_per_step": ms_ / args.steps,
                          "achieved": (ab / 1e9) / (ms_ / args.steps / 1e3), "launches_per_step": cnt_ / args.steps}
        per_kernel[kn]["frac"] = per_kernel[kn]["achieved"] / hbm
    alg_bytes = sum(v["algorithmic_bytes_per_step"] for v in per_kernel.values())
    search_ms = sum(v["ms_per_step"] for v in per_kernel.values())
    search_launches = sum(v["launches_per_step"] for v in per_kernel.values())
    unit_desc = ("gather bytes (unique non-seed evals x 4d + expansions x 4R, fp32 rows) of every beam search of the "
                 "step -- build searches of the inserted points and kNN / doubling-round searches of the queries")
    per_launch_ms = search_ms / max(search_launches, 1e-9)
    per_step_launches = search_launches
    achieved = (alg_bytes / 1e9) / (search_ms / 1e3)
    dom_ms = search_ms * args.steps

    tc = None
    if rank == 0 and not args.no_tc_sample:
        try:
            tc = brute_tc_sample()
        except Exception as e:  # noqa: BLE001 -- reported, never silently replaced
            tc = {"error": repr(e)}
    hbm_s = None
    if rank == 0 and not args.no_hbm_sample:
        try:
            hbm_s = hbm_gather_sample()
        except Exception as e:  # noqa: BLE001 -- reported, never silently replaced
            hbm_s = {"error": repr(e)}

    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        tr = json.load(open(tpath))
        for kn in per_kernel:
            per_kernel[kn]["traffic_largest_launch"] = tr.get(kn, {}).get("dram_bytes_per_launch")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, sample, secs, timings = cpu_pipeline(name, args.n)
        cpu = {"value": v, "unit": "points/s", "cores": cores, "kind": "port", "sample": sample,
               "seconds": secs}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": {0: "f64", 1: "f32 (exact: integer data)", 2: "u8/int32 (exact: integer data)"}[p.mode],
            "data": f"synthetic ({name} generator, seed 0)",
            "config": workload_config(name, args.n, world),
            "e2e": {"value": e2e_value, "unit": "points/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "step_ms": e2e_steps_ms, "step_stage_ms": e2e_stage_ms},
            "roofline": {"bound": "hbm", "kernel": "beam search walk (build_search_kernel + beam_knn_kernel)",
                         "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": (achieved / hbm) if achieved else None, "traffic": traffic,
                         "peak_source": peak_kind, "algorithmic_bytes_per_step": alg_bytes,
                         "launches_per_step": per_step_launches, "avg_launch_ms": per_launch_ms,
                         "kernel_share_of_step": dom_ms / args.steps / ms_step, "definition": unit_desc,
                         "per_kernel": per_kernel,
                         "largest_kernel_overall": overall[0],
                         "largest_kernel_share": overall[1][1] / args.steps / ms_step},
            "roofline_tensor": tc,
            "roofline_hbm_scale": hbm_s,
            "cpu_baseline": cpu,
            "gpu_launches": int(launches / args.steps) * args.steps,
            "gpu_launches_per_step": launches / args.steps,
            "clocks": clk,
            "stage_ms": {k_: v / args.steps * 1e3 for k_, v in stage.items()},
            "step_ms": [round(v, 3) for v in step_ms],
            "step_stage_ms": step_stages,
            "dependent_rounds": rounds,
            "kernels_ms_per_step": {k_: round(v[1] / args.steps, 4) for k_, v in sorted(prof.items(),
                                                                                      key=lambda kv: -kv[1][1])
                                    if k_ in TIMED_KERNELS},
            "kernel_launches_per_step": {k_: v[0] / args.steps for k_, v in sorted(prof.items())},
            "counters_per_step": {"build": bs.tolist(), "beam": be.tolist(),
                                  "legend": "build [evals, prune evals, reverse evals, expansions]; "
                                            "beam [evals, expansions] (timed steps)"},
            "unique_evaluations": uniq,
            "ari_vs_generator": ari_truth,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        main_ours(args)


if __name__ == "__main__":
    main()
