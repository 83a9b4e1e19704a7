#!/usr/bin/env python
"""Benchmark: end-to-end ANN density-peaks clustering (points/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C5] [--n N_POINTS] [--no-cpu-baseline] [--no-extras]

A step is one full pass of the hot path over the configuration's synthetic
point set: graph build, kNN densities, dependent points, policies +
union-find labels, all on the GPU.  The default workload is C5, the largest
configuration of BASELINE.json (n = 1,281,167 x d = 1024 float32,
image-embedding-shaped, Vamana R = 64 L = 200 alpha = 1.1, kth k = 16,
doubling from 32 with threshold 300, 1,000 product centers; the paper's own
headline dataset has the same n and d).  Its 5.2 GB of
points are far larger than the 126 MB L2 (L2 is still flushed before every
timed step).

* `value` = points/s with the points already resident in HBM (CUDA events
  around each step on the launching stream, max over ranks).
* `e2e` = the same through the public API (`run_pipeline(PointSet(host
  array))`): host->device upload of the points and device->host read of every
  result array inside the timed region.
* `roofline` = the beam-search walk (build searches + kNN / doubling-round
  searches: one device function behind two launch wrappers), algorithmic
  gather bytes ((unique evaluations - seeds) x 4d + expansions x 4R, counted
  by the kernels in an untimed pass) / its CUDA-event time, against the
  measured HBM copy bandwidth; `traffic` = its DRAM bytes per launch from the
  ncu capture of this configuration committed in profiles/.
* `roofline_tensor` = the exact (BruteForceIndex) kNN of all C5 points on the
  tensor cores: 2 n^2 d flops / the screening kernel's time.
* `cpu_baseline` / `--impl reference` = the reference algorithm on the host
  cores (oracle/: C restatement of _kernels.py + the numpy stages, OpenMP
  over every host thread) on a bounded sample of the same generator; the
  sample size is stated, never relabelled as the full configuration.
* `c2` = the full C2 configuration (n = 100,000) on the GPU plus the CPU port
  on the same full n.

Multi-GPU (torchrun, one rank per GPU, NCCL): the same n points are split
across the ranks (shard.py), total work fixed ("scaling": "strong"); value =
n / (max over ranks of the step time).
"""

from __future__ import annotations

import argparse
import gc
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
WALK_KERNELS = ("build_search_kernel", "beam_knn_kernel")
TIMED_KERNELS = WALK_KERNELS + ("prune_tc_build_kernel", "prune_tc_reverse_kernel", "build_prune_block_kernel",
                                "reverse_block_kernel", "reverse_big_kernel", "build_prune_kernel", "reverse_kernel",
                                "tc_screen_kernel", "dp_scan_kernel")
# oracle sample sizes (points) per configuration: ~10-20 s of CPU work on a 16-core host
CPU_SAMPLE = {"C1": 10_000, "C2": 48_000, "C3": 60_000, "C4": 24_000, "C5": 12_000}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the tensor-core pass and the C2 extra")
    ap.add_argument("--e2e-steps", type=int, default=None, help="default min(steps, 3)")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        pk = json.load(open(path))
        return pk["hbm_gbs"], pk["bf16_tflops"], pk.get("bf16_tflops_sustained"), "measured (MEASURED_PEAKS.json)"
    return 6650.0, 1590.0, None, "fallback (B200_PROFILING.md)"


def git_head():
    try:
        return subprocess.run(["git", "-C", ROOT, "rev-parse", "--short=12", "HEAD"], capture_output=True,
                              text=True, timeout=5).stdout.strip() or None
    except Exception:  # noqa: BLE001
        return None


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


# ---------------------------------------------------------------------------- CPU side (oracle)


def cpu_pipeline(name, n):
    """The reference algorithm on the host cores (oracle/ C restatement,
    OpenMP over every host thread) on an n-point instance of the generator.
    Returns (seconds, cores, stage timings, description)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    from paper_2312_03940_b200 import workloads

    w = workloads.WORKLOADS[name]
    comps = max(1, int(round(w.components * n / w.n)))
    data, _ = workloads.generate(name, n=n, components=comps)
    oracle.build()
    cores = os.cpu_count() or 1
    oracle.set_num_threads(cores)
    t = time.perf_counter()
    out = oracle.pipeline(data, index="vamana", R=w.R, L_build=w.L, L=w.L, alpha=w.alpha, seed=0, k=w.k,
                          density_kind=w.density, center_policy=("product", max(1, min(w.n_centers, comps))),
                          rho_min=0.0, initial_k=2 * w.k, threshold=300)
    secs = time.perf_counter() - t
    what = ("the full " if n == w.n else f"an n={n} instance ({comps} components) of the ") + \
        f"{name} generator through oracle/ (C restatement of _kernels.py + numpy stages), OpenMP {cores} threads"
    return secs, cores, out["timings"], what


def cpu_baseline(name, n_full, n_sample):
    secs, cores, timings, what = cpu_pipeline(name, n_sample)
    line = {"value": n_sample / secs, "unit": "points/s", "cores": cores, "kind": "port",
            "sample": what, "n": n_sample, "seconds": secs, "stage_seconds": timings}
    if n_sample != n_full:
        # linear in n: a lower bound on the port's time at full n (the reference's
        # runtime grows as n^1.12-1.2)
        line["extrapolated"] = {"n": n_full, "seconds": secs * n_full / n_sample, "rule": "linear in n (lower bound)"}
    return line


def run_reference(args):
    """--impl reference: the oracle port on the host cores, rank 0 only."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    from paper_2312_03940_b200 import workloads

    w = workloads.WORKLOADS[args.config]
    n_full = args.n or w.n
    n = min(n_full, CPU_SAMPLE.get(args.config, 10_000))
    # per-step sample bounded so that W + K steps stay within a few minutes
    n = min(n, max(2_000, int(n * 12 / max(args.steps, 1))))
    for _ in range(args.warmup):
        cpu_pipeline(args.config, min(n, 2_000))
    secs, info = [], None
    for _ in range(args.steps):
        s, cores, timings, what = cpu_pipeline(args.config, n)
        secs.append(s)
        info = (cores, timings, what)
    cores, timings, what = info
    per_step = float(np.mean(secs))
    value = n / per_step
    cfg = workload_config(args.config, n, 1)
    cfg["sample_of"] = f"{args.config} (n={n_full})" if n != n_full else None
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": f"synthetic ({args.config} generator, seed 0)",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": cores, "kind": "port", "sample": what, "n": n},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "stage_seconds": timings,
        "note": None if n == n_full else (f"each step runs an n={n} sample of {args.config} (the full n={n_full} "
                                          f"takes the CPU port far longer than a bench run); value is points/s on "
                                          f"that sample, not at full n"),
    }
    if n != n_full:
        line["extrapolated_full_n"] = {"n": n_full, "seconds": per_step * n_full / n,
                                       "points_per_s": value, "rule": "linear in n (lower bound on time)"}
    print(json.dumps(line), flush=True)


def workload_config(name, n, n_gpus):
    from paper_2312_03940_b200 import workloads

    w = workloads.WORKLOADS[name]
    par = "single GPU" if n_gpus == 1 else f"sharded x{n_gpus} (queries + build batches split, NCCL all-gather)"
    return {"workload": f"{name}: n={n} d={w.d} Vamana R={w.R} L={w.L} alpha={w.alpha} {w.density} k={w.k} "
                        f"ProductCenter({w.n_centers}) doubling from {2 * w.k}, threshold 300",
            "n": n, "d": w.d, "R": w.R, "L": w.L, "k": w.k, "density": w.density, "parallelism": par,
            "l2": ("inputs larger than L2 (126 MB); L2 also flushed (256 MiB write) before every timed step"
                   if n * w.d * 4 > (126 << 20) else "L2 flushed (256 MiB write) before every timed step"),
            "host": "python gc.freeze() after the warm-up steps (start-up heap out of the collector)"}


# ---------------------------------------------------------------------------- GPU side


def counting_pass(p, kw, comm):
    """One untimed pipeline pass in the kernels' counting mode: per-warp global
    bitmaps record every id a search evaluates, giving the exact number of
    distinct evaluations (the roofline's U) next to the expansions (X)."""
    import torch

    from paper_2312_03940_b200 import vamana
    from paper_2312_03940_b200.cluster import run_pipeline_device

    bst = torch.zeros(5, dtype=torch.int64, device="cuda")
    bem = torch.zeros(3, dtype=torch.int64, device="cuda")
    vamana.STATS["build"], vamana.STATS["beam"] = bst, bem
    os.environ["PK_COUNT_UNIQUE"] = "1"
    trace = []
    try:
        run_pipeline_device(p, **kw, comm=comm, trace=trace)
        torch.cuda.synchronize()
    finally:
        os.environ.pop("PK_COUNT_UNIQUE", None)
        vamana.STATS["build"] = vamana.STATS["beam"] = None
    b, e = bst.tolist(), bem.tolist()
    return {"build_unique": b[4], "build_evals": b[0], "build_expansions": b[3],
            "beam_unique": e[2], "beam_evals": e[0], "beam_expansions": e[1]}, trace


def traffic_record(name):
    """DRAM bytes per launch of the walk kernels from the committed ncu capture
    of this configuration (tools/ncu_traffic.py writes it)."""
    path = os.path.join(ROOT, "profiles", f"ncu_traffic_{name.lower()}.json")
    if not os.path.exists(path):
        return None
    return json.load(open(path))


def walk_roofline(prof, uniq, queries, n, w, steps, ms_step, hbm, peak_kind, name):
    """Algorithmic gather bytes of every beam search of a step / the walk
    kernels' CUDA-event time (B_q = (U_q - s) 4d + X_q 4R)."""
    s = int(np.ceil(np.sqrt(n)))
    d4 = w.d * 4
    per = {}
    for kn in WALK_KERNELS:
        if kn not in prof:
            continue
        cnt, ms = prof[kn]
        if kn == "build_search_kernel":
            ab = (uniq["build_unique"] - n * s) * d4 + uniq["build_expansions"] * w.R * 4
        else:
            ab = (uniq["beam_unique"] - queries * s) * d4 + uniq["beam_expansions"] * w.R * 4
        per[kn] = {"algorithmic_bytes_per_step": ab, "ms_per_step": ms / steps, "launches_per_step": cnt / steps,
                   "achieved": ab / 1e9 / (ms / steps / 1e3)}
        per[kn]["frac"] = per[kn]["achieved"] / hbm
    alg = sum(v["algorithmic_bytes_per_step"] for v in per.values())
    ms = sum(v["ms_per_step"] for v in per.values())
    launches = sum(v["launches_per_step"] for v in per.values())
    achieved = alg / 1e9 / (ms / 1e3)
    line = {"bound": "hbm", "kernel": "beam-search walk (build_search_kernel + beam_knn_kernel)",
            "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm, "traffic": None,
            "peak_source": peak_kind, "algorithmic_bytes_per_step": alg, "launches_per_step": launches,
            "algorithmic_bytes_per_launch": alg / launches, "avg_launch_ms": ms / launches,
            "kernel_share_of_step": ms / ms_step, "per_kernel": per,
            "definition": "(unique evaluations - seeds) x 4d + expansions x 4R over every beam search of the "
                          "step (fp32 rows at 4 B/coordinate), / the walk kernels' CUDA-event time"}
    tr = traffic_record(name)
    if tr:
        tot_b = sum(tr[k]["dram_bytes"] for k in WALK_KERNELS if k in tr)
        tot_l = sum(tr[k]["launches"] for k in WALK_KERNELS if k in tr)
        if tot_l:
            line["traffic"] = tot_b / tot_l
            line["traffic_source"] = f"profiles/ncu_traffic_{name.lower()}.json (commit {tr.get('commit')}, " \
                                     f"{tot_l} walk launches of one pipeline pass)"
            line["traffic_per_step"] = tot_b
    return line


def tensor_roofline(p, n, d, tflops, sustained, peak_kind):
    """Exact kNN (BruteForceIndex path) of all n points on the tensor cores
    (brute-force tiles are tensor-bound, 2 m n d flops)."""
    import torch

    from paper_2312_03940_b200 import _lib, index

    q = torch.arange(n, dtype=torch.int64, device="cuda")
    index.brute_device(p, q[:8192], 16)
    torch.cuda.synchronize()
    _lib.prof_collect(reset=True)
    _lib.prof_only(["tc_screen_kernel", "tc_rescore_kernel"])
    _lib.prof_enable(True)
    index.TC_STATS.update(rows=0, uncertified=0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ids, sqd = index.brute_device(p, q, 16)
    e1.record()
    torch.cuda.synchronize()
    _lib.prof_enable(False)
    prof = _lib.prof_collect(reset=True)
    cnt, scr_ms = prof["tc_screen_kernel"]
    flops = 2.0 * n * n * d
    ach = flops / (scr_ms / 1e3) / 1e12
    del ids, sqd
    return {"bound": "tensor", "kernel": "tc_screen_kernel", "achieved": ach, "peak": tflops, "unit": "TFLOP/s",
            "frac": ach / tflops, "frac_of_sustained": (ach / sustained) if sustained else None, "traffic": None,
            "peak_source": f"{peak_kind}, dense bf16 (the kernel runs fp16 operands, same rate)",
            "sample": f"exact kNN (k=16) of all {n} points x {n} points, d={d}: fp16 tcgen05 screening "
                      f"(CTA pairs, TMEM accumulators) + float64 rescoring; flops = 2 n^2 d = {flops:.3e}",
            "screen_ms": scr_ms, "screen_launches": cnt, "call_ms": e0.elapsed_time(e1),
            "rescore_ms": prof.get("tc_rescore_kernel", (0, 0.0))[1],
            "uncertified_rows": index.TC_STATS["uncertified"]}


def c2_extra(steps=5):
    """Full C2 (n = 100,000) on the GPU: device-timed steps after a warm-up."""
    import torch

    import paper_2312_03940_b200 as pk
    from paper_2312_03940_b200 import workloads
    from paper_2312_03940_b200.cluster import run_pipeline_device

    data, _ = workloads.generate("C2")
    kw = workloads.pipeline_args("C2", pk)
    p = pk.PointSet(data)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        last = run_pipeline_device(p, **kw)
    ms = []
    for _ in range(steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        last = run_pipeline_device(p, **kw)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    del last, p
    t = float(np.mean(ms))
    return {"workload": workload_config("C2", 100_000, 1)["workload"], "value": 100_000 / (t / 1e3),
            "unit": "points/s", "ms_per_step": t, "step_ms": [round(v, 3) for v in ms],
            "note": "C2 fits in L2 (51 MB): an L2-served rate, not an HBM one"}


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
    e2e_steps = args.e2e_steps or min(args.steps, 3)

    dev_pts = upload_points(data)
    p = pk.PointSet(data).attach_device(dev_pts)
    mode = p.mode
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()

    clocks = ClockSampler(local)
    clocks.start()
    # warm-up (untimed), holding the previous result alive as the timed loop does
    last = None
    for _ in range(args.warmup):
        last = run_pipeline_device(p, **kw, comm=comm)
    torch.cuda.synchronize()
    # the start-up heap leaves the collector's generations (a full collection of
    # it inside a timed step took 15-27 ms)
    gc.collect()
    gc.freeze()

    build_stats = torch.zeros(5, dtype=torch.int64, device="cuda")
    beam_stats = torch.zeros(3, dtype=torch.int64, device="cuda")
    vamana.STATS["build"] = build_stats
    vamana.STATS["beam"] = beam_stats
    _lib.prof_collect(reset=True)
    # event timing only for the kernels the roofline and the breakdown need (every
    # launch is still counted)
    _lib.prof_only(TIMED_KERNELS)
    _lib.prof_enable(os.environ.get("PK_BENCH_PROF", "1") == "1")
    clocks.wait_first()
    t_win0 = time.perf_counter()
    step_ms, step_stages, rounds = [], [], []
    stage = {"index": 0.0, "density": 0.0, "dependent": 0.0, "unionfind": 0.0}
    stream = torch.cuda.current_stream()
    last = None
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
        for k_, v in last["timings"].items():
            stage[k_] += v
        step_stages.append({k_: round(v * 1e3, 2) for k_, v in last["timings"].items()})
        rounds = trace
    clocks.mark(t_win0, time.perf_counter())
    clk = clocks.stop()
    _lib.prof_enable(False)
    prof = _lib.prof_collect(reset=True)
    vamana.STATS["build"] = vamana.STATS["beam"] = None

    t_local = torch.tensor([sum(step_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    ms_step = float(t_local.item()) / args.steps
    value = n / (ms_step / 1e3)
    labels = _lib.to_host(last["labels"])
    ari_truth = pk.ari(labels, truth)
    del last

    # end-to-end through the public API with host buffers
    pinned = torch.from_numpy(np.array(data, dtype=np.float32, copy=True)).pin_memory()
    host_view = pinned.numpy()
    del dev_pts, p
    torch.cuda.empty_cache()
    e2e_steps_ms, e2e_stage_ms = [], []
    h2d = d2h = 0
    r0 = pk.run_pipeline(pk.PointSet(host_view), **kw, comm=comm)
    r1 = pk.run_pipeline(pk.PointSet(host_view), **kw, comm=comm)
    del r0, r1
    torch.cuda.synchronize()
    for _ in range(e2e_steps):
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
        e2e_steps_ms.append(e0.elapsed_time(e1))
        e2e_stage_ms.append({k_: round(v * 1e3, 2) for k_, v in res.timings.items()})
        h2d = n * w.d * 4
        st = res.state
        arrays = [st.rho, st.lam, st.delta, res.clustering.labels, res.clustering.centers, res.clustering.noise]
        if st.neighbors is not None:  # multi-GPU: the kNN rows are gathered to rank 0 only
            arrays += [st.neighbors.ids, st.neighbors.dists]
        d2h = sum(a.nbytes for a in arrays)
    del res
    t_e2e = torch.tensor([sum(e2e_steps_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
    e2e_value = n / (float(t_e2e.item()) / e2e_steps / 1e3)

    # roofline of the walk: an untimed counting pass gives U and X
    p = pk.PointSet(host_view)
    _ = p.mode
    uniq, ctrace = counting_pass(p, kw, comm)
    queries = n + sum(r[0] for r in ctrace if isinstance(r[1], int))
    hbm, tflops, sustained, peak_kind = peaks()
    roof = walk_roofline(prof, uniq, queries, n, w, args.steps, ms_step, hbm, peak_kind, name)

    tc = c2 = None
    if rank == 0 and world == 1 and not args.no_extras:
        try:
            tc = tensor_roofline(p, n, w.d, tflops, sustained, peak_kind) if w.d >= 256 else None
        except Exception as e:  # noqa: BLE001 -- reported, never silently replaced
            tc = {"error": repr(e)}
    del p
    torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not args.no_extras and name != "C2":
        try:
            c2 = c2_extra()
        except Exception as e:  # noqa: BLE001
            c2 = {"error": repr(e)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(name, n, min(n, CPU_SAMPLE.get(name, 10_000)))
        if c2 is not None and "error" not in c2:
            secs, cores, _, what = cpu_pipeline("C2", 100_000)
            c2["cpu_port_same_n"] = {"value": 100_000 / secs, "unit": "points/s", "seconds": secs, "cores": cores,
                                     "sample": what}

    launches = sum(c for c, _ in prof.values())
    overall = max(prof.items(), key=lambda kv: kv[1][1])
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None,
            "dtype": {0: "f64 (fp32 screens, exact float64 keys)", 1: "f32 (exact: integer data)",
                      2: "u8/int32 (exact: integer data)"}[mode],
            "data": f"synthetic ({name} generator, seed 0)",
            "config": workload_config(name, n, world),
            "e2e": {"value": e2e_value, "unit": "points/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": e2e_steps, "step_ms": [round(v, 3) for v in e2e_steps_ms],
                    "step_stage_ms": e2e_stage_ms},
            "roofline": roof,
            "roofline_tensor": tc,
            "cpu_baseline": cpu,
            "c2": c2,
            "gpu_launches": int(round(launches / args.steps)) * args.steps,
            "gpu_launches_per_step": launches / args.steps,
            "clocks": clk,
            "stage_ms": {k_: v / args.steps * 1e3 for k_, v in stage.items()},
            "dependent_queries_per_s": _dep_rate(rounds, stage["dependent"] / args.steps),
            "step_ms": [round(v, 3) for v in step_ms],
            "step_stage_ms": step_stages,
            "dependent_rounds": rounds,
            "kernels_ms_per_step": {k_: round(v[1] / args.steps, 4) for k_, v in
                                    sorted(prof.items(), key=lambda kv: -kv[1][1]) if k_ in TIMED_KERNELS},
            "kernel_launches_per_step": {k_: v[0] / args.steps for k_, v in sorted(prof.items())},
            "largest_kernel": overall[0],
            "unique_evaluations": uniq,
            "counters_per_step": {"build": (_lib.to_host(build_stats) / args.steps).tolist(),
                                  "beam": (_lib.to_host(beam_stats) / args.steps).tolist(),
                                  "legend": "build [evals, prune evals, reverse evals, expansions]; "
                                            "beam [evals, expansions] (timed steps)"},
            "ari_vs_generator": ari_truth,
            "commit": git_head(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _dep_rate(rounds, dep_s):
    """Points resolved by the doubling rounds and the exact scan per second of
    the dependent stage."""
    if not rounds or dep_s <= 0:
        return None
    first = rounds[0][0]
    return {"points": first, "value": first / dep_s, "unit": "points/s"}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        main_ours(args)


if __name__ == "__main__":
    main()
