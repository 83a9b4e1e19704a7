"""Host logic of the multi-GPU split (shard.py) on CPU: world_size-2 gloo
process groups exercise the partitioning, the collectives and the build
exchange callback (called through its ctypes function pointer, the way
pk_build_vamana_sharded calls it)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2312_03940_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(world, fn):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    out = {}
    while not q.empty():
        r, res = q.get()
        out[r] = res
    codes = [p.exitcode for p in procs]
    assert codes == [0] * world, (codes, out)
    assert len(out) == world, out
    for r, res in out.items():
        assert res == "ok", (r, res)


def _worker(rank, world, port, fn, q):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        fn(shard.Comm())
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        import traceback

        q.put((rank, traceback.format_exc() + repr(e)))
    finally:
        dist.destroy_process_group()


def test_ranges_partition():
    for world in range(1, 9):
        for n in (0, 1, 2, 7, 100, 1001):
            c = shard.Comm(rank=0, world=world)
            got = []
            for r in range(world):
                c.rank = r
                lo, hi = c.my_range(n)
                assert 0 <= lo <= hi <= n
                assert lo == min(n, r * c.chunk(n))
                got.extend(range(lo, hi))
            assert got == list(range(n))


def test_largest_batch_bounds_every_batch():
    for n in (1, 2, 3, 10, 1000, 100_000, 1_281_167):
        lo, b, mx = 0, 1, 0
        while lo < n:
            mx = max(mx, min(b, n - lo))
            lo += b
            b *= 2
        assert mx <= shard.largest_batch(n) <= n


def _gathers(comm):
    r, w = comm.rank, comm.world
    assert (r, w) == (dist.get_rank(), 2)
    # equal chunks, in place, 2-D rows
    c = 3
    buf = torch.full((w * c + 1, 4), -1, dtype=torch.int64)
    buf[r * c:(r + 1) * c] = 10 * r + torch.arange(c * 4).view(c, 4)
    comm.all_gather_chunks(buf, c)
    for rr in range(w):
        assert torch.equal(buf[rr * c:(rr + 1) * c], 10 * rr + torch.arange(c * 4).view(c, 4))
    assert (buf[w * c] == -1).all()
    # variable lengths, rank order
    t = torch.arange(r + 1, dtype=torch.int64) + 100 * r
    v = comm.all_gather_varlen(t)
    assert v.tolist() == [0, 100, 101]
    e = comm.all_gather_varlen(torch.empty(0, dtype=torch.int64))
    assert e.numel() == 0
    # MAX / MIN merge of resolved entries (one owner per entry)
    lam = torch.full((6,), -1, dtype=torch.int64)
    delta = torch.full((6,), float("inf"), dtype=torch.float64)
    lam[r::2] = torch.arange(3) + 10 * r
    delta[r::2] = 0.5 + r
    comm.all_reduce(lam, "max")
    comm.all_reduce(delta, "min")
    assert lam.tolist() == [0, 10, 1, 11, 2, 12]
    assert delta.tolist() == [0.5, 1.5] * 3
    assert comm.max_time(1.0 + r, "cpu") == 2.0


def test_collectives_gloo_world2():
    _run(2, _gathers)


def _row_collectives(comm):
    """all_gather_rows / gather_rows_to_root over the my_range split (the
    sharded pipeline's rho exchange and the rank-0 gather of the kNN rows)."""
    r = comm.rank
    n = 7
    lo, hi = comm.my_range(n)
    local = torch.arange(lo * 3, hi * 3, dtype=torch.int64).view(-1, 3)
    full = comm.all_gather_rows(local, n)
    assert torch.equal(full, torch.arange(n * 3, dtype=torch.int64).view(n, 3))
    rho = torch.arange(lo, hi, dtype=torch.float64) * 0.5
    assert comm.all_gather_rows(rho, n).tolist() == [0.5 * i for i in range(n)]
    root = comm.gather_rows_to_root(local, n)
    if r == 0:
        assert torch.equal(root, torch.arange(n * 3, dtype=torch.int64).view(n, 3))
    else:
        assert root is None
    assert comm.all_gather_counts(r + 5, "cpu") == [5, 6]


def test_row_collectives_gloo_world2():
    _run(2, _row_collectives)


def _sharded_density_rows(comm):
    """kth_normalized from per-rank rows == the single-rank computation, with
    the row offset of pk_normalize_rho_rows emulated by the host restatement
    (rho_i = base_i * k / sum_j base[ids_ij]): the exchange pattern (gather raw
    kth, normalise own rows, gather rho) on two ranks."""
    import numpy as np

    n, k = 9, 3
    rng = np.random.default_rng(4)
    ids = torch.from_numpy(rng.integers(0, n, (n, k)).astype(np.int64))
    base_full = torch.from_numpy(rng.uniform(0.5, 2.0, n))
    lo, hi = comm.my_range(n)
    base = comm.all_gather_rows(base_full[lo:hi].clone(), n)
    assert torch.equal(base, base_full)
    own = base[lo:hi] * k / base[ids[lo:hi]].sum(1)
    rho = comm.all_gather_rows(own, n)
    want = base_full * k / base_full[ids].sum(1)
    assert torch.allclose(rho, want, rtol=0, atol=0)


def test_sharded_density_exchange_gloo_world2():
    _run(2, _sharded_density_rows)


def _build_exchange(comm):
    r, w = comm.rank, comm.world
    n, R = 50, 4
    ex = shard.BuildExchange(comm, n, R, "cpu")
    W = R + 2
    # PK_XCHG_OUTLISTS: a batch of m = 7 -> chunk 4; rank r wrote rows [r*4, r*4 + mine)
    m, c = 7, comm.chunk(7)
    lo, hi = comm.my_range(m)
    for t in range(lo, hi):
        ex.xids[t * R:(t + 1) * R] = torch.arange(R, dtype=torch.int32) + 100 * t
        ex.xlen[t] = t
    rc = ex.callback(None, shard.BuildExchange.OUTLISTS, c, 0)  # through the C function pointer
    assert rc == 0 and ex.error is None
    for t in range(m):
        assert ex.xids[t * R:(t + 1) * R].tolist() == [100 * t + j for j in range(R)]
        assert int(ex.xlen[t]) == t
    # PK_XCHG_ROWS: rank r packed r + 2 records [u, deg, row[R]]
    own = r + 2
    for i in range(own):
        u = 10 * r + i
        ex.xsend[i * W:(i + 1) * W] = torch.tensor([u, i] + [u + j for j in range(R)], dtype=torch.int32)
    maxc = ex.callback(None, shard.BuildExchange.ROWS, own, 0)
    assert maxc == w + 1 and ex.error is None
    assert ex.xcnt.tolist() == [2, 3]
    for rr in range(w):
        for i in range(rr + 2):
            rec = ex.xrecv[(rr * maxc + i) * W:(rr * maxc + i + 1) * W].tolist()
            u = 10 * rr + i
            assert rec == [u, i] + [u + j for j in range(R)]
    # errors surface as -1 plus the stored exception (never raised through C)
    assert ex.callback(None, 7, 0, 0) == -1 and isinstance(ex.error, ValueError)
    assert ex.calls[0] == 1 and ex.calls[1] == 1


def test_build_exchange_callback_gloo_world2():
    _run(2, _build_exchange)


def test_single_rank_comm_is_identity():
    c = shard.Comm(rank=0, world=1)
    t = torch.arange(5)
    assert c.all_gather_varlen(t) is t
    buf = torch.arange(6)
    c.all_gather_chunks(buf, 3)
    assert buf.tolist() == list(range(6))
    assert shard.Comm.auto() is None


@pytest.mark.gpu
def test_sharded_build_single_rank_matches_plain_build():
    """world = 1 through the sharded entry point is the plain build."""
    import numpy as np

    import paper_2312_03940_b200 as pk
    from paper_2312_03940_b200 import _lib, vamana

    rng = np.random.default_rng(3)
    x = rng.normal(size=(3000, 24)).astype(np.float32)
    p = pk.PointSet(x)
    starts, order = vamana.sample_starts(p.n, None, 0, False, p)
    a0, d0 = vamana.build_graph_device(p, 16, 32, 1.2, starts, order)
    ex = shard.BuildExchange(shard.Comm(rank=0, world=1), p.n, 16, _lib.device())
    adj = torch.empty_like(a0)
    deg = torch.empty_like(d0)
    st = _lib.to_dev(starts.astype(np.int32))
    od = _lib.to_dev(order.astype(np.int32))
    _lib.call("pk_build_vamana_sharded", p.device(), p.n, p.dp, p.packed(), p.dw, p.mode, 16, 32, 1.2, st,
              st.shape[0], od, adj, deg, None, 0, 0, 1, 1, *ex.pointers(), _lib.stream())
    assert torch.equal(adj, a0) and torch.equal(deg, d0)


def _pipeline_digest(comm, case="c1"):
    """Sharded pipeline on this rank; returns digests of every output array.
    case "c5": a C5-shaped instance large enough for the tensor-core start
    pre-screen and the locality order of the build batches (rank 0's order is
    broadcast: PK_XCHG_ORDER), sharded batches of >= 2,048 points."""
    import hashlib

    import paper_2312_03940_b200 as pk
    from paper_2312_03940_b200 import _lib, workloads
    from paper_2312_03940_b200.cluster import run_pipeline_device

    torch.cuda.set_device(0)
    if case == "c5":
        data, _ = workloads.generate("C5", n=70_000, components=55)
        kw = workloads.pipeline_args("C5", pk, n_centers=55)
    else:
        data, _ = workloads.generate("C1", n=6000, components=10)
        kw = workloads.pipeline_args("C1", pk, n_centers=10)
    _lib.prof_collect(reset=True)
    _lib.prof_only([])
    _lib.prof_enable(True)
    out = run_pipeline_device(pk.PointSet(data), **kw, comm=comm)
    torch.cuda.synchronize()
    _lib.prof_enable(False)
    ran_locality = "locality_keys_kernel" in _lib.prof_collect(reset=True)
    adj, deg = out["index"].graph.device_arrays()[:2]
    ids, dists = out["ids"], out["dists"]
    if comm is not None:  # each rank holds only its own rows
        assert out["rows"] == comm.my_range(data.shape[0])
        ids, dists = comm.all_gather_rows(ids, data.shape[0]), comm.all_gather_rows(dists, data.shape[0])
    h = {}
    for name, t in (("adj", adj), ("deg", deg), ("ids", ids), ("dists", dists), ("rho", out["rho"]),
                    ("lam", out["lam"]), ("delta", out["delta"]), ("labels", out["labels"])):
        h[name] = hashlib.sha256(t.detach().cpu().numpy().tobytes()).hexdigest()
    h["locality_order_ran"] = ran_locality
    return h


def _pipeline_worker(rank, world, port, q, case="c1"):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        q.put((rank, _pipeline_digest(shard.Comm(), case)))
    except Exception:  # noqa: BLE001
        import traceback

        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["c1", "c5"])
def test_sharded_pipeline_matches_single_gpu(case):
    """Functional check of the split (not a measurement): two ranks sharing
    one device, host (gloo) collectives, must reproduce the single-process
    graph, kNN rows, densities, dependents and labels bit for bit."""
    ref = _pipeline_digest(None, case)
    assert ref["locality_order_ran"] == (case == "c5")
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_pipeline_worker, args=(r, 2, port, q, case)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, h = q.get(timeout=600)
        res[r] = h
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert isinstance(res[r], dict), res[r]
        assert res[r] == ref, (r, {k: (res[r][k] == ref[k]) for k in ref})
