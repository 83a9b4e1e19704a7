"""Seeded synthetic stand-ins for the BASELINE.json configurations.

None of the paper's datasets are available offline, so each
configuration is generated from `numpy.random.default_rng(seed)` with the
shapes, sizes and value distributions BASELINE.json names:

* C1  n=10,000    d=128  10-component Gaussian mixture, centers N(0, 4I), sigma 1
* C2  n=100,000   d=128  SIFT-shaped: clip(round(N(mu_c, 20^2)), 0, 255), 100 means
* C3  n=1,000,000 d=128  same generator, 1,000 means
* C4  n=1,000,000 d=384  5,000-component mixture, Zipf(1.1) weights, sigma 0.3, L2-normalised
* C5  n=1,281,167 d=1024 1,000-component mixture, sigma 0.5, L2-normalised

`pipeline_args(name)` returns the run_pipeline keyword arguments for each
configuration (index config, k, density kind, policies, doubling params).
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

__all__ = ["Workload", "WORKLOADS", "generate", "pipeline_args"]


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    d: int
    R: int
    L: int
    alpha: float
    k: int
    density: str
    n_centers: int
    components: int


WORKLOADS = {
    "C1": Workload("C1", 10_000, 128, 32, 64, 1.2, 16, "kth", 10, 10),
    "C2": Workload("C2", 100_000, 128, 64, 128, 1.1, 16, "kth_normalized", 100, 100),
    "C3": Workload("C3", 1_000_000, 128, 64, 128, 1.1, 32, "exp_sum", 1000, 1000),
    "C4": Workload("C4", 1_000_000, 384, 64, 128, 1.1, 16, "kth", 5000, 5000),
    "C5": Workload("C5", 1_281_167, 1024, 64, 200, 1.1, 16, "kth", 1000, 1000),
}


def _gauss_mixture(rng, n, d, comps, center_scale, sigma, weights=None, seed=0, normalise=False, chunk=65536):
    """means ~ N(0, center_scale^2 I), labels from `rng`; the noise of chunk c
    comes from its own stream default_rng([seed, 0x5EED, c]) in float32, so
    the chunks are drawn (and L2-normalised) on all host threads in parallel
    -- the 1.3 G coordinates of C5 in seconds instead of a minute."""
    from concurrent.futures import ThreadPoolExecutor

    means = rng.normal(0.0, center_scale, (comps, d)).astype(np.float32)
    if weights is None:
        labels = rng.integers(0, comps, n)
    else:
        labels = rng.choice(comps, size=n, p=weights)
    out = np.empty((n, d), np.float32)

    def fill(c):
        lo, hi = c * chunk, min(n, (c + 1) * chunk)
        x = np.random.default_rng([seed, 0x5EED, c]).standard_normal((hi - lo, d), dtype=np.float32)
        x *= np.float32(sigma)
        x += means[labels[lo:hi]]
        if normalise:
            nrm = np.sqrt(np.einsum("ij,ij->i", x, x, dtype=np.float64))
            x /= nrm.astype(np.float32)[:, None]
        out[lo:hi] = x

    chunks = (n + chunk - 1) // chunk
    with ThreadPoolExecutor(max_workers=min(chunks, os.cpu_count() or 1) or 1) as ex:
        list(ex.map(fill, range(chunks)))
    return out, labels.astype(np.int64)


def _sift_shaped(rng, n, d, comps, chunk=131072):
    mu = rng.uniform(0.0, 255.0, (comps, d))
    labels = rng.integers(0, comps, n)
    out = np.empty((n, d), np.float32)
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        out[lo:hi] = np.clip(np.round(rng.normal(mu[labels[lo:hi]], 20.0)), 0, 255)
    return out, labels.astype(np.int64)


def generate(name: str, n: int | None = None, seed: int = 0, components: int | None = None):
    """(points float32 (n, d), labels int64 (n,)) for a named configuration.

    `n` and `components` may be overridden to get a reduced-size instance with
    the same generator (used by parity tests and the bounded CPU sample).
    """
    w = WORKLOADS[name]
    n = w.n if n is None else int(n)
    comps = w.components if components is None else int(components)
    rng = np.random.default_rng(seed)
    if name == "C1":
        centers = rng.normal(0.0, 2.0, (comps, w.d))
        labels = rng.integers(0, comps, n)
        x = (centers[labels] + rng.normal(0.0, 1.0, (n, w.d))).astype(np.float32)
        return x, labels.astype(np.int64)
    if name in ("C2", "C3"):
        return _sift_shaped(rng, n, w.d, comps)
    if name == "C4":
        wts = (np.arange(comps) + 1.0) ** -1.1
        wts /= wts.sum()
        return _gauss_mixture(rng, n, w.d, comps, 1.0, 0.3, wts, seed=seed, normalise=True)
    if name == "C5":
        return _gauss_mixture(rng, n, w.d, comps, 1.0, 0.5, seed=seed, normalise=True)
    raise KeyError(name)


def pipeline_args(name: str, pk, n_centers: int | None = None, seed: int = 0, brute: bool = False):
    """run_pipeline(**kwargs) for a configuration, built from module `pk`
    (this package, or the reference loaded under another name)."""
    w = WORKLOADS[name]
    if brute:
        index = pk.BruteForceConfig()
        dp = pk.DoublingParams(initial_k=2 * w.k, threshold=0)
    else:
        index = pk.VamanaConfig(R=w.R, L_build=w.L, L=w.L, alpha=w.alpha, seed=seed)
        dp = pk.DoublingParams(initial_k=2 * w.k, threshold=300)
    return dict(
        index_config=index,
        k=w.k,
        density_kind=w.density,
        center_policy=pk.ProductCenter(w.n_centers if n_centers is None else n_centers),
        noise_policy=pk.NoisePolicy(0.0),
        doubling_params=dp,
    )
