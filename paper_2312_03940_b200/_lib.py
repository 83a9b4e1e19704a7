"""ctypes binding of the C ABI in include/peakann_b200.h.

The product path has no CPU fallback: importing the kernels without a built
`libpeakann_b200.so` or without a CUDA device raises immediately.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpeakann_b200.so")

MODE_SEQ64 = 0
MODE_EXACT32 = 1
MODE_EXACT_U8 = 2

DENSITY_CODES = {"kth": 0, "kth_normalized": 1, "exp_sum": 2, "sum_exp": 3, "sum": 4}

_P = ctypes.c_void_p
_I = ctypes.c_int64
_i = ctypes.c_int
_D = ctypes.c_double

# host callback of the sharded build (pk_exchange_fn): (ctx, kind, a, b) -> int64
EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64)

# name -> argtypes (every entry returns int status)
SIGNATURES = {
    "pk_check_exact32": [_P, _I, _I, _I, _P, _P],
    "pk_pack_u8": [_P, _I, _I, _I, _P, _I, _P],
    "pk_beam_knn": [_P, _I, _I, _P, _I, _i, _P, _I, _P, _P, _I, _P, _I, _I, _I, _P, _P, _P, _i, _P, _i, _P],
    "pk_beam_knn_seeded": [_P, _I, _I, _P, _I, _i, _P, _I, _P, _P, _I, _P, _I, _I, _I, _P, _P, _P, _i, _P, _i,
                           _P, _P, _P, _P],
    "pk_beam_search_single": [_P, _I, _I, _P, _I, _P, _P, _I, _I, _P, _I, _I, _P, _P, _P, _P, _P, _I, _P, _P],
    "pk_brute_knn": [_P, _I, _I, _P, _I, _I, _P, _P, _P],
    "pk_brute_knn_vector": [_P, _I, _I, _P, _I, _P, _P, _P],
    "pk_brute_knn_tc": [_P, _I, _I, _P, _I, _I, _P, _P, _P, _P, _P],
    "pk_dp_scan_tc": [_P, _I, _I, _P, _P, _I, _P, _P, _P, _P, _P],
    "pk_build_vamana": [_P, _I, _I, _P, _I, _i, _I, _I, _D, _P, _I, _P, _P, _P, _P, _i, _P],
    "pk_build_vamana_seeds": [_P, _I, _I, _P, _I, _i, _I, _I, _D, _P, _I, _P, _P, _P, _P, _i, _P, _P, _P, _P],
    "pk_build_vamana_sharded": [_P, _I, _I, _P, _I, _i, _I, _I, _D, _P, _I, _P, _P, _P, _P, _i, _i, _i, _I,
                                EXCHANGE_FN, _P, _P, _P, _P, _P, _P, _P],
    "pk_pcg64_permutation": [_P, _i, ctypes.c_uint32, _I, _P, _P],
    "pk_find_nonfinite": [_P, _I, _P],
    "pk_parse_pecg": [_P, _I, _I, _I, _P, _P, _P],
    "pk_phase_timers": [_P, _i],
    "pk_phase_timers_build": [_P, _i],
    "pk_phase_timers_prune": [_P, _i],
    "pk_scan_points": [_P, _I, _I, _I, _P, _P],
    "pk_robust_prune": [_P, _I, _I, _I, _P, _P, _I, _P, _I, _D, _I, _P, _P, _P],
    "pk_nearest_to_centroid": [_P, _I, _I, _P, _P],
    "pk_sqrt": [_P, _I, _P, _P],
    "pk_densities": [_i, _P, _P, _I, _I, _P, _P],
    "pk_normalize_rho": [_P, _P, _I, _I, _P, _P],
    "pk_normalize_rho_rows": [_P, _P, _I, _I, _I, _P, _P],
    "pk_rank_order": [_P, _I, _P, _P, _P],
    "pk_resolve_lists": [_P, _P, _I, _P, _P, _I, _P, _P, _P, _P, _I, _P, _P, _P, _P],
    "pk_dp_scan": [_P, _I, _I, _P, _I, _i, _P, _P, _I, _P, _P, _P],
    "pk_count_below": [_P, _I, _I, _P, _I, _i, _P, _I, _P, _P, _P, _P],
    "pk_resolve_short": [_P, _I, _I, _P, _I, _i, _P, _P, _I, _I, _P, _P, _P, _P, _P],
    "pk_resolve_short_scanned": [_P, _I, _I, _P, _I, _i, _P, _I, _I, _P, _P, _P, _P, _P, _P, _P],
    "pk_tc_count_stats": [_P, _i],
    "pk_scatter_dependents": [_P, _I, _P, _P, _P, _P, _P],
    "pk_argmax_rank": [_P, _I, _P, _P],
    "pk_flag_noise": [_P, _I, _D, _P, _P, _P],
    "pk_centers_threshold": [_P, _P, _I, _D, _P, _P],
    "pk_centers_product": [_P, _P, _P, _I, _I, _P, _P],
    "pk_centers_local": [_P, _P, _I, _P, _I, _P, _P],
    "pk_promote_orphans": [_P, _P, _I, _P, _P],
    "pk_assign_clusters": [_P, _P, _P, _I, _P, _P, _P],
    "pk_flags_to_ids": [_P, _I, _P, _P, _P],
}

_lib = None


def build_library(force: bool = False) -> str:
    """Compile csrc/ for sm_100a (nvcc cross-compiles without a GPU)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", os.path.join(_HERE, "csrc")], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"peakann-b200 CUDA library not built ({LIB_PATH} missing); run __graft_entry__.build()"
            )
        L = ctypes.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        L.pk_last_error.restype = ctypes.c_char_p
        L.pk_version.restype = ctypes.c_int
        L.pk_device_info.argtypes = [ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
        L.pk_prof_enable.argtypes = [ctypes.c_int]
        L.pk_prof_enable.restype = None
        L.pk_prof_only.argtypes = [ctypes.c_char_p]
        L.pk_prof_only.restype = None
        L.pk_prof_collect.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int]
        L.pk_prof_collect.restype = ctypes.c_int
        _lib = L
    return _lib


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("peakann-b200 needs a CUDA device (B200 / sm_100a); no CPU fallback exists")


def call(name: str, *args) -> None:
    """Invoke a C-ABI entry point; raise RuntimeError on a nonzero status."""
    require_cuda()
    fn = getattr(lib(), name)
    conv = []
    for a in args:
        if isinstance(a, torch.Tensor):
            conv.append(ctypes.c_void_p(a.data_ptr()))
        elif a is None:
            conv.append(ctypes.c_void_p(0))
        else:
            conv.append(a)
    rc = fn(*conv)
    if rc != 0:
        msg = lib().pk_last_error().decode(errors="replace")
        raise RuntimeError(f"{name} failed ({rc}): {msg}")


def call_host(name: str, *args) -> None:
    """Invoke a host-only C-ABI helper (no device work, usable without a GPU)."""
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        raise RuntimeError(f"{name} failed ({rc})")


def stream() -> int:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def device() -> torch.device:
    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def to_dev(a: np.ndarray, dtype=None) -> torch.Tensor:
    t = torch.from_numpy(np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype)))
    return t.to(device(), non_blocking=False)


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def prof_enable(on: bool) -> None:
    lib().pk_prof_enable(1 if on else 0)


def prof_only(names) -> None:
    """Time only these kernels (iterable of names; empty = all)."""
    lib().pk_prof_only(",".join(names).encode())


def prof_collect(reset: bool = True) -> dict:
    """{kernel name: (launches, total device ms)} since the last reset."""
    buf = ctypes.create_string_buffer(1 << 16)
    lib().pk_prof_collect(buf, len(buf), 1 if reset else 0)
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms = line.split()
        out[name] = (int(cnt), float(ms))
    return out
