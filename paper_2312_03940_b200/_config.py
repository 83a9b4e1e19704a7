"""Worker-count API of the reference (_config.py:11-27).

The reference caps numba's CPU worker pool; the GPU build has no CPU pool,
so these keep the reference's signatures and validation and only record the
requested value (results never depend on it, as in the reference).
"""

_threads = 1


def set_num_threads(n: int) -> int:
    """Set the worker count; returns the effective value (always n here)."""
    global _threads
    if n < 1:
        raise ValueError(f"thread count must be >= 1, got {n}")
    _threads = int(n)
    return _threads


def get_num_threads() -> int:
    return _threads


def max_num_threads() -> int:
    import os

    return os.cpu_count() or 1
