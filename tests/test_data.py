"""Data module (vector / label files, the reference's generator) against
golden outputs of the reference itself (tests/golden/make_data_golden.py)."""

import hashlib
import json
import os
import sys

import numpy as np
import pytest

from conftest import ROOT, golden

sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import paper_2312_03940_b200 as pk  # noqa: E402
from make_data_golden import bad_files  # noqa: E402  (pure file builder, no reference import)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_reference_names_exported():
    for name in ("DataFormatError", "read_vectors", "read_labels", "write_clustering", "GaussianSpec",
                 "generate_gaussian"):
        assert hasattr(pk, name)
    assert issubclass(pk.DataFormatError, ValueError)


def test_generate_gaussian_bit_identical_to_reference():
    z = golden("data")
    for i in range(4):
        n, c, d, seed = (int(v) for v in z[f"g{i}__spec"])
        var = float(z[f"g{i}__var"][0])
        p, lab = pk.generate_gaussian(pk.GaussianSpec(n=n, c=c, d=d, variance=var, seed=seed))
        assert p.data.dtype == np.float32 and p.data.shape == (n, d)
        assert np.array_equal(p.data[:4], z[f"g{i}__head"])
        assert sha(p.data) == str(z[f"g{i}__sha_points"])
        assert sha(lab) == str(z[f"g{i}__sha_labels"])
    with pytest.raises(ValueError):
        pk.generate_gaussian(pk.GaussianSpec(n=3, c=4))
    with pytest.raises(ValueError):
        pk.generate_gaussian(pk.GaussianSpec(n=3, c=0))
    with pytest.raises(ValueError):
        pk.generate_gaussian(pk.GaussianSpec(n=3, c=1, d=0))


def test_malformed_files_raise_the_reference_errors(tmp_path):
    z = golden("data")
    files = bad_files(str(tmp_path))
    for name, path in files.items():
        try:
            if name.endswith(".labels"):
                pk.read_labels(path)
            else:
                pk.read_vectors(path)
            got = "OK"
        except Exception as e:  # noqa: BLE001
            got = f"{type(e).__name__}: {str(e).replace(str(tmp_path), '<dir>')}"
        assert got == str(z[f"err__{name}"]), name


def test_round_trips(tmp_path):
    from paper_2312_03940_b200 import data

    x = np.random.default_rng(3).normal(size=(37, 11)).astype(np.float32)
    for fmt, writer in (("fvecs", data.write_fvecs), ("f32bin", data.write_f32bin)):
        path = str(tmp_path / f"x.{fmt}")
        writer(x, path)
        p = pk.read_vectors(path)
        assert np.array_equal(p.data, x)
        assert np.array_equal(pk.read_vectors(path, fmt).data, x)
    lab = np.array([3, -1, 0, 7], np.int64)
    data.write_labels(lab, str(tmp_path / "l.txt"))
    assert np.array_equal(pk.read_labels(str(tmp_path / "l.txt")), lab)
    cl = pk.Clustering(lab, np.array([0, 3], np.int64), np.array([1], np.int64))
    pk.write_clustering(cl, str(tmp_path / "c.txt"), sidecar=str(tmp_path / "c.json"))
    assert np.array_equal(pk.read_labels(str(tmp_path / "c.txt")), lab)
    assert json.load(open(tmp_path / "c.json")) == {"centers": [0, 3], "noise": [1]}
    with pytest.raises(ValueError):
        pk.read_vectors(str(tmp_path / "x.fvecs"), "npy")


def test_metrics_bit_identical_to_reference():
    from paper_2312_03940_b200 import metrics

    z = golden("data")
    for i in range(6):
        a, b = z[f"m{i}__a"], z[f"m{i}__b"]
        ct = metrics.contingency(a, b)
        for f in ("rows", "cols", "counts", "row_sums", "col_sums"):
            assert np.array_equal(getattr(ct, f), z[f"m{i}__{f}"]), (i, f)
        assert ct.n == a.shape[0]
        assert pk.ari(a, b) == float(z[f"m{i}__ari"][0])
        assert pk.homogeneity_completeness(a, b) == tuple(float(v) for v in z[f"m{i}__hc"])
    assert pk.ari([0, 0, 1, 1], [0, 1, 0, 1]) == -0.5
    with pytest.raises(ValueError):
        metrics.contingency([], [])
    with pytest.raises(ValueError):
        pk.ari([1], [1])
