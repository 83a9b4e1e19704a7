"""Golden vectors for the data module, produced by the reference itself
(run here, where /root/reference exists):

    python tests/golden/make_data_golden.py

* generate_gaussian(GaussianSpec(...)) for several specs: sha256 of the points
  and labels plus the first rows;
* the exact error message of each malformed vector / label file case.
"""
import hashlib
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from refload import load_reference  # noqa: E402

SPECS = [(1000, 7, 16, 0.05, 42), (513, 1, 3, 0.3, 0), (2048, 64, 128, 0.05, 7), (10, 10, 5, 1.0, 123)]


def sha(a):
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest()


def bad_files(tmp):
    """(name, bytes, reader) cases; the reader's error text is recorded."""
    rng = np.random.default_rng(1)
    good = rng.normal(size=(5, 3)).astype("<f4")
    fv = np.empty((5, 4), "<i4")
    fv[:, 0] = 3
    fv[:, 1:] = good.view("<i4")
    cases = {
        "empty.fvecs": b"",
        "odd.fvecs": fv.tobytes()[:-2],
        "trunc.fvecs": fv.tobytes()[:-4],
        "zerodim.fvecs": np.array([0, 1, 2], "<i4").tobytes(),
        "mixed.fvecs": np.concatenate([fv.ravel(), np.array([2, 0, 0], "<i4")]).tobytes() + b"\0" * 4,
        "nan.fvecs": None,
        "short.f32bin": b"\1\0\0",
        "zero.f32bin": np.array([0, 3], "<u4").tobytes(),
        "size.f32bin": np.array([5, 3], "<u4").tobytes() + good.tobytes()[:-4],
        "inf.f32bin": None,
        "bad.labels": b"1\n2\n\nx3\n",
        "ext.txt": good.tobytes(),
    }
    nanv = good.copy()
    nanv[3, 2] = np.nan
    fvn = fv.copy()
    fvn[:, 1:] = nanv.view("<i4")
    cases["nan.fvecs"] = fvn.tobytes()
    infv = good.copy()
    infv[1, 0] = -np.inf
    cases["inf.f32bin"] = np.array([5, 3], "<u4").tobytes() + infv.tobytes()
    out = {}
    for name, blob in cases.items():
        p = os.path.join(tmp, name)
        with open(p, "wb") as f:
            f.write(blob)
        out[name] = p
    return out


def main():
    ref = load_reference()
    data = {}
    for i, (n, c, d, var, seed) in enumerate(SPECS):
        pts, lab = ref.generate_gaussian(ref.GaussianSpec(n=n, c=c, d=d, variance=var, seed=seed))
        data[f"g{i}__spec"] = np.array([n, c, d, seed], np.int64)
        data[f"g{i}__var"] = np.array([var])
        data[f"g{i}__sha_points"] = np.array(sha(pts.data))
        data[f"g{i}__sha_labels"] = np.array(sha(lab))
        data[f"g{i}__head"] = pts.data[:4]
    rng = np.random.default_rng(11)
    for i in range(6):
        n = int(rng.integers(2, 3000))
        a = rng.integers(0, int(rng.integers(1, 40)), n) * 3 - 7
        b = rng.integers(0, int(rng.integers(1, 40)), n)
        ct = ref.contingency(a, b)
        h, c = ref.homogeneity_completeness(a, b)
        data[f"m{i}__a"] = a
        data[f"m{i}__b"] = b
        data[f"m{i}__ari"] = np.array([ref.ari(a, b)])
        data[f"m{i}__hc"] = np.array([h, c])
        for f in ("rows", "cols", "counts", "row_sums", "col_sums"):
            data[f"m{i}__{f}"] = getattr(ct, f)
    with tempfile.TemporaryDirectory() as tmp:
        files = bad_files(tmp)
        for name, p in files.items():
            try:
                if name.endswith(".labels"):
                    ref.read_labels(p)
                else:
                    ref.read_vectors(p)
                msg = "OK"
            except Exception as e:  # noqa: BLE001
                msg = f"{type(e).__name__}: {str(e).replace(tmp, '<dir>')}"
            data[f"err__{name}"] = np.array(msg)
    np.savez_compressed(os.path.join(HERE, "data.npz"), **data)
    print("wrote data.npz", len(data))


if __name__ == "__main__":
    main()
