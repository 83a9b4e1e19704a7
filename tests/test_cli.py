"""The command-line front end (cli.py) against the reference's CLI contract
(/root/reference/pkg/tests/test_cli.py): key=value output, exit codes, state
dump / reapply.  score / gen and the usage errors run on the CPU; the pipeline
commands need the GPU."""
import subprocess
import sys

import numpy as np
import pytest

from conftest import FIG_COORDS, ROOT
import paper_2312_03940_b200 as pk  # noqa: E402
from paper_2312_03940_b200.cli import main  # noqa: E402
from paper_2312_03940_b200.data import read_labels, write_fvecs, write_labels  # noqa: E402


@pytest.fixture()
def fig_file(tmp_path):
    path = tmp_path / "fig.fvecs"
    write_fvecs(FIG_COORDS, path)
    return path


def run(argv):
    return main([str(a) for a in argv])


def parse_kv(capsys):
    out = capsys.readouterr().out
    return dict(line.partition("=")[::2] for line in out.strip().splitlines())


# ---- CPU: score, gen, usage errors --------------------------------------------------


def test_score_identical_and_minus_half(tmp_path, capsys):
    a, b = tmp_path / "a.txt", tmp_path / "b.txt"
    write_labels(np.array([0, 0, 1, 1]), a)
    write_labels(np.array([0, 1, 0, 1]), b)
    assert run(["score", a, a]) == 0
    assert parse_kv(capsys)["ari"] == "1.0"
    assert run(["score", a, b]) == 0
    kv = parse_kv(capsys)
    assert kv["ari"] == "-0.5"
    assert 0.0 <= float(kv["homogeneity"]) <= 1.0 and 0.0 <= float(kv["completeness"]) <= 1.0


def test_score_errors_exit_2(tmp_path):
    a, b = tmp_path / "a.txt", tmp_path / "b.txt"
    write_labels(np.array([0, 0, 1]), a)
    write_labels(np.array([0, 1]), b)
    for argv in (["score", a, b], ["score", a, tmp_path / "nope.txt"]):
        with pytest.raises(SystemExit) as exc:
            run(argv)
        assert exc.value.code == 2


def test_gen_writes_deterministic_files(tmp_path, capsys):
    p1, p2 = tmp_path / "d1", tmp_path / "d2"
    for p in (p1, p2):
        assert run(["gen", "--n", "60", "--c", "3", "--d", "8", "--seed", "1", "--out", p]) == 0
    kv = parse_kv(capsys)
    assert kv["labels"].endswith("d2.labels")
    pts = pk.read_vectors(f"{p1}.fvecs")
    assert (pts.n, pts.d) == (60, 8)
    assert read_labels(f"{p1}.labels").shape == (60,)
    assert (tmp_path / "d1.fvecs").read_bytes() == (tmp_path / "d2.fvecs").read_bytes()
    assert run(["gen", "--n", "20", "--c", "2", "--d", "4", "--format", "f32bin", "--out", tmp_path / "b"]) == 0
    assert pk.read_vectors(f"{tmp_path / 'b'}.f32bin").n == 20


@pytest.mark.parametrize("argv", [
    ["gen", "--n", "3", "--c", "5", "--out", "X"],
    ["cluster", "--input", "ABSENT", "--center", "product", "--nc", "2"],
    ["cluster", "--input", "FIG", "--center", "threshold"],
    ["cluster", "--input", "FIG", "--center", "product", "--nc", "2", "--k", "8", "--L", "4"],
    ["cluster", "--input", "FIG", "--center", "product", "--nc", "2", "--k", "4", "--Ld", "4"],
    ["exact", "--input", "FIG", "--center", "product", "--nc", "2", "--R", "16"],
    ["cluster", "--center", "product", "--nc", "2"],
])
def test_usage_errors_exit_2(argv, tmp_path, fig_file):
    argv = [str(tmp_path / "x") if a == "X" else str(tmp_path / "absent.fvecs") if a == "ABSENT"
            else str(fig_file) if a == "FIG" else a for a in argv]
    with pytest.raises(SystemExit) as exc:
        run(argv)
    assert exc.value.code == 2


def test_corrupt_input_exits_2(tmp_path):
    bad = tmp_path / "bad.fvecs"
    bad.write_bytes(b"\x02\x00\x00\x00\x00")
    assert run(["cluster", "--input", bad, "--center", "product", "--nc", "2"]) == 2


def test_module_entry_point(tmp_path):
    a = tmp_path / "a.txt"
    write_labels(np.array([0, 0, 1, 1]), a)
    out = subprocess.run([sys.executable, "-m", "paper_2312_03940_b200", "score", str(a), str(a)], cwd=ROOT,
                         capture_output=True, text=True, check=True).stdout
    assert "ari=1.0" in out


# ---- GPU: the pipeline commands ------------------------------------------------------


@pytest.mark.gpu
def test_figure_threshold_run(fig_file, tmp_path, capsys):
    out = tmp_path / "labels.txt"
    assert run(["cluster", "--input", fig_file, "--index", "bruteforce", "--k", "1", "--density", "kth",
                "--center", "threshold", "--delta-min", "2.5", "--rho-min", "0.70710678", "--output", out]) == 0
    assert list(read_labels(out)) == [1, 1, 1, 3, 4, 3]
    kv = parse_kv(capsys)
    assert kv["n_clusters"] == "3" and kv["n_noise"] == "1"
    for key in ("stage_index_s", "stage_unionfind_pct", "total_s"):
        assert key in kv


@pytest.mark.gpu
def test_vamana_run_prints_metrics(tmp_path, capsys):
    pts, labels = pk.generate_gaussian(pk.GaussianSpec(n=400, c=4, d=128, seed=2))
    vec, truth = tmp_path / "g.fvecs", tmp_path / "g.labels"
    write_fvecs(pts, vec)
    write_labels(labels, truth)
    assert run(["cluster", "--input", vec, "--index", "vamana", "--k", "8", "--L", "16", "--Ld", "16", "--R", "16",
                "--alpha", "1.1", "--center", "product", "--nc", "4", "--truth", truth, "--seed", "7"]) == 0
    kv = parse_kv(capsys)
    assert float(kv["ari"]) > 0.99


@pytest.mark.gpu
def test_state_dump_reapply_and_exact(tmp_path):
    pts, _ = pk.generate_gaussian(pk.GaussianSpec(n=200, c=4, d=8, seed=5))
    vec = tmp_path / "s.fvecs"
    write_fvecs(pts, vec)
    state, full = tmp_path / "state.npz", tmp_path / "full.txt"
    assert run(["cluster", "--input", vec, "--index", "bruteforce", "--k", "4", "--center", "product", "--nc", "4",
                "--state-out", state, "--output", full]) == 0
    re2, same = tmp_path / "re.txt", tmp_path / "same.txt"
    assert run(["cluster", "--state-in", state, "--center", "product", "--nc", "2", "--output", re2]) == 0
    assert len(np.unique(read_labels(re2))) == 2
    assert run(["cluster", "--state-in", state, "--center", "product", "--nc", "4", "--output", same]) == 0
    assert np.array_equal(read_labels(same), read_labels(full))
    a, b = tmp_path / "a.txt", tmp_path / "b.txt"
    assert run(["exact", "--input", vec, "--k", "4", "--center", "product", "--nc", "3", "--output", a]) == 0
    assert run(["cluster", "--input", vec, "--index", "bruteforce", "--k", "4", "--threshold", "0",
                "--center", "product", "--nc", "3", "--output", b]) == 0
    assert np.array_equal(read_labels(a), read_labels(b))
