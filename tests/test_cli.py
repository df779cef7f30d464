"""The bench CLI (tools/cli/spingp): kernel grammar, deterministic data
generation, CSV/JSON reports, the host comparison methods (kf, dense) and, on the GPU,
fit / predict / the scaling sweeps with fitted slopes and the CO2-style pipeline on a
synthetic NOAA-format fixture (tests/golden/co2_weekly_fixture.txt, not measured data)."""
import csv
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "cli", "spingp")
FIX = os.path.join(ROOT, "tests", "golden", "co2_weekly_fixture.txt")


@pytest.fixture(scope="module")
def cli():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tools", "cli")], check=True)
    return CLI


def run(cli, *args, ok=True):
    r = subprocess.run([cli, *map(str, args)], capture_output=True, text=True, timeout=1800)
    if ok:
        assert r.returncode == 0, r.stderr[-3000:]
    return r


def rows(path):
    with open(path) as f:
        return list(csv.DictReader(f))


def test_gen_data_is_deterministic(cli, tmp_path):
    run(cli, "gen-data", "--n", 1000, "--seed", 7, "--out", tmp_path / "a")
    run(cli, "gen-data", "--n", 1000, "--seed", 7, "--out", tmp_path / "b")
    a = (tmp_path / "a" / "data.csv").read_bytes()
    assert a == (tmp_path / "b" / "data.csv").read_bytes()
    run(cli, "gen-data", "--n", 10000, "--seed", 7, "--noise", 0, "--out", tmp_path / "c")
    d = np.loadtxt(tmp_path / "c" / "data.csv", delimiter=",", skiprows=1)
    t = d[:, 0]
    assert np.allclose(d[:, 1], np.sin(2 * np.pi * 0.04 * t) + 0.6 * np.sin(2 * np.pi * 0.17 * t), atol=1e-12)


def test_noise_variance_law_of_large_numbers(cli, tmp_path):
    run(cli, "gen-data", "--n", 100000, "--seed", 3, "--out", tmp_path / "a")
    d = np.loadtxt(tmp_path / "a" / "data.csv", delimiter=",", skiprows=1)
    eta = d[:, 1] - (np.sin(2 * np.pi * 0.04 * d[:, 0]) + 0.6 * np.sin(2 * np.pi * 0.17 * d[:, 0]))
    assert abs(eta.var() - 0.04) < 0.05 * 0.04


def test_bad_kernel_expression_fails(cli, tmp_path):
    r = run(cli, "scaling-n", "--method", "kf", "--kernel", "matern33(len=1)", "--ns", "10", "--out", tmp_path,
            ok=False)
    assert r.returncode != 0 and "unknown kernel" in (r.stderr + (tmp_path / "report.csv").read_text())


def test_scaling_n_host_methods_report(cli, tmp_path):
    run(cli, "scaling-n", "--method", "kf,dense", "--kernel", "matern32(var=1, len=5) + matern12(len=2)",
        "--ns", "100,200,400", "--out", tmp_path)
    rs = rows(tmp_path / "report.csv")
    assert len(rs) == 3 * 2  # |sweep| x |methods|
    m = json.loads((tmp_path / "metrics.json").read_text())
    assert m["schema_version"] == 1 and np.isfinite(m["slopes"]["kf"]) and np.isfinite(m["slopes"]["dense"])
    by = {(r["method"], float(r["N"])): float(r["mll"]) for r in rs}
    for n in (100, 200, 400):  # cross-method equality audit at every cell
        assert by[("kf", n)] == pytest.approx(by[("dense", n)], rel=1e-6)


@pytest.mark.gpu
def test_fit_and_predict_on_gpu(cli, tmp_path):
    run(cli, "gen-data", "--n", 400, "--seed", 5, "--out", tmp_path)
    data = tmp_path / "data.csv"
    run(cli, "fit", "--kernel", "matern32(var=1, len=3)", "--data", data, "--budget", 50, "--out", tmp_path / "fit")
    m = json.loads((tmp_path / "fit" / "metrics.json").read_text())
    assert m["schema_version"] == 1 and np.isfinite(m["mll"]) and m["iterations"] >= 1
    run(cli, "predict", "--kernel", "matern32(var=1, len=3)", "--data", data, "--grid", "0:500:101", "--out",
        tmp_path / "p")
    f = np.loadtxt(tmp_path / "p" / "forecast.csv", delimiter=",", skiprows=1)
    assert f.shape == (101, 3) and np.all(f[:, 2] >= 0)


@pytest.mark.gpu
def test_scaling_sweeps_on_gpu(cli, tmp_path):
    """spingp vs kf at the SPEC sizes (b = 12), and the GPU's own linear
    regime (N = 1M..8M points, where it is throughput-bound): slope in [0.75, 1.3].
    The cross-method audit uses a b = 12 sum of Matérn leaves: with the CLI default
    (matern32 + eq(order=10)) the SPEC's jitter on the ill-conditioned EQ-10 process noise
    (cond(P_inf) ~ 1e12) moves the sparse-precision MLL away from the
    jitter-free Kalman filter by design."""
    k12 = "matern32(len=5) + matern52(len=3) + matern32(len=20) + matern52(len=8) + matern32(len=2)"
    run(cli, "scaling-n", "--method", "spingp,kf", "--kernel", k12, "--ns", "1000,2000,4000,8000", "--out",
        tmp_path / "n")
    rs = rows(tmp_path / "n" / "report.csv")
    assert len(rs) == 8 and all(r["error"] == "" for r in rs)
    by = {(r["method"], float(r["N"])): float(r["mll"]) for r in rs}
    for n in (1000, 2000, 4000, 8000):
        assert by[("spingp", n)] == pytest.approx(by[("kf", n)], rel=1e-6)
    run(cli, "scaling-n", "--method", "spingp", "--kernel", k12, "--ns", "1000000,2000000,4000000,8000000", "--out",
        tmp_path / "big")
    s = json.loads((tmp_path / "big" / "metrics.json").read_text())["slopes"]["spingp"]
    assert 0.75 <= s <= 1.3, s
    run(cli, "scaling-b", "--method", "spingp", "--bs", "4,8,16", "--n", 1000, "--out", tmp_path / "b")
    assert len(rows(tmp_path / "b" / "report.csv")) == 3


@pytest.mark.gpu
def test_co2_pipeline_on_fixture(cli, tmp_path):
    run(cli, "co2", "--data", FIX, "--budget", 60, "--out", tmp_path)
    m = json.loads((tmp_path / "metrics.json").read_text())
    n_rows = sum(1 for ln in open(FIX) if not ln.startswith("#"))
    assert m["rows"] == n_rows - 1  # the sentinel row is dropped
    assert m["heldout_rmse"] < m["constant_mean_rmse"]
    f = np.loadtxt(tmp_path / "forecast.csv", delimiter=",", skiprows=1)
    assert len(f) == m["heldout_rows"] + 8 * 52


def test_co2_ingest_rejects_comment_only_file(cli, tmp_path):
    p = tmp_path / "empty.txt"
    p.write_text("# nothing\n# here\n")
    r = run(cli, "co2", "--data", p, "--out", tmp_path / "o", ok=False)
    assert r.returncode != 0 and "NoValidRows" in r.stderr
