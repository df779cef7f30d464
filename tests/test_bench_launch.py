"""bench.py's multi-rank launcher on CPU: `--gpus 2` outside torchrun relaunches itself
as 2 ranks; with --dry-run the ranks shard the workload, run the segment protocol (host
emulation of the kernels, gloo collectives) and rank 0 prints one line.  The
partitioned log-likelihood must equal the single-series oracle's."""
import json
import os
import subprocess
import sys

import numpy as np

import oracle_lib as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*extra):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--dry-run", *extra], capture_output=True,
                         text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    return json.loads(lines[0])


def test_two_rank_relaunch_cfg4_segments_match_oracle():
    line = _run("--gpus", "2", "--points", "3000")
    assert line["n_gpus"] == 2 and line["config"]["config"] == "cfg4"
    assert "contiguous time segments" in line["config"]["parallelism"]
    assert line["shard"] == [0, 1500]
    from paper_1610_08035_b200 import datasets
    wl = datasets.make("cfg4", n=3000)
    o = O.evaluate(wl.leaves, wl.theta, wl.t, wl.y, wl.sigma, grad=False, mean=False, var=False)
    ld = O.evaluate(wl.leaves, wl.theta, wl.t, wl.y, wl.sigma, grad=False, mean=False, var=False, precision=1)
    # cfg4 sits on its fp64 conditioning floor (4 of 6 eigenvalues of Q below the jitter,
    # SURVEY.md App. A): the fp64 oracle itself is ~6e-7 from the long-double run, so the
    # partitioned result must be as close to the long-double run as the fp64 oracle is
    floor = abs(o["loglik"] - ld["loglik"])
    assert abs(line["loglik"][0] - ld["loglik"]) <= max(1e-9 * abs(ld["loglik"]), 4 * floor)


def test_two_rank_relaunch_cfg3_shards_series():
    line = _run("--gpus", "2", "--config", "cfg3", "--points", "32")
    assert line["n_gpus"] == 2 and line["config"]["config"] == "cfg3"
    assert line["shard"] == [0, 2048]
    from paper_1610_08035_b200 import datasets
    wl = datasets.make("cfg3", n=32)
    # first two series of each rank's shard: 0, 1 (rank 0) and 2048, 2049 (rank 1)
    for k, s in enumerate([0, 1, 2048, 2049]):
        o = O.evaluate(wl.leaves, wl.theta[s], wl.t[s], wl.y[s], wl.sigma[s], grad=False, mean=False, var=False)
        assert abs(line["loglik"][k] - o["loglik"]) <= 1e-9 * abs(o["loglik"])


def test_single_rank_default_is_cfg2():
    line = _run("--points", "500")
    assert line["n_gpus"] == 1 and line["config"]["config"] == "cfg2"
    assert np.isfinite(line["loglik"][0])
