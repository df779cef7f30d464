"""The multi-rank path on CPU: world_size 2 over torch.distributed gloo, each rank
running the device algorithm (host emulation) on its own time segment and exchanging
the 2-separator records (all_gather) and the partial sums (all_reduce) exactly as the
GPU ranks do over NCCL (paper_1610_08035_b200/partition.py)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle_lib as O


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, leaves, theta, t, y, sigma, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import emu_lib as E
        from paper_1610_08035_b200.partition import split, halos
        bounds = split(len(t), world)
        a, b = bounds[rank], bounds[rank + 1]
        tl, tr = halos(t, bounds, rank)
        nrec, npart = E.seg_sizes(leaves)
        rec = torch.from_numpy(E.seg_forward(leaves, theta, t[a:b], y[a:b], tl, tr, rank, world, sigma, flags=7))
        recs = [torch.zeros(nrec, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(recs, rec)
        part, mu, v = E.seg_reverse(torch.cat(recs).numpy(), b - a, npart, mean=True, var=True)
        tp = torch.from_numpy(part)
        dist.all_reduce(tp)
        ll, g = E.seg_finalize(tp.numpy(), len(theta), len(t), sigma)
        out[rank] = (ll, g.tolist(), (a, b), mu.tolist(), v.tolist())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("leaves,theta", [([O.MATERN52], [2.0, 1.5]), ([O.MATERN32, O.MATERN12], [1.0, 0.7, 0.5, 2.0])])
def test_two_ranks_gloo_match_single_series_oracle(leaves, theta):
    rng = np.random.default_rng(5)
    n = 600
    t = np.cumsum(rng.uniform(0.05, 0.15, n))
    y = np.sin(0.5 * t) + 0.3 * rng.standard_normal(n)
    mgr = mp.get_context("spawn").Manager()  # a forked manager can deadlock on inherited thread pools
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), leaves, theta, t, y, 0.3, out), nprocs=2, join=True)
    o = O.evaluate(leaves, theta, t, y, 0.3)
    mean = np.zeros(n)
    var = np.zeros(n)
    for r in range(2):
        ll, g, (a, b), mu, v = out[r]
        assert abs(ll - o["loglik"]) <= 1e-10 * abs(o["loglik"])      # every rank holds the same result
        assert np.abs(np.array(g) - o["grad"]).max() <= 1e-9 * np.abs(o["grad"]).max()
        mean[a:b], var[a:b] = mu, v
    assert np.abs(mean - o["mean"]).max() <= 1e-9 * np.abs(o["mean"]).max()
    assert np.abs(var - o["var"]).max() <= 1e-9 * np.abs(o["var"]).max()
