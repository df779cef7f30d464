"""Multi-GPU inside the library (spingp_mctx_create + spingp_eval_partitioned): one long
series partitioned over the devices of a box with NCCL collectives enqueued by the C++
host code.  P = 1 always runs (the pool's boxes have one GPU); P = 2..8 when present."""
import numpy as np
import pytest

import oracle_lib as O
import paper_1610_08035_b200 as P
from conftest import rel

pytestmark = pytest.mark.gpu


def _series(n, seed=3):
    rng = np.random.default_rng(seed)
    t = np.cumsum(rng.uniform(0.05, 0.15, n))
    return t, np.sin(0.5 * t) + 0.3 * rng.standard_normal(n)


def _ndev():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("leaves,theta", [([P.MATERN52], [2.0, 1.5]), ([P.MATERN32, (P.QP, 6)], [1.0, 10.0, 1.0, 1.0, 1.0, 20.0])])
def test_partitioned_one_device_equals_single_context(ctx, leaves, theta):
    t, y = _series(20_000)
    with P.MultiContext([0]) as m:
        a = m.eval(leaves, theta, t, y, 0.3, grad=True, mean=True, var=True)
    b = ctx.eval(leaves, theta, t, y, 0.3, grad=True, mean=True, var=True)
    assert rel(a["loglik"], b["loglik"]) < 1e-12 and rel(a["grad"], b["grad"]) < 1e-10
    assert rel(a["mean"], b["mean"]) < 1e-10 and rel(a["var"], b["var"]) < 1e-10


@pytest.mark.parametrize("ndev", [2, 4, 8])
def test_partitioned_over_devices_matches_oracle(ndev):
    if _ndev() < ndev:
        pytest.skip(f"{ndev} GPUs needed, {_ndev()} present")
    t, y = _series(50_000)
    with P.MultiContext(list(range(ndev))) as m:
        a = m.eval([P.MATERN52], [2.0, 1.5], t, y, 0.3, grad=True, mean=True, var=True)
    o = O.evaluate([P.MATERN52], [2.0, 1.5], t, y, 0.3, threads=16)
    for k in ("loglik", "grad", "mean", "var"):
        assert rel(a[k], o[k]) < 1e-9, k
