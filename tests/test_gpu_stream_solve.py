"""The streaming cr_solve kernels (b <= 4, at most one right-hand side): the strip kernel
(csrc/strip_solve.cuh, one lane per long chunk; n >= 2 sub-tiles per lane of one CTA) and the
tile kernel (csrc/stream_solve.cuh, contiguous warp tiles; SPINGP_SOLVE_STRIP=0 or smaller n)
against the CPU oracle's block Thomas and against the partitioned
kernels they replace on that path."""
import os

import numpy as np
import pytest

import paper_1610_08035_b200 as P
import oracle_lib as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    with P.Context(0) as c:
        yield c


def rel(a, b):
    a, b = np.asarray(a, float).ravel(), np.asarray(b, float).ravel()
    assert a.shape == b.shape
    return float(np.max(np.abs(a - b)) / max(1e-300, np.max(np.abs(b))))


def system(n, b, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, b, b))
    diag = np.einsum("nij,nkj->nik", A, A) + 4 * b * np.eye(b)
    upper = rng.standard_normal((n - 1, b, b)) * (0.5 if b == 1 else 1.0)
    rhs = rng.standard_normal(n * b)
    return diag, upper, rhs


@pytest.fixture(params=["strip", "tile"])
def kernel(request):
    """Selects the streaming kernel: the strip kernel is tried first unless disabled."""
    if request.param == "tile":
        os.environ["SPINGP_SOLVE_STRIP"] = "0"
    yield request.param
    os.environ.pop("SPINGP_SOLVE_STRIP", None)


def launches(ctx, fn):
    k0 = ctx.launch_count()
    out = fn()
    return out, ctx.launch_count() - k0


# tile kernel: tile = 32 lanes x M blocks (b = 1: 224, b = 2, 3: 160, b = 4: 96), 8 warps per
# CTA; strip kernel: 256 lanes per CTA, sub-tiles of 8 / 4 / 4 / 2 blocks per lane, from
# 4096 / 2048 / 2048 / 1024 blocks (smaller n falls through to the tile kernel).  The sizes
# cover one CTA, ragged ends (odd and even remainders), several CTAs and sub-tiles.
@pytest.mark.parametrize("n,b", [(1792, 1), (1793, 1), (4096, 1), (30001, 1), (1280, 2), (1283, 2), (2049, 2),
                                 (25000, 2), (1280, 3), (1281, 3), (1282, 3), (1439, 3), (1441, 3), (2048, 3),
                                 (2049, 3), (2051, 3), (4801, 3), (60000, 3), (200001, 3), (768, 4), (769, 4),
                                 (1025, 4), (20001, 4)])
def test_stream_solve_matches_oracle(ctx, kernel, n, b):
    diag, upper, rhs = system(n, b, n + 7 * b)
    (x, ld), nl = launches(ctx, lambda: ctx.btd_cr_solve(diag, upper, rhs))
    assert nl == 1, "the streaming solve is one kernel launch"
    xo, ldo = O.btd_solve(diag, upper, rhs)
    assert rel(x, xo) < 1e-12 and abs(ld - ldo) <= 1e-12 * abs(ldo)
    (_, ld0), nl = launches(ctx, lambda: ctx.btd_cr_solve(diag, upper))  # log det only: sweep 1 + top
    assert nl == 1 and abs(ld0 - ldo) <= 1e-12 * abs(ldo)


def test_stream_solve_equals_partitioned_path(ctx, kernel):
    n, b = 50000, 3
    diag, upper, rhs = system(n, b, 5)
    x, ld = ctx.btd_cr_solve(diag, upper, rhs)
    os.environ["SPINGP_SOLVE_STREAM"] = "0"
    try:
        (xp, ldp), nl = launches(ctx, lambda: ctx.btd_cr_solve(diag, upper, rhs))
    finally:
        del os.environ["SPINGP_SOLVE_STREAM"]
    assert nl > 1
    assert rel(x, xp) < 1e-13 and abs(ld - ldp) <= 1e-13 * abs(ldp)


def test_stream_solve_below_threshold_and_multi_rhs_use_partitioned_kernels(ctx):
    diag, upper, rhs = system(600, 3, 1)  # fewer than 8 warp tiles
    (x, _), nl = launches(ctx, lambda: ctx.btd_cr_solve(diag, upper, rhs))
    assert nl > 1 and rel(x, O.btd_solve(diag, upper, rhs)[0]) < 1e-12
    diag, upper, _ = system(5000, 3, 2)
    rhs = np.random.default_rng(3).standard_normal((5000 * 3, 2))
    (x, _), nl = launches(ctx, lambda: ctx.btd_cr_solve(diag, upper, rhs))
    assert nl > 1 and rel(x, O.btd_solve(diag, upper, rhs)[0]) < 1e-12


# a non-positive-definite block inside a lane chunk and at the lane, tile / warp, run and CTA
# boundaries of both kernels (n = 4801: tile kernel 160-block tiles, 3 CTAs of 10 tiles; strip
# kernel 10 blocks per lane, 2 CTAs of 2560 blocks)
@pytest.mark.parametrize("bad", [0, 7, 9, 159, 164, 319, 1599, 2559, 3333, 4800])
def test_stream_solve_reports_the_failing_block(ctx, kernel, bad):
    n, b = 4801, 3
    diag, upper, rhs = system(n, b, 11)
    diag[bad] = -np.eye(b)
    with pytest.raises(P.NotPositiveDefinite) as e:
        ctx.btd_cr_solve(diag, upper, rhs)
    assert e.value.block_index() == bad
    # the context is usable afterwards (the grid barrier's counters stayed consistent)
    diag, upper, rhs = system(n, b, 12)
    x, _ = ctx.btd_cr_solve(diag, upper, rhs)
    assert rel(x, O.btd_solve(diag, upper, rhs)[0]) < 1e-12


def test_stream_solve_device_pointers_any_alignment(ctx, kernel):
    torch = pytest.importorskip("torch")
    n, b = 3201, 3
    diag, upper, rhs = system(n, b, 21)
    xo, ldo = O.btd_solve(diag, upper, rhs)
    dev = torch.device("cuda", 0)
    for off in (0, 1):  # 1: every array 8 bytes off a 16-byte boundary (no bulk copies)
        def put(v):
            buf = torch.empty(v.size + 2, device=dev, dtype=torch.float64)
            buf[off:off + v.size].copy_(torch.from_numpy(np.ascontiguousarray(v).ravel()))
            return buf[off:off + v.size]
        d, u, r = put(diag), put(upper), put(rhs)
        x = torch.full((n * b + 2,), float("nan"), device=dev, dtype=torch.float64)[off:off + n * b]
        ld = torch.zeros(1, device=dev, dtype=torch.float64)
        torch.cuda.synchronize()
        ctx.btd_cr_solve_device(n, b, d.data_ptr(), u.data_ptr(), r.data_ptr(), 1, x.data_ptr(), ld.data_ptr())
        ctx.status()  # synchronises the context stream, raises on a device-side failure
        assert rel(x.cpu().numpy(), xo) < 1e-12 and abs(float(ld.item()) - ldo) <= 1e-12 * abs(ldo)


@pytest.mark.parametrize("b", [3, 6])
@pytest.mark.parametrize("bad", [0, 13, 14, 3333, 4800])
def test_partitioned_kernels_report_the_failing_block(ctx, b, bad):
    """The same contract on the partitioned kernels: cr_solve with several
    right-hand sides and selective_inverse."""
    n = 4801
    diag, upper, _ = system(n, b, 31)
    rhs = np.random.default_rng(4).standard_normal((n * b, 2))
    diag[bad] = -np.eye(b)
    with pytest.raises(P.NotPositiveDefinite) as e:
        ctx.btd_cr_solve(diag, upper, rhs)
    assert e.value.block_index() == bad
    with pytest.raises(P.NotPositiveDefinite) as e:
        ctx.btd_selinv(diag, upper)
    assert e.value.block_index() == bad
