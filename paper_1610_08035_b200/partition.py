"""Host orchestration of the multi-GPU partition of one long series.

Rank r of P owns a contiguous time segment; the data path per evaluation is

    seg_forward  (device: reduce the segment to its 2-separator Schur record)
    all_gather   (P records of 3b²+2b+1 doubles — NCCL over NVLink, ~1-6 KB/rank)
    seg_reverse  (device: solve the P-block reduced system redundantly, back-substitute,
                  selected inverse, gradient terms -> partial sums)
    all_reduce   (5 + n_theta doubles)
    seg_finalize (device: loglik, gradient)

The collectives are passed in, so the same code runs with torch.distributed (NCCL on
the GPU box, gloo in the CPU tests) or with an in-process emulation of the ranks.
"""
import math

import numpy as np


def split(n, P):
    """Contiguous, balanced segment bounds [b_r, b_{r+1}) for P ranks."""
    if P < 1 or n < P:
        raise ValueError("need at least one point per rank")
    return [int(round(k * n / P)) for k in range(P + 1)]


def halos(t, bounds, rank):
    """(t_left, t_right) halo times of `rank`: the neighbours' adjacent times (NaN at the ends)."""
    P = len(bounds) - 1
    a, b = bounds[rank], bounds[rank + 1]
    tl = float(t[a - 1]) if rank > 0 else math.nan
    tr = float(t[b]) if rank < P - 1 else math.nan
    return tl, tr


def eval_partitioned(ctx, leaves, theta, d_t, d_y, n_local, n_total, t_left, t_right, rank, nranks, sigma, flags,
                     buffers, all_gather, all_reduce, d_mean=0, d_var=0):
    """One distributed evaluation on this rank.

    buffers: dict of device tensors 'record' [nrec], 'records' [P*nrec], 'partials' [npart],
             'loglik' [1], 'grad' [n_theta+1]  (torch tensors; data_ptr() is passed to the ABI)
    all_gather(out, inp) / all_reduce(t): the collectives (e.g. torch.distributed).
    """
    ctx.seg_forward_device(leaves, theta, d_t, d_y, n_local, t_left, t_right, rank, nranks, sigma, flags,
                           buffers["record"].data_ptr())
    all_gather(buffers["records"], buffers["record"])
    ctx.seg_reverse_device(leaves, theta, d_t, d_y, n_local, t_left, t_right, rank, nranks, sigma, flags,
                           buffers["records"].data_ptr(), buffers["partials"].data_ptr(), d_mean, d_var)
    all_reduce(buffers["partials"])
    ctx.seg_finalize_device(len(theta), n_total, sigma, flags, buffers["partials"].data_ptr(),
                            buffers["loglik"].data_ptr(), buffers["grad"].data_ptr())


def make_buffers(torch, device, leaves, nranks):
    from . import seg_sizes, n_theta
    nrec, npart = seg_sizes(leaves)
    f64 = torch.float64
    return {"record": torch.zeros(nrec, dtype=f64, device=device),
            "records": torch.zeros(nranks * nrec, dtype=f64, device=device),
            "partials": torch.zeros(npart, dtype=f64, device=device),
            "loglik": torch.zeros(1, dtype=f64, device=device),
            "grad": torch.zeros(n_theta(leaves) + 1, dtype=f64, device=device)}


def emulate_ranks(ctx, torch, device, leaves, theta, t, y, sigma, flags, nranks):
    """Run the P-rank protocol sequentially on one GPU (exchange done in-process).
    The library is pointed at torch's current stream so the in-process exchange
    (torch copies) is ordered after the library's kernels."""
    ctx.set_stream(torch.cuda.current_stream(device).cuda_stream)
    try:
        return _emulate(ctx, torch, device, leaves, theta, t, y, sigma, flags, nranks)
    finally:
        ctx.set_stream(None)


def _emulate(ctx, torch, device, leaves, theta, t, y, sigma, flags, nranks):
    bounds = split(len(t), nranks)
    bufs = [make_buffers(torch, device, leaves, nranks) for _ in range(nranks)]
    dt = [torch.from_numpy(np.ascontiguousarray(t[bounds[r]:bounds[r + 1]])).to(device) for r in range(nranks)]
    dy = [torch.from_numpy(np.ascontiguousarray(y[bounds[r]:bounds[r + 1]])).to(device) for r in range(nranks)]
    nrec = bufs[0]["record"].numel()
    recs = torch.zeros(nranks * nrec, dtype=torch.float64, device=device)
    for r in range(nranks):  # forward on every rank (state is per context: re-run before reverse)
        tl, tr = halos(t, bounds, r)
        ctx.seg_forward_device(leaves, theta, dt[r].data_ptr(), dy[r].data_ptr(), len(dt[r]), tl, tr, r, nranks,
                               sigma, flags, bufs[r]["record"].data_ptr())
        recs[r * nrec:(r + 1) * nrec] = bufs[r]["record"]
    total = torch.zeros_like(bufs[0]["partials"])
    mean = torch.zeros(len(t), dtype=torch.float64, device=device)
    var = torch.zeros(len(t), dtype=torch.float64, device=device)
    for r in range(nranks):
        tl, tr = halos(t, bounds, r)
        a, b = bounds[r], bounds[r + 1]
        ctx.seg_forward_device(leaves, theta, dt[r].data_ptr(), dy[r].data_ptr(), b - a, tl, tr, r, nranks, sigma,
                               flags, bufs[r]["record"].data_ptr())
        ctx.seg_reverse_device(leaves, theta, dt[r].data_ptr(), dy[r].data_ptr(), b - a, tl, tr, r, nranks, sigma,
                               flags, recs.data_ptr(), bufs[r]["partials"].data_ptr(), mean[a:b].data_ptr(),
                               var[a:b].data_ptr())
        total += bufs[r]["partials"]
    ll = torch.zeros(1, dtype=torch.float64, device=device)
    g = torch.zeros(len(theta) + 1, dtype=torch.float64, device=device)
    ctx.seg_finalize_device(len(theta), len(t), sigma, flags, total.data_ptr(), ll.data_ptr(), g.data_ptr())
    ctx.status()
    return float(ll.item()), g.cpu().numpy(), mean.cpu().numpy(), var.cpu().numpy()
