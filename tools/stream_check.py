"""Tile-streaming cr_solve (csrc/stream_solve.cuh) against the partitioned kernels
(SPINGP_SOLVE_STREAM=0) and the residual of the system, over block sizes, lengths, ragged
tails and misaligned arrays; then timings of both paths at 1 M blocks, b = 3.
Usage: python tools/stream_check.py [quick]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1610_08035_b200 as P  # noqa: E402


def system(n, b, dev, seed=7, off=0):
    g = torch.Generator(device=dev).manual_seed(seed)
    A = torch.randn(n, b, b, device=dev, dtype=torch.float64, generator=g)
    diag = A @ A.transpose(1, 2) + 4 * b * torch.eye(b, device=dev, dtype=torch.float64)
    # off-diagonal blocks scaled so that the matrix stays positive definite at b = 1
    upper = torch.randn(max(n - 1, 1), b, b, device=dev, dtype=torch.float64, generator=g) * (0.5 if b == 1 else 1.0)
    rhs = torch.randn(n * b, device=dev, dtype=torch.float64, generator=g)

    def place(v):  # optionally 8 bytes off a 16-byte boundary
        buf = torch.empty(v.numel() + 2, device=dev, dtype=torch.float64)
        out = buf[off:off + v.numel()]
        out.copy_(v.reshape(-1))
        return out

    return place(diag), place(upper), place(rhs)


def residual(n, b, diag, upper, rhs, x):
    d, u, xb = diag.view(n, b, b), upper.view(-1, b, b)[: n - 1], x.view(n, b)
    yv = torch.einsum("nij,nj->ni", d, xb)
    yv[:-1] += torch.einsum("nij,nj->ni", u, xb[1:])
    yv[1:] += torch.einsum("nji,nj->ni", u, xb[:-1])
    return float(torch.linalg.norm(yv.reshape(-1) - rhs) / torch.linalg.norm(rhs))


def solve(ctx, n, b, diag, upper, rhs, stream, k=1):
    os.environ["SPINGP_SOLVE_STREAM"] = "1" if stream else "0"
    x = torch.full((n * b,), float("nan"), device=diag.device, dtype=torch.float64)
    ld = torch.zeros(1, device=diag.device, dtype=torch.float64)
    st = P.lib().spingp_btd_cr_solve_device(ctx._h, n, b, diag.data_ptr(), upper.data_ptr(), rhs.data_ptr(), k,
                                            x.data_ptr() if k else 0, ld.data_ptr())
    torch.cuda.synchronize()
    if st != 0:
        raise RuntimeError(f"status {st}")
    return x, float(ld.item())


def main():
    dev = torch.device("cuda", 0)
    ctx = P.Context(0)
    ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
    quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
    worst = 0.0
    sizes = [1281, 1282, 1500, 1793, 4801, 20000, 100003] + ([] if quick else [1_000_000, 3_000_001])
    for b in (3, 1, 2, 4):
        for n in sizes:
            for off in (0, 1):
                if off and n > 20000:
                    continue
                diag, upper, rhs = system(n, b, dev, seed=n + b, off=off)
                xs, lds = solve(ctx, n, b, diag, upper, rhs, True)
                xo, ldo = solve(ctx, n, b, diag, upper, rhs, False)
                _, ld0 = solve(ctx, n, b, diag, upper, rhs, True, k=0)
                res = residual(n, b, diag, upper, rhs, xs)
                dx = float((xs - xo).abs().max() / xo.abs().max())
                dl = abs(lds - ldo) / abs(ldo)
                dl0 = abs(ld0 - ldo) / abs(ldo)
                worst = max(worst, dx, dl, dl0)
                flag = "" if (dx < 1e-11 and dl < 1e-12 and dl0 < 1e-12 and res < 1e-12) else "  <-- CHECK"
                print(f"b={b} n={n} off={off}: residual {res:.2e}  |x - x_old| {dx:.2e}  logdet {dl:.2e} "
                      f"(k=0 {dl0:.2e}){flag}", flush=True)
    print(f"worst relative difference {worst:.3e}")
    if quick:
        return
    # timings, L2 flushed before every call
    n, b = 1_000_000, 3
    diag, upper, rhs = system(n, b, dev)
    flush = torch.empty(64 * 1024 * 1024, device=dev, dtype=torch.float32)
    stream = torch.cuda.current_stream(dev)
    for mode, env in (("partitioned", {"SPINGP_SOLVE_STREAM": "0"}), ("stream", {"SPINGP_SOLVE_STREAM": "1"}),
                      ("stream evict_last", {"SPINGP_SOLVE_STREAM": "1", "SPINGP_SS_L2": "1"})):
        os.environ.pop("SPINGP_SS_L2", None)
        os.environ.update(env)
        x = torch.empty_like(rhs)
        ld = torch.zeros(1, device=dev, dtype=torch.float64)
        ms = []
        for it in range(25):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            P.lib().spingp_btd_cr_solve_device(ctx._h, n, b, diag.data_ptr(), upper.data_ptr(), rhs.data_ptr(), 1,
                                               x.data_ptr(), ld.data_ptr())
            e1.record(stream)
            e1.synchronize()
            if it >= 5:
                ms.append(e0.elapsed_time(e1))
        t = float(np.median(ms))
        gbs = 8 * (2 * b * b + 2 * b) * n / (t * 1e-3) / 1e9
        print(f"{mode}: {t:.4f} ms  ({gbs:.0f} GB/s algorithmic, min {min(ms):.4f} ms)")


if __name__ == "__main__":
    main()
