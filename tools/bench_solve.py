"""Solve operator (SURVEY.md §8(d) figure 1): cr_solve of a materialised SymBTD with one
right-hand side, device pointers, timed with CUDA events on the library's stream.
Compulsory bytes B_solve = 8 (2 b^2 + 2 b) per block row (diag + upper + rhs + x).
Usage: python tools/bench_solve.py [n] [b] [steps]"""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1610_08035_b200 as P  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    b = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(7)
    A = torch.randn(n, b, b, device=dev, dtype=torch.float64, generator=g)
    diag = (A @ A.transpose(1, 2) + 4 * b * torch.eye(b, device=dev, dtype=torch.float64)).contiguous()
    upper = torch.randn(n - 1, b, b, device=dev, dtype=torch.float64, generator=g).contiguous()
    rhs = torch.randn(n * b, device=dev, dtype=torch.float64, generator=g)
    x = torch.empty_like(rhs)
    ld = torch.empty(1, device=dev, dtype=torch.float64)
    flush = torch.empty(64 * 1024 * 1024, device=dev, dtype=torch.float32)
    ctx = P.Context(0)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    L = P.lib()

    def run():
        st = L.spingp_btd_cr_solve_device(ctx._h, n, b, diag.data_ptr(), upper.data_ptr(), rhs.data_ptr(), 1,
                                          x.data_ptr(), ld.data_ptr())
        if st != 0:
            raise RuntimeError(f"status {st}")

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    ms = []
    for _ in range(steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run()
        e1.record(stream)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    t = float(np.median(ms))
    # residual check: || M x - rhs || / || rhs || (matvec on the host, float64)
    d, u, r, xx = (v.cpu().numpy() for v in (diag, upper, rhs, x))
    xb = xx.reshape(n, b)
    y = np.einsum("nij,nj->ni", d, xb)
    y[:-1] += np.einsum("nij,nj->ni", u, xb[1:])
    y[1:] += np.einsum("nji,nj->ni", u, xb[:-1])
    res = float(np.linalg.norm(y.ravel() - r) / np.linalg.norm(r))
    bytes_ = 8 * (2 * b * b + 2 * b) * n
    peak = 6538.9
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "MEASURED_PEAKS.json")) as f:
            peak = float(json.load(f)["hbm_gbs"])
    except OSError:
        pass
    gbs = bytes_ / (t * 1e-3) / 1e9
    print(json.dumps({"op": "btd_cr_solve_device", "n": n, "b": b, "k": 1, "ms": t, "blocks_per_s": n / (t * 1e-3),
                      "compulsory_bytes": bytes_, "achieved_gbs": gbs, "peak_gbs": peak, "frac": gbs / peak,
                      "residual": res, "launches": ctx.launch_count()}))


if __name__ == "__main__":
    main()
