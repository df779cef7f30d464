"""Stress of the streaming cr_solve kernels: large systems, mixed sizes back to back on one
context (the grid barrier's monotonic counters), two contexts from two threads.
Usage: python tools/stream_stress.py"""
import os
import sys
import threading

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import paper_1610_08035_b200 as P  # noqa: E402
from stream_check import residual, system  # noqa: E402


def solve(ctx, n, b, diag, upper, rhs, k=1):
    x = torch.full((n * b,), float("nan"), device=diag.device, dtype=torch.float64)
    ld = torch.zeros(1, device=diag.device, dtype=torch.float64)
    torch.cuda.synchronize()
    ctx.btd_cr_solve_device(n, b, diag.data_ptr(), upper.data_ptr(), rhs.data_ptr(), k, x.data_ptr(), ld.data_ptr())
    ctx.status()
    return x, float(ld.item())


def main():
    dev = torch.device("cuda", 0)
    worst = 0.0
    with P.Context(0) as ctx:
        for n, b in ((20_000_000, 3), (50_000_000, 1), (12_000_001, 2), (6_000_003, 4)):
            diag, upper, rhs = system(n, b, dev, seed=n % 1000 + b)
            x, ld = solve(ctx, n, b, diag, upper, rhs)
            res = residual(n, b, diag, upper, rhs, x)
            worst = max(worst, res)
            print(f"large: b={b} n={n}: residual {res:.2e} logdet {ld:.6e}", flush=True)
            del diag, upper, rhs, x
            torch.cuda.empty_cache()
        # mixed sizes back to back, with and without a right-hand side
        for rep in range(3):
            for n, b in ((2049, 3), (100_003, 1), (1281, 3), (700_001, 3), (4097, 2), (33_000, 4), (1500, 3)):
                diag, upper, rhs = system(n, b, dev, seed=rep * 100 + n % 97)
                x, ld = solve(ctx, n, b, diag, upper, rhs)
                _, ld0 = solve(ctx, n, b, diag, upper, rhs, k=0)
                res = residual(n, b, diag, upper, rhs, x)
                worst = max(worst, res, abs(ld - ld0) / abs(ld))
                assert res < 1e-12 and abs(ld - ld0) <= 1e-13 * abs(ld), (n, b, res, ld, ld0)
        print("mixed sizes: ok", flush=True)
    # two contexts, two host threads, the same device
    errs = []

    def worker(seed):
        try:
            with P.Context(0) as c:
                for it in range(10):
                    n, b = 300_000 + 1000 * it + seed, 3
                    diag, upper, rhs = system(n, b, dev, seed=seed + it)
                    x, _ = solve(c, n, b, diag, upper, rhs)
                    r = residual(n, b, diag, upper, rhs, x)
                    if not r < 1e-12:
                        errs.append((seed, it, r))
        except Exception as e:  # noqa: BLE001
            errs.append((seed, repr(e)))

    th = [threading.Thread(target=worker, args=(s,)) for s in (1, 2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    print("two contexts:", "ok" if not errs else errs, flush=True)
    print(f"worst {worst:.3e}")
    if errs:
        sys.exit(1)


if __name__ == "__main__":
    main()
