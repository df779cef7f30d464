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


def measure(n=1_000_000, b=3, steps=20, device=0, check=True):
    """Median ms of one cr_solve (1 rhs) on a device-resident random SPD SymBTD, with the
    HBM roofline figures of SURVEY.md §8(d); L2 flushed before each timed call."""
    dev = torch.device("cuda", device)
    g = torch.Generator(device=dev).manual_seed(7)
    A = torch.randn(n, b, b, device=dev, dtype=torch.float64, generator=g)
    diag = (A @ A.transpose(1, 2) + 4 * b * torch.eye(b, device=dev, dtype=torch.float64)).contiguous()
    upper = torch.randn(n - 1, b, b, device=dev, dtype=torch.float64, generator=g).contiguous()
    rhs = torch.randn(n * b, device=dev, dtype=torch.float64, generator=g)
    x = torch.empty_like(rhs)
    ld = torch.empty(1, device=dev, dtype=torch.float64)
    flush = torch.empty(64 * 1024 * 1024, device=dev, dtype=torch.float32)
    ctx = P.Context(device)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    L = P.lib()

    def run():
        st = L.spingp_btd_cr_solve_device(ctx._h, n, b, diag.data_ptr(), upper.data_ptr(), rhs.data_ptr(), 1,
                                          x.data_ptr(), ld.data_ptr())
        if st != 0:
            raise RuntimeError(f"status {st}")

    def timed():
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        out = []
        for _ in range(steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run()
            e1.record(stream)
            e1.synchronize()
            out.append(e0.elapsed_time(e1))
        return out

    # the partitioned thread-per-chunk kernels (round 1) for comparison, then the default path
    # (b <= 4, one rhs: the strip-streaming kernel, csrc/strip_solve.cuh)
    prev = os.environ.get("SPINGP_SOLVE_STREAM")
    os.environ["SPINGP_SOLVE_STREAM"] = "0"
    t_part = float(np.median(timed()))
    if prev is None:
        del os.environ["SPINGP_SOLVE_STREAM"]
    else:
        os.environ["SPINGP_SOLVE_STREAM"] = prev
    k0 = ctx.launch_count()
    ms = timed()
    launches = (ctx.launch_count() - k0) // (steps + 3)
    t = float(np.median(ms))
    res = None
    if check:  # residual || M x - rhs || / || rhs || (block matvec on the device, fp64)
        xb = x.view(n, b)
        yv = torch.einsum("nij,nj->ni", diag, xb)
        yv[:-1] += torch.einsum("nij,nj->ni", upper, xb[1:])
        yv[1:] += torch.einsum("nji,nj->ni", upper, xb[:-1])
        res = float(torch.linalg.norm(yv.reshape(-1) - rhs) / torch.linalg.norm(rhs))
    bytes_ = 8 * (2 * b * b + 2 * b) * n
    peak = 6538.9
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "MEASURED_PEAKS.json")) as f:
            peak = float(json.load(f)["hbm_gbs"])
    except OSError:
        pass
    gbs = bytes_ / (t * 1e-3) / 1e9
    out = {"op": "spingp_btd_cr_solve_device", "n": n, "b": b, "k": 1, "ms": t, "blocks_per_s": n / (t * 1e-3),
           "compulsory_bytes": bytes_, "achieved_gbs": gbs, "peak_gbs": peak, "frac": gbs / peak,
           "residual": res, "launches_per_solve": launches,
           "kernel": "k_solve_strip" if launches == 1 else "k_fwdL / k_tree_* / k_revL",
           "partitioned_ms": t_part, "partitioned_frac": bytes_ / (t_part * 1e-3) / 1e9 / peak,
           "data": "random SPD blocks (seeded), L2 flushed before each call"}
    try:  # DRAM bytes per solve from the committed ncu capture (profiles/ncu_traffic.json)
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "ncu_traffic.json")) as f:
            out["traffic"] = json.load(f).get("solve_operator", {}).get(out["kernel"])
    except (OSError, ValueError):
        out["traffic"] = None
    ctx.close()
    return out


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    b = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    print(json.dumps(measure(n, b, steps)))


if __name__ == "__main__":
    main()
