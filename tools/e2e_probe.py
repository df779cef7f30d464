"""e2e probe (diagnostics): PCIe copy rates and the host-pointer eval, cfg2 shape."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1610_08035_b200 as P  # noqa: E402
from paper_1610_08035_b200 import datasets  # noqa: E402

dev = torch.device("cuda", 0)
w = datasets.make("cfg2")
n = len(w.t)
h_t = torch.from_numpy(w.t).pin_memory()
h_y = torch.from_numpy(w.y).pin_memory()
d_t = torch.empty(n, dtype=torch.float64, device=dev)
h_m = torch.empty(n, dtype=torch.float64).pin_memory()
s = torch.cuda.current_stream(dev)


def timed(f, reps=10):
    f()
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        f()
        b.record(s)
        b.synchronize()
        ms.append(a.elapsed_time(b))
    return float(np.median(ms))


h2d = timed(lambda: d_t.copy_(h_t, non_blocking=True))
d2h = timed(lambda: h_m.copy_(d_t, non_blocking=True))
print(f"H2D 8 MB {h2d:.3f} ms ({8e6 / h2d / 1e6:.1f} GB/s); D2H 8 MB {d2h:.3f} ms ({8e6 / d2h / 1e6:.1f} GB/s)")
ctx = P.Context(0)
ctx.set_stream(s.cuda_stream)
out = {"grad": np.empty(3), "mean": h_m.numpy()}
for want in (dict(grad=True), dict(grad=True, mean=True)):
    o = {k: out[k] for k in want}
    ms = timed(lambda: ctx.eval(w.leaves, w.theta, h_t.numpy(), h_y.numpy(), w.sigma, out=o, **want))
    t0 = time.perf_counter()
    for _ in range(10):
        ctx.eval(w.leaves, w.theta, h_t.numpy(), h_y.numpy(), w.sigma, out=o, **want)
    wall = (time.perf_counter() - t0) / 10 * 1e3
    print(f"eval host {sorted(want)}: events {ms:.3f} ms, wall {wall:.3f} ms "
          f"(SPINGP_PIPELINE={os.environ.get('SPINGP_PIPELINE', '1')})")

# fixed host-side cost of one host-pointer call (tiny series)
tt, yy = w.t[:1000].copy(), w.y[:1000].copy()
for _ in range(3):
    ctx.eval(w.leaves, w.theta, tt, yy, w.sigma, grad=True)
t0 = time.perf_counter()
for _ in range(200):
    ctx.eval(w.leaves, w.theta, tt, yy, w.sigma, grad=True)
print(f"host-pointer call at n=1000: {(time.perf_counter() - t0) / 200 * 1e6:.1f} us wall")
import ctypes  # noqa: E402
L = P.lib()
t0 = time.perf_counter()
for _ in range(2000):
    L.spingp_abi_version()
print(f"bare ctypes call: {(time.perf_counter() - t0) / 2000 * 1e6:.2f} us")
