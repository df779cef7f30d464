"""Timing of the tile-streaming cr_solve at 1 M blocks, b = 3 (L2 flushed before every
call), with a quick residual check.  Usage: python tools/stream_time.py [label]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1610_08035_b200 as P  # noqa: E402
from stream_check import residual, system  # noqa: E402

dev = torch.device("cuda", 0)
ctx = P.Context(0)
stream = torch.cuda.current_stream(dev)
ctx.set_stream(stream.cuda_stream)
n, b = 1_000_000, 3
diag, upper, rhs = system(n, b, dev)
flush = torch.empty(64 * 1024 * 1024, device=dev, dtype=torch.float32)
x = torch.empty_like(rhs)
ld = torch.zeros(1, device=dev, dtype=torch.float64)
ms = []
for it in range(30):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    P.lib().spingp_btd_cr_solve_device(ctx._h, n, b, diag.data_ptr(), upper.data_ptr(), rhs.data_ptr(), 1, x.data_ptr(),
                                       ld.data_ptr())
    e1.record(stream)
    e1.synchronize()
    if it >= 5:
        ms.append(e0.elapsed_time(e1))
t = float(np.median(ms))
print(f"{sys.argv[1] if len(sys.argv) > 1 else ''}: {t:.4f} ms (min {min(ms):.4f})  frac {8 * 24 * n / (t * 1e-3) / 6553.9e9:.3f}  "
      f"residual {residual(n, b, diag, upper, rhs, x):.2e}", flush=True)
