"""A few tile-streaming solves at 1 M blocks, b = 3 (profiling target)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import paper_1610_08035_b200 as P  # noqa: E402
from stream_check import system  # noqa: E402

dev = torch.device("cuda", 0)
ctx = P.Context(0)
ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
n, b = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000, 3
diag, upper, rhs = system(n, b, dev)
x = torch.empty_like(rhs)
ld = torch.zeros(1, device=dev, dtype=torch.float64)
flush = torch.empty(64 * 1024 * 1024, device=dev, dtype=torch.float32)
for it in range(4):
    flush.zero_()
    torch.cuda.synchronize()
    P.lib().spingp_btd_cr_solve_device(ctx._h, n, b, diag.data_ptr(), upper.data_ptr(), rhs.data_ptr(), 1, x.data_ptr(),
                                       ld.data_ptr())
    torch.cuda.synchronize()
print("ok", float(ld.item()))
