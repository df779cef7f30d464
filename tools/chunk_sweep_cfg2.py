"""cfg2 (1 M points, loglik + grad + mean, device-resident) against the level-0 chunk length
(spingp_ctx_set_chunk; 0 = the planner's choice)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
import paper_1610_08035_b200 as P
from paper_1610_08035_b200 import datasets
w = datasets.make("cfg2")
dev = torch.device("cuda", 0)
t = torch.from_numpy(w.t).to(dev); y = torch.from_numpy(w.y).to(dev)
n = len(w.t)
ll = torch.zeros(1, device=dev, dtype=torch.float64); g = torch.zeros(8, device=dev, dtype=torch.float64); mean = torch.zeros(n, device=dev, dtype=torch.float64)
flush = torch.empty(64 * 1024 * 1024, device=dev, dtype=torch.float32)
stream = torch.cuda.current_stream(dev)
flags = P.WANT_GRAD | P.WANT_MEAN
for m0 in (0, 10, 14, 16, 20, 27, 28, 40, 54):
    with P.Context(0) as ctx:
        ctx.set_stream(stream.cuda_stream)
        if m0: ctx.set_chunk(m0)
        def run():
            ctx.eval_device(w.leaves, w.theta, t.data_ptr(), y.data_ptr(), n, w.sigma, flags, ll.data_ptr(), g.data_ptr(), mean.data_ptr(), 0)
        for _ in range(3): run()
        torch.cuda.synchronize()
        ms = []
        for _ in range(15):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream); run(); e1.record(stream); e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        print(f"m0={m0}: {np.median(ms):.4f} ms  loglik {float(ll.item()):.10e}", flush=True)
