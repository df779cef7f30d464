"""Per-phase durations of the fused upper-level kernel (k_upper) on cfg2 (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
import paper_1610_08035_b200 as P
from paper_1610_08035_b200 import datasets
w = datasets.make(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
dev = torch.device("cuda", 0)
ctx = P.Context(0); ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
dt = torch.from_numpy(w.t).to(dev); dy = torch.from_numpy(w.y).to(dev)
ll = torch.zeros(1, dtype=torch.float64, device=dev); g = torch.zeros(8, dtype=torch.float64, device=dev)
st = torch.zeros(64, dtype=torch.int64, device=dev)
for rep in range(3):
    ctx.set_phase_stamps(st.data_ptr() if rep == 2 else 0)
    ctx.eval_device(w.leaves, w.theta, dt.data_ptr(), dy.data_ptr(), len(w.t), w.sigma, P.WANT_GRAD, ll.data_ptr(), g.data_ptr(), 0, 0)
    torch.cuda.synchronize()
s = st.cpu().numpy().astype(np.int64)
coop = np.count_nonzero(s[:16]) == 16  # k_tree_coop stamps run past slot 16
for name, lo, hi in ((("k_tree_coop", 0, 64),) if coop else (("k_tree_fwd", 0, 16), ("k_tree_one", 16, 48), ("k_tree_rev", 48, 64))):
    v = s[lo:hi]
    k = int(np.count_nonzero(v))
    if k > 1:
        d = np.diff(v[:k]) / 1e3
        print(name, "phases", k - 1, "us:", np.round(d, 2), "total", round(float(d.sum()), 1))

