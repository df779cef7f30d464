"""GPU vs host-emulation comparison of the segment protocol, rank by rank (debug tool)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
import emu_lib as E, paper_1610_08035_b200 as P
from paper_1610_08035_b200.partition import split, halos
np.set_printoptions(precision=6, linewidth=220)
rng = np.random.default_rng(0); n = 3000
t = np.cumsum(rng.uniform(0.05, 0.15, n)); y = np.sin(0.5 * t) + 0.3 * rng.standard_normal(n)
lv, th = [P.MATERN52], [2.0, 1.5]
NR = int(sys.argv[1]) if len(sys.argv) > 1 else 2
bounds = split(n, NR)
ctx = P.Context(0); dev = torch.device("cuda", 0)
ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
nrec, npart = P.seg_sizes(lv)
recs_e, recs_g = [], []
for r in range(NR):
    a, b = bounds[r], bounds[r + 1]; tl, tr = halos(t, bounds, r)
    re = E.seg_forward(lv, th, t[a:b], y[a:b], tl, tr, r, NR, 0.3, flags=7)
    dt = torch.from_numpy(t[a:b].copy()).to(dev); dy = torch.from_numpy(y[a:b].copy()).to(dev)
    rec = torch.zeros(nrec, dtype=torch.float64, device=dev)
    ctx.seg_forward_device(lv, th, dt.data_ptr(), dy.data_ptr(), b - a, tl, tr, r, NR, 0.3, 7, rec.data_ptr())
    torch.cuda.synchronize()
    rg = rec.cpu().numpy()
    print("rank", r, "rec maxdiff", np.abs(rg - re).max(), "scale", np.abs(re).max())
    if np.abs(rg - re).max() > 1e-6 * np.abs(re).max():
        print(" emu", re); print(" gpu", rg)
    recs_e.append(re); recs_g.append(rg)
    try: ctx.status()
    except Exception as e: print("status", e)
RE = np.concatenate(recs_e)
for r in range(NR):
    a, b = bounds[r], bounds[r + 1]; tl, tr = halos(t, bounds, r)
    E.seg_forward(lv, th, t[a:b], y[a:b], tl, tr, r, NR, 0.3, flags=7)
    part_e, mu_e, v_e = E.seg_reverse(RE, b - a, npart, mean=True, var=True)
    dt = torch.from_numpy(t[a:b].copy()).to(dev); dy = torch.from_numpy(y[a:b].copy()).to(dev)
    rec = torch.zeros(nrec, dtype=torch.float64, device=dev)
    ctx.seg_forward_device(lv, th, dt.data_ptr(), dy.data_ptr(), b - a, tl, tr, r, NR, 0.3, 7, rec.data_ptr())
    recs = torch.from_numpy(RE).to(dev)
    part = torch.zeros(npart, dtype=torch.float64, device=dev)
    mean = torch.zeros(b - a, dtype=torch.float64, device=dev); var = torch.zeros(b - a, dtype=torch.float64, device=dev)
    ctx.seg_reverse_device(lv, th, dt.data_ptr(), dy.data_ptr(), b - a, tl, tr, r, NR, 0.3, 7, recs.data_ptr(), part.data_ptr(), mean.data_ptr(), var.data_ptr())
    torch.cuda.synchronize()
    print("rank", r, "emu part", part_e); print("rank", r, "gpu part", part.cpu().numpy())
    mg, vg = mean.cpu().numpy(), var.cpu().numpy()
    print(" mean maxdiff", np.abs(mg - mu_e).max(), "var maxdiff", np.abs(vg - v_e).max())
    bad = np.nonzero(np.abs(vg - v_e) > 1e-6)[0]
    if len(bad): print(" bad var idx", bad[:10], bad[-10:], len(bad))
    try: ctx.status()
    except Exception as e: print("status", e)
