"""Run partition.emulate_ranks for a sequence of rank counts on one context (debug tool)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
import paper_1610_08035_b200 as P
from paper_1610_08035_b200.partition import emulate_ranks
rng = np.random.default_rng(0); n = 3000
t = np.cumsum(rng.uniform(0.05, 0.15, n)); y = np.sin(0.5 * t) + 0.3 * rng.standard_normal(n)
for seq in sys.argv[1:]:
    ctx = P.Context(0)
    for nr in [int(s) for s in seq.split(",")]:
        try:
            ll, g, m, v = emulate_ranks(ctx, torch, torch.device("cuda", 0), [P.MATERN52], [2.0, 1.5], t, y, 0.3, 7, nr)
            print(seq, nr, ll, g)
        except Exception as e:
            print(seq, nr, "ERR", e)
