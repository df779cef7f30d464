"""Parity table at BASELINE size: for every config x {loglik, grad,
mean, var} the GPU result (C ABI, sm_100a) against the fp64 oracle and against the
long-double run of the same oracle, beside the fp64 floor (the fp64 oracle's own
distance from the long-double run; with `--reversed`, the larger of the forward and
time-reversed fp64 evaluations, as tests/test_gpu_parity.py::check uses).

Errors are normwise: max|a - b| / max|b| over the quantity (per series for cfg3, then
the max over series).  Writes JSON + markdown.

Usage (GPU box): python tools/parity_table.py OUT_PREFIX [cfg ...] [--reversed]
  cfg1, cfg2, cfg3, cfg4: full BASELINE size.
  cfg5: a 1,000,000-point prefix evaluated with the full-size level-0 plan
        (spingp_ctx_set_chunk(423): the 32 M-point plan's chunk length), because the
        oracle needs hours for 32 M points (per-step 32x32 Van Loan exponentials).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import oracle_lib as O  # noqa: E402
import paper_1610_08035_b200 as P  # noqa: E402
from paper_1610_08035_b200 import datasets  # noqa: E402

THREADS = os.cpu_count() or 1
SIZES = {"cfg5": 1_000_000}
CHUNK = {"cfg5": 423}  # the full-size plan's m0 (make_plan at 32 M points)
KEYS = {"cfg1": ("loglik", "grad", "mean", "var"), "cfg2": ("loglik", "grad", "mean"), "cfg3": ("loglik", "grad"),
        "cfg4": ("loglik", "grad"), "cfg5": ("loglik", "grad", "var")}


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def rel_rows(a, b):
    """cfg3: per-series normwise error, max over series."""
    a, b = np.atleast_2d(np.asarray(a, float)), np.atleast_2d(np.asarray(b, float))
    if a.shape[0] == 1 and b.shape[0] > 1:
        a, b = a.T, b.T
    num = np.max(np.abs(a - b), axis=1)
    den = np.maximum(np.max(np.abs(b), axis=1), 1e-300)
    return float(np.max(num / den))


def oracle(wl, precision, reverse=False):
    t, y = wl.t, wl.y
    if reverse:
        t, y = -t[..., ::-1].copy(), y[..., ::-1].copy()
    keys = KEYS[wl.name]
    if wl.batched:
        ll, g = O.evaluate_batched(wl.leaves, wl.theta, t, y, wl.sigma, grad=True, precision=precision,
                                   threads=THREADS)
        return {"loglik": np.asarray(ll).reshape(-1, 1), "grad": g}
    r = O.evaluate(wl.leaves, wl.theta, t, y, wl.sigma, grad=True, mean="mean" in keys, var="var" in keys,
                   precision=precision, threads=THREADS)
    if reverse:
        for k in ("mean", "var"):
            if r.get(k) is not None:
                r[k] = np.asarray(r[k])[::-1]
    return r


def gpu(ctx, wl):
    keys = KEYS[wl.name]
    if wl.batched:
        g = ctx.eval_batched(wl.leaves, wl.theta, wl.t, wl.y, wl.sigma, grad=True)
        g["loglik"] = np.asarray(g["loglik"]).reshape(-1, 1)
        return g
    ctx.set_chunk(CHUNK.get(wl.name, 0))
    try:
        return ctx.eval(wl.leaves, wl.theta, wl.t, wl.y, wl.sigma, grad=True, mean="mean" in keys, var="var" in keys)
    finally:
        ctx.set_chunk(0)


def main():
    out = sys.argv[1]
    names = [a for a in sys.argv[2:] if a.startswith("cfg")] or ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]
    reverse = "--reversed" in sys.argv
    rows = {}
    with P.Context(0) as ctx:
        for name in names:
            wl = datasets.make(name, **({"n": SIZES[name]} if name in SIZES else {}))
            t0 = time.time()
            g = gpu(ctx, wl)
            tg = time.time() - t0
            t0 = time.time()
            o = oracle(wl, 0)
            to = time.time() - t0
            t0 = time.time()
            ld = oracle(wl, 1)
            tl = time.time() - t0
            orv = oracle(wl, 0, reverse=True) if reverse and not wl.batched else None
            f = rel_rows if wl.batched else rel
            rec = {"points": wl.points, "chunk_m0": CHUNK.get(name), "seconds": {"gpu": tg, "oracle": to, "oracle_ld": tl},
                   "threads": THREADS, "quantities": {}}
            for k in KEYS[name]:
                floor = f(o[k], ld[k])
                if orv is not None:
                    floor = max(floor, f(orv[k], ld[k]))
                e_o, e_ld = f(g[k], o[k]), f(g[k], ld[k])
                rec["quantities"][k] = {"rel_gpu_oracle": e_o, "rel_gpu_ld": e_ld, "fp64_floor": floor,
                                        "ratio_to_floor": e_ld / floor if floor > 0 else None}
            if name in ("cfg1", "cfg2", "cfg4", "cfg5"):
                rec["loglik"] = {"gpu": float(np.ravel(g["loglik"])[0]), "oracle": float(np.ravel(o["loglik"])[0]),
                                 "oracle_ld": float(np.ravel(ld["loglik"])[0])}
                rec["grad"] = {"gpu": np.ravel(g["grad"]).tolist(), "oracle": np.ravel(o["grad"]).tolist(),
                               "oracle_ld": np.ravel(ld["grad"]).tolist()}
            rows[name] = rec
            print(name, json.dumps(rec["quantities"]), flush=True)
            with open(out + ".json", "w") as fh:
                json.dump(rows, fh, indent=1)
    lines = ["| cfg | points | quantity | rel(GPU, fp64 oracle) | rel(GPU, long double) | fp64 floor "
             "rel(oracle, long double) | GPU / floor |", "|---|---|---|---|---|---|---|"]
    for name, rec in rows.items():
        pts = f"{rec['points']:,}" + (f" (plan m0={rec['chunk_m0']})" if rec["chunk_m0"] else "")
        for k, q in rec["quantities"].items():
            r = q["ratio_to_floor"]
            lines.append(f"| {name} | {pts} | {k} | {q['rel_gpu_oracle']:.2e} | {q['rel_gpu_ld']:.2e} | "
                         f"{q['fp64_floor']:.2e} | {'-' if r is None else f'{r:.2f}'} |")
    with open(out + ".md", "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
