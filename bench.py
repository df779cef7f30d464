#!/usr/bin/env python
"""Benchmark: SpInGP loglik+grad time points/s (fp64) on B200.

Default workload (N=1): BASELINE cfg2 — Matérn-5/2 (b=3), one series of 1,000,000
seeded synthetic points, log-likelihood + gradient (var, len, σ) + posterior mean,
every step the full fused hot path (closed-form discretisation -> assembly ->
partitioned block elimination -> selected inverse -> loglik/gradient reduction).

  value  : device-resident inputs, CUDA events around each step on the library's
           stream, L2 flushed (256 MiB write) between steps outside the events.
  e2e    : the same metric through the host-pointer C ABI call (spingp_eval):
           pinned host t,y -> H2D, kernels, D2H of loglik, gradient and mean.
  N > 1  : torchrun, one rank per GPU; ONE series of N x 1,000,000 points partitioned
           into contiguous time segments: each GPU reduces its
           segment to a 2-separator Schur record, the N records are all-gathered over
           NCCL (torch.distributed), the N-block reduced system is solved redundantly on
           every GPU, segments are back-substituted and the partial sums all-reduced.
           Weak scaling (1,000,000 points per GPU).  Batched configs (cfg3) shard series.
  --impl reference : the CPU oracle (restatement of the reference algorithm, Padé/
           Van Loan per step + block Thomas + Takahashi; the reference itself does
           not build here) on all host cores, same workload, rank 0 only.
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

METRIC = "SpInGP loglik+grad time points/s (fp64), 1/2/4/8 B200, % HBM roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg2", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--points", type=int, default=0, help="override N (testing only; not a bench value)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_info():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload(name, rank, points):
    from paper_1610_08035_b200 import datasets
    kw = {}
    if points:
        kw["n"] = points
    if rank:
        kw["seed"] = datasets.SEEDS[name] + 7919 * rank
    return datasets.make(name, **kw)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


FP64_PEAK_TFLOPS = 34.1  # DFMA microbenchmark on this pool's B200 (profiles/r01_box_probe.log)


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML every ~2 ms
    while the warm-up and timed steps run (B200_PROFILING.md clocks line).  Samples
    taken inside the timed region are reported when there are any; otherwise the
    whole loaded window (warm-up + timed) is, and `window` says which."""

    REASONS = [("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown")]

    def __init__(self, torch_device):
        self.dev = torch_device
        self.rows = []  # (timed?, sm_mhz, max_mhz, reasons bitmask)
        self.timed = False
        self._stop = threading.Event()
        self.nv = None

    def _handle(self):
        import pynvml as nv
        import torch
        nv.nvmlInit()
        try:
            uuid = str(torch.cuda.get_device_properties(self.dev).uuid)
            return nv, nv.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        except Exception:
            return nv, nv.nvmlDeviceGetHandleByIndex(self.dev.index or 0)

    def __enter__(self):
        try:
            self.nv, self.h = self._handle()
        except Exception:
            self.nv = None
            return self
        self.thread = threading.Thread(target=self._poll, daemon=True)
        self.thread.start()
        return self

    def _poll(self):
        nv, h = self.nv, self.h
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((self.timed, sm, mx, rs))
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv is not None:
            self.thread.join(timeout=2)

    def summary(self):
        if self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "window": "nvml unavailable"}
        rows = [r for r in self.rows if r[0]]
        window = "timed region"
        if not rows:
            rows, window = self.rows, "warm-up + timed region"
        reasons = set()
        for r in rows:
            for nm, attr in self.REASONS:
                if hasattr(self.nv, attr) and r[3] & getattr(self.nv, attr):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(r[1] for r in rows) if rows else None,
                "sm_max_mhz": max(r[2] for r in rows) if rows else None,
                "reasons": sorted(reasons), "samples": len(rows), "window": window}


def alg_bytes_per_point(kernel, wl):
    """Compulsory HBM bytes of one launch per time point (SURVEY.md §8(d) B_io split by kernel)."""
    outs = 8 * (("mean" in wl.outputs) + ("var" in wl.outputs))
    if kernel == "k_fwd0":
        return 16.0           # t, y read once
    if kernel == "k_rev0":
        return 16.0 + outs    # t, y read once, per-point outputs written once
    return 0.0


def core_flops_per_point(b, n_theta):
    """F_core = 8 b^3 + 4 b^2 (1 + n_θ) (factor + selected inverse + traces; lower bound)."""
    return 8 * b ** 3 + 4 * b ** 2 * (1 + n_theta)


def cpu_baseline(wl, seconds=10.0):
    """The oracle (restatement of the reference CPU path) on all host cores, on a
    bounded prefix of the same series, sized to ~`seconds` of CPU time."""
    import oracle_lib as O
    threads = os.cpu_count() or 1
    grad, mean, var = "grad" in wl.outputs, "mean" in wl.outputs, "var" in wl.outputs
    th = np.asarray(wl.theta, float)
    if wl.batched:
        pilot = max(1, min(wl.t.shape[0], 64))
        t0 = time.perf_counter()
        O.evaluate_batched(wl.leaves, th[:pilot], wl.t[:pilot], wl.y[:pilot], wl.sigma[:pilot], grad=grad,
                           threads=threads)
        rate = pilot * wl.t.shape[1] / (time.perf_counter() - t0)
        S = int(min(wl.t.shape[0], max(pilot, rate * seconds / wl.t.shape[1])))
        t0 = time.perf_counter()
        O.evaluate_batched(wl.leaves, th[:S], wl.t[:S], wl.y[:S], wl.sigma[:S], grad=grad, threads=threads)
        dt = time.perf_counter() - t0
        return {"value": S * wl.t.shape[1] / dt, "unit": "points/s", "cores": threads, "kind": "port",
                "sample": f"first {S} of {wl.t.shape[0]} series x {wl.t.shape[1]} points, loglik+grad, {dt:.1f} s"}
    n = len(wl.t)
    pilot = min(n, 20_000)
    t0 = time.perf_counter()
    O.evaluate(wl.leaves, th, wl.t[:pilot], wl.y[:pilot], wl.sigma, grad=grad, mean=mean, var=var, threads=threads)
    rate = pilot / (time.perf_counter() - t0)
    m = int(min(n, max(pilot, rate * seconds)))
    t0 = time.perf_counter()
    O.evaluate(wl.leaves, th, wl.t[:m], wl.y[:m], wl.sigma, grad=grad, mean=mean, var=var, threads=threads)
    dt = time.perf_counter() - t0
    return {"value": m / dt, "unit": "points/s", "cores": threads, "kind": "port",
            "sample": f"first {m} of {n} points, loglik+grad" + ("+mean" if mean else "") + ("+var" if var else "")
                      + f", {dt:.1f} s"}


def run_reference(args, ws, rank):
    if rank != 0:
        return
    wl = workload(args.config, 0, args.points)
    import oracle_lib as O
    threads = os.cpu_count() or 1
    grad, mean, var = "grad" in wl.outputs, "mean" in wl.outputs, "var" in wl.outputs
    th = np.asarray(wl.theta, float)

    def step():
        if wl.batched:
            O.evaluate_batched(wl.leaves, th, wl.t, wl.y, wl.sigma, grad=grad, threads=threads)
        else:
            O.evaluate(wl.leaves, th, wl.t, wl.y, wl.sigma, grad=grad, mean=mean, var=var, threads=threads)

    for _ in range(args.warmup):
        step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = wl.points * args.steps / total
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, BASELINE shapes)",
            "config": {"workload": wl.description, "config": wl.name, "points": wl.points,
                       "outputs": ["loglik"] + list(wl.outputs)},
            "cpu_baseline": {"value": value, "unit": "points/s", "cores": threads, "kind": "port",
                             "sample": f"full {wl.name} workload per step ({wl.points} points), all host threads; "
                                       "the reference itself cannot be built (no Eigen/GTest), oracle/ restates it"},
            "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, ws, rank, local):
    import torch
    import paper_1610_08035_b200 as P

    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    partitioned = ws > 1 and args.config != "cfg3"
    if partitioned:  # one long series, contiguous segment per rank
        from paper_1610_08035_b200 import datasets
        from paper_1610_08035_b200.partition import split, halos, make_buffers, eval_partitioned
        base = datasets.make(args.config, **({"n": args.points} if args.points else {}))
        full = datasets.make(args.config, n=len(base.t) * ws)
        bounds = split(len(full.t), ws)
        a, bb = bounds[rank], bounds[rank + 1]
        t_left, t_right = halos(full.t, bounds, rank)
        wl = full
        seg_t, seg_y = full.t[a:bb], full.y[a:bb]
        n_total = len(full.t)
    else:
        wl = workload(args.config, rank, args.points)
        seg_t, seg_y = wl.t, wl.y
    b, nt = P.kernel_dims(wl.leaves)
    flags = P.WANT_GRAD | (P.WANT_MEAN if "mean" in wl.outputs else 0) | (P.WANT_VAR if "var" in wl.outputs else 0)
    S = seg_t.shape[0] if seg_t.ndim == 2 else 1
    n = seg_t.shape[-1]
    points_per_rank = seg_t.size
    ctx = P.Context(local)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    d_t = torch.from_numpy(np.ascontiguousarray(seg_t)).to(dev)
    d_y = torch.from_numpy(np.ascontiguousarray(seg_y)).to(dev)
    d_ll = torch.zeros(S, dtype=torch.float64, device=dev)
    d_g = torch.zeros(S * (nt + 1), dtype=torch.float64, device=dev)
    d_m = torch.zeros(S * n, dtype=torch.float64, device=dev) if flags & P.WANT_MEAN else None
    d_v = torch.zeros(S * n, dtype=torch.float64, device=dev) if flags & P.WANT_VAR else None
    flush = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device=dev)
    if partitioned:
        bufs = make_buffers(torch, dev, wl.leaves, ws)

        def gather(out, inp):
            dist.all_gather_into_tensor(out, inp)

        def reduce_(x):
            dist.all_reduce(x)

    def step():
        if partitioned:
            eval_partitioned(ctx, wl.leaves, wl.theta, d_t.data_ptr(), d_y.data_ptr(), n, n_total, t_left, t_right,
                             rank, ws, wl.sigma, flags, bufs, gather, reduce_,
                             d_m.data_ptr() if d_m is not None else 0, d_v.data_ptr() if d_v is not None else 0)
        elif wl.batched:
            ctx.eval_batched_device(wl.leaves, wl.theta, S, n, d_t.data_ptr(), d_y.data_ptr(), wl.sigma, flags,
                                    d_ll.data_ptr(), d_g.data_ptr(), d_m.data_ptr() if d_m is not None else 0,
                                    d_v.data_ptr() if d_v is not None else 0)
        else:
            ctx.eval_device(wl.leaves, wl.theta, d_t.data_ptr(), d_y.data_ptr(), n, wl.sigma, flags,
                            d_ll.data_ptr(), d_g.data_ptr(), d_m.data_ptr() if d_m is not None else 0,
                            d_v.data_ptr() if d_v is not None else 0)

    with ClockSampler(dev) as clk:
        for _ in range(max(3, args.warmup)):
            flush.zero_()
            step()
        ctx.status()
        torch.cuda.synchronize(dev)
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        launches0 = ctx.launch_count()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        clk.timed = True
        for k in range(args.steps):
            flush.zero_()  # L2 flush between timed steps, outside the events
            evs[k][0].record(stream)
            step()
            evs[k][1].record(stream)
        torch.cuda.synchronize(dev)
        clk.timed = False
        launches = ctx.launch_count() - launches0
    ctx.status()  # raises on any device-side failure in the timed steps
    step_ms = [a_.elapsed_time(b_) for a_, b_ in evs]
    total_ms = float(sum(step_ms))
    if ws > 1:
        tt = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
        dist.barrier()
    value = points_per_rank * ws * args.steps / (total_ms * 1e-3)

    # per-kernel breakdown (separate, untimed profiling pass; events around every launch)
    ctx.set_profiling(True)
    kt = {}
    reps = 3
    for _ in range(reps):
        flush.zero_()
        step()
        for name, ms in ctx.kernel_times():
            kt.setdefault(name, []).append(ms)
    ctx.set_profiling(False)
    per_step = {k: sum(v) / reps for k, v in kt.items()}
    dom = max(per_step, key=per_step.get)
    dom_launch_ms = statistics.mean(kt[dom])
    launches_per_step = {k: len(v) // reps for k, v in kt.items()}

    # e2e: host inputs (pinned) -> device, evaluation, results -> host, every step
    h_t = torch.from_numpy(np.ascontiguousarray(seg_t)).pin_memory()
    h_y = torch.from_numpy(np.ascontiguousarray(seg_y)).pin_memory()
    want = dict(grad=True, mean="mean" in wl.outputs, var="var" in wl.outputs)
    h_out = torch.empty(S * (nt + 1) + S + (S * n if want["mean"] else 0) + (S * n if want["var"] else 0),
                        dtype=torch.float64).pin_memory()
    # the public API writes into caller-owned (here pinned) host arrays
    ho = h_out.numpy()
    k0 = 0
    outs = {"loglik": ho[k0:k0 + S]}
    k0 += S
    outs["grad"] = ho[k0:k0 + S * (nt + 1)].reshape((S, nt + 1) if wl.batched else (nt + 1,))
    k0 += S * (nt + 1)
    if want["mean"]:
        outs["mean"] = ho[k0:k0 + S * n].reshape((S, n) if wl.batched else (n,))
        k0 += S * n
    if want["var"]:
        outs["var"] = ho[k0:k0 + S * n].reshape((S, n) if wl.batched else (n,))

    def e2e_step():
        if partitioned:  # device entry points with explicit pinned H2D / D2H (the ABI is device-side here)
            d_t.copy_(h_t, non_blocking=True)
            d_y.copy_(h_y, non_blocking=True)
            step()
            k0 = 0
            h_out[k0:k0 + 1].copy_(bufs["loglik"], non_blocking=True)
            h_out[1:2 + nt].copy_(bufs["grad"], non_blocking=True)
            k0 = 2 + nt
            if d_m is not None:
                h_out[k0:k0 + n].copy_(d_m, non_blocking=True)
                k0 += n
            if d_v is not None:
                h_out[k0:k0 + n].copy_(d_v, non_blocking=True)
            return
        if wl.batched:
            ctx.eval_batched(wl.leaves, wl.theta, h_t.numpy(), h_y.numpy(), wl.sigma, out=outs, **want)
        else:
            ctx.eval(wl.leaves, wl.theta, h_t.numpy(), h_y.numpy(), wl.sigma, out=outs, **want)

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    e_ms = []
    for _ in range(args.steps):
        ea = torch.cuda.Event(enable_timing=True)
        eb = torch.cuda.Event(enable_timing=True)
        ea.record(stream)
        e2e_step()
        eb.record(stream)
        eb.synchronize()
        e_ms.append(ea.elapsed_time(eb))
    e_total = float(sum(e_ms))
    if ws > 1:
        tt = torch.tensor([e_total], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e_total = float(tt.item())
    e2e_value = points_per_rank * ws * args.steps / (e_total * 1e-3)
    h2d = 2 * 8 * points_per_rank
    d2h = 8 * (S + S * (nt + 1) + (S * n if want["mean"] else 0) + (S * n if want["var"] else 0))

    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return
    peak, peak_src = measured_peaks()
    abytes = alg_bytes_per_point(dom, wl) * points_per_rank
    achieved = abytes / (dom_launch_ms * 1e-3) / 1e9 if abytes else 0.0
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tr = json.load(f).get(wl.name, {}).get(dom)
        if tr is not None:
            traffic = tr
    F = core_flops_per_point(b, nt) * points_per_rank
    fp64_achieved = F / (total_ms / args.steps * 1e-3) / 1e12
    clocks = clk.summary()
    if partitioned:
        desc = f"{wl.description.split(' single')[0]} ONE series of {n_total} points partitioned over {ws} GPUs"
        par = f"{ws} ranks, contiguous time segments, NCCL all_gather of 2-separator records + all_reduce"
    else:
        desc = wl.description
        par = "single GPU" if ws == 1 else f"{ws} ranks, series sharded (independent series per rank)"
    line = {
        "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": ws, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE shapes; no public dataset)",
        "config": {"workload": desc, "config": wl.name, "points_per_gpu": int(points_per_rank),
                   "outputs": ["loglik"] + list(wl.outputs), "state_dim": b, "n_theta": nt,
                   "l2": "flushed between timed steps (256 MiB write, outside the events)",
                   "parallelism": par},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "note": f"algorithmic bytes = {alg_bytes_per_point(dom, wl):.0f} B/point x {points_per_rank} "
                             f"points per launch / {dom_launch_ms:.4f} ms mean launch; peak {peak_src}; the fused "
                             "path is FP64-bound (see roofline_fp64)"},
        "roofline_fp64": {"bound": "fp64", "achieved": fp64_achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                          "frac": fp64_achieved / FP64_PEAK_TFLOPS,
                          "note": "F_core = 8b^3 + 4b^2(1+n_theta) flop/point (SURVEY.md §8(d), lower bound) "
                                  "over the whole step; peak = measured DFMA microbenchmark"},
        "kernels_ms_per_step": {k: round(v, 5) for k, v in sorted(per_step.items(), key=lambda x: -x[1])},
        "launches_per_step": launches_per_step,
        "e2e": {"value": e2e_value, "unit": "points/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e_total / args.steps},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if ws == 1:
        # SURVEY.md §8(d) figure 1: the materialised-SymBTD solve operator at cfg2's size
        # (1 rhs, device-resident, compulsory bytes 8 (2 b^2 + 2 b) per block row)
        try:
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            import bench_solve
            line["solve_operator"] = bench_solve.measure(n=1_000_000, b=3, steps=10, device=local)
        except Exception as e:  # report, never break the metric line
            line["solve_operator"] = {"error": str(e)[:200]}
    if ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(wl)
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    ws, rank, local = dist_info()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()
