#!/usr/bin/env python
"""Benchmark: SpInGP loglik+grad time points/s (fp64) on B200.

Workloads (BASELINE.json configs, seeded synthetic inputs of the stated shapes; no
public dataset is involved):
  N = 1 (default)  cfg2 — Matérn-5/2 (b=3), one series of 1,000,000 points,
                   log-likelihood + gradient (var, len, σ) + posterior mean.  The line
                   also carries `per_config`: cfg1, cfg3, cfg4 (16 M points) and cfg5
                   (32 M points) measured the same way, each beside the CPU oracle.
  N > 1 (default)  cfg4 — EQ order 6 (b=6), ONE series of 16,000,000 points, strong
                   scaling: the series is cut into N contiguous time segments, rank r
                   uploads only its slice (+ the two halo times), reduces it to a
                   2-separator Schur record, the N records are all-gathered over NCCL,
                   the N-block reduced system is solved redundantly on every GPU,
                   segments are back-substituted and the partial sums all-reduced.
                   cfg3 shards its 4096 series over the ranks (no collective).
                   `scaling_reference` is the same workload on rank 0's GPU alone.

  value  : device-resident inputs, CUDA events around each step on the library's
           stream, L2 flushed (256 MiB write) between steps outside the events; the
           max over ranks of the summed step times.
  e2e    : the same metric through the host-pointer C ABI (spingp_eval /
           spingp_eval_batched): pinned host t,y -> H2D, kernels, D2H of loglik,
           gradient and the per-point outputs, every step.
  --gpus N without torchrun relaunches itself under torch.distributed.run with N ranks.
  --impl reference : the CPU oracle (restatement of the reference algorithm: Padé /
           Van Loan per step + block Thomas + Takahashi; the reference itself does not
           build here) on all host cores, on a bounded sample of the same workload per
           step, rank 0 only.
  --dry-run : CPU-only check of the launcher and the multi-rank plumbing (gloo, the
           host emulation of the kernels); prints a line marked "dry_run", never a
           bench value.
"""
import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

METRIC = "SpInGP loglik+grad time points/s (fp64), 1/2/4/8 B200, % HBM roofline"
FP64_PEAK_TFLOPS = 34.1  # DFMA microbenchmark on this pool's B200 (profiles/r01_box_probe.log)
PER_CONFIG_STEPS = {"cfg1": (5, 20), "cfg2": (5, 20), "cfg3": (3, 10), "cfg4": (3, 5), "cfg5": (2, 2)}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default=None, choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"],
                    help="default: cfg2 at N=1, cfg4 at N>1")
    ap.add_argument("--points", type=int, default=0, help="override N (testing only; not a bench value)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-per-config", action="store_true")
    ap.add_argument("--no-scaling-ref", action="store_true")
    ap.add_argument("--dry-run", action="store_true")
    ap.add_argument("--force-segments", action="store_true",
                    help="testing: run the N>1 segment protocol (NCCL collectives) even at one rank")
    return ap.parse_args()


def dist_info():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args):
    """--gpus N outside torchrun: run this script under torch.distributed.run, N ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.run(cmd, env=env).returncode


def config_name(args, ws):
    return args.config or ("cfg2" if ws == 1 else "cfg4")


# ------------------------------------------------------------------ workloads --

def load(name, points):
    from paper_1610_08035_b200 import datasets
    return datasets.make(name, **({"n": points} if points else {}))


def shard(wl, rank, ws, force_segments=False):
    """This rank's part of the workload: batched configs shard whole series, single
    series are cut into contiguous time segments (strong scaling)."""
    if ws == 1 and not (force_segments and not wl.batched):
        return dict(kind="single" if not wl.batched else "batched", t=wl.t, y=wl.y, theta=wl.theta, sigma=wl.sigma,
                    a=0, b=len(wl.t), n_total=wl.points)
    if wl.batched:
        S = wl.t.shape[0]
        a, b = rank * S // ws, (rank + 1) * S // ws
        return dict(kind="batched", t=wl.t[a:b], y=wl.y[a:b], theta=wl.theta[a:b], sigma=np.asarray(wl.sigma)[a:b],
                    a=a, b=b, n_total=wl.points)
    from paper_1610_08035_b200.partition import split, halos
    bounds = split(len(wl.t), ws)
    a, b = bounds[rank], bounds[rank + 1]
    tl, tr = halos(wl.t, bounds, rank)
    return dict(kind="segment", t=wl.t[a:b], y=wl.y[a:b], theta=wl.theta, sigma=wl.sigma, a=a, b=b,
                t_left=tl, t_right=tr, n_total=len(wl.t))


def describe(wl, ws):
    """The config dict both arms print (identical keys and values for one workload)."""
    if ws == 1:
        par = "single GPU"
    elif wl.batched:
        par = f"{ws} ranks, {wl.t.shape[0]} series sharded by series (no collective)"
    else:
        par = (f"{ws} ranks, contiguous time segments of one series, NCCL all_gather of the 2-separator "
               "records + all_reduce of the partial sums")
    return {"workload": wl.description, "config": wl.name, "points": wl.points,
            "outputs": ["loglik"] + list(wl.outputs), "parallelism": par,
            "l2": "flushed between timed steps (256 MiB write, outside the events)"}


def alg_bytes_per_point(kernel, wl):
    """Compulsory HBM bytes of one launch per time point (SURVEY.md §8(d) B_io split by kernel)."""
    outs = 8 * (("mean" in wl.outputs) + ("var" in wl.outputs))
    if kernel.startswith("k_fwd0"):
        return 16.0           # t, y read once
    if kernel.startswith("k_rev0"):
        return 16.0 + outs    # t, y read once, per-point outputs written once
    return 0.0


def core_flops_per_point(b, n_theta):
    """F_core = 8 b^3 + 4 b^2 (1 + n_θ), n_θ = kernel hyperparameters + 1 (σ)."""
    return 8 * b ** 3 + 4 * b ** 2 * (1 + n_theta)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------- CPU legs --

def cpu_rate(wl, threads, seconds):
    """The oracle (restatement of the reference CPU path) on `threads` host threads, on
    a bounded prefix of the workload sized to ~`seconds`: (points/s, sample text)."""
    import oracle_lib as O
    grad, mean, var = "grad" in wl.outputs, "mean" in wl.outputs, "var" in wl.outputs
    th = np.asarray(wl.theta, float)
    if wl.batched:
        S, n = wl.t.shape
        pilot = max(1, min(S, 8 * threads))
        t0 = time.perf_counter()
        O.evaluate_batched(wl.leaves, th[:pilot], wl.t[:pilot], wl.y[:pilot], wl.sigma[:pilot], grad=grad,
                           threads=threads)
        rate = pilot * n / (time.perf_counter() - t0)
        k = int(min(S, max(pilot, rate * seconds / n)))
        t0 = time.perf_counter()
        O.evaluate_batched(wl.leaves, th[:k], wl.t[:k], wl.y[:k], wl.sigma[:k], grad=grad, threads=threads)
        dt = time.perf_counter() - t0
        return k * n / dt, f"first {k} of {S} series x {n} points, loglik+grad, {dt:.1f} s"
    n = len(wl.t)
    pilot = min(n, 4000 * threads)
    t0 = time.perf_counter()
    O.evaluate(wl.leaves, th, wl.t[:pilot], wl.y[:pilot], wl.sigma, grad=grad, mean=mean, var=var, threads=threads)
    rate = pilot / (time.perf_counter() - t0)
    m = int(min(n, max(pilot, rate * seconds)))
    t0 = time.perf_counter()
    O.evaluate(wl.leaves, th, wl.t[:m], wl.y[:m], wl.sigma, grad=grad, mean=mean, var=var, threads=threads)
    dt = time.perf_counter() - t0
    outs = "loglik+grad" + ("+mean" if mean else "") + ("+var" if var else "")
    return m / dt, f"first {m} of {n} points, {outs}, {dt:.1f} s"


def cpu_baselines(wl, seconds=8.0):
    threads = os.cpu_count() or 1
    v, s = cpu_rate(wl, threads, seconds)
    v1, s1 = cpu_rate(wl, 1, seconds / 2)
    return ({"value": v, "unit": "points/s", "cores": threads, "kind": "port", "sample": s},
            {"value": v1, "unit": "points/s", "cores": 1, "kind": "port", "sample": s1})


def run_reference(args, ws, rank):
    """--impl reference: the oracle port on all host threads, rank 0 only; each step a
    bounded sample (a prefix) of the workload, so the run ends within minutes."""
    if rank != 0:
        return
    import oracle_lib as O
    name = config_name(args, max(ws, args.gpus))
    wl = load(name, args.points)
    threads = os.cpu_count() or 1
    grad, mean, var = "grad" in wl.outputs, "mean" in wl.outputs, "var" in wl.outputs
    th = np.asarray(wl.theta, float)
    budget = 3.0  # seconds of CPU work per step
    rate, _ = cpu_rate(wl, threads, 0.5)
    if wl.batched:
        S, n = wl.t.shape
        k = int(min(S, max(threads, rate * budget / n)))
        pts = k * n

        def step():
            O.evaluate_batched(wl.leaves, th[:k], wl.t[:k], wl.y[:k], wl.sigma[:k], grad=grad, threads=threads)
        sample = f"first {k} of {S} series x {n} points per step"
    else:
        n = len(wl.t)
        pts = int(min(n, max(20_000, rate * budget)))

        def step():
            O.evaluate(wl.leaves, th, wl.t[:pts], wl.y[:pts], wl.sigma, grad=grad, mean=mean, var=var,
                       threads=threads)
        sample = f"first {pts} of {n} points per step" if pts < n else f"full workload ({n} points) per step"
    for _ in range(args.warmup):
        step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = pts * args.steps / total
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": max(ws, args.gpus),
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "strong" if max(ws, args.gpus) > 1 else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE shapes)",
            "config": describe(wl, max(ws, args.gpus)),
            "cpu_baseline": {"value": value, "unit": "points/s", "cores": threads, "kind": "port",
                             "sample": sample + ", loglik+grad" + ("+mean" if mean else "") + ("+var" if var else "")
                                       + "; the reference itself cannot be built (no Eigen/GTest), oracle/ restates "
                                         "it"},
            "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------- GPU arm --

class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML every ~2 ms
    (B200_PROFILING.md clocks line).  `phase` tags each sample: 'soak' (a >= 1 s run of
    the same step right before the timed region) or 'timed'."""

    REASONS = [("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown")]

    def __init__(self, torch_device):
        self.dev = torch_device
        self.rows = []  # (phase, sm_mhz, max_mhz, reasons bitmask)
        self.phase = None
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
                if self.phase:
                    sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.rows.append((self.phase, sm, mx, rs))
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
        rows = [r for r in self.rows if r[0] == "timed"]
        window = "timed region"
        if len(rows) < 5:
            rows, window = self.rows, "clock soak (>= 1 s of the same step, just before) + timed region"
        reasons = set()
        for r in rows:
            for nm, attr in self.REASONS:
                if hasattr(self.nv, attr) and r[3] & getattr(self.nv, attr):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(r[1] for r in rows) if rows else None,
                "sm_max_mhz": max(r[2] for r in rows) if rows else None,
                "reasons": sorted(reasons), "samples": len(rows), "window": window}


class Runner:
    """One workload (or this rank's shard of it) bound to a context and device buffers."""

    def __init__(self, P, torch, ctx, dev, stream, wl, sh, ws, rank, dist):
        self.P, self.torch, self.ctx, self.dev, self.stream = P, torch, ctx, dev, stream
        self.wl, self.sh, self.ws, self.rank, self.dist = wl, sh, ws, rank, dist
        self.b, self.nt = P.kernel_dims(wl.leaves)
        outs = wl.outputs
        self.flags = P.WANT_GRAD | (P.WANT_MEAN if "mean" in outs else 0) | (P.WANT_VAR if "var" in outs else 0)
        t, y = sh["t"], sh["y"]
        self.S = t.shape[0] if t.ndim == 2 else 1
        self.n = t.shape[-1]
        self.points = int(t.size)
        f64 = torch.float64
        self.h_t = torch.from_numpy(np.ascontiguousarray(t)).pin_memory()
        self.h_y = torch.from_numpy(np.ascontiguousarray(y)).pin_memory()
        self.d_t = self.h_t.to(dev)
        self.d_y = self.h_y.to(dev)
        self.d_ll = torch.zeros(self.S, dtype=f64, device=dev)
        self.d_g = torch.zeros(self.S * (self.nt + 1), dtype=f64, device=dev)
        self.d_m = torch.zeros(self.S * self.n, dtype=f64, device=dev) if "mean" in outs else None
        self.d_v = torch.zeros(self.S * self.n, dtype=f64, device=dev) if "var" in outs else None
        self.segment = sh["kind"] == "segment"
        if self.segment:
            from paper_1610_08035_b200.partition import make_buffers
            self.bufs = make_buffers(torch, dev, wl.leaves, ws)
        # pinned host outputs of the e2e leg (caller-owned arrays the public API writes into)
        self.want = dict(grad=True, mean="mean" in outs, var="var" in outs)
        tot = self.S + self.S * (self.nt + 1) + self.S * self.n * (self.want["mean"] + self.want["var"])
        self.h_out = torch.empty(tot, dtype=f64).pin_memory()
        ho = self.h_out.numpy()
        k0 = 0
        self.outs = {"loglik": ho[k0:k0 + self.S]}
        k0 += self.S
        self.outs["grad"] = ho[k0:k0 + self.S * (self.nt + 1)].reshape(
            (self.S, self.nt + 1) if sh["kind"] == "batched" else (self.nt + 1,))
        k0 += self.S * (self.nt + 1)
        for key in ("mean", "var"):
            if self.want[key]:
                self.outs[key] = ho[k0:k0 + self.S * self.n].reshape(
                    (self.S, self.n) if sh["kind"] == "batched" else (self.n,))
                k0 += self.S * self.n
        self.h2d = 16 * self.points
        self.d2h = 8 * tot

    def ptr(self, x):
        return x.data_ptr() if x is not None else 0

    def step(self):
        sh, P = self.sh, self.P
        if self.segment:
            from paper_1610_08035_b200.partition import eval_partitioned
            eval_partitioned(self.ctx, self.wl.leaves, self.wl.theta, self.d_t.data_ptr(), self.d_y.data_ptr(), self.n,
                             sh["n_total"], sh["t_left"], sh["t_right"], self.rank, self.ws, self.wl.sigma, self.flags,
                             self.bufs, lambda o, i: self.dist.all_gather_into_tensor(o, i),
                             lambda x: self.dist.all_reduce(x), self.ptr(self.d_m), self.ptr(self.d_v))
        elif sh["kind"] == "batched":
            self.ctx.eval_batched_device(self.wl.leaves, sh["theta"], self.S, self.n, self.d_t.data_ptr(),
                                         self.d_y.data_ptr(), sh["sigma"], self.flags, self.d_ll.data_ptr(),
                                         self.d_g.data_ptr(), self.ptr(self.d_m), self.ptr(self.d_v))
        else:
            self.ctx.eval_device(self.wl.leaves, self.wl.theta, self.d_t.data_ptr(), self.d_y.data_ptr(), self.n,
                                 self.wl.sigma, self.flags, self.d_ll.data_ptr(), self.d_g.data_ptr(),
                                 self.ptr(self.d_m), self.ptr(self.d_v))

    def e2e_step(self):
        """Host inputs (pinned) -> device -> evaluation -> results to host, through the
        public API (the host-pointer C ABI; the segment protocol is device-side, so its
        copies are explicit here)."""
        if self.segment:
            self.d_t.copy_(self.h_t, non_blocking=True)
            self.d_y.copy_(self.h_y, non_blocking=True)
            self.step()
            nt1 = self.nt + 1
            self.h_out[0:1].copy_(self.bufs["loglik"], non_blocking=True)
            self.h_out[1:1 + nt1].copy_(self.bufs["grad"], non_blocking=True)
            k0 = 1 + nt1
            for d in (self.d_m, self.d_v):
                if d is not None:
                    self.h_out[k0:k0 + self.n].copy_(d, non_blocking=True)
                    k0 += self.n
            return
        if self.sh["kind"] == "batched":
            self.ctx.eval_batched(self.wl.leaves, self.sh["theta"], self.h_t.numpy(), self.h_y.numpy(),
                                  self.sh["sigma"], out=self.outs, **self.want)
        else:
            self.ctx.eval(self.wl.leaves, self.wl.theta, self.h_t.numpy(), self.h_y.numpy(), self.wl.sigma,
                          out=self.outs, **self.want)

    def barrier(self):
        self.torch.cuda.synchronize(self.dev)
        if self.ws > 1:
            self.dist.barrier()
        self.torch.cuda.synchronize(self.dev)

    def max_over_ranks(self, v):
        if self.ws == 1:
            return v
        tt = self.torch.tensor([v], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(tt, op=self.dist.ReduceOp.MAX)
        return float(tt.item())

    def measure(self, steps, warmup, flush, clk=None, soak_s=1.0):
        torch = self.torch
        for _ in range(max(3, warmup)):
            flush.zero_()
            self.step()
        self.ctx.status()
        self.barrier()
        if clk is not None:  # >= 1 s of the same step at steady clocks, sampled
            clk.phase = "soak"
            t0 = time.perf_counter()
            while True:
                flush.zero_()
                self.step()
                torch.cuda.synchronize(self.dev)
                done = time.perf_counter() - t0 >= soak_s
                if self.ws > 1:
                    f = torch.tensor([1.0 if done else 0.0], device=self.dev)
                    self.dist.all_reduce(f, op=self.dist.ReduceOp.MIN)
                    done = f.item() > 0
                if done:
                    break
            clk.phase = None
            self.barrier()
        launches0 = self.ctx.launch_count()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        if clk is not None:
            clk.phase = "timed"
        for k in range(steps):
            flush.zero_()  # L2 flush between timed steps, outside the events
            evs[k][0].record(self.stream)
            self.step()
            evs[k][1].record(self.stream)
        torch.cuda.synchronize(self.dev)
        if clk is not None:
            clk.phase = None
        launches = self.ctx.launch_count() - launches0
        self.ctx.status()  # raises on any device-side failure in the timed steps
        total_ms = self.max_over_ranks(float(sum(a.elapsed_time(b) for a, b in evs)))
        self.barrier()
        value = self.wl.points * steps / (total_ms * 1e-3) if self.ws > 1 else self.points * steps / (total_ms * 1e-3)

        # per-kernel breakdown (separate, untimed pass; CUDA events around every launch)
        self.ctx.set_profiling(True)
        kt = {}
        reps = 2
        for _ in range(reps):
            flush.zero_()
            self.step()
            for name, ms in self.ctx.kernel_times():
                kt.setdefault(name, []).append(ms)
        self.ctx.set_profiling(False)
        self.barrier()
        per_step = {k: sum(v) / reps for k, v in kt.items()}
        dom = max(per_step, key=per_step.get)

        # e2e through the public API
        e2e_steps = max(2, min(steps, 10))
        for _ in range(2):
            self.e2e_step()
        self.barrier()
        e_ms = []
        for _ in range(e2e_steps):
            ea = torch.cuda.Event(enable_timing=True)
            eb = torch.cuda.Event(enable_timing=True)
            ea.record(self.stream)
            self.e2e_step()
            eb.record(self.stream)
            eb.synchronize()
            e_ms.append(ea.elapsed_time(eb))
        e_total = self.max_over_ranks(float(sum(e_ms)))
        total_points = self.wl.points if self.ws > 1 else self.points
        return dict(value=value, ms_per_step=total_ms / steps, launches=int(launches), per_step=per_step, dom=dom,
                    dom_launch_ms=statistics.mean(kt[dom]),
                    launches_per_step={k: len(v) // reps for k, v in kt.items()},
                    e2e={"value": total_points * e2e_steps / (e_total * 1e-3), "unit": "points/s",
                         "h2d_bytes_per_step": self.h2d, "d2h_bytes_per_step": self.d2h,
                         "ms_per_step": e_total / e2e_steps, "steps": e2e_steps})

    def rooflines(self, m):
        peak, peak_src = measured_peaks()
        dom = m["dom"]
        abytes = alg_bytes_per_point(dom, self.wl) * self.points
        achieved = abytes / (m["dom_launch_ms"] * 1e-3) / 1e9 if abytes else 0.0
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            with open(tp) as f:
                traffic = json.load(f).get(self.wl.name, {}).get(dom)
        F = core_flops_per_point(self.b, self.nt + 1) * self.points
        fp64 = F / (m["ms_per_step"] * 1e-3) / 1e12
        return ({"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                 "frac": achieved / peak, "traffic": traffic,
                 "note": f"algorithmic bytes = {alg_bytes_per_point(dom, self.wl):.0f} B/point x {self.points} points "
                         f"per launch / {m['dom_launch_ms']:.4f} ms mean launch; peak {peak_src}; the fused path is "
                         "FP64-bound (see roofline_fp64)"},
                {"bound": "fp64", "achieved": fp64, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                 "frac": fp64 / FP64_PEAK_TFLOPS,
                 "note": f"F_core = 8b^3 + 4b^2(1+n_theta) = {core_flops_per_point(self.b, self.nt + 1)} flop/point "
                         f"(b={self.b}, n_theta={self.nt + 1} incl. sigma; SURVEY.md §8(d), lower bound) over the "
                         "whole step on this GPU; peak = measured DFMA microbenchmark"})


def run_ours(args, ws, rank, local):
    import torch
    import paper_1610_08035_b200 as P

    torch.cuda.set_device(local)
    dist = None
    dev = torch.device("cuda", local)
    if ws > 1 or args.force_segments:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    name = config_name(args, ws)
    wl = load(name, args.points)
    sh = shard(wl, rank, ws, args.force_segments)
    ctx = P.Context(local)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    flush = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device=dev)
    run = Runner(P, torch, ctx, dev, stream, wl, sh, ws, rank, dist)
    with ClockSampler(dev) as clk:
        m = run.measure(args.steps, args.warmup, flush, clk)
    clocks = clk.summary()
    roof, roof64 = run.rooflines(m)
    line = {
        "metric": METRIC, "value": m["value"], "unit": "points/s", "n_gpus": ws, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": m["ms_per_step"], "higher_is_better": True,
        "scaling": "strong" if ws > 1 and not wl.batched else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE shapes; no public dataset)",
        "config": describe(wl, ws),
        "points_per_gpu": run.points, "state_dim": run.b, "n_theta": run.nt + 1,
        "roofline": roof, "roofline_fp64": roof64,
        "kernels_ms_per_step": {k: round(v, 5) for k, v in sorted(m["per_step"].items(), key=lambda x: -x[1])},
        "launches_per_step": m["launches_per_step"],
        "e2e": m["e2e"], "gpu_launches": m["launches"], "clocks": clocks,
    }
    del run
    if (ws > 1 or args.force_segments) and not args.no_scaling_ref:
        # the same workload on rank 0's GPU alone (the other ranks wait): the 1-GPU point of
        # this job's scaling curve, measured in the same process and on the same box
        if rank == 0:
            r1 = Runner(P, torch, ctx, dev, stream, wl, shard(wl, 0, 1), 1, 0, None)
            m1 = r1.measure(max(2, min(args.steps, 5)), 3, flush)
            line["scaling_reference"] = {"n_gpus": 1, "value": m1["value"], "ms_per_step": m1["ms_per_step"],
                                         "efficiency": m["value"] / (ws * m1["value"]),
                                         "note": "same workload, one GPU, same job; efficiency = value / "
                                                 "(n_gpus x this value)"}
            del r1
        dist.barrier()
    if ws == 1:
        try:  # SURVEY.md §8(d) figure 1: the materialised-SymBTD solve operator at cfg2's size
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            import bench_solve
            line["solve_operator"] = bench_solve.measure(n=1_000_000, b=3, steps=10, device=local)
        except Exception as e:  # report, never break the metric line
            line["solve_operator"] = {"error": str(e)[:200]}
        if not args.no_cpu_baseline:
            line["cpu_baseline"], line["cpu_baseline_1core"] = cpu_baselines(wl)
        if not args.no_per_config and not args.points:
            line["per_config"] = per_config(P, torch, ctx, dev, stream, flush, skip=name,
                                            cpu=not args.no_cpu_baseline)
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist is not None:
        dist.destroy_process_group()


def per_config(P, torch, ctx, dev, stream, flush, skip, cpu=True):
    """Every other BASELINE config at N=1, measured like the headline (device value, e2e,
    both rooflines) beside the CPU oracle (all threads and 1 thread, bounded samples)."""
    out = {}
    for name in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
        if name == skip:
            continue
        try:
            wl = load(name, 0)
            run = Runner(P, torch, ctx, dev, stream, wl, shard(wl, 0, 1), 1, 0, None)
            w, k = PER_CONFIG_STEPS[name]
            m = run.measure(k, w, flush)
            roof, roof64 = run.rooflines(m)
            rec = {"workload": wl.description, "points": wl.points, "value": m["value"], "unit": "points/s",
                   "ms_per_step": m["ms_per_step"], "steps": k, "warmup": w, "e2e": m["e2e"], "roofline": roof,
                   "roofline_fp64": roof64,
                   "kernels_ms_per_step": {a: round(v, 5) for a, v in sorted(m["per_step"].items(),
                                                                             key=lambda x: -x[1])}}
            del run
            if cpu:
                rec["cpu_baseline"], rec["cpu_baseline_1core"] = cpu_baselines(wl, seconds=5.0)
            out[name] = rec
        except Exception as e:  # report, never break the metric line
            out[name] = {"error": str(e)[:300]}
    return out


# ----------------------------------------------------------------- dry run --

def run_dry(args, ws, rank):
    """CPU-only plumbing check (gloo; the kernels' host emulation): sharding, halos, the
    record all_gather / partial all_reduce, max-over-ranks timing and the JSON line."""
    import torch
    import torch.distributed as dist
    import emu_lib as E
    if ws > 1:
        dist.init_process_group("gloo")
    name = config_name(args, ws)
    wl = load(name, args.points or 4000)
    sh = shard(wl, rank, ws)
    t0 = time.perf_counter()
    if sh["kind"] == "segment":
        nrec, npart = E.seg_sizes(wl.leaves)
        rec = torch.from_numpy(E.seg_forward(wl.leaves, wl.theta, sh["t"], sh["y"], sh["t_left"], sh["t_right"], rank,
                                             ws, wl.sigma, flags=1))
        recs = [torch.zeros(nrec, dtype=torch.float64) for _ in range(ws)]
        dist.all_gather(recs, rec)
        part, _, _ = E.seg_reverse(torch.cat(recs).numpy(), sh["b"] - sh["a"], npart, mean=False, var=False)
        tp = torch.from_numpy(part)
        dist.all_reduce(tp)
        ll, g = E.seg_finalize(tp.numpy(), len(wl.theta), sh["n_total"], wl.sigma)
        loglik = [float(ll)]
    else:
        ts, ys = np.atleast_2d(sh["t"]), np.atleast_2d(sh["y"])
        th = np.atleast_2d(sh["theta"])
        sg = np.broadcast_to(np.asarray(sh["sigma"], float), (ts.shape[0],))
        loglik = [float(E.evaluate(wl.leaves, th[s], ts[s], ys[s], sg[s], grad=False, mean=False, var=False)["loglik"])
                  for s in range(min(2, ts.shape[0]))]  # the first series of each shard
    dt = time.perf_counter() - t0
    if ws > 1:
        tt = torch.tensor([dt], dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
        if sh["kind"] == "batched":
            gathered = [None] * ws
            dist.all_gather_object(gathered, loglik)
            loglik = [v for part in gathered for v in part]
    if rank == 0:
        print(json.dumps({"dry_run": "CPU plumbing check (gloo + host emulation); not a bench value",
                          "n_gpus": ws, "config": describe(wl, ws), "shard": [sh["a"], sh["b"]],
                          "loglik": loglik, "ms": dt * 1e3}), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    ws, rank, local = dist_info()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(relaunch(args))
    if args.gpus > 1 and ws == 1 and args.impl == "ours":
        raise SystemExit("--gpus N > 1 under a launcher with WORLD_SIZE=1")
    if args.dry_run:
        run_dry(args, ws, rank)
        return
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()
