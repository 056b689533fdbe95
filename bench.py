#!/usr/bin/env python
"""bench.py — batched symmetric-stair PCG on B200 (BASELINE.json config c4).

A "step" = one pass of the hot path (K1 Schur formation -> K3 persistent
symmetric-stair PCG, fp64, eps 1e-8, lambda0 = 0) over one batch of 4096
independent synthetic iiwa-like KKT systems (K = 64 knots, nx = 14, nu = 7)
per GPU. Weak scaling: every rank owns its own 4096 systems (contiguous
batch-index shard, seeds seed0 + global index), no inter-GPU traffic.

  value : batched solves/s, whole job, inputs resident in HBM
          (CUDA events on the launch stream, max over ranks)
  e2e   : same metric through the host-buffer C-ABI call b2p_solve_batched
          (pinned host KKT in, H2D + solve + D2H of lambda + status inside
          the timed region; host wall clock around the call)
Also reported (rank 0, outside the timed region): parity of the bench batch
against the oracle, c4 at eps 1e-4, and every other BASELINE row — c1 / c3
latency, c2 per preconditioner x eps, the c5 condition-number sweep — each
beside the CPU reference latency measured on this host in the same run.

--gpus N without WORLD_SIZE in the environment re-launches this script under
torch.distributed.run with N ranks (one per GPU).

--impl reference: the reference's CPU implementation of the path (the
oracle restatement; the reference cannot be compiled here)
on all host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2309_08079_b200.types import PcgConfig, PcgVariant, PrecondKind  # noqa: E402

METRIC = "batched PCG solves/s (symmetric-stair, fp64)"
UNIT = "solves/s"
# Measured DFMA peak of this pool's B200 (scripts/micro/lat_bench.cu: 60.9 FMA/clk/SM
# x 148 SMs x 1.965 GHz x 2); MEASURED_PEAKS.json carries no fp64 figure.
FP64_PEAK_TFLOPS = 35.4


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--batch", type=int, default=4096, help="systems per GPU")
    ap.add_argument("--knots", type=int, default=64)
    ap.add_argument("--nx", type=int, default=14)
    ap.add_argument("--nu", type=int, default=7)
    ap.add_argument("--eps", type=float, default=1e-8)
    ap.add_argument("--seed", type=int, default=2309)
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="CPU baseline sample budget (seconds)")
    ap.add_argument("--ref-budget", type=float, default=150.0,
                    help="--impl reference: total CPU seconds over warmup + steps")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-latency", action="store_true")
    return ap.parse_args()


def workload(a):
    return {
        "workload": (f"c4: {a.batch} independent synthetic iiwa-like KKT systems per GPU "
                     f"(random_kkt, seeds seed0+i), K={a.knots} knots (N={a.knots - 1}), "
                     f"nx={a.nx}, nu={a.nu}; build_schur + symmetric-stair build + PCG to "
                     f"eps={a.eps:g}, lambda0=0"),
        "batch_per_gpu": a.batch, "knots": a.knots, "nx": a.nx, "nu": a.nu,
        "precond": "symstair", "epsilon": a.eps, "dtype": "fp64",
        "l2": "inputs larger than L2 (1.19 GB per GPU vs 126 MB L2)",
        "parallelism": "batch-index shards, one process per GPU",
    }


# ------------------------------------------------------------------ helpers
def kkt_bytes(N, n, m, w=8):
    K = N + 1
    return w * (K * n * n + K * n + N * m * m + N * m + N * n * n + N * n * m + N * n + 2 * n)


def algorithmic(N, n, m, iters, w=8):
    """Per-system algorithmic bytes / flops."""
    K = N + 1
    nn = n * n
    b_in = kkt_bytes(N, n, m, w)
    b_k1 = b_in + w * (3 * K * nn + K * nn + K * n)      # read KKT, write S, theta^-1, gamma
    b_k3 = w * (3 * K * nn + K * nn + K * n + K * n)     # read S, theta^-1, gamma; write lambda
    b_full = b_in + 2 * K * n * w                         # compulsory: KKT in, lambda0 + lambda
    f_form = (K - 1) * (17 * n ** 3 + 2.33 * m ** 3 + 2 * n * m * (n + m)) + 2.33 * n ** 3
    f_iter = 4 * (3 * K - 2) * nn + 10 * K * n
    return dict(b_in=b_in, b_k1=b_k1, b_k3=b_k3, b_full=b_full, f_form=f_form,
                f_iter=f_iter, f_full=f_form + (iters + 1) * f_iter)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class ClockSampler:
    """SM clock + throttle reasons sampled every `period` s DURING the timed
    region through NVML (nvidia-ml-py); nvidia-smi -lms 20 if NVML is missing."""

    # nvmlClocksEventReasons bits (nvml.h)
    BITS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
            0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index, pci_bus_id=None, period=0.002):
        self.index = index
        self.pci = pci_bus_id
        self.period = period
        self.sm, self.mx, self.reasons = [], [], set()
        self.proc = None
        self.nvml = None
        self.stop = threading.Event()
        self.source = "none"

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = None
            if self.pci:  # the NVML device whose PCI bus id is the CUDA device's
                want = str(self.pci).lower().split(":", 1)[-1]
                for i in range(nv.nvmlDeviceGetCount()):
                    hi = nv.nvmlDeviceGetHandleByIndex(i)
                    bid = nv.nvmlDeviceGetPciInfo(hi).busId
                    bid = (bid.decode() if isinstance(bid, bytes) else str(bid)).lower()
                    if bid.endswith(want):
                        h = hi
                        break
            h = h or nv.nvmlDeviceGetHandleByIndex(self.index)
            self.nvml, self.h = nv, h
            self.mx.append(float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)))
            self.t = threading.Thread(target=self._poll_nvml, daemon=True)
            self.t.start()
            self.source = f"nvml every {self.period * 1e3:g} ms"
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read_smi, daemon=True)
            self.t.start()
            self.source = "nvidia-smi -lms 20"
        except Exception:
            self.proc = None
        return self

    def _poll_nvml(self):
        nv, h = self.nvml, self.h
        get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                r = int(get_r(h))
                self.reasons |= {name for bit, name in self.BITS.items() if r & bit}
            except Exception:
                pass
            time.sleep(self.period)

    def _read_smi(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.proc.stdout:
            p = [x.strip() for x in line.split(",")]
            if len(p) < 6:
                continue
            try:
                self.sm.append(float(p[0]))
                self.mx.append(float(p[1]))
            except ValueError:
                continue
            self.reasons |= {names[i] for i in range(4) if p[2 + i].lower().startswith("active")}

    def __exit__(self, *exc):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.nvml:
            self.t.join(timeout=1)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": max(self.mx) if self.mx else None,
                    "reasons": ["unsampled"], "samples": 0, "source": self.source}
        return {"sm_mhz": statistics.median(self.sm), "sm_min_mhz": min(self.sm),
                "sm_max_mhz": max(self.mx) if self.mx else None,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": self.source}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def maybe_relaunch(a):
    """--gpus N > 1 outside torchrun: re-exec under torch.distributed.run with N
    ranks (127.0.0.1 rendezvous); fail loudly if fewer GPUs are visible."""
    if a.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    if a.impl == "b200":
        import torch
        have = torch.cuda.device_count()
        if have < a.gpus:
            sys.stderr.write(f"bench.py: --gpus {a.gpus} but {have} CUDA device(s) visible\n")
            sys.exit(2)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def _orc():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as orc
    orc.build()
    return orc


# ------------------------------------------------------------------ CPU arm
def cpu_sample(a, seconds, seed0, want_lambda=False, native=False):
    """Oracle (restated reference) on all host threads over a bounded sample of
    the c4 workload (systems seed0 .. seed0 + sample - 1)."""
    orc = _orc()
    threads = os.cpu_count() or 1
    N = a.knots - 1
    cfg = PcgConfig(epsilon=a.eps)
    # calibrate with a small batch, then size the sample for ~`seconds`
    cal = max(threads, 8)
    kb = orc.random_kkt_batch(seed0, cal, N, a.nx, a.nu)
    secs, _, _ = orc.solve_batch(kb, PrecondKind.symmetric_stair, 1, cfg, threads=threads,
                                 want_lambda=False, native=native)
    per = secs / cal
    sample = int(min(a.batch, max(cal, seconds / max(per, 1e-9))))
    kb = orc.random_kkt_batch(seed0, sample, N, a.nx, a.nu)
    secs, lam, reps = orc.solve_batch(kb, PrecondKind.symmetric_stair, 1, cfg, threads=threads,
                                      want_lambda=want_lambda, native=native)
    return {"value": sample / secs, "sample": sample, "secs": secs, "threads": threads,
            "iters": float(np.mean([r.iterations for r in reps])), "lambda": lam,
            "iterations": np.array([r.iterations for r in reps]),
            "converged": np.array([r.converged for r in reps])}


def run_reference(a, world, rank):
    if rank != 0:
        return
    steps, warm = a.steps, a.warmup
    budget = max(0.5, min(20.0, a.ref_budget / max(1, steps + warm)))
    for _ in range(warm):
        cpu_sample(a, budget / 4, a.seed)
    vals, t_total, r = [], 0.0, None
    for _ in range(steps):
        r = cpu_sample(a, budget, a.seed)
        vals.append(r["value"])
        t_total += r["secs"]
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": a.gpus, "steps": steps, "warmup": warm,
        "ms_per_step": 1e3 * t_total / steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (random_kkt, seeded)",
        "config": workload(a),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": r["threads"], "kind": "port",
                         "sample": f"{r['sample']} systems of the c4 workload per step "
                                   f"(oracle restatement of proj/src, g++ -O3 -DNDEBUG, "
                                   f"parallel_for over instances as trajopt_cli.cpp:155; "
                                   f"inputs from the oracle's own generator)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "pcg_iters_mean": r["iters"],
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
PATHS = {0: "split", 1: "one-CTA fused", 2: "fused cluster", 3: "fused grid", 4: "fused small"}
KIND_NAMES = {"identity": PrecondKind.identity, "jacobi": PrecondKind.block_jacobi,
              "stair": PrecondKind.stair, "symstair": PrecondKind.symmetric_stair}


def c1_graph_latency(api, torch, local, reps=200, N=31, n=14, m=7):
    from paper_2309_08079_b200.types import KKTSystem
    kk = api.random_kkt(1, N, n, m)
    dev = [torch.from_numpy(np.ascontiguousarray(x)[None]).to(f"cuda:{local}") for x in kk.arrays()]
    kd = KKTSystem(N, n, m, *dev)
    lam = torch.empty((1, (N + 1) * n), dtype=torch.float64, device=f"cuda:{local}")
    ctx = api.Context(local)
    s = torch.cuda.Stream(device=local)
    ctx.set_stream(s.cuda_stream)
    cfg = PcgConfig(epsilon=1e-8)
    with torch.cuda.stream(s):
        for _ in range(3):  # workspaces allocated before capture
            api.solve_batched_device(kd, lam.data_ptr(), 1, PrecondKind.symmetric_stair, 1, cfg,
                                     ctx=ctx)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            api.solve_batched_device(kd, lam.data_ptr(), 1, PrecondKind.symmetric_stair, 1, cfg,
                                     ctx=ctx)
        for _ in range(5):
            g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
        s.synchronize()
    want = api.solve(kk, PrecondKind.symmetric_stair, 1, cfg).lambda_
    ok = bool(np.array_equal(lam.cpu().numpy()[0], want))
    ctx.close()
    return {"us_per_solve": e0.elapsed_time(e1) * 1e3 / reps, "replays": reps,
            "matches_eager": ok}


def shape_batch(api, torch, local, B, N, n, m, reps=5, check=64, c4_tflops=None):
    """An off-BASELINE shape as a device-resident batch (the reference forms and
    solves any (n, m), schur.cpp:38-82): solves/s, the kernel that ran,
    reference-algorithm flop throughput beside the c4 one (SURVEY 8d F_full with
    the measured iterations), and per-system parity against the oracle on the
    first `check` systems (outside the timed region)."""
    r = nmpc_batch_throughput(api, torch, local, B=B, N=N, n=n, m=m, reps=reps, seed=4242,
                              keep=True)
    lam, reports, kb = r.pop("_lam"), r.pop("_reports"), r.pop("_kkt")
    alg = algorithmic(N, n, m, r["iters_mean"])
    r["tflops_ref_algorithm"] = B * alg["f_full"] / (r["ms_per_batch"] * 1e-3) / 1e12
    if c4_tflops:
        r["per_flop_vs_c4"] = r["tflops_ref_algorithm"] / c4_tflops
    orc = _orc()
    sub = orc.random_kkt_batch(4242, check, N, n, m)
    _, lo, ro = orc.solve_batch(sub, PrecondKind.symmetric_stair, 1, PcgConfig(epsilon=1e-8))
    it_gpu = np.asarray(reports.iterations[:check])
    it_orc = np.array([x.iterations for x in ro])
    lg = lam[:check]
    scale = np.maximum(1.0, np.abs(lo).max(axis=1))
    r["parity"] = {"systems": check, "iterations_equal": int((it_gpu == it_orc).sum()),
                   "lambda_rel_err_max": float((np.abs(lg - lo).max(axis=1) / scale).max()),
                   "tolerance": 1e-10}
    return r


def nmpc_batch_throughput(api, torch, local, B=4096, N=32, n=2, m=1, reps=5, seed=77,
                          keep=False):
    """Many independent NMPC-shape systems (double-integrator / pendulum size, the
    SQP callers' shape) through the small-block kernel, device-resident, CUDA events."""
    from paper_2309_08079_b200.types import KKTSystem
    kb = api.random_kkt_batch(seed, B, N, n, m)
    dev = [torch.from_numpy(np.ascontiguousarray(x)).to(f"cuda:{local}") for x in kb.arrays()]
    kd = KKTSystem(N, n, m, *dev)
    lam = torch.empty((B, (N + 1) * n), dtype=torch.float64, device=f"cuda:{local}")
    ctx = api.Context(local)
    s = torch.cuda.Stream(device=local)
    ctx.set_stream(s.cuda_stream)
    cfg = PcgConfig(epsilon=1e-8)
    with torch.cuda.stream(s):
        reports = api.solve_batched_device(kd, lam.data_ptr(), B, PrecondKind.symmetric_stair, 1,
                                           cfg, ctx=ctx, want_reports=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            api.solve_batched_device(kd, lam.data_ptr(), B, PrecondKind.symmetric_stair, 1, cfg,
                                     ctx=ctx)
        e1.record(s)
        s.synchronize()
    path = ctx.last_path()
    ctx.close()
    ms = e0.elapsed_time(e1) / reps
    out = {"systems_per_s": B / (ms * 1e-3), "ms_per_batch": ms, "batch": B, "knots": N + 1,
           "nx": n, "nu": m, "kernel": PATHS.get(path, str(path)),
           "iters_mean": float(np.mean([r.iterations for r in reports]))}
    if keep:
        out.update(_lam=lam.cpu().numpy(), _reports=reports, _kkt=kb)
    return out


def gpu_single(api, kk, kind, eps, dtype=np.float64, reps=20, warm=5):
    """One fused solve through api.solve (the public API): device time (CUDA events
    around the kernels) and host wall clock of the whole call (packing, H2D,
    launch, sync, D2H, Python), medians."""
    dev, wall, r = [], [], None
    for i in range(warm + reps):
        t0 = time.perf_counter()
        r = api.solve(kk, kind, 1, PcgConfig(epsilon=eps), dtype=dtype)
        t1 = time.perf_counter()
        if i >= warm:
            dev.append(r.report.wall_time * 1e6)
            wall.append((t1 - t0) * 1e6)
    return {"us_device_median": statistics.median(dev), "us_device_min": min(dev),
            "us_host_wall_median": statistics.median(wall), "iterations": r.report.iterations,
            "converged": r.report.converged,
            "kernel": PATHS.get(api.context().last_path(), "?")}, r


def cpu_single(orc, kk, kind, eps, reps):
    """The CPU reference on this host (oracle restatement, g++ -O3): full scope
    (build_schur + build_preconditioner + pcg_solve) on 1 core, and the
    block-parallel PCG (pcg_solve_block_parallel, deterministic reductions) on
    every core; medians of `reps`."""
    def med(f):
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            f()
            ts.append((time.perf_counter() - t0) * 1e6)
        return statistics.median(ts)
    sch = orc.build_schur(kk)
    P = orc.build_preconditioner(sch, kind)
    z = sch.gamma * 0
    orc.set_threads(1)
    full = med(lambda: orc.solve(kk, kind, 1, PcgConfig(epsilon=eps)))
    r = orc.solve(kk, kind, 1, PcgConfig(epsilon=eps))
    orc.set_threads(0)
    par = med(lambda: orc.pcg_solve_auto(sch.S, P, sch.gamma, z, PcgConfig(
        epsilon=eps, variant=PcgVariant.block_parallel, deterministic_reductions=True)))
    return {"us_full_scope_1core": full, "us_pcg_block_parallel_all_cores": par,
            "iterations": r.report.iterations}, r


def kappa_estimate(S):
    """kappa(S) = lambda_max / lambda_min by Lanczos (scipy eigsh; shift-invert
    at 0 for lambda_min) on the sparse block-tridiagonal S."""
    import scipy.sparse as sp
    from scipy.sparse.linalg import eigsh
    d = S.data
    K, _, n, _ = d.shape
    blocks, idx, ptr = [], [], [0]
    for b in range(K):
        for s in range(3):
            c = b - 1 + s
            if 0 <= c < K:
                blocks.append(d[b, s])
                idx.append(c)
        ptr.append(len(idx))
    A = sp.bsr_matrix((np.array(blocks), np.array(idx), np.array(ptr)),
                      shape=(K * n, K * n)).tocsc()
    lmax = eigsh(A, k=1, which="LA", return_eigenvectors=False)[0]
    lmin = eigsh(A, k=1, sigma=0, which="LM", return_eigenvectors=False)[0]
    return float(lmax / lmin)


def baseline_rows(api, torch, local):
    """Every BASELINE.json config other than the c4 headline, each GPU number
    beside the CPU reference on this host and the oracle's iteration count."""
    orc = _orc()
    out = {"what": "device time = CUDA events around the fused kernel(s); host wall = the "
                   "api.solve call (Python, ctypes, pinned staging, H2D, kernel, D2H); "
                   "CPU = oracle restatement on this host (g++ -O3 -DNDEBUG), full scope on "
                   "1 core and block-parallel PCG on all cores",
           "host_threads": os.cpu_count()}

    def row(kk, kind, eps, dtype=np.float64, reps=20, cpu_reps=11, cpu=True):
        g, gr = gpu_single(api, kk, KIND_NAMES[kind], eps, dtype, reps=reps)
        o = orc.solve(kk, KIND_NAMES[kind], 1, PcgConfig(epsilon=eps),
                      dtype=dtype)
        g["oracle_iterations"] = o.report.iterations
        g["iterations_equal"] = g["iterations"] == o.report.iterations
        scale = max(1.0, float(np.abs(o.lambda_).max()))
        g["lambda_rel_err"] = float(np.abs(gr.lambda_ - o.lambda_).max()) / scale
        if cpu:
            c, _ = cpu_single(orc, kk, KIND_NAMES[kind], eps, cpu_reps)
            g["cpu"] = c
            g["speedup_full_scope_vs_1core"] = c["us_full_scope_1core"] / g["us_host_wall_median"]
        return g

    # c1: K 32, n 14, m 7, fp64, symstair, eps 1e-8 (+ the launch floor via a CUDA graph)
    kk1 = api.random_kkt(1, 31, 14, 7)
    out["c1"] = {"knots": 32, "nx": 14, "nu": 7, "dtype": "fp64",
                 "symstair_1e-08": row(kk1, "symstair", 1e-8)}
    try:
        out["c1"]["graph"] = c1_graph_latency(api, torch, local)
    except Exception as exc:
        out["c1"]["graph"] = {"error": str(exc)[:200]}
    # c2: K 128 — jacobi vs stair vs symstair at eps 1e-8 and 1e-4
    kk2 = api.random_kkt(2, 127, 14, 7)
    out["c2"] = {"knots": 128, "nx": 14, "nu": 7, "dtype": "fp64"}
    for kind in ("jacobi", "stair", "symstair"):
        for eps in (1e-8, 1e-4):
            out["c2"][f"{kind}_{eps:g}"] = row(kk2, kind, eps, reps=15, cpu_reps=5)
    # c3: K 256, n 12, m 4, fp32 (multi-SM single solve) at eps 1e-4 and 1e-8; the
    # CPU reference is fp64-only, so the fp32 oracle gives the iteration parity
    kk3 = api.random_kkt(3, 255, 12, 4)
    out["c3"] = {"knots": 256, "nx": 12, "nu": 4, "dtype": "fp32",
                 "note": "GPU and oracle in fp32; CPU latency is the fp64 reference"}
    for eps in (1e-4, 1e-8):
        out["c3"][f"symstair_{eps:g}"] = row(kk3, "symstair", eps, dtype=np.float32, reps=15,
                                             cpu_reps=3)
    # c5: K 512, n 28, m 14 — condition-number sweep over random_kkt_scaled
    sweep = []
    for fl in (1.0, 0.1, 0.01, 0.001):
        for cp in (0.5, 1.0, 2.0):
            kk5 = api.random_kkt_scaled(5, 511, 28, 14, fl, cp)
            g = row(kk5, "symstair", 1e-8, reps=5, cpu_reps=1, cpu=True)
            g.update({"diag_floor": fl, "coupling": cp,
                      "kappa_S": kappa_estimate(orc.build_schur(kk5).S)})
            sweep.append(g)
    out["c5"] = {"knots": 512, "nx": 28, "nu": 14, "dtype": "fp64", "epsilon": 1e-8,
                 "base_random_kkt": row(api.random_kkt(5, 511, 28, 14), "symstair", 1e-8,
                                        reps=10, cpu_reps=3),
                 "kappa_sweep": sweep}
    orc.set_threads(0)
    return out


def run_b200(a, world, rank, local):
    import torch
    import paper_2309_08079_b200.api as api

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = api.Context(local)
    # one explicit stream: the library launches on it and the timing events
    # are recorded on it (torch.cuda.Event sees only the stream it is given)
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)

    N, n, m, B = a.knots - 1, a.nx, a.nu, a.batch
    D = (N + 1) * n
    cfg = PcgConfig(epsilon=a.eps)
    from paper_2309_08079_b200.sharding import max_over_ranks, weak_shard
    first, _last = weak_shard(B, rank)
    seed0 = a.seed + first  # system i of the job <- seed + i (bench-pcg rule)

    def pinned(shape, dt):
        return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()

    kb = api.random_kkt_batch(seed0, B, N, n, m, alloc=pinned)
    # device-resident copy (value leg)
    dev = [torch.from_numpy(x).to(f"cuda:{local}", non_blocking=True) for x in kb.arrays()]
    from paper_2309_08079_b200.types import KKTSystem
    kd = KKTSystem(N, n, m, *dev)
    lam_dev = torch.empty((B, D), dtype=torch.float64, device=f"cuda:{local}")
    torch.cuda.synchronize()

    def step(c=cfg, out=lam_dev):
        api.solve_batched_device(kd, out.data_ptr(), B, PrecondKind.symmetric_stair, 1, c,
                                 ctx=ctx)

    def barrier():
        if dist is not None:
            dist.barrier()

    def allmax(x):
        return max_over_ranks(x, dist, device=f"cuda:{local}")

    # warm-up (also validates every system once)
    reps = api.solve_batched_device(kd, lam_dev.data_ptr(), B, PrecondKind.symmetric_stair, 1,
                                    cfg, ctx=ctx, want_reports=True)
    iters = reps.iterations
    assert reps.converged.all(), "unconverged systems in the bench batch"
    for _ in range(max(0, a.warmup - 1)):
        step()
    torch.cuda.synchronize()

    # ---- timed region: value (HBM-resident inputs)
    launches0 = ctx.kernel_launches()
    ctx.phase_accounting(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    try:
        pci = torch.cuda.get_device_properties(local).pci_bus_id
    except Exception:
        pci = None
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local, pci) as clk:
        ev0.record(stream)
        for _ in range(a.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    elapsed_ms = allmax(ev0.elapsed_time(ev1))
    k1_ms, k3_ms, tot_ms, nsolves = ctx.phase_totals()
    ctx.phase_accounting(False)
    launches = ctx.kernel_launches() - launches0
    value = world * B * a.steps / (elapsed_ms * 1e-3)
    lam_host_dev = lam_dev.cpu().numpy()

    # ---- c4 at the NMPC tolerance eps 1e-4, same batch, same timing
    c4_eps4 = None
    if not a.no_latency:
        cfg4 = PcgConfig(epsilon=1e-4)
        lam4 = torch.empty_like(lam_dev)
        rep4 = api.solve_batched_device(kd, lam4.data_ptr(), B, PrecondKind.symmetric_stair, 1,
                                        cfg4, ctx=ctx, want_reports=True)
        for _ in range(2):
            step(cfg4, lam4)
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.steps):
            step(cfg4, lam4)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms4 = allmax(e0.elapsed_time(e1))
        c4_eps4 = {"value": world * B * a.steps / (ms4 * 1e-3), "unit": UNIT,
                   "ms_per_step": ms4 / a.steps, "epsilon": 1e-4,
                   "pcg_iters": {"mean": float(rep4.iterations.mean()),
                                 "min": int(rep4.iterations.min()),
                                 "max": int(rep4.iterations.max())},
                   "lambda": lam4[:256].cpu().numpy(),
                   "iterations": rep4.iterations[:256]}

    # ---- e2e: host buffers through the C-ABI (pinned in, pinned out); host wall
    # clock around each call (the call returns after its final synchronisation)
    e2e = None
    if not a.no_e2e:
        lam_host = torch.empty((B, D), dtype=torch.float64, pin_memory=True).numpy()
        ctx_h = api.Context(local)
        api.solve_batched(kb, PrecondKind.symmetric_stair, 1, cfg, lambda_out=lam_host, ctx=ctx_h)
        barrier()
        wall_s, ev_ms = 0.0, 0.0
        for _ in range(a.steps):
            t0 = time.perf_counter()
            api.solve_batched(kb, PrecondKind.symmetric_stair, 1, cfg, lambda_out=lam_host,
                              ctx=ctx_h)
            wall_s += time.perf_counter() - t0
            ev_ms += ctx_h.last_solve_ms()
        barrier()
        wall_s = allmax(wall_s)
        ev_ms = allmax(ev_ms)
        assert np.array_equal(lam_host, lam_host_dev), "e2e/device outputs differ"
        sysout = 56  # sizeof(SysOut) copied back per system
        h2d = ctx_h.last_h2d_bytes()  # what the call moved (Q_k / R_k as lower triangles)
        e2e = {"value": world * B * a.steps / wall_s, "unit": UNIT,
               "h2d_bytes_per_step": h2d,
               "h2d_bytes_full_blocks": B * kkt_bytes(N, n, m),
               "d2h_bytes_per_step": B * (D * 8 + sysout + 4),
               "timing": "host wall clock around b2p_solve_batched",
               "value_cuda_events": world * B * a.steps / (ev_ms * 1e-3),
               "path": "b2p_solve_batched (host pinned buffers, 2-stream chunked H2D/compute/D2H; "
                       "Q_k and R_k sent as lower triangles and mirrored on the device — the "
                       "reference's LLT / LDLT read only the lower triangle, schur.cpp:16)"}
        ctx_h.close()

    # ---- every other BASELINE row (rank 0)
    rows = None
    latency = None
    if not a.no_latency and rank == 0:
        rows = baseline_rows(api, torch, local)
        latency = {"c1_us_median": rows["c1"]["symstair_1e-08"]["us_device_median"],
                   "c1_us_host_wall_median": rows["c1"]["symstair_1e-08"]["us_host_wall_median"]}
        kq = api.random_kkt(11, 32, 2, 1)
        wall = []
        rq = None
        for i in range(45):
            t0 = time.perf_counter()
            rq, _dz = api.sqp_step(kq, PrecondKind.symmetric_stair, 1, PcgConfig(epsilon=1e-8))
            if i >= 5:
                wall.append((time.perf_counter() - t0) * 1e6)
        latency["sqp_step_n2"] = {"us_median_host_wall": statistics.median(wall),
                                  "us_device": rq.report.wall_time * 1e6,
                                  "iterations": rq.report.iterations, "knots": 33, "nx": 2,
                                  "nu": 1, "kernel": PATHS.get(api.context().last_path(), "?")}
        try:
            latency["nmpc_graph_n2"] = c1_graph_latency(api, torch, local, N=32, n=2, m=1)
        except Exception as exc:
            latency["nmpc_graph_n2"] = {"error": str(exc)[:200]}
        try:
            latency["nmpc_batch_n2"] = nmpc_batch_throughput(api, torch, local)
        except Exception as exc:
            latency["nmpc_batch_n2"] = {"error": str(exc)[:200]}
        # off-BASELINE shapes: quadrotor-like n12 m4, n7 m2 and
        # odd n13 m7 (one-CTA kernel on an identity-padded n + 1)
        c4_tf = B * algorithmic(N, n, m, float(np.mean(iters)))["f_full"] / (
            elapsed_ms / a.steps * 1e-3) / 1e12
        shapes = {}
        for (sn, sm_) in ((12, 4), (7, 2), (13, 7)):
            try:
                shapes[f"n{sn}_m{sm_}_K{N + 1}"] = shape_batch(api, torch, local, B, N, sn, sm_,
                                                               c4_tflops=c4_tf)
            except Exception as exc:
                shapes[f"n{sn}_m{sm_}_K{N + 1}"] = {"error": str(exc)[:200]}
        latency["off_baseline_shapes"] = shapes

    # ---- reconstruct_primal on the same batch
    primal = None
    if rank == 0:
        P = (N + 1) * n + N * m
        dz_dev = torch.empty((B, P), dtype=torch.float64, device=f"cuda:{local}")
        for _ in range(3):
            api.reconstruct_primal_batched_device(kd, lam_dev.data_ptr(), dz_dev.data_ptr(), B,
                                                  ctx=ctx)
        torch.cuda.synchronize()
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        preps = 10
        p0.record(stream)
        for _ in range(preps):
            api.reconstruct_primal_batched_device(kd, lam_dev.data_ptr(), dz_dev.data_ptr(), B,
                                                  ctx=ctx)
        p1.record(stream)
        torch.cuda.synchronize()
        pms = p0.elapsed_time(p1) / preps
        pbytes = 8 * ((N + 1) * (n * n + n) + N * (m * m + m + n * n + n * m) + (N + 1) * n + P)
        hbm_p, _src = peaks()
        primal = {"systems_per_s": B / (pms * 1e-3), "ms_per_batch": pms,
                  "achieved_GBs": B * pbytes / (pms * 1e-3) / 1e9, "peak_GBs": hbm_p,
                  "frac": B * pbytes / (pms * 1e-3) / 1e9 / hbm_p,
                  "bytes_per_system": pbytes,
                  "what": "b2p_reconstruct_primal_batched_device over the bench batch "
                          "(kkt.cpp:153-181), CUDA events, inputs in HBM"}

    # ---- direct baseline (trajopt_cli.cpp:164-173)
    dense = None
    if rank == 0 and not a.no_latency:
        lam_direct = torch.empty((B, D), dtype=torch.float64, device=f"cuda:{local}")
        status = torch.empty((B,), dtype=torch.int32, device=f"cuda:{local}")
        api.direct_solve_batched_device(kd, lam_direct.data_ptr(), status.data_ptr(), B, ctx=ctx)
        torch.cuda.synchronize()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record(stream)
        for _ in range(3):
            api.direct_solve_batched_device(kd, lam_direct.data_ptr(), status.data_ptr(), B,
                                            ctx=ctx)
        d1.record(stream)
        torch.cuda.synchronize()
        dms = d0.elapsed_time(d1) / 3
        scale = torch.clamp(lam_direct.abs().amax(dim=1), min=1.0)
        rel = ((lam_direct - lam_dev).abs().amax(dim=1) / scale).max().item()
        dense = {"systems_per_s": B / (dms * 1e-3), "ms_per_batch": dms,
                 "all_ok": bool((status == -1).all().item()),
                 "max_rel_diff_vs_pcg": rel,
                 "what": "b2p_direct_solve_batched_device: build_schur + block-Thomas "
                         "cholesky_solve (block_tri.cpp:121-159), a half-warp per system, on the "
                         "bench batch; the PCG solves stop at eta' < eps, hence the difference"}

    # ---- roofline of the dominant kernel (one launch per step = the whole step)
    mean_iters = float(np.mean(iters))
    alg = algorithmic(N, n, m, mean_iters)
    hbm, peak_src = peaks()
    k1_avg = k1_ms / max(1, nsolves)
    k3_avg = k3_ms / max(1, nsolves)
    fused = ctx.last_path() >= 1
    if fused:
        dom = {1: "K13_fused", 2: "K13_fused_cluster"}.get(ctx.last_path(), "K13_fused")
        dom_ms = k1_avg + k3_avg
        dom_bytes = B * (alg["b_in"] + (N + 1) * n * 8)
    else:
        dom = "K3_pcg" if k3_avg >= k1_avg else "K1_schur_formation"
        dom_ms = max(k1_avg, k3_avg)
        dom_bytes = B * (alg["b_k3"] if dom == "K3_pcg" else alg["b_k1"])
    dom_flops = B * alg["f_full"]
    traffic = onchip = None
    tpath = os.path.join(ROOT, "profiles", "dram_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            traffic = tj[dom]["dram_bytes_per_system"] * B  # ncu capture, per system
            onchip = tj.get("onchip", {}).get(dom)
        except Exception:
            traffic = None
    fp64_ach = dom_flops / (dom_ms * 1e-3) / 1e12
    hbm_ach = dom_bytes / (dom_ms * 1e-3) / 1e9

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": elapsed_ms / a.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (random_kkt seeded draws, the reference generator restated)",
        "config": workload(a),
        "e2e": e2e,
        "gpu_launches": launches,
        # The roof that binds: formation + PCG is FP64-FMA work on on-chip
        # operands (~11 flop per compulsory byte, above the fp64 ridge). achieved =
        # reference-algorithm FLOPs of the step's systems / the kernel's average launch
        # time. The HBM view of the same launch sits beside it; "onchip" is the ncu
        # pipe utilisation that actually limits this kernel.
        "roofline": {"bound": "fp64", "kernel": dom, "achieved": fp64_ach,
                     "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": fp64_ach / FP64_PEAK_TFLOPS, "traffic": traffic,
                     "peak_source": "measured DFMA microbenchmark (scripts/micro/lat_bench.cu); "
                                    "MEASURED_PEAKS.json has no fp64 figure",
                     "flops_per_launch": dom_flops, "avg_launch_ms": dom_ms,
                     "hbm": {"achieved": hbm_ach, "peak": hbm, "unit": "GB/s",
                             "frac": hbm_ach / hbm, "peak_source": peak_src,
                             "bytes_per_launch": dom_bytes, "traffic": traffic},
                     "phase_ms_per_step": ({dom: k1_avg + k3_avg} if fused else
                                           {"K1_schur_formation": k1_avg, "K3_pcg": k3_avg}),
                     "onchip": onchip},
        "pcg_iters": {"mean": mean_iters, "min": int(min(iters)), "max": int(max(iters))},
        "c4_eps_1e-4": ({k: v for k, v in c4_eps4.items() if k not in ("lambda", "iterations")}
                        if c4_eps4 else None),
        "latency": latency,
        "baseline_configs": rows,
        "reconstruct_primal": primal,
        "dense_baseline": dense,
        "clocks": clk.summary(),
    }

    # ---- CPU baseline (N = 1) and parity of the bench batch against the oracle
    if rank == 0:
        orc = _orc()
        cb = None
        if not a.no_cpu and world == 1:
            cb = cpu_sample(a, a.cpu_seconds, a.seed, want_lambda=True)
            line["cpu_baseline"] = {
                "value": cb["value"], "unit": UNIT, "cores": cb["threads"], "kind": "port",
                "sample": f"{cb['sample']} systems of the same workload ({cb['secs']:.1f} s, "
                          f"oracle restatement g++ -O3 -DNDEBUG, all host threads)",
                "pcg_iters_mean": cb["iters"]}
            try:
                nat = cpu_sample(a, min(4.0, a.cpu_seconds / 3), a.seed, native=True)
                line["cpu_baseline"]["native_row"] = {
                    "value": nat["value"], "unit": UNIT, "cores": nat["threads"],
                    "flags": "-O3 -DNDEBUG -march=native (labelled row, BASELINE.md §2)",
                    "sample": f"{nat['sample']} systems ({nat['secs']:.1f} s)"}
            except Exception as exc:
                line["cpu_baseline"]["native_row"] = {"error": str(exc)[:200]}
        # parity: every system the oracle solved (>= 256), outside the timed region
        if cb is None or cb["sample"] < 256:
            cb = {"lambda": None}
            kbo = orc.random_kkt_batch(seed0, min(B, 256), N, n, m)
            _, lo, ro = orc.solve_batch(kbo, PrecondKind.symmetric_stair, 1, cfg)
            cb.update(lambda_=lo, it=np.array([r.iterations for r in ro]),
                      conv=np.array([r.converged for r in ro]))
        else:
            cb.update(lambda_=cb["lambda"], it=cb["iterations"], conv=cb["converged"])
        S = cb["lambda_"].shape[0]
        scale = np.maximum(1.0, np.abs(cb["lambda_"]).max(axis=1))
        rel = np.abs(lam_host_dev[:S] - cb["lambda_"]).max(axis=1) / scale
        it_g = np.array(iters[:S])
        par = {"systems": int(S), "iterations_equal": int((it_g == cb["it"]).sum()),
               "converged_equal": int((reps.converged[:S] == cb["conv"]).sum()),
               "lambda_rel_err_max": float(rel.max()), "tolerance": 1e-10,
               "what": "bench batch systems 0..S-1 (this rank's seeds) vs the oracle on the "
                       "same inputs, computed outside the timed region"}
        if c4_eps4 is not None:
            kbo = orc.random_kkt_batch(seed0, 256, N, n, m)
            _, lo4, ro4 = orc.solve_batch(kbo, PrecondKind.symmetric_stair, 1,
                                          PcgConfig(epsilon=1e-4))
            s4 = np.maximum(1.0, np.abs(lo4).max(axis=1))
            par["eps_1e-4"] = {
                "systems": 256,
                "iterations_equal": int((c4_eps4["iterations"] ==
                                         np.array([r.iterations for r in ro4])).sum()),
                "lambda_rel_err_max": float((np.abs(c4_eps4["lambda"] - lo4).max(axis=1)
                                             / s4).max())}
        line["parity"] = par
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    a = parse()
    maybe_relaunch(a)
    world, rank, local = dist_setup()
    if a.impl == "reference":
        run_reference(a, world, rank)
    else:
        run_b200(a, world, rank, local)


if __name__ == "__main__":
    main()
