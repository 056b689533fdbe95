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
          the timed region)
Also reported: single-solve latency (c1) and PCG iterations.

--impl reference: the reference's CPU implementation of the path (the
oracle restatement; the reference cannot be compiled here)
on all host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2309_08079_b200.types import PcgConfig, PrecondKind  # noqa: E402

METRIC = "batched PCG solves/s (symmetric-stair, fp64)"
UNIT = "solves/s"


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


FP64_PEAK_TFLOPS = 35.4  # measured on this pool's B200 (scripts/micro/lat_bench.cu)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------ CPU arm
def cpu_sample(a, seconds, seed0):
    """Oracle (restated reference) on all host threads over a bounded sample."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as orc
    import paper_2309_08079_b200.api as api  # host-side generator only
    orc.build()
    threads = os.cpu_count() or 1
    N = a.knots - 1
    cfg = PcgConfig(epsilon=a.eps)
    # calibrate with a small batch, then size the sample for ~`seconds`
    cal = max(threads, 8)
    kb = api.random_kkt_batch(seed0, cal, N, a.nx, a.nu)
    secs, _, reps = orc.solve_batch(kb, PrecondKind.symmetric_stair, 1, cfg, threads=threads,
                                    want_lambda=False)
    per = secs / cal
    sample = int(min(a.batch, max(cal, seconds / max(per, 1e-9))))
    kb = api.random_kkt_batch(seed0, sample, N, a.nx, a.nu)
    secs, _, reps = orc.solve_batch(kb, PrecondKind.symmetric_stair, 1, cfg, threads=threads,
                                    want_lambda=False)
    iters = float(np.mean([r.iterations for r in reps]))
    return sample / secs, sample, secs, threads, iters


def run_reference(a, world, rank):
    if rank != 0:
        return
    steps, warm = a.steps, a.warmup
    budget = max(2.0, min(20.0, 150.0 / max(1, steps + warm)))
    for _ in range(warm):
        cpu_sample(a, budget / 4, a.seed)
    vals = []
    sample = 0
    threads = 1
    iters = 0.0
    t_total = 0.0
    for s in range(steps):
        v, sample, secs, threads, iters = cpu_sample(a, budget, a.seed)
        vals.append(v)
        t_total += secs
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": a.gpus, "steps": steps, "warmup": warm,
        "ms_per_step": 1e3 * t_total / steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (random_kkt, seeded)",
        "config": workload(a),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{sample} systems of the c4 workload per step "
                                   f"(oracle restatement of proj/src, g++ -O3, "
                                   f"parallel_for over instances as trajopt_cli.cpp:155)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "pcg_iters_mean": iters,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
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


def nmpc_batch_throughput(api, torch, local, B=4096, N=32, n=2, m=1, reps=5):
    """Many independent NMPC-shape systems (double-integrator / pendulum size, the
    SQP callers' shape) through the small-block kernel, device-resident, CUDA events."""
    from paper_2309_08079_b200.types import KKTSystem
    kb = api.random_kkt_batch(77, B, N, n, m)
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
    return {"systems_per_s": B / (ms * 1e-3), "ms_per_batch": ms, "batch": B, "knots": N + 1,
            "nx": n, "nu": m, "kernel": {4: "fused small"}.get(path, str(path)),
            "iters_mean": float(np.mean([r.iterations for r in reports]))}


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

    def step():
        api.solve_batched_device(kd, lam_dev.data_ptr(), B, PrecondKind.symmetric_stair, 1, cfg,
                                 ctx=ctx)

    def barrier():
        if dist is not None:
            dist.barrier()

    def allmax(x):
        return max_over_ranks(x, dist, device=f"cuda:{local}")

    # warm-up (also validates every system once)
    reps = api.solve_batched_device(kd, lam_dev.data_ptr(), B, PrecondKind.symmetric_stair, 1,
                                    cfg, ctx=ctx, want_reports=True)
    iters = [r.iterations for r in reps]
    assert all(r.converged for r in reps), "unconverged systems in the bench batch"
    for _ in range(max(0, a.warmup - 1)):
        step()
    torch.cuda.synchronize()

    # ---- timed region: value (HBM-resident inputs)
    launches0 = ctx.kernel_launches()
    ctx.phase_accounting(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
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

    # ---- e2e: host buffers through the C-ABI (pinned in, pinned out)
    e2e = None
    if not a.no_e2e:
        lam_host = torch.empty((B, D), dtype=torch.float64, pin_memory=True).numpy()
        ctx_h = api.Context(local)
        api.solve_batched(kb, PrecondKind.symmetric_stair, 1, cfg, lambda_out=lam_host, ctx=ctx_h)
        barrier()
        e2e_ms = 0.0
        for _ in range(a.steps):
            api.solve_batched(kb, PrecondKind.symmetric_stair, 1, cfg, lambda_out=lam_host,
                              ctx=ctx_h)
            e2e_ms += ctx_h.last_solve_ms()
        barrier()
        e2e_ms = allmax(e2e_ms)
        # parity spot check of the e2e output against the device leg
        torch.cuda.synchronize()
        assert np.array_equal(lam_host, lam_dev.cpu().numpy()), "e2e/device outputs differ"
        import ctypes
        sysout = 56  # sizeof(SysOut) copied back per system
        e2e = {"value": world * B * a.steps / (e2e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": B * kkt_bytes(N, n, m),
               "d2h_bytes_per_step": B * (D * 8 + sysout + 4),
               "path": "b2p_solve_batched (host pinned buffers, 2-stream chunked H2D/compute/D2H)"}
        ctx_h.close()

    # ---- single-solve latency at the BASELINE single-system configs:
    # device time (CUDA events around the solve kernel), median of 20 after 5 warm-up
    latency = None
    if not a.no_latency and rank == 0:
        latency = {"what": "device time (CUDA events) of one fused formation + PCG solve; "
                           "host copies excluded; median of 20 after 5 warm-up solves"}
        cases = {"c1": (1, 31, 14, 7, np.float64, 1e-8), "c2": (2, 127, 14, 7, np.float64, 1e-8),
                 "c3": (3, 255, 12, 4, np.float32, 1e-4), "c5": (5, 511, 28, 14, np.float64, 1e-8)}
        names = {0: "split", 1: "one-CTA fused", 2: "fused cluster", 3: "fused grid", 4: "fused small"}
        for name, (seed, Nk, nk, mk, dt, eps) in cases.items():
            kk = api.random_kkt(seed, Nk, nk, mk)
            lat = []
            r = None
            for i in range(25):
                r = api.solve(kk, PrecondKind.symmetric_stair, 1, PcgConfig(epsilon=eps), dtype=dt)
                if i >= 5:
                    lat.append(r.report.wall_time * 1e6)
            latency[name] = {"us_median": statistics.median(lat), "us_min": min(lat),
                             "iterations": r.report.iterations, "knots": Nk + 1, "nx": nk, "nu": mk,
                             "dtype": np.dtype(dt).name, "epsilon": eps,
                             "kernel": names.get(api.context().last_path(), "?")}
        latency["c1_us_median"] = latency["c1"]["us_median"]
        # The SQP linear step of the reference's NMPC caller (sqp.cpp:171-176) at the
        # test-suite shape (double integrator, N = 32): one b2p_sqp_step call from host
        # buffers — fused solve + reconstruct_primal on one staged upload — wall clock
        # around the call (host packing, copies, launch and sync included).
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
                                  "nu": 1, "kernel": names.get(api.context().last_path(), "?")}
        # c1 through a CUDA graph ("c1 is also reported via a CUDA Graph to
        # show the launch floor"): device-resident inputs, the solve captured once and
        # replayed back to back; per-replay time = launch floor + kernel
        try:
            latency["c1_graph"] = c1_graph_latency(api, torch, local)
        except Exception as exc:  # report, do not fail the bench line
            latency["c1_graph"] = {"error": str(exc)[:200]}
        try:  # the NMPC-shape single solve replayed from a CUDA graph (launch floor)
            latency["nmpc_graph_n2"] = c1_graph_latency(api, torch, local, N=32, n=2, m=1)
        except Exception as exc:
            latency["nmpc_graph_n2"] = {"error": str(exc)[:200]}
        try:
            latency["nmpc_batch_n2"] = nmpc_batch_throughput(api, torch, local)
        except Exception as exc:
            latency["nmpc_batch_n2"] = {"error": str(exc)[:200]}

    # ---- reconstruct_primal on the same batch: dz from the
    # solved lambda, device-resident; HBM-bound (reads the KKT blocks + lambda,
    # writes dz), so its roofline fraction is meaningful
    primal = None
    if rank == 0:
        P = (N + 1) * n + N * m
        dz_dev = torch.empty((B, P), dtype=torch.float64, device=f"cuda:{local}")
        for _ in range(3):
            api.reconstruct_primal_batched_device(kd, lam_dev.data_ptr(), dz_dev.data_ptr(), B,
                                                  ctx=ctx)
        torch.cuda.synchronize()
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        p0.record(stream)
        for _ in range(reps):
            api.reconstruct_primal_batched_device(kd, lam_dev.data_ptr(), dz_dev.data_ptr(), B,
                                                  ctx=ctx)
        p1.record(stream)
        torch.cuda.synchronize()
        pms = p0.elapsed_time(p1) / reps
        # compulsory bytes per system: Q, q (all knots), R, r, A, B (k < N), lambda in, dz out
        pbytes = 8 * ((N + 1) * (n * n + n) + N * (m * m + m + n * n + n * m) + (N + 1) * n + P)
        hbm_p, _src = peaks()
        primal = {"systems_per_s": B / (pms * 1e-3), "ms_per_batch": pms,
                  "achieved_GBs": B * pbytes / (pms * 1e-3) / 1e9, "peak_GBs": hbm_p,
                  "frac": B * pbytes / (pms * 1e-3) / 1e9 / hbm_p,
                  "bytes_per_system": pbytes,
                  "what": "b2p_reconstruct_primal_batched_device over the bench batch "
                          "(kkt.cpp:153-181), CUDA events, inputs in HBM"}

    # ---- direct baseline (the reference bench's "dense_baseline"
    # row, trajopt_cli.cpp:164-173): build_schur + block-Thomas cholesky_solve of the
    # same device batch, one warp per system; CUDA events; lambda checked against PCG
    dense = None
    if rank == 0 and not a.no_latency:
        D = (N + 1) * n
        lam_direct = torch.empty((B, D), dtype=torch.float64, device=f"cuda:{local}")
        status = torch.empty((B,), dtype=torch.int32, device=f"cuda:{local}")
        api.direct_solve_batched_device(kd, lam_direct.data_ptr(), status.data_ptr(), B, ctx=ctx)
        torch.cuda.synchronize()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        d0.record(stream)
        for _ in range(reps):
            api.direct_solve_batched_device(kd, lam_direct.data_ptr(), status.data_ptr(), B,
                                            ctx=ctx)
        d1.record(stream)
        torch.cuda.synchronize()
        dms = d0.elapsed_time(d1) / reps
        scale = torch.clamp(lam_direct.abs().amax(dim=1), min=1.0)
        rel = ((lam_direct - lam_dev).abs().amax(dim=1) / scale).max().item()
        dense = {"systems_per_s": B / (dms * 1e-3), "ms_per_batch": dms,
                 "all_ok": bool((status == -1).all().item()),
                 "max_rel_diff_vs_pcg": rel,
                 "what": "b2p_direct_solve_batched_device: build_schur + block-Thomas "
                         "cholesky_solve (block_tri.cpp:121-159), one warp per system, on the "
                         "bench batch; the PCG solves stop at eta' < eps, hence the difference"}

    # ---- roofline for the dominant kernel
    mean_iters = float(np.mean(iters))
    alg = algorithmic(N, n, m, mean_iters)
    hbm, peak_src = peaks()
    k1_avg = k1_ms / max(1, nsolves)
    k3_avg = k3_ms / max(1, nsolves)
    fused = ctx.last_path() >= 1  # 1: one-CTA fused kernel, 2: fused cluster kernel
    if fused:
        # one persistent launch does K1+K2+K3: its compulsory HBM bytes are the
        # KKT inputs in and lambda out (the L/D/theta^-1 staging stays in L2)
        dom = "K13_fused" if ctx.last_path() == 1 else "K13_fused_cluster"
        dom_ms = k1_avg + k3_avg
        dom_bytes = B * (alg["b_in"] + (N + 1) * n * 8)
    else:
        dom = "K3_pcg" if k3_avg >= k1_avg else "K1_schur_formation"
        dom_ms = max(k1_avg, k3_avg)
        dom_bytes = B * (alg["b_k3"] if dom == "K3_pcg" else alg["b_k1"])
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "dram_traffic.json")
    onchip = None
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            traffic = tj.get(dom)
            onchip = tj.get("onchip", {}).get(dom)
        except Exception:
            traffic = None
    flops_step = B * alg["f_full"]

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": elapsed_ms / a.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (random_kkt seeded draws, the reference generator restated)",
        "config": workload(a),
        "e2e": e2e,
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm,
                     "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                     "peak_source": peak_src,
                     "bytes_per_launch": dom_bytes, "avg_launch_ms": dom_ms,
                     "phase_ms_per_step": ({"K13_fused": k1_avg + k3_avg} if fused else
                                           {"K1_schur_formation": k1_avg, "K3_pcg": k3_avg}),
                     "fp64_tflops_step": flops_step / (elapsed_ms / a.steps * 1e-3) / 1e12,
                     "b_full_GBs": B * alg["b_full"] / (elapsed_ms / a.steps * 1e-3) / 1e9,
                     # the on-chip roof that actually binds this kernel: FP64 FMA work of
                     # the reference algorithm (SURVEY 8d F_full) against the measured
                     # DFMA peak (scripts/micro/lat_bench.cu: 60.9 FMA/clk/SM, 35.4 TF/s)
                     "fp64": {"achieved": flops_step / (elapsed_ms / a.steps * 1e-3) / 1e12,
                              "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                              "frac": flops_step / (elapsed_ms / a.steps * 1e-3) / 1e12
                              / FP64_PEAK_TFLOPS,
                              "flops_per_step": flops_step,
                              "peak_source": "measured DFMA microbenchmark "
                                             "(scripts/micro/lat_bench.cu)"},
                     # the roof that binds: the SM's L1 / shared-memory pipe (ncu capture
                     # of the same kernel; the PCG and formation operands are on-chip)
                     "onchip": onchip},
        "pcg_iters": {"mean": mean_iters, "min": int(min(iters)), "max": int(max(iters))},
        "latency": latency,
        "reconstruct_primal": primal,
        "dense_baseline": dense,
        "clocks": clk.summary(),
    }
    if not a.no_cpu and world == 1 and rank == 0:
        v, sample, secs, threads, cit = cpu_sample(a, a.cpu_seconds, a.seed)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                                "sample": f"{sample} systems of the same workload "
                                          f"({secs:.1f} s, oracle restatement, all host threads)",
                                "pcg_iters_mean": cit}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    a = parse()
    world, rank, local = dist_setup()
    if a.impl == "reference":
        run_reference(a, world, rank)
    else:
        run_b200(a, world, rank, local)


if __name__ == "__main__":
    main()
