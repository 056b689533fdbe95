#!/usr/bin/env python
"""Single-solve latency / iteration sweep over the BASELINE configs.

c1  K=32  n14 m7  fp64 symstair eps 1e-8
c2  K=128 n14 m7  fp64 jacobi / stair / symstair, eps 1e-8 and 1e-4
c3  K=256 n12 m4  fp32 symstair, eps 1e-4 (and 1e-6), multi-SM (cluster vs cooperative grid)
c5  K=512 n28 m14 fp64 symstair eps 1e-8, conditioning sweep random_kkt_scaled
Device time = CUDA events around the solve kernels (host copies excluded).
Iteration counts are compared with the CPU oracle on the same inputs.
Prints one JSON object.
"""
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import pyoracle as orc  # noqa: E402  (checker only)
import paper_2309_08079_b200.api as api  # noqa: E402
from paper_2309_08079_b200.types import PcgConfig, PrecondKind  # noqa: E402

REPS = int(os.environ.get("REPS", "15"))


def timed(kkt, kind, eps, dtype=np.float64, env=None):
    saved = {}
    for k, v in (env or {}).items():
        saved[k] = os.environ.get(k)
        os.environ[k] = v
    try:
        cfg = PcgConfig(epsilon=eps)
        ts = []
        res = None
        for i in range(REPS + 3):
            res = api.solve(kkt, kind, 1, cfg, dtype=dtype)
            if i >= 3:
                ts.append(res.report.wall_time * 1e6)
        t0 = time.perf_counter()
        orc_res = orc.solve(kkt, kind, 1, cfg, dtype=dtype)
        cpu_us = (time.perf_counter() - t0) * 1e6
        ctx = api.context()
        path = {0: "split K1+K3", 1: "fused one-CTA", 2: "fused cluster", 3: "fused grid",
                4: "fused small"}[ctx.last_path()]
        k1_ms, k3_ms = ctx.last_phase_ms()
        return {"us_median": statistics.median(ts), "us_min": min(ts),
                "iterations": res.report.iterations,
                "oracle_iterations": orc_res.report.iterations,
                "iterations_equal": res.report.iterations == orc_res.report.iterations,
                "cpu_oracle_1thread_us": cpu_us, "path": path,
                "split_K1_us": k1_ms * 1e3 if path.startswith("split") else None,
                "split_K3_us": k3_ms * 1e3 if path.startswith("split") else None}
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def main():
    api.require_device()
    out = {"what": "single-solve device latency (CUDA events around K1+K3 or the fused kernel)",
           "reps": REPS}
    k1 = orc.random_kkt(1, 31, 14, 7)
    out["c1_symstair_1e-8"] = timed(k1, PrecondKind.symmetric_stair, 1e-8)
    out["c1_symstair_1e-8_splitpath"] = timed(k1, PrecondKind.symmetric_stair, 1e-8,
                                              env={"B2P_FUSED": "0"})
    out["c1_symstair_1e-8_onecta"] = timed(k1, PrecondKind.symmetric_stair, 1e-8,
                                           env={"B2P_FC": "0"})
    out["c1_symstair_1e-8_cluster2"] = timed(k1, PrecondKind.symmetric_stair, 1e-8,
                                             env={"B2P_FC_G": "2"})
    for rp in (1, 2):
        out[f"c1_symstair_1e-8_fusedgrid_rp{rp}"] = timed(
            k1, PrecondKind.symmetric_stair, 1e-8, env={"B2P_FG": "1", "B2P_FG_RP": str(rp)})
    # build_schur API (host buffers in/out, wall time incl. copies): fused formation
    # kernel in formation-only mode vs the split K1 kernel
    for tag, envv in (("fused_formation", {}), ("split_K1", {"B2P_FUSED": "0"})):
        saved = {kk: os.environ.get(kk) for kk in envv}
        os.environ.update(envv)
        try:
            for _ in range(3):
                api.build_schur(k1)
            ts = []
            for _ in range(20):
                t0 = time.perf_counter()
                api.build_schur(k1)
                ts.append((time.perf_counter() - t0) * 1e6)
            out[f"c1_build_schur_api_{tag}_us"] = statistics.median(ts)
        finally:
            for kk, vv in saved.items():
                if vv is None:
                    os.environ.pop(kk, None)
                else:
                    os.environ[kk] = vv
    k2 = orc.random_kkt(2, 127, 14, 7)
    for kind, name in [(PrecondKind.block_jacobi, "jacobi"), (PrecondKind.stair, "stair"),
                       (PrecondKind.symmetric_stair, "symstair")]:
        for eps in (1e-8, 1e-4):
            out[f"c2_{name}_{eps:g}"] = timed(k2, kind, eps)
    out["c2_symstair_1e-8_cluster8"] = timed(k2, PrecondKind.symmetric_stair, 1e-8,
                                             env={"B2P_FC_G": "8"})
    for rp in (1, 2, 4):
        out[f"c2_symstair_1e-8_fusedgrid_rp{rp}"] = timed(
            k2, PrecondKind.symmetric_stair, 1e-8, env={"B2P_FG": "1", "B2P_FG_RP": str(rp)})
    out["c2_symstair_1e-8_split"] = timed(k2, PrecondKind.symmetric_stair, 1e-8,
                                          env={"B2P_FC": "0"})
    k3 = orc.random_kkt(3, 255, 12, 4)
    for eps in (1e-4, 1e-6):
        out[f"c3_fp32_symstair_{eps:g}_auto"] = timed(k3, PrecondKind.symmetric_stair, eps,
                                                      dtype=np.float32)
    for G in (8, 16):
        out[f"c3_fp32_symstair_1e-4_fusedcluster{G}"] = timed(
            k3, PrecondKind.symmetric_stair, 1e-4, dtype=np.float32, env={"B2P_FC_G": str(G)})
    for rp in (2, 4, 7):
        out[f"c3_fp32_symstair_1e-4_fusedgrid_rp{rp}"] = timed(
            k3, PrecondKind.symmetric_stair, 1e-4, dtype=np.float32,
            env={"B2P_FG": "1", "B2P_FG_RP": str(rp)})
    for G in (2, 4, 8):
        out[f"c3_fp32_symstair_1e-4_split_cluster{G}"] = timed(
            k3, PrecondKind.symmetric_stair, 1e-4, dtype=np.float32,
            env={"B2P_FC": "0", "B2P_PCG_G": str(G)})
    for G in (32, 64):
        out[f"c3_fp32_symstair_1e-4_split_grid{G}"] = timed(
            k3, PrecondKind.symmetric_stair, 1e-4, dtype=np.float32,
            env={"B2P_FC": "0", "B2P_PCG_G": str(G)})
    k5 = orc.random_kkt(5, 511, 28, 14)
    out["c5_symstair_1e-8"] = timed(k5, PrecondKind.symmetric_stair, 1e-8)
    for rp in (2, 3):
        out[f"c5_symstair_1e-8_fusedgrid_rp{rp}"] = timed(
            k5, PrecondKind.symmetric_stair, 1e-8, env={"B2P_FG_RP": str(rp)})
    out["c5_symstair_1e-8_split"] = timed(k5, PrecondKind.symmetric_stair, 1e-8,
                                          env={"B2P_FG": "0"})
    sweep = {}
    for floor in (1.0, 0.1, 0.01, 0.001):
        for coupling in (0.5, 1.0, 2.0):
            kk = orc.random_kkt_scaled(50, 511, 28, 14, floor, coupling)
            r = timed(kk, PrecondKind.symmetric_stair, 1e-8)
            sweep[f"floor={floor:g},coupling={coupling:g}"] = {
                k: r[k] for k in ("us_median", "iterations", "oracle_iterations",
                                  "iterations_equal")}
    out["c5_kappa_sweep"] = sweep
    print(json.dumps(out))


if __name__ == "__main__":
    main()
