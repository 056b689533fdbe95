"""Build the in-tree sm_100a shared library libb2p.so (nvcc, no JIT cache).

The .so is git-ignored but travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libb2p.so")
SOURCES = ["b2p_api.cu", "schur_kernels.cu", "pcg_kernels.cu", "fused_kernels.cu", "fc_kernels.cu", "fg_kernels.cu", "primal_kernels.cu", "small_kernels.cu"]
HEADERS = ["common.cuh", "kernels.h", "warp_dense.cuh", "hw_dense.cuh", "wp_dense.cuh", "tmem.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    inc = os.path.join(os.path.dirname(HERE), "include")
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(inc, "b2p.h")]
    if not force and not _stale(LIB, deps):
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    common = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
                     "--expt-relaxed-constexpr", "-I", inc, "-I", CSRC]
    if verbose:
        common += ["-Xptxas", "-v"]
    objs = []
    procs = []
    hdeps = [os.path.join(CSRC, f) for f in HEADERS + ["tmem.cuh"]] + [os.path.join(inc, "b2p.h")]
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(obj)
        if not force and not verbose and not _stale(obj, [os.path.join(CSRC, src)] + hdeps):
            continue  # object up to date (per-file incremental rebuild)
        cmd = [NVCC] + common + ["-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = False
    for cmd, p in procs:
        out, _ = p.communicate()
        if out:
            sys.stderr.write(out.decode())
        if p.returncode != 0:
            failed = True
            sys.stderr.write("FAILED: " + " ".join(cmd) + "\n")
    if failed:
        raise RuntimeError("nvcc build of libb2p.so failed")
    tmp = LIB + ".tmp"
    subprocess.check_call([NVCC] + ARCH + ["-shared", "-o", tmp] + objs +
                          ["-lcudart_static", "-lpthread", "-ldl", "-lrt"])
    os.replace(tmp, LIB)
    return LIB


def build_adapter_test(force: bool = False) -> str:
    """g++ the C++ adapter test (tests/cpp/test_adapter.cpp) against libb2p.so."""
    root = os.path.dirname(HERE)
    src = os.path.join(root, "tests", "cpp", "test_adapter.cpp")
    hdr = os.path.join(root, "include", "trajopt_b200.hpp")
    out = os.path.join(root, "build", "test_adapter")
    if not force and not _stale(out, [src, hdr, LIB]):
        return out
    os.makedirs(os.path.dirname(out), exist_ok=True)
    subprocess.check_call(["g++", "-std=c++17", "-O2", "-Wall", "-I", os.path.join(root, "include"),
                           src, "-o", out, "-L", HERE, "-lb2p",
                           "-Wl,-rpath,$ORIGIN/../paper_2309_08079_b200"])
    return out


def build_dropin_test(force: bool = False) -> str:
    """g++ the drop-in acceptance test (tests/cpp/test_dropin.cpp): the reference's
    Eigen-typed trajopt:: API (include/trajopt_dropin) against libb2p.so, compiled
    with the test-only Eigen stand-in; the CPU oracle header is its checker."""
    root = os.path.dirname(HERE)
    src = os.path.join(root, "tests", "cpp", "test_dropin.cpp")
    dropin = os.path.join(root, "include", "trajopt_dropin")
    hdrs = [os.path.join(dropin, "trajopt", h)
            for h in ("b200_detail.hpp", "block_tri.hpp", "schur.hpp", "pcg.hpp")]
    hdrs += [os.path.join(root, "include", "trajopt_b200.hpp"),
             os.path.join(root, "tests", "cpp", "eigen_stub", "Eigen", "Dense"),
             os.path.join(root, "tests", "cpp", "ref_stub", "trajopt", "kkt.hpp"),
             os.path.join(root, "oracle", "trajopt_oracle.hpp")]
    out = os.path.join(root, "build", "test_dropin")
    if not force and not _stale(out, [src, LIB] + hdrs):
        return out
    os.makedirs(os.path.dirname(out), exist_ok=True)
    # include order as an integrator would set it: the drop-in ahead of the
    # reference's own include directory (here: its test-only KKT stand-in)
    subprocess.check_call(["g++", "-std=c++20", "-O2", "-Wall", "-pthread",
                           "-I", os.path.join(root, "tests", "cpp", "eigen_stub"),
                           "-I", dropin,
                           "-I", os.path.join(root, "tests", "cpp", "ref_stub"),
                           "-I", os.path.join(root, "include"), "-I", os.path.join(root, "oracle"),
                           src, "-o", out, "-L", HERE, "-lb2p",
                           "-Wl,-rpath,$ORIGIN/../paper_2309_08079_b200"])
    return out


def build_sqp_test(force: bool = False) -> str:
    """g++ the SQP / NMPC caller tests (tests/cpp/test_sqp.cpp) against libb2p.so.
    The test links the CPU oracle header as its checker (test infrastructure)."""
    root = os.path.dirname(HERE)
    src = os.path.join(root, "tests", "cpp", "test_sqp.cpp")
    hdrs = [os.path.join(root, "include", h) for h in ("trajopt_b200.hpp", "trajopt_b200_sqp.hpp")]
    hdrs.append(os.path.join(root, "oracle", "trajopt_oracle.hpp"))
    out = os.path.join(root, "build", "test_sqp")
    if not force and not _stale(out, [src, LIB] + hdrs):
        return out
    os.makedirs(os.path.dirname(out), exist_ok=True)
    subprocess.check_call(["g++", "-std=c++20", "-O2", "-Wall", "-pthread",
                           "-I", os.path.join(root, "include"), "-I", os.path.join(root, "oracle"),
                           src, "-o", out, "-L", HERE, "-lb2p",
                           "-Wl,-rpath,$ORIGIN/../paper_2309_08079_b200"])
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
