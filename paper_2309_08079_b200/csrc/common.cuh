// Shared device-side definitions for the B200 symmetric-stair PCG path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <utility>

namespace b2p {

// Per-system outcome record written by the kernels and turned into a
// b2p_solve_report / b2p_error (with the reference's message text) host-side.
struct SysOut {
  int32_t code;        // b2p_status
  int32_t knot;        // non-PD knot (build_schur) or -1
  int32_t which;       // kWhich* below
  int32_t iteration;   // PCG iteration of a breakdown / non-finite error
  int32_t iterations;  // SolveReport::iterations
  int32_t converged;   // SolveReport::converged
  double exit_eta;     // SolveReport::exit_eta
  double value;        // p'Sp for the breakdown message
  double max_drift;    // SolveReport::max_residual_drift
  int32_t trace_len;
  int32_t _pad;
};

enum : int32_t {
  kWhichNone = -1,
  kWhichQ = 0,      // "build_schur: Q at knot k is not positive definite"
  kWhichR = 1,      // "... R ..."
  kWhichTheta = 2,  // "... theta ..."
  kWhichInitNonFinite = 10,  // "pcg: non-finite initial residual"
  kWhichUpsNonFinite = 11,   // "pcg: non-finite p'Sp at iteration i"
  kWhichEtaNonFinite = 12,   // "pcg: non-finite iterate at iteration i"
  kWhichBreakdown = 13,      // "pcg: p'Sp = v at iteration i; S is not positive definite ..."
};

enum : int32_t { kOk = 0, kInvalid = 1, kRuntime = 2, kBreakdown = 3, kCuda = 4 };

// Preconditioner kinds (schur.hpp:26).
enum : int32_t { kIdentity = 0, kJacobi = 1, kStair = 2, kSymStair = 3, kPoly = 4 };

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ bool is_finite(double v) { return isfinite(v); }
__device__ __forceinline__ bool is_finite(float v) { return isfinite(v); }

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is a host call on every
// launch otherwise: set it once per (kernel, device) and size high-water mark.
// The attribute is idempotent, so a race between threads only repeats a call.
template <class F>
inline cudaError_t ensure_max_smem(F* kern, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const auto key = std::make_pair(reinterpret_cast<const void*>(kern), dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = done.find(key);
    if (it != done.end() && it->second >= bytes) return cudaSuccess;
  }
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(bytes));
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lk(mu);
    size_t& v = done[key];
    v = std::max(v, bytes);
  }
  return e;
}

}  // namespace b2p
