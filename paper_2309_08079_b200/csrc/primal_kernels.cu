// reconstruct_primal (proj/src/kkt.cpp:153-181) — the paper's "Trajopt PPCG
// finish": after the PCG returns lambda, every knot k
// independently recovers
//   dx_k = Q_k^-1 (-(q_k + lambda_k - A_k' lambda_{k+1}))      (k < N)
//   du_k = R_k^-1 (-(r_k - B_k' lambda_{k+1}))                 (k < N)
//   dx_N = Q_N^-1 (-(q_N + lambda_N))
// into dz = [x_0, u_0, x_1, u_1, ..., x_N].
//
// One warp per (system, knot, block): block 0 = the state solve, block 1 =
// the control solve. The reference solves with Eigen's LDLT (never throws);
// this kernel factors the block unpivoted as L D L' (same solution as the
// reference's for the SPD cost blocks, and like it no error path), lane i
// owning row i, the tile and the right-hand side in shared memory.
#include "kernels.h"

namespace b2p {
namespace {
constexpr int kPrWarps = 4;  // warps per CTA
}

template <class T>
__global__ void __launch_bounds__(32 * kPrWarps) k_reconstruct_primal(PrimalParams<T> p) {
  __shared__ __align__(16) T tile[kPrWarps][32 * 33];
  __shared__ T vec[kPrWarps][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int N = p.N, n = p.n, m = p.m, K = N + 1;
  const long long task = static_cast<long long>(blockIdx.x) * kPrWarps + w;
  const long long ntask = static_cast<long long>(p.B) * K * 2;
  if (task >= ntask) return;
  const int sys = static_cast<int>(task / (2 * K));
  const int k = static_cast<int>((task / 2) % K);
  const int blk = static_cast<int>(task & 1);
  if (blk == 1 && (k == N || m == 0)) return;
  const int d = blk ? m : n;
  const int LD = 33;
  T* W = tile[w];
  T* x = vec[w];
  const T* lam = p.lambda + static_cast<size_t>(sys) * K * n;
  const T* lam1 = lam + static_cast<size_t>(k + 1) * n;
  // matrix block and right-hand side
  const T* M = blk ? p.R + (static_cast<size_t>(sys) * N + k) * m * m
                   : p.Q + (static_cast<size_t>(sys) * K + k) * n * n;
  for (int idx = lane; idx < d * d; idx += 32) W[(idx / d) * LD + idx % d] = M[idx];
  if (lane < d) {
    T rhs;
    if (blk == 0) {
      const T* q = p.q + (static_cast<size_t>(sys) * K + k) * n;
      T at = T(0);
      if (k < N) {  // (A_k' lambda_{k+1})_i = sum_j A_k(j, i) lambda_{k+1, j}
        const T* A = p.A + (static_cast<size_t>(sys) * N + k) * n * n;
        for (int j = 0; j < n; ++j) at += A[j * n + lane] * lam1[j];
      }
      rhs = -(q[lane] + lam[static_cast<size_t>(k) * n + lane] - at);
    } else {
      const T* r = p.r + (static_cast<size_t>(sys) * N + k) * m;
      const T* Bm = p.B_ + (static_cast<size_t>(sys) * N + k) * n * m;
      T bt = T(0);
      for (int j = 0; j < n; ++j) bt += Bm[j * m + lane] * lam1[j];
      rhs = -(r[lane] - bt);
    }
    x[lane] = rhs;
  }
  __syncwarp();
  // unpivoted L D L' in place: W(j,j) <- D_j, W(i,j) <- L(i,j) for i > j
  for (int j = 0; j < d; ++j) {
    if (lane >= j && lane < d) {
      T s = W[lane * LD + j];
      for (int q = 0; q < j; ++q) s -= W[lane * LD + q] * W[j * LD + q] * W[q * LD + q];
      W[lane * LD + j] = s;  // lane j: D_j; lanes > j: D_j L(lane, j)
    }
    __syncwarp();
    if (lane > j && lane < d) W[lane * LD + j] = W[lane * LD + j] / W[j * LD + j];
    __syncwarp();
  }
  // L y = b (column sweep), z = D^-1 y, L' x = z
  for (int j = 0; j < d; ++j) {
    if (lane > j && lane < d) x[lane] -= W[lane * LD + j] * x[j];
    __syncwarp();
  }
  if (lane < d) x[lane] = x[lane] / W[lane * LD + lane];
  __syncwarp();
  for (int j = d - 1; j >= 0; --j) {
    if (lane < j) x[lane] -= W[j * LD + lane] * x[j];
    __syncwarp();
  }
  if (lane < d) {
    const size_t pd = static_cast<size_t>(K) * n + static_cast<size_t>(N) * m;
    const size_t off = static_cast<size_t>(sys) * pd + static_cast<size_t>(k) * (n + m) + (blk ? n : 0);
    p.dz[off + lane] = x[lane];
  }
}

template <class T>
cudaError_t launch_reconstruct_primal(const PrimalParams<T>& p, cudaStream_t st) {
  const long long tasks = static_cast<long long>(p.B) * (p.N + 1) * 2;
  const long long grid = (tasks + kPrWarps - 1) / kPrWarps;
  if (grid > 0x7fffffffLL) return cudaErrorInvalidValue;
  k_reconstruct_primal<T><<<static_cast<unsigned>(grid), 32 * kPrWarps, 0, st>>>(p);
  return cudaGetLastError();
}

template cudaError_t launch_reconstruct_primal<double>(const PrimalParams<double>&, cudaStream_t);
template cudaError_t launch_reconstruct_primal<float>(const PrimalParams<float>&, cudaStream_t);

}  // namespace b2p
