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

// ---------------------------------------------------------------------------
// Compile-time-shape variant (n, m <= 16): one 16-lane half-warp per (system,
// knot, block), lane i owning row i in registers; unpivoted L D L' with the
// pivot broadcast by shuffles, forward sweep by shuffles, backward sweep
// through the unit-lower rows in shared memory. Many half-warps per SM hide
// the short dependency chains, so the kernel runs at the HBM roofline of its
// operands (the KKT blocks, lambda in, dz out).
namespace {
constexpr int kPrHw = 16;  // half-warps per CTA (256 threads)

template <class T, int D>
__device__ __forceinline__ void hw_ldlt_solve(T (&a)[D], T& rhs, T* Lt, int l, unsigned mk) {
  // a: row l of the block (lanes l < D); rhs: b_l. Out: rhs = x_l.
  // factor: a[q] <- L(l, q) for q < l, dl = D_l
  T dl = T(1);
#pragma unroll
  for (int k = 0; k < D; ++k) {
    T s = a[k];
    // Lt[k][q] = L(k,q) d_q: row k read as broadcast 16-byte pairs when rows
    // are 16-byte aligned (fewer L1 instructions: the kernel is L1-issue-bound),
    // same subtraction order
    if constexpr (sizeof(T) == 8 && D % 2 == 0) {
#pragma unroll
      for (int q = 0; q + 1 < k; q += 2) {
        const double2 v = *reinterpret_cast<const double2*>(Lt + k * D + q);
        s -= a[q] * v.x;
        s -= a[q + 1] * v.y;
      }
      if (k & 1) s -= a[k - 1] * Lt[k * D + k - 1];
    } else {
#pragma unroll
      for (int q = 0; q < k; ++q) s -= a[q] * Lt[k * D + q];
    }
    const T dk = __shfl_sync(mk, s, k, 16);
    const T rk = T(1) / dk;
    if (l == k) dl = dk;
    if (l > k && l < D) {
      Lt[l * D + k] = s;  // unscaled L(l,k) d_k, broadcast in the later steps
      a[k] = s * rk;      // L(l,k)
    }
    __syncwarp(mk);
  }
  // L y = b (column sweep), z = y / d
#pragma unroll
  for (int q = 0; q < D; ++q) {
    const T yq = __shfl_sync(mk, rhs, q, 16);
    if (l > q && l < D) rhs -= a[q] * yq;
  }
  rhs = rhs / dl;
  // unit-lower rows to shared memory for the transposed sweep
  if (l < D) {
#pragma unroll
    for (int q = 0; q < D; ++q) Lt[l * D + q] = (q < l) ? a[q] : T(0);
  }
  __syncwarp(mk);
#pragma unroll
  for (int j = D - 1; j >= 0; --j) {
    const T xj = __shfl_sync(mk, rhs, j, 16);
    if (l < j) rhs -= Lt[j * D + l] * xj;
  }
}

template <class T, int NB, int MB>
__global__ void __launch_bounds__(16 * kPrHw) k_reconstruct_primal_hw(PrimalParams<T> p) {
  __shared__ __align__(16) T tiles[kPrHw][NB * NB];
  const int hw = threadIdx.x >> 4, l = threadIdx.x & 15;
  const unsigned mk = 0xffffu << (threadIdx.x & 16);
  const int N = p.N, K = N + 1;
  // half-warp tasks: [0, B*K) state solves, then [B*K, B*K + B*N) control
  // solves; the two half-warps of a warp always run the same kind (no
  // divergence between the n- and m-sized code paths)
  const long long nx = static_cast<long long>(p.B) * K;
  const long long nxp = (nx + 1) & ~1LL;  // state tasks padded to whole warps
  const long long g = static_cast<long long>(blockIdx.x) * kPrHw + hw;
  int sys, k, blk;
  if (g < nxp) {
    if (g >= nx) return;
    blk = 0;
    sys = static_cast<int>(g / K);
    k = static_cast<int>(g % K);
  } else {
    const long long u = g - nxp;
    if (MB == 0 || u >= static_cast<long long>(p.B) * N) return;
    blk = 1;
    sys = static_cast<int>(u / N);
    k = static_cast<int>(u % N);
  }
  T* Lt = tiles[hw];
  const T* lam = p.lambda + static_cast<size_t>(sys) * K * NB;
  const T* lam1 = lam + static_cast<size_t>(k + 1) * NB;
  const size_t pd = static_cast<size_t>(K) * NB + static_cast<size_t>(N) * MB;
  T* dz = p.dz + static_cast<size_t>(sys) * pd + static_cast<size_t>(k) * (NB + MB);
  if (blk == 0) {
    const int lr = l < NB ? l : NB - 1;
    // Q_k through the tile with coalesced 16-lane loads (each sector fetched once)
    const T* Q = p.Q + (static_cast<size_t>(sys) * K + k) * NB * NB;
    constexpr bool kVec = sizeof(T) == 8 && NB % 2 == 0;  // 16-byte blocks and rows
    T a[NB];
    if constexpr (kVec) {
      // 16-byte coalesced loads / stores (every block and row starts 16-byte aligned)
#pragma unroll
      for (int i = l; i < NB * NB / 2; i += 16)
        reinterpret_cast<double2*>(Lt)[i] = __ldg(reinterpret_cast<const double2*>(Q) + i);
      __syncwarp(mk);
#pragma unroll
      for (int j = 0; j < NB; j += 2) {
        const double2 v = *reinterpret_cast<const double2*>(Lt + lr * NB + j);
        a[j] = v.x;
        a[j + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int i = l; i < NB * NB; i += 16) Lt[i] = __ldg(Q + i);
      __syncwarp(mk);
#pragma unroll
      for (int j = 0; j < NB; ++j) a[j] = Lt[lr * NB + j];
    }
    __syncwarp(mk);
    T at = T(0);
    if (k < N) {  // (A_k' lambda_{k+1})_l = sum_j A_k(j, l) lambda_{k+1, j}
      const T* A = p.A + (static_cast<size_t>(sys) * N + k) * NB * NB;
      if constexpr (kVec) {
#pragma unroll
        for (int j = 0; j < NB; j += 2) {
          const double2 lv = __ldg(reinterpret_cast<const double2*>(lam1 + j));
          at += __ldg(A + j * NB + lr) * lv.x;
          at += __ldg(A + (j + 1) * NB + lr) * lv.y;
        }
      } else {
#pragma unroll
        for (int j = 0; j < NB; ++j) at += __ldg(A + j * NB + lr) * __ldg(lam1 + j);
      }
    }
    T rhs = -(__ldg(p.q + (static_cast<size_t>(sys) * K + k) * NB + lr) +
              __ldg(lam + static_cast<size_t>(k) * NB + lr) - at);
    hw_ldlt_solve<T, NB>(a, rhs, Lt, l, mk);
    if (l < NB) dz[l] = rhs;
  } else {
    const int lr = l < MB ? l : MB - 1;
    const T* Rm = p.R + (static_cast<size_t>(sys) * N + k) * MB * MB;
#pragma unroll
    for (int i = l; i < MB * MB; i += 16) Lt[i] = __ldg(Rm + i);
    __syncwarp(mk);
    T a[MB];
#pragma unroll
    for (int j = 0; j < MB; ++j) a[j] = Lt[lr * MB + j];
    __syncwarp(mk);
    const T* Bm = p.B_ + (static_cast<size_t>(sys) * N + k) * NB * MB;
    T bt = T(0);
    if constexpr (sizeof(T) == 8 && NB % 2 == 0) {
#pragma unroll
      for (int j = 0; j < NB; j += 2) {
        const double2 lv = __ldg(reinterpret_cast<const double2*>(lam1 + j));
        bt += __ldg(Bm + j * MB + lr) * lv.x;
        bt += __ldg(Bm + (j + 1) * MB + lr) * lv.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < NB; ++j) bt += __ldg(Bm + j * MB + lr) * __ldg(lam1 + j);
    }
    T rhs = -(__ldg(p.r + (static_cast<size_t>(sys) * N + k) * MB + lr) - bt);
    hw_ldlt_solve<T, MB>(a, rhs, Lt, l, mk);
    if (l < MB) dz[NB + l] = rhs;
  }
}
}  // namespace

template <class T>
cudaError_t launch_reconstruct_primal(const PrimalParams<T>& p, cudaStream_t st) {
  const long long tasks = static_cast<long long>(p.B) * (p.N + 1) * 2;
  auto hw_launch = [&](auto kern) {
    const long long nx = static_cast<long long>(p.B) * (p.N + 1);
    const long long ht = ((nx + 1) & ~1LL) + static_cast<long long>(p.B) * p.N;
    const long long grid = (ht + kPrHw - 1) / kPrHw;
    kern<<<static_cast<unsigned>(grid), 16 * kPrHw, 0, st>>>(p);
    return cudaGetLastError();
  };
  if (tasks / kPrHw < 0x7fffffffLL) {
    if constexpr (sizeof(T) == 8) {
      if (p.n == 14 && p.m == 7) return hw_launch(k_reconstruct_primal_hw<T, 14, 7>);
    } else {
      if (p.n == 12 && p.m == 4) return hw_launch(k_reconstruct_primal_hw<T, 12, 4>);
    }
  }
  const long long grid = (tasks + kPrWarps - 1) / kPrWarps;
  if (grid > 0x7fffffffLL) return cudaErrorInvalidValue;
  k_reconstruct_primal<T><<<static_cast<unsigned>(grid), 32 * kPrWarps, 0, st>>>(p);
  return cudaGetLastError();
}

template cudaError_t launch_reconstruct_primal<double>(const PrimalParams<double>&, cudaStream_t);
template cudaError_t launch_reconstruct_primal<float>(const PrimalParams<float>&, cudaStream_t);

}  // namespace b2p
