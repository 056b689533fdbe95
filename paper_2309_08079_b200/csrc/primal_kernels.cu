// reconstruct_primal (proj/src/kkt.cpp:153-181) — the paper's "Trajopt PPCG
// finish": after the PCG returns lambda, every knot k
// independently recovers
//   dx_k = Q_k^-1 (-(q_k + lambda_k - A_k' lambda_{k+1}))      (k < N)
//   du_k = R_k^-1 (-(r_k - B_k' lambda_{k+1}))                 (k < N)
//   dx_N = Q_N^-1 (-(q_N + lambda_N))
// into dz = [x_0, u_0, x_1, u_1, ..., x_N].
//
// The reference solves with Eigen's LDLT (never throws); these kernels factor
// each block unpivoted as L D L' (same solution as the reference's for the SPD
// cost blocks, and like it no error path). Three variants:
//   k_reconstruct_primal_bulk<14, 7> (fp64 batches of the c4 shape): CTAs of
//     4 consecutive knot tasks whose operands arrive as bulk TMA streams,
//     8-lane groups with two rows per lane (the bandwidth-bound path);
//   k_reconstruct_primal_hw (other compiled shapes): one half-warp per task;
//   k_reconstruct_primal (any n, m <= 32): one warp per (system, knot, block),
//     block 0 = the state solve, block 1 = the control solve.
#include "kernels.h"

#include <cstdint>
#include <cstdlib>

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
// ---------------------------------------------------------------------------
// 8-lane group solves for the streaming batch path: a group owns one knot
// task — the state solve of (system, k) with lane l < n/2 holding rows l and
// l + n/2, or the control solve with lane l < m holding row l — so every
// broadcast operand of the factorisation (the pivot row prefix) serves two
// rows, and a warp carries four tasks. Same unpivoted L D L' arithmetic per
// row as hw_ldlt_solve.

// reciprocal of a (positive, normal) pivot: the hardware approximation and two
// Newton steps (within an ulp of the IEEE reciprocal; the reference's LDLT
// pivots differently anyway, parity is tolerance-pinned)
__device__ __forceinline__ double recip(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ float recip(float x) { return __frcp_rn(x); }

// D x = rhs on an 8-lane group, rows l and l + H of a D x D SPD block (D = 2H):
// a0, a1 the rows, r0, r1 the right-hand sides (out: the solution rows).
template <class T, int D>
__device__ __forceinline__ void g8x2_ldlt_solve(T (&a0)[D], T (&a1)[D], T& r0, T& r1, T* Lt, int l) {
  constexpr int H = D / 2;
  const bool act = l < H;
  const int lr = act ? l : H - 1;
  T rd0 = T(1), rd1 = T(1);  // 1 / d of this lane's rows
#pragma unroll
  for (int k = 0; k < D; ++k) {
    T s0 = T(0), s1 = a1[k], u0 = T(0), u1 = T(0);
    if (k < H) s0 = a0[k];
    // two partial sums per row (even / odd q): half the dependent FMA chain
#pragma unroll
    for (int q = 0; q < k; ++q) {
      const T v = Lt[k * D + q];
      if (q & 1) {
        if (k < H) u0 -= a0[q] * v;
        u1 -= a1[q] * v;
      } else {
        if (k < H) s0 -= a0[q] * v;
        s1 -= a1[q] * v;
      }
    }
    s0 += u0;
    s1 += u1;
    const T dk = __shfl_sync(0xffffffffu, k < H ? s0 : s1, k < H ? k : k - H, 8);
    const T rk = recip(dk);  // IEEE reciprocal: bitwise T(1) / dk
    if (k < H) {
      if (lr == k) rd0 = rk;
      if (act && lr > k) {
        Lt[lr * D + k] = s0;
        a0[k] = s0 * rk;
      }
    }
    if (lr + H == k) rd1 = rk;
    if (act && lr + H > k) {
      Lt[(lr + H) * D + k] = s1;
      a1[k] = s1 * rk;
    }
    __syncwarp();
  }
  // L y = b (unit lower, column sweep)
#pragma unroll
  for (int q = 0; q < D; ++q) {
    const T yq = __shfl_sync(0xffffffffu, q < H ? r0 : r1, q < H ? q : q - H, 8);
    if (lr > q) r0 -= a0[q] * yq;
    if (lr + H > q) r1 -= a1[q] * yq;
  }
  // L' x = y / d, transposed sweep on the factorisation's unscaled entries
  // Lt(j, i) = L(j, i) d_i (i < j, stored above; no normalised copy of L is
  // written back): x_i = (y_i - sum_{j > i} Lt(j, i) x_j) / d_i, and row j is
  // final when the sweep reaches it
#pragma unroll
  for (int j = D - 1; j >= 0; --j) {
    const T xj = __shfl_sync(0xffffffffu, j < H ? r0 * rd0 : r1 * rd1, j < H ? j : j - H, 8);
    if (lr < j) r0 -= Lt[j * D + lr] * xj;
    if (lr + H < j) r1 -= Lt[j * D + lr + H] * xj;
  }
  r0 *= rd0;
  r1 *= rd1;
}

// the same on one row per lane (D <= 8; the control solve)
template <class T, int D>
__device__ __forceinline__ void g8_ldlt_solve(T (&a)[D], T& rhs, T* Lt, int l) {
  const int lr = l < D ? l : D - 1;
  T rdl = T(1);
#pragma unroll
  for (int k = 0; k < D; ++k) {
    T s = a[k];
#pragma unroll
    for (int q = 0; q < k; ++q) s -= a[q] * Lt[k * D + q];
    const T dk = __shfl_sync(0xffffffffu, s, k, 8);
    const T rk = recip(dk);  // IEEE reciprocal: bitwise T(1) / dk
    if (lr == k) rdl = rk;
    if (l < D && lr > k) {
      Lt[lr * D + k] = s;
      a[k] = s * rk;
    }
    __syncwarp();
  }
#pragma unroll
  for (int q = 0; q < D; ++q) {
    const T yq = __shfl_sync(0xffffffffu, rhs, q, 8);
    if (lr > q) rhs -= a[q] * yq;
  }
  // L' x = y / d on the unscaled entries (as in g8x2_ldlt_solve)
#pragma unroll
  for (int j = D - 1; j >= 0; --j) {
    const T xj = __shfl_sync(0xffffffffu, rhs * rdl, j, 8);
    if (lr < j) rhs -= Lt[j * D + lr] * xj;
  }
  rhs *= rdl;
}

// ---------------------------------------------------------------------------
// Streaming variant: a CTA owns kBulkTasks consecutive knot tasks of one kind and
// brings their operands in with bulk asynchronous copies (TMA, one mbarrier):
// consecutive tasks' Q_k / A_k / q_k / lambda_k blocks are contiguous in the
// b2p_kkt layout, so the CTA's HBM reads are four long sequential streams
// instead of per-lane row loads. The 8-lane groups then solve from shared
// memory (Q_k's block doubles as its L tile).
constexpr int kBulkTasks = 4;
#ifndef B2P_PR_STAGE_A
#define B2P_PR_STAGE_A 0
#endif
constexpr bool kPrStageA = B2P_PR_STAGE_A;

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          static_cast<unsigned>(__cvta_generic_to_shared(dst))),
      "l"(src), "r"(bytes), "r"(mbar)
      : "memory");
}

template <class T, int NB, int MB, bool SA>
__global__ void __launch_bounds__(8 * kBulkTasks) k_reconstruct_primal_bulk(PrimalParams<T> p) {
  constexpr int H = NB / 2, NN = NB * NB;
  extern __shared__ __align__(16) unsigned char praw[];
  T* sm = reinterpret_cast<T*>(praw);
  __shared__ __align__(8) unsigned long long mbar;
  const unsigned mb = static_cast<unsigned>(__cvta_generic_to_shared(&mbar));
  const int grp = threadIdx.x >> 3, l = threadIdx.x & 7;
  const int N = p.N, K = N + 1;
  // 32-bit task indices (the launcher guarantees B K < 2^31)
  const int nx = p.B * K, nu = p.B * N;
  const int nsc = (nx + kBulkTasks - 1) / kBulkTasks;  // state CTAs come first
  const size_t pd = static_cast<size_t>(K) * NB + static_cast<size_t>(N) * MB;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mb) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // state and control CTAs interleaved (2c: state, 2c + 1: control while both
  // remain), so every SM streams a mix of the heavy and the light tasks
  const int ncc = (nu + kBulkTasks - 1) / kBulkTasks;
  const int bx = static_cast<int>(blockIdx.x), mix = 2 * (nsc < ncc ? nsc : ncc);
  const bool is_state = bx < mix ? (bx & 1) == 0 : nsc > ncc;
  const int cta = bx < mix ? bx >> 1 : bx - mix / 2;  // index within its kind
  if (is_state) {
    // ---- state solves: tasks t = t0 .. t0 + nt - 1, t = sys K + k
    const int t0 = cta * kBulkTasks;
    const int nt = nx - t0 < kBulkTasks ? nx - t0 : kBulkTasks;
    // A blocks: a(t) = t - sys(t) for k < N; contiguous over the range
    const int sys0 = t0 / K;
    const int a_lo = t0 - sys0;  // = a(t0), or a of the next task when k0 = N
    const int t1 = t0 + nt - 1, sys1 = t1 / K, k1 = t1 - sys1 * K;
    const int a_hi = k1 < N ? t1 - sys1 : t1 - 1 - sys1;  // inclusive
    const int na = a_hi >= a_lo ? a_hi - a_lo + 1 : 0;
    const int nl = (nx - t0) < nt + 1 ? (nx - t0) : nt + 1;  // lambda blocks
    T* sQ = sm;                              // [16][NN] (then the L tiles)
    T* sA = sQ + kBulkTasks * NN;            // [16][NN] (SA: A_k staged; else read through L1)
    T* sq = sA + (SA ? kBulkTasks * NN : 0);  // [16][NB]
    T* sl = sq + kBulkTasks * NB;            // [17][NB]
    if (threadIdx.x == 0) {
      const unsigned bq = static_cast<unsigned>(sizeof(T) * nt * NN), ba = static_cast<unsigned>(sizeof(T) * na * NN);
      const unsigned bv = static_cast<unsigned>(sizeof(T) * nt * NB), bl = static_cast<unsigned>(sizeof(T) * nl * NB);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(bq + (SA ? ba : 0u) + bv + bl) : "memory");
      bulk_g2s(sQ, p.Q + static_cast<size_t>(t0) * NN, bq, mb);
      if (SA && na) bulk_g2s(sA, p.A + static_cast<size_t>(a_lo) * NN, ba, mb);
      bulk_g2s(sq, p.q + static_cast<size_t>(t0) * NB, bv, mb);
      bulk_g2s(sl, p.lambda + static_cast<size_t>(t0) * NB, bl, mb);
    }
    {
      unsigned done = 0;
      while (!done)
        asm volatile("{\n.reg .pred q;\nmbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0;\nselp.u32 %0, 1, 0, q;\n}\n"
                     : "=r"(done) : "r"(mb) : "memory");
    }
    const bool tv = grp < nt;
    const int j = tv ? grp : nt - 1;  // groups past the range duplicate the last task, store nothing
    const int t = t0 + j;
    const int sys = t / K, k = t - sys * K;
    const int lr = l < H ? l : H - 1;
    T* Qb = sQ + static_cast<size_t>(j) * NN;
    T a0[NB], a1[NB];
#pragma unroll
    for (int c = 0; c < NB; c += 2) {
      const double2 u = *reinterpret_cast<const double2*>(Qb + lr * NB + c);
      const double2 v = *reinterpret_cast<const double2*>(Qb + (lr + H) * NB + c);
      a0[c] = u.x; a0[c + 1] = u.y; a1[c] = v.x; a1[c + 1] = v.y;
    }
    T at0 = T(0), at1 = T(0);
    if (k < N) {  // (A_k' lambda_{k+1})_r = sum_c A_k(c, r) lambda_{k+1, c}
      auto ldA = [](const T* a) { return SA ? *a : __ldg(a); };
      const T* Ab = SA ? sA + static_cast<size_t>(t - sys - a_lo) * NN : p.A + static_cast<size_t>(t - sys) * NN;
      const T* l1 = sl + static_cast<size_t>(j + 1) * NB;
#pragma unroll
      for (int c = 0; c < NB; c += 2) {
        const double2 lv = *reinterpret_cast<const double2*>(l1 + c);
        at0 += ldA(Ab + c * NB + lr) * lv.x;
        at1 += ldA(Ab + c * NB + lr + H) * lv.x;
        at0 += ldA(Ab + (c + 1) * NB + lr) * lv.y;
        at1 += ldA(Ab + (c + 1) * NB + lr + H) * lv.y;
      }
    }
    const T* qk = sq + static_cast<size_t>(j) * NB;
    const T* lk = sl + static_cast<size_t>(j) * NB;
    T r0 = -(qk[lr] + lk[lr] - at0);
    T r1 = -(qk[lr + H] + lk[lr + H] - at1);
    // duplicates work in place on their own copy? no: they share the last
    // task's block, so they factor in a scratch tile instead
    T* Lt = tv ? Qb : (SA ? sA + static_cast<size_t>(kBulkTasks - 1 - grp) * NN : sQ + static_cast<size_t>(grp) * NN);
    __syncthreads();  // every group has its rows; A blocks consumed (duplicates' scratch)
    g8x2_ldlt_solve<T, NB>(a0, a1, r0, r1, Lt, l);
    if (tv && l < H) {
      T* dz = p.dz + static_cast<size_t>(sys) * pd + static_cast<size_t>(k) * (NB + MB);
      dz[lr] = r0;
      dz[lr + H] = r1;
    }
  } else {
    // ---- control solves: tasks u = u0 .. u0 + nt - 1, u = sys N + k
    const int u0 = cta * kBulkTasks;
    if (MB == 0 || u0 >= nu) return;
    const int nt = nu - u0 < kBulkTasks ? nu - u0 : kBulkTasks;
    // lambda_{k+1} blocks: index (u + sys + 1) over the range (contiguous)
    const int s0 = u0 / N, s1 = (u0 + nt - 1) / N;
    const int l_lo = u0 + s0 + 1, l_hi = u0 + nt - 1 + s1 + 1;
    const int nl = l_hi - l_lo + 1;
    T* sB = sm;                              // [16][NB MB]
    T* sl = sB + kBulkTasks * NB * MB;       // [<= 16 + #systems][NB]
    T* sR = sl + (kBulkTasks + 2 + kBulkTasks / (N > 0 ? N : 1)) * NB;  // [16][MB MB] (plain loads)
    // R_k (and r_k) blocks are 8-byte sized: bulk copies only where the range
    // happens to be 16-byte aligned (always, inside whole batches with an even
    // task count per CTA), plain loads otherwise
    const T* Rg = p.R + static_cast<size_t>(u0) * MB * MB;
    const unsigned br = static_cast<unsigned>(sizeof(T) * nt * MB * MB);
    const bool r_bulk = ((reinterpret_cast<uintptr_t>(Rg) | br) & 15u) == 0;
    T* sr_ = sR + static_cast<size_t>(2 * kBulkTasks) * MB * MB;  // [tasks][MB] r_k
    const T* rg = p.r + static_cast<size_t>(u0) * MB;
    const unsigned bv = static_cast<unsigned>(sizeof(T) * nt * MB);
    const bool v_bulk = ((reinterpret_cast<uintptr_t>(rg) | bv) & 15u) == 0;
    if (threadIdx.x == 0) {
      const unsigned bb = static_cast<unsigned>(sizeof(T) * nt * NB * MB), bl = static_cast<unsigned>(sizeof(T) * nl * NB);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb),
                   "r"(bb + bl + (r_bulk ? br : 0u) + (v_bulk ? bv : 0u)) : "memory");
      bulk_g2s(sB, p.B_ + static_cast<size_t>(u0) * NB * MB, bb, mb);
      bulk_g2s(sl, p.lambda + static_cast<size_t>(l_lo) * NB, bl, mb);
      if (r_bulk) bulk_g2s(sR, Rg, br, mb);
      if (v_bulk) bulk_g2s(sr_, rg, bv, mb);
    }
    if (!r_bulk)
      for (int i = threadIdx.x; i < nt * MB * MB; i += 8 * kBulkTasks) sR[i] = __ldg(Rg + i);
    if (!v_bulk)
      for (int i = threadIdx.x; i < nt * MB; i += 8 * kBulkTasks) sr_[i] = __ldg(rg + i);
    __syncthreads();
    {
      unsigned done = 0;
      while (!done)
        asm volatile("{\n.reg .pred q;\nmbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0;\nselp.u32 %0, 1, 0, q;\n}\n"
                     : "=r"(done) : "r"(mb) : "memory");
    }
    const bool tv = grp < nt;
    const int j = tv ? grp : nt - 1;
    const int u = u0 + j;
    const int sys = u / N, k = u - sys * N;
    const int lr = l < MB ? l : MB - 1;
    T a[MB];
#pragma unroll
    for (int c = 0; c < MB; ++c) a[c] = sR[j * MB * MB + lr * MB + c];
    const T* Bb = sB + static_cast<size_t>(j) * NB * MB;
    const T* l1 = sl + static_cast<size_t>(u + sys + 1 - l_lo) * NB;
    T bt = T(0);
#pragma unroll
    for (int c = 0; c < NB; c += 2) {
      const double2 lv = *reinterpret_cast<const double2*>(l1 + c);
      bt += Bb[c * MB + lr] * lv.x;
      bt += Bb[(c + 1) * MB + lr] * lv.y;
    }
    T rhs = -(sr_[j * MB + lr] - bt);
    T* Lt = sR + static_cast<size_t>(kBulkTasks) * MB * MB + grp * MB * MB;  // private scratch
    g8_ldlt_solve<T, MB>(a, rhs, Lt, l);
    if (tv && l < MB)
      p.dz[static_cast<size_t>(sys) * pd + static_cast<size_t>(k) * (NB + MB) + NB + lr] = rhs;
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
  auto bulk_launch = [&](auto kern, int nb, int mbk) {
    const long long nx = static_cast<long long>(p.B) * (p.N + 1);
    const long long nu = static_cast<long long>(p.B) * p.N;
    const long long grid = (nx + kBulkTasks - 1) / kBulkTasks + (nu + kBulkTasks - 1) / kBulkTasks;
    const size_t st_b = sizeof(T) * ((kPrStageA ? 2 : 1) * kBulkTasks * nb * nb + (2 * kBulkTasks + 1) * nb);
    const size_t ct_b = sizeof(T) * (kBulkTasks * nb * mbk + (kBulkTasks + 2 + kBulkTasks) * nb +
                                     2 * kBulkTasks * mbk * mbk + kBulkTasks * mbk) + 16;
    const size_t smem = st_b > ct_b ? st_b : ct_b;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<static_cast<unsigned>(grid), 8 * kBulkTasks, smem, st>>>(p);
    return cudaGetLastError();
  };
  if (tasks / kPrHw < 0x7fffffffLL) {
    if constexpr (sizeof(T) == 8) {
      if (p.n == 14 && p.m == 7 && tasks < 0x7fffffffLL && !std::getenv("B2P_PRIMAL_HW"))
        return bulk_launch(k_reconstruct_primal_bulk<T, 14, 7, kPrStageA>, 14, 7);  // 32-bit task indices
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
