// Half-warp (16-lane) dense helpers shared by the fused kernels
// (fused_kernels.cu: one CTA per system; fc_kernels.cu: one cluster per
// system). One 16-lane half-warp owns one n x n block (n <= 16): lane l owns
// row / column l. Every shuffle and __syncwarp uses the half-warp's own lane
// mask, so the two half-warps of a warp may take different branches.
#pragma once

#include "kernels.h"

namespace b2p {
namespace hwd {

constexpr unsigned FULL = 0xffffffffu;

// Predicated shared-memory stores (@p st.shared): the inverse routines' "only
// the owning lane stores" steps without the divergent branches the compiler
// otherwise builds around them.
__device__ __forceinline__ void sts_if(double* a, double v, bool pred) {
  asm volatile("{\n.reg .pred q;\nsetp.ne.u32 q, %2, 0;\n@q st.shared.f64 [%0], %1;\n}\n" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(a))),
               "d"(v), "r"(static_cast<unsigned>(pred))
               : "memory");
}
__device__ __forceinline__ void sts_if(float* a, float v, bool pred) {
  asm volatile("{\n.reg .pred q;\nsetp.ne.u32 q, %2, 0;\n@q st.shared.f32 [%0], %1;\n}\n" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(a))),
               "f"(v), "r"(static_cast<unsigned>(pred))
               : "memory");
}
__device__ __forceinline__ void sts2_if(double* a, double v0, double v1, bool pred) {
  asm volatile("{\n.reg .pred q;\nsetp.ne.u32 q, %3, 0;\n@q st.shared.v2.f64 [%0], {%1, %2};\n}\n" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(a))),
               "d"(v0), "d"(v1), "r"(static_cast<unsigned>(pred))
               : "memory");
}

template <int N>
struct Odd {
  static constexpr int v = N | 1;
};

// ---------------------------------------------------------------- half-warp dense helpers
// Each 16-lane half-warp runs these independently (the two half-warps of a
// warp may take different branches, e.g. block row 0 vs row 1), so every
// shuffle / __syncwarp uses the half-warp's own lane mask. Lanes l >= N
// compute on clamped data and never store.
__device__ __forceinline__ unsigned hw_mask() {
  return 0xffffu << (threadIdx.x & 16);
}

// In-place lower Cholesky of an N x N tile (stride LD, lower triangle read),
// left-looking like Eigen's llt_inplace::unblocked. Returns the first failing
// pivot (x <= 0; a NaN pivot passes, as in Eigen) or -1.
template <class T, int N, int LD>
__device__ __forceinline__ int hw_cholesky(T* A, T* rd, int l) {
  // In-place lower Cholesky of an N x N tile (stride LD, lower triangle read),
  // left-looking like Eigen's llt_inplace::unblocked; rd[k] = 1 / L(k,k).
  // Returns the first failing pivot (x <= 0; a NaN pivot passes, as in Eigen)
  // or -1. Divisions are replaced by one reciprocal per pivot.
  int fail = -1;
  const int lr = l < N ? l : N - 1;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    T s = A[lr * LD + k];
#pragma unroll
    for (int p = 0; p < k; ++p) s -= A[lr * LD + p] * A[k * LD + p];
    T x = __shfl_sync(hw_mask(), s, k, 16);
    const bool bad = x <= T(0);  // branch-free: fails on x <= 0, NaN passes
    fail = (bad && fail < 0) ? k : fail;
    x = bad ? T(1) : x;
    const T r = rsqrt(x);  // one MUFU sequence per pivot: 1/L(k,k) and L(k,k) = x * r
    const T val = (l == k ? x : s) * r;
    __syncwarp(hw_mask());
    if (l >= k && l < N) A[l * LD + k] = val;
    if (l == k) rd[k] = r;
    __syncwarp(hw_mask());
  }
  return fail;
}

// x = column j of (L L')^{-1} (forward then backward substitution against e_j).
template <class T, int N, int LD>
__device__ __forceinline__ void hw_inv_col(const T* L, const T* rd, int j, T (&x)[N]) {
  // __syncwarp between rows stops the scheduler from hoisting all N^2/2
  // tile loads ahead of the recurrence (register blow-up / spills).
#pragma unroll
  for (int i = 0; i < N; ++i) {
    T s = (i == j) ? T(1) : T(0);
#pragma unroll
    for (int p = 0; p < i; ++p) s -= L[i * LD + p] * x[p];
    x[i] = s * rd[i];
    __syncwarp(hw_mask());
  }
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
    T s = x[i];
#pragma unroll
    for (int p = i + 1; p < N; ++p) s -= L[p * LD + i] * x[p];
    x[i] = s * rd[i];
    __syncwarp(hw_mask());
  }
}

// column j of X -> column j of 0.5 (X + X') through the tile W (overwritten).
// FW: both half-warps of the warp call together (convergent) -> full-warp
// masks, no divergence bookkeeping around the shuffles / syncs.
template <class T, int N, int LD, bool FW = false>
__device__ __forceinline__ void hw_symmetrize_col(T* W, int j, T (&x)[N]) {
  const unsigned mk = FW ? FULL : hw_mask();
  __syncwarp(mk);
  if (j < N) {
#pragma unroll
    for (int i = 0; i < N; ++i) W[i * LD + j] = x[i];
  }
  __syncwarp(mk);
  const int jr = j < N ? j : N - 1;
#pragma unroll
  for (int i = 0; i < N; ++i) x[i] = T(0.5) * (x[i] + W[jr * LD + i]);
  __syncwarp(mk);
}

// W <- G (row-major N x N global), cooperative over the half-warp.
template <class T, int N, int LD>
__device__ __forceinline__ void hw_load(T* W, const T* __restrict__ G, int l) {
  __syncwarp(hw_mask());
#pragma unroll
  for (int idx = l; idx < N * N; idx += 16) W[(idx / N) * LD + idx % N] = G[idx];
  __syncwarp(hw_mask());
}

// spd_inverse (schur.cpp:15-23): column j of sym((W)^{-1}); returns pivot / -1.
template <class T, int N, int LD>
__device__ __forceinline__ int hw_spd_inverse(T* W, T* rd, const T* __restrict__ G, int j,
                                              T (&x)[N]) {
  hw_load<T, N, LD>(W, G, j & 15);
  const int f = hw_cholesky<T, N, LD>(W, rd, j);
  hw_inv_col<T, N, LD>(W, rd, j < N ? j : 0, x);
  hw_symmetrize_col<T, N, LD>(W, j, x);
  return f;
}

// Block sum with a single barrier: callers alternate between two `red`
// buffers, and at least one other barrier separates two uses of the same
// buffer, so no trailing barrier is needed before it is rewritten.
template <class T, int kThreads = 512>
__device__ __forceinline__ T block_reduce(T v, T* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  // pairwise tree over the warp partials (fixed order: every thread gets the
  // bit-identical sum; depth log2(#warps)): lane w holds partial w, level st
  // adds lane w + st's value — lane 0 ends with ((t0+t1)+(t2+t3))+... — then
  // broadcasts it (one shared load per lane instead of #warps)
  constexpr int NW = kThreads / 32;
  static_assert((NW & (NW - 1)) == 0 && NW <= 32, "power-of-two warp count");
  T s = lane < NW ? red[lane] : T(0);
#pragma unroll
  for (int st = 1; st < NW; st <<= 1) s += __shfl_down_sync(FULL, s, st);
  return __shfl_sync(FULL, s, 0);
}

// ---------------------------------------------------------------- PCG row products
// R independent block rows per thread are processed together (j outer, row
// inner) with two partial sums per dot product: more independent DFMA chains
// in flight per warp for the same shared-memory traffic.
template <class T, int NB, int R>
__device__ __forceinline__ void dots_row(const T* (&M)[R], const T* (&x)[R], T (&out)[R]) {
  T a[R], c[R];
#pragma unroll
  for (int r = 0; r < R; ++r) a[r] = c[r] = T(0);
#pragma unroll
  for (int j = 0; j < NB; j += 2) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double2 m2 = *reinterpret_cast<const double2*>(M[r] + j);
      const double2 v2 = *reinterpret_cast<const double2*>(x[r] + j);
      a[r] += m2.x * v2.x;
      c[r] += m2.y * v2.y;
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) out[r] = a[r] + c[r];
}
// out[r] = sum_j Mc[r][j*NB] * x[r][j]  (column of a row-major block: R_b = L_{b+1}')
template <class T, int NB, int R>
__device__ __forceinline__ void dots_col(const T* (&Mc)[R], const T* (&x)[R], T (&out)[R]) {
  T a[R], c[R];
#pragma unroll
  for (int r = 0; r < R; ++r) a[r] = c[r] = T(0);
#pragma unroll
  for (int j = 0; j < NB; j += 2) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double2 v2 = *reinterpret_cast<const double2*>(x[r] + j);
      a[r] += Mc[r][j * NB] * v2.x;
      c[r] += Mc[r][(j + 1) * NB] * v2.y;
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) out[r] = a[r] + c[r];
}
// Two rows (pr, pr + NB/2) of one block per thread (the one-CTA kernel's PCG
// mapping): out[c] = sum_j Mc[j*NB + c*NB/2] * x[j] — columns pr and pr + NB/2
// of a row-major block (Mc = block + pr), one broadcast x serving both; same
// two-accumulator order as dots_col.
template <class T, int NB, int LS>
__device__ __forceinline__ void dots_col2(const T* Mc, const T* x, T (&out)[2]) {
  constexpr int H = NB / 2;
  T a0 = T(0), c0 = T(0), a1 = T(0), c1 = T(0);
#pragma unroll
  for (int j = 0; j < NB; j += 2) {
    const double2 v2 = *reinterpret_cast<const double2*>(x + j);
    a0 += Mc[j * NB] * v2.x;
    a1 += Mc[j * NB + H] * v2.x;
    c0 += Mc[(j + 1) * NB] * v2.y;
    c1 += Mc[(j + 1) * NB + H] * v2.y;
  }
  out[0] = a0 + c0;
  out[1] = a1 + c1;
}
// Two rows (pr, pr + NB/2) of one row-major shared block per thread (M = block
// + pr NB) against one broadcast vector x: 16-byte pair loads, the same
// two-accumulator order (even j -> a, odd j -> c) as tm::dot2_row.
template <class T, int NB>
__device__ __forceinline__ void dots_row2(const T* M, const T* x, T (&out)[2]) {
  constexpr int H = NB / 2;
  T a0 = T(0), c0 = T(0), a1 = T(0), c1 = T(0);
#pragma unroll
  for (int j = 0; j < NB; j += 2) {
    const double2 v2 = *reinterpret_cast<const double2*>(x + j);
    const double2 m0 = *reinterpret_cast<const double2*>(M + j);
    const double2 m1 = *reinterpret_cast<const double2*>(M + H * NB + j);
    a0 += m0.x * v2.x;
    c0 += m0.y * v2.y;
    a1 += m1.x * v2.x;
    c1 += m1.y * v2.y;
  }
  out[0] = a0 + c0;
  out[1] = a1 + c1;
}
// out[c] = ti[c] . v for two register rows against one shared vector
template <class T, int NB>
__device__ __forceinline__ void dots_reg2(const T (&ti)[2][NB], const T* v, T (&out)[2]) {
  T a0 = T(0), c0 = T(0), a1 = T(0), c1 = T(0);
#pragma unroll
  for (int j = 0; j < NB; j += 2) {
    const double2 v2 = *reinterpret_cast<const double2*>(v + j);
    a0 += ti[0][j] * v2.x;
    c0 += ti[0][j + 1] * v2.y;
    a1 += ti[1][j] * v2.x;
    c1 += ti[1][j + 1] * v2.y;
  }
  out[0] = a0 + c0;
  out[1] = a1 + c1;
}
// out[r] = ti[r] . v[r]  (theta^-1 row held in registers)
template <class T, int NB, int R>
__device__ __forceinline__ void dots_reg(const T (&ti)[R][NB], const T* (&v)[R], T (&out)[R]) {
  T a[R], c[R];
#pragma unroll
  for (int r = 0; r < R; ++r) a[r] = c[r] = T(0);
#pragma unroll
  for (int j = 0; j < NB; j += 2) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double2 v2 = *reinterpret_cast<const double2*>(v[r] + j);
      a[r] += ti[r][j] * v2.x;
      c[r] += ti[r][j + 1] * v2.y;
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) out[r] = a[r] + c[r];
}

}  // namespace hwd
}  // namespace b2p

namespace b2p {
namespace hwd {

// ---------------------------------------------------------------------------
// Load-efficient half-warp SPD inverse (spd_inverse, schur.cpp:15-23).
// Lane l owns row l. In: a[] = row l of W (registers; only the lower part is
// used, as LLT does). Tiles (row stride N, 16-byte aligned rows for even N):
//   Lr  : rows of L as they are finalised (pivot rows are read as broadcasts),
//   LiT : rows of L^-T (= columns of L^-1).
// 1. left-looking Cholesky (Eigen llt_inplace::unblocked order; x <= 0 fails,
//    a NaN pivot passes) with the own row in registers;
// 2. column l of L^-1 by forward substitution;
// 3. X = L^-T L^-1: x[i] = sum_{p>=i} LiT[i][p] LiT[l][p] — independent dot
//    products. X is bitwise symmetric (same products in the same order for
//    X[i][l] and X[l][i]; the extra terms are exact zeros), so the
//    0.5 (X + X') of the reference is the identity on it.
// Out: x[] = row l (= column l) of W^-1. Returns the failing pivot or -1.
template <class T, int N, bool FW = false>
__device__ __forceinline__ int hw_spd_inverse_v2(T (&a)[N], T* Lr, T* LiT, T* rd, int l,
                                                 T (&x)[N]) {
  const unsigned mk = FW ? FULL : hw_mask();
  int fail = -1;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    T s = a[k];
#pragma unroll
    for (int q = 0; q < k; ++q) s -= a[q] * Lr[k * N + q];
    T piv = __shfl_sync(mk, s, k, 16);
    // branch-free pivot step (selects + predicated stores): x <= 0 fails and
    // is replaced by 1, a NaN pivot passes, as in Eigen's LLT
    const bool bad = piv <= T(0);
    fail = (bad && fail < 0) ? k : fail;
    piv = bad ? T(1) : piv;
    const T r = rsqrt(piv);
    const T val = (l == k ? piv : s) * r;
    const bool own = l >= k && l < N;
    a[k] = own ? val : a[k];
    if (own) Lr[l * N + k] = val;
    if (l == k) rd[k] = r;
    __syncwarp(mk);
  }
  // column l of L^-1 (zero above the diagonal)
  T y[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    T s = (i == l) ? T(1) : T(0);
#pragma unroll
    for (int q = 0; q < i; ++q) s -= Lr[i * N + q] * y[q];
    y[i] = s * rd[i];
  }
  if (l < N) {
#pragma unroll
    for (int q = 0; q < N; ++q) LiT[l * N + q] = y[q];
  }
  __syncwarp(mk);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    T s = T(0);
#pragma unroll
    for (int q = i; q < N; ++q) s += LiT[i * N + q] * y[q];
    x[i] = s;
  }
  __syncwarp(mk);
  return fail;
}


// hw_spd_inverse_v2 on an 8-lane group with two rows per lane: lane l < H =
// N / 2 owns rows l and l + H (lanes >= H duplicate rows H - 1, N - 1 and
// store nothing), so every broadcast operand read from the tiles serves two
// rows — half the shared-memory wavefronts per inverse of the one-row-per-lane
// half-warp version, and four blocks per warp instead of two. The arithmetic
// of every row is hw_spd_inverse_v2's (same operations in the same order), so
// the results are bitwise equal to it.
// a0, a1: rows l, l + H of W (consumed). Lr: [N][N] rows of L — may be the
// source block itself (in place: the routine first waits until every lane
// holds its rows). LiT: [N][N] rows of L^-T (may alias Lr). rd: [N].
// x0, x1: rows l, l + H of W^-1 (bitwise symmetric: also its columns).
// Every lane of the warp must call it (full-warp syncs, width-8 shuffles).
// Returns the first failing pivot (group-uniform) or -1.
template <class T, int N>
__device__ __forceinline__ int g8x2_spd_inverse(T (&a0)[N], T (&a1)[N], T* Lr, T* LiT, T* rd, int l,
                                                T (&x0)[N], T (&x1)[N]) {
  static_assert(N % 2 == 0 && N <= 16, "even N <= 16");
  constexpr int H = N / 2;
  const bool act = l < H;
  const int lr = act ? l : H - 1;
  int fail = -1;
  __syncwarp();  // Lr may be the source block: every lane has read its rows
#pragma unroll
  for (int k = 0; k < N; ++k) {
    T s0 = T(0), s1 = a1[k];
    if (k < H) s0 = a0[k];
#pragma unroll
    for (int q = 0; q < k; ++q) {
      const T v = Lr[k * N + q];
      if (k < H) s0 -= a0[q] * v;
      s1 -= a1[q] * v;
    }
    T piv = __shfl_sync(FULL, k < H ? s0 : s1, k < H ? k : k - H, 8);
    const bool bad = piv <= T(0);  // x <= 0 fails, NaN passes (Eigen LLT)
    fail = (bad && fail < 0) ? k : fail;
    piv = bad ? T(1) : piv;
    const T r = rsqrt(piv);
    // predicated stores (sts_if): no divergent branches around them
    if (k < H) {
      const T v0 = (lr == k ? piv : s0) * r;
      const bool own0 = act && lr >= k;
      a0[k] = own0 ? v0 : a0[k];
      sts_if(Lr + lr * N + k, v0, own0);
    }
    {
      const T v1 = (lr + H == k ? piv : s1) * r;
      const bool own1 = act && lr + H >= k;
      a1[k] = own1 ? v1 : a1[k];
      sts_if(Lr + (lr + H) * N + k, v1, own1);
    }
    sts_if(rd + k, r, act && lr == (k < H ? k : k - H));
    __syncwarp();
  }
  // columns l and l + H of L^-1
  T y0[N], y1[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    T t0 = (i == lr) ? T(1) : T(0), t1 = (i == lr + H) ? T(1) : T(0);
#pragma unroll
    for (int q = 0; q < i; ++q) {
      const T v = Lr[i * N + q];
      t0 -= v * y0[q];
      t1 -= v * y1[q];
    }
    const T d = rd[i];
    y0[i] = t0 * d;
    y1[i] = t1 * d;
  }
  __syncwarp();  // LiT may alias Lr
#pragma unroll
  for (int q = 0; q < N; q += 2) {
    sts2_if(LiT + lr * N + q, y0[q], y0[q + 1], act);
    sts2_if(LiT + (lr + H) * N + q, y1[q], y1[q + 1], act);
  }
  __syncwarp();
  // X[i][c] = sum_{q >= i} LiT[i][q] y_c[q]; y_c[i] dies with row i
#pragma unroll
  for (int i = 0; i < N; ++i) {
    T s0 = T(0), s1 = T(0);
#pragma unroll
    for (int q = i; q < N; ++q) {
      const T v = LiT[i * N + q];
      s0 += v * y0[q];
      s1 += v * y1[q];
    }
    x0[i] = s0;
    x1[i] = s1;
  }
  __syncwarp();
  return fail;
}

// hw_spd_inverse_v2 for N <= 8 on 8-lane groups: a half-warp inverts two
// independent matrices at once (lanes 0-7 and 8-15). l = lane & 7; every lane
// of the warp must call it (full-warp mask, width-8 shuffles); Lr / LiT / rd
// are the calling group's own tiles.
// W: group width (lanes per matrix, N <= W <= 8; W = 2 / 4 packs 16 / 8 groups per warp).
template <class T, int N, int W = 8>
__device__ __forceinline__ int g8_spd_inverse(T (&a)[N], T* Lr, T* LiT, T* rd, int l, T (&x)[N]) {
  static_assert(N <= W && W <= 8, "N <= W <= 8 lanes per group");
  int fail = -1;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    T s = a[k];
#pragma unroll
    for (int q = 0; q < k; ++q) s -= a[q] * Lr[k * N + q];
    T piv = __shfl_sync(FULL, s, k, W);
    const bool bad = piv <= T(0);  // x <= 0 fails, NaN passes (Eigen LLT)
    fail = (bad && fail < 0) ? k : fail;
    piv = bad ? T(1) : piv;
    const T r = rsqrt(piv);
    const T val = (l == k ? piv : s) * r;
    const bool own = l >= k && l < N;
    a[k] = own ? val : a[k];
    sts_if(Lr + l * N + k, val, own);
    sts_if(rd + k, r, l == k);
    __syncwarp();
  }
  T y[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    T s = (i == l) ? T(1) : T(0);
#pragma unroll
    for (int q = 0; q < i; ++q) s -= Lr[i * N + q] * y[q];
    y[i] = s * rd[i];
  }
  if (l < N) {
#pragma unroll
    for (int q = 0; q < N; ++q) LiT[l * N + q] = y[q];
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < N; ++i) {
    T s = T(0);
#pragma unroll
    for (int q = i; q < N; ++q) s += LiT[i * N + q] * y[q];
    x[i] = s;
  }
  __syncwarp();
  return fail;
}

}  // namespace hwd
}  // namespace b2p
