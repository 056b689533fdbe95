// Warp (32-lane) dense helpers for the fused grid kernel (fg_kernels.cu): one
// warp owns one n x n block (n <= 32); lane l owns row / column l. Lanes
// l >= n compute on clamped data and never store.
#pragma once

#include "kernels.h"

namespace b2p {
namespace wpd {

constexpr unsigned FULL = 0xffffffffu;

template <class T> struct V2;
template <> struct V2<double> { using t = double2; };
template <> struct V2<float> { using t = float2; };
template <class T>
__device__ __forceinline__ typename V2<T>::t ld2(const T* p) {
  return *reinterpret_cast<const typename V2<T>::t*>(p);
}

// spd_inverse (schur.cpp:15-23) of the N x N matrix whose row l is a[] (only
// the lower part is read, as Eigen's LLT does). Tiles Lr, LiT: N x N, row
// stride N (16-byte aligned rows for even N); rd: >= N.
//  1. left-looking Cholesky in Eigen's llt_inplace::unblocked order (x <= 0
//     fails, a NaN pivot passes), own row in registers, pivot rows read as
//     broadcasts from Lr;
//  2. column l of L^-1 by forward substitution;
//  3. X = L^-T L^-1: x[i] = sum_{q >= max(i,l)} LiT[i][q] LiT[l][q] — the same
//     products in the same order for X[i][l] and X[l][i], so X is bitwise
//     symmetric and the reference's 0.5 (X + X') is the identity on it.
// Out: x[] = row l (= column l) of the inverse. Returns the failing pivot or -1.
template <class T, int N>
__device__ __forceinline__ int wp_spd_inverse(T (&a)[N], T* Lr, T* LiT, T* rd, int l, T (&x)[N]) {
  int fail = -1;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    T s = a[k];
#pragma unroll
    for (int q = 0; q < k; ++q) s -= a[q] * Lr[k * N + q];
    T piv = __shfl_sync(FULL, s, k);
    // branch-free pivot step: x <= 0 fails (replaced by 1), NaN passes (Eigen LLT)
    const bool bad = piv <= T(0);
    fail = (bad && fail < 0) ? k : fail;
    piv = bad ? T(1) : piv;
    const T r = rsqrt(piv);
    const T val = (l == k ? piv : s) * r;
    const bool own = l >= k && l < N;
    a[k] = own ? val : a[k];
    if (own) Lr[l * N + k] = val;
    if (l == k) rd[k] = r;
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

// sum_j m[j] x[j]: m in registers, x (16-byte aligned) in shared memory
template <class T, int NB>
__device__ __forceinline__ T dot_reg(const T (&m)[NB], const T* x) {
  T a = T(0), c = T(0);
#pragma unroll
  for (int j = 0; j < NB; j += 2) {
    const auto v = ld2<T>(x + j);
    a += m[j] * v.x;
    c += m[j + 1] * v.y;
  }
  return a + c;
}
// row of a row-major block (Mrow = M + l*NB) times x
template <class T, int NB>
__device__ __forceinline__ T dot_row(const T* Mrow, const T* x) {
  T a = T(0), c = T(0);
#pragma unroll
  for (int j = 0; j < NB; j += 2) {
    const auto m = ld2<T>(Mrow + j);
    const auto v = ld2<T>(x + j);
    a += m.x * v.x;
    c += m.y * v.y;
  }
  return a + c;
}
// column of a row-major block (Mcol = M + l) times x
template <class T, int NB>
__device__ __forceinline__ T dot_col(const T* Mcol, const T* x) {
  T a = T(0), c = T(0);
#pragma unroll
  for (int j = 0; j < NB; j += 2) {
    const auto v = ld2<T>(x + j);
    a += Mcol[j * NB] * v.x;
    c += Mcol[(j + 1) * NB] * v.y;
  }
  return a + c;
}

}  // namespace wpd
}  // namespace b2p
