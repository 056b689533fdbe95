// Warp-cooperative small dense linear algebra on shared memory tiles
// (n <= 32). Used by Schur formation (K1), the preconditioner build (K2)
// and the block-Cholesky baseline. Operand reads are shared-memory
// broadcasts or unit-stride across lanes; tiles use an odd leading dimension
// so column access by lanes is bank-conflict free for 8-byte types.
#pragma once

#include "common.cuh"

namespace b2p {

constexpr unsigned kFull = 0xffffffffu;

template <class T>
struct Tile {
  T* p;
  int ld;
  __device__ __forceinline__ T& operator()(int i, int j) const { return p[i * ld + j]; }
};

__host__ __device__ __forceinline__ int tile_ld(int cols) { return cols | 1; }

// Copy a contiguous row-major rows x cols block from global to a tile.
template <class T>
__device__ __forceinline__ void tload(Tile<T> M, const T* __restrict__ g, int rows, int cols,
                                      int lane) {
  for (int idx = lane; idx < rows * cols; idx += 32) M(idx / cols, idx % cols) = g[idx];
  __syncwarp();
}

template <class T>
__device__ __forceinline__ void tstore(T* __restrict__ g, Tile<T> M, int rows, int cols, int lane,
                                       bool negate = false, bool transpose = false) {
  for (int idx = lane; idx < rows * cols; idx += 32) {
    const int i = idx / cols, j = idx % cols;
    const T v = transpose ? M(j, i) : M(i, j);
    g[idx] = negate ? -v : v;
  }
  __syncwarp();  // every lane has read the tile before anyone reuses it
}

template <class T>
__device__ __forceinline__ void tzero_global(T* __restrict__ g, int count, int lane) {
  for (int idx = lane; idx < count; idx += 32) g[idx] = T(0);
}

// In-place lower Cholesky, left-looking like Eigen's llt_inplace::unblocked:
// x = A(k,k) - sum_{p<k} L(k,p)^2, fail iff x <= 0 (a NaN pivot passes, as in
// Eigen), L(i,k) = (A(i,k) - sum_{p<k} L(i,p) L(k,p)) / L(k,k). Only the
// lower triangle is read. Returns the failing pivot or -1.
template <class T>
__device__ int tcholesky(Tile<T> A, int n, int lane) {
  for (int k = 0; k < n; ++k) {
    T s = T(0);
    if (lane >= k && lane < n) {
      s = A(lane, k);
      for (int p = 0; p < k; ++p) s -= A(lane, p) * A(k, p);
    }
    const T x = __shfl_sync(kFull, s, k);
    if (x <= T(0)) return k;
    const T r = rsqrt(x);  // 1/L(k,k); multiplications instead of divisions
    const T d = x * r;
    __syncwarp();
    if (lane == k) A(k, k) = d;
    else if (lane > k && lane < n) A(lane, k) = s * r;
    __syncwarp();
  }
  return -1;
}

// X = (L L')^{-1}: lane j solves L L' x = e_j (forward then backward
// substitution, LLT::solve against the identity).
template <class T>
__device__ void tllt_inverse(Tile<T> L, Tile<T> X, int n, int lane) {
  if (lane < n) {
    const int j = lane;
    // column j of L^-1 is zero above row j: start the forward sweep at j
    for (int i = 0; i < j; ++i) X(i, j) = T(0);
    for (int i = j; i < n; ++i) {
      T s = (i == j) ? T(1) : T(0);
      for (int p = j; p < i; ++p) s -= L(i, p) * X(p, j);
      X(i, j) = s * (T(1) / L(i, i));
    }
    for (int i = n - 1; i >= 0; --i) {
      T s = X(i, j);
      for (int p = i + 1; p < n; ++p) s -= L(p, i) * X(p, j);
      X(i, j) = s * (T(1) / L(i, i));
    }
  }
  __syncwarp();
}

// Solve L L' x = b in place for one vector held in a tile column `col`
// (all lanes cooperate trivially: lane 0 does the sequential work).
template <class T>
__device__ void tllt_solve_vec(Tile<T> L, T* v, int n, int lane) {
  if (lane == 0) {
    for (int i = 0; i < n; ++i) {
      T s = v[i];
      for (int p = 0; p < i; ++p) s -= L(i, p) * v[p];
      v[i] = s / L(i, i);
    }
    for (int i = n - 1; i >= 0; --i) {
      T s = v[i];
      for (int p = i + 1; p < n; ++p) s -= L(p, i) * v[p];
      v[i] = s / L(i, i);
    }
  }
  __syncwarp();
}

// X <- 0.5 (X + X') in place. 0.5*(a+b) == 0.5*(b+a) bitwise, so the
// result is exactly symmetric (schur.cpp:22).
template <class T>
__device__ __forceinline__ void tsymmetrize(Tile<T> X, int n, int lane) {
  if (lane < n) {
    const int j = lane;
    for (int i = 0; i < j; ++i) {
      const T v = T(0.5) * (X(i, j) + X(j, i));
      X(i, j) = v;
      X(j, i) = v;
    }
  }
  __syncwarp();
}

// C = op(A) * op(B) with lane = output column; A is rows x inner.
// transB: use B' (B stored cols x inner). negA: use -A (exact).
template <class T>
__device__ void tgemm(Tile<T> C, Tile<T> A, Tile<T> B, int rows, int inner, int cols, int lane,
                      bool transB = false, bool negA = false) {
  if (lane < cols) {
    const int j = lane;
    for (int i = 0; i < rows; ++i) {
      T s = T(0);
      for (int p = 0; p < inner; ++p) {
        const T a = negA ? -A(i, p) : A(i, p);
        s += a * (transB ? B(j, p) : B(p, j));
      }
      C(i, j) = s;
    }
  }
  __syncwarp();
}

// y = A x (rows x cols), x and y in shared memory; lane = output row.
template <class T>
__device__ __forceinline__ void tgemv(T* y, Tile<T> A, const T* x, int rows, int cols, int lane) {
  if (lane < rows) {
    T s = T(0);
    for (int p = 0; p < cols; ++p) s += A(lane, p) * x[p];
    y[lane] = s;
  }
  __syncwarp();
}

// SPD inverse with the reference's failure semantics (schur.cpp:15-23):
// W (tile, consumed as scratch) -> X = sym((W)^{-1}). Returns pivot or -1.
template <class T>
__device__ int tspd_inverse(Tile<T> W, Tile<T> X, int n, int lane) {
  const int f = tcholesky(W, n, lane);
  if (f >= 0) return f;
  tllt_inverse(W, X, n, lane);
  tsymmetrize(X, n, lane);
  return -1;
}

}  // namespace b2p
