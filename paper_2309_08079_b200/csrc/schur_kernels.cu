// K1 (Schur formation) and K2 (preconditioner construction) for sm_100a,
// plus the block-tridiagonal utilities behind the BlockTriMatrix API.
//
// K1 replaces build_schur's row loop (proj/src/schur.cpp:38-82): one warp per
// (system, block row); the per-knot SPD inverses (spd_inverse, :15-23) are
// warp-cooperative Cholesky + triangular solves on shared-memory tiles.
// K2 replaces build_block_jacobi / build_stair / build_symmetric_stair
// (schur.cpp:98-142): one warp per (system, block row); odd rows form
// (-theta_i^-1 L_i) theta_{i-1}^-1 and the symmetric-stair mirror writes the
// transposes into the neighbouring even rows, so every block is written once
// and no inter-row synchronisation is needed.
#include <climits>

#include <cstdlib>

#include "kernels.h"
#include "warp_dense.cuh"

namespace b2p {

// ----------------------------------------------------------------- K1
template <class T>
struct FormLayout {
  int n, m, ldn, ldm;
  // tile offsets (elements) inside one warp's scratch
  int oA, oB, oQi, oRi, oQ1, oAQ, oBR, oT, oW, vq, vr, vq1, ve, vqq, vrr, vt1, vt2, vt3, total;
  __host__ __device__ FormLayout(int n_, int m_) : n(n_), m(m_) {
    ldn = tile_ld(n);
    ldm = tile_ld(m > 0 ? m : 1);
    const int tn = n * ldn, tm = (m > 0 ? m : 1) * ldm, tnm = n * ldm;
    int o = 0;
    oA = o; o += tn;
    oB = o; o += tnm;
    oQi = o; o += tn;
    oRi = o; o += tm;
    oQ1 = o; o += tn;
    oAQ = o; o += tn;
    oBR = o; o += tnm;
    oT = o; o += tn;
    oW = o; o += tn > tm ? tn : tm;  // also the R_k factorisation scratch (m > n)
    vq = o; o += 32;
    vr = o; o += 32;
    vq1 = o; o += 32;
    ve = o; o += 32;
    vqq = o; o += 32;
    vrr = o; o += 32;
    vt1 = o; o += 32;
    vt2 = o; o += 32;
    vt3 = o; o += 32;
    total = o;
  }
};

template <class T>
size_t form_smem_per_warp(int n, int m) {
  return sizeof(T) * static_cast<size_t>(FormLayout<T>(n, m).total);
}

__device__ __forceinline__ void record_error(int* errkey, int key) {
  if (errkey) atomicMin(errkey, key);
}

template <class T>
__global__ void k_build_schur(FormParams<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int wpc = blockDim.x >> 5;
  const int K = p.N + 1, n = p.n, m = p.m;
  const long long gw = static_cast<long long>(blockIdx.x) * wpc + warp;
  if (gw >= static_cast<long long>(p.B) * K) return;
  const int sys = static_cast<int>(gw / K);
  const int b = static_cast<int>(gw % K);

  const FormLayout<T> L(n, m);
  T* base = reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(warp) * L.total;
  Tile<T> tA{base + L.oA, L.ldn}, tB{base + L.oB, L.ldm}, tQi{base + L.oQi, L.ldn},
      tRi{base + L.oRi, L.ldm}, tQ1{base + L.oQ1, L.ldn}, tAQ{base + L.oAQ, L.ldn},
      tBR{base + L.oBR, L.ldm}, tT{base + L.oT, L.ldn}, tW{base + L.oW, L.ldn};
  T* vq = base + L.vq;
  T* vr = base + L.vr;
  T* vq1 = base + L.vq1;
  T* ve = base + L.ve;
  T* vqq = base + L.vqq;
  T* vrr = base + L.vrr;
  T* vt1 = base + L.vt1;
  T* vt2 = base + L.vt2;
  T* vt3 = base + L.vt3;

  const size_t nn = static_cast<size_t>(n) * n, nm = static_cast<size_t>(n) * m,
               mm = static_cast<size_t>(m) * m;
  const T* Qs = p.Q + static_cast<size_t>(sys) * K * nn;
  const T* qs = p.q + static_cast<size_t>(sys) * K * n;
  const T* Rs = p.R + static_cast<size_t>(sys) * p.N * mm;
  const T* rs = p.r + static_cast<size_t>(sys) * p.N * m;
  const T* As = p.A + static_cast<size_t>(sys) * p.N * nn;
  const T* Bs = p.Bm + static_cast<size_t>(sys) * p.N * nm;
  const T* es = p.e + static_cast<size_t>(sys) * p.N * n;
  const T* xs = p.x_s + static_cast<size_t>(sys) * n;
  const T* x0 = p.x0 + static_cast<size_t>(sys) * n;
  T* S = p.S + static_cast<size_t>(sys) * K * 3 * nn;
  T* gam = p.gamma + static_cast<size_t>(sys) * K * n;
  T* ti = p.theta_inv + static_cast<size_t>(sys) * K * nn;
  int* ek = p.errkey ? p.errkey + sys : nullptr;

  auto blk = [&](int row, int slot) { return S + (static_cast<size_t>(row) * 3 + slot) * nn; };

  if (b == K - 1) tzero_global(blk(b, 2), static_cast<int>(nn), lane);  // right padding

  if (b == 0) {
    // schur.cpp:53-57
    tzero_global(blk(0, 0), static_cast<int>(nn), lane);  // left padding
    tload(tW, Qs, n, n, lane);
    if (tspd_inverse(tW, tQi, n, lane) >= 0) {
      if (lane == 0) record_error(ek, 0);
      return;
    }
    tstore(blk(0, 1), tQi, n, n, lane);
    // theta_inv[0] = 0.5 (Q0 + Q0')
    tload(tT, Qs, n, n, lane);
    tsymmetrize(tT, n, lane);
    tstore(ti, tT, n, n, lane);
    if (lane < n) vq[lane] = qs[lane];
    __syncwarp();
    tgemv(vt1, tQi, vq, n, n, lane);
    if (lane < n) gam[lane] = -((xs[lane] - x0[lane]) + vt1[lane]);
    return;
  }

  // schur.cpp:58-78, k = b - 1
  const int k = b - 1;
  tload(tA, As + k * nn, n, n, lane);
  tload(tB, Bs + k * nm, n, m, lane);
  if (lane < n) {
    vq[lane] = qs[static_cast<size_t>(k) * n + lane];
    vq1[lane] = qs[static_cast<size_t>(k + 1) * n + lane];
    ve[lane] = es[static_cast<size_t>(k) * n + lane];
  }
  if (lane < m) vr[lane] = rs[static_cast<size_t>(k) * m + lane];
  __syncwarp();

  tload(tW, Qs + k * nn, n, n, lane);
  if (tspd_inverse(tW, tQi, n, lane) >= 0) {
    if (lane == 0) record_error(ek, b * 4 + 0);
    return;
  }
  {
    Tile<T> tWm{tW.p, L.ldm};
    tload(tWm, Rs + k * mm, m, m, lane);
    if (tspd_inverse(tWm, tRi, m, lane) >= 0) {
      if (lane == 0) record_error(ek, b * 4 + 1);
      return;
    }
  }
  tload(tW, Qs + (k + 1) * nn, n, n, lane);
  if (tspd_inverse(tW, tQ1, n, lane) >= 0) {
    if (lane == 0) record_error(ek, b * 4 + 2);
    return;
  }

  tgemm(tAQ, tA, tQi, n, n, n, lane);  // A Qk^-1
  tgemm(tBR, tB, tRi, n, m, m, lane);  // B Rk^-1
  // theta_raw = (A Qk^-1) A' + (B Rk^-1) B' + Qk1^-1   (schur.cpp:65-66)
  if (lane < n) {
    const int j = lane;
    for (int i = 0; i < n; ++i) {
      T s1 = T(0), s2 = T(0);
      for (int q = 0; q < n; ++q) s1 += tAQ(i, q) * tA(j, q);
      for (int q = 0; q < m; ++q) s2 += tBR(i, q) * tB(j, q);
      tT(i, j) = (s1 + s2) + tQ1(i, j);
    }
  }
  __syncwarp();
  tsymmetrize(tT, n, lane);  // theta (schur.cpp:67)
  tstore(blk(b, 1), tT, n, n, lane);
  tstore(blk(b, 0), tAQ, n, n, lane, /*negate=*/true);                     // phi = -A Qk^-1
  tstore(blk(b - 1, 2), tAQ, n, n, lane, /*negate=*/true, /*transpose=*/true);  // phi'

  // zeta = -A (Qk^-1 q) - B (Rk^-1 r) + Qk1^-1 q_{k+1}  (schur.cpp:69-70)
  tgemv(vqq, tQi, vq, n, n, lane);
  tgemv(vrr, tRi, vr, m, m, lane);
  tgemv(vt1, tA, vqq, n, n, lane);
  tgemv(vt2, tB, vrr, n, m, lane);
  tgemv(vt3, tQ1, vq1, n, n, lane);
  if (lane < n) {
    const T zeta = (-vt1[lane] - vt2[lane]) + vt3[lane];
    gam[static_cast<size_t>(b) * n + lane] = -(-ve[lane] + zeta);  // -(c_b + zeta), c_b = -e_k
  }
  // theta_inv[b] = spd_inverse(theta) (schur.cpp:75)
  for (int idx = lane; idx < n * n; idx += 32) tW(idx / n, idx % n) = tT(idx / n, idx % n);
  __syncwarp();
  if (tspd_inverse(tW, tQi, n, lane) >= 0) {
    if (lane == 0) record_error(ek, b * 4 + 3);
    return;
  }
  tstore(ti + static_cast<size_t>(b) * nn, tQi, n, n, lane);
}

// ----------------------------------------------------------------- K2
template <class T>
__global__ void k_build_precond(PrecondParams<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int wpc = blockDim.x >> 5;
  const int K = p.K, n = p.nb;
  const long long gw = static_cast<long long>(blockIdx.x) * wpc + warp;
  if (gw >= static_cast<long long>(p.B) * K) return;
  const int sys = static_cast<int>(gw / K);
  const int row = static_cast<int>(gw % K);
  const int ld = tile_ld(n);
  const size_t nn = static_cast<size_t>(n) * n;
  T* base = reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(warp) * 4 * n * ld;
  Tile<T> tI{base, ld}, tL{base + n * ld, ld}, tJ{base + 2 * n * ld, ld}, tX{base + 3 * n * ld, ld};
  const T* S = p.S + static_cast<size_t>(sys) * K * 3 * nn;
  const T* ti = p.theta_inv + static_cast<size_t>(sys) * K * nn;
  T* Phi = p.phi + static_cast<size_t>(sys) * K * 3 * nn;
  auto blk = [&](T* M, int r, int slot) { return M + (static_cast<size_t>(r) * 3 + slot) * nn; };
  auto cblk = [&](const T* M, int r, int slot) {
    return M + (static_cast<size_t>(r) * 3 + slot) * nn;
  };

  // diag = theta_inv[row] for every non-identity kind
  for (int idx = lane; idx < static_cast<int>(nn); idx += 32)
    blk(Phi, row, 1)[idx] = ti[static_cast<size_t>(row) * nn + idx];
  const bool stair_like = (p.kind == kStair || p.kind == kSymStair || p.kind == kPoly);
  const bool odd = (row % 2) == 1;
  if (!stair_like || !odd) {
    // even rows: off-diagonals zero unless the symmetric-stair mirror of an
    // odd neighbour writes them (then the odd neighbour owns them).
    const bool mirror = (p.kind == kSymStair);
    if (!mirror || row == 0) tzero_global(blk(Phi, row, 0), static_cast<int>(nn), lane);
    if (!mirror || row + 1 >= K) tzero_global(blk(Phi, row, 2), static_cast<int>(nn), lane);
    return;
  }
  // odd row: left = (-theta_i^-1 L_i) theta_{i-1}^-1   (schur.cpp:119-120)
  tload(tI, ti + static_cast<size_t>(row) * nn, n, n, lane);
  tload(tL, cblk(S, row, 0), n, n, lane);
  tload(tJ, ti + static_cast<size_t>(row - 1) * nn, n, n, lane);
  tgemm(tX, tI, tL, n, n, n, lane, false, /*negA=*/true);
  tgemm(tL, tX, tJ, n, n, n, lane);
  tstore(blk(Phi, row, 0), tL, n, n, lane);
  if (p.kind == kSymStair) tstore(blk(Phi, row - 1, 2), tL, n, n, lane, false, true);
  if (row + 1 < K) {
    // right = (-theta_i^-1 R_i) theta_{i+1}^-1   (schur.cpp:121-123)
    tload(tL, cblk(S, row, 2), n, n, lane);
    tload(tJ, ti + static_cast<size_t>(row + 1) * nn, n, n, lane);
    tgemm(tX, tI, tL, n, n, n, lane, false, true);
    tgemm(tL, tX, tJ, n, n, n, lane);
    tstore(blk(Phi, row, 2), tL, n, n, lane);
    if (p.kind == kSymStair) tstore(blk(Phi, row + 1, 0), tL, n, n, lane, false, true);
  } else {
    tzero_global(blk(Phi, row, 2), static_cast<int>(nn), lane);
  }
}

// ----------------------------------------------------------------- utilities
// y = M x for one or many block-tridiagonal matrices; one thread per scalar
// row (block_tri.cpp:82-92). mode 1 = the poly_split remainder E = Psi - S
// implied by S: even rows -L, -R; odd rows zero (schur.cpp:150-159).
template <class T>
__global__ void k_blocktri_matvec(int B, int K, int nb, const T* __restrict__ M,
                                  const T* __restrict__ x, T* __restrict__ y, int mode,
                                  const T* __restrict__ add_to, T* __restrict__ acc) {
  const long long D = static_cast<long long>(K) * nb;
  const long long gid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gid >= static_cast<long long>(B) * D) return;
  const int sys = static_cast<int>(gid / D);
  const int g = static_cast<int>(gid % D);
  const int b = g / nb, i = g % nb;
  const size_t nn = static_cast<size_t>(nb) * nb;
  const T* Ms = M + static_cast<size_t>(sys) * K * 3 * nn + static_cast<size_t>(b) * 3 * nn;
  const T* xs = x + static_cast<size_t>(sys) * D;
  T out;
  if (mode == 1) {
    T sl = T(0), sr = T(0);
    if ((b % 2) == 0) {
      if (b > 0)
        for (int j = 0; j < nb; ++j) sl += -Ms[i * nb + j] * xs[(b - 1) * nb + j];
      if (b + 1 < K)
        for (int j = 0; j < nb; ++j) sr += -Ms[2 * nn + i * nb + j] * xs[(b + 1) * nb + j];
    }
    // E's diagonal block is zero: y = 0*x_b + left + right
    T sd = T(0);
    for (int j = 0; j < nb; ++j) sd += T(0) * xs[b * nb + j];
    out = (sd + sl) + sr;
  } else {
    T sd = T(0), sl = T(0), sr = T(0);
    for (int j = 0; j < nb; ++j) sd += Ms[nn + i * nb + j] * xs[b * nb + j];
    if (b > 0)
      for (int j = 0; j < nb; ++j) sl += Ms[i * nb + j] * xs[(b - 1) * nb + j];
    if (b + 1 < K)
      for (int j = 0; j < nb; ++j) sr += Ms[2 * nn + i * nb + j] * xs[(b + 1) * nb + j];
    out = b > 0 ? (sd + sl) : sd;
    if (b + 1 < K) out = out + sr;
  }
  y[gid] = out;
  if (acc) acc[gid] = add_to[gid] + out;
}

// stair_matrix (schur.cpp:84-94): even rows keep only the diagonal.
template <class T>
__global__ void k_stair_matrix(int K, int nb, const T* __restrict__ S, T* __restrict__ psi) {
  const size_t nn = static_cast<size_t>(nb) * nb;
  const size_t total = static_cast<size_t>(K) * 3 * nn;
  for (size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int row = static_cast<int>(idx / (3 * nn));
    const int slot = static_cast<int>((idx / nn) % 3);
    const bool keep = slot == 1 || (row % 2 == 1 && (slot == 0 || row + 1 < K));
    psi[idx] = keep ? S[idx] : T(0);
  }
}

// max_asymmetry / max_abs (block_tri.cpp:161-177): per-block partial maxima.
template <class T>
__global__ void k_blocktri_check(int K, int nb, const T* __restrict__ M, double* out2) {
  const size_t nn = static_cast<size_t>(nb) * nb;
  double asym = 0.0, mabs = 0.0;
  const size_t total = static_cast<size_t>(K) * nn;
  for (size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int row = static_cast<int>(idx / nn);
    const int e = static_cast<int>(idx % nn);
    const int i = e / nb, j = e % nb;
    const T* R = M + static_cast<size_t>(row) * 3 * nn;
    for (int s = 0; s < 3; ++s) mabs = fmax(mabs, fabs(static_cast<double>(R[s * nn + e])));
    asym = fmax(asym, fabs(static_cast<double>(R[nn + i * nb + j] - R[nn + j * nb + i])));
    if (row + 1 < K) {
      const T* Ln = M + static_cast<size_t>(row + 1) * 3 * nn;
      asym = fmax(asym, fabs(static_cast<double>(R[2 * nn + i * nb + j] - Ln[j * nb + i])));
    }
  }
  // block reduce (max is order independent)
  __shared__ double sa[32], sm[32];
  for (int o = 16; o > 0; o >>= 1) {
    asym = fmax(asym, __shfl_xor_sync(kFull, asym, o));
    mabs = fmax(mabs, __shfl_xor_sync(kFull, mabs, o));
  }
  if ((threadIdx.x & 31) == 0) {
    sa[threadIdx.x >> 5] = asym;
    sm[threadIdx.x >> 5] = mabs;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
      asym = fmax(asym, sa[w]);
      mabs = fmax(mabs, sm[w]);
    }
    // non-negative doubles order like their bit patterns
    atomicMax(reinterpret_cast<unsigned long long*>(out2), __double_as_longlong(asym));
    atomicMax(reinterpret_cast<unsigned long long*>(out2 + 1), __double_as_longlong(mabs));
  }
}

// BlockTriMatrix::cholesky_solve (block_tri.cpp:121-159): block Thomas, one
// warp per system (the recurrence is sequential in the block row); blockIdx.x
// is the system of a batch laid out [B][...] contiguously.
template <class T>
__global__ void k_block_cholesky(int K, int nb, const T* __restrict__ M, const T* __restrict__ rhs,
                                 T* __restrict__ x, T* __restrict__ factors, T* __restrict__ y,
                                 int* status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  if (threadIdx.x >= 32) return;
  const int n = nb, ld = tile_ld(nb);
  const size_t nn = static_cast<size_t>(n) * n;
  {
    const size_t sys = blockIdx.x, D = static_cast<size_t>(K) * n;
    M += sys * K * 3 * nn;
    rhs += sys * D;
    x += sys * D;
    y += sys * D;
    factors += sys * K * nn;
    status += sys;
  }
  T* base = reinterpret_cast<T*>(smem_raw);
  Tile<T> tF{base, ld}, tL{base + n * ld, ld}, tX{base + 2 * n * ld, ld}, tW{base + 3 * n * ld, ld};
  T* v = base + 4 * n * ld;
  T* w = v + 32;
  auto blk = [&](int r, int s) { return M + (static_cast<size_t>(r) * 3 + s) * nn; };
  for (int idx = lane; idx < K * n; idx += 32) y[idx] = rhs[idx];
  __syncwarp();
  tload(tW, blk(0, 1), n, n, lane);
  if (tcholesky(tW, n, lane) >= 0) {
    if (lane == 0) *status = 0;
    return;
  }
  tstore(factors, tW, n, n, lane);
  __syncwarp();
  for (int i = 1; i < K; ++i) {
    tload(tF, factors + (i - 1) * nn, n, n, lane);
    tload(tL, blk(i, 0), n, n, lane);
    // solved = F^-T F^-1 L_i'   (lane j: column j = L_i row j)
    if (lane < n) {
      const int j = lane;
      for (int r = 0; r < n; ++r) {
        T s = tL(j, r);
        for (int q = 0; q < r; ++q) s -= tF(r, q) * tX(q, j);
        tX(r, j) = s / tF(r, r);
      }
      for (int r = n - 1; r >= 0; --r) {
        T s = tX(r, j);
        for (int q = r + 1; q < n; ++q) s -= tF(q, r) * tX(q, j);
        tX(r, j) = s / tF(r, r);
      }
    }
    __syncwarp();
    // dhat = D_i - L_i * solved
    tload(tW, blk(i, 1), n, n, lane);
    if (lane < n) {
      const int j = lane;
      for (int r = 0; r < n; ++r) {
        T s = T(0);
        for (int q = 0; q < n; ++q) s += tL(r, q) * tX(q, j);
        tW(r, j) = tW(r, j) - s;
      }
    }
    __syncwarp();
    if (tcholesky(tW, n, lane) >= 0) {
      if (lane == 0) *status = i;
      return;
    }
    tstore(factors + i * nn, tW, n, n, lane);
    // y_i -= L_i * F_{i-1}^{-1} y_{i-1}
    if (lane < n) v[lane] = y[(i - 1) * n + lane];
    __syncwarp();
    tllt_solve_vec(tF, v, n, lane);
    if (lane < n) {
      T s = T(0);
      for (int q = 0; q < n; ++q) s += tL(lane, q) * v[q];
      y[i * n + lane] -= s;
    }
    __syncwarp();
  }
  // back substitution: x_i = F_i^{-1} (y_i - R_i x_{i+1})
  tload(tF, factors + (K - 1) * nn, n, n, lane);
  if (lane < n) v[lane] = y[(K - 1) * n + lane];
  __syncwarp();
  tllt_solve_vec(tF, v, n, lane);
  if (lane < n) x[(K - 1) * n + lane] = v[lane];
  __syncwarp();
  for (int i = K - 2; i >= 0; --i) {
    tload(tF, factors + i * nn, n, n, lane);
    tload(tL, blk(i, 2), n, n, lane);
    if (lane < n) w[lane] = x[(i + 1) * n + lane];
    __syncwarp();
    if (lane < n) {
      T s = T(0);
      for (int q = 0; q < n; ++q) s += tL(lane, q) * w[q];
      v[lane] = y[i * n + lane] - s;
    }
    __syncwarp();
    tllt_solve_vec(tF, v, n, lane);
    if (lane < n) x[i * n + lane] = v[lane];
    __syncwarp();
  }
  if (lane == 0) *status = -1;
}

// Block Thomas (BlockTriMatrix::cholesky_solve, block_tri.cpp:121-159) with the
// block dimension a compile-time constant: a half-warp per system (lane l < NB
// owns row l; lane NB carries the vector right-hand side through the block
// solves), the factor of Dhat_{i-1} and its reciprocal diagonal in shared
// memory, the next step's blocks prefetched into registers. Latency-bound by
// the 2 K dependent block factorisations / solves per system, so every system
// of a batch runs concurrently (28 per SM at c4). Same factorisation and block
// order as the reference; within-block association differs (column sweeps),
// so results agree to rounding (tests: 1e-10 of the oracle's cholesky_solve).
template <class T, int NB>
__global__ void __launch_bounds__(64, 7) k_block_thomas(int B, int K, const T* __restrict__ M,
                                                         const T* __restrict__ rhs, T* __restrict__ x,
                                                         T* __restrict__ factors, T* __restrict__ y,
                                                         int* __restrict__ status) {
  static_assert(NB >= 1 && NB < 16, "one half-warp lane per row plus the vector lane");
  constexpr int LD = NB + 1, NN = NB * NB, TS = NB * LD;
  __shared__ T sm[4][3 * TS + 2 * 16];
  const int hw = threadIdx.x >> 4, l = threadIdx.x & 15;
  // full-warp shuffles / syncs (a constant mask: no divergence handling); a
  // half-warp past the batch recomputes the last system and stores nothing
  constexpr unsigned mask = 0xffffffffu;
  const int sys_raw = blockIdx.x * 4 + hw;
  bool live = sys_raw < B;  // false also once this system failed (keeps stepping, stores nothing)
  const int sys = live ? sys_raw : B - 1;
  T* F = sm[hw];        // factor of Dhat_{i-1} (lower, row-major, ld LD)
  T* W = F + TS;        // Dhat_i, factorised in place (then swapped with F)
  T* X = W + TS;        // Dhat_{i-1}^-1 [L_i' | y_{i-1}]: column j = lane j
  T* rdF = X + TS;      // 1 / F(r, r)
  T* rdW = rdF + 16;    // 1 / W(r, r)
  const size_t D = static_cast<size_t>(K) * NB;
  M += static_cast<size_t>(sys) * K * 3 * NN;
  rhs += sys * D;
  x += sys * D;
  y += sys * D;
  factors += static_cast<size_t>(sys) * K * NN;
  status += sys;
  const bool rowc = l < NB;  // rows that compute (stores: rowc && live)
  const int lr = rowc ? l : NB - 1;
  auto blk = [&](int r, int s_) { return M + (static_cast<size_t>(r) * 3 + s_) * NN; };
  // In-place left-looking Cholesky of W (lane l: row l), Eigen's llt order;
  // returns the failing pivot (half-warp uniform) or -1.
  auto chol = [&](T* A, T* rd) -> int {
    int fail = -1;
#pragma unroll 1
    for (int k = 0; k < NB; ++k) {
      T s = A[lr * LD + k];
#pragma unroll 4
      for (int q = 0; q < k; ++q) s -= A[lr * LD + q] * A[k * LD + q];
      const T piv = __shfl_sync(mask, s, k, 16);
      if (piv <= T(0) && fail < 0) fail = k;  // x <= 0 fails, NaN passes (Eigen LLT)
      const T sq = sqrt(piv <= T(0) ? T(1) : piv);
      const T rk = T(1) / sq;  // one division per pivot
      __syncwarp(mask);
      if (rowc && l >= k) A[l * LD + k] = l == k ? sq : s * rk;
      if (l == k) rd[k] = rk;
      __syncwarp(mask);
    }
    return fail;
  };
  // F F' z = b for the calling lane's column b of X (in place, shared memory),
  // in axpy form: each step finalises one entry and updates the rest, so the
  // update chains are independent (no dot-product chains, few live loads)
  auto col_solve = [&](T* Z, const T* Fm, const T* rd) {
    T z[NB];
#pragma unroll
    for (int r = 0; r < NB; ++r) z[r] = Z[r * LD];
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      z[q] *= rd[q];
#pragma unroll
      for (int r = q + 1; r < NB; ++r) z[r] -= Fm[r * LD + q] * z[q];
    }
#pragma unroll
    for (int r = NB - 1; r >= 0; --r) {
      z[r] *= rd[r];
#pragma unroll
      for (int q = 0; q < r; ++q) z[q] -= Fm[r * LD + q] * z[r];
    }
#pragma unroll
    for (int r = 0; r < NB; ++r) Z[r * LD] = z[r];
  };
  // F F' v = b for one vector held as v (lane l: element l): column sweeps with
  // shuffles, the whole half-warp in step
  auto vec_solve = [&](T v, const T* Fm, const T* rd) -> T {
#pragma unroll
    for (int r = 0; r < NB; ++r) {
      const T zr = __shfl_sync(mask, v, r, 16) * rd[r];
      v = l == r ? zr : (l > r && rowc ? v - Fm[lr * LD + r] * zr : v);
    }
#pragma unroll
    for (int r = NB - 1; r >= 0; --r) {
      const T xr = __shfl_sync(mask, v, r, 16) * rd[r];
      v = l == r ? xr : (l < r ? v - Fm[r * LD + lr] * xr : v);
    }
    return v;
  };
  auto pf = [&](const T* p0) {  // L2 prefetch of row l of a block
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p0 + lr * NB));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p0 + lr * NB + NB - 1));
  };
  // block 0
  if (rowc)
    for (int j = 0; j < NB; ++j) F[l * LD + j] = blk(0, 1)[l * NB + j];
  T yv = rowc ? rhs[l] : T(0);
  if (K > 1) {
    pf(blk(1, 0));
    pf(blk(1, 1));
  }
  __syncwarp(mask);
  if (chol(F, rdF) >= 0) {
    if (l == 0 && live) *status = 0;
    live = false;
  }
  if (rowc && live) {
    for (int j = 0; j < NB; ++j) factors[l * NB + j] = F[l * LD + j];
    y[l] = yv;
  }
  for (int i = 1; i < K; ++i) {
    // X = Dhat_{i-1}^-1 [L_i' | y_{i-1}]: lane j < NB column j (row j of L_i),
    // lane NB the vector y_{i-1} (from the lanes holding it); L_i's rows also
    // parked in W (scratch until Dhat_i) so they are not live in registers
    // through the solves
    {
      const T* Li = blk(i, 0) + lr * NB;
#pragma unroll
      for (int q = 0; q < NB; ++q) {
        const T v = Li[q];
        const T yq = __shfl_sync(mask, yv, q, 16);
        if (rowc) {
          X[q * LD + l] = v;
          W[l * LD + q] = v;
        }
        if (l == NB) X[q * LD + NB] = yq;
      }
    }
    if (i + 1 < K) {
      pf(blk(i + 1, 0));
      pf(blk(i + 1, 1));
    }
    if (rowc || l == NB) col_solve(X + l, F, rdF);
    __syncwarp(mask);
    T Lrow[NB];  // row l of L_i
#pragma unroll
    for (int q = 0; q < NB; ++q) Lrow[q] = rowc ? W[l * LD + q] : T(0);
    // y_i = rhs_i - L_i X[:, NB]; Dhat_i = D_i - L_i X[:, :NB] (into W)
    T yi = rowc ? rhs[static_cast<size_t>(i) * NB + l] : T(0);
    {
      T sy = T(0);
#pragma unroll
      for (int q = 0; q < NB; ++q) sy += Lrow[q] * X[q * LD + NB];
      yi -= sy;
    }
    const T* Dr = blk(i, 1) + lr * NB;
#pragma unroll 2
    for (int j = 0; j < NB; ++j) {
      T s = T(0);
#pragma unroll
      for (int q = 0; q < NB; ++q) s += Lrow[q] * X[q * LD + j];
      if (rowc) W[l * LD + j] = Dr[j] - s;
    }
    __syncwarp(mask);
    if (chol(W, rdW) >= 0) {
      if (l == 0 && live) *status = i;
      live = false;
    }
    yv = yi;
    if (rowc && live) {
      T* Fo = factors + static_cast<size_t>(i) * NN;
      for (int j = 0; j < NB; ++j) Fo[l * NB + j] = W[l * LD + j];
      y[static_cast<size_t>(i) * NB + l] = yi;
    }
    {  // W becomes the factor of Dhat_i
      T* t = F;
      F = W;
      W = t;
      t = rdF;
      rdF = rdW;
      rdW = t;
    }
    __syncwarp(mask);
  }
  // back substitution: x_i = Dhat_i^-1 (y_i - R_i x_{i+1}); F holds Dhat_{K-1}
  T* xs = X;  // x_{i+1} for the R_i row products (shared by the half-warp)
  T xv = vec_solve(yv, F, rdF);  // lane l: element l of x_{K-1}
  for (int i = K - 2; i >= -1; --i) {
    if (rowc && live) x[static_cast<size_t>(i + 1) * NB + l] = xv;
    if (i < 0) break;
    __syncwarp(mask);
    if (i > 0) {  // the next step's factor and R rows into L2
      pf(factors + static_cast<size_t>(i - 1) * NN);
      pf(blk(i - 1, 2));
    }
    if (rowc && live) {
      xs[l] = xv;
      const T* Fi = factors + static_cast<size_t>(i) * NN;  // F <- factor i
      for (int j = 0; j < NB; ++j) F[l * LD + j] = Fi[l * NB + j];
      rdF[l] = T(1) / Fi[l * NB + l];
    }
    __syncwarp(mask);
    T v = T(0);
    if (rowc && live) {
      const T* Rb = blk(i, 2) + l * NB;
      T s = T(0);
#pragma unroll
      for (int q = 0; q < NB; ++q) s += Rb[q] * xs[q];
      v = y[static_cast<size_t>(i) * NB + l] - s;
    }
    __syncwarp(mask);
    xv = vec_solve(v, F, rdF);
  }
  if (l == 0 && live) *status = -1;
}

// ----------------------------------------------------------------- launchers
template <class T>
cudaError_t launch_build_schur(const FormParams<T>& p, cudaStream_t st) {
  const size_t per_warp = form_smem_per_warp<T>(p.n, p.m);
  int wpc = static_cast<int>(std::min<size_t>(8, std::max<size_t>(1, (96 * 1024) / per_warp)));
  const size_t smem = per_warp * wpc;
  if (smem > 48 * 1024)
    ensure_max_smem(k_build_schur<T>, smem);
  const long long warps = static_cast<long long>(p.B) * (p.N + 1);
  const long long grid = (warps + wpc - 1) / wpc;
  k_build_schur<T><<<static_cast<unsigned>(grid), 32 * wpc, smem, st>>>(p);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_build_precond(const PrecondParams<T>& p, cudaStream_t st) {
  const int ld = tile_ld(p.nb);
  const size_t per_warp = sizeof(T) * 4 * p.nb * ld;
  const int wpc = 4;
  const size_t smem = per_warp * wpc;
  if (smem > 48 * 1024)
    ensure_max_smem(k_build_precond<T>, smem);
  const long long warps = static_cast<long long>(p.B) * p.K;
  k_build_precond<T><<<static_cast<unsigned>((warps + wpc - 1) / wpc), 32 * wpc, smem, st>>>(p);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_blocktri_matvec(int B, int K, int nb, const T* M, const T* x, T* y, int mode,
                                   const T* add_to, T* acc, cudaStream_t st) {
  const long long total = static_cast<long long>(B) * K * nb;
  const int tpb = 256;
  k_blocktri_matvec<T><<<static_cast<unsigned>((total + tpb - 1) / tpb), tpb, 0, st>>>(
      B, K, nb, M, x, y, mode, add_to, acc);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_stair_matrix(int K, int nb, const T* S, T* psi, cudaStream_t st) {
  k_stair_matrix<T><<<148, 256, 0, st>>>(K, nb, S, psi);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_blocktri_check(int K, int nb, const T* M, double* out2, cudaStream_t st) {
  k_blocktri_check<T><<<148, 256, 0, st>>>(K, nb, M, out2);
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_block_cholesky(int B, int K, int nb, const T* M, const T* rhs, T* x, T* factors,
                                  T* y, int* status, cudaStream_t st) {
  if (nb == 14 && K >= 1 && !std::getenv("B2P_DIRECT_WARP")) {  // the c4 / c1 block dimension
    k_block_thomas<T, 14><<<(B + 3) / 4, 64, 0, st>>>(B, K, M, rhs, x, factors, y, status);
    return cudaGetLastError();
  }
  const int ld = tile_ld(nb);
  const size_t smem = sizeof(T) * (4 * nb * ld + 64);
  if (smem > 48 * 1024)
    ensure_max_smem(k_block_cholesky<T>, smem);
  k_block_cholesky<T><<<B, 32, smem, st>>>(K, nb, M, rhs, x, factors, y, status);
  return cudaGetLastError();
}

#define B2P_INST(T)                                                                            \
  template cudaError_t launch_build_schur<T>(const FormParams<T>&, cudaStream_t);              \
  template cudaError_t launch_build_precond<T>(const PrecondParams<T>&, cudaStream_t);         \
  template cudaError_t launch_blocktri_matvec<T>(int, int, int, const T*, const T*, T*, int,   \
                                                 const T*, T*, cudaStream_t);                  \
  template cudaError_t launch_stair_matrix<T>(int, int, const T*, T*, cudaStream_t);           \
  template cudaError_t launch_blocktri_check<T>(int, int, const T*, double*, cudaStream_t);    \
  template cudaError_t launch_block_cholesky<T>(int, int, int, const T*, const T*, T*, T*, T*,  \
                                                int*,                                         \
                                                cudaStream_t);
B2P_INST(double)
B2P_INST(float)
#undef B2P_INST

}  // namespace b2p
