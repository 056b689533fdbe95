// K1+K2+K3 fused for small state dimensions — one CTA per system, everything
// in shared memory. The shapes of the reference's SQP / NMPC callers
// (double integrator n=2 m=1, pendulum n=2 m=1, cart-pole n=4 m=1; any n, m <= 8)
// where the split path spends ~26 us forming a handful of 2x2 blocks and ~5 us
// per PCG iteration on generic runtime-n loops and ten barriers.
//
// Blocks are padded to compile-time sizes NP (n) and MP (m) in {1, 2, 4, 8}:
// Q, R pad with identity diagonals, A, B, q, r, e, x_s, x0 with zeros. The
// padded Cholesky / inverse act on the leading block exactly as on the
// unpadded one (pad rows do not couple), the padded entries of gamma, r, p,
// t, u, r~ and lambda stay exactly zero through every iteration (pad rows of
// D, theta^-1 are identity rows, of L zero), and every row product sums its
// n real terms first, then exact zeros — the same values as an n-term loop.
//
//   F1 (schur.cpp:15-23,49-51): one lane group (GW = max(NP, MP, 2) lanes) per knot: Q_k^-1, Q_k^-1 q_k,
//      R_k^-1, R_k^-1 r_k (Cholesky + triangular inverse in Eigen's LLT order,
//      g8_spd_inverse, which also flags the first non-PD pivot).
//   F2 (schur.cpp:53-78): one lane group per block row, lane l = row l:
//      AQ = A Q_k^-1, L_b = -AQ, BR = B R_k^-1,
//      theta = sym(AQ A' + BR B' + Q_{k+1}^-1), gamma_b = e_k - zeta,
//      theta_b^-1; row 0: D = Q_0^-1, theta^-1[0] = sym(Q_0) (the reference's).
//   P  (pcg.cpp:55-129): one thread per scalar row (strided), vectors in
//      shared memory, the stair family applied on the fly (t = theta^-1 r,
//      u = r - L t_{b-1} - L_{b+1}' t_{b+1}, r~ = theta^-1 u on corrected
//      rows), fixed-order block reductions.
#include "kernels.h"
#include "hw_dense.cuh"

namespace b2p {
namespace {

// CTA size: 128 threads when the padded system has <= 128 scalar rows (n <= 2
// at the NMPC horizons: fewer warps in every barrier and reduction, twice the
// CTAs per SM in batches), else 256
constexpr int kSmallThreadsLo = 128, kSmallThreadsHi = 256;
// lanes per block-row group: the padded block size (>= 2), so n <= 2 packs 128
// groups per CTA and a K = 33 horizon forms in one trip instead of two
template <int NP, int MP>
constexpr int group_width() {
  return (NP > MP ? NP : MP) < 2 ? 2 : (NP > MP ? NP : MP);
}

template <int NP, int MP, int TH>
struct SmallLayout {
  static constexpr int NN = NP * NP, MM = MP * MP;
  static constexpr int GW = group_width<NP, MP>(), kGroups = TH / GW;
  // per lane group: Lr, LiT, sym tile, rd (n-sized) + Lr, LiT, rd (m-sized)
  static constexpr int tile = 3 * NN + NP + 2 * MM + MP;
};

__device__ __forceinline__ unsigned long long small_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int TEAM>
__device__ __forceinline__ void team_sync() {
  if constexpr (TEAM == 32)
    __syncwarp();
  else
    __syncthreads();
}

// Fixed-order sum over the team: the warp xor tree leaves the bit-identical
// total in every lane; the CTA version combines the warp partials pairwise.
template <class T, int TEAM>
__device__ __forceinline__ T team_reduce(T v, T* red) {
  if constexpr (TEAM == 32) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  } else {
    return hwd::block_reduce<T, TEAM>(v, red);
  }
}

// P phase (pcg.cpp:55-129) on TEAM threads (the CTA; a one-warp team with
// shuffle-only reductions measured slower — rows per lane serialise). Vectors
// live in U (the dead formation scratch).
template <class T, int NP, int TEAM>
__device__ int small_pcg(const FusedParams<T>& p, int sys, int n, int K, const T* sD,
                          const T* sL, const T* sTi, const T* sG, T* U) {
  constexpr int NN = NP * NP;
  const int tid = threadIdx.x;
  const int KP = K * NP;
  T* vlam = U;
  T* vr = vlam + KP;
  T* vrt = vr + KP;
  T* vp = vrt + KP;
  T* vsp = vp + KP;
  T* vt = vsp + KP;
  T* vu = vt + KP;
  T* vbest = vu + KP;
  T* red = vbest + KP;
  // ================================================================ P
  // (formation scratch is dead: the vectors alias it)
  for (int i = tid; i < KP; i += TEAM) {
    const int b = i / NP, c = i % NP;
    vlam[i] = (p.lambda0 && c < n) ? p.lambda0[size_t(sys) * K * n + b * n + c] : T(0);
  }
  team_sync<TEAM>();
  // y_row = ((D x_b + L x_{b-1}) + R x_{b+1}), R_b = L_{b+1}' (block_tri.cpp:82-92)
  auto srow = [&](const T* x, int i) {
    const int b = i / NP, c = i % NP;
    const T* D = sD + size_t(b) * NN + c * NP;
    const T* xb = x + b * NP;
    T sd = T(0);
#pragma unroll
    for (int j = 0; j < NP; ++j) sd += D[j] * xb[j];
    T out = sd;
    if (b > 0) {
      const T* Lr = sL + size_t(b) * NN + c * NP;
      T sl = T(0);
#pragma unroll
      for (int j = 0; j < NP; ++j) sl += Lr[j] * xb[j - NP];
      out += sl;
    }
    if (b + 1 < K) {
      const T* Lc = sL + size_t(b + 1) * NN + c;  // column c of L_{b+1}
      T sr = T(0);
#pragma unroll
      for (int j = 0; j < NP; ++j) sr += Lc[j * NP] * xb[NP + j];
      out += sr;
    }
    return out;
  };
  auto trow = [&](const T* x, int i) {  // (theta_b^-1 x_b)_c
    const int b = i / NP, c = i % NP;
    const T* Ti = sTi + size_t(b) * NN + c * NP;
    const T* xb = x + b * NP;
    T s = T(0);
#pragma unroll
    for (int j = 0; j < NP; ++j) s += Ti[j] * xb[j];
    return s;
  };
  // r~ = Phi^-1 r for every kind (schur.cpp:175-194) on the own rows. A block's
  // NP rows belong to consecutive threads of one warp (NP | 32), so the
  // same-block products (theta^-1 r, theta^-1 u) only need __syncwarp; only the
  // neighbour-block product (u) needs the team barrier. Expects r visible to
  // the warp; leaves r~ valid on the own rows.
  auto precondition = [&]() {
    if (p.kind == kIdentity) {
      for (int i = tid; i < KP; i += TEAM) vrt[i] = vr[i];
      return;
    }
    for (int i = tid; i < KP; i += TEAM) vt[i] = trow(vr, i);
    if (p.kind == kJacobi) {
      for (int i = tid; i < KP; i += TEAM) vrt[i] = vt[i];
      return;
    }
    team_sync<TEAM>();
    for (int i = tid; i < KP; i += TEAM) {
      const int b = i / NP, c = i % NP;
      T v = vr[i];
      if (b > 0) {
        const T* Lr = sL + size_t(b) * NN + c * NP;
        T sl = T(0);
#pragma unroll
        for (int j = 0; j < NP; ++j) sl += Lr[j] * vt[(b - 1) * NP + j];
        v -= sl;
      }
      if (b + 1 < K) {
        const T* Lc = sL + size_t(b + 1) * NN + c;
        T sr = T(0);
#pragma unroll
        for (int j = 0; j < NP; ++j) sr += Lc[j * NP] * vt[(b + 1) * NP + j];
        v -= sr;
      }
      vu[i] = v;
    }
    __syncwarp();
    for (int i = tid; i < KP; i += TEAM) {
      const int b = i / NP;
      const bool corr = (p.kind == kSymStair) || (b & 1);
      vrt[i] = corr ? trow(vu, i) : vt[i];
    }
  };

  // r = gamma - S lambda0 (pcg.cpp:62)
  for (int i = tid; i < KP; i += TEAM)
    vr[i] = p.lambda0 ? sG[i] - srow(vlam, i) : sG[i];
  team_sync<TEAM>();
  precondition();
  T eta_part = T(0);
  for (int i = tid; i < KP; i += TEAM) {
    vp[i] = vrt[i];
    vbest[i] = vlam[i];
    eta_part += vr[i] * vrt[i];
  }
  T eta = team_reduce<T, TEAM>(eta_part, red);

  int code = kOk, which = kWhichNone, err_iter = -1, iterations = 0, converged = 0;
  double exit_eta = static_cast<double>(eta), value = 0.0;
  T best_eta = eta;
  double* trace = p.trace ? p.trace + size_t(sys) * p.trace_cap : nullptr;
  if (!is_finite(eta)) {
    code = kRuntime;
    which = kWhichInitNonFinite;
  } else if (static_cast<double>(eta) < p.epsilon) {
    converged = 1;
  } else {
    team_sync<TEAM>();
    for (int it = 1; it <= p.max_iter; ++it) {
      T up = T(0);
      for (int i = tid; i < KP; i += TEAM) {
        const T y = srow(vp, i);
        vsp[i] = y;
        up += vp[i] * y;
      }
      const T ups = team_reduce<T, TEAM>(up, red + 32);
      if (!is_finite(ups)) {
        code = kRuntime;
        which = kWhichUpsNonFinite;
        err_iter = it;
        break;
      }
      if (ups <= T(0)) {
        code = kBreakdown;
        which = kWhichBreakdown;
        err_iter = it;
        value = static_cast<double>(ups);
        break;
      }
      const T alpha = eta / ups;
      for (int i = tid; i < KP; i += TEAM) {
        vr[i] -= alpha * vsp[i];
        vlam[i] += alpha * vp[i];
      }
      __syncwarp();
      precondition();
      T ep = T(0);
      for (int i = tid; i < KP; i += TEAM) ep += vr[i] * vrt[i];
      const T eta_p = team_reduce<T, TEAM>(ep, red);
      if (!is_finite(eta_p)) {
        code = kRuntime;
        which = kWhichEtaNonFinite;
        err_iter = it;
        break;
      }
      if (trace && tid == 0) trace[it - 1] = static_cast<double>(eta_p);
      if (eta_p < best_eta) {
        best_eta = eta_p;
        for (int i = tid; i < KP; i += TEAM) vbest[i] = vlam[i];
      }
      iterations = it;
      exit_eta = static_cast<double>(eta_p);
      if (static_cast<double>(eta_p) < p.epsilon) {
        converged = 1;
        break;
      }
      if (it == p.max_iter) break;
      const T beta = eta_p / eta;
      for (int i = tid; i < KP; i += TEAM) vp[i] = vrt[i] + beta * vp[i];
      eta = eta_p;
      team_sync<TEAM>();
    }
  }
  if (code == kOk) {
    const T* src = converged ? vlam : vbest;
    for (int i = tid; i < KP; i += TEAM) {
      const int b = i / NP, c = i % NP;
      if (c < n) p.lambda_out[size_t(sys) * K * n + b * n + c] = src[i];
    }
  }
  if (tid == 0) {
    SysOut o;
    o.code = code;
    o.knot = -1;
    o.which = which;
    o.iteration = err_iter;
    o.iterations = iterations;
    o.converged = converged;
    o.exit_eta = exit_eta;
    o.value = value;
    o.max_drift = 0.0;
    o.trace_len = (trace && code == kOk) ? iterations : 0;
    o._pad = 0;
    p.out[sys] = o;
  }
  return code;
}

// The PPCG finish (reconstruct_primal, kkt.cpp:153-181) on
// the formation's resident Q_k^-1 / R_k^-1 and the solve's lambda: one lane
// group per knot, lane i = row i,
//   dx_k = Q_k^-1 (-((q_k + lambda_k) - A_k' lambda_{k+1})),
//   du_k = R_k^-1 (-(r_k - B_k' lambda_{k+1})),   dx_N = Q_N^-1 (-(q_N + lambda_N)).
// The right-hand sides are formed in the reference's association; the solve is
// the explicit inverse the formation already holds (the reference factors with
// LDLT: the same solution to rounding).
template <class T, int NP, int MP, int TH>
__device__ void small_finish(const FusedParams<T>& p, int sys, int n, int m, int K,
                             const T* sQi, const T* sRi, T* W) {
  constexpr int GW = group_width<NP, MP>(), kGroups = TH / GW;
  constexpr int NN = NP * NP, MM = MP * MP;
  const int N = K - 1, tid = threadIdx.x, g = tid / GW, l = tid % GW;
  const T* lam = p.lambda_out + size_t(sys) * K * n;
  const T* q = p.q + size_t(sys) * K * n;
  const T* r = p.r + size_t(sys) * N * m;
  const T* A = p.A + size_t(sys) * N * n * n;
  const T* Bm = p.Bm + size_t(sys) * N * n * m;
  T* dz = p.dz_out + size_t(sys) * (size_t(K) * n + size_t(N) * m);
  T* wx = W + size_t(g) * (NP + MP);  // the group's right-hand sides
  T* wu = wx + NP;
  const int kTrips = (K + kGroups - 1) / kGroups;
#pragma unroll 1
  for (int t = 0; t < kTrips; ++t) {
    const int k = g + t * kGroups;
    const bool kv = k < K;
    if (kv && l < NP) {  // pad rows: exact zeros
      T rx = T(0);
      if (l < n) {
        T at = T(0);
        if (k < N)  // (A_k' lambda_{k+1})_l
          for (int j = 0; j < n; ++j) at += A[size_t(k) * n * n + j * n + l] * lam[(k + 1) * n + j];
        rx = k < N ? -((q[k * n + l] + lam[k * n + l]) - at) : -(q[k * n + l] + lam[k * n + l]);
      }
      wx[l] = rx;
    }
    if (kv && l < MP) {
      T ru = T(0);
      if (k < N && l < m) {
        T bt = T(0);
        for (int j = 0; j < n; ++j) bt += Bm[size_t(k) * n * m + j * m + l] * lam[(k + 1) * n + j];
        ru = -(r[k * m + l] - bt);
      }
      wu[l] = ru;
    }
    __syncwarp();
    if (kv && l < n) {
      T s = T(0);
#pragma unroll
      for (int j = 0; j < NP; ++j) s += sQi[size_t(k) * NN + l * NP + j] * wx[j];
      dz[size_t(k) * (n + m) + l] = s;
    }
    if (kv && k < N && l < m) {
      T s = T(0);
#pragma unroll
      for (int j = 0; j < MP; ++j) s += sRi[size_t(k) * MM + l * MP + j] * wu[j];
      dz[size_t(k) * (n + m) + n + l] = s;
    }
    __syncwarp();
  }
}

// BATCH = true: the throughput build for batches (registers capped so 4 / 3 CTAs
// fit an SM at n <= 2 / 4: 11.6 -> 15.6 M systems/s at n = 2); BATCH = false:
// the latency build for single solves (uncapped registers: 30.6 vs 34 us).
template <class T, int NP, int MP, bool BATCH, int kSmallThreads>
__global__ void __launch_bounds__(kSmallThreads, (!BATCH ? 1 : (NP <= 2 ? 4 : (NP <= 4 ? 3 : 1))))
    k_fused_small(FusedParams<T> p, int n, int m,
                                                               int staged) {
  using L = SmallLayout<NP, MP, kSmallThreads>;
  constexpr int NN = L::NN, MM = L::MM;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);
  const int K = p.K, N = K - 1;
  const int tid = threadIdx.x;
  constexpr int GW = L::GW, kGroups = L::kGroups;
  const int g = tid / GW, l = tid % GW;
  const int lr = l < NP ? l : NP - 1;  // clamped row for duplicate lanes
  // persistent
  T* sD = smem;
  T* sL = sD + size_t(K) * NN;
  T* sTi = sL + size_t(K) * NN;
  T* sG = sTi + size_t(K) * NN;
  // with the fused finish (dz_out) Q_k^-1 and R_k^-1 stay resident past the PCG
  const bool keep = p.dz_out != nullptr;
  const size_t NR = size_t(N > 0 ? N : 1);
  T* sKeep = sG + size_t(K) * NP;
  T* U = sKeep + (keep ? size_t(K) * NN + NR * MM : 0);
  // formation scratch
  T* sQi = keep ? sKeep : U;                             // [K][NP][NP]
  T* sRi = keep ? sKeep + size_t(K) * NN : U + size_t(K) * (NN + NP);  // [N][MP][MP]
  T* sqq = keep ? U : sQi + size_t(K) * NN;              // [K][NP]
  T* srr = keep ? sqq + size_t(K) * NP : sRi + NR * MM;  // [N][MP]
  T* tiles = srr + NR * MP;
  T* tLr = tiles + size_t(g) * L::tile;
  T* tLi = tLr + NN;
  T* tSym = tLi + NN;
  T* trd = tSym + NN;
  T* tLr2 = trd + NP;  // m-sized inverse tiles
  T* tLi2 = tLr2 + MM;
  T* trd2 = tLi2 + MM;
  T* stg = tiles + size_t(kGroups) * L::tile;  // staged knot data (unpadded)
  __shared__ int s_err;

  for (int sys = blockIdx.x; sys < p.B; sys += gridDim.x) {
    __syncthreads();  // previous system done with shared memory
    unsigned long long* tm = (p.timing && tid == 0) ? p.timing + size_t(sys) * 16 : nullptr;
    if (tm) tm[0] = small_gtimer();
    // Stage the system's knot data (the b2p_kkt layout, unpadded) in shared
    // memory with coalesced cp.async copies, all issued before any is consumed: the
    // formation then reads operands at shared-memory latency instead of one
    // dependent L2/HBM round trip per product.
    const size_t cnt[9] = {size_t(K) * n * n, size_t(K) * n,     size_t(N) * m * m,
                           size_t(N) * m,     size_t(N) * n * n, size_t(N) * n * m,
                           size_t(N) * n,     size_t(n),         size_t(n)};
    const T* gsrc[9] = {p.Q, p.q, p.R, p.r, p.A, p.Bm, p.e, p.x_s, p.x0};
    const T* st[9];
    {
      T* d = stg;
#pragma unroll 1
      for (int a = 0; a < 9; ++a) {
        const T* src = gsrc[a] + size_t(sys) * cnt[a];
        if (staged) {
          // asynchronous 8-byte copies: every array's loads are in flight at
          // once (one memory latency for the whole system, not one per array)
          const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(d));
          for (size_t i = tid; i < cnt[a]; i += kSmallThreads)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst + 8u * unsigned(i)),
                         "l"(src + i)
                         : "memory");
          st[a] = d;
          d += cnt[a];
        } else {
          st[a] = src;  // too long a horizon to stage: read through L1/L2
        }
      }
    }
    const T *Qs = st[0], *qs = st[1], *Rs = st[2], *rs = st[3], *As = st[4], *Bs = st[5],
            *es = st[6], *xs = st[7], *x0 = st[8];
    if (tid == 0) s_err = 0x7fffffff;
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    if (tm) tm[1] = small_gtimer();
    int fkey = 0x7fffffff;

    // ================================================================ F1
    // Every lane of every warp runs the same trip count (clamped duplicates
    // store nothing): the group inverses use full-warp shuffles.
    const int kTrips = (K + kGroups - 1) / kGroups;
#pragma unroll 1
    for (int t = 0; t < kTrips; ++t) {
      const int k0 = g + t * kGroups;
      const bool kv = k0 < K;
      const int k = kv ? k0 : K - 1;
      T a[NP], x[NP];
#pragma unroll
      for (int j = 0; j < NP; ++j)
        a[j] = (lr < n && j < n) ? Qs[size_t(k) * n * n + lr * n + j]
                                 : (lr == j ? T(1) : T(0));
      const int f = hwd::g8_spd_inverse<T, NP, GW>(a, tLr, tLi, trd, l, x);
      if (kv && f >= 0) fkey = min(fkey, k == 0 ? 0 : 4 * k + 2);
      if (kv && l < NP) {
        T qq = T(0);
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          sQi[size_t(k) * NN + l * NP + i] = x[i];
          qq += x[i] * (i < n ? qs[size_t(k) * n + i] : T(0));
        }
        sqq[size_t(k) * NP + l] = qq;
      }
      if (N > 0) {  // R_k^-1 (knots k < N), same trip structure
        const bool rv = kv && k < N;
        const int kr = k < N ? k : N - 1;
        const int lm = l < MP ? l : MP - 1;
        T ra[MP], y[MP];
#pragma unroll
        for (int j = 0; j < MP; ++j)
          ra[j] = (lm < m && j < m) ? Rs[size_t(kr) * m * m + lm * m + j]
                                    : (lm == j ? T(1) : T(0));
        const int fr = hwd::g8_spd_inverse<T, MP, GW>(ra, tLr2, tLi2, trd2, l, y);
        if (rv && fr >= 0) fkey = min(fkey, 4 * (kr + 1) + 1);
        if (rv && l < MP) {
          T rr = T(0);
#pragma unroll
          for (int i = 0; i < MP; ++i) {
            sRi[size_t(kr) * MM + l * MP + i] = y[i];
            rr += y[i] * (i < m ? rs[size_t(kr) * m + i] : T(0));
          }
          srr[size_t(kr) * MP + l] = rr;
        }
      }
    }
    __syncthreads();
    if (tm) tm[2] = small_gtimer();

    // ================================================================ F2
#pragma unroll 1
    for (int t = 0; t < kTrips; ++t) {
      const int b0 = g + t * kGroups;
      const bool wr = b0 < K && l < NP;
      if (b0 == 0) {  // schur.cpp:53-57
        if (l < NP) {
#pragma unroll
          for (int i = 0; i < NP; ++i) {
            sD[l * NP + i] = sQi[l * NP + i];
            sL[l * NP + i] = T(0);
            sTi[l * NP + i] = (l < n && i < n) ? T(0.5) * (Qs[l * n + i] + Qs[i * n + l])
                                               : (l == i ? T(1) : T(0));
          }
          sG[l] = l < n ? -((xs[l] - x0[l]) + sqq[l]) : T(0);
        }
      }
      // rows outside [1, K) run row 1 (or row 0's data when K == 1) and store nothing
      const int b = (b0 >= 1 && b0 < K) ? b0 : (K > 1 ? 1 : 0);
      const bool general = K > 1;
      const bool store = wr && b0 >= 1;
      if (general) {
        const int k = b - 1;
        const T* Ak = As + size_t(k) * n * n;
        const T* Bk = Bs + size_t(k) * n * m;
        T arow[NP], brow[MP], aq[NP], br[MP], th[NP];
#pragma unroll
        for (int j = 0; j < NP; ++j) arow[j] = (lr < n && j < n) ? Ak[lr * n + j] : T(0);
#pragma unroll
        for (int j = 0; j < MP; ++j) brow[j] = (lr < n && j < m) ? Bk[lr * m + j] : T(0);
        // AQ row l (schur.cpp:65), L_b = -AQ (:68)
#pragma unroll
        for (int j = 0; j < NP; ++j) {
          T s = T(0);
#pragma unroll
          for (int q = 0; q < NP; ++q) s += arow[q] * sQi[size_t(k) * NN + q * NP + j];
          aq[j] = s;
        }
#pragma unroll
        for (int j = 0; j < MP; ++j) {
          T s = T(0);
#pragma unroll
          for (int q = 0; q < MP; ++q) s += brow[q] * sRi[size_t(k) * MM + q * MP + j];
          br[j] = s;
        }
        // theta row l = (AQ A')(l,:) + (BR B')(l,:) + Q_{k+1}^-1(l,:)  (schur.cpp:65-66)
#pragma unroll
        for (int j = 0; j < NP; ++j) {
          T s1 = T(0), s2 = T(0);
#pragma unroll
          for (int q = 0; q < NP; ++q) s1 += aq[q] * ((j < n && q < n) ? Ak[j * n + q] : T(0));
#pragma unroll
          for (int q = 0; q < MP; ++q) s2 += br[q] * ((j < n && q < m) ? Bk[j * m + q] : T(0));
          th[j] = (s1 + s2) + sQi[size_t(b) * NN + lr * NP + j];
        }
        // zeta, gamma_b = -(c_b + zeta), c_b = -e_k  (schur.cpp:69-77)
        T aqq = T(0), brr = T(0);
#pragma unroll
        for (int q = 0; q < NP; ++q) aqq += arow[q] * sqq[size_t(k) * NP + q];
#pragma unroll
        for (int q = 0; q < MP; ++q) brr += brow[q] * srr[size_t(k) * MP + q];
        const T zeta = (-aqq - brr) + sqq[size_t(b) * NP + lr];
        if (store) {
          sG[size_t(b) * NP + l] = l < n ? -(-es[size_t(k) * n + l] + zeta) : T(0);
#pragma unroll
          for (int j = 0; j < NP; ++j) sL[size_t(b) * NN + l * NP + j] = -aq[j];
        }
        // sym (schur.cpp:67) through the group's tile
        if (l < NP) {
#pragma unroll
          for (int j = 0; j < NP; ++j) tSym[l * NP + j] = th[j];
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < NP; ++j) th[j] = T(0.5) * (th[j] + tSym[j * NP + lr]);
        __syncwarp();
        if (store) {
#pragma unroll
          for (int j = 0; j < NP; ++j) sD[size_t(b) * NN + l * NP + j] = th[j];
        }
        T x[NP];
        const int f = hwd::g8_spd_inverse<T, NP, GW>(th, tLr, tLi, trd, l, x);
        if (store && f >= 0) fkey = min(fkey, 4 * b + 3);
        if (store) {
#pragma unroll
          for (int j = 0; j < NP; ++j) sTi[size_t(b) * NN + l * NP + j] = x[j];
        }
      }
    }
    if (l == 0 && fkey != 0x7fffffff) atomicMin(&s_err, fkey);
    __syncthreads();
    if (s_err != 0x7fffffff) {
      if (tid == 0) {
        p.errkey[sys] = s_err;
        SysOut o{};
        o.code = kRuntime;
        o.which = kWhichNone;
        o.iteration = -1;
        p.out[sys] = o;
      }
      continue;
    }
    if (tid == 0 && p.errkey) p.errkey[sys] = 0x7f7f7f7f;

    if (p.form_only) {
      // build_schur only: S in the reference layout [K][left|diag|right][n][n]
      // (row 0 left and row K-1 right zero, R_b = L_{b+1}'), theta^-1, gamma
      // — the unpadded leading blocks of the padded shared-memory arrays
      const int nn = n * n;
      T* So = p.S_out + size_t(sys) * K * 3 * nn;
      for (int i = tid; i < K * 3 * nn; i += kSmallThreads) {
        const int b = i / (3 * nn), rem = i % (3 * nn), slot = rem / nn, e = rem % nn;
        const int r = e / n, c = e % n;
        T v = T(0);
        if (slot == 0)
          v = b > 0 ? sL[size_t(b) * NN + r * NP + c] : T(0);
        else if (slot == 1)
          v = sD[size_t(b) * NN + r * NP + c];
        else
          v = b + 1 < K ? sL[size_t(b + 1) * NN + c * NP + r] : T(0);
        So[i] = v;
      }
      for (int i = tid; i < K * nn; i += kSmallThreads) {
        const int b = i / nn, e = i % nn, r = e / n, c = e % n;
        p.theta_out[size_t(sys) * K * nn + i] = sTi[size_t(b) * NN + r * NP + c];
      }
      for (int i = tid; i < K * n; i += kSmallThreads)
        p.gamma_out[size_t(sys) * K * n + i] = sG[(i / n) * NP + i % n];
      continue;
    }

    // ================================================================ P
    if (tm) tm[3] = small_gtimer();
    const int code = small_pcg<T, NP, kSmallThreads>(p, sys, n, K, sD, sL, sTi, sG, U);
    if (keep && code == kOk) {
      __syncthreads();  // lambda (global) and the PCG vectors (U) complete
      small_finish<T, NP, MP, kSmallThreads>(p, sys, n, m, K, sQi, sRi, U);
    }
    if (tm) tm[4] = small_gtimer();
  }
}

int pad_pow2(int v) { return v <= 1 ? 1 : v <= 2 ? 2 : v <= 4 ? 4 : v <= 8 ? 8 : 0; }

// Shared memory of one CTA: persistent D, L, theta^-1 [K][NP][NP] + gamma
// [K][NP], then the formation scratch (Q^-1, Q^-1 q, R^-1, R^-1 r, the
// per-group inverse tiles and, when `staged`, the system's knot data) aliased
// by the PCG vectors.
size_t small_bytes_rt(int NP, int MP, int K, bool staged, int threads, bool keep = false) {
  const size_t NN = size_t(NP) * NP, MM = size_t(MP) * MP, N = K > 1 ? K - 1 : 0;
  const size_t kept = keep ? size_t(K) * NN + std::max<size_t>(N, 1) * MM : 0;
  const int GW = std::max(2, std::max(NP, MP));
  const size_t tile = 3 * NN + NP + 2 * MM + MP;
  const size_t stg =
      staged ? size_t(K) * (NN + NP) + N * (MM + MP + NN + NP * MP + NP) + 2 * NP : 0;
  const size_t form_t = size_t(K) * (NN + NP) + std::max<size_t>(N, 1) * (MM + MP) +
                        size_t(threads / GW) * tile + stg - (keep ? kept : 0);
  const size_t fin = keep ? size_t(threads / GW) * (NP + MP) : 0;
  const size_t pcg = std::max(size_t(8) * K * NP + 64, fin);
  return sizeof(double) * (size_t(K) * (3 * NN + NP) + kept + std::max(form_t, pcg));
}

int small_threads(int NP, int K) { return K * NP <= 128 ? kSmallThreadsLo : kSmallThreadsHi; }

constexpr size_t kSmallSmemCap = 227 * 1024 - 1024;

template <class T, int NP, int MP, int TH>
cudaError_t go_small_th(const FusedParams<T>& p, int n, int m, int grid, cudaStream_t st) {
  const bool keep = p.dz_out != nullptr;
  const bool staged = small_bytes_rt(NP, MP, p.K, true, TH, keep) <= kSmallSmemCap;
  const size_t smem = small_bytes_rt(NP, MP, p.K, staged, TH, keep);
  auto kern = p.B > 1 ? k_fused_small<T, NP, MP, true, TH> : k_fused_small<T, NP, MP, false, TH>;
  cudaError_t e = ensure_max_smem(kern, smem);
  if (e != cudaSuccess) return e;
  // persistent CTAs: as many as fit co-resident (`grid` = SM count on entry)
  int per_sm = 1;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TH, smem);
  if (e != cudaSuccess) return e;
  grid = std::max(1, std::min(p.B, grid * std::max(1, per_sm)));
  kern<<<grid, TH, smem, st>>>(p, n, m, staged ? 1 : 0);
  return cudaGetLastError();
}

template <class T, int NP, int MP>
cudaError_t go_small(const FusedParams<T>& p, int n, int m, int grid, cudaStream_t st) {
  if (small_threads(NP, p.K) == kSmallThreadsLo)
    return go_small_th<T, NP, MP, kSmallThreadsLo>(p, n, m, grid, st);
  return go_small_th<T, NP, MP, kSmallThreadsHi>(p, n, m, grid, st);
}

template <class T, int NP>
cudaError_t go_small_m(const FusedParams<T>& p, int n, int m, int grid, cudaStream_t st) {
  switch (pad_pow2(m)) {
    case 1: return go_small<T, NP, 1>(p, n, m, grid, st);
    case 2: return go_small<T, NP, 2>(p, n, m, grid, st);
    case 4: return go_small<T, NP, 4>(p, n, m, grid, st);
    case 8: return go_small<T, NP, 8>(p, n, m, grid, st);
  }
  return cudaErrorNotSupported;
}

}  // namespace

template <class T>
bool small_supported(int K, int n, int m, int kind) {
  if (sizeof(T) != 8 || kind == kPoly) return false;
  if (n < 1 || n > 8 || m < 1 || m > 8 || K < 1) return false;
  const int NP = pad_pow2(n), MP = pad_pow2(m);
  return small_bytes_rt(NP, MP, K, false, small_threads(NP, K)) <= kSmallSmemCap;
}

template <class T>
bool small_supported_dz(int K, int n, int m, int kind) {
  if (!small_supported<T>(K, n, m, kind)) return false;
  const int NP = pad_pow2(n), MP = pad_pow2(m);
  return small_bytes_rt(NP, MP, K, false, small_threads(NP, K), true) <= kSmallSmemCap;
}

template <class T>
cudaError_t launch_small(const FusedParams<T>& p, int n, int m, int grid, cudaStream_t st) {
  if constexpr (sizeof(T) == 8) {
    switch (pad_pow2(n)) {
      case 1: return go_small_m<T, 1>(p, n, m, grid, st);
      case 2: return go_small_m<T, 2>(p, n, m, grid, st);
      case 4: return go_small_m<T, 4>(p, n, m, grid, st);
      case 8: return go_small_m<T, 8>(p, n, m, grid, st);
    }
  }
  return cudaErrorNotSupported;
}

template bool small_supported<double>(int, int, int, int);
template bool small_supported<float>(int, int, int, int);
template bool small_supported_dz<double>(int, int, int, int);
template bool small_supported_dz<float>(int, int, int, int);
template cudaError_t launch_small<double>(const FusedParams<double>&, int, int, int, cudaStream_t);
template cudaError_t launch_small<float>(const FusedParams<float>&, int, int, int, cudaStream_t);

}  // namespace b2p
