// K3 — persistent PCG on the block-tridiagonal Schur complement (sm_100a).
//
// Replaces pcg_solve (proj/src/pcg.cpp:55-129) and pcg_solve_block_parallel
// (pcg.cpp:157-362) with one launch per solve (or per batch of solves):
//   * a system is owned by G CTAs (G = 1, a thread-block cluster of G, or a
//     cooperative grid); each CTA owns a contiguous block-row range
//     [lo, hi) and keeps its matrix rows resident in shared memory;
//   * the two scalar reductions per iteration (upsilon = p'Sp and
//     eta' = r'r~) are warp-shuffle trees + a fixed-order CTA combine + a
//     fixed-order sum of per-CTA slots, so every CTA holds bit-identical
//     scalars and results are reproducible run to run (the GPU analog of
//     deterministic_reductions, pcg.hpp:20-22);
//   * the halo exchanges of the reference's 6-barrier loop are
//     removed by redundant halo computation: a CTA recomputes Sp, r and r~
//     for a few neighbour rows, so each iteration needs exactly two
//     inter-CTA synchronisations (the two reductions). p's halo is
//     refreshed from a global exchange buffer right after the first one.
// Operators:
//   kModeExplicit — S and a materialised Phi^-1 (the drop-in pcg_solve API);
//   kModeFused    — S and theta^-1 only; Phi^-1 r is applied on the fly:
//     stair (odd rows) / symmetric stair (all rows):
//       r~_i = theta_i^-1 (r_i - L_i t_{i-1} - R_i t_{i+1}),  t_j = theta_j^-1 r_j
//     which is the reference's materialised -theta_i^-1 L_i theta_{i-1}^-1
//     blocks (schur.cpp:109-142) re-associated; the symmetric-stair mirror of
//     the odd rows' blocks is exactly this formula on the even rows because S
//     and theta^-1 are bitwise symmetric (schur.cpp:22,67,74).
#include <cooperative_groups.h>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace b2p {

__host__ __device__ __forceinline__ int halo_of(int kind, int order) {
  return 3 + 2 * (kind == kPoly ? order : 0);
}
int pcg_halo(int kind, int order) { return halo_of(kind, order); }

__host__ __device__ __forceinline__ int num_vecs(int kind) { return kind == kPoly ? 8 : 6; }

template <class T>
size_t pcg_smem_bytes(const PcgParams<T>& p) {
  const int H = halo_of(p.kind, p.order);
  const size_t nn = static_cast<size_t>(p.nb) * p.nb;
  const size_t wrows = std::min(p.K, p.rows_per + 2 * H);
  size_t bytes = sizeof(T) * (num_vecs(p.kind) * wrows * p.nb + 64);
  if (p.stage) {
    const size_t srows = std::min(p.K, p.rows_per + 2 * (H - 1));
    size_t per_row = 3 * nn;  // S
    if (p.mode == kModeFused) {
      if (p.kind != kIdentity) per_row += nn;  // theta^-1
    } else if (p.kind != kIdentity) {
      per_row += 3 * nn;  // Phi
    }
    bytes += sizeof(T) * srows * per_row;
  }
  return bytes;
}

namespace {

// Grid barrier for the cooperative launch: one atomic arrive per CTA on a
// monotonic counter (zeroed before the launch) and an acquire-load spin by
// thread 0; bar.sync around it extends the ordering to the whole CTA.
// (cooperative_groups' grid.sync measured ~30 us per barrier at 128 CTAs.)
__device__ __forceinline__ void grid_barrier(unsigned* ctr, unsigned& target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    target += gridDim.x;
    __threadfence();
    atomicAdd(ctr, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

template <int SYNC>
__device__ __forceinline__ void gsync(unsigned* ctr, unsigned& target) {
  if constexpr (SYNC == kSyncCta) {
    __syncthreads();
  } else if constexpr (SYNC == kSyncCluster) {
    cg::this_cluster().sync();
  } else {
    grid_barrier(ctr, target);
  }
}

template <class T>
__device__ __forceinline__ T block_sum(T v, T* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  T s = T(0);
  const int nw = blockDim.x >> 5;
  for (int w = 0; w < nw; ++w) s += red[w];
  __syncthreads();
  return s;
}

// row . vector dot product: compile-time n (fully unrolled, two interleaved
// partial sums) or the runtime-n loop
template <int NBC, class T>
__device__ __forceinline__ T dotn(const T* a, const T* x, int nb) {
  if constexpr (NBC > 0) {
    T s0 = T(0), s1 = T(0);
#pragma unroll
    for (int j = 0; j + 1 < NBC; j += 2) {
      s0 += a[j] * x[j];
      s1 += a[j + 1] * x[j + 1];
    }
    if constexpr (NBC & 1) s0 += a[NBC - 1] * x[NBC - 1];
    return s0 + s1;
  } else {
    T s = T(0);
    for (int j = 0; j < nb; ++j) s += a[j] * x[j];
    return s;
  }
}

template <class T, int MODE, int NBC = 0>
struct Solver {
  const PcgParams<T>& p;
  int K, nb, nn, sys, rank;
  int lo, hi, wlo, whi, slo, shi;
  T *vp, *vr, *vrt, *vsp, *vlam, *vt, *vterm, *vs, *red;
  const T *gS, *gPhi, *gTi;
  T *sS, *sPhi, *sTi;

  __device__ Solver(const PcgParams<T>& pp, int sys_, int rank_, unsigned char* smem)
      : p(pp), K(pp.K), nb(pp.nb), nn(pp.nb * pp.nb), sys(sys_), rank(rank_) {
    const int H = halo_of(p.kind, p.order);
    lo = min(K, rank * p.rows_per);
    hi = min(K, lo + p.rows_per);
    wlo = max(0, lo - H);
    whi = min(K, hi + H);
    slo = max(0, lo - (H - 1));
    shi = min(K, hi + (H - 1));
    const int wlen = min(K, p.rows_per + 2 * H) * nb;
    T* s = reinterpret_cast<T*>(smem);
    vp = s; s += wlen;
    vr = s; s += wlen;
    vrt = s; s += wlen;
    vsp = s; s += wlen;
    vlam = s; s += wlen;
    vt = s; s += wlen;
    if (p.kind == kPoly) {
      vterm = s; s += wlen;
      vs = s; s += wlen;
    } else {
      vterm = vs = nullptr;
    }
    red = s; s += 64;
    const size_t sysoff = static_cast<size_t>(sys) * K;
    gS = p.S + sysoff * 3 * nn;
    gPhi = p.Phi ? p.Phi + sysoff * 3 * nn : nullptr;
    gTi = p.Tinv ? p.Tinv + sysoff * nn : nullptr;
    sS = sPhi = sTi = nullptr;
    if (p.stage) {
      const int srows = min(K, p.rows_per + 2 * (H - 1));
      sS = s;
      s += static_cast<size_t>(srows) * 3 * nn;
      if (MODE == kModeFused) {
        if (p.kind != kIdentity) {
          sTi = s;
          s += static_cast<size_t>(srows) * nn;
        }
      } else if (p.kind != kIdentity) {
        sPhi = s;
        s += static_cast<size_t>(srows) * 3 * nn;
      }
    }
  }

  __device__ __forceinline__ int vi(int b) const { return (b - wlo) * nb; }
  __device__ __forceinline__ const T* Srow(int b) const {
    return sS ? sS + static_cast<size_t>(b - slo) * 3 * nn : gS + static_cast<size_t>(b) * 3 * nn;
  }
  __device__ __forceinline__ const T* Phirow(int b) const {
    return sPhi ? sPhi + static_cast<size_t>(b - slo) * 3 * nn
                : gPhi + static_cast<size_t>(b) * 3 * nn;
  }
  __device__ __forceinline__ const T* Tirow(int b) const {
    return sTi ? sTi + static_cast<size_t>(b - slo) * nn : gTi + static_cast<size_t>(b) * nn;
  }

  __device__ void stage_in() {
    if (!p.stage) return;
    const int rows = shi - slo;
    const size_t n3 = static_cast<size_t>(rows) * 3 * nn;
    const T* src = gS + static_cast<size_t>(slo) * 3 * nn;
    for (size_t i = threadIdx.x; i < n3; i += blockDim.x) sS[i] = src[i];
    if (sPhi) {
      const T* sp = gPhi + static_cast<size_t>(slo) * 3 * nn;
      for (size_t i = threadIdx.x; i < n3; i += blockDim.x) sPhi[i] = sp[i];
    }
    if (sTi) {
      const size_t n1 = static_cast<size_t>(rows) * nn;
      const T* st = gTi + static_cast<size_t>(slo) * nn;
      for (size_t i = threadIdx.x; i < n1; i += blockDim.x) sTi[i] = st[i];
    }
  }

  // y_b,i of a full-layout block-tridiagonal row (block_tri.cpp:82-92):
  // ((D x_b + L x_{b-1}) + R x_{b+1}).
  __device__ __forceinline__ T bt_row(const T* M, const T* x, int b, int i) const {
    const T* D = M + nn + i * nb;
    const T* xb = x + vi(b);
    T sd = dotn<NBC>(D, xb, nb);
    T out = sd;
    if (b > 0) {
      const T* Lr = M + i * nb;
      const T* xl = xb - nb;
      T sl = dotn<NBC>(Lr, xl, nb);
      out += sl;
    }
    if (b + 1 < K) {
      const T* Rr = M + 2 * nn + i * nb;
      const T* xr = xb + nb;
      T sr = dotn<NBC>(Rr, xr, nb);
      out += sr;
    }
    return out;
  }

  // remainder E = Psi - S (schur.cpp:150-159): even rows -L, -R; odd rows 0.
  __device__ __forceinline__ T rem_row(const T* x, int b, int i) const {
    if (b & 1) return T(0);
    const T* M = Srow(b);
    T out = T(0);
    if (b > 0) {
      const T* Lr = M + i * nb;
      const T* xl = x + vi(b - 1);
      T sl = -dotn<NBC>(Lr, xl, nb);
      out += sl;
    }
    if (b + 1 < K) {
      const T* Rr = M + 2 * nn + i * nb;
      const T* xr = x + vi(b + 1);
      T sr = -dotn<NBC>(Rr, xr, nb);
      out += sr;
    }
    return out;
  }

  __device__ __forceinline__ T theta_row(const T* x, int b, int i) const {
    const T* Ti = Tirow(b) + i * nb;
    const T* xb = x + vi(b);
    return dotn<NBC>(Ti, xb, nb);
  }

  __device__ __forceinline__ int shrink_lo(int a) const { return a > 0 ? a + 1 : 0; }
  __device__ __forceinline__ int shrink_hi(int c) const { return c < K ? c - 1 : K; }

  // y[b] = S_b x over rows [a, c)
  __device__ void matvec_S(T* y, const T* x, int a, int c) const {
    for (int g = threadIdx.x; g < (c - a) * nb; g += blockDim.x) {
      const int b = a + g / nb, i = g % nb;
      y[vi(b) + i] = bt_row(Srow(b), x, b, i);
    }
  }

  // Base preconditioner (everything except the poly series): x valid on
  // [xa, xc) -> out valid on [shrink(xa), shrink(xc)). Ends synchronised.
  __device__ void apply_base(T* out, const T* x, int xa, int xc) const {
    const int a = shrink_lo(xa), c = shrink_hi(xc);
    const int kind = (p.kind == kPoly) ? kStair : p.kind;
    if (kind == kIdentity) {
      for (int g = threadIdx.x; g < (c - a) * nb; g += blockDim.x) {
        const int b = a + g / nb, i = g % nb;
        out[vi(b) + i] = x[vi(b) + i];
      }
      __syncthreads();
      return;
    }
    if (MODE == kModeExplicit) {
      for (int g = threadIdx.x; g < (c - a) * nb; g += blockDim.x) {
        const int b = a + g / nb, i = g % nb;
        out[vi(b) + i] = bt_row(Phirow(b), x, b, i);
      }
      __syncthreads();
      return;
    }
    if (kind == kJacobi) {
      for (int g = threadIdx.x; g < (c - a) * nb; g += blockDim.x) {
        const int b = a + g / nb, i = g % nb;
        out[vi(b) + i] = theta_row(x, b, i);
      }
      __syncthreads();
      return;
    }
    // stair / symmetric stair on the fly
    for (int g = threadIdx.x; g < (xc - xa) * nb; g += blockDim.x) {
      const int b = xa + g / nb, i = g % nb;
      vt[vi(b) + i] = theta_row(x, b, i);  // t = theta^-1 x
    }
    __syncthreads();
    T* u = vsp;  // Sp is dead while the preconditioner runs
    for (int g = threadIdx.x; g < (c - a) * nb; g += blockDim.x) {
      const int b = a + g / nb, i = g % nb;
      const bool corr = (kind == kSymStair) || (b & 1);
      if (!corr) continue;
      const T* M = Srow(b);
      T v = x[vi(b) + i];
      if (b > 0) {
        const T* Lr = M + i * nb;
        const T* tl = vt + vi(b - 1);
        T sl = dotn<NBC>(Lr, tl, nb);
        v -= sl;
      }
      if (b + 1 < K) {
        const T* Rr = M + 2 * nn + i * nb;
        const T* tr = vt + vi(b + 1);
        T sr = dotn<NBC>(Rr, tr, nb);
        v -= sr;
      }
      u[vi(b) + i] = v;
    }
    __syncthreads();
    for (int g = threadIdx.x; g < (c - a) * nb; g += blockDim.x) {
      const int b = a + g / nb, i = g % nb;
      const bool corr = (kind == kSymStair) || (b & 1);
      out[vi(b) + i] = corr ? theta_row(u, b, i) : vt[vi(b) + i];
    }
    __syncthreads();
  }

  // r~ = Phi^-1 r (apply_preconditioner, schur.cpp:175-194) from r valid on
  // [xa, xc); result valid on [lo-1, hi+1).
  __device__ void apply(const T* x, int xa, int xc) const {
    if (p.kind != kPoly) {
      apply_base(vrt, x, xa, xc);
      return;
    }
    // term = Phi r; acc = term; repeat order times: term = Phi (E term); acc += term
    apply_base(vterm, x, xa, xc);
    int a = shrink_lo(xa), c = shrink_hi(xc);
    for (int g = threadIdx.x; g < (c - a) * nb; g += blockDim.x) {
      const int b = a + g / nb, i = g % nb;
      vrt[vi(b) + i] = vterm[vi(b) + i];
    }
    __syncthreads();
    for (int j = 0; j < p.order; ++j) {
      const int a1 = shrink_lo(a), c1 = shrink_hi(c);
      for (int g = threadIdx.x; g < (c1 - a1) * nb; g += blockDim.x) {
        const int b = a1 + g / nb, i = g % nb;
        vs[vi(b) + i] = rem_row(vterm, b, i);
      }
      __syncthreads();
      apply_base(vterm, vs, a1, c1);
      a = shrink_lo(a1);
      c = shrink_hi(c1);
      for (int g = threadIdx.x; g < (c - a) * nb; g += blockDim.x) {
        const int b = a + g / nb, i = g % nb;
        vrt[vi(b) + i] += vterm[vi(b) + i];
      }
      __syncthreads();
    }
  }

  __device__ T dot_own(const T* x, const T* y) const {
    T s = T(0);
    for (int g = threadIdx.x; g < (hi - lo) * nb; g += blockDim.x) {
      const int b = lo + g / nb, i = g % nb;
      s += x[vi(b) + i] * y[vi(b) + i];
    }
    return block_sum(s, red);
  }
};

template <class T, int MODE, int SYNC, int NBC>
__global__ void __launch_bounds__(512) k_pcg(PcgParams<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int sys, rank;
  if constexpr (SYNC == kSyncCta) {
    sys = blockIdx.x;
    rank = 0;
  } else {
    sys = blockIdx.x / p.G;
    rank = blockIdx.x % p.G;
  }
  if (p.errkey && p.errkey[sys] < 0x7f7f7f7f) return;  // formation failed (K1)
  Solver<T, MODE, NBC> s(p, sys, rank, smem_raw);
  unsigned gtarget = 0;  // grid-barrier generation (kSyncGrid)
  const int K = p.K, nb = p.nb;
  const size_t D = static_cast<size_t>(K) * nb;
  const T* gam = p.gamma + sys * D;
  const T* l0 = p.lambda0 ? p.lambda0 + sys * D : nullptr;
  T* best = p.best + sys * D;
  T* pub = p.pub + sys * D;
  T* slot_ups = p.slots + static_cast<size_t>(sys) * 2 * p.G;
  T* slot_eta = slot_ups + p.G;
  const int hr = halo_of(p.kind, p.order) - 1;
  const int ra = max(0, s.lo - hr), rc = min(K, s.hi + hr);  // rows carrying r / Sp
  const int own = (s.hi - s.lo) * nb;

  // Sum of the G per-CTA partials: lane-parallel L2 loads and a fixed-order
  // xor tree, computed redundantly by every warp of every CTA (bit-identical
  // everywhere, no dependent chain of G global loads).
  auto reduce_slots = [&](T* slots) {
    T v = T(0);
    for (int g = threadIdx.x & 31; g < p.G; g += 32) v += __ldcg(slots + g);
    return warp_sum(v);
  };

  s.stage_in();
  for (int g = threadIdx.x; g < (s.whi - s.wlo) * nb; g += blockDim.x) {
    const int b = s.wlo + g / nb, i = g % nb;
    s.vlam[g] = l0 ? l0[static_cast<size_t>(b) * nb + i] : T(0);
  }
  __syncthreads();
  // r = gamma - S lambda0 on [ra, rc)   (pcg.cpp:62)
  for (int g = threadIdx.x; g < (rc - ra) * nb; g += blockDim.x) {
    const int b = ra + g / nb, i = g % nb;
    s.vr[s.vi(b) + i] = gam[static_cast<size_t>(b) * nb + i] - s.bt_row(s.Srow(b), s.vlam, b, i);
  }
  __syncthreads();
  s.apply(s.vr, ra, rc);  // r~ on [lo-1, hi+1)
  const int ta = max(0, s.lo - 1), tc = min(K, s.hi + 1);
  for (int g = threadIdx.x; g < (tc - ta) * nb; g += blockDim.x) {
    const int b = ta + g / nb, i = g % nb;
    s.vp[s.vi(b) + i] = s.vrt[s.vi(b) + i];
  }
  T eta = s.dot_own(s.vr, s.vrt);
  for (int g = threadIdx.x; g < own; g += blockDim.x) {
    const size_t gi = static_cast<size_t>(s.lo) * nb + g;
    pub[gi] = s.vp[s.vi(s.lo) + g];
    best[gi] = s.vlam[s.vi(s.lo) + g];
  }
  if constexpr (SYNC != kSyncCta) {
    if (threadIdx.x == 0) slot_eta[rank] = eta;
    gsync<SYNC>(p.gbar, gtarget);
    eta = reduce_slots(slot_eta);
  }

  int code = kOk, which = kWhichNone, err_iter = -1, iterations = 0, converged = 0;
  double exit_eta = static_cast<double>(eta), value = 0.0, max_drift = 0.0;
  T best_eta = eta;
  const int max_iter = p.max_iter;
  const bool emit = (rank == 0 && threadIdx.x == 0);
  double* trace = p.trace ? p.trace + static_cast<size_t>(sys) * p.trace_cap : nullptr;

  if (!is_finite(eta)) {
    code = kRuntime;
    which = kWhichInitNonFinite;
  } else if (static_cast<double>(eta) < p.epsilon) {
    converged = 1;  // warm start already satisfies the exit test (pcg.cpp:72-77)
  } else {
    for (int it = 1; it <= max_iter; ++it) {
      // --- Sp on owned rows, upsilon = p'Sp (pcg.cpp:84-85)
      s.matvec_S(s.vsp, s.vp, s.lo, s.hi);
      __syncthreads();
      T ups = s.dot_own(s.vp, s.vsp);
      if constexpr (SYNC != kSyncCta) {
        if (threadIdx.x == 0) slot_ups[rank] = ups;
        gsync<SYNC>(p.gbar, gtarget);
        ups = reduce_slots(slot_ups);
      }
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
      if constexpr (SYNC != kSyncCta) {
        // refresh p's halo from the owners, then Sp on the halo rows
        for (int g = threadIdx.x; g < (s.whi - s.wlo) * nb; g += blockDim.x) {
          const int b = s.wlo + g / nb;
          if (b >= s.lo && b < s.hi) continue;
          s.vp[g] = __ldcg(pub + static_cast<size_t>(s.wlo) * nb + g);
        }
        __syncthreads();
        if (ra < s.lo) s.matvec_S(s.vsp, s.vp, ra, s.lo);
        if (rc > s.hi) s.matvec_S(s.vsp, s.vp, s.hi, rc);
        __syncthreads();
      }
      // --- r -= alpha Sp; lambda += alpha p  (pcg.cpp:94-95)
      for (int g = threadIdx.x; g < (rc - ra) * nb; g += blockDim.x) {
        const int idx = s.vi(ra) + g;
        s.vr[idx] -= alpha * s.vsp[idx];
      }
      for (int g = threadIdx.x; g < own; g += blockDim.x) {
        const int idx = s.vi(s.lo) + g;
        s.vlam[idx] += alpha * s.vp[idx];
      }
      __syncthreads();
      // --- r~ = Phi^-1 r, eta' = r'r~  (pcg.cpp:96-97)
      s.apply(s.vr, ra, rc);
      T eta_p = s.dot_own(s.vr, s.vrt);
      if constexpr (SYNC != kSyncCta) {
        if (threadIdx.x == 0) slot_eta[rank] = eta_p;
        gsync<SYNC>(p.gbar, gtarget);
        eta_p = reduce_slots(slot_eta);
      }
      if (!is_finite(eta_p)) {
        code = kRuntime;
        which = kWhichEtaNonFinite;
        err_iter = it;
        break;
      }
      if (trace && emit) trace[it - 1] = static_cast<double>(eta_p);
      if (p.check_drift) {
        // true residual gamma - S lambda vs recurrence r (pcg.cpp:103-108); G == 1 only
        T tn = T(0), rn = T(0);
        for (int g = threadIdx.x; g < own; g += blockDim.x) {
          const int b = s.lo + g / nb, i = g % nb;
          const T tr = gam[static_cast<size_t>(b) * nb + i] - s.bt_row(s.Srow(b), s.vlam, b, i);
          tn += tr * tr;
          const T rv = s.vr[s.vi(b) + i];
          rn += rv * rv;
        }
        tn = block_sum(tn, s.red);
        rn = block_sum(rn, s.red);
        const double true_norm = static_cast<double>(sqrt(tn));
        const double drift = fabs(static_cast<double>(sqrt(rn)) - true_norm) /
                             fmax(true_norm, 2.2250738585072014e-308);
        max_drift = fmax(max_drift, drift);
      }
      if (eta_p < best_eta) {  // strict <, pcg.cpp:109-112
        best_eta = eta_p;
        for (int g = threadIdx.x; g < own; g += blockDim.x)
          best[static_cast<size_t>(s.lo) * nb + g] = s.vlam[s.vi(s.lo) + g];
      }
      iterations = it;
      exit_eta = static_cast<double>(eta_p);
      if (static_cast<double>(eta_p) < p.epsilon) {
        converged = 1;
        break;
      }
      if (it == max_iter) break;
      // --- p = r~ + beta p  (pcg.cpp:121-123)
      const T beta = eta_p / eta;
      for (int g = threadIdx.x; g < (tc - ta) * nb; g += blockDim.x) {
        const int idx = s.vi(ta) + g;
        s.vp[idx] = s.vrt[idx] + beta * s.vp[idx];
      }
      eta = eta_p;
      __syncthreads();
      if constexpr (SYNC != kSyncCta) {
        for (int g = threadIdx.x; g < own; g += blockDim.x)
          pub[static_cast<size_t>(s.lo) * nb + g] = s.vp[s.vi(s.lo) + g];
      }
    }
  }
  __syncthreads();
  // lambda if converged, else the best iterate (pcg.cpp:126-128)
  T* lout = p.lambda_out + sys * D + static_cast<size_t>(s.lo) * nb;
  if (code == kOk) {
    for (int g = threadIdx.x; g < own; g += blockDim.x)
      lout[g] = converged ? s.vlam[s.vi(s.lo) + g] : best[static_cast<size_t>(s.lo) * nb + g];
  }
  if (emit) {
    SysOut o;
    o.code = code;
    o.knot = -1;
    o.which = which;
    o.iteration = err_iter;
    o.iterations = iterations;
    o.converged = converged;
    o.exit_eta = exit_eta;
    o.value = value;
    o.max_drift = max_drift;
    o.trace_len = (trace && code == kOk) ? iterations : 0;
    o._pad = 0;
    p.out[sys] = o;
  }
}

template <class T, int MODE, int SYNC, int NBC>
cudaError_t launch_mode(const PcgParams<T>& p, cudaStream_t st) {
  const size_t smem = pcg_smem_bytes(p);
  auto kern = k_pcg<T, MODE, SYNC, NBC>;
  cudaError_t e = ensure_max_smem(kern, smem);
  if (e != cudaSuccess) return e;
  if constexpr (SYNC == kSyncCta) {
    kern<<<p.B, p.nthreads, smem, st>>>(p);
    return cudaGetLastError();
  } else if constexpr (SYNC == kSyncCluster) {
    if (p.G > 8) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.B * p.G);
    cfg.blockDim = dim3(p.nthreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.G;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
  } else {
    PcgParams<T> pc = p;
    void* args[] = {&pc};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(p.B * p.G),
                                       dim3(p.nthreads), args, smem, st);
  }
}

template <class T, int NBC>
cudaError_t launch_nb(const PcgParams<T>& p, cudaStream_t st) {
  if (p.mode == kModeFused) {
    if (p.sync == kSyncCta) return launch_mode<T, kModeFused, kSyncCta, NBC>(p, st);
    if (p.sync == kSyncCluster) return launch_mode<T, kModeFused, kSyncCluster, NBC>(p, st);
    return launch_mode<T, kModeFused, kSyncGrid, NBC>(p, st);
  }
  if (p.sync == kSyncCta) return launch_mode<T, kModeExplicit, kSyncCta, NBC>(p, st);
  if (p.sync == kSyncCluster) return launch_mode<T, kModeExplicit, kSyncCluster, NBC>(p, st);
  return launch_mode<T, kModeExplicit, kSyncGrid, NBC>(p, st);
}

}  // namespace

// compile-time block dim for the BASELINE shapes (c1/c2/c4: n = 14 fp64,
// c3: n = 12 fp32), the runtime-n kernel otherwise
template <class T>
cudaError_t launch_pcg(const PcgParams<T>& p, cudaStream_t st) {
  if constexpr (sizeof(T) == 8) {
    if (p.nb == 14) return launch_nb<T, 14>(p, st);
    if (p.nb == 2) return launch_nb<T, 2>(p, st);  // the SQP / NMPC models
    if (p.nb == 4) return launch_nb<T, 4>(p, st);
  } else {
    if (p.nb == 12) return launch_nb<T, 12>(p, st);
  }
  return launch_nb<T, 0>(p, st);
}

template cudaError_t launch_pcg<double>(const PcgParams<double>&, cudaStream_t);
template cudaError_t launch_pcg<float>(const PcgParams<float>&, cudaStream_t);
template size_t pcg_smem_bytes<double>(const PcgParams<double>&);
template size_t pcg_smem_bytes<float>(const PcgParams<float>&);

}  // namespace b2p
