// Fused cluster kernel (FC) — formation + symmetric-stair PCG for one system
// on one thread-block cluster of G CTAs (G = 1, 2, 4, 8, 16), persistent over a
// batch. Replaces build_schur (proj/src/schur.cpp:38-82), the stair-family
// builders (:98-142) and pcg_solve (proj/src/pcg.cpp:55-129) in one launch.
//
// Layout: CTA c of the cluster owns block rows [lo, hi) = [c*rp, (c+1)*rp);
// half-warp h owns block row lo + h, lane l < n owns scalar row l and keeps in
// registers its row of L_b and of theta_b^-1 (the two operators it applies
// twice per iteration). D_b and the L blocks needed for the column products
// R_b x = L_{b+1}' x live in shared memory. Neighbour data crosses CTAs through
// distributed shared memory (DSMEM).
//
// Per iteration three cluster barriers: after upsilon = p'Sp, after
// t = theta^-1 r (the stair correction reads t of the neighbour rows), after
// eta' = r'r~. p's halo rows are recomputed locally from the neighbour's
// published r~ (p_halo = r~_halo + beta p_halo), bitwise equal to the owner's
// value, so the p update needs no cluster barrier. All reductions are
// fixed-order (warp tree, 16 warp partials, G CTA partials): every CTA holds
// bit-identical scalars and results are reproducible run to run.
#include <cooperative_groups.h>

#include <climits>

#include "hw_dense.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace b2p {
namespace {

using namespace hwd;
constexpr int kFcThreads = 512;
constexpr int VS = 16;  // padded row stride of the vector arrays (16-byte aligned)

template <class T> struct V2;
template <> struct V2<double> { using t = double2; };
template <> struct V2<float> { using t = float2; };
template <class T>
__device__ __forceinline__ typename V2<T>::t ld2(const T* p) {
  return *reinterpret_cast<const typename V2<T>::t*>(p);
}

// sum_j m[j] x[j] with m in registers, x in (possibly remote) shared memory
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
// row l of a row-major NB x NB block in shared memory, times x
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
// column l of a row-major block (Mcol = M + l), times x
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

template <class T, int NB, int MB>
struct FcLayout {
  static constexpr int NN = NB * NB, MM = MB * MB, LD = NB | 1, LDM = MB | 1;
  static constexpr int per_hw = NB * LD + NB * LDM + 32;
  // PCG phase (elements)
  __host__ __device__ static int oL() { return 0; }
  __host__ __device__ static int oD(int rp) { return (rp + 1) * NN; }
  __host__ __device__ static int oP(int rp) { return oD(rp) + rp * NN; }
  __host__ __device__ static int oR(int rp) { return oP(rp) + (rp + 2) * VS; }
  __host__ __device__ static int oT(int rp) { return oR(rp) + rp * VS; }
  __host__ __device__ static int oU(int rp) { return oT(rp) + rp * VS; }
  __host__ __device__ static int oRed(int rp) { return oU(rp) + rp * VS; }
  __host__ __device__ static int oCp(int rp) { return oRed(rp) + 64; }
  __host__ __device__ static int pcg_total(int rp) { return oCp(rp) + 8; }
  // formation phase (elements, aliases the PCG phase)
  __host__ __device__ static int oQi() { return 0; }
  __host__ __device__ static int oRi(int rp) { return rp * NN; }
  __host__ __device__ static int oqq(int rp) { return oRi(rp) + rp * MM; }
  __host__ __device__ static int orr(int rp) { return oqq(rp) + rp * VS; }
  __host__ __device__ static int oScr(int rp) { return orr(rp) + rp * VS; }
  __host__ __device__ static int form_total(int rp) { return oScr(rp) + 32 * per_hw; }
  __host__ __device__ static int total(int rp) {
    const int a = pcg_total(rp), b = form_total(rp);
    return a > b ? a : b;
  }
};

}  // namespace

template <class T, int NB, int MB>
__global__ void __launch_bounds__(kFcThreads, 1) k_fc(FusedParams<T> p, int rp) {
  using FL = FcLayout<T, NB, MB>;
  constexpr int NN = FL::NN, MM = FL::MM, LD = FL::LD, LDM = FL::LDM;
  cg::cluster_group cl = cg::this_cluster();
  const int G = static_cast<int>(cl.num_blocks());
  const int c = static_cast<int>(cl.block_rank());
  const int K = p.K, N = K - 1;
  const int lo = c * rp, hi = min(K, lo + rp), nrow = max(0, hi - lo);
  const int tid = threadIdx.x, lane = tid & 31, l = lane & 15, h = tid >> 4;
  const bool lact = l < NB;
  const int lr = lact ? l : NB - 1;
  const bool rowv = h < nrow;
  const int b = lo + (rowv ? h : 0);

  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  T* sL = sm + FL::oL();
  T* sD = sm + FL::oD(rp);
  T* sP = sm + FL::oP(rp);  // rows lo-1 .. hi
  T* sR = sm + FL::oR(rp);
  T* sT = sm + FL::oT(rp);
  T* sU = sm + FL::oU(rp);
  T* red = sm + FL::oRed(rp);
  T* cpart = sm + FL::oCp(rp);
  T* sQi = sm + FL::oQi();
  T* sRi = sm + FL::oRi(rp);
  T* sqq = sm + FL::oqq(rp);
  T* srr = sm + FL::orr(rp);
  T* hw = sm + FL::oScr(rp) + h * FL::per_hw;
  T* tW = hw;
  T* tBR = tW + NB * LD;
  T* rd = tBR + NB * LDM;
  __shared__ int s_err;

  const size_t slot_stride = static_cast<size_t>(2) * rp * NN;
  T* gL = p.slot + static_cast<size_t>(blockIdx.x) * slot_stride;  // [rp][NN] own rows
  T* gD = gL + static_cast<size_t>(rp) * NN;
  const T* gLnext = gL + slot_stride;  // next CTA of the cluster: its row 0 = L_hi

  const int ncl = gridDim.x / G, cid = blockIdx.x / G;
  for (int sys = cid; sys < p.B; sys += ncl) {
    const T* Qs = p.Q + static_cast<size_t>(sys) * K * NN;
    const T* qs = p.q + static_cast<size_t>(sys) * K * NB;
    const T* Rs = p.R + static_cast<size_t>(sys) * N * MM;
    const T* rs = p.r + static_cast<size_t>(sys) * N * MB;
    const T* As = p.A + static_cast<size_t>(sys) * N * NN;
    const T* Bs = p.Bm + static_cast<size_t>(sys) * N * (NB * MB);
    const T* es = p.e + static_cast<size_t>(sys) * N * NB;
    const T* xs = p.x_s + static_cast<size_t>(sys) * NB;
    const T* x0 = p.x0 + static_cast<size_t>(sys) * NB;

    cl.sync();  // every CTA of the cluster is done with the previous system
    if (tid == 0) s_err = INT_MAX;
    int fkey = INT_MAX;

    // ======================================================== F1: own knots
    // Q_k^-1, Q_k^-1 q_k, R_k^-1, R_k^-1 r_k for k in [lo, hi) (schur.cpp:15-23)
    if (rowv) {
      const int k = b;
      T x[NB];
      const int f = hw_spd_inverse<T, NB, LD>(tW, rd, Qs + static_cast<size_t>(k) * NN, l, x);
      if (f >= 0) fkey = min(fkey, k == 0 ? 0 : 4 * k + 2);
      if (lact) {
        T qq = T(0);
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          sQi[h * NN + i * NB + l] = x[i];
          qq += x[i] * qs[k * NB + i];
        }
        sqq[h * VS + l] = qq;
      }
      if (k < N) {
        T y[MB];
        const int g = hw_spd_inverse<T, MB, LDM>(tW, rd, Rs + static_cast<size_t>(k) * MM, l, y);
        if (g >= 0) fkey = min(fkey, 4 * (k + 1) + 1);
        if (l < MB) {
          T rr = T(0);
#pragma unroll
          for (int i = 0; i < MB; ++i) {
            sRi[h * MM + i * MB + l] = y[i];
            rr += y[i] * rs[k * MB + i];
          }
          srr[h * VS + l] = rr;
        }
      }
    }
    cl.sync();  // knot data visible cluster-wide (row lo reads knot lo-1 remotely)

    // ======================================================== F2: own rows
    T ti[NB];  // row l of theta_b^-1
    T gam = T(0);
#pragma unroll
    for (int i = 0; i < NB; ++i) ti[i] = T(0);
    if (rowv) {
      if (b == 0) {
        // schur.cpp:53-57: S(0,0) = Q0^-1, theta_inv[0] = sym(Q0), gamma_0
        if (lact) {
#pragma unroll
          for (int i = 0; i < NB; ++i) {
            gD[i * NB + l] = sQi[i * NB + l];
            ti[i] = T(0.5) * (Qs[l * NB + i] + Qs[i * NB + l]);
          }
          gam = -((xs[l] - x0[l]) + sqq[l]);
        }
      } else {
        const int k = b - 1;
        const T* Qk;
        const T* Rk;
        const T* qqk;
        const T* rrk;
        if (h > 0) {
          Qk = sQi + (h - 1) * NN;
          Rk = sRi + (h - 1) * MM;
          qqk = sqq + (h - 1) * VS;
          rrk = srr + (h - 1) * VS;
        } else {  // knot lo-1 belongs to CTA c-1: read it through DSMEM
          T* rm = cl.map_shared_rank(sm, c - 1);
          Qk = rm + FL::oQi() + (rp - 1) * NN;
          Rk = rm + FL::oRi(rp) + (rp - 1) * MM;
          qqk = rm + FL::oqq(rp) + (rp - 1) * VS;
          rrk = rm + FL::orr(rp) + (rp - 1) * VS;
        }
        const T* Ak = As + static_cast<size_t>(k) * NN;
        const T* Bk = Bs + static_cast<size_t>(k) * NB * MB;
        T x[NB];
        {  // AQ = A_k Q_k^-1 column l -> L_b = -AQ  (schur.cpp:68)
          T qc[NB];
#pragma unroll
          for (int q = 0; q < NB; ++q) qc[q] = Qk[q * NB + lr];
#pragma unroll
          for (int i = 0; i < NB; ++i) {
            T s = T(0);
#pragma unroll
            for (int q = 0; q < NB; q += 2) {
              const auto a2 = __ldg(reinterpret_cast<const typename V2<T>::t*>(Ak + i * NB + q));
              s += a2.x * qc[q];
              s += a2.y * qc[q + 1];
            }
            x[i] = s;
          }
        }
        __syncwarp(hw_mask());
        if (lact) {
#pragma unroll
          for (int i = 0; i < NB; ++i) {
            tW[i * LD + l] = x[i];
            gL[static_cast<size_t>(h) * NN + i * NB + l] = -x[i];
          }
        }
        {  // BR = B_k R_k^-1 column l < m
          const int lm = l < MB ? l : MB - 1;
          T rc[MB];
#pragma unroll
          for (int q = 0; q < MB; ++q) rc[q] = Rk[q * MB + lm];
#pragma unroll
          for (int i = 0; i < NB; ++i) {
            T s = T(0);
#pragma unroll
            for (int q = 0; q < MB; ++q) s += __ldg(Bk + i * MB + q) * rc[q];
            if (l < MB) tBR[i * LDM + l] = s;
          }
        }
        __syncwarp(hw_mask());
        // theta_raw column l (schur.cpp:65-66)
        T arow[NB], brow[MB];
#pragma unroll
        for (int q = 0; q < NB; q += 2) {
          const auto a2 = __ldg(reinterpret_cast<const typename V2<T>::t*>(Ak + lr * NB + q));
          arow[q] = a2.x;
          arow[q + 1] = a2.y;
        }
#pragma unroll
        for (int q = 0; q < MB; ++q) brow[q] = __ldg(Bk + lr * MB + q);
        const T* Q1 = sQi + h * NN;  // knot b = k + 1 (own)
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          T s1 = T(0), s2 = T(0);
#pragma unroll
          for (int q = 0; q < NB; ++q) s1 += tW[i * LD + q] * arow[q];
#pragma unroll
          for (int q = 0; q < MB; ++q) s2 += tBR[i * LDM + q] * brow[q];
          x[i] = (s1 + s2) + Q1[i * NB + lr];
        }
        {  // zeta, gamma (schur.cpp:69-77)
          T aqq = T(0), brr = T(0);
#pragma unroll
          for (int q = 0; q < NB; ++q) aqq += arow[q] * qqk[q];
#pragma unroll
          for (int q = 0; q < MB; ++q) brr += brow[q] * rrk[q];
          const T zeta = (-aqq - brr) + sqq[h * VS + lr];
          gam = -(-__ldg(es + static_cast<size_t>(k) * NB + lr) + zeta);
        }
        hw_symmetrize_col<T, NB, LD>(tW, l, x);  // theta (schur.cpp:67)
        if (lact) {
#pragma unroll
          for (int i = 0; i < NB; ++i) {
            gD[static_cast<size_t>(h) * NN + i * NB + l] = x[i];
            tW[i * LD + l] = x[i];
          }
        }
        __syncwarp(hw_mask());
        {  // theta^-1 (schur.cpp:75) straight into the PCG registers
          const int f = hw_cholesky<T, NB, LD>(tW, rd, l);
          if (f >= 0) fkey = min(fkey, b * 4 + 3);
          hw_inv_col<T, NB, LD>(tW, rd, lact ? l : 0, x);
          hw_symmetrize_col<T, NB, LD>(tW, l, x);
#pragma unroll
          for (int i = 0; i < NB; ++i) ti[i] = x[i];
        }
      }
    }
    if (l == 0 && rowv && fkey != INT_MAX) atomicMin(&s_err, fkey);
    cl.sync();  // remote formation reads done; slots written; s_err final
    int err = INT_MAX;
    for (int g = 0; g < G; ++g) err = min(err, *cl.map_shared_rank(&s_err, g));
    if (err != INT_MAX) {
      if (c == 0 && tid == 0) {
        p.errkey[sys] = err;
        SysOut o{};
        o.code = kRuntime;
        o.which = kWhichNone;
        o.iteration = -1;
        p.out[sys] = o;
      }
      continue;
    }
    if (c == 0 && tid == 0) p.errkey[sys] = 0x7f7f7f7f;

    // ======================================================== P: stage
    {
      const int n_own = nrow * NN;
      for (int i = tid; i < n_own; i += kFcThreads) {
        sL[i] = __ldcg(gL + i);
        sD[i] = __ldcg(gD + i);
      }
      if (hi < K)  // L_hi from the next CTA's slot (R_{hi-1} = L_hi')
        for (int i = tid; i < NN; i += kFcThreads) sL[n_own + i] = __ldcg(gLnext + i);
    }
    T lrow[NB];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NB; ++j) lrow[j] = sL[h * NN + lr * NB + j];
    const bool hasL = rowv && b > 0;
    const bool hasR = rowv && b + 1 < K;
    const bool act = rowv && lact;
    const bool lhalo = lo > 0, rhalo = hi < K;
    T* const rmL = lhalo ? cl.map_shared_rank(sm, c - 1) : sm;  // neighbour CTAs
    T* const rmR = rhalo ? cl.map_shared_rank(sm, c + 1) : sm;
    T* myP = sP + (h + 1) * VS;  // p row b

    // (half-warps past the CTA's last row compute nothing: their rows would
    // index past the row arrays, into buffers other warps are writing)
    auto Srow = [&](const T* P) -> T {  // ((D p_b + L p_{b-1}) + R p_{b+1}), block_tri.cpp:82-92
      if (!rowv) return T(0);
      const T* pb = P + (h + 1) * VS;
      T out = dot_row<T, NB>(sD + h * NN + lr * NB, pb);
      if (hasL) out += dot_reg<T, NB>(lrow, pb - VS);
      if (hasR) out += dot_col<T, NB>(sL + (h + 1) * NN + lr, pb + VS);
      return out;
    };
    auto reduce = [&](T v, int buf) -> T {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[buf * 32 + (tid >> 5)] = v;
      __syncthreads();
      T s = T(0);
#pragma unroll
      for (int w = 0; w < kFcThreads / 32; ++w) s += red[buf * 32 + w];
      if (G == 1) return s;
      if (tid == 0) cpart[buf] = s;
      cl.sync();
      T tot = T(0);
      for (int g = 0; g < G; ++g) tot += *cl.map_shared_rank(cpart + buf, g);
      return tot;
    };
    const bool stairish = p.kind == kStair || p.kind == kSymStair;
    auto precondition = [&](T rv) -> T {
      if (p.kind == kIdentity) return rv;
      if (act) sU[h * VS + l] = rv;
      __syncwarp();
      const T tv = rowv ? dot_reg<T, NB>(ti, sU + h * VS) : T(0);  // t = theta^-1 r
      if (!stairish) return tv;                     // block Jacobi
      if (act) sT[h * VS + l] = tv;
      if (G == 1) __syncthreads(); else cl.sync();
      T uv = rv;
      if (hasL) {
        const T* tl = (h > 0) ? sT + (h - 1) * VS : rmL + FL::oT(rp) + (rp - 1) * VS;
        uv -= dot_reg<T, NB>(lrow, tl);
      }
      if (hasR) {
        const T* tr = (h + 1 < nrow) ? sT + (h + 1) * VS : rmR + FL::oT(rp);
        uv -= dot_col<T, NB>(sL + (h + 1) * NN + lr, tr);
      }
      __syncwarp();
      if (act) sU[h * VS + l] = uv;
      __syncwarp();
      const bool corr = (p.kind == kSymStair) || (b & 1);
      return (corr && rowv) ? dot_reg<T, NB>(ti, sU + h * VS) : tv;  // r~ = theta^-1 u
    };

    // r = gamma - S lambda0 (pcg.cpp:62)
    const size_t voff = static_cast<size_t>(sys) * K * NB;
    T lam = T(0);
    if (p.lambda0) {
      for (int i = tid; i < (nrow + 2) * VS; i += kFcThreads) {
        const int row = lo - 1 + i / VS, j = i % VS;
        sP[i] = (row >= 0 && row < K && j < NB) ? p.lambda0[voff + row * NB + j] : T(0);
      }
      __syncthreads();
      if (act) lam = myP[l];
    }
    T rr = act ? gam - (p.lambda0 ? Srow(sP) : T(0)) : T(0);
    __syncthreads();
    T rt = precondition(rr);
    if (act) sR[h * VS + l] = rt;
    T eta = reduce(act ? rr * rt : T(0), 1);
    // p = r~ (own rows and, from the neighbours' published r~, the halo rows)
    T pp = rt;
    if (act) myP[l] = pp;
    if (lhalo && h == 0 && lact) sP[l] = rmL[FL::oR(rp) + (rp - 1) * VS + l];
    if (rhalo && h == nrow - 1 && lact) sP[(nrow + 1) * VS + l] = rmR[FL::oR(rp) + l];
    __syncthreads();

    int code = kOk, which = kWhichNone, err_iter = -1, iterations = 0, converged = 0;
    double exit_eta = static_cast<double>(eta), value = 0.0;
    T best_eta = eta, best = lam;
    double* trace = p.trace ? p.trace + static_cast<size_t>(sys) * p.trace_cap : nullptr;
    if (!is_finite(eta)) {
      code = kRuntime;
      which = kWhichInitNonFinite;
    } else if (static_cast<double>(eta) < p.epsilon) {
      converged = 1;
    } else {
      for (int it = 1; it <= p.max_iter; ++it) {
        const T spv = rowv ? Srow(sP) : T(0);
        const T ups = reduce(act ? pp * spv : T(0), 0);
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
        rr -= alpha * spv;
        lam += alpha * pp;
        rt = precondition(rr);
        if (act) sR[h * VS + l] = rt;
        const T eta_p = reduce(act ? rr * rt : T(0), 1);
        if (!is_finite(eta_p)) {
          code = kRuntime;
          which = kWhichEtaNonFinite;
          err_iter = it;
          break;
        }
        if (trace && c == 0 && tid == 0) trace[it - 1] = static_cast<double>(eta_p);
        if (eta_p < best_eta) {
          best_eta = eta_p;
          best = lam;
        }
        iterations = it;
        exit_eta = static_cast<double>(eta_p);
        if (static_cast<double>(eta_p) < p.epsilon) {
          converged = 1;
          break;
        }
        if (it == p.max_iter) break;
        const T beta = eta_p / eta;
        pp = rt + beta * pp;
        if (act) myP[l] = pp;
        // halo p rows: the owner's arithmetic on the owner's data, bitwise equal
        if (lhalo && h == 0 && lact)
          sP[l] = rmL[FL::oR(rp) + (rp - 1) * VS + l] + beta * sP[l];
        if (rhalo && h == nrow - 1 && lact)
          sP[(nrow + 1) * VS + l] = rmR[FL::oR(rp) + l] + beta * sP[(nrow + 1) * VS + l];
        eta = eta_p;
        __syncthreads();
      }
    }
    if (code == kOk && act) p.lambda_out[voff + static_cast<size_t>(b) * NB + l] = converged ? lam : best;
    if (c == 0 && tid == 0) {
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
  }
  cl.sync();  // keep every CTA's shared memory alive until the neighbours are done
}

// ------------------------------------------------------------------ host side
namespace {
template <class T, int NB, int MB>
size_t fc_smem(int rp) {
  return sizeof(T) * static_cast<size_t>(FcLayout<T, NB, MB>::total(rp));
}
}  // namespace

template <class T>
int fc_pick_g(int K, int n, int m, int kind, int B) {
  // compiled: (14, 7), (16, 8) fp64 (the latter for padded shapes), (12, 4) fp32
  const bool shape = (sizeof(T) == 8 && ((n == 14 && m == 7) || (n == 16 && m == 8))) ||
                     (sizeof(T) == 4 && n == 12 && m == 4);
  if (!shape || kind == kPoly || K < 2) return 0;
  for (int G : {1, 2, 4, 8, 16}) {
    const int rp = (K + G - 1) / G;
    if (rp <= 32 && (K + rp - 1) / rp == G) return G;
  }
  return 0;
}

template <class T>
size_t fc_slot_elems(int K, int n, int G) {
  const int rp = (K + G - 1) / G;
  return static_cast<size_t>(2) * rp * n * n;
}

template <class T>
cudaError_t launch_fc(const FusedParams<T>& p, int G, int max_clusters, cudaStream_t st, int nb) {
  const int rp = (p.K + G - 1) / G;
  auto go = [&](auto kern, size_t smem) -> cudaError_t {
    cudaError_t e = ensure_max_smem(kern, smem);
    if (e != cudaSuccess) return e;
    if (G > 8) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = G;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(kFcThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int ncl = 0;
    cfg.gridDim = dim3(G);
    e = cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
    if (e != cudaSuccess || ncl < 1) ncl = 1;
    ncl = std::min(ncl, std::min(p.B, max_clusters));
    cfg.gridDim = dim3(G * ncl);
    return cudaLaunchKernelEx(&cfg, kern, p, rp);
  };
  if constexpr (sizeof(T) == 8) {
    if (nb == 16) return go(k_fc<T, 16, 8>, fc_smem<T, 16, 8>(rp));
    return go(k_fc<T, 14, 7>, fc_smem<T, 14, 7>(rp));
  } else {
    return go(k_fc<T, 12, 4>, fc_smem<T, 12, 4>(rp));
  }
}

template int fc_pick_g<double>(int, int, int, int, int);
template int fc_pick_g<float>(int, int, int, int, int);
template size_t fc_slot_elems<double>(int, int, int);
template size_t fc_slot_elems<float>(int, int, int);
template cudaError_t launch_fc<double>(const FusedParams<double>&, int, int, cudaStream_t, int);
template cudaError_t launch_fc<float>(const FusedParams<float>&, int, int, cudaStream_t, int);

}  // namespace b2p
