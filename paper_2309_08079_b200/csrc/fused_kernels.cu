// K1+K2+K3 fused — persistent "one CTA per system" symmetric-stair PCG for
// systems that fit one SM (c1: K=32, c4: K=64 at n=14, m=7, fp64).
//
// One launch solves a whole batch: gridDim.x CTAs (one per SM) loop over the
// systems of the batch. Per system:
//   F  (build_schur + preconditioner data, schur.cpp:38-82,109-142): each
//      16-lane half-warp owns block rows h, h+32 (the rows it will own in the
//      PCG phase) and computes, with compile-time n, m:
//        Q_{k+1}^-1, R_k^-1, Q_k^-1  (Cholesky + triangular inverse, lane j
//        holds column j in registers; symmetrised through a shared tile),
//        L_b = -A Q_k^-1, D_b = theta_b = sym((A Q_k^-1) A' + (B R_k^-1) B'
//        + Q_{k+1}^-1), gamma_b and theta_b^-1.
//      L, D and theta^-1 go to a CTA-private global slot (L2 resident: the
//      CTA rewrites the same 300 KB for every system), gamma stays in registers.
//   P  (pcg_solve, pcg.cpp:55-129): L and D are copied into shared memory
//      (row-major n x n blocks, read as 16-byte pairs along rows — conflict
//      free for n = 14 — and as 8-byte columns for the R_b = L_{b+1}' product),
//      theta^-1 rows live in registers of the thread that owns the row. The
//      stair family is applied on the fly:
//        t_j = theta_j^-1 r_j,  u_i = r_i - L_i t_{i-1} - R_i t_{i+1},
//        r~_i = theta_i^-1 u_i   (odd rows for stair, all rows for symstair),
//      the reference's materialised -theta_i^-1 L_i theta_{i-1}^-1 blocks
//      re-associated (bitwise-symmetric S and theta^-1 make the symmetric-stair
//      mirror exactly this formula on the even rows).
//      upsilon and eta' are warp-shuffle trees + a fixed-order combine of the
//      16 warp partials: bit-reproducible, no atomics.
#include "kernels.h"
#include "hw_dense.cuh"
#include "tmem.cuh"

namespace b2p {
namespace {
constexpr int kThreads = 512;  // 32 half-warps
constexpr int kHalfWarps = kThreads / 16;

using namespace hwd;

// Formation-phase shared memory (elements): per-knot Q^-1 and the products
// Q^-1 q, R^-1 r, then the 8-lane group tiles (R^-1 goes to the slot) whose
// region ends with the D blocks the PCG reads in place, then the q_k.
template <class T, int NB, int MB>
struct FLayout {
  // 8-lane group tiles of F1 (L^-T of Q_g, then the R_g^-1 tiles) and of the
  // theta^-1 pass: [max(n n, 2 MB MB)] | rd [16]
  static constexpr int g8_tile = (NB * NB > 2 * MB * MB ? NB * NB : 2 * MB * MB) + 16;
  static constexpr int tiles0 = 64 * g8_tile;
  static constexpr int ls = NB * NB + ((8 - (NB * NB) % 32) + 32) % 32;  // fused_ls(NB)
  __host__ __device__ static constexpr int oQi(int) { return 0; }
  __host__ __device__ static constexpr int oqq(int K) { return K * NB * NB; }
  __host__ __device__ static constexpr int orr(int K) { return oqq(K) + K * 16; }
  __host__ __device__ static constexpr int ohw(int K) { return orr(K) + (K - 1) * 8; }
  // The tile region also holds, at its end, the D blocks F2 leaves in place for
  // the PCG (theta_1..theta_63, D_0 = Q_0^-1 before them: oD); it is sized so
  // they clear the PCG's staged L (padded stride) and vectors below them.
  __host__ __device__ static constexpr int tiles(int K) {
    const int need = K * ls + 3 * K * NB + 32 - ohw(K) + 64 * NB * NB;
    return tiles0 > need ? tiles0 : need;
  }
  __host__ __device__ static constexpr int oD(int K) { return ohw(K) + tiles(K) - 64 * NB * NB; }
  __host__ __device__ static constexpr int osq(int K) { return ohw(K) + tiles(K); }  // q_k
  __host__ __device__ static constexpr int total(int K) { return osq(K) + K * NB; }
  // PCG vectors p, t, u (+ the reduction words) after the staged L
  __host__ __device__ static constexpr int osp(int K) { return K * ls; }
  static constexpr size_t elems(int K) {
    const size_t pcg = static_cast<size_t>(K) * (NB * NB + ls) + 3 * K * NB + 64;
    return pcg > static_cast<size_t>(total(K)) ? pcg : static_cast<size_t>(total(K));
  }
  // horizon K fits: the theta^-1 pass's group tiles (groups < K + 3) stay
  // clear of the D blocks F2 leaves in place (oD), and shared memory holds it
  static constexpr bool fits(int K) {
    return (K + 3) * g8_tile <= oD(K) && elems(K) * sizeof(T) + 64 <= 227 * 1024;
  }
  static constexpr int capacity(int kmax) {
    for (int K = kmax; K >= 2; --K)
      if (fits(K)) return K;
    return 0;
  }
  // The kernel lays shared memory out for its largest horizon (kcap(R)), not
  // for the launch's K: every region offset is a compile-time constant, so the
  // PCG's per-thread addresses are one register plus immediates (a runtime-K
  // layout had the compiler rematerialise them — S2R / LDC / IMAD — inside the
  // solve loop: 10 % of the kernel's instructions).
  static constexpr int kcap(int R) { return capacity(R == 1 ? 32 : 64); }
};

}  // namespace

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// One-thread TMA bulk copy global -> shared, completed on an mbarrier
// (16-byte aligned source, destination and size).
__device__ __forceinline__ void tma_load_1d(void* dst_smem, const void* src, unsigned bytes,
                                            unsigned mbar_addr) {
  asm volatile("fence.proxy.async;\n" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mbar_addr),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
      "[%3];\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst_smem))),
      "l"(src), "r"(bytes), "r"(mbar_addr)
      : "memory");
}
// Second bulk copy completing on the same mbarrier phase (the first call's
// expect_tx must have covered its bytes).
__device__ __forceinline__ void tma_copy_1d(void* dst_smem, const void* src, unsigned bytes,
                                            unsigned mbar_addr) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
      "[%3];\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst_smem))),
      "l"(src), "r"(bytes), "r"(mbar_addr)
      : "memory");
}
// mbar_wait on the parity held in bit `bit` of st, which is then flipped
__device__ __forceinline__ void mbar_wait_bit(unsigned mbar_addr, unsigned& st, unsigned bit) {
  unsigned done = 0;
  const unsigned phase = (st & bit) ? 1u : 0u;
  while (!done) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, "
        "1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(mbar_addr), "r"(phase)
        : "memory");
  }
  st ^= bit;
}
__device__ __forceinline__ void mbar_wait(unsigned mbar_addr, unsigned& phase) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, "
        "1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(mbar_addr), "r"(phase)
        : "memory");
  }
  phase ^= 1u;
}

// D = A B + D on the FP64 tensor cores (m8n8k4, A row-major, B column-major
// fragments): bitwise the FMA chain d = fma(a_k, b_k, d) over k = 0..3.
__device__ __forceinline__ void dmma_f64(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// ---- Tensor memory (TMEM) as a third on-chip operand store for the PCG
// phase: 512 columns x 128 lanes x 32 bit; thread t of warp w owns TMEM lane
// 32*(w%4) + t%32 and columns [128*(w/4), 128*(w/4) + 128): rows pi and
// pi + NB/2 of D_b and of L_b, 32 columns (NB <= 16 doubles) each (tmem.cuh).
// Measured tcgen05.ld throughput ~390 B/clk/SM vs 128 B/clk for shared memory
// (scripts/micro/tmem_bench.cu), so the row products come from TMEM and only
// the column products R_b = L_{b+1}' read shared memory.

// Block stride (elements) of L in the slot and in shared memory: n*n padded to
// 8 mod 32 doubles, so the four quarter-warps of a PCG warp (consecutive block
// rows) read their column-product operands from disjoint banks (n = 14: 200).
__host__ __device__ constexpr int fused_ls(int n) { return n * n + ((8 - (n * n) % 32) + 32) % 32; }

// per-CTA slot stride in elements, padded to 16 bytes (the TMA source must be aligned):
// L [K][LS] | D [K][n n] | theta^-1 [K][n n] | gamma [K][n] | R^-1 [K][m m]
// (| Q^-1 [K][n n] with the fused PPCG finish, keep_q)
template <class T>
__host__ __device__ inline size_t fused_slot_stride(int K, int n, int m, bool keep_q = false) {
  const size_t e = static_cast<size_t>(K) * fused_ls(n) +
                   static_cast<size_t>(keep_q ? 3 : 2) * K * n * n + static_cast<size_t>(K) * n +
                   static_cast<size_t>(K) * m * m;
  const size_t a = 16 / sizeof(T);
  return (e + a - 1) / a * a;
}

// NB: the state dimension n (even, <= 16); MB: the control dimension padded
// (R^-1 tiles and the slot use MB; EXM: m == MB exactly, else the runtime
// p.m_rt <= MB with identity-padded R and zero-padded B, r — the pad terms add
// exact zeros after the real ones, so every sum equals the unpadded one).
// TM: the B2P_PHASE_TIMING build (globaltimer / SM-clock stamps); the
// production instantiation carries no stamp code at all.
template <class T, int NB, int MB, int R, bool EXM, bool TM>
__global__ void __launch_bounds__(kThreads, 1) k_fused_cta(FusedParams<T> p) {
  static_assert(sizeof(T) == 8 && NB % 2 == 0 && NB <= 16 && MB <= 8,
                "one-CTA kernel: fp64, even n <= 16, m <= 8");
  constexpr int H = NB / 2;  // PCG rows per thread: pi and pi + H
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using FL = FLayout<T, NB, MB>;
  constexpr int NN = NB * NB;
  const int K = p.K, N = K - 1;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int l = lane & 15;        // row inside the block
  const int h = tid >> 4;         // half-warp index = owned block row (first)
  const bool lact = l < NB;
  T* smem = reinterpret_cast<T*>(smem_raw);
  // PCG layout. [0, K*NN): D staged from the slot at the start of the phase
  // (slot -> shared -> TMEM), then the next system's Q_k, TMA-prefetched for
  // its formation while this system's PCG runs (as are its q_k, into the q
  // region past `red`); sL: the L blocks at the padded stride LS.
  constexpr int LS = fused_ls(NB);
  T* sL = smem;                                 // [K][LS]  staging only
  constexpr int KL = FL::kcap(R);  // the layout's horizon (>= K)
  static_assert(KL >= 2, "no horizon fits the one-CTA layout");
  T* sp = smem + FL::osp(KL);                   // [K][NB]
  T* st = sp + KL * NB;
  T* su = st + KL * NB;
  T* red = su + KL * NB;                        // [32]
  // F2 leaves gamma_b in su (read once by the PCG stage, before the first
  // preconditioner application writes u) where u clears Q_k^-1 q_k / R_k^-1
  // r_k, which F2 reads, and the theta^-1 pass's group tiles (the c4 layout);
  // otherwise in the global slot
  constexpr bool kGamS = FL::osp(KL) + 2 * KL * NB >= FL::orr(KL) + (KL - 1) * 8 &&
                         FL::osp(KL) + 2 * KL * NB >= (KL + 3) * FL::g8_tile;
  // D_b rows stay where the formation left them: theta_b (b >= 1) at the end
  // of the tile region (F2), D_0 = Q_0^-1 just before (FLayout::oD)
  T* sD = smem + FL::oD(KL);                    // [K][NB][NB]  D row products
  // formation layout (aliases the PCG layout; phases are separated by barriers)
  T* sQi = smem + FL::oQi(KL);   // [K][NB][NB], column l written by lane l
  T* sqq = smem + FL::oqq(KL);   // [K][16]  Q_k^-1 q_k
  T* srr = smem + FL::orr(KL);   // [N][8]   R_k^-1 r_k
  __shared__ int s_err;
  __shared__ __align__(8) unsigned long long s_mbar;  // TMA staging barrier
  __shared__ __align__(8) unsigned long long s_mbar2;  // next system's Q prefetch
  const unsigned mbar_addr = static_cast<unsigned>(__cvta_generic_to_shared(&s_mbar));
  const unsigned mbar2_addr = static_cast<unsigned>(__cvta_generic_to_shared(&s_mbar2));
  // mbarrier phase parities and the prefetch flag packed in one register
  // (bit 0: s_mbar, bit 1: s_mbar2, bit 2: this system's Q_k / q_k already on
  // their way): loop-carried scalars that would otherwise be spilled
  unsigned mst = 0;
  __shared__ unsigned s_taddr;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mbar_addr) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mbar2_addr) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if ((tid >> 5) == 0) {  // warp 0 owns the whole TMEM of the SM (one CTA per SM)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
                     static_cast<unsigned>(__cvta_generic_to_shared(&s_taddr)))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const unsigned tbase = s_taddr + ((32u * ((tid >> 5) & 3)) << 16) + 128u * (tid >> 7);
  auto colR = [&](int r) { return tbase + 32u * r; };        // R_b = L_{b+1}' rows
  auto colL = [&](int r) { return tbase + 64u + 32u * r; };  // L_b rows
  // CTA-private slot (L2 resident): L and D (TMA-staged for the PCG phase),
  // theta^-1, gamma, R^-1
  const bool keep_q = p.dz_out != nullptr;
  T* gL = p.slot + static_cast<size_t>(blockIdx.x) * fused_slot_stride<T>(K, NB, MB, keep_q);
  T* gD = gL + static_cast<size_t>(K) * LS;
  T* gT = gD + static_cast<size_t>(K) * NN;
  T* gG = kGamS ? su : gT + static_cast<size_t>(K) * NN;  // gamma [K][NB]
  T* gR = gT + static_cast<size_t>(K) * (NN + NB);  // R_k^-1 [N][MB][MB]
  T* gQ = gR + static_cast<size_t>(K) * MB * MB;  // Q_k^-1 [K][NB][NB] (fused finish only)

  for (int sys = blockIdx.x; sys < p.B; sys += gridDim.x) {
    const int m = EXM ? MB : p.m_rt;  // control dimension of the input arrays
    const size_t nn = NN, nm = static_cast<size_t>(NB) * m, mm = MB * MB;  // mm: padded R^-1
    const T* Qs = p.Q + static_cast<size_t>(sys) * K * nn;
    const T* qs = p.q + static_cast<size_t>(sys) * K * NB;
    const T* Rs = p.R + static_cast<size_t>(sys) * N * m * m;
    const T* rs = p.r + static_cast<size_t>(sys) * N * m;
    const T* As = p.A + static_cast<size_t>(sys) * N * nn;
    const T* Bs = p.Bm + static_cast<size_t>(sys) * N * nm;
    const T* es = p.e + static_cast<size_t>(sys) * N * NB;
    const T* xs = p.x_s + static_cast<size_t>(sys) * NB;
    const T* x0 = p.x0 + static_cast<size_t>(sys) * NB;

    __syncthreads();  // previous system's PCG is done with shared memory
    unsigned long long* tm = (TM && p.timing && tid == 0) ? p.timing + static_cast<size_t>(sys) * 16 : nullptr;
    if (tm) tm[0] = gtimer();
    if (tid == 0) s_err = 0x7fffffff;

    int fkey = 0x7fffffff;

    // ============================================================ F1: knots
    // Q_k^-1 for every knot and R_k^-1 for k < N, computed once and shared
    // by the two block rows that use them (the reference recomputes them per
    // row, schur.cpp:49-51; same arithmetic). All Q_k arrive in one TMA bulk
    // copy (sQi) and are inverted in place; lanes read their rows from smem.
    T* sq = smem + FL::osq(KL);  // q_k of every knot (for Q_k^-1 q_k)
    if (mst & 4u) {
      mbar_wait_bit(mbar2_addr, mst, 2u);  // prefetched during the previous PCG
    } else {
      if (tid == 0) {
        const unsigned bq = static_cast<unsigned>(sizeof(T) * K * nn);
        const unsigned bv = static_cast<unsigned>(sizeof(T) * K * NB);
        asm volatile("fence.proxy.async;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mbar_addr),
                     "r"(bq + bv)
                     : "memory");
        tma_copy_1d(sQi, Qs, bq, mbar_addr);
        tma_copy_1d(sq, qs, bv, mbar_addr);
      }
      mbar_wait_bit(mbar_addr, mst, 1u);
    }
    mst &= ~4u;
    if (tm) tm[11] = gtimer();
    // 8-lane group g = tid / 8 inverts Q_g (lane gl < n/2 owns rows gl and
    // gl + n/2: every broadcast tile operand serves two rows) and then R_g,
    // all 64 knots in one pass. Groups past the horizon recompute a clamped
    // duplicate in their own tile and store nothing, so every shuffle and sync
    // is full-warp.
    {
      constexpr int H = NB / 2;
      const int g = tid >> 3, gl = tid & 7;
      const int glr = gl < H ? gl : H - 1;
      T* gt = smem + FL::ohw(KL) + static_cast<size_t>(g) * FL::g8_tile;
      const bool kv = g < K;
      const int kc = kv ? g : K - 1;
      // R_g row issued first: its L2 latency hides behind the Q_g inverse
      const bool rv = g < N;
      const int rc = rv ? g : N - 1;
      const int lm = gl < MB ? gl : MB - 1;
      T ra[MB];
      {
        const T* Rr = Rs + static_cast<size_t>(rc) * m * m + lm * m;
#pragma unroll
        for (int i = 0; i < MB; ++i)  // identity pad rows / columns past m
          ra[i] = (EXM || (lm < m && i < m)) ? __ldg(Rr + i) : (lm == i ? T(1) : T(0));
      }
      // r_g[gl] (for R_g^-1 r_g after the inverse; shuffled to the group then)
      const T rl = (gl < MB && (EXM || gl < m)) ? __ldg(rs + static_cast<size_t>(rc) * m + gl) : T(0);
      T a0[NB], a1[NB], x0[NB], x1[NB];
      // clamped duplicates read Q_{K-1} from global memory (its shared copy
      // is inverted in place by its owner)
      if (kv) {
        const T* Q0 = sQi + static_cast<size_t>(kc) * nn + glr * NB;
#pragma unroll
        for (int i = 0; i < NB; i += 2) {
          const double2 u = *reinterpret_cast<const double2*>(Q0 + i);
          const double2 v = *reinterpret_cast<const double2*>(Q0 + H * NB + i);
          a0[i] = u.x; a0[i + 1] = u.y; a1[i] = v.x; a1[i + 1] = v.y;
        }
      } else {
        const T* Q0 = Qs + static_cast<size_t>(kc) * nn + glr * NB;
#pragma unroll
        for (int i = 0; i < NB; i += 2) {
          const double2 u = __ldg(reinterpret_cast<const double2*>(Q0 + i));
          const double2 v = __ldg(reinterpret_cast<const double2*>(Q0 + H * NB + i));
          a0[i] = u.x; a0[i + 1] = u.y; a1[i] = v.x; a1[i + 1] = v.y;
        }
      }
      T* Lr = kv ? sQi + static_cast<size_t>(kc) * nn : gt;  // in place for owners
      const int f = g8x2_spd_inverse<T, NB>(a0, a1, Lr, gt, gt + FL::g8_tile - 16, gl, x0, x1);
      // first failing call in row order: row k as its Q_{k+1} (key 4k+2), or row 0
      if (kv && f >= 0) fkey = min(fkey, g == 0 ? 0 : 4 * g + 2);
      if (kv && gl < H) {
        // Q_g^-1 rows (bitwise symmetric: = columns, which F2 reads)
        T qq0 = T(0), qq1 = T(0);
        T* X0 = sQi + static_cast<size_t>(g) * NN + glr * NB;
#pragma unroll
        for (int i = 0; i < NB; i += 2) {
          *reinterpret_cast<double2*>(X0 + i) = make_double2(x0[i], x0[i + 1]);
          *reinterpret_cast<double2*>(X0 + H * NB + i) = make_double2(x1[i], x1[i + 1]);
        }
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          const T qi = sq[g * NB + i];
          qq0 += x0[i] * qi;
          qq1 += x1[i] * qi;
          if (keep_q) {
            gQ[static_cast<size_t>(g) * NN + glr * NB + i] = x0[i];
            gQ[static_cast<size_t>(g) * NN + (glr + H) * NB + i] = x1[i];
          }
        }
        sqq[g * 16 + glr] = qq0;
        sqq[g * 16 + glr + H] = qq1;
      }
      if (tm) tm[8] = gtimer();
      // R_g^-1 (m <= 8 rows, one per lane) in the group's tile (its L^-T is dead)
      static_assert(MB <= 8, "");
      T xr[MB];
      const int fr = g8_spd_inverse<T, MB>(ra, gt, gt + MB * MB, gt + FL::g8_tile - 16, gl, xr);
      if (rv && fr >= 0) fkey = min(fkey, 4 * (g + 1) + 1);
      T rsv[MB];
#pragma unroll
      for (int i = 0; i < MB; ++i) rsv[i] = __shfl_sync(FULL, rl, i, 8);
      if (rv && gl < MB) {
        T rr = T(0);
#pragma unroll
        for (int i = 0; i < MB; ++i) {
          gR[static_cast<size_t>(g) * mm + i * MB + gl] = xr[i];
          rr += xr[i] * rsv[i];
        }
        srr[g * 8 + gl] = rr;
      }
      if (tm) tm[9] = gtimer();
    }
    __syncthreads();

    if (tm) tm[1] = gtimer();
    // ============================================================ F2: rows
    // schur.cpp:58-78 on the FP64 tensor cores. Warp w forms rows b = w + 16 t
    // (one row at a time, warp-uniform): every block product is a chain of
    // mma.sync.m8n8k4.f64 over 16 x 16 tiles (n padded with zeros), k-steps in
    // ascending order. DMMA D = A B + C equals the scalar FMA chain from C over
    // k = 0..3 bitwise (scripts/micro/dmma_round.cu), so each element is the
    // same fma chain, in the same order, as the scalar row products — and as
    // the reference's dot products in order — with zero pads adding exact zeros.
    //   AQ = A_k Q_k^-1 (pad column NB of Q_k^-1 carries Q_k^-1 q_k, so column
    //   NB of AQ is A (Q^-1 q) for zeta), L_b = -AQ;
    //   BR = B_k R_k^-1 (pad column MB carries R_k^-1 r_k: B (R^-1 r));
    //   theta_raw = (AQ A' + BR B') + Q_{k+1}^-1, theta = (theta_raw + theta_raw')/2;
    //   gamma_b = e_k - zeta.
    // The warp's tile (stride 20: the A-fragment reads are conflict-free) moves
    // accumulator fragments into A-operand fragments and transposes theta_raw.
    {
      constexpr bool PADQ = NB < 16, PADR = MB < 8;
      const int w = tid >> 5, fr = lane >> 2, fc = lane & 3;
      // global operand fragments of row bb (A, B from L2, R_k^-1 from the
      // slot, e_k), fetched one row ahead: their L2 latency overlaps the
      // previous row's tensor-core chains. A (row r, col c), B (row c, col r).
      auto fetch = [&](int bb, T (&af)[2][4], T (&bf)[2][2], T (&rf)[2], T (&ek)[2]) {
        const bool lv = bb >= 1 && bb < K;
        const int k = lv ? bb - 1 : 0;
        const T* Ak = As + static_cast<size_t>(k) * nn;
        const T* Bk = Bs + static_cast<size_t>(k) * nm;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const int i = mt * 8 + fr;
          // e_k rows for gamma (lane (r, 0) owns rows r and r + 8)
          ek[mt] = (lv && fc == 0 && i < NB) ? __ldg(es + k * NB + i) : T(0);
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const int q = ks * 4 + fc;
            af[mt][ks] = (lv && i < NB && q < NB) ? __ldg(Ak + i * NB + q) : T(0);
          }
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            const int q = ks * 4 + fc;
            bf[mt][ks] = (lv && i < NB && q < m && (EXM || q < MB)) ? __ldg(Bk + i * m + q) : T(0);
          }
        }
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const int sr = ks * 4 + fc;
          T v = T(0);
          if (lv && sr < MB)
            v = fr < MB ? __ldcg(gR + static_cast<size_t>(k) * mm + sr * MB + fr)
                        : ((PADR && fr == MB) ? srr[k * 8 + sr] : T(0));
          rf[ks] = v;
        }
      };
      T afn[2][4], bfn[2][2], rfn[2], ekn[2];
      fetch(w, afn, bfn, rfn, ekn);
#pragma unroll 1
      for (int t = 0; t < 4; ++t) {
        const int b = w + 16 * t;
        const bool live = b >= 1 && b < K;  // warp-uniform
        T af[2][4], bf[2][2], rf[2], ek[2];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          ek[mt] = ekn[mt];
          rf[mt] = rfn[mt];
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) af[mt][ks] = afn[mt][ks];
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) bf[mt][ks] = bfn[mt][ks];
        }
        if (t < 3) fetch(b + 16, afn, bfn, rfn, ekn);
        if (b == 0) {
          // schur.cpp:53-57: S(0,0) = D_0 = Q_0^-1, theta_inv[0] = sym(Q_0), gamma_0
          if (lane < NB) {
            const T g0 = -((xs[lane] - x0[lane]) + sqq[lane]);
            gG[lane] = g0;
            if (p.form_only) p.gamma_out[static_cast<size_t>(sys) * K * NB + lane] = g0;
#pragma unroll
            for (int j = 0; j < NB; ++j) {
              const T d = sQi[lane * NB + j];
              smem[FL::oD(KL) + lane * NB + j] = d;  // D_0 in place for the PCG
              if (p.form_only) {
                p.S_out[static_cast<size_t>(sys) * K * 3 * nn + nn + lane * NB + j] = d;
                p.theta_out[static_cast<size_t>(sys) * K * nn + lane * NB + j] =
                    T(0.5) * (Qs[lane * NB + j] + Qs[j * NB + lane]);
              }
            }
          }
        }
        if (live) {
          const int k = b - 1;
          const T* Ak = As + static_cast<size_t>(k) * nn;
          const T* Bk = Bs + static_cast<size_t>(k) * nm;
          const T* Xk = sQi + static_cast<size_t>(k) * NN;
          const T* Xk1 = Xk + NN;
          // Q_k^-1 fragments (B operand, row q, col j) from shared memory; pad
          // column NB carries Q_k^-1 q_k (one predicated load, no branches)
          T xf[2][4];
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            const int j = nt * 8 + fr;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
              const int q = ks * 4 + fc;
              const T* src = j < NB ? Xk + q * NB + j : sqq + k * 16 + q;
              const bool ok = q < NB && (j < NB || (PADQ && j == NB));
              xf[nt][ks] = ok ? *src : T(0);
            }
          }
          // AQ (16 DMMA)
          T aq[2][2][2];
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
              aq[mt][nt][0] = aq[mt][nt][1] = T(0);
#pragma unroll
              for (int ks = 0; ks < 4; ++ks) dmma_f64(aq[mt][nt][0], aq[mt][nt][1], af[mt][ks], xf[nt][ks]);
            }
          // BR (4 DMMA), cols 0..7
          T br[2][2];
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            br[mt][0] = br[mt][1] = T(0);
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) dmma_f64(br[mt][0], br[mt][1], bf[mt][ks], rf[ks]);
          }
          // L_b = -AQ -> slot (padded stride LS) and, for build_schur, S.left(b) / S.right(b-1)
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
              const int i = mt * 8 + fr, j = nt * 8 + 2 * fc;
              if (i < NB && j < NB) {
                *reinterpret_cast<double2*>(gL + static_cast<size_t>(b) * LS + i * NB + j) =
                    make_double2(-aq[mt][nt][0], -aq[mt][nt][1]);
                if (p.form_only) {
                  T* Sl = p.S_out + (static_cast<size_t>(sys) * K + b) * 3 * nn;
                  T* Sr = p.S_out + ((static_cast<size_t>(sys) * K + b - 1) * 3 + 2) * nn;
                  Sl[i * NB + j] = -aq[mt][nt][0];
                  Sl[i * NB + j + 1] = -aq[mt][nt][1];
                  Sr[j * NB + i] = -aq[mt][nt][0];
                  Sr[(j + 1) * NB + i] = -aq[mt][nt][1];
                }
              }
            }
          // zeta_i = (-A(Q^-1 q) - B(R^-1 r)) + Q_{k+1}^-1 q_{k+1}; gamma_b = e_k - zeta
          // (the pad columns NB of AQ and MB of BR sit in lanes (r, NB%8/2) and
          // (r, MB/2); lane (r, 0) gathers them)
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            const int i = mt * 8 + fr;
            T aqq = T(0), brr = T(0);
            if constexpr (PADQ) aqq = __shfl_sync(FULL, aq[mt][NB / 8][(NB % 8) & 1], fr * 4 + (NB % 8) / 2);
            if constexpr (PADR) brr = __shfl_sync(FULL, br[mt][MB & 1], fr * 4 + MB / 2);
            if (fc == 0 && i < NB) {
              if constexpr (!PADQ) {
#pragma unroll
                for (int q = 0; q < NB; ++q) aqq += __ldg(Ak + i * NB + q) * sqq[k * 16 + q];
              }
              if constexpr (!PADR) {
#pragma unroll
                for (int q = 0; q < MB; ++q)
                  brr += ((EXM || q < m) ? __ldg(Bk + i * m + q) : T(0)) * srr[k * 8 + q];
              }
              const T zeta = (-aqq - brr) + sqq[(k + 1) * 16 + i];
              const T g = -(-ek[mt] + zeta);
              gG[static_cast<size_t>(b) * NB + i] = g;
              if (p.form_only) p.gamma_out[(static_cast<size_t>(sys) * K + b) * NB + i] = g;
            }
          }
          // accumulator fragment (row r, cols 2c, 2c+1 of a tile) -> A-operand
          // fragment (row r, col c of a k-step): quad shuffles
          auto to_a = [&](const T (&d)[2], int col) {  // col: column inside the 8-wide tile
            const int src = fr * 4 + (col >> 1);
            const T v0 = __shfl_sync(FULL, d[0], src), v1 = __shfl_sync(FULL, d[1], src);
            return (col & 1) ? v1 : v0;
          };
          // AQ as A operand (pad columns zeroed: no leak of the zeta column)
          T aqa[2][4];
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
              const T v = to_a(aq[mt][ks >> 1], (ks & 1) * 4 + fc);
              aqa[mt][ks] = ks * 4 + fc < NB ? v : T(0);
            }
          // theta_A = AQ A' (16 DMMA): B operand (row q, col j) = A[j][q] = af
          T ta[2][2][2];
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
              ta[mt][nt][0] = ta[mt][nt][1] = T(0);
#pragma unroll
              for (int ks = 0; ks < 4; ++ks) dmma_f64(ta[mt][nt][0], ta[mt][nt][1], aqa[mt][ks], af[nt][ks]);
            }
          T bra[2][2];
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
              const T v = to_a(br[mt], ks * 4 + fc);
              bra[mt][ks] = ks * 4 + fc < MB ? v : T(0);
            }
          // theta_raw = (AQ A' + BR B') + Q_{k+1}^-1 (schur.cpp:65-66)
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
              T s0 = T(0), s1 = T(0);
#pragma unroll
              for (int ks = 0; ks < 2; ++ks) dmma_f64(s0, s1, bra[mt][ks], bf[nt][ks]);
              const int i = mt * 8 + fr, j = nt * 8 + 2 * fc;
              double2 x1 = make_double2(0.0, 0.0);
              if (i < NB && j < NB) x1 = *reinterpret_cast<const double2*>(Xk1 + i * NB + j);
              ta[mt][nt][0] = (ta[mt][nt][0] + s0) + x1.x;
              ta[mt][nt][1] = (ta[mt][nt][1] + s1) + x1.y;
            }
          // theta = (theta_raw + theta_raw')/2 (schur.cpp:67): the transposed
          // element (j, i) of lane (r, c)'s (i, j) = (8 mt + r, 8 nt + 2c + e)
          // sits in lane (2c + e, r / 2), tile (nt, mt), element r & 1
          T* thb = smem + FL::oD(KL) + static_cast<size_t>(b) * NN;  // = the PCG's D_b
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
              const int i = mt * 8 + fr, j = nt * 8 + 2 * fc;
              T tr[2];
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int src = (2 * fc + e) * 4 + (fr >> 1);
                const T v0 = __shfl_sync(FULL, ta[nt][mt][0], src), v1 = __shfl_sync(FULL, ta[nt][mt][1], src);
                tr[e] = (fr & 1) ? v1 : v0;
              }
              const T t0 = T(0.5) * (ta[mt][nt][0] + tr[0]);
              const T t1 = T(0.5) * (ta[mt][nt][1] + tr[1]);
              if (i < NB && j < NB) {
                // theta_b rows for the theta^-1 pass (shared memory)
                *reinterpret_cast<double2*>(thb + i * NB + j) = make_double2(t0, t1);
                if (p.form_only) {
                  T* Sd = p.S_out + ((static_cast<size_t>(sys) * K + b) * 3 + 1) * nn;
                  Sd[i * NB + j] = t0;
                  Sd[i * NB + j + 1] = t1;
                }
              }
            }
          __syncwarp();
        }
      }
    }
    // ===================================================== theta^-1 (schur.cpp:75)
    // One pass over all rows on 8-lane groups: group b = tid / 8, lane gl owns
    // rows gl and gl + n/2 — exactly the PCG's quarter-warp mapping, so the
    // inverse's output rows ARE the PCG thread's theta_b^-1 register rows
    // (no slot round trip). theta_b is read from the lower triangle F2 left in
    // shared memory.
    __syncthreads();  // every theta_b is in place
    if (tm) tm[10] = gtimer();
    // warps wholly past the horizon skip the pass (their PCG rows are discarded)
    if (4 * (tid >> 5) < K) {
      constexpr int H = NB / 2;
      const int b = tid >> 3, gl = tid & 7;
      const int glr = gl < H ? gl : H - 1;
      // row 0 and the horizon warp's rows past K invert a clamped theta (row
      // 1 / K-1) in their own tile and keep nothing: convergent full-warp syncs
      // (their tiles, b < K + 3, stay clear of the theta triangles)
      const int bi = b == 0 ? 1 : (b < K ? b : K - 1);
      T* gt = smem + static_cast<size_t>(b) * FL::g8_tile;  // sQi region (dead)
      T a0[NB], a1[NB];
      const T* Th = smem + FL::oD(KL) + static_cast<size_t>(bi) * NN + glr * NB;
#pragma unroll
      for (int i = 0; i < NB; i += 2) {
        const double2 u = *reinterpret_cast<const double2*>(Th + i);
        const double2 v = *reinterpret_cast<const double2*>(Th + H * NB + i);
        a0[i] = u.x; a0[i + 1] = u.y; a1[i] = v.x; a1[i + 1] = v.y;
      }
      T x0[NB], x1[NB];
      if (tm) tm[13] = gtimer();
      const int f = g8x2_spd_inverse<T, NB>(a0, a1, gt, gt, gt + FL::g8_tile - 16, gl, x0, x1);
      if (tm) tm[14] = gtimer();
      if (b >= 1 && b < K && f >= 0) fkey = min(fkey, b * 4 + 3);
      // (row 0's theta_inv[0] = sym(Q_0) is read by the PCG stage itself)
      if (p.form_only && b >= 1 && b < K && gl < H) {  // theta_inv[b] rows
        T* To = p.theta_out + (static_cast<size_t>(sys) * K + b) * nn;
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          To[glr * NB + j] = x0[j];
          To[(glr + H) * NB + j] = x1[j];
        }
      }
      // the rows stay in the group's (now free) tile until the PCG stage loads
      // them into the same thread's registers
      if (gl < H) {
#pragma unroll
        for (int j = 0; j < NB; j += 2) {
          *reinterpret_cast<double2*>(gt + glr * NB + j) = make_double2(x0[j], x0[j + 1]);
          *reinterpret_cast<double2*>(gt + (glr + H) * NB + j) = make_double2(x1[j], x1[j + 1]);
        }
      }
    }
    if (tm) tm[12] = gtimer();
    // F2's global writes (L, D, gamma) are read back by the async proxy (TMA)
    // below: order them before the barrier
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
    if (tm) tm[2] = gtimer();
    // every failure key is 8-lane-group uniform (F1, theta^-1): each group's
    // first lane reports
    if ((l & 7) == 0 && fkey != 0x7fffffff) atomicMin(&s_err, fkey);
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
    if (p.form_only) continue;  // build_schur only

    // ================================================================ P
    // PCG mapping: warp w owns block rows 4w..4w+3, one per quarter-warp; lane
    // i < 7 of a quarter-warp owns scalar rows i and i + 7 of its block, so
    // every broadcast operand vector serves two output rows. D_b and L_b rows
    // live in TMEM, L (for the column products R_b = L_{b+1}') in shared memory,
    // theta_b^-1 rows in registers.
    const int pq = lane >> 3;  // quarter-warp
    const int pi = lane & 7;   // row pair (pi, pi + 7); lane 7 of each quarter idles
    const int pb = 4 * (tid >> 5) + pq;
    const bool pact = pi < H && pb < K;
    const int pbc = pb < K ? pb : K - 1;            // clamped block row
    const int pbl = pbc > 0 ? pbc - 1 : 0;          // neighbours, clamped into [0, K):
    const int pbn = pbc + 1 < K ? pbc + 1 : K - 1;  // edge products are discarded
    const int pr = pi < H ? pi : H - 1;             // clamped row (idle lanes)
    // theta_b^-1 rows pr, pr + n/2: the thread's own group tile (theta^-1 pass),
    // read before the staging copies overwrite the tiles
    T ti[2][NB];
    {
      const T* tt = smem + static_cast<size_t>(pb) * FL::g8_tile + pr * NB;
#pragma unroll
      for (int j = 0; j < NB; j += 2) {
        const double2 u = 4 * (tid >> 5) < K ? *reinterpret_cast<const double2*>(tt + j) : make_double2(0.0, 0.0);
        const double2 v = 4 * (tid >> 5) < K ? *reinterpret_cast<const double2*>(tt + H * NB + j) : make_double2(0.0, 0.0);
        ti[0][j] = u.x; ti[0][j + 1] = u.y; ti[1][j] = v.x; ti[1][j + 1] = v.y;
      }
    }
    __syncthreads();
    {
      // stage L from the slot (one TMA bulk copy), then every thread moves its
      // L_b rows and R_b = L_{b+1}' rows into its TMEM lane
      const unsigned bl = static_cast<unsigned>(sizeof(T) * K * LS);
      if (tid == 0) {
        asm volatile("fence.proxy.async;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mbar_addr),
                     "r"(bl)
                     : "memory");
        tma_copy_1d(sL, gL, bl, mbar_addr);
      }
    }
    if (pb == 0) {  // theta_inv[0] = sym(Q_0), not an inverse (schur.cpp:55)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int row = pr + H * c;
#pragma unroll
        for (int j = 0; j < NB; ++j) ti[c][j] = T(0.5) * (__ldg(Qs + row * NB + j) + __ldg(Qs + j * NB + row));
      }
    }
    T lam[2], rr[2], rt[2], pp[2], spv[2], best[2], gam[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int row = pr + H * c;
      gam[c] = kGamS ? gG[pbc * NB + row] : __ldcg(gG + pbc * NB + row);
      lam[c] = (pact && p.lambda0) ? p.lambda0[static_cast<size_t>(sys) * K * NB + pbc * NB + row]
                                   : T(0);
    }
    mbar_wait_bit(mbar_addr, mst, 1u);
    {
      T mrow[NB];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        // row pr + H c of R_b = column pr + H c of L_{b+1} (padded stride LS:
        // the four quarter-warps read disjoint banks)
        // (the missing neighbour blocks — L_0, R_{K-1} — are stored as exact
        // zeros, so the block products need no edge selects)
        const T* Lc = sL + static_cast<size_t>(pbn) * LS + pr + H * c;
        const bool rz = pbc + 1 >= K, lz = pbc == 0;
#pragma unroll
        for (int j = 0; j < NB; ++j) mrow[j] = rz ? T(0) : Lc[j * NB];
        tm::st_row<NB>(colR(c), mrow);
        const T* Lr = sL + static_cast<size_t>(pbc) * LS + (pr + H * c) * NB;
#pragma unroll
        for (int j = 0; j < NB; j += 2) {
          const double2 v = *reinterpret_cast<const double2*>(Lr + j);
          mrow[j] = lz ? T(0) : v.x;
          mrow[j + 1] = lz ? T(0) : v.y;
        }
        tm::st_row<NB>(colL(c), mrow);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    }
#pragma unroll
    for (int c = 0; c < 2; ++c)
      if (pact) sp[pbc * NB + pi + H * c] = lam[c];
    __syncthreads();  // sL consumed: the next system's Q may land in [0, K*NN)
    if (tm) tm[3] = gtimer();
    {
      const int nsys = sys + gridDim.x;
      if (nsys < p.B) {  // next system's Q_k, q_k straight into the formation's regions
        if (tid == 0) {
          const unsigned bq = static_cast<unsigned>(sizeof(T) * K * nn);
          const unsigned bv = static_cast<unsigned>(sizeof(T) * K * NB);
          asm volatile("fence.proxy.async;\n" ::: "memory");
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mbar2_addr),
                       "r"(bq + bv)
                       : "memory");
          tma_copy_1d(sQi, p.Q + static_cast<size_t>(nsys) * K * nn, bq, mbar2_addr);
          tma_copy_1d(smem + FL::osq(KL), p.q + static_cast<size_t>(nsys) * K * NB, bv, mbar2_addr);
        }
        mst |= 4u;
      }
      if (nsys < p.B && tid < 9) {
        // per-field contiguous ranges of the next system (16-byte aligned inside)
        // (a switch, not an indexed array: no local-memory copy of the table)
        const T* base;
        size_t per;
        switch (tid) {
          case 0: base = p.Q; per = static_cast<size_t>(K) * NN; break;
          case 1: base = p.q; per = static_cast<size_t>(K) * NB; break;
          case 2: base = p.R; per = static_cast<size_t>(N) * m * m; break;
          case 3: base = p.r; per = static_cast<size_t>(N) * m; break;
          case 4: base = p.A; per = static_cast<size_t>(N) * NN; break;
          case 5: base = p.Bm; per = static_cast<size_t>(N) * NB * m; break;
          case 6: base = p.e; per = static_cast<size_t>(N) * NB; break;
          case 7: base = p.x_s; per = NB; break;
          default: base = p.x0; per = NB; break;
        }
        const char* lo = reinterpret_cast<const char*>(base + nsys * per);
        const char* hi = lo + per * sizeof(T);
        const char* a = reinterpret_cast<const char*>((reinterpret_cast<uintptr_t>(lo) + 15) & ~uintptr_t(15));
        const char* e = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(hi) & ~uintptr_t(15));
        if (e > a)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a),
                       "r"(static_cast<unsigned>(e - a))
                       : "memory");
      }
    }

    // y_c = ((D x_b + L x_{b-1}) + R x_{b+1}) for the thread's rows pi, pi + 7,
    // R_b = L_{b+1}' (block_tri.cpp:82-92). Out-of-range neighbours are computed
    // on in-bounds shared memory and discarded by the selects.
    auto Srows = [&](const T* x, T (&y)[2]) {
      T sd[2], sl[2], sr[2];
      dots_row2<T, NB>(sD + static_cast<size_t>(pbc) * NN + pr * NB, x + pbc * NB, sd);  // D_b rows (smem)
      tm::dot2_row<NB>(colL(0), colL(1), x + pbl * NB, sl[0], sl[1]);  // L_b rows (TMEM)
      tm::dot2_row<NB>(colR(0), colR(1), x + pbn * NB, sr[0], sr[1]);  // R_b rows (TMEM)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        T out = sd[c];
        out += sl[c];  // L_0 and R_{K-1} rows are exact zeros in TMEM
        out += sr[c];
        y[c] = out;
      }
    };

    // r = gamma - S lambda0 (pcg.cpp:62)
    __syncthreads();
    {
      T sl0[2];
      if (p.lambda0) Srows(sp, sl0);
#pragma unroll
      for (int c = 0; c < 2; ++c) rr[c] = gam[c] - (p.lambda0 ? sl0[c] : T(0));
    }
    // r~ = Phi^-1 r, for every kind
    const bool corr_row = (p.kind == kSymStair) || (pbc & 1);
    // the same-block products read su; quarter-warps past the horizon (pb >= K,
    // results discarded) read sp instead: their clamped block is another
    // warp's, whose su writes are only __syncwarp-ordered, while sp is
    // barrier-ordered here
    const T* sown = pb < K ? su : sp;
    auto precondition = [&]() {
      if (p.kind == kIdentity) {
#pragma unroll
        for (int c = 0; c < 2; ++c) rt[c] = rr[c];
        return;
      }
      T tv[2];
#pragma unroll
      for (int c = 0; c < 2; ++c)
        if (pact) su[pbc * NB + pi + H * c] = rr[c];
      __syncwarp();
      dots_reg2<T, NB>(ti, sown + pbc * NB, tv);  // t = theta^-1 r
      if (p.kind == kJacobi) {
#pragma unroll
        for (int c = 0; c < 2; ++c) rt[c] = tv[c];
        return;
      }
#pragma unroll
      for (int c = 0; c < 2; ++c)
        if (pact) st[pbc * NB + pi + H * c] = tv[c];
      __syncthreads();
      // u = r - L_b t_{b-1} - R_b t_{b+1}
      T sl[2], sr[2];
      tm::dot2_row<NB>(colL(0), colL(1), st + pbl * NB, sl[0], sl[1]);
      tm::dot2_row<NB>(colR(0), colR(1), st + pbn * NB, sr[0], sr[1]);
      __syncwarp();  // every lane has read its block's r from su
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        T v = rr[c];
        v -= sl[c];
        v -= sr[c];
        if (pact) su[pbc * NB + pi + H * c] = v;
      }
      __syncwarp();
      T uv[2];
      dots_reg2<T, NB>(ti, sown + pbc * NB, uv);  // theta^-1 u
#pragma unroll
      for (int c = 0; c < 2; ++c) rt[c] = corr_row ? uv[c] : tv[c];
    };
    precondition();
    T eta_part = T(0);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      pp[c] = rt[c];
      if (pact) eta_part += rr[c] * rt[c];
      best[c] = lam[c];
    }
    T eta = block_reduce(eta_part, red);

    int code = kOk, which = kWhichNone, err_iter = -1, iterations = 0, converged = 0;
    double exit_eta = static_cast<double>(eta), value = 0.0;
    T best_eta = eta;
    double* trace = p.trace ? p.trace + static_cast<size_t>(sys) * p.trace_cap : nullptr;
    if (!is_finite(eta)) {
      code = kRuntime;
      which = kWhichInitNonFinite;
    } else if (static_cast<double>(eta) < p.epsilon) {
      converged = 1;
    } else {
#pragma unroll
      for (int c = 0; c < 2; ++c)
        if (pact) sp[pbc * NB + pi + H * c] = pp[c];
      __syncthreads();
      // B2P_PHASE_TIMING: per-segment SM-clock sums of thread 0 over the
      // iterations (Srows | upsilon reduce | update + precondition | eta
      // reduce | beta + p + barrier), packed two per stamp slot 5..7
      // (sums in shared memory: no registers or local memory in the solve path)
      __shared__ unsigned s_seg[6];
      if (tm) {
#pragma unroll
        for (int i = 0; i < 5; ++i) s_seg[i] = 0u;
        s_seg[5] = static_cast<unsigned>(clock());
      }
      auto segmark = [&](int i) {
        if (tm) {
          const unsigned c1 = static_cast<unsigned>(clock());
          s_seg[i] += c1 - s_seg[5];
          s_seg[5] = c1;
        }
      };
      for (int it = 1; it <= p.max_iter; ++it) {
        T up = T(0);
        Srows(sp, spv);
#pragma unroll
        for (int c = 0; c < 2; ++c)
          if (pact) up += pp[c] * spv[c];
        segmark(0);
        const T ups = block_reduce(up, red + 16);  // buffer B
        segmark(1);
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
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          rr[c] -= alpha * spv[c];
          lam[c] += alpha * pp[c];
        }
        precondition();
        T ep = T(0);
#pragma unroll
        for (int c = 0; c < 2; ++c)
          if (pact) ep += rr[c] * rt[c];
        segmark(2);
        const T eta_p = block_reduce(ep, red);
        segmark(3);
        if (!is_finite(eta_p)) {
          code = kRuntime;
          which = kWhichEtaNonFinite;
          err_iter = it;
          break;
        }
        if (trace && tid == 0) trace[it - 1] = static_cast<double>(eta_p);
        if (eta_p < best_eta) {
          best_eta = eta_p;
#pragma unroll
          for (int c = 0; c < 2; ++c) best[c] = lam[c];
        }
        iterations = it;
        exit_eta = static_cast<double>(eta_p);
        if (static_cast<double>(eta_p) < p.epsilon) {
          converged = 1;
          break;
        }
        if (it == p.max_iter) break;
        const T beta = eta_p / eta;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          pp[c] = rt[c] + beta * pp[c];
          if (pact) sp[pbc * NB + pi + H * c] = pp[c];
        }
        eta = eta_p;
        __syncthreads();
        segmark(4);
      }
      if (tm) {
        tm[5] = s_seg[0] | (static_cast<unsigned long long>(s_seg[1]) << 32);
        tm[6] = s_seg[2] | (static_cast<unsigned long long>(s_seg[3]) << 32);
        tm[7] = s_seg[4];
      }
    }
    if (code == kOk) {
#pragma unroll
      for (int c = 0; c < 2; ++c)
        if (pact)
          p.lambda_out[static_cast<size_t>(sys) * K * NB + pbc * NB + pi + H * c] =
              converged ? lam[c] : best[c];
    }
    if (keep_q && code == kOk) {
      // The PPCG finish (reconstruct_primal, kkt.cpp:153-181)
      // on the formation's Q_k^-1 / R_k^-1 (slot, L2) and this solve's lambda:
      // half-warp h takes knots h, h + 32, lane i = row i,
      //   dx_k = Q_k^-1 (-((q_k + lambda_k) - A_k' lambda_{k+1})),
      //   du_k = R_k^-1 (-(r_k - B_k' lambda_{k+1})), dx_N = Q_N^-1 (-(q_N + lambda_N)).
      __syncthreads();  // lambda (global) complete; sD is dead (sL may hold the next Q)
      const T* lamo = p.lambda_out + static_cast<size_t>(sys) * K * NB;
      T* dz = p.dz_out + static_cast<size_t>(sys) * (static_cast<size_t>(K) * NB + static_cast<size_t>(N) * m);
      T* W = sD + h * 32;  // this half-warp's right-hand sides
#pragma unroll 1
      for (int r = 0; r < R; ++r) {
        const int k = h + r * kHalfWarps;
        const bool kv = k < K;
        if (kv && lact) {
          T at = T(0);
          if (k < N) {
#pragma unroll
            for (int j = 0; j < NB; ++j) at += __ldg(As + static_cast<size_t>(k) * nn + j * NB + l) * lamo[(k + 1) * NB + j];
          }
          const T qk = __ldg(qs + k * NB + l) + lamo[k * NB + l];
          W[l] = k < N ? -(qk - at) : -qk;
        }
        if (kv && k < N && l < MB) {  // pad entries: exact zeros
          T bt = T(0);
          if (EXM || l < m) {
#pragma unroll
            for (int j = 0; j < NB; ++j) bt += __ldg(Bs + static_cast<size_t>(k) * nm + j * m + l) * lamo[(k + 1) * NB + j];
          }
          W[16 + l] = (EXM || l < m) ? -(__ldg(rs + k * m + l) - bt) : T(0);
        }
        __syncwarp();
        if (kv && lact) {
          T sx = T(0);
#pragma unroll
          for (int j = 0; j < NB; ++j) sx += __ldcg(gQ + static_cast<size_t>(k) * NN + j * NB + l) * W[j];
          dz[static_cast<size_t>(k) * (NB + m) + l] = sx;
        }
        if (kv && k < N && l < m) {
          T su2 = T(0);
#pragma unroll
          for (int j = 0; j < MB; ++j) su2 += __ldcg(gR + static_cast<size_t>(k) * mm + j * MB + l) * W[16 + j];
          dz[static_cast<size_t>(k) * (NB + m) + NB + l] = su2;
        }
        __syncwarp();
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
      if (tm) tm[4] = gtimer();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if ((tid >> 5) == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(s_taddr) : "memory");
}

template <class T, int NB, int MB>
size_t fused_smem_bytes(int K) {  // the layout of the instantiation K launches
  using FL = FLayout<T, NB, MB>;
  return sizeof(T) * FL::elems(FL::kcap(K <= kHalfWarps ? 1 : 2));
}

// (n, m) -> the compiled shape: (14, 7) exactly (the BASELINE iiwa shape),
// else even n in [8, 16] with m <= 8 padded to MB = 4 or 8 (runtime m).
template <class F>
bool with_fused_shape(int n, int m, F&& f) {
  using std::integral_constant;
  if (n == 14 && m == 7) return f(integral_constant<int, 14>{}, integral_constant<int, 7>{}, std::true_type{});
  if (m < 1 || m > 8) return false;
  const bool m4 = m <= 4;
  switch (n) {
    case 8: return m4 ? f(integral_constant<int, 8>{}, integral_constant<int, 4>{}, std::false_type{})
                      : f(integral_constant<int, 8>{}, integral_constant<int, 8>{}, std::false_type{});
    case 10: return m4 ? f(integral_constant<int, 10>{}, integral_constant<int, 4>{}, std::false_type{})
                       : f(integral_constant<int, 10>{}, integral_constant<int, 8>{}, std::false_type{});
    case 12: return m4 ? f(integral_constant<int, 12>{}, integral_constant<int, 4>{}, std::false_type{})
                       : f(integral_constant<int, 12>{}, integral_constant<int, 8>{}, std::false_type{});
    case 14: return m4 ? f(integral_constant<int, 14>{}, integral_constant<int, 4>{}, std::false_type{})
                       : f(integral_constant<int, 14>{}, integral_constant<int, 8>{}, std::false_type{});
    case 16: return m4 ? f(integral_constant<int, 16>{}, integral_constant<int, 4>{}, std::false_type{})
                       : f(integral_constant<int, 16>{}, integral_constant<int, 8>{}, std::false_type{});
  }
  return false;
}

template <class T>
bool fused_supported(int K, int n, int m, int kind) {
  if (sizeof(T) != 8) return false;
  if (kind == kPoly) return false;
  if (K < 2 || K > 2 * kHalfWarps) return false;
  return with_fused_shape(n, m, [&](auto nb, auto mb, auto) {
    constexpr int NB = decltype(nb)::value, MB = decltype(mb)::value;
    using FL = FLayout<T, NB, MB>;
    return K <= FL::kcap(K <= kHalfWarps ? 1 : 2);
  });
}

template <class T>
size_t fused_slot_elems(int K, int n, int m, bool keep_q) {
  int MB = m;
  with_fused_shape(n, m, [&](auto, auto mb, auto) {
    MB = decltype(mb)::value;
    return true;
  });
  return fused_slot_stride<T>(K, n, MB, keep_q);
}

template <class T>
bool fused_supported_dz(int K, int n, int m, int kind) {
  return fused_supported<T>(K, n, m, kind);
}

template <class T>
cudaError_t launch_fused(const FusedParams<T>& p, int n, int m, int grid, cudaStream_t st) {
  if constexpr (sizeof(T) == 8) {
    cudaError_t err = cudaErrorNotSupported;
    FusedParams<T> q = p;
    q.m_rt = m;
    with_fused_shape(n, m, [&](auto nb, auto mb, auto exm) {
      constexpr int NB = decltype(nb)::value, MB = decltype(mb)::value;
      constexpr bool EXM = decltype(exm)::value;
      const size_t smem = fused_smem_bytes<T, NB, MB>(q.K);
      auto kern = q.timing ? (q.K <= kHalfWarps ? k_fused_cta<T, NB, MB, 1, EXM, true>
                                                : k_fused_cta<T, NB, MB, 2, EXM, true>)
                           : (q.K <= kHalfWarps ? k_fused_cta<T, NB, MB, 1, EXM, false>
                                                : k_fused_cta<T, NB, MB, 2, EXM, false>);
      err = ensure_max_smem(kern, smem);
      if (err == cudaSuccess) {
        kern<<<grid, kThreads, smem, st>>>(q);
        err = cudaGetLastError();
      }
      return true;
    });
    return err;
  } else {
    return cudaErrorNotSupported;
  }
}

template bool fused_supported<double>(int, int, int, int);
template bool fused_supported<float>(int, int, int, int);
template size_t fused_slot_elems<double>(int, int, int, bool);
template size_t fused_slot_elems<float>(int, int, int, bool);
template bool fused_supported_dz<double>(int, int, int, int);
template bool fused_supported_dz<float>(int, int, int, int);
template cudaError_t launch_fused<double>(const FusedParams<double>&, int, int, int, cudaStream_t);
template cudaError_t launch_fused<float>(const FusedParams<float>&, int, int, int, cudaStream_t);

}  // namespace b2p
