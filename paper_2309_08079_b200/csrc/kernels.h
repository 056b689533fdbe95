// Kernel parameter blocks and launchers (host <-> device boundary inside the
// library; the public C-ABI is include/b2p.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"

namespace b2p {

template <class T>
struct FormParams {
  int B, N, n, m;
  const T *Q, *q, *R, *r, *A, *Bm, *e, *x_s, *x0;  // [B][...] contiguous (b2p_kkt layout)
  T* S;          // [B][K][3][n][n]
  T* gamma;      // [B][K*n]
  T* theta_inv;  // [B][K][n][n]
  int* errkey;   // [B], INT_MAX = ok; else row*4 + call (see k_build_schur)
};

template <class T>
struct PrecondParams {
  int B, K, nb, kind;
  const T* S;
  const T* theta_inv;
  T* phi;
};

enum : int { kModeExplicit = 0, kModeFused = 1 };
enum : int { kSyncCta = 0, kSyncCluster = 1, kSyncGrid = 2 };

template <class T>
struct PcgParams {
  int B, K, nb;
  int G;         // CTAs per system
  int rows_per;  // block rows owned per CTA
  int kind, order;
  int mode;   // kModeExplicit (user Phi) | kModeFused (theta_inv, Phi applied on the fly)
  int stage;  // 1: copy the CTA's matrix rows into shared memory once
  int sync;   // kSyncCta | kSyncCluster | kSyncGrid
  int nthreads;
  const T* S;        // [B][K][3][nb][nb]
  const T* Phi;      // explicit: [B][K][3][nb][nb]
  const T* Tinv;     // fused: [B][K][nb][nb]
  const T* gamma;    // [B][D]
  const T* lambda0;  // [B][D] or null (=> 0)
  T* lambda_out;     // [B][D]
  T* best;           // workspace [B][D]
  T* pub;            // workspace [B][D]  (p exchange between CTAs)
  T* slots;          // workspace [B][2][G]
  const int* errkey; // [B] formation status or null
  SysOut* out;       // [B]
  double* trace;     // [B][trace_cap] or null
  int trace_cap;
  double epsilon;
  int max_iter;
  int check_drift;
  unsigned* gbar;  // kSyncGrid barrier counter (zeroed before the launch)
};

// Fused persistent K1+K3 (one CTA per system; fused_kernels.cu).
template <class T>
struct FusedParams {
  int B, K, kind;
  const T *Q, *q, *R, *r, *A, *Bm, *e, *x_s, *x0;  // [B][...] b2p_kkt layout
  T* slot;            // [gridDim.x][3][K][n][n] CTA-private L, D, theta^-1 staging
  const T* lambda0;   // [B][D] or null
  T* lambda_out;      // [B][D]
  int* errkey;        // [B]
  SysOut* out;        // [B]
  double* trace;      // [B][trace_cap] or null
  int trace_cap;
  double epsilon;
  int max_iter;
  unsigned long long* timing;  // optional [B][16] globaltimer stamps per phase (debug)
  // formation only (build_schur): write S [B][K][3][n][n] (zeroed pads), gamma
  // [B][K n], theta^-1 [B][K][n][n] in the reference layout and skip the PCG
  T* S_out;
  T* gamma_out;
  T* theta_out;
  int form_only;
  // the PPCG finish fused into the solve (one-CTA and small-block kernels):
  // when non-null, every successfully solved system also gets
  // dz = [x_0, u_0, ..., x_N] ([B][K n + N m]) from the formation's Q_k^-1 /
  // R_k^-1 (reconstruct_primal, kkt.cpp:153-181)
  T* dz_out;
  int m_rt;  // control dimension (kernels compiled for a padded m read the real one here)
};
template <class T> bool fused_supported(int K, int n, int m, int kind);
// shared memory / slot need grows with dz_out (Q_k^-1 kept for the finish)
template <class T> bool fused_supported_dz(int K, int n, int m, int kind);
template <class T> size_t fused_slot_elems(int K, int n, int m, bool keep_q = false);
// one-CTA kernel shapes: (14, 7) and even n in [10, 16] with m <= 8
template <class T>
cudaError_t launch_fused(const FusedParams<T>& p, int n, int m, int grid, cudaStream_t st);

// Fused one-CTA kernel for small blocks (small_kernels.cu): n, m <= 8 padded
// to powers of two, everything in shared memory (the SQP / NMPC shapes).
template <class T> bool small_supported(int K, int n, int m, int kind);
template <class T> bool small_supported_dz(int K, int n, int m, int kind);
template <class T>
cudaError_t launch_small(const FusedParams<T>& p, int n, int m, int grid, cudaStream_t st);

// Fused cluster kernel (fc_kernels.cu): one thread-block cluster of G CTAs per
// system. fc_pick_g returns the cluster size for a shape (0 = unsupported).
template <class T> int fc_pick_g(int K, int n, int m, int kind, int B);
template <class T> size_t fc_slot_elems(int K, int n, int G);
template <class T>
cudaError_t launch_fc(const FusedParams<T>& p, int G, int max_clusters, cudaStream_t st, int nb);

// Fused grid kernel (fg_kernels.cu): one long-horizon system on G co-resident
// CTAs (cooperative launch) of rp block rows each. FgSync is the zeroed global
// workspace for its reduce-barriers and boundary-row exchanges.
template <class T>
struct FgSync {
  unsigned long long* red;  // [2][gstride] 128-byte-strided LL slots: per-CTA reduction partials
  unsigned long long* xt;   // [gstride][2][VS] LL slots: boundary rows of t
  unsigned long long* xr;   // [gstride][2][VS] LL slots: boundary rows of r~
  int gstride;
  int n;
  unsigned epoch0;  // first epoch of this launch (flags of older launches never match)
};
template <class T> int fg_pick_rp(int K, int n, int m, int kind, int sm_count, int want_rp);
// the grid kernel's compiled shape that holds (n, m) (itself, or a padded one)
template <class T> bool fg_compiled_shape(int n, int m, int* np, int* mp);
template <class T>
cudaError_t launch_fg(const FusedParams<T>& p, const FgSync<T>& sy, int rp, cudaStream_t st);

// reconstruct_primal (primal_kernels.cu): one warp per (system, knot, block).
template <class T>
struct PrimalParams {
  int B, N, n, m;
  const T *Q, *q, *R, *r, *A, *B_;  // b2p_kkt layout, [B][...]
  const T* lambda;                 // [B][(N+1) n]
  T* dz;                           // [B][(N+1) n + N m]
};
template <class T> cudaError_t launch_reconstruct_primal(const PrimalParams<T>& p, cudaStream_t st);

// Shared-memory footprint of one PCG CTA (bytes) for a parameter block.
template <class T>
size_t pcg_smem_bytes(const PcgParams<T>& p);
int pcg_halo(int kind, int order);

template <class T> cudaError_t launch_build_schur(const FormParams<T>& p, cudaStream_t st);
template <class T> cudaError_t launch_build_precond(const PrecondParams<T>& p, cudaStream_t st);
template <class T>
cudaError_t launch_blocktri_matvec(int B, int K, int nb, const T* M, const T* x, T* y, int mode,
                                   const T* add_to, T* acc, cudaStream_t st);
template <class T>
cudaError_t launch_stair_matrix(int K, int nb, const T* S, T* psi, cudaStream_t st);
template <class T>
cudaError_t launch_blocktri_check(int K, int nb, const T* M, double* out2, cudaStream_t st);
template <class T>
cudaError_t launch_block_cholesky(int B, int K, int nb, const T* M, const T* rhs, T* x, T* factors,
                                  T* y, int* status, cudaStream_t st);
template <class T> cudaError_t launch_pcg(const PcgParams<T>& p, cudaStream_t st);

}  // namespace b2p
