/*
 * b2p.h — C-ABI of the B200-native symmetric-stair PCG hot path
 * (arXiv 2309.08079, "MPCGPU"; reference artifact /root/reference/proj).
 *
 * Drop-in boundary. Each entry point names the reference
 * interface it replaces. The reference exposes Eigen-typed C++ free functions;
 * this ABI exposes the same operations over plain row-major buffers so that a
 * thin C++ adapter (include/trajopt_b200.hpp) can restore the reference's
 * names, value semantics and exception classes.
 *
 * Layouts (all row-major, no padding):
 *   BlockTriMatrix  : T[K][3][nb][nb]  slot 0 = left, 1 = diag, 2 = right;
 *                     row 0 left and row K-1 right are zero padding
 *                     (proj/src/block_tri.cpp:16-23).
 *   vectors         : T[K*nb], block b at offset b*nb.
 *   theta_inv       : T[K][nb][nb]   (SchurSystem::theta_inv, schur.hpp:23).
 *   KKT (b2p_kkt)   : SoA over K = N+1 knots, see below (kkt.hpp:13-46;
 *                     Eigen's column-major KnotData is transposed by callers).
 * T is double for B2P_F64 and float for B2P_F32.
 *
 * Errors: every call returns a b2p_status; on failure `err` (nullable)
 * carries the reference's exception message verbatim plus knot / iteration.
 * Mapping to the reference's exception classes (proj/src/pcg.cpp,
 * proj/src/schur.cpp): INVALID_ARGUMENT -> std::invalid_argument,
 * RUNTIME_ERROR -> std::runtime_error, BREAKDOWN -> trajopt::PcgBreakdown.
 *
 * Threading: one b2p_ctx per (host thread, device); calls on different
 * contexts may run concurrently. No pointer is retained after
 * a call returns.
 */
#ifndef B2P_H_
#define B2P_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define B2P_ABI_VERSION 1

typedef enum b2p_status {
  B2P_OK = 0,
  B2P_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  B2P_RUNTIME_ERROR = 2,    /* std::runtime_error (non-PD knot, non-finite) */
  B2P_BREAKDOWN = 3,        /* trajopt::PcgBreakdown (pcg.hpp:47-50) */
  B2P_CUDA_ERROR = 4        /* device / driver failure (no reference analog) */
} b2p_status;

typedef enum b2p_dtype { B2P_F64 = 0, B2P_F32 = 1 } b2p_dtype;

/* trajopt::PrecondKind (schur.hpp:26) — same order. */
typedef enum b2p_precond_kind {
  B2P_IDENTITY = 0,
  B2P_BLOCK_JACOBI = 1,
  B2P_STAIR = 2,
  B2P_SYMMETRIC_STAIR = 3,
  B2P_POLY_SPLIT = 4
} b2p_precond_kind;

/* trajopt::PcgVariant (pcg.hpp:12). */
typedef enum b2p_pcg_variant { B2P_SEQUENTIAL = 0, B2P_BLOCK_PARALLEL = 1 } b2p_pcg_variant;

/* trajopt::PcgConfig (pcg.hpp:14-29), same field order and defaults
 * (epsilon 1e-4, max_iter 0 => dim, everything else off). */
typedef struct b2p_pcg_config {
  double epsilon;
  int32_t max_iter;
  int32_t deterministic_reductions;
  int32_t variant; /* b2p_pcg_variant */
  int32_t collect_trace;
  int32_t check_residual_drift;
  int32_t _reserved;
} b2p_pcg_config;

/* trajopt::SolveReport (pcg.hpp:31-38). The trace is written to a caller
 * buffer (capacity = resolved max_iter) and its length reported here. */
typedef struct b2p_solve_report {
  int32_t iterations;
  int32_t converged;
  double exit_eta;
  double wall_time; /* seconds; device time of the solve (CUDA events) */
  double max_residual_drift;
  int32_t trace_len;
  int32_t status; /* b2p_status of this solve (per system in batched calls) */
} b2p_solve_report;

typedef struct b2p_error {
  int32_t code;      /* b2p_status */
  int32_t knot;      /* knot index for non-PD errors, else -1 */
  int32_t iteration; /* PCG iteration for breakdown / non-finite, else -1 */
  int32_t system;    /* batch index for batched calls, else -1 */
  char message[256]; /* the reference's exception text */
} b2p_error;

/* KKTSystem in per-knot SoA form (kkt.hpp:13-46). K = N + 1 knots.
 * Batched calls: every array gains a leading [batch] dimension. */
typedef struct b2p_kkt {
  int32_t N; /* horizon: N+1 state knots, N control knots */
  int32_t n; /* state dim = block dim nb */
  int32_t m; /* control dim */
  int32_t _pad;
  const void* Q;   /* [N+1][n][n] */
  const void* q;   /* [N+1][n]    */
  const void* R;   /* [N][m][m]   */
  const void* r;   /* [N][m]      */
  const void* A;   /* [N][n][n]   */
  const void* B;   /* [N][n][m]   */
  const void* e;   /* [N][n]      */
  const void* x_s; /* [n] */
  const void* x0;  /* [n] */
} b2p_kkt;

/* Mutable view used by the generator. */
typedef struct b2p_kkt_out {
  int32_t N, n, m, _pad;
  double *Q, *q, *R, *r, *A, *B, *e, *x_s, *x0;
} b2p_kkt_out;

typedef struct b2p_ctx b2p_ctx;

/* ---- library / context ------------------------------------------------ */
int b2p_abi_version(void);
/* Number of CUDA devices visible (0 on a CPU-only host). */
int b2p_device_count(void);
int b2p_ctx_create(int device, b2p_ctx** out, b2p_error* err);
void b2p_ctx_destroy(b2p_ctx* ctx);
/* Launch stream for the *_device entry points (cudaStream_t as void*; NULL
 * = the context's own stream). */
int b2p_ctx_set_stream(b2p_ctx* ctx, void* stream);
void* b2p_ctx_stream(b2p_ctx* ctx);
/* Number of kernels this context launched since creation (evidence counter). */
long long b2p_ctx_kernel_launches(b2p_ctx* ctx);
/* Which device path the most recent fused solve took: 0 = split K1 formation
 * + K3 PCG, 1 = the persistent one-CTA-per-system kernel (n14/m7 fp64),
 * 2 = the cluster kernel, 3 = the cooperative grid kernel, 4 = the small-block
 * one-CTA kernel (n, m <= 8 fp64). */
int b2p_ctx_last_path(b2p_ctx* ctx);
/* Debug (B2P_PHASE_TIMING=1): per-system %globaltimer stamps of the last
 * one-CTA fused solve, [n][16] = start, F1 end, F2 end, staging end, end (ns),
 * then kernel-specific SM-clock segment sums (scripts/phase_probe.py).
 * Returns the number of systems copied. */
int b2p_ctx_phase_stamps(b2p_ctx* ctx, unsigned long long* out, int n);

/* ---- block_tri.hpp ---------------------------------------------------- */
/* BlockTriMatrix::matvec (block_tri.cpp:70-92). */
int b2p_blocktri_matvec(b2p_ctx* ctx, int dtype, int K, int nb, const void* M, const void* x,
                        int x_len, void* y, b2p_error* err);
/* BlockTriMatrix::cholesky_solve (block_tri.cpp:121-159): the direct
 * block-Thomas baseline (bench-pcg's "dense_baseline" row). */
int b2p_blocktri_cholesky_solve(b2p_ctx* ctx, int dtype, int K, int nb, const void* M,
                                const void* rhs, int rhs_len, void* x, b2p_error* err);
/* BlockTriMatrix::max_asymmetry / max_abs (block_tri.cpp:161-177), on device. */
int b2p_blocktri_check(b2p_ctx* ctx, int dtype, int K, int nb, const void* M,
                       double* max_asymmetry, double* max_abs, b2p_error* err);

/* ---- schur.hpp -------------------------------------------------------- */
/* build_schur (schur.hpp:40, schur.cpp:38-82). Outputs: S [K][3][n][n],
 * gamma [K*n], theta_inv [K][n][n]. */
int b2p_build_schur(b2p_ctx* ctx, int dtype, const b2p_kkt* kkt, void* S, void* gamma,
                    void* theta_inv, b2p_error* err);
/* stair_matrix (schur.cpp:84-94). */
int b2p_stair_matrix(b2p_ctx* ctx, int dtype, int K, int nb, const void* S, void* psi,
                     b2p_error* err);
/* build_preconditioner (schur.hpp:51, schur.cpp:96-173): phi_inv
 * [K][3][nb][nb] (untouched for identity). For poly_split the stair
 * matrix / remainder are implied by S and not materialised. */
int b2p_build_preconditioner(b2p_ctx* ctx, int dtype, int kind, int order, int K, int nb,
                             const void* S, const void* theta_inv, void* phi_inv, b2p_error* err);
/* apply_preconditioner (schur.hpp:56, schur.cpp:175-194). S is only read for
 * poly_split (remainder E = Psi - S). */
int b2p_apply_preconditioner(b2p_ctx* ctx, int dtype, int kind, int order, int K, int nb,
                             const void* S, const void* phi_inv, const void* r, int r_len,
                             void* out, b2p_error* err);

/* ---- pcg.hpp ---------------------------------------------------------- */
/* pcg_solve / pcg_solve_block_parallel / pcg_solve_auto (pcg.hpp:57-70,
 * pcg.cpp:55-369) — dispatch on cfg->variant. trace: nullable, capacity
 * resolved max_iter. phi_inv may be NULL for identity. The *_len / phi_K /
 * phi_nb arguments carry the caller's vector and preconditioner sizes so the
 * reference's validate_inputs messages (pcg.cpp:24-47) are reproduced. */
int b2p_pcg_solve(b2p_ctx* ctx, int dtype, int K, int nb, const void* S, int kind, int order,
                  int phi_K, int phi_nb, const void* phi_inv, const void* gamma, int gamma_len,
                  const void* lambda0, int lambda0_len, const b2p_pcg_config* cfg,
                  void* lambda_out, b2p_solve_report* report, double* trace, b2p_error* err);

/* ---- fused hot path (north star): build_schur -> build_preconditioner ->
 * pcg_solve_auto for one system in one device pass. lambda0 NULL => 0. ---- */
int b2p_solve(b2p_ctx* ctx, int dtype, const b2p_kkt* kkt, int kind, int order,
              const b2p_pcg_config* cfg, const void* lambda0, void* lambda_out,
              b2p_solve_report* report, double* trace, b2p_error* err);

/* Batched independent systems (cmd_bench_pcg's parallel_for over instances,
 * proj/tools/trajopt_cli.cpp:155-191). Host buffers, [batch] leading dim;
 * H2D / compute / D2H pipelined in chunks. reports: [batch]. Per-system
 * failures are reported in reports[i].status; the call returns the first
 * failing system's status with its message in err. */
int b2p_solve_batched(b2p_ctx* ctx, int dtype, int batch, const b2p_kkt* kkt_batch, int kind,
                      int order, const b2p_pcg_config* cfg, const void* lambda0,
                      void* lambda_out, b2p_solve_report* reports, b2p_error* err);

/* Same, with every pointer (kkt arrays, lambda0, lambda_out) in device
 * memory, launched on the context stream, no host synchronisation unless
 * `reports` is non-NULL (host array, copied back after the solve).
 * status_dev (nullable, device int32[batch*4]) receives
 * {status, iterations, converged, aux} per system without a host sync. */
int b2p_solve_batched_device(b2p_ctx* ctx, int dtype, int batch, const b2p_kkt* kkt_batch_dev,
                             int kind, int order, const b2p_pcg_config* cfg,
                             const void* lambda0_dev, void* lambda_out_dev,
                             b2p_solve_report* reports, int32_t* status_dev, b2p_error* err);

/* K4: shard `batch` systems by contiguous batch index over `ndev` devices,
 * one host thread + context per device, no inter-GPU traffic.
 * The per-device contexts persist in a process-wide pool across calls (a
 * device listed k times gets k contexts); every shard's context is ready
 * before any device starts (host barrier). */
int b2p_solve_batched_multi(const int* devices, int ndev, int dtype, int batch,
                            const b2p_kkt* kkt_batch, int kind, int order,
                            const b2p_pcg_config* cfg, const void* lambda0, void* lambda_out,
                            b2p_solve_report* reports, b2p_error* err);

/* ---- reconstruct_primal (proj/include/trajopt/kkt.hpp, kkt.cpp:153-181):
 * dz = [x_0, u_0, ..., x_N] from the multipliers, per knot
 * dx_k = Q_k^-1 (-(q_k + lambda_k - A_k' lambda_{k+1})), du_k = R_k^-1 (-(r_k - B_k' lambda_{k+1})).
 * Host buffers; lambda_len must equal (N+1) n (else INVALID_ARGUMENT with the
 * reference's "reconstruct_primal: expected lambda of length D, got X");
 * dz_out holds (N+1) n + N m values. Like the reference's LDLT solve there
 * is no positive-definiteness error path. */
int b2p_reconstruct_primal(b2p_ctx* ctx, int dtype, const b2p_kkt* kkt, const void* lambda,
                           int lambda_len, void* dz_out, b2p_error* err);
/* Batched, every pointer in device memory ([batch] leading dimension),
 * launched on the context stream without a host synchronisation. */
int b2p_reconstruct_primal_batched_device(b2p_ctx* ctx, int dtype, int batch,
                                          const b2p_kkt* kkt_batch_dev, const void* lambda_dev,
                                          void* dz_dev, b2p_error* err);

/* ---- the SQP linear step (sqp.cpp:171-176): build_schur ->
 * build_preconditioner -> pcg_solve_auto(lambda0) -> reconstruct_primal(lambda)
 * on ONE upload of the knots: the fused solve and the primal kernel run
 * back to back on the context stream, then lambda_out ((N+1) n) and dz_out
 * ((N+1) n + N m) come back together. Errors as b2p_solve; dz is produced only
 * on success (the reference's exception leaves no dz either). */
int b2p_sqp_step(b2p_ctx* ctx, int dtype, const b2p_kkt* kkt, int kind, int order,
                 const b2p_pcg_config* cfg, const void* lambda0, void* lambda_out, void* dz_out,
                 b2p_solve_report* report, double* trace, b2p_error* err);

/* ---- direct baseline (trajopt_cli.cpp:164-173's
 * "dense_baseline" row): build_schur -> BlockTriMatrix::cholesky_solve(gamma)
 * (block_tri.cpp:121-159, block Thomas) for a device-resident batch, one warp
 * per system, launched on the context stream without a host sync.
 * status_dev[i] = -1 on success, else the first block row whose pivot block
 * is not positive definite. */
int b2p_direct_solve_batched_device(b2p_ctx* ctx, int dtype, int batch, const b2p_kkt* kkt_batch_dev,
                                    void* lambda_dev, int* status_dev, b2p_error* err);

/* Device time (ms) of the most recent solve kernels on this context. */
int b2p_ctx_last_solve_ms(b2p_ctx* ctx, float* ms);
/* Host -> device bytes moved by the most recent b2p_solve_batched on this
 * context (Q_k / R_k travel as lower triangles, mirrored on the device: the
 * reference's LLT / LDLT read only the lower triangle, schur.cpp:16). */
int b2p_ctx_last_h2d_bytes(b2p_ctx* ctx, unsigned long long* bytes);
/* Per-kernel split of the most recent fused solve: ms[0] = K1 Schur
 * formation, ms[1] = K3 PCG (CUDA events on the launch stream; n >= 2).
 * Valid after the caller synchronised the stream. */
int b2p_ctx_last_phase_ms(b2p_ctx* ctx, float* ms, int n);
/* Phase accounting for measurement: while enabled every fused solve records
 * its own (start, K1 end, K3 end) CUDA events on the launch stream;
 * b2p_ctx_phase_totals waits for them and returns the summed K1 / K3 / total
 * device ms (n >= 3) and the number of solves, then resets. */
int b2p_ctx_phase_accounting(b2p_ctx* ctx, int enable);
int b2p_ctx_phase_totals(b2p_ctx* ctx, float* ms, int n, int* count);

/* ---- random_problem.hpp (host-side input synthesis) -------------------- */
/* family: 0 random_kkt, 1 random_kkt_scaled(diag_floor, coupling),
 * 2 random_trajectory_kkt (random_problem.cpp:42-80). Writes f64 arrays. */
int b2p_random_kkt(int family, uint64_t seed, int N, int n, int m, double diag_floor,
                   double coupling, b2p_kkt_out* out, b2p_error* err);
/* Batch generator: system i uses seed0 + i; arrays carry a [batch] leading
 * dimension; `threads` host threads (0 = hardware concurrency). */
int b2p_random_kkt_batch(int family, uint64_t seed0, int batch, int N, int n, int m,
                         double diag_floor, double coupling, int threads, b2p_kkt_out* out,
                         b2p_error* err);

/* UniformRng(seed): `count` draws lo + (hi - lo) * ((x >> 11) * 2^-53) of
 * mt19937_64 in order (random_problem.hpp:13-37) — e.g. the seeded rollout
 * controls of a named-model problem file (problem_io.cpp:208-214). */
int b2p_uniform_draws(uint64_t seed, int count, double lo, double hi, double* out,
                      b2p_error* err);

/* ---- memory helpers (for FFI callers without a CUDA runtime) ----------- */
void* b2p_host_alloc(size_t bytes); /* pinned */
void b2p_host_free(void* p);

#ifdef __cplusplus
}
#endif

#endif /* B2P_H_ */
