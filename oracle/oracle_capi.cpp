// TEST INFRASTRUCTURE — NOT PRODUCT CODE. C shim over the oracle restatement
// (trajopt_oracle.hpp) for ctypes callers: tests/, smoke() and bench.py's CPU
// legs. Inputs and outputs are double buffers in the b2p.h layouts; `dtype`
// selects the arithmetic precision of the restatement (f64 = the reference;
// f32 = the same algorithm in float, used to pin the fp32 GPU path).
#include <cstring>
#include <memory>

#include "../include/b2p.h"
#include "trajopt_oracle.hpp"

using namespace oracle;

namespace {

void set_err(b2p_error* err, int code, const std::string& msg) {
  if (!err) return;
  err->code = code;
  err->knot = -1;
  err->iteration = -1;
  err->system = -1;
  std::snprintf(err->message, sizeof(err->message), "%s", msg.c_str());
}

template <class F>
int guard(b2p_error* err, F&& f) {
  if (err) set_err(err, B2P_OK, "");
  try {
    f();
    return B2P_OK;
  } catch (const PcgBreakdown& e) {
    set_err(err, B2P_BREAKDOWN, e.what());
    return B2P_BREAKDOWN;
  } catch (const std::invalid_argument& e) {
    set_err(err, B2P_INVALID_ARGUMENT, e.what());
    return B2P_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    set_err(err, B2P_RUNTIME_ERROR, e.what());
    return B2P_RUNTIME_ERROR;
  }
}

template <class T>
Mat<T> load_mat(const double* p, int r, int c) {
  Mat<T> M(r, c);
  for (int i = 0; i < r * c; ++i) M.a[i] = static_cast<T>(p[i]);
  return M;
}
template <class T>
Vec<T> load_vec(const double* p, int n) {
  Vec<T> v(n);
  for (int i = 0; i < n; ++i) v[i] = static_cast<T>(p[i]);
  return v;
}
template <class T>
void store(double* dst, const std::vector<T>& v) {
  for (std::size_t i = 0; i < v.size(); ++i) dst[i] = static_cast<double>(v[i]);
}

template <class T>
KKTSystem<T> load_kkt(const b2p_kkt* k) {
  KKTSystem<T> kkt;
  kkt.N = k->N;
  kkt.n = k->n;
  kkt.m = k->m;
  const int N = k->N, n = k->n, m = k->m;
  kkt.knots.resize(N + 1);
  const double* Q = static_cast<const double*>(k->Q);
  const double* q = static_cast<const double*>(k->q);
  const double* R = static_cast<const double*>(k->R);
  const double* r = static_cast<const double*>(k->r);
  const double* A = static_cast<const double*>(k->A);
  const double* B = static_cast<const double*>(k->B);
  const double* e = static_cast<const double*>(k->e);
  for (int i = 0; i <= N; ++i) {
    kkt.knots[i].Q = load_mat<T>(Q + static_cast<std::size_t>(i) * n * n, n, n);
    kkt.knots[i].q = load_vec<T>(q + static_cast<std::size_t>(i) * n, n);
    if (i < N) {
      kkt.knots[i].R = load_mat<T>(R + static_cast<std::size_t>(i) * m * m, m, m);
      kkt.knots[i].r = load_vec<T>(r + static_cast<std::size_t>(i) * m, m);
      kkt.knots[i].A = load_mat<T>(A + static_cast<std::size_t>(i) * n * n, n, n);
      kkt.knots[i].B = load_mat<T>(B + static_cast<std::size_t>(i) * n * m, n, m);
      kkt.knots[i].e = load_vec<T>(e + static_cast<std::size_t>(i) * n, n);
    }
  }
  kkt.x_s = load_vec<T>(static_cast<const double*>(k->x_s), n);
  kkt.x0 = load_vec<T>(static_cast<const double*>(k->x0), n);
  return kkt;
}

template <class T>
BlockTri<T> load_bt(const double* p, int K, int nb) {
  BlockTri<T> M(K, nb);
  for (std::size_t i = 0; i < M.raw().size(); ++i) M.raw()[i] = static_cast<T>(p[i]);
  return M;
}

template <class T>
Preconditioner<T> make_precond(int kind, int order, int K, int nb, const double* S,
                               const double* phi_inv) {
  Preconditioner<T> P;
  P.kind = static_cast<PrecondKind>(kind);
  if (kind < 0 || kind > 4) throw std::invalid_argument("build_preconditioner: unknown kind");
  if (P.kind == PrecondKind::identity) return P;
  P.phi_inv = load_bt<T>(phi_inv, K, nb);
  if (P.kind == PrecondKind::poly_split) {
    if (order < 1)
      throw std::invalid_argument("build_poly_split: order must be >= 1, got " +
                                  std::to_string(order));
    P.order = order;
    const BlockTri<T> Sm = load_bt<T>(S, K, nb);
    P.stair_psi = stair_matrix(Sm);
    P.remainder = BlockTri<T>(K, nb);
    for (int row = 0; row < K; row += 2) {
      if (row > 0) P.remainder.set_left(row, neg(Sm.left(row)));
      if (row + 1 < K) P.remainder.set_right(row, neg(Sm.right(row)));
    }
  }
  return P;
}

PcgConfig load_cfg(const b2p_pcg_config* c) {
  PcgConfig cfg;
  if (!c) return cfg;
  cfg.epsilon = c->epsilon;
  cfg.max_iter = c->max_iter;
  cfg.deterministic_reductions = c->deterministic_reductions != 0;
  cfg.variant = static_cast<PcgVariant>(c->variant);
  cfg.collect_trace = c->collect_trace != 0;
  cfg.check_residual_drift = c->check_residual_drift != 0;
  return cfg;
}

template <class T>
void store_report(const PcgResult<T>& res, b2p_solve_report* rep, double* trace) {
  if (rep) {
    rep->iterations = res.report.iterations;
    rep->converged = res.report.converged ? 1 : 0;
    rep->exit_eta = res.report.exit_eta;
    rep->wall_time = res.report.wall_time;
    rep->max_residual_drift = res.report.max_residual_drift;
    rep->trace_len = static_cast<int32_t>(res.report.trace.size());
    rep->status = B2P_OK;
  }
  if (trace)
    for (std::size_t i = 0; i < res.report.trace.size(); ++i) trace[i] = res.report.trace[i];
}

template <class T>
void do_build_schur(const b2p_kkt* k, double* S, double* gamma, double* theta_inv) {
  const KKTSystem<T> kkt = load_kkt<T>(k);
  const SchurSystem<T> s = build_schur(kkt);
  store(S, s.S.raw());
  store(gamma, s.gamma);
  const int n = kkt.n;
  for (int b = 0; b <= kkt.N; ++b)
    for (int i = 0; i < n * n; ++i)
      theta_inv[static_cast<std::size_t>(b) * n * n + i] = static_cast<double>(s.theta_inv[b].a[i]);
}

template <class T>
SchurSystem<T> load_schur(int K, int nb, const double* S, const double* theta_inv) {
  SchurSystem<T> s;
  s.n = nb;
  s.S = load_bt<T>(S, K, nb);
  s.gamma.assign(static_cast<std::size_t>(K) * nb, T(0));
  for (int b = 0; b < K; ++b)
    s.theta_inv.push_back(load_mat<T>(theta_inv + static_cast<std::size_t>(b) * nb * nb, nb, nb));
  return s;
}

template <class T>
void do_build_precond(int kind, int order, int K, int nb, const double* S, const double* theta_inv,
                      double* phi_inv, double* psi, double* remainder) {
  const SchurSystem<T> s = load_schur<T>(K, nb, S, theta_inv);
  if (kind < 0 || kind > 4) throw std::invalid_argument("build_preconditioner: unknown kind");
  const Preconditioner<T> P = build_preconditioner(s, static_cast<PrecondKind>(kind), order);
  if (P.kind != PrecondKind::identity && phi_inv) store(phi_inv, P.phi_inv.raw());
  if (P.kind == PrecondKind::poly_split) {
    if (psi) store(psi, P.stair_psi.raw());
    if (remainder) store(remainder, P.remainder.raw());
  }
}

template <class T>
void do_apply(int kind, int order, int K, int nb, const double* S, const double* phi_inv,
              const double* r, double* out) {
  const Preconditioner<T> P = make_precond<T>(kind, order, K, nb, S, phi_inv);
  store(out, apply_preconditioner(P, load_vec<T>(r, K * nb)));
}

template <class T>
void do_pcg(int K, int nb, const double* S, int kind, int order, const double* phi_inv,
            const double* gamma, const double* lambda0, const b2p_pcg_config* c, double* lam,
            b2p_solve_report* rep, double* trace, int gamma_len, int lambda0_len) {
  const BlockTri<T> Sm = load_bt<T>(S, K, nb);
  const Preconditioner<T> P = make_precond<T>(kind, order, K, nb, S, phi_inv);
  const PcgResult<T> res = pcg_solve_auto(Sm, P, load_vec<T>(gamma, gamma_len),
                                          load_vec<T>(lambda0, lambda0_len), load_cfg(c));
  store(lam, res.lambda);
  store_report(res, rep, trace);
}

template <class T>
PcgResult<T> solve_one(const KKTSystem<T>& kkt, int kind, int order, const PcgConfig& cfg,
                       const double* lambda0) {
  const SchurSystem<T> s = build_schur(kkt);
  const Preconditioner<T> P = build_preconditioner(s, static_cast<PrecondKind>(kind), order);
  Vec<T> l0(static_cast<std::size_t>(s.S.dim()), T(0));
  if (lambda0)
    for (std::size_t i = 0; i < l0.size(); ++i) l0[i] = static_cast<T>(lambda0[i]);
  return pcg_solve_auto(s.S, P, s.gamma, l0, cfg);
}

b2p_kkt slice(const b2p_kkt* k, int i) {
  const std::size_t N = k->N, n = k->n, m = k->m;
  b2p_kkt s = *k;
  auto off = [&](const void* p, std::size_t per) {
    return static_cast<const void*>(static_cast<const double*>(p) + i * per);
  };
  s.Q = off(k->Q, (N + 1) * n * n);
  s.q = off(k->q, (N + 1) * n);
  s.R = off(k->R, N * m * m);
  s.r = off(k->r, N * m);
  s.A = off(k->A, N * n * n);
  s.B = off(k->B, N * n * m);
  s.e = off(k->e, N * n);
  s.x_s = off(k->x_s, n);
  s.x0 = off(k->x0, n);
  return s;
}

void write_kkt(const KKTSystem<double>& kkt, b2p_kkt_out* o, std::size_t i) {
  const std::size_t N = kkt.N, n = kkt.n, m = kkt.m;
  for (std::size_t k = 0; k <= N; ++k) {
    std::memcpy(o->Q + i * (N + 1) * n * n + k * n * n, kkt.knots[k].Q.a.data(), n * n * 8);
    std::memcpy(o->q + i * (N + 1) * n + k * n, kkt.knots[k].q.data(), n * 8);
    if (k < N) {
      std::memcpy(o->R + i * N * m * m + k * m * m, kkt.knots[k].R.a.data(), m * m * 8);
      std::memcpy(o->r + i * N * m + k * m, kkt.knots[k].r.data(), m * 8);
      std::memcpy(o->A + i * N * n * n + k * n * n, kkt.knots[k].A.a.data(), n * n * 8);
      std::memcpy(o->B + i * N * n * m + k * n * m, kkt.knots[k].B.a.data(), n * m * 8);
      std::memcpy(o->e + i * N * n + k * n, kkt.knots[k].e.data(), n * 8);
    }
  }
  std::memcpy(o->x_s + i * n, kkt.x_s.data(), n * 8);
  std::memcpy(o->x0 + i * n, kkt.x0.data(), n * 8);
}

KKTSystem<double> gen(int family, uint64_t seed, int N, int n, int m, double f, double c) {
  if (family == 0) return random_kkt(seed, N, n, m);
  if (family == 1) return random_kkt_scaled(seed, N, n, m, f, c);
  return random_trajectory_kkt(seed, N, n, m);
}

}  // namespace

extern "C" {

int orc_set_threads(int t) {
  hw_threads_override() = t;
  return static_cast<int>(hw_threads());
}

// UniformRng stream (random_problem.hpp:17-20): out[i] = lo + (hi-lo)*u01.
void orc_uniform(uint64_t seed, int count, double lo, double hi, double* out) {
  UniformRng rng(seed);
  for (int i = 0; i < count; ++i) out[i] = rng.uniform(lo, hi);
}

int orc_random_kkt(int family, uint64_t seed, int N, int n, int m, double diag_floor,
                   double coupling, b2p_kkt_out* out, b2p_error* err) {
  return guard(err, [&] { write_kkt(gen(family, seed, N, n, m, diag_floor, coupling), out, 0); });
}

// Batch generator (the bench-pcg seeding rule, trajopt_cli.cpp:142-151): system
// i = family(seed0 + i); `threads` host threads (0 = all).
int orc_random_kkt_batch(int family, uint64_t seed0, int batch, int N, int n, int m,
                         double diag_floor, double coupling, int threads, b2p_kkt_out* out,
                         b2p_error* err) {
  const int saved = hw_threads_override();
  hw_threads_override() = threads;
  const int rc = guard(err, [&] {
    parallel_for(0, batch, [&](int i) {
      write_kkt(gen(family, seed0 + static_cast<uint64_t>(i), N, n, m, diag_floor, coupling), out,
                static_cast<std::size_t>(i));
    });
  });
  hw_threads_override() = saved;
  return rc;
}

int orc_build_schur(int dtype, const b2p_kkt* kkt, double* S, double* gamma, double* theta_inv,
                    b2p_error* err) {
  return guard(err, [&] {
    if (dtype == B2P_F32) do_build_schur<float>(kkt, S, gamma, theta_inv);
    else do_build_schur<double>(kkt, S, gamma, theta_inv);
  });
}

int orc_stair_matrix(int K, int nb, const double* S, double* psi, b2p_error* err) {
  return guard(err, [&] { store(psi, stair_matrix(load_bt<double>(S, K, nb)).raw()); });
}

int orc_build_preconditioner(int dtype, int kind, int order, int K, int nb, const double* S,
                             const double* theta_inv, double* phi_inv, double* psi,
                             double* remainder, b2p_error* err) {
  return guard(err, [&] {
    if (dtype == B2P_F32) do_build_precond<float>(kind, order, K, nb, S, theta_inv, phi_inv, psi, remainder);
    else do_build_precond<double>(kind, order, K, nb, S, theta_inv, phi_inv, psi, remainder);
  });
}

int orc_apply_preconditioner(int dtype, int kind, int order, int K, int nb, const double* S,
                             const double* phi_inv, const double* r, double* out, b2p_error* err) {
  return guard(err, [&] {
    if (dtype == B2P_F32) do_apply<float>(kind, order, K, nb, S, phi_inv, r, out);
    else do_apply<double>(kind, order, K, nb, S, phi_inv, r, out);
  });
}

int orc_matvec(int K, int nb, const double* M, const double* x, int xlen, double* y,
               b2p_error* err) {
  return guard(err, [&] { store(y, load_bt<double>(M, K, nb).matvec(load_vec<double>(x, xlen))); });
}

double orc_max_asymmetry(int K, int nb, const double* M) {
  return load_bt<double>(M, K, nb).max_asymmetry();
}
double orc_max_abs(int K, int nb, const double* M) { return load_bt<double>(M, K, nb).max_abs(); }

int orc_cholesky_solve(int K, int nb, const double* M, const double* rhs, double* x,
                       b2p_error* err) {
  return guard(err, [&] {
    store(x, load_bt<double>(M, K, nb).cholesky_solve(load_vec<double>(rhs, K * nb)));
  });
}

int orc_pcg_solve(int dtype, int K, int nb, const double* S, int kind, int order,
                  const double* phi_inv, const double* gamma, int gamma_len,
                  const double* lambda0, int lambda0_len, const b2p_pcg_config* cfg,
                  double* lambda_out, b2p_solve_report* report, double* trace, b2p_error* err) {
  return guard(err, [&] {
    if (dtype == B2P_F32)
      do_pcg<float>(K, nb, S, kind, order, phi_inv, gamma, lambda0, cfg, lambda_out, report, trace,
                    gamma_len, lambda0_len);
    else
      do_pcg<double>(K, nb, S, kind, order, phi_inv, gamma, lambda0, cfg, lambda_out, report,
                     trace, gamma_len, lambda0_len);
  });
}

// build_schur -> build_preconditioner -> pcg_solve_auto (what sqp.cpp:171-176
// and cmd_bench_pcg do per instance).
int orc_solve(int dtype, const b2p_kkt* kkt, int kind, int order, const b2p_pcg_config* cfg,
              const double* lambda0, double* lambda_out, b2p_solve_report* report, double* trace,
              b2p_error* err) {
  return guard(err, [&] {
    if (dtype == B2P_F32) {
      const auto res = solve_one(load_kkt<float>(kkt), kind, order, load_cfg(cfg), lambda0);
      store(lambda_out, res.lambda);
      store_report(res, report, trace);
    } else {
      const auto res = solve_one(load_kkt<double>(kkt), kind, order, load_cfg(cfg), lambda0);
      store(lambda_out, res.lambda);
      store_report(res, report, trace);
    }
  });
}

// Batched CPU baseline mirroring cmd_bench_pcg's instance loop
// (proj/tools/trajopt_cli.cpp:155-191): parallel_for over pre-generated
// instances, each running build_schur + build_preconditioner + pcg_solve_auto.
// `threads` host threads (0 = all). Returns elapsed seconds (steady_clock).
double orc_solve_batch(int dtype, int batch, const b2p_kkt* kkt_batch, int kind, int order,
                       const b2p_pcg_config* cfg, int threads, double* lambda_out,
                       b2p_solve_report* reports, b2p_error* err) {
  const int saved = hw_threads_override();
  hw_threads_override() = threads;
  const std::size_t D = static_cast<std::size_t>(kkt_batch->N + 1) * kkt_batch->n;
  const auto start = Clock::now();
  const int rc = guard(err, [&] {
    parallel_for(0, batch, [&](int i) {
      const b2p_kkt k = slice(kkt_batch, i);
      double* lo = lambda_out ? lambda_out + i * D : nullptr;
      b2p_solve_report* rep = reports ? reports + i : nullptr;
      if (dtype == B2P_F32) {
        const auto res = solve_one(load_kkt<float>(&k), kind, order, load_cfg(cfg), nullptr);
        if (lo) store(lo, res.lambda);
        store_report(res, rep, nullptr);
      } else {
        const auto res = solve_one(load_kkt<double>(&k), kind, order, load_cfg(cfg), nullptr);
        if (lo) store(lo, res.lambda);
        store_report(res, rep, nullptr);
      }
    });  // default grain 8, nested parallel_for inside build_schur: as the reference
  });
  const double secs = seconds_since(start);
  hw_threads_override() = saved;
  return rc == B2P_OK ? secs : -1.0;
}

int orc_reconstruct_primal(int dtype, const b2p_kkt* kkt, const double* lambda, int lambda_len,
                           double* dz, b2p_error* err) {
  return guard(err, [&] {
    if (dtype == B2P_F32)
      store(dz, reconstruct_primal(load_kkt<float>(kkt), load_vec<float>(lambda, lambda_len)));
    else
      store(dz, reconstruct_primal(load_kkt<double>(kkt), load_vec<double>(lambda, lambda_len)));
  });
}

}  // extern "C"
