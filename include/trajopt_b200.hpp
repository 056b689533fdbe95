// trajopt_b200.hpp — header-only C++ adapter over the C-ABI (b2p.h) that
// restores the reference's solver API: names, value semantics and exception
// classes of proj/include/trajopt/{block_tri,kkt,schur,pcg,random_problem}.hpp.
//
// Storage is Eigen-free (row-major std::vector<double>) so it builds in this
// image; when <Eigen/Dense> is available the overloads at the bottom accept
// Eigen types directly (column-major Eigen matrices are transposed into the
// ABI's row-major layout), which is what the reference's callers
// (sqp.cpp:171-176, trajopt_cli.cpp:93-103,158-184) would link against.
// Link with libb2p.so. Every compute call runs on the GPU.
#pragma once

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "b2p.h"

namespace trajopt_b200 {

using Vector = std::vector<double>;

/// pcg.hpp:47-50
class PcgBreakdown : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void raise(int code, const b2p_error& e) {
  if (code == B2P_OK) return;
  const std::string msg(e.message);
  if (code == B2P_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (code == B2P_BREAKDOWN) throw PcgBreakdown(msg);
  throw std::runtime_error(msg);
}

// One context per (host thread, device), created on first use.
inline b2p_ctx* context(int device = 0) {
  struct Holder {
    std::map<int, b2p_ctx*> ctxs;
    ~Holder() {
      for (auto& kv : ctxs) b2p_ctx_destroy(kv.second);
    }
  };
  thread_local Holder h;
  auto it = h.ctxs.find(device);
  if (it != h.ctxs.end()) return it->second;
  b2p_ctx* c = nullptr;
  b2p_error e{};
  raise(b2p_ctx_create(device, &c, &e), e);
  h.ctxs[device] = c;
  return c;
}
}  // namespace detail

/// Dense row-major matrix (stand-in for Eigen::MatrixXd at the boundary).
struct Matrix {
  int rows = 0, cols = 0;
  std::vector<double> a;
  Matrix() = default;
  Matrix(int r, int c) : rows(r), cols(c), a(static_cast<size_t>(r) * c, 0.0) {}
  double& operator()(int i, int j) { return a[static_cast<size_t>(i) * cols + j]; }
  double operator()(int i, int j) const { return a[static_cast<size_t>(i) * cols + j]; }
  static Matrix identity(int n) {
    Matrix m(n, n);
    for (int i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
};

/// block_tri.hpp:18-75 — [K][left|diag|right][nb][nb] row-major, zero padding.
class BlockTriMatrix {
 public:
  BlockTriMatrix() = default;
  BlockTriMatrix(int num_block_rows, int block_dim) : K_(num_block_rows), nb_(block_dim) {
    if (num_block_rows < 1 || block_dim < 1)
      throw std::invalid_argument("BlockTriMatrix: need at least one block row and block_dim >= 1");
    data_.assign(static_cast<size_t>(K_) * 3 * nb_ * nb_, 0.0);
  }
  int block_rows() const { return K_; }
  int block_dim() const { return nb_; }
  int dim() const { return K_ * nb_; }
  bool empty() const { return K_ == 0; }
  Matrix left(int row) const { return get(row, 0); }
  Matrix diag(int row) const { return get(row, 1); }
  Matrix right(int row) const { return get(row, 2); }
  void set_left(int row, const Matrix& b) {
    check(row, b);
    if (row == 0)
      throw std::invalid_argument("BlockTriMatrix: row 0 has no left block (boundary padding)");
    put(row, 0, b);
  }
  void set_diag(int row, const Matrix& b) {
    check(row, b);
    put(row, 1, b);
  }
  void set_right(int row, const Matrix& b) {
    check(row, b);
    if (row == K_ - 1)
      throw std::invalid_argument("BlockTriMatrix: last row has no right block (boundary padding)");
    put(row, 2, b);
  }
  /// block_tri.cpp:70-80 (on the GPU)
  Vector matvec(const Vector& x) const {
    Vector y(static_cast<size_t>(dim()));
    b2p_error e{};
    detail::raise(b2p_blocktri_matvec(detail::context(), B2P_F64, K_, nb_, data_.data(), x.data(),
                                      static_cast<int>(x.size()), y.data(), &e),
                  e);
    return y;
  }
  /// block_tri.cpp:121-159 (block Thomas on the GPU)
  Vector cholesky_solve(const Vector& rhs) const {
    Vector x(static_cast<size_t>(dim()));
    b2p_error e{};
    detail::raise(b2p_blocktri_cholesky_solve(detail::context(), B2P_F64, K_, nb_, data_.data(),
                                              rhs.data(), static_cast<int>(rhs.size()), x.data(),
                                              &e),
                  e);
    return x;
  }
  double max_asymmetry() const {
    double a = 0, m = 0;
    b2p_error e{};
    detail::raise(b2p_blocktri_check(detail::context(), B2P_F64, K_, nb_, data_.data(), &a, &m, &e),
                  e);
    return a;
  }
  double max_abs() const {
    double a = 0, m = 0;
    b2p_error e{};
    detail::raise(b2p_blocktri_check(detail::context(), B2P_F64, K_, nb_, data_.data(), &a, &m, &e),
                  e);
    return m;
  }
  const double* data() const { return data_.data(); }
  double* data() { return data_.data(); }
  bool structurally_symmetric = false;

 private:
  void check(int row, const Matrix& b) const {
    if (row < 0 || row >= K_)
      throw std::invalid_argument("BlockTriMatrix: block row " + std::to_string(row) +
                                  " out of range [0, " + std::to_string(K_) + ")");
    if (b.rows != nb_ || b.cols != nb_)
      throw std::invalid_argument("BlockTriMatrix: expected " + std::to_string(nb_) + "x" +
                                  std::to_string(nb_) + " block, got " + std::to_string(b.rows) +
                                  "x" + std::to_string(b.cols));
  }
  Matrix get(int row, int slot) const {
    Matrix m(nb_, nb_);
    const size_t off = (static_cast<size_t>(row) * 3 + slot) * nb_ * nb_;
    std::copy(data_.begin() + off, data_.begin() + off + m.a.size(), m.a.begin());
    return m;
  }
  void put(int row, int slot, const Matrix& b) {
    const size_t off = (static_cast<size_t>(row) * 3 + slot) * nb_ * nb_;
    std::copy(b.a.begin(), b.a.end(), data_.begin() + off);
  }
  int K_ = 0, nb_ = 0;
  std::vector<double> data_;
};

/// kkt.hpp:13-46 (per-knot data; R, r, A, B, e absent on the terminal knot).
struct KnotData {
  Matrix Q, R, A, B;
  Vector q, r, e;
};
struct KKTSystem {
  int N = 0, n = 0, m = 0;
  std::vector<KnotData> knots;  // N+1
  Vector x_s, x0;
  int primal_dim() const { return (N + 1) * n + N * m; }
  int dual_dim() const { return (N + 1) * n; }
  /// kkt.cpp:32-39 — c_0 = x_s - x_0, c_{k+1} = -e_k.
  Vector constraint_rhs() const {
    Vector c(static_cast<size_t>(dual_dim()));
    for (int i = 0; i < n; ++i) c[i] = x_s[i] - x0[i];
    for (int k = 0; k < N; ++k)
      for (int i = 0; i < n; ++i) c[static_cast<size_t>(k + 1) * n + i] = -knots[k].e[i];
    return c;
  }
  // Dense realizations (kkt.cpp:41-81; oracle bridges for small instances).
  Matrix dense_G() const {
    Matrix G(primal_dim(), primal_dim());
    int off = 0;
    for (int k = 0; k <= N; ++k) {
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) G(off + i, off + j) = knots[k].Q(i, j);
      off += n;
      if (k < N) {
        for (int i = 0; i < m; ++i)
          for (int j = 0; j < m; ++j) G(off + i, off + j) = knots[k].R(i, j);
        off += m;
      }
    }
    return G;
  }
  Vector dense_g() const {
    Vector g;
    for (int k = 0; k <= N; ++k) {
      g.insert(g.end(), knots[k].q.begin(), knots[k].q.end());
      if (k < N) g.insert(g.end(), knots[k].r.begin(), knots[k].r.end());
    }
    return g;
  }
  Matrix dense_C() const {
    Matrix C(dual_dim(), primal_dim());
    for (int i = 0; i < n; ++i) C(i, i) = 1.0;
    const int stride = n + m;
    for (int k = 0; k < N; ++k) {
      const int row = (k + 1) * n, col = k * stride;
      for (int i = 0; i < n; ++i) {
        for (int j = 0; j < n; ++j) C(row + i, col + j) = -knots[k].A(i, j);
        for (int j = 0; j < m; ++j) C(row + i, col + n + j) = -knots[k].B(i, j);
        C(row + i, col + stride + i) = 1.0;
      }
    }
    return C;
  }
};

/// kkt.hpp — primal update dz = [dx_0 du_0 ... dx_N] and multipliers lambda.
struct PrimalDual {
  Vector dz;
  Vector lambda;
};

/// SoA buffers in the b2p_kkt layout.
struct PackedKKT {
  std::vector<double> Q, q, R, r, A, B, e, x_s, x0;
  b2p_kkt view(int N, int n, int m) const {
    b2p_kkt k{};
    k.N = N;
    k.n = n;
    k.m = m;
    k.Q = Q.data();
    k.q = q.data();
    k.R = R.data();
    k.r = r.data();
    k.A = A.data();
    k.B = B.data();
    k.e = e.data();
    k.x_s = x_s.data();
    k.x0 = x0.data();
    return k;
  }
};
inline PackedKKT pack(const KKTSystem& s) {
  if (static_cast<int>(s.knots.size()) != s.N + 1)
    throw std::invalid_argument("b2p: KKTSystem needs N+1 knots, got " +
                                std::to_string(s.knots.size()));
  PackedKKT p;
  for (int k = 0; k <= s.N; ++k) {
    const KnotData& kd = s.knots[k];
    p.Q.insert(p.Q.end(), kd.Q.a.begin(), kd.Q.a.end());
    p.q.insert(p.q.end(), kd.q.begin(), kd.q.end());
    if (k < s.N) {
      p.R.insert(p.R.end(), kd.R.a.begin(), kd.R.a.end());
      p.r.insert(p.r.end(), kd.r.begin(), kd.r.end());
      p.A.insert(p.A.end(), kd.A.a.begin(), kd.A.a.end());
      p.B.insert(p.B.end(), kd.B.a.begin(), kd.B.a.end());
      p.e.insert(p.e.end(), kd.e.begin(), kd.e.end());
    }
  }
  p.x_s = s.x_s;
  p.x0 = s.x0;
  const size_t K = s.N + 1, N = s.N, n = s.n, m = s.m;
  if (p.Q.size() != K * n * n || p.q.size() != K * n || p.R.size() != N * m * m ||
      p.r.size() != N * m || p.A.size() != N * n * n || p.B.size() != N * n * m ||
      p.e.size() != N * n || p.x_s.size() != n || p.x0.size() != n)
    throw std::invalid_argument("b2p: KKTSystem knot data does not match (N, n, m)");
  return p;
}
namespace detail {
/// pcg.cpp:34-35's message for a lambda0 of the wrong length.
inline void check_lambda0(const Vector* lambda0, int dim) {
  if (lambda0 && static_cast<int>(lambda0->size()) != dim)
    throw std::invalid_argument("pcg: expected lambda0 of length " + std::to_string(dim) +
                                ", got " + std::to_string(lambda0->size()));
}
}  // namespace detail

/// random_problem.cpp:42-80 (host generator in libb2p, the reference's draw order).
inline KKTSystem random_kkt_family(int family, std::uint64_t seed, int N, int n, int m,
                                   double diag_floor = 0.1, double coupling = 1.0) {
  PackedKKT p;
  const size_t K = N + 1;
  p.Q.resize(K * n * n);
  p.q.resize(K * n);
  p.R.resize(static_cast<size_t>(N) * m * m);
  p.r.resize(static_cast<size_t>(N) * m);
  p.A.resize(static_cast<size_t>(N) * n * n);
  p.B.resize(static_cast<size_t>(N) * n * m);
  p.e.resize(static_cast<size_t>(N) * n);
  p.x_s.resize(n);
  p.x0.resize(n);
  b2p_kkt_out o{N, n, m, 0, p.Q.data(), p.q.data(), p.R.data(), p.r.data(), p.A.data(),
                p.B.data(), p.e.data(), p.x_s.data(), p.x0.data()};
  b2p_error e{};
  detail::raise(b2p_random_kkt(family, seed, N, n, m, diag_floor, coupling, &o, &e), e);
  KKTSystem s;
  s.N = N;
  s.n = n;
  s.m = m;
  s.knots.resize(N + 1);
  for (int k = 0; k <= N; ++k) {
    KnotData& kd = s.knots[k];
    kd.Q = Matrix(n, n);
    std::copy(p.Q.begin() + k * n * n, p.Q.begin() + (k + 1) * n * n, kd.Q.a.begin());
    kd.q.assign(p.q.begin() + k * n, p.q.begin() + (k + 1) * n);
    if (k < N) {
      kd.R = Matrix(m, m);
      std::copy(p.R.begin() + k * m * m, p.R.begin() + (k + 1) * m * m, kd.R.a.begin());
      kd.r.assign(p.r.begin() + k * m, p.r.begin() + (k + 1) * m);
      kd.A = Matrix(n, n);
      std::copy(p.A.begin() + k * n * n, p.A.begin() + (k + 1) * n * n, kd.A.a.begin());
      kd.B = Matrix(n, m);
      std::copy(p.B.begin() + k * n * m, p.B.begin() + (k + 1) * n * m, kd.B.a.begin());
      kd.e.assign(p.e.begin() + k * n, p.e.begin() + (k + 1) * n);
    }
  }
  s.x_s = p.x_s;
  s.x0 = p.x0;
  return s;
}
inline KKTSystem random_kkt(std::uint64_t seed, int N, int n, int m) {
  return random_kkt_family(0, seed, N, n, m);
}
inline KKTSystem random_kkt_scaled(std::uint64_t seed, int N, int n, int m, double diag_floor,
                                   double coupling) {
  return random_kkt_family(1, seed, N, n, m, diag_floor, coupling);
}
inline KKTSystem random_trajectory_kkt(std::uint64_t seed, int N, int n, int m) {
  return random_kkt_family(2, seed, N, n, m);
}

/// schur.hpp:19-56
enum class PrecondKind { identity, block_jacobi, stair, symmetric_stair, poly_split };
struct SchurSystem {
  BlockTriMatrix S;
  Vector gamma;
  std::vector<double> theta_inv;  // [K][n][n]
  int n = 0;
};
struct Preconditioner {
  PrecondKind kind = PrecondKind::identity;
  int order = 0;
  BlockTriMatrix phi_inv;
  const BlockTriMatrix* S = nullptr;  // poly_split: E = Psi - S is implied by S
};

inline std::string precond_name(PrecondKind kind, int order = 0) {
  switch (kind) {
    case PrecondKind::identity: return "identity";
    case PrecondKind::block_jacobi: return "jacobi";
    case PrecondKind::stair: return "stair";
    case PrecondKind::symmetric_stair: return "symstair";
    case PrecondKind::poly_split: return "poly:" + std::to_string(order);
  }
  return "unknown";
}

inline SchurSystem build_schur(const KKTSystem& kkt) {
  SchurSystem s;
  s.n = kkt.n;
  s.S = BlockTriMatrix(kkt.N + 1, kkt.n);
  s.gamma.resize(static_cast<size_t>(kkt.dual_dim()));
  s.theta_inv.resize(static_cast<size_t>(kkt.N + 1) * kkt.n * kkt.n);
  const PackedKKT p = pack(kkt);
  const b2p_kkt v = p.view(kkt.N, kkt.n, kkt.m);
  b2p_error e{};
  detail::raise(b2p_build_schur(detail::context(), B2P_F64, &v, s.S.data(), s.gamma.data(),
                                s.theta_inv.data(), &e),
                e);
  s.S.structurally_symmetric = true;
  return s;
}

inline Preconditioner build_preconditioner(const SchurSystem& s, PrecondKind kind, int order = 1) {
  Preconditioner P;
  P.kind = kind;
  P.order = kind == PrecondKind::poly_split ? order : 0;
  if (kind == PrecondKind::poly_split && order < 1)
    throw std::invalid_argument("build_poly_split: order must be >= 1, got " +
                                std::to_string(order));
  if (kind == PrecondKind::identity) return P;
  P.phi_inv = BlockTriMatrix(s.S.block_rows(), s.n);
  b2p_error e{};
  detail::raise(b2p_build_preconditioner(detail::context(), B2P_F64, static_cast<int>(kind),
                                         order, s.S.block_rows(), s.n, s.S.data(),
                                         s.theta_inv.data(), P.phi_inv.data(), &e),
                e);
  P.phi_inv.structurally_symmetric =
      kind == PrecondKind::block_jacobi || kind == PrecondKind::symmetric_stair;
  if (kind == PrecondKind::poly_split) P.S = &s.S;
  return P;
}
inline Preconditioner build_identity() { return Preconditioner{}; }
inline Preconditioner build_block_jacobi(const SchurSystem& s) {
  return build_preconditioner(s, PrecondKind::block_jacobi);
}
inline Preconditioner build_stair(const SchurSystem& s) {
  return build_preconditioner(s, PrecondKind::stair);
}
inline Preconditioner build_symmetric_stair(const SchurSystem& s) {
  return build_preconditioner(s, PrecondKind::symmetric_stair);
}
inline Preconditioner build_poly_split(const SchurSystem& s, int order) {
  return build_preconditioner(s, PrecondKind::poly_split, order);
}

inline Vector apply_preconditioner(const Preconditioner& P, const Vector& r) {
  if (P.kind == PrecondKind::identity) return r;
  Vector out(static_cast<size_t>(P.phi_inv.dim()));
  b2p_error e{};
  detail::raise(b2p_apply_preconditioner(detail::context(), B2P_F64, static_cast<int>(P.kind),
                                         P.order, P.phi_inv.block_rows(), P.phi_inv.block_dim(),
                                         P.S ? P.S->data() : nullptr, P.phi_inv.data(), r.data(),
                                         static_cast<int>(r.size()), out.data(), &e),
                e);
  return out;
}

/// pcg.hpp:12-70
enum class PcgVariant { sequential, block_parallel };
struct PcgConfig {
  double epsilon = 1e-4;
  int max_iter = 0;
  bool deterministic_reductions = false;
  PcgVariant variant = PcgVariant::sequential;
  bool collect_trace = false;
  bool check_residual_drift = false;
};
struct SolveReport {
  int iterations = 0;
  double exit_eta = 0.0;
  bool converged = false;
  std::vector<double> trace;
  double wall_time = 0.0;
  double max_residual_drift = 0.0;
};
struct PcgResult {
  Vector lambda;
  SolveReport report;
};

namespace detail {
inline b2p_pcg_config to_c(const PcgConfig& c) {
  return b2p_pcg_config{c.epsilon,
                        c.max_iter,
                        c.deterministic_reductions ? 1 : 0,
                        static_cast<int32_t>(c.variant),
                        c.collect_trace ? 1 : 0,
                        c.check_residual_drift ? 1 : 0,
                        0};
}
inline SolveReport from_c(const b2p_solve_report& r, const std::vector<double>& trace) {
  SolveReport s;
  s.iterations = r.iterations;
  s.exit_eta = r.exit_eta;
  s.converged = r.converged != 0;
  s.trace.assign(trace.begin(), trace.begin() + r.trace_len);
  s.wall_time = r.wall_time;
  s.max_residual_drift = r.max_residual_drift;
  return s;
}
}  // namespace detail

inline PcgResult pcg_solve_auto(const BlockTriMatrix& S, const Preconditioner& P,
                                const Vector& gamma, const Vector& lambda0, const PcgConfig& cfg) {
  const b2p_pcg_config c = detail::to_c(cfg);
  const int dim = S.dim();
  PcgResult out;
  out.lambda.resize(static_cast<size_t>(dim > 0 ? dim : 1));
  std::vector<double> trace(static_cast<size_t>(cfg.max_iter > 0 ? cfg.max_iter : dim) + 1);
  b2p_solve_report rep{};
  b2p_error e{};
  const bool id = P.kind == PrecondKind::identity;
  detail::raise(b2p_pcg_solve(detail::context(), B2P_F64, S.block_rows(), S.block_dim(), S.data(),
                              static_cast<int>(P.kind), P.order,
                              id ? 0 : P.phi_inv.block_rows(), id ? 0 : P.phi_inv.block_dim(),
                              id ? nullptr : P.phi_inv.data(), gamma.data(),
                              static_cast<int>(gamma.size()), lambda0.data(),
                              static_cast<int>(lambda0.size()), &c, out.lambda.data(), &rep,
                              trace.data(), &e),
                e);
  out.lambda.resize(static_cast<size_t>(dim));
  out.report = detail::from_c(rep, trace);
  return out;
}
inline PcgResult pcg_solve(const BlockTriMatrix& S, const Preconditioner& P, const Vector& gamma,
                           const Vector& lambda0, const PcgConfig& cfg) {
  PcgConfig c = cfg;
  c.variant = PcgVariant::sequential;
  return pcg_solve_auto(S, P, gamma, lambda0, c);
}
inline PcgResult pcg_solve_block_parallel(const BlockTriMatrix& S, const Preconditioner& P,
                                          const Vector& gamma, const Vector& lambda0,
                                          const PcgConfig& cfg) {
  PcgConfig c = cfg;
  c.variant = PcgVariant::block_parallel;
  return pcg_solve_auto(S, P, gamma, lambda0, c);
}

/// Fused hot path: build_schur -> build_preconditioner -> pcg_solve_auto.
inline PcgResult solve(const KKTSystem& kkt, PrecondKind kind, int order, const PcgConfig& cfg,
                       const Vector* lambda0 = nullptr) {
  detail::check_lambda0(lambda0, kkt.dual_dim());
  const PackedKKT p = pack(kkt);
  const b2p_kkt v = p.view(kkt.N, kkt.n, kkt.m);
  const b2p_pcg_config c = detail::to_c(cfg);
  PcgResult out;
  out.lambda.resize(static_cast<size_t>(kkt.dual_dim()));
  std::vector<double> trace(static_cast<size_t>(cfg.max_iter > 0 ? cfg.max_iter : kkt.dual_dim()) + 1);
  b2p_solve_report rep{};
  b2p_error e{};
  detail::raise(b2p_solve(detail::context(), B2P_F64, &v, static_cast<int>(kind), order, &c,
                          lambda0 ? lambda0->data() : nullptr, out.lambda.data(), &rep,
                          trace.data(), &e),
                e);
  out.report = detail::from_c(rep, trace);
  return out;
}

/// VectorXd reconstruct_primal(const KKTSystem&, const VectorXd& lambda) (kkt.hpp; kkt.cpp:153-181).
inline Vector reconstruct_primal(const KKTSystem& kkt, const Vector& lambda) {
  const PackedKKT p = pack(kkt);
  const b2p_kkt v = p.view(kkt.N, kkt.n, kkt.m);
  Vector dz(static_cast<size_t>(kkt.N + 1) * kkt.n + static_cast<size_t>(kkt.N) * kkt.m);
  b2p_error e{};
  detail::raise(b2p_reconstruct_primal(detail::context(), B2P_F64, &v, lambda.data(),
                                       static_cast<int>(lambda.size()), dz.data(), &e),
                e);
  return dz;
}

/// The SQP linear step (sqp.cpp:171-176) in one library call: fused
/// build_schur -> build_preconditioner -> pcg_solve_auto(lambda0), then
/// reconstruct_primal on the knots already resident on the device.
struct SqpStepResult {
  PcgResult pcg;
  Vector dz;
};
inline SqpStepResult sqp_step(const KKTSystem& kkt, PrecondKind kind, int order,
                              const PcgConfig& cfg, const Vector& lambda0) {
  if (!lambda0.empty()) detail::check_lambda0(&lambda0, kkt.dual_dim());
  const PackedKKT p = pack(kkt);
  const b2p_kkt v = p.view(kkt.N, kkt.n, kkt.m);
  const b2p_pcg_config c = detail::to_c(cfg);
  SqpStepResult out;
  out.pcg.lambda.resize(static_cast<size_t>(kkt.dual_dim()));
  out.dz.resize(static_cast<size_t>(kkt.N + 1) * kkt.n + static_cast<size_t>(kkt.N) * kkt.m);
  std::vector<double> trace(static_cast<size_t>(cfg.max_iter > 0 ? cfg.max_iter : kkt.dual_dim()) + 1);
  b2p_solve_report rep{};
  b2p_error e{};
  detail::raise(b2p_sqp_step(detail::context(), B2P_F64, &v, static_cast<int>(kind), order, &c,
                             lambda0.empty() ? nullptr : lambda0.data(), out.pcg.lambda.data(),
                             out.dz.data(), &rep, trace.data(), &e),
                e);
  out.pcg.report = detail::from_c(rep, trace);
  return out;
}

}  // namespace trajopt_b200

#if defined(__has_include)
#if __has_include(<Eigen/Dense>)
#include <Eigen/Dense>
namespace trajopt_b200 {
// Eigen bridge: the reference's callers pass Eigen::VectorXd / MatrixXd and
// the Eigen-typed trajopt::KKTSystem (kkt.hpp:13-46). Callers that want the
// reference's own signatures instead use the drop-in headers under
// include/trajopt_dropin.
inline Vector from_eigen(const Eigen::VectorXd& v) { return Vector(v.data(), v.data() + v.size()); }
inline Eigen::VectorXd to_eigen(const Vector& v) {
  return Eigen::Map<const Eigen::VectorXd>(v.data(), static_cast<Eigen::Index>(v.size()));
}
inline Matrix from_eigen(const Eigen::MatrixXd& M) {
  Matrix out(static_cast<int>(M.rows()), static_cast<int>(M.cols()));
  for (int i = 0; i < out.rows; ++i)
    for (int j = 0; j < out.cols; ++j) out(i, j) = M(i, j);  // column-major -> row-major
  return out;
}
/// trajopt::KKTSystem (or any type with the reference's field names: N, n, m,
/// knots[k].{Q,q,R,r,A,B,e}, x_s, x0) -> this adapter's row-major KKTSystem.
template <class EigenKKT>
inline KKTSystem to_b200(const EigenKKT& kkt) {
  KKTSystem s;
  s.N = kkt.N;
  s.n = kkt.n;
  s.m = kkt.m;
  s.knots.resize(static_cast<size_t>(kkt.N) + 1);
  for (int k = 0; k <= kkt.N; ++k) {
    const auto& kd = kkt.knots[k];
    KnotData& o = s.knots[k];
    o.Q = from_eigen(Eigen::MatrixXd(kd.Q));
    o.q = from_eigen(Eigen::VectorXd(kd.q));
    if (k < kkt.N) {
      o.R = from_eigen(Eigen::MatrixXd(kd.R));
      o.r = from_eigen(Eigen::VectorXd(kd.r));
      o.A = from_eigen(Eigen::MatrixXd(kd.A));
      o.B = from_eigen(Eigen::MatrixXd(kd.B));
      o.e = from_eigen(Eigen::VectorXd(kd.e));
    }
  }
  s.x_s = from_eigen(Eigen::VectorXd(kkt.x_s));
  s.x0 = from_eigen(Eigen::VectorXd(kkt.x0));
  return s;
}
}  // namespace trajopt_b200
#endif
#endif
