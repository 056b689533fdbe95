// trajopt_b200_sqp.hpp — the reference's callers of the hot path, over the
// B200 adapter (trajopt_b200.hpp): dynamics models and tracking cost
// (proj/include/trajopt/models.hpp, proj/src/models.cpp), the KKT
// linearisation (proj/src/kkt.cpp:83-127), the SQP outer loop with the
// parallel L1-merit line search (proj/include/trajopt/sqp.hpp,
// proj/src/sqp.cpp) and the receding-horizon NMPC loop with shifted
// multiplier warm starts (proj/include/trajopt/nmpc.hpp, proj/src/nmpc.cpp).
// SURVEY.md §8(f) rank 2.
//
// Host-side control flow only: every linear step goes to the GPU through ONE
// library call, b2p_sqp_step (fused build_schur -> build_preconditioner ->
// pcg_solve_auto(lambda warm start) -> reconstruct_primal on one upload of the
// knots). The per-knot model evaluations (n <= 4 here) stay on the host, as
// in the reference. Same names, value types, defaults and exception texts as
// the reference; Eigen-free storage (row-major Matrix / std::vector) so it
// builds in this image. Link with libb2p.so.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <limits>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "trajopt_b200.hpp"

namespace trajopt_b200 {

/// trajectory.hpp:9-17 — N+1 states, N controls, multipliers of the last solve.
struct Trajectory {
  double h = 0.01;
  std::vector<Vector> X;
  std::vector<Vector> U;
  Vector lambda;  // (N+1)*n; size 0 means "start from zero"
  int horizon() const { return static_cast<int>(U.size()); }
};

namespace la {
inline Vector matvec(const Matrix& M, const Vector& x) {
  Vector y(static_cast<size_t>(M.rows), 0.0);
  for (int i = 0; i < M.rows; ++i) {
    double s = 0.0;
    for (int j = 0; j < M.cols; ++j) s += M(i, j) * x[j];
    y[i] = s;
  }
  return y;
}
inline double dot(const Vector& a, const Vector& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
inline Vector sub(const Vector& a, const Vector& b) {
  Vector c(a.size());
  for (size_t i = 0; i < a.size(); ++i) c[i] = a[i] - b[i];
  return c;
}
inline double norm1(const Vector& a) {
  double s = 0.0;
  for (double v : a) s += std::abs(v);
  return s;
}
inline double norm_inf(const Vector& a) {
  double s = 0.0;
  for (double v : a) s = std::max(s, std::abs(v));
  return s;
}
inline bool finite(const Vector& a) {
  for (double v : a)
    if (!std::isfinite(v)) return false;
  return true;
}
inline bool finite(const Matrix& M) { return finite(M.a); }

/// Smallest eigenvalue of the symmetric matrix stored in W's lower triangle
/// (Eigen's SelfAdjointEigenSolver reads only the lower triangle), by cyclic
/// Jacobi rotations — the matrices here are n x n with n <= a few dozen.
inline double min_eigenvalue_lower(const Matrix& W) {
  const int n = W.rows;
  if (n == 0) return std::numeric_limits<double>::infinity();
  Matrix a(n, n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) a(i, j) = a(j, i) = W(i, j);
  for (int sweep = 0; sweep < 64; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int i = 0; i < n; ++i) {
      diag += a(i, i) * a(i, i);
      for (int j = i + 1; j < n; ++j) off += a(i, j) * a(i, j);
    }
    if (!(off > 1e-30 * diag)) break;  // also exits on NaN
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        if (a(p, q) == 0.0) continue;
        const double theta = (a(q, q) - a(p, p)) / (2.0 * a(p, q));
        const double t = (theta >= 0 ? 1.0 : -1.0) /
                         (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double akp = a(k, p), akq = a(k, q);
          a(k, p) = c * akp - s * akq;
          a(k, q) = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = a(p, k), aqk = a(q, k);
          a(p, k) = c * apk - s * aqk;
          a(q, k) = s * apk + c * aqk;
        }
      }
  }
  double mn = a(0, 0);
  for (int i = 1; i < n; ++i) mn = std::min(mn, a(i, i));
  return mn;
}
}  // namespace la

/// format.hpp:9-13 — locale-independent "%.9g".
inline std::string format9(double v) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.9g", v);
  return buf;
}

// --------------------------------------------------------------- models.hpp
/// models.hpp:14-27 — x+ = step(x, u, h) with analytic Jacobians.
class DynamicsModel {
 public:
  virtual ~DynamicsModel() = default;
  virtual int state_dim() const = 0;
  virtual int control_dim() const = 0;
  virtual std::string name() const = 0;
  virtual Vector step(const Vector& x, const Vector& u, double h) const = 0;
  virtual void jacobians(const Vector& x, const Vector& u, double h, Matrix& A,
                         Matrix& B) const = 0;
};

namespace models_detail {
/// models.cpp:14-34 — pos+ = pos + h vel, vel+ = vel + h u.
class DoubleIntegrator final : public DynamicsModel {
 public:
  int state_dim() const override { return 2; }
  int control_dim() const override { return 1; }
  std::string name() const override { return "double_integrator"; }
  Vector step(const Vector& x, const Vector& u, double h) const override {
    return {x[0] + h * x[1], x[1] + h * u[0]};
  }
  void jacobians(const Vector&, const Vector&, double h, Matrix& A, Matrix& B) const override {
    A = Matrix::identity(2);
    A(0, 1) = h;
    B = Matrix(2, 1);
    B(1, 0) = h;
  }
};

/// models.cpp:36-66 — point-mass pendulum, theta = 0 hanging down.
class Pendulum final : public DynamicsModel {
 public:
  int state_dim() const override { return 2; }
  int control_dim() const override { return 1; }
  std::string name() const override { return "pendulum"; }
  Vector step(const Vector& x, const Vector& u, double h) const override {
    return {x[0] + h * x[1],
            x[1] + h * (u[0] - kMass * kGravity * kLength * std::sin(x[0])) /
                       (kMass * kLength * kLength)};
  }
  void jacobians(const Vector& x, const Vector&, double h, Matrix& A, Matrix& B) const override {
    A = Matrix::identity(2);
    A(0, 1) = h;
    A(1, 0) = -h * kGravity * std::cos(x[0]) / kLength;
    B = Matrix(2, 1);
    B(1, 0) = h / (kMass * kLength * kLength);
  }

 private:
  static constexpr double kMass = 1.0, kLength = 1.0, kGravity = 9.81;
};

/// models.cpp:68-149 — cart-pole, pole angle from upright, force on the cart.
class Cartpole final : public DynamicsModel {
 public:
  int state_dim() const override { return 4; }
  int control_dim() const override { return 1; }
  std::string name() const override { return "cartpole"; }
  Vector step(const Vector& x, const Vector& u, double h) const override {
    const double s = std::sin(x[1]), c = std::cos(x[1]);
    const double total = kMassCart + kMassPole;
    const double temp = (u[0] + kMassPole * kLength * x[3] * x[3] * s) / total;
    const double tdd =
        (kGravity * s - c * temp) / (kLength * (4.0 / 3.0 - kMassPole * c * c / total));
    const double xdd = temp - kMassPole * kLength * tdd * c / total;
    return {x[0] + h * x[2], x[1] + h * x[3], x[2] + h * xdd, x[3] + h * tdd};
  }
  void jacobians(const Vector& x, const Vector& u, double h, Matrix& A, Matrix& B) const override {
    const double theta = x[1], td = x[3], f = u[0];
    const double s = std::sin(theta), c = std::cos(theta);
    const double total = kMassCart + kMassPole;
    const double temp = (f + kMassPole * kLength * td * td * s) / total;
    const double num = kGravity * s - c * temp;
    const double den = kLength * (4.0 / 3.0 - kMassPole * c * c / total);
    const double tdd = num / den;
    const double dtemp_dtheta = kMassPole * kLength * td * td * c / total;
    const double dtemp_dtd = 2.0 * kMassPole * kLength * td * s / total;
    const double dtemp_df = 1.0 / total;
    const double dnum_dtheta = kGravity * c + s * temp - c * dtemp_dtheta;
    const double dnum_dtd = -c * dtemp_dtd;
    const double dnum_df = -c * dtemp_df;
    const double dden_dtheta = 2.0 * kLength * kMassPole * c * s / total;
    const double dtdd_dtheta = (dnum_dtheta * den - num * dden_dtheta) / (den * den);
    const double dtdd_dtd = dnum_dtd / den;
    const double dtdd_df = dnum_df / den;
    const double scale = kMassPole * kLength / total;
    const double dxdd_dtheta = dtemp_dtheta - scale * (dtdd_dtheta * c - tdd * s);
    const double dxdd_dtd = dtemp_dtd - scale * c * dtdd_dtd;
    const double dxdd_df = dtemp_df - scale * c * dtdd_df;
    A = Matrix::identity(4);
    A(0, 2) = h;
    A(1, 3) = h;
    A(2, 1) = h * dxdd_dtheta;
    A(2, 3) = h * dxdd_dtd;
    A(3, 1) = h * dtdd_dtheta;
    A(3, 3) = 1.0 + h * dtdd_dtd;
    B = Matrix(4, 1);
    B(2, 0) = h * dxdd_df;
    B(3, 0) = h * dtdd_df;
  }

 private:
  static constexpr double kMassCart = 1.0, kMassPole = 0.1, kLength = 0.5, kGravity = 9.81;
};
}  // namespace models_detail

inline std::unique_ptr<DynamicsModel> double_integrator() {
  return std::make_unique<models_detail::DoubleIntegrator>();
}
inline std::unique_ptr<DynamicsModel> pendulum() {
  return std::make_unique<models_detail::Pendulum>();
}
inline std::unique_ptr<DynamicsModel> cartpole() {
  return std::make_unique<models_detail::Cartpole>();
}
/// models.cpp:155-161
inline std::unique_ptr<DynamicsModel> make_model(const std::string& name) {
  if (name == "double_integrator") return double_integrator();
  if (name == "pendulum") return pendulum();
  if (name == "cartpole") return cartpole();
  throw std::invalid_argument("unknown model \"" + name +
                              "\" (expected double_integrator, pendulum, or cartpole)");
}

/// models.hpp:35-50 — l = 1/2 (x-g)' Wx (x-g) + 1/2 u' Wu u, l_f = 1/2 (x-g)' WN (x-g).
struct CostModel {
  Matrix Wx, Wu, WN;
  std::vector<Vector> goals;  // size 1 (broadcast) or N+1
  const Vector& goal(int knot) const {
    return goals.size() == 1 ? goals.front() : goals.at(static_cast<size_t>(knot));
  }
};

inline CostModel quadratic_tracking_cost(const Matrix& Wx, const Matrix& Wu, const Matrix& WN,
                                         const Vector& goal) {  // models.cpp:163-171
  CostModel c;
  c.Wx = Wx;
  c.Wu = Wu;
  c.WN = WN;
  c.goals = {goal};
  return c;
}

inline double eval_cost(const CostModel& cost, const std::vector<Vector>& X,
                        const std::vector<Vector>& U) {  // models.cpp:173-189
  if (X.size() != U.size() + 1)
    throw std::invalid_argument("eval_cost: need N+1 states and N controls, got " +
                                std::to_string(X.size()) + " states and " +
                                std::to_string(U.size()) + " controls");
  const int N = static_cast<int>(U.size());
  double total = 0.0;
  for (int k = 0; k < N; ++k) {
    const Vector dx = la::sub(X[k], cost.goal(k));
    total += 0.5 * la::dot(dx, la::matvec(cost.Wx, dx)) +
             0.5 * la::dot(U[k], la::matvec(cost.Wu, U[k]));
  }
  const Vector dxN = la::sub(X[N], cost.goal(N));
  return total + 0.5 * la::dot(dxN, la::matvec(cost.WN, dxN));
}
inline double eval_cost(const CostModel& cost, const Trajectory& traj) {
  return eval_cost(cost, traj.X, traj.U);
}

inline Trajectory rollout(const DynamicsModel& model, const Vector& x0,
                          const std::vector<Vector>& controls, double h) {  // models.cpp:191-200
  Trajectory t;
  t.h = h;
  t.U = controls;
  t.X.reserve(controls.size() + 1);
  t.X.push_back(x0);
  for (const auto& u : controls) t.X.push_back(model.step(t.X.back(), u, h));
  return t;
}

// --------------------------------------------------------------- kkt.cpp
namespace kkt_detail {
constexpr double kEigFloor = 1e-8;  // kkt.cpp:17-18
constexpr double kRidge = 1e-6;
inline void regularize_spd(Matrix& W) {  // kkt.cpp:20-25
  if (la::min_eigenvalue_lower(W) < kEigFloor)
    for (int i = 0; i < W.rows; ++i) W(i, i) += kRidge;
}
}  // namespace kkt_detail

/// kkt.cpp:83-127 — linearise the dynamics and expand the cost around traj.
inline KKTSystem assemble_kkt(const Trajectory& traj, const DynamicsModel& model,
                              const CostModel& cost, const Vector& x_s) {
  const int N = traj.horizon(), n = model.state_dim(), m = model.control_dim();
  if (static_cast<int>(traj.X.size()) != N + 1)
    throw std::invalid_argument("assemble_kkt: trajectory needs N+1 states, got " +
                                std::to_string(traj.X.size()) + " for N = " + std::to_string(N));
  KKTSystem kkt;
  kkt.N = N;
  kkt.n = n;
  kkt.m = m;
  kkt.x_s = x_s;
  kkt.x0 = traj.X[0];
  kkt.knots.resize(static_cast<size_t>(N) + 1);
  for (int k = 0; k <= N; ++k) {
    KnotData& kd = kkt.knots[k];
    const bool terminal = k == N;
    kd.Q = terminal ? cost.WN : cost.Wx;
    kd.q = la::matvec(kd.Q, la::sub(traj.X[k], cost.goal(k)));
    kkt_detail::regularize_spd(kd.Q);
    if (!terminal) {
      kd.R = cost.Wu;
      kd.r = la::matvec(kd.R, traj.U[k]);
      kkt_detail::regularize_spd(kd.R);
      model.jacobians(traj.X[k], traj.U[k], traj.h, kd.A, kd.B);
      kd.e = la::sub(traj.X[k + 1], model.step(traj.X[k], traj.U[k], traj.h));
      if (!la::finite(kd.A) || !la::finite(kd.B) || !la::finite(kd.e) || !la::finite(kd.R) ||
          !la::finite(kd.r))
        throw std::runtime_error("assemble_kkt: non-finite linearization at knot " +
                                 std::to_string(k));
    }
    if (!la::finite(kd.Q) || !la::finite(kd.q))
      throw std::runtime_error("assemble_kkt: non-finite cost expansion at knot " +
                               std::to_string(k));
  }
  return kkt;
}

// --------------------------------------------------------------- sqp.hpp
struct MeritParams {  // sqp.hpp:16-23
  enum class MuRule { fixed, multiplier_max };
  double mu = 10.0;
  std::vector<double> alphas = {1.0, 0.5, 0.25, 0.125, 0.0625, 0.03125, 0.015625, 0.0078125};
  MuRule mu_rule = MuRule::fixed;
};

enum class SolverBackend { schur_pcg, dense_kkt };  // sqp.hpp:25

/// One SQP linear step: the multipliers, the primal step dz and the PCG report.
struct QpStep {
  Vector lambda;
  Vector dz;
  SolveReport report;
};
struct SqpConfig;
using QpSolver = std::function<QpStep(const KKTSystem&, const Vector& lambda0, const SqpConfig&)>;

struct SqpConfig {  // sqp.hpp:27-37 (field order preserved; qp_solver is an extension)
  int max_sqp_iter = 10;
  PcgConfig pcg;
  MeritParams merit;
  PrecondKind precond = PrecondKind::symmetric_stair;
  int poly_order = 1;
  double time_budget = 0.0;
  SolverBackend backend = SolverBackend::schur_pcg;
  /// Replaces the linear step. Empty: schur_pcg runs b2p_sqp_step on the GPU;
  /// dense_kkt (the reference's dense FullPivLU check backend, kkt.cpp:129-151)
  /// has no device implementation and must be supplied here.
  QpSolver qp_solver;
};

struct LineSearchResult {  // sqp.hpp:39-44
  double alpha = 0.0;
  Trajectory traj;
  double merit = 0.0;
  bool progress = false;
};
struct SqpIterStats {  // sqp.hpp:46-54
  int iter = 0;
  double mu = 0.0;
  double merit_before = 0.0;
  double merit_after = 0.0;
  double alpha = 0.0;
  double constraint_l1 = 0.0;
  SolveReport pcg;
};
struct SqpStats {  // sqp.hpp:56-61
  std::vector<SqpIterStats> iters;
  double wall_time = 0.0;
  bool hit_budget = false;
  bool stalled = false;
};
struct SqpResult {  // sqp.hpp:63-67
  Trajectory traj;
  Vector lambda;
  SqpStats stats;
};

namespace sqp_detail {
inline void validate_merit_params(const MeritParams& p) {  // sqp.cpp:19-33
  if (p.mu <= 0.0) throw std::invalid_argument("merit: mu must be positive");
  const auto& a = p.alphas;
  if (a.empty() || a.front() != 1.0)
    throw std::invalid_argument("line search: alpha set must start at 1");
  for (size_t i = 0; i < a.size(); ++i)
    if (a[i] <= 0.0 || a[i] > 1.0 || (i > 0 && a[i] >= a[i - 1]))
      throw std::invalid_argument("line search: alphas must be strictly descending in (0, 1]");
}
}  // namespace sqp_detail

/// sqp.cpp:37-43 — |x_s - x_0|_1 + sum_k |x_{k+1} - f(x_k, u_k)|_1.
inline double constraint_l1(const Trajectory& traj, const DynamicsModel& model, const Vector& x_s) {
  double total = la::norm1(la::sub(x_s, traj.X[0]));
  for (int k = 0; k < traj.horizon(); ++k)
    total += la::norm1(la::sub(traj.X[k + 1], model.step(traj.X[k], traj.U[k], traj.h)));
  return total;
}

/// sqp.cpp:45-48 — M = J + mu |c|_1.
inline double merit(const Trajectory& traj, const DynamicsModel& model, const CostModel& cost,
                    const Vector& x_s, double mu) {
  return eval_cost(cost, traj) + mu * constraint_l1(traj, model, x_s);
}

/// sqp.cpp:50-61 — lowest finite merit, ties to the largest alpha; -1 if none improves.
inline int select_line_search_candidate(double current_merit, const double* merits, size_t count) {
  int best = -1;
  double best_merit = std::numeric_limits<double>::infinity();
  for (size_t i = 0; i < count; ++i)
    if (std::isfinite(merits[i]) && merits[i] < best_merit) {
      best_merit = merits[i];
      best = static_cast<int>(i);
    }
  if (best < 0 || best_merit >= current_merit) return -1;
  return best;
}
inline int select_line_search_candidate(double current_merit, const std::vector<double>& merits) {
  return select_line_search_candidate(current_merit, merits.data(), merits.size());
}

/// sqp.cpp:63-80 — traj + alpha dz, knot by knot.
inline Trajectory apply_step(const Trajectory& traj, const Vector& dz, double alpha) {
  const int N = traj.horizon();
  const int n = static_cast<int>(traj.X[0].size());
  const int m = N > 0 ? static_cast<int>(traj.U[0].size()) : 0;
  const size_t want = static_cast<size_t>(N + 1) * n + static_cast<size_t>(N) * m;
  if (dz.size() != want)
    throw std::invalid_argument("apply_step: expected dz of length " + std::to_string(want) +
                                ", got " + std::to_string(dz.size()));
  Trajectory out = traj;
  const int stride = n + m;
  for (int k = 0; k <= N; ++k) {
    for (int i = 0; i < n; ++i) out.X[k][i] += alpha * dz[static_cast<size_t>(k) * stride + i];
    if (k < N)
      for (int i = 0; i < m; ++i)
        out.U[k][i] += alpha * dz[static_cast<size_t>(k) * stride + n + i];
  }
  return out;
}

/// sqp.cpp:82-123. The candidates are independent; at these sizes (n <= 4,
/// a few dozen knots) evaluating them in turn costs less than spawning the
/// reference's worker threads, and the selected candidate is the same.
inline LineSearchResult parallel_line_search(const Trajectory& traj, const Vector& dz,
                                             const DynamicsModel& model, const CostModel& cost,
                                             const MeritParams& params, const Vector& x_s) {
  sqp_detail::validate_merit_params(params);
  const double current = merit(traj, model, cost, x_s, params.mu);
  const size_t count = params.alphas.size();
  std::vector<double> merits(count, std::numeric_limits<double>::infinity());
  std::vector<Trajectory> candidates(count);
  for (size_t i = 0; i < count; ++i) {
    candidates[i] = apply_step(traj, dz, params.alphas[i]);
    const double mv = merit(candidates[i], model, cost, x_s, params.mu);
    if (std::isfinite(mv)) merits[i] = mv;
  }
  if (std::none_of(merits.begin(), merits.end(), [](double v) { return std::isfinite(v); }))
    throw std::runtime_error("line search: merit is non-finite at every candidate step");
  const int best = select_line_search_candidate(current, merits);
  LineSearchResult out;
  if (best < 0) {
    out.alpha = 0.0;
    out.traj = traj;
    out.merit = current;
    out.progress = false;
  } else {
    out.alpha = params.alphas[best];
    out.traj = std::move(candidates[best]);
    out.merit = merits[best];
    out.progress = true;
  }
  return out;
}

/// The default schur_pcg linear step (sqp.cpp:171-176) on the GPU.
inline QpStep gpu_qp_step(const KKTSystem& kkt, const Vector& lambda0, const SqpConfig& cfg) {
  SqpStepResult r = sqp_step(kkt, cfg.precond, cfg.poly_order, cfg.pcg, lambda0);
  return QpStep{std::move(r.pcg.lambda), std::move(r.dz), std::move(r.pcg.report)};
}

/// sqp.cpp:125-197 — linearise -> Schur/PCG (lambda warm start) -> reconstruct
/// -> parallel line search, until max_sqp_iter, the time budget, or two
/// consecutive zero-progress line searches.
inline SqpResult sqp_solve(const Trajectory& traj0, const Vector& lambda0, const Vector& x_s,
                           const DynamicsModel& model, const CostModel& cost,
                           const SqpConfig& cfg) {
  using Clock = std::chrono::steady_clock;
  if (cfg.max_sqp_iter < 1) throw std::invalid_argument("sqp_solve: max_sqp_iter must be >= 1");
  sqp_detail::validate_merit_params(cfg.merit);
  if (cfg.backend == SolverBackend::dense_kkt && !cfg.qp_solver)
    throw std::invalid_argument(
        "sqp_solve: the dense_kkt backend has no device implementation; pass "
        "SqpConfig::qp_solver or use schur_pcg");
  const QpSolver step = cfg.qp_solver ? cfg.qp_solver : QpSolver(gpu_qp_step);
  const auto start = Clock::now();
  const int n = model.state_dim();
  const int dual_dim = (traj0.horizon() + 1) * n;
  Trajectory traj = traj0;
  Vector lambda = !lambda0.empty() ? lambda0 : Vector(static_cast<size_t>(dual_dim), 0.0);
  if (static_cast<int>(lambda.size()) != dual_dim)
    throw std::invalid_argument("sqp_solve: expected lambda0 of length " +
                                std::to_string(dual_dim) + ", got " +
                                std::to_string(lambda0.size()));
  SqpResult result;
  int zero_progress = 0;
  for (int it = 1; it <= cfg.max_sqp_iter; ++it) {
    if (cfg.time_budget > 0.0 && it > 1) {
      const double elapsed = std::chrono::duration<double>(Clock::now() - start).count();
      if (elapsed >= cfg.time_budget) {
        result.stats.hit_budget = true;
        break;
      }
    }
    const KKTSystem kkt = assemble_kkt(traj, model, cost, x_s);
    double mu = cfg.merit.mu;
    if (cfg.merit.mu_rule == MeritParams::MuRule::multiplier_max)
      mu = std::max(la::norm_inf(lambda) * 1.1, cfg.merit.mu);
    SqpIterStats st;
    st.iter = it;
    st.mu = mu;
    st.constraint_l1 = constraint_l1(traj, model, x_s);
    st.merit_before = eval_cost(cost, traj) + mu * st.constraint_l1;

    QpStep qp = step(kkt, lambda, cfg);
    lambda = std::move(qp.lambda);
    if (cfg.backend == SolverBackend::schur_pcg) st.pcg = std::move(qp.report);

    MeritParams ls_params = cfg.merit;
    ls_params.mu = mu;
    ls_params.mu_rule = MeritParams::MuRule::fixed;
    LineSearchResult ls = parallel_line_search(traj, qp.dz, model, cost, ls_params, x_s);
    st.alpha = ls.alpha;
    st.merit_after = ls.merit;
    result.stats.iters.push_back(std::move(st));
    if (!ls.progress) {
      if (++zero_progress >= 2) {
        result.stats.stalled = true;
        break;
      }
    } else {
      zero_progress = 0;
      traj = std::move(ls.traj);
    }
  }
  result.stats.wall_time = std::chrono::duration<double>(Clock::now() - start).count();
  traj.lambda = lambda;
  result.traj = std::move(traj);
  result.lambda = std::move(lambda);
  return result;
}

/// sqp.cpp:199-216
inline std::string sqp_stats_csv(const SqpStats& stats) {
  std::ostringstream out;
  out << "iter,mu,merit_before,merit_after,alpha,constraint_l1,pcg_iterations,pcg_exit_eta,"
         "pcg_converged,pcg_wall_us\n";
  for (const auto& it : stats.iters)
    out << it.iter << ',' << format9(it.mu) << ',' << format9(it.merit_before) << ','
        << format9(it.merit_after) << ',' << format9(it.alpha) << ','
        << format9(it.constraint_l1) << ',' << it.pcg.iterations << ','
        << format9(it.pcg.exit_eta) << ',' << (it.pcg.converged ? "true" : "false") << ','
        << static_cast<long long>(it.pcg.wall_time * 1e6) << '\n';
  return out.str();
}

// --------------------------------------------------------------- nmpc.hpp
struct TimedGoal {  // nmpc.hpp:12-15
  double t = 0.0;
  Vector state;
};
struct NmpcConfig {  // nmpc.hpp:17-33
  double control_rate = 100.0;
  double sim_duration = 10.0;
  int N = 32;
  double h = 0.01;
  Vector x0;
  std::vector<TimedGoal> goals;
  SqpConfig solver;
  int sim_substeps = 4;
  bool warm_start_lambda = true;
  bool deterministic = false;
};
struct NmpcStepRecord {  // nmpc.hpp:35-43
  int step = 0;
  double time_s = 0.0;
  double solve_us = 0.0;
  int sqp_iters = 0;
  long pcg_iters_total = 0;
  double tracking_err = 0.0;
  bool overrun = false;
};
struct NmpcStats {  // nmpc.hpp:45-59
  std::vector<NmpcStepRecord> steps;
  std::vector<SqpStats> sqp_traces;
  std::vector<Vector> plant_trace;
  std::vector<double> segment_errors;
  double mean_solve_us = 0.0;
  double median_solve_us = 0.0;
  double p95_solve_us = 0.0;
  double max_solve_us = 0.0;
  int overruns = 0;
  bool deterministic = false;
};

namespace nmpc_detail {
inline double percentile(std::vector<double> v, double q) {  // nmpc.cpp:13-21
  if (v.empty()) return 0.0;
  std::sort(v.begin(), v.end());
  const double pos = q * (static_cast<double>(v.size()) - 1.0);
  const size_t lo = static_cast<size_t>(pos);
  const size_t hi = std::min(lo + 1, v.size() - 1);
  const double frac = pos - static_cast<double>(lo);
  return v[lo] * (1.0 - frac) + v[hi] * frac;
}
inline const Vector& active_goal(const std::vector<TimedGoal>& goals, double t) {  // :23-29
  const Vector* cur = &goals.front().state;
  for (const auto& g : goals)
    if (g.t <= t) cur = &g.state;
  return *cur;
}
}  // namespace nmpc_detail

/// nmpc.cpp:33-47 — shift states, controls and multipliers one knot earlier;
/// the vacated last knot duplicates its predecessor.
inline Trajectory shift_warm_start(const Trajectory& traj) {
  const int N = traj.horizon();
  Trajectory out = traj;
  for (int k = 0; k < N; ++k) out.X[k] = traj.X[k + 1];
  for (int k = 0; k + 1 < N; ++k) out.U[k] = traj.U[k + 1];
  if (!traj.lambda.empty()) {
    const int n = static_cast<int>(traj.X[0].size());
    for (int k = 0; k < N; ++k)
      for (int i = 0; i < n; ++i)
        out.lambda[static_cast<size_t>(k) * n + i] = traj.lambda[static_cast<size_t>(k + 1) * n + i];
  }
  return out;
}

/// nmpc.cpp:49-147 — measure, budgeted SQP solve (GPU linear steps), apply the
/// first control for one period (zero-order hold, sim_substeps Euler
/// substeps), shift-warm-start, repeat.
inline NmpcStats run_nmpc(const NmpcConfig& cfg, const DynamicsModel& model,
                          const CostModel& cost) {
  if (cfg.control_rate <= 0.0) throw std::invalid_argument("run_nmpc: control_rate must be > 0");
  if (cfg.N < 2) throw std::invalid_argument("run_nmpc: N must be >= 2");
  if (cfg.goals.empty()) throw std::invalid_argument("run_nmpc: goal sequence is empty");
  if (cfg.sim_substeps < 1) throw std::invalid_argument("run_nmpc: sim_substeps must be >= 1");
  const int n = model.state_dim(), m = model.control_dim();
  const double period = 1.0 / cfg.control_rate;
  const int steps = static_cast<int>(std::llround(cfg.control_rate * cfg.sim_duration));
  SqpConfig solver = cfg.solver;
  solver.time_budget = cfg.deterministic ? 0.0 : period;
  Vector plant = !cfg.x0.empty() ? cfg.x0 : Vector(static_cast<size_t>(n), 0.0);
  Trajectory traj;
  traj.h = cfg.h;
  traj.X.assign(static_cast<size_t>(cfg.N) + 1, plant);
  traj.U.assign(static_cast<size_t>(cfg.N), Vector(static_cast<size_t>(m), 0.0));
  traj.lambda.assign(static_cast<size_t>(cfg.N + 1) * n, 0.0);
  CostModel step_cost = cost;
  const int pos_dims = std::max(1, n / 2);
  NmpcStats stats;
  stats.deterministic = cfg.deterministic;
  stats.steps.reserve(static_cast<size_t>(std::max(steps, 0)));
  for (int step = 0; step < steps; ++step) {
    const double t = static_cast<double>(step) * period;
    const Vector& goal = nmpc_detail::active_goal(cfg.goals, t);
    step_cost.goals = {goal};
    const Vector x_s = plant;
    if (step > 0) traj = shift_warm_start(traj);
    const Vector lambda0 = cfg.warm_start_lambda
                               ? traj.lambda
                               : Vector(static_cast<size_t>(cfg.N + 1) * n, 0.0);
    SqpResult solve = sqp_solve(traj, lambda0, x_s, model, step_cost, solver);
    traj = std::move(solve.traj);
    NmpcStepRecord rec;
    rec.step = step;
    rec.time_s = t;
    rec.solve_us = solve.stats.wall_time * 1e6;
    rec.sqp_iters = static_cast<int>(solve.stats.iters.size());
    for (const auto& it : solve.stats.iters) rec.pcg_iters_total += it.pcg.iterations;
    double err2 = 0.0;
    for (int i = 0; i < pos_dims; ++i) err2 += (plant[i] - goal[i]) * (plant[i] - goal[i]);
    rec.tracking_err = std::sqrt(err2);
    rec.overrun = solve.stats.wall_time > period;
    if (rec.overrun) ++stats.overruns;
    stats.plant_trace.push_back(plant);
    stats.steps.push_back(rec);
    stats.sqp_traces.push_back(std::move(solve.stats));
    const Vector u = traj.U[0];
    const double dt = period / cfg.sim_substeps;
    for (int s = 0; s < cfg.sim_substeps; ++s) plant = model.step(plant, u, dt);
  }
  std::vector<double> times;
  times.reserve(stats.steps.size());
  for (const auto& rec : stats.steps) times.push_back(rec.solve_us);
  if (!times.empty()) {
    double sum = 0.0;
    for (double v : times) sum += v;
    stats.mean_solve_us = sum / static_cast<double>(times.size());
    stats.median_solve_us = nmpc_detail::percentile(times, 0.5);
    stats.p95_solve_us = nmpc_detail::percentile(times, 0.95);
    stats.max_solve_us = *std::max_element(times.begin(), times.end());
  }
  for (size_t g = 0; g < cfg.goals.size(); ++g) {
    const double t_begin = cfg.goals[g].t;
    const double t_end = g + 1 < cfg.goals.size() ? cfg.goals[g + 1].t : cfg.sim_duration;
    std::vector<double> seg;
    for (const auto& rec : stats.steps)
      if (rec.time_s >= t_begin && rec.time_s < t_end) seg.push_back(rec.tracking_err);
    if (seg.empty()) {
      stats.segment_errors.push_back(0.0);
      continue;
    }
    const size_t tail = std::max<size_t>(1, seg.size() / 4);
    double sum = 0.0;
    for (size_t i = seg.size() - tail; i < seg.size(); ++i) sum += seg[i];
    stats.segment_errors.push_back(sum / static_cast<double>(tail));
  }
  return stats;
}

// --------------------------------------------------------------- NMPC outputs
// problem_io.hpp:57-62, problem_io.cpp:250-303 — the run-nmpc CSV / JSON files.
namespace io_detail {
inline void write_text_file(const std::string& path, const std::string& content) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot write file: " + path);
  out << content;
}
/// nlohmann::json's number format: shortest round-trip digits, ".0" on integral values.
inline std::string json_number(double v) {
  char buf[64];
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof(buf), "%.*g", prec, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  std::string s(buf);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}
}  // namespace io_detail

/// steps.csv: step,time_s,solve_us,sqp_iters,pcg_iters_total,tracking_err
inline void write_steps_csv(const NmpcStats& stats, const std::string& path) {
  std::ostringstream out;
  out << "step,time_s,solve_us,sqp_iters,pcg_iters_total,tracking_err\n";
  for (const auto& rec : stats.steps) {
    const double solve_us = stats.deterministic ? 0.0 : rec.solve_us;
    out << rec.step << ',' << format9(rec.time_s) << ',' << format9(solve_us) << ','
        << rec.sqp_iters << ',' << rec.pcg_iters_total << ',' << format9(rec.tracking_err) << '\n';
  }
  io_detail::write_text_file(path, out.str());
}

/// cdf.csv: solve_us,cumulative_fraction (sorted ascending, monotone).
inline void write_cdf_csv(const NmpcStats& stats, const std::string& path) {
  std::vector<double> times;
  times.reserve(stats.steps.size());
  for (const auto& rec : stats.steps) times.push_back(stats.deterministic ? 0.0 : rec.solve_us);
  std::sort(times.begin(), times.end());
  std::ostringstream out;
  out << "solve_us,cumulative_fraction\n";
  for (size_t i = 0; i < times.size(); ++i)
    out << format9(times[i]) << ',' << format9(static_cast<double>(i + 1) / times.size()) << '\n';
  io_detail::write_text_file(path, out.str());
}

/// summary.json (keys sorted and indented by 2 like nlohmann::json::dump(2)).
inline void write_nmpc_summary_json(const NmpcStats& stats, const std::string& path) {
  using io_detail::json_number;
  const bool det = stats.deterministic;
  double mean_track = 0.0;
  for (const auto& rec : stats.steps) mean_track += rec.tracking_err;
  if (!stats.steps.empty()) mean_track /= static_cast<double>(stats.steps.size());
  std::ostringstream out;
  out << "{\n";
  out << "  \"max_solve_us\": " << json_number(det ? 0.0 : stats.max_solve_us) << ",\n";
  out << "  \"mean_solve_us\": " << json_number(det ? 0.0 : stats.mean_solve_us) << ",\n";
  out << "  \"mean_tracking_err\": " << json_number(mean_track) << ",\n";
  out << "  \"median_solve_us\": " << json_number(det ? 0.0 : stats.median_solve_us) << ",\n";
  out << "  \"overruns\": " << (det ? 0 : stats.overruns) << ",\n";
  out << "  \"p95_solve_us\": " << json_number(det ? 0.0 : stats.p95_solve_us) << ",\n";
  out << "  \"segment_errors\": ";
  if (stats.segment_errors.empty()) {
    out << "[]";
  } else {
    out << "[\n";
    for (size_t i = 0; i < stats.segment_errors.size(); ++i)
      out << "    " << json_number(stats.segment_errors[i])
          << (i + 1 < stats.segment_errors.size() ? ",\n" : "\n");
    out << "  ]";
  }
  out << ",\n  \"steps\": " << stats.steps.size() << "\n}\n";
  io_detail::write_text_file(path, out.str());
}

}  // namespace trajopt_b200
