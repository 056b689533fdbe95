// The reference's SQP / NMPC / model / KKT-assembly test cases
// (proj/tests/test_sqp.cpp, test_nmpc.cpp, test_models.cpp, test_kkt.cpp:30-79,144-157)
// written against include/trajopt_b200_sqp.hpp, as a reference caller would.
//
//   test_sqp cpu  — every case, with the linear step supplied by the CPU oracle
//                   (oracle/trajopt_oracle.hpp; test infrastructure) so the host
//                   logic is covered without a GPU.
//   test_sqp gpu  — every case on the B200 linear step (b2p_sqp_step), plus
//                   parity: GPU-backed and oracle-backed SQP / NMPC runs agree
//                   iteration by iteration.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>

#include "trajopt_b200_sqp.hpp"
#include "trajopt_oracle.hpp"

using namespace trajopt_b200;

static int failures = 0;
static int checks = 0;
#define CHECK(cond)                                                                \
  do {                                                                             \
    ++checks;                                                                      \
    if (!(cond)) {                                                                 \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                                  \
    }                                                                              \
  } while (0)
template <class E, class F>
static bool throws_as(F&& f, const char* contains = nullptr) {
  try {
    f();
  } catch (const E& e) {
    return !contains || std::strstr(e.what(), contains) != nullptr;
  } catch (...) {
    return false;
  }
  return false;
}

// ------------------------------------------------------------------ helpers
static Vector vec(std::initializer_list<double> v) { return Vector(v); }
static Vector rng_vec(oracle::UniformRng& rng, int n, double lo, double hi) {
  return rng.vector(n, lo, hi);
}
static Matrix scaled_identity(int n, double s) {
  Matrix M = Matrix::identity(n);
  for (double& v : M.a) v *= s;
  return M;
}
static double inf_diff(const Vector& a, const Vector& b) {
  double d = 0.0;
  for (size_t i = 0; i < a.size(); ++i) d = std::max(d, std::abs(a[i] - b[i]));
  return d;
}

// test_sqp.cpp:16-30
static CostModel default_cost(int n, int m, const Vector& goal, double wx = 1.0, double wu = 0.1,
                              double wn = 10.0) {
  return quadratic_tracking_cost(scaled_identity(n, wx), scaled_identity(m, wu),
                                 scaled_identity(n, wn), goal);
}
static Trajectory random_traj(std::uint64_t seed, int N, int n, int m, double h) {
  oracle::UniformRng rng(seed);
  Trajectory t;
  t.h = h;
  for (int k = 0; k <= N; ++k) t.X.push_back(rng_vec(rng, n, -1.0, 1.0));
  for (int k = 0; k < N; ++k) t.U.push_back(rng_vec(rng, m, -1.0, 1.0));
  return t;
}

// ------------------------------------------------------------------ linear steps
// The CPU oracle's restatement of build_schur -> build_preconditioner ->
// pcg_solve_auto -> reconstruct_primal (test infrastructure only).
static oracle::KKTSystem<double> to_oracle(const KKTSystem& k) {
  oracle::KKTSystem<double> o;
  o.N = k.N;
  o.n = k.n;
  o.m = k.m;
  o.x_s = k.x_s;
  o.x0 = k.x0;
  o.knots.resize(k.knots.size());
  auto mat = [](const Matrix& M) {
    oracle::Mat<double> R(M.rows, M.cols);
    R.a = M.a;
    return R;
  };
  for (size_t i = 0; i < k.knots.size(); ++i) {
    const KnotData& a = k.knots[i];
    oracle::KnotData<double>& b = o.knots[i];
    b.Q = mat(a.Q);
    b.q = a.q;
    if (static_cast<int>(i) < k.N) {
      b.R = mat(a.R);
      b.r = a.r;
      b.A = mat(a.A);
      b.B = mat(a.B);
      b.e = a.e;
    }
  }
  return o;
}
static QpStep oracle_qp_step(const KKTSystem& kkt, const Vector& lambda0, const SqpConfig& cfg) {
  const oracle::KKTSystem<double> o = to_oracle(kkt);
  const auto schur = oracle::build_schur(o);
  const auto P = oracle::build_preconditioner(
      schur, static_cast<oracle::PrecondKind>(static_cast<int>(cfg.precond)), cfg.poly_order);
  oracle::PcgConfig oc;
  oc.epsilon = cfg.pcg.epsilon;
  oc.max_iter = cfg.pcg.max_iter;
  oc.deterministic_reductions = cfg.pcg.deterministic_reductions;
  oc.variant = static_cast<oracle::PcgVariant>(static_cast<int>(cfg.pcg.variant));
  oc.collect_trace = cfg.pcg.collect_trace;
  oc.check_residual_drift = cfg.pcg.check_residual_drift;
  const auto res = oracle::pcg_solve_auto(schur.S, P, schur.gamma, lambda0, oc);
  QpStep out;
  out.lambda = res.lambda;
  out.dz = oracle::reconstruct_primal(o, res.lambda);
  out.report.iterations = res.report.iterations;
  out.report.exit_eta = res.report.exit_eta;
  out.report.converged = res.report.converged;
  out.report.trace = res.report.trace;
  out.report.wall_time = res.report.wall_time;
  return out;
}

// kkt.cpp:129-151 — the dense saddle-point solve, partial-pivot LU (test-side
// implementation of the reference's dense_kkt backend).
static QpStep dense_qp_step(const KKTSystem& k, const Vector&, const SqpConfig&) {
  const int N = k.N, n = k.n, m = k.m;
  const int np = (N + 1) * n + N * m, nd = (N + 1) * n, D = np + nd;
  std::vector<double> A(static_cast<size_t>(D) * D, 0.0), b(D, 0.0);
  auto at = [&](int i, int j) -> double& { return A[static_cast<size_t>(i) * D + j]; };
  int off = 0;
  for (int kk = 0; kk <= N; ++kk) {
    for (int i = 0; i < n; ++i) {
      for (int j = 0; j < n; ++j) at(off + i, off + j) = k.knots[kk].Q(i, j);
      b[off + i] = -k.knots[kk].q[i];
    }
    off += n;
    if (kk < N) {
      for (int i = 0; i < m; ++i) {
        for (int j = 0; j < m; ++j) at(off + i, off + j) = k.knots[kk].R(i, j);
        b[off + i] = -k.knots[kk].r[i];
      }
      off += m;
    }
  }
  auto setC = [&](int r, int c, double v) {
    at(np + r, c) = v;
    at(c, np + r) = v;
  };
  for (int i = 0; i < n; ++i) setC(i, i, 1.0);
  const int stride = n + m;
  for (int kk = 0; kk < N; ++kk) {
    const int row = (kk + 1) * n, col = kk * stride;
    for (int i = 0; i < n; ++i) {
      for (int j = 0; j < n; ++j) setC(row + i, col + j, -k.knots[kk].A(i, j));
      for (int j = 0; j < m; ++j) setC(row + i, col + n + j, -k.knots[kk].B(i, j));
      setC(row + i, col + stride + i, 1.0);
    }
  }
  for (int i = 0; i < n; ++i) b[np + i] = k.x_s[i] - k.x0[i];
  for (int kk = 0; kk < N; ++kk)
    for (int i = 0; i < n; ++i) b[np + (kk + 1) * n + i] = -k.knots[kk].e[i];
  for (int c = 0; c < D; ++c) {
    int p = c;
    for (int r = c + 1; r < D; ++r)
      if (std::abs(at(r, c)) > std::abs(at(p, c))) p = r;
    if (at(p, c) == 0.0) throw std::runtime_error("dense_kkt_solve: singular KKT matrix");
    if (p != c) {
      for (int j = 0; j < D; ++j) std::swap(at(c, j), at(p, j));
      std::swap(b[c], b[p]);
    }
    for (int r = c + 1; r < D; ++r) {
      const double f = at(r, c) / at(c, c);
      if (f == 0.0) continue;
      for (int j = c; j < D; ++j) at(r, j) -= f * at(c, j);
      b[r] -= f * b[c];
    }
  }
  std::vector<double> x(D);
  for (int r = D - 1; r >= 0; --r) {
    double s = b[r];
    for (int j = r + 1; j < D; ++j) s -= at(r, j) * x[j];
    x[r] = s / at(r, r);
  }
  QpStep out;
  out.dz.assign(x.begin(), x.begin() + np);
  out.lambda.assign(x.begin() + np, x.end());
  return out;
}

// The linear step every SQP case below uses (empty = the GPU default).
static QpSolver g_qp;
static SqpConfig with_backend(SqpConfig c) {
  c.qp_solver = g_qp;
  return c;
}

// ------------------------------------------------------------------ test_models.cpp
static void fd_jacobians(const DynamicsModel& model, const Vector& x, const Vector& u, double h,
                         Matrix& A, Matrix& B, double step = 1e-6) {
  const int n = model.state_dim(), m = model.control_dim();
  A = Matrix(n, n);
  B = Matrix(n, m);
  for (int j = 0; j < n; ++j) {
    Vector xp = x, xm = x;
    xp[j] += step;
    xm[j] -= step;
    const Vector fp = model.step(xp, u, h), fm = model.step(xm, u, h);
    for (int i = 0; i < n; ++i) A(i, j) = (fp[i] - fm[i]) / (2.0 * step);
  }
  for (int j = 0; j < m; ++j) {
    Vector up = u, um = u;
    up[j] += step;
    um[j] -= step;
    const Vector fp = model.step(x, up, h), fm = model.step(x, um, h);
    for (int i = 0; i < n; ++i) B(i, j) = (fp[i] - fm[i]) / (2.0 * step);
  }
}
static double jacobian_fd_error(const DynamicsModel& model, const Vector& x, const Vector& u,
                                double h) {  // test_models.cpp:35-42
  Matrix A, B, Af, Bf;
  model.jacobians(x, u, h, A, B);
  fd_jacobians(model, x, u, h, Af, Bf);
  double scale = 1.0, err = 0.0;
  for (double v : Af.a) scale = std::max(scale, std::abs(v));
  for (double v : Bf.a) scale = std::max(scale, std::abs(v));
  for (size_t i = 0; i < A.a.size(); ++i) err = std::max(err, std::abs(A.a[i] - Af.a[i]));
  for (size_t i = 0; i < B.a.size(); ++i) err = std::max(err, std::abs(B.a[i] - Bf.a[i]));
  return err / scale;
}

static void test_models() {
  {  // test_models.cpp:46-71
    auto model = double_integrator();
    CHECK(model->step(vec({0, 0}), vec({0}), 0.01) == vec({0, 0}));
    const Vector next = model->step(vec({1, 2}), vec({3}), 0.01);
    CHECK(std::abs(next[0] - 1.02) < 1e-12 && std::abs(next[1] - 2.03) < 1e-12);
    Matrix A, B;
    model->jacobians(vec({0.3, -1.1}), vec({0.7}), 0.01, A, B);
    CHECK(A(0, 1) == 0.01 && B(1, 0) == 0.01);
    CHECK(jacobian_fd_error(*model, vec({0.3, -1.1}), vec({0.7}), 0.01) <= 1e-9);
  }
  {  // :73-90
    auto model = pendulum();
    CHECK(model->step(vec({0, 0}), vec({0}), 0.05) == vec({0, 0}));
    oracle::UniformRng rng(11);
    for (int t = 0; t < 20; ++t) {
      const Vector x = rng_vec(rng, 2, -3.0, 3.0);
      const Vector u = rng_vec(rng, 1, -2.0, 2.0);
      CHECK(jacobian_fd_error(*model, x, u, 0.05) <= 1e-5);
    }
  }
  {  // :92-110
    auto model = cartpole();
    Vector x = vec({0, 0.01, 0, 0});
    for (int i = 0; i < 50; ++i) x = model->step(x, vec({0}), 0.01);
    CHECK(std::abs(x[1]) > 0.02);
    oracle::UniformRng rng(12);
    for (int t = 0; t < 20; ++t) {
      const Vector xs = rng_vec(rng, 4, -2.0, 2.0);
      const Vector u = rng_vec(rng, 1, -5.0, 5.0);
      CHECK(jacobian_fd_error(*model, xs, u, 0.01) <= 1e-5);
    }
  }
  {  // :112-122
    oracle::UniformRng rng(77);
    for (const char* name : {"double_integrator", "pendulum", "cartpole"}) {
      auto model = make_model(name);
      CHECK(model->name() == name);
      for (int t = 0; t < 100; ++t) {
        const Vector x = rng_vec(rng, model->state_dim(), -2.0, 2.0);
        const Vector u = rng_vec(rng, model->control_dim(), -2.0, 2.0);
        CHECK(jacobian_fd_error(*model, x, u, 0.02) <= 1e-5);
      }
    }
  }
  CHECK(throws_as<std::invalid_argument>([] { make_model("segway"); }, "unknown model"));
  {  // :128-183 eval_cost
    const Matrix I2 = Matrix::identity(2), I1 = Matrix::identity(1);
    const Vector goal = vec({1, -2});
    const CostModel c0 = quadratic_tracking_cost(I2, I1, I2, goal);
    CHECK(eval_cost(c0, std::vector<Vector>(4, goal), std::vector<Vector>(3, vec({0}))) == 0.0);
    const CostModel c1 = quadratic_tracking_cost(I2, I1, I2, vec({0, 0}));
    CHECK(std::abs(eval_cost(c1, {vec({1, 1})}, {}) - 1.0) < 1e-15);
    oracle::UniformRng rng(5);
    const Vector g = rng_vec(rng, 2, -1.0, 1.0);
    const CostModel c2 = quadratic_tracking_cost(scaled_identity(2, 2.0), scaled_identity(1, 0.5),
                                                 scaled_identity(2, 3.0), g);
    const int N = 5;
    std::vector<Vector> X, U;
    for (int k = 0; k <= N; ++k) X.push_back(rng_vec(rng, 2, -2.0, 2.0));
    for (int k = 0; k < N; ++k) U.push_back(rng_vec(rng, 1, -2.0, 2.0));
    double want = 0.0;
    for (int k = 0; k < N; ++k) {
      const double d0 = X[k][0] - g[0], d1 = X[k][1] - g[1];
      want += 0.5 * 2.0 * (d0 * d0 + d1 * d1) + 0.5 * 0.5 * U[k][0] * U[k][0];
    }
    const double e0 = X[N][0] - g[0], e1 = X[N][1] - g[1];
    want += 0.5 * 3.0 * (e0 * e0 + e1 * e1);
    CHECK(std::abs(eval_cost(c2, X, U) - want) <= 1e-14 * std::abs(want));
    CHECK(throws_as<std::invalid_argument>([&] { eval_cost(c2, X, X); }, "N+1 states"));
  }
  {  // rollout is feasible by construction
    auto model = pendulum();
    const Trajectory t = rollout(*model, vec({0.1, 0}), std::vector<Vector>(6, vec({0.5})), 0.05);
    CHECK(t.X.size() == 7 && constraint_l1(t, *model, t.X[0]) == 0.0);
  }
}

// ------------------------------------------------------------------ test_kkt.cpp assemble cases
static void test_assemble_kkt() {
  auto di = double_integrator();
  const Matrix I2 = Matrix::identity(2), I1 = Matrix::identity(1);
  {  // test_kkt.cpp:30-44
    const CostModel cost = quadratic_tracking_cost(I2, I1, I2, vec({0, 0}));
    Trajectory t;
    t.h = 0.01;
    t.X.assign(5, vec({0, 0}));
    t.U.assign(4, vec({0}));
    const KKTSystem k = assemble_kkt(t, *di, cost, vec({0, 0}));
    for (int i = 0; i < k.N; ++i) CHECK(la::norm_inf(k.knots[i].e) == 0.0);
    CHECK(la::norm_inf(la::sub(k.x_s, k.x0)) == 0.0);
  }
  {  // :46-61
    auto model = pendulum();
    const CostModel cost = quadratic_tracking_cost(I2, I1, I2, vec({0, 0}));
    oracle::UniformRng rng(3);
    Trajectory t;
    t.h = 0.05;
    for (int k = 0; k <= 3; ++k) t.X.push_back(rng_vec(rng, 2, -1.0, 1.0));
    for (int k = 0; k < 3; ++k) t.U.push_back(rng_vec(rng, 1, -1.0, 1.0));
    const KKTSystem k = assemble_kkt(t, *model, cost, t.X[0]);
    for (int i = 0; i < 3; ++i)
      CHECK(inf_diff(k.knots[i].e, la::sub(t.X[i + 1], model->step(t.X[i], t.U[i], t.h))) == 0.0);
  }
  {  // :63-78
    const Vector goal = vec({0.5, -0.25});
    const CostModel cost = quadratic_tracking_cost(I2, I1, I2, goal);
    oracle::UniformRng rng(4);
    Trajectory t;
    t.h = 0.01;
    for (int k = 0; k <= 2; ++k) t.X.push_back(rng_vec(rng, 2, -1.0, 1.0));
    for (int k = 0; k < 2; ++k) t.U.push_back(rng_vec(rng, 1, -1.0, 1.0));
    const KKTSystem k = assemble_kkt(t, *di, cost, t.X[0]);
    for (int i = 0; i <= 2; ++i) CHECK(inf_diff(k.knots[i].q, la::sub(t.X[i], goal)) <= 1e-15);
  }
  {  // :144-157
    const CostModel cost = quadratic_tracking_cost(I2, I1, I2, vec({0, 0}));
    Trajectory t;
    t.h = 0.01;
    t.X.assign(3, vec({0, 0}));
    t.U.assign(2, vec({0}));
    t.X[1][0] = std::numeric_limits<double>::quiet_NaN();
    CHECK(throws_as<std::runtime_error>([&] { assemble_kkt(t, *di, cost, vec({0, 0})); }, "knot"));
    t.X.pop_back();
    CHECK(throws_as<std::invalid_argument>([&] { assemble_kkt(t, *di, cost, vec({0, 0})); },
                                           "needs N+1 states"));
  }
  {  // kkt.cpp:20-25 — a singular weight gets the 1e-6 ridge, a PD one does not
    Matrix Wx(2, 2);
    Wx(0, 0) = 1.0;  // eigenvalues {1, 0}
    const CostModel cost = quadratic_tracking_cost(Wx, I1, I2, vec({0, 0}));
    Trajectory t;
    t.X.assign(2, vec({1, 1}));
    t.U.assign(1, vec({0}));
    const KKTSystem k = assemble_kkt(t, *di, cost, vec({0, 0}));
    CHECK(k.knots[0].Q(1, 1) == 1e-6 && k.knots[0].Q(0, 0) == 1.0 + 1e-6);
    CHECK(k.knots[0].q[1] == 0.0);  // q is formed before the ridge
    CHECK(k.knots[1].Q(0, 0) == 1.0 && k.knots[0].R(0, 0) == 1.0);
  }
}

// ------------------------------------------------------------------ test_sqp.cpp
static void test_merit_and_line_search() {
  auto model = double_integrator();
  const CostModel cost = default_cost(2, 1, vec({1, 0}));
  {  // test_sqp.cpp:42-58
    oracle::UniformRng rng(1);
    std::vector<Vector> controls(6);
    for (auto& u : controls) u = rng_vec(rng, 1, -1.0, 1.0);
    const Trajectory t = rollout(*model, vec({0, 0}), controls, 0.01);
    const double M = merit(t, *model, cost, t.X[0], 10.0);
    CHECK(std::abs(M - eval_cost(cost, t)) <= 1e-15 * std::abs(M));
    for (std::uint64_t seed = 0; seed < 20; ++seed) {
      const Trajectory tr = random_traj(seed, 5, 2, 1, 0.01);
      CHECK(merit(tr, *model, cost, vec({0, 0}), 10.0) >= eval_cost(cost, tr));
    }
  }
  {  // :61-79
    CHECK(select_line_search_candidate(7.2, {7.0, 6.5, 6.8}) == 1);
    CHECK(select_line_search_candidate(7.2, {6.5, 6.5, 6.8}) == 0);
    CHECK(select_line_search_candidate(7.2, {7.2, 7.3, 8.0}) == -1);
    const double inf = std::numeric_limits<double>::infinity();
    CHECK(select_line_search_candidate(7.0, {inf, 6.0, inf}) == 1);
  }
  {  // :81-108
    const Trajectory t = random_traj(3, 4, 2, 1, 0.01);
    const Vector x_s = vec({0, 0});
    MeritParams p;
    const Vector dz((4 + 1) * 2 + 4, 0.0);
    const LineSearchResult r = parallel_line_search(t, dz, *model, cost, p, x_s);
    CHECK(r.alpha == 0.0 && !r.progress);
    CHECK(std::abs(r.merit - merit(t, *model, cost, x_s, p.mu)) <= 1e-12);
    for (int k = 0; k <= 4; ++k) CHECK(inf_diff(r.traj.X[k], t.X[k]) == 0.0);
    p.alphas = {0.5, 1.0};
    CHECK(throws_as<std::invalid_argument>(
        [&] { parallel_line_search(t, dz, *model, cost, p, x_s); }, "alpha set must start at 1"));
    p.alphas = {1.0, 0.5, 0.5};
    CHECK(throws_as<std::invalid_argument>(
        [&] { parallel_line_search(t, dz, *model, cost, p, x_s); }, "strictly descending"));
    p = MeritParams{};
    p.mu = 0.0;
    CHECK(throws_as<std::invalid_argument>(
        [&] { parallel_line_search(t, dz, *model, cost, p, x_s); }, "mu must be positive"));
    CHECK(throws_as<std::invalid_argument>([&] { apply_step(t, Vector(3, 0.0), 1.0); },
                                           "expected dz of length 14"));
  }
}

static void test_sqp_solve() {
  auto model = double_integrator();
  const Vector x_s = vec({-0.4, 0.2});
  {  // test_sqp.cpp:111-140 — LQR converges in one full step
    const CostModel cost = default_cost(2, 1, vec({0.7, 0.0}));
    const Trajectory t0 = random_traj(7, 12, 2, 1, 0.05);
    SqpConfig cfg;
    cfg.max_sqp_iter = 1;
    cfg.pcg.epsilon = 1e-12;
    cfg.pcg.max_iter = 2000;
    const SqpResult res = sqp_solve(t0, {}, x_s, *model, cost, with_backend(cfg));
    CHECK(res.stats.iters.size() == 1);
    CHECK(res.stats.iters[0].alpha == 1.0);
    CHECK(constraint_l1(res.traj, *model, x_s) <= 1e-8);
    SqpConfig dense = cfg;
    dense.backend = SolverBackend::dense_kkt;
    CHECK(throws_as<std::invalid_argument>(
        [&] { sqp_solve(t0, {}, x_s, *model, cost, dense); }, "dense_kkt"));
    dense.qp_solver = dense_qp_step;
    const SqpResult rd = sqp_solve(t0, {}, x_s, *model, cost, dense);
    for (int k = 0; k <= 12; ++k) CHECK(inf_diff(res.traj.X[k], rd.traj.X[k]) <= 1e-6);
    for (int k = 0; k < 12; ++k) CHECK(inf_diff(res.traj.U[k], rd.traj.U[k]) <= 1e-6);
    CHECK(rd.stats.iters[0].pcg.iterations == 0);  // dense backend leaves the PCG report empty
  }
  {  // :142-166 — an already-optimal warm start stalls
    const CostModel cost = default_cost(2, 1, vec({0.7, 0.0}));
    SqpConfig cfg;
    cfg.max_sqp_iter = 6;
    cfg.pcg.epsilon = 1e-12;
    cfg.pcg.max_iter = 2000;
    const SqpResult first =
        sqp_solve(random_traj(9, 10, 2, 1, 0.05), {}, x_s, *model, cost, with_backend(cfg));
    const SqpResult second =
        sqp_solve(first.traj, first.lambda, x_s, *model, cost, with_backend(cfg));
    CHECK(second.stats.stalled);
    CHECK(second.stats.iters.size() <= 2);
    for (const auto& it : second.stats.iters) CHECK(it.alpha == 0.0);
    for (int k = 0; k <= 10; ++k) CHECK(inf_diff(second.traj.X[k], first.traj.X[k]) == 0.0);
  }
  {  // :168-193 — pendulum swing-up: accepted steps never increase the merit
    auto pend = pendulum();
    const CostModel cost = default_cost(2, 1, vec({M_PI, 0.0}), 1.0, 0.05, 20.0);
    Trajectory t0;
    t0.h = 0.05;
    t0.X.assign(33, vec({0, 0}));
    t0.U.assign(32, vec({0}));
    SqpConfig cfg;
    cfg.max_sqp_iter = 20;
    cfg.pcg.epsilon = 1e-10;
    cfg.pcg.max_iter = 2000;
    const SqpResult res = sqp_solve(t0, {}, vec({0, 0}), *pend, cost, with_backend(cfg));
    CHECK(!res.stats.iters.empty());
    double last = std::numeric_limits<double>::infinity();
    for (const auto& it : res.stats.iters)
      if (it.alpha > 0.0) {
        CHECK(it.merit_after <= it.merit_before);
        CHECK(it.merit_after <= last);
        last = it.merit_after;
      }
  }
  {  // :195-229 — lambda warm-start plumbing
    const CostModel cost = default_cost(2, 1, vec({1.0, 0.0}));
    const Trajectory t0 = random_traj(11, 6, 2, 1, 0.05);
    SqpConfig cfg;
    cfg.max_sqp_iter = 3;
    cfg.pcg.epsilon = 1e-30;
    cfg.pcg.max_iter = 1;
    oracle::UniformRng rng(12);
    const Vector lambda0 = rng_vec(rng, 7 * 2, -1.0, 1.0);
    const SqpResult res = sqp_solve(t0, lambda0, vec({0, 0}), *model, cost, with_backend(cfg));
    CHECK(res.lambda.size() == lambda0.size());
    SqpConfig one = cfg;
    one.max_sqp_iter = 1;
    one.pcg.epsilon = 1e-10;
    one.pcg.max_iter = 500;
    one.pcg.collect_trace = true;
    SqpConfig two = one;
    two.max_sqp_iter = 2;
    const SqpResult r1 = sqp_solve(t0, lambda0, vec({0, 0}), *model, cost, with_backend(one));
    const SqpResult r2 = sqp_solve(t0, lambda0, vec({0, 0}), *model, cost, with_backend(two));
    CHECK(r2.stats.iters.size() >= 1);
    CHECK(r1.stats.iters[0].pcg.iterations == r2.stats.iters[0].pcg.iterations);
    CHECK(throws_as<std::invalid_argument>(
        [&] { sqp_solve(t0, Vector(3, 0.0), vec({0, 0}), *model, cost, with_backend(cfg)); },
        "expected lambda0 of length 14, got 3"));
    SqpConfig bad = cfg;
    bad.max_sqp_iter = 0;
    CHECK(throws_as<std::invalid_argument>(
        [&] { sqp_solve(t0, {}, vec({0, 0}), *model, cost, bad); }, "max_sqp_iter"));
  }
  {  // :231-243 — one CSV row per iteration
    const CostModel cost = default_cost(2, 1, vec({1.0, 0.0}));
    const SqpResult res = sqp_solve(random_traj(13, 5, 2, 1, 0.05), {}, vec({0, 0}), *model,
                                    cost, with_backend(SqpConfig{}));
    const std::string csv = sqp_stats_csv(res.stats);
    CHECK(static_cast<size_t>(std::count(csv.begin(), csv.end(), '\n')) ==
          res.stats.iters.size() + 1);
    CHECK(csv.rfind("iter,mu,merit_before,merit_after,alpha,constraint_l1,", 0) == 0);
  }
}

// ------------------------------------------------------------------ test_nmpc.cpp
static NmpcConfig base_config() {  // test_nmpc.cpp:16-29
  NmpcConfig cfg;
  cfg.control_rate = 100.0;
  cfg.sim_duration = 1.0;
  cfg.N = 16;
  cfg.h = 0.01;
  cfg.sim_substeps = 4;
  cfg.deterministic = true;
  cfg.solver.max_sqp_iter = 3;
  cfg.solver.pcg.epsilon = 1e-4;
  cfg.solver.pcg.max_iter = 200;
  cfg.solver.pcg.deterministic_reductions = true;
  cfg.solver.merit.mu_rule = MeritParams::MuRule::multiplier_max;
  cfg.solver.qp_solver = g_qp;
  return cfg;
}
static CostModel tracking_cost(int n, int m) {  // :34-39
  Matrix Wx = scaled_identity(n, 100.0);
  for (int i = 0; i < n / 2; ++i) Wx(i, i) = 1000.0;
  return quadratic_tracking_cost(Wx, Matrix::identity(m), scaled_identity(n, 1e5),
                                 Vector(static_cast<size_t>(n), 0.0));
}
static double median_of(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  const size_t n = v.size();
  return n % 2 == 1 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}

static void test_nmpc() {
  {  // test_nmpc.cpp:49-80
    Trajectory t;
    t.X.assign(4, vec({1, 2}));
    t.U.assign(3, vec({1}));
    t.lambda.assign(8, 1.0);
    const Trajectory s = shift_warm_start(t);
    for (int k = 0; k <= 3; ++k) CHECK(s.X[k] == vec({1, 2}));
    CHECK(s.lambda == t.lambda);
    Trajectory u;
    for (int k = 0; k < 3; ++k) u.X.push_back(vec({static_cast<double>(k)}));
    u.U = {vec({10}), vec({11})};
    u.lambda = {100, 101, 102};
    const Trajectory v = shift_warm_start(u);
    CHECK(v.X[0][0] == 1.0 && v.X[1][0] == 2.0 && v.X[2][0] == 2.0);
    CHECK(v.U[0][0] == 11.0 && v.U[1][0] == 11.0);
    CHECK(v.lambda[0] == 101.0 && v.lambda[1] == 102.0 && v.lambda[2] == 102.0);
  }
  auto model = double_integrator();
  {  // :82-94
    NmpcConfig cfg = base_config();
    cfg.x0 = vec({0.5, 0.0});
    cfg.goals = {{0.0, vec({0.5, 0.0})}};
    const NmpcStats st = run_nmpc(cfg, *model, tracking_cost(2, 1));
    CHECK(st.steps.size() == 100);
    for (const auto& r : st.steps) CHECK(r.tracking_err <= 1e-9);
  }
  {  // :96-108
    NmpcConfig cfg = base_config();
    cfg.sim_duration = 4.0;
    cfg.N = 32;
    cfg.goals = {{0.0, vec({0.5, 0.0})}, {2.0, vec({-0.3, 0.0})}};
    const NmpcStats st = run_nmpc(cfg, *model, tracking_cost(2, 1));
    CHECK(st.segment_errors.size() == 2);
    CHECK(st.segment_errors[0] <= 1e-2 && st.segment_errors[1] <= 1e-2);
    CHECK(st.median_solve_us > 0.0 && st.p95_solve_us >= st.median_solve_us);
  }
  {  // :110-131 — warm-started multipliers cut the median PCG iterations
    NmpcConfig cfg = base_config();
    cfg.sim_duration = 2.0;
    cfg.N = 32;
    cfg.goals = {{0.0, vec({0.5, 0.0})}, {0.7, vec({-0.3, 0.0})}, {1.4, vec({0.2, 0.0})}};
    NmpcConfig cold = cfg;
    cold.warm_start_lambda = false;
    const NmpcStats w = run_nmpc(cfg, *model, tracking_cost(2, 1));
    const NmpcStats c = run_nmpc(cold, *model, tracking_cost(2, 1));
    std::vector<double> wi, ci;
    for (const auto& r : w.steps) wi.push_back(static_cast<double>(r.pcg_iters_total));
    for (const auto& r : c.steps) ci.push_back(static_cast<double>(r.pcg_iters_total));
    std::printf("nmpc median pcg iterations: warm %.1f cold %.1f\n", median_of(wi), median_of(ci));
    CHECK(median_of(wi) < median_of(ci));
  }
  {  // :133-146 — deterministic runs are bitwise identical
    NmpcConfig cfg = base_config();
    cfg.goals = {{0.0, vec({0.4, 0.0})}};
    cfg.solver.pcg.variant = PcgVariant::block_parallel;
    const NmpcStats a = run_nmpc(cfg, *model, tracking_cost(2, 1));
    const NmpcStats b = run_nmpc(cfg, *model, tracking_cost(2, 1));
    CHECK(a.plant_trace.size() == b.plant_trace.size());
    for (size_t i = 0; i < a.plant_trace.size(); ++i)
      CHECK(inf_diff(a.plant_trace[i], b.plant_trace[i]) == 0.0);
  }
  {  // :148-158
    NmpcConfig cfg = base_config();
    cfg.control_rate = 50.0;
    cfg.sim_duration = 0.8;
    cfg.goals = {{0.0, vec({0.1, 0.0})}};
    CHECK(run_nmpc(cfg, *model, tracking_cost(2, 1)).steps.size() == 40);
  }
  {  // :160-172
    NmpcConfig cfg = base_config();
    cfg.goals.clear();
    CHECK(throws_as<std::invalid_argument>([&] { run_nmpc(cfg, *model, tracking_cost(2, 1)); },
                                           "goal sequence is empty"));
    cfg = base_config();
    cfg.N = 1;
    cfg.goals = {{0.0, vec({0, 0})}};
    CHECK(throws_as<std::invalid_argument>([&] { run_nmpc(cfg, *model, tracking_cost(2, 1)); },
                                           "N must be >= 2"));
  }
}

// ------------------------------------------------------------------ test_io.cpp:98-140
static std::vector<std::string> read_lines(const std::string& path) {
  std::ifstream in(path);
  std::vector<std::string> out;
  std::string line;
  while (std::getline(in, line)) out.push_back(line);
  return out;
}
static void test_nmpc_writers() {
  NmpcStats stats;
  stats.deterministic = false;
  for (int i = 0; i < 5; ++i) {
    NmpcStepRecord rec;
    rec.step = i;
    rec.time_s = 0.01 * i;
    rec.solve_us = 100.0 - 10.0 * i;  // unsorted on purpose
    rec.sqp_iters = 2;
    rec.pcg_iters_total = 6;
    rec.tracking_err = 0.1;
    stats.steps.push_back(rec);
  }
  stats.segment_errors = {0.25, 1e-3};
  const std::string steps_path = "/tmp/b2p_test_steps.csv", cdf_path = "/tmp/b2p_test_cdf.csv",
                    json_path = "/tmp/b2p_test_summary.json";
  write_steps_csv(stats, steps_path);
  write_cdf_csv(stats, cdf_path);
  write_nmpc_summary_json(stats, json_path);
  const auto sl = read_lines(steps_path);
  CHECK(sl.size() == 6 && sl[0] == "step,time_s,solve_us,sqp_iters,pcg_iters_total,tracking_err");
  CHECK(sl[2] == "1,0.01,90,2,6,0.1");
  const auto cl = read_lines(cdf_path);
  CHECK(cl.size() == 6 && cl[0] == "solve_us,cumulative_fraction");
  double prev_t = -1.0, prev_f = 0.0;
  for (size_t i = 1; i < cl.size(); ++i) {
    const auto comma = cl[i].find(',');
    const double t = std::stod(cl[i].substr(0, comma)), f = std::stod(cl[i].substr(comma + 1));
    CHECK(t >= prev_t && f > prev_f);
    prev_t = t;
    prev_f = f;
  }
  CHECK(std::abs(prev_f - 1.0) < 1e-12);
  const auto jl = read_lines(json_path);
  CHECK(jl.size() == 13 && jl[0] == "{" && jl[1] == "  \"max_solve_us\": 0.0," && jl[3] == "  \"mean_tracking_err\": 0.1," &&
        jl[8] == "    0.25," && jl[9] == "    0.001" && jl[11] == "  \"steps\": 5");
  stats.deterministic = true;
  write_steps_csv(stats, steps_path);
  CHECK(read_lines(steps_path)[1] == "0,0,0,2,6,0.1");
  std::remove(steps_path.c_str());
  std::remove(cdf_path.c_str());
  std::remove(json_path.c_str());
}

// ------------------------------------------------------------------ GPU vs oracle parity
// Same scenario on both linear steps: every SQP iteration must take the same
// PCG iteration count and the same line-search step, with merits and final
// trajectories within floating-point tolerance.
// Identity-preconditioned CG is the one documented exception:
// its iteration count can differ by one between any two summation orders (the
// reference's own sequential and block-parallel variants included), so there
// the count may differ by one and the merits agree to the PCG tolerance.
static void compare_sqp(const char* what, const SqpResult& g, const SqpResult& o,
                        int iter_slack = 0, double merit_tol = 1e-9, double state_tol = 1e-8) {
  bool ok = g.stats.iters.size() == o.stats.iters.size();
  int max_it_diff = 0;
  double merr = 0.0, terr = 0.0;
  for (size_t i = 0; ok && i < g.stats.iters.size(); ++i) {
    const auto &a = g.stats.iters[i], &b = o.stats.iters[i];
    max_it_diff = std::max(max_it_diff, std::abs(a.pcg.iterations - b.pcg.iterations));
    // With a one-iteration slack the step lengths may legitimately differ too.
    if (iter_slack == 0) ok = ok && a.alpha == b.alpha && a.pcg.converged == b.pcg.converged;
    merr = std::max(merr, std::abs(a.merit_after - b.merit_after) /
                              std::max(1.0, std::abs(b.merit_after)));
  }
  for (size_t k = 0; k < std::min(g.traj.X.size(), o.traj.X.size()); ++k)
    terr = std::max(terr, inf_diff(g.traj.X[k], o.traj.X[k]));
  std::printf("parity %-28s sqp iters %zu/%zu  max pcg-iteration diff %d  max merit rel diff %.2e  "
              "max state diff %.2e\n",
              what, g.stats.iters.size(), o.stats.iters.size(), max_it_diff, merr, terr);
  CHECK(ok);
  CHECK(max_it_diff <= iter_slack);
  CHECK(merr <= merit_tol);
  CHECK(terr <= state_tol);
}

static void test_parity() {
  {  // pendulum swing-up (test_sqp.cpp:168-193 scenario), every preconditioner
    auto pend = pendulum();
    const CostModel cost = default_cost(2, 1, vec({M_PI, 0.0}), 1.0, 0.05, 20.0);
    Trajectory t0;
    t0.h = 0.05;
    t0.X.assign(33, vec({0, 0}));
    t0.U.assign(32, vec({0}));
    for (PrecondKind kind : {PrecondKind::symmetric_stair, PrecondKind::stair,
                             PrecondKind::block_jacobi, PrecondKind::identity}) {
      SqpConfig cfg;
      cfg.max_sqp_iter = 20;
      cfg.pcg.epsilon = 1e-10;
      cfg.pcg.max_iter = 2000;
      cfg.precond = kind;
      // identity: one SQP iteration (later iterates linearise around
      // trajectories that legitimately differ after a ±1 PCG iteration)
      if (kind == PrecondKind::identity) cfg.max_sqp_iter = 1;
      const SqpResult g = sqp_solve(t0, {}, vec({0, 0}), *pend, cost, cfg);
      cfg.qp_solver = oracle_qp_step;
      const SqpResult o = sqp_solve(t0, {}, vec({0, 0}), *pend, cost, cfg);
      if (kind == PrecondKind::identity)
        compare_sqp("pendulum identity", g, o, 1, 1e-5, 1e-3);
      else
        compare_sqp(("pendulum " + precond_name(kind)).c_str(), g, o);
    }
  }
  {  // cart-pole balance from a tilted start, long horizon
    auto cp = cartpole();
    Matrix Wx = scaled_identity(4, 1.0);
    Wx(1, 1) = 10.0;
    const CostModel cost =
        quadratic_tracking_cost(Wx, scaled_identity(1, 0.1), scaled_identity(4, 50.0), vec({0, 0, 0, 0}));
    Trajectory t0;
    t0.h = 0.02;
    t0.X.assign(129, vec({0, 0.3, 0, 0}));
    t0.U.assign(128, vec({0}));
    SqpConfig cfg;
    cfg.max_sqp_iter = 8;
    cfg.pcg.epsilon = 1e-10;
    cfg.pcg.max_iter = 4000;
    const SqpResult g = sqp_solve(t0, {}, vec({0, 0.3, 0, 0}), *cp, cost, cfg);
    cfg.qp_solver = oracle_qp_step;
    const SqpResult o = sqp_solve(t0, {}, vec({0, 0.3, 0, 0}), *cp, cost, cfg);
    compare_sqp("cartpole N=128", g, o);
  }
  {  // NMPC with warm starts: identical PCG iteration totals step by step
    auto model = double_integrator();
    NmpcConfig cfg = base_config();
    cfg.sim_duration = 1.0;
    cfg.N = 32;
    cfg.goals = {{0.0, vec({0.5, 0.0})}, {0.5, vec({-0.3, 0.0})}};
    cfg.solver.qp_solver = nullptr;
    const NmpcStats g = run_nmpc(cfg, *model, tracking_cost(2, 1));
    cfg.solver.qp_solver = oracle_qp_step;
    const NmpcStats o = run_nmpc(cfg, *model, tracking_cost(2, 1));
    bool same = g.steps.size() == o.steps.size();
    double perr = 0.0;
    for (size_t i = 0; same && i < g.steps.size(); ++i) {
      same = g.steps[i].pcg_iters_total == o.steps[i].pcg_iters_total &&
             g.steps[i].sqp_iters == o.steps[i].sqp_iters;
      perr = std::max(perr, inf_diff(g.plant_trace[i], o.plant_trace[i]));
    }
    std::printf("parity nmpc double_integrator      steps %zu  same iteration counts %d  max plant diff %.2e  "
                "median solve %.1f us (gpu) / %.1f us (oracle)\n",
                g.steps.size(), same ? 1 : 0, perr, g.median_solve_us, o.median_solve_us);
    CHECK(same);
    CHECK(perr <= 1e-9);
  }
}

// Host-visible latency of one SQP linear step through the library (pack,
// upload, fused solve + primal kernel, download) at the NMPC test size and at
// the c1 size, next to the oracle's.
static void time_linear_step() {
  using Clock = std::chrono::steady_clock;
  struct Case {
    const char* name;
    int N, n, m;
  };
  for (const Case c : {Case{"N=32 n=2 m=1", 32, 2, 1}, Case{"c1 N=31 n=14 m=7", 31, 14, 7}}) {
    const KKTSystem kkt = random_kkt(4242, c.N, c.n, c.m);
    SqpConfig cfg;
    cfg.pcg.epsilon = 1e-8;
    const Vector l0(static_cast<size_t>(kkt.dual_dim()), 0.0);
    double best[2] = {1e30, 1e30};
    for (int which = 0; which < 2; ++which) {
      const QpSolver f = which == 0 ? QpSolver(gpu_qp_step) : QpSolver(oracle_qp_step);
      for (int rep = 0; rep < 3; ++rep) f(kkt, l0, cfg);
      std::vector<double> t;
      for (int rep = 0; rep < 50; ++rep) {
        const auto t0 = Clock::now();
        f(kkt, l0, cfg);
        t.push_back(std::chrono::duration<double, std::micro>(Clock::now() - t0).count());
      }
      std::sort(t.begin(), t.end());
      best[which] = t[t.size() / 2];
    }
    std::printf("linear step %-18s median %.1f us (b2p_sqp_step) / %.1f us (oracle, 1 thread)\n",
                c.name, best[0], best[1]);
  }
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::string(argv[1]) == "gpu";
  if (!gpu) g_qp = oracle_qp_step;  // cpu mode: the oracle supplies every linear step
  test_models();
  test_assemble_kkt();
  test_merit_and_line_search();
  test_sqp_solve();
  test_nmpc();
  test_nmpc_writers();
  if (gpu) {
    test_parity();
    time_linear_step();
  }
  if (failures) {
    std::fprintf(stderr, "%d of %d checks failed\n", failures, checks);
    return 1;
  }
  std::printf("all %d checks passed (%s)\n", checks, gpu ? "gpu" : "cpu");
  return 0;
}
