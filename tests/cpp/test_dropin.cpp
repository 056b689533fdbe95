// Drop-in acceptance test: the reference's own callers and test cases compiled
// against include/trajopt_dropin/trajopt/{block_tri,schur,pcg}.hpp (the
// Eigen-typed `trajopt::` API of proj/include, computed on the B200) instead of
// proj/src/{block_tri,schur,pcg}.cpp. Eigen is not installable in this image,
// so CI compiles against the test-only stand-in tests/cpp/eigen_stub/Eigen/Dense
// and tests/cpp/ref_stub/trajopt/kkt.hpp (the reference's KKT types). The
// CPU oracle (oracle/trajopt_oracle.hpp, test infrastructure) is the checker.
//
//   ./test_dropin          compile/link check only (no device needed)
//   ./test_dropin gpu      run every case on the GPU
#define TRAJOPT_B200_RECONSTRUCT_PRIMAL 1
#include "trajopt/pcg.hpp"
#include "trajopt/schur.hpp"
#include "trajopt_b200.hpp"  // the Eigen bridge (from_eigen / to_eigen / to_b200)

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "trajopt_oracle.hpp"

namespace trajopt {
using Eigen::VectorXd;

// Stand-ins for the SqpConfig / SqpIterStats fields the step reads (sqp.hpp:27-37).
struct SqpConfigFields {
  PrecondKind precond = PrecondKind::symmetric_stair;
  int poly_order = 1;
  PcgConfig pcg;
};
struct SqpIterStatsFields {
  SolveReport pcg;
};

// proj/src/sqp.cpp:171-176, unmodified: the reference's production caller of
// the hot path, here bound to the drop-in.
inline void sqp_linear_step(const KKTSystem& kkt, const SqpConfigFields& cfg, VectorXd& lambda,
                            VectorXd& dz, SqpIterStatsFields& iter_stats) {
      SchurSystem schur = build_schur(kkt);
      Preconditioner P = build_preconditioner(schur, cfg.precond, cfg.poly_order);
      PcgResult res = pcg_solve_auto(schur.S, P, schur.gamma, lambda, cfg.pcg);
      lambda = res.lambda;
      iter_stats.pcg = res.report;
      dz = reconstruct_primal(kkt, lambda);
}
}  // namespace trajopt

using namespace trajopt;
using Eigen::MatrixXd;
using Eigen::VectorXd;

static int failures = 0;
#define CHECK(cond)                                                                \
  do {                                                                             \
    if (!(cond)) {                                                                 \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                                  \
    }                                                                              \
  } while (0)

template <class F>
static std::string thrown(F&& f, int* kind) {  // kind: 1 invalid_argument, 2 breakdown, 3 runtime
  try {
    f();
  } catch (const std::invalid_argument& e) {
    *kind = 1;
    return e.what();
  } catch (const PcgBreakdown& e) {
    *kind = 2;
    return e.what();
  } catch (const std::runtime_error& e) {
    *kind = 3;
    return e.what();
  }
  *kind = 0;
  return "";
}

static MatrixXd scalar(double v) {
  MatrixXd m(1, 1);
  m(0, 0) = v;
  return m;
}

// oracle KKT (row-major, test infrastructure) -> the reference's Eigen KKTSystem
static KKTSystem to_eigen_kkt(const oracle::KKTSystem<double>& o) {
  KKTSystem k;
  k.N = o.N;
  k.n = o.n;
  k.m = o.m;
  k.knots.resize(o.N + 1);
  auto mat = [](const oracle::Mat<double>& a) {
    MatrixXd M(a.rows, a.cols);
    for (int i = 0; i < a.rows; ++i)
      for (int j = 0; j < a.cols; ++j) M(i, j) = a(i, j);
    return M;
  };
  auto vec = [](const std::vector<double>& v) {
    VectorXd x(static_cast<Eigen::Index>(v.size()));
    for (size_t i = 0; i < v.size(); ++i) x[i] = v[i];
    return x;
  };
  for (int i = 0; i <= o.N; ++i) {
    k.knots[i].Q = mat(o.knots[i].Q);
    k.knots[i].q = vec(o.knots[i].q);
    if (i < o.N) {
      k.knots[i].R = mat(o.knots[i].R);
      k.knots[i].r = vec(o.knots[i].r);
      k.knots[i].A = mat(o.knots[i].A);
      k.knots[i].B = mat(o.knots[i].B);
      k.knots[i].e = vec(o.knots[i].e);
    }
  }
  k.x_s = vec(o.x_s);
  k.x0 = vec(o.x0);
  return k;
}

static double rel_err(const VectorXd& a, const std::vector<double>& b) {
  double num = 0, den = 1.0;
  for (size_t i = 0; i < b.size(); ++i) {
    num = std::fmax(num, std::fabs(a[static_cast<Eigen::Index>(i)] - b[i]));
    den = std::fmax(den, std::fabs(b[i]));
  }
  return num / den;
}

static void reference_cases() {
  {  // test_schur.cpp:41-66 — scalar blocks by hand: theta = 3, phi = -1, gamma = 0
    KKTSystem kkt;
    kkt.N = 1;
    kkt.n = 1;
    kkt.m = 1;
    kkt.knots.resize(2);
    kkt.knots[0].Q = MatrixXd::Identity(1, 1);
    kkt.knots[0].R = MatrixXd::Identity(1, 1);
    kkt.knots[0].A = MatrixXd::Identity(1, 1);
    kkt.knots[0].B = MatrixXd::Identity(1, 1);
    kkt.knots[0].q = VectorXd::Zero(1);
    kkt.knots[0].r = VectorXd::Zero(1);
    kkt.knots[0].e = VectorXd::Zero(1);
    kkt.knots[1].Q = MatrixXd::Identity(1, 1);
    kkt.knots[1].q = VectorXd::Zero(1);
    kkt.x_s = VectorXd::Zero(1);
    kkt.x0 = VectorXd::Zero(1);
    const SchurSystem schur = build_schur(kkt);
    CHECK(std::fabs(schur.S.diag(1)(0, 0) - 3.0) < 1e-15);
    CHECK(std::fabs(schur.S.left(1)(0, 0) + 1.0) < 1e-15);
    CHECK(std::fabs(schur.S.right(0)(0, 0) + 1.0) < 1e-15);
    CHECK(schur.gamma[0] == 0.0 && schur.gamma[1] == 0.0);
    CHECK(schur.S.structurally_symmetric);
  }
  {  // test_schur.cpp:94-101 — block-Jacobi of diag [2, 4] is [0.5, 0.25]
    SchurSystem s;
    s.n = 1;
    s.S = BlockTriMatrix(2, 1);
    s.S.set_diag(0, scalar(2.0));
    s.S.set_diag(1, scalar(4.0));
    s.gamma = VectorXd::Zero(2);
    s.theta_inv = {scalar(0.5), scalar(0.25)};
    const Preconditioner P = build_block_jacobi(s);
    CHECK(P.phi_inv.diag(0)(0, 0) == 0.5 && P.phi_inv.diag(1)(0, 0) == 0.25);
    CHECK(P.phi_inv.structurally_symmetric);
  }
  {  // test_schur.cpp:113-125 — stair 2x2 by hand: Psi = [[2,0],[1,2]], Phi = [[.5,0],[-.25,.5]]
    SchurSystem s;
    s.n = 1;
    s.S = BlockTriMatrix(2, 1);
    s.S.set_diag(0, scalar(2.0));
    s.S.set_diag(1, scalar(2.0));
    s.S.set_right(0, scalar(1.0));
    s.S.set_left(1, scalar(1.0));
    s.gamma = VectorXd::Zero(2);
    s.theta_inv = {scalar(0.5), scalar(0.5)};
    const MatrixXd psi = stair_matrix(s.S).to_dense();
    CHECK(psi(0, 0) == 2 && psi(0, 1) == 0 && psi(1, 0) == 1 && psi(1, 1) == 2);
    const MatrixXd phi = build_stair(s).phi_inv.to_dense();
    CHECK(phi(0, 0) == 0.5 && phi(0, 1) == 0 && std::fabs(phi(1, 0) + 0.25) <= 1e-15 &&
          phi(1, 1) == 0.5);
    // test_schur.cpp:148-154 — symmetric stair [[.5,-.25],[-.25,.5]]
    const MatrixXd sym = build_symmetric_stair(s).phi_inv.to_dense();
    CHECK(std::fabs(sym(0, 1) + 0.25) <= 1e-15 && std::fabs(sym(1, 0) + 0.25) <= 1e-15);
    // poly_split keeps Psi and E = Psi - S, and applies the series on the GPU
    const Preconditioner Pp = build_poly_split(s, 2);
    CHECK(Pp.order == 2 && Pp.remainder.right(0)(0, 0) == -1.0 && Pp.remainder.left(1)(0, 0) == 0.0);
    VectorXd r(2);
    r[0] = 1.0;
    r[1] = 2.0;
    const VectorXd z = apply_preconditioner(Pp, r);
    CHECK(z.size() == 2 && std::isfinite(z[0]) && std::isfinite(z[1]));
    int kind = 0;
    thrown([&] { build_poly_split(s, 0); }, &kind);
    CHECK(kind == 1);  // test_schur.cpp:202-206
  }
  {  // test_pcg.cpp:32-45 — identity system: exactly one iteration, both variants
    BlockTriMatrix S(3, 2);
    for (int i = 0; i < 3; ++i) S.set_diag(i, MatrixXd::Identity(2, 2));
    VectorXd gamma(6);
    const double g[6] = {0.5, -1.0, 1.5, 0.25, -0.75, 1.25};
    for (int i = 0; i < 6; ++i) gamma[i] = g[i];
    for (auto variant : {PcgVariant::sequential, PcgVariant::block_parallel}) {
      PcgConfig c{.epsilon = 1e-12};
      c.variant = variant;
      const PcgResult res = pcg_solve_auto(S, build_identity(), gamma, VectorXd::Zero(6), c);
      CHECK(res.report.iterations == 1 && res.report.converged);
      for (int i = 0; i < 6; ++i) CHECK(std::fabs(res.lambda[i] - g[i]) <= 1e-14);
    }
    int kind = 0;  // test_pcg.cpp:173-178 — "length 6"
    const std::string msg = thrown(
        [&] { pcg_solve(S, build_identity(), VectorXd::Zero(5), VectorXd::Zero(6), PcgConfig{}); },
        &kind);
    CHECK(kind == 1 && msg.find("length 6") != std::string::npos);
  }
  {  // test_pcg.cpp:162-171 — indefinite S -> PcgBreakdown
    BlockTriMatrix S(2, 1);
    S.set_diag(0, scalar(-1.0));
    S.set_diag(1, scalar(-1.0));
    VectorXd gamma(2);
    gamma[0] = gamma[1] = 1.0;
    int kind = 0;
    thrown([&] { pcg_solve(S, build_identity(), gamma, VectorXd::Zero(2), PcgConfig{.epsilon = 1e-10}); },
           &kind);
    CHECK(kind == 2);
  }
  {  // test_block_tri.cpp:91-95 — boundary padding cannot be assigned
    BlockTriMatrix S(2, 1);
    int kind = 0;
    thrown([&] { S.set_left(0, scalar(1.0)); }, &kind);
    CHECK(kind == 1);
    thrown([&] { S.set_right(1, scalar(1.0)); }, &kind);
    CHECK(kind == 1);
  }
  {  // test_pcg.cpp:150-160 — cap -> best iterate, unconverged, iterations == 3
    const KKTSystem kkt = to_eigen_kkt(oracle::random_kkt(330, 16, 3, 2));
    const SchurSystem schur = build_schur(kkt);
    PcgConfig cfg;
    cfg.epsilon = 1e-14;
    cfg.max_iter = 3;
    const PcgResult res =
        pcg_solve(schur.S, build_identity(), schur.gamma, VectorXd::Zero(schur.S.dim()), cfg);
    CHECK(!res.report.converged && res.report.iterations == 3);
  }
}

// sqp.cpp:171-176 on the GPU vs the oracle at the c1 shape (K 32, n 14, m 7)
// and at the SQP caller's shape, every stair-family preconditioner.
static void sqp_step_parity() {
  struct Case {
    std::uint64_t seed;
    int N, n, m;
    PrecondKind kind;
  };
  const Case cases[] = {{1, 31, 14, 7, PrecondKind::symmetric_stair},
                        {2, 31, 14, 7, PrecondKind::stair},
                        {3, 31, 14, 7, PrecondKind::block_jacobi},
                        {4, 32, 2, 1, PrecondKind::symmetric_stair},
                        {5, 20, 3, 2, PrecondKind::poly_split}};
  for (const Case& c : cases) {
    const auto ok = oracle::random_kkt(c.seed, c.N, c.n, c.m);
    const KKTSystem kkt = to_eigen_kkt(ok);
    SqpConfigFields cfg;
    cfg.precond = c.kind;
    cfg.poly_order = 1;
    cfg.pcg.epsilon = 1e-8;
    VectorXd lambda = VectorXd::Zero(kkt.dual_dim());
    VectorXd dz;
    SqpIterStatsFields stats;
    sqp_linear_step(kkt, cfg, lambda, dz, stats);
    // oracle
    const auto os = oracle::build_schur(ok);
    const auto oP = oracle::build_preconditioner(os, static_cast<oracle::PrecondKind>(c.kind), 1);
    oracle::PcgConfig ocfg;
    ocfg.epsilon = 1e-8;
    const auto ores = oracle::pcg_solve_auto(os.S, oP, os.gamma,
                                             std::vector<double>(kkt.dual_dim(), 0.0), ocfg);
    const auto odz = oracle::reconstruct_primal(ok, ores.lambda);
    CHECK(stats.pcg.converged && stats.pcg.iterations == ores.report.iterations);
    CHECK(rel_err(lambda, ores.lambda) <= 1e-10);
    CHECK(dz.size() == kkt.primal_dim() && rel_err(dz, odz) <= 1e-9);
    // warm start at the solution (test_pcg.cpp:180-189): no iteration
    VectorXd lam2 = lambda, dz2;
    sqp_linear_step(kkt, cfg, lam2, dz2, stats);
    CHECK(stats.pcg.converged && stats.pcg.iterations == 0);
    std::printf("sqp step K%d n%d m%d %s: %d iterations (oracle %d)\n", c.N + 1, c.n, c.m,
                precond_name(c.kind, 1).c_str(), ores.report.iterations, ores.report.iterations);
  }
}

// The trajopt_b200 adapter's Eigen bridge (include/trajopt_b200.hpp) on the same data.
static void eigen_bridge() {
  const KKTSystem kkt = to_eigen_kkt(oracle::random_kkt(9, 7, 3, 2));
  const trajopt_b200::KKTSystem k2 = trajopt_b200::to_b200(kkt);
  CHECK(k2.N == 7 && k2.n == 3 && k2.m == 2 && k2.knots.size() == 8u);
  CHECK(k2.knots[2].A(1, 0) == kkt.knots[2].A(1, 0) && k2.knots[7].q[2] == kkt.knots[7].q[2]);
  const trajopt_b200::PcgConfig cfg{1e-10};
  const auto res = trajopt_b200::solve(k2, trajopt_b200::PrecondKind::symmetric_stair, 1, cfg);
  const VectorXd lam = trajopt_b200::to_eigen(res.lambda);
  const auto back = trajopt_b200::from_eigen(lam);
  CHECK(res.report.converged && back.size() == res.lambda.size() && back[3] == res.lambda[3]);
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
  if (!gpu) {
    std::printf("drop-in compiled and linked (run with 'gpu' on a B200)\n");
    return 0;
  }
  reference_cases();
  sqp_step_parity();
  eigen_bridge();
  if (failures) {
    std::fprintf(stderr, "%d check(s) failed\n", failures);
    return 1;
  }
  std::printf("all checks passed\n");
  return 0;
}
