// C++ adapter tests: the reference's own test cases (proj/tests/test_pcg.cpp,
// test_schur.cpp, test_block_tri.cpp) written against include/trajopt_b200.hpp,
// exactly as a reference caller would write them. Runs on the GPU (pytest -m gpu).
#include <cmath>
#include <cstdio>
#include <string>

#include "trajopt_b200.hpp"

using namespace trajopt_b200;

static int failures = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

static BlockTriMatrix identity_system(int blocks, int nb) {  // test_pcg.cpp:18-22
  BlockTriMatrix S(blocks, nb);
  for (int i = 0; i < blocks; ++i) S.set_diag(i, Matrix::identity(nb));
  return S;
}

static void kkt_helpers() {  // kkt.cpp:32-81 on a random instance: C dz = c at the exact solve
  const KKTSystem k = random_kkt(41, 5, 3, 2);
  const Matrix G = k.dense_G(), C = k.dense_C();
  const Vector g = k.dense_g(), c = k.constraint_rhs();
  CHECK(G.rows == k.primal_dim() && C.rows == k.dual_dim() && C.cols == k.primal_dim());
  CHECK(static_cast<int>(g.size()) == k.primal_dim() && static_cast<int>(c.size()) == k.dual_dim());
  for (int i = 0; i < k.n; ++i) CHECK(c[i] == k.x_s[i] - k.x0[i]);
  CHECK(c[static_cast<size_t>(k.n)] == -k.knots[0].e[0]);
  CHECK(C(0, 0) == 1.0 && C(k.n, 0) == -k.knots[0].A(0, 0));
  CHECK(G(0, 0) == k.knots[0].Q(0, 0) && G(k.n, k.n) == k.knots[0].R(0, 0));
}

int main() {
  kkt_helpers();
  {  // test_pcg.cpp:47-60 — scalar 2x2 within two iterations
    BlockTriMatrix S(2, 1);
    Matrix two = Matrix::identity(1);
    two(0, 0) = 2.0;
    S.set_diag(0, two);
    S.set_diag(1, two);
    S.set_right(0, Matrix::identity(1));
    S.set_left(1, Matrix::identity(1));
    PcgConfig cfg;
    cfg.epsilon = 1e-12;
    const PcgResult res = pcg_solve(S, build_identity(), {3.0, 3.0}, {0.0, 0.0}, cfg);
    CHECK(res.report.converged);
    CHECK(res.report.iterations <= 2);
    CHECK(std::fabs(res.lambda[0] - 1.0) <= 1e-10 && std::fabs(res.lambda[1] - 1.0) <= 1e-10);
  }
  {  // test_pcg.cpp:32-45 — identity system, exactly one iteration, both variants
    const BlockTriMatrix S = identity_system(3, 2);
    const Vector gamma = {0.5, -1.0, 1.5, 0.25, -0.75, 1.25};
    for (PcgVariant v : {PcgVariant::sequential, PcgVariant::block_parallel}) {
      PcgConfig cfg;
      cfg.epsilon = 1e-12;
      cfg.variant = v;
      const PcgResult res = pcg_solve_auto(S, build_identity(), gamma, Vector(6, 0.0), cfg);
      CHECK(res.report.iterations == 1);
      for (int i = 0; i < 6; ++i) CHECK(std::fabs(res.lambda[i] - gamma[i]) <= 1e-14);
    }
  }
  {  // test_pcg.cpp:162-171 — breakdown is a PcgBreakdown
    BlockTriMatrix S(2, 1);
    Matrix neg = Matrix::identity(1);
    neg(0, 0) = -1.0;
    S.set_diag(0, neg);
    S.set_diag(1, neg);
    bool thrown = false;
    try {
      PcgConfig cfg;
      cfg.epsilon = 1e-10;
      pcg_solve(S, build_identity(), {1.0, 1.0}, {0.0, 0.0}, cfg);
    } catch (const PcgBreakdown&) {
      thrown = true;
    }
    CHECK(thrown);
  }
  {  // test_pcg.cpp:173-178 — dimension message
    bool thrown = false;
    try {
      pcg_solve(identity_system(3, 2), build_identity(), Vector(5, 0.0), Vector(6, 0.0),
                PcgConfig{});
    } catch (const std::invalid_argument& e) {
      thrown = std::string(e.what()).find("length 6") != std::string::npos;
    }
    CHECK(thrown);
  }
  {  // test_schur.cpp:147-154 via the full builder chain, and the fused path
    const KKTSystem kkt = random_kkt(62, 10, 3, 2);
    const SchurSystem s = build_schur(kkt);
    CHECK(s.S.max_asymmetry() <= 1e-12);
    const Preconditioner P = build_symmetric_stair(s);
    CHECK(P.phi_inv.max_asymmetry() <= 1e-12);
    PcgConfig cfg;
    cfg.epsilon = 1e-10;
    const PcgResult a = pcg_solve(s.S, P, s.gamma, Vector(s.gamma.size(), 0.0), cfg);
    const PcgResult b = solve(kkt, PrecondKind::symmetric_stair, 1, cfg);
    CHECK(a.report.converged && b.report.converged);
    CHECK(a.report.iterations == b.report.iterations);
    double worst = 0.0;
    for (size_t i = 0; i < a.lambda.size(); ++i)
      worst = std::fmax(worst, std::fabs(a.lambda[i] - b.lambda[i]));
    CHECK(worst <= 1e-9);
    // block Cholesky baseline agrees with PCG
    const Vector x = s.S.cholesky_solve(s.gamma);
    double w2 = 0.0;
    for (size_t i = 0; i < x.size(); ++i) w2 = std::fmax(w2, std::fabs(x[i] - a.lambda[i]));
    CHECK(w2 <= 1e-5);
  }
  {  // reconstruct_primal: zero multipliers and identity G give dz = -g (test_kkt.cpp:101-109)
    KKTSystem kkt = random_kkt_family(0, 31, 3, 2, 1);
    for (auto& kd : kkt.knots) {
      kd.Q = Matrix::identity(2);
      if (!kd.R.a.empty()) kd.R = Matrix::identity(1);
    }
    const Vector dz = reconstruct_primal(kkt, Vector(kkt.dual_dim(), 0.0));
    double worst = 0.0;
    size_t off = 0;
    for (int k = 0; k <= kkt.N; ++k) {
      for (double v : kkt.knots[k].q) worst = std::fmax(worst, std::fabs(dz[off++] + v));
      if (k < kkt.N)
        for (double v : kkt.knots[k].r) worst = std::fmax(worst, std::fabs(dz[off++] + v));
    }
    CHECK(off == dz.size() && worst <= 1e-14);
    bool thrown = false;
    try {
      reconstruct_primal(kkt, Vector(5, 0.0));
    } catch (const std::invalid_argument& e) {
      thrown = std::string(e.what()) == "reconstruct_primal: expected lambda of length 8, got 5";
    }
    CHECK(thrown);
  }
  {  // boundary padding rejects mutation (test_block_tri.cpp:91-95)
    BlockTriMatrix M(3, 2);
    bool t1 = false, t2 = false;
    try {
      M.set_left(0, Matrix::identity(2));
    } catch (const std::invalid_argument&) {
      t1 = true;
    }
    try {
      M.set_right(2, Matrix::identity(2));
    } catch (const std::invalid_argument&) {
      t2 = true;
    }
    CHECK(t1 && t2);
  }
  if (failures == 0) std::printf("test_adapter: all checks passed\n");
  return failures == 0 ? 0 : 1;
}
