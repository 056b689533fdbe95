// Drop-in replacement for the reference's proj/include/trajopt/schur.hpp: the
// same types (SchurSystem, PrecondKind, Preconditioner), free functions and
// signatures (schur.hpp:19-56), with build_schur / the preconditioner
// builders / apply_preconditioner computed on the B200 (include/b2p.h).
// Eigen's column-major KnotData is packed into the C-ABI's row-major SoA here.
#pragma once

#include <Eigen/Dense>
#include <string>
#include <vector>

#include "trajopt/b200_detail.hpp"
#include "trajopt/block_tri.hpp"
#include "trajopt/kkt.hpp"

namespace trajopt {

/// schur.hpp:19-24.
struct SchurSystem {
  BlockTriMatrix S;
  Eigen::VectorXd gamma;
  std::vector<Eigen::MatrixXd> theta_inv;
  int n = 0;
};

/// schur.hpp:26 (same order as b2p_precond_kind).
enum class PrecondKind { identity, block_jacobi, stair, symmetric_stair, poly_split };

/// schur.hpp:33-38.
struct Preconditioner {
  PrecondKind kind = PrecondKind::identity;
  int order = 0;
  BlockTriMatrix phi_inv;
  BlockTriMatrix stair_psi;
  BlockTriMatrix remainder;
};

/// schur.cpp:27-36.
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

namespace b200 {
/// KKTSystem (Eigen, kkt.hpp:29-46) -> the b2p_kkt row-major SoA buffers.
struct PackedKKT {
  std::vector<double> Q, q, R, r, A, B, e, x_s, x0;
  b2p_kkt view(const KKTSystem& k) const {
    return b2p_kkt{k.N,      k.n,      k.m,      0,        Q.data(),   q.data(),  R.data(),
                   r.data(), A.data(), B.data(), e.data(), x_s.data(), x0.data()};
  }
};
inline PackedKKT pack(const KKTSystem& kkt) {
  if (static_cast<int>(kkt.knots.size()) != kkt.N + 1)
    throw std::invalid_argument("b2p: KKTSystem needs N+1 knots, got " +
                                std::to_string(kkt.knots.size()));
  PackedKKT p;
  for (int k = 0; k <= kkt.N; ++k) {
    const KnotData& kd = kkt.knots[k];
    append_rowmajor(kd.Q, p.Q);
    append_vec(kd.q, p.q);
    if (k < kkt.N) {
      append_rowmajor(kd.R, p.R);
      append_vec(kd.r, p.r);
      append_rowmajor(kd.A, p.A);
      append_rowmajor(kd.B, p.B);
      append_vec(kd.e, p.e);
    }
  }
  append_vec(kkt.x_s, p.x_s);
  append_vec(kkt.x0, p.x0);
  const std::size_t K = kkt.N + 1, N = kkt.N, n = kkt.n, m = kkt.m;
  if (p.Q.size() != K * n * n || p.q.size() != K * n || p.R.size() != N * m * m ||
      p.r.size() != N * m || p.A.size() != N * n * n || p.B.size() != N * n * m ||
      p.e.size() != N * n || p.x_s.size() != n || p.x0.size() != n)
    throw std::invalid_argument("b2p: KKTSystem knot data does not match (N, n, m)");
  return p;
}
inline std::vector<double> pack_theta_inv(const SchurSystem& s) {
  std::vector<double> t;
  t.reserve(s.theta_inv.size() * s.n * s.n);
  for (const auto& M : s.theta_inv) append_rowmajor(M, t);
  return t;
}
}  // namespace b200

/// build_schur (schur.cpp:38-82) on the GPU (b2p_build_schur).
inline SchurSystem build_schur(const KKTSystem& kkt) {
  const b200::PackedKKT p = b200::pack(kkt);
  const b2p_kkt v = p.view(kkt);
  const int K = kkt.N + 1, n = kkt.n;
  SchurSystem out;
  out.n = n;
  out.S = BlockTriMatrix(K, n);
  out.gamma = Eigen::VectorXd(static_cast<Eigen::Index>(K) * n);
  std::vector<double> ti(static_cast<std::size_t>(K) * n * n);
  b2p_error e{};
  b200::raise(b2p_build_schur(b200::context(), B2P_F64, &v, out.S.b200_data(), out.gamma.data(),
                              ti.data(), &e),
              e);
  out.theta_inv.resize(K);
  for (int b = 0; b < K; ++b) {
    Eigen::MatrixXd M(n, n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) M(i, j) = ti[(static_cast<std::size_t>(b) * n + i) * n + j];
    out.theta_inv[b] = M;
  }
  out.S.structurally_symmetric = true;
  return out;
}

/// stair_matrix (schur.cpp:84-94) on the GPU.
inline BlockTriMatrix stair_matrix(const BlockTriMatrix& S) {
  BlockTriMatrix psi(S.block_rows(), S.block_dim());
  b2p_error e{};
  b200::raise(b2p_stair_matrix(b200::context(), B2P_F64, S.block_rows(), S.block_dim(),
                               S.b200_data(), psi.b200_data(), &e),
              e);
  return psi;
}

/// build_preconditioner (schur.cpp:164-173): Phi^-1 formed on the GPU.
inline Preconditioner build_preconditioner(const SchurSystem& schur, PrecondKind kind,
                                           int order = 1) {
  if (kind == PrecondKind::poly_split && order < 1)
    throw std::invalid_argument("build_poly_split: order must be >= 1, got " +
                                std::to_string(order));
  Preconditioner P;
  P.kind = kind;
  if (kind == PrecondKind::identity) return P;  // build_identity (schur.cpp:96)
  const int rows = schur.S.block_rows();
  P.phi_inv = BlockTriMatrix(rows, schur.n);
  const std::vector<double> ti = b200::pack_theta_inv(schur);
  b2p_error e{};
  b200::raise(b2p_build_preconditioner(b200::context(), B2P_F64, static_cast<int>(kind), order,
                                       rows, schur.n, schur.S.b200_data(), ti.data(),
                                       P.phi_inv.b200_data(), &e),
              e);
  P.phi_inv.structurally_symmetric =
      kind == PrecondKind::block_jacobi || kind == PrecondKind::symmetric_stair;
  if (kind == PrecondKind::poly_split) {  // schur.cpp:144-162
    P.order = order;
    P.stair_psi = stair_matrix(schur.S);
    // E = Psi - S: odd rows vanish, even rows keep the negated off-diagonals
    // (a sign flip of stored blocks, no rounding)
    P.remainder = BlockTriMatrix(rows, schur.n);
    const std::size_t nn = static_cast<std::size_t>(schur.n) * schur.n;
    for (int row = 0; row < rows; row += 2)
      for (int s = 0; s < 3; s += 2) {
        if ((s == 0 && row == 0) || (s == 2 && row + 1 >= rows)) continue;
        const double* src = schur.S.b200_data() + (static_cast<std::size_t>(row) * 3 + s) * nn;
        double* dst = P.remainder.b200_data() + (static_cast<std::size_t>(row) * 3 + s) * nn;
        for (std::size_t i = 0; i < nn; ++i) dst[i] = -src[i];
      }
  }
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

namespace b200 {
/// S = Psi - E of a poly_split preconditioner, reassembled exactly (the
/// C-ABI's series takes S; E's blocks are S's negated even-row off-diagonals).
inline std::vector<double> poly_system(const Preconditioner& P) {
  const int rows = P.stair_psi.block_rows(), nb = P.stair_psi.block_dim();
  std::vector<double> S(P.stair_psi.b200_data(),
                        P.stair_psi.b200_data() + static_cast<std::size_t>(rows) * 3 * nb * nb);
  for (std::size_t i = 0; i < S.size(); ++i) S[i] -= P.remainder.b200_data()[i];
  return S;
}
}  // namespace b200

/// apply_preconditioner (schur.cpp:175-194) on the GPU.
inline Eigen::VectorXd apply_preconditioner(const Preconditioner& P,
                                            const Eigen::Ref<const Eigen::VectorXd>& r) {
  if (P.kind == PrecondKind::identity) return Eigen::VectorXd(r);
  std::vector<double> S;
  if (P.kind == PrecondKind::poly_split) S = b200::poly_system(P);
  Eigen::VectorXd out(P.phi_inv.dim());
  b2p_error e{};
  b200::raise(b2p_apply_preconditioner(b200::context(), B2P_F64, static_cast<int>(P.kind), P.order,
                                       P.phi_inv.block_rows(), P.phi_inv.block_dim(),
                                       S.empty() ? nullptr : S.data(), P.phi_inv.b200_data(),
                                       r.data(), static_cast<int>(r.size()), out.data(), &e),
              e);
  return out;
}

}  // namespace trajopt
