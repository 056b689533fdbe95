// Drop-in replacement for the reference's proj/include/trajopt/pcg.hpp: the
// same PcgVariant / PcgConfig (field order and defaults) / SolveReport /
// PcgResult / PcgBreakdown and the three solver entry points with their exact
// signatures (pcg.hpp:12-70). The solve runs on the B200 (b2p_pcg_solve); the
// reference's validate_inputs messages and exception classes are reproduced
// by the library (pcg.cpp:24-47,66-100).
#pragma once

#include <Eigen/Dense>
#include <stdexcept>
#include <vector>

#include "trajopt/b200_detail.hpp"
#include "trajopt/block_tri.hpp"
#include "trajopt/schur.hpp"

namespace trajopt {

enum class PcgVariant { sequential, block_parallel };  // pcg.hpp:12

struct PcgConfig {  // pcg.hpp:14-29
  double epsilon = 1e-4;
  int max_iter = 0;
  bool deterministic_reductions = false;
  PcgVariant variant = PcgVariant::sequential;
  bool collect_trace = false;
  bool check_residual_drift = false;
};

struct SolveReport {  // pcg.hpp:31-38
  int iterations = 0;
  double exit_eta = 0.0;
  bool converged = false;
  std::vector<double> trace;
  double wall_time = 0.0;
  double max_residual_drift = 0.0;
};

struct PcgResult {  // pcg.hpp:40-43
  Eigen::VectorXd lambda;
  SolveReport report;
};

// PcgBreakdown (pcg.hpp:47-50) is declared in trajopt/b200_detail.hpp so the
// status -> exception mapping can throw it.

/// pcg_solve_auto (pcg.cpp:364-369): dispatch on cfg.variant, on the GPU.
inline PcgResult pcg_solve_auto(const BlockTriMatrix& S, const Preconditioner& P,
                                const Eigen::VectorXd& gamma, const Eigen::VectorXd& lambda0,
                                const PcgConfig& cfg) {
  const b2p_pcg_config c{cfg.epsilon,
                         cfg.max_iter,
                         cfg.deterministic_reductions ? 1 : 0,
                         static_cast<int32_t>(cfg.variant),
                         cfg.collect_trace ? 1 : 0,
                         cfg.check_residual_drift ? 1 : 0,
                         0};
  const int dim = S.dim();
  const bool id = P.kind == PrecondKind::identity;
  PcgResult out;
  out.lambda = Eigen::VectorXd(dim > 0 ? dim : 1);
  std::vector<double> trace(static_cast<std::size_t>(cfg.max_iter > 0 ? cfg.max_iter : dim) + 1);
  b2p_solve_report rep{};
  b2p_error e{};
  b200::raise(b2p_pcg_solve(b200::context(), B2P_F64, S.block_rows(), S.block_dim(), S.b200_data(),
                            static_cast<int>(P.kind), P.order, id ? 0 : P.phi_inv.block_rows(),
                            id ? 0 : P.phi_inv.block_dim(), id ? nullptr : P.phi_inv.b200_data(),
                            gamma.data(), static_cast<int>(gamma.size()), lambda0.data(),
                            static_cast<int>(lambda0.size()), &c, out.lambda.data(), &rep,
                            trace.data(), &e),
              e);
  if (dim <= 0) out.lambda = Eigen::VectorXd(0);
  out.report.iterations = rep.iterations;
  out.report.exit_eta = rep.exit_eta;
  out.report.converged = rep.converged != 0;
  out.report.trace.assign(trace.begin(), trace.begin() + rep.trace_len);
  out.report.wall_time = rep.wall_time;
  out.report.max_residual_drift = rep.max_residual_drift;
  return out;
}

/// pcg_solve (pcg.cpp:55-129).
inline PcgResult pcg_solve(const BlockTriMatrix& S, const Preconditioner& P,
                           const Eigen::VectorXd& gamma, const Eigen::VectorXd& lambda0,
                           const PcgConfig& cfg) {
  PcgConfig c = cfg;
  c.variant = PcgVariant::sequential;
  return pcg_solve_auto(S, P, gamma, lambda0, c);
}

/// pcg_solve_block_parallel (pcg.cpp:157-362): the device kernels' fixed-order
/// reductions are deterministic with or without deterministic_reductions.
inline PcgResult pcg_solve_block_parallel(const BlockTriMatrix& S, const Preconditioner& P,
                                          const Eigen::VectorXd& gamma,
                                          const Eigen::VectorXd& lambda0, const PcgConfig& cfg) {
  PcgConfig c = cfg;
  c.variant = PcgVariant::block_parallel;
  return pcg_solve_auto(S, P, gamma, lambda0, c);
}

}  // namespace trajopt

#ifdef TRAJOPT_B200_RECONSTRUCT_PRIMAL
namespace trajopt {
/// reconstruct_primal (kkt.hpp:65, kkt.cpp:153-181) on the GPU. Opt-in: the
/// reference defines it in kkt.cpp next to assemble_kkt, so an integrator who
/// wants the device version defines this macro in exactly one translation
/// unit and removes the CPU definition from kkt.cpp.
Eigen::VectorXd reconstruct_primal(const KKTSystem& kkt, const Eigen::VectorXd& lambda) {
  const b200::PackedKKT p = b200::pack(kkt);
  const b2p_kkt v = p.view(kkt);
  Eigen::VectorXd dz(kkt.primal_dim());
  b2p_error e{};
  b200::raise(b2p_reconstruct_primal(b200::context(), B2P_F64, &v, lambda.data(),
                                     static_cast<int>(lambda.size()), dz.data(), &e),
              e);
  return dz;
}
}  // namespace trajopt
#endif
