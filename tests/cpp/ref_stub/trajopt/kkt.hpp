// TEST-ONLY stand-in for the reference's proj/include/trajopt/kkt.hpp (which
// needs models.hpp / trajectory.hpp and the reference tree, absent on the GPU
// box). It declares the KKT data types with the reference's field names and
// Eigen types (kkt.hpp:13-46) and the reconstruct_primal prototype (kkt.hpp:65),
// which is all the drop-in headers and sqp.cpp:171-176 touch. An integrator
// uses the reference's real kkt.hpp instead of this file.
#pragma once

#include <Eigen/Dense>
#include <vector>

namespace trajopt {

struct KnotData {  // kkt.hpp:13-21
  Eigen::MatrixXd Q;
  Eigen::VectorXd q;
  Eigen::MatrixXd R;
  Eigen::VectorXd r;
  Eigen::MatrixXd A;
  Eigen::MatrixXd B;
  Eigen::VectorXd e;
};

struct KKTSystem {  // kkt.hpp:29-46
  int N = 0;
  int n = 0;
  int m = 0;
  std::vector<KnotData> knots;
  Eigen::VectorXd x_s;
  Eigen::VectorXd x0;
  int primal_dim() const { return (N + 1) * n + N * m; }
  int dual_dim() const { return (N + 1) * n; }
};

Eigen::VectorXd reconstruct_primal(const KKTSystem& kkt, const Eigen::VectorXd& lambda);

}  // namespace trajopt
