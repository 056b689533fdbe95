// Drop-in replacement for the reference's proj/include/trajopt/block_tri.hpp:
// the same class, names, signatures, storage layout ([K][left|diag|right]
// row-major nb x nb blocks, zero boundary padding, block_tri.cpp:11-29) and
// exception texts; matvec / max_asymmetry / max_abs / cholesky_solve run on
// the B200 through the C-ABI (include/b2p.h, libb2p.so). Put
// include/trajopt_dropin ahead of the reference's include directory and link
// libb2p.so instead of compiling proj/src/block_tri.cpp.
#pragma once

#include <Eigen/Dense>
#include <cstddef>
#include <stdexcept>
#include <string>
#include <vector>

#include "trajopt/b200_detail.hpp"

namespace trajopt {

using Matrix = Eigen::MatrixXd;
using Vector = Eigen::VectorXd;
using BlockRM = Eigen::Matrix<double, Eigen::Dynamic, Eigen::Dynamic, Eigen::RowMajor>;

/// block_tri.hpp:18-75.
class BlockTriMatrix {
 public:
  BlockTriMatrix() = default;
  BlockTriMatrix(int num_block_rows, int block_dim)  // block_tri.cpp:11-17
      : num_rows_(num_block_rows), block_dim_(block_dim) {
    if (num_block_rows < 1 || block_dim < 1)
      throw std::invalid_argument("BlockTriMatrix: need at least one block row and block_dim >= 1");
    data_.assign(static_cast<std::size_t>(num_rows_) * 3 * block_dim_ * block_dim_, 0.0);
  }

  int block_rows() const { return num_rows_; }
  int block_dim() const { return block_dim_; }
  int dim() const { return num_rows_ * block_dim_; }
  bool empty() const { return num_rows_ == 0; }

  Eigen::Map<const BlockRM> left(int row) const { return block(row, 0); }
  Eigen::Map<const BlockRM> diag(int row) const { return block(row, 1); }
  Eigen::Map<const BlockRM> right(int row) const { return block(row, 2); }

  void set_left(int row, const Eigen::Ref<const Matrix>& b) {  // block_tri.cpp:46-52
    check_row(row);
    check_block_shape(b);
    if (row == 0)
      throw std::invalid_argument("BlockTriMatrix: row 0 has no left block (boundary padding)");
    put(row, 0, b);
  }
  void set_diag(int row, const Eigen::Ref<const Matrix>& b) {
    check_row(row);
    check_block_shape(b);
    put(row, 1, b);
  }
  void set_right(int row, const Eigen::Ref<const Matrix>& b) {  // block_tri.cpp:60-67
    check_row(row);
    check_block_shape(b);
    if (row == num_rows_ - 1)
      throw std::invalid_argument("BlockTriMatrix: last row has no right block (boundary padding)");
    put(row, 2, b);
  }

  /// y = M x (block_tri.cpp:70-80), on the GPU (b2p_blocktri_matvec).
  Vector matvec(const Eigen::Ref<const Vector>& x) const {
    Vector y(dim());
    b2p_error e{};
    b200::raise(b2p_blocktri_matvec(b200::context(), B2P_F64, num_rows_, block_dim_, data_.data(),
                                    x.data(), static_cast<int>(x.size()), y.data(), &e),
                e);
    return y;
  }

  /// y_row = left x_{row-1} + diag x_row + right x_{row+1} (block_tri.cpp:82-92):
  /// the row of the device matvec.
  void matvec_block(int row, const Eigen::Ref<const Vector>& x, Eigen::Ref<Vector> y_block) const {
    check_row(row);
    const Vector y = matvec(x);
    for (int i = 0; i < block_dim_; ++i) y_block[i] = y[static_cast<Eigen::Index>(row) * block_dim_ + i];
  }

  Matrix to_dense() const {  // block_tri.cpp:94-104
    Matrix dense = Matrix::Zero(dim(), dim());
    const int nb = block_dim_;
    for (int row = 0; row < num_rows_; ++row)
      for (int s = 0; s < 3; ++s) {
        const int col = row - 1 + s;
        if (col < 0 || col >= num_rows_) continue;
        const auto b = block(row, s);
        for (int i = 0; i < nb; ++i)
          for (int j = 0; j < nb; ++j) dense(row * nb + i, col * nb + j) = b(i, j);
      }
    return dense;
  }

  static BlockTriMatrix from_dense(const Eigen::Ref<const Matrix>& dense, int block_dim) {
    if (dense.rows() != dense.cols() || dense.rows() % block_dim != 0)  // block_tri.cpp:106-119
      throw std::invalid_argument("BlockTriMatrix::from_dense: matrix size " +
                                  std::to_string(dense.rows()) + "x" + std::to_string(dense.cols()) +
                                  " is not square with block_dim " + std::to_string(block_dim));
    const int rows = static_cast<int>(dense.rows()) / block_dim;
    BlockTriMatrix out(rows, block_dim);
    for (int row = 0; row < rows; ++row)
      for (int s = 0; s < 3; ++s) {
        const int col = row - 1 + s;
        if (col < 0 || col >= rows) continue;
        double* d = out.data_.data() + (static_cast<std::size_t>(row) * 3 + s) * block_dim * block_dim;
        for (int i = 0; i < block_dim; ++i)
          for (int j = 0; j < block_dim; ++j)
            d[i * block_dim + j] = dense(row * block_dim + i, col * block_dim + j);
      }
    return out;
  }

  /// block_tri.cpp:167-177, on the GPU.
  double max_asymmetry() const { return check(0); }
  /// block_tri.cpp:161-165, on the GPU.
  double max_abs() const { return check(1); }

  /// Block Thomas direct solve (block_tri.cpp:121-159), on the GPU.
  Vector cholesky_solve(const Eigen::Ref<const Vector>& rhs) const {
    Vector x(dim());
    b2p_error e{};
    b200::raise(b2p_blocktri_cholesky_solve(b200::context(), B2P_F64, num_rows_, block_dim_,
                                            data_.data(), rhs.data(), static_cast<int>(rhs.size()),
                                            x.data(), &e),
                e);
    return x;
  }

  bool structurally_symmetric = false;

  /// Raw [K][3][nb][nb] storage for the other drop-in headers (not in the reference).
  const double* b200_data() const { return data_.data(); }
  double* b200_data() { return data_.data(); }

 private:
  Eigen::Map<const BlockRM> block(int row, int slot) const {
    const std::size_t bsz = static_cast<std::size_t>(block_dim_) * block_dim_;
    return Eigen::Map<const BlockRM>(data_.data() + (static_cast<std::size_t>(row) * 3 + slot) * bsz,
                                     block_dim_, block_dim_);
  }
  void put(int row, int slot, const Eigen::Ref<const Matrix>& b) {
    double* d = data_.data() + (static_cast<std::size_t>(row) * 3 + slot) * block_dim_ * block_dim_;
    for (int i = 0; i < block_dim_; ++i)
      for (int j = 0; j < block_dim_; ++j) d[i * block_dim_ + j] = b(i, j);
  }
  void check_row(int row) const {
    if (row < 0 || row >= num_rows_)
      throw std::invalid_argument("BlockTriMatrix: block row " + std::to_string(row) +
                                  " out of range [0, " + std::to_string(num_rows_) + ")");
  }
  void check_block_shape(const Eigen::Ref<const Matrix>& b) const {
    if (b.rows() != block_dim_ || b.cols() != block_dim_)
      throw std::invalid_argument("BlockTriMatrix: expected " + std::to_string(block_dim_) + "x" +
                                  std::to_string(block_dim_) + " block, got " +
                                  std::to_string(b.rows()) + "x" + std::to_string(b.cols()));
  }
  double check(int which) const {
    if (num_rows_ == 0) return 0.0;
    double v[2] = {0.0, 0.0};
    b2p_error e{};
    b200::raise(b2p_blocktri_check(b200::context(), B2P_F64, num_rows_, block_dim_, data_.data(),
                                   &v[0], &v[1], &e),
                e);
    return v[which];
  }

  int num_rows_ = 0;
  int block_dim_ = 0;
  std::vector<double> data_;
};

}  // namespace trajopt
