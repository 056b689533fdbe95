// ============================================================================
// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// Eigen-free CPU restatement of the reference hot path (arXiv 2309.08079
// artifact, /root/reference/proj). It is the results oracle for the B200
// kernels: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load it. The product library never links it.
//
// Why a restatement: the reference needs Eigen3 >= 3.3 (proj/CMakeLists.txt:10),
// doctest and CLI11 (vendor/, absent: proj/.gitignore:2); none are on disk and
// there is no network, so it cannot be compiled here.
// Eigen's packet/blocking summation order is not reproduced bit-for-bit, so
// parity against the reference is tolerance-pinned; the oracle itself is pinned
// by the reference's own known-answer tests (tests/golden/reference_kats.json,
// tests/test_oracle_*.py).
//
// Every function cites the reference file:line it follows.
// ============================================================================
#pragma once

#include <algorithm>
#include <barrier>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <exception>
#include <functional>
#include <limits>
#include <mutex>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace oracle {

// ---------------------------------------------------------------------------
// parallel.hpp:18-71 — per-call std::thread fork-join, fixed-order reductions.
// ---------------------------------------------------------------------------
inline int& hw_threads_override() {
  static int v = 0;
  return v;
}
inline unsigned hw_threads() {
  const int o = hw_threads_override();
  return o > 0 ? static_cast<unsigned>(o) : std::thread::hardware_concurrency();
}

// parallel.hpp:18-48
inline void parallel_for(int begin, int end, const std::function<void(int)>& fn, int grain = 8) {
  const int count = end - begin;
  if (count <= 0) return;
  const unsigned hw = hw_threads();
  if (hw < 2 || count <= grain) {
    for (int i = begin; i < end; ++i) fn(i);
    return;
  }
  const int workers = std::min<int>(static_cast<int>(hw), (count + grain - 1) / grain);
  std::vector<std::thread> pool;
  pool.reserve(workers);
  std::exception_ptr first_error;
  std::mutex error_mutex;
  const int chunk = (count + workers - 1) / workers;
  for (int w = 0; w < workers; ++w) {
    const int lo = begin + w * chunk;
    const int hi = std::min(end, lo + chunk);
    if (lo >= hi) break;
    pool.emplace_back([lo, hi, &fn, &first_error, &error_mutex] {
      try {
        for (int i = lo; i < hi; ++i) fn(i);
      } catch (...) {
        std::lock_guard<std::mutex> lock(error_mutex);
        if (!first_error) first_error = std::current_exception();
      }
    });
  }
  for (auto& t : pool) t.join();
  if (first_error) std::rethrow_exception(first_error);
}

// parallel.hpp:53-63 — pairwise tree with strides 1, 2, 4, ...
template <class T>
T tree_reduce(std::span<const T> slots) {
  std::vector<T> buf(slots.begin(), slots.end());
  const std::size_t n = buf.size();
  if (n == 0) return T(0);
  for (std::size_t stride = 1; stride < n; stride *= 2)
    for (std::size_t i = 0; i + stride < n; i += 2 * stride) buf[i] += buf[i + stride];
  return buf[0];
}

// parallel.hpp:67-71
template <class T>
T linear_reduce(std::span<const T> slots) {
  T acc = T(0);
  for (T v : slots) acc += v;
  return acc;
}

// ---------------------------------------------------------------------------
// Minimal dense containers (row-major). Eigen MatrixXd is column-major in the
// reference, but element values do not depend on storage order.
// ---------------------------------------------------------------------------
template <class T>
struct Mat {
  int rows = 0, cols = 0;
  std::vector<T> a;
  Mat() = default;
  Mat(int r, int c) : rows(r), cols(c), a(static_cast<std::size_t>(r) * c, T(0)) {}
  T& operator()(int i, int j) { return a[static_cast<std::size_t>(i) * cols + j]; }
  T operator()(int i, int j) const { return a[static_cast<std::size_t>(i) * cols + j]; }
  static Mat identity(int n) {
    Mat m(n, n);
    for (int i = 0; i < n; ++i) m(i, i) = T(1);
    return m;
  }
};
template <class T>
using Vec = std::vector<T>;

template <class T>
Mat<T> matmul(const Mat<T>& A, const Mat<T>& B) {
  Mat<T> C(A.rows, B.cols);
  for (int i = 0; i < A.rows; ++i)
    for (int j = 0; j < B.cols; ++j) {
      T s = T(0);
      for (int p = 0; p < A.cols; ++p) s += A(i, p) * B(p, j);
      C(i, j) = s;
    }
  return C;
}
template <class T>
Mat<T> transpose(const Mat<T>& A) {
  Mat<T> B(A.cols, A.rows);
  for (int i = 0; i < A.rows; ++i)
    for (int j = 0; j < A.cols; ++j) B(j, i) = A(i, j);
  return B;
}
template <class T>
Mat<T> add(const Mat<T>& A, const Mat<T>& B) {
  Mat<T> C(A.rows, A.cols);
  for (std::size_t i = 0; i < C.a.size(); ++i) C.a[i] = A.a[i] + B.a[i];
  return C;
}
template <class T>
Mat<T> scale(const Mat<T>& A, T s) {
  Mat<T> C(A.rows, A.cols);
  for (std::size_t i = 0; i < C.a.size(); ++i) C.a[i] = s * A.a[i];
  return C;
}
template <class T>
Mat<T> neg(const Mat<T>& A) {
  Mat<T> C(A.rows, A.cols);
  for (std::size_t i = 0; i < C.a.size(); ++i) C.a[i] = -A.a[i];
  return C;
}
// 0.5 * (X + X') — schur.cpp:22, :56, :67.
template <class T>
Mat<T> symmetrize(const Mat<T>& X) {
  Mat<T> C(X.rows, X.cols);
  for (int i = 0; i < X.rows; ++i)
    for (int j = 0; j < X.cols; ++j) C(i, j) = T(0.5) * (X(i, j) + X(j, i));
  return C;
}
template <class T>
Vec<T> matvec(const Mat<T>& A, const T* x) {
  Vec<T> y(A.rows);
  for (int i = 0; i < A.rows; ++i) {
    T s = T(0);
    for (int j = 0; j < A.cols; ++j) s += A(i, j) * x[j];
    y[i] = s;
  }
  return y;
}
template <class T>
T dot(const Vec<T>& a, const Vec<T>& b) {
  T s = T(0);
  for (std::size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
template <class T>
T norm2(const Vec<T>& a) {
  return std::sqrt(dot(a, a));
}

// Lower Cholesky in the left-looking order of Eigen's llt_inplace::unblocked
// (Eigen/src/Cholesky/LLT.h; used for sizes < 32 by the blocked driver):
// x = A(k,k) - ||L(k,0:k)||^2; fail iff x <= 0 (a NaN pivot does not fail,
// exactly as in Eigen); L(k+1:,k) = (A(k+1:,k) - L(k+1:,0:k) L(k,0:k)') / L(k,k).
// Only the lower triangle of A is read. Returns -1 on success else the pivot.
template <class T>
int cholesky_lower(const Mat<T>& A, Mat<T>& L) {
  const int n = A.rows;
  L = Mat<T>(n, n);
  for (int k = 0; k < n; ++k) {
    T x = A(k, k);
    for (int p = 0; p < k; ++p) x -= L(k, p) * L(k, p);
    if (x <= T(0)) return k;
    x = std::sqrt(x);
    L(k, k) = x;
    for (int i = k + 1; i < n; ++i) {
      T s = A(i, k);
      for (int p = 0; p < k; ++p) s -= L(i, p) * L(k, p);
      L(i, k) = s / x;
    }
  }
  return -1;
}

// L L' X = B, column by column (LLT::solve).
template <class T>
Mat<T> llt_solve(const Mat<T>& L, const Mat<T>& B) {
  const int n = L.rows;
  Mat<T> X(n, B.cols);
  std::vector<T> y(n);
  for (int c = 0; c < B.cols; ++c) {
    for (int i = 0; i < n; ++i) {
      T s = B(i, c);
      for (int p = 0; p < i; ++p) s -= L(i, p) * y[p];
      y[i] = s / L(i, i);
    }
    for (int i = n - 1; i >= 0; --i) {
      T s = y[i];
      for (int p = i + 1; p < n; ++p) s -= L(p, i) * X(p, c);
      X(i, c) = s / L(i, i);
    }
  }
  return X;
}

// ---------------------------------------------------------------------------
// block_tri.hpp:18-75 / block_tri.cpp — [K][left|diag|right][nb][nb] row-major.
// ---------------------------------------------------------------------------
template <class T>
class BlockTri {
 public:
  BlockTri() = default;
  // block_tri.cpp:11-17
  BlockTri(int rows, int nb) : K_(rows), nb_(nb) {
    if (rows < 1 || nb < 1)
      throw std::invalid_argument("BlockTriMatrix: need at least one block row and block_dim >= 1");
    data_.assign(static_cast<std::size_t>(K_) * 3 * nb_ * nb_, T(0));
  }
  int block_rows() const { return K_; }
  int block_dim() const { return nb_; }
  int dim() const { return K_ * nb_; }
  bool empty() const { return K_ == 0; }
  const T* block(int row, int slot) const {
    return data_.data() + (static_cast<std::size_t>(row) * 3 + slot) * nb_ * nb_;
  }
  T* block_mut(int row, int slot) {
    return data_.data() + (static_cast<std::size_t>(row) * 3 + slot) * nb_ * nb_;
  }
  Mat<T> get(int row, int slot) const {
    Mat<T> m(nb_, nb_);
    std::copy(block(row, slot), block(row, slot) + nb_ * nb_, m.a.begin());
    return m;
  }
  Mat<T> left(int row) const { return get(row, 0); }
  Mat<T> diag(int row) const { return get(row, 1); }
  Mat<T> right(int row) const { return get(row, 2); }
  // block_tri.cpp:31-44
  void check_row(int row) const {
    if (row < 0 || row >= K_)
      throw std::invalid_argument("BlockTriMatrix: block row " + std::to_string(row) +
                                  " out of range [0, " + std::to_string(K_) + ")");
  }
  void check_shape(const Mat<T>& b) const {
    if (b.rows != nb_ || b.cols != nb_)
      throw std::invalid_argument("BlockTriMatrix: expected " + std::to_string(nb_) + "x" +
                                  std::to_string(nb_) + " block, got " + std::to_string(b.rows) +
                                  "x" + std::to_string(b.cols));
  }
  // block_tri.cpp:46-67
  void set_left(int row, const Mat<T>& b) {
    check_row(row);
    check_shape(b);
    if (row == 0)
      throw std::invalid_argument("BlockTriMatrix: row 0 has no left block (boundary padding)");
    std::copy(b.a.begin(), b.a.end(), block_mut(row, 0));
  }
  void set_diag(int row, const Mat<T>& b) {
    check_row(row);
    check_shape(b);
    std::copy(b.a.begin(), b.a.end(), block_mut(row, 1));
  }
  void set_right(int row, const Mat<T>& b) {
    check_row(row);
    check_shape(b);
    if (row == K_ - 1)
      throw std::invalid_argument("BlockTriMatrix: last row has no right block (boundary padding)");
    std::copy(b.a.begin(), b.a.end(), block_mut(row, 2));
  }
  // block_tri.cpp:70-80
  Vec<T> matvec(const Vec<T>& x) const {
    if (static_cast<int>(x.size()) != dim())
      throw std::invalid_argument("BlockTriMatrix matvec: expected vector of length " +
                                  std::to_string(dim()) + ", got " + std::to_string(x.size()));
    Vec<T> y(dim());
    for (int row = 0; row < K_; ++row) matvec_block(row, x.data(), y.data() + row * nb_);
    return y;
  }
  // block_tri.cpp:82-92 — y_b = D_b x_b (+ L_b x_{b-1}) (+ R_b x_{b+1}).
  void matvec_block(int row, const T* x, T* y) const {
    const int n = nb_;
    const T* D = block(row, 1);
    for (int i = 0; i < n; ++i) {
      T s = T(0);
      for (int j = 0; j < n; ++j) s += D[i * n + j] * x[row * n + j];
      y[i] = s;
    }
    if (row > 0) {
      const T* L = block(row, 0);
      for (int i = 0; i < n; ++i) {
        T s = T(0);
        for (int j = 0; j < n; ++j) s += L[i * n + j] * x[(row - 1) * n + j];
        y[i] += s;
      }
    }
    if (row + 1 < K_) {
      const T* R = block(row, 2);
      for (int i = 0; i < n; ++i) {
        T s = T(0);
        for (int j = 0; j < n; ++j) s += R[i * n + j] * x[(row + 1) * n + j];
        y[i] += s;
      }
    }
  }
  // block_tri.cpp:161-165
  T max_abs() const {
    T w = T(0);
    for (T v : data_) w = std::max(w, std::abs(v));
    return w;
  }
  // block_tri.cpp:167-177
  T max_asymmetry() const {
    T w = T(0);
    const int n = nb_;
    for (int row = 0; row < K_; ++row) {
      const T* D = block(row, 1);
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) w = std::max(w, std::abs(D[i * n + j] - D[j * n + i]));
      if (row + 1 < K_) {
        const T* R = block(row, 2);
        const T* L = block(row + 1, 0);
        for (int i = 0; i < n; ++i)
          for (int j = 0; j < n; ++j) w = std::max(w, std::abs(R[i * n + j] - L[j * n + i]));
      }
    }
    return w;
  }
  // block_tri.cpp:121-159 — block Thomas / block Cholesky direct solve.
  Vec<T> cholesky_solve(const Vec<T>& rhs) const {
    if (static_cast<int>(rhs.size()) != dim())
      throw std::invalid_argument("BlockTriMatrix cholesky_solve: expected vector of length " +
                                  std::to_string(dim()) + ", got " + std::to_string(rhs.size()));
    const int n = nb_;
    std::vector<Mat<T>> factors;
    factors.reserve(K_);
    Vec<T> y = rhs;
    Mat<T> Lf;
    if (cholesky_lower(diag(0), Lf) >= 0)
      throw std::runtime_error("BlockTriMatrix cholesky_solve: block 0 is not positive definite");
    factors.push_back(Lf);
    for (int i = 1; i < K_; ++i) {
      const Mat<T> li = left(i);
      const Mat<T> solved = llt_solve(factors[i - 1], transpose(li));
      const Mat<T> dhat = add(diag(i), neg(matmul(li, solved)));
      if (cholesky_lower(dhat, Lf) >= 0)
        throw std::runtime_error("BlockTriMatrix cholesky_solve: block " + std::to_string(i) +
                                 " is not positive definite");
      factors.push_back(Lf);
      Mat<T> yprev(n, 1);
      for (int j = 0; j < n; ++j) yprev(j, 0) = y[(i - 1) * n + j];
      const Mat<T> s = llt_solve(factors[i - 1], yprev);
      const Vec<T> ls = oracle::matvec(li, s.a.data());
      for (int j = 0; j < n; ++j) y[i * n + j] -= ls[j];
    }
    Vec<T> x(dim());
    {
      Mat<T> yl(n, 1);
      for (int j = 0; j < n; ++j) yl(j, 0) = y[(K_ - 1) * n + j];
      const Mat<T> s = llt_solve(factors.back(), yl);
      for (int j = 0; j < n; ++j) x[(K_ - 1) * n + j] = s.a[j];
    }
    for (int i = K_ - 2; i >= 0; --i) {
      const Vec<T> rx = oracle::matvec(right(i), x.data() + (i + 1) * n);
      Mat<T> adj(n, 1);
      for (int j = 0; j < n; ++j) adj(j, 0) = y[i * n + j] - rx[j];
      const Mat<T> s = llt_solve(factors[i], adj);
      for (int j = 0; j < n; ++j) x[i * n + j] = s.a[j];
    }
    return x;
  }
  std::vector<T>& raw() { return data_; }
  const std::vector<T>& raw() const { return data_; }

  bool structurally_symmetric = false;  // block_tri.hpp:63-64

 private:
  int K_ = 0, nb_ = 0;
  std::vector<T> data_;
};

// ---------------------------------------------------------------------------
// kkt.hpp:13-46, kkt.cpp:32-39
// ---------------------------------------------------------------------------
template <class T>
struct KnotData {
  Mat<T> Q, R, A, B;
  Vec<T> q, r, e;
};
template <class T>
struct KKTSystem {
  int N = 0, n = 0, m = 0;
  std::vector<KnotData<T>> knots;  // N+1
  Vec<T> x_s, x0;
  int dual_dim() const { return (N + 1) * n; }
  // kkt.cpp:32-39 — c_0 = x_s - x_0, c_{k+1} = -e_k
  Vec<T> constraint_rhs() const {
    Vec<T> c(dual_dim());
    for (int i = 0; i < n; ++i) c[i] = x_s[i] - x0[i];
    for (int k = 0; k < N; ++k)
      for (int i = 0; i < n; ++i) c[(k + 1) * n + i] = -knots[k].e[i];
    return c;
  }
};

// ---------------------------------------------------------------------------
// random_problem.hpp:13-37, random_problem.cpp:10-80 — always generated in
// double (the reference is double-only); cast afterwards for f32 runs.
// ---------------------------------------------------------------------------
class UniformRng {
 public:
  explicit UniformRng(std::uint64_t seed) : gen_(seed) {}
  // random_problem.hpp:17-20
  double uniform(double lo, double hi) {
    const double u01 = static_cast<double>(gen_() >> 11) * 0x1.0p-53;
    return lo + (hi - lo) * u01;
  }
  // random_problem.hpp:22-27 — row-major draw order
  Mat<double> matrix(int rows, int cols, double lo, double hi) {
    Mat<double> M(rows, cols);
    for (int i = 0; i < rows; ++i)
      for (int j = 0; j < cols; ++j) M(i, j) = uniform(lo, hi);
    return M;
  }
  Vec<double> vector(int size, double lo, double hi) {
    Vec<double> v(size);
    for (int i = 0; i < size; ++i) v[i] = uniform(lo, hi);
    return v;
  }

 private:
  std::mt19937_64 gen_;
};

// L L' + floor*I, evaluated entrywise in p-order.
inline Mat<double> llt_plus(const Mat<double>& L, double floor_) {
  Mat<double> Q = matmul(L, transpose(L));
  for (int i = 0; i < Q.rows; ++i) Q(i, i) += floor_;
  return Q;
}

// random_problem.cpp:10-38
inline KKTSystem<double> generate(std::uint64_t seed, int N, int n, int m, double diag_floor,
                                  double coupling) {
  UniformRng rng(seed);
  KKTSystem<double> kkt;
  kkt.N = N;
  kkt.n = n;
  kkt.m = m;
  kkt.knots.resize(N + 1);
  for (int k = 0; k < N; ++k) {
    KnotData<double>& kd = kkt.knots[k];
    const Mat<double> L = rng.matrix(n, n, -1.0, 1.0);
    kd.Q = llt_plus(L, diag_floor);
    const Mat<double> Lr = rng.matrix(m, m, -1.0, 1.0);
    kd.R = llt_plus(Lr, diag_floor);
    kd.A = scale(rng.matrix(n, n, -1.0, 1.0), coupling / n);
    kd.B = scale(rng.matrix(n, m, -1.0, 1.0), coupling / n);
    kd.q = rng.vector(n, -1.0, 1.0);
    kd.r = rng.vector(m, -1.0, 1.0);
    kd.e = rng.vector(n, -1.0, 1.0);
  }
  const Mat<double> Ln = rng.matrix(n, n, -1.0, 1.0);
  kkt.knots[N].Q = llt_plus(Ln, diag_floor);
  kkt.knots[N].q = rng.vector(n, -1.0, 1.0);
  kkt.x_s = rng.vector(n, -1.0, 1.0);
  kkt.x0 = Vec<double>(n, 0.0);
  return kkt;
}
// random_problem.cpp:42-49
inline KKTSystem<double> random_kkt(std::uint64_t seed, int N, int n, int m) {
  return generate(seed, N, n, m, 0.1, 1.0);
}
inline KKTSystem<double> random_kkt_scaled(std::uint64_t seed, int N, int n, int m,
                                           double diag_floor, double coupling) {
  return generate(seed, N, n, m, diag_floor, coupling);
}
// random_problem.cpp:51-80
inline KKTSystem<double> random_trajectory_kkt(std::uint64_t seed, int N, int n, int m) {
  constexpr double kCostScale = 2e-4;
  UniformRng rng(seed);
  KKTSystem<double> kkt;
  kkt.N = N;
  kkt.n = n;
  kkt.m = m;
  kkt.knots.resize(N + 1);
  for (int k = 0; k < N; ++k) {
    KnotData<double>& kd = kkt.knots[k];
    const Mat<double> L = rng.matrix(n, n, -1.0, 1.0);
    kd.Q = scale(add(scale(matmul(L, transpose(L)), 0.3), Mat<double>::identity(n)), kCostScale);
    const Mat<double> Lr = rng.matrix(m, m, -1.0, 1.0);
    kd.R = scale(add(scale(matmul(Lr, transpose(Lr)), 0.3), Mat<double>::identity(m)), kCostScale);
    kd.A = add(scale(Mat<double>::identity(n), 0.1), scale(rng.matrix(n, n, -1.0, 1.0), 0.02 / n));
    kd.B = scale(rng.matrix(n, m, -1.0, 1.0), 1.0 / n);
    kd.q = rng.vector(n, -1.0, 1.0);
    kd.r = rng.vector(m, -1.0, 1.0);
    kd.e = rng.vector(n, -1.0, 1.0);
  }
  const Mat<double> Ln = rng.matrix(n, n, -1.0, 1.0);
  kkt.knots[N].Q =
      scale(add(scale(matmul(Ln, transpose(Ln)), 0.3), Mat<double>::identity(n)), kCostScale);
  kkt.knots[N].q = rng.vector(n, -1.0, 1.0);
  kkt.x_s = rng.vector(n, -1.0, 1.0);
  kkt.x0 = Vec<double>(n, 0.0);
  return kkt;
}

// ---------------------------------------------------------------------------
// schur.hpp:19-56, schur.cpp
// ---------------------------------------------------------------------------
enum class PrecondKind { identity = 0, block_jacobi = 1, stair = 2, symmetric_stair = 3, poly_split = 4 };

// schur.cpp:27-36
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

template <class T>
struct SchurSystem {
  BlockTri<T> S;
  Vec<T> gamma;
  std::vector<Mat<T>> theta_inv;
  int n = 0;
};

template <class T>
struct Preconditioner {
  PrecondKind kind = PrecondKind::identity;
  int order = 0;
  BlockTri<T> phi_inv;
  BlockTri<T> stair_psi;
  BlockTri<T> remainder;
};

// schur.cpp:15-23 — LLT, solve against I, symmetrise; non-PD message.
template <class T>
Mat<T> spd_inverse(const Mat<T>& W, int knot, const char* what) {
  Mat<T> L;
  if (cholesky_lower(W, L) >= 0)
    throw std::runtime_error(std::string("build_schur: ") + what + " at knot " +
                             std::to_string(knot) + " is not positive definite");
  return symmetrize(llt_solve(L, Mat<T>::identity(W.rows)));
}

// schur.cpp:38-82
template <class T>
SchurSystem<T> build_schur(const KKTSystem<T>& kkt) {
  const int N = kkt.N;
  const int n = kkt.n;
  const Vec<T> c = kkt.constraint_rhs();
  SchurSystem<T> out;
  out.n = n;
  out.S = BlockTri<T>(N + 1, n);
  out.gamma.assign(static_cast<std::size_t>(N + 1) * n, T(0));
  out.theta_inv.resize(N + 1);
  parallel_for(0, N + 1, [&](int b) {
    if (b == 0) {
      const Mat<T> q0_inv = spd_inverse(kkt.knots[0].Q, 0, "Q");
      out.S.set_diag(0, q0_inv);
      out.theta_inv[0] = symmetrize(kkt.knots[0].Q);
      const Vec<T> t = matvec(q0_inv, kkt.knots[0].q.data());
      for (int i = 0; i < n; ++i) out.gamma[i] = -(c[i] + t[i]);
    } else {
      const int k = b - 1;
      const KnotData<T>& kd = kkt.knots[k];
      const Mat<T> qk_inv = spd_inverse(kd.Q, k, "Q");
      const Mat<T> rk_inv = spd_inverse(kd.R, k, "R");
      const Mat<T> qk1_inv = spd_inverse(kkt.knots[k + 1].Q, k + 1, "Q");
      // schur.cpp:65-66 — (A Qk^-1) A' + (B Rk^-1) B' + Qk1^-1
      const Mat<T> AQ = matmul(kd.A, qk_inv);
      const Mat<T> BR = matmul(kd.B, rk_inv);
      const Mat<T> theta_raw =
          add(add(matmul(AQ, transpose(kd.A)), matmul(BR, transpose(kd.B))), qk1_inv);
      const Mat<T> theta = symmetrize(theta_raw);
      const Mat<T> phi = matmul(neg(kd.A), qk_inv);  // schur.cpp:68
      // schur.cpp:69-70 — zeta = -A (Qk^-1 q) - B (Rk^-1 r) + Qk1^-1 q_{k+1}
      const Vec<T> qq = matvec(qk_inv, kd.q.data());
      const Vec<T> rr = matvec(rk_inv, kd.r.data());
      const Vec<T> aq = matvec(kd.A, qq.data());
      const Vec<T> br = matvec(kd.B, rr.data());
      const Vec<T> q1 = matvec(qk1_inv, kkt.knots[k + 1].q.data());
      out.S.set_diag(b, theta);
      out.S.set_left(b, phi);
      out.S.set_right(b - 1, transpose(phi));
      out.theta_inv[b] = spd_inverse(theta, k, "theta");
      for (int i = 0; i < n; ++i) {
        const T zeta = -aq[i] - br[i] + q1[i];
        out.gamma[b * n + i] = -(c[b * n + i] + zeta);
      }
    }
  });
  out.S.structurally_symmetric = true;
  return out;
}

// schur.cpp:84-94
template <class T>
BlockTri<T> stair_matrix(const BlockTri<T>& S) {
  BlockTri<T> psi(S.block_rows(), S.block_dim());
  for (int row = 0; row < S.block_rows(); ++row) {
    psi.set_diag(row, S.diag(row));
    if (row % 2 == 1) {
      psi.set_left(row, S.left(row));
      if (row + 1 < S.block_rows()) psi.set_right(row, S.right(row));
    }
  }
  return psi;
}

template <class T>
Preconditioner<T> build_identity() {  // schur.cpp:96
  return Preconditioner<T>{};
}

// schur.cpp:98-107
template <class T>
Preconditioner<T> build_block_jacobi(const SchurSystem<T>& s) {
  Preconditioner<T> P;
  P.kind = PrecondKind::block_jacobi;
  P.phi_inv = BlockTri<T>(s.S.block_rows(), s.n);
  for (int row = 0; row < s.S.block_rows(); ++row) P.phi_inv.set_diag(row, s.theta_inv[row]);
  P.phi_inv.structurally_symmetric = true;
  return P;
}

// schur.cpp:109-127 — odd rows: (-theta_i^-1 L_i) theta_{i-1}^-1, ...
template <class T>
Preconditioner<T> build_stair(const SchurSystem<T>& s) {
  Preconditioner<T> P;
  P.kind = PrecondKind::stair;
  const int rows = s.S.block_rows();
  P.phi_inv = BlockTri<T>(rows, s.n);
  parallel_for(0, rows, [&](int row) {
    P.phi_inv.set_diag(row, s.theta_inv[row]);
    if (row % 2 == 1) {
      P.phi_inv.set_left(row,
                         matmul(matmul(neg(s.theta_inv[row]), s.S.left(row)), s.theta_inv[row - 1]));
      if (row + 1 < rows)
        P.phi_inv.set_right(
            row, matmul(matmul(neg(s.theta_inv[row]), s.S.right(row)), s.theta_inv[row + 1]));
    }
  });
  return P;
}

// schur.cpp:129-142
template <class T>
Preconditioner<T> build_symmetric_stair(const SchurSystem<T>& s) {
  Preconditioner<T> P = build_stair(s);
  P.kind = PrecondKind::symmetric_stair;
  const int rows = P.phi_inv.block_rows();
  for (int row = 1; row < rows; row += 2) {
    P.phi_inv.set_right(row - 1, transpose(P.phi_inv.left(row)));
    if (row + 1 < rows) P.phi_inv.set_left(row + 1, transpose(P.phi_inv.right(row)));
  }
  P.phi_inv.structurally_symmetric = true;
  return P;
}

// schur.cpp:144-162
template <class T>
Preconditioner<T> build_poly_split(const SchurSystem<T>& s, int order) {
  if (order < 1)
    throw std::invalid_argument("build_poly_split: order must be >= 1, got " +
                                std::to_string(order));
  Preconditioner<T> P = build_stair(s);
  P.kind = PrecondKind::poly_split;
  P.order = order;
  P.stair_psi = stair_matrix(s.S);
  const int rows = s.S.block_rows();
  P.remainder = BlockTri<T>(rows, s.n);
  for (int row = 0; row < rows; row += 2) {
    if (row > 0) P.remainder.set_left(row, neg(s.S.left(row)));
    if (row + 1 < rows) P.remainder.set_right(row, neg(s.S.right(row)));
  }
  return P;
}

// schur.cpp:164-173
template <class T>
Preconditioner<T> build_preconditioner(const SchurSystem<T>& s, PrecondKind kind, int order = 1) {
  switch (kind) {
    case PrecondKind::identity: return build_identity<T>();
    case PrecondKind::block_jacobi: return build_block_jacobi(s);
    case PrecondKind::stair: return build_stair(s);
    case PrecondKind::symmetric_stair: return build_symmetric_stair(s);
    case PrecondKind::poly_split: return build_poly_split(s, order);
  }
  throw std::invalid_argument("build_preconditioner: unknown kind");
}

// schur.cpp:175-194
template <class T>
Vec<T> apply_preconditioner(const Preconditioner<T>& P, const Vec<T>& r) {
  if (P.kind == PrecondKind::identity) return r;
  if (static_cast<int>(r.size()) != P.phi_inv.dim())
    throw std::invalid_argument("apply_preconditioner: expected vector of length " +
                                std::to_string(P.phi_inv.dim()) + ", got " +
                                std::to_string(r.size()));
  if (P.kind != PrecondKind::poly_split) return P.phi_inv.matvec(r);
  Vec<T> term = P.phi_inv.matvec(r);
  Vec<T> acc = term;
  for (int j = 0; j < P.order; ++j) {
    term = P.phi_inv.matvec(P.remainder.matvec(term));
    for (std::size_t i = 0; i < acc.size(); ++i) acc[i] += term[i];
  }
  return acc;
}

// ---------------------------------------------------------------------------
// pcg.hpp:12-70, pcg.cpp
// ---------------------------------------------------------------------------
enum class PcgVariant { sequential = 0, block_parallel = 1 };

struct PcgConfig {  // pcg.hpp:14-29 (field order preserved)
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

template <class T>
struct PcgResult {
  Vec<T> lambda;
  SolveReport report;
};

class PcgBreakdown : public std::runtime_error {  // pcg.hpp:47-50
 public:
  using std::runtime_error::runtime_error;
};

using Clock = std::chrono::steady_clock;
inline double seconds_since(Clock::time_point start) {
  return std::chrono::duration<double>(Clock::now() - start).count();
}

// pcg.cpp:24-47
template <class T>
void validate_inputs(const BlockTri<T>& S, const Preconditioner<T>& P, const Vec<T>& gamma,
                     const Vec<T>& lambda0) {
  if (S.empty()) throw std::invalid_argument("pcg: empty system matrix");
  if (static_cast<int>(gamma.size()) != S.dim())
    throw std::invalid_argument("pcg: expected gamma of length " + std::to_string(S.dim()) +
                                ", got " + std::to_string(gamma.size()));
  if (static_cast<int>(lambda0.size()) != S.dim())
    throw std::invalid_argument("pcg: expected lambda0 of length " + std::to_string(S.dim()) +
                                ", got " + std::to_string(lambda0.size()));
  if (P.kind != PrecondKind::identity && P.phi_inv.dim() != S.dim())
    throw std::invalid_argument("pcg: preconditioner dimension " +
                                std::to_string(P.phi_inv.dim()) + " does not match system " +
                                std::to_string(S.dim()));
  const double asym_tol = 1e-9 * std::max(1.0, static_cast<double>(S.max_abs()));
  if (S.max_asymmetry() > asym_tol)
    throw std::invalid_argument("pcg: S is not structurally symmetric (asymmetry " +
                                std::to_string(static_cast<double>(S.max_asymmetry())) + ")");
}

// pcg.cpp:49-51
template <class T>
int resolve_max_iter(const PcgConfig& cfg, const BlockTri<T>& S) {
  return cfg.max_iter > 0 ? cfg.max_iter : S.dim();
}

// pcg.cpp:55-129 — Alg. 1
template <class T>
PcgResult<T> pcg_solve(const BlockTri<T>& S, const Preconditioner<T>& P, const Vec<T>& gamma,
                       const Vec<T>& lambda0, const PcgConfig& cfg) {
  validate_inputs(S, P, gamma, lambda0);
  const auto start = Clock::now();
  const int max_iter = resolve_max_iter(cfg, S);
  const std::size_t D = static_cast<std::size_t>(S.dim());
  Vec<T> lambda = lambda0;
  Vec<T> r(D);
  {
    const Vec<T> sl = S.matvec(lambda);
    for (std::size_t i = 0; i < D; ++i) r[i] = gamma[i] - sl[i];
  }
  Vec<T> r_tilde = apply_preconditioner(P, r);
  Vec<T> p = r_tilde;
  T eta = dot(r, r_tilde);
  if (!std::isfinite(eta)) throw std::runtime_error("pcg: non-finite initial residual");
  SolveReport rep;
  rep.exit_eta = static_cast<double>(eta);
  if (static_cast<double>(eta) < cfg.epsilon) {
    rep.converged = true;
    rep.wall_time = seconds_since(start);
    return {std::move(lambda), std::move(rep)};
  }
  T best_eta = eta;
  Vec<T> best_lambda = lambda;
  for (int i = 1; i <= max_iter; ++i) {
    const Vec<T> Sp = S.matvec(p);
    const T upsilon = dot(p, Sp);
    if (!std::isfinite(upsilon))
      throw std::runtime_error("pcg: non-finite p'Sp at iteration " + std::to_string(i));
    if (upsilon <= T(0))
      throw PcgBreakdown("pcg: p'Sp = " + std::to_string(static_cast<double>(upsilon)) +
                         " at iteration " + std::to_string(i) +
                         "; S is not positive definite on the search space");
    const T alpha = eta / upsilon;
    for (std::size_t k = 0; k < D; ++k) r[k] -= alpha * Sp[k];
    for (std::size_t k = 0; k < D; ++k) lambda[k] += alpha * p[k];
    r_tilde = apply_preconditioner(P, r);
    const T eta_prime = dot(r, r_tilde);
    if (!std::isfinite(eta_prime))
      throw std::runtime_error("pcg: non-finite iterate at iteration " + std::to_string(i));
    if (cfg.collect_trace) rep.trace.push_back(static_cast<double>(eta_prime));
    if (cfg.check_residual_drift) {  // pcg.cpp:103-108
      const Vec<T> sl = S.matvec(lambda);
      Vec<T> tr(D);
      for (std::size_t k = 0; k < D; ++k) tr[k] = gamma[k] - sl[k];
      const double true_norm = static_cast<double>(norm2(tr));
      const double drift = std::abs(static_cast<double>(norm2(r)) - true_norm) /
                           std::max(true_norm, std::numeric_limits<double>::min());
      rep.max_residual_drift = std::max(rep.max_residual_drift, drift);
    }
    if (eta_prime < best_eta) {
      best_eta = eta_prime;
      best_lambda = lambda;
    }
    rep.iterations = i;
    rep.exit_eta = static_cast<double>(eta_prime);
    if (static_cast<double>(eta_prime) < cfg.epsilon) {
      rep.converged = true;
      rep.wall_time = seconds_since(start);
      return {std::move(lambda), std::move(rep)};
    }
    const T beta = eta_prime / eta;
    for (std::size_t k = 0; k < D; ++k) p[k] = r_tilde[k] + beta * p[k];
    eta = eta_prime;
  }
  rep.converged = false;
  rep.wall_time = seconds_since(start);
  return {std::move(best_lambda), std::move(rep)};
}

// pcg.cpp:157-362 — Alg. 2 analog: std::thread workers, one-block halo,
// barrier-separated scalar reductions (6 barriers per iteration).
template <class T>
PcgResult<T> pcg_solve_block_parallel(const BlockTri<T>& S, const Preconditioner<T>& P,
                                      const Vec<T>& gamma, const Vec<T>& lambda0,
                                      const PcgConfig& cfg) {
  validate_inputs(S, P, gamma, lambda0);
  const auto start = Clock::now();
  const int max_iter = resolve_max_iter(cfg, S);
  const int blocks = S.block_rows();
  const int nb = S.block_dim();
  const std::size_t D = static_cast<std::size_t>(S.dim());
  int workers = static_cast<int>(hw_threads());
  workers = std::max(1, std::min(workers, blocks));

  struct State {
    Vec<T> lambda, r, r_tilde, p, Sp, term, scratch, best_lambda;
    std::vector<T> slots;
    T eta = 0, eta_prime = 0, upsilon = 0, alpha = 0, beta = 0;
    T best_eta = std::numeric_limits<T>::infinity();
    bool done = false, converged = false, breakdown = false, nonfinite = false;
    int iterations = 0;
    double exit_eta = 0;
    std::string error;
    std::vector<double> trace;
  } st;
  st.lambda = lambda0;
  st.r.assign(D, T(0));
  st.r_tilde.assign(D, T(0));
  st.p.assign(D, T(0));
  st.Sp.assign(D, T(0));
  st.slots.assign(blocks, T(0));
  const bool poly = (P.kind == PrecondKind::poly_split);
  if (poly) {
    st.term.assign(D, T(0));
    st.scratch.assign(D, T(0));
  }
  std::barrier sync(workers);
  auto reduce_slots = [&]() {
    return cfg.deterministic_reductions ? tree_reduce<T>(st.slots) : linear_reduce<T>(st.slots);
  };
  auto dotb = [&](const Vec<T>& a, const Vec<T>& b, int blk) {
    T s = T(0);
    for (int j = 0; j < nb; ++j) s += a[blk * nb + j] * b[blk * nb + j];
    return s;
  };
  // pcg.cpp:188-221
  auto apply_precond_blocks = [&](int blo, int bhi) {
    if (P.kind == PrecondKind::identity) {
      for (int b = blo; b < bhi; ++b)
        for (int j = 0; j < nb; ++j) st.r_tilde[b * nb + j] = st.r[b * nb + j];
      return;
    }
    if (!poly) {
      for (int b = blo; b < bhi; ++b) P.phi_inv.matvec_block(b, st.r.data(), st.r_tilde.data() + b * nb);
      return;
    }
    for (int b = blo; b < bhi; ++b) {
      P.phi_inv.matvec_block(b, st.r.data(), st.term.data() + b * nb);
      for (int j = 0; j < nb; ++j) st.r_tilde[b * nb + j] = st.term[b * nb + j];
    }
    for (int j = 0; j < P.order; ++j) {
      sync.arrive_and_wait();
      for (int b = blo; b < bhi; ++b)
        P.remainder.matvec_block(b, st.term.data(), st.scratch.data() + b * nb);
      sync.arrive_and_wait();
      for (int b = blo; b < bhi; ++b) {
        Vec<T> next(nb);
        P.phi_inv.matvec_block(b, st.scratch.data(), next.data());
        for (int q = 0; q < nb; ++q) {
          st.term[b * nb + q] = next[q];
          st.r_tilde[b * nb + q] += next[q];
        }
      }
    }
  };
  auto worker = [&](int w) {
    const int chunk = (blocks + workers - 1) / workers;
    const int blo = w * chunk;
    const int bhi = std::min(blocks, blo + chunk);
    for (int b = blo; b < bhi; ++b) {
      Vec<T> sx(nb);
      S.matvec_block(b, st.lambda.data(), sx.data());
      for (int j = 0; j < nb; ++j) st.r[b * nb + j] = gamma[b * nb + j] - sx[j];
    }
    sync.arrive_and_wait();
    apply_precond_blocks(blo, bhi);
    for (int b = blo; b < bhi; ++b) {
      for (int j = 0; j < nb; ++j) st.p[b * nb + j] = st.r_tilde[b * nb + j];
      st.slots[b] = dotb(st.r, st.r_tilde, b);
    }
    sync.arrive_and_wait();
    if (w == 0) {
      st.eta = reduce_slots();
      st.exit_eta = static_cast<double>(st.eta);
      if (!std::isfinite(st.eta)) {
        st.nonfinite = true;
        st.error = "pcg: non-finite initial residual";
        st.done = true;
      } else if (static_cast<double>(st.eta) < cfg.epsilon) {
        st.converged = true;
        st.done = true;
      }
      st.best_eta = st.eta;
      st.best_lambda = st.lambda;
    }
    sync.arrive_and_wait();
    if (st.done) return;
    for (int i = 1; i <= max_iter; ++i) {
      for (int b = blo; b < bhi; ++b) {
        S.matvec_block(b, st.p.data(), st.Sp.data() + b * nb);
        st.slots[b] = dotb(st.p, st.Sp, b);
      }
      sync.arrive_and_wait();
      if (w == 0) {
        st.upsilon = reduce_slots();
        if (!std::isfinite(st.upsilon)) {
          st.nonfinite = true;
          st.error = "pcg: non-finite p'Sp at iteration " + std::to_string(i);
          st.done = true;
        } else if (st.upsilon <= T(0)) {
          st.breakdown = true;
          st.error = "pcg: p'Sp = " + std::to_string(static_cast<double>(st.upsilon)) +
                     " at iteration " + std::to_string(i) +
                     "; S is not positive definite on the search space";
          st.done = true;
        } else {
          st.alpha = st.eta / st.upsilon;
        }
      }
      sync.arrive_and_wait();
      if (st.done) return;
      for (int b = blo; b < bhi; ++b)
        for (int j = 0; j < nb; ++j) {
          st.lambda[b * nb + j] += st.alpha * st.p[b * nb + j];
          st.r[b * nb + j] -= st.alpha * st.Sp[b * nb + j];
        }
      sync.arrive_and_wait();
      apply_precond_blocks(blo, bhi);
      for (int b = blo; b < bhi; ++b) st.slots[b] = dotb(st.r, st.r_tilde, b);
      sync.arrive_and_wait();
      if (w == 0) {
        st.eta_prime = reduce_slots();
        st.iterations = i;
        st.exit_eta = static_cast<double>(st.eta_prime);
        if (cfg.collect_trace) st.trace.push_back(static_cast<double>(st.eta_prime));
        if (!std::isfinite(st.eta_prime)) {
          st.nonfinite = true;
          st.error = "pcg: non-finite iterate at iteration " + std::to_string(i);
          st.done = true;
        } else {
          if (st.eta_prime < st.best_eta) {
            st.best_eta = st.eta_prime;
            st.best_lambda = st.lambda;
          }
          if (static_cast<double>(st.eta_prime) < cfg.epsilon) {
            st.converged = true;
            st.done = true;
          } else if (i == max_iter) {
            st.done = true;
          } else {
            st.beta = st.eta_prime / st.eta;
            st.eta = st.eta_prime;
          }
        }
      }
      sync.arrive_and_wait();
      if (st.done) return;
      for (int b = blo; b < bhi; ++b)
        for (int j = 0; j < nb; ++j)
          st.p[b * nb + j] = st.r_tilde[b * nb + j] + st.beta * st.p[b * nb + j];
      sync.arrive_and_wait();
    }
  };
  if (workers == 1) {
    worker(0);
  } else {
    std::vector<std::thread> pool;
    pool.reserve(workers);
    for (int w = 0; w < workers; ++w) pool.emplace_back(worker, w);
    for (auto& t : pool) t.join();
  }
  if (st.nonfinite) throw std::runtime_error(st.error);
  if (st.breakdown) throw PcgBreakdown(st.error);
  SolveReport rep;
  rep.iterations = st.iterations;
  rep.exit_eta = st.exit_eta;
  rep.converged = st.converged;
  rep.trace = std::move(st.trace);
  rep.wall_time = seconds_since(start);
  PcgResult<T> out;
  out.lambda = st.converged ? std::move(st.lambda) : std::move(st.best_lambda);
  out.report = std::move(rep);
  return out;
}

// pcg.cpp:364-369
template <class T>
PcgResult<T> pcg_solve_auto(const BlockTri<T>& S, const Preconditioner<T>& P, const Vec<T>& gamma,
                            const Vec<T>& lambda0, const PcgConfig& cfg) {
  return cfg.variant == PcgVariant::block_parallel
             ? pcg_solve_block_parallel(S, P, gamma, lambda0, cfg)
             : pcg_solve(S, P, gamma, lambda0, cfg);
}

// kkt.cpp:153-181 — dz = -G^{-1}(g + C' lambda), blockwise (LDLT solves in the
// reference; an SPD Cholesky solve here).
template <class T>
Vec<T> reconstruct_primal(const KKTSystem<T>& kkt, const Vec<T>& lambda) {
  if (static_cast<int>(lambda.size()) != kkt.dual_dim())
    throw std::invalid_argument("reconstruct_primal: expected lambda of length " +
                                std::to_string(kkt.dual_dim()) + ", got " +
                                std::to_string(lambda.size()));
  const int N = kkt.N, n = kkt.n, m = kkt.m, stride = n + m;
  Vec<T> dz(static_cast<std::size_t>(N + 1) * n + static_cast<std::size_t>(N) * m);
  auto spd_solve = [](const Mat<T>& W, const Vec<T>& b) {
    Mat<T> L;
    cholesky_lower(W, L);
    Mat<T> B(static_cast<int>(b.size()), 1);
    for (std::size_t i = 0; i < b.size(); ++i) B.a[i] = b[i];
    return llt_solve(L, B).a;
  };
  for (int k = 0; k <= N; ++k) {
    const KnotData<T>& kd = kkt.knots[k];
    const T* lam_k = lambda.data() + k * n;
    if (k < N) {
      const T* lam_k1 = lambda.data() + (k + 1) * n;
      Vec<T> bx(n), bu(m);
      for (int i = 0; i < n; ++i) {
        T at = T(0);
        for (int j = 0; j < n; ++j) at += kd.A(j, i) * lam_k1[j];
        bx[i] = -(kd.q[i] + lam_k[i] - at);
      }
      for (int i = 0; i < m; ++i) {
        T bt = T(0);
        for (int j = 0; j < n; ++j) bt += kd.B(j, i) * lam_k1[j];
        bu[i] = -(kd.r[i] - bt);
      }
      const Vec<T> dx = spd_solve(kd.Q, bx);
      const Vec<T> du = spd_solve(kd.R, bu);
      std::copy(dx.begin(), dx.end(), dz.begin() + static_cast<std::size_t>(k) * stride);
      std::copy(du.begin(), du.end(), dz.begin() + static_cast<std::size_t>(k) * stride + n);
    } else {
      Vec<T> bx(n);
      for (int i = 0; i < n; ++i) bx[i] = -(kd.q[i] + lam_k[i]);
      const Vec<T> dx = spd_solve(kd.Q, bx);
      std::copy(dx.begin(), dx.end(), dz.begin() + static_cast<std::size_t>(N) * stride);
    }
  }
  return dz;
}

}  // namespace oracle
