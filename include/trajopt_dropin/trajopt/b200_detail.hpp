// Shared plumbing of the drop-in headers (include/trajopt_dropin/trajopt/):
// the per-(thread, device) b2p context, the status -> exception mapping of the
// reference (invalid_argument / runtime_error / PcgBreakdown, pcg.hpp:47-50)
// and Eigen <-> row-major packing. Not part of the reference's API.
#pragma once

#include <Eigen/Dense>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "b2p.h"

namespace trajopt {

/// pcg.hpp:47-50 — p'Sp <= 0 during CG.
class PcgBreakdown : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

namespace b200 {

inline void raise(int code, const b2p_error& e) {
  if (code == B2P_OK) return;
  const std::string msg(e.message);
  if (code == B2P_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (code == B2P_BREAKDOWN) throw PcgBreakdown(msg);
  throw std::runtime_error(msg);
}

/// One b2p context per (host thread, device), created on first use; the
/// reference's calls are reentrant and so are these.
inline int& device() {
  thread_local int d = 0;
  return d;
}
inline b2p_ctx* context() {
  struct Holder {
    std::map<int, b2p_ctx*> ctxs;
    ~Holder() {
      for (auto& kv : ctxs) b2p_ctx_destroy(kv.second);
    }
  };
  thread_local Holder h;
  const int dev = device();
  auto it = h.ctxs.find(dev);
  if (it != h.ctxs.end()) return it->second;
  b2p_ctx* c = nullptr;
  b2p_error e{};
  raise(b2p_ctx_create(dev, &c, &e), e);
  h.ctxs[dev] = c;
  return c;
}

/// Column-major (or any) Eigen matrix -> row-major doubles appended to `out`.
template <class M>
inline void append_rowmajor(const M& a, std::vector<double>& out) {
  for (Eigen::Index i = 0; i < a.rows(); ++i)
    for (Eigen::Index j = 0; j < a.cols(); ++j) out.push_back(a(i, j));
}
template <class V>
inline void append_vec(const V& v, std::vector<double>& out) {
  for (Eigen::Index i = 0; i < v.size(); ++i) out.push_back(v[i]);
}

}  // namespace b200
}  // namespace trajopt
