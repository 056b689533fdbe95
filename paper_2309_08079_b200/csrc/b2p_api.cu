// Host side of the C-ABI (include/b2p.h): contexts, validation with the
// reference's messages, device workspaces, launch configuration and the
// batched / multi-GPU drivers. No CPU fallback: every compute entry point
// runs on the device or fails with B2P_CUDA_ERROR.
#include <cuda_runtime.h>
#include <immintrin.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <condition_variable>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "../../include/b2p.h"
#include "kernels.h"

using namespace b2p;

// Persistent host worker pool (the packed batch upload): run(n, f) splits
// [0, n) over the workers and the calling thread and returns when all ranges
// are done.
struct HostPool {
  std::vector<std::thread> th;
  std::mutex mu;
  std::condition_variable cv, done_cv;
  std::function<void(size_t, size_t)> fn;
  size_t n = 0;
  int T = 1, pending = 0;
  unsigned long long gen = 0;
  bool stop = false;
  explicit HostPool(int t) : T(t < 1 ? 1 : t) {
    for (int i = 1; i < T; ++i) th.emplace_back([this, i] { loop(i); });
  }
  void loop(int i) {
    unsigned long long seen = 0;
    for (;;) {
      std::function<void(size_t, size_t)> f;
      size_t nn;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return stop || gen != seen; });
        if (stop) return;
        seen = gen;
        f = fn;
        nn = n;
      }
      f(nn * i / T, nn * (i + 1) / T);
      std::lock_guard<std::mutex> lk(mu);
      if (--pending == 0) done_cv.notify_one();
    }
  }
  template <class F>
  void run(size_t n_, F&& f) {
    if (T == 1 || n_ < 64) {
      f(size_t(0), n_);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(mu);
      fn = f;
      n = n_;
      pending = T - 1;
      ++gen;
    }
    cv.notify_all();
    f(size_t(0), n_ / T);
    std::unique_lock<std::mutex> lk(mu);
    done_cv.wait(lk, [&] { return pending == 0; });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu);
      stop = true;
    }
    cv.notify_all();
    for (auto& t : th) t.join();
  }
};

struct b2p_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t user = nullptr;
  cudaStream_t aux = nullptr;  // second pipeline stream for batched host calls
  std::map<std::string, std::pair<void*, size_t>> ws;
  std::map<std::string, std::pair<void*, size_t>> hws;  // pinned host staging
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;  // start, end, formation end
  bool phases = false;
  // phase accounting: one (start, formation end, end) event triple per fused solve
  bool accounting = false;
  std::vector<cudaEvent_t> pool;
  size_t pool_used = 0;
  float last_ms = 0.f;
  size_t last_h2d_bytes = 0;  // host -> device bytes of the last b2p_solve_batched
  // next LL epoch of the fused grid kernel, one counter per LL buffer (tag):
  // a buffer's words are only ever compared against its own epochs
  std::map<std::string, unsigned> fg_epoch;
  int last_path = 0;  // 0: split K1(+K2)+K3, 1: one-CTA fused, 2: fused cluster, 3: fused grid
  unsigned long long* timing = nullptr;  // B2P_PHASE_TIMING=1: per-system phase stamps
  int timing_n = 0;
  std::atomic<long long> launches{0};
  int sm_count = 148;
  size_t smem_optin = 227 * 1024;
  std::unique_ptr<HostPool> host_pool;  // created on first packed upload
  cudaStream_t stream() const { return user ? user : own; }
};

namespace {

// NVTX range per C-ABI call (header-only NVTX v3: a no-op unless a profiler
// such as nsys / ncu --nvtx attaches), so timelines show the API boundary
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// ------------------------------------------------------------------ errors
struct Fail {
  int code;
  std::string msg;
  int knot = -1, iteration = -1, system = -1;
};

void fill_err(b2p_error* err, const Fail& f) {
  if (!err) return;
  err->code = f.code;
  err->knot = f.knot;
  err->iteration = f.iteration;
  err->system = f.system;
  std::snprintf(err->message, sizeof(err->message), "%s", f.msg.c_str());
}

void clear_err(b2p_error* err) {
  if (!err) return;
  err->code = B2P_OK;
  err->knot = err->iteration = err->system = -1;
  err->message[0] = 0;
}

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      throw Fail{B2P_CUDA_ERROR, std::string("CUDA error: ") + cudaGetErrorString(e_) +    \
                                     " at " + __FILE__ + ":" + std::to_string(__LINE__)};  \
  } while (0)

template <class F>
int guard(b2p_error* err, F&& f) {
  clear_err(err);
  try {
    f();
    return B2P_OK;
  } catch (const Fail& e) {
    (void)cudaGetLastError();  // a failed launch must not surface in the next call
    fill_err(err, e);
    return e.code;
  } catch (const std::exception& e) {
    (void)cudaGetLastError();
    fill_err(err, Fail{B2P_RUNTIME_ERROR, e.what()});
    return B2P_RUNTIME_ERROR;
  }
}

Fail invalid(const std::string& m) { return Fail{B2P_INVALID_ARGUMENT, m}; }

// std::to_string(double) == "%f"
std::string fstr(double v) {
  char buf[512];
  std::snprintf(buf, sizeof(buf), "%f", v);
  return buf;
}

size_t esize(int dtype) { return dtype == B2P_F32 ? 4 : 8; }

void check_dtype(int dtype) {
  if (dtype != B2P_F64 && dtype != B2P_F32) throw invalid("b2p: unknown dtype");
}
void check_ctx(b2p_ctx* ctx) {
  if (!ctx) throw invalid("b2p: null context");
  CK(cudaSetDevice(ctx->device));
}
void check_blocktri(int K, int nb) {
  if (K < 1 || nb < 1)
    throw invalid("BlockTriMatrix: need at least one block row and block_dim >= 1");
  if (nb > 32) throw invalid("b2p: block_dim > 32 is not supported by the warp-tile kernels");
}

// ------------------------------------------------------------------ workspaces
void* ws_get(b2p_ctx* c, const std::string& name, size_t bytes) {
  auto& slot = c->ws[name];
  if (slot.second < bytes) {
    if (slot.first) CK(cudaFree(slot.first));
    slot.first = nullptr;
    slot.second = 0;
    if (bytes) CK(cudaMalloc(&slot.first, bytes));
    slot.second = bytes;
  }
  return slot.first;
}

// Pinned host staging buffer: a D2H into pageable memory blocks the host
// thread until the copy (and every kernel before it) is done, which would
// serialise the chunked H2D/compute pipeline of b2p_solve_batched.
void* hws_get(b2p_ctx* c, const std::string& name, size_t bytes) {
  auto& slot = c->hws[name];
  if (slot.second < bytes) {
    if (slot.first) CK(cudaFreeHost(slot.first));
    slot.first = nullptr;
    slot.second = 0;
    if (bytes) CK(cudaMallocHost(&slot.first, bytes));
    slot.second = bytes;
  }
  return slot.first;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

void h2d(b2p_ctx* c, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
}
void d2h(b2p_ctx* c, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
}

// ------------------------------------------------------------------ messages
std::string schur_msg(int key, int* knot) {
  const int b = key / 4, call = key % 4;
  const char* what = "Q";
  int k = 0;
  if (b == 0) {
    k = 0;
  } else {
    k = b - 1;
    if (call == 1) what = "R";
    if (call == 2) k = b;  // Q_{k+1}
    if (call == 3) what = "theta";
  }
  if (knot) *knot = k;
  return std::string("build_schur: ") + what + " at knot " + std::to_string(k) +
         " is not positive definite";
}

Fail pcg_fail(const SysOut& o) {
  Fail f{o.code, ""};
  f.iteration = o.iteration;
  switch (o.which) {
    case kWhichInitNonFinite: f.msg = "pcg: non-finite initial residual"; break;
    case kWhichUpsNonFinite:
      f.msg = "pcg: non-finite p'Sp at iteration " + std::to_string(o.iteration);
      break;
    case kWhichEtaNonFinite:
      f.msg = "pcg: non-finite iterate at iteration " + std::to_string(o.iteration);
      break;
    case kWhichBreakdown:
      f.msg = "pcg: p'Sp = " + fstr(o.value) + " at iteration " + std::to_string(o.iteration) +
              "; S is not positive definite on the search space";
      break;
    default: f.msg = "pcg: device error";
  }
  return f;
}

void fill_report(b2p_solve_report* r, const SysOut& o, double wall) {
  if (!r) return;
  r->iterations = o.iterations;
  r->converged = o.converged;
  r->exit_eta = o.exit_eta;
  r->wall_time = wall;
  r->max_residual_drift = o.max_drift;
  r->trace_len = o.trace_len;
  r->status = o.code;
}

// ------------------------------------------------------------------ launch config
int env_int(const char* name, int def) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : def;
}

template <class T>
void configure_pcg(b2p_ctx* c, PcgParams<T>& p, bool allow_grid) {
  const size_t budget = std::min<size_t>(c->smem_optin, 227 * 1024) - 2048;
  p.nthreads = env_int("B2P_PCG_THREADS", 256);
  const int forceG = env_int("B2P_PCG_G", 0);
  const int forceStage = env_int("B2P_PCG_STAGE", -1);
  auto try_cfg = [&](int G, int stage) {
    p.G = G;
    p.rows_per = (p.K + G - 1) / G;
    p.G = (p.K + p.rows_per - 1) / p.rows_per;
    p.stage = stage;
    return pcg_smem_bytes(p) <= budget;
  };
  auto set_sync = [&]() {
    p.sync = p.G == 1 ? kSyncCta : (p.G <= 16 && p.B > 1 ? kSyncCluster
                                    : (p.G <= 8 ? kSyncCluster : kSyncGrid));
  };
  if (p.check_drift) {  // the drift probe is evaluated on one CTA (sequential variant)
    if (!try_cfg(1, forceStage < 0 ? 1 : forceStage)) try_cfg(1, 0);
    p.sync = kSyncCta;
    return;
  }
  if (forceG > 0) {
    if (!try_cfg(forceG, forceStage < 0 ? 1 : forceStage)) try_cfg(forceG, 0);
    set_sync();
    if (p.sync == kSyncGrid && (!allow_grid || p.B > 1)) {
      try_cfg(1, 0);
      p.sync = kSyncCta;
    }
    return;
  }
  if (forceStage != 0 && p.B == 1 && static_cast<long long>(p.K) * p.nb > 256) {
    // one system that is not tiny: clusters of 8 or 16 CTAs with <= 112 scalar
    // rows each measured best (scripts/explicit_policy_probe.py: c1 105 -> 78 us,
    // K 64 124 -> 90, c2 134 -> 121, K 129 n 4 91 -> 70); longer horizons keep
    // the rules below
    const long long rows = static_cast<long long>(p.K) * p.nb;
    const int pref = rows <= 8 * 112 ? 8 : (rows <= 16 * 112 ? 16 : 0);
    if (pref && try_cfg(pref, 1)) {
      set_sync();
      if (p.sync != kSyncGrid || allow_grid) return;
    }
  }
  if (forceStage != 0) {
    for (int G : {1, 2, 4, 8}) {
      if (try_cfg(G, 1)) {
        set_sync();
        return;
      }
    }
    if (allow_grid && p.B == 1) {
      // one solve across many SMs: cooperative grid with staged rows
      for (int rows = 8; rows >= 1; --rows) {
        const int G = (p.K + rows - 1) / rows;
        if (G > c->sm_count) break;
        if (try_cfg(G, 1)) {
          p.sync = kSyncGrid;
          return;
        }
      }
    }
  }
  // unstaged (S rows read from global memory): the smallest CTA group whose
  // vector slices fit — long horizons of large blocks need a cluster even so
  for (int G : {1, 2, 4, 8, 16}) {
    if (!try_cfg(G, 0)) continue;
    set_sync();
    if (p.sync == kSyncGrid && (!allow_grid || p.B > 1)) continue;
    return;
  }
  throw Fail{B2P_RUNTIME_ERROR, "pcg: the PCG vectors of one system (K = " + std::to_string(p.K) +
                                    ", n = " + std::to_string(p.nb) + ") exceed 16 CTAs' shared memory"};
}

template <class T>
void pcg_common(PcgParams<T>& p, const b2p_pcg_config* cfg, int K, int nb) {
  p.K = K;
  p.nb = nb;
  p.epsilon = cfg ? cfg->epsilon : 1e-4;
  const int mi = cfg ? cfg->max_iter : 0;
  p.max_iter = mi > 0 ? mi : K * nb;  // resolve_max_iter, pcg.cpp:49-51
  // the drift probe exists in the sequential variant only (pcg.cpp:103-108)
  p.check_drift = (cfg && cfg->check_residual_drift && cfg->variant == B2P_SEQUENTIAL) ? 1 : 0;
}

// ------------------------------------------------------------------ PCG runner
template <class T>
void run_pcg(b2p_ctx* c, PcgParams<T>& p, cudaStream_t st, bool time_it) {
  const size_t D = static_cast<size_t>(p.K) * p.nb;
  p.best = static_cast<T*>(ws_get(c, "pcg_best", sizeof(T) * D * p.B));
  p.pub = static_cast<T*>(ws_get(c, "pcg_pub", sizeof(T) * D * p.B));
  p.slots = static_cast<T*>(ws_get(c, "pcg_slots", sizeof(T) * 2 * std::max(1, p.G) * p.B + 64));
  c->phases = false;
  p.gbar = static_cast<unsigned*>(ws_get(c, "pcg_gbar", 256));
  if (time_it) CK(cudaEventRecord(c->ev0, st));
  if (p.sync == kSyncGrid) CK(cudaMemsetAsync(p.gbar, 0, sizeof(unsigned), st));
  CK(launch_pcg<T>(p, st));
  c->launches++;
  if (time_it) CK(cudaEventRecord(c->ev1, st));
}

// kkt views
struct KktDev {
  const void *Q, *q, *R, *r, *A, *B, *e, *x_s, *x0;
};

// Upload `count` systems starting at `first` from a host batch into one
// contiguous device block; returns per-array device pointers.
size_t kkt_block_bytes(const b2p_kkt* k, size_t esz, int count) {
  const size_t N = k->N, n = k->n, m = k->m, K = N + 1;
  const size_t sz[9] = {K * n * n, K * n, N * m * m, N * m, N * n * n, N * n * m, N * n, n, n};
  size_t total = 0;
  for (size_t s : sz) total += (s * esz * count + 255) / 256 * 256;
  return total;
}

// Copies systems [first, first+count) of the host batch `k` into the device
// block `dst` (laid out as kkt_block_bytes). A single system is latency-bound:
// its nine arrays (plus an optional trailing `extra` host vector, returned in
// *extra_dev) are packed into one pinned staging block and sent with ONE copy
// instead of ten pageable cudaMemcpyAsync round trips. Callers synchronise the
// stream before returning, so the staging block is free again by the next call.
KktDev upload_kkt(b2p_ctx* c, const b2p_kkt* k, size_t esz, int first, int count, void* dst,
                  cudaStream_t st, const void* extra = nullptr, size_t extra_bytes = 0,
                  char** extra_dev = nullptr, bool may_stage = true) {
  const size_t N = k->N, n = k->n, m = k->m, K = N + 1;
  const size_t sz[9] = {K * n * n, K * n, N * m * m, N * m, N * n * n, N * n * m, N * n, n, n};
  const void* src[9] = {k->Q, k->q, k->R, k->r, k->A, k->B, k->e, k->x_s, k->x0};
  const void* out[9];
  char* d = static_cast<char*>(dst);
  // the chunked pipeline of b2p_solve_batched does not synchronise between
  // chunks, so it never stages (one staging block would be overwritten while
  // an earlier chunk's asynchronous H2D still reads it)
  const bool staged = count == 1 && may_stage;
  const size_t total = kkt_block_bytes(k, esz, count) + extra_bytes;
  char* h = staged ? static_cast<char*>(hws_get(c, "up_stage", total)) : nullptr;
  for (int a = 0; a < 9; ++a) {
    const size_t bytes = sz[a] * esz * count;
    if (bytes && !src[a]) throw invalid("b2p_kkt: null array");
    const char* from = static_cast<const char*>(src[a]) + sz[a] * esz * first;
    if (bytes) {
      if (staged)
        std::memcpy(h + (d - static_cast<char*>(dst)), from, bytes);
      else
        h2d(c, d, from, bytes, st);
    }
    out[a] = d;
    d += (bytes + 255) / 256 * 256;
  }
  if (extra_bytes) {
    if (staged)
      std::memcpy(h + (d - static_cast<char*>(dst)), extra, extra_bytes);
    else
      h2d(c, d, extra, extra_bytes, st);
    *extra_dev = d;
  }
  if (staged) h2d(c, dst, h, total, st);
  return KktDev{out[0], out[1], out[2], out[3], out[4], out[5], out[6], out[7], out[8]};
}

KktDev dev_view(const b2p_kkt* k) {
  return KktDev{k->Q, k->q, k->R, k->r, k->A, k->B, k->e, k->x_s, k->x0};
}

void check_kkt(const b2p_kkt* k) {
  if (!k) throw invalid("b2p: null kkt");
  if (k->N < 0 || k->n < 1 || k->m < 0)
    throw invalid("b2p_kkt: need N >= 0, n >= 1, m >= 0");
  check_blocktri(k->N + 1, k->n);
  if (k->m > 32) throw invalid("b2p: control dim > 32 is not supported");
}

// Formation (K1) for `B` systems whose inputs are at device view `kv`.
template <class T>
void launch_form(b2p_ctx* c, const b2p_kkt* k, const KktDev& kv, int B, T* S, T* gamma, T* ti,
                 int* errkey, cudaStream_t st) {
  FormParams<T> f;
  f.B = B;
  f.N = k->N;
  f.n = k->n;
  f.m = k->m;
  f.Q = static_cast<const T*>(kv.Q);
  f.q = static_cast<const T*>(kv.q);
  f.R = static_cast<const T*>(kv.R);
  f.r = static_cast<const T*>(kv.r);
  f.A = static_cast<const T*>(kv.A);
  f.Bm = static_cast<const T*>(kv.B);
  f.e = static_cast<const T*>(kv.e);
  f.x_s = static_cast<const T*>(kv.x_s);
  f.x0 = static_cast<const T*>(kv.x0);
  f.S = S;
  f.gamma = gamma;
  f.theta_inv = ti;
  f.errkey = errkey;
  CK(cudaMemsetAsync(errkey, 0x7f, sizeof(int) * B, st));  // 0x7f7f7f7f: see below
  const int K = k->N + 1;
  if (env_int("B2P_FUSED", 1) && env_int("B2P_SMALL", 1) &&
      small_supported<T>(K, k->n, k->m, kSymStair)) {
    // small blocks: the small-block kernel's formation in formation-only mode
    FusedParams<T> g{};
    g.B = B;
    g.K = K;
    g.kind = kSymStair;
    g.Q = f.Q;
    g.q = f.q;
    g.R = f.R;
    g.r = f.r;
    g.A = f.A;
    g.Bm = f.Bm;
    g.e = f.e;
    g.x_s = f.x_s;
    g.x0 = f.x0;
    g.errkey = errkey;
    g.out = static_cast<SysOut*>(ws_get(c, "form_out", sizeof(SysOut) * B));
    g.S_out = S;
    g.gamma_out = gamma;
    g.theta_out = ti;
    g.form_only = 1;
    g.max_iter = 1;
    CK(launch_small<T>(g, k->n, k->m, c->sm_count, st));
    c->launches++;
    return;
  }
  if (env_int("B2P_FUSED", 1) && fused_supported<T>(K, k->n, k->m, kSymStair)) {
    // the fused kernel's formation phase (shared Q_k^-1, half-warp rows) in
    // formation-only mode writes S / gamma / theta^-1 in the reference layout
    const int grid = std::max(1, std::min(B, c->sm_count));
    FusedParams<T> g{};
    g.B = B;
    g.K = K;
    g.kind = kSymStair;
    g.Q = f.Q;
    g.q = f.q;
    g.R = f.R;
    g.r = f.r;
    g.A = f.A;
    g.Bm = f.Bm;
    g.e = f.e;
    g.x_s = f.x_s;
    g.x0 = f.x0;
    g.slot = static_cast<T*>(
        ws_get(c, "form_slot", sizeof(T) * grid * fused_slot_elems<T>(K, k->n, k->m)));
    g.errkey = errkey;
    g.out = static_cast<SysOut*>(ws_get(c, "form_out", sizeof(SysOut) * B));
    g.S_out = S;
    g.gamma_out = gamma;
    g.theta_out = ti;
    g.form_only = 1;
    g.max_iter = 1;
    CK(cudaMemsetAsync(S, 0, sizeof(T) * static_cast<size_t>(B) * K * 3 * k->n * k->n, st));
    CK(launch_fused<T>(g, k->n, k->m, grid, st));
    c->launches++;
    return;
  }
  CK(launch_build_schur<T>(f, st));
  c->launches++;
}
// errkey is initialised with bytes 0x7f => 0x7f7f7f7f; the kernels treat any
// value >= 0x7f7f7f7f as "ok". Normalise for the PCG kernel check:
constexpr int kErrOk = 0x7f7f7f7f;

// Fused batched solve on device data: K1 formation -> K3 PCG (fused mode).
// dz_dev (nullable): the one-CTA and small-block kernels also run the PPCG
// finish (reconstruct_primal) in their epilogue; returns whether dz was
// produced (else the caller launches the primal kernel).
// out[b] (ro x co) <- in[b] (ri x ci): copy the common top-left part, fill the
// rest with zeros (diag: ones on the diagonal). Pads odd-n state blocks to
// n + 1 for the one-CTA kernel (identity Q pad, zero A / B / vector pads) and
// crops lambda back.
template <class T>
__global__ void k_reblock(const T* __restrict__ in, T* __restrict__ out, long long nblocks, int ri,
                          int ci, int ro, int co, int diag) {
  const long long total = nblocks * ro * co;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long b = e / (ro * co);
    const int i = static_cast<int>((e / co) % ro), j = static_cast<int>(e % co);
    out[e] = (i < ri && j < ci) ? in[b * ri * ci + static_cast<long long>(i) * ci + j]
                                : ((diag && i == j) ? T(1) : T(0));
  }
}
template <class T>
void reblock(const void* in, void* out, long long nblocks, int ri, int ci, int ro, int co, int diag,
             cudaStream_t st) {
  const long long total = nblocks * ro * co;
  if (total <= 0) return;
  const int grid = static_cast<int>(std::min<long long>((total + 255) / 256, 4096));
  k_reblock<T><<<grid, 256, 0, st>>>(static_cast<const T*>(in), static_cast<T*>(out), nblocks, ri,
                                      ci, ro, co, diag);
  CK(cudaGetLastError());
}

// ------------------------------------------------------------ packed upload
// The solve path reads only the lower triangles of Q_k and R_k: every
// factorisation is Eigen's LLT / LDLT, which reads the lower triangle
// (schur.cpp:16, :61-63; kkt.cpp:171-177), and only theta_inv[0] = sym(Q_0)
// (schur.cpp:56) reads an upper one. The host batch path therefore ships the
// lower triangles (+ Q_0's strict upper triangle) over PCIe and mirrors them
// on the device: 19 % fewer H2D bytes at c4, and any input — an asymmetric
// Q_k or R_k included — is read exactly as the reference reads it.
inline size_t tri(int n) { return static_cast<size_t>(n) * (n + 1) / 2; }

// block b of `nblk` n x n blocks -> its lower triangle (row-major rows 0..r);
// with k0 > 0, block s * k0 of every system s also gives its strict upper
// triangle to `up` (row-major, row r: columns r+1..n-1)
// 8-byte / 4-byte non-temporal stores: the staging is written once and read by
// the DMA engine, so the stores bypass the cache (no read-for-ownership)
inline void st_nt(double* p, double v) {
  long long b;
  std::memcpy(&b, &v, 8);
  _mm_stream_si64(reinterpret_cast<long long*>(p), b);
}
inline void st_nt(float* p, float v) {
  int b;
  std::memcpy(&b, &v, 4);
  _mm_stream_si32(reinterpret_cast<int*>(p), b);
}
template <class T>
void pack_lower(const T* src, T* dst, T* up, int n, int k0, size_t b0, size_t b1) {
  const size_t nn = static_cast<size_t>(n) * n, t = tri(n), tu = tri(n - 1);
  for (size_t b = b0; b < b1; ++b) {
    const T* a = src + b * nn;
    T* o = dst + b * t;
    for (int r = 0; r < n; ++r)
      for (int c = 0; c <= r; ++c) st_nt(o++, a[r * n + c]);
    if (k0 > 0 && b % k0 == 0) {
      T* u = up + (b / k0) * tu;
      for (int r = 0; r + 1 < n; ++r)
        for (int c = r + 1; c < n; ++c) st_nt(u++, a[r * n + c]);
    }
  }
  _mm_sfence();  // the streaming stores are visible before the DMA is issued
}

template <class T>
__global__ void k_unpack_sym(const T* __restrict__ L, const T* __restrict__ U0, T* __restrict__ out,
                             long long nblk, int n, int k0) {
  const int nn = n * n, t = n * (n + 1) / 2, tu = n * (n - 1) / 2;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < nblk * nn;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long b = e / nn;
    const int w = static_cast<int>(e - b * nn), r = w / n, c = w - r * n;
    T v;
    if (r >= c) {
      v = L[b * t + r * (r + 1) / 2 + c];
    } else if (k0 > 0 && b % k0 == 0) {
      v = U0[(b / k0) * tu + r * (n - 1) - r * (r - 1) / 2 + (c - r - 1)];
    } else {
      v = L[b * t + c * (c + 1) / 2 + r];
    }
    out[e] = v;
  }
}
template <class T>
void unpack_sym(const void* L, const void* U0, void* out, long long nblk, int n, int k0,
                cudaStream_t st) {
  const long long total = nblk * n * n;
  if (total <= 0) return;
  const int grid = static_cast<int>(std::min<long long>((total + 255) / 256, 8192));
  k_unpack_sym<T><<<grid, 256, 0, st>>>(static_cast<const T*>(L), static_cast<const T*>(U0),
                                         static_cast<T*>(out), nblk, n, k0);
  CK(cudaGetLastError());
}

// upload_kkt for the chunked batch pipeline with Q and R packed (see above):
// the other arrays go straight from the caller's memory; Q / R are packed
// into the pinned staging `hpk` (reused only after `ready`, the event of its
// previous H2D) and mirrored on the device into the same layout upload_kkt
// produces. Returns the H2D byte count through *h2d_bytes.
template <class T>
KktDev upload_kkt_packed(b2p_ctx* c, const b2p_kkt* k, int first, int count, void* dst,
                         cudaStream_t st, const std::string& tag, cudaEvent_t ready,
                         size_t* h2d_bytes) {
  const size_t es = sizeof(T);
  const size_t N = k->N, n = k->n, m = k->m, K = N + 1;
  const size_t sz[9] = {K * n * n, K * n, N * m * m, N * m, N * n * n, N * n * m, N * n, n, n};
  const void* src[9] = {k->Q, k->q, k->R, k->r, k->A, k->B, k->e, k->x_s, k->x0};
  const void* out[9];
  char* d = static_cast<char*>(dst);
  size_t bytes_total = 0;
  for (int a = 0; a < 9; ++a) {
    const size_t bytes = sz[a] * es * count;
    if (bytes && !src[a]) throw invalid("b2p_kkt: null array");
    out[a] = d;
    if (bytes && a != 0 && a != 2) {
      h2d(c, d, static_cast<const char*>(src[a]) + sz[a] * es * first, bytes, st);
      bytes_total += bytes;
    }
    d += (bytes + 255) / 256 * 256;
  }
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  const size_t nq = K * count, nr = N * count;
  const size_t bq = al(nq * tri(int(n)) * es), bu = al(count * tri(int(n) - 1) * es),
               br = al(nr * tri(int(m)) * es);
  char* h = static_cast<char*>(hws_get(c, tag + "pk", bq + bu + br));
  char* dv = static_cast<char*>(ws_get(c, tag + "pkd", bq + bu + br));
  CK(cudaEventSynchronize(ready));  // the staging's previous H2D has completed
  const T* Qs = static_cast<const T*>(k->Q) + sz[0] * first;
  const T* Rs = static_cast<const T*>(k->R) + (sz[2] ? sz[2] * first : 0);
  T* hq = reinterpret_cast<T*>(h);
  T* hu = reinterpret_cast<T*>(h + bq);
  T* hr = reinterpret_cast<T*>(h + bq + bu);
  if (!c->host_pool) {
    const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    c->host_pool.reset(new HostPool(std::min(hw, std::max(1, env_int("B2P_PACK_THREADS", 16)))));
  }
  c->host_pool->run(nq + nr, [&](size_t lo, size_t hi) {
    if (lo < nq) pack_lower<T>(Qs, hq, hu, int(n), int(K), lo, std::min(hi, nq));
    if (hi > nq && m > 0) pack_lower<T>(Rs, hr, nullptr, int(m), 0, std::max(lo, nq) - nq, hi - nq);
  });
  h2d(c, dv, h, bq + bu + br, st);
  CK(cudaEventRecord(ready, st));
  bytes_total += (nq * tri(int(n)) + count * tri(int(n) - 1) + nr * tri(int(m))) * es;
  unpack_sym<T>(dv, dv + bq, const_cast<void*>(out[0]), static_cast<long long>(nq), int(n), int(K), st);
  if (m > 0) unpack_sym<T>(dv + bq + bu, nullptr, const_cast<void*>(out[2]), static_cast<long long>(nr), int(m), 0, st);
  if (h2d_bytes) *h2d_bytes += bytes_total;
  return KktDev{out[0], out[1], out[2], out[3], out[4], out[5], out[6], out[7], out[8]};
}

template <class T>
bool solve_device_impl(b2p_ctx* c, const b2p_kkt* k, const KktDev& kv, int B, int kind,
                       int order, const b2p_pcg_config* cfg, const void* lambda0, void* lambda_out,
                       SysOut* outs_dev, int* errkey, double* trace_dev, int trace_cap,
                       cudaStream_t st, bool time_it, const std::string& tag,
                       void* dz_dev = nullptr) {
  const int K = k->N + 1, n = k->n;
  const size_t nn = static_cast<size_t>(n) * n, D = static_cast<size_t>(K) * n;
  const bool drift = cfg && cfg->check_residual_drift && cfg->variant == B2P_SEQUENTIAL;
  // Fused cluster kernel: default for single solves and for shapes the
  // one-CTA fused kernel does not cover; B2P_FC=1 forces it, =0 disables it.
  const int fc_env = env_int("B2P_FC", -1);
  int fcG = drift ? 0 : fc_pick_g<T>(K, n, k->m, kind, B);
  if (fcG > 0 && env_int("B2P_FC_G", 0) > 0) {
    const int g = env_int("B2P_FC_G", 0);
    if ((K + g - 1) / g <= 32 && (K + ((K + g - 1) / g) - 1) / ((K + g - 1) / g) == g) fcG = g;
  }
  // n = 7, 8 (n = 7 through the identity pad): the one-CTA kernel when the
  // small-block kernel does not cover the shape, and for horizons K > 24
  // (batches; single solves only at n = 8, where no pad copies are needed).
  // Measured (scripts/onecta_small_probe.py, profiles/r02_onecta_small.json):
  // 4096 x K 64: n7 m2 1.65 -> 2.49 M/s, n8 m4 1.58 -> 2.96 M/s; K 17: small-block
  // 3.9 vs 3.8 M/s; K 9: 8.7 vs 4.1 M/s. B2P_ONECTA_MIN_N=<n> overrides (n >= it).
  const int onecta_floor = env_int("B2P_ONECTA_MIN_N", -1);
  auto onecta_n = [&](int nn) -> bool {
    if (onecta_floor >= 0) return nn >= onecta_floor;
    if (nn >= 9) return true;
    if (nn < 7) return false;
    const bool small_ok = env_int("B2P_SMALL", 1) && small_supported<T>(K, nn, k->m, kind);
    return !small_ok || (K > 24 && (B > 1 || nn == 8));
  };
  const bool one_cta_ok = onecta_n(n) && fused_supported<T>(K, n, k->m, kind);
  // odd n in [7, 15] on the one-CTA kernel through the identity pad (below)
  const bool pad_ok = !drift && !dz_dev && sizeof(T) == 8 && (n & 1) && onecta_n(n) && n + 1 <= 16 &&
                      env_int("B2P_FUSED", 1) && env_int("B2P_PAD", 1) &&
                      fused_supported<T>(K, n + 1, k->m, kind);
  const bool small_ok = !drift && env_int("B2P_FUSED", 1) && env_int("B2P_SMALL", 1) &&
                        small_supported<T>(K, n, k->m, kind) &&
                        (!dz_dev || small_supported_dz<T>(K, n, k->m, kind));
  // Batches of n in [11, 16], m <= 8 that neither the one-CTA kernel (K > 64) nor
  // the small-block kernel takes: the cluster kernel compiled at (16, 8)
  // through the same pads (B2P_FC_PAD=0 disables). scripts/fc_pad_probe.py:
  // 4096 x K 128 n12 m4 98 K -> 214 K/s, K 65 n14 m5 141 K -> 303 K/s vs the
  // split path; n 9 (16 / 9 of the state) measured equal, so it stays split.
  int cnp = n, cmp = k->m;
  if (fcG == 0 && !drift && sizeof(T) == 8 && n >= 11 && n <= 16 && k->m >= 1 && k->m <= 8 &&
      !one_cta_ok && !pad_ok && !small_ok && env_int("B2P_FC_PAD", 1)) {
    fcG = fc_pick_g<T>(K, 16, 8, kind, B);
    if (fcG > 0) cnp = 16, cmp = 8;
  }
  const bool fc_padded = cnp != n || cmp != k->m;
  // Fused grid kernel: one long-horizon system over G co-resident CTAs (the
  // default for shapes no cluster / one-CTA kernel covers, e.g. c5);
  // B2P_FG=1 forces it, =0 disables it; B2P_FG_RP picks the rows per CTA.
  // Shapes it is not compiled for run on the smallest compiled (n', m') that
  // holds them (fp64 n <= 32, m <= 16), through an identity-padded state /
  // control (Q, R) and zero pads elsewhere — as the one-CTA odd-n pad below:
  // every pad entry of S, gamma, theta^-1 and the PCG vectors stays exactly 0.
  const int fg_env = env_int("B2P_FG", -1);
  int fnp = n, fmp = k->m;
  // (padded only for shapes no one-CTA / small-block kernel takes, and while
  // n' <= 2 n: n 4, m 12 on the (32, 16) kernel measured slower than the split
  // path, scripts/fg_pad_probe.py)
  const bool fg_shape_ok =
      !drift && B <= 8 && fg_compiled_shape<T>(n, k->m, &fnp, &fmp) &&
      ((fnp == n && fmp == k->m) ||
       (env_int("B2P_FG_PAD", 1) && fnp <= 2 * n && !one_cta_ok && !pad_ok && !small_ok));
  const int fgRp = !fg_shape_ok ? 0
                                : fg_pick_rp<T>(K, fnp, fmp, kind, c->sm_count,
                                                env_int("B2P_FG_RP", 0));
  const bool fg_padded = fnp != n || fmp != k->m;
  // fused kernels (one launch, no separate formation): a (start, formation end,
  // end) event triple from the context's pool when the caller times phases
  auto fused_timing_begin = [&]() {
    if (!time_it) return;
    if (!c->accounting) c->pool_used = 0;
    if (c->pool_used + 3 > c->pool.size())
      for (int q = 0; q < 3; ++q) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        c->pool.push_back(e);
      }
    c->ev0 = c->pool[c->pool_used];
    c->ev2 = c->pool[c->pool_used + 1];
    c->ev1 = c->pool[c->pool_used + 2];
    c->pool_used += 3;
    CK(cudaEventRecord(c->ev0, st));
    CK(cudaEventRecord(c->ev2, st));
  };
  // Single-solve policy (scripts/c1_policy_probe.py, profiles/r02_single_policy.json,
  // and the bench's c1 row): K <= 64 on one CTA (K 64: 87 us vs 93 on the grid
  // kernel; c1: 77 us in the bench vs 88 on the grid kernel there, although an
  // isolated probe timed the grid kernel at 73), longer fp64 horizons on the
  // grid kernel, fp32 / other shapes on the cluster kernel.
  const bool single_short = B == 1 && K <= 64 && one_cta_ok;
  const bool use_fg = fgRp > 0 && env_int("B2P_FUSED", 1) &&
                      (fg_env == 1 ||
                       (fg_env == -1 && ((fcG == 0 && !one_cta_ok && !pad_ok) ||
                                         (B == 1 && !single_short && sizeof(T) == 8 &&
                                          fc_env != 1))));
  // Identity-padded Q / R and zero-padded A, B, q, r, e, x_s, x0 (and lambda0)
  // at (np, mp) for the grid / cluster kernels' compiled shapes; points f at
  // them and returns the padded lambda the caller crops back.
  auto pad_view = [&](int np, int mp, FusedParams<T>& f) -> T* {
    const int m = k->m, N = K - 1;
    const long long Bl = B;
    const size_t eQ = size_t(K) * np * np, eq = size_t(K) * np, eR = size_t(N) * mp * mp,
                 er = size_t(N) * mp, eA = size_t(N) * np * np, eB = size_t(N) * np * mp,
                 ee = size_t(N) * np;
    const bool padm = mp != m;  // (the control blocks travel as they are when m' = m)
    const size_t per = eQ + eq + (padm ? eR + er : 0) + eA + eB + ee + 2 * np;
    T* w = static_cast<T*>(ws_get(c, tag + "xpad_kkt", sizeof(T) * per * B + 256));
    T *Qp = w, *qp = Qp + eQ * B, *Rp = qp + eq * B, *rp_ = Rp + (padm ? eR * B : 0),
      *Ap = rp_ + (padm ? er * B : 0), *Bp = Ap + eA * B, *ep = Bp + eB * B, *xsp = ep + ee * B,
      *x0p = xsp + size_t(np) * B;
    reblock<T>(kv.Q, Qp, Bl * K, n, n, np, np, 1, st);
    reblock<T>(kv.q, qp, Bl * K, n, 1, np, 1, 0, st);
    if (padm) {
      reblock<T>(kv.R, Rp, Bl * N, m, m, mp, mp, 1, st);
      reblock<T>(kv.r, rp_, Bl * N, m, 1, mp, 1, 0, st);
    }
    reblock<T>(kv.A, Ap, Bl * N, n, n, np, np, 0, st);
    reblock<T>(kv.B, Bp, Bl * N, n, m, np, mp, 0, st);
    reblock<T>(kv.e, ep, Bl * N, n, 1, np, 1, 0, st);
    reblock<T>(kv.x_s, xsp, Bl, n, 1, np, 1, 0, st);
    reblock<T>(kv.x0, x0p, Bl, n, 1, np, 1, 0, st);
    f.Q = Qp, f.q = qp, f.A = Ap, f.Bm = Bp, f.e = ep, f.x_s = xsp, f.x0 = x0p;
    f.R = padm ? Rp : static_cast<const T*>(kv.R);
    f.r = padm ? rp_ : static_cast<const T*>(kv.r);
    T* lam_pad = static_cast<T*>(ws_get(c, tag + "xpad_lam", sizeof(T) * B * K * np));
    if (lambda0) {
      T* l0p = static_cast<T*>(ws_get(c, tag + "xpad_l0", sizeof(T) * B * K * np));
      reblock<T>(lambda0, l0p, Bl * K, n, 1, np, 1, 0, st);
      f.lambda0 = l0p;
    }
    f.lambda_out = lam_pad;
    c->launches += (padm ? 9 : 7) + (lambda0 ? 1 : 0);
    return lam_pad;
  };
  if (use_fg) {
    FusedParams<T> f{};
    f.B = B;
    f.K = K;
    f.kind = kind;
    f.Q = static_cast<const T*>(kv.Q);
    f.q = static_cast<const T*>(kv.q);
    f.R = static_cast<const T*>(kv.R);
    f.r = static_cast<const T*>(kv.r);
    f.A = static_cast<const T*>(kv.A);
    f.Bm = static_cast<const T*>(kv.B);
    f.e = static_cast<const T*>(kv.e);
    f.x_s = static_cast<const T*>(kv.x_s);
    f.x0 = static_cast<const T*>(kv.x0);
    f.lambda0 = static_cast<const T*>(lambda0);
    f.lambda_out = static_cast<T*>(lambda_out);
    T* lam_pad = fg_padded ? pad_view(fnp, fmp, f) : nullptr;
    f.errkey = errkey;
    f.out = outs_dev;
    f.trace = trace_dev;
    f.trace_cap = trace_cap;
    f.epsilon = cfg ? cfg->epsilon : 1e-4;
    const int mi = cfg ? cfg->max_iter : 0;
    f.max_iter = mi > 0 ? mi : static_cast<int>(D);
    const int G = (K + fgRp - 1) / fgRp;
    FgSync<T> sy{};
    sy.gstride = (G + 31) / 32 * 32;
    sy.n = fnp;
    // LL slots: 16 bytes per value. Zeroed when (re)allocated; afterwards each
    // launch starts at a fresh epoch so words of earlier launches never match.
    const size_t slots = static_cast<size_t>(sy.gstride) * (2 * 8 + 2 * 2 * 32);
    const size_t bytes = slots * 16;
    void* cur = c->ws.count(tag + "fg_ll") ? c->ws[tag + "fg_ll"].first : nullptr;
    unsigned long long* ll = static_cast<unsigned long long*>(ws_get(c, tag + "fg_ll", bytes));
    const unsigned need = static_cast<unsigned>(
        std::min<long long>(1ll << 30, 3ll * (f.max_iter + 4) * B + 16));
    unsigned& epoch = c->fg_epoch[tag + "fg_ll"];
    if (ll != cur || epoch == 0 || epoch > (1u << 31) - need) {
      CK(cudaMemsetAsync(ll, 0, c->ws[tag + "fg_ll"].second, st));
      epoch = 1;
    }
    sy.epoch0 = epoch;
    epoch += need;
    sy.red = ll;
    sy.xt = ll + 2 * 16 * static_cast<size_t>(sy.gstride);
    sy.xr = sy.xt + 2 * static_cast<size_t>(sy.gstride) * 2 * 32;
    fused_timing_begin();
    f.timing = env_int("B2P_PHASE_TIMING", 0)
                   ? static_cast<unsigned long long*>(ws_get(c, "fused_timing", 128ull * B))
                   : nullptr;
    c->timing = f.timing;
    c->timing_n = f.timing ? B : 0;
    const cudaError_t le = launch_fg<T>(f, sy, fgRp, st);
    if (le == cudaErrorCooperativeLaunchTooLarge) {
      // The grid did not fit co-resident (SMs taken by another context):
      // fall through to the cluster / split paths below.
      (void)cudaGetLastError();
      epoch -= need;
    } else {
      CK(le);
      c->launches++;
      if (lam_pad) {
        reblock<T>(lam_pad, lambda_out, static_cast<long long>(B) * K, fnp, 1, n, 1, 0, st);
        c->launches++;
      }
      c->last_path = 3;
      c->phases = time_it;
      if (time_it) CK(cudaEventRecord(c->ev1, st));
      return false;
    }
  }
  const bool use_fc = fcG > 0 && env_int("B2P_FUSED", 1) &&
                      (fc_env == 1 || (fc_env == -1 && ((B == 1 && !single_short) || !one_cta_ok)));
  if (use_fc) {
    FusedParams<T> f{};
    f.B = B;
    f.K = K;
    f.kind = kind;
    f.Q = static_cast<const T*>(kv.Q);
    f.q = static_cast<const T*>(kv.q);
    f.R = static_cast<const T*>(kv.R);
    f.r = static_cast<const T*>(kv.r);
    f.A = static_cast<const T*>(kv.A);
    f.Bm = static_cast<const T*>(kv.B);
    f.e = static_cast<const T*>(kv.e);
    f.x_s = static_cast<const T*>(kv.x_s);
    f.x0 = static_cast<const T*>(kv.x0);
    const int max_clusters = std::max(1, c->sm_count / fcG);
    // keyed by the stream tag: chunks on two streams may run concurrently and
    // each CTA owns the slot at its blockIdx
    f.slot = static_cast<T*>(ws_get(c, tag + "fc_slot", sizeof(T) * fcG * max_clusters *
                                                       fc_slot_elems<T>(K, cnp, fcG)));
    f.lambda0 = static_cast<const T*>(lambda0);
    f.lambda_out = static_cast<T*>(lambda_out);
    f.errkey = errkey;
    f.out = outs_dev;
    f.trace = trace_dev;
    f.trace_cap = trace_cap;
    f.epsilon = cfg ? cfg->epsilon : 1e-4;
    const int mi = cfg ? cfg->max_iter : 0;
    f.max_iter = mi > 0 ? mi : static_cast<int>(D);
    fused_timing_begin();
    T* lam_pad = fc_padded ? pad_view(cnp, cmp, f) : nullptr;
    CK(launch_fc<T>(f, fcG, max_clusters, st, cnp));
    c->launches++;
    if (lam_pad) {
      reblock<T>(lam_pad, lambda_out, static_cast<long long>(B) * K, cnp, 1, n, 1, 0, st);
      c->launches++;
    }
    c->last_path = 2;
    c->phases = time_it;
    if (time_it) CK(cudaEventRecord(c->ev1, st));
    return false;
  }
  // Odd n in [7, 15] on the one-CTA kernel: the state dimension padded to n + 1
  // (Q with an identity pad, A / B / q / e / x pads zero). Every pad entry of
  // S, gamma, theta^-1 and of every PCG vector is then exactly zero, so the
  // real rows follow the unpadded recurrence (the dot products only gain
  // exact zero terms); lambda is cropped back.
  if (pad_ok) {
    const int np = n + 1, m = k->m;
    const long long Bl = B;
    const int grid = std::max(1, std::min(B, c->sm_count));
    FusedParams<T> f{};
    f.B = B;
    f.K = K;
    f.kind = kind;
    f.lambda0 = static_cast<const T*>(lambda0);
    T* lamp = pad_view(np, m, f);  // identity-padded state, control as it is
    f.slot = static_cast<T*>(
        ws_get(c, tag + "fused_slot", sizeof(T) * grid * fused_slot_elems<T>(K, np, m, false)));
    f.errkey = errkey;
    f.out = outs_dev;
    f.trace = trace_dev;
    f.trace_cap = trace_cap;
    f.epsilon = cfg ? cfg->epsilon : 1e-4;
    const int mi = cfg ? cfg->max_iter : 0;
    f.max_iter = mi > 0 ? mi : static_cast<int>(D);  // the unpadded dimension (resolve_max_iter)
    fused_timing_begin();
    CK(launch_fused<T>(f, np, m, grid, st));
    reblock<T>(lamp, lambda_out, Bl * K, np, 1, n, 1, 0, st);
    c->launches += 2;
    c->last_path = 1;
    c->phases = time_it;
    if (time_it) CK(cudaEventRecord(c->ev1, st));
    return false;
  }
  if (!drift && env_int("B2P_FUSED", 1) && one_cta_ok) {
    // persistent one-CTA-per-system K1+K3 kernel (fused_kernels.cu)
    const int grid = std::max(1, std::min(B, c->sm_count));
    FusedParams<T> f{};
    f.B = B;
    f.K = K;
    f.kind = kind;
    f.Q = static_cast<const T*>(kv.Q);
    f.q = static_cast<const T*>(kv.q);
    f.R = static_cast<const T*>(kv.R);
    f.r = static_cast<const T*>(kv.r);
    f.A = static_cast<const T*>(kv.A);
    f.Bm = static_cast<const T*>(kv.B);
    f.e = static_cast<const T*>(kv.e);
    f.x_s = static_cast<const T*>(kv.x_s);
    f.x0 = static_cast<const T*>(kv.x0);
    f.dz_out = static_cast<T*>(dz_dev);
    f.slot = static_cast<T*>(ws_get(
        c, tag + "fused_slot", sizeof(T) * grid * fused_slot_elems<T>(K, n, k->m, dz_dev != nullptr)));
    f.timing = env_int("B2P_PHASE_TIMING", 0)
                   ? static_cast<unsigned long long*>(ws_get(c, "fused_timing", 128ull * B))
                   : nullptr;
    c->timing = f.timing;
    c->timing_n = f.timing ? B : 0;
    f.lambda0 = static_cast<const T*>(lambda0);
    f.lambda_out = static_cast<T*>(lambda_out);
    f.errkey = errkey;
    f.out = outs_dev;
    f.trace = trace_dev;
    f.trace_cap = trace_cap;
    f.epsilon = cfg ? cfg->epsilon : 1e-4;
    const int mi = cfg ? cfg->max_iter : 0;
    f.max_iter = mi > 0 ? mi : static_cast<int>(D);
    fused_timing_begin();
    CK(launch_fused<T>(f, n, k->m, grid, st));
    c->launches++;
    c->last_path = 1;
    c->phases = time_it;
    if (time_it) CK(cudaEventRecord(c->ev1, st));
    return dz_dev != nullptr;
  }
  if (!drift && env_int("B2P_FUSED", 1) && env_int("B2P_SMALL", 1) &&
      small_supported<T>(K, n, k->m, kind) &&
      (!dz_dev || small_supported_dz<T>(K, n, k->m, kind))) {
    // small blocks (n, m <= 8): one CTA per system, all in shared memory
    // persistent CTAs, as many as fit co-resident (launch_small scales the SM count)
    const int grid = c->sm_count;
    FusedParams<T> f{};
    f.B = B;
    f.K = K;
    f.kind = kind;
    f.Q = static_cast<const T*>(kv.Q);
    f.q = static_cast<const T*>(kv.q);
    f.R = static_cast<const T*>(kv.R);
    f.r = static_cast<const T*>(kv.r);
    f.A = static_cast<const T*>(kv.A);
    f.Bm = static_cast<const T*>(kv.B);
    f.e = static_cast<const T*>(kv.e);
    f.x_s = static_cast<const T*>(kv.x_s);
    f.x0 = static_cast<const T*>(kv.x0);
    f.lambda0 = static_cast<const T*>(lambda0);
    f.lambda_out = static_cast<T*>(lambda_out);
    f.errkey = errkey;
    f.out = outs_dev;
    f.trace = trace_dev;
    f.trace_cap = trace_cap;
    f.dz_out = static_cast<T*>(dz_dev);
    f.epsilon = cfg ? cfg->epsilon : 1e-4;
    const int mi = cfg ? cfg->max_iter : 0;
    f.max_iter = mi > 0 ? mi : static_cast<int>(D);
    fused_timing_begin();
    f.timing = env_int("B2P_PHASE_TIMING", 0)
                   ? static_cast<unsigned long long*>(ws_get(c, "fused_timing", 128ull * B))
                   : nullptr;
    c->timing = f.timing;
    c->timing_n = f.timing ? B : 0;
    CK(launch_small<T>(f, n, k->m, grid, st));
    c->launches++;
    c->last_path = 4;
    c->phases = time_it;
    if (time_it) CK(cudaEventRecord(c->ev1, st));
    return dz_dev != nullptr;
  }
  c->last_path = 0;
  T* S = static_cast<T*>(ws_get(c, tag + "S", sizeof(T) * B * K * 3 * nn));
  T* gamma = static_cast<T*>(ws_get(c, tag + "gamma", sizeof(T) * B * D));
  T* ti = static_cast<T*>(ws_get(c, tag + "ti", sizeof(T) * B * K * nn));
  if (time_it) {
    if (!c->accounting) c->pool_used = 0;
    if (c->pool_used + 3 > c->pool.size())
      for (int q = 0; q < 3; ++q) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        c->pool.push_back(e);
      }
    c->ev0 = c->pool[c->pool_used];
    c->ev2 = c->pool[c->pool_used + 1];
    c->ev1 = c->pool[c->pool_used + 2];
    c->pool_used += 3;
    CK(cudaEventRecord(c->ev0, st));
  }
  launch_form<T>(c, k, kv, B, S, gamma, ti, errkey, st);
  if (time_it) CK(cudaEventRecord(c->ev2, st));
  c->phases = time_it;
  PcgParams<T> p{};
  p.B = B;
  pcg_common(p, cfg, K, n);
  p.kind = kind;
  p.order = order;
  p.mode = kModeFused;
  p.S = S;
  p.Phi = nullptr;
  p.Tinv = ti;
  p.gamma = gamma;
  p.lambda0 = static_cast<const T*>(lambda0);
  p.lambda_out = static_cast<T*>(lambda_out);
  p.errkey = errkey;
  p.out = outs_dev;
  p.trace = trace_dev;
  p.trace_cap = trace_cap;
  configure_pcg(c, p, /*allow_grid=*/B == 1);
  const size_t Dall = D * B;
  p.best = static_cast<T*>(ws_get(c, tag + "best", sizeof(T) * Dall));
  p.pub = static_cast<T*>(ws_get(c, tag + "pub", sizeof(T) * Dall));
  p.slots = static_cast<T*>(ws_get(c, tag + "slots", sizeof(T) * 2 * p.G * B + 64));
  p.gbar = static_cast<unsigned*>(ws_get(c, tag + "gbar", 256));
  if (p.sync == kSyncGrid) CK(cudaMemsetAsync(p.gbar, 0, sizeof(unsigned), st));
  CK(launch_pcg<T>(p, st));
  c->launches++;
  if (time_it) CK(cudaEventRecord(c->ev1, st));
  return false;
}

void check_cfg(const b2p_pcg_config* cfg) {
  if (cfg && cfg->variant != B2P_SEQUENTIAL && cfg->variant != B2P_BLOCK_PARALLEL)
    throw invalid("b2p: unknown PCG variant");
}
void check_kind(int kind, int order) {
  if (kind < B2P_IDENTITY || kind > B2P_POLY_SPLIT)
    throw invalid("build_preconditioner: unknown kind");
  if (kind == B2P_POLY_SPLIT && order < 1)
    throw invalid("build_poly_split: order must be >= 1, got " + std::to_string(order));
}

// Per-system status words for device-resident callers (b2p.h
// b2p_solve_batched_device): {status, iterations, converged, aux} with aux =
// the knot of a non-PD formation error, the PCG iteration of a breakdown /
// non-finite error, else -1. Same decoding as resolve() / schur_msg() below.
__global__ void k_pack_status(const SysOut* __restrict__ outs, const int* __restrict__ keys, int B,
                              int32_t* __restrict__ st) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  const int key = keys[i];
  int32_t w[4];
  if (key < 0x7f7f7f7f) {
    const int b = key / 4, call = key % 4;
    w[0] = B2P_RUNTIME_ERROR;
    w[1] = 0;
    w[2] = 0;
    w[3] = b == 0 ? 0 : (call == 2 ? b : b - 1);
  } else {
    const SysOut o = outs[i];
    w[0] = o.code;
    w[1] = o.iterations;
    w[2] = o.converged;
    w[3] = o.code != kOk ? o.iteration : -1;
  }
  *reinterpret_cast<int4*>(st + 4 * static_cast<size_t>(i)) = make_int4(w[0], w[1], w[2], w[3]);
}

// Resolve per-system outcomes (host copies) into reports and a first error.
void resolve(const std::vector<SysOut>& outs, const std::vector<int>& errkeys, int B,
             b2p_solve_report* reports, double wall_each, Fail* first) {
  for (int i = 0; i < B; ++i) {
    SysOut o = outs[i];
    Fail f{B2P_OK, ""};
    if (!errkeys.empty() && errkeys[i] < kErrOk) {
      f.code = B2P_RUNTIME_ERROR;
      f.msg = schur_msg(errkeys[i], &f.knot);
      o = SysOut{};
      o.code = B2P_RUNTIME_ERROR;
    } else if (o.code != kOk) {
      f = pcg_fail(o);
    }
    if (reports) fill_report(reports + i, o, wall_each);
    if (f.code != B2P_OK && first->code == B2P_OK) {
      *first = f;
      first->system = i;
    }
  }
}

// ------------------------------------------------------------------ generator
// random_problem.cpp — host-side synthetic inputs (same draw order).
struct Rng {
  std::mt19937_64 g;
  explicit Rng(uint64_t s) : g(s) {}
  double u(double lo, double hi) {
    const double u01 = static_cast<double>(g() >> 11) * 0x1.0p-53;
    return lo + (hi - lo) * u01;
  }
  void mat(double* M, int r, int c, double lo, double hi) {
    for (int i = 0; i < r * c; ++i) M[i] = u(lo, hi);
  }
};

// Q = a * (L L') + floor*I  (p-ordered dot products)
void llt(const double* L, int n, double* Q, double scale_prod, double diag, double outer) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int p = 0; p < n; ++p) s += L[i * n + p] * L[j * n + p];
      double v = scale_prod * s;
      if (i == j) v += diag;
      Q[i * n + j] = outer * v;
    }
}

void generate_one(int family, uint64_t seed, int N, int n, int m, double fl, double cp,
                  b2p_kkt_out* o, size_t i) {
  Rng rng(seed);
  const size_t K = N + 1, nn = size_t(n) * n, mm = size_t(m) * m, nm = size_t(n) * m;
  double* Q = o->Q + i * K * nn;
  double* q = o->q + i * K * n;
  double* R = o->R + i * N * mm;
  double* r = o->r + i * N * m;
  double* A = o->A + i * N * nn;
  double* B = o->B + i * N * nm;
  double* e = o->e + i * N * n;
  std::vector<double> L(std::max(nn, mm));
  const bool traj = family == 2;
  const double cs = 2e-4;
  for (int k = 0; k < N; ++k) {
    rng.mat(L.data(), n, n, -1.0, 1.0);
    if (traj) llt(L.data(), n, Q + k * nn, 0.3, 1.0, cs);
    else llt(L.data(), n, Q + k * nn, 1.0, fl, 1.0);
    rng.mat(L.data(), m, m, -1.0, 1.0);
    if (traj) llt(L.data(), m, R + k * mm, 0.3, 1.0, cs);
    else llt(L.data(), m, R + k * mm, 1.0, fl, 1.0);
    double* Ak = A + k * nn;
    rng.mat(Ak, n, n, -1.0, 1.0);
    if (traj) {
      for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b)
          Ak[a * n + b] = (a == b ? 0.1 : 0.0) + Ak[a * n + b] * (0.02 / n);
    } else {
      for (size_t a = 0; a < nn; ++a) Ak[a] *= (cp / n);
    }
    double* Bk = B + k * nm;
    rng.mat(Bk, n, m, -1.0, 1.0);
    for (size_t a = 0; a < nm; ++a) Bk[a] *= (traj ? 1.0 / n : cp / n);
    rng.mat(q + k * n, 1, n, -1.0, 1.0);
    rng.mat(r + k * m, 1, m, -1.0, 1.0);
    rng.mat(e + k * n, 1, n, -1.0, 1.0);
  }
  rng.mat(L.data(), n, n, -1.0, 1.0);
  if (traj) llt(L.data(), n, Q + N * nn, 0.3, 1.0, cs);
  else llt(L.data(), n, Q + N * nn, 1.0, fl, 1.0);
  rng.mat(q + N * n, 1, n, -1.0, 1.0);
  rng.mat(o->x_s + i * n, 1, n, -1.0, 1.0);
  for (int a = 0; a < n; ++a) o->x0[i * n + a] = 0.0;
}

}  // namespace

// ======================================================================= C-ABI
extern "C" {

int b2p_abi_version(void) { return B2P_ABI_VERSION; }

int b2p_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int b2p_ctx_create(int device, b2p_ctx** out, b2p_error* err) {
  return guard(err, [&] {
    if (!out) throw invalid("b2p_ctx_create: null out");
    *out = nullptr;
    int ndev = b2p_device_count();
    if (ndev <= 0) throw Fail{B2P_CUDA_ERROR, "b2p: no CUDA device visible"};
    if (device < 0 || device >= ndev) throw invalid("b2p_ctx_create: bad device index");
    CK(cudaSetDevice(device));
    auto* c = new b2p_ctx();
    c->device = device;
    CK(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
    for (int q = 0; q < 3; ++q) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      c->pool.push_back(e);
    }
    c->ev0 = c->pool[0];
    c->ev2 = c->pool[1];
    c->ev1 = c->pool[2];
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    c->sm_count = prop.multiProcessorCount;
    c->smem_optin = prop.sharedMemPerBlockOptin;
    *out = c;
  });
}

void b2p_ctx_destroy(b2p_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->own);
  cudaStreamSynchronize(c->aux);
  for (auto& kv : c->ws)
    if (kv.second.first) cudaFree(kv.second.first);
  for (auto& kv : c->hws)
    if (kv.second.first) cudaFreeHost(kv.second.first);
  for (cudaEvent_t e : c->pool) cudaEventDestroy(e);
  cudaStreamDestroy(c->own);
  cudaStreamDestroy(c->aux);
  delete c;
}

int b2p_ctx_set_stream(b2p_ctx* c, void* stream) {
  if (!c) return B2P_INVALID_ARGUMENT;
  c->user = static_cast<cudaStream_t>(stream);
  return B2P_OK;
}
void* b2p_ctx_stream(b2p_ctx* c) { return c ? static_cast<void*>(c->stream()) : nullptr; }
long long b2p_ctx_kernel_launches(b2p_ctx* c) { return c ? c->launches.load() : 0; }
int b2p_ctx_last_path(b2p_ctx* c) { return c ? c->last_path : -1; }

// Debug: copy the per-system globaltimer stamps of the last one-CTA fused
// solve (B2P_PHASE_TIMING=1): [n][8] = start, F1 end, F2 end, staging end, end.
int b2p_ctx_phase_stamps(b2p_ctx* c, unsigned long long* out, int n) {
  if (!c || !out || !c->timing) return B2P_INVALID_ARGUMENT;
  cudaSetDevice(c->device);
  const int m = std::min(n, c->timing_n);
  if (cudaMemcpy(out, c->timing, sizeof(unsigned long long) * 16 * m, cudaMemcpyDeviceToHost) !=
      cudaSuccess)
    return B2P_CUDA_ERROR;
  return m;
}
int b2p_ctx_last_phase_ms(b2p_ctx* c, float* ms, int n) {
  if (!c || !ms || n < 2) return B2P_INVALID_ARGUMENT;
  ms[0] = ms[1] = 0.f;
  if (!c->phases) return B2P_OK;
  cudaSetDevice(c->device);
  if (cudaEventElapsedTime(&ms[0], c->ev0, c->ev2) != cudaSuccess ||
      cudaEventElapsedTime(&ms[1], c->ev2, c->ev1) != cudaSuccess) {
    cudaGetLastError();
    return B2P_CUDA_ERROR;
  }
  return B2P_OK;
}

int b2p_ctx_phase_accounting(b2p_ctx* c, int enable) {
  if (!c) return B2P_INVALID_ARGUMENT;
  c->accounting = enable != 0;
  c->pool_used = 0;
  return B2P_OK;
}

int b2p_ctx_phase_totals(b2p_ctx* c, float* ms, int n, int* count) {
  if (!c || !ms || n < 3) return B2P_INVALID_ARGUMENT;
  cudaSetDevice(c->device);
  ms[0] = ms[1] = ms[2] = 0.f;
  const size_t used = c->pool_used;
  if (count) *count = static_cast<int>(used / 3);
  for (size_t t = 0; t + 2 < used; t += 3) {
    float a = 0.f, b = 0.f;
    if (cudaEventSynchronize(c->pool[t + 2]) != cudaSuccess ||
        cudaEventElapsedTime(&a, c->pool[t], c->pool[t + 1]) != cudaSuccess ||
        cudaEventElapsedTime(&b, c->pool[t + 1], c->pool[t + 2]) != cudaSuccess) {
      cudaGetLastError();
      return B2P_CUDA_ERROR;
    }
    ms[0] += a;
    ms[1] += b;
    ms[2] += a + b;
  }
  c->pool_used = 0;
  return B2P_OK;
}

int b2p_ctx_last_solve_ms(b2p_ctx* c, float* ms) {
  if (!c || !ms) return B2P_INVALID_ARGUMENT;
  *ms = c->last_ms;
  return B2P_OK;
}

int b2p_ctx_last_h2d_bytes(b2p_ctx* c, unsigned long long* bytes) {
  if (!c || !bytes) return B2P_INVALID_ARGUMENT;
  *bytes = static_cast<unsigned long long>(c->last_h2d_bytes);
  return B2P_OK;
}

// ---------------------------------------------------------------- block_tri
int b2p_blocktri_matvec(b2p_ctx* c, int dtype, int K, int nb, const void* M, const void* x,
                        int x_len, void* y, b2p_error* err) {
  return guard(err, [&] {
    check_dtype(dtype);
    check_blocktri(K, nb);
    if (x_len != K * nb)
      throw invalid("BlockTriMatrix matvec: expected vector of length " + std::to_string(K * nb) +
                    ", got " + std::to_string(x_len));
    check_ctx(c);
    const size_t es = esize(dtype), nn = size_t(nb) * nb, D = size_t(K) * nb;
    cudaStream_t st = c->stream();
    char* dM = static_cast<char*>(ws_get(c, "mv_M", es * K * 3 * nn));
    char* dx = static_cast<char*>(ws_get(c, "mv_x", es * D));
    char* dy = static_cast<char*>(ws_get(c, "mv_y", es * D));
    h2d(c, dM, M, es * K * 3 * nn, st);
    h2d(c, dx, x, es * D, st);
    if (dtype == B2P_F64)
      CK(launch_blocktri_matvec<double>(1, K, nb, (double*)dM, (double*)dx, (double*)dy, 0,
                                        nullptr, nullptr, st));
    else
      CK(launch_blocktri_matvec<float>(1, K, nb, (float*)dM, (float*)dx, (float*)dy, 0, nullptr,
                                       nullptr, st));
    c->launches++;
    d2h(c, y, dy, es * D, st);
    CK(cudaStreamSynchronize(st));
  });
}

int b2p_blocktri_cholesky_solve(b2p_ctx* c, int dtype, int K, int nb, const void* M,
                                const void* rhs, int rhs_len, void* x, b2p_error* err) {
  return guard(err, [&] {
    check_dtype(dtype);
    check_blocktri(K, nb);
    if (rhs_len != K * nb)
      throw invalid("BlockTriMatrix cholesky_solve: expected vector of length " +
                    std::to_string(K * nb) + ", got " + std::to_string(rhs_len));
    check_ctx(c);
    const size_t es = esize(dtype), nn = size_t(nb) * nb, D = size_t(K) * nb;
    cudaStream_t st = c->stream();
    char* dM = static_cast<char*>(ws_get(c, "ch_M", es * K * 3 * nn));
    char* db = static_cast<char*>(ws_get(c, "ch_b", es * D));
    char* dx = static_cast<char*>(ws_get(c, "ch_x", es * D));
    char* dy = static_cast<char*>(ws_get(c, "ch_y", es * D));
    char* dF = static_cast<char*>(ws_get(c, "ch_F", es * K * nn));
    int* dst = static_cast<int*>(ws_get(c, "ch_st", sizeof(int)));
    h2d(c, dM, M, es * K * 3 * nn, st);
    h2d(c, db, rhs, es * D, st);
    if (dtype == B2P_F64)
      CK(launch_block_cholesky<double>(1, K, nb, (double*)dM, (double*)db, (double*)dx, (double*)dF,
                                       (double*)dy, dst, st));
    else
      CK(launch_block_cholesky<float>(1, K, nb, (float*)dM, (float*)db, (float*)dx, (float*)dF,
                                      (float*)dy, dst, st));
    c->launches++;
    int status = 0;
    d2h(c, &status, dst, sizeof(int), st);
    d2h(c, x, dx, es * D, st);
    CK(cudaStreamSynchronize(st));
    if (status >= 0)
      throw Fail{B2P_RUNTIME_ERROR, "BlockTriMatrix cholesky_solve: block " +
                                        std::to_string(status) + " is not positive definite"};
  });
}

int b2p_blocktri_check(b2p_ctx* c, int dtype, int K, int nb, const void* M, double* asym,
                       double* mabs, b2p_error* err) {
  return guard(err, [&] {
    check_dtype(dtype);
    check_blocktri(K, nb);
    check_ctx(c);
    const size_t es = esize(dtype), nn = size_t(nb) * nb;
    cudaStream_t st = c->stream();
    char* dM = static_cast<char*>(ws_get(c, "ck_M", es * K * 3 * nn));
    double* d2 = static_cast<double*>(ws_get(c, "ck_out", 2 * sizeof(double)));
    h2d(c, dM, M, es * K * 3 * nn, st);
    CK(cudaMemsetAsync(d2, 0, 2 * sizeof(double), st));
    if (dtype == B2P_F64) CK(launch_blocktri_check<double>(K, nb, (double*)dM, d2, st));
    else CK(launch_blocktri_check<float>(K, nb, (float*)dM, d2, st));
    c->launches++;
    double h[2];
    d2h(c, h, d2, sizeof(h), st);
    CK(cudaStreamSynchronize(st));
    if (asym) *asym = h[0];
    if (mabs) *mabs = h[1];
  });
}

// ---------------------------------------------------------------- schur
int b2p_build_schur(b2p_ctx* c, int dtype, const b2p_kkt* k, void* S, void* gamma,
                    void* theta_inv, b2p_error* err) {
  NvtxRange nvtx_("b2p_build_schur");
  return guard(err, [&] {
    check_dtype(dtype);
    check_kkt(k);
    check_ctx(c);
    const size_t es = esize(dtype);
    const int K = k->N + 1, n = k->n;
    const size_t nn = size_t(n) * n, D = size_t(K) * n;
    cudaStream_t st = c->stream();
    void* in = ws_get(c, "bs_in", kkt_block_bytes(k, es, 1));
    const KktDev kv = upload_kkt(c, k, es, 0, 1, in, st);
    // outputs in one device block -> one copy back: [key | S | gamma | theta^-1]
    const size_t bS = es * K * 3 * nn, bg = es * D, bt = es * K * nn;
    const size_t oS = 256, og = oS + (bS + 255) / 256 * 256, ot = og + (bg + 255) / 256 * 256;
    const size_t obytes = ot + bt;
    char* dob = static_cast<char*>(ws_get(c, "bs_ob", obytes));
    char* hob = static_cast<char*>(hws_get(c, "bs_hob", obytes));
    char *dS = dob + oS, *dg = dob + og, *dt = dob + ot;
    int* ek = reinterpret_cast<int*>(dob);
    if (dtype == B2P_F64) launch_form<double>(c, k, kv, 1, (double*)dS, (double*)dg, (double*)dt, ek, st);
    else launch_form<float>(c, k, kv, 1, (float*)dS, (float*)dg, (float*)dt, ek, st);
    d2h(c, hob, dob, obytes, st);
    CK(cudaStreamSynchronize(st));
    int key = 0;
    std::memcpy(&key, hob, sizeof(int));
    std::memcpy(S, hob + oS, bS);
    std::memcpy(gamma, hob + og, bg);
    std::memcpy(theta_inv, hob + ot, bt);
    if (key < kErrOk) {
      Fail f{B2P_RUNTIME_ERROR, schur_msg(key, nullptr)};
      schur_msg(key, &f.knot);
      throw f;
    }
  });
}

int b2p_stair_matrix(b2p_ctx* c, int dtype, int K, int nb, const void* S, void* psi,
                     b2p_error* err) {
  return guard(err, [&] {
    check_dtype(dtype);
    check_blocktri(K, nb);
    check_ctx(c);
    const size_t es = esize(dtype), bytes = es * K * 3 * size_t(nb) * nb;
    cudaStream_t st = c->stream();
    char* dS = static_cast<char*>(ws_get(c, "sm_S", bytes));
    char* dP = static_cast<char*>(ws_get(c, "sm_P", bytes));
    h2d(c, dS, S, bytes, st);
    if (dtype == B2P_F64) CK(launch_stair_matrix<double>(K, nb, (double*)dS, (double*)dP, st));
    else CK(launch_stair_matrix<float>(K, nb, (float*)dS, (float*)dP, st));
    c->launches++;
    d2h(c, psi, dP, bytes, st);
    CK(cudaStreamSynchronize(st));
  });
}

int b2p_build_preconditioner(b2p_ctx* c, int dtype, int kind, int order, int K, int nb,
                             const void* S, const void* theta_inv, void* phi_inv,
                             b2p_error* err) {
  NvtxRange nvtx_("b2p_build_preconditioner");
  return guard(err, [&] {
    check_dtype(dtype);
    check_kind(kind, order);
    if (kind == B2P_IDENTITY) return;  // build_identity: empty phi_inv
    check_blocktri(K, nb);
    check_ctx(c);
    const size_t es = esize(dtype), nn = size_t(nb) * nb;
    cudaStream_t st = c->stream();
    // [S | theta^-1] in one pinned staging block, one copy each way
    const size_t bS = es * K * 3 * nn, bt = es * K * nn, it = (bS + 255) / 256 * 256;
    char* din = static_cast<char*>(ws_get(c, "bp_in", it + bt));
    char* hin = static_cast<char*>(hws_get(c, "bp_hin", it + bt));
    std::memcpy(hin, S, bS);
    std::memcpy(hin + it, theta_inv, bt);
    h2d(c, din, hin, it + bt, st);
    char* dS = din;
    char* dt = din + it;
    char* dP = static_cast<char*>(ws_get(c, "bp_P", bS));
    char* hP = static_cast<char*>(hws_get(c, "bp_hP", bS));
    if (dtype == B2P_F64) {
      PrecondParams<double> p{1, K, nb, kind, (double*)dS, (double*)dt, (double*)dP};
      CK(launch_build_precond<double>(p, st));
    } else {
      PrecondParams<float> p{1, K, nb, kind, (float*)dS, (float*)dt, (float*)dP};
      CK(launch_build_precond<float>(p, st));
    }
    c->launches++;
    d2h(c, hP, dP, bS, st);
    CK(cudaStreamSynchronize(st));
    std::memcpy(phi_inv, hP, bS);
  });
}

int b2p_apply_preconditioner(b2p_ctx* c, int dtype, int kind, int order, int K, int nb,
                             const void* S, const void* phi_inv, const void* r, int r_len,
                             void* out, b2p_error* err) {
  NvtxRange nvtx_("b2p_apply_preconditioner");
  return guard(err, [&] {
    check_dtype(dtype);
    check_kind(kind, order);
    const size_t es = esize(dtype);
    if (kind == B2P_IDENTITY) {  // returns r unchanged (schur.cpp:176-178)
      std::memcpy(out, r, es * r_len);
      return;
    }
    check_blocktri(K, nb);
    if (r_len != K * nb)
      throw invalid("apply_preconditioner: expected vector of length " + std::to_string(K * nb) +
                    ", got " + std::to_string(r_len));
    check_ctx(c);
    const size_t nn = size_t(nb) * nb, D = size_t(K) * nb;
    cudaStream_t st = c->stream();
    char* dP = static_cast<char*>(ws_get(c, "ap_P", es * K * 3 * nn));
    char* dr = static_cast<char*>(ws_get(c, "ap_r", es * D));
    char* dacc = static_cast<char*>(ws_get(c, "ap_acc", es * D));
    h2d(c, dP, phi_inv, es * K * 3 * nn, st);
    h2d(c, dr, r, es * D, st);
    auto mv = [&](const void* M, const void* x, void* y, int mode, const void* add, void* acc) {
      if (dtype == B2P_F64)
        CK(launch_blocktri_matvec<double>(1, K, nb, (const double*)M, (const double*)x,
                                          (double*)y, mode, (const double*)add, (double*)acc, st));
      else
        CK(launch_blocktri_matvec<float>(1, K, nb, (const float*)M, (const float*)x, (float*)y,
                                         mode, (const float*)add, (float*)acc, st));
      c->launches++;
    };
    if (kind != B2P_POLY_SPLIT) {
      mv(dP, dr, dacc, 0, nullptr, nullptr);
    } else {
      char* dS = static_cast<char*>(ws_get(c, "ap_S", es * K * 3 * nn));
      char* dterm = static_cast<char*>(ws_get(c, "ap_term", es * D));
      char* ds = static_cast<char*>(ws_get(c, "ap_s", es * D));
      char* dacc2 = static_cast<char*>(ws_get(c, "ap_acc2", es * D));
      h2d(c, dS, S, es * K * 3 * nn, st);
      mv(dP, dr, dterm, 0, nullptr, nullptr);  // term = Phi r
      CK(cudaMemcpyAsync(dacc, dterm, es * D, cudaMemcpyDeviceToDevice, st));
      for (int j = 0; j < order; ++j) {
        mv(dS, dterm, ds, 1, nullptr, nullptr);  // s = E term
        mv(dP, ds, dterm, 0, dacc, dacc2);       // term = Phi s; acc2 = acc + term
        std::swap(dacc, dacc2);
      }
    }
    d2h(c, out, dacc, es * D, st);
    CK(cudaStreamSynchronize(st));
  });
}

// ---------------------------------------------------------------- pcg
int b2p_pcg_solve(b2p_ctx* c, int dtype, int K, int nb, const void* S, int kind, int order,
                  int phi_K, int phi_nb, const void* phi_inv, const void* gamma, int gamma_len,
                  const void* lambda0, int lambda0_len, const b2p_pcg_config* cfg,
                  void* lambda_out, b2p_solve_report* report, double* trace, b2p_error* err) {
  NvtxRange nvtx_("b2p_pcg_solve");
  return guard(err, [&] {
    check_dtype(dtype);
    check_cfg(cfg);
    // validate_inputs (pcg.cpp:24-47)
    if (K <= 0) throw invalid("pcg: empty system matrix");
    const int dim = K * nb;
    if (gamma_len != dim)
      throw invalid("pcg: expected gamma of length " + std::to_string(dim) + ", got " +
                    std::to_string(gamma_len));
    if (lambda0_len != dim)
      throw invalid("pcg: expected lambda0 of length " + std::to_string(dim) + ", got " +
                    std::to_string(lambda0_len));
    check_kind(kind, order);
    if (kind != B2P_IDENTITY && phi_K * phi_nb != dim)
      throw invalid("pcg: preconditioner dimension " + std::to_string(phi_K * phi_nb) +
                    " does not match system " + std::to_string(dim));
    if (kind != B2P_IDENTITY && phi_nb != nb)
      throw invalid("b2p: preconditioner block_dim must match S");
    check_blocktri(K, nb);
    check_ctx(c);
    const size_t es = esize(dtype), nn = size_t(nb) * nb, D = size_t(dim);
    cudaStream_t st = c->stream();
    // Inputs [S | Phi | gamma | lambda0] packed into one pinned staging block and
    // sent with one copy; outputs [check | SysOut | lambda] back with one copy.
    const size_t bS = es * K * 3 * nn, bP = kind != B2P_IDENTITY ? bS : 0, bv = es * D;
    auto up = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t iP = up(bS), ig = iP + up(bP), il0 = ig + up(bv), ibytes = il0 + bv;
    char* din = static_cast<char*>(ws_get(c, "pc_in", ibytes));
    char* hin = static_cast<char*>(hws_get(c, "pc_hin", ibytes));
    std::memcpy(hin, S, bS);
    if (bP) std::memcpy(hin + iP, phi_inv, bP);
    std::memcpy(hin + ig, gamma, bv);
    std::memcpy(hin + il0, lambda0, bv);
    h2d(c, din, hin, ibytes, st);
    char* dS = din;
    char* dP = bP ? din + iP : nullptr;
    char* dg = din + ig;
    char* dl0 = din + il0;
    const size_t oOut = 256, oL = 512, obytes = oL + bv;
    char* dob = static_cast<char*>(ws_get(c, "pc_ob", obytes));
    char* hob = static_cast<char*>(hws_get(c, "pc_hob", obytes));
    char* dl = dob + oL;
    SysOut* dout = reinterpret_cast<SysOut*>(dob + oOut);
    // asymmetry check on device (validate_inputs :42-46); evaluated after the
    // solve's single synchronisation, and reported first, as the reference's
    // validation precedes the solve
    double* d2 = reinterpret_cast<double*>(dob);
    CK(cudaMemsetAsync(d2, 0, 2 * sizeof(double), st));
    if (dtype == B2P_F64) CK(launch_blocktri_check<double>(K, nb, (double*)dS, d2, st));
    else CK(launch_blocktri_check<float>(K, nb, (float*)dS, d2, st));
    c->launches++;
    int trace_cap = 0;
    double* dtr = nullptr;
    const int mi = (cfg && cfg->max_iter > 0) ? cfg->max_iter : dim;
    if (trace && cfg && cfg->collect_trace) {
      trace_cap = mi;
      dtr = static_cast<double*>(ws_get(c, "pc_tr", sizeof(double) * trace_cap));
    }
    auto go = [&](auto tag) {
      using T = decltype(tag);
      PcgParams<T> p{};
      p.B = 1;
      pcg_common(p, cfg, K, nb);
      p.kind = kind;
      p.order = order;
      p.mode = kModeExplicit;
      p.S = (const T*)dS;
      p.Phi = (const T*)dP;
      p.Tinv = nullptr;
      p.gamma = (const T*)dg;
      p.lambda0 = (const T*)dl0;
      p.lambda_out = (T*)dl;
      p.errkey = nullptr;
      p.out = dout;
      p.trace = dtr;
      p.trace_cap = trace_cap;
      configure_pcg(c, p, true);
      run_pcg<T>(c, p, st, true);
    };
    if (dtype == B2P_F64) go(double{});
    else go(float{});
    d2h(c, hob, dob, obytes, st);
    CK(cudaStreamSynchronize(st));
    CK(cudaEventElapsedTime(&c->last_ms, c->ev0, c->ev1));
    double ck[2];
    std::memcpy(ck, hob, sizeof(ck));
    if (ck[0] > 1e-9 * std::max(1.0, ck[1]))
      throw invalid("pcg: S is not structurally symmetric (asymmetry " + fstr(ck[0]) + ")");
    SysOut o;
    std::memcpy(&o, hob + oOut, sizeof(SysOut));
    if (o.code != kOk) throw pcg_fail(o);
    std::memcpy(lambda_out, hob + oL, bv);
    if (dtr && o.trace_len > 0) CK(cudaMemcpy(trace, dtr, sizeof(double) * o.trace_len,
                                             cudaMemcpyDeviceToHost));
    fill_report(report, o, c->last_ms * 1e-3);
  });
}

// ---------------------------------------------------------------- fused
}  // extern "C"
namespace {
template <class T>
void primal_impl(b2p_ctx* c, int B, const b2p_kkt* k, const KktDev& kv, const void* lam, void* dz,
                 cudaStream_t st);

int solve_one(b2p_ctx* c, int dtype, const b2p_kkt* k, int kind, int order,
              const b2p_pcg_config* cfg, const void* lambda0, void* lambda_out, void* dz_out,
              b2p_solve_report* report, double* trace, b2p_error* err) {
  return guard(err, [&] {
    check_dtype(dtype);
    check_kkt(k);
    check_kind(kind, order);
    check_cfg(cfg);
    check_ctx(c);
    const size_t es = esize(dtype);
    const int K = k->N + 1, n = k->n;
    const size_t D = size_t(K) * n;
    cudaStream_t st = c->stream();
    const size_t l0b = lambda0 ? es * D : 0;
    void* in = ws_get(c, "sv_in", kkt_block_bytes(k, es, 1) + l0b);
    char* dl0 = nullptr;
    const KktDev kv = upload_kkt(c, k, es, 0, 1, in, st, lambda0, l0b, &dl0);
    // Outputs in one device block -> one copy back: [SysOut | key | lambda | dz].
    const size_t P = static_cast<size_t>(K) * n + static_cast<size_t>(k->N) * k->m;
    const size_t oKey = 256, oL = 512, oDz = oL + (es * D + 255) / 256 * 256;
    const size_t obytes = dz_out ? oDz + es * P : oL + es * D;
    char* dob = static_cast<char*>(ws_get(c, "sv_ob", obytes));
    char* hob = static_cast<char*>(hws_get(c, "sv_hob", obytes));
    char* dl = dob + oL;
    SysOut* dout = reinterpret_cast<SysOut*>(dob);
    int* ek = reinterpret_cast<int*>(dob + oKey);
    static_assert(sizeof(SysOut) <= 256, "SysOut slot");
    const int mi = (cfg && cfg->max_iter > 0) ? cfg->max_iter : int(D);
    double* dtr = nullptr;
    if (trace && cfg && cfg->collect_trace)
      dtr = static_cast<double*>(ws_get(c, "sv_tr", sizeof(double) * mi));
    // the one-CTA / small-block kernels run reconstruct_primal in their
    // epilogue (one launch for the whole SQP linear step); other paths launch
    // the primal kernel after the solve
    bool dz_done;
    if (dtype == B2P_F64)
      dz_done = solve_device_impl<double>(c, k, kv, 1, kind, order, cfg, dl0, dl, dout, ek, dtr,
                                          mi, st, true, "sv_", dz_out ? dob + oDz : nullptr);
    else
      dz_done = solve_device_impl<float>(c, k, kv, 1, kind, order, cfg, dl0, dl, dout, ek, dtr,
                                         mi, st, true, "sv_", dz_out ? dob + oDz : nullptr);
    if (dz_out && !dz_done) {
      // reconstruct_primal on the resident knots and multipliers. If the solve
      // failed, dz is never handed back.
      if (dtype == B2P_F64)
        primal_impl<double>(c, 1, k, kv, dl, dob + oDz, st);
      else
        primal_impl<float>(c, 1, k, kv, dl, dob + oDz, st);
    }
    d2h(c, hob, dob, obytes, st);
    CK(cudaStreamSynchronize(st));
    CK(cudaEventElapsedTime(&c->last_ms, c->ev0, c->ev1));
    SysOut o;
    int key = 0;
    std::memcpy(&o, hob, sizeof(o));
    std::memcpy(&key, hob + oKey, sizeof(int));
    std::memcpy(lambda_out, hob + oL, es * D);
    Fail first{B2P_OK, ""};
    resolve({o}, {key}, 1, report, c->last_ms * 1e-3, &first);
    if (first.code != B2P_OK) {
      first.system = -1;
      throw first;
    }
    if (dz_out) std::memcpy(dz_out, hob + oDz, es * P);
    if (dtr && o.trace_len > 0)
      CK(cudaMemcpy(trace, dtr, sizeof(double) * o.trace_len, cudaMemcpyDeviceToHost));
  });
}
}  // namespace
extern "C" {

int b2p_solve(b2p_ctx* c, int dtype, const b2p_kkt* k, int kind, int order,
              const b2p_pcg_config* cfg, const void* lambda0, void* lambda_out,
              b2p_solve_report* report, double* trace, b2p_error* err) {
  NvtxRange nvtx_("b2p_solve");
  return solve_one(c, dtype, k, kind, order, cfg, lambda0, lambda_out, nullptr, report, trace,
                   err);
}

int b2p_sqp_step(b2p_ctx* c, int dtype, const b2p_kkt* k, int kind, int order,
                 const b2p_pcg_config* cfg, const void* lambda0, void* lambda_out, void* dz_out,
                 b2p_solve_report* report, double* trace, b2p_error* err) {
  if (!dz_out) return guard(err, [] { throw invalid("sqp_step: null dz buffer"); });
  NvtxRange nvtx_("b2p_sqp_step");
  return solve_one(c, dtype, k, kind, order, cfg, lambda0, lambda_out, dz_out, report, trace,
                   err);
}

// ------------------------------------------------------------------ reconstruct_primal
}  // extern "C"
namespace {
template <class T>
void primal_impl(b2p_ctx* c, int B, const b2p_kkt* k, const KktDev& kv, const void* lam, void* dz,
                 cudaStream_t st) {
  PrimalParams<T> p{};
  p.B = B;
  p.N = k->N;
  p.n = k->n;
  p.m = k->m;
  p.Q = static_cast<const T*>(kv.Q);
  p.q = static_cast<const T*>(kv.q);
  p.R = static_cast<const T*>(kv.R);
  p.r = static_cast<const T*>(kv.r);
  p.A = static_cast<const T*>(kv.A);
  p.B_ = static_cast<const T*>(kv.B);
  p.lambda = static_cast<const T*>(lam);
  p.dz = static_cast<T*>(dz);
  CK(launch_reconstruct_primal<T>(p, st));
  c->launches++;
}
}  // namespace
extern "C" {

int b2p_reconstruct_primal(b2p_ctx* c, int dtype, const b2p_kkt* k, const void* lambda,
                           int lambda_len, void* dz_out, b2p_error* err) {
  NvtxRange nvtx_("b2p_reconstruct_primal");
  return guard(err, [&] {
    check_dtype(dtype);
    check_kkt(k);
    check_ctx(c);
    const int D = (k->N + 1) * k->n;
    if (lambda_len != D)
      throw invalid("reconstruct_primal: expected lambda of length " + std::to_string(D) +
                    ", got " + std::to_string(lambda_len));
    if (!lambda || !dz_out) throw invalid("reconstruct_primal: null buffer");
    const size_t es = esize(dtype);
    const size_t P = static_cast<size_t>(k->N + 1) * k->n + static_cast<size_t>(k->N) * k->m;
    cudaStream_t st = c->stream();
    void* in = ws_get(c, "rp_in", kkt_block_bytes(k, es, 1) + es * D);
    char* dl = nullptr;
    const KktDev kv = upload_kkt(c, k, es, 0, 1, in, st, lambda, es * D, &dl);
    void* dd = ws_get(c, "rp_dz", es * P);
    void* hd = hws_get(c, "rp_hdz", es * P);
    if (dtype == B2P_F64)
      primal_impl<double>(c, 1, k, kv, dl, dd, st);
    else
      primal_impl<float>(c, 1, k, kv, dl, dd, st);
    d2h(c, hd, dd, es * P, st);
    CK(cudaStreamSynchronize(st));
    std::memcpy(dz_out, hd, es * P);
  });
}

int b2p_direct_solve_batched_device(b2p_ctx* c, int dtype, int batch, const b2p_kkt* kd,
                                    void* lambda_dev, int* status_dev, b2p_error* err) {
  NvtxRange nvtx_("b2p_direct_solve_batched_device");
  return guard(err, [&] {
    check_dtype(dtype);
    check_kkt(kd);
    check_ctx(c);
    if (batch < 1) throw invalid("direct_solve: batch must be >= 1");
    if (!lambda_dev || !status_dev) throw invalid("direct_solve: null buffer");
    const KktDev kv = dev_view(kd);
    const int K = kd->N + 1, n = kd->n;
    const size_t es = esize(dtype), nn = size_t(n) * n, D = size_t(K) * n, B = batch;
    cudaStream_t st = c->stream();
    void* S = ws_get(c, "ds_S", es * B * K * 3 * nn);
    void* g = ws_get(c, "ds_g", es * B * D);
    void* ti = ws_get(c, "ds_t", es * B * K * nn);
    void* F = ws_get(c, "ds_F", es * B * K * nn);
    void* y = ws_get(c, "ds_y", es * B * D);
    int* ek = static_cast<int*>(ws_get(c, "ds_ek", sizeof(int) * B));
    if (dtype == B2P_F64) {
      launch_form<double>(c, kd, kv, batch, (double*)S, (double*)g, (double*)ti, ek, st);
      CK(launch_block_cholesky<double>(batch, K, n, (double*)S, (double*)g, (double*)lambda_dev,
                                       (double*)F, (double*)y, status_dev, st));
    } else {
      launch_form<float>(c, kd, kv, batch, (float*)S, (float*)g, (float*)ti, ek, st);
      CK(launch_block_cholesky<float>(batch, K, n, (float*)S, (float*)g, (float*)lambda_dev,
                                      (float*)F, (float*)y, status_dev, st));
    }
    c->launches++;
  });
}

int b2p_reconstruct_primal_batched_device(b2p_ctx* c, int dtype, int batch, const b2p_kkt* kd,
                                          const void* lambda_dev, void* dz_dev, b2p_error* err) {
  NvtxRange nvtx_("b2p_reconstruct_primal_batched_device");
  return guard(err, [&] {
    check_dtype(dtype);
    check_kkt(kd);
    check_ctx(c);
    if (batch < 1) throw invalid("reconstruct_primal: batch must be >= 1");
    if (!lambda_dev || !dz_dev) throw invalid("reconstruct_primal: null buffer");
    const KktDev kv = dev_view(kd);
    if (dtype == B2P_F64)
      primal_impl<double>(c, batch, kd, kv, lambda_dev, dz_dev, c->stream());
    else
      primal_impl<float>(c, batch, kd, kv, lambda_dev, dz_dev, c->stream());
  });
}

int b2p_solve_batched_device(b2p_ctx* c, int dtype, int batch, const b2p_kkt* kd, int kind,
                             int order, const b2p_pcg_config* cfg, const void* lambda0_dev,
                             void* lambda_out_dev, b2p_solve_report* reports, int32_t* status_dev,
                             b2p_error* err) {
  NvtxRange nvtx_("b2p_solve_batched_device");
  return guard(err, [&] {
    check_dtype(dtype);
    check_kkt(kd);
    check_kind(kind, order);
    check_cfg(cfg);
    check_ctx(c);
    if (batch < 1) throw invalid("b2p_solve_batched: batch must be >= 1");
    cudaStream_t st = c->stream();
    SysOut* dout = static_cast<SysOut*>(ws_get(c, "bd_out", sizeof(SysOut) * batch));
    int* ek = static_cast<int*>(ws_get(c, "bd_ek", sizeof(int) * batch));
    const KktDev kv = dev_view(kd);
    if (dtype == B2P_F64)
      solve_device_impl<double>(c, kd, kv, batch, kind, order, cfg, lambda0_dev, lambda_out_dev,
                                dout, ek, nullptr, 0, st, true, "bd_");
    else
      solve_device_impl<float>(c, kd, kv, batch, kind, order, cfg, lambda0_dev, lambda_out_dev,
                               dout, ek, nullptr, 0, st, true, "bd_");
    if (status_dev) {
      if (reinterpret_cast<uintptr_t>(status_dev) % 16)
        throw invalid("b2p_solve_batched_device: status_dev must be 16-byte aligned");
      k_pack_status<<<(batch + 255) / 256, 256, 0, st>>>(dout, ek, batch, status_dev);
      CK(cudaGetLastError());
      c->launches++;
    }
    if (reports) {
      std::vector<SysOut> outs(batch);
      std::vector<int> keys(batch);
      d2h(c, outs.data(), dout, sizeof(SysOut) * batch, st);
      d2h(c, keys.data(), ek, sizeof(int) * batch, st);
      CK(cudaStreamSynchronize(st));
      CK(cudaEventElapsedTime(&c->last_ms, c->ev0, c->ev1));
      Fail first{B2P_OK, ""};
      resolve(outs, keys, batch, reports, c->last_ms * 1e-3 / batch, &first);
      if (first.code != B2P_OK) throw first;
    }
  });
}

// Host-buffer batched solve: chunks of systems alternate between two
// streams so the H2D copy of chunk c+1 overlaps the kernels of chunk c.
int b2p_solve_batched(b2p_ctx* c, int dtype, int batch, const b2p_kkt* k, int kind, int order,
                      const b2p_pcg_config* cfg, const void* lambda0, void* lambda_out,
                      b2p_solve_report* reports, b2p_error* err) {
  NvtxRange nvtx_("b2p_solve_batched");
  return guard(err, [&] {
    check_dtype(dtype);
    check_kkt(k);
    check_kind(kind, order);
    check_cfg(cfg);
    check_ctx(c);
    if (batch < 1) throw invalid("b2p_solve_batched: batch must be >= 1");
    const size_t es = esize(dtype);
    const int K = k->N + 1, n = k->n;
    const size_t D = size_t(K) * n;
    const int chunk = std::min(batch, std::max(1, env_int("B2P_BATCH_CHUNK", 512)));
    const int nchunks = (batch + chunk - 1) / chunk;
    cudaStream_t streams[2] = {c->stream(), c->aux};
    // per-system status words land in pinned staging (asynchronous D2H); so
    // does lambda when the caller's buffer is pageable
    SysOut* h_outs = static_cast<SysOut*>(hws_get(c, "bh_outs", sizeof(SysOut) * batch));
    int* h_keys = static_cast<int*>(hws_get(c, "bh_keys", sizeof(int) * batch));
    const bool lam_pinned = is_pinned(lambda_out);
    char* h_lam = lam_pinned ? static_cast<char*>(lambda_out)
                             : static_cast<char*>(hws_get(c, "bh_lam", es * D * batch));
    cudaEvent_t start = nullptr, stop = nullptr;
    CK(cudaEventCreate(&start));
    CK(cudaEventCreate(&stop));
    // Q / R as packed lower triangles (upload_kkt_packed); B2P_PACK_SYM=0 sends
    // the full blocks
    const bool pack = env_int("B2P_PACK_SYM", 1) != 0 && n >= 2;
    size_t h2d_total = 0;
    cudaEvent_t ready[2] = {nullptr, nullptr};
    for (auto& e : ready) {
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      CK(cudaEventRecord(e, streams[0]));
    }
    CK(cudaEventRecord(start, streams[0]));
    CK(cudaStreamWaitEvent(streams[1], start, 0));
    for (int ci = 0; ci < nchunks; ++ci) {
      const int first = ci * chunk, cnt = std::min(chunk, batch - first);
      const int sidx = ci & 1;
      cudaStream_t st = streams[sidx];
      const std::string tag = std::string("bh") + char('0' + sidx) + "_";
      void* in = ws_get(c, tag + "in", kkt_block_bytes(k, es, chunk));
      const KktDev kv =
          !pack ? upload_kkt(c, k, es, first, cnt, in, st, nullptr, 0, nullptr, false)
          : dtype == B2P_F64
              ? upload_kkt_packed<double>(c, k, first, cnt, in, st, tag, ready[sidx], &h2d_total)
              : upload_kkt_packed<float>(c, k, first, cnt, in, st, tag, ready[sidx], &h2d_total);
      char* dl0 = nullptr;
      if (lambda0) {
        dl0 = static_cast<char*>(ws_get(c, tag + "l0", es * D * chunk));
        h2d(c, dl0, static_cast<const char*>(lambda0) + es * D * first, es * D * cnt, st);
      }
      char* dl = static_cast<char*>(ws_get(c, tag + "l", es * D * chunk));
      SysOut* dout = static_cast<SysOut*>(ws_get(c, tag + "out", sizeof(SysOut) * chunk));
      int* ek = static_cast<int*>(ws_get(c, tag + "ek", sizeof(int) * chunk));
      b2p_kkt kc = *k;
      if (dtype == B2P_F64)
        solve_device_impl<double>(c, &kc, kv, cnt, kind, order, cfg, dl0, dl, dout, ek, nullptr,
                                  0, st, false, tag);
      else
        solve_device_impl<float>(c, &kc, kv, cnt, kind, order, cfg, dl0, dl, dout, ek, nullptr, 0,
                                 st, false, tag);
      d2h(c, h_lam + es * D * first, dl, es * D * cnt, st);
      d2h(c, h_outs + first, dout, sizeof(SysOut) * cnt, st);
      d2h(c, h_keys + first, ek, sizeof(int) * cnt, st);
    }
    cudaEvent_t join = nullptr;
    CK(cudaEventCreate(&join));
    CK(cudaEventRecord(join, streams[1]));
    CK(cudaStreamWaitEvent(streams[0], join, 0));
    CK(cudaEventRecord(stop, streams[0]));
    CK(cudaEventSynchronize(stop));
    CK(cudaEventElapsedTime(&c->last_ms, start, stop));
    cudaEventDestroy(start);
    cudaEventDestroy(stop);
    cudaEventDestroy(join);
    for (auto& e : ready) cudaEventDestroy(e);
    {
      const size_t Nn = k->N, nn_ = k->n, mm_ = k->m, Kk = Nn + 1;
      const size_t full = (Kk * nn_ * nn_ + Kk * nn_ + Nn * mm_ * mm_ + Nn * mm_ + Nn * nn_ * nn_ +
                           Nn * nn_ * mm_ + Nn * nn_ + 2 * nn_) * es * batch;
      c->last_h2d_bytes = (pack ? h2d_total : full) + (lambda0 ? es * D * batch : 0);
    }
    if (!lam_pinned) std::memcpy(lambda_out, h_lam, es * D * batch);
    std::vector<SysOut> outs(h_outs, h_outs + batch);
    std::vector<int> keys(h_keys, h_keys + batch);
    Fail firstf{B2P_OK, ""};
    resolve(outs, keys, batch, reports, c->last_ms * 1e-3 / batch, &firstf);
    if (firstf.code != B2P_OK) throw firstf;
  });
}

}  // extern "C"
namespace {
// Persistent per-device contexts for b2p_solve_batched_multi: a call checks one
// out per shard (creating it on first use) and returns it afterwards, so the
// streams, events, pinned staging and workspaces survive across calls.
std::mutex g_pool_mu;
std::map<int, std::vector<b2p_ctx*>> g_pool;
b2p_ctx* pool_checkout(int device, b2p_error* err, int* rc) {
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    auto& v = g_pool[device];
    if (!v.empty()) {
      b2p_ctx* c = v.back();
      v.pop_back();
      *rc = B2P_OK;
      return c;
    }
  }
  b2p_ctx* c = nullptr;
  *rc = b2p_ctx_create(device, &c, err);
  return c;
}
void pool_checkin(b2p_ctx* c) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  g_pool[c->device].push_back(c);
}
}  // namespace
extern "C" {

int b2p_solve_batched_multi(const int* devices, int ndev, int dtype, int batch,
                            const b2p_kkt* k, int kind, int order, const b2p_pcg_config* cfg,
                            const void* lambda0, void* lambda_out, b2p_solve_report* reports,
                            b2p_error* err) {
  NvtxRange nvtx_("b2p_solve_batched_multi");
  return guard(err, [&] {
    check_dtype(dtype);
    check_kkt(k);
    if (!devices || ndev < 1) throw invalid("b2p_solve_batched_multi: need >= 1 device");
    const size_t es = esize(dtype);
    const int K = k->N + 1, n = k->n, m = k->m, N = k->N;
    const size_t D = size_t(K) * n;
    std::vector<int> rc(ndev, B2P_OK);
    std::vector<b2p_error> errs(ndev);
    std::vector<std::thread> th;
    const int per = (batch + ndev - 1) / ndev;
    const int active = std::min(ndev, (batch + per - 1) / per);
    // host barrier: every shard's context is ready before any device starts
    std::mutex bm;
    std::condition_variable bcv;
    int arrived = 0;
    for (int g = 0; g < active; ++g) {
      th.emplace_back([&, g] {
        const int first = g * per, cnt = std::min(per, batch - first);
        b2p_ctx* cx = pool_checkout(devices[g], &errs[g], &rc[g]);
        {
          std::unique_lock<std::mutex> lk(bm);
          if (++arrived == active) bcv.notify_all();
          else bcv.wait(lk, [&] { return arrived == active; });
        }
        if (rc[g] != B2P_OK || !cx) return;
        // contiguous batch-index shard
        const size_t nn = size_t(n) * n, Kz = K, Nz = N;
        auto off = [&](const void* p, size_t per_sys) {
          return static_cast<const void*>(static_cast<const char*>(p) + es * per_sys * first);
        };
        b2p_kkt s = *k;
        s.Q = off(k->Q, Kz * nn);
        s.q = off(k->q, Kz * n);
        s.R = off(k->R, Nz * m * m);
        s.r = off(k->r, Nz * m);
        s.A = off(k->A, Nz * nn);
        s.B = off(k->B, Nz * n * m);
        s.e = off(k->e, Nz * n);
        s.x_s = off(k->x_s, n);
        s.x0 = off(k->x0, n);
        const void* l0 = lambda0 ? static_cast<const char*>(lambda0) + es * D * first : nullptr;
        void* lo = static_cast<char*>(lambda_out) + es * D * first;
        rc[g] = b2p_solve_batched(cx, dtype, cnt, &s, kind, order, cfg, l0, lo,
                                  reports ? reports + first : nullptr, &errs[g]);
        if (rc[g] != B2P_OK && errs[g].system >= 0) errs[g].system += first;
        pool_checkin(cx);
      });
    }
    for (auto& t : th) t.join();
    for (int g = 0; g < active; ++g)
      if (rc[g] != B2P_OK) {
        Fail f{rc[g], errs[g].message};
        f.knot = errs[g].knot;
        f.iteration = errs[g].iteration;
        f.system = errs[g].system;
        throw f;
      }
  });
}

// ---------------------------------------------------------------- generator
int b2p_uniform_draws(uint64_t seed, int count, double lo, double hi, double* out,
                      b2p_error* err) {
  return guard(err, [&] {
    if (count < 0 || (count > 0 && !out)) throw invalid("uniform_draws: bad buffer");
    Rng g(seed);
    for (int i = 0; i < count; ++i) out[i] = g.u(lo, hi);
  });
}

int b2p_random_kkt(int family, uint64_t seed, int N, int n, int m, double fl, double cp,
                   b2p_kkt_out* out, b2p_error* err) {
  return guard(err, [&] {
    if (!out || N < 0 || n < 1 || m < 0) throw invalid("b2p_random_kkt: bad arguments");
    generate_one(family, seed, N, n, m, fl, cp, out, 0);
  });
}

int b2p_random_kkt_batch(int family, uint64_t seed0, int batch, int N, int n, int m, double fl,
                         double cp, int threads, b2p_kkt_out* out, b2p_error* err) {
  return guard(err, [&] {
    if (!out || N < 0 || n < 1 || m < 0 || batch < 0)
      throw invalid("b2p_random_kkt_batch: bad arguments");
    int T = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
    T = std::max(1, std::min(T, batch));
    std::vector<std::thread> th;
    std::atomic<int> next{0};
    for (int t = 0; t < T; ++t)
      th.emplace_back([&] {
        for (int i = next++; i < batch; i = next++)
          generate_one(family, seed0 + static_cast<uint64_t>(i), N, n, m, fl, cp, out, i);
      });
    for (auto& t : th) t.join();
  });
}

void* b2p_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}
void b2p_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

}  // extern "C"
