// Microbenchmark: SPD inverse (schur.cpp:15-23) of 14x14 blocks on one SM at
// 512 threads, three lane mappings:
//   v1  the half-warp helper (hw_spd_inverse_v2): 16 lanes per block, one row
//       per lane, 32 blocks per round;
//   v2  8-lane groups with two rows per lane (rows l, l + 7): 64 blocks per
//       round, every broadcast operand serves both rows of the lane;
//   v3  v2 with 16-byte pair loads of the broadcast operands.
// Prints cycles per round and per inverse, and checks v2/v3 against v1.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2309_08079_b200/csrc scripts/micro/inv8_bench.cu
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
#include "hw_dense.cuh"
using namespace b2p;
using namespace b2p::hwd;

constexpr int N = 14, H = 7;

// 8-lane group, lane l < 7 owns rows l and l + 7 (lane 7 duplicates row 6/13,
// stores nothing). Lr: [N][N] rows of L; LiT: [N][N] rows of L^-T; rd[N];
// X: output [N][N] (row-major, bitwise symmetric). Full-warp convergent.
template <bool PAIR>
__device__ __forceinline__ int g8x2_spd_inverse(double (&a0)[N], double (&a1)[N], double* Lr,
                                                double* LiT, double* rd, int l, double* X) {
  int fail = -1;
  const bool act = l < H;
  const int lr = act ? l : H - 1;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    double s0 = 0.0, s1 = a1[k];
    if (k < H) s0 = a0[k];
    if constexpr (PAIR) {
#pragma unroll
      for (int q = 0; q + 1 < k; q += 2) {
        const double2 v = *reinterpret_cast<const double2*>(Lr + k * N + q);
        if (k < H) { s0 -= a0[q] * v.x; s0 -= a0[q + 1] * v.y; }
        s1 -= a1[q] * v.x;
        s1 -= a1[q + 1] * v.y;
      }
      if (k & 1) {
        const double v = Lr[k * N + k - 1];
        if (k < H) s0 -= a0[k - 1] * v;
        s1 -= a1[k - 1] * v;
      }
    } else {
#pragma unroll
      for (int q = 0; q < k; ++q) {
        const double v = Lr[k * N + q];
        if (k < H) s0 -= a0[q] * v;
        s1 -= a1[q] * v;
      }
    }
    double piv = __shfl_sync(FULL, k < H ? s0 : s1, k < H ? k : k - H, 8);
    const bool bad = piv <= 0.0;
    fail = (bad && fail < 0) ? k : fail;
    piv = bad ? 1.0 : piv;
    const double r = rsqrt(piv);
    if (k < H) {
      const double v0 = (lr == k ? piv : s0) * r;
      const bool own0 = act && lr >= k;
      a0[k] = own0 ? v0 : a0[k];
      if (own0) Lr[lr * N + k] = v0;
    }
    {
      const double v1 = (lr + H == k ? piv : s1) * r;
      const bool own1 = act && lr + H >= k;
      a1[k] = own1 ? v1 : a1[k];
      if (own1) Lr[(lr + H) * N + k] = v1;
    }
    if (l == (k < H ? k : k - H) && act) rd[k] = r;
    __syncwarp();
  }
  // columns l and l + 7 of L^-1
  double y0[N], y1[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double t0 = (i == lr) ? 1.0 : 0.0, t1 = (i == lr + H) ? 1.0 : 0.0;
    if constexpr (PAIR) {
#pragma unroll
      for (int q = 0; q + 1 < i; q += 2) {
        const double2 v = *reinterpret_cast<const double2*>(Lr + i * N + q);
        t0 -= v.x * y0[q];
        t0 -= v.y * y0[q + 1];
        t1 -= v.x * y1[q];
        t1 -= v.y * y1[q + 1];
      }
      if (i & 1) {
        const double v = Lr[i * N + i - 1];
        t0 -= v * y0[i - 1];
        t1 -= v * y1[i - 1];
      }
    } else {
#pragma unroll
      for (int q = 0; q < i; ++q) {
        const double v = Lr[i * N + q];
        t0 -= v * y0[q];
        t1 -= v * y1[q];
      }
    }
    const double d = rd[i];
    y0[i] = t0 * d;
    y1[i] = t1 * d;
  }
  __syncwarp();  // LiT aliases Lr
  if (act) {
#pragma unroll
    for (int q = 0; q < N; q += 2) {
      *reinterpret_cast<double2*>(LiT + lr * N + q) = make_double2(y0[q], y0[q + 1]);
      *reinterpret_cast<double2*>(LiT + (lr + H) * N + q) = make_double2(y1[q], y1[q + 1]);
    }
  }
  __syncwarp();
  // X[i][c] = sum_{q >= i} LiT[i][q] y_c[q], c = l, l + 7; written as rows c
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double x0 = 0.0, x1 = 0.0;
#pragma unroll
    for (int q = i; q < N; ++q) {
      const double v = LiT[i * N + q];
      x0 += v * y0[q];
      x1 += v * y1[q];
    }
    if (act) {
      X[lr * N + i] = x0;
      X[(lr + H) * N + i] = x1;
    }
  }
  __syncwarp();
  return fail;
}

__global__ void k_v1(const double* Q, double* out, long long* cyc, int reps) {
  extern __shared__ __align__(16) double sm[];
  const int h = threadIdx.x >> 4, l = threadIdx.x & 15;
  double* W = sm + h * (2 * 196 + 32);
  double* Xt = W + 196;
  double* rd = Xt + 196;
  const int lr = l < 14 ? l : 13;
  double a[14], x[14];
  double acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
#pragma unroll
    for (int i = 0; i < 14; ++i) a[i] = Q[lr * 14 + i] + acc * 1e-300;
    const int f = hw_spd_inverse_v2<double, 14, true>(a, W, Xt, rd, l, x);
    acc += x[0] + f;
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x < 16 && l < 14)
    for (int i = 0; i < 14; ++i) out[l * 14 + i] = x[i];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 12345.678) out[1000] = acc;
}

template <bool PAIR>
__global__ void k_v2(const double* Q, double* out, long long* cyc, int reps) {
  extern __shared__ __align__(16) double sm[];
  const int g = threadIdx.x >> 3, l = threadIdx.x & 7;
  double* Lr = sm + g * (2 * 196 + 16);
  double* LiT = Lr;
  double* X = LiT + 196;
  double* rd = X + 196;
  const int lr = l < 7 ? l : 6;
  double a0[14], a1[14];
  double acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
#pragma unroll
    for (int i = 0; i < 14; ++i) {
      a0[i] = Q[lr * 14 + i] + acc * 1e-300;
      a1[i] = Q[(lr + 7) * 14 + i] + acc * 1e-300;
    }
    const int f = g8x2_spd_inverse<PAIR>(a0, a1, Lr, LiT, rd, l, X);
    acc += X[(it % 14) * 14 + l] + f;
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < 196; ++i) out[196 + i] = X[i];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 12345.678) out[1000] = acc;
}

int main() {
  double hQ[196];
  unsigned long long s = 88172645463325252ull;
  double L[196];
  for (int i = 0; i < 196; ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    L[i] = (s >> 11) * (1.0 / 9007199254740992.0) * 2 - 1;
  }
  for (int i = 0; i < 14; ++i)
    for (int j = 0; j < 14; ++j) {
      double v = (i == j) ? 0.1 : 0.0;
      for (int k = 0; k < 14; ++k) v += L[i * 14 + k] * L[j * 14 + k];
      hQ[i * 14 + j] = v;
    }
  double *Q, *out; long long* c; long long h;
  cudaMalloc(&Q, sizeof(hQ)); cudaMalloc(&out, 1 << 20); cudaMalloc(&c, 8 * 1024);
  cudaMemcpy(Q, hQ, sizeof(hQ), cudaMemcpyHostToDevice);
  const int reps = 64;
  const size_t s1 = 32 * (2 * 196 + 32) * 8, s2 = 64 * (2 * 196 + 16) * 8;
  cudaFuncSetAttribute(k_v1, cudaFuncAttributeMaxDynamicSharedMemorySize, s1);
  cudaFuncSetAttribute(k_v2<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, s2);
  cudaFuncSetAttribute(k_v2<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, s2);
  for (int threads : {32, 256, 512}) {
    k_v1<<<1, threads, s1>>>(Q, out, c, 4);
    k_v1<<<1, threads, s1>>>(Q, out, c, reps);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("v1 threads=%3d: %6.0f cycles/round, %3d inverses/round -> %5.0f cycles/inverse/SM\n", threads,
           double(h) / reps, threads / 16, double(h) / reps / (threads / 16));
    for (int pair = 0; pair < 2; ++pair) {
      auto k = pair ? k_v2<true> : k_v2<false>;
      k<<<1, threads, s2>>>(Q, out, c, 4);
      k<<<1, threads, s2>>>(Q, out, c, reps);
      cudaDeviceSynchronize();
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      printf("v%d threads=%3d: %6.0f cycles/round, %3d inverses/round -> %5.0f cycles/inverse/SM\n",
             2 + pair, threads, double(h) / reps, threads / 8, double(h) / reps / (threads / 8));
    }
  }
  double ho[392];
  cudaMemcpy(ho, out, sizeof(ho), cudaMemcpyDeviceToHost);
  double md = 0;
  for (int i = 0; i < 196; ++i) md = fmax(md, fabs(ho[i] - ho[196 + i]) / fmax(1.0, fabs(ho[i])));
  printf("max |v1 - v3| rel = %.3e  (X[0][0] = %.6f)\n", md, ho[0]);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
