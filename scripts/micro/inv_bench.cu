// Microbenchmark: latency / throughput of the half-warp 14x14 SPD inverse
// (hw_spd_inverse_v2, the formation's building block) on one SM.
#include <cstdio>
#include <cuda_runtime.h>
#include "hw_dense.cuh"
using namespace b2p;
using namespace b2p::hwd;

__global__ void k_inv(const double* Q, double* out, long long* cyc, int reps) {
  extern __shared__ __align__(16) double tiles_raw[];
  double (*tiles)[2 * 196 + 32] = reinterpret_cast<double (*)[2 * 196 + 32]>(tiles_raw);
  const int h = threadIdx.x >> 4, l = threadIdx.x & 15;
  double* W = tiles[h];
  double* X = W + 196;
  double* rd = X + 196;
  const int lr = l < 14 ? l : 13;
  double a[14], x[14];
  double acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
#pragma unroll
    for (int i = 0; i < 14; ++i) a[i] = Q[lr * 14 + i] + acc * 1e-30;
    const int f = hw_spd_inverse_v2<double, 14, true>(a, W, X, rd, l, x);
    acc += x[0] + f;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  double hQ[196];
  for (int i = 0; i < 14; ++i)
    for (int j = 0; j < 14; ++j) hQ[i * 14 + j] = (i == j ? 20.0 : 0.0) + 1.0 / (1 + i + j);
  double *Q, *out; long long* c; long long h;
  cudaMalloc(&Q, sizeof(hQ)); cudaMalloc(&out, 1 << 20); cudaMalloc(&c, 8 * 1024);
  cudaMemcpy(Q, hQ, sizeof(hQ), cudaMemcpyHostToDevice);
  const int reps = 64;
  for (int warps : {1, 4, 8, 16}) {
    cudaFuncSetAttribute(k_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * (2 * 196 + 32) * 8);
    k_inv<<<1, 32 * warps, 32 * (2 * 196 + 32) * 8>>>(Q, out, c, 4);
    k_inv<<<1, 32 * warps, 32 * (2 * 196 + 32) * 8>>>(Q, out, c, reps);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("warps=%2d: %.0f cycles per inverse round (%d inverses per round per SM) -> %.0f cycles/inverse/SM\n",
           warps, double(h) / reps, 2 * warps, double(h) / reps / (2 * warps));
  }
  return 0;
}
