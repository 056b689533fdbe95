// Microbenchmark: single-warp dependent-chain latencies on B200 (sm_100a):
// DFMA, rsqrt(double), 1/x (double), __shfl_sync(double), LDS.64 round trip.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k_chain(double* out, long long* cyc, int iters, double seed) {
  __shared__ double sm[64];
  sm[threadIdx.x] = seed + threadIdx.x;
  __syncwarp();
  double x = seed + threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (OP == 0) x = fma(x, 0.999999, 1e-7);
      if (OP == 1) x = rsqrt(x) + 0.5;
      if (OP == 2) x = 1.0 / x + 0.5;
      if (OP == 3) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1e-9;
      if (OP == 4) x = sm[(static_cast<int>(x) & 31)] + 1e-9;
      if (OP == 5) x = sqrt(x) + 0.5;
      if (OP == 6) { x = __shfl_sync(0xffffffffu, x, 3, 16) + 1e-9; __syncwarp(); }
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

// DFMA throughput: 16 warps/SMSP-ish, independent chains
__global__ void k_dfma_tp(double* out, int iters) {
  double c[8];
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(c[i], 0.999999, 1e-7);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* d; long long* c;
  cudaMalloc(&d, 1 << 24); cudaMalloc(&c, 64);
  const char* names[] = {"DFMA", "rsqrt(f64)+DADD", "1/x(f64)+DADD", "SHFL(f64)+DADD", "LDS.64 dep", "sqrt(f64)+DADD", "SHFL16(f64)+DADD+syncwarp"};
  for (int op = 0; op < 7; ++op) {
    long long h = 0;
    for (int rep = 0; rep < 2; ++rep) {
      switch (op) {
        case 0: k_chain<0><<<1, 32>>>(d, c, 64, 1.5); break;
        case 1: k_chain<1><<<1, 32>>>(d, c, 64, 1.5); break;
        case 2: k_chain<2><<<1, 32>>>(d, c, 64, 1.5); break;
        case 3: k_chain<3><<<1, 32>>>(d, c, 64, 1.5); break;
        case 4: k_chain<4><<<1, 32>>>(d, c, 64, 1.5); break;
        case 5: k_chain<5><<<1, 32>>>(d, c, 64, 1.5); break;
        case 6: k_chain<6><<<1, 32>>>(d, c, 64, 1.5); break;
      }
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    }
    printf("%-28s %.1f cycles/op\n", names[op], h / (64.0 * 16));
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  k_dfma_tp<<<sms * 4, 512>>>(d, 1000);
  cudaEventRecord(e0);
  k_dfma_tp<<<sms * 4, 512>>>(d, 4000);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fma = double(sms) * 4 * 512 * 4000 * 8;
  printf("DFMA throughput: %.2f TFLOP/s (%.1f FMA/clk/SM at %d MHz)\n", 2 * fma / ms / 1e9, fma / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  return 0;
}
