// Microbenchmark: tcgen05.ld (TMEM -> registers) throughput per SM with 16 warps,
// vs LDS.128 shared-memory throughput, on B200 (sm_100a).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512, 1) k_tmem(float* out, int iters, long long* cyc) {
  __shared__ unsigned taddr;
  const int w = threadIdx.x >> 5;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"l"(
        reinterpret_cast<unsigned long long>(&taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const unsigned base = taddr + ((32u * (w & 3)) << 16) + 64u * (w >> 2);
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    unsigned r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
          "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
          "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(base + 32u * (it & 1)));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) acc += __uint_as_float(r[i]);
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(taddr));
}

__global__ void __launch_bounds__(512, 1) k_lds(float* out, int iters, long long* cyc) {
  __shared__ __align__(16) float sm[512 * 4 * 4];
  for (int i = threadIdx.x; i < 512 * 4 * 4; i += 512) sm[i] = i;
  __syncthreads();
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float4 v = *reinterpret_cast<const float4*>(sm + 4 * (threadIdx.x + 512 * (j & 3)) + (it & 1) * 0);
      acc += v.x + v.y + v.z + v.w;
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* d; long long* c; long long h[1];
  cudaMalloc(&d, 1 << 24); cudaMalloc(&c, 1024 * 8);
  const int iters = 4096;
  k_tmem<<<148, 512>>>(d, 16, c);
  k_tmem<<<148, 512>>>(d, iters, c);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
  printf("tmem: %s, %.1f bytes/clk/SM (32x32b.x32 per warp, 16 warps)\n", cudaGetErrorString(e),
         512.0 * 128 * iters / h[0]);
  k_lds<<<148, 512>>>(d, 16, c);
  k_lds<<<148, 512>>>(d, iters, c);
  e = cudaDeviceSynchronize();
  cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
  printf("lds.128: %s, %.1f bytes/clk/SM\n", cudaGetErrorString(e), 512.0 * 128 * iters / h[0]);
  return 0;
}
