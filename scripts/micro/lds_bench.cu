// Microbenchmark: shared-memory load cost on one SM (16 warps) by access
// pattern — 8- and 16-byte loads with 1, 2, 4 or 8 distinct (broadcast)
// addresses per warp, and with every lane distinct. Reports SM cycles per
// warp-instruction (1.0 = one wavefront per clock).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/micro/lds_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int GROUPS, int WIDTH>  // GROUPS distinct addresses per warp (0 = all lanes distinct)
__global__ void k(double* out, long long* cyc, int reps) {
  extern __shared__ __align__(16) double s[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = i * 1e-3;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int grp = GROUPS ? lane / (32 / GROUPS) : lane;
  // groups land 34 doubles apart (distinct banks), warps 1024 doubles apart
  int base = w * 256 + grp * (GROUPS ? 34 : WIDTH / 8);
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    const int o = base + ((r * 2) & 15);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (WIDTH == 16) {
        const double2 v = *reinterpret_cast<const double2*>(s + o + j * 8);
        a0 += v.x;
        a1 += v.y;
      } else {
        a0 += s[o + j * 8];
        a2 += s[o + j * 8 + 4];
      }
    }
  }
  long long t1 = clock64();
  __syncthreads();
  out[threadIdx.x] = a0 + a1 + a2 + a3;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int G, int W>
void run(const char* name, double* out, long long* c) {
  const int reps = 256, threads = 512;
  cudaFuncSetAttribute(k<G, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 8);
  k<G, W><<<1, threads, 8192 * 8>>>(out, c, 8);
  k<G, W><<<1, threads, 8192 * 8>>>(out, c, reps);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  const double instrs = double(reps) * (W == 16 ? 16 : 32) * (threads / 32);
  printf("%-34s %.2f SM cycles per warp-load\n", name, double(h) / instrs);
}

int main() {
  double* out; long long* c;
  cudaMalloc(&out, 1 << 16); cudaMalloc(&c, 64);
  run<1, 8>("LDS.64  1 address/warp", out, c);
  run<2, 8>("LDS.64  2 addresses/warp", out, c);
  run<4, 8>("LDS.64  4 addresses/warp", out, c);
  run<8, 8>("LDS.64  8 addresses/warp", out, c);
  run<0, 8>("LDS.64  32 distinct (consecutive)", out, c);
  run<1, 16>("LDS.128 1 address/warp", out, c);
  run<2, 16>("LDS.128 2 addresses/warp", out, c);
  run<4, 16>("LDS.128 4 addresses/warp", out, c);
  run<8, 16>("LDS.128 8 addresses/warp", out, c);
  run<0, 16>("LDS.128 32 distinct (consecutive)", out, c);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
