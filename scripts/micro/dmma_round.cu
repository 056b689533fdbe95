// Which scalar FMA order reproduces mma.sync.m8n8k4.row.col.f64 bitwise?
// D[i][j] = sum_k A[i][k] B[k][j] + C[i][j]; candidates:
//   chainC: fma(a3,b3, fma(a2,b2, fma(a1,b1, fma(a0,b0,c))))
//   chain0: fma(a3,b3, fma(a2,b2, fma(a1,b1, a0*b0))) + c
//   exact : the exactly rounded sum (long double reference on the host)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/micro/dmma_round.cu
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void k(const double* A, const double* B, const double* C, double* D, int reps) {
  const int lane = threadIdx.x;
  for (int t = 0; t < reps; ++t) {
    const double* a = A + t * 32;  // 8x4 row-major
    const double* b = B + t * 32;  // 4x8 row-major
    const double* c = C + t * 64;  // 8x8
    // fragments (PTX ISA m8n8k4 .f64): A: row = lane/4, col = lane%4; B: row = lane%4, col = lane/4;
    // C/D: row = lane/4, cols 2*(lane%4), +1
    const double af = a[(lane >> 2) * 4 + (lane & 3)];
    const double bf = b[(lane & 3) * 8 + (lane >> 2)];
    const int r = lane >> 2, c0 = 2 * (lane & 3);
    double d0, d1;
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
                 : "=d"(d0), "=d"(d1)
                 : "d"(af), "d"(bf), "d"(c[r * 8 + c0]), "d"(c[r * 8 + c0 + 1]));
    D[t * 64 + r * 8 + c0] = d0;
    D[t * 64 + r * 8 + c0 + 1] = d1;
  }
}

int main() {
  const int T = 4096;
  double *hA = new double[T * 32], *hB = new double[T * 32], *hC = new double[T * 64], *hD = new double[T * 64];
  srand(7);
  auto rnd = [] { return (rand() / (double)RAND_MAX * 2 - 1) * std::pow(2.0, rand() % 20 - 10); };
  for (int i = 0; i < T * 32; ++i) { hA[i] = rnd(); hB[i] = rnd(); }
  for (int i = 0; i < T * 64; ++i) hC[i] = rnd();
  double *A, *B, *C, *D;
  cudaMalloc(&A, T * 32 * 8); cudaMalloc(&B, T * 32 * 8); cudaMalloc(&C, T * 64 * 8); cudaMalloc(&D, T * 64 * 8);
  cudaMemcpy(A, hA, T * 32 * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, T * 32 * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(C, hC, T * 64 * 8, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(A, B, C, D, T);
  cudaMemcpy(hD, D, T * 64 * 8, cudaMemcpyDeviceToHost);
  long nC = 0, n0 = 0, nE = 0, nR = 0, tot = 0;
  for (int t = 0; t < T; ++t)
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) {
        const double* a = hA + t * 32 + i * 4;
        double bcol[4];
        for (int q = 0; q < 4; ++q) bcol[q] = hB[t * 32 + q * 8 + j];
        const double c = hC[t * 64 + i * 8 + j];
        double chC = c;
        for (int q = 0; q < 4; ++q) chC = std::fma(a[q], bcol[q], chC);
        double ch0 = a[0] * bcol[0];
        for (int q = 1; q < 4; ++q) ch0 = std::fma(a[q], bcol[q], ch0);
        ch0 += c;
        double rev = c;
        for (int q = 3; q >= 0; --q) rev = std::fma(a[q], bcol[q], rev);
        long double ex = c;
        for (int q = 0; q < 4; ++q) ex += (long double)a[q] * bcol[q];
        const double d = hD[t * 64 + i * 8 + j];
        nC += d == chC; n0 += d == ch0; nE += d == (double)ex; nR += d == rev; ++tot;
      }
  printf("DMMA == fma chain from C (k ascending): %ld / %ld\n", nC, tot);
  printf("DMMA == fma chain from C (k descending): %ld / %ld\n", nR, tot);
  printf("DMMA == chain from 0, then + C        : %ld / %ld\n", n0, tot);
  printf("DMMA == exact (long double) rounding  : %ld / %ld\n", nE, tot);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
