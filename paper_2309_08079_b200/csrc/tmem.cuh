// Tensor-memory (TMEM) row helpers for the fused kernels: 32x32b loads and
// stores (thread t of a warp owns TMEM lane 32*(warp%4) + t) of fp64 rows
// packed as 2 words per double, for any row length up to 16 doubles.
#pragma once

namespace b2p {
namespace tm {

// doubles per TMEM load chunk in the row products (2 rows x 2 words each live
// in registers between the load and its wait)
#ifndef TM_CHUNK
#define TM_CHUNK 4
#endif

__device__ __forceinline__ void ld16(unsigned t, unsigned* u) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];\n"
      : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]),
        "=r"(u[7]), "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]),
        "=r"(u[14]), "=r"(u[15])
      : "r"(t));
}
__device__ __forceinline__ void ld8(unsigned t, unsigned* u) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]),
                 "=r"(u[6]), "=r"(u[7])
               : "r"(t));
}
__device__ __forceinline__ void ld4(unsigned t, unsigned* u) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3])
               : "r"(t));
}
__device__ __forceinline__ void ld2(unsigned t, unsigned* u) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n"
               : "=r"(u[0]), "=r"(u[1])
               : "r"(t));
}
__device__ __forceinline__ void st16(unsigned t, const unsigned* u) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16};\n" ::"r"(t),
      "r"(u[0]), "r"(u[1]), "r"(u[2]), "r"(u[3]), "r"(u[4]), "r"(u[5]), "r"(u[6]), "r"(u[7]),
      "r"(u[8]), "r"(u[9]), "r"(u[10]), "r"(u[11]), "r"(u[12]), "r"(u[13]), "r"(u[14]), "r"(u[15])
      : "memory");
}
__device__ __forceinline__ void st8(unsigned t, const unsigned* u) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(t),
      "r"(u[0]), "r"(u[1]), "r"(u[2]), "r"(u[3]), "r"(u[4]), "r"(u[5]), "r"(u[6]), "r"(u[7])
      : "memory");
}
__device__ __forceinline__ void st4(unsigned t, const unsigned* u) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(t), "r"(u[0]),
               "r"(u[1]), "r"(u[2]), "r"(u[3])
               : "memory");
}
__device__ __forceinline__ void st2(unsigned t, const unsigned* u) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};\n" ::"r"(t), "r"(u[0]),
               "r"(u[1])
               : "memory");
}

// W words (W even) at column t, as the widest shapes that fit
template <int W>
__device__ __forceinline__ void ld_words(unsigned t, unsigned* u) {
  if constexpr (W >= 16) {
    ld16(t, u);
    ld_words<W - 16>(t + 16, u + 16);
  } else if constexpr (W >= 8) {
    ld8(t, u);
    ld_words<W - 8>(t + 8, u + 8);
  } else if constexpr (W >= 4) {
    ld4(t, u);
    ld_words<W - 4>(t + 4, u + 4);
  } else if constexpr (W >= 2) {
    ld2(t, u);
  }
}
template <int W>
__device__ __forceinline__ void st_words(unsigned t, const unsigned* u) {
  if constexpr (W >= 16) {
    st16(t, u);
    st_words<W - 16>(t + 16, u + 16);
  } else if constexpr (W >= 8) {
    st8(t, u);
    st_words<W - 8>(t + 8, u + 8);
  } else if constexpr (W >= 4) {
    st4(t, u);
    st_words<W - 4>(t + 4, u + 4);
  } else if constexpr (W >= 2) {
    st2(t, u);
  }
}

// tcgen05.wait::ld, then an empty asm per destination register: consumers read
// the registers as outputs of those asms, so none is hoisted above the wait
// (volatile asms keep their order).
template <int W>
__device__ __forceinline__ void wait_ld(unsigned* u) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < W; ++i) asm volatile("" : "+r"(u[i]));
}

__device__ __forceinline__ double word2(const unsigned* u, int j) {
  return __hiloint2double(static_cast<int>(u[2 * j + 1]), static_cast<int>(u[2 * j]));
}

// row of NB doubles -> TMEM columns [t, t + 2 NB)
template <int NB>
__device__ __forceinline__ void st_row(unsigned t, const double (&v)[NB]) {
  unsigned u[2 * NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    u[2 * j] = static_cast<unsigned>(__double2loint(v[j]));
    u[2 * j + 1] = static_cast<unsigned>(__double2hiint(v[j]));
  }
  st_words<2 * NB>(t, u);
}

// (o0, o1) += the dot products of two NB-double TMEM rows of the calling
// thread's lane with one 16-byte aligned shared vector x, over columns
// [J0, NB) in chunks of <= 8 doubles (bounded live registers); each
// broadcast x pair serves both rows. Two accumulators per row: even j -> a,
// odd j -> c (the dot_rm order).
template <int NB, int J0>
__device__ __forceinline__ void dot2_chunks(unsigned t0, unsigned t1, const double* x, double& a0,
                                            double& c0, double& a1, double& c1) {
  if constexpr (J0 < NB) {
    constexpr int C = (NB - J0) < TM_CHUNK ? (NB - J0) : TM_CHUNK;  // doubles in this chunk (even)
    unsigned u[2 * C], w[2 * C];
    ld_words<2 * C>(t0 + 2 * J0, u);
    ld_words<2 * C>(t1 + 2 * J0, w);
    // no "memory" clobber: TMEM is not compiler-visible memory, so the shared
    // loads of x are free to be scheduled across the wait (they overlap the
    // TMEM latency instead of starting after it)
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
#pragma unroll
    for (int i = 0; i < 2 * C; ++i) asm volatile("" : "+r"(u[i]), "+r"(w[i]));
#pragma unroll
    for (int j = 0; j < C; j += 2) {
      const double2 v = *reinterpret_cast<const double2*>(x + J0 + j);
      a0 += word2(u, j) * v.x;
      c0 += word2(u, j + 1) * v.y;
      a1 += word2(w, j) * v.x;
      c1 += word2(w, j + 1) * v.y;
    }
    dot2_chunks<NB, J0 + C>(t0, t1, x, a0, c0, a1, c1);
  }
}
template <int NB>
__device__ __forceinline__ void dot2_row(unsigned t0, unsigned t1, const double* x, double& o0,
                                         double& o1) {
  static_assert(NB % 2 == 0 && NB <= 16, "even rows of <= 16 doubles");
  double a0 = 0.0, c0 = 0.0, a1 = 0.0, c1 = 0.0;
  dot2_chunks<NB, 0>(t0, t1, x, a0, c0, a1, c1);
  o0 = a0 + c0;
  o1 = a1 + c1;
}

}  // namespace tm
}  // namespace b2p
