// common.cuh — shared device helpers for the MH-LatentMoE kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace mhl {

typedef __nv_bfloat16 bf16;

#ifdef __CUDACC__

// element load/store as float (E = float or bf16)
__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(bf16 v) { return __bfloat162float(v); }
template <typename E> __device__ __forceinline__ E from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ bf16 from_f<bf16>(float v) { return __float2bfloat16_rn(v); }

// exact-erf GELU (R1) and its derivative, fp32
__device__ __forceinline__ float gelu_f(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }
__device__ __forceinline__ float gelu_grad_f(float x) {
  const float cdf = 0.5f * (1.0f + erff(x * 0.70710678118654752f));
  const float pdf = 0.39894228040143268f * __expf(-0.5f * x * x);
  return cdf + x * pdf;
}

// Exact-erf GELU for a pair of values with packed f32x2 math (sm_100 FFMA2/FMUL2) and one
// ex2 + one rcp per element: Phi(x) = 1/2 (1 + sign(x) erf(|x|/sqrt 2)) with erf from
// Abramowitz-Stegun 7.1.26 (|error| <= 1.5e-7; R1 requires the erf form, not tanh).
// Returns gelu(x) = x Phi(x); if dgelu != nullptr also gelu'(x) = Phi(x) + x phi(x), reusing
// exp(-x^2/2) for phi.
__device__ __forceinline__ float fast_rcp(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float fast_ex2(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// 1/x on the FMA pipe (x >= 1 here): magic-constant seed (|rel err| <= 1/8) and three Newton steps
// (1/8 -> 1.6e-2 -> 2.4e-4 -> 6e-8), so half of the GELU reciprocals leave the MUFU (the epilogues
// are MUFU-bound at 2 MUFU ops per element).
__device__ __forceinline__ float nr_rcp(float x) {
  float r = __int_as_float(0x7EF311C7 - __float_as_int(x));
#pragma unroll
  for (int i = 0; i < 3; ++i) r = fmaf(r, fmaf(-x, r, 1.0f), r);
  return r;
}
__device__ __forceinline__ float2 gelu2(float2 h, float2* dgelu) {
  const float2 hh = __fmul2_rn(h, h);
  const float2 z = make_float2(fabsf(h.x) * 0.70710678118654752f, fabsf(h.y) * 0.70710678118654752f);
  const float2 d = __ffma2_rn(make_float2(0.3275911f, 0.3275911f), z, make_float2(1.f, 1.f));
#ifdef MHL_GELU_NR
  const float2 t = make_float2(fast_rcp(d.x), nr_rcp(d.y));
#else
  const float2 t = make_float2(fast_rcp(d.x), fast_rcp(d.y));
#endif
  float2 q = __ffma2_rn(make_float2(1.061405429f, 1.061405429f), t, make_float2(-1.453152027f, -1.453152027f));
  q = __ffma2_rn(q, t, make_float2(1.421413741f, 1.421413741f));
  q = __ffma2_rn(q, t, make_float2(-0.284496736f, -0.284496736f));
  q = __ffma2_rn(q, t, make_float2(0.254829592f, 0.254829592f));
  q = __fmul2_rn(q, t);
  const float2 ea = __fmul2_rn(hh, make_float2(-0.72134752044448170f, -0.72134752044448170f));  // -x^2/2 log2 e
  const float2 e = make_float2(fast_ex2(ea.x), fast_ex2(ea.y));                                  // exp(-x^2/2)
  const float2 erfa = __ffma2_rn(make_float2(-q.x, -q.y), e, make_float2(1.f, 1.f));             // erf(|x|/sqrt2)
  const float2 hp = __fmul2_rn(erfa, make_float2(0.5f, 0.5f));
  const float2 phi = make_float2(0.5f + copysignf(hp.x, h.x), 0.5f + copysignf(hp.y, h.y));     // Phi(x)
  if (dgelu) {
    const float2 pdf = __fmul2_rn(e, make_float2(0.39894228040143268f, 0.39894228040143268f));
    *dgelu = __ffma2_rn(h, pdf, phi);
  }
  return __fmul2_rn(h, phi);
}

// g * gelu(x) for a pair, forward only, with the fewest issued instructions: gelu(x) = x Phi(x) =
// (x + |x| erf(|x|/sqrt2)) / 2, so with hg = g / 2:  hg * (x + |x| * erfa).  erf from the same
// Abramowitz-Stegun 7.1.26 form as gelu2 (t = 1 / (1 + p |x| / sqrt2), one rcp + one ex2 per element,
// |error| <= 1.5e-7), the |x| folded into FFMA operands (18 instructions per pair instead of 23).
__device__ __forceinline__ float2 gelu2_scaled(float2 h, float hg) {
  const float2 ea = __fmul2_rn(__fmul2_rn(h, make_float2(-0.72134752044448170f, -0.72134752044448170f)), h);
  const float dx = fmaf(fabsf(h.x), 0.23164188f, 1.f), dy = fmaf(fabsf(h.y), 0.23164188f, 1.f);
  const float2 t = make_float2(fast_rcp(dx), fast_rcp(dy));
  float2 q = __ffma2_rn(make_float2(1.061405429f, 1.061405429f), t, make_float2(-1.453152027f, -1.453152027f));
  q = __ffma2_rn(q, t, make_float2(1.421413741f, 1.421413741f));
  q = __ffma2_rn(q, t, make_float2(-0.284496736f, -0.284496736f));
  q = __ffma2_rn(q, t, make_float2(0.254829592f, 0.254829592f));
  q = __fmul2_rn(q, t);
  const float2 e = make_float2(fast_ex2(ea.x), fast_ex2(ea.y));                                  // exp(-x^2/2)
  const float2 erfa = __ffma2_rn(make_float2(-q.x, -q.y), e, make_float2(1.f, 1.f));             // erf(|x|/sqrt2)
  const float2 s2 = make_float2(fmaf(fabsf(h.x), erfa.x, h.x), fmaf(fabsf(h.y), erfa.y, h.y));   // 2 gelu(x)
  return __fmul2_rn(s2, make_float2(hg, hg));
}

// Order-preserving float -> uint32 (R6): flip sign bit of non-negatives, all bits of negatives.
__device__ __forceinline__ uint32_t ord32(float v) {
  uint32_t u = __float_as_uint(v == 0.0f ? 0.0f : v);   // canonicalise -0.0
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ unsigned long long pack_key(float v, int idx) {
  return ((unsigned long long)ord32(v) << 32) | (unsigned long long)(~(uint32_t)idx);
}
// inverse of ord32 (for a canonical key: -0.0 never occurs)
__device__ __forceinline__ float unord32(uint32_t o) {
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o);
}

// Sorting networks on packed u64 keys held in registers (fully unrolled, N a power of two): block
// sort into descending order, and the top-N merge of two descending lists (a <- top N of a and b):
// c_i = max(a_i, b_{N-1-i}) is bitonic, one bitonic merge sorts it.  A compare-exchange is one
// 64-bit compare (2 ISETP) and four selects on ONE predicate: the plain C++ form (x > y ? x : y,
// x > y ? y : x) compiled to separate GT and LT compares, 8 instructions per exchange, and it is
// the router's ALU-bound inner loop (ncu: ALU pipe 76 %).  Keys of one token are distinct (the
// index is in the low word), so every network gives the same sorted list.
__device__ __forceinline__ void ce_desc(unsigned long long& a, unsigned long long& b) {   // a <- max, b <- min
  asm("{\n\t.reg .pred p;\n\t.reg .b64 t;\n\t"
      "setp.gt.u64 p, %0, %1;\n\t"
      "selp.b64 t, %0, %1, p;\n\t"
      "selp.b64 %1, %1, %0, p;\n\t"
      "mov.b64 %0, t;\n\t}"
      : "+l"(a), "+l"(b));
}
__device__ __forceinline__ unsigned long long max_u64(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("{\n\t.reg .pred p;\n\tsetp.gt.u64 p, %1, %2;\n\tselp.b64 %0, %1, %2, p;\n\t}" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
template <int N>
__device__ __forceinline__ void bitonic_sort_desc(unsigned long long (&a)[N]) {
  if constexpr (N == 8) {
    // Batcher's odd-even merge sort: 19 exchanges (bitonic: 24), checked on all 2^8 0/1 inputs
    constexpr int net[19][2] = {{0, 1}, {2, 3}, {4, 5}, {6, 7}, {0, 2}, {1, 3}, {4, 6}, {5, 7}, {1, 2}, {5, 6},
                                {0, 4}, {1, 5}, {2, 6}, {3, 7}, {2, 4}, {3, 5}, {1, 2}, {3, 4}, {5, 6}};
#pragma unroll
    for (int c = 0; c < 19; ++c) ce_desc(a[net[c][0]], a[net[c][1]]);
  } else if constexpr (N == 4) {
    constexpr int net[5][2] = {{0, 1}, {2, 3}, {0, 2}, {1, 3}, {1, 2}};
#pragma unroll
    for (int c = 0; c < 5; ++c) ce_desc(a[net[c][0]], a[net[c][1]]);
  } else {
#pragma unroll
    for (int k = 2; k <= N; k <<= 1)
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const int l = i ^ j;
          if (l > i) {
            if ((i & k) == 0) ce_desc(a[i], a[l]);
            else ce_desc(a[l], a[i]);
          }
        }
  }
}
template <int N>
__device__ __forceinline__ void merge_top_desc(unsigned long long (&a)[N], const unsigned long long (&b)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) a[i] = max_u64(a[i], b[N - 1 - i]);
#pragma unroll
  for (int j = N >> 1; j > 0; j >>= 1)
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int l = i ^ j;
      if (l > i) ce_desc(a[i], a[l]);
    }
}

#endif  // __CUDACC__

// Expert tile descriptor produced by the clustering pass (F4) and consumed by the expert kernels.
struct Tile {
  int32_t head;   // local head
  int32_t expert;
  int32_t row0;   // first sorted replica row of the tile (within the head's R rows)
  int32_t rows;   // valid rows (<= tile height)
};

}  // namespace mhl
