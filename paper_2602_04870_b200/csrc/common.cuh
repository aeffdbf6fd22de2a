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

// Order-preserving float -> uint32 (R6): flip sign bit of non-negatives, all bits of negatives.
__device__ __forceinline__ uint32_t ord32(float v) {
  uint32_t u = __float_as_uint(v == 0.0f ? 0.0f : v);   // canonicalise -0.0
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ unsigned long long pack_key(float v, int idx) {
  return ((unsigned long long)ord32(v) << 32) | (unsigned long long)(~(uint32_t)idx);
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
