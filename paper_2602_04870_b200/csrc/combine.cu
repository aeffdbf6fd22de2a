// combine.cu — F6 / B6: the k-way combine of Eq. 1, HBM-bound, 16-byte vectorized.
//
// F6: y[t][h*d_h + c] = sum_{j=0..k-1} Yrep[h][pos(t,j)][c]          (gates already applied in F5)
// B6: dXs[t][h*d_h + c] = sum_j dXrep[h][pos(t,j)][c] + sum_j dS[t][j] W_r[h][c][e_j]   (Alg. 2 l.9)
// One warp per (token, head); lane l owns 16-byte column chunks l, l+32, ...  Sums run in fixed
// j order in fp32 (deterministic), rounded once to the storage type.  Rows are written straight
// into the all-to-all send buffer (row = global token, column block = local head).
#include "kernels.h"

namespace mhl {

namespace {

template <typename E> struct Vec;
template <> struct Vec<bf16> { static constexpr int N = 8; };
template <> struct Vec<float> { static constexpr int N = 4; };

__device__ __forceinline__ void unpack(const uint4& v, float (&f)[8]) {
  const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) { const float2 t = __bfloat1622float2(p[i]); f[2 * i] = t.x; f[2 * i + 1] = t.y; }
}
__device__ __forceinline__ uint4 pack(const float (&f)[8]) {
  uint4 v;
  __nv_bfloat162* p = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) p[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return v;
}

template <typename E, bool BWD>
__global__ void __launch_bounds__(256)
combine_kernel(const E* __restrict__ rep, const int32_t* __restrict__ pos, const int32_t* __restrict__ idx,
               const float* __restrict__ dS, const float* __restrict__ W_rT, int H, int64_t T, int k, int d_h,
               int N_e, int64_t Rp, E* __restrict__ out, int64_t ldo) {
  constexpr int V = Vec<E>::N;
  const int64_t pair = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (pair >= T * H) return;
  const int lane = threadIdx.x & 31;
  const int h = (int)(pair / T);
  const int64_t t = pair % T;
  const int64_t R = T * k;
  const int32_t* ph = pos + (size_t)h * R + t * k;
  const int nchunk = d_h / V;
  for (int ch = lane; ch < nchunk; ch += 32) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int j = 0; j < k; ++j) {
      const E* src = rep + ((size_t)h * Rp + ph[j]) * d_h + ch * V;
      if constexpr (V == 8) {
        float f[8];
        unpack(__ldg(reinterpret_cast<const uint4*>(src)), f);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += f[i];
      } else {
        const float4 f = __ldg(reinterpret_cast<const float4*>(src));
        acc[0] += f.x; acc[1] += f.y; acc[2] += f.z; acc[3] += f.w;
      }
    }
    if constexpr (BWD) {
      float racc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      const int32_t* ih = idx + (size_t)h * R + t * k;
      const float* sh = dS + (size_t)h * R + t * k;
      const float* wt = W_rT + (size_t)h * N_e * d_h + ch * V;
      for (int j = 0; j < k; ++j) {
        const float ds = sh[j];
        const float4* w = reinterpret_cast<const float4*>(wt + (size_t)ih[j] * d_h);
#pragma unroll
        for (int q = 0; q < V / 4; ++q) {
          const float4 wv = __ldg(w + q);
          racc[4 * q + 0] = fmaf(ds, wv.x, racc[4 * q + 0]);
          racc[4 * q + 1] = fmaf(ds, wv.y, racc[4 * q + 1]);
          racc[4 * q + 2] = fmaf(ds, wv.z, racc[4 * q + 2]);
          racc[4 * q + 3] = fmaf(ds, wv.w, racc[4 * q + 3]);
        }
      }
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] += racc[i];
    }
    E* dst = out + t * ldo + (int64_t)h * d_h + ch * V;
    if constexpr (V == 8) {
      *reinterpret_cast<uint4*>(dst) = pack(acc);
    } else {
      *reinterpret_cast<float4*>(dst) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    }
  }
}

}  // namespace

void launch_combine_fwd(int dtype, const Routing& rt, const void* Yrep, int d_h, void* out, int64_t ldo,
                        cudaStream_t s) {
  const unsigned blocks = (unsigned)((rt.T * rt.H + 7) / 8);
  if (dtype == 1)
    combine_kernel<bf16, false><<<blocks, 256, 0, s>>>((const bf16*)Yrep, rt.pos, nullptr, nullptr, nullptr, rt.H, rt.T,
                                                       rt.k, d_h, 0, rt.Rp, (bf16*)out, ldo);
  else
    combine_kernel<float, false><<<blocks, 256, 0, s>>>((const float*)Yrep, rt.pos, nullptr, nullptr, nullptr, rt.H,
                                                        rt.T, rt.k, d_h, 0, rt.Rp, (float*)out, ldo);
}

void launch_combine_bwd(int dtype, const Routing& rt, const void* dXrep, const float* dS, const float* W_rT, int d_h,
                        void* out, int64_t ldo, cudaStream_t s) {
  const unsigned blocks = (unsigned)((rt.T * rt.H + 7) / 8);
  if (dtype == 1)
    combine_kernel<bf16, true><<<blocks, 256, 0, s>>>((const bf16*)dXrep, rt.pos, rt.idx, dS, W_rT, rt.H, rt.T, rt.k,
                                                      d_h, rt.N_e, rt.Rp, (bf16*)out, ldo);
  else
    combine_kernel<float, true><<<blocks, 256, 0, s>>>((const float*)dXrep, rt.pos, rt.idx, dS, W_rT, rt.H, rt.T,
                                                       rt.k, d_h, rt.N_e, rt.Rp, (float*)out, ldo);
}

}  // namespace mhl
