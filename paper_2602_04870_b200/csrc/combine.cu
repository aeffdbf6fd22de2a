// combine.cu — F6 / B6: the k-way combine of Eq. 1, HBM-bound, 16-byte vectorized.
//
// F6: y[t][h*d_h + c] = sum_{j=0..k-1} Yrep[h][pos(t,j)][c]          (gates already applied in F5)
// B6: dXs[t][h*d_h + c] = sum_j dXrep[h][pos(t,j)][c] + sum_j dS[t][j] W_r[h][c][e_j]   (Alg. 2 l.9)
//     (dXrep == nullptr: the router term alone, the routing sub-token's gradient of P:1565-P:1570)
// Lane l owns 16-byte column chunks l, l+32, ... of a (token, head) row.  Sums run in fixed j
// order in fp32 (deterministic), rounded once to the storage type.  Rows are written straight
// into the all-to-all send buffer (row = global token, column block = local head).
#include <cstdlib>

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

constexpr int kCombTok = 128;    // tokens of one head per CTA (F6: 8 warps x 16)
constexpr int kCombTokW = 512;   // B6 with W_r^T staged in smem: 16 warps x 32 tokens per CTA

// One CTA = (head h, 128 consecutive tokens); warp w takes tokens w, w+8, ...  Per token, lanes
// 0..k-1 fetch the k row positions (and for B6 the expert ids / dS) and broadcast them by shuffle;
// every lane then has all k 16-byte row loads of its column chunk in flight at once (KMAX-unrolled).
// B6 keeps W_r^T of the head in shared memory when it fits (SMEM_W), so the router term reads
// smem instead of re-fetching k rows of W_r^T from L2 per token.
template <typename E, bool BWD, int KMAX, bool SMEM_W, bool WIN = false>
__global__ void __launch_bounds__(SMEM_W ? 512 : 256)
combine_kernel(const E* __restrict__ rep, const int32_t* __restrict__ pos, const int32_t* __restrict__ idx,
               const float* __restrict__ dS, const float* __restrict__ W_rT, int H, int64_t T, int k, int d_h,
               int N_e, int64_t Rp, int64_t t0, int64_t nT, E* __restrict__ out, int64_t ldo, int tok_rt,
               int h0, const int32_t* __restrict__ tr, int discard) {
  constexpr int V = Vec<E>::N;
  extern __shared__ __align__(16) float s_w[];           // [N_e][d_h] when SMEM_W
  constexpr int NT = SMEM_W ? 512 : 256, NW = NT / 32;
  const int TOK = SMEM_W ? kCombTokW : tok_rt;   // tokens per CTA (smaller for small T: more CTAs in flight)
  const int h = h0 + (int)blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t tout = t0;               // output row = t - tout
  if constexpr (WIN) {             // windowed combine: head h0's tokens [tr[0], tr[1]), rows absolute
    t0 = tr[0];
    nT = tr[1] - t0;
    tout = 0;
  }
  const int64_t R = T * k;
  const float* wt_h = W_rT + (size_t)h * N_e * d_h;
  if constexpr (BWD && SMEM_W) {
    for (int i = threadIdx.x * 4; i < N_e * d_h; i += NT * 4)
      *reinterpret_cast<float4*>(s_w + i) = __ldg(reinterpret_cast<const float4*>(wt_h + i));
    __syncthreads();
  }
  const int nchunk = d_h / V;
  // tokens [t0, t0 + nT) of the head (one HP destination block, or all T); output row = t - t0
  // token blocks of TOK (grid-stride only for the windowed combine, whose grid does not know its
  // range's size; a plain launch has one block per CTA)
  for (int64_t tb = (int64_t)blockIdx.x * TOK; tb < nT; tb += WIN ? (int64_t)gridDim.x * TOK : nT)
  for (int tt = warp; tt < TOK; tt += NW) {
    if (tb + tt >= nT) break;
    const int64_t t = t0 + tb + tt;
    const size_t rb = (size_t)h * R + t * k;
    const int my_pos = lane < k ? pos[rb + lane] : 0;
    int my_e = 0;
    float my_ds = 0.f;
    if constexpr (BWD) {
      if (lane < k) { my_e = idx[rb + lane]; my_ds = dS[rb + lane]; }
    }
    // all lanes take part in the broadcasts (the column loop below may leave some lanes idle)
    int p[KMAX], ej[KMAX];
    float dsj[KMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
      p[j] = __shfl_sync(0xffffffffu, my_pos, j);
      if constexpr (BWD) { ej[j] = __shfl_sync(0xffffffffu, my_e, j); dsj[j] = __shfl_sync(0xffffffffu, my_ds, j); }
    }
    for (int ch = lane; ch < nchunk; ch += 32) {
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if constexpr (V == 8) {
        uint4 v[KMAX];
#pragma unroll
        for (int j = 0; j < KMAX; ++j)
          if (j < k && rep) v[j] = __ldg(reinterpret_cast<const uint4*>(rep + ((size_t)h * Rp + p[j]) * d_h + ch * V));
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
          if (j < k && rep) {
            float f[8];
            unpack(v[j], f);
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] += f[i];
          }
        }

      } else {
        float4 v[KMAX];
#pragma unroll
        for (int j = 0; j < KMAX; ++j)
          if (j < k && rep) v[j] = __ldg(reinterpret_cast<const float4*>(rep + ((size_t)h * Rp + p[j]) * d_h + ch * V));
#pragma unroll
        for (int j = 0; j < KMAX; ++j)
          if (j < k && rep) { acc[0] += v[j].x; acc[1] += v[j].y; acc[2] += v[j].z; acc[3] += v[j].w; }
      }
      if constexpr (BWD) {
        float racc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
          const float ds = dsj[j];
          const int e = ej[j];
          if (j < k) {
            const float* wr = (SMEM_W ? s_w : wt_h) + (size_t)e * d_h + ch * V;
#pragma unroll
            for (int q = 0; q < V / 4; ++q) {
              const float4 wv = SMEM_W ? *reinterpret_cast<const float4*>(wr + 4 * q)
                                       : __ldg(reinterpret_cast<const float4*>(wr + 4 * q));
              racc[4 * q + 0] = fmaf(ds, wv.x, racc[4 * q + 0]);
              racc[4 * q + 1] = fmaf(ds, wv.y, racc[4 * q + 1]);
              racc[4 * q + 2] = fmaf(ds, wv.z, racc[4 * q + 2]);
              racc[4 * q + 3] = fmaf(ds, wv.w, racc[4 * q + 3]);
            }
          }
        }
#pragma unroll
        for (int i = 0; i < V; ++i) acc[i] += racc[i];
      }
      E* dst = out + (t - tout) * ldo + (int64_t)h * d_h + ch * V;
      if constexpr (V == 8) {
        *reinterpret_cast<uint4*>(dst) = pack(acc);
      } else {
        *reinterpret_cast<float4*>(dst) = make_float4(acc[0], acc[1], acc[2], acc[3]);
      }
    }
    // every replica row is read exactly once: once all lanes have consumed their loads, drop the
    // rows' lines from L2 without a write-back (one lane per 128-byte line; rows are line-aligned)
    if (WIN && discard && rep) {
      __syncwarp();
      for (int ch = lane; ch < nchunk; ch += 32)
        if ((ch & 7) == 0)
#pragma unroll
          for (int j = 0; j < KMAX; ++j)
            if (j < k)
              asm volatile("discard.global.L2 [%0], 128;" ::"l"(rep + ((size_t)h * Rp + p[j]) * d_h + ch * V)
                           : "memory");
    }
  }
}

template <typename E, bool BWD, bool SMEM_W>
void launch_kw(const Routing& rt, const E* rep, const float* dS, const float* W_rT, int d_h, E* out, int64_t ldo,
               int64_t t0, int64_t nT, cudaStream_t s) {
  // tokens per CTA: kCombTok, halved down to 16 until the grid has >= 8 CTAs per SM (148 SMs)
  int tok = SMEM_W ? kCombTokW : kCombTok;
  while (!SMEM_W && tok > 16 && ((nT + tok - 1) / tok) * rt.H < 8 * 148) tok /= 2;
  const dim3 grid((unsigned)((nT + tok - 1) / tok), (unsigned)rt.H);
  const size_t smem = SMEM_W ? (size_t)rt.N_e * d_h * 4 : 0;
#define MHL_CK(KM)                                                                                          \
  {                                                                                                         \
    auto f = combine_kernel<E, BWD, KM, SMEM_W>;                                                            \
    if (smem > 48 * 1024) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
    f<<<grid, SMEM_W ? 512 : 256, smem, s>>>(rep, rt.pos, rt.idx, dS, W_rT, rt.H, rt.T, rt.k, d_h, rt.N_e, rt.Rp, t0, nT, out, ldo, tok, 0, nullptr, 0); \
  }
  if (rt.k <= 2) MHL_CK(2) else if (rt.k <= 4) MHL_CK(4) else if (rt.k <= 8) MHL_CK(8) else MHL_CK(16)
#undef MHL_CK
}

}  // namespace

void launch_combine_window(int dtype, const Routing& rt, const void* rep, int d_h, void* out, int64_t ldo, int h,
                           const int32_t* tr, int64_t max_tokens, bool discard, cudaStream_t s) {
  if (max_tokens <= 0) return;
  static const bool no_discard = getenv("MHL_WIN_DISCARD") && atoi(getenv("MHL_WIN_DISCARD")) == 0;   // A/B
  if (no_discard) discard = false;
  // max_tokens sizes the grid (the range itself is read on the device; the token loop is
  // grid-stride, so any grid covers it)
  int tok = kCombTok;
  while (tok > 16 && (max_tokens + tok - 1) / tok < 8 * 148) tok /= 2;
  const dim3 grid((unsigned)std::min<int64_t>((max_tokens + tok - 1) / tok, 16 * 148), 1u);
#define MHL_CW(E, KM)                                                                                        \
  combine_kernel<E, false, KM, false, true><<<grid, 256, 0, s>>>((const E*)rep, rt.pos, rt.idx, nullptr, nullptr, rt.H, rt.T, \
                                                           rt.k, d_h, rt.N_e, rt.Rp, 0, 0, (E*)out, ldo, tok, h, tr,     \
                                                           discard ? 1 : 0)
  if (dtype == 1) {
    if (rt.k <= 2) MHL_CW(bf16, 2); else if (rt.k <= 4) MHL_CW(bf16, 4); else if (rt.k <= 8) MHL_CW(bf16, 8);
    else MHL_CW(bf16, 16);
  } else {
    if (rt.k <= 2) MHL_CW(float, 2); else if (rt.k <= 4) MHL_CW(float, 4); else if (rt.k <= 8) MHL_CW(float, 8);
    else MHL_CW(float, 16);
  }
#undef MHL_CW
}

void launch_combine_fwd(int dtype, const Routing& rt, const void* Yrep, int d_h, void* out, int64_t ldo,
                        cudaStream_t s, int64_t t0, int64_t nT) {
  if (nT < 0) nT = rt.T - t0;
  if (nT <= 0) return;
  if (dtype == 1)
    launch_kw<bf16, false, false>(rt, (const bf16*)Yrep, nullptr, nullptr, d_h, (bf16*)out, ldo, t0, nT, s);
  else
    launch_kw<float, false, false>(rt, (const float*)Yrep, nullptr, nullptr, d_h, (float*)out, ldo, t0, nT, s);
}

void launch_combine_bwd(int dtype, const Routing& rt, const void* dXrep, const float* dS, const float* W_rT, int d_h,
                        void* out, int64_t ldo, cudaStream_t s, int64_t t0, int64_t nT) {
  if (nT < 0) nT = rt.T - t0;
  if (nT <= 0) return;
  const bool smem_w = (size_t)rt.N_e * d_h * 4 <= 160 * 1024;   // W_r^T of the head in smem (1 CTA/SM above 96 KB)
  if (dtype == 1) {
    if (smem_w) launch_kw<bf16, true, true>(rt, (const bf16*)dXrep, dS, W_rT, d_h, (bf16*)out, ldo, t0, nT, s);
    else launch_kw<bf16, true, false>(rt, (const bf16*)dXrep, dS, W_rT, d_h, (bf16*)out, ldo, t0, nT, s);
  } else {
    if (smem_w) launch_kw<float, true, true>(rt, (const float*)dXrep, dS, W_rT, d_h, (float*)out, ldo, t0, nT, s);
    else launch_kw<float, true, false>(rt, (const float*)dXrep, dS, W_rT, d_h, (float*)out, ldo, t0, nT, s);
  }
}

// Fault injection ("injected fault mode perturbs one kernel by 1e-3 -> suite fails"):
// scales a step's output tensor by f, in place.  Only launched when MHL_FAULT_INJECT names a site.
template <typename E>
__global__ void scale_kernel(E* __restrict__ p, int64_t n, float f) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = from_f<E>(to_f(p[i]) * f);
}

void launch_scale(int dtype, void* p, int64_t n, float f, cudaStream_t s) {
  if (n <= 0) return;
  const unsigned g = (unsigned)std::min<int64_t>((n + 255) / 256, 4096);
  if (dtype == 1) scale_kernel<bf16><<<g, 256, 0, s>>>((bf16*)p, n, f);
  else scale_kernel<float><<<g, 256, 0, s>>>((float*)p, n, f);
}

// dst[i] += src[i] (fp32): one pairwise step of the deterministic DP tree (MHL_FLAG_DET_DP)
__global__ void add_inplace_kernel(float4* __restrict__ dst, const float4* __restrict__ src, int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 a = dst[i];
    const float4 b = src[i];
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    dst[i] = a;
  }
}

void launch_add_inplace(float* dst, const float* src, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  const int64_t n4 = n / 4;   // n is a multiple of 4 (weight matrices with d % 8 == 0)
  add_inplace_kernel<<<(unsigned)std::min<int64_t>((n4 + 255) / 256, 4 * 148), 256, 0, s>>>((float4*)dst,
                                                                                          (const float4*)src, n4);
}

}  // namespace mhl
