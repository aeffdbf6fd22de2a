// expert_dw_sm100.cu — B5 weight gradients of the block-sparse expert FFN on tcgen05/TMEM (sm_100a).
//
// Chain rule of y_r = g_r * gelu(x W1_e^T) W2_e for the clustered replicas of one expert
// (Eq. 1), with H recomputed instead of stored (the forward never wrote it):
//   kernel dX (per 128-replica tile):
//     H   = X W1_e^T                 (tcgen05, B = W1_e K-major)
//     dA' = dY W2_e^T                (tcgen05, B = W2_e K-major)       dY = dcat rows of the tokens
//     dg  = <gelu(H), dA'>  (= <dY, E_e(x)>, the gate cotangent)
//     dH  = g dA' gelu'(H),   gA = g gelu(H)      (bf16; dH also staged in smem)
//     dXrep = dH W1_e                (tcgen05, B = W1_e read MN-major from the same smem copy)
//   kernel dW (per chunk of <= kDwChunk sorted rows of one expert), no atomics:
//     dW1_e^T += X^T dH,  dW2_e^T += dY^T gA     (tcgen05, both operands MN-major)
//   then an ordered reduction over the expert's chunks (deterministic).
#include "kernels.h"
#include "sm100.cuh"

namespace mhl {

namespace {

using namespace sm100;

constexpr int BM = kExpertBM;
constexpr int kThreads = 256;

__device__ __forceinline__ void gelu_and_grad(float h, float& a, float& da) {
  const float cdf = 0.5f * (1.0f + erff(h * 0.70710678118654752f));
  const float pdf = 0.39894228040143268f * __expf(-0.5f * h * h);
  a = h * cdf;
  da = cdf + h * pdf;
}

// =============================================================================================
// dW kernel: per chunk (<= kDwChunk rows of one (head, expert)), accumulate in TMEM
//   dW1^T[c][f] += sum_r X[r][c] dH[r][f]   dW2^T[c][f] += sum_r dY[r][c] gA[r][f]
// M = c (DH/128 MMAs of M=128), N = f (DE), K = rows (16 per MMA).  Two 64-row stages.
// =============================================================================================
constexpr int kHalf = 64;   // rows per pipeline stage

template <int DH, int DE>
struct DwSmem {
  static constexpr int STAGE = 2 * kHalf * DH * 2 + 2 * kHalf * DE * 2;     // X, dY, dH, gA
  static constexpr int X = 0, DY = kHalf * DH * 2, DHH = 2 * kHalf * DH * 2, GA = DHH + kHalf * DE * 2;
  static constexpr int BAR = 2 * STAGE;            // 2 mbarriers
  static constexpr int TOK = BAR + 16;             // [2][kHalf]
  static constexpr int TMEM = TOK + 2 * kHalf * 4;
  static constexpr int BYTES = TMEM + 16;
};

template <int DH, int DE>
__global__ void __launch_bounds__(kThreads, 1)
expert_dw_kernel(Routing rt, const bf16* __restrict__ Xs, int64_t ldx, const bf16* __restrict__ dY, int64_t ldy,
                 const bf16* __restrict__ dHg, const bf16* __restrict__ gAg, float* __restrict__ partial) {
  const Tile* chunks = rt.chunks;
  const int64_t Rp = rt.Rp;
  using L = DwSmem<DH, DE>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;   // SW128 atoms need 1024-byte alignment (checked below)
  if ((smem_u32(smem) & 1023u) != 0u) __trap();
  const uint32_t sbase = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
  int* s_tok = reinterpret_cast<int*>(smem + L::TOK);
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::TMEM);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tmem_alloc<512>(s_tmem);
  if (tid == 0) { mbar_init(&bars[0], 1); mbar_init(&bars[1], 1); fence_mbar_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  uint32_t ph[2] = {0, 0};
  constexpr int MH = DH / 128;                          // M halves (c blocks of 128)
  constexpr uint32_t IDESC = idesc_bf16(128, DE, 1, 1);
  const int nchunks = *rt.nchunks;

  for (int ci = blockIdx.x; ci < nchunks; ci += gridDim.x) {
    const Tile ch = chunks[ci];
    const int nsteps = (ch.rows + kHalf - 1) / kHalf;
    auto load_stage = [&](int st, int s) {
      const int r0 = s * kHalf;
      int* tok = s_tok + st * kHalf;
      // tokens were written before the preceding __syncthreads()
      const uint32_t base = sbase + st * L::STAGE;
      for (int i = tid; i < kHalf * DH / 8; i += kThreads) {
        const int r = i / (DH / 8), c = (i % (DH / 8)) * 8;
        const size_t so = (size_t)tok[r];   // padding rows: the zero row
        cp_async_16(base + L::X + kmaj_off(r, c, kHalf), Xs + so * ldx + (size_t)ch.head * DH + c, 16);
        cp_async_16(base + L::DY + kmaj_off(r, c, kHalf), dY + so * ldy + (size_t)ch.head * DH + c, 16);
      }
      for (int i = tid; i < kHalf * DE / 8; i += kThreads) {
        const int r = i / (DE / 8), c = (i % (DE / 8)) * 8;
        const size_t grow = (size_t)ch.head * Rp + ch.row0 + r0 + r;   // chunk rows are whole tiles
        cp_async_16(base + L::DHH + kmaj_off(r, c, kHalf), dHg + grow * DE + c, 16);
        cp_async_16(base + L::GA + kmaj_off(r, c, kHalf), gAg + grow * DE + c, 16);
      }
      cp_async_commit();
    };
    auto load_tokens = [&](int st, int s) {
      if (tid < kHalf) s_tok[st * kHalf + tid] = rt.tok_s[(size_t)ch.head * Rp + ch.row0 + s * kHalf + tid];
    };
    load_tokens(0, 0);
    __syncthreads();
    load_stage(0, 0);
    for (int s = 0; s < nsteps; ++s) {
      const int st = s & 1;
      // prefetch step s+1 into the other stage once its previous MMAs (step s-1) are done
      if (s + 1 < nsteps) {
        if (s >= 1) { mbar_wait(&bars[st ^ 1], ph[st ^ 1]); ph[st ^ 1] ^= 1; }
        load_tokens(st ^ 1, s + 1);
        __syncthreads();
        load_stage(st ^ 1, s + 1);
        cp_async_wait_group<1>();
      } else {
        cp_async_wait_group<0>();
      }
      fence_proxy_async();
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        const uint32_t base = sbase + st * L::STAGE;
#pragma unroll
        for (int ks = 0; ks < kHalf / 16; ++ks) {
          const uint32_t ko = ks * 2 * 1024;              // 16 rows = 2 K-groups of 8
#pragma unroll
          for (int m = 0; m < MH; ++m) {
            const uint32_t acc = (s > 0 || ks > 0) ? 1u : 0u;
            // A = X^T (MN-major: c atoms at kHalf*128 B, row groups at 1024 B); B = dH^T likewise
            mma_bf16(tmem + m * DE, sdesc_sw128(base + L::X + m * 2 * kHalf * 128 + ko, kHalf * 128, 1024),
                     sdesc_sw128(base + L::DHH + ko, kHalf * 128, 1024), IDESC, acc);
            mma_bf16(tmem + 256 + m * DE, sdesc_sw128(base + L::DY + m * 2 * kHalf * 128 + ko, kHalf * 128, 1024),
                     sdesc_sw128(base + L::GA + ko, kHalf * 128, 1024), IDESC, acc);
          }
        }
        mma_commit(&bars[st]);
      }
    }
    // drain: wait for the last step's MMAs (and the one before, if not yet waited)
    {
      const int last = (nsteps - 1) & 1;
      if (nsteps >= 2) { mbar_wait(&bars[last ^ 1], ph[last ^ 1]); ph[last ^ 1] ^= 1; }
      mbar_wait(&bars[last], ph[last]); ph[last] ^= 1;
    }
    tc_fence_after();
    // ---- epilogue: partial[ci][mat][f][c]  (thread = c row of the M block, coalesced over c)
    {
      const int q = warp & 3, wm = warp >> 2;            // warps 0-3: dW1, 4-7: dW2
      float* out = partial + ((size_t)ci * 2 + wm) * DE * DH;
      for (int m = 0; m < MH; ++m) {
        const int c = m * 128 + q * 32 + lane;
        for (int f0 = 0; f0 < DE; f0 += 32) {
          uint32_t v[32];
          tmem_ld32(tmem + wm * 256 + m * DE + ((uint32_t)(q * 32) << 16) + f0, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) out[(size_t)(f0 + j) * DH + c] = __uint_as_float(v[j]);
        }
      }
    }
    tc_fence_before();
    __syncthreads();
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

// dW[h][e][f][c] = sum over the expert's chunks, in chunk order (deterministic); 0 if unused
__global__ void __launch_bounds__(256)
dw_reduce_kernel(const float* __restrict__ partial, const int32_t* __restrict__ cbase,
                 const int32_t* __restrict__ ccount, int N_e, int DEDH, float* __restrict__ dW1,
                 float* __restrict__ dW2) {
  const int e = blockIdx.y, h = blockIdx.z;
  const int he = h * N_e + e;
  const int b = cbase[he], n = ccount[he];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < DEDH; i += gridDim.x * blockDim.x) {
    float a1 = 0.f, a2 = 0.f;
    for (int c = 0; c < n; ++c) {
      a1 += partial[((size_t)(b + c) * 2 + 0) * DEDH + i];
      a2 += partial[((size_t)(b + c) * 2 + 1) * DEDH + i];
    }
    if (dW1) dW1[(size_t)he * DEDH + i] = a1;
    if (dW2) dW2[(size_t)he * DEDH + i] = a2;
  }
}

template <typename K>
void set_smem(K k, int bytes) { cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes); }

}  // namespace

bool expert_bwd_sm100_supported(int d_h, int d_e) {
  return (d_h == 256 && d_e == 128) || (d_h == 256 && d_e == 64) || (d_h == 128 && d_e == 128) ||
         (d_h == 128 && d_e == 64);
}

bool launch_expert_bwd_sm100(const Routing& rt, const void* Xs, int64_t ldx, const void* dY, int64_t ldy,
                             const void* W1, const void* W2, int d_h, int d_e, void* dXrep, float* dg, void* dH,
                             void* gA, float* partial, float* dW1, float* dW2, int num_sms, cudaStream_t s,
                             bool do_dx, bool do_dw) {
  bool ok = false;
#define MHL_BWD_CASE(A, B)                                                                                       \
  if (d_h == A && d_e == B) {                                                                                    \
    ok = true;                                                                                                   \
    if (do_dx && !launch_expert_bwd_dx_sm100(rt, Xs, ldx, dY, ldy, W1, W2, d_h, d_e, dXrep, dg, dH, gA,       \
                                             num_sms, s))                                                        \
      ok = false;                                                                                                \
    if (do_dw) {                                                                                                 \
      auto kern = expert_dw_kernel<A, B>;                                                                        \
      set_smem(kern, DwSmem<A, B>::BYTES);                                                                       \
      kern<<<num_sms, kThreads, DwSmem<A, B>::BYTES, s>>>(rt, (const bf16*)Xs, ldx, (const bf16*)dY, ldy,        \
                                                          (const bf16*)dH, (const bf16*)gA, partial);            \
    }                                                                                                            \
  }
  MHL_BWD_CASE(256, 128) else MHL_BWD_CASE(256, 64) else MHL_BWD_CASE(128, 128) else MHL_BWD_CASE(128, 64)
#undef MHL_BWD_CASE
  if (ok && do_dw && (dW1 || dW2)) {
    const int dedh = d_e * d_h;
    dw_reduce_kernel<<<dim3((dedh + 255) / 256, rt.N_e, rt.H), 256, 0, s>>>(partial, rt.cbase, rt.ccount, rt.N_e, dedh,
                                                                            dW1, dW2);
  }
  return ok;
}

}  // namespace mhl
