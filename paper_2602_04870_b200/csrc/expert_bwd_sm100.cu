// expert_bwd_sm100.cu — B5: block-sparse expert FFN backward on tcgen05/TMEM (sm_100a).
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
// dX kernel
// =============================================================================================
template <int DH, int DE>
struct DxSmem {
  static constexpr int W1 = 0;                        // [DE][DH] K-major SW128
  static constexpr int W2 = W1 + DE * DH * 2;         // [DE][DH] K-major SW128
  static constexpr int XY = W2 + DE * DH * 2;         // [BM][DH] K-major: X, then dY
  static constexpr int DHS = XY + BM * DH * 2;        // [BM][DE] K-major: dH (A operand of GEMM dX)
  static constexpr int BAR = DHS + BM * DE * 2;
  static constexpr int TOK = BAR + 16;
  static constexpr int REP = TOK + BM * 4;
  static constexpr int GATE = REP + BM * 4;
  static constexpr int DG = GATE + BM * 4;            // [2][BM] partial dg per column half
  static constexpr int TMEM = DG + 2 * BM * 4;
  static constexpr int BYTES = TMEM + 16;
};

template <int DH, int DE>
__device__ __forceinline__ void gather_rows(uint32_t dst, const int* s_tok, const bf16* src, int64_t ld,
                                            int head, int tid) {
  for (int i = tid; i < BM * DH / 8; i += kThreads) {
    const int row = i / (DH / 8), c = (i % (DH / 8)) * 8;
    cp_async_16(dst + kmaj_off(row, c, BM), src + (size_t)s_tok[row] * ld + (size_t)head * DH + c, 16);
  }
}

template <int DH, int DE>
__global__ void __launch_bounds__(kThreads, 1)
expert_bwd_dx_kernel(Routing rt, const bf16* __restrict__ Xs, int64_t ldx, const bf16* __restrict__ dY, int64_t ldy,
                     const bf16* __restrict__ W1, const bf16* __restrict__ W2, bf16* __restrict__ dXrep,
                     float* __restrict__ dg, bf16* __restrict__ dHg, bf16* __restrict__ gAg) {
  const Tile* tiles = rt.tiles;
  const int N_e = rt.N_e;
  const int64_t Rp = rt.Rp, R = rt.T * rt.k;
  using L = DxSmem<DH, DE>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;   // SW128 atoms need 1024-byte alignment (checked below)
  if ((smem_u32(smem) & 1023u) != 0u) __trap();
  const uint32_t sbase = smem_u32(smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::BAR);
  int* s_tok = reinterpret_cast<int*>(smem + L::TOK);
  int* s_rep = reinterpret_cast<int*>(smem + L::REP);
  float* s_gate = reinterpret_cast<float*>(smem + L::GATE);
  float* s_dg = reinterpret_cast<float*>(smem + L::DG);
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::TMEM);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (warp == 0) tmem_alloc<512>(s_tmem);
  if (tid == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  const uint32_t tH = tmem, tD = tmem + DE, tX = tmem + 256;   // H [0,DE), dA' [DE,2DE), dX [256,256+DH)
  uint32_t phase = 0;
  const int nt = *rt.ntiles;
  const int ngroups = (nt + kTileGroup - 1) / kTileGroup;   // see expert_sm100.cu: L2-local schedule
  const int my_groups = ngroups > (int)blockIdx.x ? (ngroups - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  int cur_h = -1, cur_e = -1;
  constexpr uint32_t IDESC_H = idesc_bf16(BM, DE, 0, 0);
  constexpr uint32_t IDESC_X = idesc_bf16(BM, DH, 0, 1);
  const int q = warp & 3, half = warp >> 2, row = q * 32 + lane;

  for (int v = 0; v < my_groups * kTileGroup; ++v) {
    const int ti = ((int)blockIdx.x + (v / kTileGroup) * (int)gridDim.x) * kTileGroup + v % kTileGroup;
    if (ti >= nt) break;
    const Tile tl = tiles[ti];
    if (tid < BM) {
      const size_t q0 = (size_t)tl.head * Rp + tl.row0 + tid;
      s_tok[tid] = rt.tok_s[q0]; s_rep[tid] = rt.perm[q0]; s_gate[tid] = rt.gate_s[q0];
    }
    __syncthreads();
    if (tl.head != cur_h || tl.expert != cur_e) {
      const size_t wofs = ((size_t)tl.head * N_e + tl.expert) * DE * DH;
      for (int i = tid; i < DE * DH / 8; i += kThreads) {
        const int r = i / (DH / 8), c = (i % (DH / 8)) * 8;
        cp_async_16(sbase + L::W1 + kmaj_off(r, c, DE), W1 + wofs + (size_t)r * DH + c, 16);
        cp_async_16(sbase + L::W2 + kmaj_off(r, c, DE), W2 + wofs + (size_t)r * DH + c, 16);
      }
      cur_h = tl.head; cur_e = tl.expert;
    }
    gather_rows<DH, DE>(sbase + L::XY, s_tok, Xs, ldx, tl.head, tid);
    cp_async_commit();
    cp_async_wait_all();
    fence_proxy_async();
    __syncthreads();
    // ---- H = X W1^T
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int ks = 0; ks < DH / 16; ++ks) {
        const uint32_t ko = (ks >> 2), kk = (ks & 3) * 32;
        mma_bf16(tH, sdesc_sw128(sbase + L::XY + ko * BM * 128 + kk, 16, 1024),
                 sdesc_sw128(sbase + L::W1 + ko * DE * 128 + kk, 16, 1024), IDESC_H, ks > 0);
      }
      mma_commit(bar);
    }
    mbar_wait(bar, phase); phase ^= 1;
    // ---- dY rows into the same buffer, then dA' = dY W2^T
    gather_rows<DH, DE>(sbase + L::XY, s_tok, dY, ldy, tl.head, tid);
    cp_async_commit();
    cp_async_wait_all();
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int ks = 0; ks < DH / 16; ++ks) {
        const uint32_t ko = (ks >> 2), kk = (ks & 3) * 32;
        mma_bf16(tD, sdesc_sw128(sbase + L::XY + ko * BM * 128 + kk, 16, 1024),
                 sdesc_sw128(sbase + L::W2 + ko * DE * 128 + kk, 16, 1024), IDESC_H, ks > 0);
      }
      mma_commit(bar);
    }
    mbar_wait(bar, phase); phase ^= 1;
    tc_fence_after();
    // ---- epilogue: dg, dH, gA
    {
      const float g = s_gate[row];
      const size_t grow = (size_t)tl.head * Rp + tl.row0 + row;
      float dgp = 0.f;
      for (int c0 = half * (DE / 2); c0 < (half + 1) * (DE / 2); c0 += 32) {
        uint32_t hv[32], dv[32];
        tmem_ld32(tH + ((uint32_t)(q * 32) << 16) + c0, hv);
        tmem_ld32(tD + ((uint32_t)(q * 32) << 16) + c0, dv);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          float dh[8], ga[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            float a, dga;
            const float h = __uint_as_float(hv[j + u]);
            const float da = __uint_as_float(dv[j + u]);
            gelu_and_grad(h, a, dga);
            dgp = fmaf(a, da, dgp);
            dh[u] = g * da * dga;
            ga[u] = g * a;
          }
          uint4 p1, p2;
          p1.x = pack_bf16x2(dh[0], dh[1]); p1.y = pack_bf16x2(dh[2], dh[3]);
          p1.z = pack_bf16x2(dh[4], dh[5]); p1.w = pack_bf16x2(dh[6], dh[7]);
          p2.x = pack_bf16x2(ga[0], ga[1]); p2.y = pack_bf16x2(ga[2], ga[3]);
          p2.z = pack_bf16x2(ga[4], ga[5]); p2.w = pack_bf16x2(ga[6], ga[7]);
          *reinterpret_cast<uint4*>(smem + L::DHS + kmaj_off(row, c0 + j, BM)) = p1;
          *reinterpret_cast<uint4*>(dHg + grow * DE + c0 + j) = p1;   // padding rows: g = 0 -> zeros
          *reinterpret_cast<uint4*>(gAg + grow * DE + c0 + j) = p2;
        }
      }
      s_dg[half * BM + row] = dgp;
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    if (tid < BM && s_rep[tid] >= 0) dg[(size_t)tl.head * R + s_rep[tid]] = s_dg[tid] + s_dg[BM + tid];
    // ---- dXrep = dH W1   (B = W1 viewed MN-major: N = DH atoms at DE*128 B, K groups at 1024 B)
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int ks = 0; ks < DE / 16; ++ks) {
        mma_bf16(tX, sdesc_sw128(sbase + L::DHS + (ks >> 2) * BM * 128 + (ks & 3) * 32, 16, 1024),
                 sdesc_sw128(sbase + L::W1 + ks * 2 * 1024, DE * 128, 1024), IDESC_X, ks > 0);
      }
      mma_commit(bar);
    }
    mbar_wait(bar, phase); phase ^= 1;
    tc_fence_after();
    {
      bf16* dst = dXrep + ((size_t)tl.head * Rp + tl.row0 + row) * DH;
      for (int c0 = half * (DH / 2); c0 < (half + 1) * (DH / 2); c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tX + ((uint32_t)(q * 32) << 16) + c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          uint4 pk;
          pk.x = pack_bf16x2(__uint_as_float(v[j + 0]), __uint_as_float(v[j + 1]));
          pk.y = pack_bf16x2(__uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
          pk.z = pack_bf16x2(__uint_as_float(v[j + 4]), __uint_as_float(v[j + 5]));
          pk.w = pack_bf16x2(__uint_as_float(v[j + 6]), __uint_as_float(v[j + 7]));
          *reinterpret_cast<uint4*>(dst + c0 + j) = pk;
        }
      }
    }
    tc_fence_before();
    __syncthreads();
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
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
    if (do_dx) {                                                                                                 \
      auto kern = expert_bwd_dx_kernel<A, B>;                                                                    \
      set_smem(kern, DxSmem<A, B>::BYTES);                                                                       \
      kern<<<num_sms, kThreads, DxSmem<A, B>::BYTES, s>>>(rt, (const bf16*)Xs, ldx, (const bf16*)dY, ldy,        \
                                                          (const bf16*)W1, (const bf16*)W2, (bf16*)dXrep, dg,    \
                                                          (bf16*)dH, (bf16*)gA);                                 \
    }                                                                                                            \
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
