// router_sm100.cu — F3 on tcgen05: router GEMM + online top-k + gates (Alg. 1, P:819-P:841).
//
// Per CTA: a contiguous run of (head, 128-token tile) work items.  The fp32 router weights of the
// head are split once per call into three bf16 planes W_r = w1 + w2 + w3 (24 significant bits;
// the stored sub-token X is exact bf16), so S = X w1 + X w2 + X w3 is an fp32-accurate score
// (R3) computed on the tensor cores with fp32 accumulation in TMEM.  The score tile never
// leaves TMEM/registers (P:336-P:337): the epilogue warps read their token's row, add the bias,
// pack (score, ~index) keys (R6), keep the running top-k in registers, form the gates from
// the raw scores (R4) and emit the per-tile expert histogram for clustering (F4).
//
// Warp roles: warp 0 = TMA producer (X tiles in 64-column K-chunks through an smem ring, W planes
// once per head), warp 1 = MMA issuer (+ TMEM owner), warps 2.. = epilogue.  The TMEM accumulator
// holds kNB = 2*kEG buffers: kEG epilogue warpgroups each work on their own tile while the MMAs of
// later tiles proceed (the top-k is ALU-bound; one warpgroup left the ALU pipe half idle).
#include <cuda.h>

#include "kernels.h"
#include "sm100.cuh"
#include "tma_host.h"

namespace mhl {

namespace {

using namespace sm100;

constexpr int RT = kRouterTile;   // 128 tokens = MMA M
constexpr int kChunkBytes = RT * 128;   // one 64-column K-chunk of the X tile

template <int DH, int NE>
struct RSmem {
  // epilogue warpgroups (each owns every kEG-th tile of the CTA); fewer when the W planes fill smem
#ifndef MHL_ROUTER_EG
#define MHL_ROUTER_EG 3
#endif
  static constexpr int kEG = NE <= 64 ? MHL_ROUTER_EG : 2;
  static constexpr int THREADS = (2 + 4 * kEG) * 32;
  static constexpr int kNB = (2 * kEG * NE <= 512) ? 2 * kEG : 512 / NE;   // TMEM accumulator buffers
  static_assert(kNB >= kEG, "router: fewer TMEM buffers than epilogue warpgroups");
  static constexpr int W = 0;                                   // [3][DH/64][NE][64] SW128
  static constexpr int WBYTES = 3 * NE * DH * 2;
  static constexpr int RING = WBYTES;                           // X chunks
  static constexpr int STAGES_RAW = (225 * 1024 - WBYTES) / kChunkBytes;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int BAR = RING + STAGES * kChunkBytes;       // full[S], empty[S], wfull, wfree, tfull[NB], tempty[NB]
  static constexpr int NBAR = 2 * STAGES + 2 + 2 * kNB;
  static constexpr int BIAS = BAR + NBAR * 8;                   // [kEG][NE]
  static constexpr int HIST = BIAS + kEG * NE * 4;              // [kEG][NE]
  static constexpr int TMEMP = HIST + kEG * NE * 4;
  static constexpr int BYTES = TMEMP + 16;
  static_assert(BYTES <= 227 * 1024, "router: shared memory over the 227 KB per-CTA limit");
  static constexpr int TMEM_COLS = (kNB * NE <= 32) ? 32 : (kNB * NE <= 64) ? 64 : (kNB * NE <= 128) ? 128
                                   : (kNB * NE <= 256) ? 256 : 512;

};

template <int DH, int NE, int KMAX>
__global__ void __launch_bounds__(RSmem<DH, NE>::THREADS, 1)
router_sm100_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap wmap,
                    const float* __restrict__ bias, int H, int64_t T, int k, int32_t* __restrict__ idx,
                    float* __restrict__ gate, int32_t* __restrict__ hist, int32_t* __restrict__ flag) {
  using L = RSmem<DH, NE>;
  constexpr int S = L::STAGES;
  constexpr int KB = DH / 64;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0u) __trap();
  const uint32_t sbase = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* wfull = bars + 2 * S;
  uint64_t* wfree = wfull + 1;
  uint64_t* tfull = wfull + 2;
  constexpr int kNB = L::kNB, kEG = L::kEG, kThreads = L::THREADS;
  uint64_t* tempty = tfull + kNB;
  float* s_bias = reinterpret_cast<float*>(smem + L::BIAS);
  int* s_hist = reinterpret_cast<int*>(smem + L::HIST);
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::TMEMP);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const int n_rt = (int)((T + RT - 1) / RT);
  const int total = H * n_rt;
  const int per = (total + gridDim.x - 1) / gridDim.x;
  const int tb = min(total, (int)blockIdx.x * per), te = min(total, tb + per);

  if (tid == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(wfull, 1); mbar_init(wfree, 1);
    for (int i = 0; i < kNB; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 128); }
    fence_mbar_init();
    tma_prefetch_desc(&xmap); tma_prefetch_desc(&wmap);
  }
  if (warp == 1) tmem_alloc<L::TMEM_COLS>(s_tmem);
  for (int i = tid; i < kEG * NE; i += kThreads) s_hist[i] = 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  if (warp == 0) {
    // ============================ TMA producer
    if (lane == 0) {
      int stage = 0; uint32_t ph = 0, wfph = 0;
      int cur_h = -1;
      for (int ti = tb; ti < te; ++ti) {
        const int h = ti / n_rt, t0 = (ti % n_rt) * RT;
        if (h != cur_h) {
          if (cur_h >= 0) { mbar_wait(wfree, wfph); wfph ^= 1; }
          mbar_expect_tx(wfull, L::WBYTES);
          for (int p = 0; p < 3; ++p)
            for (int kb = 0; kb < KB; ++kb)
              tma_load_2d(sbase + L::W + (p * KB + kb) * NE * 128, &wmap, kb * 64, (h * 3 + p) * NE, wfull);
          cur_h = h;
        }
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&empty[stage], ph ^ 1);
          mbar_expect_tx(&full[stage], kChunkBytes);
          tma_load_2d(sbase + L::RING + stage * kChunkBytes, &xmap, h * DH + kb * 64, t0, &full[stage]);
          if (++stage == S) { stage = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer
    if (lane == 0) {
      constexpr uint32_t IDESC = idesc_bf16(128, NE, 0, 0);
      int stage = 0; uint32_t ph = 0, wph = 0;
      int cur_h = -1, n = 0;
      for (int ti = tb; ti < te; ++ti, ++n) {
        const int h = ti / n_rt;
        if (h != cur_h) { mbar_wait(wfull, wph); wph ^= 1; cur_h = h; }
        const int acc = n % kNB;
        mbar_wait(&tempty[acc], ((n / kNB) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * NE;
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&full[stage], ph);
          tc_fence_after();
          const uint32_t xa = sbase + L::RING + stage * kChunkBytes;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
#pragma unroll
            for (int p = 0; p < 3; ++p)
              mma_bf16(d, sdesc_sw128(xa + ks * 32, 16, 1024),
                       sdesc_sw128(sbase + L::W + (p * KB + kb) * NE * 128 + ks * 32, 16, 1024), IDESC,
                       (kb | ks | p) ? 1u : 0u);
          mma_commit(&empty[stage]);
          if (++stage == S) { stage = 0; ph ^= 1; }
        }
        mma_commit(&tfull[acc]);
        const bool head_ends = (ti + 1 >= te) || ((ti + 1) / n_rt != h);
        if (head_ends) mma_commit(wfree);
      }
    }
  } else {
    // ============================ epilogue: kEG warpgroups of 4 warps, thread = token row;
    // warpgroup g takes the CTA's tiles n = g, g + kEG, ... (accumulator buffer n % kNB)
    const int q = warp & 3, g = (warp - 2) >> 2;
    const int row = q * 32 + lane;
    const int et = (tid - 64) & 127;            // 0..127 within the warpgroup
    float* s_bias_g = s_bias + g * NE;
    int* s_hist_g = s_hist + g * NE;
    int cur_h = -1;
    bool bad = false;
    for (int ti = tb + g, n = g; ti < te; ti += kEG, n += kEG) {
      const int h = ti / n_rt, rt = ti % n_rt;
      if (h != cur_h) {
        named_bar_sync(1 + g, 128);
        for (int i = et; i < NE; i += 128) s_bias_g[i] = bias[(size_t)h * NE + i];
        named_bar_sync(1 + g, 128);
        cur_h = h;
      }
      const int acc = n % kNB;
      mbar_wait(&tfull[acc], (n / kNB) & 1);
      tc_fence_after();
      // Alg. 1 (P:829-P:834) in registers: the scores of each block of KMAX experts become packed
      // u64 keys (ord32(s + b) << 32 | ~e, P:832 / R6: a larger key wins, equal keys go to the lower
      // index), the block is sorted by a bitonic network and merged into the running top-KMAX (the
      // max of the running list against the reversed block is bitonic; one bitonic merge sorts it).
      // Branch-free: the former per-candidate insertion diverged in every warp (some lane nearly
      // always inserted), which made the router ALU-bound (ncu r2c: ALU pipe 69 %).
      unsigned long long top[KMAX];
      float chk = 0.f;   // becomes NaN if any key is NaN or +-Inf (0 * inf = NaN)
#pragma unroll 1
      for (int c0 = 0; c0 < NE; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + acc * NE + ((uint32_t)(q * 32) << 16) + c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int b0 = 0; b0 < 32; b0 += KMAX) {
          unsigned long long blk[KMAX];
#pragma unroll
          for (int u = 0; u < KMAX; ++u) {
            const float kf = __uint_as_float(v[b0 + u]) + s_bias_g[c0 + b0 + u];
            chk = fmaf(kf, 0.f, chk);
            blk[u] = pack_key(kf, c0 + b0 + u);
          }
          bitonic_sort_desc<KMAX>(blk);
          if (c0 == 0 && b0 == 0) {
#pragma unroll
            for (int u = 0; u < KMAX; ++u) top[u] = blk[u];
          } else {
            merge_top_desc<KMAX>(top, blk);
          }
        }
      }
      int kid[KMAX];
      float sraw[KMAX];
#pragma unroll
      for (int j = 0; j < KMAX; ++j) {
        kid[j] = (int)(~(uint32_t)top[j]);
        // raw score for the gates (R4): the biased key minus the bias (R25: within one fp32 rounding
        // of the score itself)
        sraw[j] = unord32((uint32_t)(top[j] >> 32)) - s_bias_g[kid[j]];
      }
      bad |= (chk != 0.f);
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      const int64_t t = (int64_t)rt * RT + row;
      if (t < T) {
        float m = sraw[0];
#pragma unroll
        for (int j = 1; j < KMAX; ++j) if (j < k) m = fmaxf(m, sraw[j]);
        float ex[KMAX], sum = 0.f;
#pragma unroll
        for (int j = 0; j < KMAX; ++j) { ex[j] = (j < k) ? expf(sraw[j] - m) : 0.f; sum += ex[j]; }
        const float inv = 1.0f / sum;
        int32_t* io = idx + ((size_t)h * T + t) * k;
        float* go = gate + ((size_t)h * T + t) * k;
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
          if (j < k) {
            const int e = kid[j];
            io[j] = e;
            go[j] = ex[j] * inv;
            atomicAdd(&s_hist_g[e], 1);
          }
        }
      }
      named_bar_sync(1 + g, 128);
      int32_t* ho = hist + ((size_t)h * n_rt + rt) * NE;
      for (int i = et; i < NE; i += 128) { ho[i] = s_hist_g[i]; s_hist_g[i] = 0; }
      named_bar_sync(1 + g, 128);
    }
    if (bad) *flag = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<L::TMEM_COLS>(tmem);
}

// planes[h][p][n][c] = bf16 split of W_r[h][c][n]:  w1 = rn(w), w2 = rn(w - w1), w3 = rn(w - w1 - w2)
__global__ void router_split_kernel(const float* __restrict__ W_r, bf16* __restrict__ planes, int H, int d_h,
                                    int N_e) {
  const int64_t n = (int64_t)H * d_h * N_e;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % d_h);
    const int e = (int)((i / d_h) % N_e);
    const int h = (int)(i / ((int64_t)d_h * N_e));
    const float w = W_r[((size_t)h * d_h + c) * N_e + e];
    const bf16 w1 = __float2bfloat16_rn(w);
    const float r1 = w - __bfloat162float(w1);
    const bf16 w2 = __float2bfloat16_rn(r1);
    const bf16 w3 = __float2bfloat16_rn(r1 - __bfloat162float(w2));
    const size_t base = ((size_t)h * 3 * N_e + e) * d_h + c;
    planes[base] = w1;
    planes[base + (size_t)N_e * d_h] = w2;
    planes[base + (size_t)2 * N_e * d_h] = w3;
  }
}

template <int DH, int NE, int KMAX>
bool launch_t(const void* Xs, int64_t ldx, const bf16* planes, const float* bias, int H, int64_t T, int k,
              int32_t* idx, float* gate, int32_t* hist, int32_t* flag, int num_sms, cudaStream_t s) {
  CUtensorMap xm, wm;
  if (!make_tmap_2d_bf16(&xm, Xs, (uint64_t)T, (uint64_t)H * DH, (uint64_t)ldx * 2, RT, 64)) return false;
  if (!make_tmap_2d_bf16(&wm, planes, (uint64_t)H * 3 * NE, DH, (uint64_t)DH * 2, NE, 64)) return false;
  auto kern = router_sm100_kernel<DH, NE, KMAX>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, RSmem<DH, NE>::BYTES);
  const int n_rt = (int)((T + RT - 1) / RT);
  const int grid = std::min(num_sms, H * n_rt);
  kern<<<grid, RSmem<DH, NE>::THREADS, RSmem<DH, NE>::BYTES, s>>>(xm, wm, bias, H, T, k, idx, gate, hist, flag);
  return true;
}

template <int DH, int NE>
bool launch_k(const void* Xs, int64_t ldx, const bf16* planes, const float* bias, int H, int64_t T, int k,
              int32_t* idx, float* gate, int32_t* hist, int32_t* flag, int num_sms, cudaStream_t s) {
  if (k <= 2) return launch_t<DH, NE, 2>(Xs, ldx, planes, bias, H, T, k, idx, gate, hist, flag, num_sms, s);
  if (k <= 4) return launch_t<DH, NE, 4>(Xs, ldx, planes, bias, H, T, k, idx, gate, hist, flag, num_sms, s);
  if (k <= 8) return launch_t<DH, NE, 8>(Xs, ldx, planes, bias, H, T, k, idx, gate, hist, flag, num_sms, s);
  return launch_t<DH, NE, 16>(Xs, ldx, planes, bias, H, T, k, idx, gate, hist, flag, num_sms, s);
}

}  // namespace

bool router_sm100_supported(int d_h, int N_e) {
  // N_e must be a multiple of 32 (the epilogue reads 32 TMEM columns at a time)
  return (d_h == 256 && (N_e == 64 || N_e == 128)) || (d_h == 192 && N_e == 64) || (d_h == 128 && N_e == 64) ||
         (d_h == 64 && N_e == 64) || (d_h == 64 && N_e == 32);
}

size_t router_sm100_planes_bytes(int H, int d_h, int N_e) { return (size_t)H * 3 * N_e * d_h * 2; }

void launch_router_split(const float* W_r, void* planes, int H, int d_h, int N_e, cudaStream_t s) {
  const int64_t n = (int64_t)H * d_h * N_e;
  router_split_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, s>>>(W_r, (bf16*)planes, H, d_h,
                                                                                         N_e);
}

bool launch_router_sm100(const void* Xs, int64_t ldx, const float* W_r, const float* bias, int H, int64_t T, int d_h,
                         int N_e, int k, void* planes, int32_t* idx, float* gate, int32_t* hist, int32_t* flag,
                         int num_sms, cudaStream_t s) {
  launch_router_split(W_r, planes, H, d_h, N_e, s);
  const bf16* pl = (const bf16*)planes;
#define MHL_R(A, B) \
  if (d_h == A && N_e == B) return launch_k<A, B>(Xs, ldx, pl, bias, H, T, k, idx, gate, hist, flag, num_sms, s);
  MHL_R(256, 64) MHL_R(256, 128) MHL_R(192, 64) MHL_R(128, 64) MHL_R(64, 64) MHL_R(64, 32)
#undef MHL_R
  return false;
}

}  // namespace mhl
