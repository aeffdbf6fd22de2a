// router_blk_sm100.cu — F3 on tcgen05 for many experts per head: Alg. 1's online top-k over expert
// blocks (P:819-P:841), for the paper's own shapes (N_e = 384-1536 per head, Tables 4-5).
//
// Same arithmetic as router_sm100.cu (fp32-accurate scores S = X w1 + X w2 + X w3 from the three
// bf16 planes of W_r, R3; bias added for selection only; gates from the raw scores, R4),
// but the head's W_r no longer fits in shared memory, so Alg. 1 is followed literally: for each
// 128-token tile, expert blocks of EB = 64 (line 5) are streamed through a two-slot smem ring, each
// block's score tile goes to TMEM (line 7) and is merged into the running top-k held in registers
// (lines 8-10, packed-key order R6 realised by visiting experts in index order with a strict >).
// The T x N_e score matrix never reaches HBM (P:336-P:337).
//
// Warp roles: warp 0 = TMA producer (X tile, then the W blocks of the tile's head), warp 1 = MMA
// issuer + TMEM owner (score buffers: kNB x EB columns), warps 2-5 = epilogue (thread = token).
#include <cuda.h>

#include "kernels.h"
#include "sm100.cuh"
#include "tma_host.h"

namespace mhl {

namespace {

using namespace sm100;

constexpr int RT = kRouterTile;          // 128 tokens = MMA M
constexpr int EB = 64;                   // experts per block (MMA N)
constexpr int kNB = 4;                   // TMEM score buffers
constexpr int kThreads = 6 * 32;
constexpr int kChunk = RT * 128;         // one 64-column K-chunk of the X tile

template <int DH>
struct BL {
  static_assert(DH == 128, "router_blk: d_h = 128 only (shared-memory budget)");
  static constexpr int KB = DH / 64;
  static constexpr int XT = KB * kChunk;                 // one X tile
  static constexpr int WBLK = 3 * KB * EB * 128;         // one expert block: 3 planes x KB chunks x EB rows
  static constexpr int X = 0, W = 2 * XT;                // X double buffer, W two slots
  static constexpr int BAR = W + 2 * WBLK;               // xfull[2] xempty[2] wfull[2] wempty[2] tfull[NB] tempty[NB]
  static constexpr int NBAR = 8 + 2 * kNB;
  static constexpr int TMEMP = BAR + NBAR * 8;
  static constexpr int DYN = TMEMP + 16;                 // + bias [N_e] f32 + hist [N_e] i32 (runtime)
};

template <int DH, int KMAX>
__global__ void __launch_bounds__(kThreads, 1)
router_blk_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap wmap,
                  const float* __restrict__ bias, int H, int64_t T, int N_e, int k, int32_t* __restrict__ idx,
                  float* __restrict__ gate, int32_t* __restrict__ hist, int32_t* __restrict__ flag) {
  using L = BL<DH>;
  constexpr int KB = L::KB;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0u) __trap();
  const uint32_t sb = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t *xfull = bars, *xempty = bars + 2, *wfull = bars + 4, *wempty = bars + 6;
  uint64_t *tfull = bars + 8, *tempty = tfull + kNB;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::TMEMP);
  float* s_bias = reinterpret_cast<float*>(smem + L::DYN);
  int* s_hist = reinterpret_cast<int*>(s_bias + N_e);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nblk = N_e / EB;

  const int n_rt = (int)((T + RT - 1) / RT);
  const int total = H * n_rt;
  const int per = (total + gridDim.x - 1) / gridDim.x;
  const int tb = min(total, (int)blockIdx.x * per), te = min(total, tb + per);

  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&xfull[i], 1); mbar_init(&xempty[i], 1); mbar_init(&wfull[i], 1); mbar_init(&wempty[i], 1);
    }
    for (int i = 0; i < kNB; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 128); }
    fence_mbar_init();
    tma_prefetch_desc(&xmap); tma_prefetch_desc(&wmap);
  }
  if (warp == 1) tmem_alloc<kNB * EB>(s_tmem);
  for (int i = tid; i < N_e; i += kThreads) s_hist[i] = 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  if (warp == 0) {
    // ============================ TMA producer: X tile n, then its head's W blocks in order
    if (lane == 0) {
      int n = 0, q = 0;                                  // tiles, blocks issued by this CTA
      for (int ti = tb; ti < te; ++ti, ++n) {
        const int h = ti / n_rt, t0 = (ti % n_rt) * RT, xb = n & 1;
        mbar_wait(&xempty[xb], ((n >> 1) & 1) ^ 1);
        mbar_expect_tx(&xfull[xb], L::XT);
        for (int kb = 0; kb < KB; ++kb)
          tma_load_2d(sb + L::X + xb * L::XT + kb * kChunk, &xmap, h * DH + kb * 64, t0, &xfull[xb]);
        for (int b = 0; b < nblk; ++b, ++q) {
          const int ws = q & 1;
          mbar_wait(&wempty[ws], ((q >> 1) & 1) ^ 1);
          mbar_expect_tx(&wfull[ws], L::WBLK);
          for (int p = 0; p < 3; ++p)
            for (int kb = 0; kb < KB; ++kb)
              tma_load_2d(sb + L::W + ws * L::WBLK + (p * KB + kb) * EB * 128, &wmap, kb * 64,
                          (h * 3 + p) * N_e + b * EB, &wfull[ws]);
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer: S_block = X (w1 + w2 + w3)ᵀ per expert block
    if (lane == 0) {
      constexpr uint32_t IDESC = idesc_bf16(RT, EB, 0, 0);
      int n = 0, q = 0;
      for (int ti = tb; ti < te; ++ti, ++n) {
        const int xb = n & 1;
        mbar_wait(&xfull[xb], (n >> 1) & 1);
        for (int b = 0; b < nblk; ++b, ++q) {
          const int ws = q & 1, tbuf = q % kNB;
          mbar_wait(&wfull[ws], (q >> 1) & 1);
          mbar_wait(&tempty[tbuf], ((q / kNB) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + tbuf * EB;
          for (int kb = 0; kb < KB; ++kb)
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
#pragma unroll
              for (int p = 0; p < 3; ++p)
                mma_bf16(d, sdesc_sw128(sb + L::X + xb * L::XT + kb * kChunk + ks * 32, 16, 1024),
                         sdesc_sw128(sb + L::W + ws * L::WBLK + (p * KB + kb) * EB * 128 + ks * 32, 16, 1024), IDESC,
                         (kb | ks | p) ? 1u : 0u);
          mma_commit(&wempty[ws]);
          mma_commit(&tfull[tbuf]);
        }
        mma_commit(&xempty[xb]);
      }
    }
  } else {
    // ============================ epilogue: thread = token row; running top-k over the blocks
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;
    const int et = tid - 64;
    int cur_h = -1, q = 0;
    bool bad = false;
    for (int ti = tb; ti < te; ++ti) {
      const int h = ti / n_rt, rt = ti % n_rt;
      if (h != cur_h) {
        named_bar_sync(1, 128);
        for (int i = et; i < N_e; i += 128) s_bias[i] = bias[(size_t)h * N_e + i];
        named_bar_sync(1, 128);
        cur_h = h;
      }
      // running top-KMAX as packed u64 keys: each KMAX-wide group of a block's scores is
      // bitonic-sorted and merged (branch-free; see router_sm100.cu)
      unsigned long long top[KMAX];
      float chk = 0.f;
      for (int b = 0; b < nblk; ++b, ++q) {              // line 5: expert blocks in index order
        const int tbuf = q % kNB;
        mbar_wait(&tfull[tbuf], (q / kNB) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c0 = 0; c0 < EB; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tmem + tbuf * EB + ((uint32_t)(q4 * 32) << 16) + c0, v);
          tmem_ld_wait();
          if (c0 + 32 >= EB) { tc_fence_before(); mbar_arrive(&tempty[tbuf]); }
#pragma unroll
          for (int g0 = 0; g0 < 32; g0 += KMAX) {
            unsigned long long blk[KMAX];
#pragma unroll
            for (int u = 0; u < KMAX; ++u) {
              const int e = b * EB + c0 + g0 + u;
              const float kf = __uint_as_float(v[g0 + u]) + s_bias[e];   // line 7
              chk = fmaf(kf, 0.f, chk);
              blk[u] = pack_key(kf, e);                                  // line 8
            }
            bitonic_sort_desc<KMAX>(blk);                                // line 9
            if (b == 0 && c0 == 0 && g0 == 0) {
#pragma unroll
              for (int u = 0; u < KMAX; ++u) top[u] = blk[u];
            } else {
              merge_top_desc<KMAX>(top, blk);                            // line 10
            }
          }
        }
      }
      int kid[KMAX];
      float sraw[KMAX];
#pragma unroll
      for (int j = 0; j < KMAX; ++j) {                   // lines 12-13: unpack, remove the bias
        kid[j] = (int)(~(uint32_t)top[j]);
        sraw[j] = unord32((uint32_t)(top[j] >> 32)) - s_bias[kid[j]];
      }
      bad |= (chk != 0.f);
      const int64_t t = (int64_t)rt * RT + row;
      if (t < T) {                                      // lines 11-12: gates from the raw scores
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
            io[j] = kid[j];
            go[j] = ex[j] * inv;
            atomicAdd(&s_hist[kid[j]], 1);
          }
        }
      }
      named_bar_sync(1, 128);
      int32_t* ho = hist + ((size_t)h * n_rt + rt) * N_e;
      for (int i = et; i < N_e; i += 128) { ho[i] = s_hist[i]; s_hist[i] = 0; }
      named_bar_sync(1, 128);
    }
    if (bad) *flag = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<kNB * EB>(tmem);
}

template <int DH, int KMAX>
bool launch_t(const void* Xs, int64_t ldx, const bf16* planes, const float* bias, int H, int64_t T, int N_e, int k,
              int32_t* idx, float* gate, int32_t* hist, int32_t* flag, int num_sms, cudaStream_t s) {
  using L = BL<DH>;
  CUtensorMap xm, wm;
  if (!make_tmap_2d_bf16(&xm, Xs, (uint64_t)T, (uint64_t)H * DH, (uint64_t)ldx * 2, RT, 64)) return false;
  if (!make_tmap_2d_bf16(&wm, planes, (uint64_t)H * 3 * N_e, DH, (uint64_t)DH * 2, EB, 64)) return false;
  const size_t bytes = L::DYN + (size_t)N_e * 8;
  if (bytes > 227 * 1024) return false;
  auto kern = router_blk_kernel<DH, KMAX>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  const int n_rt = (int)((T + RT - 1) / RT);
  const int grid = std::min(num_sms, H * n_rt);
  kern<<<grid, kThreads, bytes, s>>>(xm, wm, bias, H, T, N_e, k, idx, gate, hist, flag);
  return true;
}

template <int DH>
bool launch_k(const void* Xs, int64_t ldx, const bf16* planes, const float* bias, int H, int64_t T, int N_e, int k,
              int32_t* idx, float* gate, int32_t* hist, int32_t* flag, int num_sms, cudaStream_t s) {
  if (k <= 4) return launch_t<DH, 4>(Xs, ldx, planes, bias, H, T, N_e, k, idx, gate, hist, flag, num_sms, s);
  if (k <= 8) return launch_t<DH, 8>(Xs, ldx, planes, bias, H, T, N_e, k, idx, gate, hist, flag, num_sms, s);
  return launch_t<DH, 16>(Xs, ldx, planes, bias, H, T, N_e, k, idx, gate, hist, flag, num_sms, s);
}

}  // namespace

bool router_blk_supported(int d_h, int N_e, int k) {
  // d_h = 128 (the paper's own head width): X double buffer + two W-block slots fit in smem
  return d_h == 128 && N_e > 128 && N_e % EB == 0 && k >= 1 && k <= 16 && k <= N_e &&
         BL<128>::DYN + (size_t)N_e * 8 <= 227 * 1024;
}

bool launch_router_blk_sm100(const void* Xs, int64_t ldx, const void* planes, const float* bias, int H, int64_t T,
                             int d_h, int N_e, int k, int32_t* idx, float* gate, int32_t* hist, int32_t* flag,
                             int num_sms, cudaStream_t s) {
  const bf16* pl = (const bf16*)planes;
  if (d_h == 128) return launch_k<128>(Xs, ldx, pl, bias, H, T, N_e, k, idx, gate, hist, flag, num_sms, s);
  return false;
}

}  // namespace mhl
