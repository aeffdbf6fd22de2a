// expert_sm100.cu — F5: block-sparse expert FFN forward on tcgen05/TMEM (sm_100a).
//
// The paper's IO-aware expert computation (P:916-P:978) treats the replicas clustered by
// expert (Fig. 2) as queries and expert e's W1_e/W2_e rows as keys/values (Eq. 7):
// y = g * gelu(x W1_e^T) W2_e, with the T x k x d_e hidden activation never written to HBM.
// A tile = 128 clustered replicas of one (head, expert):
//   GEMM1  H[128 x d_e] = X[128 x d_h] W1_e^T   A = sub-tokens gathered by TMA gather4 into
//                                                 K-major SW128 smem chunks; B = W1_e (TMA)
//   epi 1  A = bf16(g * gelu(H)), written back INTO TMEM over H (exact-erf GELU, R1)
//   GEMM2  Y[128 x d_h] = A W2_e                 A read from TMEM; B = W2_e read MN-major
//   epi 2  Yrep[row] = bf16(Y)                   TMEM -> registers -> HBM
// Warp roles (320 threads): warp 0 = TMA producer (per-tile token ids / gates, X chunks through an
// smem ring, W1/W2 only when the expert changes, each loaded as soon as the previous expert's
// last GEMM that reads it has completed), warp 1 = MMA issuer (+ TMEM owner), warps 2-9 =
// epilogue.  Two TMEM H/A buffers and the issue order G1(i), G2(i-1), G1(i+1), ... overlap the
// epilogue of one tile with the MMAs of its neighbours.  Persistent CTAs take groups of
// kTileGroup consecutive tiles round-robin (weights reused within a group, the tiles in flight
// stay inside one head so its sub-tokens remain L2-resident for their k gathers).
#include <cuda.h>

#include <cstdlib>

#include "kernels.h"
#include "sm100.cuh"
#include "tma_host.h"

namespace mhl {

namespace {

using namespace sm100;

constexpr int BM = kExpertBM;        // 128 replica rows = MMA M
constexpr int kThreads = 320;
constexpr int kEpiThreads = 256;
constexpr int kXChunk = BM * 128;    // one 64-column K-chunk of the gathered X tile (16 KB)

template <int DH, int DE>
struct FwdL {
  static constexpr int WB = DE * DH * 2;
  static constexpr int W1 = 0, W2 = WB, X = 2 * WB;
  static constexpr int XS_RAW = (224 * 1024 - 2 * WB) / kXChunk;
  static constexpr int XS = XS_RAW > 12 ? 12 : XS_RAW;           // X ring stages
  static constexpr int CTRL = X + XS * kXChunk;
  // barriers
  static constexpr int B_XFULL = CTRL, B_XEMPTY = B_XFULL + 8 * XS;
  static constexpr int B_W1F = B_XEMPTY + 8 * XS, B_W1E = B_W1F + 8, B_W2F = B_W1E + 8, B_W2E = B_W2F + 8;
  static constexpr int B_HFULL = B_W2E + 8, B_AFULL = B_HFULL + 16, B_G2DONE = B_AFULL + 16, B_YEMPTY = B_G2DONE + 16;
  static constexpr int B_TOKF = B_YEMPTY + 8, B_TOKE = B_TOKF + 16;
  static constexpr int TOK = B_TOKE + 16;                         // [2][BM] int
  static constexpr int GATE = TOK + 2 * BM * 4;                   // [2][BM] float
  static constexpr int TMEMP = GATE + 2 * BM * 4;
  static constexpr int BYTES = TMEMP + 16;
};

struct Ph {   // mbarrier phase bit
  uint32_t v = 0;
  __device__ uint32_t flip() { uint32_t o = v; v ^= 1u; return o; }
};

template <int DH, int DE>
__global__ void __launch_bounds__(kThreads, 1)
expert_fwd_sm100_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap w1map,
                        const __grid_constant__ CUtensorMap w2map, const Tile* __restrict__ tiles,
                        const int32_t* __restrict__ ntiles_p, const int32_t* __restrict__ perm,
                        const float* __restrict__ gate, const bf16* __restrict__ Xg, int64_t ldx, int64_t T, int k,
                        int N_e, bf16* __restrict__ Yrep, int dbg) {
  using L = FwdL<DH, DE>;
  constexpr int XS = L::XS, KB1 = DH / 64;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0u) __trap();
  const uint32_t sb = smem_u32(smem);
  auto bar = [&](int off) { return reinterpret_cast<uint64_t*>(smem + off); };
  int* s_tok = reinterpret_cast<int*>(smem + L::TOK);
  float* s_gate = reinterpret_cast<float*>(smem + L::GATE);
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::TMEMP);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t R = T * k;

  if (tid == 0) {
    for (int i = 0; i < XS; ++i) { mbar_init(bar(L::B_XFULL + 8 * i), 32); mbar_init(bar(L::B_XEMPTY + 8 * i), 1); }
    mbar_init(bar(L::B_W1F), 1); mbar_init(bar(L::B_W1E), 1); mbar_init(bar(L::B_W2F), 1); mbar_init(bar(L::B_W2E), 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar(L::B_HFULL + 8 * b), 1);
      mbar_init(bar(L::B_AFULL + 8 * b), kEpiThreads);
      mbar_init(bar(L::B_G2DONE + 8 * b), 1);
      mbar_init(bar(L::B_TOKF + 8 * b), 1);
      mbar_init(bar(L::B_TOKE + 8 * b), kEpiThreads);
    }
    mbar_init(bar(L::B_YEMPTY), kEpiThreads);
    fence_mbar_init();
    tma_prefetch_desc(&xmap); tma_prefetch_desc(&w1map); tma_prefetch_desc(&w2map);
  }
  if (warp == 1) tmem_alloc<512>(s_tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  const int nt = *ntiles_p;
  const int ngroups = (nt + kTileGroup - 1) / kTileGroup;
  const int my_groups = ngroups > (int)blockIdx.x ? (ngroups - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  // the i-th tile of this CTA (or -1)
  auto tile_at = [&](int i) -> int {
    if (i < 0 || i >= my_groups * kTileGroup) return -1;
    const int ti = ((int)blockIdx.x + (i / kTileGroup) * (int)gridDim.x) * kTileGroup + i % kTileGroup;
    return ti < nt ? ti : -1;
  };
  auto same_expert = [&](int ta, int tb2) {
    if (ta < 0 || tb2 < 0) return false;
    const Tile a = tiles[ta], b = tiles[tb2];
    return a.head == b.head && a.expert == b.expert;
  };

  if (warp == 0) {
    // ================================================================ producer
    Ph xe[12], te[2], w1e, w2e;
    int xs = 0;
    for (int i = 0;; ++i) {
      const int ti = tile_at(i);
      if (ti < 0) {
        // W2 of the last tile, if it started a new expert run
        if (i >= 1 && lane == 0 && !same_expert(tile_at(i - 2), tile_at(i - 1))) {
          const Tile pl = tiles[tile_at(i - 1)];
          mbar_wait(bar(L::B_W2E), w2e.flip() ^ 1);
          mbar_expect_tx(bar(L::B_W2F), L::WB);
          for (int kb = 0; kb < KB1; ++kb)
            tma_load_2d(sb + L::W2 + kb * DE * 128, &w2map, kb * 64, (pl.head * N_e + pl.expert) * DE, bar(L::B_W2F));
        }
        break;
      }
      const Tile tl = tiles[ti];
      const int slot = i & 1;
      // token ids and gates of the tile (padding rows -> the zero row T)
      mbar_wait_warp(bar(L::B_TOKE + 8 * slot), te[slot].flip() ^ 1);
      for (int r = lane; r < BM; r += 32) {
        int tok = (int)T; float g = 0.f;
        if (r < tl.rows) {
          const int rep = perm[(size_t)tl.head * R + tl.row0 + r];
          tok = rep / k;
          g = gate[(size_t)tl.head * R + rep];
        }
        s_tok[slot * BM + r] = tok;
        s_gate[slot * BM + r] = g;
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(bar(L::B_TOKF + 8 * slot));
        const bool fresh = !same_expert(tile_at(i - 1), ti);
        if (fresh) {
          mbar_wait(bar(L::B_W1E), w1e.flip() ^ 1);
          mbar_expect_tx(bar(L::B_W1F), L::WB);
          for (int kb = 0; kb < KB1; ++kb)
            tma_load_2d(sb + L::W1 + kb * DE * 128, &w1map, kb * 64, (tl.head * N_e + tl.expert) * DE, bar(L::B_W1F));
        }
      }
      __syncwarp();
      {
        // X chunks: all 32 lanes gather with 16-byte cp.async (lane = 16-byte column chunk x row
        // group); each lane's completion arrives on the stage's full barrier (count 32).
        const int* tk = s_tok + slot * BM;
        for (int kb = 0; kb < KB1; ++kb) {
          mbar_wait_warp(bar(L::B_XEMPTY + 8 * xs), xe[xs].flip() ^ 1);
          const uint32_t dst = sb + L::X + xs * kXChunk;
          const bf16* src = Xg + (size_t)tl.head * DH + kb * 64;
#pragma unroll 8
          for (int j = 0; j < BM * 8 / 32; ++j) {
            const int idx = j * 32 + lane, r = idx >> 3, c = (idx & 7) * 8;
            if (!(dbg & 4)) cp_async_16(dst + kmaj_off(r, c, BM), src + (size_t)tk[r] * ldx + c, 16);
          }
          cp_async_mbar_arrive(bar(L::B_XFULL + 8 * xs));
          if (++xs == XS) xs = 0;
        }
      }
      if (lane == 0) {
        // W2 of the previous tile if that tile started a new expert run (consumed by G2(i-1),
        // which the MMA warp issues after G1(i))
        if (i >= 1 && !same_expert(tile_at(i - 2), tile_at(i - 1))) {
          const Tile pl = tiles[tile_at(i - 1)];
          mbar_wait(bar(L::B_W2E), w2e.flip() ^ 1);
          mbar_expect_tx(bar(L::B_W2F), L::WB);
          for (int kb = 0; kb < KB1; ++kb)
            tma_load_2d(sb + L::W2 + kb * DE * 128, &w2map, kb * 64, (pl.head * N_e + pl.expert) * DE, bar(L::B_W2F));
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ================================================================ MMA issuer
    if (lane == 0) {
      constexpr uint32_t ID1 = idesc_bf16(BM, DE, 0, 0);
      constexpr uint32_t ID2 = idesc_bf16(BM, DH, 0, 1);
      Ph xf[12], w1f, w2f, af[2], gd[2], ye;
      int xs = 0;
      auto gemm2 = [&](int j) {   // G2 of this CTA's j-th tile
        const int b = j & 1;
        const int tj = tile_at(j);
        if (!same_expert(tile_at(j - 1), tj)) mbar_wait(bar(L::B_W2F), w2f.flip());
        mbar_wait(bar(L::B_AFULL + 8 * b), af[b].flip());
        mbar_wait(bar(L::B_YEMPTY), ye.flip() ^ 1);
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < DE / 16; ++ks)
          mma_bf16_ts(tmem + 256, tmem + b * 128 + ks * 8,
                      sdesc_sw128(sb + L::W2 + ks * 2 * 1024, DE * 128, 1024), ID2, ks > 0);
        mma_commit(bar(L::B_G2DONE + 8 * b));
        if (!same_expert(tj, tile_at(j + 1))) mma_commit(bar(L::B_W2E));
      };
      int i = 0;
      for (;; ++i) {
        const int ti = tile_at(i);
        if (ti < 0) break;
        const int b = i & 1;
        if (!same_expert(tile_at(i - 1), ti)) mbar_wait(bar(L::B_W1F), w1f.flip());
        if (i >= 2) mbar_wait(bar(L::B_G2DONE + 8 * b), gd[b].flip());   // H/A buffer b free
        tc_fence_after();
        for (int kb = 0; kb < KB1; ++kb) {
          mbar_wait(bar(L::B_XFULL + 8 * xs), xf[xs].flip());
          fence_proxy_async();   // the chunk was written by cp.async (generic proxy); MMA reads via async proxy
          tc_fence_after();
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            mma_bf16(tmem + b * 128, sdesc_sw128(sb + L::X + xs * kXChunk + ks * 32, 16, 1024),
                     sdesc_sw128(sb + L::W1 + kb * DE * 128 + ks * 32, 16, 1024), ID1, (kb | ks) ? 1u : 0u);
          mma_commit(bar(L::B_XEMPTY + 8 * xs));
          if (++xs == XS) xs = 0;
        }
        mma_commit(bar(L::B_HFULL + 8 * b));
        if (!same_expert(ti, tile_at(i + 1))) mma_commit(bar(L::B_W1E));
        if (i >= 1) gemm2(i - 1);
      }
      if (i >= 1) gemm2(i - 1);
    }
  } else {
    // ================================================================ epilogue (8 warps)
    const int q = warp & 3, half = (warp - 2) >> 2;   // warps 2..5 -> half 0, 6..9 -> half 1
    const int row = q * 32 + lane;
    const int et = tid - 64;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    Ph hf[2], tf[2], gd[2];
    auto epi2 = [&](int j) {
      const int b = j & 1;
      const Tile tl = tiles[tile_at(j)];
      mbar_wait_warp(bar(L::B_G2DONE + 8 * b), gd[b].flip());
      tc_fence_after();
      bf16* dst = Yrep + ((size_t)tl.head * R + tl.row0 + row) * DH;
#pragma unroll 1
      for (int c0 = half * (DH / 2); c0 < (half + 1) * (DH / 2); c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + 256 + lane_off + c0, v);
        tmem_ld_wait();
        if (row < tl.rows) {
#pragma unroll
          for (int u = 0; u < 32; u += 8) {
            uint4 pk;
            pk.x = pack_bf16x2(__uint_as_float(v[u + 0]), __uint_as_float(v[u + 1]));
            pk.y = pack_bf16x2(__uint_as_float(v[u + 2]), __uint_as_float(v[u + 3]));
            pk.z = pack_bf16x2(__uint_as_float(v[u + 4]), __uint_as_float(v[u + 5]));
            pk.w = pack_bf16x2(__uint_as_float(v[u + 6]), __uint_as_float(v[u + 7]));
            if (!(dbg & 2)) *reinterpret_cast<uint4*>(dst + c0 + u) = pk;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(bar(L::B_YEMPTY));
    };
    int i = 0;
    for (;; ++i) {
      const int ti = tile_at(i);
      if (ti < 0) break;
      const int b = i & 1, slot = i & 1;
      mbar_wait_warp(bar(L::B_TOKF + 8 * slot), tf[slot].flip());
      const float g = s_gate[slot * BM + row];
      mbar_wait_warp(bar(L::B_HFULL + 8 * b), hf[b].flip());
      tc_fence_after();
      // epi 1: this warp's DE/2 columns of H -> registers; both halves of the lane quadrant
      // finish reading before either overwrites H with packed A (A col c/2 aliases H col c/2).
      constexpr int NC = DE / 2;
      uint32_t hv[NC];
#pragma unroll
      for (int c = 0; c < NC; c += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + b * 128 + lane_off + half * NC + c, v);
#pragma unroll
        for (int u = 0; u < 32; ++u) hv[c + u] = v[u];
      }
      tmem_ld_wait();
      uint32_t pa[NC / 2];
#pragma unroll
      for (int u = 0; u < NC; u += 2)
        pa[u / 2] = (dbg & 1) ? (hv[u] ^ hv[u + 1])
                              : pack_bf16x2(g * gelu_f(__uint_as_float(hv[u])), g * gelu_f(__uint_as_float(hv[u + 1])));
      named_bar_sync(2 + q, 64);
#pragma unroll
      for (int c = 0; c < NC / 2; c += 16) {
        uint32_t w[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) w[u] = pa[c + u];
        tmem_st16(tmem + b * 128 + lane_off + half * (NC / 2) + c, w);
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(bar(L::B_AFULL + 8 * b));
      mbar_arrive(bar(L::B_TOKE + 8 * slot));
      if (i >= 1) epi2(i - 1);
    }
    if (i >= 1) epi2(i - 1);
    (void)et;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

template <int DH, int DE>
bool launch_t(const Tile* tiles, const int32_t* ntiles, const void* Xs, int64_t ldx, const int32_t* perm,
              const float* gate, const void* W1, const void* W2, int H, int64_t T, int k, int N_e, void* Yrep,
              int num_sms, cudaStream_t s) {
  CUtensorMap xm, w1m, w2m;
  if (!make_tmap_2d_bf16(&xm, Xs, (uint64_t)T + 1, (uint64_t)ldx, (uint64_t)ldx * 2, 1, 64)) return false;
  if (!make_tmap_2d_bf16(&w1m, W1, (uint64_t)H * N_e * DE, DH, (uint64_t)DH * 2, DE, 64)) return false;
  if (!make_tmap_2d_bf16(&w2m, W2, (uint64_t)H * N_e * DE, DH, (uint64_t)DH * 2, DE, 64)) return false;
  auto kern = expert_fwd_sm100_kernel<DH, DE>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdL<DH, DE>::BYTES);
  kern<<<num_sms, kThreads, FwdL<DH, DE>::BYTES, s>>>(xm, w1m, w2m, tiles, ntiles, perm, gate, (const bf16*)Xs,
                                                      ldx, T, k, N_e, (bf16*)Yrep,
                                                      getenv("MHL_DBG") ? atoi(getenv("MHL_DBG")) : 0);
  return true;
}

}  // namespace

bool expert_fwd_sm100_supported(int d_h, int d_e) {
  return (d_h == 256 && d_e == 128) || (d_h == 192 && d_e == 64) || (d_h == 256 && d_e == 64) ||
         (d_h == 128 && d_e == 128) || (d_h == 64 && d_e == 64) || (d_h == 128 && d_e == 64);
}

bool launch_expert_fwd_sm100(const Tile* tiles, const int32_t* ntiles, int max_tiles, const void* Xs, int64_t ldx,
                             const int32_t* perm, const float* gate, const void* W1, const void* W2, int H, int64_t T,
                             int k, int N_e, int d_h, int d_e, void* Yrep, int num_sms, cudaStream_t s) {
  (void)max_tiles;
#define MHL_F(A, B) \
  if (d_h == A && d_e == B) return launch_t<A, B>(tiles, ntiles, Xs, ldx, perm, gate, W1, W2, H, T, k, N_e, Yrep, num_sms, s);
  MHL_F(256, 128) MHL_F(256, 64) MHL_F(192, 64) MHL_F(128, 128) MHL_F(128, 64) MHL_F(64, 64)
#undef MHL_F
  return false;
}

}  // namespace mhl
