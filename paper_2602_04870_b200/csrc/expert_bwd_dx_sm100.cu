// expert_bwd_dx_sm100.cu — B5 (input side): block-sparse expert FFN backward on tcgen05/TMEM.
//
// Chain rule of y_r = g_r * gelu(x W1_e^T) W2_e for the clustered rows of one expert (P:936,
// Eq. 1), H recomputed (the forward never stored it):
//   G_H   H   = X  W1_e^T       A = gathered sub-tokens, B = W1_e (K-major)        TMEM [0,128)
//   G_dA  dA' = dY W2_e^T       A = gathered dcat rows,  B = W2_e (K-major)        TMEM [128,256)
//   epi   dg = <gelu(H), dA'>  (= <dY, E_e(x)>, the gate cotangent)
//         dH = g dA' gelu'(H),  gA = g gelu(H)    (bf16; dH -> smem as the next A operand,
//                                                   dH and gA -> HBM for the weight gradients)
//   G_dX  dXrep = dH W1_e       A = dH (smem), B = W1_e viewed MN-major          TMEM [256,512)
// Warp roles as in the forward kernel: warps 0-3 gather X then dY chunks through an smem ring
// (W1/W2 by TMA when the expert changes), warp 4 issues the MMAs in the order
// G_H(i), G_dA(i), G_dX(i-1) (G_dX(i-1) first when tile i starts a new expert), warps 5-12 run the
// epilogue of tile i while the tensor pipe works on its neighbours.
#include <cuda.h>

#include <cstdlib>

#include "kernels.h"
#include "sm100.cuh"
#include "tma_host.h"

namespace mhl {

namespace {

using namespace sm100;

__device__ TraceBuf g_trace_dx;     // profiling aid (MHL_TRACE_DX=<file>), off by default

constexpr int BM = kExpertBM;
constexpr int kProdWarps = 4, kMmaWarp = 4, kEpiWarp0 = 5;
constexpr int kThreads = 13 * 32;
constexpr int kEpiThreads = 256;
constexpr int kChunk = BM * 128;     // one 64-column K-chunk of a gathered 128-row tile (16 KB)

template <int DH, int DE>
struct DxL {
  static constexpr int WB = DE * DH * 2;
  static constexpr int W1 = 0, W2 = WB, DHS = 2 * WB, RING = DHS + BM * DE * 2;
  static constexpr int S_RAW = (225 * 1024 - RING) / kChunk;
  static constexpr int S = S_RAW > 12 ? 12 : S_RAW;
  static constexpr int CTRL = RING + S * kChunk;
  static constexpr int B_FULL = CTRL, B_EMPTY = B_FULL + 8 * S;
  static constexpr int B_W1F = B_EMPTY + 8 * S, B_W1E = B_W1F + 8, B_W2F = B_W1E + 8, B_W2E = B_W2F + 8;
  static constexpr int B_HDFULL = B_W2E + 8, B_HDFREE = B_HDFULL + 8, B_DHFULL = B_HDFREE + 8;
  static constexpr int B_G3DONE = B_DHFULL + 8, B_DXFREE = B_G3DONE + 8;
  static constexpr int TOK = B_DXFREE + 8;                  // [BM] int (producers)
  static constexpr int DG = TOK + BM * 4;                   // [2][BM] float (epilogue pairs)
  static constexpr int TMEMP = DG + 2 * BM * 4;
  static constexpr int BYTES = TMEMP + 16;
  static constexpr uint32_t T_H = 0, T_DA = 128, T_DX = 256;
};

struct Ph {
  uint32_t v = 0;
  __device__ uint32_t flip() { uint32_t o = v; v ^= 1u; return o; }
};

template <int DH, int DE>
__global__ void __launch_bounds__(kThreads, 1)
expert_bwd_dx_kernel(const __grid_constant__ CUtensorMap w1map, const __grid_constant__ CUtensorMap w2map, Routing rt,
                     const bf16* __restrict__ Xg, int64_t ldx, const bf16* __restrict__ dYg, int64_t ldy,
                     bf16* __restrict__ dXrep, float* __restrict__ dg, bf16* __restrict__ dHg,
                     bf16* __restrict__ gAg) {
  using L = DxL<DH, DE>;
  constexpr int S = L::S, KB = DH / 64;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0u) __trap();
  const uint32_t sb = smem_u32(smem);
  auto bar = [&](int off) { return reinterpret_cast<uint64_t*>(smem + off); };
  int* s_tok = reinterpret_cast<int*>(smem + L::TOK);
  float* s_dg = reinterpret_cast<float*>(smem + L::DG);
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::TMEMP);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const Tile* tiles = rt.tiles;
  const int N_e = rt.N_e;
  const int64_t Rp = rt.Rp, R = rt.T * rt.k;

  if (tid == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(bar(L::B_FULL + 8 * i), 32 * kProdWarps); mbar_init(bar(L::B_EMPTY + 8 * i), 1); }
    mbar_init(bar(L::B_W1F), 1); mbar_init(bar(L::B_W1E), 1); mbar_init(bar(L::B_W2F), 1); mbar_init(bar(L::B_W2E), 1);
    mbar_init(bar(L::B_HDFULL), 1);
    mbar_init(bar(L::B_HDFREE), kEpiThreads);
    mbar_init(bar(L::B_DHFULL), kEpiThreads);
    mbar_init(bar(L::B_G3DONE), 1);
    mbar_init(bar(L::B_DXFREE), kEpiThreads);
    fence_mbar_init();
    tma_prefetch_desc(&w1map); tma_prefetch_desc(&w2map);
  }
  if (warp == kMmaWarp) tmem_alloc<512>(s_tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  const int nt = *rt.ntiles;
  const int ngroups = (nt + kTileGroup - 1) / kTileGroup;
  const int my_groups = ngroups > (int)blockIdx.x ? (ngroups - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
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
  auto load_w = [&](const CUtensorMap* map, int off, uint64_t* full, const Tile& t) {
    mbar_expect_tx(full, L::WB);
    for (int kb = 0; kb < KB; ++kb) tma_load_2d(sb + off + kb * DE * 128, map, kb * 64, (t.head * N_e + t.expert) * DE, full);
  };

  if (warp < kProdWarps) {
    // ================================================================ producers
    const int pw = warp;
    Ph ee[12], w1e, w2e;
    int st = 0;
    auto gather = [&](const bf16* base, int64_t ld, const Tile& tl) {
      for (int kb = 0; kb < KB; ++kb) {
        mbar_wait_warp(bar(L::B_EMPTY + 8 * st), ee[st].flip() ^ 1);
        const uint32_t dst = sb + L::RING + st * kChunk;
        const bf16* src = base + (size_t)tl.head * DH + kb * 64;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int idx = j * 32 + lane, r = pw * 32 + (idx >> 3), c = (idx & 7) * 8;
          cp_async_16(dst + kmaj_off(r, c, BM), src + (size_t)s_tok[r] * ld + c, 16);
        }
        cp_async_mbar_arrive(bar(L::B_FULL + 8 * st));
        if (++st == S) st = 0;
      }
    };
    for (int i = 0;; ++i) {
      const int ti = tile_at(i);
      if (ti < 0) break;
      const Tile tl = tiles[ti];
      const bool fresh = !same_expert(tile_at(i - 1), ti);
      __syncwarp();
      s_tok[pw * 32 + lane] = rt.tok_s[(size_t)tl.head * Rp + tl.row0 + pw * 32 + lane];
      __syncwarp();
      gather(Xg, ldx, tl);
      if (pw == 0 && lane == 0) trace_ev(g_trace_dx, 30, i);
      if (pw == 0 && lane == 0 && fresh) {
        mbar_wait(bar(L::B_W1E), w1e.flip() ^ 1);
        load_w(&w1map, L::W1, bar(L::B_W1F), tl);
        mbar_wait(bar(L::B_W2E), w2e.flip() ^ 1);
        load_w(&w2map, L::W2, bar(L::B_W2F), tl);
      }
      __syncwarp();
      gather(dYg, ldy, tl);
      if (pw == 0 && lane == 0) trace_ev(g_trace_dx, 31, i);
    }
  } else if (warp == kMmaWarp) {
    // ================================================================ MMA issuer
    if (lane == 0) {
      constexpr uint32_t ID_N_DE = idesc_bf16(BM, DE, 0, 0);
      constexpr uint32_t ID_N_DH = idesc_bf16(BM, DH, 0, 1);
      Ph ff[12], w1f, w2f, hdfr, dhf, dxfr, g3;
      int st = 0;
      auto gemm_k = [&](uint32_t d, int woff) {   // d += (ring chunks) . W^T over K = DH
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(bar(L::B_FULL + 8 * st), ff[st].flip());
          fence_proxy_async();
          tc_fence_after();
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            mma_bf16(d, sdesc_sw128(sb + L::RING + st * kChunk + ks * 32, 16, 1024),
                     sdesc_sw128(sb + woff + kb * DE * 128 + ks * 32, 16, 1024), ID_N_DE, (kb | ks) ? 1u : 0u);
          mma_commit(bar(L::B_EMPTY + 8 * st));
          if (++st == S) st = 0;
        }
      };
      int ndx = 0;   // G_dX issued so far
      auto gemm_dx = [&](int j) {
        mbar_wait(bar(L::B_DHFULL), dhf.flip());          // dH(j) in smem
        if (ndx >= 1) mbar_wait(bar(L::B_DXFREE), dxfr.flip());   // dX(j-1) drained
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < DE / 16; ++ks)
          mma_bf16(tmem + L::T_DX, sdesc_sw128(sb + L::DHS + (ks >> 2) * BM * 128 + (ks & 3) * 32, 16, 1024),
                   sdesc_sw128(sb + L::W1 + ks * 2 * 1024, DE * 128, 1024), ID_N_DH, ks > 0);
        mma_commit(bar(L::B_G3DONE));
        trace_ev(g_trace_dx, 43, j);
        if (!same_expert(tile_at(j), tile_at(j + 1))) mma_commit(bar(L::B_W1E));
        ++ndx;
      };
      int pending = -1;
      for (int i = 0;; ++i) {
        const int ti = tile_at(i);
        if (ti < 0) break;
        const bool fresh = !same_expert(tile_at(i - 1), ti);
        if (fresh && pending >= 0) { gemm_dx(pending); pending = -1; }
        if (fresh) mbar_wait(bar(L::B_W1F), w1f.flip());
        if (i >= 1) mbar_wait(bar(L::B_HDFREE), hdfr.flip());   // epilogue has read H, dA' of tile i-1
        tc_fence_after();
        trace_ev(g_trace_dx, 40, i);
        gemm_k(tmem + L::T_H, L::W1);
        if (fresh) mbar_wait(bar(L::B_W2F), w2f.flip());
        gemm_k(tmem + L::T_DA, L::W2);
        mma_commit(bar(L::B_HDFULL));
        trace_ev(g_trace_dx, 41, i);
        if (!same_expert(ti, tile_at(i + 1))) mma_commit(bar(L::B_W2E));
        if (pending >= 0) gemm_dx(pending);
        pending = i;
      }
      if (pending >= 0) gemm_dx(pending);
      (void)g3;
    }
  } else {
    // ================================================================ epilogue (8 warps)
    const int q = warp & 3, half = (warp - kEpiWarp0) >> 2;
    const int row = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    constexpr int NC = DE / 2;         // H / dA' columns per thread
    Ph hd, g3;
    auto drain_dx = [&](int j) {       // dXrep rows of tile j (G_dX(j) complete)
      const Tile tl = tiles[tile_at(j)];
      bf16* dst = dXrep + ((size_t)tl.head * Rp + tl.row0 + row) * DH + half * (DH / 2);
#pragma unroll 1
      for (int c0 = 0; c0 < DH / 2; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + L::T_DX + lane_off + half * (DH / 2) + c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 32; u += 16) {
          uint32_t p[8];
#pragma unroll
          for (int w = 0; w < 8; ++w) p[w] = pack_bf16x2(__uint_as_float(v[u + 2 * w]), __uint_as_float(v[u + 2 * w + 1]));
          st_global_v8(dst + c0 + u, p[0], p[1], p[2], p[3], p[4], p[5], p[6], p[7]);
        }
      }
      tc_fence_before();
      mbar_arrive(bar(L::B_DXFREE));
    };
    int i = 0;
    for (;; ++i) {
      const int ti = tile_at(i);
      if (ti < 0) break;
      const Tile tl = tiles[ti];
      const size_t grow = (size_t)tl.head * Rp + tl.row0 + row;
      const float g = rt.gate_s[grow];
      const int rep = rt.perm[grow];
      mbar_wait_warp(bar(L::B_HDFULL), hd.flip());
      if (tid == kEpiWarp0 * 32) trace_ev(g_trace_dx, 50, i);
      tc_fence_after();
      uint32_t hv[NC], dv[NC];
#pragma unroll
      for (int c = 0; c < NC; c += 32) {
        uint32_t v[32], w[32];
        tmem_ld32(tmem + L::T_H + lane_off + half * NC + c, v);
        tmem_ld32(tmem + L::T_DA + lane_off + half * NC + c, w);
#pragma unroll
        for (int u = 0; u < 32; ++u) { hv[c + u] = v[u]; dv[c + u] = w[u]; }
      }
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(bar(L::B_HDFREE));
      float dgp = 0.f;
      uint32_t dhp[NC / 2], gap[NC / 2];
#pragma unroll
      for (int u = 0; u < NC; u += 2) {
        const float2 h2 = make_float2(__uint_as_float(hv[u]), __uint_as_float(hv[u + 1]));
        const float2 d2 = make_float2(__uint_as_float(dv[u]), __uint_as_float(dv[u + 1]));
        float2 gp;
        const float2 a = gelu2(h2, &gp);
        dgp = fmaf(a.x, d2.x, dgp);
        dgp = fmaf(a.y, d2.y, dgp);
        const float2 dh = __fmul2_rn(__fmul2_rn(d2, gp), make_float2(g, g));
        const float2 ga = __fmul2_rn(a, make_float2(g, g));
        dhp[u / 2] = pack_bf16x2(dh.x, dh.y);
        gap[u / 2] = pack_bf16x2(ga.x, ga.y);
      }
      // dH(i) -> smem once G_dX(i-1) has finished reading the previous dH (it also left dX(i-1))
      if (tid == kEpiWarp0 * 32) trace_ev(g_trace_dx, 52, i);
      if (i >= 1) mbar_wait_warp(bar(L::B_G3DONE), g3.flip());
      if (tid == kEpiWarp0 * 32) trace_ev(g_trace_dx, 53, i);
#pragma unroll
      for (int u = 0; u < NC / 2; u += 4) {
        uint4 pk = make_uint4(dhp[u], dhp[u + 1], dhp[u + 2], dhp[u + 3]);
        *reinterpret_cast<uint4*>(smem + L::DHS + kmaj_off(row, half * NC + 2 * u, BM)) = pk;
      }
      fence_proxy_async();
      mbar_arrive(bar(L::B_DHFULL));
      if (i >= 1) { tc_fence_after(); drain_dx(i - 1); }
      if (tid == kEpiWarp0 * 32) trace_ev(g_trace_dx, 55, i);
      // dH, gA rows to HBM for the weight-gradient kernel; the gate cotangent per replica
#pragma unroll
      for (int u = 0; u < NC / 2; u += 8) {
        st_global_v8(dHg + grow * DE + half * NC + 2 * u, dhp[u], dhp[u + 1], dhp[u + 2], dhp[u + 3], dhp[u + 4],
                     dhp[u + 5], dhp[u + 6], dhp[u + 7]);
        st_global_v8(gAg + grow * DE + half * NC + 2 * u, gap[u], gap[u + 1], gap[u + 2], gap[u + 3], gap[u + 4],
                     gap[u + 5], gap[u + 6], gap[u + 7]);
      }
      s_dg[half * BM + row] = dgp;
      named_bar_sync(2 + q, 64);
      if (half == 0 && rep >= 0) dg[(size_t)tl.head * R + rep] = s_dg[row] + s_dg[BM + row];
      named_bar_sync(2 + q, 64);
    }
    if (i >= 1) { mbar_wait_warp(bar(L::B_G3DONE), g3.flip()); tc_fence_after(); drain_dx(i - 1); }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) tmem_dealloc<512>(tmem);
}

template <int DH, int DE>
bool launch_t(const Routing& rt, const void* Xs, int64_t ldx, const void* dY, int64_t ldy, const void* W1,
              const void* W2, void* dXrep, float* dg, void* dH, void* gA, int num_sms, cudaStream_t s) {
  CUtensorMap w1m, w2m;
  if (!make_tmap_2d_bf16(&w1m, W1, (uint64_t)rt.H * rt.N_e * DE, DH, (uint64_t)DH * 2, DE, 64)) return false;
  if (!make_tmap_2d_bf16(&w2m, W2, (uint64_t)rt.H * rt.N_e * DE, DH, (uint64_t)DH * 2, DE, 64)) return false;
  auto kern = expert_bwd_dx_kernel<DH, DE>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, DxL<DH, DE>::BYTES);
  static const char* trace_path = getenv("MHL_TRACE_DX");
  if (trace_path) {
    TraceBuf tb{trace_buffer(s), 0};
    cudaMemcpyToSymbolAsync(g_trace_dx, &tb, sizeof(tb), 0, cudaMemcpyHostToDevice, s);
  }
  kern<<<num_sms, kThreads, DxL<DH, DE>::BYTES, s>>>(w1m, w2m, rt, (const bf16*)Xs, ldx, (const bf16*)dY, ldy,
                                                     (bf16*)dXrep, dg, (bf16*)dH, (bf16*)gA);
  if (trace_path) {
    TraceBuf tb{nullptr, 0};
    cudaMemcpyToSymbolAsync(g_trace_dx, &tb, sizeof(tb), 0, cudaMemcpyHostToDevice, s);
    trace_dump(trace_path, s);
  }
  return true;
}

}  // namespace

bool launch_expert_bwd_dx_sm100(const Routing& rt, const void* Xs, int64_t ldx, const void* dY, int64_t ldy,
                                const void* W1, const void* W2, int d_h, int d_e, void* dXrep, float* dg, void* dH,
                                void* gA, int num_sms, cudaStream_t s) {
#define MHL_DX(A, B) \
  if (d_h == A && d_e == B) return launch_t<A, B>(rt, Xs, ldx, dY, ldy, W1, W2, dXrep, dg, dH, gA, num_sms, s);
  MHL_DX(256, 128) MHL_DX(256, 64) MHL_DX(128, 128) MHL_DX(128, 64)
#undef MHL_DX
  return false;
}

}  // namespace mhl
