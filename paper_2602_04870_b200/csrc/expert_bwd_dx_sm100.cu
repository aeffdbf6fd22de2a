// expert_bwd_dx_sm100.cu — B5 (input side): block-sparse expert FFN backward on tcgen05/TMEM.
//
// Chain rule of y_r = g_r * gelu(x W1_e^T) W2_e for the clustered rows of one expert (P:936,
// Eq. 1), H recomputed (the forward never stored it).  Two persistent kernels over the 128-row
// expert tiles of F4:
//
// kernel 1 (expert_bwd_h):
//   G_H   H   = X  W1_e^T       A = gathered sub-tokens, B = W1_e (K-major)     TMEM [256b, 256b+128)
//   G_dA  dA' = dY W2_e^T       A = gathered dcat rows,  B = W2_e (K-major)     TMEM [256b+128, 256b+256)
//   epi   dg = <gelu(H), dA'>  (= <dY, E_e(x)>, the gate cotangent, per replica)
//         dH = g dA' gelu'(H),  gA = g gelu(H)   (bf16 rows -> HBM, consumed by kernel 2 and the
//                                                 weight-gradient kernel)
//   The H/dA' accumulators are double-buffered (b = tile parity), so the MMAs and sub-token
//   gathers of tile i+1 run while the epilogue of tile i computes: the kernel streams.
//   Warps 0-3 gather X then dY chunks through an smem ring (W1/W2 by TMA on expert change),
//   warp 4 issues the MMAs, warps 5-12 run the epilogue.
//
// kernel 2 (expert_dx_gemm):
//   G_dX  dXrep = dH W1_e       A = dH tile (TMA, contiguous sorted rows), B = W1_e read MN-major
//   TMEM double buffer [0,DH) / [DH,2DH); epilogue TMEM -> bf16 -> smem -> TMA bulk store.
//   Warp 0 = TMA producer, warp 1 = MMA issuer, warps 2-9 = epilogue.
//
// Splitting G_dX off costs one extra read of dH (R*d_e*2 bytes) but lets both kernels keep every
// accumulator double-buffered in the 512 TMEM columns (the fused form needed H, dA' and dX
// resident at once: 128+128+256 columns, which serialised the gathers behind the epilogue).
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
constexpr int kChunk = BM * 128;     // one 64-column K-chunk of a 128-row tile (16 KB)
constexpr int kMaxSmem = 227 * 1024;

struct Ph {
  uint32_t v = 0;
  __device__ uint32_t flip() { uint32_t o = v; v ^= 1u; return o; }
};

__device__ __forceinline__ void tma_store_2d(const void* tmap, uint32_t src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tmap), "r"(src),
               "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Persistent schedule shared by both kernels: CTA b takes groups of kTileGroup consecutive tiles
// round-robin (weights reused within a group, the tiles in flight stay inside one head).
struct Sched {
  const Tile* tiles; int nt, my_groups;
  __device__ Sched(const Tile* t, int n) : tiles(t), nt(n) {
    const int ngroups = (nt + kTileGroup - 1) / kTileGroup;
    my_groups = ngroups > (int)blockIdx.x ? (ngroups - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  }
  __device__ int at(int i) const {
    if (i < 0 || i >= my_groups * kTileGroup) return -1;
    const int ti = ((int)blockIdx.x + (i / kTileGroup) * (int)gridDim.x) * kTileGroup + i % kTileGroup;
    return ti < nt ? ti : -1;
  }
  __device__ bool same_expert(int ta, int tb) const {
    if (ta < 0 || tb < 0) return false;
    const Tile a = tiles[ta], b = tiles[tb];
    return a.head == b.head && a.expert == b.expert;
  }
};

// =============================================================================================
// kernel 1: H, dA' -> dH, gA, dg
// =============================================================================================
constexpr int kEpiWarps = 16;
constexpr int kEpiThreads = kEpiWarps * 32;

#ifndef MHL_K1_STOREHINT
#define MHL_K1_STOREHINT 1   // dH / gA stores evict_first (1) or normal (0)
#endif
#ifndef MHL_K1_PW
#define MHL_K1_PW 8   // producer warps of the backward H kernel (8: pairs, 12: triples per chunk; 4: whole chunks)
#endif

template <int DH, int DE>
struct HL {
  static constexpr int WB = DE * DH * 2;
  static constexpr int BOXES = DE / 64;                    // 64-column output boxes per row
  // H and dA' accumulators (DE columns each) double-buffered when they fit twice in TMEM
  static constexpr int NBUF = 4 * DE <= 512 ? 2 : 1;
  // With double-buffered accumulators the 16 epilogue warps form two groups of 8 that take
  // alternate tiles (group g = buffer g): one group's MUFU-bound GELU math overlaps the other's
  // stores instead of every warp doing math, then stores, in lock step.  That epilogue stores
  // dH/gA straight from registers; giving its smem staging to the gather ring (6 stages instead
  // of 4) measured SLOWER (K1 1.10 -> 1.50 ms, r1e), so the layout keeps the 4-stage ring.
  static constexpr bool GROUPED = NBUF == 2 && kEpiWarps == 16;
#ifdef MHL_K1_RING6
  static constexpr int STGB = GROUPED ? 0 : 4 * BOXES * 4096;   // experiment: staging smem -> ring
#else
  static constexpr int STGB = 4 * BOXES * 4096;             // dH/gA staging: [quadrant][box] 32 x 64 bf16
#endif
  static constexpr int W1 = 0, W2 = WB, STG = 2 * WB, RING = STG + STGB;
  static constexpr int CTRL_MAX = 3 * 1024;
  static constexpr int S_RAW = (kMaxSmem - RING - CTRL_MAX) / kChunk;
  // producer warps and warp roles.  With a >= 4-stage ring: 8 warps, WPC of them filling each
  // chunk (128/WPC rows each): more warps issuing gathers raise the SM's gather rate
  // (tools/ring_probe.cu mech 6: 5.8 -> 8.9 TB/s for L2-resident rows).  Otherwise (d_e = 256:
  // 2-3 stages) 2 warps, each filling whole chunks.
  static constexpr bool SPLIT = S_RAW >= 4 && (MHL_K1_PW == 8 || MHL_K1_PW == 12);
  static constexpr int PW = S_RAW >= 4 ? MHL_K1_PW : 2;
  static constexpr int WPC = SPLIT ? PW / 4 : 1;            // warps per chunk (lanes split as evenly as possible)
  static constexpr int OWNERS = PW / WPC;                   // chunk owners (warp pairs or warps)
  // warps [0, PW) producers, [PW, PW + 16) epilogue, PW + 16 the MMA issuer.  With 8 producers
  // the roles are warpgroup-aligned, so producers hand registers to the epilogue (setmaxnreg).
  static constexpr int EPI_WARP0 = PW, MMA_WARP = PW + kEpiWarps, THREADS = (PW + 1 + kEpiWarps) * 32;
  static constexpr bool REGS = PW == 8 || PW == 12;
  // launch cap 72 with 25 warps (8 producers): 8*32*(72-40) >= 16*32*(88-72); 64 with 29 warps
  // (12 producers): 12*32*(64-40) >= 16*32*(80-64), and sub-partition 0 (3 producers, 4 epilogue
  // warps, the MMA warp) holds 3*40 + 4*80 + 64 <= 512
  static constexpr int PROD_REGS = 40, EPI_REGS = PW == 12 ? 80 : 88;
  // a multiple of OWNERS: chunk c -> stage c % S, owner c % OWNERS, so every stage is only ever
  // refilled by the owner that filled it before.  (S >= OWNERS alone would keep the EMPTY parity
  // exact too — the owner's previous chunk waited for the in-order consumption of chunk
  // c - OWNERS - S >= c - 2S — but the 6-stage ring it allows measured slower, see above.)
#ifdef MHL_K1_RING6
  static constexpr int S = S_RAW > 12 ? 12 : S_RAW;
#else
  static constexpr int S = (S_RAW > 12 ? 12 : S_RAW) / OWNERS * OWNERS;
#endif
  static constexpr int CTRL = RING + S * kChunk;
  static constexpr int B_FULL = CTRL, B_EMPTY = B_FULL + 8 * S;
  static constexpr int B_W1F = B_EMPTY + 8 * S, B_W1E = B_W1F + 8, B_W2F = B_W1E + 8, B_W2E = B_W2F + 8;
  static constexpr int B_HDFULL = B_W2E + 8, B_HDFREE = B_HDFULL + 16;
  static constexpr int DG = B_HDFREE + 16;                  // [kEpiWarps/4][BM] float (dg partials)
  static constexpr int TMEMP = DG + (kEpiWarps / 4) * BM * 4;
  static constexpr int BYTES = TMEMP + 16;
  static_assert(BYTES - CTRL <= CTRL_MAX, "control block overflow");
  static_assert(BYTES <= kMaxSmem, "K1: shared memory over the per-CTA limit");
  static_assert(S >= OWNERS, "ring too small");
};

template <int DH, int DE>
__global__ void __launch_bounds__(HL<DH, DE>::THREADS, 1)
expert_bwd_h_kernel(const __grid_constant__ CUtensorMap w1map, const __grid_constant__ CUtensorMap w2map,
                    const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap ymap,
                    const __grid_constant__ CUtensorMap hsmap, const __grid_constant__ CUtensorMap asmap, Routing rt,
                    float* __restrict__ dg, int dbg, uint8_t* __restrict__ dH_out, uint8_t* __restrict__ gA_out,
                    int lsu) {
  using L = HL<DH, DE>;
  constexpr int kProdWarps = L::PW, kMmaWarp = L::MMA_WARP, kEpiWarp0 = L::EPI_WARP0, NBUF = L::NBUF;
  TraceBuf trc = g_trace_dx;   // one load; trace_ev then costs a register test
  if (threadIdx.x == 0) trace_cta(trc, 60);
  constexpr int S = L::S, KB = DH / 64;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0u) __trap();
  const uint32_t sb = smem_u32(smem);
  auto bar = [&](int off) { return reinterpret_cast<uint64_t*>(smem + off); };
  float* s_dg = reinterpret_cast<float*>(smem + L::DG);
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::TMEMP);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t_lo = rt.trange ? rt.trange[0] : 0;   // tile window (NEXT-1) or every tile
  const Tile* tiles = rt.tiles + t_lo;
  const int N_e = rt.N_e;
  const int64_t Rp = rt.Rp, R = rt.T * rt.k;

  if (tid == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(bar(L::B_FULL + 8 * i), 1); mbar_init(bar(L::B_EMPTY + 8 * i), 1); }
    mbar_init(bar(L::B_W1F), 1); mbar_init(bar(L::B_W1E), 1); mbar_init(bar(L::B_W2F), 1); mbar_init(bar(L::B_W2E), 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar(L::B_HDFULL + 8 * b), 1);
      mbar_init(bar(L::B_HDFREE + 8 * b), L::GROUPED ? kEpiThreads / 2 : kEpiThreads);
    }
    fence_mbar_init();
    tma_prefetch_desc(&w1map); tma_prefetch_desc(&w2map); tma_prefetch_desc(&xmap); tma_prefetch_desc(&ymap);
    tma_prefetch_desc(&hsmap); tma_prefetch_desc(&asmap);
  }
  if (warp == kMmaWarp) tmem_alloc<512>(s_tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  const Sched sc(tiles, (rt.trange ? rt.trange[1] : *rt.ntiles) - t_lo);

  auto load_w = [&](const CUtensorMap* map, int off, uint64_t* full, const Tile& t) {
    mbar_expect_tx(full, L::WB);
    for (int kb = 0; kb < KB; ++kb) tma_load_2d(sb + off + kb * DE * 128, map, kb * 64, (t.head * N_e + t.expert) * DE, full);
  };

  if (warp < kProdWarps) {
    if constexpr (L::REGS) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(L::PROD_REGS));
    // ================================================================ producers
    // A tile is 2*KB chunks (X k-chunks, then dY k-chunks); chunk c of the CTA's stream goes to
    // ring stage c % S and is brought by warp c % kProdWarps, each of its 32 lanes issuing one TMA
    // gather4 (4 rows x 64 columns; lane l owns tile rows 4l..4l+3).  The SW128 swizzle is applied
    // by smem address, so row r lands where the K-major MMA descriptor expects it (kmaj_off).
    // Several warps with whole-chunk gathers in flight keep the TMA unit busy (tools/ring_probe.cu).
    const int pw = warp;
    Ph w1e, w2e;
    int cnt = 0;                       // chunks of this CTA's stream so far
    const uint64_t pol_keep = (dbg & 16) ? l2_evict_normal() : l2_evict_last();   // rows reused k times per head
    // owner pw/WPC fills the chunk, this warp its rows lrow.. (lanes 0..LPW-1, 4 rows each)
    // the 32 gather4 lanes of a chunk split over its WPC warps (11/11/10 with three)
    constexpr int OWN = L::OWNERS, WPC = L::WPC, LB = 32 / WPC, LX = 32 % WPC;
    const int owner = pw / WPC, wi = pw % WPC;
    const int lpw = LB + (wi < LX ? 1 : 0), lane0 = wi * LB + (wi < LX ? wi : LX);   // this warp's lanes of the chunk
    const bool issues = lane < lpw;
    const int lrow = 4 * (lane0 + (issues ? lane : 0));
    const bool tx_lead = lane == 0 && wi == 0;
    int nx[4] = {0, 0, 0, 0};          // token ids of the next tile's rows lrow..lrow+3
    auto load_tok = [&](int ti) {
      if (ti < 0) return;
      const Tile t = tiles[ti];
      const int32_t* tk = rt.tok_s + (size_t)t.head * Rp + t.row0 + lrow;
      nx[0] = tk[0]; nx[1] = tk[1]; nx[2] = tk[2]; nx[3] = tk[3];
    };
    load_tok(sc.at(0));
    for (int i = 0;; ++i) {
      const int ti = sc.at(i);
      if (ti < 0) break;
      const Tile tl = tiles[ti];
      const bool fresh = !sc.same_expert(sc.at(i - 1), ti);
      if (pw == 0 && lane == 0) trace_ev(trc, 34, i);
      const int r0 = nx[0], r1 = nx[1], r2 = nx[2], r3 = nx[3];
      load_tok(sc.at(i + 1));          // in flight while this tile's chunks are issued
      if (pw == 0 && lane == 0 && fresh) {
        mbar_wait(bar(L::B_W1E), w1e.flip() ^ 1);
        load_w(&w1map, L::W1, bar(L::B_W1F), tl);
        mbar_wait(bar(L::B_W2E), w2e.flip() ^ 1);
        load_w(&w2map, L::W2, bar(L::B_W2F), tl);
      }
      __syncwarp();
      for (int j = 0; j < 2 * KB; ++j, ++cnt) {
        if (cnt % OWN != owner) continue;
        const int st = cnt % S;
        uint64_t* full = bar(L::B_FULL + 8 * st);
        if (lane == 0) mbar_wait(bar(L::B_EMPTY + 8 * st), ((cnt / S) & 1) ^ 1);
        if (tx_lead) mbar_expect_tx(full, kChunk);
        __syncwarp();
        const int kb = j % KB;
        if (issues)
          tma_gather4_hint(sb + L::RING + st * kChunk + lrow * 128, j < KB ? &xmap : &ymap, tl.head * DH + kb * 64,
                           r0, r1, r2, r3, full, pol_keep);
      }
    }
  } else if (warp == kMmaWarp) {
    // ================================================================ MMA issuer
    if (lane == 0) {
      constexpr uint32_t ID_N_DE = idesc_bf16(BM, DE, 0, 0);
      Ph ff[12], w1f, w2f, hdfr[2];
      int st = 0, nch = 0;
      auto gemm_k = [&](uint32_t d, int woff) {   // d = (ring chunks) . W^T over K = DH
        for (int kb = 0; kb < KB; ++kb, ++nch) {
          mbar_wait(bar(L::B_FULL + 8 * st), ff[st].flip());
          if (dbg & 1) { mbar_arrive(bar(L::B_EMPTY + 8 * st)); if (++st == S) st = 0; continue; }
          tc_fence_after();
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            mma_bf16(d, sdesc_sw128(sb + L::RING + st * kChunk + ks * 32, 16, 1024),
                     sdesc_sw128(sb + woff + kb * DE * 128 + ks * 32, 16, 1024), ID_N_DE, (kb | ks) ? 1u : 0u);
          mma_commit(bar(L::B_EMPTY + 8 * st));
          if (++st == S) st = 0;
        }
      };
      for (int i = 0;; ++i) {
        const int ti = sc.at(i);
        if (ti < 0) break;
        const int b = i % NBUF;
        const bool fresh = !sc.same_expert(sc.at(i - 1), ti);
        const bool last = !sc.same_expert(ti, sc.at(i + 1));
        if (fresh) mbar_wait(bar(L::B_W1F), w1f.flip());
        if (i >= NBUF) mbar_wait(bar(L::B_HDFREE + 8 * b), hdfr[b].flip());   // epilogue read tile i-NBUF
        tc_fence_after();
        trace_ev(trc, 40, i);
        gemm_k(tmem + 2 * DE * b, L::W1);
        if (last && !(dbg & 1)) mma_commit(bar(L::B_W1E));
        if (fresh) mbar_wait(bar(L::B_W2F), w2f.flip());
        gemm_k(tmem + 2 * DE * b + DE, L::W2);
        if (dbg & 1) {
          mbar_arrive(bar(L::B_HDFULL + 8 * b));
          if (last) { mbar_arrive(bar(L::B_W1E)); mbar_arrive(bar(L::B_W2E)); }
        } else {
          mma_commit(bar(L::B_HDFULL + 8 * b));
          if (last) mma_commit(bar(L::B_W2E));
        }
        trace_ev(trc, 41, i);
      }
    }
  } else {
    if constexpr (L::REGS) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(L::EPI_REGS));
    if constexpr (L::GROUPED) {
      // ============================================================ epilogue: two groups of 8 warps
      // group grp takes tiles i = grp, grp + 2, ... (TMEM buffer grp); in a group, warp -> (lane
      // quadrant q, column half hc): one row and DE/2 columns per thread, 16 at a time: TMEM ->
      // gelu/gelu' -> bf16 -> dH, gA straight to global (32-byte st.global.v8 per lane, L2
      // evict-first; every 128-byte row segment is written whole by one thread).  dg keeps the
      // summation order of the single-group epilogue (32-column partials, added in column order).
      constexpr int NC = DE / 2;
      static_assert(NC % 32 == 0, "grouped K1 epilogue: d_e = 64 or 128");
      const int ew = warp - kEpiWarp0, grp = ew >> 3, q = warp & 3, hc = (ew >> 2) & 1;
      const int row = q * 32 + lane;
      const uint32_t lane_off = (uint32_t)(q * 32) << 16;
      const int bar_dg = 2 + grp * 4 + q;                   // the two warps of (group, quadrant)
      const uint64_t pol_out = MHL_K1_STOREHINT ? l2_evict_first() : l2_evict_normal();
      float* s_x = s_dg + grp * 2 * BM;                     // [parity][BM]: s0 + s1 of each row
      Ph hd;
      float g_n = 0.f;
      int rep_n = -1;
      Tile tl_n{};
      auto fetch = [&](int t) {
        if (t < 0) return;
        tl_n = tiles[t];
        const size_t gr = (size_t)tl_n.head * Rp + tl_n.row0 + row;
        g_n = __ldg(rt.gate_s + gr);
        rep_n = __ldg(rt.perm + gr);
      };
      fetch(sc.at(grp));
      for (int i = grp;; i += 2) {
        const int ti = sc.at(i);
        if (ti < 0) break;
        const int b = grp;
        const Tile tl = tl_n;
        const float g = g_n;
        const int rep = rep_n;
        fetch(sc.at(i + 2));
        const size_t grow = (size_t)tl.head * Rp + tl.row0 + row;
        uint8_t* dh_row = dH_out + grow * (DE * 2) + hc * NC * 2;
        uint8_t* ga_row = gA_out + grow * (DE * 2) + hc * NC * 2;
        mbar_wait_warp(bar(L::B_HDFULL + 8 * b), hd.flip());
        if (tid == kEpiWarp0 * 32) trace_ev(trc, 50, i);
        tc_fence_after();
        float sp[2] = {0.f, 0.f};                           // this thread's two DE/4-column dg partials
#pragma unroll
        for (int c = 0; c < NC; c += 16) {
          uint32_t hv[16], dv[16], wh[8], wa[8];
          const uint32_t col = lane_off + hc * NC + c;
          tmem_ld16(tmem + 2 * DE * b + col, hv);
          tmem_ld16(tmem + 2 * DE * b + DE + col, dv);
          tmem_ld_wait();
          if (c + 16 >= NC) {
            tc_fence_before();
            mbar_arrive(bar(L::B_HDFREE + 8 * b));
          }
          float dgp = sp[c / (NC / 2)];
#pragma unroll
          for (int u = 0; u < 16; u += 2) {
            const float2 h2 = make_float2(__uint_as_float(hv[u]), __uint_as_float(hv[u + 1]));
            const float2 d2 = make_float2(__uint_as_float(dv[u]), __uint_as_float(dv[u + 1]));
            float2 gp;
            const float2 a = gelu2(h2, &gp);
            dgp = fmaf(a.x, d2.x, dgp);
            dgp = fmaf(a.y, d2.y, dgp);
            const float2 dh = __fmul2_rn(__fmul2_rn(d2, gp), make_float2(g, g));
            const float2 ga = __fmul2_rn(a, make_float2(g, g));
            wh[u / 2] = pack_bf16x2(dh.x, dh.y);
            wa[u / 2] = pack_bf16x2(ga.x, ga.y);
          }
          sp[c / (NC / 2)] = dgp;
          st_global_v8_hint(dh_row + c * 2, wh[0], wh[1], wh[2], wh[3], wh[4], wh[5], wh[6], wh[7], pol_out);
          st_global_v8_hint(ga_row + c * 2, wa[0], wa[1], wa[2], wa[3], wa[4], wa[5], wa[6], wa[7], pol_out);
        }
        if (tid == kEpiWarp0 * 32) trace_ev(trc, 52, i);
        // dg = ((s0 + s1) + s2) + s3 over the four DE/4-column partials, as the single-group epilogue
        float* sx = s_x + ((i >> 1) & 1) * BM;              // parity slot: no second barrier needed
        if (hc == 0) sx[row] = sp[0] + sp[1];
        named_bar_sync(bar_dg, 64);
        if (hc == 1 && rep >= 0) dg[(size_t)tl.head * R + rep] = (sx[row] + sp[0]) + sp[1];
        if (tid == kEpiWarp0 * 32) trace_ev(trc, 55, i);
      }
    } else {
    // ================================================================ epilogue (kEpiWarps warps)
    // warp -> (lane quadrant q, column group cg); each thread owns one row and NC columns of H/dA'
    // (TMEM -> gelu/gelu' -> bf16).  dH and gA leave through smem and TMA bulk stores: the warps of
    // one 64-column box (64/NC of them) write their 32 x NC slices into the box's SW128 staging slot
    // and the box leader issues the store (dH, then gA through the same slot), so the rows reach
    // HBM as whole 128-byte lines without occupying the LSU path the gathers share.
    constexpr int NG = kEpiWarps / 4, NC = DE / NG, WPB = 64 / NC;   // warps per output box
    const int q = warp & 3, cg = (warp - kEpiWarp0) >> 2;
    const int box = cg * NC / 64, bcol = cg * NC % 64;
    const bool leader = (bcol == 0 && lane == 0);
    // named barrier ids (< 16): per (quadrant, box) only when several warps share a box
    const int bar_box = 2 + q * L::BOXES + box, bar_dg = (WPB > 1 ? 2 + 4 * L::BOXES : 2) + q;
    static_assert(WPB == 1 || 2 + 4 * L::BOXES + 4 <= 16, "K1: named barrier ids exhausted");
    auto box_sync = [&]() { if constexpr (WPB > 1) named_bar_sync(bar_box, 32 * WPB); else __syncwarp(); };
    uint8_t* slot = smem + L::STG + (q * L::BOXES + box) * 4096;
    const uint32_t slot_s = sb + L::STG + (q * L::BOXES + box) * 4096;
    const int row = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    Ph hd[2];
    auto stage = [&](const uint32_t* w) {     // this thread's NC bf16 of its row -> the box slot
#pragma unroll
      for (int u = 0; u < NC; u += 8)
        *reinterpret_cast<uint4*>(slot + kmaj_off(lane, bcol + u, 32)) =
            make_uint4(w[u / 2], w[u / 2 + 1], w[u / 2 + 2], w[u / 2 + 3]);
      fence_proxy_async();
    };
    // this row's gate and replica id, fetched one tile ahead (their L2 latency was exposed at the
    // top of every tile, ~15% of the epilogue's period)
    float g_n = 0.f;
    int rep_n = -1;
    Tile tl_n{};
    auto fetch = [&](int t) {
      if (t < 0) return;
      tl_n = tiles[t];
      const size_t gr = (size_t)tl_n.head * Rp + tl_n.row0 + row;
      g_n = __ldg(rt.gate_s + gr);
      rep_n = __ldg(rt.perm + gr);
    };
    fetch(sc.at(0));
    for (int i = 0;; ++i) {
      const int ti = sc.at(i);
      if (ti < 0) break;
      const int b = i % NBUF;
      const Tile tl = tl_n;
      const int orow = (int)((size_t)tl.head * Rp + tl.row0 + q * 32);
      const float g = g_n;
      const int rep = rep_n;
      fetch(sc.at(i + 1));
      mbar_wait_warp(bar(L::B_HDFULL + 8 * b), hd[b].flip());
      if (tid == kEpiWarp0 * 32) trace_ev(trc, 50, i);
      tc_fence_after();
      float dgp = 0.f;
      uint32_t dhp[NC / 2], gap[NC / 2];
#pragma unroll
      for (int c = 0; c < NC; c += 16) {
        uint32_t hv[16], dv[16];
        const uint32_t col = lane_off + cg * NC + c;
        tmem_ld16(tmem + 2 * DE * b + col, hv);
        tmem_ld16(tmem + 2 * DE * b + DE + col, dv);
        tmem_ld_wait();
        if (c + 16 >= NC) {                       // all of this thread's TMEM reads are done
          tc_fence_before();
          mbar_arrive(bar(L::B_HDFREE + 8 * b));
        }
#pragma unroll
        for (int u = 0; u < 16; u += 2) {
          const float2 h2 = make_float2(__uint_as_float(hv[u]), __uint_as_float(hv[u + 1]));
          const float2 d2 = make_float2(__uint_as_float(dv[u]), __uint_as_float(dv[u + 1]));
          float2 gp;
          const float2 a = gelu2(h2, &gp);
          dgp = fmaf(a.x, d2.x, dgp);
          dgp = fmaf(a.y, d2.y, dgp);
          const float2 dh = __fmul2_rn(__fmul2_rn(d2, gp), make_float2(g, g));
          const float2 ga = __fmul2_rn(a, make_float2(g, g));
          dhp[(c + u) / 2] = pack_bf16x2(dh.x, dh.y);
          gap[(c + u) / 2] = pack_bf16x2(ga.x, ga.y);
        }
      }
      if (tid == kEpiWarp0 * 32) trace_ev(trc, 52, i);
      if (!(dbg & 4) && lsu) {
        // LSU variant: the box warps copy the staged slot to global with coalesced 16-byte stores
        // (8 lanes per 128-byte row segment), leaving the TMA unit to the gathers
        const int bt = (cg % WPB) * 32 + lane;
        const uint64_t pol_out = l2_evict_first();   // streamed out once; keep L2 for the gathered rows
        auto copy_out = [&](uint8_t* dst) {
#pragma unroll
          for (int c = bt; c < 256; c += 32 * WPB) {
            const int r = c >> 3, c16 = c & 7;
            const uint4 v = *reinterpret_cast<const uint4*>(slot + r * 128 + (((c16 ^ (r & 7)) & 7) << 4));
            st_global_v4_hint(dst + ((size_t)orow + r) * (DE * 2) + box * 128 + c16 * 16, v, pol_out);
          }
        };
        box_sync();
        stage(dhp);
        box_sync();
        copy_out(dH_out);
        box_sync();
        stage(gap);
        box_sync();
        copy_out(gA_out);
      } else if (!(dbg & 4)) {
        if (leader) bulk_wait_read<0>();          // the previous tile's gA store has read the slot
        box_sync();
        stage(dhp);
        box_sync();
        if (leader) { tma_store_2d(&hsmap, slot_s, box * 64, orow); bulk_commit(); bulk_wait_read<0>(); }
        box_sync();
        stage(gap);
        box_sync();
        if (leader) { tma_store_2d(&asmap, slot_s, box * 64, orow); bulk_commit(); }
      }
      // gate cotangent: the NG column-group partial sums of this row, added in group order
      s_dg[cg * BM + row] = dgp;
      named_bar_sync(bar_dg, 32 * NG);
      if (cg == 0 && rep >= 0) {
        float acc = s_dg[row];
#pragma unroll
        for (int u = 1; u < NG; ++u) acc += s_dg[u * BM + row];
        dg[(size_t)tl.head * R + rep] = acc;
      }
      named_bar_sync(bar_dg, 32 * NG);
      if (tid == kEpiWarp0 * 32) trace_ev(trc, 55, i);
    }
    if (leader) bulk_wait_all();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) trace_cta(trc, 61);
  if (warp == kMmaWarp) tmem_dealloc<512>(tmem);
}

// =============================================================================================
// kernel 1 on CTA pairs (tcgen05 cta_group::2): two CTAs of a cluster take tiles 2u and 2u+1 of the
// same expert (segments padded to tile pairs, MHL_FLAG_PAIR) and the leader issues M = 256 MMAs;
// cta_group::2 splits each weight matrix along N (d_e), so each CTA keeps HALF of W1_e and W2_e
// and its gather ring grows from 4 to 8 chunks.  Same epilogue as kernel 1 on each CTA's rows.
// =============================================================================================
template <int DH, int DE>
struct HLP {
  static constexpr int WH = DE * DH;                        // half of one expert matrix (bytes)
  static constexpr int BOXES = DE / 64;
  static constexpr int STGB = 4 * BOXES * 4096;
  static constexpr int W1 = 0, W2 = WH, STG = 2 * WH, RING = STG + STGB;
  static constexpr int CTRL_MAX = 3 * 1024;
  static constexpr int S_RAW = (kMaxSmem - RING - CTRL_MAX) / kChunk;
  static constexpr int PW = 4;
  static constexpr int MMA_WARP = PW, EPI_WARP0 = PW + 1, THREADS = (PW + 1 + kEpiWarps) * 32;
  static constexpr int S = (S_RAW > 12 ? 12 : S_RAW) / PW * PW;
  static constexpr int NBUF = 4 * DE <= 512 ? 2 : 1;
  static constexpr int CTRL = RING + S * kChunk;
  static constexpr int B_FULL = CTRL, B_EMPTY = B_FULL + 8 * S;
  static constexpr int B_W1F = B_EMPTY + 8 * S, B_W1E = B_W1F + 8, B_W2F = B_W1E + 8, B_W2E = B_W2F + 8;
  static constexpr int B_HDFULL = B_W2E + 8, B_HDFREE = B_HDFULL + 16;
  static constexpr int DG = B_HDFREE + 16;
  static constexpr int TMEMP = DG + (kEpiWarps / 4) * BM * 4;
  static constexpr int BYTES = TMEMP + 16;
  static_assert(BYTES - CTRL <= CTRL_MAX, "control block overflow");
  static_assert(BYTES <= kMaxSmem, "K1 pair: shared memory over the per-CTA limit");
  static_assert(S >= PW, "ring too small");
};

template <int DH, int DE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(HLP<DH, DE>::THREADS, 1)
expert_bwd_h_pair_kernel(const __grid_constant__ CUtensorMap w1map, const __grid_constant__ CUtensorMap w2map,
                         const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap ymap,
                         const __grid_constant__ CUtensorMap hsmap, const __grid_constant__ CUtensorMap asmap,
                         Routing rt, float* __restrict__ dg) {
  using L = HLP<DH, DE>;
  constexpr int kProdWarps = L::PW, kMmaWarp = L::MMA_WARP, kEpiWarp0 = L::EPI_WARP0, NBUF = L::NBUF;
  constexpr int S = L::S, KB = DH / 64;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0u) __trap();
  const uint32_t sb = smem_u32(smem);
  auto bar = [&](int off) { return reinterpret_cast<uint64_t*>(smem + off); };
  auto lead = [&](int off) { return map_to_rank(sb + off, 0); };
  float* s_dg = reinterpret_cast<float*>(smem + L::DG);
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::TMEMP);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  const int t_lo = rt.trange ? rt.trange[0] : 0;   // tile window (NEXT-1) or every tile
  const Tile* tiles = rt.tiles + t_lo;
  const int N_e = rt.N_e;
  const int64_t Rp = rt.Rp, R = rt.T * rt.k;

  if (tid == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(bar(L::B_FULL + 8 * i), 1); mbar_init(bar(L::B_EMPTY + 8 * i), 1); }
    mbar_init(bar(L::B_W1F), 1); mbar_init(bar(L::B_W1E), 1); mbar_init(bar(L::B_W2F), 1); mbar_init(bar(L::B_W2E), 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar(L::B_HDFULL + 8 * b), 1);
      mbar_init(bar(L::B_HDFREE + 8 * b), 2 * kEpiWarps);      // one arrival per epilogue warp of each CTA
    }
    fence_mbar_init();
    tma_prefetch_desc(&w1map); tma_prefetch_desc(&w2map); tma_prefetch_desc(&xmap); tma_prefetch_desc(&ymap);
    tma_prefetch_desc(&hsmap); tma_prefetch_desc(&asmap);
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(s_tmem)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  // pair-tile schedule: pair-tile u = tiles (2u, 2u+1) (same head and expert); this CTA: 2u + rank
  const int npt = *rt.ntiles / 2;
  constexpr int G = kTileGroup / 2 > 0 ? kTileGroup / 2 : 1;
  const int pair = (int)blockIdx.x >> 1, npairs = (int)gridDim.x >> 1;
  const int ngroups = (npt + G - 1) / G;
  const int my_groups = ngroups > pair ? (ngroups - 1 - pair) / npairs + 1 : 0;
  auto pt_at = [&](int i) -> int {
    if (i < 0 || i >= my_groups * G) return -1;
    const int u = (pair + (i / G) * npairs) * G + i % G;
    return u < npt ? u : -1;
  };
  auto same_expert = [&](int ua, int ub) {
    if (ua < 0 || ub < 0) return false;
    const Tile a = tiles[2 * ua], b = tiles[2 * ub];
    return a.head == b.head && a.expert == b.expert;
  };
  auto load_wh = [&](const CUtensorMap* map, int off, int foff, const Tile& t) {   // this CTA's N half
    if (leader) mbar_expect_tx_local(sb + foff, 2 * L::WH);
    for (int kb = 0; kb < KB; ++kb)
      load2d_pair(sb + off + kb * (DE / 2) * 128, map, kb * 64, (t.head * N_e + t.expert) * DE + (int)rank * (DE / 2),
                  lead(foff));
  };

  if (warp < kProdWarps) {
    // ================================================================ producers
    const int pw = warp;
    Ph w1e, w2e;
    int cnt = 0;
    int nx[4] = {0, 0, 0, 0};
    auto load_tok = [&](int u) {
      if (u < 0) return;
      const Tile t = tiles[2 * u + rank];
      const int32_t* tk = rt.tok_s + (size_t)t.head * Rp + t.row0 + 4 * lane;
      nx[0] = tk[0]; nx[1] = tk[1]; nx[2] = tk[2]; nx[3] = tk[3];
    };
    load_tok(pt_at(0));
    for (int i = 0;; ++i) {
      const int u = pt_at(i);
      if (u < 0) break;
      const Tile tl = tiles[2 * u + rank];
      const bool fresh = !same_expert(pt_at(i - 1), u);
      const int r0 = nx[0], r1 = nx[1], r2 = nx[2], r3 = nx[3];
      load_tok(pt_at(i + 1));
      if (pw == 0 && lane == 0 && fresh) {
        mbar_wait(bar(L::B_W1E), w1e.flip() ^ 1);
        load_wh(&w1map, L::W1, L::B_W1F, tl);
        mbar_wait(bar(L::B_W2E), w2e.flip() ^ 1);
        load_wh(&w2map, L::W2, L::B_W2F, tl);
      }
      __syncwarp();
      for (int j = 0; j < 2 * KB; ++j, ++cnt) {
        if (cnt % kProdWarps != pw) continue;
        const int st = cnt % S;
        if (lane == 0) {
          mbar_wait(bar(L::B_EMPTY + 8 * st), ((cnt / S) & 1) ^ 1);
          if (leader) mbar_expect_tx_local(sb + L::B_FULL + 8 * st, 2 * kChunk);
        }
        __syncwarp();
        const int kb = j % KB;
        gather4_pair(sb + L::RING + st * kChunk + lane * 4 * 128, j < KB ? &xmap : &ymap, tl.head * DH + kb * 64, r0,
                     r1, r2, r3, lead(L::B_FULL + 8 * st));
      }
    }
  } else if (warp == kMmaWarp) {
    // ================================================================ MMA issuer (leader CTA only)
    if (leader && lane == 0) {
      constexpr uint32_t ID_N_DE = idesc_bf16(2 * BM, DE, 0, 0);
      Ph w1f, w2f, hdfr[2];
      int cnt = 0;
      auto gemm_k = [&](uint32_t d, int woff) {
        for (int kb = 0; kb < KB; ++kb, ++cnt) {
          const int st = cnt % S;
          mbar_wait(bar(L::B_FULL + 8 * st), (cnt / S) & 1);
          tc_fence_after();
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            mma_pair(d, sdesc_sw128(sb + L::RING + st * kChunk + ks * 32, 16, 1024),
                     sdesc_sw128(sb + woff + kb * (DE / 2) * 128 + ks * 32, 16, 1024), ID_N_DE, (kb | ks) ? 1u : 0u);
          commit_pair(bar(L::B_EMPTY + 8 * st));
        }
      };
      for (int i = 0;; ++i) {
        const int u = pt_at(i);
        if (u < 0) break;
        const int b = i % NBUF;
        const bool fresh = !same_expert(pt_at(i - 1), u);
        const bool last = !same_expert(u, pt_at(i + 1));
        if (fresh) mbar_wait(bar(L::B_W1F), w1f.flip());
        if (i >= NBUF) mbar_wait(bar(L::B_HDFREE + 8 * b), hdfr[b].flip());
        tc_fence_after();
        gemm_k(tmem + 2 * DE * b, L::W1);
        if (last) commit_pair(bar(L::B_W1E));
        if (fresh) mbar_wait(bar(L::B_W2F), w2f.flip());
        gemm_k(tmem + 2 * DE * b + DE, L::W2);
        commit_pair(bar(L::B_HDFULL + 8 * b));
        if (last) commit_pair(bar(L::B_W2E));
      }
    }
  } else {
    // ================================================================ epilogue (16 warps, this CTA's rows)
    constexpr int NG = kEpiWarps / 4, NC = DE / NG, WPB = 64 / NC;
    const int q = warp & 3, cg = (warp - kEpiWarp0) >> 2;
    const int box = cg * NC / 64, bcol = cg * NC % 64;
    const bool wleader = (bcol == 0 && lane == 0);
    const int bar_box = 2 + q * L::BOXES + box, bar_dg = (WPB > 1 ? 2 + 4 * L::BOXES : 2) + q;
    static_assert(WPB == 1 || 2 + 4 * L::BOXES + 4 <= 16, "K1 pair: named barrier ids exhausted");
    auto box_sync = [&]() { if constexpr (WPB > 1) named_bar_sync(bar_box, 32 * WPB); else __syncwarp(); };
    uint8_t* slot = smem + L::STG + (q * L::BOXES + box) * 4096;
    const uint32_t slot_s = sb + L::STG + (q * L::BOXES + box) * 4096;
    const int row = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    Ph hd[2];
    auto stage = [&](const uint32_t* w) {
#pragma unroll
      for (int c = 0; c < NC; c += 8)
        *reinterpret_cast<uint4*>(slot + kmaj_off(lane, bcol + c, 32)) =
            make_uint4(w[c / 2], w[c / 2 + 1], w[c / 2 + 2], w[c / 2 + 3]);
      fence_proxy_async();
    };
    for (int i = 0;; ++i) {
      const int u = pt_at(i);
      if (u < 0) break;
      const int b = i % NBUF;
      const Tile tl = tiles[2 * u + rank];
      const size_t grow = (size_t)tl.head * Rp + tl.row0 + row;
      const int orow = (int)((size_t)tl.head * Rp + tl.row0 + q * 32);
      const float g = rt.gate_s[grow];
      const int rep = rt.perm[grow];
      mbar_wait_warp(bar(L::B_HDFULL + 8 * b), hd[b].flip());
      tc_fence_after();
      float dgp = 0.f;
      uint32_t dhp[NC / 2], gap[NC / 2];
#pragma unroll
      for (int c = 0; c < NC; c += 16) {
        uint32_t hv[16], dv[16];
        const uint32_t col = lane_off + cg * NC + c;
        tmem_ld16(tmem + 2 * DE * b + col, hv);
        tmem_ld16(tmem + 2 * DE * b + DE + col, dv);
        tmem_ld_wait();
        if (c + 16 >= NC) {                       // this warp's TMEM reads are done: one arrival
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (leader) mbar_arrive(bar(L::B_HDFREE + 8 * b));
            else mbar_arrive_relaxed_cluster(lead(L::B_HDFREE + 8 * b));
          }
        }
#pragma unroll
        for (int x = 0; x < 16; x += 2) {
          const float2 h2 = make_float2(__uint_as_float(hv[x]), __uint_as_float(hv[x + 1]));
          const float2 d2 = make_float2(__uint_as_float(dv[x]), __uint_as_float(dv[x + 1]));
          float2 gp;
          const float2 a = gelu2(h2, &gp);
          dgp = fmaf(a.x, d2.x, dgp);
          dgp = fmaf(a.y, d2.y, dgp);
          const float2 dh = __fmul2_rn(__fmul2_rn(d2, gp), make_float2(g, g));
          const float2 ga = __fmul2_rn(a, make_float2(g, g));
          dhp[(c + x) / 2] = pack_bf16x2(dh.x, dh.y);
          gap[(c + x) / 2] = pack_bf16x2(ga.x, ga.y);
        }
      }
      if (wleader) bulk_wait_read<0>();
      box_sync();
      stage(dhp);
      box_sync();
      if (wleader) { tma_store_2d(&hsmap, slot_s, box * 64, orow); bulk_commit(); bulk_wait_read<0>(); }
      box_sync();
      stage(gap);
      box_sync();
      if (wleader) { tma_store_2d(&asmap, slot_s, box * 64, orow); bulk_commit(); }
      s_dg[cg * BM + row] = dgp;
      named_bar_sync(bar_dg, 32 * NG);
      if (cg == 0 && rep >= 0) {
        float acc = s_dg[row];
#pragma unroll
        for (int x = 1; x < NG; ++x) acc += s_dg[x * BM + row];
        dg[(size_t)tl.head * R + rep] = acc;
      }
      named_bar_sync(bar_dg, 32 * NG);
    }
    if (wleader) bulk_wait_all();
  }
  tc_fence_before();
  cluster_sync();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// =============================================================================================
// kernel 2: dXrep = dH W1_e
// =============================================================================================
constexpr int kThreads2 = 10 * 32;
constexpr int kEpiThreads2 = 8 * 32;
constexpr int kYStage = BM * 128;    // one 64-column block of the dX tile (16 KB)

template <int DH, int DE>
struct GL {
  static constexpr int WB = DE * DH * 2;
  static constexpr int ASTAGE = DE * BM * 2;                // one dH tile: DE/64 chunks of 16 KB
  static constexpr int W1 = 0, YS = WB, A = YS + 2 * kYStage;
  static constexpr int CTRL_MAX = 1024;
  static constexpr int WRB = 2 * DH * 4;                     // W_r^T[h][e] rows of two tiles (router term)
  static constexpr int AS_RAW = (kMaxSmem - A - CTRL_MAX - WRB) / ASTAGE;
  static constexpr int AS = AS_RAW > 4 ? 4 : AS_RAW;
  static constexpr int WR = A + AS * ASTAGE;
  static constexpr int CTRL = WR + WRB;
  static constexpr int B_AFULL = CTRL, B_AEMPTY = B_AFULL + 8 * AS;
  static constexpr int B_W1F = B_AEMPTY + 8 * AS, B_W1E = B_W1F + 8;
  static constexpr int B_DXFULL = B_W1E + 8, B_DXEMPTY = B_DXFULL + 16;
  static constexpr int TMEMP = B_DXEMPTY + 16;
  static constexpr int BYTES = TMEMP + 16;
  static constexpr int TMEM_COLS = 2 * DH <= 256 ? 256 : 512;
  static_assert(BYTES - CTRL <= CTRL_MAX, "control block overflow");
  static_assert(AS >= 2, "dH ring too small");
  static_assert(BYTES <= kMaxSmem, "K2: shared memory over the per-CTA limit");
};

template <int DH, int DE>
__global__ void __launch_bounds__(kThreads2, 1)
expert_dx_gemm_kernel(const __grid_constant__ CUtensorMap w1map, const __grid_constant__ CUtensorMap hmap,
                      const __grid_constant__ CUtensorMap xmap, Routing rt, const float* __restrict__ dS,
                      const float* __restrict__ W_rT, uint8_t* __restrict__ xout, int lsu) {
  using L = GL<DH, DE>;
  constexpr int AS = L::AS, KB = DH / 64;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0u) __trap();
  const uint32_t sb = smem_u32(smem);
  auto bar = [&](int off) { return reinterpret_cast<uint64_t*>(smem + off); };
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::TMEMP);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t_lo = rt.trange ? rt.trange[0] : 0;   // tile window (NEXT-1) or every tile
  const Tile* tiles = rt.tiles + t_lo;
  const int N_e = rt.N_e;
  const int64_t Rp = rt.Rp;

  if (tid == 0) {
    for (int i = 0; i < AS; ++i) { mbar_init(bar(L::B_AFULL + 8 * i), 1); mbar_init(bar(L::B_AEMPTY + 8 * i), 1); }
    mbar_init(bar(L::B_W1F), 1); mbar_init(bar(L::B_W1E), 1);
    for (int b = 0; b < 2; ++b) { mbar_init(bar(L::B_DXFULL + 8 * b), 1); mbar_init(bar(L::B_DXEMPTY + 8 * b), kEpiThreads2); }
    fence_mbar_init();
    tma_prefetch_desc(&w1map); tma_prefetch_desc(&hmap); tma_prefetch_desc(&xmap);
  }
  if (warp == 1) tmem_alloc<L::TMEM_COLS>(s_tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  const Sched sc(tiles, (rt.trange ? rt.trange[1] : *rt.ntiles) - t_lo);

  if (warp == 0) {
    // ================================================================ TMA producer
    if (lane == 0) {
      Ph ae[4], w1e;
      int st = 0;
      for (int i = 0;; ++i) {
        const int ti = sc.at(i);
        if (ti < 0) break;
        const Tile tl = tiles[ti];
        mbar_wait(bar(L::B_AEMPTY + 8 * st), ae[st].flip() ^ 1);
        mbar_expect_tx(bar(L::B_AFULL + 8 * st), L::ASTAGE);
        for (int kb = 0; kb < DE / 64; ++kb)
          tma_load_2d(sb + L::A + st * L::ASTAGE + kb * kChunk, &hmap, kb * 64, (int)((size_t)tl.head * Rp + tl.row0),
                      bar(L::B_AFULL + 8 * st));
        if (++st == AS) st = 0;
        if (!sc.same_expert(sc.at(i - 1), ti)) {
          mbar_wait(bar(L::B_W1E), w1e.flip() ^ 1);
          mbar_expect_tx(bar(L::B_W1F), L::WB);
          for (int kb = 0; kb < KB; ++kb)
            tma_load_2d(sb + L::W1 + kb * DE * 128, &w1map, kb * 64, (tl.head * N_e + tl.expert) * DE, bar(L::B_W1F));
        }
      }
    }
  } else if (warp == 1) {
    // ================================================================ MMA issuer
    if (lane == 0) {
      constexpr uint32_t ID = idesc_bf16(BM, DH, 0, 1);     // B = W1_e viewed MN-major (N = d_h)
      Ph af[4], w1f, dxe[2];
      int st = 0;
      for (int i = 0;; ++i) {
        const int ti = sc.at(i);
        if (ti < 0) break;
        const int b = i & 1;
        if (!sc.same_expert(sc.at(i - 1), ti)) mbar_wait(bar(L::B_W1F), w1f.flip());
        mbar_wait(bar(L::B_DXEMPTY + 8 * b), dxe[b].flip() ^ 1);
        mbar_wait(bar(L::B_AFULL + 8 * st), af[st].flip());
        tc_fence_after();
        const uint32_t a0 = sb + L::A + st * L::ASTAGE;
#pragma unroll
        for (int ks = 0; ks < DE / 16; ++ks)
          mma_bf16(tmem + b * DH, sdesc_sw128(a0 + (ks >> 2) * kChunk + (ks & 3) * 32, 16, 1024),
                   sdesc_sw128(sb + L::W1 + ks * 2 * 1024, DE * 128, 1024), ID, ks > 0);
        mma_commit(bar(L::B_AEMPTY + 8 * st));
        mma_commit(bar(L::B_DXFULL + 8 * b));
        if (!sc.same_expert(ti, sc.at(i + 1))) mma_commit(bar(L::B_W1E));
        if (++st == AS) st = 0;
      }
    }
  } else {
    // ================================================================ epilogue (8 warps)
    const int q = warp & 3, half = (warp - 2) >> 2;    // lane quadrant, 32-column half of a block
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const bool leader = (half == 0 && lane == 0);
    const int et = tid - 64;                            // epilogue thread 0..255
    float* s_wr = reinterpret_cast<float*>(smem + L::WR);
    // Router term of Alg. 2 l.9, fused here so B6 is a plain k-row sum: dXrep[row] += dS_s[row] *
    // W_r[h][:, e] (e = the tile's expert; dS_s = dS in sorted-row order, 0 on padding rows).  The
    // next tile's W_r^T row element and dS values are fetched one tile ahead, so their L2 latency
    // hides behind this tile's epilogue.
    const bool rterm = dS != nullptr;
    auto w_of = [&](int t) -> float {
      if (!rterm || t < 0 || et >= DH) return 0.f;
      const Tile u = tiles[t];
      return __ldg(W_rT + ((size_t)u.head * N_e + u.expert) * DH + et);
    };
    auto ds_of = [&](int t) -> float {   // dS in sorted-row order (0 on padding rows)
      if (!rterm || t < 0) return 0.f;
      const Tile u = tiles[t];
      return __ldg(dS + (size_t)u.head * Rp + u.row0 + q * 32 + lane);
    };
    float w_cur = w_of(sc.at(0));
    float ds = ds_of(sc.at(0));
    Ph dxf[2];
    int ys = 0;
    for (int i = 0;; ++i) {
      const int ti = sc.at(i);
      if (ti < 0) break;
      const int b = i & 1;
      const Tile tl = tiles[ti];
      const int tn = sc.at(i + 1);
      const float* wr = s_wr + b * DH;
      if (rterm) {
        if (et < DH) s_wr[b * DH + et] = w_cur;
        named_bar_sync(7, kEpiThreads2);   // slot b published; slot b is rewritten only after the next barrier
      }
      w_cur = w_of(tn);
      const float ds_n = ds_of(tn);
      mbar_wait_warp(bar(L::B_DXFULL + 8 * b), dxf[b].flip());
      tc_fence_after();
#pragma unroll 1
      for (int cb = 0; cb < KB; ++cb, ++ys) {
        const int st = ys & 1;
        uint32_t v[32];
        tmem_ld32(tmem + b * DH + lane_off + cb * 64 + half * 32, v);
        tmem_ld_wait();
        if (rterm) {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float4 w4 = *reinterpret_cast<const float4*>(wr + cb * 64 + half * 32 + 4 * u);
            v[4 * u + 0] = __float_as_uint(fmaf(ds, w4.x, __uint_as_float(v[4 * u + 0])));
            v[4 * u + 1] = __float_as_uint(fmaf(ds, w4.y, __uint_as_float(v[4 * u + 1])));
            v[4 * u + 2] = __float_as_uint(fmaf(ds, w4.z, __uint_as_float(v[4 * u + 2])));
            v[4 * u + 3] = __float_as_uint(fmaf(ds, w4.w, __uint_as_float(v[4 * u + 3])));
          }
        }
        if (cb == KB - 1) {
          tc_fence_before();
          mbar_arrive(bar(L::B_DXEMPTY + 8 * b));
        }
        if (leader && !lsu) bulk_wait_read<1>();   // the slab store issued from this stage 2 blocks ago has read it
        named_bar_sync(2 + q, 64);
        uint8_t* sp = smem + L::YS + st * kYStage + q * 4096;
#pragma unroll
        for (int u = 0; u < 32; u += 8) {
          uint4 pk;
          pk.x = pack_bf16x2(__uint_as_float(v[u + 0]), __uint_as_float(v[u + 1]));
          pk.y = pack_bf16x2(__uint_as_float(v[u + 2]), __uint_as_float(v[u + 3]));
          pk.z = pack_bf16x2(__uint_as_float(v[u + 4]), __uint_as_float(v[u + 5]));
          pk.w = pack_bf16x2(__uint_as_float(v[u + 6]), __uint_as_float(v[u + 7]));
          *reinterpret_cast<uint4*>(sp + kmaj_off(lane, half * 32 + u, 32)) = pk;
        }
        if (lsu) {   // coalesced 16-byte stores by the quadrant's two warps (see expert_sm100.cu)
          named_bar_sync(2 + q, 64);
          const int bt = half * 32 + lane;
          uint8_t* dst = xout + ((size_t)tl.head * Rp + tl.row0 + q * 32) * (DH * 2) + cb * 128;
#pragma unroll
          for (int c = bt; c < 256; c += 64) {
            const int r = c >> 3, c16 = c & 7;
            *reinterpret_cast<uint4*>(dst + (size_t)r * (DH * 2) + c16 * 16) =
                *reinterpret_cast<const uint4*>(sp + r * 128 + (((c16 ^ (r & 7)) & 7) << 4));
          }
        } else {
          fence_proxy_async();
          named_bar_sync(2 + q, 64);
          if (leader) {
            tma_store_2d(&xmap, sb + L::YS + st * kYStage + q * 4096, cb * 64, (int)((size_t)tl.head * Rp + tl.row0 + q * 32));
            bulk_commit();
          }
        }
      }
      ds = ds_n;
    }
    if (leader) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<L::TMEM_COLS>(tmem);
}

template <int DH, int DE>
bool launch_t(const Routing& rt, const void* Xs, int64_t ldx, const void* dY, int64_t ldy, const void* W1,
              const void* W2, void* dXrep, float* dg, void* dH, void* gA, int num_sms, cudaStream_t s) {
  CUtensorMap w1m, w2m, gxm, gym, hsm, asm_;
  // dH / gA store maps: [H*Rp rows][d_e], box = 64 columns x 32 rows (one epilogue lane quadrant)
  if (!make_tmap_2d_bf16(&hsm, dH, (uint64_t)rt.H * rt.Rp, DE, (uint64_t)DE * 2, 32, 64)) return false;
  if (!make_tmap_2d_bf16(&asm_, gA, (uint64_t)rt.H * rt.Rp, DE, (uint64_t)DE * 2, 32, 64)) return false;
  const uint64_t wrows = (uint64_t)rt.H * rt.N_e * DE;
  // gather maps over the sub-token / dcat rows (T+1 rows, row T all-zero), box = 64 columns x 1 row
  if (!make_tmap_2d_bf16(&gxm, Xs, (uint64_t)rt.T + 1, (uint64_t)rt.H * DH, (uint64_t)ldx * 2, 1, 64)) return false;
  if (!make_tmap_2d_bf16(&gym, dY, (uint64_t)rt.T + 1, (uint64_t)rt.H * DH, (uint64_t)ldy * 2, 1, 64)) return false;
  if (!make_tmap_2d_bf16(&w1m, W1, wrows, DH, (uint64_t)DH * 2, DE, 64)) return false;
  if (!make_tmap_2d_bf16(&w2m, W2, wrows, DH, (uint64_t)DH * 2, DE, 64)) return false;
  auto k1 = expert_bwd_h_kernel<DH, DE>;
  cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, HL<DH, DE>::BYTES);
  static const char* trace_path = getenv("MHL_TRACE_DX");
  if (trace_path) {
    TraceBuf tb{trace_buffer(s), 0};
    cudaMemcpyToSymbolAsync(g_trace_dx, &tb, sizeof(tb), 0, cudaMemcpyHostToDevice, s);
  }
  static const int dbg = timing_only_switch("MHL_DX_DBG");
  if (rt.seg_align % (2 * kExpertBM) == 0 && num_sms >= 2) {   // MHL_FLAG_PAIR: CTA-pair variant
    // CTA-pair variant: W maps with half-height boxes (each CTA loads its d_e/2 rows)
    CUtensorMap w1h, w2h;
    const uint64_t wr = (uint64_t)rt.H * rt.N_e * DE;
    if (!make_tmap_2d_bf16(&w1h, W1, wr, DH, (uint64_t)DH * 2, DE / 2, 64)) return false;
    if (!make_tmap_2d_bf16(&w2h, W2, wr, DH, (uint64_t)DH * 2, DE / 2, 64)) return false;
    auto kp = expert_bwd_h_pair_kernel<DH, DE>;
    cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, HLP<DH, DE>::BYTES);
    kp<<<(num_sms / 2) * 2, HLP<DH, DE>::THREADS, HLP<DH, DE>::BYTES, s>>>(w1h, w2h, gxm, gym, hsm, asm_, rt, dg);
  } else {
    k1<<<num_sms, HL<DH, DE>::THREADS, HL<DH, DE>::BYTES, s>>>(w1m, w2m, gxm, gym, hsm, asm_, rt, dg, dbg,
                                                              (uint8_t*)dH, (uint8_t*)gA, store_lsu(1));
  }
  if (trace_path) {
    TraceBuf tb{nullptr, 0};
    cudaMemcpyToSymbolAsync(g_trace_dx, &tb, sizeof(tb), 0, cudaMemcpyHostToDevice, s);
    trace_dump(trace_path, s);
  }
  return true;
}

template <int DH, int DE>
bool launch_gemm_t(const Routing& rt, const void* W1, const void* dH, void* dXrep, const float* dS, const float* W_rT,
                   int num_sms, cudaStream_t s) {
  CUtensorMap w1m, hm, xm;
  const uint64_t wrows = (uint64_t)rt.H * rt.N_e * DE, rows = (uint64_t)rt.H * rt.Rp;
  if (!make_tmap_2d_bf16(&w1m, W1, wrows, DH, (uint64_t)DH * 2, DE, 64)) return false;
  if (!make_tmap_2d_bf16(&hm, dH, rows, DE, (uint64_t)DE * 2, BM, 64)) return false;
  if (!make_tmap_2d_bf16(&xm, dXrep, rows, DH, (uint64_t)DH * 2, 32, 64)) return false;
  auto k2 = expert_dx_gemm_kernel<DH, DE>;
  cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, GL<DH, DE>::BYTES);
  k2<<<num_sms, kThreads2, GL<DH, DE>::BYTES, s>>>(w1m, hm, xm, rt, dS, W_rT, (uint8_t*)dXrep, store_lsu(0));
  return true;
}

}  // namespace

bool launch_expert_bwd_dx_sm100(const Routing& rt, const void* Xs, int64_t ldx, const void* dY, int64_t ldy,
                                const void* W1, const void* W2, int d_h, int d_e, void* dXrep, float* dg, void* dH,
                                void* gA, int num_sms, cudaStream_t s) {
#define MHL_DX(A, B) \
  if (d_h == A && d_e == B) return launch_t<A, B>(rt, Xs, ldx, dY, ldy, W1, W2, dXrep, dg, dH, gA, num_sms, s);
  MHL_DX(256, 128) MHL_DX(256, 64) MHL_DX(128, 128) MHL_DX(128, 64) MHL_DX(128, 256)
#undef MHL_DX
  return false;
}

bool launch_expert_dx_gemm_sm100(const Routing& rt, const void* W1, int d_h, int d_e, const void* dH, void* dXrep,
                                 const float* dS, const float* W_rT, int num_sms, cudaStream_t s) {
#define MHL_DX(A, B) \
  if (d_h == A && d_e == B) return launch_gemm_t<A, B>(rt, W1, dH, dXrep, dS, W_rT, num_sms, s);
  MHL_DX(256, 128) MHL_DX(256, 64) MHL_DX(128, 128) MHL_DX(128, 64) MHL_DX(128, 256)
#undef MHL_DX
  return false;
}

}  // namespace mhl
