// expert_bwd_fused_sm100.cu — B5 (input side) in ONE persistent tcgen05 kernel: H, dA', the
// epilogue and the dX contraction of each 128-row expert tile (P:936 chain rule, Eq. 1).
//
// Per tile of expert e (clustered rows r, gathered sub-tokens X_r and dcat rows dY_r, gate g_r):
//   G_dA  dA' = dY W2_e^T                  TMEM [DE, 2DE)       A = gathered dY chunks, B = W2_e
//   G_H   H   = X  W1_e^T                  TMEM [0, DE)         A = gathered X chunks,  B = W1_e
//   GELU  dg = <gelu(H), dA'>,  dH = g dA' gelu'(H),  gA = g gelu(H)
//         dH -> TMEM columns [0, DE/2) over H (bf16 pairs: the A operand of G_dX) and -> HBM,
//         gA -> HBM (dH, gA: the dW kernel's inputs), straight from registers
//   G_dX  dXrep = dH W1_e                  TMEM [2DE, 2DE+DH)   A = dH in TMEM, B = W1_e (MN-major view)
//   dX    dXrep -> bf16 -> HBM from registers
// The router term dS W_r^T of Alg. 2 l.9 is added by B6 (combine.cu, W_r^T staged in smem), so
// this kernel does not wait for the router backward: it replaces the former K1 (H, dA' -> dH, gA)
// and K2 (dH re-read from HBM -> dX GEMM) pair (the default; this kernel is MHL_FLAG_BWD_FUSED), saving K2's read of dH, its
// launch and its own pipeline per tile.
//
// TMEM: the GELU group reads H and dA' into registers and releases them at once (HDFREE), so G_dA
// of tile i+1 runs during tile i's GELU math; dH(i) then overwrites H(i)'s columns, and G_H(i+1),
// issued after G_dX(i) in program order, overwrites dH(i) only once it is consumed.  dX takes the
// other DH columns (2 DE + DH <= 512).  SMEM: W1_e, W2_e resident per expert run (re-fetched on an
// expert change) and a 6-stage ring of gathered 64-column chunks (a tile is 2 x DH/64 chunks), so
// the gathers of tile i+1 start while tile i's are still held.
// MMA issue order per tile i: G_dA(i), G_dX(i-1), G_H(i).  W2 is released after G_dA of an
// expert's last tile and W1 after its G_dX, so on an expert change the producer refetches W2
// first, issues the new tile's dY chunks, then waits for W1's release (G_dX of the previous tile,
// which follows G_dA(i) in issue order — the dY-before-X chunk order is what avoids a cycle).
// Warps: 8 producers (two owners of 4 warps, TMA gather4), 16 GELU warps (lane quadrant x column
// quarter: one row, DE/4 columns per thread), 4 dX warps (one per lane quadrant: the DH columns of
// 32 rows), 1 MMA issuer; the dX read-out of tile i overlaps the GELU math of tile i+1.
#include <cuda.h>

#include <cstdlib>

#include "kernels.h"
#include "sm100.cuh"
#include "tma_host.h"

namespace mhl {

namespace {

using namespace sm100;

__device__ __forceinline__ void tma_store_2d(const void* tmap, uint32_t src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tmap), "r"(src),
               "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ TraceBuf g_trace_fb;   // profiling aid (MHL_TRACE_FB=<file>): per-tile phase stamps of CTA 0

constexpr int BM = kExpertBM;
constexpr int kChunk = BM * 128;   // one 64-column K-chunk of a 128-row tile (16 KB)
constexpr int kMaxSmem = 227 * 1024;
constexpr int kEpiWarps = 16;     // GELU group: H, dA' -> dg, dH, gA
constexpr int kEpiThreads = kEpiWarps * 32;
constexpr int kXWarps = 4;        // dX group: one warp per TMEM lane quadrant reads dXrep out
constexpr int kXThreads = kXWarps * 32;
constexpr int kProdWarps = 8;
// dH for G_dX and for HBM: 1 = through an smem tile (SS-MMA operand + TMA bulk store; 4-stage ring),
// 0 = into TMEM over H (TS-MMA operand) + st.global from registers (6-stage ring)
#ifndef MHL_FB_SMEM_DH
#define MHL_FB_SMEM_DH 1
#endif
constexpr bool kSmemDH = MHL_FB_SMEM_DH != 0;      // in pairs: two warps (64 rows each) fill one chunk

struct Ph {
  uint32_t v = 0;
  __device__ uint32_t flip() { uint32_t o = v; v ^= 1u; return o; }
};


// Persistent schedule (as kernel 1 of expert_bwd_dx_sm100.cu): CTA b takes groups of kTileGroup
// consecutive tiles round-robin, so weights are reused within a group.
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

template <int DH, int DE>
struct FL {
  static constexpr int WB = DE * DH * 2;                    // one expert matrix (bf16)
  static constexpr int KB = DH / 64;
  static constexpr int DHS = kSmemDH ? BM * DE * 2 : 0;    // the dH tile: DE/64 SW128 chunks of 16 KB
  static constexpr int W1 = 0, W2 = WB, DHT = 2 * WB, RING = DHT + DHS;
  static constexpr int CTRL_MAX = 3 * 1024;
  static constexpr int S_RAW = (kMaxSmem - RING - CTRL_MAX) / kChunk;
  // chunk owners: pairs of producer warps fill one chunk (64 rows each), chunk c by pair c % OWNERS
  // into stage c % S.  The EMPTY parity stays exact without S being a multiple of OWNERS: chunk c
  // waits for the consumption of chunk c - S, and stage c % S cannot be consumed again before c
  // itself is filled.
  static constexpr int WPC = 2, OWNERS = kProdWarps / WPC;
  static constexpr int S = S_RAW > 12 ? 12 : S_RAW;
  static constexpr int CTRL = RING + S * kChunk;
  static constexpr int B_FULL = CTRL, B_EMPTY = B_FULL + 8 * S;
  static constexpr int B_W1F = B_EMPTY + 8 * S, B_W1E = B_W1F + 8, B_W2F = B_W1E + 8, B_W2E = B_W2F + 8;
  static constexpr int B_HDFULL = B_W2E + 8, B_HDFREE = B_HDFULL + 8, B_DHREADY = B_HDFREE + 8;
  static constexpr int B_DHFREE = B_DHREADY + 8, B_DXFULL = B_DHFREE + 8, B_DXFREE = B_DXFULL + 8;
  static constexpr int DG = B_DXFREE + 8;                   // [quarters 1..3][BM] float (dg partials)
  static constexpr int TMEMP = DG + 3 * BM * 4;
  static constexpr int BYTES = TMEMP + 16;
  // warps [0, 8) producers, [8, 24) GELU group, [24, 28) dX group, 28 the MMA issuer
  static constexpr int EPI_WARP0 = kProdWarps, X_WARP0 = kProdWarps + kEpiWarps, MMA_WARP = X_WARP0 + kXWarps;
  static constexpr int THREADS = (MMA_WARP + 1) * 32;
  // registers: 29 warps launch at 64 (sub-partition 0 holds 8: 2 producers, 4 GELU, 1 dX, the MMA
  // issuer); the producers' release to 32 covers the GELU warps' raise to 80 sub-partition by
  // sub-partition (2 x 32 = 4 x 16)
  static constexpr int LAUNCH_REGS = 64, PROD_REGS = 32, EPI_REGS = 80;
  static constexpr int NC = DE / 4, XC = DH / 4;            // H/dA' and dX columns per epilogue thread
  static_assert(2 * DE + DH <= 512, "fused backward: H, dA' and dX must fit TMEM together");
  static_assert(NC % 16 == 0 && XC % 32 == 0, "fused backward: column split");
  static_assert(BYTES - CTRL <= CTRL_MAX, "control block overflow");
  static_assert(BYTES <= kMaxSmem, "fused backward: shared memory over the per-CTA limit");
  static_assert(S >= OWNERS, "ring too small");
  static_assert(kProdWarps % OWNERS == 0 && BM % (4 * WPC) == 0 && BM / WPC <= 128, "producer split");
  static_assert(2 * (LAUNCH_REGS - PROD_REGS) >= 4 * (EPI_REGS - LAUNCH_REGS), "setmaxnreg budget");
  static_assert(THREADS == 928 && 8 * LAUNCH_REGS * 32 <= 16384, "launch register budget (8 warps on SMSP 0)");
};

template <int DH, int DE>
__global__ void __launch_bounds__(FL<DH, DE>::THREADS, 1)
expert_bwd_fused_kernel(const __grid_constant__ CUtensorMap w1map, const __grid_constant__ CUtensorMap w2map,
                        const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap ymap,
                        const __grid_constant__ CUtensorMap hsmap, Routing rt, float* __restrict__ dg,
                        uint8_t* __restrict__ dH_out,
                        uint8_t* __restrict__ gA_out, uint8_t* __restrict__ dX_out, int dbg) {
  using L = FL<DH, DE>;
  constexpr int S = L::S, KB = L::KB;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0u) __trap();
  const uint32_t sb = smem_u32(smem);
  auto bar = [&](int off) { return reinterpret_cast<uint64_t*>(smem + off); };
  float* s_dg = reinterpret_cast<float*>(smem + L::DG);
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::TMEMP);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  TraceBuf trc = g_trace_fb;
  const Tile* tiles = rt.tiles;
  const int N_e = rt.N_e;
  const int64_t Rp = rt.Rp, R = rt.T * rt.k;

  if (tid == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(bar(L::B_FULL + 8 * i), 1); mbar_init(bar(L::B_EMPTY + 8 * i), 1); }
    mbar_init(bar(L::B_W1F), 1); mbar_init(bar(L::B_W1E), 1); mbar_init(bar(L::B_W2F), 1); mbar_init(bar(L::B_W2E), 1);
    mbar_init(bar(L::B_HDFULL), 1);
    mbar_init(bar(L::B_HDFREE), kEpiThreads);
    mbar_init(bar(L::B_DHREADY), kSmemDH ? 1 : kEpiThreads);
    mbar_init(bar(L::B_DHFREE), 1);
    mbar_init(bar(L::B_DXFULL), 1);
    mbar_init(bar(L::B_DXFREE), kXThreads);
    fence_mbar_init();
    tma_prefetch_desc(&w1map); tma_prefetch_desc(&w2map); tma_prefetch_desc(&xmap); tma_prefetch_desc(&ymap);
  }
  if (warp == L::MMA_WARP) tmem_alloc<512>(s_tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  const Sched sc(tiles, *rt.ntiles);

  auto load_w = [&](const CUtensorMap* map, int off, uint64_t* full, const Tile& t) {
    mbar_expect_tx(full, L::WB);
    for (int kb = 0; kb < KB; ++kb) tma_load_2d(sb + off + kb * DE * 128, map, kb * 64, (t.head * N_e + t.expert) * DE, full);
  };

  if (warp < kProdWarps) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(L::PROD_REGS));
    // ================================================================ producers
    // A tile is 2*KB chunks (dY k-chunks, then X k-chunks); chunk c of the CTA's stream goes to
    // ring stage c % S and is filled by warp pair c % OWNERS (each warp 64 rows: 16 lanes x one
    // TMA gather4 of 4 rows).  Warp 0 lane 0 also (re)loads the weights on an expert change: W2
    // before the tile's dY chunks, W1 before its X chunks (see the header for the order).
    constexpr int OWN = L::OWNERS, WPC = L::WPC, LPW = BM / WPC / 4;   // lanes issuing per warp
    const int pw = warp, owner = pw / WPC;
    const int lrow = (pw % WPC) * (BM / WPC) + 4 * (lane % LPW);
    const bool issues = lane < LPW;
    const bool tx_lead = lane == 0 && pw % WPC == 0;
    const uint64_t pol_keep = l2_evict_last();   // rows reused k times per head
    Ph w1e, w2e;
    int cnt = 0;
    int nx[4] = {0, 0, 0, 0};
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
      const int r0 = nx[0], r1 = nx[1], r2 = nx[2], r3 = nx[3];
      load_tok(sc.at(i + 1));
      if (pw == 0 && lane == 0) trace_ev(trc, 1, i);
      for (int j = 0; j < 2 * KB; ++j, ++cnt) {
        if (j == 0 && fresh && pw == 0 && lane == 0) {
          mbar_wait(bar(L::B_W2E), w2e.flip() ^ 1);
          load_w(&w2map, L::W2, bar(L::B_W2F), tl);
        }
        if (j == KB && fresh && pw == 0 && lane == 0) {
          mbar_wait(bar(L::B_W1E), w1e.flip() ^ 1);
          load_w(&w1map, L::W1, bar(L::B_W1F), tl);
        }
        if (cnt % OWN != owner) continue;
        const int st = cnt % S;
        uint64_t* full = bar(L::B_FULL + 8 * st);
        if (lane == 0) mbar_wait(bar(L::B_EMPTY + 8 * st), ((cnt / S) & 1) ^ 1);
        if (tx_lead) mbar_expect_tx(full, kChunk);
        __syncwarp();
        const int kb = j % KB;
        if (j == KB && tx_lead) trace_ev(trc, 2, i);
        if (issues)
          tma_gather4_hint(sb + L::RING + st * kChunk + lrow * 128, j < KB ? &ymap : &xmap, tl.head * DH + kb * 64,
                           r0, r1, r2, r3, full, pol_keep);
      }
    }
  } else if (warp == L::MMA_WARP) {
    // ================================================================ MMA issuer
    if (lane == 0) {
      constexpr uint32_t ID_HD = idesc_bf16(BM, DE, 0, 0);     // N = d_e, both K-major
      constexpr uint32_t ID_DX = idesc_bf16(BM, DH, 0, 1);     // N = d_h, B = W1_e viewed MN-major
      Ph ff[12], w1f, w2f, hdfr, dhr, dxfr;
      static_assert(L::S <= 12, "ring phase array");
      int st = 0;
      auto gemm_k = [&](uint32_t d, int woff, int tev, int ti) {   // d = (ring chunks) . W^T over K = DH
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(bar(L::B_FULL + 8 * st), ff[st].flip());
          if (kb == 0) trace_ev(trc, tev, ti);
          tc_fence_after();
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            mma_bf16(d, sdesc_sw128(sb + L::RING + st * kChunk + ks * 32, 16, 1024),
                     sdesc_sw128(sb + woff + kb * DE * 128 + ks * 32, 16, 1024), ID_HD, (kb | ks) ? 1u : 0u);
          mma_commit(bar(L::B_EMPTY + 8 * st));
          if (++st == S) st = 0;
        }
      };
      // G_dX of tile i (its dH is in smem once the epilogue signals DHREADY)
      auto gemm_dx = [&](int i, bool last) {
        mbar_wait(bar(L::B_DHREADY), dhr.flip());
        if (i >= 1) mbar_wait(bar(L::B_DXFREE), dxfr.flip());   // the epilogue read dX(i-1)
        tc_fence_after();
        trace_ev(trc, 12, i);
        // A = dH(i), bf16 pairs in TMEM columns [0, DE/2) (over H(i), which the GELU group has read);
        // H(i+1) is issued after this in program order, so it overwrites dH only once it is consumed
#pragma unroll
        for (int ks = 0; ks < DE / 16; ++ks) {
          if constexpr (kSmemDH)
            mma_bf16(tmem + 2 * DE, sdesc_sw128(sb + L::DHT + (ks >> 2) * kChunk + (ks & 3) * 32, 16, 1024),
                     sdesc_sw128(sb + L::W1 + ks * 2 * 1024, DE * 128, 1024), ID_DX, ks > 0);
          else
            mma_bf16_ts(tmem + 2 * DE, tmem + ks * 8, sdesc_sw128(sb + L::W1 + ks * 2 * 1024, DE * 128, 1024), ID_DX,
                        ks > 0);
        }
        mma_commit(bar(L::B_DXFULL));
        if (kSmemDH) mma_commit(bar(L::B_DHFREE));
        if (last) mma_commit(bar(L::B_W1E));
      };
      int i = 0;
      for (;; ++i) {
        const int ti = sc.at(i);
        if (ti < 0) break;
        const bool fresh = !sc.same_expert(sc.at(i - 1), ti);
        const bool last = !sc.same_expert(ti, sc.at(i + 1));
        if (i >= 1) mbar_wait(bar(L::B_HDFREE), hdfr.flip());   // the epilogue holds H, dA'(i-1)
        trace_ev(trc, 10, i);
        if (fresh) mbar_wait(bar(L::B_W2F), w2f.flip());
        tc_fence_after();
        gemm_k(tmem + DE, L::W2, 15, i);                                  // dA'(i)
        trace_ev(trc, 11, i);
        if (last) mma_commit(bar(L::B_W2E));
        if (i >= 1) gemm_dx(i - 1, fresh);                         // dX(i-1); W1 free if i starts a run
        if (fresh) mbar_wait(bar(L::B_W1F), w1f.flip());
        tc_fence_after();
        gemm_k(tmem, L::W1, 14, i);                                       // H(i)
        mma_commit(bar(L::B_HDFULL));
        trace_ev(trc, 13, i);
      }
      if (i >= 1) gemm_dx(i - 1, true);
    }
  } else if (warp < L::X_WARP0) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(L::EPI_REGS));
    // ================================================================ GELU group (16 warps)
    constexpr int NC = L::NC;
    const int ew = warp - L::EPI_WARP0, q = warp & 3, cq = ew >> 2;   // lane quadrant, column quarter
    const int row = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const bool tw = ew == 0 && lane == 0;
    const uint64_t pol_out = l2_evict_first();
    Ph hdf, hdr, dhf;
    const bool issuer = ew == 0 && lane == 0;
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
      const Tile tl = tl_n;
      const float g = g_n;
      const int rep = rep_n;
      fetch(sc.at(i + 1));
      const size_t grow = (size_t)tl.head * Rp + tl.row0 + row;
      // ---- H, dA' -> registers; release the accumulators to the next tile's MMAs
      mbar_wait_warp(bar(L::B_HDFULL), hdf.flip());
      tc_fence_after();
      if (tw) trace_ev(trc, 20, i);
      uint32_t hv[NC], dv[NC];
#pragma unroll
      for (int c = 0; c < NC; c += 16) {
        tmem_ld16(tmem + lane_off + cq * NC + c, *reinterpret_cast<uint32_t(*)[16]>(hv + c));
        tmem_ld16(tmem + DE + lane_off + cq * NC + c, *reinterpret_cast<uint32_t(*)[16]>(dv + c));
      }
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(bar(L::B_HDFREE));
      if (tw) trace_ev(trc, 21, i);
      // ---- gelu, gelu', dg, dH, gA (fp32), bf16 pairs
      float dgp = 0.f;
      uint32_t wh[NC / 2], wa[NC / 2];
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
        wh[u / 2] = pack_bf16x2(dh.x, dh.y);
        wa[u / 2] = pack_bf16x2(ga.x, ga.y);
      }
      // gA straight to HBM (whole 32-byte sectors per lane)
      uint8_t* ga_row = gA_out + grow * (DE * 2) + cq * NC * 2;
#pragma unroll
      for (int u = 0; u < NC / 2; u += 8)
        if (!(dbg & 1))
        st_global_v8_hint(ga_row + u * 4, wa[u], wa[u + 1], wa[u + 2], wa[u + 3], wa[u + 4], wa[u + 5], wa[u + 6],
                          wa[u + 7], pol_out);
      // ---- dH -> TMEM over H (the G_dX A operand: bf16 pairs, columns [0, DE/2)) once every
      // GELU thread has read its H columns (the HDFREE phase of this tile), and -> HBM for dW
      if (tw) trace_ev(trc, 22, i);
      if constexpr (kSmemDH) {
        // smem tile, once G_dX(i-1) and the TMA store of dH(i-1) have read it
        if (issuer) bulk_wait_read0();
        if (i >= 1) mbar_wait_warp(bar(L::B_DHFREE), dhf.flip());
        named_bar_sync(1, kEpiThreads);
#pragma unroll
        for (int u = 0; u < NC; u += 8)
          *reinterpret_cast<uint4*>(smem + L::DHT + kmaj_off(row, cq * NC + u, BM)) =
              make_uint4(wh[u / 2], wh[u / 2 + 1], wh[u / 2 + 2], wh[u / 2 + 3]);
        fence_proxy_async();
        named_bar_sync(1, kEpiThreads);
        if (issuer) {
          trace_ev(trc, 23, i);
          mbar_arrive(bar(L::B_DHREADY));
          if (!(dbg & 1))
            for (int eb = 0; eb < DE / 64; ++eb)
              tma_store_2d(&hsmap, sb + L::DHT + eb * kChunk, eb * 64, (int)((size_t)tl.head * Rp + tl.row0));
          bulk_commit();
        }
      } else {
        mbar_wait_warp(bar(L::B_HDFREE), hdr.flip());
        if constexpr (NC == 32) tmem_st16(tmem + lane_off + cq * (NC / 2), *reinterpret_cast<const uint32_t(*)[16]>(wh));
        else tmem_st8(tmem + lane_off + cq * (NC / 2), *reinterpret_cast<const uint32_t(*)[8]>(wh));
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(bar(L::B_DHREADY));
        if (tw) trace_ev(trc, 23, i);
        uint8_t* dh_row = dH_out + grow * (DE * 2) + cq * NC * 2;
#pragma unroll
        for (int u = 0; u < NC / 2; u += 8)
          if (!(dbg & 1))
            st_global_v8_hint(dh_row + u * 4, wh[u], wh[u + 1], wh[u + 2], wh[u + 3], wh[u + 4], wh[u + 5], wh[u + 6],
                              wh[u + 7], pol_out);
      }
      // ---- dg: the four column-quarter partials of the row added in column order (one slot: the
      // next tile's writes follow named barrier 1, which the reading thread reaches after its read)
      if (cq > 0) s_dg[(cq - 1) * BM + row] = dgp;
      named_bar_sync(2 + q, 128);
      if (cq == 0 && rep >= 0)
        dg[(size_t)tl.head * R + rep] = ((dgp + s_dg[row]) + s_dg[BM + row]) + s_dg[2 * BM + row];
      named_bar_sync(2 + q, 128);   // s_dg is rewritten by the next tile
    }
    if (kSmemDH && issuer) bulk_wait_all();
  } else if (warp < L::MMA_WARP) {
    // ================================================================ dX group (4 warps)
    // warp q reads lane quadrant q of dXrep (all DH columns of its 32 rows), 32 columns per
    // tcgen05.ld, and stores each thread's row as whole 32-byte sectors; the TMEM columns are
    // released after the last read, so G_dX of the next tile overlaps the conversion and stores.
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const bool tw = q == 0 && lane == 0;
    const uint64_t pol_out = l2_evict_first();
    Ph dxf;
    for (int i = 0;; ++i) {
      const int ti = sc.at(i);
      if (ti < 0) break;
      const Tile tl = tiles[ti];
      uint8_t* dx_row = dX_out + ((size_t)tl.head * Rp + tl.row0 + row) * (DH * 2);
      mbar_wait_warp(bar(L::B_DXFULL), dxf.flip());
      tc_fence_after();
      if (tw) trace_ev(trc, 24, i);
#pragma unroll 1
      for (int c = 0; c < DH; c += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + 2 * DE + lane_off + c, v);
        tmem_ld_wait();
        if (c + 32 >= DH) {
          tc_fence_before();
          mbar_arrive(bar(L::B_DXFREE));
        }
        uint32_t w[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) w[u] = pack_bf16x2(__uint_as_float(v[2 * u]), __uint_as_float(v[2 * u + 1]));
        if (dbg & 2) continue;
        st_global_v8_hint(dx_row + c * 2, w[0], w[1], w[2], w[3], w[4], w[5], w[6], w[7], pol_out);
        st_global_v8_hint(dx_row + c * 2 + 32, w[8], w[9], w[10], w[11], w[12], w[13], w[14], w[15], pol_out);
      }
      if (tw) trace_ev(trc, 25, i);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == L::MMA_WARP) tmem_dealloc<512>(tmem);
}

template <int DH, int DE>
bool launch_t(const Routing& rt, const void* Xs, int64_t ldx, const void* dY, int64_t ldy, const void* W1,
              const void* W2, void* dXrep, float* dg, void* dH, void* gA, int num_sms, cudaStream_t s) {
  CUtensorMap w1m, w2m, gxm, gym, hsm;
  // dH store map: [H*Rp rows][d_e], box = 64 columns x 128 rows (one SW128 chunk of the dH tile)
  if (!make_tmap_2d_bf16(&hsm, dH, (uint64_t)rt.H * rt.Rp, DE, (uint64_t)DE * 2, BM, 64)) return false;
  const uint64_t wrows = (uint64_t)rt.H * rt.N_e * DE;
  // gather maps over the sub-token / dcat rows (T+1 rows, row T all-zero), box = 64 columns x 1 row
  if (!make_tmap_2d_bf16(&gxm, Xs, (uint64_t)rt.T + 1, (uint64_t)rt.H * DH, (uint64_t)ldx * 2, 1, 64)) return false;
  if (!make_tmap_2d_bf16(&gym, dY, (uint64_t)rt.T + 1, (uint64_t)rt.H * DH, (uint64_t)ldy * 2, 1, 64)) return false;
  if (!make_tmap_2d_bf16(&w1m, W1, wrows, DH, (uint64_t)DH * 2, DE, 64)) return false;
  if (!make_tmap_2d_bf16(&w2m, W2, wrows, DH, (uint64_t)DH * 2, DE, 64)) return false;
  auto k = expert_bwd_fused_kernel<DH, DE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, FL<DH, DE>::BYTES);
  static const char* trace_path = getenv("MHL_TRACE_FB");
  if (trace_path) {
    TraceBuf tb{trace_buffer(s), 0};
    cudaMemcpyToSymbolAsync(g_trace_fb, &tb, sizeof(tb), 0, cudaMemcpyHostToDevice, s);
  }
  static const int dbg = timing_only_switch("MHL_FB_DBG");   // A/B: 1 no dH/gA, 2 no dX stores
  k<<<num_sms, FL<DH, DE>::THREADS, FL<DH, DE>::BYTES, s>>>(w1m, w2m, gxm, gym, hsm, rt, dg, (uint8_t*)dH, (uint8_t*)gA,
                                                           (uint8_t*)dXrep, dbg);
  if (trace_path) {
    TraceBuf tb{nullptr, 0};
    cudaMemcpyToSymbolAsync(g_trace_fb, &tb, sizeof(tb), 0, cudaMemcpyHostToDevice, s);
    trace_dump(trace_path, s);
  }
  return true;
}

}  // namespace

bool expert_bwd_fused_supported(int d_h, int d_e) {
  return (d_h == 256 && d_e == 128) || (d_h == 256 && d_e == 64) || (d_h == 128 && d_e == 128) ||
         (d_h == 128 && d_e == 64);
}

bool launch_expert_bwd_fused_sm100(const Routing& rt, const void* Xs, int64_t ldx, const void* dY, int64_t ldy,
                                   const void* W1, const void* W2, int d_h, int d_e, void* dXrep, float* dg, void* dH,
                                   void* gA, int num_sms, cudaStream_t s) {
#define MHL_FB(A, B) \
  if (d_h == A && d_e == B) return launch_t<A, B>(rt, Xs, ldx, dY, ldy, W1, W2, dXrep, dg, dH, gA, num_sms, s);
  MHL_FB(256, 128) MHL_FB(256, 64) MHL_FB(128, 128) MHL_FB(128, 64)
#undef MHL_FB
  return false;
}

}  // namespace mhl
