// expert_sm100.cu — F5: block-sparse expert FFN forward on tcgen05/TMEM (sm_100a).
//
// The paper's IO-aware expert computation (P:916-P:978) treats the replicas clustered by
// expert (Fig. 2) as queries and expert e's W1_e/W2_e rows as keys/values (Eq. 7):
// y = g * gelu(x W1_e^T) W2_e, with the T x k x d_e hidden activation never written to HBM.
// A tile = 128 clustered rows of one (head, expert) (segments are padded to whole tiles; padding
// rows gather the all-zero sub-token and have gate 0):
//   GEMM1  H[128 x d_e] = X[128 x d_h] W1_e^T   A = sub-tokens gathered (TMA gather4) into
//                                                 K-major SW128 smem chunks; B = W1_e (TMA)
//   epi 1  A = bf16(g * gelu(H)) -> TMEM          (exact-erf GELU, R1; A never touches smem)
//   GEMM2  Y[128 x d_h] = A W2_e                 A read from TMEM; B = W2_e read MN-major
//   epi 2  Yrep rows = bf16(Y)                   TMEM -> registers -> smem -> TMA bulk store
// Warp roles (960 threads): warps 0-7 = producers (TMA gather4 of the sub-tokens through an smem
// ring, W1/W2 by TMA when the expert changes, each as soon as the previous expert's last GEMM
// reading it has completed), warps 8-23 = GELU epilogue (H -> A), warps 24-27 = Y epilogue (Y ->
// Yrep, one warp per TMEM lane quadrant), warp 28 = G1 issuer (+ TMEM owner), warp 29 = G2 issuer.
// TMEM: H [0,128), A double buffer [128,256), Y [256,512) in two 128-column halves.  The epilogue
// groups and the two issuers run concurrently: the GELU of tile i overlaps the Y read-out of tile
// i-1, G2 of tile i's first Y half overlaps the read-out of tile i-1's second half, and G1 never
// waits behind G2's barriers (nor G2 behind G1's gathers).  Persistent CTAs take groups of
// kTileGroup consecutive tiles round-robin (weights reused within a group; the tiles in flight
// stay inside one head, whose sub-tokens then stay L2-resident for their k gathers).
#include <cuda.h>

#include <cstdio>
#include <cstdlib>

#include "kernels.h"
#include "sm100.cuh"
#include "tma_host.h"

namespace mhl {

namespace {

using namespace sm100;

__device__ TraceBuf g_trace_fwd;     // profiling aid (MHL_TRACE_FWD=<file>), off by default

constexpr int BM = kExpertBM;        // 128 rows = MMA M
// Warp roles, warpgroup-aligned so the producers can hand registers to the GELU epilogue (setmaxnreg):
// MHL_F5_PROD_WARPS = 8 (default): producers in pairs, four Y warps; 4: four producer warps own
// whole X chunks and eight Y warps (two per lane quadrant, one per Y column half) read Y out.  The
// Y read-out is per-warp bound (one warp per quadrant moves ~50 B/clk of TMEM; the 16 GELU warps
// read H at ~190 B/clk), and two Y warps per quadrant do shorten it (3.7 k -> 2.5 k cycles per
// tile), but with four producer warps G1 waits 5.8 k instead of 3.9 k cycles for its gathers:
// F5 0.85-0.86 vs 0.77-0.78 ms (tools/ab_f5prod.sh).
#ifndef MHL_F5_PROD_WARPS
#define MHL_F5_PROD_WARPS 8
#endif
constexpr int kProdWarps = MHL_F5_PROD_WARPS;   // warps [0, kProdWarps): producers
constexpr int kOwners = 4;                      // chunk owners: whole warps (4) or warp pairs (8)
constexpr int kWpc = kProdWarps / kOwners;      // producer warps per chunk
constexpr int kGeluWarp0 = kProdWarps;          // 16 GELU warps (4 per lane quadrant, column quarters)
constexpr int kGeluWarps = 16;
constexpr int kYWarp0 = kGeluWarp0 + kGeluWarps;
constexpr int kYWarps = kProdWarps == 4 ? 8 : 4;   // Y epilogue: 1 or 2 per lane quadrant
constexpr int kYGroups = kYWarps / 4;
constexpr int kMmaWarp = kYWarp0 + kYWarps;     // G1 issuer + TMEM owner
constexpr int kMma2Warp = kMmaWarp + 1;         // G2 issuer
constexpr int kThreads = (kMma2Warp + 1) * 32;
static_assert(kThreads == 30 * 32 && (kProdWarps == 4 || kProdWarps == 8), "expert fwd: warp roles");
// Registers: setmaxnreg.inc draws only on registers the CTA's own warps released with
// setmaxnreg.dec (an increase nothing covers blocks forever).  With 30 warps ptxas launches at 64
// registers (sub-partitions 0 and 1 hold eight of them in their 16384-register files); the
// producers' release (and with eight Y warps theirs, to 56) covers the 16 GELU warps' raise to 72,
// pool-wide and on every sub-partition.  Four GELU warps per sub-partition (instead of two with
// twice the columns) hide the MUFU / FMA latency of the GELU chain (3.7 k cycles per tile with
// two, trace r2e).
constexpr int kLaunchRegs = 64, kProdRegs = 40, kGeluRegs = 72, kYRegs = kYWarps == 8 ? 56 : 64;
static_assert(kProdWarps * (kLaunchRegs - kProdRegs) + kYWarps * (kLaunchRegs - kYRegs) >=
                  kGeluWarps * (kGeluRegs - kLaunchRegs),
              "expert fwd: the GELU warps' register increase exceeds the release");
static_assert(kProdWarps / 4 * kProdRegs + 4 * kGeluRegs + kYGroups * kYRegs + kLaunchRegs <= 512,
              "expert fwd: sub-partition 0 register file");
static_assert(8 * 32 * kLaunchRegs <= 16384, "expert fwd: launch register count does not fit sub-partition 0");
constexpr int kGeluThreads = kGeluWarps * 32, kYThreads = kYWarps * 32;
constexpr int kXChunk = BM * 128;    // one 64-column K-chunk of the gathered X tile (16 KB)
constexpr int kYStage = kYWarps * 4096;   // one 4 KB slot (32 rows x 64 columns) per Y warp
// Y staging stages: each Y warp's 4 KB slot is reused once its slab store issued kYStages blocks
// earlier has read it; one stage leaves room for a 5th X ring stage
#ifndef MHL_F5_YSTAGES
#define MHL_F5_YSTAGES 1
#endif
constexpr int kYStages = MHL_F5_YSTAGES;

template <int DH, int DE>
struct FwdL {
  static constexpr int WB = DE * DH * 2;
  static constexpr int W1 = 0, W2 = WB, YS = 2 * WB, X = YS + kYStages * kYStage;
  static constexpr int XS_RAW = (224 * 1024 - X) / kXChunk;
  // chunk c -> stage c % XS, owner c % kOwners; XS >= kOwners keeps the EMPTY parity exact (an
  // owner's previous chunk waited for the in-order consumption of chunk c - kOwners - XS >= c - 2 XS)
  static constexpr int XS = XS_RAW > 6 ? 6 : XS_RAW;   // X ring stages
  static_assert(XS >= kOwners, "X ring too small");
  static constexpr int CTRL = X + XS * kXChunk;
  static constexpr int B_XFULL = CTRL, B_XEMPTY = B_XFULL + 8 * XS;
  static constexpr int B_W1F = B_XEMPTY + 8 * XS, B_W1E = B_W1F + 8, B_W2F = B_W1E + 8, B_W2E = B_W2F + 8;
  static constexpr int B_HFULL = B_W2E + 8, B_HFREE = B_HFULL + 8, B_AFULL = B_HFREE + 8, B_G2DONE = B_AFULL + 16;
  // Y in column halves (DH % 128 == 0): G2 of tile j+1's first half overwrites Y half 0 while the
  // Y warps still read half 1 of tile j, so the read-out (TMEM-read bound) overlaps the next G2
  static constexpr int YH = DH % 128 == 0 ? 2 : 1, YHC = DH / YH;
  static constexpr int B_YFULL = B_G2DONE + 16, B_YEMPTY = B_YFULL + 16;
  static constexpr int TMEMP = B_YEMPTY + 16;
  static constexpr int BYTES = TMEMP + 16;
  static_assert(BYTES <= 227 * 1024, "expert fwd: shared memory over the per-CTA limit");
  // TMEM columns: H [0, DE), A (bf16 pairs, DE/2 columns) x NA buffers, Y [T_Y, T_Y + DH).  At
  // d_e = 256 (the paper's own expert width) only one A buffer fits next to H and Y.
  static constexpr int NA = (DE + 2 * (DE / 2) + DH <= 512) ? 2 : 1;
  static constexpr uint32_t T_H = 0, T_A = DE, T_Y = DE + NA * (DE / 2);
  static_assert(T_Y + DH <= 512, "expert fwd: TMEM over 512 columns");
};

struct Ph {   // mbarrier phase bit
  uint32_t v = 0;
  __device__ uint32_t flip() { uint32_t o = v; v ^= 1u; return o; }
};

__device__ __forceinline__ void tma_store_2d(const void* tmap, uint32_t src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tmap), "r"(src),
               "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_store_2d_hint(const void* tmap, uint32_t src, int c0, int c1, uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;"
               ::"l"(tmap), "r"(src), "r"(c0), "r"(c1), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int DH, int DE>
__global__ void __launch_bounds__(kThreads, 1)
expert_fwd_sm100_kernel(const __grid_constant__ CUtensorMap w1map, const __grid_constant__ CUtensorMap w2map,
                        const __grid_constant__ CUtensorMap ymap, const __grid_constant__ CUtensorMap xmap,
                        Routing rt, int xdbg) {
  using L = FwdL<DH, DE>;
  constexpr int XS = L::XS, KB1 = DH / 64;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0u) __trap();
  const uint32_t sb = smem_u32(smem);
  auto bar = [&](int off) { return reinterpret_cast<uint64_t*>(smem + off); };
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::TMEMP);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // tile window (NEXT-1 windowed combine) or every tile
  const int t_lo = rt.trange ? rt.trange[0] : 0;
  const Tile* tiles = rt.tiles + t_lo;
  const int N_e = rt.N_e;

  if (tid == 0) {
    for (int i = 0; i < XS; ++i) { mbar_init(bar(L::B_XFULL + 8 * i), 1); mbar_init(bar(L::B_XEMPTY + 8 * i), 1); }
    mbar_init(bar(L::B_W1F), 1); mbar_init(bar(L::B_W1E), 1); mbar_init(bar(L::B_W2F), 1); mbar_init(bar(L::B_W2E), 1);
    mbar_init(bar(L::B_HFULL), 1);
    mbar_init(bar(L::B_HFREE), kGeluThreads);
    for (int b = 0; b < 2; ++b) { mbar_init(bar(L::B_AFULL + 8 * b), kGeluThreads); mbar_init(bar(L::B_G2DONE + 8 * b), 1); }
    // a Y half is released by the Y warps that read it: one group per half with two groups and
    // two halves, every Y warp otherwise
    for (int h = 0; h < 2; ++h) {
      mbar_init(bar(L::B_YFULL + 8 * h), 1);
      mbar_init(bar(L::B_YEMPTY + 8 * h), (kYGroups == 2 && L::YH == 2) ? 128 : kYThreads);
    }
    fence_mbar_init();
    tma_prefetch_desc(&w1map); tma_prefetch_desc(&w2map); tma_prefetch_desc(&ymap); tma_prefetch_desc(&xmap);
  }
  if (warp == kMmaWarp) tmem_alloc<512>(s_tmem);
  if (tid == 0) { TraceBuf tb = g_trace_fwd; trace_cta(tb, 60); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  const int nt = (rt.trange ? rt.trange[1] : *rt.ntiles) - t_lo;
  const int ngroups = (nt + kTileGroup - 1) / kTileGroup;
  const int my_groups = ngroups > (int)blockIdx.x ? (ngroups - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  auto tile_at = [&](int i) -> int {   // the i-th tile of this CTA, or -1
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
    for (int kb = 0; kb < KB1; ++kb) tma_load_2d(sb + off + kb * DE * 128, map, kb * 64, (t.head * N_e + t.expert) * DE, full);
  };

  if (warp < kProdWarps) {
    // ================================================================ producers (4 or 8 warps)
    // Chunk c of this CTA's X stream (tile c / KB1, column block c % KB1) goes to ring stage
    // c % XS and is brought by owner c % kOwners (a warp, or a warp pair with 8 producers): each
    // issuing lane brings 4 sub-token rows with one TMA gather4 (warp w of an owner holds tile rows
    // [w*128/kWpc, (w+1)*128/kWpc)).  Warp 0 lane 0 also issues the weight TMAs.
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kProdRegs));
    const int pw = warp;
    constexpr int LPW = 32 / kWpc;   // issuing lanes per warp
    const int owner = pw / kWpc, lrow = (pw % kWpc) * (BM / kWpc) + 4 * (lane % LPW);
    Ph w1e, w2e;
    int cnt = 0;
    int nx[4] = {0, 0, 0, 0};
    {
      const int t0 = tile_at(0);
      if (t0 >= 0) {
        const Tile tl = tiles[t0];
        const int32_t* tk = rt.tok_s + (size_t)tl.head * rt.Rp + tl.row0 + lrow;
        nx[0] = tk[0]; nx[1] = tk[1]; nx[2] = tk[2]; nx[3] = tk[3];
      }
    }
    for (int i = 0;; ++i) {
      const int ti = tile_at(i);
      if (ti < 0) {
        if (pw == 0 && i >= 1 && lane == 0 && !same_expert(tile_at(i - 2), tile_at(i - 1))) {
          mbar_wait(bar(L::B_W2E), w2e.flip() ^ 1);
          load_w(&w2map, L::W2, bar(L::B_W2F), tiles[tile_at(i - 1)]);
        }
        break;
      }
      const Tile tl = tiles[ti];
      const int r0 = nx[0], r1 = nx[1], r2 = nx[2], r3 = nx[3];
      const int tn = tile_at(i + 1);
      if (tn >= 0) {     // next tile's token ids, loaded while this tile's chunks are issued
        const Tile tnl = tiles[tn];
        const int32_t* tk = rt.tok_s + (size_t)tnl.head * rt.Rp + tnl.row0 + lrow;
        nx[0] = tk[0]; nx[1] = tk[1]; nx[2] = tk[2]; nx[3] = tk[3];
      }
      if (pw == 0 && lane == 0 && !same_expert(tile_at(i - 1), ti)) {
        mbar_wait(bar(L::B_W1E), w1e.flip() ^ 1);
        load_w(&w1map, L::W1, bar(L::B_W1F), tl);
      }
      __syncwarp();
      for (int kb = 0; kb < KB1; ++kb, ++cnt) {
        if (cnt % kOwners != owner) continue;
        const int xs = cnt % XS;
        uint64_t* full = bar(L::B_XFULL + 8 * xs);
        if (lane == 0) {
          mbar_wait(bar(L::B_XEMPTY + 8 * xs), ((cnt / XS) & 1) ^ 1);
          if (pw % kWpc == 0) {
            if (xdbg & 2) mbar_arrive(full);   // A/B only: no gathers (garbage X)
            else mbar_expect_tx(full, kXChunk);
          }
        }
        __syncwarp();
        if (lane < LPW && !(xdbg & 2)) {
          if (xdbg & 1) {   // A/B only: the same gather4 stream over consecutive rows
            const int c0 = (int)((tl.row0 + lrow) % rt.T);
            tma_gather4(sb + L::X + xs * kXChunk + lrow * 128, &xmap, (int)tl.head * DH + kb * 64, c0,
                        (c0 + 1) % (int)rt.T, (c0 + 2) % (int)rt.T, (c0 + 3) % (int)rt.T, full);
          } else {
            tma_gather4(sb + L::X + xs * kXChunk + lrow * 128, &xmap, (int)tl.head * DH + kb * 64, r0, r1, r2, r3,
                        full);
          }
        }
      }
      // W2 of the previous tile if it started a new expert run (read by G2(i-1), issued after G1(i))
      if (pw == 0 && lane == 0 && i >= 1 && !same_expert(tile_at(i - 2), tile_at(i - 1))) {
        mbar_wait(bar(L::B_W2E), w2e.flip() ^ 1);
        load_w(&w2map, L::W2, bar(L::B_W2F), tiles[tile_at(i - 1)]);
      }
    }
  } else if (warp == kMmaWarp) {
    // ================================================================ G1 issuer
    // Two issuing threads: G1 (this warp) waits for gathered chunks, G2 (warp kMma2Warp) for the
    // GELU's A and the Y read-out; in one thread each waited behind the other's barriers (a G2
    // behind the next tile's gathers, a G1 behind the Y read-out).  They touch disjoint TMEM
    // columns and smem operands; every cross dependency goes through an mbarrier.
    if (lane == 0) {
      constexpr uint32_t ID1 = idesc_bf16(BM, DE, 0, 0);
      Ph xf[12], w1f, hfr;
      int xs = 0;
      for (int i = 0;; ++i) {
        const int ti = tile_at(i);
        if (ti < 0) break;
        if (!same_expert(tile_at(i - 1), ti)) mbar_wait(bar(L::B_W1F), w1f.flip());
        if (i >= 1) mbar_wait(bar(L::B_HFREE), hfr.flip());   // epilogue has read H of tile i-1
        trace_ev(g_trace_fwd, 10, i);
        tc_fence_after();
        for (int kb = 0; kb < KB1; ++kb) {
          mbar_wait(bar(L::B_XFULL + 8 * xs), xf[xs].flip());
          trace_ev(g_trace_fwd, 11, i * 16 + kb);
          tc_fence_after();
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            mma_bf16(tmem + L::T_H, sdesc_sw128(sb + L::X + xs * kXChunk + ks * 32, 16, 1024),
                     sdesc_sw128(sb + L::W1 + kb * DE * 128 + ks * 32, 16, 1024), ID1, (kb | ks) ? 1u : 0u);
          mma_commit(bar(L::B_XEMPTY + 8 * xs));
          if (++xs == XS) xs = 0;
        }
        mma_commit(bar(L::B_HFULL));
        if (!same_expert(ti, tile_at(i + 1))) mma_commit(bar(L::B_W1E));
      }
    }
  } else if (warp == kMma2Warp) {
    // ================================================================ G2 issuer
    if (lane == 0) {
      constexpr uint32_t ID2 = idesc_bf16(BM, L::YHC, 0, 1);
      Ph w2f, af[2], ye[2];
      for (int j = 0;; ++j) {
        const int tj = tile_at(j);
        if (tj < 0) break;
        const int b = j % L::NA;
        if (!same_expert(tile_at(j - 1), tj)) mbar_wait(bar(L::B_W2F), w2f.flip());
        mbar_wait(bar(L::B_AFULL + 8 * b), af[b].flip());   // (NA = 1: b = 0 throughout)
#pragma unroll
        for (int hh = 0; hh < L::YH; ++hh) {
          mbar_wait(bar(L::B_YEMPTY + 8 * hh), ye[hh].flip() ^ 1);   // the Y warps read this half of Y(j-1)
          if (hh == 0) trace_ev(g_trace_fwd, 13, j);
          tc_fence_after();
          // B = W2_e's columns [hh*YHC, (hh+1)*YHC): MN-major 64-column atoms at DE*128 bytes
#pragma unroll
          for (int ks = 0; ks < DE / 16; ++ks)
            mma_bf16_ts(tmem + L::T_Y + hh * L::YHC, tmem + L::T_A + b * (DE / 2) + ks * 8,
                        sdesc_sw128(sb + L::W2 + hh * (L::YHC / 64) * DE * 128 + ks * 2 * 1024, DE * 128, 1024), ID2,
                        ks > 0);
          mma_commit(bar(L::B_YFULL + 8 * hh));
        }
        mma_commit(bar(L::B_G2DONE + 8 * b));
        trace_ev(g_trace_fwd, 14, j);
        if (!same_expert(tj, tile_at(j + 1))) mma_commit(bar(L::B_W2E));
      }
    }
  } else if (warp >= kGeluWarp0 && warp < kYWarp0) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kGeluRegs));
    // ================================================================ GELU epilogue (8 warps)
    // tile i: H (this warp's quadrant rows, DE/2 columns) -> registers, release H, A = bf16(g *
    // gelu(H)) -> TMEM A buffer i % NA once G2(i - NA) has read that buffer.
    const int q = warp & 3, sl = (warp - kGeluWarp0) >> 2;   // lane quadrant, column quarter
    const int row = q * 32 + lane;
    const int et = tid - kGeluWarp0 * 32;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    Ph hf, gd[2];
    // this row's gate, fetched one tile ahead (its L2 latency would sit at the top of every tile)
    float g_n = 0.f;
    auto fetch = [&](int t) {
      if (t < 0) return;
      const Tile u = tiles[t];
      g_n = __ldg(rt.gate_s + (size_t)u.head * rt.Rp + u.row0 + row);
    };
    fetch(tile_at(0));
    constexpr int NC = DE / 4;               // H columns of this warp
    constexpr int CW = NC < 32 ? NC : 32;    // columns per TMEM load
    auto ld = [&](uint32_t addr, uint32_t* v) {
      if constexpr (CW == 32) tmem_ld32(addr, *reinterpret_cast<uint32_t(*)[32]>(v));
      else tmem_ld16(addr, *reinterpret_cast<uint32_t(*)[16]>(v));
    };
    auto st = [&](uint32_t addr, const uint32_t* w) {
      if constexpr (CW == 32) tmem_st16(addr, *reinterpret_cast<const uint32_t(*)[16]>(w));
      else tmem_st8(addr, *reinterpret_cast<const uint32_t(*)[8]>(w));
    };
    for (int i = 0;; ++i) {
      const int ti = tile_at(i);
      if (ti < 0) break;
      const int b = i % L::NA;
      const float hg = 0.5f * g_n;
      fetch(tile_at(i + 1));
      mbar_wait_warp(bar(L::B_HFULL), hf.flip());
      if (et == 0) trace_ev(g_trace_fwd, 20, i);
      tc_fence_after();
      if constexpr (L::NA == 1) {
        // single A buffer: G2(i-1) must have read it; stream H CW columns at a time, release H after
        // the last load
        if (i >= 1) { mbar_wait_warp(bar(L::B_G2DONE), gd[0].flip()); tc_fence_after(); }
#pragma unroll 1
        for (int c = 0; c < NC; c += CW) {
          uint32_t v[CW], w[CW / 2];
          ld(tmem + L::T_H + lane_off + sl * NC + c, v);
          tmem_ld_wait();
          if (c + CW >= NC) { tc_fence_before(); mbar_arrive(bar(L::B_HFREE)); }
#pragma unroll
          for (int u = 0; u < CW; u += 2) {
            const float2 a = gelu2_scaled(make_float2(__uint_as_float(v[u]), __uint_as_float(v[u + 1])), hg);
            w[u / 2] = pack_bf16x2(a.x, a.y);
          }
          st(tmem + L::T_A + lane_off + sl * (NC / 2) + c / 2, w);
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(bar(L::B_AFULL));
        continue;
      }
      uint32_t hv[NC];
#pragma unroll
      for (int c = 0; c < NC; c += CW) ld(tmem + L::T_H + lane_off + sl * NC + c, hv + c);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(bar(L::B_HFREE));
      if (et == 0) trace_ev(g_trace_fwd, 21, i);
      uint32_t pa[NC / 2];
#pragma unroll
      for (int u = 0; u < NC; u += 2) {
        const float2 a = gelu2_scaled(make_float2(__uint_as_float(hv[u]), __uint_as_float(hv[u + 1])), hg);
        pa[u / 2] = pack_bf16x2(a.x, a.y);
      }
      // A buffer b was last read by G2(i - 2)
      if (i >= L::NA) { mbar_wait_warp(bar(L::B_G2DONE + 8 * b), gd[b].flip()); tc_fence_after(); }
#pragma unroll
      for (int c = 0; c < NC / 2; c += CW / 2) st(tmem + L::T_A + b * (DE / 2) + lane_off + sl * (NC / 2) + c, pa + c);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(bar(L::B_AFULL + 8 * b));
      if (et == 0) trace_ev(g_trace_fwd, 22, i);
    }
  } else if (warp >= kYWarp0 && warp < kMmaWarp) {
    if constexpr (kYRegs < kLaunchRegs) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kYRegs));
    // ================================================================ Y epilogue (kYWarps warps)
    // tile j: Y rows of this warp's lane quadrant (32 rows) -> bf16 -> SW128 smem slot (64-column
    // blocks) -> TMA bulk store of the 32-row slab.  With two warps per quadrant, group g reads Y
    // half g (or the blocks of its parity when Y is one half); each half is released to G2 by the
    // warps that read it, after their last TMEM load of it.
    const int q = warp & 3, yg = (warp - kYWarp0) >> 2;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    constexpr int NB = DH / 64, BPH = L::YHC / 64;   // 64-column blocks: per tile, per Y half
    auto mine = [&](int cb) { return kYGroups == 1 ? true : (L::YH == 2 ? cb / BPH == yg : cb % 2 == yg); };
    Ph yf[2];
    int ys = 0;   // running count of Y blocks stored by this warp (selects the smem stage)
    const uint32_t slot = (uint32_t)(warp - kYWarp0) * 4096;
    for (int j = 0;; ++j) {
      const int tj = tile_at(j);
      if (tj < 0) break;
      const Tile tl = tiles[tj];
#pragma unroll 1
      for (int cb = 0; cb < NB; ++cb) {
        if (!mine(cb)) continue;
        const int hh = cb / BPH;
        int first = hh * BPH, last = hh * BPH + BPH - 1;   // this warp's first / last block of half hh
        while (!mine(first)) ++first;
        while (!mine(last)) --last;
        if (cb == first) {          // wait for this Y half's G2
          mbar_wait_warp(bar(L::B_YFULL + 8 * hh), yf[hh].flip());
          if (q == 0 && lane == 0 && hh == 0) trace_ev(g_trace_fwd, 23, j);
          tc_fence_after();
        }
        const int st = ys % kYStages;
        ++ys;
        // the slab store issued from this stage kYStages blocks ago must have read the slot
        if (lane == 0) bulk_wait_read<kYStages - 1>();
        __syncwarp();
        uint8_t* sp = smem + L::YS + st * kYStage + slot;
#pragma unroll
        for (int hc = 0; hc < 2; ++hc) {      // two 32-column loads, each packed and staged at once
          uint32_t v[32], w[16];
          tmem_ld32(tmem + L::T_Y + lane_off + cb * 64 + hc * 32, v);
          tmem_ld_wait();
          if (hc == 1 && cb == last) {   // this warp's last read of the half: release it
            tc_fence_before();
            mbar_arrive(bar(L::B_YEMPTY + 8 * hh));
            if (q == 0 && lane == 0 && hh == L::YH - 1 && yg == kYGroups - 1) trace_ev(g_trace_fwd, 24, j);
          }
#pragma unroll
          for (int u = 0; u < 16; ++u) w[u] = pack_bf16x2(__uint_as_float(v[2 * u]), __uint_as_float(v[2 * u + 1]));
#pragma unroll
          for (int u = 0; u < 16; u += 4)
            *reinterpret_cast<uint4*>(sp + kmaj_off(lane, hc * 32 + 2 * u, 32)) = make_uint4(w[u], w[u + 1], w[u + 2], w[u + 3]);
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&ymap, sb + L::YS + st * kYStage + slot, cb * 64, (int)((size_t)tl.head * rt.Rp + tl.row0 + q * 32));
          bulk_commit();
        }
      }
    }
    if (lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (tid == 0) { TraceBuf tb = g_trace_fwd; trace_cta(tb, 61); }
  if (warp == kMmaWarp) tmem_dealloc<512>(tmem);
}

template <int DH, int DE>
bool launch_t(const Routing& rt, const void* Xs, int64_t ldx, const void* W1, const void* W2, void* Yrep, int num_sms,
              cudaStream_t s) {
  CUtensorMap w1m, w2m, ym, xm;
  // sub-token gather map: T+1 rows (row T all-zero), box = 64 columns x 1 row (TMA gather4)
  if (!make_tmap_2d_bf16(&xm, Xs, (uint64_t)rt.T + 1, (uint64_t)rt.H * DH, (uint64_t)ldx * 2, 1, 64)) return false;
  if (!make_tmap_2d_bf16(&w1m, W1, (uint64_t)rt.H * rt.N_e * DE, DH, (uint64_t)DH * 2, DE, 64)) return false;
  if (!make_tmap_2d_bf16(&w2m, W2, (uint64_t)rt.H * rt.N_e * DE, DH, (uint64_t)DH * 2, DE, 64)) return false;
  if (!make_tmap_2d_bf16(&ym, Yrep, (uint64_t)rt.H * rt.Rp, DH, (uint64_t)DH * 2, 32, 64)) return false;
  auto kern = expert_fwd_sm100_kernel<DH, DE>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdL<DH, DE>::BYTES);
  static const char* trace_path = getenv("MHL_TRACE_FWD");
  static unsigned long long* tbuf = nullptr;
  const size_t nslot = 64 * 4096;   // events < 64 (60 / 61: per-CTA start / end)
  if (trace_path) {
    if (!tbuf) cudaMalloc(&tbuf, nslot * sizeof(unsigned long long));
    cudaMemsetAsync(tbuf, 0, nslot * sizeof(unsigned long long), s);
    TraceBuf tb{tbuf, 0};
    cudaMemcpyToSymbolAsync(g_trace_fwd, &tb, sizeof(tb), 0, cudaMemcpyHostToDevice, s);
  }
  static const int xdbg = timing_only_switch("MHL_F5_XDBG");   // A/B only (wrong results)
  kern<<<num_sms, kThreads, FwdL<DH, DE>::BYTES, s>>>(w1m, w2m, ym, xm, rt, xdbg);
  if (trace_path) {
    TraceBuf tb{nullptr, 0};
    cudaMemcpyToSymbolAsync(g_trace_fwd, &tb, sizeof(tb), 0, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
    unsigned long long* h = (unsigned long long*)malloc(nslot * sizeof(unsigned long long));
    cudaMemcpy(h, tbuf, nslot * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    FILE* f = fopen(trace_path, "w");
    if (f) {
      for (size_t u = 0; u < nslot; ++u)
        if (h[u]) fprintf(f, "%zu %zu %llu\n", u / 4096, u % 4096, h[u]);
      fclose(f);
    }
    free(h);
  }
  return true;
}

}  // namespace

bool expert_fwd_sm100_supported(int d_h, int d_e) {
  return (d_h == 256 && d_e == 128) || (d_h == 192 && d_e == 64) || (d_h == 256 && d_e == 64) ||
         (d_h == 128 && d_e == 128) || (d_h == 128 && d_e == 64) || (d_h == 64 && d_e == 64) ||
         (d_h == 128 && d_e == 256);
}

bool launch_expert_fwd_sm100(const Routing& rt, const void* Xs, int64_t ldx, const void* W1, const void* W2, int d_h,
                             int d_e, void* Yrep, int num_sms, cudaStream_t s) {
#define MHL_F(A, B) \
  if (d_h == A && d_e == B) return launch_t<A, B>(rt, Xs, ldx, W1, W2, Yrep, num_sms, s);
  MHL_F(256, 128) MHL_F(256, 64) MHL_F(192, 64) MHL_F(128, 128) MHL_F(128, 64) MHL_F(64, 64) MHL_F(128, 256)
#undef MHL_F
  return false;
}

}  // namespace mhl
