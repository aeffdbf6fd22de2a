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
// Warp roles (416 threads): warps 0-3 = producers (TMA gather4 of the sub-tokens through an smem
// ring, W1/W2 by TMA when the expert changes, each as soon as the previous expert's last GEMM reading it has
// completed), warp 4 = MMA issuer (+ TMEM owner), warps 5-12 = epilogue.  TMEM: H [0,128),
// A double buffer [128,256), Y [256,512): the MMA order G1(i), G2(i-1), G1(i+1), ... keeps the
// tensor pipe busy while the epilogue of neighbouring tiles runs.  Persistent CTAs take groups of
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
// Warp roles, warpgroup-aligned so the producers can hand registers to the epilogue (setmaxnreg):
constexpr int kProdWarps = 8;         // warps 0-7: producers, in 4 pairs (a pair fills one X chunk)
constexpr int kOwners = kProdWarps / 2;
constexpr int kEpiWarp0 = 8;          // warps 8-15: epilogue
constexpr int kMmaWarp = 16;          // warp 16: MMA issuer + TMEM owner
constexpr int kCombWarp0 = 17;        // warps 17-19: fused combine (FwdCombine), idle without it
constexpr int kThreads = 20 * 32;
constexpr int kProdRegs = 40, kEpiRegs = 152;   // launch cap 96: 8*32*(96-40) >= 8*32*(152-96)
constexpr int kEpiThreads = 256;
constexpr int kXChunk = BM * 128;    // one 64-column K-chunk of the gathered X tile (16 KB)
constexpr int kYStage = BM * 128;    // one 64-column block of the Y tile (16 KB)

// Y store path: 0 = smem staging + TMA bulk stores, 2 = straight from registers (32-byte
// st.global.v8 per lane, no staging smem, so the X ring can take its 32 KB).  X ring depth cap.
#ifndef MHL_F5_YSTORE
#define MHL_F5_YSTORE 0
#endif
#ifndef MHL_F5_XS
#define MHL_F5_XS 4
#endif
#define L_YDIRECT (MHL_F5_YSTORE == 2)

template <int DH, int DE>
struct FwdL {
  static constexpr int WB = DE * DH * 2;
  static constexpr bool YDIRECT = MHL_F5_YSTORE == 2;
  static constexpr int W1 = 0, W2 = WB, YS = 2 * WB, X = YS + (YDIRECT ? 0 : 2 * kYStage);
  static constexpr int XS_RAW = (224 * 1024 - X) / kXChunk;
  // chunk c -> stage c % XS, pair c % kOwners; XS >= kOwners keeps the EMPTY parity exact (a
  // pair's previous chunk waited for the in-order consumption of chunk c - kOwners - XS >= c - 2 XS)
  static constexpr int XS = XS_RAW > MHL_F5_XS ? MHL_F5_XS : XS_RAW;   // X ring stages
  static_assert(XS >= kOwners, "X ring too small");
  static constexpr int CTRL = X + XS * kXChunk;
  static constexpr int B_XFULL = CTRL, B_XEMPTY = B_XFULL + 8 * XS;
  static constexpr int B_W1F = B_XEMPTY + 8 * XS, B_W1E = B_W1F + 8, B_W2F = B_W1E + 8, B_W2E = B_W2F + 8;
  static constexpr int B_HFULL = B_W2E + 8, B_HFREE = B_HFULL + 8, B_AFULL = B_HFREE + 8, B_G2DONE = B_AFULL + 16;
  static constexpr int B_YEMPTY = B_G2DONE + 16;
  static constexpr int TMEMP = B_YEMPTY + 8;
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
// L2 policies of the forward kernel (MHL_F5_L2HINT: 0 none (default), 1 both, 2 stores only; 1 and 2
// measured F5 0.87 -> 0.92-0.93 ms):
// sub-token rows gathered evict_last (each is
// re-read by its other top-k experts), Y tiles stored evict_first (streamed out once)
#ifndef MHL_F5_L2HINT
#define MHL_F5_L2HINT 0
#endif
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int DH, int DE>
__global__ void __launch_bounds__(kThreads, 1)
expert_fwd_sm100_kernel(const __grid_constant__ CUtensorMap w1map, const __grid_constant__ CUtensorMap w2map,
                        const __grid_constant__ CUtensorMap ymap, const __grid_constant__ CUtensorMap xmap,
                        Routing rt, uint8_t* __restrict__ yout, int lsu, FwdCombine fc) {
  using L = FwdL<DH, DE>;
  constexpr int XS = L::XS, KB1 = DH / 64;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0u) __trap();
  const uint32_t sb = smem_u32(smem);
  auto bar = [&](int off) { return reinterpret_cast<uint64_t*>(smem + off); };
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::TMEMP);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const Tile* tiles = rt.tiles;
  const int N_e = rt.N_e;

  if (tid == 0) {
    for (int i = 0; i < XS; ++i) { mbar_init(bar(L::B_XFULL + 8 * i), 1); mbar_init(bar(L::B_XEMPTY + 8 * i), 1); }
    mbar_init(bar(L::B_W1F), 1); mbar_init(bar(L::B_W1E), 1); mbar_init(bar(L::B_W2F), 1); mbar_init(bar(L::B_W2E), 1);
    mbar_init(bar(L::B_HFULL), 1);
    mbar_init(bar(L::B_HFREE), kEpiThreads);
    for (int b = 0; b < 2; ++b) { mbar_init(bar(L::B_AFULL + 8 * b), kEpiThreads); mbar_init(bar(L::B_G2DONE + 8 * b), 1); }
    mbar_init(bar(L::B_YEMPTY), kEpiThreads);
    fence_mbar_init();
    tma_prefetch_desc(&w1map); tma_prefetch_desc(&w2map); tma_prefetch_desc(&ymap); tma_prefetch_desc(&xmap);
  }
  if (warp == kMmaWarp) tmem_alloc<512>(s_tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  const int nt = *rt.ntiles;
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
    // ================================================================ producers (8 warps)
    // Chunk c of this CTA's X stream (tile c / KB1, column block c % KB1) goes to ring stage
    // c % XS and is brought by warp pair c % kOwners (XS is a multiple of kOwners, so a stage is
    // only ever refilled by the pair that filled it before): lanes 0-15 of each warp of the pair
    // issue one TMA gather4 of 4 sub-token rows each (warp 2p+h owns tile rows 64h..64h+63).  More
    // warps issuing gathers raise the SM's gather rate (tools/ring_probe.cu mech 6).  Warp 0 lane 0
    // also issues the weight TMAs.
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kProdRegs));
    const int pw = warp;
    const int owner = pw >> 1, lrow = (pw & 1) * 64 + 4 * (lane & 15);
    const uint64_t pol_keep = l2_evict_last();
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
          if ((pw & 1) == 0) mbar_expect_tx(full, kXChunk);
        }
        __syncwarp();
        if (lane < 16)
          if (MHL_F5_L2HINT == 1)
            tma_gather4_hint(sb + L::X + xs * kXChunk + lrow * 128, &xmap, (int)tl.head * DH + kb * 64, r0, r1, r2,
                             r3, full, pol_keep);
          else
          tma_gather4(sb + L::X + xs * kXChunk + lrow * 128, &xmap, (int)tl.head * DH + kb * 64, r0, r1, r2, r3,
                      full);
      }
      // W2 of the previous tile if it started a new expert run (read by G2(i-1), issued after G1(i))
      if (pw == 0 && lane == 0 && i >= 1 && !same_expert(tile_at(i - 2), tile_at(i - 1))) {
        mbar_wait(bar(L::B_W2E), w2e.flip() ^ 1);
        load_w(&w2map, L::W2, bar(L::B_W2F), tiles[tile_at(i - 1)]);
      }
    }
  } else if (warp == kMmaWarp) {
    // ================================================================ MMA issuer
    if (lane == 0) {
      constexpr uint32_t ID1 = idesc_bf16(BM, DE, 0, 0);
      constexpr uint32_t ID2 = idesc_bf16(BM, DH, 0, 1);
      Ph xf[12], w1f, w2f, hfr, af[2], ye;
      int xs = 0;
      auto gemm2 = [&](int j) {
        const int b = j % L::NA;
        const int tj = tile_at(j);
        if (!same_expert(tile_at(j - 1), tj)) mbar_wait(bar(L::B_W2F), w2f.flip());
        mbar_wait(bar(L::B_AFULL + 8 * b), af[b].flip());   // (NA = 1: b = 0 throughout)
        mbar_wait(bar(L::B_YEMPTY), ye.flip() ^ 1);
        trace_ev(g_trace_fwd, 13, j);
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < DE / 16; ++ks)
          mma_bf16_ts(tmem + L::T_Y, tmem + L::T_A + b * (DE / 2) + ks * 8,
                      sdesc_sw128(sb + L::W2 + ks * 2 * 1024, DE * 128, 1024), ID2, ks > 0);
        mma_commit(bar(L::B_G2DONE + 8 * b));
        trace_ev(g_trace_fwd, 14, j);
        if (!same_expert(tj, tile_at(j + 1))) mma_commit(bar(L::B_W2E));
      };
      int i = 0;
      for (;; ++i) {
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
        if (i >= 1) gemm2(i - 1);
      }
      if (i >= 1) gemm2(i - 1);
    }
  } else if (warp >= kEpiWarp0 && warp < kMmaWarp) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kEpiRegs));
    // ================================================================ epilogue (8 warps)
    const int q = warp & 3, half = (warp - kEpiWarp0) >> 2;   // lane quadrant, column half
    const int row = q * 32 + lane;
    const int et = tid - kEpiWarp0 * 32;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    Ph hf, gd[2];
    int ys = 0;   // running count of Y blocks stored (selects the smem stage)
    const uint64_t pol_stream = l2_evict_first();
    auto signal = [&](int t) {
      if (t < 0) return;
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __threadfence();
      atomicAdd(fc.wdone + fc.tilewin[t], 1);
    };
    auto epi2 = [&](int j, bool waited) {
      const int b = j % L::NA;
      const Tile tl = tiles[tile_at(j)];
      if (!waited) mbar_wait_warp(bar(L::B_G2DONE + 8 * b), gd[b].flip());
      if (et == 0) trace_ev(g_trace_fwd, 23, j);
      tc_fence_after();
      // 64-column blocks: TMEM -> regs -> bf16 -> smem stage (SW128) -> TMA bulk store.  The two
      // warps of a lane quadrant own a 32-row slab and synchronise only with each other.
      const bool leader = (half == 0 && lane == 0);
      if constexpr (L::YDIRECT) {
        // this thread's row, 32 columns per block: 2 x 32-byte stores (whole sectors), evict-first
        uint8_t* yrow = yout + ((size_t)tl.head * rt.Rp + tl.row0 + row) * (DH * 2) + half * 64;
        const uint64_t pol = l2_evict_first();
#pragma unroll 1
        for (int cb = 0; cb < DH / 64; ++cb) {
          uint32_t v[32];
          tmem_ld32(tmem + L::T_Y + lane_off + cb * 64 + half * 32, v);
          tmem_ld_wait();
          if (cb == DH / 64 - 1) {
            tc_fence_before();
            mbar_arrive(bar(L::B_YEMPTY));
            if (et == 0) trace_ev(g_trace_fwd, 24, j);
          }
          uint32_t w[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) w[u] = pack_bf16x2(__uint_as_float(v[2 * u]), __uint_as_float(v[2 * u + 1]));
          st_global_v8_hint(yrow + cb * 128, w[0], w[1], w[2], w[3], w[4], w[5], w[6], w[7], pol);
          st_global_v8_hint(yrow + cb * 128 + 32, w[8], w[9], w[10], w[11], w[12], w[13], w[14], w[15], pol);
        }
        return;
      }
#pragma unroll 1
      for (int cb = 0; cb < DH / 64; ++cb, ++ys) {
        const int st = ys & 1;
        uint32_t v[32];
        tmem_ld32(tmem + L::T_Y + lane_off + cb * 64 + half * 32, v);
        tmem_ld_wait();
        if (cb == DH / 64 - 1) {
          tc_fence_before();
          mbar_arrive(bar(L::B_YEMPTY));
          if (et == 0) trace_ev(g_trace_fwd, 24, j);
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
        if (lsu) {
          // coalesced 16-byte stores by the quadrant's two warps (8 lanes per 128-byte row segment):
          // the TMA unit stays with the gathers
          named_bar_sync(2 + q, 64);
          const int bt = half * 32 + lane;
          uint8_t* dst = yout + ((size_t)tl.head * rt.Rp + tl.row0 + q * 32) * (DH * 2) + cb * 128;
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
            if (MHL_F5_L2HINT)
              tma_store_2d_hint(&ymap, sb + L::YS + st * kYStage + q * 4096, cb * 64,
                                (int)((size_t)tl.head * rt.Rp + tl.row0 + q * 32), pol_stream);
            else
            tma_store_2d(&ymap, sb + L::YS + st * kYStage + q * 4096, cb * 64,
                         (int)((size_t)tl.head * rt.Rp + tl.row0 + q * 32));
            bulk_commit();
          }
        }
      }
      // fused combine: once the previous tile's slab stores have completed (all bulk groups but this
      // tile's DH/64), publish them to the combine warps of every CTA
      if (fc.out && leader && !lsu) {
        asm volatile("cp.async.bulk.wait_group %0;" ::"n"(DH / 64) : "memory");
        if (j >= 1) signal(tile_at(j - 1));
      }
    };
    // (the fused combine's completion signal of one tile's 32-row slab: async-proxy writes complete,
    // then made visible to other CTAs' generic loads before the counter is released)
    (void)0;
    // this row's gate, fetched one tile ahead (its L2 latency would sit at the top of every tile)
    float g_n = 0.f;
    auto fetch = [&](int t) {
      if (t < 0) return;
      const Tile u = tiles[t];
      g_n = __ldg(rt.gate_s + (size_t)u.head * rt.Rp + u.row0 + row);
    };
    fetch(tile_at(0));
    int i = 0;
    for (;; ++i) {
      const int ti = tile_at(i);
      if (ti < 0) break;
      const int b = i % L::NA;
      const float g = g_n;
      fetch(tile_at(i + 1));
      mbar_wait_warp(bar(L::B_HFULL), hf.flip());
      if (et == 0) trace_ev(g_trace_fwd, 20, i);
      tc_fence_after();
      constexpr int NC = DE / 2;
      if constexpr (L::NA == 1) {
        // single A buffer: G2(i-1) must have read it; stream H 32 columns at a time (NC = 128 values
        // would not fit in registers), release H after the last load
        if (i >= 1) { mbar_wait_warp(bar(L::B_G2DONE), gd[0].flip()); tc_fence_after(); }
#pragma unroll 1
        for (int c = 0; c < NC; c += 32) {
          uint32_t v[32], w[16];
          tmem_ld32(tmem + L::T_H + lane_off + half * NC + c, v);
          tmem_ld_wait();
          if (c + 32 >= NC) { tc_fence_before(); mbar_arrive(bar(L::B_HFREE)); }
#pragma unroll
          for (int u = 0; u < 32; u += 2) {
            const float2 a = __fmul2_rn(gelu2(make_float2(__uint_as_float(v[u]), __uint_as_float(v[u + 1])), nullptr),
                                        make_float2(g, g));
            w[u / 2] = pack_bf16x2(a.x, a.y);
          }
          tmem_st16(tmem + L::T_A + lane_off + half * (NC / 2) + c / 2, w);
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(bar(L::B_AFULL));
        if (i >= 1) epi2(i - 1, true);
        continue;
      }
      // epi 1: this warp's DE/2 columns of H -> registers, release H, GELU, A -> TMEM buffer b
      uint32_t hv[NC];
#pragma unroll
      for (int c = 0; c < NC; c += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + L::T_H + lane_off + half * NC + c, v);
#pragma unroll
        for (int u = 0; u < 32; ++u) hv[c + u] = v[u];
      }
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(bar(L::B_HFREE));
      if (et == 0) trace_ev(g_trace_fwd, 21, i);
      uint32_t pa[NC / 2];
#pragma unroll
      for (int u = 0; u < NC; u += 2) {
        const float2 a = __fmul2_rn(gelu2(make_float2(__uint_as_float(hv[u]), __uint_as_float(hv[u + 1])), nullptr),
                                    make_float2(g, g));
        pa[u / 2] = pack_bf16x2(a.x, a.y);
      }
#pragma unroll
      for (int c = 0; c < NC / 2; c += 16) {
        uint32_t w[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) w[u] = pa[c + u];
        tmem_st16(tmem + L::T_A + b * (DE / 2) + lane_off + half * (NC / 2) + c, w);
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(bar(L::B_AFULL + 8 * b));
      if (et == 0) trace_ev(g_trace_fwd, 22, i);
      if (i >= 1) epi2(i - 1, false);
    }
    if (i >= 1) epi2(i - 1, false);
    if (half == 0 && lane == 0) bulk_wait_all();
    if (fc.out && half == 0 && lane == 0 && !lsu && i >= 1) signal(tile_at(i - 1));
  } else if (warp >= kCombWarp0 && fc.out) {
    // ================================================================ fused combine (3 warps)
    // Windows (head h, part p) in order: wait until every tile of the window has been stored by all
    // CTAs (4 slab signals per tile), then combine this CTA's slice of the window's tokens
    // [wtok[h][p-1], wtok[h][p]): y[t][h*d_h + c] = sum_j Yrep[h][pos(t,j)][c] in j order, fp32,
    // rounded once — the arithmetic of combine_kernel (bit-identical).  The window's Yrep rows were
    // written moments ago and are read back from L2.  All CTAs are co-resident (one per SM), so the
    // spin cannot deadlock; a bounded spin traps instead of hanging on a bookkeeping error.
    const int cw = warp - kCombWarp0, NCW = kThreads / 32 - kCombWarp0;
    const int nwin = rt.H * kTileParts;
    const int64_t R = rt.T * rt.k;
    for (int w = 0; w < nwin; ++w) {
      const int h = w / kTileParts, p = w % kTileParts;
      if (lane == 0) {
        const int need = 4 * fc.wtiles[w];
        long long spins = 0;
        while (true) {
          int v;
          asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(fc.wdone + w) : "memory");
          if (v >= need) break;
          __nanosleep(100);
          if (++spins > (1ll << 24)) {
            printf("[mhl fused combine] CTA %d warp %d: window %d stuck at %d of %d tile-slab signals\n",
                   (int)blockIdx.x, warp, w, v, need);
            __trap();
          }
        }
      }
      __syncwarp();
      const int lo = p == 0 ? 0 : fc.wtok[w - 1], hi = fc.wtok[w];
      const int n = hi - lo;
      const int b0 = lo + (int)((int64_t)n * blockIdx.x / gridDim.x), b1 = lo + (int)((int64_t)n * (blockIdx.x + 1) / gridDim.x);
      const bf16* rep = reinterpret_cast<const bf16*>(yout) + (size_t)h * rt.Rp * DH;
      // two tokens per warp iteration (16 lanes x 32-byte loads per token row when d_h = 256) for
      // twice the loads in flight; every lane takes part in the position broadcasts
      for (int t0 = b0 + 2 * cw; t0 < b1; t0 += 2 * NCW) {
        const int sub = lane >> 4, l16 = lane & 15;            // token t0 + sub, lane l16 of its half-warp
        const int t = t0 + sub;
        const bool tok = t < b1;
        const int64_t rb = (size_t)h * R + (int64_t)t * rt.k;
        const int my_pos = (tok && l16 < rt.k) ? rt.pos[rb + l16] : 0;
        int pj[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) pj[j] = __shfl_sync(0xffffffffu, my_pos, (lane & 16) | j);
        if (tok) {
          for (int ch = l16; ch < DH / 8; ch += 16) {
            float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int j0 = 0; j0 < 16; j0 += 8) {
              if (j0 >= rt.k) break;
              uint4 v[8];
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (j0 + j < rt.k) v[j] = __ldcg(reinterpret_cast<const uint4*>(rep + (size_t)pj[j0 + j] * DH + ch * 8));
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                if (j0 + j < rt.k) {
                  const __nv_bfloat162* pv = reinterpret_cast<const __nv_bfloat162*>(&v[j]);
#pragma unroll
                  for (int u = 0; u < 4; ++u) {
                    const float2 f = __bfloat1622float2(pv[u]);
                    acc[2 * u] += f.x;
                    acc[2 * u + 1] += f.y;
                  }
                }
              }
            }
            uint4 o;
            o.x = pack_bf16x2(acc[0], acc[1]); o.y = pack_bf16x2(acc[2], acc[3]);
            o.z = pack_bf16x2(acc[4], acc[5]); o.w = pack_bf16x2(acc[6], acc[7]);
            *reinterpret_cast<uint4*>(reinterpret_cast<bf16*>(fc.out) + (size_t)t * fc.ldo + (size_t)h * DH + ch * 8) = o;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) tmem_dealloc<512>(tmem);
}

template <int DH, int DE>
bool launch_t(const Routing& rt, const void* Xs, int64_t ldx, const void* W1, const void* W2, void* Yrep, int num_sms,
              cudaStream_t s, const FwdCombine& fc) {
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
  const size_t nslot = 32 * 4096;
  if (trace_path) {
    if (!tbuf) cudaMalloc(&tbuf, nslot * sizeof(unsigned long long));
    cudaMemsetAsync(tbuf, 0, nslot * sizeof(unsigned long long), s);
    TraceBuf tb{tbuf, 0};
    cudaMemcpyToSymbolAsync(g_trace_fwd, &tb, sizeof(tb), 0, cudaMemcpyHostToDevice, s);
  }
  const int lsu = store_lsu(0);
  if (fc.out && (lsu || L_YDIRECT)) return false;   // the fused combine needs the TMA-store path's signals
  kern<<<num_sms, kThreads, FwdL<DH, DE>::BYTES, s>>>(w1m, w2m, ym, xm, rt, (uint8_t*)Yrep, lsu, fc);
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
                             int d_e, void* Yrep, int num_sms, cudaStream_t s, const FwdCombine& fc) {
#define MHL_F(A, B) \
  if (d_h == A && d_e == B) return launch_t<A, B>(rt, Xs, ldx, W1, W2, Yrep, num_sms, s, fc);
  MHL_F(256, 128) MHL_F(256, 64) MHL_F(192, 64) MHL_F(128, 128) MHL_F(128, 64) MHL_F(64, 64) MHL_F(128, 256)
#undef MHL_F
  return false;
}

}  // namespace mhl
