// expert_fwd_pair_sm100.cu — F5 on CTA pairs (tcgen05 cta_group::2): block-sparse expert FFN forward.
//
// Same computation as expert_sm100.cu (P:916-P:978, Eq. 7 semantics P:936):
//   GEMM1  H = X W1_eᵀ   →  epi 1  A = bf16(g·gelu(H)) → TMEM  →  GEMM2  Y = A W2_e  →  epi 2  Yrep
// but two CTAs of a cluster (one TPC) work on a PAIR of consecutive 128-row tiles of the same
// expert (F4 pads every expert segment to whole tile pairs) with M = 256 MMAs issued by the pair's
// leader.  cta_group::2 splits the B operand along N between the two CTAs, so each CTA keeps only
// HALF of W1_e (rows [r·d_e/2, (r+1)·d_e/2)) and HALF of W2_e (columns [r·d_h/2, (r+1)·d_h/2)) in
// shared memory.  The 64 KB this frees (at d_h = 256, d_e = 128) doubles the sub-token gather
// ring, so the next tile's rows stream in while the current tile computes — the single-CTA kernel
// could hold only one tile of X and waited a full gather latency per tile.
//
// Per CTA: warps 0-3 producers (TMA gather4 of the CTA's own 128 rows into its ring; completion
// is counted on the LEADER's barrier, .cta_group::2), warp 4 MMA (leader only; both CTAs own a
// TMEM allocation made with cta_group::2), warps 5-12 epilogue on the CTA's own rows.  Barriers
// the leader's MMA waits on live in the leader (X full, W full, H free, A full, Y empty: the peer
// arrives remotely); barriers the MMA signals are multicast to both CTAs by tcgen05.commit.
#include <cuda.h>

#include <cstdlib>

#include "kernels.h"
#include "sm100.cuh"
#include "tma_host.h"

namespace mhl {

namespace {

using namespace sm100;

__device__ TraceBuf g_trace_pair;   // profiling aid (MHL_TRACE_PAIR=<file>), CTA 0 only

constexpr int BM = kExpertBM;
constexpr int kProdWarps = 4, kMmaWarp = 4, kEpiWarp0 = 5;
constexpr int kThreads = 13 * 32;
constexpr int kEpiThreads = 256;
constexpr int kXChunk = BM * 128;
constexpr int kYStage = BM * 128;

template <int DH, int DE>
struct PL {
  static constexpr int WH = DE * DH;                               // half of one expert matrix (bytes)
  static constexpr int W1 = 0, W2 = WH, YS = 2 * WH, X = YS + 2 * kYStage;
  static constexpr int XS_RAW = (224 * 1024 - X) / kXChunk;
  static constexpr int XS = (XS_RAW > 12 ? 12 : XS_RAW) / kProdWarps * kProdWarps;
  static_assert(XS >= 2 * kProdWarps, "pair kernel: ring should hold two tiles");
  static constexpr int CTRL = X + XS * kXChunk;
  static constexpr int B_XFULL = CTRL, B_XEMPTY = B_XFULL + 8 * XS;
  static constexpr int B_W1F = B_XEMPTY + 8 * XS, B_W1E = B_W1F + 8, B_W2F = B_W1E + 8, B_W2E = B_W2F + 8;
  static constexpr int B_HFULL = B_W2E + 8, B_HFREE = B_HFULL + 8, B_AFULL = B_HFREE + 8, B_G2DONE = B_AFULL + 16;
  static constexpr int B_YEMPTY = B_G2DONE + 16;
  static constexpr int TMEMP = B_YEMPTY + 8;
  static constexpr int BYTES = TMEMP + 16;
  static_assert(BYTES <= 227 * 1024, "pair expert fwd: shared memory over the per-CTA limit");
  static constexpr uint32_t T_H = 0, T_A = 128, T_Y = 256;
};

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

template <int DH, int DE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
expert_fwd_pair_kernel(const __grid_constant__ CUtensorMap w1map, const __grid_constant__ CUtensorMap w2map,
                       const __grid_constant__ CUtensorMap ymap, const __grid_constant__ CUtensorMap xmap, Routing rt) {
  using L = PL<DH, DE>;
  constexpr int XS = L::XS, KB1 = DH / 64, KB2 = DH / 128;   // X k-chunks; W2 column chunks per CTA
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0u) __trap();
  const uint32_t sb = smem_u32(smem);
  auto bar = [&](int off) { return reinterpret_cast<uint64_t*>(smem + off); };
  auto lead = [&](int off) { return map_to_rank(sb + off, 0); };   // leader's barrier, cluster address
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::TMEMP);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  const Tile* tiles = rt.tiles;
  const int N_e = rt.N_e;
  TraceBuf trc = g_trace_pair;
  auto tev = [&](int ev, int t) {   // CTA 0 -> events ev, CTA 1 -> ev + 30 (per-SM clocks)
    if (trc.p != nullptr && blockIdx.x < 2 && t >= 0 && t < 4096) trc.p[(ev + 30 * blockIdx.x) * 4096 + t] = clock64();
  };

  if (tid == 0) {
    for (int i = 0; i < XS; ++i) { mbar_init(bar(L::B_XFULL + 8 * i), 1); mbar_init(bar(L::B_XEMPTY + 8 * i), 1); }
    mbar_init(bar(L::B_W1F), 1); mbar_init(bar(L::B_W1E), 1); mbar_init(bar(L::B_W2F), 1); mbar_init(bar(L::B_W2E), 1);
    mbar_init(bar(L::B_HFULL), 1);
    constexpr int kEpiArrivals = 2 * (kEpiThreads / 32);               // one per epilogue warp of each CTA
    mbar_init(bar(L::B_HFREE), kEpiArrivals);
    for (int b = 0; b < 2; ++b) { mbar_init(bar(L::B_AFULL + 8 * b), kEpiArrivals); mbar_init(bar(L::B_G2DONE + 8 * b), 1); }
    mbar_init(bar(L::B_YEMPTY), kEpiArrivals);
    fence_mbar_init();
    tma_prefetch_desc(&w1map); tma_prefetch_desc(&w2map); tma_prefetch_desc(&ymap); tma_prefetch_desc(&xmap);
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(s_tmem)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();                  // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  // pair-tile schedule: pair-tile u = tiles (2u, 2u+1), same (head, expert); this CTA takes tile 2u+rank
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

  if (warp < kProdWarps) {
    // ================================================================ producers (4 warps per CTA)
    const int pw = warp;
    Ph w1e, w2e;
    int cnt = 0;
    int nx[4] = {0, 0, 0, 0};
    auto load_tok = [&](int u) {
      if (u < 0) return;
      const Tile t = tiles[2 * u + rank];
      const int32_t* tk = rt.tok_s + (size_t)t.head * rt.Rp + t.row0 + 4 * lane;
      nx[0] = tk[0]; nx[1] = tk[1]; nx[2] = tk[2]; nx[3] = tk[3];
    };
    load_tok(pt_at(0));
    auto load_w1 = [&](const Tile& t) {       // this CTA's half: W1_e rows [rank*DE/2, +DE/2)
      const uint32_t f = lead(L::B_W1F);
      if (leader) mbar_expect_tx_local(sb + L::B_W1F, 2 * L::WH);
      for (int kb = 0; kb < KB1; ++kb)
        load2d_pair(sb + L::W1 + kb * (DE / 2) * 128, &w1map, kb * 64,
                    (t.head * N_e + t.expert) * DE + (int)rank * (DE / 2), f);
    };
    auto load_w2 = [&](const Tile& t) {       // this CTA's half: W2_e columns [rank*DH/2, +DH/2)
      const uint32_t f = lead(L::B_W2F);
      if (leader) mbar_expect_tx_local(sb + L::B_W2F, 2 * L::WH);
      for (int c = 0; c < KB2; ++c)
        load2d_pair(sb + L::W2 + c * DE * 128, &w2map, ((int)rank * KB2 + c) * 64, (t.head * N_e + t.expert) * DE, f);
    };
    for (int i = 0;; ++i) {
      const int u = pt_at(i);
      if (u < 0) {
        if (pw == 0 && i >= 1 && lane == 0 && !same_expert(pt_at(i - 2), pt_at(i - 1))) {
          mbar_wait(bar(L::B_W2E), w2e.flip() ^ 1);
          load_w2(tiles[2 * pt_at(i - 1)]);
        }
        break;
      }
      const Tile tl = tiles[2 * u + rank];
      const int r0 = nx[0], r1 = nx[1], r2 = nx[2], r3 = nx[3];
      load_tok(pt_at(i + 1));
      if (pw == 0 && lane == 0 && !same_expert(pt_at(i - 1), u)) {
        mbar_wait(bar(L::B_W1E), w1e.flip() ^ 1);
        load_w1(tl);
      }
      __syncwarp();
      for (int kb = 0; kb < KB1; ++kb, ++cnt) {
        if (cnt % kProdWarps != pw) continue;
        const int xs = cnt % XS;
        if (lane == 0) {
          mbar_wait(bar(L::B_XEMPTY + 8 * xs), ((cnt / XS) & 1) ^ 1);
          if (leader) mbar_expect_tx_local(sb + L::B_XFULL + 8 * xs, 2 * kXChunk);
        }
        __syncwarp();
        gather4_pair(sb + L::X + xs * kXChunk + lane * 4 * 128, &xmap, (int)tl.head * DH + kb * 64, r0, r1, r2, r3,
                     lead(L::B_XFULL + 8 * xs));
      }
      if (pw == 0 && lane == 0 && i >= 1 && !same_expert(pt_at(i - 2), pt_at(i - 1))) {
        mbar_wait(bar(L::B_W2E), w2e.flip() ^ 1);
        load_w2(tiles[2 * pt_at(i - 1)]);
      }
    }
  } else if (warp == kMmaWarp) {
    // ================================================================ MMA issuer (leader CTA only)
    if (leader && lane == 0) {
      constexpr uint32_t ID1 = idesc_bf16(2 * BM, DE, 0, 0);
      constexpr uint32_t ID2 = idesc_bf16(2 * BM, DH, 0, 1);
      Ph w1f, w2f, hfr, af[2], ye;
      int cnt = 0;
      auto gemm2 = [&](int j) {
        const int b = j & 1;
        const int uj = pt_at(j);
        if (!same_expert(pt_at(j - 1), uj)) mbar_wait(bar(L::B_W2F), w2f.flip());
        mbar_wait(bar(L::B_AFULL + 8 * b), af[b].flip());
        mbar_wait(bar(L::B_YEMPTY), ye.flip() ^ 1);
        tev(13, j);
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < DE / 16; ++ks)
          mma_pair_ts(tmem + L::T_Y, tmem + L::T_A + b * (DE / 2) + ks * 8,
                      sdesc_sw128(sb + L::W2 + ks * 2 * 1024, DE * 128, 1024), ID2, ks > 0);
        commit_pair(bar(L::B_G2DONE + 8 * b));
        if (!same_expert(uj, pt_at(j + 1))) commit_pair(bar(L::B_W2E));
      };
      int i = 0;
      for (;; ++i) {
        const int u = pt_at(i);
        if (u < 0) break;
        if (!same_expert(pt_at(i - 1), u)) mbar_wait(bar(L::B_W1F), w1f.flip());
        if (i >= 1) mbar_wait(bar(L::B_HFREE), hfr.flip());
        tev(10, i);
        tc_fence_after();
        for (int kb = 0; kb < KB1; ++kb, ++cnt) {
          const int xs = cnt % XS;
          mbar_wait(bar(L::B_XFULL + 8 * xs), (cnt / XS) & 1);
          tev(11, i * 8 + kb);
          tc_fence_after();
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            mma_pair(tmem + L::T_H, sdesc_sw128(sb + L::X + xs * kXChunk + ks * 32, 16, 1024),
                     sdesc_sw128(sb + L::W1 + kb * (DE / 2) * 128 + ks * 32, 16, 1024), ID1, (kb | ks) ? 1u : 0u);
          commit_pair(bar(L::B_XEMPTY + 8 * xs));
        }
        commit_pair(bar(L::B_HFULL));
        tev(12, i);
        if (!same_expert(u, pt_at(i + 1))) commit_pair(bar(L::B_W1E));
        if (i >= 1) gemm2(i - 1);
      }
      if (i >= 1) gemm2(i - 1);
    }
  } else {
    // ================================================================ epilogue (8 warps, this CTA's rows)
    const int q = warp & 3, half = (warp - kEpiWarp0) >> 2;
    const int row = q * 32 + lane;
    const int et = tid - kEpiWarp0 * 32;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    Ph hf, gd[2];
    int ys = 0;
    // one arrival per epilogue warp (8 per CTA) on a leader barrier once its lanes are past `fence`
    // The leader arrives on its own barrier with a plain CTA-scope arrive; the peer with a RELAXED
    // cluster-scope arrive: everything the leader's MMA depends on is TMEM state already settled by
    // tcgen05.wait::ld / wait::st before the arrive, and a release.cluster arrive measured ~1-1.5 k
    // cycles each (it made the peer's epilogue the pair's bottleneck).
    auto arrive_lead = [&](int off) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(bar(off));
        else asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(lead(off)) : "memory");
      }
    };
    auto epi2 = [&](int j) {
      const int b = j & 1;
      const Tile tl = tiles[2 * pt_at(j) + rank];
      mbar_wait_warp(bar(L::B_G2DONE + 8 * b), gd[b].flip());
      if (et == 0) tev(23, j);
      tc_fence_after();
      const bool wl = (half == 0 && lane == 0);
#pragma unroll 1
      for (int cb = 0; cb < DH / 64; ++cb, ++ys) {
        const int st = ys & 1;
        uint32_t v[32];
        tmem_ld32(tmem + L::T_Y + lane_off + cb * 64 + half * 32, v);
        tmem_ld_wait();
        if (cb == DH / 64 - 1) arrive_lead(L::B_YEMPTY);
        if (wl) bulk_wait_read<1>();
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
        fence_proxy_async();
        named_bar_sync(2 + q, 64);
        if (wl) {
          tma_store_2d(&ymap, sb + L::YS + st * kYStage + q * 4096, cb * 64,
                       (int)((size_t)tl.head * rt.Rp + tl.row0 + q * 32));
          bulk_commit();
        }
      }
    };
    int i = 0;
    for (;; ++i) {
      const int u = pt_at(i);
      if (u < 0) break;
      const Tile tl = tiles[2 * u + rank];
      const int b = i & 1;
      const float g = rt.gate_s[(size_t)tl.head * rt.Rp + tl.row0 + row];
      mbar_wait_warp(bar(L::B_HFULL), hf.flip());
      if (et == 0) tev(20, i);
      tc_fence_after();
      constexpr int NC = DE / 2;
      uint32_t hv[NC];
#pragma unroll
      for (int c = 0; c < NC; c += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + L::T_H + lane_off + half * NC + c, v);
#pragma unroll
        for (int w = 0; w < 32; ++w) hv[c + w] = v[w];
      }
      tmem_ld_wait();
      arrive_lead(L::B_HFREE);
      if (et == 0) tev(21, i);
      uint32_t pa[NC / 2];
#pragma unroll
      for (int w = 0; w < NC; w += 2) {
        // the single-CTA kernel's arithmetic (same bits, tested)
        const float2 a = gelu2_scaled(make_float2(__uint_as_float(hv[w]), __uint_as_float(hv[w + 1])), 0.5f * g);
        pa[w / 2] = pack_bf16x2(a.x, a.y);
      }
#pragma unroll
      for (int c = 0; c < NC / 2; c += 16) {
        uint32_t w[16];
#pragma unroll
        for (int x = 0; x < 16; ++x) w[x] = pa[c + x];
        tmem_st16(tmem + L::T_A + b * (DE / 2) + lane_off + half * (NC / 2) + c, w);
      }
      tmem_st_wait();
      arrive_lead(L::B_AFULL + 8 * b);
      if (et == 0) tev(22, i);
      if (i >= 1) epi2(i - 1);
      if (et == 0) tev(25, i);
    }
    if (i >= 1) epi2(i - 1);
    if (half == 0 && lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  cluster_sync();                  // the peer's TMEM / smem stay valid until the leader's MMAs are done
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

template <int DH, int DE>
bool launch_t(const Routing& rt, const void* Xs, int64_t ldx, const void* W1, const void* W2, void* Yrep, int num_sms,
              cudaStream_t s) {
  CUtensorMap w1m, w2m, ym, xm;
  if (!make_tmap_2d_bf16(&xm, Xs, (uint64_t)rt.T + 1, (uint64_t)rt.H * DH, (uint64_t)ldx * 2, 1, 64)) return false;
  if (!make_tmap_2d_bf16(&w1m, W1, (uint64_t)rt.H * rt.N_e * DE, DH, (uint64_t)DH * 2, DE / 2, 64)) return false;
  if (!make_tmap_2d_bf16(&w2m, W2, (uint64_t)rt.H * rt.N_e * DE, DH, (uint64_t)DH * 2, DE, 64)) return false;
  if (!make_tmap_2d_bf16(&ym, Yrep, (uint64_t)rt.H * rt.Rp, DH, (uint64_t)DH * 2, 32, 64)) return false;
  auto kern = expert_fwd_pair_kernel<DH, DE>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, PL<DH, DE>::BYTES);
  const int grid = (num_sms / 2) * 2;
  static const char* trace_path = getenv("MHL_TRACE_PAIR");
  if (trace_path) {
    TraceBuf tb{trace_buffer(s), 0};
    cudaMemcpyToSymbolAsync(g_trace_pair, &tb, sizeof(tb), 0, cudaMemcpyHostToDevice, s);
  }
  kern<<<grid, kThreads, PL<DH, DE>::BYTES, s>>>(w1m, w2m, ym, xm, rt);
  if (trace_path) {
    TraceBuf tb{nullptr, 0};
    cudaMemcpyToSymbolAsync(g_trace_pair, &tb, sizeof(tb), 0, cudaMemcpyHostToDevice, s);
    trace_dump(trace_path, s);
  }
  return true;
}

}  // namespace

bool expert_fwd_pair_supported(int d_h, int d_e) {
  // tiles 2u and 2u+1 must share an expert: segments padded to whole tile pairs
  return (d_h == 256 || d_h == 128) && (d_e == 128 || d_e == 64);   // caller: seg_align = 256
}

bool launch_expert_fwd_pair_sm100(const Routing& rt, const void* Xs, int64_t ldx, const void* W1, const void* W2,
                                  int d_h, int d_e, void* Yrep, int num_sms, cudaStream_t s) {
  if (rt.seg_align % (2 * kExpertBM) != 0) return false;   // tiles 2u, 2u+1 must share an expert
#define MHL_P(A, B) \
  if (d_h == A && d_e == B) return launch_t<A, B>(rt, Xs, ldx, W1, W2, Yrep, num_sms, s);
  MHL_P(256, 128) MHL_P(256, 64) MHL_P(128, 128) MHL_P(128, 64)
#undef MHL_P
  return false;
}

}  // namespace mhl
