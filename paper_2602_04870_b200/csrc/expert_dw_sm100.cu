// expert_dw_sm100.cu — B5 weight gradients of the block-sparse expert FFN on tcgen05/TMEM (sm_100a).
//
// Chain rule of y_r = g_r * gelu(x W1_e^T) W2_e over the clustered replicas of one expert
// (Eq. 1): with dH = g dA' gelu'(H) and gA = g gelu(H) from expert_bwd_dx_sm100.cu,
//   dW1_e^T = X^T dH,   dW2_e^T = dY^T gA        (X, dY = sub-token / dcat rows of the replicas)
// per chunk (one head's row part intersected with one expert segment, cluster.cu) on tcgen05 (both
// operands MN-major) into fp32 partials; the CTA finishing an expert's last chunk sums its partials
// in chunk order (deterministic, R21).  CTA b takes row part b of every head: equal rows per CTA.
#include <cuda.h>

#include "kernels.h"
#include "sm100.cuh"
#include "tma_host.h"

namespace mhl {

namespace {

using namespace sm100;

// =============================================================================================
// dW kernel: per chunk (a row part of one (head, expert)), accumulate in TMEM
//   dW1^T[c][f] += sum_r X[r][c] dH[r][f]   dW2^T[c][f] += sum_r dY[r][c] gA[r][f]
// M = c (DH/128 MMAs of M=128), N = f (DE), K = rows (16 per MMA), both operands MN-major.
// Warp roles: kDwProd producer warps bring X, dY (TMA gather4 for the token-indexed rows, one lane
// per 4 rows) and dH, gA (2-D TMA tiles of the contiguous sorted rows) into a 2-stage ring of
// 64-row steps; 8 warps flush each chunk's fp32 accumulators to its partial slot; the last warp
// issues the MMAs (+ owns TMEM).  The ring keeps filling while a chunk is flushed.
// =============================================================================================
#ifndef MHL_DW_STEP
#define MHL_DW_STEP 32
#endif
constexpr int kHalf = MHL_DW_STEP;   // rows per pipeline step (chunk boundaries stay kDwStep-aligned)
static_assert((kHalf == 64 || kHalf == 32 || kHalf == 16) && kDwStep % kHalf == 0, "dW pipeline step");

// The chunks of this CTA: part blockIdx.x of every head (cluster.cu dw_parts_kernel), in order.
struct MyChunks {
  const int32_t* pb; const int32_t* pc; int H, P;
  int h = 0, c = 0, end = 0;
  __device__ MyChunks(const Routing& rt) : pb(rt.pbase), pc(rt.pcount), H(rt.H), P(rt.dw_parts) {}
  __device__ int next() {
    while (c >= end) {
      if (h >= H) return -1;
      const int i = h * P + (int)blockIdx.x;
      c = pb[i]; end = c + pc[i]; ++h;
    }
    return c++;
  }
};
#ifndef MHL_DW_PROD
#define MHL_DW_PROD 16
#endif
constexpr int kDwProd = MHL_DW_PROD;           // producer warps 0..kDwProd-1 (8, or 16: half chunks)
constexpr int kDwFlush0 = kDwProd;             // 8 flush warps
constexpr int kDwMma = kDwProd + 8;
constexpr int kDwThreads = (kDwMma + 1) * 32;

template <int DH, int DE>
struct DwSmem {
  static constexpr int XB = kHalf * DH * 2, EB = kHalf * DE * 2;
  static constexpr int STAGE = 2 * XB + 2 * EB;                      // X, dY, dH, gA
  static constexpr int X = 0, DY = XB, DHH = 2 * XB, GA = 2 * XB + EB;
  static constexpr int S = 2 * (64 / kHalf);      // 192 KB of stages either way
  static constexpr int BAR = S * STAGE;            // full[S], empty[S], accfull, accempty
  static constexpr int LAST = BAR + 8 * (2 * S + 2);            // int: "this CTA reduces the expert"
  static constexpr int TMEM = LAST + 16;
  static constexpr int BYTES = TMEM + 16;
  static_assert(BYTES <= 227 * 1024, "dW: shared memory over the per-CTA limit");
};

template <int DH, int DE>
__global__ void __launch_bounds__(kDwThreads, 1)
expert_dw_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap ymap,
                 const __grid_constant__ CUtensorMap hmap, const __grid_constant__ CUtensorMap amap, Routing rt,
                 float* __restrict__ partial, int* __restrict__ done, float* __restrict__ dW1,
                 float* __restrict__ dW2) {
  const Tile* chunks = rt.chunks;
  const int64_t Rp = rt.Rp;
  using L = DwSmem<DH, DE>;
  constexpr int S = L::S, MH = DH / 128, XK = DH / 64, EK = DE / 64;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0u) __trap();
  const uint32_t sb = smem_u32(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* empty = full + S;
  uint64_t* accfull = full + 2 * S;
  uint64_t* accempty = accfull + 1;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::TMEM);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], kDwProd); mbar_init(&empty[i], 1); }
    mbar_init(accfull, 1); mbar_init(accempty, 256);
    fence_mbar_init();
    tma_prefetch_desc(&xmap); tma_prefetch_desc(&ymap); tma_prefetch_desc(&hmap); tma_prefetch_desc(&amap);
  }
  if (warp == kDwMma) tmem_alloc<512>(s_tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  const int nchunks = *rt.nchunks;

  // 16 producers: the launch cap falls to 72 registers; producers hand registers to the flush warps
  // (warpgroup-aligned roles: producers 0-15, flush 16-23): 16*(72-40) >= 8*(88-72)
  constexpr bool kRegs = kDwProd == 16;
  if (warp < kDwProd) {
    if constexpr (kRegs) asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
    // ================================================================ producers
    // A step needs 2*XK gathered 64-column chunks (X, dY: pair p -> operand p / XK, column block
    // p % XK) and 2*EK contiguous chunks (dH, gA).  Warp w takes pairs w, w + kDwProd, ...; in a
    // pair, lane g (mod 16) issues one gather4 for rows 4g..4g+3.
    constexpr int NP = 2 * XK, NT = 2 * EK;
    // more producer warps than chunks: WPCH warps share a chunk, warp w its rows [sub*RW, (sub+1)*RW)
    constexpr int WPCH = kDwProd > NP ? kDwProd / NP : 1, RW = kHalf / WPCH;
    const int sub = warp % WPCH;
    const int g = WPCH > 1 ? (sub * RW) / 4 + (lane & (RW / 4 - 1)) : (lane & 15);   // this lane's row group
    int mybytes = 0;
    if constexpr (WPCH > 1) mybytes += RW * 128;
    else for (int p = warp; p < NP; p += kDwProd) mybytes += kHalf * 128;
    for (int t = warp; t < NT; t += kDwProd) mybytes += kHalf * 128;
    int n = 0;                                                // steps of this CTA so far
    // X / dY rows are re-gathered by the head's other experts (keep them in L2); dH / gA stream
    // through once (evict first), so they do not push the reused rows out
    const uint64_t pol_keep = l2_evict_last(), pol_stream = l2_evict_first();
    MyChunks it(rt);
    for (int ci; (ci = it.next()) >= 0 && ci < nchunks;) {
      const Tile ch = chunks[ci];
      const int nsteps = ch.rows / kHalf;
      const int32_t* tk = rt.tok_s + (size_t)ch.head * Rp + ch.row0 + 4 * g;
      int r0 = tk[0], r1 = tk[1], r2 = tk[2], r3 = tk[3];
      int q0 = 0, q1 = 0, q2 = 0, q3 = 0;              // the next step's ids, loaded one step ahead
      if (nsteps > 1) { q0 = tk[kHalf]; q1 = tk[kHalf + 1]; q2 = tk[kHalf + 2]; q3 = tk[kHalf + 3]; }
      for (int s = 0; s < nsteps; ++s, ++n) {
        const int st = n % S;
        const uint32_t base = sb + st * L::STAGE;
        if (lane == 0) {
          mbar_wait(&empty[st], ((n / S) & 1) ^ 1);
          mbar_expect_tx(&full[st], mybytes);
          for (int t = warp; t < NT; t += kDwProd) {
            const int kb = t % EK;
            tma_load_2d_hint(base + (t < EK ? L::DHH : L::GA) + kb * kHalf * 128, t < EK ? &hmap : &amap, kb * 64,
                             (int)((size_t)ch.head * Rp + ch.row0 + s * kHalf), &full[st], pol_stream);
          }
        }
        __syncwarp();
        if constexpr (WPCH > 1) {
          const int p = warp / WPCH, kb = p % XK;
          if (lane < RW / 4)
            tma_gather4_hint(base + (p < XK ? L::X : L::DY) + kb * kHalf * 128 + 4 * g * 128, p < XK ? &xmap : &ymap,
                             ch.head * DH + kb * 64, r0, r1, r2, r3, &full[st], pol_keep);
        } else {
          for (int u = lane; u < ((NP - warp + kDwProd - 1) / kDwProd) * 16; u += 32) {
            const int p = warp + (u >> 4) * kDwProd, kb = p % XK;
            tma_gather4_hint(base + (p < XK ? L::X : L::DY) + kb * kHalf * 128 + 4 * g * 128, p < XK ? &xmap : &ymap,
                             ch.head * DH + kb * 64, r0, r1, r2, r3, &full[st], pol_keep);
          }
        }
        r0 = q0; r1 = q1; r2 = q2; r3 = q3;
        if (s + 2 < nsteps) {
          tk += kHalf;
          q0 = tk[kHalf]; q1 = tk[kHalf + 1]; q2 = tk[kHalf + 2]; q3 = tk[kHalf + 3];
        }
      }
    }
  } else if (warp == kDwMma) {
    // ================================================================ MMA issuer
    if (lane == 0) {
      constexpr uint32_t IDESC = idesc_bf16(128, DE, 1, 1);
      int n = 0, nc = 0;
      MyChunks it(rt);
      for (int ci; (ci = it.next()) >= 0 && ci < nchunks; ++nc) {
        const int nsteps = chunks[ci].rows / kHalf;
        if (nc >= 1) mbar_wait(accempty, (nc - 1) & 1);      // previous chunk flushed
        tc_fence_after();
        for (int s = 0; s < nsteps; ++s, ++n) {
          const int st = n % S;
          mbar_wait(&full[st], (n / S) & 1);
          tc_fence_after();
          const uint32_t base = sb + st * L::STAGE;
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
          mma_commit(&empty[st]);
        }
        mma_commit(accfull);
      }
    }
  } else if (warp >= kDwFlush0 && warp < kDwFlush0 + 8) {
    if constexpr (kRegs) asm volatile("setmaxnreg.inc.sync.aligned.u32 88;");
    // ================================================================ flush: partial[ci][mat][f][c]
    // Each chunk's accumulators go to its partial slot; the CTA that flushes an expert's LAST chunk
    // (counted with one atomic per chunk) then sums that expert's partials in chunk order and
    // writes dW1/dW2 — the same order as a separate reduction pass, without its launch and
    // re-read, and overlapped with the next chunk's MMAs.
    const int q = warp & 3, wm = (warp - kDwFlush0) >> 2;   // lane quadrant; 0: dW1, 1: dW2
    const int ft = tid - kDwFlush0 * 32;                    // 0..255
    constexpr int DEDH = DE * DH;
    int* s_last = reinterpret_cast<int*>(smem + L::LAST);
    static_assert(DEDH % (4 * 256 * 4) == 0, "dW reduce tiling");
    // experts without rows have no chunk: their gradients are zero
    for (int he = blockIdx.x; he < rt.H * rt.N_e; he += gridDim.x)
      if (rt.ccount[he] == 0)
        for (int i = ft; i < DEDH; i += 256) {
          if (dW1) dW1[(size_t)he * DEDH + i] = 0.f;
          if (dW2) dW2[(size_t)he * DEDH + i] = 0.f;
        }
    int nc = 0;
    MyChunks it(rt);
    for (int ci; (ci = it.next()) >= 0 && ci < nchunks; ++nc) {
      mbar_wait_warp(accfull, nc & 1);
      tc_fence_after();
      const Tile ch = chunks[ci];
      const int he = ch.head * rt.N_e + ch.expert;
      // an expert with a single chunk (small segments, e.g. the paper's N_e = 384-1536 per head)
      // is complete here: write dW directly, no partial round trip
      const bool single = rt.ccount[he] == 1;
      float* dWm = wm == 0 ? dW1 : dW2;
      if (single && dWm == nullptr) { tc_fence_before(); mbar_arrive(accempty); continue; }
      float* out = single ? dWm + (size_t)he * DE * DH : partial + ((size_t)ci * 2 + wm) * DE * DH;
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
      tc_fence_before();
      mbar_arrive(accempty);
      if ((dW1 == nullptr && dW2 == nullptr) || single) continue;
      __threadfence();
      named_bar_sync(1, 256);
      if (ft == 0) *s_last = (atomicAdd(&done[he], 1) == rt.ccount[he] - 1);
      named_bar_sync(1, 256);
      if (*s_last) {
        __threadfence();
        const int b0 = rt.cbase[he], n = rt.ccount[he];
        constexpr int U = 4;                              // float4s per thread in flight per matrix
        const float4* p4 = reinterpret_cast<const float4*>(partial);
        for (int i0 = ft; i0 < DEDH / 4; i0 += 256 * U) {
          float4 a1[U], a2[U];
#pragma unroll
          for (int u = 0; u < U; ++u) { a1[u] = make_float4(0.f, 0.f, 0.f, 0.f); a2[u] = a1[u]; }
          for (int c = 0; c < n; ++c) {
            const float4* s1 = p4 + ((size_t)(b0 + c) * 2 + 0) * (DEDH / 4);
            const float4* s2 = p4 + ((size_t)(b0 + c) * 2 + 1) * (DEDH / 4);
            float4 v1[U], v2[U];
#pragma unroll
            for (int u = 0; u < U; ++u) { v1[u] = __ldcg(s1 + i0 + 256 * u); v2[u] = __ldcg(s2 + i0 + 256 * u); }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              a1[u].x += v1[u].x; a1[u].y += v1[u].y; a1[u].z += v1[u].z; a1[u].w += v1[u].w;
              a2[u].x += v2[u].x; a2[u].y += v2[u].y; a2[u].z += v2[u].z; a2[u].w += v2[u].w;
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (dW1) reinterpret_cast<float4*>(dW1 + (size_t)he * DEDH)[i0 + 256 * u] = a1[u];
            if (dW2) reinterpret_cast<float4*>(dW2 + (size_t)he * DEDH)[i0 + 256 * u] = a2[u];
          }
        }
        if (ft == 0) done[he] = 0;   // ready for the next call
      }
      named_bar_sync(1, 256);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kDwMma) tmem_dealloc<512>(tmem);
}

template <int DH, int DE>
bool launch_dw_t(const Routing& rt, const void* Xs, int64_t ldx, const void* dY, int64_t ldy, const void* dH,
                 const void* gA, float* partial, int* done, float* dW1, float* dW2, int num_sms, cudaStream_t s) {
  CUtensorMap xm, ym, hm, am;
  const uint64_t rows = (uint64_t)rt.H * rt.Rp;
  if (!make_tmap_2d_bf16(&xm, Xs, (uint64_t)rt.T + 1, (uint64_t)rt.H * DH, (uint64_t)ldx * 2, 1, 64)) return false;
  if (!make_tmap_2d_bf16(&ym, dY, (uint64_t)rt.T + 1, (uint64_t)rt.H * DH, (uint64_t)ldy * 2, 1, 64)) return false;
  if (!make_tmap_2d_bf16(&hm, dH, rows, DE, (uint64_t)DE * 2, kHalf, 64)) return false;
  if (!make_tmap_2d_bf16(&am, gA, rows, DE, (uint64_t)DE * 2, kHalf, 64)) return false;
  auto kern = expert_dw_kernel<DH, DE>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, DwSmem<DH, DE>::BYTES);
  cudaMemsetAsync(done, 0, (size_t)rt.H * rt.N_e * sizeof(int), s);
  (void)num_sms;   // one CTA per dW row part (rt.dw_parts = kDwParts, a constant: bits independent of the device)
  kern<<<rt.dw_parts, kDwThreads, DwSmem<DH, DE>::BYTES, s>>>(xm, ym, hm, am, rt, partial, done, dW1, dW2);
  return true;
}

}  // namespace

bool expert_bwd_sm100_supported(int d_h, int d_e) {
  return (d_h == 256 && d_e == 128) || (d_h == 256 && d_e == 64) || (d_h == 128 && d_e == 128) ||
         (d_h == 128 && d_e == 64) || (d_h == 128 && d_e == 256);
}

bool launch_expert_bwd_sm100(const Routing& rt, const void* Xs, int64_t ldx, const void* dY, int64_t ldy,
                             const void* W1, const void* W2, int d_h, int d_e, void* dXrep, float* dg, void* dH,
                             void* gA, float* partial, int* done, float* dW1, float* dW2, int num_sms,
                             cudaStream_t s, bool do_dx, bool do_dw) {
  bool ok = false;
#define MHL_BWD_CASE(A, B)                                                                                       \
  if (d_h == A && d_e == B) {                                                                                    \
    ok = true;                                                                                                   \
    if (do_dx && !launch_expert_bwd_dx_sm100(rt, Xs, ldx, dY, ldy, W1, W2, d_h, d_e, dXrep, dg, dH, gA,       \
                                             num_sms, s))                                                        \
      ok = false;                                                                                                \
    if (do_dw && !launch_dw_t<A, B>(rt, Xs, ldx, dY, ldy, dH, gA, partial, done, dW1, dW2, num_sms, s)) ok = false; \
  }
  MHL_BWD_CASE(256, 128) else MHL_BWD_CASE(256, 64) else MHL_BWD_CASE(128, 128) else MHL_BWD_CASE(128, 64)
  else MHL_BWD_CASE(128, 256)
#undef MHL_BWD_CASE
  return ok;
}

}  // namespace mhl
