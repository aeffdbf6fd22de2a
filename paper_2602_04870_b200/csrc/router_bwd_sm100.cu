// router_bwd_sm100.cu — B3 on tcgen05: softmax Jacobian and router weight gradient (P:846-P:866).
//
//   dS[t][j]       = g_j (dg_j - sum_i g_i dg_i)                       (gate Jacobian, Alg. 2)
//   dW_r[h][i][e]  = sum_t X_h[t][i] * dS_dense[t][e],  dS_dense[t][e] = dS[t][j] if I[t][j] = e else 0
//
// dW_r is a (d_h x T) . (T x N_e) contraction with K = T, so it runs on the tensor cores:
// A = X_h^T read straight from the stored sub-tokens (bf16, exact) as an MN-major operand (the
// TMA box of 64 tokens x 64 features is already the MN-major SW128 atom), B = dS_dense^T built
// per 64-token step in shared memory (K-major, N_e rows).  dS is fp32; it enters the MMA as two
// bf16 planes hi = rn(dS), lo = rn(dS - hi) (16 significant bits, relative error <= 2^-17), both
// accumulated into the same fp32 TMEM accumulator.  Each CTA owns a contiguous token range of one
// head and writes one fp32 partial; a second kernel sums the partials in CTA order, so dW_r is
// deterministic (R21).
//
// Warp roles: warp 0 = TMA producer (X ring), warp 1 = MMA issuer + TMEM owner, warps 2-5 = dS
// builders (one token per thread for the Jacobian, all four zero the dense tile) and the epilogue.
#include <cuda.h>

#include <algorithm>

#include "kernels.h"
#include "sm100.cuh"
#include "tma_host.h"

namespace mhl {

namespace {

using namespace sm100;

constexpr int kStep = 64;                 // tokens (= MMA K) per pipeline step
constexpr int kThreads = 6 * 32;
constexpr int kBuilders = 128;

template <int DH, int NE>
struct RbL {
  static constexpr int XSTAGE = (DH / 64) * kStep * 128;     // one step of X: DH/64 boxes of 64 x 64
  static constexpr int BT = NE * 128;                        // one K-major bf16 plane: NE rows x 64 tokens
  static constexpr int BBUF = 2 * BT;                        // hi + lo
  static constexpr int XS_RAW = (220 * 1024 - 2 * BBUF) / XSTAGE;
  // two X stages: ~97 KB of smem at d_h = 256, N_e = 64, so two CTAs share an SM (the builders'
  // per-step chain is latency-bound; one 6-warp CTA per SM left 91 % of the warp slots empty)
  static constexpr int XS = XS_RAW > 2 ? 2 : XS_RAW;
  static constexpr int X = 0, B = XS * XSTAGE, BAR = B + 2 * BBUF;
  static constexpr int NBAR = 2 * XS + 5;                    // xfull[XS], xempty[XS], bfull[2], bempty[2], acc
  static constexpr int TMEMP = BAR + NBAR * 8;
  static constexpr int BYTES = TMEMP + 16;
  static_assert(BYTES <= 227 * 1024, "router bwd: shared memory over the per-CTA limit");
  static constexpr int ACC_COLS = (DH / 128) * NE;
  static constexpr int TMEM_COLS = ACC_COLS <= 32 ? 32 : ACC_COLS <= 64 ? 64 : ACC_COLS <= 128 ? 128
                                   : ACC_COLS <= 256 ? 256 : 512;
  static_assert(XS >= 2, "router backward: X ring too small");
};

template <int DH, int NE, int KMAX>
__global__ void __launch_bounds__(kThreads, 2)
router_bwd_sm100_kernel(const __grid_constant__ CUtensorMap xmap, const int32_t* __restrict__ idx,
                        const float* __restrict__ gate, const float* __restrict__ dg, int64_t T, int k, int nc,
                        int N_e, float* __restrict__ dS, float* __restrict__ partial) {
  // blockIdx.z = expert block [e0, e0 + NE) of N_e (the paper's own N_e = 384-1536 per head)
  const int e0 = blockIdx.z * NE;
  using L = RbL<DH, NE>;
  constexpr int XS = L::XS, XB = DH / 64;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0u) __trap();
  const uint32_t sb = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* xfull = bars;
  uint64_t* xempty = bars + XS;
  uint64_t* bfull = bars + 2 * XS;
  uint64_t* bempty = bfull + 2;
  uint64_t* accf = bfull + 4;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::TMEMP);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c = blockIdx.x, h = blockIdx.y;
  const int64_t nst = (T + kStep - 1) / kStep;
  const int64_t s0 = nst * c / nc, s1 = nst * (c + 1) / nc;   // host guarantees nc <= nst: s1 > s0
  const int ns = (int)(s1 - s0);

  if (tid == 0) {
    for (int i = 0; i < XS; ++i) { mbar_init(&xfull[i], 1); mbar_init(&xempty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&bfull[i], kBuilders); mbar_init(&bempty[i], 1); }
    mbar_init(accf, 1);
    fence_mbar_init();
    tma_prefetch_desc(&xmap);
  }
  if (warp == 1) tmem_alloc<L::TMEM_COLS>(s_tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  if (warp == 0) {
    // ============================ TMA producer: X[t0:t0+64][h*DH : (h+1)*DH] per step
    if (lane == 0) {
      int st = 0; uint32_t ph = 0;
      for (int s = 0; s < ns; ++s) {
        mbar_wait(&xempty[st], ph ^ 1);
        mbar_expect_tx(&xfull[st], L::XSTAGE);
        const int t0 = (int)((s0 + s) * kStep);
        for (int b = 0; b < XB; ++b)
          tma_load_2d(sb + L::X + st * L::XSTAGE + b * kStep * 128, &xmap, h * DH + b * 64, t0, &xfull[st]);
        if (++st == XS) { st = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer: acc[mh] (128 features x NE) += X^T . (hi + lo)
    if (lane == 0) {
      constexpr uint32_t IDESC = idesc_bf16(128, NE, 1, 0);   // A MN-major (features contiguous)
      int st = 0; uint32_t ph = 0;
      uint32_t bph[2] = {0, 0};
      for (int s = 0; s < ns; ++s) {
        const int bs = s & 1;
        mbar_wait(&xfull[st], ph);
        mbar_wait(&bfull[bs], bph[bs]); bph[bs] ^= 1;
        tc_fence_after();
        const uint32_t xa = sb + L::X + st * L::XSTAGE;
        const uint32_t bb = sb + L::B + bs * L::BBUF;
#pragma unroll
        for (int mh = 0; mh < DH / 128; ++mh)
#pragma unroll
          for (int ks = 0; ks < kStep / 16; ++ks)
#pragma unroll
            for (int p = 0; p < 2; ++p)
              mma_bf16(tmem + mh * NE, sdesc_sw128(xa + 2 * mh * kStep * 128 + ks * 2048, kStep * 128, 1024),
                       sdesc_sw128(bb + p * L::BT + ks * 32, 16, 1024), IDESC, (s | ks | p) ? 1u : 0u);
        mma_commit(&xempty[st]);
        mma_commit(&bempty[bs]);
        if (++st == XS) { st = 0; ph ^= 1; }
      }
      mma_commit(accf);
    }
  } else {
    // ============================ dS builders (thread tt < 64 = token of the step), then epilogue
    const int tt = tid - 64;
    uint32_t eph[2] = {0, 0};
    // the step's gates / dg / expert ids are prefetched two steps ahead (two register sets, the
    // step loop unrolled by two): their global-load latency stalled the builders (ncu r2c: long
    // scoreboard + the builders' barrier held 40 % of the kernel's samples with one step of lookahead)
    struct Rt { float g[KMAX], d[KMAX]; int e[KMAX]; };
    auto load = [&](Rt& r, int s) {
      const int64_t t = (s0 + s) * kStep + tt;
#pragma unroll
      for (int j = 0; j < KMAX; ++j) { r.g[j] = 0.f; r.d[j] = 0.f; r.e[j] = -1; }
      if (s < ns && tt < kStep && t < T) {
        const size_t base = ((size_t)h * T + t) * k;
#pragma unroll
        for (int j = 0; j < KMAX; ++j)
          if (j < k) { r.g[j] = __ldg(gate + base + j); r.d[j] = __ldg(dg + base + j); r.e[j] = __ldg(idx + base + j); }
      }
    };
    auto build = [&](const Rt& r, int s) {
      const int bs = s & 1;
      mbar_wait(&bempty[bs], eph[bs] ^ 1); eph[bs] ^= 1;
      uint8_t* bt = smem + L::B + bs * L::BBUF;
      for (int o = tt * 16; o < L::BBUF; o += kBuilders * 16) *reinterpret_cast<uint4*>(bt + o) = make_uint4(0, 0, 0, 0);
      named_bar_sync(1, kBuilders);
      const int64_t t = (s0 + s) * kStep + tt;
      if (tt < kStep && t < T) {
        float sum = 0.f;
#pragma unroll
        for (int j = 0; j < KMAX; ++j) if (j < k) sum = fmaf(r.g[j], r.d[j], sum);
        float* dso = dS + ((size_t)h * T + t) * k;
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
          if (j < k) {
            const float v = r.g[j] * (r.d[j] - sum);
            if (blockIdx.z == 0) dso[j] = v;
            const int el = r.e[j] - e0;
            if (el >= 0 && el < NE) {
              const bf16 hi = __float2bfloat16_rn(v);
              const bf16 lo = __float2bfloat16_rn(v - __bfloat162float(hi));
              const uint32_t off = kmaj_off(el, tt, NE);
              *reinterpret_cast<bf16*>(bt + off) = hi;
              *reinterpret_cast<bf16*>(bt + L::BT + off) = lo;
            }
          }
        }
      }
      fence_proxy_async();
      mbar_arrive(&bfull[bs]);
    };
    Rt ra, rb;
    load(ra, 0);
    load(rb, 1);
    for (int s = 0; s < ns; s += 2) {
      build(ra, s);
      load(ra, s + 2);
      if (s + 1 < ns) {
        build(rb, s + 1);
        load(rb, s + 3);
      }
    }
    // epilogue: features (TMEM lanes) x experts (columns) -> partial[h][c][i][e]
    mbar_wait(accf, 0);
    tc_fence_after();
    const int q = warp & 3;
#pragma unroll 1
    for (int mh = 0; mh < DH / 128; ++mh) {
      const int i = mh * 128 + q * 32 + lane;
      float* po = partial + (((size_t)h * nc + c) * DH + i) * N_e + e0;
#pragma unroll 1
      for (int e0 = 0; e0 < NE; e0 += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + mh * NE + e0, v);
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 32; u += 4)
          *reinterpret_cast<uint4*>(po + e0 + u) = make_uint4(v[u], v[u + 1], v[u + 2], v[u + 3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<L::TMEM_COLS>(tmem);
}

// dW_r[h][i][e] = sum over c (in order) of partial[h][c][i][e]
__global__ void __launch_bounds__(256)
router_bwd_sum_kernel(const float* __restrict__ partial, int nc, int64_t n, float* __restrict__ dW_r) {
  const int h = blockIdx.y;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int c = 0; c < nc; ++c) acc += partial[((size_t)h * nc + c) * n + o];
    dW_r[(size_t)h * n + o] = acc;
  }
}

template <int DH, int NE, int KMAX>
bool launch_t(const void* Xs, int64_t ldx, const int32_t* idx, const float* gate, const float* dg, int H, int64_t T,
              int k, int N_e, float* dS, float* partial, int nc_target, float* dW_r, cudaStream_t s) {
  using L = RbL<DH, NE>;
  CUtensorMap xm;
  if (!make_tmap_2d_bf16(&xm, Xs, (uint64_t)T, (uint64_t)H * DH, (uint64_t)ldx * 2, kStep, 64)) return false;
  const int64_t nst = (T + kStep - 1) / kStep;
  const int nc = (int)std::max<int64_t>(1, std::min<int64_t>(nc_target, nst));
  auto kern = router_bwd_sm100_kernel<DH, NE, KMAX>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::BYTES);
  kern<<<dim3(nc, H, N_e / NE), kThreads, L::BYTES, s>>>(xm, idx, gate, dg, T, k, nc, N_e, dS, partial);
  if (dW_r) {
    const int64_t n = (int64_t)DH * N_e;
    router_bwd_sum_kernel<<<dim3((unsigned)std::max<int64_t>(1, (n + 255) / 256), H), 256, 0, s>>>(partial, nc, n, dW_r);
  }
  return true;
}

template <int DH, int NE>
bool launch_k(const void* Xs, int64_t ldx, const int32_t* idx, const float* gate, const float* dg, int H, int64_t T,
              int k, int N_e, float* dS, float* partial, int nc_target, float* dW_r, cudaStream_t s) {
#define MHL_RBK(KM) return launch_t<DH, NE, KM>(Xs, ldx, idx, gate, dg, H, T, k, N_e, dS, partial, nc_target, dW_r, s);
  if (k <= 2) MHL_RBK(2)
  if (k <= 4) MHL_RBK(4)
  if (k <= 8) MHL_RBK(8)
  MHL_RBK(16)
#undef MHL_RBK
}

}  // namespace

bool router_bwd_sm100_supported(int d_h, int N_e, int k) {
  const bool blocked = N_e > 256 && N_e % 256 == 0;          // processed in blocks of 256 experts
  return (d_h == 128 || d_h == 256) && (N_e == 32 || N_e == 64 || N_e == 128 || N_e == 256 || blocked) &&
         k >= 1 && k <= 16 && k <= N_e;
}

bool launch_router_bwd_sm100(const void* Xs, int64_t ldx, const int32_t* idx, const float* gate, const float* dg,
                             int H, int64_t T, int k, int d_h, int N_e, float* dS, float* partial, int nc_target,
                             float* dW_r, cudaStream_t s) {
  if (T <= 0) return false;
  const int NEB = N_e > 256 ? 256 : N_e;                      // experts per CTA block
#define MHL_RB(A, B)        \
  if (d_h == A && NEB == B) \
    return launch_k<A, B>(Xs, ldx, idx, gate, dg, H, T, k, N_e, dS, partial, nc_target, dW_r, s);
  MHL_RB(256, 32) MHL_RB(256, 64) MHL_RB(256, 128) MHL_RB(256, 256)
  MHL_RB(128, 32) MHL_RB(128, 64) MHL_RB(128, 128) MHL_RB(128, 256)
#undef MHL_RB
  return false;
}

}  // namespace mhl
