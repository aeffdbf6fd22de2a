// expert_sm100.cu — F5: block-sparse expert FFN forward on tcgen05/TMEM (sm_100a).
//
// The paper's IO-aware expert computation (P:916-P:978) treats the replicas clustered by
// expert (Fig. 2) as queries and expert e's W1_e/W2_e rows as keys/values (Eq. 7):
// Y = gelu(X W1_e^T) W2_e, with the T x k x d_e hidden activation never written to HBM.
// Here a tile = 128 clustered replicas of one (head, expert):
//   GEMM1  H[128 x d_e]  = X[128 x d_h] . W1_e^T     tcgen05.mma, A = gathered sub-tokens
//                                                      (K-major SW128 smem), B = W1_e (K-major)
//   epi 1  A = bf16(gelu(H))  TMEM -> registers -> smem (K-major SW128), exact-erf GELU (R1)
//   GEMM2  Y[128 x d_h]  = A . W2_e                   B = W2_e read MN-major (no transpose pass)
//   epi 2  Yrep[row] = bf16(gate * Y)                 TMEM -> registers -> HBM
// Persistent CTAs (one per SM) take contiguous runs of the (head, expert)-ordered tile list,
// so W1_e / W2_e stay resident in shared memory across consecutive tiles of an expert.
#include "kernels.h"
#include "sm100.cuh"

namespace mhl {

namespace {

using namespace sm100;

constexpr int BM = kExpertBM;   // 128 replica rows = MMA M
constexpr int kThreads = 256;   // 8 warps: all load; warp 0 lane 0 issues MMAs; 8 warps run epilogues

template <int DH, int DE>
struct FwdSmem {
  static constexpr int X = 0;                         // [BM][DH]  K-major SW128
  static constexpr int W1 = X + BM * DH * 2;          // [DE][DH]  K-major SW128
  static constexpr int W2 = W1 + DE * DH * 2;         // [DE(K)][DH(N)] MN-major SW128
  static constexpr int A = W2 + DE * DH * 2;          // [BM][DE]  K-major SW128
  static constexpr int BAR = A + BM * DE * 2;         // mbarrier
  static constexpr int TOK = BAR + 16;                // [BM] token ids
  static constexpr int GATE = TOK + BM * 4;           // [BM] gates
  static constexpr int TMEM = GATE + BM * 4;          // TMEM base address
  static constexpr int TOTAL = TMEM + 16;
  static constexpr int BYTES = TOTAL;
};

template <int DH, int DE>
__global__ void __launch_bounds__(kThreads, 1)
expert_fwd_sm100_kernel(const Tile* __restrict__ tiles, const int32_t* __restrict__ ntiles_p,
                        const bf16* __restrict__ Xs, int64_t ldx, const int32_t* __restrict__ perm,
                        const float* __restrict__ gate, const bf16* __restrict__ W1, const bf16* __restrict__ W2,
                        int64_t R, int k, int N_e, bf16* __restrict__ Yrep) {
  using L = FwdSmem<DH, DE>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;   // SW128 atoms need 1024-byte alignment (checked below)
  if ((smem_u32(smem) & 1023u) != 0u) __trap();
  const uint32_t sbase = smem_u32(smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::BAR);
  int* s_tok = reinterpret_cast<int*>(smem + L::TOK);
  float* s_gate = reinterpret_cast<float*>(smem + L::GATE);
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::TMEM);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (warp == 0) tmem_alloc<512>(s_tmem);
  if (tid == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  const uint32_t tH = tmem;           // H: columns [0, DE)
  const uint32_t tY = tmem + 256;     // Y: columns [256, 256 + DH)
  uint32_t phase = 0;

  const int nt = *ntiles_p;
  const int per = (nt + gridDim.x - 1) / gridDim.x;
  const int t_begin = min(nt, (int)blockIdx.x * per), t_end = min(nt, t_begin + per);
  int cur_h = -1, cur_e = -1;
  constexpr uint32_t IDESC1 = idesc_bf16(BM, DE, 0, 0);
  constexpr uint32_t IDESC2 = idesc_bf16(BM, DH, 0, 1);
  constexpr int NA2 = DH / 64;

  for (int ti = t_begin; ti < t_end; ++ti) {
    const Tile tl = tiles[ti];
    // ---- token ids and gates of the tile's replicas
    if (tid < BM) {
      int tok = -1; float g = 0.f;
      if (tid < tl.rows) {
        const int rep = perm[(size_t)tl.head * R + tl.row0 + tid];
        tok = rep / k;
        g = gate[(size_t)tl.head * R + rep];
      }
      s_tok[tid] = tok; s_gate[tid] = g;
    }
    __syncthreads();
    // ---- expert weights (only when the (head, expert) changes)
    if (tl.head != cur_h || tl.expert != cur_e) {
      const size_t wofs = ((size_t)tl.head * N_e + tl.expert) * DE * DH;
      const bf16* w1 = W1 + wofs;
      const bf16* w2 = W2 + wofs;
      for (int i = tid; i < DE * DH / 8; i += kThreads) {
        const int row = i / (DH / 8), c = (i % (DH / 8)) * 8;
        cp_async_16(sbase + L::W1 + kmaj_off(row, c, DE), w1 + (size_t)row * DH + c, 16);
        cp_async_16(sbase + L::W2 + mnmaj_off(row, c, NA2), w2 + (size_t)row * DH + c, 16);
      }
      cur_h = tl.head; cur_e = tl.expert;
    }
    // ---- gather the tile's sub-tokens (rows of head tl.head); zero-fill padding rows
    for (int i = tid; i < BM * DH / 8; i += kThreads) {
      const int row = i / (DH / 8), c = (i % (DH / 8)) * 8;
      const int tok = s_tok[row];
      const bf16* src = Xs + (size_t)(tok < 0 ? 0 : tok) * ldx + (size_t)tl.head * DH + c;
      cp_async_16(sbase + L::X + kmaj_off(row, c, BM), src, tok < 0 ? 0u : 16u);
    }
    cp_async_commit();
    cp_async_wait_all();
    fence_proxy_async();
    __syncthreads();

    // ---- GEMM1: H = X W1^T   (K = DH in steps of 16)
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int ks = 0; ks < DH / 16; ++ks) {
        const uint32_t koff = (ks >> 2) * 0 + (ks & 3) * 32;
        const uint64_t ad = sdesc_sw128(sbase + L::X + (ks >> 2) * BM * 128 + koff, 16, 1024);
        const uint64_t bd = sdesc_sw128(sbase + L::W1 + (ks >> 2) * DE * 128 + koff, 16, 1024);
        mma_bf16(tH, ad, bd, IDESC1, ks > 0 ? 1u : 0u);
      }
      mma_commit(bar);
    }
    mbar_wait(bar, phase); phase ^= 1;
    tc_fence_after();

    // ---- epilogue 1: A = bf16(gelu(H)) into smem (8 warps: lane quadrant x column half)
    {
      const int q = warp & 3, half = warp >> 2;
      const int row = q * 32 + lane;
      for (int c0 = half * (DE / 2); c0 < (half + 1) * (DE / 2); c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tH + ((uint32_t)(q * 32) << 16) + c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          uint4 pk;
          pk.x = pack_bf16x2(gelu_f(__uint_as_float(v[j + 0])), gelu_f(__uint_as_float(v[j + 1])));
          pk.y = pack_bf16x2(gelu_f(__uint_as_float(v[j + 2])), gelu_f(__uint_as_float(v[j + 3])));
          pk.z = pack_bf16x2(gelu_f(__uint_as_float(v[j + 4])), gelu_f(__uint_as_float(v[j + 5])));
          pk.w = pack_bf16x2(gelu_f(__uint_as_float(v[j + 6])), gelu_f(__uint_as_float(v[j + 7])));
          *reinterpret_cast<uint4*>(smem + L::A + kmaj_off(row, c0 + j, BM)) = pk;
        }
      }
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();

    // ---- GEMM2: Y = A W2   (K = DE in steps of 16; W2 MN-major)
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int ks = 0; ks < DE / 16; ++ks) {
        const uint64_t ad = sdesc_sw128(sbase + L::A + (ks >> 2) * BM * 128 + (ks & 3) * 32, 16, 1024);
        const uint64_t bd = sdesc_sw128(sbase + L::W2 + ks * 2 * NA2 * 1024, 1024, NA2 * 1024);
        mma_bf16(tY, ad, bd, IDESC2, ks > 0 ? 1u : 0u);
      }
      mma_commit(bar);
    }
    mbar_wait(bar, phase); phase ^= 1;
    tc_fence_after();

    // ---- epilogue 2: Yrep[row] = bf16(gate * Y)
    {
      const int q = warp & 3, half = warp >> 2;
      const int row = q * 32 + lane;
      const float g = s_gate[row];
      bf16* dst = Yrep + ((size_t)tl.head * R + tl.row0 + row) * DH;
      for (int c0 = half * (DH / 2); c0 < (half + 1) * (DH / 2); c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tY + ((uint32_t)(q * 32) << 16) + c0, v);
        tmem_ld_wait();
        if (row < tl.rows) {
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            uint4 pk;
            pk.x = pack_bf16x2(g * __uint_as_float(v[j + 0]), g * __uint_as_float(v[j + 1]));
            pk.y = pack_bf16x2(g * __uint_as_float(v[j + 2]), g * __uint_as_float(v[j + 3]));
            pk.z = pack_bf16x2(g * __uint_as_float(v[j + 4]), g * __uint_as_float(v[j + 5]));
            pk.w = pack_bf16x2(g * __uint_as_float(v[j + 6]), g * __uint_as_float(v[j + 7]));
            *reinterpret_cast<uint4*>(dst + c0 + j) = pk;
          }
        }
      }
    }
    tc_fence_before();
    __syncthreads();
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int DH, int DE>
void launch_t(const Tile* tiles, const int32_t* ntiles, const void* Xs, int64_t ldx, const int32_t* perm,
              const float* gate, const void* W1, const void* W2, int64_t R, int k, int N_e, void* Yrep, int num_sms,
              cudaStream_t s) {
  auto kern = expert_fwd_sm100_kernel<DH, DE>;
  const int smem = FwdSmem<DH, DE>::BYTES;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<<<num_sms, kThreads, smem, s>>>(tiles, ntiles, (const bf16*)Xs, ldx, perm, gate, (const bf16*)W1,
                                       (const bf16*)W2, R, k, N_e, (bf16*)Yrep);
}

}  // namespace

bool expert_fwd_sm100_supported(int d_h, int d_e) {
  return (d_h == 256 && d_e == 128) || (d_h == 192 && d_e == 64) || (d_h == 256 && d_e == 64) ||
         (d_h == 128 && d_e == 128) || (d_h == 64 && d_e == 64);
}

void launch_expert_fwd_sm100(const Tile* tiles, const int32_t* ntiles, int max_tiles, const void* Xs, int64_t ldx,
                             const int32_t* perm, const float* gate, const void* W1, const void* W2, int64_t T, int k,
                             int N_e, int d_h, int d_e, void* Yrep, int num_sms, cudaStream_t s) {
  (void)max_tiles;
  const int64_t R = T * k;
  if (d_h == 256 && d_e == 128) launch_t<256, 128>(tiles, ntiles, Xs, ldx, perm, gate, W1, W2, R, k, N_e, Yrep, num_sms, s);
  else if (d_h == 192 && d_e == 64) launch_t<192, 64>(tiles, ntiles, Xs, ldx, perm, gate, W1, W2, R, k, N_e, Yrep, num_sms, s);
  else if (d_h == 256 && d_e == 64) launch_t<256, 64>(tiles, ntiles, Xs, ldx, perm, gate, W1, W2, R, k, N_e, Yrep, num_sms, s);
  else if (d_h == 128 && d_e == 128) launch_t<128, 128>(tiles, ntiles, Xs, ldx, perm, gate, W1, W2, R, k, N_e, Yrep, num_sms, s);
  else if (d_h == 64 && d_e == 64) launch_t<64, 64>(tiles, ntiles, Xs, ldx, perm, gate, W1, W2, R, k, N_e, Yrep, num_sms, s);
}

}  // namespace mhl
