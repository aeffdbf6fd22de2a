// router.cu — F3: fused router GEMM + bias + online top-k + gate softmax (Alg. 1, P:819-P:841).
//
// One CTA = 128 tokens of one head (Alg. 1's (b, t_block, h) parallel loop);
// one thread = one token.  The sub-token tile is staged once in shared memory
// (transposed, so the per-feature broadcast of W_r is bank-conflict free) and the
// experts are visited in blocks of M = 32 (Alg. 1 line 5).  For each block the
// fp32 scores S_block = X W_r,block + b_block are formed in registers (line 7),
// packed with their index into 64-bit keys (line 8, R6) and merged into the running
// register-resident top-k (lines 9-10).  The T x N_e score matrix never reaches
// HBM (P:336-P:337).  The raw (unbiased) score is carried next to each key, so the
// returned scores/gates exclude the bias exactly (R5) and the gate softmax
// over the k unbiased scores (Eq. 2-3, R4) is computed in the same pass.  The pass
// also emits the per-tile expert histogram consumed by the clustering pass (F4).
//
// Precision (R3): products are exact fp32 FMAs of the stored sub-token
// (bf16 values are exact in fp32) with fp32 W_r, accumulated in fp32 in fixed
// feature order.
#include "kernels.h"

namespace mhl {

namespace {

constexpr int kEB = 32;   // expert block M of Alg. 1

template <typename E, int KMAX>
__global__ void __launch_bounds__(kRouterTile)
router_topk_kernel(const E* __restrict__ Xs, int64_t ldx, const float* __restrict__ W_r,
                   const float* __restrict__ bias, int64_t T, int d_h, int N_e, int k,
                   int32_t* __restrict__ idx, float* __restrict__ gate, int32_t* __restrict__ hist,
                   int32_t* __restrict__ flag) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int h = blockIdx.y;
  const int tile = blockIdx.x;
  const int tid = threadIdx.x;
  const int64_t t0 = (int64_t)tile * kRouterTile;
  E* Xt = reinterpret_cast<E*>(smem_raw);                                   // [d_h][128]
  float* Wb = reinterpret_cast<float*>(smem_raw + sizeof(E) * (size_t)d_h * kRouterTile);  // [d_h][kEB]
  int* hcount = reinterpret_cast<int*>(Wb + (size_t)d_h * kEB);            // [N_e]

  // Alg. 1 line 3: load X_block (sub-tokens of head h are a strided column block of Xs)
  for (int i = tid; i < N_e; i += blockDim.x) hcount[i] = 0;
  for (int e = tid; e < d_h * kRouterTile; e += blockDim.x) {
    const int r = e / d_h, c = e % d_h;
    const int64_t t = t0 + r;
    E v = from_f<E>(0.0f);
    if (t < T) v = Xs[t * ldx + (int64_t)h * d_h + c];
    Xt[c * kRouterTile + r] = v;
  }

  unsigned long long key[KMAX];
  float sraw[KMAX];
#pragma unroll
  for (int j = 0; j < KMAX; ++j) { key[j] = 0ull; sraw[j] = 0.0f; }   // line 4: A = 0 (R17)
  bool bad = false;
  const float* Wh = W_r + (size_t)h * d_h * N_e;
  const float* bh = bias + (size_t)h * N_e;

  for (int e0 = 0; e0 < N_e; e0 += kEB) {                                  // line 5
    const int eb = min(kEB, N_e - e0);
    __syncthreads();
    for (int i = tid; i < d_h * kEB; i += blockDim.x) {                    // line 6
      const int f = i / kEB, e = i % kEB;
      Wb[i] = (e < eb) ? Wh[(size_t)f * N_e + e0 + e] : 0.0f;
    }
    __syncthreads();
    float acc[kEB];
#pragma unroll
    for (int e = 0; e < kEB; ++e) acc[e] = 0.0f;
    for (int f = 0; f < d_h; ++f) {                                        // line 7 (on chip)
      const float x = to_f(Xt[f * kRouterTile + tid]);
      const float4* w4 = reinterpret_cast<const float4*>(Wb + f * kEB);
#pragma unroll
      for (int q = 0; q < kEB / 4; ++q) {
        const float4 w = w4[q];
        acc[4 * q + 0] = fmaf(x, w.x, acc[4 * q + 0]);
        acc[4 * q + 1] = fmaf(x, w.y, acc[4 * q + 1]);
        acc[4 * q + 2] = fmaf(x, w.z, acc[4 * q + 2]);
        acc[4 * q + 3] = fmaf(x, w.w, acc[4 * q + 3]);
      }
    }
#pragma unroll
    for (int e = 0; e < kEB; ++e) {
      if (e < eb) {
        const float s = acc[e];
        const float kf = s + bh[e0 + e];                                    // biased key
        bad |= !isfinite(kf);
        unsigned long long kk = pack_key(kf, e0 + e);                      // line 8
        if (kk > key[KMAX - 1]) {                                          // lines 9-10: merge
          float sv = s;
#pragma unroll
          for (int j = 0; j < KMAX; ++j) {
            const bool sw = kk > key[j];
            const unsigned long long tk = key[j];
            const float ts = sraw[j];
            key[j] = sw ? kk : tk;  sraw[j] = sw ? sv : ts;
            kk = sw ? tk : kk;      sv = sw ? ts : sv;
          }
        }
      }
    }
  }

  const int64_t t = t0 + tid;
  if (bad) *flag = 1;
  if (t < T) {
    // line 12-13: unpack; the carried raw scores already exclude the bias (R5)
    float m = sraw[0];
#pragma unroll
    for (int j = 1; j < KMAX; ++j) if (j < k) m = fmaxf(m, sraw[j]);
    float ex[KMAX];
    float sum = 0.0f;
#pragma unroll
    for (int j = 0; j < KMAX; ++j) { ex[j] = (j < k) ? expf(sraw[j] - m) : 0.0f; sum += ex[j]; }
    const float inv = 1.0f / sum;
    int32_t* io = idx + ((size_t)h * T + t) * k;
    float* go = gate + ((size_t)h * T + t) * k;
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
      if (j < k) {
        const int e = (int)(~(uint32_t)(key[j] & 0xffffffffull));
        io[j] = e;
        go[j] = ex[j] * inv;
        atomicAdd(&hcount[e], 1);   // order-free count for the clustering histogram
      }
    }
  }
  __syncthreads();
  int32_t* ho = hist + ((size_t)h * gridDim.x + tile) * N_e;
  for (int i = tid; i < N_e; i += blockDim.x) ho[i] = hcount[i];
}

template <typename E, int KMAX>
void launch_t(const void* Xs, int64_t ldx, const float* W_r, const float* bias, int H, int64_t T, int d_h,
              int N_e, int k, int32_t* idx, float* gate, int32_t* hist, int32_t* flag, cudaStream_t s) {
  const size_t smem = sizeof(E) * (size_t)d_h * kRouterTile + sizeof(float) * (size_t)d_h * kEB + sizeof(int) * N_e;
  auto kern = router_topk_kernel<E, KMAX>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((unsigned)((T + kRouterTile - 1) / kRouterTile), H);
  kern<<<grid, kRouterTile, smem, s>>>(reinterpret_cast<const E*>(Xs), ldx, W_r, bias, T, d_h, N_e, k, idx, gate,
                                       hist, flag);
}

template <typename E>
void launch_k(const void* Xs, int64_t ldx, const float* W_r, const float* bias, int H, int64_t T, int d_h,
              int N_e, int k, int32_t* idx, float* gate, int32_t* hist, int32_t* flag, cudaStream_t s) {
  if (k <= 2) launch_t<E, 2>(Xs, ldx, W_r, bias, H, T, d_h, N_e, k, idx, gate, hist, flag, s);
  else if (k <= 4) launch_t<E, 4>(Xs, ldx, W_r, bias, H, T, d_h, N_e, k, idx, gate, hist, flag, s);
  else if (k <= 8) launch_t<E, 8>(Xs, ldx, W_r, bias, H, T, d_h, N_e, k, idx, gate, hist, flag, s);
  else launch_t<E, 16>(Xs, ldx, W_r, bias, H, T, d_h, N_e, k, idx, gate, hist, flag, s);
}

}  // namespace

void launch_router_topk(int dtype, const void* Xs, int64_t ldx, const float* W_r, const float* bias, int H,
                        int64_t T, int d_h, int N_e, int k, int32_t* idx, float* gate, int32_t* hist,
                        int32_t* flag, cudaStream_t s) {
  if (dtype == 1) launch_k<bf16>(Xs, ldx, W_r, bias, H, T, d_h, N_e, k, idx, gate, hist, flag, s);
  else launch_k<float>(Xs, ldx, W_r, bias, H, T, d_h, N_e, k, idx, gate, hist, flag, s);
}

}  // namespace mhl
