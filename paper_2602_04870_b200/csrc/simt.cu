// simt.cu — CUDA-core kernels of the path: block permutes, router backward (B3), and the SIMT
// versions of the expert FFN (F5/B5) used in fp32 mode and as the bf16 cross-check path
// (MHL_FLAG_SIMT).  All work on the padded clustered layout of cluster.cu (Routing).
#include <algorithm>
#include "kernels.h"

namespace mhl {

namespace {

constexpr int kSub = 32;    // rows per SIMT sub-tile
constexpr int kRbwdChunk = 128;   // tokens per router-backward partial
constexpr int kRbwdPartialFloats = 32768;   // per-block partial tile (128 KB): expert block = this / d_h

// ---------------------------------------------------------------------------------------------
// F5 (SIMT): for one 128-row expert tile, Yrep[row] = g * gelu(x W1_e^T) W2_e      (Eq. 1)
// ---------------------------------------------------------------------------------------------
template <typename E>
__global__ void __launch_bounds__(256)
expert_fwd_simt_kernel(Routing rt, const E* __restrict__ Xs, int64_t ldx, const E* __restrict__ W1,
                       const E* __restrict__ W2, int d_h, int d_e, E* __restrict__ Yrep) {
  if ((int)blockIdx.x >= *rt.ntiles) return;
  const Tile tl = rt.tiles[blockIdx.x];
  extern __shared__ __align__(16) float sm[];
  float* Xsub = sm;                                   // [kSub][d_h+1]
  float* Asub = Xsub + kSub * (d_h + 1);              // [kSub][d_e+1]
  float* gsub = Asub + kSub * (d_e + 1);              // [kSub]
  const size_t hrow = (size_t)tl.head * rt.Rp + tl.row0;
  const size_t wofs = ((size_t)tl.head * rt.N_e + tl.expert) * d_e * d_h;
  const E* w1 = W1 + wofs;
  const E* w2 = W2 + wofs;
  for (int s0 = 0; s0 < kExpertBM; s0 += kSub) {
    __syncthreads();
    for (int o = threadIdx.x; o < kSub * d_h; o += blockDim.x) {
      const int r = o / d_h, c = o % d_h;
      Xsub[r * (d_h + 1) + c] = to_f(Xs[(int64_t)rt.tok_s[hrow + s0 + r] * ldx + (int64_t)tl.head * d_h + c]);
    }
    for (int r = threadIdx.x; r < kSub; r += blockDim.x) gsub[r] = rt.gate_s[hrow + s0 + r];
    __syncthreads();
    for (int o = threadIdx.x; o < kSub * d_e; o += blockDim.x) {
      const int r = o / d_e, f = o % d_e;
      float acc = 0.0f;
      for (int c = 0; c < d_h; ++c) acc = fmaf(Xsub[r * (d_h + 1) + c], to_f(w1[(size_t)f * d_h + c]), acc);
      Asub[r * (d_e + 1) + f] = gelu_f(acc);
    }
    __syncthreads();
    for (int o = threadIdx.x; o < kSub * d_h; o += blockDim.x) {
      const int r = o / d_h, c = o % d_h;
      float acc = 0.0f;
      for (int f = 0; f < d_e; ++f) acc = fmaf(Asub[r * (d_e + 1) + f], to_f(w2[(size_t)f * d_h + c]), acc);
      Yrep[(hrow + s0 + r) * d_h + c] = from_f<E>(gsub[r] * acc);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// B5 (SIMT): recompute H, A = gelu(H); dA' = dY W2_e^T; dg = <A, dA'> (= <dY, E_e(x)>);
// dH = g dA' gelu'(H); gA = g A; dXrep = dH W1_e.
// ---------------------------------------------------------------------------------------------
template <typename E>
__global__ void __launch_bounds__(256)
expert_bwd_simt_kernel(Routing rt, const E* __restrict__ Xs, int64_t ldx, const E* __restrict__ dY, int64_t ldy,
                       const E* __restrict__ W1, const E* __restrict__ W2, int d_h, int d_e, E* __restrict__ dXrep,
                       float* __restrict__ dg, E* __restrict__ dH, E* __restrict__ gA) {
  if ((int)blockIdx.x >= *rt.ntiles) return;
  const Tile tl = rt.tiles[blockIdx.x];
  extern __shared__ __align__(16) float sm[];
  float* Xsub = sm;                                   // [kSub][d_h+1]
  float* Ysub = Xsub + kSub * (d_h + 1);              // [kSub][d_h+1]  (dY rows)
  float* Hsub = Ysub + kSub * (d_h + 1);              // [kSub][d_e+1]
  float* Dsub = Hsub + kSub * (d_e + 1);              // [kSub][d_e+1]
  float* gsub = Dsub + kSub * (d_e + 1);              // [kSub]
  const size_t hrow = (size_t)tl.head * rt.Rp + tl.row0;
  const size_t wofs = ((size_t)tl.head * rt.N_e + tl.expert) * d_e * d_h;
  const E* w1 = W1 + wofs;
  const E* w2 = W2 + wofs;
  for (int s0 = 0; s0 < kExpertBM; s0 += kSub) {
    __syncthreads();
    for (int r = threadIdx.x; r < kSub; r += blockDim.x) gsub[r] = rt.gate_s[hrow + s0 + r];
    for (int o = threadIdx.x; o < kSub * d_h; o += blockDim.x) {
      const int r = o / d_h, c = o % d_h;
      const int64_t t = rt.tok_s[hrow + s0 + r];
      Xsub[r * (d_h + 1) + c] = to_f(Xs[t * ldx + (int64_t)tl.head * d_h + c]);
      Ysub[r * (d_h + 1) + c] = to_f(dY[t * ldy + (int64_t)tl.head * d_h + c]);
    }
    __syncthreads();
    for (int o = threadIdx.x; o < kSub * d_e; o += blockDim.x) {
      const int r = o / d_e, f = o % d_e;
      float h = 0.0f, da = 0.0f;
      for (int c = 0; c < d_h; ++c) {
        h = fmaf(Xsub[r * (d_h + 1) + c], to_f(w1[(size_t)f * d_h + c]), h);
        da = fmaf(Ysub[r * (d_h + 1) + c], to_f(w2[(size_t)f * d_h + c]), da);
      }
      Hsub[r * (d_e + 1) + f] = h; Dsub[r * (d_e + 1) + f] = da;
    }
    __syncthreads();
    // dg (one thread per row, fixed f order), then dH / gA in place
    for (int r = threadIdx.x; r < kSub; r += blockDim.x) {
      const int rep = rt.perm[hrow + s0 + r];
      if (rep < 0) continue;
      float acc = 0.0f;
      for (int f = 0; f < d_e; ++f) acc = fmaf(gelu_f(Hsub[r * (d_e + 1) + f]), Dsub[r * (d_e + 1) + f], acc);
      dg[(size_t)tl.head * rt.T * rt.k + rep] = acc;
    }
    __syncthreads();
    for (int o = threadIdx.x; o < kSub * d_e; o += blockDim.x) {
      const int r = o / d_e, f = o % d_e;
      const float h = Hsub[r * (d_e + 1) + f];
      const float g = gsub[r];
      const float dh = g * Dsub[r * (d_e + 1) + f] * gelu_grad_f(h);
      const float ga = g * gelu_f(h);
      Dsub[r * (d_e + 1) + f] = dh;
      const size_t row = hrow + s0 + r;
      dH[row * d_e + f] = from_f<E>(dh);
      gA[row * d_e + f] = from_f<E>(ga);
    }
    __syncthreads();
    for (int o = threadIdx.x; o < kSub * d_h; o += blockDim.x) {
      const int r = o / d_h, c = o % d_h;
      float acc = 0.0f;
      for (int f = 0; f < d_e; ++f) acc = fmaf(Dsub[r * (d_e + 1) + f], to_f(w1[(size_t)f * d_h + c]), acc);
      dXrep[(hrow + s0 + r) * d_h + c] = from_f<E>(acc);
    }
  }
}

// B5 weight gradients (SIMT): block (f-chunk of 8, e, h); thread = feature c; padded segment rows in
// order (padding rows have dH = gA = 0).
template <typename E>
__global__ void __launch_bounds__(256)
expert_dw_simt_kernel(Routing rt, const E* __restrict__ Xs, int64_t ldx, const E* __restrict__ dY, int64_t ldy,
                      const E* __restrict__ dH, const E* __restrict__ gA, int d_h, int d_e, float* __restrict__ dW1,
                      float* __restrict__ dW2) {
  const int f0 = blockIdx.x * 8, e = blockIdx.y, h = blockIdx.z;
  const int nf = min(8, d_e - f0);
  const int32_t* offh = rt.off + (size_t)h * (rt.N_e + 1);
  const int beg = offh[e], end = offh[e + 1];
  for (int c = threadIdx.x; c < d_h; c += blockDim.x) {
    float a1[8], a2[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) { a1[q] = 0.0f; a2[q] = 0.0f; }
    for (int row = beg; row < end; ++row) {
      const size_t hr = (size_t)h * rt.Rp + row;
      const int64_t t = rt.tok_s[hr];
      const float xv = to_f(Xs[t * ldx + (int64_t)h * d_h + c]);
      const float yv = to_f(dY[t * ldy + (int64_t)h * d_h + c]);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (q < nf) {
          a1[q] = fmaf(to_f(dH[hr * d_e + f0 + q]), xv, a1[q]);
          a2[q] = fmaf(to_f(gA[hr * d_e + f0 + q]), yv, a2[q]);
        }
      }
    }
    const size_t wofs = ((size_t)h * rt.N_e + e) * d_e * d_h;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (q < nf) {
        if (dW1) dW1[wofs + (size_t)(f0 + q) * d_h + c] = a1[q];
        if (dW2) dW2[wofs + (size_t)(f0 + q) * d_h + c] = a2[q];
      }
    }
  }
}

template <typename E>
__global__ void __launch_bounds__(256)
permute_blocks_kernel(const E* __restrict__ src, E* __restrict__ dst, int G, int64_t T_loc, int64_t HD) {
  // src [G][T_loc][HD] -> dst [T_loc][G*HD]
  const int64_t total = (int64_t)G * T_loc * HD;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i % HD;
    const int64_t t = (i / HD) % T_loc;
    const int64_t g = i / (HD * T_loc);
    dst[t * G * HD + g * HD + c] = src[i];
  }
}

// ---------------------------------------------------------------------------------------------
// B3: softmax Jacobian + Alg. 2 (P:846-P:866), deterministic (R21).
// Block = (128-token chunk, head); thread = feature i.
//   dS[t][j] = g_j (dg_j - sum_i g_i dg_i)
//   partial[e][i] = sum_{t in chunk, j: I[t][j]=e} X[t][i] dS[t][j]    (fixed t, j order)
// ---------------------------------------------------------------------------------------------
template <typename E>
__global__ void __launch_bounds__(256)
router_bwd_partial_kernel(const E* __restrict__ Xs, int64_t ldx, const int32_t* __restrict__ idx,
                          const float* __restrict__ gate, const float* __restrict__ dg, int64_t T, int k, int d_h,
                          int N_e, int eblk, float* __restrict__ dS, float* __restrict__ partial) {
  // blockIdx.z selects the expert block [e0, e0 + eblk) whose partial sums this block owns (large
  // N_e: the paper's own 384-1536 experts per head do not fit one block's shared memory)
  extern __shared__ __align__(16) float smb[];
  const int e0 = blockIdx.z * eblk, ne = min(eblk, N_e - e0);
  float* part = smb;                                  // [ne][d_h]
  float* sdS = part + (size_t)eblk * d_h;             // [128][k]
  int* sI = reinterpret_cast<int*>(sdS + kRbwdChunk * k);   // [128][k]
  const int chunk = blockIdx.x, h = blockIdx.y;
  const int64_t t0 = (int64_t)chunk * kRbwdChunk;
  const int nt = (int)min((int64_t)kRbwdChunk, T - t0);
  for (int i = threadIdx.x; i < ne * d_h; i += blockDim.x) part[i] = 0.0f;
  for (int tt = threadIdx.x; tt < nt; tt += blockDim.x) {
    const size_t base = ((size_t)h * T + t0 + tt) * k;
    float s = 0.0f;
    for (int j = 0; j < k; ++j) s = fmaf(gate[base + j], dg[base + j], s);
    for (int j = 0; j < k; ++j) {
      const float v = gate[base + j] * (dg[base + j] - s);
      sdS[tt * k + j] = v;
      sI[tt * k + j] = idx[base + j] - e0;
      if (blockIdx.z == 0) dS[base + j] = v;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < d_h; i += blockDim.x) {
    for (int tt = 0; tt < nt; ++tt) {
      const float xv = to_f(Xs[(t0 + tt) * ldx + (int64_t)h * d_h + i]);
      for (int j = 0; j < k; ++j) {
        const int e = sI[tt * k + j];
        if (e >= 0 && e < ne) part[(size_t)e * d_h + i] = fmaf(xv, sdS[tt * k + j], part[(size_t)e * d_h + i]);
      }
    }
  }
  __syncthreads();
  float* po = partial + (((size_t)h * gridDim.x + chunk) * N_e + e0) * d_h;
  for (int i = threadIdx.x; i < ne * d_h; i += blockDim.x) po[i] = part[i];
}

// dW_r[h][i][e] = sum over chunks (in order) of partial[h][chunk][e][i]
__global__ void __launch_bounds__(256)
router_bwd_reduce_kernel(const float* __restrict__ partial, int n_chunks, int d_h, int N_e, float* __restrict__ dW_r) {
  const int h = blockIdx.y;
  const int64_t n = (int64_t)d_h * N_e;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(o / d_h), i = (int)(o % d_h);
    float acc = 0.0f;
    for (int c = 0; c < n_chunks; ++c) acc += partial[(((size_t)h * n_chunks + c) * N_e + e) * d_h + i];
    dW_r[((size_t)h * d_h + i) * N_e + e] = acc;
  }
}

__global__ void transpose_wr_kernel(const float* __restrict__ W_r, float* __restrict__ W_rT, int d_h, int N_e) {
  const int h = blockIdx.y;
  const int n = d_h * N_e;
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < n; o += gridDim.x * blockDim.x) {
    const int e = o / d_h, i = o % d_h;
    W_rT[(size_t)h * n + o] = W_r[(size_t)h * n + (size_t)i * N_e + e];
  }
}

template <typename F>
void set_smem(F f, size_t bytes) { cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes); }

}  // namespace

void launch_expert_fwd_simt(int dtype, const Routing& rt, const void* Xs, int64_t ldx, const void* W1, const void* W2,
                            int d_h, int d_e, void* Yrep, cudaStream_t s) {
  const size_t smem = sizeof(float) * (kSub * (d_h + 1) + kSub * (d_e + 1) + kSub);
  if (dtype == 1) {
    auto f = expert_fwd_simt_kernel<bf16>; set_smem(f, smem);
    f<<<rt.max_tiles, 256, smem, s>>>(rt, (const bf16*)Xs, ldx, (const bf16*)W1, (const bf16*)W2, d_h, d_e,
                                      (bf16*)Yrep);
  } else {
    auto f = expert_fwd_simt_kernel<float>; set_smem(f, smem);
    f<<<rt.max_tiles, 256, smem, s>>>(rt, (const float*)Xs, ldx, (const float*)W1, (const float*)W2, d_h, d_e,
                                      (float*)Yrep);
  }
}

void launch_expert_bwd_simt(int dtype, const Routing& rt, const void* Xs, int64_t ldx, const void* dY, int64_t ldy,
                            const void* W1, const void* W2, int d_h, int d_e, void* dXrep, float* dg, void* dH,
                            void* gA, cudaStream_t s) {
  const size_t smem = sizeof(float) * (2 * kSub * (d_h + 1) + 2 * kSub * (d_e + 1) + kSub);
  if (dtype == 1) {
    auto f = expert_bwd_simt_kernel<bf16>; set_smem(f, smem);
    f<<<rt.max_tiles, 256, smem, s>>>(rt, (const bf16*)Xs, ldx, (const bf16*)dY, ldy, (const bf16*)W1,
                                      (const bf16*)W2, d_h, d_e, (bf16*)dXrep, dg, (bf16*)dH, (bf16*)gA);
  } else {
    auto f = expert_bwd_simt_kernel<float>; set_smem(f, smem);
    f<<<rt.max_tiles, 256, smem, s>>>(rt, (const float*)Xs, ldx, (const float*)dY, ldy, (const float*)W1,
                                      (const float*)W2, d_h, d_e, (float*)dXrep, dg, (float*)dH, (float*)gA);
  }
}

void launch_expert_dw_simt(int dtype, const Routing& rt, const void* Xs, int64_t ldx, const void* dY, int64_t ldy,
                           const void* dH, const void* gA, int d_h, int d_e, float* dW1, float* dW2, cudaStream_t s) {
  dim3 grid((d_e + 7) / 8, rt.N_e, rt.H);
  const int threads = d_h >= 256 ? 256 : ((d_h + 31) / 32) * 32;
  if (dtype == 1)
    expert_dw_simt_kernel<bf16><<<grid, threads, 0, s>>>(rt, (const bf16*)Xs, ldx, (const bf16*)dY, ldy,
                                                         (const bf16*)dH, (const bf16*)gA, d_h, d_e, dW1, dW2);
  else
    expert_dw_simt_kernel<float><<<grid, threads, 0, s>>>(rt, (const float*)Xs, ldx, (const float*)dY, ldy,
                                                          (const float*)dH, (const float*)gA, d_h, d_e, dW1, dW2);
}

// HP block placement (F7 / B2 receive side): rows x row_bytes, 16 bytes per thread per step.
__global__ void __launch_bounds__(256)
copy_rows_kernel(const uint4* __restrict__ src, int64_t sp, uint4* __restrict__ dst, int64_t dp, int64_t rows, int64_t w) {
  const int64_t total = rows * w;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / w, c = i - r * w;
    dst[r * dp + c] = src[r * sp + c];
  }
}

void launch_copy_rows(const void* src, int64_t sp, void* dst, int64_t dp, int64_t rows, int64_t row_bytes, cudaStream_t s) {
  const int64_t w = row_bytes / 16, total = rows * w;
  if (total <= 0) return;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
  copy_rows_kernel<<<blocks, 256, 0, s>>>((const uint4*)src, sp / 16, (uint4*)dst, dp / 16, rows, w);
}

// dS in sorted-row order for the router term fused into the dX GEMM (K2)
__global__ void __launch_bounds__(256)
sort_ds_kernel(const float* __restrict__ dS, const int32_t* __restrict__ pos, int64_t R, int64_t Rp, int H,
               float* __restrict__ dS_s) {
  const int64_t total = (int64_t)H * R;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t h = i / R;
    dS_s[h * Rp + pos[i]] = dS[i];
  }
}

void launch_sort_ds(const Routing& rt, const float* dS, float* dS_s, cudaStream_t s) {
  const int64_t total = (int64_t)rt.H * rt.T * rt.k;
  if (total <= 0) return;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
  sort_ds_kernel<<<blocks, 256, 0, s>>>(dS, rt.pos, rt.T * rt.k, rt.Rp, rt.H, dS_s);
}

void launch_permute_blocks(int dtype, const void* src, void* dst, int G, int64_t T_loc, int64_t HD, cudaStream_t s) {
  const int64_t total = (int64_t)G * T_loc * HD;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  if (dtype == 1)
    permute_blocks_kernel<bf16><<<blocks, 256, 0, s>>>((const bf16*)src, (bf16*)dst, G, T_loc, HD);
  else
    permute_blocks_kernel<float><<<blocks, 256, 0, s>>>((const float*)src, (float*)dst, G, T_loc, HD);
}

void launch_router_bwd(int dtype, const void* Xs, int64_t ldx, const int32_t* idx, const float* gate, const float* dg,
                       int H, int64_t T, int k, int d_h, int N_e, float* dS, float* dwr_partial, float* dW_r,
                       cudaStream_t s) {
  const int n_chunks = (int)((T + kRbwdChunk - 1) / kRbwdChunk);
  const int eblk = std::min(N_e, std::max(1, kRbwdPartialFloats / d_h));   // experts per block
  const size_t smem = sizeof(float) * ((size_t)eblk * d_h + (size_t)kRbwdChunk * k) + sizeof(int) * kRbwdChunk * k;
  const int threads = d_h >= 256 ? 256 : ((d_h + 31) / 32) * 32;
  dim3 grid(n_chunks, H, (N_e + eblk - 1) / eblk);
  if (dtype == 1) {
    auto f = router_bwd_partial_kernel<bf16>; set_smem(f, smem);
    f<<<grid, threads, smem, s>>>((const bf16*)Xs, ldx, idx, gate, dg, T, k, d_h, N_e, eblk, dS, dwr_partial);
  } else {
    auto f = router_bwd_partial_kernel<float>; set_smem(f, smem);
    f<<<grid, threads, smem, s>>>((const float*)Xs, ldx, idx, gate, dg, T, k, d_h, N_e, eblk, dS, dwr_partial);
  }
  if (dW_r) router_bwd_reduce_kernel<<<dim3(std::max(1, d_h * N_e / 256), H), 256, 0, s>>>(dwr_partial, n_chunks, d_h, N_e, dW_r);
}

void launch_transpose_wr(const float* W_r, float* W_rT, int H, int d_h, int N_e, cudaStream_t s) {
  transpose_wr_kernel<<<dim3(std::max(1, d_h * N_e / 256), H), 256, 0, s>>>(W_r, W_rT, d_h, N_e);
}

}  // namespace mhl
