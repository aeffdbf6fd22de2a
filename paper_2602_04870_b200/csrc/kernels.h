// kernels.h — internal (non-ABI) launch interface of the kernel translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "common.cuh"

namespace mhl {

constexpr int kRouterTile = 128;   // tokens per router CTA (= clustering tile of F4)
constexpr int kExpertBM = 128;     // replica rows per expert tile (tcgen05 M)
// Expert segments are padded to a multiple of Routing::seg_align rows: one tile (128, default) or a
// tile pair (256, MHL_FLAG_PAIR), which the cta_group::2 kernels need (tiles 2u, 2u+1 share an expert).
constexpr int kDwStep = 64;        // sorted rows per dW pipeline step (dW chunk boundaries align to it)
// dW row parts per head (= the dW grid).  A constant of the decomposition, NOT the device's SM count:
// part boundaries fix the order of the dW partial sums, so dW1/dW2 bits must not depend on the device
// (§8(e)).  148 = one part per B200 SM; a device with fewer SMs runs the grid in waves, same bits.
constexpr int kDwParts = 148;
#ifndef MHL_TILE_GROUP
#define MHL_TILE_GROUP 8
#endif
constexpr int kTileGroup = MHL_TILE_GROUP;   // consecutive expert tiles a persistent CTA takes at once
#ifndef MHL_TILE_PARTS
#define MHL_TILE_PARTS 8
#endif
constexpr int kTileParts = MHL_TILE_PARTS;   // token-order parts per expert segment in the tile list (cluster.cu)

// Clustered routing of one rank's local heads (F3/F4 outputs, device pointers).
// Sorted-row arrays have a fixed per-head capacity Rp = T*k + N_e*seg_align (expert segments are
// padded to whole tiles or tile pairs; padding rows: perm -1, tok_s = T (the all-zero row), gate_s 0).
struct Routing {
  int H; int64_t T; int k; int N_e; int64_t Rp;
  int seg_align;           // expert segments padded to a multiple of this many rows (128 or 256)
  const int32_t* idx;      // [H][T][k]  expert ids, slot order = descending biased key
  const float* gate;       // [H][T][k]
  const int32_t* perm;     // [H][Rp]    sorted row -> replica t*k+j, or -1
  const int32_t* tok_s;    // [H][Rp]    sorted row -> token, or T
  const float* gate_s;     // [H][Rp]    sorted row -> gate, or 0
  const int32_t* pos;      // [H][T*k]   replica -> sorted row
  const int32_t* off;      // [H][N_e+1] padded segment offsets
  const Tile* tiles; const int32_t* ntiles; int max_tiles;        // 128-row tiles, (h, part, e, row) order
  const Tile* chunks; const int32_t* nchunks; int max_chunks;     // dW chunks
  const int32_t* cbase; const int32_t* ccount;                    // [H][N_e] chunk range per expert
  const int32_t* pbase; const int32_t* pcount; int dw_parts;       // [H][dw_parts] chunk range per (head, part)
  // optional tile window: the expert kernels then take only tiles [trange[0], trange[1]) (device
  // pointer; nullptr = every tile).  Used by the L2-resident windowed combine (NEXT-1, capi.cpp).
  const int32_t* trange = nullptr;
};

// Token windows of the windowed combine (NEXT-1): each head's tile list is cut into kWinParts
// consecutive token-order parts per window; win[(h * kWindows + w) * 4 + {0,1,2,3}] = tile range
// [lo, hi) and token range [lo, hi) of window w of head h (every replica of a token in the token
// range lies in the window's tiles or earlier ones of the same head).
constexpr int kWinParts = 2;
constexpr int kWindows = MHL_TILE_PARTS / kWinParts;
void launch_windows(int H, int N_e, int64_t T, int64_t Rp, int seg_align, const int32_t* counts, const int32_t* off,
                    const int32_t* tilepref, int n_rt, const int32_t* ntiles, const int32_t* tok_s, int32_t* win,
                    cudaStream_t s);
// F6 / B6 of one window: the k-row sum for head h's tokens [tr[0], tr[1]) (device pointer), written
// to output row t (absolute); with `discard` every replica row read is dropped from L2 afterwards
// (discard.global.L2: it is never read again, so it need not be written back to HBM).
void launch_combine_window(int dtype, const Routing& rt, const void* rep, int d_h, void* out, int64_t ldo, int h,
                           const int32_t* tr, int64_t max_tokens, bool discard, cudaStream_t s);

// ---- F3: router + online top-k + gates (SIMT fp32-FMA path). idx/gate [H][T][k];
// hist [H][ceil(T/128)][N_e]; flag set to 1 on a non-finite key.
void launch_router_topk(int dtype, const void* Xs, int64_t ldx, const float* W_r, const float* bias,
                        int H, int64_t T, int d_h, int N_e, int k, int32_t* idx, float* gate,
                        int32_t* hist, int32_t* flag, cudaStream_t s);

// ---- F3 on tcgen05 (bf16 only): splits W_r into 3 bf16 planes (scratch `planes`,
// router_sm100_planes_bytes) then runs the TMA/tcgen05 router.  Returns false if the tensor
// maps cannot be built.
bool router_sm100_supported(int d_h, int N_e);
size_t router_sm100_planes_bytes(int H, int d_h, int N_e);
bool launch_router_sm100(const void* Xs, int64_t ldx, const float* W_r, const float* bias, int H, int64_t T, int d_h,
                         int N_e, int k, void* planes, int32_t* idx, float* gate, int32_t* hist, int32_t* flag,
                         int num_sms, cudaStream_t s);

// ---- F3 for many experts (Alg. 1 over 64-expert blocks streamed through smem, d_h = 128):
// W_r split into planes by launch_router_split first
void launch_router_split(const float* W_r, void* planes, int H, int d_h, int N_e, cudaStream_t s);
bool router_blk_supported(int d_h, int N_e, int k);
bool launch_router_blk_sm100(const void* Xs, int64_t ldx, const void* planes, const float* bias, int H, int64_t T,
                             int d_h, int N_e, int k, int32_t* idx, float* gate, int32_t* hist, int32_t* flag,
                             int num_sms, cudaStream_t s);

// ---- F4: clustering.  tilepref [H][n_rt][N_e] is scratch; counts [H][N_e] receives the expert loads.
void launch_cluster(int H, int64_t T, int k, int N_e, const int32_t* idx, const float* gate, const int32_t* hist,
                    int32_t* tilepref, int32_t* counts, int32_t* off, int32_t* perm, int32_t* pos, int32_t* tok_s,
                    float* gate_s, int64_t Rp, int seg_align, Tile* tiles, int32_t* ntiles, int max_tiles,
                    Tile* chunks, int32_t* nchunks, int32_t* cbase, int32_t* ccount, int max_chunks, int dw_parts,
                    int32_t* pbase, int32_t* pcount, cudaStream_t s);

// ---- F5: Yrep[h][row][c] = gate_s * gelu(X[tok_s] W1_e^T) W2_e for every sorted row (padding rows
// produce zeros).  Xs holds T+1 rows, row T all-zero.  Yrep is [H][Rp][d_h].
void launch_expert_fwd_simt(int dtype, const Routing& rt, const void* Xs, int64_t ldx, const void* W1, const void* W2,
                            int d_h, int d_e, void* Yrep, cudaStream_t s);
bool expert_fwd_sm100_supported(int d_h, int d_e);
// the dW kernel's row-part chunks of a clustered routing (launch_cluster with dw_parts = 0 leaves
// them to this call, which the backward makes: a forward-only step does not pay for them)
void launch_dw_parts(const Routing& rt, Tile* chunks, int32_t* nchunks, int32_t* cbase, int32_t* ccount,
                     int32_t* pbase, int32_t* pcount, cudaStream_t s);

bool launch_expert_fwd_sm100(const Routing& rt, const void* Xs, int64_t ldx, const void* W1, const void* W2, int d_h,
                             int d_e, void* Yrep, int num_sms, cudaStream_t s);
// the same on CTA pairs (tcgen05 cta_group::2, half of each weight matrix per CTA)
bool expert_fwd_pair_supported(int d_h, int d_e);
bool launch_expert_fwd_pair_sm100(const Routing& rt, const void* Xs, int64_t ldx, const void* W1, const void* W2,
                                  int d_h, int d_e, void* Yrep, int num_sms, cudaStream_t s);

// ---- aux-free load balancing (NEXT-2): bias[h][e] -= gamma * sign(load[h][e]*N_e - total), with
// total = T*k the replicas per head (exact integer comparison with the mean load)
void launch_update_bias(const int32_t* load, int H, int N_e, int64_t total, float gamma, float* bias,
                        cudaStream_t s);

// ---- F6: y[t][h*d_h+c] = sum_j Yrep[h][pos[h][t*k+j]][c]  (fixed j order), out ld = ldo.
// tokens [t0, t0 + nT) (nT < 0: to the end), written to output rows 0.. (one HP destination block)
void launch_combine_fwd(int dtype, const Routing& rt, const void* Yrep, int d_h, void* out, int64_t ldo,
                        cudaStream_t s, int64_t t0 = 0, int64_t nT = -1);

// ---- deterministic DP tree step: dst[i] += src[i], n floats (a multiple of 4)
void launch_add_inplace(float* dst, const float* src, int64_t n, cudaStream_t s);

// ---- fault injection: p[i] *= f (dtype 1 = bf16, else fp32)
void launch_scale(int dtype, void* p, int64_t n, float f, cudaStream_t s);

// ---- [G][T_loc][HD] -> [T_loc][G*HD]
void launch_permute_blocks(int dtype, const void* src, void* dst, int G, int64_t T_loc, int64_t HD, cudaStream_t s);
// ---- rows x row_bytes from src (pitch sp) to dst (pitch dp); 16-byte aligned (HP block placement)
void launch_copy_rows(const void* src, int64_t sp, void* dst, int64_t dp, int64_t rows, int64_t row_bytes, cudaStream_t s);

// ---- B5: per sorted row dXrep [H][Rp][d_h], dH / gA [H][Rp][d_e] (zero on padding rows) and the
// gate cotangent dg [H][T*k] (replica order); dY holds T+1 rows, row T all-zero.
void launch_expert_bwd_simt(int dtype, const Routing& rt, const void* Xs, int64_t ldx, const void* dY, int64_t ldy,
                            const void* W1, const void* W2, int d_h, int d_e, void* dXrep, float* dg, void* dH,
                            void* gA, cudaStream_t s);
void launch_expert_dw_simt(int dtype, const Routing& rt, const void* Xs, int64_t ldx, const void* dY, int64_t ldy,
                           const void* dH, const void* gA, int d_h, int d_e, float* dW1, float* dW2, cudaStream_t s);
bool expert_bwd_sm100_supported(int d_h, int d_e);
// H/dA' recompute -> dH, gA, dg (pipelined warp-specialized kernel, expert_bwd_dx_sm100.cu)
bool launch_expert_bwd_dx_sm100(const Routing& rt, const void* Xs, int64_t ldx, const void* dY, int64_t ldy,
                                const void* W1, const void* W2, int d_h, int d_e, void* dXrep, float* dg, void* dH,
                                void* gA, int num_sms, cudaStream_t s);
// dXrep = dH W1_e (+ dS_s[h][row] W_rT[h][e] when dS_s != nullptr: the router term of Alg. 2 l.9,
// dS_s = dS in sorted-row order [H][Rp], see launch_sort_ds) per expert tile (expert_bwd_dx_sm100.cu)
bool launch_expert_dx_gemm_sm100(const Routing& rt, const void* W1, int d_h, int d_e, const void* dH, void* dXrep,
                                 const float* dS, const float* W_rT, int num_sms, cudaStream_t s);
// ONE tcgen05 kernel for the input side of B5 (expert_bwd_fused_sm100.cu): H, dA' recomputed,
// dg, dH / gA (the dW kernel's inputs) and dXrep = dH W1_e WITHOUT the router term (B6 adds it,
// launch_combine_bwd).  Shapes with 2 d_e + d_h <= 512 TMEM columns.
bool expert_bwd_fused_supported(int d_h, int d_e);
bool launch_expert_bwd_fused_sm100(const Routing& rt, const void* Xs, int64_t ldx, const void* dY, int64_t ldy,
                                   const void* W1, const void* W2, int d_h, int d_e, void* dXrep, float* dg, void* dH,
                                   void* gA, int num_sms, cudaStream_t s);
// tcgen05 dX kernel (dXrep, dg, dH, gA) and/or dW kernel (chunk partials + in-kernel ordered
// reduce; `done` = H*N_e int counters, zeroed by the launch)
bool launch_expert_bwd_sm100(const Routing& rt, const void* Xs, int64_t ldx, const void* dY, int64_t ldy,
                             const void* W1, const void* W2, int d_h, int d_e, void* dXrep, float* dg, void* dH,
                             void* gA, float* partial, int* done, float* dW1, float* dW2, int num_sms,
                             cudaStream_t s, bool do_dx, bool do_dw);

// ---- B3: dS = g (dg - sum g dg); dW_r partials per 128-token chunk; then ordered reduce.
void launch_router_bwd(int dtype, const void* Xs, int64_t ldx, const int32_t* idx, const float* gate,
                       const float* dg, int H, int64_t T, int k, int d_h, int N_e, float* dS,
                       float* dwr_partial, float* dW_r, cudaStream_t s);

// ---- B3 on tcgen05 (bf16): same dS; dW_r = X_h^T dS_dense with dS split into two bf16 planes,
// one fp32 partial per CTA (min(nc_target, ceil(T/64)) token chunks per head; partial holds
// H * nc_target * d_h * N_e floats), then an ordered sum.
bool router_bwd_sm100_supported(int d_h, int N_e, int k);
bool launch_router_bwd_sm100(const void* Xs, int64_t ldx, const int32_t* idx, const float* gate, const float* dg,
                             int H, int64_t T, int k, int d_h, int N_e, float* dS, float* partial, int nc_target,
                             float* dW_r, cudaStream_t s);

// ---- dS_s[h][pos(t,j)] = dS[h][t][j] (padding rows untouched: their dXrep rows are never read)
void launch_sort_ds(const Routing& rt, const float* dS, float* dS_s, cudaStream_t s);

// ---- W_rT[h][e][i] = W_r[h][i][e]
void launch_transpose_wr(const float* W_r, float* W_rT, int H, int d_h, int N_e, cudaStream_t s);

// ---- B6: dXs[t][h*d_h+c] = sum_j dXrep[h][pos][c] + sum_j dS[h][t][j] * W_rT[h][idx][c]
void launch_combine_bwd(int dtype, const Routing& rt, const void* dXrep, const float* dS, const float* W_rT, int d_h,
                        void* out, int64_t ldo, cudaStream_t s, int64_t t0 = 0, int64_t nT = -1);

}  // namespace mhl
