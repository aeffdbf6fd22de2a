/*
 * mhlmoe.h — C ABI of the B200-native Multi-Head LatentMoE layer under Head Parallel.
 *
 * Paper: arxiv 2602.04870.  "P:n" cites line n of the paper's LaTeX;
 * "R#" cites a reading in DESIGN.md §2.
 *
 * Conventions for every entry point:
 *   - All tensors are ROW-MAJOR, contiguous, and (unless stated) DEVICE pointers
 *     on the current CUDA device.  "E" denotes the plan's element type:
 *     bfloat16 (MHL_BF16) or float32 (MHL_F32).  Router weights/bias and every
 *     weight gradient are float32.
 *   - The caller owns every buffer (inputs, outputs, `saved`, `workspace`).
 *     Sizes come from hp_plan_query / hp_plan_info.  The library never
 *     allocates device memory inside forward/backward.
 *   - Calls are asynchronous on `stream` (a cudaStream_t passed as void*).
 *     Buffers must stay alive until the stream work completes.
 *   - Errors: argument/config validation is synchronous, before any launch.
 *     A non-OK status leaves a thread-local detail string in mhl_last_error().
 *   - Notation: T_loc = tokens of THIS rank (B*T of P:804, flattened b-major,
 *     R20); G = HP degree (the paper's P); H_loc = N_h/G heads owned by this
 *     rank (contiguous block, R12); T_glob = G*T_loc; D = N_h*d_h; R = T_glob*k.
 */
#ifndef MHLMOE_H_
#define MHLMOE_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define MHL_API __attribute__((visibility("default")))
#else
#define MHL_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MHL_OK = 0,
  MHL_ERR_INVALID_ARGUMENT = 1,   /* NULL pointer, bad handle                                   */
  MHL_ERR_CONFIG = 2,             /* k<1, k>N_e, G>N_h or N_h%G!=0, dims<=0     */
  MHL_ERR_WORKSPACE_TOO_SMALL = 3,
  MHL_ERR_UNSUPPORTED = 4,        /* shape/alignment the kernels do not support                 */
  MHL_ERR_CUDA = 5,               /* CUDA runtime / cuBLAS failure (detail in mhl_last_error)   */
  MHL_ERR_NCCL = 6,               /* NCCL failure or NCCL library not loadable                  */
  MHL_ERR_NONFINITE = 7           /* a router score / biased key was NaN or Inf (R7)            */
} mhl_status;

typedef enum { MHL_F32 = 0, MHL_BF16 = 1 } mhl_dtype;

/* plan flags */
#define MHL_FLAG_LOOPBACK 1u  /* G "virtual ranks" on ONE device; NCCL replaced by device copies.
                                 forward/backward then take the WHOLE global problem (see below). */
#define MHL_FLAG_SIMT     2u  /* bf16 mode: run the SIMT reference kernels instead of the
                                 tcgen05 kernels (debug/cross-check path; fp32 mode always SIMT). */
#define MHL_FLAG_PAIR     4u  /* bf16: CTA-pair (tcgen05 cta_group::2) expert kernels; expert
                                 segments are then padded to 256-row tile pairs   */
#define MHL_FLAG_ROUTING_TOKENS 8u  /* separate routing sub-tokens (ablation, P:1565-P:1570):
                                 [x_t1..x_tNh, r_t1..r_tNh] = split(W_in x_t), W_in is [2D, d];
                                 head i routes on r_ti and runs its experts on x_ti.  The HP
                                 scatter (and its backward mirror) carries both: twice the bytes
                                 (P:1570); dW_in is [2D, d]. */
#define MHL_FLAG_FUSED_COMBINE 16u  /* REMOVED (round 2): the in-kernel forward combine experiment
                                 measured slower than the separate pass; hp_plan / hp_plan_query
                                 return MHL_ERR_UNSUPPORTED for it. */

#define MHL_FLAG_WINDOWED_COMBINE 32u  /* G = 1, bf16 tensor-core path (NEXT-1 experiment, opt-in): the
                                 expert kernel and the combine alternate per token window (2 of
                                 the 8 token-order parts of one head), each window's per-replica
                                 rows (Yrep, dXrep) combined while L2-resident and then discarded
                                 from L2.  Same bits as the default; measured slower (the extra
                                 launches cost more than the HBM round trip they save). */

#define MHL_FLAG_DET_DP   64u  /* deterministic data-parallel weight gradients: dW_in and
                                 dW_out are formed from fixed 8192-token chunk partials (global
                                 token order) summed by a fixed pairwise tree, so with
                                 mhl_dp_reduce they are bitwise identical at every G (T_loc a
                                 multiple of 8192 with a power-of-two chunk count, G a power of
                                 two; else MHL_ERR_UNSUPPORTED).  Without LOOPBACK the backward
                                 returns the rank's subtree; mhl_dp_reduce finishes the tree. */

#define MHL_FLAG_REQUIRE_TC 128u  /* bf16: refuse (MHL_ERR_UNSUPPORTED at hp_plan / hp_plan_query) any
                                 shape for which a step would fall back from its tcgen05 kernel to
                                 the SIMT reference kernel (router, router backward, expert forward
                                 or backward); without it such shapes run, and mhl_kernel_paths
                                 tells which path ran. */
#define MHL_FLAG_BWD_FUSED 256u  /* bf16: run B5's input side (H, dA' -> dg, dH, gA; dX = dH W1) as ONE
                                 tcgen05 kernel (expert_bwd_fused_sm100.cu) with the router term of
                                 dX added by B6, instead of the default two kernels (shapes with
                                 2 d_expert + d_head <= 512; same dg, dH, gA, dW bits; measured
                                 equal step time at paper scale). */

/* Layer + HP configuration (the paper's problem statement: P:496). */
typedef struct {
  int64_t tokens;        /* T_loc: tokens on this rank (B*T of P:804)                             */
  int32_t d_model;       /* d                                                                     */
  int32_t n_heads;       /* N_h                                                                   */
  int32_t d_head;        /* d_h  (N_h*d_h == d is common practice, not required: P:768)           */
  int32_t n_experts;     /* N_e PER HEAD (R14)                                                    */
  int32_t top_k;         /* k, 1 <= k <= N_e                                                      */
  int32_t d_expert;      /* d_e                                                                   */
  int32_t dtype;         /* mhl_dtype                                                             */
  int32_t world_size;    /* G = the paper's P; P <= N_h and N_h % P == 0                 */
  int32_t rank;          /* this rank (ignored with MHL_FLAG_LOOPBACK)                            */
  uint32_t flags;        /* MHL_FLAG_*                                                            */
} mhl_config;

/* Sizes and HP facts of a plan.  Everything here is independent of k's
 * routing decisions; a2a bytes are independent of k altogether (P:811-P:812). */
typedef struct {
  int32_t head_begin, head_end;     /* local heads [head_begin, head_end) of this rank (R12)      */
  int64_t tokens_global;            /* T_glob = G*T_loc                                           */
  uint64_t a2a_bytes_per_peer;      /* the scatter all-to-all, one (src,dst) pair: T_loc*H_loc*d_h*el
                                       (x2 with MHL_FLAG_ROUTING_TOKENS; the gather is always 1x) */
  uint64_t a2a_bytes_per_rank;      /* one all-to-all, sent by one rank: per_peer*(G-1)           */
  uint64_t saved_bytes;             /* forward -> backward state                                  */
  uint64_t workspace_bytes;         /* scratch for forward and for backward                       */
  uint64_t io_bytes;                /* device staging needed by mhlmoe_train_step_host            */
  int32_t max_tiles;                /* upper bound on expert tiles per rank (diagnostic)          */
} mhl_plan_info;

typedef struct mhl_plan_s* mhl_plan;

/* Device weights.  Without LOOPBACK the router/expert tensors hold only the
 * rank's LOCAL heads (HP shards experts like EP); with LOOPBACK all N_h. */
typedef struct {
  const void*  W_in;   /* [D, d]  E      Eq. 5 (x_t -> W_in x_t), P:765  ([2D, d] with ROUTING_TOKENS) */
  const void*  W_out;  /* [d, D]  E      Eq. 6                                            */
  const float* W_r;    /* [H, d_h, N_e] f32  router (Alg. 1 REQUIRE; FP32 P:521)          */
  const float* bias;   /* [H, N_e] f32   aux-free load-balancing bias, selection only    */
  const void*  W1;     /* [H, N_e, d_e, d_h] E   expert e: gelu(x W1_e^T) W2_e (R2)       */
  const void*  W2;     /* [H, N_e, d_e, d_h] E                                                   */
} mhl_weights;

/* Device gradients (float32, overwritten).  dW_in/dW_out are rank-partial sums
 * over the rank's tokens (the DP reduction belongs to the caller, R19);
 * dW_r/dW1/dW2 are complete for the local heads (each rank owns all tokens of
 * its heads).  There is no bias gradient (R13).  Any pointer may be NULL to skip. */
typedef struct {
  float* dW_in;   /* [D, d]  ([2D, d] with MHL_FLAG_ROUTING_TOKENS) */
  float* dW_out;  /* [d, D]            */
  float* dW_r;    /* [H, d_h, N_e]     */
  float* dW1;     /* [H, N_e, d_e, d_h]*/
  float* dW2;     /* [H, N_e, d_e, d_h]*/
} mhl_grads;

/* Pure host: validate `cfg` and fill `info` (no CUDA, no NCCL).
 * Errors: MHL_ERR_INVALID_ARGUMENT (NULL), MHL_ERR_CONFIG, MHL_ERR_UNSUPPORTED. */
MHL_API mhl_status hp_plan_query(const mhl_config* cfg, mhl_plan_info* info);

/* NCCL bootstrap: rank 0 calls this, broadcasts the 128 bytes (torch.distributed),
 * every rank passes them to hp_plan.  Errors: MHL_ERR_NCCL. */
MHL_API mhl_status mhl_get_unique_id(uint8_t id[128]);

/* Create a plan on the current device: validates cfg, creates the cuBLAS handle,
 * events and (G>1 without LOOPBACK) the NCCL communicator from `nccl_id`.
 * `nccl_id` must be NULL iff G == 1 or LOOPBACK.  Collective over ranks when G>1.
 * Head Parallel partitioning (P:801-P:806): rank p owns heads [p*N_h/G, (p+1)*N_h/G). */
MHL_API mhl_status hp_plan(const mhl_config* cfg, const uint8_t* nccl_id, mhl_plan* plan);
MHL_API mhl_status hp_plan_info(mhl_plan plan, mhl_plan_info* info);
MHL_API mhl_status hp_plan_destroy(mhl_plan plan);

/* Forward of the layer (Eq. 5-6, P:763-P:775) under HP:
 *   F1 Xs = x W_in^T (split into N_h sub-tokens)          Eq. 5
 *   F2 all-to-all #1 -> every sub-token of the local heads  P:801-P:805
 *   F3 per head: fp32 router scores, biased top-k (ties to the lower index),
 *      gates = softmax of the k unbiased scores              Eq. 2-4, Alg. 1, P:885-P:886
 *   F4 clustering (stable counting sort by expert)          Fig. 2, P:941-P:972
 *   F5 block-sparse expert FFN, gated                        P:916-P:978
 *   F6 combine sum_j (Eq. 1) -> F7 all-to-all #2 -> F8 out = W_out concat  Eq. 6
 * x:   [T_loc, d] E  (LOOPBACK: [G*T_loc, d], the global batch, rank-major)
 * out: [T_loc, d] E  (LOOPBACK: [G*T_loc, d])
 * saved: saved_bytes, written here, read by mhlmoe_backward.  It begins with Xs
 *        [T_glob][H_loc*d_h] E (x2 columns with routing sub-tokens), the all-to-all #1
 *        receive buffer (R12 layout), which callers may read (e.g. conformance tests).
 * topk_idx (nullable): [H_loc, T_glob, k] int32 expert ids, slot order = descending biased key.
 * gates    (nullable): [H_loc, T_glob, k] f32.  (LOOPBACK: [N_h, T_glob, k].)
 * Token order of T_glob is global: source rank-major (R12).
 * Errors: MHL_ERR_WORKSPACE_TOO_SMALL, MHL_ERR_CUDA, MHL_ERR_NCCL.  Non-finite router
 * scores are reported asynchronously through mhl_check_device_status. */
MHL_API mhl_status mhlmoe_forward(mhl_plan plan, const void* x, const mhl_weights* w, void* out,
                          void* saved, void* workspace, size_t workspace_bytes,
                          int32_t* topk_idx, float* gates, void* stream);

/* Backward (chain rule of Eq. 1-6; router part = Alg. 2, P:846-P:866, done
 * deterministically without atomics, R21).  Same plan, x and weights as the forward
 * that filled `saved`.  d_out: [T_loc, d] E; dx: [T_loc, d] E (LOOPBACK: global).
 * Gradients: see mhl_grads.  Errors as mhlmoe_forward.  The forward's state in `saved`
 * is only read; the backward does (re)derive the weight-gradient chunk lists, a pure
 * function of that state, into scratch inside `saved`, so calls on one `saved` must not
 * run concurrently (as for any use of one plan). */
MHL_API mhl_status mhlmoe_backward(mhl_plan plan, const void* x, const mhl_weights* w, const void* d_out,
                           const void* saved, void* dx, const mhl_grads* grads,
                           void* workspace, size_t workspace_bytes, void* stream);

/* End-to-end training step from HOST buffers (x_host, dout_host: [T_loc, d] E,
 * pinned for asynchronous copies): copies x and d_out to device staging `io`
 * (io_bytes = two slots used by alternate calls), runs forward + backward, copies
 * out and dx back to out_host / dx_host ([T_loc, d] E).  Asynchronous on `stream`;
 * synchronize before reading the host outputs.  Weights and gradients are device
 * pointers.  The copies run on two plan-owned side streams (one per link direction)
 * ordered with `stream` by events: the d_out upload overlaps the forward, the out
 * download the backward, and a call's uploads overlap the previous call's backward
 * and downloads.  When `stream` completes, every output of the call is on the host.
 * Host buffers must stay valid and unmodified until then. */
MHL_API mhl_status mhlmoe_train_step_host(mhl_plan plan, const void* x_host, const void* dout_host,
                                  const mhl_weights* w, void* out_host, void* dx_host,
                                  const mhl_grads* grads, void* io, void* saved,
                                  void* workspace, size_t workspace_bytes, void* stream);

/* As mhlmoe_train_step_host, but `stream` does NOT wait for this call's downloads:
 * the next call's forward starts as soon as its own input is uploaded, so a loop of
 * calls is bound by the host link rather than by upload + compute + download in
 * series.  The host outputs (and the reuse of the host inputs) of every pipelined
 * call issued so far are safe once `stream` completes after mhl_host_drain. */
MHL_API mhl_status mhlmoe_train_step_host_pipelined(mhl_plan plan, const void* x_host, const void* dout_host,
                                            const mhl_weights* w, void* out_host, void* dx_host,
                                            const mhl_grads* grads, void* io, void* saved,
                                            void* workspace, size_t workspace_bytes, void* stream);

/* Makes `stream` wait for every host-step download issued so far (see above). */
MHL_API mhl_status mhl_host_drain(mhl_plan plan, void* stream);

/* Aux-free, global load balancing (NEXT-2): after a forward on
 * `saved`, updates this rank's router bias in place from the step's expert loads:
 *   bias[h][e] -= gamma * sign(load[h][e] - mean_e load[h][e])       (rule S:248, R24)
 * load[h][e] = replicas of local head h routed to expert e (F4's counts).  Under HP a
 * head's whole token set lives on one rank, so the load is already global: no
 * collective.  bias: DEVICE float32 [H_loc][N_e] (LOOPBACK: [N_h][N_e]), in/out, the
 * same tensor the forward used (mhl_weights.bias).  gamma >= 0 (S:267 suggests 1e-3).
 * Asynchronous on `stream`.  Errors: MHL_ERR_INVALID_ARGUMENT (NULL, gamma < 0 or NaN). */
MHL_API mhl_status mhlmoe_update_bias(mhl_plan plan, const void* saved, float* bias, float gamma, void* stream);

/* After a stream synchronize: MHL_ERR_NONFINITE if any router key seen since the
 * last call was NaN/Inf (R7), else MHL_OK.  Resets the flag. */
MHL_API mhl_status mhl_check_device_status(mhl_plan plan);

/* Number of device kernels the library launched since the plan was created
 * (diagnostic, counts every <<<>>>/cuBLAS call issued by the library). */
MHL_API uint64_t mhl_launch_count(mhl_plan plan);

/* Bytes this plan has posted to other ranks through the HP all-to-alls since creation
 * (self blocks excluded).  Independent of k and of the routing (P:811-P:812): per
 * forward (or backward) a2a_bytes_per_rank for the scatter plus T_loc*H_loc*d_h*el*(G-1)
 * for the gather (the same without routing tokens).  With LOOPBACK: summed over the
 * virtual ranks. */
MHL_API uint64_t mhl_a2a_bytes_posted(mhl_plan plan);

/* Per-step timing with CUDA events recorded on the launching stream around each
 * step (F1..F8, B8..B1) of every later forward/backward.  enable != 0 turns it on
 * and clears previous records. */
MHL_API mhl_status mhl_set_step_timing(mhl_plan plan, int enable);

/* Synchronizes on the last recorded event, accumulates the recorded steps and clears
 * them.  Writes comma-separated step names (first-seen order) to `names`
 * (capacity names_cap), per-step total milliseconds to ms[i] and call counts to
 * calls[i] (i < max_steps; arrays may be NULL).  Returns the number of steps, -1 on
 * a NULL plan. */
MHL_API int32_t mhl_step_times(mhl_plan plan, char* names, size_t names_cap, double* ms, int32_t* calls,
                               int32_t max_steps);

/* Deterministic DP reduction of the rank-partial dW_in / dW_out (MHL_FLAG_DET_DP plans, G > 1
 * without LOOPBACK): all-gathers every rank's subtree result over NCCL into `workspace`
 * (>= hp_plan_info().workspace_bytes) and sums them in the fixed tree order, in place, on every
 * rank — the caller's DP all-reduce of R19, bitwise equal to the single-GPU result.  A no-op for
 * G == 1 or LOOPBACK (the backward already returns the finished tree).  dW_in / dW_out: the same
 * device tensors the backward wrote.  Errors: MHL_ERR_INVALID_ARGUMENT (NULL, plan without
 * MHL_FLAG_DET_DP), MHL_ERR_NCCL, MHL_ERR_CUDA. */
MHL_API mhl_status mhl_dp_reduce(mhl_plan plan, float* dW_in, float* dW_out, void* workspace, size_t workspace_bytes,
                                 void* stream);

/* Fault injection (test-suite sensitivity): if the environment variable
 * MHL_FAULT_INJECT is set when hp_plan runs, that plan perturbs one step's output by a factor
 * (1 + 1e-3): "gates" (after F3), "out" (after F8), "dx" (after B1) or "dW1" (after B5); any other
 * non-empty value makes hp_plan fail with MHL_ERR_INVALID_ARGUMENT.  Never set in production. */

/* Which kernel implementation ran each step (bits OR-ed in at launch since the plan was
 * created or last reset): lets callers and tests assert that a shape took the tcgen05
 * path instead of the SIMT reference kernels, which shapes outside the tensor-core kernels'
 * support (d_h, d_e, N_e) fall back to.  reset != 0 clears the bits after reading. */
#define MHL_PATH_ROUTER_TC        (1u << 0)   /* F3 on tcgen05, N_e <= 128 (router_sm100.cu)       */
#define MHL_PATH_ROUTER_BLK       (1u << 1)   /* F3 Alg. 1 multi-block on tcgen05 (router_blk)     */
#define MHL_PATH_ROUTER_SIMT      (1u << 2)   /* F3 fp32 FMA reference kernel                      */
#define MHL_PATH_EXPERT_FWD_TC    (1u << 3)   /* F5 tcgen05, one CTA per tile                      */
#define MHL_PATH_EXPERT_FWD_PAIR  (1u << 4)   /* F5 tcgen05 cta_group::2                           */
#define MHL_PATH_EXPERT_FWD_SIMT  (1u << 5)
#define MHL_PATH_EXPERT_BWD_TC    (1u << 6)   /* B5 tcgen05 kernels                                */
#define MHL_PATH_EXPERT_BWD_SIMT  (1u << 7)
#define MHL_PATH_ROUTER_BWD_TC    (1u << 8)   /* B3 dW_r on tcgen05                                */
#define MHL_PATH_ROUTER_BWD_SIMT  (1u << 9)
#define MHL_PATH_PROJ_PINNED      (1u << 10)  /* F1/F8/B8/B1 on the plan's pinned GEMM algorithm   */
#define MHL_PATH_FUSED_COMBINE    (1u << 11)  /* (reserved: the removed in-kernel combine)         */
#define MHL_PATH_WINDOWED_COMBINE (1u << 14)  /* F5/F6 and K2/B6 alternate per token window, the
                                                 per-replica rows combined from L2 and discarded
                                                 (NEXT-1; G = 1, bf16 tensor-core path)         */
#define MHL_PATH_A2A_NCCL         (1u << 12)  /* HP exchanges through NCCL send/recv               */
#define MHL_PATH_A2A_LOOPBACK     (1u << 13)  /* HP exchanges as device copies (MHL_FLAG_LOOPBACK) */
#define MHL_PATH_EXPERT_BWD_FUSED (1u << 15)  /* B5 input side (H, dA', dH, gA, dX) in ONE tcgen05
                                                 kernel; the router term of dX moves to B6      */
MHL_API uint32_t mhl_kernel_paths(mhl_plan plan, int reset);

MHL_API const char* mhl_status_string(mhl_status s);
MHL_API const char* mhl_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* MHLMOE_H_ */
