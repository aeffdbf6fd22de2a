// capi.cpp — the C ABI (include/mhlmoe.h): plan validation/sizing, Head Parallel
// orchestration of the per-rank steps, cuBLAS projections and the NCCL all-to-alls.
//
// Per-rank data layout in HBM (R12):
//   Xs / recv1  [T_glob][HD]   HD = H_loc*d_h.  Rows are global tokens (source rank-major);
//                              local head hl is the column block [hl*d_h, (hl+1)*d_h).
//   send1       [G][T_loc][HD] destination-major output of F1 (G > 1 only)
//   send2       [T_glob][HD]   = [G(dst)][T_loc][HD]: combine output, rows in global order
//   recv2       [G(src)][T_loc][HD] -> each received block placed in its column block of cat [T_loc][D]
//   idx, gate   [H_loc][T_glob][k];  perm/pos [H_loc][T_glob*k];  Yrep/dXrep [H_loc][T_glob*k][d_h]
#include "../../include/mhlmoe.h"

#include <cublasLt.h>
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.h"
#include "tma_host.h"
#include "nccl.h"

namespace {

thread_local std::string g_last_error;

mhl_status fail(mhl_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

#define MHL_CUDA(expr)                                                                            \
  do {                                                                                            \
    cudaError_t e_ = (expr);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      return fail(MHL_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));             \
  } while (0)

#define MHL_TRY(expr)                 \
  do {                                \
    mhl_status s_ = (expr);           \
    if (s_ != MHL_OK) return s_;      \
  } while (0)

// ------------------------------------------------------------------------------------------
// NCCL, loaded at runtime (the library must load on hosts without NCCL/GPU)
// ------------------------------------------------------------------------------------------
struct NcclApi {
  bool loaded = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    const char* p = getenv("MHL_NCCL_LIB");
    if (p) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
  }
  if (!h) return api;
#define LOAD(name) api.name = reinterpret_cast<decltype(api.name)>(dlsym(h, "nccl" #name))
  LOAD(GetUniqueId); LOAD(CommInitRank); LOAD(CommDestroy); LOAD(Send); LOAD(Recv);
  LOAD(GroupStart); LOAD(GroupEnd); LOAD(GetErrorString); LOAD(AllGather);
#undef LOAD
  api.loaded = api.GetUniqueId && api.CommInitRank && api.Send && api.Recv && api.GroupStart && api.GroupEnd;
  return api;
}

#define MHL_NCCL(expr)                                                                            \
  do {                                                                                            \
    ncclResult_t e_ = (expr);                                                                     \
    if (e_ != ncclSuccess)                                                                        \
      return fail(MHL_ERR_NCCL, std::string(#expr) + ": " +                                      \
                                    (nccl().GetErrorString ? nccl().GetErrorString(e_) : "?"));  \
  } while (0)

// ------------------------------------------------------------------------------------------
// Config validation and buffer layout (pure host)
// ------------------------------------------------------------------------------------------
constexpr size_t kAlign = 256;
constexpr int kMaxA2aChunks = 8;   // token chunks of one HP exchange (hp_exchange)
constexpr int64_t kDpChunk = 8192;   // tokens per deterministic-DP weight-gradient partial
inline size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

struct Dims {
  int64_t T_loc, T_g, R, Rp;   // Rp: padded sorted-row capacity per head (R + N_e*seg_align)
  int d, N_h, d_h, N_e, k, d_e, G, H, HD, D, el, dtype, rank;
  bool loopback, simt, pair;
  bool rtok;       // MHL_FLAG_ROUTING_TOKENS (P:1565-P:1570): Xs rows carry [x part | r part]
  bool win;        // MHL_FLAG_WINDOWED_COMBINE (or MHL_WINDOWS=1)
  bool bwd_fused;  // MHL_FLAG_BWD_FUSED (or MHL_BWD_FUSED=1): B5 input side as one kernel
  bool det_dp;     // MHL_FLAG_DET_DP: dW_in / dW_out from kDpChunk-token chunk partials, fixed tree
  int dp_nc = 0;   //   chunks per rank
  int XW;          // Xs row width per rank: HD, or 2*HD with routing tokens (r part at column HD)
  int Din;         // W_in rows: D, or 2*D with routing tokens
  int n_rt, max_tiles, max_chunks, seg_align, n_rbwd;
};

struct Bump {
  size_t off = 0;
  size_t take(size_t bytes) { size_t o = off; off += align_up(bytes); return o; }
};

// offsets inside one rank's saved region
struct SavedLayout { size_t Xs, idx, gate, perm, tok_s, gate_s, pos, off, tiles, ntiles, chunks, nchunks, cbase, ccount, pbase, pcount, load, win, cat, total; };
// offsets inside one rank's workspace region (forward and backward alias each other)
struct FwdLayout { size_t send1, Yrep, send2, recv2, hist, tilepref, planes, total; };
struct BwdLayout { size_t send3, dY, dXrep, dg, dS, dS_s, dH, gA, dwr_part, W_rT, send4, recv4, dXs, dw_part, dw_done, dp_part, total; };

SavedLayout saved_layout(const Dims& m) {
  Bump b; SavedLayout L;
  L.Xs = b.take((size_t)(m.T_g + 1) * m.XW * m.el);   // + one zero row: gather target of padding rows
  L.idx = b.take((size_t)m.H * m.R * 4);
  L.gate = b.take((size_t)m.H * m.R * 4);
  L.perm = b.take((size_t)m.H * m.Rp * 4);     // padded sorted rows (cluster.cu)
  L.tok_s = b.take((size_t)m.H * m.Rp * 4);
  L.gate_s = b.take((size_t)m.H * m.Rp * 4);
  L.pos = b.take((size_t)m.H * m.R * 4);
  L.off = b.take((size_t)m.H * (m.N_e + 1) * 4);
  L.tiles = b.take((size_t)m.max_tiles * sizeof(mhl::Tile));
  L.ntiles = b.take(16);
  L.chunks = b.take((size_t)m.max_chunks * sizeof(mhl::Tile));
  L.nchunks = b.take(16);
  L.cbase = b.take((size_t)m.H * m.N_e * 4);
  L.ccount = b.take((size_t)m.H * m.N_e * 4);
  L.pbase = b.take((size_t)m.H * mhl::kDwParts * 4);
  L.pcount = b.take((size_t)m.H * mhl::kDwParts * 4);
  L.load = b.take((size_t)m.H * m.N_e * 4);             // per-head expert loads of the step (F4)
  L.win = b.take((size_t)m.H * mhl::kWindows * 4 * 4);  // windowed combine: tile / token range per window
  L.cat = b.take((size_t)m.T_loc * m.D * m.el);
  L.total = b.off;
  return L;
}

FwdLayout fwd_layout(const Dims& m) {
  Bump b; FwdLayout L;
  L.send1 = b.take(m.G > 1 ? (size_t)m.T_loc * m.G * m.XW * m.el : 0);
  L.Yrep = b.take((size_t)m.H * m.Rp * m.d_h * m.el);
  L.send2 = b.take(m.G > 1 ? (size_t)m.T_g * m.HD * m.el : 0);
  L.recv2 = b.take(m.G > 1 ? (size_t)m.T_loc * m.D * m.el : 0);
  L.hist = b.take((size_t)m.H * m.n_rt * m.N_e * 4);
  L.tilepref = b.take(((size_t)m.H * m.n_rt * m.N_e + (size_t)m.H * mhl::kTileParts * m.N_e) * 4);   // + tile bases
  L.planes = b.take(mhl::router_sm100_planes_bytes(m.H, m.d_h, m.N_e));
  L.total = b.off;
  return L;
}

BwdLayout bwd_layout(const Dims& m) {
  Bump b; BwdLayout L;
  L.send3 = b.take(m.G > 1 ? (size_t)m.T_loc * m.D * m.el : 0);
  L.dY = b.take((size_t)(m.T_g + 1) * m.HD * m.el);   // + one zero row (padding gathers)
  L.dXrep = b.take((size_t)m.H * m.Rp * m.d_h * m.el);
  L.dg = b.take((size_t)m.H * m.R * 4);
  L.dS = b.take((size_t)m.H * m.R * 4);
  L.dS_s = b.take((size_t)m.H * m.Rp * 4);   // dS in sorted-row order (K2's router term)
  L.dH = b.take((size_t)m.H * m.Rp * m.d_e * m.el);
  L.gA = b.take((size_t)m.H * m.Rp * m.d_e * m.el);
  L.dwr_part = b.take((size_t)m.H * m.n_rbwd * m.N_e * m.d_h * 4);
  L.W_rT = b.take((size_t)m.H * m.N_e * m.d_h * 4);
  L.send4 = b.take(m.G > 1 ? (size_t)m.T_g * m.XW * m.el : 0);
  L.recv4 = b.take(m.G > 1 ? (size_t)m.T_loc * m.G * m.XW * m.el : 0);
  L.dXs = b.take((size_t)m.T_loc * m.Din * m.el);
  L.dw_part = b.take(m.simt ? 0 : (size_t)m.max_chunks * 2 * m.d_e * m.d_h * 4);
  L.dw_done = b.take((size_t)m.H * m.N_e * 4);
  // MHL_FLAG_DET_DP: one fp32 weight-gradient partial per 8192-token chunk of this rank
  L.dp_part = b.take(m.det_dp ? (size_t)m.dp_nc * std::max((size_t)m.Din * m.d, (size_t)m.d * m.D) * 4 : 0);
  L.total = b.off;
  return L;
}

mhl_status make_dims(const mhl_config* c, Dims* m) {
  if (!c || !m) return fail(MHL_ERR_INVALID_ARGUMENT, "NULL config");
  if (c->tokens <= 0 || c->d_model <= 0 || c->n_heads <= 0 || c->d_head <= 0 || c->n_experts <= 0 ||
      c->d_expert <= 0 || c->world_size <= 0)
    return fail(MHL_ERR_CONFIG, "all dimensions and world_size must be positive");
  if (c->top_k < 1 || c->top_k > c->n_experts) return fail(MHL_ERR_CONFIG, "need 1 <= k <= N_e (S:213)");
  if (c->world_size > c->n_heads || c->n_heads % c->world_size != 0)
    return fail(MHL_ERR_CONFIG, "Head Parallel needs P <= N_h and N_h % P == 0 (P:803)");
  const bool loop = (c->flags & MHL_FLAG_LOOPBACK) != 0;
  if (!loop && (c->rank < 0 || c->rank >= c->world_size)) return fail(MHL_ERR_CONFIG, "rank out of range");
  if (c->dtype != MHL_F32 && c->dtype != MHL_BF16) return fail(MHL_ERR_CONFIG, "dtype must be MHL_F32 or MHL_BF16");
  if (c->top_k > 16) return fail(MHL_ERR_UNSUPPORTED, "top_k > 16 is not supported by the router kernel");
  if (c->flags & MHL_FLAG_FUSED_COMBINE)
    return fail(MHL_ERR_UNSUPPORTED, "MHL_FLAG_FUSED_COMBINE was removed: the in-kernel combine measured slower than "
                                     "the separate pass (DESIGN.md §7)");
  if (c->d_head % 8 != 0 || c->d_expert % 8 != 0 || c->d_model % 8 != 0)
    return fail(MHL_ERR_UNSUPPORTED, "d_model, d_head and d_expert must be multiples of 8");
  if (c->d_head > 512 || c->d_expert > 512) return fail(MHL_ERR_UNSUPPORTED, "d_head, d_expert <= 512");
  m->T_loc = c->tokens;
  m->G = c->world_size;
  m->T_g = m->T_loc * m->G;
  m->k = c->top_k;
  m->R = m->T_g * m->k;
  if (m->R >= (int64_t)1 << 31) return fail(MHL_ERR_UNSUPPORTED, "T_glob * k must be < 2^31");
  m->d = c->d_model; m->N_h = c->n_heads; m->d_h = c->d_head; m->N_e = c->n_experts; m->d_e = c->d_expert;
  m->H = m->N_h / m->G;
  m->HD = m->H * m->d_h;
  m->D = m->N_h * m->d_h;
  m->rtok = (c->flags & MHL_FLAG_ROUTING_TOKENS) != 0;
  m->win = (c->flags & MHL_FLAG_WINDOWED_COMBINE) != 0 || (getenv("MHL_WINDOWS") && atoi(getenv("MHL_WINDOWS")) != 0);
  m->bwd_fused = (c->flags & MHL_FLAG_BWD_FUSED) != 0 || (getenv("MHL_BWD_FUSED") && atoi(getenv("MHL_BWD_FUSED")) != 0);
  m->det_dp = (c->flags & MHL_FLAG_DET_DP) != 0;
  if (m->det_dp) {
    auto pow2 = [](int64_t v) { return v > 0 && (v & (v - 1)) == 0; };
    m->dp_nc = (int)(m->T_loc / kDpChunk);
    if (m->T_loc % kDpChunk != 0 || !pow2(m->dp_nc) || !pow2(m->G))
      return fail(MHL_ERR_UNSUPPORTED, "MHL_FLAG_DET_DP needs T_loc a power-of-two multiple of 8192 and G a power of two");
  }
  m->XW = m->HD * (m->rtok ? 2 : 1);
  m->Din = m->D * (m->rtok ? 2 : 1);
  m->dtype = c->dtype;
  m->el = c->dtype == MHL_BF16 ? 2 : 4;
  m->loopback = loop;
  m->simt = (c->flags & MHL_FLAG_SIMT) != 0 || c->dtype == MHL_F32;
  m->pair = !m->simt && (c->flags & MHL_FLAG_PAIR) != 0;
  if ((c->flags & MHL_FLAG_REQUIRE_TC) && !m->simt) {
    std::string miss;
    if (!mhl::router_sm100_supported(m->d_h, m->N_e) && !mhl::router_blk_supported(m->d_h, m->N_e, m->k)) miss += " router";
    if (!mhl::router_bwd_sm100_supported(m->d_h, m->N_e, m->k)) miss += " router-backward";
    if (!mhl::expert_fwd_sm100_supported(m->d_h, m->d_e)) miss += " expert-forward";
    if (!mhl::expert_bwd_sm100_supported(m->d_h, m->d_e)) miss += " expert-backward";
    if (!miss.empty()) return fail(MHL_ERR_UNSUPPORTED, "MHL_FLAG_REQUIRE_TC: no tcgen05 kernel for this shape:" + miss);
  }
  if ((c->flags & MHL_FLAG_REQUIRE_TC) && m->simt)
    return fail(MHL_ERR_UNSUPPORTED, "MHL_FLAG_REQUIRE_TC with the SIMT path (fp32 or MHL_FLAG_SIMT)");
  m->seg_align = m->pair ? 2 * mhl::kExpertBM : mhl::kExpertBM;
  m->Rp = m->R + (int64_t)m->N_e * m->seg_align;   // each expert segment padded by < seg_align rows
  if (m->Rp >= (int64_t)1 << 31) return fail(MHL_ERR_UNSUPPORTED, "T_glob * k + N_e * seg_align must be < 2^31");
  m->rank = loop ? 0 : c->rank;
  m->n_rt = (int)((m->T_g + mhl::kRouterTile - 1) / mhl::kRouterTile);
  // router-backward partials: one per router tile on the SIMT path, at most 2 * 148 / N_h per head on
  // the tcgen05 path (two CTAs per SM; a constant, not the device's SM count: dW_r bits stay fixed)
  m->n_rbwd = (!m->simt && mhl::router_bwd_sm100_supported(m->d_h, m->N_e, m->k))
                  ? std::min(m->n_rt, std::max(1, 2 * mhl::kDwParts / m->N_h)) : m->n_rt;
  const int64_t mt = (int64_t)m->H * ((m->R + mhl::kExpertBM - 1) / mhl::kExpertBM + 2 * m->N_e);
  if (mt >= (int64_t)1 << 31) return fail(MHL_ERR_UNSUPPORTED, "too many tiles");
  m->max_tiles = (int)mt;
  m->max_chunks = (int)((int64_t)m->H * (mhl::kDwParts + m->N_e));   // <= parts + expert boundaries
  const size_t router_smem = (size_t)m->el * m->d_h * mhl::kRouterTile + 4ull * m->d_h * 32 + 4ull * m->N_e;
  const size_t rbwd_smem = 4ull * std::min<int64_t>((int64_t)m->N_e * m->d_h, 32768) + 8ull * mhl::kRouterTile * m->k;
  if (router_smem > 200 * 1024 || rbwd_smem > 200 * 1024)
    return fail(MHL_ERR_UNSUPPORTED, "d_head * N_e too large for the router kernels' shared memory");
  return MHL_OK;
}

void fill_info(const Dims& m, mhl_plan_info* info) {
  const int vr = m.loopback ? m.G : 1;  // regions per process
  info->head_begin = m.loopback ? 0 : m.rank * m.H;
  info->head_end = m.loopback ? m.N_h : (m.rank + 1) * m.H;
  info->tokens_global = m.T_g;
  info->a2a_bytes_per_peer = (uint64_t)m.T_loc * m.XW * m.el;   // the scatter (x and, with routing tokens, r)
  info->a2a_bytes_per_rank = info->a2a_bytes_per_peer * (uint64_t)(m.G - 1);
  info->saved_bytes = (uint64_t)saved_layout(m).total * vr;
  info->workspace_bytes = (uint64_t)std::max(fwd_layout(m).total, bwd_layout(m).total) * vr;
  info->io_bytes = 8ull * align_up((size_t)m.T_loc * vr * m.d * m.el);   // 2 slots x {x, d_out, out, dx}
  info->max_tiles = m.max_tiles;
}

struct LtKey {
  bool ta, tb, c_f32, bf; int64_t N, K, Mkey;
  bool operator==(const LtKey& o) const {
    return ta == o.ta && tb == o.tb && c_f32 == o.c_f32 && bf == o.bf && N == o.N && K == o.K && Mkey == o.Mkey;
  }
};
struct LtEntry { LtKey key; cublasLtMatmulAlgo_t algo; };

}  // namespace

// ------------------------------------------------------------------------------------------
// Plan
// ------------------------------------------------------------------------------------------
struct mhl_plan_s {
  mhl_config cfg;
  Dims m;
  mhl_plan_info info;
  cublasLtHandle_t lt = nullptr;
  void* blas_ws = nullptr;
  size_t blas_ws_bytes = 32u << 20;
  std::vector<LtEntry> lt_algos;   // pinned projection-GEMM algorithms (Gemm)
  ncclComm_t comm = nullptr;
  int32_t* dflag = nullptr;   // device non-finite flag
  cudaError_t launch_err = cudaSuccess;   // first launch error harvested by a StepSpan
  const char* launch_err_at = "";
  int num_sms = 148;
  // host-buffer step (mhlmoe_train_step_host): side stream for the copies that can overlap compute
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  // per io slot (host steps alternate between two staging slots)
  cudaEvent_t ev_x[2] = {}, ev_dout[2] = {}, ev_fwd[2] = {}, ev_out[2] = {}, ev_bwd[2] = {}, ev_dx[2] = {};
  cudaEvent_t ev_drain = nullptr;
  bool io_live[2] = {false, false};   // the slot's events of a previous host step are recorded
  uint64_t host_steps = 0;
  // HP exchanges (G > 1): comm stream pipelined against the producers on the compute stream
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_prod = nullptr, ev_comm = nullptr;
  cudaEvent_t ev_chunk[kMaxA2aChunks] = {};   // chunk c of an exchange has landed (hp_exchange)
  std::atomic<uint64_t> launches{0};
  std::atomic<uint32_t> paths{0};     // MHL_PATH_* bits of the kernels launched (mhl_kernel_paths)
  // fault injection: MHL_FAULT_INJECT=gates|out|dx|dW1 at plan creation scales that
  // output by (1 + 1e-3) so the conformance suite can be shown to fail
  int fault = 0;   // 0 none, 1 gates (after F3), 2 out (after F8), 3 dx (after B1), 4 dW1 (after B5)
  uint64_t a2a_bytes_posted = 0;
  // optional per-step CUDA-event timing (mhl_set_step_timing)
  bool timing = false;
  struct Rec { const char* name; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  size_t pool_used = 0;
  cudaEvent_t next_event() {
    if (pool_used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[pool_used++];
  }
};

namespace {

// Records CUDA events around one named step on the launching stream when timing is on.
struct StepSpan {
  mhl_plan p; const char* name; cudaStream_t s; cudaEvent_t a = nullptr;
  StepSpan(mhl_plan p_, const char* n, cudaStream_t s_) : p(p_), name(n), s(s_) {
    if (p->timing) { a = p->next_event(); cudaEventRecord(a, s); }
  }
  ~StepSpan() {
    // Launch-time errors are non-sticky and a later library call (cuBLAS) may reset the runtime's
    // last-error slot, so every span harvests them immediately; check_kernels() reports the first.
    const cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess && p->launch_err == cudaSuccess) { p->launch_err = le; p->launch_err_at = name; }
    if (a) { cudaEvent_t b = p->next_event(); cudaEventRecord(b, s); p->recs.push_back({name, a, b}); }
    static const bool dbg = getenv("MHL_DEBUG_SYNC") != nullptr;
    if (dbg) {
      cudaError_t e1 = cudaGetLastError();
      cudaError_t e2 = cudaStreamSynchronize(s);
      fprintf(stderr, "[mhl debug] %s: launch=%s sync=%s\n", name, cudaGetErrorString(e1), cudaGetErrorString(e2));
    }
  }
};
#define MHL_SPAN(name) StepSpan span_##__LINE__(p, name, s)

// Projection GEMMs (F1, F8, B8, B1: Eq. 5, Eq. 6 P:772 and their chain rule) on cuBLASLt
// with a PINNED algorithm: for each (op, N, K, types) the algorithm is chosen once,
// from the heuristic at a fixed reference M (kRefM, independent of the plan's T_loc and of G), with
// split-K disabled (one sequential K loop per output tile), and then reused for every M.  Every
// output row is therefore computed by the same tile program with the same K order whatever M is,
// which is what makes out / dx bitwise independent of T_loc and so of the HP degree (§8(e)); the
// weight-gradient GEMMs (K = tokens) are pinned per shape, so they are run-to-run deterministic.
constexpr int64_t kRefM = 65536;

// cuBLASLt is column-major: row-major C[M,N] = op(A) op(B) is computed as C^T[N,M] = op(B)^T op(A)^T.
struct LtShape {
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t a = nullptr, b = nullptr, c = nullptr;
  ~LtShape() {
    if (op) cublasLtMatmulDescDestroy(op);
    if (a) cublasLtMatrixLayoutDestroy(a);
    if (b) cublasLtMatrixLayoutDestroy(b);
    if (c) cublasLtMatrixLayoutDestroy(c);
  }
  bool make(bool ta, bool tb, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb, int64_t ldc, bool c_f32,
            bool bf) {
    const cudaDataType_t ab = bf ? CUDA_R_16BF : CUDA_R_32F;
    const cudaDataType_t ct = c_f32 ? CUDA_R_32F : ab;
    const cublasComputeType_t comp = bf ? CUBLAS_COMPUTE_32F : CUBLAS_COMPUTE_32F_PEDANTIC;
    if (cublasLtMatmulDescCreate(&op, comp, CUDA_R_32F) != CUBLAS_STATUS_SUCCESS) return false;
    const cublasOperation_t opB = tb ? CUBLAS_OP_T : CUBLAS_OP_N, opA = ta ? CUBLAS_OP_T : CUBLAS_OP_N;
    // column-major "A" operand of cuBLAS = our B (N x K view), "B" operand = our A
    cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &opB, sizeof(opB));
    cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &opA, sizeof(opA));
    // stored shapes (column-major rows x cols): B^T-view is (tb ? K x N : N x K), A-view (ta ? M x K : K x M)
    if (cublasLtMatrixLayoutCreate(&a, ab, tb ? K : N, tb ? N : K, ldb) != CUBLAS_STATUS_SUCCESS) return false;
    if (cublasLtMatrixLayoutCreate(&b, ab, ta ? M : K, ta ? K : M, lda) != CUBLAS_STATUS_SUCCESS) return false;
    if (cublasLtMatrixLayoutCreate(&c, ct, N, M, ldc) != CUBLAS_STATUS_SUCCESS) return false;
    return true;
  }
};

struct Gemm {
  mhl_plan p;
  cudaStream_t s;
  // Row-major C[M,N] = alpha * op(A) op(B) + beta C; A is [M,K] (ta: stored [K,M]),
  // B is [K,N] (tb: stored [N,K]).
  mhl_status operator()(bool ta, bool tb, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                        const void* B, int64_t ldb, void* C, int64_t ldc, bool c_f32, float beta) const;
};

inline char* at(void* base, size_t off) { return static_cast<char*>(base) + off; }
inline const char* at(const void* base, size_t off) { return static_cast<const char*>(base) + off; }

mhl_status Gemm::operator()(bool ta, bool tb, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                            const void* B, int64_t ldb, void* C, int64_t ldc, bool c_f32, float beta) const {
  if (M == 0 || N == 0) return MHL_OK;
  const bool bf = p->m.dtype == MHL_BF16;
  // per-row GEMMs (fprop / dgrad: K fixed by the weights) are pinned at the reference M, the
  // weight-gradient GEMMs (ta: M, N fixed by the weights, K = tokens) per actual shape
  const LtKey key{ta, tb, c_f32, bf, N, K, ta ? M : kRefM};
  const cublasLtMatmulAlgo_t* algo = nullptr;
  for (const LtEntry& e : p->lt_algos)
    if (e.key == key) { algo = &e.algo; break; }
  if (!algo) {
    const int64_t Mh = key.Mkey;
    LtShape h;
    if (!h.make(ta, tb, Mh, N, K, ta ? Mh : K, tb ? K : N, N, c_f32, bf))
      return fail(MHL_ERR_CUDA, "cublasLt descriptor creation failed");
    cublasLtMatmulPreference_t pref;
    if (cublasLtMatmulPreferenceCreate(&pref) != CUBLAS_STATUS_SUCCESS) return fail(MHL_ERR_CUDA, "cublasLt preference");
    size_t wsb = p->blas_ws_bytes;
    cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsb, sizeof(wsb));
    // per-row GEMMs: no split-K at all (one sequential K loop per output tile); wgrad: any
    // reduction scheme cuBLASLt runs deterministically (fixed partition, no atomics)
    const uint32_t mask = ta ? (uint32_t)CUBLASLT_REDUCTION_SCHEME_MASK : (uint32_t)CUBLASLT_REDUCTION_SCHEME_NONE;
    cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_REDUCTION_SCHEME_MASK, &mask, sizeof(mask));
    cublasLtMatmulHeuristicResult_t res[8];
    int n = 0;
    const cublasStatus_t st = cublasLtMatmulAlgoGetHeuristic(p->lt, h.op, h.a, h.b, h.c, h.c, pref, 8, res, &n);
    cublasLtMatmulPreferenceDestroy(pref);
    if (st != CUBLAS_STATUS_SUCCESS || n == 0) return fail(MHL_ERR_CUDA, "cublasLt: no algorithm for a projection GEMM");
    LtEntry e{key, res[0].algo};
    if (!ta) {
      const int32_t one = 1;
      const uint32_t none = CUBLASLT_REDUCTION_SCHEME_NONE;
      cublasLtMatmulAlgoConfigSetAttribute(&e.algo, CUBLASLT_ALGO_CONFIG_SPLITK_NUM, &one, sizeof(one));
      cublasLtMatmulAlgoConfigSetAttribute(&e.algo, CUBLASLT_ALGO_CONFIG_REDUCTION_SCHEME, &none, sizeof(none));
    }
    p->lt_algos.push_back(e);
    algo = &p->lt_algos.back().algo;
  }
  LtShape sh;
  if (!sh.make(ta, tb, M, N, K, lda, ldb, ldc, c_f32, bf)) return fail(MHL_ERR_CUDA, "cublasLt descriptor creation failed");
  const float alpha = 1.0f;
  const cublasStatus_t st = cublasLtMatmul(p->lt, sh.op, &alpha, B, sh.a, A, sh.b, &beta, C, sh.c, C, sh.c, algo,
                                           p->blas_ws, p->blas_ws_bytes, s);
  if (st != CUBLAS_STATUS_SUCCESS)
    return fail(MHL_ERR_CUDA, "cublasLtMatmul (pinned algorithm) status " + std::to_string((int)st));
  p->launches++;
  p->paths |= MHL_PATH_PROJ_PINNED;
  return MHL_OK;
}

// Equal-split all-to-all (P:805-P:806), pipelined with its producer and its consumer (SURVEY
// §8(e)).  The T_loc rows of every block are cut into C token chunks (chunk boundaries c*T_loc/C,
// MHL_A2A_CHUNKS, default 4).  For chunk c, step i = 0..G-1 sends the chunk of the block rank r
// addresses to q = (r+i) mod G and receives that of src = (r-i) mod G, so at every step each rank's
// send meets its peer's receive.  produce(c, i) enqueues on the compute stream `s` whatever writes
// step i's outgoing chunk (step 0, the self block, is written straight into place); each step's
// exchange waits only for its producer and runs on the plan's comm stream while the compute stream
// produces the next one.  consume(c) — the row-chunk GEMM that needs every source's chunk c (F8,
// B1's dgrad) — is enqueued on `s` after chunk c+1 has been produced, waiting only for chunk c's
// exchange, so it overlaps chunk c+1's.  Row chunks keep the per-row GEMM programs (pinned
// algorithm, no split-K), so every output row has the same bits whatever C and G are.  tail()
// enqueues more independent work on `s`; `s` then waits for the comm stream.  Bytes are
// k-independent and counted per posted send.
//   send[v]  [G][blk]   outgoing blocks of (virtual) rank v, blk = rows * (parts * row_bytes)
//   recv[v]  [G][blk]   incoming blocks (NCCL mode; loopback copies straight to their destination)
//   place[v] optional: incoming block src is then copied into columns [src*row_bytes, ...) of the
//            [rows][pitch] matrix place[v] (F7 -> cat, B2 -> dXs), else recv itself is the target
//   parts    with routing sub-tokens a B2 block row is [dX part | dR part] (parts = 2): part pi of
//            source src goes to columns [pi*part_dst + src*row_bytes, ...) of place
struct Xfer {
  std::vector<const char*> send;
  std::vector<char*> recv, place;
  size_t blk = 0;
  int64_t rows = 0;
  size_t row_bytes = 0, pitch = 0;
  int parts = 1;
  size_t part_dst = 0;
};

int a2a_chunks(int64_t rows) {
  static const int env = getenv("MHL_A2A_CHUNKS") ? atoi(getenv("MHL_A2A_CHUNKS")) : 4;
  return (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)env, (int64_t)kMaxA2aChunks, rows}));
}
inline int64_t chunk_row(int64_t rows, int C, int c) { return rows * c / C; }

template <class Produce, class Consume, class Tail>
mhl_status hp_exchange(mhl_plan p, const Xfer& X, cudaStream_t s, Produce produce, Consume consume, Tail tail) {
  const Dims& m = p->m;
  cudaStream_t cs = p->comm_stream;
  const size_t blk = X.blk;
  const int64_t rows = X.rows;
  const size_t rb = blk / (size_t)rows;   // bytes of one block row
  const int C = a2a_chunks(rows);
  for (int c = 0; c < C; ++c) {
    const int64_t r0 = chunk_row(rows, C, c), nr = chunk_row(rows, C, c + 1) - r0;
    for (int i = 0; i < m.G; ++i) {
      MHL_TRY(produce(c, i));
      if (i == 0) continue;
      MHL_CUDA(cudaEventRecord(p->ev_prod, s));
      MHL_CUDA(cudaStreamWaitEvent(cs, p->ev_prod, 0));
      if (m.loopback) {
        for (int v = 0; v < m.G; ++v) {
          const int q = (v + i) % m.G;
          const char* src = X.send[v] + q * blk + r0 * rb;
          if (!X.place.empty())
            for (int pi = 0; pi < X.parts; ++pi)
              mhl::launch_copy_rows(src + pi * X.row_bytes, (int64_t)(X.parts * X.row_bytes),
                                    X.place[q] + r0 * X.pitch + pi * X.part_dst + v * X.row_bytes, (int64_t)X.pitch,
                                    nr, (int64_t)X.row_bytes, cs);
          else
            MHL_CUDA(cudaMemcpyAsync(X.recv[q] + v * blk + r0 * rb, src, nr * rb, cudaMemcpyDeviceToDevice, cs));
          p->a2a_bytes_posted += nr * rb;
          p->paths |= MHL_PATH_A2A_LOOPBACK;
          if (!X.place.empty()) p->launches += X.parts;
        }
      } else {
        const int r = m.rank, q = (r + i) % m.G, src = (r - i + m.G) % m.G;
        NcclApi& api = nccl();
        MHL_NCCL(api.GroupStart());
        MHL_NCCL(api.Send(X.send[0] + q * blk + r0 * rb, nr * rb, ncclUint8, q, p->comm, cs));
        MHL_NCCL(api.Recv(X.recv[0] + src * blk + r0 * rb, nr * rb, ncclUint8, src, p->comm, cs));
        MHL_NCCL(api.GroupEnd());
        p->a2a_bytes_posted += nr * rb;
        p->paths |= MHL_PATH_A2A_NCCL;
        p->launches++;
        if (!X.place.empty()) {
          for (int pi = 0; pi < X.parts; ++pi)
            mhl::launch_copy_rows(X.recv[0] + src * blk + r0 * rb + pi * X.row_bytes, (int64_t)(X.parts * X.row_bytes),
                                  X.place[0] + r0 * X.pitch + pi * X.part_dst + src * X.row_bytes, (int64_t)X.pitch,
                                  nr, (int64_t)X.row_bytes, cs);
          p->launches += X.parts;
        }
      }
    }
    MHL_CUDA(cudaEventRecord(p->ev_chunk[c], cs));
    if (c >= 1) {   // chunk c-1 is complete on every rank once its exchange is: consume it now
      MHL_CUDA(cudaStreamWaitEvent(s, p->ev_chunk[c - 1], 0));
      MHL_TRY(consume(c - 1, chunk_row(rows, C, c - 1), chunk_row(rows, C, c) - chunk_row(rows, C, c - 1)));
    }
  }
  MHL_CUDA(cudaStreamWaitEvent(s, p->ev_chunk[C - 1], 0));
  MHL_TRY(consume(C - 1, chunk_row(rows, C, C - 1), rows - chunk_row(rows, C, C - 1)));
  MHL_TRY(tail());
  MHL_CUDA(cudaEventRecord(p->ev_comm, cs));
  MHL_CUDA(cudaStreamWaitEvent(s, p->ev_comm, 0));
  return MHL_OK;
}

// MHL_FLAG_DET_DP: a weight gradient W = Σ_tokens a_tᵀ b_t (dW_out = doᵀ cat, dW_in =
// dXsᵀ x) as kDpChunk-token chunk partials in global token order (virtual rank v's chunks follow
// v-1's: R12), summed by a fixed pairwise tree ((P0+P1)+(P2+P3))+...  The same tree at every G
// (chunk counts are powers of two): with LOOPBACK all ranks' chunks are here and the tree is
// finished; otherwise the rank's subtree is returned and mhl_dp_reduce completes it.
template <class AB>
mhl_status det_wgrad(mhl_plan p, const Gemm& gemm, int VR, AB ab, int64_t M, int64_t N, int64_t lda, int64_t ldb,
                     const std::vector<char*>& part, float* out, cudaStream_t s) {
  const Dims& m = p->m;
  std::vector<float*> slot;
  for (int v = 0; v < VR; ++v) {
    const auto op = ab(v);   // (A [tokens][lda], B [tokens][ldb]) of rank v
    for (int c = 0; c < m.dp_nc; ++c) {
      float* sl = reinterpret_cast<float*>(part[v]) + (size_t)c * M * N;
      MHL_TRY(gemm(true, false, M, N, kDpChunk, at(op.first, (size_t)c * kDpChunk * lda * m.el), lda,
                   at(op.second, (size_t)c * kDpChunk * ldb * m.el), ldb, sl, N, true, 0.0f));
      slot.push_back(sl);
    }
  }
  for (size_t st = 1; st < slot.size(); st *= 2)
    for (size_t i = 0; i + st < slot.size(); i += 2 * st) {
      mhl::launch_add_inplace(slot[i], slot[i + st], M * N, s);
      p->launches++;
    }
  MHL_CUDA(cudaMemcpyAsync(out, slot[0], (size_t)M * N * 4, cudaMemcpyDeviceToDevice, s));
  return MHL_OK;
}

struct RankPtrs {   // one (virtual) rank's view
  char* saved;
  char* ws;
  const void* x;
  void* out;        // forward: out; backward: dx
  const void* dout;
  const float* W_r; const float* bias; const void* W1; const void* W2;   // local heads
  float* dW_r; float* dW1; float* dW2;
  int32_t* topk_idx; float* gates;
};

// the clustered-routing state of one rank, as stored in its `saved` region
mhl::Routing routing_view(const Dims& m, const char* saved) {
  const SavedLayout S = saved_layout(m);
  mhl::Routing rt;
  rt.H = m.H; rt.T = m.T_g; rt.k = m.k; rt.N_e = m.N_e; rt.Rp = m.Rp; rt.seg_align = m.seg_align;
  rt.idx = (const int32_t*)(saved + S.idx);
  rt.gate = (const float*)(saved + S.gate);
  rt.perm = (const int32_t*)(saved + S.perm);
  rt.tok_s = (const int32_t*)(saved + S.tok_s);
  rt.gate_s = (const float*)(saved + S.gate_s);
  rt.pos = (const int32_t*)(saved + S.pos);
  rt.off = (const int32_t*)(saved + S.off);
  rt.tiles = (const mhl::Tile*)(saved + S.tiles);
  rt.ntiles = (const int32_t*)(saved + S.ntiles);
  rt.max_tiles = m.max_tiles;
  rt.chunks = (const mhl::Tile*)(saved + S.chunks);
  rt.nchunks = (const int32_t*)(saved + S.nchunks);
  rt.max_chunks = m.max_chunks;
  rt.cbase = (const int32_t*)(saved + S.cbase);
  rt.ccount = (const int32_t*)(saved + S.ccount);
  rt.pbase = (const int32_t*)(saved + S.pbase);
  rt.pcount = (const int32_t*)(saved + S.pcount);
  rt.dw_parts = mhl::kDwParts;
  return rt;
}

// NEXT-1 (windowed, L2-resident combine): at G = 1 on the tensor-core path the expert kernel and
// the combine alternate window by window (kWinParts token-order parts of one head): each window's
// per-replica rows (Yrep forward, dXrep backward; ~67 MB at paper scale) are combined while still
// in L2 and then discarded from it, so they are never written back to HBM.  Opt-in
// (MHL_FLAG_WINDOWED_COMBINE, or MHL_WINDOWS=1 for the process):
// the 32 extra launch pairs per direction cost more than the L2 residency saves (F5 + F6 1.97 ms
// vs 1.27, K2 + B6 1.64 vs 1.08 at paper scale, tools/ab_windows.sh), so the default is one expert
// launch + one combine launch.
bool windowed(const Dims& m) {
  return m.win && m.G == 1 && !m.simt && !m.pair && !m.rtok && m.dtype == MHL_BF16 && m.d_h % 64 == 0 &&
         mhl::expert_fwd_sm100_supported(m.d_h, m.d_e) && mhl::expert_bwd_sm100_supported(m.d_h, m.d_e);
}

// B5's input side as ONE kernel (MHL_FLAG_BWD_FUSED, opt-in; expert_bwd_fused_sm100.cu, the router
// term of dX then moves to B6) where its TMEM budget holds; the default is the K1 + K2 pair, which
// measured the same step time (the fused kernel's gain went to B6's router term).
bool bwd_fused(const Dims& m) {
  return m.bwd_fused && !m.simt && !m.pair && !windowed(m) && m.dtype == MHL_BF16 &&
         mhl::expert_bwd_sm100_supported(m.d_h, m.d_e) && mhl::expert_bwd_fused_supported(m.d_h, m.d_e);
}

mhl_status check_kernels(mhl_plan p) {
  if (p->launch_err != cudaSuccess) {
    const cudaError_t e = p->launch_err;
    p->launch_err = cudaSuccess;
    return fail(MHL_ERR_CUDA, std::string("kernel launch in ") + p->launch_err_at + ": " + cudaGetErrorString(e));
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(MHL_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  return MHL_OK;
}

// B6 for tokens [t0, t0 + nT): on the split tensor-core path K2 already added the router term to
// each replica row (rterm_in_rep), so B6 is the plain k-row sum (the F6 kernel); the fused and SIMT
// paths add it here.  With
// routing sub-tokens (P:1565-P:1570) the router term is the gradient of r, not of x: dX gets the
// plain sum (out_x) and dR the router term alone (out_r).
void combine_bwd(const Dims& m, const mhl::Routing& rt, const void* dXrep, const float* dS, const float* W_rT, bool rterm_in_rep,
                 void* out_x, int64_t ld_x, void* out_r, int64_t ld_r, cudaStream_t s, int64_t t0, int64_t nT) {
  if (m.rtok) {
    mhl::launch_combine_fwd(m.dtype, rt, dXrep, m.d_h, out_x, ld_x, s, t0, nT);
    mhl::launch_combine_bwd(m.dtype, rt, nullptr, dS, W_rT, m.d_h, out_r, ld_r, s, t0, nT);
  } else if (rterm_in_rep) {
    mhl::launch_combine_fwd(m.dtype, rt, dXrep, m.d_h, out_x, ld_x, s, t0, nT);
  } else {
    mhl::launch_combine_bwd(m.dtype, rt, dXrep, dS, W_rT, m.d_h, out_x, ld_x, s, t0, nT);
  }
}

// F3-F6 for one rank's local heads; input recv1 (= saved Xs), output rows into `yout` [T_g][HD]
// (yout == nullptr: F6 is left to the caller, which runs it per HP destination block)
mhl_status moe_forward_local(mhl_plan p, const RankPtrs& R, void* yout, cudaStream_t s) {
  const Dims& m = p->m;
  const SavedLayout S = saved_layout(m);
  const FwdLayout F = fwd_layout(m);
  const void* Xs = R.saved + S.Xs;
  // routing sub-tokens: Xs itself, or its r part at column HD (MHL_FLAG_ROUTING_TOKENS)
  const void* Xr = R.saved + S.Xs + (m.rtok ? (size_t)m.HD * m.el : 0);
  int32_t* idx = (int32_t*)(R.saved + S.idx);
  float* gate = (float*)(R.saved + S.gate);
  int32_t* perm = (int32_t*)(R.saved + S.perm);
  int32_t* pos = (int32_t*)(R.saved + S.pos);
  int32_t* off = (int32_t*)(R.saved + S.off);
  mhl::Tile* tiles = (mhl::Tile*)(R.saved + S.tiles);
  int32_t* ntiles = (int32_t*)(R.saved + S.ntiles);
  int32_t* hist = (int32_t*)(R.ws + F.hist);
  {
    MHL_SPAN("F3_router_topk");
    if (!m.simt && mhl::router_sm100_supported(m.d_h, m.N_e)) {
      if (!mhl::launch_router_sm100(Xr, m.XW, R.W_r, R.bias, m.H, m.T_g, m.d_h, m.N_e, m.k, R.ws + F.planes, idx, gate,
                                    hist, p->dflag, p->num_sms, s))
        return fail(MHL_ERR_CUDA, "router: TMA tensor-map encoding failed");
      p->paths |= MHL_PATH_ROUTER_TC;
    } else if (!m.simt && mhl::router_blk_supported(m.d_h, m.N_e, m.k)) {
      mhl::launch_router_split(R.W_r, R.ws + F.planes, m.H, m.d_h, m.N_e, s);
      if (!mhl::launch_router_blk_sm100(Xr, m.XW, R.ws + F.planes, R.bias, m.H, m.T_g, m.d_h, m.N_e, m.k, idx, gate,
                                        hist, p->dflag, p->num_sms, s))
        return fail(MHL_ERR_CUDA, "router (blocked): TMA tensor-map encoding failed");
      p->paths |= MHL_PATH_ROUTER_BLK;
    } else {
      mhl::launch_router_topk(m.dtype, Xr, m.XW, R.W_r, R.bias, m.H, m.T_g, m.d_h, m.N_e, m.k, idx, gate, hist,
                              p->dflag, s);
      p->paths |= MHL_PATH_ROUTER_SIMT;
    }
  }
  if (p->fault == 1) mhl::launch_scale(0, gate, (int64_t)m.H * m.R, 1.001f, s);
  {
    MHL_SPAN("F4_cluster");
    mhl::launch_cluster(m.H, m.T_g, m.k, m.N_e, idx, gate, hist, (int32_t*)(R.ws + F.tilepref),
                        (int32_t*)(R.saved + S.load), off, perm, pos, (int32_t*)(R.saved + S.tok_s),
                        (float*)(R.saved + S.gate_s), m.Rp, m.seg_align, tiles, ntiles, m.max_tiles,
                        (mhl::Tile*)(R.saved + S.chunks),
                        (int32_t*)(R.saved + S.nchunks), (int32_t*)(R.saved + S.cbase), (int32_t*)(R.saved + S.ccount),
                        m.max_chunks, 0, (int32_t*)(R.saved + S.pbase), (int32_t*)(R.saved + S.pcount), s);
    if (windowed(m)) {
      mhl::launch_windows(m.H, m.N_e, m.T_g, m.Rp, m.seg_align, (const int32_t*)(R.saved + S.load), off,
                          (const int32_t*)(R.ws + F.tilepref), m.n_rt, ntiles, (const int32_t*)(R.saved + S.tok_s),
                          (int32_t*)(R.saved + S.win), s);
      p->launches++;
    }
  }
  const mhl::Routing rt = routing_view(m, R.saved);
  void* Yrep = R.ws + F.Yrep;
  if (yout && windowed(m)) {
    MHL_CUDA(cudaMemsetAsync(R.saved + S.Xs + (size_t)m.T_g * m.XW * m.el, 0, (size_t)m.XW * m.el, s));
    const int32_t* win = (const int32_t*)(R.saved + S.win);
    for (int h = 0; h < m.H; ++h)
      for (int w = 0; w < mhl::kWindows; ++w) {
        mhl::Routing rw = rt;
        rw.trange = win + ((size_t)h * mhl::kWindows + w) * 4;
        {
          MHL_SPAN("F5_expert_fwd");
          if (!mhl::launch_expert_fwd_sm100(rw, Xs, m.XW, R.W1, R.W2, m.d_h, m.d_e, Yrep, p->num_sms, s))
            return fail(MHL_ERR_CUDA, "expert_fwd: TMA tensor-map encoding failed");
        }
        MHL_SPAN("F6_combine");
        mhl::launch_combine_window(m.dtype, rt, Yrep, m.d_h, yout, m.HD, h, rw.trange + 2, m.T_g / mhl::kWindows, true,
                                   s);
      }
    p->paths |= MHL_PATH_EXPERT_FWD_TC | MHL_PATH_WINDOWED_COMBINE;
    p->launches += 5 + 2 * m.H * mhl::kWindows;
    if (R.topk_idx) MHL_CUDA(cudaMemcpyAsync(R.topk_idx, idx, (size_t)m.H * m.R * 4, cudaMemcpyDeviceToDevice, s));
    if (R.gates) MHL_CUDA(cudaMemcpyAsync(R.gates, gate, (size_t)m.H * m.R * 4, cudaMemcpyDeviceToDevice, s));
    return check_kernels(p);
  }
  {
    MHL_SPAN("F5_expert_fwd");
    // the all-zero sub-token row T: target of the padding rows of every expert tile
    MHL_CUDA(cudaMemsetAsync(R.saved + S.Xs + (size_t)m.T_g * m.XW * m.el, 0, (size_t)m.XW * m.el, s));
    // CTA-pair (cta_group::2) kernels with MHL_FLAG_PAIR (segments padded to tile pairs)
    if (m.simt || !mhl::expert_fwd_sm100_supported(m.d_h, m.d_e)) {
      mhl::launch_expert_fwd_simt(m.dtype, rt, Xs, m.XW, R.W1, R.W2, m.d_h, m.d_e, Yrep, s);
      p->paths |= MHL_PATH_EXPERT_FWD_SIMT;
    } else if (m.pair && mhl::expert_fwd_pair_supported(m.d_h, m.d_e) && p->num_sms >= 2 && !getenv("MHL_F5_SINGLE")) {
      if (!mhl::launch_expert_fwd_pair_sm100(rt, Xs, m.XW, R.W1, R.W2, m.d_h, m.d_e, Yrep, p->num_sms, s))
        return fail(MHL_ERR_CUDA, "expert_fwd (pair): TMA tensor-map encoding failed");
      p->paths |= MHL_PATH_EXPERT_FWD_PAIR;
    } else {
      if (!mhl::launch_expert_fwd_sm100(rt, Xs, m.XW, R.W1, R.W2, m.d_h, m.d_e, Yrep, p->num_sms, s))
        return fail(MHL_ERR_CUDA, "expert_fwd: TMA tensor-map encoding failed");
      p->paths |= MHL_PATH_EXPERT_FWD_TC;
    }
  }
  if (yout) {
    MHL_SPAN("F6_combine");
    mhl::launch_combine_fwd(m.dtype, rt, Yrep, m.d_h, yout, m.HD, s);
  }
  p->launches += yout ? 7 : 6;
  if (R.topk_idx) MHL_CUDA(cudaMemcpyAsync(R.topk_idx, idx, (size_t)m.H * m.R * 4, cudaMemcpyDeviceToDevice, s));
  if (R.gates) MHL_CUDA(cudaMemcpyAsync(R.gates, gate, (size_t)m.H * m.R * 4, cudaMemcpyDeviceToDevice, s));
  return check_kernels(p);
}

// B5, B3, B6 for one rank's local heads; input dY [T_g][HD], output dXs rows into `dxout` [T_g][HD]
// (dxout == nullptr: B6 is left to the caller, which runs it per HP destination block)
mhl_status moe_backward_local(mhl_plan p, const RankPtrs& R, const void* dY, void* dxout, cudaStream_t s,
                              void* dxout_r = nullptr) {
  const Dims& m = p->m;
  const SavedLayout S = saved_layout(m);
  const BwdLayout B = bwd_layout(m);
  const void* Xs = R.saved + S.Xs;
  const void* Xr = R.saved + S.Xs + (m.rtok ? (size_t)m.HD * m.el : 0);   // routing sub-tokens
  const int32_t* idx = (const int32_t*)(R.saved + S.idx);
  const float* gate = (const float*)(R.saved + S.gate);
  const mhl::Routing rt = routing_view(m, R.saved);
  void* dXrep = R.ws + B.dXrep;
  float* dg = (float*)(R.ws + B.dg);
  float* dS = (float*)(R.ws + B.dS);
  void* dH = R.ws + B.dH;
  void* gA = R.ws + B.gA;
  const bool tc = !m.simt && mhl::expert_bwd_sm100_supported(m.d_h, m.d_e);
  const bool fused = bwd_fused(m);
  p->paths |= tc ? MHL_PATH_EXPERT_BWD_TC : MHL_PATH_EXPERT_BWD_SIMT;
  if (fused) p->paths |= MHL_PATH_EXPERT_BWD_FUSED;
  // the all-zero row T of dY (padding rows of every expert tile gather it)
  MHL_CUDA(cudaMemsetAsync(static_cast<char*>(const_cast<void*>(dY)) + (size_t)m.T_g * m.HD * m.el, 0,
                           (size_t)m.HD * m.el, s));
  {
    MHL_SPAN("B5_expert_bwd_dx");
    if (fused) {
      if (!mhl::launch_expert_bwd_fused_sm100(rt, Xs, m.XW, dY, m.HD, R.W1, R.W2, m.d_h, m.d_e, dXrep, dg, dH, gA,
                                              p->num_sms, s))
        return fail(MHL_ERR_CUDA, "fused expert backward: TMA tensor-map encoding failed");
    } else if (tc)
      mhl::launch_expert_bwd_sm100(rt, Xs, m.XW, dY, m.HD, R.W1, R.W2, m.d_h, m.d_e, dXrep, dg, dH, gA, nullptr,
                                   nullptr, nullptr, nullptr, p->num_sms, s, true, false);
    else
      mhl::launch_expert_bwd_simt(m.dtype, rt, Xs, m.XW, dY, m.HD, R.W1, R.W2, m.d_h, m.d_e, dXrep, dg, dH, gA, s);
  }
  // B3 (needs only K1's dg) runs before K2, which folds the router term dS W_r^T into dXrep
  float* W_rT = (float*)(R.ws + B.W_rT);
  {
    MHL_SPAN("B3_router_bwd");
    if (!m.simt && m.T_g > 0 && mhl::router_bwd_sm100_supported(m.d_h, m.N_e, m.k)) {
      if (!mhl::launch_router_bwd_sm100(Xr, m.XW, idx, gate, dg, m.H, m.T_g, m.k, m.d_h, m.N_e, dS,
                                        (float*)(R.ws + B.dwr_part),
                                        // token chunks per head from T and the GLOBAL head count only,
                                        // so the partial-sum order (dW_r bits) depends neither on G
                                        // nor on the device's SM count
                                        m.n_rbwd,
                                        R.dW_r, s))
        return fail(MHL_ERR_CUDA, "router backward: TMA tensor-map encoding failed");
      p->paths |= MHL_PATH_ROUTER_BWD_TC;
    } else {
      p->paths |= MHL_PATH_ROUTER_BWD_SIMT;
      mhl::launch_router_bwd(m.dtype, Xr, m.XW, idx, gate, dg, m.H, m.T_g, m.k, m.d_h, m.N_e, dS,
                             (float*)(R.ws + B.dwr_part), R.dW_r, s);
    }
    // dS in clustered-row order for K2's router term: a separate scatter kernel (20 us faster than
    // scattering from inside the router backward, r1e)
    if (tc && !fused && !m.rtok) { mhl::launch_sort_ds(rt, dS, (float*)(R.ws + B.dS_s), s); p->launches++; }
    mhl::launch_transpose_wr(R.W_r, W_rT, m.H, m.d_h, m.N_e, s);
  }
  // windowed (NEXT-1): the dX GEMM and B6 alternate window by window after the dW kernel
  const bool win_b = tc && dxout && windowed(m);
  if (tc && !fused && !win_b) {
    MHL_SPAN("B5_expert_dx_gemm");
    if (!mhl::launch_expert_dx_gemm_sm100(rt, R.W1, m.d_h, m.d_e, dH, dXrep,
                                          m.rtok ? nullptr : (const float*)(R.ws + B.dS_s), W_rT,
                                          p->num_sms, s))
      return fail(MHL_ERR_CUDA, "expert dX GEMM: TMA tensor-map encoding failed");
  }
  if (R.dW1 || R.dW2) {
    MHL_SPAN("B5_expert_bwd_dw");
    if (tc) {
      mhl::launch_dw_parts(rt, (mhl::Tile*)(R.saved + S.chunks), (int32_t*)(R.saved + S.nchunks),
                           (int32_t*)(R.saved + S.cbase), (int32_t*)(R.saved + S.ccount),
                           (int32_t*)(R.saved + S.pbase), (int32_t*)(R.saved + S.pcount), s);
      p->launches++;
    }
    if (tc)
      mhl::launch_expert_bwd_sm100(rt, Xs, m.XW, dY, m.HD, R.W1, R.W2, m.d_h, m.d_e, dXrep, dg, dH, gA,
                                   (float*)(R.ws + B.dw_part), (int*)(R.ws + B.dw_done), R.dW1, R.dW2,
                                   p->num_sms, s, false, true);
    else
      mhl::launch_expert_dw_simt(m.dtype, rt, Xs, m.XW, dY, m.HD, dH, gA, m.d_h, m.d_e, R.dW1, R.dW2, s);
  }
  if (win_b) {
    const int32_t* win = (const int32_t*)(R.saved + S.win);
    for (int h = 0; h < m.H; ++h)
      for (int w = 0; w < mhl::kWindows; ++w) {
        mhl::Routing rw = rt;
        rw.trange = win + ((size_t)h * mhl::kWindows + w) * 4;
        {
          MHL_SPAN("B5_expert_dx_gemm");
          if (!mhl::launch_expert_dx_gemm_sm100(rw, R.W1, m.d_h, m.d_e, dH, dXrep, (const float*)(R.ws + B.dS_s),
                                                W_rT, p->num_sms, s))
            return fail(MHL_ERR_CUDA, "expert dX GEMM: TMA tensor-map encoding failed");
        }
        MHL_SPAN("B6_combine_bwd");
        mhl::launch_combine_window(m.dtype, rt, dXrep, m.d_h, dxout, m.Din, h, rw.trange + 2, m.T_g / mhl::kWindows,
                                   true, s);
      }
    p->paths |= MHL_PATH_WINDOWED_COMBINE;
    p->launches += 2 * m.H * mhl::kWindows - 2;
  } else if (dxout) {
    MHL_SPAN("B6_combine_bwd");
    combine_bwd(m, rt, dXrep, dS, W_rT, tc && !fused, dxout, m.Din, dxout_r, m.Din, s, 0, -1);
  }
  // K1 + K2 + dW (+ its in-kernel reduce) + router (2) + transpose + combine on the tensor-core path
  // (the fused kernel replaces K1 + K2)
  p->launches += (tc ? (fused ? 6 : 7) : (R.dW1 || R.dW2 ? 6 : 5)) - (dxout ? 0 : 1);
  return check_kernels(p);
}

RankPtrs rank_view(mhl_plan p, int r, void* saved, void* ws, const void* x, void* out, const void* dout,
                   const mhl_weights* w, const mhl_grads* g, int32_t* topk_idx, float* gates) {
  const Dims& m = p->m;
  const size_t sv = saved_layout(m).total;
  const size_t wsz = std::max(fwd_layout(m).total, bwd_layout(m).total);
  const int vr = m.loopback ? r : 0;            // region index
  const int hp = m.loopback ? r : 0;            // head-block index inside the weight tensors
  RankPtrs R{};
  R.saved = static_cast<char*>(saved) + (size_t)vr * sv;
  R.ws = static_cast<char*>(ws) + (size_t)vr * wsz;
  const size_t tok = (size_t)m.T_loc * m.d * m.el * (m.loopback ? r : 0);
  R.x = x ? at(x, tok) : nullptr;
  R.out = out ? at(out, tok) : nullptr;
  R.dout = dout ? at(dout, tok) : nullptr;
  const size_t H = m.H;
  R.W_r = w->W_r + (size_t)hp * H * m.d_h * m.N_e;
  R.bias = w->bias + (size_t)hp * H * m.N_e;
  const size_t we = (size_t)hp * H * m.N_e * m.d_e * m.d_h;
  R.W1 = at(w->W1, we * m.el);
  R.W2 = at(w->W2, we * m.el);
  if (g) {
    R.dW_r = g->dW_r ? g->dW_r + (size_t)hp * H * m.d_h * m.N_e : nullptr;
    R.dW1 = g->dW1 ? g->dW1 + we : nullptr;
    R.dW2 = g->dW2 ? g->dW2 + we : nullptr;
  }
  R.topk_idx = topk_idx ? topk_idx + (size_t)hp * H * m.R : nullptr;
  R.gates = gates ? gates + (size_t)hp * H * m.R : nullptr;
  return R;
}

mhl_status check_ws(mhl_plan p, const void* saved, const void* ws, size_t ws_bytes) {
  if (!p) return fail(MHL_ERR_INVALID_ARGUMENT, "NULL plan");
  if (!saved || !ws) return fail(MHL_ERR_INVALID_ARGUMENT, "NULL saved/workspace");
  if (ws_bytes < p->info.workspace_bytes)
    return fail(MHL_ERR_WORKSPACE_TOO_SMALL, "workspace_bytes < hp_plan_info().workspace_bytes");
  return MHL_OK;
}

}  // namespace

extern "C" {

mhl_status hp_plan_query(const mhl_config* cfg, mhl_plan_info* info) {
  if (!cfg || !info) return fail(MHL_ERR_INVALID_ARGUMENT, "NULL argument");
  Dims m;
  MHL_TRY(make_dims(cfg, &m));
  fill_info(m, info);
  return MHL_OK;
}

mhl_status mhl_get_unique_id(uint8_t id[128]) {
  if (!id) return fail(MHL_ERR_INVALID_ARGUMENT, "NULL id");
  NcclApi& api = nccl();
  if (!api.loaded) return fail(MHL_ERR_NCCL, "libnccl.so.2 could not be loaded");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId uid;
  MHL_NCCL(api.GetUniqueId(&uid));
  memcpy(id, &uid, 128);
  return MHL_OK;
}

mhl_status hp_plan(const mhl_config* cfg, const uint8_t* nccl_id, mhl_plan* out) {
  if (!cfg || !out) return fail(MHL_ERR_INVALID_ARGUMENT, "NULL argument");
  *out = nullptr;
  Dims m;
  MHL_TRY(make_dims(cfg, &m));
  const bool need_nccl = m.G > 1 && !m.loopback;
  if (need_nccl != (nccl_id != nullptr))
    return fail(MHL_ERR_INVALID_ARGUMENT, "nccl_id must be non-NULL iff world_size > 1 without LOOPBACK");
  mhl_plan p = new mhl_plan_s();
  p->cfg = *cfg;
  p->m = m;
  fill_info(m, &p->info);
  auto cleanup = [&](mhl_status s) { hp_plan_destroy(p); return s; };
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cleanup(fail(MHL_ERR_CUDA, "no CUDA device"));
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return cleanup(fail(MHL_ERR_CUDA, "cudaGetDeviceProperties"));
  if (prop.major != 10) return cleanup(fail(MHL_ERR_UNSUPPORTED, "this library is built for sm_100a (B200)"));
  p->num_sms = prop.multiProcessorCount;
  if (const char* f = getenv("MHL_FAULT_INJECT")) {
    const std::string v(f);
    p->fault = v == "gates" ? 1 : v == "out" ? 2 : v == "dx" ? 3 : v == "dW1" ? 4 : 0;
    if (p->fault == 0 && !v.empty()) return cleanup(fail(MHL_ERR_INVALID_ARGUMENT, "MHL_FAULT_INJECT: gates|out|dx|dW1"));
  }
  if (cublasLtCreate(&p->lt) != CUBLAS_STATUS_SUCCESS) return cleanup(fail(MHL_ERR_CUDA, "cublasLtCreate"));
  if (cudaMalloc(&p->blas_ws, p->blas_ws_bytes) != cudaSuccess) return cleanup(fail(MHL_ERR_CUDA, "cudaMalloc"));
  if (cudaMalloc(&p->dflag, 16) != cudaSuccess || cudaMemset(p->dflag, 0, 16) != cudaSuccess)
    return cleanup(fail(MHL_ERR_CUDA, "cudaMalloc flag"));
  if (m.G > 1) {
    if (cudaStreamCreateWithFlags(&p->comm_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->ev_prod, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->ev_comm, cudaEventDisableTiming) != cudaSuccess)
      return cleanup(fail(MHL_ERR_CUDA, "comm stream / events"));
    for (auto& e : p->ev_chunk)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
      return cleanup(fail(MHL_ERR_CUDA, "comm stream / events"));
  }
  if (need_nccl) {
    NcclApi& api = nccl();
    if (!api.loaded) return cleanup(fail(MHL_ERR_NCCL, "libnccl.so.2 could not be loaded"));
    ncclUniqueId uid;
    memcpy(&uid, nccl_id, 128);
    ncclResult_t r = api.CommInitRank(&p->comm, m.G, uid, m.rank);
    if (r != ncclSuccess) return cleanup(fail(MHL_ERR_NCCL, "ncclCommInitRank failed"));
  }
  *out = p;
  return MHL_OK;
}

mhl_status hp_plan_info(mhl_plan p, mhl_plan_info* info) {
  if (!p || !info) return fail(MHL_ERR_INVALID_ARGUMENT, "NULL argument");
  *info = p->info;
  return MHL_OK;
}

mhl_status hp_plan_destroy(mhl_plan p) {
  if (!p) return MHL_OK;
  if (p->comm && nccl().CommDestroy) nccl().CommDestroy(p->comm);
  if (p->lt) cublasLtDestroy(p->lt);
  if (p->blas_ws) cudaFree(p->blas_ws);
  if (p->dflag) cudaFree(p->dflag);
  for (int i = 0; i < 2; ++i)
    for (cudaEvent_t e : {p->ev_x[i], p->ev_dout[i], p->ev_fwd[i], p->ev_out[i], p->ev_bwd[i], p->ev_dx[i]})
      if (e) cudaEventDestroy(e);
  if (p->ev_drain) cudaEventDestroy(p->ev_drain);
  if (p->h2d_stream) cudaStreamDestroy(p->h2d_stream);
  if (p->comm_stream) cudaStreamDestroy(p->comm_stream);
  for (cudaEvent_t e : {p->ev_prod, p->ev_comm})
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : p->ev_chunk)
    if (e) cudaEventDestroy(e);
  if (p->d2h_stream) cudaStreamDestroy(p->d2h_stream);
  for (auto e : p->pool) cudaEventDestroy(e);
  delete p;
  return MHL_OK;
}

namespace {
mhl_status forward_impl(mhl_plan p, const void* x, const mhl_weights* w, void* out, void* saved, void* workspace,
                        size_t workspace_bytes, int32_t* topk_idx, float* gates, void* stream) {
  MHL_TRY(check_ws(p, saved, workspace, workspace_bytes));
  if (!x || !w || !out || !w->W_in || !w->W_out || !w->W_r || !w->bias || !w->W1 || !w->W2)
    return fail(MHL_ERR_INVALID_ARGUMENT, "NULL tensor");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const Dims& m = p->m;
  const int VR = m.loopback ? m.G : 1;
  const SavedLayout S = saved_layout(m);
  const FwdLayout F = fwd_layout(m);
  Gemm gemm{p, s};
  std::vector<RankPtrs> ranks;
  for (int r = 0; r < VR; ++r)
    ranks.push_back(rank_view(p, r, saved, workspace, x, out, nullptr, w, nullptr, topk_idx, gates));
  const size_t blk = (size_t)m.T_loc * m.HD * m.el;     // gather block (head outputs)
  const size_t blk_s = (size_t)m.T_loc * m.XW * m.el;  // scatter block (sub-tokens [+ routing sub-tokens])
  if (m.G == 1) {
    const RankPtrs& R = ranks[0];
    {
      MHL_SPAN("F1_proj_in");   // F1: Xs = x W_in^T (Eq. 5; [x | r] parts with routing tokens)
      MHL_TRY(gemm(false, true, m.T_loc, m.Din, m.d, R.x, m.d, w->W_in, m.d, R.saved + S.Xs, m.Din, false, 0.0f));
    }
    MHL_TRY(moe_forward_local(p, R, R.saved + S.cat, s));   // F3-F6
    MHL_SPAN("F8_proj_out");     // F8: out = cat W_out^T (Eq. 6)
    MHL_TRY(gemm(false, true, m.T_loc, m.d, m.D, R.saved + S.cat, m.D, w->W_out, m.D, R.out, m.d, false, 0.0f));
    return check_kernels(p);
  }
  auto rank_of = [&](int v) { return m.loopback ? v : m.rank; };
  // F1 + F2: destination block q of Xs = x W_in[q]^T is sent as soon as its GEMM is done
  {
    MHL_SPAN("F1F2_proj_in_a2a");
    Xfer X;
    X.blk = blk_s; X.rows = m.T_loc;
    for (auto& R : ranks) { X.send.push_back(R.ws + F.send1); X.recv.push_back(R.saved + S.Xs); }
    const int C = a2a_chunks(m.T_loc);
    MHL_TRY(hp_exchange(p, X, s, [&](int c, int i) -> mhl_status {
      const int64_t r0 = chunk_row(m.T_loc, C, c), nr = chunk_row(m.T_loc, C, c + 1) - r0;
      for (int v = 0; v < VR; ++v) {
        const RankPtrs& R = ranks[v];
        const int rk = rank_of(v), q = (rk + i) % m.G;
        char* dst = (i == 0 ? R.saved + S.Xs + rk * blk_s : R.ws + F.send1 + q * blk_s) + r0 * m.XW * m.el;
        const char* xr = at(R.x, (size_t)r0 * m.d * m.el);
        MHL_TRY(gemm(false, true, nr, m.HD, m.d, xr, m.d, at(w->W_in, (size_t)q * m.HD * m.d * m.el), m.d,
                     dst, m.XW, false, 0.0f));
        if (m.rtok)   // routing sub-tokens of q's heads: W_in rows D + q*HD.., same block
          MHL_TRY(gemm(false, true, nr, m.HD, m.d, xr, m.d,
                       at(w->W_in, ((size_t)m.D + (size_t)q * m.HD) * m.d * m.el), m.d,
                       dst + (size_t)m.HD * m.el, m.XW, false, 0.0f));
      }
      return MHL_OK;
    }, [](int, int64_t, int64_t) { return MHL_OK; }, [] { return MHL_OK; }));
  }
  // F3-F5 per rank
  for (int v = 0; v < VR; ++v) MHL_TRY(moe_forward_local(p, ranks[v], nullptr, s));
  // F6 + F7: the combine of destination block q (its tokens' head outputs) is sent as soon as it is
  // done; received blocks are placed in their column block of cat [T_loc][D]
  {
    MHL_SPAN("F6F7_combine_a2a");
    Xfer X;
    X.blk = blk; X.rows = m.T_loc; X.row_bytes = (size_t)m.HD * m.el; X.pitch = (size_t)m.D * m.el;
    for (auto& R : ranks) {
      X.send.push_back(R.ws + F.send2); X.recv.push_back(R.ws + F.recv2); X.place.push_back(R.saved + S.cat);
    }
    const int C = a2a_chunks(m.T_loc);
    MHL_TRY(hp_exchange(p, X, s, [&](int c, int i) -> mhl_status {
      const int64_t r0 = chunk_row(m.T_loc, C, c), nr = chunk_row(m.T_loc, C, c + 1) - r0;
      for (int v = 0; v < VR; ++v) {
        const RankPtrs& R = ranks[v];
        const int rk = rank_of(v), q = (rk + i) % m.G;
        const mhl::Routing rt = routing_view(m, R.saved);
        if (i == 0)
          mhl::launch_combine_fwd(m.dtype, rt, R.ws + F.Yrep, m.d_h,
                                  R.saved + S.cat + r0 * X.pitch + rk * X.row_bytes, m.D, s, (int64_t)q * m.T_loc + r0,
                                  nr);
        else
          mhl::launch_combine_fwd(m.dtype, rt, R.ws + F.Yrep, m.d_h, R.ws + F.send2 + q * blk + r0 * X.row_bytes, m.HD,
                                  s, (int64_t)q * m.T_loc + r0, nr);
        p->launches++;
      }
      return MHL_OK;
    }, [&](int, int64_t r0, int64_t nr) -> mhl_status {
      // F8 on the token chunk whose head outputs have all arrived: out = cat W_out^T (Eq. 6)
      for (auto& R : ranks) {
        MHL_SPAN("F8_proj_out");
        MHL_TRY(gemm(false, true, nr, m.d, m.D, R.saved + S.cat + r0 * X.pitch, m.D, w->W_out, m.D,
                     at(R.out, (size_t)r0 * m.d * m.el), m.d, false, 0.0f));
      }
      return MHL_OK;
    }, [] { return MHL_OK; }));
  }
  return check_kernels(p);
}

mhl_status backward_impl(mhl_plan p, const void* x, const mhl_weights* w, const void* d_out, const void* saved,
                         void* dx, const mhl_grads* grads, void* workspace, size_t workspace_bytes, void* stream) {
  MHL_TRY(check_ws(p, saved, workspace, workspace_bytes));
  if (!x || !w || !d_out || !dx || !grads) return fail(MHL_ERR_INVALID_ARGUMENT, "NULL tensor");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const Dims& m = p->m;
  const int VR = m.loopback ? m.G : 1;
  const SavedLayout S = saved_layout(m);
  const BwdLayout B = bwd_layout(m);
  Gemm gemm{p, s};
  std::vector<RankPtrs> ranks;
  for (int r = 0; r < VR; ++r)
    ranks.push_back(rank_view(p, r, const_cast<void*>(saved), workspace, x, dx, d_out, w, grads, nullptr, nullptr));
  const size_t blk = (size_t)m.T_loc * m.HD * m.el;
  // the two projection weight gradients (rank partials, R19; loopback: all virtual ranks), plain or
  // as the deterministic chunk tree (MHL_FLAG_DET_DP)
  std::vector<char*> dp_part;
  for (auto& R : ranks) dp_part.push_back(R.ws + B.dp_part);
  auto dW_out_grad = [&]() -> mhl_status {
    if (!grads->dW_out) return MHL_OK;
    if (m.det_dp)
      return det_wgrad(p, gemm, VR, [&](int v) { return std::make_pair(ranks[v].dout, (const void*)(ranks[v].saved + S.cat)); },
                       m.d, m.D, m.d, m.D, dp_part, grads->dW_out, s);
    for (int v = 0; v < VR; ++v)
      MHL_TRY(gemm(true, false, m.d, m.D, m.T_loc, ranks[v].dout, m.d, ranks[v].saved + S.cat, m.D, grads->dW_out, m.D,
                   true, v == 0 ? 0.0f : 1.0f));
    return MHL_OK;
  };
  auto dW_in_grad = [&]() -> mhl_status {
    if (!grads->dW_in) return MHL_OK;
    if (m.det_dp)
      return det_wgrad(p, gemm, VR, [&](int v) { return std::make_pair((const void*)(ranks[v].ws + B.dXs), ranks[v].x); },
                       m.Din, m.d, m.Din, m.d, dp_part, grads->dW_in, s);
    for (int v = 0; v < VR; ++v)
      MHL_TRY(gemm(true, false, m.Din, m.d, m.T_loc, ranks[v].ws + B.dXs, m.Din, ranks[v].x, m.d, grads->dW_in, m.d,
                   true, v == 0 ? 0.0f : 1.0f));
    return MHL_OK;
  };
  if (m.G == 1) {
    const RankPtrs& R = ranks[0];
    {
      MHL_SPAN("B8_proj_out_bwd");   // B8: dcat = dout W_out, dW_out = dout^T cat
      MHL_TRY(gemm(false, false, m.T_loc, m.D, m.d, R.dout, m.d, w->W_out, m.D, R.ws + B.dY, m.D, false, 0.0f));
      MHL_TRY(dW_out_grad());
    }
    MHL_TRY(moe_backward_local(p, R, R.ws + B.dY, R.ws + B.dXs, s,
                               m.rtok ? R.ws + B.dXs + (size_t)m.D * m.el : nullptr));   // B5, B3, B6
    MHL_SPAN("B1_proj_in_bwd");      // B1: dx = dXs W_in, dW_in = dXs^T x  (dXs = [dX | dR] with routing tokens)
    MHL_TRY(gemm(false, false, m.T_loc, m.d, m.Din, R.ws + B.dXs, m.Din, w->W_in, m.d, R.out, m.d, false, 0.0f));
    MHL_TRY(dW_in_grad());
    return check_kernels(p);
  }
  auto rank_of = [&](int v) { return m.loopback ? v : m.rank; };
  // B8 + B7: destination block q of dcat = dout W_out[:, q] is sent as soon as its GEMM is done; the
  // dW_out GEMM (rank partial; loopback: summed over virtual ranks) overlaps the last exchanges
  {
    MHL_SPAN("B8B7_proj_out_bwd_a2a");
    Xfer X;
    X.blk = blk; X.rows = m.T_loc;
    for (auto& R : ranks) { X.send.push_back(R.ws + B.send3); X.recv.push_back(R.ws + B.dY); }
    const int C = a2a_chunks(m.T_loc);
    MHL_TRY(hp_exchange(p, X, s, [&](int c, int i) -> mhl_status {
      const int64_t r0 = chunk_row(m.T_loc, C, c), nr = chunk_row(m.T_loc, C, c + 1) - r0;
      for (int v = 0; v < VR; ++v) {
        const RankPtrs& R = ranks[v];
        const int rk = rank_of(v), q = (rk + i) % m.G;
        char* dst = (i == 0 ? R.ws + B.dY + rk * blk : R.ws + B.send3 + q * blk) + r0 * m.HD * m.el;
        MHL_TRY(gemm(false, false, nr, m.HD, m.d, at(R.dout, (size_t)r0 * m.d * m.el), m.d,
                     at(w->W_out, (size_t)q * m.HD * m.el), m.D, dst, m.HD, false, 0.0f));
      }
      return MHL_OK;
    }, [](int, int64_t, int64_t) { return MHL_OK; }, [&]() -> mhl_status { return dW_out_grad(); }));
  }
  // B5, B3 per rank
  for (int v = 0; v < VR; ++v) MHL_TRY(moe_backward_local(p, ranks[v], ranks[v].ws + B.dY, nullptr, s));
  // B6 + B2: the dX combine of destination block q is sent as soon as it is done; received blocks
  // are placed in their column block of dXs [T_loc][D]
  {
    MHL_SPAN("B6B2_combine_bwd_a2a");
    Xfer X;
    const size_t blk4 = (size_t)m.T_loc * m.XW * m.el;   // [dX | dR] rows with routing tokens
    X.blk = blk4; X.rows = m.T_loc; X.row_bytes = (size_t)m.HD * m.el; X.pitch = (size_t)m.Din * m.el;
    X.parts = m.rtok ? 2 : 1; X.part_dst = (size_t)m.D * m.el;
    for (auto& R : ranks) {
      X.send.push_back(R.ws + B.send4); X.recv.push_back(R.ws + B.recv4); X.place.push_back(R.ws + B.dXs);
    }
    const int C = a2a_chunks(m.T_loc);
    MHL_TRY(hp_exchange(p, X, s, [&](int c, int i) -> mhl_status {
      const int64_t r0 = chunk_row(m.T_loc, C, c), nr = chunk_row(m.T_loc, C, c + 1) - r0;
      for (int v = 0; v < VR; ++v) {
        const RankPtrs& R = ranks[v];
        const int rk = rank_of(v), q = (rk + i) % m.G;
        const mhl::Routing rt = routing_view(m, R.saved);
        char* dst = i == 0 ? R.ws + B.dXs + r0 * X.pitch + rk * X.row_bytes
                           : R.ws + B.send4 + q * blk4 + r0 * (size_t)m.XW * m.el;
        char* dst_r = i == 0 ? dst + X.part_dst : dst + X.row_bytes;
        combine_bwd(m, rt, R.ws + B.dXrep, (const float*)(R.ws + B.dS), (const float*)(R.ws + B.W_rT),
                    !m.simt && mhl::expert_bwd_sm100_supported(m.d_h, m.d_e) && !bwd_fused(m), dst,
                    i == 0 ? m.Din : m.XW,
                    dst_r, i == 0 ? m.Din : m.XW, s, (int64_t)q * m.T_loc + r0, nr);
        p->launches += m.rtok ? 2 : 1;
      }
      return MHL_OK;
    }, [&](int, int64_t r0, int64_t nr) -> mhl_status {
      // B1's dgrad on the token chunk whose dXs blocks have all arrived: dx = dXs W_in
      for (int v = 0; v < VR; ++v) {
        MHL_SPAN("B1_proj_in_bwd");
        const RankPtrs& R = ranks[v];
        MHL_TRY(gemm(false, false, nr, m.d, m.Din, R.ws + B.dXs + r0 * X.pitch, m.Din, w->W_in, m.d,
                     at(R.out, (size_t)r0 * m.d * m.el), m.d, false, 0.0f));
      }
      return MHL_OK;
    }, [] { return MHL_OK; }));
  }
  // B1's wgrad: dW_in = dXs^T x (rank partial; loopback: summed in rank order)
  {
    MHL_SPAN("B1_proj_in_bwd");
    MHL_TRY(dW_in_grad());
  }
  return check_kernels(p);
}

}  // namespace

mhl_status mhlmoe_forward(mhl_plan p, const void* x, const mhl_weights* w, void* out, void* saved, void* workspace,
                          size_t workspace_bytes, int32_t* topk_idx, float* gates, void* stream) {
  MHL_TRY(forward_impl(p, x, w, out, saved, workspace, workspace_bytes, topk_idx, gates, stream));
  if (p->fault == 2)
    mhl::launch_scale(p->m.dtype, out, p->m.T_loc * (p->m.loopback ? p->m.G : 1) * p->m.d, 1.001f,
                      static_cast<cudaStream_t>(stream));
  return check_kernels(p);
}

mhl_status mhlmoe_backward(mhl_plan p, const void* x, const mhl_weights* w, const void* d_out, const void* saved,
                           void* dx, const mhl_grads* grads, void* workspace, size_t workspace_bytes, void* stream) {
  MHL_TRY(backward_impl(p, x, w, d_out, saved, dx, grads, workspace, workspace_bytes, stream));
  const Dims& m = p->m;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (p->fault == 3) mhl::launch_scale(m.dtype, dx, m.T_loc * (m.loopback ? m.G : 1) * m.d, 1.001f, s);
  if (p->fault == 4 && grads->dW1)
    mhl::launch_scale(0, grads->dW1, (int64_t)(m.loopback ? m.N_h : m.H) * m.N_e * m.d_e * m.d_h, 1.001f, s);
  return check_kernels(p);
}

namespace {
// Host-buffer training step.  Copies run on two plan-owned side streams, one per link direction,
// ordered against the compute stream by events; consecutive calls alternate between two device
// staging slots, so a call's uploads need only wait for the backward of the call two steps back.
// Within a call the d_out upload overlaps the forward and the out download the backward; across
// calls the next call's uploads overlap this call's backward and downloads.  `sync_outputs` makes
// `stream` wait for this call's downloads (outputs on the host when the stream completes);
// otherwise mhl_host_drain provides that point for all calls so far.
mhl_status host_step(mhl_plan p, const void* x_host, const void* dout_host, const mhl_weights* w, void* out_host,
                     void* dx_host, const mhl_grads* grads, void* io, void* saved, void* workspace,
                     size_t workspace_bytes, void* stream, bool sync_outputs) {
  if (!p || !x_host || !dout_host || !out_host || !dx_host || !io)
    return fail(MHL_ERR_INVALID_ARGUMENT, "NULL argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const Dims& m = p->m;
  const size_t n = (size_t)m.T_loc * (m.loopback ? m.G : 1) * m.d * m.el;
  const size_t a = align_up(n);
  const int sl = (int)(p->host_steps & 1);
  char* xd = static_cast<char*>(io) + (size_t)sl * 4 * a;
  char* dd = xd + a;
  char* od = dd + a;
  char* gd = od + a;
  if (!p->h2d_stream) {
    MHL_CUDA(cudaStreamCreateWithFlags(&p->h2d_stream, cudaStreamNonBlocking));
    MHL_CUDA(cudaStreamCreateWithFlags(&p->d2h_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i)
      for (cudaEvent_t* e : {&p->ev_x[i], &p->ev_dout[i], &p->ev_fwd[i], &p->ev_out[i], &p->ev_bwd[i], &p->ev_dx[i]})
        MHL_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    MHL_CUDA(cudaEventCreateWithFlags(&p->ev_drain, cudaEventDisableTiming));
  }
  cudaStream_t up = p->h2d_stream, down = p->d2h_stream;
  const bool live = p->io_live[sl];
  if (live) MHL_CUDA(cudaStreamWaitEvent(up, p->ev_bwd[sl], 0));     // slot's x / d_out last read there
  MHL_CUDA(cudaMemcpyAsync(xd, x_host, n, cudaMemcpyHostToDevice, up));
  MHL_CUDA(cudaEventRecord(p->ev_x[sl], up));
  MHL_CUDA(cudaMemcpyAsync(dd, dout_host, n, cudaMemcpyHostToDevice, up));
  MHL_CUDA(cudaEventRecord(p->ev_dout[sl], up));
  MHL_CUDA(cudaStreamWaitEvent(s, p->ev_x[sl], 0));
  if (live) MHL_CUDA(cudaStreamWaitEvent(s, p->ev_out[sl], 0));      // slot's previous out download
  MHL_TRY(mhlmoe_forward(p, xd, w, od, saved, workspace, workspace_bytes, nullptr, nullptr, stream));
  MHL_CUDA(cudaEventRecord(p->ev_fwd[sl], s));
  MHL_CUDA(cudaStreamWaitEvent(down, p->ev_fwd[sl], 0));
  MHL_CUDA(cudaMemcpyAsync(out_host, od, n, cudaMemcpyDeviceToHost, down));
  MHL_CUDA(cudaEventRecord(p->ev_out[sl], down));
  MHL_CUDA(cudaStreamWaitEvent(s, p->ev_dout[sl], 0));
  if (live) MHL_CUDA(cudaStreamWaitEvent(s, p->ev_dx[sl], 0));       // slot's previous dx download
  MHL_TRY(mhlmoe_backward(p, xd, w, dd, saved, gd, grads, workspace, workspace_bytes, stream));
  MHL_CUDA(cudaEventRecord(p->ev_bwd[sl], s));
  MHL_CUDA(cudaStreamWaitEvent(down, p->ev_bwd[sl], 0));
  MHL_CUDA(cudaMemcpyAsync(dx_host, gd, n, cudaMemcpyDeviceToHost, down));
  MHL_CUDA(cudaEventRecord(p->ev_dx[sl], down));
  p->io_live[sl] = true;
  p->host_steps++;
  if (sync_outputs) {
    MHL_CUDA(cudaStreamWaitEvent(s, p->ev_out[sl], 0));
    MHL_CUDA(cudaStreamWaitEvent(s, p->ev_dx[sl], 0));
  }
  return MHL_OK;
}
}  // namespace

mhl_status mhlmoe_train_step_host(mhl_plan p, const void* x_host, const void* dout_host, const mhl_weights* w,
                                  void* out_host, void* dx_host, const mhl_grads* grads, void* io, void* saved,
                                  void* workspace, size_t workspace_bytes, void* stream) {
  return host_step(p, x_host, dout_host, w, out_host, dx_host, grads, io, saved, workspace, workspace_bytes, stream,
                   true);
}

mhl_status mhlmoe_train_step_host_pipelined(mhl_plan p, const void* x_host, const void* dout_host,
                                            const mhl_weights* w, void* out_host, void* dx_host,
                                            const mhl_grads* grads, void* io, void* saved, void* workspace,
                                            size_t workspace_bytes, void* stream) {
  return host_step(p, x_host, dout_host, w, out_host, dx_host, grads, io, saved, workspace, workspace_bytes, stream,
                   false);
}

mhl_status mhl_host_drain(mhl_plan p, void* stream) {
  if (!p) return fail(MHL_ERR_INVALID_ARGUMENT, "NULL plan");
  if (!p->d2h_stream) return MHL_OK;
  MHL_CUDA(cudaEventRecord(p->ev_drain, p->d2h_stream));
  MHL_CUDA(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), p->ev_drain, 0));
  return MHL_OK;
}

mhl_status mhlmoe_update_bias(mhl_plan p, const void* saved, float* bias, float gamma, void* stream) {
  if (!p || !saved || !bias) return fail(MHL_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!(gamma >= 0.0f) || gamma != gamma) return fail(MHL_ERR_INVALID_ARGUMENT, "gamma must be a finite value >= 0");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const Dims& m = p->m;
  const SavedLayout S = saved_layout(m);
  const int VR = m.loopback ? m.G : 1;
  for (int r = 0; r < VR; ++r) {
    const char* sv = static_cast<const char*>(saved) + (size_t)r * S.total;
    mhl::launch_update_bias((const int32_t*)(sv + S.load), m.H, m.N_e, m.T_g * m.k, gamma,
                            bias + (size_t)r * m.H * m.N_e, s);
    p->launches++;
  }
  return check_kernels(p);
}

mhl_status mhl_check_device_status(mhl_plan p) {
  if (!p) return fail(MHL_ERR_INVALID_ARGUMENT, "NULL plan");
  int32_t f = 0;
  MHL_CUDA(cudaMemcpy(&f, p->dflag, 4, cudaMemcpyDeviceToHost));
  if (f) {
    MHL_CUDA(cudaMemset(p->dflag, 0, 4));
    return fail(MHL_ERR_NONFINITE, "non-finite router score/key encountered (R7)");
  }
  return MHL_OK;
}

uint64_t mhl_launch_count(mhl_plan p) { return p ? p->launches.load() : 0; }

mhl_status mhl_set_step_timing(mhl_plan p, int enable) {
  if (!p) return fail(MHL_ERR_INVALID_ARGUMENT, "NULL plan");
  p->timing = enable != 0;
  p->recs.clear();
  p->pool_used = 0;
  return MHL_OK;
}

int32_t mhl_step_times(mhl_plan p, char* names, size_t names_cap, double* ms, int32_t* calls, int32_t max_steps) {
  if (!p) return -1;
  if (!p->recs.empty()) cudaEventSynchronize(p->recs.back().b);
  std::vector<std::string> order;
  std::vector<double> tot;
  std::vector<int32_t> cnt;
  for (auto& r : p->recs) {
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    size_t i = 0;
    while (i < order.size() && order[i] != r.name) ++i;
    if (i == order.size()) { order.push_back(r.name); tot.push_back(0.0); cnt.push_back(0); }
    tot[i] += t; cnt[i] += 1;
  }
  std::string joined;
  for (size_t i = 0; i < order.size(); ++i) {
    if (i) joined += ",";
    joined += order[i];
    if ((int)i < max_steps) { if (ms) ms[i] = tot[i]; if (calls) calls[i] = cnt[i]; }
  }
  if (names && names_cap) { strncpy(names, joined.c_str(), names_cap - 1); names[names_cap - 1] = 0; }
  p->recs.clear();
  p->pool_used = 0;
  return (int32_t)order.size();
}

uint64_t mhl_a2a_bytes_posted(mhl_plan p) { return p ? p->a2a_bytes_posted : 0; }

mhl_status mhl_dp_reduce(mhl_plan p, float* dW_in, float* dW_out, void* workspace, size_t workspace_bytes,
                         void* stream) {
  if (!p || !workspace) return fail(MHL_ERR_INVALID_ARGUMENT, "NULL argument");
  const Dims& m = p->m;
  if (!m.det_dp) return fail(MHL_ERR_INVALID_ARGUMENT, "mhl_dp_reduce needs a MHL_FLAG_DET_DP plan");
  if (m.G == 1 || m.loopback) return MHL_OK;   // the backward returned the finished tree
  if (workspace_bytes < p->info.workspace_bytes)
    return fail(MHL_ERR_WORKSPACE_TOO_SMALL, "workspace_bytes < hp_plan_info().workspace_bytes");
  NcclApi& api = nccl();
  if (!api.AllGather) return fail(MHL_ERR_NCCL, "ncclAllGather not available");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int wgt = 0; wgt < 2; ++wgt) {
    float* g = wgt == 0 ? dW_in : dW_out;
    if (!g) continue;
    const size_t n = wgt == 0 ? (size_t)m.Din * m.d : (size_t)m.d * m.D;
    if (workspace_bytes < (size_t)m.G * n * 4) return fail(MHL_ERR_WORKSPACE_TOO_SMALL, "mhl_dp_reduce: G x dW bytes");
    float* all = static_cast<float*>(workspace);   // [G][n]: every rank's subtree, rank order = token order
    MHL_NCCL(api.AllGather(g, all, n, ncclFloat32, p->comm, s));
    for (int st = 1; st < m.G; st *= 2)
      for (int i = 0; i + st < m.G; i += 2 * st) mhl::launch_add_inplace(all + (size_t)i * n, all + (size_t)(i + st) * n, n, s);
    MHL_CUDA(cudaMemcpyAsync(g, all, n * 4, cudaMemcpyDeviceToDevice, s));
  }
  return check_kernels(p);
}

uint32_t mhl_kernel_paths(mhl_plan p, int reset) {
  if (!p) return 0;
  return reset ? p->paths.exchange(0u) : p->paths.load();
}

const char* mhl_status_string(mhl_status s) {
  switch (s) {
    case MHL_OK: return "MHL_OK";
    case MHL_ERR_INVALID_ARGUMENT: return "MHL_ERR_INVALID_ARGUMENT";
    case MHL_ERR_CONFIG: return "MHL_ERR_CONFIG";
    case MHL_ERR_WORKSPACE_TOO_SMALL: return "MHL_ERR_WORKSPACE_TOO_SMALL";
    case MHL_ERR_UNSUPPORTED: return "MHL_ERR_UNSUPPORTED";
    case MHL_ERR_CUDA: return "MHL_ERR_CUDA";
    case MHL_ERR_NCCL: return "MHL_ERR_NCCL";
    case MHL_ERR_NONFINITE: return "MHL_ERR_NONFINITE";
  }
  return "MHL_ERR_UNKNOWN";
}

const char* mhl_last_error(void) { return g_last_error.c_str(); }

}  // extern "C"
