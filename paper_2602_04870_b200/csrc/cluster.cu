// cluster.cu — F4: token clustering (Fig. 2, P:941-P:949, P:970-P:972).
//
// Replicas r = t*k + j of each head are stably sorted by expert (a counting sort:
// deterministic, integer-exact, dropless P:566/P:977):
//   pos(r) = off[e] + tilepref[tile(t)][e] + rank of r among the router tile's replicas of e
// where tilepref is the exclusive scan over router tiles of the per-tile expert histogram
// emitted by F3.  Each expert segment is padded to a multiple of seg_align rows (whole 128-row
// tiles; 256 = whole tile pairs for the cta_group::2 kernels, MHL_FLAG_PAIR), so the
// block-sparse mask of Eq. 7 becomes a list of whole 128-row tiles; padding rows point at
// the all-zero sub-token row (token id T) with gate 0 and contribute exactly nothing.
// Outputs per head (Rp = padded row capacity): perm (row -> replica or -1), tok_s (row -> token
// or T), gate_s (row -> gate or 0), pos (replica -> row), off, the tile list (L2-friendly
// (head, part, expert) order, see offsets_kernel) and the list of row-part chunks used by
// the weight-gradient kernel.
#include "kernels.h"

namespace mhl {

namespace {

// (1) per (h, e): exclusive scan over router tiles of hist[h][tile][e]; total -> counts[h][e]
__global__ void __launch_bounds__(256)
tile_prefix_kernel(const int32_t* __restrict__ hist, int32_t* __restrict__ tilepref, int32_t* __restrict__ counts,
                   int n_rt, int N_e) {
  const int e = blockIdx.x, h = blockIdx.y;
  __shared__ int warp_sums[8];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base = 0; base < n_rt; base += 256) {
    const int tt = base + threadIdx.x;
    const size_t o = ((size_t)h * n_rt + tt) * N_e + e;
    const int v = (tt < n_rt) ? hist[o] : 0;
    int incl = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += n;
    }
    if (lane == 31) warp_sums[wid] = incl;
    __syncthreads();
    int wpre = 0;
    for (int w = 0; w < wid; ++w) wpre += warp_sums[w];
    const int c = carry;
    if (tt < n_rt) tilepref[o] = c + wpre + incl - v;
    __syncthreads();
    if (threadIdx.x == 255) carry = c + wpre + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) counts[(size_t)h * N_e + e] = carry;
}

// block-wide exclusive scan over 1024 threads; *total (shared) receives the block sum
__device__ int block_exclusive_scan_1024(int v, int* s_warp, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += n;
  }
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const int w = s_warp[lane];
    int wi = w;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, wi, d);
      if (lane >= d) wi += n;
    }
    s_warp[32 + lane] = wi - w;
    if (lane == 31) *total = wi;
  }
  __syncthreads();
  const int r = s_warp[32 + wid] + incl - v;
  __syncthreads();
  return r;
}

// (2) padded per-head offsets off[h][e] (exclusive scan of the seg_align-padded counts), the
// per-(h, e) tile and dW-chunk bases.  The tile list is ordered (head, part, expert, tile): expert
// e's alignment units are cut into kTileParts contiguous parts (part p = units [p*n/P, (p+1)*n/P)),
// and all experts' part-p tiles come before any part-(p+1) tile.  Within an expert the rows are in
// token order, so the tiles in flight at any moment (consecutive list entries) cover one narrow
// token window of the head across many experts: every sub-token row gathered for them is re-read
// by its other top-k experts while it is still in L2.
// One CTA per head: the global tile / chunk bases of head h are the totals of heads < h, which the
// CTA recomputes itself from `counts` (H*N_e values), so the heads scan in parallel.  Warp p scans
// tile part p over the experts (32 experts per step, carry in a register) and warp 0 the padded
// segment lengths: one barrier in all (the former 1024-thread block scans, one per part and 32
// experts, took 10 us at paper scale, most of it in __syncthreads).
__device__ __forceinline__ int warp_incl_scan(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += n;
  }
  return v;
}

constexpr int kOffsetsThreads = 32 * kTileParts;
__global__ void __launch_bounds__(kOffsetsThreads)
offsets_kernel(const int32_t* __restrict__ counts, int32_t* __restrict__ off, int32_t* __restrict__ tbase,
               int32_t* __restrict__ ntiles, int H, int N_e, int max_tiles, int seg_align) {
  __shared__ int s_red[2][kOffsetsThreads / 32];
  __shared__ int s_ptot[kTileParts];
  const int TPS = seg_align / kExpertBM;                                 // tiles per alignment unit
  const int h = blockIdx.x, lane = threadIdx.x & 31, p = threadIdx.x >> 5;
  auto units = [&](int c) { return (c + seg_align - 1) / seg_align; };  // alignment units of a segment
  // tiles of all heads before h, and of all heads (order-independent integer sums)
  int t_before = 0, t_all = 0;
  for (int i = threadIdx.x; i < H * N_e; i += kOffsetsThreads) {
    const int nt = units(counts[i]) * TPS;
    if (i / N_e < h) t_before += nt;
    t_all += nt;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    t_before += __shfl_xor_sync(0xffffffffu, t_before, d);
    t_all += __shfl_xor_sync(0xffffffffu, t_all, d);
  }
  if (lane == 0) { s_red[0][p] = t_before; s_red[1][p] = t_all; }
  // part p's tile count over the experts
  const int32_t* ch = counts + (size_t)h * N_e;
  auto part_tiles = [&](int e) {
    const int nu = units(ch[e]);
    return TPS * ((p + 1) * nu / kTileParts - p * nu / kTileParts);
  };
  int ptot = 0;
  for (int e = lane; e < N_e; e += 32) ptot += part_tiles(e);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) ptot += __shfl_xor_sync(0xffffffffu, ptot, d);
  if (lane == 0) s_ptot[p] = ptot;
  __syncthreads();
  int carry = 0, tot_t = 0;
  for (int w = 0; w < kOffsetsThreads / 32; ++w) { carry += s_red[0][w]; tot_t += s_red[1][w]; }
  for (int q = 0; q < p; ++q) carry += s_ptot[q];
  // tbase[h][p][e] = tiles of earlier heads + earlier parts of this head + this part's earlier experts
  for (int b = 0; b < N_e; b += 32) {
    const int e = b + lane;
    const int v = e < N_e ? part_tiles(e) : 0;
    const int incl = warp_incl_scan(v);
    if (e < N_e) tbase[((size_t)h * kTileParts + p) * N_e + e] = carry + incl - v;
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (p == 0) {   // padded segment offsets of this head
    int carry_r = 0;
    for (int b = 0; b < N_e; b += 32) {
      const int e = b + lane;
      const int cp = e < N_e ? units(ch[e]) * seg_align : 0;
      const int incl = warp_incl_scan(cp);
      if (e < N_e) off[(size_t)h * (N_e + 1) + e] = carry_r + incl - cp;
      carry_r += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) {
      off[(size_t)h * (N_e + 1) + N_e] = carry_r;
      if (h == 0) *ntiles = min(tot_t, max_tiles);
    }
  }
}

// (2a) dW chunks.  Each head's padded rows [0, R_h) are cut into P equal parts (boundaries rounded
// down to the dW kernel's 64-row step; P = the dW grid, fixed per plan, independent of G), and a
// chunk is a part's intersection with one expert segment.  CTA b of the dW kernel takes part b of
// every head, so every CTA gets the same number of rows; the chunk list is in (head, part,
// expert) = (head, expert, row) order, so each expert's chunks are consecutive ([cbase, +ccount)),
// and its partials are summed in that order (deterministic, problem-derived boundaries).  Chunk
// ids are per-head blocks of P + N_e (the list has gaps between heads).
__device__ __forceinline__ int part_lo(int p, int P, int Rh) {
  return p >= P ? Rh : (int)(((int64_t)p * Rh / P) & ~(int64_t)(kDwStep - 1));
}

__global__ void __launch_bounds__(1024)
dw_parts_kernel(const int32_t* __restrict__ off, int H, int N_e, int P, Tile* __restrict__ chunks, int max_chunks,
                int32_t* __restrict__ nchunks, int32_t* __restrict__ cbase, int32_t* __restrict__ ccount,
                int32_t* __restrict__ pbase, int32_t* __restrict__ pcount) {
  // one CTA per head; head h's chunks live at [h*(P+N_e), ...) (a part adds one chunk per expert
  // segment it touches: at most P + N_e per head), so the heads need no cross-head scan
  __shared__ int s_warp[64];
  __shared__ int s_tot;
  const int h = blockIdx.x;
  const int32_t* o = off + (size_t)h * (N_e + 1);
  const int Rh = o[N_e];
  for (int e = threadIdx.x; e < N_e; e += blockDim.x) { ccount[(size_t)h * N_e + e] = 0; cbase[(size_t)h * N_e + e] = 0; }
  __syncthreads();
  int carry = h * (P + N_e);
  for (int base = 0; base < P; base += 1024) {
    const int p = base + threadIdx.x;
    int cnt = 0, lo = 0, hi = 0, e0 = 0;
    if (p < P) {
      lo = part_lo(p, P, Rh); hi = part_lo(p + 1, P, Rh);
      if (lo < hi) {
        int a = 0, b = N_e;                  // e0 = last expert with o[e] <= lo (its segment holds lo)
        while (a < b) { const int mid = (a + b + 1) >> 1; if (o[mid] <= lo) a = mid; else b = mid - 1; }
        e0 = a;
        for (int e = e0; e < N_e && o[e] < hi; ++e) cnt += o[e + 1] > o[e];
      }
    }
    const int ex = block_exclusive_scan_1024(cnt, s_warp, &s_tot);
    const int tot = s_tot;
    __syncthreads();
    if (p < P) {
      const int cb = carry + ex;
      pbase[(size_t)h * P + p] = cb; pcount[(size_t)h * P + p] = cnt;
      int j = 0;
      for (int e = e0; cnt > 0 && e < N_e && o[e] < hi; ++e) {
        if (o[e + 1] <= o[e]) continue;
        const int r0 = max(lo, o[e]), r1 = min(hi, o[e + 1]), ci = cb + j++;
        if (ci < max_chunks) {
          Tile tl;
          tl.head = h; tl.expert = e; tl.row0 = r0; tl.rows = r1 - r0;
          chunks[ci] = tl;
        }
        if (r0 == o[e]) {                    // the expert's first chunk: count its parts
          int n = 1;
          for (int pp = p + 1; pp < P && part_lo(pp, P, Rh) < o[e + 1]; ++pp)
            n += part_lo(pp, P, Rh) < part_lo(pp + 1, P, Rh);
          cbase[(size_t)h * N_e + e] = ci;
          ccount[(size_t)h * N_e + e] = n;
        }
      }
    }
    carry += tot;
  }
  if (h == 0 && threadIdx.x == 0) *nchunks = min(H * (P + N_e), max_chunks);   // index bound
}

// (2b) one warp per (h, e): its tiles (at the (h, part, e) positions), its dW chunks and the
// padding-row fill of its segment, lanes striding over each list.
__global__ void __launch_bounds__(256)
tiles_kernel(const int32_t* __restrict__ counts, const int32_t* __restrict__ off, const int32_t* __restrict__ tbase,
             Tile* __restrict__ tiles, int max_tiles, int H, int N_e, int64_t Rp, int32_t* __restrict__ perm, int32_t* __restrict__ tok_s,
             float* __restrict__ gate_s, int tok_zero, int seg_align) {
  const int he = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (he >= H * N_e) return;
  const int h = he / N_e, e = he % N_e;
  const int c = counts[he];
  const int TPS = seg_align / kExpertBM;
  const int nu = (c + seg_align - 1) / seg_align;
  const int cp = nu * seg_align;
  const int row_off = off[(size_t)h * (N_e + 1) + e];
  for (int p = 0; p < kTileParts; ++p) {
    const int j0 = TPS * (p * nu / kTileParts), j1 = TPS * ((p + 1) * nu / kTileParts);   // unit-aligned
    const int tb = tbase[((size_t)h * kTileParts + p) * N_e + e];
    for (int j = j0 + lane; j < j1; j += 32) {
      const int ti = tb + (j - j0);
      if (ti < max_tiles) {
        Tile tl;
        tl.head = h; tl.expert = e; tl.row0 = row_off + j * kExpertBM;
        tl.rows = max(0, min(kExpertBM, c - j * kExpertBM));
        tiles[ti] = tl;
      }
    }
  }
  // padding rows of this segment: no replica, zero sub-token, gate 0
  for (int r = row_off + c + lane; r < row_off + cp; r += 32) {
    perm[(size_t)h * Rp + r] = -1;
    tok_s[(size_t)h * Rp + r] = tok_zero;
    gate_s[(size_t)h * Rp + r] = 0.f;
  }
}

// (3) per (h, router tile), 8 warps: warp w owns a contiguous run of the tile's replicas.
// Pass 1 counts each warp's replicas per expert (warp match, no atomics); a per-expert scan over
// the warps gives every warp its stable starting rank; pass 2 recomputes the in-warp ranks and
// scatters perm/pos/tok/gate.  Replica order is preserved within every expert (stable sort).
constexpr int kScatterWarps = 8;
__global__ void __launch_bounds__(kScatterWarps * 32)
scatter_kernel(const int32_t* __restrict__ idx, const float* __restrict__ gate, const int32_t* __restrict__ off,
               const int32_t* __restrict__ tilepref, int32_t* __restrict__ perm, int32_t* __restrict__ pos,
               int32_t* __restrict__ tok_s, float* __restrict__ gate_s, int64_t T, int k, int N_e, int n_rt,
               int64_t Rp) {
  extern __shared__ int sm[];
  int* wcnt = sm;                                     // [kScatterWarps][N_e]
  int* lbase = wcnt + kScatterWarps * N_e;            // [N_e] the tile's expert runs in local sorted order
  int* s_r = lbase + N_e;                             // [kRouterTile * k] replicas in local sorted order
  int* s_e = s_r + kRouterTile * k;                   // [kRouterTile * k] their experts
  const int tt = blockIdx.x, h = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kScatterWarps * N_e; i += blockDim.x) wcnt[i] = 0;
  __syncthreads();
  const int64_t r0 = (int64_t)tt * kRouterTile * k;
  const int64_t r1 = min((int64_t)(tt + 1) * kRouterTile, T) * k;
  const int64_t per = ((r1 - r0 + kScatterWarps - 1) / kScatterWarps + 31) / 32 * 32;
  const int64_t w0 = r0 + warp * per, w1 = min(r1, w0 + per);
  const int32_t* idx_h = idx + (size_t)h * T * k;
  const float* gate_h = gate + (size_t)h * T * k;
  int* my = wcnt + warp * N_e;
  for (int64_t base = w0; base < w1; base += 32) {
    const int64_t r = base + lane;
    const bool act = r < w1;
    const int e = act ? idx_h[r] : -1 - lane;   // unique dummy per inactive lane
    const unsigned mask = __match_any_sync(0xffffffffu, e);
    if (act && __popc(mask & ((1u << lane) - 1u)) == 0) my[e] += __popc(mask);
    __syncwarp();   // orders this iteration's my[] updates before the next one's (racecheck-clean)
  }
  __syncthreads();
  for (int e = threadIdx.x; e < N_e; e += blockDim.x) {
    int run = 0;
    for (int w = 0; w < kScatterWarps; ++w) { const int c = wcnt[w * N_e + e]; wcnt[w * N_e + e] = run; run += c; }
    lbase[e] = run;                                   // the tile's count of expert e (scanned below)
  }
  __syncthreads();
  if (warp == 0) {                                    // exclusive scan of the counts over experts
    int carry = 0;
    for (int b = 0; b < N_e; b += 32) {
      const int e = b + lane;
      const int v = e < N_e ? lbase[e] : 0;
      int incl = v;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int n = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += n;
      }
      if (e < N_e) lbase[e] = carry + incl - v;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
  __syncthreads();
  const int32_t* offh = off + (size_t)h * (N_e + 1);
  const int32_t* pre = tilepref + ((size_t)h * n_rt + tt) * N_e;
  // pass 2: stable ranks -> pos (coalesced, replica order) and the tile's replicas sorted by expert in smem
  for (int64_t base = w0; base < w1; base += 32) {
    const int64_t r = base + lane;
    const bool act = r < w1;
    const int e = act ? idx_h[r] : -1 - lane;
    const unsigned mask = __match_any_sync(0xffffffffu, e);
    const int rank = __popc(mask & ((1u << lane) - 1u));
    if (act) {
      const int li = lbase[e] + my[e] + rank;
      s_r[li] = (int)(r - r0);
      s_e[li] = e;
      pos[(size_t)h * T * k + r] = offh[e] + pre[e] + my[e] + rank;
    }
    __syncwarp();
    if (act && rank == 0) my[e] += __popc(mask);
    __syncwarp();
  }
  __syncthreads();
  // pass 3: each expert's run of this tile is contiguous in the clustered rows -> coalesced stores
  const int n = (int)(r1 - r0);
  for (int li = threadIdx.x; li < n; li += blockDim.x) {
    const int e = s_e[li];
    const int64_t r = r0 + s_r[li];
    const size_t q = (size_t)h * Rp + offh[e] + pre[e] + (li - lbase[e]);
    perm[q] = (int32_t)r;
    tok_s[q] = (int32_t)(r / k);
    gate_s[q] = gate_h[r];
  }
}


// aux-free bias update (R24): one thread per (h, e); sign of load - mean as an exact integer test
__global__ void update_bias_kernel(const int32_t* __restrict__ load, int n, int N_e, int64_t total, float gamma,
                                   float* __restrict__ bias) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t d = (int64_t)load[i] * N_e - total;
  const float sgn = d > 0 ? 1.0f : (d < 0 ? -1.0f : 0.0f);
  bias[i] = bias[i] - gamma * sgn;
}

}  // namespace

void launch_dw_parts(const Routing& rt, Tile* chunks, int32_t* nchunks, int32_t* cbase, int32_t* ccount,
                     int32_t* pbase, int32_t* pcount, cudaStream_t s) {
  dw_parts_kernel<<<rt.H, 1024, 0, s>>>(rt.off, rt.H, rt.N_e, rt.dw_parts, chunks, rt.max_chunks, nchunks, cbase,
                                         ccount, pbase, pcount);
}


void launch_update_bias(const int32_t* load, int H, int N_e, int64_t total, float gamma, float* bias,
                        cudaStream_t s) {
  const int n = H * N_e;
  if (n > 0) update_bias_kernel<<<(n + 255) / 256, 256, 0, s>>>(load, n, N_e, total, gamma, bias);
}

// (4) windows of the windowed combine (kernels.h kWinParts): one block per head.  Tile range of
// window w: the first tile of its first part to the first tile of the next window (the next head's
// first tile, or the end of the list); token range: tokens below the first token of the next
// window's first part in every expert segment (rows within a segment are in token order).
__global__ void __launch_bounds__(256)
windows_kernel(const int32_t* __restrict__ counts, const int32_t* __restrict__ off, const int32_t* __restrict__ tbase,
               const int32_t* __restrict__ ntiles, const int32_t* __restrict__ tok_s, int H, int N_e, int64_t T,
               int64_t Rp, int seg_align, int32_t* __restrict__ win) {
  __shared__ int s_m[8];
  const int h = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int TPS = seg_align / kExpertBM;
  int tok_lo = 0;
  for (int w = 0; w < kWindows; ++w) {
    const int p1 = (w + 1) * kWinParts;
    int mn = (int)T;
    if (p1 < kTileParts) {
      for (int e = threadIdx.x; e < N_e; e += blockDim.x) {
        const int c = counts[(size_t)h * N_e + e];
        const int nu = (c + seg_align - 1) / seg_align;
        const int r = TPS * (p1 * nu / kTileParts) * kExpertBM;        // first row of part p1
        if (r < c) mn = min(mn, tok_s[(size_t)h * Rp + off[(size_t)h * (N_e + 1) + e] + r]);
      }
    }
    for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    if (lane == 0) s_m[warp] = mn;
    __syncthreads();
    if (threadIdx.x == 0) {
      int b = (int)T;
      for (int i = 0; i < (int)(blockDim.x / 32); ++i) b = min(b, s_m[i]);
      int32_t* o = win + ((size_t)h * kWindows + w) * 4;
      o[0] = tbase[((size_t)h * kTileParts + w * kWinParts) * N_e];
      o[1] = p1 < kTileParts ? tbase[((size_t)h * kTileParts + p1) * N_e]
                             : (h + 1 < H ? tbase[(size_t)(h + 1) * kTileParts * N_e] : *ntiles);
      o[2] = tok_lo;
      o[3] = b;
      tok_lo = b;
    }
    __syncthreads();
  }
}

void launch_windows(int H, int N_e, int64_t T, int64_t Rp, int seg_align, const int32_t* counts, const int32_t* off,
                    const int32_t* tilepref, int n_rt, const int32_t* ntiles, const int32_t* tok_s, int32_t* win,
                    cudaStream_t s) {
  const int32_t* tbase = tilepref + (size_t)H * n_rt * N_e;
  windows_kernel<<<H, 256, 0, s>>>(counts, off, tbase, ntiles, tok_s, H, N_e, T, Rp, seg_align, win);
}

void launch_cluster(int H, int64_t T, int k, int N_e, const int32_t* idx, const float* gate, const int32_t* hist,
                    int32_t* tilepref, int32_t* counts, int32_t* off, int32_t* perm, int32_t* pos, int32_t* tok_s,
                    float* gate_s, int64_t Rp, int seg_align, Tile* tiles, int32_t* ntiles, int max_tiles,
                    Tile* chunks, int32_t* nchunks, int32_t* cbase, int32_t* ccount, int max_chunks, int dw_parts,
                    int32_t* pbase, int32_t* pcount, cudaStream_t s) {
  const int n_rt = (int)((T + kRouterTile - 1) / kRouterTile);
  tile_prefix_kernel<<<dim3(N_e, H), 256, 0, s>>>(hist, tilepref, counts, n_rt, N_e);
  // tile bases [H][kTileParts][N_e] live in the (otherwise unused here) tail of tilepref's scratch
  int32_t* tbase = tilepref + (size_t)H * n_rt * N_e;
  offsets_kernel<<<H, kOffsetsThreads, 0, s>>>(counts, off, tbase, ntiles, H, N_e, max_tiles, seg_align);
  if (dw_parts > 0)
    dw_parts_kernel<<<H, 1024, 0, s>>>(off, H, N_e, dw_parts, chunks, max_chunks, nchunks, cbase, ccount, pbase, pcount);
  tiles_kernel<<<(H * N_e + 7) / 8, 256, 0, s>>>(counts, off, tbase, tiles, max_tiles, H, N_e, Rp, perm, tok_s,
                                                 gate_s, (int)T, seg_align);
  const size_t ssm = sizeof(int) * ((size_t)(kScatterWarps + 1) * N_e + 2 * (size_t)kRouterTile * k);
  if (ssm > 48 * 1024) cudaFuncSetAttribute(scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
  scatter_kernel<<<dim3(n_rt, H), kScatterWarps * 32, ssm, s>>>(idx, gate, off, tilepref, perm, pos, tok_s, gate_s,
                                                                T, k, N_e, n_rt, Rp);
}

}  // namespace mhl
