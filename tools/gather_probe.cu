// Gather-granularity probe (tools only): gathers over a working set larger than L2.
// x = [T][2048] bf16 (268 MB); every (row, head) pair of the clustered row stream is read once
// per pass (8 heads -> 268 MB of distinct bytes per pass, 2.1 GB gathered with k = 8 reuse).
//   mode 0: a warp reads one 512 B head-row at once (32 lanes x 16 B)
//   mode 1: chunk-major like the smem ring: for a 128-row tile, all rows' 128 B chunk 0, then
//           chunk 1, ... (a warp instruction covers 4 rows x 128 B)
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>
__global__ void gather(const uint4* __restrict__ x, const int* __restrict__ rows, int64_t n, int mode,
                       uint4* __restrict__ sink) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint4 acc = make_uint4(0, 0, 0, 0);
  // block = one (head, 128-row tile) at a time; 8 warps
  const int64_t ntiles = n / 128 * 8;
  for (int64_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    const int h = (int)(tl % 8);
    const int64_t r0 = (tl / 8) * 128;
    if (mode == 0) {
      // warp w: rows r0 + w*16 .. +16, each a 512 B read
      uint4 v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = x[(int64_t)rows[r0 + wib * 16 + u] * 256 + h * 32 + lane];
#pragma unroll
      for (int u = 0; u < 16; ++u) { acc.x ^= v[u].x; acc.y ^= v[u].y; }
    } else {
      // 4 chunks of 128 B; per chunk a warp instruction covers 4 rows; warp w: rows w*16..+16
      uint4 v[16];
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int r = wib * 16 + j * 4 + (lane >> 3);
          v[c * 4 + j] = x[(int64_t)rows[r0 + r] * 256 + h * 32 + c * 8 + (lane & 7)];
        }
#pragma unroll
      for (int u = 0; u < 16; ++u) { acc.x ^= v[u].x; acc.y ^= v[u].y; }
    }
  }
  if (acc.x == 0x12345678u) sink[0] = acc;
}
int main() {
  const int T = 65536, k = 8, E = 64;
  const int64_t n = (int64_t)T * k;
  std::mt19937 rng(0);
  std::vector<std::pair<int,int>> key; key.reserve(n);
  std::vector<int> perm(E); for (int e = 0; e < E; ++e) perm[e] = e;
  for (int t = 0; t < T; ++t) { std::shuffle(perm.begin(), perm.end(), rng); for (int j = 0; j < k; ++j) key.push_back({perm[j], t}); }
  std::sort(key.begin(), key.end());
  std::vector<int> clus(n), rnd(n);
  for (int64_t i = 0; i < n; ++i) { clus[i] = key[i].second; rnd[i] = rng() % T; }
  uint4 *x, *sink; int* rows;
  cudaMalloc(&x, (size_t)T * 4096); cudaMalloc(&sink, 64); cudaMalloc(&rows, n * 4);
  cudaMemset(x, 1, (size_t)T * 4096);
  char* flush; cudaMalloc(&flush, 512 << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, std::vector<int>& r, int mode, int blocks) {
    cudaMemcpy(rows, r.data(), n * 4, cudaMemcpyHostToDevice);
    float tot = 0;
    for (int i = 0; i < 6; ++i) {
      cudaMemset(flush, i, 512 << 20);
      cudaEventRecord(a);
      gather<<<blocks, 256>>>(x, rows, n, mode, sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (i >= 1) tot += ms;
    }
    const float ms = tot / 5;
    printf("%-28s mode %d grid %4d: %.3f ms  %.2f TB/s gathered\n", name, mode, blocks, ms, n * 8 * 512.0 / ms / 1e9);
  };
  for (int blocks : {148, 296, 592}) {
    run("clustered", clus, 0, blocks); run("clustered", clus, 1, blocks);
    run("random", rnd, 0, blocks); run("random", rnd, 1, blocks);
  }
  return 0;
}
