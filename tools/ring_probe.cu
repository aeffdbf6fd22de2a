// Gather-ring probe (tools only): throughput of the expert kernels' sub-token gather pipeline in
// isolation.  Producer warps fill 16 KB K-chunks (128 rows x 64 bf16 columns, SW128 K-major) of
// gathered rows into an S-stage smem ring; one consumer thread waits FULL and releases EMPTY.
//   mech 0: cp.async 16 B per lane + cp.async.mbarrier.arrive.noinc
//   mech 1: TMA tile::gather4 issued by lane 0 of each producer warp
//   mech 2: plain 16 B loads to registers, st.shared, mbarrier arrive (2-chunk software pipeline)
//   mech 7: mech 6's gathers, and the consumer writes every chunk back out with a 16 KB bulk store
//           (equal bytes in and out per tile, F5's traffic shape); TB/s counts in + out
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void cp_async_16(uint32_t dst, const void* src) { asm volatile("cp.async.cg.shared.global [%0], [%1], 16, 16;" ::"r"(dst), "l"(src) : "memory"); }
__device__ __forceinline__ void cp_async_arrive(uint64_t* b) { asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(b)) : "memory"); }
__device__ __forceinline__ void gather4(uint32_t dst, const void* map, int c0, int r0, int r1, int r2, int r3, uint64_t* b) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
               ::"r"(dst), "l"(map), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ uint32_t kmaj(int r, int c) { return r * 128 + ((((c >> 3) ^ (r & 7)) & 7) << 4); }

constexpr int kChunk = 16384;
__global__ void __launch_bounds__(1024, 1)
ring(const __grid_constant__ CUtensorMap map, const uint16_t* __restrict__ x, int ld, const int* __restrict__ rows,
     int ntiles, int S, int PW, int mech, int* sink, char* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * kChunk);
  uint64_t* empty = full + 16;
  int* stok = reinterpret_cast<int*>(empty + 16);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], mech == 5 ? 32 : (mech == 4 || mech == 6 || mech == 7) ? 1 : (mech == 1 || mech == 3) ? PW : 32 * PW); mbar_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const uint32_t sb = smem_u32(smem);
  const int RPW = 128 / PW;   // rows per producer warp
  if (mech == 5 && warp < PW) {
    // half the warps: TMA gather4 (whole chunk, 32 lanes); the other half: cp.async 16 B per lane
    int cnt = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int h = t % 8;
      const int r4[4] = {rows[(t / 8) * 128 + 4 * lane], rows[(t / 8) * 128 + 4 * lane + 1],
                         rows[(t / 8) * 128 + 4 * lane + 2], rows[(t / 8) * 128 + 4 * lane + 3]};
      for (int kb = 0; kb < 4; ++kb, ++cnt) {
        if (cnt % PW != warp) continue;
        const int st = cnt % S;
        if (lane == 0) mbar_wait(&empty[st], ((cnt / S) & 1) ^ 1);
        __syncwarp();
        if (warp & 1) {
          // cp.async: lane covers rows 4*lane..4*lane+3, 8 x 16 B each
          for (int rr = 0; rr < 4; ++rr)
            for (int c = 0; c < 8; ++c)
              cp_async_16(sb + st * kChunk + kmaj(4 * lane + rr, c * 8), x + (size_t)r4[rr] * ld + h * 256 + kb * 64 + c * 8);
          cp_async_arrive(&full[st]);
        } else {
          if (lane == 0) mbar_expect_tx(&full[st], kChunk);
          __syncwarp();
          gather4(sb + st * kChunk + 4 * lane * 128, &map, h * 256 + kb * 64, r4[0], r4[1], r4[2], r4[3], &full[st]);
          if (lane != 0) mbar_arrive(&full[st]);   // 1 expect_tx + 31 arrivals = the 32 of a cp.async warp
        }
      }
    }
  } else if ((mech == 6 || mech == 7) && warp < PW) {
    // chunk c -> stage c % S, filled by the warp pair (c % (PW/2)): each warp of the pair gathers
    // 64 of its 128 rows with 16 lanes (one gather4 per lane); stage ownership is fixed when S is a
    // multiple of PW/2, so the EMPTY parity never aliases
    int cnt = 0;
    const int pair = warp >> 1, hrow = (warp & 1) * 64;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int h = t % 8;
      const int l16 = lane & 15;
      const int base = (t / 8) * 128 + hrow + 4 * l16;
      const int r0 = rows[base], r1 = rows[base + 1], r2 = rows[base + 2], r3 = rows[base + 3];
      for (int kb = 0; kb < 4; ++kb, ++cnt) {
        if (cnt % (PW / 2) != pair) continue;
        const int st = cnt % S;
        if (lane == 0) mbar_wait(&empty[st], ((cnt / S) & 1) ^ 1);
        __syncwarp();
        if ((warp & 1) == 0 && lane == 0) mbar_expect_tx(&full[st], kChunk);
        if (lane < 16)
          gather4(sb + st * kChunk + (hrow + 4 * l16) * 128, &map, h * 256 + kb * 64, r0, r1, r2, r3, &full[st]);
      }
    }
  } else if (mech == 4 && warp < PW) {
    // warp w owns every PW-th chunk; its 32 lanes each issue one gather4 (4 rows) of it
    uint32_t eph[16] = {0};
    int cnt = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int h = t % 8;
      const int myrow = rows[(t / 8) * 128 + 4 * lane], r1 = rows[(t / 8) * 128 + 4 * lane + 1],
                r2 = rows[(t / 8) * 128 + 4 * lane + 2], r3 = rows[(t / 8) * 128 + 4 * lane + 3];
      for (int kb = 0; kb < 4; ++kb, ++cnt) {
        if (cnt % PW != warp) continue;
        const int st = cnt % S;
        if (lane == 0) { mbar_wait(&empty[st], ((cnt / S) & 1) ^ 1); mbar_expect_tx(&full[st], kChunk); }
        __syncwarp();
        gather4(sb + st * kChunk + 4 * lane * 128, &map, h * 256 + kb * 64, myrow, r1, r2, r3, &full[st]);
      }
    }
  } else if (warp < PW) {
    int st = 0; uint32_t eph[16] = {0};
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int h = t % 8;
      for (int i = lane; i < RPW; i += 32) stok[warp * RPW + i] = rows[(t / 8) * 128 + warp * RPW + i];
      __syncwarp();
      for (int kb = 0; kb < 4; ++kb) {
        if (lane == 0) mbar_wait(&empty[st], eph[st] ^ 1);
        eph[st] ^= 1;
        __syncwarp();
        const uint32_t dst = sb + st * kChunk;
        const int col = h * 256 + kb * 64;
        if (mech == 0) {
          for (int j = lane; j < RPW * 8; j += 32) {
            const int r = warp * RPW + (j >> 3), c = (j & 7) * 8;
            cp_async_16(dst + kmaj(r, c), x + (size_t)stok[r] * ld + col + c);
          }
          cp_async_arrive(&full[st]);
        } else if (mech == 3) {
          // every lane g < RPW/4 issues one gather4 (rows warp*RPW + 4g .. +4)
          if (lane == 0) mbar_expect_tx(&full[st], RPW * 128);
          __syncwarp();
          if (lane < RPW / 4) {
            const int r = warp * RPW + 4 * lane;
            gather4(dst + r * 128, &map, col, stok[r], stok[r + 1], stok[r + 2], stok[r + 3], &full[st]);
          }
        } else if (mech == 1) {
          if (lane == 0) {
            mbar_expect_tx(&full[st], RPW * 128);
            for (int g = 0; g < RPW; g += 4) {
              const int r = warp * RPW + g;
              gather4(dst + r * 128, &map, col, stok[r], stok[r + 1], stok[r + 2], stok[r + 3], &full[st]);
            }
          }
        } else {
          uint4 v[8];
          int n = 0;
          for (int j = lane; j < RPW * 8; j += 32, ++n) {
            const int r = warp * RPW + (j >> 3), c = (j & 7) * 8;
            v[n & 7] = *reinterpret_cast<const uint4*>(x + (size_t)stok[r] * ld + col + c);
          }
          n = 0;
          for (int j = lane; j < RPW * 8; j += 32, ++n) {
            const int r = warp * RPW + (j >> 3), c = (j & 7) * 8;
            *reinterpret_cast<uint4*>(smem + st * kChunk + kmaj(r, c)) = v[n & 7];
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive(&full[st]);
        }
        if (++st == S) st = 0;
      }
      __syncwarp();
    }
  } else if (warp == PW && lane == 0) {
    int st = 0; uint32_t fph[16] = {0}; int acc = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x)
      for (int kb = 0; kb < 4; ++kb) {
        mbar_wait(&full[st], fph[st]); fph[st] ^= 1;
        acc += smem[st * kChunk + 5];
        if (mech == 7) {   // write the chunk out (contiguous, like Yrep), release the stage once read
          char* dst = out + ((size_t)t * 4 + kb) * kChunk;
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                       "r"(sb + st * kChunk), "r"(kChunk) : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        mbar_arrive(&empty[st]);
        if (++st == S) st = 0;
      }
    if (mech == 7) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (acc == 123456789) *sink = acc;
  }
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  // argv[1]: mechanisms (e.g. "4,5"); argv[2]: source rows (sub-token rows gathered from: 65536 = 256 MB,
  // mostly DRAM; 8192 = 32 MB, L2-resident)
  std::vector<int> mechs;
  { const char* m = argc > 1 ? argv[1] : "4"; for (const char* c = m; *c; ++c) if (*c >= '0' && *c <= '9') mechs.push_back(*c - '0'); }
  const int Tsrc = argc > 2 ? atoi(argv[2]) : 65536;
  const int T = 65536, k = 8, E = 64;
  const int64_t n = (int64_t)T * k;
  std::mt19937 rng(0);
  std::vector<std::pair<int,int>> key; key.reserve(n);
  std::vector<int> perm(E); for (int e = 0; e < E; ++e) perm[e] = e;
  for (int t = 0; t < T; ++t) { std::shuffle(perm.begin(), perm.end(), rng); for (int j = 0; j < k; ++j) key.push_back({perm[j], t}); }
  std::sort(key.begin(), key.end());
  std::vector<int> clus(n);
  for (int64_t i = 0; i < n; ++i) clus[i] = key[i].second % Tsrc;
  uint16_t* x; int *rows, *sink;
  cudaMalloc(&x, (size_t)T * 4096); cudaMalloc(&rows, n * 4); cudaMalloc(&sink, 4);
  cudaMemset(x, 1, (size_t)T * 4096);
  cudaMemcpy(rows, clus.data(), n * 4, cudaMemcpyHostToDevice);
  PFN_cuTensorMapEncodeTiled_v12000 enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[2] = {2048, (cuuint64_t)Tsrc}; cuuint64_t str[1] = {4096}; cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int ntiles = (int)(n / 128) * 8;   // every head of every clustered tile: 2.1 GB gathered
  char* flush; cudaMalloc(&flush, 512 << 20);
  char* out; cudaMalloc(&out, (size_t)ntiles * 4 * 16384);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mech : mechs)
    for (int PW : {4, 8})
      for (int S : {4, 6, 8, 12}) {
        if ((mech == 6 || mech == 7) ? S < PW / 2 : S % PW) continue;   // mech 6/7: any S >= owners
        const int smem = S * kChunk + 2048;
        cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        float tot = 0;
        for (int it = 0; it < 3; ++it) {
          cudaMemset(flush, it, 512 << 20);
          cudaEventRecord(a);
          ring<<<148, 32 * (PW + 1), smem>>>(map, x, 2048, rows, ntiles, S, PW, mech, sink, out);
          cudaEventRecord(b); cudaEventSynchronize(b);
          float ms; cudaEventElapsedTime(&ms, a, b); if (it) tot += ms;
        }
        cudaError_t e = cudaGetLastError();
        const double bytes = ntiles * 65536.0 * (mech == 7 ? 2 : 1);   // gathered (+ stored)
        printf("mech %d PW %2d S %2d: %.3f ms  %.2f TB/s  %s\n", mech, PW, S, tot / 2, bytes / (tot / 2) / 1e9,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
  return 0;
}
