// Probe: semantics of cp.async.bulk.tensor.2d ... .tile::gather4 on sm_100a (box rows 1 vs 4),
// destination swizzle.  nvcc -gencode arch=compute_100a,code=sm_100a gather4_probe.cu -o /tmp/g4 && /tmp/g4
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void probe(const __grid_constant__ CUtensorMap map, int r0, int r1, int r2, int r3, uint16_t* out) {
  __shared__ __align__(1024) uint16_t buf[8 * 64];
  __shared__ __align__(8) uint64_t bar;
  uint32_t sb = (uint32_t)__cvta_generic_to_shared(buf);
  uint32_t bb = (uint32_t)__cvta_generic_to_shared(&bar);
  for (int i = threadIdx.x; i < 8 * 64; i += blockDim.x) buf[i] = 0xFFFF;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bb));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(4 * 128));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(sb),
        "l"(&map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bb)
        : "memory");
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(bb));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 8 * 64; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int rows = 64, cols = 64;
  std::vector<uint16_t> h(rows * cols);
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) h[r * cols + c] = (uint16_t)(r * 256 + c);   // encodes (row, col)
  uint16_t *d, *o;
  cudaMalloc(&d, h.size() * 2);
  cudaMalloc(&o, 8 * 64 * 2);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  for (int boxr : {1, 4}) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t str[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)boxr};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("box rows %d: encode=%d\n", boxr, (int)r);
    if (r != CUDA_SUCCESS) continue;
    cudaMemset(o, 0, 8 * 64 * 2);
    probe<<<1, 128>>>(m, 5, 17, 2, 40, o);
    cudaError_t e = cudaDeviceSynchronize();
    printf("  launch: %s\n", cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    std::vector<uint16_t> out(8 * 64);
    cudaMemcpy(out.data(), o, out.size() * 2, cudaMemcpyDeviceToHost);
    for (int r = 0; r < 5; ++r) {
      printf("  smem row %d:", r);
      for (int c = 0; c < 64; c += 8) printf(" (%d,%d)", out[r * 64 + c] >> 8, out[r * 64 + c] & 255);
      printf("\n");
    }
  }
  return 0;
}
