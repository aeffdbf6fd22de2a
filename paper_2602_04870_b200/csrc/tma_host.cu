// tma_host.cu — host-side TMA tensor-map encoding (driver entry point fetched through the runtime,
// so the library needs no link-time libcuda dependency).
#include "tma_host.h"

#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

namespace mhl {

bool make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t row_stride_bytes,
                       uint32_t box_rows, uint32_t box_cols) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !encode)
      return false;
  }
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {row_stride_bytes};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static unsigned long long* g_trace_dev = nullptr;

unsigned long long* trace_buffer(cudaStream_t s) {
  if (!g_trace_dev) cudaMalloc(&g_trace_dev, kTraceSlots * sizeof(unsigned long long));
  cudaMemsetAsync(g_trace_dev, 0, kTraceSlots * sizeof(unsigned long long), s);
  return g_trace_dev;
}

void trace_dump(const char* path, cudaStream_t s) {
  cudaStreamSynchronize(s);
  unsigned long long* h = (unsigned long long*)malloc(kTraceSlots * sizeof(unsigned long long));
  cudaMemcpy(h, g_trace_dev, kTraceSlots * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  FILE* f = fopen(path, "w");
  if (f) {
    for (size_t u = 0; u < kTraceSlots; ++u)
      if (h[u]) fprintf(f, "%zu %zu %llu\n", u / 4096, u % 4096, h[u]);
    fclose(f);
  }
  free(h);
}

int timing_only_switch(const char* name) {
  const char* e = getenv(name);
  const int v = e ? atoi(e) : 0;
  if (v != 0) fprintf(stderr, "[mhlmoe] timing-only A/B switch %s=%d is set: kernel results are NOT valid\n", name, v);
  return v;
}

int store_lsu(int def) {
  static const char* e = getenv("MHL_STORE_TMA");
  return e ? (atoi(e) ? 0 : 1) : def;
}

}  // namespace mhl
