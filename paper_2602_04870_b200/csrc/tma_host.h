// tma_host.h — TMA tensor-map construction (host).
#pragma once
#include <cuda.h>
#include <stdint.h>

namespace mhl {

// Row-major [rows][cols] bf16 matrix with the given row pitch; box = box_rows x box_cols
// (box_cols * 2 bytes must be 128 for the 128-byte swizzle used by the kernels).
bool make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t row_stride_bytes,
                       uint32_t box_rows, uint32_t box_cols);

}  // namespace mhl
