// tma_host.h — TMA tensor-map construction (host).
#pragma once
#include <cuda.h>
#include <stdint.h>

namespace mhl {

// Row-major [rows][cols] bf16 matrix with the given row pitch; box = box_rows x box_cols
// (box_cols * 2 bytes must be 128 for the 128-byte swizzle used by the kernels).
bool make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t row_stride_bytes,
                       uint32_t box_rows, uint32_t box_cols);

// Output-tile stores of the expert kernels: 1 = coalesced st.global from the smem staging slot
// (leaves the TMA unit to the row gathers), 0 = TMA bulk stores.  Measured per kernel (r1e,
// tools/ab_store.sh): the backward H kernel (two tiles per slot, 16 light epilogue warps) gains
// with st.global (1.39 -> 1.30 ms); the GELU-heavy forward and the dX GEMM lose (0.87 -> 1.00,
// 0.59 -> 0.65 ms).  `def` is the kernel's default; MHL_STORE_TMA=0/1 overrides all kernels.
int store_lsu(int def);
// value of a timing-only A/B environment switch (0 when unset); a nonzero value, which makes a
// kernel skip work and so produce invalid results, is reported on stderr
int timing_only_switch(const char* name);

// Event-trace profiling aid (see sm100.cuh trace_ev): a zeroed device buffer of kTraceSlots
// slots, and a dump of the non-zero slots "event tile clock" to a text file.
constexpr size_t kTraceSlots = 64 * 4096;
unsigned long long* trace_buffer(cudaStream_t s);
void trace_dump(const char* path, cudaStream_t s);

}  // namespace mhl
