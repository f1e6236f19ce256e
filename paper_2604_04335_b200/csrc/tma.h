// Host-side TMA tensor-map construction (cuTensorMapEncodeTiled via the runtime's driver
// entry point, so libgs.so does not link libcuda directly).
#pragma once
#include <cuda.h>
#include <stdint.h>

namespace gs {
// 2-D bf16 map: dims {inner, outer}, row stride in bytes, box {box_inner, box_outer},
// 128-byte swizzle, OOB elements read as zero.
bool make_tma_2d_bf16(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                      uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer);
// 2-D fp32 map, same conventions (128-byte swizzle: box_inner * 4 must be <= 128).
bool make_tma_2d_f32(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                     uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer);
// 3-D bf16 map: dims {d0, d1, d2}, strides (bytes) of dims 1 and 2, box {b0, b1, b2}.
bool make_tma_3d_bf16(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                      uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t b0, uint32_t b1,
                      uint32_t b2);
}  // namespace gs
