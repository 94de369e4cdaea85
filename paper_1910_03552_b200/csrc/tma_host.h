// Host-side TMA tensor-map helpers (driver entry point resolved at runtime, no -lcuda).
#pragma once
#include <cuda.h>
#include <stdint.h>

namespace bp {
int tma_init();        // resolve cuTensorMapEncodeTiled + SM count; BP_OK or BP_ERR_LAUNCH
int tma_num_sms();
// 2D row-major tensor [rows][cols] of `esize`-byte elements; box {box_cols (inner), box_rows};
// swz in {0, 32, 64, 128} bytes.  OOB reads are zero-filled.
int tma_make_2d(CUtensorMap* m, const void* ptr, CUtensorMapDataType dtype, int esize, long long rows,
                long long cols, int box_cols, int box_rows, int swz);
// rank-D f32 tensor, no swizzle: dims[0] innermost (contiguous); strides_b[i] = byte stride of
// dims[i + 1] (multiples of 16); box[] elements per dim (box[0] * 4 bytes a multiple of 16).
// OOB elements of a store are not written.
int tma_make_f32(CUtensorMap* m, const void* ptr, int rank, const long long* dims, const long long* strides_b,
                 const int* box);
}  // namespace bp
