// Shared host helpers of the C ABI implementation.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <string>

#include "../../include/distattn_b200.h"

namespace da {
da_status set_error(da_status s, const std::string& msg);
da_status cuda_error(cudaError_t e, const char* where);
const char* last_error();
da_status make_tmap_3d(CUtensorMap* map, const void* base, int64_t heads, int64_t rows,
                       uint32_t box_rows = 128);
// fp32 [heads][rows][128] accumulator, box {32, 32, 1} (dQ reduction): no
// swizzle (single-CTA kernel) or 128B-swizzled (CTA-pair kernel)
da_status make_tmap_f32_acc(CUtensorMap* map, void* base, int64_t heads, int64_t rows,
                            bool swizzle128 = false);
cudaError_t launch_fill(float* dst, float value, int64_t n, cudaStream_t stream);
}  // namespace da
