// span.hpp — the device entry of the span operators (span.cu) that the
// engine uses for attend_chunk over a cached bf16 range.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace sinkr {
namespace span {

// Device scratch attend_device needs for (heads, dim, len) on `sms` SMs.
size_t attend_scratch_bytes(size_t heads, size_t dim, size_t len, int sms);

// attend_chunk (attention.cpp:101-142) of q [heads][dim] (device f32) over
// the device rows K, V [len][dim] (bf16), enqueued on `st`: the chunk's
// SplitPartial lands in d_m [heads], d_l [heads], d_acc [heads][dim] (fp64).
void attend_device(cudaStream_t st, const float* d_q, size_t heads, size_t dim,
                   const __nv_bfloat16* d_k, const __nv_bfloat16* d_v, size_t len,
                   uint8_t* scratch, double* d_m, double* d_l, double* d_acc, int sms);

}  // namespace span
}  // namespace sinkr
