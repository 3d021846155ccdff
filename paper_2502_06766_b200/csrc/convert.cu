// convert.cu — TKKV section rows (row-major f32, cache.py:1-13) → scan-friendly bf16 cache rows.
//
// The reference's on-disk cache stores one (N, d) f32 section per (layer, head, keys|values)
// (cache.py:143-148). On the device each row becomes 128 bf16 values (zero-padded when
// d < 128, which leaves every dot product unchanged) in the [B, Hkv, rows, 128] layout the
// scan streams. Memory-bound: one thread per output 16-byte chunk (8 bf16), RNE rounding.
#include <cuda_bf16.h>

#include "../../include/tkv.h"
#include "common.cuh"
#include "internal.h"

namespace tkv {

__global__ void __launch_bounds__(256) convert_rows_kernel(const float* __restrict__ src, int64_t rows,
                                                          int d, __nv_bfloat16* __restrict__ dst) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // 16-byte chunk
  const int64_t row = i >> 4;
  const int part = static_cast<int>(i & 15);
  if (row >= rows) return;
  const float* s = src + row * d;
  uint32_t w[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int c0 = part * 8 + 2 * j, c1 = c0 + 1;
    const float a = c0 < d ? __ldg(s + c0) : 0.f;
    const float b = c1 < d ? __ldg(s + c1) : 0.f;
    const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    w[j] = *reinterpret_cast<const uint32_t*>(&v);
  }
  *reinterpret_cast<uint4*>(dst + row * kD + part * 8) = make_uint4(w[0], w[1], w[2], w[3]);
}

}  // namespace tkv

extern "C" int tkv_convert_rows_f32(const float* src, int64_t rows, int32_t d, void* dst, void* stream) {
  if (!src || !dst || rows < 0 || d < 1 || d > tkv::kD) return TKV_EBADSHAPE;
  if (reinterpret_cast<uintptr_t>(dst) % 16) return TKV_EBADSHAPE;
  if (rows == 0) return TKV_OK;
  const int64_t chunks = rows * 16;
  const int64_t blocks = (chunks + 255) / 256;
  tkv::convert_rows_kernel<<<static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      src, rows, d, static_cast<__nv_bfloat16*>(dst));
  return cudaGetLastError() == cudaSuccess ? TKV_OK : TKV_ECUDA;
}
