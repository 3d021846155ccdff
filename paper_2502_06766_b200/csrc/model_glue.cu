// model_glue.cu — the non-attention pieces of one batch-1 decode step (paper_2502_06766_b200/model.py,
// BASELINE cfg4), fused into four small kernels so a layer is four GEMVs (cuBLAS), one top-k
// attention call (libtkv) and these, instead of ~60 eager PyTorch elementwise launches:
//
//   tkv_model_add_rmsnorm      x += delta (bf16 residual add), h = RMSNorm(x)·w (bf16)
//   tkv_model_qkv_rope_append  RoPE of this token's q and k at position pos, q → bf16 buffer,
//                              k / v → the caches' row n_ctx + n_win (GenWindow.append,
//                              attention.py:94-100, 210; the window counter is not advanced)
//   tkv_model_silu_mul         SwiGLU activation silu(gate)·up → bf16
//   tkv_model_logits_argmax    bf16 logits → fp32 copy + greedy token (first maximal index)
//
// Numerics follow the eager code they replace (model.py history): bf16 storage, fp32 math,
// the same roundings to bf16.
#include <math.h>
#include <stdio.h>

#include "common.cuh"
#include "internal.h"
#include "tkv.h"

namespace tkv {
namespace {

constexpr int kNormThreads = 1024;

__device__ __forceinline__ float bf2f(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ __nv_bfloat16 f2bf(float v) { return __float2bfloat16_rn(v); }

__global__ void __launch_bounds__(kNormThreads) add_rmsnorm_kernel(__nv_bfloat16* x, const __nv_bfloat16* delta,
                                                                    const float* w, float eps, __nv_bfloat16* h,
                                                                    int d) {
  __shared__ float s_red[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float ss = 0.f;
  for (int i = tid; i < d; i += kNormThreads) {
    float v = bf2f(x[i]);
    if (delta) {
      v = bf2f(f2bf(v + bf2f(delta[i])));  // bf16 + bf16 → bf16 (the residual stream is bf16)
      x[i] = f2bf(v);
    }
    ss = fmaf(v, v, ss);
  }
  ss = warp_sum(ss);
  if (lane == 0) s_red[warp] = ss;
  __syncthreads();
  if (warp == 0) {
    float t = lane < kNormThreads / 32 ? s_red[lane] : 0.f;
    t = warp_sum(t);
    if (lane == 0) s_red[0] = t;
  }
  __syncthreads();
  const float r = rsqrtf(s_red[0] / static_cast<float>(d) + eps);
  for (int i = tid; i < d; i += kNormThreads) {
    h[i] = f2bf(bf2f(x[i]) * r * w[i]);
  }
}

// grid: Hq + Hkv blocks of 64 threads rotate one head each (thread j: pair (2j, 2j+1)),
// Hkv more copy the v heads
__global__ void __launch_bounds__(64) qkv_rope_append_kernel(const __nv_bfloat16* qkv, const float* cos_t,
                                                             const float* sin_t, const int64_t* pos,
                                                             __nv_bfloat16* q_out, __nv_bfloat16* kc,
                                                             __nv_bfloat16* vc, const int32_t* n_ctx,
                                                             const int32_t* n_win, int64_t cache_rows, int hq,
                                                             int hkv) {
  const int hb = blockIdx.x, j = threadIdx.x;
  const int64_t row = static_cast<int64_t>(n_ctx[0]) + n_win[0];
  if (hb < hq + hkv) {
    const __nv_bfloat16* src = qkv + static_cast<int64_t>(hb) * kD;
    const int64_t p = pos[0];
    const float c = cos_t[p * (kD / 2) + j], s = sin_t[p * (kD / 2) + j];
    const float x1 = bf2f(src[2 * j]), x2 = bf2f(src[2 * j + 1]);
    const __nv_bfloat16 o1 = f2bf(x1 * c - x2 * s), o2 = f2bf(x1 * s + x2 * c);
    __nv_bfloat16* dst;
    if (hb < hq) {
      dst = q_out + static_cast<int64_t>(hb) * kD;
    } else {
      if (row < 0 || row >= cache_rows) return;
      dst = kc + (static_cast<int64_t>(hb - hq) * cache_rows + row) * kD;
    }
    dst[2 * j] = o1;
    dst[2 * j + 1] = o2;
  } else {
    const int vh = hb - hq - hkv;
    if (row < 0 || row >= cache_rows) return;
    const __nv_bfloat16* src = qkv + static_cast<int64_t>(hq + hkv + vh) * kD;
    __nv_bfloat16* dst = vc + (static_cast<int64_t>(vh) * cache_rows + row) * kD;
    dst[2 * j] = src[2 * j];
    dst[2 * j + 1] = src[2 * j + 1];
  }
}

__global__ void __launch_bounds__(256) silu_mul_kernel(const __nv_bfloat16* gu, __nv_bfloat16* out, int f) {
  for (int i = blockIdx.x * 256 + threadIdx.x; i < f; i += gridDim.x * 256) {
    const float g = bf2f(gu[i]), u = bf2f(gu[f + i]);
    out[i] = f2bf(g / (1.f + expf(-g)) * u);
  }
}

// packed (order-preserving key of the value, ~index): the max is the largest value, ties to the
// lowest index
__device__ __forceinline__ uint64_t am_pack(float v, uint32_t i) {
  return (static_cast<uint64_t>(score_key(v)) << 32) | static_cast<uint32_t>(~i);
}

__global__ void __launch_bounds__(256) logits_argmax_kernel(const __nv_bfloat16* logits, int n, float* out_f32,
                                                            int64_t* token, unsigned long long* scratch) {
  __shared__ uint64_t s_red[8];
  __shared__ bool s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint64_t best = 0ull;
  for (int i = blockIdx.x * 256 + tid; i < n; i += gridDim.x * 256) {
    const float v = bf2f(logits[i]);
    if (out_f32) out_f32[i] = v;
    const uint64_t k = am_pack(v, static_cast<uint32_t>(i));
    best = k > best ? k : best;
  }
  best = warp_max_u64(best);
  if (lane == 0) s_red[warp] = best;
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < 8; ++w) best = s_red[w] > best ? s_red[w] : best;
    atomicMax(&scratch[0], static_cast<unsigned long long>(best));
    __threadfence();
    s_last = atomicAdd(&scratch[1], 1ull) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && tid == 0) {
    __threadfence();
    const unsigned long long m = atomicExch(&scratch[0], 0ull);  // read + reset for the next step
    token[0] = static_cast<int64_t>(~static_cast<uint32_t>(m));
    scratch[1] = 0ull;
  }
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int launched(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return TKV_OK;
  char buf[256];
  snprintf(buf, sizeof(buf), "%s launch: %s", what, cudaGetErrorString(e));
  return api_fail(TKV_ECUDA, buf);
}

}  // namespace
}  // namespace tkv

using namespace tkv;

extern "C" {

int tkv_model_add_rmsnorm(void* x, const void* delta, const float* w, float eps, void* h, int32_t d, void* stream) {
  if (!x || !w || !h || d <= 0) return api_fail(TKV_EBADSHAPE, "tkv_model_add_rmsnorm: null tensor or d <= 0");
  add_rmsnorm_kernel<<<1, kNormThreads, 0, as_stream(stream)>>>(
      static_cast<__nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(delta), w, eps,
      static_cast<__nv_bfloat16*>(h), d);
  return launched("tkv_model kernel");
}

int tkv_model_qkv_rope_append(const void* qkv, const float* cos_t, const float* sin_t, const int64_t* pos,
                              void* q_out, void* k_cache, void* v_cache, const int32_t* n_ctx,
                              const int32_t* n_win, int64_t cache_rows, int32_t n_heads, int32_t n_kv_heads,
                              int32_t head_dim, void* stream) {
  if (!qkv || !cos_t || !sin_t || !pos || !q_out || !k_cache || !v_cache || !n_ctx || !n_win)
    return api_fail(TKV_EBADSHAPE, "tkv_model_qkv_rope_append: null tensor");
  if (head_dim != kD || n_heads <= 0 || n_kv_heads <= 0 || cache_rows <= 0)
    return api_fail(TKV_EBADSHAPE, "tkv_model_qkv_rope_append: head_dim must be 128, head counts and rows > 0");
  qkv_rope_append_kernel<<<n_heads + 2 * n_kv_heads, 64, 0, as_stream(stream)>>>(
      static_cast<const __nv_bfloat16*>(qkv), cos_t, sin_t, pos, static_cast<__nv_bfloat16*>(q_out),
      static_cast<__nv_bfloat16*>(k_cache), static_cast<__nv_bfloat16*>(v_cache), n_ctx, n_win, cache_rows,
      n_heads, n_kv_heads);
  return launched("tkv_model kernel");
}

int tkv_model_silu_mul(const void* gate_up, void* out, int32_t ffn, void* stream) {
  if (!gate_up || !out || ffn <= 0) return api_fail(TKV_EBADSHAPE, "tkv_model_silu_mul: null tensor or ffn <= 0");
  int grid = (ffn + 255) / 256;
  grid = grid > 148 * 4 ? 148 * 4 : grid;
  silu_mul_kernel<<<grid, 256, 0, as_stream(stream)>>>(static_cast<const __nv_bfloat16*>(gate_up),
                                                       static_cast<__nv_bfloat16*>(out), ffn);
  return launched("tkv_model kernel");
}

int tkv_model_logits_argmax(const void* logits, int32_t n, float* logits_f32, int64_t* token, uint64_t* scratch,
                            void* stream) {
  if (!logits || !token || !scratch || n <= 0)
    return api_fail(TKV_EBADSHAPE, "tkv_model_logits_argmax: null tensor or n <= 0");
  int grid = (n + 255) / 256;
  grid = grid > 148 * 2 ? 148 * 2 : grid;
  logits_argmax_kernel<<<grid, 256, 0, as_stream(stream)>>>(static_cast<const __nv_bfloat16*>(logits), n,
                                                            logits_f32, token,
                                                            reinterpret_cast<unsigned long long*>(scratch));
  return launched("tkv_model kernel");
}

}  // extern "C"
