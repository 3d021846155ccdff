// Microbenchmark: random 256-byte row gather through per-thread async copies into shared memory
// (cp.async.cg 16 B, LDGSTS) instead of register loads. Each half-warp runs its own ring of D
// stages × RPH rows (no block barriers), so the bytes in flight per SM are bounded by shared
// memory, not by registers. Compare with gather_bw.cu (register loads, ~5.3 TB/s ceiling).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_async gather_async.cu
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}

// grid-stride over groups of RPH rows per half-warp; D groups in flight per half-warp
template <int D, int RPH>
__global__ void __launch_bounds__(256) gather_async(const uint4* V, const int* rows, int n, float* out) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int lane = threadIdx.x & 31, half = lane >> 4, part = lane & 15, warp = threadIdx.x >> 5;
  const int hw = warp * 2 + half;
  const int ghw = blockIdx.x * 16 + hw, nhw = gridDim.x * 16;
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sm)) + hw * (D * RPH * 256) + part * 16;
  const int ngroups = (n + RPH - 1) / RPH;
  float acc = 0.f;
  int g_issue = ghw;
  auto issue = [&](int slot) {
    if (g_issue < ngroups) {
#pragma unroll
      for (int j = 0; j < RPH; ++j) {
        const int r = g_issue * RPH + j;
        if (r < n) cp_async16(base + (slot * RPH + j) * 256, V + static_cast<int64_t>(rows[r]) * 16 + part);
      }
    }
    cp_commit();
    g_issue += nhw;
  };
#pragma unroll
  for (int d = 0; d < D - 1; ++d) issue(d);
  int slot = 0;
  for (int g = ghw; g < ngroups; g += nhw) {
    issue((slot + D - 1) % D);
    cp_wait<D - 1>();
    __syncwarp();
#pragma unroll
    for (int j = 0; j < RPH; ++j) {
      const uint4 v = lds128(base + (slot * RPH + j) * 256);
      acc += __uint_as_float(v.x) + __uint_as_float(v.w);
    }
    __syncwarp();
    slot = (slot + 1) % D;
  }
  cp_wait<0>();
  if (acc == 12345.f) out[0] = acc;
}

template <int D, int RPH>
void run(const uint4* V, const int* rows, int n, float* out) {
  const int smem = 16 * D * RPH * 256;
  cudaFuncSetAttribute(gather_async<D, RPH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, gather_async<D, RPH>, 256, smem);
  if (per < 1) { printf("D=%d RPH=%d: does not fit\n", D, RPH); return; }
  const int grid = 148 * per;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  gather_async<D, RPH><<<grid, 256, smem>>>(V, rows, n, out);
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i) gather_async<D, RPH><<<grid, 256, smem>>>(V, rows, n, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const cudaError_t e = cudaGetLastError();
  printf("async D=%d RPH=%d ctas/sm=%d rows in flight/SM=%d: %.1f us -> %.0f GB/s %s\n", D, RPH, per,
         per * 16 * D * RPH, ms * 100, double(n) * 256 * 10 / (ms * 1e-3) / 1e9, e ? cudaGetErrorString(e) : "");
}

int main() {
  const int64_t nrows = (2LL << 30) / 256;
  uint4* V;
  cudaMalloc(&V, nrows * 256);
  cudaMemset(V, 0, nrows * 256);
  const int n = 32 * 16384;
  std::vector<int> h(n);
  std::mt19937 g(1);
  for (int i = 0; i < n; ++i) h[i] = int(g() % nrows);
  int* rows;
  cudaMalloc(&rows, n * 4);
  cudaMemcpy(rows, h.data(), n * 4, cudaMemcpyHostToDevice);
  float* out;
  cudaMalloc(&out, 4);
  run<2, 4>(V, rows, n, out);
  run<4, 2>(V, rows, n, out);
  run<4, 4>(V, rows, n, out);
  run<3, 4>(V, rows, n, out);
  run<8, 2>(V, rows, n, out);
  run<4, 8>(V, rows, n, out);
  run<6, 4>(V, rows, n, out);
  run<8, 4>(V, rows, n, out);
  return 0;
}
