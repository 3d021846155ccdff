// Microbenchmark: random 256-byte row gather with the TMA row gather
// (cp.async.bulk.tensor.2d.tile::gather4, four indexed rows per instruction) into a shared-memory
// ring, consumed by the CTA's warps (fp32 weighted sum). Compare with gather_bw.cu (register
// loads). One CTA per SM (CTAS=2: two), ring of NSLOT slots × SLOT rows, one mbarrier per slot.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_tma4 gather_tma4.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap* map, int r0, int r1, int r2, int r3,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
      : "memory");
}

template <int NSLOT, int SLOT, int IW = 1>
__global__ void __launch_bounds__(256, 1) g4(const __grid_constant__ CUtensorMap map, const int* rows, int n,
                                             float* out) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ uint64_t bar[NSLOT];
  __shared__ int s_rows[4096];  // this CTA's row ids (indices read from shared memory at issue)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, half = lane >> 4, part = lane & 15;
  const int hw = warp * 2 + half;
  if (tid == 0) {
    for (int s = 0; s < NSLOT; ++s) mbar_init(smem_u32(&bar[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // this CTA's rows: contiguous range of the (random) row list
  const int per = (n + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * per, r1 = min(n, r0 + per);
  const int nslots_total = (r1 - r0 + SLOT - 1) / SLOT;
  for (int i = tid; i < r1 - r0 && i < 4096; i += 256) s_rows[i] = rows[r0 + i];
  __syncthreads();
  float acc = 0.f;
  auto issue = [&](int j) {  // slot j of this CTA's sequence → ring slot j % NSLOT; IW warps issue
    if (warp >= IW || j >= nslots_total) return;
    const int s = j % NSLOT;
    const uint32_t b = smem_u32(&bar[s]);
    if (warp == 0 && lane == 0) mbar_expect_tx(b, SLOT * 256);
    const uint32_t dst = smem_u32(ring) + s * SLOT * 256;
    for (int g = warp + IW * lane; g < SLOT / 4; g += 32 * IW) {
      const int base = r0 + j * SLOT + 4 * g;
      int rr[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) rr[i] = s_rows[min(base + i, r1 - 1) - r0];
      tma_gather4(dst + g * 1024, &map, rr[0], rr[1], rr[2], rr[3], b);
    }
  };
  for (int j = 0; j < NSLOT - 1; ++j) issue(j);
  for (int j = 0; j < nslots_total; ++j) {
    issue(j + NSLOT - 1);
    const int s = j % NSLOT;
    mbar_wait(smem_u32(&bar[s]), (j / NSLOT) & 1);
    const uint8_t* src = ring + s * SLOT * 256;
    for (int i = hw; i < SLOT; i += 16) {
      const uint4 v = *reinterpret_cast<const uint4*>(src + i * 256 + part * 16);
      acc += __uint_as_float(v.x << 16) + __uint_as_float(v.w & 0xFFFF0000u);
    }
    __syncthreads();  // slot s free before it is reissued
  }
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  const int64_t NROWS = 8ll * 1048576;  // 2 GiB of 256-byte rows
  const int n = 524288;                  // rows gathered (cfg3: 32 heads × 16384)
  void* V;
  cudaMalloc(&V, NROWS * 256);
  cudaMemset(V, 0, NROWS * 256);
  std::vector<int> h(n);
  std::mt19937 rng(1);
  for (int i = 0; i < n; ++i) h[i] = static_cast<int>(rng() % NROWS);
  int* rows;
  cudaMalloc(&rows, n * 4);
  cudaMemcpy(rows, h.data(), n * 4, cudaMemcpyHostToDevice);
  float* out;
  cudaMalloc(&out, 4);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  CUtensorMap map;
  const cuuint64_t dims[2] = {128, static_cast<cuuint64_t>(NROWS)};
  const cuuint64_t strides[1] = {256};
  const cuuint32_t box[2] = {128, 1};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, V, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", r);
    return 1;
  }
  auto run = [&](auto kern, int nslot, int slot, int ctas_per_sm, const char* name) {
    const int smem = nslot * slot * 256;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int grid = 148 * ctas_per_sm;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) kern<<<grid, 256, smem>>>(map, rows, n, out);
    cudaEventRecord(a);
    const int reps = 20;
    for (int w = 0; w < reps; ++w) kern<<<grid, 256, smem>>>(map, rows, n, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    printf("%-34s grid %4d smem %6d: %7.2f us  %6.2f TB/s  (%s)\n", name, grid, smem, ms * 1e3,
           n * 256.0 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  };
  run(g4<8, 64, 2>, 8, 64, 1, "ring 8 x 64, 2 issuing warps");
  run(g4<8, 64, 4>, 8, 64, 1, "ring 8 x 64, 4 issuing warps");
  run(g4<8, 64, 8>, 8, 64, 1, "ring 8 x 64, 8 issuing warps");
  run(g4<6, 128, 8>, 6, 128, 1, "ring 6 x 128, 8 issuing warps");
  run(g4<12, 64, 8>, 12, 64, 1, "ring 12 x 64, 8 issuing warps");
  run(g4<4, 64, 8>, 4, 64, 2, "ring 4 x 64, 8 iss. warps, 2 CTA/SM");
  run(g4<4, 64>, 4, 64, 1, "ring 4 x 64 rows (64 KB)");
  run(g4<8, 64>, 8, 64, 1, "ring 8 x 64 rows (128 KB)");
  run(g4<12, 64>, 12, 64, 1, "ring 12 x 64 rows (192 KB)");
  run(g4<6, 128>, 6, 128, 1, "ring 6 x 128 rows (192 KB)");
  run(g4<16, 32>, 16, 32, 1, "ring 16 x 32 rows (128 KB)");
  run(g4<4, 64>, 4, 64, 2, "ring 4 x 64 rows, 2 CTAs/SM");
  run(g4<6, 64>, 6, 64, 2, "ring 6 x 64 rows, 2 CTAs/SM");
  return 0;
}
