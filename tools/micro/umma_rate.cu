// Microbenchmark: tcgen05.mma (kind::f16, cta_group::1, A and B from shared memory, SW128
// K-major) issue throughput versus N. One CTA per SM, one thread issues `iters` MMAs over
// a 32 KB A buffer (8 K steps × 2 halves pattern of the scan), commit + wait at the end.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o umma_rate umma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
template <int M, int N>
__global__ void __launch_bounds__(128, 1) k_umma(int iters, int accumulate, int spread, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t taddr;
  const uint32_t base = (smem_u32(sm) + 1023) & ~1023u;
  for (int i = threadIdx.x; i < (32768 + 65536) / 4; i += blockDim.x) ((uint32_t*)(sm + (base - smem_u32(sm))))[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;");
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = taddr;
  constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  unsigned long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    t0 = clock64();
    if (spread == 2) {  // unrolled: 8 MMAs per iteration from precomputed descriptors
      const uint64_t da = desc(base), db = desc(base + 32768);
      for (int i = 0; i < iters; i += 8) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t off = (uint64_t)(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
          const uint64_t offb = (uint64_t)(((kk >> 2) * 32768 + (kk & 3) * 32) >> 4);
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                       ::"r"(tm + (accumulate ? 0 : kk * N)), "l"(da + off), "l"(db + offb), "r"(idesc), "r"(accumulate ? (kk > 0 ? 1u : 0u) : 0u));
        }
      }
    } else
    for (int i = 0; i < iters; ++i) {
      const int kk = i & 7, h = kk >> 2, k4 = kk & 3;
      const uint32_t a = base + h * 16384 + k4 * 32;
      const uint32_t b = base + 32768 + h * 32768 + k4 * 32;
      const uint32_t d = tm + (spread ? ((i % (512 / N)) * N) : 0);
      const uint32_t acc = accumulate ? (kk > 0) : 0;
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                   ::"r"(d), "l"(desc(a)), "l"(desc(b)), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0,1,0,p;\n}" : "=r"(done) : "r"(smem_u32(&bar)));
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int M, int N>
void run(const char* tag, int accumulate, int spread) {
  unsigned long long* d; cudaMalloc(&d, 148 * 8);
  auto k = k_umma<M, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  const int iters = 4096;
  k<<<148, 128, 100000>>>(iters, accumulate, spread, d);
  k<<<148, 128, 100000>>>(iters, accumulate, spread, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0; for (int i = 0; i < 148; ++i) s += h[i];
  printf("%-8s M=%3d N=%3d acc=%d spread=%d: %.1f cycles/MMA  (%s)\n", tag, M, N, accumulate, spread, s / 148 / iters, cudaGetErrorString(e));
  cudaFree(d);
}
int main() {
  run<128, 8>("loop", 1, 0); run<128, 8>("unroll", 1, 2); run<128, 8>("unr-ind", 0, 2); run<128, 16>("unroll", 1, 2);
  run<128, 64>("unroll", 1, 2); run<128, 128>("unroll", 1, 2); run<128, 256>("unroll", 1, 2);
  return 0;
}
