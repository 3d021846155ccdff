// Microbenchmark: producer/consumer hand-off through an mbarrier ring (depth D) between two
// warps of one CTA; cycles per hand-off for try_wait (all lanes / lane 0) and test_wait spin.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int MODE>  // 0: try_wait all lanes, 1: try_wait lane 0 + syncwarp, 2: test_wait spin all lanes, 3: try_wait with suspend hint
__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) {
  uint32_t done = 0;
  if (MODE == 1) {
    if ((threadIdx.x & 31) == 0)
      while (!done) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(done) : "r"(bar), "r"(ph) : "memory");
    __syncwarp();
  } else if (MODE == 2) {
    while (!done) asm volatile("{.reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(done) : "r"(bar), "r"(ph) : "memory");
  } else if (MODE == 3) {
    while (!done) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0,1,0,p;}" : "=r"(done) : "r"(bar), "r"(ph), "r"(20) : "memory");
  } else {
    while (!done) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(done) : "r"(bar), "r"(ph) : "memory");
  }
}
template <int MODE, int D>
__global__ void k(int iters, unsigned long long* out) {
  __shared__ __align__(8) uint64_t full[D], empty[D];
  if (threadIdx.x == 0) {
    for (int i = 0; i < D; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[i])));
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const int s = i % D;
    const uint32_t ph = (i / D) & 1;
    if (warp == 0) {
      wait<MODE>(su(&empty[s]), ph ^ 1);
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&full[s])) : "memory");
    } else {
      wait<MODE>(su(&full[s]), ph);
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}
template <int MODE, int D>
void run() {
  unsigned long long* d; cudaMalloc(&d, 148 * 8);
  k<MODE, D><<<148, 64>>>(20000, d);
  k<MODE, D><<<148, 64>>>(20000, d);
  cudaDeviceSynchronize();
  unsigned long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0; for (int i = 0; i < 148; ++i) s += h[i];
  printf("mode %d depth %d: %.1f cycles per hand-off\n", MODE, D, s / 148 / 20000);
}
int main() {
  run<0, 1>(); run<0, 4>(); run<1, 4>(); run<2, 4>(); run<3, 4>(); run<2, 1>();
}
