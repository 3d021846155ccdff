// Microbenchmark: gap between the end of a grid and the start of the next one when the next is
// (a) launched from the host into the same stream, (b) tail-launched from the first grid
// (cudaStreamTailLaunch), (c) launched with programmatic dependent launch (no early trigger).
// Each grid is 128 CTAs × 512 threads (the k-th kernel's shape), the second 592 × 256 (the
// gather's); stamps are %globaltimer (last end of A, first start of B).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -rdc=true -o launch_gap launch_gap.cu -lcudadevrt
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gt() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void kB(unsigned long long* ts) {
  if (threadIdx.x == 0) atomicMin(&ts[1], gt());
}
__global__ void kA(unsigned long long* ts, int tail) {
  // a little work so the grid is not trivially short
  __shared__ float s[512];
  s[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0 && tail) kB<<<592, 256, 0, cudaStreamTailLaunch>>>(ts);
  if (threadIdx.x == 0) atomicMax(&ts[0], gt());
}

int main() {
  unsigned long long* ts;
  cudaMalloc(&ts, 16);
  const char* names[3] = {"host launch", "tail launch", "PDL launch (implicit trigger)"};
  for (int mode = 0; mode < 3; ++mode) {
    double sum = 0;
    const int R = 50;
    for (int r = 0; r < R + 5; ++r) {
      unsigned long long init[2] = {0ull, ~0ull};
      cudaMemcpy(ts, init, 16, cudaMemcpyHostToDevice);
      kA<<<128, 512>>>(ts, mode == 1);
      if (mode == 0) kB<<<592, 256>>>(ts);
      if (mode == 2) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(592);
        cfg.blockDim = dim3(256);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kB, ts);
      }
      cudaDeviceSynchronize();
      unsigned long long h[2];
      cudaMemcpy(h, ts, 16, cudaMemcpyDeviceToHost);
      if (r >= 5) sum += (double)(long long)(h[1] - h[0]);
    }
    printf("%-32s gap end(A) -> start(B): %.2f us  (%s)\n", names[mode], sum / R / 1e3,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
