// Microbenchmark: bandwidth of gathering random 256-byte rows (bf16 V rows, d = 128) from a
// 2 GiB cache, 16 lanes per row, U rows in flight per half-warp, grid = 148 × CTAs/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>
#include <random>
#include <algorithm>
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
template <int U>
__global__ void __launch_bounds__(256) gather(const uint4* V, const int* rows, int n, float* out) {
  const int lane = threadIdx.x & 31, half = lane >> 4, part = lane & 15;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  for (int r0 = (gw * 2 + half) * U; r0 < n; r0 += nw * 2 * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = r0 + u;
      v[u] = r < n ? ldg_stream(V + static_cast<int64_t>(rows[r]) * 16 + part) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += __uint_as_float(v[u].x) + __uint_as_float(v[u].w);
  }
  if (acc == 12345.f) out[0] = acc;
}
__global__ void stream_k(const uint4* K, int64_t n16, float* out) {  // a scan-like 2 GiB read
  float a = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 v = ldg_stream(K + i);
    a += __uint_as_float(v.x);
  }
  if (a == 12345.f) out[0] = a;
}
template <int U>
void run_cold(const uint4* V, const uint4* Kb, const int* rows, int n, float* out, int per_sm, const char* tag) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int grid = 148 * per_sm;
  float tot = 0.f;
  for (int i = 0; i < 6; ++i) {
    stream_k<<<148 * 8, 256>>>(Kb, (2LL << 30) / 16, out);
    cudaEventRecord(a);
    gather<U><<<grid, 256>>>(V, rows, n, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (i > 0) tot += ms;
  }
  const double ms = tot / 5;
  printf("%s U=%d: %.1f us per gather after a 2 GiB stream -> %.0f GB/s\n", tag, U, ms * 1e3, double(n) * 256 / (ms * 1e-3) / 1e9);
}
template <int U>
void run(const uint4* V, const int* rows, int n, float* out, int per_sm) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int grid = 148 * per_sm;
  gather<U><<<grid, 256>>>(V, rows, n, out);
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i) gather<U><<<grid, 256>>>(V, rows, n, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double bytes = double(n) * 256 * 10;
  printf("U=%2d ctas/sm=%d: %.1f us per gather of %d rows -> %.0f GB/s\n", U, per_sm, ms * 100, n, bytes / (ms * 1e-3) / 1e9);
}
int main(int argc, char** argv) {
  const int64_t nrows = (2LL << 30) / 256;  // 2 GiB of V rows
  if (argc > 1) {  // row list from a file (int32, global row index into the 2 GiB buffer)
    FILE* f = fopen(argv[1], "rb");
    if (!f) { perror(argv[1]); return 1; }
    std::vector<int> h;
    int x;
    while (fread(&x, 4, 1, f) == 1) h.push_back(x);
    fclose(f);
    const int n = static_cast<int>(h.size());
    fprintf(stderr, "read %d rows\n", n);
    for (int i = 0; i < n; ++i)
      if (h[i] < 0 || h[i] >= nrows) { fprintf(stderr, "row %d out of range: %d\n", i, h[i]); return 1; }
    uint4* V = nullptr;
    if (cudaMalloc(&V, nrows * 256) != cudaSuccess) { fprintf(stderr, "cudaMalloc failed\n"); return 1; }
    cudaMemset(V, 0, nrows * 256);
    int* rows; cudaMalloc(&rows, n * 4); cudaMemcpy(rows, h.data(), n * 4, cudaMemcpyHostToDevice);
    float* out; cudaMalloc(&out, 4);
    printf("file rows (%d, in output order):\n", n);
    run<8>(V, rows, n, out, 4); run<16>(V, rows, n, out, 8);
    std::mt19937 g(2); std::shuffle(h.begin(), h.end(), g);
    cudaMemcpy(rows, h.data(), n * 4, cudaMemcpyHostToDevice);
    printf("same rows shuffled:\n"); run<8>(V, rows, n, out, 4);
    uint4* Kb = nullptr;
    if (cudaMalloc(&Kb, 2LL << 30) != cudaSuccess) { fprintf(stderr, "cudaMalloc K failed\n"); return 1; }
    cudaMemset(Kb, 0, 2LL << 30);
    run_cold<8>(V, Kb, rows, n, out, 4, "shuffled, TLB/L2 cold");
    std::vector<int> hs = h;
    std::sort(hs.begin(), hs.end());  // group-major (= kv head major), ascending rows
    cudaMemcpy(rows, hs.data(), n * 4, cudaMemcpyHostToDevice);
    run_cold<8>(V, Kb, rows, n, out, 4, "sorted (group-major), TLB/L2 cold");
    run<8>(V, rows, n, out, 4);
    return 0;
  }
  uint4* V; cudaMalloc(&V, nrows * 256); cudaMemset(V, 0, nrows * 256);
  const int n = 32 * 16384;  // cfg3: 32 heads × k
  std::vector<int> h(n); std::mt19937 g(1);
  for (int i = 0; i < n; ++i) h[i] = int(g() % nrows);
  int* rows; cudaMalloc(&rows, n * 4); cudaMemcpy(rows, h.data(), n * 4, cudaMemcpyHostToDevice);
  float* out; cudaMalloc(&out, 4);
  run<4>(V, rows, n, out, 4); run<8>(V, rows, n, out, 4); run<16>(V, rows, n, out, 4); run<8>(V, rows, n, out, 8);
  run<16>(V, rows, n, out, 8); run<32>(V, rows, n, out, 4);
  // sorted rows (ascending ids within each head, like a selection in row order)
  for (int hh = 0; hh < 32; ++hh) std::sort(h.begin() + hh * 16384, h.begin() + (hh + 1) * 16384);
  cudaMemcpy(rows, h.data(), n * 4, cudaMemcpyHostToDevice);
  printf("sorted per head:\n"); run<8>(V, rows, n, out, 4); run<16>(V, rows, n, out, 8);
  return 0;
}
