// scan.cu — K1: GQA key scan with sampled-threshold candidate emission.
//
// Reference computation: ip_scores_all (ann_kernels.py:40-47) scores every cache row of one
// head; _flat_topk (ann.py:154-167) then selects. Here one pass over the bf16 K cache of a
// KV head scores all Hq/Hkv query heads of its GQA group at once (the tile is loaded once,
// shared by the group) and, instead of materialising all N scores, emits only the rows
// whose score can still be in the top-k:
//
//   sample_kernel : scores a strided sample of S = 4096 rows per (b, kv head) and, in the
//                   last CTA of each group, picks per q head a threshold key t_h = the r-th
//                   largest sampled key with r = ceil(mu + 6 sqrt(mu) + 16), mu = k·S_b/N_b
//                   (expected ≈1.5–2·k survivors). t_h = 0 (emit all) when that would not
//                   filter. It also resets the per-head candidate counters.
//   scan_kernel   : persistent CTAs stream contiguous row ranges; each warp scores 16-row
//                   tiles on the tensor cores (HMMA, see common.cuh) and appends the
//                   composite (key, ~row) of every score with key >= t_h to a per-head
//                   staging buffer in shared memory, flushed to HBM in bulk.
//
// Exactness does not depend on the sample: the selection kernel checks that at least k
// candidates survived (then the true top-k ⊆ candidates, since every top-k key >= the k-th
// key >= t_h); if not, the head is re-scanned with t_h = 0 (scan_kernel fallback pass).
#include <math.h>

#include "common.cuh"
#include "internal.h"

namespace tkv {

// r-th largest (1-indexed) of n u32 keys held in shared memory; 8-bit radix, 4 passes.
template <int NT>
__device__ uint32_t block_kth_largest_u32(const uint32_t* keys, int n, uint32_t r, uint32_t* hist,
                                          uint32_t* scr, uint32_t* out) {
  uint32_t prefix = 0, need = r;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += NT) hist[i] = 0u;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += NT) {
      const uint32_t k = keys[i];
      if (shift == 24 || (k >> (shift + 8)) == prefix) atomicAdd(&hist[(k >> shift) & 255u], 1u);
    }
    __syncthreads();
    find_bucket<NT, 256>(hist, need, out, scr);
    need -= out[1];
    prefix = (prefix << 8) | out[0];
    __syncthreads();
  }
  return prefix;
}

__global__ void __launch_bounds__(kSampleThreads) sample_kernel(SampleParams p) {
  __shared__ uint32_t s_keys[kSamples];
  __shared__ uint32_t s_hist[256];
  __shared__ uint32_t s_scr[32];
  __shared__ uint32_t s_out[2];
  __shared__ int s_last;

  const int seg = blockIdx.y;
  const int b = seg / p.Hkv, kvh = seg % p.Hkv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, c = lane & 3;
  const int64_t N = p.n_ctx[b];
  const int64_t kb = N < p.k ? N : p.k;
  int64_t stride = 1;
  int Sb = 0;
  if (N > 0) {
    stride = (N + kSamples - 1) / kSamples;
    Sb = static_cast<int>((N + stride - 1) / stride);
  }
  const bool filter = !p.no_filter && N > 0;

  if (filter) {
    QFrag f;
    load_qfrag(f, p.q + (static_cast<int64_t>(b) * p.Hq + kvh * p.G) * kD, p.G, lane);
    const __nv_bfloat16* kbase = p.kc + (static_cast<int64_t>(b) * p.Hkv + kvh) * p.cache_rows * kD;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int s0 = blockIdx.x * (kSampleThreads / 32) * 32 + warp * 32 + u * 16;
      const int sA = s0 + g, sB = s0 + g + 8;
      uint4 a[2][4];
      load_tile(a, kbase + static_cast<int64_t>(sA) * stride * kD, sA < Sb,
                kbase + static_cast<int64_t>(sB) * stride * kD, sB < Sb, c);
      float acc[4];
      score_tile(acc, a, f);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int col = 2 * c + (i & 1);
        const int s = (i < 2) ? sA : sB;
        if (col < p.G && s < kSamples) {
          const int64_t bh = static_cast<int64_t>(b) * p.Hq + kvh * p.G + col;
          p.samp[bh * kSamples + s] = (s < Sb) ? score_key(acc[i]) : 0u;
        }
      }
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(&p.ticket[seg], 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();

  const double mu = N > 0 ? static_cast<double>(kb) * Sb / static_cast<double>(N) : 0.0;
  const double rr = ceil(mu + 6.0 * sqrt(mu) + 16.0);
  for (int n = 0; n < p.G; ++n) {
    const int64_t bh = static_cast<int64_t>(b) * p.Hq + kvh * p.G + n;
    uint32_t t = 0u;
    if (filter && kb > 0 && rr < static_cast<double>(Sb)) {
      for (int i = tid; i < Sb; i += kSampleThreads) s_keys[i] = __ldcg(&p.samp[bh * kSamples + i]);
      __syncthreads();
      t = block_kth_largest_u32<kSampleThreads>(s_keys, Sb, static_cast<uint32_t>(rr), s_hist,
                                                s_scr, s_out);
    }
    if (tid == 0) {
      p.thr[bh] = t;
      p.cand_cnt[bh] = 0u;
    }
    __syncthreads();
  }
  if (tid == 0) p.ticket[seg] = 0u;
}

// ------------------------------------------------------------------------------ scan
struct ScanState {
  int64_t seg = -1;
  int b = 0, kvh = 0;
  int64_t nctx = 0;
  bool active = false;
};

__device__ __forceinline__ void scan_flush(const ScanParams& p, const ScanState& st, uint64_t* s_buf,
                                           uint32_t* s_cnt, int warp, int lane) {
  __syncthreads();
  if (st.active && warp < p.G) {
    const uint32_t cnt = s_cnt[warp];
    __syncwarp();
    if (cnt) {
      const int64_t bh = static_cast<int64_t>(st.b) * p.Hq + st.kvh * p.G + warp;
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(&p.cand_cnt[bh], cnt);
      base = __shfl_sync(kFull, base, 0);
      uint64_t* dst = p.cand + bh * p.cap + base;
      const uint64_t* src = s_buf + warp * kScanStage;
      for (uint32_t i = lane; i < cnt; i += 32) dst[i] = src[i];
    }
    if (lane == 0) s_cnt[warp] = 0u;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kScanWarps * 32, 2) scan_kernel(ScanParams p) {
  extern __shared__ uint64_t s_buf[];  // [G][kScanStage]
  __shared__ uint32_t s_cnt[8];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, c = lane & 3;
  const int64_t tps = (p.max_ctx + kScanRows - 1) / kScanRows;
  const int64_t total = static_cast<int64_t>(p.B) * p.Hkv * tps;
  const int64_t t0 = total * blockIdx.x / gridDim.x;
  const int64_t t1 = total * (blockIdx.x + 1) / gridDim.x;
  if (tid < 8) s_cnt[tid] = 0u;
  __syncthreads();

  ScanState st;
  QFrag f;
  uint32_t thr0 = 0, thr1 = 0;
  bool en0 = false, en1 = false;
  const __nv_bfloat16* kbase = nullptr;
  int since = 0;
  const int col0 = 2 * c, col1 = 2 * c + 1;

  for (int64_t t = t0; t < t1; ++t) {
    const int64_t seg = t / tps;
    if (seg != st.seg) {
      if (st.seg >= 0) scan_flush(p, st, s_buf, s_cnt, warp, lane);
      since = 0;
      st.seg = seg;
      st.b = static_cast<int>(seg / p.Hkv);
      st.kvh = static_cast<int>(seg % p.Hkv);
      st.nctx = p.n_ctx[st.b];
      st.active = !p.fallback || p.group_fail[seg] != 0u;
      if (!st.active) {
        t = (seg + 1) * tps - 1;  // skip the rest of this segment (CTA-uniform)
        continue;
      }
      load_qfrag(f, p.q + (static_cast<int64_t>(st.b) * p.Hq + st.kvh * p.G) * kD, p.G, lane);
      kbase = p.kc + (static_cast<int64_t>(st.b) * p.Hkv + st.kvh) * p.cache_rows * kD;
      const int64_t bh0 = static_cast<int64_t>(st.b) * p.Hq + st.kvh * p.G;
      en0 = col0 < p.G && (!p.fallback || p.flag_fail[bh0 + col0] != 0u);
      en1 = col1 < p.G && (!p.fallback || p.flag_fail[bh0 + col1] != 0u);
      thr0 = (col0 < p.G && !p.fallback) ? p.thr[bh0 + col0] : 0u;
      thr1 = (col1 < p.G && !p.fallback) ? p.thr[bh0 + col1] : 0u;
    }
    const int64_t tile = t - seg * tps;
    const int64_t rbase = tile * kScanRows + warp * 16 * kScanU;
    if (rbase < st.nctx) {  // warp-uniform
      uint4 a[kScanU][2][4];
#pragma unroll
      for (int u = 0; u < kScanU; ++u) {
        const int64_t rA = rbase + u * 16 + g, rB = rA + 8;
        load_tile(a[u], kbase + rA * kD, rA < st.nctx, kbase + rB * kD, rB < st.nctx, c);
      }
#pragma unroll
      for (int u = 0; u < kScanU; ++u) {
        float acc[4];
        score_tile(acc, a[u], f);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const bool hi = (i & 1) != 0;
          const int64_t row = rbase + u * 16 + g + ((i >> 1) ? 8 : 0);
          const uint32_t key = score_key(acc[i]);
          const bool pass = (hi ? en1 : en0) && row < st.nctx && key >= (hi ? thr1 : thr0);
          const unsigned m = __ballot_sync(kFull, pass);
          if (m != 0u && pass) {
            const unsigned same = m & (0x11111111u << c);
            const int leader = __ffs(same) - 1;
            const int col = hi ? col1 : col0;
            uint32_t base = 0;
            if (lane == leader) base = atomicAdd(&s_cnt[col], static_cast<uint32_t>(__popc(same)));
            base = __shfl_sync(m, base, leader);
            const uint32_t rank = __popc(same & ((1u << lane) - 1u));
            s_buf[col * kScanStage + base + rank] =
                make_comp(key, p.row_offset + static_cast<uint32_t>(row));
          }
        }
      }
    }
    if (++since == kScanFlushEvery) {
      scan_flush(p, st, s_buf, s_cnt, warp, lane);
      since = 0;
    }
  }
  if (st.seg >= 0) scan_flush(p, st, s_buf, s_cnt, warp, lane);
}

cudaError_t launch_sample(const SampleParams& p, cudaStream_t s) {
  dim3 grid(p.no_filter ? 1 : kSamples / kSampleThreads, p.B * p.Hkv);
  sample_kernel<<<grid, kSampleThreads, 0, s>>>(p);
  return cudaGetLastError();
}

static int scan_grid(int G, size_t smem) {
  static int cached[9] = {0};
  static int dev_cached = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != dev_cached) {
    for (int i = 0; i < 9; ++i) cached[i] = 0;
    dev_cached = dev;
  }
  if (cached[G] == 0) {
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, scan_kernel, kScanWarps * 32, smem);
    cached[G] = sms * (per > 0 ? per : 1);
  }
  return cached[G];
}

cudaError_t launch_scan(const ScanParams& p, cudaStream_t s) {
  const size_t smem = static_cast<size_t>(p.G) * kScanStage * sizeof(uint64_t);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         8 * kScanStage * static_cast<int>(sizeof(uint64_t)));
    attr_set = true;
  }
  const int64_t tps = (p.max_ctx + kScanRows - 1) / kScanRows;
  const int64_t total = static_cast<int64_t>(p.B) * p.Hkv * tps;
  if (total == 0) return cudaSuccess;
  int grid = scan_grid(p.G, smem);
  if (total < grid) grid = static_cast<int>(total);
  scan_kernel<<<grid, kScanWarps * 32, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace tkv
