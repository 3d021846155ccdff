// scan.cu — K1: GQA key scan with sampled-threshold candidate emission.
//
// Reference computation: ip_scores_all (ann_kernels.py:40-47) scores every cache row of one
// head; _flat_topk (ann.py:154-167) then selects. Here one pass over the bf16 K cache of a
// KV head scores all Hq/Hkv query heads of its GQA group at once (the tile is loaded once,
// shared by the group) and, instead of materialising all N scores, emits only the rows
// whose score can still be in the top-k:
//
//   sample_kernel    : scores a sample of S = 4096 rows per (b, kv head), one per stride-wide
//                      window at a hashed offset (internal.h sample_row).
//   threshold_kernel : per (b, q head), the threshold key t_h = the r-th largest sampled key,
//                      r = ceil(mu + 6 sqrt(mu) + 16), mu = k·S_b/N_b (≈1.5–2·k survivors
//                      expected; t_h = 0 = emit all when that would not filter), and the
//                      histogram granularity for the candidates' keys; resets the counters.
//   scan_kernel      : persistent CTAs stream contiguous row ranges; each warp scores
//                      16-row tiles on the tensor cores (HMMA, see common.cuh) and appends the
//                      composite (key, ~row) of every score with key >= t_h to a per-head
//                      staging buffer in shared memory, flushed to HBM in bulk together with
//                      the candidates' 4096-bucket key histogram (consumed by select.cu).
//
// Exactness does not depend on the sample: the selection kernel checks that at least k
// candidates survived (then the true top-k ⊆ candidates, since every top-k key >= the k-th
// key >= t_h); if not, the head is re-scanned with t_h = 0 (scan_kernel fallback pass).
#include <math.h>

#include <algorithm>
#include <stdlib.h>

#include "scan_dev.cuh"

namespace tkv {

// TKV_F_HOST_Q: q from pinned host memory (PCIe reads) into the workspace copy every other
// kernel reads. The sample kernel behind it is PDL-launched and waits for this grid.
__global__ void __launch_bounds__(256) stage_kernel(StageParams p) {
  pdl_trigger();
  const int64_t n0 = p.n16[0], n1 = n0 + p.n16[1], n2 = n1 + p.n16[2];
  for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < n2; i += static_cast<int64_t>(gridDim.x) * 256) {
    const int s = i < n0 ? 0 : (i < n1 ? 1 : 2);
    const int64_t j = i - (s == 0 ? 0 : (s == 1 ? n0 : n1));
    p.dst[s][j] = p.src[s][j];
  }
}

cudaError_t launch_stage(const StageParams& p, cudaStream_t s) {
  const int64_t n = p.n16[0] + p.n16[1] + p.n16[2];
  const int grid = static_cast<int>(std::min<int64_t>((n + 1023) / 1024, 148));
  stage_kernel<<<grid > 0 ? grid : 1, 256, 0, s>>>(p);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(kSampleThreads) sample_kernel(SampleParams p) {
  pdl_wait();     // only when launched behind stage_kernel (TKV_F_HOST_Q): the staged q
  pdl_trigger();  // the threshold kernel may launch now; it waits for this grid's samples
  if (threadIdx.x == 0) tl_start(p.tl, 0);
  const int seg = blockIdx.y;
  if (p.k_new && blockIdx.x == 0) {
    // GenWindow.append (attention.py:94-100, 210) of kv head (b, kvh): the token's k/v rows go
    // after the context + window; nothing reads them before the finalising gather
    const int b = seg / p.Hkv, kvh = seg % p.Hkv;
    const int32_t cnt = p.win_count[b];
    const int64_t pos = static_cast<int64_t>(p.n_ctx[b]) + cnt;
    if (pos >= 0 && pos < p.cache_rows && threadIdx.x < 32) {
      const int which = threadIdx.x >> 4, part = threadIdx.x & 15;
      const __nv_bfloat16* src = (which ? p.v_new : p.k_new) + (static_cast<int64_t>(b) * p.Hkv + kvh) * kD + part * 8;
      __nv_bfloat16* dst = (which ? p.v_dst : p.k_dst) +
                           ((static_cast<int64_t>(b) * p.Hkv + kvh) * p.cache_rows + pos) * kD + part * 8;
      *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
    }
    // (the counter advances in threshold_kernel, after this grid — and so every read — is done)
  }
  const int b = seg / p.Hkv, kvh = seg % p.Hkv;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, c = lane & 3;
  const int64_t N = p.n_ctx[b];
  if (N <= 0) return;
  const int64_t stride = sample_stride(N, p.k);
  const int Sb = static_cast<int>((N + stride - 1) / stride);
  QFrag f;
  load_qfrag(f, p.q + (static_cast<int64_t>(b) * p.Hq + kvh * p.G) * kD, p.G, lane);
  const __nv_bfloat16* kbase = p.kc + (static_cast<int64_t>(b) * p.Hkv + kvh) * p.cache_rows * kD;
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int s0 = blockIdx.x * kSampleThreads + warp * 32 + u * 16;
    const int sA = s0 + g, sB = s0 + g + 8;
    uint4 a[2][4];
    load_tile(a, kbase + sample_row(sA, stride, seg, N) * kD, sA < Sb, kbase + sample_row(sB, stride, seg, N) * kD,
              sB < Sb, c);
    float acc[4];
    score_tile(acc, a, f);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int col = 2 * c + (i & 1);
      const int s = (i < 2) ? sA : sB;
      if (col < p.G && s < Sb)
        p.samp[(static_cast<int64_t>(b) * p.Hq + kvh * p.G + col) * kSamples + s] = score_key(acc[i]);
    }
  }
  if (threadIdx.x == 0) tl_end(p.tl, 0);
}

__global__ void __launch_bounds__(kThrThreads, 4) threshold_kernel(SampleParams p) {
  constexpr int NT = kThrThreads;
  __shared__ __align__(16) uint32_t s_keys[kSamples];
  __shared__ uint32_t s_hist[2048];
  __shared__ uint32_t s_scr[32];
  __shared__ uint32_t s_out[2];
  __shared__ uint32_t s_max[32];
  pdl_trigger();  // the scan may launch now: its TMA / MMA warps need no threshold
  if (threadIdx.x == 0) tl_start(p.tl, 1);
  pdl_wait();     // samples of the sample kernel
  if (threadIdx.x == 0) tl_start(p.tl, 2);
#ifdef TKV_DIAG
  if (threadIdx.x == 0) {
    tl_start(p.tl, 45);  // diagnostics: first / last CTA past its wait
    tl_end(p.tl, 45);
    tl_smid(p.tl, 240);  // SMs hosting a threshold CTA
  }
  uint64_t t_ph = p.tl ? ptimer() : 0ull;
#define TKV_THR_PHASE(e) \
  if (tid == 0) tl_phase(p.tl, e, t_ph)
#else
#define TKV_THR_PHASE(e)
#endif
  if (p.k_new && blockIdx.x % p.Hq == 0) {
    // GenWindow.append (attention.py:94-100, 210) for batch entry b = blockIdx.x / Hq: the rows
    // were written by the sample kernel (this kernel waited for it); with no sample kernel
    // (no_filter) they are written here. Then the window counter advances.
    const int b = blockIdx.x / p.Hq;
    const int32_t cnt = p.win_count[b];
    const int64_t pos = static_cast<int64_t>(p.n_ctx[b]) + cnt;
    if (p.no_filter && pos >= 0 && pos < p.cache_rows) {
      const int pieces = p.Hkv * 16;  // 16-byte pieces per tensor
      for (int i = threadIdx.x; i < 2 * pieces; i += blockDim.x) {
        const int which = i / pieces, rem = i % pieces, kvh = rem / 16, part = rem % 16;
        const __nv_bfloat16* src = (which ? p.v_new : p.k_new) + (static_cast<int64_t>(b) * p.Hkv + kvh) * kD + part * 8;
        __nv_bfloat16* dst = (which ? p.v_dst : p.k_dst) +
                             ((static_cast<int64_t>(b) * p.Hkv + kvh) * p.cache_rows + pos) * kD + part * 8;
        *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
      }
    }
    __syncthreads();
    // the counter advances only over a written row (a full window stays full; the host layers
    // raise InputError before enqueueing such a step, as GenWindow.append does)
    if (threadIdx.x == 0 && pos >= 0 && pos < p.cache_rows) p.win_count[b] = cnt + 1;
  }
  const int bh = blockIdx.x;
  const int b = bh / p.Hq;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t N = p.n_ctx[b];
  const int64_t kb = N < p.k ? N : p.k;
  int Sb = 0;
  if (N > 0) {
    const int64_t stride = sample_stride(N, p.k);
    Sb = static_cast<int>((N + stride - 1) / stride);
  }
  const double mu = N > 0 ? static_cast<double>(kb) * Sb / static_cast<double>(N) : 0.0;
  const double rr = ceil(mu + 6.0 * sqrt(mu) + 16.0);
  const bool filter = !p.no_filter && kb > 0 && rr < static_cast<double>(Sb);

  uint32_t thr = 0u, shift = kNoFilterShift;
  if (filter) {
    copy_g2s_u32<NT, kSamples>(s_keys, p.samp + static_cast<int64_t>(bh) * kSamples, (Sb + 3) & ~3);
    __syncthreads();
    TKV_THR_PHASE(25);
    uint32_t mx = 0u;  // the sample maximum, folded into the first histogram pass
    TKV_THR_PHASE(26);
    // r-th largest sampled key: MSB-first radix select (11/11/10-bit digits) in shared memory.
    // Stopping early when the digit's bucket is taken whole leaves the bucket's lower bound,
    // which is <= the r-th key (a threshold only has to be a lower bound).
    uint32_t prefix = 0, need = static_cast<uint32_t>(rr);
    int sh = 32;
    bool exact = false;
    for (int pi = 0; pi < 3; ++pi) {
      const int w = pi < 2 ? 11 : 10;
      const int nsh = sh - w;
      const uint32_t mask = (1u << w) - 1u;
      for (int i = tid; i <= static_cast<int>(mask); i += NT) s_hist[i] = 0u;
      __syncthreads();
      // plain shared atomics: the hardware resolves same-bin lanes faster than a match.any
      // aggregation (the samples spread over a few dozen bins of the first digit)
      for (int i = tid; i < Sb; i += NT) {
        const uint32_t k = s_keys[i];
        if (sh == 32) mx = max(mx, k);
        if (sh == 32 || (k >> sh) == prefix) atomicAdd(&s_hist[(k >> nsh) & mask], 1u);
      }
      if (sh == 32) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(kFull, mx, o));
        if (lane == 0) s_max[warp] = mx;
      }
      __syncthreads();
      if (w == 11)
        find_bucket<NT, 2048>(s_hist, need, s_out, s_scr);
      else
        find_bucket<NT, 1024>(s_hist, need, s_out, s_scr);
      need -= s_out[1];
      prefix = (prefix << w) | s_out[0];
      sh = nsh;
      const uint32_t bc = s_hist[s_out[0]];
      const bool done = bc == need;
      __syncthreads();
      if (done) break;
      if (bc <= 2048u) {
        // small bucket (the usual case after one 11-bit digit): gather it and finish with
        // rank counting instead of two more radix passes
        __shared__ uint32_t s_n, s_res;
        if (tid == 0) s_n = 0u;
        __syncthreads();
        for (int i = tid; i < Sb; i += NT) {
          const uint32_t k = s_keys[i];
          if ((k >> sh) == prefix) s_hist[atomicAdd(&s_n, 1u)] = k;
        }
        __syncthreads();
        thr = block_rank_select_par<NT>(s_hist, static_cast<int>(s_n), static_cast<int>(need), &s_res);
        exact = true;
        break;
      }
    }
    if (!exact) thr = sh > 0 ? prefix << sh : prefix;
    TKV_THR_PHASE(27);
    uint32_t smax = 0u;
    for (int w = 0; w < NT / 32; ++w) smax = max(smax, s_max[w]);
    // histogram granularity: the sampled range [thr, smax] spans ~1/4 of the 4096 buckets,
    // leaving headroom for the (unsampled) true maximum; the top bucket absorbs the rest
    const uint32_t range = smax - thr;
    const int bits = range ? 32 - __clz(range) : 0;
    shift = bits > 10 ? static_cast<uint32_t>(bits - 10) : 0u;
  }
  uint32_t* gh = p.hs.hist + static_cast<int64_t>(bh) * kHistBins;
  for (int i = tid; i < kHistBins; i += NT) gh[i] = 0u;
  for (int i = tid; i < p.pin_words; i += NT) p.pin_mask[static_cast<int64_t>(bh) * p.pin_words + i] = 0u;
  if (tid == 0) {
    p.hs.thr[bh] = thr;
    p.hs.hshift[bh] = shift;
    p.hs.cand_cnt[bh] = 0u;
    p.hs.max_comp[bh] = 0ull;
    p.hs.bkt_cnt[bh] = 0u;
    p.hs.out_cnt[bh] = 0u;
    tl_end(p.tl, 1);
  }
  {
    TKV_THR_PHASE(28);
  }
}

// ------------------------------------------------------------------------------ scan
__global__ void __launch_bounds__(kScanWarps * 32, 2) scan_kernel(ScanParams p) {
  extern __shared__ uint64_t s_buf[];  // [G][kScanStage]
  __shared__ uint32_t s_cnt[8];
  pdl_trigger();
  pdl_wait();  // thresholds, zeroed counters and histograms of threshold_kernel
  scan_body(p, s_buf, s_cnt);
}

// ------------------------------------------------------------------------------ FMA scan
// The north-star baseline for the tensor-core scans: CUDA-core FMA + warp-shuffle reductions.
// A half-warp owns 8 K rows per iteration (16 lanes × 16-byte loads, 8 rows in flight); each
// lane multiplies its 8 elements of each row with the G query heads' matching elements (FMA,
// q in registers), and one transposed butterfly reduces all 8·G partial sums at once. The
// candidate emission (threshold test, per-head staging, bulk flush with the key histogram)
// is the mma.sync scan's. Selected with TKV_SCAN=fma (A/B against the tcgen05 scan by ncu).
constexpr int kFmaRowsPerIter = kScanWarps * 2 * 8;  // 8 warps × 2 half-warps × 8 rows = 128

// one exchange of the transposed butterfly: N live values → N / 2 (lane bit o picks the half it
// keeps and adds its partner's copy of); with a single value left, a plain butterfly step
template <int N, int CAP>
__device__ __forceinline__ void fma_xstep(float (&a)[CAP], int part, int o) {
  if constexpr (N >= 2) {
    const bool up = (part & o) != 0;
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
      const float send = up ? a[i] : a[i + N / 2];
      const float keep = up ? a[i + N / 2] : a[i];
      a[i] = keep + __shfl_xor_sync(kFull, send, o);
    }
  } else {
    a[0] += __shfl_xor_sync(kFull, a[0], o);
  }
}
template <int GG>
__global__ void __launch_bounds__(kScanWarps * 32, 2) scan_fma_kernel(ScanParams p) {
  extern __shared__ uint64_t s_buf[];  // [G][kScanStage]
  __shared__ uint32_t s_cnt[8];
  pdl_trigger();
  pdl_wait();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int half = lane >> 4, part = lane & 15;
  const int64_t tps = (p.max_ctx + kFmaRowsPerIter - 1) / kFmaRowsPerIter;
  const int64_t nseg = p.seg_count ? p.seg_count : static_cast<int64_t>(p.B) * p.Hkv;
  const int64_t total = nseg * tps;
  const int64_t t0 = total * blockIdx.x / gridDim.x, t1 = total * (blockIdx.x + 1) / gridDim.x;
  if (tid < 8) s_cnt[tid] = 0u;
  __syncthreads();
  ScanState st;
  float qv[GG][8];  // [head][element]: this lane's 8 elements of every head of the group
  uint32_t thr[GG];
  const __nv_bfloat16* kbase = nullptr;
  int since = 0;
  for (int64_t t = t0; t < t1; ++t) {
    const int64_t lseg = t / tps;
    const int64_t seg = p.seg_begin + lseg;
    if (seg != st.seg) {
      if (st.seg >= 0) scan_flush(p, st, s_buf, s_cnt, warp, lane);
      since = 0;
      st.seg = seg;
      st.b = static_cast<int>(seg / p.Hkv);
      st.kvh = static_cast<int>(seg % p.Hkv);
      st.nctx = p.n_ctx[st.b];
      st.active = true;
      const int64_t bh0 = static_cast<int64_t>(st.b) * p.Hq + st.kvh * p.G;
#pragma unroll
      for (int n = 0; n < GG; ++n) {
        const bool ok = n < p.G;
        const uint4 w = ok ? *reinterpret_cast<const uint4*>(p.q + (bh0 + n) * kD + part * 8) : make_uint4(0, 0, 0, 0);
        qv[n][0] = bf16lo(w.x); qv[n][1] = bf16hi(w.x); qv[n][2] = bf16lo(w.y); qv[n][3] = bf16hi(w.y);
        qv[n][4] = bf16lo(w.z); qv[n][5] = bf16hi(w.z); qv[n][6] = bf16lo(w.w); qv[n][7] = bf16hi(w.w);
        thr[n] = ok ? p.hs.thr[bh0 + n] : 0xFFFFFFFFu;
      }
      kbase = p.kc + (static_cast<int64_t>(st.b) * p.Hkv + st.kvh) * p.cache_rows * kD + part * 8;
    }
    const int64_t rbase = (t - lseg * tps) * kFmaRowsPerIter + (warp * 2 + half) * 8;
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t r = rbase + u;
      v[u] = r < st.nctx ? ldg_stream(kbase + r * kD) : make_uint4(0, 0, 0, 0);
    }
    // partial dot products of this lane's 8 elements: a[row·GG + head]
    constexpr int NV = 8 * GG;
    float a[NV];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float x[8] = {bf16lo(v[u].x), bf16hi(v[u].x), bf16lo(v[u].y), bf16hi(v[u].y),
                          bf16lo(v[u].z), bf16hi(v[u].z), bf16lo(v[u].w), bf16hi(v[u].w)};
#pragma unroll
      for (int n = 0; n < GG; ++n) {
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) acc = fmaf(qv[n][j], x[j], acc);
        a[u * GG + n] = acc;
      }
    }
    // transposed butterfly over the 16 lanes of the half-warp: each exchange sends half of the
    // remaining values and halves the count, so 8 rows × GG heads need NV/2 + NV/4 + ... shuffles
    // (3.75 per row at GG = 4) instead of 4·GG per row; lane `part` ends with values
    // j = part·C + t (t < C = NV/16) of the flattened (row, head) index
    fma_xstep<NV>(a, part, 8);
    fma_xstep<NV / 2>(a, part, 4);
    fma_xstep<NV / 4>(a, part, 2);
    fma_xstep<NV / 8>(a, part, 1);
    constexpr int C = NV >= 16 ? NV / 16 : 1;  // values per lane after the butterfly
#pragma unroll
    for (int t = 0; t < C; ++t) {
      // (row, head) of this lane's value t: j = part·C + t; with GG = 1 lane pairs hold one row
      const int j = NV >= 16 ? part * C + t : (part >> 1);
      const int row = NV >= 16 ? j / GG : j;
      const int head = NV >= 16 ? j % GG : 0;
      const int64_t r = rbase + row;
      const uint32_t key = score_key(a[t]);
      const bool valid = r < st.nctx && (NV >= 16 || (part & 1) == 0);
#pragma unroll
      for (int n = 0; n < GG; ++n) {
        if (n >= p.G) break;
        const bool pass = valid && head == n && key >= thr[n];
        const unsigned m = __ballot_sync(kFull, pass);
        if (m == 0u) continue;
        uint32_t b0 = 0;
        if (lane == static_cast<int>(__ffs(m) - 1)) b0 = atomicAdd(&s_cnt[n], static_cast<uint32_t>(__popc(m)));
        b0 = __shfl_sync(kFull, b0, __ffs(m) - 1);
        if (pass) s_buf[n * kScanStage + b0 + __popc(m & lanemask_lt())] = make_comp(key, p.row_offset + static_cast<uint32_t>(r));
      }
    }
    if (++since == kScanFlushEvery) {
      scan_flush(p, st, s_buf, s_cnt, warp, lane);
      since = 0;
    }
  }
  if (st.seg >= 0) scan_flush(p, st, s_buf, s_cnt, warp, lane);
}

cudaError_t launch_scan_fma(const ScanParams& p, cudaStream_t s) {
  const size_t smem = static_cast<size_t>(p.G) * kScanStage * sizeof(uint64_t);
  const int grid = per_device(reinterpret_cast<const void*>(scan_fma_kernel<4>), p.G, [smem] {
    for (auto kk : {scan_fma_kernel<1>, scan_fma_kernel<2>, scan_fma_kernel<4>, scan_fma_kernel<8>})
      cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           8 * kScanStage * static_cast<int>(sizeof(uint64_t)));
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, scan_fma_kernel<4>, kScanWarps * 32, smem);
    return device_sm_count() * (per > 0 ? per : 1);
  });
  auto k = p.G <= 1 ? scan_fma_kernel<1> : p.G <= 2 ? scan_fma_kernel<2> : p.G <= 4 ? scan_fma_kernel<4> : scan_fma_kernel<8>;
  return launch_pdl(k, dim3(grid), dim3(kScanWarps * 32), smem, s, p.pdl != 0, p);
}

cudaError_t launch_sample(const SampleParams& p, cudaStream_t s) {
  per_device(reinterpret_cast<const void*>(sample_kernel), 0, [] {
    // same carveout as the scan: the scan's CTAs start beside these (PDL)
    cudaFuncSetAttribute(sample_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(threshold_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    return 1;
  });
  if (!p.no_filter) {
    const int ns = p.max_samples > 0 && p.max_samples < kSamples ? p.max_samples : kSamples;
    dim3 grid((ns + kSampleThreads - 1) / kSampleThreads, p.B * p.Hkv);
    cudaError_t e = launch_pdl(sample_kernel, grid, dim3(kSampleThreads), 0, s, p.pdl != 0, p);
    if (e != cudaSuccess) return e;
  }
  return launch_pdl(threshold_kernel, dim3(p.B * p.Hq), dim3(kThrThreads), 0, s, pdl_enabled() && !p.no_filter, p);
}

static int scan_grid(int G, size_t smem) {
  return per_device(reinterpret_cast<const void*>(scan_kernel), G, [smem] {
    cudaFuncSetAttribute(scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         8 * kScanStage * static_cast<int>(sizeof(uint64_t)));
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, scan_kernel, kScanWarps * 32, smem);
    const int cap = diag_env("TKV_SCAN_CTAS_PER_SM", 0);
    if (cap > 0 && per > cap) per = cap;
    return device_sm_count() * (per > 0 ? per : 1);
  });
}

// Grid and dynamic shared memory of the scan kernel (host), also used for the device-side
// tail launch of the exactness fallback.
void scan_launch_shape(const ScanParams& p, int* grid, int* smem_bytes) {
  const size_t smem = static_cast<size_t>(p.G) * kScanStage * sizeof(uint64_t);
  const int64_t tps = (p.max_ctx + kScanRows - 1) / kScanRows;
  const int64_t total = (p.seg_count ? p.seg_count : static_cast<int64_t>(p.B) * p.Hkv) * tps;
  int g = scan_grid(p.G, smem);
  if (total < g) g = static_cast<int>(total > 0 ? total : 1);
  *grid = g;
  *smem_bytes = static_cast<int>(smem);
}

cudaError_t launch_scan(const ScanParams& p, cudaStream_t s) {
  const size_t smem = static_cast<size_t>(p.G) * kScanStage * sizeof(uint64_t);
  const int64_t tps = (p.max_ctx + kScanRows - 1) / kScanRows;
  const int64_t total = (p.seg_count ? p.seg_count : static_cast<int64_t>(p.B) * p.Hkv) * tps;
  if (total == 0) return cudaSuccess;
  int grid = scan_grid(p.G, smem);
  if (total < grid) grid = static_cast<int>(total);
  return launch_pdl(scan_kernel, dim3(grid), dim3(kScanWarps * 32), smem, s, p.pdl != 0, p);
}

}  // namespace tkv
