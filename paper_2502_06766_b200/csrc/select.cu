// select.cu — K2: exact top-k over the emitted candidates, one CTA per (b, q head).
//
// Reference: _flat_topk (ann.py:154-167): argpartition, then every score strictly above the
// k-th score plus the LOWEST-id rows tied with it, ordered score-desc / id-asc. Here the
// candidates are 64-bit composites (score key << 32 | ~row id, common.cuh), unique per row, so
// the reference's "above + lowest-id ties" set is exactly the k largest composites. It is found
// with an MSB-first radix select (digit widths 12/10/10 over the score key, then 8-bit digits
// over the row id, used only while ties remain), each pass a shared-memory histogram over the
// candidates still matching the prefix, ending as soon as a bucket is taken whole.
//
// Passes: main (candidates from the sampled-threshold scan; fails → flags the head for the
// fallback re-scan when fewer than k survived), fallback (re-scanned heads only), merge
// (sharded: candidates gathered from every shard, empty slots = 0).
#include <math.h>

#include "common.cuh"
#include "internal.h"

namespace tkv {

namespace {
constexpr int NT = kSelectThreads;
__device__ __forceinline__ int digit_width(int pi) { return pi == 0 ? 12 : (pi < 3 ? 10 : 8); }

__device__ __forceinline__ void find_bucket_w(int w, const uint32_t* hist, uint32_t need,
                                              uint32_t* out, uint32_t* scr) {
  if (w == 12)
    find_bucket<NT, 4096>(hist, need, out, scr);
  else if (w == 10)
    find_bucket<NT, 1024>(hist, need, out, scr);
  else
    find_bucket<NT, 256>(hist, need, out, scr);
}
}  // namespace

__global__ void __launch_bounds__(NT) select_kernel(SelectParams p) {
  __shared__ uint32_t s_hist[4096];
  __shared__ uint32_t s_scr[32];
  __shared__ uint32_t s_out[2];
  __shared__ uint32_t s_wofs[32];
  __shared__ uint32_t s_tot;
  __shared__ uint32_t s_nvalid;
  __shared__ uint64_t s_rmax[32], s_rmin[32];

  const int bh = blockIdx.x;
  const int b = bh / p.Hq, h = bh % p.Hq;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (p.pass == kPassFallback && p.flag_fail[bh] == 0u) return;

  const bool merge = p.pass == kPassMerge;
  const uint64_t* src = merge ? p.src + static_cast<int64_t>(bh) * p.k
                              : p.src + static_cast<int64_t>(bh) * p.src_stride;
  int64_t n = p.src_cnt ? static_cast<int64_t>(p.src_cnt[bh]) : p.src_fixed;
  if (!merge && n > p.src_stride) n = p.src_stride;
  auto load = [&](int64_t i) -> uint64_t {
    if (!merge) return src[i];
    const int64_t s = i / p.k;
    return src[s * p.shard_stride + (i - s * p.k)];
  };

  // ---- pass 1: 12-bit histogram of the top digit + number of valid candidates
  for (int i = tid; i < 4096; i += NT) s_hist[i] = 0u;
  if (tid == 0) s_nvalid = 0u;
  __syncthreads();
  uint32_t nv = 0;
  for (int64_t i = tid; i < n; i += NT) {
    const uint64_t c = load(i);
    if (c) {
      ++nv;
      atomicAdd(&s_hist[c >> 52], 1u);
    }
  }
  nv = warp_sum(nv);
  if (lane == 0 && nv) atomicAdd(&s_nvalid, nv);
  __syncthreads();
  const int64_t nvalid = s_nvalid;

  int64_t kb;
  if (p.pass == kPassMerge) {
    kb = nvalid < p.k ? nvalid : p.k;
  } else {
    const int64_t N = p.n_ctx[b];
    kb = N < p.k ? N : p.k;
  }
  int32_t* idx_out = p.idx + static_cast<int64_t>(bh) * p.k;
  float* sc_out = p.scores + static_cast<int64_t>(bh) * p.k;
  uint64_t* pk_out = p.packed_out ? p.packed_out + static_cast<int64_t>(bh) * p.k : nullptr;

  if (p.pass == kPassMain && nvalid < kb) {
    // Sampled threshold was too high for this head: re-scan it with threshold 0.
    if (tid == 0) {
      p.flag_fail[bh] = 1u;
      p.group_fail[b * p.Hkv + h / p.G] = 1u;
      p.cand_cnt[bh] = 0u;
    }
    return;
  }

  // ---- radix select: find (shift, prefix) with selected = { c : (c >> shift) >= prefix }
  bool all = kb >= nvalid;
  int shift = 64;
  uint64_t prefix = 0;
  if (!all && kb > 0) {
    uint32_t need = static_cast<uint32_t>(kb);
    for (int pi = 0; pi < 7; ++pi) {
      const int w = digit_width(pi);
      const int nshift = shift - w;
      const uint32_t mask = (1u << w) - 1u;
      if (pi > 0) {
        for (int i = tid; i <= static_cast<int>(mask); i += NT) s_hist[i] = 0u;
        __syncthreads();
        for (int64_t i = tid; i < n; i += NT) {
          const uint64_t c = load(i);
          if (c && (c >> shift) == prefix) atomicAdd(&s_hist[(c >> nshift) & mask], 1u);
        }
        __syncthreads();
      }
      find_bucket_w(w, s_hist, need, s_out, s_scr);
      const uint32_t d = s_out[0];
      need -= s_out[1];
      prefix = (prefix << w) | d;
      shift = nshift;
      const bool done = (s_hist[d] == need);
      __syncthreads();
      if (done) break;
    }
  }

  // ---- ordered compaction of the selected candidates
  if (tid == 0) s_tot = 0u;
  uint64_t vmax = 0ull, vmin = ~0ull;
  uint32_t base = 0;
  __syncthreads();
  if (kb > 0) {
    for (int64_t start = 0; start < n; start += NT) {
      const int64_t i = start + tid;
      const uint64_t c = i < n ? load(i) : 0ull;
      const bool sel = c != 0ull && (all || (c >> shift) >= prefix);
      const unsigned bal = __ballot_sync(kFull, sel);
      if (lane == 0) s_wofs[warp] = __popc(bal);
      __syncthreads();
      if (warp == 0) {
        const uint32_t v = s_wofs[lane];
        uint32_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t t = __shfl_up_sync(kFull, incl, o);
          if (lane >= o) incl += t;
        }
        s_wofs[lane] = incl - v;
        if (lane == 31) s_tot = incl;
      }
      __syncthreads();
      if (sel) {
        const uint32_t pos = base + s_wofs[warp] + __popc(bal & ((1u << lane) - 1u));
        if (pos < static_cast<uint32_t>(kb)) {
          idx_out[pos] = static_cast<int32_t>(comp_gid(c));
          sc_out[pos] = key_score(comp_key(c));
          if (pk_out) pk_out[pos] = c;
        }
        vmax = c > vmax ? c : vmax;
        vmin = c < vmin ? c : vmin;
      }
      base += s_tot;
      __syncthreads();
    }
  }
  // pads for k > kb (reference clamps k to N, attention.py:147-149)
  for (int64_t i = kb + tid; i < p.k; i += NT) {
    idx_out[i] = -1;
    sc_out[i] = -INFINITY;
    if (pk_out) pk_out[i] = 0ull;
  }
  vmax = warp_max_u64(vmax);
  vmin = warp_min_u64(vmin);
  if (lane == 0) {
    s_rmax[warp] = vmax;
    s_rmin[warp] = vmin;
  }
  __syncthreads();
  if (warp == 0) {
    vmax = warp_max_u64(s_rmax[lane]);
    vmin = warp_min_u64(s_rmin[lane]);
    if (lane == 0) {
      p.meta_max[bh] = kb > 0 ? key_score(comp_key(vmax)) : -INFINITY;
      p.meta_kth[bh] = kb > 0 ? vmin : ~0ull;
      p.meta_kb[bh] = static_cast<int32_t>(kb);
      if (p.pass == kPassFallback) {
        p.flag_fail[bh] = 0u;
        p.group_fail[b * p.Hkv + h / p.G] = 0u;
      }
    }
  }
}

// ---------------------------------------------------------------- optional sorted output
// Bitonic sort (descending composite = score desc, id asc: TopKResult order, ann.py:166)
// of the kb selected rows in shared memory.
__global__ void __launch_bounds__(NT) sort_kernel(SortParams p) {
  extern __shared__ uint64_t s_c[];
  const int bh = blockIdx.x;
  const int kb = p.meta_kb[bh];
  if (kb <= 1) return;
  int P = 1;
  while (P < kb) P <<= 1;
  int32_t* idx = p.idx + static_cast<int64_t>(bh) * p.k;
  float* sc = p.scores + static_cast<int64_t>(bh) * p.k;
  for (int i = threadIdx.x; i < P; i += NT)
    s_c[i] = i < kb ? make_comp(score_key(sc[i]), static_cast<uint32_t>(idx[i])) : 0ull;
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P / 2; i += NT) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool desc = (lo & size) == 0;
        const uint64_t a = s_c[lo], bb = s_c[hi];
        if ((a < bb) == desc) {
          s_c[lo] = bb;
          s_c[hi] = a;
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < kb; i += NT) {
    const uint64_t c = s_c[i];
    idx[i] = static_cast<int32_t>(comp_gid(c));
    sc[i] = key_score(comp_key(c));
  }
}

cudaError_t launch_select(const SelectParams& p, cudaStream_t s) {
  select_kernel<<<p.B * p.Hq, NT, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_sort(const SortParams& p, int nbh, cudaStream_t s) {
  int P = 1;
  const int kmax = p.k < kSortMax ? p.k : kSortMax;
  while (P < kmax) P <<= 1;
  const size_t smem = static_cast<size_t>(P) * sizeof(uint64_t);
  cudaFuncSetAttribute(sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(kSortMax * sizeof(uint64_t)));
  sort_kernel<<<nbh, NT, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace tkv
