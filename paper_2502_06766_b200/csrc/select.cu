// select.cu — K2: exact top-k over the emitted candidates, one CTA per (b, q head).
//
// Reference: _flat_topk (ann.py:154-167): argpartition, then every score strictly above the
// k-th score plus the LOWEST-id rows tied with it, ordered score-desc / id-asc. Here every
// candidate is a 64-bit composite (score key << 32 | ~row id, common.cuh), unique per row, so
// the reference's "above + lowest-id ties" set is exactly the k largest composites.
//
// One pass over the candidates (typical case):
//   1. the 4096-bucket histogram of the candidates' keys (offset above the threshold, see
//      hist_digit) is already built by the scan kernel → the bucket d* holding the k-th
//      largest is found with one block-wide scan;
//   2. a single compaction pass writes every candidate of a bucket above d* straight to the
//      output and gathers the few candidates of bucket d* into shared memory;
//   3. an MSB-first radix select over the 64-bit composites of that bucket (shared memory,
//      8-bit digits, warp-aggregated histogram atomics) picks the remaining `need` rows,
//      which resolves score ties to the lower row id exactly.
// Buckets larger than shared memory fall back to radix passes over global memory.
//
// Passes: main (fails → flags the head for the exact re-scan when fewer than k candidates
// survived the sampled threshold), fallback (re-scanned heads only), merge (sharded:
// candidates gathered from every shard; histogram built here from the candidates' range).
#include <cooperative_groups.h>
#include <math.h>

#include "attend_cand_dev.cuh"
#include "scan_dev.cuh"

namespace tkv {
namespace cg = cooperative_groups;

namespace {
constexpr int SNT = kSelectThreads;
constexpr int NWARP = SNT / 32;

struct Emit {
  int32_t* idx;
  float* sc;
  uint64_t* pk;
  uint32_t kb;
  __device__ __forceinline__ void put(uint32_t pos, uint64_t c) const {
    if (pos < kb) {
      idx[pos] = static_cast<int32_t>(comp_gid(c));
      sc[pos] = key_score(comp_key(c));
      if (pk) pk[pos] = c;
    }
  }
};

// Warp-aggregated append of the lanes with `sel` set to the output (order unspecified).
__device__ __forceinline__ void emit_sel(bool sel, uint64_t c, uint32_t* counter, const Emit& e,
                                         uint64_t& vmin) {
  const unsigned bs = __ballot_sync(kFull, sel);
  uint32_t base = 0;
  if ((threadIdx.x & 31) == 0 && bs) base = atomicAdd(counter, __popc(bs));
  base = __shfl_sync(kFull, base, 0);
  if (sel) {
    e.put(base + __popc(bs & lanemask_lt()), c);
    vmin = c < vmin ? c : vmin;
  }
}
}  // namespace

__global__ void __launch_bounds__(SNT) select_kernel(SelectParams p) {
  extern __shared__ uint64_t s_bkt[];  // [kSelectBucketCap]
  __shared__ __align__(16) uint32_t s_hist[kHistBins];
  __shared__ uint32_t s_scr[32];
  __shared__ uint32_t s_out[2];
  __shared__ uint32_t s_nout, s_nbkt, s_nvalid;
  __shared__ uint32_t s_kmin[NWARP], s_kmax[NWARP];
  __shared__ uint64_t s_rmax[NWARP], s_rmin[NWARP];

  const int bh = blockIdx.x;
  const int b = bh / p.Hq, h = bh % p.Hq;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (p.pass == kPassFallback && p.hs.flag_fail[bh] == 0u) return;

  const bool merge = p.pass == kPassMerge;
  const uint64_t* src = merge ? p.src + static_cast<int64_t>(bh) * p.merge_len
                              : p.src + static_cast<int64_t>(bh) * p.src_stride;
  int64_t n = merge ? p.src_fixed : static_cast<int64_t>(p.hs.cand_cnt[bh]);
  if (!merge && n > p.src_stride) n = p.src_stride;
  auto load = [&](int64_t i) -> uint64_t {
    if (!merge) return src[i];
    const int64_t s = i / p.merge_len;
    return src[s * p.shard_stride + (i - s * p.merge_len)];
  };

  // ---- histogram of the candidate keys: from the scan (main/fallback) or built here (merge)
  uint32_t thr, shift;
  int64_t nvalid;
  if (!merge) {
    thr = p.hs.thr[bh];
    shift = p.hs.hshift[bh];
    nvalid = n;
    const uint32_t* gh = p.hs.hist + static_cast<int64_t>(bh) * kHistBins;
    copy_g2s_u32<SNT, kHistBins>(s_hist, gh, kHistBins);
    __syncthreads();
  } else {
    uint32_t kmin = 0xffffffffu, kmax = 0u, nv = 0u;
    constexpr int UNR = 8;
    for (int64_t start = 0; start < n; start += SNT * UNR) {
      uint64_t cv[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int64_t i = start + u * SNT + tid;
        cv[u] = i < n ? load(i) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        if (cv[u]) {
          ++nv;
          const uint32_t key = comp_key(cv[u]);
          kmin = key < kmin ? key : kmin;
          kmax = key > kmax ? key : kmax;
        }
      }
    }
    nv = warp_sum(nv);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      kmin = min(kmin, __shfl_xor_sync(kFull, kmin, o));
      kmax = max(kmax, __shfl_xor_sync(kFull, kmax, o));
    }
    if (lane == 0) {
      s_kmin[warp] = kmin;
      s_kmax[warp] = kmax;
      s_scr[warp] = nv;
    }
    for (int i = tid; i < kHistBins; i += SNT) s_hist[i] = 0u;
    __syncthreads();
    if (warp == 0) {
      uint32_t a = lane < NWARP ? s_kmin[lane] : 0xffffffffu;
      uint32_t z = lane < NWARP ? s_kmax[lane] : 0u;
      uint32_t v = lane < NWARP ? s_scr[lane] : 0u;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        a = min(a, __shfl_xor_sync(kFull, a, o));
        z = max(z, __shfl_xor_sync(kFull, z, o));
        v += __shfl_xor_sync(kFull, v, o);
      }
      if (lane == 0) {
        s_out[0] = a;
        s_out[1] = z;
        s_nvalid = v;
      }
    }
    __syncthreads();
    thr = s_out[0];
    const uint32_t range = s_out[1] - s_out[0];
    const int bits = range ? 32 - __clz(range) : 0;
    shift = bits > 12 ? static_cast<uint32_t>(bits - 12) : 0u;
    nvalid = s_nvalid;
    __syncthreads();
    for (int64_t start = 0; start < n; start += SNT * UNR) {
      uint64_t cv[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int64_t i = start + u * SNT + tid;
        cv[u] = i < n ? load(i) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u)
        if (cv[u]) hist_add_aggregated(s_hist, hist_digit(comp_key(cv[u]), thr, shift));
    }
    __syncthreads();
  }

  int64_t kb;
  if (merge) {
    kb = nvalid < p.k ? nvalid : p.k;
  } else {
    const int64_t N = p.n_ctx[b];
    kb = N < p.k ? N : p.k;
  }
  const Emit em{p.idx + static_cast<int64_t>(bh) * p.k, p.scores + static_cast<int64_t>(bh) * p.k,
                p.packed_out ? p.packed_out + static_cast<int64_t>(bh) * p.k : nullptr,
                static_cast<uint32_t>(kb)};

  if (p.pass == kPassMain && nvalid < kb) {
    // The sampled threshold let fewer than k rows through: re-scan this head with thr = 0.
    uint32_t* gh = p.hs.hist + static_cast<int64_t>(bh) * kHistBins;
    for (int i = tid; i < kHistBins; i += SNT) gh[i] = 0u;
    if (tid == 0) {
      p.hs.flag_fail[bh] = 1u;
      atomicAdd(p.hs.fb_heads, 1u);
      p.hs.group_fail[b * p.Hkv + h / p.G] = 1u;
      p.hs.cand_cnt[bh] = 0u;
      p.hs.thr[bh] = 0u;
      p.hs.hshift[bh] = kNoFilterShift;
    }
    return;
  }

  // ---- bucket of the k-th largest
  const bool all = kb >= nvalid;
  uint32_t dstar = kHistBins, need = 0, bcnt = 0;
  bool whole = true;
  if (!all && kb > 0) {
    find_bucket<SNT, kHistBins>(s_hist, static_cast<uint32_t>(kb), s_out, s_scr);
    dstar = s_out[0];
    need = static_cast<uint32_t>(kb) - s_out[1];
    bcnt = s_hist[dstar];
    whole = bcnt == need;
  }
  const bool refine = !all && !whole;
  const bool big = refine && bcnt > static_cast<uint32_t>(kSelectBucketCap);
  if (tid == 0) {
    s_nout = 0u;
    s_nbkt = 0u;
  }
  __syncthreads();

  // ---- compaction: buckets above d* (or d* itself when taken whole) go straight out,
  //      the candidates of d* are gathered for refinement
  uint64_t vmax = 0ull, vmin = ~0ull;
  if (kb > 0) {
    constexpr int UNR = 8;  // loads in flight per thread (the loop is latency-bound otherwise)
    for (int64_t start = 0; start < n; start += SNT * UNR) {
      uint64_t cv[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int64_t i = start + u * SNT + tid;
        cv[u] = i < n ? load(i) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const uint64_t c = cv[u];
        const bool valid = c != 0ull;
        const uint32_t dg = valid ? hist_digit(comp_key(c), thr, shift) : 0u;
        const bool sel = valid && (all || dg > dstar || (dg == dstar && whole));
        const bool inb = valid && refine && !big && dg == dstar;
        if (valid) vmax = c > vmax ? c : vmax;
        emit_sel(sel, c, &s_nout, em, vmin);
        const unsigned bb = __ballot_sync(kFull, inb);
        uint32_t base_b = 0;
        if (lane == 0 && bb) base_b = atomicAdd(&s_nbkt, __popc(bb));
        base_b = __shfl_sync(kFull, base_b, 0);
        if (inb) {
          const uint32_t pos = base_b + __popc(bb & lanemask_lt());
          if (pos < static_cast<uint32_t>(kSelectBucketCap)) s_bkt[pos] = c;
        }
      }
    }
  }
  __syncthreads();

  // ---- exact refinement inside the threshold bucket
  if (refine) {
    int cs = 64;
    uint64_t cp = 0;
    if (!big) {
      const int64_t nb = s_nbkt;
      auto ld = [&](int64_t i, uint64_t& c) {
        c = s_bkt[i];
        return true;
      };
      radix_select_u64<SNT>(ld, nb, need, s_hist, s_scr, s_out, cs, cp);
      for (int64_t start = 0; start < nb; start += SNT) {
        const int64_t i = start + tid;
        const uint64_t c = i < nb ? s_bkt[i] : 0ull;
        emit_sel(i < nb && (c >> cs) >= cp, c, &s_nout, em, vmin);
      }
    } else {
      // rare: a threshold bucket larger than shared memory (heavy exact ties) — refine with
      // radix passes over global memory restricted to bucket d*
      auto ld = [&](int64_t i, uint64_t& c) {
        c = load(i);
        return c != 0ull && hist_digit(comp_key(c), thr, shift) == dstar;
      };
      radix_select_u64<SNT>(ld, n, need, s_hist, s_scr, s_out, cs, cp);
      for (int64_t start = 0; start < n; start += SNT) {
        const int64_t i = start + tid;
        uint64_t c = 0ull;
        const bool in = i < n && ld(i, c);
        emit_sel(in && (c >> cs) >= cp, c, &s_nout, em, vmin);
      }
    }
  }

  // pads for k > kb (reference clamps k to N, attention.py:147-149)
  for (int64_t i = kb + tid; i < p.k; i += SNT) {
    em.idx[i] = -1;
    em.sc[i] = -INFINITY;
    if (em.pk) em.pk[i] = 0ull;
  }
  vmax = warp_max_u64(vmax);
  vmin = warp_min_u64(vmin);
  if (lane == 0) {
    s_rmax[warp] = vmax;
    s_rmin[warp] = vmin;
  }
  __syncthreads();
  if (warp == 0) {
    vmax = warp_max_u64(lane < NWARP ? s_rmax[lane] : 0ull);
    vmin = warp_min_u64(lane < NWARP ? s_rmin[lane] : ~0ull);
    if (lane == 0) {
      p.meta_max[bh] = kb > 0 ? key_score(comp_key(vmax)) : -INFINITY;
      p.meta_kth[bh] = kb > 0 ? vmin : ~0ull;
      p.meta_kb[bh] = static_cast<int32_t>(kb);
      if (p.pass == kPassFallback) {
        p.hs.flag_fail[bh] = 0u;
        p.hs.group_fail[b * p.Hkv + h / p.G] = 0u;
      }
    }
  }
}

// ---------------------------------------------------------------- exactness fallback scan
// Same loop as scan.cu's scan_kernel; this translation unit is compiled with -rdc=true so the
// k-th kernel can tail-launch it (the hot scan_kernel stays whole-program compiled).
#ifndef TKV_NO_CDP
__global__ void __launch_bounds__(kScanWarps * 32, 2) fb_scan_kernel(ScanParams p) {
  extern __shared__ uint64_t s_buf[];  // [G][kScanStage]
  __shared__ uint32_t s_cnt[8];
  scan_body(p, s_buf, s_cnt);
}
#endif

// ---------------------------------------------------------------- k-th threshold only
// kth_kernel: grid (kKthCtas, B*Hq). Finds the composite threshold T of each head such that
// { c >= T } is exactly the top-kb candidate set, without writing the set itself (the
// candidate-mode attend kernel filters the candidates with T while gathering V):
//   the kKthCtas CTAs of a head form a thread-block cluster; every CTA derives the bucket d* of
//   the kb-th largest from the scan's histogram and scans its slice of the candidates for the
//   maximum and for the members of d* (collected in its shared memory); cluster rank 0 pulls
//   the other CTAs' maxima and members through distributed shared memory and refines (rank
//   counting, or radix passes for huge tie buckets → exact lower-id tie resolution). Measured
//   13.2 µs at cfg3 against 14.2–14.6 with global bucket atomics and a head ticket.
// <= 32 registers (4 CTAs per SM): a kth CTA's 16 warps then fit beside a 320-thread scan CTA in
// every SM sub-partition's 16K-register file (the scan puts 3 warps x 3840 registers on some),
// so the k-th of one part runs while the next part is scanned
// CL: CTAs per head (the cluster); the body slices by gridDim.x, so any CL works. 4 by default;
// 2 when many heads share the call (their k-th then fits beside the next part's scan: cfg5
// 1454 -> 1419 us), 8 measured slower (cfg3 365 vs 358 us).
template <int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(kKthThreads, 4) kth_kernel(SelectParams p) {
  constexpr int KT = kKthThreads, KW = KT / 32;
  extern __shared__ uint64_t s_bkt[];  // [kKthSmemBucket]
  __shared__ __align__(16) uint32_t s_hist[kHistBins];
  __shared__ uint32_t s_scr[32];
  __shared__ uint32_t s_out[2];
  __shared__ uint64_t s_rmax[KW];
  __shared__ uint32_t s_nb;     // this CTA's bucket members
  __shared__ uint64_t s_vmax;   // this CTA's largest candidate

#ifdef TKV_DIAG
  if (threadIdx.x == 0) {
    tl_start(p.tl, 53);  // first / last CTA resident (before the wait)
    tl_end(p.tl, 53);
  }
#endif
  pdl_wait();  // candidates and histograms of the scan
  if (threadIdx.x == 0) tl_start(p.tl, 5);
#ifdef TKV_DIAG
  if (threadIdx.x == 0) {
    tl_start(p.tl, 54);  // first / last CTA past the wait
    tl_end(p.tl, 54);
  }
  uint64_t t_ph = p.tl ? ptimer() : 0ull;
#define TKV_KTH_PHASE(e) \
  if (threadIdx.x == 0) tl_phase(p.tl, e, t_ph)
#else
#define TKV_KTH_PHASE(e)
#endif
  const int bh = p.bh_begin + blockIdx.y, part = blockIdx.x, P = gridDim.x;
  const int b = bh / p.Hq, h = bh % p.Hq;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (p.pass == kPassFallback) {
    // The candidate-mode gather that follows the fallback rewrites every head's ids from
    // position 0: a head the small-k head kernel already finished must not append behind its
    // first copy (that would overwrite the k > kb pads)
    if (part == 0 && tid == 0) p.hs.out_cnt[bh] = 0u;
    if (p.hs.flag_fail[bh] == 0u) return;
  }

  const uint64_t* src = p.src + static_cast<int64_t>(bh) * p.src_stride;
  int64_t n = p.hs.cand_cnt[bh];
  if (n > p.src_stride) n = p.src_stride;
  const int64_t N = p.n_ctx[b];
  const int64_t kb = N < p.k ? N : p.k;

  if (p.pass == kPassMain && n < kb) {
    // The sampled threshold let fewer than k rows through: re-scan this head with thr = 0.
    if (part == 0) {
      uint32_t* gh = p.hs.hist + static_cast<int64_t>(bh) * kHistBins;
      for (int i = tid; i < kHistBins; i += KT) gh[i] = 0u;
      if (tid == 0) {
        p.hs.flag_fail[bh] = 1u;
        atomicAdd(p.hs.fb_heads, 1u);
        p.hs.group_fail[b * p.Hkv + h / p.G] = 1u;
        p.hs.cand_cnt[bh] = 0u;
        p.hs.thr[bh] = 0u;
        p.hs.hshift[bh] = kNoFilterShift;
        __threadfence();
        // First failing head of this call: tail-launch the exact re-scan and its k-th pass.
        // Tail launches start when this grid (and so every other head's flagging) is done, and
        // the next kernel of the caller's stream waits for them — no host round trip, and no
        // cost at all when no head fails.
#ifndef TKV_NO_CDP
        if (atomicExch(p.hs.fb_launched, 1u) == 0u) {
          fb_scan_kernel<<<p.fb_scan_grid, kScanWarps * 32, p.fb_scan_smem, cudaStreamTailLaunch>>>(p.fb_scan);
          SelectParams f = p;
          f.pass = kPassFallback;
          kth_kernel<kKthCtas><<<dim3(kKthCtas, p.bh_count ? p.bh_count : p.B * p.Hq), kKthThreads, kKthSmem,
                       cudaStreamTailLaunch>>>(f);
        }
#endif
      }
    }
    return;
  }
  if (kb == 0) {
    if (part == 0 && p.narrow_out)
      for (int i = tid; i < p.narrow_len; i += KT) p.narrow_out[static_cast<int64_t>(bh) * p.narrow_len + i] = 0ull;
    if (part == 0 && tid == 0) {
      p.meta_kth[bh] = ~0ull;
      p.meta_kb[bh] = 0;
      p.meta_max[bh] = -INFINITY;
      if (p.k2 > 0) p.meta_t2[bh] = 0ull;  // no rows: nothing withheld
      if (p.narrow_out) {
        p.narrow_cnt[bh] = 0u;
        p.bound_out[3 * bh + 0] = 0ull;
        p.bound_out[3 * bh + 1] = 0ull;
        p.bound_out[3 * bh + 2] = 0ull;
      }
      if (p.pass == kPassFallback) {
        p.hs.flag_fail[bh] = 0u;
        p.hs.group_fail[b * p.Hkv + h / p.G] = 0u;
        *p.hs.fb_launched = 0u;
      }
    }
    return;
  }

  const uint32_t thr = p.hs.thr[bh], shift = p.hs.hshift[bh];
  const bool all = kb >= n;
  uint32_t dstar = 0, need = 0, bcnt = 0;
  bool whole = true;
  const bool narrow2 = p.k2 > 0 && p.k2 < kb;  // a narrow list shorter than the selection
  TKV_KTH_PHASE(55);
  if (!all || narrow2) {
    const uint32_t* gh = p.hs.hist + static_cast<int64_t>(bh) * kHistBins;
    copy_g2s_u32<KT, kHistBins>(s_hist, gh, kHistBins);
    __syncthreads();
  }
  TKV_KTH_PHASE(56);
  if (!all) {
    find_bucket<KT, kHistBins>(s_hist, static_cast<uint32_t>(kb), s_out, s_scr);
    dstar = s_out[0];
    need = static_cast<uint32_t>(kb) - s_out[1];
    bcnt = s_hist[dstar];
    whole = bcnt == need;
  }
  if (narrow2 && part == 0) {  // sharded narrow list bound (tkv_shard_candidates2)
    find_bucket<KT, kHistBins>(s_hist, static_cast<uint32_t>(p.k2), s_out, s_scr);
    const uint32_t d2 = s_out[0];
    if (tid == 0)
      p.meta_t2[bh] = d2 + 1 < static_cast<uint32_t>(kHistBins)
                          ? static_cast<uint64_t>(thr + ((d2 + 1) << shift)) << 32
                          : ~0ull;  // the k2-th sits in the top (clamped) bucket: send none
  }
  const bool refine = !all && !whole;
  TKV_KTH_PHASE(21);
  // bucket members are collected in this CTA's shared memory; more than fit (heavy exact
  // ties) → radix passes over the head's candidates in the cluster's rank 0
  const bool big = refine && bcnt > static_cast<uint32_t>(kKthSmemBucket);

  // ---- slice scan: maximum + members of the threshold bucket
  if (tid == 0) s_nb = 0u;
  __syncthreads();
  const int64_t lo = n * part / P, hi = n * (part + 1) / P;
  uint64_t vmax = 0ull;
  constexpr int UNR = 8;
  for (int64_t start = lo; start < hi; start += KT * UNR) {
    uint64_t cv[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t i = start + u * KT + tid;
      cv[u] = i < hi ? src[i] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const uint64_t c = cv[u];
      vmax = c > vmax ? c : vmax;
      const bool inb = refine && !big && c != 0ull && hist_digit(comp_key(c), thr, shift) == dstar;
      const unsigned bb = __ballot_sync(kFull, inb);
      if (bb) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(&s_nb, __popc(bb));
        base = __shfl_sync(kFull, base, 0);
        const uint32_t pos = base + __popc(bb & lanemask_lt());
        if (inb && pos < static_cast<uint32_t>(kKthSmemBucket)) s_bkt[pos] = c;
      }
    }
  }
  vmax = warp_max_u64(vmax);
  if (lane == 0) s_rmax[warp] = vmax;
  __syncthreads();
  if (tid == 0) {
    uint64_t m = 0ull;
    for (int w = 0; w < KW; ++w) m = s_rmax[w] > m ? s_rmax[w] : m;
    s_vmax = m;
  }
  TKV_KTH_PHASE(22);
  // ---- the head's CTAs form a cluster: rank 0 pulls the other CTAs' maxima and bucket members
  // through distributed shared memory (no global atomics, no head ticket)
  cg::cluster_group cluster = cg::this_cluster();
  cluster.sync();  // every CTA's s_nb / s_bkt / s_vmax final
  const bool lead = cluster.block_rank() == 0;
  uint32_t nb = 0;
  if (lead) {
    vmax = s_vmax;
    nb = s_nb;
    for (int r = 1; r < P; ++r) {
      const uint32_t nr = *cluster.map_shared_rank(&s_nb, r);
      const uint64_t mr = *cluster.map_shared_rank(&s_vmax, r);
      vmax = mr > vmax ? mr : vmax;
      if (refine && !big && nb + nr <= static_cast<uint32_t>(kKthSmemBucket)) {
        const uint64_t* rb = cluster.map_shared_rank(s_bkt, r);
        for (uint32_t i = tid; i < nr; i += KT) s_bkt[nb + i] = rb[i];
      }
      nb += nr;
    }
  }
  cluster.sync();  // remote reads done: the other CTAs may exit
  if (!lead) return;
  TKV_KTH_PHASE(23);

  // ---- rank 0: exact threshold
  uint64_t T;
  if (all) {
    T = 1ull;  // every valid (non-zero) candidate
  } else if (whole) {
    T = static_cast<uint64_t>(thr + (dstar << shift)) << 32;  // lower bound of bucket d*
  } else {
    int cs = 64;
    uint64_t cp = 0;
    if (!big && nb <= static_cast<uint32_t>(kKthSmemBucket)) {  // typical: a few hundred members
      __shared__ uint64_t s_res;
      cp = block_rank_select<KT>(s_bkt, static_cast<int>(nb), static_cast<int>(need), &s_res);
      cs = 0;
    } else {
      // rare: a threshold bucket larger than shared memory (heavy exact ties) — radix passes
      // over all candidates restricted to bucket d*
      auto ld = [&](int64_t i, uint64_t& c) {
        c = __ldcg(&src[i]);
        return c != 0ull && hist_digit(comp_key(c), thr, shift) == dstar;
      };
      radix_select_u64<KT>(ld, n, need, s_hist, s_scr, s_out, cs, cp);
    }
    T = cp << cs;
  }
  if (p.narrow_out) {  // this rank's narrow list starts empty; the emit pass appends to it
    for (int i = tid; i < p.narrow_len; i += KT) p.narrow_out[static_cast<int64_t>(bh) * p.narrow_len + i] = 0ull;
    __syncthreads();  // (meta_t2 of this head was written by this CTA: part 0 is the cluster's rank 0)
    if (tid == 0) {
      const uint64_t t2 = narrow2 ? p.meta_t2[bh] : T;
      p.narrow_cnt[bh] = 0u;
      p.bound_out[3 * bh + 0] = t2;
      p.bound_out[3 * bh + 1] = kb >= p.k ? T : 0ull;  // fewer than k rows: none withheld
      p.bound_out[3 * bh + 2] = vmax;
    }
  }
  if (tid == 0) {
    p.meta_kth[bh] = T;
    p.meta_kb[bh] = static_cast<int32_t>(kb);
    p.meta_max[bh] = key_score(comp_key(vmax));
    if (p.k2 > 0 && !narrow2) p.meta_t2[bh] = T;  // the narrow list is the whole selection
    TKV_KTH_PHASE(24);
    if (p.pass == kPassFallback) {
      p.hs.flag_fail[bh] = 0u;
      p.hs.group_fail[b * p.Hkv + h / p.G] = 0u;
      *p.hs.fb_launched = 0u;
    }
    tl_end(p.tl, 5);
  }
}

void prepare_fallback_kernels() {
#ifndef TKV_NO_CDP
  per_device(reinterpret_cast<const void*>(fb_scan_kernel), 0, [] {
    cudaFuncSetAttribute(fb_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         8 * kScanStage * static_cast<int>(sizeof(uint64_t)));
    return 1;
  });
#endif
}

cudaError_t launch_kth(const SelectParams& p, cudaStream_t s) {
  prepare_fallback_kernels();
  per_device(reinterpret_cast<const void*>(kth_kernel<kKthCtas>), 0, [] {
    // same shared-memory carveout as the scan, so both can share an SM (parts pipeline)
    cudaFuncSetAttribute(kth_kernel<kKthCtas>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(kth_kernel<2>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    return 1;
  });
  const int nbh = p.bh_count ? p.bh_count : p.B * p.Hq;
  const bool pdl = p.pdl && p.pass == kPassMain;
  if (nbh >= kKthManyHeads)
    return launch_pdl(kth_kernel<2>, dim3(2, nbh), dim3(kKthThreads), kKthSmem, s, pdl, p);
  return launch_pdl(kth_kernel<kKthCtas>, dim3(kKthCtas, nbh), dim3(kKthThreads), kKthSmem, s, pdl, p);
}

// ---------------------------------------------------------------- small k: a few CTAs per head
// head_topk_kernel: grid (heads x C), 512 threads. Replaces kth_kernel +
// attend_cand_kernel when the selected set of a head is small: each of the head's C CTAs
// finds the k-th threshold itself (histogram bucket → bucket members → rank select, exactly as
// kth_kernel; the candidates are L2-resident, so the C-fold re-read is cheap and no cross-CTA
// hand-off is needed), then compacts the selected rows of its 1/C of the candidates into shared
// memory (idx/scores written on the way), gathers their V rows into partial slot c, and the
// last CTA of the head finishes it (pinned prefix, window, normalisation). C spreads a head's
// gather over several SMs: a random 256-byte-row gather runs at ~40 GB/s per SM
// (profiles/r1_micro.md), so one SM per head would leave most of HBM idle.
// A head whose sampled threshold let fewer than kb rows through is flagged as in kth_kernel,
// and the first such head tail-launches the exact chain: re-scan, k-th (fallback pass), and the
// candidate-mode gather over ALL heads of the call (it rewrites the good heads identically up
// to fp32 summation order).
#ifndef TKV_NO_CDP
__global__ void __launch_bounds__(NT, 4) attend_cand_fb_kernel(AttendParams p) {
  __shared__ AttSmem sm;
  extern __shared__ uint32_t s_pref[];
  attend_cand_run(p, sm, s_pref);
}
#endif

// (staging the V rows through shared memory with 1-D bulk copies instead measured 6.7 GB/s
// per SM — one 256-byte cp.async.bulk per ~36 ns — against ~25 GB/s for register loads)
constexpr int kHeadSmem = kHistBins * 4 + kHeadCap * 12;  // hist | bucket (= comp) | w
static_assert(kKthSmemBucket <= kHeadCap, "bucket aliases the selected composites");
static_assert((kHeadThreads / 32) * kD <= kHistBins, "reduction aliases the histogram");
static_assert(kHeadThreads >= NT, "finish group");

__global__ void __launch_bounds__(kHeadThreads, 1) head_topk_kernel(HeadParams hp) {
  constexpr int HT = kHeadThreads, HW = HT / 32, UNR = 16;
  const SelectParams& p = hp.s;
  const AttendParams& a = hp.a;
  extern __shared__ __align__(16) uint8_t s_dyn[];
  uint32_t* s_hist = reinterpret_cast<uint32_t*>(s_dyn);  // then s_red [HW][kD]
  float* s_red = reinterpret_cast<float*>(s_dyn);
  uint64_t* s_bkt = reinterpret_cast<uint64_t*>(s_dyn + kHistBins * 4);  // then s_comp
  uint64_t* s_comp = s_bkt;
  float* s_w = reinterpret_cast<float*>(s_dyn + kHistBins * 4 + kHeadCap * 8);
  static_assert(kHeadCap == HT * UNR, "one batch of candidates fits the row buffer");

  __shared__ AttSmem sm;
  __shared__ uint32_t s_scr[32], s_out[2], s_cnt;
  __shared__ uint64_t s_rmax[HW], s_res;
  __shared__ float s_l[HW];

  pdl_wait();  // candidates and histograms of the scan
  uint64_t t_ph = p.tl ? ptimer() : 0ull;
  if (threadIdx.x == 0) tl_start(p.tl, 5);
  const int C = hp.ctas_per_head;
  const int bh = p.bh_begin + static_cast<int>(blockIdx.x) / C, c = static_cast<int>(blockIdx.x) % C;
  const int b = bh / p.Hq, h = bh % p.Hq;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t* src = p.src + static_cast<int64_t>(bh) * p.src_stride;
  int64_t n = p.hs.cand_cnt[bh];
  if (n > p.src_stride) n = p.src_stride;
  const int64_t N = p.n_ctx[b];
  const int64_t kb = N < p.k ? N : p.k;
  if (tid == 0) tl_phase(p.tl, 10, t_ph);

  if (n < kb) {
    if (c == 0) {
      uint32_t* gh = p.hs.hist + static_cast<int64_t>(bh) * kHistBins;
      for (int i = tid; i < kHistBins; i += HT) gh[i] = 0u;
      if (tid == 0) {
        p.hs.flag_fail[bh] = 1u;
        atomicAdd(p.hs.fb_heads, 1u);
        p.hs.group_fail[b * p.Hkv + h / p.G] = 1u;
        p.hs.cand_cnt[bh] = 0u;
        p.hs.thr[bh] = 0u;
        p.hs.hshift[bh] = kNoFilterShift;
        __threadfence();
#ifndef TKV_NO_CDP
        if (atomicExch(p.hs.fb_launched, 1u) == 0u) {
          fb_scan_kernel<<<p.fb_scan_grid, kScanWarps * 32, p.fb_scan_smem, cudaStreamTailLaunch>>>(p.fb_scan);
          SelectParams f = p;
          f.pass = kPassFallback;
          f.pdl = 0;
          const int nbh = p.bh_count ? p.bh_count : p.B * p.Hq;
          kth_kernel<kKthCtas><<<dim3(kKthCtas, nbh), kKthThreads, kKthSmem, cudaStreamTailLaunch>>>(f);
          attend_cand_fb_kernel<<<hp.att_grid, NT, (nbh + 1) * sizeof(uint32_t), cudaStreamTailLaunch>>>(a);
        }
#endif
      }
    }
    return;
  }

  // ---- k-th threshold T: { c >= T } is exactly the top-kb candidate set. The first batch of
  // candidates is loaded before the histogram so both memory round trips overlap.
  uint64_t cv0[UNR];
#pragma unroll
  for (int u = 0; u < UNR; ++u) {
    const int64_t i = u * HT + tid;
    cv0[u] = i < n ? src[i] : 0ull;
  }
  const uint32_t thr = p.hs.thr[bh], shift = p.hs.hshift[bh];
  const bool all = kb >= n;  // includes kb == 0 (then n == 0)
  uint32_t dstar = 0, need = 0, bcnt = 0;
  bool whole = true;
  if (!all) {
    copy_g2s_u32<HT, kHistBins>(s_hist, p.hs.hist + static_cast<int64_t>(bh) * kHistBins, kHistBins);
    __syncthreads();
    find_bucket<HT, kHistBins>(s_hist, static_cast<uint32_t>(kb), s_out, s_scr);
    dstar = s_out[0];
    need = static_cast<uint32_t>(kb) - s_out[1];
    bcnt = s_hist[dstar];
    whole = bcnt == need;
  }
  if (tid == 0) tl_phase(p.tl, 11, t_ph);
  const bool refine = !all && !whole;
  bool big = refine && bcnt > static_cast<uint32_t>(kKthSmemBucket);
  if (tid == 0) s_cnt = 0u;
  __syncthreads();
  uint64_t vmax = 0ull;
  for (int64_t start = 0; start < n; start += HT * UNR) {
    uint64_t cv[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t i = start + u * HT + tid;
      cv[u] = start == 0 ? cv0[u] : (i < n ? src[i] : 0ull);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const uint64_t cc = cv[u];
      vmax = cc > vmax ? cc : vmax;
      const bool inb = refine && !big && cc != 0ull && hist_digit(comp_key(cc), thr, shift) == dstar;
      const unsigned bb = __ballot_sync(kFull, inb);
      if (bb) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(&s_cnt, __popc(bb));
        base = __shfl_sync(kFull, base, 0);
        const uint32_t pos = base + __popc(bb & lanemask_lt());
        if (inb && pos < static_cast<uint32_t>(kKthSmemBucket)) s_bkt[pos] = cc;
      }
    }
  }
  vmax = warp_max_u64(vmax);
  if (lane == 0) s_rmax[warp] = vmax;
  __syncthreads();
  vmax = 0ull;
#pragma unroll
  for (int w = 0; w < HW; ++w) vmax = s_rmax[w] > vmax ? s_rmax[w] : vmax;
  const uint32_t nbkt = s_cnt;
  if (nbkt > static_cast<uint32_t>(kKthSmemBucket)) big = refine;  // histogram/list mismatch guard
  if (tid == 0) tl_phase(p.tl, 12, t_ph);
  uint64_t T;
  if (all) {
    T = 1ull;  // every valid (non-zero) candidate
  } else if (whole) {
    T = static_cast<uint64_t>(thr + (dstar << shift)) << 32;  // lower bound of bucket d*
  } else if (!big) {
    T = block_rank_select<HT>(s_bkt, static_cast<int>(nbkt), static_cast<int>(need), &s_res);
  } else {
    int cs = 64;
    uint64_t cp = 0;
    auto ld = [&](int64_t i, uint64_t& cc) {
      cc = src[i];
      return cc != 0ull && hist_digit(comp_key(cc), thr, shift) == dstar;
    };
    radix_select_u64<HT>(ld, n, need, s_hist, s_scr, s_out, cs, cp);
    T = cp << cs;
  }
  if (tid == 0) { tl_end(p.tl, 7); tl_phase(p.tl, 13, t_ph); }
  const float zs = a.scale * kLog2e;
  const float mscore = key_score(comp_key(vmax));
  const float zref = kb > 0 ? mscore * zs : 0.f;
  int32_t* idx_o = a.idx_out + static_cast<int64_t>(bh) * p.k;
  float* sc_o = a.scores_out + static_cast<int64_t>(bh) * p.k;
  uint64_t* pk_o = a.packed_out ? a.packed_out + static_cast<int64_t>(bh) * p.k : nullptr;
  if (c == 0) {
    if (tid == 0) {
      p.meta_kth[bh] = kb > 0 ? T : ~0ull;
      p.meta_kb[bh] = static_cast<int32_t>(kb);
      p.meta_max[bh] = kb > 0 ? mscore : -INFINITY;
    }
    for (int i = static_cast<int>(kb) + tid; i < p.k; i += HT) {  // pads (attention.py:147-149)
      idx_o[i] = -1;
      sc_o[i] = -INFINITY;
      if (pk_o) pk_o[i] = 0ull;
    }
  }
  __syncthreads();  // s_bkt / s_cnt readers done
  if (tid == 0) s_cnt = 0u;
  __syncthreads();
  if (tid == 0) tl_phase(p.tl, 14, t_ph);

  // ---- streaming compaction of this CTA's share (candidate columns [u_lo, u_hi) of every
  // batch) of the selected rows into shared memory; whenever the next batch would overflow the
  // kHeadCap-row buffer, the buffered rows are flushed: output slots reserved (one atomic),
  // their V rows gathered into registers (16 lanes per 256-byte row, 8 rows in flight per
  // half-warp), ids / raw scores written (order unspecified).
  const int kvh = h / p.G;
  const int half = lane >> 4, part = lane & 15;
  const __nv_bfloat16* vb = a.vc + (static_cast<int64_t>(b) * a.Hkv + kvh) * a.cache_rows * kD + part * 8;
  float acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = 0.f;
  float lw = 0.f;
  __shared__ uint32_t s_gbase;
  auto flush = [&](uint32_t cnt) {  // rows [0, cnt) of s_comp / s_w; block-uniform cnt
    uint32_t rbase = 0u;  // published after the gather (a shared store here would stall the block)
    if (tid == 0 && cnt) rbase = atomicAdd(&a.out_cnt[bh], cnt);
    const int nr = static_cast<int>(cnt);
    if (a.gather) {
      constexpr int GU = 8;
      for (int r0 = warp * 2 + half; r0 < nr; r0 += 2 * HW * GU) {
        uint4 v[GU];
        float w[GU];
#pragma unroll
        for (int u = 0; u < GU; ++u) {
          const int r = r0 + 2 * HW * u;
          const int64_t row = r < nr ? static_cast<int64_t>(comp_gid(s_comp[r])) - a.row_offset : -1;
          w[u] = r < nr ? s_w[r] : 0.f;
          v[u] = row >= 0 ? ldg_stream(vb + row * kD) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < GU; ++u) {
          acc[0] = fmaf(w[u], bf16lo(v[u].x), acc[0]);
          acc[1] = fmaf(w[u], bf16hi(v[u].x), acc[1]);
          acc[2] = fmaf(w[u], bf16lo(v[u].y), acc[2]);
          acc[3] = fmaf(w[u], bf16hi(v[u].y), acc[3]);
          acc[4] = fmaf(w[u], bf16lo(v[u].z), acc[4]);
          acc[5] = fmaf(w[u], bf16hi(v[u].z), acc[5]);
          acc[6] = fmaf(w[u], bf16lo(v[u].w), acc[6]);
          acc[7] = fmaf(w[u], bf16hi(v[u].w), acc[7]);
        }
      }
      for (int i = tid; i < nr; i += HT) lw += s_w[i];
    }
    if (tid == 0) s_gbase = rbase;
    __syncthreads();
    const uint32_t gb = s_gbase;
    for (int i = tid; i < nr; i += HT) {
      const uint32_t o = gb + i;
      if (o < static_cast<uint32_t>(kb)) {
        const uint64_t cc = s_comp[i];
        idx_o[o] = static_cast<int32_t>(comp_gid(cc));
        sc_o[o] = key_score(comp_key(cc));
        if (pk_o) pk_o[o] = cc;
      }
    }
    __syncthreads();  // buffer reusable
  };
  const int u_lo = c * UNR / C, u_hi = (c + 1) * UNR / C;
  __shared__ uint32_t s_wsum[HW];
  uint32_t run = 0u;
  for (int64_t start = 0; start < n && kb > 0; start += HT * UNR) {
    uint64_t cv[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t i = start + u * HT + tid;
      const bool mine = u >= u_lo && u < u_hi;
      cv[u] = !mine ? 0ull : (start == 0 ? cv0[u] : (i < n ? src[i] : 0ull));
    }
    // block-ordered compaction: per-thread counts, one warp scan + one barrier per batch
    uint32_t mask = 0u;
#pragma unroll
    for (int u = 0; u < UNR; ++u) mask |= (cv[u] != 0ull && cv[u] >= T) ? (1u << u) : 0u;
    const uint32_t mine = __popc(mask);
    uint32_t incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    uint32_t woff = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < HW; ++w) {
      const uint32_t x = s_wsum[w];
      woff += w < warp ? x : 0u;
      tot += x;
    }
    if (run + tot > static_cast<uint32_t>(kHeadCap)) {  // a batch selects at most HT * UNR = kHeadCap
      flush(run);
      run = 0u;
    }
    uint32_t pos = run + woff + incl - mine;
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (mask & (1u << u)) {
        const uint64_t cc = cv[u];
        mark_pinned(a, bh, static_cast<int64_t>(comp_gid(cc)) - a.row_offset);
        s_comp[pos] = cc;
        s_w[pos] = exp2f(fmaf(key_score(comp_key(cc)), zs, -zref));
        ++pos;
      }
    }
    run += tot;
    __syncthreads();  // s_wsum reusable; rows visible
  }
  if (tid == 0) tl_phase(p.tl, 15, t_ph);
  flush(run);
  if (tid == 0) { tl_end(p.tl, 8); tl_phase(p.tl, 16, t_ph); }
  if (!a.gather) {
    if (tid == 0) tl_end(p.tl, 5);
    return;
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] += __shfl_xor_sync(kFull, acc[j], 16);
  if (half == 0) {
#pragma unroll
    for (int j = 0; j < 8; ++j) s_red[warp * kD + part * 8 + j] = acc[j];
  }
  lw = warp_sum(lw);
  if (lane == 0) s_l[warp] = lw;
  __syncthreads();
  if (tid < kD) {
    float o = 0.f;
#pragma unroll
    for (int w2 = 0; w2 < HW; ++w2) o += s_red[w2 * kD + tid];
    a.part_o[(static_cast<int64_t>(bh) * a.nchunks + c) * kD + tid] = o;
  }
  if (tid == 0) {
    float l = 0.f;
#pragma unroll
    for (int w2 = 0; w2 < HW; ++w2) l += s_l[w2];
    a.part_l[static_cast<int64_t>(bh) * a.nchunks + c] = l;
  }
  if (tid == 0) { tl_end(p.tl, 9); tl_phase(p.tl, 19, t_ph); }
  // ---- the head's last CTA finishes it: pinned prefix, window, normalisation (first 8 warps)
  if (tid >= NT) return;
  ticket_finish<WarpGrp<0, NT, 1>>(a, bh, C, sm);
  if (tid == 0) { tl_end(p.tl, 5); tl_phase(p.tl, 20, t_ph); }
}

cudaError_t launch_head_topk(const HeadParams& p, cudaStream_t s) {
  prepare_fallback_kernels();
  const int att_grid = per_device(reinterpret_cast<const void*>(head_topk_kernel), 0, [] {
    int per = 0;
#ifndef TKV_NO_CDP
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, attend_cand_fb_kernel, NT, 8192);
#endif
    cudaFuncSetAttribute(head_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kHeadSmem);
    const int g = device_sm_count() * (per > 0 ? per : 1);
    return g < kMaxGatherGrid ? g : kMaxGatherGrid;
  });
  HeadParams q = p;
  q.att_grid = att_grid;
  const int nbh = p.s.bh_count ? p.s.bh_count : p.s.B * p.s.Hq;
  return launch_pdl(head_topk_kernel, dim3(nbh * p.ctas_per_head), dim3(kHeadThreads), kHeadSmem, s, p.s.pdl != 0,
                    q);
}

// ---------------------------------------------------------------- k-th + gather + finish per cluster
// clus_topk_kernel: grid (kKthCtas, heads), one kKthCtas-CTA thread-block cluster per head,
// 256 threads per CTA (NT). Replaces kth_kernel + attend_cand_kernel (or head_topk_kernel) at
// moderate k, where the post-scan chain (k-th kernel, a launch gap, a gather kernel that
// re-derives its work split and finishes heads through global tickets) is latency-bound:
//   1. every CTA loads its 1/kKthCtas slice of the head's candidates into registers while it
//      reads the scan's histogram and finds the bucket d* of the kb-th largest;
//   2. slice scan: maximum + members of d* into shared memory; one cluster barrier;
//   3. every CTA pulls the other CTAs' members and maxima through distributed shared memory and
//      derives the same exact T itself (rank counting over 64-bit composites: lower-id ties,
//      ann.py:162-166) — no second barrier, no global hand-off;
//   4. the selected rows of its slice (c >= T; still in registers) are compacted into shared
//      memory, the output reservation atomic issued, their V rows gathered (16 lanes per
//      256-byte row, 8 rows in flight per half-warp) and weighted against the head max
//      (attention.py:158-167), ids / raw scores written;
//   5. the (l, o[128]) partial of each CTA goes to its shared memory; cluster rank 0 sums the
//      four in rank order (deterministic) over DSMEM and finishes the head: unselected pinned
//      rows, the window, normalisation (attention.py:107-122, 152-154).
// The CTAs fit beside a tcgen05 scan CTA (33 KB of shared memory, <= 85 registers), so under
// programmatic dependent launch they are resident before the scan ends. A head whose sampled
// threshold let fewer than kb rows through takes head_topk_kernel's exactness fallback.
#ifndef TKV_CLUS_PAD
// shared memory held beyond what the kernel uses, so that one CTA fills an SM's shared memory
// beside nothing else: the clusters then spread over 128 SMs instead of packing two or three
// CTAs per SM (measured: cfg1 35.9 -> 34.1 us, cfg2 80.0 -> 74.6 us per step)
#define TKV_CLUS_PAD 90000
#endif
constexpr int kClusFront = (static_cast<int>(sizeof(AttSmem)) > kHistBins * 4 ? static_cast<int>(sizeof(AttSmem))
                                                                                 : kHistBins * 4 + 15) / 16 * 16;
constexpr int kClusSmem = kClusFront + kKthSmemBucket * 8 + TKV_CLUS_PAD;  // [hist | AttSmem] [bucket members]
static_assert(kCandChunk % NT == 0, "one compaction batch = the registers of one slice batch");
#ifndef TKV_CLUS_CL
#define TKV_CLUS_CL 4  // CTAs per head (cluster size)
#endif
#ifndef TKV_CLUS_MINB
#define TKV_CLUS_MINB 2  // <= 128 registers: one CTA per SM anyway (TKV_CLUS_PAD)
#endif
#ifndef TKV_CLUS_GU
#define TKV_CLUS_GU 12  // V rows in flight per half-warp in the cluster kernel's gather (8: cfg2 +0.6 us)
#endif

__global__ void __cluster_dims__(TKV_CLUS_CL, 1, 1) __launch_bounds__(NT, TKV_CLUS_MINB) clus_topk_kernel(HeadParams hp) {
  constexpr int CL = TKV_CLUS_CL, UNR = kCandChunk / NT;
  const SelectParams& p = hp.s;
  const AttendParams& a = hp.a;
  extern __shared__ __align__(16) uint8_t s_dyn[];
  uint32_t* s_hist = reinterpret_cast<uint32_t*>(s_dyn);                 // before T
  AttSmem& sm = *reinterpret_cast<AttSmem*>(s_dyn);                      // after T (aliases s_hist)
  uint64_t* s_bkt = reinterpret_cast<uint64_t*>(s_dyn + kClusFront);  // read by peers until s_pulled completes
  float* s_sc = sm.sc;  // a batch's raw scores
  __shared__ uint32_t s_scr[32], s_out[2], s_nb;
  __shared__ uint64_t s_rmax[NW], s_vmax, s_res;
  // rank 0 receives every CTA's (l, o[128]) partial here (DSMEM stores by the peers)
  __shared__ __align__(16) float s_part[TKV_CLUS_CL][kD + 4];
  // s_pulled: the peers finished reading this CTA's bucket members (it may exit after it);
  // s_parts (rank 0): the peers' partials have landed
  __shared__ __align__(8) uint64_t s_pulled, s_parts;

  pdl_wait();  // candidates and histograms of the scan
  if (threadIdx.x == 0) tl_start(p.tl, 5);
#ifdef TKV_DIAG
  if (threadIdx.x == 0) tl_smid(p.tl, 249);  // SMs hosting a cluster CTA
  uint64_t t_ph = p.tl ? ptimer() : 0ull;
#define TKV_CL_PHASE(e) \
  if (threadIdx.x == 0) tl_phase(p.tl, e, t_ph)
#else
#define TKV_CL_PHASE(e)
#endif
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = static_cast<int>(cluster.block_rank());
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&s_pulled), CL - 1);
    mbar_init(smem_u32(&s_parts), CL - 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int bh = p.bh_begin + static_cast<int>(blockIdx.y);
  const int b = bh / p.Hq, h = bh % p.Hq;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t* src = p.src + static_cast<int64_t>(bh) * p.src_stride;
  int64_t n = p.hs.cand_cnt[bh];
  if (n > p.src_stride) n = p.src_stride;
  const int64_t N = p.n_ctx[b];
  const int64_t kb = N < p.k ? N : p.k;

  if (n < kb) {  // cluster-uniform: the whole cluster leaves without a barrier
    if (rank == 0) {
      uint32_t* gh = p.hs.hist + static_cast<int64_t>(bh) * kHistBins;
      for (int i = tid; i < kHistBins; i += NT) gh[i] = 0u;
      if (tid == 0) {
        p.hs.flag_fail[bh] = 1u;
        atomicAdd(p.hs.fb_heads, 1u);
        p.hs.group_fail[b * p.Hkv + h / p.G] = 1u;
        p.hs.cand_cnt[bh] = 0u;
        p.hs.thr[bh] = 0u;
        p.hs.hshift[bh] = kNoFilterShift;
        __threadfence();
#ifndef TKV_NO_CDP
        // exact chain over ALL heads (the good heads are rewritten identically up to fp32
        // summation order; the fallback k-th pass resets every head's output counter)
        if (atomicExch(p.hs.fb_launched, 1u) == 0u) {
          fb_scan_kernel<<<p.fb_scan_grid, kScanWarps * 32, p.fb_scan_smem, cudaStreamTailLaunch>>>(p.fb_scan);
          SelectParams f = p;
          f.pass = kPassFallback;
          f.pdl = 0;
          const int nbh = p.bh_count ? p.bh_count : p.B * p.Hq;
          kth_kernel<kKthCtas><<<dim3(kKthCtas, nbh), kKthThreads, kKthSmem, cudaStreamTailLaunch>>>(f);
          attend_cand_fb_kernel<<<hp.att_grid, NT, (nbh + 1) * sizeof(uint32_t), cudaStreamTailLaunch>>>(a);
        }
#endif
      }
    }
    return;
  }

  TKV_CL_PHASE(67);
  // ---- 1. slice registers + histogram bucket
  const int64_t lo = n * rank / CL, hi = n * (rank + 1) / CL;
  uint64_t cv0[UNR];
#pragma unroll
  for (int u = 0; u < UNR; ++u) {
    const int64_t i = lo + u * NT + tid;
    cv0[u] = i < hi ? src[i] : 0ull;
  }
  const uint32_t thr = p.hs.thr[bh], shift = p.hs.hshift[bh];
  const bool all = kb >= n;  // includes kb == 0 (then n == 0)
  uint32_t dstar = 0, need = 0, bcnt = 0;
  bool whole = true;
  if (!all) {
    copy_g2s_u32<NT, kHistBins>(s_hist, p.hs.hist + static_cast<int64_t>(bh) * kHistBins, kHistBins);
    __syncthreads();
    find_bucket<NT, kHistBins>(s_hist, static_cast<uint32_t>(kb), s_out, s_scr);
    dstar = s_out[0];
    need = static_cast<uint32_t>(kb) - s_out[1];
    bcnt = s_hist[dstar];
    whole = bcnt == need;
  }
  const bool refine = !all && !whole;
  bool big = refine && bcnt > static_cast<uint32_t>(kKthSmemBucket);
  TKV_CL_PHASE(68);

  // ---- 2. slice scan: maximum + members of bucket d*
  if (tid == 0) s_nb = 0u;
  __syncthreads();
  uint64_t vmax = 0ull;
  for (int64_t start = lo; start < hi; start += kCandChunk) {
    uint64_t cv[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t i = start + u * NT + tid;
      cv[u] = start == lo ? cv0[u] : (i < hi ? src[i] : 0ull);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const uint64_t cc = cv[u];
      vmax = cc > vmax ? cc : vmax;
      const bool inb = refine && !big && cc != 0ull && hist_digit(comp_key(cc), thr, shift) == dstar;
      const unsigned bb = __ballot_sync(kFull, inb);
      if (bb) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(&s_nb, __popc(bb));
        base = __shfl_sync(kFull, base, 0);
        const uint32_t pos = base + __popc(bb & lanemask_lt());
        if (inb && pos < static_cast<uint32_t>(kKthSmemBucket)) s_bkt[pos] = cc;
      }
    }
  }
  vmax = warp_max_u64(vmax);
  if (lane == 0) s_rmax[warp] = vmax;
  __syncthreads();
  if (tid == 0) {
    uint64_t m = 0ull;
    for (int w = 0; w < NW; ++w) m = s_rmax[w] > m ? s_rmax[w] : m;
    s_vmax = m;
  }
  TKV_CL_PHASE(69);
  cluster.sync();  // every CTA's s_nb / s_bkt / s_vmax final
  TKV_CL_PHASE(70);

  // ---- 3. every CTA: the other CTAs' members appended behind its own (peers read only
  // [0, their own count) of this buffer), the head maximum, and the exact T
  const uint32_t own = s_nb;
  uint32_t nb = own;
  vmax = s_vmax;
  for (int r = 0; r < CL; ++r) {
    if (r == rank) continue;
    const uint32_t nr = *cluster.map_shared_rank(&s_nb, r);
    const uint64_t mr = *cluster.map_shared_rank(&s_vmax, r);
    vmax = mr > vmax ? mr : vmax;
    if (refine && !big && nb + nr <= static_cast<uint32_t>(kKthSmemBucket)) {
      const uint64_t* rb = cluster.map_shared_rank(s_bkt, r);
      for (uint32_t i = tid; i < nr; i += NT) s_bkt[nb + i] = rb[i];
    }
    nb += nr;
  }
  if (nb > static_cast<uint32_t>(kKthSmemBucket) || own > static_cast<uint32_t>(kKthSmemBucket))
    big = refine;  // histogram / list mismatch guard
  __syncthreads();
  if (tid < CL && tid != rank) mbar_arrive_remote(mapa_shared(smem_u32(&s_pulled), tid));  // peers' reads done
  uint64_t T;
  if (all) {
    T = 1ull;  // every valid (non-zero) candidate
  } else if (whole) {
    T = static_cast<uint64_t>(thr + (dstar << shift)) << 32;  // lower bound of bucket d*
  } else if (!big) {
    T = block_rank_select_par<NT>(s_bkt, static_cast<int>(nb), static_cast<int>(need), &s_res);
  } else {
    int cs = 64;
    uint64_t cp = 0;
    auto ld = [&](int64_t i, uint64_t& cc) {
      cc = __ldcg(&src[i]);
      return cc != 0ull && hist_digit(comp_key(cc), thr, shift) == dstar;
    };
    radix_select_u64<NT>(ld, n, need, s_hist, s_scr, s_out, cs, cp);
    T = cp << cs;
  }
  if (tid == 0) tl_end(p.tl, 7);
  TKV_CL_PHASE(71);
  const float zs = a.scale * kLog2e;
  const float mscore = key_score(comp_key(vmax));
  const float zref = kb > 0 ? mscore * zs : 0.f;
  int32_t* idx_o = a.idx_out + static_cast<int64_t>(bh) * p.k;
  float* sc_o = a.scores_out + static_cast<int64_t>(bh) * p.k;
  uint64_t* pk_o = a.packed_out ? a.packed_out + static_cast<int64_t>(bh) * p.k : nullptr;
  if (rank == 0) {
    if (tid == 0) {
      p.meta_kth[bh] = kb > 0 ? T : ~0ull;
      p.meta_kb[bh] = static_cast<int32_t>(kb);
      p.meta_max[bh] = kb > 0 ? mscore : -INFINITY;
    }
    for (int i = static_cast<int>(kb) + tid; i < p.k; i += NT) {  // pads (attention.py:147-149)
      idx_o[i] = -1;
      sc_o[i] = -INFINITY;
      if (pk_o) pk_o[i] = 0ull;
    }
  }

  // ---- 4. this slice's selected rows: compaction, reservation, V gather, ids / scores
  float acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = 0.f;
  float lw = 0.f;
  for (int64_t start = lo; start < hi && kb > 0; start += kCandChunk) {
    uint64_t cv[UNR];
    bool sel[UNR];
    uint32_t mine = 0;
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t i = start + u * NT + tid;
      cv[u] = start == lo ? cv0[u] : (i < hi ? src[i] : 0ull);
      sel[u] = cv[u] != 0ull && cv[u] >= T;
      mine += sel[u] ? 1u : 0u;
    }
    uint32_t incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    __syncthreads();  // the previous batch's gather no longer reads sm.row / sm.w (and s_hist is dead)
    if (lane == 31) sm.wcnt[warp] = incl;
    __syncthreads();
    uint32_t woff = 0, m = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      woff += w < warp ? sm.wcnt[w] : 0u;
      m += sm.wcnt[w];
    }
    uint32_t rbase = 0u;  // published after the gather (a shared store here would stall the barrier)
    if (tid == 0 && m) rbase = atomicAdd(&a.out_cnt[bh], m);
    uint32_t pos = woff + incl - mine;
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (sel[u]) {
        const int64_t local = static_cast<int64_t>(comp_gid(cv[u])) - a.row_offset;
        mark_pinned(a, bh, local);
        const float sc = key_score(comp_key(cv[u]));
        sm.row[pos] = static_cast<int32_t>(local);
        sm.w[pos] = exp2f(fmaf(sc, zs, -zref));
        s_sc[pos] = sc;
        ++pos;
      }
    }
    __syncthreads();
    TKV_CL_PHASE(75);
    // (the candidates leave registers here: nothing but the V rows is live across the gather,
    // so every row load of a round is issued before the first use)
    if (a.gather) gather_acc<CtaGrp, TKV_CLUS_GU>(a, bh, static_cast<int>(m), sm, acc, lw);
    TKV_CL_PHASE(76);
    if (tid == 0) sm.base = rbase;
    __syncthreads();
    const uint32_t obase = sm.base;
    for (uint32_t i = tid; i < m; i += NT) {  // ids / raw scores (order unspecified)
      const uint32_t o = obase + i;
      if (o < static_cast<uint32_t>(kb)) {
        const uint32_t gid = static_cast<uint32_t>(static_cast<int64_t>(sm.row[i]) + a.row_offset);
        idx_o[o] = static_cast<int32_t>(gid);
        sc_o[o] = s_sc[i];
        if (pk_o) pk_o[o] = make_comp(score_key(s_sc[i]), gid);  // the composite, rebuilt exactly
      }
    }
  }

  TKV_CL_PHASE(72);
  // ---- 5. partials: (l, o) of this CTA into shared memory; rank 0 sums them and finishes
  if (a.gather) {
    const int half = lane >> 4, part = lane & 15;
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] += __shfl_xor_sync(kFull, acc[j], 16);
    __syncthreads();  // sm.row / sm.w readers done
    if (half == 0) {
#pragma unroll
      for (int j = 0; j < 8; ++j) sm.red[warp][part * 8 + j] = acc[j];
    }
    lw = warp_sum(lw);
    if (lane == 0) sm.l[warp] = lw;
    __syncthreads();
    // this CTA's partial → slot [rank] of rank 0's shared memory (DSMEM stores)
    float* dst = cluster.map_shared_rank(&s_part[rank][0], 0);
    if (tid < kD) {
      float o = 0.f;
#pragma unroll
      for (int w2 = 0; w2 < NW; ++w2) o += sm.red[w2][tid];
      dst[1 + tid] = o;
    }
    if (tid == 0) {
      float l = 0.f;
#pragma unroll
      for (int w2 = 0; w2 < NW; ++w2) l += sm.l[w2];
      dst[0] = l;
    }
  }
  __threadfence();  // pinned-prefix marks before the finishing CTA reads them
  __syncthreads();  // the partial stores of the whole CTA precede thread 0's release
  if (rank != 0) {
    if (tid == 0) mbar_arrive_remote(mapa_shared(smem_u32(&s_parts), 0));
    mbar_wait_cluster(smem_u32(&s_pulled), 0);  // no peer still reads this CTA's members
    TKV_CL_PHASE(73);
    if (tid == 0) tl_end(p.tl, 5);
    return;
  }
  mbar_wait_cluster(smem_u32(&s_parts), 0);  // (also: every peer is past its reads of s_bkt)
  mbar_wait_cluster(smem_u32(&s_pulled), 0);
  TKV_CL_PHASE(73);
  if (!a.gather) {
    if (tid == 0) tl_end(p.tl, 5);
    return;
  }
  float o_c = 0.f, l_c = 0.f;
  for (int r = 0; r < CL; ++r) {  // rank order: deterministic
    if (tid < kD) o_c += s_part[r][1 + tid];
    l_c += s_part[r][0];
  }
  const int kvh = h / p.G;
  const int64_t nctx = a.n_ctx[b];
  __syncthreads();
  add_pinned(a, b, h, kvh, nctx, static_cast<int>(kb), zref, l_c, o_c, sm.z, sm.scr, &sm.red[0][0]);
  if (a.partial_only) {
    sm.o[tid] = o_c;
    __syncthreads();
    float* dst = a.partial_out + static_cast<int64_t>(bh) * (kD + 1);
    if (tid == 0) dst[0] = l_c;
    if (tid < kD) dst[1 + tid] = sm.o[tid] + sm.o[tid + kD];
  } else {
    finalize_head(a, b, h, kvh, nctx, zref, l_c, o_c, sm.z, sm.scr, sm.o, &sm.red[0][0]);
  }
  TKV_CL_PHASE(74);
  if (tid == 0) tl_end(p.tl, 5);
#undef TKV_CL_PHASE
}

cudaError_t launch_clus_topk(const HeadParams& p, cudaStream_t s) {
  prepare_fallback_kernels();
  const int att_grid = per_device(reinterpret_cast<const void*>(clus_topk_kernel), 0, [] {
    int per = 0;
#ifndef TKV_NO_CDP
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, attend_cand_fb_kernel, NT, 8192);
#endif
    cudaFuncSetAttribute(clus_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kClusSmem);
    const int g = device_sm_count() * (per > 0 ? per : 1);
    return g < kMaxGatherGrid ? g : kMaxGatherGrid;
  });
  HeadParams q = p;
  q.att_grid = att_grid;
  const int nbh = p.s.bh_count ? p.s.bh_count : p.s.B * p.s.Hq;
  return launch_pdl(clus_topk_kernel, dim3(TKV_CLUS_CL, nbh), dim3(NT), kClusSmem, s, p.s.pdl != 0, q);
}

// ---------------------------------------------------------------- optional sorted output
// Bitonic sort (descending composite = score desc, id asc: TopKResult order, ann.py:166)
// of the kb selected rows in shared memory.
__global__ void __launch_bounds__(SNT) sort_kernel(SortParams p) {
  extern __shared__ uint64_t s_c[];
  const int bh = p.bh_begin + blockIdx.x;
  const int kb = p.meta_kb[bh];
  if (kb <= 1) return;
  int P = 1;
  while (P < kb) P <<= 1;
  int32_t* idx = p.idx + static_cast<int64_t>(bh) * p.k;
  float* sc = p.scores + static_cast<int64_t>(bh) * p.k;
  for (int i = threadIdx.x; i < P; i += SNT)
    s_c[i] = i < kb ? make_comp(score_key(sc[i]), static_cast<uint32_t>(idx[i])) : 0ull;
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P / 2; i += SNT) {
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
  for (int i = threadIdx.x; i < kb; i += SNT) {
    const uint64_t c = s_c[i];
    idx[i] = static_cast<int32_t>(comp_gid(c));
    sc[i] = key_score(comp_key(c));
  }
}

cudaError_t launch_select(const SelectParams& p, cudaStream_t s) {
  const int smem = kSelectBucketCap * static_cast<int>(sizeof(uint64_t));
  per_device(reinterpret_cast<const void*>(select_kernel), 0, [smem] {
    cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return 1;
  });
  select_kernel<<<p.B * p.Hq, SNT, smem, s>>>(p);
  return cudaGetLastError();
}

// k > kSortMax (TopKResult order for large k, ann.py:166): every run of kSortChunk selected rows
// is bitonic-sorted in shared memory, then log2(k / kSortChunk) merge passes double the runs.
// A merge pass places each composite directly: its rank in its own run plus the number of
// larger composites in the partner run (binary search; composites are unique, so ranks never
// collide). The last pass writes idx / scores.
__global__ void __launch_bounds__(SNT) sort_chunk_kernel(SortParams p) {
  extern __shared__ uint64_t s_c[];
  const int bh = p.bh_begin + blockIdx.y;
  const int kb = p.meta_kb[bh];
  const int c0 = blockIdx.x * kSortChunk;
  if (c0 >= kb) return;
  const int n = min(kSortChunk, kb - c0);
  int P = 1;
  while (P < n) P <<= 1;
  const int32_t* idx = p.idx + static_cast<int64_t>(bh) * p.k + c0;
  const float* sc = p.scores + static_cast<int64_t>(bh) * p.k + c0;
  for (int i = threadIdx.x; i < P; i += SNT)
    s_c[i] = i < n ? make_comp(score_key(sc[i]), static_cast<uint32_t>(idx[i])) : 0ull;
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P / 2; i += SNT) {
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
  uint64_t* dst = p.buf + static_cast<int64_t>(bh) * p.k + c0;
  for (int i = threadIdx.x; i < n; i += SNT) dst[i] = s_c[i];
}

__global__ void __launch_bounds__(256) sort_merge_kernel(SortParams p, const uint64_t* __restrict__ src,
                                                         uint64_t* __restrict__ dst, int L, int last) {
  const int bh = p.bh_begin + blockIdx.y;
  const int kb = p.meta_kb[bh];
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i >= kb) return;
  const uint64_t* run = src + static_cast<int64_t>(bh) * p.k;
  const uint64_t x = run[i];
  const int r = i / L, own = i - r * L;
  const int ps = (r ^ 1) * L;
  int larger = 0;
  if (ps < kb) {  // partner run [ps, pe), descending: count its elements > x
    int lo = ps, hi = min(ps + L, kb);
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (run[mid] > x) lo = mid + 1; else hi = mid;
    }
    larger = lo - ps;
  }
  const int pos = (r & ~1) * L + own + larger;
  if (last) {
    p.idx[static_cast<int64_t>(bh) * p.k + pos] = static_cast<int32_t>(comp_gid(x));
    p.scores[static_cast<int64_t>(bh) * p.k + pos] = key_score(comp_key(x));
  } else {
    dst[static_cast<int64_t>(bh) * p.k + pos] = x;
  }
}

cudaError_t launch_sort(const SortParams& p, int nbh, cudaStream_t s, int* launches) {
  per_device(reinterpret_cast<const void*>(sort_kernel), 0, [] {
    cudaFuncSetAttribute(sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kSortMax * sizeof(uint64_t)));
    cudaFuncSetAttribute(sort_chunk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kSortChunk * sizeof(uint64_t)));
    return 1;
  });
  *launches = 0;
  if (p.k <= kSortMax) {
    int P = 1;
    while (P < p.k) P <<= 1;
    sort_kernel<<<nbh, SNT, static_cast<size_t>(P) * sizeof(uint64_t), s>>>(p);
    *launches = 1;
    return cudaGetLastError();
  }
  if (!p.buf) return cudaErrorInvalidValue;
  const int nchunk = (p.k + kSortChunk - 1) / kSortChunk;
  sort_chunk_kernel<<<dim3(nchunk, nbh), SNT, kSortChunk * sizeof(uint64_t), s>>>(p);
  *launches = 1;
  cudaError_t e = cudaGetLastError();
  // ping-pong: run buffer a at buf + bh * k, b shifted past every head this call covers
  uint64_t* a = p.buf;
  uint64_t* b = p.buf + static_cast<int64_t>(p.bh_begin + nbh) * p.k;
  for (int L = kSortChunk; e == cudaSuccess && L < p.k; L <<= 1) {
    const int last = 2 * L >= p.k;
    sort_merge_kernel<<<dim3((p.k + 255) / 256, nbh), 256, 0, s>>>(p, a, b, L, last);
    ++*launches;
    e = cudaGetLastError();
    uint64_t* t = a;
    a = b;
    b = t;
  }
  return e;
}

// Narrow-exchange exactness rule (paper_2502_06766_b200/sharded.py narrow_exchange_exact), one
// CTA per head: floor_g = the smallest composite of shard g's list (0 when the list has an
// empty slot, i.e. the shard sent everything it has); T = max floor_g; exact iff T == 0 or at
// least k gathered composites are >= T (then no withheld row can enter the global top-k).
__global__ void __launch_bounds__(256) narrow_check_kernel(const uint64_t* __restrict__ g, int n_shards,
                                                           int L, int nbh, int k, int32_t* ok) {
  // shard by shard, every thread keeping UNR loads in flight; one block reduction per shard
  __shared__ unsigned long long s_min[2][8];
  __shared__ uint32_t s_cnt[8];
  const int bh = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int UNR = 8;
  unsigned long long T = 0ull;
  for (int s = 0; s < n_shards; ++s) {
    const uint64_t* src = g + (static_cast<int64_t>(s) * nbh + bh) * L;
    unsigned long long m = ~0ull;
    for (int base = 0; base < L; base += 256 * UNR) {
      unsigned long long v[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int i = base + u * 256 + tid;
        v[u] = i < L ? src[i] : ~0ull;
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) m = min(m, v[u]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(kFull, m, o));
    if (lane == 0) s_min[s & 1][warp] = m;  // double-buffered: one barrier per shard
    __syncthreads();
    unsigned long long f = s_min[s & 1][0];
#pragma unroll
    for (int w = 1; w < 8; ++w) f = min(f, s_min[s & 1][w]);
    T = max(T, f);  // f == 0: the shard's list has an empty slot, nothing withheld
  }
  if (T == 0ull) {
    if (tid == 0) ok[bh] = 1;
    return;
  }
  uint32_t c = 0;
  for (int s = 0; s < n_shards; ++s) {
    const uint64_t* src = g + (static_cast<int64_t>(s) * nbh + bh) * L;
    for (int base = 0; base < L; base += 256 * UNR) {
      unsigned long long v[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int i = base + u * 256 + tid;
        v[u] = i < L ? src[i] : 0ull;
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) c += v[u] >= T ? 1u : 0u;
    }
  }
  c = warp_sum(c);
  if (lane == 0) s_cnt[warp] = c;
  __syncthreads();
  if (tid == 0) {
    uint32_t t = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += s_cnt[w];
    ok[bh] = t >= static_cast<uint32_t>(k) ? 1 : 0;
  }
}

cudaError_t launch_narrow_check(const uint64_t* gathered, int n_shards, int list_len, int nbh, int k,
                                int32_t* ok, cudaStream_t s) {
  narrow_check_kernel<<<nbh, 256, 0, s>>>(gathered, n_shards, list_len, nbh, k, ok);
  return cudaGetLastError();
}

}  // namespace tkv
