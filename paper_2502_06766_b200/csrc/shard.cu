// shard.cu — the device-driven exchange of the token-range sharded layer step.
//
// Every rank g publishes, per (b, q head), in a buffer its peers can read (symmetric memory over
// NVLink; in the one-GPU emulation another local buffer):
//   full[k]     its exact local top-k composites (score key << 32 | ~global id; 0 = empty),
//   narrow[k']  the full list's entries >= t2_g, fewer than k' of them (tkv_shard_candidates2),
//   bound[3]    t2_g (every row rank g withheld from its narrow list is below it), its local k-th
//               composite when it has >= k rows (else 0: it withheld nothing from the full list),
//               and its largest composite.
// The merge (shard_merge_kernel) reads every rank's lists through device pointers and decides
// per head ON THE DEVICE whether the narrow lists suffice:
//   T* = max_g t2_g; if at least k narrow candidates are >= T*, no withheld row can enter the
//   global top-k (each is below its rank's t2_g <= T*), so the narrow lists are exact
//   (sharded.py narrow_exchange_exact restates the rule); otherwise the head is merged from the
//   full lists, which are already published — no re-scan, no second exchange, no host round trip,
//   so the sharded step is CUDA-graph capturable.
// The merge is the k-th kernel's structure (select.cu kth_kernel), a 4-CTA thread-block cluster
// per head: a 4096-bin key histogram of the candidates above a lower bound every global top-k
// row clears (T* for narrow lists; for full lists the largest local k-th), the bucket of the
// k-th largest from the cluster-summed histogram, its members pulled by cluster rank 0 over
// distributed shared memory and rank-selected → the exact threshold composite T; every CTA then
// writes its candidates >= T with one output reservation per CTA (ties → lower global id, the
// reference's order, ann.py:162-166).
#include <cooperative_groups.h>

#include "common.cuh"
#include "internal.h"

namespace tkv {
namespace cg = cooperative_groups;

// ---------------------------------------------------------------- the merge
namespace {
constexpr int MT = 512, MW = MT / 32, CL = 4;
constexpr int kMergeBkt = 2048;  // bucket members rank-selected in shared memory
constexpr int kMergeCache = 12288;  // this CTA's narrow-list entries kept in shared memory (96 KB)

struct MergeSmem {
  uint32_t hist[kHistBins];
  uint32_t tot[kHistBins / CL];
  uint64_t bkt[kMergeBkt];
  uint32_t wsum[MW];
  uint32_t slsum, nb, cnt, obase, above_loc, nout;
  uint32_t bsel[3];
  uint32_t scr[32], out[2];
  uint64_t T, res;
};

// Calls fn(c) for every candidate of this CTA's ranks (g = cta, cta + CL, ...; 0 for empty
// slots and past the end), each thread loading UNR entries before using any: one memory round
// trip per batch instead of one per entry. Every lane makes the same number of calls, so fn may
// use warp ballots.
// cmode 1: also keep every loaded entry in `cache` (shared memory); cmode 2: read the entries
// from `cache` instead of the lists (peer memory over NVLink, or L2) — the merge sweeps the same
// narrow lists up to five times.
template <int UNR = 8, class Fn>
__device__ __forceinline__ void sweep(const uint64_t* const* lists, int G, int len, int bh, int cta, Fn&& fn,
                                      uint64_t* cache = nullptr, int cmode = 0) {
  const int nr = (G - cta + CL - 1) / CL;  // ranks this CTA reads
  const int total = nr * len;
  for (int base = 0; base < total; base += MT * UNR) {
    uint64_t cv[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int i = base + u * MT + static_cast<int>(threadIdx.x);
      const int r = i / len;
      if (cmode == 2) {
        cv[u] = i < total ? cache[i] : 0ull;
      } else {
        cv[u] = i < total ? lists[cta + r * CL][static_cast<int64_t>(bh) * len + (i - r * len)] : 0ull;
        if (cmode == 1 && i < total) cache[i] = cv[u];
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) fn(cv[u]);
  }
}

// block-wide exclusive prefix of v; *total = the block's sum (every thread)
__device__ __forceinline__ uint32_t block_excl(uint32_t v, uint32_t* wsum, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  uint32_t off = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < MW; ++w) {
    off += w < warp ? wsum[w] : 0u;
    tot += wsum[w];
  }
  __syncthreads();
  *total = tot;
  return off + inc - v;
}
}  // namespace

#ifdef TKV_DIAG
#define MERGE_PHASE(e) \
  if (tid == 0) tl_phase(p.tl, e, t_ph)
#else
#define MERGE_PHASE(e)
#endif

__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(MT, 1) shard_merge_kernel(ShardMergeParams p) {
  extern __shared__ __align__(16) uint8_t dyn[];
#ifdef TKV_DIAG
  uint64_t t_ph = p.tl ? ptimer() : 0ull;
#endif
  MergeSmem& s = *reinterpret_cast<MergeSmem*>(dyn);
  cg::cluster_group cluster = cg::this_cluster();
  const int cta = static_cast<int>(cluster.block_rank());
  const int bh = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31;
  const int G = p.n_shards;

  // ---- 1. bounds of every rank: T* (narrow rule), the full-list lower bound, the maximum
  uint64_t Tstar = 0ull, Tfull = 0ull, M = 0ull;
  {
    const uint64_t* b = lane < G ? p.bound[lane] + 3 * static_cast<int64_t>(bh) : nullptr;  // G <= 16
    uint64_t t2 = b ? b[0] : 0ull, kf = b ? b[1] : 0ull, mx = b ? b[2] : 0ull;
    Tstar = warp_max_u64(t2);
    Tfull = warp_max_u64(kf);
    M = warp_max_u64(mx);
  }
  // narrow candidates >= T* (this CTA: ranks cta, cta + CL, ...)
  uint64_t* cache = reinterpret_cast<uint64_t*>(dyn + ((sizeof(MergeSmem) + 15) / 16) * 16);
  const bool cacheable = ((G - cta + CL - 1) / CL) * p.narrow_len <= kMergeCache;
  uint32_t ge = 0;
  sweep(p.narrow, G, p.narrow_len, bh, cta, [&](uint64_t c) { ge += c != 0ull && c >= Tstar; }, cache,
        cacheable ? 1 : 0);
  uint32_t ge_cta;
  block_excl(ge, s.wsum, &ge_cta);
  if (tid == 0) s.cnt = ge_cta;
  cluster.sync();
  uint32_t count = 0;
#pragma unroll
  for (int r = 0; r < CL; ++r) count += *cluster.map_shared_rank(&s.cnt, r);
  const bool exact = count >= static_cast<uint32_t>(p.k) || Tstar <= 1ull;  // <= 1: nothing withheld
  MERGE_PHASE(47);

  // ---- 2. source lists and the lower bound every global top-k row clears
  const uint64_t* const* lists = exact ? p.narrow : p.full;
  const int len = exact ? p.narrow_len : p.full_len;
  const int cm = exact && cacheable ? 2 : 0;  // later sweeps of the narrow lists: from shared memory
  const uint64_t lo = exact ? Tstar : Tfull;
  const uint32_t klo = comp_key(lo), khi = comp_key(M);
  const uint32_t range = khi > klo ? khi - klo : 0u;
  const int bits = range ? 32 - __clz(range) : 0;
  const uint32_t shift = bits > 12 ? static_cast<uint32_t>(bits - 12) : 0u;

  // ---- 3. histogram of the candidates >= lo, summed over the cluster; bucket of the kb-th
  for (int i = tid; i < kHistBins; i += MT) s.hist[i] = 0u;
  __syncthreads();
  sweep(lists, G, len, bh, cta, [&](uint64_t c) {
    if (c != 0ull && c >= lo) atomicAdd(&s.hist[hist_digit(comp_key(c), klo, shift)], 1u);
  }, cache, cm);
  __syncthreads();
  cluster.sync();
  constexpr int SB = kHistBins / CL;
  uint32_t part = 0;
  for (int j = tid; j < SB; j += MT) {  // this CTA's slice of the bins, summed over the cluster
    uint32_t v[CL];
#pragma unroll
    for (int r = 0; r < CL; ++r) v[r] = cluster.map_shared_rank(s.hist, r)[cta * SB + j];
    uint32_t t = 0;
#pragma unroll
    for (int r = 0; r < CL; ++r) t += v[r];
    s.tot[j] = t;
    part += t;
  }
  uint32_t slice_total;
  block_excl(part, s.wsum, &slice_total);
  if (tid == 0) s.slsum = slice_total;
  cluster.sync();
  uint32_t total = 0, sl[CL];
#pragma unroll
  for (int r = 0; r < CL; ++r) {
    sl[r] = *cluster.map_shared_rank(&s.slsum, r);
    total += sl[r];
  }
  const uint32_t kb = total < static_cast<uint32_t>(p.k) ? total : static_cast<uint32_t>(p.k);
  MERGE_PHASE(48);
  // the slice holding the kb-th largest (every CTA, from the 4 slice totals); its owner finds
  // the digit in its own cluster-summed bins and publishes it
  int s_star = 0;
  uint32_t above_s = 0;
  if (kb > 0) {
    for (int r = CL - 1; r >= 0; --r) {
      if (above_s + sl[r] >= kb) {
        s_star = r;
        break;
      }
      above_s += sl[r];
    }
  }
  if (kb > 0 && cta == s_star && tid < 32) {
    constexpr int PER = SB / 32;
    uint32_t loc[PER], sum = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      loc[j] = s.tot[SB - 1 - (lane * PER + j)];
      sum += loc[j];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    uint32_t cum = above_s + incl - sum;
    if (cum < kb && kb <= cum + sum) {
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        if (cum + loc[j] >= kb) {
          const int jj = SB - 1 - (lane * PER + j);
          s.bsel[0] = static_cast<uint32_t>(s_star * SB + jj);  // d*
          s.bsel[1] = cum;                                      // rows above d*
          s.bsel[2] = loc[j];                                   // rows in d* (cluster-wide)
          break;
        }
        cum += loc[j];
      }
    }
  }
  cluster.sync();
  uint32_t dstar = 0, need = 0, bcnt = 0;
  if (kb > 0) {
    const uint32_t* bs = cluster.map_shared_rank(s.bsel, s_star);
    dstar = bs[0];
    need = kb - bs[1];
    bcnt = bs[2];
  }
  const bool whole = bcnt == need;
  const bool big = kb > 0 && !whole && bcnt > static_cast<uint32_t>(kMergeBkt);
  MERGE_PHASE(49);

  // ---- 4. the exact threshold composite T = the need-th largest member of bucket d*
  if (tid == 0) {
    s.nb = 0u;
    s.nout = 0u;
  }
  {  // this CTA's rows in buckets above d* (its local histogram): selected whatever T is
    uint32_t v = 0;
    for (int d = dstar + 1 + tid; d < kHistBins; d += MT) v += s.hist[d];
    uint32_t tot;
    block_excl(v, s.wsum, &tot);
    if (tid == 0) s.above_loc = kb > 0 ? tot : 0u;
  }
  __syncthreads();
  if (kb > 0 && !whole && !big) {  // this CTA's members, compacted into its own shared memory
    sweep(lists, G, len, bh, cta, [&](uint64_t c) {
      const bool inb = c != 0ull && c >= lo && hist_digit(comp_key(c), klo, shift) == dstar;
      const unsigned bm = __ballot_sync(kFull, inb);
      if (bm) {
        uint32_t wb = 0;
        if (lane == 0) wb = atomicAdd(&s.nb, __popc(bm));
        wb = __shfl_sync(kFull, wb, 0);
        const uint32_t slot = wb + __popc(bm & lanemask_lt());
        if (inb && slot < static_cast<uint32_t>(kMergeBkt)) s.bkt[slot] = c;  // total <= kMergeBkt
      }
    }, cache, cm);
  }
  cluster.sync();  // members complete; every remote read of hist / tot / slsum done
  MERGE_PHASE(50);
  if (cta == 0) {
    uint64_t T;
    if (kb == 0) {
      T = ~0ull;
    } else if (whole) {
      const uint64_t b_lo = static_cast<uint64_t>(klo + (dstar << shift)) << 32;  // bucket lower bound
      T = b_lo > lo ? b_lo : lo;
    } else if (!big) {
      // pull the other CTAs' members behind rank 0's own (all remote loads in flight)
      uint32_t cnt[CL], start[CL], run = 0;
#pragma unroll
      for (int r = 0; r < CL; ++r) {
        cnt[r] = min(*cluster.map_shared_rank(&s.nb, r), static_cast<uint32_t>(kMergeBkt));
        start[r] = run;
        run += cnt[r];
      }
      __syncthreads();  // every thread read rank 0's own count before s.bkt is rearranged
      // rank 0's members stay in [0, cnt[0]); the others land in [start[r], start[r] + cnt[r])
      for (uint32_t i = cnt[0] + tid; i < run; i += MT) {
        int r = 1;
#pragma unroll
        for (int rr = 2; rr < CL; ++rr) r = i >= start[rr] ? rr : r;
        s.bkt[i] = cluster.map_shared_rank(s.bkt, r)[i - start[r]];
      }
      __syncthreads();
      T = block_rank_select_par<MT>(s.bkt, static_cast<int>(run), static_cast<int>(need), &s.res);
    } else {
      // rare: a bucket larger than shared memory (heavy exact ties) — radix passes over the
      // source lists restricted to bucket d*
      int cs = 64;
      uint64_t cp = 0;
      const int64_t n = static_cast<int64_t>(G) * len;
      auto ld = [&](int64_t i, uint64_t& c) {
        const int g = static_cast<int>(i / len);
        c = lists[g][static_cast<int64_t>(bh) * len + (i - static_cast<int64_t>(g) * len)];
        return c != 0ull && c >= lo && hist_digit(comp_key(c), klo, shift) == dstar;
      };
      radix_select_u64<MT>(ld, n, need, s.hist, s.scr, s.out, cs, cp);
      T = cp << cs;
    }
    if (tid == 0) s.T = T;
  }
  cluster.sync();
  const uint64_t T = *cluster.map_shared_rank(&s.T, 0);
  // this CTA's output base: the selected rows of the lower-ranked CTAs (rows above d* plus
  // their members >= T; the members are still in each CTA's own s.bkt[0, nb))
  if (tid < 32) {
    uint32_t mine = 0;
    if (kb > 0 && lane < cta) {
      const uint32_t nb = min(*cluster.map_shared_rank(&s.nb, lane), static_cast<uint32_t>(kMergeBkt));
      const uint64_t* bk = cluster.map_shared_rank(s.bkt, lane);
      uint32_t m = 0;
      if (!whole && !big)
        for (uint32_t i = 0; i < nb; ++i) m += bk[i] >= T;
      mine = *cluster.map_shared_rank(&s.above_loc, lane) + (whole ? cluster.map_shared_rank(s.hist, lane)[dstar] : m);
    }
    mine = warp_sum(mine);
    if (lane == 0) s.obase = mine;
  }
  __syncthreads();
  MERGE_PHASE(51);

  // ---- 5. emit the selected rows at this CTA's base (order inside the CTA unspecified: one
  // shared-memory reservation per warp ballot), pads, metadata. A bucket too big for shared
  // memory (rare) has no per-CTA member counts: those CTAs count and reserve globally.
  if (big) {
    uint32_t mine = 0;
    sweep(lists, G, len, bh, cta, [&](uint64_t c) { mine += c != 0ull && c >= T; }, cache, cm);
    uint32_t cta_total;
    block_excl(mine, s.wsum, &cta_total);
    if (tid == 0) s.obase = cta_total ? atomicAdd(&p.out_cnt[bh], cta_total) : 0u;
    __syncthreads();
  }
  const uint32_t obase = s.obase;
  int32_t* idx_o = p.idx + static_cast<int64_t>(bh) * p.k;
  float* sc_o = p.scores + static_cast<int64_t>(bh) * p.k;
  sweep(lists, G, len, bh, cta, [&](uint64_t c) {
    const bool sel = kb > 0 && c != 0ull && c >= T;
    const unsigned bm = __ballot_sync(kFull, sel);
    if (bm) {
      uint32_t wb = 0;
      if (lane == 0) wb = atomicAdd(&s.nout, __popc(bm));
      wb = __shfl_sync(kFull, wb, 0);
      const uint32_t o = obase + wb + __popc(bm & lanemask_lt());
      if (sel && o < kb) {
        idx_o[o] = static_cast<int32_t>(comp_gid(c));
        sc_o[o] = key_score(comp_key(c));
      }
    }
  }, cache, cm);
  cluster.sync();  // every CTA's (rare) global reservation is done: rank 0 re-arms the counter
  MERGE_PHASE(52);
  if (cta == 0) {
    for (int i = static_cast<int>(kb) + tid; i < p.k; i += MT) {
      idx_o[i] = -1;
      sc_o[i] = -INFINITY;
    }
    if (tid == 0) {
      p.out_cnt[bh] = 0u;
      p.meta_kb[bh] = static_cast<int32_t>(kb);
      p.meta_max[bh] = kb > 0 ? key_score(comp_key(M)) : -INFINITY;
      p.meta_kth[bh] = T;
      if (p.used_full) p.used_full[bh] = exact ? 0 : 1;
    }
  }
}

cudaError_t launch_shard_merge(const ShardMergeParams& p, int nbh, cudaStream_t s) {
  const int smem = static_cast<int>((sizeof(MergeSmem) + 15) / 16 * 16 + kMergeCache * sizeof(uint64_t));
  const int attr = per_device(reinterpret_cast<const void*>(shard_merge_kernel), 0, [smem] {
    return static_cast<int>(cudaFuncSetAttribute(shard_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  });
  if (attr != cudaSuccess) return static_cast<cudaError_t>(attr);
  shard_merge_kernel<<<dim3(CL, nbh), MT, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace tkv
