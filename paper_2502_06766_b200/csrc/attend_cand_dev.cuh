// attend_cand_dev.cuh — the candidate-mode V gather (filter c >= meta_kth, write idx/scores,
// gather + softmax partials, head finish), shared by attend_cand_kernel (attend.cu) and the
// exactness-fallback chain's gather tail-launched from select.cu.
// Reference: rescore + fetch_values + _joint_attend, attention.py:158-167, 107-122.
#pragma once

#include "attend_dev.cuh"

namespace tkv {
namespace {
// Persistent CTAs walk (head, S chunks of kCandChunk candidates) work items; a candidate is
// selected iff its composite >= meta_kth, which is exactly the top-kb set. Selected rows are
// appended to idx/scores (order unspecified) and, with p.gather, their V rows gathered in the
// same pass. s_pref: [heads + 1] words of dynamic shared memory.
__device__ __forceinline__ void attend_cand_run(const AttendParams& p, AttSmem& sm, uint32_t* s_pref) {
  if (threadIdx.x == 0) tl_start(p.tl, 6);
#ifdef TKV_DIAG
  uint64_t t_ph = p.tl ? ptimer() : 0ull;
#define TKV_ATT_PHASE(e) \
  if (threadIdx.x == 0) tl_phase(p.tl, e, t_ph)
#else
#define TKV_ATT_PHASE(e)
#endif
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int BH = p.bh_count ? p.bh_count : p.B * p.Hq;  // heads [bh_begin, bh_begin + BH)
  auto chunks_of = [&](int lh) -> int {  // kCandQuant-candidate quanta of a head
    int64_t n = p.cand_cnt[p.bh_begin + lh];
    if (n > p.cap) n = p.cap;
    return static_cast<int>((n + kCandQuant - 1) / kCandQuant);
  };
  // Work items: S consecutive quanta (256 candidates) of one head, S = ceil(total quanta /
  // grid), so the items fill the grid about once (the per-item fixed costs — candidate load,
  // compaction, partial write, head ticket — are paid per S quanta); an item's candidates go
  // through the compaction + gather loop in batches of up to kCandChunk. Small selections
  // (cfg2: ~4K candidates per head) thus spread over ~all CTAs instead of one item per 1024
  // candidates. Every head gets >= 1 item so its output is always finalised. Exclusive prefix
  // of items per head (block-wide).
  const int per = (BH + NT - 1) / NT;
  uint32_t csum = 0;
  for (int j = 0; j < per; ++j) {
    const int lh = tid * per + j;
    csum += lh < BH ? chunks_of(lh) : 0;
  }
  csum = warp_sum(csum);
  if (lane == 0) sm.wcnt[warp] = csum;
  __syncthreads();
  uint32_t total_chunks = 0;
  for (int w = 0; w < NW; ++w) total_chunks += sm.wcnt[w];
  const uint32_t slots = gridDim.x * static_cast<uint32_t>(p.items_mult > 0 ? p.items_mult : 1);
  const int S = total_chunks > slots ? static_cast<int>((total_chunks + slots - 1) / slots) : 1;
  __syncthreads();
  auto nslots_of = [&](int lh) -> int {
    const int c = chunks_of(lh);
    return c > 0 ? (c + S - 1) / S : 1;
  };
  {
    uint32_t sum = 0;
    for (int j = 0; j < per; ++j) {
      const int lh = tid * per + j;
      sum += lh < BH ? nslots_of(lh) : 0;
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) sm.wcnt[warp] = incl;
    __syncthreads();
    uint32_t woff = 0;
    for (int w = 0; w < warp; ++w) woff += sm.wcnt[w];
    uint32_t run = woff + incl - sum;
    for (int j = 0; j < per; ++j) {
      const int lh = tid * per + j;
      if (lh < BH) {
        s_pref[lh] = run;
        run += nslots_of(lh);
      }
    }
    if (tid == NT - 1) s_pref[BH] = run;
    __syncthreads();
  }
  const uint32_t total = s_pref[BH];
  const float zs = p.scale * kLog2e;
  TKV_ATT_PHASE(60);
  for (uint32_t item = blockIdx.x; item < total; item += gridDim.x) {
    int lo = 0, hi = BH;  // largest local head with s_pref[lh] <= item
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_pref[mid] <= item) lo = mid; else hi = mid;
    }
    const int bh = p.bh_begin + lo;
    const int slot = static_cast<int>(item - s_pref[lo]);
    const int nslots = static_cast<int>(s_pref[lo + 1] - s_pref[lo]);
    int64_t n = p.cand_cnt[bh];
    if (n > p.cap) n = p.cap;
    const int kb = p.meta_kb[bh];
    const uint64_t T = p.meta_kth[bh];
    const float zref = kb > 0 ? p.meta_max[bh] * zs : 0.f;
    int32_t* idx_o = p.idx_out + static_cast<int64_t>(bh) * p.k;
    float* sc_o = p.scores_out + static_cast<int64_t>(bh) * p.k;
    if (slot == 0) {  // pads for k > kb (reference clamps k to N, attention.py:147-149)
      for (int i = kb + tid; i < p.k; i += NT) {
        idx_o[i] = -1;
        sc_o[i] = -INFINITY;
        if (p.packed_out) p.packed_out[static_cast<int64_t>(bh) * p.k + i] = 0ull;
      }
    }
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    float lw = 0.f;
    int64_t c_end = static_cast<int64_t>(slot + 1) * S * kCandQuant;
    c_end = c_end < n ? c_end : n;
    for (int64_t c0 = static_cast<int64_t>(slot) * S * kCandQuant; c0 < c_end; c0 += kCandChunk) {
      const uint64_t* src = p.cand + static_cast<int64_t>(bh) * p.cap + c0;
      int64_t cnt = c_end - c0;
      cnt = cnt > kCandChunk ? kCandChunk : cnt;
      constexpr int PER = kCandChunk / NT;
      uint64_t cv[PER];
      bool sel[PER];
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int i = u * NT + tid;
        cv[u] = (i < cnt && kb > 0) ? src[i] : 0ull;
        sel[u] = cv[u] != 0ull && cv[u] >= T;
      }
      TKV_ATT_PHASE(61);
      // block-ordered compaction of the selected candidates
      uint32_t mine = 0;
#pragma unroll
      for (int u = 0; u < PER; ++u) mine += sel[u] ? 1u : 0u;
      uint32_t incl = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += t;
      }
      __syncthreads();  // the previous chunk's gather no longer reads sm.row / sm.w
      if (lane == 31) sm.wcnt[warp] = incl;
      __syncthreads();
      uint32_t woff = 0, m = 0;
      for (int w = 0; w < NW; ++w) {
        woff += w < warp ? sm.wcnt[w] : 0u;
        m += sm.wcnt[w];
      }
      // output reservation: thread 0 keeps the result in a register and publishes it after the
      // gather (storing it to shared memory here would stall the block's barrier on the atomic's
      // L2 round trip)
      uint32_t rbase = 0u;
      if (tid == 0 && m) rbase = atomicAdd(&p.out_cnt[bh], m);
      uint32_t pos = woff + incl - mine;
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        if (sel[u]) {
          const uint64_t c = cv[u];
          const int64_t local = static_cast<int64_t>(comp_gid(c)) - p.row_offset;
          mark_pinned(p, bh, local);
          const float sc = key_score(comp_key(c));
          sm.row[pos] = static_cast<int32_t>(local);
          sm.w[pos] = exp2f(fmaf(sc, zs, -zref));
          sm.sc[pos] = sc;
          ++pos;
        }
      }
      __syncthreads();
      TKV_ATT_PHASE(62);
      if (p.gather) gather_acc(p, bh, static_cast<int>(m), sm, acc, lw);
      TKV_ATT_PHASE(63);
      // the reservation atomic completed during the gather
      if (tid == 0) sm.base = rbase;
      __syncthreads();
      // ids / raw scores in list order from shared memory: consecutive threads, consecutive
      // slots (coalesced — the ids may live in pinned host memory, written over PCIe)
      const uint32_t obase = sm.base;
      const uint64_t t2 = p.narrow_out ? p.meta_t2[bh] : ~0ull;
      for (uint32_t i0 = 0; i0 < m; i0 += NT) {  // warp-uniform trip count (narrow-list ballots)
        const uint32_t i = i0 + tid;
        const uint32_t o = obase + i;
        bool nar = false;
        uint64_t c = 0ull;
        if (i < m && o < static_cast<uint32_t>(p.k)) {
          const uint32_t gid = static_cast<uint32_t>(static_cast<int64_t>(sm.row[i]) + p.row_offset);
          idx_o[o] = static_cast<int32_t>(gid);
          sc_o[o] = sm.sc[i];
          c = make_comp(score_key(sm.sc[i]), gid);
          if (p.packed_out) p.packed_out[static_cast<int64_t>(bh) * p.k + o] = c;
          nar = p.narrow_out && c >= t2;
        }
        if (p.narrow_out) {  // sharded: append to this rank's narrow list, one atomic per warp
          const unsigned bm = __ballot_sync(kFull, nar);
          if (bm) {
            uint32_t wb = 0;
            if (lane == 0) wb = atomicAdd(&p.narrow_cnt[bh], __popc(bm));
            wb = __shfl_sync(kFull, wb, 0);
            const uint32_t slot = wb + __popc(bm & lanemask_lt());
            if (nar && slot < static_cast<uint32_t>(p.narrow_len))
              p.narrow_out[static_cast<int64_t>(bh) * p.narrow_len + slot] = c;
          }
        }
      }
    }
    TKV_ATT_PHASE(64);
    if (p.gather) {
      partial_write(p, bh, slot, sm, acc, lw);
      TKV_ATT_PHASE(65);
      ticket_finish(p, bh, nslots, sm);
    }
    __syncthreads();
    TKV_ATT_PHASE(66);
  }
  if (threadIdx.x == 0) tl_end(p.tl, 6);
}
}  // namespace
}  // namespace tkv
