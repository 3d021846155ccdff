// scan_tc.cu — K1 on the Blackwell tensor-core pipeline: TMA → shared memory → tcgen05.mma →
// TMEM → epilogue warps. Same contract as scan_kernel (scan.cu): every score of a live row
// whose key >= t_h is appended as a composite (key, ~row) to the head's candidate list, and
// the candidates' key histogram is accumulated for select.cu. Reference computation:
// ip_scores_all (ann_kernels.py:40-47) over every cache row of a head.
//
// One CTA per SM, persistent over an even split of the 256-row units of all (b, kv head)
// segments; 192 threads in fixed roles, hand-offs through mbarriers:
//   warp 0     TMA producer: one unit = 256 rows × 128 dims bf16 = two 2-D boxes of
//              [256 rows × 64 elements] (128-byte swizzle) = 64 KB, into a 2–3 deep ring.
//   warp 1     TMEM owner + MMA issuer: at a segment change the warp writes the GQA group's
//              query rows (B operand, N = 8, rows >= G zero) into a rotating q slot; one lane
//              issues 2 sub-tiles × 8 K-steps of tcgen05.mma (M = 128, N = 8, K = 16, bf16 in,
//              f32 accumulate in TMEM), then commits the stage to the producer and the
//              accumulator to the epilogue.
//   warps 2–5  epilogue: warp w reads TMEM lanes [32·(w%4), +32) — one cache row per thread,
//              its G scores for both sub-tiles (one tcgen05.ld .x16) — tests them against the
//              heads' thresholds and appends passing composites to a warp-private staging
//              buffer (counts in registers, no shared atomics), flushed by the warp itself.
// Measured design constraints (tools/micro): an mbarrier wait+arrive hand-off costs ~170
// cycles and an M=128 N<=64 MMA ~45 cycles of issue, so the unit is 256 rows (64 KB) to keep
// the per-byte pipeline overhead well under the HBM time of the unit (~2800 cycles per SM).
// The SM's registers and warp slots stay nearly free: HBM is saturated by one 6-warp CTA per
// SM instead of the two register-staged CTAs the HMMA scan (scan.cu) needs.
#include <cudaTypedefs.h>
#include <stdlib.h>

#include "scan_tc_dev.cuh"

namespace tkv {
using namespace tc;
namespace {

#ifndef TKV_TC_STEAL
#define TKV_TC_STEAL 1  // dynamic tail: CTAs claim the last eighth of every share from a pool
#endif
#ifndef TKV_STEAL_CHUNK
#define TKV_STEAL_CHUNK 2
#endif
constexpr int kStealChunk = TKV_STEAL_CHUNK;  // units per pool claim (~3 us of one SM's HBM share)
constexpr int kStealMinShare = 64;  // units per CTA below which the split stays static: a claimed
                                    // chunk's segment switch (q reload, epilogue flush) and the
                                    // claim round trip cost more than the balance gains (cfg2:
                                    // 27 units per CTA, 75.9 -> 79.4 us with a pool)
constexpr int kClaimAhead = 3;  // static units left when the first pool claim is issued
constexpr int kStealRing = 64;  // published unit slots (>= stages + kTcAcc + 2)
static_assert(kStealRing >= kTcMaxStages + kTcAcc + 2, "unit ring too small");

#if !TKV_TC_STEAL
// Walks a CTA's units [u0, u1) of the B·Hkv segments (ups units each) without per-unit
// divisions, skipping units at or beyond the segment's context length. Every role runs the
// same walk, so they agree on the sequence of live units.
struct UnitWalk {
  int64_t u, u1, ups, seg, j;
  int64_t nctx;
  // the live unit last returned
  int64_t cur_seg = -1, cur_row0 = 0, cur_nctx = 0;
  int cur_b = 0, cur_kvh = 0;
  int b = 0, kvh = 0;

  __device__ __forceinline__ void load(const ScanParams& p) {
    b = static_cast<int>(seg / p.Hkv);
    kvh = static_cast<int>(seg - static_cast<int64_t>(b) * p.Hkv);
    nctx = p.n_ctx[b];
  }
  __device__ __forceinline__ void init(const ScanParams& p, int64_t u0, int64_t u1_, int64_t ups_) {
    u = u0;
    u1 = u1_;
    ups = ups_;
    seg = u0 / ups;
    j = u0 - seg * ups;
    if (u < u1) load(p);
  }
  // advance to the next live unit; new_seg = its segment differs from the previous live unit's
  __device__ __forceinline__ bool next(const ScanParams& p, bool& new_seg) {
    while (u < u1) {
      if (j * kTcUnit < nctx) {
        new_seg = seg != cur_seg;
        cur_seg = seg;
        cur_row0 = j * kTcUnit;
        cur_nctx = nctx;
        cur_b = b;
        cur_kvh = kvh;
        ++u;
        if (++j == ups) {
          ++seg;
          j = 0;
          if (u < u1) load(p);
        }
        return true;
      }
      u += ups - j;  // rest of this segment is beyond its context
      ++seg;
      j = 0;
      if (u < u1) load(p);
    }
    return false;
  }
};
#endif

// (diagnostic builds cap the registers at the release count: the timers would otherwise push
// the kernel past the register budget that lets threshold / k-th CTAs share its SMs)
#ifdef TKV_DIAG
__global__ void __maxnreg__(120) scan_tc_kernel(
#else
__global__ void __launch_bounds__(kTcScanThreads, 1) scan_tc_kernel(
#endif
    const __grid_constant__ CUtensorMap kmap,
                                                                ScanParams p, int n_stages, int flush_every,
                                                                int mode) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t s_bar[kTcBarWords];
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  pdl_trigger();  // the k-th kernel may launch now; it waits for this grid to complete
#ifdef TKV_DIAG
  const uint64_t t_cta = p.tl ? ptimer() : 0ull;
#endif
  if (tid == 0) {
    tl_start(p.tl, 3);
    tl_start(p.tl, 40);  // first / last CTA start
    tl_end(p.tl, 40);
#ifdef TKV_DIAG
    // SMs whose scan CTA started > 6 us after the step's first kernel
    if (p.tl && gtimer() > p.tl[0] + 6000ull) tl_smid(p.tl, 243);
    tl_smid(p.tl, 246);  // SMs hosting a scan CTA
#endif
  }
  TcPipe t = tc_setup(smem_raw, s_bar, &s_tmem, p.G, flush_every, n_stages, &kmap, tid == 0, warp == 1,
                      kTcScanGroups);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  t.tmem = s_tmem;

  const int64_t ups = (p.max_ctx + kTcUnit - 1) / kTcUnit;
  const int64_t total = (p.seg_count ? p.seg_count : static_cast<int64_t>(p.B) * p.Hkv) * ups;
  const int64_t ubase = p.seg_begin * ups;  // units of the segment range [seg_begin, +seg_count)
#if TKV_TC_STEAL
  // Units of this CTA: the front of its even share [r0, r1) statically, then chunks of the pool
  // formed by every CTA's last tc·kStealChunk units, claimed with a global atomic — so SMs that
  // started late or stream slower hand their tail to the others (the CTAs' end times spread over
  // 5 µs at cfg2 and 12 µs at cfg3 with a static split). The producer decides the sequence and
  // publishes unit i in s_unit[i % 64] before the unit's TMA; the MMA warp and the epilogue read
  // it after their barrier waits for unit i (the producer runs at most stages + kTcAcc units
  // ahead of the epilogue, so 64 slots never wrap onto an unread one). -1 ends the sequence.
  __shared__ int32_t s_unit[kStealRing];  // unit indices (< 2^23: rows < 2^31); static smem stays < 1 KB
  const int64_t r0 = ubase + total * blockIdx.x / gridDim.x, r1 = ubase + total * (blockIdx.x + 1) / gridDim.x;
  const int64_t per_cta = total / gridDim.x;
  const int64_t tcn = per_cta / (8 * kStealChunk);  // pool chunks per CTA (uniform)
  const int64_t n_pool = p.steal && per_cta >= kStealMinShare ? tcn * gridDim.x : 0;
  const int64_t s_end = n_pool ? r1 - tcn * kStealChunk : r1;

  if (warp == 0) {  // TMA producer
    uint32_t i = 0;
    int64_t pseg = -1, pnctx = 0;
    auto push = [&](int64_t u) {
      const int64_t seg = u / ups, j = u - seg * ups;
      if (seg != pseg) {
        pseg = seg;
        pnctx = p.n_ctx[static_cast<int>(seg / p.Hkv)];
      }
      if (j * kTcUnit >= pnctx) return;  // beyond the segment's context
      if (lane == 0) s_unit[i % kStealRing] = static_cast<int32_t>(u);
      tc_produce(t, i, &kmap, static_cast<int>(seg * p.cache_rows + j * kTcUnit), lane, mode);
      ++i;
    };
    // the first pool claim is issued kClaimAhead static units before the end of the static part
    // (its round trip overlaps them; the result is read only afterwards)
    uint32_t g_first = 0;
    for (int64_t u = r0; u < s_end; ++u) {
      if (n_pool && lane == 0 && u == s_end - kClaimAhead) g_first = atomicAdd(&p.steal[0], 1u);
      push(u);
    }
    if (n_pool) {
      auto claim = [&]() -> int64_t {
        uint32_t g = 0;
        if (lane == 0) g = atomicAdd(&p.steal[0], 1u);
        return static_cast<int64_t>(__shfl_sync(kFull, g, 0));
      };
      if (lane == 0 && s_end - r0 < kClaimAhead) g_first = atomicAdd(&p.steal[0], 1u);
      int64_t g = static_cast<int64_t>(__shfl_sync(kFull, g_first, 0));
      while (g < n_pool) {
        const int64_t gn = claim();  // the next claim's round trip overlaps this chunk
        const int64_t v = g / tcn, jj = g - v * tcn;
        const int64_t e_v = ubase + total * (v + 1) / gridDim.x;
        const int64_t c0 = e_v - (tcn - jj) * kStealChunk;
        for (int64_t u = c0; u < c0 + kStealChunk; ++u) push(u);
        g = gn;
      }
      // the last CTA out of the pool resets the counters for the next launch
      if (lane == 0) {
        __threadfence();
        if (atomicAdd(&p.steal[1], 1u) == gridDim.x - 1) {
          p.steal[0] = 0u;
          p.steal[1] = 0u;
        }
      }
    }
    // end marker: the MMA warp wakes on a plain arrive on the next stage and tells the epilogue
    if (lane == 0) {
      s_unit[i % kStealRing] = -1;
      s_unit[(i + 1) % kStealRing] = -1;
    }
    const int st = static_cast<int>(i % t.n_stages);
    mbar_wait(t.empty(st), ((i / t.n_stages) & 1u) ^ 1u);
    if (lane == 0) mbar_arrive(t.full(st));
    __syncwarp();
  } else if (warp == 1) {  // MMA issuer
    QRing qr;
    int64_t cur_seg = -1;
#ifdef TKV_DIAG
    uint64_t d_wait = 0, n_units = 0;  // diagnostics (tl != nullptr): MMA warp's wait for TMA
#endif
    for (uint32_t i = 0;; ++i) {
      tc_mma_acquire(t, i);
#ifdef TKV_DIAG
      const uint64_t t_w = p.tl ? ptimer() : 0ull;
#endif
      mbar_wait(t.full(static_cast<int>(i % t.n_stages)), (i / t.n_stages) & 1u);
#ifdef TKV_DIAG
      if (p.tl) {
        d_wait += ptimer() - t_w;
        ++n_units;
      }
#endif
      const int64_t u = s_unit[i % kStealRing];
      if (u < 0) {  // end: release both epilogue groups (their accumulator slots drained first)
        tc_mma_acquire(t, i + 1);
        if (lane == 0) {
          mbar_arrive(t.tfull(static_cast<int>(i % kTcAcc)));
          mbar_arrive(t.tfull(static_cast<int>((i + 1) % kTcAcc)));
        }
        __syncwarp();
        break;
      }
      const int64_t seg = u / ups;
      if (seg != cur_seg) {
        cur_seg = seg;
        const int b = static_cast<int>(seg / p.Hkv), kvh = static_cast<int>(seg - static_cast<int64_t>(b) * p.Hkv);
        tc_next_q(t, qr, p.q + (static_cast<int64_t>(b) * p.Hq + kvh * p.G) * kD, p.G, lane);
      }
      tc_mma_issue(t, i, qr.slot, lane, mode);
    }
#ifdef TKV_DIAG
    if (p.tl && lane == 0 && n_units) {
      atomicAdd(reinterpret_cast<unsigned long long*>(p.tl + 88), static_cast<unsigned long long>(d_wait));
      atomicAdd(reinterpret_cast<unsigned long long*>(p.tl + 89), static_cast<unsigned long long>(n_units));
    }
#endif
  } else {  // epilogue: two groups of four warps take alternate units
    pdl_wait();  // thresholds, zeroed counters and histograms of threshold_kernel (the TMA and
                 // MMA warps read only q and K and start streaming before it completes)
    if (lane == 0) tl_start(p.tl, 4);
    const int ew = warp - 2;
    const uint32_t group = static_cast<uint32_t>(ew / kTcEpiWarps);
    const int quarter = warp & 3;  // TMEM lanes this warp may access: [32·quarter, +32)
    uint64_t* wbuf = t.s_buf + static_cast<int64_t>(ew) * p.G * t.cap;
    uint32_t thr[8], shift[8], cnt[8];
#pragma unroll
    for (int n = 0; n < 8; ++n) cnt[n] = thr[n] = shift[n] = 0u;
    int since = 0;
    int64_t bh0 = -1, cur_seg = -1, cur_nctx = 0;
#ifdef TKV_DIAG
    uint64_t d_wait = 0, d_work = 0, d_flush = 0, n_units = 0, n_flush = 0;  // diagnostics
#endif
    for (uint32_t i = group;; i += kTcScanGroups) {
#ifdef TKV_DIAG
      uint64_t t_u = p.tl ? ptimer() : 0ull;
#endif
      mbar_wait(t.tfull(static_cast<int>(i % kTcAcc)), (i / kTcAcc) & 1u);
#ifdef TKV_DIAG
      if (p.tl) {  // diagnostics: the epilogue's wait for the unit's scores
        const uint64_t t1 = ptimer();
        d_wait += t1 - t_u;
        t_u = t1;
      }
#endif
      const int64_t u = s_unit[i % kStealRing];
      if (u < 0) break;
      const int64_t seg = u / ups;
      if (seg != cur_seg) {
        if (bh0 >= 0) tc_warp_flush(p.cand, p.cap, p.hs.cand_cnt, p.hs.hist, p.G, bh0, wbuf, t.cap, cnt, thr, shift, lane);
        since = 0;
        cur_seg = seg;
        const int b = static_cast<int>(seg / p.Hkv), kvh = static_cast<int>(seg - static_cast<int64_t>(b) * p.Hkv);
        cur_nctx = p.n_ctx[b];
        bh0 = static_cast<int64_t>(b) * p.Hq + kvh * p.G;
#pragma unroll
        for (int n = 0; n < 8; ++n) {
          thr[n] = n < p.G ? p.hs.thr[bh0 + n] : 0xFFFFFFFFu;
          shift[n] = n < p.G ? p.hs.hshift[bh0 + n] : 0u;
        }
      }
      uint32_t v[16];
      tc_epi_load(t, i, quarter, lane, v, mode);
      tc_epi_emit(v, (u - seg * ups) * kTcUnit, cur_nctx, quarter, lane, p.G, p.row_offset, thr, wbuf, t.cap, cnt,
                  !(mode & 3) /* diagnostics never emit */);
#ifdef TKV_DIAG
      if (p.tl) {
        d_work += ptimer() - t_u;
        ++n_units;
      }
      const uint64_t t_f = p.tl ? ptimer() : 0ull;
#endif
      if (++since == flush_every) {
        tc_warp_flush(p.cand, p.cap, p.hs.cand_cnt, p.hs.hist, p.G, bh0, wbuf, t.cap, cnt, thr, shift, lane);
#ifdef TKV_DIAG
        if (p.tl) {
          d_flush += ptimer() - t_f;
          ++n_flush;
        }
#endif
        since = 0;
      }
    }
    if (bh0 >= 0) tc_warp_flush(p.cand, p.cap, p.hs.cand_cnt, p.hs.hist, p.G, bh0, wbuf, t.cap, cnt, thr, shift, lane);
    if (lane == 0) tl_end(p.tl, 4);
#ifdef TKV_DIAG
    if (p.tl && lane == 0) {  // slots 42, 43, 29: (sum ns, count) per warp, one atomic pair each
      unsigned long long* tl = reinterpret_cast<unsigned long long*>(p.tl);
      atomicAdd(tl + 84, static_cast<unsigned long long>(d_wait));
      atomicAdd(tl + 85, static_cast<unsigned long long>(n_units));
      atomicAdd(tl + 86, static_cast<unsigned long long>(d_work));
      atomicAdd(tl + 87, static_cast<unsigned long long>(n_units));
      atomicAdd(tl + 58, static_cast<unsigned long long>(d_flush));
      atomicAdd(tl + 59, static_cast<unsigned long long>(n_flush));
    }
#endif
  }
#else
  UnitWalk w;
  w.init(p, ubase + total * blockIdx.x / gridDim.x, ubase + total * (blockIdx.x + 1) / gridDim.x, ups);
  bool new_seg = false;

  if (warp == 0) {  // TMA producer
    for (uint32_t i = 0; w.next(p, new_seg); ++i)
      tc_produce(t, i, &kmap, static_cast<int>(w.cur_seg * p.cache_rows + w.cur_row0), lane, mode);
  } else if (warp == 1) {  // MMA issuer
    QRing qr;
#ifdef TKV_DIAG
    uint64_t d_wait = 0, n_units = 0;  // diagnostics (tl != nullptr): MMA warp's wait for TMA
#endif
    for (uint32_t i = 0; w.next(p, new_seg); ++i) {
      tc_mma_acquire(t, i);
#ifdef TKV_DIAG
      if (p.tl) {
        const uint64_t t_w = ptimer();
        mbar_wait(t.full(static_cast<int>(i % t.n_stages)), (i / t.n_stages) & 1u);
        d_wait += ptimer() - t_w;
        ++n_units;
      }
#endif
      if (new_seg) tc_next_q(t, qr, p.q + (static_cast<int64_t>(w.cur_b) * p.Hq + w.cur_kvh * p.G) * kD, p.G, lane);
      tc_mma_issue(t, i, qr.slot, lane, mode);
    }
#ifdef TKV_DIAG
    if (p.tl && lane == 0 && n_units) {
      atomicAdd(reinterpret_cast<unsigned long long*>(p.tl + 88), static_cast<unsigned long long>(d_wait));
      atomicAdd(reinterpret_cast<unsigned long long*>(p.tl + 89), static_cast<unsigned long long>(n_units));
    }
#endif
  } else {  // epilogue: two groups of four warps take alternate units
    pdl_wait();  // thresholds, zeroed counters and histograms of threshold_kernel (the TMA and
                 // MMA warps read only q and K and start streaming before it completes)
    if (lane == 0) tl_start(p.tl, 4);
    const int ew = warp - 2;
    const uint32_t group = static_cast<uint32_t>(ew / kTcEpiWarps);
    const int quarter = warp & 3;  // TMEM lanes this warp may access: [32·quarter, +32)
    uint64_t* wbuf = t.s_buf + static_cast<int64_t>(ew) * p.G * t.cap;
    uint32_t thr[8], shift[8], cnt[8];
#pragma unroll
    for (int n = 0; n < 8; ++n) cnt[n] = thr[n] = shift[n] = 0u;
    int since = 0;
    int64_t bh0 = -1;
#ifdef TKV_DIAG
    uint64_t d_wait = 0, d_work = 0, d_flush = 0, n_units = 0, n_flush = 0;  // diagnostics
#endif
    for (uint32_t i = 0; w.next(p, new_seg); ++i) {
      if (new_seg) {
        if (bh0 >= 0) tc_warp_flush(p.cand, p.cap, p.hs.cand_cnt, p.hs.hist, p.G, bh0, wbuf, t.cap, cnt, thr, shift, lane);
        since = 0;
        bh0 = static_cast<int64_t>(w.cur_b) * p.Hq + w.cur_kvh * p.G;
#pragma unroll
        for (int n = 0; n < 8; ++n) {
          thr[n] = n < p.G ? p.hs.thr[bh0 + n] : 0xFFFFFFFFu;
          shift[n] = n < p.G ? p.hs.hshift[bh0 + n] : 0u;
        }
      }
      if (i % kTcScanGroups != group) continue;
      uint32_t v[16];
#ifdef TKV_DIAG
      uint64_t t_u = p.tl ? ptimer() : 0ull;
      if (p.tl) {  // diagnostics: the epilogue's wait for the unit's scores
        mbar_wait(t.tfull(static_cast<int>(i % kTcAcc)), (i / kTcAcc) & 1u);
        const uint64_t t1 = ptimer();
        d_wait += t1 - t_u;
        t_u = t1;
      }
#endif
      tc_epi_load(t, i, quarter, lane, v, mode);
      tc_epi_emit(v, w.cur_row0, w.cur_nctx, quarter, lane, p.G, p.row_offset, thr, wbuf, t.cap, cnt,
                  !(mode & 3) /* diagnostics never emit */);
#ifdef TKV_DIAG
      if (p.tl) {
        d_work += ptimer() - t_u;
        ++n_units;
      }
      const uint64_t t_f = p.tl ? ptimer() : 0ull;
#endif
      if (++since == flush_every) {
        tc_warp_flush(p.cand, p.cap, p.hs.cand_cnt, p.hs.hist, p.G, bh0, wbuf, t.cap, cnt, thr, shift, lane);
#ifdef TKV_DIAG
        if (p.tl) {
          d_flush += ptimer() - t_f;
          ++n_flush;
        }
#endif
        since = 0;
      }
    }
    if (bh0 >= 0) tc_warp_flush(p.cand, p.cap, p.hs.cand_cnt, p.hs.hist, p.G, bh0, wbuf, t.cap, cnt, thr, shift, lane);
    if (lane == 0) tl_end(p.tl, 4);
#ifdef TKV_DIAG
    if (p.tl && lane == 0) {  // slots 42, 43, 29: (sum ns, count) per warp, one atomic pair each
      unsigned long long* tl = reinterpret_cast<unsigned long long*>(p.tl);
      atomicAdd(tl + 84, static_cast<unsigned long long>(d_wait));
      atomicAdd(tl + 85, static_cast<unsigned long long>(n_units));
      atomicAdd(tl + 86, static_cast<unsigned long long>(d_work));
      atomicAdd(tl + 87, static_cast<unsigned long long>(n_units));
      atomicAdd(tl + 58, static_cast<unsigned long long>(d_flush));
      atomicAdd(tl + 59, static_cast<unsigned long long>(n_flush));
    }
#endif
  }

#endif  // TKV_TC_STEAL

  tc_fence_before();
  __syncthreads();
  tc_teardown(t.tmem, warp == 1);
  if (tid == 0) {
    tl_end(p.tl, 3);
    tl_start(p.tl, 41);  // first / last CTA end
    tl_end(p.tl, 41);
  }
#ifdef TKV_DIAG
  if (tid == 0) {
    uint64_t t0 = t_cta;
    tl_phase(p.tl, 46, t0);  // CTA lifetime (mean)
  }
#endif
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

}  // namespace

bool tc::make_kmap(const __nv_bfloat16* kc, int64_t rows, CUtensorMap* map) {
  if (!encode_fn()) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(kD), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(kD) * 2};
  const cuuint32_t box[2] = {64, kTcUnit};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16*>(kc), dims,
                                 strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// The K cache [B, Hkv, cache_rows, 128] bf16 as a 2-D tensor of B·Hkv·cache_rows rows.
bool scan_tc_supported(const ScanParams& p) {
  const int64_t rows = static_cast<int64_t>(p.B) * p.Hkv * p.cache_rows;
  return encode_fn() != nullptr && (reinterpret_cast<uintptr_t>(p.kc) & 15u) == 0 && rows < (int64_t(1) << 31) &&
         p.G <= 8;
}

cudaError_t launch_scan_tc(const ScanParams& p, cudaStream_t s) {
  const int64_t ups = (p.max_ctx + kTcUnit - 1) / kTcUnit;
  const int64_t total = (p.seg_count ? p.seg_count : static_cast<int64_t>(p.B) * p.Hkv) * ups;
  if (total == 0) return cudaSuccess;
  CUtensorMap map;
  if (!tc::make_kmap(p.kc, static_cast<int64_t>(p.B) * p.Hkv * p.cache_rows, &map)) return cudaErrorInvalidValue;
  // TKV_DIAG builds only (release: 0): bit 0 = no MMA, bit 1 = no emission, bit 2 = no TMA —
  // each gives wrong results by design (pipeline cost breakdown)
  const int mode = diag_env("TKV_TC_MODE", 0);
  const int stages_env = diag_env("TKV_TC_STAGES", 0);  // experiments: force the ring depth (2 or 3)
  const int flush_env = diag_env("TKV_TC_FLUSH", 0);    // experiments: cap the units between flushes
  TcShape sh = tc_shape(p.G, kTcScanGroups);
  if (stages_env >= 2 && stages_env <= kTcMaxStages && stages_env != sh.stages) {
    sh.stages = stages_env;
    const int free_b = kTcSmemLimit - 1024 - kTcQSlots * kTcQBytes - sh.stages * kTcUnitBytes;
    sh.flush = free_b / tc_stage_bytes(p.G, 1, kTcScanGroups);
    if (sh.flush > kTcMaxFlush) sh.flush = kTcMaxFlush;
    if (sh.flush < 1) return cudaErrorInvalidValue;
  }
  if (flush_env > 0) {  // experiments: set the units between a warp's flushes (bounded by smem)
    const int free_b = kTcSmemLimit - 1024 - kTcQSlots * kTcQBytes - sh.stages * kTcUnitBytes;
    const int fit = free_b / tc_stage_bytes(p.G, 1, kTcScanGroups);
    sh.flush = flush_env < fit ? flush_env : fit;
  }
  const size_t smem = tc_smem_bytes(p.G, sh, kTcScanGroups);
  const int attr = per_device(reinterpret_cast<const void*>(scan_tc_kernel), 0, [] {
    cudaError_t e = cudaFuncSetAttribute(scan_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmemLimit);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(scan_tc_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared);
    return static_cast<int>(e);
  });
  if (attr != cudaSuccess) return static_cast<cudaError_t>(attr);
  int grid = device_sm_count();
  if (total < grid) grid = static_cast<int>(total);
  return launch_pdl(scan_tc_kernel, dim3(grid), dim3(kTcScanThreads), smem, s, p.pdl != 0, map, p, sh.stages,
                    sh.flush, mode);
}

}  // namespace tkv
