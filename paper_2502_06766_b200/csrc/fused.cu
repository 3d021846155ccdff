// fused.cu — the whole layer step in ONE persistent kernel (default single-GPU path).
//
// The multi-kernel pipeline (sample → threshold → scan → kth → attend) leaves the HBM idle
// while the latency-bound stages run and pays a launch floor per kernel. Here persistent CTAs
// (256 threads, 2 per SM) claim work items IN ORDER from a global counter:
//
//   SAMPLE(g, part)   16 per (b, kv head) group g   — scores 256 sampled rows  (scan.cu)
//   THRESH(h)         one per (b, q head) h          — candidate threshold      (scan.cu)
//   SCAN(g, tile)     T per group                     — HMMA key scan + emit     (scan.cu)
//   KTH(h, slice)     4 per head                      — exact k-th composite     (select.cu)
//   ATT(h, a)         KA per head                     — filter c >= T, V gather, softmax
//
// ordered so that the selection and the V gather of group g-1 are claimed while the tiles of
// group g are being scanned:   SAMPLE(g) THRESH(g) for every g | for g: SCAN(g)[0,T/2) KTH(g-1)
// SCAN(g)[T/2,T) ATT(g-1) | KTH(last) ATT(last).
// An item only ever waits (spin on a flag) for items with a SMALLER index; the smallest
// unfinished item therefore always has its inputs ready and is being processed (a CTA holds a
// prefetched claim only while it works on a smaller one), so the schedule cannot deadlock even
// if not all CTAs are resident.
//
// Exactness fallback: a head whose sampled threshold passed fewer than k rows is flagged by
// its KTH item, which appends a job (FB_SCAN tiles of the group for that head with threshold 0,
// FB_KTH, FB_ATT) behind the static items; those are claimed through a second counter with a
// compare-and-swap, so no claimed index is ever dropped.
//
// Data produced inside the kernel (samples, candidates, histograms, thresholds, partials) is
// read with ld.global.cg (L2) after the flag's acquire — L1 is not coherent across SMs.
#include <cstdio>

#include "attend_dev.cuh"
#include "scan_tc_dev.cuh"

namespace tkv {

namespace {
constexpr int FT = 256;
constexpr int FW = FT / 32;
static_assert(FT == kAttendThreads && FT == kScanWarps * 32, "one CTA shape for every item type");
constexpr int kFStage = kScanRows * 4;  // staged candidates per head: up to 4 iterations/tile
constexpr int kFBkt = 2048;             // bucket refinement held in shared memory
constexpr uint32_t kNoItem = 0xffffffffu;

// diagnostics: time an item's dependency wait ended (set by KTH / ATT items when tracing)
__shared__ uint64_t s_item_ready;

__device__ __forceinline__ void stamp_ready(const FusedParams& p, int tid) {
  if (p.trace && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(s_item_ready));
}

enum ItemType : int { kItSample, kItThresh, kItScan, kItKth, kItAtt, kItFbScan, kItFbKth, kItFbAtt, kItNop };

struct Item {
  int type;
  int a;  // group or head
  int b;  // part / tile / slice / attend index
};

struct Ctl {
  uint32_t* w;
  int NG, NH;
  __device__ uint32_t* item() const { return w + 0; }
  __device__ uint32_t* dyn() const { return w + 1; }
  __device__ uint32_t* nfb() const { return w + 2; }
  __device__ uint32_t* fb_alloc() const { return w + 3; }
  __device__ uint32_t* exited() const { return w + 4; }
  __device__ uint32_t* samp_done(int g) const { return w + 8 + g; }
  __device__ uint32_t* scan_done(int g) const { return w + 8 + NG + g; }
  __device__ uint32_t* thr_ready(int h) const { return w + 8 + 2 * NG + h; }
  __device__ uint32_t* kth_state(int h) const { return w + 8 + 2 * NG + NH + h; }
  __device__ uint32_t* fb_scan_done(int h) const { return w + 8 + 2 * NG + 2 * NH + h; }
  __device__ uint32_t* att_ticket(int h) const { return w + 8 + 2 * NG + 3 * NH + h; }
  __device__ uint32_t* fb_head(int s) const { return w + 8 + 2 * NG + 4 * NH + s; }
};

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Back-off for spin waits; a wait that never ends (a scheduling bug) traps after ~10 s
// instead of hanging the device.
__device__ __forceinline__ void spin_pause(uint32_t& n) {
  __nanosleep(128);
  if (++n > (1u << 26)) __trap();
}

// thread 0 spins until *f >= target; the barrier then releases the whole CTA
template <class Gp>
__device__ __forceinline__ void wait_geq(const uint32_t* f, uint32_t target) {
  if (Gp::tid() == 0) {
    uint32_t n = 0;
    while (ld_acquire(f) < target) spin_pause(n);
  }
  Gp::sync();
}

// every thread's prior writes are made visible before *f is bumped
template <class Gp>
__device__ __forceinline__ void publish_add(uint32_t* f, uint32_t v) {
  __threadfence();
  Gp::sync();
  if (Gp::tid() == 0) atomicAdd(f, v);
}

__device__ __forceinline__ int group_of(const FusedParams& p, int bh) {
  const int b = bh / p.a.Hq, h = bh % p.a.Hq;
  return b * p.a.Hkv + h / p.a.G;
}
__device__ __forceinline__ int head_of(const FusedParams& p, int g, int n) {
  const int b = g / p.a.Hkv, kvh = g % p.a.Hkv;
  return b * p.a.Hq + kvh * p.a.G + n;
}

// ------------------------------------------------------------------------- schedule
struct Sched {
  int NG, NH, G, NS, T, KS, KA;
  uint32_t pre;  // SAMPLE + THRESH items
  // block g (0..NG): SCAN(g)[0,T/2) | KTH(g-1) | SCAN(g)[T/2,T) | ATT(g-1)
  __device__ int szA(int g) const { return g < NG ? T / 2 : 0; }
  __device__ int szB(int g) const { return (g >= 1 && g <= NG) ? G * KS : 0; }
  __device__ int szC(int g) const { return g < NG ? T - T / 2 : 0; }
  __device__ int szD(int g) const { return (g >= 1 && g <= NG) ? G * KA : 0; }
  __device__ int size(int g) const { return szA(g) + szB(g) + szC(g) + szD(g); }
  __device__ int nblocks() const { return NG + 1; }
};

__device__ Item decode(const Sched& s, const uint32_t* blk, uint32_t it) {
  if (it < s.pre) {  // group by group: SAMPLE(g, 0..NS) THRESH(heads of g), so g's threshold is early
    const int per = s.NS + s.G;
    const int g = static_cast<int>(it / per), o = static_cast<int>(it % per);
    if (o < s.NS) return {kItSample, g, o};
    return {kItThresh, g * s.G + (o - s.NS), 0};  // head index b·Hq + kvh·G + n = g·G + n
  }
  const uint32_t j = it - s.pre;
  int lo = 0, hi = s.nblocks();  // largest g with blk[g] <= j
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (blk[mid] <= j) lo = mid; else hi = mid;
  }
  const int g = lo;
  int o = static_cast<int>(j - blk[g]);
  if (o < s.szA(g)) return {kItScan, g, o};
  o -= s.szA(g);
  if (o < s.szB(g)) return {kItKth, (g - 1) * s.G + o / s.KS, o % s.KS};  // group-major head index
  o -= s.szB(g);
  if (o < s.szC(g)) return {kItScan, g, s.T / 2 + o};
  o -= s.szC(g);
  if (o < s.szD(g)) return {kItAtt, (g - 1) * s.G + o / s.KA, o % s.KA};
  return {kItNop, 0, 0};
}

// ------------------------------------------------------------------------- SAMPLE
template <class Gp>
__device__ void do_sample(const FusedParams& p, const Ctl& ctl, int g, int part) {
  const AttendParams& a = p.a;
  const int b = g / a.Hkv, kvh = g % a.Hkv;
  const int lane = Gp::tid() & 31, warp = Gp::tid() >> 5;
  const int gg = lane >> 2, c = lane & 3;
  const int64_t N = a.n_ctx[b];
  if (N > 0) {
    const int64_t stride = sample_stride(N);
    const int Sb = static_cast<int>((N + stride - 1) / stride);
    QFrag f;
    load_qfrag(f, a.q + (static_cast<int64_t>(b) * a.Hq + kvh * a.G) * kD, a.G, lane);
    const __nv_bfloat16* kbase = a.kc + (static_cast<int64_t>(b) * a.Hkv + kvh) * a.cache_rows * kD;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int s0 = part * FT + warp * 32 + u * 16;
      const int sA = s0 + gg, sB = s0 + gg + 8;
      uint4 t[2][4];
      load_tile(t, kbase + static_cast<int64_t>(sA) * stride * kD, sA < Sb,
                kbase + static_cast<int64_t>(sB) * stride * kD, sB < Sb, c);
      float acc[4];
      score_tile(acc, t, f);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int col = 2 * c + (i & 1);
        const int s = (i < 2) ? sA : sB;
        if (col < a.G && s < Sb)
          p.samp[static_cast<int64_t>(head_of(p, g, col)) * kSamples + s] = score_key(acc[i]);
      }
    }
  }
  publish_add<Gp>(ctl.samp_done(g), 1u);
}

// ------------------------------------------------------------------------- THRESH
template <class Gp>
__device__ void do_thresh(const FusedParams& p, const Ctl& ctl, int bh, unsigned char* smem) {
  const AttendParams& a = p.a;
  uint32_t* s_keys = reinterpret_cast<uint32_t*>(smem);          // [kSamples]
  uint32_t* s_hist = s_keys + kSamples;                           // [2048]
  uint32_t* s_scr = s_hist + 2048;                                // [32]
  uint32_t* s_out = s_scr + 32;                                   // [4]
  uint32_t* s_max = s_out + 4;                                    // [FW]
  const int tid = Gp::tid(), lane = tid & 31, warp = tid >> 5;
  const int b = bh / a.Hq;
  const int64_t N = a.n_ctx[b];
  const int64_t kb = N < a.k ? N : a.k;
  int Sb = 0;
  if (N > 0) {
    const int64_t stride = sample_stride(N);
    Sb = static_cast<int>((N + stride - 1) / stride);
  }
  const double mu = N > 0 ? static_cast<double>(kb) * Sb / static_cast<double>(N) : 0.0;
  const double rr = ceil(mu + 6.0 * sqrt(mu) + 16.0);
  const bool filter = !p.no_filter && kb > 0 && rr < static_cast<double>(Sb);
  uint32_t thr = 0u, shift = kNoFilterShift;
  if (filter) {
    wait_geq<Gp>(ctl.samp_done(group_of(p, bh)), static_cast<uint32_t>(p.NS));
    copy_g2s_u32<FT, kSamples, Gp>(s_keys, p.samp + static_cast<int64_t>(bh) * kSamples, (Sb + 3) & ~3);
    Gp::sync();
    uint32_t mx = 0u;
    for (int i = tid; i < Sb; i += FT) mx = max(mx, s_keys[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(kFull, mx, o));
    if (lane == 0) s_max[warp] = mx;
    Gp::sync();
    uint32_t prefix = 0, need = static_cast<uint32_t>(rr);
    int sh = 32;
    bool exact = false;
    for (int pi = 0; pi < 3; ++pi) {
      const int w = pi < 2 ? 11 : 10;
      const int nsh = sh - w;
      const uint32_t mask = (1u << w) - 1u;
      for (int i = tid; i <= static_cast<int>(mask); i += FT) s_hist[i] = 0u;
      Gp::sync();
      for (int i = tid; i < Sb; i += FT) {
        const uint32_t k = s_keys[i];
        if (sh == 32 || (k >> sh) == prefix) hist_add_aggregated(s_hist, (k >> nsh) & mask);
      }
      Gp::sync();
      if (w == 11)
        find_bucket<FT, 2048, Gp>(s_hist, need, s_out, s_scr);
      else
        find_bucket<FT, 1024, Gp>(s_hist, need, s_out, s_scr);
      need -= s_out[1];
      prefix = (prefix << w) | s_out[0];
      sh = nsh;
      const uint32_t bc = s_hist[s_out[0]];
      const bool done = bc == need;
      Gp::sync();
      if (done) break;
      if (bc <= 2048u) {
        if (tid == 0) s_out[2] = 0u;
        Gp::sync();
        for (int i = tid; i < Sb; i += FT) {
          const uint32_t k = s_keys[i];
          if ((k >> sh) == prefix) s_hist[atomicAdd(&s_out[2], 1u)] = k;
        }
        Gp::sync();
        thr = block_rank_select<FT, uint32_t, Gp>(s_hist, static_cast<int>(s_out[2]), static_cast<int>(need), &s_out[3]);
        exact = true;
        break;
      }
    }
    if (!exact) thr = sh > 0 ? prefix << sh : prefix;
    uint32_t smax = 0u;
    for (int w = 0; w < FW; ++w) smax = max(smax, s_max[w]);
    const uint32_t range = smax - thr;
    const int bits = range ? 32 - __clz(range) : 0;
    shift = bits > 10 ? static_cast<uint32_t>(bits - 10) : 0u;
  }
  uint4* gh = reinterpret_cast<uint4*>(p.hs.hist + static_cast<int64_t>(bh) * kHistBins);
  for (int i = tid; i < kHistBins / 4; i += FT) gh[i] = make_uint4(0, 0, 0, 0);
  for (int i = tid; i < a.pin_words; i += FT) a.pin_mask[static_cast<int64_t>(bh) * a.pin_words + i] = 0u;
  if (tid == 0) {
    p.hs.thr[bh] = thr;
    p.hs.hshift[bh] = shift;
    p.hs.cand_cnt[bh] = 0u;
    p.hs.max_comp[bh] = 0ull;
    p.hs.bkt_cnt[bh] = 0u;
    p.hs.out_cnt[bh] = 0u;
  }
  publish_add<Gp>(ctl.thr_ready(bh), 1u);
}

// ------------------------------------------------------------------------- SCAN
// Scores rows [tile*TR, (tile+1)*TR) of group g for its G heads (or, fallback, for fb_head
// only) and appends every row whose key passes the head's threshold to the candidates.
template <class Gp>
__device__ void do_scan(const FusedParams& p, const Ctl& ctl, int g, int tile, int fb_head,
                        unsigned char* smem, int& ready_group) {
  const AttendParams& a = p.a;
  const int fl = p.scan_flush_iters;                                            // iterations per flush
  const int stage = kScanRows * fl;                                              // staged per head
  uint64_t* s_buf = reinterpret_cast<uint64_t*>(smem);                          // [G][stage]
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_buf + a.G * stage);           // [8]
  const int tid = Gp::tid(), lane = tid & 31, warp = tid >> 5;
  const int gg = lane >> 2, c = lane & 3;
  const int b = g / a.Hkv, kvh = g % a.Hkv;
  const int bh0 = b * a.Hq + kvh * a.G;
  if (fb_head < 0 && ready_group != g) {
    if (tid == 0) {
      uint32_t spins = 0;
      for (int n = 0; n < a.G; ++n)
        while (ld_acquire(ctl.thr_ready(bh0 + n)) == 0u) spin_pause(spins);
    }
    ready_group = g;
  }
  if (tid < 8) s_cnt[tid] = 0u;
  Gp::sync();
  const int64_t nctx = a.n_ctx[b];
  const int TR = p.tile_iters * kScanRows;
  const int64_t r0 = static_cast<int64_t>(tile) * TR;
  int64_t r1 = r0 + TR;
  r1 = r1 < nctx ? r1 : nctx;
  const int col0 = 2 * c, col1 = 2 * c + 1;
  const bool en0 = col0 < a.G && (fb_head < 0 || bh0 + col0 == fb_head);
  const bool en1 = col1 < a.G && (fb_head < 0 || bh0 + col1 == fb_head);
  const uint32_t thr0 = col0 < a.G ? __ldcg(&p.hs.thr[bh0 + col0]) : 0u;
  const uint32_t thr1 = col1 < a.G ? __ldcg(&p.hs.thr[bh0 + col1]) : 0u;
  // flush: warp n moves head n's staged candidates to HBM and adds them to its histogram
  auto flush = [&]() {
    Gp::sync();
    if (warp < a.G) {
      const uint32_t cnt = s_cnt[warp];
      __syncwarp();
      if (cnt) {
        const int bh = bh0 + warp;
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(&p.hs.cand_cnt[bh], cnt);
        base = __shfl_sync(kFull, base, 0);
        const uint32_t thr = __ldcg(&p.hs.thr[bh]), shift = __ldcg(&p.hs.hshift[bh]);
        uint32_t* gh = p.hs.hist + static_cast<int64_t>(bh) * kHistBins;
        uint64_t* dst = const_cast<uint64_t*>(a.cand) + static_cast<int64_t>(bh) * a.cap + base;
        const uint64_t* src = s_buf + warp * stage;
        for (uint32_t i = lane; i < cnt; i += 32) {
          const uint64_t cc = src[i];
          dst[i] = cc;
          const uint32_t d = hist_digit(comp_key(cc), thr, shift);
          const unsigned peers = __match_any_sync(__activemask(), d);
          if (lane == static_cast<int>(__ffs(peers) - 1)) atomicAdd(&gh[d], __popc(peers));
        }
      }
      __syncwarp();
      if (lane == 0) s_cnt[warp] = 0u;
    }
    Gp::sync();
  };
  if (r0 < r1) {
    QFrag f;
    load_qfrag(f, a.q + static_cast<int64_t>(bh0) * kD, a.G, lane);
    const __nv_bfloat16* kbase = a.kc + (static_cast<int64_t>(b) * a.Hkv + kvh) * a.cache_rows * kD;
    for (int it = 0; it < p.tile_iters; ++it) {
      if (r0 + static_cast<int64_t>(it) * kScanRows >= r1) break;  // CTA-uniform
      const int64_t rbase = r0 + static_cast<int64_t>(it) * kScanRows + warp * 16 * kScanU;
      if (rbase < r1) {  // warp-uniform
        uint4 t[kScanU][2][4];
#pragma unroll
        for (int u = 0; u < kScanU; ++u) {
          const int64_t rA = rbase + u * 16 + gg, rB = rA + 8;
          load_tile(t[u], kbase + rA * kD, rA < r1, kbase + rB * kD, rB < r1, c);
        }
#pragma unroll
        for (int u = 0; u < kScanU; ++u) {
          float acc[4];
          score_tile(acc, t[u], f);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const bool hi = (i & 1) != 0;
            const int64_t row = rbase + u * 16 + gg + ((i >> 1) ? 8 : 0);
            const uint32_t key = score_key(acc[i]);
            const bool pass = (hi ? en1 : en0) && row < r1 && key >= (hi ? thr1 : thr0);
            const unsigned m = __ballot_sync(kFull, pass);
            if (m != 0u && pass) {
              const unsigned same = m & (0x11111111u << c);
              const int leader = __ffs(same) - 1;
              const int col = hi ? col1 : col0;
              uint32_t base = 0;
              if (lane == leader) base = atomicAdd(&s_cnt[col], static_cast<uint32_t>(__popc(same)));
              base = __shfl_sync(m, base, leader);
              const uint32_t rank = __popc(same & ((1u << lane) - 1u));
              s_buf[col * stage + base + rank] =
                  make_comp(key, static_cast<uint32_t>(a.row_offset) + static_cast<uint32_t>(row));
            }
          }
        }
      }
      if (it % fl == fl - 1 && it + 1 < p.tile_iters) flush();  // staging holds fl iterations per head
    }
  }
  flush();
  publish_add<Gp>(fb_head < 0 ? ctl.scan_done(g) : ctl.fb_scan_done(fb_head), 1u);
}

// ------------------------------------------------------------------------- KTH
template <class Gp>
__device__ void do_kth(const FusedParams& p, const Ctl& ctl, int bh, int slice, bool fb,
                       unsigned char* smem) {
  const AttendParams& a = p.a;
  uint32_t* s_hist = reinterpret_cast<uint32_t*>(smem);                   // [4096]
  uint64_t* s_bkt = reinterpret_cast<uint64_t*>(s_hist + kHistBins);      // [kFBkt]
  uint32_t* s_scr = reinterpret_cast<uint32_t*>(s_bkt + kFBkt);           // [32]
  uint32_t* s_out = s_scr + 32;                                           // [4]
  uint64_t* s_r64 = reinterpret_cast<uint64_t*>(s_out + 4);               // [FW + 2]
  const int tid = Gp::tid(), lane = tid & 31, warp = tid >> 5;
  const int b = bh / a.Hq, g = group_of(p, bh);
  if (fb)
    wait_geq<Gp>(ctl.fb_scan_done(bh), static_cast<uint32_t>(p.T));
  else
    wait_geq<Gp>(ctl.scan_done(g), static_cast<uint32_t>(p.scan_target));
  stamp_ready(p, tid);
  int64_t n = __ldcg(&p.hs.cand_cnt[bh]);
  if (n > a.cap) n = a.cap;
  const int64_t N = a.n_ctx[b];
  const int64_t kb = N < a.k ? N : a.k;
  const uint32_t final_state = fb ? 3u : 1u;

  if (!fb && n < kb) {
    // the sampled threshold passed fewer than k rows: queue an exact re-scan of this head
    if (slice == 0) {
      uint4* gh = reinterpret_cast<uint4*>(p.hs.hist + static_cast<int64_t>(bh) * kHistBins);
      for (int i = tid; i < kHistBins / 4; i += FT) gh[i] = make_uint4(0, 0, 0, 0);
      if (tid == 0) {
        p.hs.cand_cnt[bh] = 0u;
        p.hs.thr[bh] = 0u;
        p.hs.hshift[bh] = kNoFilterShift;
        p.hs.max_comp[bh] = 0ull;
        p.hs.bkt_cnt[bh] = 0u;
        p.hs.out_cnt[bh] = 0u;
        p.hs.kth_ticket[bh] = 0u;
        p.hs.flag_fail[bh] = 1u;
      }
      __threadfence();
      Gp::sync();
      if (tid == 0) {
        const uint32_t s = atomicAdd(ctl.fb_alloc(), 1u);
        *ctl.fb_head(static_cast<int>(s)) = static_cast<uint32_t>(bh);
        __threadfence();
        uint32_t spins = 0;
        while (ld_acquire(ctl.nfb()) != s) spin_pause(spins);  // publish jobs in slot order
        atomicAdd(ctl.nfb(), 1u);
        atomicExch(ctl.kth_state(bh), 2u);  // static ATT items of this head stand down
      }
      Gp::sync();
    }
    return;
  }
  if (kb == 0) {
    if (slice == 0) {
      if (tid == 0) {
        const_cast<uint64_t*>(a.meta_kth)[bh] = ~0ull;
        const_cast<int32_t*>(a.meta_kb)[bh] = 0;
        const_cast<float*>(a.meta_max)[bh] = -INFINITY;
      }
      __threadfence();
      Gp::sync();
      if (tid == 0) atomicExch(ctl.kth_state(bh), final_state);
    }
    return;
  }

  const uint32_t thr = __ldcg(&p.hs.thr[bh]), shift = __ldcg(&p.hs.hshift[bh]);
  const bool all = kb >= n;
  uint32_t dstar = 0, need = 0, bcnt = 0;
  bool whole = true;
  if (!all) {
    copy_g2s_u32<FT, kHistBins, Gp>(s_hist, p.hs.hist + static_cast<int64_t>(bh) * kHistBins, kHistBins);
    Gp::sync();
    find_bucket<FT, kHistBins, Gp>(s_hist, static_cast<uint32_t>(kb), s_out, s_scr);
    dstar = s_out[0];
    need = static_cast<uint32_t>(kb) - s_out[1];
    bcnt = s_hist[dstar];
    whole = bcnt == need;
  }
  const bool refine = !all && !whole;
  const bool big = refine && bcnt > static_cast<uint32_t>(kSelectBucketCap);
  const uint64_t* src = a.cand + static_cast<int64_t>(bh) * a.cap;
  const int64_t lo = n * slice / p.KS, hi = n * (slice + 1) / p.KS;
  uint64_t vmax = 0ull;
  uint64_t* gbkt = p.hs.bkt + static_cast<int64_t>(bh) * kSelectBucketCap;
  constexpr int UNR = 8;
  for (int64_t start = lo; start < hi; start += FT * UNR) {
    uint64_t cv[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t i = start + u * FT + tid;
      cv[u] = i < hi ? __ldcg(&src[i]) : 0ull;
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const uint64_t c = cv[u];
      vmax = c > vmax ? c : vmax;
      const bool inb = refine && !big && c != 0ull && hist_digit(comp_key(c), thr, shift) == dstar;
      const unsigned bb = __ballot_sync(kFull, inb);
      if (bb) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(&p.hs.bkt_cnt[bh], __popc(bb));
        base = __shfl_sync(kFull, base, 0);
        if (inb) {
          const uint32_t pos = base + __popc(bb & lanemask_lt());
          if (pos < static_cast<uint32_t>(kSelectBucketCap)) gbkt[pos] = c;
        }
      }
    }
  }
  vmax = warp_max_u64(vmax);
  if (lane == 0) s_r64[warp] = vmax;
  Gp::sync();
  if (tid == 0) {
    uint64_t m = 0ull;
    for (int w = 0; w < FW; ++w) m = s_r64[w] > m ? s_r64[w] : m;
    atomicMax(reinterpret_cast<unsigned long long*>(&p.hs.max_comp[bh]), static_cast<unsigned long long>(m));
  }
  __threadfence();
  Gp::sync();
  if (tid == 0) s_out[2] = (atomicAdd(&p.hs.kth_ticket[bh], 1u) == static_cast<unsigned>(p.KS - 1)) ? 1u : 0u;
  Gp::sync();
  if (!s_out[2]) return;
  __threadfence();

  uint64_t T;
  if (all) {
    T = 1ull;
  } else if (whole) {
    T = static_cast<uint64_t>(thr + (dstar << shift)) << 32;
  } else {
    int cs = 64;
    uint64_t cp = 0;
    const int64_t nb = __ldcg(&p.hs.bkt_cnt[bh]);
    if (!big && nb <= kFBkt) {
      for (int64_t i = tid; i < nb; i += FT) s_bkt[i] = __ldcg(&gbkt[i]);
      Gp::sync();
      cp = block_rank_select<FT, uint64_t, Gp>(s_bkt, static_cast<int>(nb), static_cast<int>(need), &s_r64[FW]);
      cs = 0;
    } else if (!big) {
      auto ld = [&](int64_t i, uint64_t& c) {
        c = __ldcg(&gbkt[i]);
        return true;
      };
      radix_select_u64<FT, decltype(ld), Gp>(ld, nb, need, s_hist, s_scr, s_out, cs, cp);
    } else {
      auto ld = [&](int64_t i, uint64_t& c) {
        c = __ldcg(&src[i]);
        return c != 0ull && hist_digit(comp_key(c), thr, shift) == dstar;
      };
      radix_select_u64<FT, decltype(ld), Gp>(ld, n, need, s_hist, s_scr, s_out, cs, cp);
    }
    T = cp << cs;
  }
  if (tid == 0) {
    const_cast<uint64_t*>(a.meta_kth)[bh] = T;
    const_cast<int32_t*>(a.meta_kb)[bh] = static_cast<int32_t>(kb);
    const_cast<float*>(a.meta_max)[bh] = key_score(comp_key(__ldcg(&p.hs.max_comp[bh])));
    p.hs.kth_ticket[bh] = 0u;
    p.hs.bkt_cnt[bh] = 0u;
    if (fb) p.hs.flag_fail[bh] = 0u;
  }
  __threadfence();
  Gp::sync();
  if (tid == 0) atomicExch(ctl.kth_state(bh), final_state);
}

// ------------------------------------------------------------------------- ATT
// Chunks ai, ai+KA, ... of head bh's candidate list: keep c >= T, append the kept rows to
// idx/scores, gather their V rows into per-chunk partials; the CTA that completes the head's
// chunk count combines them, adds pinned-prefix and window rows and writes out.
template <class Gp>
__device__ void do_att(const FusedParams& p, const Ctl& ctl, int bh, int ai, bool fb, unsigned char* smem) {
  const AttendParams& a = p.a;
  AttSmem& sm = *reinterpret_cast<AttSmem*>(smem);
  const int tid = Gp::tid(), lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    uint32_t st;
    uint32_t spins = 0;
    while ((st = ld_acquire(ctl.kth_state(bh))) == 0u || (fb && st != 3u)) spin_pause(spins);
    sm.base = st;
  }
  Gp::sync();
  const uint32_t state = sm.base;
  stamp_ready(p, tid);
  Gp::sync();
  if (!fb && state == 2u) return;  // failed head: its fallback job does the work

  int64_t n = __ldcg(&p.hs.cand_cnt[bh]);
  if (n > a.cap) n = a.cap;
  const int nch = n > 0 ? static_cast<int>((n + kCandChunk - 1) / kCandChunk) : 1;
  const int kb = __ldcg(&a.meta_kb[bh]);
  const uint64_t T = __ldcg(&a.meta_kth[bh]);
  const float zs = a.scale * kLog2e;
  const float zref = kb > 0 ? __ldcg(&a.meta_max[bh]) * zs : 0.f;
  int32_t* idx_o = a.idx_out + static_cast<int64_t>(bh) * a.k;
  float* sc_o = a.scores_out + static_cast<int64_t>(bh) * a.k;
  uint32_t mine = 0;
  for (int slot = ai; slot < nch; slot += p.KA) {
    const uint64_t* src = a.cand + static_cast<int64_t>(bh) * a.cap + static_cast<int64_t>(slot) * kCandChunk;
    int64_t cnt = n - static_cast<int64_t>(slot) * kCandChunk;
    cnt = cnt < 0 ? 0 : (cnt > kCandChunk ? kCandChunk : cnt);
    constexpr int PER = kCandChunk / FT;
    uint64_t cv[PER];
    bool sel[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int i = u * FT + tid;
      cv[u] = (i < cnt && kb > 0) ? __ldcg(&src[i]) : 0ull;
      sel[u] = cv[u] != 0ull && cv[u] >= T;
    }
    uint32_t my = 0;
#pragma unroll
    for (int u = 0; u < PER; ++u) my += sel[u] ? 1u : 0u;
    uint32_t incl = my;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) sm.wcnt[warp] = incl;
    Gp::sync();
    uint32_t woff = 0, m = 0;
    for (int w = 0; w < FW; ++w) {
      woff += w < warp ? sm.wcnt[w] : 0u;
      m += sm.wcnt[w];
    }
    if (tid == 0) sm.base = m ? atomicAdd(&a.out_cnt[bh], m) : 0u;
    Gp::sync();
    const uint32_t obase = sm.base;
    uint32_t pos = woff + incl - my;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      if (sel[u]) {
        const uint64_t c = cv[u];
        const uint32_t gid = comp_gid(c);
        const float s = key_score(comp_key(c));
        const uint32_t o = obase + pos;
        if (o < static_cast<uint32_t>(a.k)) {
          idx_o[o] = static_cast<int32_t>(gid);
          sc_o[o] = s;
          if (a.packed_out) a.packed_out[static_cast<int64_t>(bh) * a.k + o] = c;
        }
        mark_pinned(a, bh, static_cast<int64_t>(gid) - a.row_offset);
        sm.row[pos] = static_cast<int32_t>(static_cast<int64_t>(gid) - a.row_offset);
        sm.w[pos] = exp2f(fmaf(s, zs, -zref));
        ++pos;
      }
    }
    if (slot == 0) {  // pads for k > kb (reference clamps k to N, attention.py:147-149)
      for (int i = kb + tid; i < a.k; i += FT) {
        idx_o[i] = -1;
        sc_o[i] = -INFINITY;
        if (a.packed_out) a.packed_out[static_cast<int64_t>(bh) * a.k + i] = 0ull;
      }
    }
    Gp::sync();
    if (a.gather) gather_partial<Gp>(a, bh, slot, static_cast<int>(m), sm);
    ++mine;
  }
  if (!a.gather || mine == 0) return;
  __threadfence();
  Gp::sync();
  if (tid == 0) {
    const uint32_t old = atomicAdd(ctl.att_ticket(bh), mine);
    sm.last = (old + mine == static_cast<uint32_t>(nch)) ? 1 : 0;
  }
  Gp::sync();
  if (!sm.last) return;
  __threadfence();
  head_finish<Gp>(a, bh, nch, sm);
}

__device__ Item decode_dyn(const FusedParams& p, const Ctl& ctl, uint32_t j) {
  const int per = p.T + p.KS + p.KA;
  const int bh = static_cast<int>(__ldcg(ctl.fb_head(static_cast<int>(j / per))));
  const int o = static_cast<int>(j % per);
  if (o < p.T) return {kItFbScan, bh, o};
  if (o < p.T + p.KS) return {kItFbKth, bh, o - p.T};
  return {kItFbAtt, bh, o - p.T - p.KS};
}

// The work-queue loop, run by a thread group (the whole CTA in fused_kernel, the eight
// work-queue warps in fused_tc_kernel). Claims items in order until none is left.
template <class Gp>
__device__ void run_queue(const FusedParams& p, const Ctl& ctl, const Sched& sc, const uint32_t* blk,
                          unsigned char* work, uint32_t* s_item) {
  const int tid = Gp::tid();
  const uint32_t static_items = sc.pre + blk[sc.nblocks()];
  const uint32_t per_fb = static_cast<uint32_t>(p.T + p.KS + p.KA);
  int ready_group = -1;
  bool dyn = false;
  // thread 0: fallback jobs are claimed by CAS so an index is never lost; a static claim past
  // the static items is discarded (it is not a dynamic item)
  auto claim_dyn = [&]() -> uint32_t {
    for (;;) {
      const uint32_t cur = ld_acquire(ctl.dyn());
      if (cur >= ld_acquire(ctl.nfb()) * per_fb) return kNoItem;
      if (atomicCAS(ctl.dyn(), cur, cur + 1u) == cur) return static_items + cur;
    }
  };
  if (tid == 0) {
    const uint32_t first = atomicAdd(ctl.item(), 1u);
    if (first < static_items) {
      *s_item = first;
    } else {
      dyn = true;
      *s_item = claim_dyn();
    }
  }
  Gp::sync();
  for (;;) {
    const uint32_t it = *s_item;
    Gp::sync();
    if (it == kNoItem) break;
    uint32_t next = kNoItem;
    if (tid == 0 && !dyn) next = atomicAdd(ctl.item(), 1u);  // prefetch the next claim
    Item item;
    if (it < static_items) {
      item = decode(sc, blk, it);
    } else {
      item = decode_dyn(p, ctl, it - static_items);
    }
#ifdef TKV_DEBUG
    if (tid == 0)
      printf("[cta %d] item %u type %d a %d b %d (static %u)\n", blockIdx.x, it, item.type, item.a, item.b,
             static_items);
#endif
    uint64_t t_start = 0;
    if (p.trace && tid == 0) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
      s_item_ready = t_start;
    }
    switch (item.type) {
      case kItSample: do_sample<Gp>(p, ctl, item.a, item.b); break;
      case kItThresh: do_thresh<Gp>(p, ctl, item.a, work); break;
      case kItScan: do_scan<Gp>(p, ctl, item.a, item.b, -1, work, ready_group); break;
      case kItKth: do_kth<Gp>(p, ctl, item.a, item.b, false, work); break;
      case kItAtt: do_att<Gp>(p, ctl, item.a, item.b, false, work); break;
      case kItFbScan: do_scan<Gp>(p, ctl, group_of(p, item.a), item.b, item.a, work, ready_group); break;
      case kItFbKth: do_kth<Gp>(p, ctl, item.a, item.b, true, work); break;
      case kItFbAtt: do_att<Gp>(p, ctl, item.a, item.b, true, work); break;
      default: break;
    }
    Gp::sync();
    if (p.trace && tid == 0 && it < p.trace_cap) {
      uint64_t t_end;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
      uint64_t* r = p.trace + static_cast<uint64_t>(it) * 4;
      r[0] = t_start;
      r[1] = t_end;
      r[2] = (static_cast<uint64_t>(item.type) << 32) | blockIdx.x;
      r[3] = (static_cast<uint64_t>(static_cast<uint32_t>(item.a)) << 32) | static_cast<uint32_t>(item.b);
      r[2] |= static_cast<uint64_t>((s_item_ready - t_start) / 64u & 0xFFFFFFu) << 40 >> 0;  // wait (64 ns units)
    }
    if (tid == 0) {
      if (!dyn && next < static_items) {
        *s_item = next;
      } else {
        dyn = true;
        *s_item = claim_dyn();
      }
    }
    Gp::sync();
  }
}

__device__ __forceinline__ void build_block_table(const Sched& sc, uint32_t* blk) {
  uint32_t acc = 0;
  for (int g = 0; g < sc.nblocks(); ++g) {
    blk[g] = acc;
    acc += static_cast<uint32_t>(sc.size(g));
  }
  blk[sc.nblocks()] = acc;
}

// the last CTA out re-zeroes the control block for the next launch (block-wide call)
__device__ __forceinline__ void reset_ctl_if_last(const FusedParams& p, const Ctl& ctl, int* s_last) {
  if (threadIdx.x == 0) {
    __threadfence();
    *s_last = atomicAdd(ctl.exited(), 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (*s_last) {
    const int words = fused_ctl_words(ctl.NG, ctl.NH);
    for (int i = threadIdx.x; i < words; i += blockDim.x) p.ctl[i] = 0u;
  }
}
}  // namespace

__global__ void __launch_bounds__(FT, 2) fused_kernel(FusedParams p) {
  extern __shared__ __align__(16) unsigned char f_smem[];
  __shared__ uint32_t s_item;
  __shared__ int s_last;
  const int NG = p.a.B * p.a.Hkv, NH = p.a.B * p.a.Hq;
  const Ctl ctl{p.ctl, NG, NH};
  Sched sc{NG, NH, p.a.G, p.NS, p.T, p.KS, p.KA, static_cast<uint32_t>(p.NS * NG + NH)};
  // block-start table of the interleaved part of the schedule
  uint32_t* blk = reinterpret_cast<uint32_t*>(f_smem);
  unsigned char* work = f_smem + ((static_cast<size_t>(NG) + 3) * 4 + 15) / 16 * 16;
  if (threadIdx.x == 0) build_block_table(sc, blk);
  __syncthreads();
  run_queue<CtaGrp>(p, ctl, sc, blk, work, &s_item);
  reset_ctl_if_last(p, ctl, &s_last);
}

namespace {
// ------------------------------------------------------------------------- fused_tc_kernel
// The layer step with the key scan on the tcgen05 pipeline, warp-specialised in one persistent
// CTA per SM (448 threads):
//   warps 0–5   the scan roles of scan_tc.cu (TMA producer, MMA issuer, 4 epilogue warps),
//               walking the KV groups IN ORDER — every CTA scans its share of group 0, then of
//               group 1, … — so group g's candidates are complete early; each epilogue warp
//               bumps scan_done(g) after flushing its last candidates of g (target 4 · grid);
//   warps 6–13  the work queue of fused_kernel without SCAN items: SAMPLE/THRESH of every group
//               first (group 0 first — the epilogue waits for its thresholds), then KTH(g) and
//               ATT(g) per group, which wait for scan_done(g) and so run beside the scan of
//               groups g+1, …; the exactness fallback re-scans on these warps (mma.sync).
// The scan warps only wait on THRESH items, which never wait on the scan, and every CTA is
// co-resident (one CTA per SM, grid = #SMs, cooperative launch), so nothing can deadlock.
constexpr int kFtcThreads = tc::kTcThreads + FT;
using QueueGrp = WarpGrp<tc::kTcThreads, FT, 1>;

// live units [lo, hi) of group g scanned by this CTA: the group's units split into `grid`
// contiguous shares, share (cta + g) mod grid — rotating, so the remainder units spread evenly
__device__ __forceinline__ void group_share(const FusedParams& p, int g, int64_t ups, int64_t& lo, int64_t& hi) {
  const int grid = static_cast<int>(gridDim.x);
  const int r = static_cast<int>((static_cast<int64_t>(blockIdx.x) + g) % grid);
  lo = ups * r / grid;
  hi = ups * (r + 1) / grid;
  const int64_t nctx = p.a.n_ctx[g / p.a.Hkv];
  const int64_t live = (nctx + tc::kTcUnit - 1) / tc::kTcUnit;
  if (hi > live) hi = live;
  if (lo > hi) lo = hi;
}
}  // namespace

__global__ void __launch_bounds__(kFtcThreads, 1) fused_tc_kernel(const __grid_constant__ CUtensorMap kmap,
                                                                  FusedParams p, int n_stages, int flush_every,
                                                                  int tc_bytes) {
  using namespace tc;
  extern __shared__ __align__(16) unsigned char f_smem[];  // tc_setup aligns the pipeline to 1024
  __shared__ __align__(8) uint64_t s_bar[kTcBarWords];
  __shared__ uint32_t s_tmem;
  __shared__ uint32_t s_item;
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const AttendParams& a = p.a;
  const int NG = a.B * a.Hkv, NH = a.B * a.Hq;
  const Ctl ctl{p.ctl, NG, NH};
  Sched sc{NG, NH, a.G, p.NS, 0 /* no SCAN items */, p.KS, p.KA, static_cast<uint32_t>(p.NS * NG + NH)};
  TcPipe t = tc_setup(f_smem, s_bar, &s_tmem, a.G, flush_every, n_stages, &kmap, tid == 0, warp == 1);
  uint32_t* blk = reinterpret_cast<uint32_t*>(f_smem + tc_bytes);
  unsigned char* work = f_smem + tc_bytes + ((static_cast<size_t>(NG) + 3) * 4 + 15) / 16 * 16;
  if (tid == kTcThreads) build_block_table(sc, blk);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  t.tmem = s_tmem;
  const int64_t ups = (p.max_ctx + kTcUnit - 1) / kTcUnit;

  if (warp == 0) {  // TMA producer
    uint32_t i = 0;
    for (int g = 0; g < NG; ++g) {
      int64_t lo, hi;
      group_share(p, g, ups, lo, hi);
      for (int64_t u = lo; u < hi; ++u, ++i)
        tc_produce(t, i, &kmap, static_cast<int>(g * a.cache_rows + u * kTcUnit), lane, 0);
    }
  } else if (warp == 1) {  // MMA issuer
    uint32_t i = 0;
    QRing qr;
    for (int g = 0; g < NG; ++g) {
      int64_t lo, hi;
      group_share(p, g, ups, lo, hi);
      for (int64_t u = lo; u < hi; ++u, ++i) {
        tc_mma_acquire(t, i);
        if (u == lo) tc_next_q(t, qr, a.q + static_cast<int64_t>(g) * a.G * kD, a.G, lane);
        tc_mma_issue(t, i, qr.slot, lane, 0);
      }
    }
  } else if (warp < kTcThreads / 32) {  // epilogue
    const int ew = warp - 2;
    const int quarter = warp & 3;  // TMEM lanes this warp may access: [32·quarter, +32)
    uint64_t* wbuf = t.s_buf + static_cast<int64_t>(ew) * a.G * t.cap;
    uint32_t thr[8], shift[8], cnt[8];
#pragma unroll
    for (int n = 0; n < 8; ++n) cnt[n] = thr[n] = shift[n] = 0u;
    uint32_t i = 0;
    for (int g = 0; g < NG; ++g) {
      int64_t lo, hi;
      group_share(p, g, ups, lo, hi);
      const int64_t bh0 = static_cast<int64_t>(g) * a.G;
      uint64_t t_start = 0, t_ready = 0;
      if (p.trace && lane == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
      if (lo < hi) {
        // the group's thresholds come from THRESH items of the work queue
        if (lane < a.G) {
          uint32_t spins = 0;
          while (ld_acquire(ctl.thr_ready(static_cast<int>(bh0) + lane)) == 0u) spin_pause(spins);
        }
        __syncwarp();
        if (p.trace && lane == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_ready));
#pragma unroll
        for (int n = 0; n < 8; ++n) {
          thr[n] = n < a.G ? __ldcg(&p.hs.thr[bh0 + n]) : 0xFFFFFFFFu;
          shift[n] = n < a.G ? __ldcg(&p.hs.hshift[bh0 + n]) : 0u;
        }
        const int64_t nctx = a.n_ctx[g / a.Hkv];
        int since = 0;
        for (int64_t u = lo; u < hi; ++u, ++i) {
          uint32_t v[16];
          tc_epi_load(t, i, quarter, lane, v, 0);
          tc_epi_emit(v, u * kTcUnit, nctx, quarter, lane, a.G, static_cast<uint32_t>(a.row_offset), thr, wbuf,
                      t.cap, cnt, true);
          if (++since == flush_every) {
            tc_warp_flush(const_cast<uint64_t*>(a.cand), a.cap, p.hs.cand_cnt, p.hs.hist, a.G, bh0, wbuf, t.cap,
                          cnt, thr, shift, lane);
            since = 0;
          }
        }
        tc_warp_flush(const_cast<uint64_t*>(a.cand), a.cap, p.hs.cand_cnt, p.hs.hist, a.G, bh0, wbuf, t.cap, cnt,
                      thr, shift, lane);
      }
      // this warp's share of group g is in HBM: count it towards scan_done(g)
      __threadfence();
      __syncwarp();
      if (lane == 0) atomicAdd(ctl.scan_done(g), 1u);
      if (p.trace && lane == 0) {  // diagnostics: per (group, CTA, epilogue warp) scan window
        const uint32_t slot = sc.pre + blk[sc.nblocks()] + 4096u + (static_cast<uint32_t>(g) * gridDim.x + blockIdx.x) * 4u + ew;
        if (slot < p.trace_cap) {
          uint64_t t_end;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
          uint64_t* r = p.trace + static_cast<uint64_t>(slot) * 4;
          r[0] = t_start;
          r[1] = t_end;
          r[2] = (static_cast<uint64_t>(kItScan) << 32) | blockIdx.x;
          r[3] = (static_cast<uint64_t>(static_cast<uint32_t>(g)) << 32) |
                 static_cast<uint32_t>(t_ready ? (t_ready - t_start) : 0);
        }
      }
    }
  } else {  // work queue
    run_queue<QueueGrp>(p, ctl, sc, blk, work, &s_item);
  }

  tc_fence_before();
  __syncthreads();
  tc_teardown(t.tmem, warp == 1);
  reset_ctl_if_last(p, ctl, &s_last);
}

cudaError_t launch_fused(const FusedParams& p, cudaStream_t s) {
  const int NG = p.a.B * p.a.Hkv;
  const size_t tbl = ((static_cast<size_t>(NG) + 3) * 4 + 15) / 16 * 16;
  const size_t scan_sm = static_cast<size_t>(p.a.G) * kFStage * 8 + 64;
  const size_t thr_sm = (kSamples + 2048 + 32 + 4 + FW) * 4;
  const size_t kth_sm = kHistBins * 4 + kFBkt * 8 + (32 + 4) * 4 + (FW + 2) * 8;
  const size_t att_sm = sizeof(AttSmem);
  size_t work = scan_sm;
  work = thr_sm > work ? thr_sm : work;
  work = kth_sm > work ? kth_sm : work;
  work = att_sm > work ? att_sm : work;
  const size_t smem = tbl + work;
  static int grid_cache[2] = {0, 0};  // (smem, grid)
  if (grid_cache[0] != static_cast<int>(smem)) {
    cudaFuncSetAttribute(fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fused_kernel, FT, smem);
    grid_cache[0] = static_cast<int>(smem);
    grid_cache[1] = sms * (per > 0 ? per : 1);
  }
  fused_kernel<<<grid_cache[1], FT, smem, s>>>(p);
  return cudaGetLastError();
}

// Work-queue shared memory of the tc layer kernel: the fallback scan flushes every iteration.
static size_t ftc_work_bytes(int G) {
  const size_t scan_sm = static_cast<size_t>(G) * kScanRows * 8 + 64;
  const size_t thr_sm = (kSamples + 2048 + 32 + 4 + FW) * 4;
  const size_t kth_sm = kHistBins * 4 + kFBkt * 8 + (32 + 4) * 4 + (FW + 2) * 8;
  const size_t att_sm = sizeof(AttSmem);
  size_t work = scan_sm;
  work = thr_sm > work ? thr_sm : work;
  work = kth_sm > work ? kth_sm : work;
  work = att_sm > work ? att_sm : work;
  return work;
}

bool fused_tc_supported(const FusedParams& p) {
  const int64_t rows = static_cast<int64_t>(p.a.B) * p.a.Hkv * p.a.cache_rows;
  return (reinterpret_cast<uintptr_t>(p.a.kc) & 15u) == 0 && rows < (int64_t(1) << 31) && p.a.G <= 8;
}

cudaError_t launch_fused_tc(FusedParams p, cudaStream_t s) {
  using namespace tc;
  CUtensorMap map;
  if (!make_kmap(p.a.kc, static_cast<int64_t>(p.a.B) * p.a.Hkv * p.a.cache_rows, &map)) return cudaErrorInvalidValue;
  const int NG = p.a.B * p.a.Hkv;
  const size_t tbl = ((static_cast<size_t>(NG) + 3) * 4 + 15) / 16 * 16;
  const size_t work = ftc_work_bytes(p.a.G);
  // scan pipeline: two stages, the largest flush interval (<= 4 units) that fits beside the queue
  TcShape sh{2, kTcMaxFlush};
  size_t tcb = 0;
  for (; sh.flush >= 1; --sh.flush) {
    tcb = (tc_smem_bytes(p.a.G, sh) + 15) / 16 * 16;
    if (tcb + tbl + work <= static_cast<size_t>(kTcSmemLimit)) break;
  }
  if (sh.flush < 1) return cudaErrorInvalidConfiguration;
  const size_t smem = tcb + tbl + work;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(fused_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmemLimit);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(fused_tc_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fused_tc_kernel, kFtcThreads, smem);
  if (per < 1) return cudaErrorInvalidConfiguration;
  p.scan_target = 4 * sms;  // every epilogue warp of every CTA reports each group
  p.scan_flush_iters = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(kFtcThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  // every CTA must be resident (the queue warps wait on other CTAs' scan progress): a
  // cooperative launch guarantees it, or fails instead of hanging; inside stream capture a
  // plain launch of one CTA per SM (the shared memory allows no more) is used
  cudaLaunchAttribute attr_coop[1];
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cap);
  attr_coop[0].id = cudaLaunchAttributeCooperative;
  attr_coop[0].val.cooperative = 1;
  cfg.attrs = attr_coop;
  cfg.numAttrs = cap == cudaStreamCaptureStatusNone ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, fused_tc_kernel, map, p, sh.stages, sh.flush, static_cast<int>(tcb));
}

}  // namespace tkv
