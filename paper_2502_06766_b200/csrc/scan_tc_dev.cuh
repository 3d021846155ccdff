// scan_tc_dev.cuh — building blocks of the TMA + tcgen05 key scan (see scan_tc.cu for the
// pipeline): constants, PTX wrappers, the per-CTA pipeline state (mbarrier ring, TMEM
// accumulators, q slots, warp-private candidate staging) and the per-unit steps of the three
// roles, used by scan_tc_kernel (scan_tc.cu).
#pragma once

#include <cuda.h>

#include "common.cuh"
#include "internal.h"

namespace tkv {
namespace tc {


constexpr int kTcM = 128;                          // UMMA M: cache rows per MMA sub-tile
constexpr int kTcSub = 2;                          // sub-tiles per unit
constexpr int kTcUnit = kTcM * kTcSub;             // cache rows per pipeline unit
constexpr int kTcN = 8;                            // UMMA N: query rows (G <= 8)
constexpr int kTcKSteps = kD / 16;                 // UMMA K = 16
constexpr int kTcUnitBytes = kTcUnit * kD * 2;     // 64 KB per ring stage
constexpr int kTcHalfBytes = kTcUnitBytes / 2;     // [256 rows × 64 elements]: one swizzle span wide
constexpr int kTcSubBytes = kTcM * 128;            // one sub-tile inside a half
constexpr int kTcMaxStages = 3;
// TMEM is a deep score buffer: 32 units (8192 rows per SM, ~45 us of streaming) may be scored
// before the epilogue drains them, so the TMA/MMA stream keeps going while the epilogue still
// waits for the candidate thresholds (threshold_kernel overlaps the scan through PDL)
#ifndef TKV_TC_ACC
#define TKV_TC_ACC 32
#endif
constexpr int kTcAcc = TKV_TC_ACC;                 // unit accumulators in flight
constexpr int kTcAccCols = kTcSub * kTcN;          // TMEM columns per unit
constexpr uint32_t kTcTmemCols = kTcAcc * kTcAccCols <= 32 ? 32 : kTcAcc * kTcAccCols;  // power of two
static_assert((kTcTmemCols & (kTcTmemCols - 1)) == 0 && kTcTmemCols <= 512, "TMEM columns");
constexpr int kTcQSlots = 4;                       // q slots, each released by a tcgen05.commit
constexpr int kTcQBytes = kTcN * kD * 2;           // 2 KB: one 8-row swizzle atom per half
constexpr int kTcEpiWarps = 4;                     // epilogue warps per unit (one per TMEM lane quarter)
constexpr int kTcScanGroups = 2;                   // scan_tc_kernel: two groups alternate units
constexpr int kTcScanThreads = 64 + 32 * kTcEpiWarps * kTcScanGroups;
constexpr int kTcWarpRows = kTcUnit / 4;           // rows per unit one epilogue warp handles
constexpr int kTcMaxFlush = 4;  // units between a warp's flushes (flat from 4 to 16; 4 leaves room beside the CTA)
constexpr int kTcSmemLimit = 227 * 1024 - 1024;    // opt-in maximum minus the static barriers (<= 1 KB)

static_assert(kTcTmemCols >= kTcAcc * kTcAccCols, "TMEM allocation too small");

// dynamic shared memory: [staging: 4 warps × G × flush·64 × 8 B][q slots][K ring]
struct TcShape {
  int stages, flush;
};
// staging: every epilogue warp (4 per group) holds flush units' worth of rows per head
inline int tc_stage_bytes(int G, int flush, int groups = 1) { return groups * kTcEpiWarps * G * flush * kTcWarpRows * 8; }
inline TcShape tc_shape(int G, int groups = 1) {
  // two stages and the rest of shared memory as staging: measured faster on cfg3 than three
  // stages with 3-unit flushes (fewer flush round trips beat a deeper ring)
  for (int st = 2; st >= 2; --st) {
    const int free_b = kTcSmemLimit - 1024 - kTcQSlots * kTcQBytes - st * kTcUnitBytes;
    int f = free_b / tc_stage_bytes(G, 1, groups);
    // own units between a warp's flushes: 4 with one group; 2 with two (the same rows per flush,
    // and the staging stays small enough for the k-th / gather kernels to share the SM)
    const int fmax = kTcMaxFlush / groups;
    if (f > fmax) f = fmax;
    if (f >= 2 || st == 2) return {st, f};
  }
  return {2, 1};
}
inline size_t tc_smem_bytes(int G, const TcShape& sh, int groups = 1) {
  return 1024 + ((tc_stage_bytes(G, sh.flush, groups) + 1023) & ~1023) + kTcQSlots * kTcQBytes +
         static_cast<size_t>(sh.stages) * kTcUnitBytes;
}

// ---------------------------------------------------------------- PTX wrappers (sm_100a)
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
// the same with an L2 eviction-priority policy (createpolicy): the K stream is read exactly
// once, so it goes in evict-first and does not push the candidates, histograms, per-head state
// and the later kernels' code out of L2
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_2d_hint(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
// one row (TMEM lane) × 16 consecutive 32-bit columns per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UMMA shared-memory descriptor, K-major operand with the 128-byte swizzle: rows of 128 bytes,
// 8-row atoms of 1024 bytes (stride byte offset), descriptor version 1 (sm_100).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);  // start address
  d |= static_cast<uint64_t>(1u) << 16;                // leading byte offset (unused for SW128 K-major)
  d |= static_cast<uint64_t>(1024u >> 4) << 32;        // stride byte offset: next 8-row atom
  d |= static_cast<uint64_t>(1u) << 46;                // version
  d |= static_cast<uint64_t>(2u) << 61;                // layout: SWIZZLE_128B
  return d;
}
// instruction descriptor: kind::f16, A/B bf16 K-major, D f32, M = 128, N = 8
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(kTcN >> 3) << 17) |
                            (static_cast<uint32_t>(kTcM >> 4) << 24);


// Per-CTA pipeline state. Dynamic shared memory: [staging: 4 warps × G × cap × 8 B]
// [q slots][K ring], the last two 1024-byte aligned.
struct TcPipe {
  uint32_t sA, sQ, bar0, tmem;
  uint8_t* q_generic;  // generic pointer of the q slots (written by the MMA warp)
  uint64_t* s_buf;     // staging
  int n_stages, cap;
  __device__ __forceinline__ uint32_t full(int s) const { return bar0 + 8u * s; }
  __device__ __forceinline__ uint32_t empty(int s) const { return bar0 + 8u * (kTcMaxStages + s); }
  __device__ __forceinline__ uint32_t tfull(int a) const { return bar0 + 8u * (2 * kTcMaxStages + a); }
  __device__ __forceinline__ uint32_t tempty(int a) const { return bar0 + 8u * (2 * kTcMaxStages + kTcAcc + a); }
  __device__ __forceinline__ uint32_t qfree(int s) const { return bar0 + 8u * (2 * kTcMaxStages + 2 * kTcAcc + s); }
};
constexpr int kTcBarWords = 2 * kTcMaxStages + 2 * kTcAcc + kTcQSlots;

// Lays out the pipeline in `smem_raw` (dynamic shared memory) and, on the calling threads,
// initialises it: thread `init_tid` the barriers, warp `alloc_warp` the TMEM accumulators. All
// threads of the CTA must then pass tc_fence_before(); __syncthreads(); tc_fence_after(); and
// read the TMEM base with tc_tmem_base().
__device__ __forceinline__ TcPipe tc_setup(uint8_t* smem_raw, uint64_t* s_bar, uint32_t* s_tmem, int G,
                                           int flush_every, int n_stages, const CUtensorMap* kmap,
                                           bool init_thread, bool alloc_warp, int groups = 1) {
  TcPipe t;
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;  // 1024-byte alignment for the swizzle atoms
  uint8_t* gbase = smem_raw + (base - raw);
  t.cap = flush_every * kTcWarpRows;
  const int stage_b = (groups * kTcEpiWarps * G * t.cap * 8 + 1023) & ~1023;
  t.s_buf = reinterpret_cast<uint64_t*>(gbase);
  t.sQ = base + stage_b;
  t.sA = t.sQ + kTcQSlots * kTcQBytes;
  t.q_generic = gbase + stage_b;
  t.bar0 = smem_u32(s_bar);
  t.n_stages = n_stages;
  t.tmem = 0;
  if (init_thread) {
    for (int s = 0; s < n_stages; ++s) {
      mbar_init(t.full(s), 1);
      mbar_init(t.empty(s), 1);
    }
    for (int a = 0; a < kTcAcc; ++a) {
      mbar_init(t.tfull(a), 1);
      mbar_init(t.tempty(a), kTcEpiWarps);
    }
    for (int q = 0; q < kTcQSlots; ++q) mbar_init(t.qfree(q), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(kmap)) : "memory");
  }
  if (alloc_warp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                 "n"(kTcTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  return t;
}

__device__ __forceinline__ void tc_teardown(uint32_t tmem, bool alloc_warp) {
  if (alloc_warp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTcTmemCols)
                 : "memory");
  }
}

// producer, whole warp: unit i (64 KB: rows [grow, grow + 256) of the 2-D K view) → ring stage
__device__ __forceinline__ void tc_produce(const TcPipe& t, uint32_t i, const CUtensorMap* kmap, int grow, int lane,
                                           int mode) {
  const int st = static_cast<int>(i % t.n_stages);
  const uint32_t ph = (i / t.n_stages) & 1u;
  mbar_wait(t.empty(st), ph ^ 1u);
  if (lane == 0 && (mode & 4)) {  // diagnostics: no HBM traffic (MMAs on stale tiles)
    mbar_arrive(t.full(st));
  } else if (lane == 0) {
    mbar_expect_tx(t.full(st), kTcUnitBytes);
#ifndef TKV_TC_NO_EVICT_FIRST
    const uint64_t pol = l2_evict_first_policy();
    tma_load_2d_hint(t.sA + st * kTcUnitBytes, kmap, 0, grow, t.full(st), pol);
    tma_load_2d_hint(t.sA + st * kTcUnitBytes + kTcHalfBytes, kmap, 64, grow, t.full(st), pol);
#else
    tma_load_2d(t.sA + st * kTcUnitBytes, kmap, 0, grow, t.full(st));
    tma_load_2d(t.sA + st * kTcUnitBytes + kTcHalfBytes, kmap, 64, grow, t.full(st));
#endif
  }
  __syncwarp();
}

// MMA warp, step 1 of unit i: wait until accumulator i % kTcAcc is drained by the epilogue
__device__ __forceinline__ void tc_mma_acquire(const TcPipe& t, uint32_t i) {
  mbar_wait(t.tempty(static_cast<int>(i % kTcAcc)), ((i / kTcAcc) & 1u) ^ 1u);
}

// MMA warp: the GQA group's query rows → q slot (B operand, 8 rows, rows >= G zero), in the
// 128-byte-swizzled K-major layout: chunk (h, j) of row n at h·1024 + n·128 + (j ^ n)·16.
// Prefer tc_next_q, which also manages the slot's release.
__device__ __forceinline__ void tc_load_q(const TcPipe& t, int slot, const __nv_bfloat16* qg, int G, int lane) {
  uint8_t* qs = t.q_generic + slot * kTcQBytes;
  for (int e = lane; e < kTcN * 16; e += 32) {
    const int n = e >> 4, cj = e & 15, h = cj >> 3, j = cj & 7;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (n < G) v = *reinterpret_cast<const uint4*>(qg + n * kD + cj * 8);
    *reinterpret_cast<uint4*>(qs + h * (kTcQBytes / 2) + n * 128 + ((j ^ n) << 4)) = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
}

// The MMA warp's q-slot ring. Switching to a new segment releases the current slot with a
// tcgen05.commit on qfree[slot] (it fires once every MMA that read the slot has completed);
// a slot is rewritten only after its previous release fired.
struct QRing {
  int slot = -1;
  uint32_t used = 0;    // bit s: slot s has been used before
  uint32_t parity = 0;  // bit s: phase parity of slot s's next release
};
__device__ __forceinline__ void tc_next_q(const TcPipe& t, QRing& r, const __nv_bfloat16* qg, int G, int lane) {
  if (r.slot >= 0 && lane == 0) umma_commit(t.qfree(r.slot));
  r.slot = (r.slot + 1) % kTcQSlots;
  const uint32_t bit = 1u << r.slot;
  if (r.used & bit) {
    mbar_wait(t.qfree(r.slot), (r.parity & bit) ? 1u : 0u);
    r.parity ^= bit;
  }
  r.used |= bit;
  tc_load_q(t, r.slot, qg, G, lane);
}

// MMA warp, step 2 of unit i: wait for the tile, one lane issues 2 sub-tiles × 8 K-steps, then
// commits the stage (to the producer) and the accumulator (to the epilogue)
__device__ __forceinline__ void tc_mma_issue(const TcPipe& t, uint32_t i, int slot, int lane, int mode) {
  const int st = static_cast<int>(i % t.n_stages);
  const int acc = static_cast<int>(i % kTcAcc);
  mbar_wait(t.full(st), (i / t.n_stages) & 1u);
  tc_fence_after();
  if (lane == 0 && (mode & 1)) {  // diagnostics: TMA stream only
    mbar_arrive(t.empty(st));
    mbar_arrive(t.tfull(acc));
  } else if (lane == 0) {
    const uint64_t qd = sw128_desc(t.sQ + slot * kTcQBytes);
    const uint64_t kd = sw128_desc(t.sA + st * kTcUnitBytes);
#pragma unroll
    for (int u = 0; u < kTcSub; ++u) {
#pragma unroll
      for (int kk = 0; kk < kTcKSteps; ++kk) {
        const int h = kk >> 2, k4 = kk & 3;  // 64-element half, 16-element step inside it
        const uint32_t koff = (h * kTcHalfBytes + u * kTcSubBytes + k4 * 32) >> 4;
        const uint32_t qoff = (h * (kTcQBytes / 2) + k4 * 32) >> 4;
        umma_bf16(t.tmem + acc * kTcAccCols + u * kTcN, kd + koff, qd + qoff, kIdesc, kk > 0 ? 1u : 0u);
      }
    }
    umma_commit(t.empty(st));
    umma_commit(t.tfull(acc));
  }
  __syncwarp();
}

// epilogue warp (TMEM lane quarter `quarter`): unit i's scores → v[u·8 + n] = sub-tile u, head n
// of row quarter·32 + lane; releases the accumulator
__device__ __forceinline__ void tc_epi_load(const TcPipe& t, uint32_t i, int quarter, int lane, uint32_t (&v)[16],
                                            int mode) {
  const int acc = static_cast<int>(i % kTcAcc);
  mbar_wait(t.tfull(acc), (i / kTcAcc) & 1u);
  tc_fence_after();
  if (!(mode & 1)) {
    tmem_ld16(t.tmem + (static_cast<uint32_t>(quarter * 32) << 16) + acc * kTcAccCols, v);
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = 0u;
  }
  tc_fence_before();
  __syncwarp();
  if (lane == 0) mbar_arrive(t.tempty(acc));
}

// epilogue warp: threshold test of the unit's rows, warp-aggregated append to the warp's
// staging (counts in registers; en = per-head emission mask)
__device__ __forceinline__ void tc_epi_emit(const uint32_t (&v)[16], int64_t row0, int64_t nctx, int quarter,
                                            int lane, int G, uint32_t row_offset, const uint32_t (&thr)[8],
                                            uint64_t* wbuf, int cap, uint32_t (&cnt)[8], bool emit) {
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int u = 0; u < kTcSub; ++u) {
    const int64_t row = row0 + u * kTcM + quarter * 32 + lane;
    const bool live = emit && row < nctx;
    const uint32_t rid = row_offset + static_cast<uint32_t>(row);
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      if (n >= G) break;
      const uint32_t key = score_key(__uint_as_float(v[u * kTcN + n]));
      const bool pass = live && key >= thr[n];
      const unsigned m = __ballot_sync(kFull, pass);
      if (pass) wbuf[n * cap + cnt[n] + __popc(m & lt)] = make_comp(key, rid);
      cnt[n] += __popc(m);
    }
  }
}

// Warp-private flush of one epilogue warp's staged candidates (all heads bh0 .. bh0+G-1):
// lanes 0..G-1 reserve the heads' output ranges with one global atomic each (one round trip),
// then the warp copies the composites out and adds them to the heads' key histograms.
__device__ __forceinline__ void tc_warp_flush(uint64_t* cand, int64_t cand_cap, uint32_t* cand_cnt, uint32_t* hist,
                                              int G, int64_t bh0, const uint64_t* wbuf, int cap,
                                              uint32_t (&cnt)[8], const uint32_t (&thr)[8],
                                              const uint32_t (&shift)[8], int lane) {
  __syncwarp();
  uint32_t mine = 0;
#pragma unroll
  for (int n = 0; n < 8; ++n)
    if (lane == n) mine = cnt[n];
  uint32_t base = 0;
  if (lane < G && mine) base = atomicAdd(&cand_cnt[bh0 + lane], mine);
#pragma unroll
  for (int n = 0; n < 8; ++n) {
    if (n >= G) break;
    const uint32_t c = cnt[n];
    const uint32_t b = __shfl_sync(kFull, base, n);
    if (c == 0u) continue;
    uint64_t* dst = cand + (bh0 + n) * cand_cap + b;
    uint32_t* gh = hist + (bh0 + n) * kHistBins;
    const uint64_t* src = wbuf + n * cap;
    for (uint32_t i = lane; i < c; i += 32) {
      const uint64_t cc = src[i];
      dst[i] = cc;
      const uint32_t d = hist_digit(comp_key(cc), thr[n], shift[n]);
      const unsigned peers = __match_any_sync(__activemask(), d);
      if (lane == static_cast<int>(__ffs(peers) - 1)) atomicAdd(&gh[d], __popc(peers));
    }
    cnt[n] = 0u;
  }
  __syncwarp();
}

// host: the K cache [B, Hkv, cache_rows, 128] bf16 as a 2-D TMA tensor of B·Hkv·cache_rows rows
bool make_kmap(const __nv_bfloat16* kc, int64_t rows, CUtensorMap* map);

}  // namespace tc
}  // namespace tkv
