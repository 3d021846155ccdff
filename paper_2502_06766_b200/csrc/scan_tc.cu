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
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdlib.h>

#include "common.cuh"
#include "internal.h"

namespace tkv {
namespace {

constexpr int kTcM = 128;                          // UMMA M: cache rows per MMA sub-tile
constexpr int kTcSub = 2;                          // sub-tiles per unit
constexpr int kTcUnit = kTcM * kTcSub;             // cache rows per pipeline unit
constexpr int kTcN = 8;                            // UMMA N: query rows (G <= 8)
constexpr int kTcKSteps = kD / 16;                 // UMMA K = 16
constexpr int kTcUnitBytes = kTcUnit * kD * 2;     // 64 KB per ring stage
constexpr int kTcHalfBytes = kTcUnitBytes / 2;     // [256 rows × 64 elements]: one swizzle span wide
constexpr int kTcSubBytes = kTcM * 128;            // one sub-tile inside a half
constexpr int kTcMaxStages = 3;
constexpr int kTcAcc = 4;                          // unit accumulators in flight
constexpr int kTcAccCols = kTcSub * kTcN;          // TMEM columns per unit
constexpr uint32_t kTcTmemCols = 64;               // >= kTcAcc * kTcAccCols, power of two >= 32
constexpr int kTcQSlots = kTcAcc;                  // q slots: reuse is safe once kTcAcc units drained
constexpr int kTcQBytes = kTcN * kD * 2;           // 2 KB: one 8-row swizzle atom per half
constexpr int kTcEpiWarps = 4;
constexpr int kTcThreads = 64 + 32 * kTcEpiWarps;
constexpr int kTcWarpRows = kTcUnit / 4;           // rows per unit one epilogue warp handles
constexpr int kTcMaxFlush = 4;  // units between a warp's flushes (flat from 4 to 16; 4 leaves room beside the CTA)
constexpr int kTcSmemLimit = 227 * 1024 - 512;     // opt-in maximum minus the static barriers

static_assert(kTcTmemCols >= kTcAcc * kTcAccCols, "TMEM allocation too small");

// dynamic shared memory: [staging: 4 warps × G × flush·64 × 8 B][q slots][K ring]
struct TcShape {
  int stages, flush;
};
inline int tc_stage_bytes(int G, int flush) { return kTcEpiWarps * G * flush * kTcWarpRows * 8; }
inline TcShape tc_shape(int G) {
  // two stages and the rest of shared memory as staging: measured faster on cfg3 than three
  // stages with 3-unit flushes (fewer flush round trips beat a deeper ring)
  for (int st = 2; st >= 2; --st) {
    const int free_b = kTcSmemLimit - 1024 - kTcQSlots * kTcQBytes - st * kTcUnitBytes;
    int f = free_b / tc_stage_bytes(G, 1);
    if (f > kTcMaxFlush) f = kTcMaxFlush;
    if (f >= 2 || st == 2) return {st, f};
  }
  return {2, 1};
}
inline size_t tc_smem_bytes(int G, const TcShape& sh) {
  return 1024 + ((tc_stage_bytes(G, sh.flush) + 1023) & ~1023) + kTcQSlots * kTcQBytes +
         static_cast<size_t>(sh.stages) * kTcUnitBytes;
}

// ---------------------------------------------------------------- PTX wrappers (sm_100a)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
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

// Warp-private flush of one epilogue warp's staged candidates (all heads of the segment):
// lanes 0..G-1 reserve the heads' output ranges with one global atomic each (one round trip),
// then the warp copies the composites out and adds them to the heads' key histograms.
__device__ __forceinline__ void tc_warp_flush(const ScanParams& p, int64_t bh0, const uint64_t* wbuf, int cap,
                                              uint32_t (&cnt)[8], const uint32_t (&thr)[8],
                                              const uint32_t (&shift)[8], int lane) {
  __syncwarp();
  uint32_t mine = 0;
#pragma unroll
  for (int n = 0; n < 8; ++n)
    if (lane == n) mine = cnt[n];
  uint32_t base = 0;
  if (lane < p.G && mine) base = atomicAdd(&p.hs.cand_cnt[bh0 + lane], mine);
#pragma unroll
  for (int n = 0; n < 8; ++n) {
    if (n >= p.G) break;
    const uint32_t c = cnt[n];
    const uint32_t b = __shfl_sync(kFull, base, n);
    if (c == 0u) continue;
    uint64_t* dst = p.cand + (bh0 + n) * p.cap + b;
    uint32_t* gh = p.hs.hist + (bh0 + n) * kHistBins;
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

__global__ void __launch_bounds__(kTcThreads, 1) scan_tc_kernel(const __grid_constant__ CUtensorMap kmap,
                                                                ScanParams p, int n_stages, int flush_every,
                                                                int mode) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t s_bar[2 * kTcMaxStages + 2 * kTcAcc];
  __shared__ uint32_t s_tmem;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;  // 1024-byte alignment for the swizzle atoms
  uint8_t* gbase = smem_raw + (base - raw);
  const int cap = flush_every * kTcWarpRows;  // staged candidates per (epilogue warp, head)
  const int stage_b = (kTcEpiWarps * p.G * cap * 8 + 1023) & ~1023;
  uint64_t* s_buf = reinterpret_cast<uint64_t*>(gbase);
  const uint32_t sQ = base + stage_b, sA = sQ + kTcQSlots * kTcQBytes;
  const uint32_t bar0 = smem_u32(s_bar);
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (kTcMaxStages + s); };
  auto tfull_bar = [&](int a) { return bar0 + 8u * (2 * kTcMaxStages + a); };
  auto tempty_bar = [&](int a) { return bar0 + 8u * (2 * kTcMaxStages + kTcAcc + a); };

  if (tid == 0) {
    for (int s = 0; s < n_stages; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < kTcAcc; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), kTcEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&kmap)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "n"(kTcTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;

  const int64_t ups = (p.max_ctx + kTcUnit - 1) / kTcUnit;
  const int64_t total = (p.seg_count ? p.seg_count : static_cast<int64_t>(p.B) * p.Hkv) * ups;
  const int64_t ubase = p.seg_begin * ups;  // units of the segment range [seg_begin, +seg_count)
  UnitWalk w;
  w.init(p, ubase + total * blockIdx.x / gridDim.x, ubase + total * (blockIdx.x + 1) / gridDim.x, ups);
  bool new_seg = false;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    for (uint32_t i = 0; w.next(p, new_seg); ++i) {
      const int st = static_cast<int>(i % n_stages);
      const uint32_t ph = (i / n_stages) & 1u;
      mbar_wait(empty_bar(st), ph ^ 1u);
      if (lane == 0 && (mode & 4)) {  // diagnostics: no HBM traffic (MMAs on stale tiles)
        mbar_arrive(full_bar(st));
      } else if (lane == 0) {
        const int grow = static_cast<int>(w.cur_seg * p.cache_rows + w.cur_row0);
        mbar_expect_tx(full_bar(st), kTcUnitBytes);
        tma_load_2d(sA + st * kTcUnitBytes, &kmap, 0, grow, full_bar(st));
        tma_load_2d(sA + st * kTcUnitBytes + kTcHalfBytes, &kmap, 64, grow, full_bar(st));
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    int slot = -1;
    for (uint32_t i = 0; w.next(p, new_seg); ++i) {
      const int st = static_cast<int>(i % n_stages);
      const uint32_t ph = (i / n_stages) & 1u;
      const int acc = static_cast<int>(i % kTcAcc);
      const uint32_t aph = (i / kTcAcc) & 1u;
      mbar_wait(tempty_bar(acc), aph ^ 1u);  // accumulator drained: MMAs of units <= i-kTcAcc done
      if (new_seg) {
        // query rows of the GQA group → next slot; its previous user is >= kTcQSlots units back,
        // so its MMAs completed (drained above)
        slot = (slot + 1) % kTcQSlots;
        const __nv_bfloat16* qg = p.q + (static_cast<int64_t>(w.cur_b) * p.Hq + w.cur_kvh * p.G) * kD;
        uint8_t* qs = gbase + stage_b + slot * kTcQBytes;
        // 8 rows × 16 chunks of 16 bytes; chunk (h, j) of row n at h·1024 + n·128 + (j ^ n)·16
        for (int e = lane; e < kTcN * 16; e += 32) {
          const int n = e >> 4, cj = e & 15, h = cj >> 3, j = cj & 7;
          uint4 v = make_uint4(0u, 0u, 0u, 0u);
          if (n < p.G) v = *reinterpret_cast<const uint4*>(qg + n * kD + cj * 8);
          *reinterpret_cast<uint4*>(qs + h * (kTcQBytes / 2) + n * 128 + ((j ^ n) << 4)) = v;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
      }
      mbar_wait(full_bar(st), ph);
      tc_fence_after();
      if (lane == 0 && (mode & 1)) {  // diagnostics: TMA stream only
        mbar_arrive(empty_bar(st));
        mbar_arrive(tfull_bar(acc));
      } else if (lane == 0) {
        const uint64_t qd = sw128_desc(sQ + slot * kTcQBytes);
        const uint64_t kd = sw128_desc(sA + st * kTcUnitBytes);
#pragma unroll
        for (int u = 0; u < kTcSub; ++u) {
#pragma unroll
          for (int kk = 0; kk < kTcKSteps; ++kk) {
            const int h = kk >> 2, k4 = kk & 3;  // 64-element half, 16-element step inside it
            const uint32_t koff = (h * kTcHalfBytes + u * kTcSubBytes + k4 * 32) >> 4;
            const uint32_t qoff = (h * (kTcQBytes / 2) + k4 * 32) >> 4;
            umma_bf16(tmem + acc * kTcAccCols + u * kTcN, kd + koff, qd + qoff, kIdesc, kk > 0 ? 1u : 0u);
          }
        }
        umma_commit(empty_bar(st));
        umma_commit(tfull_bar(acc));
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 2;
    const int quarter = warp & 3;  // TMEM lanes this warp may access: [32·quarter, +32)
    uint64_t* wbuf = s_buf + static_cast<int64_t>(ew) * p.G * cap;
    uint32_t thr[8], shift[8], cnt[8];
#pragma unroll
    for (int n = 0; n < 8; ++n) cnt[n] = thr[n] = shift[n] = 0u;
    int since = 0;
    int64_t bh0 = -1;
    const unsigned lt = lanemask_lt();
    for (uint32_t i = 0; w.next(p, new_seg); ++i) {
      if (new_seg) {
        if (bh0 >= 0) tc_warp_flush(p, bh0, wbuf, cap, cnt, thr, shift, lane);
        since = 0;
        bh0 = static_cast<int64_t>(w.cur_b) * p.Hq + w.cur_kvh * p.G;
#pragma unroll
        for (int n = 0; n < 8; ++n) {
          thr[n] = n < p.G ? p.hs.thr[bh0 + n] : 0xFFFFFFFFu;
          shift[n] = n < p.G ? p.hs.hshift[bh0 + n] : 0u;
        }
      }
      const int acc = static_cast<int>(i % kTcAcc);
      const uint32_t aph = (i / kTcAcc) & 1u;
      mbar_wait(tfull_bar(acc), aph);
      tc_fence_after();
      uint32_t v[16];
      if (!(mode & 1)) {
        tmem_ld16(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + acc * kTcAccCols, v);
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0u;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty_bar(acc));
#pragma unroll
      for (int u = 0; u < kTcSub; ++u) {
        const int64_t row = w.cur_row0 + u * kTcM + quarter * 32 + lane;
        const bool live = row < w.cur_nctx && !(mode & 3);  // diagnostics never emit
        const uint32_t rid = p.row_offset + static_cast<uint32_t>(row);
        uint64_t* ub = wbuf + (u * 32);  // rows of sub-tile u follow those of sub-tile 0 in order
#pragma unroll
        for (int n = 0; n < 8; ++n) {
          if (n >= p.G) break;
          const uint32_t key = score_key(__uint_as_float(v[u * kTcN + n]));
          const bool pass = live && key >= thr[n];
          const unsigned m = __ballot_sync(kFull, pass);
          if (pass) ub[n * cap + cnt[n] + __popc(m & lt) - u * 32] = make_comp(key, rid);
          cnt[n] += __popc(m);
        }
      }
      if (++since == flush_every) {
        tc_warp_flush(p, bh0, wbuf, cap, cnt, thr, shift, lane);
        since = 0;
      }
    }
    if (bh0 >= 0) tc_warp_flush(p, bh0, wbuf, cap, cnt, thr, shift, lane);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTcTmemCols)
                 : "memory");
  }
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
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(kD),
                              static_cast<cuuint64_t>(p.B) * p.Hkv * static_cast<cuuint64_t>(p.cache_rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(kD) * 2};
  const cuuint32_t box[2] = {64, kTcUnit};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16*>(p.kc), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  static const int mode = [] {  // diagnostics: bit 0 = no MMA, bit 1 = no emission, bit 2 = no TMA
    const char* e = getenv("TKV_TC_MODE");
    return e ? atoi(e) : 0;
  }();
  static const int stages_env = [] {  // experiments: force the ring depth (2 or 3)
    const char* e = getenv("TKV_TC_STAGES");
    return e ? atoi(e) : 0;
  }();
  static const int flush_env = [] {  // experiments: cap the units between flushes
    const char* e = getenv("TKV_TC_FLUSH");
    return e ? atoi(e) : 0;
  }();
  TcShape sh = tc_shape(p.G);
  if (stages_env >= 2 && stages_env <= kTcMaxStages && stages_env != sh.stages) {
    sh.stages = stages_env;
    const int free_b = kTcSmemLimit - 1024 - kTcQSlots * kTcQBytes - sh.stages * kTcUnitBytes;
    sh.flush = free_b / tc_stage_bytes(p.G, 1);
    if (sh.flush > kTcMaxFlush) sh.flush = kTcMaxFlush;
    if (sh.flush < 1) return cudaErrorInvalidValue;
  }
  if (flush_env > 0 && flush_env < sh.flush) sh.flush = flush_env;
  const size_t smem = tc_smem_bytes(p.G, sh);
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(scan_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmemLimit);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(scan_tc_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  static const int sms = [] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  int grid = sms;
  if (total < grid) grid = static_cast<int>(total);
  scan_tc_kernel<<<grid, kTcThreads, smem, s>>>(map, p, sh.stages, sh.flush, mode);
  return cudaGetLastError();
}

}  // namespace tkv
