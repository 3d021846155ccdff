// scan_dev.cuh — the key-scan loop (see scan.cu), shared by the host-launched scan kernel
// (scan.cu) and the device-tail-launched exactness fallback (select.cu).
#pragma once

#include "common.cuh"
#include "internal.h"

namespace tkv {
namespace {
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
      if (lane == 0) base = atomicAdd(&p.hs.cand_cnt[bh], cnt);
      base = __shfl_sync(kFull, base, 0);
      const uint32_t thr = p.hs.thr[bh], shift = p.hs.hshift[bh];
      uint32_t* gh = p.hs.hist + bh * kHistBins;
      uint64_t* dst = p.cand + bh * p.cap + base;
      const uint64_t* src = s_buf + warp * kScanStage;
      for (uint32_t i = lane; i < cnt; i += 32) {
        const uint64_t cc = src[i];
        dst[i] = cc;
        const uint32_t d = hist_digit(comp_key(cc), thr, shift);
        const unsigned peers = __match_any_sync(__activemask(), d);
        if (lane == static_cast<int>(__ffs(peers) - 1)) atomicAdd(&gh[d], __popc(peers));
      }
    }
    if (lane == 0) s_cnt[warp] = 0u;
  }
  __syncthreads();
}

__device__ __forceinline__ void scan_body(const ScanParams& p, uint64_t* s_buf, uint32_t* s_cnt) {

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, c = lane & 3;
  const int64_t tps = (p.max_ctx + kScanRows - 1) / kScanRows;
  const int64_t nseg = p.seg_count ? p.seg_count : static_cast<int64_t>(p.B) * p.Hkv;
  const int64_t total = nseg * tps;
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
    const int64_t lseg = t / tps;  // segment index inside [seg_begin, seg_begin + nseg)
    const int64_t seg = p.seg_begin + lseg;
    if (seg != st.seg) {
      if (st.seg >= 0) scan_flush(p, st, s_buf, s_cnt, warp, lane);
      since = 0;
      st.seg = seg;
      st.b = static_cast<int>(seg / p.Hkv);
      st.kvh = static_cast<int>(seg % p.Hkv);
      st.nctx = p.n_ctx[st.b];
      st.active = !p.fallback || p.hs.group_fail[seg] != 0u;
      if (!st.active) {
        t = (lseg + 1) * tps - 1;  // skip the rest of this segment (CTA-uniform)
        continue;
      }
      load_qfrag(f, p.q + (static_cast<int64_t>(st.b) * p.Hq + st.kvh * p.G) * kD, p.G, lane);
      kbase = p.kc + (static_cast<int64_t>(st.b) * p.Hkv + st.kvh) * p.cache_rows * kD;
      const int64_t bh0 = static_cast<int64_t>(st.b) * p.Hq + st.kvh * p.G;
      en0 = col0 < p.G && (!p.fallback || p.hs.flag_fail[bh0 + col0] != 0u);
      en1 = col1 < p.G && (!p.fallback || p.hs.flag_fail[bh0 + col1] != 0u);
      thr0 = col0 < p.G ? p.hs.thr[bh0 + col0] : 0u;
      thr1 = col1 < p.G ? p.hs.thr[bh0 + col1] : 0u;
    }
    const int64_t tile = t - lseg * tps;
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

}  // namespace
}  // namespace tkv
