// attend_dev.cuh — device pieces of the V gather + softmax (attention.py:158-167, 107-122),
// shared by attend.cu and select.cu (head kernel, exactness-fallback gather).
#pragma once

#include <math.h>

#include "common.cuh"
#include "internal.h"

namespace tkv {
namespace {
constexpr int NT = kAttendThreads;
constexpr int NW = NT / 32;

// Online softmax accumulation over local rows [r_begin, r_end) of kv head (b, kvh) for q head
// h. State (m, l, o) in the log2-scaled domain; thread t holds o for d = t % 128 (the two
// halves t / 128 are summed by the caller). With `skip` (a bitmask over local rows), a row
// whose bit is set — it is among the selected top-k — is skipped. Per 128-row block: the rows are scored with the scan's
// HMMA tile (bit-identical scores), weighted once per row, and their V rows gathered 16 bytes
// per lane with 8 rows in flight per half-warp; s_red: NW × 128 floats.
template <class Gp = CtaGrp>
__device__ void accumulate_rows(const AttendParams& p, int b, int h, int kvh, int64_t r_begin,
                                int64_t r_end, const uint32_t* skip, float& m, float& l,
                                float& o, float* s_z, float* s_scr, float* s_red) {
  const int tid = Gp::tid(), lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, c = lane & 3;
  const int half = lane >> 4, part = lane & 15;
  const int n = h - kvh * p.G;
  const float zs = p.scale * kLog2e;
  QFrag f;
  load_qfrag(f, p.q + (static_cast<int64_t>(b) * p.Hq + kvh * p.G) * kD, p.G, lane);
  const int64_t head_off = (static_cast<int64_t>(b) * p.Hkv + kvh) * p.cache_rows * kD;
  const __nv_bfloat16* kb = p.kc + head_off;
  const __nv_bfloat16* vb = p.vc + head_off + part * 8;
  float acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = 0.f;
  float mrun = m, lrun = 0.f;  // acc and lrun are relative to mrun (rows of this call only)
  for (int64_t base = r_begin; base < r_end; base += 8 * 16) {
    {
      const int64_t rA = base + warp * 16 + g, rB = rA + 8;
      uint4 a[2][4];
      load_tile(a, kb + rA * kD, rA < r_end, kb + rB * kD, rB < r_end, c);
      float sc[4];
      score_tile(sc, a, f);
      if (c == (n >> 1)) {
        const float sA = sc[n & 1], sB = sc[2 + (n & 1)];
        bool okA = rA < r_end, okB = rB < r_end;
        if (skip) {
          okA = okA && !((__ldcg(&skip[rA >> 5]) >> (rA & 31)) & 1u);
          okB = okB && !((__ldcg(&skip[rB >> 5]) >> (rB & 31)) & 1u);
        }
        s_z[warp * 16 + g] = okA ? sA * zs : -INFINITY;
        s_z[warp * 16 + g + 8] = okB ? sB * zs : -INFINITY;
      }
    }
    Gp::sync();
    float v = tid < 128 ? s_z[tid] : -INFINITY;
    v = warp_max(v);
    if (lane == 0) s_scr[warp] = v;
    Gp::sync();
    float cm = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) cm = fmaxf(cm, s_scr[w]);
    const float mn = fmaxf(mrun, cm);
    if (mn != -INFINITY) {  // block-uniform
      const float fold = (mrun == -INFINITY) ? 0.f : exp2f(mrun - mn);
      if (tid < 128) {  // weights, once per row, in place
        const float z = s_z[tid];
        const float w = z == -INFINITY ? 0.f : exp2f(z - mn);
        s_z[tid] = w;
        const float ws = warp_sum(w);
        if (lane == 0) s_scr[8 + warp] = ws;
      }
      Gp::sync();
      const float lsum = s_scr[8] + s_scr[9] + s_scr[10] + s_scr[11];
      uint4 vv[8];
      float wt[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int r = warp * 16 + 2 * u + half;
        wt[u] = s_z[r];
        vv[u] = wt[u] != 0.f ? ldg_stream(vb + (base + r) * kD) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] *= fold;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        acc[0] = fmaf(wt[u], bf16lo(vv[u].x), acc[0]);
        acc[1] = fmaf(wt[u], bf16hi(vv[u].x), acc[1]);
        acc[2] = fmaf(wt[u], bf16lo(vv[u].y), acc[2]);
        acc[3] = fmaf(wt[u], bf16hi(vv[u].y), acc[3]);
        acc[4] = fmaf(wt[u], bf16lo(vv[u].z), acc[4]);
        acc[5] = fmaf(wt[u], bf16hi(vv[u].z), acc[5]);
        acc[6] = fmaf(wt[u], bf16lo(vv[u].w), acc[6]);
        acc[7] = fmaf(wt[u], bf16hi(vv[u].w), acc[7]);
      }
      lrun = lrun * fold + lsum;
      mrun = mn;
    }
    Gp::sync();
  }
  if (mrun == -INFINITY) return;  // no row of the range contributes
  // per-lane partial sums → per-dimension totals (thread d of parity 0 takes the whole sum)
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] += __shfl_xor_sync(kFull, acc[j], 16);
  if (half == 0) {
#pragma unroll
    for (int j = 0; j < 8; ++j) s_red[warp * kD + part * 8 + j] = acc[j];
  }
  Gp::sync();
  const int d = tid & (kD - 1);
  float tot = 0.f;
  if (tid < kD) {
#pragma unroll
    for (int w = 0; w < NW; ++w) tot += s_red[w * kD + d];
  }
  const float F = (m == -INFINITY) ? 0.f : exp2f(m - mrun);
  o = o * F + tot;
  l = l * F + lrun;
  m = mrun;
  Gp::sync();
}

// Pinned-prefix rows [0, p) that the top-k did not select join the context softmax
// (attention.py:152-154 unions them into the retrieved ids). Local rows of this shard only.
template <class Gp = CtaGrp>
__device__ void add_pinned(const AttendParams& p, int b, int h, int kvh, int64_t nctx, int kb,
                           float zref, float& l, float& o, float* s_z, float* s_scr, float* s_red) {
  if (p.pinned <= 0 || kb <= 0) return;
  int64_t lo = -p.row_offset;
  if (lo < 0) lo = 0;
  int64_t hi = static_cast<int64_t>(p.pinned) - p.row_offset;
  if (hi > nctx) hi = nctx;
  if (hi <= lo) return;
  const int bh = b * p.Hq + h;
  float m = zref;
  // rows the top-k selected are marked in pin_mask by the gather / filter pass
  accumulate_rows<Gp>(p, b, h, kvh, lo, hi, p.pin_mask + static_cast<int64_t>(bh) * p.pin_words, m, l, o, s_z,
                      s_scr, s_red);
  // every unselected row scores <= the k-th selected score <= M, so m stays zref
}

// Window rows + normalisation. Inputs: context state (zref, l_c, o_c) where o_c is this
// thread's share (d = tid % 128, parity tid / 128). Writes out[bh, :].
template <class Gp = CtaGrp>
__device__ void finalize_head(const AttendParams& p, int b, int h, int kvh, int64_t nctx, float zref,
                              float l_c, float o_c, float* s_z, float* s_scr, float* s_o, float* s_red) {
  const int tid = Gp::tid();
  const int bh = b * p.Hq + h;
  // precondition n_ctx + n_win <= cache_rows (tkv.h); a window past the cache is clamped
  // rather than read from the next head's rows
  int64_t nwin = p.n_win ? p.n_win[b] : 0;
  if (nwin > p.cache_rows - nctx) nwin = p.cache_rows - nctx;
  float m_w = -INFINITY, l_w = 0.f, o_w = 0.f;
  if (nwin > 0)
    accumulate_rows<Gp>(p, b, h, kvh, nctx, nctx + nwin, nullptr, m_w, l_w, o_w, s_z, s_scr, s_red);
  float val;
  if (p.combine == 0) {  // joint (attention.py:109-114)
    const float mm = fmaxf(l_c > 0.f ? zref : -INFINITY, m_w);
    const float fc = (l_c > 0.f) ? exp2f(zref - mm) : 0.f;
    const float fw = (l_w > 0.f) ? exp2f(m_w - mm) : 0.f;
    const float L = l_c * fc + l_w * fw;
    val = L > 0.f ? (o_c * fc + o_w * fw) / L : 0.f;
  } else {  // additive (attention.py:115-121)
    val = (l_c > 0.f ? o_c / l_c : 0.f) + (l_w > 0.f ? o_w / l_w : 0.f);
  }
  s_o[tid] = val;
  Gp::sync();
  if (tid < kD) p.out[static_cast<int64_t>(bh) * kD + tid] = s_o[tid] + s_o[tid + kD];
}

// a selected row inside the pinned prefix: mark it so the pinned pass does not add it again
__device__ __forceinline__ void mark_pinned(const AttendParams& p, int bh, int64_t local) {
  if (p.pin_mask && local >= 0 && local < static_cast<int64_t>(p.pin_words) * 32 &&
      local < static_cast<int64_t>(p.pinned) - p.row_offset)
    atomicOr(&p.pin_mask[static_cast<int64_t>(bh) * p.pin_words + (local >> 5)], 1u << (local & 31));
}

struct AttSmem {
  __align__(16) float w[kCandChunk];
  __align__(16) int32_t row[kCandChunk];
  float sc[kCandChunk];  // candidate mode: raw scores of the batch's selected rows (coalesced id writes)
  float red[NW][kD];
  float l[NW];
  float z[128];
  float scr[32];
  float o[NT];
  uint32_t wcnt[NW];
  uint32_t base;
  int last;
};

// Accumulate the V rows listed in sm.row (local rows, -1 = skip) weighted by sm.w into this
// thread's registers: lane part·8 .. +7 of the 128 dims (16 lanes per 256-byte row, 16-byte
// loads), and the weight sum. A half-warp takes 8 consecutive list entries per round — their
// ids and weights arrive as two broadcast 16-byte shared loads each instead of eight scalar
// ones (ncu, cfg3: the per-row id load and its bounds test were 11 % of the kernel's
// instructions) — and keeps their 8 rows in flight. Leaves sm.row / sm.w intact.
template <class Gp = CtaGrp, int UNR = 8>
__device__ void gather_acc(const AttendParams& p, int bh, int nrows, const AttSmem& sm, float (&acc)[8],
                           float& lw) {
  static_assert(UNR % 4 == 0, "list entries come in 16-byte groups of four");
  const int b = bh / p.Hq, h = bh % p.Hq, kvh = h / p.G;
  const int tid = Gp::tid(), lane = tid & 31, warp = tid >> 5;
  const int half = lane >> 4, part = lane & 15;
  const __nv_bfloat16* vb =
      p.vc + (static_cast<int64_t>(b) * p.Hkv + kvh) * p.cache_rows * kD + part * 8;
  for (int r0 = (warp * 2 + half) * UNR; r0 < nrows; r0 += 2 * NW * UNR) {
    int rr[UNR];
    float ww[UNR];
#pragma unroll
    for (int g = 0; g < UNR / 4; ++g) {
      const int4 ra = *reinterpret_cast<const int4*>(&sm.row[r0 + 4 * g]);
      const float4 wa = *reinterpret_cast<const float4*>(&sm.w[r0 + 4 * g]);
      rr[4 * g] = ra.x, rr[4 * g + 1] = ra.y, rr[4 * g + 2] = ra.z, rr[4 * g + 3] = ra.w;
      ww[4 * g] = wa.x, ww[4 * g + 1] = wa.y, ww[4 * g + 2] = wa.z, ww[4 * g + 3] = wa.w;
    }
    uint4 v[UNR];
    float w[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const bool ok = r0 + u < nrows && rr[u] >= 0;
      w[u] = ok ? ww[u] : 0.f;
      v[u] = ok ? ldg_stream(vb + static_cast<int64_t>(rr[u]) * kD) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (part == 0) lw += w[u];
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
}

// Reduce the per-thread (acc, lw) of gather_acc over the block into the head's partial slot
// (l, o[128]). Ends with a barrier (smem reusable).
template <class Gp = CtaGrp>
__device__ void partial_write(const AttendParams& p, int bh, int slot, AttSmem& sm, float (&acc)[8], float lw) {
  const int tid = Gp::tid(), lane = tid & 31, warp = tid >> 5;
  const int half = lane >> 4, part = lane & 15;
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] += __shfl_xor_sync(kFull, acc[j], 16);
  Gp::sync();  // sm.row / sm.w readers are done before the reduction buffers are reused
  if (half == 0) {
#pragma unroll
    for (int j = 0; j < 8; ++j) sm.red[warp][part * 8 + j] = acc[j];
  }
  lw = warp_sum(lw);
  if (lane == 0) sm.l[warp] = lw;
  Gp::sync();
  if (tid < kD) {
    float o = 0.f;
#pragma unroll
    for (int w2 = 0; w2 < NW; ++w2) o += sm.red[w2][tid];
    p.part_o[(static_cast<int64_t>(bh) * p.nchunks + slot) * kD + tid] = o;
  }
  if (tid == 0) {
    float l = 0.f;
#pragma unroll
    for (int w2 = 0; w2 < NW; ++w2) l += sm.l[w2];
    p.part_l[static_cast<int64_t>(bh) * p.nchunks + slot] = l;
  }
  Gp::sync();
}

// Gather the V rows listed in sm.row weighted by sm.w and reduce them into the head's partial
// slot (l, o[128]). Ends with a barrier (smem reusable).
template <class Gp = CtaGrp>
__device__ void gather_partial(const AttendParams& p, int bh, int slot, int nrows, AttSmem& sm) {
  float acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = 0.f;
  float lw = 0.f;
  gather_acc<Gp>(p, bh, nrows, sm, acc, lw);
  partial_write<Gp>(p, bh, slot, sm, acc, lw);
}

// The last CTA of a head (caller decided, after a __threadfence): combine the nslots partials
// in slot order (deterministic), add the unselected pinned-prefix rows and the window, write out
// (or the (l, o) partial in sharded mode).
template <class Gp = CtaGrp>
__device__ void head_finish(const AttendParams& p, int bh, int nslots, AttSmem& sm) {
  const int b = bh / p.Hq, h = bh % p.Hq, kvh = h / p.G;
  const int tid = Gp::tid();
  const int kb = __ldcg(&p.meta_kb[bh]);
  const float zref = kb > 0 ? __ldcg(&p.meta_max[bh]) * p.scale * kLog2e : 0.f;
  const int64_t nctx = p.n_ctx[b];
  // sum the partials in slot order (deterministic), 8 slots' loads in flight at a time (a
  // dependent load per slot made the finish a serial chain of L2 round trips: ~18 slots per
  // head at cfg3)
  float o_c = 0.f, l_c = 0.f;
  const float* po = p.part_o + static_cast<int64_t>(bh) * p.nchunks * kD + (tid & (kD - 1));
  const float* pl = p.part_l + static_cast<int64_t>(bh) * p.nchunks;
  for (int c0 = 0; c0 < nslots; c0 += 8) {
    float vo[8], vl[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const bool ok = c0 + u < nslots;
      vo[u] = ok && tid < kD ? __ldcg(po + static_cast<int64_t>(c0 + u) * kD) : 0.f;
      vl[u] = ok ? __ldcg(pl + c0 + u) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      o_c += vo[u];
      l_c += vl[u];
    }
  }
  add_pinned<Gp>(p, b, h, kvh, nctx, kb, zref, l_c, o_c, sm.z, sm.scr, &sm.red[0][0]);
  if (p.partial_only) {
    sm.o[tid] = o_c;
    Gp::sync();
    float* dst = p.partial_out + static_cast<int64_t>(bh) * (kD + 1);
    if (tid == 0) dst[0] = l_c;
    if (tid < kD) dst[1 + tid] = sm.o[tid] + sm.o[tid + kD];
    Gp::sync();
    return;
  }
  finalize_head<Gp>(p, b, h, kvh, nctx, zref, l_c, o_c, sm.z, sm.scr, sm.o, &sm.red[0][0]);
  Gp::sync();
}

// Per-head ticket after a partial slot was written; the last CTA of the head finishes it.
template <class Gp = CtaGrp>
__device__ void ticket_finish(const AttendParams& p, int bh, int nslots, AttSmem& sm) {
  __threadfence();
  Gp::sync();
  if (Gp::tid() == 0) sm.last = (atomicAdd(&p.ticket[bh], 1u) == static_cast<unsigned>(nslots - 1));
  Gp::sync();
  if (!sm.last) return;
  __threadfence();
  if (Gp::tid() == 0) p.ticket[bh] = 0u;
  head_finish<Gp>(p, bh, nslots, sm);
}

// gather_partial + per-head ticket; the last CTA of the head finishes it.
template <class Gp = CtaGrp>
__device__ void chunk_body(const AttendParams& p, int bh, int slot, int nslots, int nrows, AttSmem& sm) {
  gather_partial<Gp>(p, bh, slot, nrows, sm);
  ticket_finish<Gp>(p, bh, nslots, sm);
}
}  // namespace

}  // namespace tkv
