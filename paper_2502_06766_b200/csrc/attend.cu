// attend.cu — K3: V gather + softmax over exactly the selected rows (+ window, + pinned
// prefix), and K4: KV append.
//
// Reference (attention.py:158-167, 107-122): s_ctx = (K[ids]·q)/sqrt(d), v_ctx = V[ids],
// s_gen = (K_gen·q)/sqrt(d); joint: softmax over [s_ctx, s_gen] applied to [v_ctx; v_gen];
// additive: two independently normalised softmaxes summed. All f64 in the reference; here fp32
// with exp2 of pre-scaled scores.
//
// Gather: grid (ceil(k / 512), B*Hq). The selection kernel already produced each selected
// row's exact score and the per-head maximum M, so every chunk weights its rows with
// w = 2^((s - M)·scale·log2e) <= 1 directly (no running-max rescale): a CTA loads its 512
// (row, score) pairs, streams the V rows with 16-byte loads (16 lanes per 256-byte row) and
// reduces (l, o[128]) into a per-chunk partial. The last CTA of each head (atomic ticket) sums
// the partials in chunk order (deterministic), adds the pinned-prefix rows that were not
// selected and the window rows (online softmax, scores from the same HMMA tile function as
// the scan so pinned-row membership is decided on bit-identical scores), normalises and
// writes out[b, h, :].
#include <math.h>

#include "common.cuh"
#include "internal.h"

namespace tkv {

namespace {
constexpr int NT = kAttendThreads;
constexpr int NW = NT / 32;

// Online softmax accumulation over local rows [r_begin, r_end) of kv head (b, kvh) for q head
// h. State (m, l, o) in the log2-scaled domain; thread t accumulates o for d = t % 128 over rows
// of parity t / 128. With `pinned`, a row is skipped when it is among the selected top-k
// (composite >= kth).
__device__ void accumulate_rows(const AttendParams& p, int b, int h, int kvh, int64_t r_begin,
                                int64_t r_end, bool pinned, uint64_t kth, float& m, float& l,
                                float& o, float* s_z, float* s_scr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, c = lane & 3;
  const int n = h - kvh * p.G;
  const float zs = p.scale * kLog2e;
  QFrag f;
  load_qfrag(f, p.q + (static_cast<int64_t>(b) * p.Hq + kvh * p.G) * kD, p.G, lane);
  const int64_t head_off = (static_cast<int64_t>(b) * p.Hkv + kvh) * p.cache_rows * kD;
  const __nv_bfloat16* kb = p.kc + head_off;
  const __nv_bfloat16* vb = p.vc + head_off;
  const int d = tid & (kD - 1), par = tid >> 7;
  for (int64_t base = r_begin; base < r_end; base += 8 * 16) {
    {
      const int64_t rA = base + warp * 16 + g, rB = rA + 8;
      uint4 a[2][4];
      load_tile(a, kb + rA * kD, rA < r_end, kb + rB * kD, rB < r_end, c);
      float acc[4];
      score_tile(acc, a, f);
      if (c == (n >> 1)) {
        const float sA = acc[n & 1], sB = acc[2 + (n & 1)];
        bool okA = rA < r_end, okB = rB < r_end;
        if (pinned) {
          okA = okA && make_comp(score_key(sA), static_cast<uint32_t>(p.row_offset + rA)) < kth;
          okB = okB && make_comp(score_key(sB), static_cast<uint32_t>(p.row_offset + rB)) < kth;
        }
        s_z[warp * 16 + g] = okA ? sA * zs : -INFINITY;
        s_z[warp * 16 + g + 8] = okB ? sB * zs : -INFINITY;
      }
    }
    __syncthreads();
    float v = tid < 128 ? s_z[tid] : -INFINITY;
    v = warp_max(v);
    if (lane == 0) s_scr[warp] = v;
    __syncthreads();
    float cm = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) cm = fmaxf(cm, s_scr[w]);
    const float mn = fmaxf(m, cm);
    if (mn != -INFINITY) {
      const float fold = (m == -INFINITY) ? 0.f : exp2f(m - mn);
      float lsum = 0.f, osum = 0.f;
      for (int r = 0; r < 128; ++r) {
        const float z = s_z[r];
        if (z == -INFINITY) continue;
        const float w = exp2f(z - mn);
        lsum += w;
        if ((r & 1) == par) osum += w * __bfloat162float(vb[(base + r) * kD + d]);
      }
      l = l * fold + lsum;
      o = o * fold + osum;
      m = mn;
    }
    __syncthreads();
  }
}

// Pinned-prefix rows [0, p) that the top-k did not select join the context softmax
// (attention.py:152-154 unions them into the retrieved ids). Local rows of this shard only.
__device__ void add_pinned(const AttendParams& p, int b, int h, int kvh, int64_t nctx, int kb,
                           float zref, float& l, float& o, float* s_z, float* s_scr) {
  if (p.pinned <= 0 || kb <= 0) return;
  int64_t lo = -p.row_offset;
  if (lo < 0) lo = 0;
  int64_t hi = static_cast<int64_t>(p.pinned) - p.row_offset;
  if (hi > nctx) hi = nctx;
  if (hi <= lo) return;
  const int bh = b * p.Hq + h;
  float m = zref;
  accumulate_rows(p, b, h, kvh, lo, hi, true, p.meta_kth[bh], m, l, o, s_z, s_scr);
  // every unselected row scores <= the k-th selected score <= M, so m stays zref
}

// Window rows + normalisation. Inputs: context state (zref, l_c, o_c) where o_c is this
// thread's share (d = tid % 128, parity tid / 128). Writes out[bh, :].
__device__ void finalize_head(const AttendParams& p, int b, int h, int kvh, int64_t nctx, float zref,
                              float l_c, float o_c, float* s_z, float* s_scr, float* s_o) {
  const int tid = threadIdx.x;
  const int bh = b * p.Hq + h;
  const int64_t nwin = p.n_win ? p.n_win[b] : 0;
  float m_w = -INFINITY, l_w = 0.f, o_w = 0.f;
  if (nwin > 0) accumulate_rows(p, b, h, kvh, nctx, nctx + nwin, false, 0ull, m_w, l_w, o_w, s_z, s_scr);
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
  __syncthreads();
  if (tid < kD) p.out[static_cast<int64_t>(bh) * kD + tid] = s_o[tid] + s_o[tid + kD];
}

struct AttSmem {
  float w[kCandChunk];
  int32_t row[kCandChunk];
  float red[NW][kD];
  float l[NW];
  float z[128];
  float scr[32];
  float o[NT];
  uint32_t wcnt[NW];
  uint32_t base;
  int last;
};

// Gather the V rows listed in sm.row (local rows, -1 = skip) weighted by sm.w, reduce into the
// head's partial slot, and let the last CTA of the head (atomic ticket over nslots) combine
// the partials in slot order (deterministic), add the pinned-prefix rows and the window, and
// write out (or the (l, o) partial in sharded mode).
__device__ void chunk_body(const AttendParams& p, int bh, int slot, int nslots, int nrows, AttSmem& sm) {
  const int b = bh / p.Hq, h = bh % p.Hq, kvh = h / p.G;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int half = lane >> 4, part = lane & 15;
  const __nv_bfloat16* vb =
      p.vc + (static_cast<int64_t>(b) * p.Hkv + kvh) * p.cache_rows * kD + part * 8;
  float acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = 0.f;
  constexpr int UNR = 8;
  for (int r0 = warp * 2 + half; r0 < nrows; r0 += 2 * NW * UNR) {
    uint4 v[UNR];
    float w[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int r = r0 + 2 * NW * u;
      const int row = r < nrows ? sm.row[r] : -1;
      w[u] = r < nrows ? sm.w[r] : 0.f;
      v[u] = row >= 0 ? ldg_nc(vb + static_cast<int64_t>(row) * kD) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
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
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] += __shfl_xor_sync(kFull, acc[j], 16);
  if (half == 0) {
#pragma unroll
    for (int j = 0; j < 8; ++j) sm.red[warp][part * 8 + j] = acc[j];
  }
  float lw = 0.f;
  for (int i = tid; i < nrows; i += NT) lw += sm.w[i];
  lw = warp_sum(lw);
  if (lane == 0) sm.l[warp] = lw;
  __syncthreads();
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
  __threadfence();
  __syncthreads();
  if (tid == 0) sm.last = (atomicAdd(&p.ticket[bh], 1u) == static_cast<unsigned>(nslots - 1));
  __syncthreads();
  if (!sm.last) return;
  __threadfence();

  // ---- last CTA of this head: deterministic slot-order combine
  const int kb = p.meta_kb[bh];
  const float zref = kb > 0 ? p.meta_max[bh] * p.scale * kLog2e : 0.f;
  const int64_t nctx = p.n_ctx[b];
  float o_c = 0.f, l_c = 0.f;
  for (int c2 = 0; c2 < nslots; ++c2) {
    if (tid < kD) o_c += __ldcg(&p.part_o[(static_cast<int64_t>(bh) * p.nchunks + c2) * kD + tid]);
    l_c += __ldcg(&p.part_l[static_cast<int64_t>(bh) * p.nchunks + c2]);
  }
  if (tid == 0) p.ticket[bh] = 0u;
  add_pinned(p, b, h, kvh, nctx, kb, zref, l_c, o_c, sm.z, sm.scr);
  if (p.partial_only) {
    sm.o[tid] = o_c;
    __syncthreads();
    float* dst = p.partial_out + static_cast<int64_t>(bh) * (kD + 1);
    if (tid == 0) dst[0] = l_c;
    if (tid < kD) dst[1 + tid] = sm.o[tid] + sm.o[tid + kD];
    __syncthreads();
    return;
  }
  finalize_head(p, b, h, kvh, nctx, zref, l_c, o_c, sm.z, sm.scr, sm.o);
  __syncthreads();
}
}  // namespace

// List mode (sharded partial): the selected (idx, score) list is given.
__global__ void __launch_bounds__(NT) attend_kernel(AttendParams p) {
  __shared__ AttSmem sm;
  const int ch = blockIdx.x, bh = blockIdx.y;
  const int b = bh / p.Hq;
  const int kb = p.meta_kb[bh];
  const int lo = ch * kAttendChunk;
  int nrows = kb - lo;
  nrows = nrows < 0 ? 0 : (nrows > kAttendChunk ? kAttendChunk : nrows);
  const float zs = p.scale * kLog2e;
  const float zref = kb > 0 ? p.meta_max[bh] * zs : 0.f;
  const int64_t nctx = p.n_ctx[b];
  for (int i = threadIdx.x; i < nrows; i += NT) {
    const int64_t gid = p.idx[static_cast<int64_t>(bh) * p.k + lo + i];
    const float s = p.scores[static_cast<int64_t>(bh) * p.k + lo + i];
    const int64_t local = gid - p.row_offset;
    const bool owned = local >= 0 && local < nctx;
    sm.row[i] = owned ? static_cast<int32_t>(local) : -1;
    sm.w[i] = owned ? exp2f(fmaf(s, zs, -zref)) : 0.f;
  }
  __syncthreads();
  chunk_body(p, bh, ch, p.nchunks, nrows, sm);
}

// Candidate mode (single GPU): persistent CTAs walk (head, chunk of kCandChunk candidates)
// work items; a candidate is selected iff its composite >= meta_kth (kth_kernel), which is
// exactly the top-kb set. Selected rows are appended to idx/scores (order unspecified) and,
// with p.gather, their V rows are gathered in the same pass.
__global__ void __launch_bounds__(NT) attend_cand_kernel(AttendParams p) {
  __shared__ AttSmem sm;
  extern __shared__ uint32_t s_pref[];  // [B*Hq + 1] work-item prefix over heads
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int BH = p.B * p.Hq;
  auto nslots_of = [&](int bh) -> int {
    int64_t n = p.cand_cnt[bh];
    if (n > p.cap) n = p.cap;
    const int c = static_cast<int>((n + kCandChunk - 1) / kCandChunk);
    return c > 0 ? c : 1;  // every head gets >= 1 item so its output is always finalized
  };
  // exclusive prefix of work items per head (block-wide, BH <= a few thousand)
  {
    const int per = (BH + NT - 1) / NT;
    uint32_t sum = 0;
    for (int j = 0; j < per; ++j) {
      const int bh = tid * per + j;
      sum += bh < BH ? nslots_of(bh) : 0;
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
      const int bh = tid * per + j;
      if (bh < BH) {
        s_pref[bh] = run;
        run += nslots_of(bh);
      }
    }
    if (tid == NT - 1) s_pref[BH] = run;
    __syncthreads();
  }
  const uint32_t total = s_pref[BH];
  const float zs = p.scale * kLog2e;
  for (uint32_t item = blockIdx.x; item < total; item += gridDim.x) {
    int lo = 0, hi = BH;  // largest bh with s_pref[bh] <= item
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_pref[mid] <= item) lo = mid; else hi = mid;
    }
    const int bh = lo;
    const int slot = static_cast<int>(item - s_pref[bh]);
    const int nslots = static_cast<int>(s_pref[bh + 1] - s_pref[bh]);
    const int b = bh / p.Hq;
    int64_t n = p.cand_cnt[bh];
    if (n > p.cap) n = p.cap;
    const int kb = p.meta_kb[bh];
    const uint64_t T = p.meta_kth[bh];
    const float zref = kb > 0 ? p.meta_max[bh] * zs : 0.f;
    const uint64_t* src = p.cand + static_cast<int64_t>(bh) * p.cap + static_cast<int64_t>(slot) * kCandChunk;
    int64_t cnt = n - static_cast<int64_t>(slot) * kCandChunk;
    cnt = cnt < 0 ? 0 : (cnt > kCandChunk ? kCandChunk : cnt);
    constexpr int PER = kCandChunk / NT;
    uint64_t cv[PER];
    bool sel[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int i = u * NT + tid;
      cv[u] = (i < cnt && kb > 0) ? src[i] : 0ull;
      sel[u] = cv[u] != 0ull && cv[u] >= T;
    }
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
    if (lane == 31) sm.wcnt[warp] = incl;
    __syncthreads();
    uint32_t woff = 0, m = 0;
    for (int w = 0; w < NW; ++w) {
      woff += w < warp ? sm.wcnt[w] : 0u;
      m += sm.wcnt[w];
    }
    if (tid == 0) sm.base = m ? atomicAdd(&p.out_cnt[bh], m) : 0u;
    __syncthreads();
    const uint32_t obase = sm.base;
    uint32_t pos = woff + incl - mine;
    int32_t* idx_o = p.idx_out + static_cast<int64_t>(bh) * p.k;
    float* sc_o = p.scores_out + static_cast<int64_t>(bh) * p.k;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      if (sel[u]) {
        const uint64_t c = cv[u];
        const uint32_t gid = comp_gid(c);
        const float s = key_score(comp_key(c));
        const uint32_t o = obase + pos;
        if (o < static_cast<uint32_t>(p.k)) {
          idx_o[o] = static_cast<int32_t>(gid);
          sc_o[o] = s;
          if (p.packed_out) p.packed_out[static_cast<int64_t>(bh) * p.k + o] = c;
        }
        sm.row[pos] = static_cast<int32_t>(static_cast<int64_t>(gid) - p.row_offset);
        sm.w[pos] = exp2f(fmaf(s, zs, -zref));
        ++pos;
      }
    }
    if (slot == 0) {  // pads for k > kb (reference clamps k to N, attention.py:147-149)
      for (int i = kb + tid; i < p.k; i += NT) {
        idx_o[i] = -1;
        sc_o[i] = -INFINITY;
        if (p.packed_out) p.packed_out[static_cast<int64_t>(bh) * p.k + i] = 0ull;
      }
    }
    __syncthreads();
    if (p.gather) chunk_body(p, bh, slot, nslots, static_cast<int>(m), sm);
    (void)b;
  }
}

// Sharded finalize: partial_in holds the all-reduced (l, o[128]) per head.
__global__ void __launch_bounds__(NT) finalize_kernel(AttendParams p) {
  __shared__ float s_z[128];
  __shared__ float s_scr[32];
  __shared__ float s_o[NT];
  const int bh = blockIdx.x;
  const int b = bh / p.Hq, h = bh % p.Hq, kvh = h / p.G;
  const int tid = threadIdx.x;
  const int kb = p.meta_kb[bh];
  const float zs = p.scale * kLog2e;
  const float zref = kb > 0 ? p.meta_max[bh] * zs : 0.f;
  const float* src = p.partial_in + static_cast<int64_t>(bh) * (kD + 1);
  const float l_c = kb > 0 ? src[0] : 0.f;
  const float o_c = (kb > 0 && tid < kD) ? src[1 + tid] : 0.f;
  finalize_head(p, b, h, kvh, p.n_ctx[b], zref, l_c, o_c, s_z, s_scr, s_o);
}

// K4: KV append (GenWindow.append, attention.py:94-100) — one CTA per batch entry.
__global__ void __launch_bounds__(256) append_kernel(AppendParams p) {
  const int b = blockIdx.x;
  const int32_t cnt = p.count[b];
  const int32_t pos = (p.base ? p.base[b] : 0) + cnt;
  const int pieces = p.Hkv * 16;  // 16-byte pieces per tensor
  if (pos >= 0 && pos < p.cache_rows) {
    for (int i = threadIdx.x; i < 2 * pieces; i += blockDim.x) {
      const int which = i / pieces, rem = i % pieces;
      const int kvh = rem / 16, part = rem % 16;
      const __nv_bfloat16* src = (which ? p.v_new : p.k_new) + (static_cast<int64_t>(b) * p.Hkv + kvh) * kD + part * 8;
      __nv_bfloat16* dst = (which ? p.vc : p.kc) +
                           ((static_cast<int64_t>(b) * p.Hkv + kvh) * p.cache_rows + pos) * kD + part * 8;
      *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && p.advance) p.count[b] = cnt + 1;
}

cudaError_t launch_attend(const AttendParams& p, cudaStream_t s) {
  dim3 grid(p.nchunks, p.B * p.Hq);
  attend_kernel<<<grid, NT, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_attend_cand(const AttendParams& p, cudaStream_t s) {
  static int grid = 0;
  if (!grid) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, attend_cand_kernel, NT, 8192);
    grid = sms * (per > 0 ? per : 1);
  }
  const size_t smem = (static_cast<size_t>(p.B) * p.Hq + 1) * sizeof(uint32_t);
  attend_cand_kernel<<<grid, NT, smem, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_finalize(const AttendParams& p, cudaStream_t s) {
  finalize_kernel<<<p.B * p.Hq, NT, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_append(const AppendParams& p, cudaStream_t s) {
  append_kernel<<<p.B, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace tkv
