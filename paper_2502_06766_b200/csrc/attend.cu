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
}  // namespace

__global__ void __launch_bounds__(NT) attend_kernel(AttendParams p) {
  __shared__ float s_w[kAttendChunk];
  __shared__ int32_t s_row[kAttendChunk];
  __shared__ float s_red[NW][kD];
  __shared__ float s_l[NW];
  __shared__ float s_z[128];
  __shared__ float s_scr[32];
  __shared__ float s_o[NT];
  __shared__ int s_last;

  const int ch = blockIdx.x, bh = blockIdx.y;
  const int b = bh / p.Hq, h = bh % p.Hq, kvh = h / p.G;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kb = p.meta_kb[bh];
  const int lo = ch * kAttendChunk;
  int nrows = kb - lo;
  nrows = nrows < 0 ? 0 : (nrows > kAttendChunk ? kAttendChunk : nrows);
  const float zs = p.scale * kLog2e;
  const float zref = kb > 0 ? p.meta_max[bh] * zs : 0.f;
  const int64_t nctx = p.n_ctx[b];

  for (int i = tid; i < nrows; i += NT) {
    const int64_t gid = p.idx[static_cast<int64_t>(bh) * p.k + lo + i];
    const float s = p.scores[static_cast<int64_t>(bh) * p.k + lo + i];
    const int64_t local = gid - p.row_offset;
    const bool owned = local >= 0 && local < nctx;
    s_row[i] = owned ? static_cast<int32_t>(local) : -1;
    s_w[i] = owned ? exp2f(fmaf(s, zs, -zref)) : 0.f;
  }
  __syncthreads();

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
      const int row = r < nrows ? s_row[r] : -1;
      w[u] = r < nrows ? s_w[r] : 0.f;
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
    for (int j = 0; j < 8; ++j) s_red[warp][part * 8 + j] = acc[j];
  }
  float lw = 0.f;
  for (int i = tid; i < nrows; i += NT) lw += s_w[i];
  lw = warp_sum(lw);
  if (lane == 0) s_l[warp] = lw;
  __syncthreads();
  if (tid < kD) {
    float o = 0.f;
#pragma unroll
    for (int w2 = 0; w2 < NW; ++w2) o += s_red[w2][tid];
    p.part_o[(static_cast<int64_t>(bh) * p.nchunks + ch) * kD + tid] = o;
  }
  if (tid == 0) {
    float l = 0.f;
#pragma unroll
    for (int w2 = 0; w2 < NW; ++w2) l += s_l[w2];
    p.part_l[static_cast<int64_t>(bh) * p.nchunks + ch] = l;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(&p.ticket[bh], 1u) == static_cast<unsigned>(p.nchunks - 1));
  __syncthreads();
  if (!s_last) return;
  __threadfence();

  // ---- last CTA of this head: deterministic chunk-order combine
  float o_c = 0.f, l_c = 0.f;
  for (int c2 = 0; c2 < p.nchunks; ++c2) {
    if (tid < kD) o_c += __ldcg(&p.part_o[(static_cast<int64_t>(bh) * p.nchunks + c2) * kD + tid]);
    l_c += __ldcg(&p.part_l[static_cast<int64_t>(bh) * p.nchunks + c2]);
  }
  if (tid == 0) p.ticket[bh] = 0u;
  add_pinned(p, b, h, kvh, nctx, kb, zref, l_c, o_c, s_z, s_scr);
  if (p.partial_only) {
    s_o[tid] = o_c;
    __syncthreads();
    float* dst = p.partial_out + static_cast<int64_t>(bh) * (kD + 1);
    if (tid == 0) dst[0] = l_c;
    if (tid < kD) dst[1 + tid] = s_o[tid] + s_o[tid + kD];
    return;
  }
  finalize_head(p, b, h, kvh, nctx, zref, l_c, o_c, s_z, s_scr, s_o);
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

cudaError_t launch_finalize(const AttendParams& p, cudaStream_t s) {
  finalize_kernel<<<p.B * p.Hq, NT, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_append(const AppendParams& p, cudaStream_t s) {
  append_kernel<<<p.B, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace tkv
