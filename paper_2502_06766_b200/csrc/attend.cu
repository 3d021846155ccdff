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

#include "attend_cand_dev.cuh"

namespace tkv {

// CTAs per SM the gather kernels are compiled for. With 4 (64 registers) the compiler
// interleaves the FMAs with the loads and keeps ~3 of the 8 V-row loads per lane in flight;
// with 3 (85 registers) all 8 are issued before the first use — but the step time measured the
// same for 2, 3 and 4 (cfg3 383-388 us, within noise), and 4 was the fastest run.
#ifndef TKV_ATT_MINB
#define TKV_ATT_MINB 4
#endif


// List mode (sharded partial): the selected (idx, score) list is given.
__global__ void __launch_bounds__(NT, 4) attend_kernel(AttendParams p) {
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
    if (owned) mark_pinned(p, bh, local);
    sm.row[i] = owned ? static_cast<int32_t>(local) : -1;
    sm.w[i] = owned ? exp2f(fmaf(s, zs, -zref)) : 0.f;
  }
  __syncthreads();
  chunk_body(p, bh, ch, gridDim.x, nrows, sm);  // one partial slot per chunk of the k list
}

// Candidate mode (single GPU): persistent CTAs walk (head, chunk of kCandChunk candidates)
// work items; a candidate is selected iff its composite >= meta_kth (kth_kernel), which is
// exactly the top-kb set. Selected rows are appended to idx/scores (order unspecified) and,
// with p.gather, their V rows are gathered in the same pass.
__global__ void __launch_bounds__(NT, TKV_ATT_MINB) attend_cand_kernel(AttendParams p) {
  __shared__ AttSmem sm;
  extern __shared__ uint32_t s_pref[];  // [B*Hq + 1] work-item prefix over heads
  attend_cand_run(p, sm, s_pref);
}

// List gather (after a filter pass wrote each head's kb selected rows to idx/scores). The
// concatenation of all heads' lists (T rows) is split into one equal contiguous range per CTA
// — perfectly balanced, like a flat gather — and a CTA walks the head segments of its range:
// every half-warp streams rows (id and score straight from global memory, 16-byte V loads, 8
// rows in flight), one reduction per segment goes to the head's partial slot (CTA index minus
// the head's first CTA), and the head ticket counts the CTAs whose ranges overlap the head.
__global__ void __launch_bounds__(NT, TKV_ATT_MINB) attend_list_kernel(AttendParams p) {
  __shared__ AttSmem sm;
  extern __shared__ uint32_t s_pref[];  // [heads + 1] prefix of kb over heads
  if (threadIdx.x == 0) tl_start(p.tl, 6);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int half = lane >> 4, part = lane & 15, hw = warp * 2 + half;
  const int BH = p.bh_count ? p.bh_count : p.B * p.Hq;
  auto kb_of = [&](int lh) -> uint32_t { return static_cast<uint32_t>(max(p.meta_kb[p.bh_begin + lh], 0)); };
  {
    const int per = (BH + NT - 1) / NT;
    uint32_t sum = 0;
    for (int j = 0; j < per; ++j) {
      const int lh = tid * per + j;
      sum += lh < BH ? kb_of(lh) : 0u;
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
        run += kb_of(lh);
      }
    }
    if (tid == NT - 1) s_pref[BH] = run;
    __syncthreads();
  }
  const int64_t T = s_pref[BH];
  // CTAs in use: ranges of at least kFlatMinRows rows (bounds the slots per head)
  int64_t G = (T + kFlatMinRows - 1) / kFlatMinRows;
  if (G > gridDim.x) G = gridDim.x;
  if (G < 1) G = 1;
  auto start_of = [&](int64_t c) -> int64_t { return T * c / G; };
  auto cta_of = [&](int64_t r) -> int64_t {  // the CTA whose range holds flat row r
    int64_t lo = 0, hi = G;                   // largest c with start_of(c) <= r
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (start_of(mid) <= r) lo = mid; else hi = mid;
    }
    return lo;
  };
  const float zs = p.scale * kLog2e;
  // heads with nothing selected still need their output: CTA (head mod G) finishes them
  for (int lh = static_cast<int>(blockIdx.x); lh < BH; lh += static_cast<int>(G)) {
    if (blockIdx.x >= G) break;
    if (s_pref[lh + 1] != s_pref[lh]) continue;
    float acc0[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    partial_write(p, p.bh_begin + lh, 0, sm, acc0, 0.f);
    ticket_finish(p, p.bh_begin + lh, 1, sm);
    __syncthreads();
  }
  if (blockIdx.x < G) {
    const int64_t r_lo = start_of(blockIdx.x), r_hi = start_of(blockIdx.x + 1);
    int lh;
    {  // first head whose rows reach past r_lo
      int lo = 0, hi = BH;  // largest lh with s_pref[lh] <= r_lo
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s_pref[mid] <= r_lo) lo = mid; else hi = mid;
      }
      lh = lo;
    }
    for (; lh < BH && static_cast<int64_t>(s_pref[lh]) < r_hi; ++lh) {
      const int64_t h0 = s_pref[lh], h1 = s_pref[lh + 1];
      if (h1 <= r_lo || h1 == h0) continue;
      const int64_t s0 = r_lo > h0 ? r_lo : h0, s1 = r_hi < h1 ? r_hi : h1;
      const int64_t c_first = cta_of(h0), c_last = cta_of(h1 - 1);
      const int slot = static_cast<int>(blockIdx.x - c_first);
      const int nslots = static_cast<int>(c_last - c_first + 1);
      const int bh = p.bh_begin + lh;
      const int b = bh / p.Hq, kvh = (bh % p.Hq) / p.G;
      const int kb = p.meta_kb[bh];
      const float zref = kb > 0 ? p.meta_max[bh] * zs : 0.f;
      const int32_t* ids = p.idx_out + static_cast<int64_t>(bh) * p.k - h0;  // index by flat row
      const float* scs = p.scores_out + static_cast<int64_t>(bh) * p.k - h0;
      const __nv_bfloat16* vb =
          p.vc + (static_cast<int64_t>(b) * p.Hkv + kvh) * p.cache_rows * kD + part * 8;
      float acc[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = 0.f;
      float lw = 0.f;
      constexpr int UNR = 8;
      constexpr int STEP = 2 * NW * UNR;  // rows per round of the CTA
      // software pipeline: the next round's ids / scores load while this round's V rows are
      // in flight (one memory latency per round instead of two)
      int idn[UNR];
      float scn[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int64_t r = s0 + hw + 2 * NW * u;
        idn[u] = r < s1 ? __ldcg(&ids[r]) : -1;
        scn[u] = r < s1 ? __ldcg(&scs[r]) : 0.f;
      }
      for (int64_t r0 = s0 + hw; r0 < s1; r0 += STEP) {
        int id[UNR];
        float sc[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          id[u] = idn[u];
          sc[u] = scn[u];
        }
        uint4 v[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u)
          v[u] = id[u] >= 0 ? ldg_stream(vb + (static_cast<int64_t>(id[u]) - p.row_offset) * kD)
                            : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const int64_t r = r0 + STEP + 2 * NW * u;
          idn[u] = r < s1 ? __ldcg(&ids[r]) : -1;
          scn[u] = r < s1 ? __ldcg(&scs[r]) : 0.f;
        }
        float w[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          w[u] = id[u] >= 0 ? exp2f(fmaf(sc[u], zs, -zref)) : 0.f;
          if (part == 0) lw += w[u];
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
#ifdef TKV_GATHER_DIAG  // timing only: no reduction / head ticket (results are wrong)
      if (acc[0] == 12345.f) p.part_l[0] = acc[1] + lw + slot + nslots;
      continue;
#endif
      partial_write(p, bh, slot, sm, acc, lw);
      ticket_finish(p, bh, nslots, sm);
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) tl_end(p.tl, 6);
}

cudaError_t launch_attend_list(const AttendParams& p, cudaStream_t s) {
  const int grid = per_device(reinterpret_cast<const void*>(attend_list_kernel), 0, [] {
    cudaFuncSetAttribute(attend_list_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, attend_list_kernel, NT, 8192);
    return device_sm_count() * (per > 0 ? per : 1);
  });
  const size_t nbh = p.bh_count ? static_cast<size_t>(p.bh_count) : static_cast<size_t>(p.B) * p.Hq;
  attend_list_kernel<<<grid, NT, (nbh + 1) * sizeof(uint32_t), s>>>(p);
  return cudaGetLastError();
}

// Sharded finalize: partial_in holds the all-reduced (l, o[128]) per head.
__global__ void __launch_bounds__(NT) finalize_kernel(AttendParams p) {
  __shared__ float s_z[128];
  __shared__ float s_scr[32];
  __shared__ float s_o[NT];
  __shared__ float s_red[NW * kD];
  const int bh = blockIdx.x;
  const int b = bh / p.Hq, h = bh % p.Hq, kvh = h / p.G;
  const int tid = threadIdx.x;
  const int kb = p.meta_kb[bh];
  const float zs = p.scale * kLog2e;
  const float zref = kb > 0 ? p.meta_max[bh] * zs : 0.f;
  float l_c = 0.f, o_c = 0.f;
  if (kb > 0 && p.n_peers > 0) {  // every rank's partial, read from its buffer (peer memory)
    // all G pointer loads, then all G partial loads in flight at once (one peer round trip, not
    // G dependent ones: 9.5 us at G = 8 in the one-GPU emulation, more over NVLink), summed in
    // rank order (deterministic)
    const float* src[kMaxShards];
#pragma unroll
    for (int g = 0; g < kMaxShards; ++g)
      src[g] = g < p.n_peers ? p.partial_peers[g] + static_cast<int64_t>(bh) * (kD + 1) : nullptr;
    float lv[kMaxShards], ov[kMaxShards];
#pragma unroll
    for (int g = 0; g < kMaxShards; ++g) {
      lv[g] = src[g] ? __ldcg(src[g]) : 0.f;
      ov[g] = src[g] && tid < kD ? __ldcg(src[g] + 1 + tid) : 0.f;
    }
#pragma unroll
    for (int g = 0; g < kMaxShards; ++g) {
      l_c += lv[g];
      o_c += ov[g];
    }
  } else if (kb > 0) {
    const float* src = p.partial_in + static_cast<int64_t>(bh) * (kD + 1);
    l_c = src[0];
    o_c = tid < kD ? src[1 + tid] : 0.f;
  }
  finalize_head(p, b, h, kvh, p.n_ctx[b], zref, l_c, o_c, s_z, s_scr, s_o, s_red);
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
  if (threadIdx.x == 0 && p.advance && pos >= 0 && pos < p.cache_rows) p.count[b] = cnt + 1;  // written rows only
}

cudaError_t launch_attend(const AttendParams& p, cudaStream_t s) {
  // chunks of kAttendChunk selected rows: the k-list needs ceil(k / kAttendChunk) of them (the
  // workspace's partial slots, nchunks, are sized for the candidate-mode gather and can be far
  // more: launching nchunks CTAs per head would mostly launch empty ones)
  const int nch = (p.k + kAttendChunk - 1) / kAttendChunk;
  dim3 grid(nch < p.nchunks ? nch : p.nchunks, p.B * p.Hq);
  attend_kernel<<<grid, NT, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_attend_cand(const AttendParams& p, cudaStream_t s) {
  const int grid = per_device(reinterpret_cast<const void*>(attend_cand_kernel), 0, [] {
    // same shared-memory carveout as the scan, so both can share an SM (parts pipeline)
    cudaFuncSetAttribute(attend_cand_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, attend_cand_kernel, NT, 8192);
    const int g = device_sm_count() * (per > 0 ? per : 1);
    return g < kMaxGatherGrid ? g : kMaxGatherGrid;
  });
  const size_t nbh = p.bh_count ? static_cast<size_t>(p.bh_count) : static_cast<size_t>(p.B) * p.Hq;
  attend_cand_kernel<<<grid, NT, (nbh + 1) * sizeof(uint32_t), s>>>(p);
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
