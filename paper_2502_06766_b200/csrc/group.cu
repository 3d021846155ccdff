// group.cu — the small-context layer step: ONE thread-block cluster per (b, kv head) does the
// key scan, the exact top-k selection and the V gather of that KV group's G q heads.
//
// Reference computation (per q head, attention.py:125-167): ip_scores_all (ann_kernels.py:40-47),
// _flat_topk (ann.py:154-167: the k largest scores, ties to the lower row id), rescore + gather
// + _joint_attend (attention.py:158-167, 107-122).
//
// Why a separate path: at small contexts (cfg1 16K rows, cfg2 128K rows, a G = 8 token shard of
// cfg3) the multi-kernel pipeline (sample → threshold → scan → k-th → gather) is a chain of
// dependent launches and global round trips that costs as much as the key scan itself. Here a
// cluster of `cs` CTAs (one per SM, up to 16) splits the group's rows; every CTA keeps the
// order-preserving score keys of its rows for all G heads in shared memory, so the selection
// needs no sampled threshold, no candidate lists and no exactness fallback:
//
//   1. scan      each warp scores 32-row slabs with the HMMA tile (common.cuh score_tile; the
//                pinned-prefix / window code scores rows with the same function), keys → smem.
//   2. select    MSB-first radix select per head across the cluster: every CTA histograms its
//                keys (11-bit digits), CTA r sums bin slice r over the cluster through
//                distributed shared memory, every CTA finds the digit holding the kb-th largest
//                from the slice totals. Up to three levels (11 / 11 / 10 bits), stopping as soon
//                as the threshold bucket has <= kMemCap members: those are then sent (as
//                (key, ~row) composites) to the head's owner CTA, which rank-selects the exact
//                threshold composite T — selected ⇔ composite >= T, which is exactly the
//                reference's "above the k-th score plus the lowest-id ties". A bucket that is
//                still larger after the last level is a run of exactly equal keys: its rows are
//                taken in row order through cluster prefix counts (lower id first).
//   3. emit      every CTA counts its selected rows per head; cluster prefix sums give each CTA
//                its output range, so idx / scores are written in ascending row order.
//   4. gather    the selected rows' V rows (16 lanes per 256-byte row, 8 rows in flight per
//                half-warp, warps split between the heads) → one partial (l, o[128]) per CTA and
//                head in the head's partial slot `rank`.
//   5. finish    after a cluster barrier the head's owner CTA combines the cs partials, adds the
//                unselected pinned-prefix rows and the window, normalises (head_finish,
//                attend_dev.cuh — shared with the multi-kernel path).
// A decode step's window append (GenWindow.append, attention.py:94-100, 210) is folded in: the
// cluster's rank 0 writes the token's k/v row before any window read, the call attends with it,
// and the last cluster of the batch entry advances the window counter.
#include <cooperative_groups.h>

#include "attend_dev.cuh"

namespace tkv {
namespace cg = cooperative_groups;

namespace {
constexpr int GT = kGrpThreads, GW = GT / 32;
constexpr int kMemCap = 1024;  // threshold-bucket members per head sent to its owner CTA
constexpr int kListCap = 1024;  // selected rows per head staged per gather round

struct GrpShared {
  uint32_t kmax[8];     // this CTA's largest key per head
  uint32_t slsum[8];    // this CTA's bin-slice total per head (current level)
  uint32_t prefix[8];   // selected digits so far (per head, identical in every CTA)
  uint32_t need[8];     // rank still to place inside the prefix set
  uint32_t mode[8];     // 0 open, 1 threshold known (T), 2 members, 3 exact-key ties
  uint32_t dstar[8], above[8], bcnt[8];
  uint32_t nmem[8];     // owner: members received per head
  uint64_t T[8];        // exact threshold composite (modes 1, 2)
  uint32_t tkey[8];     // mode 3: the tied key
  uint32_t hshift[8];   // mode 2: members are the keys with key >> hshift == prefix
  uint32_t cnt_gt[8];   // this CTA: rows strictly above the threshold (mode 3) or all selected
  uint32_t cnt_tie[8];  // this CTA: rows equal to the tied key (mode 3)
  uint32_t sel[8];      // this CTA: selected rows per head
  uint32_t out_base[8]; // this CTA's first output position per head
  uint32_t tie_base[8]; // mode 3: tied rows in lower-ranked CTAs
  float mscore[8];      // head maximum score (cluster-wide)
  uint32_t scr[64];
  uint32_t out2[2];
  uint64_t res;
  float red[GW][kD];  // gather reduction
  float lsum[GW];
  AttSmem att;        // head_finish
};

}  // namespace

#ifdef TKV_DIAG
#define GRP_PHASE(e) \
  if (tid == 0) tl_phase(p.tl, e, t_ph)
#else
#define GRP_PHASE(e)
#endif

template <int CS>
__global__ void __launch_bounds__(GT, 1) group_topk_kernel(GroupParams gp) {
  const AttendParams& p = gp.a;
#ifdef TKV_DIAG
  uint64_t t_ph = p.tl ? gtimer() : 0ull;
#endif
  cg::cluster_group cluster = cg::this_cluster();
  constexpr int cs = CS;
  const int rank = static_cast<int>(cluster.block_rank());
  const int seg = static_cast<int>(blockIdx.x) / cs;
  const int b = seg / p.Hkv, kvh = seg % p.Hkv;
  const int G = p.G;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int R = gp.rows_per_cta;
  extern __shared__ __align__(16) uint8_t dyn[];
  uint32_t* s_key = reinterpret_cast<uint32_t*>(dyn);      // [G][R]
  uint32_t* s_hist = s_key + static_cast<size_t>(G) * R;   // [G][kGrpBins]
  constexpr int SBmax = kGrpBins / cs;
  uint32_t* s_tot = s_hist + static_cast<size_t>(G) * kGrpBins;  // [G][kGrpBins / cs]
  uint64_t* s_mem = reinterpret_cast<uint64_t*>(s_hist);   // owner: [G][kMemCap] (aliases hist)
  int32_t* s_lrow = reinterpret_cast<int32_t*>(s_hist);    // gather lists [G][kListCap] (alias)
  float* s_lw = reinterpret_cast<float*>(s_hist) + static_cast<size_t>(G) * kListCap;
  __shared__ GrpShared sh;

  int64_t N = p.n_ctx[b];
  N = N < 0 ? 0 : (N > gp.max_ctx ? gp.max_ctx : N);
  const int64_t r0 = static_cast<int64_t>(rank) * R;
  const int nrow = static_cast<int>(N - r0 < 0 ? 0 : (N - r0 > R ? R : N - r0));
  const int64_t kb = N < p.k ? N : p.k;
  const int bh0 = b * p.Hq + kvh * G;
  const int64_t head_off = (static_cast<int64_t>(b) * p.Hkv + kvh) * p.cache_rows * kD;

  // ---- window append (decode step): the token's k / v row of this kv head, before any read
  if (gp.k_new && rank == 0 && tid < 32) {
    const int64_t pos = N + gp.win_count[b];
    if (pos >= 0 && pos < p.cache_rows) {
      const int which = tid >> 4, part = tid & 15;
      const __nv_bfloat16* src = (which ? gp.v_new : gp.k_new) + (static_cast<int64_t>(b) * p.Hkv + kvh) * kD + part * 8;
      __nv_bfloat16* dst = (which ? gp.v_dst : gp.k_dst) + head_off + pos * kD + part * 8;
      *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
      __threadfence();
    }
  }
  if (tid < 8) {
    sh.kmax[tid] = 0u;
    sh.nmem[tid] = 0u;
    sh.prefix[tid] = 0u;
    sh.need[tid] = static_cast<uint32_t>(kb);
    sh.mode[tid] = kb == 0 ? 1u : 0u;  // nothing to select: T above every composite
    sh.T[tid] = ~0ull;
  }
  // pin masks of the heads this CTA owns (set by the emit pass below, read by head_finish)
  for (int g = rank; g < G; g += cs)
    for (int i = tid; i < p.pin_words; i += GT) p.pin_mask[static_cast<int64_t>(bh0 + g) * p.pin_words + i] = 0u;
  __syncthreads();

  // ---- 1. scan: 32-row slabs per warp (two 16-row HMMA tiles), keys → shared memory
  {
    QFrag f;
    load_qfrag(f, p.q + static_cast<int64_t>(bh0) * kD, G, lane);
    const __nv_bfloat16* kbase = p.kc + head_off + r0 * kD;
    const int g4 = lane >> 2, c4 = lane & 3;
    uint32_t m0 = 0u, m1 = 0u;
    for (int base = warp * 32; base < nrow; base += GW * 32) {
      uint4 t0[2][4], t1[2][4];
      const int a0 = base + g4, a1 = base + 16 + g4;
      load_tile(t0, kbase + static_cast<int64_t>(a0) * kD, a0 < nrow, kbase + static_cast<int64_t>(a0 + 8) * kD,
                a0 + 8 < nrow, c4);
      load_tile(t1, kbase + static_cast<int64_t>(a1) * kD, a1 < nrow, kbase + static_cast<int64_t>(a1 + 8) * kD,
                a1 + 8 < nrow, c4);
      float s0[4], s1[4];
      score_tile(s0, t0, f);
      score_tile(s1, t1, f);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int col = 2 * c4 + (i & 1);
        const int ra = a0 + (i >= 2 ? 8 : 0), rb = a1 + (i >= 2 ? 8 : 0);
        if (col < G) {
          if (ra < nrow) {
            const uint32_t key = score_key(s0[i]);
            s_key[col * R + ra] = key;
            if (i & 1) m1 = max(m1, key); else m0 = max(m0, key);
          }
          if (rb < nrow) {
            const uint32_t key = score_key(s1[i]);
            s_key[col * R + rb] = key;
            if (i & 1) m1 = max(m1, key); else m0 = max(m0, key);
          }
        }
      }
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      m0 = max(m0, __shfl_xor_sync(kFull, m0, o));
      m1 = max(m1, __shfl_xor_sync(kFull, m1, o));
    }
    if (g4 == 0) {
      if (2 * c4 < G) atomicMax(&sh.kmax[2 * c4], m0);
      if (2 * c4 + 1 < G) atomicMax(&sh.kmax[2 * c4 + 1], m1);
    }
  }
  __syncthreads();

  GRP_PHASE(47);
  // ---- 2. cluster radix select per head (levels of 11 / 11 / 10 bits)
  for (int level = 0; level < 3; ++level) {
    bool open = false;
    for (int g = 0; g < G; ++g) open |= sh.mode[g] == 0u;
    if (!open) break;  // identical in every CTA of the cluster
    const int width = level < 2 ? 11 : 10;
    const int shf = level == 0 ? 21 : (level == 1 ? 10 : 0);
    const uint32_t mask = (1u << width) - 1u;
    const int nb = 1 << width, SB = nb / cs;
    for (int i = tid; i < G * kGrpBins; i += GT) s_hist[i] = 0u;
    __syncthreads();
    for (int g = 0; g < G; ++g) {
      if (sh.mode[g] != 0u) continue;
      const uint32_t pre = sh.prefix[g];
      const uint32_t* keys = s_key + g * R;
      uint32_t* hist = s_hist + g * kGrpBins;
      for (int i = tid; i < nrow; i += GT) {
        const uint32_t key = keys[i];
        if (level == 0 || (key >> (shf + width)) == pre) atomicAdd(&hist[(key >> shf) & mask], 1u);
      }
    }
    __syncthreads();
    cluster.sync();  // every CTA's histograms complete
    // CTA `rank` sums bin slice [rank·SB, +SB) of every head over the cluster
    for (int e = tid; e < G * SB; e += GT) {
      const int g = e / SB, j = e - g * SB;
      if (sh.mode[g] != 0u) continue;
      const int bin = g * kGrpBins + rank * SB + j;
      uint32_t v[cs];
#pragma unroll
      for (int r = 0; r < cs; ++r) v[r] = cluster.map_shared_rank(s_hist, r)[bin];  // all loads in flight
      uint32_t sum = 0u;
#pragma unroll
      for (int r = 0; r < cs; ++r) sum += v[r];
      s_tot[g * SBmax + j] = sum;
    }
    __syncthreads();
    if (warp < G && sh.mode[warp] == 0u) {
      uint32_t v = 0u;
      for (int j = lane; j < SB; j += 32) v += s_tot[warp * SBmax + j];
      v = warp_sum(v);
      if (lane == 0) sh.slsum[warp] = v;
    }
    __syncthreads();
    cluster.sync();  // slice totals complete
    // every CTA: the digit holding the need-th largest (warp g for head g)
    if (warp < G && sh.mode[warp] == 0u) {
      const int g = warp;
      const uint32_t need = sh.need[g];
      // slices in descending digit order: slice r covers digits [r·SB, (r+1)·SB)
      const uint32_t mine = lane < cs ? *cluster.map_shared_rank(&sh.slsum[g], lane) : 0u;
      // suffix sums over slices (higher slice = larger digits)
      uint32_t suf = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_down_sync(kFull, suf, o);
        if (lane + o < 32) suf += t;
      }
      const uint32_t above_s = suf - mine;  // rows in slices above this one
      const bool hit = lane < cs && above_s < need && need <= suf;
      const unsigned hm = __ballot_sync(kFull, hit);
      const int s_star = hm ? __ffs(hm) - 1 : 0;
      const uint32_t above0 = __shfl_sync(kFull, above_s, s_star);
      // digits of slice s_star, descending: lane handles SB/32 consecutive digits
      const uint32_t* tot = cluster.map_shared_rank(s_tot, s_star) + g * SBmax;
      const int per = (SB + 31) / 32;
      uint32_t loc[16];
      uint32_t sum = 0u;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int pos = lane * per + j;  // descending position inside the slice
        loc[j] = (j < per && pos < SB) ? tot[SB - 1 - pos] : 0u;
        sum += loc[j];
      }
      uint32_t incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += t;
      }
      uint32_t cum = above0 + incl - sum;
      const uint32_t need_local = need;
      const bool in = cum < need_local && need_local <= cum + sum;
      if (in) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (j < per && cum + loc[j] >= need_local) {
            sh.dstar[g] = static_cast<uint32_t>(s_star * SB + SB - 1 - (lane * per + j));
            sh.above[g] = cum;
            sh.bcnt[g] = loc[j];
            break;
          }
          cum += loc[j];
        }
      }
    }
    __syncthreads();
    if (tid < G && sh.mode[tid] == 0u) {
      const int g = tid;
      const uint32_t need = sh.need[g] - sh.above[g];
      const uint32_t pre = (sh.prefix[g] << width) | sh.dstar[g];
      sh.need[g] = need;
      sh.prefix[g] = pre;
      sh.hshift[g] = static_cast<uint32_t>(shf);
      if (sh.bcnt[g] == need) {  // the whole bucket: threshold = its lower bound
        sh.mode[g] = 1u;
        sh.T[g] = static_cast<uint64_t>(pre << shf) << 32;
      } else if (sh.bcnt[g] <= static_cast<uint32_t>(kMemCap)) {
        sh.mode[g] = 2u;
      } else if (level == 2) {
        sh.mode[g] = 3u;  // a run of > kMemCap exactly equal keys
        sh.tkey[g] = pre;
      }
    }
    __syncthreads();
  }
  // ---- threshold-bucket members (mode 2): each CTA compacts its own into its shared memory
  // (s_mem aliases s_hist: after the last level's second barrier nobody reads it remotely)
  bool any_mem = false;
  for (int g = 0; g < G; ++g) any_mem |= sh.mode[g] == 2u;
  if (any_mem) {
    for (int g = 0; g < G; ++g) {
      if (sh.mode[g] != 2u) continue;
      const uint32_t pre = sh.prefix[g], hs = sh.hshift[g];
      const uint32_t* keys = s_key + g * R;
      uint64_t* mem = s_mem + g * kMemCap;
      for (int base = 0; base < nrow; base += GT) {
        const int i = base + tid;
        const uint32_t key = i < nrow ? keys[i] : 0u;
        const bool inb = i < nrow && (key >> hs) == pre;
        const unsigned bm = __ballot_sync(kFull, inb);
        if (!bm) continue;
        uint32_t wb = 0;
        if (lane == 0) wb = atomicAdd(&sh.nmem[g], __popc(bm));
        wb = __shfl_sync(kFull, wb, 0);
        if (inb) {
          const uint32_t slot = wb + __popc(bm & lanemask_lt());
          if (slot < static_cast<uint32_t>(kMemCap)) mem[slot] = make_comp(key, static_cast<uint32_t>(p.row_offset + r0 + i));
        }
      }
    }
  }
  GRP_PHASE(48);
  cluster.sync();  // every CTA's kmax and bucket members are final
  // cluster maximum score per head (softmax reference, attention.py:109-114 subtracts the max)
  if (warp < G) {
    const uint32_t m = lane < cs ? *cluster.map_shared_rank(&sh.kmax[warp], lane) : 0u;
    uint32_t mm = m;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mm = max(mm, __shfl_xor_sync(kFull, mm, o));
    if (lane == 0) sh.mscore[warp] = key_score(mm);
  }
  if (any_mem) {
    // owners pull the other CTAs' members behind their own (all remote loads in flight at once),
    // then rank-select the exact threshold composite
    for (int g = rank; g < G; g += cs) {
      if (sh.mode[g] != 2u) continue;
      uint32_t* start = sh.scr;      // [cs] first slot of each rank's block (own block at 0)
      uint32_t* cnt = sh.scr + 16;   // [cs] members of each foreign rank (own: 0)
      if (warp == 0) {
        const uint32_t c = lane < cs ? min(*cluster.map_shared_rank(&sh.nmem[g], lane), static_cast<uint32_t>(kMemCap)) : 0u;
        const uint32_t own = __shfl_sync(kFull, c, rank);
        const uint32_t c2 = lane == rank ? 0u : c;
        uint32_t inc = c2;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t t = __shfl_up_sync(kFull, inc, o);
          if (lane >= o) inc += t;
        }
        if (lane < cs) {
          start[lane] = own + inc - c2;
          cnt[lane] = c2;
        }
        if (lane == 31) sh.out2[0] = min(own + inc, static_cast<uint32_t>(kMemCap));
        if (lane == 0) sh.out2[1] = own;
      }
      __syncthreads();
      uint64_t* mem = s_mem + g * kMemCap;
      const uint32_t total = sh.out2[0];
      for (uint32_t i = sh.out2[1] + tid; i < total; i += GT) {
        int r = 0;
#pragma unroll
        for (int rr = 0; rr < cs; ++rr)
          if (cnt[rr] && i >= start[rr]) r = rr;  // blocks are in rank order
        mem[i] = cluster.map_shared_rank(s_mem, r)[g * kMemCap + (i - start[r])];
      }
      __syncthreads();
      const int m = static_cast<int>(total);
      const int need = static_cast<int>(sh.need[g]);
      uint64_t T;
      if (m <= 256) {
        T = block_rank_select<GT>(mem, m, need, &sh.res);
      } else {
        int cs_ = 64;
        uint64_t cp = 0;
        auto ld = [&](int64_t i, uint64_t& c) {
          c = mem[i];
          return true;
        };
        radix_select_u64<GT>(ld, m, static_cast<uint32_t>(need), s_tot /* 256 bins, free here */, sh.scr + 32,
                             sh.out2, cs_, cp);
        T = cp << cs_;
      }
      if (tid == 0) sh.T[g] = T;
      __syncthreads();
    }
    cluster.sync();  // thresholds published by the owners (and every pull done)
    if (tid < G && sh.mode[tid] == 2u) sh.T[tid] = *cluster.map_shared_rank(&sh.T[tid], tid % cs);
    __syncthreads();
  }

  GRP_PHASE(49);
  // ---- 3. selection counts. Warp w owns the contiguous rows [w·WR, (w+1)·WR) of this CTA and
  // walks them 32 at a time (lane = row, conflict-free), so ballots give row-ordered ranks.
  const int WR = ((nrow + GW - 1) / GW + 31) & ~31;
  const int w0 = warp * WR, w1 = min(nrow, w0 + WR);
  const unsigned lt = lanemask_lt();
  uint32_t c_gt[8], c_tie[8];
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    c_gt[g] = c_tie[g] = 0u;
    if (g >= G) continue;
    const uint32_t* keys = s_key + g * R;
    const uint32_t md = sh.mode[g], tk = sh.tkey[g];
    const uint64_t T = sh.T[g];
    for (int i = w0 + lane; i - lane < w1; i += 32) {
      const bool v = i < w1;
      const uint32_t key = v ? keys[i] : 0u;
      bool gt, tie = false;
      if (md == 3u) {
        gt = v && key > tk;
        tie = v && key == tk;
      } else {
        gt = v && make_comp(key, static_cast<uint32_t>(p.row_offset + r0 + i)) >= T;
      }
      c_gt[g] += __popc(__ballot_sync(kFull, gt));
      c_tie[g] += __popc(__ballot_sync(kFull, tie));
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      if (g >= G) continue;
      s_tot[g * 32 + warp] = c_gt[g];  // per-warp counts (s_tot is free again)
      s_tot[256 + g * 32 + warp] = c_tie[g];
    }
  }
  __syncthreads();
  if (warp < G) {  // warp g: exclusive per-warp offsets of head g, and the CTA totals
    const int g = warp;
    const uint32_t a = lane < GW ? s_tot[g * 32 + lane] : 0u, t = lane < GW ? s_tot[256 + g * 32 + lane] : 0u;
    uint32_t ia = a, it = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t ua = __shfl_up_sync(kFull, ia, o), ut = __shfl_up_sync(kFull, it, o);
      if (lane >= o) {
        ia += ua;
        it += ut;
      }
    }
    if (lane < GW) {
      s_tot[512 + g * 32 + lane] = ia - a;
      s_tot[768 + g * 32 + lane] = it - t;
    }
    if (lane == 31) {
      sh.cnt_gt[g] = ia;
      sh.cnt_tie[g] = it;
    }
  }
  __syncthreads();
  cluster.sync();  // every CTA's counts published
  // output ranges: selected rows of lower-ranked CTAs; mode 3 takes tied rows in rank order
  if (warp < G) {
    const int g = warp;
    const uint32_t gt_r = lane < cs ? *cluster.map_shared_rank(&sh.cnt_gt[g], lane) : 0u;
    const uint32_t tie_r = lane < cs ? *cluster.map_shared_rank(&sh.cnt_tie[g], lane) : 0u;
    uint32_t it = tie_r;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t ut = __shfl_up_sync(kFull, it, o);
      if (lane >= o) it += ut;
    }
    const uint32_t tie_ex = it - tie_r;
    const uint32_t need = sh.mode[g] == 3u ? sh.need[g] : 0u;
    const uint32_t take = tie_ex >= need ? 0u : min(tie_r, need - tie_ex);
    const uint32_t sel = gt_r + take;
    uint32_t is = sel;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t us = __shfl_up_sync(kFull, is, o);
      if (lane >= o) is += us;
    }
    if (lane == rank) {
      sh.out_base[g] = is - sel;
      sh.tie_base[g] = tie_ex;
      sh.sel[g] = sel;
    }
  }
  __syncthreads();

  GRP_PHASE(50);
  // ---- 4. emit idx / scores (row order) and stage the gather lists; gather in rounds of
  // kListCap rows per head (usually one)
  const float zs = p.scale * kLog2e;
  const int half = lane >> 4, part = lane & 15;
  const int wph = GW / G;          // warps per head in the gather
  const int hg = warp / wph;       // this warp's head
  const int wi = warp - hg * wph;  // its index among the head's warps
  float acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = 0.f;
  float lw = 0.f;
  uint32_t max_sel = 0u;
  for (int g = 0; g < G; ++g) max_sel = max(max_sel, sh.sel[g]);
  const int rounds = p.gather ? max(1, static_cast<int>((max_sel + kListCap - 1) / kListCap)) : 1;
  for (int rd = 0; rd < rounds; ++rd) {
    __syncthreads();  // previous round's lists consumed
    for (int g = 0; g < G; ++g) {
      const uint32_t* keys = s_key + g * R;
      const uint32_t md = sh.mode[g], tk = sh.tkey[g], need = sh.need[g];
      const uint64_t T = sh.T[g];
      // ranks of this warp's first row: selected rows before it in this CTA; tied rows before
      // it in the cluster (mode 3)
      uint32_t tie_rank = sh.tie_base[g] + s_tot[768 + g * 32 + warp];
      uint32_t local = s_tot[512 + g * 32 + warp];
      if (md == 3u) {
        const uint32_t tb = sh.tie_base[g], tw = s_tot[768 + g * 32 + warp];
        local += tb >= need ? 0u : min(tw, need - tb);
      }
      const int bh = bh0 + g;
      const float zref = sh.mscore[g] * zs;
      int32_t* idx_o = p.idx_out + static_cast<int64_t>(bh) * p.k;
      float* sc_o = p.scores_out + static_cast<int64_t>(bh) * p.k;
      uint64_t* pk_o = p.packed_out ? p.packed_out + static_cast<int64_t>(bh) * p.k : nullptr;
      const uint32_t lo = static_cast<uint32_t>(rd) * kListCap, hi = lo + kListCap;
      for (int i = w0 + lane; i - lane < w1; i += 32) {
        const bool v = i < w1;
        const uint32_t key = v ? keys[i] : 0u;
        const uint32_t gid = static_cast<uint32_t>(p.row_offset + r0 + i);
        bool sel;
        if (md == 3u) {
          const bool tie = v && key == tk;
          const unsigned tm = __ballot_sync(kFull, tie);
          sel = (v && key > tk) || (tie && tie_rank + __popc(tm & lt) < need);
          tie_rank += __popc(tm);
        } else {
          sel = v && make_comp(key, gid) >= T;
        }
        const unsigned sm_ = __ballot_sync(kFull, sel);
        const uint32_t my = local + __popc(sm_ & lt);
        local += __popc(sm_);
        if (!sel) continue;
        if (rd == 0) {
          const uint32_t o = sh.out_base[g] + my;
          if (o < static_cast<uint32_t>(kb)) {
            idx_o[o] = static_cast<int32_t>(gid);
            sc_o[o] = key_score(key);
            if (pk_o) pk_o[o] = make_comp(key, gid);
          }
          mark_pinned(p, bh, r0 + i);
        }
        if (p.gather && my >= lo && my < hi) {
          s_lrow[g * kListCap + (my - lo)] = static_cast<int32_t>(r0 + i);
          s_lw[g * kListCap + (my - lo)] = exp2f(fmaf(key_score(key), zs, -zref));
        }
      }
    }
    __syncthreads();
    if (!p.gather) break;
    // gather this round's rows: the warps of head hg, 8 rows in flight per half-warp
    const uint32_t done = static_cast<uint32_t>(rd) * kListCap;
    const int n_g = sh.sel[hg] > done ? static_cast<int>(min(sh.sel[hg] - done, static_cast<uint32_t>(kListCap))) : 0;
    const __nv_bfloat16* vb = p.vc + head_off + part * 8;
    const int32_t* lrow = s_lrow + hg * kListCap;
    const float* lwt = s_lw + hg * kListCap;
    constexpr int UNR = 8;
    for (int r = wi * 2 + half; r < n_g; r += 2 * wph * UNR) {
      uint4 v[UNR];
      float w[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int rr = r + 2 * wph * u;
        w[u] = rr < n_g ? lwt[rr] : 0.f;
        v[u] = rr < n_g ? ldg_stream(vb + static_cast<int64_t>(lrow[rr]) * kD) : make_uint4(0, 0, 0, 0);
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
    for (int r = wi * 32 + lane; r < n_g; r += wph * 32) lw += lwt[r];
  }

  GRP_PHASE(51);
  // ---- head metadata and pads (owner), then the gather partials (every CTA, slot = rank)
  for (int g = rank; g < G; g += cs) {
    const int bh = bh0 + g;
    if (tid == 0) {
      // the workspace's head metadata (const in AttendParams: the gather kernels only read it)
      const_cast<int32_t*>(p.meta_kb)[bh] = static_cast<int32_t>(kb);
      const_cast<float*>(p.meta_max)[bh] = kb > 0 ? sh.mscore[g] : -INFINITY;
      const_cast<uint64_t*>(p.meta_kth)[bh] = sh.mode[g] == 3u ? static_cast<uint64_t>(sh.tkey[g]) << 32 : sh.T[g];
    }
    for (int64_t i = kb + tid; i < p.k; i += GT) {  // pads for k > n_ctx (attention.py:147-149)
      p.idx_out[static_cast<int64_t>(bh) * p.k + i] = -1;
      p.scores_out[static_cast<int64_t>(bh) * p.k + i] = -INFINITY;
      if (p.packed_out) p.packed_out[static_cast<int64_t>(bh) * p.k + i] = 0ull;
    }
  }
  if (p.gather) {
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] += __shfl_xor_sync(kFull, acc[j], 16);
    if (half == 0) {
#pragma unroll
      for (int j = 0; j < 8; ++j) sh.red[warp][part * 8 + j] = acc[j];
    }
    lw = warp_sum(lw);
    if (lane == 0) sh.lsum[warp] = lw;
    __syncthreads();
    for (int e = tid; e < G * kD; e += GT) {
      const int g = e / kD, d = e - g * kD;
      float o = 0.f;
      for (int w2 = g * wph; w2 < (g + 1) * wph; ++w2) o += sh.red[w2][d];
      p.part_o[(static_cast<int64_t>(bh0 + g) * p.nchunks + rank) * kD + d] = o;
    }
    if (tid < G) {
      float l = 0.f;
      for (int w2 = tid * wph; w2 < (tid + 1) * wph; ++w2) l += sh.lsum[w2];
      p.part_l[static_cast<int64_t>(bh0 + tid) * p.nchunks + rank] = l;
    }
  }
  __threadfence();
  cluster.sync();  // partials, pin marks and meta visible to the owners
  GRP_PHASE(52);

  // ---- 5. owners finish their heads (pinned prefix, window, normalisation): first 8 warps
  if (p.gather && tid < kAttendThreads) {
    for (int g = rank; g < G; g += cs) head_finish<WarpGrp<0, kAttendThreads, 1>>(p, bh0 + g, cs, sh.att);
    if (rank < G) GRP_PHASE(53);
  }
  // ---- the last cluster of batch entry b advances its window counter (decode step)
  if (gp.k_new && rank == 0 && tid == 0) {
    __threadfence();
    if (atomicAdd(&gp.win_ticket[b], 1u) == static_cast<uint32_t>(p.Hkv - 1)) {
      gp.win_ticket[b] = 0u;
      const int32_t cnt = gp.win_count[b];
      if (N + cnt < p.cache_rows) gp.win_count[b] = cnt + 1;
    }
  }
}

int group_max_rows(int G) { return kGrpKeyBytes / (G * 4); }

size_t group_smem_bytes(int G, int rows_per_cta, int cs) {
  const size_t keys = static_cast<size_t>(G) * rows_per_cta * 4;
  const size_t hist = static_cast<size_t>(G) * kGrpBins * 4;  // >= members / gather lists (G x 8 KB)
  size_t tot = static_cast<size_t>(G) * (kGrpBins / cs) * 4;
  if (tot < 32 * 32 * 4) tot = 32 * 32 * 4;  // reused for the block prefix sums of the counts
  return keys + hist + tot;
}

template <int CS>
static cudaError_t group_attributes_cs() {
  cudaError_t e = cudaFuncSetAttribute(group_topk_kernel<CS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       227 * 1024 - static_cast<int>(sizeof(GrpShared)) - 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(group_topk_kernel<CS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  return e;
}
static cudaError_t group_attributes() {
  return static_cast<cudaError_t>(per_device(reinterpret_cast<const void*>(group_topk_kernel<16>), 0, [] {
    cudaError_t e = group_attributes_cs<4>();
    if (e == cudaSuccess) e = group_attributes_cs<8>();
    if (e == cudaSuccess) e = group_attributes_cs<16>();
    return static_cast<int>(e);
  }));
}

cudaError_t launch_group(const GroupParams& p, cudaStream_t s) {
  const cudaError_t attr = group_attributes();
  if (attr != cudaSuccess) return attr;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.a.B * p.a.Hkv * p.cs);
  cfg.blockDim = dim3(GT);
  cfg.dynamicSmemBytes = group_smem_bytes(p.a.G, p.rows_per_cta, p.cs);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = p.cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  switch (p.cs) {
    case 4: return cudaLaunchKernelEx(&cfg, group_topk_kernel<4>, p);
    case 8: return cudaLaunchKernelEx(&cfg, group_topk_kernel<8>, p);
    case 16: return cudaLaunchKernelEx(&cfg, group_topk_kernel<16>, p);
    default: return cudaErrorInvalidValue;
  }
}

// Largest cluster size (16, 8, 4, 2) whose clusters can be resident with this shared memory,
// or 0 (queried once per device and size)
int group_cluster_ok(int cs, size_t smem) {
  if (group_attributes() != cudaSuccess) return 0;
  if (smem + sizeof(GrpShared) + 1024 > 227 * 1024) return 0;
  return per_device(reinterpret_cast<const void*>(group_topk_kernel<16>), 1000 + cs * 1000000 + static_cast<int>(smem / 1024),
                    [cs, smem] {
                      cudaLaunchConfig_t cfg{};
                      cfg.gridDim = dim3(cs);
                      cfg.blockDim = dim3(GT);
                      cfg.dynamicSmemBytes = smem;
                      cudaLaunchAttribute at[1];
                      at[0].id = cudaLaunchAttributeClusterDimension;
                      at[0].val.clusterDim.x = cs;
                      at[0].val.clusterDim.y = 1;
                      at[0].val.clusterDim.z = 1;
                      cfg.attrs = at;
                      cfg.numAttrs = 1;
                      int n = 0;
                      const cudaError_t e = cs == 4   ? cudaOccupancyMaxActiveClusters(&n, group_topk_kernel<4>, &cfg)
                                            : cs == 8 ? cudaOccupancyMaxActiveClusters(&n, group_topk_kernel<8>, &cfg)
                                                      : cudaOccupancyMaxActiveClusters(&n, group_topk_kernel<16>, &cfg);
                      if (e != cudaSuccess) {
                        cudaGetLastError();
                        n = 0;
                      }
                      return n;
                    });
}

}  // namespace tkv
