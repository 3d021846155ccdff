// common.cuh — shared device helpers for the sm_100a top-k decode-attention kernels.
//
// Numerics contract (reference: ann_kernels.py:31-47, ann.py:154-167, attention.py:107-167):
//   * scores are raw dot products q·K[row] of bf16 inputs; products are exact in fp32 and the
//     128-term sum is accumulated in fp32 on the tensor cores (HMMA, fp32 accumulate). The
//     reference accumulates in f64; the difference (~1e-6 relative) is far inside the
//     near-tie exemption of the parity contract (|Δs| < 1e-3·|s_k|).
//   * selection order is the reference's: larger score first, ties to the LOWER row id
//     (ann.py:162-166). It is realised as one 64-bit composite per row:
//        comp = (order-preserving key of the f32 score) << 32 | ~global_row_id
//     so "top-k by composite, descending" == reference order, and composites are unique.
//   * -0.0 is canonicalised to +0.0 before keying (the reference compares f64 values, where
//     -0.0 == +0.0 and the lower id wins).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace tkv {

constexpr int kD = 128;                 // head dim this build supports
constexpr unsigned kFull = 0xffffffffu;
constexpr float kLog2e = 1.4426950408889634f;

// ---------------------------------------------------------------- score keys / composites
__device__ __forceinline__ uint32_t score_key(float f) {
  uint32_t b = __float_as_uint(f);
  if (b == 0x80000000u) b = 0u;  // -0.0 -> +0.0
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key_score(uint32_t k) {
  uint32_t b = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(b);
}
__device__ __forceinline__ uint64_t make_comp(uint32_t key, uint32_t gid) {
  return (static_cast<uint64_t>(key) << 32) | static_cast<uint32_t>(~gid);
}
__device__ __forceinline__ uint32_t comp_gid(uint64_t c) { return ~static_cast<uint32_t>(c); }
__device__ __forceinline__ uint32_t comp_key(uint64_t c) { return static_cast<uint32_t>(c >> 32); }

// ---------------------------------------------------------------- memory
// Streaming 128-bit load: read-only path, no L1 allocation, 256B L2 prefetch (K is read once).
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// Gather load (V rows): read-only path, no L1 allocation.
__device__ __forceinline__ uint4 ldg_nc(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ uint32_t u4_word(const uint4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// ---------------------------------------------------------------- HMMA key-scan tile
// One warp scores a 16-row × 128 tile of K against up to 8 q heads of one GQA group with
// 8 × mma.m16n8k16 (bf16 in, fp32 accumulate). The k-dimension is permuted so that every
// thread's A/B fragments come straight from 16-byte contiguous global loads (no shared
// memory, no ldmatrix):
//   thread (g = lane/4, c = lane%4) loads, for its rows g and g+8, the 16-byte chunks
//   j = 0..3 at element offset 32*j + 8*c  (a warp instruction covers 64 contiguous bytes of
//   each of 8 rows = whole 32-byte sectors);
//   mma step s = 2*j + h consumes elements 32*j + 8*c + 4*h + {0,1,2,3} of that chunk as the
//   A slots {2c, 2c+1, 2c+8, 2c+9}; the B fragment (q head n = g) uses the same map.
// The accumulator layout is the standard one:
//   acc[0] = S[row g][head 2c], acc[1] = S[row g][head 2c+1],
//   acc[2] = S[row g+8][head 2c], acc[3] = S[row g+8][head 2c+1].
// A row's score depends only on that row and q (fixed step order 0..7), so any kernel that
// scores a row with this function gets bit-identical values (used for pinned-row membership).
struct QFrag {
  uint32_t w[8][2];
};

__device__ __forceinline__ void load_qfrag(QFrag& f, const __nv_bfloat16* qgroup, int G, int lane) {
  const int g = lane >> 2, c = lane & 3;
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    if (g < G) {
      const uint2 v = *reinterpret_cast<const uint2*>(qgroup + g * kD + 32 * (s >> 1) + 8 * c +
                                                      4 * (s & 1));
      f.w[s][0] = v.x;
      f.w[s][1] = v.y;
    } else {
      f.w[s][0] = 0u;
      f.w[s][1] = 0u;
    }
  }
}

__device__ __forceinline__ void mma_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                          uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// rowA / rowB: pointers to the two rows this thread loads (row g and row g+8 of the tile);
// invalid rows are zero-filled (never dereferenced).
__device__ __forceinline__ void load_tile(uint4 (&a)[2][4], const __nv_bfloat16* rowA, bool okA,
                                          const __nv_bfloat16* rowB, bool okB, int c) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    a[0][j] = okA ? ldg_stream(rowA + 32 * j + 8 * c) : make_uint4(0, 0, 0, 0);
    a[1][j] = okB ? ldg_stream(rowB + 32 * j + 8 * c) : make_uint4(0, 0, 0, 0);
  }
}

__device__ __forceinline__ void score_tile(float (&acc)[4], const uint4 (&a)[2][4], const QFrag& f) {
  acc[0] = acc[1] = acc[2] = acc[3] = 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int s = 2 * j + h;
      mma_16816(acc, u4_word(a[0][j], 2 * h), u4_word(a[1][j], 2 * h), u4_word(a[0][j], 2 * h + 1),
                u4_word(a[1][j], 2 * h + 1), f.w[s][0], f.w[s][1]);
    }
  }
}

// ---------------------------------------------------------------- candidate histogram
// Emitted candidates have key >= thr; their histogram bucket is the key offset above the
// threshold at a per-head granularity `shift` (chosen from the sampled score range so the
// candidates spread over the buckets instead of piling into a few top-bit buckets),
// clamped into the top bucket.
constexpr int kHistBins = 4096;
__device__ __forceinline__ uint32_t hist_digit(uint32_t key, uint32_t thr, uint32_t shift) {
  const uint32_t d = (key - thr) >> shift;
  return d < static_cast<uint32_t>(kHistBins - 1) ? d : static_cast<uint32_t>(kHistBins - 1);
}

// Warp-aggregated shared-memory histogram increment: lanes with equal digits combine into one
// atomic (score keys are concentrated, so per-lane atomics would serialise on a few bins).
__device__ __forceinline__ void hist_add_aggregated(uint32_t* hist, uint32_t digit) {
  const unsigned peers = __match_any_sync(__activemask(), digit);
  if ((threadIdx.x & 31) == static_cast<unsigned>(__ffs(peers) - 1)) atomicAdd(&hist[digit], __popc(peers));
}

// ---------------------------------------------------------------- thread groups
// Block-wide helpers run on a thread group: the whole CTA (default), or a contiguous range of
// warps synchronised by a named barrier (the work-queue warps of the warp-specialised layer
// kernel run beside the tcgen05 scan warps, which must not take part in their barriers).
struct CtaGrp {
  __device__ static __forceinline__ int tid() { return static_cast<int>(threadIdx.x); }
  __device__ static __forceinline__ void sync() { __syncthreads(); }
};
template <int kBase, int kCount, int kBarId>
struct WarpGrp {
  static_assert(kBase % 32 == 0 && kCount % 32 == 0 && kBarId > 0 && kBarId < 16, "warp-aligned group");
  __device__ static __forceinline__ int tid() { return static_cast<int>(threadIdx.x) - kBase; }
  __device__ static __forceinline__ void sync() { asm volatile("bar.sync %0, %1;" ::"n"(kBarId), "n"(kCount) : "memory"); }
};

// Copy n (multiple of 4, 16-byte aligned) u32 words global → shared with every load of a
// thread issued before its first store (one memory round trip instead of n / NT). L2 path.
template <int NT, int MAXN, class Gp = CtaGrp>
__device__ __forceinline__ void copy_g2s_u32(uint32_t* dst, const uint32_t* src, int n) {
  constexpr int PER = (MAXN / 4 + NT - 1) / NT;
  uint4 v[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int i = (u * NT + Gp::tid()) * 4;
    v[u] = i < n ? __ldcg(reinterpret_cast<const uint4*>(src + i)) : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int i = (u * NT + Gp::tid()) * 4;
    if (i < n) *reinterpret_cast<uint4*>(dst + i) = v[u];
  }
}

// ---------------------------------------------------------------- small-set selection
// need-th largest (1-indexed) of m values in shared memory by rank counting: thread-parallel
// O(m^2 / NT) compares, two barriers — for the few hundred elements of a threshold bucket
// this beats any multi-pass radix. Duplicates allowed: returns the value v with
// #{> v} < need <= #{>= v}. Result broadcast through *out. Block-wide call.
template <int NT, typename T, class Gp = CtaGrp>
__device__ __forceinline__ T block_rank_select(const T* vals, int m, int need, T* out) {
  for (int i = Gp::tid(); i < m; i += NT) {
    const T v = vals[i];
    int gt = 0, ge = 0;
    for (int j = 0; j < m; ++j) {
      const T w = vals[j];
      gt += w > v;
      ge += w >= v;
    }
    if (gt < need && need <= ge) *out = v;  // all qualifying threads hold the same value
  }
  Gp::sync();
  const T r = *out;
  Gp::sync();
  return r;
}

// Same contract as block_rank_select, with the compare loop split over P = NT / m threads per
// element (P a power of two <= 32, the element's threads adjacent lanes) so that small sets
// (a few hundred elements) take a few hundred cycles instead of m dependent shared loads.
template <int NT, typename T, class Gp = CtaGrp>
__device__ __forceinline__ T block_rank_select_par(const T* vals, int m, int need, T* out) {
  if (m > NT / 2) return block_rank_select<NT, T, Gp>(vals, m, need, out);
  int P = 1;
  while (P < 32 && P * 2 * m <= NT) P <<= 1;
  const int tid = Gp::tid();
  const int i = tid / P, sub = tid % P;
  int gt = 0, ge = 0;
  T v{};
  if (i < m) {
    v = vals[i];
    for (int j = sub; j < m; j += P) {
      const T w = vals[j];
      gt += w > v;
      ge += w >= v;
    }
  }
  for (int o = 1; o < P; o <<= 1) {  // the P threads of element i are lanes of one warp
    gt += __shfl_xor_sync(kFull, gt, o);
    ge += __shfl_xor_sync(kFull, ge, o);
  }
  if (i < m && sub == 0 && gt < need && need <= ge) *out = v;
  Gp::sync();
  const T r = *out;
  Gp::sync();
  return r;
}

// ---------------------------------------------------------------- block helpers
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
  return v;
}
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t t = __shfl_xor_sync(kFull, v, o);
    v = t > v ? t : v;
  }
  return v;
}
__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t t = __shfl_xor_sync(kFull, v, o);
    v = t < v ? t : v;
  }
  return v;
}

// Given a histogram hist[NB] (shared memory), find the bucket d* in LARGEST-first order such
// that above(d*) < need <= above(d*) + hist[d*], where above(d) = sum of hist over buckets > d.
// Requires 1 <= need <= sum(hist). Result in out[0] = d*, out[1] = above(d*). Block-wide;
// every thread must call it. scratch: >= NT/32 words.
template <int NT, int NB, class Gp = CtaGrp>
__device__ __forceinline__ void find_bucket(const uint32_t* hist, uint32_t need, uint32_t* out,
                                            uint32_t* scratch) {
  constexpr int PER = (NB + NT - 1) / NT;
  const int tid = Gp::tid(), lane = tid & 31, warp = tid >> 5;
  uint32_t local[PER];
  uint32_t sum = 0;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int pos = tid * PER + j;  // descending position
    local[j] = pos < NB ? hist[NB - 1 - pos] : 0u;
    sum += local[j];
  }
  // block exclusive scan of `sum`
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) scratch[warp] = incl;
  Gp::sync();
  if (warp == 0) {
    constexpr int NW = NT / 32;
    uint32_t w = lane < NW ? scratch[lane] : 0u;
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(kFull, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < NW) scratch[lane] = wi - w;  // exclusive warp offsets
  }
  Gp::sync();
  const uint32_t excl = scratch[warp] + incl - sum;
  if (excl < need && need <= excl + sum) {
    uint32_t cum = excl;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      if (cum + local[j] >= need) {
        out[0] = NB - 1 - (tid * PER + j);
        out[1] = cum;
        break;
      }
      cum += local[j];
    }
  }
  Gp::sync();
}

// ---------------------------------------------------------------- generic radix select
// Radix select of the `need` largest composites among the elements accepted by `load`
// (load(i, c) -> bool), MSB first with 8-bit digits. Result: selected ⇔ (c >> shift) >= prefix.
template <int T, typename Load, class Gp = CtaGrp>
__device__ void radix_select_u64(Load load, int64_t n, uint32_t need, uint32_t* hist, uint32_t* scr,
                                 uint32_t* out, int& shift_out, uint64_t& prefix_out) {
  int shift = 64;
  uint64_t prefix = 0;
  while (shift > 0) {
    const int nshift = shift - 8;
    for (int i = Gp::tid(); i < 256; i += T) hist[i] = 0u;
    Gp::sync();
    for (int64_t i = Gp::tid(); i < n; i += T) {
      uint64_t c;
      if (load(i, c) && (shift == 64 || (c >> shift) == prefix))
        hist_add_aggregated(hist, static_cast<uint32_t>(c >> nshift) & 255u);
    }
    Gp::sync();
    find_bucket<T, 256, Gp>(hist, need, out, scr);
    const uint32_t d = out[0];
    need -= out[1];
    prefix = (prefix << 8) | d;
    shift = nshift;
    const bool done = hist[d] == need;
    Gp::sync();
    if (done) break;
  }
  shift_out = shift;
  prefix_out = prefix;
}

// Programmatic dependent launch (sm_90+): a kernel launched with programmatic stream
// serialisation may start while its predecessor still runs; pdl_wait() blocks until the
// predecessor grid has completed and its memory is visible, pdl_trigger() lets this grid's
// successor launch early. Both are no-ops for ordinary launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Diagnostics (tkv_debug_timeline): first-start (slot 2e) / last-end (slot 2e+1) %globaltimer
// stamps of pipeline event e; tl == nullptr when not requested.
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// durations inside one CTA: the SM clock (%globaltimer ticks too coarsely for sub-us phases),
// scaled to ~ns at the B200's 1965 MHz boost clock
__device__ __forceinline__ uint64_t ptimer() { return static_cast<uint64_t>(clock64()) * 509ull / 1000ull; }
__device__ __forceinline__ void tl_start(uint64_t* tl, int e) {
  if (tl) atomicMin(reinterpret_cast<unsigned long long*>(tl + 2 * e), static_cast<unsigned long long>(gtimer()));
}
__device__ __forceinline__ void tl_end(uint64_t* tl, int e) {
  if (tl) atomicMax(reinterpret_cast<unsigned long long*>(tl + 2 * e + 1), static_cast<unsigned long long>(gtimer()));
}
// diagnostics: set this CTA's SM in the 3-word SM bitmask at tl[w]
__device__ __forceinline__ void tl_smid(uint64_t* tl, int w) {
  uint32_t sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  if (tl && sm < 192) atomicOr(reinterpret_cast<unsigned long long*>(tl + w + sm / 64), 1ull << (sm % 64));
}

// ---------------------------------------------------------------- mbarrier / bulk-copy PTX (sm_100a)
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
// cluster-scope hand-offs (thread-block clusters): arrive on a barrier in another CTA's shared
// memory (release at cluster scope: this thread's — and, after a CTA barrier, its CTA's — prior
// writes, DSMEM stores included, are visible to a thread that then acquires the barrier), and
// wait with acquire at cluster scope
__device__ __forceinline__ uint32_t mapa_shared(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
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
// 1-D bulk copy global → shared (async proxy), completion counted on mbarrier `bar`
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

// per-CTA phase durations: slot e accumulates (sum of ns, count) — averaged by tools/timeline.py
__device__ __forceinline__ void tl_phase(uint64_t* tl, int e, uint64_t& t_prev) {
  if (tl) {
    const uint64_t t = ptimer();
    atomicAdd(reinterpret_cast<unsigned long long*>(tl + 2 * e), static_cast<unsigned long long>(t - t_prev));
    atomicAdd(reinterpret_cast<unsigned long long*>(tl + 2 * e + 1), 1ull);
    t_prev = t;
  }
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

}  // namespace tkv
