// api.cu — extern "C" boundary of libtkv.so (declared in include/tkv.h).
//
// Host-side validation mirrors the reference's error behaviour where it can be checked
// without touching device data (errors.py:4-42; attention.py:144-145; ann.py:210-213;
// attention.py:122); the Python shim maps the status codes back onto the reference's
// exception classes. Device-resident values (n_ctx, n_win, finiteness of q/K) are not
// inspected here — that would cost a host synchronisation or a full scan.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/tkv.h"
#include "common.cuh"
#include "internal.h"

using namespace tkv;

namespace {

thread_local std::string g_err;
thread_local int g_launches = 0;
thread_local cudaEvent_t g_scan_start = nullptr, g_scan_stop = nullptr;
thread_local uint64_t* g_tl = nullptr;
thread_local bool g_staged = false;  // q staged by stage_kernel in this call (TKV_F_HOST_Q)

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define TKV_LAUNCH(expr)                                                            \
  do {                                                                              \
    cudaError_t e__ = (expr);                                                       \
    ++g_launches;                                                                   \
    if (e__ != cudaSuccess) return fail(TKV_ECUDA, "%s: %s", #expr, cudaGetErrorString(e__)); \
  } while (0)

// TopKResult ordering (one kernel up to kSortMax, chunk sort + merge passes above)
#define TKV_SORT(so, nbh, st)                                                          \
  do {                                                                              \
    int n__ = 0;                                                                    \
    cudaError_t e__ = launch_sort((so), (nbh), (st), &n__);                         \
    g_launches += n__;                                                              \
    if (e__ != cudaSuccess) return fail(TKV_ECUDA, "launch_sort: %s", cudaGetErrorString(e__)); \
  } while (0)

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Layout {
  size_t ticket_g, ticket_k, flag, gflag, fbl, fbh, mout, steal, ctrl_end;
  size_t maxc, bktc, bkt, outc;
  size_t cnt, thr, hshift, hist, mmax, mkth, mkb, mt2, ncnt, samp, cand, sidx, sscore, pl, po, pinm, qs, sortb, total;
  int pin_words;
  int64_t cap;
  int nchunks;
};

Layout make_layout(const tkv_problem* p) {
  Layout L{};
  const size_t BH = static_cast<size_t>(p->batch) * p->n_q_heads;
  const size_t BK = static_cast<size_t>(p->batch) * p->n_kv_heads;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + (bytes ? bytes : 1), 256);
    return o;
  };
  L.ticket_g = take(BH * 4);
  L.ticket_k = take(BH * 4);
  L.flag = take(BH * 4);
  L.gflag = take(BK * 4);
  L.fbl = take(4 * kMaxParts);
  L.fbh = take(4);
  L.mout = take(BH * 4);  // sharded merge output counters (self-resetting)
  L.steal = take(2 * 4 * kMaxParts);  // tcgen05 scan work pool, one counter pair per part (self-resetting)
  L.ctrl_end = off;
  L.cnt = take(BH * 4);
  L.thr = take(BH * 4);
  L.hshift = take(BH * 4);
  L.hist = take(BH * kHistBins * 4);
  L.maxc = take(BH * 8);
  L.bktc = take(BH * 4);
  L.outc = take(BH * 4);
  L.bkt = take(BH * kSelectBucketCap * 8);
  L.mmax = take(BH * 4);
  L.mkth = take(BH * 8);
  L.mkb = take(BH * 4);
  L.mt2 = take(BH * 8);  // sharded narrow-list bound t2 per head
  L.ncnt = take(BH * 4);  // sharded narrow-list append counters (zeroed by the k-th kernel)
  L.samp = take(BH * kSamples * 4);
  L.cap = p->max_ctx > 0 ? p->max_ctx : 1;
  L.cand = take(BH * static_cast<size_t>(L.cap) * 8);
  L.sidx = take(BH * static_cast<size_t>(p->k) * 4);
  L.sscore = take(BH * static_cast<size_t>(p->k) * 4);
  {
    // partial slots per head: list mode (k / kAttendChunk) or candidate mode (cap / kCandQuant)
    const int64_t a = (p->k + kAttendChunk - 1) / kAttendChunk;
    // candidate-mode items per head: ceil(quanta_h / S) <= min(quanta_h, grid + 1) (S =
    // ceil(all quanta / grid), grid <= kMaxGatherGrid)
    int64_t c = (L.cap + kCandQuant - 1) / kCandQuant + 1;
    c = c < kMaxGatherGrid + 1 ? c : kMaxGatherGrid + 1;
    const int64_t f = (p->k + kFlatMinRows - 1) / kFlatMinRows + 1;  // flat list gather ranges
    int64_t m = a > c ? a : c;
    L.nchunks = static_cast<int>(m > f ? m : f);
  }
  {
    const int64_t pin = p->pinned_prefix < p->max_ctx ? p->pinned_prefix : p->max_ctx;
    L.pin_words = pin > 0 ? static_cast<int>((pin + 31) / 32) : 0;
  }
  L.pinm = take(BH * static_cast<size_t>(L.pin_words) * 4);
  L.qs = take((BH + 2 * BK) * kD * 2);  // TKV_F_HOST_Q staging copies of q | k_new | v_new
  L.pl = take(BH * L.nchunks * 4);
  L.po = take(BH * L.nchunks * kD * 4);
  // large-k TopKResult ordering (k > kSortMax): merge ping-pong buffers
  L.sortb = take((p->flags & TKV_F_SORTED) && p->k > kSortMax ? 2 * BH * static_cast<size_t>(p->k) * 8 : 0);
  L.total = off;
  return L;
}

int validate(const tkv_problem* p) {
  if (!p) return fail(TKV_EBADSHAPE, "problem is NULL");
  if (p->batch < 1 || p->n_q_heads < 1 || p->n_kv_heads < 1)
    return fail(TKV_EBADSHAPE, "batch/heads must be >= 1 (got B=%d Hq=%d Hkv=%d)", p->batch,
                p->n_q_heads, p->n_kv_heads);
  if (p->n_q_heads % p->n_kv_heads != 0)
    return fail(TKV_EBADSHAPE, "Hq=%d not a multiple of Hkv=%d", p->n_q_heads, p->n_kv_heads);
  const int G = p->n_q_heads / p->n_kv_heads;
  if (G != 1 && G != 2 && G != 4 && G != 8)
    return fail(TKV_EBADSHAPE, "GQA group size Hq/Hkv=%d must be 1, 2, 4 or 8", G);
  if (p->head_dim != kD) return fail(TKV_EBADSHAPE, "head_dim=%d unsupported (this build: %d)", p->head_dim, kD);
  if (p->k < 1) return fail(TKV_EBADK, "k must be >= 1 (got %d)", p->k);
  if (p->max_ctx < 0 || p->max_ctx > 0x7fffffffLL)
    return fail(TKV_EBADSHAPE, "max_ctx=%lld out of range", static_cast<long long>(p->max_ctx));
  if (p->cache_rows < p->max_ctx)
    return fail(TKV_EBADSHAPE, "cache_rows=%lld < max_ctx=%lld", static_cast<long long>(p->cache_rows),
                static_cast<long long>(p->max_ctx));
  if (p->row_offset < 0 || p->row_offset + p->max_ctx > 0x7fffffffLL)
    return fail(TKV_EBADSHAPE, "row_offset=%lld out of range", static_cast<long long>(p->row_offset));
  if (p->combine != TKV_COMBINE_JOINT && p->combine != TKV_COMBINE_ADDITIVE)
    return fail(TKV_ECONFIG, "unknown combine mode %d", p->combine);
  if (p->pinned_prefix < 0) return fail(TKV_EBADK, "pinned_prefix must be >= 0");
  return TKV_OK;
}

int check_ptr(const void* ptr, const char* name, size_t align) {
  if (!ptr) return fail(TKV_EBADSHAPE, "%s is NULL", name);
  if (reinterpret_cast<uintptr_t>(ptr) % align)
    return fail(TKV_EBADSHAPE, "%s must be %zu-byte aligned", name, align);
  return TKV_OK;
}

int check_ws(const tkv_problem* p, void* ws, size_t bytes, Layout* L) {
  *L = make_layout(p);
  if (!ws) return fail(TKV_EWORKSPACE, "workspace is NULL");
  if (reinterpret_cast<uintptr_t>(ws) % 256) return fail(TKV_EWORKSPACE, "workspace must be 256-byte aligned");
  if (bytes < L->total)
    return fail(TKV_EWORKSPACE, "workspace too small: %zu < %zu bytes", bytes, L->total);
  return TKV_OK;
}

template <typename T>
T* at(void* ws, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(ws) + off);
}

#define TRY(x)                 \
  do {                         \
    const int r__ = (x);       \
    if (r__ != TKV_OK) return r__; \
  } while (0)

HeadState head_state(void* ws, const Layout& L) {
  HeadState hs{};
  hs.thr = at<uint32_t>(ws, L.thr);
  hs.hshift = at<uint32_t>(ws, L.hshift);
  hs.cand_cnt = at<uint32_t>(ws, L.cnt);
  hs.hist = at<uint32_t>(ws, L.hist);
  hs.flag_fail = at<uint32_t>(ws, L.flag);
  hs.group_fail = at<uint32_t>(ws, L.gflag);
  hs.max_comp = at<uint64_t>(ws, L.maxc);
  hs.bkt_cnt = at<uint32_t>(ws, L.bktc);
  hs.bkt = at<uint64_t>(ws, L.bkt);
  hs.kth_ticket = at<uint32_t>(ws, L.ticket_k);
  hs.out_cnt = at<uint32_t>(ws, L.outc);
  hs.fb_launched = at<uint32_t>(ws, L.fbl);
  hs.fb_heads = at<uint32_t>(ws, L.fbh);
  return hs;
}

// sample → threshold for every head; fills the scan / k-th parameter templates
// window append folded into threshold_kernel for this thread's next run_prefix (decode step)
struct AppendFold {
  const void* k_new = nullptr;
  const void* v_new = nullptr;
  void* k_cache = nullptr;
  void* v_cache = nullptr;
  int32_t* n_win = nullptr;
};
thread_local AppendFold g_fold;

int run_prefix(const tkv_problem* p, const void* q, const void* k_cache, const int32_t* n_ctx, void* ws,
               const Layout& L, cudaStream_t st, ScanParams* cp_out, SelectParams* sl_out) {
  const int G = p->n_q_heads / p->n_kv_heads;
  const HeadState hs = head_state(ws, L);
  SampleParams sp{};
  sp.q = static_cast<const __nv_bfloat16*>(q);
  sp.kc = static_cast<const __nv_bfloat16*>(k_cache);
  sp.cache_rows = p->cache_rows;
  sp.B = p->batch;
  sp.Hq = p->n_q_heads;
  sp.Hkv = p->n_kv_heads;
  sp.G = G;
  sp.k = p->k;
  sp.n_ctx = n_ctx;
  sp.no_filter = (p->flags & TKV_F_NO_FILTER) ? 1 : 0;
  sp.max_samples = sample_max(p->max_ctx, p->k);
  sp.samp = at<uint32_t>(ws, L.samp);
  sp.hs = hs;
  sp.tl = g_tl;
  sp.pin_words = L.pin_words;
  sp.pin_mask = L.pin_words ? at<uint32_t>(ws, L.pinm) : nullptr;
  sp.k_new = static_cast<const __nv_bfloat16*>(g_fold.k_new);
  sp.v_new = static_cast<const __nv_bfloat16*>(g_fold.v_new);
  sp.k_dst = static_cast<__nv_bfloat16*>(g_fold.k_cache);
  sp.v_dst = static_cast<__nv_bfloat16*>(g_fold.v_cache);
  sp.win_count = g_fold.n_win;
  g_fold = AppendFold{};
  sp.pdl = g_staged && pdl_enabled() ? 1 : 0;
  TKV_LAUNCH(launch_sample(sp, st));
  if (!sp.no_filter) ++g_launches;  // sample + threshold kernels

  ScanParams cp{};
  cp.q = sp.q;
  cp.kc = sp.kc;
  cp.cache_rows = p->cache_rows;
  cp.B = p->batch;
  cp.Hq = p->n_q_heads;
  cp.Hkv = p->n_kv_heads;
  cp.G = G;
  cp.max_ctx = p->max_ctx;
  cp.n_ctx = n_ctx;
  cp.row_offset = static_cast<uint32_t>(p->row_offset);
  cp.cand = at<uint64_t>(ws, L.cand);
  cp.cap = L.cap;
  cp.hs = hs;
  cp.fallback = 0;
  cp.tl = g_tl;
  cp.seg_begin = 0;
  cp.seg_count = static_cast<int64_t>(p->batch) * p->n_kv_heads;
  cp.steal = at<uint32_t>(ws, L.steal);

  SelectParams sl{};
  sl.src = cp.cand;
  sl.src_stride = L.cap;
  sl.B = p->batch;
  sl.Hq = p->n_q_heads;
  sl.Hkv = p->n_kv_heads;
  sl.G = G;
  sl.k = p->k;
  sl.n_ctx = n_ctx;
  sl.meta_max = at<float>(ws, L.mmax);
  sl.meta_kth = at<uint64_t>(ws, L.mkth);
  sl.meta_kb = at<int32_t>(ws, L.mkb);
  sl.hs = hs;
  sl.pass = kPassMain;
  sl.tl = g_tl;
  *cp_out = cp;
  *sl_out = sl;
  return TKV_OK;
}

}  // namespace

// Programmatic dependent launch between sample → threshold → scan → k-th (default on;
// TKV_PDL=0 disables it, e.g. for A/B timing).
bool tkv::pdl_enabled() { return diag_env("TKV_PDL", 1) != 0; }

namespace {

bool use_tc_scan(const tkv_problem* p, const ScanParams& cp) {
  return !(p->flags & TKV_F_SCAN_HMMA) && scan_tc_supported(cp);
}

// key scan of segments [s0, s1) on stream `st`
int run_scan_part(const tkv_problem* p, ScanParams cp, int64_t s0, int64_t s1, cudaStream_t st, bool pdl,
                  int part = 0, bool steal = true) {
  // the dynamic tail only where nothing absorbs the CTAs' uneven ends: in the chained parts
  // pipeline the next part's CTAs take over SMs as they free up (cfg5: 1448 us static, 1475-1490
  // with every part balanced, 1459 with the last part balanced), so the parts stay static
  cp.steal = steal ? cp.steal + 2 * part : nullptr;  // overlapping part scans each own a counter pair
  cp.seg_begin = s0;
  cp.seg_count = s1 - s0;
  cp.pdl = pdl ? 1 : 0;
  // the north star's CUDA-core FMA scan, kept for the ncu A/B (TKV_DIAG builds: TKV_SCAN_FMA=1)
  if (diag_env("TKV_SCAN_FMA", 0))
    TKV_LAUNCH(launch_scan_fma(cp, st));
  else if (use_tc_scan(p, cp))
    TKV_LAUNCH(launch_scan_tc(cp, st));
  else
    TKV_LAUNCH(launch_scan(cp, st));
  return TKV_OK;
}

// exact k-th threshold of the heads of segments [s0, s1) (+ the exactness fallback: re-scan /
// k-th of failing heads, tail-launched on device); the selected set of a head is
// { candidates c : c >= meta_kth }, materialised by run_emit
int run_kth_part(const tkv_problem* p, ScanParams cp, SelectParams sl, int64_t s0, int64_t s1, int part,
                 cudaStream_t st, bool pdl) {
  const int G = p->n_q_heads / p->n_kv_heads;
  cp.seg_begin = s0;
  cp.seg_count = s1 - s0;
  cp.fallback = 1;
  cp.pdl = 0;  // the device-launched fallback scan
  sl.pdl = pdl ? 1 : 0;
  sl.bh_begin = static_cast<int>(s0 * G);
  sl.bh_count = static_cast<int>((s1 - s0) * G);
  sl.hs.fb_launched += part;
  sl.fb_scan = cp;
  scan_launch_shape(cp, &sl.fb_scan_grid, &sl.fb_scan_smem);
  TKV_LAUNCH(launch_kth(sl, st));
  return TKV_OK;
}

// Parts of the overlapped pipeline: the scan of part i+1 runs on the caller's stream while
// the k-th selection and the V gather of part i run on a side stream beside it (both fit on
// an SM next to the tcgen05 scan CTA). One part when the scan is too short to hide them.
int pipeline_parts(const tkv_problem* p, bool tc) {
  const int env = diag_env("TKV_PARTS", 0);
  const int64_t nseg = static_cast<int64_t>(p->batch) * p->n_kv_heads;
  int P;
  const int forced = static_cast<int>((p->flags & TKV_F_PARTS_MASK) >> 8);
  if (forced > 0) {
    P = forced;
  } else if (env > 0) {
    P = env;
  } else {
    // measured on cfg3 (2.1 GB of keys): each extra scan launch costs ~12 us of fill/drain, more
    // than the overlap hides, so one part; four parts only for very long scans (cfg5: 8.6 GB)
    const double kbytes = static_cast<double>(nseg) * static_cast<double>(p->max_ctx) * kD * 2;
    P = tc && kbytes >= 4e9 ? 4 : 1;
  }
  if (P > nseg) P = static_cast<int>(nseg);
  if (P > kMaxParts) P = kMaxParts;
  return P < 1 ? 1 : P;
}

// per-thread, per-device side stream and fork/join events of the overlapped pipeline
struct PipeRes {
  cudaStream_t side = nullptr;   // k-th of each part
  cudaStream_t side2 = nullptr;  // gather of each part (after its k-th; beside the next k-th)
  cudaEvent_t ev[kMaxParts + 1] = {};
  cudaEvent_t evk[kMaxParts] = {};
};
thread_local PipeRes g_pipe[16];

int pipe_res(PipeRes** out) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 16) return fail(TKV_ECUDA, "device ordinal %d unsupported", dev);
  PipeRes& r = g_pipe[dev];
  if (!r.side) {
    cudaError_t e = cudaStreamCreateWithFlags(&r.side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&r.side2, cudaStreamNonBlocking);
    for (int i = 0; e == cudaSuccess && i <= kMaxParts; ++i) e = cudaEventCreateWithFlags(&r.ev[i], cudaEventDisableTiming);
    for (int i = 0; e == cudaSuccess && i < kMaxParts; ++i) e = cudaEventCreateWithFlags(&r.evk[i], cudaEventDisableTiming);
    if (e != cudaSuccess) return fail(TKV_ECUDA, "side stream / events: %s", cudaGetErrorString(e));
  }
  *out = &r;
  return TKV_OK;
}

// tkv_shard_candidates2's narrow-list append, carried into the emit pass's AttendParams
struct NarrowEmit {
  uint64_t* out = nullptr;
  int len = 0;
  uint32_t* cnt = nullptr;
  const uint64_t* t2 = nullptr;
};
thread_local NarrowEmit g_narrow;

AttendParams make_attend(const tkv_problem* p, const void* q, const void* k_cache, const void* v_cache,
                         const int32_t* n_ctx, const int32_t* n_win, const int32_t* idx,
                         const float* scores, void* ws, const Layout& L) {
  AttendParams a{};
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.kc = static_cast<const __nv_bfloat16*>(k_cache);
  a.vc = static_cast<const __nv_bfloat16*>(v_cache);
  a.cache_rows = p->cache_rows;
  a.B = p->batch;
  a.Hq = p->n_q_heads;
  a.Hkv = p->n_kv_heads;
  a.G = p->n_q_heads / p->n_kv_heads;
  a.k = p->k;
  a.n_ctx = n_ctx;
  a.n_win = n_win;
  a.row_offset = p->row_offset;
  a.pinned = p->pinned_prefix;
  a.scale = p->scale;
  a.combine = p->combine;
  a.idx = idx;
  a.scores = scores;
  a.meta_max = at<float>(ws, L.mmax);
  a.meta_kth = at<uint64_t>(ws, L.mkth);
  a.meta_kb = at<int32_t>(ws, L.mkb);
  a.part_l = at<float>(ws, L.pl);
  a.part_o = at<float>(ws, L.po);
  a.ticket = at<uint32_t>(ws, L.ticket_g);
  a.nchunks = L.nchunks;
  a.items_mult = diag_env("TKV_ATT_MULT", 1);  // experiments (TKV_DIAG builds): items per gather CTA
  a.cand = at<uint64_t>(ws, L.cand);
  a.cap = L.cap;
  a.cand_cnt = at<uint32_t>(ws, L.cnt);
  a.out_cnt = at<uint32_t>(ws, L.outc);
  a.tl = g_tl;
  a.pin_words = L.pin_words;
  a.pin_mask = L.pin_words ? at<uint32_t>(ws, L.pinm) : nullptr;
  a.narrow_out = g_narrow.out;
  a.narrow_len = g_narrow.len;
  a.narrow_cnt = g_narrow.cnt;
  a.meta_t2 = g_narrow.t2;
  return a;
}

// Gather structure: one fused filter + gather pass over the candidates, or (many selected
// rows) a filter pass writing idx/scores followed by a streaming gather over those lists —
// measured faster from ~1M selected rows per step (cfg5 family), slower below (cfg1-3).
// TKV_LIST_GATHER=0/1 forces either.
bool list_gather_used(const tkv_problem* p, int bh_count, int gather) {
  const int list_env = diag_env("TKV_LIST_GATHER", -1);
  const double sel_rows = static_cast<double>(bh_count) * p->k;
  return gather && ((p->flags & TKV_F_GATHER_LIST) ? true : (list_env >= 0 ? list_env != 0 : sel_rows >= 1.0e6));
}

// Materialise the selected rows (idx/scores[/packed]) from the candidates, with the V
// gather + softmax fused when gather != 0; then the optional TopKResult-order sort.
int run_emit(const tkv_problem* p, const void* q, const void* k_cache, const void* v_cache,
             const int32_t* n_ctx, const int32_t* n_win, int32_t* idx, float* scores,
             uint64_t* packed, float* out, int gather, void* ws, const Layout& L, cudaStream_t st,
             int bh_begin, int bh_count) {
  AttendParams a = make_attend(p, q, k_cache, v_cache, n_ctx, n_win, idx, scores, ws, L);
  a.bh_begin = bh_begin;
  a.bh_count = bh_count;
  a.idx_out = idx;
  a.scores_out = scores;
  a.packed_out = packed;
  a.out = out;
  a.gather = gather;
  a.partial_only = 0;
  const bool list_gather = list_gather_used(p, bh_count, gather);
  if (gather && list_gather) {
    a.gather = 0;  // filter only: idx / scores
    TKV_LAUNCH(launch_attend_cand(a, st));
    a.gather = 1;
    TKV_LAUNCH(launch_attend_list(a, st));
  } else {
    TKV_LAUNCH(launch_attend_cand(a, st));
  }
  if (p->flags & TKV_F_SORTED) {
    SortParams so{idx, scores, at<int32_t>(ws, L.mkb), p->k, bh_begin, at<uint64_t>(ws, L.sortb)};
    TKV_SORT(so, bh_count, st);
  }
  return TKV_OK;
}

// Small k: C CTAs per head do the k-th selection, the V gather and the finish
// (head_topk_kernel) instead of kth_kernel + attend_cand_kernel. Measured (tools/scan_ab.py):
// cfg1 (k = 256) 41.9 -> 37.4 us per step; cfg2 (k = 2048) 90.2 vs 91.5; cfg3 (k = 16384)
// 373 vs 390 — with one 512-thread CTA per SM the head kernel keeps ~64 KB of V rows in flight
// per SM (~25 GB/s), half of what attend_cand's four CTAs per SM sustain. TKV_HEAD_TOPK=0/1
// forces either (any k: the selected rows stream through a kHeadCap-row buffer); the
// TKV_F_HEAD / TKV_F_NO_HEAD flags force it per call.
// Moderate k: one 4-CTA cluster per head does the k-th selection, the V gather and the finish
// (clus_topk_kernel) — no k-th → gather launch gap, no global tickets. TKV_CLUS=0/1 (TKV_DIAG
// builds) forces either; TKV_F_CLUSTER / TKV_F_NO_CLUSTER per call.
// Automatic: few heads (one wave of 4-CTA clusters over the SMs) and moderate k (a CTA gathers
// <= k/4 rows: at cfg3's k = 16384 the candidate gather's four CTAs per SM keep more rows in
// flight — 361 vs 391 us). Measured: cfg1 (32 heads, k = 256) 38.3 -> 34.1 us, cfg2 (k = 2048)
// 76.1 -> 74.1 us.
bool use_clus_topk(const tkv_problem* p) {
  const int env = diag_env("TKV_CLUS", -1);
  if (p->flags & TKV_F_CLUSTER) return true;
  if ((p->flags & (TKV_F_GATHER_LIST | TKV_F_NO_CLUSTER | TKV_F_HEAD)) || env == 0) return false;
  if (env > 0) return true;
  const int nbh = p->batch * p->n_q_heads;
  return p->k <= 4096 && nbh * 4 <= device_sm_count();
}

bool use_head_topk(const tkv_problem* p, int gather) {
  const int env = diag_env("TKV_HEAD_TOPK", -1);
  if (p->flags & TKV_F_HEAD) return true;
  if ((p->flags & (TKV_F_GATHER_LIST | TKV_F_NO_HEAD)) || env == 0) return false;
  if (env > 0) return true;
  (void)gather;
  return p->k <= 1024;
}

int run_head(const tkv_problem* p, const void* q, const void* k_cache, const void* v_cache, const int32_t* n_ctx,
             const int32_t* n_win, int32_t* idx, float* scores, uint64_t* packed, float* out, int gather, void* ws,
             const Layout& L, cudaStream_t st, ScanParams cp, SelectParams sl, int nbh, bool pdl, bool clus = false) {
  HeadParams hp{};
  cp.seg_begin = 0;
  cp.seg_count = static_cast<int64_t>(p->batch) * p->n_kv_heads;
  cp.fallback = 1;
  cp.pdl = 0;
  sl.pdl = pdl ? 1 : 0;
  sl.bh_begin = 0;
  sl.bh_count = nbh;
  sl.fb_scan = cp;
  scan_launch_shape(cp, &sl.fb_scan_grid, &sl.fb_scan_smem);
  hp.s = sl;
  AttendParams& a = hp.a;
  a = make_attend(p, q, k_cache, v_cache, n_ctx, n_win, idx, scores, ws, L);
  a.bh_begin = 0;
  a.bh_count = nbh;
  a.idx_out = idx;
  a.scores_out = scores;
  a.packed_out = packed;
  a.out = out;
  a.gather = gather;
  a.partial_only = 0;
  // CTAs per head: enough heads x CTAs to cover the SMs in one wave (the gather is per-SM
  // bound), at least ~128 selected rows per CTA, at most one partial slot each
  const int sms = device_sm_count();
  const int env_c = diag_env("TKV_HEAD_CTAS", 0);
  int C = env_c > 0 ? env_c : sms / nbh;  // one wave: the kernel holds one CTA per SM
  const int c_rows = (p->k + 127) / 128 > 2 ? (p->k + 127) / 128 : 2;  // >= 128 rows per CTA, >= 2 CTAs
  if (env_c <= 0 && C > c_rows) C = c_rows;  // cfg1 (k = 256): C = 2 37.0 us, C = 1 40.6-43.3 us
  if (C > 8) C = 8;
  if (C > L.nchunks) C = L.nchunks;
  hp.ctas_per_head = C < 1 ? 1 : C;
  if (clus)
    TKV_LAUNCH(launch_clus_topk(hp, st));
  else
    TKV_LAUNCH(launch_head_topk(hp, st));
  if (p->flags & TKV_F_SORTED) {
    SortParams so{idx, scores, at<int32_t>(ws, L.mkb), p->k, 0, at<uint64_t>(ws, L.sortb)};
    TKV_SORT(so, nbh, st);
  }
  return TKV_OK;
}

// The whole layer step (multi-kernel pipeline).
int run_layer_dev(const tkv_problem* p, const void* q, const void* k_cache, const void* v_cache,
                  const int32_t* n_ctx, const int32_t* n_win, int32_t* idx, float* scores,
                  uint64_t* packed, float* out, int gather, void* ws, const Layout& L, cudaStream_t st);

// TKV_F_HOST_Q: stage q from pinned host memory into the workspace (one small kernel; the
// sample kernel is PDL-launched behind it), then run the layer on the device copy
int run_layer(const tkv_problem* p, const void* q, const void* k_cache, const void* v_cache,
              const int32_t* n_ctx, const int32_t* n_win, int32_t* idx, float* scores,
              uint64_t* packed, float* out, int gather, void* ws, const Layout& L, cudaStream_t st) {
  if (!(p->flags & TKV_F_HOST_Q))
    return run_layer_dev(p, q, k_cache, v_cache, n_ctx, n_win, idx, scores, packed, out, gather, ws, L, st);
  const int64_t nq = static_cast<int64_t>(p->batch) * p->n_q_heads * kD * 2 / 16;
  const int64_t nkv = static_cast<int64_t>(p->batch) * p->n_kv_heads * kD * 2 / 16;
  uint4* qs = at<uint4>(ws, L.qs);
  StageParams sp{};
  sp.src[0] = static_cast<const uint4*>(q);
  sp.dst[0] = qs;
  sp.n16[0] = nq;
  if (g_fold.k_new) {  // decode step: the window append reads the staged rows
    sp.src[1] = static_cast<const uint4*>(g_fold.k_new);
    sp.dst[1] = qs + nq;
    sp.n16[1] = nkv;
    sp.src[2] = static_cast<const uint4*>(g_fold.v_new);
    sp.dst[2] = qs + nq + nkv;
    sp.n16[2] = nkv;
    g_fold.k_new = qs + nq;
    g_fold.v_new = qs + nq + nkv;
  }
  TKV_LAUNCH(launch_stage(sp, st));
  g_staged = true;
  const int rc = run_layer_dev(p, at<uint4>(ws, L.qs), k_cache, v_cache, n_ctx, n_win, idx, scores, packed, out,
                               gather, ws, L, st);
  g_staged = false;
  return rc;
}

int run_layer_dev(const tkv_problem* p, const void* q, const void* k_cache, const void* v_cache,
                  const int32_t* n_ctx, const int32_t* n_win, int32_t* idx, float* scores,
                  uint64_t* packed, float* out, int gather, void* ws, const Layout& L, cudaStream_t st) {
  {
    ScanParams cp;
    SelectParams sl;
    TRY(run_prefix(p, q, k_cache, n_ctx, ws, L, st, &cp, &sl));
    const int G = p->n_q_heads / p->n_kv_heads;
    const int64_t nseg = static_cast<int64_t>(p->batch) * p->n_kv_heads;
    const int P = pipeline_parts(p, use_tc_scan(p, cp));
    const bool prof = g_scan_start && g_scan_stop;
    if (P == 1) {
      if (prof) cudaEventRecord(g_scan_start, st);
      // with the profiling events in the stream the launches stay ordinary (an event record
      // between two kernels would hide the overlap anyway)
      TRY(run_scan_part(p, cp, 0, nseg, st, pdl_enabled() && !prof));
      if (prof) cudaEventRecord(g_scan_stop, st);
      if (use_clus_topk(p))
        return run_head(p, q, k_cache, v_cache, n_ctx, n_win, idx, scores, packed, out, gather, ws, L, st, cp, sl,
                        static_cast<int>(nseg * G), pdl_enabled() && !prof, true);
      if (use_head_topk(p, gather))
        return run_head(p, q, k_cache, v_cache, n_ctx, n_win, idx, scores, packed, out, gather, ws, L, st, cp, sl,
                        static_cast<int>(nseg * G), pdl_enabled() && !prof);
      TRY(run_kth_part(p, cp, sl, 0, nseg, 0, st, pdl_enabled() && !prof));
      return run_emit(p, q, k_cache, v_cache, n_ctx, n_win, idx, scores, packed, out, gather, ws, L, st, 0,
                      static_cast<int>(nseg * G));
    }
    PipeRes* r = nullptr;
    TRY(pipe_res(&r));
    const bool serial = diag_env("TKV_PIPE_SERIAL", 0) != 0;  // diagnostics: split scans, no overlap
    if (serial) {
      if (prof) cudaEventRecord(g_scan_start, st);
      for (int part = 0; part < P; ++part)
        TRY(run_scan_part(p, cp, nseg * part / P, nseg * (part + 1) / P, st, false, part));
      if (prof) cudaEventRecord(g_scan_stop, st);
      for (int part = 0; part < P; ++part) {
        const int64_t s0 = nseg * part / P, s1 = nseg * (part + 1) / P;
        TRY(run_kth_part(p, cp, sl, s0, s1, part, st, false));
        TRY(run_emit(p, q, k_cache, v_cache, n_ctx, n_win, idx, scores, packed, out, gather, ws, L, st,
                     static_cast<int>(s0 * G), static_cast<int>((s1 - s0) * G)));
      }
      return TKV_OK;
    }
    // part boundaries: even, or (TKV_PARTS_TAIL=1) a last part of one eighth of the groups so
    // less k-th + gather work remains after the final scan
    const bool tail_split = diag_env("TKV_PARTS_TAIL", 0) != 0;
    auto bound = [&](int part) -> int64_t {
      if (!tail_split || P < 2) return nseg * part / P;
      int64_t last = nseg / 8;
      if (last < 1) last = 1;
      if (part >= P) return nseg;
      return (nseg - last) * part / (P - 1);
    };
    if (prof) cudaEventRecord(g_scan_start, st);
    const bool chain = diag_env("TKV_PARTS_CHAIN", 1) != 0;  // experiments: PDL-chained part scans
    for (int part = 0; part < P; ++part) {
      const int64_t s0 = bound(part), s1 = bound(part + 1);
      // the first part's scan overlaps sample / threshold (PDL); later parts' CTAs take over SMs
      // as the previous part's retire (its epilogue waits for that grid; TMEM buffers the gap)
      TRY(run_scan_part(p, cp, s0, s1, st, pdl_enabled() && !prof && (part == 0 || chain), part, false));
      if (cudaEventRecord(r->ev[part], st) != cudaSuccess || cudaStreamWaitEvent(r->side, r->ev[part], 0) != cudaSuccess)
        return fail(TKV_ECUDA, "pipeline fork failed");
      TRY(run_kth_part(p, cp, sl, s0, s1, part, r->side, false));
      // the gather of this part on its own stream, so the next part's k-th need not wait for it
      if (cudaEventRecord(r->evk[part], r->side) != cudaSuccess ||
          cudaStreamWaitEvent(r->side2, r->evk[part], 0) != cudaSuccess)
        return fail(TKV_ECUDA, "pipeline fork failed");
      TRY(run_emit(p, q, k_cache, v_cache, n_ctx, n_win, idx, scores, packed, out, gather, ws, L, r->side2,
                   static_cast<int>(s0 * G), static_cast<int>((s1 - s0) * G)));
    }
    if (cudaEventRecord(r->evk[0], r->side2) != cudaSuccess || cudaStreamWaitEvent(r->side, r->evk[0], 0) != cudaSuccess)
      return fail(TKV_ECUDA, "pipeline join failed");
    if (prof) cudaEventRecord(g_scan_stop, st);
    if (cudaEventRecord(r->ev[P], r->side) != cudaSuccess || cudaStreamWaitEvent(st, r->ev[P], 0) != cudaSuccess)
      return fail(TKV_ECUDA, "pipeline join failed");
    return TKV_OK;
  }
}

}  // namespace

extern "C" {

int tkv_version(void) { return TKV_VERSION; }

const char* tkv_last_error(void) { return g_err.c_str(); }

int tkv_last_launch_count(void) { return g_launches; }

int tkv_debug_timeline(void* buf) {
  g_tl = static_cast<uint64_t*>(buf);
  return TKV_OK;
}

int tkv_profile_scan_events(void* start, void* stop) {
  g_scan_start = static_cast<cudaEvent_t>(start);
  g_scan_stop = static_cast<cudaEvent_t>(stop);
  return TKV_OK;
}

int tkv_device_check(void) {
  int dev = 0, n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(TKV_ECUDA, "no CUDA device: %s", e == cudaSuccess ? "count is 0" : cudaGetErrorString(e));
  cudaGetDevice(&dev);
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0)
    return fail(TKV_ECUDA, "device %d is sm_%d%d; libtkv is built for sm_100a only", dev, major, minor);
  return TKV_OK;
}

int tkv_workspace_bytes(const tkv_problem* p, size_t* bytes) {
  TRY(validate(p));
  if (!bytes) return fail(TKV_EBADSHAPE, "bytes is NULL");
  *bytes = make_layout(p).total;
  return TKV_OK;
}

int tkv_workspace_fallbacks(const tkv_problem* p, const void* ws, size_t bytes, uint32_t* heads) {
  TRY(validate(p));
  Layout L;
  TRY(check_ws(p, const_cast<void*>(ws), bytes, &L));
  if (!heads) return fail(TKV_EBADSHAPE, "heads is NULL");
  const cudaError_t e = cudaMemcpy(heads, static_cast<const char*>(ws) + L.fbh, 4, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return fail(TKV_ECUDA, "cudaMemcpy: %s", cudaGetErrorString(e));
  return TKV_OK;
}

int tkv_workspace_init(const tkv_problem* p, void* ws, size_t bytes, void* stream) {
  g_launches = 0;
  TRY(validate(p));
  Layout L;
  TRY(check_ws(p, ws, bytes, &L));
  cudaError_t e = cudaMemsetAsync(ws, 0, L.ctrl_end, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(TKV_ECUDA, "cudaMemsetAsync: %s", cudaGetErrorString(e));
  return TKV_OK;
}

int tkv_topk_decode_attention(const tkv_problem* p, const void* q, const void* k_cache,
                              const void* v_cache, const int32_t* n_ctx, const int32_t* n_win,
                              float* out, int32_t* idx, float* scores, void* ws, size_t ws_bytes,
                              void* stream) {
  g_launches = 0;
  TRY(validate(p));
  Layout L;
  TRY(check_ws(p, ws, ws_bytes, &L));
  TRY(check_ptr(q, "q", 16));
  TRY(check_ptr(k_cache, "k_cache", 16));
  TRY(check_ptr(v_cache, "v_cache", 16));
  TRY(check_ptr(n_ctx, "n_ctx", 4));
  TRY(check_ptr(out, "out", 4));
  TRY(check_ptr(idx, "idx", 4));
  if (n_win) TRY(check_ptr(n_win, "n_win", 4));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float* sc = scores ? scores : at<float>(ws, L.sscore);
  return run_layer(p, q, k_cache, v_cache, n_ctx, n_win, idx, sc, nullptr, out, 1, ws, L, st);
}

int tkv_topk_search(const tkv_problem* p, const void* q, const void* k_cache, const int32_t* n_ctx,
                    int32_t* idx, float* scores, void* ws, size_t ws_bytes, void* stream) {
  g_launches = 0;
  TRY(validate(p));
  Layout L;
  TRY(check_ws(p, ws, ws_bytes, &L));
  TRY(check_ptr(q, "q", 16));
  TRY(check_ptr(k_cache, "k_cache", 16));
  TRY(check_ptr(n_ctx, "n_ctx", 4));
  TRY(check_ptr(idx, "idx", 4));
  float* sc = scores ? scores : at<float>(ws, L.sscore);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return run_layer(p, q, k_cache, k_cache, n_ctx, nullptr, idx, sc, nullptr, nullptr, 0, ws, L, st);
}

int tkv_topk_decode_step(const tkv_problem* p, const void* q, const void* k_new, const void* v_new, void* k_cache,
                         void* v_cache, const int32_t* n_ctx, int32_t* n_win, float* out, int32_t* idx,
                         float* scores, void* ws, size_t ws_bytes, void* stream) {
  g_launches = 0;
  TRY(validate(p));
  Layout L;
  TRY(check_ws(p, ws, ws_bytes, &L));
  TRY(check_ptr(q, "q", 16));
  TRY(check_ptr(k_new, "k_new", 16));
  TRY(check_ptr(v_new, "v_new", 16));
  TRY(check_ptr(k_cache, "k_cache", 16));
  TRY(check_ptr(v_cache, "v_cache", 16));
  TRY(check_ptr(n_ctx, "n_ctx", 4));
  TRY(check_ptr(n_win, "n_win", 4));
  TRY(check_ptr(out, "out", 4));
  TRY(check_ptr(idx, "idx", 4));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float* sc = scores ? scores : at<float>(ws, L.sscore);
  g_fold = AppendFold{k_new, v_new, k_cache, v_cache, n_win};
  const int rc = run_layer(p, q, k_cache, v_cache, n_ctx, n_win, idx, sc, nullptr, out, 1, ws, L, st);
  g_fold = AppendFold{};
  return rc;
}

int tkv_kv_append(int32_t batch, int32_t n_kv_heads, int32_t head_dim, int64_t cache_rows,
                  void* k_cache, void* v_cache, const void* k_new, const void* v_new,
                  const int32_t* base, int32_t* count, int32_t advance, void* stream) {
  g_launches = 0;
  if (batch < 1 || n_kv_heads < 1) return fail(TKV_EBADSHAPE, "batch/heads must be >= 1");
  if (head_dim != kD) return fail(TKV_EBADSHAPE, "head_dim=%d unsupported (this build: %d)", head_dim, kD);
  if (cache_rows < 1) return fail(TKV_EBADSHAPE, "cache_rows must be >= 1");
  TRY(check_ptr(k_cache, "k_cache", 16));
  TRY(check_ptr(v_cache, "v_cache", 16));
  TRY(check_ptr(k_new, "k_new", 16));
  TRY(check_ptr(v_new, "v_new", 16));
  TRY(check_ptr(count, "count", 4));
  if (base) TRY(check_ptr(base, "base", 4));
  AppendParams a{};
  a.B = batch;
  a.Hkv = n_kv_heads;
  a.cache_rows = cache_rows;
  a.kc = static_cast<__nv_bfloat16*>(k_cache);
  a.vc = static_cast<__nv_bfloat16*>(v_cache);
  a.k_new = static_cast<const __nv_bfloat16*>(k_new);
  a.v_new = static_cast<const __nv_bfloat16*>(v_new);
  a.base = base;
  a.count = count;
  a.advance = advance;
  TKV_LAUNCH(launch_append(a, static_cast<cudaStream_t>(stream)));
  return TKV_OK;
}

int tkv_shard_candidates(const tkv_problem* p, const void* q, const void* k_cache, const int32_t* n_ctx,
                         uint64_t* cand, void* ws, size_t ws_bytes, void* stream) {
  g_launches = 0;
  TRY(validate(p));
  Layout L;
  TRY(check_ws(p, ws, ws_bytes, &L));
  TRY(check_ptr(q, "q", 16));
  TRY(check_ptr(k_cache, "k_cache", 16));
  TRY(check_ptr(n_ctx, "n_ctx", 4));
  TRY(check_ptr(cand, "cand", 8));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  tkv_problem pu = *p;
  pu.flags &= ~TKV_F_SORTED;
  return run_layer(&pu, q, k_cache, k_cache, n_ctx, nullptr, at<int32_t>(ws, L.sidx), at<float>(ws, L.sscore),
                  cand, nullptr, 0, ws, L, st);
}

int tkv_shard_candidates2(const tkv_problem* p, int32_t narrow_k, const void* q, const void* k_cache,
                          const int32_t* n_ctx, uint64_t* cand_narrow, uint64_t* cand_full, uint64_t* bounds,
                          void* ws, size_t ws_bytes, void* stream) {
  g_launches = 0;
  TRY(validate(p));
  Layout L;
  TRY(check_ws(p, ws, ws_bytes, &L));
  TRY(check_ptr(q, "q", 16));
  TRY(check_ptr(k_cache, "k_cache", 16));
  TRY(check_ptr(n_ctx, "n_ctx", 4));
  TRY(check_ptr(cand_narrow, "cand_narrow", 8));
  TRY(check_ptr(cand_full, "cand_full", 8));
  TRY(check_ptr(bounds, "bounds", 8));
  if (narrow_k < 1 || narrow_k > p->k) return fail(TKV_EBADK, "narrow_k must be in [1, k] (got %d)", narrow_k);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // one key scan and one exact k-th selection for k; the k-th kernel also marks the narrow
  // bound t2 (fewer than narrow_k candidates above it) from the same histogram; the emit pass
  // writes the full list, a small filter kernel the narrow list and the bounds
  tkv_problem pu = *p;
  pu.flags = (pu.flags & ~(TKV_F_SORTED | TKV_F_PARTS_MASK | TKV_F_HEAD | TKV_F_HOST_Q)) | TKV_F_NO_HEAD;
  ScanParams cp;
  SelectParams sl;
  TRY(run_prefix(&pu, q, k_cache, n_ctx, ws, L, st, &cp, &sl));
  const int64_t nseg = static_cast<int64_t>(p->batch) * p->n_kv_heads;
  const int nbh = p->batch * p->n_q_heads;
  sl.k2 = narrow_k;
  sl.meta_t2 = at<uint64_t>(ws, L.mt2);
  // the narrow list + bounds are produced by the k-th kernel (zeroed list, bounds) and the emit
  // pass (selected candidates >= t2 appended) — no separate filter kernel over the full list
  sl.narrow_out = cand_narrow;
  sl.narrow_len = narrow_k;
  sl.narrow_cnt = at<uint32_t>(ws, L.ncnt);
  sl.bound_out = bounds;
  TRY(run_scan_part(&pu, cp, 0, nseg, st, pdl_enabled()));
  TRY(run_kth_part(&pu, cp, sl, 0, nseg, 0, st, pdl_enabled()));
  g_narrow = NarrowEmit{cand_narrow, narrow_k, at<uint32_t>(ws, L.ncnt), at<uint64_t>(ws, L.mt2)};
  const int rc = run_emit(&pu, q, k_cache, k_cache, n_ctx, nullptr, at<int32_t>(ws, L.sidx), at<float>(ws, L.sscore),
                          cand_full, nullptr, 0, ws, L, st, 0, nbh);
  g_narrow = NarrowEmit{};
  (void)bounds;
  return rc;
}

int tkv_shard_exchange_merge(const tkv_problem* p, const uint64_t* const* narrow_lists,
                             const uint64_t* const* full_lists, const uint64_t* const* bounds, int32_t n_shards,
                             int32_t narrow_k, int32_t* idx, float* scores, int32_t* used_full, void* ws,
                             size_t ws_bytes, void* stream) {
  g_launches = 0;
  TRY(validate(p));
  Layout L;
  TRY(check_ws(p, ws, ws_bytes, &L));
  TRY(check_ptr(narrow_lists, "narrow_lists", 8));
  TRY(check_ptr(full_lists, "full_lists", 8));
  TRY(check_ptr(bounds, "bounds", 8));
  TRY(check_ptr(idx, "idx", 4));
  TRY(check_ptr(scores, "scores", 4));
  if (n_shards < 1 || n_shards > kMaxShards) return fail(TKV_EBADSHAPE, "n_shards must be in [1, %d]", kMaxShards);
  if (narrow_k < 1 || narrow_k > p->k) return fail(TKV_EBADK, "narrow_k must be in [1, k] (got %d)", narrow_k);
  ShardMergeParams mp{};
  mp.narrow = narrow_lists;
  mp.full = full_lists;
  mp.bound = bounds;
  mp.n_shards = n_shards;
  mp.narrow_len = narrow_k;
  mp.full_len = p->k;
  mp.k = p->k;
  mp.idx = idx;
  mp.scores = scores;
  mp.meta_max = at<float>(ws, L.mmax);
  mp.meta_kth = at<uint64_t>(ws, L.mkth);
  mp.meta_kb = at<int32_t>(ws, L.mkb);
  mp.out_cnt = at<uint32_t>(ws, L.mout);
  mp.used_full = used_full;
  mp.tl = g_tl;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nbh = p->batch * p->n_q_heads;
  TKV_LAUNCH(launch_shard_merge(mp, nbh, st));
  if (p->flags & TKV_F_SORTED) {
    SortParams so{idx, scores, mp.meta_kb, p->k, 0, at<uint64_t>(ws, L.sortb)};
    TKV_SORT(so, nbh, st);
  }
  return TKV_OK;
}

int tkv_shard_combine(const tkv_problem* p, const float* const* partials, int32_t n_shards, const void* q,
                      const void* k_cache, const void* v_cache, const int32_t* n_ctx, const int32_t* n_win,
                      float* out, void* ws, size_t ws_bytes, void* stream) {
  g_launches = 0;
  TRY(validate(p));
  Layout L;
  TRY(check_ws(p, ws, ws_bytes, &L));
  TRY(check_ptr(partials, "partials", 8));
  TRY(check_ptr(q, "q", 16));
  TRY(check_ptr(k_cache, "k_cache", 16));
  TRY(check_ptr(v_cache, "v_cache", 16));
  TRY(check_ptr(n_ctx, "n_ctx", 4));
  TRY(check_ptr(out, "out", 4));
  if (n_shards < 1 || n_shards > kMaxShards) return fail(TKV_EBADSHAPE, "n_shards must be in [1, %d]", kMaxShards);
  AttendParams a = make_attend(p, q, k_cache, v_cache, n_ctx, n_win, nullptr, nullptr, ws, L);
  a.partial_peers = partials;
  a.n_peers = n_shards;
  a.out = out;
  TKV_LAUNCH(launch_finalize(a, static_cast<cudaStream_t>(stream)));
  return TKV_OK;
}

int tkv_shard_merge(const tkv_problem* p, const uint64_t* gathered, int32_t n_shards, int32_t* idx,
                    float* scores, void* ws, size_t ws_bytes, void* stream) {
  TRY(validate(p));
  return tkv_shard_merge_lists(p, gathered, n_shards, p->k, idx, scores, ws, ws_bytes, stream);
}

int tkv_shard_narrow_check(const tkv_problem* p, const uint64_t* gathered, int32_t n_shards,
                           int32_t list_len, int32_t* ok, void* stream) {
  g_launches = 0;
  TRY(validate(p));
  TRY(check_ptr(gathered, "gathered", 8));
  TRY(check_ptr(ok, "ok", 4));
  if (n_shards < 1) return fail(TKV_EBADSHAPE, "n_shards must be >= 1");
  if (list_len < 1 || list_len > p->k) return fail(TKV_EBADK, "list_len must be in [1, k]");
  if (static_cast<int64_t>(n_shards) * list_len > (1ll << 30))
    return fail(TKV_EBADSHAPE, "n_shards * list_len too large");
  const int nbh = p->batch * p->n_q_heads;
  TKV_LAUNCH(launch_narrow_check(gathered, n_shards, list_len, nbh, p->k, ok,
                                 static_cast<cudaStream_t>(stream)));
  return TKV_OK;
}

int tkv_shard_merge_lists(const tkv_problem* p, const uint64_t* gathered, int32_t n_shards,
                          int32_t list_len, int32_t* idx, float* scores, void* ws, size_t ws_bytes,
                          void* stream) {
  g_launches = 0;
  TRY(validate(p));
  Layout L;
  TRY(check_ws(p, ws, ws_bytes, &L));
  TRY(check_ptr(gathered, "gathered", 8));
  TRY(check_ptr(idx, "idx", 4));
  TRY(check_ptr(scores, "scores", 4));
  if (n_shards < 1) return fail(TKV_EBADSHAPE, "n_shards must be >= 1");
  if (list_len < 1 || list_len > p->k) return fail(TKV_EBADK, "list_len must be in [1, k]");
  // gathered is [n_shards][B*Hq*list_len] (all_gather_into_tensor layout), read in place.
  const int G = p->n_q_heads / p->n_kv_heads;
  SelectParams sl{};
  sl.src = gathered;
  sl.merge_len = list_len;
  sl.src_stride = static_cast<int64_t>(n_shards) * list_len;
  sl.shard_stride = static_cast<int64_t>(p->batch) * p->n_q_heads * list_len;
  sl.src_fixed = static_cast<int64_t>(n_shards) * list_len;
  sl.B = p->batch;
  sl.Hq = p->n_q_heads;
  sl.Hkv = p->n_kv_heads;
  sl.G = G;
  sl.k = p->k;
  sl.n_ctx = nullptr;
  sl.idx = idx;
  sl.scores = scores;
  sl.meta_max = at<float>(ws, L.mmax);
  sl.meta_kth = at<uint64_t>(ws, L.mkth);
  sl.meta_kb = at<int32_t>(ws, L.mkb);
  sl.hs = head_state(ws, L);
  sl.packed_out = nullptr;
  sl.pass = kPassMerge;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  TKV_LAUNCH(launch_select(sl, st));
  if (p->flags & TKV_F_SORTED) {
    SortParams so{idx, scores, sl.meta_kb, p->k, 0, at<uint64_t>(ws, L.sortb)};
    TKV_SORT(so, p->batch * p->n_q_heads, st);
  }
  return TKV_OK;
}

int tkv_shard_partial(const tkv_problem* p, const void* q, const void* k_cache, const void* v_cache,
                      const int32_t* n_ctx, const int32_t* idx, const float* scores, float* partial,
                      void* ws, size_t ws_bytes, void* stream) {
  g_launches = 0;
  TRY(validate(p));
  Layout L;
  TRY(check_ws(p, ws, ws_bytes, &L));
  TRY(check_ptr(q, "q", 16));
  TRY(check_ptr(k_cache, "k_cache", 16));
  TRY(check_ptr(v_cache, "v_cache", 16));
  TRY(check_ptr(n_ctx, "n_ctx", 4));
  TRY(check_ptr(idx, "idx", 4));
  TRY(check_ptr(scores, "scores", 4));
  TRY(check_ptr(partial, "partial", 4));
  AttendParams a = make_attend(p, q, k_cache, v_cache, n_ctx, nullptr, idx, scores, ws, L);
  a.partial_only = 1;
  a.partial_out = partial;
  if (a.pin_mask) {  // the list pass marks the selected pinned rows; start from none
    const cudaError_t e = cudaMemsetAsync(a.pin_mask, 0, static_cast<size_t>(p->batch) * p->n_q_heads * L.pin_words * 4,
                                          static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return fail(TKV_ECUDA, "cudaMemsetAsync: %s", cudaGetErrorString(e));
  }
  TKV_LAUNCH(launch_attend(a, static_cast<cudaStream_t>(stream)));
  return TKV_OK;
}

int tkv_shard_finalize(const tkv_problem* p, const void* q, const void* k_cache, const void* v_cache,
                       const int32_t* n_ctx, const int32_t* n_win, const float* partial, float* out,
                       void* ws, size_t ws_bytes, void* stream) {
  g_launches = 0;
  TRY(validate(p));
  Layout L;
  TRY(check_ws(p, ws, ws_bytes, &L));
  TRY(check_ptr(q, "q", 16));
  TRY(check_ptr(k_cache, "k_cache", 16));
  TRY(check_ptr(v_cache, "v_cache", 16));
  TRY(check_ptr(n_ctx, "n_ctx", 4));
  TRY(check_ptr(partial, "partial", 4));
  TRY(check_ptr(out, "out", 4));
  AttendParams a = make_attend(p, q, k_cache, v_cache, n_ctx, n_win, nullptr, nullptr, ws, L);
  a.partial_in = partial;
  a.out = out;
  TKV_LAUNCH(launch_finalize(a, static_cast<cudaStream_t>(stream)));
  return TKV_OK;
}

}  // extern "C"

// error reporting for the other translation units' C entry points (model_glue.cu)
int tkv::api_fail(int code, const char* msg) { return fail(code, "%s", msg); }
