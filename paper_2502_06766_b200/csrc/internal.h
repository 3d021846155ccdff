// internal.h — kernel parameter blocks and launchers shared by the .cu translation units.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>
#include <utility>

namespace tkv {

#ifndef TKV_SAMPLES
#define TKV_SAMPLES 4096
#endif
constexpr int kSamples = TKV_SAMPLES;  // sampled rows per (b, kv head) for the threshold estimate
constexpr int kSampleThreads = 256;  // sample-scoring CTA
#ifndef TKV_THR_THREADS
#define TKV_THR_THREADS 512
#endif
constexpr int kThrThreads = TKV_THR_THREADS;  // threshold CTA (one per (b, q head))
constexpr int kScanWarps = 8;        // scan kernel CTA = 8 warps
constexpr int kScanU = 2;            // 16-row tiles per warp per iteration
constexpr int kScanRows = kScanWarps * 16 * kScanU;  // rows per CTA iteration
constexpr int kScanFlushEvery = 4;                   // iterations between staging flushes
constexpr int kScanStage = kScanRows * kScanFlushEvery;  // staged candidates per head
constexpr int kSelectThreads = 1024;
constexpr int kSelectBucketCap = 8192;  // threshold-bucket candidates refined in shared memory
constexpr int kKthThreads = 512;        // kth_kernel CTA
#ifndef TKV_KTH_CTAS
#define TKV_KTH_CTAS 4
#endif
constexpr int kKthCtas = TKV_KTH_CTAS;  // kth_kernel CTAs per (b, q head) (one cluster)
constexpr int kKthManyHeads = 128;      // from this many heads per call: 2-CTA clusters
constexpr int kKthSmemBucket = 2048;    // threshold-bucket members rank-selected in shared memory
constexpr int kKthSmem = kKthSmemBucket * 8;  // kth_kernel dynamic shared memory (fits beside the scan)
constexpr int kAttendThreads = 256;
#ifndef TKV_ATTEND_CHUNK
#define TKV_ATTEND_CHUNK 1024
#endif
constexpr int kAttendChunk = TKV_ATTEND_CHUNK;  // selected rows per gather CTA (list mode)
#ifndef TKV_CAND_CHUNK
#define TKV_CAND_CHUNK 2048
#endif
constexpr int kCandChunk = TKV_CAND_CHUNK;  // candidates per compaction + gather batch (candidate mode)
static_assert(kAttendChunk <= kCandChunk, "a list chunk fits the gather's row buffer");
constexpr int kCandQuant = 256;             // candidate-mode work items are multiples of this
constexpr int kMaxGatherGrid = 1023;        // candidate-mode gather CTAs (bounds the partial slots)
constexpr int kFlatMinRows = 256;           // flat list gather: rows per CTA range, at least
constexpr int kSortMax = 16384;      // one-CTA shared-memory sort up to this k; chunk sort + merge passes above
constexpr uint32_t kNoFilterShift = 20;  // histogram shift when every score is a candidate
constexpr int kMinSampleStride = 8;      // small contexts sample at most every 8th row
constexpr int kMaxParts = 16;            // KV-group parts of the overlapped layer pipeline

// Half the sample (kSamples / 2) for contexts of at most kSmallCtxRows rows whose k is at most
// 1/32 of them: there the threshold kernel ends while the key scan waits for it (its epilogue
// cannot emit before), so the shorter radix select and the smaller sample grid shorten the step
// (cfg2 70.0 -> 68.1 us). Beyond it the threshold is off the critical path and the tighter full
// sample (fewer candidates) wins (cfg3 with 2048: 357.9 -> 361.5 us), and so it does at a large
// k / N (a G = 8 shard of cfg3, 131K rows with k = 16384: candidates stage 92.4 -> 95.4 us).
#ifndef TKV_SMALL_CTX_LOG2
#define TKV_SMALL_CTX_LOG2 17
#endif
constexpr int64_t kSmallCtxRows = int64_t(1) << TKV_SMALL_CTX_LOG2;

// samples of a context of n rows with top-k size k (at most; also sizes the sample grid)
__host__ __device__ inline int sample_max(int64_t n, int64_t k) {
  return (n <= kSmallCtxRows && k * 32 <= n) ? kSamples / 2 : kSamples;
}

// rows between two sampled rows: up to sample_max(n, k) samples, never denser than 1 in 8
__host__ __device__ inline int64_t sample_stride(int64_t n, int64_t k) {
  const int64_t target = sample_max(n, k);
  const int64_t s = (n + target - 1) / target;
  return s > kMinSampleStride ? s : kMinSampleStride;
}

// Sampled row s of segment seg (= b * Hkv + kv head): one row per stride-wide window, at an
// offset hashed from the segment, so a cache with period `stride` cannot line up with the
// sample the same way in every segment (a per-sample offset measured 8 us slower at cfg3: the
// faster sample kernel let threshold CTAs land where they hold scan CTAs off their SM).
// tests/conftest.py sample_rows() restates it for adversarial caches.
__host__ __device__ inline int64_t sample_row(int64_t s, int64_t stride, int seg, int64_t n) {
  const uint32_t h = static_cast<uint32_t>(seg) * 0x9E3779B9u + 0x7F4A7C15u;
  const int64_t r = s * stride + static_cast<int64_t>((h >> 8) % static_cast<uint32_t>(stride));
  return r < n ? r : n - 1;
}

// per-(b, q head) state shared by the kernels of one call, in the workspace
struct HeadState {
  uint32_t* thr;         // [B*Hq] candidate threshold key (0 = emit all)
  uint32_t* hshift;      // [B*Hq] histogram granularity
  uint32_t* cand_cnt;    // [B*Hq]
  uint32_t* hist;        // [B*Hq][kHistBins] histogram of the emitted candidates
  uint32_t* flag_fail;   // [B*Hq] sampled threshold too high → re-scan with thr = 0
  uint32_t* group_fail;  // [B*Hkv]
  uint64_t* max_comp;    // [B*Hq] largest candidate composite (reset by threshold_kernel)
  uint32_t* bkt_cnt;     // [B*Hq] candidates of the threshold bucket gathered so far
  uint64_t* bkt;         // [B*Hq][kSelectBucketCap] threshold-bucket candidates
  uint32_t* kth_ticket;  // [B*Hq] kth_kernel CTAs done (self-resetting)
  uint32_t* out_cnt;     // [B*Hq] selected rows written so far (reset by threshold_kernel)
  uint32_t* fb_launched; // the exactness fallback has been tail-launched for this call (one flag
                         // per pipeline part; the part's SelectParams points at its own)
  uint32_t* fb_heads;    // heads that needed the exactness fallback since tkv_workspace_init
};

struct SampleParams {
  uint64_t* tl;  // diagnostics timeline (tkv_debug_timeline), nullptr normally
  const __nv_bfloat16* q;
  const __nv_bfloat16* kc;
  int64_t cache_rows;
  int B, Hq, Hkv, G, k;
  const int32_t* n_ctx;
  int no_filter;
  uint32_t* samp;  // [B*Hq*kSamples]
  HeadState hs;
  uint32_t* pin_mask;  // [B*Hq][pin_words] selected pinned-prefix rows (zeroed by threshold_kernel)
  int pin_words;
  // optional window append folded into threshold_kernel (tkv_topk_decode_step): rows
  // n_ctx[b] + win_count[b] of K/V <- k_new/v_new[b], then win_count[b] += 1
  const __nv_bfloat16* k_new;  // [B, Hkv, 128] or nullptr
  const __nv_bfloat16* v_new;
  __nv_bfloat16* k_dst;
  __nv_bfloat16* v_dst;
  int32_t* win_count;
  int pdl;  // sample_kernel launched behind the q staging kernel (TKV_F_HOST_Q)
  int max_samples;  // largest sample of any batch entry (sample_max(max_ctx)): sizes the grid
};

// TKV_F_HOST_Q: q copied from pinned host memory into the workspace by one small kernel
struct StageParams {
  const uint4* src[3];  // q, and for tkv_topk_decode_step k_new / v_new
  uint4* dst[3];
  int64_t n16[3];  // 16-byte words per segment (0 = unused)
};
cudaError_t launch_stage(const StageParams& p, cudaStream_t s);

struct ScanParams {
  uint64_t* tl;  // diagnostics timeline (tkv_debug_timeline), nullptr normally
  const __nv_bfloat16* q;
  const __nv_bfloat16* kc;
  int64_t cache_rows;
  int B, Hq, Hkv, G;
  int64_t max_ctx;
  const int32_t* n_ctx;
  uint32_t row_offset;
  uint64_t* cand;  // [B*Hq][cap]
  int64_t cap;
  HeadState hs;
  int fallback;
  int64_t seg_begin, seg_count;  // (b, kv head) segments to scan; seg_count 0 = all B*Hkv
  int pdl;                       // launch with programmatic dependent launch (see launch_pdl)
  uint32_t* steal;  // tcgen05 scan: [2] pool claim counter + CTAs done (self-resetting); nullptr = static split
};

enum SelectPass { kPassMain = 0, kPassFallback = 1, kPassMerge = 2 };

struct SelectParams {
  uint64_t* tl;  // diagnostics timeline (tkv_debug_timeline), nullptr normally
  const uint64_t* src;   // candidates: src + bh*src_stride (main/fallback)
  int64_t src_stride;    // merge: element i of head bh is
  int64_t shard_stride;  //   src[(i / L) * shard_stride + bh * L + i % L], L = merge_len
  int64_t src_fixed;     // merge: candidates per head (n_shards * merge_len)
  int64_t merge_len;     // merge: list length per shard and head (k, or k' < k: narrow exchange)
  int B, Hq, Hkv, G, k;
  const int32_t* n_ctx;  // kb = min(k, n_ctx[b]) (main/fallback); merge: min(k, #valid)
  int32_t* idx;          // [B*Hq*k]
  float* scores;         // [B*Hq*k]
  float* meta_max;       // [B*Hq]
  uint64_t* meta_kth;    // [B*Hq]
  int32_t* meta_kb;      // [B*Hq]
  HeadState hs;
  uint64_t* packed_out;  // optional [B*Hq*k] composites (shard candidates)
  int pass;
  int bh_begin, bh_count;  // heads handled (kth_kernel); bh_count 0 = all B*Hq
  int pdl;                 // launch kth_kernel with programmatic dependent launch
  // sharded narrow list (tkv_shard_candidates2): k2 > 0 → kth_kernel also writes, per head, a
  // composite t2 with fewer than k2 candidates >= t2 (the lower bound of the histogram bucket
  // above the one holding the k2-th largest; T itself when every candidate is selected)
  int k2;
  uint64_t* meta_t2;
  // ... and (narrow_out != nullptr) zeroes this rank's narrow list [B*Hq][narrow_len] and its
  // append counters, and writes the bounds [B*Hq][3] = {t2, local k-th floor, max composite};
  // the emit pass then appends the selected candidates >= t2 (no separate filter kernel)
  uint64_t* narrow_out;
  int narrow_len;
  uint32_t* narrow_cnt;
  uint64_t* bound_out;
  // exactness fallback, tail-launched by kth_kernel (main pass) when a head failed
  ScanParams fb_scan;
  int fb_scan_grid;
  int fb_scan_smem;
};

// sets tkv_last_error's message and returns code (api.cu)
int api_fail(int code, const char* msg);

// host-side preparation of the device-tail-launched fallback kernels (select.cu)
void prepare_fallback_kernels();

struct SortParams {
  int32_t* idx;
  float* scores;
  const int32_t* meta_kb;
  int k;
  int bh_begin;
  uint64_t* buf;  // k > kSortMax: 2 x [heads][k] composites (merge ping-pong), workspace
};
constexpr int kSortChunk = 8192;  // k > kSortMax: runs sorted in shared memory, then merged

struct AttendParams {
  uint64_t* tl;  // diagnostics timeline (tkv_debug_timeline), nullptr normally
  const __nv_bfloat16* q;
  const __nv_bfloat16* kc;
  const __nv_bfloat16* vc;
  int64_t cache_rows;
  int B, Hq, Hkv, G, k;
  const int32_t* n_ctx;
  const int32_t* n_win;
  int64_t row_offset;
  int pinned;
  float scale;
  int combine;
  const int32_t* idx;
  const float* scores;
  const float* meta_max;
  const uint64_t* meta_kth;
  const int32_t* meta_kb;
  float* part_l;  // [B*Hq*nchunks]
  float* part_o;  // [B*Hq*nchunks*D]
  uint32_t* ticket;
  int nchunks;       // list mode: chunks per head; candidate mode: partial slots per head
  int partial_only;  // 1: write (l, o) to partial_out; 0: finalize into out
  float* partial_out;
  const float* partial_in;  // finalize kernel input
  float* out;
  // candidate mode (single GPU): read the scan's candidates, keep c >= meta_kth, write
  // idx/scores (and packed composites) as a side effect, gather V of the kept rows
  const uint64_t* cand;
  int64_t cap;
  const uint32_t* cand_cnt;
  uint32_t* out_cnt;
  int32_t* idx_out;
  float* scores_out;
  uint64_t* packed_out;
  int gather;  // 0: only write the selected rows (no attention)
  // selected rows inside the pinned prefix, one bit per local row, set by the gather / filter
  // pass; the pinned pass skips them (membership by id, not by a recomputed score)
  uint32_t* pin_mask;  // [B*Hq][pin_words] or nullptr
  int pin_words;
  int bh_begin, bh_count;  // heads handled by attend_cand_kernel; bh_count 0 = all B*Hq
  // sharded finalize (finalize_kernel): partial_in is replaced by the sum over n_peers ranks'
  // (l, o[128]) partials read through device pointers, when n_peers > 0
  const float* const* partial_peers;
  int n_peers;
  int items_mult;  // candidate mode: work items per CTA, about (0 = 1)
  // sharded candidates (tkv_shard_candidates2): selected candidates >= meta_t2[bh] are also
  // appended to narrow_out[bh][0, narrow_len) (order unspecified; kth_kernel zeroed the list)
  uint64_t* narrow_out;
  int narrow_len;
  uint32_t* narrow_cnt;
  const uint64_t* meta_t2;
};

// shard_merge_kernel (shard.cu): exact global top-k over every rank's published candidate lists
// (device pointers: peers' buffers over NVLink, or local buffers in the one-GPU emulation), the
// narrow-vs-full choice made per head on the device
constexpr int kMaxShards = 16;
struct ShardMergeParams {
  const uint64_t* const* narrow;  // [n_shards] → [B*Hq][narrow_len]
  const uint64_t* const* full;    // [n_shards] → [B*Hq][full_len]
  const uint64_t* const* bound;   // [n_shards] → [B*Hq][3]: narrow floor t2, full floor, max
  int n_shards, narrow_len, full_len, k;
  int32_t* idx;
  float* scores;
  float* meta_max;
  uint64_t* meta_kth;
  int32_t* meta_kb;
  uint32_t* out_cnt;
  int32_t* used_full;  // [B*Hq] or nullptr: 1 where the head was merged from the full lists
  uint64_t* tl;        // diagnostics timeline (TKV_DIAG builds: per-phase means)
};
cudaError_t launch_shard_merge(const ShardMergeParams& p, int nbh, cudaStream_t s);
// head_topk_kernel (select.cu): k-th selection + V gather + finish of a head by ctas_per_head
// CTAs (selected rows streamed through a kHeadCap-row shared buffer). att_grid: grid of the candidate-mode gather the exactness fallback
// tail-launches over all heads.
constexpr int kHeadThreads = 512;
constexpr int kHeadCap = 8192;
struct HeadParams {
  SelectParams s;
  AttendParams a;
  int ctas_per_head;  // <= nchunks (partial slots)
  int att_grid;
};

struct AppendParams {
  int B, Hkv;
  int64_t cache_rows;
  __nv_bfloat16* kc;
  __nv_bfloat16* vc;
  const __nv_bfloat16* k_new;
  const __nv_bfloat16* v_new;
  const int32_t* base;  // nullable
  int32_t* count;
  int advance;
};

// Launch with programmatic stream serialisation (the kernel calls pdl_wait() before touching
// its predecessor's outputs), or an ordinary launch when pdl is false.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
bool pdl_enabled();

// host_state.cu: per-device memoisation (key, tag, current device) -> compute(), the current
// device's SM count, and the TKV_DIAG-only environment overrides (release: always dflt)
int current_device();
int per_device(const void* key, int tag, const std::function<int()>& compute);
int device_sm_count();
int diag_env(const char* name, int dflt);

cudaError_t launch_sample(const SampleParams& p, cudaStream_t s);
cudaError_t launch_scan(const ScanParams& p, cudaStream_t s);
cudaError_t launch_scan_tc(const ScanParams& p, cudaStream_t s);
cudaError_t launch_scan_fma(const ScanParams& p, cudaStream_t s);
bool scan_tc_supported(const ScanParams& p);
void scan_launch_shape(const ScanParams& p, int* grid, int* smem_bytes);
cudaError_t launch_select(const SelectParams& p, cudaStream_t s);
cudaError_t launch_narrow_check(const uint64_t* gathered, int n_shards, int list_len, int nbh, int k,
                                int32_t* ok, cudaStream_t s);
cudaError_t launch_kth(const SelectParams& p, cudaStream_t s);
cudaError_t launch_head_topk(const HeadParams& p, cudaStream_t s);
cudaError_t launch_clus_topk(const HeadParams& p, cudaStream_t s);
cudaError_t launch_attend_cand(const AttendParams& p, cudaStream_t s);
cudaError_t launch_attend_list(const AttendParams& p, cudaStream_t s);
cudaError_t launch_sort(const SortParams& p, int nbh, cudaStream_t s, int* launches);
cudaError_t launch_attend(const AttendParams& p, cudaStream_t s);
cudaError_t launch_finalize(const AttendParams& p, cudaStream_t s);
cudaError_t launch_append(const AppendParams& p, cudaStream_t s);

}  // namespace tkv
