/*
 * tkv.h — C ABI of the B200-native exact top-k decode-attention library (libtkv.so).
 *
 * This is the drop-in boundary for the hot path of the reference package `topk_kv`
 * (arXiv 2502.06766 desk realisation, /root/reference/pkg/src/topk_kv). Every entry point
 * below replaces one reference interface; the citation is given per function.
 *
 * Conventions
 *   - Plain C types only: device pointers, sizes, an opaque CUDA stream (cudaStream_t passed
 *     as void*). No torch / C++ types cross this boundary.
 *   - All compute entry points are stream-ordered and asynchronous: they enqueue kernels on
 *     `stream` and return without a host synchronisation (CUDA-graph capturable).
 *   - The caller owns every buffer (q, caches, outputs, workspace). Nothing is allocated
 *     inside a compute call. Size the scratch with tkv_workspace_bytes() and zero it once
 *     with tkv_workspace_init(); kernels leave its control words zeroed again on exit.
 *     One workspace per stream (calls sharing a workspace must be stream-ordered).
 *   - Return value: TKV_OK (0) or a negative TKV_E* code; tkv_last_error() gives a
 *     thread-local message for the last failing call on the calling thread.
 *
 * Data layout (HBM)
 *   q        [B, Hq, d]            bf16   (query of the current decode token, post-RoPE)
 *   k_cache  [B, Hkv, cache_rows, d] bf16  (rows [0, n_ctx[b]) = context: the top-k domain;
 *   v_cache  [B, Hkv, cache_rows, d] bf16   rows [n_ctx[b], n_ctx[b]+n_win[b]) = generation
 *                                            window, always attended, never retrieved —
 *                                            reference GenWindow, attention.py:76-104)
 *   n_ctx, n_win [B]               int32  device arrays, n_ctx[b] + n_win[b] <= cache_rows
 *                                          (n_ctx[b] <= max_ctx; a window past the cache is clamped)
 *   out      [B, Hq, d]            f32
 *   idx      [B, Hq, k]            int32  global row ids (row_offset + local row); -1 pads
 *                                          when k > n_ctx[b] (reference clamps, attention.py:147-149)
 *   scores   [B, Hq, k]            f32    raw (unscaled) dot products q·K[idx]
 *                                          (TopKResult.vals, ann.py:47-55); -inf pads
 *   GQA: q head h reads kv head h / (Hq/Hkv) (contiguous-group convention; the reference is
 *   MHA, SPEC.md:13 — with Hq == Hkv this is exactly the reference mapping).
 */
#ifndef TKV_H_
#define TKV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TKV_VERSION 1

/* status codes (reference error taxonomy, errors.py:4-42, mapped by the Python shim) */
#define TKV_OK 0
#define TKV_EBADSHAPE (-1)  /* -> ShapeError  (ann.py:210-211, tensor.py:33-36)          */
#define TKV_EBADK (-2)      /* -> InputError  (attention.py:144-145, ann.py:212-213)     */
#define TKV_ECONFIG (-3)    /* -> ConfigError (attention.py:122)                          */
#define TKV_ECUDA (-4)      /* CUDA runtime failure (launch, bad pointer, no device)      */
#define TKV_EWORKSPACE (-5) /* workspace too small / misaligned                           */

/* combine modes (reference _joint_attend, attention.py:107-122) */
#define TKV_COMBINE_JOINT 0
#define TKV_COMBINE_ADDITIVE 1

/* flags */
#define TKV_F_SORTED 1u    /* idx/scores ordered score-desc, id-asc (TopKResult order, ann.py:166) */
#define TKV_F_NO_FILTER 2u /* disable the sampled-threshold pre-filter (emit every score)       */
/* flag bit 4u is reserved (was a persistent single-kernel layer step, measured slower; removed) */
#define TKV_F_PARTS(n) ((uint32_t)(n) << 8) /* pipeline parts: scan of part i+1 overlaps the  \
                              k-th selection + V gather of part i (1..15; 0 = automatic)         */
#define TKV_F_PARTS_MASK 0xF00u
#define TKV_F_GATHER_LIST 16u /* V gather as filter pass + balanced list gather (automatic from  \
                                 ~1M selected rows per call)                                    */
#define TKV_F_HOST_Q 128u  /* q (and tkv_topk_decode_step's k_new/v_new) are pinned host buffers   \
                              (device-accessible through UVA): one small kernel stages q into the \
                              workspace, so a host-I/O step needs no H2D copy of its inputs      */
#define TKV_F_HEAD 32u     /* k-th + V gather by the per-head kernel (head_topk_kernel) at any k   */
#define TKV_F_NO_HEAD 64u  /* never the per-head kernel (automatic: k <= 1024, one part)          */
#define TKV_F_CLUSTER 4096u /* k-th + V gather + finish by one 4-CTA thread-block cluster per head  \
                               (clus_topk_kernel; automatic at moderate k, one part)              */
#define TKV_F_NO_CLUSTER 8192u /* never the cluster kernel                                      */
#define TKV_F_SCAN_HMMA 8u /* key scan on register-staged mma.sync (scan.cu) instead of the TMA +  
                              tcgen05 pipeline (scan_tc.cu, the default)                         */

typedef struct tkv_problem {
  int32_t batch;         /* B                                                                  */
  int32_t n_q_heads;     /* Hq                                                                 */
  int32_t n_kv_heads;    /* Hkv; Hq % Hkv == 0 and Hq / Hkv in {1, 2, 4, 8}                     */
  int32_t head_dim;      /* d; this build supports d == 128 (Llama-3 head shape)               */
  int64_t cache_rows;    /* row stride between kv heads in k_cache / v_cache                   */
  int64_t max_ctx;       /* host-side upper bound on n_ctx[b] (grid and workspace sizing)      */
  int32_t k;             /* rows retrieved per q head (clamped per batch entry to n_ctx[b])    */
  int32_t pinned_prefix; /* rows [0, p) always attended (attention.py:152-154); 0 = off        */
  float scale;           /* softmax scale; reference uses 1/sqrt(d) (attention.py:159)         */
  int32_t combine;       /* TKV_COMBINE_*                                                      */
  uint32_t flags;        /* TKV_F_*                                                            */
  int64_t row_offset;    /* global id of local row 0 (token-range shard); 0 when unsharded     */
} tkv_problem;

/* Library / device identification. */
int tkv_version(void);
const char* tkv_last_error(void);
/* Checks that a CUDA device of compute capability 10.0 is current. */
int tkv_device_check(void);

/* Scratch sizing and one-time zeroing of the workspace control words. */
int tkv_workspace_bytes(const tkv_problem* p, size_t* bytes);
int tkv_workspace_init(const tkv_problem* p, void* workspace, size_t bytes, void* stream);

/*
 * One layer's top-k decode attention for all (b, q head): key scan, exact top-k selection
 * (ties to the lower row id), V gather + numerically stable softmax jointly with the
 * window rows.
 * Replaces: topk_attend            attention.py:125-167 (batched over heads and batch)
 *           knn_search (flat)      ann.py:203-218 → _flat_topk ann.py:154-167
 *           ip_scores_all          ann_kernels.py:40-47
 *           _joint_attend          attention.py:107-122
 *           the per-head loop of decode_step, attention.py:213-230
 * `scores` may be NULL (kept in the workspace).
 */
int tkv_topk_decode_attention(const tkv_problem* p, const void* q, const void* k_cache,
                              const void* v_cache, const int32_t* n_ctx, const int32_t* n_win,
                              float* out, int32_t* idx, float* scores, void* workspace,
                              size_t workspace_bytes, void* stream);

/*
 * Exact top-k search only (no attention): knn_search flat, ann.py:203-218 / _flat_topk
 * ann.py:154-167. With TKV_F_SORTED the result is TopKResult-ordered.
 */
int tkv_topk_search(const tkv_problem* p, const void* q, const void* k_cache,
                    const int32_t* n_ctx, int32_t* idx, float* scores, void* workspace,
                    size_t workspace_bytes, void* stream);

/*
 * One decode step of one layer: the window append of this token's k/v (GenWindow.append,
 * attention.py:210; rows n_ctx[b] + n_win[b], then n_win[b] += 1 on device) folded into the
 * attention call (tkv_topk_decode_attention over context + the grown window) — no separate
 * append kernel. n_win is required. k_new/v_new [B, Hkv, d] bf16.
 */
int tkv_topk_decode_step(const tkv_problem* p, const void* q, const void* k_new, const void* v_new,
                         void* k_cache, void* v_cache, const int32_t* n_ctx, int32_t* n_win, float* out,
                         int32_t* idx, float* scores, void* workspace, size_t workspace_bytes, void* stream);

/*
 * Append this token's post-RoPE k/v rows ([B, Hkv, d] bf16) at row base[b] + count[b] of
 * every kv head (base may be NULL → row count[b]). Replaces GenWindow.append,
 * attention.py:94-100 (with base = n_ctx, count = n_win: the window grows after the context).
 * With advance != 0, count[b] += 1 on device, so a decode loop needs no host sync.
 * Rows >= cache_rows are not written (capacity is the caller's, as GenWindow's, :96-97).
 */
int tkv_kv_append(int32_t batch, int32_t n_kv_heads, int32_t head_dim, int64_t cache_rows,
                  void* k_cache, void* v_cache, const void* k_new, const void* v_new,
                  const int32_t* base, int32_t* count, int32_t advance, void* stream);

/*
 * Token-range sharded stages (decode-time context parallelism; the reference is
 * single-process). Shard g holds global rows [row_offset, row_offset+n_ctx[b]).
 *   1. tkv_shard_candidates: local exact top-k → packed candidates cand[B*Hq*k] (uint64,
 *      (order-preserving score key << 32) | ~global_id; 0 = empty slot).
 *   2. caller all-gathers cand from every shard → gathered[n_shards][B*Hq*k].
 *   3. tkv_shard_merge: exact global top-k over the gathered candidates (ties → lower
 *      global id ⇔ lower shard), writes idx/scores (global ids) and the softmax reference max.
 *   4. tkv_shard_partial: V rows this shard owns → partial[B*Hq*(d+1)] = (l, o[d]) against
 *      the global max (no rescale needed on combine).
 *   5. caller all-reduces partial with SUM.
 *   6. tkv_shard_finalize: window rows + normalisation → out.
 */
int tkv_shard_candidates(const tkv_problem* p, const void* q, const void* k_cache,
                         const int32_t* n_ctx, uint64_t* cand, void* workspace,
                         size_t workspace_bytes, void* stream);
int tkv_shard_merge(const tkv_problem* p, const uint64_t* gathered, int32_t n_shards,
                    int32_t* idx, float* scores, void* workspace, size_t workspace_bytes,
                    void* stream);
/*
 * Narrow candidate exchange (sharded.py narrow_exchange_exact): every shard sent only its
 * local top-list_len (list_len <= k), gathered[n_shards][B*Hq*list_len].
 *   tkv_shard_narrow_check: ok[B*Hq] = 1 where the global top-k over the lists is provably
 *     exact (no withheld row can enter it), else 0 — the caller then re-runs the full-k
 *     exchange. tkv_shard_merge_lists: tkv_shard_merge over lists of list_len.
 * (Replaces no reference interface: the reference is single-process.)
 */
int tkv_shard_narrow_check(const tkv_problem* p, const uint64_t* gathered, int32_t n_shards,
                           int32_t list_len, int32_t* ok, void* stream);
int tkv_shard_merge_lists(const tkv_problem* p, const uint64_t* gathered, int32_t n_shards,
                          int32_t list_len, int32_t* idx, float* scores, void* workspace,
                          size_t workspace_bytes, void* stream);
/*
 * Device-driven exchange (no host round trip, CUDA-graph capturable). Every rank publishes its
 * lists in buffers its peers can read (symmetric memory over NVLink; in a one-GPU emulation,
 * plain device buffers):
 *   tkv_shard_candidates2: one key scan; cand_full[B*Hq*k] = the exact local top-k (as
 *     tkv_shard_candidates); cand_narrow[B*Hq*narrow_k] = its entries >= a bound t2 (fewer
 *     than narrow_k of them, zero-padded); bounds[B*Hq*3] = {t2 (every withheld row is below
 *     it), the local k-th composite when the shard has >= k rows else 0, the largest composite}.
 *   tkv_shard_exchange_merge: narrow_lists / full_lists / bounds are DEVICE arrays of n_shards
 *     (<= 16) pointers to the ranks' buffers. Per head, on the device: when at least k narrow
 *     candidates clear T* = max of the ranks' t2, the global top-k is merged from the narrow
 *     lists (exact: no withheld row can enter it), else from the full lists (used_full[B*Hq],
 *     optional, records which). Outputs as tkv_shard_merge; with TKV_F_SORTED, TopKResult order.
 *   tkv_shard_combine: partials is a device array of n_shards pointers to the ranks'
 *     tkv_shard_partial outputs; sums them (the all-reduce) and finishes as tkv_shard_finalize.
 * (Replace no reference interface: the reference is single-process.)
 */
int tkv_shard_candidates2(const tkv_problem* p, int32_t narrow_k, const void* q, const void* k_cache,
                          const int32_t* n_ctx, uint64_t* cand_narrow, uint64_t* cand_full, uint64_t* bounds,
                          void* workspace, size_t workspace_bytes, void* stream);
int tkv_shard_exchange_merge(const tkv_problem* p, const uint64_t* const* narrow_lists,
                             const uint64_t* const* full_lists, const uint64_t* const* bounds, int32_t n_shards,
                             int32_t narrow_k, int32_t* idx, float* scores, int32_t* used_full, void* workspace,
                             size_t workspace_bytes, void* stream);
int tkv_shard_combine(const tkv_problem* p, const float* const* partials, int32_t n_shards, const void* q,
                      const void* k_cache, const void* v_cache, const int32_t* n_ctx, const int32_t* n_win,
                      float* out, void* workspace, size_t workspace_bytes, void* stream);
int tkv_shard_partial(const tkv_problem* p, const void* q, const void* k_cache,
                      const void* v_cache, const int32_t* n_ctx, const int32_t* idx,
                      const float* scores, float* partial, void* workspace,
                      size_t workspace_bytes, void* stream);
int tkv_shard_finalize(const tkv_problem* p, const void* q, const void* k_cache,
                       const void* v_cache, const int32_t* n_ctx, const int32_t* n_win,
                       const float* partial, float* out, void* workspace,
                       size_t workspace_bytes, void* stream);

/*
 * TKKV cache loading (reference on-disk format, cache.py:1-13, 120-257): convert `rows` rows
 * of one f32 section (row-major, d <= 128 floats per row, device memory) into bf16 cache rows
 * of 128 values (zero-padded) at dst (16-byte aligned), stream-ordered. The host side
 * (header validation, section offsets, staging) is paper_2502_06766_b200/cache.py.
 */
int tkv_convert_rows_f32(const float* src, int64_t rows, int32_t d, void* dst, void* stream);

/*
 * Diagnostics (synchronous): how many (b, q head) selections needed the exactness fallback (the
 * sampled threshold admitted fewer than k rows, so the head was re-scanned with threshold 0)
 * on this workspace since tkv_workspace_init.
 */
int tkv_workspace_fallbacks(const tkv_problem* p, const void* workspace, size_t workspace_bytes,
                            uint32_t* heads);

/* ---- Decode-step integration helpers (paper_2502_06766_b200/model.py, BASELINE cfg4): the
 * non-attention elementwise work of one batch-1 layer step, fused (csrc/model_glue.cu). They
 * replace the reference model's per-step NumPy glue around decode_step (reference
 * model.py:255-263 projections / MLP, attention.py:202-233 per-layer loop); all tensors are
 * device pointers, bf16 unless noted, batch 1.
 *   add_rmsnorm:      x[d] += delta[d] (delta may be NULL), h[d] = RMSNorm(x) * w (w f32)
 *   qkv_rope_append:  qkv = [Hq + 2 Hkv][head_dim] projections of this token; RoPE (cos/sin f32
 *                     tables [rows][head_dim/2], row *pos) of q -> q_out [Hq][head_dim] and of k;
 *                     k, v written to the caches' row n_ctx[0] + n_win[0] (caches
 *                     [Hkv][cache_rows][head_dim]); the window counter is not advanced
 *   silu_mul:         out[f] = silu(gate_up[f]) * gate_up[ffn + f]
 *   logits_argmax:    token[0] = first index of the maximum of logits[n] (bf16); logits_f32
 *                     (may be NULL) receives the f32 copy; scratch: 2 zeroed uint64 words,
 *                     left zeroed for the next call */
int tkv_model_add_rmsnorm(void* x, const void* delta, const float* w, float eps, void* h, int32_t d, void* stream);
int tkv_model_qkv_rope_append(const void* qkv, const float* cos_t, const float* sin_t, const int64_t* pos,
                              void* q_out, void* k_cache, void* v_cache, const int32_t* n_ctx,
                              const int32_t* n_win, int64_t cache_rows, int32_t n_heads, int32_t n_kv_heads,
                              int32_t head_dim, void* stream);
int tkv_model_silu_mul(const void* gate_up, void* out, int32_t ffn, void* stream);
int tkv_model_logits_argmax(const void* logits, int32_t n, float* logits_f32, int64_t* token, uint64_t* scratch,
                            void* stream);

/* Number of kernels the last compute call on this thread enqueued (for launch accounting). */
int tkv_last_launch_count(void);

/*
 * Measurement hook: when both events are non-NULL (cudaEvent_t as void*), subsequent compute
 * calls on this thread record `start` / `stop` on their stream immediately before / after the
 * dominant kernel launch (the key-scan kernel: scan_tc_kernel, or scan_kernel with
 * TKV_F_SCAN_HMMA),
 * so a caller can time it with CUDA events on the stream it runs on. Pass NULLs to disable.
 */
int tkv_profile_scan_events(void* start, void* stop);

/*
 * Diagnostics: with a non-NULL device buffer of TKV_TIMELINE_WORDS uint64 (words 0..19:
 * even words initialised to UINT64_MAX, odd words to 0; words 20.. to 0), subsequent
 * multi-kernel compute calls on this thread record %globaltimer first-start / last-end stamps
 * (slot e = words 2e, 2e+1) of: 0 sample, 1 threshold, 2 threshold past its dependency wait,
 * 3 key scan, 4 scan epilogue past its dependency wait, 5 k-th (or the small-k head kernel),
 * 6 gather, 7-9 head kernel: threshold found / rows compacted / V gathered; and slots 10-20
 * accumulate (sum of ns, count) of the head kernel's per-CTA phase durations; slots 21-119 more
 * first/last stamps and phase sums of the other kernels, words 240-248 SM bitmasks (see
 * tools/timeline.py; diagnostic builds record most of them). NULL disables.
 */
#define TKV_TIMELINE_WORDS 256
int tkv_debug_timeline(void* buf);


#ifdef __cplusplus
}
#endif

#endif /* TKV_H_ */
