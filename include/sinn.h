/*
 * sinn.h — C ABI of the B200-native Sinnamon hot path (arXiv 2301.10622).
 *
 * Sinnamon: approximate top-k Maximum Inner Product Search over streaming sparse real vectors.
 * The index holds, per document id i, an ids-only inverted list entry for every active
 * coordinate (I[j]) and a 2m-cell sketch: an upper half U (cell = max of the values
 * hashed into it) and a lower half L (cell = min), built by Alg. 5.  Search walks
 * the inverted lists of each query coordinate and accumulates q_j * decode into per-query
 * scores (Alg. 6), selects the top-k' and re-ranks them to top-k by exact inner
 * product (Alg. 7).  Deletion removes i from the lists and recycles column i
 * (P:460-468).  Every step runs in this library's own CUDA kernels for sm_100a.
 *
 * Conventions (all calls):
 *   - Return value: a sinn_status (SINN_OK == 0).  Validation is all-or-nothing: a call that
 *     returns SINN_EINVAL / SINN_EEXIST / SINN_ENOTFOUND leaves the index unchanged.
 *   - A CUDA error inside a call returns SINN_ECUDA and poisons the handle: every later call
 *     returns SINN_EPOISONED.  sinn_last_error() returns a message for the last failure.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  All device
 *     work is enqueued on it; device pointers must stay valid until that work has run.
 *   - "device" pointers are CUDA device (or managed) memory; "host" pointers are host memory.
 *   - One handle per stream; no internal locking — callers serialise calls on a handle.
 *   - Document ids are caller-chosen uint32 values < 0xFFFFFFFF; the id is the sketch column
 *     (the paper's identifier i).  0xFFFFFFFF pads result rows.
 *   - The index owns all of its device memory (grown geometrically; freed by sinn_destroy).
 */
#ifndef SINN_H_
#define SINN_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sinn_index sinn_index; /* opaque; owns all index device memory */
typedef int32_t sinn_status;

#define SINN_OK 0
#define SINN_EINVAL 1     /* malformed arguments or input rows */
#define SINN_ENOMEM 2     /* device allocation failed (index unchanged) */
#define SINN_EEXIST 3     /* insert of an id that is already live */
#define SINN_ENOTFOUND 4  /* delete of an id that is not live */
#define SINN_ECUDA 5      /* CUDA error; the handle is now poisoned */
#define SINN_EPOISONED 6  /* an earlier call hit a CUDA error */
#define SINN_EAGAIN 7     /* a SINN_SEARCH_NOSYNC search needs a synchronous re-run (see sinn_sync) */

#define SINN_NO_ID 0xFFFFFFFFu

/* sinn_create flags */
#define SINN_UPPER_ONLY 1u /* Sinnamon+ (P:358): non-negative data, upper sketch U only */
#define SINN_SKETCH_BF16 2u /* sketch cells stored in bfloat16: each U cell
                               the exact max rounded UP, each L cell the min rounded DOWN, so decodes
                               still bound x from the correct side and Theorem 1 holds
                               (R21).  Halves the sketch bytes.  Requires m % 8 == 0. */

#define SINN_BITMAP_CONTAINERS 4u /* Roaring-style bitmap containers for dense lists (SURVEY §8(f)
                               F3): the ids-only inverted index I is held per 32-id tile (DESIGN.md
                               §4); where a term has >= 2 of a tile's documents (its list is locally
                               dense), bulk loads store the pair (term, 32-bit document mask) instead
                               of one entry per document — up to 32 such containers per tile, the
                               densest first.  Searches, exports and the exact mode read both forms;
                               ids recycled or deleted later lose their container bits (their new
                               entries are stored one by one).  DESIGN.md §5.7. */

/* sinn_search flags */
#define SINN_SEARCH_NOSYNC 1u /* do not wait for the stream; errors surface at sinn_sync (see there) */

/* Limits (SINN_EINVAL beyond them) */
#define SINN_MAX_N (1 << 27) /* dimensionality: index entries pack (term << 5) | document-in-tile in 32 bits */
#define SINN_MAX_M 4096      /* sketch cells per side */
#define SINN_MAX_H 8         /* random mappings */
#define SINN_MAX_KPRIME 16384

/* Library version string, e.g. "sinn-b200 0.1 sm_100a". */
const char* sinn_version(void);

/* Create an empty index.  [P:312 h random maps pi_o: [n] -> [m]; P:333 sketch 2m x |X|]
 *   n          dimensionality (1..SINN_MAX_N = 2^27: an index entry packs (j << 5) | (i mod 32) into
 *              32 bits, so larger term ids would wrap; rejected with SINN_EINVAL)
 *   m          sketch cells per side (1..SINN_MAX_M)
 *   h          number of random mappings (1..SINN_MAX_H)
 *   hash_table host int32[n*h], row-major: pi_o(j) = hash_table[j*h + o], each in [0, m).
 *              Copied at create; the caller keeps ownership.
 *   flags      0 or a combination of SINN_UPPER_ONLY, SINN_SKETCH_BF16, SINN_BITMAP_CONTAINERS
 *   out        receives the handle (NULL on failure)
 * Errors: SINN_EINVAL (bad n/m/h/table/out), SINN_ENOMEM, SINN_ECUDA. Synchronises `stream`. */
sinn_status sinn_create(int32_t n, int32_t m, int32_t h, const int32_t* hash_table, uint32_t flags, void* stream,
                        sinn_index** out);

/* Free every device allocation of the index (waits for the device).  NULL is a no-op. */
sinn_status sinn_destroy(sinn_index* index);

/* Insert a batch of documents (Alg. 5): append id i to I[j] for every active j, write
 * column i of U (and L): u[k] = max, l[k] = min over active j with some pi_o(j) = k; untouched
 * cells hold -inf (U) / +inf (L).  A stored entry is active even when its value is 0 (P:473
 * footnote); -0.0 is stored as +0.0.
 *   nrows     number of rows (>= 0)
 *   indptr    device int64[nrows+1], non-decreasing (any base: row r is [indptr[r], indptr[r+1]))
 *   indices   device int32[...], strictly increasing within a row, each in [0, n)
 *   values    device float32[...], finite; >= 0 under SINN_UPPER_ONLY
 *   ids       device uint32[nrows]: distinct, not live, != SINN_NO_ID.  A vacant (deleted) id is
 *             recycled: its column is fully overwritten.
 * Errors: SINN_EINVAL (malformed rows, duplicate ids), SINN_EEXIST (live id), SINN_ENOMEM.
 * Synchronises `stream` twice (validation flags, capacity). */
sinn_status sinn_insert(sinn_index* index, int64_t nrows, const int64_t* indptr, const int32_t* indices,
                        const float* values, const uint32_t* ids, void* stream);

/* As sinn_insert, with HOST pointers; the rows are copied to the device inside the call. */
sinn_status sinn_insert_host(sinn_index* index, int64_t nrows, const int64_t* indptr, const int32_t* indices,
                             const float* values, const uint32_t* ids, void* stream);

/* Reserve device capacity for ids < max_docs and `postings` stored entries in total (index entries
 * and raw-store entries), so that a bulk load does not grow the arrays batch by batch.  Never
 * shrinks; the index contents are unchanged.  Errors: SINN_EINVAL (negative sizes, max_docs above
 * the id range), SINN_ENOMEM.  Stream-ordered (allocations come from the device's stream-ordered
 * pool). */
sinn_status sinn_reserve(sinn_index* index, int64_t max_docs, int64_t postings, void* stream);

/* Delete documents: remove every instance of each id from the inverted lists; the
 * sketch column is left stale and the id becomes reusable by a later insert.
 *   count  number of ids (>= 0);  ids  device uint32[count], distinct, all live.
 * Errors: SINN_ENOTFOUND (an id not live), SINN_EINVAL (duplicates).  Synchronises `stream`. */
sinn_status sinn_delete(sinn_index* index, int64_t count, const uint32_t* ids, void* stream);

/* As sinn_delete with a HOST id array. */
sinn_status sinn_delete_host(sinn_index* index, int64_t count, const uint32_t* ids, void* stream);

/* Search a batch of queries (Alg. 6 + Alg. 7, T = infinity).
 *   nq          number of queries (>= 0)
 *   q_indptr    device int64[nq+1];  q_indices device int32 (strictly increasing per row, < n);
 *   q_values    device float32, finite.  Entries with q_j == 0 are skipped (nz(q)).
 *               Under SINN_UPPER_ONLY a negative q_j contributes 0 (0 lower-bounds x >= 0).
 *   k, kprime   1 <= k <= kprime <= SINN_MAX_KPRIME (k' >= k).  If kprime exceeds the
 *               live count, every live document is a candidate.
 *   rerank      nonzero: V = top-k' by approximate score, re-scored exactly against the stored
 *               raw vectors, top-k of those returned (Alg. 7); zero: top-k by approximate score.
 *   out_ids     device uint32[nq*k], out_scores device float32[nq*k]: row q best first;
 *               rows with fewer than k results are padded with (SINN_NO_ID, -inf).
 *               Untouched live documents score 0 and are eligible; deleted ids never appear.
 *               Ties are broken by ascending id.
 *   flags       0 or SINN_SEARCH_NOSYNC.
 * Errors: SINN_EINVAL (arguments, or malformed query rows: then outputs are undefined).
 * Without SINN_SEARCH_NOSYNC the call waits for `stream` (validation flag, completion of queries
 * whose candidate buffer overflowed, on the dense path). */
sinn_status sinn_search(sinn_index* index, int64_t nq, const int64_t* q_indptr, const int32_t* q_indices,
                        const float* q_values, int32_t k, int32_t kprime, int32_t rerank, uint32_t* out_ids,
                        float* out_scores, uint32_t flags, void* stream);

/* As sinn_search with HOST query and output arrays: the queries are copied to the device and the
 * results back inside the call, which returns after the results have landed in host memory. */
sinn_status sinn_search_host(sinn_index* index, int64_t nq, const int64_t* q_indptr, const int32_t* q_indices,
                             const float* q_values, int32_t k, int32_t kprime, int32_t rerank, uint32_t* out_ids,
                             float* out_scores, void* stream);

/* sinn_search with the anytime budget of Alg. 6: stage 1 scores
 * only each query's first max_terms non-zero terms in the order of descending abs(q_j) (ties by
 * ascending j) — the GPU's form of the paper's time budget T (R20); the exact re-rank
 * (Alg. 7) uses the whole query.  max_terms = 0 is T = infinity (= sinn_search).  Other arguments,
 * outputs and errors as sinn_search; SINN_EINVAL also for max_terms < 0. */
sinn_status sinn_search_anytime(sinn_index* index, int64_t nq, const int64_t* q_indptr, const int32_t* q_indices,
                                const float* q_values, int32_t k, int32_t kprime, int32_t rerank, int32_t max_terms,
                                uint32_t* out_ids, float* out_scores, uint32_t flags, void* stream);

/* Constrained search (Eq. 3): sinn_search whose solution set holds only the
 * documents that pass the caller's constraints, given as a column mask — the paper's "masking out
 * those columns in X~ that do not satisfy the given conditions".
 *   allow        device uint32[allow_words]: document i may be returned iff bit (i & 31) of word
 *                i >> 5 is set; ids at or beyond 32 * allow_words are masked out.  One mask for the
 *                whole batch (group queries by constraint set).  allow_words = 0 masks out everything.
 * Other arguments, outputs and errors as sinn_search (SINN_EINVAL also for a bad mask); a masked-out
 * document behaves exactly as a vacant one. */
sinn_status sinn_search_filtered(sinn_index* index, int64_t nq, const int64_t* q_indptr, const int32_t* q_indices,
                                 const float* q_values, int32_t k, int32_t kprime, int32_t rerank,
                                 const uint32_t* allow, int64_t allow_words, uint32_t* out_ids, float* out_scores,
                                 uint32_t flags, void* stream);

/* Constrained search with a constraint set PER QUERY (Eq. 3): query q's solution
 * set holds only the documents of mask qmask[q] of a table of column masks, so queries with different
 * filters share one batch.
 *   masks        device uint32[nmasks * mask_words], mask r = words [r * mask_words, (r + 1) * mask_words):
 *                document i passes mask r iff bit (i & 31) of word r * mask_words + (i >> 5) is set; ids at
 *                or beyond 32 * mask_words fail every mask
 *   qmask        device int32[nq]: the mask of query q, in [0, nmasks), or -1 for no constraint
 * Other arguments, outputs and errors as sinn_search; SINN_EINVAL also for nmasks < 0, mask_words < 0,
 * a null table with nmasks > 0, or a null qmask.  A query's masked-out documents behave for it exactly as
 * vacant ones; qmask entries outside [-1, nmasks) are SINN_EINVAL (checked on the device, reported by
 * this call, or by sinn_sync under SINN_SEARCH_NOSYNC). */
sinn_status sinn_search_masked(sinn_index* index, int64_t nq, const int64_t* q_indptr, const int32_t* q_indices,
                               const float* q_values, int32_t k, int32_t kprime, int32_t rerank, const uint32_t* masks,
                               int64_t mask_words, int32_t nmasks, const int32_t* qmask, uint32_t* out_ids,
                               float* out_scores, uint32_t flags, void* stream);

/* Exact top-k MIPS over the live documents (Alg. 2, LinScan retrieval; the ground truth
 * of recall@k): s_i = sum_j q_j x_ij from the stored values (the re-rank store), documents that
 * share no coordinate with q score 0; negative q_j count under SINN_UPPER_ONLY too.  The
 * same walk as sinn_search with each entry's stored value in place of its sketch decode, fp32
 * accumulation.  Device arrays as sinn_search (out_ids/out_scores nq*k, padded with
 * (SINN_NO_ID, -inf), ties by ascending id).  1 <= k <= SINN_MAX_KPRIME.  Synchronises `stream`. */
sinn_status sinn_search_exact(sinn_index* index, int64_t nq, const int64_t* q_indptr, const int32_t* q_indices,
                              const float* q_values, int32_t k, uint32_t* out_ids, float* out_scores,
                              void* stream);

/* Stage 1 only (Alg. 6 + Alg. 7 line 1): the top-k' candidates V with their approximate scores,
 * best first (ties by ascending id), padded with (SINN_NO_ID, -inf).  Device outputs
 * cand_ids uint32[nq*kprime], cand_scores float32[nq*kprime].  Synchronises `stream`. */
sinn_status sinn_search_stage1(sinn_index* index, int64_t nq, const int64_t* q_indptr, const int32_t* q_indices,
                               const float* q_values, int32_t kprime, uint32_t* cand_ids, float* cand_scores,
                               void* stream);

/* ---- document sharding across GPUs (the paper's Sinnamon|| splits list segments across
 * threads and merges their heaps).  Shard r of W holds the documents with global id g, g % W == r,
 * under the local id g / W (global = local * W + r); every shard scores the whole query batch
 * (sinn_search_stage1), the per-shard candidate lists are exchanged once (an all-gather: NCCL, the
 * caller's), merged into the global V (sinn_merge_topk), re-ranked by their owners (sinn_rerank) and the
 * per-shard top-k lists merged again.  The result equals the unsharded search of the same documents:
 * the global top-k' is contained in the union of the shards' top-k'. */

/* sinn_search_stage1 whose select kernels store the rows straight into every shard's gather buffer: the
 * all-gather of step 2 done by the producing kernel's own stores (peer-mapped memory over NVLink /
 * NVSwitch; no collective launch).
 *   world, slot   number of shards (1..8) and this shard's slot
 *   dst_ids, dst_scores   HOST arrays of `world` DEVICE pointers: buffer d is shard d's gather buffer,
 *                 uint32 / float32 [world][nq][kprime] (dst[slot] is this shard's own; the others are
 *                 peer-mapped, or local in a single-process test).  This call writes rows
 *                 [slot][0..nq) of every buffer; rows of other slots are untouched.
 * The caller synchronises the shards (a barrier) before reading a buffer.  Other arguments, errors and
 * synchronisation as sinn_search_stage1. */
sinn_status sinn_search_stage1_gather(sinn_index* index, int64_t nq, const int64_t* q_indptr, const int32_t* q_indices,
                                      const float* q_values, int32_t kprime, int32_t world, int32_t slot,
                                      uint32_t* const* dst_ids, float* const* dst_scores, void* stream);

/* Exact re-rank of caller-supplied candidates (Alg. 7 lines 2-5, on this shard's part of V).
 *   q_*        the query batch (device CSR, as sinn_search; rows are not re-validated: pass the batch
 *              that stage 1 accepted)
 *   kc         candidates per query (1..SINN_MAX_KPRIME); cand_ids device uint32[nq*kc] GLOBAL ids,
 *              SINN_NO_ID = none.  A candidate g is re-ranked iff g % id_mul == id_add and its local id
 *              (g - id_add) / id_mul is live in this index; every other candidate is skipped.
 *   id_mul, id_add   the shard's id map (W and r; 1 and 0 for an unsharded index)
 *   k          1 <= k <= kc; out_ids device uint32[nq*k] GLOBAL ids, out_scores float32[nq*k]: the top-k
 *              of the owned candidates by exact inner product, best first, ties by ascending id, padded
 *              with (SINN_NO_ID, -inf).
 * Stream-ordered (no synchronisation).  Errors: SINN_EINVAL, SINN_ENOMEM, SINN_ECUDA (poisons). */
sinn_status sinn_rerank(sinn_index* index, int64_t nq, const int64_t* q_indptr, const int32_t* q_indices,
                        const float* q_values, int32_t kc, const uint32_t* cand_ids, uint32_t id_mul, uint32_t id_add,
                        int32_t k, uint32_t* out_ids, float* out_scores, void* stream);

/* Merge `parts` per-shard result lists into one top-kout per query (FindLargest, Alg. 3, over
 * the union; needs no index).
 *   ids, scores   device uint32 / float32 [parts][nq][kin] (the layout an all-gather of [nq][kin] leaves),
 *                 SINN_NO_ID entries are skipped
 *   id_mul, id_add   host uint32[parts] id_add (NULL = zeros): an id of part p becomes id * id_mul +
 *                 id_add[p] (local -> global; 1 and zeros when the ids are global already); results
 *                 at or beyond SINN_NO_ID are dropped
 *   kout          entries written per query: out_ids uint32[nq*kout], out_scores float32[nq*kout], by
 *                 (score descending, global id ascending), padded with (SINN_NO_ID, -inf)
 * Limits: 1 <= parts <= 64, parts * kin <= 16384, 1 <= kout <= 16384 (SINN_EINVAL beyond).
 * Stream-ordered.  Errors: SINN_EINVAL, SINN_ECUDA. */
sinn_status sinn_merge_topk(int64_t nq, int32_t parts, int32_t kin, const uint32_t* ids, const float* scores,
                            uint32_t id_mul, const uint32_t* id_add, int32_t kout, uint32_t* out_ids, float* out_scores,
                            void* stream);

/* Wait for `stream` and return the deferred status of SINN_SEARCH_NOSYNC searches (then cleared):
 * SINN_EINVAL for a malformed query row, SINN_EAGAIN when a query of such a batch overflowed its
 * candidate buffer (or the batch term table overflowed): its output rows are then incomplete and
 * the batch must be re-run without SINN_SEARCH_NOSYNC, which completes such queries on the dense
 * path.  Synchronous searches never return SINN_EAGAIN. */
sinn_status sinn_sync(sinn_index* index, void* stream);

/* Message describing the last failure on this handle ("" if none).  Owned by the handle. */
const char* sinn_last_error(const sinn_index* index);

/* ---- debug / parity exports (not on the timed path) ---- */

/* Copy the sketch columns of `ids` (device uint32[count], each < capacity): device U float32[count*m]
 * and, unless SINN_UPPER_ONLY, device L float32[count*m] (L may be NULL to skip); bfloat16 cells
 * (SINN_SKETCH_BF16) are widened to float32 exactly.  Synchronises. */
sinn_status sinn_export_sketch(sinn_index* index, int64_t count, const uint32_t* ids, float* U, float* L,
                               void* stream);

/* Copy I[term] (sorted ascending) into device `out` (capacity `cap` entries); *len (host) receives the
 * list length (the copy is truncated to cap).  Synchronises. */
sinn_status sinn_export_postings(sinn_index* index, int32_t term, uint32_t* out, int64_t cap, int64_t* len,
                                 void* stream);

/* Decode estimates with the scoring path's own decode: out[t] = min_o U[ids[t]][pi_o(terms[t])] if
 * positive[t] != 0, else max_o L[ids[t]][pi_o(terms[t])] (0 under SINN_UPPER_ONLY).  Device arrays of
 * length count.  The caller guarantees terms[t] is active for ids[t].  Synchronises. */
sinn_status sinn_decode(sinn_index* index, int64_t count, const uint32_t* ids, const int32_t* terms,
                        const uint8_t* positive, float* out, void* stream);

typedef struct {
  int64_t live;            /* live documents */
  int64_t capacity;        /* sketch columns allocated */
  int64_t postings;        /* live postings of the inverted index (entries + container bits) */
  int64_t raw_entries;     /* entries held by the raw-vector store (incl. garbage of deleted ids) */
  int64_t bytes_postings;  /* device bytes of the inverted index */
  int64_t bytes_sketch;    /* device bytes of U and L */
  int64_t bytes_raw;       /* device bytes of the raw-vector store */
  int64_t bytes_workspace; /* device bytes of cached search/insert workspaces */
  int64_t containers;      /* bitmap containers in use (SINN_BITMAP_CONTAINERS), 8 bytes each */
  int64_t container_postings; /* postings held as container bits (live documents) */
  int64_t sample_stride;   /* the last search's threshold sample: every sample_stride-th tile (0: none yet) */
  int64_t sample_rows_kept;/* 1 if that sample kept its documents' score rows, i.e. the full scoring pass
                              covered the other (1 - 1 / sample_stride) of the tiles */
} sinn_stats_t;

/* Fill *out (host).  No device work. */
sinn_status sinn_stats(const sinn_index* index, sinn_stats_t* out);

/* ---- in-process profiling (CUDA events around each kernel phase, on the call's stream) ---- */
#define SINN_NUM_PHASES 12
enum {
  SINN_PH_INIT = 0,      /* threshold: sample pass(es) + theta (dense path: row init) */
  SINN_PH_SCORE = 1,     /* postings walk + decode + accumulate (Alg. 6), the full pass */
  SINN_PH_SELECT = 2,    /* top-k' selection (Alg. 7 line 1)             */
  SINN_PH_RERANK = 3,    /* exact re-rank gather-dot (Alg. 7 lines 2-4)  */
  SINN_PH_FINAL = 4,     /* final top-k (Alg. 7 line 5)                  */
  SINN_PH_VALIDATE = 5,  /* insert/delete validation                     */
  SINN_PH_SKETCH = 6,    /* sketch build (Alg. 5 lines 3-9)              */
  SINN_PH_POSTINGS = 7,  /* postings sort + merge (Alg. 5 line 2)        */
  SINN_PH_RAW = 8,       /* raw-vector store append                      */
  SINN_PH_DELETE = 9,    /* delete compaction                            */
  SINN_PH_PREP = 10      /* query prep: batch term table + directory (Alg. 6 lines 1-2) */
};
typedef struct {
  double ms[SINN_NUM_PHASES];       /* summed CUDA-event time per phase since sinn_profile(.., 1) */
  int64_t calls[SINN_NUM_PHASES];   /* phase executions (one per chunk / call)                    */
  int64_t launches[SINN_NUM_PHASES];/* kernel launches of this library per phase                  */
} sinn_profile_t;

/* enable != 0: start recording (clears totals); enable == 0: stop.  No device work. */
sinn_status sinn_profile(sinn_index* index, int32_t enable);

/* Wait for `stream`, fold all recorded event pairs into *out (host) and keep recording. */
sinn_status sinn_profile_read(sinn_index* index, sinn_profile_t* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SINN_H_ */
