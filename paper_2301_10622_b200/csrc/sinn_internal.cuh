// sinn_internal.cuh — device data layout of the index and the launch wrappers shared by the
// translation units of libsinn.so.  (Product code; shares nothing with oracle/.)
//
// HBM layout:
//   pi      uint16[n*h]          packed random maps, pi[j*h+o] = pi_o(j)
//   U, L    fp32[cap*m] each     doc-major SoA: column i of the sketch is the m contiguous
//                                cells U[i*m .. i*m+m) (one 256 B-1 KB row per document)
//   live    uint8[cap]           1 = id in X
//   post    uint32[post_len]     inverted index I, tile-major: documents are grouped in tiles of
//                                32 consecutive ids; tile t holds the entries (j << 5) | (i & 31)
//                                for i in tile t, j in nz(x_i), ordered by (i, j) — the lists I[j]
//                                chunked by id range (P:361 Roaring chunks ids likewise),
//                                grouped per document so a warp can own a document's score row
//   off     int64[cap/32 + 1]    tile offsets into post
//   raw     int32 idx / fp32 val pool + per-id (offset int64, nnz int32): vector storage S
//                                for the exact re-rank
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/sinn.h"

namespace sinn {

constexpr uint32_t kNoId = SINN_NO_ID;

// device error bits (validation flags written by kernels, read back by the host)
enum : uint32_t {
  kErrRow = 1u << 0,       // malformed CSR row (index range/order, non-finite, negative under U-only)
  kErrIdReserved = 1u << 1,
  kErrDupId = 1u << 2,
  kErrLive = 1u << 3,      // insert of a live id
  kErrNotLive = 1u << 4,   // delete of a vacant id
  kErrIndptr = 1u << 5,
  kErrNull = 1u << 6,      // indices/values null while some row has entries
  kErrBeyond = 1u << 7,    // (not an error) insert pre-check: some ids lie beyond the current capacity
};

struct DevInfo {  // small device-resident struct read back by the host after validation
  uint32_t err;
  uint32_t max_id;         // insert: largest id; search: number of queries needing the dense path
  uint32_t ids_unsorted;   // insert: 0 if ids[r] < ids[r+1] for all r
  uint32_t pad;            // search: 1 if the batch term table overflowed (retry with a larger one);
                           // insert: the batch's first id
};

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;  // elements allocated
};

}  // namespace sinn

struct sinn_index {
  int32_t n = 0, m = 0, h = 0;
  uint32_t flags = 0;
  bool upper_only = false;
  bool poisoned = false;
  sinn_status deferred = SINN_OK;
  std::string last_error;

  uint16_t* pi = nullptr;  // n*h
  uint2* pi4 = nullptr;    // h <= 4: the term's maps padded to four u16 (one 8-byte load per entry in the sketch build; same allocation as pi)
  int32_t* df = nullptr;   // n: live documents per term (|I[j]|), for the dense-head split
  int64_t max_df = 0;      // max_j df[j] after the last insert (host copy; chooses the scoring kernel)
  int64_t last_stride = 0; // the last tile-path search's sample stride and whether its rows were kept (sinn_stats)
  int64_t last_rows = 0;
  cudaEvent_t df_ready = nullptr;  // recorded after the async copy of max df (read lazily by search)
  bool df_pending = false;

  int64_t cap = 0;  // sketch columns
  int64_t id_end = 0;  // 1 + the largest id ever inserted (tiles at or beyond round-up(id_end, 32) are empty)
  float* U = nullptr;  // fp32 sketch cells (null with bf16)
  float* L = nullptr;
  bool bf16 = false;       // SINN_SKETCH_BF16 (F3, R21): cells in bfloat16, U rounded up, L down
  uint16_t* Ub = nullptr;  // bfloat16 sketch cells (bits), same layout
  uint16_t* Lb = nullptr;
  const void* sU() const { return bf16 ? (const void*)Ub : (const void*)U; }
  const void* sL() const { return bf16 ? (const void*)Lb : (const void*)L; }
  uint8_t* live = nullptr;
  int32_t* ecnt = nullptr;    // per id: entries of the id stored in its tile (tombstones included: a deleted
                              // document keeps its entries until its tile is merged or compacted)
  int32_t* tdead = nullptr;   // per tile: entries of deleted documents still stored in the tile
  int64_t* d_dead = nullptr;  // device: sum of tdead (dead entries in the index)
  int64_t dead_known = 0;     // host copy of *d_dead as of the last round trip
  uint32_t* stamp = nullptr;  // per-id batch stamp for duplicate detection
  uint32_t epoch = 0;
  int64_t live_count = 0;

  // raw-vector store (vector storage S)
  int64_t* raw_off = nullptr;  // cap
  int32_t* raw_nnz = nullptr;  // cap
  int32_t* raw_idx = nullptr;
  float* raw_val = nullptr;
  int64_t raw_used = 0, raw_cap = 0;

  // inverted index (tile-major CSR), double-buffered for merge / compaction
  int64_t* off = nullptr;      // cap/32 + 1
  int64_t* off_alt = nullptr;  // cap/32 + 1
  uint32_t* post = nullptr;
  uint32_t* post_alt = nullptr;
  int64_t post_len = 0, post_cap = 0;
  // tile regions with slack: region t = [off[t], off[t+1]), its first tsz[t] entries in use; tiles from
  // t_region_end on have no region (off = post_len); an insert merges in place while every touched
  // tile fits its region (O(touched tiles)), else the index is re-laid out with fresh slack
  int32_t* tsz = nullptr;     // cap/32
  int64_t t_region_end = 0;
  // bitmap containers (SINN_BITMAP_CONTAINERS, F3): per tile up to 32 (term, 32-bit document mask)
  // pairs, slots [0, cnum[t]) of cont[t * 32 ..); d_cstat = {container slots in use, bits set, bits of
  // deleted documents not yet cleared}
  bool containers = false;
  uint2* cont = nullptr;     // cap/32 * 32
  uint8_t* cnum = nullptr;   // cap/32
  int64_t* d_cstat = nullptr;
  int32_t* ccand = nullptr;  // [64 + 1]: the last bulk load's candidate terms, then their count
  int8_t* cslot = nullptr;   // n: a term's candidate slot, -1 if none

  sinn::DevInfo* d_info = nullptr;    // device: insert/delete validation
  sinn::DevInfo* d_sinfo = nullptr;   // device: search validation (deferred under SINN_SEARCH_NOSYNC)
  sinn::DevInfo* h_info = nullptr;    // pinned host mirror
  int64_t* h_i64 = nullptr;           // pinned host scratch (indptr ends, list bounds)

  // cached workspaces (grow-only)
  void* ws = nullptr;
  size_t ws_bytes = 0;
  void* ws2 = nullptr;
  size_t ws2_bytes = 0;
  void* ws3 = nullptr;  // dense-path score rows
  size_t ws3_bytes = 0;
  uint32_t pair_cap = 0;  // batch term-table capacity (pairs)
  void* hstage = nullptr;  // pinned host staging for the *_host entry points
  size_t hstage_bytes = 0;
  void* dstage = nullptr;  // device staging for the *_host entry points
  size_t dstage_bytes = 0;

  // profiling (sinn_profile): event pairs per phase, folded into totals on read
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<int> ev_phase;  // per recorded pair
  double prof_ms[SINN_NUM_PHASES] = {};
  int64_t prof_calls[SINN_NUM_PHASES] = {};
  int64_t prof_launches[SINN_NUM_PHASES] = {};
};

namespace sinn {

// ---- profiling helpers (api.cu): RAII scope around a phase (an NVTX range named after the phase,
// always; CUDA events when sinn_profile is on); count_launch per kernel launch
struct NvtxScope {  // an NVTX range per ABI call (nsight / ncu --nvtx); a no-op without a tool attached
  explicit NvtxScope(const char* name);
  ~NvtxScope();
};
struct PhaseScope {
  sinn_index* x;
  int ph;
  cudaStream_t s;
  PhaseScope(sinn_index* x_, int ph_, cudaStream_t s_);
  ~PhaseScope();
};
inline void count_launch(sinn_index* x, int ph, int n = 1) {
  if (x->prof) x->prof_launches[ph] += n;
}

// ---- k_util.cu
// SM count of the current device (cudaDevAttrMultiProcessorCount), cached per device: grids are sized
// from it, never from a hard-coded 148
int sm_count();
// *out = sum of v[i] (i < n, w[i] != 0 when w is given): stream-ordered, int64
void launch_sum_i32(const int32_t* v, const uint8_t* w, int64_t n, int64_t* out, cudaStream_t s);
// a launch with an invalid configuration (test hook of the failure semantics: a real, non-sticky error)
void launch_fault_probe(cudaStream_t s);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize = the per-block opt-in maximum less the kernel's
// static shared memory) once per (kernel,
// device): the attribute is per device, so a process with indexes on several GPUs sets it on each
void smem_optin(const void* func);
void exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* tmp, cudaStream_t s);
size_t exclusive_scan_u32_tmp_elems(int64_t n);
void exclusive_scan_i64_small(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s);  // n <= ~1e7
void radix_sort_u64(uint64_t* keys, uint64_t* tmp, int64_t n, int lo_bit, int hi_bit, uint32_t* hist,
                    uint32_t* scan_tmp, cudaStream_t s);
size_t radix_sort_hist_elems(int64_t n);
void fill_u8(uint8_t* p, uint8_t v, int64_t n, cudaStream_t s);
void fill_f32(float* p, float v, int64_t n, cudaStream_t s);
void fill_u16(uint16_t* p, uint16_t v, int64_t n, cudaStream_t s);

// ---- k_insert.cu
void launch_validate_rows(const int64_t* indptr, const int32_t* indices, const float* values, const uint32_t* ids,
                          int64_t nrows, int32_t n, bool upper_only, DevInfo* info, cudaStream_t s);
void launch_check_ids(const uint32_t* ids, int64_t nrows, const uint8_t* live, uint32_t* stamp, uint32_t epoch,
                      bool want_live, int64_t cap, DevInfo* info, cudaStream_t s);
// validate = true: the insert's row validation fused in (flags in info; columns written only when the
// ids passed k_check_ids, the row is well formed and the id < cap)
void launch_sketch_build(const int64_t* indptr, const int32_t* indices, const float* values, const uint32_t* ids,
                         int64_t nrows, const uint16_t* pi, int32_t m, int32_t h, void* U, void* L, bool bf16,
                         cudaStream_t s, bool validate = false, int32_t n = 0, bool upper_only = false,
                         int64_t cap = 0, DevInfo* info = nullptr, const uint2* pi4 = nullptr);
void launch_make_pairs(const int64_t* indptr, const int32_t* indices, const uint32_t* ids, int64_t nrows,
                       uint64_t* keys, uint32_t* direct, unsigned long long* tile_count, cudaStream_t s);
// a batch whose ids do not ascend: rows sorted by id (radix sort of (id << 32 | row) keys on the id
// bits), then placed entry by entry in (id, term) order; per-tile entry counts
void launch_row_sorted_batch(const int64_t* indptr, const int32_t* indices, const uint32_t* ids, int64_t nrows,
                             int hi_bit, uint64_t* keys, uint64_t* keys_tmp, uint32_t* hist, uint32_t* scan_tmp,
                             int64_t* rlen, int64_t* rdst, uint32_t* out, unsigned long long* tile_count, cudaStream_t s);
void launch_unpack_ids(const uint64_t* keys, int64_t nnz, uint32_t* ids_out, cudaStream_t s);
// merge tile by tile; entries of documents that are not live (tombstones, and the old entries of ids
// the batch recycles) are dropped, their ecnt and the tiles' tdead reset
void launch_merge_postings(const int64_t* old_off, const uint32_t* old_post, const int64_t* batch_off,
                           const uint32_t* batch_post, int64_t n, int64_t* new_off, uint32_t* new_post,
                           const uint8_t* live, int32_t* ecnt, int32_t* tdead, int32_t* tsz, cudaStream_t s,
                           int64_t stage_entries = 0);
void launch_merge_fit(const int64_t* off, const int32_t* tsz, const int32_t* tdead, const unsigned long long* tcount,
                      int64_t n, int64_t t_new, int64_t t_last, int32_t last_docs, uint32_t* misfit, int64_t* newcap,
                      int64_t* newscan, cudaStream_t s);
void launch_new_regions(int64_t* off, int64_t t_new, int64_t n, int64_t base, const int64_t* newscan, cudaStream_t s);
void launch_tsz_add(int32_t* tsz, const unsigned long long* tcount, int64_t n, cudaStream_t s);
void fill_i64(int64_t* p, int64_t v, int64_t n, cudaStream_t s);
void launch_raw_append(const int64_t* indptr, const int32_t* indices, const float* values, const uint32_t* ids,
                       int64_t nrows, int64_t pool_base, int32_t* raw_idx, float* raw_val, int64_t* raw_off,
                       int32_t* raw_nnz, uint8_t* live, int32_t* ecnt, int32_t n, int32_t* df, cudaStream_t s);
// new tile sizes of a merge: old size - dead entries + batch entries (tombstones are dropped)
void launch_merge_sizes(const int32_t* tsz, const int32_t* tdead, const unsigned long long* tcount, int64_t n,
                        int64_t t_end, int32_t last_docs, int64_t* sizes, cudaStream_t s);
void launch_add_i64(const int64_t* a, const int64_t* b, int64_t* out, int64_t n, cudaStream_t s);
void launch_df_add(const int32_t* indices, int64_t nnz, int32_t n, int32_t* df, cudaStream_t s);
void launch_raw_compact(const int32_t* raw_nnz, const uint8_t* live, int64_t cap, int64_t* raw_off,
                        const int32_t* old_idx, const float* old_val, int32_t* new_idx, float* new_val,
                        uint32_t* cnt, uint32_t* scan_tmp, cudaStream_t s);
void launch_df_max(const int32_t* df, int32_t n, int64_t* out, cudaStream_t s);

// ---- k_delete.cu
// delete as tombstones, O(deleted entries): ids vacant, df of their terms decremented from the
// raw rows, their entries counted into tdead / d_dead (dropped later by a merge or compaction)
void launch_delete_mark(const uint32_t* ids, int64_t count, uint8_t* live, const int32_t* ecnt, int32_t* tdead,
                        int64_t* d_dead, const int64_t* raw_off, const int32_t* raw_nnz, const int32_t* raw_idx,
                        int32_t* df, const uint2* cont, const uint8_t* cnum, int64_t* cstat, cudaStream_t s);
void launch_count_live_postings(const int32_t* tsz, const int32_t* tdead, int64_t n, int64_t t_end, int64_t* counts,
                                cudaStream_t s);
void launch_compact_postings(const int64_t* off, const uint32_t* post, const uint8_t* live, int64_t n,
                             const int64_t* new_off, uint32_t* new_post, int32_t* ecnt, int32_t* tdead, int32_t* tsz,
                             cudaStream_t s);
void launch_export_term(const int64_t* off, const int32_t* tsz, const uint32_t* post, const uint8_t* live,
                        const uint2* cont, const uint8_t* cnum, int64_t ntiles, uint32_t term, uint32_t* cnt,
                        uint32_t* pos, uint32_t* scan_tmp, uint32_t* out, int64_t cap, cudaStream_t s);
void launch_gather_rows(const uint32_t* ids, int64_t count, const void* src, bool bf16, int32_t m, float* out,
                        cudaStream_t s);
void launch_decode(const uint32_t* ids, const int32_t* terms, const uint8_t* positive, int64_t count,
                   const void* U, const void* L, bool bf16, const uint16_t* pi, int32_t m, int32_t h,
                   bool upper_only, float* out, cudaStream_t s);

// ---- k_search.cu
// Stage-1 rows stored straight into every shard's gather buffer (document sharding): the
// select kernels write each (id, score) row to `n` more destinations — peer-mapped device memory of the
// other GPUs over NVLink, or local buffers — at element offset `off` (= slot * nq * k'), so the
// all-gather of the candidate lists is the select kernel's own stores
constexpr int kGatherMax = 8;
struct GatherDst {
  uint32_t* ids[kGatherMax];
  float* scores[kGatherMax];
  int n = 0;
  int64_t off = 0;
};

struct SearchArgs {
  int64_t nq;
  const int64_t* q_indptr;
  const int32_t* q_indices;
  const float* q_values;
  int32_t k, kprime;
  bool rerank;
  uint32_t* out_ids;     // nq*k (may be null when only stage 1 is wanted)
  float* out_scores;
  uint32_t* cand_ids;    // nq*kprime (stage-1 output; workspace if null)
  float* cand_scores;
  bool exact = false;    // exact MIPS (Alg. 2): entries score with their stored values, no sketch
  int32_t max_terms = 0; // anytime budget: query terms scored per query (0 = T infinity), R20
  const uint32_t* allow = nullptr;  // constrained search (Eq. 3): column mask (bit i of word i/32)
  int64_t allow_words = 0;
  const uint32_t* qmasks = nullptr; // per-query constraint sets (F4): mask table [nmasks][qmask_words]
  int64_t qmask_words = 0;
  int32_t nmasks = 0;
  const int32_t* qmask = nullptr;   // [nq]: mask of each query, -1 = none
  GatherDst gather;                 // extra destinations of the stage-1 rows (n = 0: none)
};
// Returns cudaSuccess or the first CUDA error.  Query validation errors go to idx->d_sinfo->err.
// sync: wait for the batch and complete overflowed queries on the dense path; *needs_retry is set
// when the batch term table was too small (the caller re-issues the call).  Without sync, pending
// dense-path work is reported by sinn_sync as SINN_EAGAIN.
cudaError_t search_batch(sinn_index* idx, const SearchArgs& a, bool sync, cudaStream_t s, std::string* why,
                         bool* needs_retry);

// document sharding: owner re-rank of global candidates, merge of per-shard lists
constexpr int kMergeMaxParts = 64;
constexpr int kMergeMaxItems = 16384;  // parts * kin composites sorted in shared memory per query
cudaError_t rerank_candidates(sinn_index* idx, int64_t nq, const int64_t* q_indptr, const int32_t* q_indices,
                              const float* q_values, int32_t kc, const uint32_t* cand_gids, uint32_t mul, uint32_t add,
                              int32_t k, uint32_t* out_ids, float* out_scores, cudaStream_t s, std::string* why);
cudaError_t launch_merge_topk(int64_t nq, int32_t parts, int32_t kin, const uint32_t* ids, const float* scores,
                              uint32_t mul, const uint32_t* add, int32_t kout, uint32_t* out_ids, float* out_scores,
                              cudaStream_t s);

// ---- k_tile.cu
bool tile_path_supported(int m, bool lower);
int tile_qmax();
int theta_bins();
void launch_qtab(const int64_t* q_indptr, const int32_t* q_indices, const float* q_values, const int32_t* qlist,
                 int64_t q0, int64_t G, int32_t n, bool upper_only, uint32_t* cnt, uint32_t* qoff, uint32_t* cursor,
                 uint32_t* scan_tmp, uint2* pairs, uint32_t pair_cap, uint32_t* sgn, uint4* dir, const uint16_t* pi,
                 int32_t h, uint32_t* bm, DevInfo* info, cudaStream_t s, int32_t max_terms = 0);
struct QMaskArgs {  // per-query constraint sets of one pass (F4); qmask points at the pass's first query
  const uint32_t* masks = nullptr;
  int64_t words = 0;
  int32_t nmasks = 0;
  const int32_t* qmask = nullptr;
};
void launch_doc_score(bool emit, const int64_t* toff, const uint32_t* post, int64_t ntiles_total, int64_t stride,
                      const uint8_t* live, const int32_t* nnz, const void* U, const void* L, bool bf16,
                      const uint16_t* pi, int32_t m, int32_t h, const uint4* dir, const uint2* pairs, int32_t nqc,
                      const float* theta, const uint32_t* list_ok, unsigned long long* cand, uint32_t* cand_cnt,
                      uint32_t cand_cap, uint32_t* hist, uint32_t* nsampled, const float* Qh,
                      const uint32_t* head_cnt, const float* raw_val, const int64_t* raw_off, const uint32_t* allow,
                      int64_t allow_words, uint32_t* sched, cudaStream_t s, QMaskArgs qm = QMaskArgs(),
                      const uint2* cont = nullptr, const uint8_t* cnum = nullptr, const int32_t* raw_idx = nullptr,
                      const int32_t* raw_nnz = nullptr, float* rows = nullptr, int64_t skip = 0);
// candidates of the sampled documents from the rows the sample pass kept (the full pass skips those tiles)
void launch_emit_rows(const float* rows, int64_t ntiles_total, int64_t stride, const uint8_t* live, int32_t nqc,
                      const float* theta, unsigned long long* cand, uint32_t* cand_cnt, uint32_t cand_cap,
                      const uint32_t* allow, int64_t allow_words, QMaskArgs qm, cudaStream_t s);
// per-query constraint sets: live, allowed documents of the sampled tiles for each query of a pass
// (the sample's size per query, for k_theta)
void launch_qmask_sampled(const uint8_t* live, const uint32_t* allow, int64_t allow_words, int64_t ntiles,
                          int64_t stride, QMaskArgs qm, int32_t nqc, uint32_t* nsamp_q, cudaStream_t s);
// k_tile_bf16.cu: the bfloat16-cell instantiation (args: the launcher's DocArgs)
void launch_doc_score_bf16(bool emit, const void* args, bool lower, bool head, cudaStream_t s);
int doc_head_max(int m, bool lower, bool bf16 = false);
void launch_theta(const uint32_t* hist, const uint32_t* nsampled, int nqc, int kprime, float* theta,
                  uint32_t* list_ok, cudaStream_t s, const uint32_t* nsamp_q = nullptr);
void launch_cand_select(const unsigned long long* cand, const uint32_t* cand_cnt, uint32_t cand_cap, int64_t q0,
                        int nqc, int kprime, uint32_t* cand_ids, float* cand_scores, uint8_t* overflow,
                        DevInfo* info, cudaStream_t s, bool final_pass = true, int64_t expected = -1,
                        const float* theta = nullptr, const GatherDst* gather = nullptr);

// ---- k_head.cu (head-term selection of a pass)
int head_cand_cap();

// ---- k_cont.cu (bitmap containers, SINN_BITMAP_CONTAINERS)
int cont_cand_cap();
void launch_cont_bulk(int64_t* off, uint32_t* post, int64_t ta, int64_t nt, int64_t ntiles, const int32_t* df,
                      int32_t n, int64_t live, int32_t* cand, int32_t* ncand, int8_t* slotmap, uint2* cont,
                      uint8_t* cnum, uint32_t* tmp, int64_t* kept, int64_t* scan, int64_t* rel, int32_t* ecnt,
                      int32_t* tsz, int64_t* cstat, cudaStream_t s);
void launch_cont_clear(uint2* cont, const uint8_t* cnum, const uint8_t* live, int64_t ntiles, int64_t* cstat,
                       cudaStream_t s);
// head terms of a pass (coverage df/live x queries/nq >= tau, the best hmax): Qh rows, and the term's
// head mark in dir (k_doc_score's 32-byte directory)
void launch_head_select(const uint32_t* qoff, const int32_t* df, int32_t n, int64_t live, int64_t nq, float tau,
                        const uint2* pairs, uint4* dir, float* Qh, uint32_t* head_cnt, unsigned long long* hcand,
                        uint32_t* nhcand, int hmax, int qrow, cudaStream_t s);

}  // namespace sinn
