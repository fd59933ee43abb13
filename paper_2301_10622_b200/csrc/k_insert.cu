// k_insert.cu — insert path (Alg. 5): batch validation, the sketch-build kernel
// (warp per document, shared-memory max/min), postings build (batch (term,id) pairs, stable radix
// sort, per-term merge into the CSR inverted index) and the raw-vector store append.
#include <math.h>

#include "sinn_device.cuh"
#include <algorithm>

#include "sinn_internal.cuh"

namespace sinn {

namespace {

inline unsigned grid_for(int64_t n, int threads, int64_t cap_blocks = 0) {
  if (cap_blocks <= 0) cap_blocks = (int64_t)sm_count() * 32;
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap_blocks) b = cap_blocks;
  return (unsigned)b;
}

// order-preserving int image of a float (signed compare == float compare, -0 < +0)
__device__ __forceinline__ int f2ord(float f) {
  int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float ord2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

// ---------------------------------------------------------------- validation
// one warp per row: indices in [0,n), strictly increasing, values finite (>= 0 under Sinnamon+)
__global__ void k_validate_rows(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                                const float* __restrict__ values, const uint32_t* __restrict__ ids, int64_t nrows,
                                int32_t n, int upper_only, DevInfo* info) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint32_t err = 0, maxid = 0, unsorted = 0;
  for (int64_t r = warp; r < nrows; r += nwarps) {
    const int64_t b = indptr[r], e = indptr[r + 1];
    if (e < b) { err |= kErrIndptr; continue; }
    if (lane == 0) {
      uint32_t id = ids[r];
      if (id == kNoId) err |= kErrIdReserved;
      maxid = max(maxid, id);
      if (r + 1 < nrows && !(id < ids[r + 1])) unsorted = 1;
      if (r == 0) info->pad = id;
    }
    if (e > b && (!indices || !values)) {  // null arrays: no entry is read (SINN_EINVAL, not a fault)
      err |= kErrNull;
      continue;
    }
    for (int64_t p = b + lane; p < e; p += 32) {
      const int32_t j = indices[p];
      const float x = values[p];
      if (j < 0 || j >= n) err |= kErrRow;
      if (p > b && indices[p - 1] >= j) err |= kErrRow;
      if (!isfinite(x)) err |= kErrRow;
      if (upper_only && x < 0.0f) err |= kErrRow;
    }
  }
  err = __reduce_or_sync(0xffffffffu, err);
  maxid = __reduce_max_sync(0xffffffffu, maxid);
  unsorted = __reduce_or_sync(0xffffffffu, unsorted);
  if (lane == 0) {
    if (err) atomicOr(&info->err, err);
    atomicMax(&info->max_id, maxid);
    if (unsorted) atomicOr(&info->ids_unsorted, 1u);
  }
}

// insert (want_live = false): id must be vacant; delete (want_live = true): id must be live.
// duplicates within the batch detected with a per-id stamp (atomicExch returns the old stamp).
// Insert runs this before the capacity grows (one host round trip with k_validate_rows): an id at or
// beyond the capacity is vacant by definition and only flagged (kErrBeyond) — the host re-checks the
// batch for duplicates after growing only when such ids exist and the batch's ids do not ascend.
__global__ void k_check_ids(const uint32_t* __restrict__ ids, int64_t nrows, const uint8_t* __restrict__ live,
                            uint32_t* __restrict__ stamp, uint32_t epoch, int want_live, int64_t cap,
                            DevInfo* info) {
  uint32_t err = 0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t id = ids[r];
    if ((int64_t)id >= cap) {
      err |= want_live ? kErrNotLive : (id == kNoId ? kErrIdReserved : kErrBeyond);
      continue;
    }
    const bool is_live = live[id] != 0;
    if (want_live && !is_live) err |= kErrNotLive;
    if (!want_live && is_live) err |= kErrLive;
    if (atomicExch(&stamp[id], epoch) == epoch) err |= kErrDupId;
  }
  if (err) atomicOr(&info->err, err);
}

// ---------------------------------------------------------------- sketch build (Alg. 5 lines 3-9)
// One warp per document.  The warp keeps the m-cell u and l vectors in shared memory as
// order-preserving ints, folds its active coordinates in with smem atomicMax/atomicMin (max/min
// are exact, so the result is independent of the order), then writes column i of U and L with
// coalesced stores.  Untouched cells keep the identities -inf (U) / +inf (L).  BF (F3, R21): the
// exact fp32 extremes are stored as bfloat16 bits, U rounded up and L rounded down.
// VAL: the insert's validation pass fused in (one read of the batch instead of two): the rows are
// checked as k_validate_rows does (range, order, finite, sign, indptr, null arrays, reserved id, max /
// first id, id order) while they are folded, and a column is written only when the batch passed
// k_check_ids (launched just before: no live or repeated id — a live document's column is never
// touched), the row is well formed and the id lies below the capacity (else the host re-runs the
// plain build after growing).  A rejected batch may thus have rewritten columns of vacant ids, which
// nothing reads (R18: observable all-or-nothing).
template <bool BF, bool VAL>
__global__ void k_sketch_build(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                               const float* __restrict__ values, const uint32_t* __restrict__ ids, int64_t nrows,
                               const uint16_t* __restrict__ pi, int32_t m, int32_t h, void* __restrict__ U_,
                               void* __restrict__ L_, int32_t n, int upper_only, int64_t cap, DevInfo* info,
                               const uint2* __restrict__ pi4) {
  extern __shared__ int sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const bool lower = L_ != nullptr;
  float* U = reinterpret_cast<float*>(U_);
  float* L = reinterpret_cast<float*>(L_);
  uint16_t* Ub = reinterpret_cast<uint16_t*>(U_);
  uint16_t* Lb = reinterpret_cast<uint16_t*>(L_);
  int* su = sm + (size_t)w * 2 * m;
  int* sl = su + m;
  const int kNegInf = f2ord(-INFINITY), kPosInf = f2ord(INFINITY);
  uint32_t err = 0, maxid = 0, unsorted = 0;
  // (VAL) k_check_ids ran before in stream order: any live, repeated or reserved id blocks every write
  // (the flag word is loaded here and tested only where a column is written: its latency hides behind the
  // first document's fold instead of stalling every warp at its start — 12 % of the stall samples, ncu)
  const uint32_t err_ids = VAL ? *(volatile uint32_t*)&info->err : 0u;
  for (int64_t r = (int64_t)blockIdx.x * nw + w; r < nrows; r += (int64_t)gridDim.x * nw) {
    for (int k = lane; k < m; k += 32) {
      su[k] = kNegInf;
      sl[k] = kPosInf;
    }
    __syncwarp();
    const int64_t b = indptr[r], e = indptr[r + 1];
    bool row_bad = false;
    if (VAL) {
      const uint32_t id = ids[r];
      if (lane == 0) {
        if (id == kNoId) err |= kErrIdReserved;
        maxid = max(maxid, id);
        if (r + 1 < nrows && !(id < ids[r + 1])) unsorted = 1;
        if (r == 0) info->pad = id;
      }
      if (e < b) err |= kErrIndptr;
      if (e > b && (!indices || !values)) err |= kErrNull;  // no entry is read (SINN_EINVAL, not a fault)
      if (e < b || (e > b && (!indices || !values))) {
        __syncwarp();
        continue;
      }
    }
    // a long document with padded maps: EIGHT entries per lane per round (a 250-entry document is one
    // round: indptr -> entries -> maps -> fold, three dependent memory round trips instead of five)
    if (pi4 && h <= 4 && e - b > 128) {
      for (int64_t p0 = b + lane; p0 < e; p0 += 256) {
        int32_t j[8], jp[8];
        float xv[8];
        int xo[8];
        // every load of the round is issued before the first check: the checks are branch-free (a
        // short-circuit `||` made each entry's loads wait for the previous entry's comparison)
#pragma unroll
        for (int u = 0; u < 8; u++) {
          const int64_t p = p0 + 32 * u;
          const bool in = p < e;
          j[u] = in ? __ldg(indices + p) : -1;
          xv[u] = in ? __ldg(values + p) : 0.0f;
          jp[u] = (VAL && in && p > b) ? __ldg(indices + p - 1) : -1;
        }
#pragma unroll
        for (int u = 0; u < 8; u++) {
          const bool in = p0 + 32 * u < e;
          float x = xv[u];
          if (VAL) {
            const bool bad = in & ((j[u] < 0) | (j[u] >= n) | (jp[u] >= j[u]) | !isfinite(x) | ((upper_only != 0) & (x < 0.0f)));
            row_bad |= bad;
            if (bad) j[u] = -1;
          }
          if (x == 0.0f) x = 0.0f;
          xo[u] = f2ord(x);
        }
        uint2 pk[8];
#pragma unroll
        for (int u = 0; u < 8; u++) pk[u] = j[u] >= 0 ? __ldg(pi4 + j[u]) : make_uint2(0xffffffffu, 0xffffffffu);
#pragma unroll
        for (int u = 0; u < 8; u++) {
          if (j[u] < 0) continue;
          const uint32_t kk[4] = {pk[u].x & 0xffffu, pk[u].x >> 16, pk[u].y & 0xffffu, pk[u].y >> 16};
#pragma unroll
          for (int o = 0; o < 4; o++)
            if (o < h) {
              atomicMax(&su[kk[o]], xo[u]);
              if (lower) atomicMin(&sl[kk[o]], xo[u]);
            }
        }
      }
    } else
    // four entries per lane per round: every load of the round (entries, then their buckets) is issued
    // before the first atomic, so the warp waits on one memory round trip per round, not per entry
    for (int64_t p0 = b + lane; p0 < e; p0 += 128) {
      int32_t j[4], jp[4];
      float xv[4];
      int xo[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {  // loads first, branch-free checks after (see the 8-entry round)
        const int64_t p = p0 + 32 * u;
        const bool in = p < e;
        j[u] = in ? __ldg(indices + p) : -1;
        xv[u] = in ? __ldg(values + p) : 0.0f;
        jp[u] = (VAL && in && p > b) ? __ldg(indices + p - 1) : -1;
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const bool in = p0 + 32 * u < e;
        float x = xv[u];
        if (VAL) {  // a malformed entry is flagged and not folded (its bucket would be out of range)
          const bool bad = in & ((j[u] < 0) | (j[u] >= n) | (jp[u] >= j[u]) | !isfinite(x) | ((upper_only != 0) & (x < 0.0f)));
          row_bad |= bad;
          if (bad) j[u] = -1;
        }
        if (x == 0.0f) x = 0.0f;  // -0.0 is stored as +0.0 (R19)
        xo[u] = f2ord(x);
      }
      if (h <= 4) {
        int k[4][4];
        if (pi4) {
          // the term's maps padded to four u16: ONE 8-byte load per entry instead of h 2-byte loads (90 %
          // of this kernel's L1 requests; insert +3.6 % on config 5, +7 % on config 2 with the larger
          // document-frequency histogram of k_raw_append)
#pragma unroll
          for (int u = 0; u < 4; u++) {
            const uint2 pk = j[u] >= 0 ? __ldg(pi4 + j[u]) : make_uint2(0xffffffffu, 0xffffffffu);
            const uint32_t kk[4] = {pk.x & 0xffffu, pk.x >> 16, pk.y & 0xffffu, pk.y >> 16};
#pragma unroll
            for (int o = 0; o < 4; o++) k[u][o] = (j[u] >= 0 && o < h) ? (int)kk[o] : -1;
          }
        } else {
#pragma unroll
          for (int u = 0; u < 4; u++)
#pragma unroll
            for (int o = 0; o < 4; o++) k[u][o] = (j[u] >= 0 && o < h) ? (int)__ldg(pi + (int64_t)j[u] * h + o) : -1;
        }
#pragma unroll
        for (int u = 0; u < 4; u++)
#pragma unroll
          for (int o = 0; o < 4; o++)
            if (k[u][o] >= 0) {
              atomicMax(&su[k[u][o]], xo[u]);
              if (lower) atomicMin(&sl[k[u][o]], xo[u]);
            }
      } else {
#pragma unroll
        for (int u = 0; u < 4; u++)
          if (j[u] >= 0)
            for (int o = 0; o < h; o++) {
              const int k = pi[(int64_t)j[u] * h + o];
              atomicMax(&su[k], xo[u]);
              if (lower) atomicMin(&sl[k], xo[u]);
            }
      }
    }
    __syncwarp();
    if (VAL) {
      row_bad = __any_sync(0xffffffffu, row_bad);
      if (row_bad) err |= kErrRow;
      const bool ids_bad = (err_ids & (kErrLive | kErrDupId | kErrIdReserved)) != 0;
      if (row_bad || ids_bad || (int64_t)ids[r] >= cap) continue;
    }
    const int64_t col = (int64_t)ids[r] * m;
    for (int k = lane; k < m; k += 32) {
      if (BF) {
        Ub[col + k] = bf16_up_bits(ord2f(su[k]));
        if (lower) Lb[col + k] = bf16_down_bits(ord2f(sl[k]));
      } else {
        U[col + k] = ord2f(su[k]);
        if (lower) L[col + k] = ord2f(sl[k]);
      }
    }
    __syncwarp();
  }
  if (VAL) {
    err = __reduce_or_sync(0xffffffffu, err);
    maxid = __reduce_max_sync(0xffffffffu, maxid);
    unsorted = __reduce_or_sync(0xffffffffu, unsorted);
    if (lane == 0) {
      if (err) atomicOr(&info->err, err);
      atomicMax(&info->max_id, maxid);
      if (unsorted) atomicOr(&info->ids_unsorted, 1u);
    }
  }
}

// ---------------------------------------------------------------- postings build
// Tile-major inverted index: documents are grouped in tiles of 32 consecutive ids and tile t holds
// the entries (term << 5) | (id & 31) of its documents ordered by (id, term) — the inverted lists
// I[j] chunked by id range (as Roaring chunks ids), grouped per document inside a tile.
// keys[p] = (id << 32) | term for every entry of the batch (sorted when the batch ids are not
// ascending); with ascending ids the CSR order already is (id, term) and the entries are written
// straight to `direct`.  Per-tile entry counts.
__global__ void k_make_pairs(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                             const uint32_t* __restrict__ ids, int64_t nrows, uint64_t* __restrict__ keys,
                             uint32_t* __restrict__ direct, unsigned long long* __restrict__ tile_count) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t base = indptr[0];
  for (int64_t r = warp; r < nrows; r += nwarps) {
    const int64_t b = indptr[r], e = indptr[r + 1];
    const uint32_t id = ids[r];
    for (int64_t p = b + lane; p < e; p += 32) {
      const uint32_t j = (uint32_t)indices[p];
      if (keys) keys[p - base] = ((uint64_t)id << 32) | j;
      else direct[p - base] = (j << 5) | (id & 31u);
    }
    if (lane == 0 && e > b) atomicAdd(&tile_count[id >> 5], (unsigned long long)(e - b));
  }
}

// A batch whose ids do not ascend: its ROWS are sorted by id (keys (id << 32) | row), not its entries —
// each row's terms already ascend (validated), so the rows in id order, entries in row order, are the
// (id, term) order the tiles need.  rlen[i] = the i-th row's entries (scanned into its destination).
__global__ void k_row_keys(const int64_t* __restrict__ indptr, const uint32_t* __restrict__ ids, int64_t nrows,
                           uint64_t* __restrict__ keys, unsigned long long* __restrict__ tile_count) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t id = ids[r];
    keys[r] = ((uint64_t)id << 32) | (uint64_t)r;
    const int64_t len = indptr[r + 1] - indptr[r];
    if (len > 0) atomicAdd(&tile_count[id >> 5], (unsigned long long)len);
  }
}
__global__ void k_row_lens(const int64_t* __restrict__ indptr, const uint64_t* __restrict__ keys, int64_t nrows,
                           int64_t* __restrict__ rlen) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = (int64_t)(keys[i] & 0xffffffffu);
    rlen[i] = indptr[r + 1] - indptr[r];
  }
}
// warp per sorted row: its entries (term << 5) | (id & 31) at its destination
__global__ void k_row_place(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                            const uint64_t* __restrict__ keys, const int64_t* __restrict__ rdst, int64_t nrows,
                            uint32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < nrows; i += nwarps) {
    const uint64_t k = keys[i];
    const int64_t r = (int64_t)(k & 0xffffffffu);
    const uint32_t d = (uint32_t)(k >> 32) & 31u;
    const int64_t b = indptr[r], e = indptr[r + 1];
    uint32_t* o = out + rdst[i];
    for (int64_t p = b + lane; p < e; p += 32) o[p - b] = ((uint32_t)indices[p] << 5) | d;
  }
}

__global__ void k_fill_i64(int64_t* __restrict__ p, int64_t v, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void k_unpack_ids(const uint64_t* __restrict__ keys, int64_t nnz, uint32_t* __restrict__ out) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x)
    out[p] = ((uint32_t)keys[p] << 5) | ((uint32_t)(keys[p] >> 32) & 31u);
}

__global__ void k_add_i64(const int64_t* __restrict__ a, const int64_t* __restrict__ b, int64_t* __restrict__ out,
                          int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a[i] + b[i];
}

// (document, term) order of a tile entry (j << 5) | d  (j < 2^27)
__device__ __forceinline__ uint32_t rot(uint32_t e) { return ((e & 31u) << 27) | (e >> 5); }

// One block per tile: T'[t] = (T[t] without its tombstones) ∪ B[t] as one sorted list at new_off[t].
// A tile without tombstones merges as before: fresh ids (every new id above every old one) reduce to
// two coalesced copies; otherwise each entry goes to its document's new start + its rank inside the
// document (the kept and the batch documents are disjoint).  A tile with tombstones (entries of documents that are not live — deleted ids, including
// the old entries of ids this batch recycles) first stages its live entries in shared memory in order
// (block scan), then merges those; its dead documents' ecnt and its tdead are reset.
constexpr int kMergeStage = 12288;  // kept entries of a tile merged in shared memory (48 KB) ...
constexpr int kMergeBStage = 4096;  // ... plus the batch's entries of the tile (16 KB: a whole tile of config 4)

// COPY = true: the tiles the batch leaves alone (no batch entries, no tombstones) — plain coalesced
// copies, no shared memory (full occupancy).  COPY = false: the others — the tile's live entries and
// its batch entries are staged in shared memory (in order; a block scan drops tombstones) and every
// rank comes from a binary search in shared memory, not in global memory.
// Tiles have slack: tile t's region is [off[t], off[t+1]) and its first tsz[t]
// entries are in use.  With new_post == old_post (and new_off == old_off) the kernel merges IN PLACE
// (the slack layout's O(touched tiles) insert): every stored entry of a touched tile is staged in
// shared memory before the tile is written back, untouched tiles are not visited (COPY = false only).
template <bool COPY>
__global__ void __launch_bounds__(256) k_merge_postings(const int64_t* __restrict__ old_off,
                                                        const uint32_t* old_post,
                                                        const int64_t* __restrict__ batch_off,
                                                        const uint32_t* __restrict__ batch_post, int64_t n,
                                                        const int64_t* __restrict__ new_off,
                                                        uint32_t* new_post,
                                                        const uint8_t* __restrict__ live, int32_t* __restrict__ ecnt,
                                                        int32_t* __restrict__ tdead, int32_t* __restrict__ tsz,
                                                        int64_t stage_cap) {
  extern __shared__ uint32_t stage[];  // [stage_cap]: the merged tile
  __shared__ uint32_t sOc[32], sBc[32], sOs[32], sBs[32], sNs[32];
  __shared__ uint8_t sLv[32];
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
    const int64_t oo = old_off[j], ol = tsz[j];
    const int64_t bo = batch_off[j], bl = batch_off[j + 1] - bo;
    const int64_t no = new_off[j];
    const uint32_t* A = old_post + oo;
    const uint32_t* B = batch_post + bo;
    uint32_t* O = new_post + no;
    const int32_t dead = tdead[j];  // (uniform: read before any write of this tile below)
    const bool plain = dead == 0 && bl == 0;
    if (plain != COPY) continue;
    if (COPY) {
      for (int64_t t = threadIdx.x; t < ol; t += blockDim.x) O[t] = A[t];
      continue;
    }
    __syncthreads();  // (the previous tile's shared state is free)
    if (threadIdx.x < 32) {  // per document: stored entries (tombstones included), liveness
      const int64_t id = (j << 5) | threadIdx.x;
      sOc[threadIdx.x] = (uint32_t)ecnt[id];
      sLv[threadIdx.x] = live[id] != 0;
      sBc[threadIdx.x] = 0;
    }
    if (threadIdx.x == 0) {
      tdead[j] = 0;
      tsz[j] = (int32_t)(ol - dead + bl);  // (every thread read ol above; the next tile's read follows a barrier)
    }
    if (dead == 0 && (bl == 0 || ol == 0 || rot(A[ol - 1]) < rot(B[0]))) {  // fresh ids past the old ones
      if (O != A)
        for (int64_t t = threadIdx.x; t < ol; t += blockDim.x) O[t] = A[t];
      for (int64_t t = threadIdx.x; t < bl; t += blockDim.x) O[ol + t] = B[t];
      continue;
    }
    if (ol - dead + bl <= stage_cap) {
      // the merged tile in document order: the kept documents (live, not in the batch) and the batch's
      // documents are disjoint (batch ids are not live), each one's entries contiguous and in term
      // order in its source — so an entry's place is its document's new start + its rank inside the
      // document: per-document counts and starts (warp scans), then one placement pass into shared
      // memory (every read of the old tile before the barrier: safe in place) and one copy out
      __syncthreads();
      for (int64_t t0 = threadIdx.x; t0 < bl; t0 += 4 * (int64_t)blockDim.x) {
        uint32_t e[4];
#pragma unroll
        for (int u = 0; u < 4; u++) e[u] = t0 + u * (int64_t)blockDim.x < bl ? B[t0 + u * (int64_t)blockDim.x] : 0xffffffffu;
#pragma unroll
        for (int u = 0; u < 4; u++)
          if (e[u] != 0xffffffffu) atomicAdd(&sBc[e[u] & 31u], 1u);
      }
      __syncthreads();
      if (threadIdx.x < 32) {
        const uint32_t oc = sOc[threadIdx.x], bc = sBc[threadIdx.x], kc = sLv[threadIdx.x] ? oc : 0u;
        uint32_t io = oc, ib = bc, in = kc + bc;
#pragma unroll
        for (int dd = 1; dd < 32; dd <<= 1) {
          const uint32_t yo = __shfl_up_sync(0xffffffffu, io, dd), yb = __shfl_up_sync(0xffffffffu, ib, dd),
                         yn = __shfl_up_sync(0xffffffffu, in, dd);
          if ((int)threadIdx.x >= dd) {
            io += yo;
            ib += yb;
            in += yn;
          }
        }
        sOs[threadIdx.x] = io - oc;
        sBs[threadIdx.x] = ib - bc;
        sNs[threadIdx.x] = in - (kc + bc);
      }
      __syncthreads();
      // eight loads in flight per thread before their stores (a tile is ~4 K entries: latency-bound
      // otherwise)
      for (int64_t t0 = threadIdx.x; t0 < ol; t0 += 8 * (int64_t)blockDim.x) {
        uint32_t e[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
          const int64_t t = t0 + u * (int64_t)blockDim.x;
          e[u] = t < ol ? A[t] : 0xffffffffu;
        }
#pragma unroll
        for (int u = 0; u < 8; u++) {
          const int64_t t = t0 + u * (int64_t)blockDim.x;
          const uint32_t d = e[u] & 31u;
          if (t < ol && sLv[d]) stage[sNs[d] + (uint32_t)t - sOs[d]] = e[u];
        }
      }
      for (int64_t t0 = threadIdx.x; t0 < bl; t0 += 4 * (int64_t)blockDim.x) {
        uint32_t e[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int64_t t = t0 + u * (int64_t)blockDim.x;
          e[u] = t < bl ? B[t] : 0u;
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int64_t t = t0 + u * (int64_t)blockDim.x;
          const uint32_t d = e[u] & 31u;
          if (t < bl) stage[sNs[d] + (uint32_t)t - sBs[d]] = e[u];
        }
      }
      __syncthreads();
      const int64_t total = ol - dead + bl;
      for (int64_t t = threadIdx.x; t < total; t += blockDim.x) O[t] = stage[t];
    } else if (threadIdx.x == 0) {  // an oversized tile (a full merge only, never in place): sequential
      int64_t a = 0, b = 0, o = 0;
      while (a < ol || b < bl) {
        if (a < ol && !live[(j << 5) | (A[a] & 31u)]) {
          a++;
          continue;
        }
        if (b >= bl || (a < ol && rot(A[a]) < rot(B[b]))) O[o++] = A[a++];
        else O[o++] = B[b++];
      }
    }
    __syncthreads();
    if (threadIdx.x < 32 && !sLv[threadIdx.x]) ecnt[(j << 5) | threadIdx.x] = 0;  // tombstones dropped
  }
}

// slack of a tile region holding s entries: an eighth + 32, so that the next rounds of a stream
// (recycled ids replacing deleted ones: sizes drift by a few documents) merge in place
__host__ __device__ inline int64_t tile_slack(int64_t s) { return (s >> 3) + 32; }
// region of a tile holding s entries of `docs` documents: s + slack, scaled to 32 documents when the tile
// is the partly filled last one (the next fresh ids fill it in place)
__host__ __device__ inline int64_t tile_region(int64_t s, int docs) {
  const int64_t r = s + tile_slack(s);
  return docs > 0 && docs < 32 ? r * 32 / docs : r;
}

// new tile regions of a full merge: stored entries - tombstones + the batch's entries, plus slack for
// the tiles below t_end (tiles at or beyond it hold nothing and get no region)
__global__ void k_merge_sizes(const int32_t* __restrict__ tsz, const int32_t* __restrict__ tdead,
                              const unsigned long long* __restrict__ tcount, int64_t n, int64_t t_end,
                              int32_t last_docs, int64_t* __restrict__ sizes) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t sz = (int64_t)tsz[t] - tdead[t] + (int64_t)tcount[t];
    sizes[t] = t < t_end ? tile_region(sz, t == t_end - 1 ? last_docs : 32) : sz;
  }
}

// can the batch merge in place?  A touched tile (batch entries or tombstones) below t_new must fit
// its region and the shared-memory stage; tiles from t_new on have no region yet: their new region
// sizes (entries + slack) go to newcap[t - t_new] (0 for tiles without batch entries)
__global__ void k_merge_fit(const int64_t* __restrict__ off, const int32_t* __restrict__ tsz,
                            const int32_t* __restrict__ tdead, const unsigned long long* __restrict__ tcount,
                            int64_t n, int64_t t_new, int64_t t_last, int32_t last_docs, uint32_t* __restrict__ misfit,
                            int64_t* __restrict__ newcap) {
  // misfit[0]: some touched tile does not fit; misfit[1]: the most entries a touched tile will hold
  // (the merge's shared-memory stage is sized to it: small tiles, more blocks per SM)
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t bl = (int64_t)tcount[t], live_old = (int64_t)tsz[t] - tdead[t];
    const int64_t sz = live_old + bl;
    if (t < t_new) {
      const bool touched = bl > 0 || tdead[t] > 0;
      if (touched) {
        if (sz > off[t + 1] - off[t] || sz > kMergeStage + kMergeBStage) misfit[0] = 1u;
        atomicMax(&misfit[1], sz < 0x7fffffff ? (uint32_t)sz : 0x7fffffffu);
      }
    } else {
      if (tsz[t] != 0) *misfit = 1u;  // (no region beyond t_new holds entries)
      newcap[t - t_new] = bl > 0 ? tile_region(sz, t == t_last - 1 ? last_docs : 32) : 0;
    }
  }
}

// regions of the new tiles [t_new, n): off[t] = base + scan[t - t_new]
__global__ void k_new_regions(int64_t* __restrict__ off, int64_t t_new, int64_t n, int64_t base,
                              const int64_t* __restrict__ scan) {
  for (int64_t t = t_new + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t <= n; t += (int64_t)gridDim.x * blockDim.x)
    off[t] = base + scan[t - t_new];
}

// bulk append: the new tiles' entries in use
__global__ void k_tsz_add(int32_t* __restrict__ tsz, const unsigned long long* __restrict__ tcount, int64_t n) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    tsz[t] += (int32_t)tcount[t];
}

// ---------------------------------------------------------------- document frequencies
// df[j] += entries of term j in the batch.  Terms < 16,384 (the Zipf head of the skewed configs)
// are first counted in a shared-memory histogram per block, so hot terms see one global atomic
// per block instead of one per entry.
constexpr int kDfSmem = 49152;  // (192 KB of dynamic shared memory, one 1,024-thread block per SM: the terms below it take no global atomic per entry — config 5: 88 % of the entries instead of 66 % with 16 K)
__global__ void k_df_add(const int32_t* __restrict__ indices, int64_t nnz, int32_t n, int32_t* __restrict__ df) {
  extern __shared__ int32_t hs[];
  for (int t = threadIdx.x; t < kDfSmem; t += blockDim.x) hs[t] = 0;
  __syncthreads();
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t j = indices[p];
    if (j < kDfSmem) atomicAdd(&hs[j], 1);
    else atomicAdd(&df[j], 1);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < kDfSmem && t < n; t += blockDim.x)
    if (hs[t]) atomicAdd(&df[t], hs[t]);
}

__global__ void k_df_max(const int32_t* __restrict__ df, int32_t n, int64_t* __restrict__ out) {
  int32_t mx = 0;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    mx = max(mx, df[j]);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0 && mx > 0) atomicMax(reinterpret_cast<unsigned long long*>(out), (unsigned long long)mx);
}

// ---------------------------------------------------------------- raw-vector store append
// (the batch's document frequencies are counted in the same pass: df[j] += 1 per entry, terms below
// kDfSmem in a shared-memory histogram per block — the Zipf head sees one global atomic per block)
__global__ void k_raw_append(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                             const float* __restrict__ values, const uint32_t* __restrict__ ids, int64_t nrows,
                             int64_t pool_base, int32_t* __restrict__ raw_idx, float* __restrict__ raw_val,
                             int64_t* __restrict__ raw_off, int32_t* __restrict__ raw_nnz,
                             uint8_t* __restrict__ live, int32_t* __restrict__ ecnt, int32_t n, int32_t* __restrict__ df) {
  extern __shared__ int32_t hs[];
  for (int t = threadIdx.x; t < kDfSmem; t += blockDim.x) hs[t] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t base = indptr[0];
  for (int64_t r = warp; r < nrows; r += nwarps) {
    const int64_t b = indptr[r], e = indptr[r + 1];
    const int64_t dst = pool_base + (b - base);
    // four entries per lane in flight: the copy is latency-bound at one load pair per iteration
    for (int64_t p0 = b + lane; p0 < e; p0 += 128) {
      int32_t j[4];
      float x[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int64_t p = p0 + 32 * u;
        j[u] = p < e ? __ldg(indices + p) : -1;
        x[u] = p < e ? __ldg(values + p) : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int64_t p = p0 + 32 * u;
        if (p < e) {
          raw_idx[dst + (p - b)] = j[u];
          raw_val[dst + (p - b)] = x[u] == 0.0f ? 0.0f : x[u];
          if (j[u] < kDfSmem) atomicAdd(&hs[j[u]], 1);
          else atomicAdd(&df[j[u]], 1);
        }
      }
    }
    if (lane == 0) {
      const uint32_t id = ids[r];
      raw_off[id] = dst;
      raw_nnz[id] = (int32_t)(e - b);
      ecnt[id] = (int32_t)(e - b);  // its entries in its tile (inserted by this batch's merge / append)
      live[id] = 1;
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < kDfSmem && t < n; t += blockDim.x)
    if (hs[t]) atomicAdd(&df[t], hs[t]);
}

// raw-store compaction (the store is append-only between compactions: a deleted row keeps its
// entries until then): per-id live entry counts, then a warp per live id copies its row to the
// exclusive-scan offset in the new pool
__global__ void k_raw_counts(const int32_t* __restrict__ raw_nnz, const uint8_t* __restrict__ live, int64_t cap,
                             uint32_t* __restrict__ cnt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += (int64_t)gridDim.x * blockDim.x)
    cnt[i] = live[i] ? (uint32_t)raw_nnz[i] : 0u;
}

__global__ void k_raw_compact(const uint32_t* __restrict__ new_off, const uint8_t* __restrict__ live, int64_t cap,
                              const int32_t* __restrict__ raw_nnz, int64_t* __restrict__ raw_off,
                              const int32_t* __restrict__ old_idx, const float* __restrict__ old_val,
                              int32_t* __restrict__ new_idx, float* __restrict__ new_val) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < cap; i += nwarps) {
    if (!live[i]) continue;
    const int64_t src = raw_off[i], dst = new_off[i];
    const int32_t c = raw_nnz[i];
    for (int32_t p = lane; p < c; p += 32) {
      new_idx[dst + p] = old_idx[src + p];
      new_val[dst + p] = old_val[src + p];
    }
    __syncwarp();
    if (lane == 0) raw_off[i] = dst;
  }
}

}  // namespace

void launch_raw_compact(const int32_t* raw_nnz, const uint8_t* live, int64_t cap, int64_t* raw_off,
                        const int32_t* old_idx, const float* old_val, int32_t* new_idx, float* new_val,
                        uint32_t* cnt, uint32_t* scan_tmp, cudaStream_t s) {
  if (cap <= 0) return;
  k_raw_counts<<<grid_for(cap, 256), 256, 0, s>>>(raw_nnz, live, cap, cnt);
  exclusive_scan_u32(cnt, cnt, cap, scan_tmp, s);
  k_raw_compact<<<grid_for(cap * 32, 256), 256, 0, s>>>(cnt, live, cap, raw_nnz, raw_off, old_idx, old_val, new_idx,
                                                        new_val);
}

void launch_validate_rows(const int64_t* indptr, const int32_t* indices, const float* values, const uint32_t* ids,
                          int64_t nrows, int32_t n, bool upper_only, DevInfo* info, cudaStream_t s) {
  k_validate_rows<<<grid_for(nrows * 32, 256), 256, 0, s>>>(indptr, indices, values, ids, nrows, n, upper_only ? 1 : 0,
                                                           info);
}

void launch_check_ids(const uint32_t* ids, int64_t nrows, const uint8_t* live, uint32_t* stamp, uint32_t epoch,
                      bool want_live, int64_t cap, DevInfo* info, cudaStream_t s) {
  k_check_ids<<<grid_for(nrows, 256), 256, 0, s>>>(ids, nrows, live, stamp, epoch, want_live ? 1 : 0, cap, info);
}

void launch_sketch_build(const int64_t* indptr, const int32_t* indices, const float* values, const uint32_t* ids,
                         int64_t nrows, const uint16_t* pi, int32_t m, int32_t h, void* U, void* L, bool bf16,
                         cudaStream_t s, bool validate, int32_t n, bool upper_only, int64_t cap, DevInfo* info,
                         const uint2* pi4) {
  // warps per block bounded by shared memory (2*m ints per warp)
  int wpb = (int)(96 * 1024 / (8 * (size_t)m));
  if (wpb > 8) wpb = 8;
  if (wpb < 1) wpb = 1;
  size_t smem = (size_t)wpb * 2 * m * sizeof(int);
  int64_t blocks = (nrows + wpb - 1) / wpb;
  // all blocks resident at once (a warp then folds ~10 documents of a 100 K batch: its start-up — flag
  // word, first indptr — is paid once, not per document)
  if (blocks > (int64_t)sm_count() * 8) blocks = (int64_t)sm_count() * 8;
  if (blocks < 1) blocks = 1;
  auto go = [&](auto kern) {
    smem_optin((const void*)kern);
    kern<<<(unsigned)blocks, wpb * 32, smem, s>>>(indptr, indices, values, ids, nrows, pi, m, h, U, L, n,
                                                   upper_only ? 1 : 0, cap, info, h <= 4 ? pi4 : nullptr);
  };
  if (bf16) {
    if (validate) go(k_sketch_build<true, true>); else go(k_sketch_build<true, false>);
  } else {
    if (validate) go(k_sketch_build<false, true>); else go(k_sketch_build<false, false>);
  }
}

void launch_make_pairs(const int64_t* indptr, const int32_t* indices, const uint32_t* ids, int64_t nrows,
                       uint64_t* keys, uint32_t* direct, unsigned long long* tile_count, cudaStream_t s) {
  k_make_pairs<<<grid_for(nrows * 32, 256), 256, 0, s>>>(indptr, indices, ids, nrows, keys, direct, tile_count);
}

void fill_i64(int64_t* p, int64_t v, int64_t n, cudaStream_t s) {
  if (n > 0) k_fill_i64<<<grid_for(n, 256), 256, 0, s>>>(p, v, n);
}

void launch_row_sorted_batch(const int64_t* indptr, const int32_t* indices, const uint32_t* ids, int64_t nrows,
                             int hi_bit, uint64_t* keys, uint64_t* keys_tmp, uint32_t* hist, uint32_t* scan_tmp,
                             int64_t* rlen, int64_t* rdst, uint32_t* out, unsigned long long* tile_count, cudaStream_t s) {
  k_row_keys<<<grid_for(nrows, 256), 256, 0, s>>>(indptr, ids, nrows, keys, tile_count);
  radix_sort_u64(keys, keys_tmp, nrows, 32, hi_bit, hist, scan_tmp, s);
  k_row_lens<<<grid_for(nrows, 256), 256, 0, s>>>(indptr, keys, nrows, rlen);
  exclusive_scan_i64_small(rlen, rdst, nrows, s);
  k_row_place<<<grid_for(nrows * 32, 256), 256, 0, s>>>(indptr, indices, keys, rdst, nrows, out);
}

void launch_unpack_ids(const uint64_t* keys, int64_t nnz, uint32_t* ids_out, cudaStream_t s) {
  if (nnz > 0) k_unpack_ids<<<grid_for(nnz, 256), 256, 0, s>>>(keys, nnz, ids_out);
}

void launch_merge_postings(const int64_t* old_off, const uint32_t* old_post, const int64_t* batch_off,
                           const uint32_t* batch_post, int64_t n, int64_t* new_off, uint32_t* new_post,
                           const uint8_t* live, int32_t* ecnt, int32_t* tdead, int32_t* tsz, cudaStream_t s,
                           int64_t stage_entries) {
  int64_t blocks = std::min<int64_t>(n, (int64_t)sm_count() * 64);
  if (blocks < 1) blocks = 1;
  smem_optin((const void*)k_merge_postings<false>);
  const int64_t cap = stage_entries > 0 ? std::min<int64_t>(((stage_entries + 1023) / 1024) * 1024,
                                                           kMergeStage + kMergeBStage)
                                        : kMergeStage + kMergeBStage;
  if (new_post != old_post)  // a full merge copies the untouched tiles; in place they stay where they are
    k_merge_postings<true><<<(unsigned)blocks, 256, 0, s>>>(old_off, old_post, batch_off, batch_post, n, new_off,
                                                            new_post, live, ecnt, tdead, tsz, 0);
  k_merge_postings<false><<<(unsigned)blocks, 256, sizeof(uint32_t) * (size_t)cap, s>>>(
      old_off, old_post, batch_off, batch_post, n, new_off, new_post, live, ecnt, tdead, tsz, cap);
}

void launch_merge_fit(const int64_t* off, const int32_t* tsz, const int32_t* tdead, const unsigned long long* tcount,
                      int64_t n, int64_t t_new, int64_t t_last, int32_t last_docs, uint32_t* misfit, int64_t* newcap,
                      int64_t* newscan, cudaStream_t s) {
  cudaMemsetAsync(misfit, 0, 2 * sizeof(uint32_t), s);
  k_merge_fit<<<grid_for(n, 256), 256, 0, s>>>(off, tsz, tdead, tcount, n, t_new, t_last, last_docs, misfit, newcap);
  exclusive_scan_i64_small(newcap, newscan, n - t_new, s);  // newscan[n - t_new] = the new regions' total
}

void launch_new_regions(int64_t* off, int64_t t_new, int64_t n, int64_t base, const int64_t* newscan, cudaStream_t s) {
  k_new_regions<<<grid_for(n - t_new + 1, 256), 256, 0, s>>>(off, t_new, n, base, newscan);
}

void launch_tsz_add(int32_t* tsz, const unsigned long long* tcount, int64_t n, cudaStream_t s) {
  k_tsz_add<<<grid_for(n, 256), 256, 0, s>>>(tsz, tcount, n);
}

void launch_raw_append(const int64_t* indptr, const int32_t* indices, const float* values, const uint32_t* ids,
                       int64_t nrows, int64_t pool_base, int32_t* raw_idx, float* raw_val, int64_t* raw_off,
                       int32_t* raw_nnz, uint8_t* live, int32_t* ecnt, int32_t n, int32_t* df, cudaStream_t s) {
  smem_optin((const void*)k_raw_append);
  k_raw_append<<<grid_for(nrows * 32, 1024, (int64_t)sm_count()), 1024, sizeof(int32_t) * kDfSmem, s>>>(
      indptr, indices, values, ids, nrows, pool_base, raw_idx, raw_val, raw_off, raw_nnz, live, ecnt, n, df);
}

void launch_merge_sizes(const int32_t* tsz, const int32_t* tdead, const unsigned long long* tcount, int64_t n,
                        int64_t t_end, int32_t last_docs, int64_t* sizes, cudaStream_t s) {
  k_merge_sizes<<<grid_for(n, 256), 256, 0, s>>>(tsz, tdead, tcount, n, t_end, last_docs, sizes);
}

void launch_df_add(const int32_t* indices, int64_t nnz, int32_t n, int32_t* df, cudaStream_t s) {
  smem_optin((const void*)k_df_add);
  if (nnz > 0)
    k_df_add<<<grid_for(nnz, 1024, (int64_t)sm_count()), 1024, sizeof(int32_t) * kDfSmem, s>>>(indices, nnz, n, df);
}

void launch_df_max(const int32_t* df, int32_t n, int64_t* out, cudaStream_t s) {
  cudaMemsetAsync(out, 0, sizeof(int64_t), s);
  k_df_max<<<grid_for(n, 256, (int64_t)sm_count() * 4), 256, 0, s>>>(df, n, out);
}

void launch_add_i64(const int64_t* a, const int64_t* b, int64_t* out, int64_t n, cudaStream_t s) {
  k_add_i64<<<grid_for(n, 256), 256, 0, s>>>(a, b, out, n);
}

}  // namespace sinn
