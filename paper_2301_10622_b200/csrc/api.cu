// api.cu — the C ABI (include/sinn.h) and the host-side index manager: argument checks,
// stream-ordered validation round trips, geometric capacity growth, buffer swaps.
// All arithmetic of the method runs in the kernels of k_insert.cu / k_delete.cu / k_search.cu.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "sinn_internal.cuh"

using sinn::DevInfo;

namespace {

const char* kVersion = "sinn-b200 0.1 sm_100a";

struct Fail {
  sinn_status st;
};

// record an error; CUDA errors poison the handle
sinn_status fail(sinn_index* x, sinn_status st, const std::string& msg) {
  if (x) {
    x->last_error = msg;
    if (st == SINN_ECUDA) x->poisoned = true;
  }
  // a failed allocation also sets the runtime's last error: clear it, or the next call's launch
  // check (cudaGetLastError) would report this stale error and poison a healthy handle
  if (st == SINN_ENOMEM) (void)cudaGetLastError();
  return st;
}

#define CU(call)                                                                                        \
  do {                                                                                                  \
    cudaError_t e_ = (call);                                                                            \
    if (e_ != cudaSuccess) {                                                                            \
      return fail(x, e_ == cudaErrorMemoryAllocation ? SINN_ENOMEM : SINN_ECUDA,                       \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                                  \
    }                                                                                                   \
  } while (0)

#define GUARD(x)                                                                                        \
  do {                                                                                                  \
    if (!(x)) return SINN_EINVAL;                                                                       \
    if ((x)->poisoned) return SINN_EPOISONED;                                                           \
  } while (0)

// Index arrays and workspaces come from the device's stream-ordered pool (cudaMallocAsync /
// cudaFreeAsync on the call's stream): growing a buffer is allocate + copy + free in stream order,
// with no device-wide synchronisation; the pool keeps freed memory for reuse.
template <typename T>
cudaError_t grow_copy(T** p, int64_t old_n, int64_t new_n, cudaStream_t s) {
  T* q = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&q, sizeof(T) * (size_t)std::max<int64_t>(new_n, 1), s);
  if (e != cudaSuccess) return e;
  if (getenv("SINN_POISON")) cudaMemsetAsync(q, 0xA5, sizeof(T) * (size_t)std::max<int64_t>(new_n, 1), s);
  if (*p && old_n > 0) {
    e = cudaMemcpyAsync(q, *p, sizeof(T) * (size_t)old_n, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return e;
  }
  if (*p) {
    e = cudaFreeAsync(*p, s);
    if (e != cudaSuccess) return e;
  }
  *p = q;
  return cudaSuccess;
}

void keep_pool_memory() {  // freed pool memory stays reserved for the next growth (no OS round trip)
  static bool done[256] = {};  // per device: the default pool is a per-device object
  int dev = 0;
  cudaMemPool_t pool;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 256 || done[dev]) return;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev] = true;
}

// sketch-column capacity >= need (U, L, live, stamp, raw_off, raw_nnz)
sinn_status ensure_cap(sinn_index* x, int64_t need, cudaStream_t s) {
  if (need <= x->cap) return SINN_OK;
  int64_t c = std::max<int64_t>({need, x->cap + x->cap / 2, 1024});
  c = ((c + 31) / 32) * 32;
  const int64_t old = x->cap, m = x->m;
  if (x->bf16) {
    CU(grow_copy(&x->Ub, old * m, c * m, s));
    if (!x->upper_only) CU(grow_copy(&x->Lb, old * m, c * m, s));
  } else {
    CU(grow_copy(&x->U, old * m, c * m, s));
    if (!x->upper_only) CU(grow_copy(&x->L, old * m, c * m, s));
  }
  CU(grow_copy(&x->live, old, c, s));
  CU(grow_copy(&x->ecnt, old, c, s));
  CU(grow_copy(&x->tdead, old / 32, c / 32, s));
  CU(grow_copy(&x->tsz, old / 32, c / 32, s));
  CU(grow_copy(&x->stamp, old, c, s));
  CU(grow_copy(&x->raw_off, old, c, s));
  CU(grow_copy(&x->raw_nnz, old, c, s));
  if (x->bf16) {  // -inf / +inf in bfloat16
    sinn::fill_u16(x->Ub + old * m, 0xff80u, (c - old) * m, s);
    if (!x->upper_only) sinn::fill_u16(x->Lb + old * m, 0x7f80u, (c - old) * m, s);
  } else {
    sinn::fill_f32(x->U + old * m, -INFINITY, (c - old) * m, s);
    if (!x->upper_only) sinn::fill_f32(x->L + old * m, INFINITY, (c - old) * m, s);
  }
  CU(cudaMemsetAsync(x->live + old, 0, (size_t)(c - old), s));
  CU(cudaMemsetAsync(x->ecnt + old, 0, sizeof(int32_t) * (size_t)(c - old), s));
  CU(cudaMemsetAsync(x->tdead + old / 32, 0, sizeof(int32_t) * (size_t)(c / 32 - old / 32), s));
  CU(cudaMemsetAsync(x->tsz + old / 32, 0, sizeof(int32_t) * (size_t)(c / 32 - old / 32), s));
  CU(cudaMemsetAsync(x->stamp + old, 0, sizeof(uint32_t) * (size_t)(c - old), s));
  CU(cudaMemsetAsync(x->raw_nnz + old, 0, sizeof(int32_t) * (size_t)(c - old), s));
  CU(cudaMemsetAsync(x->raw_off + old, 0, sizeof(int64_t) * (size_t)(c - old), s));
  if (x->containers) {  // container slots of the new tiles: none in use
    CU(grow_copy(&x->cont, old, c, s));
    CU(grow_copy(&x->cnum, old / 32, c / 32, s));
    CU(cudaMemsetAsync(x->cnum + old / 32, 0, (size_t)(c / 32 - old / 32), s));
  }
  // tile offsets of the inverted index: new (empty) tiles start at the current end
  CU(grow_copy(&x->off, old / 32 + 1, c / 32 + 1, s));
  CU(grow_copy(&x->off_alt, 0, c / 32 + 1, s));
  sinn::fill_i64(x->off + old / 32 + 1, x->post_len, c / 32 - old / 32, s);
  x->cap = c;
  return SINN_OK;
}

// raw-store capacity >= raw_used + add.  The store is append-only between compactions (a deleted
// row keeps its entries, a re-inserted id appends a new row); when it must grow while a quarter or
// more of it is dead, the live rows are first compacted into a fresh pool (k_raw_compact), which
// reclaims the dead entries and usually makes the growth unnecessary.
sinn_status ensure_raw(sinn_index* x, int64_t add, cudaStream_t s) {
  const int64_t need = x->raw_used + add;
  if (need <= x->raw_cap) return SINN_OK;
  // the live documents' raw entries (a device sum: the stored postings have slack and containers,
  // so they do not count them; growth is rare, so this round trip is too)
  int64_t* d_sum = reinterpret_cast<int64_t*>(x->d_info + 2);  // (the max-df scratch: not in use here)
  sinn::launch_sum_i32(x->raw_nnz, x->live, x->cap, d_sum, s);
  CU(cudaMemcpyAsync(x->h_i64 + 6, d_sum, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  const int64_t live_entries = x->h_i64[6];
  if (x->raw_used - live_entries >= x->raw_used / 4 && live_entries < ((int64_t)1 << 32) && x->cap > 0) {
    const int64_t c = std::max<int64_t>({live_entries + add, x->raw_cap, 1 << 16});
    int32_t* nidx = nullptr;
    float* nval = nullptr;
    uint32_t* cnt = nullptr;
    uint32_t* tmp = nullptr;
    CU(cudaMallocAsync((void**)&nidx, sizeof(int32_t) * (size_t)c, s));
    CU(cudaMallocAsync((void**)&nval, sizeof(float) * (size_t)c, s));
    CU(cudaMallocAsync((void**)&cnt, sizeof(uint32_t) * (size_t)x->cap, s));
    CU(cudaMallocAsync((void**)&tmp, sizeof(uint32_t) * sinn::exclusive_scan_u32_tmp_elems(x->cap), s));
    sinn::launch_raw_compact(x->raw_nnz, x->live, x->cap, x->raw_off, x->raw_idx, x->raw_val, nidx, nval, cnt, tmp,
                             s);
    CU(cudaGetLastError());
    CU(cudaFreeAsync(x->raw_idx, s));
    CU(cudaFreeAsync(x->raw_val, s));
    CU(cudaFreeAsync(cnt, s));
    CU(cudaFreeAsync(tmp, s));
    x->raw_idx = nidx;
    x->raw_val = nval;
    x->raw_cap = c;
    x->raw_used = live_entries;
    return SINN_OK;
  }
  int64_t c = std::max<int64_t>({need, x->raw_cap + x->raw_cap / 2, 1 << 16});
  CU(grow_copy(&x->raw_idx, x->raw_used, c, s));
  CU(grow_copy(&x->raw_val, x->raw_used, c, s));
  x->raw_cap = c;
  return SINN_OK;
}

sinn_status ensure_post(sinn_index* x, int64_t need, cudaStream_t s) {
  if (need <= x->post_cap) return SINN_OK;
  int64_t c = std::max<int64_t>({need, x->post_cap + x->post_cap / 2, 1 << 16});
  CU(grow_copy(&x->post, x->post_len, c, s));
  CU(grow_copy(&x->post_alt, 0, c, s));
  x->post_cap = c;
  return SINN_OK;
}

sinn_status ensure_ws2(sinn_index* x, size_t bytes, cudaStream_t s) {
  if (bytes <= x->ws2_bytes) return SINN_OK;
  // 25 % headroom: batches of one size vary a few percent in entries, and a regrowth (new pool
  // memory) inside a streaming insert costs tens of milliseconds
  bytes = std::max(bytes + bytes / 4, x->ws2_bytes + x->ws2_bytes / 2);
  if (x->ws2) CU(cudaFreeAsync(x->ws2, s));
  x->ws2 = nullptr;
  x->ws2_bytes = 0;
  CU(cudaMallocAsync(&x->ws2, bytes, s));
  x->ws2_bytes = bytes;
  return SINN_OK;
}

sinn_status ensure_stage(sinn_index* x, size_t bytes) {
  if (bytes <= x->dstage_bytes) return SINN_OK;
  if (x->dstage) cudaFree(x->dstage);
  if (x->hstage) cudaFreeHost(x->hstage);
  x->dstage = x->hstage = nullptr;
  x->dstage_bytes = x->hstage_bytes = 0;
  size_t b = std::max<size_t>(bytes, 1 << 20);
  CU(cudaMalloc(&x->dstage, b));
  CU(cudaMallocHost(&x->hstage, b));
  x->dstage_bytes = x->hstage_bytes = b;
  return SINN_OK;
}

inline size_t a256(size_t b) { return ((b + 255) / 256) * 256; }

int bits_for(uint64_t v) {
  int b = 0;
  while (v) {
    b++;
    v >>= 1;
  }
  return b;
}

sinn_status read_info(sinn_index* x, DevInfo* d, cudaStream_t s) {
  CU(cudaMemcpyAsync(x->h_info, d, sizeof(DevInfo), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  return SINN_OK;
}

}  // namespace

namespace sinn {

NvtxScope::NvtxScope(const char* name) { nvtxRangePushA(name); }
NvtxScope::~NvtxScope() { nvtxRangePop(); }

static const char* const kPhaseName[SINN_NUM_PHASES] = {
    "sinn:threshold", "sinn:score", "sinn:select", "sinn:rerank", "sinn:final", "sinn:validate",
    "sinn:sketch",    "sinn:postings", "sinn:raw", "sinn:delete", "sinn:prep"};

PhaseScope::PhaseScope(sinn_index* x_, int ph_, cudaStream_t s_) : x(x_), ph(ph_), s(s_) {
  nvtxRangePushA(ph_ >= 0 && ph_ < SINN_NUM_PHASES && kPhaseName[ph_] ? kPhaseName[ph_] : "sinn:phase");
  if (!x->prof) return;
  if (x->ev_used + 2 > x->ev_pool.size()) {
    for (int t = 0; t < 64; t++) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return;
      x->ev_pool.push_back(e);
    }
  }
  cudaEventRecord(x->ev_pool[x->ev_used], s);
}

PhaseScope::~PhaseScope() {
  nvtxRangePop();
  if (!x->prof || x->ev_used + 2 > x->ev_pool.size()) return;
  cudaEventRecord(x->ev_pool[x->ev_used + 1], s);
  x->ev_used += 2;
  x->ev_phase.push_back(ph);
  x->prof_calls[ph]++;
}

}  // namespace sinn

extern "C" {

const char* sinn_version(void) { return kVersion; }

sinn_status sinn_create(int32_t n, int32_t m, int32_t h, const int32_t* hash_table, uint32_t flags, void* stream,
                        sinn_index** out) {
  sinn::NvtxScope nvtx_("sinn_create");
  if (!out) return SINN_EINVAL;
  *out = nullptr;
  if (n < 1 || n > SINN_MAX_N || m < 1 || m > SINN_MAX_M || h < 1 || h > SINN_MAX_H || !hash_table) return SINN_EINVAL;
  if ((flags & ~(SINN_UPPER_ONLY | SINN_SKETCH_BF16 | SINN_BITMAP_CONTAINERS)) != 0) return SINN_EINVAL;
  if ((flags & SINN_SKETCH_BF16) && (m % 8) != 0) return SINN_EINVAL;  // 16-byte column copies
  for (int64_t t = 0; t < (int64_t)n * h; t++)
    if (hash_table[t] < 0 || hash_table[t] >= m) return SINN_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  keep_pool_memory();
  sinn_index* x = new sinn_index();
  x->n = n;
  x->m = m;
  x->h = h;
  x->flags = flags;
  x->upper_only = (flags & SINN_UPPER_ONLY) != 0;
  x->bf16 = (flags & SINN_SKETCH_BF16) != 0;
  x->containers = (flags & SINN_BITMAP_CONTAINERS) != 0;
  auto bail = [&](sinn_status st) {
    sinn_destroy(x);
    return st;
  };
  // pi: u16[n*h]; for h <= 4 followed (8-byte aligned) by the same maps padded to four u16 per term
  const size_t b_pi = ((sizeof(uint16_t) * (size_t)n * h + 7) / 8) * 8;
  const size_t b_pi4 = h <= 4 ? sizeof(uint16_t) * 4 * (size_t)n : 0;
  uint16_t* packed = (uint16_t*)malloc(b_pi + b_pi4);
  for (int64_t t = 0; t < (int64_t)n * h; t++) packed[t] = (uint16_t)hash_table[t];
  if (b_pi4) {
    uint16_t* p4 = packed + b_pi / sizeof(uint16_t);
    for (int64_t j = 0; j < n; j++)
      for (int o = 0; o < 4; o++) p4[4 * j + o] = o < h ? (uint16_t)hash_table[j * h + o] : (uint16_t)0xffff;
  }
  cudaError_t e = cudaMalloc(&x->pi, b_pi + b_pi4);
  if (e == cudaSuccess) e = cudaMemcpyAsync(x->pi, packed, b_pi + b_pi4, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  free(packed);
  if (e == cudaSuccess && b_pi4) x->pi4 = reinterpret_cast<uint2*>(reinterpret_cast<char*>(x->pi) + b_pi);
  if (e == cudaSuccess) e = cudaMalloc(&x->df, sizeof(int32_t) * (size_t)n);
  if (e == cudaSuccess) e = cudaMemsetAsync(x->df, 0, sizeof(int32_t) * (size_t)n, s);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&x->off, sizeof(int64_t), s);  // grown in stream order
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&x->off_alt, sizeof(int64_t), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(x->off, 0, sizeof(int64_t), s);
  // d_info: [0] insert/delete validation, [1] search validation, then two int64: max df scratch and
  // the index's dead (tombstoned) entries
  if (e == cudaSuccess) e = cudaMalloc(&x->d_info, 2 * sizeof(DevInfo) + 2 * sizeof(int64_t));
  if (e == cudaSuccess) e = cudaMemsetAsync(x->d_info, 0, 2 * sizeof(DevInfo) + 2 * sizeof(int64_t), s);
  if (e == cudaSuccess) e = cudaMalloc(&x->d_cstat, 4 * sizeof(int64_t));  // [3]: stats scratch
  if (e == cudaSuccess) e = cudaMemsetAsync(x->d_cstat, 0, 4 * sizeof(int64_t), s);
  if (x->containers) {
    if (e == cudaSuccess) e = cudaMalloc(&x->ccand, sizeof(int32_t) * (size_t)(sinn::cont_cand_cap() + 1));
    if (e == cudaSuccess) e = cudaMemsetAsync(x->ccand, 0, sizeof(int32_t) * (size_t)(sinn::cont_cand_cap() + 1), s);
    if (e == cudaSuccess) e = cudaMalloc(&x->cslot, (size_t)n);
    if (e == cudaSuccess) e = cudaMemsetAsync(x->cslot, 0xff, (size_t)n, s);
  }
  if (e == cudaSuccess) e = cudaMallocHost(&x->h_info, sizeof(DevInfo));
  if (e == cudaSuccess) e = cudaMallocHost(&x->h_i64, 8 * sizeof(int64_t));
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return bail(e == cudaErrorMemoryAllocation ? SINN_ENOMEM : SINN_ECUDA);
  x->d_sinfo = x->d_info + 1;
  x->d_dead = reinterpret_cast<int64_t*>(x->d_info + 2) + 1;
  *out = x;
  return SINN_OK;
}

sinn_status sinn_destroy(sinn_index* x) {
  sinn::NvtxScope nvtx_("sinn_destroy");
  if (!x) return SINN_OK;
  cudaDeviceSynchronize();
  for (cudaEvent_t e : x->ev_pool) cudaEventDestroy(e);
  if (x->df_ready) cudaEventDestroy(x->df_ready);
  // stream-ordered pool allocations go back with cudaFreeAsync, the rest with cudaFree
  void* pooled[] = {x->U, x->L, x->Ub, x->Lb, x->live, x->ecnt, x->tdead, x->stamp, x->raw_off, x->raw_nnz, x->raw_idx, x->raw_val,
                    x->off, x->off_alt, x->post, x->post_alt, x->ws, x->ws2, x->ws3, x->cont, x->cnum, x->tsz};
  for (void* p : pooled)
    if (p) cudaFreeAsync(p, 0);
  cudaDeviceSynchronize();
  void* plain[] = {x->pi, x->df, x->d_info, x->dstage, x->d_cstat, x->ccand, x->cslot};
  for (void* p : plain)
    if (p) cudaFree(p);
  if (x->h_info) cudaFreeHost(x->h_info);
  if (x->h_i64) cudaFreeHost(x->h_i64);
  if (x->hstage) cudaFreeHost(x->hstage);
  delete x;
  return SINN_OK;
}

sinn_status sinn_insert(sinn_index* x, int64_t nrows, const int64_t* indptr, const int32_t* indices,
                        const float* values, const uint32_t* ids, void* stream) {
  sinn::NvtxScope nvtx_("sinn_insert");
  GUARD(x);
  if (nrows < 0) return fail(x, SINN_EINVAL, "insert: nrows < 0");
  if (nrows == 0) return SINN_OK;
  if (!indptr || !ids) return fail(x, SINN_EINVAL, "insert: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  // 1. ONE round trip: the id checks (vacant, distinct) against the current capacity (ids beyond it
  //    are vacant by definition), then the sketch build with the row validation fused in (max id,
  //    indptr ends; columns of vacant ids below the capacity written only if the ids passed)
  x->epoch++;
  CU(cudaMemsetAsync(x->d_info, 0, sizeof(DevInfo), s));
  {
    sinn::PhaseScope ps(x, SINN_PH_VALIDATE, s);
    sinn::count_launch(x, SINN_PH_VALIDATE, 2);
    if (x->cap > 0) sinn::launch_check_ids(ids, nrows, x->live, x->stamp, x->epoch, false, x->cap, x->d_info, s);
    else CU(cudaMemsetAsync(&x->d_info->err, sinn::kErrBeyond, 1, s));  // (every id is beyond an empty index)
    sinn::launch_sketch_build(indptr, indices, values, ids, nrows, x->pi, x->m, x->h, (void*)x->sU(),
                              x->upper_only ? nullptr : (void*)x->sL(), x->bf16, s, true, x->n, x->upper_only,
                              x->cap, x->d_info, x->pi4);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(x->h_i64, indptr, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(x->h_i64 + 1, indptr + nrows, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(x->h_i64 + 3, x->d_dead, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  }
  if (read_info(x, x->d_info, s)) return SINN_ECUDA;
  x->dead_known = x->h_i64[3];
  const DevInfo v = *x->h_info;
  const int64_t base = x->h_i64[0], nnz = x->h_i64[1] - x->h_i64[0];
  if (v.err & sinn::kErrNull) return fail(x, SINN_EINVAL, "insert: null pointer");
  if (v.err & (sinn::kErrRow | sinn::kErrIndptr)) return fail(x, SINN_EINVAL, "insert: malformed row");
  if (v.err & sinn::kErrIdReserved) return fail(x, SINN_EINVAL, "insert: id 0xFFFFFFFF is reserved");
  if (nnz < 0) return fail(x, SINN_EINVAL, "insert: indptr decreasing");
  if (nnz > 0 && (!indices || !values)) return fail(x, SINN_EINVAL, "insert: null pointer");
  if (v.err & sinn::kErrLive) return fail(x, SINN_EEXIST, "insert: id already live");
  if (v.err & sinn::kErrDupId) return fail(x, SINN_EINVAL, "insert: duplicate ids in batch");
  (void)base;
  // 2. capacity; ids beyond the old capacity in a batch whose ids do not ascend may repeat among
  //    themselves: only then a second check over the grown capacity (ascending ids cannot repeat)
  if (sinn_status st = ensure_cap(x, (int64_t)v.max_id + 1, s)) return st;
  if ((v.err & sinn::kErrBeyond) && v.ids_unsorted) {
    x->epoch++;
    CU(cudaMemsetAsync(x->d_info, 0, sizeof(DevInfo), s));
    {
      sinn::PhaseScope ps(x, SINN_PH_VALIDATE, s);
      sinn::count_launch(x, SINN_PH_VALIDATE);
      sinn::launch_check_ids(ids, nrows, x->live, x->stamp, x->epoch, false, x->cap, x->d_info, s);
    }
    CU(cudaGetLastError());
    if (read_info(x, x->d_info, s)) return SINN_ECUDA;
    if (x->h_info->err & sinn::kErrLive) return fail(x, SINN_EEXIST, "insert: id already live");
    if (x->h_info->err) return fail(x, SINN_EINVAL, "insert: duplicate ids in batch");
  }
  // 3. capacities for raw store, postings and the batch workspace (before any mutation)
  if (sinn_status st = ensure_raw(x, nnz, s)) return st;
  if (sinn_status st = ensure_post(x, x->post_len + nnz, s)) return st;
  const int64_t ntiles = x->cap / 32;
  const int64_t kn = std::max<int64_t>({nnz, nrows, 1});  // sort keys: one per row (ids not ascending)
  const size_t hist_e = sinn::radix_sort_hist_elems(kn);
  const size_t need = 2 * a256(sizeof(uint64_t) * (size_t)kn) + 2 * a256(sizeof(int64_t) * (size_t)(nrows + 1)) +
                      a256(sizeof(uint32_t) * hist_e) + a256(sizeof(uint32_t) * sinn::exclusive_scan_u32_tmp_elems(hist_e)) +
                      a256(sizeof(unsigned long long) * (size_t)ntiles) + 2 * a256(sizeof(int64_t) * (size_t)(ntiles + 1)) +
                      a256(sizeof(uint32_t) * (size_t)std::max<int64_t>(nnz, 1)) +
                      (x->containers ? 3 * a256(sizeof(int64_t) * (size_t)(ntiles + 1)) : 0) +
                      a256(sizeof(int64_t) * (size_t)(ntiles + 1)) + a256(sizeof(uint32_t));
  if (sinn_status st = ensure_ws2(x, need, s)) return st;
  char* p = (char*)x->ws2;
  auto take = [&](size_t b) {
    char* r = p;
    p += a256(b);
    return r;
  };
  uint64_t* keys = (uint64_t*)take(sizeof(uint64_t) * (size_t)kn);
  uint64_t* keys_tmp = (uint64_t*)take(sizeof(uint64_t) * (size_t)kn);
  int64_t* rlen = (int64_t*)take(sizeof(int64_t) * (size_t)(nrows + 1));
  int64_t* rdst = (int64_t*)take(sizeof(int64_t) * (size_t)(nrows + 1));
  uint32_t* hist = (uint32_t*)take(sizeof(uint32_t) * hist_e);
  uint32_t* scan_tmp = (uint32_t*)take(sizeof(uint32_t) * sinn::exclusive_scan_u32_tmp_elems(hist_e));
  unsigned long long* tcount = (unsigned long long*)take(sizeof(unsigned long long) * (size_t)ntiles);
  int64_t* boff = (int64_t*)take(sizeof(int64_t) * (size_t)(ntiles + 1));
  int64_t* tsizes = (int64_t*)take(sizeof(int64_t) * (size_t)(ntiles + 1));  // merged tile sizes
  uint32_t* bpost = (uint32_t*)take(sizeof(uint32_t) * (size_t)std::max<int64_t>(nnz, 1));
  int64_t* nscan = (int64_t*)take(sizeof(int64_t) * (size_t)(ntiles + 1));  // in-place merge: new regions
  uint32_t* misfit = (uint32_t*)take(2 * sizeof(uint32_t));
  int64_t* ckept = x->containers ? (int64_t*)take(sizeof(int64_t) * (size_t)(ntiles + 1)) : nullptr;
  int64_t* cscan = x->containers ? (int64_t*)take(sizeof(int64_t) * (size_t)(ntiles + 1)) : nullptr;
  int64_t* crel = x->containers ? (int64_t*)take(sizeof(int64_t) * (size_t)(ntiles + 1)) : nullptr;

  // 4. sketch columns (Alg. 5 lines 3-9): built with the validation above unless some id lay beyond the
  //    old capacity (its column could not be written before the growth)
  if (v.err & sinn::kErrBeyond) {
    sinn::PhaseScope ps(x, SINN_PH_SKETCH, s);
    sinn::count_launch(x, SINN_PH_SKETCH);
    sinn::launch_sketch_build(indptr, indices, values, ids, nrows, x->pi, x->m, x->h, (void*)x->sU(),
                              x->upper_only ? nullptr : (void*)x->sL(), x->bf16, s, false, 0, false, 0, nullptr, x->pi4);
  }
  CU(cudaGetLastError());
  // 5. postings (Alg. 5 line 2): batch entries sorted by (tile, term, id), merged tile by tile into I
  bool append = false;
  {
    sinn::PhaseScope ps(x, SINN_PH_POSTINGS, s);
    CU(cudaMemsetAsync(tcount, 0, sizeof(unsigned long long) * (size_t)ntiles, s));
    // append fast path: ascending ids that all lie in tiles past every tile holding entries (a bulk
    // load of fresh ids) leave the old tiles untouched, so the batch's tile-ordered entries are
    // written straight to the end of the index instead of merging (copying) it
    append = nnz > 0 && !v.ids_unsorted && (int64_t)v.pad >= ((x->id_end + 31) / 32) * 32;
    if (nnz > 0 && !v.ids_unsorted) {  // ascending ids: CSR order is (id, term) already
      sinn::count_launch(x, SINN_PH_POSTINGS);
      sinn::launch_make_pairs(indptr, indices, ids, nrows, nullptr, append ? x->post + x->post_len : bpost, tcount, s);
    } else if (nnz > 0) {
      // the rows sorted by id (each id once, validated), each row's terms ascending (validated): the
      // rows in id order give the (id, term) order — a sort of nrows keys, not of nnz entries
      const int hi = 32 + bits_for((uint64_t)v.max_id);
      sinn::count_launch(x, SINN_PH_POSTINGS, 4 + 3 * ((hi - 32 + 7) / 8));
      sinn::launch_row_sorted_batch(indptr, indices, ids, nrows, hi, keys, keys_tmp, hist, scan_tmp, rlen, rdst,
                                    bpost, tcount, s);
    }
    sinn::exclusive_scan_i64_small((const int64_t*)tcount, boff, ntiles, s);
    const int64_t t_last = (int64_t)v.max_id / 32 + 1;  // 1 + the last tile the batch touches
    // documents of the last tile after this batch (a partly filled last tile gets a region for 32)
    const int64_t id_end_new = std::max<int64_t>(x->id_end, (int64_t)v.max_id + 1);
    const int32_t last_docs = (int32_t)(id_end_new - 32 * ((id_end_new - 1) / 32));
    if (append) {
      sinn::launch_add_i64(x->off, boff, x->off_alt, ntiles + 1, s);
      sinn::launch_tsz_add(x->tsz, tcount, ntiles, s);
      sinn::count_launch(x, SINN_PH_POSTINGS, 3);
      std::swap(x->off, x->off_alt);
      x->post_len += nnz;
      x->t_region_end = std::max(x->t_region_end, t_last);
    } else {
      // container bits of documents that are not live (deleted, or recycled by this batch: their new
      // entries are merged one by one) are cleared before the recycled ids become live again
      if (x->containers) sinn::launch_cont_clear(x->cont, x->cnum, x->live, ntiles, x->d_cstat, s);
      // in place when every touched tile fits its region (slack): O(touched tiles); tiles from
      // t_region_end on get new regions at the end (ids past every region)
      const int64_t t_new = std::min(x->t_region_end, ntiles);
      sinn::launch_merge_fit(x->off, x->tsz, x->tdead, tcount, ntiles, t_new, (id_end_new + 31) / 32, last_docs, misfit,
                             tsizes, nscan, s);
      sinn::count_launch(x, SINN_PH_POSTINGS, 3);
      CU(cudaMemcpyAsync(x->h_i64 + 5, nscan + (ntiles - t_new), sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      CU(cudaMemcpyAsync(&x->h_info->pad, misfit, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
      CU(cudaMemcpyAsync(x->h_i64 + 7, misfit + 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
      CU(cudaStreamSynchronize(s));
      static const bool dbg = getenv("SINN_DEBUG") != nullptr;
      if (dbg)
        fprintf(stderr, "[sinn insert] rows %lld nnz %lld: %s merge (tiles %lld, regions below %lld, new %lld)\n",
                (long long)nrows, (long long)nnz, x->h_info->pad ? "full" : "in-place", (long long)ntiles,
                (long long)t_new, (long long)x->h_i64[5]);
      if (x->h_info->pad == 0) {
        const int64_t grow = x->h_i64[5];
        if (sinn_status st = ensure_post(x, x->post_len + grow, s)) return st;
        sinn::launch_new_regions(x->off, t_new, ntiles, x->post_len, nscan, s);
        const int64_t stage = (int64_t)(uint32_t)x->h_i64[7];  // (the low word: the largest touched tile)
        sinn::launch_merge_postings(x->off, x->post, boff, bpost, ntiles, x->off, x->post, x->live, x->ecnt,
                                    x->tdead, x->tsz, s, std::max<int64_t>(stage, 2048));
        CU(cudaMemsetAsync(x->d_dead, 0, sizeof(int64_t), s));
        sinn::count_launch(x, SINN_PH_POSTINGS, 3);
        x->post_len += grow;
        x->t_region_end = std::max(t_new, t_last);
      } else {
        // a full merge into fresh regions (entries + slack): tombstones dropped, untouched tiles copied
        const int64_t t_end = std::max(x->t_region_end, t_last);
        const int64_t used = x->post_len + nnz;  // >= the entries after the merge
        if (sinn_status st = ensure_post(x, used + used / 8 + 32 * t_end + 8192 + 32 * used / std::max<int64_t>(
                                                  x->live_count + nrows, 1), s))
          return st;  // (+ the last tile's room for 32 documents)
        sinn::launch_merge_sizes(x->tsz, x->tdead, tcount, ntiles, t_end, t_end == (id_end_new + 31) / 32 ? last_docs : 32,
                                 tsizes, s);
        sinn::exclusive_scan_i64_small(tsizes, x->off_alt, ntiles, s);
        sinn::launch_merge_postings(x->off, x->post, boff, bpost, ntiles, x->off_alt, x->post_alt, x->live, x->ecnt,
                                    x->tdead, x->tsz, s);
        CU(cudaMemsetAsync(x->d_dead, 0, sizeof(int64_t), s));
        CU(cudaMemcpyAsync(x->h_i64 + 5, x->off_alt + ntiles, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        sinn::count_launch(x, SINN_PH_POSTINGS, 5);
        std::swap(x->off, x->off_alt);
        std::swap(x->post, x->post_alt);
        x->post_len = x->h_i64[5];
        x->t_region_end = t_end;
      }
      x->dead_known = 0;  // every tombstone was dropped (touched tiles are exactly those holding some)
    }
  }
  CU(cudaGetLastError());
  x->id_end = std::max<int64_t>(x->id_end, (int64_t)v.max_id + 1);
  // 6. raw-vector store + live marks
  {
    sinn::PhaseScope ps(x, SINN_PH_RAW, s);
    sinn::count_launch(x, SINN_PH_RAW);
    sinn::launch_raw_append(indptr, indices, values, ids, nrows, x->raw_used, x->raw_idx, x->raw_val, x->raw_off,
                            x->raw_nnz, x->live, x->ecnt, x->n, x->df, s);
  }
  CU(cudaGetLastError());
  x->raw_used += nnz;
  x->live_count += nrows;
  // document frequencies (dense-head split of the scoring path); max df read back for the
  // host's choice of scoring kernel
  // (the batch's document frequencies were counted by k_raw_append)
  int64_t* d_maxdf = reinterpret_cast<int64_t*>(x->d_info + 2);
  sinn::launch_df_max(x->df, x->n, d_maxdf, s);
  CU(cudaGetLastError());
  // 7. bitmap containers of a bulk load (the batch's tiles are new: [first id / 32, last id / 32])
  if (x->containers && append) {
    sinn::PhaseScope ps(x, SINN_PH_POSTINGS, s);
    const int64_t ta = (int64_t)v.pad / 32, nt = (int64_t)v.max_id / 32 + 1 - ta;
    sinn::count_launch(x, SINN_PH_POSTINGS, 6);
    sinn::launch_cont_bulk(x->off, x->post, ta, nt, ntiles, x->df, x->n, x->live_count, x->ccand,
                           x->ccand + sinn::cont_cand_cap(), x->cslot, x->cont, x->cnum, bpost, ckept, cscan, crel,
                           x->ecnt, x->tsz, x->d_cstat, s);
    CU(cudaGetLastError());
    // the new end of the postings (the tiles' remaining entries moved down): a second round trip,
    // only for bulk loads with containers
    CU(cudaMemcpyAsync(x->h_i64 + 4, x->off + ntiles, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    x->post_len = x->h_i64[4];
  }
  // read back lazily: the next search waits on the event (by then long complete) instead of this
  // insert synchronising a third time
  CU(cudaMemcpyAsync(x->h_i64 + 2, d_maxdf, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  if (!x->df_ready) CU(cudaEventCreateWithFlags(&x->df_ready, cudaEventDisableTiming));
  CU(cudaEventRecord(x->df_ready, s));
  x->df_pending = true;
  return SINN_OK;
}

sinn_status sinn_reserve(sinn_index* x, int64_t max_docs, int64_t postings, void* stream) {
  sinn::NvtxScope nvtx_("sinn_reserve");
  GUARD(x);
  if (max_docs < 0 || postings < 0 || max_docs > (int64_t)SINN_NO_ID)
    return fail(x, SINN_EINVAL, "reserve: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  if (sinn_status st = ensure_cap(x, max_docs, s)) return st;
  if (sinn_status st = ensure_raw(x, postings - x->raw_used, s)) return st;
  if (sinn_status st = ensure_post(x, postings, s)) return st;
  CU(cudaGetLastError());
  return SINN_OK;
}

sinn_status sinn_delete(sinn_index* x, int64_t count, const uint32_t* ids, void* stream) {
  sinn::NvtxScope nvtx_("sinn_delete");
  GUARD(x);
  if (count < 0) return fail(x, SINN_EINVAL, "delete: count < 0");
  if (count == 0) return SINN_OK;
  if (!ids) return fail(x, SINN_EINVAL, "delete: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  x->epoch++;
  CU(cudaMemsetAsync(x->d_info, 0, sizeof(DevInfo), s));
  {
    sinn::PhaseScope ps(x, SINN_PH_VALIDATE, s);
    sinn::count_launch(x, SINN_PH_VALIDATE);
    sinn::launch_check_ids(ids, count, x->live, x->stamp, x->epoch, true, x->cap, x->d_info, s);
    CU(cudaMemcpyAsync(x->h_i64 + 3, x->d_dead, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  }
  CU(cudaGetLastError());
  if (read_info(x, x->d_info, s)) return SINN_ECUDA;
  x->dead_known = x->h_i64[3];
  if (x->h_info->err & sinn::kErrNotLive) return fail(x, SINN_ENOTFOUND, "delete: id not live");
  if (x->h_info->err) return fail(x, SINN_EINVAL, "delete: duplicate ids");
  // tombstones (O(deleted entries)): vacant, df of the rows' terms decremented, entries counted dead
  {
    sinn::PhaseScope ps(x, SINN_PH_DELETE, s);
    sinn::count_launch(x, SINN_PH_DELETE);
    sinn::launch_delete_mark(ids, count, x->live, x->ecnt, x->tdead, x->d_dead, x->raw_off, x->raw_nnz, x->raw_idx,
                             x->df, x->containers ? x->cont : nullptr, x->cnum, x->d_cstat, s);
  }
  CU(cudaGetLastError());
  x->live_count -= count;
  // amortised compaction once the tombstones (known as of this call's round trip, plus this call's
  // estimated share) pass a quarter of the stored entries
  const int64_t est = x->dead_known + (x->live_count + count > 0 ? count * x->post_len / (x->live_count + count) : 0);
  if (est * 4 < x->post_len) return SINN_OK;
  const int64_t n = x->cap / 32;  // tiles
  if (sinn_status st = ensure_ws2(x, a256(sizeof(int64_t) * (size_t)(n + 1)), s)) return st;
  // the compacted regions: live entries + slack (<= the stored entries + an eighth + 32 per tile)
  const int64_t t_end = std::min(x->t_region_end, n);
  if (sinn_status st = ensure_post(x, x->post_len + x->post_len / 8 + 32 * t_end + 64, s)) return st;
  int64_t* counts = (int64_t*)x->ws2;
  {
    sinn::PhaseScope ps(x, SINN_PH_DELETE, s);
    sinn::count_launch(x, SINN_PH_DELETE, 3);
    sinn::launch_count_live_postings(x->tsz, x->tdead, n, t_end, counts, s);
    sinn::exclusive_scan_i64_small(counts, x->off_alt, n, s);
    sinn::launch_compact_postings(x->off, x->post, x->live, n, x->off_alt, x->post_alt, x->ecnt, x->tdead, x->tsz, s);
    if (x->containers) sinn::launch_cont_clear(x->cont, x->cnum, x->live, n, x->d_cstat, s);
  }
  CU(cudaGetLastError());
  CU(cudaMemsetAsync(x->d_dead, 0, sizeof(int64_t), s));
  CU(cudaMemcpyAsync(x->h_i64, x->off_alt + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  std::swap(x->off, x->off_alt);
  std::swap(x->post, x->post_alt);
  x->post_len = x->h_i64[0];
  x->dead_known = 0;
  return SINN_OK;
}

static sinn_status check_search_args(sinn_index* x, int64_t nq, const int64_t* qp, int32_t k, int32_t kp) {
  if (nq < 0) return fail(x, SINN_EINVAL, "search: nq < 0");
  if (k < 1 || kp < k || kp > SINN_MAX_KPRIME) return fail(x, SINN_EINVAL, "search: need 1 <= k <= kprime <= 16384");
  if (nq > 0 && !qp) return fail(x, SINN_EINVAL, "search: null pointer");
  return SINN_OK;
}

// run one search; synchronous calls retry once when the batch term table had to grow
static sinn_status run_search(sinn_index* x, const sinn::SearchArgs& a, bool sync, cudaStream_t s) {
  if (x->df_pending) {  // the last insert's max document frequency (chooses the scoring kernel)
    CU(cudaEventSynchronize(x->df_ready));
    x->max_df = x->h_i64[2];
    x->df_pending = false;
  }
  // failure-semantics test hook (tests/test_gpu_edges.py): a real launch error (1,025-thread block of
  // 1,024 max: cudaErrorInvalidConfiguration, not sticky) raised inside the call, which must return
  // SINN_ECUDA and poison the handle
  if (const char* f = getenv("SINN_TEST_FAULT")) {
    if (f[0] == '1') {
      sinn::launch_fault_probe(s);
      CU(cudaGetLastError());
    }
  }
  for (int attempt = 0; attempt < 3; attempt++) {
    if (sync) CU(cudaMemsetAsync(x->d_sinfo, 0, sizeof(DevInfo), s));
    std::string why;
    bool retry = false;
    cudaError_t e = sinn::search_batch(x, a, sync, s, &why, &retry);
    if (e != cudaSuccess)
      return fail(x, e == cudaErrorMemoryAllocation ? SINN_ENOMEM : SINN_ECUDA,
                  why.empty() ? std::string("search: ") + cudaGetErrorString(e) : why);
    if (!sync) return SINN_OK;
    if (read_info(x, x->d_sinfo, s)) return SINN_ECUDA;
    if (x->h_info->err) return fail(x, SINN_EINVAL, "search: malformed query row");
    if (!retry) return SINN_OK;
  }
  return fail(x, SINN_ECUDA, "search: term table did not converge");
}

sinn_status sinn_search(sinn_index* x, int64_t nq, const int64_t* q_indptr, const int32_t* q_indices,
                        const float* q_values, int32_t k, int32_t kprime, int32_t rerank, uint32_t* out_ids,
                        float* out_scores, uint32_t flags, void* stream) {
  sinn::NvtxScope nvtx_("sinn_search");
  GUARD(x);
  if (sinn_status st = check_search_args(x, nq, q_indptr, k, kprime)) return st;
  if (nq > 0 && (!out_ids || !out_scores)) return fail(x, SINN_EINVAL, "search: null output");
  if (nq == 0) return SINN_OK;
  sinn::SearchArgs a{nq, q_indptr, q_indices, q_values, k, kprime, rerank != 0, out_ids, out_scores, nullptr, nullptr};
  return run_search(x, a, !(flags & SINN_SEARCH_NOSYNC), (cudaStream_t)stream);
}

sinn_status sinn_search_stage1(sinn_index* x, int64_t nq, const int64_t* q_indptr, const int32_t* q_indices,
                               const float* q_values, int32_t kprime, uint32_t* cand_ids, float* cand_scores,
                               void* stream) {
  sinn::NvtxScope nvtx_("sinn_search_stage1");
  GUARD(x);
  if (sinn_status st = check_search_args(x, nq, q_indptr, 1, kprime)) return st;
  if (nq > 0 && (!cand_ids || !cand_scores)) return fail(x, SINN_EINVAL, "stage1: null output");
  if (nq == 0) return SINN_OK;
  sinn::SearchArgs a{nq, q_indptr, q_indices, q_values, 1, kprime, false, nullptr, nullptr, cand_ids, cand_scores};
  return run_search(x, a, true, (cudaStream_t)stream);
}

sinn_status sinn_search_stage1_gather(sinn_index* x, int64_t nq, const int64_t* q_indptr, const int32_t* q_indices,
                                      const float* q_values, int32_t kprime, int32_t world, int32_t slot,
                                      uint32_t* const* dst_ids, float* const* dst_scores, void* stream) {
  sinn::NvtxScope nvtx_("sinn_search_stage1_gather");
  GUARD(x);
  if (sinn_status st = check_search_args(x, nq, q_indptr, 1, kprime)) return st;
  if (world < 1 || world > sinn::kGatherMax || slot < 0 || slot >= world || !dst_ids || !dst_scores)
    return fail(x, SINN_EINVAL, "stage1_gather: need 1 <= world <= 8, 0 <= slot < world, destination arrays");
  for (int d = 0; d < world; d++)
    if (nq > 0 && (!dst_ids[d] || !dst_scores[d])) return fail(x, SINN_EINVAL, "stage1_gather: null destination");
  if (nq == 0) return SINN_OK;
  // the local copy of the rows is destination `slot` itself (no second buffer)
  uint32_t* own_ids = dst_ids[slot] + (int64_t)slot * nq * kprime;
  float* own_scores = dst_scores[slot] + (int64_t)slot * nq * kprime;
  sinn::SearchArgs a{nq, q_indptr, q_indices, q_values, 1, kprime, false, nullptr, nullptr, own_ids, own_scores};
  for (int d = 0; d < world; d++) {
    if (d == slot) continue;
    a.gather.ids[a.gather.n] = dst_ids[d];
    a.gather.scores[a.gather.n] = dst_scores[d];
    a.gather.n++;
  }
  a.gather.off = (int64_t)slot * nq * kprime;
  return run_search(x, a, true, (cudaStream_t)stream);
}

sinn_status sinn_search_anytime(sinn_index* x, int64_t nq, const int64_t* q_indptr, const int32_t* q_indices,
                                const float* q_values, int32_t k, int32_t kprime, int32_t rerank, int32_t max_terms,
                                uint32_t* out_ids, float* out_scores, uint32_t flags, void* stream) {
  sinn::NvtxScope nvtx_("sinn_search_anytime");
  GUARD(x);
  if (sinn_status st = check_search_args(x, nq, q_indptr, k, kprime)) return st;
  if (max_terms < 0) return fail(x, SINN_EINVAL, "search_anytime: max_terms < 0");
  if (nq > 0 && (!out_ids || !out_scores)) return fail(x, SINN_EINVAL, "search: null output");
  if (nq == 0) return SINN_OK;
  sinn::SearchArgs a{nq, q_indptr, q_indices, q_values, k, kprime, rerank != 0, out_ids, out_scores, nullptr, nullptr};
  a.max_terms = max_terms;
  return run_search(x, a, !(flags & SINN_SEARCH_NOSYNC), (cudaStream_t)stream);
}

sinn_status sinn_search_filtered(sinn_index* x, int64_t nq, const int64_t* q_indptr, const int32_t* q_indices,
                                 const float* q_values, int32_t k, int32_t kprime, int32_t rerank, const uint32_t* allow,
                                 int64_t allow_words, uint32_t* out_ids, float* out_scores, uint32_t flags,
                                 void* stream) {
  sinn::NvtxScope nvtx_("sinn_search_filtered");
  GUARD(x);
  if (sinn_status st = check_search_args(x, nq, q_indptr, k, kprime)) return st;
  if (allow_words < 0 || (allow_words > 0 && !allow)) return fail(x, SINN_EINVAL, "search_filtered: bad mask");
  if (nq > 0 && (!out_ids || !out_scores)) return fail(x, SINN_EINVAL, "search: null output");
  if (nq == 0) return SINN_OK;
  static const uint32_t kNone = 0;
  sinn::SearchArgs a{nq, q_indptr, q_indices, q_values, k, kprime, rerank != 0, out_ids, out_scores, nullptr, nullptr};
  a.allow = allow_words > 0 ? allow : &kNone;  // an empty mask admits nothing (kNone is never read: 0 words)
  a.allow_words = allow_words;
  return run_search(x, a, !(flags & SINN_SEARCH_NOSYNC), (cudaStream_t)stream);
}

// F4: qmask entries in [-1, nmasks) (device check; the flag joins the search validation word)
__global__ void k_check_qmask(const int32_t* __restrict__ qmask, int64_t nq, int32_t nmasks, sinn::DevInfo* info) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = qmask[q];
    if (r < -1 || r >= nmasks) atomicOr(&info->err, sinn::kErrRow);
  }
}

sinn_status sinn_search_masked(sinn_index* x, int64_t nq, const int64_t* q_indptr, const int32_t* q_indices,
                               const float* q_values, int32_t k, int32_t kprime, int32_t rerank, const uint32_t* masks,
                               int64_t mask_words, int32_t nmasks, const int32_t* qmask, uint32_t* out_ids,
                               float* out_scores, uint32_t flags, void* stream) {
  sinn::NvtxScope nvtx_("sinn_search_masked");
  GUARD(x);
  if (sinn_status st = check_search_args(x, nq, q_indptr, k, kprime)) return st;
  if (nmasks < 0 || mask_words < 0 || (nmasks > 0 && mask_words > 0 && !masks) || (nq > 0 && !qmask))
    return fail(x, SINN_EINVAL, "search_masked: bad mask table");
  if (nq > 0 && (!out_ids || !out_scores)) return fail(x, SINN_EINVAL, "search: null output");
  if (nq == 0) return SINN_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const bool sync = !(flags & SINN_SEARCH_NOSYNC);
  if (sync) CU(cudaMemsetAsync(x->d_sinfo, 0, sizeof(DevInfo), s));
  k_check_qmask<<<(unsigned)std::min<int64_t>((nq + 255) / 256, 1024), 256, 0, s>>>(qmask, nq, nmasks, x->d_sinfo);
  CU(cudaGetLastError());
  if (sync) {  // a bad mask index is an argument error: nothing is searched
    if (read_info(x, x->d_sinfo, s)) return SINN_ECUDA;
    if (x->h_info->err) return fail(x, SINN_EINVAL, "search_masked: qmask entry outside [-1, nmasks)");
  }
  static const uint32_t kNone = 0;
  sinn::SearchArgs a{nq, q_indptr, q_indices, q_values, k, kprime, rerank != 0, out_ids, out_scores, nullptr, nullptr};
  a.qmasks = (nmasks > 0 && mask_words > 0) ? masks : &kNone;  // (kNone is never read: 0 words)
  a.qmask_words = (nmasks > 0) ? mask_words : 0;
  a.nmasks = nmasks;
  a.qmask = qmask;
  return run_search(x, a, sync, s);
}

sinn_status sinn_search_exact(sinn_index* x, int64_t nq, const int64_t* q_indptr, const int32_t* q_indices,
                              const float* q_values, int32_t k, uint32_t* out_ids, float* out_scores, void* stream) {
  sinn::NvtxScope nvtx_("sinn_search_exact");
  GUARD(x);
  if (sinn_status st = check_search_args(x, nq, q_indptr, k, k)) return st;
  if (nq > 0 && (!out_ids || !out_scores)) return fail(x, SINN_EINVAL, "search_exact: null output");
  if (nq == 0) return SINN_OK;
  sinn::SearchArgs a{nq, q_indptr, q_indices, q_values, k, k, false, out_ids, out_scores, nullptr, nullptr};
  a.exact = true;
  return run_search(x, a, true, (cudaStream_t)stream);
}

sinn_status sinn_rerank(sinn_index* x, int64_t nq, const int64_t* q_indptr, const int32_t* q_indices,
                        const float* q_values, int32_t kc, const uint32_t* cand_ids, uint32_t id_mul, uint32_t id_add,
                        int32_t k, uint32_t* out_ids, float* out_scores, void* stream) {
  sinn::NvtxScope nvtx_("sinn_rerank");
  GUARD(x);
  if (sinn_status st = check_search_args(x, nq, q_indptr, k, kc)) return st;
  if (id_mul < 1 || id_add >= id_mul) return fail(x, SINN_EINVAL, "rerank: need id_mul >= 1 and id_add < id_mul");
  if (nq > 0 && (!cand_ids || !out_ids || !out_scores)) return fail(x, SINN_EINVAL, "rerank: null pointer");
  if (nq == 0) return SINN_OK;
  std::string why;
  cudaError_t e = sinn::rerank_candidates(x, nq, q_indptr, q_indices, q_values, kc, cand_ids, id_mul, id_add, k, out_ids,
                                          out_scores, (cudaStream_t)stream, &why);
  if (e != cudaSuccess)
    return fail(x, e == cudaErrorMemoryAllocation ? SINN_ENOMEM : SINN_ECUDA,
                why.empty() ? std::string("rerank: ") + cudaGetErrorString(e) : why);
  return SINN_OK;
}

sinn_status sinn_merge_topk(int64_t nq, int32_t parts, int32_t kin, const uint32_t* ids, const float* scores,
                            uint32_t id_mul, const uint32_t* id_add, int32_t kout, uint32_t* out_ids, float* out_scores,
                            void* stream) {
  sinn::NvtxScope nvtx_("sinn_merge_topk");
  if (nq < 0 || nq > 0x7fffffffLL || parts < 1 || parts > sinn::kMergeMaxParts || kin < 1 ||
      (int64_t)parts * kin > sinn::kMergeMaxItems || kout < 1 || kout > sinn::kMergeMaxItems || id_mul < 1)
    return SINN_EINVAL;
  if (nq > 0 && (!ids || !scores || !out_ids || !out_scores)) return SINN_EINVAL;
  if (nq == 0) return SINN_OK;
  cudaError_t e = sinn::launch_merge_topk(nq, parts, kin, ids, scores, id_mul, id_add, kout, out_ids, out_scores,
                                          (cudaStream_t)stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return SINN_ECUDA;
  }
  return SINN_OK;
}

sinn_status sinn_sync(sinn_index* x, void* stream) {
  GUARD(x);
  cudaStream_t s = (cudaStream_t)stream;
  if (read_info(x, x->d_sinfo, s)) return SINN_ECUDA;
  const DevInfo inf = *x->h_info;
  CU(cudaMemsetAsync(x->d_sinfo, 0, sizeof(DevInfo), s));
  CU(cudaStreamSynchronize(s));
  if (inf.err) return fail(x, SINN_EINVAL, "search: malformed query row (deferred)");
  if (inf.pad || inf.max_id)
    return fail(x, SINN_EAGAIN, "search: some queries need a synchronous search (re-run without SINN_SEARCH_NOSYNC)");
  return SINN_OK;
}

sinn_status sinn_insert_host(sinn_index* x, int64_t nrows, const int64_t* indptr, const int32_t* indices,
                             const float* values, const uint32_t* ids, void* stream) {
  sinn::NvtxScope nvtx_("sinn_insert_host");
  GUARD(x);
  if (nrows < 0) return fail(x, SINN_EINVAL, "insert: nrows < 0");
  if (nrows == 0) return SINN_OK;
  if (!indptr || !ids) return fail(x, SINN_EINVAL, "insert: null pointer");
  const int64_t base = indptr[0], nnz = indptr[nrows] - indptr[0];
  if (nnz < 0) return fail(x, SINN_EINVAL, "insert: indptr decreasing");
  if (nnz > 0 && (!indices || !values)) return fail(x, SINN_EINVAL, "insert: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t b_ip = a256(sizeof(int64_t) * (size_t)(nrows + 1)), b_ix = a256(sizeof(int32_t) * (size_t)nnz),
               b_v = a256(sizeof(float) * (size_t)nnz), b_id = a256(sizeof(uint32_t) * (size_t)nrows);
  if (sinn_status st = ensure_stage(x, b_ip + b_ix + b_v + b_id)) return st;
  char* d = (char*)x->dstage;
  char* h = (char*)x->hstage;
  int64_t* hip = (int64_t*)h;
  for (int64_t r = 0; r <= nrows; r++) hip[r] = indptr[r] - base;
  memcpy(h + b_ip, indices + base, sizeof(int32_t) * (size_t)nnz);
  memcpy(h + b_ip + b_ix, values + base, sizeof(float) * (size_t)nnz);
  memcpy(h + b_ip + b_ix + b_v, ids, sizeof(uint32_t) * (size_t)nrows);
  CU(cudaMemcpyAsync(d, h, b_ip + b_ix + b_v + b_id, cudaMemcpyHostToDevice, s));
  return sinn_insert(x, nrows, (const int64_t*)d, (const int32_t*)(d + b_ip), (const float*)(d + b_ip + b_ix),
                     (const uint32_t*)(d + b_ip + b_ix + b_v), stream);
}

sinn_status sinn_delete_host(sinn_index* x, int64_t count, const uint32_t* ids, void* stream) {
  sinn::NvtxScope nvtx_("sinn_delete_host");
  GUARD(x);
  if (count < 0) return fail(x, SINN_EINVAL, "delete: count < 0");
  if (count == 0) return SINN_OK;
  if (!ids) return fail(x, SINN_EINVAL, "delete: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  if (sinn_status st = ensure_stage(x, sizeof(uint32_t) * (size_t)count)) return st;
  memcpy(x->hstage, ids, sizeof(uint32_t) * (size_t)count);
  CU(cudaMemcpyAsync(x->dstage, x->hstage, sizeof(uint32_t) * (size_t)count, cudaMemcpyHostToDevice, s));
  return sinn_delete(x, count, (const uint32_t*)x->dstage, stream);
}

sinn_status sinn_search_host(sinn_index* x, int64_t nq, const int64_t* q_indptr, const int32_t* q_indices,
                             const float* q_values, int32_t k, int32_t kprime, int32_t rerank, uint32_t* out_ids,
                             float* out_scores, void* stream) {
  sinn::NvtxScope nvtx_("sinn_search_host");
  GUARD(x);
  if (sinn_status st = check_search_args(x, nq, q_indptr, k, kprime)) return st;
  if (nq > 0 && (!out_ids || !out_scores)) return fail(x, SINN_EINVAL, "search: null output");
  if (nq == 0) return SINN_OK;
  const int64_t base = q_indptr[0], nnz = q_indptr[nq] - q_indptr[0];
  if (nnz < 0) return fail(x, SINN_EINVAL, "search: indptr decreasing");
  if (nnz > 0 && (!q_indices || !q_values)) return fail(x, SINN_EINVAL, "search: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t b_ip = a256(sizeof(int64_t) * (size_t)(nq + 1)), b_ix = a256(sizeof(int32_t) * (size_t)nnz),
               b_v = a256(sizeof(float) * (size_t)nnz), b_oi = a256(sizeof(uint32_t) * (size_t)(nq * k)),
               b_os = a256(sizeof(float) * (size_t)(nq * k));
  if (sinn_status st = ensure_stage(x, b_ip + b_ix + b_v + b_oi + b_os)) return st;
  char* d = (char*)x->dstage;
  char* h = (char*)x->hstage;
  int64_t* hip = (int64_t*)h;
  for (int64_t r = 0; r <= nq; r++) hip[r] = q_indptr[r] - base;
  memcpy(h + b_ip, q_indices + base, sizeof(int32_t) * (size_t)nnz);
  memcpy(h + b_ip + b_ix, q_values + base, sizeof(float) * (size_t)nnz);
  CU(cudaMemcpyAsync(d, h, b_ip + b_ix + b_v, cudaMemcpyHostToDevice, s));
  uint32_t* doi = (uint32_t*)(d + b_ip + b_ix + b_v);
  float* dos = (float*)(d + b_ip + b_ix + b_v + b_oi);
  sinn_status st = sinn_search(x, nq, (const int64_t*)d, (const int32_t*)(d + b_ip), (const float*)(d + b_ip + b_ix),
                               k, kprime, rerank, doi, dos, 0, stream);
  if (st) return st;
  CU(cudaMemcpyAsync(h + b_ip + b_ix + b_v, doi, b_oi + b_os, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  memcpy(out_ids, h + b_ip + b_ix + b_v, sizeof(uint32_t) * (size_t)(nq * k));
  memcpy(out_scores, h + b_ip + b_ix + b_v + b_oi, sizeof(float) * (size_t)(nq * k));
  return SINN_OK;
}

sinn_status sinn_profile(sinn_index* x, int32_t enable) {
  GUARD(x);
  x->prof = enable != 0;
  if (enable) {
    x->ev_used = 0;
    x->ev_phase.clear();
    for (int p = 0; p < SINN_NUM_PHASES; p++) {
      x->prof_ms[p] = 0;
      x->prof_calls[p] = 0;
      x->prof_launches[p] = 0;
    }
  }
  return SINN_OK;
}

sinn_status sinn_profile_read(sinn_index* x, sinn_profile_t* out, void* stream) {
  GUARD(x);
  if (!out) return SINN_EINVAL;
  CU(cudaStreamSynchronize((cudaStream_t)stream));
  CU(cudaDeviceSynchronize());
  for (size_t t = 0; t < x->ev_phase.size(); t++) {
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, x->ev_pool[2 * t], x->ev_pool[2 * t + 1]));
    x->prof_ms[x->ev_phase[t]] += ms;
  }
  x->ev_used = 0;
  x->ev_phase.clear();
  for (int p = 0; p < SINN_NUM_PHASES; p++) {
    out->ms[p] = x->prof_ms[p];
    out->calls[p] = x->prof_calls[p];
    out->launches[p] = x->prof_launches[p];
  }
  return SINN_OK;
}

const char* sinn_last_error(const sinn_index* x) { return x ? x->last_error.c_str() : "null handle"; }

sinn_status sinn_export_sketch(sinn_index* x, int64_t count, const uint32_t* ids, float* U, float* L, void* stream) {
  GUARD(x);
  if (count < 0 || (count > 0 && (!ids || !U))) return fail(x, SINN_EINVAL, "export_sketch: bad arguments");
  if (count == 0) return SINN_OK;
  cudaStream_t s = (cudaStream_t)stream;
  // bounds check on the host (debug path)
  uint32_t* hid = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)count);
  cudaError_t e = cudaMemcpyAsync(hid, ids, sizeof(uint32_t) * (size_t)count, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  bool ok = true;
  for (int64_t r = 0; r < count && e == cudaSuccess; r++) ok &= (int64_t)hid[r] < x->cap;
  free(hid);
  CU(e);
  if (!ok) return fail(x, SINN_EINVAL, "export_sketch: id beyond capacity");
  sinn::launch_gather_rows(ids, count, x->sU(), x->bf16, x->m, U, s);
  if (L && !x->upper_only) sinn::launch_gather_rows(ids, count, x->sL(), x->bf16, x->m, L, s);
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(s));
  return SINN_OK;
}

sinn_status sinn_export_postings(sinn_index* x, int32_t term, uint32_t* out, int64_t cap, int64_t* len,
                                 void* stream) {
  GUARD(x);
  if (term < 0 || term >= x->n || !len || cap < 0 || (cap > 0 && !out))
    return fail(x, SINN_EINVAL, "export_postings: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t ntiles = x->cap / 32;
  *len = 0;
  if (ntiles == 0) return SINN_OK;
  const size_t b_cnt = a256(sizeof(uint32_t) * (size_t)(ntiles + 1));
  if (sinn_status st = ensure_ws2(x, 2 * b_cnt + a256(sizeof(uint32_t) * sinn::exclusive_scan_u32_tmp_elems(ntiles + 1)), s))
    return st;
  uint32_t* cnt = (uint32_t*)x->ws2;
  uint32_t* pos = (uint32_t*)((char*)x->ws2 + b_cnt);
  uint32_t* tmp = (uint32_t*)((char*)x->ws2 + 2 * b_cnt);
  CU(cudaMemsetAsync(cnt, 0, b_cnt, s));
  sinn::launch_export_term(x->off, x->tsz, x->post, x->live, x->containers ? x->cont : nullptr, x->cnum, ntiles,
                           (uint32_t)term, cnt, pos, tmp, out, cap, s);
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(x->h_info, pos + ntiles, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  *len = (int64_t)*(uint32_t*)x->h_info;
  return SINN_OK;
}

sinn_status sinn_decode(sinn_index* x, int64_t count, const uint32_t* ids, const int32_t* terms,
                        const uint8_t* positive, float* out, void* stream) {
  GUARD(x);
  if (count < 0 || (count > 0 && (!ids || !terms || !positive || !out)))
    return fail(x, SINN_EINVAL, "decode: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  sinn::launch_decode(ids, terms, positive, count, x->sU(), x->sL(), x->bf16, x->pi, x->m, x->h, x->upper_only,
                      out, s);
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(s));
  return SINN_OK;
}

sinn_status sinn_stats(const sinn_index* x, sinn_stats_t* out) {
  if (!x || !out) return SINN_EINVAL;
  int64_t dead = 0;  // tombstoned entries (device counter; this debug call reads it synchronously)
  if (x->d_dead && cudaMemcpy(&dead, x->d_dead, sizeof(int64_t), cudaMemcpyDeviceToHost) != cudaSuccess) dead = 0;
  int64_t cs[3] = {0, 0, 0};  // container slots, bits set, bits of deleted documents
  if (x->d_cstat && cudaMemcpy(cs, x->d_cstat, sizeof(cs), cudaMemcpyDeviceToHost) != cudaSuccess) cs[0] = cs[1] = cs[2] = 0;
  int64_t stored = 0;  // entries in use in the tile regions (their slack excluded)
  if (x->tsz && x->cap >= 32) {
    sinn::launch_sum_i32(x->tsz, nullptr, x->cap / 32, x->d_cstat + 3, 0);
    if (cudaMemcpy(&stored, x->d_cstat + 3, sizeof(int64_t), cudaMemcpyDeviceToHost) != cudaSuccess) stored = 0;
  }
  out->live = x->live_count;
  out->capacity = x->cap;
  out->postings = stored - dead + cs[1] - cs[2];
  out->containers = cs[0];
  out->container_postings = cs[1] - cs[2];
  out->raw_entries = x->raw_used;
  out->bytes_postings = (int64_t)(2 * x->post_cap * sizeof(uint32_t) + 2 * (x->cap / 32 + 1) * sizeof(int64_t)) +
                        (x->containers ? (int64_t)(x->cap * sizeof(uint2) + x->cap / 32) : 0);
  out->bytes_sketch = (int64_t)((x->upper_only ? 1 : 2) * x->cap * x->m * (x->bf16 ? 2 : 4));
  out->bytes_raw = (int64_t)(x->raw_cap * (sizeof(int32_t) + sizeof(float)) + x->cap * (sizeof(int64_t) + sizeof(int32_t)));
  out->bytes_workspace = (int64_t)(x->ws_bytes + x->ws2_bytes + x->ws3_bytes + x->dstage_bytes);
  out->sample_stride = x->last_stride;
  out->sample_rows_kept = x->last_rows;
  return SINN_OK;
}

}  // extern "C"
