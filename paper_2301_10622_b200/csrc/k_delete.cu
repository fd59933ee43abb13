// k_delete.cu — deletion: ids become vacant at once and leave I[term] observably (searches
// skip vacant documents, df drops, export_postings filters them); their stored entries stay as
// tombstones, counted per tile, until the next merge of an insert drops them or the dead share of the
// index passes a quarter (order-preserving compaction, amortised) — a delete is O(deleted entries),
// not O(index).  The sketch column stays stale until the id is recycled.  Also the stand-alone decode
// kernel used for bit-exact decode parity.
#include "sinn_device.cuh"
#include <algorithm>

#include "sinn_internal.cuh"

namespace sinn {

namespace {

// warp per deleted id: vacant; its tile's dead-entry count and the index total grow by the entries it
// keeps as tombstones; every term of its stored row leaves I[term] (df - 1): O(deleted entries)
__global__ void k_delete_mark(const uint32_t* __restrict__ ids, int64_t count, uint8_t* __restrict__ live,
                              const int32_t* __restrict__ ecnt, int32_t* __restrict__ tdead,
                              unsigned long long* __restrict__ d_dead, const int64_t* __restrict__ raw_off,
                              const int32_t* __restrict__ raw_nnz, const int32_t* __restrict__ raw_idx,
                              int32_t* __restrict__ df, const uint2* __restrict__ cont,
                              const uint8_t* __restrict__ cnum, int64_t* __restrict__ cstat) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < count; r += nwarps) {
    const uint32_t id = ids[r];
    if (lane == 0) {
      live[id] = 0;
      const int32_t c = ecnt[id];
      if (c) {
        atomicAdd(&tdead[id >> 5], c);
        atomicAdd(d_dead, (unsigned long long)c);
      }
    }
    const int64_t ro = raw_off[id];
    const int32_t rn = raw_nnz[id];
    for (int32_t p = lane; p < rn; p += 32) atomicSub(&df[raw_idx[ro + p]], 1);
    if (cont) {  // its postings held as container bits become bits of a deleted document
      const int64_t t = id >> 5;
      const bool bit = lane < (int)cnum[t] && ((cont[t * 32 + lane].y >> (id & 31u)) & 1u);
      const uint32_t nb = __popc(__ballot_sync(0xffffffffu, bit));
      if (lane == 0 && nb) atomicAdd(reinterpret_cast<unsigned long long*>(cstat + 2), (unsigned long long)nb);
    }
  }
}

// the compacted tiles' regions: live entries (stored - dead) + slack below t_end (k_insert.cu's rule)
__global__ void k_count_live(const int32_t* __restrict__ tsz, const int32_t* __restrict__ tdead, int64_t n,
                             int64_t t_end, int64_t* __restrict__ counts) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t sz = (int64_t)tsz[t] - tdead[t];
    counts[t] = t < t_end ? sz + (sz >> 3) + 32 : sz;
  }
}

// one block per tile: stable compaction of the live entries of tile t to new_post[new_off[t] ..); the
// tile's dead documents lose their entries (ecnt 0) and the tile its tombstone count
__global__ void k_compact(const int64_t* __restrict__ off, const uint32_t* __restrict__ post,
                          const uint8_t* __restrict__ live, int64_t n, const int64_t* __restrict__ new_off,
                          uint32_t* __restrict__ new_post, int32_t* __restrict__ ecnt, int32_t* __restrict__ tdead,
                          int32_t* __restrict__ tsz) {
  __shared__ uint32_t wsum[32];
  __shared__ int64_t carry;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
    const int64_t b = off[j], e = b + tsz[j];
    uint32_t* out = new_post + new_off[j];
    if (threadIdx.x == 0) carry = 0;
    if (threadIdx.x < 32 && !live[(j << 5) | threadIdx.x]) ecnt[(j << 5) | threadIdx.x] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
      tsz[j] -= tdead[j];
      tdead[j] = 0;
    }
    for (int64_t t0 = b; t0 < e; t0 += blockDim.x) {
      const int64_t p = t0 + threadIdx.x;
      uint32_t id = 0;
      bool keep = false;
      if (p < e) {
        id = post[p];
        keep = live[(j << 5) | (id & 31u)] != 0;
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, keep);
      const uint32_t rank = __popc(bal & ((1u << lane) - 1u));
      if (lane == 0) wsum[w] = __popc(bal);
      __syncthreads();
      uint32_t before = 0, total = 0;
      for (int ww = 0; ww < nw; ww++) {
        if (ww < w) before += wsum[ww];
        total += wsum[ww];
      }
      if (keep) out[carry + before + rank] = id;
      __syncthreads();
      if (threadIdx.x == 0) carry += total;
      __syncthreads();
    }
  }
}

template <class T>  // sketch cell: float, or bfloat16 bits (F3)
__global__ void k_decode(const uint32_t* __restrict__ ids, const int32_t* __restrict__ terms,
                         const uint8_t* __restrict__ positive, int64_t count, const T* __restrict__ U,
                         const T* __restrict__ L, const uint16_t* __restrict__ pi, int32_t m, int32_t h,
                         int upper_only, float* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t j = terms[t];
    int cells[SINN_MAX_H];
    for (int o = 0; o < h; o++) cells[o] = pi[(int64_t)j * h + o];
    float e;
    if (positive[t]) e = decode_upper(U + (int64_t)ids[t] * m, cells, h);
    else if (upper_only) e = 0.0f;
    else e = decode_lower(L + (int64_t)ids[t] * m, cells, h);
    out[t] = e;
  }
}

template <class T>
__global__ void k_gather_rows(const uint32_t* __restrict__ ids, int64_t count, const T* __restrict__ src,
                              int32_t m, float* __restrict__ out) {
  const int64_t total = count * m;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = cellf(src[(int64_t)ids[t / m] * m + t % m]);
}

inline unsigned grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > (int64_t)sm_count() * 32) b = (int64_t)sm_count() * 32;
  return (unsigned)b;
}

}  // namespace

void launch_delete_mark(const uint32_t* ids, int64_t count, uint8_t* live, const int32_t* ecnt, int32_t* tdead,
                        int64_t* d_dead, const int64_t* raw_off, const int32_t* raw_nnz, const int32_t* raw_idx,
                        int32_t* df, const uint2* cont, const uint8_t* cnum, int64_t* cstat, cudaStream_t s) {
  k_delete_mark<<<grid_for(count * 32, 256), 256, 0, s>>>(ids, count, live, ecnt, tdead,
                                                          reinterpret_cast<unsigned long long*>(d_dead), raw_off,
                                                          raw_nnz, raw_idx, df, cont, cnum, cstat);
}

void launch_count_live_postings(const int32_t* tsz, const int32_t* tdead, int64_t n, int64_t t_end, int64_t* counts,
                                cudaStream_t s) {
  k_count_live<<<grid_for(n, 256), 256, 0, s>>>(tsz, tdead, n, t_end, counts);
}

void launch_compact_postings(const int64_t* off, const uint32_t* post, const uint8_t* live, int64_t n,
                             const int64_t* new_off, uint32_t* new_post, int32_t* ecnt, int32_t* tdead, int32_t* tsz,
                             cudaStream_t s) {
  int64_t blocks = std::min<int64_t>(n, (int64_t)sm_count() * 64);
  if (blocks < 1) blocks = 1;
  k_compact<<<(unsigned)blocks, 256, 0, s>>>(off, post, live, n, new_off, new_post, ecnt, tdead, tsz);
}

// export of I[term] from the tile-major index: inside a tile the entries are grouped by document,
// so the (at most one per document) entries of `term` are found by a linear scan of the tile; they
// come out in ascending id order.
// the live documents of tile t holding `term`: its entries and (SINN_BITMAP_CONTAINERS) its container
// bits, as a 32-bit mask (tombstones are not in I[term]); bit order is id order
__device__ __forceinline__ uint32_t term_mask(const int64_t* __restrict__ off, const int32_t* __restrict__ tsz,
                                              const uint32_t* __restrict__ post,
                                              const uint8_t* __restrict__ live, const uint2* __restrict__ cont,
                                              const uint8_t* __restrict__ cnum, int64_t t, uint32_t term) {
  uint32_t mk = 0;
  for (int64_t p = off[t]; p < off[t] + tsz[t]; p++) {
    const uint32_t e = post[p];
    if ((e >> 5) == term) mk |= 1u << (e & 31u);
  }
  if (cont)
    for (int c = 0; c < (int)cnum[t]; c++) {
      const uint2 v = cont[t * 32 + c];
      if (v.x == term) mk |= v.y;
    }
  uint32_t lm = 0;
  for (uint32_t b = mk; b; b &= b - 1) {
    const int d = __ffs(b) - 1;
    if (live[(t << 5) | d]) lm |= 1u << d;
  }
  return lm;
}

__global__ void k_term_count(const int64_t* __restrict__ off, const int32_t* __restrict__ tsz,
                             const uint32_t* __restrict__ post,
                             const uint8_t* __restrict__ live, const uint2* __restrict__ cont,
                             const uint8_t* __restrict__ cnum, int64_t ntiles, uint32_t term,
                             uint32_t* __restrict__ cnt) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += (int64_t)gridDim.x * blockDim.x)
    cnt[t] = __popc(term_mask(off, tsz, post, live, cont, cnum, t, term));
}

__global__ void k_term_write(const int64_t* __restrict__ off, const int32_t* __restrict__ tsz,
                             const uint32_t* __restrict__ post,
                             const uint8_t* __restrict__ live, const uint2* __restrict__ cont,
                             const uint8_t* __restrict__ cnum, int64_t ntiles, uint32_t term,
                             const uint32_t* __restrict__ pos, uint32_t* __restrict__ out, int64_t cap) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t w = pos[t];
    for (uint32_t b = term_mask(off, tsz, post, live, cont, cnum, t, term); b; b &= b - 1) {
      if (w < cap) out[w] = (uint32_t)((t << 5) | (uint32_t)(__ffs(b) - 1));
      w++;
    }
  }
}

void launch_export_term(const int64_t* off, const int32_t* tsz, const uint32_t* post, const uint8_t* live,
                        const uint2* cont, const uint8_t* cnum, int64_t ntiles, uint32_t term, uint32_t* cnt,
                        uint32_t* pos, uint32_t* scan_tmp, uint32_t* out, int64_t cap, cudaStream_t s) {
  if (ntiles <= 0) return;
  k_term_count<<<grid_for(ntiles, 256), 256, 0, s>>>(off, tsz, post, live, cont, cnum, ntiles, term, cnt);
  exclusive_scan_u32(cnt, pos, ntiles + 1, scan_tmp, s);
  k_term_write<<<grid_for(ntiles, 256), 256, 0, s>>>(off, tsz, post, live, cont, cnum, ntiles, term, pos, out, cap);
}

void launch_gather_rows(const uint32_t* ids, int64_t count, const void* src, bool bf16, int32_t m, float* out,
                        cudaStream_t s) {
  if (count <= 0) return;
  if (bf16)
    k_gather_rows<<<grid_for(count * m, 256), 256, 0, s>>>(ids, count, (const uint16_t*)src, m, out);
  else
    k_gather_rows<<<grid_for(count * m, 256), 256, 0, s>>>(ids, count, (const float*)src, m, out);
}

void launch_decode(const uint32_t* ids, const int32_t* terms, const uint8_t* positive, int64_t count,
                   const void* U, const void* L, bool bf16, const uint16_t* pi, int32_t m, int32_t h,
                   bool upper_only, float* out, cudaStream_t s) {
  if (count <= 0) return;
  if (bf16)
    k_decode<<<grid_for(count, 256), 256, 0, s>>>(ids, terms, positive, count, (const uint16_t*)U,
                                                   (const uint16_t*)L, pi, m, h, upper_only ? 1 : 0, out);
  else
    k_decode<<<grid_for(count, 256), 256, 0, s>>>(ids, terms, positive, count, (const float*)U, (const float*)L,
                                                   pi, m, h, upper_only ? 1 : 0, out);
}

}  // namespace sinn
