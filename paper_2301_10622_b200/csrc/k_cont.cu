// k_cont.cu — Roaring-style bitmap containers of the tile-major inverted index (SINN_BITMAP_CONTAINERS;
// the paper keeps I as Roaring bitmaps, whose containers switch from a
// sorted id array to a bitmap where a chunk of the id space is dense).  Here the chunk is the
// 32-id tile: where a term holds >= 2 of a tile's documents, the bulk load stores (term, 32-bit
// document mask) in one of the tile's 32 container slots instead of one entry (term << 5 | d) per
// document.  A term is a container candidate when its list is dense enough to fill slots across
// tiles: document frequency >= kContMinFrac of the live documents (the 64 most frequent such terms
// after the batch's df update); each tile then keeps the (up to) 32 candidates with the most of its
// documents.  Later changes never extend containers: a recycled id's new entries are stored one by
// one, and the bits of documents that are not live are cleared when a merge or a compaction
// rewrites the index (k_cont_clear; until then the walks skip them like any tombstone).
#include <stdint.h>

#include <algorithm>

#include "sinn_internal.cuh"

namespace sinn {

namespace {

constexpr int kContCand = 64;          // candidate terms per bulk load
constexpr int kContCandMax = 4096;     // terms over the frequency bar considered for the candidates
constexpr float kContMinFrac = 0.05f;  // df / live for a candidate (2 of a tile's 32 documents expected: 0.06)

inline unsigned grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  b = std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)sm_count() * 32));
  return (unsigned)b;
}

// one block: the candidate terms (df >= bar, the kContCand most frequent, ties by term id) -> cand[],
// their slot in slotmap (int8[n]; the previous candidates' slots are cleared first), ncand
__global__ void __launch_bounds__(1024) k_cont_cands(const int32_t* __restrict__ df, int32_t n, int32_t bar,
                                                     int32_t* __restrict__ cand, int32_t* __restrict__ ncand,
                                                     int8_t* __restrict__ slotmap) {
  __shared__ unsigned long long sb[kContCandMax];
  __shared__ uint32_t cnt;
  const int prev = *ncand;
  for (int t = threadIdx.x; t < prev; t += blockDim.x) slotmap[cand[t]] = -1;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int32_t j = threadIdx.x; j < n; j += blockDim.x) {
    const int32_t f = df[j];
    if (f >= bar && f > 0) {
      const uint32_t pos = atomicAdd(&cnt, 1u);
      if (pos < (uint32_t)kContCandMax) sb[pos] = ((unsigned long long)(uint32_t)f << 32) | (uint32_t)~(uint32_t)j;
    }
  }
  __syncthreads();
  const int c = (int)min(cnt, (uint32_t)kContCandMax);
  int N = 1;
  while (N < c) N <<= 1;
  for (int t = c + threadIdx.x; t < N; t += blockDim.x) sb[t] = 0ull;
  for (int k = 2; k <= N; k <<= 1)
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const int l = i ^ jj;
        if (l > i) {
          const unsigned long long a = sb[i], b = sb[l];
          if (((i & k) == 0) ? (a < b) : (a > b)) {
            sb[i] = b;
            sb[l] = a;
          }
        }
      }
    }
  __syncthreads();
  const int nc = min(c, kContCand);
  for (int t = threadIdx.x; t < nc; t += blockDim.x) {
    const int32_t j = (int32_t)~(uint32_t)(sb[t] & 0xffffffffu);
    cand[t] = j;
    slotmap[j] = (int8_t)t;
  }
  if (threadIdx.x == 0) *ncand = nc;
}

// one block per tile of the bulk load (tiles [ta, ta + nt)): the candidates' document masks, the (up
// to) 32 with the most documents (>= 2) become the tile's containers (slot = rank), and the tile's
// other entries are compacted, in order, to tmp[off[t] - off[ta] ..); kept[t - ta] = their count;
// ecnt of the tile's documents drops by the entries now held as container bits
__global__ void __launch_bounds__(256) k_cont_build(const int64_t* __restrict__ off, const uint32_t* __restrict__ post,
                                                    int64_t ta, int64_t nt, const int8_t* __restrict__ slotmap,
                                                    const int32_t* __restrict__ cand, const int32_t* __restrict__ ncand,
                                                    uint2* __restrict__ cont, uint8_t* __restrict__ cnum,
                                                    uint32_t* __restrict__ tmp, int64_t* __restrict__ kept,
                                                    int32_t* __restrict__ ecnt, int32_t* __restrict__ tsz,
                                                    int64_t* __restrict__ cstat) {
  __shared__ uint32_t mask[kContCand];
  __shared__ int8_t csel[kContCand];
  __shared__ int32_t rem[32];
  __shared__ uint32_t wsum[8];
  __shared__ uint32_t s_kept;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nc = *ncand;
  for (int64_t u = blockIdx.x; u < nt; u += gridDim.x) {
    const int64_t t = ta + u;
    const int64_t b = off[t], e = off[t + 1];
    __syncthreads();
    if (threadIdx.x < kContCand) {
      mask[threadIdx.x] = 0;
      csel[threadIdx.x] = -1;
    }
    if (threadIdx.x < 32) rem[threadIdx.x] = 0;
    if (threadIdx.x == 0) s_kept = 0;
    __syncthreads();
    for (int64_t p = b + threadIdx.x; p < e; p += blockDim.x) {
      const uint32_t en = post[p];
      const int sl = slotmap[en >> 5];
      if (sl >= 0) atomicOr(&mask[sl], 1u << (en & 31u));
    }
    __syncthreads();
    if (threadIdx.x < kContCand) {  // rank by (documents desc, slot asc); slots under 2 documents stay out
      const int sidx = threadIdx.x;
      const int pc = sidx < nc ? __popc(mask[sidx]) : 0;
      int rank = 0;
      for (int o = 0; o < nc; o++) {
        const int po = __popc(mask[o]);
        rank += (po > pc) || (po == pc && o < sidx);
      }
      if (pc >= 2 && rank < 32) {
        csel[sidx] = (int8_t)rank;
        cont[t * 32 + rank] = make_uint2((uint32_t)cand[sidx], mask[sidx]);
      }
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // slots in use: the ranks below the number of selected candidates
      uint32_t sel = 0;
      for (int o = 0; o < nc; o++) sel += csel[o] >= 0;
      if (threadIdx.x == 0) {
        cnum[t] = (uint8_t)sel;
        uint32_t bits = 0;
        for (int o = 0; o < nc; o++)
          if (csel[o] >= 0) bits += __popc(mask[o]);
        if (sel) {
          atomicAdd(reinterpret_cast<unsigned long long*>(cstat), (unsigned long long)sel);
          atomicAdd(reinterpret_cast<unsigned long long*>(cstat + 1), (unsigned long long)bits);
        }
      }
    }
    // the entries that stay entries, in order (block scan per 256-entry round)
    uint32_t* out = tmp + (b - off[ta]);
    for (int64_t p0 = b; p0 < e; p0 += blockDim.x) {
      const int64_t p = p0 + threadIdx.x;
      uint32_t en = 0;
      bool keep = false;
      if (p < e) {
        en = post[p];
        const int sl = slotmap[en >> 5];
        keep = !(sl >= 0 && csel[sl] >= 0);
        if (!keep) atomicAdd(&rem[en & 31u], 1);
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, keep);
      if (lane == 0) wsum[w] = __popc(bal);
      __syncthreads();
      uint32_t before = 0, total = 0;
      for (int k = 0; k < (int)(blockDim.x >> 5); k++) {
        before += k < w ? wsum[k] : 0u;
        total += wsum[k];
      }
      const uint32_t base = s_kept;
      if (keep) out[base + before + __popc(bal & ((1u << lane) - 1u))] = en;
      __syncthreads();
      if (threadIdx.x == 0) s_kept = base + total;
      __syncthreads();
    }
    if (threadIdx.x < 32 && rem[threadIdx.x]) ecnt[t * 32 + threadIdx.x] -= rem[threadIdx.x];
    if (threadIdx.x == 0) {
      kept[u] = s_kept;
      tsz[t] = (int32_t)s_kept;
    }
  }
}

// new offsets of the bulk-load tiles (noff = exclusive scan of kept, from off[ta]) and of every tile
// after them (empty): off[t] for t in (ta, ntiles]
__global__ void k_cont_offsets(int64_t* __restrict__ off, int64_t ta, int64_t nt, int64_t ntiles,
                               const int64_t* __restrict__ scan) {
  const int64_t base = off[ta];
  for (int64_t t = ta + 1 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t <= ntiles;
       t += (int64_t)gridDim.x * blockDim.x)
    off[t] = base + scan[min(t - ta, nt)];
}

// copy the kept entries of tile ta + u from tmp (at its old offset) to post (at its new one)
__global__ void __launch_bounds__(256) k_cont_copy(const int64_t* __restrict__ old_off_rel,
                                                   const int64_t* __restrict__ off, int64_t ta, int64_t nt,
                                                   const int64_t* __restrict__ kept, const uint32_t* __restrict__ tmp,
                                                   uint32_t* __restrict__ post) {
  for (int64_t u = blockIdx.x; u < nt; u += gridDim.x) {
    const uint32_t* src = tmp + old_off_rel[u];
    uint32_t* dst = post + off[ta + u];
    for (int64_t k = threadIdx.x; k < kept[u]; k += blockDim.x) dst[k] = src[k];
  }
}

// relative old offsets of the bulk-load tiles (before k_cont_offsets rewrites off)
__global__ void k_cont_rel(const int64_t* __restrict__ off, int64_t ta, int64_t nt, int64_t* __restrict__ rel) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < nt; u += (int64_t)gridDim.x * blockDim.x)
    rel[u] = off[ta + u] - off[ta];
}

// warp per tile with containers: the bits of documents that are not live are cleared (before a
// merge or compaction rewrites the index, and before recycled ids become live again), and the
// statistics drop by them (they were counted as bits of deleted documents by k_delete_mark, or are
// the stale bits of ids being recycled, whose delete counted them the same way)
__global__ void k_cont_clear(uint2* __restrict__ cont, const uint8_t* __restrict__ cnum,
                             const uint8_t* __restrict__ live, int64_t ntiles, int64_t* __restrict__ cstat) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = warp; t < ntiles; t += nwarps) {
    const int c = cnum[t];
    if (c == 0) continue;
    const uint32_t lm = __ballot_sync(0xffffffffu, live[t * 32 + lane] != 0);
    uint32_t cleared = 0;
    if (lane < c) {
      uint2 v = cont[t * 32 + lane];
      cleared = __popc(v.y & ~lm);
      if (cleared) {
        v.y &= lm;
        cont[t * 32 + lane] = v;
      }
    }
    cleared = __reduce_add_sync(0xffffffffu, cleared);
    if (lane == 0 && cleared) {
      atomicAdd(reinterpret_cast<unsigned long long*>(cstat + 1), (unsigned long long)(-(int64_t)cleared));
      atomicAdd(reinterpret_cast<unsigned long long*>(cstat + 2), (unsigned long long)(-(int64_t)cleared));
    }
  }
}

}  // namespace

// bulk load of the tiles [ta, ta + nt) (their entries at post[off[ta] .. off[ta + nt])): containers,
// compaction of the remaining entries, new offsets; returns through *new_len the new end of post.
// Workspace: tmp (entries of the tiles), kept / scan / rel (nt + 1 int64 each).
void launch_cont_bulk(int64_t* off, uint32_t* post, int64_t ta, int64_t nt, int64_t ntiles, const int32_t* df,
                      int32_t n, int64_t live, int32_t* cand, int32_t* ncand, int8_t* slotmap, uint2* cont,
                      uint8_t* cnum, uint32_t* tmp, int64_t* kept, int64_t* scan, int64_t* rel, int32_t* ecnt,
                      int32_t* tsz, int64_t* cstat, cudaStream_t s) {
  if (nt <= 0) return;
  const int32_t bar = std::max<int32_t>(2, (int32_t)(kContMinFrac * (double)live));
  k_cont_cands<<<1, 1024, 0, s>>>(df, n, bar, cand, ncand, slotmap);
  k_cont_rel<<<grid_for(nt, 256), 256, 0, s>>>(off, ta, nt, rel);
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nt, (int64_t)sm_count() * 8));
  k_cont_build<<<blocks, 256, 0, s>>>(off, post, ta, nt, slotmap, cand, ncand, cont, cnum, tmp, kept, ecnt, tsz, cstat);
  exclusive_scan_i64_small(kept, scan, nt, s);  // scan[nt] = the tiles' new total
  k_cont_offsets<<<grid_for(ntiles - ta, 256), 256, 0, s>>>(off, ta, nt, ntiles, scan);
  k_cont_copy<<<blocks, 256, 0, s>>>(rel, off, ta, nt, kept, tmp, post);
}

int cont_cand_cap() { return kContCand; }

void launch_cont_clear(uint2* cont, const uint8_t* cnum, const uint8_t* live, int64_t ntiles, int64_t* cstat,
                       cudaStream_t s) {
  if (ntiles > 0) k_cont_clear<<<grid_for(ntiles * 32, 256), 256, 0, s>>>(cont, cnum, live, ntiles, cstat);
}

}  // namespace sinn
