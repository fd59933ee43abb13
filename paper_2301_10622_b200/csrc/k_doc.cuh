// k_doc.cuh — the document-owned scoring kernel k_doc_score (S1 + S2 of the hot path) and its
// launcher, as a header so that the fp32-sketch and bfloat16-sketch (F3) instantiations are
// compiled in two translation units (k_tile.cu, k_tile_bf16.cu).  See k_tile.cu for the overview.
#pragma once
#include <math.h>
#include <stdlib.h>

#include <algorithm>
#include <type_traits>

#include "sinn_device.cuh"
#include "sinn_internal.cuh"

namespace sinn {

namespace {

constexpr int kTile = 32;          // documents per tile (entry low 5 bits)
constexpr int kQMax = 1024;        // queries per pass (score row length)
constexpr int kHistBins = 4096;    // key >> 20 (k_cand_select's fallback radix levels)
constexpr int kThetaShift = 19;    // sample histogram: key >> 19 (sign, exponent, 4 mantissa bits)
constexpr int kThetaBins = 1 << (32 - kThetaShift);
constexpr uint32_t kNegZeroBits = 0x80000000u;  // untouched-cell sentinel (-0.0f)
constexpr uint32_t kFull = 0xffffffffu;
constexpr int kSelPer = 32;  // candidate keys per thread held in registers by k_cand_select
constexpr int kNarrowMax = 8;  // terms with more queries take the warp-cooperative path

// ---------------------------------------------------------------- S1 + S2: document-owned scoring
enum { kModeHist = 0, kModeEmit = 1 };

struct DocArgs {
  const int64_t* toff;
  const uint32_t* post;
  int64_t ntiles;      // tiles visited: t = it * stride, it < ntiles
  int64_t stride;
  const uint8_t* live;
  const int32_t* nnz;  // per-id entries stored in its tile (ecnt: tombstones of deleted ids included)
  const void* U;       // sketch cells: fp32, or bfloat16 bits (BF, F3)
  const void* L;       // null under Sinnamon+
  const uint16_t* pi;
  int32_t m, h;
  const uint4* dir;
  const uint2* pairs;
  int32_t nqc;         // queries in this pass (<= kQMax)
  const float* theta;  // [nqc]
  const uint32_t* list_ok;  // EMIT: 1 if every theta_q > 0 (untouched documents can never qualify)
  unsigned long long* cand;  // [nqc][cand_cap]
  uint32_t* cand_cnt;        // [nqc]
  uint32_t cand_cap;
  uint32_t* hist;            // [nqc][kThetaBins] (non-zero sample scores)
  uint32_t* nsampled;        // live documents in the sample
  int32_t parts;             // work unit = 32 / parts documents of one tile
  const float* Qh;           // HD > 0: [kDocHead][kQMax] q values of the batch's head terms (0 if absent)
  const uint32_t* head_cnt;  // HD > 0: number of head terms
  const float* raw_val;      // exact mode (non-null): an entry's estimate is its stored value x_ij
  const int64_t* raw_off;    //   (a document's entries and its raw row are in the same term order)
  uint32_t* sched;           // work-unit counter (zeroed before the launch), or null: static striding
  const uint32_t* allow;     // constrained search (Eq. 3): column mask, bit i of word i/32; null = all
  int64_t allow_words;
  int32_t single_buf;        // one sketch-column buffer per warp (large columns: more warps); the next
                             // document's column is staged after the current one's last decode
  QMaskArgs qm;              // per-query constraint sets (F4): a cell (q, i) counts only if i passes q's mask
  const uint2* cont;         // bitmap containers (F3, k_cont.cu): per tile [32] (term, document mask), or null
  const uint8_t* cnum;       //   containers in use per tile
  const int32_t* raw_idx;    // exact mode with containers: the stored value by binary search of the row
  const int32_t* raw_nnz;
  int32_t tma;               // stage sketch columns with bulk copies (cp.async.bulk + mbarrier)
  float* rows = nullptr;     // HIST: the score rows of the sampled documents are kept ([it * 32 + d][kQMax]),
                             //   so the full pass need not score the sampled tiles again (k_emit_rows)
  int64_t skip = 0;          // EMIT: tiles that are multiples of `skip` are left to k_emit_rows (0: none)
};

// F4: does document id pass query q's constraint set (qm.qmask[q] = -1: no constraint)
__device__ __forceinline__ bool qmask_pass(const QMaskArgs& qm, uint32_t q, uint32_t id) {
  if (!qm.qmask) return true;
  const int32_t r = __ldg(qm.qmask + q);
  if (r < 0) return true;
  const int64_t wd = id >> 5;
  return wd < qm.words && ((__ldg(qm.masks + (int64_t)r * qm.words + wd) >> (id & 31)) & 1u);
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void emit(const DocArgs& A, uint32_t q, float x, uint32_t id) {
  const uint32_t pos = atomicAdd(&A.cand_cnt[q], 1u);
  if (pos < A.cand_cap)
    A.cand[(int64_t)q * A.cand_cap + pos] = ((unsigned long long)f2key(x) << 32) | (unsigned long long)(~id);
}

// per-warp shared slot: score row S[kQMax] fp32, conflict tags[kQMax] u8, two sketch-column
// buffers (m or 2m cells each, fp32 or bfloat16: the next document's column streams in with
// cp.async)

__host__ __device__ inline size_t col_cells(int m, bool lower) { return (size_t)m * (lower ? 2 : 1); }

__host__ __device__ inline size_t warp_slot_bytes(int m, bool lower, bool bf = false, bool single = false,
                                                  bool claim_bits = false) {
  size_t b = sizeof(float) * (size_t)kQMax + (claim_bits ? (size_t)kQMax / 8 : (size_t)kQMax) +
             (single ? 1 : 2) * (bf ? 2 : 4) * col_cells(m, lower);
  return ((b + 15) & ~(size_t)15) + 16;  // + the two column buffers' mbarriers (bulk copies)
}

constexpr size_t kSmemBudget = 227 * 1024;  // the sm_100 per-block maximum (232,448 B)
constexpr int kDocHead = 8;        // head terms handled as a per-document dense product (HD > 0) ...
constexpr int kDocHeadWide = 16;   // ... or 16 (the most TMEM holds: 16 rows x 32 queries per lane)
constexpr uint32_t kHeadMarkD = 0x80000000u;

// head terms per batch for the dense product: 16 one-sided, 8 two-sided (the sign-split rows take
// twice the TMEM columns); SINN_HEAD_W=8 for A/B runs
inline int doc_head_width(bool lower) {
  const char* e = getenv("SINN_HEAD_W");  // (read per search: tests switch it within one process)
  if (e && atoi(e) == kDocHead) return kDocHead;
  if (e && atoi(e) == kDocHeadWide) return kDocHeadWide;
  return lower ? kDocHead : kDocHeadWide;
}

// shared memory outside the warp slots: theta [kQMax], and with head terms the per-warp decoded
// estimates E+/E- [32 warps][2][hd] (the head query rows Q[hd][kQMax] live in TMEM)
inline size_t doc_fixed_smem(int hd) { return sizeof(float) * kQMax + sizeof(float) * 64 * (size_t)hd; }

int warps_per_cta(int m, bool lower, int hd = 0, bool bf = false, bool single = false) {
  const size_t avail = kSmemBudget - doc_fixed_smem(hd);
  int w = (int)(avail / warp_slot_bytes(m, lower, bf, single));
  w = std::min(w, 32);
  // SINN_DOC_WARPS caps the warps per CTA (the warps-vs-L1 sweep, profiles/r1/sweep_warps_*)
  if (const char* e = getenv("SINN_DOC_WARPS")) w = std::max(1, std::min(w, atoi(e)));
  return w;
}

// a term's 32-byte directory sector in ONE 256-bit load (sm_100 LDG.E.ENL2.256): one L1 request of
// 32 sectors per warp instead of two (the directory is 32-byte aligned: dir[2j], dir[2j+1])
__device__ __forceinline__ void ldg_dir(const uint4* p, uint4& a, uint4& b) {
  asm("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
      : "l"(p));
}

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gsrc));
}
__device__ __forceinline__ void cp_async4(void* sdst, const void* gsrc) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// column of document `id` (U, then L) -> `dst`, asynchronously (one commit group); cells are
// fp32 or, with BF, bfloat16 bits (m % 8 == 0, checked at create)
template <bool LOWER, bool BF>
__device__ __forceinline__ void stage_column(const DocArgs& A, int64_t id, void* dst_, int lane) {
  if (A.raw_val) {  // exact mode reads no sketch (an empty group keeps the wait accounting)
    cp_async_commit();
    return;
  }
  const int m = A.m;
  if (BF) {
    uint16_t* dst = reinterpret_cast<uint16_t*>(dst_);
    const uint4* gu = reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(A.U) + id * m);
    for (int k = lane; k < (m >> 3); k += 32) cp_async16(dst + 8 * k, gu + k);
    if (LOWER) {
      const uint4* gl = reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(A.L) + id * m);
      for (int k = lane; k < (m >> 3); k += 32) cp_async16(dst + m + 8 * k, gl + k);
    }
  } else {
    float* dst = reinterpret_cast<float*>(dst_);
    const float* U = reinterpret_cast<const float*>(A.U);
    const float* L = reinterpret_cast<const float*>(A.L);
    if ((m & 3) == 0) {
      const float4* gu = reinterpret_cast<const float4*>(U + id * m);
      for (int k = lane; k < (m >> 2); k += 32) cp_async16(dst + 4 * k, gu + k);
      if (LOWER) {
        const float4* gl = reinterpret_cast<const float4*>(L + id * m);
        for (int k = lane; k < (m >> 2); k += 32) cp_async16(dst + m + 4 * k, gl + k);
      }
    } else {
      for (int k = lane; k < m; k += 32) cp_async4(dst + k, U + id * m + k);
      if (LOWER)
        for (int k = lane; k < m; k += 32) cp_async4(dst + m + k, L + id * m + k);
    }
  }
  cp_async_commit();
}

// ---- column staging by the tensor memory accelerator's bulk copy (cp.async.bulk, sm_90+): lane 0
// issues one copy per sketch half into the warp's column buffer, completing on the buffer's mbarrier;
// the warp waits on the barrier's phase (no LSU load/store per 16 bytes as with cp.async)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(smem_u32(b)), "r"(parity) : "memory");
  } while (!done);
}
// lane 0 of the warp: the column of document `id` (U, then L) -> dst, completing on barrier b
template <bool LOWER, bool BF>
__device__ __forceinline__ void bulk_column(const DocArgs& A, int64_t id, void* dst, uint64_t* b) {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // the buffer's last generic reads first
  if (A.raw_val) {  // exact mode reads no sketch: complete the phase without data
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
    return;
  }
  const uint32_t half = (uint32_t)A.m * (BF ? 2u : 4u);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(LOWER ? 2 * half : half)
               : "memory");
  const char* gu = reinterpret_cast<const char*>(A.U) + (size_t)id * half;
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)), "l"(gu), "r"(half), "r"(smem_u32(b))
               : "memory");
  if (LOWER) {
    const char* gl = reinterpret_cast<const char*>(A.L) + (size_t)id * half;
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(reinterpret_cast<char*>(dst) + half)), "l"(gl), "r"(half), "r"(smem_u32(b))
                 : "memory");
  }
}

// one 32-entry chunk of a document: entry lane -> term j, its directory sector
struct Chunk {
  uint32_t j;   // 0xffffffff: no entry
  uint4 a, b;   // dir[2j], dir[2j+1]
};

__device__ __forceinline__ Chunk load_chunk(const DocArgs& A, int64_t eb, uint32_t p0, uint32_t cnt, int lane) {
  Chunk c;
  const uint32_t p = p0 + lane;
  c.j = p < cnt ? (__ldg(A.post + eb + p) >> 5) : 0xffffffffu;
  c.a = make_uint4(0, 0, 0, 0);
  c.b = make_uint4(0, 0, 0, 0);
  if (c.j != 0xffffffffu) {
    ldg_dir(A.dir + 2 * (int64_t)c.j, c.a, c.b);
  }
  return c;
}

// H: number of maps (1..4 unrolled from the directory; 0 = generic h read from the pi table).
// LOWER: the index keeps the lower sketch L (false under Sinnamon+).
// HD: 0, kDocHead or kDocHeadWide: the batch's head terms (marked in the directory) only record their
// decoded estimates E+/E- while the document's entries are walked; when the document is complete the
// warp adds sum_hh Q[hh][q] * E(sign)[hh] to every cell (a per-document dense product instead of a
// walk over the head terms' long query lists).  Q sits in TMEM, replicated in the four
// sub-partitions: lane 32p + t, column (k * HD + hh) * 4 + c holds Q[hh][4t + 128k + c] — exactly the
// four queries thread t of any warp handles in round k — so the product reads its Q values with
// tcgen05.ld (16 columns = 4 head terms per load), off the shared-memory pipe, and costs no shared
// memory (round 2: Q in shared memory took 32-64 KB, i.e. 4-8 warps per SM).  With the lower sketch
// the term's columns are split by sign: (k * HD + hh) * 8 + c holds q+ = max(q, 0) and + 4 + c holds
// q- = min(q, 0), so Alg. 6's choice of estimate (lines 7-10) costs no per-cell select:
// s += q+ * E+ + q- * E- (one of the two products is an exact zero).  8 two-sided head terms fill
// the 512 columns.
// CONT: the index has bitmap containers (F3, SINN_BITMAP_CONTAINERS); false compiles the walk without them
template <int MODE, int H, bool LOWER, int HD, bool BF, bool CONT>
__global__ void __launch_bounds__(1024, 1) k_doc_score(DocArgs A) {
  using Cell = typename std::conditional<BF, uint16_t, float>::type;  // sketch cell (F3: bfloat16 bits)
  // two-sided head rows: 8 split by sign (q+ and q- columns, no per-cell choice), or 16 unsplit
  // (Alg. 6's choice by max(fma(q, E+, x), fma(q, E-, x)), E from lane hh by shuffle — no E registers)
  constexpr bool kSplit = LOWER && HD > 0 && HD <= kDocHead;
  constexpr bool kShflE = HD > kDocHead;
  extern __shared__ float4 smem4[];
  __shared__ uint32_t tmem_base_s;
  float* th_s = reinterpret_cast<float*>(smem4);  // [kQMax] theta (EMIT; +inf beyond nqc)
  float* Ew_all = th_s + kQMax;                   // HD > 0: per warp [2][HD] (E+, E-)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, W = blockDim.x >> 5;
  const int m = A.m, h = H > 0 ? H : A.h;
  const bool single = A.single_buf != 0;
  const bool exact = A.raw_val != nullptr;
  const size_t slot = warp_slot_bytes(m, LOWER, BF, single);
  float* Ew = Ew_all + w * 2 * (HD > 0 ? HD : 1);
  int hc = 0;
  uint32_t tq = 0;  // HD > 0: this warp's TMEM lanes (sub-partition w % 4), column 0
  if (HD > 0) {
    hc = (int)*A.head_cnt;
    if (lane < 2 * HD) Ew[lane] = 0.0f;
    if (w == 0) tmem_alloc512(&tmem_base_s);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    tq = tmem_base_s + ((uint32_t)(32 * (w & 3)) << 16);
    if (w < 4) {  // warp p fills sub-partition p (layout: kHeadCols)
      for (int k = 0; k < kQMax / 128; k++)
        for (int g = 0; g < HD; g += (kSplit ? 2 : 4)) {
          float v[16];
#pragma unroll
          for (int t2 = 0; t2 < (kSplit ? 2 : 4); t2++) {
            const float4 q4 = __ldg(reinterpret_cast<const float4*>(A.Qh + (g + t2) * kQMax + 4 * lane + 128 * k));
            if (kSplit) {  // q+ = max(q, 0) then q- = min(q, 0)
              v[8 * t2] = fmaxf(q4.x, 0.0f);
              v[8 * t2 + 1] = fmaxf(q4.y, 0.0f);
              v[8 * t2 + 2] = fmaxf(q4.z, 0.0f);
              v[8 * t2 + 3] = fmaxf(q4.w, 0.0f);
              v[8 * t2 + 4] = fminf(q4.x, 0.0f);
              v[8 * t2 + 5] = fminf(q4.y, 0.0f);
              v[8 * t2 + 6] = fminf(q4.z, 0.0f);
              v[8 * t2 + 7] = fminf(q4.w, 0.0f);
            } else {
              v[4 * t2] = q4.x;
              v[4 * t2 + 1] = q4.y;
              v[4 * t2 + 2] = q4.z;
              v[4 * t2 + 3] = q4.w;
            }
          }
          tmem_st16(tq + (uint32_t)((k * HD + g) * (kSplit ? 8 : 4)), v);
        }
      tmem_wait_st();
    }
    tmem_fence_before();
  }
  char* base = reinterpret_cast<char*>(Ew_all + (HD > 0 ? 32 * 2 * HD : 0)) + (size_t)w * slot;
  float* S = reinterpret_cast<float*>(base);
  // conflict detection for the lane = entry rounds: a tag byte per query (claim bits, kClaimBits,
  // were the head-heavy instantiation's way to save shared memory while Q sat there)
  constexpr bool kClaimBits = false;
  uint8_t* tag = reinterpret_cast<uint8_t*>(S + kQMax);
  uint32_t* claim = reinterpret_cast<uint32_t*>(S + kQMax);  // [kQMax / 32]
  Cell* colbuf = reinterpret_cast<Cell*>(tag + (kClaimBits ? kQMax / 8 : kQMax));  // 2 (or 1) x col_cells
  uint64_t* mbar = reinterpret_cast<uint64_t*>(base + slot - 16);  // [2]: the column buffers' barriers
  // bulk copies (opt-in, SINN_TMA=1) need 16-byte halves (m % 4 == 0 fp32, m % 8 == 0 bfloat16)
  const bool tma = A.tma && ((size_t)m * sizeof(Cell)) % 16 == 0;
  uint32_t use0 = 0, use1 = 0;  // bulk copies issued into buffer 0 / 1 (phase k completes copy k)
  if (lane == 0) {
    mbar_init(mbar);
    mbar_init(mbar + 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  // stage document id's column into buffer b (0: colbuf, 1: colbuf + cf); wait for the buffer in use
  auto stage_b = [&](int b, int64_t id) {
    if (tma) {
      if (lane == 0) bulk_column<LOWER, BF>(A, id, colbuf + (b ? col_cells(m, LOWER) : 0), mbar + b);
      if (b) use1++; else use0++;
    } else {
      stage_column<LOWER, BF>(A, id, colbuf + (b ? col_cells(m, LOWER) : 0), lane);
    }
  };
  const int cf = (int)col_cells(m, LOWER);
  const int nqc = A.nqc;
  if (MODE == kModeEmit)
    for (int q = threadIdx.x; q < kQMax; q += blockDim.x) th_s[q] = q < nqc ? A.theta[q] : INFINITY;
  else  // HIST: a positive floor from a smaller nested sample (cells below it cannot be its k'-th)
    for (int q = threadIdx.x; q < kQMax; q += blockDim.x) {
      const float f = (A.theta && q < nqc) ? A.theta[q] : -INFINITY;
      th_s[q] = f > 0.0f ? f : -INFINITY;
    }
  for (int q = lane; q < kQMax; q += 32) S[q] = __uint_as_float(kNegZeroBits);
  if (kClaimBits) claim[lane] = 0u;  // kQMax / 32 == 32 words
  // without head rows TMEM is free: theta goes there (lane 32p + t, column 4k + c: theta of query
  // 4t + 128k + c, the cells thread t compares in round k), so the document-completion scan reads
  // it with tcgen05.ld instead of a 128-bit shared load per four cells (off the L1 data pipe)
  uint32_t tth = 0;
  if (HD == 0) {
    if (w == 0) tmem_alloc32(&tmem_base_s);
    tmem_fence_before();
    __syncthreads();  // (th_s written above)
    tmem_fence_after();
    tth = tmem_base_s + ((uint32_t)(32 * (w & 3)) << 16);
    if (w < 4) {
      float v[16];
#pragma unroll
      for (int half = 0; half < 2; half++) {
#pragma unroll
        for (int k2 = 0; k2 < 4; k2++) {
          const float4 t4 = reinterpret_cast<const float4*>(th_s)[(4 * lane + 128 * (4 * half + k2)) >> 2];
          v[4 * k2] = t4.x;
          v[4 * k2 + 1] = t4.y;
          v[4 * k2 + 2] = t4.z;
          v[4 * k2 + 3] = t4.w;
        }
        tmem_st16(tth + (uint32_t)(16 * half), v);
      }
      tmem_wait_st();
    }
    tmem_fence_before();
  }
  __syncthreads();
  tmem_fence_after();
  const int parts = A.parts, per_part = kTile / parts;
  uint32_t nsampled = 0;  // HIST: live documents scored by this warp
  const int64_t gw = (int64_t)blockIdx.x * W + w, GW = (int64_t)gridDim.x * W;
  const int64_t units = A.ntiles * parts;
  // work units (tile parts) are handed out by an atomic counter, so a warp that drew short
  // documents takes more and the launch ends when the work does (c3 score -4%); a null counter
  // falls back to static striding
  int64_t u_static = gw;
  auto take_unit = [&]() -> int64_t {
    if (!A.sched) {
      const int64_t v = u_static;
      u_static += GW;
      return v;
    }
    uint32_t v = 0;
    if (lane == 0) v = atomicAdd(A.sched, 1u);
    return (int64_t)__shfl_sync(kFull, v, 0);
  };
  for (int64_t u = take_unit(); u < units; u = take_unit()) {
    const int64_t t = (u / parts) * A.stride;
    if (MODE == kModeEmit && A.skip > 1 && t % A.skip == 0) continue;  // scored by the sample pass (A.rows)
    const int d0 = (int)(u % parts) * per_part;
    const int64_t i_lane = t * kTile + lane;
    const bool lv = A.live[i_lane] != 0;
    const uint32_t c_lane = (uint32_t)A.nnz[i_lane];  // entries stored (a deleted id's tombstones included)
    uint32_t inc = c_lane;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, inc, d);
      if (lane >= d) inc += y;
    }
    const uint32_t start_lane = inc - c_lane;
    const uint32_t partmask = per_part == 32 ? kFull : (((1u << per_part) - 1u) << d0);
    // constrained search: masked-out documents are skipped like vacant ones (their entries still
    // count in the offsets above)
    const uint32_t amask = A.allow ? (t < A.allow_words ? __ldg(A.allow + t) : 0u) : kFull;
    uint32_t todo = __ballot_sync(kFull, lv) & partmask & amask;
    if (!todo) continue;
    const int64_t tbase = A.toff[t];
    // bitmap containers of the tile (F3): lane L holds container L (term, document mask); a document
    // with container bits walks them first, as one virtual chunk of 32 entries (lane L: term L if the
    // document's bit is set), then its stored entries
    const int cn = CONT ? (int)A.cnum[t] : 0;
    uint2 cv = make_uint2(0u, 0u);
    if (CONT && lane < cn) cv = __ldg(A.cont + t * kTile + lane);
    // pipeline over the unit's (document, chunk) sequence, three chunks deep: while chunk c0 is
    // processed, the directory sectors of c1 and the entries of c2 are in flight, and the next
    // document's sketch column streams into the other column buffer (cp.async)
    // pipeline stage: a (document, chunk) with the document's entry count and first entry (both
    // warp-uniform, shuffled once per document)
    struct Stage {
      int d;        // document within the tile, -1: none
      uint32_t p;   // first entry of the chunk (virtual: the container chunk, if any, is 0..31)
      uint32_t c;   // the document's entry count, + 32 with container bits
      uint32_t e0;  // the document's first entry, relative to the tile's
      uint32_t cb;  // lanes whose container holds the document (0: no container chunk)
    };
    auto doc_stage = [&](int dd) {
      Stage st;
      st.d = dd;
      st.p = 0;
      const int src = dd < 0 ? 0 : dd;
      st.c = __shfl_sync(kFull, c_lane, src);
      st.e0 = __shfl_sync(kFull, start_lane, src);
      st.cb = cn ? __ballot_sync(kFull, dd >= 0 && ((cv.y >> src) & 1u)) : 0u;
      if (st.cb) st.c += 32;
      return st;
    };
    auto next_doc = [&]() {
      const int dd = todo ? __ffs(todo) - 1 : -1;
      if (dd >= 0) todo &= todo - 1;
      return dd;
    };
    // raw entry ((j << 5) | d), 0xffffffff past the document; the shift is left to the consumer so
    // that the load is not waited on where it is issued
    auto entry_raw = [&](const Stage& st) -> uint32_t {
      uint32_t v = 0xffffffffu;
      if (st.d >= 0) {
        if (st.cb && st.p == 0) {
          if ((st.cb >> lane) & 1u) v = (cv.x << 5) | (uint32_t)st.d;
        } else if (st.p + lane < st.c) {
          v = __ldg(A.post + tbase + (st.e0 + st.p - (st.cb ? 32u : 0u) + lane));
        }
      }
      return v;
    };
    auto term_of = [](uint32_t v) { return v == 0xffffffffu ? v : v >> 5; };
    auto advance = [&](const Stage& st) {  // (warp-uniform)
      if constexpr (HD == 0) {  // one branch (fewer instructions; the head variants keep the form
                                // that fits their registers without spills)
        Stage n = st;
        n.p += 32;
        if (st.d >= 0 && n.p >= st.c) n = doc_stage(next_doc());
        return n;
      } else {
        if (st.d < 0) return st;
        if (st.p + 32 < st.c) {
          Stage n = st;
          n.p += 32;
          return n;
        }
        return doc_stage(next_doc());
      }
    };
    Stage s0 = doc_stage(next_doc());
    int coff = 0;  // the current column's offset in colbuf (0 or cf; always 0 with one buffer)
    stage_b(0, t * kTile + s0.d);
    Chunk cur;
    cur.j = term_of(entry_raw(s0));
    cur.a = make_uint4(0, 0, 0, 0);
    cur.b = make_uint4(0, 0, 0, 0);
    if (cur.j != 0xffffffffu) {
      ldg_dir(A.dir + 2 * (int64_t)cur.j, cur.a, cur.b);
    }
    Stage s1 = advance(s0);
    uint32_t r1 = entry_raw(s1);
    if (!single && s1.d >= 0 && s1.d != s0.d) stage_b(1, t * kTile + s1.d);
    Stage s2 = advance(s1);
    int d = s0.d, d1 = s1.d;
    uint32_t p0 = s0.p;
    while (true) {
      const bool newdoc = d1 != d;
      // directory sectors of c1, entries of c2
      Chunk nxt;
      nxt.j = term_of(r1);
      nxt.a = make_uint4(0, 0, 0, 0);
      nxt.b = make_uint4(0, 0, 0, 0);
      if (nxt.j != 0xffffffffu) {
        ldg_dir(A.dir + 2 * (int64_t)nxt.j, nxt.a, nxt.b);
      }
      const uint32_t r2 = entry_raw(s2);
      if (tma) {  // the current document's buffer: its latest copy's phase
        if (coff) mbar_wait(mbar + 1, (use1 - 1) & 1u);
        else mbar_wait(mbar, (use0 - 1) & 1u);
      } else if (!single && newdoc && d1 >= 0) {
        cp_async_wait<1>();  // a newer column (d1's) may stay in flight
      } else {
        cp_async_wait<0>();
      }
      __syncwarp();
      const Cell* colU = colbuf + coff;
      const Cell* colL = colU + m;
      // ---- process the current chunk
      const uint32_t qb = cur.a.x;
      uint32_t nr = (cur.a.y & 0x3fffffffu) - qb;
      float eu = 0.0f, el = 0.0f;
      const bool headent = HD > 0 && (cur.b.x & kHeadMarkD) != 0;
      if (HD == 0 ? exact : A.raw_val != nullptr) {  // exact scoring (Alg. 2, LinScan): the stored value
        if (nr > 0) {
          const int64_t ro = A.raw_off[t * kTile + d];
          if (!CONT) {  // the document's entries and its raw row are in the same term order
            eu = el = __ldg(A.raw_val + ro + p0 + lane);
          } else {  // with containers they are not: binary search of the term in the row
            const int32_t* ri = A.raw_idx + ro;
            int32_t lo = 0, hi = A.raw_nnz[t * kTile + d];
            while (lo < hi) {
              const int32_t mid = (lo + hi) >> 1;
              if (__ldg(ri + mid) < (int32_t)cur.j) lo = mid + 1; else hi = mid;
            }
            eu = el = __ldg(A.raw_val + ro + lo);
          }
        }
      } else if (nr > 0 || headent) {
        const uint32_t j = cur.j;
        const uint4 dd = cur.a;
        // pi_o(j): packed in the directory for h <= 4, else from the table
        auto cell = [&](int o) -> int {
          if (H == 0) return (int)__ldg(A.pi + (int64_t)j * h + o);
          const uint32_t wv = o < 2 ? dd.z : dd.w;
          return (int)((o & 1) ? (wv >> 16) : (wv & 0xffffu));
        };
        if (dd.y & (1u << 30)) eu = decode_upper_by(colU, h, cell);
        if (LOWER && (dd.y & (1u << 31))) el = decode_lower_by(colL, h, cell);
      }
      if (single && newdoc && d1 >= 0) {  // the document's last decode is done: stage the next column
        __syncwarp();
        stage_b(0, t * kTile + d1);
      }
      if (headent) {  // head term: record the estimates; no walk over its queries
        const int hh = (int)(cur.b.x & 0xffffu);
        Ew[hh] = eu;
        if (LOWER) Ew[HD + hh] = el;
      }
      // wide terms: the whole warp walks the term's queries (distinct queries: no conflicts)
      uint32_t wide = __ballot_sync(kFull, nr > (uint32_t)kNarrowMax);
      // the estimate a query value multiplies: upper for q_j > 0, lower otherwise; without a lower
      // sketch (Sinnamon+) S0 keeps only q_j > 0, and exact mode passes the stored value as both
      auto sgn_est = [](float v, float u, float l) { return LOWER ? (v > 0.0f ? u : l) : u; };
      auto wide_rmw = [&](uint2 pr, uint32_t r, uint32_t nn, float wu, float wl) {
        if (r < nn) {
          const float v = __uint_as_float(pr.y);
          S[pr.x] = __fadd_rn(S[pr.x], __fmul_rn(v, sgn_est(v, wu, wl)));
        }
      };
      while (wide) {
        const int src = __ffs(wide) - 1;
        wide &= wide - 1;
        const uint32_t b = __shfl_sync(kFull, qb, src), nn = __shfl_sync(kFull, nr, src);
        const float wu = __shfl_sync(kFull, eu, src), wl = __shfl_sync(kFull, el, src);
        // four pair loads per lane in flight before the read-modify-writes (L2 latency); the
        // term's pairs are placed bank-major by S0, so a warp's 32 cells mostly sit in distinct banks
        if (nn <= 64) {  // up to two passes: both loads in flight, no idle 4-pass body
          const uint32_t r = lane;
          const uint2 p1 = r < nn ? __ldg(A.pairs + b + r) : make_uint2(0, 0);
          const uint2 p2 = r + 32 < nn ? __ldg(A.pairs + b + r + 32) : make_uint2(0, 0);
          // a second short term: its loads join the first's, one L2 round trip for both
          const int src2 = wide ? __ffs(wide) - 1 : 0;
          const uint32_t nn2 = wide ? __shfl_sync(kFull, nr, src2) : 0u;
          if (nn2 > 0 && nn2 <= 64) {
            wide &= wide - 1;
            const uint32_t b2 = __shfl_sync(kFull, qb, src2);
            const float wu2 = __shfl_sync(kFull, eu, src2), wl2 = __shfl_sync(kFull, el, src2);
            const uint2 q1 = r < nn2 ? __ldg(A.pairs + b2 + r) : make_uint2(0, 0);
            const uint2 q2 = r + 32 < nn2 ? __ldg(A.pairs + b2 + r + 32) : make_uint2(0, 0);
            wide_rmw(p1, r, nn, wu, wl);
            wide_rmw(p2, r + 32, nn, wu, wl);
            __syncwarp();  // the two terms may share a query
            wide_rmw(q1, r, nn2, wu2, wl2);
            wide_rmw(q2, r + 32, nn2, wu2, wl2);
          } else {
            wide_rmw(p1, r, nn, wu, wl);
            wide_rmw(p2, r + 32, nn, wu, wl);
          }
        } else {
          for (uint32_t r = lane; r < nn; r += 128) {
            uint2 pr[4];
#pragma unroll
            for (int u = 0; u < 4; u++)
              pr[u] = r + 32 * u < nn ? __ldg(A.pairs + b + r + 32 * u) : make_uint2(0, 0);
#pragma unroll
            for (int u = 0; u < 4; u++) wide_rmw(pr[u], r + 32 * u, nn, wu, wl);
          }
        }
        __syncwarp();
      }
      if (nr > (uint32_t)kNarrowMax) nr = 0;
      // narrow terms: lane = entry, serial over the term's queries (the first three inline in the
      // directory, the rest prefetched one ahead); lanes hitting the same query in one round are
      // serialised through the tag array
      const uint32_t maxr = __reduce_max_sync(kFull, nr);
      // one update round: lanes with pend add cval into S[q]; lanes holding the same query are
      // serialised through the tag array (a query sharing two terms with the document)
      // branch-free: every lane loads (q is a valid cell even when idle), only pending winners store
      auto update = [&](bool pend, uint32_t q, float cval) {
        if (kClaimBits) {  // one bit per query, claimed with atomicOr (frees 7/8 of the tag bytes)
        q &= (kQMax - 1);
          const uint32_t bit = 1u << (q & 31);
          uint32_t* word = claim + (q >> 5);
          bool win = false;
          if (pend) win = (atomicOr(word, bit) & bit) == 0;  // first claim of q this round wins
          float x = __fadd_rn(S[q], cval);
          if (win) S[q] = x;
          __syncwarp();
          if (win) atomicAnd(word, ~bit);  // release for the next round
          pend = pend && !win;
          __syncwarp();
          while (__any_sync(kFull, pend)) {
            win = false;
            if (pend) win = (atomicOr(word, bit) & bit) == 0;
            x = __fadd_rn(S[q], cval);
            if (win) S[q] = x;
            __syncwarp();
            if (win) atomicAnd(word, ~bit);
            pend = pend && !win;
            __syncwarp();
          }
        } else {  // one tag byte per query
        q &= (kQMax - 1);
          if (pend) tag[q] = (uint8_t)lane;
          __syncwarp();
          bool win = pend && tag[q] == (uint8_t)lane;
          float x = __fadd_rn(S[q], cval);
          if (win) S[q] = x;
          pend = pend && !win;
          __syncwarp();
          while (__any_sync(kFull, pend)) {
            if (pend) tag[q] = (uint8_t)lane;
            __syncwarp();
            win = pend && tag[q] == (uint8_t)lane;
            x = __fadd_rn(S[q], cval);
            if (win) S[q] = x;
            pend = pend && !win;
            __syncwarp();
          }
        }
      };
      // a narrow term's fourth pair: its load issued before the inline rounds, which hide its latency
      uint2 pf = make_uint2(0, 0);
      if (nr > 3) pf = __ldg(A.pairs + qb + 3);
      if (maxr > 0) {  // first query of each term (inline in the directory)
        const float v = __uint_as_float(cur.b.y);
        update(nr > 0, cur.b.x & 0x3ffu, __fmul_rn(v, sgn_est(v, eu, el)));
      }
      if (maxr > 1) {  // second query (inline)
        const float v = __uint_as_float(cur.b.z);
        update(nr > 1, (cur.b.x >> 10) & 0x3ffu, __fmul_rn(v, sgn_est(v, eu, el)));
      }
      if (maxr > 2) {  // third query (inline)
        const float v = __uint_as_float(cur.b.w);
        update(nr > 2, (cur.b.x >> 20) & 0x3ffu, __fmul_rn(v, sgn_est(v, eu, el)));
      }
      if (maxr > 3) {  // the rest from the pair table, prefetched one ahead
        for (uint32_t r = 3; r < maxr; r++) {
          const uint2 pr = pf;
          if (r + 1 < nr) pf = __ldg(A.pairs + qb + r + 1);
          const float v = __uint_as_float(pr.y);
          update(r < nr, pr.x, __fmul_rn(v, sgn_est(v, eu, el)));
        }
      }
      if (newdoc) {
        // ---- document d complete: compare every cell with theta_q (or find the non-zero ones to
        // histogram); lane L owns cells 4L + 128k + c; the qualifying cells are collected in a bit
        // mask and handled by all lanes together; the scan resets every other cell to the sentinel
        // (the emission loop resets the qualifying ones)
        nsampled++;
        const uint32_t uid = (uint32_t)(t * kTile + d);
        uint32_t em = 0;
        float ep[HD > 0 && !kShflE ? HD : 1], en[HD > 0 && !kShflE ? HD : 1];
        float ep_l = 0.0f, en_l = 0.0f;  // kShflE: lane hh holds term hh's E+ / E-
        if (HD > 0) {
          __syncwarp();
          if constexpr (kShflE) {
            if (lane < HD) {
              ep_l = Ew[lane];
              en_l = LOWER ? Ew[HD + lane] : 0.0f;
            }
          } else {
#pragma unroll
            for (int hh = 0; hh < HD; hh++) {
              ep[hh] = Ew[hh];
              en[hh] = LOWER ? Ew[HD + hh] : 0.0f;
            }
          }
          __syncwarp();
          if (lane < 2 * HD) Ew[lane] = 0.0f;  // for the next document
        }
        const float4 sent = make_float4(-0.0f, -0.0f, -0.0f, -0.0f);
#pragma unroll
        for (int k = 0; k < kQMax / 128; k++) {
          const int q0 = 4 * lane + 128 * k;
          float4 x4 = reinterpret_cast<const float4*>(S)[q0 >> 2];
          if (HD > 0) {  // dense head product for these four queries (Q from TMEM, four terms per load)
            // terms per TMEM load (16 columns): 4, or 2 sign-split terms with the lower sketch
            constexpr int TPL = kSplit ? 1 : 4;
#pragma unroll
            for (int g = 0; g < HD; g += TPL) {
              if (g >= hc) break;
              float qv[kSplit ? 8 : 16];
              if constexpr (kSplit) tmem_ld8(tq + (uint32_t)((k * HD + g) * 8), qv);
              else tmem_ld16(tq + (uint32_t)((k * HD + g) * 4), qv);
              tmem_wait_ld();
#pragma unroll
            for (int t2 = 0; t2 < TPL; t2++) {
              const int hh = g + t2;
              if (hh < hc) {
                if (kShflE && !LOWER) {  // Sinnamon+: Q >= 0, the upper estimate only
                  const float eu = __shfl_sync(kFull, ep_l, hh);
                  const float2 e2 = make_float2(eu, eu);
                  const float2 lo = __ffma2_rn(make_float2(qv[4 * t2], qv[4 * t2 + 1]), e2, make_float2(x4.x, x4.y));
                  const float2 hi = __ffma2_rn(make_float2(qv[4 * t2 + 2], qv[4 * t2 + 3]), e2, make_float2(x4.z, x4.w));
                  x4 = make_float4(lo.x, lo.y, hi.x, hi.y);
                } else if (kShflE) {  // max(fma(q, E+, x), fma(q, E-, x)) = fma(q, E(sign q), x): E+ >= x_ij >= E- 
                  const float eu = __shfl_sync(kFull, ep_l, hh), el = __shfl_sync(kFull, en_l, hh);
                  const float* qp = qv + 4 * t2;
                  const float2 eu2 = make_float2(eu, eu), el2 = make_float2(el, el);
                  const float2 xl = make_float2(x4.x, x4.y), xh = make_float2(x4.z, x4.w);
                  const float2 q01 = make_float2(qp[0], qp[1]), q23 = make_float2(qp[2], qp[3]);
                  const float2 a = __ffma2_rn(q01, eu2, xl), b = __ffma2_rn(q01, el2, xl);
                  const float2 c = __ffma2_rn(q23, eu2, xh), d = __ffma2_rn(q23, el2, xh);
                  x4 = make_float4(fmaxf(a.x, b.x), fmaxf(a.y, b.y), fmaxf(c.x, d.x), fmaxf(c.y, d.y));
                } else if (kSplit) {  // x += q+ E+ then q- E- (FFMA2: two round-to-nearest FMAs, as fmaf)
                  const float* qp = qv + 8 * t2;
                  const float2 ep2 = make_float2(ep[hh], ep[hh]), en2 = make_float2(en[hh], en[hh]);
                  float2 lo = __ffma2_rn(make_float2(qp[0], qp[1]), ep2, make_float2(x4.x, x4.y));
                  float2 hi = __ffma2_rn(make_float2(qp[2], qp[3]), ep2, make_float2(x4.z, x4.w));
                  lo = __ffma2_rn(make_float2(qp[4], qp[5]), en2, lo);
                  hi = __ffma2_rn(make_float2(qp[6], qp[7]), en2, hi);
                  x4 = make_float4(lo.x, lo.y, hi.x, hi.y);
                } else {
                  const float4 v4 = make_float4(qv[4 * t2], qv[4 * t2 + 1], qv[4 * t2 + 2], qv[4 * t2 + 3]);  // Sinnamon+: S0 drops negative q_j, so Q >= 0 and only the upper estimate is used
                  // (packed FFMA2 on sm_100: two independent round-to-nearest FMAs, as fmaf)
                  const float2 e2 = make_float2(ep[hh], ep[hh]);
                  const float2 lo = __ffma2_rn(make_float2(v4.x, v4.y), e2, make_float2(x4.x, x4.y));
                  const float2 hi = __ffma2_rn(make_float2(v4.z, v4.w), e2, make_float2(x4.z, x4.w));
                  x4 = make_float4(lo.x, lo.y, hi.x, hi.y);
                }
              }
            }
            }
          }
          if (MODE == kModeHist && A.rows)  // the sampled document's row, for k_emit_rows (coalesced 16-byte stores)
            reinterpret_cast<float4*>(A.rows + ((t / A.stride) * kTile + d) * (int64_t)kQMax)[q0 >> 2] = x4;
          uint32_t e4;
          float4 t4;
          if (HD == 0) {
            float tv[4];
            tmem_ld4(tth + (uint32_t)(4 * k), tv);
            tmem_wait_ld();
            t4 = make_float4(tv[0], tv[1], tv[2], tv[3]);
          } else {
            t4 = reinterpret_cast<const float4*>(th_s)[q0 >> 2];
          }
          if (MODE == kModeEmit) {
            // -0.0 (untouched) compares equal to +0.0
            e4 = (x4.x >= t4.x ? 1u : 0u) | (x4.y >= t4.y ? 2u : 0u) | (x4.z >= t4.z ? 4u : 0u) |
                 (x4.w >= t4.w ? 8u : 0u);
          } else {
            e4 = (x4.x != 0.0f && x4.x >= t4.x ? 1u : 0u) | (x4.y != 0.0f && x4.y >= t4.y ? 2u : 0u) |
                 (x4.z != 0.0f && x4.z >= t4.z ? 4u : 0u) | (x4.w != 0.0f && x4.w >= t4.w ? 8u : 0u);
          }
          em |= e4 << (4 * k);
          // qualifying cells keep their score for the emission loop (which resets them), the others
          // are reset here
          reinterpret_cast<float4*>(S)[q0 >> 2] =
              e4 ? make_float4((e4 & 1u) ? x4.x : sent.x, (e4 & 2u) ? x4.y : sent.y, (e4 & 4u) ? x4.z : sent.z,
                               (e4 & 8u) ? x4.w : sent.w)
                 : sent;
        }
        __syncwarp();
        while (__any_sync(kFull, em)) {
          if (em) {
            const int b = __ffs(em) - 1;
            em &= em - 1;
            const uint32_t q = 4 * lane + 128 * (b >> 2) + (b & 3);
            float x = S[q];
            S[q] = __uint_as_float(kNegZeroBits);
            if (x == 0.0f) x = 0.0f;  // -0.0 -> +0.0 (R19)
            if ((int)q >= nqc || !qmask_pass(A.qm, q, uid)) continue;  // (F4: masked out for this query)
            if (MODE == kModeEmit) emit(A, q, x, uid);
            else atomicAdd(&A.hist[(int64_t)q * kThetaBins + (f2key(x) >> kThetaShift)], 1u);
          }
        }
        __syncwarp();
        coff = single ? 0 : cf - coff;
      }
      if (d1 < 0) break;
      // rotate: c1 -> c0, c2 -> c1; a new document entering c1 gets its column staged
      cur = nxt;
      s0 = s1;
      s1 = s2;
      r1 = r2;
      d = s0.d;
      p0 = s0.p;
      d1 = s1.d;
      if (!single && d1 >= 0 && d1 != d)
        stage_b(coff ? 0 : 1, t * kTile + d1);
      s2 = advance(s1);
    }
  }
  if (MODE == kModeHist && lane == 0 && nsampled) atomicAdd(A.nsampled, nsampled);
  // every warp's last TMEM read is done before the allocating warp frees the columns
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (w == 0) {
    if (HD > 0) tmem_dealloc512(tmem_base_s);
    else tmem_dealloc32(tmem_base_s);
  }
}

int num_sms() { return sm_count(); }

// launcher of k_doc_score for one sketch-cell type (BF: bfloat16, F3); A fully set up except parts
template <bool BF>
void launch_doc_score_tpl(bool emit, DocArgs A, bool lower, bool head, cudaStream_t s) {
  const int m = A.m, h = A.h;
  cudaMemsetAsync(A.sched, 0, sizeof(uint32_t), s);
  // the head width is chosen on the fp32 slot size for both cell types (the same head split for a
  // bfloat16 index; its smaller slot would admit 16 head terms where they do not pay, config 5)
  const int HDv = head ? doc_head_width(lower) : 0;
  // one column buffer per warp whenever the second would cost a warp per SM: the extra warps hide
  // more latency than the earlier column staging does (config 5: 21 -> 27 warps, score -18 %;
  // config 2: 31 -> 32, -3 %; config 3: 28 -> 29, -1 %).  SINN_SINGLE_BUF=0/1 forces either.
  const int sb_env = getenv("SINN_SINGLE_BUF") ? atoi(getenv("SINN_SINGLE_BUF")) : -1;
  const bool single = sb_env >= 0 ? sb_env != 0
                                  : warps_per_cta(m, lower, HDv, BF, true) > warps_per_cta(m, lower, HDv, BF);
  A.single_buf = single ? 1 : 0;
  const int W = warps_per_cta(m, lower, HDv, BF, single);
  // split tiles into parts while there are fewer than 4 work units per warp (the sample pass: a
  // sampled tile's 32 documents are spread over several warps; config 3 sample pass -8 % vs 2)
  static const int64_t parts_env = getenv("SINN_PARTS_X") ? atoi(getenv("SINN_PARTS_X")) : 0;
  // the full pass with head terms spends ~75 K clocks per document and warp (config 5), so a 32-document
  // unit is 1.2 ms of one warp: quarter tiles shorten the tail of the dynamic schedule (config 5 full
  // pass -1.1 %); without head terms (configs 2, 4) a document is cheap and the tile header is not
  const bool heavy = emit && HDv > 0;
  const int64_t parts_x = parts_env ? parts_env : (heavy ? 80 : 4);
  const int parts_max = (heavy && !parts_env) ? 4 : kTile;
  while (A.parts < parts_max && A.ntiles * A.parts < parts_x * num_sms() * W) A.parts *= 2;
  size_t smem = doc_fixed_smem(HDv) + (size_t)W * warp_slot_bytes(m, lower, BF, single);
  // a CTA with head terms owns all 512 TMEM columns: one CTA per SM (a second one would wait in
  // tcgen05.alloc until the first exits)
  if (HDv > 0) smem = std::max<size_t>(smem, kSmemBudget / 2 + 1024);
  const int H = h <= 4 ? h : 0;
  auto go = [&](void (*kern)(DocArgs), int, int, int, int) {
    smem_optin((const void*)kern);
    const int64_t ctas_needed = (A.ntiles * A.parts + W - 1) / W;
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(num_sms(), ctas_needed));
    kern<<<grid, W * 32, smem, s>>>(A);
  };
#define SINN_DOC_CASE(MO, HH, LO)                                                                          \
  if ((emit ? kModeEmit : kModeHist) == MO && H == HH && lower == LO) {                                    \
    if (ct) {                                                                                              \
      if (HDv == kDocHeadWide) return go(k_doc_score<MO, HH, LO, kDocHeadWide, BF, true>, MO, HH, LO, 2);  \
      if (HDv) return go(k_doc_score<MO, HH, LO, kDocHead, BF, true>, MO, HH, LO, 1);                      \
      return go(k_doc_score<MO, HH, LO, 0, BF, true>, MO, HH, LO, 0);                                      \
    }                                                                                                      \
    if (HDv == kDocHeadWide) return go(k_doc_score<MO, HH, LO, kDocHeadWide, BF, false>, MO, HH, LO, 2);  \
    if (HDv) return go(k_doc_score<MO, HH, LO, kDocHead, BF, false>, MO, HH, LO, 1);                       \
    return go(k_doc_score<MO, HH, LO, 0, BF, false>, MO, HH, LO, 0);                                       \
  }
  const bool ct = A.cont != nullptr;
#define SINN_DOC_H(MO, LO) \
  SINN_DOC_CASE(MO, 0, LO) SINN_DOC_CASE(MO, 1, LO) SINN_DOC_CASE(MO, 2, LO) SINN_DOC_CASE(MO, 3, LO) \
  SINN_DOC_CASE(MO, 4, LO)
  SINN_DOC_H(kModeHist, false)
  SINN_DOC_H(kModeHist, true)
  SINN_DOC_H(kModeEmit, false)
  SINN_DOC_H(kModeEmit, true)
#undef SINN_DOC_H
#undef SINN_DOC_CASE
}

}  // namespace

}  // namespace sinn
