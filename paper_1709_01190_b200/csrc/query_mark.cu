// query_mark.cu — Q1-Q3 by an occupancy bitmap over the id range (sm_100a), for indexes
// whose ids fit a shared-memory bitmap (max_id < 8 * kMarkMaxBitmapBytes).
//
// What the top-k needs (Alg. 3; R#11-R#13): every id seen at least twice, with
// its full multiplicity, and — when fewer than k ids repeat — the smallest `need` ids seen
// exactly once (ties at count 1 go by ascending id).  On the webspam graph a query has
// ~1,060 candidates of which ~80 are repeats of ~4 ids (a near-duplicate family seen in
// most of the L tables), and the 124-odd surviving singletons are the smallest ids, so a
// full sort of the candidates (query_sort.cu) does mostly unneeded work.  Instead, one
// CTA owns one query at a time (persistent over the queries):
//   Q1 gather   thread t < L holds bucket t's extent (loaded during the previous query); a
//               scan gives each non-empty bucket's first flattened position: a start bitmap
//               over the positions, the number of starts below each of its words, and one
//               base pointer per bucket, so position p's bucket is a popc away; 32-position
//               blocks go round-robin to the warps, 4 loads in flight per lane.
//   Q2 count    each candidate sets its bit in the id bitmap with one shared-memory
//               atomicOr; a bit already set means a repeat, and only repeats go to a small
//               open-addressing table (id -> extra occurrences; new slots are listed).
//               Full multiplicity = 1 + extra (R#11).  The excluded id (self, R#14) is
//               dropped at the gather.
//   Q3 top-k    warp 0 compacts the listed repeated ids into (count desc, id asc) keys and
//               clears their bits, so the bitmap holds exactly the singletons, and ranks
//               them by counting; the CTA then scans the bitmap from id 0 (2,048 words per
//               round, a block scan of the per-thread bit counts) writing the first `need`
//               set bits in ascending order (R#12); pads (EMPTY, 0) fill the rest (R#13).
//   reset       the bitmap words of the staged candidates (their u16 word indices, M <=
//               kStage; else the whole bitmap) and the listed table slots.
// A query with more than kRepMax distinct repeated ids (or a probe sequence longer than
// kRepProbes) is appended to a fallback list and answered by the CTA sort kernel
// (k_query_csort) afterwards; the results do not depend on which kernel answers a query
// (both compute the same (count desc, id asc) top-k).
#include <cstdlib>

#include "flash_internal.cuh"

namespace flash {
namespace {

constexpr int kMarkThreads = 256;
constexpr uint32_t kMarkWarps = kMarkThreads / 32;
constexpr uint32_t kConsWarps = kMarkWarps - 1;  // consumer warps (Q2-Q3); the last warp is the producer (Q1)
constexpr uint32_t kConsThreads = kConsWarps * 32;
constexpr uint32_t kRepLog2 = 8;
constexpr uint32_t kRepSlots = 1u << kRepLog2;  // open-addressing table of repeated ids
constexpr uint32_t kRepMax = 112;               // distinct repeated ids ranked here (more: fallback)
constexpr uint32_t kRepProbes = 32;             // a longer probe sequence also falls back
constexpr uint32_t kMarkMaxL = 128;             // Q1: one thread per bucket, 8-bit bucket ranks
constexpr uint32_t kStage = 2048;               // candidates staged for the bitmap reset
constexpr uint32_t kScanWpt = 8;                // bitmap words per thread per scan round
constexpr size_t kMarkMaxBitmapBytes = 96 * 1024;  // >= 2 CTAs per SM (and u16 word indices)
constexpr uint32_t kMarkMinCandidates = 768;     // fewer: the size-class sort kernels

#ifdef FLASH_QPROF  // per-phase cycle counters of thread 0 (diagnostic builds only: build.py --qprof)
__device__ unsigned long long g_mprof[8];
#define MMARK(i)                                                                 \
  do {                                                                           \
    const long long now_ = clock64();                                            \
    if (tid == 0) atomicAdd(&g_mprof[i], (unsigned long long)(now_ - mp_last)); \
    mp_last = now_;                                                              \
  } while (0)
#else
#define MMARK(i) \
  do {           \
  } while (0)
#endif

struct MarkHdr {
  uint32_t nrep, overflow;
  uint32_t M[2], excl[2];  // per query buffer (Q1 output): candidates, excluded id
  uint64_t q[2];           // and the query's index
  uint32_t rsum[2][kConsWarps];
};

__host__ __device__ inline uint32_t mark_words(uint32_t max_id) {  // bitmap words, multiple of 128
  const uint64_t bits = (uint64_t)max_id + 1;
  return (uint32_t)(((bits + 32 * 128 - 1) / (32 * 128)) * 128);
}
__host__ __device__ inline uint32_t mark_bmap_words(uint64_t mmax) { return (uint32_t)((mmax / 32 + 2 + 7) & ~7ull); }
__host__ __device__ inline uint32_t mark_stage(uint64_t mmax) {
  return mmax < kStage ? (uint32_t)((mmax + 7) & ~7ull) : kStage;
}

__host__ __device__ inline size_t mark_smem_bytes(uint32_t nwords, uint32_t L, uint64_t mmax) {
  size_t b = (size_t)nwords * 4                      // id bitmap
             + (size_t)kRepSlots * 10                // repeated ids, their extra occurrences, slot list
             + (size_t)kRepMax * 8                   // ranked repeated ids (u64 keys)
             + (size_t)2 * ((L + 1) & ~1u) * 8       // base of each non-empty bucket (x2 queries)
             + (size_t)2 * mark_bmap_words(mmax) * 8  // bucket-start bitmap over positions (x2)
             + (size_t)mark_stage(mmax) * 2;         // staged bitmap word indices (reset)
  return (b + 15) & ~(size_t)15;
}

// shared-memory atomics on 32-bit shared-window addresses (no generic-address conversion
// per access)
__device__ __forceinline__ uint32_t smem_or(uint32_t addr, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.or.b32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ uint32_t smem_cas(uint32_t addr, uint32_t cmp, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "r"(addr), "r"(cmp), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void smem_add(uint32_t addr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// word j (< 8) of a thread's scan words, without indexing registers dynamically
__device__ __forceinline__ uint32_t pick8(const uint32_t (&w)[8], uint32_t j) {
  const uint32_t a = (j & 1) ? w[1] : w[0], b = (j & 1) ? w[3] : w[2];
  const uint32_t c = (j & 1) ? w[5] : w[4], d = (j & 1) ? w[7] : w[6];
  const uint32_t ab = (j & 2) ? b : a, cd = (j & 2) ? d : c;
  return (j & 4) ? cd : ab;
}

// named barriers (id 0 is __syncthreads): 1 = the consumer warps, 2 + b = buffer b full
// (the producer arrives, the consumers wait), 4 + b = buffer b empty (the consumers arrive,
// the producer waits)
// (immediate ids, so that ptxas reserves only the barriers used)
template <uint32_t kId, uint32_t kN>
__device__ __forceinline__ void bar_sync() {
  asm volatile("bar.sync %0, %1;" ::"n"(kId), "n"(kN) : "memory");
}
template <uint32_t kId, uint32_t kN>
__device__ __forceinline__ void bar_arrive() {
  asm volatile("bar.arrive %0, %1;" ::"n"(kId), "n"(kN) : "memory");
}
constexpr uint32_t kBarCons = 1, kBarFull = 2, kBarEmpty = 4;
__device__ __forceinline__ void bar_full_sync(uint32_t b) {
  if (b) bar_sync<kBarFull + 1, kMarkThreads>(); else bar_sync<kBarFull, kMarkThreads>();
}
__device__ __forceinline__ void bar_full_arrive(uint32_t b) {
  if (b) bar_arrive<kBarFull + 1, kMarkThreads>(); else bar_arrive<kBarFull, kMarkThreads>();
}
__device__ __forceinline__ void bar_empty_sync(uint32_t b) {
  if (b) bar_sync<kBarEmpty + 1, kMarkThreads>(); else bar_sync<kBarEmpty, kMarkThreads>();
}
__device__ __forceinline__ void bar_empty_arrive(uint32_t b) {
  if (b) bar_arrive<kBarEmpty + 1, kMarkThreads>(); else bar_arrive<kBarEmpty, kMarkThreads>();
}
__device__ __forceinline__ void bar_cons() { bar_sync<kBarCons, kConsThreads>(); }

__global__ void __launch_bounds__(kMarkThreads, 4)
    k_query_mark(QueryArgs a, const uint32_t* __restrict__ qlist, const uint32_t* __restrict__ qcount,
                 uint32_t nwords, uint32_t rep_max, uint32_t* __restrict__ fb_list, uint32_t* __restrict__ fb_count) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ MarkHdr hdr;
  const uint32_t L = a.L, k = a.k;
  const uint32_t Lp = (L + 1) & ~1u;
  const uint32_t nbw = mark_bmap_words(a.mmax);
  const uint32_t stage_cap = mark_stage(a.mmax);
  uint32_t* bits = reinterpret_cast<uint32_t*>(sm);                     // [nwords]
  uint32_t* rkey = bits + nwords;                                       // [kRepSlots]
  uint32_t* rcnt = rkey + kRepSlots;                                    // [kRepSlots]
  uint64_t* rlist = reinterpret_cast<uint64_t*>(rcnt + kRepSlots);      // [kRepMax]
  // base pointer of each non-empty bucket (its start minus its first flattened position)
  // (u32 offsets instead of 64-bit pointers measured slower: graph 4.49 vs 4.42 ms,
  // tools/variants_graph.py; so was a plain load before the repeat table's CAS)
  const uint32_t** nbase = reinterpret_cast<const uint32_t**>(rlist + kRepMax);
  // word w of a bucket-start bitmap over positions: .x = the starts in [32w, 32w + 32),
  // .y = the number of starts below 32w
  uint2* bmap = reinterpret_cast<uint2*>(nbase + 2 * Lp);              // [2][nbw]
  uint16_t* stage = reinterpret_cast<uint16_t*>(bmap + 2 * nbw);        // [stage_cap], 16-B aligned
  uint16_t* rslot = stage + stage_cap;                                  // [kRepSlots] slots in use
  const uint32_t tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
  const uint32_t* __restrict__ gids = a.ids;
  const uint32_t lim = a.shared ? a.shared : a.range;
  const uint32_t nbits = nwords * 32u;
  const uint64_t nq = qlist ? (uint64_t)*qcount : a.nq;  // this launch's queries
  auto query_at = [&](uint64_t it) -> uint64_t { return qlist ? (uint64_t)qlist[it] : it; };

  {  // one-time reset (later queries reset what they touched)
    uint4* b4 = reinterpret_cast<uint4*>(bits);
    for (uint32_t j = tid; j < nwords / 4; j += kMarkThreads) b4[j] = make_uint4(0, 0, 0, 0);
    for (uint32_t j = tid; j < kRepSlots; j += kMarkThreads) {
      rkey[j] = kEmpty;
      rcnt[j] = 0;
    }
    for (uint32_t j = tid; j < 2 * nbw; j += kMarkThreads) bmap[j] = make_uint2(0, 0);
    for (uint32_t j = tid; j < stage_cap; j += kMarkThreads) stage[j] = 0;
    if (tid == 0) hdr.nrep = hdr.overflow = 0;
  }
  __syncthreads();

  if (wib == kConsWarps) {
    // ==== the producer warp: Q1 of this CTA's queries, into two alternating buffers.  Lane
    //      `lane` holds tables t = 4 lane + u (u < 4).  Loads run ahead: a query's extents
    //      one query early, its addresses two, its index three. ====
    uint32_t nad[4];               // addresses of query j + 1
    uint64_t est[4], nst[4];       // extents: of query j (est/esz), of query j + 1 (nst/nen,
    uint32_t esz[4];               // raw: the end offset or segment length, subtracted at use
    uint64_t nen[4];
    uint64_t eq = 0, nq1 = 0, q2 = 0;  // query indices j, j + 1, j + 2
    uint32_t eex = kEmpty, nex = kEmpty;
    const uint64_t g = gridDim.x;
    auto addrs_of = [&](uint64_t q) {
#pragma unroll
      for (uint32_t u = 0; u < 4; ++u) {
        const uint32_t t = 4 * lane + u;
        nad[u] = t < L ? (a.direct ? (uint32_t)q : a.addrs[q * L + t]) : kEmpty;
      }
    };
    auto extents_of = [&](uint64_t q) {  // of the addresses in nad -> nst/nsz/nex
#pragma unroll
      for (uint32_t u = 0; u < 4; ++u) {
        const uint32_t t = 4 * lane + u, ad = nad[u];
        nst[u] = 0;
        nen[u] = 0;
        if (ad < lim) {
          const uint64_t i = a.shared ? (uint64_t)ad : (uint64_t)t * a.range + ad;
          nst[u] = a.goff[i];
          nen[u] = a.seg_len ? (uint64_t)a.seg_len[i] : a.goff[i + 1];
        } else if (ad != kEmpty) {
          atomicAdd(a.err, 1ull);  // an address outside the table
        }
      }
      nex = a.exclude ? a.exclude[q] : (a.exclude_self ? a.self_base + (uint32_t)q : kEmpty);
    };
    uint64_t it = blockIdx.x;
    if (it < nq) {
      eq = query_at(it);
      addrs_of(eq);
      extents_of(eq);
#pragma unroll
      for (uint32_t u = 0; u < 4; ++u) {
        est[u] = nst[u];
        esz[u] = a.seg_len ? (uint32_t)nen[u] : (uint32_t)(nen[u] - nst[u]);
      }
      eex = nex;
    }
    if (it + g < nq) {
      nq1 = query_at(it + g);
      addrs_of(nq1);
    }
    if (it + 2 * g < nq) q2 = query_at(it + 2 * g);
    uint32_t j = 0;
    for (; it < nq; it += g, ++j) {
      const uint32_t b = j & 1;
      if (it + g < nq) extents_of(nq1);     // query j + 1 (its addresses arrived last round)
      if (it + 2 * g < nq) addrs_of(q2);    // query j + 2
      const uint64_t q3 = it + 3 * g < nq ? query_at(it + 3 * g) : 0;
      // Q1 of query j: a warp scan of (size, non-empty) over its L buckets (sizes clamped
      // above L*R: the sum then stays below 2^24; ranks < 2^8), the start bitmap and one
      // base pointer per non-empty bucket, so that position p's bucket is a popc away
      uint32_t v[4], tot = 0;
#pragma unroll
      for (uint32_t u = 0; u < 4; ++u) {
        const uint32_t sz = esz[u] <= a.mmax ? esz[u] : (uint32_t)a.mmax + 1;
        v[u] = tot;
        tot += sz | ((uint32_t)(sz > 0) << 24);
      }
      uint32_t incl = tot;
#pragma unroll
      for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
      }
      const uint32_t M = __shfl_sync(0xFFFFFFFFu, incl, 31) & 0xFFFFFFu;
      const uint32_t base = incl - tot;
      if (j >= 2) bar_empty_sync(b);  // the consumers are done with buffer b
      if (M <= a.mmax) {
        uint2* bm = bmap + b * nbw;
#pragma unroll
        for (uint32_t u = 0; u < 4; ++u) {
          const uint32_t sz = esz[u];
          if (sz > 0) {
            const uint32_t ex = base + v[u];  // exclusive prefix: position | rank << 24
            const uint32_t pos = ex & 0xFFFFFFu, r = ex >> 24;
            nbase[b * Lp + r] = gids + (int64_t)(est[u] - (uint64_t)pos);
            atomicOr(&bm[pos >> 5].x, 1u << (pos & 31));
          }
        }
        __syncwarp();
        // .y of each word: the starts below it (an exclusive scan of the words' popcounts,
        // lanes over words; was a per-bucket fill loop, divergent with the bucket sizes)
        uint32_t carry = 0;
        for (uint32_t w0 = 0; w0 < (M + 31) >> 5; w0 += 32) {
          const uint32_t w = w0 + lane;
          const uint32_t c = w < nbw ? __popc(bm[w].x) : 0u;
          uint32_t in = c;
#pragma unroll
          for (uint32_t o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, in, o);
            if (lane >= o) in += y;
          }
          if (w < nbw) bm[w].y = carry + in - c;
          carry += __shfl_sync(0xFFFFFFFFu, in, 31);
        }
      }
      if (lane == 0) {
        hdr.M[b] = M;
        hdr.excl[b] = eex;
        hdr.q[b] = eq;
      }
      bar_full_arrive(b);
#pragma unroll
      for (uint32_t u = 0; u < 4; ++u) {
        est[u] = nst[u];
        esz[u] = a.seg_len ? (uint32_t)nen[u] : (uint32_t)(nen[u] - nst[u]);
      }
      eex = nex;
      eq = nq1;
      nq1 = q2;
      q2 = q3;
    }
    // match the consumers' last two arrivals on the empty barriers
    for (uint32_t r = j >= 2 ? j - 2 : 0; r < j; ++r) bar_empty_sync(r & 1);
    return;
  }

  // ==== the consumer warps (kConsWarps): Q2-Q3 of one query at a time ====
  const uint32_t s_bits = (uint32_t)__cvta_generic_to_shared(bits);
  const uint32_t s_rkey = (uint32_t)__cvta_generic_to_shared(rkey);
  const uint32_t s_rcnt = (uint32_t)__cvta_generic_to_shared(rcnt);
  uint32_t lanele;
  asm("mov.u32 %0, %%lanemask_le;" : "=r"(lanele));
#ifdef FLASH_QPROF
  long long mp_last = clock64();
#endif
  uint32_t cb = 0;  // this query's Q1 buffer
  for (uint64_t it = blockIdx.x; it < nq; it += gridDim.x, cb ^= 1) {
    // this query's Q1 is written; every consumer is past the previous query's reset
    bar_full_sync(cb);
    MMARK(0);
    const uint32_t M = hdr.M[cb], excl = hdr.excl[cb];
    const uint64_t q = hdr.q[cb];
    const bool bad = M > a.mmax || M == 0;  // more than L*R candidates (bad direct segments): error + pads
    const bool staged = M <= stage_cap;

    // ---- Q2: gather 32-position blocks (block b -> warp b mod kConsWarps, 8 in flight per
    //      lane), mark the bitmap, table the repeats.  Position p lies in bucket
    //      (#starts <= p) - 1.  The excluded id (R#14) is dropped here. ----
    if (!bad) {
      const uint2* bm = bmap + cb * nbw;
      const uint32_t* const* nbs = nbase + cb * Lp;
      const uint32_t nblk = (M + 31) >> 5;
      for (uint32_t b0 = wib; b0 < nblk; b0 += 8 * kConsWarps) {
        uint32_t idv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t b = b0 + u * kConsWarps, p = b * 32 + lane;
          idv[u] = kEmpty;
          if (p < M) {
            const uint2 e = bm[b];
            idv[u] = __ldg(nbs[e.y + __popc(e.x & lanele) - 1] + p);
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t id = idv[u];
          const uint32_t p = (b0 + u * kConsWarps) * 32 + lane;
          if (id < nbits) {
            if (staged) stage[p] = (uint16_t)(id >> 5);
            if (id != excl) {
              const uint32_t bit = 1u << (id & 31);
              const uint32_t old = smem_or(s_bits + ((id >> 5) << 2), bit);
              if (old & bit) {  // a repeat: one more occurrence of id in the table
                uint32_t s = (id * 0x9E3779B1u) >> (32 - kRepLog2);
#pragma unroll 1
                for (uint32_t probe = 0;; ++probe) {
                  const uint32_t c = smem_cas(s_rkey + (s << 2), kEmpty, id);
                  if (c == kEmpty || c == id) {
                    smem_add(s_rcnt + (s << 2), 1u);
                    if (c == kEmpty) rslot[atomicAdd(&hdr.nrep, 1u)] = (uint16_t)s;
                    break;
                  }
                  if (probe == kRepProbes) {  // (a crowded table) -> the fallback kernel
                    atomicExch(&hdr.overflow, 1u);
                    break;
                  }
                  s = (s + 1) & (kRepSlots - 1);
                }
              }
            }
          } else if (id != kEmpty) {
            atomicAdd(a.err, 1ull);  // an id above max_id: contract violation
            if (staged) stage[p] = 0;
          }
        }
      }
    }
    bar_cons();  // B: the gather is done
    MMARK(1);

    // ---- Q3a: each listed repeated id becomes a (count desc, id asc) key and leaves the
    //      bitmap, which then holds exactly the ids seen once; its slot is cleared.  Full
    //      multiplicity = 1 + extra (R#11).  The start bitmap is cleared for the producer. ----
    const uint32_t nrep = hdr.nrep;
    const bool ovf = !bad && (hdr.overflow != 0 || nrep > rep_max);
    for (uint32_t e = tid; e < nrep; e += kConsThreads) {
      const uint32_t s = rslot[e], key = rkey[s], c = rcnt[s];
      if (!ovf) {
        rlist[e] = ((uint64_t)(0xFFFFFFFEu - (c + 1)) << 32) | key;
        atomicAnd(&bits[key >> 5], ~(1u << (key & 31)));
      }
      rkey[s] = kEmpty;
      rcnt[s] = 0;
    }
    if (!bad) {
      uint2* bm = bmap + cb * nbw;
      for (uint32_t w = tid; w <= (M >> 5) + 1 && w < nbw; w += kConsThreads) bm[w].x = 0;
    }
    bar_empty_arrive(cb);  // buffer cb may be refilled
    if (tid == 0) {
      if (ovf) fb_list[atomicAdd(fb_count, 1u)] = (uint32_t)q;
      if (bad && M) atomicAdd(a.err, 1ull);
    }
    bar_cons();  // C: the bitmap holds the singletons, rlist the repeated ids
    MMARK(2);

    uint32_t* oid = a.out_ids + q * k;
    uint32_t* ocnt = a.out_counts + q * k;
    if (bad) {
      for (uint32_t j = tid; j < k; j += kConsThreads) {
        oid[j] = kEmpty;
        ocnt[j] = 0;
      }
    } else if (!ovf) {
      // ---- Q3c: the smallest `need` singletons, in ascending id order (R#12) ----
      const uint32_t nhi = nrep < k ? nrep : k;
      const uint32_t target = k - nhi;
      uint32_t* osg = oid + nhi;
      uint32_t found = 0, buf = 0;
      for (uint32_t w0 = 0; found < target && w0 < nwords; w0 += kConsThreads * kScanWpt) {
        const uint32_t wt = w0 + tid * kScanWpt;
        uint32_t wv[kScanWpt];
        const bool in = wt < nwords;  // (nwords is a multiple of kScanWpt)
#pragma unroll
        for (uint32_t j = 0; j < kScanWpt; j += 4) {
          const uint4 b4 = in ? *reinterpret_cast<const uint4*>(bits + wt + j) : make_uint4(0, 0, 0, 0);
          wv[j] = b4.x;
          wv[j + 1] = b4.y;
          wv[j + 2] = b4.z;
          wv[j + 3] = b4.w;
        }
        uint32_t c = 0;
#pragma unroll
        for (uint32_t j = 0; j < kScanWpt; ++j) c += __popc(wv[j]);
        uint32_t incl = c;
#pragma unroll
        for (uint32_t o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
          if (lane >= o) incl += y;
        }
        if (lane == 31) hdr.rsum[buf][wib] = incl;
        bar_cons();
        const uint32_t rs = lane < kConsWarps ? hdr.rsum[buf][lane] : 0u;
        const uint32_t wpre = __reduce_add_sync(0xFFFFFFFFu, lane < wib ? rs : 0u);
        const uint32_t rtot = __reduce_add_sync(0xFFFFFFFFu, rs);
        uint32_t pos = found + wpre + incl - c;
        uint32_t nz = 0;
        if (c && pos < target) {
#pragma unroll
          for (uint32_t j = 0; j < kScanWpt; ++j) nz |= (wv[j] != 0 ? 1u : 0u) << j;
        }
        while (nz && pos < target) {  // this thread's non-empty words, in order
          const uint32_t j = __ffs(nz) - 1;
          nz &= nz - 1;
          uint32_t xw = pick8(wv, j);
          const uint32_t idb = (wt + j) * 32 - 1;
          do {
            osg[pos++] = idb + __ffs(xw);
            xw &= xw - 1;
          } while (xw && pos < target);
        }
        found += rtot;
        buf ^= 1;
      }
      MMARK(3);
      // ---- Q3b (warp 0): rank the repeated ids (count desc, id asc) ----
      if (wib == 0) {
        for (uint32_t e0 = 0; e0 < nrep; e0 += 32) {
          const uint32_t e = e0 + lane;
          const uint64_t me = e < nrep ? rlist[e] : ~0ull;
          uint32_t rank = 0;
          if (nrep <= 32) {
            for (uint32_t j = 0; j < nrep; ++j) rank += __shfl_sync(0xFFFFFFFFu, me, j) < me;
          } else {
            for (uint32_t j = 0; j < nrep; ++j) rank += rlist[j] < me;
          }
          if (e < nrep && rank < nhi) {
            oid[rank] = (uint32_t)me;
            ocnt[rank] = 0xFFFFFFFEu - (uint32_t)(me >> 32);
          }
        }
      }
      // counts of the singletons, then pads (EMPTY, 0)
      const uint32_t nsg = found < target ? found : target;
      for (uint32_t j = nhi + tid; j < k; j += kConsThreads) {
        const bool pad = j >= nhi + nsg;
        if (pad) oid[j] = kEmpty;
        ocnt[j] = pad ? 0u : 1u;
      }
    }
    MMARK(4);

    // ---- reset for the next query (its full barrier orders it before the next gather):
    //      the bitmap is no longer read once every consumer has passed barrier C or the
    //      last scan round's ----
    if (!bad) {
      if (staged) {  // 8 staged word indices per thread
        for (uint32_t j = tid * 8; j < M; j += kConsThreads * 8) {
          const uint4 s4 = *reinterpret_cast<const uint4*>(stage + j);
          bits[s4.x & 0xFFFFu] = 0;
          bits[s4.x >> 16] = 0;
          bits[s4.y & 0xFFFFu] = 0;
          bits[s4.y >> 16] = 0;
          bits[s4.z & 0xFFFFu] = 0;
          bits[s4.z >> 16] = 0;
          bits[s4.w & 0xFFFFu] = 0;
          bits[s4.w >> 16] = 0;
        }
      } else {
        uint4* b4 = reinterpret_cast<uint4*>(bits);
        for (uint32_t j = tid; j < nwords / 4; j += kConsThreads) b4[j] = make_uint4(0, 0, 0, 0);
      }
    }
    if (tid == 0) hdr.nrep = hdr.overflow = 0;  // (read by every consumer before barrier C)
    MMARK(5);
  }
}

}  // namespace

static bool query_mark_eligible(const QueryArgs& a) {
  const char* e = getenv("FLASH_QUERY_MARK");  // tests: 0 = the sort kernels
  if ((e && e[0] == '0') || a.L > kMarkMaxL || a.mmax > FLASH_MAX_CANDIDATES) return false;
  if ((size_t)mark_words(a.max_id) * 4 > kMarkMaxBitmapBytes) return false;
  return mark_smem_bytes(mark_words(a.max_id), a.L, a.mmax) <= 227 * 1024;
}

// Queries with more candidates than this go to the bitmap kernel, the rest to the size-class
// sort kernels: the bitmap kernel's cost per query is nearly flat in M (its bitmap scan ends
// further out when fewer ids were seen), the sort kernels' grows with M; measured crossover
// on the webspam sweep ~850 candidates (profiles/r02_sweep.txt).  FLASH_QUERY_MARK_MIN
// (tests, tuning) overrides.
uint32_t query_mark_min(const QueryArgs& a) {
  if (!query_mark_eligible(a)) return 0xFFFFFFFFu;
  const char* e = getenv("FLASH_QUERY_MARK_MIN");
  return e ? (uint32_t)strtoul(e, nullptr, 10) : kMarkMinCandidates;
}

int launch_query_mark(const QueryArgs& a, const uint32_t* list, const uint32_t* count, uint32_t* fb,
                      cudaStream_t s) {
  if (a.nq == 0) return 0;
  const uint32_t nwords = mark_words(a.max_id);
  const size_t smem = mark_smem_bytes(nwords, a.L, a.mmax);
  if (!ensure_smem_attr((const void*)k_query_mark, smem)) return -1;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_query_mark, kMarkThreads, smem);
  if (per_sm < 1) return -1;
  uint32_t* fb_list = fb;
  uint32_t* fb_count = fb + a.nq;
  cudaMemsetAsync(fb_count, 0, sizeof(uint32_t), s);
  uint64_t grid = (uint64_t)device_sms() * per_sm;
  if (grid > a.nq) grid = a.nq;
  // FLASH_QUERY_MARK_REPMAX (tests): a lower cap on distinct repeated ids, so that queries
  // take the fallback path
  const char* e = getenv("FLASH_QUERY_MARK_REPMAX");
  uint32_t rep_max = e ? (uint32_t)strtoul(e, nullptr, 10) : kRepMax;
  if (rep_max > kRepMax) rep_max = kRepMax;
  k_query_mark<<<(unsigned)grid, kMarkThreads, smem, s>>>(a, list, count, nwords, rep_max, fb_list, fb_count);
  // the queries with more than rep_max distinct repeated ids: the CTA sort kernel
  const int r = launch_csort(a, (uint32_t)a.mmax, fb_list, fb_count, s);
  if (r < 0) return -1;
  return 2 + r;
}

}  // namespace flash

#ifdef FLASH_QPROF
extern "C" int flash_debug_mprof(unsigned long long out[8], int reset) {
  if (cudaMemcpyFromSymbol(out, flash::g_mprof, sizeof(unsigned long long) * 8) != cudaSuccess) return 1;
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(flash::g_mprof, z, sizeof z);
  }
  return 0;
}
#endif
