// query_sort.cu — Q1-Q3 by radix partition: one warp owns one query at a time (sm_100a).
//
// COUNTFREQUENCY (Alg. 3) needs equal candidate ids brought together.  The
// L addressed buckets hold M ~ 1K ids, so a warp sorts them in shared memory:
//   Q1 gather   the non-empty buckets of the query are located by a bitmap over the
//               flattened candidate positions (one word + popc per 32 positions).
//   Q2 sort     pass A counts the candidates per digit (the top 10 significant bits of
//               the id range), a warp scan turns counts into bin offsets, pass B gathers
//               again and scatters each id into its bin; each lane then insertion-sorts
//               the 32 bins it owns (a bin spans a narrow id range, so inversions are
//               few).  The array is now sorted by id.
//   Q3 count    run lengths of equal ids are the full multiplicities (R#11), found with
//   + top-k     a ballot of run starts per 32 elements; a histogram of the counts (<= L)
//               gives the threshold count c*; runs of >= 2 ids (a query's near-
//               duplicates, few) are listed in ascending id order.  Ids with count > c*
//               go from that list to per-count output cursors (higher counts first, ids
//               ascending within a count); the ties at c* that survive are the first
//               `need` in ascending id order (R#12) — from the list when c* >= 2, else
//               the once-seen ids, scanned from the start of the sorted array only until
//               `need` are found.  No final sort.  Pads are (EMPTY, 0) (R#13).  The
//               excluded id (self, R#14) is dropped at the gather.
// No hash table, no probing, no CAS: two shared-memory atomics per candidate.
#include "flash_internal.cuh"

namespace flash {
namespace {

constexpr uint32_t kFullS = 0xFFFFFFFFu;

#ifdef FLASH_QPROF  // per-phase cycle counters (diagnostic builds only: build.py --qprof)
__device__ unsigned long long g_qprof[8];
#define QMARK(i)                                                                  \
  do {                                                                            \
    const long long now_ = clock64();                                             \
    if (lane == 0) atomicAdd(&g_qprof[i], (unsigned long long)(now_ - qp_last)); \
    qp_last = now_;                                                               \
  } while (0)
#else
#define QMARK(i) \
  do {           \
  } while (0)
#endif

__device__ __forceinline__ uint32_t lanemask_lt_s() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ uint32_t lanemask_le_s() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
  return m;
}

// bitonic sort of E*32 keys held E per lane, key index r*32+lane (ascending)
template <int E>
__device__ __forceinline__ void warp_bitonic(uint32_t (&v)[E], uint32_t lane) {
#pragma unroll
  for (uint32_t k = 2; k <= 32u * E; k <<= 1) {
#pragma unroll
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      if (j == 32) {  // partner is the other register of this lane (k == 64: ascending)
        const uint32_t a = min(v[0], v[1]), b = max(v[0], v[1]);
        v[0] = a;
        v[1] = b;
      } else {
        const bool lower = (lane & j) == 0;
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const uint32_t w = __shfl_xor_sync(0xFFFFFFFFu, v[r], j);
          const bool asc = ((lane + 32u * r) & k) == 0;
          v[r] = (lower == asc) ? min(v[r], w) : max(v[r], w);
        }
      }
    }
  }
}

// whole-warp ascending sort of arr[lo, lo+n), n <= 64
__device__ __forceinline__ void warp_sort_range(uint32_t* arr, uint32_t lo, uint32_t n, uint32_t lane) {
  if (n <= 32) {
    uint32_t v[1] = {lane < n ? arr[lo + lane] : 0xFFFFFFFFu};
    warp_bitonic<1>(v, lane);
    if (lane < n) arr[lo + lane] = v[0];
  } else {
    uint32_t v[2] = {arr[lo + lane], lane + 32 < n ? arr[lo + 32 + lane] : 0xFFFFFFFFu};
    warp_bitonic<2>(v, lane);
    arr[lo + lane] = v[0];
    if (lane + 32 < n) arr[lo + 32 + lane] = v[1];
  }
}

__host__ __device__ inline size_t sort_slice_bytes(uint32_t mcap, uint32_t kBins, uint32_t L, uint32_t CM) {
  size_t b = (size_t)mcap * 4            // ids, sorted in place by bin
             + (size_t)(kBins * 2 > mcap ? kBins * 2 : mcap)  // u16 bin counters, later the u16 run list
             + (size_t)L * 8              // base of each non-empty segment (bucket)
             + ((size_t)mcap / 32 + 2) * 4  // bucket-start bitmap
             + (size_t)(CM + 1) * 4;      // count histogram
  return (b + 15) & ~(size_t)15;
}

template <int MCAP, int BINS_LOG2, int NW>
__global__ void __launch_bounds__(32 * NW) k_query_sort(QueryArgs a, const uint32_t* __restrict__ qlist,
                                                   const uint32_t* __restrict__ qcount, uint32_t shift,
                                                   uint32_t* __restrict__ next) {
  constexpr uint32_t NBW = MCAP / 32 + 2;
  constexpr uint32_t kBins = 1u << BINS_LOG2;
  extern __shared__ __align__(16) uint8_t sms[];
  const uint32_t L = a.L, k = a.k;  // L segments (table buckets) per query
  const uint32_t CM = a.cmax;        // counts are <= CM (the index's L)
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint8_t* my = sms + sort_slice_bytes(MCAP, kBins, L, CM) * wib;
  uint32_t* arr = reinterpret_cast<uint32_t*>(my);                  // [MCAP]
  uint32_t* binw = arr + MCAP;                                      // [kBins/2] packed u16
  constexpr uint32_t CW = (kBins * 2 > MCAP ? kBins * 2 : MCAP) / 4;  // words of the u16 area
  // nbase[j]: address of candidate position 0 if it lay in the j-th non-empty bucket,
  // so candidate p of that bucket is nbase[j][p] (one wide multiply-add per gather)
  const uint32_t** nbase = reinterpret_cast<const uint32_t**>(binw + CW);  // [L]
  uint32_t* bmap = reinterpret_cast<uint32_t*>(nbase + L);                 // [NBW]
  uint32_t* hcnt = bmap + NBW;                                      // [CM+1]
  const uint16_t* bin16 = reinterpret_cast<const uint16_t*>(binw);
  const uint32_t* __restrict__ gids = a.ids;

  for (uint32_t j = lane; j < kBins / 2; j += 32) binw[j] = 0;
  for (uint32_t j = lane; j < NBW; j += 32) bmap[j] = 0;
  for (uint32_t j = lane; j <= CM; j += 32) hcnt[j] = 0;
  __syncwarp();

  const uint32_t nq = *qcount;
  const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + wib, nw = gridDim.x * (blockDim.x >> 5);
  // queries handed out by a global counter (next; null: statically), so warps that drew
  // larger queries take fewer and none forms a tail
  auto grab = [&](uint32_t cur) -> uint32_t {
    if (!next) return cur + nw;
    uint32_t c = 0;
    if (lane == 0) c = atomicAdd(next, 1u);
    return __shfl_sync(0xFFFFFFFFu, c, 0);
  };
  for (uint32_t it = next ? grab(0) : gw; it < nq; it = grab(it)) {
#ifdef FLASH_QPROF
    long long qp_last = clock64();
#endif
    const uint64_t q = qlist[it];
    const uint32_t excl = a.exclude ? a.exclude[q] : (a.exclude_self ? a.self_base + (uint32_t)q : kEmpty);

    // ---- Q1: non-empty buckets in table order: start bitmap + bases ----
    uint32_t M = 0, nne = 0;
    for (uint32_t t0 = 0; t0 < L; t0 += 32) {
      const uint32_t t = t0 + lane;
      uint32_t sz = 0;
      uint64_t st = 0;
      if (t < L) {
        const uint32_t ad = a.direct ? (uint32_t)q : a.addrs[q * L + t];
        if (ad < (a.shared ? a.shared : a.range)) {
          const uint64_t i = a.shared ? (uint64_t)ad : (uint64_t)t * a.range + ad;
          st = a.goff[i];
          sz = a.seg_len ? a.seg_len[i] : (uint32_t)(a.goff[i + 1] - st);
        }
      }
      uint32_t x = sz;
#pragma unroll
      for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFullS, x, o);
        if (lane >= o) x += y;
      }
      const uint32_t pos = M + x - sz;
      const uint32_t ne = __ballot_sync(kFullS, sz > 0);
      if (sz > 0) {
        nbase[nne + __popc(ne & lanemask_lt_s())] = gids + (int64_t)(st - (uint64_t)pos);
        atomicOr(&bmap[pos >> 5], 1u << (pos & 31));
      }
      nne += __popc(ne);
      M += __shfl_sync(kFullS, x, 31);
    }
    __syncwarp();
    QMARK(0);

    // ---- Q2a: count candidates per digit ----
    {
      uint32_t before = 0;
      for (uint32_t r0 = 0; r0 < M; r0 += 128) {
        uint32_t idv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t w = r0 + u * 32 < M ? bmap[(r0 >> 5) + u] : 0u;  // stay inside the slice
          const uint32_t p = r0 + u * 32 + lane;
          const uint32_t ti = before + __popc(w & lanemask_le_s()) - 1;
          idv[u] = p < M ? __ldg(nbase[ti] + p) : kEmpty;
          before += __popc(w);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t id = idv[u];
          if (id != kEmpty && id != excl) {
            const uint32_t d = (id >> shift) & (kBins - 1);
            atomicAdd(&binw[d >> 1], 1u << ((d & 1) * 16));
          }
        }
      }
    }
    __syncwarp();
    QMARK(1);
    // exclusive scan of the kBins counters (lane owns kBins/32 consecutive bins, 2 per word)
    constexpr uint32_t WPL = kBins / 64;  // words per lane
    uint32_t mtot;
    {
      uint32_t sum = 0;
#pragma unroll
      for (uint32_t i = 0; i < WPL; ++i) {
        const uint32_t w = binw[lane * WPL + i];
        sum += (w & 0xFFFFu) + (w >> 16);
      }
      uint32_t x = sum;
#pragma unroll
      for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFullS, x, o);
        if (lane >= o) x += y;
      }
      mtot = __shfl_sync(kFullS, x, 31);
      uint32_t run = x - sum;
#pragma unroll
      for (uint32_t i = 0; i < WPL; ++i) {
        const uint32_t w = binw[lane * WPL + i];
        const uint32_t c0 = w & 0xFFFFu, c1 = w >> 16;
        binw[lane * WPL + i] = run | ((run + c0) << 16);
        run += c0 + c1;
      }
    }
    __syncwarp();
    QMARK(2);

    // ---- Q2b: gather again, scatter into bins ----
    {
      uint32_t before = 0;
      for (uint32_t r0 = 0; r0 < M; r0 += 128) {
        uint32_t idv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t w = r0 + u * 32 < M ? bmap[(r0 >> 5) + u] : 0u;  // stay inside the slice
          const uint32_t p = r0 + u * 32 + lane;
          const uint32_t ti = before + __popc(w & lanemask_le_s()) - 1;
          idv[u] = p < M ? __ldg(nbase[ti] + p) : kEmpty;
          before += __popc(w);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t id = idv[u];
          if (id != kEmpty && id != excl) {
            const uint32_t d = (id >> shift) & (kBins - 1);
            const uint32_t old = atomicAdd(&binw[d >> 1], 1u << ((d & 1) * 16));
            arr[(old >> ((d & 1) * 16)) & 0xFFFFu] = id;
          }
        }
      }
    }
    __syncwarp();  // every lane is done reading the bitmap (independent thread scheduling)
    for (uint32_t j = lane; j <= (M >> 5) + 1 && j < NBW; j += 32) bmap[j] = 0;
    __syncwarp();
    QMARK(3);
    // bin d now ends at bin16[d].  A bin spans 2^shift ids and holds ~M/kBins of them,
    // so the array is sorted except inside bins, with few inversions (~300 per query on
    // webspam, tools/binstats.py).  Each lane insertion-sorts a contiguous run of whole
    // bins: lane j starts at the bin holding element j*mtot/32, so the runs are balanced
    // even when a near-duplicate's L copies make one bin large; such a bin (16..64 ids)
    // is bitonic-sorted by the whole warp first.  The in-order scan checks four elements
    // per step.  (Measured alternatives, all slower: bubble passes, LSD
    // radix passes, per-bin min-extraction, a descent queue + warp bitonic sort of big
    // bins alone, register-held ids.)
    {
      const uint32_t p = (uint32_t)(((uint64_t)lane * mtot) >> 5);
      uint32_t lo = 0, bsz = 0;
      if (mtot) {
        const uint32_t d = (arr[p] >> shift) & (kBins - 1);
        lo = d ? bin16[d - 1] : 0u;
        bsz = bin16[d] - lo;
      }
      {  // a bin of 16..64 ids found at a split point is sorted by the whole warp first
        const uint32_t plo = __shfl_up_sync(kFullS, lo, 1);
        uint32_t bm = __ballot_sync(kFullS, (lane == 0 || plo != lo) && bsz >= 16 && bsz <= 64);
        while (bm) {
          const uint32_t src = __ffs(bm) - 1;
          warp_sort_range(arr, __shfl_sync(kFullS, lo, src), __shfl_sync(kFullS, bsz, src), lane);
          bm &= bm - 1;
        }
        __syncwarp();
      }
      uint32_t hi = __shfl_down_sync(kFullS, lo, 1);
      if (lane == 31) hi = mtot;
      uint32_t prev = lo < hi ? arr[lo] : 0u;
      uint32_t i = lo + 1;
      while (i < hi) {
        if (i + 3 < hi) {
          const uint32_t x0 = arr[i], x1 = arr[i + 1], x2 = arr[i + 2], x3 = arr[i + 3];
          if (prev <= x0 && x0 <= x1 && x1 <= x2 && x2 <= x3) {
            prev = x3;
            i += 4;
            continue;
          }
        }
        const uint32_t x = arr[i];
        if (x >= prev) {
          prev = x;
        } else {
          uint32_t j = i;
          while (j > lo && arr[j - 1] > x) {
            arr[j] = arr[j - 1];
            --j;
          }
          arr[j] = x;
        }
        ++i;
      }
    }
    __syncwarp();
    QMARK(4);

    // ---- Q3a: run lengths of equal ids are the multiplicities (R#11).  The count histogram
    //      is built on the way (runs of one id, the bulk, aggregated per warp); runs of two
    //      or more are listed by their end index (and count), in ascending id order, in the
    //      area of the finished bin counters.  The sorted array itself is left in place. ----
    // (kBins >= MCAP: the area holds MCAP/2 (end << 16 | count) words; otherwise only u16 end
    // indices fit, and the count is recovered by walking back over the run)
    constexpr bool kList16 = MCAP > kBins;
    uint16_t* mlist16 = reinterpret_cast<uint16_t*>(binw);
    uint32_t* mlist32 = binw;
    uint32_t nd = 0, nm = 0;
    {
      uint32_t carry = 0;  // start index of the run open at the chunk boundary
      for (uint32_t i0 = 0; i0 < mtot; i0 += 32) {
        const uint32_t i = i0 + lane;
        const uint32_t x = i < mtot ? arr[i] : kEmpty;
        const bool start = i < mtot && (i == 0 || arr[i - 1] != x);
        const bool end = i < mtot && (i + 1 == mtot || arr[i + 1] != x);
        const uint32_t sm = __ballot_sync(kFullS, start);
        const uint32_t em = __ballot_sync(kFullS, end);
        const uint32_t below = sm & lanemask_le_s();
        const uint32_t st = below ? i0 + 31 - __clz(below) : carry;
        const uint32_t c = end ? i - st + 1 : 0u;
        const uint32_t ones = __ballot_sync(kFullS, c == 1);
        if (lane == 0 && ones) atomicAdd(&hcnt[1], __popc(ones));
        const uint32_t mm = __ballot_sync(kFullS, c >= 2);
        if (c >= 2) {
          const uint32_t slot = nm + __popc(mm & lanemask_lt_s());
          if (kList16) mlist16[slot] = (uint16_t)i;
          else mlist32[slot] = (i << 16) | c;
          atomicAdd(&hcnt[c < CM ? c : CM], 1u);
        }
        nm += __popc(mm);
        nd += __popc(em);
        if (sm) carry = i0 + 31 - __clz(sm);
      }
    }
    __syncwarp();
    QMARK(5);

    // ---- Q3b: threshold count c*, how many ties to keep, how many counts above c*; the
    //      histogram becomes the output cursor of each count above c* (higher counts first) ----
    uint32_t cstar = 0, need = 0xFFFFFFFFu, nhi = nd;
    {
      const uint32_t cs = (CM + 31) / 32;
      const int32_t hi = (int32_t)CM - (int32_t)(lane * cs);
      const int32_t lo = hi - (int32_t)cs + 1 > 1 ? hi - (int32_t)cs + 1 : 1;
      uint32_t sum = 0;
      for (int32_t c = hi; c >= lo; --c) sum += hcnt[c];
      uint32_t x = sum;
#pragma unroll
      for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFullS, x, o);
        if (lane >= o) x += y;
      }
      const uint32_t bef = x - sum;
      if (nd > k) {
        const uint32_t hit = __ballot_sync(kFullS, bef < k && x >= k);
        const uint32_t src = __ffs(hit) - 1;
        if (lane == src) {
          uint32_t cum = bef;
          for (int32_t c = hi; c >= lo; --c) {
            if (cum + hcnt[c] >= k) {
              cstar = (uint32_t)c;
              need = k - cum;
              nhi = cum;
              break;
            }
            cum += hcnt[c];
          }
        }
        cstar = __shfl_sync(kFullS, cstar, src);
        need = __shfl_sync(kFullS, need, src);
        nhi = __shfl_sync(kFullS, nhi, src);
      }
      __syncwarp();
      uint32_t cur = bef;  // exclusive prefix in descending count order
      for (int32_t c = hi; c >= lo; --c) {
        const uint32_t h = hcnt[c];
        hcnt[c] = cur;
        cur += h;
      }
    }
    __syncwarp();

    // ---- Q3c: (1) the listed runs of >= 2, ascending id: a count above c* is written at
    //      its count's cursor (equal counts stay in id order), ties at c* >= 2 take the
    //      first `need` slots after all of them; (2) the runs of one id (count 1), scanned
    //      in ascending order only as far as needed: count 1 is above c* when c* = 0 (every
    //      distinct id fits) and a tie when c* = 1. ----
    uint32_t* oid = a.out_ids + q * k;
    uint32_t* ocnt = a.out_counts + q * k;
    uint32_t nt = 0;
    for (uint32_t j0 = 0; j0 < nm; j0 += 32) {
      const uint32_t j = j0 + lane;
      uint32_t x = 0, c = 0;
      if (j < nm) {
        if (kList16) {  // the run ends at e; walk back over it for its length
          const uint32_t e = mlist16[j];
          x = arr[e];
          uint32_t b = e;
          while (b > 0 && arr[b - 1] == x) --b;
          c = e - b + 1;
        } else {
          const uint32_t e = mlist32[j];
          x = arr[e >> 16];
          c = e & 0xFFFFu;
        }
      }
      const bool up = j < nm && c > cstar;
      const bool tie = j < nm && cstar >= 2 && c == cstar;
      uint32_t um = __ballot_sync(kFullS, up);
      while (um) {  // one group per distinct count in this chunk
        const uint32_t c0 = __shfl_sync(kFullS, c, __ffs(um) - 1);
        const uint32_t m = __ballot_sync(kFullS, up && c == c0);
        const uint32_t base = hcnt[c0 < CM ? c0 : CM];
        if (up && c == c0) {
          const uint32_t pos = base + __popc(m & lanemask_lt_s());
          oid[pos] = x;
          ocnt[pos] = c;
        }
        __syncwarp();
        if (lane == 0) hcnt[c0 < CM ? c0 : CM] = base + __popc(m);
        __syncwarp();
        um &= ~m;
      }
      const uint32_t mt = __ballot_sync(kFullS, tie);
      const uint32_t rank = nt + __popc(mt & lanemask_lt_s());
      if (tie && rank < need) {
        oid[nhi + rank] = x;
        ocnt[nhi + rank] = c;
      }
      nt += __popc(mt);
    }
    if (cstar <= 1) {
      const bool all1 = cstar == 0;
      uint32_t base1 = all1 ? hcnt[1] : 0u;  // count-1 cursor (descending-count prefix)
      for (uint32_t i0 = 0; i0 < mtot && (all1 || nt < need); i0 += 32) {
        const uint32_t i = i0 + lane;
        const uint32_t x = i < mtot ? arr[i] : kEmpty;
        const bool single = i < mtot && (i == 0 || arr[i - 1] != x) && (i + 1 == mtot || arr[i + 1] != x);
        const uint32_t sg = __ballot_sync(kFullS, single);
        if (all1) {
          if (single) {
            const uint32_t pos = base1 + __popc(sg & lanemask_lt_s());
            oid[pos] = x;
            ocnt[pos] = 1;
          }
          base1 += __popc(sg);
        } else {
          const uint32_t rank = nt + __popc(sg & lanemask_lt_s());
          if (single && rank < need) {
            oid[nhi + rank] = x;
            ocnt[nhi + rank] = 1;
          }
          nt += __popc(sg);
        }
      }
    }
    __syncwarp();
    if (nt > need) nt = need;
    for (uint32_t j = lane; j <= CM; j += 32) hcnt[j] = 0;
    for (uint32_t j = lane; j < kBins / 2; j += 32) binw[j] = 0;
    for (uint32_t j = nhi + nt + lane; j < k; j += 32) {
      oid[j] = kEmpty;
      ocnt[j] = 0;
    }
    __syncwarp();
    QMARK(6);
  }
}

// NW warps per CTA (one query each).
template <int MCAP, int BL, int NW>
int launch_sort_nw(const QueryArgs& a, const uint32_t* list, const uint32_t* count, uint32_t* next, cudaStream_t s) {
  // digit = the top BL bits of the id range [0, max_id]
  const uint32_t bits = a.max_id ? 32u - (uint32_t)__builtin_clz(a.max_id) : 1u;
  const uint32_t shift = bits > (uint32_t)BL ? bits - BL : 0u;
  // FLASH_QSORT_PAD (diagnostic): extra shared memory per CTA, to probe how the kernel's
  // time depends on resident warps
  static const size_t pad = [] { const char* e = getenv("FLASH_QSORT_PAD"); return e ? (size_t)atol(e) : (size_t)0; }();
  const size_t smem = sort_slice_bytes(MCAP, 1u << BL, a.L, a.cmax) * NW + pad;
  if (!ensure_smem_attr((const void*)k_query_sort<MCAP, BL, NW>, smem)) return 0;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_query_sort<MCAP, BL, NW>, 32 * NW, smem);
  if (per_sm < 1) return 0;  // the caller runs the class on the CTA sort kernel instead
  uint64_t grid = (uint64_t)device_sms() * per_sm;
  const uint64_t need = (a.nq + NW - 1) / NW;
  if (grid > need) grid = need;
  if (next) cudaMemsetAsync(next, 0, sizeof(uint32_t), s);
  k_query_sort<MCAP, BL, NW><<<(unsigned)grid, 32 * NW, smem, s>>>(a, list, count, shift, next);
  return 1;
}

// Resident warps per SM of an NW-warp CTA of this class (0 if it does not fit).
template <int MCAP, int BL, int NW>
int resident_warps(const QueryArgs& a) {
  const size_t smem = sort_slice_bytes(MCAP, 1u << BL, a.L, a.cmax) * NW;
  if (!ensure_smem_attr((const void*)k_query_sort<MCAP, BL, NW>, smem)) return 0;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_query_sort<MCAP, BL, NW>, 32 * NW, smem);
  return per_sm * NW;
}

// 4 warps per CTA, or 5 where that packs more warps into an SM's shared memory (the slice
// size depends on L: e.g. MCAP 4096 at L = 128 is 22.5 KB per warp — 2 CTAs of 4 = 8
// warps per SM, 2 CTAs of 5 = 10).  Cached per (class, L, cmax).
template <int MCAP, int BL>
int launch_sort_t(const QueryArgs& a, const uint32_t* list, const uint32_t* count, uint32_t* next, cudaStream_t s) {
  static thread_local uint64_t key = ~0ull;
  static thread_local bool five = false;
  const uint64_t k2 = ((uint64_t)a.L << 32) | a.cmax;
  if (k2 != key) {
    five = resident_warps<MCAP, BL, 5>(a) > resident_warps<MCAP, BL, 4>(a);
    key = k2;
  }
  return five ? launch_sort_nw<MCAP, BL, 5>(a, list, count, next, s) : launch_sort_nw<MCAP, BL, 4>(a, list, count, next, s);
}

}  // namespace

int launch_query_sort(const QueryArgs& a, uint32_t mcap, const uint32_t* list, const uint32_t* count,
                      cudaStream_t s, uint32_t* next) {
  if (mcap <= 768) return launch_sort_t<768, 10>(a, list, count, next, s);
  if (mcap <= 1024) return launch_sort_t<1024, 10>(a, list, count, next, s);
  if (mcap <= 1280) return launch_sort_t<1280, 10>(a, list, count, next, s);
  if (mcap <= 1536) return launch_sort_t<1536, 10>(a, list, count, next, s);
  // the 2048 class: 1024 bins (u16 run list, 10.8 instead of 12.9 KB per warp at L = 32)
  // when it is the top class — L*R <= 2048, saturated buckets put most queries there
  // (friendster graph query 1494 -> 1358 ms) — else 2048 bins (fewer inversions; webspam)
  if (mcap <= 2048)
    return a.mmax <= 2048 ? launch_sort_t<2048, 10>(a, list, count, next, s)
                                              : launch_sort_t<2048, 11>(a, list, count, next, s);
  if (mcap <= 3072) return launch_sort_t<3072, 11>(a, list, count, next, s);
  return launch_sort_t<4096, 11>(a, list, count, next, s);
}

}  // namespace flash

#ifdef FLASH_QPROF
extern "C" int flash_debug_qprof(unsigned long long out[8], int reset) {
  if (cudaMemcpyFromSymbol(out, flash::g_qprof, sizeof(unsigned long long) * 8) != cudaSuccess) return 1;
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(flash::g_qprof, z, sizeof z);
  }
  return 0;
}
#endif
