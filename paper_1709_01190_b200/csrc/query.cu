// query.cu — Q1-Q3: the querying phase (Alg. 3) on sm_100a.
//
// k_query_plan: one lane per query sums the sizes M of its L addressed buckets and
//   files the query into a size class: M <= 768 / 1024 / 1280 / 1536 / 2048 / 3072 / 4096
//   go to the warp-per-query radix-partition kernel (query_sort.cu), 4096 < M <= 8192 to the
//   CTA hash kernel below (count table of 2^14 slots, load factor <= 1/2), 8192 < M <= 32768
//   to the CTA sort kernel (k_query_csort, candidates sorted in shared memory).
// k_query<LOG2S, NT>: one CTA owns one query at a time (persistent over its class list):
//   Q1 gather   warp 0 scans the L bucket sizes into prefix offsets; each warp then walks
//               its own contiguous chunk of the flattened candidate positions p (4 loads in
//               flight per lane, table index advanced monotonically), reading
//               ids[goff[t*range+a_t] + ...].
//   Q2 count    each id goes into a shared-memory open-addressing table (u32 keys, u16
//               counts updated through their u32 word): CAS on a new key, RED.ADD on its
//               count; new slots are appended (warp-aggregated) to a list so later passes
//               touch only the D distinct candidates (COUNTFREQUENCY, full multiplicity,
//               R#11).  The excluded id (self in the k-NN graph, R#14) is skipped.
//   Q3 top-k    counts are <= L: a count histogram gives the threshold count c* (warp-
//               parallel suffix search); the ids tied at c* are cut at the need-th smallest
//               id by a radix select (digits of <= 10 bits from the top set bit of the
//               largest candidate id), stopping as soon as a digit bucket is taken whole
//               (ties by ascending id, R#12).  The <= k survivors are sorted by (count desc,
//               id asc) in one warp's registers (bitonic) and written, padded with
//               (EMPTY, 0) (R#13).  The collect pass also resets the touched table slots.
#include "flash_internal.cuh"

namespace flash {
namespace {

constexpr uint32_t kFullMask = 0xFFFFFFFFu;


__device__ __forceinline__ uint32_t pow2_ceil_q(uint32_t x) {
  return x <= 1 ? 1u : 1u << (32 - __clz(x - 1));
}
__device__ __forceinline__ uint32_t lanemask_lt_q() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Query size classes by M (candidates): the first kSortClasses run one query per warp
// (query_sort.cu; a smaller class uses less shared memory per warp, so more warps per
// SM, up to MCAP 4096); M <= 8192 runs one query per CTA with 2^14 count slots (below).
constexpr int kSortClasses = 7;
__host__ __device__ constexpr uint32_t class_max(int c) {
  return c == 0 ? 768u : c == 1 ? 1024u : c == 2 ? 1280u : c == 3 ? 1536u : c == 4 ? 2048u
         : c == 5 ? 3072u : c == 6 ? 4096u : c == 7 ? 8192u : 32768u;
}
// the last class (8192 < M <= 32768, indexes with L*R > 8192): one 1024-thread CTA per query
// sorts its candidates in shared memory (k_query_csort; 128 KB of ids)
constexpr int kClasses = kSortClasses + 2;
// one more list: queries with more than mark_min candidates, for the occupancy-bitmap kernel
// (query_mark.cu) when the index's ids fit its bitmap
constexpr int kLists = kClasses + 1;
constexpr uint64_t kFewQueries = 65536;  // below: the 3072 < M <= 4096 class runs CTA-per-query

__global__ void k_query_plan(const uint32_t* __restrict__ addrs, uint64_t nq, const uint64_t* __restrict__ goff,
                             const uint32_t* __restrict__ seg_len,
                             uint32_t L, uint32_t range, int direct, uint32_t shared, uint64_t mmax,
                             uint32_t mark_min, uint32_t k,
                             uint32_t* __restrict__ out_ids, uint32_t* __restrict__ out_counts,
                             uint32_t* __restrict__ lists, uint32_t* __restrict__ counts, unsigned long long* err) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t q0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31ull; q0 < nq;
       q0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t q = q0 + lane;
    uint64_t M = 0;
    if (q < nq) {
      const uint32_t lim = shared ? shared : range;
      // 8 tables per step: the address loads, then the offset loads, all independent, so
      // each lane has up to 16 loads in flight instead of one dependent pair per table
      for (uint32_t t0 = 0; t0 < L; t0 += 8) {
        uint32_t a[8];
#pragma unroll
        for (uint32_t u = 0; u < 8; ++u)
          a[u] = t0 + u < L ? (direct ? (uint32_t)q : addrs[q * L + t0 + u]) : kEmpty;
        uint64_t lo[8], hi[8];
#pragma unroll
        for (uint32_t u = 0; u < 8; ++u) {
          lo[u] = hi[u] = 0;
          if (a[u] < lim) {
            const uint64_t i = shared ? (uint64_t)a[u] : (uint64_t)(t0 + u) * range + a[u];
            lo[u] = goff[i];
            hi[u] = seg_len ? lo[u] + seg_len[i] : goff[i + 1];
          } else if (a[u] != kEmpty) {
            atomicAdd(err, 1ull);
          }
        }
#pragma unroll
        for (uint32_t u = 0; u < 8; ++u) M += hi[u] - lo[u];
      }
    }
    int cls = 0;
    while (cls < kClasses - 1 && M > class_max(cls)) ++cls;
    if (M > mark_min || mark_min == 0) cls = kClasses;  // the bitmap kernel's list (it pads M = 0)
    if (q < nq && M > mmax) {  // more candidates than L*R: only possible for bad direct segments
      // (flash.h flash_count_topk: counted in the error counter, k pads)
      atomicAdd(err, 1ull);
      for (uint32_t j = 0; j < k; ++j) {
        out_ids[q * k + j] = kEmpty;
        out_counts[q * k + j] = 0;
      }
      cls = kLists;  // in no list
    }
#pragma unroll
    for (int c = 0; c < kLists; ++c) {
      const uint32_t m = __ballot_sync(kFullMask, q < nq && cls == c);
      if (!m) continue;
      uint32_t b = 0;
      if (lane == 0) b = atomicAdd(&counts[c], __popc(m));
      b = __shfl_sync(kFullMask, b, 0);
      if ((m >> lane) & 1) lists[(uint64_t)c * nq + b + __popc(m & lanemask_lt_q())] = (uint32_t)q;
    }
  }
}

// Sort KP*32 keys (outbuf[0..nout), padded with ~0) ascending in registers of one warp
// (element e = r*32 + lane) and write the first nout as (id, count).
template <int KP>
__device__ __forceinline__ void warp_sort_out(const uint64_t* outbuf, uint32_t nout, uint32_t* oid,
                                              uint32_t* ocnt) {
  const uint32_t lane = threadIdx.x & 31;
  constexpr uint32_t n = KP * 32;
  uint64_t v[KP];
#pragma unroll
  for (int r = 0; r < KP; ++r) {
    const uint32_t e = r * 32 + lane;
    v[r] = e < nout ? outbuf[e] : ~0ull;
  }
#pragma unroll
  for (uint32_t kk = 2; kk <= n; kk <<= 1) {
#pragma unroll
    for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const uint32_t rj = j >> 5;
#pragma unroll
        for (int r = 0; r < KP; ++r) {
          if ((r & rj) == 0) {
            const uint32_t e = r * 32 + lane;
            const bool up = (e & kk) == 0;
            const uint64_t x = v[r], y = v[r | rj];
            if ((x > y) == up) {
              v[r] = y;
              v[r | rj] = x;
            }
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < KP; ++r) {
          const uint32_t e = r * 32 + lane;
          const uint64_t other = __shfl_xor_sync(kFullMask, v[r], j);
          const bool up = (e & kk) == 0;
          const bool lower = (lane & j) == 0;
          v[r] = (lower == up) ? (v[r] < other ? v[r] : other) : (v[r] > other ? v[r] : other);
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < KP; ++r) {
    const uint32_t e = r * 32 + lane;
    if (e < nout) {
      oid[e] = (uint32_t)v[r];
      ocnt[e] = 0xFFFFu - (uint32_t)(v[r] >> 32);
    }
  }
}


struct QueryShared {
  uint32_t M, nlist, nout, cstar, need, ties, theta, maxid, done, prefix;
};

template <int LOG2S, int NT>
__global__ void __launch_bounds__(NT) k_query(QueryArgs a, const uint32_t* __restrict__ qlist,
                                             const uint32_t* __restrict__ qcount, uint32_t hist_len) {
  constexpr uint32_t S = 1u << LOG2S;
  constexpr uint32_t MASK = S - 1;
  extern __shared__ __align__(16) uint8_t sm[];
  const uint32_t L = a.L, CM = a.cmax, k = a.k;  // L segments per query; counts <= CM
  const uint32_t kp2 = pow2_ceil_q(k);
  uint64_t* outbuf = reinterpret_cast<uint64_t*>(sm);      // [kp2]
  uint64_t* base = outbuf + kp2;                             // [L]
  uint32_t* pref = reinterpret_cast<uint32_t*>(base + L);    // [L+1]
  uint32_t* hist = pref + L + 1;                             // [hist_len]
  uint32_t* keys = hist + hist_len;                          // [S]
  uint32_t* cnt32 = keys + S;                                // [S/2] (u16 counts)
  uint16_t* cnt = reinterpret_cast<uint16_t*>(cnt32);
  uint16_t* list = reinterpret_cast<uint16_t*>(cnt32 + S / 2);  // [S]
  auto ldk = [&](uint32_t slot) -> uint32_t { return keys[slot]; };
  auto ldc = [&](uint32_t slot) -> uint32_t { return (uint32_t)cnt[slot]; };
  auto ldl = [&](uint32_t j) -> uint32_t { return (uint32_t)list[j]; };
  __shared__ QueryShared sh;

  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (uint32_t j = tid; j < S; j += NT) keys[j] = kEmpty;
  for (uint32_t j = tid; j < S / 2; j += NT) cnt32[j] = 0;
  for (uint32_t j = tid; j < hist_len; j += NT) hist[j] = 0;
  if (tid == 0) {
    sh.nlist = 0;
    sh.maxid = 0;
  }
  __syncthreads();

  const uint32_t nq = *qcount;
  for (uint32_t it = blockIdx.x; it < nq; it += gridDim.x) {
    const uint64_t q = qlist[it];
    const uint32_t excl = a.exclude ? a.exclude[q] : (a.exclude_self ? a.self_base + (uint32_t)q : kEmpty);

    // ---- Q1: bucket segments -> prefix offsets (warp 0) ----
    if (warp == 0) {
      uint32_t carry = 0;
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
          const uint32_t y = __shfl_up_sync(kFullMask, x, o);
          if (lane >= o) x += y;
        }
        const uint32_t ex = carry + x - sz;
        if (t < L) {
          pref[t] = ex;
          base[t] = st - ex;
        }
        carry += __shfl_sync(kFullMask, x, 31);
      }
      if (lane == 0) {
        pref[L] = carry;
        sh.M = carry;
      }
    }
    __syncthreads();
    const uint32_t M = sh.M;

    // ---- Q2: gather + count; warp w walks its own contiguous chunk of the M positions,
    //      4 x 32 positions per step, advancing each lane's table index monotonically ----
    uint32_t mymax = 0;
    {
      constexpr uint32_t NWARP = NT / 32;
      const uint32_t chunk = ((M + NWARP * 128 - 1) / (NWARP * 128)) * 128;
      const uint32_t pbeg = warp * chunk;
      const uint32_t pend = M < pbeg + chunk ? M : pbeg + chunk;
      uint32_t t = 0;
      if (pbeg + lane < pend) {
        const uint32_t p = pbeg + lane;
        uint32_t lo = 0, hi = L - 1;
        while (lo < hi) {
          const uint32_t mid = (lo + hi + 1) >> 1;
          if (pref[mid] <= p) lo = mid; else hi = mid - 1;
        }
        t = lo;
      }
      for (uint32_t p0 = pbeg; p0 < pend; p0 += 128) {
        uint32_t idv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t p = p0 + u * 32 + lane;
          idv[u] = kEmpty;
          if (p < pend) {
            while (pref[t + 1] <= p) ++t;
            idv[u] = a.ids[base[t] + p];
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t id = idv[u];
          uint32_t newslot = 0xFFFFFFFFu;
          if (id != kEmpty && id != excl) {
            mymax = id > mymax ? id : mymax;
            uint32_t slot = (id * 0x9E3779B1u) >> (32 - LOG2S);
            while (true) {
              uint32_t cur = ldk(slot);
              if (cur == kEmpty) {
                cur = atomicCAS(&keys[slot], kEmpty, id);
                if (cur == kEmpty) {
                  newslot = slot;
                  cur = id;
                }
              }
              if (cur == id) {
                atomicAdd(&cnt32[slot >> 1], 1u << ((slot & 1) * 16));
                break;
              }
              slot = (slot + 1) & MASK;
            }
          }
          const uint32_t m = __ballot_sync(kFullMask, newslot != 0xFFFFFFFFu);
          if (m) {
            uint32_t b = 0;
            if (lane == 0) b = atomicAdd(&sh.nlist, __popc(m));
            b = __shfl_sync(kFullMask, b, 0);
            if (newslot != 0xFFFFFFFFu) list[b + __popc(m & lanemask_lt_q())] = (uint16_t)newslot;
          }
        }
      }
    }
#pragma unroll
    for (uint32_t o = 16; o > 0; o >>= 1) {
      const uint32_t y = __shfl_xor_sync(kFullMask, mymax, o);
      mymax = y > mymax ? y : mymax;
    }
    if (lane == 0 && mymax) atomicMax(&sh.maxid, mymax);
    __syncthreads();
    const uint32_t D = sh.nlist;

    // ---- Q3a: count histogram (count-1 ids, the bulk, aggregated per warp) ----
    for (uint32_t j0 = warp * 32; j0 < D; j0 += NT) {
      const uint32_t j = j0 + lane;
      uint32_t c = 0;
      if (j < D) c = ldc(ldl(j));
      const uint32_t ones = __ballot_sync(kFullMask, c == 1);
      if (lane == 0 && ones) atomicAdd(&hist[1], __popc(ones));
      if (c > 1) atomicAdd(&hist[c < CM ? c : CM], 1u);
    }
    __syncthreads();

    // ---- Q3b: threshold count c* and how many of its ties to keep (warp 0) ----
    if (warp == 0) {
      uint32_t cstar = 0, need = 0, ties = 0;
      if (D > k) {
        const uint32_t cs = (CM + 31) / 32;  // counts per lane, lane 0 = highest counts
        const int32_t hi = (int32_t)CM - (int32_t)(lane * cs);
        const int32_t lo = hi - (int32_t)cs + 1 > 1 ? hi - (int32_t)cs + 1 : 1;
        uint32_t sum = 0;
        for (int32_t c = hi; c >= lo; --c) sum += hist[c];
        uint32_t x = sum;
#pragma unroll
        for (uint32_t o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFullMask, x, o);
          if (lane >= o) x += y;
        }
        const uint32_t before = x - sum;
        const uint32_t hit = __ballot_sync(kFullMask, before < k && x >= k);
        const uint32_t src = __ffs(hit) - 1;
        if (lane == src) {
          uint32_t cum = before;
          for (int32_t c = hi; c >= lo; --c) {
            if (cum + hist[c] >= k) {
              cstar = (uint32_t)c;
              need = k - cum;
              ties = hist[c];
              break;
            }
            cum += hist[c];
          }
        }
        cstar = __shfl_sync(kFullMask, cstar, src);
        need = __shfl_sync(kFullMask, need, src);
        ties = __shfl_sync(kFullMask, ties, src);
      }
      if (lane == 0) {
        sh.cstar = cstar;
        sh.need = need;
        sh.ties = ties;
        sh.theta = 0xFFFFFFFFu;
        sh.nout = 0;
        sh.done = 0;
        sh.prefix = 0;
      }
    }
    __syncthreads();
    const uint32_t cstar = sh.cstar;

    // ---- Q3c: the need-th smallest id among those tied at c* (radix select, digits of
    //      up to 10 bits from the top set bit; stops when a digit bucket is taken whole) ----
    if (cstar > 0 && sh.need < sh.ties) {
      const uint32_t hb = 31 - __clz(sh.maxid | 1u);
      uint32_t width = hb + 1 < 10 ? hb + 1 : 10;
      int32_t shift = (int32_t)(hb + 1 - width);
      uint32_t pmask = 0;
      while (true) {
        const uint32_t nbins = 1u << width;
        const uint32_t dmask = nbins - 1;
        for (uint32_t d = tid; d < nbins; d += NT) hist[d] = 0;
        __syncthreads();
        const uint32_t prefix = sh.prefix;
        for (uint32_t j = tid; j < D; j += NT) {
          const uint32_t slot = ldl(j);
          const uint32_t id = ldk(slot);
          if (ldc(slot) == cstar && (id & pmask) == prefix) atomicAdd(&hist[(id >> shift) & dmask], 1u);
        }
        __syncthreads();
        if (warp == 0) {
          const uint32_t per = (nbins + 31) >> 5;
          const uint32_t d0 = lane * per < nbins ? lane * per : nbins;
          const uint32_t d1 = d0 + per < nbins ? d0 + per : nbins;
          uint32_t sum = 0;
          for (uint32_t d = d0; d < d1; ++d) sum += hist[d];
          uint32_t x = sum;
#pragma unroll
          for (uint32_t o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFullMask, x, o);
            if (lane >= o) x += y;
          }
          const uint32_t need = sh.need;
          const uint32_t before = x - sum;
          const uint32_t hit = __ballot_sync(kFullMask, before < need && x >= need);
          const uint32_t src = __ffs(hit) - 1;
          if (lane == src) {
            uint32_t cum = before, d = d0;
            for (; d + 1 < d1; ++d) {
              if (cum + hist[d] >= need) break;
              cum += hist[d];
            }
            const uint32_t rem = need - cum;
            const uint32_t np = prefix | (d << shift);
            sh.need = rem;
            sh.prefix = np;
            if (hist[d] == rem || shift == 0) {  // take this digit bucket whole / last digit
              sh.theta = np | ((1u << shift) - 1u);
              sh.done = 1;
            }
          }
        }
        __syncthreads();
        if (sh.done) break;
        pmask |= dmask << shift;
        width = shift >= 10 ? 10u : (uint32_t)shift;
        shift -= (int32_t)width;
      }
    }
    const uint32_t theta = sh.theta;

    // ---- Q3d: collect <= k survivors (and reset the touched table state) ----
    for (uint32_t j0 = warp * 32; j0 < D; j0 += NT) {
      const uint32_t j = j0 + lane;
      bool keep = false;
      uint64_t key = 0;
      if (j < D) {
        const uint32_t slot = ldl(j);
        const uint32_t c = ldc(slot);
        const uint32_t id = ldk(slot);
        keep = c > cstar || (c == cstar && id <= theta);
        key = ((uint64_t)(0xFFFFu - c) << 32) | id;
        keys[slot] = kEmpty;
        cnt[slot] = 0;
      }
      const uint32_t m = __ballot_sync(kFullMask, keep);
      if (m) {
        uint32_t b = 0;
        if (lane == 0) b = atomicAdd(&sh.nout, __popc(m));
        b = __shfl_sync(kFullMask, b, 0);
        if (keep) outbuf[b + __popc(m & lanemask_lt_q())] = key;
      }
    }
    for (uint32_t j = tid; j < hist_len; j += NT) hist[j] = 0;
    __syncthreads();
    const uint32_t nout = sh.nout;
    uint32_t* oid = a.out_ids + q * k;
    uint32_t* ocnt = a.out_counts + q * k;
    // ---- Q3e: order by (count desc, id asc): one warp, keys in registers ----
    if (kp2 <= 256) {
      if (warp == 0) {
        if (kp2 <= 32) warp_sort_out<1>(outbuf, nout, oid, ocnt);
        else if (kp2 == 64) warp_sort_out<2>(outbuf, nout, oid, ocnt);
        else if (kp2 == 128) warp_sort_out<4>(outbuf, nout, oid, ocnt);
        else warp_sort_out<8>(outbuf, nout, oid, ocnt);
      }
    } else {
      for (uint32_t j = nout + tid; j < kp2; j += NT) outbuf[j] = ~0ull;
      __syncthreads();
      for (uint32_t kk = 2; kk <= kp2; kk <<= 1) {
        for (uint32_t jj = kk >> 1; jj > 0; jj >>= 1) {
          for (uint32_t p = tid; p < (kp2 >> 1); p += NT) {
            const uint32_t i = ((p & ~(jj - 1)) << 1) | (p & (jj - 1));
            const uint64_t x = outbuf[i], y = outbuf[i + jj];
            if ((x > y) == ((i & kk) == 0)) {
              outbuf[i] = y;
              outbuf[i + jj] = x;
            }
          }
          __syncthreads();
        }
      }
      for (uint32_t j = tid; j < nout; j += NT) {
        const uint64_t key = outbuf[j];
        oid[j] = (uint32_t)key;
        ocnt[j] = 0xFFFFu - (uint32_t)(key >> 32);
      }
    }
    for (uint32_t j = nout + tid; j < k; j += NT) {
      oid[j] = kEmpty;
      ocnt[j] = 0;
    }
    __syncthreads();
    if (tid == 0) {
      sh.nlist = 0;
      sh.maxid = 0;
    }
  }
}


// ---------------------------------------------------------------------------
// k_query_csort: one 1024-thread CTA owns one query at a time (persistent over its class
// list) and sorts the query's candidates in shared memory — the class 8192 < M <= 32768
// (indexes with L*R > 8192, up to FLASH_MAX_CANDIDATES: 128 KB of ids), and the fallback
// of a warp sort class whose per-warp slices do not fit for the index's L.
//   Q1 gather   warp 0 scans the L segment sizes into prefix offsets; every warp then walks
//               its own contiguous chunk of the M flattened positions (as k_query).
//   Q2 sort     pass A counts the candidates per digit (the top 12 bits of the id range,
//               4096 bins), a block scan turns the counts into bin starts, pass B gathers
//               again and scatters each id into its bin; each thread insertion-sorts its
//               bins (<= 64 ids), warp 0 bitonic-sorts the few larger ones (a near-
//               duplicate's L copies) with the freed bin counters as scratch.
//   Q3 count    run lengths of equal ids are the multiplicities (R#11): each warp owns a
//   + top-k     contiguous chunk of the sorted array (a run is attributed to the chunk where
//               it ends; its start is carried across rounds and, at the chunk's first run,
//               found by walking back); a count histogram (counts <= L) gives the threshold
//               c* and how many ties to keep; the ties' ranks in ascending id order are the
//               per-warp tie counts scanned in chunk order (R#12), so the first `need` of
//               them survive with every id above c*; the <= k survivors are sorted by
//               (count desc, id asc) in registers (warp_sort_out) and written, padded with
//               (EMPTY, 0) (R#13).  The excluded id (self, R#14) is dropped at the gather.
constexpr int kCsortThreads = 1024;
constexpr uint32_t kCsortWarps = kCsortThreads / 32;
constexpr uint32_t kCsortBins = 4096;
constexpr uint32_t kCsortSmallBin = 64;   // larger bins: warp 0, bitonic
constexpr uint32_t kCsortBigList = 512;   // >= M / (kCsortSmallBin + 1) for M <= 32768

struct CsortShared {
  uint32_t M, mtot, cstar, need, nout, nbig;
};

__host__ __device__ inline size_t csort_smem_bytes(uint32_t cap, uint32_t L, uint32_t cm, uint32_t k) {
  uint32_t kp2 = 1;
  while (kp2 < k) kp2 <<= 1;
  size_t b = (size_t)kp2 * 8                 // outbuf: survivors (u64 keys)
             + (size_t)L * 8                  // base of each segment
             + (size_t)kCsortBigList * 8      // large bins (start << 32 | size)
             + (size_t)cap * 4                // candidate ids, sorted in place
             + (size_t)kCsortBins * 4         // bin counters (later: bitonic scratch)
             + (size_t)(L + 1) * 4            // segment prefix offsets
             + (size_t)(cm + 1) * 4           // count histogram
             + (size_t)kCsortWarps * 4 * 2;   // per-warp sums
  return (b + 15) & ~(size_t)15;
}

__global__ void __launch_bounds__(kCsortThreads, 1) k_query_csort(QueryArgs a, const uint32_t* __restrict__ qlist,
                                                                 const uint32_t* __restrict__ qcount, uint32_t cap,
                                                                 uint32_t shift) {
  extern __shared__ __align__(16) uint8_t sm[];
  const uint32_t L = a.L, CM = a.cmax, k = a.k;
  const uint32_t kp2 = pow2_ceil_q(k);
  uint64_t* outbuf = reinterpret_cast<uint64_t*>(sm);        // [kp2]
  int64_t* base = reinterpret_cast<int64_t*>(outbuf + kp2);  // [L]
  uint64_t* bigl = reinterpret_cast<uint64_t*>(base + L);    // [kCsortBigList]
  uint32_t* arr = reinterpret_cast<uint32_t*>(bigl + kCsortBigList);  // [cap]
  uint32_t* bins = arr + cap;                                // [kCsortBins]
  uint32_t* pref = bins + kCsortBins;                        // [L+1]
  uint32_t* hist = pref + L + 1;                             // [CM+1]
  uint32_t* wsum = hist + CM + 1;                            // [kCsortWarps]
  uint32_t* wtie = wsum + kCsortWarps;                       // [kCsortWarps]
  __shared__ CsortShared sh;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t* __restrict__ gids = a.ids;

  for (uint32_t j = tid; j < kCsortBins; j += kCsortThreads) bins[j] = 0;
  for (uint32_t j = tid; j <= CM; j += kCsortThreads) hist[j] = 0;
  if (tid == 0) {
    sh.nout = 0;
    sh.nbig = 0;
  }
  __syncthreads();

  // visit(id) for every candidate position, each warp over its own contiguous chunk
  auto gather = [&](uint32_t M, auto&& visit) {
    const uint32_t chunk = ((M + kCsortWarps * 128 - 1) / (kCsortWarps * 128)) * 128;
    const uint32_t pbeg = warp * chunk;
    const uint32_t pend = M < pbeg + chunk ? M : pbeg + chunk;
    uint32_t t = 0;
    if (pbeg + lane < pend) {
      const uint32_t p = pbeg + lane;
      uint32_t lo = 0, hi = L - 1;
      while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (pref[mid] <= p) lo = mid; else hi = mid - 1;
      }
      t = lo;
    }
    for (uint32_t p0 = pbeg; p0 < pend; p0 += 128) {
      uint32_t idv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t p = p0 + u * 32 + lane;
        idv[u] = kEmpty;
        if (p < pend) {
          while (pref[t + 1] <= p) ++t;
          idv[u] = __ldg(gids + base[t] + p);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (idv[u] != kEmpty) visit(idv[u]);
    }
  };

  const uint32_t nq = *qcount;
  for (uint32_t it = blockIdx.x; it < nq; it += gridDim.x) {
    const uint64_t q = qlist[it];
    const uint32_t excl = a.exclude ? a.exclude[q] : (a.exclude_self ? a.self_base + (uint32_t)q : kEmpty);

    // ---- Q1: segment prefix offsets (warp 0) ----
    if (warp == 0) {
      uint32_t carry = 0;
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
          const uint32_t y = __shfl_up_sync(kFullMask, x, o);
          if (lane >= o) x += y;
        }
        const uint32_t ex = carry + x - sz;
        if (t < L) {
          pref[t] = ex;
          base[t] = (int64_t)st - (int64_t)ex;
        }
        carry += __shfl_sync(kFullMask, x, 31);
      }
      if (lane == 0) {
        pref[L] = carry;
        sh.M = carry;
      }
    }
    __syncthreads();
    const uint32_t M = sh.M < cap ? sh.M : cap;  // the plan guarantees M <= cap

    // ---- Q2a: candidates per digit ----
    gather(M, [&](uint32_t id) {
      if (id != excl) atomicAdd(&bins[(id >> shift) & (kCsortBins - 1)], 1u);
    });
    __syncthreads();
    // exclusive block scan of the bins (4 consecutive bins per thread)
    {
      const uint32_t b0 = tid * 4;
      const uint32_t c0 = bins[b0], c1 = bins[b0 + 1], c2 = bins[b0 + 2], c3 = bins[b0 + 3];
      const uint32_t sum = c0 + c1 + c2 + c3;
      uint32_t x = sum;
#pragma unroll
      for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFullMask, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) wsum[warp] = x;
      __syncthreads();
      if (warp == 0) {
        const uint32_t w = wsum[lane];
        uint32_t y = w;
#pragma unroll
        for (uint32_t o = 1; o < 32; o <<= 1) {
          const uint32_t z = __shfl_up_sync(kFullMask, y, o);
          if (lane >= o) y += z;
        }
        wsum[lane] = y - w;
        if (lane == 31) sh.mtot = y;
      }
      __syncthreads();
      const uint32_t run = wsum[warp] + x - sum;
      bins[b0] = run;
      bins[b0 + 1] = run + c0;
      bins[b0 + 2] = run + c0 + c1;
      bins[b0 + 3] = run + c0 + c1 + c2;
    }
    __syncthreads();
    const uint32_t mtot = sh.mtot;

    // ---- Q2b: gather again, scatter into the bins ----
    gather(M, [&](uint32_t id) {
      if (id != excl) arr[atomicAdd(&bins[(id >> shift) & (kCsortBins - 1)], 1u)] = id;
    });
    __syncthreads();
    // bin d is now arr[bins[d-1], bins[d]): sort each bin
    for (uint32_t d = tid; d < kCsortBins; d += kCsortThreads) {
      const uint32_t s0 = d ? bins[d - 1] : 0u, e0 = bins[d];
      if (e0 - s0 <= 1) continue;
      if (e0 - s0 > kCsortSmallBin) {
        const uint32_t slot = atomicAdd(&sh.nbig, 1u);
        if (slot < kCsortBigList) bigl[slot] = ((uint64_t)s0 << 32) | (e0 - s0);
        continue;
      }
      for (uint32_t i = s0 + 1; i < e0; ++i) {
        const uint32_t x = arr[i];
        uint32_t j = i;
        while (j > s0 && arr[j - 1] > x) {
          arr[j] = arr[j - 1];
          --j;
        }
        arr[j] = x;
      }
    }
    __syncthreads();
    if (warp == 0) {  // the large bins; the bin counters are free now and serve as scratch
      const uint32_t nbig = sh.nbig < kCsortBigList ? sh.nbig : kCsortBigList;
      for (uint32_t b = 0; b < nbig; ++b) {
        const uint32_t s0 = (uint32_t)(bigl[b] >> 32), n = (uint32_t)bigl[b];
        if (n <= kCsortBins) {
          const uint32_t n2 = pow2_ceil_q(n);
          for (uint32_t j = lane; j < n2; j += 32) bins[j] = j < n ? arr[s0 + j] : kEmpty;
          __syncwarp();
          for (uint32_t kk = 2; kk <= n2; kk <<= 1) {
            for (uint32_t jj = kk >> 1; jj > 0; jj >>= 1) {
              for (uint32_t p = lane; p < (n2 >> 1); p += 32) {
                const uint32_t i = ((p & ~(jj - 1)) << 1) | (p & (jj - 1));
                const uint32_t x = bins[i], y = bins[i + jj];
                if ((x > y) == ((i & kk) == 0)) {
                  bins[i] = y;
                  bins[i + jj] = x;
                }
              }
              __syncwarp();
            }
          }
          for (uint32_t j = lane; j < n; j += 32) arr[s0 + j] = bins[j];
          __syncwarp();
        } else if (lane == 0) {  // (more ids than the scratch: one lane, insertion sort)
          for (uint32_t i = s0 + 1; i < s0 + n; ++i) {
            const uint32_t x = arr[i];
            uint32_t j = i;
            while (j > s0 && arr[j - 1] > x) {
              arr[j] = arr[j - 1];
              --j;
            }
            arr[j] = x;
          }
        }
        __syncwarp();
      }
    }
    __syncthreads();

    // ---- Q3: runs of equal ids over each warp's chunk.  f(x, c, active) is called every
    //      32-element round with c = the run length at a run's last element (else 0). ----
    const uint32_t chunk = ((mtot + kCsortWarps * 32 - 1) / (kCsortWarps * 32)) * 32;
    const uint32_t cb = warp * chunk < mtot ? warp * chunk : mtot;
    const uint32_t ce = cb + chunk < mtot ? cb + chunk : mtot;
    uint32_t carry0 = cb;
    if (lane == 0 && cb < ce) {
      const uint32_t x = arr[cb];
      while (carry0 > 0 && arr[carry0 - 1] == x) --carry0;
    }
    carry0 = __shfl_sync(kFullMask, carry0, 0);
    auto runs = [&](auto&& f) {
      uint32_t carry = carry0;
      for (uint32_t i0 = cb; i0 < ce; i0 += 32) {
        const uint32_t i = i0 + lane;
        const uint32_t x = i < ce ? arr[i] : kEmpty;
        const bool start = i < ce && (i == 0 || arr[i - 1] != x);
        const bool end = i < ce && (i + 1 == mtot || arr[i + 1] != x);
        const uint32_t smk = __ballot_sync(kFullMask, start);
        uint32_t le;
        asm("mov.u32 %0, %%lanemask_le;" : "=r"(le));
        const uint32_t below = smk & le;
        const uint32_t st = below ? i0 + 31 - __clz(below) : carry;
        f(x, end ? i - st + 1 : 0u);
        if (smk) carry = i0 + 31 - __clz(smk);
      }
    };
    // count histogram; distinct ids per warp
    {
      uint32_t nd = 0;
      runs([&](uint32_t x, uint32_t c) {
        const uint32_t ones = __ballot_sync(kFullMask, c == 1);
        if (lane == 0 && ones) atomicAdd(&hist[1], __popc(ones));
        if (c >= 2) atomicAdd(&hist[c < CM ? c : CM], 1u);
        nd += __popc(__ballot_sync(kFullMask, c > 0));
      });
      if (lane == 0) wsum[warp] = nd;
    }
    __syncthreads();
    // threshold count c* and how many of its ties to keep (warp 0)
    if (warp == 0) {
      uint32_t D = 0;
      D = wsum[lane];
#pragma unroll
      for (uint32_t o = 16; o > 0; o >>= 1) D += __shfl_xor_sync(kFullMask, D, o);
      uint32_t cstar = 0, need = 0;
      if (D > k) {
        const uint32_t cs = (CM + 31) / 32;  // counts per lane, lane 0 = highest counts
        const int32_t hi = (int32_t)CM - (int32_t)(lane * cs);
        const int32_t lo = hi - (int32_t)cs + 1 > 1 ? hi - (int32_t)cs + 1 : 1;
        uint32_t sum = 0;
        for (int32_t c = hi; c >= lo; --c) sum += hist[c];
        uint32_t x = sum;
#pragma unroll
        for (uint32_t o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFullMask, x, o);
          if (lane >= o) x += y;
        }
        const uint32_t before = x - sum;
        const uint32_t hit = __ballot_sync(kFullMask, before < k && x >= k);
        const uint32_t src = __ffs(hit) - 1;
        if (lane == src) {
          uint32_t cum = before;
          for (int32_t c = hi; c >= lo; --c) {
            if (cum + hist[c] >= k) {
              cstar = (uint32_t)c;
              need = k - cum;
              break;
            }
            cum += hist[c];
          }
        }
        cstar = __shfl_sync(kFullMask, cstar, src);
        need = __shfl_sync(kFullMask, need, src);
      }
      if (lane == 0) {
        sh.cstar = cstar;
        sh.need = need;
      }
    }
    __syncthreads();
    const uint32_t cstar = sh.cstar, need = sh.need;
    // ties at c* per warp chunk (ascending id order = chunk order)
    if (cstar > 0) {
      uint32_t nt = 0;
      runs([&](uint32_t, uint32_t c) { nt += __popc(__ballot_sync(kFullMask, c > 0 && c == cstar)); });
      if (lane == 0) wtie[warp] = nt;
    }
    __syncthreads();
    // survivors: every id counted above c*, and the first `need` ties
    {
      uint32_t tbase = 0;
      if (cstar > 0) {
        const uint32_t w = lane < warp ? wtie[lane] : 0u;
        tbase = w;
#pragma unroll
        for (uint32_t o = 16; o > 0; o >>= 1) tbase += __shfl_xor_sync(kFullMask, tbase, o);
      }
      runs([&](uint32_t x, uint32_t c) {
        const bool tie = c > 0 && c == cstar;
        const uint32_t tm = __ballot_sync(kFullMask, tie);
        const bool keep = c > cstar || (tie && tbase + __popc(tm & lanemask_lt_q()) < need);
        tbase += __popc(tm);
        const uint32_t m = __ballot_sync(kFullMask, keep);
        if (m) {
          uint32_t b = 0;
          if (lane == 0) b = atomicAdd(&sh.nout, __popc(m));
          b = __shfl_sync(kFullMask, b, 0);
          if (keep) outbuf[b + __popc(m & lanemask_lt_q())] = ((uint64_t)(0xFFFFu - c) << 32) | x;
        }
      });
    }
    for (uint32_t j = tid; j < kCsortBins; j += kCsortThreads) bins[j] = 0;
    for (uint32_t j = tid; j <= CM; j += kCsortThreads) hist[j] = 0;
    __syncthreads();
    const uint32_t nout = sh.nout;
    uint32_t* oid = a.out_ids + q * k;
    uint32_t* ocnt = a.out_counts + q * k;
    // ---- order by (count desc, id asc) ----
    if (kp2 <= 256) {
      if (warp == 0) {
        if (kp2 <= 32) warp_sort_out<1>(outbuf, nout, oid, ocnt);
        else if (kp2 == 64) warp_sort_out<2>(outbuf, nout, oid, ocnt);
        else if (kp2 == 128) warp_sort_out<4>(outbuf, nout, oid, ocnt);
        else warp_sort_out<8>(outbuf, nout, oid, ocnt);
      }
    } else {
      for (uint32_t j = nout + tid; j < kp2; j += kCsortThreads) outbuf[j] = ~0ull;
      __syncthreads();
      for (uint32_t kk = 2; kk <= kp2; kk <<= 1) {
        for (uint32_t jj = kk >> 1; jj > 0; jj >>= 1) {
          for (uint32_t p = tid; p < (kp2 >> 1); p += kCsortThreads) {
            const uint32_t i = ((p & ~(jj - 1)) << 1) | (p & (jj - 1));
            const uint64_t x = outbuf[i], y = outbuf[i + jj];
            if ((x > y) == ((i & kk) == 0)) {
              outbuf[i] = y;
              outbuf[i + jj] = x;
            }
          }
          __syncthreads();
        }
      }
      for (uint32_t j = tid; j < nout; j += kCsortThreads) {
        const uint64_t key = outbuf[j];
        oid[j] = (uint32_t)key;
        ocnt[j] = 0xFFFFu - (uint32_t)(key >> 32);
      }
    }
    for (uint32_t j = nout + tid; j < k; j += kCsortThreads) {
      oid[j] = kEmpty;
      ocnt[j] = 0;
    }
    __syncthreads();
    if (tid == 0) {
      sh.nout = 0;
      sh.nbig = 0;
    }
  }
}

size_t class_smem(uint32_t log2s, uint32_t L, uint32_t k, uint32_t hist_len) {
  uint32_t kp2 = 1;
  while (kp2 < k) kp2 <<= 1;
  const size_t S = (size_t)1 << log2s;
  return (size_t)kp2 * 8 + (size_t)L * 8 + S * 4 + (size_t)(L + 1) * 4 + (size_t)hist_len * 4 + S * 2 + S * 2;
}

template <int LOG2S, int NT>
int launch_class(const QueryArgs& a, const uint32_t* list, const uint32_t* count, uint32_t hist_len, cudaStream_t s) {
  const size_t smem = class_smem(LOG2S, a.L > a.cmax ? a.L : a.cmax, a.k, hist_len);
  if (!ensure_smem_attr((const void*)k_query<LOG2S, NT>, smem)) return 0;  // -> the CTA sort kernel
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_query<LOG2S, NT>, NT, smem);
  if (per_sm < 1) return 0;
  uint64_t grid = (uint64_t)device_sms() * per_sm;
  if (grid > a.nq) grid = a.nq;
  k_query<LOG2S, NT><<<(unsigned)grid, NT, smem, s>>>(a, list, count, hist_len);
  return 1;
}

}  // namespace

// the CTA sort kernel for queries of at most `cap` candidates (cap <= FLASH_MAX_CANDIDATES)
int launch_csort(const QueryArgs& a, uint32_t cap, const uint32_t* list, const uint32_t* count, cudaStream_t s) {
  cap = (cap + 127) & ~127u;
  const size_t smem = csort_smem_bytes(cap, a.L, a.cmax, a.k);
  if (!ensure_smem_attr((const void*)k_query_csort, smem)) return -1;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_query_csort, kCsortThreads, smem);
  if (per_sm < 1) return -1;
  // digit = the top 12 bits of the id range [0, max_id]
  const uint32_t bits = a.max_id ? 32u - (uint32_t)__builtin_clz(a.max_id) : 1u;
  const uint32_t shift = bits > 12u ? bits - 12u : 0u;
  uint64_t grid = (uint64_t)device_sms() * per_sm;
  if (grid > a.nq) grid = a.nq;
  k_query_csort<<<(unsigned)grid, kCsortThreads, smem, s>>>(a, list, count, cap, shift);
  return 1;
}

bool query_shape_fits(uint32_t L, uint32_t R, uint32_t k) {
  const uint64_t mmax = (uint64_t)L * R;
  if (mmax > FLASH_MAX_CANDIDATES) return false;
  // the CTA sort kernel serves every query size (and any class that does not fit)
  const uint32_t cap = (uint32_t)(((mmax < 8192 ? 8192 : mmax) + 127) & ~127ull);
  return csort_smem_bytes(cap, L, L, k) <= 227 * 1024;
}

// lists [kLists][nq], counts [kLists], then the bitmap kernel's fallback list [nq] + count,
// then the sort classes' query counter
size_t query_scratch_bytes(uint64_t nq) { return sizeof(uint32_t) * (nq * (kLists + 1) + kLists + 4); }

int launch_query_plan(const QueryArgs& a, void* scratch, cudaStream_t s) {
  if (a.nq == 0) return 0;
  uint32_t* lists = reinterpret_cast<uint32_t*>(scratch);
  uint32_t* counts = lists + a.nq * kLists;
  cudaMemsetAsync(counts, 0, sizeof(uint32_t) * kLists, s);
  const uint64_t warps = (a.nq + 31) / 32;
  uint64_t blocks = (warps + 7) / 8;
  if (blocks > (uint64_t)device_sms() * 16) blocks = (uint64_t)device_sms() * 16;
  k_query_plan<<<(unsigned)blocks, 256, 0, s>>>(a.addrs, a.nq, a.goff, a.seg_len, a.L, a.range, a.direct, a.shared, a.mmax,
                                                 query_mark_min(a), a.k, a.out_ids, a.out_counts, lists, counts, a.err);
  return 1;
}

int launch_query(const QueryArgs& a, void* scratch, cudaStream_t s) {
  if (a.nq == 0) return 0;
  uint32_t* lists = reinterpret_cast<uint32_t*>(scratch);
  uint32_t* counts = lists + a.nq * kLists;
  const uint32_t mark_min = query_mark_min(a);
  // the size classes hold the queries with at most min(L*R, mark_min) candidates
  const uint64_t max_m = a.mmax < mark_min ? a.mmax : mark_min;
  const int planned = a.planned ? 0 : launch_query_plan(a, scratch, s);
  const uint32_t hist_len = (a.cmax + 1) > 1024 ? a.cmax + 1 : 1024;
  // The class kernels are persistent over their device-side query lists and run back to
  // back on the caller's stream (measured: overlapping them on side streams is slower,
  // since kernels with different shared-memory footprints then share the SMs).
  const char* few_env = getenv("FLASH_QUERY_FEW");  // tests: force either 4096-class kernel
  const uint64_t few = few_env ? strtoull(few_env, nullptr, 10) : kFewQueries;
  // FLASH_QUERY_CSORT=1 (tests): every class runs the CTA sort kernel
  const char* cs_env = getenv("FLASH_QUERY_CSORT");
  const bool all_csort = cs_env && cs_env[0] == '1';
  // (a spare scratch word after the fallback list: the sort classes' query counter)
  uint32_t* next_q = lists + (uint64_t)(kLists + 1) * a.nq + kLists + 1;
  int n = planned;
  for (int c = 0; c < kClasses && max_m; ++c) {
    if (c > 0 && class_max(c - 1) >= max_m) break;  // no query can be this large
    const uint32_t* lc = lists + (uint64_t)c * a.nq;
    const uint32_t cap = class_max(c) < max_m ? class_max(c) : (uint32_t)max_m;
    int r;
    // (the 4096 class holds 22.5 KB of shared memory per warp; with few queries the CTA
    // kernel, 8 warps on each query, finishes sooner: url 10 K queries 1.24 vs 1.31 ms)
    if (all_csort || c == kClasses - 1) r = launch_csort(a, cap, lc, counts + c, s);
    else if (c == kSortClasses - 1 && a.nq < few) r = launch_class<13, 256>(a, lc, counts + c, hist_len, s);
    else if (c < kSortClasses) r = launch_query_sort(a, class_max(c), lc, counts + c, s, next_q);
    else r = launch_class<14, 256>(a, lc, counts + c, hist_len, s);
    if (r == 0) r = launch_csort(a, cap, lc, counts + c, s);  // a warp class that does not fit
    if (r < 0) return -1;
    n += r;
  }
  if (mark_min < a.mmax) {  // the queries with more than mark_min candidates (query_mark.cu)
    const int r = launch_query_mark(a, lists + (uint64_t)kClasses * a.nq, counts + kClasses,
                                    lists + (uint64_t)kLists * a.nq + kLists, s);
    if (r < 0) return -1;
    n += r;
  }
  return n;
}

}  // namespace flash
