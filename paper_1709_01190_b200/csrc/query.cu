// query.cu — Q1-Q3: the querying phase (Alg. 3) on sm_100a.
//
// k_query_plan: one lane per query sums the sizes M of its L addressed buckets and
//   files the query into a size class: M <= 768 / 1024 / 1280 / 1536 / 2048 / 3072 / 4096
//   go to the warp-per-query radix-partition kernel (query_sort.cu), larger M to the CTA
//   kernel below (count table of 2^14 slots, load factor <= 1/2; 2^16 slots in global
//   memory above 8192).
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
// the last class (M <= 32768, indexes with L*R > 8192) keeps its count table of 2^16 slots
// in a per-CTA region of global memory (L2-resident), since it exceeds shared memory
constexpr int kClasses = kSortClasses + 2;
constexpr uint32_t kHugeLog2 = 16;
constexpr uint64_t kFewQueries = 65536;  // below: the 3072 < M <= 4096 class runs CTA-per-query
constexpr uint32_t kHugeCtas = 296;  // 2 per SM: 114 MB of slices, about the L2 (148: 2.24 s, 592: 2.25 s for the K=2, L=128, R=256 graph; 296: 2.10 s)

__global__ void k_query_plan(const uint32_t* __restrict__ addrs, uint64_t nq, const uint64_t* __restrict__ goff,
                             uint32_t L, uint32_t range, int direct, uint32_t shared, uint64_t mmax, uint32_t k,
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
            hi[u] = goff[i + 1];
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
    if (q < nq && M > mmax) {  // more candidates than L*R: only possible for bad direct segments
      atomicAdd(err, 1ull);
      for (uint32_t j = 0; j < k; ++j) {
        out_ids[q * k + j] = kEmpty;
        out_counts[q * k + j] = 0;
      }
      cls = kClasses;  // in no list
    }
#pragma unroll
    for (int c = 0; c < kClasses; ++c) {
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

// GLOBAL: keys / counts / list live in this CTA's slice of `gtab` (kept clean between
// queries and launches: every query resets the slots it touched), read with ld.global.cg
// so no stale L1 copy is seen after another thread's atomic.
template <int LOG2S, int NT, bool GLOBAL>
__global__ void __launch_bounds__(NT) k_query(QueryArgs a, const uint32_t* __restrict__ qlist,
                                             const uint32_t* __restrict__ qcount, uint32_t hist_len,
                                             uint8_t* __restrict__ gtab) {
  constexpr uint32_t S = 1u << LOG2S;
  constexpr uint32_t MASK = S - 1;
  extern __shared__ __align__(16) uint8_t sm[];
  const uint32_t L = a.L, CM = a.cmax, k = a.k;  // L segments per query; counts <= CM
  const uint32_t kp2 = pow2_ceil_q(k);
  uint64_t* outbuf = reinterpret_cast<uint64_t*>(sm);      // [kp2]
  uint64_t* base = outbuf + kp2;                             // [L]
  uint32_t* pref = reinterpret_cast<uint32_t*>(base + L);    // [L+1]
  uint32_t* hist = pref + L + 1;                             // [hist_len]
  uint32_t* keys;                                            // [S]
  uint32_t* cnt32;                                           // [S/2] (u16 counts)
  if (GLOBAL) {
    if (blockIdx.x >= *qcount) return;
    keys = reinterpret_cast<uint32_t*>(gtab) + (size_t)blockIdx.x * S;
    cnt32 = reinterpret_cast<uint32_t*>(gtab) + (size_t)kHugeCtas * S + (size_t)blockIdx.x * (S / 2);
  } else {
    keys = hist + hist_len;
    cnt32 = keys + S;
  }
  uint16_t* cnt = reinterpret_cast<uint16_t*>(cnt32);
  uint16_t* list = GLOBAL ? reinterpret_cast<uint16_t*>(reinterpret_cast<uint32_t*>(gtab) + (size_t)kHugeCtas * S * 3 / 2) +
                                (size_t)blockIdx.x * S
                          : reinterpret_cast<uint16_t*>(cnt32 + S / 2);  // [S]
  auto ldk = [&](uint32_t slot) -> uint32_t { return GLOBAL ? __ldcg(&keys[slot]) : keys[slot]; };
  auto ldc = [&](uint32_t slot) -> uint32_t { return GLOBAL ? (uint32_t)__ldcg(&cnt[slot]) : (uint32_t)cnt[slot]; };
  auto ldl = [&](uint32_t j) -> uint32_t { return GLOBAL ? (uint32_t)__ldcg(&list[j]) : (uint32_t)list[j]; };
  __shared__ QueryShared sh;

  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (!GLOBAL) {
    for (uint32_t j = tid; j < S; j += NT) keys[j] = kEmpty;
    for (uint32_t j = tid; j < S / 2; j += NT) cnt32[j] = 0;
  }
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
            sz = (uint32_t)(a.goff[i + 1] - st);
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


size_t class_smem(uint32_t log2s, uint32_t L, uint32_t k, uint32_t hist_len, bool global_table = false) {
  uint32_t kp2 = 1;
  while (kp2 < k) kp2 <<= 1;
  const size_t S = global_table ? 0 : (size_t)1 << log2s;
  return (size_t)kp2 * 8 + (size_t)L * 8 + S * 4 + (size_t)(L + 1) * 4 + (size_t)hist_len * 4 + S * 2 + S * 2;
}

template <int LOG2S, int NT, bool GLOBAL>
int launch_class(const QueryArgs& a, const uint32_t* list, const uint32_t* count, uint32_t hist_len,
                 uint8_t* gtab, cudaStream_t s) {
  const size_t smem = class_smem(LOG2S, a.L > a.cmax ? a.L : a.cmax, a.k, hist_len, GLOBAL);
  if (!ensure_smem_attr((const void*)k_query<LOG2S, NT, GLOBAL>, smem)) return 0;
  uint64_t grid;
  if (GLOBAL) {
    grid = kHugeCtas;  // one table slice each (query_huge_table_bytes)
  } else {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_query<LOG2S, NT, GLOBAL>, NT, smem);
    if (per_sm < 1) per_sm = 1;
    grid = (uint64_t)device_sms() * per_sm;
  }
  if (grid > a.nq) grid = a.nq;
  k_query<LOG2S, NT, GLOBAL><<<(unsigned)grid, NT, smem, s>>>(a, list, count, hist_len, gtab);
  return 1;
}

}  // namespace

uint32_t query_table_log2(uint32_t L, uint32_t R) {
  uint64_t need = 2ull * L * R;  // worst case: every candidate distinct, load factor 1/2
  uint32_t lg = 11;
  while ((1ull << lg) < need) ++lg;
  return lg;
}

size_t query_smem_bytes(uint32_t table_log2, uint32_t L, uint32_t k) {
  const uint32_t hist_len = (L + 1) > 1024 ? L + 1 : 1024;
  uint32_t lg = table_log2 < 11 ? 11 : table_log2;
  if (lg > 14) lg = 14;  // the largest class keeps its table in global memory
  return class_smem(lg, L, k, hist_len);
}

size_t query_huge_table_bytes() {
  const size_t S = (size_t)1 << kHugeLog2;
  return kHugeCtas * (S * 4 + S * 2 + S * 2);  // keys, u16 counts, u16 list per CTA
}

void query_huge_table_init(void* gtab, cudaStream_t s) {
  const size_t S = (size_t)1 << kHugeLog2;
  cudaMemsetAsync(gtab, 0xFF, kHugeCtas * S * 4, s);                               // keys = EMPTY
  cudaMemsetAsync(static_cast<uint8_t*>(gtab) + kHugeCtas * S * 4, 0, kHugeCtas * S * 2, s);  // counts
}

size_t query_scratch_bytes(uint64_t nq) { return sizeof(uint32_t) * (nq * kClasses + kClasses); }

int launch_query_plan(const QueryArgs& a, void* scratch, cudaStream_t s) {
  if (a.nq == 0) return 0;
  uint32_t* lists = reinterpret_cast<uint32_t*>(scratch);
  uint32_t* counts = lists + a.nq * kClasses;
  cudaMemsetAsync(counts, 0, sizeof(uint32_t) * kClasses, s);
  const uint64_t warps = (a.nq + 31) / 32;
  uint64_t blocks = (warps + 7) / 8;
  if (blocks > (uint64_t)device_sms() * 16) blocks = (uint64_t)device_sms() * 16;
  const uint64_t max_m = 1ull << (a.table_log2 - 1);  // M <= L*R <= 2^(table_log2 - 1)
  k_query_plan<<<(unsigned)blocks, 256, 0, s>>>(a.addrs, a.nq, a.goff, a.L, a.range, a.direct, a.shared, max_m, a.k,
                                                 a.out_ids, a.out_counts, lists, counts, a.err);
  return 1;
}

int launch_query(const QueryArgs& a, void* scratch, void* huge_tab_v, cudaStream_t s) {
  uint8_t* huge_tab = static_cast<uint8_t*>(huge_tab_v);
  if (a.nq == 0) return 0;
  uint32_t* lists = reinterpret_cast<uint32_t*>(scratch);
  uint32_t* counts = lists + a.nq * kClasses;
  const uint64_t max_m = 1ull << (a.table_log2 - 1);
  const int planned = a.planned ? 0 : launch_query_plan(a, scratch, s);
  const uint32_t hist_len = (a.cmax + 1) > 1024 ? a.cmax + 1 : 1024;
  // The class kernels are persistent over their device-side query lists and run back to
  // back on the caller's stream (measured: overlapping them on side streams is slower,
  // since kernels with different shared-memory footprints then share the SMs).
  const char* few_env = getenv("FLASH_QUERY_FEW");  // tests: force either 4096-class kernel
  const uint64_t few = few_env ? strtoull(few_env, nullptr, 10) : kFewQueries;
  int n = planned;
  for (int c = 0; c < kClasses; ++c) {
    if (c > 0 && class_max(c - 1) >= max_m) break;  // no query can be this large
    const uint32_t* lc = lists + (uint64_t)c * a.nq;
    // (the 4096 class holds 22.5 KB of shared memory per warp; with few queries the CTA
    // kernel, 8 warps on each query, finishes sooner: url 10 K queries 1.24 vs 1.31 ms)
    if (c == kSortClasses - 1 && a.nq < few)
      n += launch_class<13, 256, false>(a, lc, counts + c, hist_len, nullptr, s);
    else if (c < kSortClasses) n += launch_query_sort(a, class_max(c), lc, counts + c, s);
    else if (c == kSortClasses) n += launch_class<14, 256, false>(a, lc, counts + c, hist_len, nullptr, s);
    else n += launch_class<kHugeLog2, 256, true>(a, lc, counts + c, hist_len, huge_tab, s);
  }
  return n;
}

}  // namespace flash

