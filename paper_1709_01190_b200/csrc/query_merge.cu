// query_merge.cu — Q1-Q3 by merging: one warp owns one query at a time (sm_100a).
//
// The L addressed buckets are already sorted by id (B2 stores them ascending, R#10), so
// COUNTFREQUENCY (Alg. 3) is run-length counting of their merge:
//   Q1 gather  the buckets are copied into a warp-private shared-memory buffer as L runs
//              (table-major loop, coalesced reads).
//   Q2 count   ceil(log2 L) levels of pairwise merge-path merging (each lane produces an
//              equal share of the output, ping-ponging between two buffers); then the
//              run starts of the sorted multiset give every distinct id and its full
//              multiplicity (R#11), in ascending id order.  The excluded id (self in the
//              k-NN graph, R#14) is skipped.
//   Q3 top-k   a histogram of the counts (<= L) gives the threshold count c*; because
//              the distinct ids are visited in ascending order, the ids tied at c* that
//              survive are simply the first `need` of them (ties by ascending id, R#12),
//              already in output order; only the few ids with count > c* are sorted
//              (by count desc, id asc) in registers.  Pads are (EMPTY, 0) (R#13).
// Versus hashing (query.cu), this needs no atomics and no probing, and about a third
// of the instructions per query.
#include "flash_internal.cuh"

namespace flash {
namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t lanemask_lt_m() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Sort up to KP*32 u64 keys from buf[0..n) ascending in one warp's registers; write
// element e (< n) to dst_ids[e] / dst_cnt[e] as (id = low 32 bits, count = 0xFFFF - high).
template <int KP>
__device__ __forceinline__ void warp_sort64(const unsigned long long* buf, uint32_t n, uint32_t* dst_ids,
                                            uint32_t* dst_cnt) {
  const uint32_t lane = threadIdx.x & 31;
  constexpr uint32_t N = KP * 32;
  unsigned long long v[KP];
#pragma unroll
  for (int r = 0; r < KP; ++r) {
    const uint32_t e = r * 32 + lane;
    v[r] = e < n ? buf[e] : ~0ull;
  }
#pragma unroll
  for (uint32_t kk = 2; kk <= N; kk <<= 1) {
#pragma unroll
    for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const uint32_t rj = j >> 5;
#pragma unroll
        for (int r = 0; r < KP; ++r) {
          if ((r & rj) == 0) {
            const bool up = ((r * 32 + lane) & kk) == 0;
            const unsigned long long x = v[r], y = v[r | rj];
            if ((x > y) == up) {
              v[r] = y;
              v[r | rj] = x;
            }
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < KP; ++r) {
          const unsigned long long other = __shfl_xor_sync(kFull, v[r], j);
          const bool keep_min = (((r * 32 + lane) & kk) == 0) == ((lane & j) == 0);
          v[r] = keep_min ? (v[r] < other ? v[r] : other) : (v[r] > other ? v[r] : other);
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < KP; ++r) {
    const uint32_t e = r * 32 + lane;
    if (e < n) {
      dst_ids[e] = (uint32_t)v[r];
      dst_cnt[e] = 0xFFFFu - (uint32_t)(v[r] >> 32);
    }
  }
}

__host__ __device__ inline size_t merge_slice_bytes(uint32_t mcap, uint32_t L) {
  // two id buffers + two run-offset arrays + count histogram
  size_t b = (size_t)mcap * 4 * 2 + (size_t)(L + 1) * 4 * 3;
  return (b + 15) & ~(size_t)15;
}

template <int MCAP>
__global__ void __launch_bounds__(128) k_query_merge(QueryArgs a, const uint32_t* __restrict__ qlist,
                                                    const uint32_t* __restrict__ qcount) {
  extern __shared__ __align__(16) uint8_t smm[];
  const uint32_t L = a.L, k = a.k;
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint8_t* my = smm + merge_slice_bytes(MCAP, L) * wib;
  uint32_t* bufA = reinterpret_cast<uint32_t*>(my);  // [MCAP]
  uint32_t* bufB = bufA + MCAP;                       // [MCAP]
  uint32_t* offA = bufB + MCAP;                       // [L+1]
  uint32_t* offB = offA + L + 1;                      // [L+1]
  uint32_t* hcnt = offB + L + 1;                      // [L+1]
  for (uint32_t j = lane; j <= L; j += 32) hcnt[j] = 0;
  __syncwarp();

  const uint32_t nq = *qcount;
  const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + wib, nw = gridDim.x * (blockDim.x >> 5);
  for (uint32_t it = gw; it < nq; it += nw) {
    const uint64_t q = qlist[it];
    const uint32_t excl = a.exclude ? a.exclude[q] : (a.exclude_self ? a.self_base + (uint32_t)q : kEmpty);

    // ---- Q1: run offsets (offA) and global starts (staged in bufB), then copy the L
    //      buckets into bufA, 8 tables' loads in flight per step ----
    uint64_t* tst = reinterpret_cast<uint64_t*>(bufB);  // [L], free until the first merge level
    uint32_t M = 0;
    for (uint32_t t0 = 0; t0 < L; t0 += 32) {
      const uint32_t t = t0 + lane;
      uint32_t sz = 0;
      uint64_t st = 0;
      if (t < L) {
        const uint32_t ad = a.addrs[q * L + t];
        if (ad < a.range) {
          const uint64_t i = (uint64_t)t * a.range + ad;
          st = a.goff[i];
          sz = (uint32_t)(a.goff[i + 1] - st);
        }
      }
      uint32_t x = sz;
#pragma unroll
      for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
      }
      if (t < L) {
        offA[t] = M + x - sz;
        tst[t] = st;
      }
      M += __shfl_sync(kFull, x, 31);
    }
    if (lane == 0) offA[L] = M;
    __syncwarp();
    for (uint32_t t0 = 0; t0 < L; t0 += 8) {
      uint32_t v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t t = t0 + u;
        v[u] = 0;
        if (t < L && lane < offA[t + 1] - offA[t]) v[u] = a.ids[tst[t] + lane];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t t = t0 + u;
        if (t < L) {
          const uint32_t o = offA[t], n = offA[t + 1] - o;
          if (lane < n) bufA[o + lane] = v[u];
          for (uint32_t j = 32 + lane; j < n; j += 32) bufA[o + j] = a.ids[tst[t] + j];  // long buckets
        }
      }
    }
    __syncwarp();

    // ---- Q2: pairwise merge-path levels until one run remains ----
    uint32_t* src = bufA;
    uint32_t* dst = bufB;
    uint32_t* off = offA;
    uint32_t* noff = offB;
    uint32_t nr = L;
    const uint32_t c = (M + 31) >> 5;  // outputs per lane
    const uint32_t o0 = lane * c < M ? lane * c : M;
    const uint32_t o1 = o0 + c < M ? o0 + c : M;
    while (nr > 1) {
      const uint32_t nr2 = (nr + 1) >> 1;
      // pair containing o0: largest p with off[2p] <= o0
      uint32_t lo = 0, hi = nr2 - 1;
      while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (off[2 * mid] <= o0) lo = mid; else hi = mid - 1;
      }
      uint32_t p = lo, o = o0;
      while (o < o1) {
        const uint32_t xs = off[2 * p];
        const uint32_t ys = off[2 * p + 1 < nr ? 2 * p + 1 : nr];
        const uint32_t ye = off[2 * p + 2 < nr ? 2 * p + 2 : nr];
        const uint32_t seg_end = o1 < ye ? o1 : ye;
        if (o < seg_end) {
          const uint32_t nx = ys - xs, ny = ye - ys, d = o - xs;
          uint32_t l2 = d > ny ? d - ny : 0, h2 = d < nx ? d : nx;
          while (l2 < h2) {  // merge path: how many of the first d outputs come from X
            const uint32_t mid = (l2 + h2) >> 1;
            if (src[xs + mid] <= src[ys + d - 1 - mid]) l2 = mid + 1; else h2 = mid;
          }
          uint32_t i = l2, j = d - l2;
          uint32_t xv = i < nx ? src[xs + i] : 0xFFFFFFFFu;
          uint32_t yv = j < ny ? src[ys + j] : 0xFFFFFFFFu;
          // branch-free merge: both heads reloaded every step (an exhausted side reads
          // the sentinel 0xFFFFFFFF, never a valid id)
          for (; o < seg_end; ++o) {
            const bool tx = xv <= yv;
            dst[o] = tx ? xv : yv;
            i += tx;
            j += !tx;
            xv = i < nx ? src[xs + i] : 0xFFFFFFFFu;
            yv = j < ny ? src[ys + j] : 0xFFFFFFFFu;
          }
        }
        ++p;
      }
      for (uint32_t r = lane; r <= nr2; r += 32) noff[r] = off[2 * r < nr ? 2 * r : nr];
      __syncwarp();
      uint32_t* tb = src;
      src = dst;
      dst = tb;
      tb = off;
      off = noff;
      noff = tb;
      nr = nr2;
    }
    // src: the M candidates sorted ascending.  dst is free: run starts (u16, M < 2^16) go
    // to its front, the staging area for counts above c* right after them.
    uint16_t* rs = reinterpret_cast<uint16_t*>(dst);  // [D+1]

    // ---- Q2b: run starts -> distinct ids and counts; count histogram ----
    uint32_t D = 0;
    for (uint32_t i0 = 0; i0 < M; i0 += 32) {
      const uint32_t i = i0 + lane;
      bool start = false;
      if (i < M) {
        const uint32_t x = src[i];
        start = (i == 0 || src[i - 1] != x);
      }
      const uint32_t m = __ballot_sync(kFull, start);
      if (start) rs[D + __popc(m & lanemask_lt_m())] = (uint16_t)i;
      D += __popc(m);
    }
    if (lane == 0) rs[D] = (uint16_t)M;
    __syncwarp();
    uint32_t nd = 0;  // distinct ids other than the excluded one
    for (uint32_t d0 = 0; d0 < D; d0 += 32) {
      const uint32_t d = d0 + lane;
      uint32_t cnt = 0;
      if (d < D && src[rs[d]] != excl) cnt = rs[d + 1] - rs[d];
      const uint32_t ones = __ballot_sync(kFull, cnt == 1);
      if (lane == 0 && ones) hcnt[1] += __popc(ones);
      __syncwarp();
      if (cnt > 1) atomicAdd(&hcnt[cnt < L ? cnt : L], 1u);
      nd += __popc(__ballot_sync(kFull, cnt > 0));
    }
    __syncwarp();

    // ---- Q3a: threshold count c* ----
    uint32_t cstar = 0, need = 0;
    if (nd > k) {
      const uint32_t cs = (L + 31) / 32;
      const int32_t hi = (int32_t)L - (int32_t)(lane * cs);
      const int32_t lo = hi - (int32_t)cs + 1 > 1 ? hi - (int32_t)cs + 1 : 1;
      uint32_t sum = 0;
      for (int32_t cc = hi; cc >= lo; --cc) sum += hcnt[cc];
      uint32_t x = sum;
#pragma unroll
      for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
      }
      const uint32_t before = x - sum;
      const uint32_t hit = __ballot_sync(kFull, before < k && x >= k);
      const uint32_t src_l = __ffs(hit) - 1;
      if (lane == src_l) {
        uint32_t cum = before;
        for (int32_t cc = hi; cc >= lo; --cc) {
          if (cum + hcnt[cc] >= k) {
            cstar = (uint32_t)cc;
            need = k - cum;
            break;
          }
          cum += hcnt[cc];
        }
      }
      cstar = __shfl_sync(kFull, cstar, src_l);
      need = __shfl_sync(kFull, need, src_l);
    } else {
      need = 0xFFFFFFFFu;  // everything survives; no tie cut
    }
    __syncwarp();
    for (uint32_t j = lane; j <= L; j += 32) hcnt[j] = 0;

    // ---- Q3b: survivors in ascending id order: counts above c* go to the staging area
    //      (sorted next), ids tied at c* are written straight to the output after them ----
    uint32_t* oid = a.out_ids + q * k;
    uint32_t* ocnt = a.out_counts + q * k;
    unsigned long long* hiq =
        reinterpret_cast<unsigned long long*>(reinterpret_cast<uint8_t*>(dst) + (((MCAP + 1) * 2 + 15) & ~15));
    uint32_t nhi = 0, ntie = 0;
    // first pass: how many counts above c* (their output block precedes the ties)
    for (uint32_t d0 = 0; d0 < D; d0 += 32) {
      const uint32_t d = d0 + lane;
      uint32_t cnt = 0, id = 0;
      if (d < D) {
        id = src[rs[d]];
        if (id != excl) cnt = rs[d + 1] - rs[d];
      }
      const bool up = cnt > cstar;
      const uint32_t mh = __ballot_sync(kFull, up);
      if (up) hiq[nhi + __popc(mh & lanemask_lt_m())] = ((unsigned long long)(0xFFFFu - cnt) << 32) | id;
      nhi += __popc(mh);
    }
    __syncwarp();
    for (uint32_t d0 = 0; d0 < D && ntie < need; d0 += 32) {
      const uint32_t d = d0 + lane;
      uint32_t cnt = 0, id = 0;
      if (d < D) {
        id = src[rs[d]];
        if (id != excl) cnt = rs[d + 1] - rs[d];
      }
      const bool tie = cnt > 0 && cnt == cstar;
      const uint32_t mt = __ballot_sync(kFull, tie);
      const uint32_t rank = ntie + __popc(mt & lanemask_lt_m());
      if (tie && rank < need) {
        oid[nhi + rank] = id;
        ocnt[nhi + rank] = cnt;
      }
      ntie += __popc(mt);
    }
    if (ntie > need) ntie = need;
    if (nhi <= 32) warp_sort64<1>(hiq, nhi, oid, ocnt);
    else if (nhi <= 64) warp_sort64<2>(hiq, nhi, oid, ocnt);
    else if (nhi <= 128) warp_sort64<4>(hiq, nhi, oid, ocnt);
    else warp_sort64<8>(hiq, nhi, oid, ocnt);
    for (uint32_t j = nhi + ntie + lane; j < k; j += 32) {
      oid[j] = kEmpty;
      ocnt[j] = 0;
    }
    __syncwarp();
  }
}

template <int MCAP>
int launch_merge_t(const QueryArgs& a, const uint32_t* list, const uint32_t* count, cudaStream_t s) {
  constexpr int kWarps = 4;
  const size_t smem = merge_slice_bytes(MCAP, a.L) * kWarps;
  static size_t attr = 48 * 1024;
  if (smem > attr) {
    if (cudaFuncSetAttribute(k_query_merge<MCAP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return 0;
    attr = smem;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_query_merge<MCAP>, 32 * kWarps, smem);
  if (per_sm < 1) per_sm = 1;
  uint64_t grid = 148ull * per_sm;
  const uint64_t need = (a.nq + kWarps - 1) / kWarps;
  if (grid > need) grid = need;
  k_query_merge<MCAP><<<(unsigned)grid, 32 * kWarps, smem, s>>>(a, list, count);
  return 1;
}

}  // namespace

int launch_query_merge(const QueryArgs& a, uint32_t mcap, const uint32_t* list, const uint32_t* count,
                       cudaStream_t s) {
  if (mcap <= 1536) return launch_merge_t<1536>(a, list, count, s);
  return launch_merge_t<3072>(a, list, count, s);
}

}  // namespace flash
