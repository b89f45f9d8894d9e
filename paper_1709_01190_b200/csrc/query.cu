// query.cu — Q1-Q3: the querying phase (Alg. 3) on sm_100a.
//
// One CTA owns one query at a time (persistent over queries):
//   Q1 gather   warp w walks tables t = w, w+8, ...; lanes read the bucket
//               ids[goff[t*range+a_t] .. goff[t*range+a_t+1]) (coalesced, ascending ids).
//   Q2 count    each id is inserted into a shared-memory open-addressing table
//               (keys u32, counts u16 packed in u32 words): CAS on a new key, RED.ADD on
//               its count.  New keys are appended to a slot list so later passes touch
//               only the D distinct candidates (COUNTFREQUENCY with full multiplicity, R#11).
//   Q3 top-k    counts are <= L, so a histogram of counts gives the threshold count c*;
//               the ids tied at c* are cut by an 8-bit radix select on the id (ties broken
//               by ascending id, R#12); the <= k survivors are bitonic-sorted by
//               (count desc, id asc) and written, padded with (EMPTY, 0) (R#13).
//   The excluded id (self in the k-NN graph, R#14) is dropped before counting.
#include "flash_internal.cuh"

namespace flash {
namespace {

constexpr int kQThreads = 256;
constexpr int kQWarps = kQThreads / 32;

__device__ __forceinline__ uint32_t pow2_ceil_q(uint32_t x) {
  return x <= 1 ? 1u : 1u << (32 - __clz(x - 1));
}

__device__ __forceinline__ uint32_t get_count(const uint32_t* cnt32, uint32_t slot) {
  return (cnt32[slot >> 1] >> ((slot & 1) * 16)) & 0xFFFFu;
}

template <typename T>
__device__ void cta_bitonic(T* a, uint32_t n) {
  for (uint32_t k = 2; k <= n; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t p = threadIdx.x; p < (n >> 1); p += blockDim.x) {
        const uint32_t i = ((p & ~(j - 1)) << 1) | (p & (j - 1));
        const uint32_t ixj = i + j;
        const T x = a[i], y = a[ixj];
        const bool up = (i & k) == 0;
        if ((x > y) == up) { a[i] = y; a[ixj] = x; }
      }
      __syncthreads();
    }
  }
}

struct QSmem {
  uint32_t* keys;    // [S]
  uint32_t* cnt32;   // [S/2] packed u16 counts
  uint32_t* list;    // [S] slots of distinct keys, in insertion order
  uint64_t* outbuf;  // [pow2(k)]
  uint32_t* hist;    // [max(L+1, 256)]
};

__global__ void __launch_bounds__(kQThreads)
k_query(QueryArgs a, uint32_t hist_len) {
  extern __shared__ __align__(16) uint8_t qsm[];
  const uint32_t S = 1u << a.table_log2;
  const uint32_t mask = S - 1;
  const uint32_t kp2 = pow2_ceil_q(a.k);
  uint64_t* outbuf = reinterpret_cast<uint64_t*>(qsm);
  uint32_t* keys = reinterpret_cast<uint32_t*>(outbuf + kp2);
  uint32_t* cnt32 = keys + S;
  uint32_t* list = cnt32 + S / 2;
  uint32_t* hist = list + S;
  __shared__ uint32_t s_nlist, s_nout, s_cstar, s_need, s_ties, s_theta, s_prefix;

  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t j = threadIdx.x; j < S; j += blockDim.x) keys[j] = kEmpty;
  for (uint32_t j = threadIdx.x; j < S / 2; j += blockDim.x) cnt32[j] = 0;
  for (uint32_t j = threadIdx.x; j < hist_len; j += blockDim.x) hist[j] = 0;
  if (threadIdx.x == 0) s_nlist = 0;
  __syncthreads();

  for (uint64_t q = blockIdx.x; q < a.nq; q += gridDim.x) {
    const uint32_t excl = a.exclude ? a.exclude[q] : (a.exclude_self ? a.self_base + (uint32_t)q : kEmpty);

    // ---- Q1 + Q2: gather and count ----
    for (uint32_t t = warp; t < a.L; t += kQWarps) {
      const uint32_t addr = a.addrs[q * a.L + t];
      if (addr == kEmpty) continue;
      if (addr >= a.range) {
        if (lane == 0) atomicAdd(a.err, 1ull);
        continue;
      }
      const uint64_t i = (uint64_t)t * a.range + addr;
      const uint64_t s = a.goff[i], e = a.goff[i + 1];
      for (uint64_t p = s + lane; p < e; p += 32) {
        const uint32_t id = a.ids[p];
        if (id == excl) continue;
        uint32_t slot = (id * 0x9E3779B1u) >> (32 - a.table_log2);
        while (true) {
          uint32_t cur = keys[slot];
          if (cur == kEmpty) {
            cur = atomicCAS(&keys[slot], kEmpty, id);
            if (cur == kEmpty) {
              list[atomicAdd(&s_nlist, 1u)] = slot;
              cur = id;
            }
          }
          if (cur == id) {
            atomicAdd(&cnt32[slot >> 1], 1u << ((slot & 1) * 16));
            break;
          }
          slot = (slot + 1) & mask;
        }
      }
    }
    __syncthreads();
    const uint32_t D = s_nlist;

    // ---- Q3: threshold count c*, then the ids tied at c* ----
    for (uint32_t j = threadIdx.x; j < D; j += blockDim.x) {
      const uint32_t c = get_count(cnt32, list[j]);
      atomicAdd(&hist[c < a.L ? c : a.L], 1u);  // counts <= L unless ids repeat (contract)
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t cum = 0, c = a.L, cstar = 0, need = 0, ties = 0;
      if (D > a.k) {
        for (; c >= 1; --c) {
          if (cum + hist[c] >= a.k) break;
          cum += hist[c];
        }
        cstar = c;
        need = a.k - cum;  // how many of the hist[c*] tied ids to keep
        ties = hist[c];
      }
      s_cstar = cstar;
      s_need = need;
      s_ties = ties;
      s_theta = 0xFFFFFFFFu;
      s_nout = 0;
    }
    __syncthreads();
    const uint32_t cstar = s_cstar;
    if (cstar > 0 && s_need < s_ties) {
      // radix select: the need-th smallest id among those with count == c*
      uint32_t need = s_need, prefix = 0, pmask = 0;
      for (int shift = 24; shift >= 0; shift -= 8) {
        for (uint32_t d = threadIdx.x; d < 256; d += blockDim.x) hist[d] = 0;
        __syncthreads();
        for (uint32_t j = threadIdx.x; j < D; j += blockDim.x) {
          const uint32_t slot = list[j];
          const uint32_t id = keys[slot];
          if (get_count(cnt32, slot) == cstar && (id & pmask) == prefix)
            atomicAdd(&hist[(id >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          uint32_t cum = 0, d = 0;
          for (; d < 255; ++d) {
            if (cum + hist[d] >= need) break;
            cum += hist[d];
          }
          s_need = need - cum;
          s_prefix = prefix | (d << shift);
        }
        __syncthreads();
        need = s_need;
        prefix = s_prefix;
        pmask |= 255u << shift;
        __syncthreads();
      }
      if (threadIdx.x == 0) s_theta = prefix;
      __syncthreads();
    }
    const uint32_t theta = s_theta;

    // ---- collect <= k survivors, sort by (count desc, id asc) ----
    for (uint32_t j = threadIdx.x; j < D; j += blockDim.x) {
      const uint32_t slot = list[j];
      const uint32_t c = get_count(cnt32, slot);
      const uint32_t id = keys[slot];
      if (c > cstar || (c == cstar && id <= theta))
        outbuf[atomicAdd(&s_nout, 1u)] = ((uint64_t)(0xFFFFu - c) << 32) | id;
    }
    __syncthreads();
    const uint32_t nout = s_nout;
    for (uint32_t j = nout + threadIdx.x; j < kp2; j += blockDim.x) outbuf[j] = ~0ull;
    __syncthreads();
    cta_bitonic(outbuf, kp2);
    for (uint32_t j = threadIdx.x; j < a.k; j += blockDim.x) {
      const uint64_t key = outbuf[j];
      const bool ok = j < nout;
      a.out_ids[q * a.k + j] = ok ? (uint32_t)key : kEmpty;
      a.out_counts[q * a.k + j] = ok ? 0xFFFFu - (uint32_t)(key >> 32) : 0u;
    }

    // ---- reset the touched state for the next query ----
    for (uint32_t j = threadIdx.x; j < D; j += blockDim.x) {
      const uint32_t slot = list[j];
      keys[slot] = kEmpty;
      reinterpret_cast<uint16_t*>(cnt32)[slot] = 0;
    }
    for (uint32_t j = threadIdx.x; j < hist_len; j += blockDim.x) hist[j] = 0;
    if (threadIdx.x == 0) s_nlist = 0;
    __syncthreads();
  }
}

}  // namespace

uint32_t query_table_log2(uint32_t L, uint32_t R) {
  // >= 2x the maximal number of distinct candidates (load factor <= 1/2), >= 2^10
  uint64_t need = 2ull * L * R;
  uint32_t lg = 10;
  while ((1ull << lg) < need) ++lg;
  return lg;
}

size_t query_smem_bytes(uint32_t table_log2, uint32_t k) {
  const size_t S = (size_t)1 << table_log2;
  uint32_t kp2 = 1;
  while (kp2 < k) kp2 <<= 1;
  return kp2 * 8 + S * 4 + S * 2 + S * 4 + 0;  // hist appended separately
}

int launch_query(const QueryArgs& a, cudaStream_t s) {
  if (a.nq == 0) return 0;
  const uint32_t hist_len = (a.L + 1) > 256 ? a.L + 1 : 256;
  const size_t smem = query_smem_bytes(a.table_log2, a.k) + hist_len * 4;
  static size_t attr = 48 * 1024;
  if (smem > attr) {
    if (cudaFuncSetAttribute(k_query, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return 0;  // the launch below then fails and the caller reports it
    attr = smem;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_query, kQThreads, smem);
  if (per_sm < 1) per_sm = 1;
  uint64_t grid = 148ull * per_sm;
  if (grid > a.nq) grid = a.nq;
  k_query<<<(unsigned)grid, kQThreads, smem, s>>>(a, hist_len);
  return 1;
}

}  // namespace flash
