// exchange.cu — the sender side of the multi-GPU candidate exchange (north_star (d)).
//
// With the L tables partitioned over G GPUs (rank g owns the table window [t0, t1)),
// query q's candidate multiset (Alg. 3 lines 4-7) is the union over ranks of
// the buckets it addresses in each rank's window.  The owner of a table window gathers,
// for every query, the concatenation of its window buckets (table order); the lists are
// sent to the query's owner (NCCL all-to-all-v, paper_1709_01190_b200/dist.py), which
// counts and selects over all G segments (flash_count_topk: the query kernels in
// `direct` segment mode).  The result equals the single-GPU query exactly: the multiset
// is the same and the count / top-k rule does not depend on candidate order.
//
//   k_window_sizes   lane per query: sum of its window bucket sizes (the per-destination
//                    byte counts of the exchange), then an exclusive scan to offsets
//   k_window_gather  warp per query: bucket-by-bucket coalesced copies into the send
//                    buffer at the query's offset
#include <cub/cub.cuh>

#include "flash_internal.cuh"

namespace flash {
namespace {

__global__ void k_window_sizes(const uint32_t* __restrict__ addrs, uint64_t n, uint32_t t0, uint32_t W,
                               uint32_t range, const uint64_t* __restrict__ goff, uint32_t* __restrict__ sizes,
                               unsigned long long* err) {
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t m = 0;
    for (uint32_t j = 0; j < W; ++j) {
      const uint32_t a = addrs[q * W + j];
      if (a < range) {
        const uint64_t i = (uint64_t)(t0 + j) * range + a;
        m += goff[i + 1] - goff[i];
      } else if (a != kEmpty) {
        atomicAdd(err, 1ull);
      }
    }
    sizes[q] = (uint32_t)m;
  }
}

__global__ void k_window_gather(const uint32_t* __restrict__ addrs, uint64_t n, uint32_t t0, uint32_t W,
                                uint32_t range, const uint64_t* __restrict__ goff, const uint32_t* __restrict__ ids,
                                const uint64_t* __restrict__ off, uint32_t* __restrict__ out) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t q = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < n; q += nw) {
    uint64_t d = off[q];
    for (uint32_t j0 = 0; j0 < W; j0 += 32) {
      // lane j holds bucket j0+j's extent; the warp then copies the buckets in order
      uint64_t st = 0;
      uint32_t sz = 0;
      if (j0 + lane < W) {
        const uint32_t a = addrs[q * W + j0 + lane];
        if (a < range) {
          const uint64_t i = (uint64_t)(t0 + j0 + lane) * range + a;
          st = goff[i];
          sz = (uint32_t)(goff[i + 1] - st);
        }
      }
      const uint32_t nb = W - j0 < 32 ? W - j0 : 32;
      for (uint32_t b = 0; b < nb; ++b) {
        const uint64_t bst = __shfl_sync(0xFFFFFFFFu, st, b);
        const uint32_t bsz = __shfl_sync(0xFFFFFFFFu, sz, b);
        for (uint32_t e = lane; e < bsz; e += 32) out[d + e] = __ldg(ids + bst + e);
        d += bsz;
      }
    }
  }
}

// Scan input: sizes[i] widened to uint64 for i < n, and 0 at i = n, so the exclusive
// scan over n+1 entries ends with the total at off[n].
struct Guard {
  const uint32_t* p;
  uint64_t n;
  __host__ __device__ uint64_t operator()(uint64_t i) const { return i < n ? (uint64_t)p[i] : 0ull; }
};
using GuardIt = cub::TransformInputIterator<uint64_t, Guard, cub::CountingInputIterator<uint64_t>>;

}  // namespace

size_t scan_u32_to_u64_tmp_bytes(uint64_t n) {
  size_t bytes = 0;
  GuardIt it(cub::CountingInputIterator<uint64_t>(0), Guard{nullptr, n});
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, it, (uint64_t*)nullptr, (int64_t)(n + 1));
  return bytes;
}

int launch_scan_sizes(const uint32_t* sizes, uint64_t n, uint64_t* off, void* scan_tmp, size_t scan_tmp_bytes,
                      cudaStream_t s) {
  GuardIt it(cub::CountingInputIterator<uint64_t>(0), Guard{sizes, n});
  size_t tmp = scan_tmp_bytes;
  cub::DeviceScan::ExclusiveSum(scan_tmp, tmp, it, off, (int64_t)(n + 1), s);
  return 0;  // library (CUB) kernel, not counted as ours
}

int launch_window_sizes(const uint32_t* addrs, uint64_t n, uint32_t t0, uint32_t t1, uint32_t range,
                        const uint64_t* goff, uint32_t* sizes, uint64_t* off, void* scan_tmp,
                        size_t scan_tmp_bytes, unsigned long long* err, cudaStream_t s) {
  if (n == 0) return 0;
  const uint64_t want = (n + 255) / 256;
  const unsigned blocks = (unsigned)(want < (uint64_t)device_sms() * 16 ? want : (uint64_t)device_sms() * 16);
  k_window_sizes<<<blocks, 256, 0, s>>>(addrs, n, t0, t1 - t0, range, goff, sizes, err);
  launch_scan_sizes(sizes, n, off, scan_tmp, scan_tmp_bytes, s);
  return 1;
}

int launch_window_gather(const uint32_t* addrs, uint64_t n, uint32_t t0, uint32_t t1, uint32_t range,
                         const uint64_t* goff, const uint32_t* ids, const uint64_t* off, uint32_t* out,
                         cudaStream_t s) {
  if (n == 0 || t1 == t0) return 0;
  const uint64_t want = (n + 7) / 8;
  const unsigned blocks = (unsigned)(want < (uint64_t)device_sms() * 16 ? want : (uint64_t)device_sms() * 16);
  k_window_gather<<<blocks, 256, 0, s>>>(addrs, n, t0, t1 - t0, range, goff, ids, off, out);
  return 1;
}

}  // namespace flash
