// doph.cu — H1-H3: DOPH of CSR rows straight to table addresses (sm_100a).
//
// H1 (Eq. 1 per bin; DOPH §2.3): one pass over a row's nonzeros,
//    bin minima of pi(c) in a warp-private shared-memory array v[B], B = K*L.
// H2 (optimal densification [36]; R#4): an empty bin copies the first originally
//    non-empty bin on its data-independent probe chain; donors read from v only.
// H3 (MapKHashesToAddress, Alg. 2 line 5 P:215; R#5): fmix32 fold of each table's
//    K-tuple, reduced to [0, range) with a multiply-high.
//
// One warp owns one row at a time.  HBM traffic per row: its col_idx (4 B/nnz), two
// row_ptr entries and L addresses (4*L B) — the kernel never writes codes unless
// flash_hash asks for them.  The bin update is a shared-memory atomicMin (RED.MIN): on
// B200 it issues at the LDS rate (profiles/r01_microbench_smem.txt), so no
// read-before-update filter is needed.
#include "flash_internal.cuh"

namespace flash {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 ld_stream4(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void bin_min(uint32_t* v, uint32_t B, const HashKeys& k, uint32_t c) {
  const uint32_t h = perm(k, c);
  atomicMin(&v[__umulhi(h, B)], h);
}

template <bool kCodes, bool kAddrs>
__global__ void __launch_bounds__(kThreads) k_doph(const int64_t* __restrict__ row_ptr,
                                                   const uint32_t* __restrict__ col_idx,
                                                   uint64_t n_rows, uint32_t K, uint32_t L,
                                                   uint32_t range, HashKeys keys,
                                                   uint32_t* __restrict__ codes,
                                                   uint32_t* __restrict__ addrs, uint32_t world) {
  extern __shared__ uint32_t smem[];
  const uint32_t B = K * L;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t wpb = blockDim.x >> 5;
  uint32_t* v = smem + (size_t)warp * 2 * B;  // bin minima (pre-densification)
  uint32_t* code = v + B;                      // densified codes of the current row

  for (uint64_t r = (uint64_t)blockIdx.x * wpb + warp; r < n_rows; r += (uint64_t)gridDim.x * wpb) {
    for (uint32_t i = lane; i < B; i += 32) v[i] = kEmpty;
    __syncwarp();

    // ---- H1: stream the row.  16-byte loads once the cursor is 16-B aligned. ----
    int64_t e = row_ptr[r];
    const int64_t end = row_ptr[r + 1];
    const uint32_t mis = (uint32_t)(reinterpret_cast<uintptr_t>(col_idx + e) & 15u);
    const int64_t head = min(end, e + (int64_t)(((16u - mis) & 15u) >> 2));
    if (e + (int64_t)lane < head) bin_min(v, B, keys, ld_stream(col_idx + e + lane));
    e = head;
    const int64_t vec_end2 = e + ((end - e) & ~(int64_t)255);  // pairs of 512-B warp tiles
    for (; e < vec_end2; e += 256) {  // two 16-B loads in flight per lane
      const uint4 q0 = ld_stream4(reinterpret_cast<const uint4*>(col_idx + e) + lane);
      const uint4 q1 = ld_stream4(reinterpret_cast<const uint4*>(col_idx + e + 128) + lane);
      bin_min(v, B, keys, q0.x);
      bin_min(v, B, keys, q0.y);
      bin_min(v, B, keys, q0.z);
      bin_min(v, B, keys, q0.w);
      bin_min(v, B, keys, q1.x);
      bin_min(v, B, keys, q1.y);
      bin_min(v, B, keys, q1.z);
      bin_min(v, B, keys, q1.w);
    }
    if (end - e >= 128) {  // one more whole tile
      const uint4 q = ld_stream4(reinterpret_cast<const uint4*>(col_idx + e) + lane);
      bin_min(v, B, keys, q.x);
      bin_min(v, B, keys, q.y);
      bin_min(v, B, keys, q.z);
      bin_min(v, B, keys, q.w);
      e += 128;
    }
    for (e += lane; e < end; e += 32) bin_min(v, B, keys, ld_stream(col_idx + e));
    __syncwarp();

    // ---- H2: densify (donors from v only) ----
    bool nonempty = false;
    for (uint32_t i = lane; i < B; i += 32) nonempty |= (v[i] != kEmpty);
    nonempty = __any_sync(0xFFFFFFFFu, nonempty);
    for (uint32_t i = lane; i < B; i += 32) {
      uint32_t x = v[i];
      if (x == kEmpty && nonempty) {
        uint32_t j = 0;
        for (uint32_t a = 1; a <= kProbes; ++a) {
          j = __umulhi(fmix32(keys.s_dens ^ ((i << 8) | a)), B);
          x = v[j];
          if (x != kEmpty) break;
        }
        if (x == kEmpty) {  // circular scan from the last probed bin
          for (uint32_t m = 1; m <= B; ++m) {
            uint32_t jj = j + m;
            if (jj >= B) jj -= B;
            x = v[jj];
            if (x != kEmpty) break;
          }
        }
      }
      code[i] = x;
      if (kCodes) codes[r * B + i] = x;
    }
    __syncwarp();

    // ---- H3: L table addresses ----
    if (kAddrs) {
      for (uint32_t t = lane; t < L; t += 32) {
        uint32_t a = kEmpty;
        if (nonempty) {
          uint32_t x = fmix32(keys.s_addr ^ t);
          for (uint32_t j = 0; j < K; ++j) x = fmix32(x ^ code[t * K + j]);
          a = __umulhi(x, range);
        }
        if (world == 1) {
          addrs[r * L + t] = a;
        } else {  // owner-blocked: table t goes to the block of the rank whose window holds it
          const uint32_t g = ((t + 1) * world - 1) / L;
          const uint32_t g0 = (g * L) / world, g1 = ((g + 1) * L) / world;
          addrs[n_rows * g0 + r * (g1 - g0) + (t - g0)] = a;
        }
      }
    }
    __syncwarp();
  }
}

template <bool C, bool A>
int launch_t(const int64_t* row_ptr, const uint32_t* col_idx, uint64_t n_rows, uint32_t K,
             uint32_t L, uint32_t range, const HashKeys& keys, uint32_t* codes, uint32_t* addrs,
             uint32_t world, cudaStream_t s) {
  const uint32_t B = K * L;
  const size_t per_warp = (size_t)2 * B * sizeof(uint32_t);
  int wpb = (int)((96 * 1024) / per_warp);
  wpb = wpb < 1 ? 1 : (wpb > kThreads / 32 ? kThreads / 32 : wpb);
  const size_t smem = per_warp * wpb;
  static size_t attr = 48 * 1024;
  if (smem > attr) {
    cudaFuncSetAttribute(k_doph<C, A>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  uint64_t blocks = (n_rows + wpb - 1) / wpb;  // one warp per row: the block scheduler balances
  const uint64_t cap = 0x7FFFFFFFull;             // the skewed row lengths
  if (blocks > cap) blocks = cap;
  if (blocks == 0) return 0;
  k_doph<C, A><<<(unsigned)blocks, wpb * 32, smem, s>>>(row_ptr, col_idx, n_rows, K, L, range, keys,
                                                         codes, addrs, world);
  return 1;
}

}  // namespace

int launch_doph(const int64_t* row_ptr, const uint32_t* col_idx, uint64_t n_rows, uint32_t K,
                uint32_t L, uint32_t range, const HashKeys& keys, uint32_t* codes, uint32_t* addrs,
                uint32_t world, cudaStream_t s) {
  if (codes && addrs)
    return launch_t<true, true>(row_ptr, col_idx, n_rows, K, L, range, keys, codes, addrs, world, s);
  if (codes) return launch_t<true, false>(row_ptr, col_idx, n_rows, K, L, range, keys, codes, addrs, world, s);
  return launch_t<false, true>(row_ptr, col_idx, n_rows, K, L, range, keys, codes, addrs, world, s);
}

}  // namespace flash
