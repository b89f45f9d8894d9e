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
#include <algorithm>
#include <cstdlib>

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

// Two 16-byte streaming loads issued back to back (one asm block, so the compiler cannot
// sink the second load below the first one's uses: two tiles in flight per lane).
__device__ __forceinline__ void ld_stream4x2(const uint4* p0, const uint4* p1, uint4& a, uint4& b) {
  asm volatile(
      "ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%8];\n\t"
      "ld.global.nc.L1::no_allocate.v4.u32 {%4, %5, %6, %7}, [%9];"
      : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
      : "l"(p0), "l"(p1));
}

__host__ __device__ __forceinline__ uint32_t warp_words(uint32_t B) {
  return 2 * B + (B + 1) / 2;  // v[B], code[B], u16 elist[B]
}

__device__ __forceinline__ uint32_t lanemask_lt_d() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ void smem_min(uint32_t addr, uint32_t v) {
  asm volatile("red.shared.min.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ void bin_min(uint32_t* v, uint32_t B, const HashKeys& k, uint32_t c) {
  const uint32_t h = perm(k, c);
  atomicMin(&v[__umulhi(h, B)], h);
}

// H3 for one row (lanes over tables): fmix32 fold of each table's K-tuple, multiply-high to
// [0, range).  out.world > 1 writes owner-blocked (flash_hash_blocked), or with out.peers
// straight into each table owner's window-address buffer (the multi-GPU X1 exchange fused
// into the hash: P2P stores over NVLink when the owner is another GPU).
__device__ __forceinline__ void write_addrs(const uint32_t* code, bool nonempty, uint32_t K, uint32_t L,
                                            uint32_t range, const HashKeys& keys, const AddrOut& out,
                                            uint64_t n_rows, uint64_t r, uint32_t lane) {
  // K % 4 == 0 with a 16-B aligned code array: the tuple in 16-byte shared loads (lanes 16 B
  // apart: conflict-free, where 4-byte loads at a 4K-byte lane stride conflict K-way)
  const bool vec = (K & 3) == 0 && (reinterpret_cast<uintptr_t>(code) & 15) == 0;
  for (uint32_t t = lane; t < L; t += 32) {
    uint32_t a = kEmpty;
    if (nonempty) {
      uint32_t x = fmix32(keys.s_addr ^ t);
      if (vec) {
        const uint4* c4 = reinterpret_cast<const uint4*>(code + t * K);
        for (uint32_t j = 0; j < K / 4; ++j) {
          const uint4 q = c4[j];
          x = fmix32(x ^ q.x);
          x = fmix32(x ^ q.y);
          x = fmix32(x ^ q.z);
          x = fmix32(x ^ q.w);
        }
      } else {
        for (uint32_t j = 0; j < K; ++j) x = fmix32(x ^ code[t * K + j]);
      }
      a = __umulhi(x, range);
    }
    if (out.world == 1) {
      out.addrs[r * L + t] = a;
    } else {  // owner-blocked: table t goes to the block of the rank whose window holds it
      const uint32_t g = ((t + 1) * out.world - 1) / L;
      const uint32_t g0 = (g * L) / out.world, g1 = ((g + 1) * L) / out.world;
      if (out.peers)
        out.peers[g][(out.row0 + r) * (g1 - g0) + (t - g0)] = a;
      else
        out.addrs[n_rows * g0 + r * (g1 - g0) + (t - g0)] = a;
    }
  }
}

template <bool kCodes, bool kAddrs>
__global__ void __launch_bounds__(kThreads, 8) k_doph(const int64_t* __restrict__ row_ptr,
                                                   const uint32_t* __restrict__ col_idx,
                                                   uint64_t n_rows, uint32_t K, uint32_t L,
                                                   uint32_t range, HashKeys keys,
                                                   uint32_t* __restrict__ codes, AddrOut out,
                                                   int64_t skip_le, const uint32_t* __restrict__ long_rows,
                                                   uint32_t long_cap) {
  extern __shared__ uint32_t smem[];
  const uint32_t B = K * L;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t wpb = blockDim.x >> 5;
  uint32_t* v = smem + (size_t)warp * warp_words(B);  // bin minima (pre-densification)
  uint32_t* code = v + B;                              // densified codes of the current row
  uint16_t* elist = reinterpret_cast<uint16_t*>(code + B);  // empty bins of the current row

  auto do_row = [&](const uint64_t r, int64_t e, const int64_t end) {
    for (uint32_t i = lane; i < B; i += 32) v[i] = kEmpty;
    __syncwarp();

    // ---- H1: stream the row.  16-byte loads once the cursor is 16-B aligned. ----
    const uint32_t mis = (uint32_t)(reinterpret_cast<uintptr_t>(col_idx + e) & 15u);
    const int64_t head = min(end, e + (int64_t)(((16u - mis) & 15u) >> 2));
    if (e + (int64_t)lane < head) bin_min(v, B, keys, ld_stream(col_idx + e + lane));
    e = head;
    const int64_t vec_end2 = e + ((end - e) & ~(int64_t)255);  // pairs of 512-B warp tiles
    if (e < vec_end2) {  // software-pipelined: the next pair of tiles loads while this one hashes
      uint4 q0, q1;
      ld_stream4x2(reinterpret_cast<const uint4*>(col_idx + e) + lane,
                   reinterpret_cast<const uint4*>(col_idx + e + 128) + lane, q0, q1);
      while (true) {
        const int64_t en = e + 256;
        const bool more = en < vec_end2;
        uint4 n0 = q0, n1 = q1;
        if (more)
          ld_stream4x2(reinterpret_cast<const uint4*>(col_idx + en) + lane,
                       reinterpret_cast<const uint4*>(col_idx + en + 128) + lane, n0, n1);
        bin_min(v, B, keys, q0.x);
        bin_min(v, B, keys, q0.y);
        bin_min(v, B, keys, q0.z);
        bin_min(v, B, keys, q0.w);
        bin_min(v, B, keys, q1.x);
        bin_min(v, B, keys, q1.y);
        bin_min(v, B, keys, q1.z);
        bin_min(v, B, keys, q1.w);
        e = en;
        if (!more) break;
        q0 = n0;
        q1 = n1;
      }
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
    // Pass 1: non-empty bins keep their minimum; the empty bins are listed (ascending).
    uint32_t ne = 0;
    for (uint32_t i0 = 0; i0 < B; i0 += 32) {
      const uint32_t i = i0 + lane;
      const uint32_t x = i < B ? v[i] : 0u;
      const bool empty = i < B && x == kEmpty;
      if (i < B && !empty) code[i] = x;
      const uint32_t m = __ballot_sync(0xFFFFFFFFu, empty);
      if (empty) elist[ne + __popc(m & lanemask_lt_d())] = (uint16_t)i;
      ne += __popc(m);
    }
    const bool nonempty = ne < B;
    __syncwarp();
    if (!nonempty) {  // empty row: every code stays EMPTY
      for (uint32_t i = lane; i < B; i += 32) code[i] = kEmpty;
    } else if (ne) {
      // Pass 2: the probe chains of the empty bins, dynamically balanced over the lanes:
      // a lane that finds its donor takes the next listed bin, so every step of the
      // warp-uniform loop advances ~32 chains (a probe count per bin is geometric; a
      // static bin-per-lane split would wait for the longest chain of each round).  Each
      // step evaluates 4 consecutive probes of the lane's chain (independent hashes and
      // loads) and takes the first hit in chain order, amortising the bookkeeping.
      constexpr uint32_t kBatch = 4;  // divides kProbes
      uint32_t e = lane, a = 1, next = 32;
      uint32_t i = e < ne ? elist[e] : 0u;
      while (__any_sync(0xFFFFFFFFu, e < ne)) {
        const bool active = e < ne;
        bool hit = false;
        uint32_t x = kEmpty;
        if (active) {
          uint32_t jl = 0;
#pragma unroll
          for (uint32_t u = 0; u < kBatch; ++u) {
            const uint32_t j = __umulhi(fmix32(keys.s_dens ^ ((i << 8) | (a + u))), B);
            const uint32_t y = v[j];
            if (x == kEmpty) x = y;  // the first hit in chain order wins
            jl = j;
          }
          hit = x != kEmpty;
          if (!hit && a + kBatch > kProbes) {  // chain exhausted: circular scan from its last bin
            for (uint32_t m = 1; m <= B; ++m) {
              uint32_t jj = jl + m;
              if (jj >= B) jj -= B;
              x = v[jj];
              if (x != kEmpty) break;
            }
            hit = true;  // the row is non-empty, so the scan found a donor
          }
        }
        const uint32_t done = __ballot_sync(0xFFFFFFFFu, hit);
        if (hit) {
          code[i] = x;
          e = next + __popc(done & lanemask_lt_d());
          a = 1;
          if (e < ne) i = elist[e];
        } else if (active) {
          a += kBatch;
        }
        next += __popc(done);
      }
    }
    __syncwarp();
    if (kCodes)
      for (uint32_t i = lane; i < B; i += 32) codes[r * B + i] = code[i];

    // ---- H3: L table addresses ----
    if (kAddrs) write_addrs(code, nonempty, K, L, range, keys, out, n_rows, r, lane);
    __syncwarp();
  };

  // one warp per row, the block scheduler balances skewed row lengths; rows with <= skip_le
  // nonzeros belong to k_doph_sparse (their extents are read here anyway)
  // the rows k_doph_sparse listed: those over kHugeNnz from the front (lowest warp indices:
  // dispatched first, so the longest rows do not form the tail), the rest from the back
  const uint32_t nfront = long_rows ? long_rows[long_cap] : 0u;
  const uint32_t nback = long_rows ? long_rows[long_cap + 1] : 0u;
  if (long_rows && (uint64_t)nfront + nback <= long_cap) {
    for (uint32_t x = blockIdx.x * wpb + warp; x < nfront + nback; x += gridDim.x * wpb) {
      const uint64_t r = x < nfront ? long_rows[x] : long_rows[long_cap - 1 - (x - nfront)];
      do_row(r, row_ptr[r], row_ptr[r + 1]);
    }
    return;
  }
  for (uint64_t r = (uint64_t)blockIdx.x * wpb + warp; r < n_rows; r += (uint64_t)gridDim.x * wpb) {
    const int64_t e0 = row_ptr[r], e1 = row_ptr[r + 1];
    if (e1 - e0 > skip_le) do_row(r, e0, e1);
  }
}

// ---------------------------------------------------------------------------
// Very sparse rows (nnz <= kSparseNnz, B <= kSparseMaxB: the kdd12 shape, 11 nnz into
// 128 bins).  Probing costs ~B/|NE| probes per empty bin, each a dependent hash + load,
// with per-lane divergence; here the chains are tabulated once per CTA instead:
//   first[j*B + i] = the first position a <= T at which bin i's chain probes bin j
//                    (255: never), data-independent (HASHSPEC H2).
// An empty bin's donor is then the non-empty bin j minimising first[j*B + i] — the same
// bin the chain reaches first.  Lane l owns bins 4l..4l+3 of every 128-bin chunk: for each
// of the |NE| (<= nnz) non-empty bins j it loads the 4 table bytes of its bins in one word
// and keeps two packed 16-bit minima of (first << 8 | rank of j in the NE list)
// (__vminu2), so the argmin over j costs ~7 instructions per 4 bins, uniform, no
// divergence.  A bin whose T probes all miss falls back to the circular scan from its
// last probe, i.e. the first non-empty bin after it (a search in the sorted NE list).
// One warp per row; persistent CTAs (the table is built once per CTA).
constexpr uint32_t kSparseNnz = 32;
// listed rows longer than this go first to k_doph (webspam, A/B in one process: hash 1.178 ->
// 1.100 ms, graph 4.445 -> 4.368 ms; 2,048 and 8,192 the same within noise; a third class
// (rows over 1,024 next) 1.095 ms, not kept)
constexpr int64_t kHugeNnz = 4096;
constexpr uint32_t kSparseMaxB = 256;

__host__ __device__ __forceinline__ uint32_t sparse_stride(uint32_t B) { return (B + 127) & ~127u; }
__host__ __device__ __forceinline__ uint32_t sparse_warp_words(uint32_t B) {
  return 2 * B + (B + 3) / 4 + 8;  // v[B], code[B], u8 NE list, NE bitmap (<= 256 bins)
}
// the CTA tables: first[B][Bs] and jt[Bs] (each bin's T-th probe), in 32-bit words
__host__ __device__ __forceinline__ uint32_t sparse_table_words(uint32_t B) {
  return (B + 1) * sparse_stride(B) / 4;
}

template <bool kCodes, bool kAddrs>
__global__ void __launch_bounds__(kThreads, 8) k_doph_sparse(const int64_t* __restrict__ row_ptr,
                                                          const uint32_t* __restrict__ col_idx,
                                                          uint64_t n_rows, uint32_t K, uint32_t L,
                                                          uint32_t range, HashKeys keys,
                                                          uint32_t* __restrict__ codes, AddrOut out,
                                                          uint32_t* __restrict__ long_rows, uint32_t long_cap,
                                                          unsigned long long* __restrict__ next_chunk) {
  extern __shared__ uint32_t smem[];
  const uint32_t B = K * L;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const uint32_t Bs = sparse_stride(B);               // table row stride (bytes), 128-multiple
  uint8_t* first = reinterpret_cast<uint8_t*>(smem);  // [B][Bs], 255 = never
  uint8_t* jt = first + B * Bs;                        // [Bs] bin i's T-th (last) probe
  uint32_t* v = smem + sparse_table_words(B) + (size_t)warp * sparse_warp_words(B);
  uint32_t* code = v + B;
  uint8_t* nel = reinterpret_cast<uint8_t*>(code + B);  // non-empty bins, ascending
  uint32_t* nebits = code + B + (B + 3) / 4;            // [8] non-empty bins as a bitmap

  for (uint32_t x = threadIdx.x; x < B * Bs / 4; x += blockDim.x) smem[x] = 0xFFFFFFFFu;
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < B; i += blockDim.x) {
    for (uint32_t a = kProbes; a >= 1; --a)  // descending: the smallest position wins
      first[__umulhi(fmix32(keys.s_dens ^ ((i << 8) | a)), B) * Bs + i] = (uint8_t)a;
    jt[i] = (uint8_t)__umulhi(fmix32(keys.s_dens ^ ((i << 8) | kProbes)), B);
  }
  __syncthreads();

  const uint64_t nw = (uint64_t)gridDim.x * wpb;
  // chunks of 32 rows per warp (handed out by a global counter when next_chunk is set): one
  // coalesced read of their extents, then the sparse ones
  auto grab = [&](uint64_t cur) -> uint64_t {
    if (!next_chunk) return cur + nw * 32;
    unsigned long long c = 0;
    if (lane == 0) c = atomicAdd(next_chunk, 32ull);
    return __shfl_sync(0xFFFFFFFFu, c, 0);
  };
  for (uint64_t r0 = next_chunk ? grab(0) : ((uint64_t)blockIdx.x * wpb + warp) * 32; r0 < n_rows; r0 = grab(r0)) {
   const uint64_t rl = r0 + lane;
   const int64_t my_e0 = rl < n_rows ? row_ptr[rl] : 0, my_e1 = rl < n_rows ? row_ptr[rl + 1] : 0;
   uint32_t todo = __ballot_sync(0xFFFFFFFFu, rl < n_rows && my_e1 - my_e0 <= (int64_t)kSparseNnz);
   if (long_rows) {  // list the others for k_doph: rows over kHugeNnz from the front, the
                     // rest from the back (past long_cap in total they are counted only)
     const int64_t len = my_e1 - my_e0;
     const bool lg = rl < n_rows && len > (int64_t)kSparseNnz;
     const bool hg = lg && len > (int64_t)kHugeNnz;
     const uint32_t hm = __ballot_sync(0xFFFFFFFFu, hg), om = __ballot_sync(0xFFFFFFFFu, lg && !hg);
     if (hm | om) {
       uint32_t bh = 0, bo = 0;
       if (lane == 0) {
         if (hm) bh = atomicAdd(&long_rows[long_cap], (uint32_t)__popc(hm));
         if (om) bo = atomicAdd(&long_rows[long_cap + 1], (uint32_t)__popc(om));
       }
       bh = __shfl_sync(0xFFFFFFFFu, bh, 0);
       bo = __shfl_sync(0xFFFFFFFFu, bo, 0);
       if (hg) {
         const uint32_t x = bh + __popc(hm & lanemask_lt_d());
         if (x < long_cap) long_rows[x] = (uint32_t)rl;
       } else if (lg) {
         const uint32_t x = bo + __popc(om & lanemask_lt_d());
         if (x < long_cap) long_rows[long_cap - 1 - x] = (uint32_t)rl;  // (overlap: counted, then ignored)
       }
     }
   }
   while (todo) {  // the others are k_doph's
    const uint32_t src = __ffs(todo) - 1;
    todo &= todo - 1;
    const uint64_t r = r0 + src;
    const int64_t e0 = __shfl_sync(0xFFFFFFFFu, my_e0, src), e1 = __shfl_sync(0xFFFFFFFFu, my_e1, src);
    for (uint32_t i = lane; i < B; i += 32) v[i] = kEmpty;
    __syncwarp();
    if (e0 + (int64_t)lane < e1) bin_min(v, B, keys, col_idx[e0 + lane]);  // H1
    __syncwarp();
    // NE list (ascending bin order)
    uint32_t nne = 0;
    for (uint32_t i0 = 0; i0 < B; i0 += 32) {
      const uint32_t i = i0 + lane;
      const bool full = i < B && v[i] != kEmpty;
      const uint32_t mf = __ballot_sync(0xFFFFFFFFu, full);
      if (full) nel[nne + __popc(mf & lanemask_lt_d())] = (uint8_t)i;
      if (lane == 0) nebits[i0 >> 5] = mf;
      nne += __popc(mf);
    }
    __syncwarp();
    const bool nonempty = nne > 0;
    // H2 (R#4): per 128-bin chunk, lane l's bins 4l..4l+3 take the NE bin of smallest first
    for (uint32_t c0 = 0; c0 < B; c0 += 128) {
      const uint32_t ib = c0 + 4 * lane;
      uint32_t m01 = 0xFFFFFFFFu, m23 = 0xFFFFFFFFu;  // (first << 8 | NE rank) per bin, 16-bit
      for (uint32_t kk = 0; kk < nne; ++kk) {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(first + nel[kk] * Bs + ib);
        m01 = __vminu2(m01, __byte_perm(w, kk, 0x1404));  // bins ib, ib+1
        m23 = __vminu2(m23, __byte_perm(w, kk, 0x3424));  // bins ib+2, ib+3
      }
#pragma unroll
      for (uint32_t q = 0; q < 4; ++q) {
        const uint32_t i = ib + q;
        if (i >= B) break;
        uint32_t x = v[i];
        if (x == kEmpty && nonempty) {
          const uint32_t r16 = ((q < 2 ? m01 : m23) >> (16 * (q & 1))) & 0xFFFFu;
          uint32_t dj;
          if ((r16 >> 8) != 255) {
            dj = nel[r16 & 0xFF];
          } else {  // every probe missed: the first non-empty bin after the T-th probe, circularly
            const uint32_t nwb = (B + 31) >> 5;
            uint32_t jj = jt[i] + 1u;
            if (jj == B) jj = 0;
            uint32_t wi = jj >> 5, word = nebits[wi] & (0xFFFFFFFFu << (jj & 31));
            while (!word) {  // (the row is non-empty: a bit is found within nwb + 1 words)
              wi = wi + 1 == nwb ? 0u : wi + 1;
              word = nebits[wi];
            }
            dj = wi * 32 + __ffs(word) - 1;
          }
          x = v[dj];
        }
        code[i] = x;
      }
    }
    __syncwarp();
    if (kCodes)
      for (uint32_t i = lane; i < B; i += 32) codes[r * B + i] = code[i];
    if (kAddrs) write_addrs(code, nonempty, K, L, range, keys, out, n_rows, r, lane);
    __syncwarp();
   }
  }
}

// ---------------------------------------------------------------------------
// Rows that leave most of B > 256 bins empty (nnz <= B/2: the url shape, ~116 nnz into 512
// bins, ~100 non-empty).  Probing (k_doph) spends ~1/p dependent hash + load probes per
// empty bin, p = |NE|/B ~ 0.2, with divergent chain lengths (url: ~3,900 warp-instructions
// per row).  Here the chains are inverted once per CTA:
//   inv[j]   = kMidC entries (a << 11 | i) with probe(i, a) = j, taken in increasing a
//              (a <= kMidT1) until the list is full; short lists are padded with entries
//              that hit a dummy slot;
//   cover[i] = the depth up to which every probe of bin i's chain is listed (one less than
//              the first of its entries a full list dropped; else kMidT1).
// A row scatters, for each non-empty bin j, the key (a << 11 | j) of all kMidC entries of
// inv[j] into best[i] with shared-memory atomicMin (every list has the same length: lanes
// take (bin, 8-entry chunk) items, no divergence).  When best[i]'s depth is <= cover[i] it
// is the first position at which bin i's chain reaches a non-empty bin, so its j is the
// donor of R#4; otherwise (rare: ~0.8^cover[i]) the warp's lanes probe positions
// cover[i]+1..T in parallel (one ballot per 32 probes), then the circular scan.  Densified
// codes are written in place after every miss is resolved (a donor is always an originally
// non-empty bin, which nothing overwrites).  Lane l owns bins 128c + 4l .. +3 (16-byte
// shared-memory accesses, conflict-free).
constexpr uint32_t kMidMaxB = 2047;  // 11-bit bin field; B itself is the dummy slot
constexpr uint32_t kMidT1 = 31;      // deepest listed chain position (5-bit field)
constexpr uint32_t kMidC = 32;       // entries per inverted list (4 chunks of 8; FLASH_DOPH_MIDC: 8/16/32)
constexpr int kMidThreads = 512;

__host__ __device__ __forceinline__ uint32_t mid_pad(uint32_t B) { return (B + 127) & ~127u; }
__host__ __device__ __forceinline__ uint32_t mid_table_words(uint32_t B, uint32_t C) {
  return B * C / 2 + (B + 3) / 4;  // inv u16[B][C], cover u8[B]
}
__host__ __device__ __forceinline__ uint32_t mid_warp_words(uint32_t B) {
  // v[Bp] (codes in place), best[Bp + 4] (dummy slot B), NE list u16[B/2 + 2]
  return (mid_pad(B) + mid_pad(B) + 4 + (B / 2 + 2) / 2 + 3) & ~3u;  // (16-B aligned)
}

template <bool kCodes, bool kAddrs>
__global__ void __launch_bounds__(kMidThreads, 2) k_doph_mid(const int64_t* __restrict__ row_ptr,
                                                          const uint32_t* __restrict__ col_idx,
                                                          uint64_t n_rows, uint32_t K, uint32_t L,
                                                          uint32_t range, HashKeys keys,
                                                          uint32_t* __restrict__ codes, AddrOut out,
                                                          uint32_t T1, uint32_t C, int64_t mid_le,
                                                          unsigned long long* __restrict__ next_chunk) {
  extern __shared__ __align__(16) uint32_t smem[];
  const uint32_t B = K * L, Bp = mid_pad(B), nc = Bp >> 7;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const uint32_t nchk = C / 8;
  const uint4* inv = reinterpret_cast<const uint4*>(smem);                    // [B][C / 8]
  uint8_t* cover = reinterpret_cast<uint8_t*>(smem + B * C / 2);              // [B]
  uint32_t* v = smem + ((mid_table_words(B, C) + 3) & ~3u) + (size_t)warp * mid_warp_words(B);
  uint32_t* best = v + Bp;                                                     // [Bp + 4]
  uint16_t* nel = reinterpret_cast<uint16_t*>(best + Bp + 4);                 // [B / 2 + 2]
  uint4* v4 = reinterpret_cast<uint4*>(v);
  uint4* best4 = reinterpret_cast<uint4*>(best);
  const uint32_t* cover4 = reinterpret_cast<const uint32_t*>(cover);

  // ---- the CTA table, in increasing depth a (warp 0's v serves as the list cursors) ----
  {
    uint32_t* cnt = v - (size_t)warp * mid_warp_words(B);
    uint16_t* ent = reinterpret_cast<uint16_t*>(smem);
    const uint32_t pad = (31u << 11) | B;  // -> the dummy slot best[B]
    for (uint32_t x = threadIdx.x; x < B * C; x += blockDim.x) ent[x] = (uint16_t)pad;
    for (uint32_t j = threadIdx.x; j < B; j += blockDim.x) {
      cnt[j] = 0;
      cover[j] = (uint8_t)T1;
    }
    for (uint32_t a = 1; a <= T1; ++a) {
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < B; i += blockDim.x) {
        const uint32_t j = __umulhi(fmix32(keys.s_dens ^ ((i << 8) | a)), B);
        const uint32_t pos = atomicAdd(&cnt[j], 1u);
        if (pos < C) ent[j * C + pos] = (uint16_t)((a << 11) | i);
        else if (cover[i] == T1) cover[i] = (uint8_t)(a - 1);
      }
    }
    __syncthreads();
  }
  for (uint32_t x = lane; x < (Bp + 4) / 4; x += 32) best4[x] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
  __syncwarp();

  // 32-row chunks handed out dynamically (a global counter; with next_chunk null, statically):
  // warps whose chunks held longer rows take fewer, so no warp's share forms a tail
  const uint64_t nw = (uint64_t)gridDim.x * wpb;
  auto grab = [&](uint64_t cur) -> uint64_t {
    if (!next_chunk) return cur + nw * 32;
    unsigned long long c = 0;
    if (lane == 0) c = atomicAdd(next_chunk, 32ull);
    return __shfl_sync(0xFFFFFFFFu, c, 0);
  };
  for (uint64_t r0 = next_chunk ? grab(0) : ((uint64_t)blockIdx.x * wpb + warp) * 32; r0 < n_rows; r0 = grab(r0)) {
    const uint64_t rl = r0 + lane;
    const int64_t my_e0 = rl < n_rows ? row_ptr[rl] : 0, my_e1 = rl < n_rows ? row_ptr[rl + 1] : 0;
    uint32_t todo = __ballot_sync(0xFFFFFFFFu, rl < n_rows && my_e1 - my_e0 <= mid_le);
    while (todo) {  // the others are k_doph's
      const uint32_t src = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint64_t r = r0 + src;
      const int64_t e0 = __shfl_sync(0xFFFFFFFFu, my_e0, src), e1 = __shfl_sync(0xFFFFFFFFu, my_e1, src);
      for (uint32_t c = 0; c < nc; ++c) v4[c * 32 + lane] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
      __syncwarp();
      // ---- H1: 4 loads in flight per lane ----
      for (int64_t e = e0 + lane; e < e1; e += 128) {
        uint32_t cv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) cv[u] = e + 32 * u < e1 ? ld_stream(col_idx + e + 32 * u) : 0u;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (e + 32 * u < e1) bin_min(v, B, keys, cv[u]);
      }
      __syncwarp();
      // ---- the non-empty bins, listed in (bin mod 4, lane) order per chunk ----
      uint32_t nne = 0;
      for (uint32_t c = 0; c < nc; ++c) {
        const uint4 q = v4[c * 32 + lane];
        const uint32_t x[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) {
          const bool full = x[k] != kEmpty;  // (bins >= B stay EMPTY)
          const uint32_t m = __ballot_sync(0xFFFFFFFFu, full);
          if (full) nel[nne + __popc(m & lanemask_lt_d())] = (uint16_t)(c * 128 + 4 * lane + k);
          nne += __popc(m);
        }
      }
      __syncwarp();
      if (nne) {
        // ---- H2a: scatter (a << 11 | j) of the NE bins' lists, one 8-entry chunk per item ----
        const uint32_t s_best = (uint32_t)__cvta_generic_to_shared(best);
        for (uint32_t it = lane; it < nne * nchk; it += 32) {
          const uint32_t j = nel[nchk == 2 ? it >> 1 : (nchk == 1 ? it : it / nchk)];
          const uint4 q = inv[j * nchk + (it - (it / nchk) * nchk)];
          const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {  // per entry: mask, address, key, RED.MIN
            const uint32_t hi = w[u] >> 16;
            smem_min(s_best + ((w[u] & 0x7FFu) << 2), (w[u] & 0xF800u) | j);
            smem_min(s_best + ((hi & 0x7FFu) << 2), (hi & 0xF800u) | j);
          }
        }
        __syncwarp();
        // ---- H2b: bins the lists do not settle (no listed hit, or one deeper than cover[i])
        //      probe on from depth cover[i] + 1 on pre-densification v, one bin at a time, the
        //      warp's lanes evaluating 32 consecutive positions per ballot (a lane-parallel
        //      probing loop over the missed bins measured slower: url 10.9 vs 8.2 ms) ----
        for (uint32_t c = 0; c < nc; ++c) {
          const uint4 qv = v4[c * 32 + lane], qb = best4[c * 32 + lane];
          const uint32_t cov = cover4[c * 32 + lane];  // (bins >= B: never a miss)
          const uint32_t x[4] = {qv.x, qv.y, qv.z, qv.w}, kb[4] = {qb.x, qb.y, qb.z, qb.w};
          uint32_t mk = 0;
#pragma unroll
          for (uint32_t k = 0; k < 4; ++k) {
            const uint32_t i = c * 128 + 4 * lane + k;
            const uint32_t depth = kb[k] == kEmpty ? 32u : kb[k] >> 11;
            if (i < B && x[k] == kEmpty && depth > ((cov >> (8 * k)) & 0xFFu)) mk |= 1u << k;
          }
          uint32_t lm = __ballot_sync(0xFFFFFFFFu, mk != 0);
          while (lm) {  // warp-uniform: one missed bin at a time
            const uint32_t sl = __ffs(lm) - 1;
            const uint32_t smk = __shfl_sync(0xFFFFFFFFu, mk, sl);
            const uint32_t k = __ffs(smk) - 1;
            if (lane == sl) mk &= mk - 1;
            if ((smk & (smk - 1)) == 0) lm &= lm - 1;
            const uint32_t bi = c * 128 + 4 * sl + k;
            uint32_t donor = kEmpty;
            for (uint32_t a0 = cover[bi] + 1u; a0 <= kProbes && donor == kEmpty; a0 += 32) {
              const uint32_t a = a0 + lane;
              const uint32_t jp = __umulhi(fmix32(keys.s_dens ^ ((bi << 8) | a)), B);
              const bool hit = a <= kProbes && v[jp] != kEmpty;
              const uint32_t hm = __ballot_sync(0xFFFFFFFFu, hit);
              if (hm) donor = __shfl_sync(0xFFFFFFFFu, jp, __ffs(hm) - 1);
            }
            if (donor == kEmpty) {  // circular scan after the T-th probe (the row is non-empty)
              const uint32_t st = __umulhi(fmix32(keys.s_dens ^ ((bi << 8) | kProbes)), B) + 1;
              for (uint32_t o0 = 0; o0 < B && donor == kEmpty; o0 += 32) {
                uint32_t p = st + o0 + lane;
                while (p >= B) p -= B;
                const bool hit = o0 + lane < B && v[p] != kEmpty;
                const uint32_t hm = __ballot_sync(0xFFFFFFFFu, hit);
                if (hm) donor = __shfl_sync(0xFFFFFFFFu, p, __ffs(hm) - 1);
              }
            }
            if (lane == 0) best[bi] = donor;  // depth 0: taken as is below
          }
        }
        __syncwarp();
        // ---- H2c: densify in place, reset best ----
        for (uint32_t c = 0; c < nc; ++c) {
          uint4 qv = v4[c * 32 + lane];
          const uint4 qb = best4[c * 32 + lane];
          best4[c * 32 + lane] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
          const uint32_t base = c * 128 + 4 * lane;
          if (qv.x == kEmpty && base + 0 < B) qv.x = v[qb.x & 0x7FFu];
          if (qv.y == kEmpty && base + 1 < B) qv.y = v[qb.y & 0x7FFu];
          if (qv.z == kEmpty && base + 2 < B) qv.z = v[qb.z & 0x7FFu];
          if (qv.w == kEmpty && base + 3 < B) qv.w = v[qb.w & 0x7FFu];
          __syncwarp();  // (every lane's donor reads of this chunk precede its stores)
          v4[c * 32 + lane] = qv;
        }
        if (lane == 0) best[B] = kEmpty;
      }
      __syncwarp();
      if (kCodes)
        for (uint32_t i = lane; i < B; i += 32) codes[r * B + i] = v[i];
      if (kAddrs) write_addrs(v, nne > 0, K, L, range, keys, out, n_rows, r, lane);
      __syncwarp();
    }
  }
}

template <bool C, bool A>
int launch_t(const int64_t* row_ptr, const uint32_t* col_idx, uint64_t n_rows, uint32_t K,
             uint32_t L, uint32_t range, const HashKeys& keys, uint32_t* codes, const AddrOut& out,
             cudaStream_t s, uint32_t* long_rows, uint32_t long_cap) {
  const uint32_t B = K * L;
  int launched = 0;
  int64_t skip_le = -1;
  unsigned long long* chunk_ctr = nullptr;
  if (B <= kSparseMaxB) {  // rows with <= kSparseNnz nonzeros: the table-driven kernel
    const size_t smem = ((size_t)sparse_table_words(B) + (size_t)sparse_warp_words(B) * (kThreads / 32)) * 4;
    ensure_smem_attr((const void*)k_doph_sparse<C, A>, 100 * 1024, true);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_doph_sparse<C, A>, kThreads, smem);
    if (per_sm < 1) per_sm = 1;
    uint64_t blocks = (uint64_t)device_sms() * per_sm;
    const uint64_t need = (n_rows + kThreads - 1) / kThreads;  // 32 rows per warp-chunk
    if (blocks > need) blocks = need;
    // (the scratch: the list, its two counts, then an 8-byte chunk counter)
    unsigned long long* nc =
        long_rows ? reinterpret_cast<unsigned long long*>(long_rows + ((long_cap + 3) & ~1u)) : nullptr;
    if (long_rows) cudaMemsetAsync(long_rows + long_cap, 0, ((long_cap + 3) & ~1u) * 4 + 8 - long_cap * 4, s);
    k_doph_sparse<C, A><<<(unsigned)blocks, kThreads, smem, s>>>(row_ptr, col_idx, n_rows, K, L, range, keys,
                                                                 codes, out, long_rows, long_cap, nc);
    ++launched;
    skip_le = kSparseNnz;
  } else {
    // (only the sparse kernel lists the rows it leaves; the mid kernel takes the scratch's
    // first 8 bytes as its chunk counter)
    if (long_rows) chunk_ctr = reinterpret_cast<unsigned long long*>(long_rows);
    long_rows = nullptr;
  }
  if (B > kSparseMaxB && B <= kMidMaxB) {  // rows with <= B/2 nonzeros: the inverted-chain kernel
    // FLASH_DOPH_MID_LE (tests, tuning): the row-length cut, -1 = off; FLASH_DOPH_T1 (tests):
    // a shallower inverted depth T1 (more rows' bins take the probing path)
    const char* e = getenv("FLASH_DOPH_MID_LE");
    int64_t mid_le = e ? strtoll(e, nullptr, 10) : (int64_t)(B / 2);
    if (mid_le > (int64_t)(B / 2)) mid_le = B / 2;
    const char* et = getenv("FLASH_DOPH_T1");
    uint32_t T1 = et ? (uint32_t)strtoul(et, nullptr, 10) : kMidT1;
    T1 = T1 < 1 ? 1 : (T1 > kMidT1 ? kMidT1 : T1);
    const char* ec = getenv("FLASH_DOPH_MIDC");
    uint32_t mc = ec ? (uint32_t)strtoul(ec, nullptr, 10) : kMidC;
    mc = mc <= 8 ? 8 : (mc <= 16 ? 16 : 32);
    if (mid_le >= 0) {
      // as many warps (<= 16) as fit beside the table in one CTA's shared memory
      const size_t tbytes = (size_t)((mid_table_words(B, mc) + 3) & ~3u) * 4, wbytes = (size_t)mid_warp_words(B) * 4;
      const size_t cap = 227 * 1024;
      const uint32_t wpb = tbytes + 4 * wbytes <= cap ? (uint32_t)std::min<size_t>(kMidThreads / 32, (cap - tbytes) / wbytes) : 0;
      const size_t smem = tbytes + wpb * wbytes;
      if (wpb && ensure_smem_attr((const void*)k_doph_mid<C, A>, smem, true)) {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_doph_mid<C, A>, wpb * 32, smem);
        if (per_sm >= 1) {
          uint64_t blocks = (uint64_t)device_sms() * per_sm;
          const uint64_t need = (n_rows + wpb * 32 - 1) / (wpb * 32);  // 32 rows per warp-chunk
          if (blocks > need) blocks = need;
          if (blocks) {
            unsigned long long* nc = chunk_ctr;
            if (nc) cudaMemsetAsync(nc, 0, sizeof(unsigned long long), s);
            k_doph_mid<C, A><<<(unsigned)blocks, wpb * 32, smem, s>>>(row_ptr, col_idx, n_rows, K, L, range,
                                                                      keys, codes, out, T1, mc, mid_le, nc);
            ++launched;
          }
          skip_le = mid_le;
        }
      }
    }
  }
  const size_t per_warp = (size_t)warp_words(B) * sizeof(uint32_t);
  int wpb = (int)((96 * 1024) / per_warp);
  wpb = wpb < 1 ? 1 : (wpb > kThreads / 32 ? kThreads / 32 : wpb);
  const size_t smem = per_warp * wpb;
  // the column stream bypasses L1 (no_allocate): give the whole carveout to shared memory,
  // so the per-warp bin arrays never cap the resident warps below the thread limit
  ensure_smem_attr((const void*)k_doph<C, A>, smem, true);
  uint64_t blocks = (n_rows + wpb - 1) / wpb;  // one warp per row: the block scheduler balances
  // the skewed row lengths; with the sparse kernel in use, a grid-stride cap keeps the launch
  // from scheduling millions of CTAs that would only skip sparse rows
  const uint64_t cap = skip_le >= 0 ? 65536ull : 0x7FFFFFFFull;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) return launched;
  k_doph<C, A><<<(unsigned)blocks, wpb * 32, smem, s>>>(row_ptr, col_idx, n_rows, K, L, range, keys,
                                                         codes, out, skip_le, long_rows, long_cap);
  return launched + 1;
}

}  // namespace

int launch_doph(const int64_t* row_ptr, const uint32_t* col_idx, uint64_t n_rows, uint32_t K,
                uint32_t L, uint32_t range, const HashKeys& keys, uint32_t* codes, const AddrOut& out,
                cudaStream_t s, uint32_t* long_rows, uint32_t long_cap) {
  const bool addrs = out.addrs || out.peers;
  if (codes && addrs)
    return launch_t<true, true>(row_ptr, col_idx, n_rows, K, L, range, keys, codes, out, s, long_rows, long_cap);
  if (codes)
    return launch_t<true, false>(row_ptr, col_idx, n_rows, K, L, range, keys, codes, out, s, long_rows, long_cap);
  return launch_t<false, true>(row_ptr, col_idx, n_rows, K, L, range, keys, codes, out, s, long_rows, long_cap);
}

}  // namespace flash
