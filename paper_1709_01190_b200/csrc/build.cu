// build.cu — B1-B2: the adding phase (Alg. 2) with deterministic bottom-R
// reservoirs (north_star; R#7, R#9, R#10), sm_100a.
//
// For every bucket (t, b):  S = old kept ids ∪ newly arriving ids,
//   arrivals[t][b] += #new arrivals                              (ReservoirCounter)
//   kept(t,b) = the min(|S|, R) members of S with smallest (prio(t,b,id), id), ascending id.
// Using old KEPT ids instead of all old arrivals is exact: an id outside the bottom-R of
// a subset can never enter the bottom-R of a superset.  The result does not depend on the
// order in which ids arrive or on atomic ordering: the pool order written by the
// scatter is erased by the per-bucket (prio, id) selection and the final id sort.
//
// Kernels: k_count (B1 histogram) -> k_pool_sizes -> 2 scans -> k_fill_old / k_fill_new
// (scatter every member into a bucket-contiguous pool; or the shared-memory / table-major
// variants) -> k_select_small (buckets with <= 32 members: a warp per 32 buckets, staged
// in shared memory and insertion-sorted) -> k_select_mid (33..256 members, registers) ->
// k_select_warp (one warp per bucket up to 512 members: priority-threshold filter to
// ~R+6sqrt(R) survivors, shared-memory bitonic sort) -> k_select_big (one CTA per larger or
// leftover bucket: the same filter with the whole CTA, exact radix select on the priority
// as the fallback).
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>

#include "flash_internal.cuh"

namespace flash {
namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr int kSelThreads = 256;
constexpr int kBigThreads = 1024;     // k_select_big: one wide CTA per large bucket
constexpr uint32_t kWarpMax = 512;    // buckets above this go to the CTA path
constexpr uint32_t kWarpCap = 1024;   // per-warp sort buffer (u64 keys)
constexpr uint32_t kBigCap = 4096;    // CTA path: kept ids sorted in smem (R <= kBigCap)
constexpr uint32_t kMidMax = 256;     // register path (k_select_mid): m, R <= kMidMax

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ uint32_t pow2_ceil(uint32_t x) {
  return x <= 1 ? 1u : 1u << (32 - __clz(x - 1));
}

// Ascending bitonic sort of one u64 key per lane.
__device__ __forceinline__ uint64_t warp_sort32(uint64_t key) {
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll
  for (uint32_t k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      const uint64_t other = __shfl_xor_sync(kFull, key, j);
      const bool up = (lane & k) == 0;
      const bool lower = (lane & j) == 0;
      key = (lower == up) ? (key < other ? key : other) : (key > other ? key : other);
    }
  }
  return key;
}

// Ascending bitonic sort of one u32 key per lane.
__device__ __forceinline__ uint32_t warp_sort32_u32(uint32_t key) {
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll
  for (uint32_t k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      const uint32_t other = __shfl_xor_sync(kFull, key, j);
      const bool keep_min = ((lane & k) == 0) == ((lane & j) == 0);
      key = keep_min ? min(key, other) : max(key, other);
    }
  }
  return key;
}

// Ascending bitonic sort of n (power of two) keys in shared memory by one warp.
template <typename T>
__device__ void warp_bitonic(T* a, uint32_t n) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t k = 2; k <= n; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t p = lane; p < (n >> 1); p += 32) {
        const uint32_t i = ((p & ~(j - 1)) << 1) | (p & (j - 1));
        const uint32_t ixj = i + j;
        const T x = a[i], y = a[ixj];
        const bool up = (i & k) == 0;
        if ((x > y) == up) { a[i] = y; a[ixj] = x; }
      }
      __syncwarp();
    }
  }
}

// Same, by a whole CTA.
template <typename T>
__device__ void block_bitonic(T* a, uint32_t n) {
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

// B1: per-bucket arrival histogram of the new rows (warp per row, lanes over tables).
__global__ void k_count(const uint32_t* __restrict__ addrs, uint64_t n, uint32_t L, uint32_t acol0,
                        uint32_t range, uint32_t t0, uint32_t t1, uint32_t shared, uint32_t* __restrict__ cnt,
                        unsigned long long* err) {
  const uint32_t lim = shared ? shared : range;  // shared: addrs are reservoir indices
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t r = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += nw) {
    for (uint32_t t = t0 + lane; t < t1; t += 32) {
      const uint32_t a = addrs[r * L + t - acol0];
      if (a == kEmpty) continue;
      if (a >= lim) { atomicAdd(err, 1ull); continue; }
      atomicAdd(&cnt[shared ? a : t * range + a], 1u);
    }
  }
}

// Table-major build (large indexes).  When the per-bucket arrays (cursor 4 B + pool
// offset 8 B per bucket) outgrow L2, the row-major passes above touch every table's arrays
// from every warp and each atomic misses L2.  Instead the window's addresses are first
// transposed to [W][n] (k_transpose_cols), and the histogram / scatter kernels run with a
// table-major grid (block b covers table b / chunks, rows of chunk b % chunks): blocks are
// dispatched in order, so the resident blocks share one or two tables whose arrays stay
// L2-resident while every row passes through.
constexpr uint32_t kTmRows = 4096;  // rows per block in the table-major passes

__global__ void __launch_bounds__(256) k_transpose_cols(const uint32_t* __restrict__ addrs, uint64_t n,
                                                        uint32_t astride, uint32_t c0, uint32_t W,
                                                        uint32_t* __restrict__ out) {
  __shared__ uint32_t tile[32][257];
  const uint64_t r0 = (uint64_t)blockIdx.x * 256;
  const uint32_t nr = (uint32_t)(n - r0 < 256 ? n - r0 : 256);
  for (uint32_t cb = 0; cb < W; cb += 32) {
    const uint32_t wc = W - cb < 32 ? W - cb : 32;
    for (uint32_t k = threadIdx.x; k < nr * wc; k += 256) {  // row-major reads
      const uint32_t rr = k / wc, cc = k - rr * wc;
      tile[cc][rr] = addrs[(r0 + rr) * astride + c0 + cb + cc];
    }
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < 256 * wc; k += 256) {  // column-major writes
      const uint32_t cc = k >> 8, rr = k & 255;
      if (rr < nr) out[(uint64_t)(cb + cc) * n + r0 + rr] = tile[cc][rr];
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) k_count_tm(const uint32_t* __restrict__ addrsT, uint64_t n, uint32_t t0,
                                                  uint32_t range, uint32_t chunks, uint32_t* __restrict__ cnt,
                                                  unsigned long long* err) {
  const uint32_t j = blockIdx.x / chunks, ch = blockIdx.x - j * chunks;
  const uint64_t r0 = (uint64_t)ch * kTmRows;
  const uint64_t r1 = n - r0 < kTmRows ? n : r0 + kTmRows;
  const uint32_t* col = addrsT + (uint64_t)j * n;
  uint32_t* c = cnt + (uint64_t)(t0 + j) * range;
  for (uint64_t r = r0 + threadIdx.x; r < r1; r += 4 * 256) {
    uint32_t a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = r + u * 256 < r1 ? col[r + u * 256] : kEmpty;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (a[u] == kEmpty) continue;
      if (a[u] >= range) atomicAdd(err, 1ull);
      else atomicAdd(&c[a[u]], 1u);
    }
  }
}

__global__ void __launch_bounds__(256) k_fill_tm(const uint32_t* __restrict__ addrsT, uint64_t n, uint32_t t0,
                                                 uint32_t range, uint32_t chunks, uint32_t id_base,
                                                 uint32_t* __restrict__ cursor, const uint64_t* __restrict__ pool_off,
                                                 uint32_t* __restrict__ pool) {
  const uint32_t j = blockIdx.x / chunks, ch = blockIdx.x - j * chunks;
  const uint64_t r0 = (uint64_t)ch * kTmRows;
  const uint64_t r1 = n - r0 < kTmRows ? n : r0 + kTmRows;
  const uint32_t* col = addrsT + (uint64_t)j * n;
  const uint64_t tb = (uint64_t)(t0 + j) * range;
  for (uint64_t r = r0 + threadIdx.x; r < r1; r += 4 * 256) {
    uint32_t a[4], pos[4];
    uint64_t po[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = r + u * 256 < r1 ? col[r + u * 256] : kEmpty;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (a[u] < range) {
        pos[u] = atomicAdd(&cursor[tb + a[u]], 1u);
        po[u] = pool_off[tb + a[u]];
      }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (a[u] < range) pool[po[u] + pos[u]] = id_base + (uint32_t)(r + u * 256);
  }
}

// Grouped table-major passes (fresh builds of tables whose per-bucket arrays do not fit
// L2, e.g. kdd12: 32 tables x 2^20 buckets, ~143 arrivals per bucket).  The plain
// table-major scatter (k_count_tm / k_fill_tm) issues one global atomic and one isolated
// 4-B store per (table, row) into a 600 MB-per-table pool, so almost every store is a
// partial-sector write to HBM.  Instead the (table, row) entries are first partitioned by
// bucket GROUP (2^gshift consecutive buckets, <= 2048 groups per table, so each chunk's
// CTA has <= 2048 open output runs and the partial sectors combine in L2):
//   k_gcount    CTA per (table, 2^21-row chunk): group histogram in shared memory;
//   scan        (table, group, chunk)-major exclusive scan -> each chunk's slot range in
//               every group (the entries of a group are contiguous, chunks in order);
//   k_gscatter  the same CTAs write packed entries (bucket within the group << 21 | row
//               within the chunk) into their group slots — runs of ~250 entries;
//   k_gplace    1024-thread CTA per group, one per SM: counts its buckets (the arrivals,
//               into `cursor` for k_pool_sizes), and places its rows bucket by bucket into
//               the pool range the group occupies — exactly where the later exclusive scan
//               of the bucket counts puts these buckets (a fresh build has no old kept ids,
//               and group order is bucket order); the 148 ranges in flight (~290 KB each for
//               kdd12) stay in L2, so the scattered stores combine there.
// The bucket-contiguous pool then goes through the usual k_pool_sizes / scans / selects.
constexpr uint32_t kGChunkLog2 = 21;  // rows per chunk: local row ids in 21 bits
constexpr uint32_t kGMaxGroups = 2048;
constexpr int kGThreads = 1024;
constexpr int kGPlaceThreads = 1024;

struct GroupGeom {
  uint32_t gshift, ng, nch;
};

GroupGeom group_geom(uint32_t range, uint64_t n) {
  uint32_t gs = 7;
  while ((((uint64_t)range + (1ull << gs) - 1) >> gs) > kGMaxGroups) ++gs;
  return {gs, (uint32_t)(((uint64_t)range + (1ull << gs) - 1) >> gs),
          (uint32_t)((n + (1ull << kGChunkLog2) - 1) >> kGChunkLog2)};
}

__global__ void __launch_bounds__(kGThreads) k_gcount(const uint32_t* __restrict__ addrsT, uint64_t n,
                                                      uint32_t range, GroupGeom g, uint64_t* __restrict__ ghist,
                                                      unsigned long long* err) {
  extern __shared__ uint32_t gcnt[];  // [ng]
  const uint32_t j = blockIdx.x / g.nch, c = blockIdx.x - j * g.nch;
  for (uint32_t i = threadIdx.x; i < g.ng; i += blockDim.x) gcnt[i] = 0;
  __syncthreads();
  const uint64_t r0 = (uint64_t)c << kGChunkLog2;
  const uint64_t r1 = n - r0 < (1ull << kGChunkLog2) ? n : r0 + (1ull << kGChunkLog2);
  const uint32_t* col = addrsT + (uint64_t)j * n;
  for (uint64_t r = r0 + threadIdx.x; r < r1; r += 4 * kGThreads) {
    uint32_t a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = r + u * kGThreads < r1 ? col[r + u * kGThreads] : kEmpty;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (a[u] < range) atomicAdd(&gcnt[a[u] >> g.gshift], 1u);
      else if (a[u] != kEmpty) atomicAdd(err, 1ull);
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < g.ng; i += blockDim.x) ghist[((uint64_t)j * g.ng + i) * g.nch + c] = gcnt[i];
}

// (tiles of kGTile rows are counting-sorted by group in shared memory first, so each
// warp store writes runs of one group's consecutive slots)
// (8 K-row tiles in 512-thread CTAs, two per SM, measured slower: kdd12 insert 204.7 vs
// 189.4 ms)
constexpr uint32_t kGTile = 16384;
constexpr int kGSThreads = kGThreads;
constexpr int kGSMinBlocks = 1;

__host__ __device__ inline size_t gscatter_smem(uint32_t ng) {
  return (size_t)ng * (8 + 4 + 4) + (size_t)kGTile * (4 + 2);
}

__global__ void __launch_bounds__(kGSThreads, kGSMinBlocks) k_gscatter(const uint32_t* __restrict__ addrsT, uint64_t n,
                                                           uint32_t range, GroupGeom g,
                                                           const uint64_t* __restrict__ goffs, uint32_t* __restrict__ ent) {
  // [ng] each group's next slot in this chunk; during a tile's write-out, minus the group's
  // start in the tile's staging order (so an entry's slot is gbase[gi] + its stage index)
  extern __shared__ uint64_t gbase[];
  uint32_t* tcnt = reinterpret_cast<uint32_t*>(gbase + g.ng);       // [ng] this tile's counts
  uint32_t* toff = tcnt + g.ng;                                     // [ng] this tile's group starts
  uint32_t* stage = toff + g.ng;                                    // [kGTile] entries, by group
  uint16_t* sgrp = reinterpret_cast<uint16_t*>(stage + kGTile);     // [kGTile] their groups
  __shared__ uint32_t wsum[kGSThreads / 32];
  constexpr uint32_t E = kGTile / kGSThreads;
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t j = blockIdx.x / g.nch, c = blockIdx.x - j * g.nch;
  for (uint32_t i = threadIdx.x; i < g.ng; i += blockDim.x) gbase[i] = goffs[((uint64_t)j * g.ng + i) * g.nch + c];
  const uint64_t r0 = (uint64_t)c << kGChunkLog2;
  const uint64_t r1 = n - r0 < (1ull << kGChunkLog2) ? n : r0 + (1ull << kGChunkLog2);
  const uint32_t* col = addrsT + (uint64_t)j * n;
  const uint32_t gmask = (1u << g.gshift) - 1;
  const uint32_t gpt = (g.ng + kGSThreads - 1) / kGSThreads;  // groups per thread in the scan
  for (uint64_t t0 = r0; t0 < r1; t0 += kGTile) {
    for (uint32_t i = threadIdx.x; i < g.ng; i += blockDim.x) tcnt[i] = 0;
    uint32_t a[E], rk[E];
#pragma unroll
    for (uint32_t u = 0; u < E; ++u) {
      const uint64_t r = t0 + u * kGSThreads + threadIdx.x;
      a[u] = r < r1 ? col[r] : kEmpty;
    }
    __syncthreads();
#pragma unroll
    for (uint32_t u = 0; u < E; ++u)
      if (a[u] < range) rk[u] = atomicAdd(&tcnt[a[u] >> g.gshift], 1u);
    __syncthreads();
    // exclusive scan of the tile's group counts (thread t: groups [t*gpt, t*gpt + gpt))
    uint32_t run = 0;
    for (uint32_t q = 0; q < gpt; ++q) run += threadIdx.x * gpt + q < g.ng ? tcnt[threadIdx.x * gpt + q] : 0u;
    uint32_t x = run;
#pragma unroll
    for (uint32_t o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wib] = x;
    __syncthreads();
    uint32_t before = 0;
    for (uint32_t w = 0; w < wib; ++w) before += wsum[w];
    uint32_t pos = before + x - run;
    for (uint32_t q = 0; q < gpt; ++q) {
      const uint32_t gi = threadIdx.x * gpt + q;
      if (gi < g.ng) {
        toff[gi] = pos;
        gbase[gi] -= pos;
        pos += tcnt[gi];
      }
    }
    __syncthreads();
    const uint32_t tot = toff[g.ng - 1] + tcnt[g.ng - 1];
#pragma unroll
    for (uint32_t u = 0; u < E; ++u)
      if (a[u] < range) {
        const uint32_t gi = a[u] >> g.gshift;
        const uint32_t s = toff[gi] + rk[u];
        stage[s] = ((a[u] & gmask) << kGChunkLog2) | (uint32_t)(t0 + u * kGSThreads + threadIdx.x - r0);
        sgrp[s] = (uint16_t)gi;
      }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < tot; i += blockDim.x) ent[gbase[sgrp[i]] + i] = stage[i];
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < g.ng; i += blockDim.x) gbase[i] += toff[i] + tcnt[i];
  }
}

__host__ __device__ inline size_t gplace_smem(uint32_t gshift, uint32_t nch) {
  return (size_t)(nch + 1) * 8 + ((size_t)4 << gshift);
}

// kMode 0: count each group's buckets into `cursor` (the arrivals k_pool_sizes adds);
// 1: place the rows, bucket b's slots starting at pool_off[b] (the scan of the counts, which
// for a fresh build is exactly where the group ranges of k_gscatter put them); 2: both in
// one pass (the bucket starts from a block scan of the counts; when nothing has to run
// beside the placement)
template <int kMode>
__global__ void __launch_bounds__(kGPlaceThreads, 1) k_gplace(uint32_t W, uint32_t t0, uint32_t range, GroupGeom g,
                                                              const uint64_t* __restrict__ goffs,
                                                              const uint32_t* __restrict__ ent, uint32_t id_base,
                                                              uint32_t* __restrict__ cursor,
                                                              const uint64_t* __restrict__ pool_off,
                                                              uint32_t* __restrict__ pool) {
  extern __shared__ uint64_t co[];                                   // [nch + 1] chunk slot ranges
  uint32_t* bc = reinterpret_cast<uint32_t*>(co + g.nch + 1);        // [2^gshift] counts / cursors
  const uint32_t gsz = 1u << g.gshift;
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint64_t ngroups = (uint64_t)W * g.ng;
  for (uint64_t gid = blockIdx.x; gid < ngroups; gid += gridDim.x) {
    const uint32_t j = (uint32_t)(gid / g.ng), gi = (uint32_t)(gid - (uint64_t)j * g.ng);
    const uint32_t b0 = gi << g.gshift;
    const uint32_t nbk = range - b0 < gsz ? range - b0 : gsz;
    const uint64_t tb = (uint64_t)(t0 + j) * range + b0;
    for (uint32_t c = threadIdx.x; c <= g.nch; c += blockDim.x) co[c] = goffs[gid * g.nch + c];
    __syncthreads();
    const uint64_t e0 = co[0], e1 = co[g.nch];
    if (kMode != 1) {
      for (uint32_t b = threadIdx.x; b < gsz; b += blockDim.x) bc[b] = 0;
      __syncthreads();
      // 4 entry loads in flight per thread before their counter updates
      for (uint64_t p0 = e0 + threadIdx.x; p0 < e1; p0 += 4 * (uint64_t)blockDim.x) {
        uint32_t ev[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint64_t p = p0 + (uint64_t)u * blockDim.x;
          ev[u] = p < e1 ? ent[p] : 0xFFFFFFFFu;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (ev[u] != 0xFFFFFFFFu) atomicAdd(&bc[ev[u] >> kGChunkLog2], 1u);
      }
      __syncthreads();
      for (uint32_t b = threadIdx.x; b < nbk; b += blockDim.x) cursor[tb + b] = bc[b];
      __syncthreads();
      if (kMode == 0) continue;
      // exclusive scan of the group's counts (thread t owns buckets [t*per, t*per + per))
      __shared__ uint32_t wsum[kGPlaceThreads / 32];
      const uint32_t per = (gsz + kGPlaceThreads - 1) / kGPlaceThreads;
      const uint32_t bl = threadIdx.x * per;
      uint32_t run = 0;
      for (uint32_t q = 0; q < per && bl + q < gsz; ++q) run += bc[bl + q];
      uint32_t x = run;
#pragma unroll
      for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) wsum[wib] = x;
      __syncthreads();
      uint32_t pos = x - run;
      for (uint32_t w = 0; w < wib; ++w) pos += wsum[w];
      for (uint32_t q = 0; q < per && bl + q < gsz; ++q) {
        const uint32_t cnt = bc[bl + q];
        bc[bl + q] = pos;
        pos += cnt;
      }
    } else {
      for (uint32_t b = threadIdx.x; b < nbk; b += blockDim.x) bc[b] = (uint32_t)(pool_off[tb + b] - e0);
    }
    __syncthreads();
    // place the rows: each warp walks a contiguous range of 32-slot blocks, finding the chunk
    // of its first slot by a binary search over the chunk ranges and advancing it from there
    // (a chunk's entries carry its rows' low 21 bits; a block straddles few chunk ends)
    const uint64_t nblk = (e1 - e0 + 31) >> 5;
    const uint64_t wb0 = nblk * wib / (kGPlaceThreads / 32), wb1 = nblk * (wib + 1) / (kGPlaceThreads / 32);
    uint32_t c = 0;
    if (wb0 < wb1) {
      const uint64_t pb = e0 + (wb0 << 5);
      uint32_t hi = g.nch;  // the chunk c with co[c] <= pb < co[c + 1]
      while (hi - c > 1) {
        const uint32_t mid = (c + hi) >> 1;
        if (co[mid] <= pb) c = mid;
        else hi = mid;
      }
    }
    for (uint64_t blk0 = wb0; blk0 < wb1; blk0 += 4) {  // 4 blocks' entry loads in flight per lane
      uint32_t ev[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint64_t p = e0 + ((blk0 + u) << 5) + lane;
        ev[u] = blk0 + u < wb1 && p < e1 ? ent[p] : 0u;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (blk0 + u >= wb1) break;
        const uint64_t pb = e0 + ((blk0 + u) << 5);
        while (co[c + 1] <= pb) ++c;
        const uint64_t p = pb + lane;
        if (p < e1) {
          uint32_t cl = c;
          while (co[cl + 1] <= p) ++cl;
          const uint32_t e = ev[u];
          const uint32_t slot = atomicAdd(&bc[e >> kGChunkLog2], 1u);
          pool[e0 + slot] = id_base + (cl << kGChunkLog2) + (e & ((1u << kGChunkLog2) - 1));
        }
      }
    }
    __syncthreads();
  }
}

// Shared-memory build passes (tables whose bucket counters fit shared memory, e.g. webspam /
// url: 2^15 buckets).  Global L2 atomics cap k_count / k_fill_new at ~1 atomic per L2 slice
// per clock; here the W tables' (table, row) pairs — units j*n + r, table-major — are cut
// into C equal ranges, one 1024-thread CTA each (C = one per SM when every table's pool
// region fits L2 together, so no SM idles for want of a whole table slice).  A CTA's range
// is one or more segments (j, [r0, r1)); for each it histograms the transposed address
// column in shared memory and publishes the segment histogram (hbuf slot b + j: a table's
// segments have consecutive slots, in row order) plus the table's arrival totals.  The
// scatter pass then starts each segment's bucket cursors at the bucket's old kept count
// plus the earlier segments' counts, so the pool positions are disjoint without global
// atomics.
constexpr uint32_t kSmemBuildThreads = 1024;
constexpr uint32_t kSmemBuildMaxRange = 40960;  // 160 KB of u32 counters

// the CTA whose unit range holds unit x: the largest b with floor(b*U/C) <= x
__host__ __device__ __forceinline__ uint64_t cta_of_unit(uint64_t x, uint64_t U, uint64_t C) {
  return ((x + 1) * C - 1) / U;
}

__global__ void __launch_bounds__(kSmemBuildThreads) k_count_smem(const uint32_t* __restrict__ addrsT, uint64_t n,
                                                                  uint32_t t0, uint32_t range, uint32_t W, uint32_t C,
                                                                  uint32_t* __restrict__ cursor,
                                                                  uint32_t* __restrict__ hbuf,
                                                                  unsigned long long* err) {
  extern __shared__ uint32_t hsm[];  // [range]
  const uint64_t U = (uint64_t)W * n, b = blockIdx.x;
  const uint64_t u0 = b * U / C, u1 = (b + 1) * U / C;
  if (u0 >= u1) return;
  for (uint32_t j = (uint32_t)(u0 / n); j <= (uint32_t)((u1 - 1) / n); ++j) {
    const uint64_t r0 = max(u0, (uint64_t)j * n) - (uint64_t)j * n;
    const uint64_t r1 = min(u1, (uint64_t)(j + 1) * n) - (uint64_t)j * n;
    const uint32_t* col = addrsT + (uint64_t)j * n;
    for (uint32_t bb = threadIdx.x; bb < range; bb += blockDim.x) hsm[bb] = 0;
    __syncthreads();
    for (uint64_t r = r0 + threadIdx.x; r < r1; r += 4ull * blockDim.x) {
      uint32_t a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = r + u * blockDim.x < r1 ? col[r + u * blockDim.x] : kEmpty;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (a[u] == kEmpty) continue;
        if (a[u] >= range) atomicAdd(err, 1ull);
        else atomicAdd(&hsm[a[u]], 1u);
      }
    }
    __syncthreads();
    uint32_t* hb = hbuf + (b + j) * range;
    uint32_t* cur = cursor + (uint64_t)(t0 + j) * range;
    for (uint32_t bb = threadIdx.x; bb < range; bb += blockDim.x) {
      const uint32_t v = hsm[bb];
      hb[bb] = v;
      if (v) atomicAdd(&cur[bb], v);
    }
    __syncthreads();
  }
}

// Each segment's first pool position in every bucket of its table, relative to the table's
// pool start: the bucket's offset, then its old kept ids (their count is in cursor after
// k_pool_sizes), then the earlier segments' arrivals — an exclusive scan over the table's
// segments, written over the segment histograms.
__global__ void k_slice_bases(uint32_t W, uint32_t t0, uint32_t range, uint64_t n, uint32_t C,
                              const uint32_t* __restrict__ cursor, const uint64_t* __restrict__ pool_off,
                              uint32_t* __restrict__ hbuf) {
  const uint64_t total = (uint64_t)W * range, U = (uint64_t)W * n;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t j = (uint32_t)(x / range), b = (uint32_t)(x - (uint64_t)j * range);
    const uint64_t tb = (uint64_t)(t0 + j) * range;
    const uint64_t s0 = cta_of_unit((uint64_t)j * n, U, C) + j, s1 = cta_of_unit((uint64_t)(j + 1) * n - 1, U, C) + j + 1;
    uint32_t run = (uint32_t)(pool_off[tb + b] - pool_off[tb]) + cursor[tb + b];
    uint32_t* h = hbuf + b;
    for (uint64_t c0 = s0; c0 < s1; c0 += 8) {  // 8 independent loads in flight
      uint32_t v[8];
#pragma unroll
      for (uint32_t u = 0; u < 8; ++u) v[u] = c0 + u < s1 ? h[(c0 + u) * range] : 0u;
#pragma unroll
      for (uint32_t u = 0; u < 8; ++u) {
        if (c0 + u < s1) h[(c0 + u) * range] = run;
        run += v[u];
      }
    }
  }
}

__global__ void __launch_bounds__(kSmemBuildThreads) k_fill_smem(const uint32_t* __restrict__ addrsT, uint64_t n,
                                                                 uint32_t t0, uint32_t range, uint32_t W, uint32_t C,
                                                                 uint32_t id_base, const uint32_t* __restrict__ cursor,
                                                                 const uint32_t* __restrict__ hbuf,
                                                                 const uint64_t* __restrict__ pool_off,
                                                                 uint32_t* __restrict__ pool, int prefixed) {
  // [range] this segment's next pool position in each bucket, relative to the table's pool
  // start (a table's pool holds < 2^32 entries: its rows' arrivals plus its old kept ids)
  extern __shared__ uint32_t csm[];
  const uint64_t U = (uint64_t)W * n, cb = blockIdx.x;
  const uint64_t u0 = cb * U / C, u1 = (cb + 1) * U / C;
  if (u0 >= u1) return;
  const uint32_t bd = blockDim.x;
  for (uint32_t j = (uint32_t)(u0 / n); j <= (uint32_t)((u1 - 1) / n); ++j) {
    const uint64_t r0 = max(u0, (uint64_t)j * n) - (uint64_t)j * n;
    const uint64_t r1 = min(u1, (uint64_t)(j + 1) * n) - (uint64_t)j * n;
    const uint64_t tb = (uint64_t)(t0 + j) * range;
    const uint64_t pbase = pool_off[tb];
    const uint32_t* col = addrsT + (uint64_t)j * n;
    const uint64_t slot = cb + j;
    if (prefixed) {  // k_slice_bases turned the segment histograms into first positions
      for (uint32_t b = threadIdx.x; b < range; b += bd) csm[b] = hbuf[slot * range + b];
    } else {  // few segments per table: the same scan, here
      const uint64_t s0 = cta_of_unit((uint64_t)j * n, U, C) + j;
      for (uint32_t b = threadIdx.x; b < range; b += bd) {
        // the bucket's old kept ids come first (k_pool_sizes left their count in cursor)
        uint32_t base = (uint32_t)(pool_off[tb + b] - pbase) + cursor[tb + b];
        for (uint64_t s2 = s0; s2 < slot; ++s2) base += hbuf[s2 * range + b];
        csm[b] = base;
      }
    }
    __syncthreads();
    // Rows go in chunks of blockDim with a barrier between chunks, so a bucket's entries from
    // different chunks land in row (= id) order; only rows of one chunk that share a bucket
    // (rare: ~blockDim^2 / 2range pairs per chunk) may land out of order.  k_select_small
    // then finds most buckets already ascending.  The next chunks' addresses are loaded
    // ahead (4 chunks in flight).
    uint32_t* tpool = pool + pbase;
    uint32_t a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t r = r0 + threadIdx.x + (uint64_t)u * bd;
      a[u] = r < r1 ? col[r] : kEmpty;
    }
    for (uint64_t base = r0; base < r1; base += 4ull * bd) {
      uint32_t nx[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint64_t r = base + 4ull * bd + threadIdx.x + (uint64_t)u * bd;
        nx[u] = r < r1 ? col[r] : kEmpty;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (a[u] < range)
          tpool[atomicAdd(&csm[a[u]], 1u)] = id_base + (uint32_t)(base + threadIdx.x + (uint64_t)u * bd);
        __syncthreads();
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = nx[u];
    }
  }
}

// Per bucket: pool size m (old kept ids + new arrivals) and kept count; buckets with
// m > early_min go to early_list (their k_select_big can start as soon as the pool is filled).
__global__ void k_pool_sizes(uint32_t nb, uint32_t R, const uint64_t* __restrict__ goff_old,
                             uint32_t* __restrict__ cursor, uint32_t* __restrict__ arrivals,
                             uint64_t* __restrict__ pool_cnt, uint64_t* __restrict__ keep_cnt,
                             uint64_t early_min, uint32_t* __restrict__ early_list,
                             uint32_t* __restrict__ early_count) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= nb; i += gridDim.x * blockDim.x) {
    if (i == nb) { pool_cnt[nb] = 0; keep_cnt[nb] = 0; continue; }
    const uint64_t old = goff_old ? goff_old[i + 1] - goff_old[i] : 0;
    const uint32_t c = cursor[i];
    arrivals[i] += c;
    const uint64_t m = old + c;
    pool_cnt[i] = m;
    keep_cnt[i] = m < R ? m : R;
    cursor[i] = (uint32_t)old;
    if (m > early_min) early_list[atomicAdd(early_count, 1u)] = i;
  }
}

__global__ void k_fill_old(uint32_t nb, const uint64_t* __restrict__ goff_old,
                           const uint32_t* __restrict__ ids_old, const uint64_t* __restrict__ pool_off,
                           uint32_t* __restrict__ pool) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nw = gridDim.x * (blockDim.x >> 5);
  for (uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < nb; i += nw) {
    const uint64_t s = goff_old[i], m = goff_old[i + 1] - s, d = pool_off[i];
    for (uint64_t j = lane; j < m; j += 32) pool[d + j] = ids_old[s + j];
  }
}

__global__ void k_fill_new(const uint32_t* __restrict__ addrs, uint64_t n, uint32_t L, uint32_t acol0,
                           uint32_t range, uint32_t t0, uint32_t t1, uint32_t shared, uint32_t id_base,
                           uint32_t* __restrict__ cursor,
                           const uint64_t* __restrict__ pool_off, uint32_t* __restrict__ pool) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t r = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += nw) {
    for (uint32_t t = t0 + lane; t < t1; t += 32) {
      const uint32_t a = addrs[r * L + t - acol0];
      if (a >= (shared ? shared : range)) continue;  // EMPTY or invalid (counted by k_count)
      const uint32_t i = shared ? a : t * range + a;
      const uint32_t pos = atomicAdd(&cursor[i], 1u);
      pool[pool_off[i] + pos] = id_base + (uint32_t)r;
    }
  }
}

// Reservoir sharing pre-pass (R#23): warp per row, the row's L reservoir indices staged
// in shared memory so each entry can drop itself when an earlier table of the row points
// to the same reservoir.
__global__ void __launch_bounds__(256) k_shared_reservoirs(const uint32_t* __restrict__ addrs, uint64_t n,
                                                           uint32_t L, uint32_t range, uint32_t P, HashKeys keys,
                                                           uint32_t* __restrict__ out, unsigned long long* err) {
  extern __shared__ uint32_t rbuf_all[];
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t* rbuf = rbuf_all + (size_t)w * L;
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t r = (uint64_t)blockIdx.x * (blockDim.x >> 5) + w; r < n; r += nw) {
    for (uint32_t t = lane; t < L; t += 32) {
      const uint32_t a = addrs[r * L + t];
      uint32_t v = kEmpty;
      if (a < range) v = shared_reservoir(keys, t, a, P);
      else if (a != kEmpty) atomicAdd(err, 1ull);
      rbuf[t] = v;
    }
    __syncwarp();
    for (uint32_t t = lane; t < L; t += 32) {
      const uint32_t v = rbuf[t];
      bool dup = false;
      for (uint32_t j = 0; j < t && !dup; ++j) dup = rbuf[j] == v;
      out[r * L + t] = (v == kEmpty || dup) ? kEmpty : v;
    }
    __syncwarp();
  }
}

__device__ __forceinline__ void push_big(uint32_t i, uint32_t* big_list, uint32_t* big_count) {
  if ((threadIdx.x & 31) == 0) big_list[atomicAdd(big_count, 1u)] = i;
}

// B2, buckets with <= 32 members (the vast majority).  A warp takes 32 consecutive buckets
// at a time.  When all of them keep every member (m <= 32 and m <= R: their pool range and
// output range are contiguous and equal) it stages the range in shared memory with
// coalesced loads, each lane insertion-sorts its bucket there (the chunk-ordered scatter of
// k_fill_smem leaves buckets nearly ascending, so this is ~m steps), and the warp stores the
// range back coalesced.  In a mixed chunk each lane stages, sorts and writes its own
// all-kept bucket; a bucket with more than R (<= 32) members sorts its (prio, id) keys with
// the whole warp; larger buckets are listed for k_select_mid / k_select_warp / k_select_big
// (or the exact CTA path when FLASH_DEBUG_FORCE_BIG is set).
constexpr uint32_t kSmallChunk = 32;                 // buckets per warp step
constexpr uint32_t kSmallBuf = kSmallChunk * 32;     // ids staged per warp

// bottom-R of bucket i (R < m <= 32) by (prio, id) with the whole warp, written ascending
__device__ __forceinline__ void select_over_r(uint32_t i, uint32_t m, uint64_t p, uint64_t g, uint32_t range,
                                              uint32_t R, const HashKeys& keys, const uint32_t* __restrict__ pool,
                                              uint32_t* __restrict__ ids_out) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t id = lane < m ? pool[p + lane] : kEmpty;
  const uint32_t t = i / range, b = i - t * range;
  const uint64_t tb = prio_bucket_key(keys, t, b);
  uint64_t key = lane < m ? ((uint64_t)prio_of(tb, id) << 32) | id : ~0ull;
  key = warp_sort32(key);
  id = lane < R ? (uint32_t)key : kEmpty;
  id = warp_sort32_u32(id);  // ascending id; EMPTY (> any id) sorts last
  if (lane < R) ids_out[g + lane] = id;
}

__device__ __forceinline__ void insertion_sort(uint32_t* buf, uint32_t s0, uint32_t e0) {
  for (uint32_t a = s0 + 1; a < e0; ++a) {  // ascending id within the bucket (R#10)
    const uint32_t x = buf[a];
    uint32_t b = a;
    while (b > s0 && buf[b - 1] > x) {
      buf[b] = buf[b - 1];
      --b;
    }
    buf[b] = x;
  }
}

__global__ void __launch_bounds__(256)
k_select_small(uint32_t nb, uint32_t range, uint32_t R, HashKeys keys, int force_big, int early_listed,
               const uint64_t* __restrict__ pool_off, const uint32_t* __restrict__ pool,
               const uint64_t* __restrict__ goff, uint32_t* __restrict__ ids_out,
               uint32_t* __restrict__ mid_list, uint32_t* __restrict__ mid_count,
               uint32_t* __restrict__ reg_list, uint32_t* __restrict__ reg_count,
               uint32_t* __restrict__ big_list, uint32_t* __restrict__ big_count) {
  __shared__ uint32_t sbuf[256 / 32][kSmallBuf];
  const uint32_t lane = threadIdx.x & 31;
  uint32_t* buf = sbuf[threadIdx.x >> 5];
  const uint32_t nw = gridDim.x * (blockDim.x >> 5);
  const uint32_t nchunks = (nb + kSmallChunk - 1) / kSmallChunk;
  for (uint32_t c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c < nchunks; c += nw) {
    const uint32_t i0 = c * kSmallChunk, i = i0 + lane;
    const uint64_t pl = pool_off[i < nb ? i : nb];
    const uint64_t pe = pool_off[i < nb ? i + 1 : nb];
    const uint32_t m = (uint32_t)(pe - pl);
    if (__all_sync(kFull, m <= 32 && m <= R)) {
      const uint64_t p0 = __shfl_sync(kFull, pl, 0);
      const uint32_t T = (uint32_t)(__shfl_sync(kFull, pe, 31) - p0);  // <= kSmallBuf
      const uint64_t g0 = goff[i0];
#pragma unroll 4
      for (uint32_t j = lane; j < T; j += 32) buf[j] = pool[p0 + j];
      __syncwarp();
      insertion_sort(buf, (uint32_t)(pl - p0), (uint32_t)(pl - p0) + m);
      __syncwarp();
#pragma unroll 4
      for (uint32_t j = lane; j < T; j += 32) ids_out[g0 + j] = buf[j];
      __syncwarp();
    } else {
      const bool kept_all = i < nb && m <= 32 && m <= R;
      const uint32_t ps = kept_all ? m : 0u;
      uint32_t x = ps;
#pragma unroll
      for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
      }
      const uint32_t so = x - ps;  // this lane's staging offset
      for (uint32_t e = 0; e < ps; ++e) buf[so + e] = pool[pl + e];
      insertion_sort(buf, so, so + ps);
      if (ps) {
        const uint64_t go = goff[i];
        for (uint32_t e = 0; e < ps; ++e) ids_out[go + e] = buf[so + e];
      }
      if (i < nb && m > 32) {  // > kWarpMax members: the CTA path streams them with 1024 threads
        if (force_big || m > kWarpMax) {
          if (!early_listed) big_list[atomicAdd(big_count, 1u)] = i;  // else k_pool_sizes listed it
        }
        else if (m <= kMidMax && R <= kMidMax) reg_list[atomicAdd(reg_count, 1u)] = i;
        else mid_list[atomicAdd(mid_count, 1u)] = i;
      }
      uint32_t over = __ballot_sync(kFull, i < nb && m <= 32 && m > R);
      const uint64_t gi = (i < nb && m <= 32 && m > R) ? goff[i] : 0ull;
      while (over) {
        const uint32_t u = __ffs(over) - 1;
        over &= over - 1;
        select_over_r(i0 + u, __shfl_sync(kFull, m, u), __shfl_sync(kFull, pl, u), __shfl_sync(kFull, gi, u), range,
                      R, keys, pool, ids_out);
      }
      __syncwarp();
    }
  }
}

// Ascending bitonic sort of E*32 u32 keys held E per lane (element index r*32 + lane).
template <int E>
__device__ __forceinline__ void warp_sort_regs(uint32_t (&v)[E]) {
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll
  for (uint32_t k = 2; k <= 32u * E; k <<= 1) {
#pragma unroll
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const uint32_t rj = j >> 5;
#pragma unroll
        for (int r = 0; r < E; ++r) {
          if ((r & rj) == 0) {
            const bool up = ((r * 32 + lane) & k) == 0;
            const uint32_t x = v[r], y = v[r | rj];
            v[r] = up ? min(x, y) : max(x, y);
            v[r | rj] = up ? max(x, y) : min(x, y);
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const uint32_t w = __shfl_xor_sync(kFull, v[r], j);
          const bool up = ((r * 32 + lane) & k) == 0, lower = (lane & j) == 0;
          v[r] = (lower == up) ? min(v[r], w) : max(v[r], w);
        }
      }
    }
  }
}

// Sort the first n (<= E*32) ids of buf ascending and store them to out (one warp).
template <int E>
__device__ __forceinline__ void sort_store(const uint32_t* buf, uint32_t n, uint32_t* out) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t v[E];
#pragma unroll
  for (int r = 0; r < E; ++r) v[r] = r * 32 + lane < n ? buf[r * 32 + lane] : kEmpty;
  warp_sort_regs<E>(v);
#pragma unroll
  for (int r = 0; r < E; ++r)
    if (r * 32 + lane < n) out[r * 32 + lane] = v[r];
}

template <int E>
__device__ __forceinline__ void sort_store_upto(const uint32_t* buf, uint32_t n, uint32_t* out) {
  if (E > 1 && n <= 32u * (E / 2)) {
    sort_store_upto<(E > 1 ? E / 2 : 1)>(buf, n, out);
    return;
  }
  sort_store<E>(buf, n, out);
}

// B2, buckets with 33..256 members (and R <= 256): one warp per bucket, members in
// registers (8 per lane).  When m > R the bottom-R priority threshold is found by a radix
// select over the 32-bit priorities in 4-bit digits (a 16-bin shared-memory histogram per
// digit, stopping as soon as the R-th smallest is pinned down, ~log16(m) + 1 digits); the
// kept ids are then sorted ascending in registers.  Exact priority ties at the threshold (probability
// ~m^2/2^33) go to the exact CTA path.
// one bucket of m <= 32*E members (E = ceil(m / 32): only the register slots that hold
// members are hashed, counted and compacted)
// (false: priorities tie at the threshold, nothing written — the caller lists the bucket for
// the exact CTA path)
template <int E>
__device__ __forceinline__ bool select_mid_bucket(uint32_t i, uint32_t m, uint64_t p0, uint32_t range, uint32_t R,
                                                  const HashKeys& keys, const uint32_t* pool, uint32_t* out,
                                                  uint32_t* kbuf, uint32_t* hist, uint32_t lane) {
  uint32_t id[E];
#pragma unroll
  for (int u = 0; u < E; ++u) id[u] = lane + 32u * u < m ? pool[p0 + lane + 32u * u] : kEmpty;
  uint32_t keep = m;
  if (m > R) {
    const uint32_t t = i / range, b = i - t * range;
    const uint64_t tb = prio_bucket_key(keys, t, b);
    uint32_t pr[E];
#pragma unroll
    for (int u = 0; u < E; ++u) pr[u] = lane + 32u * u < m ? prio_of(tb, id[u]) : 0xFFFFFFFFu;
    // radix select over 4-bit digits, most significant first: a per-warp shared-memory
    // histogram of the candidates still matching `prefix`; the R-th smallest priority lies
    // in digit d of the current position, everything in the digits below d is kept
    uint32_t prefix = 0, need = R, ubound = 0;
    bool done = false;
    for (int sh = 28; sh >= 0 && !done; sh -= 4) {
      const uint32_t hi_mask = sh == 28 ? 0u : ~((16u << sh) - 1u);
      if (lane < 16) hist[lane] = 0;
      __syncwarp();
#pragma unroll
      for (int u = 0; u < E; ++u)
        if ((lane + 32u * u < m) && (pr[u] & hi_mask) == prefix) atomicAdd(&hist[(pr[u] >> sh) & 15u], 1u);
      __syncwarp();
      const uint32_t hc = lane < 16 ? hist[lane] : 0u;
      uint32_t x = hc;
#pragma unroll
      for (uint32_t o = 1; o < 16; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
      }
      const uint32_t d = __ffs(__ballot_sync(kFull, lane < 16 && x >= need)) - 1;
      const uint32_t below = __shfl_sync(kFull, x - hc, d), cd = __shfl_sync(kFull, hc, d);
      need -= below;  // still needed inside digit d (1 <= need <= cd)
      prefix |= d << sh;
      if (need == cd) {
        ubound = prefix + (1u << sh);  // keep every priority < ubound (0: 2^32)
        done = true;
      }
      __syncwarp();
    }
    if (!done) return false;  // priorities tie at the threshold: exact CTA path
    // compact the kept ids (priority < ubound; ubound == 0 means 2^32) into shared memory
    uint32_t base = 0;
#pragma unroll
    for (int u = 0; u < E; ++u) {
      const bool k_ = (lane + 32u * u < m) && (ubound == 0 || pr[u] < ubound);
      const uint32_t bal = __ballot_sync(kFull, k_);
      if (k_) kbuf[base + __popc(bal & lanemask_lt())] = id[u];
      base += __popc(bal);
    }
    keep = R;
  } else {
#pragma unroll
    for (int u = 0; u < E; ++u)
      if (lane + 32u * u < m) kbuf[lane + 32u * u] = id[u];
  }
  __syncwarp();
  sort_store_upto<8>(kbuf, keep, out);  // kept ids ascending (R#10)
  __syncwarp();
  return true;
}

// select_mid_bucket with E = ceil(m / 32) (warp-uniform), m <= kMidMax
__device__ __forceinline__ bool select_mid_any(uint32_t i, uint32_t m, uint64_t p0, uint32_t range, uint32_t R,
                                               const HashKeys& keys, const uint32_t* pool, uint32_t* out,
                                               uint32_t* kbuf, uint32_t* hist, uint32_t lane) {
  switch ((m + 31) >> 5) {
    case 0:
    case 1: return select_mid_bucket<1>(i, m, p0, range, R, keys, pool, out, kbuf, hist, lane);
    case 2: return select_mid_bucket<2>(i, m, p0, range, R, keys, pool, out, kbuf, hist, lane);
    case 3: return select_mid_bucket<3>(i, m, p0, range, R, keys, pool, out, kbuf, hist, lane);
    case 4: return select_mid_bucket<4>(i, m, p0, range, R, keys, pool, out, kbuf, hist, lane);
    case 5: return select_mid_bucket<5>(i, m, p0, range, R, keys, pool, out, kbuf, hist, lane);
    case 6: return select_mid_bucket<6>(i, m, p0, range, R, keys, pool, out, kbuf, hist, lane);
    default: return select_mid_bucket<8>(i, m, p0, range, R, keys, pool, out, kbuf, hist, lane);
  }
}

__global__ void __launch_bounds__(256)
k_select_mid(uint32_t range, uint32_t R, HashKeys keys, const uint32_t* __restrict__ mid_list,
             const uint32_t* __restrict__ mid_count, const uint64_t* __restrict__ pool_off,
             const uint32_t* __restrict__ pool, const uint64_t* __restrict__ goff,
             uint32_t* __restrict__ ids_out, uint32_t* __restrict__ big_list, uint32_t* __restrict__ big_count) {
  __shared__ uint32_t kept_s[8][kMidMax];
  __shared__ uint32_t hist_s[8][16];
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t* kbuf = kept_s[w];
  uint32_t* hist = hist_s[w];
  const uint32_t nw = gridDim.x * (blockDim.x >> 5);
  const uint32_t nmid = *mid_count;
  for (uint32_t it = blockIdx.x * (blockDim.x >> 5) + w; it < nmid; it += nw) {
    const uint32_t i = mid_list[it];
    const uint64_t p0 = pool_off[i];
    const uint32_t m = (uint32_t)(pool_off[i + 1] - p0);
    uint32_t* out = ids_out + goff[i];
    if (!select_mid_any(i, m, p0, range, R, keys, pool, out, kbuf, hist, lane)) push_big(i, big_list, big_count);
  }
}

// Grouped placement fused with the bottom-R select (fresh builds of big tables on the
// grouped path, R <= kMidMax; after the bucket counts are scanned).  One 1,024-thread CTA
// per group at a time: the group's buckets go in sub-ranges of kGSelSub; the members of a
// sub-range's buckets with <= kMidMax members are placed into shared memory (bucket-major,
// at the block scan of their counts) instead of the pool, and each warp then selects the
// bottom-R of its buckets there (select_mid_any) and writes the kept ids, ascending, to
// their final place — the pool write and the selects' re-read of it (19 GB each for kdd12)
// disappear.  Larger buckets, and every bucket of a sub-range whose members exceed the
// stage, are placed into the pool as k_gplace does and listed for the select kernels
// (reg_list: k_select_mid, mid_list: k_select_warp, > kWarpMax: k_pool_sizes' early list
// or big_list); a bucket whose priorities tie at the threshold is copied to the pool and
// listed for the exact CTA path.
constexpr uint32_t kGSelSub = 256;

__host__ __device__ inline size_t gsel_fixed_smem(uint32_t nch) {
  return (size_t)(nch + 1) * 8 + (size_t)(3 * kGSelSub + 1 + 32) * 4 + (size_t)(kGPlaceThreads / 32) * (kMidMax + 16) * 4;
}

__global__ void __launch_bounds__(kGPlaceThreads, 1)
k_gplace_sel(uint32_t W, uint32_t t0, uint32_t range, GroupGeom g, const uint64_t* __restrict__ goffs,
             const uint32_t* __restrict__ ent, uint32_t id_base, const uint64_t* __restrict__ pool_off,
             uint32_t* __restrict__ pool, uint32_t stage_cap, uint32_t R, HashKeys keys,
             const uint64_t* __restrict__ goff, uint32_t* __restrict__ ids_out, int early_listed,
             uint32_t* __restrict__ mid_list, uint32_t* __restrict__ mid_count,
             uint32_t* __restrict__ reg_list, uint32_t* __restrict__ reg_count,
             uint32_t* __restrict__ big_list, uint32_t* __restrict__ big_count) {
  extern __shared__ uint64_t co[];                                        // [nch + 1] chunk slot ranges
  uint32_t* msz = reinterpret_cast<uint32_t*>(co + g.nch + 1);            // [kGSelSub] members
  uint32_t* soff = msz + kGSelSub;                                        // [kGSelSub + 1] stage offsets
  uint32_t* cur = soff + kGSelSub + 1;                                    // [kGSelSub] placement cursors
  uint32_t* wsum = cur + kGSelSub;                                        // [32]
  uint32_t* kbuf_all = wsum + 32;                                         // [32][kMidMax]
  uint32_t* hist_all = kbuf_all + (kGPlaceThreads / 32) * kMidMax;        // [32][16]
  uint32_t* stage = hist_all + (kGPlaceThreads / 32) * 16;                // [stage_cap]
  const uint32_t gsz = 1u << g.gshift;
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint32_t* kbuf = kbuf_all + wib * kMidMax;
  uint32_t* hist = hist_all + wib * 16;
  const uint64_t ngroups = (uint64_t)W * g.ng;
  for (uint64_t gid = blockIdx.x; gid < ngroups; gid += gridDim.x) {
    const uint32_t j = (uint32_t)(gid / g.ng), gi = (uint32_t)(gid - (uint64_t)j * g.ng);
    const uint32_t b0 = gi << g.gshift;
    const uint32_t nbk = range - b0 < gsz ? range - b0 : gsz;
    const uint64_t tb = (uint64_t)(t0 + j) * range + b0;
    for (uint32_t c = threadIdx.x; c <= g.nch; c += blockDim.x) co[c] = goffs[gid * g.nch + c];
    __syncthreads();
    const uint64_t e0 = co[0], e1 = co[g.nch];
    for (uint32_t s0 = 0; s0 < nbk; s0 += kGSelSub) {
      const uint32_t ns = nbk - s0 < kGSelSub ? nbk - s0 : kGSelSub;
      // members per bucket, and the stage offsets of the staged ones (a block scan)
      uint32_t m = 0, sv = 0;
      if (threadIdx.x < kGSelSub) {
        if (threadIdx.x < ns) {
          const uint64_t i = tb + s0 + threadIdx.x;
          m = (uint32_t)(pool_off[i + 1] - pool_off[i]);
        }
        sv = m <= kMidMax ? m : 0u;
        uint32_t x = sv;
#pragma unroll
        for (uint32_t o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, x, o);
          if (lane >= o) x += y;
        }
        if (lane == 31) wsum[wib] = x;
        msz[threadIdx.x] = m;
        cur[threadIdx.x] = 0;
        sv = x - sv;  // exclusive within the warp
      }
      __syncthreads();
      if (threadIdx.x < kGSelSub) {
        uint32_t before = 0;
        for (uint32_t w = 0; w < wib; ++w) before += wsum[w];
        soff[threadIdx.x] = before + sv;
        if (threadIdx.x == kGSelSub - 1) soff[kGSelSub] = before + sv + (m <= kMidMax ? m : 0u);
      }
      __syncthreads();
      const bool overflow = soff[kGSelSub] > stage_cap;
      // place: each warp walks a contiguous range of 32-slot blocks of the group's entries
      // (as k_gplace), 4 blocks' loads in flight per lane; entries of other sub-ranges skip
      const uint64_t nblk = (e1 - e0 + 31) >> 5;
      const uint64_t wb0 = nblk * wib / (kGPlaceThreads / 32), wb1 = nblk * (wib + 1) / (kGPlaceThreads / 32);
      uint32_t c = 0;
      if (wb0 < wb1) {
        const uint64_t pb = e0 + (wb0 << 5);
        uint32_t hi = g.nch;
        while (hi - c > 1) {
          const uint32_t mid = (c + hi) >> 1;
          if (co[mid] <= pb) c = mid;
          else hi = mid;
        }
      }
      // (positions relative to e0 in 32 bits: a group holds < 2^32 entries; the next chunk
      // end is kept in a register, so a block costs one compare unless it crosses it)
      const uint32_t* gent = ent + e0;
      const uint32_t ge = (uint32_t)(e1 - e0);
      uint32_t cend = (uint32_t)(co[c + 1] - e0);
      for (uint32_t blk0 = (uint32_t)wb0; blk0 < (uint32_t)wb1; blk0 += 4) {
        uint32_t ev[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t p = ((blk0 + u) << 5) + lane;
          ev[u] = blk0 + u < (uint32_t)wb1 && p < ge ? gent[p] : 0xFFFFFFFFu;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (blk0 + u >= (uint32_t)wb1) break;
          const uint32_t pb = (blk0 + u) << 5;
          while (cend <= pb) cend = (uint32_t)(co[++c + 1] - e0);
          const uint32_t p = pb + lane;
          const uint32_t bl = (ev[u] >> kGChunkLog2) - s0;  // bucket within the sub-range
          if (p < ge && bl < ns) {
            uint32_t cl = c;
            if (p >= cend) {  // (a block that straddles chunk ends)
              ++cl;
              while ((uint32_t)(co[cl + 1] - e0) <= p) ++cl;
            }
            const uint32_t id = id_base + (cl << kGChunkLog2) + (ev[u] & ((1u << kGChunkLog2) - 1));
            const uint32_t slot = atomicAdd(&cur[bl], 1u);
            if (!overflow && msz[bl] <= kMidMax) stage[soff[bl] + slot] = id;
            else pool[pool_off[tb + s0 + bl] + slot] = id;
          }
        }
      }
      __syncthreads();
      // select: warp per bucket
      for (uint32_t b = wib; b < ns; b += kGPlaceThreads / 32) {
        const uint64_t i = tb + s0 + b;
        const uint32_t mb = msz[b];
        if (mb == 0) continue;
        if (overflow || mb > kMidMax) {  // in the pool: listed for the select kernels
          if (lane == 0) {
            if (mb > kWarpMax) {
              if (!early_listed) big_list[atomicAdd(big_count, 1u)] = (uint32_t)i;  // else k_pool_sizes listed it
            } else if (mb <= kMidMax) {
              reg_list[atomicAdd(reg_count, 1u)] = (uint32_t)i;
            } else {
              mid_list[atomicAdd(mid_count, 1u)] = (uint32_t)i;
            }
          }
          continue;
        }
        const uint32_t* src = stage + soff[b];
        if (!select_mid_any((uint32_t)i, mb, 0, range, R, keys, src, ids_out + goff[i], kbuf, hist, lane)) {
          const uint64_t po = pool_off[i];  // a priority tie: the exact CTA path reads the pool
          for (uint32_t x = lane; x < mb; x += 32) pool[po + x] = src[x];
          __syncwarp();
          push_big((uint32_t)i, big_list, big_count);
        }
      }
      __syncthreads();
    }
  }
}

// B2, buckets with > 32 members: one warp per listed bucket.
__global__ void __launch_bounds__(kSelThreads)
k_select_warp(uint32_t range, uint32_t R, HashKeys keys, const uint32_t* __restrict__ mid_list,
              const uint32_t* __restrict__ mid_count, const uint64_t* __restrict__ pool_off,
              const uint32_t* __restrict__ pool, const uint64_t* __restrict__ goff,
              uint32_t* __restrict__ ids_out, uint32_t* __restrict__ big_list, uint32_t* __restrict__ big_count) {
  extern __shared__ uint64_t sel_smem[];
  const uint32_t lane = threadIdx.x & 31;
  uint64_t* buf = sel_smem + (size_t)(threadIdx.x >> 5) * kWarpCap;
  const uint32_t nw = gridDim.x * (blockDim.x >> 5);
  const uint32_t nmid = *mid_count;
  for (uint32_t it = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); it < nmid; it += nw) {
    const uint32_t i = mid_list[it];
    const uint64_t p0 = pool_off[i];
    const uint32_t m = (uint32_t)(pool_off[i + 1] - p0);
    if (m == 0) continue;
    const uint32_t keep = m < R ? m : R;
    uint32_t* out = ids_out + goff[i];
    const uint32_t t = i / range, b = i - t * range;

    if (m <= R) {  // keep every member; sort ids
      if (m > kWarpCap) { push_big(i, big_list, big_count); continue; }
      const uint32_t n2 = pow2_ceil(m);
      for (uint32_t j = lane; j < n2; j += 32) buf[j] = j < m ? (uint64_t)pool[p0 + j] : ~0ull;
      __syncwarp();
      warp_bitonic(buf, n2);
      for (uint32_t j = lane; j < m; j += 32) out[j] = (uint32_t)buf[j];
      __syncwarp();
      continue;
    }

    // m > R: keep every member whose priority is below a threshold that leaves
    // ~R + 6 sqrt(R) + 16 survivors in expectation; the bottom-R of the survivors is
    // the bottom-R of the bucket whenever at least R survive (else: exact CTA path).
    const double expect = (double)R + 6.0 * sqrt((double)R) + 16.0;
    const uint64_t tau = expect >= (double)m ? (1ull << 32)
                                             : (uint64_t)ceil(expect / (double)m * 4294967296.0);
    const uint64_t tb = prio_bucket_key(keys, t, b);
    uint32_t cnt = 0;
    for (uint32_t j0 = 0; j0 < m; j0 += 32) {
      const uint32_t j = j0 + lane;
      bool pass = false;
      uint64_t key = 0;
      if (j < m) {
        const uint32_t id = pool[p0 + j];
        const uint32_t pr = prio_of(tb, id);
        pass = (uint64_t)pr < tau;
        key = ((uint64_t)pr << 32) | id;
      }
      const uint32_t ballot = __ballot_sync(kFull, pass);
      const uint32_t pos = cnt + __popc(ballot & lanemask_lt());
      if (pass && pos < kWarpCap) buf[pos] = key;
      cnt += __popc(ballot);
    }
    if (cnt < keep || cnt > kWarpCap) {
      __syncwarp();
      push_big(i, big_list, big_count);
      continue;
    }
    const uint32_t n2 = pow2_ceil(cnt);
    for (uint32_t j = cnt + lane; j < n2; j += 32) buf[j] = ~0ull;
    __syncwarp();
    warp_bitonic(buf, n2);  // by (prio, id)
    const uint32_t n3 = pow2_ceil(keep);
    for (uint32_t j = lane; j < n3; j += 32) buf[j] = j < keep ? (buf[j] & 0xFFFFFFFFull) : ~0ull;
    __syncwarp();
    warp_bitonic(buf, n3);  // kept ids ascending
    for (uint32_t j = lane; j < keep; j += 32) out[j] = (uint32_t)buf[j];
    __syncwarp();
  }
}

// B2, large buckets (and anything the warp path could not finish): one CTA per bucket.
// First a priority-threshold filter with the whole CTA (4 loads in flight per thread)
// keeps ~R + 6 sqrt(R) + 16 candidates in shared memory; if at least `keep` and at most
// kBigCap survive, a CTA bitonic sort by (prio, id) picks the bottom-R.  Otherwise an
// exact radix select of the keep-th smallest (prio, id), 8 bits at a time, decides.
__global__ void __launch_bounds__(kBigThreads)
k_select_big(uint32_t range, uint32_t R, HashKeys keys, int exact_only, const uint64_t* __restrict__ pool_off,
             const uint32_t* __restrict__ pool, const uint64_t* __restrict__ goff,
             uint32_t* __restrict__ ids_out, const uint32_t* __restrict__ big_list,
             const uint32_t* __restrict__ big_count) {
  __shared__ uint32_t hist[256];
  __shared__ uint64_t kbuf[kBigCap];
  __shared__ uint32_t s_prefix, s_need, s_ties, s_n;
  const uint32_t nbig = *big_count;
  for (uint32_t it = blockIdx.x; it < nbig; it += gridDim.x) {
    const uint32_t i = big_list[it];
    const uint64_t p0 = pool_off[i];
    const uint32_t m = (uint32_t)(pool_off[i + 1] - p0);
    const uint32_t keep = m < R ? m : R;
    uint32_t* out = ids_out + goff[i];
    const uint32_t t = i / range, b = i - t * range;
    const uint64_t tb = prio_bucket_key(keys, t, b);

    if (m <= R) {  // every member is kept (m <= R <= kBigCap): sort the ids
      const uint32_t n2 = pow2_ceil(m);
      for (uint32_t j = threadIdx.x; j < n2; j += blockDim.x) kbuf[j] = j < m ? (uint64_t)pool[p0 + j] : ~0ull;
      __syncthreads();
      block_bitonic(kbuf, n2);
      for (uint32_t j = threadIdx.x; j < m; j += blockDim.x) out[j] = (uint32_t)kbuf[j];
      __syncthreads();
      continue;
    }

    // ---- threshold filter ----
    const double expect = (double)R + 6.0 * sqrt((double)R) + 16.0;
    const uint64_t tau = expect >= (double)m ? (1ull << 32) : (uint64_t)ceil(expect / (double)m * 4294967296.0);
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    for (uint32_t j0 = threadIdx.x; j0 < m; j0 += 4 * blockDim.x) {
      uint32_t idv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t j = j0 + u * blockDim.x;
        idv[u] = j < m ? pool[p0 + j] : kEmpty;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (j0 + u * blockDim.x < m) {
          const uint32_t pr = prio_of(tb, idv[u]);
          if ((uint64_t)pr < tau) {
            const uint32_t pos = atomicAdd(&s_n, 1u);
            if (pos < kBigCap) kbuf[pos] = ((uint64_t)pr << 32) | idv[u];
          }
        }
      }
    }
    __syncthreads();
    const uint32_t cnt = s_n;
    if (cnt >= keep && cnt <= kBigCap && !exact_only) {
      const uint32_t n2 = pow2_ceil(cnt);
      for (uint32_t j = cnt + threadIdx.x; j < n2; j += blockDim.x) kbuf[j] = ~0ull;
      __syncthreads();
      block_bitonic(kbuf, n2);  // by (prio, id)
      const uint32_t n3 = pow2_ceil(keep);
      for (uint32_t j = threadIdx.x; j < n3; j += blockDim.x) kbuf[j] = j < keep ? (kbuf[j] & 0xFFFFFFFFull) : ~0ull;
      __syncthreads();
      block_bitonic(kbuf, n3);  // kept ids ascending
      for (uint32_t j = threadIdx.x; j < keep; j += blockDim.x) out[j] = (uint32_t)kbuf[j];
      __syncthreads();
      continue;
    }

    // ---- exact fallback: radix select on the priority, then on the id among ties ----
    uint32_t pstar, theta = 0xFFFFFFFFu;
    {
      uint32_t prefix = 0, pmask = 0, need = keep, ties = 0;
      for (int shift = 24; shift >= 0; shift -= 8) {
        for (uint32_t d = threadIdx.x; d < 256; d += blockDim.x) hist[d] = 0;
        __syncthreads();
        for (uint32_t j = threadIdx.x; j < m; j += blockDim.x) {
          const uint32_t pr = prio_of(tb, pool[p0 + j]);
          if ((pr & pmask) == prefix) atomicAdd(&hist[(pr >> shift) & 255u], 1u);
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
          s_ties = hist[d];
        }
        __syncthreads();
        need = s_need;
        prefix = s_prefix;
        ties = s_ties;
        pmask |= 255u << shift;
        __syncthreads();
      }
      pstar = prefix;
      if (need < ties) {
        uint32_t iprefix = 0, imask = 0;
        for (int shift = 24; shift >= 0; shift -= 8) {
          for (uint32_t d = threadIdx.x; d < 256; d += blockDim.x) hist[d] = 0;
          __syncthreads();
          for (uint32_t j = threadIdx.x; j < m; j += blockDim.x) {
            const uint32_t id = pool[p0 + j];
            if (prio_of(tb, id) == pstar && (id & imask) == iprefix) atomicAdd(&hist[(id >> shift) & 255u], 1u);
          }
          __syncthreads();
          if (threadIdx.x == 0) {
            uint32_t cum = 0, d = 0;
            for (; d < 255; ++d) {
              if (cum + hist[d] >= need) break;
              cum += hist[d];
            }
            s_need = need - cum;
            s_prefix = iprefix | (d << shift);
          }
          __syncthreads();
          need = s_need;
          iprefix = s_prefix;
          imask |= 255u << shift;
          __syncthreads();
        }
        theta = iprefix;
      }
    }
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < m; j += blockDim.x) {
      const uint32_t id = pool[p0 + j];
      const uint32_t pr = prio_of(tb, id);
      if (pr < pstar || (pr == pstar && id <= theta)) kbuf[atomicAdd(&s_n, 1u)] = id;
    }
    __syncthreads();
    const uint32_t n2 = pow2_ceil(keep);
    for (uint32_t j = keep + threadIdx.x; j < n2; j += blockDim.x) kbuf[j] = ~0ull;
    __syncthreads();
    block_bitonic(kbuf, n2);
    for (uint32_t j = threadIdx.x; j < keep; j += blockDim.x) out[j] = (uint32_t)kbuf[j];
    __syncthreads();
  }
}

}  // namespace

uint32_t smem_build_ctas(uint32_t W, uint64_t n) {
  // CTAs over the W*n (table, row) units: one per SM (or one per table if W is larger)
  // when every table's pool region (4 B per row) fits L2 together; otherwise S equal row
  // slices per table, S large enough that the CTAs resident at once cover only the few
  // tables whose regions fit ~96 MB of L2, so the scattered pool writes stay in L2 (the
  // units are table-major)
  const uint32_t sms = device_sms();
  const uint64_t region = 4 * (n ? n : 1);
  uint64_t tc = (96ull << 20) / region;  // tables whose regions fit L2 at once
  if (tc < 1) tc = 1;
  uint64_t c;
  if (tc >= W) {
    c = W > sms ? W : sms;
  } else {
    uint64_t s = (sms + tc - 1) / tc;
    c = (uint64_t)W * (s < 1 ? 1 : (s > 64 ? 64 : s));
  }
  // every CTA must own at least one unit (an empty one would leave its hbuf slot unwritten)
  const uint64_t units = (uint64_t)W * (n ? n : 1);
  return (uint32_t)(c < units ? c : units);
}

bool smem_build_fits(uint32_t range) { return range <= kSmemBuildMaxRange; }

uint64_t build_group_slots(uint32_t range, uint64_t n, uint32_t W) {
  const GroupGeom g = group_geom(range, n);
  return (uint64_t)W * g.ng * g.nch + 1;
}

size_t build_scan_tmp_bytes(uint64_t nb) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                (int64_t)(nb + 1));
  return bytes;
}

int launch_shared_reservoirs(const uint32_t* addrs, uint64_t n, uint32_t L, uint32_t range, uint32_t P,
                             const HashKeys& keys, uint32_t* out, unsigned long long* err, cudaStream_t s) {
  if (n == 0) return 0;
  const size_t smem = (size_t)8 * L * sizeof(uint32_t);
  ensure_smem_attr((const void*)k_shared_reservoirs, smem);
  const uint64_t want = (n + 7) / 8;
  const unsigned blocks = (unsigned)(want < (uint64_t)device_sms() * 16 ? want : (uint64_t)device_sms() * 16);
  k_shared_reservoirs<<<blocks, 256, smem, s>>>(addrs, n, L, range, P, keys, out, err);
  return 1;
}

int launch_build(const BuildArgs& a, cudaStream_t s) {
  const uint32_t nb = a.shared ? a.shared : a.L * a.range;
  int launches = 0;
  const unsigned rows_blocks = (unsigned)((a.n + 7) / 8 < (uint64_t)device_sms() * 32 ? (a.n + 7) / 8 : (uint64_t)device_sms() * 32);
  const unsigned nb_blocks = (unsigned)(((uint64_t)nb + 256) / 256 < (uint64_t)device_sms() * 32 ? ((uint64_t)nb + 256) / 256 : (uint64_t)device_sms() * 32);
  cudaMemsetAsync(a.cursor, 0, sizeof(uint32_t) * (size_t)nb, s);
  cudaMemsetAsync(a.big_count, 0, 4 * sizeof(uint32_t), s);  // big, mid, register-path, early list counters
  const uint32_t W = a.t1 > a.t0 ? a.t1 - a.t0 : 0;
  const bool sm_build = a.hbuf != nullptr && a.addrsT != nullptr && a.n && W && !a.shared;  // k_count_smem
  const bool tm = !sm_build && a.addrsT != nullptr && a.n && W && !a.shared;  // table-major passes (k_count_tm)
  // grouped table-major passes: fresh builds whose group slot table fits the pool_cnt /
  // keep_cnt scratch (W*ng*nch + 1 <= nb + 1), FLASH_BUILD_GROUPED=0 disables (tests)
  const GroupGeom gg = group_geom(a.range, a.n);
  const char* gp_env = getenv("FLASH_BUILD_GROUPED");
  const bool grouped = tm && !a.goff_old && a.gslots && a.range <= (1u << 24) &&
                       (uint64_t)W * gg.ng * gg.nch <= (uint64_t)nb &&  // (the scan's temp storage is sized for nb)
                       !(gp_env && gp_env[0] == '0');
  // FLASH_DEBUG_FORCE_BIG=1: every bucket with > 32 members takes the CTA path;
  // =2: and the CTA path skips its filter (exact radix select).  Tests only.
  const char* fb = getenv("FLASH_DEBUG_FORCE_BIG");
  const int force_big = fb ? (fb[0] == '2' ? 2 : 1) : 0;
  // grouped placement fused with the select (k_gplace_sel; FLASH_BUILD_GSEL=0 disables, tests)
  const char* gs_env = getenv("FLASH_BUILD_GSEL");
  // it pays where most buckets select (kdd12: ~143 arrivals per bucket, R = 64); where most
  // keep every member (friendster: ~63 per bucket, R = 64) k_select_small's staged copies win
  // (friendster build 97 vs 139 ms fused); FLASH_BUILD_GSEL=1 forces it (tests)
  const bool gsel = grouped && a.R <= kMidMax && !force_big &&
                    (gs_env ? gs_env[0] == '1' : a.n > (uint64_t)a.R * a.range);
  uint32_t* pool = a.pool;  // the grouped passes leave the bucket-ordered pool in addrsT
  unsigned gplace_grid = 1;
  const uint64_t chunks = (a.n + kTmRows - 1) / kTmRows;
  const uint32_t C = smem_build_ctas(W, a.n);
  if (sm_build) {
    ensure_smem_attr((const void*)k_count_smem, (size_t)kSmemBuildMaxRange * 4);
    ensure_smem_attr((const void*)k_fill_smem, (size_t)kSmemBuildMaxRange * 4);
    k_transpose_cols<<<(unsigned)((a.n + 255) / 256), 256, 0, s>>>(a.addrs, a.n, a.astride, a.t0 - a.acol0, W,
                                                                   a.addrsT);
    k_count_smem<<<C, kSmemBuildThreads, (size_t)a.range * 4, s>>>(a.addrsT, a.n, a.t0, a.range, W, C, a.cursor,
                                                                      a.hbuf, a.err);
    launches += 2;
  } else if (grouped) {
    k_transpose_cols<<<(unsigned)((a.n + 255) / 256), 256, 0, s>>>(a.addrs, a.n, a.astride, a.t0 - a.acol0, W,
                                                                   a.addrsT);
    uint64_t* ghist = a.gslots;  // group histograms, scanned in place into slot offsets
    uint64_t* goffs = a.gslots;
    const uint64_t nslots = (uint64_t)W * gg.ng * gg.nch;
    ensure_smem_attr((const void*)k_gscatter, gscatter_smem(gg.ng));
    k_gcount<<<W * gg.nch, kGThreads, (size_t)gg.ng * 4, s>>>(a.addrsT, a.n, a.range, gg, ghist, a.err);
    cudaMemsetAsync(ghist + nslots, 0, sizeof(uint64_t), s);
    size_t tmp = a.scan_tmp_bytes;
    cub::DeviceScan::ExclusiveSum(a.scan_tmp, tmp, ghist, goffs, (int64_t)nslots + 1, s);
    k_gscatter<<<W * gg.nch, kGSThreads, gscatter_smem(gg.ng), s>>>(a.addrsT, a.n, a.range, gg, goffs, a.pool);
    const size_t psm = gplace_smem(gg.gshift, gg.nch);
    const uint64_t ngroups = (uint64_t)W * gg.ng;
    gplace_grid = (unsigned)((uint64_t)device_sms() < ngroups ? device_sms() : ngroups);  // one group per SM
    if (a.after_scan || gsel) {  // count now, place after the scans (the callback's work overlaps it)
      ensure_smem_attr((const void*)k_gplace<0>, psm);
      ensure_smem_attr((const void*)k_gplace<1>, psm);
      k_gplace<0><<<gplace_grid, kGPlaceThreads, psm, s>>>(W, a.t0, a.range, gg, goffs, a.pool, a.id_base, a.cursor,
                                                           nullptr, nullptr);
    } else {  // count and place in one pass
      ensure_smem_attr((const void*)k_gplace<2>, psm);
      k_gplace<2><<<gplace_grid, kGPlaceThreads, psm, s>>>(W, a.t0, a.range, gg, goffs, a.pool, a.id_base, a.cursor,
                                                           nullptr, a.addrsT);
    }
    pool = a.addrsT;
    launches += 3;
  } else if (tm) {
    k_transpose_cols<<<(unsigned)((a.n + 255) / 256), 256, 0, s>>>(a.addrs, a.n, a.astride, a.t0 - a.acol0, W,
                                                                   a.addrsT);
    k_count_tm<<<(unsigned)(chunks * W), 256, 0, s>>>(a.addrsT, a.n, a.t0, a.range, (uint32_t)chunks, a.cursor,
                                                       a.err);
    launches += 2;
  } else if (a.n) {
    k_count<<<rows_blocks, 256, 0, s>>>(a.addrs, a.n, a.astride, a.acol0, a.range, a.t0, a.t1, a.shared, a.cursor,
                                        a.err);
    launches++;
  }
  // buckets with > kWarpMax members are listed here and selected on the side stream
  const bool early = a.early_list && a.side_stream && !force_big;
  uint32_t* early_count = a.big_count + 3;
  k_pool_sizes<<<nb_blocks, 256, 0, s>>>(nb, a.R, a.goff_old, a.cursor, a.arrivals, a.pool_cnt, a.keep_cnt,
                                         early ? (uint64_t)kWarpMax : ~0ull, a.early_list, early_count);
  launches++;
  size_t tmp = a.scan_tmp_bytes;
  cub::DeviceScan::ExclusiveSum(a.scan_tmp, tmp, a.pool_cnt, a.pool_off, (int64_t)nb + 1, s);
  tmp = a.scan_tmp_bytes;
  cub::DeviceScan::ExclusiveSum(a.scan_tmp, tmp, a.keep_cnt, a.goff_new, (int64_t)nb + 1, s);
  // (the two CUB scans launch library kernels; they are not counted as ours)
  cudaStream_t side = static_cast<cudaStream_t>(a.side_stream);
  bool side_used = false;
  if (a.after_scan && side) {  // e.g. the graph's query planning, beside the scatter/selects
    cudaEventRecord(static_cast<cudaEvent_t>(a.side_fork), s);
    cudaStreamWaitEvent(side, static_cast<cudaEvent_t>(a.side_fork), 0);
    a.after_scan(a.after_scan_ctx, side);
    side_used = true;
  }
  if (a.goff_old) {
    const unsigned wb = (unsigned)(((uint64_t)nb + 7) / 8 < (uint64_t)device_sms() * 32 ? ((uint64_t)nb + 7) / 8 : (uint64_t)device_sms() * 32);
    k_fill_old<<<wb, 256, 0, s>>>(nb, a.goff_old, a.ids_old, a.pool_off, a.pool);
    launches++;
  }
  if (sm_build) {
    const bool prefixed = C > 4 * W;  // many segments per table: scan them once up front
    if (prefixed) {
      const uint64_t sb = ((uint64_t)W * a.range + 255) / 256;
      k_slice_bases<<<(unsigned)(sb < (uint64_t)device_sms() * 16 ? sb : (uint64_t)device_sms() * 16), 256, 0,
                      s>>>(W, a.t0, a.range, a.n, C, a.cursor, a.pool_off, a.hbuf);
      launches++;
    }
    k_fill_smem<<<C, kSmemBuildThreads, (size_t)a.range * 4, s>>>(a.addrsT, a.n, a.t0, a.range, W, C, a.id_base,
                                                                 a.cursor, a.hbuf, a.pool_off, a.pool, prefixed);
    launches++;
  } else if (gsel) {  // placement + bottom-R select of the small buckets, in one pass
    const size_t fixed = gsel_fixed_smem(gg.nch);
    const size_t gsm = 227 * 1024;
    uint32_t stage_cap = (uint32_t)((gsm - fixed) / 4);
    const char* cap_env = getenv("FLASH_BUILD_GSEL_CAP");  // tests: a smaller stage (sub-range overflow)
    if (cap_env) stage_cap = std::min<uint32_t>(stage_cap, (uint32_t)strtoul(cap_env, nullptr, 10));
    ensure_smem_attr((const void*)k_gplace_sel, gsm);
    k_gplace_sel<<<gplace_grid, kGPlaceThreads, gsm, s>>>(W, a.t0, a.range, gg, a.gslots, a.pool, a.id_base, a.pool_off,
                                                          a.addrsT, stage_cap, a.R, a.keys, a.goff_new, a.ids_new,
                                                          early, a.cursor, a.big_count + 1,
                                                          reinterpret_cast<uint32_t*>(a.pool_cnt), a.big_count + 2,
                                                          a.big_list, a.big_count);
    launches++;
  } else if (grouped) {
    if (a.after_scan) {  // (after the scans: the callback's work above overlaps the placement)
      const size_t psm = gplace_smem(gg.gshift, gg.nch);
      k_gplace<1><<<gplace_grid, kGPlaceThreads, psm, s>>>(W, a.t0, a.range, gg, a.gslots, a.pool, a.id_base, nullptr,
                                                           a.pool_off, a.addrsT);
      launches++;
    }
  } else if (tm) {
    k_fill_tm<<<(unsigned)(chunks * W), 256, 0, s>>>(a.addrsT, a.n, a.t0, a.range, (uint32_t)chunks, a.id_base,
                                                      a.cursor, a.pool_off, a.pool);
    launches++;
  } else if (a.n) {
    k_fill_new<<<rows_blocks, 256, 0, s>>>(a.addrs, a.n, a.astride, a.acol0, a.range, a.t0, a.t1, a.shared,
                                           a.id_base, a.cursor, a.pool_off, a.pool);
    launches++;
  }
  const size_t sel_smem = (size_t)(kSelThreads / 32) * kWarpCap * sizeof(uint64_t);
  ensure_smem_attr((const void*)k_select_warp, sel_smem);
  if (early) {  // the early-listed big buckets, concurrently with the kernels below
    cudaEventRecord(static_cast<cudaEvent_t>(a.side_fork), s);
    cudaStreamWaitEvent(side, static_cast<cudaEvent_t>(a.side_fork), 0);
    k_select_big<<<device_sms(), kBigThreads, 0, side>>>(a.range, a.R, a.keys, 0, a.pool_off, pool, a.goff_new,
                                                        a.ids_new, a.early_list, early_count);
    side_used = true;
    launches += 1;
  }
  uint32_t* mid_list = a.cursor;  // free once k_fill_new is done
  uint32_t* mid_count = a.big_count + 1;
  uint32_t* reg_list = reinterpret_cast<uint32_t*>(a.pool_cnt);  // free once pool_off is scanned
  uint32_t* reg_count = a.big_count + 2;
  const uint64_t small_warps = ((uint64_t)nb + kSmallChunk - 1) / kSmallChunk;  // 32 buckets per warp step
  const unsigned small_blocks = (unsigned)((small_warps + 7) / 8 < (uint64_t)device_sms() * 64 ? (small_warps + 7) / 8 : (uint64_t)device_sms() * 64);
  if (!gsel)  // (k_gplace_sel selected the small buckets and listed the rest)
    k_select_small<<<small_blocks, 256, 0, s>>>(nb, a.range, a.R, a.keys, force_big, early, a.pool_off, pool,
                                               a.goff_new, a.ids_new, mid_list, mid_count, reg_list, reg_count,
                                               a.big_list, a.big_count);
  k_select_mid<<<device_sms() * 8, 256, 0, s>>>(a.range, a.R, a.keys, reg_list, reg_count, a.pool_off, pool, a.goff_new,
                                       a.ids_new, a.big_list, a.big_count);
  launches += 1;
  k_select_warp<<<device_sms() * 3, kSelThreads, sel_smem, s>>>(a.range, a.R, a.keys, mid_list, mid_count, a.pool_off,
                                                      pool, a.goff_new, a.ids_new, a.big_list, a.big_count);
  launches += 2;
  k_select_big<<<device_sms(), kBigThreads, 0, s>>>(a.range, a.R, a.keys, force_big == 2, a.pool_off, pool, a.goff_new,
                                              a.ids_new, a.big_list, a.big_count);  // the late list
  launches += 1;
  if (side_used) {  // join everything queued on the side stream
    cudaEventRecord(static_cast<cudaEvent_t>(a.side_join), side);
    cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(a.side_join), 0);
  }
  return launches;
}

}  // namespace flash
