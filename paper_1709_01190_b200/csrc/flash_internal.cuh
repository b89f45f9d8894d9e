// flash_internal.cuh — device primitives and kernel launchers of libflash.so (sm_100a).
//
// The integer definitions implemented here are DESIGN.md §2 (HASHSPEC); they are
// written independently of the CPU oracle (oracle/), which shares no code with this
// directory.  Citations: P:n = PAPER.md line n; R#n = DESIGN.md readings ledger.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "flash.h"

namespace flash {

constexpr uint32_t kEmpty = 0xFFFFFFFFu;  // R#3
constexpr uint32_t kProbes = 64;          // densification chain cap T (R#4)

// Per-index hash keys derived from the single seed (R#2).
struct HashKeys {
  uint32_t a1, m1, a2, s_dens;  // DOPH's "4 random numbers"
  uint32_t s_addr;              // K-tuple -> address key (R#5)
  uint32_t s_pool;              // shared-reservoir binding key (R#23)
  uint64_t s_prio;              // bottom-R priority key (R#9)
  uint32_t tbase;               // global index of local table 0 (a multi-GPU table window; else 0):
                                // priorities are keyed by the GLOBAL table index
};

__host__ __device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  h ^= h >> 16;
  return h;
}

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

inline HashKeys derive_keys(uint64_t seed) {
  uint64_t w[4];
  for (int k = 0; k < 4; ++k) w[k] = mix64(seed + (uint64_t)(k + 1) * 0x9E3779B97F4A7C15ull);
  HashKeys s;
  s.a1 = (uint32_t)w[0];
  s.m1 = (uint32_t)(w[0] >> 32) | 1u;
  s.a2 = (uint32_t)w[1];
  s.s_dens = (uint32_t)(w[1] >> 32);
  s.s_addr = (uint32_t)w[2];
  s.s_pool = (uint32_t)(w[2] >> 32);
  s.s_prio = w[3];
  s.tbase = 0;
  return s;
}

// pi(c): keyed bijection on uint32 standing in for the random permutation of Eq. 1.
__device__ __forceinline__ uint32_t perm(const HashKeys& k, uint32_t c) {
  return fmix32(((c ^ k.a1) * k.m1) + k.a2);
}

// Reservoir sharing (R#23): table t's bucket b points to shared reservoir
// mulhi(fmix32(fmix32(s_pool ^ t) ^ b), P) of a pool of P reservoirs.
__device__ __forceinline__ uint32_t shared_reservoir(const HashKeys& k, uint32_t t, uint32_t b, uint32_t P) {
  return __umulhi(fmix32(fmix32(k.s_pool ^ t) ^ b), P);
}

// prio(t, b, id) = hi32(mix64(tb ^ id)) with tb = mix64(s_prio ^ (t<<32 | b)), t the global
// table index (local table index + tbase).
__device__ __forceinline__ uint64_t prio_bucket_key(const HashKeys& k, uint32_t t, uint32_t b) {
  return mix64(k.s_prio ^ (((uint64_t)(t + k.tbase) << 32) | (uint64_t)b));
}
__device__ __forceinline__ uint32_t prio_of(uint64_t tb, uint32_t id) {
  return (uint32_t)(mix64(tb ^ (uint64_t)id) >> 32);
}

// Set a kernel's dynamic shared-memory limit (and optionally the max carveout) once per
// (kernel, device) for at least `bytes` (util.cu).
bool ensure_smem_attr(const void* func, size_t bytes, bool carveout_max = false);
// SM count of the current device (cached per device; 148 on B200)
uint32_t device_sms();

// ---------------------------------------------------------------------------
// Launchers (each returns the number of kernels it launched).
// ---------------------------------------------------------------------------

// Where the hash writes the L addresses of each row.
struct AddrOut {
  uint32_t* addrs;         // world == 1: [n_rows][L]; world > 1 (peers null): owner-blocked for a
                           // floor-block partition of the L tables over `world` ranks (table window
                           // of rank g: [floor(gL/world), floor((g+1)L/world))), rank g's block
                           // [n_rows][L_g] starting at element n_rows * t0(g)
  uint32_t* const* peers;  // or (dist mode, device array [world]): rank g's window-address buffer
                           // [N][L_g]; this call's row r is global row row0 + r
  uint64_t row0;
  uint32_t world;
};
inline AddrOut addr_out(uint32_t* addrs, uint32_t world = 1) { return AddrOut{addrs, nullptr, 0, world}; }

// H1-H3: DOPH bin minima, densification, addresses.  codes may be null; addresses are
// written when out.addrs or out.peers is set.
// long_rows (optional, [long_cap + 2] u32 scratch): when the sparse kernel runs, it lists the
// rows it leaves to k_doph there (the longest from the front, the rest from the back; the
// last two words count them), so k_doph need not scan every row's extent and starts with
// the longest rows; counts above long_cap make k_doph scan as without the list.
int launch_doph(const int64_t* row_ptr, const uint32_t* col_idx, uint64_t n_rows, uint32_t K,
                uint32_t L, uint32_t range, const HashKeys& keys, uint32_t* codes, const AddrOut& out,
                cudaStream_t s, uint32_t* long_rows = nullptr, uint32_t long_cap = 0);

// Reservoir sharing (R#23): addrs [n][L] -> reservoir indices [n][L]: entry (r, t) is
// shared_reservoir(t, addrs[r][t]) unless the address is EMPTY/invalid or an earlier table of
// the same row points to the same reservoir (then EMPTY: a row enters / a query aggregates
// each distinct reservoir once).
int launch_shared_reservoirs(const uint32_t* addrs, uint64_t n, uint32_t L, uint32_t range, uint32_t P,
                             const HashKeys& keys, uint32_t* out, unsigned long long* err, cudaStream_t s);

// Build scratch / state.  All bucket-indexed arrays have nb = L*range entries (+1).
struct BuildArgs {
  const uint32_t* addrs;  // row r, table t at addrs[r*astride + t - acol0]
  uint32_t astride, acol0;  // [n][L]: L, 0; a column window [n][t1-t0]: t1-t0, t0
  uint32_t* addrsT;         // scratch [t1-t0][n] for the table-major / shared-memory passes, or null
  uint32_t* hbuf;           // scratch [C + (t1-t0)][range] segment histograms: shared-memory passes, or null
  uint32_t shared;          // 0: bucket (t, a) is t*range + a; else addrs hold shared-reservoir
                            // indices < shared (k_shared_reservoirs output) used as the bucket
  uint64_t n;
  uint32_t id_base;
  uint32_t L, R, range;
  uint32_t t0, t1;  // only tables [t0, t1) receive the new rows (others keep their content)
  HashKeys keys;
  // old tables (null when empty)
  const uint64_t* goff_old;  // [nb+1]
  const uint32_t* ids_old;
  // outputs / scratch
  uint32_t* arrivals;         // [nb], accumulated
  uint32_t* cursor;           // [nb] scratch
  uint64_t* pool_cnt;         // [nb+1] scratch (becomes pool offsets after scan)
  uint64_t* pool_off;         // [nb+1]
  uint64_t* keep_cnt;         // [nb+1]
  uint64_t* goff_new;         // [nb+1]
  uint32_t* pool;             // [pool capacity]
  uint32_t* ids_new;          // [kept capacity]
  uint32_t* big_list;         // [nb] bucket indices for the CTA path
  uint32_t* big_count;        // [4]: CTA-path, warp-path (mid), register-path and early list counts
  uint32_t* early_list;       // [nb] buckets with > 512 members, listed by k_pool_sizes, or null
  void* side_stream;          // with early_list: k_select_big runs these on this stream,
  void* side_fork;            //   concurrently with the other select kernels (events fork /
  void* side_join;            //   join it with the caller's stream)
  uint64_t* gslots;           // [build_group_slots(range, n, t1-t0)] scratch of the grouped
                              // table-major passes (fresh table-major builds), or null
  unsigned long long* err;    // device error counter
  void* scan_tmp;
  size_t scan_tmp_bytes;
  // optional: called once the new bucket offsets (goff_new) are final, with the side stream
  // already ordered after them (flash_knn_graph plans its queries there, concurrently with
  // the scatter and selects); the build joins the side stream before it returns
  void (*after_scan)(void* ctx, cudaStream_t side);
  void* after_scan_ctx;
};
size_t build_scan_tmp_bytes(uint64_t nb);
uint32_t smem_build_ctas(uint32_t W, uint64_t n);  // CTAs of the shared-memory passes (hbuf: (C + W) slots)
bool smem_build_fits(uint32_t range);
uint64_t build_group_slots(uint32_t range, uint64_t n, uint32_t W);
int launch_build(const BuildArgs& a, cudaStream_t s);

struct QueryArgs {
  // Segment t (t < L) of query q is ids[goff[i] .. goff[i+1]) with i = t*range + addrs[q*L+t]
  // (a table bucket), or i = t*range + q when `direct` (pre-gathered candidate segments,
  // range = nq: the candidate-exchange owner side).  Counts are <= cmax (the index's L).
  const uint32_t* addrs;  // [nq][L] (unused when direct)
  uint64_t nq;
  const uint64_t* goff;   // [L*range+1]
  const uint32_t* ids;
  uint32_t L, range, k;
  uint32_t cmax;          // largest possible count (= the index's L)
  int direct;
  uint32_t shared;        // 0, or: addrs hold shared-reservoir indices (bucket = the index itself)
  const uint32_t* exclude;  // [nq] or null
  int exclude_self;         // exclude id = self_base + q
  uint32_t self_base;
  uint32_t* out_ids;
  uint32_t* out_counts;
  unsigned long long* err;
  const uint32_t* seg_len;  // direct mode only (or null): segment i has seg_len[i] ids starting at
                            // goff[i] (segments need not be contiguous); null: goff[i+1] - goff[i]
  uint64_t mmax;            // a query has at most mmax = L*R candidates (more: error counter + pads)
  uint32_t max_id;          // largest id inserted (the sort kernel's digit range)
  int planned;              // launch_query_plan already ran for these queries (skip it)
};
// scratch: query_scratch_bytes(nq) bytes of device memory (size-class lists).  Returns the
// number of kernels launched, or -1 if some size class could not be launched.
int launch_query(const QueryArgs& a, void* scratch, cudaStream_t s);
// the size-class planning step of launch_query alone (needs only addrs and goff)
int launch_query_plan(const QueryArgs& a, void* scratch, cudaStream_t s);
size_t query_scratch_bytes(uint64_t nq);
// every size class of an index with L tables, R per bucket, top-k has a kernel that fits
// (L*R <= FLASH_MAX_CANDIDATES and the CTA sort kernel's shared memory fits)
bool query_shape_fits(uint32_t L, uint32_t R, uint32_t k);
// occupancy-bitmap CTA-per-query kernel (query_mark.cu) for indexes whose ids fit a
// shared-memory bitmap: launch_query routes the queries with more than query_mark_min(a)
// candidates to it (0xFFFFFFFF: never); the queries it cannot finish go to the CTA sort
// kernel.  list/count: device-side query list; fb: scratch for nq + 1 u32 (fallback list)
uint32_t query_mark_min(const QueryArgs& a);
int launch_query_mark(const QueryArgs& a, const uint32_t* list, const uint32_t* count, uint32_t* fb, cudaStream_t s);
// CTA sort kernel over a device-side query list (list[0..*count)), M <= cap
int launch_csort(const QueryArgs& a, uint32_t cap, const uint32_t* list, const uint32_t* count, cudaStream_t s);
// radix-partition warp-per-query kernel for queries with M <= mcap candidates (k <= 256)
int launch_query_sort(const QueryArgs& a, uint32_t mcap, const uint32_t* list, const uint32_t* count,
                      cudaStream_t s, uint32_t* next = nullptr);

// Candidate exchange, sender side (exchange.cu).  addrs: [n][t1-t0] (a table window's
// columns).  sizes[q] = sum of the window buckets' sizes; off = exclusive scan (n+1).
int launch_window_sizes(const uint32_t* addrs, uint64_t n, uint32_t t0, uint32_t t1, uint32_t range,
                        const uint64_t* goff, uint32_t* sizes, uint64_t* off, void* scan_tmp,
                        size_t scan_tmp_bytes, unsigned long long* err, cudaStream_t s);
size_t scan_u32_to_u64_tmp_bytes(uint64_t n);
// out[off[q] ..] = concatenation of query q's window buckets (table order).
int launch_window_gather(const uint32_t* addrs, uint64_t n, uint32_t t0, uint32_t t1, uint32_t range,
                         const uint64_t* goff, const uint32_t* ids, const uint64_t* off, uint32_t* out,
                         cudaStream_t s);
// exclusive scan of n uint32 sizes into n+1 uint64 offsets
int launch_scan_sizes(const uint32_t* sizes, uint64_t n, uint64_t* off, void* scan_tmp, size_t scan_tmp_bytes,
                      cudaStream_t s);

}  // namespace flash
