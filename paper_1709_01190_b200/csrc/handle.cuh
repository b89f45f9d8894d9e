// handle.cuh — the flash_index handle and the host-side helpers the C ABI entry points
// share (flash_api.cu: single-GPU calls; dist.cu: the multi-GPU handle).  Internal to
// libflash.so.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "flash.h"
#include "flash_internal.cuh"

namespace flash {
namespace api {

// Record `st` with a printf-style message as this thread's flash_last_error and return it.
flash_status fail(flash_status st, const char* fmt, ...);

#define CUDA_TRY(expr)                                                                        \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess) {                                                                  \
      cudaGetLastError();                                                                     \
      return ::flash::api::fail(e_ == cudaErrorMemoryAllocation ? FLASH_ENOMEM : FLASH_ECUDA, \
                                "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__,    \
                                __LINE__);                                                    \
    }                                                                                         \
  } while (0)

#define TRY(expr)                    \
  do {                               \
    flash_status st_ = (expr);       \
    if (st_ != FLASH_OK) return st_; \
  } while (0)

struct PendingPhase {
  int phase;
  cudaEvent_t a, b;
};

// A grow-only device buffer (cudaMalloc: one allocation each, so it can be exported to a
// peer process with cudaIpcGetMemHandle).
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  template <typename T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};
flash_status ensure(DevBuf& b, size_t bytes);
void release(DevBuf& b);

struct DistState;  // dist.cu

}  // namespace api
}  // namespace flash

struct flash_index {
  uint32_t K, L, R, range;
  uint32_t shared = 0;  // reservoir sharing (R#23): pool size P < L*range, or 0 (unshared)
  uint64_t seed;
  flash::HashKeys keys;
  int device;
  // tables: goff / ids double-buffered; `have_tables` false before the first insert
  uint32_t* arrivals = nullptr;  // [L*range]
  flash::api::DevBuf goff[2], ids[2];
  int cur = 0;
  bool have_tables = false;
  uint64_t kept_ub = 0;     // host upper bound on kept ids
  uint64_t n_inserted = 0;  // rows passed to insert (host count)
  uint64_t max_id = 0;      // largest id inserted so far (host count)
  // scratch
  flash::api::DevBuf addrs, cursor, pool_cnt, pool_off, keep_cnt, pool, big_list, scan_tmp, qscratch, off_tmp;
  flash::api::DevBuf seg_off, xscan_tmp;  // flash_count_topk segment offsets; exchange scans
  flash::api::DevBuf addrsT;              // build: window addresses transposed to [W][n] (table-major passes)
  flash::api::DevBuf raddr, qraddr;       // shared mode: rows' / queries' distinct reservoir indices
  flash::api::DevBuf hbuf;                // build: slice histograms of the shared-memory passes
  flash::api::DevBuf gslots;              // build: group slot offsets of the grouped table-major passes
  flash::api::DevBuf long_rows;           // hash: [cap] rows k_doph_sparse leaves to k_doph, + counter
  flash::api::DevBuf h_rp, h_col, h_ids, h_cnt;  // flash_knn_graph_host staging
  flash::api::DevBuf zero;                // 16 zero bytes (a valid device pointer for empty inputs)
  unsigned long long* err = nullptr;
  cudaStream_t last_stream = nullptr;
  bool have_last = false;
  cudaEvent_t order_ev = nullptr;
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> copy_events;
  cudaStream_t side_stream = nullptr;  // build: k_select_big of the early-listed buckets
  cudaEvent_t side_fork = nullptr, side_join = nullptr;

  // profiling
  int profiling = 0;
  int phase_depth[4] = {0, 0, 0, 0};  // open Phase scopes per phase (nested ones are not timed twice)
  std::vector<flash::api::PendingPhase> pending;
  double phase_ms[4] = {0, 0, 0, 0};
  uint64_t phase_calls[4] = {0, 0, 0, 0};
  uint64_t launches = 0;

  // multi-GPU handle (flash_create_dist / flash_create_dist_local): null for a plain index
  flash::api::DistState* dist = nullptr;
};

namespace flash {
namespace api {

// Order this call after everything previously enqueued on the handle (and make its device
// current).
flash_status enter(const flash_index* h, cudaStream_t s);

// CUDA events around one phase of a call on stream s, when profiling is on.
struct Phase {
  flash_index* h;
  int phase;
  cudaStream_t s;
  cudaEvent_t a = nullptr, b = nullptr;
  Phase(const flash_index* hc, int p, cudaStream_t st);
  ~Phase();
};

// True when the GPU can dereference p (device, managed, or mapped host memory).
bool device_accessible(const void* p);

// buckets (reservoirs) the index holds: L*range, or the shared pool's P (R#23)
uint64_t nbuckets(const flash_index* h);

// tables = false: the handle never holds tables itself (a multi-GPU handle's outer handle)
flash_index* new_handle(uint32_t K, uint32_t L, uint32_t R, uint32_t range, uint64_t seed, uint32_t shared,
                        flash_status* st, bool tables = true);
void free_handle(flash_index* h);

flash_status do_hash(const flash_index* h, const int64_t* row_ptr, const uint32_t* col_idx, uint64_t n,
                     uint32_t* codes, const AddrOut& out, cudaStream_t s);
flash_status do_insert_addrs(flash_index* h, const uint32_t* addrs, uint64_t n, uint32_t id_base, cudaStream_t s,
                             uint32_t t0 = 0, uint32_t t1 = UINT32_MAX, bool cols = false, bool converted = false,
                             void (*after_scan)(void*, cudaStream_t) = nullptr, void* after_scan_ctx = nullptr);
QueryArgs query_args(const flash_index* h, const uint32_t* addrs, uint64_t nq, uint32_t k, const uint32_t* exclude,
                     int exclude_self, uint32_t self_base, uint32_t* out_ids, uint32_t* out_counts, int cur);
flash_status do_query_addrs(const flash_index* h, const uint32_t* addrs, uint64_t nq, uint32_t k,
                            const uint32_t* exclude, int exclude_self, uint32_t self_base, uint32_t* out_ids,
                            uint32_t* out_counts, cudaStream_t s, bool converted = false, bool planned = false);
// the count / top-k step (Q2-Q3) over a prepared QueryArgs (direct segments, dist.cu)
flash_status run_query(flash_index* h, const QueryArgs& a, cudaStream_t s);
flash_status check_query_shape(const flash_index* h, uint32_t k);

}  // namespace api
}  // namespace flash
