// flash_api.cu — the C ABI of libflash.so (include/flash.h): handle, validation,
// handle-owned device arena, phase orchestration, profiling counters.  The multi-GPU
// handle's collective calls live in dist.cu.
//
// Every entry point validates on the host before enqueueing anything, enqueues on the
// caller's stream, and returns without synchronizing (except where flash.h says so).
// Device memory: the handle owns every buffer the path needs (tables double-buffered,
// scratch sized to the largest call so far).  Buffers only grow, so steady-state calls
// never allocate (growth uses cudaMalloc/cudaFree, which synchronize the device).
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "dist.cuh"
#include "flash.h"
#include "flash_internal.cuh"
#include "handle.cuh"

using namespace flash;
using namespace flash::api;

namespace {
thread_local std::string g_last_error;

__global__ void k_table_off(const uint64_t* goff, uint32_t t, uint32_t range, uint32_t* off) {
  const uint64_t base = goff[(uint64_t)t * range];
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b <= range; b += gridDim.x * blockDim.x)
    off[b] = (uint32_t)(goff[(uint64_t)t * range + b] - base);
}

// flash_import_tables' consistency check: goff[0] == 0, goff non-decreasing, goff[nb] ==
// n_ids (bad[0] counts violations), and the largest imported id (bad[1]).
__global__ void k_import_check(const uint64_t* __restrict__ goff, uint64_t nb, const uint32_t* __restrict__ ids,
                               uint64_t n_ids, unsigned long long* bad) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long nbad = 0;
  for (uint64_t i = i0; i < nb; i += stride)
    if (goff[i + 1] < goff[i]) ++nbad;
  if (i0 == 0 && (goff[0] != 0 || goff[nb] != n_ids)) ++nbad;
  uint32_t mx = 0;
  for (uint64_t i = i0; i < n_ids; i += stride) mx = ids[i] > mx ? ids[i] : mx;
  if (nbad) atomicAdd(&bad[0], nbad);
  if (mx) atomicMax(&bad[1], (unsigned long long)mx);
}
}  // namespace

namespace flash {
namespace api {

flash_status fail(flash_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

flash_status ensure(DevBuf& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (b.cap >= bytes) return FLASH_OK;
  if (b.p) CUDA_TRY(cudaFree(b.p));
  b.p = nullptr;
  b.cap = 0;
  const size_t want = bytes + bytes / 8;  // headroom against repeated regrowth
  CUDA_TRY(cudaMalloc(&b.p, want));
  b.cap = want;
  return FLASH_OK;
}

void release(DevBuf& b) {
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
}

flash_status enter(const flash_index* hc, cudaStream_t s) {
  flash_index* h = const_cast<flash_index*>(hc);
  CUDA_TRY(cudaSetDevice(h->device));
  if (h->have_last && h->last_stream != s) {
    CUDA_TRY(cudaEventRecord(h->order_ev, h->last_stream));
    CUDA_TRY(cudaStreamWaitEvent(s, h->order_ev, 0));
  }
  h->last_stream = s;
  h->have_last = true;
  return FLASH_OK;
}

Phase::Phase(const flash_index* hc, int p, cudaStream_t st) : h(const_cast<flash_index*>(hc)), phase(p), s(st) {
  if (h->profiling && h->phase_depth[p]++ == 0) {  // the outermost scope of this phase times it
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
  }
}
Phase::~Phase() {
  if (h->profiling) --h->phase_depth[phase];
  if (a) {
    cudaEventRecord(b, s);
    h->pending.push_back({phase, a, b});
  }
}

bool device_accessible(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged ||
         (at.type == cudaMemoryTypeHost && at.devicePointer != nullptr);
}

#define REQUIRE_DEV(p)                                                                     \
  do {                                                                                     \
    if (!device_accessible(p)) return fail(FLASH_EINVAL, "%s is not a device pointer", #p); \
  } while (0)

uint64_t nbuckets(const flash_index* h) { return h->shared ? h->shared : (uint64_t)h->L * h->range; }

flash_index* new_handle(uint32_t K, uint32_t L, uint32_t R, uint32_t range, uint64_t seed, uint32_t shared,
                        flash_status* st, bool tables) {
  *st = FLASH_OK;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *st = fail(FLASH_ECUDA, "flash_create: %s", cudaGetErrorString(e));
    return nullptr;
  }
  flash_index* h = new (std::nothrow) flash_index();
  if (!h) {
    *st = fail(FLASH_ENOMEM, "host allocation failed");
    return nullptr;
  }
  h->K = K;
  h->L = L;
  h->R = R;
  h->range = range;
  h->seed = seed;
  h->keys = derive_keys(seed);
  h->device = dev;
  h->shared = shared;
  const size_t nb = !tables ? 1 : shared ? shared : (size_t)L * range;
  e = cudaMalloc(&h->arrivals, sizeof(uint32_t) * (nb ? nb : 1));
  if (e == cudaSuccess) e = cudaMemset(h->arrivals, 0, sizeof(uint32_t) * (nb ? nb : 1));
  if (e == cudaSuccess) e = cudaMalloc(&h->err, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(h->err, 0, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->order_ev, cudaEventDisableTiming);
  if (e == cudaSuccess && ensure(h->zero, 16) == FLASH_OK) e = cudaMemset(h->zero.p, 0, 16);
  if (e != cudaSuccess || !h->zero.p) {
    cudaGetLastError();
    free_handle(h);
    *st = fail(e == cudaErrorMemoryAllocation ? FLASH_ENOMEM : FLASH_ECUDA, "flash_create: %s",
               cudaGetErrorString(e));
    return nullptr;
  }
  return h;
}

void free_handle(flash_index* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  for (auto& p : h->pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : h->copy_events) cudaEventDestroy(e);
  if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
  if (h->side_stream) cudaStreamDestroy(h->side_stream);
  if (h->side_fork) cudaEventDestroy(h->side_fork);
  if (h->side_join) cudaEventDestroy(h->side_join);
  cudaFree(h->arrivals);
  cudaFree(h->err);
  for (DevBuf* b : {&h->goff[0], &h->goff[1], &h->ids[0], &h->ids[1], &h->addrs, &h->cursor, &h->pool_cnt,
                    &h->pool_off, &h->keep_cnt, &h->pool, &h->big_list, &h->scan_tmp, &h->qscratch, &h->off_tmp,
                    &h->seg_off, &h->xscan_tmp, &h->addrsT, &h->raddr, &h->qraddr, &h->hbuf, &h->gslots, &h->long_rows, &h->h_rp, &h->h_col,
                    &h->h_ids, &h->h_cnt, &h->zero})
    release(*b);
  if (h->order_ev) cudaEventDestroy(h->order_ev);
  delete h;
}

flash_status do_hash(const flash_index* h, const int64_t* row_ptr, const uint32_t* col_idx, uint64_t n,
                     uint32_t* codes, const AddrOut& out, cudaStream_t s) {
  Phase ph(h, 0, s);
  // the rows k_doph_sparse leaves to k_doph are listed (up to kLongCap; more: k_doph scans
  // every row's extent) when K*L <= 256, so that k_doph does not read all n extents
  flash_index* hm = const_cast<flash_index*>(h);
  uint32_t* long_rows = nullptr;
  uint32_t long_cap = 0;
  if ((uint64_t)h->K * h->L > 256 && n > 0) {  // the mid kernel's chunk counter (8 B)
    TRY(ensure(hm->long_rows, 8));
    long_rows = hm->long_rows.as<uint32_t>();
  } else if ((uint64_t)h->K * h->L <= 256 && n > 0) {
    const char* ce = getenv("FLASH_DOPH_LONGCAP");  // tests: a small cap (the full-scan fallback)
    const uint64_t kLongCap = ce ? strtoull(ce, nullptr, 10) : (1ull << 25);
    long_cap = (uint32_t)(n < kLongCap ? n : kLongCap);
    TRY(ensure(hm->long_rows, sizeof(uint32_t) * (((size_t)long_cap + 3) & ~(size_t)1) + 8));
    long_rows = hm->long_rows.as<uint32_t>();
  }
  hm->launches += launch_doph(row_ptr, col_idx, n, h->K, h->L, h->range, h->keys, codes, out, s, long_rows,
                              long_cap);
  CUDA_TRY(cudaGetLastError());
  return FLASH_OK;
}

flash_status do_insert_addrs(flash_index* h, const uint32_t* addrs, uint64_t n, uint32_t id_base, cudaStream_t s,
                             uint32_t t0, uint32_t t1, bool cols, bool converted,
                             void (*after_scan)(void*, cudaStream_t), void* after_scan_ctx) {
  if (t1 > h->L) t1 = h->L;
  const uint64_t nb = nbuckets(h);
  if (h->shared && !converted) {  // table addresses -> each row's distinct shared reservoirs
    TRY(ensure(h->raddr, sizeof(uint32_t) * n * h->L));
    Phase ph(h, 1, s);
    h->launches += launch_shared_reservoirs(addrs, n, h->L, h->range, h->shared, h->keys,
                                            h->raddr.as<uint32_t>(), h->err, s);
    CUDA_TRY(cudaGetLastError());
    addrs = h->raddr.as<uint32_t>();
  }
  const uint64_t pool_cap = h->kept_ub + n * h->L;
  const uint64_t kept_cap = pool_cap < nb * h->R ? pool_cap : nb * h->R;
  const int nxt = h->have_tables ? 1 - h->cur : h->cur;
  // buffers first (growth synchronizes; it happens outside the profiled phase)
  TRY(ensure(h->cursor, sizeof(uint32_t) * nb));
  TRY(ensure(h->pool_cnt, sizeof(uint64_t) * (nb + 1)));
  TRY(ensure(h->pool_off, sizeof(uint64_t) * (nb + 1)));
  TRY(ensure(h->keep_cnt, sizeof(uint64_t) * (nb + 1)));
  TRY(ensure(h->goff[nxt], sizeof(uint64_t) * (nb + 1)));
  TRY(ensure(h->pool, sizeof(uint32_t) * pool_cap));
  TRY(ensure(h->ids[nxt], sizeof(uint32_t) * kept_cap));
  TRY(ensure(h->big_list, sizeof(uint32_t) * (2 * nb + 4)));  // late list, 4 counters, early list
  if (!h->side_stream) {
    CUDA_TRY(cudaStreamCreateWithFlags(&h->side_stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&h->side_fork, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&h->side_join, cudaEventDisableTiming));
  }
  TRY(ensure(h->scan_tmp, build_scan_tmp_bytes(nb)));
  // Table-major passes once the per-bucket arrays (cursor + pool offset, 12 B per bucket)
  // no longer fit comfortably in L2 and each table has enough buckets that the resident
  // CTAs' atomics (all on one or two tables) do not pile onto the same counters (measured:
  // kdd12, 2^20 buckets/table, 3.6x faster; url, 2^15, 2.6x slower); FLASH_BUILD_TM=0/1
  // forces the choice (tests).
  const char* tm_env = getenv("FLASH_BUILD_TM");
  const bool tm = !h->shared &&
                  (tm_env ? tm_env[0] == '1' : (nb * 12 > (32ull << 20) && h->range >= (1u << 18)));
  // shared-memory passes when a table's bucket counters fit shared memory (the default
  // there; FLASH_BUILD_SMEM=0 disables them, tests)
  const char* sm_env = getenv("FLASH_BUILD_SMEM");
  const bool smb = !tm && !h->shared && t1 > t0 && n > 0 && smem_build_fits(h->range) &&
                   !(sm_env && sm_env[0] == '0');
  if ((tm || smb) && t1 > t0) TRY(ensure(h->addrsT, sizeof(uint32_t) * n * (t1 - t0)));
  if (smb)
    TRY(ensure(h->hbuf, sizeof(uint32_t) * ((size_t)(t1 - t0) + smem_build_ctas(t1 - t0, n)) * h->range));
  const bool grouped = tm && !h->have_tables && t1 > t0 && n > 0;  // (launch_build may still decline)
  if (grouped) TRY(ensure(h->gslots, sizeof(uint64_t) * build_group_slots(h->range, n, t1 - t0)));

  Phase ph(h, 1, s);
  BuildArgs a;
  memset(&a, 0, sizeof a);
  a.addrs = addrs;
  a.astride = cols ? t1 - t0 : h->L;  // cols: addrs holds only the window's columns
  a.acol0 = cols ? t0 : 0;
  a.addrsT = ((tm || smb) && t1 > t0) ? h->addrsT.as<uint32_t>() : nullptr;
  a.hbuf = smb ? h->hbuf.as<uint32_t>() : nullptr;
  a.gslots = grouped ? h->gslots.as<uint64_t>() : nullptr;
  a.shared = h->shared;
  a.n = n;
  a.id_base = id_base;
  a.L = h->L;
  a.R = h->R;
  a.range = h->range;
  a.t0 = t0;
  a.t1 = t1;
  a.keys = h->keys;
  a.goff_old = h->have_tables ? h->goff[h->cur].as<uint64_t>() : nullptr;
  a.ids_old = h->have_tables ? h->ids[h->cur].as<uint32_t>() : nullptr;
  a.arrivals = h->arrivals;
  a.err = h->err;
  a.cursor = h->cursor.as<uint32_t>();
  a.pool_cnt = h->pool_cnt.as<uint64_t>();
  a.pool_off = h->pool_off.as<uint64_t>();
  a.keep_cnt = h->keep_cnt.as<uint64_t>();
  a.goff_new = h->goff[nxt].as<uint64_t>();
  a.pool = h->pool.as<uint32_t>();
  a.ids_new = h->ids[nxt].as<uint32_t>();
  a.big_list = h->big_list.as<uint32_t>();
  a.big_count = h->big_list.as<uint32_t>() + nb;
  a.early_list = h->big_list.as<uint32_t>() + nb + 4;
  a.side_stream = h->side_stream;
  a.side_fork = h->side_fork;
  a.side_join = h->side_join;
  a.after_scan = after_scan;
  a.after_scan_ctx = after_scan_ctx;
  a.scan_tmp = h->scan_tmp.p;
  a.scan_tmp_bytes = h->scan_tmp.cap;
  h->launches += launch_build(a, s);
  CUDA_TRY(cudaGetLastError());
  h->cur = nxt;
  h->have_tables = true;
  h->kept_ub = kept_cap;
  h->n_inserted += n;
  if ((uint64_t)id_base + n - 1 > h->max_id) h->max_id = (uint64_t)id_base + n - 1;
  return FLASH_OK;
}

QueryArgs query_args(const flash_index* h, const uint32_t* addrs, uint64_t nq, uint32_t k, const uint32_t* exclude,
                     int exclude_self, uint32_t self_base, uint32_t* out_ids, uint32_t* out_counts, int cur) {
  QueryArgs a;
  memset(&a, 0, sizeof a);
  a.addrs = addrs;
  a.nq = nq;
  a.goff = h->goff[cur].as<uint64_t>();
  a.ids = h->ids[cur].as<uint32_t>();
  a.L = h->L;
  a.range = h->range;
  a.k = k;
  a.cmax = h->L;
  a.direct = 0;
  a.shared = h->shared;
  a.exclude = exclude;
  a.exclude_self = exclude_self;
  a.self_base = self_base;
  a.out_ids = out_ids;
  a.out_counts = out_counts;
  a.err = h->err;
  a.seg_len = nullptr;
  a.mmax = (uint64_t)h->L * h->R;
  a.max_id = (uint32_t)h->max_id;
  return a;
}

flash_status run_query(flash_index* h, const QueryArgs& a, cudaStream_t s) {
  const int n = launch_query(a, h->qscratch.p, s);
  if (n < 0)
    return fail(FLASH_ECUDA, "query kernels could not be launched for L=%u, R=%u, k=%u (shared memory)", h->L, h->R,
                a.k);
  h->launches += (uint64_t)n;
  CUDA_TRY(cudaGetLastError());
  return FLASH_OK;
}

flash_status do_query_addrs(const flash_index* hc, const uint32_t* addrs, uint64_t nq, uint32_t k,
                            const uint32_t* exclude, int exclude_self, uint32_t self_base,
                            uint32_t* out_ids, uint32_t* out_counts, cudaStream_t s, bool converted,
                            bool planned) {
  flash_index* h = const_cast<flash_index*>(hc);
  if (h->shared && !converted && h->have_tables) {  // each distinct reservoir aggregated once
    TRY(ensure(h->qraddr, sizeof(uint32_t) * nq * h->L));
    Phase ph(h, 2, s);
    h->launches += launch_shared_reservoirs(addrs, nq, h->L, h->range, h->shared, h->keys,
                                            h->qraddr.as<uint32_t>(), h->err, s);
    CUDA_TRY(cudaGetLastError());
    addrs = h->qraddr.as<uint32_t>();
  }
  if (!h->have_tables) {  // nothing inserted: every query returns k pads
    Phase ph(h, 2, s);
    CUDA_TRY(cudaMemsetAsync(out_ids, 0xFF, sizeof(uint32_t) * nq * k, s));
    CUDA_TRY(cudaMemsetAsync(out_counts, 0, sizeof(uint32_t) * nq * k, s));
    return FLASH_OK;
  }
  TRY(ensure(h->qscratch, query_scratch_bytes(nq)));
  Phase ph(h, 2, s);
  QueryArgs a = query_args(h, addrs, nq, k, exclude, exclude_self, self_base, out_ids, out_counts, h->cur);
  a.planned = planned ? 1 : 0;
  return run_query(h, a, s);
}

flash_status check_query_shape(const flash_index* h, uint32_t k) {
  if (k == 0 || k > FLASH_MAX_TOPK) return fail(FLASH_EINVAL, "k=%u outside [1, %u]", k, FLASH_MAX_TOPK);
  if ((uint64_t)h->L * h->R > FLASH_MAX_CANDIDATES)
    return fail(FLASH_EINVAL, "L*R=%llu too large for the count kernels (limit L*R <= %u)",
                (unsigned long long)h->L * h->R, FLASH_MAX_CANDIDATES);
  if (!query_shape_fits(h->L, h->R, k))
    return fail(FLASH_EINVAL, "query shared memory for L=%u, R=%u, k=%u exceeds 227 KB", h->L, h->R, k);
  return FLASH_OK;
}

}  // namespace api
}  // namespace flash

extern "C" {

const char* flash_last_error(void) { return g_last_error.c_str(); }

flash_status flash_create(uint32_t K, uint32_t L, uint32_t R, uint32_t range, uint64_t seed,
                          flash_index** out) {
  return flash_create_pool(K, L, R, range, 0, seed, out);
}

flash_status flash_create_pool(uint32_t K, uint32_t L, uint32_t R, uint32_t range, uint64_t pool, uint64_t seed,
                               flash_index** out) {
  if (!out) return fail(FLASH_EINVAL, "out is NULL");
  *out = nullptr;
  if (K < 1 || L < 1 || (uint64_t)K * L > FLASH_MAX_BINS)
    return fail(FLASH_EINVAL, "need 1 <= K, 1 <= L, K*L <= %u (K=%u L=%u)", FLASH_MAX_BINS, K, L);
  if (R < 1 || R > FLASH_MAX_R) return fail(FLASH_EINVAL, "R=%u outside [1, %u]", R, FLASH_MAX_R);
  if (range < 1 || range > (1u << 31)) return fail(FLASH_EINVAL, "range=%u outside [1, 2^31]", range);
  if ((uint64_t)L * range > (1ull << 31)) return fail(FLASH_EINVAL, "L*range must be <= 2^31");
  if (pool > (uint64_t)L * range)
    return fail(FLASH_EINVAL, "pool=%llu exceeds L*range=%llu", (unsigned long long)pool,
                (unsigned long long)L * range);
  const uint32_t shared = (pool == 0 || pool == (uint64_t)L * range) ? 0u : (uint32_t)pool;
  flash_status st;
  *out = new_handle(K, L, R, range, seed, shared, &st);
  return st;
}

void flash_destroy(flash_index* h) {
  if (!h) return;
  if (h->dist) dist_destroy(h);
  free_handle(h);
}

flash_status flash_hash(const flash_index* h, const int64_t* row_ptr, const uint32_t* col_idx, uint64_t n_rows,
                        uint32_t* codes, uint32_t* addrs, void* stream) {
  if (!h) return fail(FLASH_EINVAL, "handle is NULL");
  if (!codes && !addrs) return fail(FLASH_EINVAL, "codes and addrs are both NULL");
  if (n_rows == 0) return FLASH_OK;
  REQUIRE_DEV(row_ptr);
  REQUIRE_DEV(col_idx);
  if (codes) REQUIRE_DEV(codes);
  if (addrs) REQUIRE_DEV(addrs);
  cudaStream_t s = (cudaStream_t)stream;
  TRY(enter(h, s));
  return do_hash(h, row_ptr, col_idx, n_rows, codes, addr_out(addrs), s);
}

flash_status flash_insert_addrs(flash_index* h, const uint32_t* addrs, uint64_t n_rows, uint32_t id_base,
                                void* stream) {
  if (!h) return fail(FLASH_EINVAL, "handle is NULL");
  if (h->dist) return fail(FLASH_ESTATE, "flash_insert_addrs: not a call of a multi-GPU handle");
  if (n_rows == 0) return FLASH_OK;
  REQUIRE_DEV(addrs);
  if ((uint64_t)id_base + n_rows - 1 >= 0xFFFFFFFFull)
    return fail(FLASH_EINVAL, "ids id_base..id_base+n_rows-1 must stay below 0xFFFFFFFF");
  cudaStream_t s = (cudaStream_t)stream;
  TRY(enter(h, s));
  return do_insert_addrs(h, addrs, n_rows, id_base, s);
}

flash_status flash_insert_addrs_window(flash_index* h, const uint32_t* addrs, uint64_t n_rows, uint32_t id_base,
                                       uint32_t t_begin, uint32_t t_end, void* stream) {
  if (!h) return fail(FLASH_EINVAL, "handle is NULL");
  if (h->dist) return fail(FLASH_ESTATE, "flash_insert_addrs_window: not a call of a multi-GPU handle");
  if (h->shared) return fail(FLASH_EINVAL, "table windows are undefined when tables share reservoirs (R#23)");
  if (t_begin > t_end || t_end > h->L) return fail(FLASH_EINVAL, "table window [%u, %u) outside [0, %u)", t_begin, t_end, h->L);
  if (n_rows == 0) return FLASH_OK;
  REQUIRE_DEV(addrs);
  if ((uint64_t)id_base + n_rows - 1 >= 0xFFFFFFFFull)
    return fail(FLASH_EINVAL, "ids id_base..id_base+n_rows-1 must stay below 0xFFFFFFFF");
  cudaStream_t s = (cudaStream_t)stream;
  TRY(enter(h, s));
  return do_insert_addrs(h, addrs, n_rows, id_base, s, t_begin, t_end);
}

flash_status flash_table_arrays(const flash_index* hc, const uint64_t** goff, const uint32_t** ids,
                                const uint32_t** arrivals, uint64_t* n_ids) {
  if (!hc) return fail(FLASH_EINVAL, "handle is NULL");
  flash_index* h = const_cast<flash_index*>(hc);
  if (h->dist) return fail(FLASH_ESTATE, "flash_table_arrays: a multi-GPU handle holds only its table window");
  if (!h->have_tables) return fail(FLASH_ESTATE, "nothing inserted yet");
  CUDA_TRY(cudaSetDevice(h->device));
  if (h->have_last) CUDA_TRY(cudaStreamSynchronize(h->last_stream));
  const uint64_t* g = h->goff[h->cur].as<uint64_t>();
  uint64_t total = 0;
  CUDA_TRY(cudaMemcpy(&total, g + nbuckets(h), sizeof total, cudaMemcpyDeviceToHost));
  if (goff) *goff = g;
  if (ids) *ids = h->ids[h->cur].as<uint32_t>();
  if (arrivals) *arrivals = h->arrivals;
  if (n_ids) *n_ids = total;
  return FLASH_OK;
}

flash_status flash_import_tables(flash_index* h, const uint64_t* goff, const uint32_t* ids, uint64_t n_ids,
                                 const uint32_t* arrivals, void* stream) {
  if (!h) return fail(FLASH_EINVAL, "handle is NULL");
  if (h->dist) return fail(FLASH_ESTATE, "flash_import_tables: not a call of a multi-GPU handle");
  REQUIRE_DEV(goff);
  if (n_ids) REQUIRE_DEV(ids);
  if (arrivals) REQUIRE_DEV(arrivals);
  if (n_ids >= 0x100000000ull * 64) return fail(FLASH_EINVAL, "n_ids=%llu too large", (unsigned long long)n_ids);
  cudaStream_t s = (cudaStream_t)stream;
  TRY(enter(h, s));
  const uint64_t nb = nbuckets(h);
  // validate the offsets and find the largest id before anything changes (synchronizes)
  TRY(ensure(h->off_tmp, 2 * sizeof(unsigned long long)));
  unsigned long long* chk = h->off_tmp.as<unsigned long long>();
  CUDA_TRY(cudaMemsetAsync(chk, 0, 2 * sizeof(unsigned long long), s));
  const uint64_t work = nb > n_ids ? nb : n_ids;
  const unsigned blocks = (unsigned)((work + 255) / 256 < (uint64_t)device_sms() * 8 ? (work + 255) / 256
                                                                                   : (uint64_t)device_sms() * 8);
  k_import_check<<<blocks ? blocks : 1, 256, 0, s>>>(goff, nb, n_ids ? ids : h->zero.as<uint32_t>(), n_ids, chk);
  h->launches++;
  unsigned long long hv[2] = {0, 0};
  CUDA_TRY(cudaMemcpyAsync(hv, chk, sizeof hv, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (hv[0])
    return fail(FLASH_EINVAL, "flash_import_tables: goff must start at 0, be non-decreasing and end at n_ids=%llu",
                (unsigned long long)n_ids);
  const int nxt = h->have_tables ? 1 - h->cur : h->cur;
  TRY(ensure(h->goff[nxt], sizeof(uint64_t) * (nb + 1)));
  TRY(ensure(h->ids[nxt], sizeof(uint32_t) * (n_ids ? n_ids : 1)));
  CUDA_TRY(cudaMemcpyAsync(h->goff[nxt].p, goff, sizeof(uint64_t) * (nb + 1), cudaMemcpyDeviceToDevice, s));
  if (n_ids) CUDA_TRY(cudaMemcpyAsync(h->ids[nxt].p, ids, sizeof(uint32_t) * n_ids, cudaMemcpyDeviceToDevice, s));
  if (arrivals)
    CUDA_TRY(cudaMemcpyAsync(h->arrivals, arrivals, sizeof(uint32_t) * nb, cudaMemcpyDeviceToDevice, s));
  else
    CUDA_TRY(cudaMemsetAsync(h->arrivals, 0, sizeof(uint32_t) * nb, s));
  h->cur = nxt;
  h->have_tables = true;
  h->kept_ub = n_ids;
  h->max_id = hv[1];
  h->n_inserted = hv[1] + 1;
  return FLASH_OK;
}

flash_status flash_insert(flash_index* h, const int64_t* row_ptr, const uint32_t* col_idx, uint64_t n_rows,
                          uint32_t id_base, void* stream) {
  if (!h) return fail(FLASH_EINVAL, "handle is NULL");
  if (n_rows == 0 && !h->dist) return FLASH_OK;  // (a multi-GPU insert is collective: every rank calls)
  if (n_rows) {
    REQUIRE_DEV(row_ptr);
    REQUIRE_DEV(col_idx);
  }
  if ((uint64_t)id_base + n_rows - 1 >= 0xFFFFFFFFull)
    return fail(FLASH_EINVAL, "ids id_base..id_base+n_rows-1 must stay below 0xFFFFFFFF");
  cudaStream_t s = (cudaStream_t)stream;
  if (h->dist) return dist_insert(h, row_ptr, col_idx, n_rows, id_base, s);
  TRY(enter(h, s));
  TRY(ensure(h->addrs, sizeof(uint32_t) * n_rows * h->L));
  uint32_t* addrs = h->addrs.as<uint32_t>();
  TRY(do_hash(h, row_ptr, col_idx, n_rows, nullptr, addr_out(addrs), s));
  return do_insert_addrs(h, addrs, n_rows, id_base, s);
}

flash_status flash_query_addrs(const flash_index* h, const uint32_t* addrs, uint64_t n_q, uint32_t k,
                               const uint32_t* exclude, uint32_t* out_ids, uint32_t* out_counts, void* stream) {
  if (!h) return fail(FLASH_EINVAL, "handle is NULL");
  if (h->dist) return fail(FLASH_ESTATE, "flash_query_addrs: not a call of a multi-GPU handle");
  TRY(check_query_shape(h, k));
  if (n_q == 0) return FLASH_OK;
  REQUIRE_DEV(addrs);
  REQUIRE_DEV(out_ids);
  REQUIRE_DEV(out_counts);
  if (exclude) REQUIRE_DEV(exclude);
  cudaStream_t s = (cudaStream_t)stream;
  TRY(enter(h, s));
  return do_query_addrs(h, addrs, n_q, k, exclude, 0, 0, out_ids, out_counts, s);
}

flash_status flash_query_topk(const flash_index* hc, const int64_t* row_ptr, const uint32_t* col_idx,
                              uint64_t n_q, uint32_t k, const uint32_t* exclude, uint32_t* out_ids,
                              uint32_t* out_counts, void* stream) {
  if (!hc) return fail(FLASH_EINVAL, "handle is NULL");
  flash_index* h = const_cast<flash_index*>(hc);
  TRY(check_query_shape(h, k));
  if (n_q == 0 && !h->dist) return FLASH_OK;
  if (n_q) {
    REQUIRE_DEV(row_ptr);
    REQUIRE_DEV(col_idx);
    REQUIRE_DEV(out_ids);
    REQUIRE_DEV(out_counts);
    if (exclude) REQUIRE_DEV(exclude);
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (h->dist) return dist_query_topk(h, row_ptr, col_idx, n_q, k, exclude, out_ids, out_counts, s);
  TRY(enter(h, s));
  TRY(ensure(h->addrs, sizeof(uint32_t) * n_q * h->L));
  uint32_t* addrs = h->addrs.as<uint32_t>();
  TRY(do_hash(h, row_ptr, col_idx, n_q, nullptr, addr_out(addrs), s));
  return do_query_addrs(h, addrs, n_q, k, exclude, 0, 0, out_ids, out_counts, s);
}

flash_status flash_knn_graph(flash_index* h, const int64_t* row_ptr, const uint32_t* col_idx, uint64_t n_rows,
                             uint32_t k, uint32_t* out_ids, uint32_t* out_counts, void* stream) {
  if (!h) return fail(FLASH_EINVAL, "handle is NULL");
  if (h->have_tables || h->n_inserted) return fail(FLASH_ESTATE, "flash_knn_graph needs a fresh handle");
  TRY(check_query_shape(h, k));
  if (n_rows == 0 && !h->dist) return FLASH_OK;
  if (n_rows >= 0xFFFFFFFFull) return fail(FLASH_EINVAL, "n_rows must be < 2^32-1");
  if (n_rows) {
    REQUIRE_DEV(row_ptr);
    REQUIRE_DEV(col_idx);
    REQUIRE_DEV(out_ids);
    REQUIRE_DEV(out_counts);
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (h->dist) return dist_knn_graph(h, row_ptr, col_idx, n_rows, k, out_ids, out_counts, s);
  TRY(enter(h, s));
  TRY(ensure(h->addrs, sizeof(uint32_t) * n_rows * h->L));
  uint32_t* addrs = h->addrs.as<uint32_t>();
  TRY(do_hash(h, row_ptr, col_idx, n_rows, nullptr, addr_out(addrs), s));
  if (h->shared) {  // the rows' distinct reservoirs are the queries' too
    TRY(do_insert_addrs(h, addrs, n_rows, 0, s));
    return do_query_addrs(h, h->raddr.as<uint32_t>(), n_rows, k, nullptr, 1, 0, out_ids, out_counts, s, true);
  }
  // The queries' size-class plan needs only their addresses and the new bucket offsets, so
  // it runs on the build's side stream as soon as the offsets are scanned, beside the
  // scatter and selects; the build joins it before returning.
  TRY(ensure(h->qscratch, query_scratch_bytes(n_rows)));
  struct PlanCtx {
    flash_index* h;
    QueryArgs a;
    void* scratch;
    uint64_t launches;
  } ctx{h, query_args(h, addrs, n_rows, k, nullptr, 1, 0, out_ids, out_counts, h->cur), h->qscratch.p, 0};
  // the ids about to be inserted are 0..n_rows-1 (a fresh handle): the plan's routing between
  // the bitmap and sort kernels must see the same max_id as the query launch after the build
  ctx.a.max_id = (uint32_t)(n_rows - 1);
  auto plan = [](void* c, cudaStream_t side) {
    PlanCtx* p = static_cast<PlanCtx*>(c);
    // a fresh handle builds into goff[cur]; allocated by now
    p->a.goff = p->h->goff[p->h->cur].as<uint64_t>();
    p->launches += launch_query_plan(p->a, p->scratch, side);
  };
  TRY(do_insert_addrs(h, addrs, n_rows, 0, s, 0, UINT32_MAX, false, false, plan, &ctx));
  h->launches += ctx.launches;
  return do_query_addrs(h, addrs, n_rows, k, nullptr, 1, 0, out_ids, out_counts, s, false, true);
}

flash_status flash_knn_graph_host(flash_index* h, const int64_t* row_ptr, const uint32_t* col_idx,
                                  uint64_t n_rows, uint32_t k, uint32_t* out_ids, uint32_t* out_counts,
                                  void* stream) {
  if (!h) return fail(FLASH_EINVAL, "handle is NULL");
  if (h->have_tables || h->n_inserted) return fail(FLASH_ESTATE, "flash_knn_graph_host needs a fresh handle");
  TRY(check_query_shape(h, k));
  if (n_rows == 0 && !h->dist) return FLASH_OK;
  if (n_rows >= 0xFFFFFFFFull) return fail(FLASH_EINVAL, "n_rows must be < 2^32-1");
  if (!row_ptr || (n_rows && (!col_idx || !out_ids || !out_counts))) return fail(FLASH_EINVAL, "NULL buffer");
  cudaStream_t s = (cudaStream_t)stream;
  if (h->dist) return dist_knn_graph_host(h, row_ptr, col_idx, n_rows, k, out_ids, out_counts, s);
  TRY(enter(h, s));
  const int64_t nnz_begin = row_ptr[0], nnz_end = row_ptr[n_rows];
  if (nnz_end < nnz_begin) return fail(FLASH_EINVAL, "row_ptr must be non-decreasing");
  const uint64_t nnz = (uint64_t)(nnz_end - nnz_begin);
  TRY(ensure(h->h_rp, sizeof(int64_t) * (n_rows + 1)));
  TRY(ensure(h->h_col, sizeof(uint32_t) * nnz));
  TRY(ensure(h->addrs, sizeof(uint32_t) * n_rows * h->L));
  TRY(ensure(h->h_ids, sizeof(uint32_t) * n_rows * k));
  TRY(ensure(h->h_cnt, sizeof(uint32_t) * n_rows * k));
  if (!h->copy_stream) CUDA_TRY(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
  int64_t* d_rp = h->h_rp.as<int64_t>();
  uint32_t* d_col = h->h_col.as<uint32_t>();
  uint32_t* d_addrs = h->addrs.as<uint32_t>();
  uint32_t* d_ids = h->h_ids.as<uint32_t>();
  uint32_t* d_cnt = h->h_cnt.as<uint32_t>();
  const uint32_t* d_col_abs = d_col - nnz_begin;  // absolute CSR offsets index this
  cudaStream_t cs = h->copy_stream;
  {
    Phase ph(h, 3, s);
    CUDA_TRY(cudaMemcpyAsync(d_rp, row_ptr, sizeof(int64_t) * (n_rows + 1), cudaMemcpyHostToDevice, s));
  }
  // chunked H2D of col_idx on the copy stream; chunk i is hashed while chunk i+1 copies
  const uint64_t chunk_bytes = 256ull << 20;
  size_t ev_used = 0;
  auto next_event = [&](cudaEvent_t* ev) -> flash_status {
    if (ev_used == h->copy_events.size()) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      h->copy_events.push_back(e);
    }
    *ev = h->copy_events[ev_used++];
    return FLASH_OK;
  };
  cudaEvent_t ready;
  TRY(next_event(&ready));
  CUDA_TRY(cudaEventRecord(ready, s));  // previous users of the staging buffers are done
  CUDA_TRY(cudaStreamWaitEvent(cs, ready, 0));
  uint64_t r0 = 0;
  while (r0 < n_rows) {
    uint64_t lo = r0 + 1, hi = n_rows;
    while (lo < hi) {
      const uint64_t mid = lo + (hi - lo + 1) / 2;
      if ((uint64_t)(row_ptr[mid] - row_ptr[r0]) * 4 <= chunk_bytes) lo = mid; else hi = mid - 1;
    }
    const uint64_t r1 = lo;
    const uint64_t e0 = (uint64_t)(row_ptr[r0] - nnz_begin), e1 = (uint64_t)(row_ptr[r1] - nnz_begin);
    cudaEvent_t ev;
    TRY(next_event(&ev));
    {
      Phase ph(h, 3, cs);
      if (e1 > e0)
        CUDA_TRY(cudaMemcpyAsync(d_col + e0, col_idx + nnz_begin + e0, sizeof(uint32_t) * (e1 - e0),
                                 cudaMemcpyHostToDevice, cs));
    }
    CUDA_TRY(cudaEventRecord(ev, cs));
    CUDA_TRY(cudaStreamWaitEvent(s, ev, 0));
    TRY(do_hash(h, d_rp + r0, d_col_abs, r1 - r0, nullptr, addr_out(d_addrs + r0 * h->L), s));
    r0 = r1;
  }
  TRY(do_insert_addrs(h, d_addrs, n_rows, 0, s));
  if (h->shared)
    TRY(do_query_addrs(h, h->raddr.as<uint32_t>(), n_rows, k, nullptr, 1, 0, d_ids, d_cnt, s, true));
  else
    TRY(do_query_addrs(h, d_addrs, n_rows, k, nullptr, 1, 0, d_ids, d_cnt, s));
  {
    Phase ph(h, 3, s);
    CUDA_TRY(cudaMemcpyAsync(out_ids, d_ids, sizeof(uint32_t) * n_rows * k, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(out_counts, d_cnt, sizeof(uint32_t) * n_rows * k, cudaMemcpyDeviceToHost, s));
  }
  CUDA_TRY(cudaStreamSynchronize(s));
  return FLASH_OK;
}

flash_status flash_hash_blocked(const flash_index* h, const int64_t* row_ptr, const uint32_t* col_idx,
                                uint64_t n_rows, uint32_t world, uint32_t* addrs, void* stream) {
  if (!h) return fail(FLASH_EINVAL, "handle is NULL");
  if (world < 1 || world > 65536) return fail(FLASH_EINVAL, "world=%u outside [1, 65536]", world);
  if (n_rows == 0) return FLASH_OK;
  REQUIRE_DEV(row_ptr);
  REQUIRE_DEV(col_idx);
  REQUIRE_DEV(addrs);
  cudaStream_t s = (cudaStream_t)stream;
  TRY(enter(h, s));
  return do_hash(h, row_ptr, col_idx, n_rows, nullptr, addr_out(addrs, world), s);
}

flash_status flash_insert_addrs_cols(flash_index* h, const uint32_t* addrs, uint64_t n_rows, uint32_t id_base,
                                     uint32_t t_begin, uint32_t t_end, void* stream) {
  if (!h) return fail(FLASH_EINVAL, "handle is NULL");
  if (h->dist) return fail(FLASH_ESTATE, "flash_insert_addrs_cols: not a call of a multi-GPU handle");
  if (h->shared) return fail(FLASH_EINVAL, "table windows are undefined when tables share reservoirs (R#23)");
  if (t_begin >= t_end || t_end > h->L)
    return fail(FLASH_EINVAL, "table window [%u, %u) must be non-empty and inside [0, %u)", t_begin, t_end, h->L);
  if (n_rows == 0) return FLASH_OK;
  REQUIRE_DEV(addrs);
  if ((uint64_t)id_base + n_rows - 1 >= 0xFFFFFFFFull)
    return fail(FLASH_EINVAL, "ids id_base..id_base+n_rows-1 must stay below 0xFFFFFFFF");
  cudaStream_t s = (cudaStream_t)stream;
  TRY(enter(h, s));
  return do_insert_addrs(h, addrs, n_rows, id_base, s, t_begin, t_end, true);
}

flash_status flash_window_sizes(const flash_index* hc, const uint32_t* addrs, uint64_t n_q, uint32_t t_begin,
                                uint32_t t_end, uint32_t* sizes, uint64_t* offsets, void* stream) {
  if (!hc) return fail(FLASH_EINVAL, "handle is NULL");
  flash_index* h = const_cast<flash_index*>(hc);
  if (h->dist) return fail(FLASH_ESTATE, "flash_window_sizes: not a call of a multi-GPU handle");
  if (h->shared) return fail(FLASH_EINVAL, "table windows are undefined when tables share reservoirs (R#23)");
  if (t_begin > t_end || t_end > h->L)
    return fail(FLASH_EINVAL, "table window [%u, %u) outside [0, %u)", t_begin, t_end, h->L);
  REQUIRE_DEV(offsets);
  if (n_q) {
    REQUIRE_DEV(sizes);
    if (t_end > t_begin) REQUIRE_DEV(addrs);
  }
  cudaStream_t s = (cudaStream_t)stream;
  TRY(enter(h, s));
  if (!h->have_tables || t_end == t_begin || n_q == 0) {
    if (n_q) CUDA_TRY(cudaMemsetAsync(sizes, 0, sizeof(uint32_t) * n_q, s));
    CUDA_TRY(cudaMemsetAsync(offsets, 0, sizeof(uint64_t) * (n_q + 1), s));
    return FLASH_OK;
  }
  TRY(ensure(h->xscan_tmp, scan_u32_to_u64_tmp_bytes(n_q)));
  Phase ph(h, 2, s);
  h->launches += launch_window_sizes(addrs, n_q, t_begin, t_end, h->range, h->goff[h->cur].as<uint64_t>(), sizes,
                                     offsets, h->xscan_tmp.p, h->xscan_tmp.cap, h->err, s);
  CUDA_TRY(cudaGetLastError());
  return FLASH_OK;
}

flash_status flash_window_gather(const flash_index* hc, const uint32_t* addrs, uint64_t n_q, uint32_t t_begin,
                                 uint32_t t_end, const uint64_t* offsets, uint32_t* out_ids, void* stream) {
  if (!hc) return fail(FLASH_EINVAL, "handle is NULL");
  flash_index* h = const_cast<flash_index*>(hc);
  if (h->dist) return fail(FLASH_ESTATE, "flash_window_gather: not a call of a multi-GPU handle");
  if (h->shared) return fail(FLASH_EINVAL, "table windows are undefined when tables share reservoirs (R#23)");
  if (t_begin > t_end || t_end > h->L)
    return fail(FLASH_EINVAL, "table window [%u, %u) outside [0, %u)", t_begin, t_end, h->L);
  if (n_q == 0 || t_end == t_begin || !h->have_tables) return FLASH_OK;
  REQUIRE_DEV(addrs);
  REQUIRE_DEV(offsets);
  REQUIRE_DEV(out_ids);
  cudaStream_t s = (cudaStream_t)stream;
  TRY(enter(h, s));
  Phase ph(h, 2, s);
  h->launches += launch_window_gather(addrs, n_q, t_begin, t_end, h->range, h->goff[h->cur].as<uint64_t>(),
                                      h->ids[h->cur].as<uint32_t>(), offsets, out_ids, s);
  CUDA_TRY(cudaGetLastError());
  return FLASH_OK;
}

flash_status flash_count_topk(const flash_index* hc, const uint32_t* cand, const uint32_t* seg_sizes,
                              uint32_t n_seg, uint64_t n_q, uint32_t k, const uint32_t* exclude, uint32_t max_id,
                              uint32_t* out_ids, uint32_t* out_counts, void* stream) {
  if (!hc) return fail(FLASH_EINVAL, "handle is NULL");
  flash_index* h = const_cast<flash_index*>(hc);
  if (h->dist) return fail(FLASH_ESTATE, "flash_count_topk: not a call of a multi-GPU handle");
  TRY(check_query_shape(h, k));
  if (n_seg < 1 || n_seg > 4096) return fail(FLASH_EINVAL, "n_seg=%u outside [1, 4096]", n_seg);
  if (n_q >= 0x80000000ull) return fail(FLASH_EINVAL, "n_q must be < 2^31");
  if (n_q == 0) return FLASH_OK;
  REQUIRE_DEV(seg_sizes);
  REQUIRE_DEV(out_ids);
  REQUIRE_DEV(out_counts);
  if (exclude) REQUIRE_DEV(exclude);
  if (cand && !device_accessible(cand)) return fail(FLASH_EINVAL, "cand is not a device pointer");
  cudaStream_t s = (cudaStream_t)stream;
  TRY(enter(h, s));
  const uint64_t nsq = (uint64_t)n_seg * n_q;
  TRY(ensure(h->seg_off, sizeof(uint64_t) * (nsq + 1)));
  TRY(ensure(h->xscan_tmp, scan_u32_to_u64_tmp_bytes(nsq)));
  TRY(ensure(h->qscratch, query_scratch_bytes(n_q)));
  Phase ph(h, 2, s);
  launch_scan_sizes(seg_sizes, nsq, h->seg_off.as<uint64_t>(), h->xscan_tmp.p, h->xscan_tmp.cap, s);
  QueryArgs a;
  memset(&a, 0, sizeof a);
  a.addrs = nullptr;
  a.nq = n_q;
  a.goff = h->seg_off.as<uint64_t>();
  // cand == NULL: every segment must be empty (a non-empty one would read the 16 zero bytes)
  a.ids = cand ? cand : h->zero.as<uint32_t>();
  a.L = n_seg;
  a.range = (uint32_t)n_q;
  a.k = k;
  a.cmax = h->L;
  a.direct = 1;
  a.exclude = exclude;
  a.exclude_self = 0;
  a.out_ids = out_ids;
  a.out_counts = out_counts;
  a.err = h->err;
  a.seg_len = nullptr;
  a.mmax = cand ? (uint64_t)h->L * h->R : 0;  // NULL cand: any candidate is an error (pads)
  a.max_id = max_id;
  return run_query(h, a, s);
}

flash_status flash_clear(flash_index* h, void* stream) {
  if (!h) return fail(FLASH_EINVAL, "handle is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  if (h->dist) return dist_clear(h, s);
  TRY(enter(h, s));
  CUDA_TRY(cudaMemsetAsync(h->arrivals, 0, sizeof(uint32_t) * nbuckets(h), s));
  h->have_tables = false;
  h->kept_ub = 0;
  h->n_inserted = 0;
  h->max_id = 0;
  return FLASH_OK;
}

flash_status flash_get_table(const flash_index* hc, uint32_t t, const uint32_t** off, const uint32_t** ids,
                             const uint32_t** arrivals, uint64_t* n_ids) {
  if (!hc) return fail(FLASH_EINVAL, "handle is NULL");
  flash_index* h = const_cast<flash_index*>(hc);
  if (t >= h->L) return fail(FLASH_EINVAL, "table %u >= L=%u", t, h->L);
  if (h->dist) return dist_get_table(h, t, off, ids, arrivals, n_ids);
  if (h->shared) return fail(FLASH_ESTATE, "tables share reservoirs: use flash_table_arrays");
  if (!h->have_tables) return fail(FLASH_ESTATE, "nothing inserted yet");
  CUDA_TRY(cudaSetDevice(h->device));
  if (h->have_last) CUDA_TRY(cudaStreamSynchronize(h->last_stream));
  TRY(ensure(h->off_tmp, sizeof(uint32_t) * ((size_t)h->range + 1)));
  const uint64_t* goff = h->goff[h->cur].as<uint64_t>();
  uint64_t b[2];
  CUDA_TRY(cudaMemcpy(&b[0], goff + (uint64_t)t * h->range, sizeof(uint64_t), cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(&b[1], goff + (uint64_t)(t + 1) * h->range, sizeof(uint64_t), cudaMemcpyDeviceToHost));
  const unsigned blocks = (h->range + 256) / 256 < 4096 ? (h->range + 256) / 256 : 4096;
  k_table_off<<<blocks, 256>>>(goff, t, h->range, h->off_tmp.as<uint32_t>());
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaDeviceSynchronize());
  h->launches++;
  if (off) *off = h->off_tmp.as<uint32_t>();
  if (ids) *ids = h->ids[h->cur].as<uint32_t>() + b[0];
  if (arrivals) *arrivals = h->arrivals + (uint64_t)t * h->range;
  if (n_ids) *n_ids = b[1] - b[0];
  return FLASH_OK;
}

flash_status flash_check(const flash_index* h, uint64_t* n_errors) {
  if (!h) return fail(FLASH_EINVAL, "handle is NULL");
  if (h->dist) return dist_check(h, n_errors);
  CUDA_TRY(cudaSetDevice(h->device));
  if (h->have_last) CUDA_TRY(cudaStreamSynchronize(h->last_stream));
  unsigned long long e = 0;
  CUDA_TRY(cudaMemcpy(&e, h->err, sizeof e, cudaMemcpyDeviceToHost));
  if (n_errors) *n_errors = e;
  return FLASH_OK;
}

flash_status flash_set_profiling(flash_index* h, int enable) {
  if (!h) return fail(FLASH_EINVAL, "handle is NULL");
  h->profiling = enable;
  return FLASH_OK;
}

flash_status flash_phase_ms(const flash_index* hc, double ms_out[4], uint64_t calls_out[4]) {
  if (!hc) return fail(FLASH_EINVAL, "handle is NULL");
  flash_index* h = const_cast<flash_index*>(hc);
  for (auto& p : h->pending) {
    CUDA_TRY(cudaEventSynchronize(p.b));
    float ms = 0;
    CUDA_TRY(cudaEventElapsedTime(&ms, p.a, p.b));
    h->phase_ms[p.phase] += ms;
    h->phase_calls[p.phase] += 1;
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  h->pending.clear();
  for (int i = 0; i < 4; ++i) {
    if (ms_out) ms_out[i] = h->phase_ms[i];
    if (calls_out) calls_out[i] = h->phase_calls[i];
  }
  return FLASH_OK;
}

uint64_t flash_launch_count(const flash_index* h) { return h ? h->launches : 0; }

flash_status flash_reset_counters(flash_index* h) {
  if (!h) return fail(FLASH_EINVAL, "handle is NULL");
  TRY(flash_phase_ms(h, nullptr, nullptr));
  for (int i = 0; i < 4; ++i) {
    h->phase_ms[i] = 0;
    h->phase_calls[i] = 0;
  }
  h->launches = 0;
  return FLASH_OK;
}

}  // extern "C"
