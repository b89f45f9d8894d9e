// dist.cu — the multi-GPU handle (flash_create_dist / flash_create_dist_local): FLASH's
// k-NN graph, insert and query with the L tables partitioned over the GPUs of one node and
// each query's candidates counted on the GPU that owns the query (north_star (d); SURVEY
// §8(e); queries are data-parallel, §3.4).
//
// Rank g owns the table window [t0(g), t1(g)) = [floor(gL/G), floor((g+1)L/G)) (R#22) and
// holds it as an ordinary index of W = t1 - t0 tables whose priorities are keyed by the
// global table index (HashKeys::tbase), so a window equals those tables of a 1-GPU build.
// A collective call (every rank calls it with its own contiguous row shard):
//   C0   all-gather of the shard sizes (host: sizes the exchange and fixes the global row ids)
//   H+X1 the DOPH kernel writes each row's addresses straight into the table owners' window-
//        address buffers [N][W_g] (P2P stores over NVLink: the exchange is fused into the hash)
//   B    each rank builds its window over all N rows (B1-B2; bottom-R is per bucket)
//   Q1+X2 per round of <= B queries of every owner: each rank gathers the query's window
//        buckets and stores them straight into the owner's receive region for this sender
//        (regions sized by the worst case W_s*R per query, so no size exchange is needed;
//        the sizes go along, also as peer stores), rounds alternate two receive buffers
//   Q2-Q3 the owner counts over its G segments per query and selects the top-k (the query
//        kernels in direct-segment mode).
// The candidate multiset of a query is exactly the union of its L buckets and the count /
// top-k rule does not depend on candidate order, so the output equals the 1-GPU result
// byte for byte at every G.  Stream-ordered barriers separate the peer stores from their
// readers; the host synchronizes only on C0 (and when buffers grow).
//
// Transports: NCCL (one process per GPU; NCCL is loaded with dlopen — the torch-bundled
// libnccl.so.2 when torch is already loaded — and provides the bootstrap, C0 and the stream
// barriers; the receive buffers are mapped into the peers with CUDA IPC) or a local group
// (virtual ranks in one process, one host thread each, on one or several devices: host
// barriers plus CUDA events; peers' buffers are plain device pointers).
#include <cub/block/block_scan.cuh>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <type_traits>
#include <vector>

#include "dist.cuh"
#include "flash.h"
#include "flash_internal.cuh"
#include "handle.cuh"

using namespace flash;
using namespace flash::api;

namespace flash {
namespace api {
namespace {

// ---------------------------------------------------------------------------
// NCCL, resolved at run time
// ---------------------------------------------------------------------------
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*CommAbort)(ncclComm_t);
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    void* lib = nullptr;
    for (const char* n : names)
      if ((lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!lib) {
      api.why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    bool all = true;
    auto sym = [&](auto& f, const char* n) {
      f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(lib, n));
      if (!f) {
        all = false;
        api.why = std::string("libnccl lacks ") + n;
      }
    };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommSplit, "ncclCommSplit");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.CommAbort, "ncclCommAbort");
    sym(api.CommGetAsyncError, "ncclCommGetAsyncError");
    sym(api.AllGather, "ncclAllGather");
    sym(api.AllReduce, "ncclAllReduce");
    sym(api.GetErrorString, "ncclGetErrorString");
    api.ok = all;
  });
  return api;
}

#define NCCL_TRY(expr)                                                                                  \
  do {                                                                                                  \
    ncclResult_t r_ = (expr);                                                                           \
    if (r_ != ncclSuccess)                                                                              \
      return fail(FLASH_ENCCL, "%s: %s (%s:%d)", #expr, nccl().GetErrorString(r_), __FILE__, __LINE__); \
  } while (0)

// ---------------------------------------------------------------------------
// Transports
// ---------------------------------------------------------------------------
struct Transport {
  int rank = 0, world = 1;
  virtual ~Transport() {}
  // host all-gather of n uint64 per rank (all: [world][n]); synchronizes the host with the
  // other ranks, NOT the caller's stream
  virtual flash_status allgather(const uint64_t* mine, uint64_t* all, int n) = 0;
  // stream-ordered barrier on s: every rank's work enqueued before it (including stores into
  // other ranks' buffers) completes before any rank's work enqueued after it
  virtual flash_status barrier(cudaStream_t s) = 0;
  // collective: out[g] = rank g's buffer `mine` (a cudaMalloc base) as seen by this rank
  virtual flash_status map(void* mine, std::vector<void*>& out) = 0;
  virtual void unmap(std::vector<void*>& ptrs) = 0;
  virtual flash_status check() { return FLASH_OK; }
};

struct NcclTransport : Transport {
  ncclComm_t comm = nullptr;  // barriers, on the caller's stream
  ncclComm_t ctl = nullptr;   // C0 and the IPC handle exchange, on a private stream
  cudaStream_t cs = nullptr;
  int device = 0;
  void* dbuf = nullptr;       // device staging
  size_t dcap = 0;
  int* dflag = nullptr;

  ~NcclTransport() override {
    if (comm) nccl().CommDestroy(comm);
    if (ctl) nccl().CommDestroy(ctl);
    if (cs) cudaStreamDestroy(cs);
    if (dbuf) cudaFree(dbuf);
    if (dflag) cudaFree(dflag);
  }
  flash_status stage(size_t bytes) {
    if (dcap >= bytes) return FLASH_OK;
    if (dbuf) CUDA_TRY(cudaFree(dbuf));
    dbuf = nullptr;
    CUDA_TRY(cudaMalloc(&dbuf, bytes));
    dcap = bytes;
    return FLASH_OK;
  }
  flash_status gather_bytes(const void* mine, void* all, size_t bytes) {
    TRY(stage(bytes * (world + 1)));
    uint8_t* d = static_cast<uint8_t*>(dbuf);
    CUDA_TRY(cudaMemcpyAsync(d, mine, bytes, cudaMemcpyHostToDevice, cs));
    NCCL_TRY(nccl().AllGather(d, d + bytes, bytes, ncclUint8, ctl, cs));
    CUDA_TRY(cudaMemcpyAsync(all, d + bytes, bytes * world, cudaMemcpyDeviceToHost, cs));
    CUDA_TRY(cudaStreamSynchronize(cs));
    return FLASH_OK;
  }
  flash_status allgather(const uint64_t* mine, uint64_t* all, int n) override {
    return gather_bytes(mine, all, sizeof(uint64_t) * n);
  }
  flash_status barrier(cudaStream_t s) override {
    if (world == 1) return FLASH_OK;
    NCCL_TRY(nccl().AllReduce(dflag, dflag, 1, ncclInt32, ncclSum, comm, s));
    return FLASH_OK;
  }
  flash_status map(void* mine, std::vector<void*>& out) override {
    out.assign(world, nullptr);
    out[rank] = mine;
    if (world == 1) return FLASH_OK;
    cudaIpcMemHandle_t hm;
    CUDA_TRY(cudaIpcGetMemHandle(&hm, mine));
    std::vector<cudaIpcMemHandle_t> all(world);
    TRY(gather_bytes(&hm, all.data(), sizeof hm));
    for (int g = 0; g < world; ++g)
      if (g != rank) CUDA_TRY(cudaIpcOpenMemHandle(&out[g], all[g], cudaIpcMemLazyEnablePeerAccess));
    return FLASH_OK;
  }
  void unmap(std::vector<void*>& ptrs) override {
    for (int g = 0; g < (int)ptrs.size(); ++g)
      if (g != rank && ptrs[g]) cudaIpcCloseMemHandle(ptrs[g]);
    ptrs.clear();
  }
  flash_status check() override {
    ncclResult_t r = ncclSuccess;
    NCCL_TRY(nccl().CommGetAsyncError(comm, &r));
    if (r != ncclSuccess && r != ncclInProgress)
      return fail(FLASH_ENCCL, "NCCL asynchronous error: %s", nccl().GetErrorString(r));
    return FLASH_OK;
  }
};

// Virtual ranks of one process (one host thread per rank).
struct LocalGroup {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  int refs = 0;
  std::vector<uint64_t> words;   // all-gather staging
  std::vector<void*> ptrs;       // map staging
  std::vector<cudaEvent_t> ev;   // [world][2] barrier events
  explicit LocalGroup(int w) : world(w), ptrs(w, nullptr), ev(2 * w, nullptr) {}
  ~LocalGroup() {
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
  }
  void host_barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct LocalTransport : Transport {
  std::shared_ptr<LocalGroup> grp;
  int par = 0;
  flash_status allgather(const uint64_t* mine, uint64_t* all, int n) override {
    {
      std::lock_guard<std::mutex> lk(grp->mu);
      if (grp->words.size() < (size_t)world * n) grp->words.resize((size_t)world * n);
    }
    grp->host_barrier();  // everyone sized the staging before anyone writes it
    memcpy(&grp->words[(size_t)rank * n], mine, sizeof(uint64_t) * n);
    grp->host_barrier();
    memcpy(all, grp->words.data(), sizeof(uint64_t) * n * world);
    grp->host_barrier();  // everyone read before the next all-gather writes
    return FLASH_OK;
  }
  flash_status barrier(cudaStream_t s) override {
    if (world == 1) return FLASH_OK;
    cudaEvent_t mine = grp->ev[2 * rank + par];
    CUDA_TRY(cudaEventRecord(mine, s));
    grp->host_barrier();
    for (int g = 0; g < world; ++g)
      if (g != rank) CUDA_TRY(cudaStreamWaitEvent(s, grp->ev[2 * g + par], 0));
    par ^= 1;
    return FLASH_OK;
  }
  flash_status map(void* mine, std::vector<void*>& out) override {
    grp->ptrs[rank] = mine;
    grp->host_barrier();
    out = grp->ptrs;
    grp->host_barrier();
    return FLASH_OK;
  }
  void unmap(std::vector<void*>& ptrs) override { ptrs.clear(); }
};

// Worst-case receive bytes of one candidate buffer (two are kept): 4 GiB, i.e. B = 4 GiB /
// (L*R*4) queries per round; FLASH_DIST_CAND_BYTES overrides it (tests force many rounds).
uint64_t cand_buffer_bytes() {
  const char* e = getenv("FLASH_DIST_CAND_BYTES");
  return e ? strtoull(e, nullptr, 10) : (4ull << 30);
}

}  // namespace

struct DistState {
  int rank = 0, world = 1;
  std::unique_ptr<Transport> tr;
  flash_index* win = nullptr;  // this rank's table window as W local tables (null when W == 0)
  uint32_t t0 = 0, t1 = 0;
  // receive buffers (peers store into them)
  DevBuf x1;                   // [rows][W]: window addresses of every row of the call
  DevBuf cand[2], segs[2];     // [B*L*R] candidate regions; [world][B] segment sizes
  std::vector<void*> px1, pcand[2], pseg[2];
  DevBuf dpeer;                // device copy: [world] x1, [2][world] cand, [2][world] segs
  uint64_t rows_cap = 0, batch = 0, cand_cap = 0;
  bool mapped = false;
  // local scratch
  DevBuf sizes, offs, goffq, dbounds, scan_tmp;
  uint64_t max_id = 0;         // largest id inserted on any rank
  bool have_any = false;       // some rank has inserted something
  std::vector<uint64_t> bounds;  // global row bounds of the last call [world+1]
};

namespace {

uint32_t win_t0(uint32_t L, int world, int g) { return (uint32_t)(((uint64_t)L * g) / world); }

// ---------------------------------------------------------------------------
// Kernels
// ---------------------------------------------------------------------------

// Q1 + X2 fused, sender side: for every query of this round (owner g's local rows
// [round*B, round*B + B)), copy its window buckets into owner g's receive region for this
// sender, at the query's offset within the owner's batch, and store its segment size.
// One warp per query; bucket extents one per lane, copies coalesced.
__global__ void k_dist_gather(const uint32_t* __restrict__ x1, uint32_t W, uint32_t range,
                              const uint64_t* __restrict__ goff, const uint32_t* __restrict__ ids,
                              const uint32_t* __restrict__ sizes, const uint64_t* __restrict__ offs,
                              const uint64_t* __restrict__ bounds, int world, int me, uint64_t round,
                              uint64_t B, uint64_t region, uint32_t* const* __restrict__ pcand,
                              uint32_t* const* __restrict__ pseg) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nv = (uint64_t)world * B;
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t v = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); v < nv; v += nw) {
    const int g = (int)(v / B);
    const uint64_t j = v - (uint64_t)g * B;
    const uint64_t lr = round * B + j;
    if (lr >= bounds[g + 1] - bounds[g]) continue;
    const uint64_t q = bounds[g] + lr;
    const uint32_t sz = W ? sizes[q] : 0u;
    const uint64_t rel = offs[q] - offs[bounds[g] + round * B];  // within this sender's region
    if (lane == 0) {
      pseg[g][(uint64_t)me * B + j] = sz;                        // segment size
      pseg[g][nv + (uint64_t)me * B + j] = (uint32_t)rel;        // and start (< 2^32: <= 4 GiB)
    }
    if (!sz) continue;
    uint32_t* dst = pcand[g] + region + rel;
    // 32 buckets at a time: lane b holds bucket b's extent and its exclusive position; each
    // 32 consecutive output positions find their bucket by a binary search over the lanes
    for (uint32_t j0 = 0; j0 < W; j0 += 32) {
      uint64_t st = 0;
      uint32_t bsz = 0;
      if (j0 + lane < W) {
        const uint32_t a = x1[q * W + j0 + lane];
        if (a < range) {
          const uint64_t i = (uint64_t)(j0 + lane) * range + a;
          st = goff[i];
          bsz = (uint32_t)(goff[i + 1] - st);
        }
      }
      uint32_t incl = bsz;
#pragma unroll
      for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
      }
      const uint32_t tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
      const uint64_t base = st - (incl - bsz);  // ids + base + p: position p's id, p in this bucket
      for (uint32_t p0 = 0; p0 < tot; p0 += 32) {
        const uint32_t p = p0 + lane;
        // the bucket of p: the first lane b with incl_b > p (never an empty bucket)
        uint32_t lo = 0;
#pragma unroll
        for (uint32_t step = 16; step; step >>= 1)
          if (__shfl_sync(0xFFFFFFFFu, incl, lo + step - 1) <= p) lo += step;
        const uint64_t bb = __shfl_sync(0xFFFFFFFFu, base, lo);
        if (p < tot) dst[p] = __ldg(ids + bb + p);
      }
      dst += tot;
    }
  }
}

// Owner side: segment (s, j) of this round starts at region(s) + the start the sender stored
// beside its size (segs[nv + s*B + j]).
__global__ void k_dist_seg_offsets(const uint32_t* __restrict__ segs, uint64_t B, uint64_t nb, int world,
                                   const uint64_t* __restrict__ region, uint64_t* __restrict__ goffq) {
  const uint64_t nv = (uint64_t)world * B;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = v / B, j = v - s * B;
    if (j < nb) goffq[v] = region[s] + segs[nv + v];
  }
}

// ---------------------------------------------------------------------------
// Host orchestration
// ---------------------------------------------------------------------------
DistState* D(const flash_index* h) { return h->dist; }

// profiling / launch counters of the window handle go to the outer handle
void absorb(flash_index* h, flash_index* w) {
  if (!w) return;
  h->launches += w->launches;
  w->launches = 0;
  for (auto& p : w->pending) h->pending.push_back(p);
  w->pending.clear();
}

flash_status unmap_all(DistState* d) {
  if (!d->mapped) return FLASH_OK;
  d->tr->unmap(d->px1);
  for (int p = 0; p < 2; ++p) {
    d->tr->unmap(d->pcand[p]);
    d->tr->unmap(d->pseg[p]);
  }
  d->mapped = false;
  return FLASH_OK;
}

// Size the receive buffers for a call over N global rows (largest shard maxn) and map them
// into every rank.  Every input is global, so every rank takes the same decisions (growth
// and remapping are collective).
flash_status prepare(flash_index* h, uint64_t N, uint64_t maxn, cudaStream_t s) {
  DistState* d = D(h);
  const uint64_t wmax = (h->L + d->world - 1) / d->world;
  const uint64_t per_q = (uint64_t)h->L * h->R * sizeof(uint32_t);
  uint64_t B = cand_buffer_bytes() / (per_q ? per_q : 1);
  if (B < 1) B = 1;
  if (B > maxn) B = maxn ? maxn : 1;
  const bool grow_rows = N * wmax * 4 > d->x1.cap;
  const bool grow_b = B > d->batch;  // the segment-size rows are B apart: B changes only upward
  if (!grow_b) B = d->batch;
  const uint64_t cand_need = B * h->L * h->R * 4;
  const bool grow_cand = cand_need > d->cand[0].cap;
  if (d->mapped && !grow_rows && !grow_b && !grow_cand) return FLASH_OK;
  // every rank is done with the old buffers before anyone releases them
  TRY(d->tr->barrier(s));
  CUDA_TRY(cudaStreamSynchronize(s));
  TRY(unmap_all(d));
  uint64_t dummy = 0, all[4096];
  TRY(d->tr->allgather(&dummy, all, 1));  // (host barrier: every rank has unmapped)
  if (grow_rows) TRY(ensure(d->x1, (N + N / 8 + 1) * wmax * 4));
  d->batch = B;
  for (int p = 0; p < 2; ++p) {
    TRY(ensure(d->cand[p], cand_need));
    TRY(ensure(d->segs[p], (uint64_t)d->world * B * 8));  // sizes, then starts
  }
  TRY(d->tr->map(d->x1.p, d->px1));
  for (int p = 0; p < 2; ++p) {
    TRY(d->tr->map(d->cand[p].p, d->pcand[p]));
    TRY(d->tr->map(d->segs[p].p, d->pseg[p]));
  }
  d->mapped = true;
  std::vector<void*> tab;
  tab.insert(tab.end(), d->px1.begin(), d->px1.end());
  for (int p = 0; p < 2; ++p) tab.insert(tab.end(), d->pcand[p].begin(), d->pcand[p].end());
  for (int p = 0; p < 2; ++p) tab.insert(tab.end(), d->pseg[p].begin(), d->pseg[p].end());
  TRY(ensure(d->dpeer, tab.size() * sizeof(void*)));
  CUDA_TRY(cudaMemcpy(d->dpeer.p, tab.data(), tab.size() * sizeof(void*), cudaMemcpyHostToDevice));
  return FLASH_OK;
}

uint32_t* const* peer_x1(DistState* d) { return d->dpeer.as<uint32_t* const>(); }
uint32_t* const* peer_cand(DistState* d, int p) { return d->dpeer.as<uint32_t* const>() + d->world * (1 + p); }
uint32_t* const* peer_seg(DistState* d, int p) { return d->dpeer.as<uint32_t* const>() + d->world * (3 + p); }

// C0: every rank's (n, extra) pair; fills d->bounds.
flash_status exchange_shards(flash_index* h, uint64_t n, uint64_t extra, std::vector<uint64_t>& all) {
  DistState* d = D(h);
  TRY(d->tr->check());
  uint64_t mine[2] = {n, extra};
  all.assign(2 * (size_t)d->world, 0);
  TRY(d->tr->allgather(mine, all.data(), 2));
  d->bounds.assign(d->world + 1, 0);
  for (int g = 0; g < d->world; ++g) d->bounds[g + 1] = d->bounds[g] + all[2 * g];
  return FLASH_OK;
}

// H1-H3 of this rank's rows with the addresses stored into every owner's window buffer
// (X1), bracketed by barriers.
flash_status hash_exchange(flash_index* h, const int64_t* row_ptr, const uint32_t* col_idx, uint64_t n,
                           cudaStream_t s) {
  DistState* d = D(h);
  Phase ph(h, 0, s);
  TRY(d->tr->barrier(s));  // the owners are done reading their window buffers
  if (n) {
    AddrOut out;
    if (d->world == 1) {
      out = addr_out(d->x1.as<uint32_t>());
    } else {
      out.addrs = nullptr;
      out.peers = peer_x1(d);
      out.row0 = d->bounds[d->rank];
      out.world = (uint32_t)d->world;
    }
    TRY(do_hash(h, row_ptr, col_idx, n, nullptr, out, s));
  }
  TRY(d->tr->barrier(s));  // every row's addresses have landed
  return FLASH_OK;
}

// Q1-Q3 for the queries whose window addresses are in x1 (Q = bounds.back() global rows,
// this rank's are bounds[rank] ..): per round, gather + store to the owners, barrier, count.
flash_status query_rounds(flash_index* h, uint32_t k, const uint32_t* exclude, bool exclude_self,
                          uint32_t* out_ids, uint32_t* out_counts, cudaStream_t s) {
  DistState* d = D(h);
  Phase ph(h, 2, s);
  const uint64_t Q = d->bounds.back();
  const uint32_t W = d->t1 - d->t0;
  flash_index* w = d->win;
  const bool tables = w && w->have_tables;
  TRY(ensure(d->sizes, (Q + 1) * 4));
  TRY(ensure(d->offs, (Q + 1) * 8));
  TRY(ensure(d->dbounds, (d->world + 1) * 8 + (uint64_t)d->world * 8));
  TRY(ensure(d->goffq, (uint64_t)d->world * d->batch * 8));
  CUDA_TRY(cudaMemcpyAsync(d->dbounds.p, d->bounds.data(), (d->world + 1) * 8, cudaMemcpyHostToDevice, s));
  std::vector<uint64_t> region(d->world);
  for (int g = 0; g < d->world; ++g) region[g] = d->batch * h->R * win_t0(h->L, d->world, g);
  uint64_t* dregion = d->dbounds.as<uint64_t>() + d->world + 1;
  CUDA_TRY(cudaMemcpyAsync(dregion, region.data(), d->world * 8, cudaMemcpyHostToDevice, s));
  if (tables && Q) {
    TRY(ensure(d->scan_tmp, scan_u32_to_u64_tmp_bytes(Q)));
    h->launches += launch_window_sizes(d->x1.as<uint32_t>(), Q, 0, W, h->range, w->goff[w->cur].as<uint64_t>(),
                                       d->sizes.as<uint32_t>(), d->offs.as<uint64_t>(), d->scan_tmp.p,
                                       d->scan_tmp.cap, h->err, s);
  } else if (Q) {
    CUDA_TRY(cudaMemsetAsync(d->sizes.p, 0, Q * 4, s));
    CUDA_TRY(cudaMemsetAsync(d->offs.p, 0, (Q + 1) * 8, s));
  }
  uint64_t maxn = 0;
  for (int g = 0; g < d->world; ++g) maxn = std::max(maxn, d->bounds[g + 1] - d->bounds[g]);
  const uint64_t B = d->batch;
  const uint64_t rounds = (maxn + B - 1) / B;
  const uint64_t mine = d->bounds[d->rank + 1] - d->bounds[d->rank];
  TRY(ensure(h->qscratch, query_scratch_bytes(B)));
  for (uint64_t r = 0; r < rounds; ++r) {
    const int p = (int)(r & 1);
    const uint64_t nv = (uint64_t)d->world * B;
    const uint64_t want = (nv + 7) / 8;
    const unsigned blocks = (unsigned)std::min<uint64_t>(want, (uint64_t)device_sms() * 16);
    k_dist_gather<<<blocks, 256, 0, s>>>(d->x1.as<uint32_t>(), tables ? W : 0, h->range,
                                         tables ? w->goff[w->cur].as<uint64_t>() : nullptr,
                                         tables ? w->ids[w->cur].as<uint32_t>() : nullptr, d->sizes.as<uint32_t>(),
                                         d->offs.as<uint64_t>(), d->dbounds.as<uint64_t>(), d->world, d->rank, r, B,
                                         region[d->rank], peer_cand(d, p), peer_seg(d, p));
    h->launches++;
    CUDA_TRY(cudaGetLastError());
    TRY(d->tr->barrier(s));  // every sender's candidates for this round have landed
    const uint64_t lo = r * B;
    if (lo >= mine) continue;
    const uint64_t nb = std::min(B, mine - lo);
    const uint64_t sv = (uint64_t)d->world * B;
    k_dist_seg_offsets<<<(unsigned)std::min<uint64_t>((sv + 255) / 256, (uint64_t)device_sms() * 8), 256, 0, s>>>(
        d->segs[p].as<uint32_t>(), B, nb, d->world, dregion, d->goffq.as<uint64_t>());
    h->launches++;
    QueryArgs a;
    memset(&a, 0, sizeof a);
    a.nq = nb;
    a.goff = d->goffq.as<uint64_t>();
    a.seg_len = d->segs[p].as<uint32_t>();
    a.ids = d->cand[p].as<uint32_t>();
    a.L = (uint32_t)d->world;  // segments per query: one per sender
    a.range = (uint32_t)B;     // segment (s, j) at index s*B + j
    a.k = k;
    a.cmax = h->L;
    a.direct = 1;
    a.exclude = exclude ? exclude + lo : nullptr;
    a.exclude_self = exclude_self ? 1 : 0;
    a.self_base = (uint32_t)(d->bounds[d->rank] + lo);
    a.out_ids = out_ids + lo * k;
    a.out_counts = out_counts + lo * k;
    a.err = h->err;
    a.mmax = (uint64_t)h->L * h->R;
    a.max_id = (uint32_t)d->max_id;
    TRY(run_query(h, a, s));
  }
  return FLASH_OK;
}

flash_status check_ids(const std::vector<uint64_t>& all, int world) {
  for (int g = 0; g < world; ++g)
    if (all[2 * g] && all[2 * g + 1] + all[2 * g] - 1 >= 0xFFFFFFFFull)
      return fail(FLASH_EINVAL, "rank %d: ids id_base..id_base+n_rows-1 must stay below 0xFFFFFFFF", g);
  return FLASH_OK;
}

}  // namespace

flash_status dist_insert(flash_index* h, const int64_t* row_ptr, const uint32_t* col_idx, uint64_t n,
                         uint32_t id_base, cudaStream_t s) {
  DistState* d = D(h);
  TRY(enter(h, s));
  std::vector<uint64_t> all;
  TRY(exchange_shards(h, n, id_base, all));
  TRY(check_ids(all, d->world));
  const uint64_t N = d->bounds.back();
  if (N == 0) return FLASH_OK;
  uint64_t maxn = 0;
  for (int g = 0; g < d->world; ++g) maxn = std::max(maxn, all[2 * g]);
  TRY(prepare(h, N, maxn, s));
  TRY(hash_exchange(h, row_ptr, col_idx, n, s));
  if (d->win) {
    // ids of rank g's rows are id_base_g + r; consecutive ranks with contiguous ids build in one pass
    d->win->profiling = h->profiling;
    const uint32_t W = d->t1 - d->t0;
    int g = 0;
    while (g < d->world) {
      if (!all[2 * g]) {
        ++g;
        continue;
      }
      int e = g + 1;
      uint64_t cnt = all[2 * g];
      while (e < d->world && all[2 * e] && all[2 * e + 1] == all[2 * g + 1] + cnt) cnt += all[2 * e++];
      TRY(do_insert_addrs(d->win, d->x1.as<uint32_t>() + d->bounds[g] * W, cnt, (uint32_t)all[2 * g + 1], s));
      g = e;
    }
    absorb(h, d->win);
  }
  for (int g = 0; g < d->world; ++g)
    if (all[2 * g]) d->max_id = std::max(d->max_id, all[2 * g + 1] + all[2 * g] - 1);
  d->have_any = true;
  h->n_inserted += N;
  h->have_tables = true;
  return FLASH_OK;
}

flash_status dist_query_topk(flash_index* h, const int64_t* row_ptr, const uint32_t* col_idx, uint64_t n_q,
                             uint32_t k, const uint32_t* exclude, uint32_t* out_ids, uint32_t* out_counts,
                             cudaStream_t s) {
  DistState* d = D(h);
  TRY(enter(h, s));
  std::vector<uint64_t> all;
  TRY(exchange_shards(h, n_q, 0, all));
  const uint64_t Q = d->bounds.back();
  if (Q == 0) return FLASH_OK;
  if (!d->have_any) {  // nothing inserted on any rank (a global state): k pads, no exchange
    if (n_q) {
      CUDA_TRY(cudaMemsetAsync(out_ids, 0xFF, sizeof(uint32_t) * n_q * k, s));
      CUDA_TRY(cudaMemsetAsync(out_counts, 0, sizeof(uint32_t) * n_q * k, s));
    }
    return FLASH_OK;
  }
  uint64_t maxn = 0;
  for (int g = 0; g < d->world; ++g) maxn = std::max(maxn, all[2 * g]);
  TRY(prepare(h, Q, maxn, s));
  TRY(hash_exchange(h, row_ptr, col_idx, n_q, s));
  return query_rounds(h, k, exclude, false, out_ids, out_counts, s);
}

flash_status dist_knn_graph(flash_index* h, const int64_t* row_ptr, const uint32_t* col_idx, uint64_t n,
                            uint32_t k, uint32_t* out_ids, uint32_t* out_counts, cudaStream_t s) {
  DistState* d = D(h);
  TRY(enter(h, s));
  std::vector<uint64_t> all;
  TRY(exchange_shards(h, n, 0, all));
  const uint64_t N = d->bounds.back();
  if (N == 0) return FLASH_OK;
  if (N >= 0xFFFFFFFFull) return fail(FLASH_EINVAL, "the graph's %llu rows must be < 2^32-1", (unsigned long long)N);
  uint64_t maxn = 0;
  for (int g = 0; g < d->world; ++g) maxn = std::max(maxn, all[2 * g]);
  TRY(prepare(h, N, maxn, s));
  TRY(hash_exchange(h, row_ptr, col_idx, n, s));
  if (d->win) {  // B1-B2: this rank's window over all N rows (global ids 0..N-1)
    d->win->profiling = h->profiling;
    TRY(do_insert_addrs(d->win, d->x1.as<uint32_t>(), N, 0, s));
    absorb(h, d->win);
  }
  d->max_id = N - 1;
  d->have_any = true;
  h->n_inserted = N;
  h->have_tables = true;
  return query_rounds(h, k, nullptr, true, out_ids, out_counts, s);
}

flash_status dist_knn_graph_host(flash_index* h, const int64_t* row_ptr, const uint32_t* col_idx, uint64_t n,
                                 uint32_t k, uint32_t* out_ids, uint32_t* out_counts, cudaStream_t s) {
  TRY(enter(h, s));
  const int64_t e0 = n ? row_ptr[0] : 0, e1 = n ? row_ptr[n] : 0;
  if (e1 < e0) return fail(FLASH_EINVAL, "row_ptr must be non-decreasing");
  const uint64_t nnz = (uint64_t)(e1 - e0);
  TRY(ensure(h->h_rp, sizeof(int64_t) * (n + 1)));
  TRY(ensure(h->h_col, sizeof(uint32_t) * (nnz ? nnz : 1)));
  TRY(ensure(h->h_ids, sizeof(uint32_t) * (n ? n : 1) * k));
  TRY(ensure(h->h_cnt, sizeof(uint32_t) * (n ? n : 1) * k));
  {
    Phase ph(h, 3, s);
    CUDA_TRY(cudaMemcpyAsync(h->h_rp.p, row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
    if (nnz)
      CUDA_TRY(cudaMemcpyAsync(h->h_col.p, col_idx + e0, sizeof(uint32_t) * nnz, cudaMemcpyHostToDevice, s));
  }
  TRY(dist_knn_graph(h, h->h_rp.as<int64_t>(), h->h_col.as<uint32_t>() - e0, n, k, h->h_ids.as<uint32_t>(),
                     h->h_cnt.as<uint32_t>(), s));
  if (n) {
    Phase ph(h, 3, s);
    CUDA_TRY(cudaMemcpyAsync(out_ids, h->h_ids.p, sizeof(uint32_t) * n * k, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(out_counts, h->h_cnt.p, sizeof(uint32_t) * n * k, cudaMemcpyDeviceToHost, s));
  }
  CUDA_TRY(cudaStreamSynchronize(s));
  return FLASH_OK;
}

flash_status dist_clear(flash_index* h, cudaStream_t s) {
  DistState* d = D(h);
  TRY(enter(h, s));
  if (d->win) {
    flash_index* w = d->win;
    CUDA_TRY(cudaMemsetAsync(w->arrivals, 0, sizeof(uint32_t) * nbuckets(w), s));
    w->have_tables = false;
    w->kept_ub = 0;
    w->n_inserted = 0;
    w->max_id = 0;
  }
  d->max_id = 0;
  d->have_any = false;
  h->have_tables = false;
  h->n_inserted = 0;
  return FLASH_OK;
}

flash_status dist_get_table(flash_index* h, uint32_t t, const uint32_t** off, const uint32_t** ids,
                            const uint32_t** arrivals, uint64_t* n_ids) {
  DistState* d = D(h);
  if (t < d->t0 || t >= d->t1 || !d->win)
    return fail(FLASH_ESTATE, "table %u is not in rank %d's window [%u, %u)", t, d->rank, d->t0, d->t1);
  if (!d->win->have_tables) return fail(FLASH_ESTATE, "nothing inserted yet");
  if (h->have_last) {
    CUDA_TRY(cudaSetDevice(h->device));
    CUDA_TRY(cudaStreamSynchronize(h->last_stream));
  }
  return flash_get_table(d->win, t - d->t0, off, ids, arrivals, n_ids);
}

flash_status dist_check(const flash_index* hc, uint64_t* n_errors) {
  flash_index* h = const_cast<flash_index*>(hc);
  DistState* d = D(h);
  TRY(d->tr->check());
  CUDA_TRY(cudaSetDevice(h->device));
  if (h->have_last) CUDA_TRY(cudaStreamSynchronize(h->last_stream));
  unsigned long long e = 0, e2 = 0;
  CUDA_TRY(cudaMemcpy(&e, h->err, sizeof e, cudaMemcpyDeviceToHost));
  if (d->win) CUDA_TRY(cudaMemcpy(&e2, d->win->err, sizeof e2, cudaMemcpyDeviceToHost));
  if (n_errors) *n_errors = e + e2;
  return FLASH_OK;
}

void dist_destroy(flash_index* h) {
  DistState* d = D(h);
  if (!d) return;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  if (d->mapped) unmap_all(d);
  if (d->win) free_handle(d->win);
  for (DevBuf* b : {&d->x1, &d->cand[0], &d->cand[1], &d->segs[0], &d->segs[1], &d->dpeer, &d->sizes, &d->offs,
                    &d->goffq, &d->dbounds, &d->scan_tmp})
    release(*b);
  delete d;  // the transport (NCCL communicators / local group reference) goes with it
  h->dist = nullptr;
}

namespace {

flash_status validate(uint32_t K, uint32_t L, uint32_t R, uint32_t range) {
  if (K < 1 || L < 1 || (uint64_t)K * L > FLASH_MAX_BINS)
    return fail(FLASH_EINVAL, "need 1 <= K, 1 <= L, K*L <= %u (K=%u L=%u)", FLASH_MAX_BINS, K, L);
  if (R < 1 || R > FLASH_MAX_R) return fail(FLASH_EINVAL, "R=%u outside [1, %u]", R, FLASH_MAX_R);
  if (range < 1 || range > (1u << 31)) return fail(FLASH_EINVAL, "range=%u outside [1, 2^31]", range);
  if ((uint64_t)L * range > (1ull << 31)) return fail(FLASH_EINVAL, "L*range must be <= 2^31");
  return FLASH_OK;
}

// The outer handle (hashes all L tables of its rows; holds no tables) and its window.
flash_status make_dist(uint32_t K, uint32_t L, uint32_t R, uint32_t range, uint64_t seed, int rank, int world,
                       std::unique_ptr<Transport> tr, flash_index** out) {
  flash_status st;
  flash_index* h = new_handle(K, L, R, range, seed, 0, &st, false);
  if (!h) return st;
  DistState* d = new (std::nothrow) DistState();
  if (!d) {
    free_handle(h);
    return fail(FLASH_ENOMEM, "host allocation failed");
  }
  d->rank = rank;
  d->world = world;
  d->t0 = win_t0(L, world, rank);
  d->t1 = win_t0(L, world, rank + 1);
  tr->rank = rank;
  tr->world = world;
  d->tr = std::move(tr);
  h->dist = d;
  if (d->t1 > d->t0) {
    d->win = new_handle(K, d->t1 - d->t0, R, range, seed, 0, &st);
    if (!d->win) {
      flash_destroy(h);
      return st;
    }
    d->win->keys.tbase = d->t0;  // priorities keyed by the global table index
  }
  *out = h;
  return FLASH_OK;
}

}  // namespace
}  // namespace api
}  // namespace flash

extern "C" {

flash_status flash_get_unique_id(void* unique_id) {
  if (!unique_id) return fail(FLASH_EINVAL, "unique_id is NULL");
  const NcclApi& n = nccl();
  if (!n.ok) return fail(FLASH_ENCCL, "%s", n.why.c_str());
  ncclUniqueId id;
  NCCL_TRY(n.GetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == FLASH_UNIQUE_ID_BYTES, "ncclUniqueId size");
  memcpy(unique_id, &id, sizeof id);
  return FLASH_OK;
}

flash_status flash_create_dist(uint32_t K, uint32_t L, uint32_t R, uint32_t range, uint64_t seed, int rank,
                               int world, const void* unique_id, flash_index** out) {
  if (!out) return fail(FLASH_EINVAL, "out is NULL");
  *out = nullptr;
  TRY(validate(K, L, R, range));
  if (world < 1 || world > 4096 || rank < 0 || rank >= world)
    return fail(FLASH_EINVAL, "need 0 <= rank < world <= 4096 (rank=%d world=%d)", rank, world);
  if (!unique_id) return fail(FLASH_EINVAL, "unique_id is NULL");
  const NcclApi& n = nccl();
  if (!n.ok) return fail(FLASH_ENCCL, "%s", n.why.c_str());
  std::unique_ptr<NcclTransport> tr(new (std::nothrow) NcclTransport());
  if (!tr) return fail(FLASH_ENOMEM, "host allocation failed");
  CUDA_TRY(cudaGetDevice(&tr->device));
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof id);
  NCCL_TRY(n.CommInitRank(&tr->comm, world, id, rank));
  NCCL_TRY(n.CommSplit(tr->comm, 0, rank, &tr->ctl, nullptr));
  CUDA_TRY(cudaStreamCreateWithFlags(&tr->cs, cudaStreamNonBlocking));
  CUDA_TRY(cudaMalloc(&tr->dflag, sizeof(int)));
  CUDA_TRY(cudaMemset(tr->dflag, 0, sizeof(int)));
  TRY(tr->stage(64 * 1024));  // (staging never regrows in steady state: a cudaFree would sync the device)
  return make_dist(K, L, R, range, seed, rank, world, std::move(tr), out);
}

flash_status flash_create_dist_local(uint32_t K, uint32_t L, uint32_t R, uint32_t range, uint64_t seed, int world,
                                     const int* devices, flash_index** out) {
  if (!out) return fail(FLASH_EINVAL, "out is NULL");
  if (world < 1 || world > 4096) return fail(FLASH_EINVAL, "world=%d outside [1, 4096]", world);
  for (int g = 0; g < world; ++g) out[g] = nullptr;
  TRY(validate(K, L, R, range));
  int cur = 0;
  CUDA_TRY(cudaGetDevice(&cur));
  auto grp = std::make_shared<LocalGroup>(world);
  flash_status st = FLASH_OK;
  for (int g = 0; g < world && st == FLASH_OK; ++g) {
    const int dev = devices ? devices[g] : cur;
    if (cudaSetDevice(dev) != cudaSuccess) {
      cudaGetLastError();
      st = fail(FLASH_EINVAL, "device %d is not available", dev);
      break;
    }
    for (int p = 0; p < 2 && st == FLASH_OK; ++p)
      if (cudaEventCreateWithFlags(&grp->ev[2 * g + p], cudaEventDisableTiming) != cudaSuccess)
        st = fail(FLASH_ECUDA, "cudaEventCreate failed");
    if (devices)  // peer stores between the group's devices
      for (int o = 0; o < world; ++o)
        if (devices[o] != dev) {
          const cudaError_t e = cudaDeviceEnablePeerAccess(devices[o], 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
            cudaGetLastError();
            st = fail(FLASH_ECUDA, "peer access %d -> %d: %s", dev, devices[o], cudaGetErrorString(e));
          }
          cudaGetLastError();
        }
    if (st != FLASH_OK) break;
    std::unique_ptr<LocalTransport> tr(new LocalTransport());
    tr->grp = grp;
    st = make_dist(K, L, R, range, seed, g, world, std::move(tr), &out[g]);
  }
  cudaSetDevice(cur);
  if (st != FLASH_OK) {
    for (int g = 0; g < world; ++g) {
      flash_destroy(out[g]);
      out[g] = nullptr;
    }
  }
  // the events live as long as the group (destroyed with the last reference)
  return st;
}

flash_status flash_dist_info(const flash_index* h, int* rank, int* world, uint32_t* t_begin, uint32_t* t_end) {
  if (!h) return fail(FLASH_EINVAL, "handle is NULL");
  if (!h->dist) {
    if (rank) *rank = 0;
    if (world) *world = 1;
    if (t_begin) *t_begin = 0;
    if (t_end) *t_end = h->L;
    return FLASH_OK;
  }
  if (rank) *rank = h->dist->rank;
  if (world) *world = h->dist->world;
  if (t_begin) *t_begin = h->dist->t0;
  if (t_end) *t_end = h->dist->t1;
  return FLASH_OK;
}

}  // extern "C"
