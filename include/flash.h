/*
 * flash.h — C ABI of libflash.so, the B200 (sm_100a) hot path of FLASH
 * (Wang, Shrivastava, Wang, Ryu, SIGMOD'18, arXiv 1709.01190).
 *
 * Citations: P:n = PAPER.md line n; DESIGN.md §2 (HASHSPEC) gives the exact integer
 * definitions; R#n = DESIGN.md readings ledger.
 *
 * Conventions (all calls):
 *   - Pointers are DEVICE pointers unless a function says "host".  The caller owns
 *     every input and output buffer; the library never frees them.
 *   - `stream` is a cudaStream_t passed as void* (NULL = the legacy default stream).
 *     Every call is stream-ordered and returns after enqueueing; results are valid
 *     once the stream reaches that point.  No call synchronizes the host unless it
 *     says so.
 *   - CSR input: row r's column indices are col_idx[row_ptr[r] .. row_ptr[r+1])
 *     (absolute indexing into col_idx, so a row slice of a larger CSR can be passed
 *     with the same col_idx).  Rows are sets: order and duplicates do not matter.
 *     Column indices must be < 0xFFFFFFFF.  An empty row hashes to all-EMPTY codes and
 *     EMPTY addresses, is never inserted, and a query on it returns k pads (R#15).
 *   - Ids are uint32, unique across inserts (caller contract, as SPEC S:213) and
 *     < 0xFFFFFFFF.
 *   - Errors: argument errors are detected on the host before anything is enqueued
 *     and leave the index unchanged (FLASH_EINVAL).  CUDA errors surface as
 *     FLASH_ECUDA from the call that observes them.  flash_last_error() returns a
 *     thread-local message for the last non-OK status.  No C++ exception crosses
 *     the ABI.
 *   - Thread safety: one handle must not be used concurrently from several host
 *     threads; distinct handles are independent.
 */
#ifndef FLASH_H_
#define FLASH_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FLASH_EMPTY 0xFFFFFFFFu /* empty code / no address / output pad id */

/* Limits checked by flash_create (FLASH_EINVAL otherwise). */
#define FLASH_MAX_BINS 8192u    /* K*L */
#define FLASH_MAX_R 4096u
#define FLASH_MAX_TOPK 1024u

typedef struct flash_index flash_index; /* opaque; owned by the library */

typedef enum {
    FLASH_OK = 0,
    FLASH_EINVAL = 1, /* bad argument; nothing enqueued */
    FLASH_ENOMEM = 2, /* device allocation failed */
    FLASH_ECUDA = 3,  /* CUDA runtime error (message in flash_last_error) */
    FLASH_ENCCL = 4,  /* NCCL failed (multi-GPU handle; message in flash_last_error) */
    FLASH_ESTATE = 5  /* call not valid in the handle's state */
} flash_status;

/* Create an empty index: L hash tables of `range` buckets, each bucket a reservoir of
 * at most R ids; every table key is a K-tuple of DOPH hashes (§2.2,
 * P:185-195 §3.2).  seed: the single 64-bit seed all hash keys derive from (R#2).
 * Requires 1 <= K, 1 <= L, K*L <= FLASH_MAX_BINS, 1 <= R <= FLASH_MAX_R,
 * 1 <= range <= 2^31, and a CUDA device (the current device at create time is
 * the handle's device).  Allocates O(L*range) device memory. */
flash_status flash_create(uint32_t K, uint32_t L, uint32_t R, uint32_t range, uint64_t seed,
                          flash_index **out);

/* flash_create with reservoir sharing across tables (§3.2(4); §3.5 P:352-362;
 * R#23): the L*range table buckets point into one pool of `pool` reservoirs
 * (pool = ceil(F*L*range) for the paper's fraction F).  Bucket (t, b) is bound to
 * reservoir mulhi(fmix32(fmix32(s_pool ^ t) ^ b), pool) (data-independent, so the index is
 * order-free); a row enters each of its distinct reservoirs once and a query aggregates each
 * distinct reservoir once (counts <= L).  pool = 0 or L*range: the unshared index (exactly
 * flash_create).  1 <= pool <= L*range, else FLASH_EINVAL.  With sharing, flash_get_table
 * and the table-window calls (multi-GPU) return FLASH_ESTATE / FLASH_EINVAL;
 * flash_table_arrays reports the pool ([pool+1] offsets, [pool] arrivals). */
flash_status flash_create_pool(uint32_t K, uint32_t L, uint32_t R, uint32_t range, uint64_t pool, uint64_t seed,
                               flash_index **out);

/* Free the tables and the handle (synchronizes the device first).  NULL is a no-op. */
void flash_destroy(flash_index *h);

/* DOPH of n_rows CSR rows (H1-H3; §2.3, Alg. 2 lines 3-5 P:213-215).
 * codes: [n_rows][K*L] uint32, table t owns [t*K, (t+1)*K) — or NULL.
 * addrs: [n_rows][L] uint32 bucket addresses in [0, range) or FLASH_EMPTY — or NULL.
 * At least one of codes / addrs must be non-NULL. */
flash_status flash_hash(const flash_index *h, const int64_t *row_ptr, const uint32_t *col_idx,
                        uint64_t n_rows, uint32_t *codes, uint32_t *addrs, void *stream);

/* Adding phase (Alg. 2): hash n_rows rows and insert ids id_base + r into
 * every table's addressed bucket under the bottom-R rule (R#7): each bucket keeps the
 * min(arrivals, R) ids with smallest (prio(t,b,id), id), ascending by id.  Inserting in
 * several batches gives the same tables as one batch (bottom-R is composable). */
flash_status flash_insert(flash_index *h, const int64_t *row_ptr, const uint32_t *col_idx,
                          uint64_t n_rows, uint32_t id_base, void *stream);

/* Same as flash_insert with precomputed addresses addrs [n_rows][L] (e.g. gathered from
 * other ranks).  Entries >= range other than FLASH_EMPTY are invalid: they are skipped
 * and counted in the handle's device error counter (flash_check). */
flash_status flash_insert_addrs(flash_index *h, const uint32_t *addrs, uint64_t n_rows,
                                uint32_t id_base, void *stream);

/* flash_insert_addrs restricted to tables [t_begin, t_end): the rows' addresses for
 * other tables are ignored and those tables keep their content.  The multi-GPU graph
 * (paper_1709_01190_b200/dist.py) builds each GPU's table window with this and then
 * assembles the full tables on every GPU (flash_table_arrays / flash_import_tables).
 * The tables of a window are exactly those a full insert would build (bottom-R is
 * per-bucket; the priority uses the global table index). */
flash_status flash_insert_addrs_window(flash_index *h, const uint32_t *addrs, uint64_t n_rows,
                                       uint32_t id_base, uint32_t t_begin, uint32_t t_end,
                                       void *stream);

/* Device pointers to the whole index: goff [L*range+1] (uint64 absolute offsets: table t,
 * bucket b holds ids[goff[t*range+b] .. goff[t*range+b+1])), ids [*n_ids], arrivals
 * [L*range].  Synchronizes the handle's last stream.  Valid until the next insert,
 * import, clear or destroy.  Before any insert: FLASH_ESTATE. */
flash_status flash_table_arrays(const flash_index *h, const uint64_t **goff, const uint32_t **ids,
                                const uint32_t **arrivals, uint64_t *n_ids);

/* Replace the index content with copies of device arrays in flash_table_arrays' layout
 * (arrivals may be NULL: zeros).  The offsets are validated first (goff[0] == 0,
 * non-decreasing, goff[L*range] == n_ids; else FLASH_EINVAL and the index is unchanged) and
 * the largest imported id is taken from ids (it sets the query kernels' digit range): both
 * on the device, then the call synchronizes `stream` once. */
flash_status flash_import_tables(flash_index *h, const uint64_t *goff, const uint32_t *ids, uint64_t n_ids,
                                 const uint32_t *arrivals, void *stream);

/* Querying phase (Alg. 3) for n_q CSR query rows: aggregate the L addressed
 * buckets, count each candidate's multiplicity (full count, R#11), drop exclude[q] (if
 * exclude != NULL, R#14), order by (count desc, id asc) (R#12), keep k, pad with
 * (FLASH_EMPTY, 0) (R#13).  out_ids / out_counts: [n_q][k] uint32.  1 <= k <= FLASH_MAX_TOPK.
 * Every query call (also flash_query_addrs, flash_knn_graph*, flash_count_topk) requires
 * L*R <= FLASH_MAX_CANDIDATES (the count tables' capacity), else FLASH_EINVAL. */
#define FLASH_MAX_CANDIDATES 32768u
flash_status flash_query_topk(const flash_index *h, const int64_t *row_ptr, const uint32_t *col_idx,
                              uint64_t n_q, uint32_t k, const uint32_t *exclude, uint32_t *out_ids,
                              uint32_t *out_counts, void *stream);

/* Same as flash_query_topk with precomputed query addresses addrs [n_q][L]. */
flash_status flash_query_addrs(const flash_index *h, const uint32_t *addrs, uint64_t n_q, uint32_t k,
                               const uint32_t *exclude, uint32_t *out_ids, uint32_t *out_counts,
                               void *stream);

/* Approximate k-NN graph from scratch: insert rows as ids 0..n_rows-1, then
 * query every row with its own addresses, excluding itself.  Requires a fresh handle
 * (nothing inserted yet), else FLASH_ESTATE.  out_ids / out_counts: [n_rows][k]. */
flash_status flash_knn_graph(flash_index *h, const int64_t *row_ptr, const uint32_t *col_idx,
                             uint64_t n_rows, uint32_t k, uint32_t *out_ids, uint32_t *out_counts,
                             void *stream);

/* flash_knn_graph on HOST buffers (row_ptr [n_rows+1], col_idx [row_ptr[n_rows]],
 * out_ids / out_counts [n_rows][k], all host; pinned memory is fastest): copies the CSR
 * to the device (chunked, overlapped with hashing), runs the graph, copies the results
 * back, and synchronizes `stream` before returning. */
flash_status flash_knn_graph_host(flash_index *h, const int64_t *row_ptr, const uint32_t *col_idx,
                                  uint64_t n_rows, uint32_t k, uint32_t *out_ids, uint32_t *out_counts,
                                  void *stream);

/* ---- Multi-GPU candidate exchange (north_star (d)) ----------
 * The L tables are partitioned over `world` GPUs by floor blocks: rank g owns the table
 * window [t0(g), t1(g)) = [floor(g*L/world), floor((g+1)*L/world)).  A query's candidate
 * multiset (Alg. 3 lines 4-7) is the union over ranks of the buckets it
 * addresses in each window, so the owner of a query can count and select (Q2-Q3) over
 * the per-rank lists exactly as a single GPU does over the L buckets. */

/* flash_hash writing only addresses, laid out by table owner (the exchange's send layout
 * for the address all-to-all, X1): rank g's block is [n_rows][t1(g)-t0(g)] uint32 and
 * starts at element n_rows * t0(g) of addrs (total n_rows * L elements).  world == 1 is
 * the plain [n_rows][L] layout.  1 <= world <= 65536. */
flash_status flash_hash_blocked(const flash_index *h, const int64_t *row_ptr, const uint32_t *col_idx,
                                uint64_t n_rows, uint32_t world, uint32_t *addrs, void *stream);

/* flash_insert_addrs_window where addrs holds only the window's columns: addrs
 * [n_rows][t_end - t_begin], column j = table t_begin + j (the address all-to-all's
 * receive layout).  Builds tables [t_begin, t_end) exactly as a full insert would
 * (bottom-R is per bucket, keyed by the global table index); other tables are kept. */
flash_status flash_insert_addrs_cols(flash_index *h, const uint32_t *addrs, uint64_t n_rows,
                                     uint32_t id_base, uint32_t t_begin, uint32_t t_end, void *stream);

/* Per-query candidate counts of the table window [t_begin, t_end) for n_q queries whose
 * window addresses are addrs [n_q][t_end - t_begin]: sizes[q] (uint32, [n_q]) = sum of
 * the addressed buckets' sizes; offsets (uint64, [n_q+1]) = their exclusive scan, total
 * at offsets[n_q].  These are the per-destination sizes of the candidate all-to-all (X2).
 * Before any insert every size is 0. */
flash_status flash_window_sizes(const flash_index *h, const uint32_t *addrs, uint64_t n_q, uint32_t t_begin,
                                uint32_t t_end, uint32_t *sizes, uint64_t *offsets, void *stream);

/* Gather (Q1 restricted to the window): out_ids[offsets[q] .. offsets[q+1]) = the
 * concatenation, in table order, of query q's window buckets (ascending ids within each).
 * offsets from flash_window_sizes with the same arguments; out_ids has offsets[n_q]
 * entries (caller-allocated). */
flash_status flash_window_gather(const flash_index *h, const uint32_t *addrs, uint64_t n_q, uint32_t t_begin,
                                 uint32_t t_end, const uint64_t *offsets, uint32_t *out_ids, void *stream);

/* Q2-Q3 on pre-gathered candidate segments (the owner side of X2): query q's candidates
 * are the n_seg segments (s, q), s < n_seg, stored consecutively in (s, q) order in cand:
 * segment (s, q) has seg_sizes[s*n_q + q] ids.  Counts multiplicities (R#11), drops
 * exclude[q] (if exclude != NULL), orders by (count desc, id asc), keeps k, pads (R#12,
 * R#13) — the same result as flash_query_addrs when the segments are the query's
 * buckets split by table window.  Preconditions (the exchange guarantees them): an id
 * occurs at most once per table, so counts are <= the handle's L, and a query has at most
 * L*R candidates (a query with more is counted in the device error counter, flash_check,
 * and gets k pads).  max_id bounds every candidate id.  cand may be NULL when every size is
 * 0 (a query with candidates then counts as an error and gets k pads).  1 <= n_seg <= 4096,
 * n_q < 2^31.  The handle's tables are not used. */
flash_status flash_count_topk(const flash_index *h, const uint32_t *cand, const uint32_t *seg_sizes,
                              uint32_t n_seg, uint64_t n_q, uint32_t k, const uint32_t *exclude, uint32_t max_id,
                              uint32_t *out_ids, uint32_t *out_counts, void *stream);

/* ---- Multi-GPU handle (north_star (d)) ---------------
 * One handle per GPU (rank g of `world`, one node).  The L tables are partitioned over the
 * ranks by floor blocks — rank g owns [floor(g*L/world), floor((g+1)*L/world)) — and every
 * query is answered on the rank that passed its row (queries are data-parallel, P:322
 * §3.4).  On such a handle flash_insert, flash_query_topk, flash_knn_graph(_host) are
 * COLLECTIVE: every rank calls them, in the same order, with its own contiguous row shard
 * (n_rows may differ per rank and may be 0):
 *   - flash_knn_graph: the shards in rank order are rows 0..N-1 of ONE graph (global ids =
 *     rank offset + local row); out_ids / out_counts [n_rows][k] are this rank's rows.
 *   - flash_insert: rank g's rows get ids id_base_g + r (id_base per rank).
 *   - flash_query_topk: this rank's queries against the whole (distributed) index;
 *     exclude [n_q] per local query.
 * Results are byte-identical to a single-GPU handle with the same (K, L, R, range, seed) fed
 * the concatenated shards.  Row addresses travel to the table owners and candidate lists to
 * the query owners as stores into the peers' memory (NVLink P2P), separated by stream-ordered
 * barriers; the host synchronizes once per call to exchange the shard sizes.
 * flash_get_table works for the rank's own tables; flash_clear is local; flash_hash works on
 * the rank's rows (all L tables); the single-GPU step calls (flash_insert_addrs*,
 * flash_query_addrs, flash_table_arrays, flash_import_tables, flash_count_topk, window calls)
 * return FLASH_ESTATE. */
#define FLASH_UNIQUE_ID_BYTES 128

/* NCCL bootstrap id (host buffer of FLASH_UNIQUE_ID_BYTES): rank 0 creates it and hands it to
 * every rank out of band (e.g. torch.distributed broadcast). */
flash_status flash_get_unique_id(void *unique_id);

/* Collective over `world` processes (one GPU each, the current device): rank `rank` of a
 * multi-GPU handle with an NCCL communicator owned by the handle.  NCCL (libnccl.so.2) is
 * loaded at run time; FLASH_ENCCL if it is missing or fails.  Peer buffers are mapped with
 * CUDA IPC, so the ranks must share a node.  0 <= rank < world <= 4096. */
flash_status flash_create_dist(uint32_t K, uint32_t L, uint32_t R, uint32_t range, uint64_t seed, int rank,
                               int world, const void *unique_id, flash_index **out);

/* The same for `world` virtual ranks in ONE process: out[g] (host array [world]) is rank g's
 * handle, on device devices[g] (host array, or NULL: every rank on the current device; peer
 * access is enabled between distinct devices).  Each rank's collective calls must come from
 * its own host thread (they wait for each other), each on its own stream. */
flash_status flash_create_dist_local(uint32_t K, uint32_t L, uint32_t R, uint32_t range, uint64_t seed, int world,
                                     const int *devices, flash_index **out);

/* rank, world and table window [t_begin, t_end) of a handle (a plain handle: 0, 1, [0, L)). */
flash_status flash_dist_info(const flash_index *h, int *rank, int *world, uint32_t *t_begin, uint32_t *t_end);

/* Drop every inserted id (stream-ordered): the handle returns to its freshly created
 * state (arrivals zero, no tables), keeping K, L, R, range and seed. */
flash_status flash_clear(flash_index *h, void *stream);

/* Device pointers to table t: off [range+1] (bucket b holds ids[off[b]..off[b+1])),
 * ids [*n_ids] (ascending within each bucket), arrivals [range] (ReservoirCounter).
 * Synchronizes the handle's last stream.  Pointers stay valid until the next insert or
 * destroy.  Before any insert: FLASH_ESTATE. */
flash_status flash_get_table(const flash_index *h, uint32_t t, const uint32_t **off,
                             const uint32_t **ids, const uint32_t **arrivals, uint64_t *n_ids);

/* Synchronize the handle's last stream and report the device-side error counter
 * (invalid addresses seen by flash_insert_addrs / flash_query_addrs) in *n_errors (host). */
flash_status flash_check(const flash_index *h, uint64_t *n_errors);

/* Profiling: when enabled, every call records CUDA events around its phases on the
 * caller's stream.  flash_phase_ms (host out, synchronizes) returns the accumulated
 * milliseconds of phase i: 0 = hash (H1-H3), 1 = build (B1-B2), 2 = query (Q1-Q3),
 * 3 = host<->device copies (flash_knn_graph_host), and their launch counts.
 * flash_launch_count returns the number of kernels this handle has launched. */
flash_status flash_set_profiling(flash_index *h, int enable);
flash_status flash_phase_ms(const flash_index *h, double ms_out[4], uint64_t calls_out[4]);
uint64_t flash_launch_count(const flash_index *h);
flash_status flash_reset_counters(flash_index *h);

/* Thread-local message for the last non-OK status returned on this thread. */
const char *flash_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* FLASH_H_ */
