/*
 * oracle/flash_oracle.c — plain, slow, obviously-correct CPU oracle for FLASH's hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant generator with the CUDA path (paper_1709_01190_b200/);
 * the two meet only at the written specification.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (section / equation /
 * algorithm named alongside); "S:n" = SPEC.md line n; "R#n" = reading n of the
 * DESIGN.md readings ledger (where the paper is silent or garbled).
 *
 * What each function computes, in the paper's order:
 *   oracle_doph        DOPH of one CSR row per row: one-permutation bin minima
 *                      (Eq. 1 per bin; §2.3) then optimal
 *                      densification (ref [36]; reading R#4).
 *   oracle_addresses   MapKHashesToAddress (Alg. 2 line 5; "universal random
 *                      mapping function to the desired address range"; R#5).
 *   oracle_build       Adding phase (Alg. 2) with the bottom-R reservoir
 *                      rule (north_star; same law as Vitter's Alg. 1; R#7, R#9, R#10).
 *   oracle_query       Querying phase (Alg. 3): aggregate, KSELECT =
 *                      SORTINPLACE, COUNTFREQUENCY (full multiplicity, R#11),
 *                      SORTBYVALUE (count desc, id asc, R#12), top-k (pad R#13).
 *   oracle_bruteforce_topk / oracle_pair_similarity
 *                      exact Jaccard (Eq. 2) and binary cosine (Eq. 3)
 *                      in fp64 — the recall reference (O-2), pins nothing bit-exactly.
 *
 * Parity status: the hash constants (fmix32/mix64 family, probe, fold, prio) are our
 * HASHSPEC choices; the paper prints no hash values, so they are "parity unpinned"
 * against the paper and pinned only statistically (Eq. 2 calibration, Vitter's law)
 * and by the MurmurHash3 / SplitMix64 reference vectors (tests/golden/).
 * All arithmetic is uint32/uint64 modulo 2^32/2^64; fp64 only in the brute force.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_EMPTY 0xFFFFFFFFu /* empty-bin / no-address sentinel (R#3) */
#define ORACLE_T_PROBES 64u      /* probe-chain cap before the circular scan (R#4) */

/* ------------------------------------------------------------------------- */
/* Hash primitives (HASHSPEC).                                               */
/* ------------------------------------------------------------------------- */

/* MurmurHash3 32-bit finalizer: a bijection on uint32. */
uint32_t oracle_fmix32(uint32_t h) {
    h ^= h >> 16;
    h *= 0x85EBCA6Bu;
    h ^= h >> 13;
    h *= 0xC2B2AE35u;
    h ^= h >> 16;
    return h;
}

/* SplitMix64 output function (Steele, Lea, Flood 2014). */
uint64_t oracle_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* Uniform reduction of a 32-bit hash to [0, n): floor(h * n / 2^32). */
static uint32_t mulhi_range(uint32_t h, uint32_t n) {
    return (uint32_t)(((uint64_t)h * (uint64_t)n) >> 32);
}

typedef struct {
    uint32_t a1, m1, a2, s_dens; /* DOPH's "4 random numbers" */
    uint32_t s_addr;             /* address-map key (R#5) */
    uint32_t s_pool;             /* shared-reservoir map key (R#23) */
    uint64_t s_prio;             /* bottom-R priority key (R#9) */
} oracle_seeds;

/* One 64-bit seed -> the first four outputs of a SplitMix64 stream (R#2). */
void oracle_derive_seeds(uint64_t seed, oracle_seeds *s) {
    uint64_t w[4];
    for (int k = 0; k < 4; ++k) w[k] = oracle_mix64(seed + (uint64_t)(k + 1) * 0x9E3779B97F4A7C15ull);
    s->a1 = (uint32_t)w[0];
    s->m1 = (uint32_t)(w[0] >> 32) | 1u;
    s->a2 = (uint32_t)w[1];
    s->s_dens = (uint32_t)(w[1] >> 32);
    s->s_addr = (uint32_t)w[2];
    s->s_pool = (uint32_t)(w[2] >> 32);
    s->s_prio = w[3];
}

/* pi(c): the random permutation of Eq. 1, a keyed bijection on uint32 (R#1). */
uint32_t oracle_perm(uint64_t seed, uint32_t c) {
    oracle_seeds s;
    oracle_derive_seeds(seed, &s);
    return oracle_fmix32(((c ^ s.a1) * s.m1) + s.a2);
}

/* probe(i, a): a-th bin on empty bin i's data-independent densification chain (R#4). */
uint32_t oracle_probe(uint64_t seed, uint32_t i, uint32_t a, uint32_t B) {
    oracle_seeds s;
    oracle_derive_seeds(seed, &s);
    return mulhi_range(oracle_fmix32(s.s_dens ^ ((i << 8) | a)), B);
}

/* prio(t, b, id): hashed reservoir priority (north_star "hash(seed,table,bucket,id)"; R#9). */
uint32_t oracle_prio(uint64_t seed, uint32_t t, uint32_t b, uint32_t id) {
    oracle_seeds s;
    oracle_derive_seeds(seed, &s);
    uint64_t tb = oracle_mix64(s.s_prio ^ (((uint64_t)t << 32) | (uint64_t)b));
    return (uint32_t)(oracle_mix64(tb ^ (uint64_t)id) >> 32);
}

/* oracle_prio for n (t, b, id) triples (a loop over oracle_prio; for sampled checks). */
void oracle_prio_batch(uint64_t seed, const uint32_t *t, const uint32_t *b, const uint32_t *id, uint64_t n,
                       uint32_t *out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = oracle_prio(seed, t[i], b[i], id[i]);
}

/* ------------------------------------------------------------------------- */
/* DOPH (§2.3; §3.2(1)).                               */
/* ------------------------------------------------------------------------- */

/* codes[r*B + i] for B = K*L bins; table t owns bins [t*K, (t+1)*K).
 * Returns 0, or 1 on bad arguments.  An empty row gets all-EMPTY codes (R#15). */
int oracle_doph(uint32_t K, uint32_t L, uint64_t seed, const int64_t *row_ptr,
                const uint32_t *col_idx, uint64_t n_rows, uint32_t *codes) {
    if (K == 0 || L == 0 || (uint64_t)K * L > 65535u) return 1;
    const uint32_t B = K * L;
    oracle_seeds s;
    oracle_derive_seeds(seed, &s);
#pragma omp parallel
    {
        uint32_t *v = (uint32_t *)malloc(sizeof(uint32_t) * B);
#pragma omp for schedule(dynamic, 64)
        for (int64_t r = 0; r < (int64_t)n_rows; ++r) {
            /* H1 — one pass over the nonzeros: bin b holds min pi(c) over the row's
             * indices c whose pi(c) falls in b's range (Eq. 1 restricted to bin b). */
            for (uint32_t i = 0; i < B; ++i) v[i] = ORACLE_EMPTY;
            for (int64_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) { /* absolute CSR indexing */
                uint32_t h = oracle_fmix32(((col_idx[e] ^ s.a1) * s.m1) + s.a2); /* pi(c) */
                uint32_t b = mulhi_range(h, B);                                  /* bin */
                if (h < v[b]) v[b] = h;
            }
            /* H2 — densification: an empty bin copies the value of the first
             * originally non-empty bin on its probe chain; donors are read from v,
             * never from already-densified codes (R#4). */
            uint32_t *code = codes + (uint64_t)r * B;
            for (uint32_t i = 0; i < B; ++i) {
                if (v[i] != ORACLE_EMPTY) { code[i] = v[i]; continue; }
                uint32_t found = ORACLE_EMPTY, j = 0;
                int ok = 0;
                for (uint32_t a = 1; a <= ORACLE_T_PROBES; ++a) {
                    j = mulhi_range(oracle_fmix32(s.s_dens ^ ((i << 8) | a)), B);
                    if (v[j] != ORACLE_EMPTY) { found = v[j]; ok = 1; break; }
                }
                if (!ok) { /* circular scan from the last probed bin */
                    for (uint32_t m = 1; m <= B; ++m) {
                        uint32_t jj = (uint32_t)(((uint64_t)j + m) % B);
                        if (v[jj] != ORACLE_EMPTY) { found = v[jj]; break; }
                    }
                }
                code[i] = found; /* stays EMPTY only when the whole row is empty */
            }
        }
        free(v);
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* MapKHashesToAddress (Alg. 2 line 5).                        */
/* ------------------------------------------------------------------------- */

/* addrs[r*L + t] in [0, range), or EMPTY for an empty row (R#15). */
int oracle_addresses(uint32_t K, uint32_t L, uint32_t range, uint64_t seed, const uint32_t *codes,
                     uint64_t n_rows, uint32_t *addrs) {
    if (K == 0 || L == 0 || range == 0 || (uint64_t)K * L > 65535u) return 1;
    oracle_seeds s;
    oracle_derive_seeds(seed, &s);
    const uint32_t B = K * L;
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < (int64_t)n_rows; ++r) {
        const uint32_t *code = codes + (uint64_t)r * B;
        for (uint32_t t = 0; t < L; ++t) {
            if (code[0] == ORACLE_EMPTY) { addrs[(uint64_t)r * L + t] = ORACLE_EMPTY; continue; }
            uint32_t x = oracle_fmix32(s.s_addr ^ t);
            for (uint32_t j = 0; j < K; ++j) x = oracle_fmix32(x ^ code[t * K + j]);
            addrs[(uint64_t)r * L + t] = mulhi_range(x, range);
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Adding phase with bottom-R reservoirs (Alg. 2).                */
/* ------------------------------------------------------------------------- */

typedef struct { uint32_t b, prio, id; } arrival;

static int cmp_arrival(const void *x, const void *y) {
    const arrival *a = (const arrival *)x, *c = (const arrival *)y;
    if (a->b != c->b) return a->b < c->b ? -1 : 1;
    if (a->prio != c->prio) return a->prio < c->prio ? -1 : 1;
    if (a->id != c->id) return a->id < c->id ? -1 : 1;
    return 0;
}
static int cmp_u32(const void *x, const void *y) {
    uint32_t a = *(const uint32_t *)x, b = *(const uint32_t *)y;
    return a < b ? -1 : (a > b);
}

/* Every id inserted so far, grouped per table t and bucket b:
 *   S(t,b) = { id : addr_t(id) = b }            arrivals[t][b] = |S| (ReservoirCounter)
 *   kept(t,b) = the min(|S|, R) members of S with the smallest (prio(t,b,id), id),
 *               stored ascending by id (R#7, R#10)
 *   off[t][b] = sum over b' < b of |kept(t,b')|   (the table's bucket offsets)
 * Table t's kept ids are written at kept_ids + t*n_rows (capacity n_rows per table).
 * addrs is [n_rows][L]; rows whose address is EMPTY are not inserted (R#15). */
int oracle_build(uint32_t L, uint32_t R, uint32_t range, uint64_t seed, const uint32_t *addrs,
                 const uint32_t *ids, uint64_t n_rows, uint32_t *arrivals, uint32_t *off,
                 uint32_t *kept_ids) {
    if (L == 0 || R == 0 || range == 0) return 1;
    oracle_seeds s;
    oracle_derive_seeds(seed, &s);
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t t = 0; t < (int64_t)L; ++t) {
        arrival *A = (arrival *)malloc(sizeof(arrival) * (n_rows ? n_rows : 1));
        uint64_t m = 0;
        for (uint64_t r = 0; r < n_rows; ++r) {
            uint32_t b = addrs[r * L + t];
            if (b == ORACLE_EMPTY) continue;
            if (b >= range) { bad = 1; continue; }
            uint64_t tb = oracle_mix64(s.s_prio ^ (((uint64_t)t << 32) | (uint64_t)b));
            A[m].b = b;
            A[m].prio = (uint32_t)(oracle_mix64(tb ^ (uint64_t)ids[r]) >> 32);
            A[m].id = ids[r];
            m++;
        }
        qsort(A, m, sizeof(arrival), cmp_arrival); /* group by bucket, then (prio, id) */
        uint32_t *arr = arrivals + (uint64_t)t * range;
        uint32_t *o = off + (uint64_t)t * ((uint64_t)range + 1);
        uint32_t *kept = kept_ids + (uint64_t)t * n_rows;
        memset(arr, 0, sizeof(uint32_t) * range);
        uint64_t i = 0, w = 0;
        for (uint32_t b = 0; b < range; ++b) {
            o[b] = (uint32_t)w;
            uint64_t j = i;
            while (j < m && A[j].b == b) j++;
            arr[b] = (uint32_t)(j - i);
            uint64_t keep = (j - i) < R ? (j - i) : R;
            for (uint64_t q = 0; q < keep; ++q) kept[w + q] = A[i + q].id;
            qsort(kept + w, keep, sizeof(uint32_t), cmp_u32); /* ascending id in the bucket */
            w += keep;
            i = j;
        }
        o[range] = (uint32_t)w;
        free(A);
    }
    return bad;
}

/* ------------------------------------------------------------------------- */
/* Querying phase (Alg. 3).                                       */
/* ------------------------------------------------------------------------- */

typedef struct { uint32_t id, count; } kvpair;

static int cmp_by_value(const void *x, const void *y) {
    const kvpair *a = (const kvpair *)x, *b = (const kvpair *)y;
    if (a->count != b->count) return a->count > b->count ? -1 : 1; /* count desc */
    return a->id < b->id ? -1 : (a->id > b->id);                    /* id asc */
}

/* For each query q (addresses q_addrs[q*L + t]):
 *   A = concatenation over tables t of kept(t, addr_t(q))            (Alg. 3 lines 4-7)
 *   KSELECT(A): SORTINPLACE(A); COUNTFREQUENCY(A) with full multiplicity (R#11);
 *   drop exclude[q] (R#14); SORTBYVALUE by (count desc, id asc) (R#12);
 *   return KVPair[0:k], padded with (EMPTY, 0) (R#13).
 * Tables: off [L][range+1] and kept_ids with per-table stride `table_stride`. */
int oracle_query(uint32_t L, uint32_t range, const uint32_t *off, const uint32_t *kept_ids,
                 uint64_t table_stride, const uint32_t *q_addrs, uint64_t n_q, uint32_t k,
                 const uint32_t *exclude, uint32_t *out_ids, uint32_t *out_counts) {
    if (L == 0 || range == 0 || k == 0) return 1;
    int bad = 0;
#pragma omp parallel
    {
        uint64_t cap = 1024;
        uint32_t *A = (uint32_t *)malloc(sizeof(uint32_t) * cap);
        kvpair *kv = (kvpair *)malloc(sizeof(kvpair) * cap);
#pragma omp for schedule(dynamic, 16)
        for (int64_t q = 0; q < (int64_t)n_q; ++q) {
            /* Initialize A; for each Table_i: Append A with Table_i[Key] */
            uint64_t m = 0;
            for (uint32_t t = 0; t < L; ++t) {
                uint32_t a = q_addrs[(uint64_t)q * L + t];
                if (a == ORACLE_EMPTY) continue;
                if (a >= range) { bad = 1; continue; }
                const uint32_t *o = off + (uint64_t)t * ((uint64_t)range + 1);
                const uint32_t *bucket = kept_ids + (uint64_t)t * table_stride;
                uint64_t len = o[a + 1] - o[a];
                if (m + len > cap) {
                    while (m + len > cap) cap *= 2;
                    A = (uint32_t *)realloc(A, sizeof(uint32_t) * cap);
                    kv = (kvpair *)realloc(kv, sizeof(kvpair) * cap);
                }
                memcpy(A + m, bucket + o[a], sizeof(uint32_t) * len);
                m += len;
            }
            /* KSELECT: SORTINPLACE(A) */
            qsort(A, m, sizeof(uint32_t), cmp_u32);
            /* COUNTFREQUENCY(A): one (key, multiplicity) pair per distinct key */
            uint64_t nkv = 0;
            for (uint64_t i = 0; i < m; ++i) {
                if (i > 0 && A[i] == A[i - 1]) { kv[nkv - 1].count++; continue; }
                kv[nkv].id = A[i];
                kv[nkv].count = 1;
                nkv++;
            }
            /* the query's own id never reports itself (k-NN graph, R#14) */
            if (exclude) {
                uint64_t w = 0;
                for (uint64_t i = 0; i < nkv; ++i)
                    if (kv[i].id != exclude[q]) kv[w++] = kv[i];
                nkv = w;
            }
            /* SORTBYVALUEINPLACE(KVPair); return KVPair[0:TopK] */
            qsort(kv, nkv, sizeof(kvpair), cmp_by_value);
            for (uint32_t j = 0; j < k; ++j) {
                out_ids[(uint64_t)q * k + j] = j < nkv ? kv[j].id : ORACLE_EMPTY;
                out_counts[(uint64_t)q * k + j] = j < nkv ? kv[j].count : 0u;
            }
        }
        free(A);
        free(kv);
    }
    return bad;
}

/* ------------------------------------------------------------------------- */
/* Reservoir sharing across tables (§3.2(4); §3.5, Fig. 3/4). */
/* ------------------------------------------------------------------------- */

/* The reservoir that table t's bucket b points to in a shared pool of P reservoirs
 * ("one shared chunk of reservoirs ... the pointer points to a randomly selected shared
 * reservoir"; "Allocated Range = F * Actual Range", so P = ceil(F*L*range)).
 * P = L*range (F = 1) is the unshared index: reservoir t*range + b.  Otherwise a keyed
 * hash of (t, b) reduced to [0, P) — a data-independent binding with the paper's law (a
 * uniformly random reservoir), so the index does not depend on insertion order (R#23). */
uint32_t oracle_reservoir(uint64_t seed, uint32_t t, uint32_t b, uint32_t L, uint32_t range, uint64_t P) {
    if (P == (uint64_t)L * range) return t * range + b;
    oracle_seeds s;
    oracle_derive_seeds(seed, &s);
    return mulhi_range(oracle_fmix32(oracle_fmix32(s.s_pool ^ t) ^ b), (uint32_t)P);
}

/* The distinct reservoirs of one row (addresses a[0..L)), in table order: a reservoir
 * that several of the row's tables point to is listed once (R#23).  Returns the count. */
static uint32_t row_reservoirs(uint64_t seed, const uint32_t *a, uint32_t L, uint32_t range, uint64_t P,
                               uint32_t *res, int *bad) {
    uint32_t n = 0;
    for (uint32_t t = 0; t < L; ++t) {
        if (a[t] == ORACLE_EMPTY) continue;
        if (a[t] >= range) { *bad = 1; continue; }
        uint32_t r = oracle_reservoir(seed, t, a[t], L, range, P);
        int dup = 0;
        for (uint32_t j = 0; j < n; ++j) dup |= res[j] == r;
        if (!dup) res[n++] = r;
    }
    return n;
}

/* Adding phase over a shared pool of P reservoirs.  For every reservoir r:
 *   S(r) = { id : r is one of the row's distinct reservoirs }   arrivals[r] = |S(r)|
 *   kept(r) = the min(|S|, R) members with the smallest (prio(r div range, r mod range, id), id),
 *             ascending id;  off[r] = sum over r' < r of |kept(r')|  (off has P+1 entries).
 * kept_ids needs n_rows*L entries.  P = L*range gives exactly oracle_build's tables laid out
 * table after table. */
int oracle_build_pool(uint32_t L, uint32_t R, uint32_t range, uint64_t P, uint64_t seed,
                      const uint32_t *addrs, const uint32_t *ids, uint64_t n_rows, uint32_t *arrivals,
                      uint32_t *off, uint32_t *kept_ids) {
    if (L == 0 || R == 0 || range == 0 || P == 0 || P > (uint64_t)L * range) return 1;
    oracle_seeds s;
    oracle_derive_seeds(seed, &s);
    int bad = 0;
    arrival *A = (arrival *)malloc(sizeof(arrival) * (n_rows * L + 1));
    uint32_t *res = (uint32_t *)malloc(sizeof(uint32_t) * (L + 1));
    uint64_t m = 0;
    for (uint64_t r = 0; r < n_rows; ++r) {
        uint32_t nr = row_reservoirs(seed, addrs + r * L, L, range, P, res, &bad);
        for (uint32_t j = 0; j < nr; ++j) {
            uint32_t v = res[j];
            uint64_t tb = oracle_mix64(s.s_prio ^ (((uint64_t)(v / range) << 32) | (uint64_t)(v % range)));
            A[m].b = v;
            A[m].prio = (uint32_t)(oracle_mix64(tb ^ (uint64_t)ids[r]) >> 32);
            A[m].id = ids[r];
            m++;
        }
    }
    qsort(A, m, sizeof(arrival), cmp_arrival); /* group by reservoir, then (prio, id) */
    uint64_t i = 0, w = 0;
    for (uint64_t v = 0; v < P; ++v) {
        off[v] = (uint32_t)w;
        uint64_t j = i;
        while (j < m && A[j].b == v) j++;
        arrivals[v] = (uint32_t)(j - i);
        uint64_t keep = (j - i) < R ? (j - i) : R;
        for (uint64_t q = 0; q < keep; ++q) kept_ids[w + q] = A[i + q].id;
        qsort(kept_ids + w, keep, sizeof(uint32_t), cmp_u32); /* ascending id (R#10) */
        w += keep;
        i = j;
    }
    off[P] = (uint32_t)w;
    free(A);
    free(res);
    return bad;
}

/* Querying phase over a shared pool: A = concatenation of kept(r) over the query's
 * DISTINCT reservoirs in table order (a shared reservoir is aggregated once, R#23), then
 * KSELECT exactly as oracle_query (full multiplicity, drop exclude, (count desc, id asc),
 * pad (EMPTY, 0)). */
int oracle_query_pool(uint32_t L, uint32_t range, uint64_t P, uint64_t seed, const uint32_t *off,
                      const uint32_t *kept_ids, const uint32_t *q_addrs, uint64_t n_q, uint32_t k,
                      const uint32_t *exclude, uint32_t *out_ids, uint32_t *out_counts) {
    if (L == 0 || range == 0 || k == 0 || P == 0) return 1;
    int bad = 0;
#pragma omp parallel
    {
        uint64_t cap = 1024;
        uint32_t *A = (uint32_t *)malloc(sizeof(uint32_t) * cap);
        kvpair *kv = (kvpair *)malloc(sizeof(kvpair) * cap);
        uint32_t *res = (uint32_t *)malloc(sizeof(uint32_t) * (L + 1));
#pragma omp for schedule(dynamic, 16)
        for (int64_t q = 0; q < (int64_t)n_q; ++q) {
            int lbad = 0;
            uint32_t nr = row_reservoirs(seed, q_addrs + (uint64_t)q * L, L, range, P, res, &lbad);
            if (lbad) bad = 1;
            uint64_t m = 0;
            for (uint32_t j = 0; j < nr; ++j) {
                uint64_t len = off[res[j] + 1] - off[res[j]];
                if (m + len > cap) {
                    while (m + len > cap) cap *= 2;
                    A = (uint32_t *)realloc(A, sizeof(uint32_t) * cap);
                    kv = (kvpair *)realloc(kv, sizeof(kvpair) * cap);
                }
                memcpy(A + m, kept_ids + off[res[j]], sizeof(uint32_t) * len);
                m += len;
            }
            qsort(A, m, sizeof(uint32_t), cmp_u32);
            uint64_t nkv = 0;
            for (uint64_t i = 0; i < m; ++i) {
                if (i > 0 && A[i] == A[i - 1]) { kv[nkv - 1].count++; continue; }
                kv[nkv].id = A[i];
                kv[nkv].count = 1;
                nkv++;
            }
            if (exclude) {
                uint64_t w = 0;
                for (uint64_t i = 0; i < nkv; ++i)
                    if (kv[i].id != exclude[q]) kv[w++] = kv[i];
                nkv = w;
            }
            qsort(kv, nkv, sizeof(kvpair), cmp_by_value);
            for (uint32_t j = 0; j < k; ++j) {
                out_ids[(uint64_t)q * k + j] = j < nkv ? kv[j].id : ORACLE_EMPTY;
                out_counts[(uint64_t)q * k + j] = j < nkv ? kv[j].count : 0u;
            }
        }
        free(A);
        free(kv);
        free(res);
    }
    return bad;
}

/* Full k-NN graph: insert ids 0..n-1 (Alg. 2), then query every row with its
 * own addresses and exclude = own id (Alg. 3).  Scratch is allocated here. */
int oracle_knn_graph(uint32_t K, uint32_t L, uint32_t R, uint32_t range, uint64_t seed,
                     const int64_t *row_ptr, const uint32_t *col_idx, uint64_t n_rows, uint32_t k,
                     uint32_t *out_ids, uint32_t *out_counts) {
    uint64_t B = (uint64_t)K * L;
    uint32_t *codes = (uint32_t *)malloc(sizeof(uint32_t) * (n_rows * B + 1));
    uint32_t *addrs = (uint32_t *)malloc(sizeof(uint32_t) * (n_rows * L + 1));
    uint32_t *ids = (uint32_t *)malloc(sizeof(uint32_t) * (n_rows + 1));
    uint32_t *arr = (uint32_t *)malloc(sizeof(uint32_t) * (uint64_t)L * range);
    uint32_t *off = (uint32_t *)malloc(sizeof(uint32_t) * (uint64_t)L * ((uint64_t)range + 1));
    uint32_t *kept = (uint32_t *)malloc(sizeof(uint32_t) * (n_rows * L + 1));
    int rc = 0;
    if (!codes || !addrs || !ids || !arr || !off || !kept) rc = 2;
    for (uint64_t r = 0; r < n_rows && !rc; ++r) ids[r] = (uint32_t)r;
    if (!rc) rc = oracle_doph(K, L, seed, row_ptr, col_idx, n_rows, codes);
    if (!rc) rc = oracle_addresses(K, L, range, seed, codes, n_rows, addrs);
    if (!rc) rc = oracle_build(L, R, range, seed, addrs, ids, n_rows, arr, off, kept);
    if (!rc) rc = oracle_query(L, range, off, kept, n_rows, addrs, n_rows, k, ids, out_ids, out_counts);
    free(codes); free(addrs); free(ids); free(arr); free(off); free(kept);
    return rc;
}

/* ------------------------------------------------------------------------- */
/* O-2: exact similarities (Eq. 2; Eq. 3), rows as sets.       */
/* ------------------------------------------------------------------------- */

/* Sorted, de-duplicated copy of every row (binary vectors are sets). */
static void normalize_rows(const int64_t *row_ptr, const uint32_t *col_idx, uint64_t n,
                           int64_t **rp_out, uint32_t **col_out) {
    int64_t base = row_ptr[0];
    uint64_t nnz = (uint64_t)(row_ptr[n] - base);
    uint32_t *tmp = (uint32_t *)malloc(sizeof(uint32_t) * (nnz + 1));
    memcpy(tmp, col_idx + base, sizeof(uint32_t) * nnz); /* absolute CSR indexing */
    int64_t *len = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t r = 0; r < (int64_t)n; ++r) {
        uint32_t *x = tmp + (row_ptr[r] - base);
        int64_t m = row_ptr[r + 1] - row_ptr[r];
        qsort(x, (size_t)m, sizeof(uint32_t), cmp_u32);
        int64_t w = 0;
        for (int64_t i = 0; i < m; ++i)
            if (i == 0 || x[i] != x[i - 1]) x[w++] = x[i];
        len[r] = w;
    }
    int64_t *rp = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
    rp[0] = 0;
    for (uint64_t r = 0; r < n; ++r) rp[r + 1] = rp[r] + len[r];
    uint32_t *col = (uint32_t *)malloc(sizeof(uint32_t) * ((uint64_t)rp[n] + 1));
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < (int64_t)n; ++r)
        memcpy(col + rp[r], tmp + (row_ptr[r] - base), sizeof(uint32_t) * (size_t)len[r]);
    free(tmp);
    free(len);
    *rp_out = rp;
    *col_out = col;
}

static uint64_t intersect(const uint32_t *a, uint64_t na, const uint32_t *b, uint64_t nb) {
    uint64_t i = 0, j = 0, c = 0;
    while (i < na && j < nb) {
        if (a[i] < b[j]) i++;
        else if (a[i] > b[j]) j++;
        else { c++; i++; j++; }
    }
    return c;
}

/* metric 0: Jaccard |x∩y| / (|x|+|y|-|x∩y|) (Eq. 2); metric 1: cosine |x∩y| / sqrt(|x||y|)
 * (Eq. 3).  Both 0 when undefined (empty vectors). */
static double similarity(uint64_t inter, uint64_t na, uint64_t nb, int metric) {
    if (metric == 0) {
        uint64_t u = na + nb - inter;
        return u ? (double)inter / (double)u : 0.0;
    }
    return (na && nb) ? (double)inter / sqrt((double)na * (double)nb) : 0.0;
}

int oracle_pair_similarity(const int64_t *row_ptr, const uint32_t *col_idx, uint64_t n,
                           const uint64_t *pairs /* [np][2] */, uint64_t np, int metric, double *out) {
    int64_t *rp;
    uint32_t *col;
    normalize_rows(row_ptr, col_idx, n, &rp, &col);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)np; ++i) {
        uint64_t x = pairs[2 * i], y = pairs[2 * i + 1];
        uint64_t nx = (uint64_t)(rp[x + 1] - rp[x]), ny = (uint64_t)(rp[y + 1] - rp[y]);
        out[i] = similarity(intersect(col + rp[x], nx, col + rp[y], ny), nx, ny, metric);
    }
    free(rp);
    free(col);
    return 0;
}

typedef struct { double sim; uint32_t id; } scored;
static int cmp_scored(const void *x, const void *y) {
    const scored *a = (const scored *)x, *b = (const scored *)y;
    if (a->sim != b->sim) return a->sim > b->sim ? -1 : 1; /* similarity desc */
    return a->id < b->id ? -1 : (a->id > b->id);            /* id asc */
}

/* Exact top-k neighbours of rows `queries` among all n rows (self excluded if asked),
 * ties by ascending id; padded with (EMPTY, -1). */
int oracle_bruteforce_topk(const int64_t *row_ptr, const uint32_t *col_idx, uint64_t n,
                           const uint64_t *queries, uint64_t nq, uint32_t k, int metric,
                           int exclude_self, uint32_t *out_ids, double *out_sim) {
    int64_t *rp;
    uint32_t *col;
    normalize_rows(row_ptr, col_idx, n, &rp, &col);
#pragma omp parallel
    {
        scored *S = (scored *)malloc(sizeof(scored) * (n + 1));
#pragma omp for schedule(dynamic, 1)
        for (int64_t qi = 0; qi < (int64_t)nq; ++qi) {
            uint64_t q = queries[qi];
            uint64_t nqq = (uint64_t)(rp[q + 1] - rp[q]);
            uint64_t m = 0;
            for (uint64_t x = 0; x < n; ++x) {
                if (exclude_self && x == q) continue;
                uint64_t nx = (uint64_t)(rp[x + 1] - rp[x]);
                S[m].sim = similarity(intersect(col + rp[q], nqq, col + rp[x], nx), nqq, nx, metric);
                S[m].id = (uint32_t)x;
                m++;
            }
            qsort(S, m, sizeof(scored), cmp_scored);
            for (uint32_t j = 0; j < k; ++j) {
                out_ids[qi * k + j] = j < m ? S[j].id : ORACLE_EMPTY;
                out_sim[qi * k + j] = j < m ? S[j].sim : -1.0;
            }
        }
        free(S);
    }
    free(rp);
    free(col);
    return 0;
}
