/*
 * synth/gen.c — seeded synthetic sparse-binary CSR generator.
 *
 * Shared by BOTH the CPU oracle tests and the CUDA path (the only shared module).
 * It holds none of FLASH's arithmetic: no DOPH, no address mapping, no priority
 * hash.  Its random numbers come from PCG32 (O'Neill 2014), a generator unrelated
 * to the method's hash functions.
 *
 * Recipe ("core + near-duplicate families"):
 *   - rows come in families; family size s = fam_min + Poisson(fam_extra);
 *   - a family root has n = round(LogNormal(mu, sigma)) features (clipped to
 *     [1, D]) with mu = ln(mean_nnz) - sigma^2/2 so that E[n] = mean_nnz;
 *     min(round(f_core*n), V_c) of them are drawn without replacement from a
 *     shared "core" vocabulary of V_c ids, the rest uniformly from the tail;
 *   - every other family member copies the root and replaces each feature,
 *     independently with probability mu_f, by a fresh uniform tail feature;
 *   - final row order is a seeded Fisher-Yates shuffle of family order.
 * Feature id space: vocabulary index j in [0, D) maps to col = (j*P + O) mod D
 * with gcd(P, D) = 1, so core ids are a pseudo-random subset of [0, D) and tail
 * ids never coincide with core ids.  Rows are multisets: a tail draw can repeat
 * (probability ~ n^2 / 2D per row); every consumer treats a row as a set.
 *
 * Determinism: row r's content depends only on (params, seed, r), never on the
 * thread count, so any row range can be generated independently (multi-GPU
 * ranks each generate their own shard).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    uint64_t N;          /* rows */
    uint64_t D;          /* dimensionality (feature ids in [0, D)) */
    double mean_nnz;     /* E[row length] before clipping */
    double sigma;        /* log-normal shape */
    double f_core;       /* fraction of a root's features drawn from the core */
    uint64_t V_c;        /* core vocabulary size (< D) */
    uint32_t fam_min;    /* minimum family size (>= 1) */
    double fam_extra;    /* Poisson mean of extra family members */
    double mu_f;         /* per-feature replacement probability for members */
    uint64_t seed;
    int32_t shuffle;     /* 1: seeded row shuffle; 0: family order */
} synth_params;

/* ---- PCG32 (XSH-RR), O'Neill 2014 ---- */
typedef struct { uint64_t state, inc; } pcg32;

static uint32_t pcg32_next(pcg32 *r) {
    uint64_t old = r->state;
    r->state = old * 6364136223846793005ULL + r->inc;
    uint32_t xorshifted = (uint32_t)(((old >> 18u) ^ old) >> 27u);
    uint32_t rot = (uint32_t)(old >> 59u);
    return (xorshifted >> rot) | (xorshifted << ((-rot) & 31));
}
static void pcg32_seed(pcg32 *r, uint64_t initstate, uint64_t stream) {
    r->state = 0u;
    r->inc = (stream << 1u) | 1u;
    pcg32_next(r);
    r->state += initstate;
    pcg32_next(r);
}
static double unif01(pcg32 *r) { /* 53-bit uniform in [0,1) */
    uint64_t a = pcg32_next(r) >> 5, b = pcg32_next(r) >> 6;
    return (double)(a * 67108864.0 + b) * (1.0 / 9007199254740992.0);
}
static uint64_t unif_below(pcg32 *r, uint64_t n) { /* uniform in [0, n), n <= 2^53 */
    return (uint64_t)(unif01(r) * (double)n);
}
static double gauss(pcg32 *r) { /* Box-Muller */
    double u1 = unif01(r), u2 = unif01(r);
    if (u1 < 1e-300) u1 = 1e-300;
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}
static uint32_t poisson(pcg32 *r, double lam) { /* Knuth, small lambda */
    double L = exp(-lam), p = 1.0;
    uint32_t k = 0;
    do { k++; p *= unif01(r); } while (p > L);
    return k - 1;
}
static uint64_t gcd64(uint64_t a, uint64_t b) { while (b) { uint64_t t = a % b; a = b; b = t; } return a; }

/* ---- family layout (sequential, cheap) ---- */
typedef struct {
    uint64_t N, F;
    uint32_t *fam_of;     /* family-order row -> family */
    uint64_t *fam_start;  /* family -> first family-order row */
    uint64_t *perm;       /* final row -> family-order row */
    uint64_t P, O;        /* vocabulary affine map */
} layout;

static void make_layout(const synth_params *p, layout *L) {
    pcg32 r; pcg32_seed(&r, p->seed, 0);
    L->N = p->N;
    L->fam_of = (uint32_t *)malloc(sizeof(uint32_t) * (p->N ? p->N : 1));
    uint64_t cap = 1024, F = 0, i = 0;
    L->fam_start = (uint64_t *)malloc(sizeof(uint64_t) * cap);
    while (i < p->N) {
        uint64_t s = p->fam_min + poisson(&r, p->fam_extra);
        if (s < 1) s = 1;
        if (F == cap) { cap *= 2; L->fam_start = (uint64_t *)realloc(L->fam_start, sizeof(uint64_t) * cap); }
        L->fam_start[F] = i;
        for (uint64_t m = 0; m < s && i < p->N; ++m) L->fam_of[i++] = (uint32_t)F;
        F++;
    }
    L->F = F;
    L->perm = (uint64_t *)malloc(sizeof(uint64_t) * (p->N ? p->N : 1));
    for (uint64_t j = 0; j < p->N; ++j) L->perm[j] = j;
    if (p->shuffle) {
        pcg32 q; pcg32_seed(&q, p->seed, 1);
        for (uint64_t j = p->N; j > 1; --j) {
            uint64_t k = unif_below(&q, j);
            uint64_t t = L->perm[j - 1]; L->perm[j - 1] = L->perm[k]; L->perm[k] = t;
        }
    }
    /* affine vocabulary map col = (j*P + O) mod D with gcd(P, D) = 1 */
    pcg32 a; pcg32_seed(&a, p->seed, 2);
    uint64_t D = p->D;
    uint64_t P = (D > 2) ? (unif_below(&a, D - 2) + 2) : 1;
    while (gcd64(P, D) != 1) P = (P + 1) % D ? (P + 1) % D : 1;
    L->P = P;
    L->O = D ? unif_below(&a, D) : 0;
}
static void free_layout(layout *L) { free(L->fam_of); free(L->fam_start); free(L->perm); }

static inline uint32_t vocab(const synth_params *p, const layout *L, uint64_t j) {
    return (uint32_t)(((unsigned __int128)j * L->P + L->O) % p->D);
}

static uint64_t root_len(const synth_params *p, uint64_t fam) {
    pcg32 r; pcg32_seed(&r, p->seed, 3 + 2 * (uint64_t)fam);
    double mu = log(p->mean_nnz) - 0.5 * p->sigma * p->sigma;
    double x = exp(mu + p->sigma * gauss(&r));
    double n = floor(x + 0.5);
    if (n < 1) n = 1;
    if (n > (double)p->D) n = (double)p->D;
    return (uint64_t)n;
}

/* writes the root's n features; `mark` is a zeroed scratch bitmap of V_c bits */
static void root_row(const synth_params *p, const layout *L, uint64_t fam, uint32_t *out,
                     uint64_t n, uint8_t *mark) {
    pcg32 r; pcg32_seed(&r, p->seed, 3 + 2 * (uint64_t)fam);
    (void)gauss(&r); /* same draw root_len consumed */
    uint64_t c = (uint64_t)floor(p->f_core * (double)n + 0.5);
    if (c > p->V_c) c = p->V_c;
    if (c > n) c = n;
    /* Floyd's algorithm: c distinct values from [0, V_c) */
    uint64_t w = 0;
    for (uint64_t j = p->V_c - c; j < p->V_c; ++j) {
        uint64_t t = unif_below(&r, j + 1);
        uint64_t pick = (mark[t >> 3] >> (t & 7)) & 1 ? j : t;
        mark[pick >> 3] |= (uint8_t)(1u << (pick & 7));
        out[w++] = vocab(p, L, pick);
    }
    memset(mark, 0, (size_t)((p->V_c + 7) / 8)); /* scratch back to all-zero */
    for (; w < n; ++w) out[w] = vocab(p, L, p->V_c + unif_below(&r, p->D - p->V_c));
}

static void member_mutate(const synth_params *p, const layout *L, uint64_t fo_row, uint32_t *row, uint64_t n) {
    pcg32 r; pcg32_seed(&r, p->seed, 3 + 2 * (uint64_t)L->F + 2 * fo_row + 1);
    for (uint64_t q = 0; q < n; ++q)
        if (unif01(&r) < p->mu_f) row[q] = vocab(p, L, p->V_c + unif_below(&r, p->D - p->V_c));
}

/* Row lengths of final rows [r0, r1): len[i] for row r0+i. Returns 0 on success. */
int synth_row_lengths(const synth_params *p, uint64_t r0, uint64_t r1, int64_t *len) {
    if (r1 < r0 || r1 > p->N || p->V_c >= p->D) return 1;
    layout L; make_layout(p, &L);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)(r1 - r0); ++i) {
        uint64_t fo = L.perm[r0 + i];
        len[i] = (int64_t)root_len(p, L.fam_of[fo]);
    }
    free_layout(&L);
    return 0;
}

/* Fill rows [r0, r1) into col_idx using row_ptr (row_ptr[0] may be nonzero; it is
 * used as an absolute offset into col_idx, i.e. col_idx[row_ptr[i] - row_ptr[0]]). */
int synth_fill(const synth_params *p, uint64_t r0, uint64_t r1, const int64_t *row_ptr, uint32_t *col_idx) {
    if (r1 < r0 || r1 > p->N || p->V_c >= p->D) return 1;
    layout L; make_layout(p, &L);
    size_t mark_bytes = (size_t)((p->V_c + 7) / 8);
#pragma omp parallel
    {
        uint8_t *mark = (uint8_t *)calloc(mark_bytes ? mark_bytes : 1, 1);
#pragma omp for schedule(dynamic, 256)
        for (int64_t i = 0; i < (int64_t)(r1 - r0); ++i) {
            uint64_t fo = L.perm[r0 + i];
            uint64_t fam = L.fam_of[fo];
            uint64_t n = root_len(p, fam);
            uint32_t *row = col_idx + (row_ptr[i] - row_ptr[0]);
            root_row(p, &L, fam, row, n, mark);
            if (fo != L.fam_start[fam]) member_mutate(p, &L, fo, row, n);
        }
        free(mark);
    }
    free_layout(&L);
    return 0;
}

/* Family id of final rows [r0, r1) (ground truth for planted-neighbour checks). */
int synth_family_of(const synth_params *p, uint64_t r0, uint64_t r1, uint64_t *fam) {
    if (r1 < r0 || r1 > p->N) return 1;
    layout L; make_layout(p, &L);
    for (uint64_t i = r0; i < r1; ++i) fam[i - r0] = L.fam_of[L.perm[i]];
    free_layout(&L);
    return 0;
}
