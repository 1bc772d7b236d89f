/*
 * oracle/gace_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU definition of the GACE Measurement
 * Engine's selectivity probe (arxiv 2512.19750, §III-B "Measurement
 * Engine", §III-C Eq. 1-3; probe semantics fixed in SURVEY.md §8(c) steps 1-6
 * and DESIGN.md "Readings").  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or constant generator with the CUDA product
 * under paper_2512_19750_b200/ and include/ (the record layouts and op codes
 * below are restated from the interface, not included).
 *
 * Every output is the definition evaluated row by row, with each predicate
 * evaluated by its operator exactly as written (no interval normalisation, no
 * bucketing, no breakpoint tables).  The only re-ordering is OpenMP
 * partitioning of the rows: each thread keeps its own integer counters and
 * registers and they are merged by exact integer sum / max at the end.
 *
 * Pinned by tests/test_oracle_*.py against: JDK SplittableRandom and
 * MurmurHash3 known answers, a pure-Python brute force (oracle/reference.py)
 * over exhaustive tiny tables, closed forms and invariants.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* interface record layouts (gace_pred / gace_pair, 24 B and 8 B) */
typedef struct { uint32_t col; uint16_t op; uint16_t flags; int64_t a; int64_t b; } or_pred;
typedef struct { uint32_t i; uint32_t j; } or_pair;

enum { OR_EQ = 0, OR_LT = 1, OR_LE = 2, OR_GT = 3, OR_GE = 4, OR_BETWEEN = 5 };
enum { OR_NEGATE = 1 };
enum { OR_I32 = 0, OR_I64 = 1 };

#define OR_GAMMA 0x9E3779B97F4A7C15ULL

/* SplitMix64 finaliser (Steele, Lea, Flood 2014; JDK SplittableRandom.mix64). */
uint64_t oracle_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* u(seed, r): the (r+1)-th output of SplitMix64 seeded with `seed`. */
uint64_t oracle_u(uint64_t seed, uint64_t r) {
    return oracle_mix64(seed + (r + 1) * OR_GAMMA);
}

/* SURVEY §8(c).2 / reading L8: T = floor(rate * 2^64) for 0 <= rate < 1. */
uint64_t oracle_threshold(double rate) {
    return (uint64_t)ldexp(rate, 64);
}

/* keep(r) = 1 if rate == 1, else u(seed, r) < T. */
int oracle_keep(double rate, uint64_t seed, uint64_t r) {
    if (rate == 1.0) return 1;
    return oracle_u(seed, r) < oracle_threshold(rate);
}

/* MurmurHash3 fmix32 (= MurmurHash3_x86_32 of the empty key with seed h). */
uint32_t oracle_fmix32(uint32_t h) {
    h ^= h >> 16;
    h *= 0x85EBCA6BU;
    h ^= h >> 13;
    h *= 0xC2B2AE35U;
    h ^= h >> 16;
    return h;
}

static int clz32(uint32_t x) { int n = 0; while (n < 32 && !(x & 0x80000000U)) { x <<= 1; n++; } return n; }
static int clz64(uint64_t x) { int n = 0; while (n < 64 && !(x & 0x8000000000000000ULL)) { x <<= 1; n++; } return n; }

/* HLL (index, rank) of one int32 key: top p bits of fmix32 = index; rank = leading zeros of
 * the remaining 32-p bits + 1, or 32-p+1 if they are all zero (reading L3). */
void oracle_hll_i32(int32_t x, int p, uint32_t *idx, uint32_t *rank) {
    uint32_t h = oracle_fmix32((uint32_t)x);
    uint32_t w = h << p;
    *idx = h >> (32 - p);
    *rank = (w == 0) ? (uint32_t)(32 - p + 1) : (uint32_t)(clz32(w) + 1);
}

/* int64 key: h = mix64(x + gamma) (= first SplittableRandom(x).nextLong()). */
void oracle_hll_i64(int64_t x, int p, uint32_t *idx, uint32_t *rank) {
    uint64_t h = oracle_mix64((uint64_t)x + OR_GAMMA);
    uint64_t w = h << p;
    *idx = (uint32_t)(h >> (64 - p));
    *rank = (w == 0) ? (uint32_t)(64 - p + 1) : (uint32_t)(clz64(w) + 1);
}

/* SURVEY §8(c).4 / SPEC.md S:45 operators; reading L9/L10: exact signed int64 compare. */
int oracle_pred(const or_pred *p, int64_t v) {
    int t;
    switch (p->op) {
        case OR_EQ: t = (v == p->a); break;
        case OR_LT: t = (v < p->a); break;
        case OR_LE: t = (v <= p->a); break;
        case OR_GT: t = (v > p->a); break;
        case OR_GE: t = (v >= p->a); break;
        case OR_BETWEEN: t = (p->a <= v && v <= p->b); break;
        default: return -1;
    }
    if (p->flags & OR_NEGATE) t = !t;
    return t;
}

static int64_t col_value(const void *col, int dtype, uint64_t r) {
    if (dtype == OR_I32) return (int64_t)((const int32_t *)col)[r];
    return ((const int64_t *)col)[r];
}

/*
 * The probe over rows [0, nrows) of a table shard whose first row has global id row_offset.
 *   n_sampled            = sum_r keep(r)
 *   counts[p]            = sum_r keep(r) * pred_p(x_{col_p}[r])
 *   joints[q]            = sum_r keep(r) * pred_{i_q}(row r) * pred_{j_q}(row r)
 *   regs[k][idx]         = max over kept rows of rank, for the k-th column of hll_col_mask
 *                          (ascending column order), 2^p registers each, starting at 0.
 * Returns 0, or -1 on an invalid argument (nothing written).
 */
int oracle_probe(const void *const *cols, const int *dtypes, uint32_t ncols,
                 uint64_t nrows, uint64_t row_offset,
                 const or_pred *preds, uint32_t npreds,
                 const or_pair *pairs, uint32_t npairs,
                 double rate, uint64_t seed, uint64_t hll_col_mask, int hll_p, int nthreads,
                 uint64_t *n_sampled, uint64_t *counts, uint64_t *joints, uint8_t *regs) {
    if (!(rate >= 0.0 && rate <= 1.0)) return -1;
    if (hll_p < 4 || hll_p > 16) return -1;
    if (ncols > 64) return -1;
    for (uint32_t p = 0; p < npreds; p++) {
        if (preds[p].col >= ncols || preds[p].op > OR_BETWEEN) return -1;
    }
    for (uint32_t q = 0; q < npairs; q++) {
        if (pairs[q].i >= npreds || pairs[q].j >= npreds) return -1;
    }
    uint32_t hll_cols[64];
    uint32_t nh = 0;
    for (uint32_t c = 0; c < ncols; c++)
        if (hll_col_mask & (1ULL << c)) hll_cols[nh++] = c;
    if (ncols < 64 && (hll_col_mask >> ncols)) return -1;
    const uint64_t m = 1ULL << hll_p;

    uint64_t total = 0;
    memset(counts, 0, sizeof(uint64_t) * npreds);
    memset(joints, 0, sizeof(uint64_t) * npairs);
    if (nh) memset(regs, 0, nh * m);

#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#else
    nthreads = 1;
#endif
    int err = 0;
#pragma omp parallel num_threads(nthreads) reduction(+ : total)
    {
        uint64_t *my_counts = calloc(npreds ? npreds : 1, sizeof(uint64_t));
        uint64_t *my_joints = calloc(npairs ? npairs : 1, sizeof(uint64_t));
        uint8_t *my_regs = calloc(nh ? nh * m : 1, 1);
        unsigned char *bit = calloc(npreds ? npreds : 1, 1);
        if (!my_counts || !my_joints || !my_regs || !bit) {
#pragma omp atomic write
            err = 1;
        } else {
#pragma omp for schedule(static)
            for (int64_t rr = 0; rr < (int64_t)nrows; rr++) {
                uint64_t r = (uint64_t)rr;
                uint64_t g = row_offset + r;                     /* global row id (reading L7) */
                if (!oracle_keep(rate, seed, g)) continue;
                total += 1;
                for (uint32_t p = 0; p < npreds; p++) {
                    int64_t v = col_value(cols[preds[p].col], dtypes[preds[p].col], r);
                    bit[p] = (unsigned char)oracle_pred(&preds[p], v);
                    my_counts[p] += bit[p];
                }
                for (uint32_t q = 0; q < npairs; q++)
                    my_joints[q] += (uint64_t)(bit[pairs[q].i] & bit[pairs[q].j]);
                for (uint32_t k = 0; k < nh; k++) {
                    uint32_t c = hll_cols[k], idx, rank;
                    if (dtypes[c] == OR_I32)
                        oracle_hll_i32(((const int32_t *)cols[c])[r], hll_p, &idx, &rank);
                    else
                        oracle_hll_i64(((const int64_t *)cols[c])[r], hll_p, &idx, &rank);
                    if (rank > my_regs[k * m + idx]) my_regs[k * m + idx] = (uint8_t)rank;
                }
            }
#pragma omp critical
            {
                for (uint32_t p = 0; p < npreds; p++) counts[p] += my_counts[p];
                for (uint32_t q = 0; q < npairs; q++) joints[q] += my_joints[q];
                for (uint64_t i = 0; i < nh * m; i++)
                    if (my_regs[i] > regs[i]) regs[i] = my_regs[i];
            }
        }
        free(my_counts);
        free(my_joints);
        free(my_regs);
        free(bit);
    }
    if (err) return -1;
    *n_sampled = total;
    return 0;
}

/* Bit-packed sample mask of rows [0, nrows): bit (r % 64) of word r / 64 = keep(row_offset + r). */
int oracle_sample_mask(uint64_t nrows, uint64_t row_offset, double rate, uint64_t seed, uint64_t *bits) {
    if (!(rate >= 0.0 && rate <= 1.0)) return -1;
    memset(bits, 0, sizeof(uint64_t) * ((nrows + 63) / 64));
    for (uint64_t r = 0; r < nrows; r++)
        if (oracle_keep(rate, seed, row_offset + r)) bits[r / 64] |= 1ULL << (r % 64);
    return 0;
}

/*
 * Candidate-set conjunction counts (§IV-H "Experiment D: Replacing Dynamic
 * Sampling (Key-Only + Bitmask)", lines 250-270: M candidate predicate sets of K
 * predicates each; SPEC.md evaluate_bitmasks: "per-set count = popcount of AND-ed
 * bitmaps").  Over rows [0, nrows) of a shard whose first row has global id row_offset:
 *   set_counts[m] = sum_r keep(r) * prod_{p in members(m)} pred_p(row r)
 * members(m) = set_members[set_offsets[m] .. set_offsets[m+1]); an empty set counts every
 * kept row.  Each member predicate is evaluated by its operator as written, per row and per
 * set (no sharing, no bucketing).  Returns 0, or -1 on an invalid argument.
 */
int oracle_probe_sets(const void *const *cols, const int *dtypes, uint32_t ncols,
                      uint64_t nrows, uint64_t row_offset,
                      const or_pred *preds, uint32_t npreds,
                      const uint32_t *set_offsets, const uint32_t *set_members, uint32_t nsets,
                      double rate, uint64_t seed, int nthreads,
                      uint64_t *n_sampled, uint64_t *set_counts) {
    if (!(rate >= 0.0 && rate <= 1.0)) return -1;
    if (ncols > 64) return -1;
    for (uint32_t p = 0; p < npreds; p++)
        if (preds[p].col >= ncols || preds[p].op > OR_BETWEEN) return -1;
    if (nsets && set_offsets[0] != 0) return -1;
    for (uint32_t m = 0; m < nsets; m++) {
        if (set_offsets[m + 1] < set_offsets[m]) return -1;
        for (uint32_t k = set_offsets[m]; k < set_offsets[m + 1]; k++)
            if (set_members[k] >= npreds) return -1;
    }
    memset(set_counts, 0, sizeof(uint64_t) * nsets);
    uint64_t total = 0;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#else
    nthreads = 1;
#endif
    int err = 0;
#pragma omp parallel num_threads(nthreads) reduction(+ : total)
    {
        uint64_t *my = calloc(nsets ? nsets : 1, sizeof(uint64_t));
        if (!my) {
#pragma omp atomic write
            err = 1;
        } else {
#pragma omp for schedule(static)
            for (int64_t rr = 0; rr < (int64_t)nrows; rr++) {
                uint64_t r = (uint64_t)rr;
                if (!oracle_keep(rate, seed, row_offset + r)) continue;
                total += 1;
                for (uint32_t m = 0; m < nsets; m++) {
                    int all = 1;
                    for (uint32_t k = set_offsets[m]; k < set_offsets[m + 1] && all; k++) {
                        const or_pred *p = &preds[set_members[k]];
                        all = oracle_pred(p, col_value(cols[p->col], dtypes[p->col], r));
                    }
                    my[m] += (uint64_t)all;
                }
            }
#pragma omp critical
            {
                for (uint32_t m = 0; m < nsets; m++) set_counts[m] += my[m];
            }
        }
        free(my);
    }
    if (err) return -1;
    *n_sampled = total;
    return 0;
}
