/*
 * gace.h -- C-ABI of the B200-native GACE selectivity probe.
 *
 * What it computes: the Measurement Engine's probe (arxiv 2512.19750,
 * PAPER.md §III-B "Measurement Engine (GPU-based Probing)", lines 54-55, and
 * §IV-H "Key-Only + Bitmask", lines 250-251): one key-only pass over columnar
 * int32 / int64 keys, optionally Bernoulli-sampled by a seeded per-row hash,
 * producing per-predicate match counts, pairwise joint counts (the P(A,B) of
 * PCS, Eq. 3, lines 73-78) and per-column HyperLogLog registers (the NDV_est
 * of the drift D, Eq. 1, lines 60-65).  Exact semantics: DESIGN.md
 * "Semantics" (= SURVEY.md §8(c) steps 1-8) and the readings listed there.
 *
 * Conventions (all calls):
 *  - Every call returns gace_status.  On any non-OK status no output is
 *    written (all validation happens before any launch); gace_last_error()
 *    returns a thread-local message.  No C++ exception crosses this ABI.
 *  - Host pointers are read only during the call.  Device pointers are
 *    borrowed, never freed.  The library owns all scratch it allocates.
 *  - No CPU fallback: without a usable CUDA device attach fails with
 *    GACE_ECUDA.  gace_derive / gace_gate are host-only (no device needed).
 */
#ifndef GACE_H_
#define GACE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GACE_OK = 0,
    GACE_EINVAL = 1,        /* invalid argument (NULL, range, alignment, index)          */
    GACE_ENOMEM = 2,        /* device / pinned allocation failed                         */
    GACE_ECUDA = 3,         /* CUDA runtime error, or no CUDA device                     */
    GACE_ENCCL = 4,         /* NCCL unavailable or failed                                */
    GACE_EHANDLE = 5,       /* NULL or already-detached table handle                     */
    GACE_EUNSUPPORTED = 6   /* legal request outside this build's limits (see below)     */
} gace_status;

typedef enum { GACE_I32 = 0, GACE_I64 = 1 } gace_dtype;

/* Predicate operators (=, <, <=, >, >=, BETWEEN; reading L9).
 * Comparison is exact signed int64: v = (int64)x[r] against int64 bounds, also
 * on int32 columns, so bounds outside the column dtype are legal (L10).        */
typedef enum {
    GACE_EQ = 0,            /* v == a                                                    */
    GACE_LT = 1,            /* v <  a                                                    */
    GACE_LE = 2,            /* v <= a                                                    */
    GACE_GT = 3,            /* v >  a                                                    */
    GACE_GE = 4,            /* v >= a                                                    */
    GACE_BETWEEN = 5        /* a <= v && v <= b  (inclusive; a > b is the empty predicate) */
} gace_op;

#define GACE_PRED_NEGATE 1u /* flags bit: logical NOT of the operator (gives !=, NOT BETWEEN) */

/* One candidate predicate, 24 bytes.  `b` is read for BETWEEN only. */
typedef struct {
    uint32_t col;           /* column index into the attached table, < ncols             */
    uint16_t op;            /* gace_op                                                   */
    uint16_t flags;         /* 0 or GACE_PRED_NEGATE                                     */
    int64_t a;
    int64_t b;
} gace_pred;

/* A pair flagged for a correlation check: joint = #{sampled rows where predicates
 * i and j both hold} (reading L18: i == j, same-column pairs, duplicates allowed). */
typedef struct {
    uint32_t i, j;          /* indices into the predicate batch, < npreds                */
} gace_pair;

/* Multi-GPU description: rows are sharded contiguously, one
 * process per GPU.  row_offset = global id of this shard's first row (reading
 * L7: the sample bit uses global row ids, so results are shard-invariant);
 * row_offset + nrows_local <= nrows_total (GACE_EINVAL otherwise).
 * Either nccl_unique_id (128 bytes from ncclGetUniqueId on rank 0, broadcast by
 * the caller) or an existing nccl_comm (ncclComm_t, not destroyed by detach).
 * With either, results are merged over NCCL at any nranks (1 included); with
 * neither (nranks must then be 1) the table is a plain single-GPU table with an
 * offset.  An NCCL table's attach is collective: the ranks all-reduce their
 * shards' per-column minima / maxima so every rank plans over the same global
 * value domains, and -- when the loaded libnccl has the 2.28 device API and every
 * rank is NVLink load/store reachable -- register a 128 KB symmetric window per
 * rank for the fused merge (§IV-B "Reduction"; SURVEY.md §8(f) NEXT-2b;
 * GACE_NCCL_FUSED=0 keeps the grouped all-reduce).  Its detach is collective too.
 * Waits on an NCCL table poll ncclCommGetAsyncError: an asynchronous error, or no
 * progress within GACE_NCCL_TIMEOUT_MS (default 300000), aborts the communicator
 * and returns GACE_ENCCL (the table cannot merge again; detach it).  */
typedef struct {
    int rank;
    int nranks;
    uint64_t row_offset;
    uint64_t nrows_total;
    const void *nccl_unique_id;
    void *nccl_comm;
} gace_dist;

typedef struct gace_table gace_table;   /* opaque */

/* Limits of this build (GACE_EINVAL beyond the first three, GACE_EUNSUPPORTED beyond
 * the rest):  ncols <= 64; npreds <= 4096; npairs <= 4096; hll_p == 12; at most 8
 * distinct probed columns (columns referenced by a predicate or by hll_col_mask)
 * per gace_probe call; the per-probe plan must fit one CTA's shared memory.     */
#define GACE_MAX_COLS 64
#define GACE_MAX_PREDS 4096
#define GACE_MAX_PAIRS 4096
#define GACE_MAX_PROBED_COLS 8
#define GACE_HLL_P 12

/*
 * Attach a device-resident table.
 *   col_dev_ptrs[c]  device pointer to nrows_local values of column c, dtype dtypes[c],
 *                    16-byte aligned (GACE_EINVAL otherwise).  Borrowed: must stay valid
 *                    and unmodified until detach.  Column-major, one array per column.
 *   dist             NULL = single GPU, row_offset 0; else gace_dist above (collective:
 *                    every rank calls attach; NCCL comm created here if an id is given).
 *   device           CUDA device ordinal.
 *   cuda_stream      cudaStream_t all work is issued on, including the attach-time pass
 *                    below: pass the stream that produced the columns (NULL = a
 *                    library-owned stream, which is NOT ordered after other streams -- the
 *                    caller must then have synchronised the columns before attach).
 * One-time work: a min/max pass per column (the table is immutable while attached); the
 * lookup tables are built over that domain, so columns still being written at attach
 * give wrong results, not an error.
 */
gace_status gace_table_attach(const void *const *col_dev_ptrs, const gace_dtype *dtypes,
                              uint32_t ncols, uint64_t nrows_local, const gace_dist *dist,
                              int device, void *cuda_stream, gace_table **out);

/*
 * Attach a HOST-resident table (§IV-B Exp. A "Key-only = True": the keys cross
 * PCIe on every probe).  col_host_ptrs[c] are host arrays (pinned for full speed);
 * every gace_probe streams the probed columns to the device in chunks on a copy
 * stream, overlapped with the scan of the previous chunk.  Same ownership rules.
 */
gace_status gace_table_attach_host(const void *const *col_host_ptrs, const gace_dtype *dtypes,
                                   uint32_t ncols, uint64_t nrows_local, const gace_dist *dist,
                                   int device, void *cuda_stream, gace_table **out);

/* Free everything the library allocated for t (never the borrowed columns; never a
 * caller-passed communicator).  Collective for a table attached with NCCL. */
gace_status gace_table_detach(gace_table *t);

/*
 * CUDA-graph replay of repeated probes (graph half; BJ:5-11: the
 * probe's fixed per-call cost).  enable != 0: on a device table attached on a non-default
 * stream with one rank, the second gace_probe with the same plan (predicates, pairs, HLL
 * mask), sample_rate, seed and scratch buffers captures the probe's device work (memsets,
 * scan, finalize, result D2H, stage events) into one graph; later identical calls launch
 * that graph.  Results are the same as without graphs (the same kernels run); host tables,
 * multi-rank tables and the legacy default stream always run eagerly.  enable == 0 frees
 * the graph.  Default: disabled.  Errors: GACE_EHANDLE on an invalid handle.
 * gace_table_graph_stats: captures and replays so far (either pointer may be NULL).
 */
gace_status gace_table_set_graphs(gace_table *t, int enable);
gace_status gace_table_graph_stats(const gace_table *t, uint64_t *captures, uint64_t *replays);

/*
 * The probe (north star: counts, joint_counts, hll_regs).
 *   preds[npreds], pairs[npairs]   host arrays (validated before any launch)
 *   sample_rate                    in [0,1]; 1 = every row (NaN / out of range: EINVAL)
 *   seed                           sample seed: keep(r) = u(seed,r) < floor(rate*2^64),
 *                                  u = (r+1)-th SplitMix64 output (reading L6/L8)
 *   hll_col_mask                   bit c = HLL over column c (< ncols)
 *   hll_p                          must be 12 (GACE_EUNSUPPORTED otherwise)
 * Outputs (host, caller-allocated; merged over all ranks when attached with dist):
 *   *n_sampled                     number of kept rows
 *   counts[npreds]                 count[p] = #{kept r : pred_p(x[r])}
 *   joint_counts[npairs]           may be NULL iff npairs == 0
 *   hll_regs[popcount(mask)][4096] u8 registers, ascending column order; may be NULL
 *                                  iff mask == 0 (sampled rows only, reading L4)
 * Synchronous: returns once the results are in host memory.  One probe in flight per
 * handle.  Collective over ranks when attached with NCCL (identical arguments): a batch
 * new to the table is agreed on first (all-reduce of the ranks' planning status and a
 * hash of the batch), so a batch no rank can plan fails on every rank (its own status),
 * and ranks passing different batches all get GACE_EINVAL -- none enters a merge the
 * others would not join.
 */
gace_status gace_probe(gace_table *t, const gace_pred *preds, uint32_t npreds,
                       const gace_pair *pairs, uint32_t npairs, double sample_rate,
                       uint64_t seed, uint64_t hll_col_mask, uint32_t hll_p,
                       uint64_t *n_sampled, uint64_t *counts, uint64_t *joint_counts,
                       uint8_t *hll_regs);

/*
 * Candidate-set conjunction counts (§IV-H "Experiment D: Replacing Dynamic
 * Sampling (Key-Only + Bitmask)", lines 250-270: M candidate sets of K predicates; SPEC.md
 * evaluate_bitmasks: "per-set count = popcount of AND-ed bitmaps").
 *   preds[npreds]                  host array, validated as for gace_probe
 *   set_offsets[nsets + 1]         CSR offsets into set_members (set_offsets[0] == 0,
 *                                  non-decreasing); set m = set_members[off[m] .. off[m+1])
 *   set_members[set_offsets[nsets]] predicate indices (< npreds); duplicates allowed;
 *                                  an empty set holds on every row
 *   sample_rate, seed              the sample of gace_probe (same rows for the same rate/seed)
 * Outputs (host, caller-allocated; merged over ranks when attached with dist):
 *   *n_sampled                     number of kept rows
 *   set_counts[nsets]              #{kept r : every member predicate of set m holds on row r}
 * Limits: nsets <= GACE_MAX_SETS, members <= GACE_MAX_SET_MEMBERS (GACE_EUNSUPPORTED
 * beyond); members on at most 8 distinct columns; device tables only (GACE_EUNSUPPORTED
 * for host tables); the plan must fit one CTA's shared memory (GACE_EUNSUPPORTED).
 * Synchronous; one call in flight per handle; collective over ranks with dist.
 * gace_last_timing reports it like a probe (scan_ms = the set kernel).
 */
#define GACE_MAX_SETS 256
#define GACE_MAX_SET_MEMBERS 65536
gace_status gace_probe_sets(gace_table *t, const gace_pred *preds, uint32_t npreds,
                            const uint32_t *set_offsets, const uint32_t *set_members, uint32_t nsets,
                            double sample_rate, uint64_t seed, uint64_t *n_sampled,
                            uint64_t *set_counts);

/*
 * Est.CV vs budget (§IV-C "Experiment B: Estimation Stability (Est.CV vs. Budget)",
 * lines 121-141): run the probe once per seed
 * (nseeds >= 2, same batch and sample_rate) and report, per predicate, the coefficient of
 * variation CV = sample standard deviation (R - 1) / mean over the seeds of S_p = count/n;
 * per pair, the CV of the joint selectivity J/n and of PCS (Eq. 3).  A mean of 0 or a NaN
 * estimate (n = 0, zero marginal) gives NaN.  Outputs are host arrays [npreds] / [npairs];
 * cv_joint / cv_pcs may be NULL iff npairs == 0.  Collective with dist, like gace_probe.
 */
gace_status gace_estimate_cv(gace_table *t, const gace_pred *preds, uint32_t npreds,
                             const gace_pair *pairs, uint32_t npairs, double sample_rate,
                             const uint64_t *seeds, uint32_t nseeds, double *cv_sel,
                             double *cv_joint, double *cv_pcs);

/*
 * Probe cache (§V item 3, line 314: "Probing results should be cached by bind value
 * (or value range) to amortize the measurement cost across subsequent queries"; SPEC.md
 * S:354-403).  Host-only; thread-safe (one mutex per cache).
 * Key: table_id + the conjunction's predicates normalised as (col, op, flags, bind bucket of
 * a, bind bucket of b for BETWEEN), sorted and de-duplicated -- A and B == B and A.  Bind
 * bucket: with range_buckets > 0 and a domain [lo, hi] per predicate (domains[2i], [2i+1]),
 * the equal-width bucket of the bind (-1 below lo, range_buckets above hi); otherwise the
 * exact bind.  Capacity (0 = 4096 entries): least recently inserted evicted first.
 */
typedef struct {
    double s_probe;         /* measured selectivity, in [0, 1] (put: GACE_EINVAL otherwise) */
    uint64_t count;         /* matching sampled rows                                      */
    uint64_t n_sampled;     /* sample size used                                           */
    uint64_t hits;          /* lookups that returned this entry (put resets it)            */
} gace_cache_entry;
typedef struct gace_cache gace_cache;

gace_status gace_cache_create(uint32_t capacity, uint32_t range_buckets, gace_cache **out);
gace_status gace_cache_destroy(gace_cache *c);
/* Insert or replace (a replaced entry moves to the back of the eviction order). */
gace_status gace_cache_put(gace_cache *c, uint64_t table_id, const gace_pred *conj, uint32_t k,
                           const int64_t *domains, const gace_cache_entry *entry);
/* *hit = 1 and *entry (may be NULL) = the stored entry with its hit count incremented, or
 * *hit = 0 on a miss. */
gace_status gace_cache_lookup(gace_cache *c, uint64_t table_id, const gace_pred *conj, uint32_t k,
                              const int64_t *domains, gace_cache_entry *entry, uint32_t *hit);
/* Drop every entry of table_id (the table was mutated). */
gace_status gace_cache_invalidate(gace_cache *c, uint64_t table_id);
gace_status gace_cache_stats(gace_cache *c, uint64_t *hits, uint64_t *misses, uint64_t *evictions,
                             uint64_t *size);

/* Test hook: the deterministic sample mask of this shard's rows, bit-packed:
 * bit (r % 64) of bits[r / 64] = keep(row_offset + r); bits has ceil(nrows_local/64)
 * words (host).  Device tables only.                                               */
gace_status gace_sample_mask(gace_table *t, double sample_rate, uint64_t seed, uint64_t *bits);

/*
 * Derived doubles (host only, Eq. 1-3):
 *   sel[p]     = counts[p] / n_sampled                   (NaN when n_sampled == 0)
 *   pcs[q]     = (J/n) / ((A/n) * (B/n))                 (NaN when n == 0 or A*B == 0)
 *   ndv_est[c] = HLL estimate of regs[c] (raw, linear counting when E <= 2.5m and V > 0)
 *   drift[c]   = |ndv_hist[c] - ndv_est[c]| / ndv_hist[c] (ndv_hist[c] <= 0: EINVAL)
 * Any of the output arrays may be NULL (not computed).  regs may be NULL iff
 * ncols_hll == 0; ndv_hist may be NULL iff drift is NULL.
 */
gace_status gace_derive(uint64_t n_sampled, const uint64_t *counts, uint32_t npreds,
                        const gace_pair *pairs, const uint64_t *joints, uint32_t npairs,
                        const uint8_t *regs, uint32_t ncols_hll, uint32_t hll_p,
                        const double *ndv_hist, double *sel, double *pcs, double *ndv_est,
                        double *drift);

/* Gate thresholds; NULL = the paper's: D >= 0.25 (line 65), |dS| > 0.01 (line 69),
 * PCS > 1.6 or PCS < 0.7 (line 78). */
typedef struct {
    double d_threshold;
    double sel_err_threshold;
    double pcs_high;
    double pcs_low;
} gace_thresholds;

enum { GACE_SIG_DRIFT = 1, GACE_SIG_SEL_ERROR = 2, GACE_SIG_CORRELATION = 4 };

/*
 * Risky Gate (§III-A, lines 45-52): fired_mask = OR of
 *   DRIFT        if any drift[k] >= d_threshold
 *   SEL_ERROR    if any |s_est[k] - s_probe[k]| > sel_err_threshold
 *   CORRELATION  if any pcs[k] > pcs_high or pcs[k] < pcs_low
 * NaN never fires.  per_signal_fired (optional) gets nd + ns + np bytes (0/1) in
 * that order.  The probe is recommended iff fired_mask != 0.
 */
gace_status gace_gate(const double *drift, uint32_t nd, const double *s_est,
                      const double *s_probe, uint32_t ns, const double *pcs, uint32_t np,
                      const gace_thresholds *th, uint32_t *fired_mask,
                      uint8_t *per_signal_fired);

/*
 * Break-even cost accounting (§III-C Eq. 4, lines 80-83: the measurement cost is
 * modelled from the measured kernel time, "Cost_measurement ~ 0.85 ms"; §V item 2: a
 * break-even point exists).
 *   est_probe_cost_ms = c0 + c_t * N + c_e * K * M * N / p
 *   est_benefit_ms    = benefit_weight * (max - min candidate plan cost)   (SPEC reading S:249)
 * Host only (no device needed).
 */
typedef struct {
    double c0_ms;           /* fixed cost per probe (launch, plan upload, D2H)               */
    double ct_ms_per_row;   /* per scanned row                                              */
    double ce_ms_per_eval;  /* per row x predicate x set evaluation                         */
    double p;               /* parallelism factor, >= 1                                     */
    double benefit_weight;  /* >= 0; gace_cost_fit sets 0.5 when it is not >= 0 on entry   */
} gace_cost_model;

enum { GACE_NO_RISK = 0, GACE_RISK_BUT_NOT_WORTH = 1, GACE_PROBE = 2 };

/* Least-squares fit of (c0, c_t, c_e) >= 0 to npts >= 3 measured probe times ms[i] at
 * (n[i], k[i], m[i]) for a given p >= 1: every non-negativity active
 * set is solved and the feasible fit with the least squared residual is kept.  out->p = p.
 * GACE_EINVAL: NULL, npts < 3, p < 1, non-finite inputs.                                   */
gace_status gace_cost_fit(const double *n, const double *k, const double *m, const double *ms,
                          uint32_t npts, double p, gace_cost_model *out);

/* GateDecision: probe = fired_mask != 0 && est_benefit > est_cost
 * (strict); reason = GACE_NO_RISK (nothing fired), GACE_RISK_BUT_NOT_WORTH, GACE_PROBE.
 * est_cost_ms / est_benefit_ms may be NULL.  GACE_EINVAL: negative coefficients, p < 1.   */
gace_status gace_gate_decide(uint32_t fired_mask, const gace_cost_model *cm, double n_sample,
                             double k, double m, double plan_cost_spread_ms, double *est_cost_ms,
                             double *est_benefit_ms, uint32_t *probe, uint32_t *reason);

/* Per-stage device times of the last gace_probe on t, in ms (CUDA events on the
 * table's stream; §IV-B overhead decomposition H2D / kernel / D2H / reduction). */
typedef struct {
    double plan_upload_ms;  /* H2D of the predicate plan                               */
    double h2d_ms;          /* H2D of key columns (host tables; 0 for device tables)   */
    double scan_ms;         /* probe kernel(s): the HBM pass                           */
    double finalize_ms;     /* block partials -> counts / joints / registers           */
    double merge_ms;        /* NCCL all-reduce sum + max (0 on one GPU)                */
    double d2h_ms;          /* results to host                                         */
    double total_ms;        /* first to last event                                     */
    uint64_t scan_launches; /* probe-kernel launches in that call                      */
    uint64_t bytes_scanned; /* algorithmic bytes: rows x sum of probed column widths   */
    int32_t jit;            /* scan kernel of the call's large launches: 0 generic
                               (precompiled) kernel, 1 specialised for the plan's
                               structure, 2 specialised for its structure and layout,
                               -1 specialisation failed, generic kernel used            */
    int32_t merge;          /* cross-GPU merge of that call: 0 none (one rank, no NCCL),
                               1 grouped ncclAllReduce sum + max, 2 fused peer-memory
                               kernel over an NCCL symmetric window (NVLink loads)      */
    double jit_compile_ms;  /* NVRTC compile time spent in that call (0 when cached)   */
} gace_timing;

gace_status gace_last_timing(const gace_table *t, gace_timing *out);

/*
 * Plan-specialised scan kernels are compiled with NVRTC off the call path:
 * a probe whose specialised kernel is not compiled yet runs the precompiled generic kernel
 * (same results) and queues the compile on a background thread; the kernel specialised
 * for the batch's structure serves every later batch of that structure, the one
 * specialised for its layout too replaces it for repeats of the same batch.  (Env
 * GACE_JIT=1 compiles synchronously instead; GACE_JIT=0 never specialises.)
 * gace_jit_sync waits up to timeout_ms until no compile is queued or running
 * (GACE_EUNSUPPORTED on timeout); the counters (each may be NULL) report compiles
 * finished, failed and still pending.  GACE_EINVAL: timeout_ms negative or NaN.
 */
gace_status gace_jit_sync(double timeout_ms, uint64_t *compiled, uint64_t *failed, uint64_t *pending);

/* Stop the background compile worker (process exit): queued compiles are dropped, one in
 * progress finishes first; later batches run on the kernels already compiled or the generic
 * one (no compile is started again).  Idempotent; always GACE_OK.  The Python binding calls
 * it from its atexit hook, before the interpreter tears down CUDA state the worker uses. */
gace_status gace_jit_shutdown(void);

/* Rank 0 of a multi-GPU job: fill id[128] with a fresh ncclUniqueId to broadcast to
 * the other ranks (GACE_ENCCL if libnccl.so.2 cannot be loaded). */
gace_status gace_nccl_unique_id(void *id128);

/* Test hook (host only; no device needed): plan a predicate batch for a table with
 * value domains [dlo[c], dhi[c]] (host = 0: device table; 1: host table) and resolve
 * values[n] of column `col` through the planned lookup table with the kernel's own
 * lookup code (csrc/gace_plan.h lut_lookup), bounds-checked.  out[k] = bucket of
 * values[k] relative to the column's bucket 0 (= #{breakpoints <= v}); *mode = 0 lookup
 * table, 1 binary search; the column's sorted breakpoints go to bps[cap], *nbp = count.
 * GACE_EUNSUPPORTED "internal: ..." reports a plan that would read out of range.     */
gace_status gace_debug_buckets(uint32_t ncols, const gace_dtype *dtypes, const int64_t *dlo,
                               const int64_t *dhi, int host, const gace_pred *preds,
                               uint32_t npreds, const gace_pair *pairs, uint32_t npairs,
                               uint64_t hll_mask, uint32_t col, const int64_t *values, uint64_t n,
                               uint32_t *out, uint32_t *mode, int64_t *bps, uint32_t cap,
                               uint32_t *nbp);

/* Test hook (host only; needs libnvrtc, no device): plan a batch as gace_debug_buckets
 * does and compile its plan-specialised probe kernel without launching
 * it; *cubin_bytes = size of the compiled image.  GACE_EUNSUPPORTED carries the NVRTC log. */
gace_status gace_debug_jit_compile(uint32_t ncols, const gace_dtype *dtypes, const int64_t *dlo,
                                   const int64_t *dhi, int host, const gace_pred *preds,
                                   uint32_t npreds, const gace_pair *pairs, uint32_t npairs,
                                   uint64_t hll_mask, double sample_rate, uint64_t *cubin_bytes);

/* Number of this library's CUDA kernels launched since load (all tables). */
uint64_t gace_kernel_launches(void);

/* Thread-local message for the last non-OK status on this thread ("" if none). */
const char *gace_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* GACE_H_ */
