// gace_host.cpp -- C-ABI of the GACE selectivity probe (include/gace.h):
// table handles, the predicate planner, launch orchestration, the NCCL merge
// and the host-side derive / gate arithmetic.
//
// Planner: every predicate becomes a
// closed int64 interval (plus a negate flag), clipped to the column's value
// domain; the interval ends give the column's sorted breakpoints T, so each
// predicate is a contiguous range of buckets bucket(v) = #{t in T : t <= v} and
// count = (prefix-sum difference over a per-column bucket histogram).  Pairs on
// one column are interval intersections of those ranges (no per-row work);
// pairs across two columns share one 2-D histogram per column pair over the
// sub-buckets of only the pair-relevant predicates.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <unistd.h>   // environ

#include <algorithm>
#include <array>
#include <deque>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <functional>
#include <map>
#include <memory>
#include <charconv>
#include <chrono>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/gace.h"
#include "gace_jit.h"
#include "gace_kernels.h"
#include "gace_merge.h"
#include "gace_plan.h"
#include "gace_sets.h"

using namespace gace;

namespace {

thread_local std::string g_err;

// Design / test switches (GACE_*) read by the probe path: one pass over the environment at the
// start of each probe call (refresh_knobs) instead of a getenv per switch -- at C1's size ten
// getenv scans were a visible part of the per-call host time.  Tests change them between calls.
struct KnobSnap {
    std::vector<std::pair<std::string, std::string>> kv;
};
thread_local KnobSnap g_knobs;
thread_local bool g_knobs_valid = false;
void refresh_knobs() {
    g_knobs.kv.clear();
    for (char **e = environ; e && *e; ++e) {
        const char *v = *e;
        if (v[0] != 'G' || strncmp(v, "GACE_", 5) != 0) continue;
        const char *eq = strchr(v, '=');
        if (eq) g_knobs.kv.emplace_back(std::string(v, eq - v), std::string(eq + 1));
    }
    g_knobs_valid = true;
}
const char *knob(const char *name) {
    if (!g_knobs_valid) return getenv(name);
    for (const auto &p : g_knobs.kv)
        if (p.first == name) return p.second.c_str();
    return nullptr;
}
std::atomic<uint64_t> g_launches{0};

gace_status fail(gace_status s, const std::string &msg) {
    g_err = msg;
    return s;
}

#define CUDA_TRY(x)                                                                              \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess) return fail(GACE_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// ------------------------------------------------------------------ NCCL via dlopen

struct NcclUid { char internal[128]; };
struct Nccl {
    void *h = nullptr;
    int (*GetUniqueId)(NcclUid *) = nullptr;
    int (*CommInitRank)(void **, int, NcclUid, int) = nullptr;
    int (*AllReduce)(const void *, void *, size_t, int, int, void *, cudaStream_t) = nullptr;
    int (*GroupStart)() = nullptr;
    int (*GroupEnd)() = nullptr;
    int (*CommDestroy)(void *) = nullptr;
    int (*CommAbort)(void *) = nullptr;
    int (*CommGetAsyncError)(void *, int *) = nullptr;
    const char *(*GetErrorString)(int) = nullptr;
};
constexpr int kNcclUint8 = 1, kNcclInt64 = 4, kNcclUint64 = 5, kNcclSum = 0, kNcclMax = 2, kNcclMin = 3;
constexpr int kNcclInProgress = 7;

Nccl *nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        const char *names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char *nm : names) {
            n.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (n.h) break;
        }
        if (!n.h) return;
        n.GetUniqueId = (int (*)(NcclUid *))dlsym(n.h, "ncclGetUniqueId");
        n.CommInitRank = (int (*)(void **, int, NcclUid, int))dlsym(n.h, "ncclCommInitRank");
        n.AllReduce = (int (*)(const void *, void *, size_t, int, int, void *, cudaStream_t))dlsym(n.h, "ncclAllReduce");
        n.GroupStart = (int (*)())dlsym(n.h, "ncclGroupStart");
        n.GroupEnd = (int (*)())dlsym(n.h, "ncclGroupEnd");
        n.CommDestroy = (int (*)(void *))dlsym(n.h, "ncclCommDestroy");
        n.CommAbort = (int (*)(void *))dlsym(n.h, "ncclCommAbort");
        n.CommGetAsyncError = (int (*)(void *, int *))dlsym(n.h, "ncclCommGetAsyncError");
        n.GetErrorString = (const char *(*)(int))dlsym(n.h, "ncclGetErrorString");
        if (!n.GetUniqueId || !n.CommInitRank || !n.AllReduce || !n.GroupStart || !n.GroupEnd || !n.CommDestroy ||
            !n.CommAbort || !n.CommGetAsyncError)
            n.h = nullptr;
    });
    return n.h ? &n : nullptr;
}

// ------------------------------------------------------------------ buffers

struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t n) {
        if (n <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaMalloc(&p, n);
        if (e == cudaSuccess) cap = n;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <class T> T *as(size_t byte_off = 0) const { return reinterpret_cast<T *>(static_cast<char *>(p) + byte_off); }
};

struct HostBuf {
    void *p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t n) {
        if (n <= cap) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaMallocHost(&p, n);
        if (e == cudaSuccess) cap = n;
        return e;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
    }
    template <class T> T *as(size_t byte_off = 0) const { return reinterpret_cast<T *>(static_cast<char *>(p) + byte_off); }
};

size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

}  // namespace

constexpr uint32_t kMagic = 0x47414345u;   // "GACE"
// per-rank symmetric window of the fused merge: the largest packed result,
// [1 + 4096 + 4096 u64 | 8 HLL columns x 4096 registers], rounded up
constexpr size_t kMergeBytes = 128 * 1024;

// what a captured probe graph bakes in: plan, sampling, seed, ablation bits, scratch buffers
struct GraphKey {
    uint64_t plan = 0;       // plan generation of the table (never reused, unlike addresses)
    double rate = 0;
    uint64_t seed = 0;
    uint32_t dbg = 0;
    const void *buf[7] = {};
    GraphKey() = default;
    GraphKey(uint64_t pl, double r, uint64_t sd, uint32_t d, const void *a, const void *b, const void *c,
             const void *e, const void *f, const void *g, const void *h)
        : plan(pl), rate(r), seed(sd), dbg(d), buf{a, b, c, e, f, g, h} {}
    bool operator==(const GraphKey &o) const {
        if (plan != o.plan || rate != o.rate || seed != o.seed || dbg != o.dbg) return false;
        for (int i = 0; i < 7; ++i)
            if (buf[i] != o.buf[i]) return false;
        return true;
    }
};
constexpr int kNumEv = 8;

struct gace_table {
    uint32_t magic = kMagic;
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool host = false;
    uint32_t ncols = 0;
    uint64_t nrows = 0;
    std::vector<const void *> cols;
    std::vector<int> dtypes;
    std::vector<int64_t> dlo, dhi;     // value domain per column (measured for device tables)
    std::vector<uint8_t> clustered;    // >= half of the aligned row quads hold one key (device tables)
    bool has_dist = false;
    gace_dist dist{};
    // NCCL merge: whenever the caller gave a communicator or a unique id (any nranks,
    // including 1), the results are merged by the grouped all-reduce before the D2H copy
    bool use_nccl = false;
    void *comm = nullptr;
    bool own_comm = false;
    bool comm_dead = false;            // aborted after an asynchronous NCCL error / timeout
    MergeState *merge = nullptr;       // fused merge over a symmetric window (gace_merge.cu), or none
    DevBuf d_coll;                     // small collective scratch (attach domains, plan agreement)
    int sms = 148;
    DevBuf d_plan, d_accb[2], d_pre, d_part, d_out, d_nsamp, d_mask, d_stage[2];
    HostBuf h_plan, h_out;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev[kNumEv]{};
    cudaEvent_t ev_copied[2]{}, ev_free[2]{}, ev_c0{}, ev_c1{};
    gace_timing last{};
    // stage times are read from the events only when asked (gace_last_timing): 0 none,
    // 1 probe (ev[0..5]), 2 candidate sets (no finalize stage); host tables add the copy span
    int timing_kind = 0;
    bool dirty = false;     // a call returned mid-way: its work may still be queued
    std::mutex mu;
    // plan cache: the last batch's plan and its uploaded device blob (repeated probes of the
    // same batch skip planning and the H2D of the tables)
    std::string plan_key;
    std::shared_ptr<void> plan;
    // specialised kernel of the cached plan (index: sampled): kind 1 = keyed on the plan
    // structure, 2 = keyed on its layout too; the layout-keyed one is compiled in the
    // background (jit_lsrc) and replaces the structure-keyed one once it is loaded
    void *jit_fn[2] = {nullptr, nullptr};
    int jit_kind[2] = {0, 0};
    std::string jit_ssrc[2], jit_lsrc[2];
    uint64_t plan_calls = 0;           // probes of the cached plan (layout-keyed compile on the 2nd)
    // CUDA-graph replay of repeated identical probes (gace_table_set_graphs)
    bool graphs = false;
    uint64_t plan_gen = 0;
    // double-buffered accumulators: each call's fin_output zeroes the other buffer, so the
    // next call needs no memset (a buffer is "clean" only after a call that zeroed it completed)
    int acc_next = 0;
    bool acc_clean[2] = {false, false};
    cudaGraphExec_t gexec = nullptr;
    GraphKey gkey, gprev;
    bool gprev_ok = false;
    uint64_t g_scan_launches = 0, g_nl = 0, g_captures = 0, g_replays = 0;
    int g_jit = 0;
    size_t blob = 0, o_img = 0, o_dir = 0, o_job = 0, o_fp = 0, o_fq = 0, o_bps = 0;
    // HLL register ceilings per column (u8[ncols][4096]), computed on first use
    DevBuf d_hceil, d_hceil32;
    std::vector<uint8_t> hceil_ready;
    // candidate-set probe (gace_probe_sets): plan cache and buffers
    std::string sets_key;
    std::shared_ptr<void> sets_plan;
    DevBuf d_sets_img, d_sets_out;
    HostBuf h_sets_img, h_sets_out;
};

namespace {

// ------------------------------------------------------------------ NCCL-aware waits

// Wait for the table's stream.  Tables merged over NCCL poll instead of blocking: an
// asynchronous NCCL error (a peer died, a network fault) or a collective that does not
// finish within GACE_NCCL_TIMEOUT_MS (default 300000) aborts the communicator -- which
// releases the kernels blocked in it -- and the call returns GACE_ENCCL instead of hanging.
gace_status wait_stream(gace_table *t, cudaStream_t s) {
    if (!t->use_nccl || !t->comm) {
        CUDA_TRY(cudaStreamSynchronize(s));
        return GACE_OK;
    }
    if (t->comm_dead) return fail(GACE_ENCCL, "NCCL communicator was aborted by an earlier error");
    Nccl *n = nccl();
    static const double limit_ms = [] {
        const char *e = getenv("GACE_NCCL_TIMEOUT_MS");
        return e ? atof(e) : 300000.0;
    }();
    const auto t0 = std::chrono::steady_clock::now();
    for (uint32_t spin = 0;; ++spin) {
        const cudaError_t q = cudaStreamQuery(s);
        if (q == cudaSuccess) return GACE_OK;
        if (q != cudaErrorNotReady) return fail(GACE_ECUDA, std::string("stream: ") + cudaGetErrorString(q));
        int async = 0;
        const int r = n->CommGetAsyncError(t->comm, &async);
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (r != 0 || (async != 0 && async != kNcclInProgress) || ms > limit_ms) {
            n->CommAbort(t->comm);
            t->comm_dead = true;
            const int code = r ? r : async;
            return fail(GACE_ENCCL, ms > limit_ms ? std::string("NCCL collective timed out; communicator aborted")
                                                  : std::string("NCCL asynchronous error: ") +
                                                        (n->GetErrorString ? n->GetErrorString(code) : "?"));
        }
        if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(spin > 4096 ? 200 : 5));
    }
}

// ------------------------------------------------------------------ planner

struct Interval {      // closed int64 interval after clipping to the column domain
    bool empty = true;
    int64_t lo = 0, hi = 0;
};

// PAPER-side semantics (DESIGN.md "Semantics" 4, readings L9/L10): op -> closed interval.
Interval op_interval(const gace_pred &p) {
    Interval I;
    const int64_t a = p.a, b = p.b;
    I.empty = false;
    switch (p.op) {
        case GACE_EQ: I.lo = a; I.hi = a; break;
        case GACE_LT:
            if (a == INT64_MIN) I.empty = true; else { I.lo = INT64_MIN; I.hi = a - 1; }
            break;
        case GACE_LE: I.lo = INT64_MIN; I.hi = a; break;
        case GACE_GT:
            if (a == INT64_MAX) I.empty = true; else { I.lo = a + 1; I.hi = INT64_MAX; }
            break;
        case GACE_GE: I.lo = a; I.hi = INT64_MAX; break;
        default:   // BETWEEN
            if (a > b) I.empty = true; else { I.lo = a; I.hi = b; }
    }
    return I;
}

Interval clip(Interval I, int64_t dl, int64_t dh) {
    if (I.empty) return I;
    I.lo = std::max(I.lo, dl);
    I.hi = std::min(I.hi, dh);
    if (I.lo > I.hi) I.empty = true;
    return I;
}

void add_breakpoints(const Interval &I, int64_t dl, int64_t dh, std::vector<int64_t> &T) {
    if (I.empty) return;
    if (I.lo > dl) T.push_back(I.lo);
    if (I.hi < dh) T.push_back(I.hi + 1);
}

// #{t in T : t <= x} over sorted T -- branch-free halving (the planner calls it per predicate
// bound and per bucket: branchy searches mispredicted at ~100 ns per call on C3's 1024 binds)
uint32_t count_le(const std::vector<int64_t> &T, int64_t x) {
    const int64_t *base = T.data();
    size_t len = T.size();
    if (!len) return 0;
    while (len > 1) {
        const size_t half = len >> 1;
        base = base[half - 1] <= x ? base + half : base;
        len -= half;
    }
    return (uint32_t)(base - T.data()) + (*base <= x ? 1u : 0u);
}

struct SlotPlan {
    int col = -1;
    int dtype = 0;
    bool has_preds = false, has_hll = false;
    int64_t dl = 0, dh = 0;
    std::vector<int64_t> T;            // sorted unique breakpoints
    uint32_t nb = 1;                   // buckets
    // lookup table
    uint8_t mode = MODE_NOPRED;
    bool clamp = false;
    int64_t base = 0, clamp_lo = 0, clamp_hi = 0;
    uint32_t s1 = 0;
    uint8_t fmt = FMT32;               // level-1 cell format (gace_plan.h LutFmt)
    uint32_t sb = 16;                  // FMT1T: bucket field width of bs
    std::vector<uint32_t> l1;          // level-1 cells in FMT32 encoding (boundary: slot-relative record index)
    std::vector<uint4> l2;             // records and nested blocks (slot-relative indices)
    std::vector<uint32_t> lst;         // list thresholds (breakpoint offsets)
    uint64_t n_l1 = 0, n_l2 = 0, n_lst = 0;   // table sizes at s1 (built, or estimated: lut_estimate)
    bool built = false;                // l1 / l2 / lst hold the table at s1
    // roles in the pair grids
    int hist_grp = -1;                 // group whose grid row sums give this column's histogram
    int prim_b = -1;                   // group whose sub-bucket the entries pack
    const std::vector<int64_t> *TBp = nullptr;   // that group's sub-bucket breakpoints
    // layout
    uint32_t lut_idx = 0, l2_idx = 0, lst_idx = 0, hist_w = kNone, hll_idx = kNone, bps_off = 0;
    uint32_t pre = 0, pre_stride = 1;  // finalize: bucket-count prefix of this column
    // HLL by presence bitmap (gace_plan.h SlotParams::bm_addr)
    bool bm = false;
    bool fdirect = false;              // exact cells hold the byte address of the own histogram bin
    int64_t bm_base = 0;
    uint32_t bm_words = 0, bm_w = kNone, bm_goff = 0, hll_out = 0;
};

uint32_t ceil_log2(uint64_t x) {
    uint32_t r = 0;
    while ((1ull << r) < x) ++r;
    return r;
}

// Build the lookup table of a slot for level-1 shift s1 over offsets u in [0, span]
// (formats: gace_plan.h).  Indices are RELATIVE here; make_plan adds the slot's
// shared-memory offsets.  A cell without breakpoints is a plain u32 (bucket + packed
// sub-bucket of the column's primary B role); a boundary cell points to a record: direct
// (<= 3 breakpoints), list (<= 8) or a block of uniform sub-cells built recursively.
bool build_lut(SlotPlan &S, uint64_t span, uint32_t s1) {
    std::vector<uint64_t> toff;
    toff.reserve(S.T.size());
    for (int64_t t : S.T) toff.push_back((uint64_t)t - (uint64_t)S.base);   // in [1, span]
    auto le = [&](uint64_t x) { return (uint32_t)(std::upper_bound(toff.begin(), toff.end(), x) - toff.begin()); };
    // sub-bucket of bucket b in the packed group, and whether breakpoint T[i] cuts it
    // (tabulated once: the cell loops below look them up per cell)
    std::vector<uint32_t> sub_tab(S.T.size() + 1, 0);
    std::vector<uint8_t> cut_tab(S.T.size(), 0);
    if (S.TBp) {
        for (size_t b = 1; b <= S.T.size(); ++b) sub_tab[b] = count_le(*S.TBp, S.T[b - 1]);
        for (size_t i = 0; i < S.T.size(); ++i) cut_tab[i] = std::binary_search(S.TBp->begin(), S.TBp->end(), S.T[i]);
    }
    auto sub_of = [&](uint32_t b) -> uint32_t { return sub_tab[b]; };
    auto cuts = [&](uint32_t i) -> bool { return cut_tab[i] != 0; };
    // #{t in toff : t <= x} for non-decreasing x along a cell sweep (amortised O(1))
    struct Sweep {
        const std::vector<uint64_t> &t;
        uint32_t j = 0;
        uint32_t operator()(uint64_t x) {
            while (j < t.size() && t[j] <= x) ++j;
            return j;
        }
    };
    S.s1 = s1;
    S.l1.clear();
    S.l2.clear();
    S.lst.clear();
    bool ok = true;
    auto done = [&]() {
        S.n_l1 = S.l1.size();
        S.n_l2 = S.l2.size();
        S.n_lst = S.lst.size();
        S.built = true;
        return ok;
    };
    std::function<uint4(uint64_t, uint64_t, uint32_t)> node = [&](uint64_t lo, uint64_t hi, uint32_t s) -> uint4 {
        const uint32_t b0 = le(lo), b1 = le(hi), cnt = b1 - b0;   // breakpoints in (lo, hi]
        if (cnt <= 3) {
            uint32_t t[3] = {kNoThr, kNoThr, kNoThr}, flags = 0;
            for (uint32_t i = 0; i < cnt; ++i) {
                t[i] = (uint32_t)(toff[b0 + i] - 1);               // u > t  <=>  u >= breakpoint
                if (cuts(b0 + i)) flags |= 1u << (kIncShift + i);
            }
            return make_uint4(b0 | (sub_of(b0) << kSubShift) | flags, t[0], t[1], t[2]);
        }
        if (cnt <= 8 || s == 0) {
            uint4 e = make_uint4(kSpecial | kList | (cnt << 24) | b0, (uint32_t)S.lst.size(), 0, 0);
            for (uint32_t i = b0; i < b1; ++i) S.lst.push_back((uint32_t)toff[i]);
            return e;
        }
        // sub-cells at the minimum breakpoint gap when affordable (then each holds <= 1),
        // else about two sub-cells per breakpoint
        uint64_t gap = UINT64_MAX;
        for (uint32_t i = b0 + 1; i < b1; ++i) gap = std::min(gap, toff[i] - toff[i - 1]);
        uint32_t sc = 0;
        while (sc + 1 < s && (2ull << sc) <= gap) ++sc;          // 2^sc <= gap, sc < s
        if (((hi - lo) >> sc) + 1 > 4ull * cnt + 16) {
            const uint32_t want = ceil_log2(cnt) + 1;
            sc = s > want ? s - want : 0;
        }
        const uint64_t nsub = ((hi - lo) >> sc) + 1;
        if (S.l2.size() + nsub > (1u << 20)) { ok = false; return make_uint4(b0, kNoThr, kNoThr, kNoThr); }
        const uint32_t first = (uint32_t)S.l2.size();
        S.l2.resize(first + nsub);
        for (uint64_t j = 0; j < nsub; ++j) {
            const uint64_t slo = lo + (j << sc), shi = std::min<uint64_t>(slo + (1ull << sc) - 1, hi);
            const uint4 e = node(slo, shi, sc);
            S.l2[first + j] = e;
        }
        return make_uint4(kSpecial | (sc << 24), first, 0, 0);
    };
    const uint64_t ncells = (span >> s1) + 1;
    const uint64_t csize = 1ull << s1;
    S.l1.reserve(ncells);
    Sweep at_lo{toff}, at_hi{toff};
    // runs of cells without a breakpoint inside share one plain entry: the sweeps below jump
    // from one breakpoint-holding cell to the next and fill the run between with std::fill
    // (planning cost O(cells) memory writes + O(breakpoints) work, not per-cell searches)
    auto run_end = [&](uint64_t k) -> uint64_t {      // first cell >= k holding a breakpoint in (lo, hi]
        const uint32_t j = at_lo(k << s1);             // first breakpoint above this cell's start
        if (j >= toff.size()) return ncells;
        const uint64_t kn = toff[j] >> s1;             // its cell (at that cell's start: it bounds it)
        return std::min<uint64_t>(kn, ncells);
    };
    // a record of <= 3 breakpoints (the common boundary cell), from the sweep's own indices:
    // node()'s first case without its searches
    auto direct = [&](uint32_t b0, uint32_t cnt) -> uint4 {
        uint32_t t[3] = {kNoThr, kNoThr, kNoThr}, flags = 0;
        for (uint32_t i = 0; i < cnt; ++i) {
            t[i] = (uint32_t)(toff[b0 + i] - 1);                   // u > t  <=>  u >= breakpoint
            if (cuts(b0 + i)) flags |= 1u << (kIncShift + i);
        }
        return make_uint4(b0 | (sub_of(b0) << kSubShift) | flags, t[0], t[1], t[2]);
    };
    if (S.fmt == FMT1T) {      // one in-cell threshold per cell (gace_plan.h FMT1T)
        auto bs = [&](uint32_t b) { return (b + 1) | (sub_of(b) << S.sb); };
        for (uint64_t k = 0; k < ncells && ok; ++k) {
            const uint64_t ke = run_end(k);
            if (ke > k) {                                          // plain run [k, ke)
                S.l1.insert(S.l1.end(), ke - k, bs(at_lo(k << s1)) - 1);
                k = ke - 1;
                continue;
            }
            const uint64_t lo = k << s1, hi = std::min<uint64_t>(lo + csize - 1, span);
            const uint32_t b0 = at_lo(lo), cnt = at_hi(hi) - b0;   // breakpoints in (lo, hi]
            if (cnt == 0) {
                S.l1.push_back(bs(b0) - 1);                        // t = 0: always "crossed"
            } else if (cnt == 1) {
                const uint32_t t = (uint32_t)(toff[b0] - lo);      // in [1, 2^s1)
                S.l1.push_back((t << (32 - s1)) | (cuts(b0) ? 1u << (30 - s1) : 0u) | bs(b0));
            } else {
                const uint4 e = cnt <= 3 ? direct(b0, cnt) : node(lo, hi, s1);
                S.l1.push_back(t1_special(s1) | (uint32_t)S.l2.size());   // slot-relative record
                S.l2.push_back(e);
            }
        }
        return done();
    }
    for (uint64_t k = 0; k < ncells && ok; ++k) {
        const uint64_t ke = run_end(k);
        if (ke > k) {                                              // plain run [k, ke)
            const uint32_t b0 = at_lo(k << s1);
            S.l1.insert(S.l1.end(), ke - k, b0 | (sub_of(b0) << kSubShift));
            k = ke - 1;
            continue;
        }
        const uint64_t lo = k << s1, hi = std::min<uint64_t>(lo + csize - 1, span);
        const uint32_t b0 = at_lo(lo), cnt = at_hi(hi) - b0;
        if (cnt == 0) {                                            // plain cell
            S.l1.push_back(b0 | (sub_of(b0) << kSubShift));
        } else {                                                   // boundary cell -> record
            const uint4 e = cnt <= 3 ? direct(b0, cnt) : node(lo, hi, s1);
            S.l1.push_back(kSpecial | (uint32_t)S.l2.size());
            S.l2.push_back(e);
        }
    }
    return done();
}

size_t lut_bytes(const SlotPlan &S) {
    return (S.fmt == FMT16 ? 2 : 4) * S.n_l1 + 16 * S.n_l2 + 4 * S.n_lst + 48;
}

// The sizes build_lut would produce at level-1 shift s1, without building (the planner sizes
// candidate resolutions with this and builds each table once): every cell is one level-1
// entry; a cell holding breakpoints (FMT1T: >= 2) adds one record.  A breakpoint exactly at a
// cell start bounds that cell and lies inside none.  exact = false when some cell holds more
// than 3 (nested blocks or lists): then the table has to be built to be sized.
struct LutEst {
    uint64_t l1 = 0, l2 = 0;
    bool exact = false;
};
LutEst lut_estimate(const SlotPlan &S, uint64_t span, uint32_t s1) {
    LutEst E;
    E.l1 = (span >> s1) + 1;
    const uint32_t need = S.fmt == FMT1T ? 2u : 1u;
    const uint64_t m = (1ull << s1) - 1;
    uint64_t cur = UINT64_MAX;
    uint32_t cnt = 0;
    for (int64_t t : S.T) {
        const uint64_t o = (uint64_t)t - (uint64_t)S.base;
        if (o > span || (o & m) == 0) continue;
        const uint64_t k = o >> s1;
        if (k != cur) {
            if (cnt > 3) return E;
            E.l2 += cnt >= need ? 1 : 0;
            cur = k;
            cnt = 0;
        }
        ++cnt;
    }
    if (cnt > 3) return E;
    E.l2 += cnt >= need ? 1 : 0;
    E.exact = true;
    return E;
}

// FMT1T field budget: bucket + 1 in sb bits, the packed sub-bucket above it, and record
// indices (< 2^14 uint4 in 227 KB) all within the 30 - s1 data bits.
uint32_t t1_max_s1(const SlotPlan &S, uint32_t nsub) {
    const uint32_t need = std::max<uint32_t>(S.sb + ceil_log2(nsub), 14);
    return need >= 29 ? 0 : std::min<uint32_t>(20, 30 - need);
}

// MurmurHash3 fmix32 (the int32 HLL hash, DESIGN.md §2 step 6) for exact-cell tables.
uint32_t host_fmix32(uint32_t h) {
    h ^= h >> 16;
    h *= 0x85EBCA6BU;
    h ^= h >> 13;
    h *= 0xC2B2AE35U;
    h ^= h >> 16;
    return h;
}

struct Group {
    int a = -1, b = -1;                // oriented: a = full-resolution side, b = sub-bucket side
    int s0, s1;                        // the two slots (s0 < s1), before orientation
    std::vector<uint32_t> pq;          // its cross-column pairs
    std::vector<int64_t> TB;           // sub-bucket breakpoints on b (b-side predicates of pq)
    uint32_t na = 1, nbs = 1;
    bool direct = false, packed = false;
    uint32_t grid_w = 0, map_w = 0, sat = 0;
};

struct Plan {
    std::vector<SlotPlan> slots;
    std::vector<int> col2slot;
    std::vector<Interval> iv;          // per predicate, clipped
    std::vector<int> pslot;            // per predicate
    std::vector<Group> groups;
    std::map<std::pair<int, int>, int> gidx;
    bool clamp = false;
    // layout results
    std::vector<uint8_t> image;        // shared-memory image (tables + maps)
    uint32_t acc_idx = 0, acc_words = 0, hll_off = 0, hll_bytes = 0, smem_bytes = 0;
    uint32_t pre_words = 0;
    uint32_t bm_gwords = 0;            // merged presence bitmaps (u32 words in g_bm)
    std::vector<DirectPair> direct;
    std::vector<FinJob> jobs;
    std::vector<FinPred> fpreds;
    std::vector<FinPair> fpairs;
    std::vector<int64_t> bps;          // MODE_SEARCH breakpoints, concatenated
    ProbeParams P{};
};

// dynamic shared memory a plan may use: the 227 KB less the kernel's static reservation
// (gace_plan.h static_smem_reserve: a full scan's kernels carry no row queue)
constexpr size_t smem_budget(bool full) { return (size_t)(kMaxSmem - static_smem_reserve(!full)); }

// Plan summary on stderr (env GACE_PLAN_DUMP; design inspection only).
void dump_plan(const Plan &pl) {
    for (size_t i = 0; i < pl.slots.size(); ++i) {
        const SlotPlan &S = pl.slots[i];
        size_t special = 0;
        for (uint32_t c : S.l1) special += (c & (S.fmt == FMT1T ? t1_special(S.s1) : kSpecial)) ? 1 : 0;
        fprintf(stderr, "slot %zu col %d dt %d mode %d fmt %d s1 %u sb %u nb %u cells %zu special %zu (%.2f%%) l2 %zu lst %zu "
                "hll %d%s hist_grp %d prim_b %d span %llu\n", i, S.col, S.dtype, (int)S.mode, (int)S.fmt, S.s1, S.sb, S.nb,
                S.l1.size(), special, S.l1.empty() ? 0.0 : 100.0 * special / S.l1.size(), S.l2.size(), S.lst.size(),
                (int)S.has_hll, S.bm ? " (bitmap)" : "", S.hist_grp, S.prim_b, (unsigned long long)((uint64_t)S.dh - (uint64_t)S.dl));
    }
    for (size_t g = 0; g < pl.groups.size(); ++g) {
        const Group &G = pl.groups[g];
        fprintf(stderr, "group %zu a %d b %d na %u nbs %u pairs %zu direct %d packed %d\n", g, G.a, G.b, G.na, G.nbs,
                G.pq.size(), (int)G.direct, (int)G.packed);
    }
    fprintf(stderr, "smem %u image %zu acc_words %u hll_bytes %u\n", pl.smem_bytes, pl.image.size(), pl.acc_words,
            pl.hll_bytes);
}

// Folded addressing (int32 lookup column without clamp, FMTEX, or FMT1T whose cells are
// aligned key multiples): the specialised kernel indexes the level-1 table with the key
// itself and the base folded into fold_b / fold_z (gace_plan.h SlotParams).
bool slot_foldable(const SlotParams &Q) {
    if (Q.dtype != 0 || Q.mode != MODE_LUT || Q.clamp_lo != INT32_MIN || Q.clamp_hi != INT32_MAX) return false;
    if (Q.fmt == FMTEX) return true;
    return Q.fmt == FMT1T && Q.s1 >= 1 && ((uint64_t)Q.base & ((1ull << Q.s1) - 1)) == 0 && Q.base >= 0;
}

// sparse = the probe's sample rate is below 1/8: only the few kept rows are looked up, so the
// level-1 tables are planned ~8x coarser (the lookup resolution barely matters there, while a
// new batch's planning, plan upload and per-CTA table load all scale with the table size)
gace_status make_plan(const gace_table *t, const gace_pred *preds, uint32_t np, const gace_pair *pairs,
                      uint32_t nq, uint64_t hll_mask, Plan &pl, bool sparse = false, bool full = false) {
    const size_t kSmemBudget = smem_budget(full);
    // design inspection: GACE_PLAN_PROFILE=1 prints the planner's phase times (stderr)
    static const bool prof = getenv("GACE_PLAN_PROFILE") != nullptr;
    auto tp0 = std::chrono::steady_clock::now();
    auto phase = [&](const char *name) {
        if (!prof) return;
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "plan %-12s %8.1f us\n", name, std::chrono::duration<double, std::micro>(now - tp0).count());
        tp0 = std::chrono::steady_clock::now();     // (the print is not part of the next phase)
    };
    // ---- slots: probed columns in ascending order
    std::vector<bool> probed(t->ncols, false);
    for (uint32_t p = 0; p < np; ++p) probed[preds[p].col] = true;
    for (uint32_t c = 0; c < t->ncols; ++c)
        if (hll_mask >> c & 1ull) probed[c] = true;
    pl.col2slot.assign(t->ncols, -1);
    for (uint32_t c = 0; c < t->ncols; ++c) {
        if (!probed[c]) continue;
        if (pl.slots.size() == (size_t)kMaxSlots)
            return fail(GACE_EUNSUPPORTED, "more than 8 probed columns in one probe");
        pl.col2slot[c] = (int)pl.slots.size();
        SlotPlan S;
        S.col = (int)c;
        S.dtype = t->dtypes[c];
        S.dl = t->dlo[c];
        S.dh = t->dhi[c];
        S.has_hll = (hll_mask >> c) & 1ull;
        pl.slots.push_back(S);
    }
    // ---- predicates -> clipped intervals -> breakpoints
    pl.iv.resize(np);
    pl.pslot.resize(np);
    for (uint32_t p = 0; p < np; ++p) {
        const int s = pl.col2slot[preds[p].col];
        SlotPlan &S = pl.slots[s];
        pl.pslot[p] = s;
        S.has_preds = true;
        pl.iv[p] = clip(op_interval(preds[p]), S.dl, S.dh);
        add_breakpoints(pl.iv[p], S.dl, S.dh, S.T);
    }
    for (auto &S : pl.slots) {
        std::sort(S.T.begin(), S.T.end());
        S.T.erase(std::unique(S.T.begin(), S.T.end()), S.T.end());
        S.nb = (uint32_t)S.T.size() + 1;
    }
    phase("intervals");
    // ---- cross-column pairs -> groups (one per unordered column pair)
    for (uint32_t q = 0; q < nq; ++q) {
        const int si = pl.pslot[pairs[q].i], sj = pl.pslot[pairs[q].j];
        if (si == sj) continue;
        auto key = std::make_pair(std::min(si, sj), std::max(si, sj));
        if (!pl.gidx.count(key)) {
            pl.gidx[key] = (int)pl.groups.size();
            Group G;
            G.s0 = key.first;
            G.s1 = key.second;
            pl.groups.push_back(G);
        }
        pl.groups[pl.gidx[key]].pq.push_back(q);
    }
    auto side_bps = [&](const Group &G, int side) {      // breakpoints of G's predicates on `side`
        std::vector<int64_t> TB;
        for (uint32_t q : G.pq) {
            const uint32_t p = pl.pslot[pairs[q].i] == side ? pairs[q].i : pairs[q].j;
            add_breakpoints(pl.iv[p], pl.slots[side].dl, pl.slots[side].dh, TB);
        }
        std::sort(TB.begin(), TB.end());
        TB.erase(std::unique(TB.begin(), TB.end()), TB.end());
        return TB;
    };
    // orientation: every column should be the full-resolution (A) side of some group -- its
    // histogram then comes from that grid's row sums -- and the packed sub-bucket (B) side
    // of at most one group.  Chosen from the group topology only (exhaustively for up to 12
    // groups, ties to the lowest orientation mask; greedily beyond), never from the grid
    // sizes: the orientation is part of the specialised kernel's structure, so a bind sweep
    // that moves the predicate bounds keeps its kernel.
    {
        const size_t G_ = pl.groups.size(), ns = pl.slots.size();
        std::vector<std::vector<int64_t>> tb[2];            // tb[o][g]: B-side breakpoints if oriented o
        for (int o = 0; o < 2; ++o)
            for (auto &G : pl.groups) tb[o].push_back(side_bps(G, o ? G.s0 : G.s1));
        auto score_of = [&](uint32_t mask, int upto) {
            std::vector<int> has_hist(ns, 0), has_prim(ns, 0);
            int sc = 0;
            for (int g = 0; g < upto; ++g) {
                const int o = (mask >> g) & 1;
                const Group &G = pl.groups[g];
                const int A = o ? G.s1 : G.s0, B = o ? G.s0 : G.s1;
                if (!has_hist[A]) { has_hist[A] = 1; sc += 4; }
                if (!has_prim[B] && tb[o][g].size() + 1 <= kSubMax) { has_prim[B] = 1; sc += 2; }
            }
            return sc;
        };
        uint32_t best_mask = 0;
        if (const char *om = knob("GACE_ORIENT_MASK")) {        // design experiments: force one
            best_mask = (uint32_t)strtoul(om, nullptr, 0);
        } else if (G_ <= 12) {
            int best = -1;
            for (uint32_t m = 0; m < (1u << G_); ++m) {
                const int sc = score_of(m, (int)G_);
                if (sc > best) { best = sc; best_mask = m; }
            }
        } else {
            for (size_t g = 0; g < G_; ++g)
                if (score_of(best_mask | (1u << g), (int)g + 1) > score_of(best_mask, (int)g + 1)) best_mask |= 1u << g;
        }
        for (size_t g = 0; g < G_; ++g) {
            Group &G = pl.groups[g];
            const int o = (best_mask >> g) & 1;
            G.a = o ? G.s1 : G.s0;
            G.b = o ? G.s0 : G.s1;
            G.TB = tb[o][g];
            G.na = pl.slots[G.a].nb;
            // row stride = sub-bucket count rounded up to odd: rows then start in different
            // shared-memory banks, so a warp whose rows share one sub-bucket (a sorted B
            // column) does not serialise on a single bank (the extra column stays zero)
            G.nbs = ((uint32_t)G.TB.size() + 1) | 1u;
        }
    }
    phase("groups");
    // ---- budget: grids (+ the B side's bucket -> sub-bucket map) in increasing size while
    // they fit with 4 KB per predicate column kept for its lookup table; the rest per row
    size_t fixed = 256;
    for (auto &S : pl.slots)
        if (S.has_hll) fixed += 4 * kHllM;
    size_t lut_reserve = 0;
    for (auto &S : pl.slots) {
        lut_reserve += S.has_preds ? 4096 : 0;
        fixed += S.has_preds ? 4ull * S.nb : 0;        // worst case: every column keeps its own histogram
    }
    {
        std::vector<int> order(pl.groups.size());
        for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
        std::sort(order.begin(), order.end(), [&](int x, int y) {
            return (uint64_t)pl.groups[x].na * pl.groups[x].nbs < (uint64_t)pl.groups[y].na * pl.groups[y].nbs;
        });
        size_t used = 0;
        for (int gi : order) {
            Group &G = pl.groups[gi];
            const size_t need = 4ull * ((uint64_t)G.na * G.nbs + pl.slots[G.b].nb) + 64;
            if (fixed + used + need + lut_reserve <= kSmemBudget) used += need;
            else G.direct = true;
        }
        fixed += used;
    }
    size_t ndirect = 0;
    for (auto &G : pl.groups) ndirect += G.direct ? G.pq.size() : 0;
    fixed += 4 * ndirect;
    if (fixed > kSmemBudget)
        return fail(GACE_EUNSUPPORTED, "probe plan exceeds one CTA's shared memory (" + std::to_string(fixed) + " B)");
    // roles among the groups that got a grid
    for (size_t g = 0; g < pl.groups.size(); ++g) {
        Group &G = pl.groups[g];
        if (G.direct) continue;
        if (pl.slots[G.a].hist_grp < 0) pl.slots[G.a].hist_grp = (int)g;
        if (G.nbs <= kSubMax && pl.slots[G.b].prim_b < 0) {
            pl.slots[G.b].prim_b = (int)g;
            pl.slots[G.b].TBp = &G.TB;
            G.packed = true;
        }
    }

    phase("budget");
    // ---- lookup tables within the remaining budget
    const size_t lut_budget = kSmemBudget - fixed;
    for (auto &S : pl.slots) {
        if (!S.has_preds) continue;
        S.mode = MODE_LUT;
        S.clamp = false;
        if (S.T.empty()) {                       // every value in bucket 0
            S.base = S.dl;
            S.clamp = true;
            S.clamp_lo = S.clamp_hi = S.dl;
        } else if ((uint64_t)S.dh - (uint64_t)S.dl < (1ull << 32) && !t->host &&
                   ((uint64_t)S.T.back() - ((uint64_t)S.T.front() - 1)) * 4 > (uint64_t)S.dh - (uint64_t)S.dl) {
            S.base = S.dl;                       // domain cover, values never leave it
        } else if ((uint64_t)S.T.back() - ((uint64_t)S.T.front() - 1) < (1ull << 32)) {
            // breakpoint-span cover (host tables, or breakpoints in a small part of the domain:
            // much finer cells for two extra ops per key), keys clamped into it
            S.base = S.T.front() - 1;            // breakpoint-span cover, clamp into it
            S.clamp = true;
            S.clamp_lo = S.base;
            S.clamp_hi = S.T.back();
        } else {
            S.mode = MODE_SEARCH;
        }
    }
    // level-1 size target: 16 cells per breakpoint, 64..4096; coarsen the largest table while over budget
    std::vector<uint32_t> s1(pl.slots.size(), 0);
    auto span_of = [](const SlotPlan &S) -> uint64_t {
        return S.clamp ? (uint64_t)S.clamp_hi - (uint64_t)S.clamp_lo : (uint64_t)S.dh - (uint64_t)S.base;
    };
    // FMT1T on a non-negative (or all-negative) int32 domain: cells aligned to multiples of
    // 2^s1 of the key itself, so the kernel indexes with key >> s1 and folds the base into
    // the address immediate (one op per key less)
    auto t1_rebase = [](SlotPlan &S, uint32_t sh) {
        if (S.fmt != FMT1T || S.clamp || S.dtype != GACE_I32 || !(S.dl >= 0 || S.dh < 0)) return;
        S.base = (int64_t)((uint64_t)S.dl & ~((1ull << sh) - 1));
    };
    auto to_search = [](SlotPlan &S) {
        S.mode = MODE_SEARCH;
        S.clamp = false;
        S.l1.clear();
        S.l2.clear();
        S.lst.clear();
        S.n_l1 = S.n_l2 = S.n_lst = 0;
        S.built = false;
    };
    // S at level-1 shift s: sized by lut_estimate (built at the end), or built when the
    // estimate cannot size it; false = the table cannot be built
    auto size_lut = [&](SlotPlan &S, uint32_t s) -> bool {
        const LutEst E = lut_estimate(S, span_of(S), s);
        if (!E.exact || knob("GACE_NO_LUT_ESTIMATE")) return build_lut(S, span_of(S), s);
        S.s1 = s;
        S.l1.clear();
        S.l2.clear();
        S.lst.clear();
        S.n_l1 = E.l1;
        S.n_l2 = E.l2;
        S.n_lst = 0;
        S.built = false;
        return true;
    };
    // level-1 formats: exact cells (one per key value, HLL info folded in) for small int32
    // domains; 16-bit cells when buckets <= 512 and packed sub-buckets <= 64; else 32-bit
    auto small_subs = [&](const SlotPlan &S) { return S.prim_b < 0 || pl.groups[S.prim_b].nbs <= 64; };
    auto nsub_of = [&](const SlotPlan &S) -> uint32_t {
        return S.prim_b < 0 ? 1u : (uint32_t)pl.groups[S.prim_b].TB.size() + 1;
    };
    const bool use_t1 = !knob("GACE_NO_T1");      // design A/B switch (GACE_NO_T1=1: older formats)
    for (size_t i = 0; i < pl.slots.size(); ++i) {
        SlotPlan &S = pl.slots[i];
        if (S.mode != MODE_LUT) continue;
        const uint64_t span = span_of(S);
        const bool narrow = S.nb <= 512 && small_subs(S);
        S.sb = ceil_log2((uint64_t)S.nb + 1);
        uint32_t t1s = 0;                    // FMT1T level-1 shift: ~128 cells per breakpoint, <= 32K cells
        {
            uint64_t target = 64;
            while (target < (sparse ? 4096u : 32768u) && target < (sparse ? 16ull : 128ull) * S.T.size()) target <<= 1;
            while (t1s < 31 && (span >> t1s) + 1 > target) ++t1s;
            t1s = std::max<uint32_t>(t1s, 1);
            const uint32_t mx = t1_max_s1(S, nsub_of(S));     // finer than the target when the fields force it
            if (t1s > mx && mx >= 1 && (span >> mx) + 1 <= 32768) t1s = mx;
        }
        // exact cells: small int32 spans; up to 32767 buckets when no sub-bucket is packed
        // (bucket field bits 0..14: C3's 1025 EQ binds); a clamped span too -- keys outside
        // it land in an edge cell, so such a column never takes its HLL from the cells
        if (S.dtype == GACE_I32 && span < 16384 && (narrow || (S.prim_b < 0 && S.nb < 32768))) {
            S.fmt = FMTEX;
            s1[i] = 0;
        } else if (use_t1 && t1s <= t1_max_s1(S, nsub_of(S))) {
            S.fmt = FMT1T;
            s1[i] = t1s;
            t1_rebase(S, t1s);
        } else {
            S.fmt = narrow ? FMT16 : FMT32;
            const uint64_t cap = S.fmt == FMT16 ? 16384 : 8192;
            uint64_t target = 64;
            while (target < (sparse ? cap / 8 : cap) && target < (sparse ? 4ull : 32ull) * S.T.size()) target <<= 1;
            uint32_t sh = 0;
            while (sh < 31 && (span >> sh) + 1 > target) ++sh;
            s1[i] = sh;
        }
        if (!size_lut(S, s1[i]) || (S.fmt == FMT16 && S.n_l2 > kRecMask16)) to_search(S);
    }
    const std::vector<uint32_t> s1_target = s1;
    phase("luts-size");
    auto lut_total = [&]() {
        size_t tot = 0;
        for (auto &S : pl.slots)
            if (S.mode == MODE_LUT) tot += lut_bytes(S);
        return tot;
    };
    for (int iter = 0; iter < 256; ++iter) {
        size_t tot = 0;
        int worst = -1;
        size_t worst_sz = 0;
        for (size_t i = 0; i < pl.slots.size(); ++i) {
            const SlotPlan &S = pl.slots[i];
            if (S.mode != MODE_LUT) continue;
            const size_t sz = lut_bytes(S);
            tot += sz;
            if (sz > worst_sz) { worst_sz = sz; worst = (int)i; }
        }
        if (tot <= lut_budget || worst < 0) break;
        SlotPlan &S = pl.slots[worst];
        if (S.fmt == FMTEX) S.fmt = small_subs(S) && S.nb <= 512 ? FMT16 : FMT32;   // exact cells cost too much
        if (S.fmt == FMT1T && s1[worst] + 1 > t1_max_s1(S, nsub_of(S)))
            S.fmt = small_subs(S) && S.nb <= 512 ? FMT16 : FMT32;                  // thresholds no longer fit
        // a coarser level 1 roughly halves it; when nested blocks / lists dominate (dense
        // breakpoints) that column falls back to a binary search in global memory
        if (s1[worst] >= 31 || S.n_l1 <= 64 || 16 * S.n_l2 + 4 * S.n_lst > 4 * S.n_l1) {
            to_search(S);
            continue;
        }
        ++s1[worst];
        if (S.fmt == FMT1T) t1_rebase(S, s1[worst]);
        else if (!S.clamp && S.mode == MODE_LUT) S.base = S.dl;          // left FMT1T: plain domain cover
        if (!size_lut(S, s1[worst]) || (S.fmt == FMT16 && S.n_l2 > kRecMask16)) to_search(S);
    }
    phase("luts-fit");
    // refine again where the halving steps above left room: the table whose keys most often
    // land in a boundary cell (a record walk, and for the warp a divergent branch; keys taken
    // as uniform over the span) first, never finer than its target, same format
    for (int iter = 0; iter < 64 && !knob("GACE_NO_REFINE"); ++iter) {
        std::vector<std::pair<double, int>> cand;
        for (size_t i = 0; i < pl.slots.size(); ++i) {
            const SlotPlan &S = pl.slots[i];
            if (S.mode != MODE_LUT || S.fmt == FMTEX || s1[i] <= s1_target[i] || !S.n_l1) continue;
            // a clustered (sorted) column passes each boundary cell once per run, not per key
            if ((size_t)S.col < t->clustered.size() && t->clustered[S.col]) continue;
            // boundary cells (records) per cell
            if (S.n_l2) cand.push_back({-(double)S.n_l2 / (double)S.n_l1, (int)i});
        }
        std::sort(cand.begin(), cand.end());
        bool done = false;
        for (auto &c : cand) {
            const int i = c.second;
            SlotPlan keep = pl.slots[i];
            SlotPlan &S = pl.slots[i];
            --s1[i];
            if (S.fmt == FMT1T) t1_rebase(S, s1[i]);
            if (size_lut(S, s1[i]) && !(S.fmt == FMT16 && S.n_l2 > kRecMask16) && S.mode == MODE_LUT &&
                lut_total() <= lut_budget) {
                done = true;
                break;
            }
            S = keep;
            ++s1[i];
        }
        if (!done) break;
    }
    phase("luts-refine");
    // the tables sized by estimate: built once, at their final shift
    for (auto &S : pl.slots) {
        if (S.mode != MODE_LUT || S.built) continue;
        const uint64_t n1 = S.n_l1, n2 = S.n_l2;
        if (!build_lut(S, span_of(S), S.s1) || (S.fmt == FMT16 && S.n_l2 > kRecMask16)) {
            to_search(S);
            continue;
        }
        if (S.n_l1 != n1 || S.n_l2 != n2 || S.n_lst)
            return fail(GACE_EUNSUPPORTED, "internal: lookup-table size estimate differs from the built table");
    }

    phase("luts");
    // ---- HLL mode per column: a presence bitmap (one bit per value of a small int32 domain;
    // the finalize hashes each present value once) instead of hashing every key, when it
    // fits where the u32 registers were budgeted (exact: registers depend only on the set
    // of distinct kept values).  Exact-cell columns keep their per-cell (index, rank).
    {
        size_t used = fixed;
        for (auto &S : pl.slots)
            if (S.mode == MODE_LUT) used += lut_bytes(S);
        for (auto &S : pl.slots) {
            if (!S.has_hll || S.dtype != GACE_I32 || t->host || knob("GACE_NO_BITMAP")) continue;
            if (S.mode == MODE_LUT && S.fmt == FMTEX && !S.clamp) continue;   // (index, rank) in the cells
            const int64_t base = (int64_t)((uint64_t)S.dl & ~31ull);
            const uint64_t words = (((uint64_t)S.dh - (uint64_t)base) >> 5) + 1;
            if (words > 32768) continue;                        // <= 128 KB
            // zeroing and merging the bitmap costs ~words per CTA (and the finalize hashes every
            // present value on one CTA): worth it when every CTA scans many rows per bitmap word
            // (C4: 200M rows, 2K words; not C1's 1M rows, nor C3's 100M rows over 32K words --
            // measured there: scan unchanged, finalize +0.15 ms).  Rows per rank, not this
            // shard's own count, so every rank of a multi-GPU table makes the same choice.
            const uint64_t rows = t->has_dist ? t->dist.nrows_total / (uint64_t)t->dist.nranks : t->nrows;
            if (rows < 32ull * words * (uint64_t)t->sms && !knob("GACE_FORCE_BITMAP")) continue;
            const size_t bytes = 4 * words;
            if (bytes > 4ull * kHllM && used + bytes - 4ull * kHllM > kSmemBudget) continue;
            used = used + bytes - 4ull * kHllM;
            S.bm = true;
            S.bm_base = base;
            S.bm_words = (uint32_t)words;
        }
    }

    phase("hll");
    // ---- layout: image [per slot: L1 | nested | lists][maps] | acc [own hists][grids][direct] |
    //      presence bitmaps | hll registers
    uint32_t w = 0;    // u32 cursor
    for (auto &S : pl.slots) {
        if (S.mode != MODE_LUT) continue;
        w = (w + 3) & ~3u;
        S.l2_idx = w / 4;
        w += 4 * (uint32_t)S.l2.size();
        S.lut_idx = w;
        w += S.fmt == FMT16 ? ((uint32_t)S.l1.size() + 1) / 2 : (uint32_t)S.l1.size();
        S.lst_idx = w;
        w += (uint32_t)S.lst.size();
    }
    w = (w + 3) & ~3u;
    for (auto &G : pl.groups) {
        if (G.direct) continue;
        G.map_w = w;
        w += pl.slots[G.b].nb;
    }
    w = (w + 3) & ~3u;
    const uint32_t image_words = w;
    pl.acc_idx = w;
    for (auto &S : pl.slots) {
        if (!S.has_preds || S.hist_grp >= 0) continue;
        S.hist_w = w;
        w += S.nb;
    }
    for (auto &G : pl.groups) {
        if (G.direct) continue;
        G.grid_w = w;
        w += G.na * G.nbs;
    }
    const uint32_t direct_idx = w;
    w += (uint32_t)ndirect;
    w = (w + 3) & ~3u;
    pl.acc_words = w - pl.acc_idx;
    uint32_t gbm = 0;
    for (auto &S : pl.slots) {
        if (!S.bm) continue;
        S.bm_w = w;
        w += S.bm_words;
        S.bm_goff = gbm;
        gbm += (S.bm_words + 3) & ~3u;
    }
    pl.bm_gwords = gbm;
    w = (w + 3) & ~3u;
    pl.hll_off = w * 4;
    uint32_t nh = 0, nreg = 0;
    for (auto &S : pl.slots) {
        if (!S.has_hll) continue;
        S.hll_out = nh++;
        if (S.bm) continue;
        S.hll_idx = w + nreg * kHllM;
        ++nreg;
    }
    pl.hll_bytes = nh * kHllM;
    pl.smem_bytes = (uint32_t)align16(pl.hll_off + 4ull * nreg * kHllM);
    if (pl.smem_bytes > kSmemBudget)
        return fail(GACE_EUNSUPPORTED, "probe plan exceeds one CTA's shared memory");

    phase("layout");
    // exact cells of a clamped column in no pair group (C3's bind span) hold the byte address
    // of the key's own histogram bin: the kernel adds to it directly (SlotParams::fdirect)
    {
        std::vector<uint8_t> in_group(pl.slots.size(), 0);
        for (auto &G : pl.groups) in_group[G.s0] = in_group[G.s1] = 1;
        for (size_t i = 0; i < pl.slots.size(); ++i) {
            SlotPlan &S = pl.slots[i];
            S.fdirect = S.has_preds && S.mode == MODE_LUT && S.fmt == FMTEX && S.clamp && !in_group[i] &&
                        S.hist_grp < 0 && S.prim_b < 0 && S.hist_w != kNone && !knob("GACE_NO_FDIRECT");
        }
    }
    // ---- fill the image (absolute shared-memory indices)
    pl.image.assign((size_t)image_words * 4, 0);
    uint4 *img4 = reinterpret_cast<uint4 *>(pl.image.data());
    uint32_t *img32 = reinterpret_cast<uint32_t *>(pl.image.data());
    auto fix = [&](uint4 e, const SlotPlan &S) {   // relative record / list indices -> absolute
        if (!(e.x & kSpecial)) return e;
        if (e.x & kList) e.y += S.lst_idx;
        else e.y += S.l2_idx;
        return e;
    };
    for (auto &S : pl.slots) {
        if (S.mode != MODE_LUT) continue;
        uint16_t *img16 = reinterpret_cast<uint16_t *>(img32 + S.lut_idx);
        uint32_t *dst = img32 + S.lut_idx;
        const uint32_t *src = S.l1.data();
        const size_t n1 = S.l1.size();
        // one branch-free loop per format (vectorised; records are rare)
        if (S.fmt == FMT1T) {
            const uint32_t sp = t1_special(S.s1), dm = t1_dmask(S.s1), l2i = S.l2_idx;
            for (size_t k = 0; k < n1; ++k) {
                const uint32_t c = src[k];
                dst[k] = (c & sp) ? sp | (l2i + (c & dm)) : c;
            }
        } else if (S.fmt == FMT16) {
            const uint32_t l2i = S.l2_idx;
            for (size_t k = 0; k < n1; ++k) {
                const uint32_t c = src[k];
                img16[k] = (uint16_t)((c & kSpecial) ? 0x8000u | (l2i + (c & kRecMask))
                                                     : (c & kIdxMask) | (((c >> kSubShift) & kSubMask) << 9));
            }
        } else if (S.fmt == FMTEX) {                       // cell k is the key base + k
            const bool hll_cells = S.has_hll && !S.clamp && !S.bm;
            for (size_t k = 0; k < n1; ++k) {
                const uint32_t c = src[k];
                const uint32_t idx = c & kIdxMask, sub = (c >> kSubShift) & kSubMask;
                uint32_t hidx = 0, rank = 0;
                if (hll_cells) {
                    const uint32_t h = host_fmix32((uint32_t)(int32_t)(S.base + (int64_t)k));
                    hidx = h >> (32 - kHllP);
                    rank = (uint32_t)__builtin_clz((h << kHllP) | (1u << (kHllP - 1))) + 1;
                }
                dst[k] = S.fdirect ? 4 * (S.hist_w + idx) : idx | (sub << 9) | (hidx << 15) | (rank << 27);
            }
        } else {
            const uint32_t l2i = S.l2_idx;
            for (size_t k = 0; k < n1; ++k) {
                const uint32_t c = src[k];
                dst[k] = (c & kSpecial) ? kSpecial | (l2i + (c & kRecMask)) : c;
            }
        }
        for (size_t k = 0; k < S.l2.size(); ++k) img4[S.l2_idx + k] = fix(S.l2[k], S);
        for (size_t k = 0; k < S.lst.size(); ++k) img32[S.lst_idx + k] = S.lst[k];
    }
    for (auto &G : pl.groups) {
        if (G.direct) continue;
        const SlotPlan &B = pl.slots[G.b];
        for (uint32_t r = 0; r < B.nb; ++r) img32[G.map_w + r] = r == 0 ? 0 : count_le(G.TB, B.T[r - 1]);
    }

    phase("image");
    // ---- finalize plan
    uint32_t pre = 0;
    for (auto &S : pl.slots) {
        if (!S.has_preds || S.hist_grp >= 0) continue;
        S.pre = pre;
        S.pre_stride = 1;
        pl.jobs.push_back(FinJob{JOB_HIST, S.hist_w - pl.acc_idx, pre, 0, S.nb});
        pre += S.nb + 1;
    }
    for (auto &G : pl.groups) {
        if (G.direct) continue;
        G.sat = pre;
        pl.jobs.push_back(FinJob{JOB_SAT, G.grid_w - pl.acc_idx, pre, G.na, G.nbs});
        pre += (G.na + 1) * (G.nbs + 1);
    }
    for (auto &S : pl.slots) {           // grid-provided histograms: the SAT's last column
        if (S.hist_grp < 0) continue;
        const Group &G = pl.groups[S.hist_grp];
        S.pre = G.sat + G.nbs;
        S.pre_stride = G.nbs + 1;
    }
    pl.pre_words = pre;
    auto bucket_iv = [&](uint32_t p, const std::vector<int64_t> &T, uint32_t &lo, uint32_t &hi) {
        if (pl.iv[p].empty) { lo = 1; hi = 0; return; }
        lo = count_le(T, pl.iv[p].lo);
        hi = count_le(T, pl.iv[p].hi);
    };
    auto negated = [&](uint32_t p) -> uint32_t { return (preds[p].flags & GACE_PRED_NEGATE) ? 1 : 0; };
    // bucket intervals of the predicates on their own columns: every clipped interval end is a
    // breakpoint of the column (lo, or hi + 1), so its bucket is that breakpoint's position --
    // found in an open-addressing index of each column's breakpoints (O(1), not a search)
    struct BpIndex {
        std::vector<int64_t> key;
        std::vector<uint32_t> pos;
        uint64_t mask = 0;
        void build(const std::vector<int64_t> &T) {
            size_t cap = 16;
            while (cap < 2 * T.size()) cap <<= 1;
            key.assign(cap, 0);
            pos.assign(cap, kNone);
            mask = cap - 1;
            for (size_t i = 0; i < T.size(); ++i) {
                uint64_t h = ((uint64_t)T[i] * 0x9E3779B97F4A7C15ull) >> 20;
                while (pos[h & mask] != kNone) ++h;
                key[h & mask] = T[i];
                pos[h & mask] = (uint32_t)i;
            }
        }
        uint32_t find(int64_t x) const {            // index of x in T, or kNone
            for (uint64_t h = ((uint64_t)x * 0x9E3779B97F4A7C15ull) >> 20;; ++h) {
                if (pos[h & mask] == kNone) return kNone;
                if (key[h & mask] == x) return pos[h & mask];
            }
        }
    };
    std::vector<BpIndex> bpx(pl.slots.size());
    for (size_t i = 0; i < pl.slots.size(); ++i) bpx[i].build(pl.slots[i].T);
    auto bucket_iv_fast = [&](uint32_t p, int sl, uint32_t &lo, uint32_t &hi) {
        const Interval &I = pl.iv[p];
        const SlotPlan &S = pl.slots[sl];
        if (I.empty) { lo = 1; hi = 0; return; }
        const uint32_t a = I.lo > S.dl ? bpx[sl].find(I.lo) : kNone;
        const uint32_t b = I.hi < S.dh ? bpx[sl].find(I.hi + 1) : kNone;
        lo = I.lo > S.dl ? (a != kNone ? a + 1 : count_le(S.T, I.lo)) : 0u;
        hi = I.hi < S.dh ? (b != kNone ? b : count_le(S.T, I.hi)) : (uint32_t)S.T.size();
    };
    phase("fin-jobs");
    pl.fpreds.resize(np);
    for (uint32_t p = 0; p < np; ++p) {
        const SlotPlan &S = pl.slots[pl.pslot[p]];
        FinPred F{};
        F.pre = S.pre;
        F.stride = S.pre_stride;
        bucket_iv_fast(p, pl.pslot[p], F.lo, F.hi);
        F.neg = negated(p);
        pl.fpreds[p] = F;
    }
    phase("fin-preds");
    pl.fpairs.resize(nq);
    struct DEnt { uint32_t g, q; DirectPair D; };
    std::vector<DEnt> dlist;
    for (uint32_t q = 0; q < nq; ++q) {
        const uint32_t i = pairs[q].i, j = pairs[q].j;
        const int si = pl.pslot[i], sj = pl.pslot[j];
        FinPair F{};
        if (si == sj) {
            F.kind = PAIR_SAME;
            F.pre = pl.slots[si].pre;
            F.stride = pl.slots[si].pre_stride;
            bucket_iv(i, pl.slots[si].T, F.li, F.hi);
            bucket_iv(j, pl.slots[sj].T, F.lj, F.hj);
            F.negi = negated(i);
            F.negj = negated(j);
        } else {
            const int g = pl.gidx[std::make_pair(std::min(si, sj), std::max(si, sj))];
            const Group &G = pl.groups[g];
            const uint32_t pa = (si == G.a) ? i : j, pb = (si == G.a) ? j : i;
            if (G.direct) {
                DirectPair D{};
                bucket_iv(pa, pl.slots[G.a].T, D.la, D.ha);
                bucket_iv(pb, pl.slots[G.b].T, D.lb, D.hb);
                D.nega = negated(pa);
                D.negb = negated(pb);
                dlist.push_back({(uint32_t)g, q, D});
                F.kind = PAIR_DIRECT;
            } else {
                F.kind = PAIR_GRID;
                F.pre = G.sat;
                F.na = G.na;
                F.nb = G.nbs;
                bucket_iv(pa, pl.slots[G.a].T, F.li, F.hi);     // full resolution on A
                bucket_iv(pb, G.TB, F.lj, F.hj);                // sub-buckets on B
                F.negi = negated(pa);
                F.negj = negated(pb);
            }
        }
        pl.fpairs[q] = F;
    }
    // direct pairs grouped by column pair; each counter's slot = its position
    std::stable_sort(dlist.begin(), dlist.end(), [](const DEnt &x, const DEnt &y) { return x.g < y.g; });
    std::vector<uint32_t> dbeg(pl.groups.size(), 0), dend(pl.groups.size(), 0);
    for (uint32_t k = 0; k < dlist.size(); ++k) {
        DEnt &E = dlist[k];
        E.D.acc_idx = direct_idx + k;
        const Group &G = pl.groups[E.g];
        if (pl.slots[G.a].fmt == FMT1T) { ++E.D.la; ++E.D.ha; }      // 1-based buckets
        if (pl.slots[G.b].fmt == FMT1T) { ++E.D.lb; ++E.D.hb; }
        pl.fpairs[E.q].pre = direct_idx + k - pl.acc_idx;
        if (dend[E.g] == 0) dbeg[E.g] = k;
        dend[E.g] = k + 1;
        pl.direct.push_back(E.D);
    }

    phase("finalize");
    // ---- kernel parameters (pointers filled in at launch)
    ProbeParams &P = pl.P;
    memset(&P, 0, sizeof(P));
    P.nslots = (uint32_t)pl.slots.size();
    uint32_t bps = 0;
    for (size_t i = 0; i < pl.slots.size(); ++i) {
        SlotPlan &S = pl.slots[i];
        SlotParams &Q = P.slot[i];
        Q.dtype = (uint8_t)S.dtype;
        Q.mode = S.has_preds ? S.mode : (uint8_t)MODE_NOPRED;
        Q.has_hll = S.has_hll ? 1 : 0;
        Q.hll_idx = S.hll_idx;
        Q.bm_addr = S.bm ? 4 * S.bm_w : kNone;
        Q.bm_words = S.bm_words;
        Q.bm_goff = S.bm_goff;
        Q.bm_base = S.bm_base;
        Q.bm_nvals = S.bm ? (uint32_t)((uint64_t)S.dh - (uint64_t)S.dl + 1) : 0u;
        // register ceilings: R[j] can never exceed the largest rank among the domain values
        // with index j, so once the merged registers reach them the column is complete and
        // the scan stops hashing its keys (register columns, domains <= 2^25 values)
        // (a property of the column, not of the batch: computed once per attached column on
        // the GPU -- gace_probe launches it the first time a plan needs it -- and kept in the
        // table's d_hceil at byte offset col * 4096)
        Q.hceil_off = kNone;
        if (S.has_hll && !S.bm && !(S.has_preds && S.mode == MODE_LUT && S.fmt == FMTEX && !S.clamp) &&
            (uint64_t)S.dh - (uint64_t)S.dl < (1ull << 25) && !t->host && !knob("GACE_NO_CEIL"))
            Q.hceil_off = (uint32_t)S.col * kHllM;
        Q.hll_out = S.hll_out;
        Q.hist_addr = S.hist_w == kNone ? kNone : 4 * S.hist_w;
        Q.fdirect = S.fdirect ? 1 : 0;
        Q.prim_b = (int8_t)S.prim_b;
        Q.base = S.base;
        Q.s1 = S.s1;
        Q.lut_w = S.lut_idx;
        Q.fmt = S.fmt;
        // bs layout per format: the plain level-1 word is used as bs directly
        const bool lutm = S.has_preds && S.mode == MODE_LUT;
        Q.sb = (uint8_t)(!lutm ? 16 : S.fmt == FMT1T ? S.sb : S.fmt == FMT32 ? kSubShift
                                                : (S.fmt == FMTEX && S.nb > 512) ? 15 : 9);
        Q.bmask = (1u << Q.sb) - 1u;
        Q.submask = !lutm || S.fmt == FMT1T ? 0xFFFFFFFFu : S.fmt == FMT32 ? kSubMask : 63u;
        Q.sub_mul = 1u << (32 - Q.sb);
        Q.cell_mul = S.s1 >= 1 ? 1u << (32 - S.s1) : 0u;
        if (S.fmt == FMT1T) {
            Q.t1_mul = 1u << (32 - S.s1);
            Q.t1_ones = Q.t1_mul - 1u;
            Q.t1_dmask = t1_dmask(S.s1);
            Q.t1_sp = t1_special(S.s1);
            Q.t1_cutsh = 30 - S.s1 - S.sb;
            Q.t1_cutmul = Q.t1_cutsh ? 1u << (32 - Q.t1_cutsh) : 0u;
        }
        if (S.fmt == FMT1T && S.hist_w != kNone) Q.hist_addr -= 4;     // 1-based buckets
        if (S.dtype == GACE_I32) { Q.clamp_lo = INT32_MIN; Q.clamp_hi = INT32_MAX; }
        else { Q.clamp_lo = INT64_MIN; Q.clamp_hi = INT64_MAX; }
        if (S.has_preds && S.mode == MODE_LUT && S.clamp) {
            Q.clamp_lo = S.clamp_lo;
            Q.clamp_hi = S.clamp_hi;
            pl.clamp = true;
        }
        if (slot_foldable(Q)) {
            Q.fold_b = 4 * Q.lut_w - 4 * (uint32_t)((uint64_t)Q.base >> Q.s1);
            Q.fold_z = Q.fmt == FMT1T ? Q.t1_ones - (uint32_t)Q.base * Q.t1_mul : 0u;
        }
        if (S.has_preds && S.mode == MODE_SEARCH) {
            S.bps_off = bps;
            Q.nbp = (uint32_t)S.T.size();
            for (int64_t x : S.T) pl.bps.push_back(x);
            bps += (uint32_t)S.T.size();
        }
    }
    for (size_t g = 0; g < pl.groups.size(); ++g) {
        const Group &G = pl.groups[g];
        GroupParams &R = P.grp[g];
        R.a = (uint8_t)G.a;
        R.b = (uint8_t)G.b;
        R.dbeg = (uint16_t)dbeg[g];
        R.dend = (uint16_t)dend[g];
        R.has_grid = G.direct ? 0 : 1;
        R.packed = G.packed ? 1 : 0;
        R.nbs = G.nbs;
        R.grid_addr = G.direct ? kNone : 4 * G.grid_w;
        R.map_addr = G.direct ? kNone : 4 * G.map_w;
        if (!G.direct && pl.slots[G.a].fmt == FMT1T) R.grid_addr -= 4 * G.nbs;   // 1-based A buckets
        if (!G.direct && pl.slots[G.b].fmt == FMT1T) R.map_addr -= 4;          // 1-based B buckets
    }
    P.ngroups = (uint32_t)pl.groups.size();
    P.c1 = 1;
    P.c4 = 4;
    P.c_hll = 1u << kHllP;
    P.clamp = pl.clamp ? 1u : 0u;      // (the specialised kernel bakes this in: set it here)
    P.ndirect = (uint32_t)pl.direct.size();
    P.image_u4 = image_words / 4;
    P.acc_idx = pl.acc_idx;
    P.acc_words = pl.acc_words;
    P.hll_off = pl.hll_off;
    P.hll_bytes = pl.hll_bytes;
    P.smem_bytes = pl.smem_bytes;
    phase("params");
    if (knob("GACE_PLAN_DUMP")) dump_plan(pl);
    return GACE_OK;
}

// ------------------------------------------------------------------ validation helpers

int popcount64(uint64_t x) { return __builtin_popcountll(x); }

gace_status check_table(const gace_table *t) {
    if (!t || t->magic != kMagic) return fail(GACE_EHANDLE, "invalid or detached table handle");
    return GACE_OK;
}

// per_item = false: the batch is byte-identical to the table's cached (validated) batch, so
// the per-predicate / per-pair checks are skipped (repeated probes: no O(P) host work)
gace_status validate_batch(const gace_table *t, const gace_pred *preds, uint32_t np, const gace_pair *pairs,
                           uint32_t nq, double rate, uint64_t hll_mask, uint32_t hll_p, bool per_item = true) {
    if (np > GACE_MAX_PREDS) return fail(GACE_EINVAL, "npreds > 4096");
    if (nq > GACE_MAX_PAIRS) return fail(GACE_EINVAL, "npairs > 4096");
    if (np && !preds) return fail(GACE_EINVAL, "preds is NULL");
    if (nq && !pairs) return fail(GACE_EINVAL, "pairs is NULL");
    if (!(rate >= 0.0 && rate <= 1.0)) return fail(GACE_EINVAL, "sample_rate must be in [0, 1]");
    if (t->ncols < 64 && (hll_mask >> t->ncols)) return fail(GACE_EINVAL, "hll_col_mask names a column >= ncols");
    if (!per_item) return hll_p != GACE_HLL_P ? fail(GACE_EUNSUPPORTED, "hll_p must be 12") : GACE_OK;
    for (uint32_t p = 0; p < np; ++p) {
        if (preds[p].col >= t->ncols) return fail(GACE_EINVAL, "predicate column out of range");
        if (preds[p].op > GACE_BETWEEN) return fail(GACE_EINVAL, "unknown predicate op");
        if (preds[p].flags & ~GACE_PRED_NEGATE) return fail(GACE_EINVAL, "unknown predicate flags");
    }
    for (uint32_t q = 0; q < nq; ++q)
        if (pairs[q].i >= np || pairs[q].j >= np) return fail(GACE_EINVAL, "pair index out of range");
    if (hll_p != GACE_HLL_P) return fail(GACE_EUNSUPPORTED, "hll_p must be 12");
    return GACE_OK;
}

uint64_t threshold_of(double rate) { return rate >= 1.0 ? ~0ull : (uint64_t)std::ldexp(rate, 64); }

gace_status attach_common(const void *const *ptrs, const gace_dtype *dtypes, uint32_t ncols, uint64_t nrows,
                          const gace_dist *dist, int device, void *stream, bool host, gace_table **out) {
    refresh_knobs();
    if (!out) return fail(GACE_EINVAL, "out is NULL");
    if (!ptrs || !dtypes) return fail(GACE_EINVAL, "column pointers / dtypes are NULL");
    if (ncols == 0 || ncols > GACE_MAX_COLS) return fail(GACE_EINVAL, "ncols must be in [1, 64]");
    for (uint32_t c = 0; c < ncols; ++c) {
        if (dtypes[c] != GACE_I32 && dtypes[c] != GACE_I64) return fail(GACE_EINVAL, "unknown dtype");
        if (!ptrs[c] && nrows) return fail(GACE_EINVAL, "NULL column pointer");
        if (!host && ((uintptr_t)ptrs[c] & 15)) return fail(GACE_EINVAL, "column pointer not 16-byte aligned");
    }
    if (dist) {
        if (dist->nranks < 1 || dist->rank < 0 || dist->rank >= dist->nranks)
            return fail(GACE_EINVAL, "bad rank / nranks");
        if (dist->nranks > 1 && !dist->nccl_unique_id && !dist->nccl_comm)
            return fail(GACE_EINVAL, "multi-rank attach needs an NCCL unique id or comm");
        if (dist->row_offset > dist->nrows_total || nrows > dist->nrows_total - dist->row_offset)
            return fail(GACE_EINVAL, "row_offset + nrows_local exceeds nrows_total");
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(GACE_ECUDA, "no CUDA device");
    if (device < 0 || device >= ndev) return fail(GACE_EINVAL, "bad device ordinal");
    CUDA_TRY(cudaSetDevice(device));
    gace_table *t = new gace_table();
    t->device = device;
    t->host = host;
    t->ncols = ncols;
    t->nrows = nrows;
    t->cols.assign(ptrs, ptrs + ncols);
    for (uint32_t c = 0; c < ncols; ++c) t->dtypes.push_back((int)dtypes[c]);
    cudaDeviceGetAttribute(&t->sms, cudaDevAttrMultiProcessorCount, device);
    auto bail = [&](gace_status s) {
        gace_table_detach(t);
        return s;
    };
    if (stream) {
        t->stream = (cudaStream_t)stream;
    } else {
        if (cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking) != cudaSuccess)
            return bail(fail(GACE_ECUDA, "stream create failed"));
        t->own_stream = true;
    }
    for (int i = 0; i < kNumEv; ++i)
        if (cudaEventCreate(&t->ev[i]) != cudaSuccess) return bail(fail(GACE_ECUDA, "event create failed"));
    // value domains
    t->dlo.resize(ncols);
    t->dhi.resize(ncols);
    for (uint32_t c = 0; c < ncols; ++c) {
        t->dlo[c] = dtypes[c] == GACE_I32 ? INT32_MIN : INT64_MIN;
        t->dhi[c] = dtypes[c] == GACE_I32 ? INT32_MAX : INT64_MAX;
    }
    t->clustered.assign(ncols, 0);
    t->hceil_ready.assign(ncols, 0);
    if (!host && (t->d_hceil.ensure((size_t)ncols * kHllM) != cudaSuccess || t->d_hceil32.ensure(4 * kHllM) != cudaSuccess))
        return bail(fail(GACE_ENOMEM, "HLL ceiling buffers"));
    if (!host && nrows) {
        DevBuf mm;
        if (mm.ensure(24 * ncols) != cudaSuccess) return bail(fail(GACE_ENOMEM, "minmax scratch"));
        std::vector<long long> init(3 * ncols);
        for (uint32_t c = 0; c < ncols; ++c) { init[3 * c] = LLONG_MAX; init[3 * c + 1] = LLONG_MIN; init[3 * c + 2] = 0; }
        cudaMemcpyAsync(mm.p, init.data(), 24 * ncols, cudaMemcpyHostToDevice, t->stream);
        for (uint32_t c = 0; c < ncols; ++c) {
            if (launch_minmax(ptrs[c], dtypes[c], nrows, mm.as<long long>(24 * c), t->sms, t->stream) != cudaSuccess) {
                mm.release();
                return bail(fail(GACE_ECUDA, "minmax launch failed"));
            }
            ++g_launches;
        }
        cudaMemcpyAsync(init.data(), mm.p, 24 * ncols, cudaMemcpyDeviceToHost, t->stream);
        cudaError_t e = cudaStreamSynchronize(t->stream);
        mm.release();
        if (e != cudaSuccess) return bail(fail(GACE_ECUDA, std::string("attach scan: ") + cudaGetErrorString(e)));
        for (uint32_t c = 0; c < ncols; ++c) {
            t->dlo[c] = init[3 * c];
            t->dhi[c] = init[3 * c + 1];
            t->clustered[c] = 2ull * (uint64_t)init[3 * c + 2] >= nrows / 4 && nrows >= 4;
        }
    }
    if (host) {
        if (cudaStreamCreateWithFlags(&t->copy_stream, cudaStreamNonBlocking) != cudaSuccess)
            return bail(fail(GACE_ECUDA, "copy stream create failed"));
        for (int b = 0; b < 2; ++b) {
            if (cudaEventCreateWithFlags(&t->ev_copied[b], cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&t->ev_free[b], cudaEventDisableTiming) != cudaSuccess)
                return bail(fail(GACE_ECUDA, "event create failed"));
        }
        if (cudaEventCreate(&t->ev_c0) != cudaSuccess || cudaEventCreate(&t->ev_c1) != cudaSuccess)
            return bail(fail(GACE_ECUDA, "event create failed"));
    }
    if (dist) {
        t->has_dist = true;
        t->dist = *dist;
        t->dist.nccl_unique_id = nullptr;
        t->use_nccl = dist->nranks > 1 || dist->nccl_unique_id || dist->nccl_comm;
        if (t->use_nccl) {
            if (dist->nccl_comm) {
                t->comm = dist->nccl_comm;
            } else {
                Nccl *n = nccl();
                if (!n) return bail(fail(GACE_ENCCL, "libnccl.so.2 not loadable"));
                NcclUid id;
                memcpy(&id, dist->nccl_unique_id, sizeof(id));
                int r = n->CommInitRank(&t->comm, dist->nranks, id, dist->rank);
                if (r != 0) return bail(fail(GACE_ENCCL, std::string("ncclCommInitRank: ") + (n->GetErrorString ? n->GetErrorString(r) : "")));
                t->own_comm = true;
            }
            // every rank plans over the same global value domains (min of the minima, max of
            // the maxima), so identical batches give identical plans -- the same lookup
            // tables, grids, limits and errors -- on every rank; an empty shard is neutral
            if (!host) {
                std::vector<long long> dom(2 * ncols);
                for (uint32_t c = 0; c < ncols; ++c) {
                    dom[c] = nrows ? t->dlo[c] : LLONG_MAX;
                    dom[ncols + c] = nrows ? t->dhi[c] : LLONG_MIN;
                }
                Nccl *n = nccl();
                if (t->d_coll.ensure(std::max<size_t>(16ull * ncols, 64)) != cudaSuccess)
                    return bail(fail(GACE_ENOMEM, "collective scratch"));
                long long *d = t->d_coll.as<long long>();
                if (cudaMemcpyAsync(d, dom.data(), 16ull * ncols, cudaMemcpyHostToDevice, t->stream) != cudaSuccess)
                    return bail(fail(GACE_ECUDA, "domain agreement copy"));
                n->GroupStart();
                const int r1 = n->AllReduce(d, d, ncols, kNcclInt64, kNcclMin, t->comm, t->stream);
                const int r2 = n->AllReduce(d + ncols, d + ncols, ncols, kNcclInt64, kNcclMax, t->comm, t->stream);
                const int r3 = n->GroupEnd();
                if (r1 || r2 || r3) return bail(fail(GACE_ENCCL, "domain agreement all-reduce failed"));
                if (cudaMemcpyAsync(dom.data(), d, 16ull * ncols, cudaMemcpyDeviceToHost, t->stream) != cudaSuccess)
                    return bail(fail(GACE_ECUDA, "domain agreement copy"));
                const gace_status ws = wait_stream(t, t->stream);
                if (ws) return bail(ws);
                for (uint32_t c = 0; c < ncols; ++c) {
                    if (dom[c] > dom[ncols + c]) continue;          // every shard empty: dtype range
                    t->dlo[c] = dom[c];
                    t->dhi[c] = dom[ncols + c];
                }
            }
            // the fused merge (NCCL device API, NVLink peer loads; gace_merge.cu) when every
            // rank is load/store reachable; else the grouped all-reduce (GACE_NCCL_FUSED=0 forces it)
            const char *fz = knob("GACE_NCCL_FUSED");
            if (!(fz && !atoi(fz)) && merge_available()) {
                std::string why;
                if (!merge_create(t->comm, dist->nranks, kMergeBytes, &t->merge, &why)) t->merge = nullptr;
            }
        }
    }
    *out = t;
    return GACE_OK;
}

// Planning is deterministic in (global domains, batch), so ranks given the same batch
// build the same plan.  A new plan is still agreed on before any data collective: every
// rank contributes its planning status and a hash of its batch; if any rank failed, or
// the batches differ, every rank returns an error instead of entering the merge that the
// others would never join (identical arguments are part of the collective contract).
gace_status agree_plan(gace_table *t, gace_status local, const std::string &key) {
    if (!t->use_nccl || !t->comm) return local;
    if (t->comm_dead) return fail(GACE_ENCCL, "NCCL communicator was aborted by an earlier error");
    Nccl *n = nccl();
    const std::string err = local ? g_err : std::string();
    const long long h = (long long)(std::hash<std::string>{}(key) >> 1);
    long long v[4] = {local ? 1 : 0, h, h, 0};
    CUDA_TRY(cudaSetDevice(t->device));
    if (t->d_coll.ensure(64) != cudaSuccess) return fail(GACE_ENOMEM, "collective scratch");
    long long *d = t->d_coll.as<long long>();
    CUDA_TRY(cudaMemcpyAsync(d, v, 32, cudaMemcpyHostToDevice, t->stream));
    n->GroupStart();
    const int r1 = n->AllReduce(d, d, 2, kNcclInt64, kNcclMax, t->comm, t->stream);
    const int r2 = n->AllReduce(d + 2, d + 2, 1, kNcclInt64, kNcclMin, t->comm, t->stream);
    const int r3 = n->GroupEnd();
    if (r1 || r2 || r3) return fail(GACE_ENCCL, "plan agreement all-reduce failed");
    CUDA_TRY(cudaMemcpyAsync(v, d, 32, cudaMemcpyDeviceToHost, t->stream));
    const gace_status ws = wait_stream(t, t->stream);
    if (ws) return ws;
    if (local) return fail(local, err);
    if (v[0]) return fail(GACE_EINVAL, "another rank failed to plan this batch (collective call aborted)");
    if (v[1] != v[2]) return fail(GACE_EINVAL, "ranks passed different batches to a collective probe");
    return GACE_OK;
}

}  // namespace

namespace {

// Source of `struct JitShape` for gace_probe.cuh: the plan's structural decisions as
// constexpr answers (predicate values stay in the kernel parameters).
// Threads per CTA of a plan's specialised kernel (gace_plan.h kThreads): 768 (<= 80 registers)
// when the column-streamed keys of one row unit need >= 24 registers (4 per int32 column, 8
// per int64), 1024 (<= 64) otherwise.  Measured (profiles/r02_threads_sweep.txt): C4's 8
// columns 1.43 -> 1.29 ms, C5_i64 2.88 -> 2.76 ms at 768; C5's 4 int32 columns 2.06 at 1024,
// 2.16 at 768.  GACE_JIT_THREADS overrides (1024 / 768 / 512).
int jit_threads(const Plan &pl) {
    if (const char *e = knob("GACE_JIT_THREADS")) {
        const int v = atoi(e);
        if (v == 1024 || v == 768 || v == 512) return v;
    }
    uint32_t key_regs = 0;
    for (uint32_t i = 0; i < pl.P.nslots; ++i) key_regs += pl.P.slot[i].dtype ? 8 : 4;
    return key_regs >= 24 ? 768 : 1024;
}

// layout = false: the structure only (layout read from the parameters, gace_probe.cuh
// RtLayout), so every batch with this structure shares one compiled kernel; layout = true:
// offsets, shifts and masks baked in as immediates too (one kernel per batch layout).
std::string jit_shape_source(const Plan &pl, bool sample, bool i64, const std::vector<uint8_t> &clustered,
                             bool layout) {
    // (every piece appended in place: a new batch's structure-keyed source is generated on the
    // probe's host path, so no temporaries per term)
    const ProbeParams &P = pl.P;
    const int nc = (int)P.nslots;
    std::string o;
    o.reserve(layout ? 8192 : 4096);
    char nb[64];
    auto num = [&](long long v) { o.append(nb, (size_t)(std::to_chars(nb, nb + sizeof nb, v).ptr - nb)); };
    auto bit = [&](bool v) { o += v ? '1' : '0'; };
    auto tf = [&](bool v) { o += v ? "true" : "false"; };
    // "s == 0 ? f(0) : s == 1 ? f(1) : ... 0" (f appends its term)
    auto chain = [&](auto f, int n) {
        for (int i = 0; i < n; ++i) {
            o += "s == ";
            num(i);
            o += " ? ";
            f(i);
            o += " : ";
        }
        o += '0';
    };
    auto gchain = [&](auto f) {
        for (uint32_t g = 0; g < P.ngroups; ++g) {
            o += "g == ";
            num(g);
            o += " ? ";
            f(g);
            o += " : ";
        }
        o += '0';
    };
    // one trait: "  __device__ static constexpr <type> <name>(<args>) { return <chain>; }\n"
    auto trait = [&](const char *head, auto body) {
        o += "  __device__ static constexpr ";
        o += head;
        o += " { return ";
        body();
        o += "; }\n";
    };
    const int threads = jit_threads(pl);
    if (threads != 1024) {
        o += "#define GACE_THREADS ";
        num(threads);
        o += '\n';
    }
    o += "namespace gace {\nstruct JitShape : RtLayout {\n";
    o += "  static constexpr int NC = ";
    num(nc);
    o += ";\n  static constexpr bool SAMPLE = ";
    tf(sample);
    o += ";\n  static constexpr bool I64 = ";
    tf(i64);
    o += ";\n  static constexpr bool STATIC = true;\n";
    o += "  static constexpr int U = NC >= 4 ? 1 : 4 / NC;\n";
    o += "  static constexpr int NG = ";
    num(P.ngroups);
    o += ";\n";
    {   // no HLL column: the skip-bound refresh points are compiled out
        bool any_hll = false;
        for (uint32_t i = 0; i < P.nslots; ++i) any_hll |= P.slot[i].has_hll != 0;
        o += "  static constexpr bool ANY_HLL = ";
        tf(any_hll);
        o += ";\n";
    }
    o += "  __device__ static constexpr bool active(const ProbeParams &, int s) { return s < NC; }\n";
    auto slot_bits = [&](const char *head, auto pred) {
        trait(head, [&] { chain([&](int i) { bit(pred(i)); }, nc); });
    };
    trait("int mode(const ProbeParams &, int s)", [&] { chain([&](int i) { num((int)P.slot[i].mode); }, nc); });
    slot_bits("bool is32(const ProbeParams &, int s)", [&](int i) { return P.slot[i].dtype == 0; });
    slot_bits("bool hll(const ProbeParams &, int s)", [&](int i) { return P.slot[i].has_hll != 0; });
    trait("bool clamp(const ProbeParams &)", [&] { tf(P.clamp != 0); });
    slot_bits("bool packs(const ProbeParams &, int s)", [&](int i) { return P.slot[i].prim_b >= 0; });
    trait("int fmt(const ProbeParams &, int s)", [&] { chain([&](int i) { num((int)P.slot[i].fmt); }, nc); });
    slot_bits("bool clust(const ProbeParams &, int s)", [&](int i) { return clustered[i] != 0; });
    slot_bits("bool fdirect(const ProbeParams &, int s)", [&](int i) { return P.slot[i].fdirect != 0; });
    slot_bits("bool ownh(const ProbeParams &, int s)",
              [&](int i) { return P.slot[i].mode != MODE_NOPRED && P.slot[i].hist_addr != kNone; });
    trait("int ga(int g)", [&] { gchain([&](uint32_t g) { num((int)P.grp[g].a); }); });
    trait("int gb(int g)", [&] { gchain([&](uint32_t g) { num((int)P.grp[g].b); }); });
    trait("bool gpacked(int g)", [&] { gchain([&](uint32_t g) { bit(P.grp[g].packed != 0); }); });
    trait("bool ggrid(int g)", [&] { gchain([&](uint32_t g) { bit(P.grp[g].has_grid != 0); }); });
    trait("bool gdirect(int g)", [&] { gchain([&](uint32_t g) { bit(P.grp[g].dend > P.grp[g].dbeg); }); });
    {
        const char *ab = knob("GACE_ABLATE");          // design experiments: ablations baked in
        trait("uint32_t dbg(const ProbeParams &)", [&] {
            num(ab ? (long long)(uint32_t)strtoul(ab, nullptr, 0) : 0ll);
            o += 'u';
        });
    }
    slot_bits("bool hllbm(const ProbeParams &, int s)", [&](int i) { return P.slot[i].bm_addr != kNone; });
    slot_bits("bool fold(const ProbeParams &, int s)", [&](int i) { return slot_foldable(P.slot[i]); });
    slot_bits("bool sclamp(const ProbeParams &, int s)", [&](int i) {
        const SlotParams &Q = P.slot[i];
        return Q.dtype == 0 ? (Q.clamp_lo != INT32_MIN || Q.clamp_hi != INT32_MAX)
                            : (Q.clamp_lo != INT64_MIN || Q.clamp_hi != INT64_MAX);
    });
    if (!layout) {
        o += "};\n}  // namespace gace\n";
        return o;
    }
    // plan layout as immediates (the lookup-table contents stay in shared memory)
    auto u32 = [&](uint32_t v) {
        num(v);
        o += 'u';
    };
    auto i64v = [&](int64_t v) {
        if (v == INT64_MIN) o += "(int64_t)(-9223372036854775807LL - 1)";
        else {
            o += "(int64_t)";
            num((long long)v);
            o += "LL";
        }
    };
    auto slot_u32 = [&](const char *name, auto f) {
        o += "  __device__ static constexpr uint32_t ";
        o += name;
        o += "(const ProbeParams &, int s) { return ";
        chain([&](int i) { u32(f(P.slot[i])); }, nc);
        o += "; }\n";
    };
    auto slot_i64 = [&](const char *name, auto f) {
        o += "  __device__ static constexpr int64_t ";
        o += name;
        o += "(const ProbeParams &, int s) { return ";
        chain([&](int i) { i64v(f(P.slot[i])); }, nc);
        o += "; }\n";
    };
    auto grp_u32 = [&](const char *name, auto f) {
        o += "  __device__ static constexpr uint32_t ";
        o += name;
        o += "(const ProbeParams &, int g) { return ";
        gchain([&](uint32_t g) { u32(f(P.grp[g])); });
        o += "; }\n";
    };
    slot_i64("base", [](const SlotParams &Q) { return Q.base; });
    slot_u32("foldb", [&](const SlotParams &Q) { return Q.fold_b; });
    slot_u32("foldz", [&](const SlotParams &Q) { return Q.fold_z; });
    slot_i64("clo", [](const SlotParams &Q) { return Q.clamp_lo; });
    slot_i64("chi", [](const SlotParams &Q) { return Q.clamp_hi; });
    slot_u32("s1", [](const SlotParams &Q) { return Q.s1; });
    slot_u32("lutb", [](const SlotParams &Q) { return 4 * Q.lut_w; });
    slot_u32("histb", [](const SlotParams &Q) { return Q.hist_addr; });
    slot_u32("hllw", [](const SlotParams &Q) { return Q.hll_idx; });
    slot_u32("bmaddr", [](const SlotParams &Q) { return Q.bm_addr; });
    slot_u32("bmbase", [](const SlotParams &Q) { return (uint32_t)Q.bm_base; });
    slot_u32("bmnv", [](const SlotParams &Q) { return Q.bm_nvals; });
    slot_u32("hllout", [](const SlotParams &Q) { return Q.hll_out; });
    slot_u32("sb", [](const SlotParams &Q) { return (uint32_t)Q.sb; });
    slot_u32("bmask", [](const SlotParams &Q) { return Q.bmask; });
    slot_u32("t1mul", [](const SlotParams &Q) { return Q.t1_mul; });
    slot_u32("t1ones", [](const SlotParams &Q) { return Q.t1_ones; });
    slot_u32("t1dmask", [](const SlotParams &Q) { return Q.t1_dmask; });
    slot_u32("t1sp", [](const SlotParams &Q) { return Q.t1_sp; });
    slot_u32("t1cutsh", [](const SlotParams &Q) { return Q.t1_cutsh; });
    slot_u32("t1cutmul", [](const SlotParams &Q) { return Q.t1_cutmul; });
    slot_u32("submask", [](const SlotParams &Q) { return Q.submask; });
    slot_u32("submul", [](const SlotParams &Q) { return Q.sub_mul; });
    slot_u32("cellmul", [](const SlotParams &Q) { return Q.cell_mul; });
    slot_u32("mapb", [&](const SlotParams &Q) { return Q.prim_b >= 0 ? P.grp[Q.prim_b].map_addr : kNone; });
    grp_u32("ggridb", [](const GroupParams &G) { return G.grid_addr; });
    grp_u32("gnbs", [](const GroupParams &G) { return G.nbs; });
    grp_u32("gmapb", [](const GroupParams &G) { return G.map_addr; });
    o += "};\n}  // namespace gace\n";
    return o;
}

// Which specialised kernels (GACE_JIT_LAYOUT): 0 the structure-keyed one only; 1 the
// layout-keyed one only (compiled per batch layout); unset / 2: the structure-keyed one at
// once and the layout-keyed one compiled in the background, used once it is loaded.
int jit_layout_mode() {
    const char *e = knob("GACE_JIT_LAYOUT");
    if (!e) return 2;
    const int v = atoi(e);
    return v < 0 || v > 2 ? 2 : v;
}
bool jit_layout() { return jit_layout_mode() == 1; }

// Launches of at least this many rows use a specialised kernel once it is compiled
// (GACE_JIT_MIN_ROWS, default 65536): even C1's 1M rows gain from it (scan 0.035 -> 0.026 ms,
// wall p50 0.088 -> 0.078 ms, profiles/r02_c1_jit.txt); below the default a table is too
// small for a background compile to be worth it.
uint64_t jit_min_rows() {
    const char *e = knob("GACE_JIT_MIN_ROWS");
    return (e && *e) ? strtoull(e, nullptr, 10) : 65536ull;
}

// GACE_JIT=0: never specialise; 1: always, compiling a missing kernel synchronously; unset:
// launches of >= jit_min_rows() rows use a specialised kernel if one is compiled, else the generic
// kernel while the specialised one compiles in the background (no call waits for NVRTC).
int jit_mode() {
    const char *e = knob("GACE_JIT");
    if (!e) return 2;
    return atoi(e) ? 1 : 0;
}

}  // namespace

// ====================================================================== C-ABI

// ------------------------------------------------------------------ candidate sets

namespace {

// Operator as written (DESIGN.md §2 step 4), used to evaluate each member predicate on a
// bucket's representative value: independent of the interval normalisation that places
// the breakpoints, so a breakpoint slip shows up as a parity failure, not as agreement.
bool eval_pred(const gace_pred &p, int64_t v) {
    bool r;
    switch (p.op) {
        case GACE_EQ: r = v == p.a; break;
        case GACE_LT: r = v < p.a; break;
        case GACE_LE: r = v <= p.a; break;
        case GACE_GT: r = v > p.a; break;
        case GACE_GE: r = v >= p.a; break;
        default: r = p.a <= v && v <= p.b;
    }
    return (p.flags & GACE_PRED_NEGATE) ? !r : r;
}

struct SetsPlan {
    SetsParams P{};
    std::vector<uint32_t> cols;        // table column of each slot
    std::vector<uint8_t> image;        // cells | breakpoints | sat masks
    bool i64 = false;
    uint64_t bytes_per_row = 0;
};

constexpr size_t kSetsSmemHard = 200 * 1024;   // one 1024-thread CTA per SM

// Planner of gace_probe_sets (DESIGN.md §6 "Candidate sets").  For each probed column:
// sorted breakpoints of its member predicates' intervals clipped to the column domain
// (every predicate is constant on each bucket), sat[b] = bitmask of the sets all of whose
// members on this column hold on bucket b, and a cell table over the domain (cell word =
// first bucket of the cell | breakpoints inside << 20) sized to the shared-memory budget.
gace_status make_sets_plan(const gace_table *t, const gace_pred *preds, const uint32_t *offs,
                           const uint32_t *mem, uint32_t nsets, SetsPlan &out) {
    const uint32_t W = nsets <= 32 ? 1 : nsets <= 64 ? 2 : nsets <= 128 ? 4 : 8;
    const bool fold = nsets <= 31;             // bit 31 of a cell word is free: masks in the cells
    std::map<uint32_t, uint32_t> slot_of;      // table column -> slot
    for (uint32_t m = 0; m < nsets; ++m)
        for (uint32_t k = offs[m]; k < offs[m + 1]; ++k) {
            const uint32_t c = preds[mem[k]].col;
            if (!slot_of.count(c)) {
                if (slot_of.size() == (size_t)kSetsMaxCols)
                    return fail(GACE_EUNSUPPORTED, "candidate sets reference more than 8 columns");
                const uint32_t sl = (uint32_t)slot_of.size();
                slot_of[c] = sl;
            }
        }
    const uint32_t ns = (uint32_t)slot_of.size();
    out.cols.assign(ns, 0);
    for (auto &kv : slot_of) out.cols[kv.second] = kv.first;
    std::vector<std::vector<uint64_t>> bps(ns);        // offsets t - dlo, sorted, unique
    std::vector<std::vector<uint32_t>> sat(ns);
    size_t fixed = 0;
    for (uint32_t sl = 0; sl < ns; ++sl) {
        const uint32_t c = out.cols[sl];
        const int64_t dl = t->dlo[c], dh = t->dhi[c];
        std::vector<int64_t> T;
        for (uint32_t m = 0; m < nsets; ++m)
            for (uint32_t k = offs[m]; k < offs[m + 1]; ++k)
                if (preds[mem[k]].col == c) add_breakpoints(clip(op_interval(preds[mem[k]]), dl, dh), dl, dh, T);
        std::sort(T.begin(), T.end());
        T.erase(std::unique(T.begin(), T.end()), T.end());
        const uint32_t nb = (uint32_t)T.size() + 1;
        if (nb >= (1u << kSetsCellB0Bits)) return fail(GACE_EUNSUPPORTED, "too many breakpoints on one column");
        for (int64_t x : T) bps[sl].push_back((uint64_t)x - (uint64_t)dl);
        sat[sl].assign((size_t)nb * W, 0xFFFFFFFFu);
        for (uint32_t b = 0; b < nb; ++b) {
            const int64_t rep = b == 0 ? dl : T[b - 1];       // every value of bucket b behaves alike
            for (uint32_t m = 0; m < nsets; ++m)
                for (uint32_t k = offs[m]; k < offs[m + 1]; ++k) {
                    const gace_pred &p = preds[mem[k]];
                    if (p.col == c && !eval_pred(p, rep)) {
                        sat[sl][(size_t)b * W + m / 32] &= ~(1u << (m % 32));
                        break;
                    }
                }
        }
        fixed += 8 * bps[sl].size() + 4 * sat[sl].size() + 16;
    }
    if (fixed > kSetsSmemHard) return fail(GACE_EUNSUPPORTED, "candidate-set plan exceeds shared memory");
    const size_t cell_words = ns ? (kSetsSmemHard - fixed) / 4 / ns : 0;     // per slot
    std::vector<std::vector<uint32_t>> cells(ns);
    for (uint32_t sl = 0; sl < ns; ++sl) {
        const uint32_t c = out.cols[sl];
        const uint64_t span = (uint64_t)t->dhi[c] - (uint64_t)t->dlo[c];
        const std::vector<uint64_t> &B = bps[sl];
        // ~256 cells per bucket: few keys land in a cell holding a breakpoint
        const uint64_t want = std::min<uint64_t>(cell_words, std::max<uint64_t>(256ull * (B.size() + 1), 1024));
        uint32_t sh = 0;
        while (sh < 63 && (span >> sh) >= want) ++sh;
        for (;; --sh) {                       // finer cells while a cell holds too many breakpoints
            const uint64_t nc = (span >> sh) + 1;
            if (nc > cell_words) return fail(GACE_EUNSUPPORTED, "candidate-set cells exceed shared memory");
            std::vector<uint32_t> cw(nc);
            size_t i = 0;
            bool ok = true;
            // b0 = #{t <= cell start}: a breakpoint at the cell start does not split the cell;
            // n = #{t in (start, end]}, searched in bps[b0 .. b0 + n)
            for (uint64_t cell = 0; cell < nc; ++cell) {
                const uint64_t cs = cell << sh;
                while (i < B.size() && B[i] <= cs) ++i;
                size_t e = i;
                const uint64_t ce_minus1 = cs + ((sh >= 64) ? ~0ull : ((1ull << sh) - 1));   // inclusive end
                while (e < B.size() && B[e] <= ce_minus1) ++e;
                if (e - i > kSetsCellNMax) { ok = false; break; }
                cw[cell] = (uint32_t)i | ((uint32_t)(e - i) << kSetsCellB0Bits);
                if (fold) cw[cell] = e == i ? sat[sl][i] & ~kSetsImpure : cw[cell] | kSetsImpure;
            }
            if (ok) { cells[sl].swap(cw); out.P.col[sl].shift = sh; break; }
            if (sh == 0) return fail(GACE_EUNSUPPORTED, "candidate-set cell overflow");
        }
    }
    // image: cells (u32) | breakpoints (u64, 8-aligned) | sat (u32)
    size_t w32 = 0;
    for (uint32_t sl = 0; sl < ns; ++sl) { out.P.col[sl].cell_off = (uint32_t)w32; w32 += cells[sl].size(); }
    w32 = (w32 + 1) & ~size_t(1);
    size_t w64 = w32 / 2;
    for (uint32_t sl = 0; sl < ns; ++sl) { out.P.col[sl].bps_off = (uint32_t)w64; w64 += bps[sl].size(); }
    w32 = 2 * w64;
    for (uint32_t sl = 0; sl < ns; ++sl) { out.P.col[sl].sat_off = (uint32_t)w32; w32 += sat[sl].size(); }
    const size_t bytes = std::max<size_t>(align16(4 * w32), 16);
    if (bytes > kSetsSmemHard) return fail(GACE_EUNSUPPORTED, "candidate-set plan exceeds shared memory");
    out.image.assign(bytes, 0);
    uint32_t *i32 = reinterpret_cast<uint32_t *>(out.image.data());
    uint64_t *i64p = reinterpret_cast<uint64_t *>(out.image.data());
    for (uint32_t sl = 0; sl < ns; ++sl) {
        std::copy(cells[sl].begin(), cells[sl].end(), i32 + out.P.col[sl].cell_off);
        std::copy(bps[sl].begin(), bps[sl].end(), i64p + out.P.col[sl].bps_off);
        std::copy(sat[sl].begin(), sat[sl].end(), i32 + out.P.col[sl].sat_off);
        const uint32_t c = out.cols[sl];
        out.P.col[sl].dlo = t->dlo[c];
        out.P.col[sl].is64 = t->dtypes[c] == GACE_I64 ? 1u : 0u;
        out.i64 |= t->dtypes[c] == GACE_I64;
        out.bytes_per_row += t->dtypes[c] == GACE_I64 ? 8 : 4;
    }
    out.P.ncols = ns;
    out.P.W = W;
    out.P.fold = fold ? 1u : 0u;
    out.P.image_u4 = (uint32_t)(bytes / 16);
    return GACE_OK;
}

}  // namespace

extern "C" {

const char *gace_last_error(void) { return g_err.c_str(); }

uint64_t gace_kernel_launches(void) { return g_launches.load(); }

gace_status gace_nccl_unique_id(void *id128) {
    if (!id128) return fail(GACE_EINVAL, "id is NULL");
    Nccl *n = nccl();
    if (!n) return fail(GACE_ENCCL, "libnccl.so.2 not loadable");
    NcclUid id;
    int r = n->GetUniqueId(&id);
    if (r != 0) return fail(GACE_ENCCL, "ncclGetUniqueId failed");
    memcpy(id128, &id, sizeof(id));
    return GACE_OK;
}

gace_status gace_table_attach(const void *const *col_dev_ptrs, const gace_dtype *dtypes, uint32_t ncols,
                              uint64_t nrows_local, const gace_dist *dist, int device, void *cuda_stream,
                              gace_table **out) {
    return attach_common(col_dev_ptrs, dtypes, ncols, nrows_local, dist, device, cuda_stream, false, out);
}

gace_status gace_table_attach_host(const void *const *col_host_ptrs, const gace_dtype *dtypes, uint32_t ncols,
                                   uint64_t nrows_local, const gace_dist *dist, int device, void *cuda_stream,
                                   gace_table **out) {
    return attach_common(col_host_ptrs, dtypes, ncols, nrows_local, dist, device, cuda_stream, true, out);
}

gace_status gace_table_detach(gace_table *t) {
    if (!t || t->magic != kMagic) return fail(GACE_EHANDLE, "invalid or detached table handle");
    cudaSetDevice(t->device);
    if (t->stream) cudaStreamSynchronize(t->stream);
    if (t->copy_stream) cudaStreamSynchronize(t->copy_stream);
    if (t->merge && !t->comm_dead) merge_destroy(t->merge);
    t->merge = nullptr;
    if (t->own_comm && t->comm && !t->comm_dead) {
        Nccl *n = nccl();
        if (n) n->CommDestroy(t->comm);
    }
    t->d_coll.release();
    t->d_hceil.release();
    t->d_hceil32.release();
    for (auto &e : t->ev) if (e) cudaEventDestroy(e);
    for (int b = 0; b < 2; ++b) {
        if (t->ev_copied[b]) cudaEventDestroy(t->ev_copied[b]);
        if (t->ev_free[b]) cudaEventDestroy(t->ev_free[b]);
        t->d_stage[b].release();
    }
    if (t->ev_c0) cudaEventDestroy(t->ev_c0);
    if (t->ev_c1) cudaEventDestroy(t->ev_c1);
    if (t->gexec) cudaGraphExecDestroy(t->gexec);
    t->d_plan.release(); t->d_accb[0].release(); t->d_accb[1].release(); t->d_pre.release(); t->d_part.release();
    t->d_out.release(); t->d_nsamp.release(); t->d_mask.release();
    t->h_plan.release(); t->h_out.release();
    t->d_sets_img.release(); t->d_sets_out.release(); t->h_sets_img.release(); t->h_sets_out.release();
    if (t->copy_stream) cudaStreamDestroy(t->copy_stream);
    if (t->own_stream && t->stream) cudaStreamDestroy(t->stream);
    t->magic = 0;
    delete t;
    return GACE_OK;
}

gace_status gace_table_set_graphs(gace_table *t, int enable) {
    gace_status st = check_table(t);
    if (st) return st;
    std::lock_guard<std::mutex> lock(t->mu);
    t->graphs = enable != 0;
    t->gprev_ok = false;
    if (!t->graphs && t->gexec) {
        cudaSetDevice(t->device);
        if (t->stream) cudaStreamSynchronize(t->stream);
        cudaGraphExecDestroy(t->gexec);
        t->gexec = nullptr;
    }
    return GACE_OK;
}

gace_status gace_table_graph_stats(const gace_table *t, uint64_t *captures, uint64_t *replays) {
    gace_status st = check_table(t);
    if (st) return st;
    if (captures) *captures = t->g_captures;
    if (replays) *replays = t->g_replays;
    return GACE_OK;
}

gace_status gace_probe(gace_table *t, const gace_pred *preds, uint32_t npreds, const gace_pair *pairs,
                       uint32_t npairs, double sample_rate, uint64_t seed, uint64_t hll_col_mask, uint32_t hll_p,
                       uint64_t *n_sampled, uint64_t *counts, uint64_t *joint_counts, uint8_t *hll_regs) {
    gace_status st = check_table(t);
    if (st) return st;
    refresh_knobs();
    std::lock_guard<std::mutex> lock(t->mu);
    if (npreds > GACE_MAX_PREDS || npairs > GACE_MAX_PAIRS) return fail(GACE_EINVAL, "npreds / npairs > 4096");
    if ((npreds && !preds) || (npairs && !pairs)) return fail(GACE_EINVAL, "preds / pairs is NULL");
    const bool sparse_plan = sample_rate < 0.125;          // make_plan's sparse hint (part of the key)
    const bool full_plan = sample_rate >= 1.0;             // full scan: the larger smem budget (idem)
    std::string key;
    key.reserve(24 * (size_t)npreds + 8 * (size_t)npairs + 9);
    key.push_back(sparse_plan ? 's' : full_plan ? 'f' : 'd');
    key.append(reinterpret_cast<const char *>(&hll_col_mask), 8);
    if (npreds) key.append(reinterpret_cast<const char *>(preds), sizeof(gace_pred) * npreds);
    if (npairs) key.append(reinterpret_cast<const char *>(pairs), sizeof(gace_pair) * npairs);
    const bool cached = t->plan && key == t->plan_key;
    st = validate_batch(t, preds, npreds, pairs, npairs, sample_rate, hll_col_mask, hll_p, !cached);
    if (st) return st;
    const int nh = popcount64(hll_col_mask);
    if (!n_sampled) return fail(GACE_EINVAL, "n_sampled is NULL");
    if (npreds && !counts) return fail(GACE_EINVAL, "counts is NULL");
    if (npairs && !joint_counts) return fail(GACE_EINVAL, "joint_counts is NULL");
    if (nh && !hll_regs) return fail(GACE_EINVAL, "hll_regs is NULL");

    CUDA_TRY(cudaSetDevice(t->device));
    if (t->dirty) {                                              // an aborted call's work is done
        st = wait_stream(t, t->stream);
        if (st) return st;
    }
    t->dirty = true;                                             // (a completed call synchronised)
    t->timing_kind = 0;
    if (!cached) {
        auto fresh = std::make_shared<Plan>();
        st = agree_plan(t, make_plan(t, preds, npreds, pairs, npairs, hll_col_mask, *fresh, sparse_plan, full_plan), key);
        if (st) return st;
        const Plan &q = *fresh;
        // the cached plan is replaced below: until then (and on any failure) no plan is
        // current, so a later call can never launch the old plan over a half-written blob
        t->plan.reset();
        t->plan_key.clear();
        // ---- one pinned blob -> one H2D copy: image | direct | jobs | fpreds | fpairs | bps
        size_t off = 0;
        t->o_img = off; off = align16(off + q.image.size());
        t->o_dir = off; off = align16(off + q.direct.size() * sizeof(DirectPair));
        t->o_job = off; off = align16(off + q.jobs.size() * sizeof(FinJob));
        t->o_fp = off; off = align16(off + q.fpreds.size() * sizeof(FinPred));
        t->o_fq = off; off = align16(off + q.fpairs.size() * sizeof(FinPair));
        t->o_bps = off; off = align16(off + q.bps.size() * sizeof(int64_t));
        t->blob = std::max<size_t>(off, 16);
        if (t->h_plan.ensure(t->blob) != cudaSuccess || t->d_plan.ensure(t->blob) != cudaSuccess)
            return fail(GACE_ENOMEM, "plan buffers");
        char *hb = t->h_plan.as<char>();
        memcpy(hb + t->o_img, q.image.data(), q.image.size());
        if (!q.direct.empty()) memcpy(hb + t->o_dir, q.direct.data(), q.direct.size() * sizeof(DirectPair));
        if (!q.jobs.empty()) memcpy(hb + t->o_job, q.jobs.data(), q.jobs.size() * sizeof(FinJob));
        if (!q.fpreds.empty()) memcpy(hb + t->o_fp, q.fpreds.data(), q.fpreds.size() * sizeof(FinPred));
        if (!q.fpairs.empty()) memcpy(hb + t->o_fq, q.fpairs.data(), q.fpairs.size() * sizeof(FinPair));
        if (!q.bps.empty()) memcpy(hb + t->o_bps, q.bps.data(), q.bps.size() * sizeof(int64_t));
        CUDA_TRY(cudaMemcpyAsync(t->d_plan.p, hb, t->blob, cudaMemcpyHostToDevice, t->stream));
        t->plan = fresh;
        t->plan_key.swap(key);
        t->plan_gen++;
        t->plan_calls = 0;
        for (int i = 0; i < 2; ++i) {
            t->jit_fn[i] = nullptr;
            t->jit_kind[i] = 0;
            t->jit_ssrc[i].clear();
            t->jit_lsrc[i].clear();
        }
    }
    const Plan &pl = *static_cast<const Plan *>(t->plan.get());
    const size_t o_img = t->o_img, o_dir = t->o_dir, o_job = t->o_job, o_fp = t->o_fp, o_fq = t->o_fq, o_bps = t->o_bps;

    // persistent grid: one CTA per SM; a small table gets fewer CTAs (GACE_ROWS_PER_CTA: at
    // least that many rows each), since every CTA pays a fixed cost -- zeroing its shared
    // accumulators and registers, loading the plan image, flushing its partials
    int grid = t->sms;
    if (const char *rp = knob("GACE_ROWS_PER_CTA")) {
        const uint64_t per = strtoull(rp, nullptr, 10);
        if (per && !t->host) grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(t->sms, (t->nrows + per - 1) / per));
    }
    // + merged HLL bound registers + merged presence bitmaps
    // + n_sampled counter at the end, so one memset clears the whole accumulator
    const size_t nsamp_off = align16(8ull * pl.acc_words + 4ull * pl.hll_bytes + 4ull * pl.bm_gwords + 4ull * kMaxSlots + 16);
    const size_t acc_bytes = nsamp_off + 16;
    const size_t part_bytes = std::max<size_t>((size_t)grid * pl.hll_bytes, 16);
    const size_t out_words = 1 + npreds + npairs;
    const size_t out_bytes = align16(8 * out_words) + pl.hll_bytes;
    const bool use_graph = t->graphs && !t->host && t->nrows > 0 && t->stream != nullptr && !t->use_nccl;
    // graphs bake in one accumulator buffer and keep the memset; eager calls alternate
    const bool dbuf = !use_graph && !knob("GACE_NO_ACC_DBUF");
    const int ab = dbuf ? t->acc_next : 0, ob = ab ^ 1;
    DevBuf &acc = t->d_accb[ab];
    const bool need_memset = !(dbuf && t->acc_clean[ab] && acc.cap >= acc_bytes);
    t->acc_clean[0] = t->acc_clean[1] = false;
    if (dbuf && t->d_accb[ob].ensure(acc_bytes) != cudaSuccess) return fail(GACE_ENOMEM, "probe scratch");
    if (acc.ensure(acc_bytes) != cudaSuccess || t->d_pre.ensure(std::max<size_t>(8ull * pl.pre_words, 8)) != cudaSuccess ||
        t->d_part.ensure(part_bytes) != cudaSuccess || t->d_out.ensure(out_bytes) != cudaSuccess ||
        t->h_out.ensure(out_bytes) != cudaSuccess)
        return fail(GACE_ENOMEM, "probe scratch");

    cudaStream_t s = t->stream;
    // CUDA-graph replay (gace_table_set_graphs): the second call with the same plan, sample,
    // seed and scratch buffers captures the enqueue below (memsets, scan, finalize, D2H and
    // the stage events as external records); later identical calls launch the graph.
    uint64_t nl = 0;                 // our kernel launches enqueued by this call
    int merge_kind = 0;              // 0 one rank, 1 grouped all-reduce, 2 fused peer-memory kernel
    uint64_t launches = 0;
    double jit_ms = 0;
    int jit_used = 0;
    uint64_t bytes_per_row = 0;
    for (auto &S : pl.slots) bytes_per_row += S.dtype == GACE_I32 ? 4 : 8;
    const char *ab_env = knob("GACE_ABLATE");
    // ---- scan kernel for this call's large launches (gace_probe.cuh)
    const bool sample = sample_rate < 1.0;
    bool i64 = false;
    for (auto &S : pl.slots) i64 |= S.dtype == GACE_I64;
    const int jm = jit_mode(), jl = jit_layout_mode();
    ++t->plan_calls;
    // rows per launch: keep every CTA's u32 bins below 2^31
    // (and unit indices within 32 bits: <= 2^31 units of 4..16 rows)
    // (sampled launches: <= 2^31 rows, so the compacted row ids fit 32 bits)
    uint64_t max_rows = std::min<uint64_t>((uint64_t)grid * kThreads * (1ull << 19),
                                           sample_rate < 1.0 ? (1ull << 31) : (1ull << 33));
    if (const char *ml = knob("GACE_MAX_LAUNCH_ROWS")) {     // tests: force chunked launches
        const uint64_t m = strtoull(ml, nullptr, 10) & ~3ull;
        if (m) max_rows = std::min(max_rows, m);
    }
    const uint64_t big_launch = t->host ? std::min<uint64_t>(t->nrows, 1ull << 24) : std::min(t->nrows, max_rows);
    void *scan_fn = nullptr;
    int scan_kind = 0;
    std::string jit_err;
    if (pl.P.nslots > 0 && (jm == 1 || (jm == 2 && big_launch >= jit_min_rows()))) {
        const int si = sample ? 1 : 0;
        void *&fn = t->jit_fn[si];
        if (fn && t->jit_kind[si] == 1 && !t->jit_lsrc[si].empty()) {     // layout-keyed kernel loaded yet?
            void *f2 = nullptr;
            if (jit_lookup(t->device, t->jit_lsrc[si], &f2)) {
                fn = f2;
                t->jit_kind[si] = 2;
                t->jit_lsrc[si].clear();
            }
        }
        if (!fn) {
            std::vector<uint8_t> cl(pl.slots.size(), 0);
            for (size_t i = 0; i < pl.slots.size(); ++i) cl[i] = t->clustered[pl.slots[i].col];
            if (t->jit_ssrc[si].empty()) t->jit_ssrc[si] = jit_shape_source(pl, sample, i64, cl, jl == 1);
            if (jl == 2 && !t->jit_lsrc[si].empty() && jit_lookup(t->device, t->jit_lsrc[si], &fn)) {
                t->jit_kind[si] = 2;                               // repeat of a batch seen before
                t->jit_lsrc[si].clear();
            } else if (!jit_lookup(t->device, t->jit_ssrc[si], &fn)) {
                fn = nullptr;
                if (jm == 1) {
                    if (!jit_get(t->device, t->jit_ssrc[si], &fn, &jit_ms, &jit_err)) fn = nullptr;
                } else {
                    jit_prefetch(t->device, t->jit_ssrc[si]);      // generic kernel meanwhile
                }
            }
            if (fn && t->jit_kind[si] != 2) t->jit_kind[si] = jl == 1 ? 2 : 1;
        }
        // a batch probed again is worth its own layout-keyed kernel (compiled in the
        // background; a stream of distinct batches never generates or queues one)
        if (jl == 2 && t->plan_calls >= 2 && t->jit_kind[si] == 1 && t->jit_lsrc[si].empty()) {
            std::vector<uint8_t> cl(pl.slots.size(), 0);
            for (size_t i = 0; i < pl.slots.size(); ++i) cl[i] = t->clustered[pl.slots[i].col];
            t->jit_lsrc[si] = jit_shape_source(pl, sample, i64, cl, true);
            jit_prefetch(t->device, t->jit_lsrc[si]);
        }
        scan_fn = fn;
        scan_kind = fn ? t->jit_kind[si] : 0;
        if (!fn && jm == 1) {
            scan_kind = -1;
            g_err = "jit unavailable, generic kernel used: " + jit_err;
        }
    }
    GraphKey gk{t->plan_gen, sample_rate, seed, ab_env ? (uint32_t)strtoul(ab_env, nullptr, 0) : 0u,
                acc.p, t->d_pre.p, t->d_part.p, t->d_out.p, t->h_out.p, scan_fn, t->d_plan.p};
    const bool replay = use_graph && t->gexec && gk == t->gkey;
    bool capt = use_graph && !replay && t->gprev_ok && gk == t->gprev;
    if (use_graph && !replay) {
        t->gprev = gk;
        t->gprev_ok = true;
    }
    if (replay) {
        CUDA_TRY(cudaGraphLaunch(t->gexec, s));
        launches = t->g_scan_launches;
        jit_used = t->g_jit;
        g_launches += t->g_nl;
        t->g_replays++;
    } else {
    if (capt && cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
        (void)cudaGetLastError();
        capt = false;
    }
    auto rec = [&](cudaEvent_t e, cudaStream_t st) {
        return capt ? cudaEventRecordWithFlags(e, st, cudaEventRecordExternal) : cudaEventRecord(e, st);
    };
    const gace_status est = [&]() -> gace_status {
    CUDA_TRY(rec(t->ev[0], s));
    if (need_memset) CUDA_TRY(cudaMemsetAsync(acc.p, 0, acc_bytes, s));
    CUDA_TRY(rec(t->ev[1], s));

    ProbeParams P = pl.P;
    P.image = t->d_plan.as<const uint4>(o_img);
    P.direct = t->d_plan.as<const DirectPair>(o_dir);
    P.g_hceil = t->d_hceil.as<const uint8_t>();
    for (size_t i = 0; i < pl.slots.size(); ++i) {       // ceilings of the columns that need them
        const int c = pl.slots[i].col;
        if (P.slot[i].hceil_off == kNone || t->hceil_ready[c]) continue;
        CUDA_TRY(launch_hll_ceilings(t->dlo[c], (uint64_t)t->dhi[c] - (uint64_t)t->dlo[c], t->dtypes[c] == GACE_I64,
                                     t->d_hceil32.as<uint32_t>(), t->d_hceil.as<uint8_t>((size_t)c * kHllM), t->sms, s));
        nl += 2;
        t->hceil_ready[c] = 1;
    }
    for (size_t i = 0; i < pl.slots.size(); ++i)
        if (P.slot[i].mode == MODE_SEARCH) P.slot[i].bps = t->d_plan.as<const int64_t>(o_bps) + pl.slots[i].bps_off;
    P.g_acc = acc.as<unsigned long long>();
    P.g_hll_glob = acc.as<uint32_t>(8ull * pl.acc_words);
    P.g_bm = acc.as<uint32_t>(8ull * pl.acc_words + 4ull * pl.hll_bytes);
    P.g_bmcnt = acc.as<uint32_t>(8ull * pl.acc_words + 4ull * pl.hll_bytes + 4ull * pl.bm_gwords);
    P.g_hll_part = t->d_part.as<uint8_t>();
    P.g_nsamp = acc.as<unsigned long long>(nsamp_off);
    P.thr = threshold_of(sample_rate);
    P.seed = seed;
    P.sample_all = sample_rate >= 1.0 ? 1u : 0u;
    // samples below 3/8: kept rows compacted per warp (gace_probe.cuh s_queue); above, the
    // whole-quad path.  Measured on C5 (tools/compact_sweep.py): compaction 2.64 / 2.32 / 2.02 ms
    // at rates 0.3 / 0.2 / 0.1 against 3.23 / 3.24 / 3.38 for whole quads, 3.84 against 3.16 at
    // 0.5.  GACE_COMPACT=0/1 overrides.
    P.compact = knob("GACE_COMPACT") ? (uint32_t)(atoi(knob("GACE_COMPACT")) != 0) : (sample_rate < 0.375 ? 1u : 0u);
    if (ab_env) P.dbg = (uint32_t)strtoul(ab_env, nullptr, 0);   // design experiments only
    const uint64_t row_offset = t->has_dist ? t->dist.row_offset : 0;

    // the specialised kernel (resolved above) for large launches, generic precompiled otherwise
    auto launch_scan = [&](const ProbeParams &PP, uint64_t n) -> cudaError_t {
        if (scan_fn && (jm == 1 || n >= jit_min_rows())) {
            std::string err;
            if (jit_launch_fn(scan_fn, PP, grid, jit_threads(pl), s, &err)) {
                jit_used = scan_kind;
                return cudaSuccess;
            }
            jit_used = -1;     // fall back to the generic GPU kernel; reason in gace_last_error()
            g_err = "jit launch failed, generic kernel used: " + err;
        } else if (scan_kind < 0) {
            jit_used = -1;
        }
        return launch_probe(PP, sample, i64, grid, s);
    };
    if (t->nrows == 0) {
        CUDA_TRY(cudaMemsetAsync(t->d_part.p, 0, part_bytes, s));
    } else if (!t->host) {
        for (uint64_t r0 = 0; r0 < t->nrows; r0 += max_rows) {
            const uint64_t n = std::min(max_rows, t->nrows - r0);
            for (size_t i = 0; i < pl.slots.size(); ++i) {
                const size_t w = pl.slots[i].dtype == GACE_I32 ? 4 : 8;
                P.slot[i].ptr = static_cast<const char *>(t->cols[pl.slots[i].col]) + r0 * w;
            }
            P.nrows = n;
            P.row0 = row_offset + r0;
            P.part_merge = launches ? 1u : 0u;
            CUDA_TRY(launch_scan(P, n));
            ++launches;
        }
    } else {
        // host table: double-buffered H2D of the probed columns, overlapped with the scan
        const uint64_t chunk = std::min<uint64_t>((t->nrows + 3) & ~3ull, 1ull << 24);
        const size_t stage_bytes = align16(chunk * bytes_per_row) + 16 * pl.slots.size();
        if (t->d_stage[0].ensure(stage_bytes) != cudaSuccess || t->d_stage[1].ensure(stage_bytes) != cudaSuccess)
            return fail(GACE_ENOMEM, "host-table staging");
        CUDA_TRY(cudaEventRecord(t->ev_free[0], s));
        CUDA_TRY(cudaEventRecord(t->ev_free[1], s));
        CUDA_TRY(cudaStreamWaitEvent(t->copy_stream, t->ev[1], 0));
        CUDA_TRY(cudaEventRecord(t->ev_c0, t->copy_stream));
        uint64_t k = 0;
        for (uint64_t r0 = 0; r0 < t->nrows; r0 += chunk, ++k) {
            const int b = (int)(k & 1);
            const uint64_t n = std::min(chunk, t->nrows - r0);
            CUDA_TRY(cudaStreamWaitEvent(t->copy_stream, t->ev_free[b], 0));
            size_t so = 0;
            for (size_t i = 0; i < pl.slots.size(); ++i) {
                const size_t w = pl.slots[i].dtype == GACE_I32 ? 4 : 8;
                char *dst = t->d_stage[b].as<char>(so);
                CUDA_TRY(cudaMemcpyAsync(dst, static_cast<const char *>(t->cols[pl.slots[i].col]) + r0 * w, n * w,
                                         cudaMemcpyHostToDevice, t->copy_stream));
                P.slot[i].ptr = dst;
                so = align16(so + chunk * w);
            }
            CUDA_TRY(cudaEventRecord(t->ev_copied[b], t->copy_stream));
            CUDA_TRY(cudaStreamWaitEvent(s, t->ev_copied[b], 0));
            P.nrows = n;
            P.row0 = row_offset + r0;
            P.part_merge = launches ? 1u : 0u;
            CUDA_TRY(launch_scan(P, n));
            ++launches;
            CUDA_TRY(cudaEventRecord(t->ev_free[b], s));
        }
        CUDA_TRY(cudaEventRecord(t->ev_c1, t->copy_stream));
    }
    nl += launches;
    CUDA_TRY(rec(t->ev[2], s));

    FinParams F{};
    F.jobs = t->d_plan.as<const FinJob>(o_job);
    F.njobs = (uint32_t)pl.jobs.size();
    F.hll_bytes = pl.hll_bytes;
    F.nparts = (t->nrows == 0) ? 1 : (uint32_t)grid;
    F.hll_blocks = pl.hll_bytes ? (pl.hll_bytes / 4 + 63) / 64 : 0;      // fin_prefix: 64 register words per block
    F.g_acc = acc.as<const unsigned long long>();
    F.g_pre = t->d_pre.as<unsigned long long>();
    F.g_hll_part = t->d_part.as<const uint8_t>();
    F.g_nsamp = acc.as<const unsigned long long>(nsamp_off);
    F.preds = t->d_plan.as<const FinPred>(o_fp);
    F.npreds = npreds;
    F.pairs = t->d_plan.as<const FinPair>(o_fq);
    F.npairs = npairs;
    // one rank: the finalize kernels write the packed result straight into the pinned host
    // buffer (mapped under UVA, same address), so no D2H copy is queued; with several ranks
    // the result stays on the device for the NCCL merge and is copied back after it
    const bool zero_copy = !t->use_nccl && !knob("GACE_NO_ZERO_COPY");
    // fused merge: the finalize writes into this rank's symmetric window, the merge kernel
    // reads every rank's window into d_out
    size_t win_bytes = 0;
    char *win = t->merge ? static_cast<char *>(merge_buffer(t->merge, &win_bytes)) : nullptr;
    const bool fused = win && out_bytes <= win_bytes;
    char *out_base = fused ? win : zero_copy ? t->h_out.as<char>() : t->d_out.as<char>();
    F.out = reinterpret_cast<unsigned long long *>(out_base);
    F.out_regs = reinterpret_cast<uint8_t *>(out_base + align16(8 * out_words));
    F.g_bm = P.g_bm;
    F.zero = dbuf ? t->d_accb[ob].as<uint4>() : nullptr;          // the next call's accumulators
    F.zero_vec = dbuf ? t->d_accb[ob].cap / 16 : 0;
    F.nbm = 0;
    for (auto &S : pl.slots) {
        if (!S.bm) continue;
        FinParams::BmJob &J = F.bm[F.nbm++];
        J.goff = S.bm_goff;
        J.words = S.bm_words;
        J.out = S.hll_out;
        J.is64 = 0;
        J.base = S.bm_base;
    }
    CUDA_TRY(launch_finalize(F, s));
    nl += (F.njobs + F.hll_blocks ? 2 : 1) + (F.nbm ? 1 : 0);
    CUDA_TRY(rec(t->ev[3], s));

    if (fused) {
        CUDA_TRY(merge_launch(t->merge, (uint32_t)out_words, (uint32_t)align16(8 * out_words), pl.hll_bytes,
                              t->d_out.p, s));
        ++nl;
        merge_kind = 2;
    } else if (t->use_nccl) {
        merge_kind = 1;
        Nccl *n = nccl();
        if (!n) return fail(GACE_ENCCL, "libnccl.so.2 not loadable");
        n->GroupStart();
        int r1 = n->AllReduce(F.out, F.out, out_words, kNcclUint64, kNcclSum, t->comm, s);
        int r2 = pl.hll_bytes ? n->AllReduce(F.out_regs, F.out_regs, pl.hll_bytes, kNcclUint8, kNcclMax, t->comm, s) : 0;
        int r3 = n->GroupEnd();
        if (r1 || r2 || r3) return fail(GACE_ENCCL, "ncclAllReduce failed");
    }
    CUDA_TRY(rec(t->ev[4], s));
    if (!zero_copy) CUDA_TRY(cudaMemcpyAsync(t->h_out.p, t->d_out.p, out_bytes, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(rec(t->ev[5], s));
    return GACE_OK;
    }();
    if (capt) {
        cudaGraph_t g = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(s, &g);
        if (est) {
            if (g) cudaGraphDestroy(g);
            return est;
        }
        if (ce != cudaSuccess || !g) return fail(GACE_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
        if (t->gexec) cudaGraphExecDestroy(t->gexec);
        t->gexec = nullptr;
        const cudaError_t ie = cudaGraphInstantiate(&t->gexec, g, 0);
        cudaGraphDestroy(g);
        if (ie != cudaSuccess) {
            t->gexec = nullptr;
            return fail(GACE_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(ie));
        }
        t->gkey = gk;
        t->g_scan_launches = launches;
        t->g_jit = jit_used;
        t->g_nl = nl;
        t->g_captures++;
        CUDA_TRY(cudaGraphLaunch(t->gexec, s));
    } else if (est) {
        return est;
    }
    g_launches += nl;
    }
    st = wait_stream(t, s);
    if (st) return st;

    const uint64_t *ho = t->h_out.as<uint64_t>();
    *n_sampled = ho[0];
    if (npreds) memcpy(counts, ho + 1, 8ull * npreds);
    if (npairs) memcpy(joint_counts, ho + 1 + npreds, 8ull * npairs);
    if (nh) memcpy(hll_regs, t->h_out.as<uint8_t>(align16(8 * out_words)), pl.hll_bytes);

    gace_timing &T = t->last;
    T = gace_timing{};
    t->timing_kind = 1;          // stage times from the events in gace_last_timing
    t->dirty = false;
    if (dbuf) {                  // this call's fin_output zeroed the other buffer
        t->acc_clean[ob] = true;
        t->acc_next = ob;
    }
    T.scan_launches = launches;
    T.jit = jit_used;
    T.merge = merge_kind;
    T.jit_compile_ms = jit_ms;
    T.bytes_scanned = t->nrows * bytes_per_row;
    return GACE_OK;
}

gace_status gace_probe_sets(gace_table *t, const gace_pred *preds, uint32_t npreds, const uint32_t *set_offsets,
                            const uint32_t *set_members, uint32_t nsets, double sample_rate, uint64_t seed,
                            uint64_t *n_sampled, uint64_t *set_counts) {
    gace_status st = check_table(t);
    if (st) return st;
    refresh_knobs();
    std::lock_guard<std::mutex> lock(t->mu);
    st = validate_batch(t, preds, npreds, nullptr, 0, sample_rate, 0, GACE_HLL_P);
    if (st) return st;
    if (!n_sampled) return fail(GACE_EINVAL, "n_sampled is NULL");
    if (nsets > GACE_MAX_SETS) return fail(GACE_EUNSUPPORTED, "nsets > 256");
    if (nsets && (!set_offsets || !set_counts)) return fail(GACE_EINVAL, "set_offsets / set_counts is NULL");
    if (nsets && set_offsets[0] != 0) return fail(GACE_EINVAL, "set_offsets[0] must be 0");
    for (uint32_t m = 0; m < nsets; ++m)
        if (set_offsets[m + 1] < set_offsets[m]) return fail(GACE_EINVAL, "set_offsets must be non-decreasing");
    const uint32_t nmem = nsets ? set_offsets[nsets] : 0;
    if (nmem > GACE_MAX_SET_MEMBERS) return fail(GACE_EUNSUPPORTED, "more than 65536 set members");
    if (nmem && !set_members) return fail(GACE_EINVAL, "set_members is NULL");
    for (uint32_t k = 0; k < nmem; ++k)
        if (set_members[k] >= npreds) return fail(GACE_EINVAL, "set member index out of range");
    if (t->host) return fail(GACE_EUNSUPPORTED, "gace_probe_sets needs a device table");

    CUDA_TRY(cudaSetDevice(t->device));
    if (t->dirty) {
        st = wait_stream(t, t->stream);
        if (st) return st;
    }
    t->dirty = true;
    t->timing_kind = 0;
    std::string key;
    key.append(reinterpret_cast<const char *>(&nsets), 4);
    if (npreds) key.append(reinterpret_cast<const char *>(preds), sizeof(gace_pred) * npreds);
    if (nsets) key.append(reinterpret_cast<const char *>(set_offsets), 4ull * (nsets + 1));
    if (nmem) key.append(reinterpret_cast<const char *>(set_members), 4ull * nmem);
    cudaStream_t s = t->stream;
    CUDA_TRY(cudaEventRecord(t->ev[0], s));
    if (!t->sets_plan || key != t->sets_key) {
        auto fresh = std::make_shared<SetsPlan>();
        st = agree_plan(t, make_sets_plan(t, preds, set_offsets, set_members, nsets, *fresh), key);
        if (st) return st;
        const size_t n = fresh->image.size();
        if (t->h_sets_img.ensure(n) != cudaSuccess || t->d_sets_img.ensure(n) != cudaSuccess)
            return fail(GACE_ENOMEM, "candidate-set plan buffers");
        memcpy(t->h_sets_img.p, fresh->image.data(), n);
        CUDA_TRY(cudaMemcpyAsync(t->d_sets_img.p, t->h_sets_img.p, n, cudaMemcpyHostToDevice, s));
        t->sets_plan = fresh;
        t->sets_key.swap(key);
    }
    const SetsPlan &pl = *static_cast<const SetsPlan *>(t->sets_plan.get());
    const size_t out_words = 1 + 32ull * pl.P.W;          // [n_sampled, counts of W*32 sets]
    if (t->d_sets_out.ensure(8 * out_words) != cudaSuccess || t->h_sets_out.ensure(8 * out_words) != cudaSuccess)
        return fail(GACE_ENOMEM, "candidate-set scratch");
    CUDA_TRY(cudaMemsetAsync(t->d_sets_out.p, 0, 8 * out_words, s));
    CUDA_TRY(cudaEventRecord(t->ev[1], s));
    SetsParams P = pl.P;
    P.image = t->d_sets_img.as<const uint4>();
    P.g_nsamp = t->d_sets_out.as<unsigned long long>();
    P.g_counts = t->d_sets_out.as<unsigned long long>(8);
    P.seed = seed;
    P.thr = threshold_of(sample_rate);
    const bool sample = sample_rate < 1.0;
    const uint64_t row_offset = t->has_dist ? t->dist.row_offset : 0;
    const int grid = t->sms;
    // rows per launch: per-warp u32 counters and per-CTA u32 sums stay below 2^32
    const uint64_t max_rows = 1ull << 33;
    uint64_t launches = 0;
    for (uint64_t r0 = 0; r0 < t->nrows; r0 += max_rows) {
        const uint64_t n = std::min(max_rows, t->nrows - r0);
        for (uint32_t sl = 0; sl < P.ncols; ++sl) {
            const size_t w = pl.P.col[sl].is64 ? 8 : 4;
            P.col[sl].ptr = static_cast<const char *>(t->cols[pl.cols[sl]]) + r0 * w;
        }
        P.nrows = n;
        P.row0 = row_offset + r0;
        CUDA_TRY(launch_sets(P, sample, pl.i64, grid, s));
        ++launches;
    }
    g_launches += launches;
    CUDA_TRY(cudaEventRecord(t->ev[2], s));
    CUDA_TRY(cudaEventRecord(t->ev[3], s));
    if (t->use_nccl) {
        Nccl *nc = nccl();
        if (!nc) return fail(GACE_ENCCL, "libnccl.so.2 not loadable");
        void *buf = t->d_sets_out.p;
        if (nc->AllReduce(buf, buf, out_words, kNcclUint64, kNcclSum, t->comm, s))
            return fail(GACE_ENCCL, "ncclAllReduce failed");
    }
    CUDA_TRY(cudaEventRecord(t->ev[4], s));
    CUDA_TRY(cudaMemcpyAsync(t->h_sets_out.p, t->d_sets_out.p, 8 * out_words, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaEventRecord(t->ev[5], s));
    st = wait_stream(t, s);
    if (st) return st;
    const uint64_t *ho = t->h_sets_out.as<uint64_t>();
    *n_sampled = ho[0];
    if (nsets) memcpy(set_counts, ho + 1, 8ull * nsets);

    gace_timing &T = t->last;
    T = gace_timing{};
    t->timing_kind = 2;
    t->dirty = false;
    T.scan_launches = launches;
    T.bytes_scanned = t->nrows * pl.bytes_per_row;
    return GACE_OK;
}

// ------------------------------------------------------------------ Est.CV (NEXT-4, PAPER.md Exp. B)

gace_status gace_estimate_cv(gace_table *t, const gace_pred *preds, uint32_t npreds, const gace_pair *pairs,
                             uint32_t npairs, double sample_rate, const uint64_t *seeds, uint32_t nseeds,
                             double *cv_sel, double *cv_joint, double *cv_pcs) {
    gace_status st = check_table(t);
    if (st) return st;
    if (nseeds < 2) return fail(GACE_EINVAL, "Est.CV needs >= 2 seeds");
    if (!seeds) return fail(GACE_EINVAL, "seeds is NULL");
    if (npreds && !cv_sel) return fail(GACE_EINVAL, "cv_sel is NULL");
    if (npairs && (!cv_joint || !cv_pcs)) return fail(GACE_EINVAL, "cv_joint / cv_pcs is NULL");
    st = validate_batch(t, preds, npreds, pairs, npairs, sample_rate, 0, GACE_HLL_P);
    if (st) return st;
    // per seed: S_p = count_p / n, S_q = joint_q / n, PCS_q (Eq. 3 order) -- one probe each
    const size_t P = npreds, Q = npairs;
    std::vector<double> sel(P * nseeds), js(Q * nseeds), pcs(Q * nseeds);
    std::vector<uint64_t> counts(std::max<size_t>(P, 1)), joints(std::max<size_t>(Q, 1));
    for (uint32_t r = 0; r < nseeds; ++r) {
        uint64_t n = 0;
        st = gace_probe(t, preds, npreds, pairs, npairs, sample_rate, seeds[r], 0, GACE_HLL_P, &n, counts.data(),
                        joints.data(), nullptr);
        if (st) return st;
        std::vector<double> s(P), pq(Q);
        st = gace_derive(n, counts.data(), npreds, pairs, joints.data(), npairs, nullptr, 0, GACE_HLL_P, nullptr,
                         s.data(), pq.data(), nullptr, nullptr);
        if (st) return st;
        for (size_t p = 0; p < P; ++p) sel[p * nseeds + r] = s[p];
        for (size_t q = 0; q < Q; ++q) {
            js[q * nseeds + r] = n ? (double)joints[q] / (double)n : NAN;
            pcs[q * nseeds + r] = pq[q];
        }
    }
    // CV = sample standard deviation (R - 1) / mean; mean 0 or any NaN -> NaN
    auto cv = [&](const double *x) {
        double mean = 0.0;
        for (uint32_t r = 0; r < nseeds; ++r) mean += x[r];
        mean /= (double)nseeds;
        double ss = 0.0;
        for (uint32_t r = 0; r < nseeds; ++r) ss += (x[r] - mean) * (x[r] - mean);
        const double sd = std::sqrt(ss / (double)(nseeds - 1));
        return mean == 0.0 ? NAN : sd / mean;
    };
    for (size_t p = 0; p < P; ++p) cv_sel[p] = cv(&sel[p * nseeds]);
    for (size_t q = 0; q < Q; ++q) {
        cv_joint[q] = cv(&js[q * nseeds]);
        cv_pcs[q] = cv(&pcs[q * nseeds]);
    }
    return GACE_OK;
}

// ------------------------------------------------------------------ probe cache (NEXT-4, §V item 3)

struct gace_cache {
    uint32_t magic = 0x47434348u;   // "GCCH"
    uint32_t capacity = 4096, buckets = 64;
    struct Entry {
        gace_cache_entry v;
        uint64_t seq;
        uint64_t table;
    };
    std::map<std::string, Entry> map;
    std::deque<std::pair<uint64_t, std::string>> order;   // insertion order (FIFO eviction)
    uint64_t seq = 0, hits = 0, misses = 0, evictions = 0;
    std::mutex mu;
};

namespace {

gace_status check_cache(const gace_cache *c) {
    if (!c || c->magic != 0x47434348u) return fail(GACE_EHANDLE, "invalid or destroyed cache handle");
    return GACE_OK;
}

// Bind bucket of value x on a column with domain [lo, hi]: buckets equal-width intervals
// (SPEC.md S:397 reading: 64 per column), -1 below the domain, `buckets` above; exact value
// when buckets == 0 or no domain is given.
int64_t bind_bucket(int64_t x, uint32_t buckets, const int64_t *dom) {
    if (!buckets || !dom) return x;
    const int64_t lo = dom[0], hi = dom[1];
    if (x < lo) return -1;
    if (x > hi) return (int64_t)buckets;
    const long double w = ((long double)hi - (long double)lo + 1.0L) / (long double)buckets;
    int64_t b = (int64_t)(((long double)x - (long double)lo) / w);
    return std::min<int64_t>(std::max<int64_t>(b, 0), (int64_t)buckets - 1);
}

// CacheKey: table id + the conjunction's predicates as (col, op, flags,
// bind bucket(a), bind bucket(b) for BETWEEN), sorted -- A and B == B and A.
std::string cache_key(const gace_cache *c, uint64_t table, const gace_pred *conj, uint32_t k, const int64_t *dom) {
    std::vector<std::array<int64_t, 5>> items(k);
    for (uint32_t i = 0; i < k; ++i) {
        const gace_pred &p = conj[i];
        const int64_t *d = dom ? dom + 2 * i : nullptr;
        items[i] = {(int64_t)p.col, (int64_t)p.op, (int64_t)p.flags, bind_bucket(p.a, c->buckets, d),
                    p.op == GACE_BETWEEN ? bind_bucket(p.b, c->buckets, d) : 0};
    }
    std::sort(items.begin(), items.end());
    items.erase(std::unique(items.begin(), items.end()), items.end());   // A and A == A
    std::string key(reinterpret_cast<const char *>(&table), 8);
    for (auto &it : items) key.append(reinterpret_cast<const char *>(it.data()), sizeof(int64_t) * 5);
    return key;
}

}  // namespace

gace_status gace_cache_create(uint32_t capacity, uint32_t range_buckets, gace_cache **out) {
    if (!out) return fail(GACE_EINVAL, "out is NULL");
    gace_cache *c = new gace_cache();
    c->capacity = capacity ? capacity : 4096;
    c->buckets = range_buckets;
    *out = c;
    return GACE_OK;
}

gace_status gace_cache_destroy(gace_cache *c) {
    gace_status st = check_cache(c);
    if (st) return st;
    c->magic = 0;
    delete c;
    return GACE_OK;
}

gace_status gace_cache_put(gace_cache *c, uint64_t table_id, const gace_pred *conj, uint32_t k,
                           const int64_t *domains, const gace_cache_entry *entry) {
    gace_status st = check_cache(c);
    if (st) return st;
    if ((k && !conj) || !entry) return fail(GACE_EINVAL, "NULL argument");
    if (!(entry->s_probe >= 0.0 && entry->s_probe <= 1.0)) return fail(GACE_EINVAL, "s_probe must be in [0, 1]");
    std::lock_guard<std::mutex> lock(c->mu);
    const std::string key = cache_key(c, table_id, conj, k, domains);
    auto it = c->map.find(key);
    const uint64_t seq = ++c->seq;
    if (it != c->map.end()) {                       // replace: re-inserted at the back
        it->second.v = *entry;
        it->second.v.hits = 0;
        it->second.seq = seq;
    } else {
        c->map[key] = {*entry, seq, table_id};
        c->map[key].v.hits = 0;
    }
    c->order.emplace_back(seq, key);
    while (c->map.size() > c->capacity && !c->order.empty()) {      // least recently inserted
        auto [s, kk] = c->order.front();
        c->order.pop_front();
        auto f = c->map.find(kk);
        if (f != c->map.end() && f->second.seq == s) {
            c->map.erase(f);
            ++c->evictions;
        }
    }
    if (c->order.size() > 2ull * c->capacity + 64) {       // re-puts leave stale entries: compact
        std::deque<std::pair<uint64_t, std::string>> live;
        for (auto &e : c->order) {
            auto f = c->map.find(e.second);
            if (f != c->map.end() && f->second.seq == e.first) live.push_back(std::move(e));
        }
        c->order.swap(live);
    }
    return GACE_OK;
}

gace_status gace_cache_lookup(gace_cache *c, uint64_t table_id, const gace_pred *conj, uint32_t k,
                              const int64_t *domains, gace_cache_entry *entry, uint32_t *hit) {
    gace_status st = check_cache(c);
    if (st) return st;
    if ((k && !conj) || !hit) return fail(GACE_EINVAL, "NULL argument");
    std::lock_guard<std::mutex> lock(c->mu);
    auto it = c->map.find(cache_key(c, table_id, conj, k, domains));
    if (it == c->map.end()) {
        ++c->misses;
        *hit = 0;
        return GACE_OK;
    }
    ++c->hits;
    ++it->second.v.hits;
    if (entry) *entry = it->second.v;
    *hit = 1;
    return GACE_OK;
}

gace_status gace_cache_invalidate(gace_cache *c, uint64_t table_id) {
    gace_status st = check_cache(c);
    if (st) return st;
    std::lock_guard<std::mutex> lock(c->mu);
    for (auto it = c->map.begin(); it != c->map.end();)
        it = it->second.table == table_id ? c->map.erase(it) : std::next(it);
    return GACE_OK;
}

gace_status gace_cache_stats(gace_cache *c, uint64_t *hits, uint64_t *misses, uint64_t *evictions, uint64_t *size) {
    gace_status st = check_cache(c);
    if (st) return st;
    std::lock_guard<std::mutex> lock(c->mu);
    if (hits) *hits = c->hits;
    if (misses) *misses = c->misses;
    if (evictions) *evictions = c->evictions;
    if (size) *size = c->map.size();
    return GACE_OK;
}

gace_status gace_sample_mask(gace_table *t, double sample_rate, uint64_t seed, uint64_t *bits) {
    gace_status st = check_table(t);
    if (st) return st;
    std::lock_guard<std::mutex> lock(t->mu);
    if (!(sample_rate >= 0.0 && sample_rate <= 1.0)) return fail(GACE_EINVAL, "sample_rate must be in [0, 1]");
    if (!bits && t->nrows) return fail(GACE_EINVAL, "bits is NULL");
    const uint64_t words = (t->nrows + 63) / 64;
    if (!words) return GACE_OK;
    CUDA_TRY(cudaSetDevice(t->device));
    if (t->d_mask.ensure(8 * words) != cudaSuccess) return fail(GACE_ENOMEM, "mask buffer");
    const uint64_t row0 = t->has_dist ? t->dist.row_offset : 0;
    CUDA_TRY(launch_sample_mask(t->nrows, row0, seed, threshold_of(sample_rate), sample_rate >= 1.0,
                                t->d_mask.as<unsigned long long>(), t->stream));
    ++g_launches;
    CUDA_TRY(cudaMemcpyAsync(bits, t->d_mask.p, 8 * words, cudaMemcpyDeviceToHost, t->stream));
    CUDA_TRY(cudaStreamSynchronize(t->stream));
    return GACE_OK;
}

gace_status gace_jit_sync(double timeout_ms, uint64_t *compiled, uint64_t *failed, uint64_t *pending) {
    if (!(timeout_ms >= 0)) return fail(GACE_EINVAL, "timeout_ms must be >= 0");
    const bool ok = jit_bg_wait(timeout_ms);
    jit_bg_stats(compiled, failed, pending);
    return ok ? GACE_OK : fail(GACE_EUNSUPPORTED, "background kernel compiles still running at the timeout");
}

gace_status gace_jit_shutdown(void) {
    jit_bg_shutdown();
    return GACE_OK;
}

gace_status gace_last_timing(const gace_table *t, gace_timing *out) {
    gace_status st = check_table(t);
    if (st) return st;
    if (!out) return fail(GACE_EINVAL, "out is NULL");
    *out = t->last;
    if (t->timing_kind) {        // the call synchronised its stream: every event has completed
        float ms;
        cudaSetDevice(t->device);
        cudaEventElapsedTime(&ms, t->ev[0], t->ev[1]); out->plan_upload_ms = ms;
        cudaEventElapsedTime(&ms, t->ev[1], t->ev[2]); out->scan_ms = ms;
        if (t->timing_kind == 1) { cudaEventElapsedTime(&ms, t->ev[2], t->ev[3]); out->finalize_ms = ms; }
        cudaEventElapsedTime(&ms, t->ev[3], t->ev[4]); out->merge_ms = ms;
        cudaEventElapsedTime(&ms, t->ev[4], t->ev[5]); out->d2h_ms = ms;
        cudaEventElapsedTime(&ms, t->ev[0], t->ev[5]); out->total_ms = ms;
        if (t->timing_kind == 1 && t->host && t->nrows) { cudaEventElapsedTime(&ms, t->ev_c0, t->ev_c1); out->h2d_ms = ms; }
    }
    return GACE_OK;
}

// ---------------------------------------------------------------- derive / gate (host doubles)

static double hll_estimate(const uint8_t *R, uint32_t m) {
    double z = 0.0;
    uint32_t v = 0;
    for (uint32_t j = 0; j < m; ++j) {
        z += std::ldexp(1.0, -(int)R[j]);
        v += R[j] == 0;
    }
    const double md = (double)m;
    const double alpha = 0.7213 / (1.0 + 1.079 / md);
    const double e = alpha * md * md / z;
    if (e <= 2.5 * md && v > 0) return md * std::log(md / (double)v);
    return e;
}

gace_status gace_derive(uint64_t n, const uint64_t *counts, uint32_t npreds, const gace_pair *pairs,
                        const uint64_t *joints, uint32_t npairs, const uint8_t *regs, uint32_t ncols_hll,
                        uint32_t hll_p, const double *ndv_hist, double *sel, double *pcs, double *ndv_est,
                        double *drift) {
    if ((npreds && !counts && (sel || pcs)) || (npairs && (!pairs || !joints) && pcs))
        return fail(GACE_EINVAL, "NULL input array");
    if (ncols_hll && !regs && (ndv_est || drift)) return fail(GACE_EINVAL, "regs is NULL");
    if (drift && ncols_hll && !ndv_hist) return fail(GACE_EINVAL, "ndv_hist is NULL");
    if (ncols_hll && (ndv_est || drift) && hll_p != GACE_HLL_P) return fail(GACE_EUNSUPPORTED, "hll_p must be 12");
    if (pcs)
        for (uint32_t q = 0; q < npairs; ++q)
            if (pairs[q].i >= npreds || pairs[q].j >= npreds) return fail(GACE_EINVAL, "pair index out of range");
    if (drift)
        for (uint32_t c = 0; c < ncols_hll; ++c)
            if (!(ndv_hist[c] > 0)) return fail(GACE_EINVAL, "ndv_hist must be > 0");
    const double nan = std::nan("");
    const double fn = (double)n;
    if (sel)
        for (uint32_t p = 0; p < npreds; ++p) sel[p] = n ? (double)counts[p] / fn : nan;
    if (pcs)
        for (uint32_t q = 0; q < npairs; ++q) {
            const uint64_t a = counts[pairs[q].i], b = counts[pairs[q].j];
            if (!n || !a || !b) { pcs[q] = nan; continue; }
            const double pa = (double)a / fn, pb = (double)b / fn, pj = (double)joints[q] / fn;
            pcs[q] = pj / (pa * pb);
        }
    for (uint32_t c = 0; c < ncols_hll && (ndv_est || drift); ++c) {
        const double e = hll_estimate(regs + (size_t)c * kHllM, kHllM);
        if (ndv_est) ndv_est[c] = e;
        if (drift) drift[c] = std::fabs(ndv_hist[c] - e) / ndv_hist[c];
    }
    return GACE_OK;
}

// ------------------------------------------------------------------ break-even cost accounting (NEXT-3)

static double cost_of(const gace_cost_model &c, double n, double k, double m) {
    return c.c0_ms + c.ct_ms_per_row * n + c.ce_ms_per_eval * k * m * n / c.p;
}

gace_status gace_cost_fit(const double *n, const double *k, const double *m, const double *ms, uint32_t npts,
                          double p, gace_cost_model *out) {
    if (!n || !k || !m || !ms || !out) return fail(GACE_EINVAL, "NULL argument");
    if (npts < 3) return fail(GACE_EINVAL, "cost fit needs >= 3 points");
    if (!(p >= 1.0) || !std::isfinite(p)) return fail(GACE_EINVAL, "parallelism factor p must be >= 1");
    for (uint32_t i = 0; i < npts; ++i)
        if (!std::isfinite(n[i]) || !std::isfinite(k[i]) || !std::isfinite(m[i]) || !std::isfinite(ms[i]))
            return fail(GACE_EINVAL, "non-finite calibration point");
    // design columns: 1, N, K*M*N/p, each scaled by its max |.|
    std::vector<double> X[3];
    double scale[3];
    for (int j = 0; j < 3; ++j) {
        X[j].resize(npts);
        scale[j] = 0.0;
        for (uint32_t i = 0; i < npts; ++i) {
            X[j][i] = j == 0 ? 1.0 : j == 1 ? n[i] : k[i] * m[i] * n[i] / p;
            scale[j] = std::max(scale[j], std::fabs(X[j][i]));
        }
        if (scale[j] > 0)
            for (uint32_t i = 0; i < npts; ++i) X[j][i] /= scale[j];
    }
    double best_r = 0.0, best[3] = {0, 0, 0};
    for (uint32_t i = 0; i < npts; ++i) best_r += ms[i] * ms[i];
    const double tss = best_r;
    // every non-negativity active set in mask order 1..7, least squares by modified
    // Gram-Schmidt with one re-orthogonalisation pass; a later set replaces the best only
    // when its residual is smaller by more than 1e-9 of sum(ms^2) (near-ties keep the
    // earlier set, e.g. collinear N and K*M*N columns)
    for (int mask = 1; mask < 8; ++mask) {
        int cols[3], nc = 0;
        for (int j = 0; j < 3; ++j)
            if (mask >> j & 1) cols[nc++] = j;
        std::vector<double> Q[3];
        double R[3][3] = {{0}};
        bool ok = true;
        for (int a = 0; a < nc; ++a) {
            Q[a] = X[cols[a]];
            for (int pass = 0; pass < 2; ++pass)
                for (int b = 0; b < a; ++b) {
                    double d = 0;
                    for (uint32_t i = 0; i < npts; ++i) d += Q[b][i] * Q[a][i];
                    R[b][a] += d;
                    for (uint32_t i = 0; i < npts; ++i) Q[a][i] -= d * Q[b][i];
                }
            double nr = 0;
            for (uint32_t i = 0; i < npts; ++i) nr += Q[a][i] * Q[a][i];
            nr = std::sqrt(nr);
            if (!(nr > 1e-12)) { ok = false; break; }     // rank-deficient subset: skipped
            R[a][a] = nr;
            for (uint32_t i = 0; i < npts; ++i) Q[a][i] /= nr;
        }
        if (!ok) continue;
        double qb[3], sol[3];
        for (int a = 0; a < nc; ++a) {
            qb[a] = 0;
            for (uint32_t i = 0; i < npts; ++i) qb[a] += Q[a][i] * ms[i];
        }
        for (int a = nc - 1; a >= 0; --a) {
            double s = qb[a];
            for (int b = a + 1; b < nc; ++b) s -= R[a][b] * sol[b];
            sol[a] = s / R[a][a];
        }
        bool feasible = true;
        double coef[3] = {0, 0, 0};
        for (int a = 0; a < nc; ++a) {
            if (sol[a] < 0) feasible = false;
            coef[cols[a]] = scale[cols[a]] > 0 ? sol[a] / scale[cols[a]] : 0.0;
        }
        if (!feasible) continue;
        double r = 0;
        for (uint32_t i = 0; i < npts; ++i) {
            const double pred = coef[0] + coef[1] * n[i] + coef[2] * k[i] * m[i] * n[i] / p;
            r += (pred - ms[i]) * (pred - ms[i]);
        }
        if (r < best_r - 1e-9 * tss) {
            best_r = r;
            best[0] = coef[0]; best[1] = coef[1]; best[2] = coef[2];
        }
    }
    out->c0_ms = best[0];
    out->ct_ms_per_row = best[1];
    out->ce_ms_per_eval = best[2];
    out->p = p;
    if (!(out->benefit_weight >= 0.0)) out->benefit_weight = 0.5;    // SPEC.md S:249 default
    return GACE_OK;
}

gace_status gace_gate_decide(uint32_t fired_mask, const gace_cost_model *cm, double n_sample, double k, double m,
                             double plan_cost_spread_ms, double *est_cost_ms, double *est_benefit_ms,
                             uint32_t *probe, uint32_t *reason) {
    if (!cm || !probe || !reason) return fail(GACE_EINVAL, "NULL argument");
    if (!(cm->p >= 1.0) || !(cm->c0_ms >= 0) || !(cm->ct_ms_per_row >= 0) || !(cm->ce_ms_per_eval >= 0) ||
        !(cm->benefit_weight >= 0))
        return fail(GACE_EINVAL, "cost model coefficients must be >= 0 and p >= 1");
    const double cost = cost_of(*cm, n_sample, k, m);
    const double benefit = cm->benefit_weight * plan_cost_spread_ms;
    uint32_t pr = 0, rs = GACE_NO_RISK;
    if (fired_mask) {
        pr = benefit > cost ? 1u : 0u;             // strict: a tie is not worth it
        rs = pr ? GACE_PROBE : GACE_RISK_BUT_NOT_WORTH;
    }
    if (est_cost_ms) *est_cost_ms = cost;
    if (est_benefit_ms) *est_benefit_ms = benefit;
    *probe = pr;
    *reason = rs;
    return GACE_OK;
}

gace_status gace_gate(const double *drift, uint32_t nd, const double *s_est, const double *s_probe, uint32_t ns,
                      const double *pcs, uint32_t np, const gace_thresholds *th, uint32_t *fired_mask,
                      uint8_t *per_signal_fired) {
    if (!fired_mask) return fail(GACE_EINVAL, "fired_mask is NULL");
    if ((nd && !drift) || (ns && (!s_est || !s_probe)) || (np && !pcs)) return fail(GACE_EINVAL, "NULL signal array");
    const gace_thresholds def = {0.25, 0.01, 1.6, 0.7};
    const gace_thresholds &T = th ? *th : def;
    uint32_t mask = 0, k = 0;
    for (uint32_t i = 0; i < nd; ++i, ++k) {
        const bool f = drift[i] >= T.d_threshold;                            // NaN: false
        if (f) mask |= GACE_SIG_DRIFT;
        if (per_signal_fired) per_signal_fired[k] = f;
    }
    for (uint32_t i = 0; i < ns; ++i, ++k) {
        const bool f = std::fabs(s_est[i] - s_probe[i]) > T.sel_err_threshold;
        if (f) mask |= GACE_SIG_SEL_ERROR;
        if (per_signal_fired) per_signal_fired[k] = f;
    }
    for (uint32_t i = 0; i < np; ++i, ++k) {
        const bool f = pcs[i] > T.pcs_high || pcs[i] < T.pcs_low;
        if (f) mask |= GACE_SIG_CORRELATION;
        if (per_signal_fired) per_signal_fired[k] = f;
    }
    *fired_mask = mask;
    return GACE_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- planner test hook

namespace {
struct CheckedTables {
    const std::vector<uint8_t> *img;
    mutable bool oob = false;
    uint4 u4(uint32_t i) const {
        if ((size_t)i * 16 + 16 > img->size()) { oob = true; return make_uint4(0, kNoThr, kNoThr, kNoThr); }
        return reinterpret_cast<const uint4 *>(img->data())[i];
    }
    uint32_t u32(uint32_t i) const {
        if ((size_t)i * 4 + 4 > img->size()) { oob = true; return 0; }
        return reinterpret_cast<const uint32_t *>(img->data())[i];
    }
    uint32_t u16(uint32_t i) const {
        if ((size_t)i * 2 + 2 > img->size()) { oob = true; return 0; }
        return reinterpret_cast<const uint16_t *>(img->data())[i];
    }
};
}  // namespace

extern "C" gace_status gace_debug_buckets(uint32_t ncols, const gace_dtype *dtypes, const int64_t *dlo,
                                          const int64_t *dhi, int host, const gace_pred *preds, uint32_t npreds,
                                          const gace_pair *pairs, uint32_t npairs, uint64_t hll_mask, uint32_t col,
                                          const int64_t *values, uint64_t n, uint32_t *out, uint32_t *mode,
                                          int64_t *bps, uint32_t cap, uint32_t *nbp) {
    if (!dtypes || !dlo || !dhi || ncols == 0 || ncols > GACE_MAX_COLS || col >= ncols || (n && (!values || !out)))
        return fail(GACE_EINVAL, "bad arguments");
    refresh_knobs();
    gace_table t;
    t.ncols = ncols;
    t.host = host != 0;
    t.nrows = getenv("GACE_DEBUG_ROWS") ? strtoull(getenv("GACE_DEBUG_ROWS"), nullptr, 10) : 0;   // row-count heuristics
    for (uint32_t c = 0; c < ncols; ++c) {
        t.dtypes.push_back((int)dtypes[c]);
        t.dlo.push_back(dlo[c]);
        t.dhi.push_back(dhi[c]);
    }
    gace_status st = validate_batch(&t, preds, npreds, pairs, npairs, 1.0, hll_mask, GACE_HLL_P);
    if (st) return st;
    Plan pl;
    st = make_plan(&t, preds, npreds, pairs, npairs, hll_mask, pl, false, true);    // the plan a full scan uses
    if (st) return st;
    const int s = pl.col2slot[col];
    if (s < 0 || !pl.slots[s].has_preds) return fail(GACE_EINVAL, "column has no predicates");
    const SlotPlan &S = pl.slots[s];
    const SlotParams &Q = pl.P.slot[s];
    if (mode) *mode = Q.mode;
    if (nbp) *nbp = (uint32_t)S.T.size();
    for (uint32_t i = 0; bps && i < S.T.size() && i < cap; ++i) bps[i] = S.T[i];
    // static layout checks: every grid cell a (bucket, sub-bucket) pair can address lies
    // inside the accumulators, and every map entry is a valid sub-bucket
    for (const Group &G : pl.groups) {
        if (G.direct) continue;
        const uint32_t *m32 = reinterpret_cast<const uint32_t *>(pl.image.data());
        for (uint32_t r = 0; r < pl.slots[G.b].nb; ++r)
            if (m32[G.map_w + r] >= G.nbs) return fail(GACE_EUNSUPPORTED, "internal: sub-bucket map out of range");
        if (G.grid_w + G.na * G.nbs > pl.acc_idx + pl.acc_words) return fail(GACE_EUNSUPPORTED, "internal: grid out of range");
    }
    CheckedTables M{&pl.image};
    for (uint64_t k = 0; k < n; ++k) {
        uint32_t b;
        if (Q.mode == MODE_SEARCH) {
            b = count_le(S.T, values[k]);
        } else if (Q.dtype == GACE_I32) {
            int32_t x = (int32_t)values[k];
            if (pl.clamp) x = std::min(std::max(x, (int32_t)Q.clamp_lo), (int32_t)Q.clamp_hi);
            if (Q.fmt == FMTEX && Q.fdirect)       // the kernel's decode: a bin address -> its bucket
                b = (M.u32(Q.lut_w + ((uint32_t)x - (uint32_t)Q.base)) - Q.hist_addr) / 4;
            else if (Q.fmt == FMTEX)               // the kernel's decode: the cell word's bucket field
                b = M.u32(Q.lut_w + ((uint32_t)x - (uint32_t)Q.base)) & Q.bmask;
            else
                b = lut_lookup(M, Q.fmt, Q.lut_w, Q.s1, (uint32_t)x - (uint32_t)Q.base, Q.sb);
        } else {
            int64_t x = values[k];
            if (pl.clamp) x = std::min(std::max(x, Q.clamp_lo), Q.clamp_hi);
            b = lut_lookup(M, Q.fmt, Q.lut_w, Q.s1, (uint32_t)((uint64_t)x - (uint64_t)Q.base), Q.sb);
        }
        if (M.oob) return fail(GACE_EUNSUPPORTED, "internal: table read out of range");
        if (b >= S.nb) return fail(GACE_EUNSUPPORTED, "internal: bucket out of range");
        out[k] = b;
        // the packed sub-bucket of a direct entry must agree with the group's map
        if (Q.mode == MODE_LUT && S.prim_b >= 0) {
            const Group &G = pl.groups[S.prim_b];
            const uint32_t u = Q.dtype == GACE_I32
                ? (uint32_t)std::min(std::max((int32_t)values[k], pl.clamp ? (int32_t)Q.clamp_lo : INT32_MIN),
                                     pl.clamp ? (int32_t)Q.clamp_hi : INT32_MAX) - (uint32_t)Q.base
                : (uint32_t)((uint64_t)std::min(std::max(values[k], pl.clamp ? Q.clamp_lo : INT64_MIN),
                                                pl.clamp ? Q.clamp_hi : INT64_MAX) - (uint64_t)Q.base);
            uint32_t sub;
            if (Q.fmt == FMT1T) {
                const uint32_t v = t1_bs(M, Q.lut_w, Q.s1, Q.sb, u);
                sub = (v & 0x80000000u) ? kNone : v >> Q.sb;
            } else {
                sub = entry_sub(lut_entry(M, Q.fmt, Q.lut_w, Q.s1, u), u);
            }
            const uint32_t want = reinterpret_cast<const uint32_t *>(pl.image.data())[G.map_w + b];
            if (sub != kNone && sub != want) return fail(GACE_EUNSUPPORTED, "internal: packed sub-bucket differs from the map");
        }
    }
    return GACE_OK;
}

// Test hook: plan a batch (as gace_debug_buckets) and compile its specialised probe kernel
// with NVRTC without launching it.  *cubin_bytes = size of the compiled kernel image.
// Test hook: the generated JitShape source of a batch (structure-keyed, or layout-keyed with
// layout != 0), without compiling it.  out[cap] receives it NUL-terminated; *len its length.
extern "C" gace_status gace_debug_jit_source(uint32_t ncols, const gace_dtype *dtypes, const int64_t *dlo,
                                             const int64_t *dhi, int host, const gace_pred *preds,
                                             uint32_t npreds, const gace_pair *pairs, uint32_t npairs,
                                             uint64_t hll_mask, double sample_rate, int layout, char *out,
                                             uint64_t cap, uint64_t *len) {
    if (!dtypes || !dlo || !dhi || ncols == 0 || ncols > GACE_MAX_COLS) return fail(GACE_EINVAL, "bad arguments");
    refresh_knobs();
    gace_table t;
    t.ncols = ncols;
    t.host = host != 0;
    t.nrows = getenv("GACE_DEBUG_ROWS") ? strtoull(getenv("GACE_DEBUG_ROWS"), nullptr, 10) : 0;   // row-count heuristics
    for (uint32_t c = 0; c < ncols; ++c) {
        t.dtypes.push_back((int)dtypes[c]);
        t.dlo.push_back(dlo[c]);
        t.dhi.push_back(dhi[c]);
    }
    gace_status st = validate_batch(&t, preds, npreds, pairs, npairs, sample_rate, hll_mask, GACE_HLL_P);
    if (st) return st;
    Plan pl;
    st = make_plan(&t, preds, npreds, pairs, npairs, hll_mask, pl, sample_rate < 0.125, sample_rate >= 1.0);   // as gace_probe
    if (st) return st;
    bool i64 = false;
    for (auto &S : pl.slots) i64 |= S.dtype == GACE_I64;
    const std::string src = jit_shape_source(pl, sample_rate < 1.0, i64, std::vector<uint8_t>(pl.slots.size(), 0),
                                             layout != 0);
    if (len) *len = src.size();
    if (out && cap) {
        const size_t n = std::min<size_t>(cap - 1, src.size());
        memcpy(out, src.data(), n);
        out[n] = 0;
    }
    return GACE_OK;
}

extern "C" gace_status gace_debug_jit_compile(uint32_t ncols, const gace_dtype *dtypes, const int64_t *dlo,
                                              const int64_t *dhi, int host, const gace_pred *preds,
                                              uint32_t npreds, const gace_pair *pairs, uint32_t npairs,
                                              uint64_t hll_mask, double sample_rate, uint64_t *cubin_bytes) {
    if (!dtypes || !dlo || !dhi || ncols == 0 || ncols > GACE_MAX_COLS) return fail(GACE_EINVAL, "bad arguments");
    refresh_knobs();
    gace_table t;
    t.ncols = ncols;
    t.host = host != 0;
    t.nrows = getenv("GACE_DEBUG_ROWS") ? strtoull(getenv("GACE_DEBUG_ROWS"), nullptr, 10) : 0;   // row-count heuristics
    for (uint32_t c = 0; c < ncols; ++c) {
        t.dtypes.push_back((int)dtypes[c]);
        t.dlo.push_back(dlo[c]);
        t.dhi.push_back(dhi[c]);
    }
    gace_status st = validate_batch(&t, preds, npreds, pairs, npairs, sample_rate, hll_mask, GACE_HLL_P);
    if (st) return st;
    // GACE_DEBUG_CLUSTERED = bit mask of columns taken as clustered (planner and kernel path)
    const unsigned long clm = getenv("GACE_DEBUG_CLUSTERED") ? strtoul(getenv("GACE_DEBUG_CLUSTERED"), nullptr, 0) : 0ul;
    t.clustered.assign(ncols, 0);
    for (uint32_t c = 0; c < ncols; ++c) t.clustered[c] = (clm >> c) & 1ul;
    Plan pl;
    st = make_plan(&t, preds, npreds, pairs, npairs, hll_mask, pl, sample_rate < 0.125, sample_rate >= 1.0);   // as gace_probe
    if (st) return st;
    if (pl.P.nslots == 0) return fail(GACE_EINVAL, "no probed columns");
    bool i64 = false;
    for (auto &S : pl.slots) i64 |= S.dtype == GACE_I64;
    std::string err;
    size_t n = 0;
    std::vector<uint8_t> cl(pl.slots.size(), 0);
    for (size_t i = 0; i < cl.size(); ++i) cl[i] = t.clustered[pl.slots[i].col];
    if (getenv("GACE_PLAN_PROFILE")) {       // design inspection: cost of generating the source
        const auto t0 = std::chrono::steady_clock::now();
        for (int r = 0; r < 20; ++r) (void)jit_shape_source(pl, sample_rate < 1.0, i64, cl, false);
        fprintf(stderr, "jit_shape_source (structure-keyed) %.1f us\n",
                std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / 20);
    }
    if (!jit_compile_check(jit_shape_source(pl, sample_rate < 1.0, i64, cl, jit_layout()), &n, &err))
        return fail(GACE_EUNSUPPORTED, err);
    if (cubin_bytes) *cubin_bytes = n;
    return GACE_OK;
}
