// gace_merge.cu -- the cross-GPU merge fused into one kernel over NVLink peer memory
// (SURVEY.md §8(f) NEXT-2b; §8(a) a9; §IV-B P:100 "Reduction").
//
// Every rank's finalize writes its packed result [n_sampled, counts, joints | HLL registers]
// into a symmetric NCCL window (ncclMemAlloc + ncclCommWindowRegister, NCCL 2.28 device
// API).  One CTA per rank then
//   1. meets the other ranks at an LSA barrier (every result is in its window),
//   2. reads the same words from every peer's window through NVLink load/store addresses
//      (ncclGetLsaPointer) and writes the sum of the u64 counters and the byte-wise max of the
//      registers into this rank's output buffer,
//   3. meets them at the barrier again, so no rank's next probe overwrites a window a peer is
//      still reading.
// That replaces the grouped ncclAllReduce(sum u64) + ncclAllReduce(max u8) -- two collective
// launches with their protocol set-up -- by one small kernel whose reads are the exchange.
// Used when every rank is in one load/store-accessible (LSA, NVLink) team; otherwise, or when
// the NCCL device API is not available, gace_probe keeps the grouped all-reduce.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>

#include <string>

#include "gace_merge.h"

#if GACE_NCCL_DEVICE
#include <nccl.h>
#include <nccl_device.h>

namespace gace {

struct MergeState {
    void *buf = nullptr;               // ncclMemAlloc'd symmetric buffer (this rank's window)
    size_t bytes = 0;
    ncclWindow_t win = nullptr;
    ncclDevComm dc{};
    void *comm = nullptr;
    bool dc_ok = false;
};

namespace {

struct Api {
    ncclResult_t (*MemAlloc)(void **, size_t) = nullptr;
    ncclResult_t (*MemFree)(void *) = nullptr;
    ncclResult_t (*WinReg)(ncclComm_t, void *, size_t, ncclWindow_t *, int) = nullptr;
    ncclResult_t (*WinDereg)(ncclComm_t, ncclWindow_t) = nullptr;
    ncclResult_t (*DevCommCreate)(ncclComm_t, ncclDevCommRequirements_t const *, ncclDevComm_t *) = nullptr;
    ncclResult_t (*DevCommDestroy)(ncclComm_t, ncclDevComm_t const *) = nullptr;
    bool ok = false;
};

Api &api() {
    static Api a;
    static bool done = false;
    if (done) return a;
    done = true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);     // the library the comm came from
    if (!h) return a;
    a.MemAlloc = (decltype(a.MemAlloc))dlsym(h, "ncclMemAlloc");
    a.MemFree = (decltype(a.MemFree))dlsym(h, "ncclMemFree");
    a.WinReg = (decltype(a.WinReg))dlsym(h, "ncclCommWindowRegister");
    a.WinDereg = (decltype(a.WinDereg))dlsym(h, "ncclCommWindowDeregister");
    a.DevCommCreate = (decltype(a.DevCommCreate))dlsym(h, "ncclDevCommCreate");
    a.DevCommDestroy = (decltype(a.DevCommDestroy))dlsym(h, "ncclDevCommDestroy");
    a.ok = a.MemAlloc && a.MemFree && a.WinReg && a.WinDereg && a.DevCommCreate && a.DevCommDestroy;
    return a;
}

struct MergeParams {
    ncclDevComm dc;
    ncclWindow_t win;
    uint32_t nwords;                   // u64 counters at window offset 0
    uint32_t regs_off;                 // byte offset of the registers in the window
    uint32_t regs_words;               // u32 words of registers (4 registers each)
    unsigned long long *out;           // this rank's merged result (same layout as the window)
};

__global__ void __launch_bounds__(1024) fin_merge_lsa(const __grid_constant__ MergeParams M) {
    // launched with programmatic stream serialisation: the launch overlaps the finalize's
    // tail, and this waits for it (its window writes complete and visible) before anything
    asm volatile("griddepcontrol.wait;" ::: "memory");
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), M.dc, ncclTeamTagLsa(), blockIdx.x);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);     // every rank's result is in its window
    const int n = M.dc.lsaSize;
    for (uint32_t i = threadIdx.x; i < M.nwords; i += blockDim.x) {
        unsigned long long s = 0;
        for (int p = 0; p < n; ++p) s += static_cast<const volatile unsigned long long *>(ncclGetLsaPointer(M.win, 0, p))[i];
        M.out[i] = s;
    }
    uint32_t *oreg = reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(M.out) + M.regs_off);
    for (uint32_t i = threadIdx.x; i < M.regs_words; i += blockDim.x) {
        uint32_t m = 0;
        for (int p = 0; p < n; ++p)
            m = __vmaxu4(m, static_cast<const volatile uint32_t *>(ncclGetLsaPointer(M.win, M.regs_off, p))[i]);
        oreg[i] = m;
    }
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);     // peers are done reading this window
}

}  // namespace

bool merge_available() { return api().ok; }

bool merge_create(void *comm, int nranks, size_t bytes, MergeState **out, std::string *err) {
    Api &A = api();
    *out = nullptr;
    if (!A.ok) { *err = "NCCL device API (ncclMemAlloc / ncclDevCommCreate) not in the loaded libnccl"; return false; }
    MergeState *m = new MergeState();
    m->comm = comm;
    m->bytes = bytes;
    ncclComm_t c = static_cast<ncclComm_t>(comm);
    ncclResult_t r = A.MemAlloc(&m->buf, bytes);
    if (r == ncclSuccess) r = A.WinReg(c, m->buf, bytes, &m->win, NCCL_WIN_COLL_SYMMETRIC);
    if (r == ncclSuccess) {
        ncclDevCommRequirements_t req{};
        req.lsaBarrierCount = 1;
        r = A.DevCommCreate(c, &req, &m->dc);
        m->dc_ok = r == ncclSuccess;
    }
    if (r != ncclSuccess || m->dc.lsaSize != nranks || m->dc.nRanks != nranks) {
        *err = r != ncclSuccess ? "NCCL window / device communicator set-up failed"
                                : "not every rank is load/store reachable (LSA team smaller than the job)";
        merge_destroy(m);
        return false;
    }
    *out = m;
    return true;
}

void merge_destroy(MergeState *m) {
    if (!m) return;
    Api &A = api();
    ncclComm_t c = static_cast<ncclComm_t>(m->comm);
    if (m->dc_ok) A.DevCommDestroy(c, &m->dc);
    if (m->win) A.WinDereg(c, m->win);
    if (m->buf) A.MemFree(m->buf);
    delete m;
}

void *merge_buffer(MergeState *m, size_t *bytes) {
    if (bytes) *bytes = m->bytes;
    return m->buf;
}

cudaError_t merge_launch(MergeState *m, uint32_t nwords, uint32_t regs_off, uint32_t regs_bytes, void *out,
                         cudaStream_t s) {
    MergeParams P;
    P.dc = m->dc;
    P.win = m->win;
    P.nwords = nwords;
    P.regs_off = regs_off;
    P.regs_words = regs_bytes / 4;
    P.out = static_cast<unsigned long long *>(out);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(1024);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fin_merge_lsa, P);
}

}  // namespace gace

#else   // built without the NCCL device headers: the grouped all-reduce is the merge

namespace gace {
struct MergeState {};
bool merge_available() { return false; }
bool merge_create(void *, int, size_t, MergeState **out, std::string *err) {
    *out = nullptr;
    *err = "built without the NCCL device API headers";
    return false;
}
void merge_destroy(MergeState *) {}
void *merge_buffer(MergeState *, size_t *bytes) {
    if (bytes) *bytes = 0;
    return nullptr;
}
cudaError_t merge_launch(MergeState *, uint32_t, uint32_t, uint32_t, void *, cudaStream_t) {
    return cudaErrorNotSupported;
}
}  // namespace gace

#endif
