// ajm.cu -- host runtime + C ABI (include/ajm.h) of the B200-native AJM solver.
//
// create : validate (host row_ptr scan + device column/value kernel, optional symmetry kernel),
//          D per dmode (eq-J-diag on the device), ||b|| (deterministic two-level
//          reduction), and the row-length-binned layout:
//            rows <= AJM_SELL_MAX nonzeros -> SELL-32-sigma chunks (sigma = 1 when natural order
//              pads < 5%, else rows sorted by length inside windows of 4096), thread per row;
//            longer rows -> warp segments of <= AJM_SEG nonzeros (several segments: split row,
//              finished by an owner CTA);
//          SELL chunks grouped into TMA staging units (<= 8 chunks, <= AJM_UNIT_EL elements);
//          segments and units assigned to the CTAs of a persistent grid (#SMs x resident
//          CTAs/SM) in contiguous cost-balanced ranges.
// solve  : init kernel -> ONE cooperative launch of ajm_solve_kernel that runs every pass of
//          Alg. 3 with a grid barrier per pass and device-side control (no host round trip, no
//          relaunch) -> copy-out of the answer buffer, histories and the control block.
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <functional>
#include <omp.h>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges visible to nsys / ncu, no link dependency

#include "ajm.h"
#include "ajm_kernels.cuh"

namespace {

thread_local std::string g_create_error;
thread_local bool g_poison = false;  // AJM_DEBUG_POISON during a create (tests)

// NVTX range for the duration of a scope (SURVEY §5 tracing: create / solve / destroy)
struct NvtxScope {
    explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
    ~NvtxScope() { nvtxRangePop(); }
};

typedef void (*SolveFn)(AjmPass);

// Solver kernel instantiations (ajm_solve_kernel<stages, kSeg, kCluster, kJB, kGMeta, kCol8>,
// DESIGN.md §4).  The TMA ring depth sets how much of the SM's unified L1/shared memory is left to
// the L1, which holds the x~ gathers' lines in flight.
// int32 columns: ring depth 2-4, with or without the segment phases
SolveFn ring_fn(bool seg, int stages) {
    switch (stages) {
        case 2: return seg ? ajm_solve_kernel<2, true> : ajm_solve_kernel<2, false>;
        case 3: return seg ? ajm_solve_kernel<3, true> : ajm_solve_kernel<3, false>;
        default: return seg ? ajm_solve_kernel<4, true> : ajm_solve_kernel<4, false>;
    }
}
// byte-coded columns: ring depth 3-6 (18 KB stages)
SolveFn col8_fn(bool seg, int stages) {
    switch (stages) {
        case 3: return seg ? ajm_solve_kernel<3, true, false, 0, false, true> : ajm_solve_kernel<3, false, false, 0, false, true>;
        case 5: return seg ? ajm_solve_kernel<5, true, false, 0, false, true> : ajm_solve_kernel<5, false, false, 0, false, true>;
        case 6: return seg ? ajm_solve_kernel<6, true, false, 0, false, true> : ajm_solve_kernel<6, false, false, 0, false, true>;
        default: return seg ? ajm_solve_kernel<4, true, false, 0, false, true> : ajm_solve_kernel<4, false, false, 0, false, true>;
    }
}
// pair-coded entries (1 byte per entry, no values streamed; 2 KB stages): ring depth 4 or 8,
// with or without the segment phases
SolveFn pair_fn(bool seg, int stages) {
    if (stages == 8) return seg ? ajm_solve_kernel<8, true, false, 0, false, 2> : ajm_solve_kernel<8, false, false, 0, false, 2>;
    return seg ? ajm_solve_kernel<4, true, false, 0, false, 2> : ajm_solve_kernel<4, false, false, 0, false, 2>;
}
// banded staging (natural-order pair-coded stencils): ring depth 2-4 (stages of 12-30 KB)
SolveFn band_fn(int stages, int ku) {
    if (ku == 16) return stages >= 3 ? ajm_band_kernel<3, 16> : ajm_band_kernel<2, 16>;
    return stages >= 4 ? ajm_band_kernel<4, 8> : stages == 3 ? ajm_band_kernel<3, 8> : ajm_band_kernel<2, 8>;
}
// block-diagonal J (natural order, no segments), cooperative grid or single cluster
SolveFn jblock_fn(int bs, bool cluster) {
    if (cluster)
        return bs == 2 ? ajm_solve_kernel<4, false, true, 2> : bs == 4 ? ajm_solve_kernel<4, false, true, 4>
             : bs == 8 ? ajm_solve_kernel<4, false, true, 8> : ajm_solve_kernel<4, false, true, -1>;
    return bs == 2 ? ajm_solve_kernel<4, false, false, 2> : bs == 4 ? ajm_solve_kernel<4, false, false, 4>
         : bs == 8 ? ajm_solve_kernel<4, false, false, 8> : ajm_solve_kernel<4, false, false, -1>;
}
// block-diagonal J on pair-coded entries (natural-order stencils; 1-byte stages)
SolveFn jblock_pair_fn(int bs) {
    return bs == 2 ? ajm_solve_kernel<4, false, false, 2, false, 2> : bs == 4 ? ajm_solve_kernel<4, false, false, 4, false, 2>
         : bs == 8 ? ajm_solve_kernel<4, false, false, 8, false, 2> : ajm_solve_kernel<4, false, false, -1, false, 2>;
}
SolveFn gmeta_fn(bool seg) { return seg ? ajm_solve_kernel<4, true, false, 0, true> : ajm_solve_kernel<4, false, false, 0, true>; }
SolveFn cluster_fn(bool seg) { return seg ? ajm_solve_kernel<4, true, true> : ajm_solve_kernel<4, false, true>; }

// The Lanczos twin (kLz) of a handle's solver kernel: same template arguments, same ring and shared
// memory, Lanczos epilogue (ajm_estimate_spectrum).  Instantiated for the layouts create picks by
// default; nullptr for block-J handles and experiment-only ring depths.
SolveFn lanczos_fn(bool seg, bool cluster, bool gmeta, int col_bytes, int stages, bool pair) {
    if (pair) {
        if (stages == 8) return seg ? ajm_solve_kernel<8, true, false, 0, false, 2, true> : ajm_solve_kernel<8, false, false, 0, false, 2, true>;
        return seg ? ajm_solve_kernel<4, true, false, 0, false, 2, true> : ajm_solve_kernel<4, false, false, 0, false, 2, true>;
    }
    if (cluster) return seg ? ajm_solve_kernel<4, true, true, 0, false, false, true> : ajm_solve_kernel<4, false, true, 0, false, false, true>;
    if (gmeta) return seg ? ajm_solve_kernel<4, true, false, 0, true, false, true> : ajm_solve_kernel<4, false, false, 0, true, false, true>;
    if (col_bytes == 1) {
        if (stages == 4) return seg ? ajm_solve_kernel<4, true, false, 0, false, true, true> : ajm_solve_kernel<4, false, false, 0, false, true, true>;
        if (stages == 5) return seg ? ajm_solve_kernel<5, true, false, 0, false, true, true> : ajm_solve_kernel<5, false, false, 0, false, true, true>;
        return nullptr;
    }
    if (stages == 3) return seg ? ajm_solve_kernel<3, true, false, 0, false, false, true> : ajm_solve_kernel<3, false, false, 0, false, false, true>;
    if (stages == 4) return seg ? ajm_solve_kernel<4, true, false, 0, false, false, true> : ajm_solve_kernel<4, false, false, 0, false, false, true>;
    return nullptr;
}

// One rank of a row-block sharded solve: int32 columns at ring depth 3 / 4 or byte-coded columns at
// 4 / 5, with or without the segment phases -- the layouts create picks for shards; emu: the
// emulated-group kernel (kShard = 2) instead of the per-process one (kShard = 1)
template <int kSh>
SolveFn shard_fn_t(int col_bytes, bool seg, int stages, bool pair) {
    if (pair) return ajm_solve_kernel<4, false, false, 0, false, 2, false, kSh>;  // (no segments)
    if (col_bytes == 1) {
        if (stages == 5) return seg ? ajm_solve_kernel<5, true, false, 0, false, true, false, kSh> : ajm_solve_kernel<5, false, false, 0, false, true, false, kSh>;
        return seg ? ajm_solve_kernel<4, true, false, 0, false, true, false, kSh> : ajm_solve_kernel<4, false, false, 0, false, true, false, kSh>;
    }
    if (stages == 4) return seg ? ajm_solve_kernel<4, true, false, 0, false, false, false, kSh> : ajm_solve_kernel<4, false, false, 0, false, false, false, kSh>;
    return seg ? ajm_solve_kernel<3, true, false, 0, false, false, false, kSh> : ajm_solve_kernel<3, false, false, 0, false, false, false, kSh>;
}
SolveFn shard_fn(int col_bytes, bool seg, int stages, bool emu, bool pair) {
    return emu ? shard_fn_t<2>(col_bytes, seg, stages, pair) : shard_fn_t<1>(col_bytes, seg, stages, pair);
}

// Threads per CTA of a solver kernel: 8 consumer warps + the TMA producer warp (kProd, layouts
// without warp segments), or the 8 warps alone (segment layouts: the last warp to release a stage
// refills it, and 128 registers per thread fit).  Every kernel a handle uses shares its nseg > 0.
int block_threads(bool seg) { return seg ? AJM_BLOCK : AJM_BLOCK + 32; }

// Kernel attributes (max dynamic shared memory, carve-out) belong to the kernel, which every handle
// of that layout shares: they are set -- and occupancy is queried -- under one library-wide lock,
// and each launch sets its own handle's values and launches before releasing it.
std::mutex g_attr_mu;

// set the attributes of fn and return the resident CTAs per SM (0 on failure); caller holds g_attr_mu
cudaError_t fn_occupancy(SolveFn fn, size_t dyn_smem, int carveout, int* occ, int threads) {
    cudaError_t e = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, fn, threads, dyn_smem);
    return e;
}

// Persisting-L2 limit: raised by creates whose vectors fit the L2 and restored (with the
// persisting lines reset) when the last such handle is destroyed, so no handle's L2 state leaks
// into later work.
struct PersistState {
    int holders = 0;
    size_t saved_limit = 0;
};
PersistState g_persist[64];

}  // namespace

struct ajm_ctx {
    int device = 0;
    int sm_count = 0;
    int ctas_per_sm = 0;
    int64_t n = 0, nnz = 0, n_pad = 0;
    int64_t nchunks = 0, n_sell = 0, sell_elems = 0;
    int64_t nseg = 0, nsplit = 0, seg_rows = 0, long_rows = 0, seg_nnz = 0;
    int sigma = 1;
    bool relabel = false;           // SELL slot order != caller's row order: vectors live in slot order
    int* perm_fwd = nullptr;        // [n] internal (layout) index -> caller's row
    int* perm_inv = nullptr;        // [n] caller's row -> internal index
    SolveFn fn = nullptr;
    SolveFn fn_lz = nullptr;           // Lanczos twin of fn (ajm_estimate_spectrum), or nullptr
    double* lzw = nullptr;             // Lanczos workspace: p x3, Qp x3, g x2 (n_pad each)
    size_t dyn_smem = 0;
    int64_t nunits = 0;
    int meta_units = 0, meta_chunks = 0;
    int l2_mode = 2;
    int cluster = 0;                   // grid <= 16 CTAs launched as one cluster (DSMEM barrier)
    int gmeta = 0;                     // per-CTA unit/chunk tables in global memory (huge layouts)
    int* g_uc0 = nullptr;
    int* g_coff = nullptr;
    long long* g_ubase = nullptr;
    long long* g_cbase = nullptr;
    unsigned long long* ts = nullptr;  // debug phase timestamps (AJM_TS=1)
    double* vecs = nullptr;            // X0 X1 X2 Qxp b D, one allocation
    int l2persist = 1;
    bool persist_holder = false;       // this handle raised the device's persisting-L2 limit
    size_t win_bytes = 0;
    float win_hit = 0.f;
    size_t prime_bytes = 0;  // (l2_mode 3) window over all six vectors for the per-solve L2 priming
    float prime_hit = 0.f;
    int grid = 0;
    uint32_t flags = 0;
    // device arrays
    long long* rp = nullptr;   // int64 row offsets (create-time kernels; nnz may exceed 2^31)
    int* col = nullptr;
    double* val = nullptr;
    double* b = nullptr;
    double* D = nullptr;
    double* X[3] = {nullptr, nullptr, nullptr};
    double* Qxp = nullptr;
    double* sval = nullptr;
    int* scol = nullptr;
    long long* chunk_off = nullptr;
    int* seg_row = nullptr;
    int* seg_k0 = nullptr;
    int* seg_k1 = nullptr;
    int* seg_split = nullptr;
    double* seg_part = nullptr;
    int* split_row = nullptr;
    int* split_seg0 = nullptr;
    unsigned* split_cnt = nullptr;
    int* cta_split = nullptr;
    int* owner_split = nullptr;
    int* unit_c0 = nullptr;
    int* cta_seg = nullptr;
    int* seg_list = nullptr;
    int* seg_order = nullptr;       // dynamic segment queue: segments in claim order (longest first)
    int* seg_grp = nullptr;         // claim g -> seg_order[seg_grp[g] .. seg_grp[g+1])
    int64_t nsegq = 0;              // claim groups
    int dynseg = 0;                 // segments claimed dynamically by warps (else static LPT plan)
    int* cta_unit = nullptr;
    int* seg_meta = nullptr;        // int4 {row, k0, k1, split} per static seg_list position
    int4* grp = nullptr;            // sub-warp groups: 3 int4 per group ({rows}, {k0}, {k1})
    int64_t ngrp = 0, grp_rows = 0;
    double* partials = nullptr;
    AjmCtrl* ctrl = nullptr;
    double* hist = nullptr;  // 4 x hist_cap: res, f, d, dabs
    int64_t hist_cap = 0;
    double* scratch = nullptr;  // reductions at create
    int* err = nullptr;
    AjmCtrl* h_ctrl = nullptr;  // host copy of the control block
    double* b_in = nullptr;     // b as given (caller's order), until the layout exists
    int dmode = 0;
    int jbs = 0;                // AJM_D_JBLOCK block size (0: diagonal metric)
    double* Jblk = nullptr;     // [s][bs][bs] blocks of eq-J-blkdiag
    double* Jinv = nullptr;     // rows of their inverses, per SELL chunk [bs][32]
    uint8_t* scode = nullptr;   // byte-coded SELL columns (col = row + ctab[code]), replaces scol
    int* ctab = nullptr;        // [AJM_CTAB] ascending column offsets of the codes
    long long* ptab = nullptr;  // [AJM_CTAB][2] pair-coded entries {value bits, offset}
    int col_bytes = 4;          // bytes per streamed column index: 4 (int32) or 1 (byte code)
    int pair = 0;               // 1: the byte code carries the value too (no values streamed)
    int band = 0;               // 1: ajm_band_kernel (x~ bands and row operands staged by the TMA)
    AjmBand bd = {};            // its band layout
    long long* bptab = nullptr; // [AJM_CTAB][2] {value bits, stage offset} of the pair codes
    int* band_c0 = nullptr;     // [grid+1] first SELL chunk of each band-kernel CTA
    int* smid = nullptr;        // [grid] placement probe output (SM of each CTA)
    double band_skew = 0.0;     // work skew applied between the two CTAs sharing an SM (0: none)
    int ring_stages = 4;        // TMA ring depth of the chosen solver kernel
    bool seg_fn = true;         // the chosen plain/col8 ring kernel has the segment phases
    bool ring_fn = false;       // h->fn is a ring_fn/col8_fn kernel (ring depth selectable)
    bool wide_rows = false;     // SELL chunks average >= 16 entries per row
    size_t meta_bytes = 0;      // shared-memory unit/chunk tables behind the ring
    int carveout = 100;         // preferred shared-memory carve-out (%), set before every launch
    double nb = 0.0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    double last_loop_ms = 0.0;
    int64_t last_passes = 0;
    int64_t last_launches = 0;
    int64_t last_iterations = -1;
    std::string err_msg;
    // ---- row-block shard (NEXT-2; ajm_shard_create) ----
    int resident = 0;                  // the resident single-cluster kernel (ajm_resident_kernel)
    std::vector<int> cta_nchk;         // (AJM_TS_ALL diagnostics) SELL chunks planned per CTA
    size_t lz_dyn_smem = 0;            // dynamic shared memory of the Lanczos twin
    int shard = 0;                     // 1: one rank of a sharded group
    int rank = 0, nranks = 1;
    int colocated = 0;                 // AJM_SHARD_COLOCATED: the group runs as one launch here
    int64_t n_glob = 0, row0 = 0;
    int64_t h_lo = 0, h_hi = 0;        // halo entries below / above the own rows
    int64_t lo_pad = 0, xstride = 0;   // X_k = vecs + k * xstride + lo_pad
    double bsq_local = 0.0;            // ||b_r||^2 of the own rows
    std::vector<int64_t> halo_cnt, send_cnt;  // [nranks]
    std::vector<int4> snd_host;        // per CTA: {internal row, peer, k-th entry of the list to peer, 0}
    std::vector<int> snd_cta_host;     // [grid+1]
    int* snd_cta = nullptr;
    int4* snd = nullptr;
    double* xch = nullptr;             // cudaMalloc (IPC-exportable): slots [2][MAXR][NPART] + counter
    AjmPeer* peers = nullptr;          // [nranks] device
    std::vector<AjmPeer> peers_host;
    std::vector<void*> ipc_opened;     // peer allocations opened through CUDA IPC
    bool connected = false;
    bool broken = false;               // a cross-rank wait timed out: the counters are out of step
    unsigned long long bar_base = 0;   // cross-rank arrivals of earlier solves
    AjmPass* emu = nullptr;            // (colocated, rank 0) device array of the group's pass structs
};

namespace {

ajm_status_t fail(ajm_ctx* h, ajm_status_t s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (h) h->err_msg = buf;
    else g_create_error = buf;
    return s;
}

#define AJM_CUDA(h, call)                                                                      \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess) {                                                               \
            ajm_status_t s_ = (e_ == cudaErrorMemoryAllocation) ? AJM_ERR_OOM : AJM_ERR_CUDA;  \
            return fail(h, s_, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                        __LINE__);                                                             \
        }                                                                                      \
    } while (0)

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

cudaMemcpyKind kind_to_device(const void* src) {
    return is_device_ptr(src) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
}

cudaMemcpyKind kind_from_device(const void* dst) {
    return is_device_ptr(dst) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
}

// Device memory comes from a library-owned stream-ordered pool that keeps freed memory (up to a
// release threshold), so the allocations of a create after a destroy cost no cudaMalloc and a
// destroy costs no synchronising cudaFree.
cudaMemPool_t ajm_pool(int dev) {
    static cudaMemPool_t pools[64] = {};
    static std::mutex mu;  // first use from several threads at once
    if (dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> lock(mu);
    if (!pools[dev]) {
        cudaMemPoolProps pp = {};
        pp.allocType = cudaMemAllocationTypePinned;
        pp.handleTypes = cudaMemHandleTypeNone;
        pp.location.type = cudaMemLocationTypeDevice;
        pp.location.id = dev;
        cudaMemPool_t mp = nullptr;
        if (cudaMemPoolCreate(&mp, &pp) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        // keep up to 16 GiB of freed memory for the next create; anything above goes back to the
        // driver at the next synchronisation (so a huge solver does not hoard HBM after destroy)
        uint64_t thr = 16ull << 30;
        cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr);
        pools[dev] = mp;
    }
    return pools[dev];
}

template <class T>
cudaError_t dalloc(T** p, size_t count, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t mp = ajm_pool(dev);
    const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    if (!mp) return cudaMalloc((void**)p, bytes);
    cudaError_t e = cudaMallocFromPoolAsync((void**)p, bytes, mp, s);
    // AJM_POISON (tests): fill new allocations with 0xff so a read of memory the library never
    // wrote shows up deterministically instead of depending on what the pool hands back
    if (e == cudaSuccess && g_poison) cudaMemsetAsync(*p, 0xff, bytes, s);
    return e;
}

void dfree(void* p) {
    if (p) cudaFreeAsync(p, 0);  // nothing of the handle is in flight when it is freed
}

void free_all(ajm_ctx* h) {
    void* ptrs[] = {h->rp, h->col, h->val, h->shard ? nullptr : h->vecs,
                    h->sval, h->scol, h->chunk_off, h->seg_row, h->seg_k0, h->seg_k1,
                    h->seg_split, h->seg_part, h->split_row, h->split_seg0, h->split_cnt,
                    h->cta_split, h->owner_split, h->unit_c0, h->cta_seg, h->seg_list, h->cta_unit, h->partials, h->ctrl,
                    h->hist, h->scratch, h->err, h->ts, h->perm_fwd, h->perm_inv, h->b_in, h->Jblk, h->Jinv, h->seg_order, h->seg_grp,
                    h->g_uc0, h->g_coff, h->g_ubase, h->g_cbase, h->scode, h->ctab, h->seg_meta, h->lzw, h->grp, h->ptab, h->bptab,
                    h->band_c0, h->smid};
    for (void* p : ptrs) dfree(p);
    dfree(h->snd_cta);
    dfree(h->snd);
    dfree(h->peers);
    dfree(h->emu);
    for (void* p : h->ipc_opened) cudaIpcCloseMemHandle(p);
    h->ipc_opened.clear();
    if (h->xch) cudaFree(h->xch);
    if (h->shard && h->vecs) {  // cudaMalloc'd (IPC-exportable), not from the pool
        cudaFree(h->vecs);
        h->vecs = nullptr;
    }
    if (h->persist_holder) {  // the last holder restores the limit and drops the persisting lines
        std::lock_guard<std::mutex> lock(g_attr_mu);
        PersistState& ps = g_persist[h->device];
        if (--ps.holders == 0) {
            int cur_dev = 0;
            cudaGetDevice(&cur_dev);
            if (cur_dev != h->device) cudaSetDevice(h->device);
            cudaCtxResetPersistingL2Cache();
            cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, ps.saved_limit);
            if (cur_dev != h->device) cudaSetDevice(cur_dev);
            cudaGetLastError();
        }
        h->persist_holder = false;
    }
    if (h->h_ctrl) free(h->h_ctrl);
    if (h->ev0) cudaEventDestroy(h->ev0);
    if (h->ev1) cudaEventDestroy(h->ev1);
}

AjmPass make_pass(ajm_ctx* h, int max_passes) {
    AjmPass p;
    p.rp = h->rp;
    p.col = h->col;
    p.val = h->val;
    p.sval = h->sval;
    p.scol = h->scol;
    p.chunk_off = h->chunk_off;
    p.seg_row = h->seg_row;
    p.seg_k0 = h->seg_k0;
    p.seg_k1 = h->seg_k1;
    p.seg_split = h->seg_split;
    p.seg_part = h->seg_part;
    p.split_row = h->split_row;
    p.split_seg0 = h->split_seg0;
    p.split_cnt = h->split_cnt;
    p.cta_split = h->cta_split;
    p.owner_split = h->owner_split;
    p.unit_c0 = h->unit_c0;
    p.cta_seg = h->cta_seg;
    p.seg_list = h->seg_list;
    p.seg_order = h->seg_order;
    p.dynseg = h->dynseg;
    p.nseg = (int)h->nsegq;
    p.seg_grp = h->seg_grp;
    p.cta_unit = h->cta_unit;
    p.b = h->b;
    p.D = h->D;
    p.X0 = h->X[0];
    p.X1 = h->X[1];
    p.X2 = h->X[2];
    p.Qxp = h->Qxp;
    p.partials = h->partials;
    p.ctrl = h->ctrl;
    p.n = (int)h->n;
    p.n_sell = (int)h->n_sell;
    p.max_passes = max_passes;
    p.meta_units = h->meta_units;
    p.meta_chunks = h->meta_chunks;
    p.l2_mode = h->l2_mode;
    p.ts = h->ts;
    p.g_uc0 = h->g_uc0;
    p.g_coff = h->g_coff;
    p.g_ubase = h->g_ubase;
    p.g_cbase = h->g_cbase;
    p.Jinv = h->Jinv;
    p.jbs = h->jbs;
    p.scode = h->scode;
    p.seg_meta = reinterpret_cast<const int4*>(h->seg_meta);
    p.grp = h->grp;
    p.ctab = h->ctab;
    p.ptab = h->ptab;
    p.sh = AjmShard{};
    p.sh.nranks = 1;
    p.bd = h->bd;
    p.bptab = h->bptab;
    p.band_c0 = h->band_c0;
    p.smid_out = nullptr;
    if (h->shard) {
        p.sh.rank = h->rank;
        p.sh.nranks = h->nranks;
        p.sh.peers = h->peers;
        p.sh.snd_cta = h->snd_cta;
        p.sh.snd = h->snd;
        p.sh.slot = h->xch;
        p.sh.bar = reinterpret_cast<unsigned long long*>(h->xch + 2 * AJM_MAX_RANKS * AJM_NPART);
        p.sh.bar_base = h->bar_base;
    }
    return p;
}

// cooperative launch of the persistent solver kernel, with the L2 access-policy window over the
// iterate vectors (persisting hits, streaming misses)
cudaError_t launch_solver(ajm_ctx* h, AjmPass& p, cudaStream_t st, SolveFn fn = nullptr) {
    // the solver kernel, or its Lanczos twin (which keeps the ring kernel's shared-memory layout and
    // block when the solver is the resident single-cluster kernel)
    const bool lz = fn != nullptr && fn != h->fn;
    if (!fn) fn = h->fn;
    const size_t dyn = lz ? h->lz_dyn_smem : h->dyn_smem;
    const int threads = (h->resident && !lz) ? AJM_BLOCK : block_threads(h->nseg > 0);
    // the attributes belong to the kernel, which other handles share: set this handle's own, and
    // launch before another thread's handle can change them (the launch itself is asynchronous)
    std::lock_guard<std::mutex> lock(g_attr_mu);
    cudaError_t e = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributePreferredSharedMemoryCarveout, h->carveout);
    if (e == cudaSuccess && h->cluster && h->grid > 8)
        e = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(h->grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = dyn;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    if (h->cluster) {  // the grid is one thread-block cluster (co-scheduled by construction)
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)h->grid;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
    } else {
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
    }
    int na = 1;
    if (h->win_bytes) {
        at[1].id = cudaLaunchAttributeAccessPolicyWindow;
        at[1].val.accessPolicyWindow.base_ptr = h->vecs;
        at[1].val.accessPolicyWindow.num_bytes = h->win_bytes;
        at[1].val.accessPolicyWindow.hitRatio = h->win_hit;
        at[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        at[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        na = 2;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, fn, p);
}

ajm_status_t ensure_hist(ajm_ctx* h, int64_t need, cudaStream_t st) {
    if (need <= h->hist_cap) return AJM_OK;
    if (h->hist) {
        dfree(h->hist);
        h->hist = nullptr;
    }
    int64_t cap = std::max<int64_t>(need, 1024);
    AJM_CUDA(h, dalloc(&h->hist, (size_t)cap * 4, st));
    h->hist_cap = cap;
    return AJM_OK;
}

// ---- symmetric tridiagonal T_k (Lanczos coefficients) on the host: k <= a few thousand ----
// Sturm count: eigenvalues of T (diag a[0..k), off-diagonal b[0..k-1)) strictly below x
int tri_sturm(const std::vector<double>& a, const std::vector<double>& b, int k, double x) {
    int cnt = 0;
    double d = 1.0;
    for (int i = 0; i < k; ++i) {
        const double bb = i ? b[(size_t)i - 1] * b[(size_t)i - 1] : 0.0;
        d = a[(size_t)i] - x - (i ? bb / d : 0.0);
        if (d == 0.0) d = -1e-300;  // x is (numerically) an eigenvalue: count it as below
        if (d < 0.0) ++cnt;
    }
    return cnt;
}

// the m-th smallest eigenvalue (m = 0 .. k-1) by bisection on the Sturm count, to full precision
double tri_eig(const std::vector<double>& a, const std::vector<double>& b, int k, int m) {
    double lo = a[0], hi = a[0];
    for (int i = 0; i < k; ++i) {  // Gershgorin
        const double r = (i ? std::fabs(b[(size_t)i - 1]) : 0.0) + (i + 1 < k ? std::fabs(b[(size_t)i]) : 0.0);
        lo = std::min(lo, a[(size_t)i] - r);
        hi = std::max(hi, a[(size_t)i] + r);
    }
    for (int it = 0; it < 200; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (mid <= lo || mid >= hi) break;
        if (tri_sturm(a, b, k, mid) > m) hi = mid;
        else lo = mid;
    }
    return 0.5 * (lo + hi);
}

// |last component| of the unit eigenvector of T for the eigenvalue theta: two steps of inverse
// iteration with a tridiagonal LU with partial pivoting (shift perturbed off the exact eigenvalue)
double tri_last_component(const std::vector<double>& a, const std::vector<double>& b, int k, double theta) {
    if (k == 1) return 1.0;
    double scale = 0.0;
    for (int i = 0; i < k; ++i) scale = std::max(scale, std::fabs(a[(size_t)i]) + (i + 1 < k ? std::fabs(b[(size_t)i]) : 0.0));
    const double sh = theta + 1e-13 * std::max(scale, 1e-300);
    std::vector<double> y((size_t)k, 1.0);
    for (int rep = 0; rep < 3; ++rep) {
        // (T - sh I) x = y: rows i of the banded system, partial pivoting (dgtsv-style)
        std::vector<double> dl((size_t)k, 0.0), d((size_t)k), du((size_t)k, 0.0), du2((size_t)k, 0.0), x = y;
        for (int i = 0; i < k; ++i) {
            d[(size_t)i] = a[(size_t)i] - sh;
            if (i + 1 < k) { du[(size_t)i] = b[(size_t)i]; dl[(size_t)i] = b[(size_t)i]; }
        }
        for (int i = 0; i + 1 < k; ++i) {
            if (std::fabs(d[(size_t)i]) >= std::fabs(dl[(size_t)i])) {  // no interchange
                if (d[(size_t)i] == 0.0) d[(size_t)i] = 1e-300;
                const double f = dl[(size_t)i] / d[(size_t)i];
                d[(size_t)i + 1] -= f * du[(size_t)i];
                x[(size_t)i + 1] -= f * x[(size_t)i];
                du2[(size_t)i] = 0.0;
            } else {  // swap rows i and i+1
                const double f = d[(size_t)i] / dl[(size_t)i];
                d[(size_t)i] = dl[(size_t)i];
                const double tmp = d[(size_t)i + 1];
                d[(size_t)i + 1] = du[(size_t)i] - f * tmp;
                if (i + 2 < k) {
                    du2[(size_t)i] = du[(size_t)i + 1];
                    du[(size_t)i + 1] = -f * du2[(size_t)i];
                }
                du[(size_t)i] = tmp;
                const double tx = x[(size_t)i];
                x[(size_t)i] = x[(size_t)i + 1];
                x[(size_t)i + 1] = tx - f * x[(size_t)i + 1];
            }
        }
        if (d[(size_t)k - 1] == 0.0) d[(size_t)k - 1] = 1e-300;
        x[(size_t)k - 1] /= d[(size_t)k - 1];
        if (k >= 2) x[(size_t)k - 2] = (x[(size_t)k - 2] - du[(size_t)k - 2] * x[(size_t)k - 1]) / d[(size_t)k - 2];
        for (int i = k - 3; i >= 0; --i)
            x[(size_t)i] = (x[(size_t)i] - du[(size_t)i] * x[(size_t)i + 1] - du2[(size_t)i] * x[(size_t)i + 2]) / d[(size_t)i];
        double nrm = 0.0;
        for (double v : x) nrm += v * v;
        nrm = std::sqrt(nrm);
        if (!(nrm > 0.0) || !std::isfinite(nrm)) return 1.0;  // no information: the worst case
        for (int i = 0; i < k; ++i) y[(size_t)i] = x[(size_t)i] / nrm;
    }
    return std::fabs(y[(size_t)k - 1]);
}

// What ajm_shard_create hands to the common create path (host data of the rank's plan)
struct ShardIn {
    int rank = 0, nranks = 1;
    int colocated = 0;
    int64_t n_glob = 0, row0 = 0;
    int64_t h_lo = 0, h_hi = 0;
    std::vector<int64_t> halo_cnt, send_cnt;  // [nranks]
    std::vector<int64_t> send_rows;           // own local rows, grouped by destination rank
};

}  // namespace

extern "C" {

int32_t ajm_abi_version(void) { return AJM_ABI_VERSION; }

const char* ajm_last_error(ajm_handle_t h) {
    return h ? h->err_msg.c_str() : g_create_error.c_str();
}

// The create path of ajm_create and (sh != NULL) ajm_shard_create: a shard's rows are an ordinary
// n-row matrix whose columns may also reach its halo, [-H_lo, n + H_hi).
static ajm_status_t create_impl(ajm_handle_t* out, int64_t n, int64_t nnz, const int64_t* row_ptr,
                                const int32_t* col_idx, const double* vals, const double* b, int32_t dmode,
                                const double* d, uint32_t flags, void* cuda_stream, const ShardIn* sh) {
    NvtxScope nvtx_scope_(sh ? "ajm_shard_create" : "ajm_create");
    g_create_error.clear();
    g_poison = (flags & AJM_DEBUG_POISON) != 0;
    struct PoisonReset { ~PoisonReset() { g_poison = false; } } poison_reset_;
    // debug (AJM_TS): host wall time of each create phase
    const bool tsc = getenv("AJM_TS") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    std::string tsc_log;
    auto mark = [&](const char* what, cudaStream_t s_) {
        if (!tsc) return;
        if (s_ != (cudaStream_t)-1) {
            cudaError_t e_ = cudaStreamSynchronize(s_);
            if (e_ != cudaSuccess) fprintf(stderr, "[ajm create] error after phase before '%s': %s\n", what, cudaGetErrorString(e_));
        }
        auto now = std::chrono::steady_clock::now();
        char b[96];
        snprintf(b, sizeof b, " %s %.2f", what, std::chrono::duration<double, std::milli>(now - t_last).count());
        tsc_log += b;
        t_last = now;
    };
    if (!out) return fail(nullptr, AJM_ERR_INVALID_ARG, "out is NULL");
    if (n < 1 || nnz < 0) return fail(nullptr, AJM_ERR_INVALID_ARG, "n must be >= 1 and nnz >= 0");
    if (n >= (int64_t)1 << 31)
        return fail(nullptr, AJM_ERR_UNSUPPORTED, "n must be < 2^31 (int32 column indices)");
    if (!row_ptr || !b || (nnz > 0 && (!col_idx || !vals)))
        return fail(nullptr, AJM_ERR_INVALID_ARG, "NULL array argument");
    if (dmode < 0 || dmode > 3) return fail(nullptr, AJM_ERR_INVALID_ARG, "bad dmode %d", dmode);
    const int jbs = dmode == AJM_D_JBLOCK ? (int)AJM_JBLOCK_SIZE_OF(flags) : 0;
    if (dmode == AJM_D_JBLOCK && (jbs < 1 || jbs > 32 || (jbs & (jbs - 1))))
        return fail(nullptr, AJM_ERR_INVALID_ARG, "AJM_D_JBLOCK needs AJM_JBLOCK_SIZE(bs) with bs in {1,2,4,8,16,32}");
    if (dmode == AJM_D_USER && !d) return fail(nullptr, AJM_ERR_INVALID_ARG, "AJM_D_USER needs d");
    if (sh && dmode == AJM_D_JBLOCK) return fail(nullptr, AJM_ERR_UNSUPPORTED, "sharded handles support diagonal metrics only");
    if (sh && (flags & (AJM_VALIDATE_SYMMETRY | AJM_GLOBAL_TABLES | AJM_LOOP_HOST)))
        return fail(nullptr, AJM_ERR_UNSUPPORTED, "AJM_VALIDATE_SYMMETRY / AJM_GLOBAL_TABLES / AJM_LOOP_HOST are not available for shards");
    const int64_t clo = sh ? -sh->h_lo : 0, chi = sh ? n + sh->h_hi : n;  // column range
    if (chi >= ((int64_t)1 << 31) - 1) return fail(nullptr, AJM_ERR_UNSUPPORTED, "n + halo must be < 2^31");
    cudaStream_t st = (cudaStream_t)cuda_stream;

    // the O(1) consistency checks before any copy: with row_ptr[0] = 0 and row_ptr[n] = nnz the
    // arrays the copies below read have the sizes the caller declared
    {
        int64_t ends[2] = {0, 0};
        if (is_device_ptr(row_ptr)) {
            cudaError_t e = cudaMemcpyAsync(&ends[0], row_ptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaMemcpyAsync(&ends[1], row_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) return fail(nullptr, AJM_ERR_CUDA, "row_ptr copy: %s", cudaGetErrorString(e));
        } else {
            ends[0] = row_ptr[0];
            ends[1] = row_ptr[n];
        }
        if (ends[0] != 0) return fail(nullptr, AJM_ERR_CSR_INVALID, "row_ptr[0] = %lld != 0", (long long)ends[0]);
        if (ends[1] != nnz)
            return fail(nullptr, AJM_ERR_CSR_INVALID, "row_ptr[n] = %lld != nnz = %lld", (long long)ends[1], (long long)nnz);
    }
    ajm_ctx* h = new ajm_ctx();
    h->n = n;
    h->nnz = nnz;
    if (sh) {
        h->shard = 1;
        h->rank = sh->rank;
        h->nranks = sh->nranks;
        h->colocated = sh->colocated;
        h->n_glob = sh->n_glob;
        h->row0 = sh->row0;
        h->h_lo = sh->h_lo;
        h->h_hi = sh->h_hi;
        h->halo_cnt = sh->halo_cnt;
        h->send_cnt = sh->send_cnt;
        // one process per GPU: the rank's iterate buffers get the device's persisting L2 window like a
        // single-GPU handle (emulated groups share one device and one launch: none)
        h->l2persist = sh->colocated ? 0 : 1;
    }
    h->flags = flags;
    h->dmode = dmode;
    h->jbs = jbs;
    auto bail = [&](ajm_status_t s) {
        cudaStreamSynchronize(st);  // no copy into the handle's memory still in flight
        cudaGetLastError();
        g_create_error = h->err_msg;
        free_all(h);
        delete h;
        return s;
    };
#define CC(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return bail(fail(h, e_ == cudaErrorMemoryAllocation ? AJM_ERR_OOM : AJM_ERR_CUDA,      \
                             "%s: %s", #call, cudaGetErrorString(e_)));                           \
    } while (0)

    CC(cudaGetDevice(&h->device));
    CC(cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, h->device));
    int coop = 0;
    CC(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, h->device));
    if (!coop) return bail(fail(h, AJM_ERR_UNSUPPORTED, "device does not support cooperative launch"));
    // experiment overrides, read once per create (never per solve): AJM_STAGES / AJM_COL8_STAGES
    // (ring depth), AJM_CARVEOUT (%), AJM_NO_CLUSTER; the supported layout switches are create flags
    const int env_stages = getenv("AJM_STAGES") ? atoi(getenv("AJM_STAGES")) : 0;
    const int env_col8_stages = getenv("AJM_COL8_STAGES") ? atoi(getenv("AJM_COL8_STAGES")) : 0;
    const int env_carveout = getenv("AJM_CARVEOUT") ? atoi(getenv("AJM_CARVEOUT")) : -1;
    const bool env_no_cluster = getenv("AJM_NO_CLUSTER") != nullptr;

    // ---- the CSR arrays and b go to the device now; the copies overlap the host planning ----
    CC(dalloc(&h->rp, n + 1, st));
    CC(dalloc(&h->col, nnz + 8, st));
    CC(dalloc(&h->val, nnz + 8, st));
    CC(dalloc(&h->b_in, n, st));
    CC(cudaMemcpyAsync(h->rp, row_ptr, sizeof(int64_t) * (n + 1), kind_to_device(row_ptr), st));
    if (nnz > 0) {
        CC(cudaMemcpyAsync(h->col, col_idx, sizeof(int32_t) * nnz, kind_to_device(col_idx), st));
        CC(cudaMemcpyAsync(h->val, vals, sizeof(double) * nnz, kind_to_device(vals), st));
    }
    CC(cudaMemcpyAsync(h->b_in, b, sizeof(double) * n, kind_to_device(b), st));
    mark("h2d-issue", st);

    // host scan of row_ptr (needed anyway for the layout) while the copies above run; read in
    // place when it is host memory.  (The copies move exactly the nnz / n entries the caller
    // declared, so a row_ptr rejected here never made them read out of bounds.)
    const bool rp_dev = is_device_ptr(row_ptr);
    std::vector<int64_t> hrp_copy;
    const int64_t* hrp = row_ptr;
    if (rp_dev) {
        hrp_copy.resize((size_t)n + 1);
        CC(cudaMemcpyAsync(hrp_copy.data(), row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, st));
        CC(cudaStreamSynchronize(st));
        hrp = hrp_copy.data();
    }
    {
        int64_t bad = n;  // first row whose offsets decrease (n: none)
#pragma omp parallel for reduction(min : bad) schedule(static)
        for (int64_t i = 0; i < n; ++i)
            if (hrp[i + 1] < hrp[i] && i < bad) bad = i;
        if (bad < n) return bail(fail(h, AJM_ERR_CSR_INVALID, "row_ptr decreases at row %lld", (long long)bad));
    }
    mark("rowptr", st);

    // rows validated by a warp each (ajm_validate_long_kernel), caller's numbering
    constexpr int64_t kValidateLong = 2048;
    std::vector<int> vlong_h;
    // ---- row-length-binned layout (host, O(n log sigma)) ----
    auto rlen = [&](int64_t r) { return hrp[(size_t)r + 1] - hrp[(size_t)r]; };
    std::vector<int> perm_h, seg_row_h, seg_k0_h, seg_k1_h, seg_split_h, split_row_h, split_seg0_h;
    std::vector<int> inv_keep;  // (shards, relabelled) caller's local row -> internal row
    std::vector<int> row_cta;   // (shards) internal row -> the CTA that computes it
    std::vector<int4> grp_h;    // sub-warp groups: {rows}, {k0}, {k1} per group
    std::vector<long long> choff;
    std::vector<double> chcost;
    // fast path (stencil-like matrices): every row short and natural order pads < 5% -> SELL-32
    // in natural order, no relabelling, no segments; one pass over the row lengths
    // (host loops below are OpenMP-parallel where the result does not depend on the split)
    bool fast = false;
    {
        const int64_t nch = (n + 31) / 32;
        std::vector<long long> fo((size_t)nch + 1, 0);
        std::vector<double> fc((size_t)nch, 0.0);
        int64_t maxlen = 0;
#pragma omp parallel for schedule(static) reduction(max : maxlen)
        for (int64_t c = 0; c < nch; ++c) {
            int64_t w = 1;
            const int64_t r1 = std::min<int64_t>(n, c * 32 + 32);
            for (int64_t r = c * 32; r < r1; ++r) w = std::max<int64_t>(w, rlen(r));
            maxlen = std::max(maxlen, w);
            fo[(size_t)c + 1] = 32 * w;
            // a chunk costs its row operands plus one gather round trip per batch of 8 entries
            // (the natural-order cost model below)
            fc[(size_t)c] = 2600.0 * (double)((w + 7) / 8) + 56.0 * (double)(r1 - c * 32) + 64.0;
        }
        for (int64_t c = 0; c < nch; ++c) fo[(size_t)c + 1] += fo[(size_t)c];
        if (jbs && maxlen > AJM_SELL_MAX)
            return bail(fail(h, AJM_ERR_UNSUPPORTED, "AJM_D_JBLOCK needs every row to have <= %d nonzeros "
                                                       "(the longest has %lld)", AJM_SELL_MAX, (long long)maxlen));
        // block-diagonal J solves each block inside a warp: natural order whatever the padding
        if (maxlen <= AJM_SELL_MAX && (jbs || (double)fo.back() <= 1.05 * (double)std::max<int64_t>(nnz, 1))) {
            fast = true;
            h->long_rows = 0;
            h->sigma = 1;
            h->n_sell = n;
            h->nchunks = nch;
            h->relabel = false;
            choff.swap(fo);
            chcost.swap(fc);
            h->sell_elems = choff.back();
            split_seg0_h.push_back(0);
            h->nseg = h->nsplit = h->seg_rows = 0;
        }
        mark("L-fast", (cudaStream_t)-1);
    }
    if (!fast) {
        int64_t seg_len = AJM_SEG;  // nonzeros per warp segment (AJM_SEGLEN: tuning experiments)
        std::vector<int> short_rows, split_rows, whole_rows;
        short_rows.reserve((size_t)n);
        // dynamic segment queue when long rows carry >= 90% of the nonzeros (e.g. the §4.1 dense
        // SDD matrix: 1.2-1.3x faster); with a SELL majority (config 4) the static LPT plan is
        // faster (873 vs 964 us/pass).  AJM_DYNSEG overrides.
        {
            int64_t long_nnz = 0;
#pragma omp parallel for schedule(static) reduction(+ : long_nnz)
            for (int64_t i = 0; i < n; ++i)
                if (rlen(i) > AJM_SELL_MAX) long_nnz += rlen(i);
            h->dynseg = (double)long_nnz >= 0.9 * (double)std::max<int64_t>(nnz, 1) ? 1 : 0;
            if (flags & AJM_SEGMENTS_STATIC) h->dynseg = 0;
            if (flags & AJM_SEGMENTS_DYNAMIC) h->dynseg = 1;
        }
        {
            // per-thread bins over contiguous row ranges, concatenated in thread order (so every
            // list stays in ascending row order, as a serial pass would give)
            std::vector<std::vector<int>> tb[4];
            int nt = 1;
#pragma omp parallel
            {
#pragma omp single
                {
                    nt = omp_get_num_threads();
                    for (auto& v : tb) v.resize((size_t)nt);
                }
                const int tid = omp_get_thread_num();
                const int64_t lo = n * tid / nt, hi = n * (tid + 1) / nt;
                for (int64_t i = lo; i < hi; ++i) {
                    const int64_t len = rlen(i);
                    if (len <= AJM_SELL_MAX) tb[0][(size_t)tid].push_back((int)i);
                    else if (len <= seg_len) tb[1][(size_t)tid].push_back((int)i);
                    else tb[2][(size_t)tid].push_back((int)i);
                    if (len > kValidateLong) tb[3][(size_t)tid].push_back((int)i);
                }
            }
            std::vector<int>* dst[4] = {&short_rows, &whole_rows, &split_rows, &vlong_h};
            for (int q = 0; q < 4; ++q)
                for (auto& v : tb[q]) dst[q]->insert(dst[q]->end(), v.begin(), v.end());
        }
        h->long_rows = (int64_t)split_rows.size();
        // the SELL path indexes with 64-bit offsets; warp segments keep int32 CSR offsets
        if (nnz >= ((int64_t)1 << 31) && !(split_rows.empty() && whole_rows.empty()))
            return bail(fail(h, AJM_ERR_UNSUPPORTED, "nnz >= 2^31 needs every row to have <= %d nonzeros",
                             AJM_SELL_MAX));
        mark("L-bins", (cudaStream_t)-1);
        auto padded = [&](const std::vector<int>& order) {
            int64_t tot = 0;
            const int64_t nc = ((int64_t)order.size() + 31) / 32;
#pragma omp parallel for schedule(static) reduction(+ : tot)
            for (int64_t c = 0; c < nc; ++c) {
                int64_t w = 1;
                for (size_t j = (size_t)c * 32; j < std::min(order.size(), (size_t)c * 32 + 32); ++j)
                    w = std::max<int64_t>(w, rlen(order[j]));
                tot += 32 * w;
            }
            return tot;
        };
        int64_t short_nnz = 0;
        const int64_t nshort = (int64_t)short_rows.size();
#pragma omp parallel for schedule(static) reduction(+ : short_nnz)
        for (int64_t j = 0; j < nshort; ++j) short_nnz += rlen(short_rows[(size_t)j]);
        std::vector<int> order = short_rows;
        h->sigma = 1;
        if (!short_rows.empty() && (double)padded(order) > 1.05 * (double)std::max<int64_t>(short_nnz, 1)) {
            // sort by decreasing length inside windows of 4096 consecutive row indices (stable)
            // (a stable counting sort: row lengths are <= AJM_SELL_MAX here)
            h->sigma = 4096;
            std::vector<size_t> wlo;  // window boundaries in `order` (ascending row index)
            for (int64_t wb = 0; wb * h->sigma < n; ++wb) {
                const size_t lo = (size_t)(std::lower_bound(order.begin(), order.end(), (int)(wb * h->sigma)) - order.begin());
                if (lo < order.size() && (wlo.empty() || lo > wlo.back())) wlo.push_back(lo);
            }
            wlo.push_back(order.size());
            const int64_t nwin = (int64_t)wlo.size() - 1;
#pragma omp parallel
            {
                std::vector<int> tmp;
#pragma omp for schedule(static)
                for (int64_t wi = 0; wi < nwin; ++wi) {
                    const size_t lo = wlo[(size_t)wi], hi = wlo[(size_t)wi + 1];
                    int cnt[AJM_SELL_MAX + 2] = {0};
                    for (size_t j = lo; j < hi; ++j) ++cnt[AJM_SELL_MAX - rlen(order[j]) + 1];
                    for (int b2 = 1; b2 <= AJM_SELL_MAX + 1; ++b2) cnt[b2] += cnt[b2 - 1];
                    tmp.resize(hi - lo);
                    for (size_t j = lo; j < hi; ++j) tmp[(size_t)cnt[AJM_SELL_MAX - rlen(order[j])]++] = order[j];
                    std::copy(tmp.begin(), tmp.end(), order.begin() + (long)lo);
                }
            }
        }
        mark("L-sort", (cudaStream_t)-1);
        h->n_sell = (int64_t)order.size();
        h->nchunks = (h->n_sell + 31) / 32;
        // Relabelling: the solver works in "internal" row numbering -- SELL rows in
        // slot order, then the segment rows (split rows first) -- so every row operand of a SELL
        // chunk is contiguous (coalesced / TMA-stageable) whatever the sorting window.  Values
        // and the order of each row's entries are unchanged (the row sums are the same).
        h->relabel = !(h->sigma == 1 && split_rows.empty() && whole_rows.empty());
        perm_h.assign((size_t)n, 0);
        const int64_t nord = (int64_t)order.size();
#pragma omp parallel for schedule(static)
        for (int64_t j = 0; j < nord; ++j) perm_h[(size_t)j] = order[(size_t)j];
        {
            size_t k = order.size();
            for (int r : split_rows) perm_h[k++] = r;
            for (int r : whole_rows) perm_h[k++] = r;
        }
        std::vector<int> inv_h;
        if (h->relabel) {
            inv_h.assign((size_t)n, 0);
#pragma omp parallel for schedule(static)
            for (int64_t k = 0; k < n; ++k) inv_h[(size_t)perm_h[(size_t)k]] = (int)k;
        }
        auto irow = [&](int r) { return h->relabel ? inv_h[(size_t)r] : r; };
        mark("L-perm", (cudaStream_t)-1);
        choff.assign((size_t)h->nchunks + 1, 0);
        chcost.assign((size_t)h->nchunks, 0.0);
        const int64_t nchk_h = h->nchunks, nsell_h = h->n_sell;
        // A wide chunk fills a staging unit alone (<= 2048 entries), so a ring of S stages keeps
        // only S * floor(64 / w) of the CTA's 8 warps busy: weight such chunks by the idle share
        // (config 4: the first sorted windows hold the 40-64-wide rows, and the CTAs planned on
        // them finished ~90 us after the median)
        const double par_stages = h->relabel ? 3.0 : 4.0;
        // softened to (8 / busy)^0.5: config 4 495 -> 444 us/pass, config 3 79.1 -> 79.7 (exponent
        // 1: 452 / 81.0; 0.7: 440 / 80.3; the idle-share weight on one-chunk units only: 452 / 79.1)
        const double par_alpha = 0.5;
#pragma omp parallel for schedule(static)
        for (int64_t c = 0; c < nchk_h; ++c) {
            int64_t w = 1, rows = 0;
            for (int64_t j = c * 32; j < std::min<int64_t>(nsell_h, c * 32 + 32); ++j) {
                w = std::max<int64_t>(w, rlen(order[(size_t)j]));
                ++rows;
            }
            choff[(size_t)c + 1] = 32 * w;
            const double busy = std::min<double>(AJM_WARPS, par_stages * std::max<int64_t>(1, AJM_UNIT_EL / (32 * w)));
            // natural-order layouts (stencils): a chunk costs its row operands plus one gather round
            // trip per batch of 8 entries -- measured per chunk (config 2, pair-coded): 6-wide
            // boundary chunks take as long as 7-wide ones (0.12 us per chunk and CTA; the byte model
            // gave the boundary CTAs 242 chunks instead of 221 and they finished last), and on config
            // 5 an 18-wide chunk (3 batches) takes 0.78 of a 27-wide one (4 batches)
            const double body = h->relabel ? 12.0 * 32 * w : 2600.0 * (double)((w + 7) / 8);
            chcost[(size_t)c] = (body + 56.0 * rows + 64.0) * std::pow((double)AJM_WARPS / busy, par_alpha);
        }
        for (int64_t c = 0; c < nchk_h; ++c) choff[(size_t)c + 1] += choff[(size_t)c];
        h->sell_elems = choff.back();
        mark("L-chunks", (cudaStream_t)-1);
        // segments: split rows first (consecutive per row), then whole rows
        for (int r : split_rows) {
            const int sidx = (int)split_row_h.size();
            split_row_h.push_back(irow(r));
            split_seg0_h.push_back((int)seg_row_h.size());
            for (int64_t k = hrp[(size_t)r]; k < hrp[(size_t)r + 1]; k += seg_len) {
                seg_row_h.push_back(irow(r));
                seg_k0_h.push_back((int)k);
                seg_k1_h.push_back((int)std::min<int64_t>(k + seg_len, hrp[(size_t)r + 1]));
                seg_split_h.push_back(sidx);
            }
        }
        if (!h->dynseg) split_seg0_h.push_back((int)seg_row_h.size());
        // sub-warp groups (static plan): rows of 65 .. AJM_GRP_MAX nonzeros four to a warp, 8 lanes
        // per row, so four rows' latency chains (operands, gathers, epilogue) overlap in one warp
        // (north_star "one warp or sub-warp per row, chosen by row-length histogram")
        std::vector<int> grp_members;
        const bool use_groups = !h->dynseg && !getenv("AJM_NO_GROUPS");
        for (int r : whole_rows) {
            if (use_groups && rlen(r) <= AJM_GRP_MAX) {
                grp_members.push_back(r);
                continue;
            }
            // dynamic segments: every segment row is finished by a fixed owner CTA (one segment)
            const int sidx = h->dynseg ? (int)split_row_h.size() : -1;
            if (h->dynseg) {
                split_row_h.push_back(irow(r));
                split_seg0_h.push_back((int)seg_row_h.size());
            }
            seg_row_h.push_back(irow(r));
            seg_k0_h.push_back((int)hrp[(size_t)r]);
            seg_k1_h.push_back((int)hrp[(size_t)r + 1]);
            seg_split_h.push_back(sidx);
        }
        if (h->dynseg) split_seg0_h.push_back((int)seg_row_h.size());
        if (!grp_members.empty()) {
            // longest first, so the rows of a group have similar lengths (balanced 8-lane groups)
            std::stable_sort(grp_members.begin(), grp_members.end(), [&](int x, int y) { return rlen(x) > rlen(y); });
            const int64_t ng = ((int64_t)grp_members.size() + AJM_GRP_ROWS - 1) / AJM_GRP_ROWS;
            grp_h.assign((size_t)ng * 3, make_int4(-1, -1, -1, -1));
            for (int64_t g = 0; g < ng; ++g) {
                int rr[4] = {-1, -1, -1, -1}, k0[4] = {0, 0, 0, 0}, k1[4] = {0, 0, 0, 0};
                int64_t tot = 0;
                for (int q = 0; q < AJM_GRP_ROWS; ++q) {
                    const int64_t m = g * AJM_GRP_ROWS + q;
                    if (m >= (int64_t)grp_members.size()) break;
                    const int r = grp_members[(size_t)m];
                    rr[q] = irow(r);
                    k0[q] = (int)hrp[(size_t)r];
                    k1[q] = (int)hrp[(size_t)r + 1];
                    tot += rlen(r);
                }
                grp_h[(size_t)g * 3 + 0] = make_int4(rr[0], rr[1], rr[2], rr[3]);
                grp_h[(size_t)g * 3 + 1] = make_int4(k0[0], k0[1], k0[2], k0[3]);
                grp_h[(size_t)g * 3 + 2] = make_int4(k1[0], k1[1], k1[2], k1[3]);
                seg_row_h.push_back((int)g);  // a group item: {group id, 0, its nonzeros, -2}
                seg_k0_h.push_back(0);
                seg_k1_h.push_back((int)tot);
                seg_split_h.push_back(-2);
            }
            h->ngrp = ng;
            h->grp_rows = (int64_t)grp_members.size();
        }
        h->nseg = (int64_t)seg_row_h.size();
        for (int64_t k = 0; k < h->nseg; ++k) h->seg_nnz += seg_k1_h[(size_t)k] - seg_k0_h[(size_t)k];
        h->nsplit = (int64_t)split_row_h.size();
        h->seg_rows = (int64_t)(split_rows.size() + whole_rows.size());
        if (h->relabel) {
            CC(dalloc(&h->perm_fwd, n, st));
            CC(dalloc(&h->perm_inv, n, st));
            CC(cudaMemcpyAsync(h->perm_fwd, perm_h.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st));
            CC(cudaMemcpyAsync(h->perm_inv, inv_h.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st));
            CC(cudaStreamSynchronize(st));
            if (sh) inv_keep.swap(inv_h);
        }
    }
    mark("layout", st);
    // ---- TMA staging units, persistent grid, cost-balanced CTA ranges ----
    std::vector<int> unit_c0_h, cta_seg_h, cta_unit_h, cta_split_h, owner_split_h, seg_list_h, seg_order_h, seg_grp_h;
    if (h->dynseg) {  // claim order of the dynamic segment queue: longest first (LPT-like)
        seg_order_h.resize((size_t)h->nseg);
        for (int64_t k = 0; k < h->nseg; ++k) seg_order_h[(size_t)k] = (int)k;
        std::stable_sort(seg_order_h.begin(), seg_order_h.end(), [&](int x, int y) {
            return seg_k1_h[(size_t)x] - seg_k0_h[(size_t)x] > seg_k1_h[(size_t)y] - seg_k0_h[(size_t)y];
        });
        // claim groups: consecutive segments of the order with >= seg_group_nnz nonzeros (<= 16
        // segments), so the queue costs one atomic per ~1k nonzeros, not per short row
        int64_t gnnz = 1024;
        int64_t acc = 0, cntg = 0;
        seg_grp_h.push_back(0);
        for (int64_t k = 0; k < h->nseg; ++k) {
            const int sg = seg_order_h[(size_t)k];
            acc += seg_k1_h[(size_t)sg] - seg_k0_h[(size_t)sg];
            ++cntg;
            if (acc >= gnnz || cntg >= 16 || k + 1 == h->nseg) {
                seg_grp_h.push_back((int)(k + 1));
                acc = cntg = 0;
            }
        }
        h->nsegq = (int64_t)seg_grp_h.size() - 1;
    }
    {
        // one item sequence: segments (split rows first), then SELL chunks; contiguous CTA ranges
        // balanced by cost at chunk granularity; each CTA's chunks are then grouped into TMA
        // staging units of <= AJM_WARPS chunks and <= AJM_UNIT_EL elements
        const int64_t nitems = h->nseg + h->nchunks;
        std::vector<double> cost;
        cost.reserve((size_t)nitems);
        // segments are latency-bound (one warp, direct loads): weight their bytes twice
        const double segw = 24.0, segc = 568.0;
        for (int64_t s2 = 0; s2 < h->nseg; ++s2)  // (dynamic segments are outside the static plan)
            cost.push_back(h->dynseg ? 0.0 : segw * (seg_k1_h[(size_t)s2] - seg_k0_h[(size_t)s2]) + segc);
        for (int64_t c2 = 0; c2 < h->nchunks; ++c2) cost.push_back(chcost[(size_t)c2]);
        double total = 0.0;
        for (double x : cost) total += x;
        mark("P-cost", (cudaStream_t)-1);
        // LPT order of the segments (largest cost first, index order among equals): independent
        // of the grid size, so computed once for every plan() call below
        std::vector<int64_t> lpt_order;
        if (!h->dynseg) {
            // the cost is increasing in the segment length: a counting sort by length
            int64_t seg_len_max = 0;
            for (int64_t k = 0; k < h->nseg; ++k) seg_len_max = std::max<int64_t>(seg_len_max, seg_k1_h[(size_t)k] - seg_k0_h[(size_t)k]);
            lpt_order.resize((size_t)h->nseg);
            std::vector<int64_t> cnt((size_t)seg_len_max + 2, 0);
            for (int64_t k = 0; k < h->nseg; ++k) ++cnt[(size_t)(seg_len_max - (seg_k1_h[(size_t)k] - seg_k0_h[(size_t)k]) + 1)];
            for (size_t q = 1; q < cnt.size(); ++q) cnt[q] += cnt[q - 1];
            for (int64_t k = 0; k < h->nseg; ++k)
                lpt_order[(size_t)cnt[(size_t)(seg_len_max - (seg_k1_h[(size_t)k] - seg_k0_h[(size_t)k]))]++] = k;
        }
        mark("P-lptsort", (cudaStream_t)-1);
        auto plan = [&](int G) {
            // (a) segments: largest first onto the least-loaded CTA (LPT), so the latency-bound
            //     long rows spread over every SM; (b) SELL chunks: contiguous ranges topping every
            //     CTA up to the same cumulative cost
            const double target = total / (double)G;
            std::vector<double> segload((size_t)G, 0.0);
            std::vector<std::vector<int>> segs((size_t)G);
            if (!h->dynseg) {
                // least-loaded CTA first, lower index among equal loads; the costs are integers,
                // so (load << 10 | cta) orders exactly like (load, cta) in one 64-bit key
                std::vector<uint64_t> heap;
                for (int cc = 0; cc < G; ++cc) heap.push_back((uint64_t)cc);
                std::make_heap(heap.begin(), heap.end(), std::greater<uint64_t>());
                for (int64_t k : lpt_order) {
                    std::pop_heap(heap.begin(), heap.end(), std::greater<uint64_t>());
                    const int cc = (int)(heap.back() & 1023u);
                    segload[(size_t)cc] += cost[(size_t)k];
                    heap.back() = ((uint64_t)segload[(size_t)cc] << 10) | (uint64_t)cc;
                    segs[(size_t)cc].push_back((int)k);
                    std::push_heap(heap.begin(), heap.end(), std::greater<uint64_t>());
                }
            }
            mark("p-lpt", (cudaStream_t)-1);
            seg_list_h.clear();
            cta_seg_h.assign((size_t)G + 1, 0);
            for (int cc = 0; cc < G; ++cc) {
                // split-row segments first (their owners wait for them), then longest first
                // (round robin over the warps; config 4: 500.6 -> 496.1 us/pass vs segment order);
                // LPT handed them out longest first already, so a stable partition suffices
                std::stable_partition(segs[(size_t)cc].begin(), segs[(size_t)cc].end(),
                                      [&](int x) { return seg_split_h[(size_t)x] >= 0; });
                cta_seg_h[(size_t)cc] = (int)seg_list_h.size();
                for (int k : segs[(size_t)cc]) seg_list_h.push_back(k);
            }
            cta_seg_h[(size_t)G] = (int)seg_list_h.size();
            mark("p-segsort", (cudaStream_t)-1);
            std::vector<int64_t> cstart((size_t)G + 1, h->nchunks);
            int64_t i = 0;
            double pref = 0.0, cumseg = 0.0;
            // a small grid with a chunk per consumer warp (the single-cluster kernels): exactly
            // AJM_WARPS consecutive chunks per CTA -- the pass lasts as long as its slowest warp
            const bool one_per_warp = h->nseg == 0 && G <= 16 && (int64_t)G * AJM_WARPS >= h->nchunks;
            for (int cc = 0; cc < G; ++cc) {
                if (one_per_warp) {
                    cstart[(size_t)cc] = std::min<int64_t>((int64_t)cc * AJM_WARPS, h->nchunks);
                    continue;
                }
                cstart[(size_t)cc] = i;
                cumseg += segload[(size_t)cc];
                if (cc == G - 1) break;
                const double lim = target * (double)(cc + 1) - cumseg;
                while (i < h->nchunks && pref + 0.5 * cost[(size_t)(h->nseg + i)] < lim) pref += cost[(size_t)(h->nseg + i++)];
            }
            cstart[(size_t)G] = h->nchunks;
            cta_unit_h.assign((size_t)G + 1, 0);
            unit_c0_h.clear();
            int mu = 1, mc = 1;
            for (int cc = 0; cc < G; ++cc) {
                cta_unit_h[(size_t)cc] = (int)unit_c0_h.size();
                const int64_t c0 = cstart[(size_t)cc], c1 = cstart[(size_t)cc + 1];
                int64_t c2 = c0;
                while (c2 < c1) {
                    const int64_t ub = c2;
                    unit_c0_h.push_back((int)ub);
                    int64_t k = 0;
                    while (c2 < c1 && k < AJM_WARPS && choff[(size_t)c2 + 1] - choff[(size_t)ub] <= AJM_UNIT_EL) {
                        ++c2;
                        ++k;
                    }
                }
                mu = std::max(mu, (int)(unit_c0_h.size() - cta_unit_h[(size_t)cc]) + 1);
                mc = std::max(mc, (int)(c1 - c0) + 1);
            }
            cta_unit_h[(size_t)G] = (int)unit_c0_h.size();
            unit_c0_h.push_back((int)h->nchunks);
            h->nunits = (int64_t)unit_c0_h.size() - 1;
            h->meta_units = (mu + 3) & ~3;
            h->meta_chunks = (mc + 3) & ~3;
        };
        const double avg_w = h->nchunks ? (double)h->sell_elems / (32.0 * (double)h->nchunks) : 0.0;
        h->wide_rows = avg_w >= 16.0;
        int ring_stages = 4;
        if (h->jbs) {  // block-diagonal J: its own instantiation (natural order, no segments)
            h->fn = jblock_fn(h->jbs, false);
        } else {
            // without long rows the instantiation without the segment phases (its ring loop has more
            // registers to spare: config 2 47.5 -> 45.5 us/pass, config 3 81.5 -> 76.2).  Ring depth:
            // 3 stages and the L1 they free win where the gathers are scattered (sorted-window graph
            // layouts: config 3 135 -> 82, config 4 880 -> 535 us/pass) and on narrow natural-order
            // rows (config 2 int32: 45.7 -> 44.7); natural-order wide rows (units of 2-3 chunks) keep
            // 4 (config 5 int32: 1189 vs 1350 at 3)
            h->seg_fn = h->nseg > 0;
            h->ring_fn = true;
            ring_stages = (!h->relabel && avg_w >= 16.0) ? 4 : 3;
            if (env_stages) ring_stages = std::min(4, std::max(2, env_stages));
            h->fn = ring_fn(h->seg_fn, ring_stages);
        }
        h->ring_stages = ring_stages;
        size_t ring = (size_t)ring_stages * AJM_UNIT_EL * 12;  // val/col of a unit per stage
        size_t meta = 4096;  // initial allowance, grown until the plan fits
        int smem_optin = 0;
        CC(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
        mark("P-pre", (cudaStream_t)-1);
        int planned_grid = -1;
        for (int iter = 0;; ++iter) {
            // tables too large for shared memory next to the ring: read them from global memory
            if (!h->gmeta && !h->jbs && (ring + meta + 2048 > (size_t)smem_optin || (flags & AJM_GLOBAL_TABLES))) {
                if (sh) return bail(fail(h, AJM_ERR_UNSUPPORTED, "shard layout tables do not fit shared memory"));
                h->gmeta = 1;
                h->fn = gmeta_fn(h->nseg > 0);
                h->ring_fn = false;
                h->ring_stages = 4;
                ring = (size_t)4 * AJM_UNIT_EL * 12;
            }
            h->dyn_smem = ring + (h->gmeta ? 0 : meta);
            h->meta_bytes = h->gmeta ? 0 : meta;
            int occ = 0;
            cudaError_t eo;
            {
                std::lock_guard<std::mutex> lock(g_attr_mu);
                eo = fn_occupancy(h->fn, h->dyn_smem, 100, &occ, block_threads(h->nseg > 0));
            }
            CC(eo);
            if (occ < 1) return bail(fail(h, AJM_ERR_UNSUPPORTED, "solver kernel cannot be resident (%zu B smem)", h->dyn_smem));
            h->ctas_per_sm = occ;
            const int64_t g = (int64_t)h->sm_count * occ;
            h->grid = (int)std::max<int64_t>(1, std::min<int64_t>(g, nitems));
            // an emulated group shares the device: every rank takes the same 1/nranks of the
            // resident CTAs (one launch runs them all)
            if (sh && sh->colocated) h->grid = (int)std::max<int64_t>(1, g / sh->nranks);
            // <= 128 work items: one item per consumer warp on <= 16 CTAs, launched below as a
            // single cluster whose barrier lives in distributed shared memory
            if (!sh && nitems <= 16 * AJM_WARPS && !env_no_cluster)
                h->grid = (int)std::max<int64_t>(1, (nitems + AJM_WARPS - 1) / AJM_WARPS);
            if (h->grid != planned_grid) {  // plan() depends on the grid size only
                plan(h->grid);
                planned_grid = h->grid;
            }
            const size_t need = (size_t)(h->meta_units + h->meta_chunks) * sizeof(int);
            if (h->gmeta || need <= meta) break;
            if (iter > 6) return bail(fail(h, AJM_ERR_UNSUPPORTED, "layout metadata does not fit shared memory"));
            meta = need;
        }
        mark("P-loop", (cudaStream_t)-1);
        const int G = h->grid;
        // small problems: the grid as ONE thread-block cluster, barrier and partial exchange in
        // distributed shared memory (AJM_NO_CLUSTER disables, for experiments)
        if (!sh && G <= 16 && !env_no_cluster && (h->jbs || h->ring_fn)) {
            const SolveFn cf = h->jbs ? jblock_fn(h->jbs, true) : cluster_fn(h->seg_fn);
            // (the cluster kernels keep a 4-deep ring: per-pass latency, not L1, bounds them)
            const size_t cdyn = h->ring_fn ? (size_t)4 * AJM_UNIT_EL * 12 + h->meta_bytes : h->dyn_smem;
            std::lock_guard<std::mutex> lock(g_attr_mu);
            cudaFuncSetAttribute((const void*)cf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cdyn);
            cudaFuncSetAttribute((const void*)cf, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
            if (G > 8) cudaFuncSetAttribute((const void*)cf, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            cudaLaunchConfig_t qc = {};
            qc.gridDim = dim3(G);
            qc.blockDim = dim3(block_threads(h->nseg > 0));
            qc.dynamicSmemBytes = cdyn;
            cudaLaunchAttribute qa[1];
            qa[0].id = cudaLaunchAttributeClusterDimension;
            qa[0].val.clusterDim.x = (unsigned)G;
            qa[0].val.clusterDim.y = 1;
            qa[0].val.clusterDim.z = 1;
            qc.attrs = qa;
            qc.numAttrs = 1;
            int ncl = 0;
            if (cudaOccupancyMaxActiveClusters(&ncl, (const void*)cf, &qc) == cudaSuccess && ncl >= 1) {
                h->fn = cf;
                h->cluster = 1;
                h->dyn_smem = cdyn;
                if (h->ring_fn) h->ring_stages = 4;
                h->ring_fn = false;
            }
            cudaGetLastError();
        }
        h->lz_dyn_smem = h->dyn_smem;
        // natural-order SELL rows only, diagonal D: the whole solve resident in the cluster
        // (ajm_resident_kernel: matrix slices and an x~ replica in shared memory, row state in
        // registers); AJM_NO_RESIDENT=1 keeps the kCluster ring kernel (experiments)
        if (h->cluster && !h->relabel && h->nseg == 0 && !h->jbs && !getenv("AJM_NO_RESIDENT")) {
            int64_t max_el = 0;
            int max_chk = 0;  // the kernel runs one chunk per warp: every CTA needs <= AJM_WARPS
            for (int cc = 0; cc < G; ++cc) {
                const int ua = cta_unit_h[(size_t)cc], ub = cta_unit_h[(size_t)cc + 1];
                if (ub > ua) {
                    max_el = std::max<int64_t>(max_el, choff[(size_t)unit_c0_h[(size_t)ub]] - choff[(size_t)unit_c0_h[(size_t)ua]]);
                    max_chk = std::max(max_chk, unit_c0_h[(size_t)ub] - unit_c0_h[(size_t)ua]);
                }
            }
            const size_t rdyn = (size_t)2 * 8 * (size_t)((n + 31) / 32 * 32) + (size_t)max_el * 12 + 64;
            const SolveFn rf = ajm_resident_kernel;
            std::lock_guard<std::mutex> lock(g_attr_mu);
            if (rdyn <= (size_t)smem_optin && max_chk <= AJM_WARPS &&
                cudaFuncSetAttribute((const void*)rf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rdyn) == cudaSuccess) {
                if (G > 8) cudaFuncSetAttribute((const void*)rf, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                cudaLaunchConfig_t qc = {};
                qc.gridDim = dim3(G);
                qc.blockDim = dim3(AJM_BLOCK);
                qc.dynamicSmemBytes = rdyn;
                cudaLaunchAttribute qa[1];
                qa[0].id = cudaLaunchAttributeClusterDimension;
                qa[0].val.clusterDim.x = (unsigned)G;
                qa[0].val.clusterDim.y = 1;
                qa[0].val.clusterDim.z = 1;
                qc.attrs = qa;
                qc.numAttrs = 1;
                int ncl = 0;
                if (cudaOccupancyMaxActiveClusters(&ncl, (const void*)rf, &qc) == cudaSuccess && ncl >= 1) {
                    h->fn = rf;
                    h->resident = 1;
                    h->dyn_smem = rdyn;
                }
            }
            cudaGetLastError();
        }
        if (getenv("AJM_TS_ALL")) {
            h->cta_nchk.assign((size_t)G, 0);
            for (int cc = 0; cc < G; ++cc)
                h->cta_nchk[(size_t)cc] = unit_c0_h[(size_t)cta_unit_h[(size_t)cc + 1]] - unit_c0_h[(size_t)cta_unit_h[(size_t)cc]];
        }
        mark("P-cluster", (cudaStream_t)-1);
        // owner of a split row = the CTA that runs its last segment
        std::vector<int> seg_cta((size_t)h->nseg, 0);
        for (int cc = 0; cc < G; ++cc)
            for (int k2 = cta_seg_h[(size_t)cc]; k2 < cta_seg_h[(size_t)cc + 1]; ++k2) seg_cta[(size_t)seg_list_h[(size_t)k2]] = cc;
        std::vector<std::vector<int>> per((size_t)G);
        for (int64_t sp = 0; sp < h->nsplit; ++sp) {
            // static: the CTA that runs the row's last segment; dynamic: contiguous equal shares
            const int own = h->dynseg ? (int)(sp * G / std::max<int64_t>(h->nsplit, 1))
                                      : seg_cta[(size_t)split_seg0_h[(size_t)sp + 1] - 1];
            per[(size_t)own].push_back((int)sp);
        }
        cta_split_h.assign((size_t)G + 1, 0);
        for (int cc = 0; cc < G; ++cc) {
            cta_split_h[(size_t)cc + 1] = cta_split_h[(size_t)cc] + (int)per[(size_t)cc].size();
            for (int sp : per[(size_t)cc]) owner_split_h.push_back(sp);
        }
        if (sh) {  // which CTA writes each row's x~^{t+1} (and so pushes its halo entries)
            row_cta.assign((size_t)n, 0);
            for (int cc = 0; cc < G; ++cc) {
                const int u0 = cta_unit_h[(size_t)cc], u1 = cta_unit_h[(size_t)cc + 1];
                if (u1 <= u0) continue;
                const int64_t r0 = (int64_t)unit_c0_h[(size_t)u0] * 32;
                const int64_t r1 = std::min<int64_t>(h->n_sell, (int64_t)unit_c0_h[(size_t)u1] * 32);
                for (int64_t r = r0; r < r1; ++r) row_cta[(size_t)r] = cc;
            }
            for (int64_t k = 0; k < h->nseg; ++k) {
                if (seg_split_h[(size_t)k] == -1) row_cta[(size_t)seg_row_h[(size_t)k]] = seg_cta[(size_t)k];
                if (seg_split_h[(size_t)k] == -2) {
                    const int4 gr = grp_h[(size_t)seg_row_h[(size_t)k] * 3];
                    for (int r2 : {gr.x, gr.y, gr.z, gr.w})
                        if (r2 >= 0) row_cta[(size_t)r2] = seg_cta[(size_t)k];
                }
            }
            for (int cc = 0; cc < G; ++cc)
                for (int sp : per[(size_t)cc]) row_cta[(size_t)split_row_h[(size_t)sp]] = cc;
        }
    }

    mark("plan", st);
    // ---- device allocations ----
    // the six n-vectors in ONE allocation [X0 X1 X2 Qxp b D] (each padded to whole SELL chunks,
    // 256-byte aligned): the L2 persistence window below covers them with a single range
    h->n_pad = (std::max<int64_t>(n, h->nchunks * 32) + 31) / 32 * 32;
    size_t vec_elems = (size_t)6 * h->n_pad;
    if (sh) {
        // a shard's iterate buffers carry its halo around the own rows: X_k = base + lo_pad, the
        // lower halo at X_k[-H_lo .. -1], the upper at X_k[n .. n + H_hi - 1]; cudaMalloc (not the
        // pool) so the allocation can be exported through CUDA IPC to the other ranks' processes
        h->lo_pad = (h->h_lo + 31) / 32 * 32;
        h->xstride = h->lo_pad + h->n_pad + (h->h_hi + 31) / 32 * 32;
        vec_elems = (size_t)3 * h->xstride + (size_t)3 * h->n_pad;
        CC(cudaMalloc((void**)&h->vecs, sizeof(double) * vec_elems));
        for (int k = 0; k < 3; ++k) h->X[k] = h->vecs + (size_t)k * h->xstride + h->lo_pad;
        double* rest = h->vecs + (size_t)3 * h->xstride;
        h->Qxp = rest;
        h->b = rest + (size_t)h->n_pad;
        h->D = rest + (size_t)2 * h->n_pad;
        CC(cudaMalloc((void**)&h->xch, sizeof(double) * (2 * AJM_MAX_RANKS * AJM_NPART + 1)));
        CC(cudaMemsetAsync(h->xch, 0, sizeof(double) * (2 * AJM_MAX_RANKS * AJM_NPART + 1), st));
    } else {
        CC(dalloc(&h->vecs, vec_elems, st));
        for (int k = 0; k < 3; ++k) h->X[k] = h->vecs + (size_t)k * h->n_pad;
        h->Qxp = h->vecs + (size_t)3 * h->n_pad;
        h->b = h->vecs + (size_t)4 * h->n_pad;
        h->D = h->vecs + (size_t)5 * h->n_pad;
    }
    CC(cudaMemsetAsync(h->vecs, 0, sizeof(double) * vec_elems, st));
    // L2 residency: keep as much of the iterate vectors as the device allows in a
    // persisting L2 carve-out; the matrix stream goes through with evict_first hints
    h->win_bytes = 0;
    int l2size = 0;
    CC(cudaDeviceGetAttribute(&l2size, cudaDevAttrL2CacheSize, h->device));
    const size_t vec_bytes = sizeof(double) * vec_elems;
    // vectors larger than the whole L2 (configs 4, 5): a persisting carve-out only takes L2 away
    // from everything else (measured 1138 -> 919 us/pass on config 4): eviction hints only
    if (vec_bytes > (size_t)l2size) {
        h->l2persist = 0;
        h->l2_mode = 3;
    }
    if (getenv("AJM_NO_PERSIST")) h->l2persist = 0;  // (experiments)
    if (h->l2persist) {
        int maxp = 0, maxw = 0;
        CC(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, h->device));
        CC(cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, h->device));
        if (maxp > 0 && maxw > 0) {
            const size_t persist = std::min<size_t>((size_t)maxp, vec_bytes);
            size_t cur = 0;
            cudaError_t el;
            {   // raise the device limit; the first holder remembers the value to restore at destroy
                std::lock_guard<std::mutex> lock(g_attr_mu);
                PersistState& ps = g_persist[h->device];
                el = cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
                if (el == cudaSuccess && ps.holders == 0) ps.saved_limit = cur;
                if (el == cudaSuccess && cur < persist) el = cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist);
                if (el == cudaSuccess) el = cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
                if (el == cudaSuccess) {
                    ps.holders += 1;
                    h->persist_holder = true;
                }
            }
            CC(el);
            // mode 2: all six vectors in the window (they fit 3/4 of the carve-out: config 3);
            // mode 3: only the three rotating iterate buffers X0..X2 (the gathered x~ lives there),
            // b, D, Qx streamed with evict_first
            h->l2_mode = (double)vec_bytes <= 0.75 * (double)maxp ? 2 : 3;
            const size_t wb = h->l2_mode == 3 ? sizeof(double) * 3 * (size_t)(h->shard ? h->xstride : h->n_pad) : vec_bytes;
            h->win_bytes = std::min<size_t>(wb, (size_t)maxw);
            h->win_hit = (float)std::min(1.0, (double)cur / (double)h->win_bytes);
            // mode 3 on vectors that fit the L2 (config 2): before each solve one touch pass over
            // all six vectors under a window covering them (the carve-out's share persists), then
            // the solver's own window keeps the x~ buffers at hit ratio 1 (55.3 -> 47.0 us/pass)
            if (h->l2_mode == 3 && vec_bytes <= (size_t)l2size) {
                h->prime_bytes = std::min<size_t>(vec_bytes, (size_t)maxw);
                h->prime_hit = (float)std::min(1.0, (double)cur / (double)h->prime_bytes);
            }
        }
    }
    CC(dalloc(&h->sval, h->sell_elems, st));
    CC(dalloc(&h->scol, h->sell_elems, st));
    CC(dalloc(&h->chunk_off, h->nchunks + 1, st));
    CC(dalloc(&h->seg_row, h->nseg, st));
    CC(dalloc(&h->seg_k0, h->nseg, st));
    CC(dalloc(&h->seg_k1, h->nseg, st));
    CC(dalloc(&h->seg_split, h->nseg, st));
    CC(dalloc(&h->seg_part, h->nseg, st));
    CC(dalloc(&h->split_row, h->nsplit, st));
    CC(dalloc(&h->split_seg0, h->nsplit + 1, st));
    CC(dalloc(&h->split_cnt, h->nsplit, st));
    CC(dalloc(&h->cta_split, h->grid + 1, st));
    CC(dalloc(&h->owner_split, h->nsplit, st));
    CC(dalloc(&h->unit_c0, unit_c0_h.size(), st));
    CC(dalloc(&h->cta_seg, cta_seg_h.size(), st));
    std::vector<int> seg_meta_h(4 * seg_list_h.size());
    for (size_t k = 0; k < seg_list_h.size(); ++k) {
        const int sg = seg_list_h[k];
        seg_meta_h[4 * k + 0] = seg_row_h[(size_t)sg];
        seg_meta_h[4 * k + 1] = seg_k0_h[(size_t)sg];
        seg_meta_h[4 * k + 2] = seg_k1_h[(size_t)sg];
        seg_meta_h[4 * k + 3] = seg_split_h[(size_t)sg];
    }
    CC(dalloc(&h->seg_meta, seg_meta_h.size(), st));
    CC(dalloc(&h->seg_list, seg_list_h.size(), st));
    CC(dalloc(&h->seg_order, seg_order_h.size(), st));
    CC(dalloc(&h->seg_grp, seg_grp_h.size(), st));
    CC(dalloc(&h->cta_unit, cta_unit_h.size(), st));
    CC(dalloc(&h->partials, (size_t)2 * h->grid * AJM_NPART, st));
    CC(dalloc(&h->ctrl, 1, st));
    CC(dalloc(&h->scratch, 512, st));
    CC(dalloc(&h->err, 1, st));
    if (getenv("AJM_TS")) {
        CC(dalloc(&h->ts, 512 + 4 * (size_t)h->grid, st));
        CC(cudaMemsetAsync(h->ts, 0, (512 + 4 * (size_t)h->grid) * sizeof(unsigned long long), st));
    }
    h->h_ctrl = (AjmCtrl*)malloc(sizeof(AjmCtrl));
    if (!h->h_ctrl) return bail(fail(h, AJM_ERR_OOM, "host allocation failed"));
    CC(cudaEventCreate(&h->ev0));
    CC(cudaEventCreate(&h->ev1));

    mark("alloc", st);
    // ---- copies ----
    // b (and below D) arrive in the caller's row order; with relabelling they are gathered into
    // internal order (D through the X[2] scratch buffer, free until the first solve)
    if (h->relabel) {
        ajm_gather_kernel<<<1024, 256, 0, st>>>(n, h->perm_fwd, h->b_in, h->b);
        CC(cudaGetLastError());
    } else {
        CC(cudaMemcpyAsync(h->b, h->b_in, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    }
    CC(cudaFreeAsync(h->b_in, st));
    h->b_in = nullptr;
    double* dtmp = nullptr;
    if (dmode == AJM_D_USER) {
        CC(dalloc(&dtmp, n, st));
        CC(cudaMemcpyAsync(dtmp, d, sizeof(double) * n, kind_to_device(d), st));
    }
    auto h2d = [&](void* dst, const void* src, size_t bytes) {
        return bytes ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st) : cudaSuccess;
    };
    CC(h2d(h->chunk_off, choff.data(), sizeof(long long) * choff.size()));
    CC(h2d(h->seg_row, seg_row_h.data(), sizeof(int) * seg_row_h.size()));
    CC(h2d(h->seg_k0, seg_k0_h.data(), sizeof(int) * seg_k0_h.size()));
    CC(h2d(h->seg_k1, seg_k1_h.data(), sizeof(int) * seg_k1_h.size()));
    CC(h2d(h->seg_split, seg_split_h.data(), sizeof(int) * seg_split_h.size()));
    CC(h2d(h->split_row, split_row_h.data(), sizeof(int) * split_row_h.size()));
    CC(h2d(h->split_seg0, split_seg0_h.data(), sizeof(int) * split_seg0_h.size()));
    CC(h2d(h->cta_split, cta_split_h.data(), sizeof(int) * cta_split_h.size()));
    CC(h2d(h->owner_split, owner_split_h.data(), sizeof(int) * owner_split_h.size()));
    CC(h2d(h->unit_c0, unit_c0_h.data(), sizeof(int) * unit_c0_h.size()));
    CC(h2d(h->cta_seg, cta_seg_h.data(), sizeof(int) * cta_seg_h.size()));
    CC(h2d(h->seg_meta, seg_meta_h.data(), sizeof(int) * seg_meta_h.size()));
    if (!grp_h.empty()) {
        CC(dalloc(&h->grp, grp_h.size(), st));
        CC(h2d(h->grp, grp_h.data(), sizeof(int4) * grp_h.size()));
    }
    CC(h2d(h->seg_list, seg_list_h.data(), sizeof(int) * seg_list_h.size()));
    CC(h2d(h->seg_order, seg_order_h.data(), sizeof(int) * seg_order_h.size()));
    CC(h2d(h->seg_grp, seg_grp_h.data(), sizeof(int) * seg_grp_h.size()));
    CC(h2d(h->cta_unit, cta_unit_h.data(), sizeof(int) * cta_unit_h.size()));
    if (h->gmeta) {  // the per-CTA tables the kernel would otherwise stage in shared memory
        std::vector<int> guc, gco;
        std::vector<long long> gub((size_t)h->grid), gcb((size_t)h->grid);
        for (int cc = 0; cc < h->grid; ++cc) {
            const int u0 = cta_unit_h[(size_t)cc], u1 = cta_unit_h[(size_t)cc + 1];
            const int cf = u1 > u0 ? unit_c0_h[(size_t)u0] : 0;
            const int cl = u1 > u0 ? unit_c0_h[(size_t)u1] : 0;
            const long long ef = u1 > u0 ? choff[(size_t)cf] : 0;
            gub[(size_t)cc] = (long long)guc.size();
            for (int i = 0; i <= u1 - u0; ++i) guc.push_back(unit_c0_h[(size_t)(u0 + i)] - cf);
            gcb[(size_t)cc] = (long long)gco.size();
            for (int i = 0; i <= cl - cf; ++i) gco.push_back((int)(choff[(size_t)(cf + i)] - ef));
        }
        CC(dalloc(&h->g_uc0, guc.size(), st));
        CC(dalloc(&h->g_coff, gco.size(), st));
        CC(dalloc(&h->g_ubase, gub.size(), st));
        CC(dalloc(&h->g_cbase, gcb.size(), st));
        CC(h2d(h->g_uc0, guc.data(), sizeof(int) * guc.size()));
        CC(h2d(h->g_coff, gco.data(), sizeof(int) * gco.size()));
        CC(h2d(h->g_ubase, gub.data(), sizeof(long long) * gub.size()));
        CC(h2d(h->g_cbase, gcb.data(), sizeof(long long) * gcb.size()));
        CC(cudaStreamSynchronize(st));  // the host vectors die here
    }
    CC(cudaMemsetAsync(h->err, 0, sizeof(int), st));

    mark("copies", st);
    // ---- validation + D (device) ----
    const int nblk = (int)((n + 255) / 256);
    ajm_validate_diag_kernel<<<nblk, 256, 0, st>>>((int)n, (int)clo, (int)chi, h->rp, h->col, h->val, dmode == AJM_D_JBLOCK ? 0 : dmode, dtmp,
                                                   h->relabel ? h->X[2] : h->D, h->err,
                                                   vlong_h.empty() ? LLONG_MAX : (long long)kValidateLong);
    CC(cudaGetLastError());
    if (!vlong_h.empty()) {
        int* vl = nullptr;
        CC(dalloc(&vl, vlong_h.size(), st));
        CC(cudaMemcpyAsync(vl, vlong_h.data(), sizeof(int) * vlong_h.size(), cudaMemcpyHostToDevice, st));
        const int nl = (int)vlong_h.size();
        ajm_validate_long_kernel<<<(nl + 7) / 8, 256, 0, st>>>((int)clo, (int)chi, vl, nl, h->rp, h->col, h->val,
                                                               dmode == AJM_D_JBLOCK ? 0 : dmode, dtmp,
                                                               h->relabel ? h->X[2] : h->D, h->err);
        CC(cudaGetLastError());
        CC(cudaStreamSynchronize(st));  // vlong_h lives until the copy has run
        CC(cudaFreeAsync(vl, st));
    }
    if (h->relabel) {
        ajm_gather_kernel<<<1024, 256, 0, st>>>(n, h->perm_fwd, h->X[2], h->D);
        CC(cudaGetLastError());
    }
    ajm_finite_kernel<<<1024, 256, 0, st>>>(n, h->b, h->err);
    CC(cudaGetLastError());
    int herr = 0;
    CC(cudaMemcpyAsync(&herr, h->err, sizeof(int), cudaMemcpyDeviceToHost, st));
    CC(cudaStreamSynchronize(st));
    if (dtmp) cudaFreeAsync(dtmp, st);
    if (herr & AJM_EB_CSR) return bail(fail(h, AJM_ERR_CSR_INVALID, "column index out of range or not strictly increasing"));
    if (herr & AJM_EB_NONFINITE) return bail(fail(h, AJM_ERR_NONFINITE, "non-finite value in Q, b or d"));
    if (herr & AJM_EB_NEGDIAG) return bail(fail(h, AJM_ERR_NEGATIVE_DIAG, "negative diagonal entry: Q is not SPSD"));
    if (herr & AJM_EB_ZERODIAG) return bail(fail(h, AJM_ERR_ZERO_DIAG, "zero (or non-positive user) diagonal metric entry: D_kk = 0"));
    if (flags & AJM_VALIDATE_SYMMETRY) {
        ajm_symmetry_kernel<<<nblk, 256, 0, st>>>((int)n, h->rp, h->col, h->val, h->err);
        CC(cudaGetLastError());
        CC(cudaMemcpyAsync(&herr, h->err, sizeof(int), cudaMemcpyDeviceToHost, st));
        CC(cudaStreamSynchronize(st));
        if (herr & AJM_EB_ASYM) return bail(fail(h, AJM_ERR_NOT_SYMMETRIC, "Q is not symmetric"));
    }
    // eq-J-blkdiag: blocks, their inverses (per-chunk rows) and D = diag(J)
    if (h->jbs) {
        const int64_t sblk = (n + jbs - 1) / jbs;
        CC(dalloc(&h->Jblk, (size_t)sblk * jbs * jbs, st));
        CC(dalloc(&h->Jinv, (size_t)h->nchunks * jbs * 32, st));
        CC(cudaMemsetAsync(h->Jinv, 0, sizeof(double) * (size_t)h->nchunks * jbs * 32, st));
        const int tb = 64, gb = (int)((sblk + tb - 1) / tb);
        switch (jbs) {
            case 1: ajm_jblock_build_kernel<1><<<gb, tb, 0, st>>>((int)n, h->rp, h->col, h->val, h->Jblk, h->Jinv, h->D, h->err); break;
            case 2: ajm_jblock_build_kernel<2><<<gb, tb, 0, st>>>((int)n, h->rp, h->col, h->val, h->Jblk, h->Jinv, h->D, h->err); break;
            case 4: ajm_jblock_build_kernel<4><<<gb, tb, 0, st>>>((int)n, h->rp, h->col, h->val, h->Jblk, h->Jinv, h->D, h->err); break;
            case 8: ajm_jblock_build_kernel<8><<<gb, tb, 0, st>>>((int)n, h->rp, h->col, h->val, h->Jblk, h->Jinv, h->D, h->err); break;
            case 16: ajm_jblock_build_kernel<16><<<gb, tb, 0, st>>>((int)n, h->rp, h->col, h->val, h->Jblk, h->Jinv, h->D, h->err); break;
            default: ajm_jblock_build_kernel<32><<<gb, tb, 0, st>>>((int)n, h->rp, h->col, h->val, h->Jblk, h->Jinv, h->D, h->err); break;
        }
        CC(cudaGetLastError());
        CC(cudaMemcpyAsync(&herr, h->err, sizeof(int), cudaMemcpyDeviceToHost, st));
        CC(cudaStreamSynchronize(st));
        if (herr & AJM_EB_JBLOCK)
            return bail(fail(h, AJM_ERR_ZERO_DIAG, "a block J^{ii} of eq-J-blkdiag is not positive definite"));
    }
    mark("validate", st);
    // columns in internal numbering (after validation, which needs the caller's order)
    if (h->relabel && nnz > 0) {
        ajm_remap_kernel<<<2048, 256, 0, st>>>(nnz, (int)n, h->perm_inv, h->col);
        CC(cudaGetLastError());
    }
    mark("remap", st);
    // SELL copy of the short rows (slot -> caller's row through perm_fwd when relabelled)
    if (h->nchunks > 0) {
        const int ns = (int)(h->nchunks * 32);
        ajm_sell_fill_kernel<<<(ns + 255) / 256, 256, 0, st>>>(ns, (int)h->n_sell, h->perm_fwd, h->relabel ? 0 : 1,
                                                               h->rp, h->col, h->val, h->chunk_off, h->sval, h->scol);
        CC(cudaGetLastError());
    }
    mark("fill", st);
    // byte-coded columns: when the offsets col - row of the SELL entries take at most
    // AJM_CTAB distinct values (stencils: 7 / 27), stream one byte per entry instead of an int32
    // column (12 -> 9 bytes per stored entry) -- plain-ring variant-0 layouts only
    // (block J: there is no value-streamed byte-coded block-J kernel, so the codes are built with the
    //  int32 columns kept, and committed only if the pair coding below succeeds)
    bool jb_pending = false;
    if (h->nchunks > 0 && (h->ring_fn || (h->jbs && !sh)) && !h->cluster && !h->gmeta && !(flags & AJM_INT32_COLUMNS) &&
        !(h->jbs && (flags & AJM_VALUE_STREAM))) {
        const int ns = (int)(h->nchunks * 32);
        int* tmp = nullptr;
        CC(dalloc(&tmp, AJM_CTAB_HASH + 2, st));
        std::vector<int> htab(AJM_CTAB_HASH + 2, INT_MIN);
        htab[AJM_CTAB_HASH] = htab[AJM_CTAB_HASH + 1] = 0;
        CC(cudaMemcpyAsync(tmp, htab.data(), sizeof(int) * htab.size(), cudaMemcpyHostToDevice, st));
        ajm_coloff_collect_kernel<<<(ns + 255) / 256, 256, 0, st>>>(ns, (int)h->n_sell, h->chunk_off, h->scol, tmp,
                                                                     tmp + AJM_CTAB_HASH);
        CC(cudaGetLastError());
        CC(cudaMemcpyAsync(htab.data(), tmp, sizeof(int) * htab.size(), cudaMemcpyDeviceToHost, st));
        CC(cudaStreamSynchronize(st));
        // ring depth of the byte-coded kernels (18 KB stages): stencils' gathers hit L1 anyway, so
        // the depth goes to the ring -- 4 for narrow rows (config 2: 43.7 -> 43.0 us/pass vs 3), 5
        // for wide ones, whose units hold only 2-3 chunks (config 5: 1414 / 1139 / 1126 us/pass
        // at 3 / 4 / 5); AJM_COL8_STAGES=3..6 overrides (experiments)
        // Without warp segments the byte-coded kernel is always the variant compiled without the
        // segment phases (config 5: 1104 -> 1088 us/pass; the int32 layouts keep the seg variant
        // for wide rows, where it measured faster)
        int st8 = h->wide_rows ? 5 : 4;
        if (env_col8_stages) st8 = std::min(6, std::max(3, env_col8_stages));
        SolveFn f8 = col8_fn(h->nseg > 0, st8);

        const size_t dyn8 = (size_t)st8 * AJM_UNIT_EL * 9 + h->meta_bytes;
        int occ8 = 0;
        if (htab[AJM_CTAB_HASH + 1] == 0 && htab[AJM_CTAB_HASH] <= AJM_CTAB) {
            cudaError_t eo;
            {
                std::lock_guard<std::mutex> lock(g_attr_mu);
                eo = fn_occupancy(f8, dyn8, 100, &occ8, block_threads(h->nseg > 0));
            }
            CC(eo);
        }
        if (h->jbs && htab[AJM_CTAB_HASH + 1] == 0 && htab[AJM_CTAB_HASH] <= AJM_CTAB) occ8 = h->ctas_per_sm;
        if (occ8 >= h->ctas_per_sm && occ8 > 0) {
            std::vector<int> keys;
            for (int i = 0; i < AJM_CTAB_HASH; ++i)
                if (htab[(size_t)i] != INT_MIN) keys.push_back(htab[(size_t)i]);
            std::sort(keys.begin(), keys.end());
            const int m = (int)keys.size();
            keys.resize(AJM_CTAB, keys.empty() ? 0 : keys.back());
            CC(dalloc(&h->ctab, AJM_CTAB, st));
            CC(cudaMemcpyAsync(h->ctab, keys.data(), sizeof(int) * AJM_CTAB, cudaMemcpyHostToDevice, st));
            CC(dalloc(&h->scode, (size_t)h->sell_elems, st));
            ajm_coloff_encode_kernel<<<(ns + 255) / 256, 256, 0, st>>>(ns, (int)h->n_sell, h->chunk_off, h->scol,
                                                                        h->ctab, m, h->scode);
            CC(cudaGetLastError());
            if (h->jbs) {
                jb_pending = true;  // the int32 columns stay until the pair coding commits
            } else {
                CC(cudaFreeAsync(h->scol, st));
                h->scol = nullptr;
                h->fn = f8;
                h->dyn_smem = dyn8;
                h->ring_stages = st8;
            }
            h->col_bytes = 1;
        }
        CC(cudaStreamSynchronize(st));  // keys / htab live until the copies have run
        CC(cudaFreeAsync(tmp, st));
    }
    mark("col8", st);
    // pair-coded entries: when the byte-coded layout's (offset, value) pairs take at
    // most AJM_CTAB distinct values (constant-coefficient stencils: 7 / 27 / a few boundary
    // diagonals), the code byte indexes a table of pairs and the values are not streamed at all
    // (9 -> 1 byte per stored entry); the same values and columns in the same order, so bitwise the
    // same iterates.  AJM_VALUE_STREAM keeps the values (experiments, tests).
    if (h->col_bytes == 1 && !(flags & AJM_VALUE_STREAM) && !(sh && h->nseg > 0) && getenv("AJM_NO_PAIR") == nullptr) {
        const long long ne = (long long)h->sell_elems;
        unsigned long long* vt = nullptr;
        CC(dalloc(&vt, AJM_VTAB_HASH + 1, st));
        CC(cudaMemsetAsync(vt, 0xff, sizeof(unsigned long long) * AJM_VTAB_HASH, st));
        CC(cudaMemsetAsync(vt + AJM_VTAB_HASH, 0, sizeof(unsigned long long), st));
        int* vcnt = reinterpret_cast<int*>(vt + AJM_VTAB_HASH);
        const int gblocks = (int)std::min<long long>((ne + 255) / 256, 148LL * 16);
        ajm_val_collect_kernel<<<gblocks, 256, 0, st>>>(ne, h->sval, vt, vcnt);
        CC(cudaGetLastError());
        std::vector<unsigned long long> vh(AJM_VTAB_HASH + 1);
        CC(cudaMemcpyAsync(vh.data(), vt, sizeof(unsigned long long) * vh.size(), cudaMemcpyDeviceToHost, st));
        CC(cudaStreamSynchronize(st));
        int cnt2[2];
        std::memcpy(cnt2, &vh[AJM_VTAB_HASH], sizeof(cnt2));
        if (cnt2[1] == 0 && cnt2[0] <= AJM_CTAB) {
            std::vector<unsigned long long> vk;
            for (int i = 0; i < AJM_VTAB_HASH; ++i)
                if (vh[(size_t)i] != ~0ull) vk.push_back(vh[(size_t)i]);
            std::sort(vk.begin(), vk.end());
            const int mv = (int)vk.size();
            vk.resize(AJM_CTAB, ~0ull);
            // flags of the present (offset code, value code) pairs
            uint8_t* fl = nullptr;
            CC(dalloc(&fl, (size_t)AJM_CTAB * AJM_CTAB, st));
            CC(cudaMemsetAsync(fl, 0, (size_t)AJM_CTAB * AJM_CTAB, st));
            CC(cudaMemcpyAsync(vt, vk.data(), sizeof(unsigned long long) * AJM_CTAB, cudaMemcpyHostToDevice, st));
            ajm_pair_code_kernel<<<gblocks, 256, 0, st>>>(ne, h->sval, vt, mv, h->scode, fl, 0);
            CC(cudaGetLastError());
            std::vector<uint8_t> fh((size_t)AJM_CTAB * AJM_CTAB);
            std::vector<int> ch(AJM_CTAB);
            CC(cudaMemcpyAsync(fh.data(), fl, fh.size(), cudaMemcpyDeviceToHost, st));
            CC(cudaMemcpyAsync(ch.data(), h->ctab, sizeof(int) * AJM_CTAB, cudaMemcpyDeviceToHost, st));
            CC(cudaStreamSynchronize(st));
            std::vector<long long> pt;
            std::vector<uint8_t> map((size_t)AJM_CTAB * AJM_CTAB, 0);
            for (int k = 0; k < AJM_CTAB * AJM_CTAB; ++k)
                if (fh[(size_t)k]) {
                    if (pt.size() >= 2 * (size_t)AJM_CTAB) { pt.clear(); break; }
                    map[(size_t)k] = (uint8_t)(pt.size() / 2);
                    pt.push_back((long long)vk[(size_t)(k % AJM_CTAB)]);
                    pt.push_back((long long)ch[(size_t)(k / AJM_CTAB)]);
                }
            // more than AJM_CTAB pairs (pt cleared) or none: keep the values streamed
            if (!pt.empty()) {
                const char* es = getenv("AJM_PAIR_STAGES");  // (experiments) 4 or 8
                const int stp = h->jbs ? 4 : es ? (std::atoi(es) >= 8 ? 8 : 4) : (h->wide_rows ? 8 : 4);
                SolveFn fp = h->jbs ? jblock_pair_fn(h->jbs) : pair_fn(h->nseg > 0, stp);
                const size_t dynp = (size_t)stp * AJM_UNIT_EL * 1 + h->meta_bytes;
                int occp = 0;
                cudaError_t eo;
                {
                    std::lock_guard<std::mutex> lock(g_attr_mu);
                    eo = fn_occupancy(fp, dynp, 100, &occp, block_threads(h->nseg > 0));
                }
                CC(eo);
                if (occp >= h->ctas_per_sm) {
                    pt.resize(2 * (size_t)AJM_CTAB, 0);
                    CC(dalloc(&h->ptab, 2 * (size_t)AJM_CTAB, st));
                    CC(cudaMemcpyAsync(h->ptab, pt.data(), sizeof(long long) * pt.size(), cudaMemcpyHostToDevice, st));
                    CC(cudaMemcpyAsync(fl, map.data(), map.size(), cudaMemcpyHostToDevice, st));
                    ajm_pair_code_kernel<<<gblocks, 256, 0, st>>>(ne, h->sval, vt, mv, h->scode, fl, 1);
                    CC(cudaGetLastError());
                    CC(cudaFreeAsync(h->sval, st));
                    h->sval = nullptr;
                    if (jb_pending) {  // block J: the pair coding commits, the int32 columns go
                        CC(cudaFreeAsync(h->scol, st));
                        h->scol = nullptr;
                        jb_pending = false;
                    }
                    h->fn = fp;
                    h->dyn_smem = dynp;
                    h->ring_stages = stp;
                    h->pair = 1;
                }
            }
            CC(cudaStreamSynchronize(st));  // map / pt live until the copies have run
            CC(cudaFreeAsync(fl, st));
        }
        CC(cudaFreeAsync(vt, st));
    }
    if (jb_pending) {  // block J without a pair coding: back to the int32 columns
        CC(cudaStreamSynchronize(st));
        CC(cudaFreeAsync(h->scode, st));
        CC(cudaFreeAsync(h->ctab, st));
        h->scode = nullptr;
        h->ctab = nullptr;
        h->col_bytes = 4;
    }
    mark("pair", st);
    // banded staging (ajm_band_kernel): natural-order pair-coded layouts without long
    // rows and with a diagonal D whose column offsets fall into <= AJM_MAX_BANDS bands of width
    // <= 1024: every operand of a 256- or 512-row unit is staged by the TMA -- x~ over each band, b,
    // D, x^{t-1}, Q x^{t-1} -- next to its codes.  Same sums, same reduction order: bitwise the pair
    // kernel (AJM_NO_BAND=1 keeps it, experiments / tests).
    if (h->pair && !sh && h->nseg == 0 && !h->relabel && !h->jbs && !h->cluster && !h->gmeta && !h->resident &&
        getenv("AJM_NO_BAND") == nullptr && !(flags & AJM_NO_BAND_STAGING)) {
        std::vector<long long> pt(2 * (size_t)AJM_CTAB);
        std::vector<int> offs(AJM_CTAB);
        CC(cudaMemcpyAsync(pt.data(), h->ptab, sizeof(long long) * pt.size(), cudaMemcpyDeviceToHost, st));
        CC(cudaMemcpyAsync(offs.data(), h->ctab, sizeof(int) * AJM_CTAB, cudaMemcpyDeviceToHost, st));
        CC(cudaStreamSynchronize(st));
        std::vector<int> ko(offs.begin(), offs.end());
        ko.push_back(0);  // x~_row itself is always staged
        std::sort(ko.begin(), ko.end());
        ko.erase(std::unique(ko.begin(), ko.end()), ko.end());
        AjmBand bd = {};
        int maxw = 0;
        for (int64_t c = 0; c < h->nchunks; ++c) maxw = std::max<int>(maxw, (int)((choff[(size_t)c + 1] - choff[(size_t)c]) / 32));
        // two offset ranges share a band when the gap between them is below a unit's rows: the merged
        // band is then no longer than the two (config 2: the y-neighbour bands join the centre one,
        // 31.6 -> 28.5 us/pass; AJM_BAND_GAP overrides for experiments)
        // the band layout for units of ku chunks (32 ku rows); false if the offsets do not band
        auto plan_band = [&](int ku, AjmBand& out) {
            AjmBand q = {};
            const int urows = 32 * ku;
            const long long gap = getenv("AJM_BAND_GAP") ? std::atoll(getenv("AJM_BAND_GAP")) : urows;
            for (size_t i = 0; i < ko.size(); ++i) {
                if (q.nb > 0 && (long long)ko[i] - q.hi[q.nb - 1] <= gap) {
                    q.hi[q.nb - 1] = ko[i];
                } else if (q.nb < AJM_MAX_BANDS) {
                    q.lo[q.nb] = q.hi[q.nb] = ko[i];
                    q.nb += 1;
                } else {
                    return false;
                }
            }
            int xd = 0;
            for (int b = 0; b < q.nb; ++b) {
                if (q.hi[b] - q.lo[b] > 1024) return false;
                q.pos[b] = xd;
                const int len = urows + (q.hi[b] - q.lo[b]) + 2;
                xd += len + (len & 1);
            }
            q.urows = urows;
            q.xdoubles = xd;
            q.code_bytes = (urows * maxw + 15) / 16 * 16;
            q.stage_bytes = q.code_bytes + 8 * q.xdoubles + 4 * urows * 8;
            q.n_pad = (int)h->n_pad;
            out = q;
            return true;
        };
        auto soff_of = [&](int off) {
            for (int b = 0; b < bd.nb; ++b)
                if (off >= bd.lo[b] && off <= bd.hi[b]) return bd.pos[b] + off - bd.lo[b] + (bd.lo[b] & 1);
            return -1;
        };
        // (unit chunks, stages) in order of preference: the largest unit whose ring of >= 2 stages
        // keeps ctas_per_sm CTAs resident (config 2: 16 x 3 22.3 us/pass, 16 x 2 22.9, 8 x 4 27.2;
        // config 5's 27-wide 512-row stages do not fit, it takes 8 x 4); AJM_BAND_UNIT / AJM_BAND_STAGES
        // restrict the search (experiments)
        const int env_ku = getenv("AJM_BAND_UNIT") ? std::atoi(getenv("AJM_BAND_UNIT")) : 0;
        const int smax = getenv("AJM_BAND_STAGES") ? std::max(2, std::min(4, std::atoi(getenv("AJM_BAND_STAGES")))) : 4;
        const int cand[5][2] = {{16, 3}, {16, 2}, {8, 4}, {8, 3}, {8, 2}};
        int stb = 0, kub = 0;
        size_t dynb = 0;
        for (int ci = 0; ci < 5 && !stb && h->n_pad < INT_MAX / 2; ++ci) {
            const int ku = cand[ci][0], sgs = cand[ci][1];
            if ((env_ku && ku != env_ku) || sgs > smax) continue;
            AjmBand q;
            if (!plan_band(ku, q)) continue;
            const size_t dyn = (size_t)sgs * (size_t)q.stage_bytes + h->meta_bytes;
            int occ = 0;
            cudaError_t eo;
            {
                std::lock_guard<std::mutex> lock(g_attr_mu);
                eo = fn_occupancy(band_fn(sgs, ku), dyn, 100, &occ, block_threads(false));
            }
            CC(eo);
            if (occ >= h->ctas_per_sm) {
                stb = sgs;
                kub = ku;
                dynb = dyn;
                bd = q;
            }
        }
        bd.xt_soff = soff_of(0);
        if (stb) {
            bd.vpk = h->l2_mode == 3 ? 1 : (h->l2_mode >= 2 ? 2 : 0);
            bd.xpk = h->l2_mode >= 2 ? 2 : 0;
            if (getenv("AJM_BAND_VPK")) bd.vpk = std::atoi(getenv("AJM_BAND_VPK"));  // (experiments)
            if (getenv("AJM_BAND_XPK")) bd.xpk = std::atoi(getenv("AJM_BAND_XPK"));
            std::vector<long long> bp(2 * (size_t)AJM_CTAB, 0);
            for (int cc = 0; cc < AJM_CTAB; ++cc) {
                bp[2 * (size_t)cc] = pt[2 * (size_t)cc];
                const int so = soff_of((int)pt[2 * (size_t)cc + 1]);
                bp[2 * (size_t)cc + 1] = 8LL * (so < 0 ? bd.xt_soff : so);  // bytes (unused slots: any in-range offset)
            }
            CC(dalloc(&h->bptab, bp.size(), st));
            CC(cudaMemcpyAsync(h->bptab, bp.data(), sizeof(long long) * bp.size(), cudaMemcpyHostToDevice, st));
            CC(cudaStreamSynchronize(st));
            h->bd = bd;
            h->band = 1;
            h->fn = band_fn(stb, kub);
            h->dyn_smem = dynb;
            h->ring_stages = stb;
        }
    }
    mark("band", st);
    // shared-memory carve-out: the smallest that keeps ctas_per_sm CTAs resident, so the rest of
    // the SM's 256 KB stays L1 for the gathers; AJM_CARVEOUT=<pct> overrides
    {
        cudaFuncAttributes fa = {};
        CC(cudaFuncGetAttributes(&fa, (const void*)h->fn));
        int smem_sm = 0;
        CC(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, h->device));
        const double need = (double)h->ctas_per_sm * ((double)h->dyn_smem + (double)fa.sharedSizeBytes + 1024.0);
        int pct = (int)std::ceil(100.0 * need / std::max(1, smem_sm)) + 1;
        if (env_carveout >= 0) pct = env_carveout;
        pct = std::min(100, std::max(0, pct));
        int occ = 0;
        cudaError_t eo;
        {
            std::lock_guard<std::mutex> lock(g_attr_mu);
            if (h->resident) pct = 100;  // one CTA per SM of the cluster: all of it to shared memory
            eo = fn_occupancy(h->fn, h->dyn_smem, pct, &occ, h->resident ? AJM_BLOCK : block_threads(h->nseg > 0));
            if (eo == cudaSuccess && occ < h->ctas_per_sm && !h->cluster) {
                pct = 100;
                eo = cudaFuncSetAttribute((const void*)h->fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
            }
        }
        CC(eo);
        h->carveout = pct;
    }
    // Band kernel: the CTAs' chunk ranges re-planned for the band kernel.
    //  - chunk cost 123 + w (w = chunk width): measured per CTA (AJM_TS_ALL, config 5) the 18-wide
    //    z-boundary chunks take 0.94 of a 27-wide one -- the stage's x~ bands, row operands and
    //    per-row work weigh as much as the entries -- where the register kernels' batch-count cost
    //    gave them 0.75, and the two boundary CTAs finished 30-60 us after the others;
    //  - the SM-sharing skew: of the two CTAs on an SM the one launched first (lower index) is
    //    issued first by the warp schedulers and runs ~10 % faster while both are resident (config
    //    2: 16.9 vs 18.8 us, config 5: 343 vs 370 us per pass, every SM), and the pass waits for the
    //    later one.  A probe launch of the solver kernel itself (max_passes = 0) records each CTA's
    //    SM; the older CTA of every SM gets (1 + skew) of the mean cost, the younger (1 - skew).  A
    //    placement that differs at solve time only costs balance, never correctness (the
    //    arithmetic of a chunk does not depend on its CTA; a fixed plan keeps every solve of the
    //    handle bitwise the same).  Measured (tools/env_ab.py, profiles/r2i_band_replan_ab.log):
    //    config 2 21.89 (generic plan) -> 21.88 (band cost) -> 21.52 us/pass (skew 0.07; 0.045:
    //    21.67, 0.1: 21.97, 0.13: 22.24); config 5 411 -> 387 -> 381 (0.045 and 0.07 alike).
    //    AJM_BAND_SKEW=<x> overrides (experiments; 0 disables), AJM_BAND_NO_REPLAN keeps the
    //    generic plan's ranges (tests comparing partial sums bitwise with the other kernels).
    if (h->band) {
        const int G = h->grid;
        std::vector<int> c0h((size_t)G + 1);
        for (int cc = 0; cc <= G; ++cc) c0h[(size_t)cc] = unit_c0_h[(size_t)cta_unit_h[(size_t)cc]];
        const double skew = getenv("AJM_BAND_SKEW") ? std::atof(getenv("AJM_BAND_SKEW")) : AJM_BAND_SKEW;
        std::vector<int> age((size_t)G, -1);  // 0: first CTA on its SM, 1: second, ...
        if (h->ctas_per_sm >= 2 && skew != 0.0 && !sh) {
            CC(dalloc(&h->smid, G, st));
            CC(cudaMemsetAsync(h->smid, 0xff, sizeof(int) * (size_t)G, st));
        }
        std::vector<int> smid_h((size_t)G, -1);
        if (h->smid) {
            // the probe needs the (unchanged) plan's ranges: upload them first
            CC(dalloc(&h->band_c0, (size_t)G + 1, st));
            CC(cudaMemcpyAsync(h->band_c0, c0h.data(), sizeof(int) * ((size_t)G + 1), cudaMemcpyHostToDevice, st));
            AjmPass pp = make_pass(h, 0);
            pp.smid_out = h->smid;
            CC(launch_solver(h, pp, st));
            CC(cudaMemcpyAsync(smid_h.data(), h->smid, sizeof(int) * (size_t)G, cudaMemcpyDeviceToHost, st));
            CC(cudaStreamSynchronize(st));
            std::vector<int> seen;  // CTAs seen so far per SM (bid order = launch order)
            for (int cc = 0; cc < G; ++cc) {
                const int sm = smid_h[(size_t)cc];
                if (sm < 0) { age.assign((size_t)G, -1); break; }
                if ((size_t)sm >= seen.size()) seen.resize((size_t)sm + 1, 0);
                age[(size_t)cc] = seen[(size_t)sm]++;
            }
        }
        // weights: the older CTA of a shared SM (1 + skew), the younger (1 - skew); alone: 1
        std::vector<double> wt((size_t)G, 1.0);
        {
            std::vector<int> per_sm;
            for (int cc = 0; cc < G; ++cc)
                if (age[(size_t)cc] >= 0) {
                    const int sm = smid_h[(size_t)cc];
                    if ((size_t)sm >= per_sm.size()) per_sm.resize((size_t)sm + 1, 0);
                    per_sm[(size_t)sm]++;
                }
            for (int cc = 0; cc < G; ++cc)
                if (age[(size_t)cc] >= 0 && per_sm[(size_t)smid_h[(size_t)cc]] == 2)
                    wt[(size_t)cc] = age[(size_t)cc] == 0 ? 1.0 + skew : 1.0 - skew;
        }
        const int64_t nc = h->nchunks;
        std::vector<double> cpre((size_t)nc + 1, 0.0);
        for (int64_t cidx = 0; cidx < nc; ++cidx)
            cpre[(size_t)cidx + 1] = cpre[(size_t)cidx] + 123.0 + (double)((choff[(size_t)cidx + 1] - choff[(size_t)cidx]) >> 5);
        double wsum = 0.0;
        for (double w : wt) wsum += w;
        std::vector<int> nh((size_t)G + 1, 0);
        double wacc = 0.0;
        int64_t i = 0;
        for (int cc = 0; cc < G; ++cc) {
            nh[(size_t)cc] = (int)i;
            wacc += wt[(size_t)cc];
            const double lim = cpre[(size_t)nc] * wacc / wsum;
            while (i < nc && 0.5 * (cpre[(size_t)i] + cpre[(size_t)i + 1]) < lim) ++i;
        }
        nh[(size_t)G] = (int)nc;
        // the band kernel keeps a CTA's chunk offsets in the shared-memory table behind its ring
        int mx = 0;
        for (int cc = 0; cc < G; ++cc) mx = std::max(mx, nh[(size_t)cc + 1] - nh[(size_t)cc] + 1);
        if ((size_t)mx * sizeof(int) <= h->meta_bytes && !getenv("AJM_BAND_NO_REPLAN")) {  // (experiments)
            c0h.swap(nh);
            h->band_skew = h->smid ? skew : 0.0;
        }
        if (!h->band_c0) CC(dalloc(&h->band_c0, (size_t)G + 1, st));
        CC(cudaMemcpyAsync(h->band_c0, c0h.data(), sizeof(int) * ((size_t)G + 1), cudaMemcpyHostToDevice, st));
        CC(cudaStreamSynchronize(st));
        if (!h->cta_nchk.empty())
            for (int cc = 0; cc < G; ++cc) h->cta_nchk[(size_t)cc] = c0h[(size_t)cc + 1] - c0h[(size_t)cc];
    }
    // ||b||
    ajm_sumsq_partial_kernel<<<256, 256, 0, st>>>(n, h->b, h->scratch);
    ajm_sum_final_kernel<<<1, 32, 0, st>>>(256, h->scratch, h->scratch + 256);
    CC(cudaGetLastError());
    double bb = 0.0;
    CC(cudaMemcpyAsync(&bb, h->scratch + 256, sizeof(double), cudaMemcpyDeviceToHost, st));
    CC(cudaStreamSynchronize(st));
    if (sh) {
        h->bsq_local = bb;  // ||b|| of the whole system: ajm_shard_connect, in rank order
    } else {
        if (!(bb > 0.0)) return bail(fail(h, AJM_ERR_ZERO_RHS, "||b|| = 0: relative residual undefined"));
        h->nb = std::sqrt(bb);
    }
    // without warp segments the solver never reads the CSR copy again (everything is in the SELL
    // copy): release it, halving the matrix footprint (config 5: 5.4 GB)
    if (h->nseg == 0) {
        CC(cudaFreeAsync(h->col, st));
        CC(cudaFreeAsync(h->val, st));
        h->col = nullptr;
        h->val = nullptr;
    }
    if (!h->jbs && !sh) h->fn_lz = lanczos_fn(h->nseg > 0, h->cluster != 0, h->gmeta != 0, h->col_bytes, h->ring_stages, h->pair != 0);
    if (sh) {
        // the rank's kernel: the same layout class with the halo exchange compiled in
        h->fn = shard_fn(h->col_bytes, h->nseg > 0, h->ring_stages, sh->colocated != 0, h->pair != 0);
        {
            std::lock_guard<std::mutex> lock(g_attr_mu);
            int occ = 0;
            cudaError_t eo = fn_occupancy(h->fn, h->dyn_smem, h->carveout, &occ, block_threads(h->nseg > 0));
            if (eo == cudaSuccess && occ < h->ctas_per_sm) {  // (its pass-struct copy in shared memory)
                h->carveout = 100;
                eo = fn_occupancy(h->fn, h->dyn_smem, h->carveout, &occ, block_threads(h->nseg > 0));
            }
            if (eo == cudaSuccess && occ < h->ctas_per_sm)
                return bail(fail(h, AJM_ERR_UNSUPPORTED, "shard kernel cannot keep %d CTAs per SM resident", h->ctas_per_sm));
            CC(eo);
        }
        // send entries grouped by the CTA that writes the row: {internal row, peer, k, 0}, k = the
        // entry's position in this rank's list to that peer (turned into an offset at connect)
        std::vector<std::vector<int4>> per_cta((size_t)h->grid);
        size_t pos = 0;
        for (int r = 0; r < sh->nranks; ++r)
            for (int64_t k = 0; k < sh->send_cnt[(size_t)r]; ++k, ++pos) {
                const int64_t j = sh->send_rows[pos];
                const int ir = h->relabel ? inv_keep[(size_t)j] : (int)j;
                per_cta[(size_t)row_cta[(size_t)ir]].push_back(make_int4(ir, r, (int)k, 0));
            }
        h->snd_cta_host.assign((size_t)h->grid + 1, 0);
        h->snd_host.clear();
        for (int cc = 0; cc < h->grid; ++cc) {
            h->snd_cta_host[(size_t)cc] = (int)h->snd_host.size();
            h->snd_host.insert(h->snd_host.end(), per_cta[(size_t)cc].begin(), per_cta[(size_t)cc].end());
        }
        h->snd_cta_host[(size_t)h->grid] = (int)h->snd_host.size();
    }
    mark("validate+fill+norm", st);
    if (tsc) fprintf(stderr, "[ajm create ms]%s\n", tsc_log.c_str());
    *out = h;
#undef CC
    return AJM_OK;
}

// ---- ajm_solve in phases (shared with ajm_group_solve) ----
static ajm_status_t solve_check(ajm_ctx* h, const double* x_out, double tol, int64_t maxit, ajm_policy_t policy,
                                const int64_t* restart_iters, int64_t restart_cap) {
    h->err_msg.clear();
    if (!x_out) return fail(h, AJM_ERR_INVALID_ARG, "x_out is NULL");
    if (!(tol >= 0.0)) return fail(h, AJM_ERR_INVALID_ARG, "tol must be >= 0");
    if (maxit < 1) return fail(h, AJM_ERR_INVALID_ARG, "maxit must be >= 1");
    if (maxit >= (int64_t)INT32_MAX) return fail(h, AJM_ERR_INVALID_ARG, "maxit must be < 2^31 - 1");
    if (policy.k0 < 2) return fail(h, AJM_ERR_INVALID_ARG, "k0 must be >= 2 (P:460)");
    if (policy.restart && !policy.momentum)
        return fail(h, AJM_ERR_INVALID_ARG, "restart requires momentum (Alg. 2/3)");
    if (restart_iters && restart_cap < 0) return fail(h, AJM_ERR_INVALID_ARG, "restart_cap < 0");
    if (h->shard && !h->connected) return fail(h, AJM_ERR_INVALID_ARG, "shard handle is not connected (ajm_shard_connect)");
    if (h->broken) return fail(h, AJM_ERR_CUDA, "an earlier solve of this shard group timed out: re-create the group");
    return AJM_OK;
}

// x~^0, x^{-1}, Q x^{-1}, the control block (the own rows; a shard's halo of x~^0 is exchanged by
// the kernel's round 0)
static ajm_status_t solve_prep(ajm_ctx* h, const double* x0, double tol, int64_t maxit, ajm_policy_t policy,
                               cudaStream_t st) {
    const int64_t n = h->n;
    ajm_status_t s = ensure_hist(h, maxit + 2, st);
    if (s != AJM_OK) return s;

    // x~^0 = x0 and x^{-1} := x0 (beta_0 = 0 makes it unused); Q x^{-1} := 0 (finite, times 0)
    if (x0) {
        const cudaMemcpyKind k = kind_to_device(x0);
        if (h->relabel) {  // caller's order -> internal order (X[2] is free at this point)
            AJM_CUDA(h, cudaMemcpyAsync(h->X[2], x0, sizeof(double) * n, k, st));
            ajm_gather_kernel<<<1024, 256, 0, st>>>(n, h->perm_fwd, h->X[2], h->X[0]);
            AJM_CUDA(h, cudaGetLastError());
        } else {
            AJM_CUDA(h, cudaMemcpyAsync(h->X[0], x0, sizeof(double) * n, k, st));
        }
        AJM_CUDA(h, cudaMemsetAsync(h->err, 0, sizeof(int), st));
        ajm_finite_kernel<<<1024, 256, 0, st>>>(n, h->X[0], h->err);
        AJM_CUDA(h, cudaGetLastError());
        int herr = 0;
        AJM_CUDA(h, cudaMemcpyAsync(&herr, h->err, sizeof(int), cudaMemcpyDeviceToHost, st));
        AJM_CUDA(h, cudaStreamSynchronize(st));
        if (herr) return fail(h, AJM_ERR_NONFINITE, "x0 has a non-finite entry");
        AJM_CUDA(h, cudaMemcpyAsync(h->X[1], h->X[0], sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    } else {
        AJM_CUDA(h, cudaMemsetAsync(h->X[0], 0, sizeof(double) * h->n_pad, st));
        AJM_CUDA(h, cudaMemsetAsync(h->X[1], 0, sizeof(double) * h->n_pad, st));
    }
    AJM_CUDA(h, cudaMemsetAsync(h->Qxp, 0, sizeof(double) * h->n_pad, st));
    if (h->nsplit) AJM_CUDA(h, cudaMemsetAsync(h->split_cnt, 0, sizeof(unsigned) * h->nsplit, st));
    double* hr = h->hist;
    double* hf = h->hist + h->hist_cap;
    double* hd = h->hist + 2 * h->hist_cap;
    double* hda = h->hist + 3 * h->hist_cap;
    if (h->prime_bytes) {  // L2 priming pass (see ajm_create)
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)h->sm_count * 4);
        cfg.blockDim = dim3(256);
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeAccessPolicyWindow;
        at[0].val.accessPolicyWindow.base_ptr = h->vecs;
        at[0].val.accessPolicyWindow.num_bytes = h->prime_bytes;
        at[0].val.accessPolicyWindow.hitRatio = h->prime_hit;
        at[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        at[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        AJM_CUDA(h, cudaLaunchKernelEx(&cfg, ajm_l2_touch_kernel, (const double*)h->vecs,
                                       (long long)(h->prime_bytes / sizeof(double)), h->scratch + 300));
    }
    ajm_init_ctrl_kernel<<<1, 32, 0, st>>>(h->ctrl, tol, maxit, policy.momentum ? 1 : 0,
                                           policy.restart ? 1 : 0, policy.k0, h->nb, hr, hf, hd, hda);
    AJM_CUDA(h, cudaGetLastError());

    return AJM_OK;
}

// after the loop: the control block, the answer in the caller's order and the histories
static ajm_status_t solve_post(ajm_ctx* h, int64_t launches, float ms, double* x_out, ajm_result_t* res,
                               double* res_hist, double* f_hist, int64_t* restart_iters, int64_t restart_cap,
                               cudaStream_t st) {
    const int64_t n = h->n;
    AJM_CUDA(h, cudaMemcpyAsync(h->h_ctrl, h->ctrl, sizeof(AjmCtrl), cudaMemcpyDeviceToHost, st));
    AJM_CUDA(h, cudaStreamSynchronize(st));
    const AjmCtrl& c = *h->h_ctrl;
    if (h->shard) {  // every other rank added one arrival per round to this rank's counter
        if (c.timeout_flag || !c.s.done) h->broken = true;
        else h->bar_base += (unsigned long long)(h->nranks - 1) * (unsigned long long)(c.s.iterations + 2);
    }
    if (c.timeout_flag) return fail(h, AJM_ERR_CUDA, "device barrier wait timed out (internal error)");
    if (!c.s.done) return fail(h, AJM_ERR_CUDA, "iteration loop ended without a termination decision");
    h->last_loop_ms = ms;
    h->last_passes = c.s.iterations + 1;
    h->last_launches = launches;
    h->last_iterations = c.s.iterations;
    double* hr = h->hist;
    double* hf = h->hist + h->hist_cap;
    if (h->ts) {  // debug: mean phase durations of CTA 0 over the first passes
        unsigned long long hts[64 * 8];
        AJM_CUDA(h, cudaMemcpy(hts, h->ts, sizeof(hts), cudaMemcpyDeviceToHost));
        double acc[5] = {0, 0, 0, 0, 0}, seg = 0, chk = 0, ctl = 0;
        int np = 0;
        for (int k = 2; k + 1 < 64 && k + 1 <= c.s.iterations; ++k) {
            if (!hts[k * 8 + 5] || !hts[(k + 1) * 8]) break;
            for (int j = 0; j < 4; ++j) acc[j] += (double)(hts[k * 8 + j + 1] - hts[k * 8 + j]);
            acc[4] += (double)(hts[(k + 1) * 8] - hts[k * 8 + 4]);
            seg += (double)(hts[k * 8 + 6] - hts[k * 8 + 0]);
            chk += (double)(hts[k * 8 + 7] - hts[k * 8 + 6]);
            ctl += (double)(hts[k * 8 + 5] - hts[k * 8 + 4]);
            ++np;
        }
        std::vector<unsigned long long> cta((size_t)4 * h->grid);
        AJM_CUDA(h, cudaMemcpy(cta.data(), h->ts + 512, sizeof(unsigned long long) * cta.size(), cudaMemcpyDeviceToHost));
        if (c.s.iterations >= 6 && hts[5 * 8]) {  // pass-5 work-end of every CTA relative to the pass start
            std::vector<std::pair<double, int>> endt;
            for (int g = 0; g < h->grid; ++g)
                endt.push_back({(double)(cta[(size_t)4 * g] - hts[5 * 8]) / 1e3, (int)cta[(size_t)4 * g + 1]});
            std::sort(endt.begin(), endt.end());
            auto q = [&](double f) { return endt[(size_t)std::min<double>(endt.size() - 1, f * (endt.size() - 1))]; };
            fprintf(stderr, "[ajm ts] pass 5 CTA work-end us: min %.2f (sm %d) p10 %.2f p50 %.2f p90 %.2f max %.2f (sm %d)\n",
                    endt.front().first, endt.front().second, q(0.1).first, q(0.5).first, q(0.9).first,
                    endt.back().first, endt.back().second);
            if (getenv("AJM_TS_ALL")) {
                for (int g = 0; g < h->grid; ++g)
                    fprintf(stderr, "[ajm cta] %d sm %d seg-end %.2f chunk-end %.2f end %.2f chunks %d\n", g, (int)cta[(size_t)4 * g + 1],
                            (double)(cta[(size_t)4 * g + 2] - hts[5 * 8]) / 1e3, (double)(cta[(size_t)4 * g + 3] - hts[5 * 8]) / 1e3,
                            (double)(cta[(size_t)4 * g] - hts[5 * 8]) / 1e3, h->cta_nchk.empty() ? -1 : h->cta_nchk[(size_t)g]);
            }
        }
        if (np)
            fprintf(stderr, "[ajm ts] passes %d: work %.2f us, block-reduce %.2f, grid-barrier %.2f, "
                            "partials %.2f, control+sync %.2f (control %.2f) | segments %.2f, chunks %.2f\n", np, acc[0] / np / 1e3,
                    acc[1] / np / 1e3, acc[2] / np / 1e3, acc[3] / np / 1e3, acc[4] / np / 1e3, ctl / np / 1e3, seg / np / 1e3,
                    chk / np / 1e3);
    }

    if (h->relabel) {  // internal order -> caller's order, through a buffer that is not the answer
        double* tmp = h->X[(c.s.answer + 1) % 3];
        ajm_gather_kernel<<<1024, 256, 0, st>>>(n, h->perm_inv, h->X[c.s.answer], tmp);
        AJM_CUDA(h, cudaGetLastError());
        AJM_CUDA(h, cudaMemcpyAsync(x_out, tmp, sizeof(double) * n, kind_from_device(x_out), st));
    } else {
        AJM_CUDA(h, cudaMemcpyAsync(x_out, h->X[c.s.answer], sizeof(double) * n, kind_from_device(x_out), st));
    }
    const int64_t cnt = c.s.iterations + 1;
    if (res_hist) AJM_CUDA(h, cudaMemcpyAsync(res_hist, hr, sizeof(double) * cnt, kind_from_device(res_hist), st));
    if (f_hist) AJM_CUDA(h, cudaMemcpyAsync(f_hist, hf, sizeof(double) * cnt, kind_from_device(f_hist), st));
    AJM_CUDA(h, cudaStreamSynchronize(st));
    const int64_t nlog = std::min<int64_t>(c.s.nlogged, restart_iters ? restart_cap : 0);
    for (int64_t i = 0; i < nlog; ++i) restart_iters[i] = c.restart_log[i];
    if (res) {
        res->status = c.s.status;
        res->n_restarts = c.s.nres;
        res->iterations = c.s.iterations;
        res->rel_residual = c.s.res_last;
        res->f = c.s.f_last;
        res->x_is_prerestart = c.s.prerestart;
        res->restarts_logged = (int32_t)nlog;
    }
    return AJM_OK;
}


ajm_status_t ajm_solve(ajm_handle_t h, const double* x0, double tol, int64_t maxit,
                       ajm_policy_t policy, double* x_out, ajm_result_t* res, double* res_hist,
                       double* f_hist, int64_t* restart_iters, int64_t restart_cap,
                       void* cuda_stream) {
    NvtxScope nvtx_scope_("ajm_solve");
    if (!h) return fail(nullptr, AJM_ERR_INVALID_ARG, "NULL handle");
    ajm_status_t s = solve_check(h, x_out, tol, maxit, policy, restart_iters, restart_cap);
    if (s != AJM_OK) return s;
    if (h->colocated) return fail(h, AJM_ERR_INVALID_ARG, "an AJM_SHARD_COLOCATED group is solved by ajm_group_solve");
    cudaStream_t st = (cudaStream_t)cuda_stream;
    s = solve_prep(h, x0, tol, maxit, policy, st);
    if (s != AJM_OK) return s;
    AJM_CUDA(h, cudaEventRecord(h->ev0, st));
    int64_t launches = 0;
    if (!(h->flags & AJM_LOOP_HOST)) {
        // the whole Alg. 3 loop: one cooperative launch
        AjmPass p = make_pass(h, (int)(maxit + 1));
        AJM_CUDA(h, launch_solver(h, p, st));
        launches = 1;
    } else {
        // debug host loop: one pass per launch, the control state round-trips through global memory
        AjmPass p = make_pass(h, 1);
        int64_t issued = 0;
        for (;;) {
            const int64_t chunk = std::min<int64_t>(64, maxit + 1 - issued);
            for (int64_t i = 0; i < chunk; ++i) AJM_CUDA(h, launch_solver(h, p, st));
            issued += chunk;
            AJM_CUDA(h, cudaMemcpyAsync(h->h_ctrl, h->ctrl, sizeof(AjmCtrl), cudaMemcpyDeviceToHost, st));
            AJM_CUDA(h, cudaStreamSynchronize(st));
            if (h->h_ctrl->s.done || issued >= maxit + 1) break;
        }
        launches = issued;
    }
    AJM_CUDA(h, cudaEventRecord(h->ev1, st));
    AJM_CUDA(h, cudaEventSynchronize(h->ev1));
    float ms = 0.f;
    AJM_CUDA(h, cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    return solve_post(h, launches, ms, x_out, res, res_hist, f_hist, restart_iters, restart_cap, st);
}

// ------------------------------------------------------------------------------------------------
// Row-block sharded solve (NEXT-2; include/ajm.h)
// ------------------------------------------------------------------------------------------------

ajm_status_t ajm_create(ajm_handle_t* out, int64_t n, int64_t nnz, const int64_t* row_ptr,
                        const int32_t* col_idx, const double* vals, const double* b, int32_t dmode,
                        const double* d, uint32_t flags, void* cuda_stream) {
    return create_impl(out, n, nnz, row_ptr, col_idx, vals, b, dmode, d, flags, cuda_stream, nullptr);
}

ajm_status_t ajm_partition_rows(int64_t n, const int64_t* row_ptr, int32_t nranks, int64_t* row_starts) {
    g_create_error.clear();
    if (!row_ptr || !row_starts) return fail(nullptr, AJM_ERR_INVALID_ARG, "NULL argument");
    if (nranks < 1 || nranks > AJM_MAX_RANKS || n < nranks)
        return fail(nullptr, AJM_ERR_INVALID_ARG, "need 1 <= nranks <= min(%d, n)", AJM_MAX_RANKS);
    if (row_ptr[0] != 0) return fail(nullptr, AJM_ERR_CSR_INVALID, "row_ptr[0] != 0");
    for (int64_t i = 0; i < n; ++i)
        if (row_ptr[i + 1] < row_ptr[i]) return fail(nullptr, AJM_ERR_CSR_INVALID, "row_ptr decreases at row %lld", (long long)i);
    // block r starts at the first row whose prefix cost reaches r/nranks of the total (12 B per
    // nonzero + 56 B per row: the pass's bytes), at least one row per block
    const double total = 12.0 * (double)row_ptr[n] + 56.0 * (double)n;
    row_starts[0] = 0;
    int64_t i = 0;
    for (int r = 1; r < nranks; ++r) {
        const double lim = total * (double)r / (double)nranks;
        while (i < n && 12.0 * (double)row_ptr[i] + 56.0 * (double)i < lim) ++i;
        row_starts[r] = std::min<int64_t>(std::max<int64_t>(i, row_starts[r - 1] + 1), n - (nranks - r));
        i = row_starts[r];
    }
    row_starts[nranks] = n;
    return AJM_OK;
}

namespace {
// The plan of one rank (host only): local columns, halo (sorted global indices), send lists.
ajm_status_t shard_plan_host(int rank, int R, const int64_t* starts, const int64_t* rp, const int32_t* colg,
                             std::vector<int32_t>* col_loc, std::vector<int64_t>* halo_glob,
                             std::vector<int64_t>* send_rows, ShardIn& out) {
    if (R < 1 || R > AJM_MAX_RANKS || rank < 0 || rank >= R || !starts || !rp)
        return fail(nullptr, AJM_ERR_INVALID_ARG, "bad rank / nranks / NULL argument");
    if (starts[0] != 0) return fail(nullptr, AJM_ERR_INVALID_ARG, "row_starts[0] != 0");
    for (int r = 0; r < R; ++r)
        if (starts[r + 1] <= starts[r]) return fail(nullptr, AJM_ERR_INVALID_ARG, "row_starts must increase (every block non-empty)");
    const int64_t n = starts[R], r0 = starts[rank], r1 = starts[rank + 1], nl = r1 - r0;
    if (n >= ((int64_t)1 << 31)) return fail(nullptr, AJM_ERR_UNSUPPORTED, "n must be < 2^31");
    if (rp[0] != 0) return fail(nullptr, AJM_ERR_CSR_INVALID, "row_ptr[0] != 0");
    for (int64_t i = 0; i < nl; ++i)
        if (rp[i + 1] < rp[i]) return fail(nullptr, AJM_ERR_CSR_INVALID, "row_ptr decreases at local row %lld", (long long)i);
    const int64_t nnz = rp[nl];
    if (nnz > 0 && !colg) return fail(nullptr, AJM_ERR_INVALID_ARG, "col_idx is NULL");
    auto owner = [&](int64_t j) { return (int)(std::upper_bound(starts, starts + R + 1, j) - starts) - 1; };
    // halo: the distinct out-of-block columns, sorted (lower ranks' entries first)
    int bad = 0;
    std::vector<int32_t> hal;
    {
        std::vector<std::vector<int32_t>> th;
#pragma omp parallel
        {
#pragma omp single
            th.resize((size_t)omp_get_num_threads());
            std::vector<int32_t>& v = th[(size_t)omp_get_thread_num()];
#pragma omp for schedule(static) reduction(| : bad)
            for (int64_t k = 0; k < nnz; ++k) {
                const int64_t j = colg[k];
                if (j < 0 || j >= n) bad |= 1;
                else if (j < r0 || j >= r1) v.push_back((int32_t)j);
            }
        }
        for (auto& v : th) hal.insert(hal.end(), v.begin(), v.end());
    }
    if (bad) return fail(nullptr, AJM_ERR_CSR_INVALID, "column index out of [0, n)");
    std::sort(hal.begin(), hal.end());
    hal.erase(std::unique(hal.begin(), hal.end()), hal.end());
    const int64_t hlo = (int64_t)(std::lower_bound(hal.begin(), hal.end(), (int32_t)r0) - hal.begin());
    out.rank = rank;
    out.nranks = R;
    out.n_glob = n;
    out.row0 = r0;
    out.h_lo = hlo;
    out.h_hi = (int64_t)hal.size() - hlo;
    out.halo_cnt.assign((size_t)R, 0);
    for (int32_t j : hal) ++out.halo_cnt[(size_t)owner(j)];
    if (halo_glob) halo_glob->assign(hal.begin(), hal.end());
    if (col_loc) {
        col_loc->resize((size_t)nnz);
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < nnz; ++k) {
            const int32_t j = colg[k];
            int64_t l;
            if (j >= r0 && j < r1) l = j - r0;
            else {
                const int64_t pos = (int64_t)(std::lower_bound(hal.begin(), hal.end(), j) - hal.begin());
                l = pos < hlo ? pos - hlo : nl + (pos - hlo);
            }
            (*col_loc)[(size_t)k] = (int32_t)l;
        }
    }
    // send lists: by symmetry of the structure, rank s reads own row i iff row i has a column in s's block
    std::vector<std::vector<std::vector<int64_t>>> ts;  // [thread][dest] rows, contiguous row ranges
    int nt = 1;
#pragma omp parallel
    {
#pragma omp single
        {
            nt = omp_get_num_threads();
            ts.assign((size_t)nt, std::vector<std::vector<int64_t>>((size_t)R));
        }
        const int tid = omp_get_thread_num();
        const int64_t lo = nl * tid / nt, hi = nl * (tid + 1) / nt;
        std::vector<int64_t> last((size_t)R, -1);
        for (int64_t i = lo; i < hi; ++i)
            for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
                const int64_t j = colg[k];
                if (j >= r0 && j < r1) continue;
                const int s = owner(j);
                if (last[(size_t)s] != i) {
                    last[(size_t)s] = i;
                    ts[(size_t)tid][(size_t)s].push_back(i);
                }
            }
    }
    out.send_cnt.assign((size_t)R, 0);
    std::vector<int64_t> sr;
    for (int s = 0; s < R; ++s)
        for (int t2 = 0; t2 < nt; ++t2) {
            out.send_cnt[(size_t)s] += (int64_t)ts[(size_t)t2][(size_t)s].size();
            sr.insert(sr.end(), ts[(size_t)t2][(size_t)s].begin(), ts[(size_t)t2][(size_t)s].end());
        }
    out.send_rows = sr;
    if (send_rows) send_rows->swap(sr);
    return AJM_OK;
}

// The connection record of one rank (ajm_shard_export / ajm_shard_connect)
struct ShardBlob {
    uint32_t magic;
    int32_t version, rank, nranks;
    int32_t device, pid, colocated, grid;
    int64_t n_loc, row0, n_glob;
    cudaIpcMemHandle_t vec_h, xch_h;
    int32_t ipc_ok, carveout;
    uint64_t vec_ptr, xch_ptr, fn;
    int64_t x_off[3];
    int64_t dyn_smem;
    int64_t halo_off[AJM_MAX_RANKS], halo_cnt[AJM_MAX_RANKS], send_cnt[AJM_MAX_RANKS];
    double bsq;
};
static_assert(sizeof(ShardBlob) <= AJM_SHARD_BLOB_BYTES, "shard record size");
constexpr uint32_t kBlobMagic = 0x414a4d53u;  // "AJMS"
}  // namespace

ajm_status_t ajm_shard_plan(int32_t rank, int32_t nranks, const int64_t* row_starts, const int64_t* row_ptr,
                            const int32_t* col_glob, int32_t* col_loc, int64_t* halo_glob, int64_t* send_rows,
                            int64_t* counts) {
    g_create_error.clear();
    if (!counts) return fail(nullptr, AJM_ERR_INVALID_ARG, "counts is NULL");
    ShardIn sp;
    std::vector<int32_t> cl;
    std::vector<int64_t> hg, sr;
    ajm_status_t s = shard_plan_host(rank, nranks, row_starts, row_ptr, col_glob, col_loc ? &cl : nullptr,
                                     halo_glob ? &hg : nullptr, send_rows ? &sr : nullptr, sp);
    if (s != AJM_OK) return s;
    counts[0] = sp.h_lo;
    counts[1] = sp.h_hi;
    for (int r = 0; r < nranks; ++r) {
        counts[2 + r] = sp.halo_cnt[(size_t)r];
        counts[2 + nranks + r] = sp.send_cnt[(size_t)r];
    }
    if (col_loc) std::copy(cl.begin(), cl.end(), col_loc);
    if (halo_glob) std::copy(hg.begin(), hg.end(), halo_glob);
    if (send_rows) std::copy(sr.begin(), sr.end(), send_rows);
    return AJM_OK;
}

ajm_status_t ajm_shard_create(ajm_handle_t* out, int32_t rank, int32_t nranks, const int64_t* row_starts,
                              int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx, const double* vals,
                              const double* b, int32_t dmode, const double* d, uint32_t flags,
                              void* cuda_stream) {
    g_create_error.clear();
    if (!out || !row_starts || !row_ptr || !b || (nnz > 0 && (!col_idx || !vals)))
        return fail(nullptr, AJM_ERR_INVALID_ARG, "NULL argument");
    if (nranks < 1 || nranks > AJM_MAX_RANKS || rank < 0 || rank >= nranks)
        return fail(nullptr, AJM_ERR_INVALID_ARG, "bad rank / nranks (1 <= nranks <= %d)", AJM_MAX_RANKS);
    if (nnz < 0) return fail(nullptr, AJM_ERR_INVALID_ARG, "nnz < 0");
    for (int r = 0; r < nranks; ++r)
        if (row_starts[r + 1] <= row_starts[r]) return fail(nullptr, AJM_ERR_INVALID_ARG, "row_starts must increase");
    const int64_t nl = row_starts[rank + 1] - row_starts[rank];
    // the plan needs the rank's structure on the host
    std::vector<int64_t> rph;
    std::vector<int32_t> colh;
    const int64_t* rpp = row_ptr;
    const int32_t* cp = col_idx;
    if (is_device_ptr(row_ptr)) {
        rph.resize((size_t)nl + 1);
        if (cudaMemcpy(rph.data(), row_ptr, sizeof(int64_t) * (nl + 1), cudaMemcpyDeviceToHost) != cudaSuccess)
            return fail(nullptr, AJM_ERR_CUDA, "row_ptr copy failed");
        rpp = rph.data();
    }
    if (rpp[nl] != nnz) return fail(nullptr, AJM_ERR_CSR_INVALID, "row_ptr[n_loc] != nnz");
    if (nnz > 0 && is_device_ptr(col_idx)) {
        colh.resize((size_t)nnz);
        if (cudaMemcpy(colh.data(), col_idx, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost) != cudaSuccess)
            return fail(nullptr, AJM_ERR_CUDA, "col_idx copy failed");
        cp = colh.data();
    }
    ShardIn sp;
    std::vector<int32_t> cl;
    ajm_status_t s = shard_plan_host(rank, nranks, row_starts, rpp, cp, &cl, nullptr, nullptr, sp);
    if (s != AJM_OK) return s;
    sp.colocated = (flags & AJM_SHARD_COLOCATED) ? 1 : 0;
    return create_impl(out, nl, nnz, rpp, cl.data(), vals, b, dmode, d, flags & ~AJM_SHARD_COLOCATED, cuda_stream, &sp);
}

ajm_status_t ajm_shard_export(ajm_handle_t h, void* blob) {
    if (!h || !blob) return fail(h, AJM_ERR_INVALID_ARG, "NULL argument");
    if (!h->shard) return fail(h, AJM_ERR_INVALID_ARG, "not a shard handle");
    ShardBlob bl;
    memset(&bl, 0, sizeof bl);
    bl.magic = kBlobMagic;
    bl.version = AJM_ABI_VERSION;
    bl.rank = h->rank;
    bl.nranks = h->nranks;
    bl.device = h->device;
    bl.pid = (int32_t)getpid();
    bl.colocated = h->colocated;
    bl.grid = h->grid;
    bl.n_loc = h->n;
    bl.row0 = h->row0;
    bl.n_glob = h->n_glob;
    bl.ipc_ok = (cudaIpcGetMemHandle(&bl.vec_h, h->vecs) == cudaSuccess &&
                 cudaIpcGetMemHandle(&bl.xch_h, h->xch) == cudaSuccess) ? 1 : 0;
    cudaGetLastError();
    bl.carveout = h->carveout;
    bl.vec_ptr = (uint64_t)(uintptr_t)h->vecs;
    bl.xch_ptr = (uint64_t)(uintptr_t)h->xch;
    bl.fn = (uint64_t)(uintptr_t)h->fn;
    for (int k = 0; k < 3; ++k) bl.x_off[k] = (int64_t)(h->X[k] - h->vecs);
    bl.dyn_smem = (int64_t)h->dyn_smem;
    int64_t lo = -h->h_lo, hi = h->n;  // where each source rank's entries start in this rank's halo
    for (int r = 0; r < h->nranks; ++r) {
        bl.halo_cnt[r] = h->halo_cnt[(size_t)r];
        bl.send_cnt[r] = h->send_cnt[(size_t)r];
        if (r < h->rank) { bl.halo_off[r] = lo; lo += h->halo_cnt[(size_t)r]; }
        else if (r > h->rank) { bl.halo_off[r] = hi; hi += h->halo_cnt[(size_t)r]; }
    }
    bl.bsq = h->bsq_local;
    memset(blob, 0, AJM_SHARD_BLOB_BYTES);
    memcpy(blob, &bl, sizeof bl);
    return AJM_OK;
}

ajm_status_t ajm_shard_connect(ajm_handle_t h, const void* blobs) {
    if (!h || !blobs) return fail(h, AJM_ERR_INVALID_ARG, "NULL argument");
    if (!h->shard) return fail(h, AJM_ERR_INVALID_ARG, "not a shard handle");
    if (h->connected) return fail(h, AJM_ERR_INVALID_ARG, "already connected");
    h->err_msg.clear();
    const int R = h->nranks, me = h->rank;
    std::vector<ShardBlob> bl((size_t)R);
    for (int r = 0; r < R; ++r) memcpy(&bl[(size_t)r], (const char*)blobs + (size_t)r * AJM_SHARD_BLOB_BYTES, sizeof(ShardBlob));
    for (int r = 0; r < R; ++r) {
        const ShardBlob& b = bl[(size_t)r];
        if (b.magic != kBlobMagic || b.version != AJM_ABI_VERSION || b.rank != r || b.nranks != R || b.n_glob != h->n_glob)
            return fail(h, AJM_ERR_INVALID_ARG, "record %d is not rank %d of this group", r, r);
        if (r + 1 < R && b.row0 + b.n_loc != bl[(size_t)r + 1].row0)
            return fail(h, AJM_ERR_INVALID_ARG, "records disagree on the row partition");
        if (r != me && (b.halo_cnt[me] != h->send_cnt[(size_t)r] || b.send_cnt[me] != h->halo_cnt[(size_t)r]))
            return fail(h, AJM_ERR_NOT_SYMMETRIC, "rank %d's halo from rank %d (%lld entries) differs from rank %d's send "
                        "list (%lld): Q is not structurally symmetric", r, me, (long long)b.halo_cnt[me], me,
                        (long long)h->send_cnt[(size_t)r]);
        if (h->colocated && (b.pid != (int32_t)getpid() || b.device != h->device || !b.colocated))
            return fail(h, AJM_ERR_INVALID_ARG, "an AJM_SHARD_COLOCATED group must live in one process on one device");
    }
    // ||b||^2 summed in rank order: the same bits on every rank
    double bb = 0.0;
    for (int r = 0; r < R; ++r) bb += bl[(size_t)r].bsq;
    if (!(bb > 0.0)) return fail(h, AJM_ERR_ZERO_RHS, "||b|| = 0: relative residual undefined");
    h->peers_host.assign((size_t)R, AjmPeer{});
    for (int r = 0; r < R; ++r) {
        const ShardBlob& b = bl[(size_t)r];
        double* vec = nullptr;
        double* xch = nullptr;
        if (r == me) {
            vec = h->vecs;
            xch = h->xch;
        } else if (b.pid == (int32_t)getpid()) {
            vec = (double*)(uintptr_t)b.vec_ptr;
            xch = (double*)(uintptr_t)b.xch_ptr;
            if (b.device != h->device) {
                cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                    return fail(h, AJM_ERR_CUDA, "peer access to device %d: %s", b.device, cudaGetErrorString(e));
                cudaGetLastError();
            }
        } else {
            if (!b.ipc_ok) return fail(h, AJM_ERR_CUDA, "rank %d could not export CUDA IPC handles", r);
            void* pv = nullptr;
            void* px = nullptr;
            AJM_CUDA(h, cudaIpcOpenMemHandle(&pv, b.vec_h, cudaIpcMemLazyEnablePeerAccess));
            h->ipc_opened.push_back(pv);
            AJM_CUDA(h, cudaIpcOpenMemHandle(&px, b.xch_h, cudaIpcMemLazyEnablePeerAccess));
            h->ipc_opened.push_back(px);
            vec = (double*)pv;
            xch = (double*)px;
        }
        AjmPeer& pe = h->peers_host[(size_t)r];
        for (int k = 0; k < 3; ++k) pe.x[k] = vec + b.x_off[k];
        pe.slot = xch;
        pe.bar = reinterpret_cast<unsigned long long*>(xch + 2 * AJM_MAX_RANKS * AJM_NPART);
    }
    // the send entries' positions become offsets into the destination's buffers
    std::vector<int4> snd = h->snd_host;
    for (int4& e : snd) e.z = (int)(bl[(size_t)e.y].halo_off[me] + e.z);
    AJM_CUDA(h, cudaMalloc((void**)&h->peers, sizeof(AjmPeer) * R));
    AJM_CUDA(h, cudaMemcpy(h->peers, h->peers_host.data(), sizeof(AjmPeer) * R, cudaMemcpyHostToDevice));
    AJM_CUDA(h, cudaMalloc((void**)&h->snd_cta, sizeof(int) * h->snd_cta_host.size()));
    AJM_CUDA(h, cudaMemcpy(h->snd_cta, h->snd_cta_host.data(), sizeof(int) * h->snd_cta_host.size(), cudaMemcpyHostToDevice));
    AJM_CUDA(h, cudaMalloc((void**)&h->snd, sizeof(int4) * std::max<size_t>(1, snd.size())));
    if (!snd.empty()) AJM_CUDA(h, cudaMemcpy(h->snd, snd.data(), sizeof(int4) * snd.size(), cudaMemcpyHostToDevice));
    h->nb = std::sqrt(bb);
    h->connected = true;
    return AJM_OK;
}

ajm_status_t ajm_group_solve(const ajm_handle_t* hs, int32_t nranks, const double* x0, double tol,
                             int64_t maxit, ajm_policy_t policy, double* x_out, ajm_result_t* res,
                             double* res_hist, double* f_hist, int64_t* restart_iters, int64_t restart_cap,
                             void* cuda_stream) {
    NvtxScope nvtx_scope_("ajm_group_solve");
    if (!hs || nranks < 1 || nranks > AJM_MAX_RANKS || !hs[0]) return fail(nullptr, AJM_ERR_INVALID_ARG, "bad handle array");
    ajm_ctx* h0 = hs[0];
    for (int r = 0; r < nranks; ++r) {
        ajm_ctx* h = hs[r];
        if (!h || !h->shard || !h->colocated || h->rank != r || h->nranks != nranks)
            return fail(h0, AJM_ERR_INVALID_ARG, "handle %d is not rank %d of an AJM_SHARD_COLOCATED group of %d", r, r, nranks);
        if (h->col_bytes != h0->col_bytes || h->pair != h0->pair || h->grid != h0->grid)
            return fail(h0, AJM_ERR_UNSUPPORTED, "ranks 0 and %d chose different column encodings / grids: one launch "
                        "cannot run both (create the group with AJM_INT32_COLUMNS)", r);
        ajm_status_t s = solve_check(h, x_out, tol, maxit, policy, restart_iters, restart_cap);
        if (s != AJM_OK) return s == AJM_OK ? s : fail(h0, s, "rank %d: %s", r, h->err_msg.c_str());
    }
    // ONE kernel for every rank: the segment phases if any rank has long rows, the deepest ring of
    // the ranks (each rank's tables sit behind the ring in shared memory)
    bool any_seg = false;
    int stages = 0;
    size_t meta = 0;
    for (int r = 0; r < nranks; ++r) {
        any_seg = any_seg || hs[r]->nseg > 0;
        stages = std::max(stages, hs[r]->ring_stages);
        meta = std::max(meta, hs[r]->meta_bytes);
    }
    if (h0->pair) stages = 4;
    else if (h0->col_bytes == 1) stages = std::max(4, std::min(5, stages));
    else stages = std::max(3, std::min(4, stages));
    const SolveFn gfn = shard_fn(h0->col_bytes, any_seg, stages, true, h0->pair != 0);
    const size_t gdyn = (size_t)stages * AJM_UNIT_EL * (h0->pair ? 1 : h0->col_bytes == 1 ? 9 : 12) + meta;
    cudaStream_t st = (cudaStream_t)cuda_stream;
    for (int r = 0; r < nranks; ++r) {
        ajm_ctx* h = hs[r];
        ajm_status_t s = solve_prep(h, x0 ? x0 + h->row0 : nullptr, tol, maxit, policy, st);
        if (s != AJM_OK) return fail(h0, s, "rank %d: %s", r, h->err_msg.c_str());
    }
    std::vector<AjmPass> ps((size_t)nranks);
    for (int r = 0; r < nranks; ++r) ps[(size_t)r] = make_pass(hs[r], (int)(maxit + 1));
    if (!h0->emu) AJM_CUDA(h0, cudaMalloc((void**)&h0->emu, sizeof(AjmPass) * AJM_MAX_RANKS));
    AJM_CUDA(h0, cudaMemcpyAsync(h0->emu, ps.data(), sizeof(AjmPass) * nranks, cudaMemcpyHostToDevice, st));
    AjmPass p = ps[0];
    p.sh.emu = h0->emu;
    p.sh.emu_grid = h0->grid;
    AJM_CUDA(h0, cudaStreamSynchronize(st));  // ps lives until the copy has run
    AJM_CUDA(h0, cudaEventRecord(h0->ev0, st));
    {
        std::lock_guard<std::mutex> lock(g_attr_mu);
        int occ = 0;
        cudaError_t e = fn_occupancy(gfn, gdyn, 100, &occ, block_threads(any_seg));
        if (e == cudaSuccess && (int64_t)occ * h0->sm_count < (int64_t)h0->grid * nranks)
            return fail(h0, AJM_ERR_UNSUPPORTED, "the group's %d CTAs cannot be co-resident (%d per SM)", h0->grid * nranks, occ);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(h0->grid * nranks));
        cfg.blockDim = dim3(block_threads(any_seg));
        cfg.dynamicSmemBytes = gdyn;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;  // every rank's CTAs co-resident
        at[0].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, gfn, p);
        AJM_CUDA(h0, e);
    }
    AJM_CUDA(h0, cudaEventRecord(h0->ev1, st));
    AJM_CUDA(h0, cudaEventSynchronize(h0->ev1));
    float ms = 0.f;
    AJM_CUDA(h0, cudaEventElapsedTime(&ms, h0->ev0, h0->ev1));
    // every rank took the same decisions: its own control block says so
    ajm_result_t r0res = {};
    for (int r = 0; r < nranks; ++r) {
        ajm_ctx* h = hs[r];
        ajm_result_t rr = {};
        ajm_status_t s = solve_post(h, 1, ms, x_out + h->row0, &rr, r == 0 ? res_hist : nullptr, r == 0 ? f_hist : nullptr,
                                    r == 0 ? restart_iters : nullptr, restart_cap, st);
        if (s != AJM_OK) return fail(h0, s, "rank %d: %s", r, h->err_msg.c_str());
        if (r == 0) r0res = rr;
        else if (rr.iterations != r0res.iterations || rr.status != r0res.status || rr.n_restarts != r0res.n_restarts ||
                 memcmp(&rr.rel_residual, &r0res.rel_residual, sizeof(double)) != 0)
            return fail(h0, AJM_ERR_CUDA, "rank %d's control decisions differ from rank 0's (internal error)", r);
    }
    if (res) *res = r0res;
    return AJM_OK;
}

ajm_status_t ajm_estimate_spectrum(ajm_handle_t h, const double* v0, uint64_t seed, int64_t max_steps,
                                   double tol, ajm_spectrum_t* out, double* alpha, double* beta,
                                   void* cuda_stream) {
    NvtxScope nvtx_scope_("ajm_estimate_spectrum");
    if (!h) return fail(nullptr, AJM_ERR_INVALID_ARG, "NULL handle");
    h->err_msg.clear();
    if (!out) return fail(h, AJM_ERR_INVALID_ARG, "out is NULL");
    if (max_steps < 1 || max_steps > (1 << 20)) return fail(h, AJM_ERR_INVALID_ARG, "max_steps must be in [1, 2^20]");
    if (!(tol >= 0.0)) return fail(h, AJM_ERR_INVALID_ARG, "tol must be >= 0");
    if (!h->fn_lz)
        return fail(h, AJM_ERR_UNSUPPORTED, "no Lanczos pass for this layout (block-J handles, experiment ring depths)");
    cudaStream_t st = (cudaStream_t)cuda_stream;
    const int64_t n = h->n;
    const size_t np = (size_t)h->n_pad;
    if (!h->lzw) AJM_CUDA(h, dalloc(&h->lzw, 8 * np, st));
    AJM_CUDA(h, cudaMemsetAsync(h->lzw, 0, sizeof(double) * 8 * np, st));
    double* Lg0 = h->lzw + 6 * np;
    // start vector (internal order)
    if (v0) {
        const cudaMemcpyKind k = kind_to_device(v0);
        if (h->relabel) {
            AJM_CUDA(h, cudaMemcpyAsync(h->lzw + 7 * np, v0, sizeof(double) * n, k, st));
            ajm_gather_kernel<<<1024, 256, 0, st>>>(n, h->perm_fwd, h->lzw + 7 * np, Lg0);
            AJM_CUDA(h, cudaGetLastError());
        } else {
            AJM_CUDA(h, cudaMemcpyAsync(Lg0, v0, sizeof(double) * n, k, st));
        }
        AJM_CUDA(h, cudaMemsetAsync(h->err, 0, sizeof(int), st));
        ajm_finite_kernel<<<1024, 256, 0, st>>>(n, Lg0, h->err);
        AJM_CUDA(h, cudaGetLastError());
        int herr = 0;
        AJM_CUDA(h, cudaMemcpyAsync(&herr, h->err, sizeof(int), cudaMemcpyDeviceToHost, st));
        AJM_CUDA(h, cudaStreamSynchronize(st));
        if (herr) return fail(h, AJM_ERR_NONFINITE, "v0 has a non-finite entry");
        AJM_CUDA(h, cudaMemsetAsync(h->lzw + 7 * np, 0, sizeof(double) * np, st));
    } else {
        ajm_start_vector_kernel<<<1024, 256, 0, st>>>(n, h->relabel ? h->perm_fwd : nullptr, seed, Lg0);
        AJM_CUDA(h, cudaGetLastError());
    }
    // steps: step 0 normalises the start, step j >= 1 is Lanczos step j (an SpMV pass for alpha_j
    // and a vector pass for beta_j); T_k needs k + 1 steps (alpha_1..alpha_k and beta_1..beta_k, the
    // last one for the residual bounds)
    const int64_t passes = max_steps + 1;  // Lanczos steps
    {
        const ajm_status_t hs = ensure_hist(h, passes + 2, st);
        if (hs != AJM_OK) return hs;
    }
    double* ha = h->hist;                 // alpha_{t+1} at [t]
    double* hb = h->hist + h->hist_cap;   // beta_t at [t] (t = 0: ||v0||_D)
    if (h->nsplit) AJM_CUDA(h, cudaMemsetAsync(h->split_cnt, 0, sizeof(unsigned) * h->nsplit, st));
    ajm_init_lanczos_kernel<<<1, 32, 0, st>>>(h->ctrl, passes, ha, hb, h->hist + 2 * h->hist_cap,
                                              h->hist + 3 * h->hist_cap);
    AJM_CUDA(h, cudaGetLastError());
    AjmPass p = make_pass(h, 0);
    p.Lp0 = h->lzw;
    p.Lp1 = h->lzw + np;
    p.Lp2 = h->lzw + 2 * np;
    p.Lq = h->lzw + 3 * np;
    p.Lv = Lg0;
    std::vector<double> va, vb;
    int64_t done_passes = 0, chunk = 32;
    int64_t kchk = 0;    // beta_1 .. beta_kchk checked for a (numerical) breakdown
    double tnorm = 0.0;  // max |alpha_i|, beta_i seen so far (the scale of T_k)
    ajm_spectrum_t r = {};
    AJM_CUDA(h, cudaEventRecord(h->ev0, st));
    int64_t launches = 0;
    for (;;) {
        // a chunk of steps (two passes each) in one persistent launch; the state continues across
        // launches
        p.max_passes = (int)(2 * std::min<int64_t>(chunk, passes - done_passes + 1));
        AJM_CUDA(h, launch_solver(h, p, st, h->fn_lz));
        ++launches;
        AJM_CUDA(h, cudaMemcpyAsync(h->h_ctrl, h->ctrl, sizeof(AjmCtrl), cudaMemcpyDeviceToHost, st));
        AJM_CUDA(h, cudaStreamSynchronize(st));
        const AjmCtrl& c = *h->h_ctrl;
        if (c.timeout_flag) return fail(h, AJM_ERR_CUDA, "device barrier wait timed out (internal error)");
        done_passes = c.s.iterations;
        va.resize((size_t)done_passes);
        vb.resize((size_t)done_passes);
        AJM_CUDA(h, cudaMemcpy(va.data(), ha, sizeof(double) * done_passes, cudaMemcpyDeviceToHost));
        AJM_CUDA(h, cudaMemcpy(vb.data(), hb, sizeof(double) * done_passes, cudaMemcpyDeviceToHost));
        if (c.s.done && c.s.status == 2) return fail(h, AJM_ERR_NONFINITE, "non-finite Lanczos coefficient");
        bool breakdown = c.s.done && c.s.status == 0;  // beta = 0: invariant subspace
        // T_k: alpha_1..alpha_k = va[0..k), beta_1..beta_{k-1} = vb[1..k), residual coefficient
        // beta_k = vb[k] (0 at a breakdown)
        int k = (int)(breakdown ? done_passes : done_passes - 1);
        // a NUMERICAL breakdown -- beta_k at rounding level against ||T_k|| (the Krylov space is
        // invariant: e.g. the §4.1 matrix has two distinct eigenvalues) -- ends the run at T_k: the
        // steps after it are rounding noise without reorthogonalisation, not more information
        for (int64_t kk = kchk + 1; kk < done_passes && !breakdown; ++kk) {
            tnorm = std::max(tnorm, std::fabs(va[(size_t)kk - 1]));
            if (kk >= 2) tnorm = std::max(tnorm, vb[(size_t)kk - 1]);
            if (vb[(size_t)kk] <= 1e-12 * tnorm) {
                breakdown = true;
                k = (int)kk;
            }
            kchk = kk;
        }
        if (k >= 1) {
            std::vector<double> ta(va.begin(), va.begin() + k), tb;
            for (int i = 1; i < k; ++i) tb.push_back(vb[(size_t)i]);
            tb.push_back(0.0);
            const double bk = (breakdown && (int64_t)k >= done_passes) ? 0.0 : vb[(size_t)k];
            const double lmin = tri_eig(ta, tb, k, 0), lmax = tri_eig(ta, tb, k, k - 1);
            r.lambda_min = lmin;
            r.lambda_max = lmax;
            r.err_min = bk * tri_last_component(ta, tb, k, lmin);
            r.err_max = bk * tri_last_component(ta, tb, k, lmax);
            r.steps = k;
            r.breakdown = breakdown ? 1 : 0;
            const double scale = std::max(std::fabs(lmax), std::fabs(lmin));
            r.converged = (r.err_min <= tol * scale && r.err_max <= tol * scale) ? 1 : 0;
            r.omega_opt = 2.0 / (lmin + lmax);
            if (r.converged || breakdown) break;
        }
        if (c.s.done || done_passes >= passes) break;
        chunk = std::min<int64_t>(2 * chunk, 1024);
    }
    AJM_CUDA(h, cudaEventRecord(h->ev1, st));
    AJM_CUDA(h, cudaEventSynchronize(h->ev1));
    float ms = 0.f;
    AJM_CUDA(h, cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    h->last_loop_ms = ms;
    h->last_passes = done_passes;
    h->last_launches = launches;
    const int64_t kk = std::min<int64_t>(r.steps, done_passes);
    if (alpha) for (int64_t i = 0; i < kk; ++i) alpha[i] = va[(size_t)i];
    if (beta) for (int64_t i = 0; i < kk; ++i) beta[i] = (size_t)i + 1 < vb.size() ? vb[(size_t)i + 1] : 0.0;
    *out = r;
    return AJM_OK;
}

ajm_status_t ajm_get_trace(ajm_handle_t h, int32_t which, double* out, int64_t count) {
    if (!h) return fail(nullptr, AJM_ERR_INVALID_ARG, "NULL handle");
    if (which < 0 || which > 3 || !out || count < 0)
        return fail(h, AJM_ERR_INVALID_ARG, "bad trace request");
    if (h->last_iterations < 0 || count > h->last_iterations + 1)
        return fail(h, AJM_ERR_INVALID_ARG, "count exceeds iterations + 1 of the last solve");
    AJM_CUDA(h, cudaMemcpy(out, h->hist + (size_t)which * h->hist_cap, sizeof(double) * count,
                           kind_from_device(out)));
    return AJM_OK;
}

ajm_status_t ajm_get_diag(ajm_handle_t h, double* out) {
    if (!h || !out) return fail(h, AJM_ERR_INVALID_ARG, "NULL argument");
    if (h->relabel) {
        double* tmp = nullptr;
        AJM_CUDA(h, dalloc(&tmp, h->n, (cudaStream_t)0));
        ajm_gather_kernel<<<1024, 256>>>(h->n, h->perm_inv, h->D, tmp);
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaMemcpy(out, tmp, sizeof(double) * h->n, kind_from_device(out));
        dfree(tmp);
        AJM_CUDA(h, e);
        return AJM_OK;
    }
    AJM_CUDA(h, cudaMemcpy(out, h->D, sizeof(double) * h->n, kind_from_device(out)));
    return AJM_OK;
}

ajm_status_t ajm_get_jblock(ajm_handle_t h, double* out) {
    if (!h || !out) return fail(h, AJM_ERR_INVALID_ARG, "NULL argument");
    if (!h->jbs) return fail(h, AJM_ERR_INVALID_ARG, "handle was not created with AJM_D_JBLOCK");
    const size_t cnt = (size_t)((h->n + h->jbs - 1) / h->jbs) * h->jbs * h->jbs;
    AJM_CUDA(h, cudaMemcpy(out, h->Jblk, sizeof(double) * cnt, kind_from_device(out)));
    return AJM_OK;
}

ajm_status_t ajm_get_info(ajm_handle_t h, ajm_info_t* info) {
    if (!h || !info) return fail(h, AJM_ERR_INVALID_ARG, "NULL argument");
    info->n = h->n;
    info->nnz = h->nnz;
    info->units = h->nunits + h->nseg;
    info->long_rows = h->long_rows;
    info->grid = h->grid;
    info->block = AJM_BLOCK;
    info->sm_count = h->sm_count;
    info->ctas_per_sm = h->ctas_per_sm;
    // the diagonal D (8 B/row) is replaced by bs doubles per row of J^{-1} for AJM_D_JBLOCK
    info->model_bytes_per_iter = 12.0 * (double)h->nnz + (48.0 + 8.0 * (h->jbs ? h->jbs : 1)) * (double)h->n +
                                 4.0 * (double)(h->n + 1);
    info->last_loop_ms = h->last_loop_ms;
    info->last_passes = h->last_passes;
    info->last_launches = h->last_launches;
    info->sell_rows = h->n_sell;
    info->seg_rows = h->seg_rows;
    info->split_rows = h->nsplit;
    info->sigma = h->sigma;
    info->variant = h->nseg > 0 ? 1 : 0;  // 1: no producer warp, 128 registers (layouts with segments)
    info->l2_window_bytes = (int64_t)h->win_bytes;
    info->l2_hit_ratio = h->win_hit;
    info->mode = h->resident ? 6 : (h->cluster ? 5 : 0);
    info->sell_elems = h->sell_elems;
    info->l2_mode = h->l2_mode;
    info->launches_per_solve = (int32_t)(1 + (h->prime_bytes ? 1 : 0) + std::max<int64_t>(h->last_launches, 1));
    info->col_bytes = h->col_bytes;
    info->val_bytes = h->pair ? 0 : 8;
    info->band_staged = h->band;
    info->seg_nnz = h->seg_nnz;
    info->rank = h->rank;
    info->nranks = h->nranks;
    info->halo = h->h_lo + h->h_hi;
    info->send = (int64_t)h->snd_host.size();
    info->group_rows = h->grp_rows;
    return AJM_OK;
}

ajm_status_t ajm_destroy(ajm_handle_t h) {
    NvtxScope nvtx_scope_("ajm_destroy");
    if (!h) return AJM_OK;
    free_all(h);
    delete h;
    return AJM_OK;
}

}  // extern "C"
