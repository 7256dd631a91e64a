// ajm.cu -- host runtime + C ABI (include/ajm.h) of the B200-native AJM solver.
//
// create : validate (host row_ptr scan + device column/value kernel, optional symmetry kernel),
//          D per dmode (eq-J-diag on the device), ||b|| (deterministic two-level
//          reduction), and the row-length-binned layout:
//            rows <= AJM_SELL_MAX nonzeros -> SELL-32-sigma chunks (sigma = 1 when natural order
//              pads < 5%, else rows sorted by length inside windows of 4096), thread per row;
//            rows <= AJM_WARP_MAX -> warp per row;  longer rows -> CTA per row;
//          on a persistent grid of (#SMs x resident CTAs/SM) CTAs: long rows spread largest-first
//          onto the least-loaded CTA, then mid rows and chunks in contiguous cost-balanced ranges.
// solve  : init kernel -> one CUDA-graph launch whose WHILE conditional node re-runs the fused
//          pass until the last CTA's finalize clears the condition (no host round trip per
//          iteration) -> copy-out of the answer buffer, histories and the control block.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ajm.h"
#include "ajm_kernels.cuh"

namespace {

thread_local std::string g_create_error;

typedef void (*PassFn)(AjmPass);
struct PassVariant {
    PassFn ident, general;
    const char* name;
};
// SELL batch depth x min resident CTAs per SM (register budget); AJM_KVARIANT selects (tuning)
const PassVariant kVariants[] = {
    {ajm_pass_kernel<true, 8, 3>, ajm_pass_kernel<false, 8, 3>, "b8m3"},
    {ajm_pass_kernel<true, 8, 2>, ajm_pass_kernel<false, 8, 2>, "b8m2"},
    {ajm_pass_kernel<true, 6, 4>, ajm_pass_kernel<false, 6, 4>, "b6m4"},
    {ajm_pass_kernel<true, 4, 4>, ajm_pass_kernel<false, 4, 4>, "b4m4"},
};
const int kNumVariants = sizeof(kVariants) / sizeof(kVariants[0]);

}  // namespace

struct ajm_ctx {
    int device = 0;
    int sm_count = 0;
    int ctas_per_sm = 0;
    int64_t n = 0, nnz = 0;
    int64_t units = 0, long_rows = 0, mid_rows_n = 0, nchunks = 0, n_sell = 0;
    int64_t sell_elems = 0;
    int sigma = 1;
    bool ident = true;
    int variant = 0;
    PassFn pass = nullptr;
    int grid = 0;
    uint32_t flags = 0;
    // device arrays
    int* rp = nullptr;
    int* col = nullptr;
    double* val = nullptr;
    double* b = nullptr;
    double* D = nullptr;
    double* X[3] = {nullptr, nullptr, nullptr};
    double* Qxp = nullptr;
    double* sval = nullptr;
    int* scol = nullptr;
    long long* chunk_off = nullptr;
    int* perm = nullptr;
    int* mid_rows = nullptr;
    int* long_rows_d = nullptr;
    int* cta_chunk = nullptr;
    int* cta_mid = nullptr;
    int* cta_long = nullptr;
    double* partials = nullptr;
    AjmCtrl* ctrl = nullptr;
    double* hist = nullptr;  // 4 x hist_cap: res, f, d, dabs
    int64_t hist_cap = 0;
    double* scratch = nullptr;  // reductions at create
    int* err = nullptr;
    AjmCtrl* h_ctrl = nullptr;  // pinned
    double nb = 0.0;
    // graph
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t graph_exec = nullptr;
    cudaGraphConditionalHandle cond = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    double last_loop_ms = 0.0;
    int64_t last_passes = 0;
    int64_t last_graph_launches = 0;
    int64_t last_iterations = -1;
    std::string err_msg;
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

template <class T>
cudaError_t dalloc(T** p, size_t count) {
    return cudaMalloc((void**)p, std::max<size_t>(count, 1) * sizeof(T));
}

void free_all(ajm_ctx* h) {
    if (h->graph_exec) cudaGraphExecDestroy(h->graph_exec);
    if (h->graph) cudaGraphDestroy(h->graph);
    void* ptrs[] = {h->rp, h->col, h->val, h->b, h->D, h->X[0], h->X[1], h->X[2], h->Qxp,
                    h->sval, h->scol, h->chunk_off, h->perm, h->mid_rows, h->long_rows_d,
                    h->cta_chunk, h->cta_mid, h->cta_long, h->partials, h->ctrl, h->hist,
                    h->scratch, h->err};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    if (h->h_ctrl) cudaFreeHost(h->h_ctrl);
    if (h->ev0) cudaEventDestroy(h->ev0);
    if (h->ev1) cudaEventDestroy(h->ev1);
}

AjmPass make_pass(ajm_ctx* h, int use_cond) {
    AjmPass p;
    p.rp = h->rp;
    p.col = h->col;
    p.val = h->val;
    p.b = h->b;
    p.D = h->D;
    p.X0 = h->X[0];
    p.X1 = h->X[1];
    p.X2 = h->X[2];
    p.Qxp = h->Qxp;
    p.sval = h->sval;
    p.scol = h->scol;
    p.chunk_off = h->chunk_off;
    p.perm = h->perm;
    p.mid_rows = h->mid_rows;
    p.long_rows = h->long_rows_d;
    p.cta_chunk = h->cta_chunk;
    p.cta_mid = h->cta_mid;
    p.cta_long = h->cta_long;
    p.n_sell = (int)h->n_sell;
    p.partials = h->partials;
    p.ctrl = h->ctrl;
    p.cond = h->cond;
    p.use_cond = use_cond;
    p.n = (int)h->n;
    return p;
}

ajm_status_t build_graph(ajm_ctx* h) {
    AJM_CUDA(h, cudaGraphCreate(&h->graph, 0));
    AJM_CUDA(h, cudaGraphConditionalHandleCreate(&h->cond, h->graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h->cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    AJM_CUDA(h, cudaGraphAddNode(&cnode, h->graph, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    AjmPass p = make_pass(h, 1);
    void* args[] = {&p};
    cudaKernelNodeParams kp = {};
    kp.func = (void*)h->pass;
    kp.gridDim = dim3(h->grid);
    kp.blockDim = dim3(AJM_BLOCK);
    kp.sharedMemBytes = 0;
    kp.kernelParams = args;
    cudaGraphNode_t knode;
    AJM_CUDA(h, cudaGraphAddKernelNode(&knode, body, nullptr, 0, &kp));
    AJM_CUDA(h, cudaGraphInstantiate(&h->graph_exec, h->graph, 0));
    return AJM_OK;
}

ajm_status_t ensure_hist(ajm_ctx* h, int64_t need) {
    if (need <= h->hist_cap) return AJM_OK;
    if (h->hist) {
        AJM_CUDA(h, cudaFree(h->hist));
        h->hist = nullptr;
    }
    int64_t cap = std::max<int64_t>(need, 1024);
    AJM_CUDA(h, dalloc(&h->hist, (size_t)cap * 4));
    h->hist_cap = cap;
    return AJM_OK;
}

}  // namespace

extern "C" {

int32_t ajm_abi_version(void) { return AJM_ABI_VERSION; }

const char* ajm_last_error(ajm_handle_t h) {
    return h ? h->err_msg.c_str() : g_create_error.c_str();
}

ajm_status_t ajm_create(ajm_handle_t* out, int64_t n, int64_t nnz, const int64_t* row_ptr,
                        const int32_t* col_idx, const double* vals, const double* b, int32_t dmode,
                        const double* d, uint32_t flags, void* cuda_stream) {
    g_create_error.clear();
    if (!out) return fail(nullptr, AJM_ERR_INVALID_ARG, "out is NULL");
    if (n < 1 || nnz < 0) return fail(nullptr, AJM_ERR_INVALID_ARG, "n must be >= 1 and nnz >= 0");
    if (n >= (int64_t)1 << 31 || nnz >= (int64_t)1 << 31)
        return fail(nullptr, AJM_ERR_UNSUPPORTED, "n and nnz must be < 2^31 (int32 device offsets)");
    if (!row_ptr || !b || (nnz > 0 && (!col_idx || !vals)))
        return fail(nullptr, AJM_ERR_INVALID_ARG, "NULL array argument");
    if (dmode < 0 || dmode > 2) return fail(nullptr, AJM_ERR_INVALID_ARG, "bad dmode %d", dmode);
    if (dmode == AJM_D_USER && !d) return fail(nullptr, AJM_ERR_INVALID_ARG, "AJM_D_USER needs d");
    cudaStream_t st = (cudaStream_t)cuda_stream;

    // host scan of row_ptr (needed anyway for the unit layout)
    std::vector<int64_t> hrp((size_t)n + 1);
    {
        cudaError_t e = cudaMemcpyAsync(hrp.data(), row_ptr, sizeof(int64_t) * (n + 1),
                                        is_device_ptr(row_ptr) ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return fail(nullptr, AJM_ERR_CUDA, "row_ptr copy: %s", cudaGetErrorString(e));
    }
    if (hrp[0] != 0) return fail(nullptr, AJM_ERR_CSR_INVALID, "row_ptr[0] = %lld != 0", (long long)hrp[0]);
    for (int64_t i = 0; i < n; ++i)
        if (hrp[i + 1] < hrp[i])
            return fail(nullptr, AJM_ERR_CSR_INVALID, "row_ptr decreases at row %lld", (long long)i);
    if (hrp[n] != nnz)
        return fail(nullptr, AJM_ERR_CSR_INVALID, "row_ptr[n] = %lld != nnz = %lld", (long long)hrp[n], (long long)nnz);

    ajm_ctx* h = new ajm_ctx();
    h->n = n;
    h->nnz = nnz;
    h->flags = flags;
    auto bail = [&](ajm_status_t s) {
        g_create_error = h->err_msg;
        free_all(h);
        delete h;
        return s;
    };
#define CK(call)                                         \
    do {                                                 \
        ajm_status_t s__ = (call);                       \
        if (s__ != AJM_OK) return bail(s__);             \
    } while (0)
#define CC(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return bail(fail(h, e_ == cudaErrorMemoryAllocation ? AJM_ERR_OOM : AJM_ERR_CUDA,      \
                             "%s: %s", #call, cudaGetErrorString(e_)));                           \
    } while (0)

    CC(cudaGetDevice(&h->device));
    CC(cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, h->device));

    // ---- row-length-binned layout (host, O(n log sigma)) ----
    std::vector<int> perm_h, mid_h, long_h;
    std::vector<long long> choff;
    std::vector<double> chcost;
    {
        std::vector<int> short_rows;
        short_rows.reserve((size_t)n);
        for (int64_t i = 0; i < n; ++i) {
            const int64_t len = hrp[i + 1] - hrp[i];
            if (len <= AJM_SELL_MAX) short_rows.push_back((int)i);
            else if (len <= AJM_WARP_MAX) mid_h.push_back((int)i);
            else long_h.push_back((int)i);
        }
        auto rlen = [&](int r) { return hrp[r + 1] - hrp[r]; };
        auto padded = [&](const std::vector<int>& order) {
            int64_t tot = 0;
            for (size_t c0 = 0; c0 < order.size(); c0 += 32) {
                int64_t w = 1;
                for (size_t j = c0; j < std::min(order.size(), c0 + 32); ++j) w = std::max<int64_t>(w, rlen(order[j]));
                tot += 32 * w;
            }
            return tot;
        };
        int64_t short_nnz = 0;
        for (int r : short_rows) short_nnz += rlen(r);
        std::vector<int> order = short_rows;
        h->sigma = 1;
        if (!short_rows.empty() && (double)padded(order) > 1.05 * (double)std::max<int64_t>(short_nnz, 1)) {
            // sort by decreasing length inside windows of 4096 consecutive row indices (stable)
            h->sigma = 4096;
            size_t lo = 0;
            while (lo < order.size()) {
                const int wbase = order[lo] / h->sigma;
                size_t hi = lo;
                while (hi < order.size() && order[hi] / h->sigma == wbase) ++hi;
                std::stable_sort(order.begin() + lo, order.begin() + hi,
                                 [&](int x, int y) { return rlen(x) > rlen(y); });
                lo = hi;
            }
        }
        h->n_sell = (int64_t)order.size();
        h->nchunks = (h->n_sell + 31) / 32;
        h->ident = (h->sigma == 1 && mid_h.empty() && long_h.empty());
        perm_h.assign((size_t)h->nchunks * 32, -1);
        for (size_t j = 0; j < order.size(); ++j) perm_h[j] = order[j];
        choff.assign((size_t)h->nchunks + 1, 0);
        chcost.assign((size_t)h->nchunks, 0.0);
        for (int64_t c = 0; c < h->nchunks; ++c) {
            int64_t w = 1, rows = 0;
            for (int64_t j = c * 32; j < std::min<int64_t>(h->n_sell, c * 32 + 32); ++j) {
                w = std::max<int64_t>(w, rlen(order[(size_t)j]));
                ++rows;
            }
            choff[(size_t)c + 1] = choff[(size_t)c] + 32 * w;
            chcost[(size_t)c] = 12.0 * 32 * w + 56.0 * rows;
        }
        h->sell_elems = choff.back();
        if (h->sell_elems >= ((int64_t)1 << 40)) return bail(fail(h, AJM_ERR_UNSUPPORTED, "SELL layout too large"));
        h->mid_rows_n = (int64_t)mid_h.size();
        h->long_rows = (int64_t)long_h.size();
        h->units = h->nchunks + h->mid_rows_n + h->long_rows;
    }
    std::vector<int> cta_chunk, cta_mid, cta_long, long_sorted;
    {
        if (const char* ev = getenv("AJM_KVARIANT")) h->variant = std::max(0, std::min(kNumVariants - 1, atoi(ev)));
        h->pass = h->ident ? kVariants[h->variant].ident : kVariants[h->variant].general;
        int occ = 0;
        CC(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, h->pass, AJM_BLOCK, 0));
        h->ctas_per_sm = std::max(occ, 1);
        const int64_t g = (int64_t)h->sm_count * h->ctas_per_sm;
        // at least ~8 work items per CTA (one per warp) before adding CTAs
        const int64_t want = std::max<int64_t>(1, (h->nchunks + h->mid_rows_n) / 8 + h->long_rows);
        h->grid = (int)std::max<int64_t>(1, std::min<int64_t>(g, want));
        const int G = h->grid;
        std::vector<double> load((size_t)G, 0.0);
        // long rows: largest first onto the least-loaded CTA (LPT)
        std::vector<int> lr = long_h;
        std::stable_sort(lr.begin(), lr.end(), [&](int x, int y) { return hrp[x + 1] - hrp[x] > hrp[y + 1] - hrp[y]; });
        std::vector<std::vector<int>> per((size_t)G);
        for (int r : lr) {
            size_t best = 0;
            for (size_t c = 1; c < (size_t)G; ++c)
                if (load[c] < load[best]) best = c;
            load[best] += 12.0 * (double)(hrp[r + 1] - hrp[r]) + 56.0;
            per[best].push_back(r);
        }
        cta_long.assign((size_t)G + 1, 0);
        for (int c = 0; c < G; ++c) {
            cta_long[(size_t)c + 1] = cta_long[(size_t)c] + (int)per[(size_t)c].size();
            for (int r : per[(size_t)c]) long_sorted.push_back(r);
        }
        // mid rows then chunks as one sequence, contiguous ranges balancing total load
        const int64_t nm = h->mid_rows_n, nc = h->nchunks, nseq = nm + nc;
        auto cost = [&](int64_t i) {
            if (i < nm) { const int r = mid_h[(size_t)i]; return 12.0 * (double)(hrp[r + 1] - hrp[r]) + 56.0 + 256.0; }
            return chcost[(size_t)(i - nm)];
        };
        double total = 0.0;
        for (double l : load) total += l;
        for (int64_t i = 0; i < nseq; ++i) total += cost(i);
        const double target = total / G;
        std::vector<int64_t> start((size_t)G + 1, nseq);
        int64_t i = 0;
        for (int c = 0; c < G; ++c) {
            start[(size_t)c] = i;
            double acc = load[(size_t)c];
            if (c == G - 1) { i = nseq; break; }
            while (i < nseq && acc + 0.5 * cost(i) < target) acc += cost(i++);
        }
        start[(size_t)G] = nseq;
        cta_mid.assign((size_t)G + 1, 0);
        cta_chunk.assign((size_t)G + 1, 0);
        for (int c = 0; c <= G; ++c) {
            cta_mid[(size_t)c] = (int)std::min(start[(size_t)c], nm);
            cta_chunk[(size_t)c] = (int)std::max<int64_t>(start[(size_t)c] - nm, 0);
        }
    }

    // ---- device allocations ----
    CC(dalloc(&h->rp, n + 1));
    CC(dalloc(&h->col, nnz));
    CC(dalloc(&h->val, nnz));
    CC(dalloc(&h->b, n));
    CC(dalloc(&h->D, n));
    for (int k = 0; k < 3; ++k) CC(dalloc(&h->X[k], n));
    CC(dalloc(&h->Qxp, n));
    CC(dalloc(&h->sval, h->sell_elems));
    CC(dalloc(&h->scol, h->sell_elems));
    CC(dalloc(&h->chunk_off, h->nchunks + 1));
    CC(dalloc(&h->perm, h->nchunks * 32));
    CC(dalloc(&h->mid_rows, h->mid_rows_n));
    CC(dalloc(&h->long_rows_d, h->long_rows));
    CC(dalloc(&h->cta_chunk, h->grid + 1));
    CC(dalloc(&h->cta_mid, h->grid + 1));
    CC(dalloc(&h->cta_long, h->grid + 1));
    CC(dalloc(&h->partials, (size_t)h->grid * AJM_NPART));
    CC(dalloc(&h->ctrl, 1));
    CC(dalloc(&h->scratch, 512));
    CC(dalloc(&h->err, 1));
    CC(cudaMallocHost((void**)&h->h_ctrl, sizeof(AjmCtrl)));
    CC(cudaEventCreate(&h->ev0));
    CC(cudaEventCreate(&h->ev1));

    // ---- copies ----
    {
        int64_t* rp64 = nullptr;
        CC(dalloc(&rp64, n + 1));
        CC(cudaMemcpyAsync(rp64, hrp.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, st));
        ajm_rowptr_narrow_kernel<<<1024, 256, 0, st>>>(n + 1, (const long long*)rp64, h->rp);
        CC(cudaGetLastError());
        CC(cudaStreamSynchronize(st));
        cudaFree(rp64);
    }
    if (nnz > 0) {
        CC(cudaMemcpyAsync(h->col, col_idx, sizeof(int32_t) * nnz, kind_to_device(col_idx), st));
        CC(cudaMemcpyAsync(h->val, vals, sizeof(double) * nnz, kind_to_device(vals), st));
    }
    CC(cudaMemcpyAsync(h->b, b, sizeof(double) * n, kind_to_device(b), st));
    double* dtmp = nullptr;
    if (dmode == AJM_D_USER) {
        CC(dalloc(&dtmp, n));
        CC(cudaMemcpyAsync(dtmp, d, sizeof(double) * n, kind_to_device(d), st));
    }
    auto h2d = [&](void* dst, const void* src, size_t bytes) {
        return bytes ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st) : cudaSuccess;
    };
    CC(h2d(h->chunk_off, choff.data(), sizeof(long long) * choff.size()));
    CC(h2d(h->perm, perm_h.data(), sizeof(int) * perm_h.size()));
    CC(h2d(h->mid_rows, mid_h.data(), sizeof(int) * mid_h.size()));
    CC(h2d(h->long_rows_d, long_sorted.data(), sizeof(int) * long_sorted.size()));
    CC(h2d(h->cta_chunk, cta_chunk.data(), sizeof(int) * cta_chunk.size()));
    CC(h2d(h->cta_mid, cta_mid.data(), sizeof(int) * cta_mid.size()));
    CC(h2d(h->cta_long, cta_long.data(), sizeof(int) * cta_long.size()));
    CC(cudaMemsetAsync(h->err, 0, sizeof(int), st));

    // ---- validation + D (device) ----
    const int nblk = (int)((n + 255) / 256);
    ajm_validate_diag_kernel<<<nblk, 256, 0, st>>>((int)n, h->rp, h->col, h->val, dmode, dtmp, h->D, h->err);
    CC(cudaGetLastError());
    ajm_finite_kernel<<<1024, 256, 0, st>>>(n, h->b, h->err);
    CC(cudaGetLastError());
    int herr = 0;
    CC(cudaMemcpyAsync(&herr, h->err, sizeof(int), cudaMemcpyDeviceToHost, st));
    CC(cudaStreamSynchronize(st));
    if (dtmp) cudaFree(dtmp);
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
    // SELL copy of the short rows
    if (h->nchunks > 0) {
        const int ns = (int)(h->nchunks * 32);
        ajm_sell_fill_kernel<<<(ns + 255) / 256, 256, 0, st>>>(ns, (int)h->n_sell, h->perm, h->ident ? 1 : 0,
                                                               h->rp, h->col, h->val, h->chunk_off, h->sval, h->scol);
        CC(cudaGetLastError());
    }
    // ||b||
    ajm_sumsq_partial_kernel<<<256, 256, 0, st>>>(n, h->b, h->scratch);
    ajm_sum_final_kernel<<<1, 32, 0, st>>>(256, h->scratch, h->scratch + 256);
    CC(cudaGetLastError());
    double bb = 0.0;
    CC(cudaMemcpyAsync(&bb, h->scratch + 256, sizeof(double), cudaMemcpyDeviceToHost, st));
    CC(cudaStreamSynchronize(st));
    if (!(bb > 0.0)) return bail(fail(h, AJM_ERR_ZERO_RHS, "||b|| = 0: relative residual undefined"));
    h->nb = std::sqrt(bb);
    if (!(flags & AJM_LOOP_HOST)) CK(build_graph(h));
    *out = h;
#undef CK
#undef CC
    return AJM_OK;
}

ajm_status_t ajm_solve(ajm_handle_t h, const double* x0, double tol, int64_t maxit,
                       ajm_policy_t policy, double* x_out, ajm_result_t* res, double* res_hist,
                       double* f_hist, int64_t* restart_iters, int64_t restart_cap,
                       void* cuda_stream) {
    if (!h) return fail(nullptr, AJM_ERR_INVALID_ARG, "NULL handle");
    h->err_msg.clear();
    if (!x_out) return fail(h, AJM_ERR_INVALID_ARG, "x_out is NULL");
    if (!(tol >= 0.0)) return fail(h, AJM_ERR_INVALID_ARG, "tol must be >= 0");
    if (maxit < 1) return fail(h, AJM_ERR_INVALID_ARG, "maxit must be >= 1");
    if (policy.k0 < 2) return fail(h, AJM_ERR_INVALID_ARG, "k0 must be >= 2 (P:460)");
    if (policy.restart && !policy.momentum)
        return fail(h, AJM_ERR_INVALID_ARG, "restart requires momentum (Alg. 2/3)");
    if (restart_iters && restart_cap < 0) return fail(h, AJM_ERR_INVALID_ARG, "restart_cap < 0");
    cudaStream_t st = (cudaStream_t)cuda_stream;
    const int64_t n = h->n;
    ajm_status_t s = ensure_hist(h, maxit + 2);
    if (s != AJM_OK) return s;

    // x~^0 = x0 and x^{-1} := x0 (beta_0 = 0 makes it unused); Q x^{-1} := 0 (finite, times 0)
    if (x0) {
        const cudaMemcpyKind k = kind_to_device(x0);
        AJM_CUDA(h, cudaMemcpyAsync(h->X[0], x0, sizeof(double) * n, k, st));
        AJM_CUDA(h, cudaMemsetAsync(h->err, 0, sizeof(int), st));
        ajm_finite_kernel<<<1024, 256, 0, st>>>(n, h->X[0], h->err);
        AJM_CUDA(h, cudaGetLastError());
        int herr = 0;
        AJM_CUDA(h, cudaMemcpyAsync(&herr, h->err, sizeof(int), cudaMemcpyDeviceToHost, st));
        AJM_CUDA(h, cudaStreamSynchronize(st));
        if (herr) return fail(h, AJM_ERR_NONFINITE, "x0 has a non-finite entry");
        AJM_CUDA(h, cudaMemcpyAsync(h->X[1], h->X[0], sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    } else {
        AJM_CUDA(h, cudaMemsetAsync(h->X[0], 0, sizeof(double) * n, st));
        AJM_CUDA(h, cudaMemsetAsync(h->X[1], 0, sizeof(double) * n, st));
    }
    AJM_CUDA(h, cudaMemsetAsync(h->Qxp, 0, sizeof(double) * n, st));
    double* hr = h->hist;
    double* hf = h->hist + h->hist_cap;
    double* hd = h->hist + 2 * h->hist_cap;
    double* hda = h->hist + 3 * h->hist_cap;
    ajm_init_ctrl_kernel<<<1, 32, 0, st>>>(h->ctrl, tol, maxit, policy.momentum ? 1 : 0,
                                           policy.restart ? 1 : 0, policy.k0, h->nb, hr, hf, hd, hda);
    AJM_CUDA(h, cudaGetLastError());

    AJM_CUDA(h, cudaEventRecord(h->ev0, st));
    int64_t launches = 0;
    if (h->graph_exec) {
        AJM_CUDA(h, cudaGraphLaunch(h->graph_exec, st));
        launches = 1;
    } else {
        // debug host loop: chunks of passes, each pass exits at once when the control block is done
        AjmPass p = make_pass(h, 0);
        int64_t issued = 0;
        for (;;) {
            const int64_t chunk = std::min<int64_t>(64, maxit + 1 - issued);
            for (int64_t i = 0; i < chunk; ++i) h->pass<<<h->grid, AJM_BLOCK, 0, st>>>(p);
            AJM_CUDA(h, cudaGetLastError());
            issued += chunk;
            AJM_CUDA(h, cudaMemcpyAsync(h->h_ctrl, h->ctrl, sizeof(AjmCtrl), cudaMemcpyDeviceToHost, st));
            AJM_CUDA(h, cudaStreamSynchronize(st));
            if (h->h_ctrl->done || issued >= maxit + 1) break;
        }
        launches = issued;
    }
    AJM_CUDA(h, cudaEventRecord(h->ev1, st));
    AJM_CUDA(h, cudaMemcpyAsync(h->h_ctrl, h->ctrl, sizeof(AjmCtrl), cudaMemcpyDeviceToHost, st));
    AJM_CUDA(h, cudaStreamSynchronize(st));
    const AjmCtrl& c = *h->h_ctrl;
    if (!c.done) return fail(h, AJM_ERR_CUDA, "iteration loop ended without a termination decision");
    float ms = 0.f;
    AJM_CUDA(h, cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    h->last_loop_ms = ms;
    h->last_passes = c.iterations + 1;
    h->last_graph_launches = launches;
    h->last_iterations = c.iterations;

    AJM_CUDA(h, cudaMemcpyAsync(x_out, h->X[c.answer], sizeof(double) * n, kind_from_device(x_out), st));
    const int64_t cnt = c.iterations + 1;
    if (res_hist) AJM_CUDA(h, cudaMemcpyAsync(res_hist, hr, sizeof(double) * cnt, kind_from_device(res_hist), st));
    if (f_hist) AJM_CUDA(h, cudaMemcpyAsync(f_hist, hf, sizeof(double) * cnt, kind_from_device(f_hist), st));
    AJM_CUDA(h, cudaStreamSynchronize(st));
    const int64_t nlog = std::min<int64_t>(c.nlogged, restart_iters ? restart_cap : 0);
    for (int64_t i = 0; i < nlog; ++i) restart_iters[i] = c.restart_log[i];
    if (res) {
        res->status = c.status;
        res->n_restarts = c.nres;
        res->iterations = c.iterations;
        res->rel_residual = c.res_last;
        res->f = c.f_last;
        res->x_is_prerestart = c.prerestart;
        res->restarts_logged = (int32_t)nlog;
    }
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
    AJM_CUDA(h, cudaMemcpy(out, h->D, sizeof(double) * h->n, kind_from_device(out)));
    return AJM_OK;
}

ajm_status_t ajm_get_info(ajm_handle_t h, ajm_info_t* info) {
    if (!h || !info) return fail(h, AJM_ERR_INVALID_ARG, "NULL argument");
    info->n = h->n;
    info->nnz = h->nnz;
    info->units = h->units;
    info->long_rows = h->long_rows;
    info->grid = h->grid;
    info->block = AJM_BLOCK;
    info->sm_count = h->sm_count;
    info->ctas_per_sm = h->ctas_per_sm;
    info->model_bytes_per_iter = 12.0 * (double)h->nnz + 56.0 * (double)h->n + 4.0 * (double)(h->n + 1);
    info->last_loop_ms = h->last_loop_ms;
    info->last_passes = h->last_passes;
    info->last_graph_launches = h->last_graph_launches;
    return AJM_OK;
}

ajm_status_t ajm_destroy(ajm_handle_t h) {
    if (!h) return AJM_OK;
    free_all(h);
    delete h;
    return AJM_OK;
}

}  // extern "C"
