// ajm_kernels.cuh -- sm_100a device code of the AJM hot path (arXiv 2407.03272, Alg. 3).
//
// One fused pass per iteration:
//   a2  SpMV  q = Q x~^t                     (Alg. 3 line 4 Q y^t via the identity below)
//   a3  partials of ||b - q||^2, <x~,q>, <b,x~>  (stopping rule P:505; f, eq-qp P:25-28)
//   a4  restart branch or Nesterov extrapolation (Alg. 3 lines 6-13):
//         restart_t: y = x^{t-1}, Qy = Q x^{t-1}
//         else     : y = x~ + beta_t (x~ - x^{t-1}),  Qy = q + beta_t (q - Q x^{t-1}),  Q x^t := q
//   a5  Jacobi-type step x~^{t+1} = y + (b - Qy) / D   (IEEE division)
//   a6  partials of d_{t+1} = <Qy - b, x~^{t+1} - x^t> and sum |terms|  (restart test P:465)
//   a7  last-CTA finalize: fixed-order reduction of the per-CTA partials, residual / f history,
//       stopping test, restart decision for t+1, alpha/beta schedule, buffer rotation, and the
//       CUDA-graph WHILE condition.  Deterministic: no floating-point atomics anywhere.
// Q is streamed from HBM exactly once per iteration; y and Qy are never stored.
//
// The translation unit is compiled with --fmad=false so that no multiply-add is contracted
// (R14): the per-row sums of rows with <= 32 nonzeros run sequentially in ascending
// column order from 0.0 exactly like the oracle's, and the elementwise update rounds like it.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define AJM_BLOCK 256
#define AJM_SELL_MAX 64     // rows up to this length go to SELL (thread per row)
#define AJM_WARP_MAX 8192    // rows up to this length: one warp per row; longer: one CTA per row
#define AJM_NPART 5       // rr, <x,q>, <b,x>, d, sum|d terms|
#define AJM_LOG_CAP 64

struct AjmCtrl {
    long long t;        // index of the iterate x~^t the current pass multiplies
    long long maxit;
    long long K;        // K_l (prohibition period)
    long long Kre;      // K_re
    double tol;
    double nb;          // ||b||_2
    double alpha;       // alpha_t of the iteration whose y the current pass forms (see finalize)
    double beta;        // beta_t used by the current pass
    int restart_t;      // restart decision for iteration t (applied by the current pass)
    int cur, prev, fre; // X buffer indices: x~^t, x^{t-1}, free (receives x~^{t+1})
    int momentum, restart_enabled;
    int done, status;
    long long iterations;
    int answer;         // buffer index holding the answer when done
    int prerestart;
    int nres, nlogged;
    unsigned int ticket;
    int pad0;
    double res_last, f_last;
    double* res_hist;
    double* f_hist;
    double* d_hist;
    double* dabs_hist;
    long long restart_log[AJM_LOG_CAP];
};

struct AjmPass {
    // CSR (rows longer than AJM_SELL_MAX: warp- and CTA-per-row work)
    const int* __restrict__ rp;       // int32 row offsets [n+1]
    const int* __restrict__ col;      // int32 [nnz]
    const double* __restrict__ val;   // [nnz]
    // SELL-32-sigma copy of the short rows (<= AJM_SELL_MAX nonzeros): chunk c holds 32 slots,
    // element k of slot l at chunk_off[c] + 32 k + l (column-major: a warp's loads are coalesced)
    const double* __restrict__ sval;
    const int* __restrict__ scol;
    const long long* __restrict__ chunk_off; // [nchunks+1]
    const int* __restrict__ perm;     // slot -> row (-1 for tail slots); unused when identity
    const int* __restrict__ mid_rows; // warp-per-row list, grouped by CTA
    const int* __restrict__ long_rows;// CTA-per-row list, grouped by CTA
    const int* __restrict__ cta_chunk;// [grid+1] chunk range of each CTA
    const int* __restrict__ cta_mid;  // [grid+1]
    const int* __restrict__ cta_long; // [grid+1]
    const double* __restrict__ b;     // [n]
    const double* __restrict__ D;     // [n]
    double* X0;
    double* X1;
    double* X2;
    double* Qxp;                      // Q x^{t-1} in, Q x^t out (in place per row)
    double* partials;                 // [grid * AJM_NPART]
    AjmCtrl* ctrl;
    cudaGraphConditionalHandle cond;
    int use_cond;
    int n;
    int n_sell;                       // slots holding a row
};

__device__ __forceinline__ double ajm_warp_sum(double v) {
    // xor butterfly: a + b == b + a in IEEE, so every lane ends with the same bits
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    return v;
}

struct AjmAcc {
    double rr, xq, bx, d, dabs;
};

// a3-a6 for one row i with q = (Q x~^t)_i; the five row operands are loaded by the caller
__device__ __forceinline__ void ajm_row_update(double* __restrict__ Qxp, double* __restrict__ xf,
                                               int i, double q, double bi, double Di, double xt,
                                               double xpi, double qxp, double beta, int restart_t,
                                               AjmAcc& a) {
    const double r = bi - q;
    a.rr += r * r;
    a.xq += xt * q;
    a.bx += bi * xt;
    double y, qy, xnow;
    if (!restart_t) {
        y = xt + beta * (xt - xpi);
        qy = q + beta * (q - qxp);
        Qxp[i] = q;
        xnow = xt;
    } else {
        y = xpi;
        qy = qxp;
        xnow = xpi;
    }
    const double xn = y + (bi - qy) / Di;
    xf[i] = xn;
    const double term = (qy - bi) * (xn - xnow);
    a.d += term;
    a.dabs += fabs(term);
}

__device__ __forceinline__ void ajm_row_epilogue(const AjmPass& p, int i, double q, double beta,
                                                 int restart_t, const double* __restrict__ xc,
                                                 const double* __restrict__ xp,
                                                 double* __restrict__ xf, AjmAcc& a) {
    ajm_row_update(p.Qxp, xf, i, q, __ldg(p.b + i), __ldg(p.D + i), __ldg(xc + i), __ldg(xp + i),
                   p.Qxp[i], beta, restart_t, a);
}

__device__ __forceinline__ double* ajm_sel(const AjmPass& p, int k) {
    return k == 0 ? p.X0 : (k == 1 ? p.X1 : p.X2);
}

// Fixed-order CTA reduction of the 5 accumulators; result valid in thread 0.
__device__ __forceinline__ void ajm_block_reduce(AjmAcc& a, double (*s_red)[AJM_NPART]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double v[AJM_NPART] = {a.rr, a.xq, a.bx, a.d, a.dabs};
#pragma unroll
    for (int j = 0; j < AJM_NPART; ++j) v[j] = ajm_warp_sum(v[j]);
    if (lane == 0) {
#pragma unroll
        for (int j = 0; j < AJM_NPART; ++j) s_red[warp][j] = v[j];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s[AJM_NPART] = {0, 0, 0, 0, 0};
        for (int w = 0; w < AJM_BLOCK / 32; ++w)
#pragma unroll
            for (int j = 0; j < AJM_NPART; ++j) s[j] += s_red[w][j];
        a.rr = s[0]; a.xq = s[1]; a.bx = s[2]; a.d = s[3]; a.dabs = s[4];
    }
}

// a7: executed by thread 0 of the last CTA with the grid-wide sums
__device__ void ajm_finalize_ctrl(const AjmPass& p, const double* tot) {
    AjmCtrl* c = p.ctrl;
    const long long t = c->t;
    const double res = sqrt(tot[0]) / c->nb;
    const double f = 0.5 * tot[1] - tot[2];
    c->res_hist[t] = res;
    c->f_hist[t] = f;
    c->d_hist[t + 1] = tot[3];
    c->dabs_hist[t + 1] = tot[4];
    c->res_last = res;
    c->f_last = f;
    int stop = 0;
    if (res <= c->tol) {  // stopping rule on x~^t before the restart logic (R5)
        c->status = 0;
        c->answer = c->cur;
        c->prerestart = (t >= 1) ? c->restart_t : 0;
        stop = 1;
    } else if (t >= 1 && !(res <= 1e8)) {  // divergence guard (R19), NaN included
        c->status = 2;
        c->answer = c->cur;
        stop = 1;
    } else {
        if (t >= 1 && c->restart_t) {  // the restart decided for t is executed now (counted here)
            c->nres += 1;
            if (c->nlogged < AJM_LOG_CAP) c->restart_log[c->nlogged++] = t;
        }
        if (t == c->maxit) {  // output the post-iteration x^t (R10)
            c->status = 1;
            c->answer = c->restart_t ? c->prev : c->cur;
            stop = 1;
        }
    }
    if (stop) {
        c->iterations = t;
        c->done = 1;
    } else {
        // restart decision for iteration t+1 (Alg. 3 line 5): d_{t+1} was formed by this pass
        const long long tn = t + 1;
        int rs = 0;
        if (c->restart_enabled && tn > c->Kre + c->K) rs = (tot[3] >= 0.0);  // tie restarts (R7)
        if (rs) {  // lines 6-10: K_re = t, K_{l+1} = 2 K_l, alpha_{t+1} = 1 (R9)
            c->Kre = tn;
            c->K = 2 * c->K;
            c->alpha = 1.0;
            c->beta = 0.0;
        } else {   // lines 12-13: alpha_{t+1} = (1 + sqrt(1 + 4 alpha_t^2))/2, beta_t = (alpha_t - 1)/alpha_{t+1}
            const double a = c->alpha;
            const double an = (1.0 + sqrt(1.0 + 4.0 * a * a)) / 2.0;
            c->beta = c->momentum ? (a - 1.0) / an : 0.0;
            c->alpha = an;
        }
        // rotate: x^t = x~^t unless iteration t restarted (then x^t = x^{t-1})
        const int cur = c->cur, prev = c->prev, fre = c->fre;
        if (!c->restart_t) {
            c->prev = cur;
            c->cur = fre;
            c->fre = prev;
        } else {
            c->cur = fre;
            c->fre = cur;
        }
        c->restart_t = rs;
        c->t = tn;
    }
    c->ticket = 0;
    if (p.use_cond) cudaGraphSetConditional(p.cond, stop ? 0u : 1u);
}

// The fused pass.  Persistent grid (#SMs x resident CTAs); CTA c owns, fixed at create time,
//   (1) long rows  cta_long[c]..   : the whole CTA per row (strided sums + fixed CTA tree),
//   (2) mid rows   cta_mid[c]..    : one warp per row (lane-strided sums + xor tree),
//   (3) SELL chunks cta_chunk[c].. : one warp per chunk, one thread per row, sequential
//       ascending-column sums (bitwise the oracle's per-row order).
// Every assignment is static, so per-CTA partials and hence all reductions are deterministic.
template <bool kIdent, int kBatch, int kMinCtas>
__global__ void __launch_bounds__(AJM_BLOCK, kMinCtas) ajm_pass_kernel(AjmPass p) {
    __shared__ double s_red[AJM_BLOCK / 32][AJM_NPART];
    __shared__ double s_w[AJM_BLOCK / 32];
    __shared__ double s_tot[AJM_NPART];
    __shared__ int s_last;

    AjmCtrl* c = p.ctrl;
    if (*(volatile int*)&c->done) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int restart_t = c->restart_t;
    const double beta = c->beta;
    const double* __restrict__ xc = ajm_sel(p, c->cur);
    const double* __restrict__ xp = ajm_sel(p, c->prev);
    double* __restrict__ xf = ajm_sel(p, c->fre);
    AjmAcc acc = {0.0, 0.0, 0.0, 0.0, 0.0};
    const int bid = blockIdx.x;

    // (1) long rows: whole CTA
    for (int li = p.cta_long[bid]; li < p.cta_long[bid + 1]; ++li) {
        const int row = p.long_rows[li];
        const int k0 = p.rp[row], k1 = p.rp[row + 1];
        double s = 0.0;
        for (int k = k0 + tid; k < k1; k += 4 * AJM_BLOCK) {
            double v[4], xg[4];
            int cc[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int kk = k + j * AJM_BLOCK;
                v[j] = 0.0;
                cc[j] = row;
                if (kk < k1) { v[j] = __ldcs(p.val + kk); cc[j] = __ldcs(p.col + kk); }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) xg[j] = __ldg(xc + cc[j]);
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (k + j * AJM_BLOCK < k1) s += v[j] * xg[j];
        }
        s = ajm_warp_sum(s);
        if (lane == 0) s_w[warp] = s;
        __syncthreads();
        if (tid == 0) {
            double q = 0.0;
            for (int w = 0; w < AJM_BLOCK / 32; ++w) q += s_w[w];
            ajm_row_epilogue(p, row, q, beta, restart_t, xc, xp, xf, acc);
        }
        __syncthreads();
    }

    // (2) mid rows: one warp per row
    for (int mi = p.cta_mid[bid] + warp; mi < p.cta_mid[bid + 1]; mi += AJM_BLOCK / 32) {
        const int row = p.mid_rows[mi];
        const int k0 = p.rp[row], k1 = p.rp[row + 1];
        double s = 0.0;
        for (int k = k0 + lane; k < k1; k += 4 * 32) {
            double v[4], xg[4];
            int cc[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int kk = k + j * 32;
                v[j] = 0.0;
                cc[j] = row;
                if (kk < k1) { v[j] = __ldcs(p.val + kk); cc[j] = __ldcs(p.col + kk); }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) xg[j] = __ldg(xc + cc[j]);
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (k + j * 32 < k1) s += v[j] * xg[j];
        }
        s = ajm_warp_sum(s);
        if (lane == 0) ajm_row_epilogue(p, row, s, beta, restart_t, xc, xp, xf, acc);
    }

    // (3) SELL chunks: one warp per chunk of 32 rows, one thread per row
    for (int ch = p.cta_chunk[bid] + warp; ch < p.cta_chunk[bid + 1]; ch += AJM_BLOCK / 32) {
        const long long base = p.chunk_off[ch];
        const int w = (int)((p.chunk_off[ch + 1] - base) >> 5);
        const int slot = ch * 32 + lane;
        const int row = kIdent ? (slot < p.n_sell ? slot : -1) : __ldg(p.perm + slot);
        double bi = 0.0, Di = 1.0, xt = 0.0, xpi = 0.0, qxp = 0.0;
        if (row >= 0) {  // row operands first: independent of the SpMV, so they overlap it
            bi = __ldcs(p.b + row);
            Di = __ldcs(p.D + row);
            xt = __ldg(xc + row);
            xpi = __ldg(xp + row);
            qxp = __ldcs(p.Qxp + row);
        }
        const double* __restrict__ sv = p.sval + base + lane;
        const int* __restrict__ sc = p.scol + base + lane;
        double s = 0.0;
        for (int k0 = 0; k0 < w; k0 += kBatch) {
            double v[kBatch], xg[kBatch];
            int cc[kBatch];
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                if (k0 + j < w) {
                    v[j] = __ldcs(sv + (size_t)(k0 + j) * 32);
                    cc[j] = __ldcs(sc + (size_t)(k0 + j) * 32);
                }
            }
#pragma unroll
            for (int j = 0; j < kBatch; ++j)
                if (k0 + j < w) xg[j] = __ldg(xc + cc[j]);
#pragma unroll
            for (int j = 0; j < kBatch; ++j)
                if (k0 + j < w) s += v[j] * xg[j];
        }
        if (row >= 0) ajm_row_update(p.Qxp, xf, row, s, bi, Di, xt, xpi, qxp, beta, restart_t, acc);
    }

    ajm_block_reduce(acc, s_red);
    if (tid == 0) {
        double* dst = p.partials + (size_t)bid * AJM_NPART;
        dst[0] = acc.rr; dst[1] = acc.xq; dst[2] = acc.bx; dst[3] = acc.d; dst[4] = acc.dabs;
        __threadfence();
        const unsigned v = atomicAdd(&c->ticket, 1u);
        s_last = (v == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // last CTA: fixed-order reduction over all CTA partials
    AjmAcc t = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int k = tid; k < (int)gridDim.x; k += AJM_BLOCK) {
        const double* src = p.partials + (size_t)k * AJM_NPART;
        t.rr += __ldcg(src + 0);
        t.xq += __ldcg(src + 1);
        t.bx += __ldcg(src + 2);
        t.d += __ldcg(src + 3);
        t.dabs += __ldcg(src + 4);
    }
    __syncthreads();
    ajm_block_reduce(t, s_red);
    if (tid == 0) {
        s_tot[0] = t.rr; s_tot[1] = t.xq; s_tot[2] = t.bx; s_tot[3] = t.d; s_tot[4] = t.dabs;
        ajm_finalize_ctrl(p, s_tot);
        __threadfence();
    }
}

// SELL fill: slot-parallel copy of each short row's entries into its chunk column; padding
// (k >= row length, and tail slots) is val 0 / col = own row (or 0), appended AFTER the row's
// entries so the sequential sum order is unchanged.
__global__ void ajm_sell_fill_kernel(int nslots_padded, int n_sell, const int* __restrict__ perm,
                                     int ident, const int* __restrict__ rp, const int* __restrict__ col,
                                     const double* __restrict__ val, const long long* __restrict__ chunk_off,
                                     double* __restrict__ sval, int* __restrict__ scol) {
    const int slot = blockIdx.x * blockDim.x + threadIdx.x;
    if (slot >= nslots_padded) return;
    const int ch = slot >> 5, lane = slot & 31;
    const long long base = chunk_off[ch];
    const int w = (int)((chunk_off[ch + 1] - base) >> 5);
    const int row = ident ? (slot < n_sell ? slot : -1) : perm[slot];
    int k0 = 0, len = 0;
    if (row >= 0) { k0 = rp[row]; len = rp[row + 1] - k0; }
    for (int k = 0; k < w; ++k) {
        const long long e = base + (long long)k * 32 + lane;
        if (k < len) { sval[e] = val[k0 + k]; scol[e] = col[k0 + k]; }
        else { sval[e] = 0.0; scol[e] = row >= 0 ? row : 0; }
    }
}

// ------------------------------------------------------------------------------------------------
// setup kernels (create time, "setup J" of P:798)
// ------------------------------------------------------------------------------------------------

// error bits
#define AJM_EB_CSR 1
#define AJM_EB_NONFINITE 2
#define AJM_EB_NEGDIAG 4
#define AJM_EB_ZERODIAG 8
#define AJM_EB_ASYM 16

// Column range / strict order / finiteness / diagonal, and D per dmode.  One thread per row,
// ascending-column sequential sums: D_kk = Q_kk + sum_{j != k}|Q_kj| (eq-J-diag).
__global__ void ajm_validate_diag_kernel(int n, const int* __restrict__ rp, const int* __restrict__ col,
                                         const double* __restrict__ val, int dmode,
                                         const double* __restrict__ duser, double* __restrict__ D,
                                         int* __restrict__ err) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int e = 0;
    double qkk = 0.0, off = 0.0;
    int last = -1;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
        const int j = col[k];
        const double v = val[k];
        if (j < 0 || j >= n || j <= last) e |= AJM_EB_CSR;
        last = j;
        if (!isfinite(v)) e |= AJM_EB_NONFINITE;
        if (j == i) qkk = v;
        else off += fabs(v);
    }
    if (qkk < 0.0) e |= AJM_EB_NEGDIAG;
    double d;
    if (dmode == 0) d = qkk + off;
    else if (dmode == 2) d = qkk;
    else {
        d = duser[i];
        if (!isfinite(d)) e |= AJM_EB_NONFINITE;
        if (!(d > 0.0)) e |= AJM_EB_ZERODIAG;
    }
    if (d == 0.0) e |= AJM_EB_ZERODIAG;
    D[i] = d;
    if (e) atomicOr(err, e);
}

// Q_ij == Q_ji for every stored entry (binary search of column i in row j).
__global__ void ajm_symmetry_kernel(int n, const int* __restrict__ rp, const int* __restrict__ col,
                                    const double* __restrict__ val, int* __restrict__ err) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
        const int j = col[k];
        int lo = rp[j], hi = rp[j + 1] - 1, found = -1;
        while (lo <= hi) {
            const int mid = (lo + hi) >> 1;
            const int cm = col[mid];
            if (cm == i) { found = mid; break; }
            if (cm < i) lo = mid + 1; else hi = mid - 1;
        }
        if (found < 0 || val[found] != val[k]) { atomicOr(err, AJM_EB_ASYM); return; }
    }
}

__global__ void ajm_finite_kernel(long long n, const double* __restrict__ v, int* __restrict__ err) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        if (!isfinite(v[i])) { atomicOr(err, AJM_EB_NONFINITE); return; }
}

__global__ void ajm_rowptr_narrow_kernel(long long n1, const long long* __restrict__ src,
                                         int* __restrict__ dst) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n1;
         i += (long long)gridDim.x * blockDim.x)
        dst[i] = (int)src[i];
}

// ||b||^2: fixed grid of 256 CTAs, grid-strided sequential per thread, then fixed trees.
__global__ void __launch_bounds__(256) ajm_sumsq_partial_kernel(long long n, const double* __restrict__ v,
                                                                double* __restrict__ part) {
    __shared__ double s[256 / 32];
    double a = 0.0;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += 256LL * gridDim.x) a += v[i] * v[i];
    a = ajm_warp_sum(a);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += s[w];
        part[blockIdx.x] = t;
    }
}

__global__ void ajm_sum_final_kernel(int m, const double* __restrict__ part, double* __restrict__ out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < m; ++i) t += part[i];
        *out = t;
    }
}

// Per-solve initialisation of the control block (t = 0: x~^0 = x0, x^{-1} := x0, beta_0 = 0,
// alpha_1 = 1, K = K_0, K_re = 0, ell = 0).
__global__ void ajm_init_ctrl_kernel(AjmCtrl* c, double tol, long long maxit, int momentum,
                                     int restart, long long k0, double nb, double* res_hist,
                                     double* f_hist, double* d_hist, double* dabs_hist) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    c->t = 0;
    c->maxit = maxit;
    c->K = k0;
    c->Kre = 0;
    c->tol = tol;
    c->nb = nb;
    c->alpha = 1.0;
    c->beta = 0.0;
    c->restart_t = 0;
    c->cur = 0;
    c->prev = 1;
    c->fre = 2;
    c->momentum = momentum;
    c->restart_enabled = restart;
    c->done = 0;
    c->status = 1;
    c->iterations = 0;
    c->answer = 0;
    c->prerestart = 0;
    c->nres = 0;
    c->nlogged = 0;
    c->ticket = 0;
    c->res_last = 0.0;
    c->f_last = 0.0;
    c->res_hist = res_hist;
    c->f_hist = f_hist;
    c->d_hist = d_hist;
    c->dabs_hist = dabs_hist;
    d_hist[0] = 0.0;
    dabs_hist[0] = 0.0;
}
