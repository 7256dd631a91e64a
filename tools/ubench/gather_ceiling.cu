// gather_ceiling.cu -- measured ceilings for the AJM pass's two memory streams on this GPU:
//   (1) streaming read of a large array (HBM)                      -> GB/s
//   (2) random 8-byte gathers x[idx[k]] from an array of X MB      -> Ggathers/s  (idx streamed)
//   (3) the same with the idx stream replaced by a hash (no idx traffic)
// Each thread sums what it reads (so nothing is dead code); grid = 148 x 8 CTAs x 256 threads,
// grid-strided.  CUDA events, best of 5 after warm-up.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_ceiling gather_ceiling.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void stream_read(const double2* __restrict__ a, long long n4, double* out) {
    double s = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
        double2 v = __ldcs(a + i);
        s += v.x + v.y;
    }
    if (s == 12345.678) *out = s;
}

__global__ void gather_idx(const double* __restrict__ x, const int* __restrict__ idx, long long m, double* out) {
    double s = 0;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < m; k += (long long)gridDim.x * blockDim.x)
        s += x[__ldcs(idx + k)];
    if (s == 12345.678) *out = s;
}

__global__ void gather_hash(const double* __restrict__ x, unsigned nmask, long long m, double* out) {
    double s = 0;
#pragma unroll 8
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < m; k += (long long)gridDim.x * blockDim.x) {
        unsigned h = (unsigned)k * 2654435761u;
        h ^= h >> 15;
        s += x[h & nmask];
    }
    if (s == 12345.678) *out = s;
}

template <class F>
float best_ms(F f) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    f();
    f();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        f();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * 8, block = 256;
    double* out;
    cudaMalloc(&out, 8);
    // (1) streaming read, 4 GiB
    const long long nbytes = 4LL << 30;
    double2* a;
    cudaMalloc(&a, nbytes);
    cudaMemset(a, 0, nbytes);
    float ms = best_ms([&] { stream_read<<<grid, block>>>(a, nbytes / 16, out); });
    printf("{\"test\": \"stream_read\", \"bytes\": %lld, \"ms\": %.4f, \"GBps\": %.1f}\n", nbytes, ms, nbytes / (ms * 1e-3) / 1e9);
    cudaFree(a);
    // (2)/(3) gathers from arrays of 8, 32, 128, 512 MB
    const long long m = 64LL << 20;  // 64 Mi gathers
    int* idx;
    cudaMalloc(&idx, m * 4);
    int* hidx = (int*)malloc(m * 4);
    for (int mb : {8, 32, 128, 512}) {
        const long long nx = (long long)mb << 17;  // doubles
        double* x;
        cudaMalloc(&x, nx * 8);
        cudaMemset(x, 0, nx * 8);
        uint64_t st = 0x9E3779B97F4A7C15ull;
        for (long long k = 0; k < m; ++k) {
            st ^= st << 13; st ^= st >> 7; st ^= st << 17;
            hidx[k] = (int)(st % (uint64_t)nx);
        }
        cudaMemcpy(idx, hidx, m * 4, cudaMemcpyHostToDevice);
        float mi = best_ms([&] { gather_idx<<<grid, block>>>(x, idx, m, out); });
        float mh = best_ms([&] { gather_hash<<<grid, block>>>(x, (unsigned)(nx - 1), m, out); });
        printf("{\"test\": \"gather\", \"array_MB\": %d, \"gathers\": %lld, \"idx_ms\": %.4f, \"idx_Ggps\": %.2f, "
               "\"hash_ms\": %.4f, \"hash_Ggps\": %.2f}\n", mb, m, mi, m / (mi * 1e-3) / 1e9, mh, m / (mh * 1e-3) / 1e9);
        cudaFree(x);
    }
    return 0;
}
