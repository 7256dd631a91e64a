// gather_mlp.cu -- random 8-byte gathers from an L2-resident array (8 MB / 32 MB) as a function of
// warps per SM and gathers in flight per thread (G independent loads per loop step).
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_mlp gather_mlp.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int G>
__global__ void gather_g(const double* __restrict__ x, unsigned nmask, long long m, double* out) {
    double s = 0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < m; k += stride * G) {
        double v[G];
#pragma unroll
        for (int j = 0; j < G; ++j) {
            unsigned h = (unsigned)(k + j * stride) * 2654435761u;
            h ^= h >> 15;
            v[j] = x[h & nmask];
        }
#pragma unroll
        for (int j = 0; j < G; ++j) s += v[j];
    }
    if (s == 12345.678) *out = s;
}

template <int G>
float run(const double* x, unsigned mask, long long m, int ctas_per_sm, int sms, double* out) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    gather_g<G><<<sms * ctas_per_sm, 256>>>(x, mask, m, out);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        gather_g<G><<<sms * ctas_per_sm, 256>>>(x, mask, m, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    return best;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    const long long m = 64LL << 20;
    for (int mb : {8, 32}) {
        const long long nx = (long long)mb << 17;
        double* x;
        cudaMalloc(&x, nx * 8);
        cudaMemset(x, 0, nx * 8);
        for (int cps : {1, 2, 8}) {
            float t1 = run<1>(x, (unsigned)(nx - 1), m, cps, sms, out);
            float t8 = run<8>(x, (unsigned)(nx - 1), m, cps, sms, out);
            float t16 = run<16>(x, (unsigned)(nx - 1), m, cps, sms, out);
            printf("{\"array_MB\": %d, \"warps_per_sm\": %d, \"Ggps_G1\": %.1f, \"Ggps_G8\": %.1f, \"Ggps_G16\": %.1f}\n", mb,
                   cps * 8, m / (t1 * 1e-3) / 1e9, m / (t8 * 1e-3) / 1e9, m / (t16 * 1e-3) / 1e9);
        }
        cudaFree(x);
    }
    return 0;
}
