// Probe: plain vectorised LDG/STG streaming copy (1 GiB in + 1 GiB out) with
// U independent 16-byte loads in flight per thread, by grid size — the
// ceiling a non-TMA streaming kernel reaches (cf. cuFFT's 1024-point batch
// at ~6.9 TB/s). Best of 10 back-to-back launches.
#include <cstdio>
#include <cuda_runtime.h>

template <int U, int ST>
__global__ void __launch_bounds__(256) copy_u(const float4* __restrict__ in, float4* __restrict__ out, long long n) {
    const long long stride = (long long)gridDim.x * blockDim.x * U;
    for (long long base = (long long)blockIdx.x * blockDim.x * U + threadIdx.x; base < n; base += stride) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            long long i = base + (long long)u * blockDim.x;
            if (i < n) v[u] = __ldcs(in + i);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            long long i = base + (long long)u * blockDim.x;
            if (i < n) {
                if (ST == 0) __stcs(out + i, v[u]);
                else out[i] = v[u];
            }
        }
    }
}

template <int U, int ST>
void run(const float4* a, float4* b, long long n, int blocks) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9;
    for (int r = 0; r < 12; ++r) {
        cudaEventRecord(e0);
        copy_u<U, ST><<<blocks, 256>>>(a, b, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r >= 2 && ms < best) best = ms;
    }
    printf("{\"U\": %d, \"store\": \"%s\", \"blocks\": %d, \"ms\": %.4f, \"gbps\": %.0f}\n", U, ST ? "plain" : "cs",
           blocks, best, 2.0 * n * 16 / best / 1e6);
}

int main() {
    const size_t bytes = 1ull << 30;
    float4 *a, *b;
    cudaMalloc(&a, bytes);
    cudaMalloc(&b, bytes);
    cudaMemset(a, 1, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const long long n = bytes / 16;
    for (int per : {4, 8, 16}) {
        run<4, 0>(a, b, n, sms * per);
        run<8, 0>(a, b, n, sms * per);
        run<4, 1>(a, b, n, sms * per);
    }
    run<1, 1>(a, b, n, (int)(n / 256));
    run<4, 1>(a, b, n, (int)(n / 1024));
    return 0;
}
