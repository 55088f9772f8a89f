// Probe: HBM streaming efficiency of read-once/write-once copies by how the
// rows are assigned to a persistent grid — contiguous per-CTA ranges (K3's
// assignment) vs interleaved batches (one advancing front) — and by chunk
// size. 1 GiB in, 1 GiB out; bytes = in + out; best of 10 back-to-back.
#include <cstdio>
#include <cuda_runtime.h>

template <int CONTIG>
__global__ void __launch_bounds__(512) copy_rows(const float4* __restrict__ in, float4* __restrict__ out,
                                                 long long n_chunks, int chunk_f4) {
    const long long per = (n_chunks + gridDim.x - 1) / gridDim.x;
    for (long long k = 0; k < per; ++k) {
        const long long c = CONTIG ? blockIdx.x * per + k : k * gridDim.x + blockIdx.x;
        if (c >= n_chunks) break;
        const float4* src = in + c * chunk_f4;
        float4* dst = out + c * chunk_f4;
        for (int i = threadIdx.x; i < chunk_f4; i += blockDim.x) {
            float4 v = __ldcs(src + i);
            __stcs(dst + i, v);
        }
    }
}

int main() {
    const size_t bytes = 1ull << 30;
    float4 *a, *b;
    cudaMalloc(&a, bytes);
    cudaMalloc(&b, bytes);
    cudaMemset(a, 1, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int chunk_kb : {8, 48, 256}) {
        const int chunk_f4 = chunk_kb * 1024 / 16;
        const long long n = bytes / (chunk_kb * 1024);
        for (int contig = 0; contig < 2; ++contig) {
            for (int per_sm : {1, 2, 4}) {
                float best = 1e9;
                for (int r = 0; r < 12; ++r) {
                    cudaEventRecord(e0);
                    if (contig) copy_rows<1><<<sms * per_sm, 512>>>(a, b, n, chunk_f4);
                    else copy_rows<0><<<sms * per_sm, 512>>>(a, b, n, chunk_f4);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (r >= 2 && ms < best) best = ms;
                }
                printf("{\"chunk_kb\": %d, \"assign\": \"%s\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"gbps\": %.0f}\n",
                       chunk_kb, contig ? "contiguous" : "interleaved", per_sm, best, 2.0 * bytes / best / 1e6);
            }
        }
    }
    float best = 1e9;
    for (int r = 0; r < 12; ++r) {
        cudaEventRecord(e0);
        cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r >= 2 && ms < best) best = ms;
    }
    printf("{\"cudaMemcpy\": true, \"ms\": %.4f, \"gbps\": %.0f}\n", best, 2.0 * bytes / best / 1e6);
    return 0;
}
