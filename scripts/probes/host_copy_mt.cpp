// Probe: host copy throughput on the GPU box by thread count and store kind
// (memcpy vs AVX non-temporal streaming stores), pageable <-> pinned 1 GiB
// buffers, in 8 MiB jobs split over the threads (as the library's CopyPool).
#include <cuda_runtime.h>
#include <immintrin.h>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static void copy_nt(char* d, const char* s, size_t n) {
    // 32-byte aligned bulk with streaming stores; head/tail by memcpy
    size_t head = (32 - (reinterpret_cast<uintptr_t>(d) & 31)) & 31;
    if (head > n) head = n;
    std::memcpy(d, s, head);
    d += head; s += head; n -= head;
    size_t i = 0;
    for (; i + 128 <= n; i += 128) {
        __m256i a = _mm256_loadu_si256((const __m256i*)(s + i));
        __m256i b = _mm256_loadu_si256((const __m256i*)(s + i + 32));
        __m256i c = _mm256_loadu_si256((const __m256i*)(s + i + 64));
        __m256i e = _mm256_loadu_si256((const __m256i*)(s + i + 96));
        _mm256_stream_si256((__m256i*)(d + i), a);
        _mm256_stream_si256((__m256i*)(d + i + 32), b);
        _mm256_stream_si256((__m256i*)(d + i + 64), c);
        _mm256_stream_si256((__m256i*)(d + i + 96), e);
    }
    std::memcpy(d + i, s + i, n - i);
    _mm_sfence();
}

int main() {
    const size_t N = size_t(1) << 30, JOB = size_t(8) << 20;
    char* pg = static_cast<char*>(aligned_alloc(4096, N));
    char* pg2 = static_cast<char*>(aligned_alloc(4096, N));
    char* pin = nullptr;
    cudaHostAlloc(&pin, N, cudaHostAllocDefault);
    std::memset(pg, 1, N);
    std::memset(pg2, 2, N);
    std::memset(pin, 3, N);
    printf("{\"hw_threads\": %u}\n", std::thread::hardware_concurrency());
    for (int nt : {1, 2, 4, 8, 12, 16}) {
        for (int kind = 0; kind < 2; ++kind) {
            for (int dir = 0; dir < 2; ++dir) {
                char* dst = dir ? pg2 : pin;
                const char* src = dir ? pin : pg;
                auto t0 = std::chrono::steady_clock::now();
                for (int rep = 0; rep < 2; ++rep) {
                    for (size_t o = 0; o < N; o += JOB) {
                        // one job: split over nt threads
                        std::vector<std::thread> th;
                        const size_t per = JOB / nt;
                        for (int k = 0; k < nt; ++k)
                            th.emplace_back([=] {
                                if (kind) copy_nt(dst + o + k * per, src + o + k * per, per);
                                else std::memcpy(dst + o + k * per, src + o + k * per, per);
                            });
                        for (auto& t : th) t.join();
                    }
                }
                double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                printf("{\"threads\": %d, \"kind\": \"%s\", \"dir\": \"%s\", \"GBps\": %.1f}\n", nt,
                       kind ? "nt-avx" : "memcpy", dir ? "pinned->pageable" : "pageable->pinned", 2.0 * N / s / 1e9);
            }
        }
    }
    return 0;
}
