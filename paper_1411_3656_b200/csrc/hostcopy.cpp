// hostcopy.cpp — the host copy kernel of the library's copy pool (ppfg.cu
// CopyPool): pageable <-> pinned staging of the host-buffer paths. Large
// pieces are copied with AVX2 non-temporal (streaming) stores: the
// destination is not read back by this copy, so streaming skips the
// read-for-ownership of every destination line — on the GPU box (16-vCPU
// Xeon VM) 8 threads copy 37 GB/s this way against 31 GB/s with memcpy
// (profiles/round2/probes/host_copy_mt.jsonl). Compiled as plain C++ with
// -mavx2 for this unit only; used only when the CPU reports AVX2.
#include <immintrin.h>

#include <cstddef>
#include <cstdint>
#include <cstring>

namespace ppfg {

namespace {
bool have_avx2() {
    static const bool ok = __builtin_cpu_supports("avx2");
    return ok;
}
} // namespace

void copy_piece(void* dst, const void* src, std::size_t n) {
    constexpr std::size_t kStreamMin = std::size_t(256) << 10;
    if (n < kStreamMin || !have_avx2()) {
        std::memcpy(dst, src, n);
        return;
    }
    char* d = static_cast<char*>(dst);
    const char* s = static_cast<const char*>(src);
    const std::size_t head = (32 - (reinterpret_cast<std::uintptr_t>(d) & 31)) & 31;
    std::memcpy(d, s, head);
    d += head;
    s += head;
    n -= head;
    std::size_t i = 0;
    for (; i + 128 <= n; i += 128) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 32));
        const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 64));
        const __m256i e = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 96));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), a);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 32), b);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 64), c);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 96), e);
    }
    std::memcpy(d + i, s + i, n - i);
    _mm_sfence(); // the streamed lines are visible before the caller signals completion
}

} // namespace ppfg
