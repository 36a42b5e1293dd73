// Host staging-copy bandwidth on the GPU box: pageable source -> pinned ring buffer, the copy cspq_encode_host does
// for pageable input.  Variants: memcpy / AVX2 non-temporal stores, 1..32 threads, thread pool vs spawn per batch.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <thread>
#include <vector>
#include <atomic>
#include <immintrin.h>
#include <cuda_runtime.h>
static void nt_copy(char *dst, const char *src, size_t n) {
    size_t i = 0;
    for (; i + 128 <= n; i += 128) {
        __m256i a = _mm256_loadu_si256((const __m256i *)(src + i)), b = _mm256_loadu_si256((const __m256i *)(src + i + 32));
        __m256i c = _mm256_loadu_si256((const __m256i *)(src + i + 64)), d = _mm256_loadu_si256((const __m256i *)(src + i + 96));
        _mm256_stream_si256((__m256i *)(dst + i), a); _mm256_stream_si256((__m256i *)(dst + i + 32), b);
        _mm256_stream_si256((__m256i *)(dst + i + 64), c); _mm256_stream_si256((__m256i *)(dst + i + 96), d);
    }
    memcpy(dst + i, src + i, n - i);
    _mm_sfence();
}
int main() {
    const size_t total = 4ull << 30, batch = 192ull << 20;
    char *src = (char *)malloc(total);
    for (size_t i = 0; i < total; i += 4096) src[i] = (char)i;  // touch
    char *dst;
    cudaHostAlloc((void **)&dst, batch * 2, cudaHostAllocDefault);
    memset(dst, 1, batch * 2);
    printf("hw threads %u\n", std::thread::hardware_concurrency());
    for (int nt : {1, 2, 4, 8, 16, 32}) for (int mode = 0; mode < 2; ++mode) {
        auto t0 = std::chrono::steady_clock::now();
        size_t done = 0; int slot = 0;
        while (done + batch <= total) {
            std::vector<std::thread> th;
            const size_t per = (batch + nt - 1) / nt / 128 * 128 + 128;
            for (int t = 0; t < nt; ++t) {
                const size_t lo = t * per; if (lo >= batch) break;
                const size_t len = std::min(per, batch - lo);
                char *d = dst + slot * batch + lo; const char *s = src + done + lo;
                th.emplace_back([=] { if (mode) nt_copy(d, s, len); else memcpy(d, s, len); });
            }
            for (auto &t : th) t.join();
            done += batch; slot ^= 1;
        }
        double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        printf("threads %2d %-6s %6.1f GB/s\n", nt, mode ? "nt" : "memcpy", done / dt / 1e9);
    }
    // with H2D overlapped (the real pipeline): copy batch b+1 while batch b goes over PCIe
    void *dX; cudaMalloc(&dX, batch); cudaStream_t st; cudaStreamCreate(&st);
    for (int nt : {8, 16, 32}) for (int mode = 0; mode < 2; ++mode) {
        auto t0 = std::chrono::steady_clock::now();
        size_t done = 0; int slot = 0;
        cudaEvent_t ev[2]; cudaEventCreate(&ev[0]); cudaEventCreate(&ev[1]);
        bool used[2] = {false, false};
        while (done + batch <= total) {
            if (used[slot]) cudaEventSynchronize(ev[slot]);
            std::vector<std::thread> th;
            const size_t per = (batch + nt - 1) / nt / 128 * 128 + 128;
            for (int t = 0; t < nt; ++t) {
                const size_t lo = t * per; if (lo >= batch) break;
                const size_t len = std::min(per, batch - lo);
                char *d = dst + slot * batch + lo; const char *s = src + done + lo;
                th.emplace_back([=] { if (mode) nt_copy(d, s, len); else memcpy(d, s, len); });
            }
            for (auto &t : th) t.join();
            cudaMemcpyAsync(dX, dst + slot * batch, batch, cudaMemcpyHostToDevice, st);
            cudaEventRecord(ev[slot], st); used[slot] = true;
            done += batch; slot ^= 1;
        }
        cudaStreamSynchronize(st);
        double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        printf("pipeline threads %2d %-6s %6.1f GB/s\n", nt, mode ? "nt" : "memcpy", done / dt / 1e9);
    }
    return 0;
}
