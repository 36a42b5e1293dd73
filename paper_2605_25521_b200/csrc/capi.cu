// capi.cu -- the extern "C" boundary (include/cspq_b200.h) and the native
// host-side runtime around the kernels: argument validation with the
// reference's error classes, the end-to-end host->device->host encode
// pipeline (pinned ring, multi-stream overlap), and per-thread errors.

#include <atomic>
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#if defined(__x86_64__)
#include <immintrin.h>
#endif
#include <vector>

#include "common.cuh"

namespace cspq {

// kernels (encode.cu / lloyd.cu)
int encode_prepare(const float *CB, const float *B, int m, int k, int sub, float *guard, cudaStream_t st);
int encode_stats(unsigned long long *flagged, int reset);
int encode_set_tiling(int t);
size_t encode_tc_image_bytes(int m, int k, int sub);
int encode_tc_prepare(const float *CB, const float *B, int m, int k, int sub, void *img, cudaStream_t st);
int encode_tc(const void *X, int in_dtype, int64_t n, int64_t xrs, const float *CB, const float *B,
              const float *guard, const void *img, int m, int k, int sub, uint8_t *codes, int64_t crs, float *best,
              cudaStream_t st);
int encode_tc_stats(unsigned long long *flagged, int reset);
int encode_tc_max_subspaces(int sub, int in_dtype);
int recompute_biases(const float *CB, int m, int k, int sub, float *Bo, cudaStream_t st);
int encode_device(const void *X, int in_dtype, int64_t n, int d, int64_t xrs, const float *CB, const float *B,
                  const float *guard, int m, int k, int sub, void *codes, int64_t crs, int variant, int mode,
                  cudaStream_t st);
int encode_subspace_major(const float *P, int64_t n, int m, int sub, const float *CB, const float *B, int k,
                          int32_t *assign, int variant, cudaStream_t st);
int encode_with_scores(const void *X, int in_dtype, int64_t n, int64_t xrs, const float *CB, const float *B,
                       int m, int k, int sub, int32_t *codes, float *best, int variant, cudaStream_t st);
size_t lloyd_workspace_bytes(int64_t n, int m, int sub, int k);
size_t crc32_workspace_bytes(int64_t n);
int adc_tables(const float *Q, int64_t nq, int d, const float *CB, int m, int k, int sub, float *T, cudaStream_t st);
int adc_scores(const float *T, int64_t nq, const void *codes, int code_bytes, int64_t n, int m, int k, float *S,
               cudaStream_t st);
int topn_select(const void *vals, int val_bytes, int64_t nq, int64_t n, int topn, int64_t *idx, void *out_vals,
                cudaStream_t st);
int gt_distances(const float *Qm, int64_t nq, const float *X, int64_t n, int d, double *nrm, double *D,
                 cudaStream_t st);
int crc32_device_api(const void *data, int64_t n, uint32_t crc_in, uint32_t *crc_out, void *ws, cudaStream_t st);
uint32_t crc32_combine_host(uint32_t crc1, uint32_t crc2, int64_t len2);
int unpack_vecs(const void *records, int64_t n, int d, int value_bytes, int check_finite, int64_t off0, void *rows,
                unsigned long long *bad, cudaStream_t st);
int encode_vecs_file(const char *in_path, int fmt, const char *out_path, const float *CB, const float *B,
                     const float *guard, const void *tc_img, int m, int k, int sub, int variant, int mode,
                     int64_t batch_rows, int n_streams, int device, int64_t *n_out, int64_t *err);
int lloyd_assign(const void *P, int pf64, int64_t n, int m, int sub, int k, const double *C64,
                 const int32_t *state, int64_t b, int64_t e, int32_t *assign, double *sq, void *ws, cudaStream_t st);
int lloyd_accumulate(const void *P, int pf64, int64_t n, int m, int sub, int k, const int32_t *state,
                     const int32_t *assign, const double *sq, int64_t b, int64_t e, double *counts,
                     double *sums, double *obj, void *ws, cudaStream_t st);
int lloyd_update(const double *counts, const double *sums, int m, int k, int sub, const int32_t *state,
                 double *C64, int32_t *empties, int32_t *nempty, cudaStream_t st);
int lloyd_repair(const void *P, int pf64, int64_t n, int m, int sub, int k, const int32_t *assign,
                 const int32_t *state, const int32_t *empties, const int32_t *nempty, double *C64, void *ws,
                 cudaStream_t st);
int lloyd_stop(const double *obj, int m, int max_iters, double tol, int32_t *state, double *prev,
               int32_t *iterations, double *objectives, cudaStream_t st);
int lloyd_final_objective(const void *P, int pf64, int64_t n, int m, int sub, int k, const float *C32,
                          const int32_t *assign, double *obj, void *ws, cudaStream_t st);
int lloyd_train(const void *P, int pf64, int64_t n, int m, int sub, int k, double *C64, int max_iters, double tol,
                float *C32, int32_t *assign, double *objectives, int32_t *iterations, void *ws, cudaStream_t st);
int kmeanspp(const void *P, int pf64, int64_t n, int m, int sub, int k, const int64_t *first, const double *u,
             double *C64, int32_t *status, void *ws, cudaStream_t st);

namespace {
thread_local char g_err[1024] = "";

int check_shape(int64_t n, int m, int k, int sub) {
    CSPQ_REQUIRE(n >= 0, CSPQ_E_CONFIG, "n must be >= 0, got %lld", (long long)n);
    CSPQ_REQUIRE(m >= 1, CSPQ_E_CONFIG, "m must be >= 1, got %d", m);
    CSPQ_REQUIRE(k >= 1 && k <= 65536, CSPQ_E_CONFIG, "k must be in [1, 65536], got %d", k);
    CSPQ_REQUIRE(sub >= 1, CSPQ_E_CONFIG, "sub_dim must be >= 1, got %d", sub);
    return CSPQ_OK;
}

bool is_pinned(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// Streaming copy (AVX2 non-temporal stores): the staging copies never re-read their destination on the
// host, so they should not pull it through the caches.  scripts/micro/host_copy.cu on the GPU box
// (16 cores), pageable source -> pinned ring with the H2D copy of the previous batch in flight:
// memcpy 16 threads 41 GB/s (32 threads 33), non-temporal 16 threads 47 GB/s.
#if defined(__x86_64__)
__attribute__((target("avx2"))) static void stream_copy_avx2(char *dst, const char *src, size_t n) {
    size_t i = 0;
    const size_t head = std::min(n, (size_t)((32 - (reinterpret_cast<uintptr_t>(dst) & 31)) & 31));
    if (head) { std::memcpy(dst, src, head); i = head; }
    for (; i + 128 <= n; i += 128) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(src + i));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(src + i + 32));
        const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(src + i + 64));
        const __m256i d = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(src + i + 96));
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i), a);
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i + 32), b);
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i + 64), c);
        _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i + 96), d);
    }
    if (i < n) std::memcpy(dst + i, src + i, n - i);
    _mm_sfence();
}
#endif
static void stream_copy(char *dst, const char *src, size_t n) {
#if defined(__x86_64__)
    static const bool avx2 = __builtin_cpu_supports("avx2") && !(getenv("CSPQ_HOST_COPY_NT") && atoi(getenv("CSPQ_HOST_COPY_NT")) == 0);
    if (avx2) { stream_copy_avx2(dst, src, n); return; }
#endif
    std::memcpy(dst, src, n);
}

void par_memcpy(void *dst, const void *src, size_t bytes) {
    const size_t kMin = 8u << 20;
    const unsigned nt = std::min<unsigned>(16u, std::max(1u, std::thread::hardware_concurrency()));
    if (bytes < kMin || nt == 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    std::vector<std::thread> th;
    const size_t per = ((bytes + nt - 1) / nt + 127) / 128 * 128;
    for (unsigned i = 0; i < nt; ++i) {
        const size_t lo = i * per;
        if (lo >= bytes) break;
        const size_t len = std::min(per, bytes - lo);
        th.emplace_back([=] { stream_copy((char *)dst + lo, (const char *)src + lo, len); });
    }
    for (auto &t : th) t.join();
}

// Per-device pipeline resources for cspq_encode_host, grown on demand.
struct Pipeline {
    int device = -1;
    int ns = 0;
    size_t xbytes = 0, cbytes = 0;
    std::vector<cudaStream_t> st;
    std::vector<void *> dX, dC, hX, hC;
    std::vector<cudaEvent_t> ev0, ev1;
    float *guard = nullptr;
    size_t guard_floats = 0;
    std::mutex mu;

    void release() {
        for (auto s : st) cudaStreamDestroy(s);
        for (auto p : dX) cudaFree(p);
        for (auto p : dC) cudaFree(p);
        for (auto p : hX) if (p) cudaFreeHost(p);
        for (auto p : hC) if (p) cudaFreeHost(p);
        for (auto e : ev0) cudaEventDestroy(e);
        for (auto e : ev1) cudaEventDestroy(e);
        st.clear(); dX.clear(); dC.clear(); hX.clear(); hC.clear(); ev0.clear(); ev1.clear();
        ns = 0; xbytes = cbytes = 0;
    }
    int ensure(int n_streams, size_t xb, size_t cb) {
        if (n_streams <= ns && xb <= xbytes && cb <= cbytes) return CSPQ_OK;
        cudaDeviceSynchronize();
        release();
        for (int i = 0; i < n_streams; ++i) {
            cudaStream_t s;
            CSPQ_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            st.push_back(s);
            void *p;
            CSPQ_CUDA_TRY(cudaMalloc(&p, xb)); dX.push_back(p);
            CSPQ_CUDA_TRY(cudaMalloc(&p, cb)); dC.push_back(p);
            CSPQ_CUDA_TRY(cudaHostAlloc(&p, xb, cudaHostAllocDefault)); hX.push_back(p);
            CSPQ_CUDA_TRY(cudaHostAlloc(&p, cb, cudaHostAllocDefault)); hC.push_back(p);
            cudaEvent_t e;
            CSPQ_CUDA_TRY(cudaEventCreate(&e)); ev0.push_back(e);
            CSPQ_CUDA_TRY(cudaEventCreate(&e)); ev1.push_back(e);
        }
        ns = n_streams; xbytes = xb; cbytes = cb;
        return CSPQ_OK;
    }
};

Pipeline g_pipes[64];
}  // namespace

std::atomic<unsigned long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

}  // namespace cspq

using namespace cspq;

extern "C" {

int cspq_abi_version(void) { return CSPQ_ABI_VERSION; }
const char *cspq_last_error(void) { return g_err; }

int cspq_encode_set_tiling(int32_t tiling) { return encode_set_tiling(tiling); }

uint64_t cspq_launch_count(int32_t reset) {
    return reset ? g_launches.exchange(0, std::memory_order_relaxed) : g_launches.load(std::memory_order_relaxed);
}

int cspq_encode_stats(uint64_t *flagged, int32_t reset) {
    unsigned long long v = 0, w = 0;
    int rc = encode_stats(flagged ? &v : nullptr, reset);
    if (rc) return rc;
    rc = encode_tc_stats(flagged ? &w : nullptr, reset);
    if (flagged) *flagged = v + w;
    return rc;
}

size_t cspq_encode_tc_image_bytes(int32_t m, int32_t k, int32_t sub) { return encode_tc_image_bytes(m, k, sub); }

int cspq_encode_tc_prepare(const float *CB, const float *B, int32_t m, int32_t k, int32_t sub, void *img,
                           void *stream) {
    int rc = check_shape(0, m, k, sub);
    if (rc) return rc;
    CSPQ_REQUIRE(CB && B && img, CSPQ_E_CONFIG, "null pointer");
    return encode_tc_prepare(CB, B, m, k, sub, img, as_stream(stream));
}

int cspq_encode_tc(const void *X, int32_t in_dtype, int64_t n, int32_t d, int64_t x_row_stride, const float *CB,
                   const float *B, const float *guard, const void *img, int32_t m, int32_t k, int32_t sub, void *codes,
                   int64_t codes_row_stride, float *best, void *stream) {
    int rc = check_shape(n, m, k, sub);
    if (rc) return rc;
    CSPQ_REQUIRE(d == m * sub, CSPQ_E_CONFIG,
                 "dataset dimensionality %d does not match codebooks' d=%d", d, m * sub);
    CSPQ_REQUIRE(in_dtype == CSPQ_IN_F32 || in_dtype == CSPQ_IN_U8, CSPQ_E_CONFIG, "bad in_dtype %d", in_dtype);
    CSPQ_REQUIRE(x_row_stride >= d && codes_row_stride >= m, CSPQ_E_CONFIG, "bad strides");
    if (n == 0) return CSPQ_OK;
    CSPQ_REQUIRE(X && CB && B && guard && img && codes, CSPQ_E_CONFIG, "null pointer");
    return encode_tc(X, in_dtype, n, x_row_stride, CB, B, guard, img, m, k, sub, reinterpret_cast<uint8_t *>(codes),
                     codes_row_stride, best, as_stream(stream));
}

int32_t cspq_encode_tc_max_subspaces(int32_t sub, int32_t in_dtype) { return encode_tc_max_subspaces(sub, in_dtype); }

int cspq_encode_prepare(const float *CB, const float *B, int32_t m, int32_t k, int32_t sub, float *guard,
                        void *stream) {
    int rc = check_shape(0, m, k, sub);
    if (rc) return rc;
    CSPQ_REQUIRE(CB && guard, CSPQ_E_CONFIG, "null pointer");
    return encode_prepare(CB, B, m, k, sub, guard, as_stream(stream));
}

int cspq_recompute_biases_f32(const float *CB, int32_t m, int32_t k, int32_t sub, float *B_out, void *stream) {
    int rc = check_shape(0, m, k, sub);
    if (rc) return rc;
    CSPQ_REQUIRE(CB && B_out, CSPQ_E_CONFIG, "null pointer");
    return recompute_biases(CB, m, k, sub, B_out, as_stream(stream));
}

int cspq_encode(const void *X, int32_t in_dtype, int64_t n, int32_t d, int64_t x_row_stride, const float *CB,
                const float *B, const float *guard, int32_t m, int32_t k, int32_t sub, void *codes,
                int64_t codes_row_stride, int32_t variant, int32_t mode, void *stream) {
    int rc = check_shape(n, m, k, sub);
    if (rc) return rc;
    CSPQ_REQUIRE(d == m * sub, CSPQ_E_CONFIG,
                 "dataset dimensionality %d does not match codebooks' d=%d", d, m * sub);
    CSPQ_REQUIRE(in_dtype == CSPQ_IN_F32 || in_dtype == CSPQ_IN_U8, CSPQ_E_CONFIG, "bad in_dtype %d", in_dtype);
    CSPQ_REQUIRE(variant >= 0 && variant <= 2, CSPQ_E_CONFIG, "bad variant %d", variant);
    CSPQ_REQUIRE(mode >= 0 && mode <= 2, CSPQ_E_CONFIG, "bad mode %d", mode);
    CSPQ_REQUIRE(x_row_stride >= d && codes_row_stride >= m, CSPQ_E_CONFIG, "bad strides");
    if (n == 0) return CSPQ_OK;
    CSPQ_REQUIRE(X && CB && codes && (B || variant == CSPQ_VARIANT_REFERENCE), CSPQ_E_CONFIG, "null pointer");
    cudaStream_t st = as_stream(stream);
    float *tmp = nullptr;
    const bool needs_guard = variant != CSPQ_VARIANT_REFERENCE && mode != CSPQ_MODE_EXACT;
    if (needs_guard && !guard) {
        CSPQ_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void **>(&tmp), sizeof(float) * 2 * m, st));
        if ((rc = encode_prepare(CB, B, m, k, sub, tmp, st))) return rc;
        guard = tmp;
    }
    rc = encode_device(X, in_dtype, n, d, x_row_stride, CB, B, guard, m, k, sub, codes, codes_row_stride, variant,
                       mode, st);
    if (tmp) cudaFreeAsync(tmp, st);
    return rc;
}

int cspq_encode_with_scores(const void *X, int32_t in_dtype, int64_t n, int32_t d, int64_t x_row_stride,
                            const float *CB, const float *B, int32_t m, int32_t k, int32_t sub, int32_t *codes,
                            float *best, int32_t variant, void *stream) {
    int rc = check_shape(n, m, k, sub);
    if (rc) return rc;
    CSPQ_REQUIRE(d == m * sub, CSPQ_E_CONFIG, "vector length %d does not match d=%d", d, m * sub);
    CSPQ_REQUIRE(x_row_stride >= d, CSPQ_E_CONFIG, "bad stride");
    if (n == 0) return CSPQ_OK;
    return encode_with_scores(X, in_dtype, n, x_row_stride, CB, B, m, k, sub, codes, best, variant, as_stream(stream));
}

int cspq_encode_subspace_major(const float *P, int64_t n, int32_t m, int32_t sub, const float *CB, const float *B,
                               int32_t k, int32_t *assign, int32_t variant, void *stream) {
    int rc = check_shape(n, m, k, sub);
    if (rc) return rc;
    if (n == 0) return CSPQ_OK;
    return encode_subspace_major(P, n, m, sub, CB, B, k, assign, variant, as_stream(stream));
}

int cspq_encode_host(const void *X_host, int32_t in_dtype, int64_t n, int32_t d, const float *CB, const float *B,
                     const float *guard, const void *tc_img, int32_t m, int32_t k, int32_t sub, void *codes_host,
                     int32_t variant, int32_t mode, int64_t batch_rows, int32_t n_streams, double *batch_ms,
                     int32_t device) {
    int rc = check_shape(n, m, k, sub);
    if (rc) return rc;
    CSPQ_REQUIRE(d == m * sub, CSPQ_E_CONFIG,
                 "dataset dimensionality %d does not match codebooks' d=%d", d, m * sub);
    CSPQ_REQUIRE(batch_rows >= 1 && n_streams >= 1 && n_streams <= 16, CSPQ_E_CONFIG, "bad pipeline shape");
    CSPQ_REQUIRE(device >= 0 && device < 64, CSPQ_E_CONFIG, "bad device %d", device);
    if (n == 0) return CSPQ_OK;
    CSPQ_CUDA_TRY(cudaSetDevice(device));
    Pipeline &P = g_pipes[device];
    std::lock_guard<std::mutex> lock(P.mu);
    const size_t esz = in_dtype == CSPQ_IN_U8 ? 1 : 4;
    const size_t cb = k <= 256 ? 1 : 2;
    const size_t xrow = (size_t)d * esz, crow = (size_t)m * cb;
    // buffers for what this call can use (a 10-row call does not pin a 600 MB ring)
    batch_rows = std::min<int64_t>(batch_rows, n);
    if ((rc = P.ensure(n_streams, batch_rows * xrow, batch_rows * crow))) return rc;
    bool pin_in = is_pinned(X_host);
    const bool pin_out = is_pinned(codes_host);
    // pageable input: staged batch by batch through the pinned ring by a multi-threaded copy
    // (30.8 GB/s of rows on the B200 box); CSPQ_HOST_REGISTER=1 page-locks the caller's array
    // for the call instead (cudaHostRegister + DMA: 9.4 GB/s there -- registration dominates;
    // scripts/probe_pageable.py)
    bool registered = false;
    if (!pin_in) {
        const char *env = getenv("CSPQ_HOST_REGISTER");
        const size_t in_bytes = (size_t)n * xrow;
        const bool want = env && atoi(env) != 0;
        void *hp = const_cast<void *>(X_host);
        if (want && (cudaHostRegister(hp, in_bytes, cudaHostRegisterReadOnly) == cudaSuccess ||
                     (cudaGetLastError(), cudaHostRegister(hp, in_bytes, cudaHostRegisterDefault) == cudaSuccess))) {
            registered = pin_in = true;
        } else {
            cudaGetLastError();  // registration refused (e.g. already registered, or unsupported): stage instead
        }
    }
    const bool needs_guard = variant != CSPQ_VARIANT_REFERENCE && mode != CSPQ_MODE_EXACT;
    const int64_t nb = (n + batch_rows - 1) / batch_rows;
    std::vector<int64_t> slot_batch(n_streams, -1);
    auto retire = [&](int s) -> int {
        const int64_t b = slot_batch[s];
        if (b < 0) return CSPQ_OK;
        CSPQ_CUDA_TRY(cudaEventSynchronize(P.ev1[s]));
        const int64_t r0 = b * batch_rows, rows = std::min<int64_t>(batch_rows, n - r0);
        if (!pin_out) par_memcpy((char *)codes_host + r0 * crow, P.hC[s], rows * crow);
        if (batch_ms) {
            float ms = 0.f;
            CSPQ_CUDA_TRY(cudaEventElapsedTime(&ms, P.ev0[s], P.ev1[s]));
            batch_ms[b] = ms;
        }
        slot_batch[s] = -1;
        return CSPQ_OK;
    };
    auto run = [&]() -> int {
        int rc2;
        if (needs_guard && !guard) {
            if (P.guard_floats < (size_t)2 * m) {
                if (P.guard) cudaFree(P.guard);
                P.guard = nullptr;
                P.guard_floats = 0;
                CSPQ_CUDA_TRY(cudaMalloc(reinterpret_cast<void **>(&P.guard), sizeof(float) * 2 * m));
                P.guard_floats = 2 * m;
            }
            if ((rc2 = encode_prepare(CB, B, m, k, sub, P.guard, P.st[0]))) return rc2;
            CSPQ_CUDA_TRY(cudaStreamSynchronize(P.st[0]));
            guard = P.guard;
        }
        for (int64_t b = 0; b < nb; ++b) {
            const int s = (int)(b % n_streams);
            if ((rc2 = retire(s))) return rc2;
            const int64_t r0 = b * batch_rows, rows = std::min<int64_t>(batch_rows, n - r0);
            const char *src = (const char *)X_host + r0 * xrow;
            if (!pin_in) {
                par_memcpy(P.hX[s], src, rows * xrow);
                src = (const char *)P.hX[s];
            }
            cudaStream_t st = P.st[s];
            CSPQ_CUDA_TRY(cudaEventRecord(P.ev0[s], st));
            CSPQ_CUDA_TRY(cudaMemcpyAsync(P.dX[s], src, rows * xrow, cudaMemcpyHostToDevice, st));
            slot_batch[s] = b;  // from here on the stream may touch the caller's buffers
            if (tc_img && variant != CSPQ_VARIANT_REFERENCE)
                rc2 = encode_tc(P.dX[s], in_dtype, rows, d, CB, B, guard, tc_img, m, k, sub,
                                reinterpret_cast<uint8_t *>(P.dC[s]), m, nullptr, st);
            else
                rc2 = encode_device(P.dX[s], in_dtype, rows, d, d, CB, B, guard, m, k, sub, P.dC[s], m, variant,
                                    mode, st);
            if (rc2) return rc2;
            void *dst = pin_out ? (char *)codes_host + r0 * crow : P.hC[s];
            CSPQ_CUDA_TRY(cudaMemcpyAsync(dst, P.dC[s], rows * crow, cudaMemcpyDeviceToHost, st));
            CSPQ_CUDA_TRY(cudaEventRecord(P.ev1[s], st));
        }
        for (int s = 0; s < n_streams; ++s)
            if ((rc2 = retire(s))) return rc2;
        return CSPQ_OK;
    };
    rc = run();
    if (rc != CSPQ_OK) {
        // never return while copies into / out of the caller's buffers are still in flight
        for (int s = 0; s < P.ns; ++s) cudaStreamSynchronize(P.st[s]);
        cudaGetLastError();
    }
    if (registered) cudaHostUnregister(const_cast<void *>(X_host));
    return rc;
}

size_t cspq_crc32_workspace_bytes(int64_t n) { return crc32_workspace_bytes(n); }

int cspq_adc_tables(const float *Q, int64_t nq, int32_t d, const float *CB, int32_t m, int32_t k, int32_t sub,
                    float *tables, void *stream) {
    int rc = check_shape(nq, m, k, sub);
    if (rc) return rc;
    CSPQ_REQUIRE(d == m * sub, CSPQ_E_CONFIG, "query length %d does not match d=%d", d, m * sub);
    if (nq == 0) return CSPQ_OK;
    CSPQ_REQUIRE(Q && CB && tables, CSPQ_E_CONFIG, "null pointer");
    return adc_tables(Q, nq, d, CB, m, k, sub, tables, as_stream(stream));
}

int cspq_adc_scores(const float *tables, int64_t nq, const void *codes, int64_t n, int32_t m, int32_t k, float *scores,
                    void *stream) {
    int rc = check_shape(n, m, k, 1);
    if (rc) return rc;
    CSPQ_REQUIRE(nq >= 0, CSPQ_E_CONFIG, "nq must be >= 0");
    if (nq == 0 || n == 0) return CSPQ_OK;
    CSPQ_REQUIRE(tables && codes && scores, CSPQ_E_CONFIG, "null pointer");
    return adc_scores(tables, nq, codes, k <= 256 ? 1 : 2, n, m, k, scores, as_stream(stream));
}

int cspq_topn(const void *values, int32_t value_bytes, int64_t nq, int64_t n, int32_t topn, int64_t *indices,
              void *top_values, void *stream) {
    CSPQ_REQUIRE(value_bytes == 4 || value_bytes == 8, CSPQ_E_CONFIG, "value_bytes must be 4 (f32) or 8 (f64)");
    CSPQ_REQUIRE(nq >= 0 && n >= 0, CSPQ_E_CONFIG, "bad shape");
    if (nq == 0) return CSPQ_OK;
    CSPQ_REQUIRE(values && indices && top_values, CSPQ_E_CONFIG, "null pointer");
    return topn_select(values, value_bytes, nq, n, topn, indices, top_values, as_stream(stream));
}

int cspq_exact_distances(const float *queries, int64_t nq, const float *db, int64_t n, int32_t d, double *norms,
                         double *dist, void *stream) {
    CSPQ_REQUIRE(nq >= 0 && n >= 0 && d >= 1, CSPQ_E_CONFIG, "bad shape");
    if (nq == 0 || n == 0) return CSPQ_OK;
    CSPQ_REQUIRE(queries && db && norms && dist, CSPQ_E_CONFIG, "null pointer");
    return gt_distances(queries, nq, db, n, d, norms, dist, as_stream(stream));
}

int cspq_crc32_device(const void *data, int64_t n, uint32_t crc_in, uint32_t *crc_out, void *workspace,
                      void *stream) {
    CSPQ_REQUIRE(n >= 0, CSPQ_E_CONFIG, "n must be >= 0");
    CSPQ_REQUIRE(crc_out && workspace && (data || n == 0), CSPQ_E_CONFIG, "null pointer");
    return crc32_device_api(data, n, crc_in, crc_out, workspace, as_stream(stream));
}

uint32_t cspq_crc32_combine(uint32_t crc_a, uint32_t crc_b, int64_t len_b) {
    return crc32_combine_host(crc_a, crc_b, len_b);
}

int cspq_unpack_vecs(const void *records, int64_t n, int32_t d, int32_t value_bytes, int32_t check_finite,
                     int64_t offset0, void *rows, uint64_t *bad, void *stream) {
    CSPQ_REQUIRE(n >= 0 && d >= 1, CSPQ_E_CONFIG, "bad shape");
    CSPQ_REQUIRE(value_bytes == 1 || value_bytes == 4, CSPQ_E_CONFIG, "value_bytes must be 1 or 4");
    if (n == 0) return CSPQ_OK;
    CSPQ_REQUIRE(records && rows && bad, CSPQ_E_CONFIG, "null pointer");
    return unpack_vecs(records, n, d, value_bytes, check_finite, offset0, rows,
                       reinterpret_cast<unsigned long long *>(bad), as_stream(stream));
}

int cspq_encode_vecs_file(const char *in_path, int32_t in_format, const char *out_path, const float *CB,
                          const float *B, const float *guard, const void *tc_img, int32_t m, int32_t k, int32_t sub,
                          int32_t variant, int32_t mode, int64_t batch_rows, int32_t n_streams, int32_t device,
                          int64_t *n_rows, int64_t *err) {
    int rc = check_shape(0, m, k, sub);
    if (rc) return rc;
    CSPQ_REQUIRE(in_path && out_path && n_rows && err && CB, CSPQ_E_CONFIG, "null pointer");
    CSPQ_REQUIRE(in_format == 0 || in_format == 1, CSPQ_E_CONFIG, "in_format must be 0 (fvecs) or 1 (bvecs)");
    CSPQ_REQUIRE(variant >= 0 && variant <= 2 && mode >= 0 && mode <= 2, CSPQ_E_CONFIG, "bad variant/mode");
    CSPQ_REQUIRE(B || variant == CSPQ_VARIANT_REFERENCE, CSPQ_E_CONFIG, "null biases");
    CSPQ_REQUIRE(batch_rows >= 1 && n_streams >= 1 && n_streams <= 8, CSPQ_E_CONFIG, "bad pipeline shape");
    CSPQ_REQUIRE(device >= 0 && device < 64, CSPQ_E_CONFIG, "bad device %d", device);
    return encode_vecs_file(in_path, in_format, out_path, CB, B, guard, tc_img, m, k, sub, variant, mode, batch_rows,
                            n_streams, device, n_rows, err);
}

size_t cspq_lloyd_workspace_bytes(int64_t n, int32_t m, int32_t sub, int32_t k) {
    return lloyd_workspace_bytes(n, m, sub, k);
}

#define CSPQ_LLOYD_CHECK(n, m, sub, k, P, ws)                                                   \
    do {                                                                                        \
        int rc_ = check_shape(n, m, k, sub);                                                    \
        if (rc_) return rc_;                                                                    \
        CSPQ_REQUIRE((P) && (ws), CSPQ_E_CONFIG, "null points or workspace");                   \
        CSPQ_REQUIRE((n) <= 0x7fffffffLL, CSPQ_E_CONFIG, "training sample too large (%lld)", (long long)(n)); \
    } while (0)

int cspq_lloyd_assign(const void *P, int32_t p_f64, int64_t n, int32_t m, int32_t sub, int32_t k, const double *C64,
                      const int32_t *state, int64_t row_begin, int64_t row_end, int32_t *assign, double *sq,
                      void *workspace, void *stream) {
    CSPQ_LLOYD_CHECK(n, m, sub, k, P, workspace);
    CSPQ_REQUIRE(0 <= row_begin && row_begin <= row_end && row_end <= n, CSPQ_E_CONFIG, "bad row range");
    return lloyd_assign(P, p_f64, n, m, sub, k, C64, state, row_begin, row_end, assign, sq, workspace,
                        as_stream(stream));
}

int cspq_lloyd_accumulate(const void *P, int32_t p_f64, int64_t n, int32_t m, int32_t sub, int32_t k,
                          const int32_t *state, const int32_t *assign, const double *sq, int64_t row_begin,
                          int64_t row_end, double *counts, double *sums, double *obj, void *workspace,
                          void *stream) {
    CSPQ_LLOYD_CHECK(n, m, sub, k, P, workspace);
    CSPQ_REQUIRE(0 <= row_begin && row_begin <= row_end && row_end <= n, CSPQ_E_CONFIG, "bad row range");
    return lloyd_accumulate(P, p_f64, n, m, sub, k, state, assign, sq, row_begin, row_end, counts, sums, obj,
                            workspace, as_stream(stream));
}

int cspq_lloyd_update(const double *counts, const double *sums, int32_t m, int32_t k, int32_t sub,
                      const int32_t *state, double *C64, int32_t *empties, int32_t *n_empty, void *stream) {
    int rc = check_shape(0, m, k, sub);
    if (rc) return rc;
    return lloyd_update(counts, sums, m, k, sub, state, C64, empties, n_empty, as_stream(stream));
}

int cspq_lloyd_repair(const void *P, int32_t p_f64, int64_t n, int32_t m, int32_t sub, int32_t k,
                      const int32_t *assign, const int32_t *state, const int32_t *empties, const int32_t *n_empty,
                      double *C64, void *workspace, void *stream) {
    CSPQ_LLOYD_CHECK(n, m, sub, k, P, workspace);
    return lloyd_repair(P, p_f64, n, m, sub, k, assign, state, empties, n_empty, C64, workspace, as_stream(stream));
}

int cspq_lloyd_stop(const double *obj, int32_t m, int32_t max_iters, double tol, int32_t *state, double *prev,
                    int32_t *iterations, double *objectives, void *stream) {
    CSPQ_REQUIRE(m >= 1 && max_iters >= 1 && tol >= 0, CSPQ_E_CONFIG, "bad stop arguments");
    return lloyd_stop(obj, m, max_iters, tol, state, prev, iterations, objectives, as_stream(stream));
}

int cspq_lloyd_train(const void *P, int32_t p_f64, int64_t n, int32_t m, int32_t sub, int32_t k, double *C64,
                     int32_t max_iters, double tol, float *C32, int32_t *assign, double *objectives,
                     int32_t *iterations, void *workspace, void *stream) {
    CSPQ_LLOYD_CHECK(n, m, sub, k, P, workspace);
    CSPQ_REQUIRE(n >= 1, CSPQ_E_TRAINING, "need at least one training point");
    CSPQ_REQUIRE(max_iters >= 1, CSPQ_E_TRAINING, "max_iters must be >= 1, got %d", max_iters);
    CSPQ_REQUIRE(tol >= 0, CSPQ_E_TRAINING, "tol must be >= 0");
    return lloyd_train(P, p_f64, n, m, sub, k, C64, max_iters, tol, C32, assign, objectives, iterations, workspace,
                       as_stream(stream));
}

int cspq_lloyd_final_objective(const void *P, int32_t p_f64, int64_t n, int32_t m, int32_t sub, int32_t k,
                               const float *C32, const int32_t *assign, double *obj, void *workspace, void *stream) {
    CSPQ_LLOYD_CHECK(n, m, sub, k, P, workspace);
    return lloyd_final_objective(P, p_f64, n, m, sub, k, C32, assign, obj, workspace, as_stream(stream));
}

int cspq_kmeanspp(const void *P, int32_t p_f64, int64_t n, int32_t m, int32_t sub, int32_t k, const int64_t *first,
                  const double *u, double *C64, int32_t *status, void *workspace, void *stream) {
    CSPQ_LLOYD_CHECK(n, m, sub, k, P, workspace);
    CSPQ_REQUIRE(n >= 1, CSPQ_E_TRAINING, "need at least one training point");
    return kmeanspp(P, p_f64, n, m, sub, k, first, u, C64, status, workspace, as_stream(stream));
}

}  // extern "C"
