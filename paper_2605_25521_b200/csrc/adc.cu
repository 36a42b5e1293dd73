// adc.cu -- flat ADC search and its exact ground truth on the GPU (SURVEY.md §8(f)
// row 4; reference /root/reference/pkg/src/cspq/evaluation.py).
//
//   tables[q, j, l] = sum_t (c_jl[t] - q_j[t])^2  in float32, summed the way numpy's
//       einsum("kt,kt->k") does it (evaluation.py:66-74): four strided partial sums
//       acc[t % 4] in t order, then (acc0 + acc1) + (acc2 + acc3); bit-identical to the
//       reference for sub <= 12 (measured; every configuration), one rounding apart above.
//   scores[q, i]   = ((0 + T[0][c_i0]) + T[1][c_i1]) + ...  float32 in chunk order
//       (evaluation.py:91-96).
//   top-N          = the N smallest (score, index) pairs in lexsort order
//       (evaluation.py:99-103): a radix select over unique keys (orderable float bits,
//       then the index) finds the N-th pair, the <= N survivors are compacted and
//       bitonic-sorted in shared memory.  No ties or NaN ordering question is left open:
//       NaN maps above +inf, as lexsort places it.
//   ground truth   = the same selection over float64 distances ||x||^2 - 2 q.x
//       (evaluation.py:114-129; ascending-t fused products: neighbour lists equal the
//       reference's except for float64 near-ties of dgemm's summation order).

#include <cstdint>

#include "common.cuh"

namespace cspq {
namespace {

constexpr int kSelThreads = 1024;
constexpr int kMaxTopN = 1024;

__device__ __forceinline__ uint32_t f32_key(float f) {
    uint32_t u = __float_as_uint(f);
    if (f != f) return 0xffffffffu;  // NaN after +inf (lexsort)
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ uint64_t f64_key(double f) {
    uint64_t u = (uint64_t)__double_as_longlong(f);
    if (f != f) return ~0ull;
    return (u >> 63) ? ~u : (u | (1ull << 63));
}

// tables (nq, m, k): one thread per (q, j, l)
__global__ void adc_tables_kernel(const float *__restrict__ Q, int64_t nq, int d, const float *__restrict__ CB, int m,
                                  int k, int sub, float *__restrict__ T) {
    const int64_t total = nq * m * (int64_t)k;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
        const int l = (int)(g % k);
        const int64_t qj = g / k;
        const int j = (int)(qj % m);
        const int64_t q = qj / m;
        const float *c = CB + ((int64_t)j * k + l) * sub;
        const float *x = Q + q * d + (int64_t)j * sub;
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        for (int t = 0; t < sub; ++t) {
            const float df = __fsub_rn(c[t], x[t]);
            acc[t & 3] = __fadd_rn(acc[t & 3], __fmul_rn(df, df));
        }
        T[g] = __fadd_rn(__fadd_rn(acc[0], acc[1]), __fadd_rn(acc[2], acc[3]));
    }
}

// scores (nq, n): tables of one query staged in shared memory, one thread per row
template <typename C>
__global__ void adc_scores_kernel(const float *__restrict__ T, const C *__restrict__ codes, int64_t n, int m, int k,
                                  float *__restrict__ S) {
    extern __shared__ float sT[];
    const int64_t q = blockIdx.y;
    const float *Tq = T + q * (int64_t)m * k;
    for (int i = threadIdx.x; i < m * k; i += blockDim.x) sT[i] = Tq[i];
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const C *ci = codes + i * m;
        float s = 0.f;
        for (int j = 0; j < m; ++j) s = __fadd_rn(s, sT[j * k + ci[j]]);
        S[q * n + i] = s;
    }
}

// float64 squared norms of the database rows (ascending t, fused)
__global__ void row_norms_kernel(const float *__restrict__ X, int64_t n, int d, double *__restrict__ nrm) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float *x = X + i * d;
        double s = 0.0;
        for (int t = 0; t < d; ++t) s = fma((double)x[t], (double)x[t], s);
        nrm[i] = s;
    }
}

// D[q, i] = ||x_i||^2 - 2 q.x_i in float64; 32 x 32 tiles of (query, row), d in 32-wide slabs
__global__ void gt_dist_kernel(const float *__restrict__ Qm, int64_t nq, const float *__restrict__ X, int64_t n, int d,
                               const double *__restrict__ nrm, double *__restrict__ D) {
    __shared__ double sq[32][33], sx[32][33];
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8 threads, 4 queries each
    const int64_t i0 = blockIdx.x * 32, q0 = blockIdx.y * 32;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int t0 = 0; t0 < d; t0 += 32) {
        for (int r = ty; r < 32; r += 8) {
            const int64_t qi = q0 + r, xi = i0 + r;
            const int t = t0 + tx;
            sq[r][tx] = (qi < nq && t < d) ? (double)Qm[qi * d + t] : 0.0;
            sx[r][tx] = (xi < n && t < d) ? (double)X[xi * d + t] : 0.0;
        }
        __syncthreads();
        const int tl = d - t0 < 32 ? d - t0 : 32;
        for (int t = 0; t < tl; ++t) {
            const double xv = sx[tx][t];
#pragma unroll
            for (int a = 0; a < 4; ++a) acc[a] = fma(sq[ty + 8 * a][t], xv, acc[a]);
        }
        __syncthreads();
    }
    const int64_t i = i0 + tx;
    if (i < n)
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const int64_t q = q0 + ty + 8 * a;
            if (q < nq) D[q * n + i] = nrm[i] - 2.0 * acc[a];
        }
}

// ---- per-query exact top-N selection: one CTA per query ----
// An element's ordering value is (key, index), key 32 bits (float32 scores) or 64 bits
// (float64 distances), index 32 bits: digits are taken 8 bits at a time from the top.
template <bool K64>
struct Sel {
    static constexpr int kKeyBits = K64 ? 64 : 32;
    static constexpr int kPasses = (kKeyBits + 32) / 8;
    __device__ static uint64_t key(const void *v, int64_t i) {
        if constexpr (K64) return f64_key(reinterpret_cast<const double *>(v)[i]);
        else return f32_key(reinterpret_cast<const float *>(v)[i]);
    }
    // digit p (0 = most significant) of (key, index)
    __device__ static uint32_t digit(uint64_t k, uint32_t idx, int p) {
        const int bit = kKeyBits + 32 - 8 * (p + 1);
        if (bit >= 32) return (uint32_t)(k >> (bit - 32)) & 0xff;
        return (idx >> bit) & 0xff;
    }
    // does (k, idx) agree with the chosen prefix on digits < p
    __device__ static bool match(uint64_t k, uint32_t idx, int p, uint64_t pk, uint32_t pi) {
        for (int q = 0; q < p; ++q)
            if (digit(k, idx, q) != digit(pk, pi, q)) return false;
        return true;
    }
};

template <bool K64>
__global__ void __launch_bounds__(kSelThreads) topn_kernel(const void *__restrict__ vals, int64_t n, int topn,
                                                           int64_t *__restrict__ out_idx, void *__restrict__ out_val) {
    using SL = Sel<K64>;
    __shared__ uint32_t hist[256];
    __shared__ uint64_t s_pk;
    __shared__ uint32_t s_pi, s_rank, s_cnt;
    __shared__ uint64_t ck[kMaxTopN];
    __shared__ uint32_t ci[kMaxTopN];
    const int tid = threadIdx.x;
    const int64_t q = blockIdx.x;
    const char *base = reinterpret_cast<const char *>(vals) + q * n * (K64 ? 8 : 4);
    if (tid == 0) { s_pk = 0; s_pi = 0; s_rank = (uint32_t)topn; }  // want the topn-th smallest (1-based)
    __syncthreads();
    for (int p = 0; p < SL::kPasses; ++p) {
        for (int b = tid; b < 256; b += blockDim.x) hist[b] = 0;
        __syncthreads();
        const uint64_t pk = s_pk;
        const uint32_t pi = s_pi;
        for (int64_t i = tid; i < n; i += blockDim.x) {
            const uint64_t kk = SL::key(base, i);
            if (SL::match(kk, (uint32_t)i, p, pk, pi)) atomicAdd(&hist[SL::digit(kk, (uint32_t)i, p)], 1u);
        }
        __syncthreads();
        if (tid == 0) {
            uint32_t r = s_rank, b = 0;
            while (hist[b] < r) { r -= hist[b]; ++b; }
            s_rank = r;
            const int bit = SL::kKeyBits + 32 - 8 * (p + 1);
            if (bit >= 32) s_pk |= (uint64_t)b << (bit - 32);
            else s_pi |= b << bit;
        }
        __syncthreads();
    }
    // (s_pk, s_pi) is the topn-th smallest pair: keep every pair <= it (exactly topn)
    const uint64_t tk = s_pk;
    const uint32_t ti = s_pi;
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    for (int64_t i = tid; i < n; i += blockDim.x) {
        const uint64_t kk = SL::key(base, i);
        if (kk < tk || (kk == tk && (uint32_t)i <= ti)) {
            const uint32_t slot = atomicAdd(&s_cnt, 1u);
            if (slot < kMaxTopN) { ck[slot] = kk; ci[slot] = (uint32_t)i; }
        }
    }
    __syncthreads();
    // bitonic sort of topn (padded to a power of two) by (key, index)
    int P = 1;
    while (P < topn) P <<= 1;
    for (int s = tid + topn; s < P; s += blockDim.x) { ck[s] = ~0ull; ci[s] = 0xffffffffu; }
    __syncthreads();
    for (int size = 2; size <= P; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int a = tid; a < P; a += blockDim.x) {
                const int b = a ^ stride;
                if (b > a) {
                    const bool up = (a & size) == 0;
                    const bool gt = ck[a] > ck[b] || (ck[a] == ck[b] && ci[a] > ci[b]);
                    if (gt == up) {
                        const uint64_t t1 = ck[a]; ck[a] = ck[b]; ck[b] = t1;
                        const uint32_t t2 = ci[a]; ci[a] = ci[b]; ci[b] = t2;
                    }
                }
            }
            __syncthreads();
        }
    for (int s = tid; s < topn; s += blockDim.x) {
        const uint32_t i = ci[s];
        out_idx[q * topn + s] = i;
        if constexpr (K64) reinterpret_cast<double *>(out_val)[q * topn + s] = reinterpret_cast<const double *>(base)[i];
        else reinterpret_cast<float *>(out_val)[q * topn + s] = reinterpret_cast<const float *>(base)[i];
    }
}

int grid_for(int64_t work, int threads) {
    const int64_t g = (work + threads - 1) / threads;
    return (int)(g < 148 * 32 ? (g < 1 ? 1 : g) : 148 * 32);
}

}  // namespace

int adc_tables(const float *Q, int64_t nq, int d, const float *CB, int m, int k, int sub, float *T, cudaStream_t st) {
    if (nq == 0) return CSPQ_OK;
    adc_tables_kernel<<<grid_for(nq * m * (int64_t)k, 256), 256, 0, st>>>(Q, nq, d, CB, m, k, sub, T);
    CSPQ_LAUNCH_CHECK();
    return CSPQ_OK;
}

int adc_scores(const float *T, int64_t nq, const void *codes, int code_bytes, int64_t n, int m, int k, float *S,
               cudaStream_t st) {
    if (nq == 0 || n == 0) return CSPQ_OK;
    const size_t smem = (size_t)m * k * sizeof(float);
    CSPQ_REQUIRE(smem <= 200 * 1024, CSPQ_E_CONFIG, "ADC tables of one query (%d x %d) exceed shared memory", m, k);
    CSPQ_REQUIRE(nq <= 65535, CSPQ_E_CONFIG, "at most 65535 queries per call");
    const dim3 grid((unsigned)((n + 255) / 256 < 148 * 8 ? (n + 255) / 256 : 148 * 8), (unsigned)nq);
    if (code_bytes == 1) {
        auto kern = adc_scores_kernel<uint8_t>;
        CSPQ_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<grid, 256, smem, st>>>(T, reinterpret_cast<const uint8_t *>(codes), n, m, k, S);
    } else {
        auto kern = adc_scores_kernel<uint16_t>;
        CSPQ_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<grid, 256, smem, st>>>(T, reinterpret_cast<const uint16_t *>(codes), n, m, k, S);
    }
    CSPQ_LAUNCH_CHECK();
    return CSPQ_OK;
}

int topn_select(const void *vals, int val_bytes, int64_t nq, int64_t n, int topn, int64_t *idx, void *out_vals,
                cudaStream_t st) {
    if (nq == 0 || topn == 0) return CSPQ_OK;
    CSPQ_REQUIRE(topn >= 1 && topn <= kMaxTopN && topn <= n, CSPQ_E_CONFIG, "topn must be in [1, min(n, %d)]", kMaxTopN);
    CSPQ_REQUIRE(n <= 0xffffffffll, CSPQ_E_CONFIG, "at most 2^32 - 1 database rows");
    CSPQ_REQUIRE(nq <= 0x7fffffffll, CSPQ_E_CONFIG, "too many queries");
    if (val_bytes == 8) topn_kernel<true><<<(unsigned)nq, kSelThreads, 0, st>>>(vals, n, topn, idx, out_vals);
    else topn_kernel<false><<<(unsigned)nq, kSelThreads, 0, st>>>(vals, n, topn, idx, out_vals);
    CSPQ_LAUNCH_CHECK();
    return CSPQ_OK;
}

int gt_distances(const float *Qm, int64_t nq, const float *X, int64_t n, int d, double *nrm, double *D,
                 cudaStream_t st) {
    if (nq == 0 || n == 0) return CSPQ_OK;
    row_norms_kernel<<<grid_for(n, 256), 256, 0, st>>>(X, n, d, nrm);
    CSPQ_LAUNCH_CHECK();
    CSPQ_REQUIRE((nq + 31) / 32 <= 65535, CSPQ_E_CONFIG, "too many queries per call");
    gt_dist_kernel<<<dim3((unsigned)((n + 31) / 32), (unsigned)((nq + 31) / 32)), dim3(32, 8), 0, st>>>(Qm, nq, X, n, d,
                                                                                                     nrm, D);
    CSPQ_LAUNCH_CHECK();
    return CSPQ_OK;
}

}  // namespace cspq
