// encode.cu -- PQ encode kernels for sm_100a.
//
// Replaces the reference's bulk driver _drive_chunk_major and the kernels it
// calls (/root/reference/pkg/src/cspq/kernels.py:84-316, driven from
// bulk.py:108-157).  For every (row i, subspace j) the code is
//     argmin_l  s_l,   s_l = b_l - sum_t x_t * c_{l,t}      (REFORMULATED/BLOCKED)
// or  argmin_l  (vv + cc_l) - 2 * dd_l                        (REFERENCE)
// with the oracle's tie rule (strict '<' from +inf: first index wins, NaN
// never wins, all-NaN -> 0).  The oracle scores are strict IEEE fp32 with a
// separate rounding per multiply and per add (kernels.py:4-9).
//
// Two arithmetic modes, both returning the oracle's codes bit for bit:
//  * EXACT   -- the oracle's own chains (__fmul_rn / __fadd_rn, ascending t).
//  * GUARDED -- one FFMA per MAC with the bias folded in (s = fma(-x_t, c_t, .. b)),
//               plus a rigorous forward-error guard: |s_ffma - s_oracle| <=
//               E = 2*gamma_{sub+1} * (|b| + ||x|| ||c||).  A (row, subspace)
//               whose runner-up approximate score lies within 2E (x2 safety)
//               of the best is "flagged" and re-encoded exactly by its warp
//               (lanes split the centroids, warp-shuffle argmin).  Unflagged
//               codes are provably the oracle's.
//
// Kernel shape (fast path, k == 256, sub in {4, 8}): a CTA owns a tile of
// 128*R rows and walks all m subspaces chunk-major (one codebook resident
// while the tile streams through it -- the paper's cache idea).
// Codebook j+1 and the tile's subvectors for j+1 are staged into shared
// memory with cp.async while subspace j is computed.  Each thread keeps R
// rows' subvectors in registers and sweeps all 256 centroids from shared
// memory with warp-uniform (broadcast) loads: "vectorising across
// centroids" becomes one thread scoring every centroid against R rows,
// which keeps the FFMA pipe busy with no cross-lane reductions.  The argmin
// runs on blocks of 8 centroids: block minimum with 3-input FMNMX3, running
// best/runner-up per row, and the winner's in-block index recovered at the
// end by re-scoring the winning block.

#include "common.cuh"

namespace cspq {

namespace {

constexpr int kK = 256;    // centroids (fast path)
constexpr int kBlk = 8;    // centroids per argmin block

template <typename TIn>
__device__ __forceinline__ float to_f(TIn v) { return static_cast<float>(v); }

// strict oracle chain: dd = x0*c0 (+) x1*c1 (+) ... ; s = b - dd
template <int SUB>
__device__ __forceinline__ float score_exact(const float (&x)[SUB], const float *c, float b) {
    float dd = __fmul_rn(x[0], c[0]);
#pragma unroll
    for (int t = 1; t < SUB; ++t) dd = __fadd_rn(dd, __fmul_rn(x[t], c[t]));
    return __fsub_rn(b, dd);
}

// FFMA chain with the bias folded: s = fma(nx_{SUB-1}, c, ... fma(nx_0, c_0, b))
template <int SUB>
__device__ __forceinline__ float score_ffma(const float (&nx)[SUB], const float *c, float b) {
    float a = b;
#pragma unroll
    for (int t = 0; t < SUB; ++t) a = __fmaf_rn(nx[t], c[t], a);
    return a;
}

template <int SUB>
__device__ __forceinline__ void load_cent(const float *p, float (&c)[SUB]) {
    if constexpr (SUB % 4 == 0) {
#pragma unroll
        for (int q = 0; q < SUB / 4; ++q) {
            float4 v = reinterpret_cast<const float4 *>(p)[q];
            c[4 * q + 0] = v.x; c[4 * q + 1] = v.y; c[4 * q + 2] = v.z; c[4 * q + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int t = 0; t < SUB; ++t) c[t] = p[t];
    }
}

// tiling of the fast kernel (cspq_encode_set_tiling; default 3, the fastest
// on B200 in scripts/sweep_tiling.py): 0 = R8/T128/2 CTAs,
// 1 = R8/T128/3, 2 = R4/T256/2, 3 = R4/T128/4 -- codes never depend on it
int g_tiling = 3;

// flagged-subvector counter (telemetry: cspq_encode_stats)
__device__ unsigned long long g_flagged = 0;

// gamma_n = n u / (1 - n u), u = 2^-24
__host__ __device__ constexpr double gamma_n(int n) { return n * 5.9604644775390625e-8 / (1.0 - n * 5.9604644775390625e-8); }

// Shared-memory codebook: one record per block of kBlk centroids = the
// block's centroids (kBlk*SUB floats) followed by its kBlk biases, padded
// to an odd number of 16-byte chunks so that lanes reading different
// records (the winner-block re-score) spread over all 8 bank groups.
template <int SUB>
struct Rec {
    static constexpr int kChunks = (kBlk * SUB + kBlk) / 4;                 // 16-byte chunks of payload
    static constexpr int kStride = (kChunks % 2 == 0) ? kChunks + 1 : kChunks;  // chunks per record
    static constexpr int kFloats = kStride * 4;
    static constexpr int kBias = kBlk * SUB;                                 // bias offset in a record
    static constexpr int kTotal = (kK / kBlk) * kFloats;                     // floats per staged codebook
};

template <int SUB, typename TIn>
struct TileCopy {
    static constexpr int kBytes = SUB * (int)sizeof(TIn);
    __device__ __forceinline__ static void copy(TIn *dst, const TIn *src, bool valid) {
        const int sb = valid ? 16 : 0;
        if constexpr (kBytes == 32) {
            cp_async16(dst, src, sb);
            cp_async16(dst + 16 / sizeof(TIn), src + 16 / sizeof(TIn), sb);
        } else if constexpr (kBytes == 16) {
            cp_async16(dst, src, sb);
        } else if constexpr (kBytes == 8) {
            cp_async8(dst, src, valid ? 8 : 0);
        } else {
            static_assert(kBytes == 4, "unsupported subvector width");
            cp_async4(dst, src, valid ? 4 : 0);
        }
    }
};

// ---------------------------------------------------------------------------
// Fast path: k = 256, sub in {4, 8}, f32 or u8 rows.
// ---------------------------------------------------------------------------
template <int SUB, int R, int kT, int MINB, typename TIn, bool EXACT>
__global__ void __launch_bounds__(kT, MINB)
encode_k256_kernel(const TIn *__restrict__ X, int64_t n, int m, int64_t xs,
                   const float *__restrict__ CB, const float *__restrict__ B,
                   const float *__restrict__ guard, uint8_t *__restrict__ codes, int64_t cs) {
    using RC = Rec<SUB>;
    constexpr int CBF = RC::kTotal;     // floats per staged codebook (records)
    constexpr int XE = R * kT * SUB;    // elements per staged x tile
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float *cbuf = reinterpret_cast<float *>(smem_raw);
    TIn *xbuf = reinterpret_cast<TIn *>(cbuf + 2 * CBF);

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int64_t row0 = (int64_t)blockIdx.x * (kT * R);

    auto issue = [&](int j, int buf) {
        const float *gc = CB + (int64_t)j * kK * SUB;
        const float *gb = B + (int64_t)j * kK;
        float *sc = cbuf + buf * CBF;
        constexpr int CPB = kBlk * SUB / 4;  // centroid chunks per record
        for (int q = tid; q < (kK / kBlk) * (CPB + kBlk / 4); q += kT) {
            const int rec = q / (CPB + kBlk / 4), w = q % (CPB + kBlk / 4);
            float *dst = sc + rec * RC::kFloats + 4 * w;
            const float *src = w < CPB ? gc + (rec * kBlk * SUB + 4 * w) : gb + (rec * kBlk + 4 * (w - CPB));
            cp_async16(dst, src);
        }
        TIn *sx = xbuf + buf * XE;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t row = row0 + r * kT + tid;
            const bool valid = row < n;
            const TIn *src = X + (valid ? row * xs + (int64_t)j * SUB : 0);
            TileCopy<SUB, TIn>::copy(sx + (r * kT + tid) * SUB, src, valid);
        }
        cp_async_commit();
    };

    issue(0, 0);
    for (int j = 0; j < m; ++j) {
        if (j + 1 < m) issue(j + 1, (j + 1) & 1);
        else cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();

        const float *sc = cbuf + (j & 1) * CBF;
        const TIn *sx = xbuf + (j & 1) * XE;

        // this thread's R subvectors (negated for the FFMA chain)
        float x[R][SUB];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const TIn *p = sx + (r * kT + tid) * SUB;
            if constexpr (sizeof(TIn) == 4 && SUB % 4 == 0) {
                float tmp[SUB];
                load_cent<SUB>(reinterpret_cast<const float *>(p), tmp);
#pragma unroll
                for (int t = 0; t < SUB; ++t) x[r][t] = EXACT ? tmp[t] : -tmp[t];
            } else {
#pragma unroll
                for (int t = 0; t < SUB; ++t) x[r][t] = EXACT ? to_f(p[t]) : -to_f(p[t]);
            }
        }

        float m1[R], m2[R];
        int wb[R];
#pragma unroll
        for (int r = 0; r < R; ++r) { m1[r] = pos_inf_f(); m2[r] = pos_inf_f(); wb[r] = 0; }

#pragma unroll 1
        for (int blk = 0; blk < kK / kBlk; ++blk) {
            const float *cblk = sc + blk * RC::kFloats;
            float bb[kBlk];
            {
                const float4 *bp = reinterpret_cast<const float4 *>(cblk + RC::kBias);
#pragma unroll
                for (int q = 0; q < kBlk / 4; ++q) {
                    float4 v = bp[q];
                    bb[4 * q] = v.x; bb[4 * q + 1] = v.y; bb[4 * q + 2] = v.z; bb[4 * q + 3] = v.w;
                }
            }
            float bm[R];
#pragma unroll
            for (int cc = 0; cc < kBlk; cc += 2) {
                float ca[SUB], cb[SUB];
                load_cent<SUB>(cblk + cc * SUB, ca);
                load_cent<SUB>(cblk + (cc + 1) * SUB, cb);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    float sa, sbv;
                    if constexpr (EXACT) {
                        sa = score_exact<SUB>(x[r], ca, bb[cc]);
                        sbv = score_exact<SUB>(x[r], cb, bb[cc + 1]);
                    } else {
                        sa = score_ffma<SUB>(x[r], ca, bb[cc]);
                        sbv = score_ffma<SUB>(x[r], cb, bb[cc + 1]);
                    }
                    bm[r] = (cc == 0) ? fminf(sa, sbv) : fmin3(bm[r], sa, sbv);
                }
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if constexpr (!EXACT) m2[r] = fminf(m2[r], fmaxf(m1[r], bm[r]));
                wb[r] = (bm[r] < m1[r]) ? blk : wb[r];
                m1[r] = fminf(m1[r], bm[r]);
            }
        }

        // resolve each row's code: re-score the winning block for the first index
        float gbmax = 0.f, gcmax = 0.f;
        if constexpr (!EXACT) { gbmax = guard[2 * j]; gcmax = guard[2 * j + 1]; }
        int code[R];
        bool flag[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            code[r] = 0;
            flag[r] = false;
            float thr = m1[r];
            if constexpr (!EXACT) {
                float ss = 0.f;
#pragma unroll
                for (int t = 0; t < SUB; ++t) ss = __fmaf_rn(x[r][t], x[r][t], ss);
                const float nrm = __fsqrt_ru(ss) * 1.000001f;
                constexpr float kG = (float)(8.0 * gamma_n(SUB + 1));
                thr = m1[r] + (kG * (gbmax + nrm * gcmax) + 1e-36f);
            }
            if (m1[r] < pos_inf_f()) {
                const float *rec = sc + wb[r] * RC::kFloats;
                float rb[kBlk];
                {
                    const float4 *bp = reinterpret_cast<const float4 *>(rec + RC::kBias);
#pragma unroll
                    for (int q = 0; q < kBlk / 4; ++q) {
                        float4 v = bp[q];
                        rb[4 * q] = v.x; rb[4 * q + 1] = v.y; rb[4 * q + 2] = v.z; rb[4 * q + 3] = v.w;
                    }
                }
                int first = -1, others = 0;
#pragma unroll
                for (int cc = 0; cc < kBlk; ++cc) {
                    float c[SUB];
                    load_cent<SUB>(rec + cc * SUB, c);
                    const float s = EXACT ? score_exact<SUB>(x[r], c, rb[cc]) : score_ffma<SUB>(x[r], c, rb[cc]);
                    if (first < 0 && s == m1[r]) first = cc;
                    else if (!EXACT && s <= thr) ++others;
                }
                code[r] = wb[r] * kBlk + (first < 0 ? 0 : first);
                if constexpr (!EXACT) flag[r] = (others > 0) || (m2[r] <= thr) || !(thr < pos_inf_f()) || first < 0;
            } else {
                if constexpr (!EXACT) flag[r] = true;  // all approximate scores NaN/inf: decide exactly
            }
        }

        if constexpr (!EXACT) {
            // warp-cooperative exact re-encode of flagged (row, subspace) pairs
#pragma unroll
            for (int r = 0; r < R; ++r) {
                unsigned mask = __ballot_sync(0xffffffffu, flag[r]);
                if (lane == 0 && mask) atomicAdd(&g_flagged, (unsigned long long)__popc(mask));
                while (mask) {
                    const int src = __ffs(mask) - 1;
                    mask &= mask - 1;
                    float xv[SUB];
#pragma unroll
                    for (int t = 0; t < SUB; ++t) xv[t] = -__shfl_sync(0xffffffffu, x[r][t], src);
                    float best = pos_inf_f();
                    int bl = kK;
                    for (int l = lane; l < kK; l += 32) {
                        float c[SUB];
                        const float *rec = sc + (l / kBlk) * RC::kFloats;
                        load_cent<SUB>(rec + (l % kBlk) * SUB, c);
                        const float s = score_exact<SUB>(xv, c, rec[RC::kBias + l % kBlk]);
                        if (s < best) { best = s; bl = l; }
                    }
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) {
                        const float ob = __shfl_xor_sync(0xffffffffu, best, off);
                        const int ol = __shfl_xor_sync(0xffffffffu, bl, off);
                        if (ob < best || (ob == best && ol < bl)) { best = ob; bl = ol; }
                    }
                    if (lane == src) code[r] = (best < pos_inf_f()) ? bl : 0;
                }
            }
        }

#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t row = row0 + r * kT + tid;
            if (row < n) codes[row * cs + j] = static_cast<uint8_t>(code[r]);
        }
        __syncthreads();  // buffer (j & 1) is refilled by issue(j + 2)
    }
}

// ---------------------------------------------------------------------------
// Generic exact path: any k, any sub, any strides; also the REFERENCE variant.
// One thread per (row, subspace); warps share the subspace so centroid loads
// are warp-uniform.
// ---------------------------------------------------------------------------
template <typename TIn, int VARIANT, int SUBC>
__global__ void __launch_bounds__(256)
encode_generic_kernel(const TIn *__restrict__ X, int64_t n, int m, int k, int sub_rt, int64_t xrs,
                      int64_t xss, const float *__restrict__ CB, const float *__restrict__ B,
                      void *__restrict__ codes, int code_bytes, int64_t crs, int64_t css,
                      float *__restrict__ best_out) {
    const int sub = SUBC > 0 ? SUBC : sub_rt;
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    const float *C = CB + (int64_t)j * k * sub;
    // REFERENCE: cc_l = sum_t c_t * c_t does not depend on the row -- the CTA computes the
    // subspace's chains once (the same ascending mul-then-add, so the same bits) for k <= 1024
    constexpr int kCcMax = 1024;
    __shared__ float s_cc[VARIANT == CSPQ_VARIANT_REFERENCE ? kCcMax : 1];
    const bool cc_tab = VARIANT == CSPQ_VARIANT_REFERENCE && k <= kCcMax;
    if (cc_tab) {
        for (int l = threadIdx.x; l < k; l += blockDim.x) {
            float cc = 0.f;
            for (int t = 0; t < sub; ++t) { const float cv = __ldg(C + (int64_t)l * sub + t); cc = __fadd_rn(cc, __fmul_rn(cv, cv)); }
            s_cc[l] = cc;
        }
        __syncthreads();
    }
    if (row >= n) return;
    const TIn *x = X + row * xrs + (int64_t)j * xss;
    float best = pos_inf_f();
    int bidx = 0;
    if constexpr (SUBC > 0) {
        float xv[SUBC];
#pragma unroll
        for (int t = 0; t < SUBC; ++t) xv[t] = to_f(x[t]);
        float vv = 0.f;
        if constexpr (VARIANT == CSPQ_VARIANT_REFERENCE) {
#pragma unroll
            for (int t = 0; t < SUBC; ++t) vv = __fadd_rn(vv, __fmul_rn(xv[t], xv[t]));
        }
        for (int l = 0; l < k; ++l) {
            const float *c = C + (int64_t)l * SUBC;
            float s;
            if constexpr (VARIANT == CSPQ_VARIANT_REFERENCE) {
                float cc = 0.f, dd = 0.f;
                if (cc_tab) {
                    cc = s_cc[l];
#pragma unroll
                    for (int t = 0; t < SUBC; ++t) dd = __fadd_rn(dd, __fmul_rn(xv[t], __ldg(c + t)));
                } else {
#pragma unroll
                    for (int t = 0; t < SUBC; ++t) {
                        const float cv = __ldg(c + t);
                        cc = __fadd_rn(cc, __fmul_rn(cv, cv));
                        dd = __fadd_rn(dd, __fmul_rn(xv[t], cv));
                    }
                }
                s = __fsub_rn(__fadd_rn(vv, cc), __fmul_rn(2.0f, dd));
            } else {
                float dd = 0.f;
#pragma unroll
                for (int t = 0; t < SUBC; ++t) dd = __fadd_rn(dd, __fmul_rn(xv[t], __ldg(c + t)));
                s = __fsub_rn(__ldg(B + (int64_t)j * k + l), dd);
            }
            if (s < best) { best = s; bidx = l; }
        }
    } else {
        float vv = 0.f;
        if constexpr (VARIANT == CSPQ_VARIANT_REFERENCE) {
            for (int t = 0; t < sub; ++t) { const float v = to_f(x[t]); vv = __fadd_rn(vv, __fmul_rn(v, v)); }
        }
        for (int l = 0; l < k; ++l) {
            const float *c = C + (int64_t)l * sub;
            float s;
            if constexpr (VARIANT == CSPQ_VARIANT_REFERENCE) {
                float cc = 0.f, dd = 0.f;
                for (int t = 0; t < sub; ++t) {
                    const float v = to_f(x[t]);
                    const float cv = __ldg(c + t);
                    if (!cc_tab) cc = __fadd_rn(cc, __fmul_rn(cv, cv));
                    dd = __fadd_rn(dd, __fmul_rn(v, cv));
                }
                if (cc_tab) cc = s_cc[l];
                s = __fsub_rn(__fadd_rn(vv, cc), __fmul_rn(2.0f, dd));
            } else {
                float dd = 0.f;
                for (int t = 0; t < sub; ++t) dd = __fadd_rn(dd, __fmul_rn(to_f(x[t]), __ldg(c + t)));
                s = __fsub_rn(__ldg(B + (int64_t)j * k + l), dd);
            }
            if (s < best) { best = s; bidx = l; }
        }
    }
    if (best_out) best_out[row * crs + (int64_t)j * css] = best;
    char *o = reinterpret_cast<char *>(codes) + (row * crs + (int64_t)j * css) * code_bytes;
    if (code_bytes == 1) *reinterpret_cast<uint8_t *>(o) = static_cast<uint8_t>(bidx);
    else if (code_bytes == 2) *reinterpret_cast<uint16_t *>(o) = static_cast<uint16_t>(bidx);
    else *reinterpret_cast<int32_t *>(o) = bidx;
}

// guard[2j] = max |b|, guard[2j+1] = max ||c||_2 (rounded up)
__global__ void guard_kernel(const float *__restrict__ CB, const float *__restrict__ B, int k, int sub,
                             float *__restrict__ guard) {
    const int j = blockIdx.x;
    float bmax = 0.f, cmax = 0.f;
    for (int l = threadIdx.x; l < k; l += blockDim.x) {
        const float *c = CB + ((int64_t)j * k + l) * sub;
        double s = 0.0;
        for (int t = 0; t < sub; ++t) s = fma((double)c[t], (double)c[t], s);
        const float cn = __double2float_ru(sqrt(s) * (1.0 + 1e-12));
        const float b = B ? fabsf(B[(int64_t)j * k + l]) : 0.f;
        // NaN-propagating maxima: a non-finite table poisons the guard (=> every row flagged)
        bmax = (b != b || b > bmax) ? b : bmax;
        cmax = (cn != cn || cn > cmax) ? cn : cmax;
    }
    __shared__ float sbm[256], scm[256];
    sbm[threadIdx.x] = bmax;
    scm[threadIdx.x] = cmax;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < blockDim.x; ++i) {
            bmax = (sbm[i] != sbm[i] || sbm[i] > bmax) ? sbm[i] : bmax;
            cmax = (scm[i] != scm[i] || scm[i] > cmax) ? scm[i] : cmax;
        }
        guard[2 * j] = bmax;
        guard[2 * j + 1] = cmax;
    }
}

// precomputed_bias=False table: 0.5f * (c0*c0 (+) c1*c1 (+) ...), kernels.py:146-157
__global__ void nobias_kernel(const float *__restrict__ CB, int m, int k, int sub, float *__restrict__ Bo) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)m * k) return;
    const float *c = CB + i * sub;
    float acc = 0.f;
    for (int t = 0; t < sub; ++t) acc = __fadd_rn(acc, __fmul_rn(c[t], c[t]));
    Bo[i] = __fmul_rn(0.5f, acc);
}

template <int SUB, int R, int kT, int MINB, typename TIn, bool EXACT>
int launch_fast(const TIn *X, int64_t n, int m, int64_t xs, const float *CB, const float *B,
                const float *guard, uint8_t *codes, int64_t cs, cudaStream_t st) {
    constexpr size_t smem = 2 * (size_t)Rec<SUB>::kTotal * sizeof(float) + 2 * (size_t)R * kT * SUB * sizeof(TIn);
    auto kern = encode_k256_kernel<SUB, R, kT, MINB, TIn, EXACT>;
    static bool attr_set = false;  // benign race: idempotent attribute
    if (!attr_set) {
        CSPQ_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_set = true;
    }
    const int64_t tile = (int64_t)kT * R;
    const int64_t grid = (n + tile - 1) / tile;
    CSPQ_REQUIRE(grid <= 0x7fffffff, CSPQ_E_CONFIG, "too many rows (%lld)", (long long)n);
    kern<<<(unsigned)grid, kT, smem, st>>>(X, n, m, xs, CB, B, guard, codes, cs);
    CSPQ_LAUNCH_CHECK();
    return CSPQ_OK;
}

template <typename TIn, int VARIANT>
int launch_generic(const TIn *X, int64_t n, int m, int k, int sub, int64_t xrs, int64_t xss,
                   const float *CB, const float *B, void *codes, int code_bytes, int64_t crs,
                   int64_t css, cudaStream_t st, float *best = nullptr) {
    CSPQ_REQUIRE(m <= 65535, CSPQ_E_CONFIG, "m=%d exceeds the generic kernel's grid limit", m);
    dim3 grid((unsigned)((n + 255) / 256), (unsigned)m);
    if (sub == 4)
        encode_generic_kernel<TIn, VARIANT, 4><<<grid, 256, 0, st>>>(X, n, m, k, sub, xrs, xss, CB, B, codes, code_bytes, crs, css, best);
    else if (sub == 8)
        encode_generic_kernel<TIn, VARIANT, 8><<<grid, 256, 0, st>>>(X, n, m, k, sub, xrs, xss, CB, B, codes, code_bytes, crs, css, best);
    else if (sub == 16)
        encode_generic_kernel<TIn, VARIANT, 16><<<grid, 256, 0, st>>>(X, n, m, k, sub, xrs, xss, CB, B, codes, code_bytes, crs, css, best);
    else
        encode_generic_kernel<TIn, VARIANT, 0><<<grid, 256, 0, st>>>(X, n, m, k, sub, xrs, xss, CB, B, codes, code_bytes, crs, css, best);
    CSPQ_LAUNCH_CHECK();
    return CSPQ_OK;
}

template <typename TIn>
int dispatch(const TIn *X, int64_t n, int d, int64_t xrs, const float *CB, const float *B,
             const float *guard, int m, int k, int sub, void *codes, int64_t crs, int variant,
             int mode, cudaStream_t st) {
    const int code_bytes = k <= 256 ? 1 : 2;
    const bool reform = variant != CSPQ_VARIANT_REFERENCE;
    const size_t esz = sizeof(TIn);
    const size_t vec = (size_t)sub * esz;  // bytes per subvector copy
    const bool aligned = (vec == 32 || vec == 16 || vec == 8 || vec == 4) &&
                         (reinterpret_cast<uintptr_t>(X) % (vec >= 16 ? 16 : vec) == 0) &&
                         ((xrs * esz) % (vec >= 16 ? 16 : vec) == 0) &&
                         (reinterpret_cast<uintptr_t>(CB) % 16 == 0) &&
                         (reinterpret_cast<uintptr_t>(B) % 16 == 0);
    const bool fast = reform && k == kK && (sub == 4 || sub == 8) && aligned;
    if (fast) {
        const bool exact = mode == CSPQ_MODE_EXACT;
        uint8_t *c8 = reinterpret_cast<uint8_t *>(codes);
        const int tiling = g_tiling;
#define CSPQ_FAST(SUBV, RV, TV, MB)                                                                     \
    return exact ? launch_fast<SUBV, RV, TV, MB, TIn, true>(X, n, m, xrs, CB, B, guard, c8, crs, st)   \
                 : launch_fast<SUBV, RV, TV, MB, TIn, false>(X, n, m, xrs, CB, B, guard, c8, crs, st)
        if (sub == 8) {
            switch (tiling) {
                case 1: CSPQ_FAST(8, 8, 128, 3);
                case 2: CSPQ_FAST(8, 4, 256, 2);
                case 3: CSPQ_FAST(8, 4, 128, 4);
                default: CSPQ_FAST(8, 8, 128, 2);
            }
        } else {
            switch (tiling) {
                case 1: CSPQ_FAST(4, 8, 128, 3);
                case 2: CSPQ_FAST(4, 4, 256, 2);
                case 3: CSPQ_FAST(4, 4, 128, 4);
                default: CSPQ_FAST(4, 8, 128, 2);
            }
        }
#undef CSPQ_FAST
    }
    (void)d;
    if (reform)
        return launch_generic<TIn, CSPQ_VARIANT_REFORMULATED>(X, n, m, k, sub, xrs, sub, CB, B, codes, code_bytes, crs, 1, st);
    return launch_generic<TIn, CSPQ_VARIANT_REFERENCE>(X, n, m, k, sub, xrs, sub, CB, B, codes, code_bytes, crs, 1, st);
}

}  // namespace

int encode_set_tiling(int t) {
    CSPQ_REQUIRE(t >= 0 && t <= 3, CSPQ_E_CONFIG, "tiling must be in [0, 3], got %d", t);
    g_tiling = t;
    return CSPQ_OK;
}

int encode_stats(unsigned long long *flagged, int reset) {
    if (flagged) CSPQ_CUDA_TRY(cudaMemcpyFromSymbol(flagged, g_flagged, sizeof(unsigned long long)));
    if (reset) {
        const unsigned long long z = 0;
        CSPQ_CUDA_TRY(cudaMemcpyToSymbol(g_flagged, &z, sizeof(z)));
    }
    return CSPQ_OK;
}

int encode_prepare(const float *CB, const float *B, int m, int k, int sub, float *guard, cudaStream_t st) {
    guard_kernel<<<m, 256, 0, st>>>(CB, B, k, sub, guard);
    CSPQ_LAUNCH_CHECK();
    return CSPQ_OK;
}

int recompute_biases(const float *CB, int m, int k, int sub, float *Bo, cudaStream_t st) {
    const int64_t tot = (int64_t)m * k;
    nobias_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(CB, m, k, sub, Bo);
    CSPQ_LAUNCH_CHECK();
    return CSPQ_OK;
}

int encode_device(const void *X, int in_dtype, int64_t n, int d, int64_t xrs, const float *CB,
                  const float *B, const float *guard, int m, int k, int sub, void *codes,
                  int64_t crs, int variant, int mode, cudaStream_t st) {
    if (in_dtype == CSPQ_IN_U8)
        return dispatch<uint8_t>(reinterpret_cast<const uint8_t *>(X), n, d, xrs, CB, B, guard, m, k, sub, codes, crs, variant, mode, st);
    return dispatch<float>(reinterpret_cast<const float *>(X), n, d, xrs, CB, B, guard, m, k, sub, codes, crs, variant, mode, st);
}

int encode_with_scores(const void *X, int in_dtype, int64_t n, int64_t xrs, const float *CB, const float *B,
                       int m, int k, int sub, int32_t *codes, float *best, int variant, cudaStream_t st) {
    const bool ref = variant == CSPQ_VARIANT_REFERENCE;
    if (in_dtype == CSPQ_IN_U8) {
        const uint8_t *x = reinterpret_cast<const uint8_t *>(X);
        return ref ? launch_generic<uint8_t, CSPQ_VARIANT_REFERENCE>(x, n, m, k, sub, xrs, sub, CB, B, codes, 4, m, 1, st, best)
                   : launch_generic<uint8_t, CSPQ_VARIANT_REFORMULATED>(x, n, m, k, sub, xrs, sub, CB, B, codes, 4, m, 1, st, best);
    }
    const float *x = reinterpret_cast<const float *>(X);
    return ref ? launch_generic<float, CSPQ_VARIANT_REFERENCE>(x, n, m, k, sub, xrs, sub, CB, B, codes, 4, m, 1, st, best)
               : launch_generic<float, CSPQ_VARIANT_REFORMULATED>(x, n, m, k, sub, xrs, sub, CB, B, codes, 4, m, 1, st, best);
}

int encode_subspace_major(const float *P, int64_t n, int m, int sub, const float *CB, const float *B,
                          int k, int32_t *assign, int variant, cudaStream_t st) {
    // rows of subspace j live at P + j*n*sub, stride sub; codes (m, n) int32
    if (variant == CSPQ_VARIANT_REFERENCE)
        return launch_generic<float, CSPQ_VARIANT_REFERENCE>(P, n, m, k, sub, sub, n * (int64_t)sub, CB, B, assign, 4, 1, n, st);
    return launch_generic<float, CSPQ_VARIANT_REFORMULATED>(P, n, m, k, sub, sub, n * (int64_t)sub, CB, B, assign, 4, 1, n, st);
}

}  // namespace cspq
