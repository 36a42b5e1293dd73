/*
 * oracle/pq_oracle.c -- CPU ORACLE for the PQ-construction hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links, loads or
 * calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it, and only as the checker (or as
 * the timed CPU baseline).  The product path is the CUDA library under
 * paper_2605_25521_b200/csrc and fails loudly when that is missing.
 *
 * What it restates (reference = /root/reference/pkg/src/cspq, read-only):
 *
 *   encode, REFORMULATED / BLOCKED variants   kernels.py:108-122 (_reform_one),
 *       kernels.py:125-168 (_blocked_one), kernels.py:171-245 (_blocked_quad),
 *       driven by kernels.py:271-316 (_drive_chunk_major) from bulk.py:108-157.
 *       score s_l = fl(b_l - dd_l), dd_l = fl(..fl(fl(0 + x0*c0) + x1*c1)..)
 *       summed in ascending t, strict IEEE fp32, NO fused multiply-add
 *       (kernels.py:4-9: the numba kernels are built without fastmath; the
 *       survey checked the generated asm: 0 FMA).  argmin with strict '<'
 *       from +inf, index 0 initially => first index on ties, NaN never wins.
 *       Blocked == reformulated bit-for-bit for every lane width w
 *       (pkg/tests/test_kernels.py:99-119), so one routine serves both.
 *   encode, REFERENCE variant                 kernels.py:84-105 (_ref_one):
 *       vv, cc, dd accumulated together, dist = (vv + cc) - 2*dd.
 *   encode, precomputed_bias=False ablation   kernels.py:146-157 / 213-217:
 *       s = 0.5f*bacc - acc with bacc = fl-chain of c*c.
 *   Lloyd k-means                              training.py:57-73 (_assign),
 *       training.py:109-159 (lloyd_iterate): float64 assignment by
 *       argmin_l ||c_l||^2 - 2 x.c_l (BLAS dgemm in the reference: the dot
 *       is restated as an ascending fused chain, the order of a dgemm
 *       micro-kernel's rank-1 updates), objective = pairwise sum of
 *       max(d_min + ||x||^2, 0) (numpy's pairwise summation), point-ordered
 *       float64 sums (np.add.at is an in-order loop), mean update, empty-cluster
 *       teleport to the farthest residual (ties -> smallest point index),
 *       tol stop rule, float32 cast, final REFERENCE-variant assignment pass
 *       and final objective.
 *
 * Parity pin: tests/test_oracle_golden.py checks every routine here against
 * golden vectors produced by importing the reference itself
 * (tests/golden/make_golden.py).  Encode is bit-exact; the float64 squared
 * norms follow np.einsum's own order (oracle_einsum_dot), so Lloyd differs
 * from the reference only where OpenBLAS's dgemm order would differ from the
 * ascending fused chain (none observed).
 *
 * Build: oracle/Makefile (gcc -O3 -fopenmp -ffp-contract=off; the clones are
 * vectorised across centroids only, which never reorders a centroid's own
 * accumulation chain -- the paper's centroid-parallel SIMD idea).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

#if defined(__GNUC__) && !defined(__clang__)
#pragma GCC optimize("fp-contract=off")
#define ORACLE_CLONES __attribute__((target_clones("avx512f", "avx2", "default")))
#else
#define ORACLE_CLONES
#endif

enum { OR_VARIANT_REFERENCE = 0, OR_VARIANT_REFORM = 1, OR_VARIANT_NOBIAS = 2 };

int oracle_version(void) { return 1; }

static inline float load_x(const void *X, int in_u8, int64_t off) {
    return in_u8 ? (float)((const uint8_t *)X)[off] : ((const float *)X)[off];
}

/* One (row, subspace) through the REFERENCE formula (kernels.py:84-105). */
static int32_t ref_one(const float *x, const float *C, int k, int sub, float *best_out) {
    float best = INFINITY;
    int32_t bidx = 0;
    for (int l = 0; l < k; ++l) {
        float vv = 0.0f, cc = 0.0f, dd = 0.0f;
        const float *c = C + (int64_t)l * sub;
        for (int t = 0; t < sub; ++t) {
            float v = x[t], cv = c[t];
            float p;
            p = v * v;  vv = vv + p;
            p = cv * cv; cc = cc + p;
            p = v * cv; dd = dd + p;
        }
        float dist = (vv + cc) - 2.0f * dd;
        if (dist < best) { best = dist; bidx = l; }
    }
    if (best_out) *best_out = best;
    return bidx;
}

/*
 * Reformulated / blocked scores for a block of rows against one codebook,
 * vectorised across centroids with the dimension-major copy CT (sub, k)
 * (core.py:218-229): acc[l] += x_t * CT[t][l] for t ascending -- each lane's
 * chain is exactly the scalar chain of kernels.py:117-119.
 */
ORACLE_CLONES
static void reform_rows(const float *xs, int64_t nrows, int64_t xstride, const float *CT,
                        const float *b, int k, int sub, int nobias, float *acc, float *bacc,
                        int32_t *codes_out, float *best_out) {
    if (nobias) {
        for (int l = 0; l < k; ++l) bacc[l] = 0.0f;
        for (int t = 0; t < sub; ++t) {
            const float *ct = CT + (int64_t)t * k;
            for (int l = 0; l < k; ++l) { float p = ct[l] * ct[l]; bacc[l] = bacc[l] + p; }
        }
        for (int l = 0; l < k; ++l) bacc[l] = 0.5f * bacc[l];
    }
    for (int64_t r = 0; r < nrows; ++r) {
        const float *x = xs + r * xstride;
        for (int l = 0; l < k; ++l) acc[l] = 0.0f;
        for (int t = 0; t < sub; ++t) {
            const float xt = x[t];
            const float *ct = CT + (int64_t)t * k;
            for (int l = 0; l < k; ++l) { float p = xt * ct[l]; acc[l] = acc[l] + p; }
        }
        const float *bb = nobias ? bacc : b;
        float best = INFINITY;
        int32_t bidx = 0;
        for (int l = 0; l < k; ++l) {
            float s = bb[l] - acc[l];
            if (s < best) { best = s; bidx = l; }
        }
        codes_out[r] = bidx;
        if (best_out) best_out[r] = best;
    }
}

/*
 * oracle_encode: codes (n, m) for X (n, d) row-major (f32 or u8 widened to
 * f32 exactly, bulk.py:122-125).  CB (m, k, sub) row-major centroids, B (m, k)
 * biases (the bias bits are an input, as in the reference).  variant: 0
 * REFERENCE, 1 REFORMULATED/BLOCKED, 2 blocked with precomputed_bias=False.
 * code_bytes 1 -> uint8, 2 -> uint16 (bulk.py:127).  best (n, m) optional:
 * the winning score/distance, for the bitwise score tests.
 */
int oracle_encode(const void *X, int in_u8, int64_t n, int d, const float *CB, const float *B,
                  int m, int k, int sub, int variant, void *codes, int code_bytes, float *best,
                  int nthreads) {
    if (n < 0 || m <= 0 || k <= 0 || sub <= 0 || d != m * sub) return -1;
    if (code_bytes != 1 && code_bytes != 2 && code_bytes != 4) return -2;
    if (n == 0) return 0;
    if (nthreads > 0) omp_set_num_threads(nthreads);
    const int64_t ROWS = 256;
    const int64_t nblk = (n + ROWS - 1) / ROWS;
    int err = 0;
#pragma omp parallel
    {
        float *CT = (float *)malloc(sizeof(float) * (size_t)k * sub);
        float *acc = (float *)malloc(sizeof(float) * (size_t)k);
        float *bacc = (float *)malloc(sizeof(float) * (size_t)k);
        float *xs = (float *)malloc(sizeof(float) * (size_t)ROWS * sub);
        int32_t *cc = (int32_t *)malloc(sizeof(int32_t) * (size_t)ROWS);
        float *bb = (float *)malloc(sizeof(float) * (size_t)ROWS);
        const int ok = CT && acc && bacc && xs && cc && bb;
        if (!ok) {
#pragma omp atomic write
            err = -3;
        }
        {
            /* chunk-major inside a block of rows: subspace outer, rows inner */
#pragma omp for schedule(dynamic, 4)
            for (int64_t blk = 0; blk < nblk; ++blk) {
                if (!ok) continue;
                const int64_t r0 = blk * ROWS;
                const int64_t nr = (r0 + ROWS <= n) ? ROWS : n - r0;
                for (int j = 0; j < m; ++j) {
                    const float *C = CB + (int64_t)j * k * sub;
                    for (int64_t r = 0; r < nr; ++r)
                        for (int t = 0; t < sub; ++t)
                            xs[r * sub + t] = load_x(X, in_u8, (r0 + r) * d + (int64_t)j * sub + t);
                    if (variant == OR_VARIANT_REFERENCE) {
                        for (int64_t r = 0; r < nr; ++r)
                            cc[r] = ref_one(xs + r * sub, C, k, sub, &bb[r]);
                    } else {
                        for (int l = 0; l < k; ++l)
                            for (int t = 0; t < sub; ++t) CT[(int64_t)t * k + l] = C[(int64_t)l * sub + t];
                        reform_rows(xs, nr, sub, CT, B + (int64_t)j * k, k, sub,
                                    variant == OR_VARIANT_NOBIAS, acc, bacc, cc, bb);
                    }
                    for (int64_t r = 0; r < nr; ++r) {
                        const int64_t o = (r0 + r) * m + j;
                        if (code_bytes == 1) ((uint8_t *)codes)[o] = (uint8_t)cc[r];
                        else if (code_bytes == 2) ((uint16_t *)codes)[o] = (uint16_t)cc[r];
                        else ((int32_t *)codes)[o] = cc[r];
                        if (best) best[o] = bb[r];
                    }
                }
            }
        }
        free(CT); free(acc); free(bacc); free(xs); free(cc); free(bb);
    }
    return err;
}

/* ------------------------------------------------------------------------ */
/* float64 helpers for Lloyd                                                */
/* ------------------------------------------------------------------------ */

/* np.einsum("it,it->i") / ("kt,kt->k") on contiguous float64 rows of length n
 * (training.py:61/70/88/134/154, core.py via the same routine): numpy's
 * sum_of_products_contig_contig_outstride0_two with 2-lane (SSE2 baseline)
 * vectors.  Each 8-element block is folded into the two lane accumulators
 * back to front (acc = p[t+L] + (p[t+2+L] + (p[t+4+L] + (p[t+6+L] + acc))),
 * npyv_muladd without FMA = product rounded, then added), the tail adds one
 * lane pair at a time, and the result is lane0 + lane1.  Checked bit-exact
 * against np.einsum for n = 1..24 (tests/test_oracle_golden.py). */
double oracle_einsum_dot(const double *a, const double *b, int n) {
    double l0 = 0.0, l1 = 0.0;
    int t = 0;
    for (; n - t >= 8; t += 8) {
        l0 = a[t + 6] * b[t + 6] + l0; l1 = a[t + 7] * b[t + 7] + l1;
        l0 = a[t + 4] * b[t + 4] + l0; l1 = a[t + 5] * b[t + 5] + l1;
        l0 = a[t + 2] * b[t + 2] + l0; l1 = a[t + 3] * b[t + 3] + l1;
        l0 = a[t] * b[t] + l0;         l1 = a[t + 1] * b[t + 1] + l1;
    }
    for (; t < n; t += 2) {
        l0 = a[t] * b[t] + l0;
        if (t + 1 < n) l1 = a[t + 1] * b[t + 1] + l1;
    }
    return l0 + l1;
}

/* numpy's pairwise summation for a contiguous float64 array (what
 * ndarray.sum() does for training.py:73/154): <8 sequential, <=128 eight
 * accumulators, else split at n/2 rounded down to a multiple of 8. */
double oracle_pairwise_sum(const double *a, int64_t n) {
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; ++i) r += a[i];
        return r;
    } else if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return oracle_pairwise_sum(a, n2) + oracle_pairwise_sum(a + n2, n - n2);
}

/* training.py:57-73: argmin_l (||c_l||^2 - 2 x.c_l), first index on ties,
 * sq_i = max(d_min + ||x||^2, 0).  Returns the pairwise-summed objective.
 * The dot products run across centroids in lanes (dimension-major copy CT),
 * each lane an ascending fused chain. */
#if defined(__GNUC__) && !defined(__clang__)
__attribute__((target_clones("arch=skylake-avx512", "arch=haswell", "default")))
#endif
static void lloyd_assign_rows(const double *P, int64_t i0, int64_t i1, int sub, const double *CT,
                              const double *cn, int k, int64_t *assign, double *sq, double *dot) {
    for (int64_t i = i0; i < i1; ++i) {
        const double *x = P + i * sub;
        for (int l = 0; l < k; ++l) dot[l] = 0.0;
        for (int t = 0; t < sub; ++t) {
            const double xt = x[t];
            const double *ct = CT + (int64_t)t * k;
            for (int l = 0; l < k; ++l) dot[l] = fma(xt, ct[l], dot[l]);
        }
        double best = cn[0] - 2.0 * dot[0];
        int64_t bi = 0;
        for (int l = 1; l < k; ++l) {
            double dl = cn[l] - 2.0 * dot[l];
            if (dl < best) { best = dl; bi = l; }
        }
        double v = best + oracle_einsum_dot(x, x, sub);
        assign[i] = bi;
        sq[i] = v > 0.0 ? v : 0.0;
    }
}

static double lloyd_assign(const double *P, int64_t n, int sub, const double *C, int k,
                           int64_t *assign, double *sq, double *cn) {
    double *CT = (double *)malloc(sizeof(double) * (size_t)k * sub);
    for (int l = 0; l < k; ++l) {
        for (int t = 0; t < sub; ++t) CT[(int64_t)t * k + l] = C[(int64_t)l * sub + t];
        cn[l] = oracle_einsum_dot(C + (int64_t)l * sub, C + (int64_t)l * sub, sub);
    }
    const int64_t ROWS = 1024;
#pragma omp parallel
    {
        double *dot = (double *)malloc(sizeof(double) * (size_t)k);
#pragma omp for schedule(static)
        for (int64_t i0 = 0; i0 < n; i0 += ROWS)
            lloyd_assign_rows(P, i0, i0 + ROWS < n ? i0 + ROWS : n, sub, CT, cn, k, assign, sq, dot);
        free(dot);
    }
    free(CT);
    return oracle_pairwise_sum(sq, n);
}

/*
 * oracle_lloyd: training.py:109-159 for one subspace.
 *   P (n, sub) float64 points, C (k, sub) float64 initial centroids (updated
 *   in place to the final float64 centroids), objectives: room for
 *   max_iters + 1 values, assign_out (n) int64 final assignments, cast_out
 *   (k, sub) float32 centroids.  Returns the number of objectives written;
 *   *iters_out = iterations run.
 */
int oracle_lloyd(const double *P, int64_t n, int sub, double *C, int k, int max_iters,
                 double tol, double *objectives, int64_t *assign_out, float *cast_out,
                 int *iters_out, int nthreads) {
    if (nthreads > 0) omp_set_num_threads(nthreads);
    int64_t *assign = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    double *sq = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double *cn = (double *)malloc(sizeof(double) * (size_t)k);
    double *sums = (double *)malloc(sizeof(double) * (size_t)k * sub);
    double *counts = (double *)malloc(sizeof(double) * (size_t)k);
    double *resid = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    if (!assign || !sq || !cn || !sums || !counts || !resid) return -3;
    int nobj = 0, iters = 0;
    double prev = INFINITY;
    for (int it = 0; it < max_iters; ++it) {
        ++iters;
        double obj = lloyd_assign(P, n, sub, C, k, assign, sq, cn);
        objectives[nobj++] = obj;
        memset(sums, 0, sizeof(double) * (size_t)k * sub);
        memset(counts, 0, sizeof(double) * (size_t)k);
        for (int64_t i = 0; i < n; ++i) { /* np.add.at: in point order */
            counts[assign[i]] += 1.0;
            for (int t = 0; t < sub; ++t) sums[assign[i] * sub + t] += P[i * sub + t];
        }
        int nempty = 0;
        for (int l = 0; l < k; ++l) {
            if (counts[l] > 0) {
                for (int t = 0; t < sub; ++t) C[(int64_t)l * sub + t] = sums[(int64_t)l * sub + t] / counts[l];
            } else {
                ++nempty;
            }
        }
        if (nempty) { /* training.py:129-136 */
            double *df = (double *)malloc(sizeof(double) * (size_t)sub);
            for (int64_t i = 0; i < n; ++i) {
                for (int t = 0; t < sub; ++t) df[t] = P[i * sub + t] - C[assign[i] * sub + t];
                resid[i] = oracle_einsum_dot(df, df, sub);
            }
            free(df);
            for (int l = 0; l < k; ++l) {
                if (counts[l] > 0) continue;
                int64_t cand = 0;
                for (int64_t i = 1; i < n; ++i) if (resid[i] > resid[cand]) cand = i;
                for (int t = 0; t < sub; ++t) C[(int64_t)l * sub + t] = P[cand * sub + t];
                resid[cand] = -1.0;
            }
        }
        if (obj == 0.0) break;
        if (prev < INFINITY && (prev - obj) <= tol * (prev > 1e-300 ? prev : 1e-300)) break;
        prev = obj;
    }
    /* cast, then the float32 REFERENCE-variant final pass (training.py:143-152) */
    for (int64_t q = 0; q < (int64_t)k * sub; ++q) cast_out[q] = (float)C[q];
    float *p32 = (float *)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1) * sub);
    for (int64_t q = 0; q < n * sub; ++q) p32[q] = (float)P[q];
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) assign_out[i] = ref_one(p32 + i * sub, cast_out, k, sub, NULL);
    double *df = (double *)malloc(sizeof(double) * (size_t)sub);
    for (int64_t i = 0; i < n; ++i) {
        for (int t = 0; t < sub; ++t) df[t] = P[i * sub + t] - (double)cast_out[assign_out[i] * sub + t];
        sq[i] = oracle_einsum_dot(df, df, sub);
    }
    free(df);
    objectives[nobj++] = oracle_pairwise_sum(sq, n);
    *iters_out = iters;
    free(p32); free(assign); free(sq); free(cn); free(sums); free(counts); free(resid);
    return nobj;
}
