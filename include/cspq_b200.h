/*
 * cspq_b200.h -- C ABI of the B200-native PQ-construction engine.
 *
 * This is the drop-in boundary for the reference package `cspq`
 * (/root/reference/pkg/src/cspq).  The reference has no FFI: its operator
 * seam is the jitted bulk driver
 *     _drive_chunk_major(X, b0, b1, CB, CT, B, w, variant, precomp, out)
 *         kernels.py:271-316, called at bulk.py:145-148
 * and the Lloyd assignment/update of training.py:57-159.  Each entry point
 * below replaces one of those and cites it.  Python binds them with ctypes
 * (paper_2605_25521_b200/_native.py); INTEGRATION.md shows the binding the
 * reference side would add.
 *
 * Conventions (all entry points):
 *   - plain pointers and sizes only; no torch types;
 *   - device pointers unless the name says _host; caller-allocated;
 *   - stream-ordered on `stream` (a cudaStream_t passed as void*, NULL =
 *     legacy default stream); no hidden device synchronisation except where
 *     documented (the _host pipeline is synchronous by contract);
 *   - return 0 on success or a negative CSPQ_E* code; cspq_last_error()
 *     returns a per-thread message for the last failure (like the
 *     reference's ConfigError / DataError messages, core.py:14-44);
 *   - re-entrant: concurrent calls on different streams are safe
 *     (bulk.py:150-155 runs drivers concurrently on disjoint row ranges).
 *
 * Layouts (the reference's, bulk.py:53-81 and core.py:88-124):
 *   X      (n, d) row-major, float32 or uint8 (uint8 is widened exactly to
 *          float32 in-kernel; the reference widens on the host, bulk.py:125);
 *          x_row_stride = elements between rows (>= d).
 *   CB     (m, k, sub) float32 row-major centroids ("rowmajor").
 *   B      (m, k) float32 biases 0.5*||c||^2 (compute_biases, core.py:232-243);
 *          the bias bits are an input contract, never recomputed here.
 *   codes  (n, m) row-major, uint8 when k <= 256 else uint16 (bulk.py:127).
 */
#ifndef CSPQ_B200_H
#define CSPQ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CSPQ_ABI_VERSION 1

/* error codes */
#define CSPQ_OK 0
#define CSPQ_E_CONFIG (-1)   /* bad shape / parameter   -> cspq ConfigError   */
#define CSPQ_E_DATA (-2)     /* bad data                -> cspq DataError     */
#define CSPQ_E_CUDA (-3)     /* CUDA runtime failure                          */
#define CSPQ_E_NOMEM (-4)    /* allocation failure                            */
#define CSPQ_E_TRAINING (-5) /* cannot train            -> cspq TrainingError */
#define CSPQ_E_FORMAT (-6)   /* malformed file          -> cspq FormatError   */

/* input element type of X */
#define CSPQ_IN_F32 0
#define CSPQ_IN_U8 1

/* encoder variants (kernels.py:36-51 EncoderVariant / _VARIANT_IDS) */
#define CSPQ_VARIANT_REFERENCE 0    /* (vv + cc) - 2 dd, kernels.py:84-105      */
#define CSPQ_VARIANT_REFORMULATED 1 /* b - dd,            kernels.py:108-122     */
#define CSPQ_VARIANT_BLOCKED 2      /* b - dd (== REFORMULATED bit for bit),
                                       kernels.py:125-245                        */

/* arithmetic modes; every mode returns the oracle's codes bit for bit */
#define CSPQ_MODE_AUTO 0    /* fastest provably-exact path for the shape      */
#define CSPQ_MODE_EXACT 1   /* strict fp32 mul-then-add chains, no FMA        */
#define CSPQ_MODE_GUARDED 2 /* FFMA scores + error-bound guard + exact fix-up */

int cspq_abi_version(void);
const char *cspq_last_error(void);

/* Guard constants of a codebook set: guard[2*j] = max_l |B[j,l]|,
 * guard[2*j+1] = max_l ||CB[j,l,:]||_2 (rounded up).  Computed once per
 * codebook set (the reference's "built once per train/load", bulk.py:55-58)
 * and passed to cspq_encode; (m, 2) float32 device buffer. */
int cspq_encode_prepare(const float *CB, const float *B, int32_t m, int32_t k, int32_t sub,
                        float *guard, void *stream);

/* Tuning knob for benchmarks: thread-block tiling of the fast encode kernel
 * (0 = 8 rows x 128 threads, 2 CTAs/SM; 1 = 8 x 128, 3 CTAs/SM;
 * 2 = 4 rows x 256 threads; 3 = 4 rows x 128 threads, 4 CTAs/SM [default]).
 * Process-global; never changes the codes. */
int cspq_encode_set_tiling(int32_t tiling);

/* Telemetry of the fast encode kernels (device-global, all streams):
 * number of (row, subspace) pairs whose best score had a runner-up inside
 * the guard band and were therefore re-encoded exactly.  Synchronises the
 * device.  reset != 0 zeroes the counter after reading. */
int cspq_encode_stats(uint64_t *flagged, int32_t reset);

/* Number of kernels this library has launched in the process (host-side count, one per launch
 * site execution); reset != 0 returns the count and zeroes it.  bench.py's gpu_launches. */
uint64_t cspq_launch_count(int32_t reset);

/* Bias table of the precomputed_bias=False ablation (kernels.py:146-157):
 * B_out[j,l] = 0.5f * fl-chain(sum_t c_t*c_t) in float32, exactly as the
 * reference recomputes it per vector.  (m, k) float32 device buffer. */
int cspq_recompute_biases_f32(const float *CB, int32_t m, int32_t k, int32_t sub, float *B_out,
                              void *stream);

/* Bulk encode of device-resident rows: replaces _drive_chunk_major over all
 * blocks (kernels.py:271-316, bulk.py:139-155).  `guard` may be NULL (it is
 * then computed on the stream with stream-ordered scratch).  B is ignored
 * for CSPQ_VARIANT_REFERENCE.  codes_row_stride = elements between code rows
 * (>= m). */
int cspq_encode(const void *X, int32_t in_dtype, int64_t n, int32_t d, int64_t x_row_stride,
                const float *CB, const float *B, const float *guard, int32_t m, int32_t k,
                int32_t sub, void *codes, int64_t codes_row_stride, int32_t variant, int32_t mode,
                void *stream);

/* Exact encode that also returns each winning score -- the per-subvector
 * API encode_*_with_score (kernels.py:349-404, the ScoreBlock best_score of
 * core.py:183-201).  codes (n, m) int32, best (n, m) float32 (the oracle's
 * score: b - dd for REFORMULATED/BLOCKED, (vv + cc) - 2 dd for REFERENCE). */
int cspq_encode_with_scores(const void *X, int32_t in_dtype, int64_t n, int32_t d, int64_t x_row_stride,
                            const float *CB, const float *B, int32_t m, int32_t k, int32_t sub,
                            int32_t *codes, float *best, int32_t variant, void *stream);

/* Tensor-core encode (tcgen05.mma kind::f16 on fp16 hi/lo splits of the
 * power-of-two scaled rows and codebook, fp32 accumulation, sm_100a): the same
 * codes as cspq_encode -- the oracle's, bit for bit -- computed as a GEMM with
 * the bias folded in, an exact argmin/runner-up epilogue on the TMEM
 * accumulators and an exact fix-up of every subvector whose runner-up lies
 * within the tensor-core error band.  Needs k == 256, sub in {4, 8},
 * REFORMULATED/BLOCKED semantics and 16-byte aligned float32 rows (or uint8
 * rows).  `img` is the prepared codebook image (cspq_encode_tc_prepare,
 * cspq_encode_tc_image_bytes(m, k, sub) bytes), `guard` as for cspq_encode.
 * best (optional, (n, m) float32) receives the tensor-core score of each
 * winner (diagnostics). */
size_t cspq_encode_tc_image_bytes(int32_t m, int32_t k, int32_t sub);
/* Largest m the tensor-core kernel takes for this sub / in_dtype (0: sub unsupported); callers
 * use cspq_encode beyond it. */
int32_t cspq_encode_tc_max_subspaces(int32_t sub, int32_t in_dtype);
int cspq_encode_tc_prepare(const float *CB, const float *B, int32_t m, int32_t k, int32_t sub, void *img,
                           void *stream);
int cspq_encode_tc(const void *X, int32_t in_dtype, int64_t n, int32_t d, int64_t x_row_stride,
                   const float *CB, const float *B, const float *guard, const void *img, int32_t m,
                   int32_t k, int32_t sub, void *codes, int64_t codes_row_stride, float *best,
                   void *stream);

/* Same as cspq_encode for a subspace-major batch (m, n, sub) -- the layout
 * of Lloyd's training sample -- writing codes as (m, n) int32.  This is the
 * final REFERENCE-variant assignment pass of lloyd_iterate
 * (training.py:143-150). */
int cspq_encode_subspace_major(const float *P, int64_t n, int32_t m, int32_t sub, const float *CB,
                               const float *B, int32_t k, int32_t *assign, int32_t variant,
                               void *stream);

/* End-to-end encode from HOST memory: pinned or pageable X (n, d) -> host
 * codes (n, m), pipelined in batches of `batch_rows` over `n_streams` CUDA
 * streams (H2D copy, encode, D2H copy overlapped; pageable buffers are
 * staged through a pinned ring).  CB/B/guard are device pointers on
 * `device`.  Synchronous: returns when codes are in host memory.
 * batch_ms (optional, ceil(n / batch_rows) doubles) receives each batch's
 * host-observed latency from its H2D enqueue to its codes landing in host
 * memory (BASELINE config 5's per-batch p50/p99).  tc_img (optional): the
 * prepared tensor-core codebook image; when given, each batch is encoded by
 * cspq_encode_tc instead of the FFMA kernel (same codes). */
int cspq_encode_host(const void *X_host, int32_t in_dtype, int64_t n, int32_t d, const float *CB,
                     const float *B, const float *guard, const void *tc_img, int32_t m, int32_t k,
                     int32_t sub, void *codes_host, int32_t variant, int32_t mode, int64_t batch_rows,
                     int32_t n_streams, double *batch_ms, int32_t device);

/* ---------------- Lloyd k-means (training.py:57-159), all M subspaces at once.
 * P      (m, n, sub) training points, float32 (p_f64 = 0; widened exactly to
 *        float64 in registers, as pts64 = float64(pts32) in the reference)
 *        or float64 (p_f64 = 1; lloyd_iterate's public float64 input);
 * C64    (m, k, sub) float64 centroids, in/out;
 * state  (m) int32: 1 = still iterating, 0 = stopped (the per-subspace
 *        early stop of training.py:137-141 -- each subspace runs exactly the
 *        iterations the reference's sequential loop would);
 * workspace: cspq_lloyd_workspace_bytes() bytes of device memory,
 *        zero-initialised once by the caller. */
size_t cspq_lloyd_workspace_bytes(int64_t n, int32_t m, int32_t sub, int32_t k);

/* Assignment step (training.py:57-73, _assign) for rows [row_begin, row_end)
 * of every active subspace: assign (m, n) int32 = argmin_l ||c_l||^2 -
 * 2 x.c_l in float64 (first index on ties), sq (m, n) float64 =
 * max(d_min + ||x||^2, 0).  Row ranges let a multi-GPU run shard the
 * assignment; rows outside the range are left untouched. */
int cspq_lloyd_assign(const void *P, int32_t p_f64, int64_t n, int32_t m, int32_t sub, int32_t k,
                      const double *C64, const int32_t *state, int64_t row_begin, int64_t row_end,
                      int32_t *assign, double *sq, void *workspace, void *stream);

/* Statistics of rows [row_begin, row_end) (training.py:73, 121-124):
 * counts (m, k) float64 (np.bincount), sums (m, k, sub) float64 accumulated
 * in ascending point order exactly like np.add.at (a stable counting sort by
 * cluster, then one sequential chain per (cluster, coordinate)), and
 * obj (m) float64 = numpy's pairwise sum of sq over the range.  With the
 * full range these are the reference's bits (given identical assignments);
 * sub-ranges give per-rank partials of a row-sharded run. */
int cspq_lloyd_accumulate(const void *P, int32_t p_f64, int64_t n, int32_t m, int32_t sub, int32_t k,
                          const int32_t *state, const int32_t *assign, const double *sq,
                          int64_t row_begin, int64_t row_end, double *counts, double *sums,
                          double *obj, void *workspace, void *stream);

/* Mean update for non-empty clusters (training.py:125-126) and the list of
 * empty clusters: empties (m, k) int32 gets the ascending empty ids,
 * n_empty (m) int32 their number. */
int cspq_lloyd_update(const double *counts, const double *sums, int32_t m, int32_t k,
                      int32_t sub, const int32_t *state, double *C64, int32_t *empties,
                      int32_t *n_empty, void *stream);

/* Empty-cluster teleport (training.py:129-136): residual ||x - c_assign||^2
 * against the updated centroids, then each empty cluster in ascending order
 * takes the current argmax-residual point (ties -> smallest point index)
 * and that residual is set to -1. */
int cspq_lloyd_repair(const void *P, int32_t p_f64, int64_t n, int32_t m, int32_t sub, int32_t k,
                      const int32_t *assign, const int32_t *state, const int32_t *empties,
                      const int32_t *n_empty, double *C64, void *workspace, void *stream);

/* Stop rule (training.py:137-141): record obj into
 * objectives[j, iterations[j]], increment iterations[j], and stop subspace
 * j if obj == 0 or prev - obj <= tol * max(prev, 1e-300) (or max_iters is
 * reached).  prev (m) float64 starts at +inf; objectives is
 * (m, max_iters + 1). */
int cspq_lloyd_stop(const double *obj, int32_t m, int32_t max_iters, double tol, int32_t *state,
                    double *prev, int32_t *iterations, double *objectives, void *stream);

/* Whole single-device Lloyd run: max_iters x (assign, accumulate, update,
 * repair, stop), then the float32 cast, the REFERENCE-variant final
 * assignment of float32(points) and the final objective
 * (training.py:143-154).  Outputs: C32 (m, k, sub) float32, assign (m, n)
 * int32 (final pass), objectives (m, max_iters + 1) float64 with
 * iterations[j] + 1 valid entries, iterations (m) int32. */
int cspq_lloyd_train(const void *P, int32_t p_f64, int64_t n, int32_t m, int32_t sub, int32_t k,
                     double *C64, int32_t max_iters, double tol, float *C32, int32_t *assign,
                     double *objectives, int32_t *iterations, void *workspace, void *stream);

/* Final objective of training.py:151-154: obj (m) = pairwise sum over
 * points of ||x - float64(C32[assign])||^2. */
int cspq_lloyd_final_objective(const void *P, int32_t p_f64, int64_t n, int32_t m, int32_t sub,
                               int32_t k, const float *C32, const int32_t *assign, double *obj,
                               void *workspace, void *stream);

/* k-means++ seeding (training.py:76-92) for every subspace: C64[j, 0] =
 * P[j, first[j]], then for c = 1..k-1 the reference's
 * rng.choice(n, p = d2 / d2.sum()) -- cdf = cumsum(p) (sequential),
 * cdf /= cdf[-1], searchsorted(cdf, u[j, c-1], 'right') -- and
 * d2 = minimum(d2, ||x - c||^2).  first (m) int64 and u (m, k-1) float64
 * are the host generator's draws (rng.integers(n), then one rng.random()
 * per choice).  status (m) int32 = -c if step c met zero total mass (the
 * reference draws rng.integers(n) for steps c..k-1 instead; the caller
 * replays those draws), 3 if the total was NaN, else 0. */
int cspq_kmeanspp(const void *P, int32_t p_f64, int64_t n, int32_t m, int32_t sub, int32_t k,
                  const int64_t *first, const double *u, double *C64, int32_t *status,
                  void *workspace, void *stream);

/* ---------------------------------------------------------------------------
 * Data formats either side of the path (io.py).  CRC-32 is zlib's, the
 * trailer of the PQCB / PQCD containers (io.py:140-151, 213-219).
 * ------------------------------------------------------------------------- */

/* Scratch bytes cspq_crc32_device needs for n input bytes. */
size_t cspq_crc32_workspace_bytes(int64_t n);

/* *crc_out (device uint32) = zlib.crc32(data[0:n], crc_in) for n device
 * bytes: per-thread pieces merged in GF(2) (crc(A|B) = x^(8|B|) crc(A) ^
 * crc(B)).  Replaces the host zlib.crc32 pass of write_codes (io.py:213-219)
 * for codes that live on the GPU. */
int cspq_crc32_device(const void *data, int64_t n, uint32_t crc_in, uint32_t *crc_out,
                      void *workspace, void *stream);

/* Host helper: the CRC of A || B from crc(A), crc(B) and |B| (zlib's
 * crc32_combine). */
uint32_t cspq_crc32_combine(uint32_t crc_a, uint32_t crc_b, int64_t len_b);

/* texmex records (fvecs: value_bytes 4, bvecs: 1; io.py:35-62, 100-104) ->
 * dense (n, d) rows, validating on the device: bad[0] (uint64, init
 * ~0) = min file offset of a record header != d, bad[1] = min file offset
 * of a non-finite value (check_finite, io.py:70-77); offset0 = file offset
 * of the first record. */
int cspq_unpack_vecs(const void *records, int64_t n, int32_t d, int32_t value_bytes,
                     int32_t check_finite, int64_t offset0, void *rows, uint64_t *bad,
                     void *stream);

/* Streaming file encoder: fvecs (in_format 0) or bvecs (1) file -> PQCD
 * codes file (io.py:213-219), i.e. read_fvecs/read_bvecs + encode_dataset +
 * write_codes (bulk.py:108-157) without materialising the dataset: batches
 * of batch_rows records are pread into pinned buffers, copied raw to the
 * GPU, unpacked and validated there, encoded (tc_img != NULL: tcgen05 path),
 * checksummed on the GPU and written with pwrite, n_streams batches in
 * flight.  bvecs rows are encoded as uint8 (no float32 widening copy).
 * On a format problem returns CSPQ_E_FORMAT, removes out_path and sets
 * err[0] = kind (1 empty dataset, 2 truncated record header, 3 non-positive
 * record length, 4 inconsistent record length, 5 truncated record body,
 * 6 non-finite value), err[1] = byte offset, err[2] = the offending record
 * length (kinds 3, 4) -- the reference reader's checks and precedence
 * (io.py:35-77).  *n_rows = records encoded.  Synchronous. */
int cspq_encode_vecs_file(const char *in_path, int32_t in_format, const char *out_path,
                          const float *CB, const float *B, const float *guard, const void *tc_img,
                          int32_t m, int32_t k, int32_t sub, int32_t variant, int32_t mode,
                          int64_t batch_rows, int32_t n_streams, int32_t device, int64_t *n_rows,
                          int64_t *err);

/* ---------------------------------------------------------------------------
 * Flat ADC search and its exact ground truth (evaluation.py), query time.
 * ------------------------------------------------------------------------- */

/* tables (nq, m, k) float32: tables[q, j, l] = ||c_jl - q_j||^2 summed like
 * numpy's einsum("kt,kt->k") (evaluation.py:66-88; bit-identical for
 * sub <= 12).  Q (nq, d) row-major float32. */
int cspq_adc_tables(const float *Q, int64_t nq, int32_t d, const float *CB, int32_t m, int32_t k,
                    int32_t sub, float *tables, void *stream);

/* scores (nq, n) float32: table sums over the m chunks in chunk order from
 * 0.0 (adc_scores, evaluation.py:91-96); codes (n, m) uint8 (k <= 256) or
 * uint16. */
int cspq_adc_scores(const float *tables, int64_t nq, const void *codes, int64_t n, int32_t m,
                    int32_t k, float *scores, void *stream);

/* Per row q of values (nq, n) (float32: value_bytes 4, float64: 8): the
 * topn smallest (value, index) pairs in lexsort order -- ties toward the
 * smaller index, NaN last (evaluation.py:99-103, 124-128).  indices (nq,
 * topn) int64, top_values (nq, topn).  1 <= topn <= min(n, 1024). */
int cspq_topn(const void *values, int32_t value_bytes, int64_t nq, int64_t n, int32_t topn,
              int64_t *indices, void *top_values, void *stream);

/* Ground-truth distances (exact_topn, evaluation.py:114-129): norms (n)
 * float64 = ||x||^2, dist (nq, n) float64 = norms - 2 q.x, float32 inputs
 * widened, float64 fused products in ascending t. */
int cspq_exact_distances(const float *queries, int64_t nq, const float *db, int64_t n, int32_t d,
                         double *norms, double *dist, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* CSPQ_B200_H */
