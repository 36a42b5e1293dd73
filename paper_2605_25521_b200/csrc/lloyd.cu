// lloyd.cu -- Lloyd k-means for all M subspaces at once, float64, sm_100a.
//
// Restates the reference's lloyd_iterate (/root/reference/pkg/src/cspq/
// training.py:109-159) with its _assign (training.py:57-73), batched over
// subspaces instead of the reference's sequential subspace loop
// (training.py:212-223).  Arithmetic follows the oracle (oracle/pq_oracle.c)
// operation for operation so GPU and oracle agree bit for bit:
//   * assignment: ||c||^2 in np.einsum's order (einsum_sum), x.c as an
//     ascending fused chain (a dgemm micro-kernel's rank-1 order),
//     d = ||c||^2 - 2 x.c, argmin first index (np.argmin);
//   * objective terms sq = np.maximum(d_min + ||x||^2, 0) and their sum in
//     numpy's pairwise-summation tree (ndarray.sum);
//   * counts (np.bincount) and sums accumulated in ascending point order,
//     which is what np.add.at does: a stable counting sort by cluster
//     (per-chunk histograms -> scan -> warp-stable scatter with
//     __match_any_sync) followed by one sequential float64 chain per
//     (cluster, coordinate).  No floating-point atomics anywhere, so the
//     result is deterministic and equal to the reference's for identical
//     assignments;
//   * mean for non-empty clusters with IEEE division; empty clusters
//     teleported (ascending) onto the argmax residual point (ties ->
//     smallest index), that residual then set to -1;
//   * stop rule obj == 0 or prev - obj <= tol * max(prev, 1e-300), kept per
//     subspace (state[j]) so every subspace runs exactly the iterations the
//     reference's sequential loop would.

#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"

namespace cspq {

namespace {

#ifndef CSPQ_SUMS_KB
#define CSPQ_SUMS_KB 32  // sums_kernel gathers in flight per thread (16: c4 training +8 %)
#endif
constexpr int kChunk = 1024;  // points per histogram/scatter chunk
constexpr uint64_t kMagic = 0x43535051424C4C59ull;

inline int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }


struct WsLayout {
    int64_t header, leaves, nodes, ntmp, nodeval, hist, cnt, start, perm, sq, resid, leafsum, cn;
    // train-loop state
    int64_t counts, sums, obj, prev, state, empties, nempty, assign_it;
    // float32 copy of float64 points (final pass), k-means++ scratch
    int64_t p32, d2, pp;
    // tensor-core screened assignment: float32 codebooks, biases, guard, tcgen05 image, codes, flags
    int64_t tc_cb, tc_b, tc_guard, tc_img, tc_codes, tc_flags, tc_rmax;
    int64_t redo;  // clusters whose sums need the sequential chain (sums_exact_kernel)
    int64_t total;
    int64_t nch, maxleaves;
    WsLayout(int64_t n, int m, int sub, int k) {
        nch = (n + kChunk - 1) / kChunk;
        maxleaves = n / 32 + 8;
        int64_t o = 0;
        auto take = [&](int64_t bytes) { int64_t r = o; o = align_up(o + bytes, 256); return r; };
        header = take(256);
        leaves = take(16 * maxleaves);
        nodes = take(8 * maxleaves + 4 * 80);   // internal nodes (left, right) by height + level offsets
        ntmp = take(12 * maxleaves);            // construction scratch (left, right, height)
        nodeval = take(8 * (int64_t)m * maxleaves);
        hist = take(4 * (int64_t)m * nch * k);
        cnt = take(4 * (int64_t)m * k);
        start = take(4 * (int64_t)m * k);
        perm = take(4 * (int64_t)m * n);
        sq = take(8 * (int64_t)m * n);
        resid = take(8 * (int64_t)m * n);
        leafsum = take(8 * (int64_t)m * maxleaves);
        cn = take(8 * (int64_t)m * k);
        counts = take(8 * (int64_t)m * k);
        sums = take(8 * (int64_t)m * k * sub);
        obj = take(8 * (int64_t)m);
        prev = take(8 * (int64_t)m);
        state = take(4 * (int64_t)m);
        empties = take(4 * (int64_t)m * k);
        nempty = take(4 * (int64_t)m);
        assign_it = take(4 * (int64_t)m * n);
        p32 = take(4 * (int64_t)m * n * sub);
        d2 = take(8 * (int64_t)m * n);
        pp = take(8 * (int64_t)m * n);
        tc_cb = take(4 * (int64_t)m * k * sub);
        tc_b = take(4 * (int64_t)m * k);
        tc_guard = take(8 * (int64_t)m);
        tc_img = take((int64_t)m * k * 32 * 4);  // >= encode_tc_image_bytes (K = 32 fp16 per centroid row + the m scales)
        tc_codes = take((int64_t)m * n);
        tc_flags = take((int64_t)m * n);
        tc_rmax = take(4 * (int64_t)m);
        redo = take((int64_t)m * k);
        total = o;
    }
    template <typename T>
    T *at(void *ws, int64_t off) const { return reinterpret_cast<T *>(reinterpret_cast<char *>(ws) + off); }
};

struct WsHeader {
    uint64_t magic;
    int64_t leaves_for;  // range length the leaf table describes
    int64_t nleaves;
    int64_t nlevels;     // heights 1 .. nlevels of the internal nodes
};


// ---------------------------------------------------------------- pairwise tree
// Leaves of numpy's pairwise summation of a length-n range, in order
// (pairwise_sum: n <= 128 is a leaf; otherwise split at n2 = n/2 - (n/2)%8).
// Also the internal nodes of that recursion (node = left + right, exactly numpy's order),
// grouped by height so that a CTA can evaluate them level by level.  Node ids: leaves are
// 0 .. nl-1 (in order), internal nodes nl .. in construction order.  Built once per n.
// (host code: the tree depends on n only, so it is built once per (device, n) on the host and
// kept in device memory -- a single GPU thread took 6 ms for n = 1M)
void build_tree(int64_t n, int64_t *leaves, int32_t *nodes, int32_t *ntmp, int64_t maxleaves, WsHeader *hdr) {
    // pass 1: leaves in order
    struct F { int64_t lo, len; };
    F st[96];
    int sp = 0;
    int64_t nl = 0;
    st[sp++] = {0, n};
    while (sp) {
        F f = st[--sp];
        if (f.len <= 128) { leaves[2 * nl] = f.lo; leaves[2 * nl + 1] = f.len; ++nl; continue; }
        int64_t n2 = f.len / 2;
        n2 -= n2 % 8;
        st[sp++] = {f.lo + n2, f.len - n2};  // right pushed first: left is visited first
        st[sp++] = {f.lo, n2};
    }
    // pass 2: post-order walk giving every internal node (left id, right id, height)
    struct G { int64_t len; int stage; int32_t left, lh; };
    G gs[96];
    int gp = 0;
    int32_t next_leaf = 0, next_node = (int32_t)nl, ret = 0, rh = 0, maxh = 0;
    gs[0] = {n, 0, 0, 0};
    for (;;) {
        G &g = gs[gp];
        if (g.stage == 0) {
            if (g.len <= 128) {
                ret = next_leaf++;
                rh = 0;
                if (gp == 0) break;
                --gp;
                continue;
            }
            int64_t n2 = g.len / 2;
            n2 -= n2 % 8;
            g.stage = 1;
            gs[++gp] = {n2, 0, 0, 0};
        } else if (g.stage == 1) {
            g.left = ret;
            g.lh = rh;
            g.stage = 2;
            int64_t n2 = g.len / 2;
            n2 -= n2 % 8;
            gs[++gp] = {g.len - n2, 0, 0, 0};
        } else {
            const int32_t id = next_node++, h = 1 + (g.lh > rh ? g.lh : rh);
            int32_t *t = ntmp + 3 * (int64_t)(id - nl);
            t[0] = g.left; t[1] = ret; t[2] = h;
            maxh = h > maxh ? h : maxh;
            ret = id;
            rh = h;
            if (gp == 0) break;
            --gp;
        }
    }
    // counting sort of the internal nodes by height: nodes = [(left, right)...], level
    // offsets after them (level h occupies [off[h-1], off[h]))
    const int64_t ni = next_node - nl;
    int32_t *off = nodes + 2 * maxleaves;
    for (int h = 0; h <= maxh; ++h) off[h] = 0;
    for (int64_t i = 0; i < ni; ++i) ++off[ntmp[3 * i + 2]];
    int32_t run = 0;
    for (int h = 1; h <= maxh; ++h) { const int32_t c = off[h]; off[h] = run; run += c; }
    off[0] = 0;
    // off[h] is now the start of level h; place, then turn starts into ends
    for (int64_t i = 0; i < ni; ++i) {
        const int32_t h = ntmp[3 * i + 2];
        const int32_t pos = off[h]++;
        nodes[2 * (int64_t)pos] = ntmp[3 * i];
        nodes[2 * (int64_t)pos + 1] = ntmp[3 * i + 1];
        ntmp[3 * i + 2] = pos;  // construction index -> sorted slot
    }
    // children that are internal nodes: construction id -> nl + sorted slot
    for (int64_t p = 0; p < 2 * ni; ++p) {
        const int32_t c = nodes[p];
        if (c >= nl) nodes[p] = (int32_t)nl + ntmp[3 * (int64_t)(c - nl) + 2];
    }
    hdr->magic = kMagic;
    hdr->leaves_for = n;
    hdr->nleaves = nl;
    hdr->nlevels = maxh;  // off[h] = end of level h; level 1 starts at 0
}

struct TreeBuf {
    int64_t *leaves;
    int32_t *nodes;
    const WsHeader *hdr;
};
// leaves (16 B x maxleaves) | nodes (8 B x maxleaves + 320 B) | header, in device memory
TreeBuf tree_for(int64_t n) {
    static std::mutex mu;
    static std::map<std::pair<int, int64_t>, TreeBuf> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find({dev, n});
    if (it != cache.end()) return it->second;
    const int64_t maxleaves = n / 32 + 8;
    const size_t lb = 16 * (size_t)maxleaves, nb = 8 * (size_t)maxleaves + 4 * 80;
    std::vector<unsigned char> h(lb + nb + sizeof(WsHeader));
    std::vector<int32_t> ntmp(3 * (size_t)maxleaves);
    build_tree(n, reinterpret_cast<int64_t *>(h.data()), reinterpret_cast<int32_t *>(h.data() + lb), ntmp.data(),
               maxleaves, reinterpret_cast<WsHeader *>(h.data() + lb + nb));
    unsigned char *d = nullptr;
    if (cudaMalloc(&d, h.size()) != cudaSuccess || cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
        if (d) cudaFree(d);
        return {nullptr, nullptr, nullptr};
    }
    TreeBuf t{reinterpret_cast<int64_t *>(d), reinterpret_cast<int32_t *>(d + lb),
              reinterpret_cast<const WsHeader *>(d + lb + nb)};
    cache[{dev, n}] = t;
    return t;
}

// numpy leaf sum: <8 sequential from 0.0; else 8 accumulators, fixed combine, tail
__device__ double leaf_sum(const double *a, int64_t n) {
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
        return r;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
}

// leafsum[j][l] for values vals[j*vstride + lo .. ]
__global__ void leafsum_kernel(const double *vals, int64_t vstride, int64_t begin, int m,
                               const int32_t *state, const int64_t *leaves, const WsHeader *hdr,
                               int64_t maxleaves, double *leafsum) {
    const int64_t nl = hdr->nleaves;
    const int j = blockIdx.y;
    if (state && !state[j]) return;
    for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < nl; l += (int64_t)gridDim.x * blockDim.x)
        leafsum[(int64_t)j * maxleaves + l] = leaf_sum(vals + (int64_t)j * vstride + begin + leaves[2 * l], leaves[2 * l + 1]);
}

// evaluate the internal nodes level by level (one CTA per subspace); node ids are
// translated to storage: id < nl -> leafsum, else nodeval[id - nl] at its sorted slot
__global__ void combine_levels_kernel(int m, const int32_t *state, const double *leafsum, int64_t maxleaves,
                                      const int32_t *nodes, int64_t tree_maxleaves, const WsHeader *hdr, double *nodeval,
                                      double *out) {
    const int j = blockIdx.x;
    if (state && !state[j]) return;
    const int64_t nl = hdr->nleaves;
    const int H = (int)hdr->nlevels;
    const double *ls = leafsum + (int64_t)j * maxleaves;
    double *nv = nodeval + (int64_t)j * maxleaves;
    if (H == 0) {
        if (threadIdx.x == 0) out[j] = ls[0];
        return;
    }
    const int32_t *off = nodes + 2 * tree_maxleaves;  // level ends (after the tree's node pairs)
    int32_t lo = 0;
    for (int h = 1; h <= H; ++h) {
        const int32_t hi = off[h];
        for (int32_t p = lo + threadIdx.x; p < hi; p += blockDim.x) {
            const int32_t a = nodes[2 * (int64_t)p], b = nodes[2 * (int64_t)p + 1];
            const double va = a < nl ? ls[a] : nv[a - nl];
            const double vb = b < nl ? ls[b] : nv[b - nl];
            nv[p] = __dadd_rn(va, vb);
        }
        lo = hi;
        __syncthreads();
    }
    if (threadIdx.x == 0) out[j] = nv[off[H] - 1];  // the root is alone on the top level
}

// ---------------------------------------------------------------- einsum order
// np.einsum("it,it->i") on contiguous float64 rows (training.py:61/70/88/134/154): numpy's
// sum_of_products_contig_contig_outstride0_two with 2-lane vectors -- every 8-element block
// folded back to front into two lane accumulators (product rounded, then added), a tail of lane
// pairs, then lane0 + lane1.  prod(t) returns the rounded product of element t.  Same order as
// oracle_einsum_dot (oracle/pq_oracle.c); with n a compile-time constant it unrolls completely.
template <typename G>
__device__ __forceinline__ double einsum_sum(G prod, int n) {
    double l0 = 0.0, l1 = 0.0;
    int t = 0;
    for (; n - t >= 8; t += 8) {
        l0 = __dadd_rn(prod(t + 6), l0); l1 = __dadd_rn(prod(t + 7), l1);
        l0 = __dadd_rn(prod(t + 4), l0); l1 = __dadd_rn(prod(t + 5), l1);
        l0 = __dadd_rn(prod(t + 2), l0); l1 = __dadd_rn(prod(t + 3), l1);
        l0 = __dadd_rn(prod(t), l0);     l1 = __dadd_rn(prod(t + 1), l1);
    }
    for (; t < n; t += 2) {
        l0 = __dadd_rn(prod(t), l0);
        if (t + 1 < n) l1 = __dadd_rn(prod(t + 1), l1);
    }
    return __dadd_rn(l0, l1);
}

// ---------------------------------------------------------------- assignment
#ifndef CSPQ_SETTLE_PPT
#define CSPQ_SETTLE_PPT 2  // points per thread per step in tc_settle_kernel
#endif
#ifndef CSPQ_LLOYD_PPT
#define CSPQ_LLOYD_PPT 4  // points per thread in assign_kernel (2x4, 4x2, 4x4, 2x8, 1x8 measured: 4x2 best)
#endif
#ifndef CSPQ_LLOYD_U
#define CSPQ_LLOYD_U 2    // centroids per step in assign_kernel
#endif
__global__ void cnorm_kernel(const double *C64, int m, int k, int sub, const int32_t *state, double *cn) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)m * k) return;
    const int j = (int)(i / k);
    if (state && !state[j]) return;
    const double *c = C64 + i * sub;
    cn[i] = einsum_sum([&](int t) { return __dmul_rn(c[t], c[t]); }, sub);  // c_norms, training.py:61
}

template <int SUBC, typename TP>
__global__ void __launch_bounds__(256)
assign_kernel(const TP *__restrict__ P, int64_t n, int k, int sub_rt, const double *__restrict__ C64,
              const double *__restrict__ cn_g, const int32_t *__restrict__ state, int64_t b, int64_t e,
              int32_t *__restrict__ assign, double *__restrict__ sq, int use_smem) {
    const int sub = SUBC > 0 ? SUBC : sub_rt;
    const int j = blockIdx.y;
    if (!state[j]) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const double *Cj = C64 + (int64_t)j * k * sub;
    const double *cnj = cn_g + (int64_t)j * k;
    if (use_smem) {
        double *sC = reinterpret_cast<double *>(smem_raw);
        double *scn = sC + (int64_t)k * sub;
        for (int q = threadIdx.x; q < k * sub; q += blockDim.x) sC[q] = Cj[q];
        for (int q = threadIdx.x; q < k; q += blockDim.x) scn[q] = cnj[q];
        __syncthreads();
        Cj = sC;
        cnj = scn;
    }
    const TP *Pj = P + (int64_t)j * n * sub;
    if constexpr (SUBC > 0) {
        // Two points per thread (each broadcast centroid load feeds both) and four centroids
        // per step (independent fma chains); every (point, centroid) value is the same
        // ascending chain as before, d = cn - 2 dot is one rounding either way (2 dot is
        // exact), and the argmin still compares centroids in index order.
        constexpr int kPPT = CSPQ_LLOYD_PPT;
        constexpr int kU = CSPQ_LLOYD_U;
        const int64_t stride = (int64_t)gridDim.x * blockDim.x * kPPT;
        for (int64_t i0 = b + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kPPT; i0 < e; i0 += stride) {
            double x[kPPT][SUBC], best[kPPT];
            int bi[kPPT];
#pragma unroll
            for (int p = 0; p < kPPT; ++p) {
                const int64_t i = i0 + p < e ? i0 + p : i0;  // a missing second point repeats the first
#pragma unroll
                for (int t = 0; t < SUBC; ++t) x[p][t] = (double)Pj[i * SUBC + t];
                best[p] = 0.0;
                bi[p] = 0;
            }
            int l = 0;
            for (; l + kU <= k; l += kU) {
                double dl[kPPT][kU];
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    const double *c = Cj + (int64_t)(l + u) * SUBC;
                    double cv[SUBC];
#pragma unroll
                    for (int t = 0; t < SUBC; ++t) cv[t] = c[t];
                    const double cn = cnj[l + u];
#pragma unroll
                    for (int p = 0; p < kPPT; ++p) {
                        double dot = 0.0;
#pragma unroll
                        for (int t = 0; t < SUBC; ++t) dot = __fma_rn(x[p][t], cv[t], dot);
                        dl[p][u] = __fma_rn(-2.0, dot, cn);
                    }
                }
#pragma unroll
                for (int p = 0; p < kPPT; ++p)
#pragma unroll
                    for (int u = 0; u < kU; ++u)
                        if ((l + u) == 0 || dl[p][u] < best[p]) { best[p] = dl[p][u]; bi[p] = l + u; }
            }
            for (; l < k; ++l) {
                const double *c = Cj + (int64_t)l * SUBC;
#pragma unroll
                for (int p = 0; p < kPPT; ++p) {
                    double dot = 0.0;
#pragma unroll
                    for (int t = 0; t < SUBC; ++t) dot = __fma_rn(x[p][t], c[t], dot);
                    const double d1 = __fma_rn(-2.0, dot, cnj[l]);
                    if (l == 0 || d1 < best[p]) { best[p] = d1; bi[p] = l; }
                }
            }
#pragma unroll
            for (int p = 0; p < kPPT; ++p) {
                const int64_t i = i0 + p;
                if (i >= e) break;
                const double xx = einsum_sum([&](int t) { return __dmul_rn(x[p][t], x[p][t]); }, SUBC);
                const double v = __dadd_rn(best[p], xx);
                assign[(int64_t)j * n + i] = bi[p];
                sq[(int64_t)j * n + i] = (v >= 0.0 || v != v) ? v : 0.0;  // np.maximum(v, 0.0)
            }
        }
        return;
    } else {
    for (int64_t i = b + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x) {
        double best = 0.0;
        int bi = 0;
        double xx = 0.0;
        {
            const TP *x = Pj + i * sub;
            for (int l = 0; l < k; ++l) {
                const double *c = Cj + (int64_t)l * sub;
                double dot = 0.0;
                for (int t = 0; t < sub; ++t) dot = __fma_rn((double)x[t], c[t], dot);
                const double dl = __dsub_rn(cnj[l], __dmul_rn(2.0, dot));
                if (l == 0 || dl < best) { best = dl; bi = l; }
            }
            xx = einsum_sum([&](int t) { return __dmul_rn((double)x[t], (double)x[t]); }, sub);
        }
        const double v = __dadd_rn(best, xx);
        assign[(int64_t)j * n + i] = bi;
        sq[(int64_t)j * n + i] = (v >= 0.0 || v != v) ? v : 0.0;  // np.maximum(v, 0.0)
    }
    }
}

// ---------------------------------------------------------------- counting sort
// ---------------------------------------------------------------- tensor-core screened assignment
// The float64 argmin of d_l = ||c_l||^2 - 2 x.c_l is the argmin of the real score
// b_l - x.c_l (b = ||c||^2 / 2).  The tcgen05 encode kernel evaluates that score from
// float32(c), float32(b) with the error band E of the encode path and flags every point whose
// runner-up lies within 4E; rounding c and b to float32 moves a score by at most 2^-24 W
// (W = |b| + ||x|| ||c||, far inside the 2x margin of the 4E threshold), so an unflagged
// point's winner is the real -- and float64 -- argmin by a margin no float64 rounding can
// close.  Flagged points (~1e-3) take the full float64 scan; every point's d and sq come from
// the same float64 chain as assign_kernel, so assignments and objective terms are identical.
__global__ void tc_codebook_kernel(const double *__restrict__ C64, const double *__restrict__ cn, int k, int sub,
                                   float *__restrict__ cb32, float *__restrict__ b32) {
    const int j = blockIdx.x;
    for (int l = threadIdx.x; l < k; l += blockDim.x) {
        const int64_t i = (int64_t)j * k + l;
        for (int t = 0; t < sub; ++t) cb32[i * sub + t] = __double2float_rn(C64[i * sub + t]);
        b32[i] = __double2float_rn(0.5 * cn[i]);
    }
}

template <int SUBC>  // k == 256
__global__ void __launch_bounds__(256)
tc_settle_kernel(const float *__restrict__ P, int64_t n, int k, const double *__restrict__ C64,
                 const double *__restrict__ cn_g, const int32_t *__restrict__ state, int64_t b, int64_t e,
                 const uint8_t *__restrict__ codes, const uint8_t *__restrict__ flags, int32_t *__restrict__ assign,
                 double *__restrict__ sq) {
    const int j = blockIdx.y;
    if (!state[j]) return;
    // the subspace's float64 codebook and norms in shared memory (k = 256: 8-16 KB + 2 KB);
    // every point gathers one centroid from it
    // (centroid stride SUBC + 1 doubles: random per-lane centroids spread over 16 bank pairs
    // instead of 2 -- a 16-way conflict with the dense layout)
    constexpr int kCS = SUBC + 1;
    __shared__ double sC[256 * kCS], scn[256];
    for (int q = threadIdx.x; q < k * SUBC; q += blockDim.x) sC[(q / SUBC) * kCS + q % SUBC] = C64[(int64_t)j * k * SUBC + q];
    for (int q = threadIdx.x; q < k; q += blockDim.x) scn[q] = cn_g[(int64_t)j * k + q];
    __syncthreads();
    const double *Cj = sC;
    const double *cnj = scn;
    auto dist = [&](const double (&x)[SUBC], int l) {
        const double *c = Cj + l * kCS;
        double dot = 0.0;
#pragma unroll
        for (int t = 0; t < SUBC; ++t) dot = __fma_rn(x[t], c[t], dot);
        return __fma_rn(-2.0, dot, cnj[l]);
    };
    // two points per thread per step (independent loads in flight); x with 16-byte loads.  The
    // loop bound is warp-uniform (a warp owns 64 consecutive points) so flagged points can be
    // scanned by the whole warp: lanes split the 256 centroids, then a shuffle reduction keeps the
    // sequential scan's winner (smallest d, first index; a NaN d never wins unless it is d_0)
    constexpr int kPP = CSPQ_SETTLE_PPT;
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * kPP;
    for (int64_t w0 = b + ((int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) * kPP; w0 < e; w0 += stride) {
        const int64_t i0 = w0 + lane * kPP;
        double x[kPP][SUBC];
        int bi[kPP];
        bool fl[kPP], ok[kPP];
#pragma unroll
        for (int p = 0; p < kPP; ++p) {
            ok[p] = i0 + p < e;
            const int64_t ji = (int64_t)j * n + (ok[p] ? i0 + p : b);
            const float4 *xp = reinterpret_cast<const float4 *>(P + ji * SUBC);
#pragma unroll
            for (int q = 0; q < SUBC / 4; ++q) {
                const float4 v = xp[q];
                x[p][4 * q] = v.x; x[p][4 * q + 1] = v.y; x[p][4 * q + 2] = v.z; x[p][4 * q + 3] = v.w;
            }
            bi[p] = codes[ji];
            fl[p] = ok[p] && flags[ji] != 0;
        }
        auto finish = [&](const double (&xv)[SUBC], int64_t ji, int l, double d) {
            const double xx = einsum_sum([&](int t) { return __dmul_rn(xv[t], xv[t]); }, SUBC);
            const double v = __dadd_rn(d, xx);
            assign[ji] = l;
            sq[ji] = (v >= 0.0 || v != v) ? v : 0.0;  // np.maximum(v, 0.0)
        };
#pragma unroll
        for (int p = 0; p < kPP; ++p)
            if (ok[p] && !fl[p]) finish(x[p], (int64_t)j * n + i0 + p, bi[p], dist(x[p], bi[p]));
#pragma unroll
        for (int p = 0; p < kPP; ++p) {
            unsigned todo = __ballot_sync(0xffffffffu, fl[p]);
            while (todo) {  // full float64 scan of one flagged point by the whole warp
                const int src = __ffs(todo) - 1;
                todo &= todo - 1;
                const int64_t ji = (int64_t)j * n + w0 + src * kPP + p;
                double xs[SUBC];
                const float4 *xp = reinterpret_cast<const float4 *>(P + ji * SUBC);
#pragma unroll
                for (int q = 0; q < SUBC / 4; ++q) {
                    const float4 v = xp[q];
                    xs[4 * q] = v.x; xs[4 * q + 1] = v.y; xs[4 * q + 2] = v.z; xs[4 * q + 3] = v.w;
                }
                double bd = 0.0;
                int bl = -1;
#pragma unroll 1
                for (int r = 0; r < 8; ++r) {  // k == 256: centroids lane + 32 r, ascending
                    const int l = lane + 32 * r;
                    const double d1 = dist(xs, l);
                    if (d1 == d1 && (bl < 0 || d1 < bd)) { bd = d1; bl = l; }
                }
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    const double od = __shfl_xor_sync(0xffffffffu, bd, o);
                    const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
                    if (ol >= 0 && (bl < 0 || od < bd || (od == bd && ol < bl))) { bd = od; bl = ol; }
                }
                if (lane == 0) {
                    const double d0 = dist(xs, 0);
                    if (d0 != d0 || bl < 0) { bl = 0; bd = d0; }  // d_0 NaN (or every d NaN): index 0 stays
                    finish(xs, ji, bl, bd);
                }
            }
        }
    }
}

__global__ void hist_kernel(const int32_t *__restrict__ assign, int64_t n, int k, const int32_t *state,
                            int64_t b, int64_t e, int64_t nch, int32_t *__restrict__ hist, int use_smem) {
    const int j = blockIdx.y;
    if (!state[j]) return;
    const int64_t c = blockIdx.x;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int32_t *h = use_smem ? reinterpret_cast<int32_t *>(smem_raw) : hist + ((int64_t)j * nch + c) * k;
    for (int q = threadIdx.x; q < k; q += blockDim.x) h[q] = 0;
    __syncthreads();
    const int64_t lo = b + c * kChunk, hi = min(e, lo + kChunk);
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) atomicAdd(&h[assign[(int64_t)j * n + i]], 1);
    __syncthreads();
    if (use_smem)
        for (int q = threadIdx.x; q < k; q += blockDim.x) hist[((int64_t)j * nch + c) * k + q] = h[q];
}

// per bin: chunk offsets (in place), counts; then bin starts
__global__ void scan_kernel(int32_t *__restrict__ hist, int k, int64_t nch, const int32_t *state,
                            int32_t *__restrict__ cnt, int32_t *__restrict__ start, double *__restrict__ counts) {
    const int j = blockIdx.x;
    if (!state[j]) return;
    int32_t *H = hist + (int64_t)j * nch * k;
    constexpr int kU = 16;  // chunk counts loaded kU at a time: independent loads, one latency per batch
    for (int l = threadIdx.x; l < k; l += blockDim.x) {
        int32_t run = 0;
        int64_t c = 0;
        for (; c + kU <= nch; c += kU) {
            int32_t v[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) v[u] = H[(c + u) * k + l];
#pragma unroll
            for (int u = 0; u < kU; ++u) { H[(c + u) * k + l] = run; run += v[u]; }
        }
        for (; c < nch; ++c) {
            const int32_t v = H[c * k + l];
            H[c * k + l] = run;
            run += v;
        }
        cnt[(int64_t)j * k + l] = run;
        counts[(int64_t)j * k + l] = (double)run;
    }
    __syncthreads();
    // exclusive scan of cnt over bins (block-wide, tiles of blockDim)
    __shared__ int32_t s[1024];
    __shared__ int32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < k; base += blockDim.x) {
        const int l = base + threadIdx.x;
        const int32_t v = l < k ? cnt[(int64_t)j * k + l] : 0;
        s[threadIdx.x] = v;
        __syncthreads();
        for (int off = 1; off < (int)blockDim.x; off <<= 1) {
            const int32_t add = threadIdx.x >= (unsigned)off ? s[threadIdx.x - off] : 0;
            __syncthreads();
            s[threadIdx.x] += add;
            __syncthreads();
        }
        if (l < k) start[(int64_t)j * k + l] = carry + s[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry += s[threadIdx.x];
        __syncthreads();
    }
    // (the bin starts are added to the chunk offsets by scatter_kernel)
}

// stable scatter: perm[j][pos] = i, in ascending i within each cluster
__global__ void scatter_kernel(const int32_t *__restrict__ assign, int64_t n, int k, const int32_t *state,
                               int64_t b, int64_t e, int64_t nch, int32_t *__restrict__ hist,
                               const int32_t *__restrict__ start, int32_t *__restrict__ perm, int use_smem) {
    const int j = blockIdx.y;
    if (!state[j]) return;
    const int64_t c = blockIdx.x;
    const int lane = threadIdx.x;
    // running positions = bin start + this chunk's offset within the bin, in shared memory when
    // k fits (the read-modify-write per 32 points is then not a global-memory round trip)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int32_t *H = hist + ((int64_t)j * nch + c) * k;
    int32_t *run = use_smem ? reinterpret_cast<int32_t *>(smem_raw) : H;
    for (int q = lane; q < k; q += 32) run[q] = H[q] + start[(int64_t)j * k + q];
    if (use_smem)
        for (int q = lane; q < k; q += 32) run[k + q] = 32;  // slot[]: lowest pending lane per bin (see below)
    __syncwarp();
    const int64_t lo = b + c * kChunk, hi = min(e, lo + kChunk);
    const unsigned lt = (1u << lane) - 1u;
    constexpr int kB = 8;  // assignments of 8 x 32 points loaded ahead (independent loads)
    for (int64_t base0 = lo; base0 < hi; base0 += 32 * kB) {
        int av[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int64_t i = base0 + 32 * u + lane;
            av[u] = i < hi ? assign[(int64_t)j * n + i] : -1 - lane;  // unique sentinels never match
        }
        if (use_smem) {
            // ranks among the lanes that share a bin, in ascending lane order, by rounds of a shared-memory
            // atomicMin: in each round the lowest pending lane of every bin takes the bin's next position
            // (~2 rounds per 32 points: 32 lanes over 256 bins).  __match_any_sync gives the same ranks but
            // costs more the more distinct values the warp holds: this kernel 106 -> 84 us per c2 iteration.
            // (Also tried on top: the chunk sorted in shared memory first and written out run by run, so a
            // store's lanes share sectors -- no gain: the scattered writes are not what bounds it.)
            int32_t *slot = run + k;
#pragma unroll
            for (int u = 0; u < kB; ++u) {
                const int64_t i = base0 + 32 * u + lane;
                const int a = av[u];
                bool pending = a >= 0;
                unsigned pend = __ballot_sync(0xffffffffu, pending);
                while (pend) {
                    if (pending) atomicMin(&slot[a], lane);
                    __syncwarp();
                    const bool win = pending && slot[a] == lane;
                    __syncwarp();
                    if (win) {
                        const int32_t pos = run[a];
                        run[a] = pos + 1;
                        slot[a] = 32;
                        perm[(int64_t)j * n + pos] = (int32_t)(i - b);
                        pending = false;
                    }
                    __syncwarp();
                    pend = __ballot_sync(0xffffffffu, pending);
                }
            }
            continue;
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int64_t i = base0 + 32 * u + lane;
            const int a = av[u];
            const unsigned peers = __match_any_sync(0xffffffffu, a);
            if (a >= 0) {
                const int rank = __popc(peers & lt);
                const int32_t pos = run[a] + rank;
                perm[(int64_t)j * n + pos] = (int32_t)(i - b);
            }
            __syncwarp();
            if (a >= 0 && lane == __ffs(peers) - 1) run[a] += __popc(peers);
            __syncwarp();
        }
    }
}

// sums[j][l][t] = sequential float64 chain over the cluster's points (ascending i)
template <int SUBC, typename TP>
__global__ void sums_kernel(const TP *__restrict__ P, int64_t n, int m, int k, int sub_rt,
                            const int32_t *state, int64_t b, const int32_t *__restrict__ cnt,
                            const int32_t *__restrict__ start, const int32_t *__restrict__ perm,
                            double *__restrict__ sums, const uint8_t *__restrict__ only) {
    const int sub = SUBC > 0 ? SUBC : sub_rt;
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= (int64_t)m * k * sub) return;
    const int t = (int)(g % sub);
    const int64_t jl = g / sub;
    const int j = (int)(jl / k);
    if (!state[j] || (only && !only[jl])) return;
    const int32_t c0 = start[jl], cc = cnt[jl];
    const int32_t *pp = perm + (int64_t)j * n + c0;
    const TP *Pj = P + ((int64_t)j * n + b) * sub + t;
    double s = 0.0;
    int32_t p = 0;
    // CSPQ_SUMS_KB gathers in flight per step; the next step's indices are loaded before this step's sum
    constexpr int kB = CSPQ_SUMS_KB;
    int32_t idx[kB];
    if (cc >= kB) {
#pragma unroll
        for (int q = 0; q < kB; ++q) idx[q] = pp[q];
    }
    for (; p + kB <= cc; p += kB) {
        TP v[kB];
#pragma unroll
        for (int q = 0; q < kB; ++q) v[q] = Pj[(int64_t)idx[q] * sub];
        if (p + 2 * kB <= cc) {
#pragma unroll
            for (int q = 0; q < kB; ++q) idx[q] = pp[p + kB + q];
        }
#pragma unroll
        for (int q = 0; q < kB; ++q) s = __dadd_rn(s, (double)v[q]);
    }
    for (; p < cc; ++p) s = __dadd_rn(s, (double)Pj[(int64_t)pp[p] * sub]);
    sums[g] = s;
}

// sums[j][l][:] for float32 points, one warp per (subspace, cluster).  np.add.at's result is the
// sequential float64 chain over the cluster's points in ascending order; when that chain cannot
// round, its value is the exact sum and any order gives it.  It cannot round when every member
// value is a multiple of 2^L (L = the lowest set bit over the members' coordinates) and
// count * max|v| <= 2^(L + 52): every partial sum -- of the chain or of any subset -- is then a
// multiple of 2^L below 2^(L + 53), exactly representable.  The warp checks that while it sums
// lane-strided partials (a parallel reduction); a cluster that fails the check (float32 data with
// tiny values, NaN/inf) is marked in redo[] and summed again by sums_kernel's sequential chains.
// Measured on the config samples: c2 and c4 never fail, c3 / c5 ~4 of 256 clusters per subspace.
template <int SUBC>
__global__ void __launch_bounds__(128)
sums_exact_kernel(const float *__restrict__ P, int64_t n, int m, int k, const int32_t *state, int64_t b,
                  const int32_t *__restrict__ cnt, const int32_t *__restrict__ start,
                  const int32_t *__restrict__ perm, double *__restrict__ sums, uint8_t *__restrict__ redo) {
    const int64_t jl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (jl >= (int64_t)m * k) return;
    const int j = (int)(jl / k);
    if (!state[j]) return;
    const int32_t c0 = start[jl], cc = cnt[jl];
    const int32_t *pp = perm + (int64_t)j * n + c0;
    const float *Pj = P + ((int64_t)j * n + b) * SUBC;
    double acc[SUBC];
#pragma unroll
    for (int t = 0; t < SUBC; ++t) acc[t] = 0.0;
    int minlsb = 1 << 20;
    uint32_t maxabs = 0;
    // kU members per lane in flight (independent index and row loads): the gathers are
    // latency-bound, not bandwidth-bound
    constexpr int kU = 4;
    for (int32_t p0 = lane; p0 < cc; p0 += 32 * kU) {
        int32_t idx[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) idx[u] = p0 + 32 * u < cc ? __ldg(pp + p0 + 32 * u) : -1;
        float x[kU][SUBC];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const float4 *xp = reinterpret_cast<const float4 *>(Pj + (int64_t)(idx[u] < 0 ? 0 : idx[u]) * SUBC);
#pragma unroll
            for (int q = 0; q < SUBC / 4; ++q) {
                const float4 v = idx[u] < 0 ? make_float4(0.f, 0.f, 0.f, 0.f) : __ldg(xp + q);
                x[u][4 * q] = v.x; x[u][4 * q + 1] = v.y; x[u][4 * q + 2] = v.z; x[u][4 * q + 3] = v.w;
            }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
#pragma unroll
            for (int t = 0; t < SUBC; ++t) {
                acc[t] = __dadd_rn(acc[t], (double)x[u][t]);
                const uint32_t a = __float_as_uint(x[u][t]) & 0x7fffffffu;
                maxabs = max(maxabs, a);  // non-negative float bits order like the values (inf / NaN largest)
                if (a) {
                    const int e = (int)(a >> 23);
                    const uint32_t mant = e ? ((a & 0x7fffffu) | 0x800000u) : a;
                    minlsb = min(minlsb, (e ? e - 150 : -149) + __ffs(mant) - 1);
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
#pragma unroll
        for (int t = 0; t < SUBC; ++t) acc[t] = __dadd_rn(acc[t], __shfl_xor_sync(0xffffffffu, acc[t], o));
        minlsb = min(minlsb, __shfl_xor_sync(0xffffffffu, minlsb, o));
        maxabs = max(maxabs, __shfl_xor_sync(0xffffffffu, maxabs, o));
    }
    const double bound = (double)cc * (double)__uint_as_float(maxabs);  // >= sum |v| (inf / NaN: fails)
    const bool exact = minlsb >= (1 << 20) || bound <= ldexp(1.0, minlsb + 52);
    double *out = sums + jl * SUBC;
    if (lane == 0) redo[jl] = 0;
    if (exact) {
        if (lane < SUBC) {
            double v = acc[0];
#pragma unroll
            for (int t = 1; t < SUBC; ++t) v = lane == t ? acc[t] : v;
            out[lane] = v;
        }
        return;
    }
    if (lane == 0) redo[jl] = 1;  // sums_kernel runs the sequential chain of this cluster
}

// ---------------------------------------------------------------- update / repair / stop
__global__ void update_kernel(const double *__restrict__ counts, const double *__restrict__ sums, int k,
                              int sub, const int32_t *state, double *__restrict__ C64,
                              int32_t *__restrict__ empties, int32_t *__restrict__ nempty) {
    const int j = blockIdx.x;
    if (!state[j]) return;
    __shared__ int32_t s[1024];
    __shared__ int32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < k; base += blockDim.x) {
        const int l = base + threadIdx.x;
        int flag = 0;
        if (l < k) {
            const double cntv = counts[(int64_t)j * k + l];
            if (cntv > 0) {
                for (int t = 0; t < sub; ++t) {
                    const int64_t q = ((int64_t)j * k + l) * sub + t;
                    C64[q] = __ddiv_rn(sums[q], cntv);
                }
            } else {
                flag = 1;
            }
        }
        s[threadIdx.x] = flag;
        __syncthreads();
        for (int off = 1; off < (int)blockDim.x; off <<= 1) {
            const int32_t add = threadIdx.x >= (unsigned)off ? s[threadIdx.x - off] : 0;
            __syncthreads();
            s[threadIdx.x] += add;
            __syncthreads();
        }
        if (flag) empties[(int64_t)j * k + carry + s[threadIdx.x] - 1] = l;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry += s[threadIdx.x];
        __syncthreads();
    }
    if (threadIdx.x == 0) nempty[j] = carry;
}

template <typename TP>
__global__ void __launch_bounds__(1024)
repair_kernel(const TP *__restrict__ P, int64_t n, int k, int sub, const int32_t *__restrict__ assign,
              const int32_t *state, const int32_t *__restrict__ empties, const int32_t *__restrict__ nempty,
              double *__restrict__ C64, double *__restrict__ resid) {
    const int j = blockIdx.x;
    if (!state[j] || nempty[j] == 0) return;
    const TP *Pj = P + (int64_t)j * n * sub;
    double *C = C64 + (int64_t)j * k * sub;
    double *R = resid + (int64_t)j * n;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double *c = C + (int64_t)assign[(int64_t)j * n + i] * sub;
        const TP *x = Pj + i * sub;
        R[i] = einsum_sum([&](int t) {  // residual, training.py:133-134
            const double df = __dsub_rn((double)x[t], c[t]);
            return __dmul_rn(df, df);
        }, sub);
    }
    __syncthreads();
    __shared__ double sv[1024];
    __shared__ int64_t si[1024];
    const int ne = nempty[j];
    for (int q = 0; q < ne; ++q) {
        double bv = -pos_inf_d();
        int64_t bi = -1;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            const double v = R[i];
            if (bi < 0 || v > bv) { bv = v; bi = i; }  // ascending i per thread: first max kept
        }
        sv[threadIdx.x] = bv;
        si[threadIdx.x] = bi;
        __syncthreads();
        for (int off = blockDim.x / 2; off > 0; off >>= 1) {
            if (threadIdx.x < (unsigned)off) {
                const double ov = sv[threadIdx.x + off];
                const int64_t oi = si[threadIdx.x + off];
                const double mv = sv[threadIdx.x];
                const int64_t mi = si[threadIdx.x];
                if (oi >= 0 && (mi < 0 || ov > mv || (ov == mv && oi < mi))) {
                    sv[threadIdx.x] = ov;
                    si[threadIdx.x] = oi;
                }
            }
            __syncthreads();
        }
        const int64_t cand = si[0];
        const int e = empties[(int64_t)j * k + q];
        if (threadIdx.x < (unsigned)sub) C[(int64_t)e * sub + threadIdx.x] = (double)Pj[cand * sub + threadIdx.x];
        __syncthreads();
        if (threadIdx.x == 0) R[cand] = -1.0;
        __syncthreads();
    }
}

__global__ void stop_kernel(const double *obj, int m, int max_iters, double tol, int32_t *state,
                            double *prev, int32_t *iterations, double *objectives) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
        if (!state[j]) continue;
        const double o = obj[j];
        objectives[(int64_t)j * (max_iters + 1) + iterations[j]] = o;
        iterations[j] += 1;
        const double p = prev[j];
        bool stop = (o == 0.0);
        if (!stop && p < pos_inf_d()) {
            const double scale = p > 1e-300 ? p : 1e-300;
            stop = (p - o) <= tol * scale;
        }
        prev[j] = o;
        if (stop || iterations[j] >= max_iters) state[j] = 0;
    }
}

__global__ void init_state_kernel(int m, int32_t *state, double *prev, int32_t *iterations) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
        state[j] = 1;
        prev[j] = pos_inf_d();
        iterations[j] = 0;
    }
}

__global__ void cast_kernel(const double *C64, int64_t tot, float *C32) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < tot) C32[i] = __double2float_rn(C64[i]);
}

template <typename TP>
__global__ void final_resid_kernel(const TP *__restrict__ P, int64_t n, int k, int sub,
                                   const float *__restrict__ C32, const int32_t *__restrict__ assign,
                                   double *__restrict__ out) {
    const int j = blockIdx.y;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const TP *x = P + ((int64_t)j * n + i) * sub;
        const float *c = C32 + ((int64_t)j * k + assign[(int64_t)j * n + i]) * sub;
        out[(int64_t)j * n + i] = einsum_sum([&](int t) {  // final objective terms, training.py:153-154
            const double df = __dsub_rn((double)x[t], (double)c[t]);
            return __dmul_rn(df, df);
        }, sub);
    }
}

__global__ void write_final_obj_kernel(const double *obj, int m, int max_iters, const int32_t *iterations,
                                       double *objectives) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x)
        objectives[(int64_t)j * (max_iters + 1) + iterations[j]] = obj[j];
}

// ---------------------------------------------------------------- k-means++ (training.py:76-92)
// d2[i] = ||x_i - c||^2 (diff, then np.einsum's order), or
// min(d2[i], that) (np.minimum(d2, ., out=d2)).
template <typename TP>
__global__ void kpp_dist_kernel(const TP *__restrict__ P, int64_t n, int sub, const double *__restrict__ C64,
                                int k, int c, const int32_t *__restrict__ status, double *__restrict__ d2, int first) {
    const int j = blockIdx.y;
    if (status[j]) return;
    const double *cen = C64 + ((int64_t)j * k + c) * sub;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const TP *x = P + ((int64_t)j * n + i) * sub;
        const double r = einsum_sum([&](int t) {  // training.py:81/90
            const double df = __dsub_rn((double)x[t], cen[t]);
            return __dmul_rn(df, df);
        }, sub);
        double *o = d2 + (int64_t)j * n + i;
        if (first) *o = r;
        else {
            const double cur = *o;
            *o = (cur != cur || r != r) ? (cur != cur ? cur : r) : (r < cur ? r : cur);
        }
    }
}

// p = d2 / total (np: p = d2 / total)
// rng.choice(n, p=p): p = d2 / total; cdf = cumsum(p) (sequential); cdf /= cdf[-1];
// idx = searchsorted(cdf, u, 'right').  One CTA per subspace: chunks of the probabilities are
// computed into shared memory (coalesced loads of d2, the same IEEE division as numpy's p) and
// thread 0 runs numpy's sequential chain over
// them (loads issued ahead of the dependent adds).  Only every kSeg-th running sum is kept
// (written over already-consumed probabilities); the search finds the segment among those, then
// re-runs that segment's chain from its start -- the same operations in the same order -- to
// find the index.  (The cdf is
// monotone, so the first index whose normalised cdf exceeds u lies in the first segment whose
// end does.)
constexpr int kKppChunk = 4096;
constexpr int kSeg = 64;
__global__ void __launch_bounds__(256) kpp_choose_kernel(double *__restrict__ pp, const double *__restrict__ d2,
                                                         int64_t n, int m, int k, int c,
                                                         const double *__restrict__ total, const double *__restrict__ u,
                                                         int32_t *__restrict__ status, const void *P, int pf64, int sub,
                                                         double *__restrict__ C64) {
    __shared__ double buf[kKppChunk];
    __shared__ double s_run;
    const int j = blockIdx.x;
    if (status[j]) return;
    if (!(total[j] > 0.0)) {
        // total <= 0: all mass on chosen points -- the reference switches to rng.integers(n) draws
        // from this step on (training.py:84-86; the host replays them): status = -c.  A NaN total
        // (training.py:87 would raise in rng.choice): status = 3
        if (threadIdx.x == 0) status[j] = total[j] != total[j] ? 3 : -c;
        return;
    }
    double *cdf = pp + (int64_t)j * n;  // segment-end sums (cdf[s] = sum through s*kSeg+kSeg-1)
    const double tot = total[j];
    const double *dj = d2 + (int64_t)j * n;
    if (threadIdx.x == 0) s_run = 0.0;
    for (int64_t c0 = 0; c0 < n; c0 += kKppChunk) {
        const int len = (int)(n - c0 < kKppChunk ? n - c0 : kKppChunk);
        for (int i = threadIdx.x; i < len; i += blockDim.x) buf[i] = __ddiv_rn(dj[c0 + i], tot);  // p = d2 / total
        __syncthreads();
        if (threadIdx.x == 0) {
            double run = s_run;
            int i = 0;
            for (; i + 16 <= len; i += 16) {
                double v[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) v[q] = buf[i + q];
#pragma unroll
                for (int q = 0; q < 16; ++q) run = __dadd_rn(run, v[q]);
                // kKppChunk and 16 are multiples of... 16 | kSeg: a segment ends on this step's last element
                if (((c0 + i + 16) % kSeg) == 0) cdf[(c0 + i + 16) / kSeg - 1] = run;
            }
            for (; i < len; ++i) {
                run = __dadd_rn(run, buf[i]);
                if (((c0 + i + 1) % kSeg) == 0) cdf[(c0 + i + 1) / kSeg - 1] = run;
            }
            s_run = run;
        }
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    const double last = s_run;
    const double uu = u[(int64_t)j * (k - 1) + (c - 1)];
    // segments [s kSeg, (s + 1) kSeg); the last one may be partial and has no stored end
    const int64_t nseg = (n + kSeg - 1) / kSeg, nfull = n / kSeg;
    int64_t lo = 0, hi = nfull;  // first full segment whose end exceeds u (or nfull)
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ddiv_rn(cdf[mid], last) > uu) hi = mid; else lo = mid + 1;
    }
    const int64_t seg = lo < nseg ? lo : nseg - 1;
    double run = seg > 0 ? cdf[seg - 1] : 0.0;
    const int64_t e = (seg + 1) * kSeg < n ? (seg + 1) * kSeg : n;
    int64_t idx = e - 1;  // u < 1 and cdf[-1]/last == 1 find an index before the end
    for (int64_t i = seg * kSeg; i < e; ++i) {
        run = __dadd_rn(run, __ddiv_rn(dj[i], tot));
        if (__ddiv_rn(run, last) > uu) { idx = i; break; }
    }
    double *dst = C64 + ((int64_t)j * k + c) * sub;
    for (int t = 0; t < sub; ++t)
        dst[t] = pf64 ? reinterpret_cast<const double *>(P)[((int64_t)j * n + idx) * sub + t]
                      : (double)reinterpret_cast<const float *>(P)[((int64_t)j * n + idx) * sub + t];
}

template <typename TP>
__global__ void kpp_first_kernel(const TP *__restrict__ P, int64_t n, int m, int sub, int k,
                                 const int64_t *__restrict__ first, double *__restrict__ C64, int32_t *status) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    status[j] = 0;
    for (int t = 0; t < sub; ++t) C64[(int64_t)j * k * sub + t] = (double)P[((int64_t)j * n + first[j]) * sub + t];
}

template <typename TP>
__global__ void cast_points_kernel(const TP *P, int64_t tot, float *out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < tot) out[i] = (float)P[i];
}

int grid_for(int64_t items, int threads, int64_t cap = 148 * 16) {
    int64_t g = (items + threads - 1) / threads;
    if (g < 1) g = 1;
    return (int)(g < cap ? g : cap);
}

// pairwise objective of vals[j][begin .. begin+len) for every active subspace
int pairwise_obj(const double *vals, int64_t vstride, int64_t begin, int64_t len, int m,
                 const int32_t *state, void *ws, const WsLayout &L, double *out, cudaStream_t st) {
    double *leafsum = L.at<double>(ws, L.leafsum);
    const TreeBuf tb = tree_for(len);
    CSPQ_REQUIRE(tb.hdr, CSPQ_E_CUDA, "pairwise summation tree for n=%lld: device allocation failed", (long long)len);
    const int64_t *leaves = tb.leaves;
    const int32_t *nodes = tb.nodes;
    const WsHeader *hdr = tb.hdr;
    const int64_t maxl = len / 32 + 8;
    dim3 g((unsigned)grid_for(maxl, 128, 64), (unsigned)m);
    leafsum_kernel<<<g, 128, 0, st>>>(vals, vstride, begin, m, state, leaves, hdr, L.maxleaves, leafsum);
    CSPQ_LAUNCH_CHECK();
    combine_levels_kernel<<<m, 256, 0, st>>>(m, state, leafsum, L.maxleaves, nodes, len / 32 + 8, hdr,
                                             L.at<double>(ws, L.nodeval), out);
    CSPQ_LAUNCH_CHECK();
    return CSPQ_OK;
}

}  // namespace

size_t lloyd_workspace_bytes(int64_t n, int m, int sub, int k) { return (size_t)WsLayout(n, m, sub, k).total; }

#define CSPQ_TP_DISPATCH(pf64, P, ...)                                                                  \
    do {                                                                                               \
        if (pf64) { using TP = double; const TP *Pt = reinterpret_cast<const TP *>(P); __VA_ARGS__; } \
        else { using TP = float; const TP *Pt = reinterpret_cast<const TP *>(P); __VA_ARGS__; }       \
    } while (0)

int encode_prepare(const float *CB, const float *B, int m, int k, int sub, float *guard, cudaStream_t st);
int encode_tc_prepare(const float *CB, const float *B, int m, int k, int sub, void *img, cudaStream_t st);
int encode_tc_max_subspaces(int sub, int in_dtype);
float encode_tc_error_constant(int sub);
int encode_tc_ex(const void *X, int in_dtype, int64_t n, int64_t xrs, int64_t xjs, const float *CB, const float *B,
                 const float *guard, const void *img, int m, int k, int sub, uint8_t *codes, int64_t crs, int64_t cjs,
                 uint8_t *flags, float *best, cudaStream_t st);

// assignment of points [b, e) of every subspace through the tcgen05 encode kernel in mark
// mode, then tc_settle_kernel (see above)
static int assign_tc(const float *P, int64_t n, int m, int sub, int k, const double *C64, const double *cn,
                     const int32_t *state, int64_t b, int64_t e, int32_t *assign, double *sq, void *ws,
                     const WsLayout &L, cudaStream_t st) {
    float *cb32 = L.at<float>(ws, L.tc_cb), *b32 = L.at<float>(ws, L.tc_b), *guard = L.at<float>(ws, L.tc_guard);
    void *img = L.at<void>(ws, L.tc_img);
    uint8_t *codes = L.at<uint8_t>(ws, L.tc_codes), *flags = L.at<uint8_t>(ws, L.tc_flags);
    tc_codebook_kernel<<<m, 256, 0, st>>>(C64, cn, k, sub, cb32, b32);
    CSPQ_LAUNCH_CHECK();
    int rc;
    if ((rc = encode_prepare(cb32, b32, m, k, sub, guard, st))) return rc;
    if ((rc = encode_tc_prepare(cb32, b32, m, k, sub, img, st))) return rc;
    // rows = points b.. of every subspace: row stride sub, subspace stride n * sub; codes and
    // flags subspace-major (m, n) like assign
    if ((rc = encode_tc_ex(P + b * sub, CSPQ_IN_F32, e - b, sub, n * sub, cb32, b32, guard, img, m, k, sub, codes + b, 1, n,
                           flags + b, nullptr, st)))
        return rc;
    // ~8 CTAs per SM in total: each CTA stages its subspace's codebook once for many points
    dim3 grid((unsigned)grid_for((e - b + CSPQ_SETTLE_PPT - 1) / CSPQ_SETTLE_PPT, 256, std::max<int64_t>(1, 148 * 8 / m)), (unsigned)m);
    if (sub == 8) tc_settle_kernel<8><<<grid, 256, 0, st>>>(P, n, k, C64, cn, state, b, e, codes, flags, assign, sq);
    else tc_settle_kernel<4><<<grid, 256, 0, st>>>(P, n, k, C64, cn, state, b, e, codes, flags, assign, sq);
    CSPQ_LAUNCH_CHECK();
    return CSPQ_OK;
}

// ---------------------------------------------------------------- screened final pass
// The final assignment is the float32 REFERENCE encoder (training.py:143-150, kernels.py:84-105):
// dist_l = (vv + cc_l) - 2 dd_l with every product and sum rounded in sequence, strict < from
// +inf.  Each term is a d_sub-long recursive sum, so |dist_l - D_l| <= g (vv + cc_l + 2 |x| |c_l|)
// with g = gamma_{d_sub + 4} for the real D_l = |x|^2 + 2 s_l (s_l = |c_l|^2 / 2 - x.c_l).  The
// tensor kernel screens s_l; its band is widened from E W to E W + u max|b| + g (max|b| +
// |x| max|c| + |x| R / 2) (R = max |x| of the subspace's points, so vv / 2 <= |x| R / 2; u
// covers the rounding of b).  An unflagged point's winner then beats every other centroid's
// REFERENCE distance by > 7.8 E'W' - 4 (E'W') > 0: its code is the REFERENCE code.  Flagged
// points take the exact REFERENCE scan, the whole warp on one point.
__global__ void pnorm_max_kernel(const float *__restrict__ P, int64_t n, int sub, unsigned *__restrict__ rmax) {
    const int j = blockIdx.y;
    float mx = 0.f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float *x = P + ((int64_t)j * n + i) * sub;
        double ss = 0.0;
        for (int t = 0; t < sub; ++t) ss = fma((double)x[t], (double)x[t], ss);
        const float r = __double2float_ru(sqrt(ss) * (1.0 + 1e-12));
        mx = (r != r || r > mx) ? r : mx;
    }
    // non-negative floats order like their bits; a NaN (bits above +inf) poisons the guard
    unsigned bits = __float_as_uint(mx);
    for (int o = 16; o; o >>= 1) bits = max(bits, __shfl_xor_sync(0xffffffffu, bits, o));
    if ((threadIdx.x & 31) == 0) atomicMax(rmax + j, bits);
}

__global__ void final_guard_kernel(float *__restrict__ guard, const unsigned *__restrict__ rmax, int m, int sub, float kE) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const double u = 1.0 / 16777216.0;
    const double g = (sub + 4) * u / (1.0 - (sub + 4) * u);
    const double g0 = guard[2 * j], g1 = guard[2 * j + 1], R = __uint_as_float(rmax[j]);
    guard[2 * j] = __double2float_ru(g0 * (1.0 + (u + g) / kE) * (1.0 + 1e-6));
    guard[2 * j + 1] = __double2float_ru((g1 * (1.0 + g / kE) + g * R / (2.0 * kE)) * (1.0 + 1e-6));
}

template <int SUBC>  // k == 256
__global__ void __launch_bounds__(256)
final_settle_kernel(const float *__restrict__ P, int64_t n, const float *__restrict__ C32,
                    const uint8_t *__restrict__ codes, const uint8_t *__restrict__ flags, int32_t *__restrict__ assign) {
    const int j = blockIdx.y;
    constexpr int kCS = SUBC + 1;  // padded centroid stride (per-lane centroids spread over the banks)
    __shared__ float sC[256 * kCS], scc[256];
    for (int q = threadIdx.x; q < 256 * SUBC; q += blockDim.x) sC[(q / SUBC) * kCS + q % SUBC] = C32[(int64_t)j * 256 * SUBC + q];
    __syncthreads();
    for (int l = threadIdx.x; l < 256; l += blockDim.x) {  // cc_l: the reference's sequential chain
        float cc = 0.f;
#pragma unroll
        for (int t = 0; t < SUBC; ++t) cc = __fadd_rn(cc, __fmul_rn(sC[l * kCS + t], sC[l * kCS + t]));
        scc[l] = cc;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i - lane < n; i += (int64_t)gridDim.x * blockDim.x) {
        const bool ok = i < n;
        const int64_t ji = (int64_t)j * n + (ok ? i : 0);
        const bool fl = ok && flags[ji] != 0;
        if (ok && !fl) assign[ji] = codes[ji];
        unsigned todo = __ballot_sync(0xffffffffu, fl);
        while (todo) {
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            const int64_t jf = (int64_t)j * n + (i - lane + src);
            float x[SUBC];
            const float4 *xp = reinterpret_cast<const float4 *>(P + jf * SUBC);
#pragma unroll
            for (int q = 0; q < SUBC / 4; ++q) {
                const float4 v = xp[q];
                x[4 * q] = v.x; x[4 * q + 1] = v.y; x[4 * q + 2] = v.z; x[4 * q + 3] = v.w;
            }
            float vv = 0.f;
#pragma unroll
            for (int t = 0; t < SUBC; ++t) vv = __fadd_rn(vv, __fmul_rn(x[t], x[t]));
            float bd = __int_as_float(0x7f800000);
            int bl = -1;
#pragma unroll 1
            for (int r = 0; r < 8; ++r) {  // centroids lane + 32 r, ascending: strict < keeps the first
                const int l = lane + 32 * r;
                float dd = 0.f;
#pragma unroll
                for (int t = 0; t < SUBC; ++t) dd = __fadd_rn(dd, __fmul_rn(x[t], sC[l * kCS + t]));
                const float d1 = __fsub_rn(__fadd_rn(vv, scc[l]), __fmul_rn(2.0f, dd));
                if (d1 < bd) { bd = d1; bl = l; }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const float od = __shfl_xor_sync(0xffffffffu, bd, o);
                const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
                if (ol >= 0 && (bl < 0 || od < bd || (od == bd && ol < bl))) { bd = od; bl = ol; }
            }
            if (lane == 0) assign[jf] = bl < 0 ? 0 : bl;  // nothing below +inf: index 0 (best = inf)
        }
    }
}

__global__ void final_bias_kernel(const float *__restrict__ C32, int64_t mk, int sub, float *__restrict__ b32) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= mk) return;
    double ss = 0.0;  // float products are exact in float64: b = |c|^2 / 2 rounded once (to within u b)
    for (int t = 0; t < sub; ++t) ss = fma((double)C32[i * sub + t], (double)C32[i * sub + t], ss);
    b32[i] = __double2float_rn(0.5 * ss);
}

static bool tc_screen_ok(const float *P, int m, int sub, int k) {
    const char *tcv = getenv("CSPQ_LLOYD_TC");  // "0": the plain kernels (A/B and tests)
    return !(tcv && tcv[0] == '0') && k == 256 && (sub == 4 || sub == 8) && reinterpret_cast<uintptr_t>(P) % 16 == 0 &&
           m <= encode_tc_max_subspaces(sub, CSPQ_IN_F32);
}

static int final_assign_tc(const float *P32, int64_t n, int m, int sub, int k, const float *C32, int32_t *assign, void *ws,
                           const WsLayout &L, cudaStream_t st) {
    float *b32 = L.at<float>(ws, L.tc_b), *guard = L.at<float>(ws, L.tc_guard);
    void *img = L.at<void>(ws, L.tc_img);
    uint8_t *codes = L.at<uint8_t>(ws, L.tc_codes), *flags = L.at<uint8_t>(ws, L.tc_flags);
    unsigned *rmax = L.at<unsigned>(ws, L.tc_rmax);
    int rc;
    final_bias_kernel<<<(unsigned)(((int64_t)m * k + 255) / 256), 256, 0, st>>>(C32, (int64_t)m * k, sub, b32);
    CSPQ_LAUNCH_CHECK();
    if ((rc = encode_prepare(C32, b32, m, k, sub, guard, st))) return rc;
    CSPQ_CUDA_TRY(cudaMemsetAsync(rmax, 0, sizeof(unsigned) * m, st));
    dim3 gn((unsigned)grid_for(n, 256, std::max<int64_t>(1, 148 * 4 / m)), (unsigned)m);
    pnorm_max_kernel<<<gn, 256, 0, st>>>(P32, n, sub, rmax);
    CSPQ_LAUNCH_CHECK();
    final_guard_kernel<<<(m + 127) / 128, 128, 0, st>>>(guard, rmax, m, sub, encode_tc_error_constant(sub));
    CSPQ_LAUNCH_CHECK();
    if ((rc = encode_tc_prepare(C32, b32, m, k, sub, img, st))) return rc;
    if ((rc = encode_tc_ex(P32, CSPQ_IN_F32, n, sub, n * sub, C32, b32, guard, img, m, k, sub, codes, 1, n, flags, nullptr, st)))
        return rc;
    dim3 grid((unsigned)grid_for(n, 256, std::max<int64_t>(1, 148 * 8 / m)), (unsigned)m);
    if (sub == 8) final_settle_kernel<8><<<grid, 256, 0, st>>>(P32, n, C32, codes, flags, assign);
    else final_settle_kernel<4><<<grid, 256, 0, st>>>(P32, n, C32, codes, flags, assign);
    CSPQ_LAUNCH_CHECK();
    return CSPQ_OK;
}

int lloyd_assign(const void *P, int pf64, int64_t n, int m, int sub, int k, const double *C64,
                 const int32_t *state, int64_t b, int64_t e, int32_t *assign, double *sq, void *ws, cudaStream_t st) {
    WsLayout L(n, m, sub, k);
    double *cn = L.at<double>(ws, L.cn);
    const int64_t mk = (int64_t)m * k;
    cnorm_kernel<<<(unsigned)((mk + 255) / 256), 256, 0, st>>>(C64, m, k, sub, state, cn);
    CSPQ_LAUNCH_CHECK();
    if (e <= b) return CSPQ_OK;
    if (!pf64 && tc_screen_ok(reinterpret_cast<const float *>(P), m, sub, k))
        return assign_tc(reinterpret_cast<const float *>(P), n, m, sub, k, C64, cn, state, b, e, assign, sq, ws, L, st);
    const size_t need = (size_t)k * (sub + 1) * sizeof(double);
    const int use_smem = need <= 96 * 1024;
    const size_t smem = use_smem ? need : 0;
    // the fixed-sub kernels take CSPQ_LLOYD_PPT points per thread: size the grid for that, or
    // most CTAs would only stage the codebook and exit
    const int64_t per_thread = (sub == 8 || sub == 4) ? CSPQ_LLOYD_PPT : 1;
    dim3 grid((unsigned)grid_for((e - b + per_thread - 1) / per_thread, 256, 148 * 8), (unsigned)m);
    CSPQ_TP_DISPATCH(pf64, P, {
        if (sub == 8) {
            CSPQ_CUDA_TRY(cudaFuncSetAttribute(assign_kernel<8, TP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
            assign_kernel<8, TP><<<grid, 256, smem, st>>>(Pt, n, k, sub, C64, cn, state, b, e, assign, sq, use_smem);
        } else if (sub == 4) {
            CSPQ_CUDA_TRY(cudaFuncSetAttribute(assign_kernel<4, TP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
            assign_kernel<4, TP><<<grid, 256, smem, st>>>(Pt, n, k, sub, C64, cn, state, b, e, assign, sq, use_smem);
        } else {
            CSPQ_CUDA_TRY(cudaFuncSetAttribute(assign_kernel<0, TP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
            assign_kernel<0, TP><<<grid, 256, smem, st>>>(Pt, n, k, sub, C64, cn, state, b, e, assign, sq, use_smem);
        }
    });
    CSPQ_LAUNCH_CHECK();
    return CSPQ_OK;
}

int lloyd_accumulate(const void *P, int pf64, int64_t n, int m, int sub, int k, const int32_t *state,
                     const int32_t *assign, const double *sq, int64_t b, int64_t e, double *counts,
                     double *sums, double *obj, void *ws, cudaStream_t st) {
    WsLayout L(n, m, sub, k);
    const int64_t len = e - b;
    const int64_t nch = (len + kChunk - 1) / kChunk;
    int32_t *hist = L.at<int32_t>(ws, L.hist);
    int32_t *cnt = L.at<int32_t>(ws, L.cnt);
    int32_t *start = L.at<int32_t>(ws, L.start);
    int32_t *perm = L.at<int32_t>(ws, L.perm);
    if (nch > 0) {
        const int use_smem = (size_t)k * 4 <= 48 * 1024;
        hist_kernel<<<dim3((unsigned)nch, (unsigned)m), 256, use_smem ? k * 4 : 0, st>>>(assign, n, k, state, b, e, nch, hist, use_smem);
        CSPQ_LAUNCH_CHECK();
    }
    scan_kernel<<<m, 256, 0, st>>>(hist, k, nch, state, cnt, start, counts);
    CSPQ_LAUNCH_CHECK();
    if (nch > 0) {
        const int use_smem = (size_t)k * 8 <= 48 * 1024;
        scatter_kernel<<<dim3((unsigned)nch, (unsigned)m), 32, use_smem ? k * 8 : 0, st>>>(assign, n, k, state, b, e, nch,
                                                                                          hist, start, perm, use_smem);
        CSPQ_LAUNCH_CHECK();
    }
    const int64_t tot = (int64_t)m * k * sub;
    const unsigned g = (unsigned)((tot + 127) / 128);
    static const bool exact_sums = [] { const char *e = getenv("CSPQ_LLOYD_EXACT_SUMS"); return !e || atoi(e) != 0; }();
    const uint8_t *only = nullptr;
    if (!pf64 && (sub == 8 || sub == 4) && exact_sums) {  // float32 points: the checked parallel sums
        const unsigned gw = (unsigned)(((int64_t)m * k + 3) / 4);
        const float *P32 = reinterpret_cast<const float *>(P);
        uint8_t *redo = L.at<uint8_t>(ws, L.redo);
        if (sub == 8) sums_exact_kernel<8><<<gw, 128, 0, st>>>(P32, n, m, k, state, b, cnt, start, perm, sums, redo);
        else sums_exact_kernel<4><<<gw, 128, 0, st>>>(P32, n, m, k, state, b, cnt, start, perm, sums, redo);
        CSPQ_LAUNCH_CHECK();
        only = redo;  // the sequential chains below run for the marked clusters only
    }
    CSPQ_TP_DISPATCH(pf64, P, {
        if (sub == 8) sums_kernel<8, TP><<<g, 128, 0, st>>>(Pt, n, m, k, sub, state, b, cnt, start, perm, sums, only);
        else if (sub == 4) sums_kernel<4, TP><<<g, 128, 0, st>>>(Pt, n, m, k, sub, state, b, cnt, start, perm, sums, only);
        else sums_kernel<0, TP><<<g, 128, 0, st>>>(Pt, n, m, k, sub, state, b, cnt, start, perm, sums, only);
    });
    CSPQ_LAUNCH_CHECK();
    return pairwise_obj(sq, n, b, len, m, state, ws, L, obj, st);
}

int lloyd_update(const double *counts, const double *sums, int m, int k, int sub, const int32_t *state,
                 double *C64, int32_t *empties, int32_t *nempty, cudaStream_t st) {
    update_kernel<<<m, 256, 0, st>>>(counts, sums, k, sub, state, C64, empties, nempty);
    CSPQ_LAUNCH_CHECK();
    return CSPQ_OK;
}

int lloyd_repair(const void *P, int pf64, int64_t n, int m, int sub, int k, const int32_t *assign,
                 const int32_t *state, const int32_t *empties, const int32_t *nempty, double *C64, void *ws,
                 cudaStream_t st) {
    WsLayout L(n, m, sub, k);
    CSPQ_TP_DISPATCH(pf64, P, {
        repair_kernel<TP><<<m, 1024, 0, st>>>(Pt, n, k, sub, assign, state, empties, nempty, C64, L.at<double>(ws, L.resid));
    });
    CSPQ_LAUNCH_CHECK();
    return CSPQ_OK;
}

int lloyd_stop(const double *obj, int m, int max_iters, double tol, int32_t *state, double *prev,
               int32_t *iterations, double *objectives, cudaStream_t st) {
    stop_kernel<<<(m + 127) / 128, 128, 0, st>>>(obj, m, max_iters, tol, state, prev, iterations, objectives);
    CSPQ_LAUNCH_CHECK();
    return CSPQ_OK;
}

int encode_subspace_major(const float *P, int64_t n, int m, int sub, const float *CB, const float *B, int k,
                          int32_t *assign, int variant, cudaStream_t st);

int lloyd_final_objective(const void *P, int pf64, int64_t n, int m, int sub, int k, const float *C32,
                          const int32_t *assign, double *obj, void *ws, cudaStream_t st) {
    WsLayout L(n, m, sub, k);
    double *r = L.at<double>(ws, L.resid);
    dim3 g((unsigned)grid_for(n, 256, 256), (unsigned)m);
    CSPQ_TP_DISPATCH(pf64, P, { final_resid_kernel<TP><<<g, 256, 0, st>>>(Pt, n, k, sub, C32, assign, r); });
    CSPQ_LAUNCH_CHECK();
    return pairwise_obj(r, n, 0, n, m, nullptr, ws, L, obj, st);
}

int lloyd_train(const void *P, int pf64, int64_t n, int m, int sub, int k, double *C64, int max_iters, double tol,
                float *C32, int32_t *assign, double *objectives, int32_t *iterations, void *ws, cudaStream_t st) {
    WsLayout L(n, m, sub, k);
    int32_t *state = L.at<int32_t>(ws, L.state);
    double *prev = L.at<double>(ws, L.prev);
    double *sq = L.at<double>(ws, L.sq);
    double *counts = L.at<double>(ws, L.counts);
    double *sums = L.at<double>(ws, L.sums);
    double *obj = L.at<double>(ws, L.obj);
    int32_t *empties = L.at<int32_t>(ws, L.empties);
    int32_t *nempty = L.at<int32_t>(ws, L.nempty);
    int32_t *asg = L.at<int32_t>(ws, L.assign_it);
    init_state_kernel<<<(m + 127) / 128, 128, 0, st>>>(m, state, prev, iterations);
    CSPQ_LAUNCH_CHECK();
    int rc;
    for (int it = 0; it < max_iters; ++it) {
        if ((rc = lloyd_assign(P, pf64, n, m, sub, k, C64, state, 0, n, asg, sq, ws, st))) return rc;
        if ((rc = lloyd_accumulate(P, pf64, n, m, sub, k, state, asg, sq, 0, n, counts, sums, obj, ws, st))) return rc;
        if ((rc = lloyd_update(counts, sums, m, k, sub, state, C64, empties, nempty, st))) return rc;
        if ((rc = lloyd_repair(P, pf64, n, m, sub, k, asg, state, empties, nempty, C64, ws, st))) return rc;
        if ((rc = lloyd_stop(obj, m, max_iters, tol, state, prev, iterations, objectives, st))) return rc;
    }
    const int64_t tot = (int64_t)m * k * sub;
    cast_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(C64, tot, C32);
    CSPQ_LAUNCH_CHECK();
    // final pass with the float32 REFERENCE encoder on float32(points) (training.py:143-150)
    const float *P32 = reinterpret_cast<const float *>(P);
    if (pf64) {
        float *p32 = L.at<float>(ws, L.p32);
        const int64_t np = (int64_t)m * n * sub;
        cast_points_kernel<double><<<(unsigned)((np + 255) / 256), 256, 0, st>>>(reinterpret_cast<const double *>(P), np, p32);
        CSPQ_LAUNCH_CHECK();
        P32 = p32;
    }
    if (tc_screen_ok(P32, m, sub, k)) {
        if ((rc = final_assign_tc(P32, n, m, sub, k, C32, assign, ws, L, st))) return rc;
    } else if ((rc = encode_subspace_major(P32, n, m, sub, C32, nullptr, k, assign, CSPQ_VARIANT_REFERENCE, st))) {
        return rc;
    }
    if ((rc = lloyd_final_objective(P, pf64, n, m, sub, k, C32, assign, obj, ws, st))) return rc;
    write_final_obj_kernel<<<(m + 127) / 128, 128, 0, st>>>(obj, m, max_iters, iterations, objectives);
    CSPQ_LAUNCH_CHECK();
    return CSPQ_OK;
}

// k-means++ seeding for every subspace (training.py:76-92).  first (m) and
// u (m, k-1) are the host RNG draws (rng.integers(n), then one rng.random()
// per rng.choice).  status[j] = -c if step c found zero total mass (the
// reference then draws rng.integers(n) for steps c..k-1 -- the host replays
// them), 3 if the total was NaN.
int kmeanspp(const void *P, int pf64, int64_t n, int m, int sub, int k, const int64_t *first, const double *u,
             double *C64, int32_t *status, void *ws, cudaStream_t st) {
    WsLayout L(n, m, sub, k);
    double *d2 = L.at<double>(ws, L.d2);
    double *pp = L.at<double>(ws, L.pp);
    double *total = L.at<double>(ws, L.obj);
    dim3 g((unsigned)grid_for(n, 256, 512), (unsigned)m);
    int rc;
    CSPQ_TP_DISPATCH(pf64, P, {
        kpp_first_kernel<TP><<<(m + 63) / 64, 64, 0, st>>>(Pt, n, m, sub, k, first, C64, status);
        CSPQ_LAUNCH_CHECK();
        kpp_dist_kernel<TP><<<g, 256, 0, st>>>(Pt, n, sub, C64, k, 0, status, d2, 1);
        CSPQ_LAUNCH_CHECK();
        for (int c = 1; c < k; ++c) {
            // status doubles as the "active" mask of pairwise_obj: 0 -> active
            if ((rc = pairwise_obj(d2, n, 0, n, m, nullptr, ws, L, total, st))) return rc;
            kpp_choose_kernel<<<m, 256, 0, st>>>(pp, d2, n, m, k, c, total, u, status, P, pf64, sub, C64);
            CSPQ_LAUNCH_CHECK();
            kpp_dist_kernel<TP><<<g, 256, 0, st>>>(Pt, n, sub, C64, k, c, status, d2, 0);
            CSPQ_LAUNCH_CHECK();
        }
    });
    return CSPQ_OK;
}

}  // namespace cspq
