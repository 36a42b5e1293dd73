// fileio.cu -- the data formats either side of the encode path.
//
//   * texmex vector files (fvecs: int32 d + d float32 per record; bvecs: int32 d
//     + d uint8), reference /root/reference/pkg/src/cspq/io.py:35-121: raw records
//     are copied to the GPU as they are and unpacked there into dense rows, which
//     also validates every record header and (fvecs) every value.  bvecs rows are
//     encoded as uint8 directly -- no float32 widening copy.
//   * the PQCD codes container (io.py:9-17, 213-219): header | codes | CRC-32 of
//     header and codes.  The CRC of each batch of codes is computed on the GPU
//     next to the codes and the per-batch CRCs are merged on the host, so codes
//     never need a second pass on the CPU.
//   * cspq_encode_vecs_file: the streaming file -> codes-file encoder: pread into
//     pinned buffers, H2D, unpack, encode (SIMT or tcgen05), CRC, D2H, pwrite,
//     several batches in flight on separate streams.
//
// CRC-32 is zlib's (reflected polynomial 0xEDB88320, init and final xor ~0).  It
// is linear over GF(2), so crc(A || B) = (x^(8|B|) mod P) * crc(A) xor crc(B): every
// thread checksums one piece and pieces merge up a tree.

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <climits>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace cspq {

int encode_device(const void *X, int in_dtype, int64_t n, int d, int64_t xrs, const float *CB, const float *B,
                  const float *guard, int m, int k, int sub, void *codes, int64_t crs, int variant, int mode,
                  cudaStream_t st);
int encode_tc(const void *X, int in_dtype, int64_t n, int64_t xrs, const float *CB, const float *B,
              const float *guard, const void *img, int m, int k, int sub, uint8_t *codes, int64_t crs, float *best,
              cudaStream_t st);
int encode_prepare(const float *CB, const float *B, int m, int k, int sub, float *guard, cudaStream_t st);

namespace {

constexpr uint32_t kPoly = 0xEDB88320u;
constexpr int kPiece = 1024;                    // bytes per thread
constexpr int kCrcThreads = 256;
constexpr int64_t kBlockBytes = (int64_t)kPiece * kCrcThreads;
constexpr int kMergeThreads = 1024;
__host__ __device__ inline int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

// a(x) * b(x) mod P in the reflected representation (bit 31 = x^0); a != 0
__host__ __device__ inline uint32_t gf_mul(uint32_t a, uint32_t b) {
    uint32_t prod = 0;
    for (uint32_t bit = 1u << 31; bit; bit >>= 1) {
        if (a & bit) prod ^= b;
        b = (b & 1) ? (b >> 1) ^ kPoly : b >> 1;  // b *= x
    }
    return prod;
}

struct X2n {  // x^(2^i) mod P, i = 0..63
    uint32_t t[64];
};
__host__ __device__ inline void x2n_fill(X2n &x) {
    x.t[0] = 1u << 30;  // x^1
    for (int i = 1; i < 64; ++i) x.t[i] = gf_mul(x.t[i - 1], x.t[i - 1]);
}
// x^(8 len) mod P
__host__ __device__ inline uint32_t x8n(const X2n &x, int64_t len) {
    uint32_t p = 1u << 31;  // x^0
    uint64_t e = (uint64_t)len;
    for (int i = 3; e; e >>= 1, ++i)
        if (e & 1) p = gf_mul(x.t[i], p);
    return p;
}
__host__ __device__ inline uint32_t crc_merge(const X2n &x, uint32_t crc_a, uint32_t crc_b, int64_t len_b) {
    return len_b == 0 ? crc_a : gf_mul(x8n(x, len_b), crc_a) ^ crc_b;
}

// Pass 1: CRC of each kBlockBytes block (slicing-by-8 tables in shared memory).
__global__ void __launch_bounds__(kCrcThreads) crc_blocks_kernel(const uint8_t *__restrict__ data, int64_t n,
                                                                 uint32_t *__restrict__ block_crc) {
    __shared__ uint32_t T[8][256];
    __shared__ X2n X;
    __shared__ uint32_t part[kCrcThreads];
    const int t = threadIdx.x;
    {
        uint32_t c = t;
        for (int i = 0; i < 8; ++i) c = (c & 1) ? (c >> 1) ^ kPoly : c >> 1;
        T[0][t] = c;
    }
    if (t == 0) x2n_fill(X);
    __syncthreads();
    for (int s = 1; s < 8; ++s) {
        T[s][t] = (T[s - 1][t] >> 8) ^ T[0][T[s - 1][t] & 0xff];
        __syncthreads();
    }
    const int64_t b0 = (int64_t)blockIdx.x * kBlockBytes;
    const int64_t p0 = b0 + (int64_t)t * kPiece;
    const int64_t len = p0 >= n ? 0 : (n - p0 < kPiece ? n - p0 : kPiece);
    uint32_t c = 0xffffffffu;
    const uint8_t *p = data + p0;
    int64_t i = 0;
    if ((reinterpret_cast<uintptr_t>(p) & 7) == 0) {
        for (; i + 8 <= len; i += 8) {
            const uint2 w = *reinterpret_cast<const uint2 *>(p + i);
            const uint32_t lo = w.x ^ c, hi = w.y;
            c = T[7][lo & 0xff] ^ T[6][(lo >> 8) & 0xff] ^ T[5][(lo >> 16) & 0xff] ^ T[4][lo >> 24] ^
                T[3][hi & 0xff] ^ T[2][(hi >> 8) & 0xff] ^ T[1][(hi >> 16) & 0xff] ^ T[0][hi >> 24];
        }
    }
    for (; i < len; ++i) c = (c >> 8) ^ T[0][(c ^ p[i]) & 0xff];
    part[t] = ~c;
    __syncthreads();
    // merge pieces pairwise: after the level with stride s, part[t] (t % 2s == 0)
    // covers pieces t .. t + 2s - 1
    for (int s = 1; s < kCrcThreads; s <<= 1) {
        if ((t & (2 * s - 1)) == 0) {
            const int64_t rb = b0 + (int64_t)(t + s) * kPiece;  // right run start
            const int64_t rl = rb >= n ? 0 : min64(n - rb, (int64_t)s * kPiece);
            part[t] = crc_merge(X, part[t], part[t + s], rl);
        }
        __syncthreads();
    }
    if (t == 0) block_crc[blockIdx.x] = part[0];
}

// Pass 2: merge the block CRCs in order (one CTA), then continue crc_in.
__global__ void __launch_bounds__(kMergeThreads) crc_merge_kernel(const uint32_t *__restrict__ block_crc,
                                                                  int64_t nblocks, int64_t n, uint32_t crc_in,
                                                                  uint32_t *__restrict__ out) {
    __shared__ X2n X;
    __shared__ uint32_t part[kMergeThreads];
    __shared__ int64_t plen[kMergeThreads];
    const int t = threadIdx.x;
    if (t == 0) x2n_fill(X);
    __syncthreads();
    const int64_t per = (nblocks + kMergeThreads - 1) / kMergeThreads;
    const int64_t lo = min64(nblocks, t * per), hi = min64(nblocks, lo + per);
    uint32_t c = 0;
    int64_t covered = 0;
    for (int64_t b = lo; b < hi; ++b) {
        const int64_t bl = min64(kBlockBytes, n - b * kBlockBytes);
        c = covered ? crc_merge(X, c, block_crc[b], bl) : block_crc[b];
        covered += bl;
    }
    part[t] = c;
    plen[t] = covered;
    __syncthreads();
    for (int s = 1; s < kMergeThreads; s <<= 1) {
        if ((t & (2 * s - 1)) == 0) {
            if (plen[t + s]) part[t] = plen[t] ? crc_merge(X, part[t], part[t + s], plen[t + s]) : part[t + s];
            plen[t] += plen[t + s];
        }
        __syncthreads();
    }
    if (t == 0) *out = crc_merge(X, crc_in, part[0], n);
}

// texmex records -> dense rows.  One CTA per group of records; bad[0] = file offset of
// the first record header != d, bad[1] = file offset of the first non-finite value.
template <typename V>
__global__ void unpack_kernel(const uint8_t *__restrict__ rec, int64_t n, int d, int check_finite, int64_t off0,
                              V *__restrict__ rows, unsigned long long *__restrict__ bad) {
    const int64_t rb = 4 + (int64_t)d * sizeof(V);
    for (int64_t r = blockIdx.x; r < n; r += gridDim.x) {
        const uint8_t *src = rec + r * rb;
        if (threadIdx.x == 0) {
            int32_t h;
            memcpy(&h, src, 4);
            if (h != d) atomicMin(&bad[0], (unsigned long long)(off0 + r * rb));
        }
        V *dst = rows + r * d;
        for (int i = threadIdx.x; i < d; i += blockDim.x) {
            V v;
            memcpy(&v, src + 4 + (int64_t)i * sizeof(V), sizeof(V));
            if constexpr (sizeof(V) == 4) {
                if (check_finite && !isfinite(v)) atomicMin(&bad[1], (unsigned long long)(off0 + r * rb + 4 + 4 * (int64_t)i));
            }
            dst[i] = v;
        }
    }
}

int crc32_device(const void *data, int64_t n, uint32_t crc_in, uint32_t *crc_out, void *ws, cudaStream_t st) {
    const int64_t nb = (n + kBlockBytes - 1) / kBlockBytes;
    uint32_t *blk = reinterpret_cast<uint32_t *>(ws);
    if (nb > 0) {
        CSPQ_REQUIRE(nb <= INT_MAX, CSPQ_E_CONFIG, "CRC input too large");
        crc_blocks_kernel<<<(unsigned)nb, kCrcThreads, 0, st>>>(reinterpret_cast<const uint8_t *>(data), n, blk);
        CSPQ_LAUNCH_CHECK();
    }
    crc_merge_kernel<<<1, kMergeThreads, 0, st>>>(blk, nb, n, crc_in, crc_out);
    CSPQ_LAUNCH_CHECK();
    return CSPQ_OK;
}

const X2n &host_x2n() {
    static X2n x = [] {
        X2n v;
        x2n_fill(v);
        return v;
    }();
    return x;
}

uint32_t crc32_host(uint32_t crc, const uint8_t *p, size_t len) {  // bytewise, for small headers
    static uint32_t T[256];
    static std::once_flag once;
    std::call_once(once, [] {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ kPoly : c >> 1;
            T[i] = c;
        }
    });
    crc = ~crc;
    for (size_t i = 0; i < len; ++i) crc = (crc >> 8) ^ T[(crc ^ p[i]) & 0xff];
    return ~crc;
}

bool pread_all(int fd, void *buf, size_t len, off_t off) {
    char *p = reinterpret_cast<char *>(buf);
    while (len) {
        const ssize_t r = pread(fd, p, len, off);
        if (r <= 0) return false;
        p += r; len -= (size_t)r; off += r;
    }
    return true;
}
bool pwrite_all(int fd, const void *buf, size_t len, off_t off) {
    const char *p = reinterpret_cast<const char *>(buf);
    while (len) {
        const ssize_t r = pwrite(fd, p, len, off);
        if (r <= 0) return false;
        p += r; len -= (size_t)r; off += r;
    }
    return true;
}

struct Fd {
    int fd = -1;
    ~Fd() { if (fd >= 0) close(fd); }
};

// one in-flight batch of the file encoder
struct Slot {
    cudaStream_t st = nullptr;
    cudaEvent_t done = nullptr;
    void *h_rec = nullptr, *h_codes = nullptr, *d_rec = nullptr, *d_rows = nullptr, *d_codes = nullptr, *d_ws = nullptr;
    uint32_t *h_crc = nullptr;
    int64_t batch = -1, r0 = 0, rows = 0;
};

}  // namespace

size_t crc32_workspace_bytes(int64_t n) {
    return (size_t)std::max<int64_t>(1, (n + kBlockBytes - 1) / kBlockBytes) * sizeof(uint32_t);
}
int crc32_device_api(const void *data, int64_t n, uint32_t crc_in, uint32_t *crc_out, void *ws, cudaStream_t st) {
    return crc32_device(data, n, crc_in, crc_out, ws, st);
}
uint32_t crc32_combine_host(uint32_t crc1, uint32_t crc2, int64_t len2) { return crc_merge(host_x2n(), crc1, crc2, len2); }

int unpack_vecs(const void *records, int64_t n, int d, int value_bytes, int check_finite, int64_t off0, void *rows,
                unsigned long long *bad, cudaStream_t st) {
    if (n == 0) return CSPQ_OK;
    const int grid = (int)std::min<int64_t>(n, 148 * 16);
    const int threads = d >= 256 ? 256 : (d >= 64 ? 64 : 32);
    if (value_bytes == 4)
        unpack_kernel<float><<<grid, threads, 0, st>>>(reinterpret_cast<const uint8_t *>(records), n, d, check_finite,
                                                      off0, reinterpret_cast<float *>(rows), bad);
    else
        unpack_kernel<uint8_t><<<grid, threads, 0, st>>>(reinterpret_cast<const uint8_t *>(records), n, d, 0, off0,
                                                        reinterpret_cast<uint8_t *>(rows), bad);
    CSPQ_LAUNCH_CHECK();
    return CSPQ_OK;
}

// Streaming fvecs/bvecs -> PQCD encoder.  On a format problem returns CSPQ_E_FORMAT
// with err[0] = kind (1 empty, 2 truncated header, 3 non-positive d, 4 inconsistent d,
// 5 truncated body, 6 non-finite value), err[1] = byte offset, err[2] = the offending
// record length (kinds 3/4); the output file is removed.
int encode_vecs_file(const char *in_path, int fmt, const char *out_path, const float *CB, const float *B,
                     const float *guard, const void *tc_img, int m, int k, int sub, int variant, int mode,
                     int64_t batch_rows, int n_streams, int device, int64_t *n_out, int64_t *err) {
    err[0] = err[1] = err[2] = 0;
    CSPQ_CUDA_TRY(cudaSetDevice(device));
    const int vb = fmt == 0 ? 4 : 1;
    const int in_dtype = fmt == 0 ? CSPQ_IN_F32 : CSPQ_IN_U8;
    Fd in;
    in.fd = open(in_path, O_RDONLY);
    CSPQ_REQUIRE(in.fd >= 0, CSPQ_E_CONFIG, "cannot open %s", in_path);
    struct stat sb;
    CSPQ_REQUIRE(fstat(in.fd, &sb) == 0, CSPQ_E_CONFIG, "cannot stat %s", in_path);
    const int64_t size = sb.st_size;
    auto fail = [&](int64_t kind, int64_t off, int64_t val) {
        err[0] = kind; err[1] = off; err[2] = val;
        set_error("format error in %s (kind %lld at byte %lld)", in_path, (long long)kind, (long long)off);
        return CSPQ_E_FORMAT;
    };
    if (size == 0) return fail(1, 0, 0);
    if (size < 4) return fail(2, 0, 0);
    int32_t d = 0;
    CSPQ_REQUIRE(pread_all(in.fd, &d, 4, 0), CSPQ_E_CONFIG, "read error on %s", in_path);
    if (d <= 0) return fail(3, 0, d);
    const int64_t rb = 4 + (int64_t)d * vb;
    const int64_t n = size / rb, tail = size - n * rb;
    CSPQ_REQUIRE(d == m * sub, CSPQ_E_CONFIG, "dataset dimensionality %d does not match codebooks' d=%d", d, m * sub);
    const int cw = k <= 256 ? 1 : 2;
    const int64_t crow = (int64_t)m * cw;

    Fd out;
    out.fd = open(out_path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
    CSPQ_REQUIRE(out.fd >= 0, CSPQ_E_CONFIG, "cannot create %s", out_path);
    // PQCD header: magic | version u32 | n u64 | m u32 | k u32 | width u32 (io.py:213-219)
    uint8_t hdr[28];
    memcpy(hdr, "PQCD", 4);
    const uint32_t ver = 1, um = (uint32_t)m, uk = (uint32_t)k, uw = (uint32_t)cw;
    const uint64_t un = (uint64_t)n;
    memcpy(hdr + 4, &ver, 4); memcpy(hdr + 8, &un, 8); memcpy(hdr + 16, &um, 4); memcpy(hdr + 20, &uk, 4);
    memcpy(hdr + 24, &uw, 4);
    uint32_t crc = crc32_host(0, hdr + 4, 24);

    const bool tc = tc_img && variant != CSPQ_VARIANT_REFERENCE && k == 256 && (sub == 4 || sub == 8) &&
                    (in_dtype == CSPQ_IN_U8 || (d * 4) % 16 == 0);
    float *tmp_guard = nullptr;
    std::vector<Slot> S(std::max(1, std::min(n_streams, 8)));
    unsigned long long *d_bad = nullptr;
    int rc = CSPQ_OK;
    auto cleanup = [&]() {
        for (auto &s : S) {
            if (s.st) cudaStreamSynchronize(s.st);
            if (s.st) cudaStreamDestroy(s.st);
            if (s.done) cudaEventDestroy(s.done);
            if (s.h_rec) cudaFreeHost(s.h_rec);
            if (s.h_codes) cudaFreeHost(s.h_codes);
            if (s.h_crc) cudaFreeHost(s.h_crc);
            cudaFree(s.d_rec); cudaFree(s.d_rows); cudaFree(s.d_codes); cudaFree(s.d_ws);
        }
        if (d_bad) cudaFree(d_bad);
        if (tmp_guard) cudaFree(tmp_guard);
    };
    const int64_t br = std::max<int64_t>(1, std::min<int64_t>(batch_rows, std::max<int64_t>(n, 1)));
    unsigned long long bad[2] = {~0ull, ~0ull};
    auto run = [&]() -> int {
    for (auto &s : S) {
        CSPQ_CUDA_TRY(cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking));
        CSPQ_CUDA_TRY(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
        CSPQ_CUDA_TRY(cudaHostAlloc(&s.h_rec, br * rb, cudaHostAllocDefault));
        CSPQ_CUDA_TRY(cudaHostAlloc(&s.h_codes, br * crow, cudaHostAllocDefault));
        CSPQ_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void **>(&s.h_crc), 4, cudaHostAllocDefault));
        CSPQ_CUDA_TRY(cudaMalloc(&s.d_rec, br * rb));
        CSPQ_CUDA_TRY(cudaMalloc(&s.d_rows, br * (int64_t)d * vb));
        CSPQ_CUDA_TRY(cudaMalloc(&s.d_codes, br * crow + 8));  // + the batch CRC at the next 4-aligned offset
        CSPQ_CUDA_TRY(cudaMalloc(&s.d_ws, crc32_workspace_bytes(br * crow)));
    }
    CSPQ_CUDA_TRY(cudaMalloc(reinterpret_cast<void **>(&d_bad), 2 * sizeof(unsigned long long)));
    CSPQ_CUDA_TRY(cudaMemset(d_bad, 0xff, 2 * sizeof(unsigned long long)));
    const bool needs_guard = variant != CSPQ_VARIANT_REFERENCE && mode != CSPQ_MODE_EXACT;
    if (needs_guard && !guard) {
        CSPQ_CUDA_TRY(cudaMalloc(reinterpret_cast<void **>(&tmp_guard), sizeof(float) * 2 * m));
        if ((rc = encode_prepare(CB, B, m, k, sub, tmp_guard, S[0].st))) return rc;
        CSPQ_CUDA_TRY(cudaStreamSynchronize(S[0].st));
        guard = tmp_guard;
    }
    const int64_t nb = (n + br - 1) / br;
    auto retire = [&](Slot &s) -> int {
        if (s.batch < 0) return CSPQ_OK;
        CSPQ_CUDA_TRY(cudaEventSynchronize(s.done));
        if (!pwrite_all(out.fd, s.h_codes, s.rows * crow, 28 + s.r0 * crow)) {
            set_error("write error on %s", out_path);
            return CSPQ_E_CONFIG;
        }
        crc = crc32_combine_host(crc, *s.h_crc, s.rows * crow);  // batches retire in file order
        s.batch = -1;
        return CSPQ_OK;
    };
    for (int64_t b = 0; b < nb && rc == CSPQ_OK; ++b) {
        Slot &s = S[b % S.size()];
        if ((rc = retire(s))) break;
        s.batch = b; s.r0 = b * br; s.rows = std::min<int64_t>(br, n - s.r0);
        if (!pread_all(in.fd, s.h_rec, s.rows * rb, s.r0 * rb)) { set_error("read error on %s", in_path); rc = CSPQ_E_CONFIG; break; }
        CSPQ_CUDA_TRY(cudaMemcpyAsync(s.d_rec, s.h_rec, s.rows * rb, cudaMemcpyHostToDevice, s.st));
        if ((rc = unpack_vecs(s.d_rec, s.rows, d, vb, fmt == 0, s.r0 * rb, s.d_rows, d_bad, s.st))) break;
        if (tc)
            rc = encode_tc(s.d_rows, in_dtype, s.rows, d, CB, B, guard, tc_img, m, k, sub,
                           reinterpret_cast<uint8_t *>(s.d_codes), m, nullptr, s.st);
        else
            rc = encode_device(s.d_rows, in_dtype, s.rows, d, d, CB, B, guard, m, k, sub, s.d_codes, m, variant, mode, s.st);
        if (rc) break;
        uint32_t *d_crc = reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(s.d_codes) + ((br * crow + 3) & ~3ll));
        if ((rc = crc32_device(s.d_codes, s.rows * crow, 0, d_crc, s.d_ws, s.st))) break;
        CSPQ_CUDA_TRY(cudaMemcpyAsync(s.h_codes, s.d_codes, s.rows * crow, cudaMemcpyDeviceToHost, s.st));
        CSPQ_CUDA_TRY(cudaMemcpyAsync(s.h_crc, d_crc, 4, cudaMemcpyDeviceToHost, s.st));
        CSPQ_CUDA_TRY(cudaEventRecord(s.done, s.st));
    }
    // drain in order
    for (int64_t b = std::max<int64_t>(0, nb - (int64_t)S.size()); b < nb && rc == CSPQ_OK; ++b)
        rc = retire(S[b % S.size()]);
    if (rc == CSPQ_OK) CSPQ_CUDA_TRY(cudaMemcpy(bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost));
    return rc;
    };
    rc = run();  // every CUDA failure inside returns here, so the resources are always released
    cleanup();
    if (rc) { unlink(out_path); return rc; }
    // the reference walks records in order (io.py:35-62): a bad header or a truncated
    // tail is reported before any value check (io.py:70-77)
    if (bad[0] != ~0ull) {
        int32_t v = 0;
        pread_all(in.fd, &v, 4, (off_t)bad[0]);
        unlink(out_path);
        return fail(v <= 0 ? 3 : 4, (int64_t)bad[0], v);
    }
    if (tail) {
        const int64_t off = n * rb;
        int32_t v = 0;
        unlink(out_path);
        if (tail < 4) return fail(2, off, 0);
        pread_all(in.fd, &v, 4, off);
        if (v <= 0) return fail(3, off, v);
        if (v != d) return fail(4, off, v);
        return fail(5, off + 4, v);
    }
    if (bad[1] != ~0ull) {
        unlink(out_path);
        return fail(6, (int64_t)bad[1], 0);
    }
    if (!pwrite_all(out.fd, hdr, 28, 0) || !pwrite_all(out.fd, &crc, 4, 28 + n * crow)) {
        unlink(out_path);
        set_error("write error on %s", out_path);
        return CSPQ_E_CONFIG;
    }
    *n_out = n;
    return CSPQ_OK;
}

}  // namespace cspq
