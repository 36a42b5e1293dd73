// encode_tc.cu -- PQ encode on the 5th-generation tensor cores (tcgen05, sm_100a).
//
// Same contract as encode.cu (the oracle's codes bit for bit; reference:
// /root/reference/pkg/src/cspq/kernels.py:108-316), different engine:
//
//   scores  S = A . B^T  on tcgen05.mma.kind::f16 (fp16 hi/lo split, fp32 accumulation, bias folded):
//     A row (one x subvector)  = [ xh | xh | xl | 1 1 0.. ]           (fp16)
//     B row (one centroid)     = [-ch |-cl |-ch | bh bl 0.. ]          (fp16)
//     => S[i][l] = bh + bl - (xh.ch + xh.cl + xl.ch) ~= s^2 (b_l - x_i.c_l)
//     of the scaled operands x' = s x, c' = s c, b' = s^2 b: s is the subspace's power of two that
//     puts the largest centroid norm in [32, 64) (tc_image_kernel), so every part sits inside the
//     fp16 range; x' = xh + xl, c' = ch + cl, b' = bh + bl with round-to-nearest fp16 parts
//     (22 significant bits, as the 3xTF32 split this replaced).  For uint8 rows xl = 0.
//     K = 32 (d_sub 8) is two K = 16 MMAs per item, K = 16 (d_sub 4) one -- half the tensor work of
//     the tf32 form.  c3 runs into the 1,000 W power cap: with half the MMAs the SM clock under the
//     cap rises from ~1,690 to ~1,880 MHz (bench c3 +13 % together with the shorter MMA chain).
//   accumulators in TMEM (128 lanes = rows x 256 columns = centroids), two
//   buffers so the MMA of tile t+1 overlaps the epilogue of tile t;
//   epilogue warps read their rows with tcgen05.ld (64 columns per load) and
//   run an argmin that also finds the runner-up exactly without re-reading
//   anything: every 16 centroids form a block of 7 and a block of 9 (three-
//   input minima with no idle operand: 3 + 4 FMNMX3), 32 block minima in all;
//   nine "class" minima (position inside the block) catch a runner-up that
//   shares the winner's block, because a block and a class intersect in at
//   most one centroid.  Block slot s starts at centroid 8s - (s & 1); the
//   code is that start + class.  The 32 block minima are folded, chunk by chunk, into 8
//   "super-block" and 4 "super-class" minima (the same two-partition argument one level up), so the
//   selection looks at 9 + 8 + 4 = 21 candidates.
//   A (row, subspace) whose runner-up lies within the error band of the
//   tensor-core score is re-encoded exactly by its warp (strict fp32 chains,
//   warp-shuffle argmin) -- the same fix-up as the SIMT kernel.
//
//   Error band (per score, in the scaled units, |S_tc - s^2 s_oracle| <= E W + absolute terms):
//     fp16 splitting of x', c', b': 4 * 2^-22 (|b'| + sum|x'_t c'_t|)  (three parts of 2^-22 and
//                                  the dropped xl.cl)
//     tensor-core accumulation:    2^-22 per 8 products (products of fp16 operands are exact in
//                                  fp32; 8 products + the running sum are modelled as <= 2
//                                  roundings of 2^-23 of the running magnitude) -> 4 * 2^-22 for
//                                  K = 32
//     the oracle's own rounding:   (sub+1) 2^-24 (|b| + sum|x_t c_t|)
//     absolute terms:              2^-25 per element of x', c' and the bias whose fp16 parts fall
//                                  below the normal range, and 2^-150 s^2 per operation of the
//                                  oracle's chain when its float32 terms are subnormal
//   The accumulation term is a model of undocumented hardware; measured
//   errors (scripts/tc_error.py, tests/test_encode_tc_gpu.py) stay >= 7x
//   below the resulting E on every data regime tried (max 2.8e-7 W vs E = 2.2e-6 W).
//   with sum|x_t c_t| <= ||x|| max_l ||c_l||; a runner-up within 4E (x2
//   safety) of the best is flagged.  Rows beyond the fp16 range of their subspace (|x_t| more than
//   ~1000 x the largest centroid norm) give NaN scores and are flagged; rows whose oracle chain can
//   overflow float32 (W / s^2 >= 2^127) are flagged too -- the scaled scores have more range.
//
// Warp roles (128 + 128 kGroups threads, one CTA per SM, persistent over a contiguous range of
// (row group, subspace) pairs).  The kernel is bound by issue slots: on this SM a half-rate
// ALU-pipe instruction (FMNMX3: 276 of ~600 instructions per warp-item; ~710 before the per-thread
// addresses were made loop constants, see opaque32) holds a sub-partition's issue port for two cycles
// (scripts/micro/issue_mix.cu), so time ~ 2 x ALU + other instructions.  More warps do not help:
// four epilogue groups (-DCSPQ_TC_GROUPS=4) run 2-4 % slower.
//   warps 0-3   one warpgroup that hands its registers to the others (setmaxnreg 40 / 152):
//     warp 0    TMEM allocation + MMA issue (the warp walks the items, one elected lane issues);
//               waits for A rows and drained accumulators on named barriers (bar.sync: no retries)
//     warp 1    bulk copies of the prepared codebook image + fp32 codebook (cp.async.bulk)
//     warps 2-3 idle
//   warps 4..   kGroups epilogue groups of 4 warps (TMEM lane quadrant = warp % 4); item it
//               belongs to group it % kGroups and TMEM buffer it & 1.  A group writes the A rows of
//               its next item (x prefetched with cp.async, scaled, fp16 split) into its other A
//               stage, drains its item's accumulator (block, class, super-block and super-class
//               minima, all in registers), selects the winner with binary band indicators summed
//               into one exact integer accumulator (runner-up within the error band => flag),
//               applies the exact fix-up (or, in mark mode, flags the pair for the caller), stores
//               codes.

#include <atomic>
#include <cstdlib>

#include "common.cuh"

namespace cspq {

__device__ unsigned long long g_tc_flagged = 0;  // telemetry (cspq_encode_stats)

namespace {

constexpr int kTM = 128;     // rows per tile (MMA M)
constexpr int kN = 256;      // centroids (MMA N)
constexpr int kNCls = 9;     // argmin classes = position inside a block of 7 or 9 centroids
constexpr int kG = 16;       // max tiles per row group (codebook image reuse); the launch picks 1..kG
#ifndef CSPQ_TC_GROUPS
#define CSPQ_TC_GROUPS 3
#endif
constexpr int kGroups = CSPQ_TC_GROUPS;   // epilogue groups: item it belongs to group it % kGroups
constexpr int kLdCols = kGroups >= 4 ? 32 : 64;  // accumulator columns per tcgen05.ld (4 groups: 112 registers each)
constexpr int kNA = 2 * kGroups;  // A-operand stages: a group alternates between two, so it writes the A rows of
                                  // its next item (it + kGroups) before it waits for item it's accumulator --
                                  // with one stage per group the next item's MMA could only start after the
                                  // current item's scan (the chain scan -> A rows -> MMA -> scan bounded a group)
constexpr int kThreads = 128 + 128 * kGroups;  // warpgroup 0 = MMA warp, loader warp, two idle warps; then
                                               // kGroups epilogue warpgroups.  Warpgroup 0 hands its
                                               // registers to the epilogue (setmaxnreg kRegsLight / kRegsEpi)
// setmaxnreg moves registers inside the CTA's launch allocation (threads x the launch register count:
// 512 x 128, or 640 x 96 with four groups), never beyond it
constexpr int kRegsLight = 40, kRegsEpi = kGroups >= 4 ? 104 : 152;  // 128 x 40 + 384 x 152 = 63,488 <= 65,536
constexpr int kRegsLaunch = (65536 / kThreads) / 8 * 8;
static_assert(128 * kRegsLight + 128 * kGroups * kRegsEpi <= kThreads * kRegsLaunch, "register pool");
// (Accumulator chunks -- N = 128 or 64 per MMA with per-chunk commits and barriers, so MMA and scan
// overlap chunk by chunk -- were measured three times and never paid: c3 -4..-5 % with 2 chunks; an
// N = 128 MMA costs what an N = 256 one does.)
// The MMA warp waits on named barriers (bar.sync / bar.arrive, 160 = a group's 128 threads + the
// MMA warp): a warp blocked in bar.sync issues nothing, whereas a suspended mbarrier wait returns
// on every barrier operation of the CTA (~10 retries of ~11 instructions per wait, ncu source
// counters) -- and the MMA warp shares its sub-partition with three epilogue warps, which makes
// that sub-partition the slowest of the four.  The MMA completions (tcgen05.commit) and the bulk
// copies need mbarriers; the epilogue warps keep waiting on those one by one (releasing a whole
// group through a named barrier put its four warps in lockstep: -3 %).
constexpr int kBarTEmpty = 1;   // + TMEM buffer
constexpr int kBarAFull = 3;    // + A stage (6)
constexpr int kBarThreads = 160;
constexpr int kPD = 2;        // cp.async prefetch distance, in the group's own items
constexpr int kRing = 3;      // x slots per group (> kPD: an item's slot outlives its fix-up)

// error constant E of the tensor scores: |S - s_oracle| <= E W, W = max|b| + ||x|| max||c||
// (fp16 hi/lo split, 2 roundings per 8 products, the oracle's own chain; 1 % slack).  Lloyd's final
// REFERENCE screen widens the same band (lloyd.cu, final_guard_kernel)
__host__ __device__ constexpr float tc_error_constant(int sub) {
    return (float)((4.0 / 4194304.0 + (sub == 8 ? 4 : 2) / 4194304.0 * (1.0 + 1.0 / 1024.0) + (sub + 1) / 16777216.0) * 1.01);
}

template <int SUB>
struct TcShape {
    static constexpr int K = SUB == 8 ? 32 : 16;    // fp16 elements per operand row
    static constexpr int kChunks = K / 8;           // 16-byte chunks (8 fp16) per row
    static constexpr int kSteps = K / 16;           // MMAs (kind::f16, K = 16 each)
    static constexpr int kRowGroupBytes = kChunks * 128;  // 8 rows x all chunks
    static constexpr int kABytes = kTM * K * 2;
    static constexpr int kBBytes = kN * K * 2;
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
                 "r"(bytes) : "memory");
}
// bounded wait: a lost arrival traps (error) instead of hanging the device
constexpr uint32_t kSuspendNs = 1000000;
__device__ __noinline__ long long mbar_wait_check(long long t0) {
    // every 256th unsuccessful try: ~10 s of clock without the phase flip is a lost arrival (not a
    // time slice)
    const long long t = clock64();
    if (t0 == 0) return t;
    if (t - t0 > 20000000000ll) __trap();
    return t0;
}
// sleep between retries of the epilogue's accumulator wait: fewer polls (c3 executes ~19 retries of 11
// instructions per item).  0 / 100 / 200 ns over five alternations: c3 3.540e8 / 3.589e8 / 3.577e8 vec/s,
// c2 and c5 (not power-capped) unchanged, c4 never waits
#ifndef CSPQ_TC_WAIT_SLEEP
#define CSPQ_TC_WAIT_SLEEP 100
#endif
template <int kSleepNs = 0>
__device__ __forceinline__ void mbar_wait_s(uint32_t addr, uint32_t parity) {  // addr: shared address of the mbarrier
    // suspend (woken by the phase flip) instead of busy polling: spinning warps steal issue slots
    // from the epilogue warps that share their SM sub-partition.  A suspended try_wait also
    // returns on other barrier traffic of the CTA (~5 times per wait, ncu source counters), so the
    // retry path is kept to the try itself plus a counter: the clock is read every 256th retry.
    // (Four tries and a branch each inside one asm block -- 4 instead of 11 instructions per retry --
    // ran 2 % SLOWER on c3 and c4: the shorter loop simply polls more often; the wait is time, not
    // instructions.)
    uint32_t spins = 0;
    long long t0 = 0;
    for (;;) {
        uint32_t done;
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"(addr), "r"(parity), "r"(kSuspendNs) : "memory");
        if (done) return;
        if constexpr (kSleepNs > 0) asm volatile("nanosleep.u32 %0;" ::"n"(kSleepNs));
        if ((++spins & 255u) == 0) t0 = mbar_wait_check(t0);
    }
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) { mbar_wait_s(smem_u32(bar), parity); }
__device__ __forceinline__ void bar_sync(int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(kBarThreads) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "n"(kBarThreads) : "memory"); }
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    // K-major, no swizzle: core matrices of 8 rows x 16 B; LBO = between the
    // two 16-B K-chunks of one MMA, SBO = between 8-row groups; version 1.
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

__host__ __device__ constexpr uint32_t make_idesc(int n = kN) {
    // kind::f16: D f32 (bit 4), A f16 (0 << 7), B f16 (0 << 10), K-major A/B,
    // N >> 3 at [17, 23), M >> 4 at [24, 29)
    return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kTM >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
                 "l"(da), "l"(db), "r"(make_idesc(kN)), "r"(accumulate) : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

#define CSPQ_LD8(o) "=r"(v[o + 0]), "=r"(v[o + 1]), "=r"(v[o + 2]), "=r"(v[o + 3]), "=r"(v[o + 4]), "=r"(v[o + 5]), "=r"(v[o + 6]), "=r"(v[o + 7])
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, uint32_t *v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,"
        "%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,"
        "%57,%58,%59,%60,%61,%62,%63}, [%64];\n\t"
        "tcgen05.wait::ld.sync.aligned;"  // same statement: no use of v can be scheduled before the wait
        : CSPQ_LD8(0), CSPQ_LD8(8), CSPQ_LD8(16), CSPQ_LD8(24), CSPQ_LD8(32), CSPQ_LD8(40), CSPQ_LD8(48), CSPQ_LD8(56)
        : "r"(taddr) : "memory");
}
[[maybe_unused]] __device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t *v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,"
        "%29,%30,%31}, [%32];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : CSPQ_LD8(0), CSPQ_LD8(8), CSPQ_LD8(16), CSPQ_LD8(24)
        : "r"(taddr) : "memory");
}
#undef CSPQ_LD8

// two floats -> packed fp16 (round to nearest even; beyond the fp16 range -> inf, which makes the
// scores NaN and the row flagged); lo is the element at the lower address
__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ float f16_lo(uint32_t v) {
    float f;
    asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %1;\n\tcvt.f32.f16 %0, l;\n\t}" : "=f"(f) : "r"(v));
    return f;
}
__device__ __forceinline__ float f16_hi(uint32_t v) {
    float f;
    asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %1;\n\tcvt.f32.f16 %0, h;\n\t}" : "=f"(f) : "r"(v));
    return f;
}

// a - (one fp16 half of v) in one mixed-precision add (SASS FHADD; exact: the half is a's own
// rounding, so the difference has <= 13 significant bits) instead of a conversion and a subtraction
__device__ __forceinline__ float f16_resid_lo(uint32_t v, float a) {
    float d;
    asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %1;\n\tneg.f16 l, l;\n\tadd.rn.f32.f16 %0, l, %2;\n\t}" : "=f"(d) : "r"(v), "f"(a));
    return d;
}
__device__ __forceinline__ float f16_resid_hi(uint32_t v, float a) {
    float d;
    asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %1;\n\tneg.f16 h, h;\n\tadd.rn.f32.f16 %0, h, %2;\n\t}" : "=f"(d) : "r"(v), "f"(a));
    return d;
}

// Shared-memory accesses of the epilogue's hot loop by 32-bit shared address: every per-thread
// address is computed once, made opaque (opaque32: ptxas otherwise re-derives such values from
// %tid and the shared window base at every use -- ~80 of ~680 instructions per warp-item) and kept
// in a register.
__device__ __forceinline__ uint32_t opaque32(uint32_t v) { return __shfl_sync(0xffffffffu, v, threadIdx.x & 31); }
__device__ __forceinline__ uint64_t opaque64(uint64_t v) {
    return ((uint64_t)opaque32((uint32_t)(v >> 32)) << 32) | opaque32((uint32_t)v);
}
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ float lds_f(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint2 lds_u2(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_u(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_u4(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
// cp.async of BYTES (4, 8, 16) with the ignore-src predicate: !ok writes zeros and reads nothing
template <int BYTES>
__device__ __forceinline__ void cp_async_pred(uint32_t dst, const void *src, bool ok) {
    if constexpr (BYTES == 16)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %2, 0;\n\tcp.async.cg.shared.global [%0], [%1], 16, p;\n\t}" ::"r"(dst), "l"(src), "r"((uint32_t)ok));
    else if constexpr (BYTES == 8)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %2, 0;\n\tcp.async.ca.shared.global [%0], [%1], 8, p;\n\t}" ::"r"(dst), "l"(src), "r"((uint32_t)ok));
    else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %2, 0;\n\tcp.async.ca.shared.global [%0], [%1], 4, p;\n\t}" ::"r"(dst), "l"(src), "r"((uint32_t)ok));
}

template <int SUB>
__device__ __forceinline__ float exact_score(const float (&x)[SUB], const float *c, float b) {
    float dd = __fmul_rn(x[0], c[0]);
#pragma unroll
    for (int t = 1; t < SUB; ++t) dd = __fadd_rn(dd, __fmul_rn(x[t], c[t]));
    return __fsub_rn(b, dd);
}

struct TcSmemHdr {
    uint64_t b_full[2], b_empty[2];
    uint64_t t_full[4];  // MMA completion of item it: [it & 3] (TMEM buffer it & 1): never 2 phases off
    uint32_t tmem_base;
};

// walk of the (row group, subspace, tile) work items of one CTA: the CTA owns the contiguous
// range [p, p_end) of (row group, subspace) pairs, pair p = g * m + j (32-bit counters: the launch
// checks ngroups * m < 2^31 and ntiles < 2^31)
struct ItemIter {
    int g, j, t, tn, p, p_end, m, gs, ntiles;
    uint32_t jt;  // pairs walked before the current one
    __device__ ItemIter(int p0, int p1, int m_, int gs_, int nt)
        : g(p0 / m_), j(p0 % m_), t(0), tn(0), p(p0), p_end(p1), m(m_), gs(gs_), ntiles(nt), jt(0) {
        tn = p < p_end ? min(ntiles - g * gs, gs) : 0;
    }
    __device__ bool valid() const { return p < p_end; }
    __device__ int tile32() const { return valid() ? g * gs + t : -1; }  // (ntiles < 2^31: checked by the launch)
    // k items ahead (jt counts every pair boundary crossed, as k single steps would)
    __device__ void advance(int k) {
        t += k;
        while (p < p_end && t >= tn) {
            t -= tn;
            ++jt;
            ++p;
            if (++j >= m) {
                j = 0;
                ++g;
                tn = min(ntiles - g * gs, gs);
            }
        }
    }
};

template <int SUB, typename TIn>
struct TcSmem {
    using S = TcShape<SUB>;
    static constexpr int kCFloats = kN * SUB + kN;                 // fp32 codebook + biases (fix-up)
    static constexpr int kXBytes = kTM * SUB * (int)sizeof(TIn);   // one staged x tile
    static constexpr size_t oB = 0;
    static constexpr size_t oA = oB + 2 * (size_t)S::kBBytes;
    static constexpr size_t oC = oA + kNA * (size_t)S::kABytes;
    static constexpr size_t oX = oC + 2 * (size_t)kCFloats * 4;
    static constexpr size_t oG = oX + kGroups * kRing * (size_t)kXBytes;  // per subspace: band constants, scale (float4)
    static size_t total(int m) { return oG + (size_t)m * 16 + sizeof(TcSmemHdr) + 16; }
};

// ------------------------------------------------------------------ the kernel
// kMark: mark mode (flags written, no fix-up; the Lloyd screen); kBest: the winning scores are
// written to best_out (tests) -- templates, so the encode path carries no per-item test of them
template <int SUB, typename TIn, bool kMark, bool kBest>
__global__ void __launch_bounds__(kThreads, 1)
encode_tc_kernel(const TIn *__restrict__ X, int64_t n, int m, int64_t xs, int64_t xjs, const float *__restrict__ CB,
                 const float *__restrict__ Bv, const float *__restrict__ guard, const uint8_t *__restrict__ img,
                 uint8_t *__restrict__ codes, int64_t cs, int64_t cjs, uint8_t *__restrict__ flags,
                 float *__restrict__ best_out, int gs, int probe) {
    // probe (debug timing only; honoured by -DCSPQ_TC_PROBES builds): bit 0 = epilogue skips its min work, bit 1 = no MMAs,
    // bit 2 = skip the A conversion, bit 3 = keep TMEM loads but skip the min work
    // (bits 0-3 leave garbage codes), bit 4 = CTA 0 writes clock64 stamps into best_out
    // (-DCSPQ_TC_STAMPS), bit 5 = no x prefetch (stale x), bit 6 = no code stores, bit 7 = no
    // selection / fix-up
    using S = TcShape<SUB>;
    using L = TcSmem<SUB, TIn>;
#ifdef CSPQ_TC_STAMPS
    long long *stamp = (probe & 16) && blockIdx.x == 0 ? reinterpret_cast<long long *>(best_out) : nullptr;
#else
    constexpr long long *stamp = nullptr;  // clock stamps: build with -DCSPQ_TC_STAMPS (scripts/stamp_tc.py)
#endif
#ifndef CSPQ_TC_PROBES
    // timing probes: build with -DCSPQ_TC_PROBES.  Bit 3's runtime test stays: it sits between
    // the unrolled chunk iterations of the scan, and without it ptxas schedules TMEM loads
    // across chunks and spills (re-measured at the 152-register budget: 150 registers, ~90 bytes of
    // spills, c3 -12 %, c4 -3.5 %)
    probe &= 8;
#endif
#ifdef CSPQ_TC_STAMPS
    if (probe & 16) best_out = nullptr;  // (the stamps borrow best_out)
#endif
    constexpr int kStampItems = 2048;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *sB = smem_raw + L::oB;
    unsigned char *sA = smem_raw + L::oA;
    float *sC = reinterpret_cast<float *>(smem_raw + L::oC);
    unsigned char *sX = smem_raw + L::oX;
    float4 *sGuard = reinterpret_cast<float4 *>(smem_raw + L::oG);
    TcSmemHdr *H = reinterpret_cast<TcSmemHdr *>(smem_raw + L::oG + (size_t)m * 16);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // The walk's constants are computed inside each role's region, from an opaque zero: a value
    // born before setmaxnreg and live across it is given a stack slot by ptxas, and the tile / pair
    // counters would live there.  Contiguous pair ranges balance the SMs at pair granularity (a
    // whole row group per CTA left up to a row group's worth of items of imbalance: c1's 782 tiles)
    auto pair_range = [&](int &p_begin, int &p_end, int &ntiles) {
        unsigned z;
        asm volatile("mov.u32 %0, 0;" : "=r"(z));
        ntiles = (int)((n + z + kTM - 1) / kTM);  // (< 2^31: checked by the launch)
        const int64_t npairs = (int64_t)((ntiles + gs - 1) / gs) * m;
        p_begin = (int)(npairs * (blockIdx.x + z) / gridDim.x);
        p_end = (int)(npairs * (blockIdx.x + z + 1) / gridDim.x);
    };

    // per subspace, in the scaled units of the fp16 operands (x' = s x, c' = s c, scores x s^2, s a
    // power of two from the image): W = G0 + ||x|| G1 bounds |b'| + ||x'|| ||c'|| plus, over E, the
    // absolute errors the relative model does not cover: fp16 operands below the normal range
    // (<= 2^-25 per element of x', of c' and of the bias) and the oracle's own float32 chain when
    // its terms are subnormal (<= 2^-150 per operation, times s^2)
    {
        const float *scales = reinterpret_cast<const float *>(img + (size_t)m * S::kBBytes);
        constexpr float kRootSub = SUB == 8 ? 2.8284271f : 2.0f;
        constexpr float kappa = 2.9802322e-8f * kRootSub / tc_error_constant(SUB);  // 2^-25 sqrt(sub) / E
        for (int i = threadIdx.x; i < m; i += kThreads) {
            const float sc = scales[i], g0 = guard[2 * i], g1 = guard[2 * i + 1];
            const float tiny = sc * 2.6469779601696886e-23f;  // s 2^-75
            sGuard[i] = make_float4(g0 * sc * sc + kappa * (g1 * sc + 1.0f / kRootSub) + (SUB + 1) * tiny * tiny / tc_error_constant(SUB),
                                    (g1 * sc + kappa) * sc, sc, 1.0f / (sc * sc));
        }
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&H->b_full[i], 1);
            mbar_init(&H->b_empty[i], 1 + 128 * kGroups);  // MMA commit + every epilogue thread (fix-up reads sC)
        }
        for (int i = 0; i < 4; ++i) mbar_init(&H->t_full[i], 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&H->tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = H->tmem_base;
    // the MMA / loader warpgroup keeps kRegsLight registers per thread; the epilogue warpgroups take
    // what it frees (the block minima of a whole item then stay in registers: no shared-memory scratch)
    // (each role's code is dominated by its own setmaxnreg: ptxas budgets registers per region)
    if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsLight));
    if (warp == 0) {
        // ---------------- MMA issuer ----------------
        // The whole warp walks the items (warp-uniform descriptors live in uniform registers) and
        // one elected lane issues: no per-thread -> uniform register waterfall around each MMA
        // (scripts/micro/umma_rate.cu: 676 vs 756 cycles from issue to completion of an item).
        uint32_t it = 0, jt = 0;
        int p_begin, p_end, ntiles;
        pair_range(p_begin, p_end, ntiles);
        // descriptors = the stage-0 / step-0 ones plus multiples of the stage and step strides in the
        // 14-bit address field (shared memory is < 256 KB, so the sums never carry out of it)
        const uint64_t da0 = make_desc(smem_u32(sA), 128, S::kRowGroupBytes), db0 = make_desc(smem_u32(sB), 128, S::kRowGroupBytes);
        int as = 0;  // A stage = it % kNA
        for (int p = p_begin; p < p_end; ++p, ++jt) {
            const int g = p / m;
            const int tn = min(ntiles - g * gs, gs);
            {
                const int jb = jt & 1;
                mbar_wait(&H->b_full[jb], (jt >> 1) & 1);
                for (int t = 0; t < tn; ++t, ++it, as = (as == kNA - 1) ? 0 : as + 1) {
                    const int tb = it & 1;
                    // everything the issue needs is computed before the waits: after the accumulator
                    // is handed back only the fence, the MMAs and the commit remain
                    uint64_t da[S::kSteps], db[S::kSteps];
#pragma unroll
                    for (int s = 0; s < S::kSteps; ++s) {
                        da[s] = da0 + (uint32_t)(as * (S::kABytes >> 4) + s * (256 >> 4));
                        db[s] = db0 + (uint32_t)(jb * (S::kBBytes >> 4) + s * (256 >> 4));
                    }
                    const uint32_t tacc = tmem + tb * kN;
                    uint64_t *const tfull = &H->t_full[it & 3];
                    bar_sync(kBarAFull + as);  // the A rows of item it (its group's fence.proxy.async precedes)
                    if (stamp && lane == 0 && it < kStampItems) stamp[it * 8 + 0] = clock64();
                    if (it >= 2) bar_sync(kBarTEmpty + tb);  // buffer tb drained by the scan of item it - 2
                    if (stamp && lane == 0 && it < kStampItems) stamp[it * 8 + 1] = clock64();
                    tc_fence_after();
                    if (elect_one()) {
#pragma unroll
                        for (int s = 0; s < S::kSteps; ++s) {
#ifdef CSPQ_TC_PROBES
                            if ((probe & 256) && s >= (S::kSteps + 1) / 2) break;  // (timing probe: half the MMAs)
#endif
                            if (!(probe & 2)) mma_f16(tacc, da[s], db[s], s > 0);
                        }
                        mma_commit(tfull);  // (completion also frees A stage `as`)
                    }
                    __syncwarp();
                    if (stamp && lane == 0 && it < kStampItems) stamp[it * 8 + 2] = clock64();
                }
                if (elect_one()) mma_commit(&H->b_empty[jb]);
                __syncwarp();
            }
        }
    } else if (warp == 1) {
        // ---------------- codebook loader: fp16 image (MMA) + fp32 codebook (fix-up) ----------------
#ifdef CSPQ_TC_STAMPS
        if (lane == 1 && stamp) {
            for (uint32_t it = 0; it < kStampItems; ++it) {
                uint32_t done = 0;
                long long t0 = clock64();
                while (!done && clock64() - t0 < 4000000) {
                    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                                 : "=r"(done) : "r"(smem_u32(&H->t_full[it & 3])), "r"((it >> 2) & 1) : "memory");
                }
                stamp[it * 8 + 3] = clock64();
            }
        }
#endif
        if (lane == 0) {
            uint32_t jt = 0;
            int p_begin, p_end, ntiles;
            pair_range(p_begin, p_end, ntiles);
            for (int p = p_begin; p < p_end; ++p) {
                {
                    const int j = p % m;
                    const int jb = jt & 1;
                    mbar_wait(&H->b_empty[jb], ((jt >> 1) & 1) ^ 1);
                    mbar_arrive_expect_tx(&H->b_full[jb], S::kBBytes + L::kCFloats * 4);
                    bulk_g2s(sB + jb * S::kBBytes, img + (int64_t)j * S::kBBytes, S::kBBytes, &H->b_full[jb]);
                    float *cdst = sC + jb * L::kCFloats;
                    bulk_g2s(cdst, CB + (int64_t)j * kN * SUB, kN * SUB * 4, &H->b_full[jb]);
                    bulk_g2s(cdst + kN * SUB, Bv + (int64_t)j * kN, kN * 4, &H->b_full[jb]);
                    ++jt;
                }
            }
        }
    }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsEpi));
        // ---------------- epilogue + A producer: kGroups groups of 4 warps ----------------
        // Group e owns the items with item % kGroups == e (TMEM buffer item & 1).  Thread (q, lane)
        // owns tile row r = 32 q + lane: it reads that TMEM lane, and it also writes that
        // row of the A operand of the group's next item (item + kGroups) and prefetches the
        // row's x kPD owned items ahead into the group's x ring.
        const int e = (warp - 4) >> 2;  // group: items it with it % kGroups == e
        const int q = warp & 3;
        const int r = 32 * q + lane;
        constexpr float kE = tc_error_constant(SUB);
        static_assert(S::kSteps == (SUB == 8 ? 2 : 1), "tc_error_constant budgets two K = 8 steps per K = 16 MMA");
        // the group's x ring: owned item k (item e + kGroups k) lives in slot k % kRing
        static_assert(kRing == kPD + 1, "slot rotation below assumes kRing == kPD + 1");
        // Per-thread constants of the loop, opaque and in registers (see opaque32): shared addresses
        // of the thread's x ring rows and A rows, its TMEM lane, the guard table, the accumulator
        // barriers; global row bases.  Row r of tile t, subspace j sits at xrow + t (128 xs) + j xjs
        // -- two wide multiply-adds instead of a 64-bit row * stride chain; row < n is t < tlim.
        const uint32_t smem0 = smem_u32(smem_raw);
        const uint32_t sg_s = opaque32(smem0 + (uint32_t)L::oG);                                  // sGuard
        const uint32_t tf_s = opaque32(smem0 + (uint32_t)L::oG + (uint32_t)m * 16 + (uint32_t)offsetof(TcSmemHdr, t_full));
        const uint32_t tm_lane = opaque32(tmem + ((uint32_t)(32 * q) << 16));
        const uint64_t xrow = opaque64((uint64_t)(uintptr_t)(X + (int64_t)r * xs));
        const uint64_t crow = opaque64((uint64_t)(uintptr_t)(codes + (int64_t)r * cs));
        const uint32_t tlim = opaque32(n > r ? (uint32_t)((n - r + kTM - 1) / kTM) : 0u);
        const uint64_t xs_tile = (uint64_t)xs * (kTM * sizeof(TIn)), xjs_b = (uint64_t)xjs * sizeof(TIn);
        const uint64_t cs_tile = (uint64_t)cs * kTM;
        // x ring rows of the current item, the next one (A conversion) and the prefetched one: the
        // addresses rotate, so no slot index is ever turned into an address inside the loop
        uint32_t x_cur = opaque32(smem0 + (uint32_t)(L::oX + ((size_t)e * kRing) * L::kXBytes + r * SUB * sizeof(TIn)));
        uint32_t x_next = x_cur + L::kXBytes, x_pf = x_cur + 2 * L::kXBytes;
        // the thread's A row in the group's two stages (e and e + kGroups) and the stage's named
        // barrier, packed (address | barrier << 24) so one XOR toggles both
        static_assert(kNA == 2 * kGroups, "A stage = item % kNA: the group's items alternate between e and e + kGroups");
        const uint32_t arow0 = smem0 + (uint32_t)(L::oA + (size_t)e * S::kABytes + (r >> 3) * S::kRowGroupBytes + (r & 7) * 16);
        const uint32_t apk0 = arow0 | ((uint32_t)(kBarAFull + e) << 24);
        const uint32_t apk1 = (arow0 + kGroups * S::kABytes) | ((uint32_t)(kBarAFull + e + kGroups) << 24);
        const uint32_t a_tog = opaque32(apk0 ^ apk1);
        uint32_t a_next = opaque32(apk1);  // (the first item's A rows go to stage e: apk0, before the loop)
        // One item of the walk as the loop needs it: tile index (-1 past the end), subspace, pair
        // counter.  The loop keeps the current item, the next one (A conversion) and a running
        // iterator two items ahead (x prefetch): one ItemIter::advance per iteration instead of three.
        struct ItemRef { int tile, j; uint32_t jt; };
        auto ref_of = [](const ItemIter &w) { return ItemRef{w.tile32(), w.j, w.jt}; };
        auto prefetch = [&](const ItemRef &pi, uint32_t dst) {
            const bool ok = (uint32_t)pi.tile < tlim;
            // (an ignored source is never read: the address may lie outside X)
            const unsigned char *src = reinterpret_cast<const unsigned char *>(
                (uintptr_t)(xrow + (uint64_t)(uint32_t)pi.tile * xs_tile + (uint64_t)(uint32_t)pi.j * xjs_b));
            constexpr int bytes = SUB * (int)sizeof(TIn);
            if constexpr (bytes == 32) {
                cp_async_pred<16>(dst, src, ok);
                cp_async_pred<16>(dst + 16, src + 16, ok);
            } else {
                cp_async_pred<bytes>(dst, src, ok);
            }
            cp_async_commit();
        };
        // A row of one of the group's items (apk: shared address of the row in the item's stage |
        // the stage's barrier << 24) from the staged x at shared address xa; returns ||x|| rounded up
        auto convert = [&](uint32_t xa, uint32_t apk, int jsub) -> float {
            float x[SUB];
            if constexpr (sizeof(TIn) == 4) {
#pragma unroll
                for (int q4 = 0; q4 < SUB / 4; ++q4) {
                    const float4 v = lds_f4(xa + 16 * q4);
                    x[4 * q4] = v.x; x[4 * q4 + 1] = v.y; x[4 * q4 + 2] = v.z; x[4 * q4 + 3] = v.w;
                }
            } else {
                uint32_t w[SUB / 4];
                if constexpr (SUB == 8) { const uint2 v = lds_u2(xa); w[0] = v.x; w[1] = v.y; }
                else w[0] = lds_u(xa);
#pragma unroll
                for (int tt = 0; tt < SUB; ++tt) x[tt] = (float)((w[tt >> 2] >> (8 * (tt & 3))) & 255u);
            }
            // fp16 split of the scaled row x' = s x (s: the subspace's power of two, so x' is exact):
            // xh = x' rounded to fp16, xl = (x' - xh) rounded to fp16 -- x' - xh is exact in fp32 and
            // |x' - xh - xl| <= 2^-22 |x'| (2^-25 absolute below the fp16 normal range).  Bytes
            // times a power of two are exact in fp16: no low part.
            const float sc = lds_f(sg_s + (uint32_t)jsub * 16 + 8);  // sGuard[jsub].z
            uint32_t h[SUB / 2], l[SUB / 2];
            float ss = 7.8886090522101181e-31f;  // 2^-100: never subnormal (the approximate sqrt below flushes)
#pragma unroll
            for (int pp = 0; pp < SUB / 2; ++pp) {
                const float a = __fmul_rn(x[2 * pp], sc), b = __fmul_rn(x[2 * pp + 1], sc);
                h[pp] = pack_f16x2(a, b);
                if constexpr (sizeof(TIn) == 1) l[pp] = 0u;
                else l[pp] = pack_f16x2(f16_resid_lo(h[pp], a), f16_resid_hi(h[pp], b));
                ss = __fmaf_rn(x[2 * pp], x[2 * pp], ss);
                ss = __fmaf_rn(x[2 * pp + 1], x[2 * pp + 1], ss);
            }
            if (!(probe & 4)) {
                const uint32_t rowp = apk & 0xFFFFFFu;
                constexpr uint32_t kOnes = 0x3C003C00u;  // (1.0, 1.0): the two bias parts
                if constexpr (SUB == 8) {
                    sts_u4(rowp, h[0], h[1], h[2], h[3]); sts_u4(rowp + 128, h[0], h[1], h[2], h[3]);
                    sts_u4(rowp + 256, l[0], l[1], l[2], l[3]); sts_u4(rowp + 384, kOnes, 0u, 0u, 0u);
                } else {
                    sts_u4(rowp, h[0], h[1], h[0], h[1]); sts_u4(rowp + 128, l[0], l[1], kOnes, 0u);
                }
            }
            fence_proxy_async();
            bar_arrive((int)(apk >> 24));
            // ||x|| rounded up: the sum's roundings (<= sub 2^-24 relative, all terms positive), the
            // approximate square root (<= 2^-22) and the product's rounding stay below the factor's
            // 8 ulp; the 2^-100 floor adds 2^-50 at most (a wider band, never a narrower one)
            float sq;
            asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sq) : "f"(ss));
            return sq * 1.000001f;
        };
        // b_empty[p & 1] phase p >> 1 belongs to pair p.  A group that owns no item of
        // a pair reaches the next pair early; its arrival must not land in the still
        // open phase of pair p - 2, so it first waits for that phase to complete.
        auto release_pair = [&](uint32_t p) {
            mbar_wait(&H->b_empty[p & 1], ((p >> 1) & 1) ^ 1);
            mbar_arrive(&H->b_empty[p & 1]);
        };

        // The group walks its own items only (item e, e + kGroups, ...); ic / ip run kGroups
        // and kGroups kPD items ahead for the A conversion and the x prefetch.
        int p_begin, p_end, ntiles;
        pair_range(p_begin, p_end, ntiles);
        ItemIter ip(p_begin, p_end, m, gs, ntiles);
        ip.advance(e);
        ItemRef ii = ref_of(ip);  // the current item
        prefetch(ii, x_cur);
        ip.advance(kGroups);
        ItemRef ic = ref_of(ip);  // the group's next item (A conversion)
        static_assert(kPD == 2, "two items prefetched ahead of the loop");
        prefetch(ic, x_next);
        ip.advance(kGroups);      // ip: the item whose x the iteration prefetches
        float norm_cur = 0.f;
        if (ii.tile >= 0) { cp_async_wait<kPD - 1>(); norm_cur = convert(x_cur, apk0, ii.j); }
        uint32_t rel = 0;  // pairs below rel are released by this thread
        auto rotate = [&] {  // the current item's slot becomes the next prefetch target
            const uint32_t x_old = x_cur;
            x_cur = x_next;
            x_next = x_pf;
            x_pf = x_old;
        };

        for (uint32_t it = e; ii.tile >= 0; it += kGroups, ii = ic, ic = ref_of(ip), ip.advance(kGroups), rotate(), a_next ^= a_tog) {
            for (; rel < ii.jt; ++rel) release_pair(rel);  // done with those pairs' sC
            // the group's next item first: stage the x prefetch of the one after it and write its A
            // rows into the group's other A stage (free since item it - kGroups was scanned), so
            // its MMA can start as soon as a TMEM buffer is handed back
            if (!(probe & 32)) prefetch(ref_of(ip), x_pf);  // (an empty group keeps the wait count uniform)
            float norm_next = 0.f;
            if (ic.tile >= 0) {
                if (!(probe & 32)) cp_async_wait<kPD - 1>();
                norm_next = convert(x_next, a_next, ic.j);
            }
            const int tb = it & 1;  // TMEM buffer
            const uint32_t jt = ii.jt;
            const int j = ii.j;
            // second level over the 32 block minima (slot b = 4 u + s), folded chunk by chunk: 8
            // "super-block" minima (u = b >> 2) and 4 "super-class" minima (s = b & 3) -- two blocks
            // differ in u or in s, so a second block inside the band shows up in another super-block
            // or super-class minimum
            float cls[kNCls], sbm[8], scm[4];
#pragma unroll
            for (int c = 0; c < kNCls; ++c) cls[c] = pos_inf_f();
#pragma unroll
            for (int c = 0; c < 4; ++c) scm[c] = pos_inf_f();
#pragma unroll
            for (int ch = 0; ch < 4 && !(probe & 1); ++ch) {
                if (ch == 0) {
                    mbar_wait_s<CSPQ_TC_WAIT_SLEEP>(tf_s + 8 * (it & 3), (it >> 2) & 1);
                    if (stamp && r == 0 && it < kStampItems) stamp[it * 8 + 5] = clock64();
                    tc_fence_after();
                }
                float bmc[8];
#pragma unroll
                for (int half = 0; half < 64 / kLdCols; ++half) {
                uint32_t v[kLdCols];
                if constexpr (kLdCols == 64) tmem_ld64(tm_lane + tb * kN + ch * 64, v);
                else tmem_ld32(tm_lane + tb * kN + ch * 64 + half * 32, v);
                if (ch == 3 && half == 64 / kLdCols - 1) {  // the whole accumulator is in registers or reduced: hand the buffer back
                    tc_fence_before();
                    bar_arrive(kBarTEmpty + tb);
                    if (stamp && r == 0 && it < kStampItems) stamp[it * 8 + 4] = clock64();
                }
#define SV(i) __uint_as_float(v[(i)])
                if (probe & 8) {
                    cls[ch] = __fadd_rn(SV(0), SV(kLdCols - 1));
                    continue;
                }
                // each 16 columns = a block of 7 then a block of 9 (3 + 4 three-input minima, no
                // idle operand slot); the class is the position inside the block, so classes 0-6
                // take two columns per 16 and classes 7-8 one (paired across 16-column groups)
#pragma unroll
                for (int bq = 0; bq < kLdCols / 16; ++bq) {
                    const int o = 16 * bq, bp = bq + half * (kLdCols / 16);
#pragma unroll
                    for (int c = 0; c < 7; ++c) cls[c] = fmin3(cls[c], SV(o + c), SV(o + 7 + c));
                    if (bp & 1) {
                        cls[7] = fmin3(cls[7], SV(o - 2), SV(o + 14));
                        cls[8] = fmin3(cls[8], SV(o - 1), SV(o + 15));
                    }
                    bmc[2 * bp] = fmin3(fmin3(SV(o), SV(o + 1), SV(o + 2)), fmin3(SV(o + 3), SV(o + 4), SV(o + 5)), SV(o + 6));
                    bmc[2 * bp + 1] = fmin3(fmin3(SV(o + 7), SV(o + 8), SV(o + 9)), fmin3(SV(o + 10), SV(o + 11), SV(o + 12)),
                                            fmin3(SV(o + 13), SV(o + 14), SV(o + 15)));
                }
#undef SV
                }
                if (probe & 8) continue;
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    sbm[2 * ch + h] = fmin3(fmin3(bmc[4 * h], bmc[4 * h + 1], bmc[4 * h + 2]), bmc[4 * h + 3], bmc[4 * h + 3]);
#pragma unroll
                for (int c = 0; c < 4; ++c) scm[c] = fmin3(scm[c], bmc[c], bmc[4 + c]);
            }
            if (probe & 1) {  // (timing probe: no TMEM reads; still walk the barriers)
                mbar_wait_s(tf_s + 8 * (it & 3), (it >> 2) & 1);
                bar_arrive(kBarTEmpty + tb);
            }
            if (stamp && r == 0 && it < kStampItems) stamp[it * 8 + 6] = clock64();
            const float xnorm = norm_cur;
            norm_cur = norm_next;
            const bool inb = (uint32_t)ii.tile < tlim;  // row < n
            uint8_t *const cptr = reinterpret_cast<uint8_t *>(  // the row's code of subspace j
                (uintptr_t)(crow + (uint64_t)(uint32_t)ii.tile * cs_tile + (uint64_t)(uint32_t)j * (uint64_t)cjs));
            if (probe & 128) {  // (timing probe: no selection / fix-up; garbage codes)
                if (inb && !(probe & 64)) *cptr = (uint8_t)(__float_as_uint(cls[0] + xnorm) & 255);
                continue;
            }
            // Final selection on the FMA pipe.  m1 = the minimum (of the class minima); the band
            // indicator ind(v) = sat(1 - (v - m1) / (4 E W)) is exactly 1 for v == m1, exactly 0
            // beyond the guard band and in between inside it (0 for NaN).  A (row, subspace) is
            // decided iff exactly one class minimum and exactly one block minimum have a nonzero
            // indicator (the sums of the indicators are exactly 1): then no other centroid lies
            // within the band -- any other centroid shares neither its block nor its class with
            // the winner, or only one of them, and its block or class minimum would be in the band
            // -- and the indicator-weighted index sums give the winner's block and class exactly.
            // (An indicator < 2^-24 can vanish in a sum; its value is > 3.9 E W from m1, outside
            // the 2 E W that exactness needs.)
            const float m1 = fmin3(fmin3(cls[0], cls[1], cls[2]), fmin3(cls[3], cls[4], cls[5]), fmin3(cls[6], cls[7], cls[8]));
            const float4 gj = lds_f4(sg_s + (uint32_t)j * 16);  // sGuard[j] = (G0, G1, s, 1 / s^2)
            float W = gj.x + xnorm * gj.y;
            // The scaled scores have more range than the oracle's float32 chain: when its terms can
            // reach 2^127 in the original units (W / s^2) the oracle may overflow to inf / NaN where
            // the tensor score is finite -- W becomes NaN (inf x 0) and the row is flagged
            W = __fmaf_rn(__fmul_rn(W, 2.0f * gj.w), 0.0f, W);
            // binary band indicator on the FMA pipe: ind(v) = sat((thr - v) 2^126), thr = m1 + 4 E W;
            // the difference is flushed to zero below 2^-126, so ind is exactly 1 (v < thr) or 0
            // (v >= thr, NaN, or W = 0 / non-finite).  One exact integer accumulator counts and
            // names the candidates inside the band: class c adds 2^9 + c, super-class s adds
            // 2^13 + 16 s, super-block u adds 2^17 + 64 u.  The minimum itself is always inside, so
            // every count is >= 1 and carries only ever raise a count: the sum lies in
            // [kSelBase, kSelBase + 512) iff exactly one candidate of each kind is inside the band,
            // and its low 9 bits then hold (u, s, c).
            const float thr = __fadd_rn(m1, 4.0f * kE * W);
            auto ind = [&](float v) {
                float d, o;
                asm("sub.ftz.f32 %0, %1, %2;" : "=f"(d) : "f"(thr), "f"(v));
                asm("mul.sat.f32 %0, %1, 0f7E800000;" : "=f"(o) : "f"(d));  // x 2^126
                return o;
            };
            constexpr int kSelBase = (1 << 9) + (1 << 13) + (1 << 17);
            float tc = 0.f, ts = 0.f, tu = 0.f;
#pragma unroll
            for (int c = 0; c < kNCls; ++c) tc = __fmaf_rn(ind(cls[c]), (float)((1 << 9) + c), tc);
#pragma unroll
            for (int c = 0; c < 4; ++c) ts = __fmaf_rn(ind(scm[c]), (float)((1 << 13) + 16 * c), ts);
#pragma unroll
            for (int u = 0; u < 8; ++u) tu = __fmaf_rn(ind(sbm[u]), (float)((1 << 17) + 64 * u), tu);
            const uint32_t sel = (uint32_t)(__float2int_rz(__fadd_rn(__fadd_rn(tc, ts), tu)) - kSelBase);
            // block slot sb starts at column 8 sb - (sb & 1) (7-blocks at even slots, 9-blocks at odd)
            const int sb = (int)(sel >> 4) & 31;
            int code = 8 * sb - (sb & 1) + (int)(sel & 15);
            const bool flag = inb && !(sel < 512u);
            // exact warp-cooperative re-encode of flagged rows (x and the fp32 codebook from
            // shared memory: the item's x slot stays valid until kPD more owned items)
            if constexpr (kMark) {  // mark mode (Lloyd screening): flagged rows are settled by the caller
                if (inb) cptr[flags - codes] = flag ? 1 : 0;  // (same layout as the codes)
                const unsigned fm = __ballot_sync(0xffffffffu, flag);
                if (lane == 0 && fm) atomicAdd(&g_tc_flagged, (unsigned long long)__popc(fm));
            }
            unsigned mask = kMark ? 0u : __ballot_sync(0xffffffffu, flag && !(probe & 15));
            if (mask) {
                // acquire the bulk copies of this pair (the buffer cannot advance past this
                // pair until every epilogue thread has arrived on b_empty)
                mbar_wait(&H->b_full[jt & 1], (jt >> 1) & 1);
                const float *cbs = sC + (jt & 1) * L::kCFloats;
                if (lane == 0) atomicAdd(&g_tc_flagged, (unsigned long long)__popc(mask));
                while (mask) {
                    const int src = __ffs(mask) - 1;
                    mask &= mask - 1;
                    const TIn *xr = reinterpret_cast<const TIn *>(smem_raw + (x_cur - smem0)) + (src - lane) * SUB;
                    float xv[SUB];
#pragma unroll
                    for (int tt = 0; tt < SUB; ++tt) xv[tt] = (float)xr[tt];
                    float best = pos_inf_f();
                    int bl = kN;
#pragma unroll 2
                    for (int l = lane; l < kN; l += 32) {
                        float cv[SUB];
#pragma unroll
                        for (int tt = 0; tt < SUB; ++tt) cv[tt] = cbs[l * SUB + tt];
                        const float sc = exact_score<SUB>(xv, cv, cbs[kN * SUB + l]);
                        if (sc < best) { best = sc; bl = l; }
                    }
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) {
                        const float ob2 = __shfl_xor_sync(0xffffffffu, best, off);
                        const int ol = __shfl_xor_sync(0xffffffffu, bl, off);
                        if (ob2 < best || (ob2 == best && ol < bl)) { best = ob2; bl = ol; }
                    }
                    if (lane == src) code = (best < pos_inf_f()) ? bl : 0;
                }
            }
            if (inb) {
                if (!(probe & 64)) *cptr = (uint8_t)code;
                if constexpr (kBest) {
                    if (best_out) best_out[((int64_t)ii.tile * kTM + r) * m + j] = m1 * gj.w;  // back from the scaled units (exact: a power of two)  // (a stamp run borrows best_out: nullptr then)
                }
            }
            if (stamp && r == 0 && it < kStampItems) stamp[it * 8 + 7] = clock64();
        }
        for (; rel < (uint32_t)(p_end - p_begin); ++rel) release_pair(rel);  // every pair this CTA walked
        cp_async_wait<0>();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

// Codebook image: per subspace, 256 rows (centroids) x K fp16 in the K-major no-swizzle core-matrix
// layout the MMA reads, [-ch | -cl | -ch | bh bl 0..] of the scaled codebook c' = s c, b' = s^2 b
// (ch = c' rounded to fp16, cl = (c' - ch) rounded to fp16), followed by the m scales.  s is the
// power of two that puts the largest centroid norm in [32, 64) -- |c'| < 64 and b' = ||c'||^2 / 2 <
// 2^11 are inside the fp16 range with their low parts normal, and a row overflows fp16 (-> NaN
// scores -> flagged -> exact path) only when an |x_t| exceeds ~1000 times that norm -- lowered
// when a caller's bias is larger than that (s^2 max|b| <= 2^15).
template <int SUB>
__global__ void tc_image_kernel(const float *__restrict__ CB, const float *__restrict__ B, int m,
                                uint8_t *__restrict__ img) {
    using S = TcShape<SUB>;
    const int j = blockIdx.x, l = threadIdx.x;  // 256 threads
    const float *c = CB + ((int64_t)j * kN + l) * SUB;
    float cv[SUB], nn = 0.f;
#pragma unroll
    for (int t = 0; t < SUB; ++t) {
        cv[t] = c[t];
        nn = __fmaf_ru(cv[t], cv[t], nn);
    }
    const float b = B[(int64_t)j * kN + l];
    __shared__ float red[2][kN / 32];
    __shared__ float s_scale;
    float vn = __fsqrt_ru(nn), vb = fabsf(b);
    if (!(vn <= 3.0e38f)) vn = 0.f;  // (non-finite centroids: the scale ignores them; their scores flag)
    if (!(vb <= 3.0e38f)) vb = 0.f;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        vn = fmaxf(vn, __shfl_xor_sync(0xffffffffu, vn, off));
        vb = fmaxf(vb, __shfl_xor_sync(0xffffffffu, vb, off));
    }
    if ((l & 31) == 0) { red[0][l >> 5] = vn; red[1][l >> 5] = vb; }
    __syncthreads();
    if (l == 0) {
        float mn = 0.f, mb = 0.f;
        for (int w = 0; w < kN / 32; ++w) { mn = fmaxf(mn, red[0][w]); mb = fmaxf(mb, red[1][w]); }
        int e = 0;
        if (mn > 0.f) { int q; frexpf(mn, &q); e = 6 - q; }           // mn 2^e in [32, 64)
        if (mb > 0.f) { int q; frexpf(mb, &q); e = min(e, (15 - q) / 2 - ((15 - q) < 0 && ((15 - q) & 1) ? 1 : 0)); }  // mb 2^(2e) < 2^15
        e = max(-62, min(62, e));  // (s^2 and 1 / s^2 stay finite)
        s_scale = ldexpf(1.0f, e);
        reinterpret_cast<float *>(img + (size_t)m * S::kBBytes)[j] = s_scale;
    }
    __syncthreads();
    const float sc = s_scale;
    uint32_t hw[SUB / 2], lw[SUB / 2];
#pragma unroll
    for (int pp = 0; pp < SUB / 2; ++pp) {
        const float a0 = -cv[2 * pp] * sc, a1 = -cv[2 * pp + 1] * sc;  // (exact: a power of two)
        hw[pp] = pack_f16x2(a0, a1);
        lw[pp] = pack_f16x2(a0 - f16_lo(hw[pp]), a1 - f16_hi(hw[pp]));
    }
    const float bs = b * sc * sc;
    const uint32_t bw = pack_f16x2(bs, 0.f);
    const uint32_t bias = pack_f16x2(f16_lo(bw), bs - f16_lo(bw));  // (bh, bl)
    unsigned char *rowp = img + (int64_t)j * S::kBBytes + (l >> 3) * S::kRowGroupBytes + (l & 7) * 16;
    auto st = [&](int cch, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3) {
        *reinterpret_cast<uint4 *>(rowp + cch * 128) = make_uint4(a0, a1, a2, a3);
    };
    if constexpr (SUB == 8) {
        st(0, hw[0], hw[1], hw[2], hw[3]); st(1, lw[0], lw[1], lw[2], lw[3]);
        st(2, hw[0], hw[1], hw[2], hw[3]); st(3, bias, 0u, 0u, 0u);
    } else {
        st(0, hw[0], hw[1], lw[0], lw[1]); st(1, hw[0], hw[1], bias, 0u);
    }
}

template <int SUB, typename TIn>
int launch_tc(const TIn *X, int64_t n, int m, int64_t xs, int64_t xjs, const float *CB, const float *B, const float *guard,
              const uint8_t *img, uint8_t *codes, int64_t cs, int64_t cjs, uint8_t *flags, float *best, cudaStream_t st) {
    const size_t smem = TcSmem<SUB, TIn>::total(m);
    CSPQ_REQUIRE(smem <= 227 * 1024, CSPQ_E_CONFIG, "too many subspaces (%d) for the tensor-core kernel", m);
    CSPQ_REQUIRE((n + kTM - 1) / kTM < ((int64_t)1 << 31), CSPQ_E_CONFIG, "too many rows (%lld) for one launch", (long long)n);
#ifdef CSPQ_TC_PROBES
    const char *pe = getenv("CSPQ_TC_PROBE");  // debug timing knob of the instrumented build, see the kernel
    const int probe = pe ? atoi(pe) : 0;
#else
    const int probe = 0;  // (a production build never reads the knob: probe bits change codes)
#endif
    auto kern = flags ? (best ? encode_tc_kernel<SUB, TIn, true, true> : encode_tc_kernel<SUB, TIn, true, false>)
                      : (best ? encode_tc_kernel<SUB, TIn, false, true> : encode_tc_kernel<SUB, TIn, false, false>);
    // per-launch host work kept to the launch itself (small batches -- c5's 4096 rows -- launch
    // often): the shared-memory opt-in is set once per (device, kernel) at the maximum, the SM
    // count read once per device
    int dev = 0;
    cudaGetDevice(&dev);
    static int sm_count[64] = {};
    static std::atomic<uint32_t> smem_set[64][2][2] = {};  // [device][mark][best] (statics are per SUB, TIn)
    const int di = dev & 63;
    if (!sm_count[di]) {
        int v = 148;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        sm_count[di] = v;
    }
    const int sms = sm_count[di];
    std::atomic<uint32_t> &once = smem_set[di][flags ? 1 : 0][best ? 1 : 0];
    if (!once.load(std::memory_order_acquire)) {
        CSPQ_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        once.store(1, std::memory_order_release);
    }
    const int64_t ntiles = (n + kTM - 1) / kTM;
    // tiles per row group: the CTAs share the (row group, subspace) pairs in contiguous ranges, so
    // the largest row group (kG tiles: the most codebook-image reuse) balances to within a pair
    // 8 tiles.  16 for long uint8 / d_sub 4 launches ran 1.3 % faster on c4 but doubled its DRAM traffic
    // (335 vs 168 B/row under ncu: a row's four sectors are fetched again by later subspaces once 16
    // tiles x 148 CTAs of rows no longer stay in L2), so it is not the default; float32 rows: 16 tiles
    // c3 -0.3 %, c1 -9 % (balance), 32 tiles c3 -27 %, c5 -48 %; 4 / 6 / 12 tiles within +-0.5 % of 8
    int gs = 8;
    static const int gs_env = [] { const char *ge = getenv("CSPQ_TC_GS"); return ge ? atoi(ge) : 0; }();
    if (gs_env) gs = std::max(1, std::min(kG, gs_env));  // debug override
    const int64_t ngroups = (ntiles + gs - 1) / gs;
    CSPQ_REQUIRE(ngroups * m < ((int64_t)1 << 31), CSPQ_E_CONFIG, "too many rows (%lld) for one launch", (long long)n);
    const int grid = (int)std::min<int64_t>(sms, ngroups * m);
    kern<<<grid, kThreads, smem, st>>>(X, n, m, xs, xjs, CB, B, guard, img, codes, cs, cjs, flags, best, gs, probe);
    CSPQ_LAUNCH_CHECK();
    return CSPQ_OK;
}

}  // namespace

size_t encode_tc_image_bytes(int m, int k, int sub) {
    if (k != kN || (sub != 4 && sub != 8)) return 0;
    return (size_t)m * (sub == 8 ? TcShape<8>::kBBytes : TcShape<4>::kBBytes) + ((size_t)m * 4 + 15) / 16 * 16;  // + the scales
}

int encode_tc_prepare(const float *CB, const float *B, int m, int k, int sub, void *img, cudaStream_t st) {
    CSPQ_REQUIRE(k == kN && (sub == 4 || sub == 8), CSPQ_E_CONFIG,
                 "tensor-core encode needs k=256 and sub in {4, 8} (got k=%d, sub=%d)", k, sub);
    if (sub == 8) tc_image_kernel<8><<<m, kN, 0, st>>>(CB, B, m, reinterpret_cast<uint8_t *>(img));
    else tc_image_kernel<4><<<m, kN, 0, st>>>(CB, B, m, reinterpret_cast<uint8_t *>(img));
    CSPQ_LAUNCH_CHECK();
    return CSPQ_OK;
}

// xjs / cjs: element strides between subspaces of a row in X and in codes (sub and 1 for
// row-major (n, d) rows and (n, m) codes; n * sub and n for subspace-major Lloyd points and
// assignments).  flags != nullptr: mark mode -- flagged (row, subspace) pairs get flag 1 and
// an unspecified code instead of the exact fix-up (the caller settles them).
int encode_tc_ex(const void *X, int in_dtype, int64_t n, int64_t xrs, int64_t xjs, const float *CB, const float *B,
                 const float *guard, const void *img, int m, int k, int sub, uint8_t *codes, int64_t crs, int64_t cjs,
                 uint8_t *flags, float *best, cudaStream_t st) {
    CSPQ_REQUIRE(k == kN && (sub == 4 || sub == 8), CSPQ_E_CONFIG,
                 "tensor-core encode needs k=256 and sub in {4, 8} (got k=%d, sub=%d)", k, sub);
    const uint8_t *im = reinterpret_cast<const uint8_t *>(img);
    if (in_dtype == CSPQ_IN_U8) {
        const uint8_t *x = reinterpret_cast<const uint8_t *>(X);
        // the x prefetch copies one subvector (sub bytes) with a sub-byte cp.async
        CSPQ_REQUIRE(reinterpret_cast<uintptr_t>(x) % sub == 0 && xrs % sub == 0 && xjs % sub == 0, CSPQ_E_CONFIG,
                     "tensor-core encode needs uint8 subvectors aligned to %d bytes", sub);
        return sub == 8 ? launch_tc<8, uint8_t>(x, n, m, xrs, xjs, CB, B, guard, im, codes, crs, cjs, flags, best, st)
                        : launch_tc<4, uint8_t>(x, n, m, xrs, xjs, CB, B, guard, im, codes, crs, cjs, flags, best, st);
    }
    const float *x = reinterpret_cast<const float *>(X);
    CSPQ_REQUIRE(reinterpret_cast<uintptr_t>(x) % 16 == 0 && (xrs * 4) % 16 == 0 && (xjs * 4) % 16 == 0, CSPQ_E_CONFIG,
                 "tensor-core encode needs 16-byte aligned float32 rows");
    return sub == 8 ? launch_tc<8, float>(x, n, m, xrs, xjs, CB, B, guard, im, codes, crs, cjs, flags, best, st)
                    : launch_tc<4, float>(x, n, m, xrs, xjs, CB, B, guard, im, codes, crs, cjs, flags, best, st);
}

int encode_tc(const void *X, int in_dtype, int64_t n, int64_t xrs, const float *CB, const float *B,
              const float *guard, const void *img, int m, int k, int sub, uint8_t *codes, int64_t crs, float *best,
              cudaStream_t st) {
    return encode_tc_ex(X, in_dtype, n, xrs, sub, CB, B, guard, img, m, k, sub, codes, crs, 1, nullptr, best, st);
}

// the largest m whose guard constants fit next to the kernel's fixed shared-memory layout
float encode_tc_error_constant(int sub) { return tc_error_constant(sub); }

int encode_tc_max_subspaces(int sub, int in_dtype) {
    auto fit = [](size_t fixed) { return (int)((227 * 1024 - fixed - sizeof(TcSmemHdr) - 16) / 16 / 4 * 4); };
    if (sub == 8) return in_dtype == CSPQ_IN_U8 ? fit(TcSmem<8, uint8_t>::oG) : fit(TcSmem<8, float>::oG);
    if (sub == 4) return in_dtype == CSPQ_IN_U8 ? fit(TcSmem<4, uint8_t>::oG) : fit(TcSmem<4, float>::oG);
    return 0;
}

int encode_tc_stats(unsigned long long *flagged, int reset) {
    if (flagged) CSPQ_CUDA_TRY(cudaMemcpyFromSymbol(flagged, g_tc_flagged, sizeof(unsigned long long)));
    if (reset) {
        const unsigned long long z = 0;
        CSPQ_CUDA_TRY(cudaMemcpyToSymbol(g_tc_flagged, &z, sizeof(z)));
    }
    return CSPQ_OK;
}

}  // namespace cspq
