// tcgen05.mma issue-rate microbenchmark (sm_100a): one CTA per SM, one thread issues
// `items` x `ksteps` MMAs (M = 128, N = 256 or 128, K = 8 tf32 / 16 bf16 per instruction)
// into two alternating TMEM accumulators, one commit per item, no waits until the end.
// Prints cycles per item (clock64 on the issuing thread) -- the tensor-pipe floor of the
// encode kernel's item (M=128, N=256, K=32 tf32 = 4 MMAs).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
template <int KIND>  // 0 tf32, 1 bf16
__device__ __forceinline__ void mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    if (KIND == 0)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
                     "l"(da), "l"(db), "r"(idesc), "r"(acc) : "memory");
    else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
                     "l"(da), "l"(db), "r"(idesc), "r"(acc) : "memory");
}

template <int KIND, int N, int KSTEPS>
__global__ void __launch_bounds__(128, 1) k_umma(int items, long long *cycles) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int K = KSTEPS * 8;  // tf32 elements per row (32 B per K-step)
    unsigned char *sA = sm, *sB = sm + 128 * K * 4;
    for (int i = threadIdx.x; i < (128 + N) * K; i += blockDim.x) reinterpret_cast<float *>(sm)[i] = 0.f;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tbase;
    const uint32_t fmt = KIND == 0 ? 2u : 1u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const int rg = KSTEPS * 2 * 128;  // bytes per 8-row group (K-major core matrices)
    if (threadIdx.x == 0) {
        const long long t0 = clock64();
        for (int it = 0; it < items; ++it) {
#pragma unroll
            for (int s = 0; s < KSTEPS; ++s) {
                const uint64_t da = make_desc(smem_u32(sA) + 2 * s * 128, 128, rg);
                const uint64_t db = make_desc(smem_u32(sB) + 2 * s * 128, 128, rg);
                mma<KIND>(tmem + (it & 1) * 256, da, db, idesc, s > 0);
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
        cycles[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

template <int KIND, int N, int KSTEPS>
void run(const char *name, long long *d_cyc) {
    const int items = 4096;
    const size_t smem = (size_t)(128 + N) * KSTEPS * 8 * 4;
    auto k = k_umma<KIND, N, KSTEPS>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<<<148, 128, smem>>>(16, d_cyc);
    cudaEventRecord(e0);
    k<<<148, 128, smem>>>(items, d_cyc);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    long long h[148]; cudaMemcpy(h, d_cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
    const double macs = 128.0 * N * KSTEPS * (KIND == 0 ? 8 : 16);
    printf("%-22s %s  %8.1f cycles/item  %7.1f MAC/clk/SM  %7.1f TFLOP/s (events %.3f ms)\n", name, cudaGetErrorString(err),
           avg / items, macs / (avg / items), 2 * macs * items * 148 / (ms * 1e-3) / 1e12, ms);
}


// latency of one item (KSTEPS dependent MMAs) issued into an idle pipe: issue time and
// issue -> commit-barrier completion, averaged over `items` bursts
template <int N, int KSTEPS>
__global__ void __launch_bounds__(128, 1) k_umma_lat(int items, long long *cycles) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int K = KSTEPS * 8;
    unsigned char *sA = sm, *sB = sm + 128 * K * 4;
    for (int i = threadIdx.x; i < (128 + N) * K; i += blockDim.x) reinterpret_cast<float *>(sm)[i] = 0.f;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tbase;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const int rg = KSTEPS * 2 * 128;
    if (threadIdx.x == 0) {
        long long iss = 0, lat = 0;
        for (int it = 0; it < items; ++it) {
            const long long t0 = clock64();
#pragma unroll
            for (int s = 0; s < KSTEPS; ++s) {
                const uint64_t da = make_desc(smem_u32(sA) + 2 * s * 128, 128, rg);
                const uint64_t db = make_desc(smem_u32(sB) + 2 * s * 128, 128, rg);
                mma<0>(tmem + (it & 1) * 256, da, db, idesc, s > 0);
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
            const long long t1 = clock64();
            uint32_t done = 0;
            while (!done)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(done) : "r"(smem_u32(&bar)), "r"((uint32_t)(it & 1)) : "memory");
            const long long t2 = clock64();
            iss += t1 - t0; lat += t2 - t0;
        }
        cycles[2 * blockIdx.x] = iss; cycles[2 * blockIdx.x + 1] = lat;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}
template <int N, int KSTEPS>
void run_lat(const char *name, long long *d) {
    const int items = 512;
    const size_t smem = (size_t)(128 + N) * KSTEPS * 8 * 4;
    auto k = k_umma_lat<N, KSTEPS>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<148, 128, smem>>>(items, d);
    cudaError_t err = cudaDeviceSynchronize();
    long long h[296]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double a = 0, b = 0; for (int i = 0; i < 148; ++i) { a += h[2 * i]; b += h[2 * i + 1]; }
    printf("%-22s %s  issue %7.1f cycles  issue->done %7.1f cycles (idle pipe, per item)\n", name, cudaGetErrorString(err),
           a / 148 / items, b / 148 / items);
}

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    return pred != 0;
}
// same as k_umma_lat, but the whole warp runs the loop and one elected lane issues
// (warp-uniform descriptors: no per-thread -> uniform register waterfall around each MMA)
template <int N, int KSTEPS>
__global__ void __launch_bounds__(128, 1) k_umma_lat_warp(int items, long long *cycles) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int K = KSTEPS * 8;
    unsigned char *sA = sm, *sB = sm + 128 * K * 4;
    for (int i = threadIdx.x; i < (128 + N) * K; i += blockDim.x) reinterpret_cast<float *>(sm)[i] = 0.f;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tbase;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const int rg = KSTEPS * 2 * 128;
    if (threadIdx.x < 32) {
        long long iss = 0, lat = 0;
        for (int it = 0; it < items; ++it) {
            const long long t0 = clock64();
            if (elect_one()) {
#pragma unroll
                for (int s = 0; s < KSTEPS; ++s) {
                    const uint64_t da = make_desc(smem_u32(sA) + 2 * s * 128, 128, rg);
                    const uint64_t db = make_desc(smem_u32(sB) + 2 * s * 128, 128, rg);
                    mma<0>(tmem + (it & 1) * 256, da, db, idesc, s > 0);
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
            }
            __syncwarp();
            const long long t1 = clock64();
            uint32_t done = 0;
            while (!done)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(done) : "r"(smem_u32(&bar)), "r"((uint32_t)(it & 1)) : "memory");
            const long long t2 = clock64();
            iss += t1 - t0; lat += t2 - t0;
        }
        if (threadIdx.x == 0) { cycles[2 * blockIdx.x] = iss; cycles[2 * blockIdx.x + 1] = lat; }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}
template <int N, int KSTEPS>
void run_lat_warp(const char *name, long long *d) {
    const int items = 512;
    const size_t smem = (size_t)(128 + N) * KSTEPS * 8 * 4;
    auto k = k_umma_lat_warp<N, KSTEPS>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<148, 128, smem>>>(items, d);
    cudaError_t err = cudaDeviceSynchronize();
    long long h[296]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double a = 0, b = 0; for (int i = 0; i < 148; ++i) { a += h[2 * i]; b += h[2 * i + 1]; }
    printf("%-22s %s  issue %7.1f cycles  issue->done %7.1f cycles (idle pipe, per item, warp+elect)\n", name, cudaGetErrorString(err),
           a / 148 / items, b / 148 / items);
}

int main() {
    long long *d; cudaMalloc(&d, 296 * sizeof(long long));
    run<0, 256, 4>("tf32 N256 K32", d);
    run<0, 256, 3>("tf32 N256 K24", d);
    run<0, 256, 2>("tf32 N256 K16", d);
    run<0, 128, 4>("tf32 N128 K32", d);
    run<1, 256, 2>("bf16 N256 K32", d);
    run<1, 256, 4>("bf16 N256 K64", d);
    run_lat<256, 4>("lat tf32 N256 K32", d);
    run_lat<256, 1>("lat tf32 N256 K8", d);
    run_lat<128, 4>("lat tf32 N128 K32", d);
    run_lat_warp<256, 4>("latw tf32 N256 K32", d);
    run_lat_warp<256, 1>("latw tf32 N256 K8", d);
    return 0;
}
