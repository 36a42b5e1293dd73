// min/max issue-rate microbenchmark (sm_100a): FMNMX3, FMNMX, IMNMX, HMNMX2, FSETP+SEL
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#define NC 16
__device__ float g_seed[64];
__device__ __forceinline__ float fmin3(float a, float b, float c) { float d; asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }
__global__ void k_min3(float *out, int iters) {
    float a[NC], x = g_seed[threadIdx.x & 63], y = g_seed[(threadIdx.x + 7) & 63];
    for (int i = 0; i < NC; ++i) a[i] = g_seed[(i + threadIdx.x) & 63];
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NC; ++i) a[i] = fmin3(a[i], a[(i + 3) % NC], a[(i + 7) % NC]);
    }
    float s = 0; for (int i = 0; i < NC; ++i) s += a[i]; out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_min2(float *out, int iters) {
    float a[NC], x = g_seed[threadIdx.x & 63];
    for (int i = 0; i < NC; ++i) a[i] = g_seed[(i + threadIdx.x) & 63];
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NC; ++i) a[i] = fmaxf(a[i], a[(i + 5) % NC]);
    }
    float s = 0; for (int i = 0; i < NC; ++i) s += a[i]; out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_imin(float *out, int iters) {
    int a[NC], x = __float_as_int(g_seed[threadIdx.x & 63]);
    for (int i = 0; i < NC; ++i) a[i] = __float_as_int(g_seed[(i + threadIdx.x) & 63]);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NC; ++i) a[i] = max(a[i], a[(i + 5) % NC]);
    }
    int s = 0; for (int i = 0; i < NC; ++i) s += a[i]; out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_hmin2(float *out, int iters) {
    __half2 a[NC], x = __floats2half2_rn(g_seed[threadIdx.x & 63], g_seed[1]);
    for (int i = 0; i < NC; ++i) a[i] = __floats2half2_rn(g_seed[(i + threadIdx.x) & 63], g_seed[i]);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NC; ++i) a[i] = __hmax2(a[i], a[(i + 5) % NC]);
    }
    float s = 0; for (int i = 0; i < NC; ++i) s += __low2float(a[i]); out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float *out; cudaMalloc(&out, 148 * 4 * 1024 * 4);
    float h[64]; for (int i = 0; i < 64; ++i) h[i] = 1000.0f + i; cudaMemcpyToSymbol(g_seed, h, 256);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 1 << 14; dim3 g(148 * 4), b(256);
    const char *nm[] = {"fmnmx3", "fmnmx", "imnmx", "hmnmx2"};
    for (int k = 0; k < 4; ++k) for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (k == 0) k_min3<<<g, b>>>(out, iters);
        if (k == 1) k_min2<<<g, b>>>(out, iters);
        if (k == 2) k_imin<<<g, b>>>(out, iters);
        if (k == 3) k_hmin2<<<g, b>>>(out, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)NC * iters * g.x * b.x;  // thread-level min ops
        // per-SMSP warp-instructions per cycle at 1.965 GHz
        double ipc = ops / 32.0 / (148 * 4) / (ms * 1e-3 * 1.965e9);
        if (rep) printf("%-7s %.3f ms  %.3f warp-instr/clk/SMSP (incl. the adds)\n", nm[k], ms, ipc);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
