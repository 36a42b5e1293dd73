// FFMA issue-rate microbenchmark: which operand forms reach 1 warp-FFMA/clk/SMSP on sm_100a?
#include <cstdio>
#include <cuda_runtime.h>
#define N_CHAIN 16
#define ITERS 4096
__device__ float g_seed[64];

__global__ void k_reg3(float *out, const float *cb, int iters) {
    float acc[N_CHAIN], x[N_CHAIN], y[N_CHAIN];
    for (int i = 0; i < N_CHAIN; ++i) { acc[i] = cb[(threadIdx.x + i) & 63]; x[i] = cb[(i * 3 + threadIdx.x) & 63]; y[i] = cb[(i * 5 + 7) & 63]; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < N_CHAIN; ++i) acc[i] = __fmaf_rn(x[i], y[(i + it) & 1 ? i : (N_CHAIN - 1 - i)], acc[i]);
    }
    float s = 0; for (int i = 0; i < N_CHAIN; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// one shared multiplicand per step (like a broadcast centroid value), reused by all chains
__global__ void k_reuse(float *out, const float *cb, int iters) {
    float acc[N_CHAIN], x[N_CHAIN];
    for (int i = 0; i < N_CHAIN; ++i) { acc[i] = g_seed[(threadIdx.x + i) & 63]; x[i] = g_seed[(i * 3 + threadIdx.x) & 63]; }
    float c0 = cb[0], c1 = cb[1];
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < N_CHAIN; ++i) acc[i] = __fmaf_rn(x[i], c0, acc[i]);
#pragma unroll
        for (int i = 0; i < N_CHAIN; ++i) acc[i] = __fmaf_rn(x[i], c1, acc[i]);
        c0 += 1e-7f; c1 -= 1e-7f;
    }
    float s = 0; for (int i = 0; i < N_CHAIN; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_imm(float *out, int iters) {
    float acc[N_CHAIN], x[N_CHAIN];
    for (int i = 0; i < N_CHAIN; ++i) { acc[i] = g_seed[(threadIdx.x + i) & 63]; x[i] = g_seed[(i * 3 + threadIdx.x) & 63]; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < N_CHAIN; ++i) acc[i] = __fmaf_rn(x[i], 1.00001f, acc[i]);
    }
    float s = 0; for (int i = 0; i < N_CHAIN; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__constant__ float kc[64];
__global__ void k_const(float *out, int iters) {
    float acc[N_CHAIN], x[N_CHAIN];
    for (int i = 0; i < N_CHAIN; ++i) { acc[i] = g_seed[(threadIdx.x + i) & 63]; x[i] = g_seed[(i * 3 + threadIdx.x) & 63]; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < N_CHAIN; ++i) acc[i] = __fmaf_rn(x[i], kc[i], acc[i]);
    }
    float s = 0; for (int i = 0; i < N_CHAIN; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// FFMA2 (paired fp32) via float2 fma: sm_100 has FFMA2?
__global__ void k_ffma2(float *out, const float *cb, int iters) {
    float2 acc[N_CHAIN / 2], x[N_CHAIN / 2];
    for (int i = 0; i < N_CHAIN / 2; ++i) { acc[i] = make_float2(g_seed[(threadIdx.x + i) & 63], g_seed[i]); x[i] = make_float2(g_seed[(i * 3 + threadIdx.x) & 63], g_seed[(i*7)&63]); }
    float2 c = make_float2(cb[0], cb[1]);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < N_CHAIN / 2; ++i) {
            float2 r;
            asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(*(unsigned long long*)&r) : "l"(*(unsigned long long*)&x[i]), "l"(*(unsigned long long*)&c), "l"(*(unsigned long long*)&acc[i]));
            acc[i] = r;
        }
        c.x += 1e-7f;
    }
    float s = 0; for (int i = 0; i < N_CHAIN / 2; ++i) s += acc[i].x + acc[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    float *out, *cb; cudaMalloc(&out, 148 * 64 * 1024 * 4); cudaMalloc(&cb, 256);
    float h[64]; for (int i = 0; i < 64; ++i) h[i] = 1.0f + i * 1e-5f;
    cudaMemcpy(cb, h, 256, cudaMemcpyHostToDevice); cudaMemcpyToSymbol(kc, h, 256); cudaMemcpyToSymbol(g_seed, h, 256);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int bpsm : {1, 2, 4}) for (int thr : {128, 256}) {
        dim3 g(sms * bpsm), b(thr);
        double flops = 2.0 * N_CHAIN * ITERS * (double)g.x * thr;
        const char *names[] = {"reg3", "reuse", "imm", "const", "ffma2"};
        for (int kk = 0; kk < 5; ++kk) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                if (kk == 0) k_reg3<<<g, b>>>(out, cb, ITERS);
                if (kk == 1) k_reuse<<<g, b>>>(out, cb, ITERS / 2);
                if (kk == 2) k_imm<<<g, b>>>(out, ITERS);
                if (kk == 3) k_const<<<g, b>>>(out, ITERS);
                if (kk == 4) k_ffma2<<<g, b>>>(out, cb, ITERS);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                if (rep == 1) printf("blocks/SM=%d thr=%d %-6s %.2f ms %.1f TFLOP/s\n", bpsm, thr, names[kk], ms, flops / ms / 1e9);
            }
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
