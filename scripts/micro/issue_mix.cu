// Issue-slot model of one SM sub-partition (sm_100a): how many FMA-pipe instructions fit beside a
// stream of half-rate ALU-pipe FMNMX3?  Loops of NA FMNMX3 + NF FFMA (independent chains), W warps per
// sub-partition, one CTA per SM.  Prints warp-instructions per clock per sub-partition.
#include <cstdio>
#include <cuda_runtime.h>
__device__ float g_seed[64];
__device__ __forceinline__ float fmin3(float a, float b, float c) { float d; asm volatile("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }
__device__ __forceinline__ float ffma(float a, float b, float c) { float d; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }
template <int NA, int NF>
__global__ void k_mix(float *out, int iters, long long *cyc) {
    float a[16], f[16];
    for (int i = 0; i < 16; ++i) { a[i] = g_seed[(i + threadIdx.x) & 63]; f[i] = g_seed[(i * 3 + threadIdx.x) & 63]; }
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
#pragma unroll
            for (int i = 0; i < (NA > NF ? NA : NF); ++i) {
                if (i < NA) a[i & 15] = fmin3(a[i & 15], a[(i + 3) & 15], a[(i + 7) & 15]);
                if (i < NF) f[i & 15] = ffma(f[i & 15], 1.0001f, f[(i + 5) & 15]);
            }
        }
    }
    const long long t1 = clock64();
    float s = 0; for (int i = 0; i < 16; ++i) s += a[i] + f[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int NA, int NF>
void run(int warps_per_smsp, float *out, long long *dcyc) {
    const int iters = 4096;
    k_mix<NA, NF><<<148, 128 * warps_per_smsp>>>(out, iters, dcyc);
    k_mix<NA, NF><<<148, 128 * warps_per_smsp>>>(out, iters, dcyc);
    long long c; cudaMemcpy(&c, dcyc, 8, cudaMemcpyDeviceToHost);
    const double instr = (double)iters * 4 * (NA + NF) * warps_per_smsp;  // per sub-partition
    printf("W=%d  ALU %2d : FMA %2d   %.3f instr/clk/SMSP   ALU %.3f/clk  FMA %.3f/clk\n", warps_per_smsp, NA, NF, instr / c,
           (double)iters * 4 * NA * warps_per_smsp / c, (double)iters * 4 * NF * warps_per_smsp / c);
}
int main() {
    float *out; cudaMalloc(&out, 148 * 1024 * 4); long long *dcyc; cudaMalloc(&dcyc, 8);
    float h[64]; for (int i = 0; i < 64; ++i) h[i] = 1000.0f + i; cudaMemcpyToSymbol(g_seed, h, 256);
    for (int w = 1; w <= 4; ++w) {
        if (w == 2) continue;
        run<16, 0>(w, out, dcyc); run<0, 16>(w, out, dcyc); run<16, 4>(w, out, dcyc); run<16, 8>(w, out, dcyc);
        run<16, 16>(w, out, dcyc); run<8, 16>(w, out, dcyc);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
