// Shared-memory atomic throughput on B200: float64 add vs uint64 add vs uint32 add, 256 clusters x 8
// coordinates, random cluster per point (the Lloyd accumulation pattern).  nvcc -arch=sm_100a
#include <cstdio>
#include <cstdint>
template <int KIND>
__global__ void kern(const uint32_t *lab, int n, double *out) {
    __shared__ double sd[2048];
    __shared__ unsigned long long su[2048];
    __shared__ unsigned su32[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) { sd[i] = 0; su[i] = 0; su32[i] = 0; }
    __syncthreads();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t l = lab[i] & 255;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            if (KIND == 0) atomicAdd(&sd[l * 8 + t], (double)(i & 1023));
            if (KIND == 1) atomicAdd(&su[l * 8 + t], (unsigned long long)(i & 1023));
            if (KIND == 2) atomicAdd(&su32[l * 8 + t], (unsigned)(i & 1023));
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) out[blockIdx.x * 2048 + i] = sd[i] + su[i] + su32[i];
}
int main() {
    const int n = 12000000;
    uint32_t *lab; double *out;
    cudaMalloc(&lab, n * 4); cudaMalloc(&out, 148 * 8 * 2048 * 8);
    uint32_t *h = new uint32_t[n];
    uint32_t s = 1; for (int i = 0; i < n; ++i) { s = s * 1664525u + 1013904223u; h[i] = s >> 8; }
    cudaMemcpy(lab, h, n * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int kind = 0; kind < 3; ++kind) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            if (kind == 0) kern<0><<<148 * 4, 256>>>(lab, n, out);
            if (kind == 1) kern<1><<<148 * 4, 256>>>(lab, n, out);
            if (kind == 2) kern<2><<<148 * 4, 256>>>(lab, n, out);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep == 2) printf("kind %d (%s): %.3f ms for %d points x 8 atomics = %.2f Gatom/s\n", kind,
                                 kind == 0 ? "f64 add" : kind == 1 ? "u64 add" : "u32 add", ms, n, n * 8.0 / ms / 1e6);
        }
    }
    return 0;
}
