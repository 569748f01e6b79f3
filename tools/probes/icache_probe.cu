// Instruction-fetch probe: straight-line code vs a loop with the same dynamic
// instruction count (one CTA per SM).  nvcc -arch=sm_100a -O3 icache_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int N>
__device__ __forceinline__ void chain(float (&a)[8]) {
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], 1.0001f, 0.5f);
}

__global__ void straight(float *out, float x) {
    float a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = x + j;
    chain<512>(a);                       // 4096 FFMA, ~64 KB of SASS
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += a[j];
    if (s == 123.f) out[threadIdx.x] = s;
}

__global__ void looped(float *out, float x, int n) {
    float a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = x + j;
    for (int it = 0; it < n; ++it) chain<8>(a);   // n * 64 FFMA
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += a[j];
    if (s == 123.f) out[threadIdx.x] = s;
}

__global__ void evict(float *buf, size_t n) {   // stream through a big buffer (evicts L2)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        buf[i] = buf[i] * 0.5f + 1.f;
}

int main() {
    float *out, *big;
    size_t nbig = 256ull << 20;   // 1 GB
    cudaMalloc(&out, 4096);
    cudaMalloc(&big, nbig * 4);
    cudaMemset(big, 0, nbig * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int ctas : {1, 148}) {
        for (int ev = 0; ev < 2; ++ev) {
            for (int rep = 0; rep < 3; ++rep) {
                float ts, tl;
                if (ev) evict<<<1184, 512>>>(big, nbig);
                cudaEventRecord(e0);
                straight<<<ctas, 128>>>(out, 1.f);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ts, e0, e1);
                if (ev) evict<<<1184, 512>>>(big, nbig);
                cudaEventRecord(e0);
                looped<<<ctas, 128>>>(out, 1.f, 64);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&tl, e0, e1);
                printf("ctas %3d evictL2 %d rep %d: straight %.2f us, looped %.2f us\n", ctas, ev, rep, ts * 1e3, tl * 1e3);
            }
        }
    }
    return 0;
}
