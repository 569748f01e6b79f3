// ffma2_rate.cu — register-only FP32 FMA throughput of the KM-SIMT thread tile
// (8 filters x 6 pixels, FFMA2 with a broadcast scalar) against other forms,
// at 4 and 8 warps per SM sub-partition.  No memory traffic in the loop.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2212_00404_b200/csrc
//        tools/probes/ffma2_rate.cu -o tools/probes/bin/ffma2_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace b200;

__device__ __forceinline__ void ffma2p(float &d0, float &d1, float a0, float a1, float b0, float b1) {
    uint64_t d, av, bv;
    asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(d0), "f"(d1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(av) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(bv) : "f"(b0), "f"(b1));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(av), "l"(bv));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(d));
}

// MODE 0: FFMA2 scalar-broadcast a, 8 x 6 tile (the KM-SIMT form)
// MODE 1: FFMA2 with a as a duplicated pair
// MODE 2: plain FFMA, 8 x 6
// MODE 3: FFMA2 scalar a, 8 x 8 tile
// MODE 4: FFMA2 scalar a, 4 x 12 tile (fewer distinct a, longer b)
template <int MODE>
__global__ void __launch_bounds__(256) rate_kernel(const float *in, float *out, int iters) {
    constexpr int TM = MODE == 4 ? 4 : 8, TN = MODE == 3 ? 8 : (MODE == 4 ? 12 : 6);
    float acc[TM][TN];
    float a[TM], b[TN];
#pragma unroll
    for (int i = 0; i < TM; ++i) a[i] = in[(threadIdx.x + i) & 63];
#pragma unroll
    for (int j = 0; j < TN; ++j) b[j] = in[(threadIdx.x + 7 * j) & 63];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
            for (int i = 0; i < TM; ++i) {
#pragma unroll
                for (int j = 0; j < TN; j += 2) {
                    if (MODE == 2) {
                        acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
                        acc[i][j + 1] = fmaf(a[i], b[j + 1], acc[i][j + 1]);
                    } else if (MODE == 1) {
                        ffma2p(acc[i][j], acc[i][j + 1], a[i], a[i], b[j], b[j + 1]);
                    } else {
                        ffma2(acc[i][j], acc[i][j + 1], a[i], b[j], b[j + 1]);
                    }
                }
            }
            // perturb operands so nothing is loop-invariant
#pragma unroll
            for (int i = 0; i < TM; ++i) a[i] = __int_as_float(__float_as_int(a[i]) ^ 1);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) s += acc[i][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(const char *name, float *in, float *out, int ctas_per_sm) {
    constexpr int TM = MODE == 4 ? 4 : 8, TN = MODE == 3 ? 8 : (MODE == 4 ? 12 : 6);
    const int iters = 4000, grid = 148 * ctas_per_sm;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    rate_kernel<MODE><<<grid, 256>>>(in, out, 10);
    cudaEventRecord(e0);
    rate_kernel<MODE><<<grid, 256>>>(in, out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double fma = (double)grid * 256 * iters * 4 * TM * TN;
    const double peak = 148.0 * 128 * clk * 1e3;    // FMA / s at the max clock
    printf("%-34s ctas/SM %d: %8.3f ms  %6.2f TFMA/s  = %5.1f %% of 128 FMA/clk/SM @ %d MHz  (%s)\n", name,
           ctas_per_sm, ms, fma / (ms * 1e-3) / 1e12, 100.0 * fma / (ms * 1e-3) / peak, clk / 1000,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    float *in, *out;
    cudaMalloc(&in, 64 * 4);
    cudaMemset(in, 0, 64 * 4);
    cudaMalloc(&out, 148 * 8 * 256 * 4);
    for (int c : {2, 4}) {
        run<0>("FFMA2 scalar-a 8x6 (KM-SIMT)", in, out, c);
        run<1>("FFMA2 pair-a 8x6", in, out, c);
        run<2>("FFMA 8x6", in, out, c);
        run<3>("FFMA2 scalar-a 8x8", in, out, c);
        run<4>("FFMA2 scalar-a 4x12", in, out, c);
    }
    return 0;
}
