// conv_single.cu — kernel KS: single-channel direct convolution, strict FP32 on
// CUDA cores (§2.1 Eq. 2; the paper's single-channel
// kernel, §3.1, re-designed for sm_100a).
//
//   O[m][y][x] = sum_{r,c} I[y+r][x+c] * F[m][r][c]
//
// B200 design (not the paper's P/Q planner):
//  * One CTA = one output tile of TY rows x BX columns x R filters.  The
//    paper's "both feature maps and filters are divided" option
//    becomes the (x, y, m) grid; grids hold many waves of 148 SMs.
//  * The halo band I[y0 .. y0+TY+K-1)[x0 .. x0+BX+K-1) is staged once in
//    shared memory with coalesced loads (I is L2-resident: <= 200 KB).
//  * The R*K*K filter taps live in registers ("filters fully to registers",
//    P:665-667); every thread computes a TY x R register tile of one output
//    column, so each staged input value feeds up to K*R FMAs.
//  * Stores are the HBM-binding stream for K <= 3 (O is >= 94 % of all bytes
//    for Wx >= 56): each warp store writes 32 consecutive x of one (m, y) row
//    (128 B, fully coalesced), with the streaming .cs hint.
#include <cstdint>
#include "kernels.h"
#include "ptx.cuh"

namespace b200 {

template <int K, int R, int TY>
__global__ void __launch_bounds__(256)
ks_kernel(const float *__restrict__ I, int Wx, int Wy, const float *__restrict__ F, int M,
          float *__restrict__ O) {
    extern __shared__ float s_in[];                  // (TY+K-1) x SW
    const int Wo = Wx - K + 1, Ho = Wy - K + 1;
    const int BX = blockDim.x;
    const int SW = BX + K - 1;
    const int x0 = blockIdx.x * BX, y0 = blockIdx.y * TY, m0 = blockIdx.z * R;
    const int tx = threadIdx.x;

    // stage the halo band (zero outside the map; those lanes produce no output)
    const int n_in = (TY + K - 1) * SW;
    for (int idx = tx; idx < n_in; idx += BX) {
        const int rr = idx / SW, cc = idx - rr * SW;
        const int gy = y0 + rr, gx = x0 + cc;
        s_in[idx] = (gy < Wy && gx < Wx) ? __ldg(I + (int64_t)gy * Wx + gx) : 0.f;
    }
    // filter taps -> registers (warp-uniform addresses: broadcast loads)
    float w[R][K * K];
#pragma unroll
    for (int f = 0; f < R; ++f) {
        const bool ok = (m0 + f) < M;
        const float *Ff = F + (int64_t)(m0 + f) * K * K;
#pragma unroll
        for (int t = 0; t < K * K; ++t) w[f][t] = ok ? __ldg(Ff + t) : 0.f;
    }
    __syncthreads();

    float acc[TY][R];
#pragma unroll
    for (int ty = 0; ty < TY; ++ty)
#pragma unroll
        for (int f = 0; f < R; ++f) acc[ty][f] = 0.f;

    // input row iy feeds output row ty with filter row r = iy - ty
#pragma unroll
    for (int iy = 0; iy < TY + K - 1; ++iy) {
        float v[K];
#pragma unroll
        for (int c = 0; c < K; ++c) v[c] = s_in[iy * SW + tx + c];
#pragma unroll
        for (int ty = 0; ty < TY; ++ty) {
            const int r = iy - ty;
            if (r >= 0 && r < K) {
#pragma unroll
                for (int f = 0; f < R; ++f)
#pragma unroll
                    for (int c = 0; c < K; ++c) acc[ty][f] = fmaf(v[c], w[f][r * K + c], acc[ty][f]);
            }
        }
    }

    const int x = x0 + tx;
    if (x < Wo) {
#pragma unroll
        for (int f = 0; f < R; ++f) {
            if (m0 + f >= M) break;
            float *Of = O + (int64_t)(m0 + f) * Ho * Wo + x;
#pragma unroll
            for (int ty = 0; ty < TY; ++ty) {
                const int y = y0 + ty;
                if (y < Ho) st_cs(Of + (int64_t)y * Wo, acc[ty][f]);
            }
        }
    }
}

// Generic-K fallback (any K, e.g. K = Wx = Wy): no staging, loads through L1.
template <int R, int TY>
__global__ void __launch_bounds__(256)
ks_kernel_generic(const float *__restrict__ I, int Wx, int Wy, const float *__restrict__ F, int K,
                  int M, float *__restrict__ O) {
    const int Wo = Wx - K + 1, Ho = Wy - K + 1;
    const int x0 = blockIdx.x * blockDim.x, y0 = blockIdx.y * TY, m0 = blockIdx.z * R;
    const int x = x0 + threadIdx.x;
    if (x >= Wo) return;
    float acc[TY][R];
#pragma unroll
    for (int ty = 0; ty < TY; ++ty)
#pragma unroll
        for (int f = 0; f < R; ++f) acc[ty][f] = 0.f;
#pragma unroll
    for (int ty = 0; ty < TY; ++ty) {
        const int y = min(y0 + ty, Ho - 1);
        for (int r = 0; r < K; ++r)
            for (int c = 0; c < K; ++c) {
                const float v = __ldg(I + (int64_t)(y + r) * Wx + x + c);
#pragma unroll
                for (int f = 0; f < R; ++f) {
                    const int m = min(m0 + f, M - 1);
                    acc[ty][f] = fmaf(v, __ldg(F + ((int64_t)m * K + r) * K + c), acc[ty][f]);
                }
            }
    }
    for (int f = 0; f < R && m0 + f < M; ++f)
#pragma unroll
        for (int ty = 0; ty < TY; ++ty)
            if (y0 + ty < Ho) st_cs(O + ((int64_t)(m0 + f) * Ho + y0 + ty) * Wo + x, acc[ty][f]);
}

namespace {
struct KsCfg { int R, TY; };
// (R filters, TY rows) per thread: registers = R*K*K taps + TY*R accumulators.
KsCfg ks_cfg(int K) {
    switch (K) {
        case 1: return {8, 8};
        case 2: return {8, 4};
        case 3: return {8, 4};
        case 4: return {4, 8};
        case 5: return {4, 8};
        case 6: return {2, 8};
        case 7: return {2, 8};
        default: return {4, 4};
    }
}
int ks_bx(int Wo) {
    int bx = ((Wo + 31) / 32) * 32;
    return bx > 256 ? 256 : bx;
}
}  // namespace

int plan_single(int Wx, int Wy, int K, int M, conv_plan *p) {
    const int Wo = Wx - K + 1, Ho = Wy - K + 1;
    const KsCfg c = ks_cfg(K);
    const int bx = ks_bx(Wo);
    p->kernel = 0;
    p->block_x = bx;
    p->grid_x = (Wo + bx - 1) / bx;
    p->grid_y = (Ho + c.TY - 1) / c.TY;
    p->grid_z = (M + c.R - 1) / c.R;
    p->cluster_x = 1;
    p->tile_m = c.R;
    p->tile_n = bx * c.TY;
    p->smem_bytes = (K <= 7) ? (c.TY + K - 1) * (bx + K - 1) * 4 : 0;
    p->tma_f = 0;
    return 0;
}

template <int K>
static cudaError_t launch_ks(const conv_plan &p, const float *I, int Wx, int Wy, const float *F,
                             int M, float *O, cudaStream_t s) {
    constexpr int R = (K == 1 || K == 2 || K == 3) ? 8 : (K == 4 || K == 5) ? 4 : 2;
    constexpr int TY = (K == 2 || K == 3) ? 4 : 8;
    auto kern = ks_kernel<K, R, TY>;
    if (p.smem_bytes > 48 * 1024)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem_bytes);
    kern<<<dim3(p.grid_x, p.grid_y, p.grid_z), p.block_x, p.smem_bytes, s>>>(I, Wx, Wy, F, M, O);
    return cudaGetLastError();
}

cudaError_t launch_single(const float *I, int Wx, int Wy, const float *F, int K, int M, float *O,
                          cudaStream_t s) {
    conv_plan p;
    plan_single(Wx, Wy, K, M, &p);
    switch (K) {
        case 1: return launch_ks<1>(p, I, Wx, Wy, F, M, O, s);
        case 2: return launch_ks<2>(p, I, Wx, Wy, F, M, O, s);
        case 3: return launch_ks<3>(p, I, Wx, Wy, F, M, O, s);
        case 4: return launch_ks<4>(p, I, Wx, Wy, F, M, O, s);
        case 5: return launch_ks<5>(p, I, Wx, Wy, F, M, O, s);
        case 6: return launch_ks<6>(p, I, Wx, Wy, F, M, O, s);
        case 7: return launch_ks<7>(p, I, Wx, Wy, F, M, O, s);
        default: {
            ks_kernel_generic<4, 4><<<dim3(p.grid_x, p.grid_y, p.grid_z), p.block_x, 0, s>>>(
                I, Wx, Wy, F, K, M, O);
            return cudaGetLastError();
        }
    }
}

}  // namespace b200
