// conv_single.cu — kernel KS: single-channel direct convolution, strict FP32 on
// CUDA cores (§2.1 Eq. 2; the paper's single-channel
// kernel, §3.1, re-designed for sm_100a).
//
//   O[m][y][x] = sum_{r,c} I[y+r][x+c] * F[m][r][c]
//
// For K <= 3 the output stream (O is >= 94 % of all bytes for Wx >= 56) binds
// to HBM; for K >= 5 the FP32 FMA pipe binds.  Design:
//  * One CTA owns a band of TY full output rows and a chunk of filters.  Because
//    the band spans whole rows, O[m][y0 : y0+TY][:] is ONE contiguous range of
//    TY*Wo floats per filter.  The paper's "only the feature maps are divided
//    ... processed by all filters" option at CTA level: the halo
//    band I[y0 .. y0+TY+K-1) is staged once in shared memory and reused for
//    every filter of the chunk ("FMA operations per loaded data").
//  * Filters are processed in groups of R; their taps sit in registers
//    ("filters fully to registers").  Each thread computes R filters
//    x 4 consecutive pixels (16-B shared loads of the input window, sliding
//    window reuse across the K taps of a row).
//  * Results go to a double-buffered shared-memory image of the contiguous
//    output range (laid out so that smem and global addresses agree mod 16 B)
//    and leave through ONE bulk TMA store per filter (cp.async.bulk
//    shared->global): the write stream costs no per-element instructions.
//    The <= 3 unaligned head/tail elements of a range are stored by threads.
#include <cstdint>
#include "kernels.h"
#include "ptx.cuh"

namespace b200 {

constexpr int kKsThreads = 256;
constexpr int kKsWarps = kKsThreads / 32;

// One work item = (row block, filter group): a warp computes RI output rows
// x R filters.  Normal mode (rows >= 16 px): lane l owns TX consecutive pixels of
// RR rows (vertical register blocking: an input row feeds up to min(RR, K)
// output rows).  Small-map mode (TX == 1, Wo <= 16): the warp's lanes cover
// RW = 32 / Wo whole rows, one pixel each.  Warps run independently after the
// staging barrier: each writes its tile into a warp-private double-buffered
// smem image of the contiguous global range O[m][y : y+RI][:], and lanes
// 0..R-1 each stream one filter's range out with a bulk store.
template <int K, int R, int TX, int RR>
__global__ void __launch_bounds__(kKsThreads)
ks_kernel(const float *__restrict__ I, int Wx, int Wy, const float *__restrict__ F, int M,
          float *__restrict__ O, int m_per_cta, int TY) {
    constexpr int KK = K * K;
    constexpr int GS = (R * KK + 3) & ~3;            // floats per filter group (16-B rows)
    constexpr int WN = TX + K - 1;                   // input window per lane and row
    extern __shared__ __align__(16) float smem[];
    const int Wo = Wx - K + 1, Ho = Wy - K + 1;
    const int RW = (TX == 1 && Wo <= 16) ? 32 / Wo : 1;      // small-map rows per warp
    const int RI = RW > 1 ? RW : RR;                          // output rows per item
    const int SW = ((RW > 1 ? Wx : 32 * TX + K - 1) + 3) & ~3;
    const int y0 = blockIdx.y * TY;
    const int rows = min(TY, Ho - y0);
    const int n_ri = (rows + RI - 1) / RI;
    const int CHW = ((RI * Wo + 3) & ~3) + 4;        // smem floats per (filter) output image
    const int mc0 = blockIdx.x * m_per_cta;
    const int mc1 = min(M, mc0 + m_per_cta);
    const int ngroups = (mc1 - mc0 + R - 1) / R;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t plane = (int64_t)Ho * Wo;

    float *s_w = smem;                                           // [groups][GS]
    float *s_in = s_w + ((m_per_cta + R - 1) / R) * GS;          // (TY+K-1) x SW
    float *s_out = s_in + (TY + K - 1) * SW + warp * 2 * R * CHW; // this warp: [2][R][CHW]

    pdl_wait();
    // stage taps and the halo band with fire-and-forget cp.async (zero-filled
    // outside the map), one wait for all of them
    for (int idx = tid; idx < ngroups * GS; idx += kKsThreads) {
        const int g = idx / GS, e = idx - g * GS;
        const int f = e / KK, t = e - f * KK;
        const int m = mc0 + g * R + f;
        const bool ok = f < R && m < mc1;
        cp_async4(s_w + idx, ok ? F + (int64_t)m * KK + t : F, ok);
    }
    const int hr = rows + K - 1;
    for (int rr = warp; rr < TY + K - 1; rr += kKsWarps) {
        const float *src = I + (int64_t)(y0 + rr) * Wx;
        for (int cc = lane; cc < SW; cc += 32) {
            const bool ok = rr < hr && cc < Wx;
            cp_async4(s_in + rr * SW + cc, ok ? src + cc : I, ok);
        }
    }
    cp_async_commit();
    pdl_trigger();
    cp_async_wait<0>();
    __syncthreads();

    // lane -> (row within the item, first pixel)
    int lrow, lx;
    if (RW > 1) { lrow = lane / Wo; lx = lane - lrow * Wo; }
    else        { lrow = 0;         lx = lane * TX; }
    const bool lane_ok = (RW > 1) ? (lrow < RW) : (lx < Wo);
    const bool lane_full = (RW > 1) || (lx + TX <= Wo);       // no per-pixel bounds checks

    const int n_items = n_ri * ngroups;
    int local = 0;
    for (int it = warp; it < n_items; it += kKsWarps, ++local) {
        const int ri = it % n_ri, g = it / n_ri;
        float *ob = s_out + (local & 1) * R * CHW;
        if (local >= 2) {
            if (lane < R) bulk_wait_read<1>();        // this lane's store of 2 items ago read ob
            __syncwarp();
        }
        const int yb = ri * RI;                       // first band row of this item
        const int nrows = min(RI, rows - yb);         // rows in this item
        const int len = nrows * Wo;                   // contiguous floats per filter
        const int m0 = mc0 + g * R;
        const int64_t g00 = ((int64_t)m0 * Ho + y0 + yb) * Wo;   // range start of filter m0
        if (lane_ok && lrow < nrows) {
            float w[GS];
#pragma unroll
            for (int q = 0; q < GS / 4; ++q) {
                const float4 v = *reinterpret_cast<const float4 *>(s_w + g * GS + 4 * q);
                w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
            }
            constexpr int RL = RR;                    // rows computed per lane (1 in small mode)
            const int nr = (RW > 1) ? 1 : nrows;      // valid rows of this lane's block
            float acc[RL][R][TX];
#pragma unroll
            for (int q = 0; q < RL; ++q)
#pragma unroll
                for (int f = 0; f < R; ++f)
#pragma unroll
                    for (int j = 0; j < TX; ++j) acc[q][f][j] = 0.f;
            const float *base = s_in + (yb + lrow) * SW + lx;
#pragma unroll
            for (int ir = 0; ir < RL + K - 1; ++ir) {
                float win[WN];
#pragma unroll
                for (int u = 0; u < WN; ++u) win[u] = base[ir * SW + u];
#pragma unroll
                for (int q = 0; q < RL; ++q) {
                    const int r = ir - q;             // filter row feeding output row q
                    if (r >= 0 && r < K) {
#pragma unroll
                        for (int c = 0; c < K; ++c)
#pragma unroll
                            for (int f = 0; f < R; ++f)
#pragma unroll
                                for (int j = 0; j < TX; ++j)
                                    acc[q][f][j] = fmaf(win[j + c], w[f * KK + r * K + c], acc[q][f][j]);
                    }
                }
            }
            const int e = lrow * Wo + lx;
#pragma unroll
            for (int f = 0; f < R; ++f) {
                float *d = ob + f * CHW + (int)((g00 + (int64_t)f * plane) & 3) + e;
#pragma unroll
                for (int q = 0; q < RL; ++q) {
                    if (q < nr) {
                        if (lane_full) {
#pragma unroll
                            for (int j = 0; j < TX; ++j) d[q * Wo + j] = acc[q][f][j];
                        } else {
#pragma unroll
                            for (int j = 0; j < TX; ++j)
                                if (lx + j < Wo) d[q * Wo + j] = acc[q][f][j];
                        }
                    }
                }
            }
        }
        fence_proxy_async_smem();                     // smem image -> visible to the bulk copy
        __syncwarp();
        // lane f < R: bulk store of filter f's 16-B aligned body; all lanes: the
        // <= 3 head and <= 3 tail elements (or a whole range shorter than 8)
        if (lane < R) {
            if (m0 + lane < mc1) {
                const int64_t g0 = g00 + (int64_t)lane * plane;
                const int64_t a0 = (g0 + 3) & ~(int64_t)3, a1 = (g0 + len) & ~(int64_t)3;
                if (a1 > a0)
                    bulk_store(O + a0, ob + lane * CHW + (int)(g0 & 3) + (int)(a0 - g0),
                               (uint32_t)((a1 - a0) * 4));
            }
            bulk_commit();
        }
        for (int t = lane; t < 8 * R; t += 32) {
            const int f = t >> 3, j = t & 7;
            if (m0 + f >= mc1) continue;
            const int64_t g0 = g00 + (int64_t)f * plane;
            const int64_t a0 = (g0 + 3) & ~(int64_t)3, a1 = (g0 + len) & ~(int64_t)3;
            int64_t gi = -1;
            if (a1 > a0) {
                if (j < 4) { if (g0 + j < a0) gi = g0 + j; }
                else if (a1 + (j - 4) < g0 + len) gi = a1 + (j - 4);
            } else if (j < len) {
                gi = g0 + j;
            }
            if (gi >= 0) O[gi] = ob[f * CHW + (int)(g0 & 3) + (int)(gi - g0)];
        }
    }
    if (lane < R) bulk_wait<0>();                     // keep smem alive until the copies finish
}

// Generic fallback (any K, e.g. K = Wx = Wy, or rows too wide for smem): no
// staging, loads through L1.
template <int R, int TY>
__global__ void __launch_bounds__(256)
ks_kernel_generic(const float *__restrict__ I, int Wx, int Wy, const float *__restrict__ F, int K,
                  int M, float *__restrict__ O) {
    const int Wo = Wx - K + 1, Ho = Wy - K + 1;
    const int x0 = blockIdx.x * blockDim.x, y0 = blockIdx.y * TY, m0 = blockIdx.z * R;
    const int x = x0 + threadIdx.x;
    pdl_wait();
    pdl_trigger();
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
constexpr int kKsMaxSmem = 110 * 1024;

// (R filters, RR rows) per lane and item: K=1 store-bound -> more filters;
// K>=5 FMA-bound -> more rows (an input row feeds min(RR, K) output rows)
__host__ __device__ constexpr int ks_R(int K) { return K <= 1 ? 4 : (K <= 5 ? 2 : 1); }
__host__ __device__ constexpr int ks_RR(int K) { return K <= 1 ? 1 : (K <= 5 ? 2 : 4); }
int ks_TX(int Wo) { return (Wo + 31) / 32; }
int ks_smem(int K, int R, int TX, int TY, int Wx, int Wo, int m_per) {
    const int RW = (TX == 1 && Wo <= 16) ? 32 / Wo : 1;
    const int RI = RW > 1 ? RW : ks_RR(K);
    const int SW = ((RW > 1 ? Wx : 32 * TX + K - 1) + 3) & ~3;
    const int GS = (R * K * K + 3) & ~3;
    const int CHW = ((RI * Wo + 3) & ~3) + 4;
    return (((m_per + R - 1) / R) * GS + (TY + K - 1) * SW + kKsWarps * 2 * R * CHW) * 4;
}
}  // namespace

int plan_single(int Wx, int Wy, int K, int M, conv_plan *p) {
    const int Wo = Wx - K + 1, Ho = Wy - K + 1;
    p->cluster_x = 1;
    p->tma_f = 0;
    p->launches = 1;
    const int TX = ks_TX(Wo);
    if (K <= 7 && TX <= 8) {
        const int R = ks_R(K);
        // (band rows TY, filters per CTA m_per): minimise waves x work per CTA on
        // 148 SMs x 2 CTAs (+ a per-CTA staging cost), i.e. avoid a ragged last wave
        const int slots = 2 * kNumSMs;
        int TY = Ho < 16 ? Ho : 16, m_per = R;
        double best = -1.0;
        for (int ty : {8, 16}) {
            const int t = Ho < ty ? Ho : ty;
            const int nb = (Ho + t - 1) / t;
            for (int mp = R; mp < M + R; mp += R) {
                const int ctas = nb * ((M + mp - 1) / mp);
                const int waves = (ctas + slots - 1) / slots;
                const double cost = waves * ((double)t * mp + 4.0 * (t + K - 1));
                if (best < 0 || cost < best - 1e-9) { best = cost; TY = t; m_per = mp; }
                if (ctas <= slots) break;                 // larger chunks only lengthen the wave
            }
            if (Ho <= ty) break;
        }
        const int bands = (Ho + TY - 1) / TY;
        p->kernel = 0;
        p->block_x = kKsThreads;
        p->grid_x = (M + m_per - 1) / m_per;
        p->grid_y = bands;
        p->grid_z = 1;
        p->tile_m = m_per;                               // filters per CTA (groups of R)
        p->tile_n = TY;                                  // output rows per CTA band (full width)
        p->smem_bytes = ks_smem(K, R, TX, TY, Wx, Wo, m_per);
        if (p->smem_bytes <= kKsMaxSmem) return 0;
    }
    // generic fallback: (x, y, m) tiles of 1 column x 4 rows x 4 filters per thread
    const int bx = Wo >= 128 ? 128 : ((Wo + 31) / 32) * 32;
    p->kernel = 0;
    p->block_x = bx;
    p->grid_x = (Wo + bx - 1) / bx;
    p->grid_y = (Ho + 3) / 4;
    p->grid_z = (M + 3) / 4;
    p->tile_m = 4;
    p->tile_n = -1;                                      // marks the generic kernel
    p->smem_bytes = 0;
    return 0;
}

static cudaLaunchAttribute pdl_attr() {
    cudaLaunchAttribute a;
    a.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a.val.programmaticStreamSerializationAllowed = pdl_enabled();
    return a;
}

template <int K, int TX>
static cudaError_t launch_ks(const conv_plan &p, const float *I, int Wx, int Wy, const float *F,
                             int M, float *O, cudaStream_t s) {
    auto kern = ks_kernel<K, ks_R(K), TX, ks_RR(K)>;
    if (p.smem_bytes > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             p.smem_bytes);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.grid_x, p.grid_y, p.grid_z);
    cfg.blockDim = dim3(p.block_x);
    cfg.dynamicSmemBytes = p.smem_bytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1] = {pdl_attr()};
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, I, Wx, Wy, F, M, O, p.tile_m, p.tile_n);
}

template <int K>
static cudaError_t launch_ks_v(const conv_plan &p, const float *I, int Wx, int Wy, const float *F,
                               int M, float *O, cudaStream_t s) {
    switch (ks_TX(Wx - K + 1)) {
        case 1: return launch_ks<K, 1>(p, I, Wx, Wy, F, M, O, s);
        case 2: return launch_ks<K, 2>(p, I, Wx, Wy, F, M, O, s);
        case 3: return launch_ks<K, 3>(p, I, Wx, Wy, F, M, O, s);
        case 4: return launch_ks<K, 4>(p, I, Wx, Wy, F, M, O, s);
        case 5: return launch_ks<K, 5>(p, I, Wx, Wy, F, M, O, s);
        case 6: return launch_ks<K, 6>(p, I, Wx, Wy, F, M, O, s);
        case 7: return launch_ks<K, 7>(p, I, Wx, Wy, F, M, O, s);
        default: return launch_ks<K, 8>(p, I, Wx, Wy, F, M, O, s);
    }
}

cudaError_t launch_single(const float *I, int Wx, int Wy, const float *F, int K, int M, float *O,
                          cudaStream_t s) {
    conv_plan p;
    plan_single(Wx, Wy, K, M, &p);
    if (p.tile_n > 0) {
        switch (K) {
            case 1: return launch_ks_v<1>(p, I, Wx, Wy, F, M, O, s);
            case 2: return launch_ks_v<2>(p, I, Wx, Wy, F, M, O, s);
            case 3: return launch_ks_v<3>(p, I, Wx, Wy, F, M, O, s);
            case 4: return launch_ks_v<4>(p, I, Wx, Wy, F, M, O, s);
            case 5: return launch_ks_v<5>(p, I, Wx, Wy, F, M, O, s);
            case 6: return launch_ks_v<6>(p, I, Wx, Wy, F, M, O, s);
            case 7: return launch_ks_v<7>(p, I, Wx, Wy, F, M, O, s);
            default: break;
        }
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.grid_x, p.grid_y, p.grid_z);
    cfg.blockDim = dim3(p.block_x);
    cfg.stream = s;
    cudaLaunchAttribute attr[1] = {pdl_attr()};
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, ks_kernel_generic<4, 4>, I, Wx, Wy, F, K, M, O);
}

}  // namespace b200
