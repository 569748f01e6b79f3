// conv_multi_simt.cu — kernel KM-SIMT: multi-channel direct convolution in
// strict FP32 on CUDA cores (§2.1 Eq. 1; the paper's
// stride-fixed-block kernel, §3.2, re-designed for sm_100a).
//
//   O[m][y][x] = sum_{ch,r,c} I[ch][y+r][x+c] * F[m][ch][r][c]
//
// Design:
//  * Output tile = BM filters x BN "wide" pixels.  A wide pixel p = y*Wx + x
//    runs over the full input width (x in [0, Wx)); columns x >= Wo are
//    computed and discarded.  With that indexing the input patch a tile needs
//    for one channel is ONE contiguous range I[ch][p0 .. p0+BN+(K-1)*Wx+K-1),
//    so staging is a plain 1-D copy for any alignment.
//  * The reduction runs over channel chunks of CB channels (the paper's
//    "segment along ch" of S bytes per filter, with S = CB*K*K*4 B),
//    double-buffered with cp.async (the paper's prefetch rounds).
//  * F chunks are stored transposed in smem (k-major, m contiguous) so each
//    thread reads its 8 filters with two 16-B loads; each thread owns an 8x8
//    register tile (8 filters x 8 pixels strided by BN/8 -> conflict-free).
//  * Small layers cannot fill 148 SMs with output tiles, so the channel sum is
//    split across a thread-block cluster of S CTAs (the paper's rejected
//    Fig. 2(b) split along ch): partial tiles are reduced through
//    distributed shared memory in fixed rank order (deterministic, no global
//    atomics, O written once) instead of through global memory.
#include <cstdint>
#include "kernels.h"
#include "ptx.cuh"

namespace b200 {


constexpr int kSimtBM = 64;
constexpr int kSimtBN = 128;

// channels per staged chunk (the paper's segment S = CB*K*K*4 bytes per filter)
__host__ __device__ constexpr int simt_cb(int K) { return (K == 1 || K == 3) ? 8 : (K == 5 ? 4 : 2); }
constexpr int kSimtMaxSmem = 200 * 1024;

// Fallback for shapes whose staged patch exceeds shared memory (very large K,
// e.g. K = Wx = Wy): one thread per output, loads through L1, same sum order.
__global__ void __launch_bounds__(256)
kmn_kernel(const float *__restrict__ I, int C, int Wx, int Wy, const float *__restrict__ F, int K,
           int M, float *__restrict__ O) {
    const int Ho = Wy - K + 1, Wo = Wx - K + 1;
    const int64_t n = (int64_t)M * Ho * Wo;
    pdl_wait();
    pdl_trigger();
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < n;
         o += (int64_t)gridDim.x * blockDim.x) {
        const int m = (int)(o / ((int64_t)Ho * Wo));
        const int rem = (int)(o - (int64_t)m * Ho * Wo);
        const int y = rem / Wo, x = rem - y * Wo;
        float acc = 0.f;
        for (int ch = 0; ch < C; ++ch) {
            const float *Ic = I + (int64_t)ch * Wx * Wy + (int64_t)y * Wx + x;
            const float *Fc = F + ((int64_t)m * C + ch) * K * K;
            for (int r = 0; r < K; ++r)
                for (int c = 0; c < K; ++c) acc = fmaf(__ldg(Ic + (int64_t)r * Wx + c), __ldg(Fc + r * K + c), acc);
        }
        O[o] = acc;
    }
}

// KT = compile-time K (1..7) or 0 for a runtime K.
template <int KT, int BM, int BN, int CB>
__global__ void __launch_bounds__((BM / 8) * (BN / 8))
kms_kernel(const float *__restrict__ I, int C, int Wx, int Wy, const float *__restrict__ F,
           int Krt, int M, float *__restrict__ O, int ch_per_split, int NP) {
    constexpr int NT = (BM / 8) * (BN / 8);
    constexpr int TNS = BN / 8;                     // pixel stride inside a thread tile
    constexpr int FS = BM + 4;                      // transposed-F row stride (floats)
    const int K = KT > 0 ? KT : Krt;
    const int KK = K * K;
    const int Ho = Wy - K + 1, Wo = Wx - K + 1;
    const int HW = Wx * Wy;
    const int Ktot = C * KK;

    extern __shared__ __align__(16) float smem[];
    const int f_floats = CB * KK * FS;
    const int i_floats = CB * NP;
    const int buf_floats = f_floats + i_floats;     // buffer b: F at b*buf, I at b*buf + f

    const int S = gridDim.x;                        // cluster size == split
    const int split = blockIdx.x;
    const int p0 = blockIdx.y * BN;
    const int m0 = blockIdx.z * BM;
    const int ch_begin = split * ch_per_split;
    const int ch_end = min(C, ch_begin + ch_per_split);
    const int nchunks = ch_end > ch_begin ? (ch_end - ch_begin + CB - 1) / CB : 0;
    const int tid = threadIdx.x;
    const int tn = tid % TNS, tm = tid / TNS;

    auto load_chunk = [&](int chunk, int b) {
        const int ch0 = ch_begin + chunk * CB;
        const int nk = CB * KK;
        for (int idx = tid; idx < BM * nk; idx += NT) {
            const int m = idx / nk, kk = idx - m * nk;
            const bool ok = (m0 + m < M) && (ch0 * KK + kk < ch_end * KK);
            const float *src = ok ? F + (int64_t)(m0 + m) * Ktot + ch0 * KK + kk : F;
            cp_async4(smem + b * buf_floats + kk * FS + m, src, ok);
        }
        for (int idx = tid; idx < CB * NP; idx += NT) {
            const int ch = idx / NP, q = idx - ch * NP;
            const bool ok = (ch0 + ch < ch_end) && (p0 + q < HW);
            const float *src = ok ? I + (int64_t)(ch0 + ch) * HW + p0 + q : I;
            cp_async4(smem + b * buf_floats + f_floats + idx, src, ok);
        }
    };

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

    pdl_wait();
    pdl_trigger();
    if (nchunks > 0) load_chunk(0, 0);
    cp_async_commit();
    for (int chunk = 0; chunk < nchunks; ++chunk) {
        const int b = chunk & 1;
        if (chunk + 1 < nchunks) load_chunk(chunk + 1, b ^ 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        const float *Fs = smem + b * buf_floats;
        const float *Is = Fs + f_floats;
#pragma unroll 1
        for (int ch = 0; ch < CB; ++ch) {
#pragma unroll
            for (int r = 0; r < (KT > 0 ? KT : 1); ++r) {
                for (int rr = (KT > 0 ? r : 0); rr < (KT > 0 ? r + 1 : K); ++rr) {
                    const float *ip = Is + ch * NP + rr * Wx + tn;
#pragma unroll
                    for (int c = 0; c < (KT > 0 ? KT : 1); ++c) {
                        for (int cc = (KT > 0 ? c : 0); cc < (KT > 0 ? c + 1 : K); ++cc) {
                            float bv[8];
#pragma unroll
                            for (int j = 0; j < 8; ++j) bv[j] = ip[cc + j * TNS];
                            const float *fp = Fs + ((ch * K + rr) * K + cc) * FS + tm * 8;
                            const float4 a0 = *reinterpret_cast<const float4 *>(fp);
                            const float4 a1 = *reinterpret_cast<const float4 *>(fp + 4);
                            const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
                            for (int i = 0; i < 8; ++i)
#pragma unroll
                                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
                        }
                    }
                }
            }
        }
        __syncthreads();
    }
    cp_async_wait<0>();
    __syncthreads();

    // ---- partial tile -> own smem, then fixed-order (DSMEM) reduction ------
    float *P = smem;                                // BM x BN
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) P[(tm * 8 + i) * BN + tn + j * TNS] = acc[i][j];
    if (S > 1) cluster_sync_all(); else __syncthreads();

    const int rows = BM / S;
    const int mlo = split * rows;
    const uint32_t Pbase = smem_u32(P);
    for (int idx = tid; idx < rows * BN; idx += NT) {
        const int m = mlo + idx / BN, n = idx % BN;
        const int p = p0 + n;
        const int y = p / Wx, x = p - y * Wx;
        float v = 0.f;
        if (S > 1) {
            for (int t = 0; t < S; ++t) v += ld_dsmem_f32(mapa_shared(Pbase + (m * BN + n) * 4, t));
        } else {
            v = P[m * BN + n];
        }
        if (m0 + m < M && y < Ho && x < Wo) O[(int64_t)(m0 + m) * Ho * Wo + (int64_t)y * Wo + x] = v;
    }
    if (S > 1) cluster_sync_all();
}

static int simt_np(int Wx, int K) {
    int np = kSimtBN + (K - 1) * Wx + (K - 1);
    return (np + 3) & ~3;
}
static int simt_smem(int Wx, int K) {
    const int CB = simt_cb(K);
    const int stage = CB * K * K * (kSimtBM + 4) + CB * simt_np(Wx, K);
    int bytes = 2 * stage * 4;
    const int pbytes = kSimtBM * kSimtBN * 4;
    return bytes > pbytes ? bytes : pbytes;
}

int plan_multi_simt(int C, int Wx, int Wy, int K, int M, conv_plan *p) {
    const int Ho = Wy - K + 1;
    if (simt_smem(Wx, K) > kSimtMaxSmem) {           // naive fallback
        const int64_t n = (int64_t)M * Ho * (Wx - K + 1);
        int64_t blocks = (n + 255) / 256;
        p->kernel = 1;
        p->grid_x = (int)(blocks < 4 * kNumSMs ? blocks : 4 * kNumSMs);
        p->grid_y = p->grid_z = 1;
        p->block_x = 256;
        p->cluster_x = 1;
        p->tile_m = 1;
        p->tile_n = 1;
        p->smem_bytes = 0;
        p->tma_f = 0;
        return 0;
    }
    const int npt = (Ho * Wx + kSimtBN - 1) / kSimtBN;
    const int nmt = (M + kSimtBM - 1) / kSimtBM;
    const int tiles = npt * nmt;
    int S = 1;
    while (S < 8 && tiles * S < kNumSMs && 2 * S <= C) S *= 2;
    p->kernel = 1;
    p->grid_x = S;
    p->grid_y = npt;
    p->grid_z = nmt;
    p->block_x = (kSimtBM / 8) * (kSimtBN / 8);
    p->cluster_x = S;
    p->tile_m = kSimtBM;
    p->tile_n = kSimtBN;
    p->smem_bytes = simt_smem(Wx, K);
    p->tma_f = 0;
    return 0;
}

template <int KT, int CB>
static cudaError_t launch_kms(const conv_plan &p, const float *I, int C, int Wx, int Wy,
                              const float *F, int K, int M, float *O, cudaStream_t s) {
    auto kern = kms_kernel<KT, kSimtBM, kSimtBN, CB>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         p.smem_bytes);
    if (e != cudaSuccess) return e;
    const int ch_per_split = (C + p.cluster_x - 1) / p.cluster_x;
    const int NP = simt_np(Wx, K);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.grid_x, p.grid_y, p.grid_z);
    cfg.blockDim = dim3(p.block_x);
    cfg.dynamicSmemBytes = p.smem_bytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.cluster_x;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled();
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kern, I, C, Wx, Wy, F, K, M, O, ch_per_split, NP);
}

cudaError_t launch_multi_simt(const float *I, int C, int Wx, int Wy, const float *F, int K, int M,
                              float *O, cudaStream_t s) {
    conv_plan p;
    plan_multi_simt(C, Wx, Wy, K, M, &p);
    if (p.tile_m == 1) {
        kmn_kernel<<<p.grid_x, p.block_x, 0, s>>>(I, C, Wx, Wy, F, K, M, O);
        return cudaGetLastError();
    }
    switch (K) {
        case 1: return launch_kms<1, simt_cb(1)>(p, I, C, Wx, Wy, F, K, M, O, s);
        case 3: return launch_kms<3, simt_cb(3)>(p, I, C, Wx, Wy, F, K, M, O, s);
        case 5: return launch_kms<5, simt_cb(5)>(p, I, C, Wx, Wy, F, K, M, O, s);
        case 7: return launch_kms<7, simt_cb(7)>(p, I, C, Wx, Wy, F, K, M, O, s);
        default: return launch_kms<0, simt_cb(0)>(p, I, C, Wx, Wy, F, K, M, O, s);
    }
}

}  // namespace b200
