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


constexpr int kSimtThreads = 256;              // (BM/8) x (BN/8) threads, 8x8 outputs each
constexpr int kSimtMaxSplit = 16;              // non-portable cluster size on B200
constexpr int kSimtStageBudget = 48 * 1024;    // bytes per pipeline stage
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

// KT = compile-time K (1..7) or 0 for a runtime K; CB = channels per stage.
template <int KT, int BM, int BN>
__global__ void __launch_bounds__(kSimtThreads, 2)
kms_kernel(const float *__restrict__ I, int C, int Wx, int Wy, const float *__restrict__ F,
           int Krt, int M, float *__restrict__ O, int ch_per_split, int NP, int CB) {
    static_assert((BM / 8) * (BN / 8) == kSimtThreads, "tile must map to 256 threads");
    constexpr int NT = (BM / 8) * (BN / 8);
    constexpr int TNS = BN / 8;                     // pixel stride inside a thread tile
    constexpr int FS = BM + 4;                      // transposed-F row stride (floats)
    const int K = KT > 0 ? KT : Krt;
    const int KK = K * K;
    const int Ho = Wy - K + 1, Wo = Wx - K + 1;
    const int HW = Wx * Wy;
    const int Ktot = C * KK;

    extern __shared__ __align__(16) float smem[];
    // smem: F_s[2][CB*KK][FS] (transposed, m contiguous) | I_s[2][CB][NP] | Fraw[BM][RS]
    const int CK = CB * KK;
    const int RS = ((CK - 4 + 31) / 32) * 32 + 4;   // raw row stride, == 4 (mod 32)
    const int f_floats = CK * FS;
    const int i_floats = CB * NP;
    float *Fs_buf = smem;
    float *Is_buf = smem + 2 * f_floats;
    float *Fraw = Is_buf + 2 * i_floats;

    const int S = gridDim.x;                        // cluster size == split
    const int split = blockIdx.x;
    const int p0 = blockIdx.y * BN;
    const int m0 = blockIdx.z * BM;
    const int ch_begin = split * ch_per_split;
    const int ch_end = min(C, ch_begin + ch_per_split);
    const int nchunks = ch_end > ch_begin ? (ch_end - ch_begin + CB - 1) / CB : 0;
    const int tid = threadIdx.x;
    const int tn = tid % TNS, tm = tid / TNS;
    // 16-B copies of F rows when every row start of every chunk is 16-B aligned
    const bool vec_f = ((Ktot & 3) == 0) && ((CK & 3) == 0) && ((ch_per_split * KK & 3) == 0) &&
                       ((reinterpret_cast<uintptr_t>(F) & 15) == 0);

    // F rows (row-major, as stored) -> Fraw with coalesced cp.async over the flat
    // (row, 16-B vector) space: every lane busy, one division per copy
    auto load_f = [&](int chunk) {
        const int ch0 = ch_begin + chunk * CB;
        const int nk = min(CB, ch_end - ch0) * KK;            // valid k of this chunk
        const float *fbase = F + (int64_t)m0 * Ktot + (int64_t)ch0 * KK;
        if (vec_f) {
            const int nv = CK >> 2;
            for (int idx = tid; idx < BM * nv; idx += NT) {
                const int m = idx / nv, v = idx - m * nv;
                const bool ok = (m0 + m < M) && 4 * v < nk;      // nk is a multiple of 4 here
                const float *src = ok ? fbase + (int64_t)m * Ktot + 4 * v : F;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;"
                             ::"r"(smem_u32(Fraw + m * RS + 4 * v)), "l"(src), "r"(ok ? 16 : 0)
                             : "memory");
            }
        } else {
            for (int idx = tid; idx < BM * CK; idx += NT) {
                const int m = idx / CK, kk = idx - m * CK;
                const bool ok = (m0 + m < M) && kk < nk;
                cp_async4(Fraw + m * RS + kk, ok ? fbase + (int64_t)m * Ktot + kk : F, ok);
            }
        }
    };
    auto load_i = [&](int chunk, int b) {
        const int ch0 = ch_begin + chunk * CB;
        float *is = Is_buf + b * i_floats;
        for (int idx = tid; idx < CB * NP; idx += NT) {
            const int ch = idx / NP, q = idx - ch * NP;
            const bool ok = (ch0 + ch < ch_end) && (p0 + q < HW);
            cp_async4(is + idx, ok ? I + (int64_t)(ch0 + ch) * HW + p0 + q : I, ok);
        }
    };
    // Fraw[m][k..k+3] (16-B loads along m: RS == 4 mod 32 -> conflict-free)
    //   -> F_s[k+i][m] (scalar stores, consecutive m -> conflict-free)
    auto transpose_f = [&](int b) {
        float *fs = Fs_buf + b * f_floats;
        const int nq = (CK + 3) / 4;
        for (int u = tid; u < BM * nq; u += NT) {
            const int m = u % BM, q = u / BM;
            const float4 v = *reinterpret_cast<const float4 *>(Fraw + m * RS + 4 * q);
            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (4 * q + i < CK) fs[(4 * q + i) * FS + m] = vv[i];
        }
    };

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

    pdl_wait();
    pdl_trigger();
    // pipeline: F of chunk c+1 lands in Fraw and I of chunk c+1 in I_s[(c+1)&1]
    // while chunk c computes; then Fraw is transposed into F_s[(c+1)&1]
    if (nchunks > 0) {
        load_f(0);
        load_i(0, 0);
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        transpose_f(0);
        __syncthreads();
        if (nchunks > 1) { load_f(1); load_i(1, 1); }
        cp_async_commit();
    }
    for (int chunk = 0; chunk < nchunks; ++chunk) {
        const int b = chunk & 1;
        const float *Fs = Fs_buf + b * f_floats;
        const float *Is = Is_buf + b * i_floats;
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
        if (chunk + 1 < nchunks) {
            cp_async_wait<0>();                     // chunk c+1 staged
            __syncthreads();                        // ... and everyone is done with chunk c
            transpose_f(b ^ 1);
            __syncthreads();
            if (chunk + 2 < nchunks) { load_f(chunk + 2); load_i(chunk + 2, b); }
            cp_async_commit();
        }
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

namespace {
struct SimtTile { int BM, BN; };
constexpr SimtTile kSimtTiles[3] = {{128, 128}, {64, 256}, {256, 64}};

int simt_np(int BN, int Wx, int K) { return (BN + (K - 1) * Wx + (K - 1) + 3) & ~3; }
// channels per stage: a multiple of 4 (16-B F rows) within the stage budget
int simt_cb_for(int BM, int BN, int Wx, int K, int C) {
    const int per_ch = (K * K * (2 * BM + 5) + 2 * simt_np(BN, Wx, K)) * 4;
    int cb = (2 * kSimtStageBudget / per_ch) & ~3;
    if (cb > 8) cb = 8;
    if (cb < 4) cb = 4;
    if (cb > C) cb = C;
    return cb < 1 ? 1 : cb;
}
// channels per split, a multiple of CB (chunk starts stay 16-B aligned in F)
void simt_split(int C, int S, int BM, int BN, int Wx, int K, int *CB, int *cps) {
    int per = (C + S - 1) / S;
    int cb = simt_cb_for(BM, BN, Wx, K, C);
    if (cb > per) cb = per >= 4 ? (per & ~3) : per;
    *CB = cb;
    *cps = ((per + cb - 1) / cb) * cb;
}
int simt_smem(int BM, int BN, int Wx, int K, int CB) {
    const int CK = CB * K * K;
    const int RS = ((CK - 4 + 31) / 32) * 32 + 4;
    const int bytes = (2 * CK * (BM + 4) + 2 * CB * simt_np(BN, Wx, K) + BM * RS) * 4;
    const int pbytes = BM * BN * 4;
    return bytes > pbytes ? bytes : pbytes;
}
}  // namespace

int plan_multi_simt(int C, int Wx, int Wy, int K, int M, conv_plan *p) {
    const int Ho = Wy - K + 1;
    const int64_t px = (int64_t)Ho * Wx;                  // wide pixels
    // tile shape with the least padded work (ties: the first, 128 x 128)
    int best = 0;
    int64_t best_pad = -1;
    for (int i = 0; i < 3; ++i) {
        const int64_t pad = ((px + kSimtTiles[i].BN - 1) / kSimtTiles[i].BN) * kSimtTiles[i].BN *
                            (((int64_t)M + kSimtTiles[i].BM - 1) / kSimtTiles[i].BM) * kSimtTiles[i].BM;
        if (best_pad < 0 || pad < best_pad) { best_pad = pad; best = i; }
    }
    const int BM = kSimtTiles[best].BM, BN = kSimtTiles[best].BN;
    const int CB = simt_cb_for(BM, BN, Wx, K, C);
    const int smem = simt_smem(BM, BN, Wx, K, CB);
    if (smem > kSimtMaxSmem) {                           // naive fallback (huge K * Wx)
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
    const int npt = (int)((px + BN - 1) / BN);
    const int nmt = (M + BM - 1) / BM;
    const int tiles = npt * nmt;
    int S = 1;        // split the channel sum over a cluster until ~2 CTAs per SM
    while (S < kSimtMaxSplit && tiles * S < 2 * kNumSMs && 2 * S <= C) S *= 2;
    p->kernel = 1;
    p->grid_x = S;
    p->grid_y = npt;
    p->grid_z = nmt;
    p->block_x = kSimtThreads;
    p->cluster_x = S;
    p->tile_m = BM;
    p->tile_n = BN;
    p->smem_bytes = smem;
    p->tma_f = 0;
    return 0;
}

template <int KT, int BM, int BN>
static cudaError_t launch_kms(const conv_plan &p, const float *I, int C, int Wx, int Wy,
                              const float *F, int K, int M, float *O, cudaStream_t s) {
    auto kern = kms_kernel<KT, BM, BN>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         p.smem_bytes);
    if (e != cudaSuccess) return e;
    if (p.cluster_x > 8) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    int CB, ch_per_split;
    simt_split(C, p.cluster_x, BM, BN, Wx, K, &CB, &ch_per_split);
    const int NP = simt_np(BN, Wx, K);
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
    return cudaLaunchKernelEx(&cfg, kern, I, C, Wx, Wy, F, K, M, O, ch_per_split, NP, CB);
}

template <int KT>
static cudaError_t launch_kms_tile(const conv_plan &p, const float *I, int C, int Wx, int Wy,
                                   const float *F, int K, int M, float *O, cudaStream_t s) {
    if (p.tile_m == 64) return launch_kms<KT, 64, 256>(p, I, C, Wx, Wy, F, K, M, O, s);
    if (p.tile_m == 256) return launch_kms<KT, 256, 64>(p, I, C, Wx, Wy, F, K, M, O, s);
    return launch_kms<KT, 128, 128>(p, I, C, Wx, Wy, F, K, M, O, s);
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
        case 1: return launch_kms_tile<1>(p, I, C, Wx, Wy, F, K, M, O, s);
        case 3: return launch_kms_tile<3>(p, I, C, Wx, Wy, F, K, M, O, s);
        case 5: return launch_kms_tile<5>(p, I, C, Wx, Wy, F, K, M, O, s);
        case 7: return launch_kms_tile<7>(p, I, C, Wx, Wy, F, K, M, O, s);
        default: return launch_kms_tile<0>(p, I, C, Wx, Wy, F, K, M, O, s);
    }
}

}  // namespace b200
