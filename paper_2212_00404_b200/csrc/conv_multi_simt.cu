// conv_multi_simt.cu — kernel KM-SIMT: multi-channel direct convolution in
// strict FP32 on CUDA cores (§2.1 Eq. 1; the paper's
// stride-fixed-block kernel, §3.2, re-designed for sm_100a).
//
//   O[m][y][x] = sum_{ch,r,c} I[ch][y+r][x+c] * F[m][ch][r][c]
//
// Design: an implicit GEMM on the FP32 pipes,
//   D[m][n] = sum_k F[m][k] * B[k][n],  k = (ch, r, c),  n = output pixel y*Wo+x
//  * CTA tile = BM filters x BN output pixels (compact indexing: no garbage
//    columns), 256 threads, 8 x 8 register tile per thread taken as two 4-wide
//    halves in m and in n so every operand load is a 16-B shared load.
//  * The reduction runs over channel chunks of CB channels — the paper's
//    segment of S = CB*K*K*4 bytes per filter — double buffered
//    (the paper's prefetch rounds):
//      F: 16-B cp.async of the rows as stored into a raw buffer, then an
//         in-smem transpose to [k][m];
//      B: the im2col tile [k][n] gathered straight from global/L2 by 4-B
//         cp.async (one pixel per lane: coalesced), offsets from a small
//         per-chunk k -> (ch, r, c) table in shared memory.
//  * Small layers cannot fill 148 SMs with output tiles, so the channel sum is
//    split across a thread-block cluster of up to 16 CTAs (the paper's
//    rejected Fig. 2(b) split along ch): partial tiles are reduced
//    through distributed shared memory in fixed rank order (deterministic, no
//    global atomics, O written once).
#include <cstdint>
#include "kernels.h"
#include "ptx.cuh"

namespace b200 {

constexpr int kSimtThreads = 256;              // (BM/8) x (BN/8) threads, 8x8 outputs each
constexpr int kSimtMaxSplit = 16;              // non-portable cluster size on B200
constexpr int kSimtMaxSmem = 110 * 1024;       // 2 CTAs per SM

// Fallback for shapes whose chunk does not fit in shared memory (huge K):
// one thread per output, loads through L1.
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

// smem layout (floats): F_s[CK][BM] | B_s[2][CK][BN] | Fraw[BM][RS] | koff[CK] (int)
// (F is double buffered through Fraw: chunk c+1 lands in Fraw while chunk c
// computes from F_s, and is transposed into F_s once every thread is done.)
__host__ __device__ constexpr int simt_rs(int CK) { return ((CK - 4 + 31) / 32) * 32 + 4; }

template <int BM, int BN>
__global__ void __launch_bounds__(kSimtThreads, 2)
kms_kernel(const float *__restrict__ I, int C, int Wx, int Wy, const float *__restrict__ F,
           int K, int M, float *__restrict__ O, int ch_per_split, int CB) {
    static_assert((BM / 8) * (BN / 8) == kSimtThreads, "tile must map to 256 threads");
    constexpr int NT = kSimtThreads;
    constexpr int TNG = BN / 8;                     // thread columns
    const int KK = K * K;
    const int Ho = Wy - K + 1, Wo = Wx - K + 1;
    const int HW = Wx * Wy;
    const int HoWo = Ho * Wo;
    const int Ktot = C * KK;
    const int CK = CB * KK;
    const int RS = simt_rs(CK);

    extern __shared__ __align__(16) float smem[];
    float *Fs_buf = smem;                           // [CK][BM]
    float *Bs_buf = smem + CK * BM;                 // [2][CK][BN]
    float *Fraw = Bs_buf + 2 * CK * BN;             // [BM][RS]
    int *koff = reinterpret_cast<int *>(Fraw + BM * RS);   // [CK]

    const int S = gridDim.x;                        // cluster size == split
    const int split = blockIdx.x;
    const int p0 = blockIdx.y * BN;
    const int m0 = blockIdx.z * BM;
    const int ch_begin = split * ch_per_split;
    const int ch_end = min(C, ch_begin + ch_per_split);
    const int nchunks = ch_end > ch_begin ? (ch_end - ch_begin + CB - 1) / CB : 0;
    const int tid = threadIdx.x;
    const int tn = tid % TNG, tm = tid / TNG;
    // widest copy of F rows (16, 8 or 4 B) that keeps every row start of every
    // chunk aligned
    auto fits = [&](int w) {
        return (Ktot % w) == 0 && (CK % w) == 0 && ((ch_per_split * KK) % w) == 0 &&
               (reinterpret_cast<uintptr_t>(F) % (4 * w)) == 0;
    };
    const int vw = fits(4) ? 4 : (fits(2) ? 2 : 1);

    // k -> input offset within a chunk (channel relative to the chunk start)
    for (int k = tid; k < CK; k += NT) {
        const int ch = k / KK, rem = k - ch * KK, r = rem / K;
        koff[k] = ch * HW + r * Wx + (rem - r * K);
    }
    // this thread's im2col pixel (fixed for the whole kernel) and k-lane
    constexpr int KL = NT / BN > 0 ? NT / BN : 1;
    const int bn = tid % BN, bkl = tid / BN;
    const int bo = p0 + bn;
    const bool bvalid = bo < HoWo;
    const int by = bvalid ? bo / Wo : 0;
    const int bbase = by * Wx + (bvalid ? bo - by * Wo : 0);

    auto load_f = [&](int chunk) {
        const int ch0 = ch_begin + chunk * CB;
        const int nk = min(CB, ch_end - ch0) * KK;            // valid k of this chunk
        const float *fbase = F + (int64_t)m0 * Ktot + (int64_t)ch0 * KK;
        // thread -> fixed vector column v of rows mr, mr + rpt, ...: no division in the loop
        const int nv = CK / vw;
        const int rpt = NT / nv;
        if (tid < nv * rpt) {
            const int v = tid % nv, mr = tid / nv;
            const bool kok = vw * v < nk;                     // nk is a multiple of vw
            const float *src = fbase + (int64_t)mr * Ktot + vw * v;
            uint32_t dst = smem_u32(Fraw + mr * RS + vw * v);
            for (int m = mr; m < BM; m += rpt) {
                const bool ok = kok && (m0 + m < M);
                const float *sp = ok ? src : F;
                if (vw == 4)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;"
                                 ::"r"(dst), "l"(sp), "r"(ok ? 16 : 0) : "memory");
                else if (vw == 2)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;"
                                 ::"r"(dst), "l"(sp), "r"(ok ? 8 : 0) : "memory");
                else
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;"
                                 ::"r"(dst), "l"(sp), "r"(ok ? 4 : 0) : "memory");
                src += (int64_t)rpt * Ktot;
                dst += rpt * RS * 4;
            }
        }
    };
    // im2col tile B[k][n] = I[ch0 + ch][y_n + r][x_n + c] (zero past the valid range)
    auto load_b = [&](int chunk, int b) {
        const int ch0 = ch_begin + chunk * CB;
        const int nk = min(CB, ch_end - ch0) * KK;
        const float *src = I + (int64_t)ch0 * HW + bbase;
        float *dst = Bs_buf + b * CK * BN + bn;
        for (int k = bkl; k < CK; k += KL) {
            const bool ok = bvalid && k < nk;
            cp_async4(dst + k * BN, ok ? src + koff[k] : I, ok);
        }
    };
    // Fraw[m][k..k+3] (16-B loads along m: RS == 4 mod 32 -> conflict-free)
    //   -> F_s[k+i][m] (scalar stores, consecutive m -> conflict-free)
    auto transpose_f = [&]() {
        float *fs = Fs_buf;
        const int nq = (CK + 3) / 4;
        for (int u = tid; u < BM * nq; u += NT) {
            const int m = u % BM, q = u / BM;
            const float4 v = *reinterpret_cast<const float4 *>(Fraw + m * RS + 4 * q);
            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (4 * q + i < CK) fs[(4 * q + i) * BM + m] = vv[i];
        }
    };

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

    pdl_wait();
    pdl_trigger();
    __syncthreads();                                // koff table
    if (nchunks > 0) {
        load_f(0);
        load_b(0, 0);
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        transpose_f();
        __syncthreads();
        if (nchunks > 1) { load_f(1); load_b(1, 1); }
        cp_async_commit();
    }
    for (int chunk = 0; chunk < nchunks; ++chunk) {
        const int b = chunk & 1;
        const float *Fs = Fs_buf + tm * 4;
        const float *Bs = Bs_buf + b * CK * BN + tn * 4;
#pragma unroll 4
        for (int k = 0; k < CK; ++k) {
            const float4 a0 = *reinterpret_cast<const float4 *>(Fs + k * BM);
            const float4 a1 = *reinterpret_cast<const float4 *>(Fs + k * BM + BM / 2);
            const float4 b0 = *reinterpret_cast<const float4 *>(Bs + k * BN);
            const float4 b1 = *reinterpret_cast<const float4 *>(Bs + k * BN + BN / 2);
            const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        if (chunk + 1 < nchunks) {
            cp_async_wait<0>();                     // chunk c+1 staged
            __syncthreads();                        // ... and everyone is done with chunk c
            transpose_f();
            __syncthreads();
            if (chunk + 2 < nchunks) { load_f(chunk + 2); load_b(chunk + 2, b); }
            cp_async_commit();
        }
    }
    cp_async_wait<0>();
    __syncthreads();

    // ---- partial tile -> own smem, then fixed-order (DSMEM) reduction ------
    float *P = smem;                                // [BM][BN]
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int m = (i < 4) ? tm * 4 + i : BM / 2 + tm * 4 + (i - 4);
        *reinterpret_cast<float4 *>(P + m * BN + tn * 4) =
            make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        *reinterpret_cast<float4 *>(P + m * BN + BN / 2 + tn * 4) =
            make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
    }
    if (S > 1) cluster_sync_all(); else __syncthreads();

    const int mlo = split * BM / S;                 // rows [mlo, mhi) reduced by this rank
    const int rows = (split + 1) * BM / S - mlo;
    const uint32_t Pbase = smem_u32(P);
    const int nvalid = min(BN, HoWo - p0);
    for (int idx = tid; idx < rows * BN; idx += NT) {
        const int m = mlo + idx / BN, n = idx % BN;
        float v = 0.f;
        if (S > 1) {
            for (int t = 0; t < S; ++t) v += ld_dsmem_f32(mapa_shared(Pbase + (m * BN + n) * 4, t));
        } else {
            v = P[m * BN + n];
        }
        if (m0 + m < M && n < nvalid) O[(int64_t)(m0 + m) * HoWo + p0 + n] = v;   // compact: coalesced
    }
    if (S > 1) cluster_sync_all();
}

namespace {
struct SimtTile { int BM, BN; };
constexpr SimtTile kSimtTiles[3] = {{128, 128}, {64, 256}, {256, 64}};

int simt_smem(int BM, int BN, int CK) {
    const int bytes = (CK * BM + 2 * CK * BN + BM * simt_rs(CK)) * 4 + CK * 4;
    const int pbytes = BM * BN * 4;
    return bytes > pbytes ? bytes : pbytes;
}
// channels per stage: a multiple of 4 (16-B F rows) that fits the smem budget
int simt_cb_for(int BM, int BN, int K, int C) {
    int cb = (64 / (K * K) + 3) & ~3;               // ~64 k-steps per chunk
    if (cb < 8) cb = 8;
    while (cb > 4 && simt_smem(BM, BN, cb * K * K) > kSimtMaxSmem) cb -= 4;
    while (cb > 1 && simt_smem(BM, BN, cb * K * K) > kSimtMaxSmem + 16 * 1024) --cb;
    if (cb > C) cb = C;
    return cb < 1 ? 1 : cb;
}
// channels per split, a multiple of CB (chunk starts stay 16-B aligned in F)
void simt_split(int C, int S, int BM, int BN, int K, int *CB, int *cps) {
    const int per = (C + S - 1) / S;
    const int budget = simt_cb_for(BM, BN, K, C);
    // largest chunk in {8, 4, 2, 1} (<= budget) that wastes < 1/8 of a split
    int cb = 1;
    for (int c : {8, 4, 2}) {
        if (c > budget || c > per) continue;
        const int waste = ((per + c - 1) / c) * c - per;
        if (8 * waste <= per) { cb = c; break; }
    }
    *CB = cb;
    *cps = ((per + cb - 1) / cb) * cb;
}
}  // namespace

int plan_multi_simt(int C, int Wx, int Wy, int K, int M, conv_plan *p) {
    const int Ho = Wy - K + 1, Wo = Wx - K + 1;
    const int64_t px = (int64_t)Ho * Wo;                  // compact output pixels
    // tile shape with the least padded work (ties: the first, 128 x 128)
    int best = 0;
    int64_t best_pad = -1;
    for (int i = 0; i < 3; ++i) {
        const int64_t pad = ((px + kSimtTiles[i].BN - 1) / kSimtTiles[i].BN) * kSimtTiles[i].BN *
                            (((int64_t)M + kSimtTiles[i].BM - 1) / kSimtTiles[i].BM) * kSimtTiles[i].BM;
        if (best_pad < 0 || pad < best_pad) { best_pad = pad; best = i; }
    }
    const int BM = kSimtTiles[best].BM, BN = kSimtTiles[best].BN;
    const int CB = simt_cb_for(BM, BN, K, C);
    if (simt_smem(BM, BN, CB * K * K) > kSimtMaxSmem + 64 * 1024) {   // naive fallback (huge K)
        const int64_t n = (int64_t)M * px;
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
    // split the channel sum over a cluster (unit = 1 channel of a 16K-output
    // tile, ~0.6 us per 9 taps; DSMEM reduction ~1 us)
    const int smem = simt_smem(BM, BN, CB * K * K);
    const int S = choose_split(tiles, C, kSimtMaxSplit, smem <= 113 * 1024 ? 2 : 1,
                               0.6f * (float)(K * K) / 9.f, 1.0f);
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

template <int BM, int BN>
static cudaError_t launch_kms(const conv_plan &p, const float *I, int C, int Wx, int Wy,
                              const float *F, int K, int M, float *O, cudaStream_t s) {
    auto kern = kms_kernel<BM, BN>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         p.smem_bytes);
    if (e != cudaSuccess) return e;
    if (p.cluster_x > 8) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    int CB, ch_per_split;
    simt_split(C, p.cluster_x, BM, BN, K, &CB, &ch_per_split);
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
    return cudaLaunchKernelEx(&cfg, kern, I, C, Wx, Wy, F, K, M, O, ch_per_split, CB);
}

int simt_max_clusters(int cluster, int smem) {
    auto kern = kms_kernel<128, 128>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cluster, 1, 1);
    cfg.blockDim = dim3(kSimtThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = -1;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) { cudaGetLastError(); return -1; }
    return n;
}

cudaError_t launch_multi_simt(const float *I, int C, int Wx, int Wy, const float *F, int K, int M,
                              float *O, cudaStream_t s) {
    conv_plan p;
    plan_multi_simt(C, Wx, Wy, K, M, &p);
    if (p.tile_m == 1) {
        kmn_kernel<<<p.grid_x, p.block_x, 0, s>>>(I, C, Wx, Wy, F, K, M, O);
        return cudaGetLastError();
    }
    if (p.tile_m == 64) return launch_kms<64, 256>(p, I, C, Wx, Wy, F, K, M, O, s);
    if (p.tile_m == 256) return launch_kms<256, 64>(p, I, C, Wx, Wy, F, K, M, O, s);
    return launch_kms<128, 128>(p, I, C, Wx, Wy, F, K, M, O, s);
}

}  // namespace b200
