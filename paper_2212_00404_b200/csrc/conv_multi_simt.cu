// conv_multi_simt.cu — kernel KM-SIMT: multi-channel direct convolution in
// strict FP32 on CUDA cores (§2.1 Eq. 1; the paper's
// stride-fixed-block kernel, §3.2, re-designed for sm_100a).
//
//   O[m][y][x] = sum_{ch,r,c} I[ch][y+r][x+c] * F[m][ch][r][c]
//
// Design: an implicit GEMM on the FP32 pipes,
//   D[m][n] = sum_k F[m][k] * B[k][n],  k = (ch, r, c),  n = output pixel y*Wo+x
//  * CTA tile = BM filters x BN output pixels (compact indexing: no garbage
//    columns), 256 threads, 8 x TN register tile per thread (TN = 8, 6 or 4),
//    every operand load a 16-B (or 8-B) shared load.
//  * The reduction runs over channel chunks of CB channels — the paper's
//    segment of S = CB*K*K*4 bytes per filter — in a two-stage
//    cp.async pipeline (the paper's prefetch rounds):
//      F: 16-B cp.async of the rows as stored into a raw buffer, then an
//         in-smem transpose to [k][m] (a transpose-free [k/4][m][4] layout
//         was measured slower: ptxas interleaves the four k of a quad into
//         short dependent FFMA chains);
//      B: the im2col tile [k][n] gathered straight from global/L2 by 4-B
//         cp.async (one pixel per lane: coalesced), offsets from a small
//         per-chunk k -> (ch, r, c) table in shared memory.
//  * Small layers cannot fill 148 SMs with output tiles, so the channel sum is
//    split S ways (the paper's rejected Fig. 2(b) split along ch):
//    either across a thread-block cluster (partials reduced through
//    distributed shared memory in fixed rank order) or, when more splits pay
//    than clusters can co-reside, through the split-K workspace and a
//    fixed-order reduction kernel (workspace.cu).  Both are deterministic.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include "kernels.h"
#include "latency_model.h"
#include "ptx.cuh"

namespace b200 {

#ifndef B200CONV_SIMT_UNROLL2
#define B200CONV_SIMT_UNROLL2 0
#endif
constexpr bool kUnroll2 = B200CONV_SIMT_UNROLL2;   // (A/B build switch: kq loop unrolled by 2)
constexpr int kSimtThreads = 256;              // (BM/8) x (BN/8) threads, 8x8 outputs each
constexpr int kSimtMaxSplit = 16;              // non-portable cluster size on B200
constexpr int kSimtMaxSmem = 110 * 1024;       // 2 CTAs per SM
#ifndef B200CONV_SIMT_FIXED_CK
#define B200CONV_SIMT_FIXED_CK 1
#endif
constexpr bool kSimtFixedCk = B200CONV_SIMT_FIXED_CK;   // (A/B build switch: compile-time 36-k chunks)
#ifndef B200CONV_SIMT_FIXED_UNROLL
#define B200CONV_SIMT_FIXED_UNROLL 9
#endif
// k-quad unroll of the fixed-chunk loop: all 9 (every operand address an
// immediate off two per-chunk bases; measured configs[4] 124.9 -> 114.4 us
// against no unroll, 119.2 us with 3)
constexpr int kSimtFixedUnroll = B200CONV_SIMT_FIXED_UNROLL;

// diagnostics (B200CONV_SIMT_DBG=1): per-CTA globaltimer stamps [start, after
// griddepcontrol.wait, chunk 0 staged, main loop done, end << 8 | smid]
__device__ unsigned long long g_simt_cta[5 * 1024];
__device__ __forceinline__ unsigned long long simt_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned long long simt_smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}
int simt_read_stamps(unsigned long long *host) {
    return cudaMemcpyFromSymbol(host, g_simt_cta, sizeof(g_simt_cta)) == cudaSuccess ? 0 : 1;
}

// Fallback for shapes whose chunk does not fit in shared memory (huge K):
// one thread per output, loads through L1.
__global__ void __launch_bounds__(256)
kmn_kernel(const float *__restrict__ I, int C, int Wx, int Wy, const float *__restrict__ F, int K,
           int M, float *__restrict__ O, int sd) {
    const int Ho = (Wy - K) / sd + 1, Wo = (Wx - K) / sd + 1;
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
            const float *Ic = I + (int64_t)ch * Wx * Wy + (int64_t)y * sd * Wx + (int64_t)x * sd;
            const float *Fc = F + ((int64_t)m * C + ch) * K * K;
            for (int r = 0; r < K; ++r)
                for (int c = 0; c < K; ++c) acc = fmaf(__ldg(Ic + (int64_t)r * Wx + c), __ldg(Fc + r * K + c), acc);
        }
        O[o] = acc;
    }
}

// smem layout (floats): F[2][BM][RS] | B[2][CKP][BN] | koff[CKP] (int): a
// two-stage ring of (F rows as stored, im2col tile); CKP = the chunk's k padded
// to whole 16-B quads.  The main loop reads F in place, four k per 16-B load
// (no transpose pass), and issues paired FMAs (FFMA2, ptx.cuh ffma2).
__host__ __device__ constexpr int simt_rs(int CK) { return ((CK - 4 + 31) / 32) * 32 + 4; }

// Thread tile: 8 filters (two 4-row halves, BM/2 apart) x TN pixels, TN in
// {8, 6, 4}: columns tn*4 .. tn*4+3 of the first region (width R1 = 4*TNG) and,
// for TN > 4, TN-4 more columns at R1 + tn*(TN-4) — every operand load is one
// 16-B (or 8-B) shared load.
template <int BM, int BN, int TN>
struct SimtShape {
    static constexpr int TNG = BN / TN;             // thread columns
    static constexpr int TMG = BM / 8;              // thread rows
    static constexpr int R1 = 4 * TNG;
    static constexpr int T2 = TN - 4;               // 0, 2 or 4
    static_assert(TMG * TNG == kSimtThreads && TNG * TN == BN, "tile must map to 256 threads");
    __device__ static int row(int tm, int i) { return tm + TMG * i; }     // interleaved thread rows
};

// NST: ring stages (NST = 2: two CTAs per SM, 128 registers; NST >= 3: one
// CTA per SM, up to 255 registers).  One barrier per chunk: right after it,
// the stage chunk c - 1 used — which every thread has finished, as the
// barrier guarantees — is refilled with chunk c + NST - 1.
// kCKP > 0: the chunk's k count is a compile-time constant (the TMA-fed
// K = 3, 4-channel chunk of every 3x3 bench layer: 36), so every shared-memory
// operand address in the main loop is one base register plus an immediate
// (measured: the runtime row stride cost ~14 integer instructions per k-quad,
// each an issue slot the FFMA2 stream needs)
template <int BM, int BN, int TN, bool kTmaF, int NST, int kCKP = 0>
__global__ void __launch_bounds__(kSimtThreads, NST == 2 ? 2 : 1)
kms_kernel(const __grid_constant__ CUtensorMap tmapF, const float *__restrict__ I, int C, int Wx, int Wy,
           const float *__restrict__ F,
           int K, int M, float *__restrict__ O, int ch_per_split, int CB, float *__restrict__ W, int dbg_in,
           int sd, int Nimg) {
    using SH = SimtShape<BM, BN, TN>;
    const int dbg = kDiag ? dbg_in : 0;
    const unsigned cta_lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    const bool tl = dbg && threadIdx.x == 0 && cta_lin < 1024;
    if (tl) g_simt_cta[5 * cta_lin] = simt_gtimer();
    constexpr int NT = kSimtThreads;
    constexpr int TNG = SH::TNG;
    constexpr int T2 = SH::T2;
    const int KK = K * K;
    const int Ho = (Wy - K) / sd + 1, Wo = (Wx - K) / sd + 1;   // stride sd (NEXT-3)
    const int HW = Wx * Wy;
    const int HoWo = Ho * Wo;
    const int Ptot = Nimg * HoWo;                   // compact pixels of all images (batch)
    const int Ktot = C * KK;
    const int CK = CB * KK;

    const int CKP = kCKP > 0 ? kCKP : (CK + 3) & ~3;   // k per chunk, padded to whole 16-B quads
    // F row stride: RS = 4 mod 32 words (cp.async rows); TMA boxes land dense
    // (CKP = CK, CK / 4 not a multiple of 4: consecutive rows still hit
    // different 16-B bank quads)
    const int RS = kTmaF ? CKP : simt_rs(CKP);

    extern __shared__ __align__(128) float smem[];
    float *Fst = smem;                              // [NST][BM][RS]   F rows as stored (k fastest)
    float *Bst = smem + NST * BM * RS;              // [NST][CKP][BN]  im2col tile
    int *koff = reinterpret_cast<int *>(Bst + NST * CKP * BN);   // [CKP]
    uint64_t *fbar = reinterpret_cast<uint64_t *>(koff + ((CKP + 1) & ~1));   // [NST] F stage barriers (TMA)

    const int S = gridDim.x;                        // split count (== cluster size when W == nullptr)
    const int split = blockIdx.x;
    const int p0 = blockIdx.y * BN;
    const int m0 = blockIdx.z * BM;
    // the ceil(C / CB) channel chunks dealt to the S splits as evenly as whole
    // chunks allow (sizes differ by at most one chunk; the host's ch_per_split
    // is the largest share, ceil-rounded, used only for planning)
    (void)ch_per_split;
    const int nch_all = (C + CB - 1) / CB;
    const int ch_begin = (int)((int64_t)split * nch_all / S) * CB;
    const int ch_end = min(C, (int)((int64_t)(split + 1) * nch_all / S) * CB);
    const int nchunks = ch_end > ch_begin ? (ch_end - ch_begin + CB - 1) / CB : 0;
    const int tid = threadIdx.x;
    const int tn = tid % TNG, tm = tid / TNG;
    // widest copy of F rows (16, 8 or 4 B) that keeps every row start of every
    // chunk aligned
    auto fits = [&](int w) {
        return (Ktot % w) == 0 && (CK % w) == 0 &&
               (reinterpret_cast<uintptr_t>(F) % (4 * w)) == 0;
    };
    const int vw = fits(4) ? 4 : (fits(2) ? 2 : 1);

    // k -> input offset within a chunk (channel relative to the chunk start)
    for (int k = tid; k < CKP; k += NT) {
        const int ch = k / KK, rem = k - ch * KK, r = rem / K;
        koff[k] = k < CK ? ch * HW + r * Wx + (rem - r * K) : 0;
    }
    // this thread's im2col pixel (fixed for the whole kernel) and k-lane
    constexpr int KL = NT / BN > 0 ? NT / BN : 1;
    const int bn = tid % BN, bkl = tid / BN;
    const int bo = p0 + bn;
    const bool bvalid = bo < Ptot;
    const int bimg = bvalid ? bo / HoWo : 0;
    const int bpix = bvalid ? bo - bimg * HoWo : 0;
    const int by = bpix / Wo;
    // input pixel of output (by, bx) of image bimg
    const int64_t bbase = (int64_t)bimg * C * HW + sd * (by * Wx + (bpix - by * Wo));

    // F rows straight into Fst[stage][m][0..CKP): thread -> fixed vector column
    // v (+ NT, ... when a row has more than NT vectors) of rows mr, mr + rpt, ...
    // (chunk invariant, decoded once); columns past the chunk's valid k and
    // rows past M are zero-filled
    const int f_nv = CKP / vw;
    const int f_rpt = NT / f_nv > 0 ? NT / f_nv : 1;
    const int f_vstep = f_nv < NT ? f_nv : NT;
    const bool f_act = tid < f_vstep * f_rpt;
    const int f_v = f_act ? tid % f_vstep : 0, f_mr = f_act ? tid / f_vstep : 0;
    const int64_t f_step = (int64_t)f_rpt * Ktot;
    auto load_f = [&](int chunk, int st) {
        if constexpr (kTmaF) {
            // one 2-D TMA box [BM rows][CK k] of F seen as [M][Ktot]: rows past
            // M and k past Ktot (the last, partial chunk) are zero-filled
            if (tid == 0) {
                mbar_arrive_expect_tx(&fbar[st], BM * CKP * 4);
                tma_load_2d(Fst + st * BM * RS, &tmapF, &fbar[st], (ch_begin + chunk * CB) * KK, m0);
            }
            return;
        }
        if (!f_act) return;
        const int ch0 = ch_begin + chunk * CB;
        const int nk = min(CB, ch_end - ch0) * KK;            // valid k of this chunk
        const uint32_t dstep = f_rpt * RS * 4;
        for (int v = f_v; v < f_nv; v += f_vstep) {
            const bool kok = vw * v < nk;                     // nk is a multiple of vw
            const float *src = F + (int64_t)(m0 + f_mr) * Ktot + (int64_t)ch0 * KK + vw * v;
            uint32_t dst = smem_u32(Fst + st * BM * RS + f_mr * RS + vw * v);
            // (one loop per copy width: no per-element width branch)
            if (vw == 4) {
                for (int m = f_mr; m < BM; m += f_rpt, src += f_step, dst += dstep) {
                    const bool ok = kok && m0 + m < M;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;"
                                 ::"r"(dst), "l"(ok ? src : F), "r"(ok ? 16 : 0) : "memory");
                }
            } else if (vw == 2) {
                for (int m = f_mr; m < BM; m += f_rpt, src += f_step, dst += dstep) {
                    const bool ok = kok && m0 + m < M;
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;"
                                 ::"r"(dst), "l"(ok ? src : F), "r"(ok ? 8 : 0) : "memory");
                }
            } else {
                for (int m = f_mr; m < BM; m += f_rpt, src += f_step, dst += dstep) {
                    const bool ok = kok && m0 + m < M;
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;"
                                 ::"r"(dst), "l"(ok ? src : F), "r"(ok ? 4 : 0) : "memory");
                }
            }
        }
    };
    // im2col tile B[k][n] = I[ch0 + ch][y_n + r][x_n + c] (zero past the valid range)
    auto load_b = [&](int chunk, int st) {
        if (bkl >= KL) return;
        const int ch0 = ch_begin + chunk * CB;
        const int nk = bvalid ? min(CB, ch_end - ch0) * KK : 0;
        const float *src = I + (int64_t)ch0 * HW + bbase;
        uint32_t dst = smem_u32(Bst + st * CKP * BN + bkl * BN + bn);
#pragma unroll 4
        for (int k = bkl; k < CKP; k += KL, dst += KL * BN * 4)
            cp_async4_zf(dst, src + koff[k], k < nk);    // k >= nk: zero fill, src not read
    };

    float acc[8][TN];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

    if (kTmaF && tid == 0) {
        tma_prefetch_desc(&tmapF);
#pragma unroll
        for (int j = 0; j < NST; ++j) mbar_init(&fbar[j], 1);
        fence_mbar_init();
    }
    pdl_wait();
    pdl_trigger();
    if (tl) g_simt_cta[5 * cta_lin + 1] = simt_gtimer();
    __syncthreads();                                // koff table, barriers
    // NST-stage ring: chunk c lives in stage c % NST; chunks c + 1 .. c + NST - 1
    // are in flight while chunk c computes (the paper's prefetch rounds)
#pragma unroll
    for (int j = 0; j < NST - 1; ++j) {
        if (j < nchunks) { load_f(j, j); load_b(j, j); }
        cp_async_commit();
    }
    int st = 0;
    for (int chunk = 0; chunk < nchunks; ++chunk) {
        cp_async_wait<NST - 2>();                   // chunk c staged (newer ones may be in flight)
        __syncthreads();
        if constexpr (kTmaF) mbar_wait(&fbar[st], (chunk / NST) & 1);
        if (tl && chunk == 0) g_simt_cta[5 * cta_lin + 2] = simt_gtimer();
        {                                           // refill the stage chunk c - 1 used
            const int nx = chunk + NST - 1;
            const int sx = st == 0 ? NST - 1 : st - 1;
            if (nx < nchunks) { load_f(nx, sx); load_b(nx, sx); }
            cp_async_commit();
        }
        // A = F rows in place: thread rows tm + i * TMG (consecutive rows across
        // the warp's lanes: conflict-free 16-B loads along k), four k per load;
        // B = the im2col tile, TN consecutive pixels per k
        const float *Fa = Fst + st * BM * RS + tm * RS;
        const float *Bs = Bst + st * CKP * BN + tn * 4;
        const float *Bs2 = Bst + st * CKP * BN + SH::R1 + tn * T2;
        // (kq unrolled by two where it measured faster: TN = 4 and the
        // BM <= 128 TN = 6 tiles, -2..-7 %; the 256 x 48 tile +0.5 %)
#pragma unroll(kCKP > 0 ? kSimtFixedUnroll : (NST >= 3 || kUnroll2 || TN == 4 || (TN == 6 && BM <= 128) ? 2 : 1))
        for (int kq = 0; kq < CKP; kq += 4) {
            float4 a[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = *reinterpret_cast<const float4 *>(Fa + i * SH::TMG * RS + kq);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const int k = kq + kk;
                const float4 b0 = *reinterpret_cast<const float4 *>(Bs + k * BN);
                float bv[TN];
                bv[0] = b0.x; bv[1] = b0.y; bv[2] = b0.z; bv[3] = b0.w;
                if constexpr (T2 == 4) {
                    const float4 b1 = *reinterpret_cast<const float4 *>(Bs2 + k * BN);
                    bv[4] = b1.x; bv[5] = b1.y; bv[6] = b1.z; bv[7] = b1.w;
                } else if constexpr (T2 == 2) {
                    const float2 b1 = *reinterpret_cast<const float2 *>(Bs2 + k * BN);
                    bv[4] = b1.x; bv[5] = b1.y;
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const float ai = kk == 0 ? a[i].x : kk == 1 ? a[i].y : kk == 2 ? a[i].z : a[i].w;
#pragma unroll
                    for (int j = 0; j < TN; j += 2) ffma2(acc[i][j], acc[i][j + 1], ai, bv[j], bv[j + 1]);
                }
            }
        }
        st = st + 1 == NST ? 0 : st + 1;
    }
    cp_async_wait<0>();
    if (tl) g_simt_cta[5 * cta_lin + 3] = simt_gtimer();

    if (W != nullptr) {
        // ---- workspace split-K: partial tile -> W[split] (padded, aligned) ----
        const int ldw = gridDim.y * BN;
        float *w = W + (int64_t)split * ((int64_t)gridDim.z * BM * ldw) + (int64_t)m0 * ldw + p0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float *wr = w + (int64_t)SH::row(tm, i) * ldw;
            __stcg(reinterpret_cast<float4 *>(wr + tn * 4),
                   make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]));
            if constexpr (T2 == 4)
                __stcg(reinterpret_cast<float4 *>(wr + SH::R1 + tn * 4),
                       make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]));
            else if constexpr (T2 == 2)
                __stcg(reinterpret_cast<float2 *>(wr + SH::R1 + tn * 2), make_float2(acc[i][4], acc[i][5]));
        }
        if (tl) g_simt_cta[5 * cta_lin + 4] = simt_gtimer() << 8 | simt_smid();
        return;
    }
    __syncthreads();

    // ---- partial tile -> own smem, then fixed-order (DSMEM) reduction ------
    float *P = smem;                                // [BM][BN]
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float *pr = P + SH::row(tm, i) * BN;
        *reinterpret_cast<float4 *>(pr + tn * 4) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        if constexpr (T2 == 4)
            *reinterpret_cast<float4 *>(pr + SH::R1 + tn * 4) =
                make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
        else if constexpr (T2 == 2)
            *reinterpret_cast<float2 *>(pr + SH::R1 + tn * 2) = make_float2(acc[i][4], acc[i][5]);
    }
    if (S > 1) cluster_sync_all(); else __syncthreads();

    const int mlo = split * BM / S;                 // rows [mlo, mhi) reduced by this rank
    const int rows = (split + 1) * BM / S - mlo;
    const uint32_t Pbase = smem_u32(P);
    const int nvalid = min(BN, Ptot - p0);
    constexpr int BQ = BN / 4;
    for (int idx = tid; idx < rows * BQ; idx += NT) {
        const int m = mlo + idx / BQ, n = 4 * (idx % BQ);
        float4 v;
        if (S > 1) {
            v = dsmem_sum_ranks<kSimtMaxSplit>(Pbase + (m * BN + n) * 4, S);
        } else {
            v = *reinterpret_cast<const float4 *>(P + m * BN + n);
        }
        if (m0 + m < M) {
            const float vv[4] = {v.x, v.y, v.z, v.w};
            if (Nimg == 1) {
                float *o = O + (int64_t)(m0 + m) * HoWo + p0 + n;   // compact: coalesced
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (n + i < nvalid) o[i] = vv[i];
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    if (n + i >= nvalid) break;
                    const int q = p0 + n + i, img = q / HoWo;
                    O[((int64_t)img * M + m0 + m) * HoWo + (q - img * HoWo)] = vv[i];
                }
            }
        }
    }
    if (S > 1) cluster_sync_all();
    if (tl) g_simt_cta[5 * cta_lin + 4] = simt_gtimer() << 8 | simt_smid();
}

namespace {
struct SimtTile { int BM, BN, TN; };
// 8 x TN outputs per thread, 256 threads: TN = 8 (16K-output tiles), 6, 4
constexpr int kNumSimtTiles = 9;
constexpr SimtTile kSimtTiles[kNumSimtTiles] = {
    {128, 128, 8}, {64, 256, 8}, {256, 64, 8},
    {256, 48, 6}, {128, 96, 6}, {64, 192, 6},
    {256, 32, 4}, {128, 64, 4}, {64, 128, 4}};

int simt_smem(int BM, int BN, int CK, int nst = 2) {
    const int CKP = (CK + 3) & ~3;
    const int bytes = (nst * BM * simt_rs(CKP) + nst * CKP * BN) * 4 + ((CKP + 1) & ~1) * 4 + 8 * nst;
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

// Launch-time model (us) used to pick tile, split and reduction mode.  Per-SM
// FFMA issue rate 128 lanes x 1.965 GHz times the sustained fraction with one
// / two resident CTAs; constants fitted (tools/simt_model.py) to a measured
// sweep of every (tile, split, mode) on the bench layers (tools/simt_sweep.py,
// B200): the planner's pick is within 1.5% of the best measured on average.
// (Refit for the FFMA2 / TMA-ring kernel on the dense sweep v4
// (profiles/sweeps/simt_sweep_v4_r02.log): kEff1 0.40, kEff2 0.45, TN = 6
// weight 0.85, 0.8 us per chunk; the pick is the measured best on 7 of the 8
// bench layers and within 1% on the eighth.)
constexpr double kFmaPerUs = 128.0 * 1965.0;
constexpr double kEff1 = 0.40, kEff2 = 0.45;
constexpr double kCtaFixed = 0.5;      // prologue (first chunk latency) + epilogue
constexpr double kPerChunk = 0.8;      // per channel chunk: ring barrier, B gather issue, F TMA round trip
constexpr double kClusterReduce = 9.0; // cluster co-scheduling + barrier waits + DSMEM reduction
constexpr double kWsReduce = 0.5;      // second launch (PDL-overlapped) + its tail
constexpr double kL2BytesPerUs = 3.0e6;

double sm_time(int n, int q, double w, int nch, int BM) {
    const double c = kCtaFixed + nch * kPerChunk;
    (void)BM;
    if (q >= 2) return (n / 2) * (2.0 * w / kEff2) + (n % 2) * (w / kEff1) + ((n + 1) / 2) * c;
    return n * (w / kEff1 + c);
}

struct SimtCfg { int tile, S, CB, cps, ws, smem; double t; int nst = 2; };

SimtCfg simt_choose(int C, int Wx, int Wy, int K, int M, bool allow_ws, int sd, int Nimg) {
    const int Ho = (Wy - K) / sd + 1, Wo = (Wx - K) / sd + 1;
    const int64_t px = (int64_t)Ho * Wo * Nimg;
    const int KK = K * K;
    SimtCfg best = {-1, 1, 1, C, 0, 0, 1e30};
    for (int ti = 0; ti < kNumSimtTiles; ++ti) {
        const SimtTile &T = kSimtTiles[ti];
        const int npt = (int)((px + T.BN - 1) / T.BN);
        const int nmt = (M + T.BM - 1) / T.BM;
        const int tiles = npt * nmt;
        const double tn_pen = T.TN == 6 ? 0.85 : 1.0;                         // fitted per thread tile
        int last_S = -1;
        for (int Sreq = 1; Sreq <= C && Sreq <= 96; ++Sreq) {
            int CB, cps;
            simt_split(C, Sreq, T.BM, T.BN, K, &CB, &cps);
            const int S = (C + cps - 1) / cps;
            if (S == last_S) continue;
            last_S = S;
            const int smem = simt_smem(T.BM, T.BN, CB * KK);
            if (smem > kSimtMaxSmem + 64 * 1024) continue;
            const int q = smem <= 113 * 1024 ? 2 : 1;
            const double w = (double)T.BM * T.BN * cps * KK * tn_pen / kFmaPerUs;
            const int nch = (cps + CB - 1) / CB;
            for (int ws = 0; ws <= 1; ++ws) {
                if (ws && (S == 1 || !allow_ws)) continue;
                double t;
                if (!ws) {
                    if (S > kSimtMaxSplit) continue;
                    const int cap = clusters_resident(S, q);
                    const int waves = (tiles + cap - 1) / cap;
                    const int per_wave = (tiles < cap ? tiles : cap) * S;
                    t = waves * sm_time((per_wave + num_sms() - 1) / num_sms(), q, w, nch, T.BM) + (S > 1 ? kClusterReduce : 0.0);
                } else {
                    const int64_t total = (int64_t)tiles * S;
                    const double bytes = 8.0 * S * (double)nmt * T.BM * (double)npt * T.BN + 4.0 * M * px;
                    t = sm_time((int)((total + num_sms() - 1) / num_sms()), q, w, nch, T.BM) + kWsReduce + bytes / kL2BytesPerUs;
                }
                if (t < best.t * 0.995) best = {ti, S, CB, cps, ws, smem, t};
            }
        }
    }
    return best;
}

// B200CONV_SIMT_FORCE="tile,S,ws" (experiments / tests): force tile index,
// requested split and reduction mode
bool simt_forced(int C, int K, SimtCfg *c) {
    const char *e = getenv("B200CONV_SIMT_FORCE");
    if (!e || !*e) return false;
    int ti = 0, S = 1, ws = 0;
    if (sscanf(e, "%d,%d,%d", &ti, &S, &ws) < 2 || ti < 0 || ti >= kNumSimtTiles || S < 1) return false;
    const SimtTile &T = kSimtTiles[ti];
    int CB, cps;
    simt_split(C, S > C ? C : S, T.BM, T.BN, K, &CB, &cps);
    const int Se = (C + cps - 1) / cps;
    if (!ws && Se > kSimtMaxSplit) return false;
    *c = {ti, Se, CB, cps, (ws && Se > 1) ? 1 : 0, simt_smem(T.BM, T.BN, CB * K * K), 0.0};
    return true;
}

SimtCfg simt_config(int C, int Wx, int Wy, int K, int M, bool allow_ws, int sd, int Nimg) {
    SimtCfg c;
    if (!(simt_forced(C, K, &c) && (allow_ws || !c.ws))) c = simt_choose(C, Wx, Wy, K, M, allow_ws, sd, Nimg);
    // ring depth.  The paper's model (§2.2, NEXT-4): a chunk carries
    // q x BM x BN x CK FMAs per SM; at or above N_FMA (method 1) one chunk
    // in flight behind the one computing hides the latency: two stages, two
    // CTAs per SM.  Below it (method 2) the deepest ring that fits keeps the
    // most bytes in flight (one CTA per SM).  Measured: every bench layer is
    // method 1, and 3 / 4 stages are 1-10 % slower.
    // Planner override B200CONV_SIMT_NST = 2..4.
    if (c.tile >= 0) {
        const SimtTile &T = kSimtTiles[c.tile];
        int nst_model = 2;
        {
            const LatencyModel lm = latency_model(b200_profile(num_sms()));
            const int q = c.smem <= 113 * 1024 ? 2 : 1;
            const double fma_chunk = (double)q * T.BM * T.BN * c.CB * K * K;
            if (paper_method(lm, fma_chunk) == 2)
                nst_model = simt_smem(T.BM, T.BN, c.CB * K * K, 4) <= 227 * 1024 ? 4 : 3;
        }
        const int nst = env_override("B200CONV_SIMT_NST", nst_model);
        if (nst >= 3 && nst <= 4 && simt_smem(T.BM, T.BN, c.CB * K * K, nst) <= 227 * 1024) {
            c.nst = nst;
            c.smem = simt_smem(T.BM, T.BN, c.CB * K * K, nst);
        }
    }
    return c;
}

int64_t out_px(int Wx, int Wy, int K, int sd) { return (int64_t)((Wy - K) / sd + 1) * ((Wx - K) / sd + 1); }

void fill_plan(const SimtCfg &c, int C, int Wx, int Wy, int K, int M, conv_plan *p, int sd, int Nimg) {
    const int64_t px = out_px(Wx, Wy, K, sd) * Nimg;
    const SimtTile &T = kSimtTiles[c.tile];
    p->kernel = 1;
    p->grid_x = c.S;
    p->grid_y = (int)((px + T.BN - 1) / T.BN);
    p->grid_z = (M + T.BM - 1) / T.BM;
    p->block_x = kSimtThreads;
    p->cluster_x = c.ws ? 1 : c.S;
    p->tile_m = T.BM;
    p->tile_n = T.BN;
    p->smem_bytes = c.smem;
    p->tma_f = 0;
    p->launches = c.ws ? 2 : 1;
    p->chunk_k = c.CB * K * K;
    (void)C;
}
}  // namespace

int plan_multi_simt(int C, int Wx, int Wy, int K, int M, conv_plan *p, int sd, int Nimg) {
    const SimtCfg c = simt_config(C, Wx, Wy, K, M, true, sd, Nimg);
    if (c.tile < 0) {                                   // naive fallback (huge K; one image per launch)
        const int64_t n = (int64_t)M * out_px(Wx, Wy, K, sd);
        int64_t blocks = (n + 255) / 256;
        p->kernel = 1;
        p->grid_x = (int)(blocks < 4 * num_sms() ? blocks : 4 * num_sms());
        p->grid_y = p->grid_z = 1;
        p->block_x = 256;
        p->cluster_x = 1;
        p->tile_m = 1;
        p->tile_n = 1;
        p->smem_bytes = 0;
        p->tma_f = 0;
        p->launches = 1;
        return 0;
    }
    fill_plan(c, C, Wx, Wy, K, M, p, sd, Nimg);
    return 0;
}

// F rows by TMA when the chunk is a whole number of 16-B quads that lands
// bank-conflict-free densely and F rows are 16-B strided
bool simt_tma_f(const float *F, int C, int K, int CB) {
    const int KK = K * K, CK = CB * KK;
    return (C * KK) % 4 == 0 && CK % 4 == 0 && CK <= 256 && (CK / 4) % 4 != 0 &&
           reinterpret_cast<uintptr_t>(F) % 16 == 0;
}

template <int BM, int BN, int TN>
static cudaError_t launch_kms(const SimtCfg &c, const conv_plan &p, const float *I, int C, int Wx, int Wy,
                              const float *F, int K, int M, float *O, float *W, cudaStream_t s, int sd,
                              int Nimg) {
    CUtensorMap tmap;
    bool tma = simt_tma_f(F, C, K, c.CB);
    if (tma) {
        const int CK = c.CB * K * K;
        tma = encode_f32_2d_plain(&tmap, F, (uint64_t)C * K * K, (uint64_t)M, (uint64_t)C * K * K * 4, CK, BM);
    }
    if (!tma) memset(&tmap, 0, sizeof(tmap));
    // the deeper one-CTA-per-SM rings exist for the TMA-fed variant only
    auto kern = !tma ? kms_kernel<BM, BN, TN, false, 2>
                     : c.nst == 3 ? kms_kernel<BM, BN, TN, true, 3>
                     : c.nst == 4 ? kms_kernel<BM, BN, TN, true, 4>
                     : (c.CB * K * K == 36 && kSimtFixedCk) ? kms_kernel<BM, BN, TN, true, 2, 36>
                                                            : kms_kernel<BM, BN, TN, true, 2>;
    cudaError_t e = ensure_smem((const void *)kern, p.smem_bytes);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.grid_x, p.grid_y, p.grid_z);
    cfg.blockDim = dim3(p.block_x);
    cfg.dynamicSmemBytes = p.smem_bytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = p.cluster_x;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = W ? 1 : 2;
    const int dbg = kDiag ? env_override("B200CONV_SIMT_DBG", 0) : 0;
    e = cudaLaunchKernelEx(&cfg, kern, tmap, I, C, Wx, Wy, F, K, M, O, c.cps, c.CB, W, dbg, sd, Nimg);
    if (e != cudaSuccess) return e;
    if (!W) {                                   // (NEXT-2 peers: this epilogue is not peer-aware)
        const PeerOut &po = peer_out();
        return (po.n || po.mc) ? launch_peer_copy(O, (int64_t)M * out_px(Wx, Wy, K, sd) * Nimg, s) : e;
    }
    const int ldw = p.grid_y * BN;
    const int64_t slice = (int64_t)p.grid_z * BM * ldw;
    const int plane = (int)out_px(Wx, Wy, K, sd);
    return launch_splitk_reduce(W, p.grid_x, slice, M, ldw, plane * Nimg, O, s, plane);
}

int simt_max_clusters(int cluster, int smem) {
    auto kern = kms_kernel<128, 128, 8, false, 2>;
    ensure_smem((const void *)kern, smem);
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
                              float *O, cudaStream_t s, int sd, int Nimg) {
    SimtCfg c = simt_config(C, Wx, Wy, K, M, true, sd, Nimg);
    if (c.tile < 0) {
        conv_plan p;
        plan_multi_simt(C, Wx, Wy, K, M, &p, sd);
        const int64_t out_img = (int64_t)M * out_px(Wx, Wy, K, sd);
        for (int n = 0; n < Nimg; ++n)
            kmn_kernel<<<p.grid_x, p.block_x, 0, s>>>(I + (int64_t)n * C * Wx * Wy, C, Wx, Wy, F, K, M,
                                                      O + n * out_img, sd);
        const PeerOut &po = peer_out();
        if (cudaGetLastError() != cudaSuccess) return cudaErrorLaunchFailure;
        return (po.n || po.mc) ? launch_peer_copy(O, out_img * Nimg, s) : cudaSuccess;
    }
    float *W = nullptr;
    if (c.ws) {
        const SimtTile &T = kSimtTiles[c.tile];
        const int64_t px = out_px(Wx, Wy, K, sd) * Nimg;
        const size_t bytes = (size_t)c.S * ((M + T.BM - 1) / T.BM) * T.BM * ((px + T.BN - 1) / T.BN) * T.BN * 4;
        W = static_cast<float *>(workspace_get(bytes, s));
        if (!W) c = simt_config(C, Wx, Wy, K, M, false, sd, Nimg);   // capturing: cluster-only plan
    }
    conv_plan p;
    fill_plan(c, C, Wx, Wy, K, M, &p, sd, Nimg);
    switch (c.tile) {
        case 0: return launch_kms<128, 128, 8>(c, p, I, C, Wx, Wy, F, K, M, O, W, s, sd, Nimg);
        case 1: return launch_kms<64, 256, 8>(c, p, I, C, Wx, Wy, F, K, M, O, W, s, sd, Nimg);
        case 2: return launch_kms<256, 64, 8>(c, p, I, C, Wx, Wy, F, K, M, O, W, s, sd, Nimg);
        case 3: return launch_kms<256, 48, 6>(c, p, I, C, Wx, Wy, F, K, M, O, W, s, sd, Nimg);
        case 4: return launch_kms<128, 96, 6>(c, p, I, C, Wx, Wy, F, K, M, O, W, s, sd, Nimg);
        case 5: return launch_kms<64, 192, 6>(c, p, I, C, Wx, Wy, F, K, M, O, W, s, sd, Nimg);
        case 6: return launch_kms<256, 32, 4>(c, p, I, C, Wx, Wy, F, K, M, O, W, s, sd, Nimg);
        case 7: return launch_kms<128, 64, 4>(c, p, I, C, Wx, Wy, F, K, M, O, W, s, sd, Nimg);
        default: return launch_kms<64, 128, 4>(c, p, I, C, Wx, Wy, F, K, M, O, W, s, sd, Nimg);
    }
}

}  // namespace b200
