// conv_multi_gemm.cu — kernel pair KM-TC/G: multi-channel direct convolution
// (§2.1 Eq. 1) on the tcgen05 tensor cores with BOTH operands
// fed by TMA (TF32 or BF16 inputs, FP32 accumulate).
//
//   X[p][k] = I[ch][(y*s + r)*Wx + x*s + c]   (k = (ch, r, c) = ch*K*K + r*K + c,
//                                              p = y*Wo + x compact, stride s)
//   D       = X . F^T               (F as stored: row-major [M][C*K*K])
//   O[m][y][x] = D[y*Wo + x][m]
//
// Why not the implicit kernel (conv_multi_tc.cu) for these layers: there the
// im2col tile of every k-block is rebuilt by eight warps for every filter
// tile, which makes the main loop shared-memory-bandwidth bound (patch read
// + tile write + MMA read per element) at ~0.45 us per k-block, i.e. 10-40 %
// of the tensor pipe.  The im2col matrix of the paper's layers is small
// (0.9-7 MB, it stays in the 126 MB L2), so kernel 1 writes it ONCE per call
// and kernel 2 is a plain warp-specialised TMA -> tcgen05 GEMM: one thread
// issues the TMA loads of both operands (SWIZZLE_128B, K-major, straight
// into the canonical UMMA layout), one thread issues tcgen05.mma into TMEM,
// four warps drain TMEM.  The k-order (ch, r, c) is the filter layout of the
// paper, so F is never re-laid out.
//
// Two operand roles (chosen per layer by the planner):
//  * mode P (pixels on the 128-lane M side): A = X tile (128 pixels),
//    B = F tile (BN filters); many-pixel layers.
//  * mode F (filters on M): A = F tile (128 filters), B = X tile (all wide
//    pixels of the map, N <= 256); few-pixel layers (ResNet 14x14 / 7x7, the
//    configs[4] sweep): every F element is read from HBM exactly once.
// Small layers split the k loop over a thread-block cluster; the partial tile
// leaves by one bulk store to an L2 workspace and each rank bulk-loads its
// slice of every partial and sums them in rank order (deterministic).
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>
#include "kernels.h"
#include "ptx.cuh"

namespace b200 {

constexpr int kGmThreads = 192;       // warp 0 TMA producer, warp 1 MMA + TMEM, warps 2..5 epilogue
constexpr int kGmBM = 128;            // UMMA M
constexpr int kGmMaxSplit = 16;
constexpr int kGmMaxStages = 8;
constexpr int kGmSmemMax = 225 * 1024;

// ---------------------------------------------------------------- kernel 1
// X[p][k] for p < P, k < Kp (row stride Kp; zero for k >= C*K*K and outside
// the channel).  One 16-B vector of consecutive k per thread: coalesced rows.
// Pixel p = y*Wp + x (compact, Wp = Wo) reads input row y*sd, column x*sd.
// Batched (strided calls): pixels p < Ptot = N*Pimg, image n = p / Pimg reads
// I[n]; rows Ptot <= p < P are zero.
template <typename T>
struct Im2col {
    const T *I;
    int C, Wx, Wy, K, Kp, sd, Wp, Pimg, Ptot;
    // the 16-B vector kv (V = 16 / sizeof(T) consecutive k) of X row pg
    __device__ __forceinline__ uint4 vec(int pg, int kv) const {
        constexpr int V = 16 / sizeof(T);
        const int KK = K * K, HW = Wx * Wy, Ktot = C * KK;
        const int n = pg / Pimg, p = pg - n * Pimg;          // image, pixel within the image
        const T *In = I + (int64_t)n * C * HW;
        const int py = p / Wp;
        const int base = sd * (py * Wx + (p - py * Wp));   // input offset of the pixel's window
        const bool live = pg < Ptot;
        int k = kv * V;
        int ch = k / KK, rem = k - ch * KK, r = rem / K, c = rem - r * K;
        union { uint4 u; T e[V]; } v;
#pragma unroll
        for (int e = 0; e < V; ++e) {
            const int off = base + r * Wx + c;
            v.e[e] = (live && k < Ktot && off < HW) ? In[(int64_t)ch * HW + off] : T(0.f);
            ++k;
            if (++c == K) { c = 0; if (++r == K) { r = 0; ++ch; } }
        }
        return v.u;
    }
};

template <typename T>
__global__ void __launch_bounds__(256)
im2col_kernel(const Im2col<T> a, int P, T *__restrict__ X) {
    constexpr int V = 16 / sizeof(T);
    const int nv = a.Kp / V;
    const int64_t total = (int64_t)P * nv;
    pdl_wait();
    pdl_trigger();
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int pg = (int)(idx / nv), kv = (int)(idx - (int64_t)pg * nv);
        *reinterpret_cast<uint4 *>(X + (int64_t)pg * a.Kp + (int64_t)kv * V) = a.vec(pg, kv);
    }
}

// ---------------------------------------------------------------- kernel 2
struct GmArgs {
    int nkb;          // k-blocks of the whole reduction
    int kbps;         // k-blocks per split
    int M, Ho, Wo, Wx;
    int N;            // images (strided batched calls: compact pixels p = (n*Ho + y)*Wo + x)
    int stages, stage_bytes;
    float *O;
    float *Wk;        // split-K partials [S][tiles][BN][PS] (nullptr: DSMEM reduction)
    PeerOut po;       // NEXT-2: extra / multicast destinations of every O store
    int dbg;          // diagnostics (kDiag builds only)
};

// Filters-on-M partial / transpose tile in shared memory: [BN pixels][kGmPS]
// floats, filter rows contiguous (the 4-float pad keeps both the row-per-lane
// writes from TMEM and the pixel-per-lane float4 reads conflict-free).
constexpr int kGmPS = kGmBM + 4;
#ifndef B200CONV_GM_OWN_GRAIN
#define B200CONV_GM_OWN_GRAIN 8
#endif
constexpr int kGmOwnGrain = B200CONV_GM_OWN_GRAIN;   // split-K rank pixel ranges: whole groups of this many

// diagnostics (-DB200CONV_DIAG builds, B200CONV_GM_DBG=1): per-CTA globaltimer
// stamps [start, after griddepcontrol.wait, first stage full (MMA warp),
// MMAs done (epilogue), partial stored (workspace split), cluster barrier
// passed, end << 8 | smid, partial slices loaded (workspace split)]
__device__ unsigned long long g_gm_cta[8 * 1024];
__device__ unsigned long long g_gm_loop[8 * 1024];   // clock64 at each store-loop iteration (thread 0)
int gm_read_cta_stamps(unsigned long long *host) {
    return cudaMemcpyFromSymbol(host, g_gm_cta, sizeof(g_gm_cta)) == cudaSuccess &&
                   cudaMemcpyFromSymbol(host + 8 * 1024, g_gm_loop, sizeof(g_gm_loop)) == cudaSuccess
               ? 0 : 1;
}
__device__ __forceinline__ unsigned long long gm_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Rank-ordered sum of the S partial tiles' float4 at local_addr across the
// cluster (DSMEM).  Out of line: the epilogue runs once per CTA, so its code
// is fetched cold; keeping the loop body small keeps that fetch short.
__device__ __noinline__ float4 gm_dsmem_sum(uint32_t local_addr, int S) {
    float4 v = ld_dsmem_f32x4(mapa_shared(local_addr, 0u));
#pragma unroll 1
    for (int t = 1; t < S; ++t) {
        const float4 u = ld_dsmem_f32x4(mapa_shared(local_addr, (uint32_t)t));
        v.x += u.x; v.y += u.y; v.z += u.z; v.w += u.w;
    }
    return v;
}

template <bool kTF32, int BN, bool kModeF>
__global__ void __launch_bounds__(kGmThreads, 1)
gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const GmArgs g) {
    constexpr int ELEM = kTF32 ? 4 : 2;
    constexpr int BK = 128 / ELEM;                    // k per stage: one 128-B swizzle row
    constexpr int UK = 32 / ELEM;                     // k per tcgen05.mma
    constexpr int A_BYTES = kGmBM * 128;
    constexpr int B_BYTES = BN * 128;
    constexpr uint32_t IDESC = umma_idesc(kTF32 ? 2u : 1u, kGmBM, BN);
    constexpr uint32_t TCOLS = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));

    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t *smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    const int NS = g.stages, STAGE = g.stage_bytes;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + NS * STAGE);
    uint64_t *empty = full + kGmMaxStages;
    uint64_t *tmem_full = empty + kGmMaxStages;
    uint64_t *red_bar = tmem_full + 1;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(red_bar + 1);
    float *P = reinterpret_cast<float *>(smem);       // partial / transpose tile, aliases the stages

    const int S = gridDim.x, split = blockIdx.x;
    const int a0 = blockIdx.y * kGmBM;                // first A row of the tile
    const int b0 = blockIdx.z * BN;                   // first B row
    const int tile_lin = blockIdx.y + gridDim.y * blockIdx.z;
    const int kb0 = split * g.kbps;
    const int kb1 = min(g.nkb, kb0 + g.kbps);
    const int niter = kb1 > kb0 ? kb1 - kb0 : 0;
    const uint32_t warp = warp_id(), lane = lane_id();
    const unsigned cta_lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    const bool tl = kDiag && g.dbg && cta_lin < 1024;
    if (tl && threadIdx.x == 0) g_gm_cta[8 * cta_lin] = gm_gtimer();

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        mbar_init(tmem_full, 1);
        mbar_init(red_bar, 1);
        fence_mbar_init();
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
    }
    if (warp == 1) tmem_alloc<TCOLS>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();                                       // kernel 1 (im2col) complete and visible
    pdl_trigger();
    if (tl && threadIdx.x == 0) g_gm_cta[8 * cta_lin + 1] = gm_gtimer();

    if (warp == 0) {
        // -------------------------------------------- TMA producer
        if (lane == 0) {
            for (int i = 0; i < niter; ++i) {
                const int s = i % NS;
                mbar_wait(&empty[s], ((i / NS) & 1) ^ 1);
                uint8_t *st = smem + s * STAGE;
                const int k0 = (kb0 + i) * BK;
                mbar_arrive_expect_tx(&full[s], A_BYTES + B_BYTES);
                tma_load_2d(st, &tmA, &full[s], k0, a0);
                tma_load_2d(st + A_BYTES, &tmB, &full[s], k0, b0);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // -------------------------------------------- MMA issuer
        if (lane == 0) {
            for (int i = 0; i < niter; ++i) {
                const int s = i % NS;
                mbar_wait(&full[s], (i / NS) & 1);
                tc_fence_after();
                if (tl && i == 0) g_gm_cta[8 * cta_lin + 2] = gm_gtimer();
                const uint32_t a_addr = smem_u32(smem + s * STAGE);
                const uint32_t b_addr = a_addr + A_BYTES;
#pragma unroll
                for (int kk = 0; kk < BK / UK; ++kk)
                    umma_ss<kTF32>(tmem, umma_desc_k_sw128(a_addr + kk * 32), umma_desc_k_sw128(b_addr + kk * 32),
                                   IDESC, (i > 0 || kk > 0) ? 1u : 0u);
                umma_commit(&empty[s]);
            }
            umma_commit(tmem_full);
        }
        __syncwarp();
    } else {
        // -------------------------------------------- epilogue (warps 2..5)
        const int q = (int)(warp & 3);                // TMEM lane quarter
        const int row = q * 32 + (int)lane;           // A row within the tile == TMEM lane
        const int plane = g.Ho * g.Wo;
        if (niter > 0) {
            mbar_wait(tmem_full, 0);
            tc_fence_after();
        }
        if (tl && warp == 2 && lane == 0) g_gm_cta[8 * cta_lin + 3] = gm_gtimer();
        constexpr int NCB = (BN + 31) / 32;           // 32-column blocks; BN % 32 == 16: a 16-column tail
#pragma unroll 1
        for (int cb = 0; cb < NCB; ++cb) {
            uint32_t r[32];
            const int ncol = (BN % 32 != 0 && cb == NCB - 1) ? BN % 32 : 32;
            if (niter > 0 && ncol == 32) {
                tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(cb * 32), r);
                tmem_ld_wait();
            } else if (niter > 0) {
                tmem_ld_32x32b_x16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(cb * 32), r);
                tmem_ld_wait();
#pragma unroll
                for (int j = 16; j < 32; ++j) r[j] = 0u;
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) r[j] = 0u;
            }
            if constexpr (kModeF) {
                // row = filter, column = pixel: P[pixel][filter] (stored below,
                // pixel-fastest, so every warp store is one run of pixels)
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (j < ncol) P[(cb * 32 + j) * kGmPS + row] = __uint_as_float(r[j]);
            } else if (S == 1) {
                // row = pixel, columns = filters b0 + cb*32 + j
                const int p = a0 + row;
                int y = p / g.Wx;
                const int x = p - y * g.Wx, n = y / g.Ho;      // n = image (0 unless batched)
                y -= n * g.Ho;
                if (n < g.N && x < g.Wo) {
                    const int64_t o = (int64_t)n * g.M * plane + (int64_t)y * g.Wo + x;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int m = b0 + cb * 32 + j;
                        if (m < g.M) out_store(g.po, g.O, o + (int64_t)m * plane, __uint_as_float(r[j]));
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (j < ncol) P[(cb * 32 + j) * kGmBM + row] = __uint_as_float(r[j]);
            }
        }
        if (S > 1 && g.Wk) fence_proxy_async_smem();    // P -> visible to the bulk store
        tc_fence_before();
    }
    __syncthreads();

    if constexpr (kModeF) {
        // ---------------------------------------------- store / split-K reduction
        // rank `split` owns pixels [nlo, nhi) of the tile (all S ranks' partials
        // summed in rank order: deterministic); threads run along pixels, so
        // each of the four filter rows a thread stores is a coalesced warp
        // store.  The ranges are whole 8-pixel groups: every 8 lanes write one
        // full 32-B sector (a sector written in parts costs a DRAM
        // read-modify-write; measured configs[4] BF16: the O stores took
        // ~8 us of the call with 36-pixel ranges)
        const int plane = g.Ho * g.Wo;
        constexpr int G = kGmOwnGrain;
        const int nlo = (split * (BN / G) / S) * G;
        const int nhi = split == S - 1 ? BN : ((split + 1) * (BN / G) / S) * G, np = nhi - nlo;
        const float *src = P;                         // [.][kGmPS] rows of pixel nlo.. (local / workspace)
        int src_p0 = 0;
        if (S > 1 && g.Wk) {
            if (threadIdx.x == 0) {
                bulk_store(g.Wk + ((int64_t)split * gridDim.y * gridDim.z + tile_lin) * BN * kGmPS, P,
                           (uint32_t)(BN * kGmPS * 4));
                bulk_commit();
                bulk_wait<0>();
                fence_proxy_async_global();
                if (tl) g_gm_cta[8 * cta_lin + 4] = gm_gtimer();
            }
            cluster_sync_all();
            if (tl && threadIdx.x == 0) g_gm_cta[8 * cta_lin + 5] = gm_gtimer();
            if (threadIdx.x == 0) {
                const int64_t wslice = (int64_t)gridDim.y * gridDim.z * BN * kGmPS;
                const float *wt = g.Wk + ((int64_t)tile_lin * BN + nlo) * kGmPS;
                const uint32_t bytes = (uint32_t)(np * kGmPS * 4);
                mbar_arrive_expect_tx(red_bar, bytes * S);
                if (np > 0)
                    for (int t = 0; t < S; ++t) bulk_load(P + t * np * kGmPS, wt + t * wslice, bytes, red_bar);
            }
            mbar_wait(red_bar, 0);
            if (tl && threadIdx.x == 0) g_gm_cta[8 * cta_lin + 7] = gm_gtimer();
            src_p0 = nlo;
        } else if (S > 1) {
            cluster_sync_all();                       // every rank's partial is in its smem
            if (tl && threadIdx.x == 0) g_gm_cta[8 * cta_lin + 5] = gm_gtimer();
        }
        const uint32_t Pbase = smem_u32(P);
        // items (filter quad qd, pixel p) dealt round-robin to the threads,
        // four per thread per batch: all their shared-memory loads issue
        // before the sums and stores (the loop ran once per CTA, latency-bound
        // at ~700 clk per item with one item in flight); item indices advance
        // without divisions
        const int total = np * (kGmBM / 4);
        int qd = np > 0 ? (int)threadIdx.x / np : 0, pp = (int)threadIdx.x - qd * np;
        const int dq = np > 0 ? kGmThreads / np : 0, dp = kGmThreads - dq * np;
        int it_dbg = 0;
        for (int idx0 = threadIdx.x; idx0 < ((kDiag && (g.dbg & 4)) ? 0 : total); idx0 += 4 * kGmThreads) {
            if (tl && threadIdx.x == 0 && it_dbg < 8) g_gm_loop[8 * cta_lin + it_dbg++] = clock64();
            float4 v[4];
            int qv[4], pv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                qv[u] = qd;
                pv[u] = nlo + pp;
                if (idx0 + u * kGmThreads < total) {
                    if (S > 1 && g.Wk) {
                        const float *sl = src + (pv[u] - src_p0) * kGmPS + 4 * qd;
                        v[u] = *reinterpret_cast<const float4 *>(sl);
#pragma unroll 4
                        for (int t = 1; t < S; ++t) {
                            const float4 w = *reinterpret_cast<const float4 *>(sl + t * np * kGmPS);
                            v[u].x += w.x; v[u].y += w.y; v[u].z += w.z; v[u].w += w.w;
                        }
                    } else if (S > 1) {
                        v[u] = gm_dsmem_sum(Pbase + (uint32_t)((pv[u] * kGmPS + 4 * qd) * 4), S);
                    } else {
                        v[u] = *reinterpret_cast<const float4 *>(P + pv[u] * kGmPS + 4 * qd);
                    }
                }
                pp += dp;
                qd += dq;
                if (pp >= np) { pp -= np; ++qd; }
            }
            if (kDiag && (g.dbg & 2)) continue;       // (diag: no O stores)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (idx0 + u * kGmThreads >= total) break;
                const int m0 = a0 + 4 * qv[u];
                const int pg = b0 + pv[u];            // compact pixel over all images
                const int n = g.N > 1 ? pg / plane : (pg < plane ? 0 : 1);   // rows past the map: n = N
                if (n >= g.N) continue;
                const int64_t o = ((int64_t)n * g.M + m0) * plane + (pg - n * plane);
                const float vv[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
                if (!g.po.mc && g.po.n == 0 && m0 + 3 < g.M) {
                    float *op = g.O + o;
                    op[0] = vv[0]; op[plane] = vv[1]; op[2 * plane] = vv[2]; op[3 * plane] = vv[3];
                } else {
#pragma unroll 1
                    for (int e = 0; e < 4; ++e)
                        if (m0 + e < g.M) out_store(g.po, g.O, o + (int64_t)e * plane, vv[e]);
                }
            }
        }
        if (S > 1 && !g.Wk) cluster_sync_all();      // keep this CTA's partial alive for the others
    } else if (S > 1) {
        // ---------------------------------------------- split-K reduction (pixels on M)
        if (g.Wk && threadIdx.x == 0) {
            bulk_store(g.Wk + ((int64_t)split * gridDim.y * gridDim.z + tile_lin) * BN * kGmBM, P,
                       (uint32_t)(BN * kGmBM * 4));
            bulk_commit();
            bulk_wait<0>();
            fence_proxy_async_global();
        }
        cluster_sync_all();
        if (tl && threadIdx.x == 0) g_gm_cta[8 * cta_lin + 5] = gm_gtimer();
        const int nlo = split * BN / S;               // columns [nlo, nhi) reduced by this rank
        const int rows = (split + 1) * BN / S - nlo;
        float *slices = P;                            // [S][rows][128]
        if (g.Wk) {
            if (threadIdx.x == 0) {
                const int64_t wslice = (int64_t)gridDim.y * gridDim.z * BN * kGmBM;
                const float *wt = g.Wk + ((int64_t)tile_lin * BN + nlo) * kGmBM;
                const uint32_t bytes = (uint32_t)(rows * kGmBM * 4);
                mbar_arrive_expect_tx(red_bar, bytes * S);
                for (int t = 0; t < S; ++t) bulk_load(slices + t * rows * kGmBM, wt + t * wslice, bytes, red_bar);
            }
            mbar_wait(red_bar, 0);
        }
        const uint32_t Pbase = smem_u32(P);
        const int plane = g.Ho * g.Wo;
        for (int idx = threadIdx.x; idx < rows * (kGmBM / 4); idx += kGmThreads) {
            const int nl = nlo + idx / (kGmBM / 4), row0 = 4 * (idx % (kGmBM / 4));
            float4 v;
            if (g.Wk) {
                const float *sl = slices + (nl - nlo) * kGmBM + row0;
                v = *reinterpret_cast<const float4 *>(sl);
                for (int t = 1; t < S; ++t) {
                    const float4 u = *reinterpret_cast<const float4 *>(sl + t * rows * kGmBM);
                    v.x += u.x; v.y += u.y; v.z += u.z; v.w += u.w;
                }
            } else {
                v = dsmem_sum_ranks<kGmMaxSplit>(Pbase + (uint32_t)((nl * kGmBM + row0) * 4), S);
            }
            const float vv[4] = {v.x, v.y, v.z, v.w};
            // column = filter, rows = 4 pixels
            const int m = b0 + nl;
            if (m < g.M) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int p = a0 + row0 + e;
                    int y = p / g.Wx;
                    const int x = p - y * g.Wx, n = y / g.Ho;
                    y -= n * g.Ho;
                    if (n < g.N && x < g.Wo) out_store(g.po, g.O, ((int64_t)n * g.M + m) * plane + y * g.Wo + x, vv[e]);
                }
            }
        }
        if (!g.Wk) cluster_sync_all();                // keep this CTA's partial alive for the others
    }
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<TCOLS>(tmem);
    }
    if (tl && threadIdx.x == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_gm_cta[8 * cta_lin + 6] = gm_gtimer() << 8 | smid;
    }
}

// ---------------------------------------------------------------- host side
namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

bool encode_2d(CUtensorMap *m, bool tf32, const void *base, uint64_t inner, uint64_t outer, uint64_t stride_bytes,
               uint32_t box_inner, uint32_t box_outer) {
    auto enc = encode_fn();
    if (!enc) return false;
    memset(m, 0, sizeof(*m));
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {stride_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, tf32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
               const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool encode_f32_2d_plain(CUtensorMap *m, const void *base, uint64_t inner, uint64_t outer, uint64_t stride_bytes,
                         uint32_t box_inner, uint32_t box_outer) {
    auto enc = encode_fn();
    if (!enc) return false;
    memset(m, 0, sizeof(*m));
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {stride_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

namespace {
// pixel-side tile width (mode F: N of the MMA): the smallest instantiated
// width >= n (every X byte a CTA streams is TMA ingest, ~53 B/clk per SM)
int round_bn(int n) {
    return n <= 32 ? 32 : (n <= 64 ? 64 : (n <= 128 ? 128 : (n <= 144 ? 144 : (n <= 160 ? 160 : (n <= 192 ? 192 : 256)))));
}

struct GmPlan {
    bool ok, modeF;
    int BN, S, tilesA, tilesB, nkb, kbps, Prows, Kp, stages, stage_bytes, smem;
    size_t x_bytes, w_bytes;
};

// sd > 1 (strided calls): compact pixels, and this path is taken whenever it
// is legal (the implicit kernel is stride-1 only)
GmPlan gm_plan(int C, int Wx, int Wy, int K, int M, bool bf16, int sd = 1, int N = 1) {
    GmPlan p = {};
    const int elem = bf16 ? 2 : 4, BK = 128 / elem;
    const int Ho = (Wy - K) / sd + 1;
    const int64_t Ktot = (int64_t)C * K * K;
    // (wide) pixels that carry outputs; strided calls: compact, all N images
    // compact output pixels (p = (n*Ho + y)*Wo + x) of all N images: no wide
    // columns x >= Wo in the X operand (the sweep: 144 instead of 168 rows)
    const int64_t Pw = (int64_t)Ho * N * ((Wx - K) / sd + 1);
    // F rows must be TMA-able (strided calls re-stride them instead: launch_multi_gemm)
    if (((Ktot * elem) % 16 != 0 && sd == 1) || Ktot > (1 << 24) || Pw > (1 << 24)) return p;
    p.Kp = (int)((Ktot + BK - 1) / BK * BK);
    p.nkb = p.Kp / BK;
    p.modeF = Pw <= 256;
    if (p.modeF) {
        p.BN = round_bn((int)Pw);
        p.tilesA = (M + kGmBM - 1) / kGmBM;
        p.tilesB = 1;
        p.Prows = p.BN;
    } else {
        p.BN = M <= 64 ? 64 : (M <= 128 ? 128 : 256);
        p.tilesA = (int)((Pw + kGmBM - 1) / kGmBM);
        p.tilesB = (M + p.BN - 1) / p.BN;
        p.Prows = p.tilesA * kGmBM;
    }
    // Measured (tools/mc_variants.py, B200): per-SM TMA ingest is ~53 B/clk,
    // so a tile pays for every operand byte it streams.  The explicit-im2col
    // GEMM wins where the implicit kernel's per-filter-tile patch rebuild is
    // the cost and the X tile is shared by many filter tiles: filters on M
    // with >= 4 filter tiles (ResNet 7x7: 8.4 vs 11.8 us bf16; configs[4]
    // sweep: 24.4 vs 30.2 us bf16).  Pixels-on-M layers stay on the implicit
    // kernel (e.g. 28x28x256: 10.1 vs 16.9 us), B200CONV_GM=2 forces this path.
    // TF32 (round 2, tools/gm_vs_implicit.py): the GEMM re-streams a 4-byte X
    // tile per filter tile; where the implicit kernel's wide-pixel waste is
    // small ((K-1)/Wx <= 1/6: the 14x14 layers, 17 %) it builds A on chip for
    // less — configs[4] at M = 4096 / 2048 / 1024 / 512: 27.8 / 19.8 / 15.7 /
    // 12.3 us against 32.5 / 23.0 / 18.2 / 15.5 us.  BF16 keeps the GEMM
    // (24.4 vs 29.0 us at M = 4096), as do the 7x7 layers (40 % waste).
    const bool tf32_implicit = !bf16 && 6 * (K - 1) <= Wx;
    if ((!(p.modeF && p.tilesA >= 4) || tf32_implicit) && env_override("B200CONV_GM", 1) != 2 && sd == 1) return p;
    const int tiles = p.tilesA * p.tilesB;
    // split the k loop over a cluster: fill the SMs, >= 2 k-blocks per split,
    // and only when the saved k-loop time beats the ~3 us partial exchange
    int S = tiles >= num_sms() ? 1 : num_sms() / tiles;
    if (S > kGmMaxSplit) S = kGmMaxSplit;
    if (S > p.nkb / 2) S = p.nkb / 2 > 0 ? p.nkb / 2 : 1;
    while (S > 1 && tiles > clusters_resident(S, 1)) --S;
    if (S > 1 && p.nkb <= 8) S = 1;
    if (const int v = env_override("B200CONV_GM_SPLIT", 0); v >= 1 && v <= kGmMaxSplit) S = v;
    p.kbps = (p.nkb + S - 1) / S;
    p.S = (p.nkb + p.kbps - 1) / p.kbps;
    p.stage_bytes = kGmBM * 128 + p.BN * 128;
    int ns = (kGmSmemMax - 1024 - 256) / p.stage_bytes;
    p.stages = ns > kGmMaxStages ? kGmMaxStages : ns;
    p.smem = 1024 + p.stages * p.stage_bytes + 256;
    // the partial / transpose tile (plus the workspace slices' rounding) aliases the stages
    const int ptile = p.modeF ? (p.BN + kGmOwnGrain * p.S) * kGmPS * 4 : p.BN * kGmBM * 4;
    if (p.stages < 2 || ptile > p.stages * p.stage_bytes) return p;
    p.x_bytes = ((size_t)p.Prows * p.Kp * elem + 1023) & ~(size_t)1023;
    p.w_bytes = p.S > 1 ? (size_t)p.S * tiles * p.BN * (p.modeF ? kGmPS : kGmBM) * 4 : 0;

    p.ok = true;
    return p;
}

template <bool kTF32, int BN, bool kModeF>
cudaError_t launch_gemm(const GmPlan &p, const CUtensorMap &ta, const CUtensorMap &tb, const GmArgs &g,
                        cudaStream_t s) {
    auto kern = gemm_kernel<kTF32, BN, kModeF>;
    cudaError_t e = ensure_smem((const void *)kern, p.smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.S, p.tilesA, p.tilesB);
    cfg.blockDim = dim3(kGmThreads);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled();
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kern, ta, tb, g);
}

template <bool kTF32, bool kModeF>
cudaError_t launch_gemm_bn(const GmPlan &p, const CUtensorMap &ta, const CUtensorMap &tb, const GmArgs &g,
                           cudaStream_t s) {
    switch (p.BN) {
        case 32: return launch_gemm<kTF32, 32, kModeF>(p, ta, tb, g, s);
        case 64: return launch_gemm<kTF32, 64, kModeF>(p, ta, tb, g, s);
        case 144: return launch_gemm<kTF32, 144, kModeF>(p, ta, tb, g, s);
        case 160: return launch_gemm<kTF32, 160, kModeF>(p, ta, tb, g, s);
        case 128: return launch_gemm<kTF32, 128, kModeF>(p, ta, tb, g, s);
        case 192: return launch_gemm<kTF32, 192, kModeF>(p, ta, tb, g, s);
        default: return launch_gemm<kTF32, 256, kModeF>(p, ta, tb, g, s);
    }
}
}  // namespace

int plan_multi_gemm(int C, int Wx, int Wy, int K, int M, bool bf16, conv_plan *out, int sd, int N) {
    const GmPlan p = gm_plan(C, Wx, Wy, K, M, bf16, sd, sd > 1 ? N : 1);
    if (!p.ok) return 1;
    out->kernel = 3;
    out->grid_x = p.S;
    out->grid_y = p.tilesA;
    out->grid_z = p.tilesB;
    out->block_x = kGmThreads;
    out->cluster_x = p.S;
    out->tile_m = p.modeF ? kGmBM : p.BN;               // filters per tile
    out->tile_n = p.modeF ? p.BN : kGmBM;               // pixels per tile
    out->smem_bytes = p.smem;
    out->tma_f = 1 | 4 | (p.modeF ? 8 : 0);             // F by TMA, X (im2col) by TMA, filters-on-M
    out->launches = 2;
    return 0;
}

// Returns cudaErrorNotSupported when the shape / alignment / workspace does
// not allow this path (the caller then uses the implicit kernel).
cudaError_t launch_multi_gemm(const void *I, int C, int Wx, int Wy, const void *F, int K, int M, float *O,
                              bool bf16, cudaStream_t s, int sd, int N) {
    if (sd == 1) N = 1;                                     // stride 1: one image (the implicit kernel batches)
    const GmPlan p = gm_plan(C, Wx, Wy, K, M, bf16, sd, N);
    if (!p.ok) return cudaErrorNotSupported;
    const int64_t Ktot0 = (int64_t)C * K * K;
    // strided calls have no other tensor-core path: filter rows that are not
    // 16-B strided / aligned are first copied to [M][Kp] with zero tails
    const bool fpad = ((Ktot0 * (bf16 ? 2 : 4)) % 16 != 0) || (reinterpret_cast<uintptr_t>(F) % 16) != 0;
    if (fpad && sd == 1) return cudaErrorNotSupported;
    if (env_override("B200CONV_GM", 1) == 0 && sd == 1) return cudaErrorNotSupported;
    const int Ho = (Wy - K) / sd + 1, Wo = (Wx - K) / sd + 1;
    const int Wp = Wo;                                      // compact pixel rows
    const int elem = bf16 ? 2 : 4;
    // split-K exchange: the L2 workspace round trip (measured faster than
    // DSMEM even at S = 4 here: configs[4] BF16 21.6 vs 23.0 us);
    // B200CONV_GM_DSMEM = 1 exchanges through DSMEM instead
    const bool dsmem = p.S > 1 && env_override("B200CONV_GM_DSMEM", 0) == 1;
    uint8_t *ws = static_cast<uint8_t *>(workspace_get(p.x_bytes + (dsmem ? 0 : p.w_bytes), s));
    if (!ws) return cudaErrorNotSupported;
    void *X = ws;
    float *Wk = p.S > 1 && !dsmem ? reinterpret_cast<float *>(ws + p.x_bytes) : nullptr;
    int64_t Ktot = Ktot0;
    if (fpad) {
        void *Fp = auxbuf_get((size_t)M * p.Kp * elem, s);
        if (!Fp) return cudaErrorNotSupported;
        cudaError_t e = launch_pad_rows(F, M, (int)Ktot0, p.Kp, elem, Fp, s);
        if (e != cudaSuccess) return e;
        F = Fp;
        Ktot = p.Kp;
    }
    CUtensorMap tf, tx;
    const int BK = 128 / elem;
    const int frows = p.modeF ? kGmBM : p.BN, xrows = p.modeF ? p.BN : kGmBM;
    if (!encode_2d(&tf, !bf16, F, (uint64_t)Ktot, (uint64_t)M, (uint64_t)Ktot * elem, BK, frows) ||
        !encode_2d(&tx, !bf16, X, (uint64_t)p.Kp, (uint64_t)p.Prows, (uint64_t)p.Kp * elem, BK, xrows))
        return cudaErrorNotSupported;
    Im2col<float> im32 = {static_cast<const float *>(I), C, Wx, Wy, K, p.Kp, sd, Wp, Ho * Wp, N * Ho * Wp};
    Im2col<__nv_bfloat16> im16 = {static_cast<const __nv_bfloat16 *>(I), C, Wx, Wy, K, p.Kp, sd, Wp, Ho * Wp,
                                  N * Ho * Wp};
    {
        // kernel 1: im2col into the (L2-resident) workspace
        const int64_t vecs = (int64_t)p.Prows * (p.Kp / (16 / elem));
        int blocks = (int)((vecs + 255) / 256);
        if (blocks > 8 * num_sms()) blocks = 8 * num_sms();
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(blocks);
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaError_t e = bf16 ? cudaLaunchKernelEx(&cfg, im2col_kernel<__nv_bfloat16>, im16, p.Prows,
                                                  static_cast<__nv_bfloat16 *>(X))
                             : cudaLaunchKernelEx(&cfg, im2col_kernel<float>, im32, p.Prows, static_cast<float *>(X));
        if (e != cudaSuccess) return e;
    }
    GmArgs g;
    g.po = N == 1 ? peer_out() : PeerOut{};
    g.dbg = kDiag ? env_override("B200CONV_GM_DBG", 0) : 0;
    g.nkb = p.nkb;
    g.kbps = p.kbps;
    g.M = M;
    g.Ho = Ho;
    g.Wo = Wo;
    g.Wx = Wp;
    g.N = N;
    g.stages = p.stages;
    g.stage_bytes = p.stage_bytes;
    g.O = O;
    g.Wk = Wk;
    const CUtensorMap &ta = p.modeF ? tf : tx;
    const CUtensorMap &tb = p.modeF ? tx : tf;
    if (bf16)
        return p.modeF ? launch_gemm_bn<false, true>(p, ta, tb, g, s) : launch_gemm_bn<false, false>(p, ta, tb, g, s);
    return p.modeF ? launch_gemm_bn<true, true>(p, ta, tb, g, s) : launch_gemm_bn<true, false>(p, ta, tb, g, s);
}

}  // namespace b200
