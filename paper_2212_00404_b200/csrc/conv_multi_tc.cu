// conv_multi_tc.cu — kernel KM-TC: multi-channel direct convolution (PAPER.md
// §2.1 Eq. 1) as an implicit GEMM on the 5th-generation tensor cores
// (tcgen05.mma, accumulators in TMEM), TF32 or BF16 inputs, FP32 accumulate.
//
//   D[p][m] = sum_k A[p][k] * B[m][k],   k = (ch, r, c) = ch*K*K + r*K + c
//   A[p][k] = I[ch][p + r*Wx + c]        (im2col of I, built on chip)
//   B[m][k] = F[m][ch][r][c] = F[m*Ktot + k]  (F as stored, row-major [M][Ktot])
//   O[m][y][x] = D[y*Wx + x][m]          for x < Wo ("wide" pixel p = y*Wx + x)
//
// The reduction order k = (ch, r, c) is exactly the filter layout of the paper
// ("along the dimension ch first"), so B is F itself: a TMA tensor
// map loads [BN filters] x [128 B of k] boxes with the 128-B swizzle straight
// into the canonical K-major UMMA layout (the paper's stride-fixed segment S,
// P:603-612, becomes one 128-B TMA row).
//
// A is never materialised in global memory.  For every k-block the TMA
// producer also loads the input "patch" of the channels that k-block touches:
// with wide-pixel indexing the pixels a 128-pixel tile needs from one channel
// form ONE contiguous range I[ch][p0 .. p0 + 128 + (K-1)*Wx + K-1), fetched by
// 1-D TMA boxes (any alignment, zero fill past the end).  Eight gather warps
// then expand the patch into the im2col tile in TMEM with conflict-free
// shared loads (one pixel row per thread pair) and tcgen05.st, and arrive on
// the stage's mbarrier; one thread issues tcgen05.mma.
// Pixels sit on the 128-lane M side, so the epilogue (tcgen05.ld -> registers
// -> st.global) writes 32 consecutive pixels per warp instruction.  Small
// layers split the k loop over a thread-block cluster and reduce the partial
// tiles through DSMEM in fixed rank order (deterministic, O written once).
//
// The im2col tile never touches shared memory: the gather warps store it
// straight into tensor memory (tcgen05.st, 16 columns per thread) and the MMA
// reads A from TMEM (tcgen05.mma [d], [a_tmem], b_desc) — the main loop was
// shared-memory-bandwidth bound (patch read + tile write + MMA tile read per
// element); A in TMEM removes two of those three passes (measured: 28x28x256
// batched N = 64 TF32 357 -> 447 TFLOP/s, single-image layers 3-10 % faster).
//
// Warp roles (352 threads):
//   warps 0..7  im2col build of A into TMEM (2 threads per pixel row), then epilogue
//   warp 8      TMA producer: F tile (B) + input patch
//   warp 9      TMEM allocator + MMA issuer                  [elected lane]
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>
#include "kernels.h"
#include "ptx.cuh"

namespace b200 {

constexpr int kTcProducers = 2;       // producer warps (alternate stages)
constexpr int kTcThreads = 32 * (8 + kTcProducers + 1);
// Warp roles.  The SM sub-partition scheduler favours higher warp ids, so the
// single-thread producer and MMA roles take the two highest ids: spinning
// im2col warps on the same sub-partition can never starve them.
constexpr uint32_t kProdWarp = 8;     // TMA producers: warps 8 .. 8+kTcProducers-1
constexpr uint32_t kMmaWarp = 8 + kTcProducers;   // TMEM allocator + tcgen05.mma issuer
constexpr int kTcBM = 128;            // pixels per tile (UMMA M)
constexpr int kTcMaxSplit = 16;      // non-portable cluster size on B200
constexpr int kTcSmemMax = 225 * 1024;
#ifndef B200CONV_TC_MAX_STAGES
#define B200CONV_TC_MAX_STAGES 8
#endif
constexpr int kTcMaxStages = B200CONV_TC_MAX_STAGES;   // (A/B builds: -DB200CONV_TC_MAX_STAGES=12)

template <bool kTF32>
struct TcTraits {
    using T = typename std::conditional<kTF32, float, __nv_bfloat16>::type;
    static constexpr int kElem = kTF32 ? 4 : 2;
    static constexpr int kBK = 128 / kElem;           // k per stage (one 128-B swizzle row)
    static constexpr int kUmmaK = 32 / kElem;         // k per tcgen05.mma (32 B)
    static constexpr uint32_t kFmt = kTF32 ? 2u : 1u; // instr-desc a/b format
};

// Per-launch geometry shared by host and device.
struct TcGeom {
    int np;       // patch length per channel (elements)
    int pb;       // 1-D TMA box (elements)
    int nbox;     // boxes per channel
    int npp;      // patch stride per channel in smem (elements) = nbox * pb
    int pch;      // max channels touched by one k-block
    int patch_bytes;
    int tab_bytes;
    int stages;
    int stage_bytes;
    int smem;
};

__host__ __device__ inline TcGeom tc_geom(int Wx, int K, int BN, int elem, bool patch, int extra = 0) {
    TcGeom g;
    const int BK = 128 / elem;
    // a box must start 16-B aligned in global memory: the patch starts up to
    // 16/elem - 1 elements before the channel's first pixel
    g.np = kTcBM + (K - 1) * Wx + (K - 1) + 16 / elem - 1;
    const int align = 128 / elem;             // TMA smem destinations: 128-B aligned
    const int npa = (g.np + align - 1) / align * align;
    g.pb = npa < 256 ? npa : 256;
    g.nbox = (g.np + g.pb - 1) / g.pb;
    g.npp = g.nbox * g.pb;
    g.pch = (BK + K * K - 1) / (K * K) + 1;
    g.patch_bytes = patch ? ((g.pch * g.npp * elem + 1023) & ~1023) : 0;
    // the im2col A tile lives in TMEM (columns BN + 32*s), so a stage holds
    // only the B (filter) tile and the input patch
    g.stage_bytes = BN * 128 + g.patch_bytes;
    // k -> patch offset table for every phase (k0 mod K*K) of a k-block (K <= 7)
    g.tab_bytes = (patch && K <= 7) ? K * K * BK * 4 : 0;
    int st = (kTcSmemMax - 1024 - 512 - g.tab_bytes - extra) / g.stage_bytes;
    g.stages = st > kTcMaxStages ? kTcMaxStages : st;
    if (g.stages > (512 - BN) / 32) g.stages = (512 - BN) / 32;       // TMEM: BN + 32 * stages <= 512
    g.smem = 1024 + g.stages * g.stage_bytes + 512 + g.tab_bytes + extra;
    return g;
}

// Byte offset of 16-B chunk j of row g in a K-major SWIZZLE_128B tile.
__device__ __forceinline__ uint32_t sw128_off(int g, int j) {
    return (uint32_t)((g >> 3) * 1024 + (g & 7) * 128 + ((j ^ (g & 7)) << 4));
}

__device__ unsigned long long g_tc_stamps[1024];   // diagnostics (dbg & 128)

// dbg & 256: per-CTA timeline, globaltimer ns: [start, after griddepcontrol.wait,
// first k-block ready (MMA warp), last MMA retired (tmem_full), partial/epilogue
// done, end (after the cluster reduction) << 8 | smid], CTAs 0..1023 (linear id)
__device__ unsigned long long g_tc_cta[8 * 1024];

int tc_read_stamps(unsigned long long *host) {
    return cudaMemcpyFromSymbol(host, g_tc_stamps, sizeof(g_tc_stamps)) == cudaSuccess ? 0 : 1;
}
int tc_read_cta_stamps(unsigned long long *host) {
    return cudaMemcpyFromSymbol(host, g_tc_cta, sizeof(g_tc_cta)) == cudaSuccess ? 0 : 1;
}
__device__ __forceinline__ unsigned long long tc_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Rank-ordered sum of the S partial tiles' float4 at local_addr across the
// cluster (DSMEM); out of line, so the once-per-CTA reduction loop stays small
// (its code is fetched cold).
__device__ __noinline__ float4 tc_dsmem_sum(uint32_t local_addr, int S) {
    float4 v = ld_dsmem_f32x4(mapa_shared(local_addr, 0u));
#pragma unroll 1
    for (int t = 1; t < S; ++t) {
        const float4 u = ld_dsmem_f32x4(mapa_shared(local_addr, (uint32_t)t));
        v.x += u.x; v.y += u.y; v.z += u.z; v.w += u.w;
    }
    return v;
}

template <bool kTF32, int BN, bool kTmaB, bool kPatch>
__global__ void __launch_bounds__(kTcThreads, 1)
kmtc_kernel(const __grid_constant__ CUtensorMap tmapF, const __grid_constant__ CUtensorMap tmapI,
            const void *__restrict__ Iv, const void *__restrict__ Fv, int C, int Wx, int Wy,
            int K, int M, float *__restrict__ O, int kb_per_split, int patch2d, int dbg_in,
            float *__restrict__ Wk, int Nimg, int Wv) {
    const int dbg = kDiag ? dbg_in : 0;
    using Tr = TcTraits<kTF32>;
    using T = typename Tr::T;
    constexpr int BK = Tr::kBK;
    constexpr int A_BYTES = 0;                        // A (im2col) tile: in TMEM, not smem
    constexpr int B_BYTES = BN * 128;
    constexpr uint32_t IDESC = umma_idesc(Tr::kFmt, kTcBM, BN);

    const int KK = K * K;
    const int Ktot = C * KK;
    const int HW = Wx * Wy;
    const int64_t CHW = (int64_t)C * HW;
    // Wv: valid input width (padded calls: the row stride Wx is rounded up to
    // 16 B; columns >= Wv are zeros whose outputs are wide-pixel garbage)
    const int Ho = Wy - K + 1, Wo = (Wv > 0 ? Wv : Wx) - K + 1;
    // batch: blockIdx.y = image * (pixel tiles per image) + pixel tile
    const int npt_img = gridDim.y / Nimg;
    const int img = blockIdx.y / npt_img;
    const int chb = img * C;                              // first channel of this image in I viewed as [N*C][HW]
    const T *__restrict__ I = static_cast<const T *>(Iv) + (int64_t)img * CHW;
    const T *__restrict__ F = static_cast<const T *>(Fv);
    O += (int64_t)img * M * Ho * Wo;
    const int nkb = (Ktot + BK - 1) / BK;
    const TcGeom geo = tc_geom(Wx, K, BN, Tr::kElem, kPatch);
    const int NS = geo.stages;
    const int STAGE = geo.stage_bytes;

    const int S = gridDim.x;
    const int split = blockIdx.x;
    const int tile_lin = blockIdx.y + gridDim.y * blockIdx.z;
    const int p0 = (blockIdx.y - img * npt_img) * kTcBM;
    const int n0 = blockIdx.z * BN;
    const int kb0 = split * kb_per_split;
    const int kb1 = min(nkb, kb0 + kb_per_split);
    const int niter = kb1 > kb0 ? kb1 - kb0 : 0;

    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t *smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + NS * STAGE);   // A+B ready (MMA)
    uint64_t *pfull = full + kTcMaxStages;                               // patch landed
    uint64_t *empty = pfull + kTcMaxStages;                              // MMA done with stage
    uint64_t *tmem_full = empty + kTcMaxStages;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_full + 1);
    uint64_t *red_bar = tmem_full + 2;                                   // split-K slices landed
    float *P = reinterpret_cast<float *>(smem);      // [BN][128] partial tile (split > 1), aliases the stages
    int *ktab = reinterpret_cast<int *>(smem + NS * STAGE + 512);        // [K*K][BK]
    const bool use_tab = kPatch && patch2d && geo.tab_bytes > 0;
    if (use_tab) {
        for (int idx = threadIdx.x; idx < KK * BK; idx += kTcThreads) {
            const int u = idx / BK + idx % BK;             // phase + j
            const int rem = u % KK;
            ktab[idx] = (u / KK) * geo.npp + (rem / K) * Wx + (rem % K);
        }
    }

    const uint32_t warp = warp_id();
    const uint32_t lane = lane_id();
    const unsigned cta_lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    const bool tl = (dbg & 256) && cta_lin < 1024;
    if (tl && threadIdx.x == 0) g_tc_cta[8 * cta_lin] = tc_gtimer();
    // dbg & 128: CTA (0,0,0) records globaltimer stamps per iteration into O
    //   O[i] producer issue, O[256+i] gather(warp 2) arrive, O[512+i] MMA commit
    const bool stamp = (dbg & 128) && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0;
    auto gtime = []() { uint64_t t; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)); return t; };
    auto wait = [&](uint64_t *bar, uint32_t par) {
        if (dbg & 64) mbar_wait_poll(bar, par); else mbar_wait(bar, par);
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 8 + (kTmaB ? 1 : 0));   // 8 gather warps (+1 TMA expect_tx)
            mbar_init(&pfull[s], 1);
            mbar_init(&empty[s], 1);                    // tcgen05.commit
        }
        mbar_init(tmem_full, 1);
        mbar_init(red_bar, 1);
        fence_mbar_init();
        if (kTmaB) tma_prefetch_desc(&tmapF);
        if (kPatch) tma_prefetch_desc(&tmapI);
    }
    if (warp == kMmaWarp) tmem_alloc<512>(tmem_slot);    // accumulator [0, BN) + A stages [BN, BN + 32*NS)
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();                     // prologue above overlaps the previous kernel's tail
    pdl_trigger();
    if (tl && threadIdx.x == 0) g_tc_cta[8 * cta_lin + 1] = tc_gtimer();

    if (warp >= kProdWarp && warp < kMmaWarp) {
        // ------------------------------------------------ TMA producer
        // The whole warp runs the loop; lane 0 owns the barriers and the F
        // tile, lanes 0..nch-1 issue one channel's patch boxes each, so the
        // per-stage issue latency is not one thread's serial chain.
        const int ch_mask = 16 / Tr::kElem - 1;
        const int pw = (int)(warp - kProdWarp);          // this producer takes stages pw, pw+P, ...
        int k0 = (kb0 + pw) * BK;
        int ch_lo = k0 / KK;                             // incremental from here on
        for (int i = pw; i < niter; i += kTcProducers, k0 += kTcProducers * BK) {
            const int s = i % NS, ph = (i / NS) & 1;
            if (stamp && lane == 0 && i < 128) g_tc_stamps[768 + i] = gtime();
            if (lane == 0) wait(&empty[s], ph ^ 1);
            __syncwarp();
            if (stamp && lane == 0 && i < 128) g_tc_stamps[896 + i] = gtime();
            uint8_t *st = smem + s * STAGE;
            if (kPatch) {
                while ((ch_lo + 1) * KK <= k0) ++ch_lo;
                const int k_end = min(k0 + BK, Ktot) - 1;
                int ch_hi = ch_lo;
                while ((ch_hi + 1) * KK <= k_end) ++ch_hi;
                const int nch = ch_hi - ch_lo + 1;
                if (patch2d) {
                    // one 2-D box [pch channels][pb pixels] (I viewed as [C][HW])
                    if (lane == 0) {
                        mbar_arrive_expect_tx(&pfull[s], (uint32_t)(geo.pch * geo.pb * Tr::kElem));
                        tma_load_2d(st + A_BYTES + B_BYTES, &tmapI, &pfull[s], p0, chb + ch_lo);
                    }
                } else {
                    if (lane == 0) {
                        if (dbg & 8) mbar_arrive(&pfull[s]);
                        else mbar_arrive_expect_tx(&pfull[s], (uint32_t)(nch * geo.npp * Tr::kElem));
                    }
                    __syncwarp();
                    if (!(dbg & 8) && (int)lane < nch) {
                        T *patch = reinterpret_cast<T *>(st + A_BYTES + B_BYTES) + lane * geo.npp;
                        const int start = ((chb + ch_lo + (int)lane) * HW + p0) & ~ch_mask;
                        for (int b = 0; b < geo.nbox; ++b)
                            tma_load_1d(patch + b * geo.pb, &tmapI, &pfull[s], start + b * geo.pb);
                    }
                }
            }
            if (lane == 0) {
                if (stamp && i < 256) g_tc_stamps[i] = gtime();
                if (kTmaB) {
                    if (dbg & 2) {
                        mbar_arrive(&full[s]);
                    } else {
                        mbar_arrive_expect_tx(&full[s], B_BYTES);
                        tma_load_2d(st + A_BYTES, &tmapF, &full[s], k0, n0);
                    }
                }
            }
        }
    } else if (warp == kMmaWarp) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            for (int i = 0; i < niter; ++i) {
                const int s = i % NS;
                wait(&full[s], (i / NS) & 1);
                tc_fence_after();
                if (tl && i == 0) g_tc_cta[8 * cta_lin + 2] = tc_gtimer();
                const uint32_t b_addr = smem_u32(smem + s * STAGE);
                const uint32_t a_tmem = tmem + (uint32_t)(BN + 32 * s);
#pragma unroll
                for (int kk = 0; kk < BK / Tr::kUmmaK; ++kk) {
                    if (dbg & 4) break;
                    umma_ts<kTF32>(tmem, a_tmem + 8 * kk, umma_desc_k_sw128(b_addr + kk * 32), IDESC,
                                   (i > 0 || kk > 0) ? 1u : 0u);
                }
                if (dbg & 16) mbar_arrive(&empty[s]); else umma_commit(&empty[s]);
                if (stamp && i < 256) g_tc_stamps[512 + i] = gtime();
            }
            umma_commit(tmem_full);       // fires when all MMAs above are complete
        }
        __syncwarp();
    } else {
        // ------------------------------------------------ im2col build of A
        const int gt = threadIdx.x;                      // 0..255 (warps 0..7)
        const int g = gt & 127;                          // pixel row in the tile
        const int h = gt >> 7;                           // which half of the 128-B row
        const int p = p0 + g;
        const bool prow = p < Ho * Wx;
        // stage / parity / first channel of the k-block advanced incrementally
        // (no integer division per k-block on the gather warps)
        int ch_lo = (kb0 * BK) / KK;
        for (int i = 0, s = 0, ph = 0, k0 = kb0 * BK; i < niter;
             ++i, k0 += BK, (++s == NS) ? (s = 0, ph ^= 1) : 0) {
            uint8_t *a_s = smem + s * STAGE;
            while ((ch_lo + 1) * KK <= k0) ++ch_lo;
            // stage free (non-patch path) / patch landed (patch path; the producer
            // only loads it after the MMA released the stage)
            if (kPatch) wait(&pfull[s], (uint32_t)ph);
            else wait(&empty[s], (uint32_t)(ph ^ 1));
            if (dbg & 1) {
                if (!(dbg & 32)) fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[s]);
                if (stamp && warp == 0 && lane == 0 && i < 256) g_tc_stamps[256 + i] = gtime();
                continue;
            }
            uint32_t v[16];
            if (use_tab && k0 + BK <= Ktot) {
                // offsets of this thread's BK/2 k values from the phase table (16-B broadcast loads)
                const int4 *trow = reinterpret_cast<const int4 *>(ktab + (k0 - ch_lo * KK) * BK + (BK / 2) * h);
                if constexpr (kTF32) {
                    const float *src = reinterpret_cast<const float *>(a_s + A_BYTES + B_BYTES) + g;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int4 o = trow[q];
                        v[4 * q] = __float_as_uint(src[o.x]);
                        v[4 * q + 1] = __float_as_uint(src[o.y]);
                        v[4 * q + 2] = __float_as_uint(src[o.z]);
                        v[4 * q + 3] = __float_as_uint(src[o.w]);
                    }
                } else {
                    const unsigned short *src =
                        reinterpret_cast<const unsigned short *>(a_s + A_BYTES + B_BYTES) + g;
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int4 o = trow[q];
                        v[2 * q] = (uint32_t)src[o.x] | ((uint32_t)src[o.y] << 16);
                        v[2 * q + 1] = (uint32_t)src[o.z] | ((uint32_t)src[o.w] << 16);
                    }
                }
            } else {
                // each lane decodes the source offset of BK/32 k values
                int koff[BK / 32];
#pragma unroll
                for (int t = 0; t < BK / 32; ++t) {
                    const int k = k0 + t * 32 + (int)lane;
                    const int ch = k / KK, rem = k - ch * KK, r = rem / K, c = rem - r * K;
                    if (kPatch)   // + the channel's misalignment inside its 16-B aligned patch
                        koff[t] = k < Ktot ? (ch - ch_lo) * geo.npp + (((chb + ch) * HW) & (16 / Tr::kElem - 1)) +
                                                 r * Wx + c
                                           : -1;
                    else koff[t] = k < Ktot ? ch * HW + r * Wx + c : -1;
                }
                // this thread's half row: 16-B chunks [4h, 4h+4) = BK/2 consecutive k
                if constexpr (kTF32) {
                    const float *src = kPatch ? reinterpret_cast<const float *>(a_s + A_BYTES + B_BYTES)
                                              : reinterpret_cast<const float *>(I);
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int off = __shfl_sync(0xffffffffu, koff[0], 16 * h + j);
                        if (kPatch) {
                            v[j] = off >= 0 ? __float_as_uint(src[off + g]) : 0u;
                        } else {
                            const int64_t a = (int64_t)p + off;
                            v[j] = (prow && off >= 0 && a < CHW) ? __float_as_uint(__ldg(src + a)) : 0u;
                        }
                    }
                } else {
                    const unsigned short *src =
                        kPatch ? reinterpret_cast<const unsigned short *>(a_s + A_BYTES + B_BYTES)
                               : reinterpret_cast<const unsigned short *>(I);
                    const int kh = h ? koff[BK / 32 - 1] : koff[0];   // this half's k offsets
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        uint32_t lohi[2];
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int off = __shfl_sync(0xffffffffu, kh, 2 * j + e);
                            if (kPatch) {
                                lohi[e] = off >= 0 ? (uint32_t)src[off + g] : 0u;
                            } else {
                                const int64_t a = (int64_t)p + off;
                                lohi[e] = (prow && off >= 0 && a < CHW) ? (uint32_t)__ldg(src + a) : 0u;
                            }
                        }
                        v[j] = lohi[0] | (lohi[1] << 16);
                    }
                }
            }
            // A row g, columns [16h, 16h + 16) of stage s -> TMEM (lane quarter = warp & 3)
            tmem_st_32x32b_x16(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(BN + 32 * s + 16 * h), v);
            tmem_st_wait();
            if constexpr (!kTmaB) {
                // B rows (filters) gathered too when F rows are not 16-B aligned
                uint8_t *b_s = a_s + A_BYTES;
                for (int nr = g; nr < BN; nr += 128) {
                    const int m = n0 + nr;
                    uint32_t w[16];
                    if constexpr (kTF32) {
                        const float *Fm = reinterpret_cast<const float *>(F) + (int64_t)m * Ktot;
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const int k = k0 + 16 * h + j;
                            w[j] = (m < M && k < Ktot) ? __float_as_uint(__ldg(Fm + k)) : 0u;
                        }
                    } else {
                        const unsigned short *Fm =
                            reinterpret_cast<const unsigned short *>(F) + (int64_t)m * Ktot;
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const int k = k0 + 32 * h + 2 * j;
                            const uint32_t lo = (m < M && k < Ktot) ? (uint32_t)__ldg(Fm + k) : 0u;
                            const uint32_t hi = (m < M && k + 1 < Ktot) ? (uint32_t)__ldg(Fm + k + 1) : 0u;
                            w[j] = lo | (hi << 16);
                        }
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        *reinterpret_cast<uint4 *>(b_s + sw128_off(nr, 4 * h + q)) =
                            make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
                }
            }
            if constexpr (!kTmaB) fence_proxy_async_smem();   // gathered B -> visible to tcgen05
            tc_fence_before();               // TMEM stores ordered before the arrive
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[s]);
            if (stamp && warp == 0 && lane == 0 && i < 256) g_tc_stamps[256 + i] = gtime();
        }

        // ------------------------------------------------ epilogue
        const int q = (int)(warp & 3);                   // TMEM lane quarter of this warp
        const int half = (int)warp >> 2;                 // which half of the BN columns
        const int row = q * 32 + (int)lane;              // pixel row == TMEM lane
        const int pe = p0 + row;
        const int y = pe / Wx, x = pe - y * Wx;
        const bool valid = (pe < Ho * Wx) && (x < Wo);
        const int64_t obase = (int64_t)y * Wo + x;
        const int64_t plane = (int64_t)Ho * Wo;
        if (niter > 0) {
            mbar_wait(tmem_full, 0);
            tc_fence_after();
        }
        if (tl && threadIdx.x == 0) g_tc_cta[8 * cta_lin + 3] = tc_gtimer();
        // the split-K partial tile P reuses the ring's smem: every gather warp's
        // patch reads are ordered before it through the stage barriers and the
        // MMA commit; this named barrier (the 8 gather / epilogue warps only)
        // states that ordering explicitly (compute-sanitizer racecheck does not
        // follow the tcgen05.commit chain)
        if (S > 1) asm volatile("bar.sync 1, 256;" ::: "memory");
        constexpr int NCB = BN / 32;                     // 32-column blocks
        for (int cb = half; cb < NCB; cb += 2) {
            uint32_t r[32];
            if (niter > 0) {
                tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(cb * 32), r);
                tmem_ld_wait();
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) r[j] = 0u;
            }
            if (S == 1) {
                if (valid) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int m = n0 + cb * 32 + j;
                        if (m < M) O[(int64_t)m * plane + obase] = __uint_as_float(r[j]);
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) P[(cb * 32 + j) * kTcBM + row] = __uint_as_float(r[j]);
            }
        }
        if (S > 1 && Wk) fence_proxy_async_smem();       // P -> visible to the bulk store
        tc_fence_before();
    }

    __syncthreads();
    if (tl && threadIdx.x == 0) g_tc_cta[8 * cta_lin + 4] = tc_gtimer();
    if (S > 1) {
        // ---------------------------------------------- split-K reduce
        // L2 path: the partial tile leaves in ONE bulk store to the workspace
        // [split][tile][BN][128]; after the cluster barrier each rank bulk-loads
        // its filter rows of all S partials into (the now free) smem and sums
        // them in rank order.  DSMEM path (no workspace): sums the ranks' smem
        // tiles directly.
        if (Wk && threadIdx.x == 0) {
            float *wmine = Wk + ((int64_t)split * gridDim.y * gridDim.z + tile_lin) * BN * kTcBM;
            bulk_store(wmine, P, (uint32_t)(BN * kTcBM * 4));
            bulk_commit();
            bulk_wait<0>();
            fence_proxy_async_global();
        }
        cluster_sync_all();
        if (tl && threadIdx.x == 0) g_tc_cta[8 * cta_lin + 6] = tc_gtimer();
        const int nlo = split * BN / S;                  // filters [nlo, nhi) owned by this rank
        const int rows = (split + 1) * BN / S - nlo;
        const uint32_t Pbase = smem_u32(smem);
        const int64_t plane = (int64_t)Ho * Wo;
        // 4 pixels per thread: 16-B loads of every rank's partial (L2 workspace
        // or DSMEM), all in flight at once, summed in rank order
        float *slices = P;                               // [S][rows][128]
        if (Wk) {
            if (threadIdx.x == 0) {
                const int64_t wslice = (int64_t)gridDim.y * gridDim.z * BN * kTcBM;
                const float *wt = Wk + ((int64_t)tile_lin * BN + nlo) * kTcBM;
                const uint32_t bytes = (uint32_t)(rows * kTcBM * 4);
                mbar_arrive_expect_tx(red_bar, bytes * S);
                for (int t = 0; t < S; ++t) bulk_load(slices + t * rows * kTcBM, wt + t * wslice, bytes, red_bar);
            }
            mbar_wait(red_bar, 0);
            if (tl && threadIdx.x == 0) g_tc_cta[8 * cta_lin + 7] = tc_gtimer();
        }
        // thread -> 4 fixed pixels (row0 = 4 * lane) and filter rows lane-warp
        // + kTcWarps * j; four rows per batch, every partial load of a batch
        // in flight before the sums and stores (this loop runs once per CTA:
        // one item at a time it was latency-bound, ~6 us on configs[4] TF32)
        constexpr int kTcWarps = kTcThreads / 32;
        const int row0 = 4 * (int)lane;
        int64_t opix[4];
        bool pvalid[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int pe = p0 + row0 + e;
            const int y = pe / Wx, x = pe - y * Wx;
            pvalid[e] = pe < Ho * Wx && x < Wo;
            opix[e] = (int64_t)y * Wo + x;
        }
        for (int nb = (int)warp; nb < rows; nb += 4 * kTcWarps) {
            float4 v[4];
            if (!Wk && S <= 4 && !(dbg & 512)) {
                // DSMEM, up to 4 ranks: all 16 remote loads of the batch first
                float4 w[4][4];
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int t = 0; t < 4; ++t)
                        if (t < S && nb + u * kTcWarps < rows)
                            w[u][t] = ld_dsmem_f32x4(mapa_shared(
                                Pbase + (uint32_t)(((nlo + nb + u * kTcWarps) * kTcBM + row0) * 4), (uint32_t)t));
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    v[u] = w[u][0];                      // rank order: 0, 1, ..., S-1
#pragma unroll
                    for (int t = 1; t < 4; ++t)
                        if (t < S && nb + u * kTcWarps < rows) {
                            v[u].x += w[u][t].x; v[u].y += w[u][t].y; v[u].z += w[u][t].z; v[u].w += w[u][t].w;
                        }
                }
            } else
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int nl = nlo + nb + u * kTcWarps;
                v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (nb + u * kTcWarps >= rows || (dbg & 512)) continue;
                if (Wk) {
                    const float *sl = slices + (nl - nlo) * kTcBM + row0;
                    v[u] = *reinterpret_cast<const float4 *>(sl);
#pragma unroll 4
                    for (int t = 1; t < S; ++t) {
                        const float4 w = *reinterpret_cast<const float4 *>(sl + t * rows * kTcBM);
                        v[u].x += w.x; v[u].y += w.y; v[u].z += w.z; v[u].w += w.w;
                    }
                } else {
                    v[u] = tc_dsmem_sum(Pbase + (uint32_t)((nl * kTcBM + row0) * 4), S);
                }
            }
            if (dbg & 1024) continue;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int m = n0 + nlo + nb + u * kTcWarps;
                if (nb + u * kTcWarps >= rows || m >= M) continue;
                float *o = O + (int64_t)m * plane;
                if (pvalid[0]) o[opix[0]] = v[u].x;
                if (pvalid[1]) o[opix[1]] = v[u].y;
                if (pvalid[2]) o[opix[2]] = v[u].z;
                if (pvalid[3]) o[opix[3]] = v[u].w;
            }
        }
        if (!Wk) cluster_sync_all();          // keep this CTA's partial alive for the others
    }
    if (tl && threadIdx.x == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_tc_cta[8 * cta_lin + 5] = (tc_gtimer() << 8) | smid;
    }
    if (warp == kMmaWarp) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

// ---------------------------------------------------------------- persistent variant
// Batched calls with many tiles (S = 1, TMA filters, one 2-D patch box per
// k-block, C*K*K a multiple of BK): one CTA per SM walks the tiles
// t = blockIdx.x, + gridDim.x, ...  The rings (stage / parity counters) run
// on across tiles, so the producers and gather warps start tile t+1 while
// four dedicated epilogue warps drain tile t's accumulator; the MMA issuer
// starts tile t+1's MMAs once the epilogue has released TMEM (tmem_empty).
// This removes the per-tile prologue (TMEM alloc, barrier init, descriptor
// prefetch) and the pipeline fill that the one-tile-per-CTA kernel pays at
// every tile.
#ifndef B200CONV_TP_EPI_GROUPS
#define B200CONV_TP_EPI_GROUPS 2
#endif
constexpr int kTpEpiGroups = B200CONV_TP_EPI_GROUPS;         // epilogue warp groups (4 warps each)
constexpr int kTpEpiWarp = 8 + kTcProducers + 1;            // warps 11..: epilogue
constexpr int kTpThreads = 32 * (kTpEpiWarp + 4 * kTpEpiGroups);
// epilogue staging: per group, 16 filters x 128 pixels of the accumulator,
// transposed so each filter's outputs leave as one contiguous run of O
constexpr int kTpEpiBytes = kTpEpiGroups * 16 * kTcBM * 4;

template <bool kTF32, int BN>
__global__ void __launch_bounds__(kTpThreads, 1)
kmtc_persist_kernel(const __grid_constant__ CUtensorMap tmapF, const __grid_constant__ CUtensorMap tmapI,
                    int C, int Wx, int Wy, int K, int M, float *__restrict__ O, int Nimg, int tiles_y, int Wv) {
    using Tr = TcTraits<kTF32>;
    constexpr int BK = Tr::kBK;
    constexpr int B_BYTES = BN * 128;
    constexpr uint32_t IDESC = umma_idesc(Tr::kFmt, kTcBM, BN);
    const int KK = K * K;
    const int Ktot = C * KK;
    const int Ho = Wy - K + 1, Wo = (Wv > 0 ? Wv : Wx) - K + 1;   // Wv: see kmtc_kernel
    const int nkb = Ktot / BK;                           // plan: Ktot % BK == 0
    const TcGeom geo = tc_geom(Wx, K, BN, Tr::kElem, true, kTpEpiBytes);
    const int NS = geo.stages;
    const int STAGE = geo.stage_bytes;
    const int nft = (M + BN - 1) / BN;
    const int ntiles = tiles_y * nft;                    // tile t: y = t / nft (image x pixel tile), z = t % nft
    const int npt_img = tiles_y / Nimg;
    const int64_t plane = (int64_t)Ho * Wo;

    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t *smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + NS * STAGE);
    uint64_t *pfull = full + kTcMaxStages;
    uint64_t *empty = pfull + kTcMaxStages;
    uint64_t *tmem_full = empty + kTcMaxStages;          // MMA -> epilogue (one phase per tile)
    uint64_t *tmem_empty = tmem_full + 1;                // epilogue -> MMA
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_empty + 1);
    int *ktab = reinterpret_cast<int *>(smem + NS * STAGE + 512);
    for (int idx = threadIdx.x; idx < KK * BK; idx += kTpThreads) {
        const int u = idx / BK + idx % BK;
        const int rem = u % KK;
        ktab[idx] = (u / KK) * geo.npp + (rem / K) * Wx + (rem % K);
    }
    const uint32_t warp = warp_id();
    const uint32_t lane = lane_id();
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 8 + 1);                  // 8 gather warps + the filter TMA
            mbar_init(&pfull[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
        mbar_init(tmem_empty, 4 * kTpEpiGroups);         // every epilogue warp
        fence_mbar_init();
        tma_prefetch_desc(&tmapF);
        tma_prefetch_desc(&tmapI);
    }
    if (warp == kMmaWarp) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();
    pdl_trigger();

    // diagnostic build: clock64 stamps of CTA 0's first 256 ring iterations
    // (P: producer past empty, G0: gather warp 0 past pfull, G1: its arrive,
    // M: MMA issuer past full) -> g_tc_stamps, tools/tc_stamp_persist.py
    const bool pst = kDiag && blockIdx.x == 0;
    auto pstamp = [&](int slot, int i) {
        if (pst && i < 256) g_tc_stamps[slot * 256 + i] = (unsigned long long)clock64();
    };
    auto tile_of = [&](int t, int *p0, int *n0, int *img) {
        const int y = t / nft;
        *n0 = (t - y * nft) * BN;
        *img = y / npt_img;
        *p0 = (y - *img * npt_img) * kTcBM;
    };

    if (warp >= kProdWarp && warp < kMmaWarp) {
        // ------------------------------------------------ TMA producers (alternate k-blocks)
        const int pw = (int)(warp - kProdWarp);
        if (lane == 0) {
            int i = 0;                                   // ring iteration across tiles
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                int p0, n0, img;
                tile_of(t, &p0, &n0, &img);
                int ch_lo = 0;
                for (int kb = 0; kb < nkb; ++kb, ++i) {
                    const int k0 = kb * BK;
                    while ((ch_lo + 1) * KK <= k0) ++ch_lo;
                    if ((i % kTcProducers) != pw) continue;
                    const int s = i % NS, ph = (i / NS) & 1;
                    mbar_wait(&empty[s], ph ^ 1);
                    pstamp(0, i);
                    uint8_t *st = smem + s * STAGE;
                    mbar_arrive_expect_tx(&pfull[s], (uint32_t)(geo.pch * geo.pb * Tr::kElem));
                    tma_load_2d(st + B_BYTES, &tmapI, &pfull[s], p0, img * C + ch_lo);
                    mbar_arrive_expect_tx(&full[s], B_BYTES);
                    tma_load_2d(st, &tmapF, &full[s], k0, n0);
                }
            }
        }
        __syncwarp();
    } else if (warp == kMmaWarp) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            int i = 0, nt = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++nt) {
                if (nt > 0) {                            // the epilogue has drained the previous tile
                    mbar_wait(tmem_empty, (uint32_t)((nt - 1) & 1));
                    tc_fence_after();
                }
                for (int kb = 0; kb < nkb; ++kb, ++i) {
                    const int s = i % NS;
                    mbar_wait(&full[s], (uint32_t)((i / NS) & 1));
                    pstamp(3, i);
                    tc_fence_after();
                    const uint32_t b_addr = smem_u32(smem + s * STAGE);
                    const uint32_t a_tmem = tmem + (uint32_t)(BN + 32 * s);
#pragma unroll
                    for (int kk = 0; kk < BK / Tr::kUmmaK; ++kk)
                        umma_ts<kTF32>(tmem, a_tmem + 8 * kk, umma_desc_k_sw128(b_addr + kk * 32), IDESC,
                                       (kb > 0 || kk > 0) ? 1u : 0u);
                    umma_commit(&empty[s]);
                }
                umma_commit(tmem_full);                  // this tile's accumulator is complete
            }
        }
        __syncwarp();
    } else if (warp < 8) {
        // ------------------------------------------------ im2col build of A (table path)
        const int gt = threadIdx.x;
        const int g = gt & 127;
        const int h = gt >> 7;
        int i = 0, s = 0, ph = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            int ch_lo = 0;
            for (int kb = 0, k0 = 0; kb < nkb; ++kb, k0 += BK, ++i, (++s == NS) ? (s = 0, ph ^= 1) : 0) {
                while ((ch_lo + 1) * KK <= k0) ++ch_lo;
                mbar_wait(&pfull[s], (uint32_t)ph);
                if (gt == 0) pstamp(1, i);
                const uint8_t *patch = smem + s * STAGE + B_BYTES;
                uint32_t v[16];
                const int4 *trow = reinterpret_cast<const int4 *>(ktab + (k0 - ch_lo * KK) * BK + (BK / 2) * h);
                if constexpr (kTF32) {
                    const float *src = reinterpret_cast<const float *>(patch) + g;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int4 o = trow[q];
                        v[4 * q] = __float_as_uint(src[o.x]);
                        v[4 * q + 1] = __float_as_uint(src[o.y]);
                        v[4 * q + 2] = __float_as_uint(src[o.z]);
                        v[4 * q + 3] = __float_as_uint(src[o.w]);
                    }
                } else {
                    const unsigned short *src = reinterpret_cast<const unsigned short *>(patch) + g;
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int4 o = trow[q];
                        v[2 * q] = (uint32_t)src[o.x] | ((uint32_t)src[o.y] << 16);
                        v[2 * q + 1] = (uint32_t)src[o.z] | ((uint32_t)src[o.w] << 16);
                    }
                }
                tmem_st_32x32b_x16(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(BN + 32 * s + 16 * h), v);
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[s]);
                if (gt == 0) pstamp(2, i);
            }
        }
    } else {
        // ------------------------------------------------ epilogue (warps 11..14)
        // The tile's valid pixels form ONE contiguous compact range
        // [q0, q0 + nv) of every O plane (wide pixels run row after row).
        // Per 32-filter chunk: TMEM -> registers -> smem [filter][pixel], then
        // each warp writes 8 filters' runs with lanes along the run.  (Direct
        // stores from the TMEM layout wrote 32-pixel pieces of 32 planes that
        // start mid-line: the drain took ~15 K clk per tile while the MMA
        // waited on tmem_empty — profiles/tc_persist_stamps_r02.txt.)
        // kTpEpiGroups groups of four warps (one per TMEM lane quarter) take
        // interleaved 16-column chunks, each through its own staging buffer
        // (direct stores -> 1 -> 2 -> 4 groups: the MMA issuer waited 15 K ->
        // 9.3 K -> 8.2 K -> 7.2 K clk at each tile boundary; 2 groups measured
        // fastest overall, profiles/tc_persist_stamps_r02.txt).
        const int q = (int)(warp & 3);                   // TMEM lane quarter
        const int row = q * 32 + (int)lane;
        const int eg = (int)(warp - kTpEpiWarp) >> 2;    // epilogue group
        float *ep = reinterpret_cast<float *>(smem + NS * STAGE + 512 + geo.tab_bytes) + eg * 16 * kTcBM;
        int nt = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++nt) {
            int p0, n0, img;
            tile_of(t, &p0, &n0, &img);
            const int pend = min(p0 + kTcBM, Ho * Wx);
            int y0 = p0 / Wx, x0 = p0 - y0 * Wx;
            if (x0 >= Wo) { x0 = 0; ++y0; }              // first valid wide pixel: (y0, x0)
            const int q0 = y0 * Wo + x0;
            int nv = 0;
            if (y0 * Wx + x0 < pend) {
                const int yl = (pend - 1) / Wx, xl = pend - 1 - yl * Wx;
                nv = yl * Wo + min(xl, Wo - 1) - q0 + 1;
            }
            // wide offsets (from p0) of this lane's compact elements k = lane + 32 i
            int woff[kTcBM / 32];
#pragma unroll
            for (int i = 0; i < kTcBM / 32; ++i) {
                const int k = (int)lane + 32 * i;
                const int yy = (x0 + k) / Wo, xx = x0 + k - yy * Wo;
                woff[i] = k < nv ? (y0 + yy) * Wx + xx - p0 : -1;
            }
            float *Ot = O + (int64_t)img * M * plane + q0 + lane;
            mbar_wait(tmem_full, (uint32_t)(nt & 1));
            tc_fence_after();
#pragma unroll 1
            for (int cb = eg; cb < BN / 16; cb += kTpEpiGroups) {
                uint32_t r[16];
                tmem_ld_32x32b_x16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(cb * 16), r);
                tmem_ld_wait();
                if (cb + kTpEpiGroups >= BN / 16) {      // this warp's last TMEM read of the tile
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(tmem_empty);
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) ep[j * kTcBM + row] = __uint_as_float(r[j]);
                asm volatile("bar.sync %0, 128;" ::"r"(2 + eg) : "memory");   // this group's 4 warps
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const int j = q * 4 + jj;
                    const int m = n0 + cb * 16 + j;
                    if (m < M) {
                        float *Om = Ot + (int64_t)m * plane;
#pragma unroll
                        for (int i = 0; i < kTcBM / 32; ++i)
                            if (woff[i] >= 0) Om[32 * i] = ep[j * kTcBM + woff[i]];
                    }
                }
                asm volatile("bar.sync %0, 128;" ::"r"(2 + eg) : "memory");
            }
            if (eg >= BN / 16) {                         // no chunk for this group (BN < 16 * groups)
                __syncwarp();
                if (lane == 0) mbar_arrive(tmem_empty);
            }
        }
    }
    __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

// ---------------------------------------------------------------- host side
namespace {
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess && q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// filters per CTA tile (UMMA N).  N = 256 halves how often one im2col tile is
// rebuilt (once per filter tile) when there are many filters.
// (pixel_tiles: 128-pixel tiles of the whole call.  N = 256 once there are
// enough pixel tiles to fill the SMs without splitting k — one im2col build
// per 256 filters: batched 28x28x256, N = 32: 105 vs 125 us TF32, 64 vs 84 us
// BF16; single images keep N = 128 tiles and split k instead.)
int tc_bn(int M, int pixel_tiles) {
    if (const int v = env_override("B200CONV_TC_BN", 0); v == 32 || v == 64 || v == 128 || v == 256) return v;
    if (M <= 32) return 32;
    if (M <= 64) return 64;
    if (M >= 1024 || (M >= 256 && pixel_tiles >= 64)) return 256;
    return 128;
}
}  // namespace

static int plan_tc(int C, int Wx, int Wy, int K, int M, bool bf16, const void *F, conv_plan *p, int N,
                   bool allow_persist) {
    const int Ho = Wy - K + 1;
    const int elem = bf16 ? 2 : 4;
    const int BK = 128 / elem;
    const int64_t Ktot = (int64_t)C * K * K;
    const int nkb = (int)((Ktot + BK - 1) / BK);
    const int npt = N * ((Ho * Wx + kTcBM - 1) / kTcBM);   // pixel tiles of all N images
    const int BN = tc_bn(M, npt);
    const int nft = (M + BN - 1) / BN;
    const int tiles = npt * nft;
    // split the k loop over a cluster (measured: ~0.45 us per k-block, ~3.5 us
    // for the partial-tile exchange through L2), at least 2 k-blocks per split
    // (no split once the tiles alone occupy most SMs: measured slower at every
    // batched shape tried, e.g. 28x28x256 N=32 TF32 105 vs 94 us with S = 2)
    int S = tiles >= 128 ? 1
                         : choose_split(tiles, nkb, nkb / 2 < kTcMaxSplit ? (nkb / 2 > 0 ? nkb / 2 : 1) : kTcMaxSplit,
                                        1, 0.45f, 3.5f);
    if (const int v = env_override("B200CONV_TC_SPLIT", 0); v >= 1 && v <= kTcMaxSplit && v <= nkb) S = v;
    const TcGeom gp = tc_geom(Wx, K, BN, elem, true);
    const bool patch = gp.stages >= 2;
    const TcGeom g = patch ? gp : tc_geom(Wx, K, BN, elem, false);
    if (g.stages * g.stage_bytes < BN * kTcBM * 4) S = 1;   // the split partial tile aliases the stages
    p->kernel = 2;
    p->grid_x = S;
    p->grid_y = npt;
    p->grid_z = nft;
    p->block_x = kTcThreads;
    p->cluster_x = S;
    p->tile_m = BN;
    p->tile_n = kTcBM;
    p->smem_bytes = g.smem;
    const bool aligned = ((Ktot * elem) % 16 == 0) &&
                         (F == nullptr || (reinterpret_cast<uintptr_t>(F) % 16) == 0);
    p->tma_f = (aligned ? 1 : 0) | (patch ? 2 : 0);    // bit 0: F by TMA, bit 1: I patch by TMA
    p->launches = 1;
    // persistent variant (kmtc_persist_kernel): more tiles than SMs, no k split,
    // one 2-D patch box per k-block, whole k-blocks; B200CONV_TC_PERSIST=0 disables
    const bool persist_on = allow_persist && env_override("B200CONV_TC_PERSIST", 1) != 0;
    if (persist_on && S == 1 && aligned && patch && tiles > num_sms() && gp.nbox == 1 &&
        ((int64_t)Wx * Wy * elem) % 16 == 0 && Ktot % BK == 0 && gp.tab_bytes > 0 &&
        tc_geom(Wx, K, BN, elem, true, kTpEpiBytes).stages >= 2) {
        p->tma_f |= 32;                                    // bit 5: persistent CTAs
        p->smem_bytes = tc_geom(Wx, K, BN, elem, true, kTpEpiBytes).smem;
        p->grid_x = 1;
        p->grid_y = num_sms();
        p->grid_z = 1;
        p->block_x = kTpThreads;
    }
    return 0;
}

int plan_multi_tc(int C, int Wx, int Wy, int K, int M, bool bf16, const void *F, conv_plan *p, int N) {
    return plan_tc(C, Wx, Wy, K, M, bf16, F, p, N, true);
}
static int plan_tc_nopersist(int C, int Wx, int Wy, int K, int M, bool bf16, const void *F, conv_plan *p, int N) {
    return plan_tc(C, Wx, Wy, K, M, bf16, F, p, N, false);
}

template <bool kTF32, int BN, bool kTmaB, bool kPatch>
static cudaError_t launch_tc(const conv_plan &p, const CUtensorMap &tf, const CUtensorMap &ti,
                             const void *I, int C, int Wx, int Wy, const void *F, int K, int M,
                             float *O, int patch2d, cudaStream_t s, int N) {
    auto kern = kmtc_kernel<kTF32, BN, kTmaB, kPatch>;
    cudaError_t e = ensure_smem((const void *)kern, p.smem_bytes);
    if (e != cudaSuccess) return e;
    const int BK = kTF32 ? 32 : 64;
    const int nkb = (int)(((int64_t)C * K * K + BK - 1) / BK);
    const int kb_per_split = (nkb + p.cluster_x - 1) / p.cluster_x;
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
    const int dbg = kDiag ? env_override("B200CONV_TC_DBG", 0) : 0;
    // split-K partials go through the L2 workspace (DSMEM reduction when the
    // workspace cannot grow during stream capture, or with B200CONV_TC_DSMEM=1)
    float *Wk = nullptr;
    // split-K exchange: the L2 round trip (bulk store + bulk loads, 2 x the
    // tile per CTA at ~50 B/clk) or DSMEM ((S-1)/S of the tile at ~20 B/clk):
    // DSMEM wins for S <= 4 (configs[4] TF32: 25.9 vs 27.9 us), L2 above
    // (ResNet / AlexNet / target layers, S = 5..15: 0.5-1 us faster)
    const int dsmem_default = p.cluster_x <= 4 ? 1 : 0;
    if (p.cluster_x > 1 && env_override("B200CONV_TC_DSMEM", dsmem_default) != 1) {
        const size_t bytes = (size_t)p.cluster_x * p.grid_y * p.grid_z * BN * kTcBM * 4;
        Wk = static_cast<float *>(workspace_get(bytes, s));
    }
    return cudaLaunchKernelEx(&cfg, kern, tf, ti, I, F, C, Wx, Wy, K, M, O, kb_per_split, patch2d, dbg, Wk, N,
                              valid_width());
}

template <bool kTF32, int BN>
static cudaError_t launch_tc_persist(const conv_plan &p, const CUtensorMap &tf, const CUtensorMap &ti, int C, int Wx,
                                     int Wy, int K, int M, float *O, cudaStream_t s, int N) {
    auto kern = kmtc_persist_kernel<kTF32, BN>;
    cudaError_t e = ensure_smem((const void *)kern, p.smem_bytes);
    if (e != cudaSuccess) return e;
    const int tiles_y = N * (((Wy - K + 1) * Wx + kTcBM - 1) / kTcBM);   // images x pixel tiles per image
    const int tiles = tiles_y * ((M + BN - 1) / BN);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(tiles < num_sms() ? tiles : num_sms());
    cfg.blockDim = dim3(kTpThreads);
    cfg.dynamicSmemBytes = p.smem_bytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, tf, ti, C, Wx, Wy, K, M, O, N, tiles_y, valid_width());
}

template <bool kTF32, int BN>
static cudaError_t launch_tc_bn(const conv_plan &p, const void *I, int C, int Wx, int Wy,
                                const void *F, int K, int M, float *O, cudaStream_t s, int N) {
    const int elem = kTF32 ? 4 : 2;
    const CUtensorMapDataType dt =
        kTF32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    CUtensorMap tf, ti;
    memset(&tf, 0, sizeof(tf));
    memset(&ti, 0, sizeof(ti));
    const bool tma_b = (p.tma_f & 1) != 0;
    bool patch = (p.tma_f & 2) != 0 && (reinterpret_cast<uintptr_t>(I) % 16) == 0;
    auto encode = get_encode();
    if ((tma_b || patch) && !encode) return cudaErrorNotSupported;
    if (tma_b) {
        const cuuint64_t Ktot = (cuuint64_t)C * K * K;
        cuuint64_t dims[2] = {Ktot, (cuuint64_t)M};
        cuuint64_t strides[1] = {Ktot * elem};
        cuuint32_t box[2] = {(cuuint32_t)(128 / elem), (cuuint32_t)BN};
        cuuint32_t estr[2] = {1, 1};
        if (encode(&tf, dt, 2, const_cast<void *>(F), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    int patch2d = 0;
    if (patch) {
        const TcGeom g = tc_geom(Wx, K, BN, elem, true);
        const int HW = Wx * Wy;
        // one 2-D box per stage when channel rows are 16-B strided and one box
        // covers the patch; else one 1-D box per channel (any alignment)
        if (g.nbox == 1 && ((int64_t)HW * elem) % 16 == 0) {
            cuuint64_t dims[2] = {(cuuint64_t)HW, (cuuint64_t)N * C};
            cuuint64_t strides[1] = {(cuuint64_t)HW * elem};
            cuuint32_t box[2] = {(cuuint32_t)g.pb, (cuuint32_t)g.pch};
            cuuint32_t estr[2] = {1, 1};
            if (encode(&ti, dt, 2, const_cast<void *>(I), dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
                patch2d = 1;
        }
        if (!patch2d) {
            cuuint64_t dims[1] = {(cuuint64_t)N * C * HW};
            cuuint64_t strides[1] = {0};
            cuuint32_t box[1] = {(cuuint32_t)g.pb};
            cuuint32_t estr[1] = {1};
            if (encode(&ti, dt, 1, const_cast<void *>(I), dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
                patch = false;
        }
    }
    conv_plan q = p;
    if ((p.tma_f & 32) && tma_b && patch && patch2d)
        return launch_tc_persist<kTF32, BN>(p, tf, ti, C, Wx, Wy, K, M, O, s, N);
    if (p.tma_f & 32) {                               // planned persistent, but the patch map failed
        conv_plan r;
        plan_tc_nopersist(C, Wx, Wy, K, M, !kTF32, F, &r, N);
        q = r;
    }
    if (!patch) {
        q.smem_bytes = tc_geom(Wx, K, BN, elem, false).smem;
        return tma_b ? launch_tc<kTF32, BN, true, false>(q, tf, ti, I, C, Wx, Wy, F, K, M, O, patch2d, s, N)
                     : launch_tc<kTF32, BN, false, false>(q, tf, ti, I, C, Wx, Wy, F, K, M, O, patch2d, s, N);
    }
    return tma_b ? launch_tc<kTF32, BN, true, true>(q, tf, ti, I, C, Wx, Wy, F, K, M, O, patch2d, s, N)
                 : launch_tc<kTF32, BN, false, true>(q, tf, ti, I, C, Wx, Wy, F, K, M, O, patch2d, s, N);
}

template <bool kTF32>
static cudaError_t launch_tc_prec(const conv_plan &p, const void *I, int C, int Wx, int Wy,
                                  const void *F, int K, int M, float *O, cudaStream_t s, int N) {
    switch (p.tile_m) {
        case 32: return launch_tc_bn<kTF32, 32>(p, I, C, Wx, Wy, F, K, M, O, s, N);
        case 64: return launch_tc_bn<kTF32, 64>(p, I, C, Wx, Wy, F, K, M, O, s, N);
        case 256: return launch_tc_bn<kTF32, 256>(p, I, C, Wx, Wy, F, K, M, O, s, N);
        default: return launch_tc_bn<kTF32, 128>(p, I, C, Wx, Wy, F, K, M, O, s, N);
    }
}

int tc_max_clusters(int cluster, int smem) {
    auto kern = kmtc_kernel<true, 128, true, true>;
    ensure_smem((const void *)kern, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cluster, 1, 1);
    cfg.blockDim = dim3(kTcThreads);
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

cudaError_t launch_multi_tc(const void *I, int C, int Wx, int Wy, const void *F, int K, int M,
                            float *O, bool bf16, cudaStream_t s, int N) {
    conv_plan p;
    plan_multi_tc(C, Wx, Wy, K, M, bf16, F, &p, N);
    return bf16 ? launch_tc_prec<false>(p, I, C, Wx, Wy, F, K, M, O, s, N)
                : launch_tc_prec<true>(p, I, C, Wx, Wy, F, K, M, O, s, N);
}

}  // namespace b200
