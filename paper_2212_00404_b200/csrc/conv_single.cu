// conv_single.cu — kernel KS: single-channel direct convolution, strict FP32 on
// CUDA cores (§2.1 Eq. 2; the paper's single-channel
// kernel, §3.1, re-designed for sm_100a).
//
//   O[m][y][x] = sum_{r,c} I[y+r][x+c] * F[m][r][c]
//
// For K <= 3 the output stream (O is >= 94 % of all bytes for Wx >= 56) binds
// to HBM; for K >= 5 the FP32 FMA pipe binds.  Design:
//  * Work is a grid of tasks (a block of RB full-width output rows) x (a group
//    of R filters), each cut into 32-lane segments; the segments of the whole
//    problem are dealt to ALL warps of one wave (3 CTAs x 8 warps per SM) in
//    contiguous ranges that differ by at most one segment, so every SM gets the
//    same work (no ragged last wave, no idle SMs) — the B200 counterpart of the
//    paper's SM-assignment scheme (§3.1, Eqs. 4-9).
//  * A CTA's range covers a contiguous band of row blocks: the band's input
//    rows (ONE contiguous range of I) and the taps of its filter groups are
//    staged once in shared memory with cp.async — "only the feature maps are
//    divided ... processed by all filters", maximising FMAs per
//    loaded byte.  Taps of the current group sit in registers
//    ("filters fully to registers").
//  * A lane computes TX consecutive pixels x RR consecutive rows x R filters
//    from a (RR+K-1) x (TX+K-1) shared-memory window (vector loads; an input
//    row feeds min(RR, K) output rows), and writes each (row, filter) result
//    as VS-wide vector stores.  Consecutive lanes own consecutive pixels of a
//    row, so every warp store is coalesced.  VS divides Wo, so stores stay
//    aligned for any output offset.
#include <cstdint>
#include <cstdlib>
#include <type_traits>
#include <cuda_bf16.h>
#include "kernels.h"
#include "latency_model.h"
#include "ptx.cuh"

namespace b200 {

constexpr int kKsThreads = 256;
constexpr int kKsWarps = kKsThreads / 32;
// resident CTAs per SM: 3 (24 warps, <= 80 registers) for the store-bound small
// K; 2 (16 warps, <= 128 registers) for the FMA-bound K >= 5, whose 4 x 4 pixel
// register tiles need the room
__host__ __device__ constexpr int ks_min_blocks(int K) { return K >= 5 ? 2 : 3; }

// Launch parameters of one KS call (computed by plan_ks on the host).
struct KsArgs {
    const void *I;    // float (or bf16 for the C = 3 variant)
    const void *F;
    float *O;
    int Wx, Wy, M;
    int L;        // lane slots per output row: ceil(Wo / TX)
    int RWt;      // row groups (of RR rows) per task: a task is RB = RWt*RR rows x R filters
    int NG;       // filter groups ceil(M / R)
    int nseg;     // 32-slot segments per task: ceil(RWt * L / 32)
    int U;        // work units = tasks * nseg   (task t = (row block t / NG, group t % NG))
    int NW;       // warps in the grid
    int ub, ur;   // U = ub * NW + ur: warp w owns units [w*ub + min(w, ur), (w+1)*ub + min(w+1, ur))
    int gmax;     // filter-group capacity of the smem tap table
    int dbg;      // diagnostics: 1 = per-CTA globaltimer stamps into g_ks_stamps
    int prefetch; // L2 prefetch of the CTA's inputs before griddepcontrol.wait (B200CONV_PREFETCH=0: off)
    int cstride;  // kC > 1: floats per staged channel in shared memory
};

// diagnostics (B200CONV_KS_DBG=1): per CTA [start, after griddepcontrol.wait,
// staged, done << 8 | smid] globaltimer stamps of the last launch, CTAs 0..1023
__device__ unsigned long long g_ks_stamps[4 * 1024];
__device__ unsigned long long g_ks_fine[16];   // dbg == 2: CTA 0 warp 0 lane 0, first unit
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
int ks_read_fine(unsigned long long *host) {
    return cudaMemcpyFromSymbol(host, g_ks_fine, sizeof(g_ks_fine)) == cudaSuccess ? 0 : 1;
}
int ks_read_stamps(unsigned long long *host) {
    return cudaMemcpyFromSymbol(host, g_ks_stamps, sizeof(g_ks_stamps)) == cudaSuccess ? 0 : 1;
}

template <int V>
__device__ __forceinline__ void lds_vec(const float *p, float *d) {
    if constexpr (V == 4) {
        const float4 v = *reinterpret_cast<const float4 *>(p);
        d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
    } else if constexpr (V == 2) {
        const float2 v = *reinterpret_cast<const float2 *>(p);
        d[0] = v.x; d[1] = v.y;
    } else {
        d[0] = *p;
    }
}
template <int V>
__device__ __forceinline__ void stg_vec(float *p, const float *v) {
    if constexpr (V == 4) *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
    else if constexpr (V == 2) *reinterpret_cast<float2 *>(p) = make_float2(v[0], v[1]);
    else *p = v[0];
}

// Work unit = one 32-slot segment of one task.  Slot s of a task = (row group
// rg = s / L, column slot xv = s % L); its lane computes pixels x = TX*xv ..
// x+TX-1 (the last slot of a row may be partial) of rows y0 .. y0+RR-1.
// Loads are VL-wide (VL | Wx and the I alignment), stores VS-wide (VS | Wo).
//
// kC > 1 (the RGB stem layers, C = 3): the same kernel summing kC channels —
// each CTA stages kC planes' rows (converted to f32; T = float or bf16) and
// the lane's window loop runs over the channels (Eq. 1 with small C).
template <typename T> __device__ __forceinline__ float to_f32(T v) { return static_cast<float>(v); }
template <> __device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <int K, int TX, int VL, int VS, int R, int RR, int kC = 1, typename T = float>
__global__ void __launch_bounds__(kKsThreads, kC > 1 ? 2 : ks_min_blocks(K))
ks_kernel(const KsArgs a) {
    constexpr int KK = K * K;
    constexpr int CKK = kC * KK;                     // taps per filter
    constexpr bool kPlain = kC == 1 && std::is_same<T, float>::value;
    constexpr int GS = (R * CKK + 3) & ~3;           // floats per filter group (16-B rows)
    constexpr int NV = (TX + K - 1 + VL - 1) / VL;   // load vectors per window row
    extern __shared__ __align__(16) float smem[];
    const int Wx = a.Wx, Wy = a.Wy, M = a.M, L = a.L, NG = a.NG, nseg = a.nseg;
    const int Wo = Wx - K + 1, Ho = Wy - K + 1;
    const int RB = a.RWt * RR;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int dbg = kDiag ? a.dbg : 0;
    const bool stamp = dbg && tid == 0 && blockIdx.x < 1024;
    if (stamp) g_ks_stamps[4 * blockIdx.x] = gtimer();

    // this CTA's unit range -> task range -> row blocks and filter groups
    // (all decoding happens before griddepcontrol.wait: it overlaps the
    // previous kernel's tail)
    const int c0 = blockIdx.x * kKsWarps;
    const int u0 = c0 * a.ub + min(c0, a.ur);
    const int u1 = (c0 + kKsWarps) * a.ub + min(c0 + kKsWarps, a.ur);
    if (u0 >= u1) { pdl_trigger(); return; }
    const int t0 = u0 / nseg, t1 = (u1 - 1) / nseg + 1;
    const int row_lo = (t0 / NG) * RB;
    const int row_hi = min(Wy, ((t1 - 1) / NG + 1) * RB + K - 1);
    const int g_first = t0 % NG;
    const int ngr = min(NG, t1 - t0);

    // this warp's unit range, decoded once; then advanced incrementally
    const int gw = c0 + warp;
    const int w0 = gw * a.ub + min(gw, a.ur), w1 = (gw + 1) * a.ub + min(gw + 1, a.ur);
    int t = w0 / nseg, j = w0 - t * nseg;
    int rb = t / NG, g = t - rb * NG;
    const int q32 = 32 / L, r32 = 32 - q32 * L;        // slot step of one segment
    const int rg_l = lane / L, xv_l = lane - rg_l * L;  // slot of this lane in segment 0
    int rg = rg_l + j * q32, xv = xv_l + j * r32;       // slot of this lane in segment j
    while (xv >= L) { xv -= L; ++rg; }
    int gi = g - g_first;
    if (gi < 0) gi += NG;

    const T *__restrict__ Ig = static_cast<const T *>(a.I);
    const T *__restrict__ Fg = static_cast<const T *>(a.F);
    float *s_w = smem;                                // [gmax][GS]
    float *s_in = smem + a.gmax * GS;                 // input rows [row_lo, row_hi), + pad (per channel)
    // s_in[pad + e - e0] = I[e]: smem and global agree mod 16 B (kC == 1)
    const int64_t e0 = (int64_t)row_lo * Wx, e1 = (int64_t)row_hi * Wx;
    const int pad = kPlain ? (int)(((reinterpret_cast<uintptr_t>(a.I) >> 2) + e0) & 3) : 0;
    // bf16 rows can move as 4-B pairs when every channel's range starts 4-B aligned
    const bool pairs_ok = !kPlain && sizeof(T) == 2 && ((int64_t)Wx * Wy) % 2 == 0 && e0 % 2 == 0 &&
                          (reinterpret_cast<uintptr_t>(a.I) & 3) == 0 && ((e1 - e0) & 1) == 0;

    // warm L2 with this CTA's input rows and taps while the previous kernel drains
    if (a.prefetch) {
    for (int64_t e = e0 + 32 * tid; e < e1; e += 32 * kKsThreads) prefetch_l2(Ig + e);
    if (tid < ngr) {
        int g = g_first + tid;
        if (g >= NG) g -= NG;
        prefetch_l2(Fg + (int64_t)g * R * CKK);
    }
    }
    pdl_wait();
    if (stamp) g_ks_stamps[4 * blockIdx.x + 1] = gtimer();
    if constexpr (kPlain) {
    for (int idx = tid; idx < ngr * GS; idx += kKsThreads) {
        const int gi = idx / GS, e = idx - gi * GS;
        const int t = e / R, f = e - t * R;         // taps [t][f]: filter pairs adjacent (FFMA2)
        int g = g_first + gi;
        if (g >= NG) g -= NG;
        const int m = g * R + f;
        const bool ok = f < R && m < M;
        cp_async4(s_w + idx, ok ? Fg + (int64_t)m * KK + t : Fg, ok);
    }
    {
        const int nch = (int)((pad + (e1 - e0) + 3) >> 2);  // 16-B chunks of s_in
        for (int c = tid; c < nch; c += kKsThreads) {
            const int64_t e = e0 - pad + 4 * c;            // global element of the chunk's first float
            if (e >= e0 && e + 4 <= e1) {
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                             ::"r"(smem_u32(s_in + 4 * c)), "l"(Ig + e) : "memory");
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const bool ok = e + i >= e0 && e + i < e1;
                    cp_async4(s_in + 4 * c + i, ok ? Ig + e + i : Ig, ok);
                }
            }
        }
    }
    } else {
        // kC channels (f32 or bf16) -> f32 shared copies, plain loads
        for (int idx = tid; idx < ngr * GS; idx += kKsThreads) {
            const int gi = idx / GS, e = idx - gi * GS;
            const int t = e / R, f = e - t * R;     // taps [t][f]
            int g = g_first + gi;
            if (g >= NG) g -= NG;
            const int m = g * R + f;
            s_w[idx] = (f < R && m < M) ? to_f32(Fg[(int64_t)m * CKK + t]) : 0.f;
        }
        const int64_t HWp = (int64_t)Wx * Wy;
        const int n = (int)(e1 - e0);
        if constexpr (std::is_same<T, float>::value) {
            // asynchronous 4-B copies, all in flight at once
            for (int c = 0; c < kC; ++c)
                for (int e = tid; e < n; e += kKsThreads)
                    cp_async4(s_in + c * a.cstride + e, Ig + c * HWp + e0 + e, true);
        } else if (pairs_ok) {
            // bf16 pairs by 4-B copies into a raw area, widened after the wait
            __nv_bfloat16 *raw = reinterpret_cast<__nv_bfloat16 *>(s_in + kC * a.cstride);
            for (int c = 0; c < kC; ++c)
                for (int e = 2 * tid; e < n; e += 2 * kKsThreads)
                    cp_async4(raw + c * a.cstride + e, Ig + c * HWp + e0 + e, true);
        } else {
            // 16 independent loads in flight per thread
            constexpr int kUnr = 16;
            for (int b0 = tid; b0 < kC * n; b0 += kKsThreads * kUnr) {
                float v[kUnr];
#pragma unroll
                for (int u = 0; u < kUnr; ++u) {
                    const int idx = b0 + u * kKsThreads;
                    const int c = idx / n, e = idx - c * n;
                    v[u] = idx < kC * n ? to_f32(Ig[c * HWp + e0 + e]) : 0.f;
                }
#pragma unroll
                for (int u = 0; u < kUnr; ++u) {
                    const int idx = b0 + u * kKsThreads;
                    const int c = idx / n, e = idx - c * n;
                    if (idx < kC * n) s_in[c * a.cstride + e] = v[u];
                }
            }
        }
    }
    cp_async_commit();
    pdl_trigger();
    cp_async_wait<0>();
    __syncthreads();
    if constexpr (!kPlain && !std::is_same<T, float>::value) {
        if (pairs_ok) {                              // widen the raw bf16 rows
            const __nv_bfloat16 *raw = reinterpret_cast<const __nv_bfloat16 *>(s_in + kC * a.cstride);
            const int n = (int)(e1 - e0);
            for (int c = 0; c < kC; ++c)
                for (int e = tid; e < n; e += kKsThreads)
                    s_in[c * a.cstride + e] = __bfloat162float(raw[c * a.cstride + e]);
            __syncthreads();
        }
    }
    if (stamp) g_ks_stamps[4 * blockIdx.x + 2] = gtimer();

    if (w0 >= w1 && !dbg) return;

    const float *sin = s_in + pad - (int64_t)row_lo * Wx;   // sin[y*Wx + x] = I[y][x]
    const int64_t plane = (int64_t)Ho * Wo;
    float w[R * CKK];
    bool need_w = true;
    for (int u = w0; u < w1; ++u) {
        const bool fine = dbg == 2 && blockIdx.x == 0 && threadIdx.x == 0 && u == w0;
        if (fine) g_ks_fine[0] = gtimer();
        if (need_w) {                                 // (warp-uniform) new task: load its taps
            need_w = false;
            const float *ws = s_w + gi * GS;
#pragma unroll
            for (int q = 0; q < (R * CKK) / 4; ++q) {
                const float4 v = *reinterpret_cast<const float4 *>(ws + 4 * q);
                w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
            }
#pragma unroll
            for (int q = (R * CKK) & ~3; q < R * CKK; ++q) w[q] = ws[q];
        }
        if (fine) g_ks_fine[1] = gtimer();
        const int y0 = rb * RB + rg * RR;
        const int x = TX * xv;
        if (rg < a.RWt && y0 < Ho) {
            float acc[RR][R][TX];
#pragma unroll
            for (int q = 0; q < RR; ++q)
#pragma unroll
                for (int f = 0; f < R; ++f)
#pragma unroll
                    for (int v = 0; v < TX; ++v) acc[q][f][v] = 0.f;
#pragma unroll
            for (int ch = 0; ch < kC; ++ch) {
            const float *base = sin + ch * a.cstride + y0 * Wx + x;
#pragma unroll
            for (int ir = 0; ir < RR + K - 1; ++ir) {
                float win[NV * VL];
#pragma unroll
                for (int i = 0; i < NV; ++i) lds_vec<VL>(base + ir * Wx + i * VL, win + i * VL);
                // c outermost: consecutive FMAs update RR*R*TX different
                // accumulators (a lone warp on an SMSP stays at full issue rate)
#pragma unroll
                for (int c = 0; c < K; ++c)
#pragma unroll
                    for (int q = 0; q < RR; ++q) {
                        const int r = ir - q;         // filter row feeding output row q
                        if (r >= 0 && r < K) {
                            const int tap = (ch * KK + r * K + c) * R;
                            // paired FMAs (FFMA2, ptx.cuh) along filter pairs
                            // (broadcast input pixel; taps staged [t][f], so
                            // a pair is one aligned register pair); bitwise the
                            // same as fmaf.  (Pairing along pixels needs the
                            // odd-c window pairs re-formed by moves: measured
                            // slower on K = 5 / 7, R = 1, so those stay FFMA.)
                            if constexpr (R % 2 == 0) {
#pragma unroll
                                for (int f = 0; f < R; f += 2)
#pragma unroll
                                    for (int v = 0; v < TX; ++v)
                                        ffma2(acc[q][f][v], acc[q][f + 1][v], win[v + c], w[tap + f], w[tap + f + 1]);
                            } else {
#pragma unroll
                                for (int f = 0; f < R; ++f)
#pragma unroll
                                    for (int v = 0; v < TX; ++v)
                                        acc[q][f][v] = fmaf(win[v + c], w[tap + f], acc[q][f][v]);
                            }
                        }
                    }
            }
            }
            if (fine) g_ks_fine[2] = gtimer() + (unsigned long long)(acc[0][0][0] == 12345.f);
            float *of = a.O + ((int64_t)g * R * Ho + y0) * Wo + x;
            const int nvs = min(TX, Wo - x);          // valid pixels of this slot (multiple of VS)
            const int nq = min(RR, Ho - y0), nf = min(R, M - g * R);
#pragma unroll
            for (int f = 0; f < R; ++f, of += plane) {
                if (f >= nf) break;
                float *o = of;
#pragma unroll
                for (int q = 0; q < RR; ++q, o += Wo) {
                    if (q >= nq) break;
#pragma unroll
                    for (int v = 0; v < TX; v += VS)
                        if (TX == VS || v < nvs) stg_vec<VS>(o + v, &acc[q][f][v]);
                }
            }
        }
        if (fine) g_ks_fine[3] = gtimer();
        // next unit: next segment of this task, or segment 0 of the next task
        if (++j == nseg) {
            j = 0;
            rg = rg_l;
            xv = xv_l;
            need_w = true;
            if (++g == NG) { g = 0; ++rb; }
            if (++gi == NG) gi = 0;
        } else {
            rg += q32;
            xv += r32;
            if (xv >= L) { xv -= L; ++rg; }
        }
    }
    if (dbg) {
        __syncthreads();
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        if (stamp) g_ks_stamps[4 * blockIdx.x + 3] = (gtimer() << 8) | smid;
    }
}

// ---------------------------------------------------------------- KS-L: line-aligned flat units
// K = 3 maps whose output rows are not whole 128-B lines (Wo % 32 != 0, e.g.
// 224x224 -> 222 = 888-B rows): the row-block units above cut every row into
// 32-lane pieces that start mid-line, so each piece boundary's line is written
// by two warp stores (measured 1.51x L2 write requests and 13.95 vs 10.82 us
// against the 16-B/128-B aligned 226x226 map, profiles/ks_alignment_r02.txt).
// Here a unit is one 128-B-aligned 64-float chunk of ONE filter plane's flat
// output (rows run on into the next row): lane l computes the pixel pair at
// flat p = h + 64 (c - 1) + 2 l for four filters, so each of its four warp
// stores writes exactly two whole lines.  The four filters of a lane are
// m, m + P, m + 2P, m + 3P, where P is the alignment period of the planes
// (P * Ho * Wo == 0 mod 32 floats): they share the line offset h of their
// planes, so one pixel mapping is aligned for all four.  Rows of the pair
// never split (Wo even, p even).  Units (group, chunk) are dealt evenly over
// one wave of 3 CTAs per SM (equal work per SM: 11.9-12.2 vs 12.9 us with
// CTAs owning chunk ranges of one group, which left SMs with 2 or 3 CTAs);
// each CTA stages the input rows of its (at most two) groups' chunk ranges.
struct KfArgs {
    const float *I;
    const float *F;
    float *O;
    int Wx, Wy, M;
    int P;        // plane alignment period (filters)
    int R;        // filters per lane (4, or 8 at 2 CTAs per SM)
    int NG;       // filter groups: ceil(M / (4P)) * P
    int nch;      // 64-float chunks per plane (incl. the partial head chunk)
    int ub, ur;   // units U = NG * nch (u = g * nch + c) dealt to warps: [w*ub + min(w, ur), ...)
};

#ifndef B200CONV_KSL_ALIGN
#define B200CONV_KSL_ALIGN 4
#endif
constexpr int kKslAlign = B200CONV_KSL_ALIGN;   // staged block B alignment (floats, power of 2)

// first line-aligned flat index h of the planes of filter group g
__device__ __forceinline__ int ksl_h(int g, int P, int64_t plane) {
    return (32 - (int)(((int64_t)(g % P) * (plane & 31)) & 31)) & 31;
}

// Input rows [row_lo, row_hi) of chunks [c0, c1) of a group with head h.
__device__ __forceinline__ void ksl_rows(int h, int c0, int c1, int HW, int Wo, int Wy, int *lo, int *hi) {
    const int p_lo = max(0, h + 64 * (c0 - 1)), p_hi = min(HW - 1, h + 64 * c1 - 1);
    *lo = p_lo / Wo;
    *hi = max(*lo, min(Wy, p_hi / Wo + 3));
}

template <int R, int MB>   // R filters per lane (P apart), MB CTAs per SM
__global__ void __launch_bounds__(kKsThreads, MB) ks_flat_kernel(const KfArgs a) {
    constexpr int K = 3;
    extern __shared__ __align__(16) float smem[];
    const int Wx = a.Wx, Wy = a.Wy, M = a.M, P = a.P, nch = a.nch;
    const int Wo = Wx - K + 1, Ho = Wy - K + 1;
    const int HW = Ho * Wo;
    const int64_t plane = HW;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // Units u = g * nch + c (group-major: a warp writes long contiguous runs of
    // its group's four planes) dealt evenly over every warp of one wave of 3
    // CTAs per SM (equal work per SM).  A CTA's range covers at most two
    // groups (the planner checks): the end of group gA's planes and the start
    // of group gA + 1's, each with its own staged row block.
    const int cw = blockIdx.x * kKsWarps;
    const int u0 = cw * a.ub + min(cw, a.ur), u1 = (cw + kKsWarps) * a.ub + min(cw + kKsWarps, a.ur);
    if (u0 >= u1) { pdl_trigger(); return; }
    // (small planes: a CTA spanning three or more groups stages the whole map once)
    const int gA = u0 / nch, gB = (u1 - 1) / nch;
    const bool whole = gB > gA + 1;
    const int cA0 = u0 - gA * nch, cA1 = gB == gA ? u1 - gA * nch : nch;
    const int cB1 = gB == gA ? 0 : u1 - gB * nch;
    int rA0 = 0, rA1 = Wy, rB0 = 0, rB1 = 0;
    if (!whole) {
        ksl_rows(ksl_h(gA, P, plane), cA0, cA1, HW, Wo, Wy, &rA0, &rA1);
        if (gB != gA) ksl_rows(ksl_h(gB, P, plane), 0, cB1, HW, Wo, Wy, &rB0, &rB1);
    }
    const int64_t eA = (int64_t)rA0 * Wx, eB = (int64_t)rB0 * Wx;
    const int padA = (int)(((reinterpret_cast<uintptr_t>(a.I) >> 2) + eA) & 3);
    const int padB = (int)(((reinterpret_cast<uintptr_t>(a.I) >> 2) + eB) & 3);
    // block B follows block A's actual extent (16-B aligned)
    float *sA = smem, *sB = smem + ((padA + (rA1 - rA0) * Wx + 3 + kKslAlign) & ~(kKslAlign - 1));
    pdl_wait();
#pragma unroll 1
    for (int b = 0; b < 2; ++b) {
        const int64_t e0 = b ? eB : eA, e1 = b ? (int64_t)rB1 * Wx : (int64_t)rA1 * Wx;
        const int pad = b ? padB : padA;
        float *dst = b ? sB : sA;
        const int n16 = (int)((pad + (e1 - e0) + 3) >> 2);
        for (int c = tid; c < n16; c += kKsThreads) {
            const int64_t e = e0 - pad + 4 * c;
            if (e >= e0 && e + 4 <= e1) {
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                             ::"r"(smem_u32(dst + 4 * c)), "l"(a.I + e) : "memory");
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const bool ok = e + i >= e0 && e + i < e1;
                    cp_async4(dst + 4 * c + i, ok ? a.I + e + i : a.I, ok);
                }
            }
        }
    }
    cp_async_commit();
    pdl_trigger();
    cp_async_wait<0>();
    __syncthreads();
    const int gw = cw + warp;
    const int w0 = gw * a.ub + min(gw, a.ur), w1 = (gw + 1) * a.ub + min(gw + 1, a.ur);
    if (w0 >= w1) return;
    int g = w0 / nch, c = w0 - g * nch;
    float w[9 * R];
    float *O0 = a.O;
    const float *sin = sA;
    int64_t e0 = eA;
    int m0 = 0, p = 0, y = 0, x = 0;
    bool fresh = true;
    for (int u = w0; u < w1; ++u) {
        if (fresh) {                                     // (warp-uniform) first unit of a group run
            fresh = false;
            const int gb = g / P, r = g - gb * P;
            m0 = gb * P * R + r;
#pragma unroll
            for (int i = 0; i < R; ++i) {
                const int m = m0 + P * i;
#pragma unroll
                for (int t = 0; t < 9; ++t) w[t * R + i] = m < M ? __ldg(a.F + (int64_t)m * 9 + t) : 0.f;
            }
            O0 = a.O + (int64_t)m0 * plane;
            const bool inA = whole || g == gA;
            sin = (inA ? sA + padA : sB + padB) - (inA ? eA : eB);   // sin[y*Wx + x] = I[y][x]
            e0 = inA ? eA : eB;
            p = ksl_h(g, P, plane) + 64 * (c - 1) + 2 * lane;
            y = 0; x = p;
            if (p >= 0) { y = p / Wo; x = p - y * Wo; }
        }
        const bool valid = p >= 0 && p < HW;
        const float *base = sin + (valid ? (int64_t)y * Wx + x : e0);
        float acc[R][2];
#pragma unroll
        for (int i = 0; i < R; ++i) acc[i][0] = acc[i][1] = 0.f;
#pragma unroll
        for (int rr = 0; rr < K; ++rr) {
            float win[4];
            lds_vec<2>(base + rr * Wx, win);
            lds_vec<2>(base + rr * Wx + 2, win + 2);
#pragma unroll
            for (int cc = 0; cc < K; ++cc) {
                const int t = rr * K + cc;
#pragma unroll
                for (int v = 0; v < 2; ++v)
#pragma unroll
                    for (int f = 0; f < R; f += 2)
                        ffma2(acc[f][v], acc[f + 1][v], win[v + cc], w[t * R + f], w[t * R + f + 1]);
            }
        }
        if (valid) {
#pragma unroll
            for (int i = 0; i < R; ++i)
                if (m0 + P * i < M) stg_vec<2>(O0 + (int64_t)P * i * plane + p, acc[i]);
        }
        if (++c == nch) {
            c = 0;
            ++g;
            fresh = true;
        } else {
            p += 64;
            x += 64;
            while (x >= Wo) { x -= Wo; ++y; }
        }
    }
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

// per lane: TX pixels x RR rows x R filters.  K = 1 is store-bound -> many
// filters; large K is FMA-bound -> 4 pixels x 4 rows (an input row feeds
// min(RR, K) outputs, a window row of TX+K-1 loads feeds TX*K FMAs per filter)
__host__ __device__ constexpr int ks_TX(int K) { return K == 1 ? 4 : (K <= 3 ? 2 : 4); }
__host__ __device__ constexpr int ks_R(int K) { return K <= 1 ? 8 : (K <= 3 ? 4 : 1); }
__host__ __device__ constexpr int ks_RR(int K) { return K <= 1 ? 1 : (K <= 3 ? 2 : 4); }
// filters per lane of the C = 3 variant (weights: R * 3 * K * K registers)
__host__ __device__ constexpr int ks_R_c3(int K) { return K <= 3 ? 2 : 1; }

struct KsPlan {
    KsArgs a;
    int RR, VL, VS, G, smem;
};

bool al(const void *p, int bytes) { return p == nullptr || reinterpret_cast<uintptr_t>(p) % bytes == 0; }

// Max dynamic smem over the CTAs of a grid of G CTAs (filter taps + input rows).
void ks_cta_needs(const KsArgs &a, int K, int R, int RR, int TX, int G, int *gmax, int *smem, int kC,
                  int *cstride) {
    const int KK = K * K, GS = (R * kC * KK + 3) & ~3, RB = a.RWt * RR;
    int rows_max = 0, g = 1;
    for (int c = 0; c < G; ++c) {
        const int c0 = c * kKsWarps, c1 = c0 + kKsWarps;
        const int u0 = c0 * a.ub + (c0 < a.ur ? c0 : a.ur), u1 = c1 * a.ub + (c1 < a.ur ? c1 : a.ur);
        if (u0 >= u1) continue;
        const int t0 = u0 / a.nseg, t1 = (u1 - 1) / a.nseg + 1;
        const int n = t1 - t0 < a.NG ? t1 - t0 : a.NG;
        const int rows = ((t1 - 1) / a.NG - t0 / a.NG + 1) * RB + K - 1;
        if (n > g) g = n;
        if (rows > rows_max) rows_max = rows;
    }
    *gmax = g;
    *cstride = (rows_max * a.Wx + 2 * TX + 8 + 3) & ~3;        // floats per staged channel
    *smem = (g * GS + kC * *cstride) * 4;
}

// Returns false when the band kernel does not apply (K > 7 or the staged rows
// of a CTA do not fit in shared memory).
bool plan_ks(const void *I, int Wx, int Wy, const void *F, int K, int M, float *O, KsPlan *kp, int kC = 1,
             int elem = 4) {
    if (K > 7) return false;
    const int Wo = Wx - K + 1, Ho = Wy - K + 1;
    // small maps with K >= 3: one row per lane (a multi-row register block
    // would be mostly rows past Ho, lengthening every warp's serial FMA chain)
    // (measured, tools/ks_variants.py: 7x7 K=7 2.9 -> 2.2 us, 7x7 K=3 2.5 ->
    // 2.0 us, 28x28 K=3 2.24 -> 2.05 us; K >= 5 at 28x28 and K = 3 at 56x56
    // get slower).  B200CONV_KS_SMALL=<max Ho> overrides (0: off).
    const int small_ho = kDiag ? env_override("B200CONV_KS_SMALL", K == 3 ? 32 : 16) : (K == 3 ? 32 : 16);
    bool small = K >= 3 && Ho <= small_ho;
    if (planner_paper_model() && K >= 3) {
        // the paper's procedure (§2.2; NEXT-4): each SM's data set
        // is its share of the layer (the band a CTA stages, all filters);
        // fewer than N_FMA FMAs per SM -> method 2 (volume / latency bound):
        // 1-row blocks, the most independent units in flight; else method 1:
        // register row blocks, more FMAs per staged byte
        const LatencyModel lm = latency_model(b200_profile(num_sms()));
        const double fma_per_sm = (double)M * Ho * Wo * K * K / num_sms();
        small = paper_method(lm, fma_per_sm) == 2;
    }
    const int TX = ks_TX(K), R = kC > 1 ? ks_R_c3(K) : ks_R(K), RR = small ? 1 : ks_RR(K);
    KsArgs a = {};
    a.I = I; a.F = F; a.O = O;
    a.Wx = Wx; a.Wy = Wy; a.M = M;
    a.L = (Wo + TX - 1) / TX;
    // row groups per task: fewest lane-steps per filter group,
    //   ceil(Ho / (RWt*RR)) row blocks x ceil(RWt*L / 32) segments
    // (within 5 % of the minimum, the shortest task: finer work ranges and
    // fewer staged rows; two row blocks of input must fit in ~40 KB)
    int64_t cost[33];
    int64_t best = -1;
    int nr = 0;
    for (int rwt = 1; rwt <= 32; ++rwt) {
        if (rwt > 1 && (int64_t)(rwt - 1) * RR >= Ho) break;      // taller than the map
        if (rwt > 1 && (int64_t)(2 * rwt * RR + K - 1) * Wx * 4 > 40 * 1024) break;
        cost[rwt] = (int64_t)((Ho + rwt * RR - 1) / (rwt * RR)) * ((rwt * a.L + 31) / 32);
        if (best < 0 || cost[rwt] < best) best = cost[rwt];
        nr = rwt;
    }
    a.RWt = 1;
    for (int rwt = 1; rwt <= nr; ++rwt)
        if (cost[rwt] * 100 <= best * 105) { a.RWt = rwt; break; }
    a.NG = (M + R - 1) / R;
    a.nseg = (a.RWt * a.L + 31) / 32;
    const int64_t NRB = (Ho + a.RWt * RR - 1) / (a.RWt * RR);
    const int64_t U = NRB * a.NG * a.nseg;
    if (U > (int64_t)1 << 30) return false;
    a.U = (int)U;
    // one wave of ks_min_blocks(K) CTAs per SM, or one unit per warp if fewer
    // (K = 1, pure store stream: one CTA per SM measured fastest — 9.4 vs
    // 11.5 us for 224x224 M=256 — fewer warps per SM keep the store traffic
    // fairer across SMs; see tools/ks_variants.py)
    const int cap = (K == 1 ? 1 : (kC > 1 ? 2 : ks_min_blocks(K))) * num_sms();
    const int max_smem = (kC == 1 && ks_min_blocks(K) == 3 ? 72 : 110) * 1024;
    // (B200CONV_KS_SPREAD=1: at least one CTA per SM up to one unit per CTA;
    // measured neutral on the small maps, so off by default)
    int G = (a.U + kKsWarps - 1) / kKsWarps;
    if (kDiag && env_override("B200CONV_KS_SPREAD", 0) == 1) {
        const int spread = a.U < num_sms() ? a.U : num_sms();
        if (G < spread) G = spread;
    }
    if (G > cap) G = cap;
    if (const int g = kDiag ? env_override("B200CONV_KS_G", 0) : 0; g > 0)   // experiments: CTA count
        G = g < a.U ? g : a.U;
    for (;;) {
        a.NW = G * kKsWarps;
        a.ub = a.U / a.NW;
        a.ur = a.U - a.ub * a.NW;
        int smem;
        ks_cta_needs(a, K, R, RR, TX, G, &a.gmax, &smem, kC, &a.cstride);
        if (kC > 1 && elem == 2) smem += kC * a.cstride * 2;     // raw bf16 rows before widening
        if (smem <= max_smem || G >= a.U) {
            if (smem > 200 * 1024) return false;
            kp->a = a;
            kp->RR = RR;
            // window loads: TX-wide vectors, or 8-B pairs when rows are only
            // 8-B strided (Wx = 2 mod 4 with TX = 4: 230x230 K=7 M=256 went
            // scalar, 40.5 vs 26.6 us on 224x224)
            kp->VL = (kC == 1 && elem == 4 && Wx % TX == 0 && al(I, 4 * TX)) ? TX
                     : (kC == 1 && elem == 4 && TX == 4 && Wx % 2 == 0 && al(I, 8)) ? 2 : 1;
            kp->VS = (Wo % TX == 0 && al(O, 4 * TX)) ? TX : ((TX >= 2 && Wo % 2 == 0 && al(O, 8)) ? 2 : 1);
            if (RR != ks_RR(K)) kp->VL = kp->VS = 1;    // small-map variant: scalar loads / stores
            // channel planes are staged from offset 0 of 16-B aligned regions
            if (kC > 1) kp->VL = (Wx % TX == 0) ? TX : 1;
            kp->G = G;
            kp->smem = smem;
            return true;
        }
        if (G >= 4 * cap) return false;
        G = G * 2 > a.U ? a.U : G * 2;               // finer ranges -> fewer rows per CTA
    }
}
}  // namespace

// KS-L plan (K = 3 maps with rows that are not whole lines); false when it
// does not apply.  B200CONV_KS_FLAT=0 disables it, =1 uses it wherever legal.
static bool plan_ks_flat(const void *I, int Wx, int Wy, int K, int M, const float *O, KfArgs *fa, int *Gout,
                         int *smem_bytes) {
    const int v = env_override("B200CONV_KS_FLAT", -1);
    if (v == 0 || K != 3) return false;
    const int Wo = Wx - K + 1, Ho = Wy - K + 1;
    const int64_t HW = (int64_t)Ho * Wo;
    if (Wo < 2 || Ho < 1 || Wo % 2 != 0 || Wx % 2 != 0 || !al(I, 8) || !al(O, 128)) return false;
    if (HW + 64 > ((int64_t)1 << 30) / 4) return false;
    // measured (tools/ks_variants.py, 8 filters per lane): 224x224 M=256
    // 11.0 vs 13.7 us, M=128 7.1 vs 7.4; slower at M <= 64 and on 56-114 px
    // maps (the row-block kernel's two-row register blocks matter more there)
    if (v != 1 && (Wo % 32 == 0 || Ho < 128 || M < 128)) return false;
    int gcd = 32, q = (int)(HW & 31);
    for (int b = q; b != 0;) { const int t = gcd % b; gcd = b; b = t; }
    const int P = 32 / gcd;
    KfArgs a = {};
    a.Wx = Wx; a.Wy = Wy; a.M = M;
    a.P = P;
    // 8 filters per lane at 2 CTAs per SM (128 registers: 72 taps + 16
    // accumulators) measured faster than 4 at 3 CTAs per SM: 224x224 M=256
    // 11.1 vs 12.2 us, M=512 20.9 vs 21.8, M=1024 40.8 vs 57.9 (4-filter
    // version out of smem: row-block kernel)
    a.R = kDiag ? env_override("B200CONV_KSL_R", 8) : 8;
    if (a.R != 4) a.R = 8;
    const int MB = a.R == 8 ? 2 : 3;
    a.NG = (M + a.R * P - 1) / (a.R * P) * P;
    a.nch = (int)(1 + (HW + 63) / 64);
    const int64_t U = (int64_t)a.NG * a.nch;
    if (U > ((int64_t)1 << 30)) return false;
    // one wave of 3 CTAs per SM, units dealt evenly over its warps
    int G = (int)((U + kKsWarps - 1) / kKsWarps);
    if (G > MB * num_sms()) G = MB * num_sms();
    const int NW = G * kKsWarps;
    a.ub = (int)(U / NW);
    a.ur = (int)(U - (int64_t)a.ub * NW);
    const int64_t upc = (int64_t)kKsWarps * (a.ub + 1);      // units of the largest CTA
    // the two staged blocks together: the rows of at most upc chunks, each
    // block + head / tail slack and K - 1 halo rows; a CTA that may span three
    // or more groups (upc > nch: small planes) stages the whole map
    // (upc > nch: either both blocks can be the whole map, or one whole-map block)
    const int64_t rows = upc > a.nch ? 2 * (int64_t)Wy : ((upc + 2) * 64 + 64) / Wo + 2 * (K + 2);
    const int64_t sm = ((rows < 2 * Wy ? rows : 2 * Wy) * Wx + 20 + 2 * kKslAlign) * 4;
    if (sm > (MB == 3 ? 72 : 110) * 1024) return false;
    *fa = a;
    *Gout = G;
    *smem_bytes = (int)sm;
    return true;
}

int plan_single(int Wx, int Wy, int K, int M, conv_plan *p) {
    const int Wo = Wx - K + 1, Ho = Wy - K + 1;
    p->cluster_x = 1;
    p->tma_f = 0;
    p->launches = 1;
    p->kernel = 0;
    KfArgs fa;
    int fg = 0, fsm = 0;
    if (plan_ks_flat(reinterpret_cast<const float *>(256), Wx, Wy, K, M, reinterpret_cast<float *>(256), &fa, &fg,
                     &fsm)) {
        p->block_x = kKsThreads;
        p->grid_x = fg;
        p->grid_y = 1;
        p->grid_z = 1;
        p->tile_m = fa.R;                                 // filters per lane (P apart)
        p->tile_n = -2;                                   // marks KS-L (64-float flat chunks)
        p->smem_bytes = fsm;
        return 0;
    }
    KsPlan kp;
    // plans are computed for 16-B aligned I / O (torch allocations)
    if (plan_ks(reinterpret_cast<const float *>(256), Wx, Wy, nullptr, K, M,
                reinterpret_cast<float *>(256), &kp)) {
        p->block_x = kKsThreads;
        p->grid_x = kp.G;
        p->grid_y = 1;
        p->grid_z = 1;
        p->tile_m = ks_R(K);                              // filters per task
        p->tile_n = kp.a.RWt * kp.RR;                     // output rows per task (full width)
        p->smem_bytes = kp.smem;
        return 0;
    }
    // generic fallback: (x, y, m) tiles of 1 column x 4 rows x 4 filters per thread
    const int bx = Wo >= 128 ? 128 : ((Wo + 31) / 32) * 32;
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

template <int K, int VL, int VS, int RR = ks_RR(K)>
static cudaError_t launch_ks(const KsPlan &kp, cudaStream_t s) {
    auto kern = ks_kernel<K, ks_TX(K), VL, VS, ks_R(K), RR>;
    if (cudaError_t e = ensure_smem((const void *)kern, kp.smem); e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kp.G);
    cfg.blockDim = dim3(kKsThreads);
    cfg.dynamicSmemBytes = kp.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1] = {pdl_attr()};
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    KsArgs a = kp.a;
    a.dbg = kDiag ? env_override("B200CONV_KS_DBG", 0) : 0;
    a.prefetch = kDiag ? env_override("B200CONV_PREFETCH", 1) != 0 : 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

// VL in {TX, 2 (TX = 4), 1}; VS in {TX, 2, 1} (2 only when TX = 4)
template <int K>
static cudaError_t launch_ks_v(const KsPlan &kp, cudaStream_t s) {
    constexpr int TX = ks_TX(K);
    constexpr int V2 = TX >= 2 ? 2 : 1;
    if constexpr (ks_RR(K) != 1)
        if (kp.RR == 1) return launch_ks<K, 1, 1, 1>(kp, s);
    if constexpr (TX == 4) {
        if (kp.VL == 2) {
            if (kp.VS == TX) return launch_ks<K, 2, TX>(kp, s);
            if (kp.VS == 2) return launch_ks<K, 2, 2>(kp, s);
            return launch_ks<K, 2, 1>(kp, s);
        }
    }
    if (kp.VL == TX) {
        if (kp.VS == TX) return launch_ks<K, TX, TX>(kp, s);
        if (kp.VS == 2) return launch_ks<K, TX, V2>(kp, s);
        return launch_ks<K, TX, 1>(kp, s);
    }
    if (kp.VS == TX) return launch_ks<K, 1, TX>(kp, s);
    if (kp.VS == 2) return launch_ks<K, 1, V2>(kp, s);
    return launch_ks<K, 1, 1>(kp, s);
}

// ---------------------------------------------------------------- C = 3 (RGB stems)
// The multi-channel layers with three input channels (VGG / AlexNet / ResNet
// first layers) are output-store bound (C*K*K = 27 MACs per output) with too
// little reduction for a GEMM: the channel-summing KS variant runs them for
// every precision (TF32 inputs are consumed in full FP32 — more accurate than
// the TF32 tolerance needs; BF16 inputs are widened to FP32).
template <int K, int VL, int VS, typename T>
static cudaError_t launch_ks_c3(const KsPlan &kp, cudaStream_t s) {
    constexpr int RR = ks_RR(K);
    auto kern = ks_kernel<K, ks_TX(K), VL, VS, ks_R_c3(K), RR, 3, T>;
    if (cudaError_t e = ensure_smem((const void *)kern, kp.smem); e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kp.G);
    cfg.blockDim = dim3(kKsThreads);
    cfg.dynamicSmemBytes = kp.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1] = {pdl_attr()};
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    KsArgs a = kp.a;
    a.dbg = kDiag ? env_override("B200CONV_KS_DBG", 0) : 0;
    a.prefetch = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

template <int K, typename T>
static cudaError_t launch_ks_c3_v(const KsPlan &kp, cudaStream_t s) {
    constexpr int TX = ks_TX(K);
    constexpr int V2 = TX >= 2 ? 2 : 1;
    if (kp.VL == TX) {
        if (kp.VS == TX) return launch_ks_c3<K, TX, TX, T>(kp, s);
        if (kp.VS == 2) return launch_ks_c3<K, TX, V2, T>(kp, s);
        return launch_ks_c3<K, TX, 1, T>(kp, s);
    }
    if (kp.VS == TX) return launch_ks_c3<K, 1, TX, T>(kp, s);
    if (kp.VS == 2) return launch_ks_c3<K, 1, V2, T>(kp, s);
    return launch_ks_c3<K, 1, 1, T>(kp, s);
}

static bool c3_applies(int C, int K, int Wy) {
    if (env_override("B200CONV_C3", 1) == 0) return false;
    return C == 3 && (K == 3 || K == 5) && Wy - K + 1 > 16;   // (the 1-row small-map variant is not built)
}

int plan_multi_c3(int C, int Wx, int Wy, int K, int M, conv_plan *p) {
    if (!c3_applies(C, K, Wy)) return 1;
    KsPlan kp;
    if (!plan_ks(reinterpret_cast<const float *>(256), Wx, Wy, nullptr, K, M, reinterpret_cast<float *>(256), &kp, 3))
        return 1;
    p->kernel = 4;
    p->block_x = kKsThreads;
    p->grid_x = kp.G;
    p->grid_y = 1;
    p->grid_z = 1;
    p->cluster_x = 1;
    p->tile_m = ks_R_c3(K);                              // filters per task
    p->tile_n = kp.a.RWt * kp.RR;                        // output rows per task (full width)
    p->smem_bytes = kp.smem;
    p->tma_f = 0;
    p->launches = 1;
    return 0;
}

cudaError_t launch_multi_c3(const void *I, int C, int Wx, int Wy, const void *F, int K, int M, float *O,
                            bool bf16, cudaStream_t s) {
    if (!c3_applies(C, K, Wy)) return cudaErrorNotSupported;
    KsPlan kp;
    if (!plan_ks(I, Wx, Wy, F, K, M, O, &kp, 3, bf16 ? 2 : 4) || kp.RR != ks_RR(K)) return cudaErrorNotSupported;
    if (bf16) return K == 3 ? launch_ks_c3_v<3, __nv_bfloat16>(kp, s) : launch_ks_c3_v<5, __nv_bfloat16>(kp, s);
    return K == 3 ? launch_ks_c3_v<3, float>(kp, s) : launch_ks_c3_v<5, float>(kp, s);
}

cudaError_t launch_single(const float *I, int Wx, int Wy, const float *F, int K, int M, float *O,
                          cudaStream_t s) {
    {
        KfArgs fa;
        int G = 0, sm = 0;
        if (plan_ks_flat(I, Wx, Wy, K, M, O, &fa, &G, &sm)) {
            fa.I = I; fa.F = F; fa.O = O;
            auto kern = fa.R == 8 ? ks_flat_kernel<8, 2> : ks_flat_kernel<4, 3>;
            if (cudaError_t e = ensure_smem((const void *)kern, sm); e != cudaSuccess) return e;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(G);
            cfg.blockDim = dim3(kKsThreads);
            cfg.dynamicSmemBytes = sm;
            cfg.stream = s;
            cudaLaunchAttribute attr[1] = {pdl_attr()};
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            return cudaLaunchKernelEx(&cfg, kern, fa);
        }
    }
    KsPlan kp;
    if (plan_ks(I, Wx, Wy, F, K, M, O, &kp)) {
        switch (K) {
            case 1: return launch_ks_v<1>(kp, s);
            case 2: return launch_ks_v<2>(kp, s);
            case 3: return launch_ks_v<3>(kp, s);
            case 4: return launch_ks_v<4>(kp, s);
            case 5: return launch_ks_v<5>(kp, s);
            case 6: return launch_ks_v<6>(kp, s);
            case 7: return launch_ks_v<7>(kp, s);
            default: break;
        }
    }
    const int Wo = Wx - K + 1, Ho = Wy - K + 1;
    const int bx = Wo >= 128 ? 128 : ((Wo + 31) / 32) * 32;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((Wo + bx - 1) / bx, (Ho + 3) / 4, (M + 3) / 4);
    cfg.blockDim = dim3(bx);
    cfg.stream = s;
    cudaLaunchAttribute attr[1] = {pdl_attr()};
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, ks_kernel_generic<4, 4>, I, Wx, Wy, F, K, M, O);
}

}  // namespace b200
