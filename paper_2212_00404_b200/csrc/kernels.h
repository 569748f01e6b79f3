// kernels.h — internal launch interface between the C ABI (abi.cu) and the
// three kernels (KS, KM-SIMT, KM-TC).  Not part of the public ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../include/b200conv.h"

namespace b200 {

// SM count of the current device (cudaDevAttrMultiProcessorCount, cached per
// device; 148 on B200, and the fallback when no device is present, so plans
// stay computable on a host without a GPU).  Planners size grids against it.
int num_sms();

// Diagnostic builds (-DB200CONV_DIAG, `python -m paper_2212_00404_b200.build
// --diag` -> libb200conv_diag.so) compile the timeline stamps and the work-
// skipping switches of B200CONV_{KS,SIMT,TC}_DBG; the product library has
// none of them (the kernels see dbg == 0 as a constant).
#ifdef B200CONV_DIAG
constexpr bool kDiag = true;
#else
constexpr bool kDiag = false;
#endif

// NEXT-4: B200CONV_PLANNER=paper makes the KS row-block decision follow the
// paper's latency model (§2.2 procedure) instead of the measured
// threshold; A/B in profiles/planner_ab_r02.txt (the model is 4 % slower over
// the 17 layers where the two differ, so the threshold is the default).  The
// KM-SIMT ring depth always follows the model (its choice is the measured best).
bool planner_paper_model();

// Documented planner overrides (include/b200conv.h "Planner overrides"): an
// integer environment variable, or `def` when unset.  They only choose among
// correct plans (tests force every path with them); read at each call.
int env_override(const char *name, int def);

// Raise a kernel's dynamic shared memory limit to at least `bytes` (and allow
// non-portable cluster sizes).  The limit only ever grows, under a mutex, so a
// concurrent launch of the same kernel with a smaller footprint never fails.
cudaError_t ensure_smem(const void *kernel, int bytes);

// Programmatic dependent launch on/off (env B200CONV_PDL=0 disables it).
int pdl_enabled();

// KS: single-channel FP32 (conv_single.cu)
int plan_single(int Wx, int Wy, int K, int M, conv_plan *p);
cudaError_t launch_single(const float *I, int Wx, int Wy, const float *F, int K, int M, float *O,
                          cudaStream_t s);

// KS-C3: the channel-summing KS variant for C = 3 (RGB stem) layers, every
// precision (conv_single.cu); plan nonzero / cudaErrorNotSupported otherwise
int plan_multi_c3(int C, int Wx, int Wy, int K, int M, conv_plan *p);
cudaError_t launch_multi_c3(const void *I, int C, int Wx, int Wy, const void *F, int K, int M, float *O,
                            bool bf16, cudaStream_t s);

// KM-SIMT: multi-channel strict FP32 (conv_multi_simt.cu); sd = stride
// (output (Wy-K)/sd+1 x (Wx-K)/sd+1)
// Nimg > 1: a batch I [Nimg][C][Wy][Wx] -> O [Nimg][M][Ho][Wo] in one launch
// (pixel tiles over all images' compact pixels)
int plan_multi_simt(int C, int Wx, int Wy, int K, int M, conv_plan *p, int sd = 1, int Nimg = 1);
cudaError_t launch_multi_simt(const float *I, int C, int Wx, int Wy, const float *F, int K, int M,
                              float *O, cudaStream_t s, int sd = 1, int Nimg = 1);

// KM-TC: multi-channel tcgen05 implicit GEMM, TF32 or BF16 (conv_multi_tc.cu)
// N > 1: a batch of N images, I [N][C][Wy][Wx], O [N][M][Ho][Wo] (shared F)
int plan_multi_tc(int C, int Wx, int Wy, int K, int M, bool bf16, const void *F, conv_plan *p, int N = 1);
cudaError_t launch_multi_tc(const void *I, int C, int Wx, int Wy, const void *F, int K, int M,
                            float *O, bool bf16, cudaStream_t s, int N = 1);

// KM-TC/G: explicit im2col (L2-resident workspace) + TMA-fed tcgen05 GEMM
// (conv_multi_gemm.cu).  plan returns nonzero / launch returns
// cudaErrorNotSupported when the shape, alignment or workspace rules it out.
// sd > 1: stride (compact pixels; the only tensor-core path for strided calls).
// N > 1 with sd > 1: all N images (I [N][C][Wy][Wx], O [N][M][Ho][Wo]) in one GEMM.
int plan_multi_gemm(int C, int Wx, int Wy, int K, int M, bool bf16, conv_plan *p, int sd = 1, int N = 1);
cudaError_t launch_multi_gemm(const void *I, int C, int Wx, int Wy, const void *F, int K, int M, float *O,
                              bool bf16, cudaStream_t s, int sd = 1, int N = 1);

// Split-K chooser: cluster size S (1..max_split) minimising
//   waves(S) * (ceil(units / S) * t_unit + (S > 1) * t_reduce),
// waves(S) = ceil(tiles / clusters_resident(S)), with the co-resident cluster
// counts MEASURED on B200 (cudaOccupancyMaxActiveClusters; tools/cluster_occ.py)
// for kernels that fit 1 or 2 CTAs per SM.
int choose_split(int tiles, int units, int max_split, int ctas_per_sm, float t_unit,
                 float t_reduce);
// co-resident clusters of size S (1..16) for 1 or 2 CTAs per SM (same table)
int clusters_resident(int S, int ctas_per_sm);

// NEXT-2 (epilogue-fused all-gather of the filter-sharded O): the final-store
// sites of the split-K reduce kernel and of the KM-TC/G GEMM write every
// output value to the primary O and to up to kMaxPeers - 1 more buffers (peer
// memory mapped into this process, e.g. torch symmetric memory), or ONE
// multimem store to a multicast address covering all of them.  n == 0 and
// mc == nullptr: a plain call.  Set by conv_multi_allgather_ex for the
// duration of its launches (thread-local), read by those launchers.
constexpr int kMaxPeers = 8;
struct PeerOut {
    float *p[kMaxPeers - 1];   // extra destinations, each offset like the primary O
    float *mc;                 // multicast address of the primary O (replaces every store)
    int n;                     // number of extra destinations
};
const PeerOut &peer_out();
void set_peer_out(const PeerOut *po);       // nullptr: back to plain calls
__device__ __forceinline__ void out_store(const PeerOut &po, float *O, int64_t idx, float v) {
    if (po.mc) {
        asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(po.mc + idx), "f"(v) : "memory");
        return;
    }
    O[idx] = v;
    for (int r = 0; r < po.n; ++r) po.p[r][idx] = v;
}
// copy n floats from src to every peer destination (fallback for plans whose
// final stores are not peer-aware)
cudaError_t launch_peer_copy(const float *src, int64_t n, cudaStream_t s);

// Valid input width of the map the KM-TC kernels read (padded calls, NEXT-3):
// the zero-padded copy of I has 16-B-multiple row strides (Wx) so the patch
// keeps its 2-D TMA boxes, and only Wv - K + 1 output columns are real.
// 0 = Wx.  Thread-local, set by conv_multi_pad_ex around its launch.
void set_valid_width(int Wv);
int valid_width();

// Every ABI entry point holds a CallScope for the duration of the call: the
// graph-private scratch allocated while a stream is being captured is freed
// (cudaFreeAsync, in stream order) when the outermost scope ends.
struct CallScope {
    CallScope();
    ~CallScope();
    CallScope(const CallScope &) = delete;
    CallScope &operator=(const CallScope &) = delete;
};

// split-K workspace (workspace.cu): >= bytes of device memory owned by the
// library for (current device, stream); during stream capture a graph memory
// allocation private to the captured graph (needs a CallScope); nullptr on OOM
void *workspace_get(size_t bytes, cudaStream_t s);
// zero-padded input copies (padded calls): a second per-(device, stream) buffer
void *padbuf_get(size_t bytes, cudaStream_t s);
// filter rows re-strided for the strided tensor-core path: a third buffer
void *auxbuf_get(size_t bytes, cudaStream_t s);
// Fp[m][k] = F[m][k] (k < Ktot), 0 (Ktot <= k < Kp)
cudaError_t launch_pad_rows(const void *F, int M, int Ktot, int Kp, int elem, void *Fp, cudaStream_t s);
// Ip = I with a zero border of `pad` on every side of each of NC planes
cudaError_t launch_pad(const void *I, int NC, int Wx, int Wy, int pad, int elem, void *Ip, cudaStream_t s,
                       int Wps = 0);   // Wps: row stride of Ip (>= Wx + 2 pad; 0 = Wx + 2 pad), extra columns zero
// O[m][n] = sum_{s<S} W[s*slice + m*ldw + n] in order s = 0..S-1; plane < N:
// a batch, column n is pixel n % plane of image n / plane, O [N/plane][M][plane]
cudaError_t launch_splitk_reduce(const float *W, int S, int64_t slice, int M, int ldw, int N, float *O,
                                 cudaStream_t s, int plane = 0);

// 2-D FP32 tensor map, no swizzle, zero fill out of bounds (conv_multi_gemm.cu):
// [outer][inner] elements, row stride stride_bytes, box [box_outer][box_inner]
bool encode_f32_2d_plain(CUtensorMap *m, const void *base, uint64_t inner, uint64_t outer, uint64_t stride_bytes,
                         uint32_t box_inner, uint32_t box_outer);

// empty PDL-attributed kernel (the launch floor, diagnostics)
cudaError_t launch_nop(cudaStream_t s);

// max co-resident clusters (diagnostics)
int tc_max_clusters(int cluster, int smem);
int tc_read_stamps(unsigned long long *host);
int ks_read_stamps(unsigned long long *host);
int ks_read_fine(unsigned long long *host);
int tc_read_cta_stamps(unsigned long long *host);
int gm_read_cta_stamps(unsigned long long *host);
int simt_max_clusters(int cluster, int smem);
int simt_read_stamps(unsigned long long *host);

}  // namespace b200
