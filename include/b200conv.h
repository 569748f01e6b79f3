/*
 * b200conv.h — C ABI of libb200conv.so, the B200 (sm_100a) hot path of
 * arXiv 2212.00404: direct, valid-mode, stride-1 convolution.
 *
 * Operation (§2.1 "The Convolution Models", Eq. 1):
 *
 *   O^m(x,y) = sum_{ch=1}^{C} sum_{i=0}^{K-1} sum_{j=0}^{K-1} I^ch(x+i, y+j) * F^{ch,m}(i,j),
 *   x in [0, Wx-K+1), y in [0, Wy-K+1), m in [1, M]
 *
 * and its single-channel case C = 1 (Eq. 2).  With the reading Q1
 * of DESIGN.md (filter row r pairs with the map row y) and
 * 0-based indices this is
 *
 *   O[m][y][x] = sum_{ch,r,c} I[ch][y+r][x+c] * F[m][ch][r][c]
 *
 * i.e. cross-correlation (no kernel flip), identical to
 * torch.nn.functional.conv2d(I[None], F)[0] on contiguous NCHW/OIHW tensors.
 *
 * Layouts (row-major, x fastest, no padding, no row pitch):
 *   I : [C][Wy][Wx]                         (single-channel: [Wy][Wx])
 *   F : [M][C][K][K], element (((m*C+ch)*K+r)*K+c)
 *       "stored along the dimension ch first, and then along the dimension m"
 *       (P:337-338); single-channel [M][K][K] "stored ... continuously"
 *   O : [M][Wy-K+1][Wx-K+1], fully overwritten, never accumulated into.
 *
 * Ownership: every array pointer of the device entry points is a CUDA device
 * pointer owned by the caller; the library keeps no pointer after the call.
 * The library allocates (i) its workspace — split-K partial tiles and the
 * KM-TC/G im2col matrix — and (ii) the zero-padded input copy of the padded
 * calls: one device buffer each per (device, stream), grown on demand
 * (geometric growth; superseded buffers stay allocated, since work in flight
 * may still reference them) and kept for the process lifetime.  A call made
 * while its stream is being captured into a CUDA graph bakes in that stream's
 * buffer if it is big enough, else a graph memory allocation (cudaMallocAsync
 * node before its kernels, cudaFreeAsync node after them) private to the
 * graph.  Hence: graphs captured on the SAME stream may share scratch and must
 * be replayed in stream order (not concurrently on different streams); to
 * replay graphs concurrently, capture them on different streams.  Likewise
 * two threads issuing calls on the same stream handle (cudaStreamPerThread is
 * one value for all threads; the legacy stream) share its buffers and must be
 * ordered by that stream, as any work on one stream is.  The *_host entry
 * points take host pointers and use a library-owned stream-ordered memory
 * pool.  O must not overlap I or F.
 *
 * Execution: asynchronous and stream-ordered on the given stream (a
 * cudaStream_t / CUstream passed as void*; NULL = legacy default stream);
 * no host synchronisation inside the device entry points.  Kernel faults
 * surface at the caller's next synchronisation.  Reentrant: the only mutable
 * global state is the per-kernel shared-memory limit (raised monotonically
 * under a mutex, never lowered), the per-device SM-count / cluster-occupancy
 * cache and the workspace cache (mutex-protected).
 *
 * Planner overrides (environment, read at each call; they only choose among
 * correct plans, the tests force every path with them, unset = the planner):
 *   B200CONV_PDL=0          no programmatic dependent launch
 *   B200CONV_GM=0|2         KM-TC/G im2col+GEMM path off | forced where legal
 *   B200CONV_GM_SPLIT=S     KM-TC/G k split (cluster size) S
 *   B200CONV_GM_DSMEM=1     KM-TC/G split-K partials through DSMEM instead of
 *                           the L2 workspace
 *   B200CONV_TC_BN=32..256  KM-TC filter-tile width
 *   B200CONV_TC_SPLIT=S     KM-TC k split S
 *   B200CONV_TC_PERSIST=0   no persistent KM-TC for batched calls
 *   B200CONV_TC_DSMEM=0|1   KM-TC split-K partials exchanged through L2 (0) or
 *                           DSMEM (1); default DSMEM for splits <= 4
 *   B200CONV_SIMT_FORCE=t,S,ws  KM-SIMT thread tile t, channel split S, ws=1:
 *                           reduced through the workspace
 *   B200CONV_C3=0           no KS-C3 (C = 3 stems take the general kernels)
 *   B200CONV_PLANNER=paper  KS row blocks by the paper's N_FMA rule instead
 *                           of the measured row threshold (NEXT-4 A/B)
 *   B200CONV_SIMT_NST=2..4  KM-SIMT ring depth (3, 4: one CTA per SM)
 *   B200CONV_KS_FLAT=0|1    KS-L (line-aligned flat chunks for K = 3 maps whose
 *                           output rows are not whole 128-B lines) off | used
 *                           wherever legal (default: Ho >= 128, M >= 256)
 * Timeline stamps and work-skipping diagnostics exist only in the separate
 * -DB200CONV_DIAG build (libb200conv_diag.so), never in this library.
 *
 * Errors: the return value is a conv_status.  On any argument error nothing is
 * launched and O is untouched.  Checks, in order:
 *   CONV_E_SHAPE      any of C, Wx, Wy, K, M < 1, K > min(Wx, Wy),
 *                     or an element count above 2^31-1
 *   CONV_E_NULL       a null array pointer
 *   CONV_E_ALIGN      a pointer not aligned to its element size
 *   CONV_E_PRECISION  unknown precision
 *   CONV_E_DEVICE     the current CUDA device is not sm_100 (or none exists)
 *   CONV_E_LAUNCH     the launch itself failed (cudaGetLastError after launch)
 */
#ifndef B200CONV_H
#define B200CONV_H

#include <stdint.h>

#if defined(__GNUC__)
#define B200CONV_API __attribute__((visibility("default")))
#else
#define B200CONV_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CONV_OK = 0,
    CONV_E_SHAPE = 1,
    CONV_E_NULL = 2,
    CONV_E_ALIGN = 3,
    CONV_E_PRECISION = 4,
    CONV_E_DEVICE = 5,
    CONV_E_LAUNCH = 6
} conv_status;

/* Arithmetic of the multi-channel path (north_star: "TF32 and BF16 inputs
 * with FP32 accumulate ... alongside a strict-FP32 SIMT direct kernel").
 *   CONV_FP32: I, F float; FP32 FFMA on CUDA cores (kernel KM-SIMT)
 *   CONV_TF32: I, F float; tcgen05.mma kind::tf32, FP32 accumulate in TMEM
 *              (operands enter the tensor core as TF32: the low 13 mantissa
 *              bits are ignored by the hardware) (kernel KM-TC)
 *   CONV_BF16: I, F __nv_bfloat16 (caller converts, RNE); tcgen05.mma
 *              kind::f16 with BF16 inputs, FP32 accumulate (kernel KM-TC)
 * O is always float. */
typedef enum { CONV_FP32 = 0, CONV_TF32 = 1, CONV_BF16 = 2 } conv_precision;

/* Single-channel convolution, Eq. 2, strict FP32 on CUDA cores
 * (kernel KS), legacy default stream.  I [Wy][Wx], F [M][K][K], O [M][Ho][Wo]. */
B200CONV_API int conv_single(const float *I, int Wx, int Wy, const float *F, int K, int M, float *O);

/* Multi-channel convolution, Eq. 1, strict FP32 (kernel KM-SIMT),
 * legacy default stream.  I [C][Wy][Wx], F [M][C][K][K], O [M][Ho][Wo]. */
B200CONV_API int conv_multi(const float *I, int C, int Wx, int Wy, const float *F, int K, int M, float *O);

/* As conv_single on an explicit stream. */
B200CONV_API int conv_single_ex(const float *I, int Wx, int Wy, const float *F, int K, int M, float *O,
                   void *stream);

/* As conv_multi with an explicit precision (conv_precision) and stream.
 * For CONV_BF16, I and F point to bfloat16 arrays of the same shapes. */
B200CONV_API int conv_multi_ex(const void *I, int C, int Wx, int Wy, const void *F, int K, int M, float *O,
                  int precision, void *stream);

/* Batch of N images sharing one filter bank (the layers as CNNs run them,
 * P:25-42): I [N][C][Wy][Wx], O [N][M][Wy-K+1][Wx-K+1] (device
 * pointers, same element types as conv_multi_ex).  TF32 / BF16: ONE launch of
 * the implicit tensor-core kernel whose pixel tiles span all N images (no
 * split-K needed once N fills the machine).  CONV_FP32: ONE KM-SIMT launch
 * whose pixel tiles span all N images (+ the split-K reduce when planned);
 * the C = 3 stem layers (KS-C3) and N == 1: one conv_multi_ex call per image.  N < 1 or N*C*Wx*Wy / N*M*Ho*Wo > INT_MAX:
 * CONV_E_SHAPE; other errors as conv_multi_ex. */
B200CONV_API int conv_multi_batched_ex(const void *I, int N, int C, int Wx, int Wy, const void *F, int K, int M,
                          float *O, int precision, void *stream);

/* Zero ("same"-style) padding, stride 1: the input is
 * read as if surrounded by `pad` zero rows / columns, so
 * O [N][M][Wy+2*pad-K+1][Wx+2*pad-K+1].  A pre-pass kernel writes the padded
 * copy of I into a library-owned per-stream buffer, then the same kernels as
 * conv_single_ex / conv_multi_batched_ex run on it (one extra launch).
 * pad == 0 is exactly the unpadded call.  pad < 0, N < 1 or a size overflow:
 * CONV_E_SHAPE.  CONV_E_LAUNCH if the buffer would have to grow while the
 * stream is being captured (run the shape once before capturing). */
B200CONV_API int conv_single_pad_ex(const float *I, int Wx, int Wy, const float *F, int K, int M, int pad, float *O,
                       void *stream);
B200CONV_API int conv_multi_pad_ex(const void *I, int N, int C, int Wx, int Wy, const void *F, int K, int M, int pad,
                      float *O, int precision, void *stream);

/* Stride (PAPER.md treats stride 1 only): output
 * pixel (y, x) is the window at input (y*stride, x*stride) of the zero-padded
 * input, so O [N][M][Ho][Wo] with Ho = (Wy+2*pad-K)/stride+1 and
 * Wo = (Wx+2*pad-K)/stride+1 (torch.nn.functional.conv2d(I, F, stride=stride,
 * padding=pad)).  stride == 1 is exactly conv_*_pad_ex.  stride > 1:
 *   CONV_FP32  KM-SIMT with strided im2col gathers, one launch (+ split-K
 *              reduce) over all N images;
 *   CONV_TF32 / CONV_BF16  KM-TC/G: the strided im2col of all N images into
 *              the workspace, then ONE TMA-fed tcgen05 GEMM; filter rows that are not 16-B
 *              strided are first copied to zero-padded rows in a third
 *              library-owned per-stream buffer (one extra launch).
 * conv_single_strided_ex is the C = 1 case on the FP32 path.  stride < 1,
 * pad < 0, N < 1 or a size overflow: CONV_E_SHAPE; CONV_E_LAUNCH if a library
 * buffer would have to grow while the stream is being captured. */
B200CONV_API int conv_single_strided_ex(const float *I, int Wx, int Wy, const float *F, int K, int M, int pad,
                           int stride, float *O, void *stream);
B200CONV_API int conv_multi_strided_ex(const void *I, int N, int C, int Wx, int Wy, const void *F, int K, int M,
                          int pad, int stride, float *O, int precision, void *stream);

/* End-to-end entry points on HOST buffers (pageable or pinned): copy I and F
 * host->device, run the same kernels as the *_ex calls, copy O device->host,
 * and synchronise the stream before returning.  Device scratch comes from a
 * library-owned stream-ordered memory pool (allocated once, then reused).  For CONV_BF16
 * the host I and F are bfloat16 arrays. */
B200CONV_API int conv_single_host(const float *I, int Wx, int Wy, const float *F, int K, int M, float *O,
                     void *stream);
B200CONV_API int conv_multi_host(const void *I, int C, int Wx, int Wy, const void *F, int K, int M, float *O,
                    int precision, void *stream);

/* Asynchronous host-buffer entry points: the same copies and kernels enqueued
 * on `stream`, WITHOUT the final synchronisation, so a caller can keep several
 * calls in flight on different streams and overlap their host->device and
 * device->host copies (two copy engines).  I, F and O must be page-locked
 * (cudaHostAlloc / torch pin_memory) for the copies to be asynchronous; they
 * must stay valid, and O must not be read, until the caller synchronises
 * `stream`.  Argument errors are returned before anything is enqueued; copy
 * or kernel faults surface at that synchronisation. */
B200CONV_API int conv_single_host_async(const float *I, int Wx, int Wy, const float *F, int K, int M, float *O,
                           void *stream);
B200CONV_API int conv_multi_host_async(const void *I, int C, int Wx, int Wy, const void *F, int K, int M, float *O,
                          int precision, void *stream);

/* Launch plan the device entry points use for a shape (a function of the
 * shape and of the current device's SM count / cluster occupancy, queried
 * once; B200 values when no device is present; no device memory access).  A call of the hot path is one kernel launch, or two when
 * the channel split is reduced through the library's split-K workspace
 * (launches == 2: a deterministic fixed-order reduction kernel follows). */
typedef struct {
    int kernel;        /* 0 = KS (single FP32), 1 = KM-SIMT (multi FP32), 2 = KM-TC implicit (tf32/bf16),
                          3 = KM-TC/G: im2col kernel + TMA-fed tcgen05 GEMM (tf32/bf16),
                          4 = KS-C3: channel-summing KS for C = 3, K = 3 / 5 layers (every precision) */
    int grid_x, grid_y, grid_z;
    int block_x;
    int cluster_x;     /* split-K factor over channels / K-blocks (1 = none) */
    int tile_m;        /* filters per CTA tile (KS: per task; KS-L: per lane, P planes apart) */
    int tile_n;        /* (wide) output pixels per CTA tile (KS: rows per task; -1: the generic
                          single-channel kernel; -2: KS-L, 64-float line-aligned flat chunks) */
    int smem_bytes;    /* dynamic shared memory per CTA */
    int tma_f;         /* bit 0: F tiles by TMA; bit 1: I patch by TMA (KM-TC); bit 2: im2col tiles by
                          TMA (KM-TC/G); bit 3: filters on the 128-lane M side (KM-TC/G); bit 5:
                          persistent KM-TC (grid_y CTAs, one per SM, walk all tiles; block_x 480) */
    int launches;      /* kernel launches per call: 1, or 2 (split-K through the workspace;
                          cluster_x is then 1 and grid_x is the split count) */
    int chunk_k;       /* KM-SIMT: k-steps (channels x K x K) per pipeline stage; 0 = other kernels */
} conv_plan;

B200CONV_API int conv_plan_single(int Wx, int Wy, int K, int M, conv_plan *out);
B200CONV_API int conv_plan_multi(int C, int Wx, int Wy, int K, int M, int precision, conv_plan *out);
/* Plan of conv_multi_batched_ex (N == 1 and the C = 3 stem layers in FP32:
 * the per-image plan). */
B200CONV_API int conv_plan_multi_batched(int N, int C, int Wx, int Wy, int K, int M, int precision, conv_plan *out);
/* Plan of conv_multi_strided_ex (stride > 1: kernel 1 = the KM-SIMT launch
 * for CONV_FP32, kernel 3 = the KM-TC/G GEMM for CONV_TF32 / CONV_BF16, both
 * over all N images; stride 1: conv_plan_multi_batched of the padded map). */
B200CONV_API int conv_plan_multi_strided(int N, int C, int Wx, int Wy, int K, int M, int pad, int stride,
                            int precision, conv_plan *out);

/* Filter-sharded call with the all-gather fused into the epilogue (SURVEY
 * §8(f) NEXT-2; Fig. 2(c), lifted to GPUs): this rank's
 * F [M][C][K][K] (filters m0 .. m0+M-1 of M_total) produces O rows
 * [m0, m0+M) of the full O [M_total][Ho][Wo], and the final stores of the
 * kernels write them straight into every rank's copy of O: O_peers[0..n_peers)
 * are device pointers valid in this process (the local O and the peers' O
 * mapped over NVLink, e.g. torch symmetric-memory buffer_ptrs), n_peers <= 8.
 * O_mc, when non-null, is a multicast address of that buffer (NVSwitch
 * multicast object, e.g. symmetric-memory multicast_ptr): every value is then
 * ONE multimem.st reaching all GPUs, and O_peers[0] is still required.  The
 * final-store sites of the KM-SIMT split-K reduce and of the KM-TC/G GEMM are
 * peer-aware; other plans (implicit KM-TC, KS-C3, unsplit KM-SIMT) store
 * locally and a copy kernel in the same stream pushes the rows to the peers.
 * The data is complete on a rank once every rank's call has finished (e.g.
 * stream sync + a process-group barrier).  Errors as conv_multi_ex, plus
 * CONV_E_SHAPE for m0 < 0, m0 + M > M_total, n_peers outside 1..8. */
B200CONV_API int conv_multi_allgather_ex(const void *I, int C, int Wx, int Wy, const void *F, int K, int M, int m0,
                                         int M_total, float *const *O_peers, int n_peers, float *O_mc, int precision,
                                         void *stream);

/* The paper's latency-hiding model (§2.2; SURVEY §8(f)
 * NEXT-4) for a device profile: profile 0 = the current B200 (577-clock DRAM
 * latency, 128 FP32 lanes and the measured 6554 GB/s at 1965 MHz), 1 = the
 * paper's GTX 1080Ti (Table 1).  out[5] receives N_FMA (FMAs per
 * SM per data set for method 1), the latency volume (bytes per clock x
 * latency), the 4-B loading threads per SM that move it (rounded up to the
 * core count), V_s (the minimum volume they move) and bytes per clock.
 * CONV_E_NULL / CONV_E_SHAPE (unknown profile) on bad arguments.  The KM-SIMT
 * planner sets its ring depth from it; the KS planner does with
 * B200CONV_PLANNER=paper. */
B200CONV_API int conv_latency_model(int profile, double *out);

B200CONV_API const char *conv_status_string(int status);

/* ABI version: (major << 16) | minor. */
B200CONV_API int conv_version(void);

#ifdef __cplusplus
}
#endif
#endif /* B200CONV_H */
