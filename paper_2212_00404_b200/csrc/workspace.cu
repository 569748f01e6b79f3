// workspace.cu — split-K partial-sum workspace and its deterministic
// reduction kernel (shared by KM-SIMT and KM-TC).
//
// When a layer has too few output tiles to fill 148 SMs, the channel sum of
// Eq. 1 is split S ways (the paper's Fig. 2(b) split along ch,
// P:350-361).  Up to 16 splits can be reduced through distributed shared
// memory inside one thread-block cluster; beyond that (or when clusters of the
// needed size do not co-reside) each split writes its partial tile to a
// device workspace W[S][Mpad][Npad] and `splitk_reduce_kernel` sums the S
// slices in fixed order s = 0..S-1 (deterministic: no atomics) into the
// compact O[M][Ho*Wo].
//
// The workspace is owned by the library: one buffer per (device, stream),
// grown (never shrunk) on demand outside stream capture; a call made while
// the stream is being captured that would need a bigger buffer gets nullptr
// and the caller falls back to a cluster-only plan.
#include <cstdint>
#include <map>
#include <mutex>
#include <utility>
#include "kernels.h"
#include "ptx.cuh"

namespace b200 {

namespace {
struct WsBuf { void *p = nullptr; size_t bytes = 0; };
std::mutex g_ws_mu;
std::map<std::pair<int, cudaStream_t>, WsBuf> g_ws;
}  // namespace

void *workspace_get(size_t bytes, cudaStream_t s) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    std::lock_guard<std::mutex> lk(g_ws_mu);
    WsBuf &b = g_ws[{dev, s}];
    if (b.bytes >= bytes) return b.p;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    if (cs != cudaStreamCaptureStatusNone) return nullptr;
    // in-flight work on this stream may still read the old buffer
    if (b.p) {
        if (cudaStreamSynchronize(s) != cudaSuccess) { cudaGetLastError(); return nullptr; }
        cudaFree(b.p);
        b.p = nullptr;
        b.bytes = 0;
    }
    size_t want = bytes < (size_t(16) << 20) ? (size_t(16) << 20) : bytes;
    if (cudaMalloc(&b.p, want) != cudaSuccess) { cudaGetLastError(); b.p = nullptr; return nullptr; }
    b.bytes = want;
    return b.p;
}

// O[m][n] = sum_{s=0}^{S-1} W[s][m][n], m < M, n < N (compact O, row stride N;
// W rows padded to ldw, a multiple of 4; slice = Mpad * ldw floats).
__global__ void __launch_bounds__(256)
splitk_reduce_kernel(const float *__restrict__ W, int S, int64_t slice, int M, int ldw, int N,
                     float *__restrict__ O) {
    pdl_wait();
    pdl_trigger();
    const int q_per_row = (N + 3) >> 2;
    const int64_t total = (int64_t)M * q_per_row;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total;
         u += (int64_t)gridDim.x * blockDim.x) {
        const int m = (int)(u / q_per_row);
        const int n = 4 * (int)(u - (int64_t)m * q_per_row);
        const float *w = W + (int64_t)m * ldw + n;
        float4 a = __ldcs(reinterpret_cast<const float4 *>(w));
        for (int s = 1; s < S; ++s) {
            const float4 b = __ldcs(reinterpret_cast<const float4 *>(w + s * slice));
            a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
        }
        float *o = O + (int64_t)m * N + n;
        const float v[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (n + i < N) o[i] = v[i];
    }
}

cudaError_t launch_splitk_reduce(const float *W, int S, int64_t slice, int M, int ldw, int N, float *O,
                                 cudaStream_t s) {
    const int64_t total = (int64_t)M * ((N + 3) / 4);
    int64_t blocks = (total + 255) / 256;
    if (blocks > 8 * kNumSMs) blocks = 8 * kNumSMs;
    if (blocks < 1) blocks = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, splitk_reduce_kernel, W, S, slice, M, ldw, N, O);
}

}  // namespace b200
