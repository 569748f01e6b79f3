// workspace.cu — split-K partial-sum workspace and its deterministic
// reduction kernel (shared by KM-SIMT and KM-TC).
//
// When a layer has too few output tiles to fill 148 SMs, the channel sum of
// Eq. 1 is split S ways (the paper's Fig. 2(b) split along ch,
// P:350-361).  Up to 16 splits can be reduced through distributed shared
// memory inside one thread-block cluster; beyond that (or when clusters of the
// needed size do not co-reside) each split writes its partial tile to a
// device workspace W[S][Mpad][Npad] and `splitk_reduce_kernel` sums the S
// slices in a fixed order (deterministic: no atomics) into the compact
// O[M][Ho*Wo].
//
// The workspace is owned by the library: one buffer per (device, stream),
// grown (never shrunk, old buffers retired but kept alive) on demand.  A call
// captured into a CUDA graph uses its stream's buffer when that is big
// enough (graph memory nodes measured 2-7 us slower per call on the bench
// layers); when it is not, the buffer cannot grow during capture and the call
// gets a graph memory allocation (cudaMallocAsync inside the capture, freed by
// cudaFreeAsync after the call's last kernel) private to that graph.  So
// graphs captured on one stream may share its buffer: replay them in stream
// order (the header states this).
#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>
#include <vector>
#include <cuda_bf16.h>
#include "kernels.h"
#include "ptx.cuh"

namespace b200 {

namespace {
struct WsBuf { void *p = nullptr; size_t bytes = 0; };
std::mutex g_ws_mu;
std::map<std::pair<int, cudaStream_t>, WsBuf> g_ws;
std::map<std::pair<int, cudaStream_t>, WsBuf> g_pad;
std::map<std::pair<int, cudaStream_t>, WsBuf> g_aux;
std::vector<void *> g_ws_retired;
// graph-private scratch of the calls being captured on this thread, released
// when the outermost entry point returns
thread_local std::vector<std::pair<void *, cudaStream_t>> t_graph_scratch;
thread_local int t_call_depth = 0;
}  // namespace

namespace {
thread_local PeerOut t_peer_out = {};
}
thread_local int t_valid_width = 0;
const PeerOut &peer_out() { return t_peer_out; }
void set_valid_width(int Wv) { t_valid_width = Wv; }
int valid_width() { return t_valid_width; }
void set_peer_out(const PeerOut *po) { t_peer_out = po ? *po : PeerOut{}; }

CallScope::CallScope() { ++t_call_depth; }
CallScope::~CallScope() {
    if (--t_call_depth > 0) return;
    for (auto &ps : t_graph_scratch) cudaFreeAsync(ps.first, ps.second);
    t_graph_scratch.clear();
}

static void *buffer_get(std::map<std::pair<int, cudaStream_t>, WsBuf> &pool, size_t bytes, cudaStream_t s);

void *workspace_get(size_t bytes, cudaStream_t s) { return buffer_get(g_ws, bytes, s); }

// The zero-padded copy of I for padded calls: a second per-(device, stream)
// buffer, so the kernels of the same call can still use the workspace.
void *padbuf_get(size_t bytes, cudaStream_t s) { return buffer_get(g_pad, bytes, s); }

// A third per-(device, stream) buffer: filter rows re-strided to a 16-B
// multiple for the strided tensor-core path (launch_multi_gemm).
void *auxbuf_get(size_t bytes, cudaStream_t s) { return buffer_get(g_aux, bytes, s); }

static void *buffer_get(std::map<std::pair<int, cudaStream_t>, WsBuf> &pool, size_t bytes, cudaStream_t s) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    std::unique_lock<std::mutex> lk(g_ws_mu);
    WsBuf &b = pool[{dev, s}];
    if (b.bytes >= bytes) return b.p;
    if (cs != cudaStreamCaptureStatusNone) {
        // the stream's buffer is too small and cannot grow during capture:
        // graph-private scratch (a memory node of the captured graph)
        lk.unlock();
        if (t_call_depth == 0) return nullptr;
        void *p = nullptr;
        if (cudaMallocAsync(&p, bytes, s) != cudaSuccess) { cudaGetLastError(); return nullptr; }
        t_graph_scratch.emplace_back(p, s);
        return p;
    }
    // The old buffer is retired, not freed: in-flight work, or a CUDA graph
    // captured earlier on this stream, may still reference it.  Growth is
    // geometric, so retired buffers total less than the live one.
    if (b.p) {
        g_ws_retired.push_back(b.p);
        b.p = nullptr;
    }
    size_t want = bytes < (size_t(16) << 20) ? (size_t(16) << 20) : bytes;
    if (want < 2 * b.bytes) want = 2 * b.bytes;
    b.bytes = 0;
    if (cudaMalloc(&b.p, want) != cudaSuccess) { cudaGetLastError(); b.p = nullptr; return nullptr; }
    b.bytes = want;
    return b.p;
}

// O[m][n] = sum_{s=0}^{S-1} W[s][m][n], m < M, n < N (compact O, row stride N;
// W rows padded to ldw, a multiple of 4; slice = Mpad * ldw floats).
// G (1 or 8) adjacent lanes share one float4 of outputs: lane g sums the
// slices s = g, g + G, ... in order (8 loads in flight), then the G lane sums
// combine by a fixed xor tree — the same order on every run, so the result is
// deterministic.
template <int kRedG, bool kBatch>
__global__ void __launch_bounds__(256)
splitk_reduce_kernel(const float *__restrict__ W, int S, int64_t slice, int M, int ldw, int N,
                     float *__restrict__ O, int plane, const PeerOut po) {
    pdl_wait();
    pdl_trigger();
    // plain compact output, 16-B aligned rows: vector stores (peer / multicast
    // destinations keep the per-element out_store).  Only with one lane per
    // float4 (kRedG == 1): with 8-lane groups (S > 16) the vector store made
    // the PDL-chained call 4 us slower on ResNet 14x14 (S = 32: 15.3 vs
    // 11.4 us) although the reduce kernel alone was 4 % faster; configs[4]
    // (S = 6): 114.4 -> 113.9 us.
    const bool vec_ok = kRedG == 1 && !kBatch && po.mc == nullptr && po.n == 0 && (N & 3) == 0 &&
                        (reinterpret_cast<uintptr_t>(O) & 15) == 0;
    // 32-bit indexing: M * N <= INT_MAX is an ABI precondition
    const int q_per_row = (N + 3) >> 2;
    const int total = M * q_per_row;
    const int g = threadIdx.x % kRedG;
    constexpr int kGroupsPerWarp = 32 / kRedG;
    const int stride = gridDim.x * (blockDim.x / kRedG);
    // warp-uniform trip count (the shuffles below need all 32 lanes)
    for (int ub = blockIdx.x * (blockDim.x / kRedG) + (threadIdx.x / 32) * kGroupsPerWarp; ub < total;
         ub += stride) {
        const int u = ub + (threadIdx.x % 32) / kRedG;
        const bool valid = u < total;
        const int m = valid ? u / q_per_row : 0;
        const int n = valid ? 4 * (u - m * q_per_row) : 0;
        const float *w = W + (int64_t)m * ldw + n;
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        const int Sv = valid ? S : 0;
        // 8 loads in flight per lane (the partials sit in L2: latency-bound)
        for (int s0 = g; s0 < Sv; s0 += 8 * kRedG) {
            float4 b[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (s0 + j * kRedG < Sv) b[j] = __ldcs(reinterpret_cast<const float4 *>(w + (s0 + j * kRedG) * slice));
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (s0 + j * kRedG < Sv) { a.x += b[j].x; a.y += b[j].y; a.z += b[j].z; a.w += b[j].w; }
        }
#pragma unroll
        for (int o = kRedG / 2; o >= 1; o >>= 1) {   // (no-op for kRedG == 1)
            a.x += __shfl_xor_sync(0xffffffffu, a.x, o);
            a.y += __shfl_xor_sync(0xffffffffu, a.y, o);
            a.z += __shfl_xor_sync(0xffffffffu, a.z, o);
            a.w += __shfl_xor_sync(0xffffffffu, a.w, o);
        }
        if (valid && g == 0) {
            const float v[4] = {a.x, a.y, a.z, a.w};
            if constexpr (!kBatch) {
                const int64_t o = (int64_t)m * N + n;
                if (vec_ok && n + 4 <= N) {
                    // one 16-B store per thread (consecutive lanes: consecutive
                    // float4 of the compact O rows): whole sectors per warp store
                    // (four scalar stores strided by 16 B wrote every sector in
                    // up to four partial pieces, configs[4]: 925 K L2 write
                    // sectors for a 2.36 MB output)
                    *reinterpret_cast<float4 *>(O + o) = a;
                } else {
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        if (n + i < N) out_store(po, O, o + i, v[i]);
                }
            } else {
                // batch of N / plane images: column n + i is pixel (n+i) % plane of image (n+i) / plane
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    if (n + i >= N) break;
                    const int img = (n + i) / plane;
                    O[((int64_t)img * M + m) * plane + (n + i - img * plane)] = v[i];
                }
            }
        }
    }
}

// Ip[n][c][y][x] = I[n][c][y - pad][x - pad] inside, 0 in the border and in
// the columns Wx + 2 pad <= x < Wp of a wider row stride Wp (elem = 4 or 2
// bytes; one element per thread, grid-stride).
template <typename T>
__global__ void __launch_bounds__(256)
pad_kernel(const T *__restrict__ I, int NC, int Wx, int Wy, int pad, T *__restrict__ Ip, int Wp) {
    pdl_wait();
    pdl_trigger();
    const int Hp = Wy + 2 * pad;
    const int64_t total = (int64_t)NC * Hp * Wp;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t plane = i / ((int64_t)Hp * Wp);
        const int rem = (int)(i - plane * Hp * Wp);
        const int y = rem / Wp - pad, x = rem % Wp - pad;
        T v = T(0.f);
        if (y >= 0 && y < Wy && x >= 0 && x < Wx) v = I[(plane * Wy + y) * Wx + x];
        Ip[i] = v;
    }
}

// The same with 16-B output rows (Wp * sizeof(T) a multiple of 16, Ip 16-B
// aligned): one 16-B vector of a padded row per thread, one index decode per
// vector instead of per element.
template <typename T>
__global__ void __launch_bounds__(256)
pad_vec_kernel(const T *__restrict__ I, int NC, int Wx, int Wy, int pad, T *__restrict__ Ip, int Wp) {
    constexpr int V = 16 / sizeof(T);
    pdl_wait();
    pdl_trigger();
    const int Hp = Wy + 2 * pad, nv = Wp / V;
    const int64_t total = (int64_t)NC * Hp * nv;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / nv;                      // plane * Hp + yp
        const int xv = (int)(i - row * nv) * V;
        const int64_t plane = row / Hp;
        const int y = (int)(row - plane * Hp) - pad;
        union { uint4 u; T e[V]; } v;
        const T *src = I + (plane * Wy + y) * Wx;
        const bool yok = y >= 0 && y < Wy;
#pragma unroll
        for (int e = 0; e < V; ++e) {
            const int x = xv + e - pad;
            v.e[e] = (yok && x >= 0 && x < Wx) ? src[x] : T(0.f);
        }
        reinterpret_cast<uint4 *>(Ip)[i] = v.u;
    }
}

cudaError_t launch_pad(const void *I, int NC, int Wx, int Wy, int pad, int elem, void *Ip, cudaStream_t s,
                       int Wps) {
    if (Wps < Wx + 2 * pad) Wps = Wx + 2 * pad;
    if ((Wps * elem) % 16 == 0 && reinterpret_cast<uintptr_t>(Ip) % 16 == 0) {
        const int64_t vecs = (int64_t)NC * (Wy + 2 * pad) * (Wps * elem / 16);
        int64_t blocks = (vecs + 255) / 256;
        if (blocks > 8 * num_sms()) blocks = 8 * num_sms();
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(blocks < 1 ? 1 : blocks));
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (elem == 2)
            return cudaLaunchKernelEx(&cfg, pad_vec_kernel<__nv_bfloat16>, static_cast<const __nv_bfloat16 *>(I),
                                      NC, Wx, Wy, pad, static_cast<__nv_bfloat16 *>(Ip), Wps);
        return cudaLaunchKernelEx(&cfg, pad_vec_kernel<float>, static_cast<const float *>(I), NC, Wx, Wy, pad,
                                  static_cast<float *>(Ip), Wps);
    }
    const int64_t total = (int64_t)NC * (Wy + 2 * pad) * Wps;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 8 * num_sms()) blocks = 8 * num_sms();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(blocks < 1 ? 1 : blocks));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (elem == 2)
        return cudaLaunchKernelEx(&cfg, pad_kernel<__nv_bfloat16>, static_cast<const __nv_bfloat16 *>(I), NC, Wx,
                                  Wy, pad, static_cast<__nv_bfloat16 *>(Ip), Wps);
    return cudaLaunchKernelEx(&cfg, pad_kernel<float>, static_cast<const float *>(I), NC, Wx, Wy, pad,
                              static_cast<float *>(Ip), Wps);
}

// Fp[m][k] = F[m][k] for k < Ktot, 0 for Ktot <= k < Kp (elem-byte elements)
template <typename T>
__global__ void __launch_bounds__(256)
pad_rows_kernel(const T *__restrict__ F, int M, int Ktot, int Kp, T *__restrict__ Fp) {
    pdl_wait();
    pdl_trigger();
    const int64_t total = (int64_t)M * Kp;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = i / Kp;
        const int k = (int)(i - m * Kp);
        Fp[i] = k < Ktot ? F[m * Ktot + k] : T(0.f);
    }
}

cudaError_t launch_pad_rows(const void *F, int M, int Ktot, int Kp, int elem, void *Fp, cudaStream_t s) {
    const int64_t total = (int64_t)M * Kp;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 8 * num_sms()) blocks = 8 * num_sms();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(blocks < 1 ? 1 : blocks));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (elem == 2)
        return cudaLaunchKernelEx(&cfg, pad_rows_kernel<__nv_bfloat16>, static_cast<const __nv_bfloat16 *>(F), M,
                                  Ktot, Kp, static_cast<__nv_bfloat16 *>(Fp));
    return cudaLaunchKernelEx(&cfg, pad_rows_kernel<float>, static_cast<const float *>(F), M, Ktot, Kp,
                              static_cast<float *>(Fp));
}

cudaError_t launch_splitk_reduce(const float *W, int S, int64_t slice, int M, int ldw, int N, float *O,
                                 cudaStream_t s, int plane) {
    if (plane <= 0) plane = N;
    const PeerOut po = plane == N ? peer_out() : PeerOut{};
    // few splits: one lane per float4 of outputs; many: 8 lanes (latency)
    const int Gd = S > 16 ? 8 : 1;
    const int G = kDiag ? (env_override("B200CONV_REDG", Gd) == 8 ? 8 : 1) : Gd;
    const int64_t total = (int64_t)M * ((N + 3) / 4);
    int64_t blocks = (total * G + 255) / 256;          // one float4 group per G lanes
    if (blocks > 4 * num_sms()) blocks = 4 * num_sms();        // grid-stride: CTA launch rate, not work, bounds tiny CTAs
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
    // a batch (plane < N) maps columns to (image, pixel): its own instantiation,
    // so the single-image store path is the plain one
    if (plane != N) {
        if (G == 8) return cudaLaunchKernelEx(&cfg, splitk_reduce_kernel<8, true>, W, S, slice, M, ldw, N, O, plane, po);
        return cudaLaunchKernelEx(&cfg, splitk_reduce_kernel<1, true>, W, S, slice, M, ldw, N, O, plane, po);
    }
    if (G == 8) return cudaLaunchKernelEx(&cfg, splitk_reduce_kernel<8, false>, W, S, slice, M, ldw, N, O, plane, po);
    return cudaLaunchKernelEx(&cfg, splitk_reduce_kernel<1, false>, W, S, slice, M, ldw, N, O, plane, po);
}

__global__ void __launch_bounds__(256) peer_copy_kernel(const float *__restrict__ src, int64_t n, const PeerOut po) {
    pdl_wait();
    pdl_trigger();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float v = src[i];
        if (po.mc) {
            multimem_st_f32(po.mc + i, v);
        } else {
            for (int r = 0; r < po.n; ++r) po.p[r][i] = v;
        }
    }
}

cudaError_t launch_peer_copy(const float *src, int64_t n, cudaStream_t s) {
    const PeerOut &po = peer_out();
    if (n <= 0 || (!po.mc && po.n == 0)) return cudaSuccess;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 4 * num_sms()) blocks = 4 * num_sms();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, peer_copy_kernel, src, n, po);
}

// empty kernel with the same launch attributes as the hot-path kernels: the
// dependent-launch floor every call of the library pays (bench launch_floor_us)
__global__ void nop_kernel() {
    pdl_wait();
    pdl_trigger();
}

cudaError_t launch_nop(cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(32);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, nop_kernel);
}

}  // namespace b200
