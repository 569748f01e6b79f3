// abi.cu — the C ABI declared in include/b200conv.h: argument validation,
// device check, dispatch to one kernel launch per call, host-buffer entry
// points.  Every compute step of the hot path runs in the kernels; this file
// only checks and launches.
#include <array>
#include <atomic>
#include <climits>
#include <cstdlib>
#include <cstdint>
#include <map>
#include <mutex>
#include <utility>
#include <cuda_runtime.h>
#include "kernels.h"
#include "latency_model.h"

using namespace b200;

int b200::pdl_enabled() { return env_override("B200CONV_PDL", 1) != 0; }

bool b200::planner_paper_model() {
    const char *e = getenv("B200CONV_PLANNER");
    return e && e[0] == 'p';
}

int b200::env_override(const char *name, int def) {
    const char *e = getenv(name);
    if (!e || !*e) return def;
    char *end = nullptr;
    const long v = strtol(e, &end, 10);
    return end == e ? def : (int)v;
}

static int current_device() {
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return -1; }
    return dev;
}

int b200::num_sms() {
    static std::atomic<int> cache[64];
    const int dev = current_device();
    if (dev < 0 || dev >= 64) return 148;
    int v = cache[dev].load(std::memory_order_relaxed);
    if (v > 0) return v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) {
        cudaGetLastError();
        return 148;
    }
    cache[dev].store(v, std::memory_order_relaxed);
    return v;
}

cudaError_t b200::ensure_smem(const void *kernel, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void *>, int> limit;
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(mu);
    int &cur = limit[{dev, kernel}];
    if (bytes <= cur) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e == cudaSuccess) cur = bytes;
    return e;
}

// Co-resident clusters of size S for kernels that fit 1 or 2 CTAs per SM:
// cudaOccupancyMaxActiveClusters of a probe kernel with the same residency
// (256 threads, 200 KB or 100 KB of shared memory), queried once per device.
// Without a device (host-only plan queries) the values measured on B200 are
// used (148 SMs, 8 GPCs; tools/cluster_occ.py).
static const int kClusters1[17] = {0, 148, 74, 45, 33, 26, 22, 15, 15, 15, 11, 7, 7, 7, 7, 7, 7};
static const int kClusters2[17] = {0, 296, 148, 93, 71, 56, 45, 37, 33, 30, 26, 21, 21, 17, 14, 14, 14};

__global__ void occ_probe_kernel() {}

static const int *cluster_table(int ctas_per_sm) {
    static std::mutex mu;
    static std::map<int, std::array<int, 34>> tabs;
    const int dev = current_device();
    const int which = ctas_per_sm >= 2 ? 1 : 0;
    if (dev < 0) return which ? kClusters2 : kClusters1;
    std::lock_guard<std::mutex> lk(mu);
    auto it = tabs.find(dev);
    if (it == tabs.end()) {
        std::array<int, 34> t{};
        bool ok = true;
        for (int w = 0; w < 2 && ok; ++w) {
            const int smem = w ? 100 * 1024 : 200 * 1024;
            ok = ensure_smem((const void *)occ_probe_kernel, smem) == cudaSuccess;
            for (int S = 1; S <= 16 && ok; ++S) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(S);
                cfg.blockDim = dim3(256);
                cfg.dynamicSmemBytes = smem;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = S;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                int n = 0;
                ok = cudaOccupancyMaxActiveClusters(&n, occ_probe_kernel, &cfg) == cudaSuccess && n > 0;
                t[17 * w + S] = n;
            }
        }
        if (!ok) {
            cudaGetLastError();
            for (int S = 0; S < 17; ++S) { t[S] = kClusters1[S]; t[17 + S] = kClusters2[S]; }
        }
        it = tabs.emplace(dev, t).first;
    }
    return it->second.data() + 17 * which;
}

int b200::choose_split(int tiles, int units, int max_split, int ctas_per_sm, float t_unit,
                       float t_reduce) {
    const int *tab = cluster_table(ctas_per_sm);
    if (max_split > 16) max_split = 16;
    if (max_split > units) max_split = units;
    int best = 1;
    float best_t = -1.f;
    for (int S = 1; S <= (max_split < 1 ? 1 : max_split); ++S) {
        const int waves = (tiles + tab[S] - 1) / tab[S];
        // every wave of clusters pays its own partial exchange
        const float t = waves * (((units + S - 1) / S) * t_unit + (S > 1 ? t_reduce : 0.f));
        if (best_t < 0.f || t < best_t - 1e-6f) { best_t = t; best = S; }
    }
    return best;
}

int b200::clusters_resident(int S, int ctas_per_sm) {
    if (S < 1) S = 1;
    if (S > 16) S = 16;
    return cluster_table(ctas_per_sm)[S];
}

namespace {

int check_shape(int C, int Wx, int Wy, int K, int M) {
    if (C < 1 || Wx < 1 || Wy < 1 || K < 1 || M < 1) return CONV_E_SHAPE;
    if (K > Wx || K > Wy) return CONV_E_SHAPE;
    const int64_t Ho = Wy - K + 1, Wo = Wx - K + 1;
    if ((int64_t)C * Wx * Wy > INT_MAX) return CONV_E_SHAPE;
    if ((int64_t)M * C * K * K > INT_MAX) return CONV_E_SHAPE;
    if ((int64_t)M * Ho * Wo > INT_MAX) return CONV_E_SHAPE;
    return CONV_OK;
}

bool aligned(const void *p, int a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

int check_ptrs(const void *I, const void *F, const void *O, int in_elem) {
    if (!I || !F || !O) return CONV_E_NULL;
    if (!aligned(I, in_elem) || !aligned(F, in_elem) || !aligned(O, 4)) return CONV_E_ALIGN;
    return CONV_OK;
}

int check_device() {
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return CONV_E_DEVICE; }
    int major = 0, minor = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess) {
        cudaGetLastError();
        return CONV_E_DEVICE;
    }
    return (major == 10 && minor == 0) ? CONV_OK : CONV_E_DEVICE;
}

int launch_status(cudaError_t e) {
    if (e == cudaSuccess) return CONV_OK;
    cudaGetLastError();
    return CONV_E_LAUNCH;
}

int run_multi(const void *I, int C, int Wx, int Wy, const void *F, int K, int M, float *O,
              int precision, cudaStream_t s) {
    if (precision >= CONV_FP32 && precision <= CONV_BF16) {
        const cudaError_t e = launch_multi_c3(I, C, Wx, Wy, F, K, M, O, precision == CONV_BF16, s);
        if (e != cudaErrorNotSupported) return launch_status(e);
        cudaGetLastError();
    }
    switch (precision) {
        case CONV_FP32:
            return launch_status(launch_multi_simt(static_cast<const float *>(I), C, Wx, Wy,
                                                   static_cast<const float *>(F), K, M, O, s));
        case CONV_TF32:
        case CONV_BF16: {
            const bool bf16 = precision == CONV_BF16;
            cudaError_t e = launch_multi_gemm(I, C, Wx, Wy, F, K, M, O, bf16, s);
            if (e == cudaErrorNotSupported) {   // shape / alignment / capture: implicit kernel
                cudaGetLastError();
                e = launch_multi_tc(I, C, Wx, Wy, F, K, M, O, bf16, s);
            }
            return launch_status(e);
        }
        default:
            return CONV_E_PRECISION;
    }
}

// the C = 3 stem layers the channel-summing KS variant takes (per image)
bool c3_layer(int C, int Wx, int Wy, int K, int M) {
    conv_plan tmp;
    return plan_multi_c3(C, Wx, Wy, K, M, &tmp) == 0;
}

// stride sd > 1: FP32 on KM-SIMT, TF32 / BF16 on KM-TC/G
// (explicit strided im2col + one TMA GEMM); each as ONE launch over all N images
int run_strided(const void *I, int N, int C, int Wx, int Wy, const void *F, int K, int M, float *O,
                int precision, int sd, cudaStream_t s) {
    switch (precision) {
        case CONV_FP32:
            return launch_status(launch_multi_simt(static_cast<const float *>(I), C, Wx, Wy,
                                                   static_cast<const float *>(F), K, M, O, s, sd, N));
        case CONV_TF32:
        case CONV_BF16:
            return launch_status(launch_multi_gemm(I, C, Wx, Wy, F, K, M, O, precision == CONV_BF16, s, sd, N));
        default:
            return CONV_E_PRECISION;
    }
}

}  // namespace

extern "C" {

int conv_single_ex(const float *I, int Wx, int Wy, const float *F, int K, int M, float *O,
                   void *stream) {
    CallScope scope;
    int st = check_shape(1, Wx, Wy, K, M);
    if (st) return st;
    if ((st = check_ptrs(I, F, O, 4))) return st;
    if ((st = check_device())) return st;
    return launch_status(launch_single(I, Wx, Wy, F, K, M, O, static_cast<cudaStream_t>(stream)));
}

int conv_single(const float *I, int Wx, int Wy, const float *F, int K, int M, float *O) {
    return conv_single_ex(I, Wx, Wy, F, K, M, O, nullptr);
}

int conv_multi_ex(const void *I, int C, int Wx, int Wy, const void *F, int K, int M, float *O,
                  int precision, void *stream) {
    CallScope scope;
    int st = check_shape(C, Wx, Wy, K, M);
    if (st) return st;
    if (precision < CONV_FP32 || precision > CONV_BF16) return CONV_E_PRECISION;
    if ((st = check_ptrs(I, F, O, precision == CONV_BF16 ? 2 : 4))) return st;
    if ((st = check_device())) return st;
    return run_multi(I, C, Wx, Wy, F, K, M, O, precision, static_cast<cudaStream_t>(stream));
}

int conv_multi(const float *I, int C, int Wx, int Wy, const float *F, int K, int M, float *O) {
    return conv_multi_ex(I, C, Wx, Wy, F, K, M, O, CONV_FP32, nullptr);
}

int conv_multi_batched_ex(const void *I, int N, int C, int Wx, int Wy, const void *F, int K, int M, float *O,
                          int precision, void *stream) {
    CallScope scope;
    if (N < 1) return CONV_E_SHAPE;
    int st = check_shape(C, Wx, Wy, K, M);
    if (st) return st;
    const int64_t Ho = Wy - K + 1, Wo = Wx - K + 1;
    if ((int64_t)N * C * Wx * Wy > INT_MAX || (int64_t)N * M * Ho * Wo > INT_MAX) return CONV_E_SHAPE;
    if (precision < CONV_FP32 || precision > CONV_BF16) return CONV_E_PRECISION;
    const int e = precision == CONV_BF16 ? 2 : 4;
    if ((st = check_ptrs(I, F, O, e))) return st;
    if ((st = check_device())) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (precision == CONV_FP32 && N > 1 && !c3_layer(C, Wx, Wy, K, M)) {
        // strict FP32: ONE KM-SIMT launch whose pixel tiles span all N images
        return launch_status(launch_multi_simt(static_cast<const float *>(I), C, Wx, Wy,
                                               static_cast<const float *>(F), K, M, O, s, 1, N));
    }
    if (precision == CONV_FP32 || N == 1) {
        // N == 1, and the C = 3 stem layers (KS-C3): one call per image
        for (int n = 0; n < N; ++n) {
            st = run_multi(static_cast<const uint8_t *>(I) + (size_t)n * C * Wx * Wy * e, C, Wx, Wy, F, K, M,
                           O + (size_t)n * M * Ho * Wo, precision, s);
            if (st) return st;
        }
        return CONV_OK;
    }
    // TF32 / BF16: ONE launch of the implicit tensor-core kernel over all N images
    return launch_status(launch_multi_tc(I, C, Wx, Wy, F, K, M, O, precision == CONV_BF16, s, N));
}

// ------------------------------------------------------------ host buffers
// Library-owned stream-ordered pool per device with no release threshold: the
// device staging buffers of the host entry points are recycled across calls
// instead of being returned to the driver at every synchronisation.
static cudaMemPool_t host_pool() {
    static cudaMemPool_t pools[64] = {};
    static std::mutex mu;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> lk(mu);
    if (!pools[dev]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t p = nullptr;
        if (cudaMemPoolCreate(&p, &props) != cudaSuccess) { cudaGetLastError(); return nullptr; }
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
        // a block freed on one stream is reused only by that stream: cross-
        // stream reuse would insert a wait on the freeing stream and serialise
        // callers that overlap copies on several streams (*_host_async)
        int no = 0;
        cudaMemPoolSetAttribute(p, cudaMemPoolReuseFollowEventDependencies, &no);
        cudaMemPoolSetAttribute(p, cudaMemPoolReuseAllowOpportunistic, &no);
        cudaMemPoolSetAttribute(p, cudaMemPoolReuseAllowInternalDependencies, &no);
        pools[dev] = p;
    }
    return pools[dev];
}

static cudaError_t pool_alloc(void **ptr, size_t bytes, cudaStream_t s) {
    cudaMemPool_t p = host_pool();
    return p ? cudaMallocFromPoolAsync(ptr, bytes, p, s) : cudaMallocAsync(ptr, bytes, s);
}

static int host_roundtrip(const void *Ih, size_t i_bytes, const void *Fh, size_t f_bytes, float *Oh,
                          size_t o_bytes, cudaStream_t s,
                          int (*body)(const void *, const void *, float *, void *), void *ctx,
                          bool sync = true) {
    void *Id = nullptr, *Fd = nullptr, *Od = nullptr;
    if (pool_alloc(&Id, i_bytes, s) != cudaSuccess || pool_alloc(&Fd, f_bytes, s) != cudaSuccess ||
        pool_alloc(&Od, o_bytes, s) != cudaSuccess) {
        cudaGetLastError();
        if (Id) cudaFreeAsync(Id, s);
        if (Fd) cudaFreeAsync(Fd, s);
        return CONV_E_LAUNCH;
    }
    int st = CONV_OK;
    if (cudaMemcpyAsync(Id, Ih, i_bytes, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(Fd, Fh, f_bytes, cudaMemcpyHostToDevice, s) != cudaSuccess)
        st = CONV_E_LAUNCH;
    if (st == CONV_OK) st = body(Id, Fd, static_cast<float *>(Od), ctx);
    if (st == CONV_OK && cudaMemcpyAsync(Oh, Od, o_bytes, cudaMemcpyDeviceToHost, s) != cudaSuccess)
        st = CONV_E_LAUNCH;
    cudaFreeAsync(Id, s);
    cudaFreeAsync(Fd, s);
    cudaFreeAsync(Od, s);
    if (sync && cudaStreamSynchronize(s) != cudaSuccess && st == CONV_OK) st = CONV_E_LAUNCH;
    cudaGetLastError();
    return st;
}

struct MultiCtx { int C, Wx, Wy, K, M, precision; cudaStream_t s; };
static int multi_body(const void *I, const void *F, float *O, void *c) {
    MultiCtx *m = static_cast<MultiCtx *>(c);
    return run_multi(I, m->C, m->Wx, m->Wy, F, m->K, m->M, O, m->precision, m->s);
}
static int single_body(const void *I, const void *F, float *O, void *c) {
    MultiCtx *m = static_cast<MultiCtx *>(c);
    return launch_status(launch_single(static_cast<const float *>(I), m->Wx, m->Wy,
                                       static_cast<const float *>(F), m->K, m->M, O, m->s));
}

int conv_single_host(const float *I, int Wx, int Wy, const float *F, int K, int M, float *O,
                     void *stream) {
    CallScope scope;
    int st = check_shape(1, Wx, Wy, K, M);
    if (st) return st;
    if ((st = check_ptrs(I, F, O, 4))) return st;
    if ((st = check_device())) return st;
    MultiCtx ctx{1, Wx, Wy, K, M, CONV_FP32, static_cast<cudaStream_t>(stream)};
    const size_t Ho = Wy - K + 1, Wo = Wx - K + 1;
    return host_roundtrip(I, (size_t)Wx * Wy * 4, F, (size_t)M * K * K * 4, O, (size_t)M * Ho * Wo * 4,
                          ctx.s, single_body, &ctx);
}

int conv_multi_host(const void *I, int C, int Wx, int Wy, const void *F, int K, int M, float *O,
                    int precision, void *stream) {
    CallScope scope;
    int st = check_shape(C, Wx, Wy, K, M);
    if (st) return st;
    if (precision < CONV_FP32 || precision > CONV_BF16) return CONV_E_PRECISION;
    const int e = precision == CONV_BF16 ? 2 : 4;
    if ((st = check_ptrs(I, F, O, e))) return st;
    if ((st = check_device())) return st;
    MultiCtx ctx{C, Wx, Wy, K, M, precision, static_cast<cudaStream_t>(stream)};
    const size_t Ho = Wy - K + 1, Wo = Wx - K + 1;
    return host_roundtrip(I, (size_t)C * Wx * Wy * e, F, (size_t)M * C * K * K * e, O,
                          (size_t)M * Ho * Wo * 4, ctx.s, multi_body, &ctx);
}

// Asynchronous variants: identical, minus the final stream synchronisation.
int conv_single_host_async(const float *I, int Wx, int Wy, const float *F, int K, int M, float *O,
                           void *stream) {
    CallScope scope;
    int st = check_shape(1, Wx, Wy, K, M);
    if (st) return st;
    if ((st = check_ptrs(I, F, O, 4))) return st;
    if ((st = check_device())) return st;
    MultiCtx ctx{1, Wx, Wy, K, M, CONV_FP32, static_cast<cudaStream_t>(stream)};
    const size_t Ho = Wy - K + 1, Wo = Wx - K + 1;
    return host_roundtrip(I, (size_t)Wx * Wy * 4, F, (size_t)M * K * K * 4, O, (size_t)M * Ho * Wo * 4,
                          ctx.s, single_body, &ctx, false);
}

int conv_multi_host_async(const void *I, int C, int Wx, int Wy, const void *F, int K, int M, float *O,
                          int precision, void *stream) {
    CallScope scope;
    int st = check_shape(C, Wx, Wy, K, M);
    if (st) return st;
    if (precision < CONV_FP32 || precision > CONV_BF16) return CONV_E_PRECISION;
    const int e = precision == CONV_BF16 ? 2 : 4;
    if ((st = check_ptrs(I, F, O, e))) return st;
    if ((st = check_device())) return st;
    MultiCtx ctx{C, Wx, Wy, K, M, precision, static_cast<cudaStream_t>(stream)};
    const size_t Ho = Wy - K + 1, Wo = Wx - K + 1;
    return host_roundtrip(I, (size_t)C * Wx * Wy * e, F, (size_t)M * C * K * K * e, O,
                          (size_t)M * Ho * Wo * 4, ctx.s, multi_body, &ctx, false);
}

// ------------------------------------------------------------ plans / misc
int conv_plan_single(int Wx, int Wy, int K, int M, conv_plan *out) {
    int st = check_shape(1, Wx, Wy, K, M);
    if (st) return st;
    if (!out) return CONV_E_NULL;
    *out = conv_plan{};
    plan_single(Wx, Wy, K, M, out);
    return CONV_OK;
}

int conv_plan_multi(int C, int Wx, int Wy, int K, int M, int precision, conv_plan *out) {
    int st = check_shape(C, Wx, Wy, K, M);
    if (st) return st;
    if (!out) return CONV_E_NULL;
    *out = conv_plan{};
    if (precision >= CONV_FP32 && precision <= CONV_BF16 && plan_multi_c3(C, Wx, Wy, K, M, out) == 0)
        return CONV_OK;
    switch (precision) {
        case CONV_FP32: plan_multi_simt(C, Wx, Wy, K, M, out); return CONV_OK;
        case CONV_TF32:
        case CONV_BF16: {
            const bool bf16 = precision == CONV_BF16;
            if (env_override("B200CONV_GM", 1) == 0 || plan_multi_gemm(C, Wx, Wy, K, M, bf16, out) != 0)
                plan_multi_tc(C, Wx, Wy, K, M, bf16, nullptr, out);
            return CONV_OK;
        }
        default: return CONV_E_PRECISION;
    }
}

// ------------------------------------------------------------ zero padding
int conv_single_pad_ex(const float *I, int Wx, int Wy, const float *F, int K, int M, int pad, float *O,
                       void *stream) {
    CallScope scope;
    if (pad < 0) return CONV_E_SHAPE;
    if (pad == 0) return conv_single_ex(I, Wx, Wy, F, K, M, O, stream);
    if (Wx < 1 || Wy < 1 || (int64_t)Wx + 2 * pad > INT_MAX / 2 || (int64_t)Wy + 2 * pad > INT_MAX / 2)
        return CONV_E_SHAPE;
    const int Wxp = Wx + 2 * pad, Wyp = Wy + 2 * pad;
    int st = check_shape(1, Wxp, Wyp, K, M);
    if (st) return st;
    if ((st = check_ptrs(I, F, O, 4))) return st;
    if ((st = check_device())) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    void *Ip = padbuf_get((size_t)Wxp * Wyp * 4, s);
    if (!Ip) return CONV_E_LAUNCH;
    if ((st = launch_status(launch_pad(I, 1, Wx, Wy, pad, 4, Ip, s)))) return st;
    return launch_status(launch_single(static_cast<const float *>(Ip), Wxp, Wyp, F, K, M, O, s));
}

int conv_multi_pad_ex(const void *I, int N, int C, int Wx, int Wy, const void *F, int K, int M, int pad, float *O,
                      int precision, void *stream) {
    CallScope scope;
    if (pad < 0 || N < 1) return CONV_E_SHAPE;
    if (pad == 0) return conv_multi_batched_ex(I, N, C, Wx, Wy, F, K, M, O, precision, stream);
    if (Wx < 1 || Wy < 1 || C < 1 || (int64_t)Wx + 2 * pad > INT_MAX / 2 || (int64_t)Wy + 2 * pad > INT_MAX / 2)
        return CONV_E_SHAPE;
    const int Wxp = Wx + 2 * pad, Wyp = Wy + 2 * pad;
    int st = check_shape(C, Wxp, Wyp, K, M);
    if (st) return st;
    if ((int64_t)N * C * Wxp * Wyp > INT_MAX) return CONV_E_SHAPE;
    if (precision < CONV_FP32 || precision > CONV_BF16) return CONV_E_PRECISION;
    const int e = precision == CONV_BF16 ? 2 : 4;
    if ((st = check_ptrs(I, F, O, e))) return st;
    if ((st = check_device())) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (precision != CONV_FP32) {
        // the implicit tensor-core kernel (every TF32 / BF16 batch; single
        // images unless KM-TC/G takes them) reads the padded copy with its row
        // stride rounded up to 16 B: the patch keeps one 2-D TMA box per stage
        // and the offset-table gather (30-wide BF16 rows are 60 B, not a 16-B
        // multiple); the columns past Wx + 2 pad are zeros whose outputs the
        // kernel drops (valid width Wxp)
        const bool bf16 = precision == CONV_BF16;
        const int v = 16 / e, Wps = (Wxp + v - 1) / v * v;
        conv_plan tmp;
        if (Wps != Wxp && !c3_layer(C, Wxp, Wyp, K, M) && (int64_t)N * C * Wps * Wyp <= INT_MAX &&
            (N > 1 || plan_multi_gemm(C, Wxp, Wyp, K, M, bf16, &tmp) != 0)) {
            void *Ip = padbuf_get((size_t)N * C * Wps * Wyp * e, s);
            if (!Ip) return CONV_E_LAUNCH;
            if ((st = launch_status(launch_pad(I, N * C, Wx, Wy, pad, e, Ip, s, Wps)))) return st;
            set_valid_width(Wxp);
            const cudaError_t er = launch_multi_tc(Ip, C, Wps, Wyp, F, K, M, O, bf16, s, N);
            set_valid_width(0);
            return launch_status(er);
        }
    }
    void *Ip = padbuf_get((size_t)N * C * Wxp * Wyp * e, s);
    if (!Ip) return CONV_E_LAUNCH;
    if ((st = launch_status(launch_pad(I, N * C, Wx, Wy, pad, e, Ip, s)))) return st;
    return conv_multi_batched_ex(Ip, N, C, Wxp, Wyp, F, K, M, O, precision, stream);
}

int conv_plan_multi_batched(int N, int C, int Wx, int Wy, int K, int M, int precision, conv_plan *out) {
    if (N < 1) return CONV_E_SHAPE;
    int st = check_shape(C, Wx, Wy, K, M);
    if (st) return st;
    if (!out) return CONV_E_NULL;
    *out = conv_plan{};
    if (precision == CONV_FP32 && N > 1 && !c3_layer(C, Wx, Wy, K, M)) {
        plan_multi_simt(C, Wx, Wy, K, M, out, 1, N);
        return CONV_OK;
    }
    if (precision == CONV_FP32 || N == 1) return conv_plan_multi(C, Wx, Wy, K, M, precision, out);
    if (precision != CONV_TF32 && precision != CONV_BF16) return CONV_E_PRECISION;
    plan_multi_tc(C, Wx, Wy, K, M, precision == CONV_BF16, nullptr, out, N);
    return CONV_OK;
}

int conv_multi_strided_ex(const void *I, int N, int C, int Wx, int Wy, const void *F, int K, int M, int pad,
                          int stride, float *O, int precision, void *stream) {
    CallScope scope;
    if (stride < 1 || pad < 0 || N < 1) return CONV_E_SHAPE;
    if (stride == 1) return conv_multi_pad_ex(I, N, C, Wx, Wy, F, K, M, pad, O, precision, stream);
    if (Wx < 1 || Wy < 1 || C < 1 || (int64_t)Wx + 2 * pad > INT_MAX / 2 || (int64_t)Wy + 2 * pad > INT_MAX / 2)
        return CONV_E_SHAPE;
    const int Wxp = Wx + 2 * pad, Wyp = Wy + 2 * pad;
    int st = check_shape(C, Wxp, Wyp, K, M);
    if (st) return st;
    if ((int64_t)N * C * Wxp * Wyp > INT_MAX) return CONV_E_SHAPE;
    if ((int64_t)N * M * ((Wyp - K) / stride + 1) * ((Wxp - K) / stride + 1) > INT_MAX) return CONV_E_SHAPE;
    if (precision < CONV_FP32 || precision > CONV_BF16) return CONV_E_PRECISION;
    const int e = precision == CONV_BF16 ? 2 : 4;
    if ((st = check_ptrs(I, F, O, e))) return st;
    if ((st = check_device())) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const void *Ic = I;
    if (pad > 0) {
        void *Ip = padbuf_get((size_t)N * C * Wxp * Wyp * e, s);
        if (!Ip) return CONV_E_LAUNCH;
        if ((st = launch_status(launch_pad(I, N * C, Wx, Wy, pad, e, Ip, s)))) return st;
        Ic = Ip;
    }
    return run_strided(Ic, N, C, Wxp, Wyp, F, K, M, O, precision, stride, s);
}

int conv_single_strided_ex(const float *I, int Wx, int Wy, const float *F, int K, int M, int pad, int stride,
                           float *O, void *stream) {
    if (stride == 1) return conv_single_pad_ex(I, Wx, Wy, F, K, M, pad, O, stream);
    return conv_multi_strided_ex(I, 1, 1, Wx, Wy, F, K, M, pad, stride, O, CONV_FP32, stream);
}

int conv_plan_multi_strided(int N, int C, int Wx, int Wy, int K, int M, int pad, int stride, int precision,
                            conv_plan *out) {
    if (!out) return CONV_E_NULL;
    *out = conv_plan{};
    if (N < 1 || stride < 1 || pad < 0 || (int64_t)Wx + 2 * pad > INT_MAX / 2 || (int64_t)Wy + 2 * pad > INT_MAX / 2)
        return CONV_E_SHAPE;
    const int Wxp = Wx + 2 * pad, Wyp = Wy + 2 * pad;
    if (stride == 1) return conv_plan_multi_batched(N, C, Wxp, Wyp, K, M, precision, out);
    int st = check_shape(C, Wxp, Wyp, K, M);
    if (st) return st;
    switch (precision) {
        case CONV_FP32: plan_multi_simt(C, Wxp, Wyp, K, M, out, stride, N); return CONV_OK;
        case CONV_TF32:
        case CONV_BF16:
            return plan_multi_gemm(C, Wxp, Wyp, K, M, precision == CONV_BF16, out, stride, N) ? CONV_E_SHAPE : CONV_OK;
        default: return CONV_E_PRECISION;
    }
}

int conv_multi_allgather_ex(const void *I, int C, int Wx, int Wy, const void *F, int K, int M, int m0, int M_total,
                            float *const *O_peers, int n_peers, float *O_mc, int precision, void *stream) {
    CallScope scope;
    int st = check_shape(C, Wx, Wy, K, M_total);
    if (st) return st;
    if (M < 1 || m0 < 0 || (int64_t)m0 + M > M_total || n_peers < 1 || n_peers > kMaxPeers) return CONV_E_SHAPE;
    if (precision < CONV_FP32 || precision > CONV_BF16) return CONV_E_PRECISION;
    if (!O_peers) return CONV_E_NULL;
    for (int r = 0; r < n_peers; ++r)
        if ((st = check_ptrs(I, F, O_peers[r], precision == CONV_BF16 ? 2 : 4))) return st;
    if (O_mc && !aligned(O_mc, 4)) return CONV_E_ALIGN;
    if ((st = check_device())) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t plane = (int64_t)(Wy - K + 1) * (Wx - K + 1);
    const int64_t off = (int64_t)m0 * plane;
    float *O0 = O_peers[0] + off;
    PeerOut po = {};
    for (int r = 1; r < n_peers; ++r) po.p[r - 1] = O_peers[r] + off;
    po.n = n_peers - 1;
    po.mc = O_mc ? O_mc + off : nullptr;
    struct Reset { ~Reset() { set_peer_out(nullptr); } } reset;
    cudaError_t e;
    if (c3_layer(C, Wx, Wy, K, M)) {            // KS-C3: plain stores, then the peer copy
        set_peer_out(nullptr);
        e = launch_multi_c3(I, C, Wx, Wy, F, K, M, O0, precision == CONV_BF16, s);
        set_peer_out(&po);
        if (e == cudaSuccess) e = launch_peer_copy(O0, M * plane, s);
    } else if (precision == CONV_FP32) {        // split-K reduce stores to every peer (else a copy)
        set_peer_out(&po);
        e = launch_multi_simt(static_cast<const float *>(I), C, Wx, Wy, static_cast<const float *>(F), K, M, O0, s);
    } else {                                    // KM-TC/G epilogue stores to every peer
        const bool bf16 = precision == CONV_BF16;
        set_peer_out(&po);
        e = launch_multi_gemm(I, C, Wx, Wy, F, K, M, O0, bf16, s);
        if (e == cudaErrorNotSupported) {       // implicit kernel: plain stores, then the peer copy
            cudaGetLastError();
            set_peer_out(nullptr);
            e = launch_multi_tc(I, C, Wx, Wy, F, K, M, O0, bf16, s);
            set_peer_out(&po);
            if (e == cudaSuccess) e = launch_peer_copy(O0, M * plane, s);
        }
    }
    return launch_status(e);
}

int conv_latency_model(int profile, double *out) {
    if (!out) return CONV_E_NULL;
    if (profile != 0 && profile != 1) return CONV_E_SHAPE;
    const DeviceProfile d = profile == 1 ? kGtx1080Ti : b200_profile(num_sms());
    const LatencyModel m = latency_model(d);
    out[0] = m.n_fma;
    out[1] = m.volume;
    out[2] = m.threads_per_sm;
    out[3] = m.v_s;
    out[4] = d.bytes_per_clk;
    return CONV_OK;
}

const char *conv_status_string(int status) {
    switch (status) {
        case CONV_OK: return "ok";
        case CONV_E_SHAPE: return "shape error: a dimension < 1, K > min(Wx, Wy), or size overflow";
        case CONV_E_NULL: return "null pointer";
        case CONV_E_ALIGN: return "pointer not aligned to its element size";
        case CONV_E_PRECISION: return "unknown precision";
        case CONV_E_DEVICE: return "current CUDA device is not sm_100 (B200) or no device";
        case CONV_E_LAUNCH: return "kernel launch or CUDA runtime error";
        default: return "unknown status";
    }
}

int conv_version(void) { return (1 << 16) | 6; }   // 1.2: + *_host_async; 1.3: + batched; 1.4: + padding; 1.5: + stride; 1.6: graph-private scratch

}  // extern "C"

// ------------------------------------------------------------ diagnostics
// Max co-resident clusters for a kernel family at a cluster size (tools only).
extern "C" B200CONV_API int conv_diag_nop(void *stream) {
    return launch_status(launch_nop(static_cast<cudaStream_t>(stream)));
}
extern "C" B200CONV_API int conv_diag_stamps(unsigned long long *host) { return tc_read_stamps(host); }
extern "C" B200CONV_API int conv_diag_ks_stamps(unsigned long long *host) { return ks_read_stamps(host); }
extern "C" B200CONV_API int conv_diag_ks_fine(unsigned long long *host) { return ks_read_fine(host); }
extern "C" B200CONV_API int conv_diag_simt_stamps(unsigned long long *host) { return simt_read_stamps(host); }
extern "C" B200CONV_API int conv_diag_tc_cta_stamps(unsigned long long *host) { return tc_read_cta_stamps(host); }
extern "C" B200CONV_API int conv_diag_gm_cta_stamps(unsigned long long *host) { return gm_read_cta_stamps(host); }
extern "C" B200CONV_API int conv_diag_max_clusters(int kernel, int cluster, int smem_bytes) {
    return kernel == 2 ? tc_max_clusters(cluster, smem_bytes) : simt_max_clusters(cluster, smem_bytes);
}
