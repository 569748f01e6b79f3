// Dependent-launch floor on B200: a graph of N back-to-back launches of a tiny
// kernel (griddepcontrol.wait / launch_dependents, PDL attribute) — the time
// per launch when the kernel does (a) nothing, (b) one global load + store per
// thread (a minimal dependent read -> write chain).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_empty(float *o) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0 && blockIdx.x == 100000) o[0] = 1.f;
}
__global__ void k_rw(const float *i, float *o) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    o[t] = i[t] * 2.f + 1.f;
}
int main() {
    float *a, *b;
    cudaMalloc(&a, 1 << 24); cudaMalloc(&b, 1 << 24);
    cudaMemset(a, 0, 1 << 24);
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (int pdl = 0; pdl < 2; ++pdl)
    for (int variant = 0; variant < 2; ++variant)
    for (int ctas : {1, 16, 148}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(ctas); cfg.blockDim = dim3(256); cfg.stream = s;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = pdl; cfg.attrs = at; cfg.numAttrs = 1;
        cudaGraph_t g; cudaGraphExec_t ge;
        const int N = 50;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int n = 0; n < N; ++n) {
            if (variant == 0) cudaLaunchKernelEx(&cfg, k_empty, b);
            else cudaLaunchKernelEx(&cfg, k_rw, (n & 1) ? b : a, (n & 1) ? a : b);
        }
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0, s); cudaGraphLaunch(ge, s); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
        }
        printf("pdl %d %-10s ctas %3d: %.2f us per launch\n", pdl, variant ? "read-write" : "empty", ctas, best * 1e3 / N);
    }
    return 0;
}
