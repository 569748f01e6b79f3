// dsmem_push.cu — split-K partial exchange inside a cluster of S CTAs: each
// CTA holds a `tile`-byte partial in shared memory and every rank needs its
// 1/S slice of all S partials.  Three ways, timed with clock64 per CTA:
//   mode 0: ld.shared::cluster float4 loads of the S-1 remote slices (pull)
//   mode 1: cp.async.bulk.shared::cluster.shared::cta pushes of each slice to
//           its owner's receive buffer, completing on the owner's mbarrier
//   mode 2: the L2 round trip (bulk store to global, cluster barrier, bulk
//           loads of the slices)
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2212_00404_b200/csrc
//        tools/probes/dsmem_push.cu -o tools/probes/bin/dsmem_push
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace b200;

__device__ __forceinline__ void bulk_s2s(uint32_t dst_cluster, uint32_t src, uint32_t bytes, uint32_t bar_cluster) {
    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst_cluster), "r"(src), "r"(bytes), "r"(bar_cluster) : "memory");
}

__device__ __forceinline__ uint32_t cluster_nctarank_probe() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}

__global__ void __launch_bounds__(256, 1) xchg(int mode, int tile, float *ws, long long *cyc, float *sink) {
    extern __shared__ __align__(128) uint8_t sm[];
    float *P = reinterpret_cast<float *>(sm);                       // own partial [tile]
    float *R = reinterpret_cast<float *>(sm + tile);                // receive [S][slice]
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + 2 * tile);
    const int S = (int)cluster_nctarank_probe();
    const int rank = (int)cluster_ctarank();
    const int slice = tile / S;                                     // bytes
    for (int i = threadIdx.x; i < tile / 4; i += blockDim.x) P[i] = (float)(i + rank);
    if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
    fence_proxy_async_smem();                                       // P -> visible to the bulk copies
    __syncthreads();
    cluster_sync_all();
    const long long t0 = clock64();
    float acc = 0.f;
    if (mode == 0) {
        for (int off = threadIdx.x * 16; off < slice; off += blockDim.x * 16) {
            for (int t = 0; t < S; ++t) {
                const float4 v = ld_dsmem_f32x4(mapa_shared(smem_u32(P) + rank * slice + off, (uint32_t)t));
                acc += v.x + v.y + v.z + v.w;
            }
        }
        cluster_sync_all();
    } else if (mode == 1) {
        if (threadIdx.x == 0) mbar_arrive_expect_tx(bar, (uint32_t)(slice * S));
        cluster_sync_all();                                         // every receive barrier armed
        if (threadIdx.x < S) {
            const int t = threadIdx.x;                              // push my slice t to rank t
            bulk_s2s(mapa_shared(smem_u32(R) + rank * slice, (uint32_t)t), smem_u32(P) + t * slice,
                     (uint32_t)slice, mapa_shared(smem_u32(bar), (uint32_t)t));
        }
        mbar_wait(bar, 0);
        for (int off = threadIdx.x * 16; off < slice; off += blockDim.x * 16)
            for (int t = 0; t < S; ++t) {
                const float4 v = *reinterpret_cast<const float4 *>(reinterpret_cast<uint8_t *>(R) + t * slice + off);
                acc += v.x + v.y + v.z + v.w;
            }
        cluster_sync_all();                                         // sources stay alive until consumed
    } else {
        float *wme = ws + (size_t)blockIdx.x * (tile / 4);
        if (threadIdx.x == 0) {
            fence_proxy_async_smem();
            bulk_store(wme, P, (uint32_t)tile);
            bulk_commit();
            bulk_wait<0>();
            fence_proxy_async_global();
        }
        cluster_sync_all();
        if (threadIdx.x == 0) {
            mbar_arrive_expect_tx(bar, (uint32_t)(slice * S));
            const int base = blockIdx.x - rank;
            for (int t = 0; t < S; ++t)
                bulk_load(reinterpret_cast<uint8_t *>(R) + t * slice,
                          reinterpret_cast<const uint8_t *>(ws + (size_t)(base + t) * (tile / 4)) + rank * slice,
                          (uint32_t)slice, bar);
        }
        mbar_wait(bar, 0);
        for (int off = threadIdx.x * 16; off < slice; off += blockDim.x * 16)
            for (int t = 0; t < S; ++t) {
                const float4 v = *reinterpret_cast<const float4 *>(reinterpret_cast<uint8_t *>(R) + t * slice + off);
                acc += v.x + v.y + v.z + v.w;
            }
    }
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (acc == 1234.5f) sink[0] = acc;
}

int main() {
    float *ws, *sink;
    long long *cyc;
    cudaMalloc(&ws, 256 << 20);
    cudaMalloc(&sink, 64);
    cudaMalloc(&cyc, 4096 * 8);
    cudaFuncSetAttribute(xchg, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(xchg, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int S : {4, 9}) {
        for (int tile : {65536, 73728, 98304}) {
            if (tile % (S * 16)) continue;
            for (int mode = 0; mode < 3; ++mode) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(S * (S == 4 ? 32 : 12));
                cfg.blockDim = dim3(256);
                cfg.dynamicSmemBytes = 2 * tile + 64;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = S; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
                cfg.attrs = at; cfg.numAttrs = 1;
                long long best = 1LL << 60;
                for (int r = 0; r < 5; ++r) {
                    cudaLaunchKernelEx(&cfg, xchg, mode, tile, ws, cyc, sink);
                    cudaDeviceSynchronize();
                    long long h[4096];
                    cudaMemcpy(h, cyc, cfg.gridDim.x * 8, cudaMemcpyDeviceToHost);
                    long long mx = 0;
                    for (unsigned i = 0; i < cfg.gridDim.x; ++i) mx = h[i] > mx ? h[i] : mx;
                    best = mx < best ? mx : best;
                }
                printf("S %d tile %6d B  mode %d (%s): %7lld clk max over CTAs  %s\n", S, tile, mode,
                       mode == 0 ? "DSMEM pull" : mode == 1 ? "DSMEM bulk push" : "L2 round trip", best,
                       cudaGetErrorString(cudaGetLastError()));
            }
        }
    }
    return 0;
}
