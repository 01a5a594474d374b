// Microbenchmark: cluster barrier latency, DSMEM per-thread store bandwidth,
// async bulk shared::cta -> shared::cluster copy latency / bandwidth on B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_bench dsmem_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void expect_tx(uint64_t *b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mwait(uint64_t *b, uint32_t ph) {
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) { uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }
__device__ __forceinline__ void bulk(uint32_t d, uint32_t s, uint32_t n, uint32_t mb) {
    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d), "r"(s), "r"(n), "r"(mb) : "memory");
}

// 1) cluster barrier latency
__global__ void __cluster_dims__(2, 1, 1) k_barrier(int iters, long long *out) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) cg::this_cluster().sync();
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / iters;
}

// 2) bulk ping-pong latency between rank 0 and 1 of a pair cluster
__global__ void __cluster_dims__(2, 1, 1) k_pingpong(int iters, int bytes, long long *out) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *mb = (uint64_t *)sm;
    unsigned char *buf = sm + 128;
    const int rank = cg::this_cluster().block_rank();
    if (threadIdx.x == 0) { mbar_init(mb, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    cg::this_cluster().sync();
    long long t0 = clock64();
    if (threadIdx.x == 0) {
        const uint32_t peer = rank ^ 1;
        for (int i = 0; i < iters; ++i) {
            if (rank == 0) {
                bulk(mapa(su32(buf + 65536), peer), su32(buf), bytes, mapa(su32(mb), peer));
                expect_tx(mb, bytes);
                mwait(mb, i & 1);
            } else {
                expect_tx(mb, bytes);
                mwait(mb, i & 1);
                bulk(mapa(su32(buf + 65536), peer), su32(buf), bytes, mapa(su32(mb), peer));
            }
        }
        asm volatile("cp.async.bulk.commit_group; cp.async.bulk.wait_group 0;" ::: "memory");
    }
    long long t1 = clock64();
    __syncthreads();
    cg::this_cluster().sync();
    if (threadIdx.x == 0 && rank == 0) out[0] = (t1 - t0) / iters;
}

// 3) one-way streaming bandwidth: rank 0 sends `bytes` chunks to rank 1, rank 1 acks with 16 B
template <int C>
__global__ void k_stream(int iters, int bytes, long long *out) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *mb = (uint64_t *)sm;  // [0]: data arrived at receivers, [1]: ack at rank 0
    unsigned char *buf = sm + 128;
    const int rank = cg::this_cluster().block_rank();
    if (threadIdx.x == 0) { mbar_init(&mb[0], 1); mbar_init(&mb[1], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    cg::this_cluster().sync();
    long long t0 = clock64();
    if (threadIdx.x == 0) {
        for (int i = 0; i < iters; ++i) {
            if (rank == 0) {
                for (int d = 1; d < C; ++d)
                    bulk(mapa(su32(buf + 100000), d), su32(buf), bytes, mapa(su32(&mb[0]), d));
                expect_tx(&mb[1], 16 * (C - 1));
                mwait(&mb[1], i & 1);
            } else {
                expect_tx(&mb[0], bytes);
                mwait(&mb[0], i & 1);
                bulk(mapa(su32(buf + 200000), 0), su32(buf), 16, mapa(su32(&mb[1]), 0));
            }
        }
        asm volatile("cp.async.bulk.commit_group; cp.async.bulk.wait_group 0;" ::: "memory");
    }
    long long t1 = clock64();
    __syncthreads();
    cg::this_cluster().sync();
    if (threadIdx.x == 0 && rank == 0) out[0] = (t1 - t0) / iters;
}

// 4) per-thread remote stores: every thread of rank 0 stores 16 B into rank 1, then cluster sync
__global__ void __cluster_dims__(2, 1, 1) k_st_remote(int iters, int bytes, long long *out) {
    extern __shared__ __align__(128) unsigned char sm[];
    float4 *buf = (float4 *)(sm);
    const int rank = cg::this_cluster().block_rank();
    cg::cluster_group cl = cg::this_cluster();
    float4 *remote = cl.map_shared_rank(buf, rank ^ 1);
    const int n16 = bytes / 16;
    cl.sync();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        for (int j = threadIdx.x; j < n16; j += blockDim.x) remote[j] = make_float4(i, j, 0, 0);
        cl.sync();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && rank == 0) out[0] = (t1 - t0) / iters;
}

int main() {
    long long *d, h;
    cudaMalloc(&d, 8);
    k_barrier<<<2, 256>>>(1000, d);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("cluster(2) barrier: %lld cycles\n", h);
    cudaFuncSetAttribute(k_pingpong, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int b : {16, 256, 2048, 16384, 65536}) {
        k_pingpong<<<2, 128, 200 * 1024>>>(200, b, d);
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("bulk ping-pong %6d B: round trip %lld cycles\n", b, h);
    }
    auto run_stream = [&](auto kern, int C, int b) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(C); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 220 * 1024; cfg.attrs = at; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kern, 100, b, d);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("bulk stream C=%2d %6d B to each of %d peers: %lld cycles/iter (%.1f B/cycle out of rank 0) %s\n", C, b, C - 1, h,
               (double)b * (C - 1) / h, e == cudaSuccess ? "" : cudaGetErrorString(e));
    };
    for (int b : {2048, 16384, 65536}) { run_stream(k_stream<2>, 2, b); run_stream(k_stream<8>, 8, b); }
    run_stream(k_stream<16>, 16, 2048);
    cudaFuncSetAttribute(k_st_remote, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int b : {2048, 16384, 65536}) {
        for (int th : {128, 512}) {
            k_st_remote<<<2, th, 200 * 1024>>>(200, b, d);
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            printf("st.shared::cluster %6d B by %d threads + cluster sync: %lld cycles (%.1f B/cycle)\n", b, th, h, (double)b / h);
        }
    }
    return 0;
}
