// tc_rate_probe.cu -- issue-rate of small tcgen05 kind::tf32 MMAs (the shapes
// of the blocked Jacobi): cycles for 96 MMAs M x N x 8 from SW128 K-major
// operands, into one accumulator (dependent chain) or round-robin over 4.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -o tools/tc_rate_probe tools/tc_rate_probe.cu
#include <cstdio>
#include "../paper_2506_05617_b200/csrc/cs_tcb.cuh"
using namespace cs;
using namespace cs::tcb;
__global__ void __launch_bounds__(128, 1) k(long long *out, int M, int nacc, int N, int cnt, int f16, int nw) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tb;
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x; i < 65536 / 4; i += 128) reinterpret_cast<float *>(sm)[i] = 1e-3f * (i % 7);
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tb)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) { mbar_init(&bar, nw); fence_mbar_init(); }
    fence_proxy_async_smem();
    __syncthreads();
    tc_after_sync();
    const uint32_t t = tb;
    const uint32_t id = f16 ? ((1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24)) : idesc_tf32(M, N);
    uint32_t ph = 0;
    long long best = 1LL << 60;
    for (int rep = 0; rep < 5; ++rep) {
        __syncthreads();
        const long long c0 = clock64();
        const int w = threadIdx.x >> 5;
        if (w < nw) {
            if ((threadIdx.x & 31) == 0)
            for (int i = 0; i < cnt / nw; ++i) {
                const int a = nw > 1 ? w : i % nacc;
                const uint64_t da = desc_sw128(smem_u32(sm) + (i & 3) * 32), db = desc_sw128(smem_u32(sm) + 32768 + (i & 3) * 32);
                if (f16)
                    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, q;\n\t}" ::"r"(t + 64 * a),
                                 "l"(da), "l"(db), "r"(id), "r"(i >= nacc ? 1u : 0u));
                else
                    mma_tf32(t + 64 * a, da, db, id, i >= nacc ? 1u : 0u);
            }
            if ((threadIdx.x & 31) == 0) mma_commit(&bar);
            __syncwarp();
        }
        mbar_wait(&bar, ph);
        ph ^= 1;
        const long long c1 = clock64();
        if (c1 - c0 < best) best = c1 - c0;
    }
    if (threadIdx.x == 0) out[blockIdx.x] = best;
    tc_before_sync();
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(512));
}
int main() {
    long long *d, h;
    cudaMalloc(&d, 8 * 148);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    int cases[][6] = {{128, 1, 64, 96, 0, 1}, {128, 1, 64, 96, 0, 2}, {128, 1, 64, 96, 0, 4},
                      {64, 1, 64, 96, 0, 1}, {64, 1, 64, 96, 0, 4}, {128, 1, 256, 96, 0, 1}, {128, 1, 256, 96, 0, 2},
                      // latency of the Jacobi's small batches: 1 and 8 MMAs issue -> commit -> mbarrier
                      {128, 1, 64, 1, 0, 1}, {128, 1, 64, 8, 0, 1}, {128, 1, 128, 8, 0, 1}, {128, 1, 128, 32, 0, 1},
                      {128, 1, 128, 96, 0, 1},
                      // one issuing warp, independent accumulators round-robin
                      {128, 2, 64, 96, 0, 1}, {128, 4, 64, 96, 0, 1}, {128, 4, 128, 96, 0, 1}, {128, 4, 64, 8, 0, 1},
                      {128, 8, 64, 96, 0, 1}, {128, 4, 64, 32, 0, 1}};
    for (auto &c : cases) {
        k<<<148, 128, 65536>>>(d, c[0], c[1], c[2], c[3], c[4], c[5]);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        const double macs = (double)c[3] * c[0] * c[2] * (c[4] ? 16 : 8);
        printf("%d issuing warps: %s M=%d N=%d x%d: %lld cycles, %.0f cyc/instr (%.0f MAC/clk/SM) %s\n", c[5], c[4] ? "bf16" : "tf32", c[0], c[2], c[3], h,
               (double)h / c[3], macs / h, cudaGetErrorString(e));
    }
    return 0;
}
