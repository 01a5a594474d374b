// tmem_m64_probe.cu -- where does an M = 64 tcgen05.mma (cta_group::1) put
// its accumulator rows in TMEM?  D = A B^T with A[r][0] = r + 1, B[n][0] = 1
// (other K entries 0), so D[r][n] = r + 1; every (lane, column) of the 128 x
// 64 TMEM window is read back and the row found there printed per lane.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tmem_m64_probe tools/tmem_m64_probe.cu
#include <cstdint>
#include <cstdio>

constexpr int M = 64, N = 64, K = 8, LBO = 128, SBO = (K / 4) * 128;

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
    return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)(LBO >> 4) << 16) | ((uint64_t)(SBO >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ int canon(int r, int k) { return (r % 8) * 4 + (r / 8) * (SBO / 4) + (k % 4) + (k / 4) * (LBO / 4); }

__global__ void probe(float *out) {
    __shared__ __align__(1024) float A[128 * K], B[N * K];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 128 * K; i += blockDim.x) A[i] = 0.f;
    for (int i = tid; i < N * K; i += blockDim.x) B[i] = 0.f;
    __syncthreads();
    if (tid < M) A[canon(tid, 0)] = (float)(tid + 1);
    if (tid < N) B[canon(tid, 0)] = 1.f;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(&tbase)), "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t t = tbase;
    // zero the window first (uninitialised TMEM would confuse the map): store 0s
    {
        uint32_t z[16] = {};
        for (int c = 0; c < 64; c += 16)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                         ::"r"(t + ((uint32_t)(warp * 32) << 16) + c), "r"(z[0]), "r"(z[1]), "r"(z[2]), "r"(z[3]), "r"(z[4]), "r"(z[5]),
                         "r"(z[6]), "r"(z[7]), "r"(z[8]), "r"(z[9]), "r"(z[10]), "r"(z[11]), "r"(z[12]), "r"(z[13]), "r"(z[14]), "r"(z[15]));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid == 0) {
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, 0, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, q;\n\t}" ::"r"(t),
                     "l"(desc(sa(A))), "l"(desc(sa(B))), "r"(idesc));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)) : "memory");
    }
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" ::"r"(sa(&bar)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t v[16];
    for (int c = 0; c < 64; c += 16) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(t + ((uint32_t)(warp * 32) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int i = 0; i < 16; ++i) out[(warp * 32 + lane) * 64 + c + i] = __uint_as_float(v[i]);
    }
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(64));
}

int main() {
    float *d, h[128 * 64];
    cudaMalloc(&d, sizeof(h));
    probe<<<1, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    // per lane: the row value in columns 0 and 32 (and whether all 64 columns agree)
    for (int l = 0; l < 128; ++l) {
        int agree = 1;
        for (int c = 1; c < 64; ++c) agree &= h[l * 64 + c] == h[l * 64];
        printf("lane %3d: col0 %5.0f col32 %5.0f col63 %5.0f %s\n", l, h[l * 64], h[l * 64 + 32], h[l * 64 + 63],
               agree ? "" : "(columns differ)");
    }
}
