// tc_probe.cu -- tcgen05 (5th-gen tensor core) TF32 GEMM probe for the
// planned tensor-core blocked Jacobi: one CTA computes
// C[128 x 64] = A[128 x K] * B[64 x K]^T from shared memory (canonical
// K-major, no swizzle), accumulator in TMEM, read back with tcgen05.ld.
// Variants: plain TF32 (1 MMA per K step) and 3xTF32 (hi*hi + hi*lo + lo*hi,
// hi = x with the low 13 mantissa bits cleared), which is what the Gram
// G = P^H P and the update P += P D need for fp32-level accuracy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tc_probe tools/tc_probe.cu
// Prints max error vs fp64 for both variants and the sustained rate of a
// persistent grid (MMA FLOP/s counted per issued MMA).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

constexpr int M = 128, N = 64, K = 64;  // one tile; K steps of 8
constexpr int LBO = 128;                // bytes between K core matrices (8 rows x 16 B)
constexpr int SBO_A = (K / 4) * 128;    // bytes between 8-row groups
constexpr int SBO_B = (K / 4) * 128;

__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version 1 (sm100)
    // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
    return d;
}

// kind::tf32, fp32 accumulate, both K-major, M = 128, N = 64
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);

// element (r, k) of a [rows x K] K-major tile in the canonical no-swizzle layout
__host__ __device__ __forceinline__ int canon(int r, int k, int sbo_bytes) {
    return (r % 8) * 4 + (r / 8) * (sbo_bytes / 4) + (k % 4) + (k / 4) * (LBO / 4);
}

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

template <int NPROD>
__global__ void __launch_bounds__(128) tc_gemm(const float *__restrict__ A, const float *__restrict__ B,
                                               float *__restrict__ C, int iters) {
    extern __shared__ __align__(1024) unsigned char sm[];
    float *Ah = (float *)sm, *Al = Ah + M * K, *Bh = Al + M * K, *Bl = Bh + N * K;
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t mbar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < M * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        const float x = A[i], h = tf32_hi(x);
        Ah[canon(r, k, SBO_A)] = h;
        Al[canon(r, k, SBO_A)] = x - h;
    }
    for (int i = tid; i < N * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        const float x = B[i], h = tf32_hi(x);
        Bh[canon(r, k, SBO_B)] = h;
        Bl[canon(r, k, SBO_B)] = x - h;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_base)), "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy (MMA)
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base;
    if (tid == 0) {
        const uint32_t a[2] = {smem_addr(Ah), smem_addr(Al)}, b[2] = {smem_addr(Bh), smem_addr(Bl)};
        const int pa[3] = {0, 0, 1}, pb[3] = {0, 1, 0};  // hi*hi, hi*lo, lo*hi
        for (int it = 0; it < iters; ++it)
            for (int ks = 0; ks < K / 8; ++ks)
#pragma unroll
                for (int p = 0; p < NPROD; ++p) {
                    const uint64_t da = make_desc(a[pa[p]] + ks * 2 * LBO, LBO, SBO_A);
                    const uint64_t db = make_desc(b[pb[p]] + ks * 2 * LBO, LBO, SBO_B);
                    const uint32_t acc = (it | ks | p) ? 1u : 0u;
                    asm volatile(
                        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, q;\n\t}" ::"r"(tmem),
                        "l"(da), "l"(db), "r"(IDESC), "r"(acc));
                }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(&mbar))
                     : "memory");
    }
    // wait for the MMAs (phase 0)
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(&mbar))
        : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // warp w reads TMEM lanes 32w..32w+31 (rows), 64 fp32 columns
    uint32_t v[64];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll
    for (int c = 0; c < 64; c += 16)
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[c + 0]), "=r"(v[c + 1]), "=r"(v[c + 2]), "=r"(v[c + 3]), "=r"(v[c + 4]), "=r"(v[c + 5]),
              "=r"(v[c + 6]), "=r"(v[c + 7]), "=r"(v[c + 8]), "=r"(v[c + 9]), "=r"(v[c + 10]), "=r"(v[c + 11]),
              "=r"(v[c + 12]), "=r"(v[c + 13]), "=r"(v[c + 14]), "=r"(v[c + 15])
            : "r"(taddr + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int row = warp * 32 + lane;
    float *out = C + (size_t)blockIdx.x * M * N + (size_t)row * N;
#pragma unroll
    for (int c = 0; c < 64; ++c) out[c] = __uint_as_float(v[c]);
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}

int main() {
    std::vector<float> A(M * K), B(N * K);
    srand(7);
    for (auto &x : A) x = (float)rand() / RAND_MAX * 2.f - 1.f;
    for (auto &x : B) x = (float)rand() / RAND_MAX * 2.f - 1.f;
    std::vector<double> ref(M * N, 0.0);
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
            double s = 0;
            for (int k = 0; k < K; ++k) s += (double)A[i * K + k] * (double)B[j * K + k];
            ref[i * N + j] = s;
        }
    float *dA, *dB, *dC;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms;
    cudaMalloc(&dC, (size_t)grid * M * N * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    const size_t smem = (size_t)(2 * M * K + 2 * N * K) * 4;
    cudaFuncSetAttribute(tc_gemm<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(tc_gemm<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int np = 1; np <= 3; np += 2) {
        if (np == 1) tc_gemm<1><<<1, 128, smem>>>(dA, dB, dC, 1);
        else tc_gemm<3><<<1, 128, smem>>>(dA, dB, dC, 1);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("kernel error: %s\n", cudaGetErrorString(e)); return 1; }
        std::vector<float> Cv(M * N);
        cudaMemcpy(Cv.data(), dC, Cv.size() * 4, cudaMemcpyDeviceToHost);
        double err = 0, mx = 0;
        for (int i = 0; i < M * N; ++i) {
            err = fmax(err, fabs(Cv[i] - ref[i]));
            mx = fmax(mx, fabs(ref[i]));
        }
        printf("%dxTF32: max |C - C_fp64| = %.3e (rel to max|C| %.3e), C[0]=%.6f ref %.6f\n", np, err, err / mx,
               Cv[0], ref[0]);
    }
    // sustained rate: every SM runs `iters` x (K/8) x NPROD MMAs of 128x64x8
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4000;
    for (int np = 1; np <= 3; np += 2) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (np == 1) tc_gemm<1><<<grid, 128, smem>>>(dA, dB, dC, iters);
            else tc_gemm<3><<<grid, 128, smem>>>(dA, dB, dC, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double flops = 2.0 * M * N * 8 * (K / 8) * np * (double)iters * grid;
            if (rep) printf("%dxTF32 sustained: %.1f TFLOP/s of MMA work (%.1f TFLOP/s fp32-accurate GEMM)\n", np,
                            flops / ms / 1e9, flops / np / ms / 1e9);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
