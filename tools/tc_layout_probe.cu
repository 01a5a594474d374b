// tc_layout_probe.cu -- unit check of the tcgen05 tf32 operand layouts used by
// the blocked Jacobi: one MMA per case from a 128-row x 64-real-column buffer
// in 128-byte core matrices (offset(row, c) = (row>>3)*2048 + (c>>2)*128 +
// (row&7)*16 + (c&3)*4), compared with a host product.
//   case 0: MN-major Gram, M = N = 64 (cols), K = 8 rows (LBO 2048, SBO 128)
//   case 1: K-major A (M = 128 rows, K = 8 cols, LBO 128, SBO 2048) x
//           K-major B (N = 64, K = 8) from a separate N x K buffer
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tc_layout_probe tools/tc_layout_probe.cu
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t mdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, int amaj, int bmaj) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)amaj << 15) | ((uint32_t)bmaj << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ uint64_t mdesc_sw128(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return mdesc(addr, lbo, sbo) | (2ull << 61);
}
__global__ void __launch_bounds__(128) k(const float *A, const float *B, float *out, int cas, uint32_t lbo, uint32_t sbo) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char *Ab = sm, *Bb = sm + 32768;
    __shared__ uint32_t tb;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int x = tid; x < 128 * 64; x += 128) {
        const int r = x / 64, c = x % 64;
        *reinterpret_cast<float *>(Ab + (r >> 3) * 2048 + (c >> 2) * 128 + (r & 7) * 16 + (c & 3) * 4) = A[x];
    }
    for (int x = tid; x < 64 * 8; x += 128) {  // B: N=64 rows x K=8, K-major canonical (SBO 256: 2 chunks per n-group)
        const int n = x / 8, kk = x % 8;
        *reinterpret_cast<float *>(Bb + (n >> 3) * 256 + (kk >> 2) * 128 + (n & 7) * 16 + (kk & 3) * 4) = B[x];
    }
    if (cas == 5) {  // Bb = SW128 MN-major copy of A rows 0..7 (K) x cols 0..63 (MN): two 1 KB atoms
        for (int x = tid; x < 8 * 64; x += 128) {
            const int kk = x / 64, c = x % 64;
            const int atom = c / 32, ch = ((c % 32) / 4) ^ (kk & 7);
            *reinterpret_cast<float *>(Bb + atom * lbo + kk * 128 + ch * 16 + (c % 4) * 4) = A[kk * 64 + c];
        }
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(&tb)), "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t t = tb;
    if (tid == 0) {
        uint64_t da, db;
        uint32_t id;
        if (cas == 0) {
            da = db = mdesc(sa(Ab), lbo, sbo);
            id = idesc(64, 64, 1, 1);
        } else if (cas == 2) {  // A MN-major (cols x rows), B K-major from Bb (N=64 x K=8)
            da = mdesc(sa(Ab), lbo, sbo);
            db = mdesc(sa(Bb), 128, 256);
            id = idesc(64, 64, 1, 0);
        } else if (cas == 3) {  // M = 128 MN-major A and B
            da = db = mdesc(sa(Ab), lbo, sbo);
            id = idesc(128, 64, 1, 1);
        } else if (cas == 4) {  // A K-major (rows x cols), B MN-major
            da = mdesc(sa(Ab), 128, 2048);
            db = mdesc(sa(Ab), lbo, sbo);
            id = idesc(128, 64, 0, 1);
        } else if (cas == 5) {  // Gram: A MN-major interleave, B MN-major SW128
            da = mdesc(sa(Ab), 2048, 128);
            db = mdesc_sw128(sa(Bb), lbo, sbo);
            id = idesc(64, 64, 1, 1);
        } else {
            da = mdesc(sa(Ab), lbo, sbo);
            db = mdesc(sa(Bb), 128, 256);
            id = idesc(128, 64, 0, 0);
        }
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, q;\n\t}" ::"r"(t),
                     "l"(da), "l"(db), "r"(id), "r"(0u));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)) : "memory");
    }
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}"
                 ::"r"(sa(&bar)), "r"(0) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int c = 0; c < 64; c += 16) {
        uint32_t v[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(t + ((uint32_t)(warp * 32) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int i = 0; i < 16; ++i) out[(warp * 32 + lane) * 64 + c + i] = __uint_as_float(v[i]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(64));
}

// SW128 K-major: offset(row, k) = (k>>5)*ATOM + (row>>3)*1024 + (row&7)*128 + ((((k&31)>>2) ^ (row&7))<<4) + (k&3)*4
__device__ __forceinline__ uint32_t sw_off(int row, int kk, uint32_t atom) {
    return (kk >> 5) * atom + (row >> 3) * 1024 + (row & 7) * 128 + ((((kk & 31) >> 2) ^ (row & 7)) << 4) + (kk & 3) * 4;
}
__global__ void __launch_bounds__(128) ksw(const float *A, const float *B, float *out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char *Ab = sm, *Bb = sm + 32768;  // A: 128 x 64 (2 atoms of 16 KB), B: 64 x 64 (2 atoms of 8 KB)
    __shared__ uint32_t tb;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int x = tid; x < 128 * 64; x += 128) *reinterpret_cast<float *>(Ab + sw_off(x / 64, x % 64, 16384)) = A[x];
    for (int x = tid; x < 64 * 64; x += 128) *reinterpret_cast<float *>(Bb + sw_off(x / 64, x % 64, 8192)) = B[x];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(&tb)), "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t t = tb;
    if (tid == 0) {
        for (int ks = 0; ks < 8; ++ks) {
            const uint32_t ao = (ks >> 2) * 16384 + (ks & 3) * 32, bo = (ks >> 2) * 8192 + (ks & 3) * 32;
            const uint64_t da = mdesc_sw128(sa(Ab) + ao, 16, 1024), db = mdesc_sw128(sa(Bb) + bo, 16, 1024);
            asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, q;\n\t}" ::"r"(t),
                         "l"(da), "l"(db), "r"(idesc(128, 64, 0, 0)), "r"(ks ? 1u : 0u));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)) : "memory");
    }
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}"
                 ::"r"(sa(&bar)), "r"(0) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int c = 0; c < 64; c += 16) {
        uint32_t v[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(t + ((uint32_t)(warp * 32) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int i = 0; i < 16; ++i) out[(warp * 32 + lane) * 64 + c + i] = __uint_as_float(v[i]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(64));
}

int main() {
    std::vector<float> A(128 * 64), B(64 * 8), O(128 * 64);
    for (int i = 0; i < 128 * 64; ++i) A[i] = (float)((i * 37) % 17 - 8) / 8.f;  // exact in tf32
    for (int i = 0; i < 64 * 8; ++i) B[i] = (float)((i * 11) % 13 - 6) / 4.f;
    float *dA, *dB, *dO;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dO, O.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    struct { int cas; uint32_t lbo, sbo; const char *name; } cases[] = {
        {0, 2048, 128, "MN-major Gram LBO=2048 SBO=128"},
        {0, 128, 2048, "MN-major Gram LBO=128 SBO=2048"},
        {1, 128, 2048, "K-major A LBO=128 SBO=2048"},
        {1, 2048, 128, "K-major A LBO=2048 SBO=128"},
        {2, 2048, 128, "A MN-major only LBO=2048 SBO=128"},
        {2, 128, 2048, "A MN-major only LBO=128 SBO=2048"},
        {3, 2048, 128, "M128 MN-major LBO=2048 SBO=128"},
        {4, 2048, 128, "B MN-major only LBO=2048 SBO=128"},
        {4, 128, 2048, "B MN-major only LBO=128 SBO=2048"},
        {5, 1024, 2048, "Gram A inter, B SW128 LBO=1024"},
        {5, 2048, 1024, "Gram A inter, B SW128 LBO=2048 SBO=1024"},
    };
    {   // truncation test: A = 1 + f*2^-10 (f in {0.25, 0.5, 0.75}) -> tf32 trunc = 1, rn = 1 or 1+2^-10
        std::vector<float> A2(128 * 64, 0.f), B2(64 * 8, 0.f);
        const float fr[4] = {0.f, 0.25f, 0.5f, 0.75f};
        for (int m = 0; m < 128; ++m) A2[m * 64 + 0] = 1.f + fr[m % 4] * ldexpf(1.f, -10) + (m / 4 % 2 ? ldexpf(1.f, -20) : 0.f);
        B2[0] = 1.f;  // n = 0, k = 0
        cudaMemcpy(dA, A2.data(), A2.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B2.data(), B2.size() * 4, cudaMemcpyHostToDevice);
        cudaMemset(dO, 0, O.size() * 4);
        k<<<1, 128, 65536>>>(dA, dB, dO, 1, 128, 2048);
        cudaDeviceSynchronize();
        cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
        printf("tf32 operand rounding: A = 1 + f*2^-10 (+2^-20 on odd quads) -> D:\n");
        for (int m = 0; m < 8; ++m) printf("  A=%.10f  D=%.10f  trunc=%.10f\n", A2[m * 64], O[m * 64],
                                           (double)__builtin_bit_cast(float, __builtin_bit_cast(unsigned, A2[m * 64]) & 0xFFFFE000u));
        cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    }
    {   // SW128 K-major, full K = 64 over 8 MMAs
        std::vector<float> B3(64 * 64);
        for (int i = 0; i < 64 * 64; ++i) B3[i] = (float)((i * 29) % 19 - 9) / 8.f;
        float *dB3;
        cudaMalloc(&dB3, B3.size() * 4);
        cudaMemcpy(dB3, B3.data(), B3.size() * 4, cudaMemcpyHostToDevice);
        cudaFuncSetAttribute(ksw, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
        cudaMemset(dO, 0, O.size() * 4);
        ksw<<<1, 128, 65536>>>(dA, dB3, dO);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
        double err = 0, mx = 0;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < 64; ++n) {
                double ref = 0;
                for (int kk = 0; kk < 64; ++kk) ref += (double)A[m * 64 + kk] * B3[n * 64 + kk];
                err = fmax(err, fabs(O[m * 64 + n] - ref)); mx = fmax(mx, fabs(ref));
            }
        printf("SW128 K-major 128x64x64 (8 MMAs): %s max err %.3e (max ref %.3e)\n", cudaGetErrorString(e), err, mx);
    }
    for (auto &cs : cases) {
        cudaMemset(dO, 0, O.size() * 4);
        k<<<1, 128, 65536>>>(dA, dB, dO, cs.cas, cs.lbo, cs.sbo);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s: error %s\n", cs.name, cudaGetErrorString(e)); return 1; }
        cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
        double err = 0, mx = 0, gotmax = 0;
        int bad = 0;
        if (cs.cas == 2) {  // D[i][n] = sum_k A[k][i] B[n][k], M=64 layout
            for (int i = 0; i < 64; ++i)
                for (int n = 0; n < 64; ++n) {
                    double ref = 0;
                    for (int r = 0; r < 8; ++r) ref += (double)A[r * 64 + i] * B[n * 8 + r];
                    const double got = O[(32 * (i / 16) + i % 16) * 64 + n];
                    err = fmax(err, fabs(got - ref)); mx = fmax(mx, fabs(ref)); gotmax = fmax(gotmax, fabs(got));
                    bad += fabs(got - ref) > 1e-5;
                }
        } else if (cs.cas == 0 || cs.cas == 5) {  // G[i][j] = sum_{r<8} A[r][i] A[r][j]; row i in lane 32(i/16) + i%16
            for (int i = 0; i < 64; ++i)
                for (int j = 0; j < 64; ++j) {
                    double ref = 0;
                    for (int r = 0; r < 8; ++r) ref += (double)A[r * 64 + i] * A[r * 64 + j];
                    const double got = O[(32 * (i / 16) + i % 16) * 64 + j];
                    err = fmax(err, fabs(got - ref)); mx = fmax(mx, fabs(ref)); gotmax = fmax(gotmax, fabs(got));
                    bad += fabs(got - ref) > 1e-5;
                }
        } else if (cs.cas != 1) {  // just report magnitude
            for (int i = 0; i < 128 * 64; ++i) gotmax = fmax(gotmax, fabs(O[i]));
        } else {  // D[m][n] = sum_{k<8} A[m][k] B[n][k]
            for (int m = 0; m < 128; ++m)
                for (int n = 0; n < 64; ++n) {
                    double ref = 0;
                    for (int kk = 0; kk < 8; ++kk) ref += (double)A[m * 64 + kk] * B[n * 8 + kk];
                    const double got = O[m * 64 + n];
                    err = fmax(err, fabs(got - ref)); mx = fmax(mx, fabs(ref)); gotmax = fmax(gotmax, fabs(got));
                    bad += fabs(got - ref) > 1e-5;
                }
        }
        printf("%-34s max err %.3e (max ref %.3e, max got %.3e), %d bad\n", cs.name, err, mx, gotmax, bad);
    }
    return 0;
}
