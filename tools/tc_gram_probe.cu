// tc_gram_probe.cu -- the Gram G = P^H P of a panel pair (X rows 256, 2w = 32
// complex columns) on tcgen05, from the panel kernel's shared-memory layout
// (column-major, interleaved complex, column stride LD): staged 64 rows at a
// time into canonical K-major hi/lo operands ([Re P | Im P]^T, 64 x 64 real
// per stage = 4 x 16 KB, the size of the panel kernel's spare buffer), 3xTF32
// M = 64 / N = 64 MMAs, the four real blocks combined into G_re / G_im.
// Compared with an fp64 Gram, and timed (clock64 per CTA) against the
// CUDA-core gram_phase cost measured in the Gram variant (~64k cycles per
// super-round).  Groundwork for the tensor-core blocked Jacobi.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tc_gram_probe tools/tc_gram_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

constexpr int ROWS = 256, NCOL = 32, LD = 520, KS = 64;  // rows per stage
constexpr int LBO = 128, SBO = (KS / 4) * 128;
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(64 >> 4) << 24);

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
    return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)(LBO >> 4) << 16) | ((uint64_t)(SBO >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ int canon(int r, int k) { return (r & 7) * 4 + (r >> 3) * (SBO / 4) + (k & 3) + (k >> 2) * (LBO / 4); }

__global__ void __launch_bounds__(128) gram(const float2 *P, float *D, long long *cyc, int reps) {
    extern __shared__ __align__(1024) unsigned char sm[];
    float2 *pan = reinterpret_cast<float2 *>(sm);                       // NCOL x LD complex (the panel pair)
    float *Oh = reinterpret_cast<float *>(sm + NCOL * LD * 8);          // 64 x KS hi
    float *Ol = Oh + 64 * KS;                                           // 64 x KS lo
    __shared__ uint32_t tb;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const float2 *src = P + (size_t)blockIdx.x * NCOL * LD;
    for (int i = tid; i < NCOL * LD; i += blockDim.x) pan[i] = src[i];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(&tb)), "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t t = tb;
    uint32_t phase = 0;
    const long long c0 = clock64();
    for (int rep = 0; rep < reps; ++rep)
        for (int st = 0; st < ROWS / KS; ++st) {
            // stage rows st*KS.. : operand row m < 32 -> Re col m, m >= 32 -> Im col m - 32;
            // a thread converts 4 consecutive rows of one column (one 16-byte chunk)
            for (int it = tid; it < NCOL * (KS / 4); it += blockDim.x) {
                const int c = it % NCOL, k4 = it / NCOL;
                const float2 *col = pan + (size_t)c * LD + st * KS + 4 * k4;
                float re[4], im[4], h, l;
                float4 hr, lr, hi, li;
#pragma unroll
                for (int j = 0; j < 4; ++j) { re[j] = col[j].x; im[j] = col[j].y; }
                float *hp = &hr.x, *lp = &lr.x, *hq = &hi.x, *lq = &li.x;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    h = __uint_as_float(__float_as_uint(re[j]) & 0xFFFFE000u); l = re[j] - h; hp[j] = h; lp[j] = l;
                    h = __uint_as_float(__float_as_uint(im[j]) & 0xFFFFE000u); l = im[j] - h; hq[j] = h; lq[j] = l;
                }
                *reinterpret_cast<float4 *>(Oh + canon(c, 4 * k4)) = hr;
                *reinterpret_cast<float4 *>(Ol + canon(c, 4 * k4)) = lr;
                *reinterpret_cast<float4 *>(Oh + canon(32 + c, 4 * k4)) = hi;
                *reinterpret_cast<float4 *>(Ol + canon(32 + c, 4 * k4)) = li;
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (tid == 0) {
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t h = sa(Oh), l = sa(Ol);
#pragma unroll
                for (int ks = 0; ks < KS / 8; ++ks)
#pragma unroll
                    for (int p = 0; p < 3; ++p) {
                        const uint64_t da = desc((p == 2 ? l : h) + ks * 2 * LBO), db = desc((p == 1 ? l : h) + ks * 2 * LBO);
                        const uint32_t acc = (st | ks | p) ? 1u : 0u;
                        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, q;\n\t}" ::"r"(t),
                                     "l"(da), "l"(db), "r"(IDESC), "r"(acc));
                    }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)) : "memory");
            }
            asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}"
                         ::"r"(sa(&bar)), "r"(phase) : "memory");
            phase ^= 1;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
    const long long c1 = clock64();
    if (tid == 0) cyc[blockIdx.x] = (c1 - c0) / reps;
    // D rows: warp w lanes 0..15 hold rows 16w + lane (M = 64 layout); the
    // .sync.aligned load is warp-wide, only the lower half-warp stores
    for (int c = 0; c < 64; c += 16) {
        uint32_t v[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(t + ((uint32_t)(warp * 32) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (lane < 16)
            for (int i = 0; i < 16; ++i) D[(size_t)blockIdx.x * 64 * 64 + (16 * warp + lane) * 64 + c + i] = __uint_as_float(v[i]);
    }
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(64));
}

int main(int argc, char **argv) {
    const int B = argc > 1 ? atoi(argv[1]) : 148, reps = argc > 2 ? atoi(argv[2]) : 20;
    std::vector<float2> P((size_t)B * NCOL * LD);
    srand(11);
    for (auto &z : P) z = make_float2((float)rand() / RAND_MAX - 0.5f, (float)rand() / RAND_MAX - 0.5f);
    float2 *dP; float *dD; long long *dc;
    cudaMalloc(&dP, P.size() * 8); cudaMalloc(&dD, (size_t)B * 64 * 64 * 4); cudaMalloc(&dc, B * 8);
    cudaMemcpy(dP, P.data(), P.size() * 8, cudaMemcpyHostToDevice);
    const size_t smem = NCOL * LD * 8 + 2 * 64 * KS * 4;
    cudaFuncSetAttribute(gram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    gram<<<B, 128, smem>>>(dP, dD, dc, 1);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<float> D((size_t)B * 64 * 64);
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double err = 0, mx = 0;
    for (int b = 0; b < B; b += 7) {
        const float2 *p = P.data() + (size_t)b * NCOL * LD;
        const float *d = D.data() + (size_t)b * 64 * 64;
        for (int i = 0; i < NCOL; ++i)
            for (int j = 0; j < NCOL; ++j) {
                double re = 0, im = 0;
                for (int r = 0; r < ROWS; ++r) {
                    const float2 x = p[(size_t)i * LD + r], y = p[(size_t)j * LD + r];
                    re += (double)x.x * y.x + (double)x.y * y.y;
                    im += (double)x.x * y.y - (double)x.y * y.x;
                }
                const double gre = (double)d[i * 64 + j] + d[(32 + i) * 64 + 32 + j];
                const double gim = (double)d[i * 64 + 32 + j] - d[(32 + i) * 64 + j];
                err = fmax(err, hypot(gre - re, gim - im));
                mx = fmax(mx, hypot(re, im));
            }
    }
    gram<<<B, 128, smem>>>(dP, dD, dc, reps);
    cudaDeviceSynchronize();
    std::vector<long long> cyc(B);
    cudaMemcpy(cyc.data(), dc, B * 8, cudaMemcpyDeviceToHost);
    double s = 0;
    for (auto c : cyc) s += c;
    printf("tcgen05 3xTF32 Gram of a 256 x 32 complex panel pair (%d CTAs): max |G - G_fp64| / max|G| = %.2e, "
           "%.0f cycles per Gram (staging + 96 MMAs)\n", B, err / mx, s / B);
    return 0;
}
