// k1_tune.cu -- standalone timing of K1 (symbol assembly) variants at cfg5
// shape (5x5, c=256, 256x256 half grid, fp32).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/k1_tune tools/k1_tune.cu
// Prints ms and GB/s (algorithmic bytes F_u*c*c*8) per variant, best of 10.
#include <cstdio>
#include <vector>

#include "../paper_2506_05617_b200/csrc/cs_common.cuh"

using namespace cs;

__device__ __forceinline__ long long imod2(long long a, long long n) {
    long long r = a % n;
    return r < 0 ? r + n : r;
}
__device__ __forceinline__ double2 uph(long long e, long long n) {
    double s, c;
    sincospi(2.0 * (double)imod2(e, n) / (double)n, &s, &c);
    return make_double2(c, s);
}

// V: store kind 0 = plain, 1 = st.global.cs, 2 = st.global.L1::no_allocate
template <int EPT, int KH, int JC, int NT, int ST>
__global__ void __launch_bounds__(NT) k1v(const float *__restrict__ W, int co, int ci, int kw, int n,
                                           int m, float2 *__restrict__ out) {
    __shared__ double2 rowph[16];
    __shared__ float2 colph[JC][KH];
    const HalfGrid hg(n, m);
    const int i = blockIdx.y;
    const long long base = hg.row_start(i);
    const int rlen = hg.row_len(i);
    const int j0 = blockIdx.z * JC;
    const int jn = min(JC, rlen - j0);
    if (jn <= 0) return;
    const int t = threadIdx.x;
    if (t < kw) rowph[t] = uph((long long)i * (t - kw / 2), n);
    for (int x = t; x < JC * KH; x += NT) {
        const int jj = x / KH, p = x % KH;
        const double2 z = uph((long long)(j0 + jj) * (p - KH / 2), m);
        colph[jj][p] = make_float2((float)z.x, (float)z.y);
    }
    __syncthreads();
    const long long nel = (long long)co * ci;
    const long long e0 = ((long long)blockIdx.x * NT + t) * EPT;
    if (e0 >= nel) return;
    float2 G[EPT][KH];
#pragma unroll
    for (int e = 0; e < EPT; ++e)
#pragma unroll
        for (int p = 0; p < KH; ++p) {
            double gr = 0.0, gi = 0.0;
            const float *w = W + (e0 + e) * (long long)(KH * kw) + p * kw;
            for (int q = 0; q < kw; ++q) {
                const double wv = (double)w[q];
                gr += wv * rowph[q].x;
                gi += wv * rowph[q].y;
            }
            G[e][p] = make_float2((float)gr, (float)gi);
        }
    for (int jj = 0; jj < jn; ++jj) {
        float2 v[EPT];
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
            float ar = 0, ai = 0;
#pragma unroll
            for (int p = 0; p < KH; ++p) {
                const float2 ph = colph[jj][p];
                ar += ph.x * G[e][p].x - ph.y * G[e][p].y;
                ai += ph.x * G[e][p].y + ph.y * G[e][p].x;
            }
            v[e] = make_float2(ar, ai);
        }
        float2 *dst = out + (base + j0 + jj) * nel + e0;
#pragma unroll
        for (int e = 0; e < EPT; e += 2) {
            float4 q = make_float4(v[e].x, v[e].y, v[e + 1].x, v[e + 1].y);
            float4 *d = reinterpret_cast<float4 *>(dst + e);
            if (ST == 0) *d = q;
            else if (ST == 1) __stcs(d, q);
            else asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(d), "f"(q.x), "f"(q.y), "f"(q.z), "f"(q.w) : "memory");
        }
    }
}

// interleaved-warp variant: a warp's 32 lanes x EPT entries are consecutive,
// but EPT=4 lanes store as two float4 at lane*16 and 512+lane*16 (fully
// coalesced 1 KB per warp per frequency)
template <int KH, int JC, int NT>
__global__ void __launch_bounds__(NT) k1w(const float *__restrict__ W, int co, int ci, int kw, int n,
                                          int m, float2 *__restrict__ out) {
    __shared__ double2 rowph[16];
    __shared__ float2 colph[JC][KH];
    const HalfGrid hg(n, m);
    const int i = blockIdx.y;
    const long long base = hg.row_start(i);
    const int rlen = hg.row_len(i);
    const int j0 = blockIdx.z * JC;
    const int jn = min(JC, rlen - j0);
    if (jn <= 0) return;
    const int t = threadIdx.x;
    if (t < kw) rowph[t] = uph((long long)i * (t - kw / 2), n);
    for (int x = t; x < JC * KH; x += NT) {
        const int jj = x / KH, p = x % KH;
        const double2 z = uph((long long)(j0 + jj) * (p - KH / 2), m);
        colph[jj][p] = make_float2((float)z.x, (float)z.y);
    }
    __syncthreads();
    const long long nel = (long long)co * ci;
    const int lane = t & 31, warp = t >> 5;
    const long long wbase = ((long long)blockIdx.x * (NT / 32) + warp) * 128;  // 128 entries per warp
    if (wbase >= nel) return;
    long long ee[4] = {wbase + 2 * lane, wbase + 2 * lane + 1, wbase + 64 + 2 * lane, wbase + 65 + 2 * lane};
    float2 G[4][KH];
#pragma unroll
    for (int e = 0; e < 4; ++e)
#pragma unroll
        for (int p = 0; p < KH; ++p) {
            double gr = 0.0, gi = 0.0;
            const float *w = W + ee[e] * (long long)(KH * kw) + p * kw;
            for (int q = 0; q < kw; ++q) {
                const double wv = (double)w[q];
                gr += wv * rowph[q].x;
                gi += wv * rowph[q].y;
            }
            G[e][p] = make_float2((float)gr, (float)gi);
        }
    for (int jj = 0; jj < jn; ++jj) {
        float2 v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            float ar = 0, ai = 0;
#pragma unroll
            for (int p = 0; p < KH; ++p) {
                const float2 ph = colph[jj][p];
                ar += ph.x * G[e][p].x - ph.y * G[e][p].y;
                ai += ph.x * G[e][p].y + ph.y * G[e][p].x;
            }
            v[e] = make_float2(ar, ai);
        }
        float2 *dst = out + (base + j0 + jj) * nel;
        __stcs(reinterpret_cast<float4 *>(dst + ee[0]), make_float4(v[0].x, v[0].y, v[1].x, v[1].y));
        __stcs(reinterpret_cast<float4 *>(dst + ee[2]), make_float4(v[2].x, v[2].y, v[3].x, v[3].y));
    }
}

int main() {
    const int co = 256, ci = 256, kh = 5, kw = 5, n = 256, m = 256;
    const HalfGrid hg(n, m);
    const long long nel = (long long)co * ci, Fu = hg.count;
    const double bytes = (double)Fu * nel * 8 + (double)nel * kh * kw * 4;
    float *W;
    float2 *out;
    cudaMalloc(&W, nel * kh * kw * 4);
    cudaMemset(W, 0, nel * kh * kw * 4);
    cudaMalloc(&out, Fu * nel * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char *name, auto launch) {
        float best = 1e9;
        for (int r = 0; r < 12; ++r) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r >= 2 && ms < best) best = ms;
        }
        cudaError_t e = cudaGetLastError();
        printf("%-40s %8.3f ms  %7.1f GB/s  %s\n", name, best, bytes / best / 1e6, cudaGetErrorString(e));
    };
    const int rows = hg.rows();
#define V(EPT, JC, NT, ST)                                                                          \
    run("ept" #EPT " jc" #JC " nt" #NT " st" #ST, [&] {                                            \
        dim3 g((unsigned)(nel / (NT * EPT)), rows, (m + JC - 1) / JC);                              \
        k1v<EPT, 5, JC, NT, ST><<<g, NT>>>(W, co, ci, kw, n, m, out);                             \
    });
    V(2, 64, 256, 0)
    V(2, 64, 256, 1)
    V(2, 64, 256, 2)
    V(2, 128, 256, 1)
    V(2, 256, 256, 1)
    V(2, 32, 256, 1)
    V(4, 64, 256, 1)
    V(4, 128, 128, 1)
    V(2, 64, 512, 1)
    V(2, 128, 128, 1)
    run("warp1KB jc64 nt256", [&] {
        dim3 g((unsigned)(nel / (256 * 4)), rows, (m + 63) / 64);
        k1w<5, 64, 256><<<g, 256>>>(W, co, ci, kw, n, m, out);
    });
    run("warp1KB jc128 nt256", [&] {
        dim3 g((unsigned)(nel / (256 * 4)), rows, (m + 127) / 128);
        k1w<5, 128, 256><<<g, 256>>>(W, co, ci, kw, n, m, out);
    });
    run("memset (write-only peak)", [&] { cudaMemsetAsync(out, 1, Fu * nel * 8); });
    return 0;
}
