// cayley_probe.cu -- cs_tcb.cu's cross-pair Cayley map (cayley_cross) on random
// B blocks, one CTA of 512 threads; prints max |D - D_ref| against a host
// solve of 2 (I - K)^-1 K in double.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I paper_2506_05617_b200/csrc -o tools/cayley_probe tools/cayley_probe.cu -lcufft
#include <complex>
#include <cstdio>
#include <random>
#include <vector>
#include "../paper_2506_05617_b200/csrc/cs_tcb.cu"
namespace cs {
int cuda_status(cudaError_t, const char *) { return 1; }
int fail(int s, const std::string &) { return s; }
}
using namespace cs::tcb;
__global__ void k(const float2 *Bin, float2 *Dout) {
    __shared__ float2 Bm[W * (W + 1)], g0[W * LDJ], g1[W * LDJ], D[N2 * LDG];
    for (int x = threadIdx.x; x < W * (W + 1); x += blockDim.x) Bm[x] = make_float2(0.f, 0.f);
    __syncthreads();
    if (threadIdx.x < W * W) Bm[(threadIdx.x / W) * (W + 1) + threadIdx.x % W] = Bin[threadIdx.x];
    __syncthreads();
    cayley_cross(Bm, g0, g1, D);
    for (int x = threadIdx.x; x < N2 * N2; x += blockDim.x) Dout[x] = D[(x / N2) * LDG + x % N2];
}
typedef std::complex<double> cd;
int main() {
    std::mt19937 rng(3);
    std::normal_distribution<double> nd(0.0, 0.2);
    std::vector<float2> hB(W * W), hD(N2 * N2);
    for (auto &v : hB) v = make_float2((float)nd(rng), (float)nd(rng));
    float2 *dB, *dD;
    cudaMalloc(&dB, sizeof(float2) * W * W);
    cudaMalloc(&dD, sizeof(float2) * N2 * N2);
    cudaMemcpy(dB, hB.data(), sizeof(float2) * W * W, cudaMemcpyHostToDevice);
    k<<<1, 512>>>(dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hD.data(), dD, sizeof(float2) * N2 * N2, cudaMemcpyDeviceToHost);
    // host: M = [I - K | 2K], Gauss-Jordan in double
    std::vector<cd> M(32 * 64, 0.0);
    for (int i = 0; i < 32; ++i) M[i * 64 + i] = 1.0;
    for (int i = 0; i < W; ++i)
        for (int j = 0; j < W; ++j) {
            cd b(hB[i * W + j].x, hB[i * W + j].y);
            M[i * 64 + W + j] -= b;            // I - K, K_ab = B
            M[(W + j) * 64 + i] += std::conj(b);  // K_ba = -B^H
            M[i * 64 + 32 + W + j] += 2.0 * b;
            M[(W + j) * 64 + 32 + i] -= 2.0 * std::conj(b);
        }
    for (int kk = 0; kk < 32; ++kk) {
        cd p = M[kk * 64 + kk];
        for (int j = 0; j < 64; ++j) M[kk * 64 + j] /= p;
        for (int i = 0; i < 32; ++i)
            if (i != kk) {
                cd f = M[i * 64 + kk];
                for (int j = 0; j < 64; ++j) M[i * 64 + j] -= f * M[kk * 64 + j];
            }
    }
    double err = 0, uerr = 0;
    for (int i = 0; i < 32; ++i)
        for (int j = 0; j < 32; ++j) {
            cd d(hD[i * 32 + j].x, hD[i * 32 + j].y);
            err = std::max(err, std::abs(d - M[i * 64 + 32 + j]));
        }
    for (int i = 0; i < 32; ++i)  // unitarity of I + D
        for (int j = 0; j < 32; ++j) {
            cd s = 0;
            for (int r = 0; r < 32; ++r) {
                cd a(hD[r * 32 + i].x, hD[r * 32 + i].y), b(hD[r * 32 + j].x, hD[r * 32 + j].y);
                if (r == i) a += 1.0;
                if (r == j) b += 1.0;
                s += std::conj(a) * b;
            }
            uerr = std::max(uerr, std::abs(s - (i == j ? 1.0 : 0.0)));
        }
    printf("cayley_cross: max |D - D_ref| = %.3e, max |Q^H Q - I| = %.3e (%s)\n", err, uerr, cudaGetErrorString(e));
    return 0;
}
