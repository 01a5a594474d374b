// inner_probe.cu -- the inner phase of the Gram-blocked super-round (the w
// cross rounds of rotations on the 2w x 2w Gram G, with D = Q - I
// accumulated), measured in isolation: the shipped inner_phase (column pass,
// row pass, 3 CTA barriers per round) against a fused form in which each of
// 256 threads owns one 2x2 pair block of G and applies the left and right
// rotations at once (2 barriers per round, one pass).  Same rotations, same
// result up to rounding.  Groundwork for the tensor-core blocked variant
// (the inner phase must shrink before tcgen05 Gram/update pay).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -o tools/inner_probe tools/inner_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "../paper_2506_05617_b200/csrc/cs_panel.cuh"

using namespace cs;

constexpr int W = 16, N2 = 32, LDG = N2 + 1;

__global__ void __launch_bounds__(512) shipped(const float2 *Gin, float2 *Gout, float2 *Dout, long long *cyc,
                                               float tol) {
    __shared__ float2 G[N2 * LDG], D[N2 * LDG];
    __shared__ Prm<float> prm[W];
    const float2 *g = Gin + (size_t)blockIdx.x * N2 * N2;
    for (int x = threadIdx.x; x < N2 * N2; x += blockDim.x) {
        G[(x / N2) * LDG + x % N2] = g[x];
        D[(x / N2) * LDG + x % N2] = make_float2(0.f, 0.f);
    }
    __syncthreads();
    const long long c0 = clock64();
    inner_phase<float>(W, G, D, prm, tol);
    __syncthreads();
    const long long c1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
    for (int x = threadIdx.x; x < N2 * N2; x += blockDim.x) {
        Gout[(size_t)blockIdx.x * N2 * N2 + x] = G[(x / N2) * LDG + x % N2];
        Dout[(size_t)blockIdx.x * N2 * N2 + x] = D[(x / N2) * LDG + x % N2];
    }
}

// fused: thread (P, Q) = (t / 16, t % 16) owns rows {p_P, q_P} x cols {p_Q, q_Q}
// of G (pair P: p = P, q = W + (P + sr) % W); G' = J^H G J on that 2x2 block.
// D' = D J + (J - I): the same threads own D rows {p_P, q_P} x cols {p_Q, q_Q}.
__global__ void __launch_bounds__(256) fused(const float2 *Gin, float2 *Gout, float2 *Dout, long long *cyc,
                                             float tol) {
    __shared__ float2 G[N2 * LDG], D[N2 * LDG];
    __shared__ Prm<float> prm[W];
    const float2 *g = Gin + (size_t)blockIdx.x * N2 * N2;
    for (int x = threadIdx.x; x < N2 * N2; x += blockDim.x) {
        G[(x / N2) * LDG + x % N2] = g[x];
        D[(x / N2) * LDG + x % N2] = make_float2(0.f, 0.f);
    }
    __syncthreads();
    const long long c0 = clock64();
    const int P = threadIdx.x / W, Q = threadIdx.x % W;
#pragma unroll 1
    for (int sr = 0; sr < W; ++sr) {
        if (threadIdx.x < W) {
            const int p = threadIdx.x, q = W + (threadIdx.x + sr) % W;
            const float2 gpq = G[p * LDG + q];
            Rot<float> R;
            const int act = rot_params<float>(G[p * LDG + p].x, G[q * LDG + q].x, gpq.x, gpq.y, tol, R);
            Prm<float> pm;
            pm.cm1 = R.cm1; pm.wr = R.wr; pm.wi = R.wi; pm.act = act;
            prm[threadIdx.x] = pm;
        }
        __syncthreads();
        const int pP = P, qP = W + (P + sr) % W, pQ = Q, qQ = W + (Q + sr) % W;
        const Prm<float> mP = prm[P], mQ = prm[Q];
        float2 a = G[pP * LDG + pQ], b = G[pP * LDG + qQ], c = G[qP * LDG + pQ], d = G[qP * LDG + qQ];
        if (mQ.act > 0) {  // right: columns (pQ, qQ) of rows pP and qP
            Rot<float> R;
            R.cm1 = mQ.cm1; R.wr = mQ.wr; R.wi = mQ.wi;
            rot_apply<float>(a, b, R);
            rot_apply<float>(c, d, R);
        }
        if (mP.act > 0) {  // left: rows (pP, qP) with conj(J) (rot_apply on conjugates)
            Rot<float> R;
            R.cm1 = mP.cm1; R.wr = mP.wr; R.wi = mP.wi;
            a.y = -a.y; c.y = -c.y; b.y = -b.y; d.y = -d.y;
            rot_apply<float>(a, c, R);
            rot_apply<float>(b, d, R);
            a.y = -a.y; c.y = -c.y; b.y = -b.y; d.y = -d.y;
        }
        // D: the same 2x2 block positions, right rotation + (J - I) on the diagonal pair block
        float2 da = D[pP * LDG + pQ], db = D[pP * LDG + qQ], dc = D[qP * LDG + pQ], dd = D[qP * LDG + qQ];
        if (mQ.act > 0) {
            Rot<float> R;
            R.cm1 = mQ.cm1; R.wr = mQ.wr; R.wi = mQ.wi;
            rot_apply<float>(da, db, R);
            rot_apply<float>(dc, dd, R);
            if (P == Q) {  // rows pP = pQ, qP = qQ: + (J - I)
                da.x += R.cm1; db.x += R.wr; db.y += R.wi;
                dc.x -= R.wr; dc.y += R.wi; dd.x += R.cm1;
            }
        }
        __syncthreads();  // every block read before any is written
        G[pP * LDG + pQ] = a; G[pP * LDG + qQ] = b; G[qP * LDG + pQ] = c; G[qP * LDG + qQ] = d;
        D[pP * LDG + pQ] = da; D[pP * LDG + qQ] = db; D[qP * LDG + pQ] = dc; D[qP * LDG + qQ] = dd;
        __syncthreads();
    }
    const long long c1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
    for (int x = threadIdx.x; x < N2 * N2; x += blockDim.x) {
        Gout[(size_t)blockIdx.x * N2 * N2 + x] = G[(x / N2) * LDG + x % N2];
        Dout[(size_t)blockIdx.x * N2 * N2 + x] = D[(x / N2) * LDG + x % N2];
    }
}

int main(int argc, char **argv) {
    const int B = argc > 1 ? atoi(argv[1]) : 148;
    std::vector<float2> G((size_t)B * N2 * N2);
    srand(3);
    // Hermitian G = P^H P of a random 64 x 32 complex P, columns of mixed scale
    for (int b = 0; b < B; ++b) {
        std::vector<float> pr(64 * N2), pi(64 * N2);
        for (int i = 0; i < 64 * N2; ++i) {
            const float s = 1.f + (i % N2) * 0.1f;
            pr[i] = s * ((float)rand() / RAND_MAX - 0.5f);
            pi[i] = s * ((float)rand() / RAND_MAX - 0.5f);
        }
        for (int i = 0; i < N2; ++i)
            for (int j = 0; j < N2; ++j) {
                double re = 0, im = 0;
                for (int r = 0; r < 64; ++r) {
                    const double ar = pr[r * N2 + i], ai = pi[r * N2 + i], br = pr[r * N2 + j], bi = pi[r * N2 + j];
                    re += ar * br + ai * bi;
                    im += ar * bi - ai * br;
                }
                G[(size_t)b * N2 * N2 + i * N2 + j] = make_float2((float)re, (float)im);
            }
    }
    float2 *dG, *g1, *d1, *g2, *d2;
    long long *c1, *c2;
    const size_t bytes = G.size() * sizeof(float2);
    cudaMalloc(&dG, bytes); cudaMalloc(&g1, bytes); cudaMalloc(&d1, bytes); cudaMalloc(&g2, bytes); cudaMalloc(&d2, bytes);
    cudaMalloc(&c1, B * 8); cudaMalloc(&c2, B * 8);
    cudaMemcpy(dG, G.data(), bytes, cudaMemcpyHostToDevice);
    const float tol = 5e-6f;
    for (int rep = 0; rep < 2; ++rep) {
        shipped<<<B, 512>>>(dG, g1, d1, c1, tol);
        fused<<<B, 256>>>(dG, g2, d2, c2, tol);
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<float2> h1(G.size()), h2(G.size()), e1(G.size()), e2(G.size());
    std::vector<long long> k1(B), k2(B);
    cudaMemcpy(h1.data(), g1, bytes, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2.data(), g2, bytes, cudaMemcpyDeviceToHost);
    cudaMemcpy(e1.data(), d1, bytes, cudaMemcpyDeviceToHost);
    cudaMemcpy(e2.data(), d2, bytes, cudaMemcpyDeviceToHost);
    cudaMemcpy(k1.data(), c1, B * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(k2.data(), c2, B * 8, cudaMemcpyDeviceToHost);
    double dg = 0, dd = 0, gm = 0;
    for (size_t i = 0; i < G.size(); ++i) {
        dg = fmax(dg, hypot(h1[i].x - h2[i].x, h1[i].y - h2[i].y));
        dd = fmax(dd, hypot(e1[i].x - e2[i].x, e1[i].y - e2[i].y));
        gm = fmax(gm, hypot(G[i].x, G[i].y));
    }
    double s1 = 0, s2 = 0;
    for (int b = 0; b < B; ++b) { s1 += k1[b]; s2 += k2[b]; }
    printf("inner phase, 16 rounds on 32x32 G (+D), %d matrices:\n", B);
    printf("  shipped (col pass + row pass, 3 barriers/round, 512 thr): %.0f cycles\n", s1 / B);
    printf("  fused 2x2 blocks (2 barriers/round, 256 thr):            %.0f cycles\n", s2 / B);
    printf("  max |G_shipped - G_fused| / max|G| = %.2e, max |D diff| = %.2e\n", dg / gm, dd);
    return 0;
}
