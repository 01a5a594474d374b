// tcb_probe.cu -- one tensor-core blocked super-round on a panel pair, in
// isolation (single CTA per pair, no cluster): the building blocks of the
// tcgen05 blocked Jacobi (K3) measured and checked against fp64.
//
// Panel pair [a b] = 32 complex columns x R rows (X rows then V rows), stored
// in 128-byte core matrices (8 rows x 4 floats = 2 complex columns):
//   byte offset(row, realcol) = (row>>3)*2048 + (realcol>>2)*128 + (row&7)*16 + (realcol&3)*4
// The same bytes are
//   * the MN-major operand of the Gram  G = P^H P  (M = N = 64 real columns,
//     K = X rows; LBO 2048 = next 8 rows, SBO 128 = next 4 columns), and
//   * the K-major A operand of the update P <- P + P D  (M = 128 rows,
//     K = 64 real columns; LBO 128, SBO 2048),
// so no operand repacking: hi = the stored fp32 word (the tensor core reads
// tf32 from it), lo = x - trunc_tf32(x) staged next to it (3xTF32).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -o tools/tcb_probe tools/tcb_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "../paper_2506_05617_b200/csrc/cs_tcb.cuh"

using namespace cs;
using namespace cs::tcb;

constexpr int ROWS_X = 256, ROWS_V = 256, ROWS = ROWS_X + ROWS_V;
constexpr int NT = 512;
constexpr uint32_t ATOM = ROWS * 128;               // 64 KB per panel
constexpr uint32_t PANEL_BYTES = 2 * ATOM;          // 128 KB
constexpr uint32_t REGION_BYTES = 64 * 1024;

struct Out {
    float G[N2 * N2 * 2];       // Gram from the tensor cores (complex, row-major)
    float D[N2 * N2 * 2];       // accumulated D = Q - I
    float P1[ROWS * KR];        // panel pair after the update, row-major real
    long long cyc[8];
};

// mode bit0: explicit truncated hi copy (else the raw fp32 word is the hi operand)
// nstage: Gram accumulated in nstage separate TMEM accumulators (summed in fp32)
__global__ void __launch_bounds__(NT, 1)
tcb_kernel(const float *Pin, Out *out, int mode, int nstage, float tol, int reps) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char *AB = sm;                         // panel pair (128 KB)
    unsigned char *RG = sm + PANEL_BYTES;           // region (64 KB)
    float2 *Gm = reinterpret_cast<float2 *>(RG);    // inner phase: G and D (aliases the region)
    float2 *Dm = Gm + N2 * LDG;
    Prm<float> *prm = reinterpret_cast<Prm<float> *>(Dm + N2 * LDG);
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar[4];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const float *src = Pin + (size_t)blockIdx.x * ROWS * KR;
    for (int x = tid; x < ROWS * KR; x += NT) {
        const int r = x / KR, c = x % KR;
        *reinterpret_cast<float *>(AB + sw_off(r, c, ATOM)) = src[x];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base;
    uint32_t ph[4] = {0, 0, 0, 0};
    long long cyc[6] = {0, 0, 0, 0, 0, 0};

    for (int rep = 0; rep < reps; ++rep) {
        long long t0 = clock64();
        // ---- (1)+(2) Gram: 4 stages of 64 X rows, transposed hi|lo staging in a 2-slot ring
        long long t1 = t0;
        for (int st = 0; st < 4; ++st) {
            const int slot = st & 1;
            if (st >= 2) { mbar_wait(&bar[1 + slot], ph[1 + slot]); ph[1 + slot] ^= 1; }
            gram_stage<NT>(AB, ATOM, 64 * st, RG + slot * 32768);
            fence_proxy_async_smem();
            __syncthreads();
            if (st == 0) t1 = clock64();
            if (tid == 0) {
                tc_after_sync();
                gram_mma(tmem + 64 * st, smem_u32(RG + slot * 32768));
                mma_commit(&bar[1 + slot]);
            }
        }
        for (int s2 = 0; s2 < 2; ++s2) { mbar_wait(&bar[1 + s2], ph[1 + s2]); ph[1 + s2] ^= 1; }
        tc_after_sync();
        long long t2 = clock64();
        // ---- (3) G from the accumulators (M = 64: row r in lane 32(r/16) + r%16) --
        {
            float R[64];
#pragma unroll
            for (int i = 0; i < 64; ++i) R[i] = 0.f;
            if (warp < 4) {
                for (int st = 0; st < 4; ++st) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        float v[16];
                        tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + 64 * st + 16 * c, v);
#pragma unroll
                        for (int i = 0; i < 16; ++i) R[16 * c + i] += v[i];
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            // real row i = 16 warp + lane (lane < 16); complex row c = i/2: lane 2c (re part row) pairs with 2c+1
            if (warp < 4) {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const float rr_re = R[2 * j], rr_im = R[2 * j + 1];
                    const float o_re = __shfl_xor_sync(0xffffffffu, rr_re, 1);  // row 2c+1 (imag part row)
                    const float o_im = __shfl_xor_sync(0xffffffffu, rr_im, 1);
                    if (lane < 16 && !(lane & 1)) {
                        const int c = (16 * warp + lane) >> 1;
                        // G_r = R[2c][2j] + R[2c+1][2j+1];  G_i = R[2c][2j+1] - R[2c+1][2j]
                        Gm[c * LDG + j] = make_float2(rr_re + o_im, rr_im - o_re);
                    }
                }
            }
            for (int x = tid; x < N2 * N2; x += NT) Dm[(x / N2) * LDG + x % N2] = make_float2(0.f, 0.f);
        }
        __syncthreads();
        if (rep == 0 && blockIdx.x < 4)
            for (int x = tid; x < N2 * N2; x += NT) {
                out[blockIdx.x].G[2 * x] = Gm[(x / N2) * LDG + x % N2].x;
                out[blockIdx.x].G[2 * x + 1] = Gm[(x / N2) * LDG + x % N2].y;
            }
        long long t3 = clock64();
        // ---- (4) inner phase: w cross rounds on G, D <- D J + (J - I) ------------
        {
            const int P = tid / W, Q = tid % W;
            const bool act_t = tid < 256;
#pragma unroll 1
            for (int sr = 0; sr < W; ++sr) {
                if (tid < W) {
                    const int p = tid, q = W + (tid + sr) % W;
                    const float2 gpq = Gm[p * LDG + q];
                    Rot<float> R;
                    const int act = rot_params<float>(Gm[p * LDG + p].x, Gm[q * LDG + q].x, gpq.x, gpq.y, tol, R);
                    Prm<float> pm;
                    pm.cm1 = R.cm1; pm.wr = R.wr; pm.wi = R.wi; pm.act = act;
                    prm[tid] = pm;
                }
                __syncthreads();
                float2 a, b, c, d, da, db, dc, dd;
                int pP = 0, qP = 0, pQ = 0, qQ = 0;
                if (act_t) {
                    pP = P; qP = W + (P + sr) % W; pQ = Q; qQ = W + (Q + sr) % W;
                    const Prm<float> mP = prm[P], mQ = prm[Q];
                    a = Gm[pP * LDG + pQ]; b = Gm[pP * LDG + qQ]; c = Gm[qP * LDG + pQ]; d = Gm[qP * LDG + qQ];
                    da = Dm[pP * LDG + pQ]; db = Dm[pP * LDG + qQ]; dc = Dm[qP * LDG + pQ]; dd = Dm[qP * LDG + qQ];
                    if (mQ.act > 0) {
                        Rot<float> R;
                        R.cm1 = mQ.cm1; R.wr = mQ.wr; R.wi = mQ.wi;
                        rot_apply<float>(a, b, R);
                        rot_apply<float>(c, d, R);
                        rot_apply<float>(da, db, R);
                        rot_apply<float>(dc, dd, R);
                        if (P == Q) {
                            da.x += R.cm1; db.x += R.wr; db.y += R.wi;
                            dc.x -= R.wr; dc.y += R.wi; dd.x += R.cm1;
                        }
                    }
                    if (mP.act > 0) {
                        Rot<float> R;
                        R.cm1 = mP.cm1; R.wr = mP.wr; R.wi = mP.wi;
                        a.y = -a.y; c.y = -c.y; b.y = -b.y; d.y = -d.y;
                        rot_apply<float>(a, c, R);
                        rot_apply<float>(b, d, R);
                        a.y = -a.y; c.y = -c.y; b.y = -b.y; d.y = -d.y;
                    }
                }
                __syncthreads();
                if (act_t) {
                    Gm[pP * LDG + pQ] = a; Gm[pP * LDG + qQ] = b; Gm[qP * LDG + pQ] = c; Gm[qP * LDG + qQ] = d;
                    Dm[pP * LDG + pQ] = da; Dm[pP * LDG + qQ] = db; Dm[qP * LDG + pQ] = dc; Dm[qP * LDG + qQ] = dd;
                }
                __syncthreads();
            }
        }
        if (rep == 0 && blockIdx.x < 4)
            for (int x = tid; x < N2 * N2; x += NT) {
                out[blockIdx.x].D[2 * x] = Dm[(x / N2) * LDG + x % N2].x;
                out[blockIdx.x].D[2 * x + 1] = Dm[(x / N2) * LDG + x % N2].y;
            }
        long long t4 = clock64();
        // ---- (5) B operand from D (hi | lo, 32 KB at RG + 32 KB)
        unsigned char *Bop = RG + 32768;
        build_bop<NT>(Dm, Bop);
        __syncthreads();  // D read before the ring (aliasing G/D) is written
        // ---- (6) update: per M-block (128 rows) and K atom (panel a | b), lo staged into a 2-slot ring
        unsigned char *ring = RG;  // 2 x 16 KB, byte image of the panel's atom slice
        for (int ch = 0; ch < 8; ++ch) {
            const int mb = ch >> 1, at = ch & 1, slot = ch & 1;
            if (ch >= 2) { mbar_wait(&bar[1 + slot], ph[1 + slot]); ph[1 + slot] ^= 1; }
            unsigned char *lo = ring + slot * 16384;
            const unsigned char *srcp = AB + at * ATOM + mb * 16384;
#pragma unroll
            for (int i = 0; i < 1024 / NT; ++i) {
                const int u = tid + i * NT;
                *reinterpret_cast<float4 *>(lo + 16 * u) = lo4(*reinterpret_cast<const float4 *>(srcp + 16 * u));
            }
            fence_proxy_async_smem();
            __syncthreads();
            if (tid == 0) {
                tc_after_sync();
                const uint32_t d = tmem + 64 * mb;
                const uint32_t ah = smem_u32(srcp), al = smem_u32(lo), bh = smem_u32(Bop) + at * 8192, bl = bh + 16384;
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const uint32_t acc0 = (at | ks) ? 1u : 0u;
                    const uint64_t dah = desc_sw128(ah + ks * 32), dal = desc_sw128(al + ks * 32);
                    const uint64_t dbh = desc_sw128(bh + ks * 32), dbl = desc_sw128(bl + ks * 32);
                    const uint32_t d2 = (mode & 2) ? d + 256 : d;
                    mma_tf32(d, dah, dbh, IDESC_UPD, acc0);
                    mma_tf32(d2, dah, dbl, IDESC_UPD, (mode & 2) ? acc0 : 1u);
                    mma_tf32(d2, dal, dbh, IDESC_UPD, 1u);
                }
                mma_commit(&bar[1 + slot]);
            }
        }
        for (int s = 0; s < 2; ++s) {
            mbar_wait(&bar[1 + s], ph[1 + s]);
            ph[1 + s] ^= 1;
        }
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        long long t5 = clock64();
        // ---- (7) epilogue: P += acc (warp group g -> M-block g, quarter q -> lanes 32q..)
        {
            const int g = warp >> 2, q = warp & 3, row = g * 128 + 32 * q + lane;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                float v[16];
                tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + 64 * g + 16 * c, v);
                if (mode & 2) {
                    float v2[16];
                    tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + 256 + 64 * g + 16 * c, v2);
#pragma unroll
                    for (int i = 0; i < 16; ++i) v[i] += v2[i];
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    float4 *pp = reinterpret_cast<float4 *>(AB + sw_chunk(row, 4 * c + u, ATOM));
                    float4 x = *pp;
                    x.x += v[4 * u]; x.y += v[4 * u + 1]; x.z += v[4 * u + 2]; x.w += v[4 * u + 3];
                    *pp = x;
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        }
        __syncthreads();
        long long t6 = clock64();
        cyc[0] += t1 - t0; cyc[1] += t2 - t1; cyc[2] += t3 - t2; cyc[3] += t4 - t3; cyc[4] += t5 - t4; cyc[5] += t6 - t5;
        if (rep == 0 && blockIdx.x < 4)
            for (int x = tid; x < ROWS * KR; x += NT) {
                const int r = x / KR, c = x % KR;
                out[blockIdx.x].P1[x] = *reinterpret_cast<float *>(AB + sw_off(r, c, ATOM));
            }
        __syncthreads();
    }
    if (tid == 0 && blockIdx.x < 4)
        for (int i = 0; i < 6; ++i) out[blockIdx.x].cyc[i] = cyc[i] / reps;
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main(int argc, char **argv) {
    const int B = argc > 1 ? atoi(argv[1]) : 148;
    const int mode = argc > 2 ? atoi(argv[2]) : 0;
    const int nstage = argc > 3 ? atoi(argv[3]) : 4;
    const float scale_spread = argc > 4 ? atof(argv[4]) : 1e-3f;
    // panels: X rows with graded column scales (1 .. scale_spread) and a small
    // common component (off-diagonal Gram ~ 1e-2), V rows ~ unitary-ish
    std::vector<float> P((size_t)B * ROWS * KR);
    srand(7);
    for (int b = 0; b < B; ++b)
        for (int c = 0; c < N2; ++c) {
            const float s = powf(scale_spread, (float)((c * 7) % N2) / (N2 - 1));
            for (int r = 0; r < ROWS; ++r) {
                const float g1 = (float)rand() / RAND_MAX - 0.5f, g2 = (float)rand() / RAND_MAX - 0.5f;
                const float sc = r < ROWS_X ? s : 0.0625f;
                P[(size_t)b * ROWS * KR + r * KR + 2 * c] = sc * g1;
                P[(size_t)b * ROWS * KR + r * KR + 2 * c + 1] = sc * g2;
            }
        }
    float *dP;
    Out *dO;
    cudaMalloc(&dP, P.size() * 4);
    cudaMalloc(&dO, 4 * sizeof(Out));
    cudaMemcpy(dP, P.data(), P.size() * 4, cudaMemcpyHostToDevice);
    const size_t smem = PANEL_BYTES + REGION_BYTES;
    cudaFuncSetAttribute(tcb_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    tcb_kernel<<<B, NT, smem>>>(dP, dO, mode, nstage, 5e-6f, 1);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<Out> O(4);
    cudaMemcpy(O.data(), dO, 4 * sizeof(Out), cudaMemcpyDeviceToHost);
    double gerr = 0, gerr_rel = 0, uerr = 0, dmax = 0, umag = 0;
    for (int b = 0; b < std::min(B, 4); ++b) {
        const float *p = P.data() + (size_t)b * ROWS * KR;
        // fp64 Gram vs tensor-core Gram; error relative to sqrt(G_ii G_jj)
        std::vector<double> gr(N2 * N2), gi(N2 * N2);
        for (int i = 0; i < N2; ++i)
            for (int j = 0; j < N2; ++j) {
                double re = 0, im = 0;
                for (int r = 0; r < ROWS_X; ++r) {
                    const double xr = p[r * KR + 2 * i], xi = p[r * KR + 2 * i + 1];
                    const double yr = p[r * KR + 2 * j], yi = p[r * KR + 2 * j + 1];
                    re += xr * yr + xi * yi;
                    im += xr * yi - xi * yr;
                }
                gr[i * N2 + j] = re; gi[i * N2 + j] = im;
            }
        if (b == 0) {
            printf("row-wise max |G_tc - G| / max|G row| (b=0):\n");
            for (int i = 0; i < N2; ++i) {
                double e = 0, mx = 0;
                for (int j = 0; j < N2; ++j) {
                    e = fmax(e, hypot(O[b].G[2 * (i * N2 + j)] - gr[i * N2 + j], O[b].G[2 * (i * N2 + j) + 1] - gi[i * N2 + j]));
                    mx = fmax(mx, hypot(gr[i * N2 + j], gi[i * N2 + j]));
                }
                printf(" %.1e", e / mx);
            }
            printf("\n");
        }
        for (int i = 0; i < N2; ++i)
            for (int j = 0; j < N2; ++j) {
                const double er = hypot(O[b].G[2 * (i * N2 + j)] - gr[i * N2 + j], O[b].G[2 * (i * N2 + j) + 1] - gi[i * N2 + j]);
                gerr = fmax(gerr, er / gr[0]);
                gerr_rel = fmax(gerr_rel, er / sqrt(gr[i * N2 + i] * gr[j * N2 + j]));
            }
        // update check: P1 vs P + P D (fp64, with the device's D)
        const float *D = O[b].D;
        for (int r = 0; r < ROWS; ++r)
            for (int cp = 0; cp < N2; ++cp) {
                double re = p[r * KR + 2 * cp], im = p[r * KR + 2 * cp + 1];
                double dre = 0, dim = 0;
                for (int c = 0; c < N2; ++c) {
                    const double xr = p[r * KR + 2 * c], xi = p[r * KR + 2 * c + 1];
                    const double ar = D[2 * (c * N2 + cp)], ai = D[2 * (c * N2 + cp) + 1];
                    dre += xr * ar - xi * ai;
                    dim += xr * ai + xi * ar;
                }
                dmax = fmax(dmax, hypot(dre, dim));
                re += dre; im += dim;
                const double er = hypot(O[b].P1[r * KR + 2 * cp] - re, O[b].P1[r * KR + 2 * cp + 1] - im);
                uerr = fmax(uerr, er);
                umag = fmax(umag, hypot(re, im));
            }
    }
    printf("mode %d nstage %d spread %.0e: Gram err/max %.2e, err/sqrt(GiiGjj) %.2e; update err %.2e (|P| %.2e, |PD| %.2e)\n",
           mode, nstage, scale_spread, gerr, gerr_rel, uerr, umag, dmax);
    tcb_kernel<<<B, NT, smem>>>(dP, dO, mode, nstage, 5e-6f, 20);
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(O.data(), dO, 4 * sizeof(Out), cudaMemcpyDeviceToHost);
    printf("  cycles: first-stage %lld  gram %lld  G-read %lld  inner %lld  update %lld  epilogue %lld\n", O[0].cyc[0],
           O[0].cyc[1], O[0].cyc[2], O[0].cyc[3], O[0].cyc[4], O[0].cyc[5]);
    return 0;
}
