// cs_tcb.cu -- K3 "tcb": tensor-core blocked one-sided Jacobi for large
// blocks with vectors (fp32; cfg5's 256 x 256 + V).
//
// Same partition and block-circle ordering as the panel kernel
// (cs_panel.cuh): a cluster of C CTAs holds one matrix, CTA c owns two
// panels of W = 16 columns (all X and V rows), and 2C-1 super-rounds per
// sweep pair every panel with every other.  What changes is how a
// super-round treats its panel pair P = [a b] (X rows then V rows):
//
//   1. G = P_X^H P_X on tcgen05 (3xTF32, 64 x 64 real, 4 row stages whose
//      TMEM accumulators are summed in fp32);
//   2. every pair's rotation is computed from G at once -- the reference's
//      test |gamma| <= tol sqrt(alpha beta) and angle t = tan(theta)
//      (blocksvd.py:97-109, rot_params) -- and the rotations are combined
//      into one unitary Q = exp(E), E_pq = theta phi, E_qp = -theta conj(phi)
//      (a pair's own exp is exactly its Jacobi rotation); D = Q - I comes
//      from a Horner/scaling-squaring series on 32 x 32 complex matrices;
//   3. P <- P + P D on tcgen05 (3xTF32, M = 128 rows per block).
// The first super-round of a sweep treats all pairs of the 32 columns
// (within a, within b, cross), the others the cross pairs a x b, so every
// column pair is tested once per sweep; a sweep in which no pair passes
// the threshold ends the solve exactly as in the reference (blocksvd.py:
// 121-123).  Simultaneous rotations replace the w sequential rounds whose
// dependency chain bounds the scalar kernel; a CPU study of the block
// ordering (warm-started cfg5 blocks, f64) needs 6.8 instead of 6.0 sweeps.
//
// The panels live in shared memory in the 128-byte-swizzled K-major layout
// the update reads directly (cs_tcb.cuh); the Gram reads a transposed hi|lo
// copy staged per 64 rows.  Between super-rounds panels move across the
// cluster through DSMEM as in the panel kernel.
#include "cs_tcb.cuh"

namespace cs {
namespace tcb {

constexpr int NT = 512;

#ifdef CS_TCB_CLOCKS
// experiment builds only (tools/ab_build.sh with CS_AB_FLAGS=-DCS_TCB_CLOCKS):
// CTA-0-thread-0 cycles per phase, summed over super-rounds
__device__ unsigned long long g_tcb_cycles[10];  // [7] cluster wait, [9] super-round count
#define TCB_MARK(i)                                                                  \
    do {                                                                             \
        if (tid == 0) {                                                              \
            const long long _c = clock64();                                          \
            atomicAdd(&g_tcb_cycles[i], (unsigned long long)(_c - tcb_t));           \
            tcb_t = _c;                                                              \
        }                                                                            \
    } while (0)
#else
#define TCB_MARK(i) do { } while (0)
#endif

template <int MR, int NC>
struct Cfg {
    static constexpr int C = NC / N2;
    static constexpr int ROWS = MR + NC;
    static constexpr uint32_t ATOM = ROWS * 128;
    static constexpr uint32_t RG_OFF = 2 * ATOM;
    static constexpr uint32_t RG_BYTES = 65536;
    static constexpr uint32_t SIG_OFF = RG_OFF + RG_BYTES;
    static constexpr uint32_t PERM_OFF = SIG_OFF + NC * 4;
    static constexpr uint32_t FLAG_OFF = PERM_OFF + 2 * NC * 4;
    static constexpr uint32_t RED_OFF = FLAG_OFF + 68 * 4;
    static constexpr uint32_t BAR_OFF = (RED_OFF + 64 * 4 + 15) & ~15u;
    static constexpr uint32_t TM_OFF = BAR_OFF + 4 * 8;
    static constexpr uint32_t SMEM = TM_OFF + 16;
    static constexpr int STAGES = MR / 64;
    static constexpr int MBLK = ROWS / 128;
    static_assert(MR % 64 == 0 && ROWS % 128 == 0 && NC % N2 == 0, "tcb shape");
    static_assert(STAGES <= 4 && MBLK <= 4, "tcb TMEM budget (4 accumulators of 128 columns)");
    static_assert(C >= 2 && C <= 8, "tcb cluster size");
    static_assert(SMEM <= 227 * 1024, "tcb shared memory");
};

// scratch offsets inside the region during the rotation phase (bytes)
// (HH, HL: real 64 x 65 partial Grams read from TMEM; dead once G is built)
constexpr uint32_t SC_D = 0, SC_PRM = 8448, SC_E = 16384, SC_T = 24832, SC_HH = 0, SC_HL = 16640, SC_G = 33792,
                   SC_BOP = 32768;
constexpr int LDR = 65;

// C = s * A B (+ I) on 32 x 32 complex matrices in shared memory (stride LDG)
__device__ __forceinline__ void cgemm32(const float2 *A, const float2 *B, float2 *Cm, float s, bool addI) {
    const int t = threadIdx.x, i = t >> 4, j = t & 15;
    float2 c0 = make_float2(0.f, 0.f), c1 = c0;
#pragma unroll 8
    for (int k = 0; k < N2; ++k) {
        const float2 a = A[i * LDG + k], b0 = B[k * LDG + j], b1 = B[k * LDG + j + 16];
        c0.x = fmaf(a.x, b0.x, fmaf(-a.y, b0.y, c0.x));
        c0.y = fmaf(a.x, b0.y, fmaf(a.y, b0.x, c0.y));
        c1.x = fmaf(a.x, b1.x, fmaf(-a.y, b1.y, c1.x));
        c1.y = fmaf(a.x, b1.y, fmaf(a.y, b1.x, c1.y));
    }
    c0.x *= s; c0.y *= s; c1.x *= s; c1.y *= s;
    if (addI) {
        if (i == j) c0.x += 1.f;
        if (i == j + 16) c1.x += 1.f;
    }
    Cm[i * LDG + j] = c0;
    Cm[i * LDG + j + 16] = c1;
}

// D = exp(E) - I for a skew-Hermitian E (in Em, overwritten by the scaled E;
// Tm scratch): ||E||_inf scaled by 2^-s to <= 1/2, Horner of the lowest
// degree d with (1/2)^(d+1)/(d+1)! <= 1e-9, then s squarings
// (I + D)^2 = I + (2D + D D).  512 threads.
__device__ void expm_minus_identity(float2 *Em, float2 *Tm, float2 *Dm, float *red) {
    const int tid = threadIdx.x;
    if (tid < N2) {
        float sum = 0.f;
        for (int k = 0; k < N2; ++k) sum += hypotf(Em[tid * LDG + k].x, Em[tid * LDG + k].y);
        red[tid] = sum;
    }
    __syncthreads();
    float nrm = 0.f;
#pragma unroll 8
    for (int k = 0; k < N2; ++k) nrm = fmaxf(nrm, red[k]);
    int s = 0;
    while (nrm > 0.5f && s < 16) { nrm *= 0.5f; ++s; }
    int deg = 1;
    float term = nrm * nrm * 0.5f;  // nrm^(deg+1)/(deg+1)!
    while (term > 1e-9f && deg < 10) { ++deg; term *= nrm / (float)(deg + 1); }
    const float sc = ldexpf(1.f, -s), inv = 1.f / (float)deg;
    for (int x = tid; x < N2 * N2; x += blockDim.x) {
        const int i = x >> 5, j = x & 31;
        float2 e = Em[i * LDG + j];
        e.x *= sc; e.y *= sc;
        Em[i * LDG + j] = e;
        Tm[i * LDG + j] = make_float2(e.x * inv + (i == j ? 1.f : 0.f), e.y * inv);
    }
    __syncthreads();
    float2 *Xc = Tm, *Xn = Dm;
    for (int k = deg - 1; k >= 2; --k) {  // X_k = I + E X_{k+1} / k
        cgemm32(Em, Xc, Xn, 1.f / (float)k, true);
        __syncthreads();
        float2 *tt = Xc; Xc = Xn; Xn = tt;
    }
    if (deg >= 2) {
        cgemm32(Em, Xc, Xn, 1.f, false);  // E X_2
        __syncthreads();
        if (Xn != Dm)
            for (int x = tid; x < N2 * LDG; x += blockDim.x) Dm[x] = Xn[x];
    } else {
        for (int x = tid; x < N2 * LDG; x += blockDim.x) Dm[x] = Em[x];
    }
    __syncthreads();
    for (int k = 0; k < s; ++k) {
        cgemm32(Dm, Dm, Tm, 1.f, false);
        __syncthreads();
        for (int x = tid; x < N2 * N2; x += blockDim.x) {
            const int i = x >> 5, j = x & 31;
            const float2 d = Dm[i * LDG + j], e = Tm[i * LDG + j];
            Dm[i * LDG + j] = make_float2(2.f * d.x + e.x, 2.f * d.y + e.y);
        }
        __syncthreads();
    }
}

template <int MR, int NC>
__global__ void __launch_bounds__(NT, 1) jacobi_tcb_kernel(const JacArgs<float> a) {
    using K = Cfg<MR, NC>;
    constexpr int C = K::C;
    constexpr uint32_t ATOM = K::ATOM;
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char *AB = sm;
    unsigned char *RG = sm + K::RG_OFF;
    float *sig2 = reinterpret_cast<float *>(sm + K::SIG_OFF);
    int *perm = reinterpret_cast<int *>(sm + K::PERM_OFF);
    int *flags = reinterpret_cast<int *>(sm + K::FLAG_OFF);
    int *pos = flags + 4;
    float *red = reinterpret_cast<float *>(sm + K::RED_OFF);
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + K::BAR_OFF);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sm + K::TM_OFF);
    float2 *Dm = reinterpret_cast<float2 *>(RG + SC_D);
    float2 *Gm = reinterpret_cast<float2 *>(RG + SC_G);
    unsigned char *Bop = RG + SC_BOP;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int rank = (int)cg::this_cluster().block_rank();
    const long long cid = blockIdx.x / C;
    const float tol = a.tol;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    tc_after_sync();
    const uint32_t tmem = *tmem_slot;
    uint32_t ph1 = 0, ph2 = 0;  // parities of the two ring barriers (bar[1], bar[2])
    auto ring_wait = [&](int slot) {
        if (slot == 0) { mbar_wait(&bar[1], ph1); ph1 ^= 1; }
        else { mbar_wait(&bar[2], ph2); ph2 ^= 1; }
    };

    for (long long f = cid; f < a.count; f += a.s.num_clusters) {
        const long long mid = a.index ? a.index[f] : f;
        if (tid < 2 * C) pos[tid] = tid;
        // ---- load the two panels: a = columns [rank W, +W), b = [(2C-1-rank) W, +W)
        {
            const float2 *X0 = a.initX ? a.initX + (size_t)f * MR * NC : nullptr;
            const float2 *V0 = a.initV ? a.initV + (size_t)a.initV_index[f] * NC * NC : nullptr;
            const float2 *A = a.blocks + (size_t)mid * a.co * a.ci;
            for (int half = 0; half < 2; ++half) {
                const int c0 = (half == 0 ? rank : 2 * C - 1 - rank) * W;
                for (int idx = tid; idx < K::ROWS * W; idx += NT) {
                    const int r = idx / W, jj = idx % W, j = c0 + jj;
                    float2 v;
                    if (r < MR) {
                        if (X0) v = X0[(size_t)r * NC + j];
                        else if (!a.s.wide) v = A[(size_t)r * a.ci + j];
                        else { v = A[(size_t)j * a.ci + r]; v.y = -v.y; }
                    } else {
                        const int rv = r - MR;
                        if (V0) v = V0[(size_t)rv * NC + j];
                        else v = make_float2(rv == j ? 1.f : 0.f, 0.f);
                    }
                    *reinterpret_cast<float2 *>(AB + sw_off(r, 32 * half + 2 * jj, ATOM)) = v;
                }
            }
        }
        __syncthreads();

        int info = -1;
        for (int sweep = 0; sweep < a.max_sweeps; ++sweep) {
            bool rot = false, bad = false;
#pragma unroll 1
            for (int t = 0; t < 2 * C - 1; ++t) {
                const bool full = (t == 0);
#ifdef CS_TCB_CLOCKS
                long long tcb_t = clock64();
                if (tid == 0) atomicAdd(&g_tcb_cycles[9], 1ull);
#endif
                // ---- (1) Gram: STAGES x 64 X rows, transposed hi|lo staging, 2-slot ring
#pragma unroll 1
                for (int st = 0; st < K::STAGES; ++st) {
                    const int slot = st & 1;
                    if (st >= 2) ring_wait(slot);
                    gram_stage<NT>(AB, ATOM, 64 * st, RG + slot * 32768);
                    fence_proxy_async_smem();
                    __syncthreads();
                    if (warp == (st & 3)) {  // one issuing warp per stage (issuers overlap)
                        if (lane == 0) {
                            tc_after_sync();
                            gram_mma(tmem + 128 * (st & 3), smem_u32(RG + slot * 32768));
                            mma_commit(&bar[1 + slot]);
                        }
                        __syncwarp();
                    }
                }
                if (K::STAGES >= 2) { ring_wait(K::STAGES & 1); ring_wait((K::STAGES + 1) & 1); }
                else ring_wait(0);
                tc_after_sync();
                TCB_MARK(0);
                // ---- (2) G (complex, 32 x 32) from the stage accumulators: row i < 64
                // of a 128 x 128 accumulator is TMEM lane i; columns [0, 64) = hi*hi,
                // [64, 128) = hi*lo.  R = HH + HL + HL^T (real 64 x 64 Gram of the
                // real columns), summed over stages in fp32.
                {
                    float *HH = reinterpret_cast<float *>(RG + SC_HH);
                    float *HL = reinterpret_cast<float *>(RG + SC_HL);
                    const int q = warp & 3, cb = 32 * (warp >> 2);
                    if (q < 2) {  // lanes 0..63: warps with quarter 0, 1; 32 columns each
                        float acc[32];
#pragma unroll
                        for (int i = 0; i < 32; ++i) acc[i] = 0.f;
#pragma unroll 1
                        for (int st = 0; st < K::STAGES; ++st) {
                            float v[16];
                            tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + 128 * st + cb, v);
#pragma unroll
                            for (int i = 0; i < 16; ++i) acc[i] += v[i];
                            tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + 128 * st + cb + 16, v);
#pragma unroll
                            for (int i = 0; i < 16; ++i) acc[16 + i] += v[i];
                        }
                        const int row = 32 * q + lane;
                        float *dst = cb < 64 ? HH + row * LDR + cb : HL + row * LDR + (cb - 64);
#pragma unroll
                        for (int i = 0; i < 32; ++i) dst[i] = acc[i];
                    }
                    tc_before_sync();
                    __syncthreads();
                    for (int x = tid; x < N2 * N2; x += NT) {
                        const int c = x >> 5, j = x & 31;
                        auto R = [&](int i, int k) { return HH[i * LDR + k] + HL[i * LDR + k] + HL[k * LDR + i]; };
                        // G_r = R[2c][2j] + R[2c+1][2j+1], G_i = R[2c][2j+1] - R[2c+1][2j]
                        Gm[c * LDG + j] = make_float2(R(2 * c, 2 * j) + R(2 * c + 1, 2 * j + 1),
                                                      R(2 * c, 2 * j + 1) - R(2 * c + 1, 2 * j));
                    }
                    __syncthreads();
                }
                for (int x = tid; x < N2 * LDG; x += NT) Dm[x] = make_float2(0.f, 0.f);
                __syncthreads();
                TCB_MARK(1);
                // ---- (3) every pair's rotation from G at once (the reference's test
                // and root, rot_params), slot k of round r at prm[16 r + k]
                Prm<float> *prm = reinterpret_cast<Prm<float> *>(RG + SC_PRM);
                const int nround = full ? N2 - 1 : W;
                int act = 0;
                if (tid < nround * W) {
                    int p, qq;
                    inner_pair(full, tid % W, tid / W, p, qq);
                    const float2 g = Gm[p * LDG + qq];
                    Rot<float> R;
                    act = rot_params<float>(Gm[p * LDG + p].x, Gm[qq * LDG + qq].x, g.x, g.y, tol, R);
                    Prm<float> pm;
                    pm.cm1 = R.cm1; pm.wr = R.wr; pm.wi = R.wi; pm.act = act;
                    prm[tid] = pm;
                }
                const int any_rot = __syncthreads_or(act > 0);
                const int any_big = __syncthreads_or(act > 1);
                if (__syncthreads_or(act < 0)) bad = true;
                TCB_MARK(2);
                if (any_rot && !bad) {
                    rot = true;
                    if (!any_big) {
                        // ---- (4a) small angles (every |gamma| / sqrt(alpha beta) <=
                        // GCHECK_TAU): D = Q - I for Q = the product of the rounds'
                        // rotations, D <- D J_r + (J_r - I).  Rows evolve independently,
                        // so the 16 threads of a row (half a warp) only sync warp-wide.
                        const int i = tid >> 4, k = tid & 15;
#pragma unroll 1
                        for (int r = 0; r < nround; ++r) {
                            const Prm<float> pm = prm[r * W + k];
                            if (pm.act > 0) {
                                int p, qq;
                                inner_pair(full, k, r, p, qq);
                                float2 x = Dm[i * LDG + p], y = Dm[i * LDG + qq];
                                Rot<float> R;
                                R.cm1 = pm.cm1; R.wr = pm.wr; R.wi = pm.wi;
                                rot_apply<float>(x, y, R);
                                if (i == p) { x.x += R.cm1; y.x += R.wr; y.y += R.wi; }
                                if (i == qq) { x.x -= R.wr; x.y += R.wi; y.x += R.cm1; }
                                Dm[i * LDG + p] = x;
                                Dm[i * LDG + qq] = y;
                            }
                            __syncwarp();
                        }
                        __syncthreads();
                    } else {
                        // ---- (4b) some large angle: the product of stale rotations can
                        // stall, so the rotations are combined symmetrically instead:
                        // Q = exp(E), E_pq = theta phi, E_qp = -theta conj(phi)
                        // (a single pair's exp is exactly its Jacobi rotation)
                        float2 *Em = reinterpret_cast<float2 *>(RG + SC_E);
                        float2 *Tm = reinterpret_cast<float2 *>(RG + SC_T);
                        for (int x = tid; x < N2 * LDG; x += NT) Em[x] = make_float2(0.f, 0.f);
                        __syncthreads();
                        if (tid < nround * W) {
                            const Prm<float> pm = prm[tid];
                            if (pm.act > 0) {
                                int p, qq;
                                inner_pair(full, tid % W, tid / W, p, qq);
                                const float sn = sqrtf(pm.wr * pm.wr + pm.wi * pm.wi);  // sin(theta)
                                const float th = atan2f(sn, 1.f + pm.cm1);
                                const float f = th / sn;
                                Em[p * LDG + qq] = make_float2(f * pm.wr, f * pm.wi);
                                Em[qq * LDG + p] = make_float2(-f * pm.wr, f * pm.wi);
                            }
                        }
                        __syncthreads();
                        expm_minus_identity(Em, Tm, Dm, red);
                    }
                    TCB_MARK(3);
                    // ---- (5) B operand (D~, hi | lo) and (6) update P += P D
                    build_bop<NT>(Dm, Bop);
                    __syncthreads();  // D read before the ring (aliasing it) is written
#pragma unroll 1
                    for (int ch = 0; ch < 2 * K::MBLK; ++ch) {
                        const int mb = ch >> 1, at = ch & 1, slot = ch & 1;
                        if (ch >= 2) ring_wait(slot);
                        unsigned char *lo = RG + slot * 16384;
                        const unsigned char *srcp = AB + at * ATOM + mb * 16384;
#pragma unroll
                        for (int i = 0; i < 1024 / NT; ++i) {
                            const int u = tid + i * NT;
                            *reinterpret_cast<float4 *>(lo + 16 * u) =
                                lo4(*reinterpret_cast<const float4 *>(srcp + 16 * u));
                        }
                        fence_proxy_async_smem();
                        __syncthreads();
                        if (warp == 4 + slot) {  // one issuing warp per ring slot
                            if (lane == 0) {
                                tc_after_sync();
                                const uint32_t d = tmem + 128 * mb;
                                const uint32_t ah = smem_u32(srcp), al = smem_u32(lo);
                                const uint32_t bb = smem_u32(Bop) + at * 16384;
#pragma unroll
                                for (int ks = 0; ks < 4; ++ks) {
                                    const uint64_t dah = desc_sw128(ah + ks * 32), dal = desc_sw128(al + ks * 32);
                                    const uint64_t db = desc_sw128(bb + ks * 32);
                                    const uint32_t acc0 = (at | ks) ? 1u : 0u;
                                    mma_tf32(d, dah, db, IDESC_UPD, acc0);          // [hi*hi | hi*lo]
                                    mma_tf32(d + 64, dal, db, IDESC_UPD_LO, 1u);    // + lo*hi -> correction
                                }
                                mma_commit(&bar[1 + slot]);
                            }
                            __syncwarp();
                        }
                    }
                    ring_wait(0);
                    ring_wait(1);
                    tc_after_sync();
                    TCB_MARK(4);
                    // ---- (7) P += acc: warp group g -> M-blocks g, g+4, ..; quarter q -> lanes
                    {
                        const int q = warp & 3;
#pragma unroll 1
                        for (int mb = warp >> 2; mb < K::MBLK; mb += NT / 128) {
                            const int row = mb * 128 + 32 * q + lane;
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                float v[16], vc[16];
                                tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + 128 * mb + 16 * c, v);
                                tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + 128 * mb + 64 + 16 * c, vc);
#pragma unroll
                                for (int i = 0; i < 16; ++i) v[i] += vc[i];
#pragma unroll
                                for (int u = 0; u < 4; ++u) {
                                    float4 *pp = reinterpret_cast<float4 *>(AB + sw_chunk(row, 4 * c + u, ATOM));
                                    float4 x = *pp;
                                    x.x += v[4 * u]; x.y += v[4 * u + 1]; x.z += v[4 * u + 2]; x.w += v[4 * u + 3];
                                    *pp = x;
                                }
                            }
                        }
                        tc_before_sync();
                    }
                }
                __syncthreads();
                TCB_MARK(5);
                // ---- (8) panel rotation across the cluster (circle method over 2C
                // positions, position 0 fixed): new a <- position rank+1, new b <-
                // position 2C-rank; staged through registers (peers read this CTA's
                // panels until the second cluster barrier)
                if (t < 2 * C - 2) {
                    cluster_sync_all();
                    TCB_MARK(7);  // waiting for the slowest CTA of the cluster
                    const uint32_t own = smem_u32(AB);
                    const uint32_t src_a = rank == 0 ? own : (rank == C - 1 ? own + ATOM : map_rank(own, rank + 1));
                    const uint32_t src_b = rank == 0 ? map_rank(own, 1) : map_rank(own + ATOM, rank - 1);
                    constexpr int PER = (int)(ATOM / 16 / NT);
                    float4 ra[PER], rb[PER];
#pragma unroll
                    for (int i = 0; i < PER; ++i) {
                        const uint32_t o = 16u * (tid + i * NT);
                        if (rank != 0) {
                            asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];"
                                         : "=f"(ra[i].x), "=f"(ra[i].y), "=f"(ra[i].z), "=f"(ra[i].w)
                                         : "r"(src_a + o) : "memory");
                        }
                        asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];"
                                     : "=f"(rb[i].x), "=f"(rb[i].y), "=f"(rb[i].z), "=f"(rb[i].w)
                                     : "r"(src_b + o) : "memory");
                    }
                    int np = 0;
                    if (tid < 2 * C) np = (tid == 0) ? pos[0] : (tid == 2 * C - 1 ? pos[1] : pos[tid + 1]);
                    cluster_sync_all();
#pragma unroll
                    for (int i = 0; i < PER; ++i) {
                        const uint32_t o = 16u * (tid + i * NT);
                        if (rank != 0) *reinterpret_cast<float4 *>(AB + o) = ra[i];
                        *reinterpret_cast<float4 *>(AB + ATOM + o) = rb[i];
                    }
                    if (tid < 2 * C) pos[tid] = np;
                    __syncthreads();
                }
                TCB_MARK(6);
            }
            // ---- sweep verdict, OR-ed over the cluster
            if (tid == 0) {
                flags[0] = rot ? 1 : 0;
                flags[1] = bad ? 1 : 0;
            }
            cluster_sync_all();
            int any_rot = 0, any_bad = 0;
            {
                cg::cluster_group cl = cg::this_cluster();
                for (int d = 0; d < C; ++d) {
                    const int *pf = cl.map_shared_rank(flags, d);
                    any_rot |= pf[0];
                    any_bad |= pf[1];
                }
            }
            cluster_sync_all();
            if (any_bad) break;
            if (!any_rot) {
                info = sweep + 1;
                break;
            }
        }

        // ---- epilogue: exact fp32 column norms of the local panels, gathered
        // over the cluster; stable descending order; U = X / sigma, V
        const int pa = pos[rank], pb = pos[2 * C - 1 - rank];
        for (int c = warp; c < N2; c += NT / 32) {
            const int half = c / W, jj = c % W;
            float acc = 0.f;
            for (int r = lane; r < MR; r += 32) {
                const float2 v = *reinterpret_cast<const float2 *>(AB + sw_off(r, 32 * half + 2 * jj, ATOM));
                acc = fmaf(v.x, v.x, fmaf(v.y, v.y, acc));
            }
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            if (lane == 0) sig2[(half == 0 ? pa : pb) * W + jj] = acc;
        }
        cluster_sync_all();
        {
            float *stage = reinterpret_cast<float *>(RG);
            cg::cluster_group cl = cg::this_cluster();
            for (int j = tid; j < NC; j += NT) {
                const int panel = j / W;
                int p0 = 0;
                for (int p = 0; p < 2 * C; ++p)
                    if (pos[p] == panel) p0 = p;
                const int owner = pos_owner(p0, C);
                stage[j] = owner == rank ? sig2[j] : cl.map_shared_rank(sig2, owner)[j];
            }
            cluster_sync_all();
            for (int j = tid; j < NC; j += NT) sig2[j] = sqrtf(stage[j]);
            __syncthreads();
        }
        for (int j = tid; j < NC; j += NT) perm[j] = j;
        __syncthreads();
        if (info >= 0) {
            int *rnk = perm + NC;
            for (int j = tid; j < NC; j += NT) {
                const float sj = sig2[j];
                int pp = 0;
                for (int i = 0; i < NC; ++i) {
                    const float si = sig2[i];
                    pp += (si > sj) || (si == sj && i < j);
                }
                rnk[j] = pp;
            }
            __syncthreads();
            for (int j = tid; j < NC; j += NT) perm[rnk[j]] = j;
            __syncthreads();
        }
        if (rank == 0) {
            for (int p = tid; p < NC; p += NT) a.sigma[(size_t)mid * NC + p] = sig2[perm[p]];
            if (tid == 0) a.info[mid] = info;
        }
        int *ipos = perm + NC;
        __syncthreads();
        for (int p = tid; p < NC; p += NT) ipos[perm[p]] = p;
        __syncthreads();
        for (int half = 0; half < 2; ++half) {
            const int c0 = (half == 0 ? pa : pb) * W;
            if (a.Uw) {
                for (int idx = tid; idx < MR * W; idx += NT) {
                    const int r = idx / W, jj = idx % W, j = c0 + jj;
                    const float sj = sig2[j];
                    const float den = sj > 0.f ? sj : 1.f;
                    const float2 v = *reinterpret_cast<const float2 *>(AB + sw_off(r, 32 * half + 2 * jj, ATOM));
                    a.Uw[((size_t)mid * MR + r) * NC + ipos[j]] = make_float2(__fdividef(v.x, den), __fdividef(v.y, den));
                }
            }
            if (a.Vw) {
                for (int idx = tid; idx < NC * W; idx += NT) {
                    const int r = idx / W, jj = idx % W, j = c0 + jj;
                    a.Vw[((size_t)mid * NC + r) * NC + ipos[j]] =
                        *reinterpret_cast<const float2 *>(AB + sw_off(MR + r, 32 * half + 2 * jj, ATOM));
                }
            }
        }
        if (a.zero_sigma && rank == 0 && tid == 0) {
            int z = 0;
            for (int j = 0; j < NC; ++j) z |= !(sig2[j] > 0.f);
            a.zero_sigma[mid] = z;
        }
        cluster_sync_all();  // peers done reading this CTA's buffers
        __syncthreads();
    }
    tc_before_sync();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int MR, int NC>
static int launch(const JacArgs<float> &args0, cudaStream_t st, bool dry, long long *ncl_out) {
    using K = Cfg<MR, NC>;
    JacArgs<float> args = args0;
    auto kern = jacobi_tcb_kernel<MR, NC>;
    CS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::SMEM));
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = K::C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = K::SMEM;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(K::C);
    int maxc = 0;
    CS_CUDA_TRY(cudaOccupancyMaxActiveClusters(&maxc, (void *)kern, &cfg));
    if (maxc <= 0) return fail(CS_ENOMEM, "tcb SVD: cluster configuration cannot be scheduled");
    const long long ncl = lmin(args.count, (long long)maxc);
    if (ncl_out) *ncl_out = ncl;
    if (dry) return CS_OK;
    args.s.num_clusters = ncl;
    cfg.gridDim = dim3((unsigned)(ncl * K::C));
    CS_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, args));
    return check_launch("jacobi_tcb_kernel");
}

}  // namespace tcb

// shapes the tensor-core blocked kernel is instantiated for (working
// orientation mr x nc, vectors requested, fp32)
bool tcb_supported(int mr, int nc, bool wantv) { return wantv && mr == 256 && nc == 256; }

#ifdef CS_TCB_CLOCKS
extern "C" int cs_debug_tcb_cycles(unsigned long long *out, int reset) {
    if (cudaDeviceSynchronize() != cudaSuccess) return 4;
    cudaMemcpyFromSymbol(out, tcb::g_tcb_cycles, sizeof(unsigned long long) * 10);
    if (reset) {
        unsigned long long z[10] = {};
        cudaMemcpyToSymbol(tcb::g_tcb_cycles, z, sizeof(z));
    }
    return 0;
}
#endif

int tcb_dispatch(const JacArgs<float> &a, cudaStream_t st) {
    if (a.s.mr == 256 && a.s.nc == 256) return tcb::launch<256, 256>(a, st, false, nullptr);
    return fail(CS_EINVAL, "tcb SVD: unsupported shape");
}

}  // namespace cs
