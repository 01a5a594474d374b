// cs_tcb.cu -- K3 "tcb": tensor-core blocked one-sided Jacobi for large
// blocks with vectors (fp32; cfg5's 256 x 256 + V).
//
// A group of C CTAs solves one matrix; CTA c holds two panels of W = 16
// columns (all X and V rows), and 2C-1 super-rounds per sweep pair every
// panel with every other.  A super-round treats its panel pair P = [a b]
// (X rows then V rows):
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
// dependency chain bounds the scalar kernel.
//
// Panel exchange (the part that bounds a super-round once the O(rows) work
// is on the tensor cores).  The 2C-1 pairings of a sweep are a fixed
// 1-factorisation of the 2C panels (circle method on panel labels); between
// two consecutive pairings every CTA keeps one panel and swaps the other --
// possible for ANY two perfect matchings (their union is a set of even
// alternating cycles; orienting each cycle gives every CTA one panel in and
// one out).  So only ONE panel (64 KB) moves per CTA and super-round instead
// of two, and odd sweeps run the pairings backwards (no exchange at sweep
// boundaries).  Panels move through L2 rather than DSMEM: the sender pushes
// the outgoing panel into its mailbox in global memory with TMA bulk stores
// (X rows first, then V rows, each published by a release flag); the
// receiver pulls it with TMA bulk loads into its free shared-memory slot and
// acknowledges.  No cluster barrier, only pairwise flags: a CTA waits only
// for the one CTA it receives from.  Without the cluster-placement limit
// (15 clusters of 8 = 120 SMs) the groups fill 144 of 148 SMs; co-residency
// of a group's CTAs is guaranteed by a cooperative launch.
//
// Shared memory: three 64 KB slots (panel a, panel b, scratch) whose roles
// rotate -- the incoming panel lands in the scratch slot, the outgoing
// panel's slot becomes the next scratch.
#include <cstdio>

#include "cs_tcb.cuh"

namespace cs {
namespace tcb {

constexpr int NT = 512;
#ifndef CS_K3_TAU
#define CS_K3_TAU 0.35f  // measured: 0.05 2901 ms, 0.2 2722, 0.35 2666, 0.5 2689, never-exp 2728 (cfg5 warm SVD)
#endif
constexpr float K3_TAU = CS_K3_TAU;  // small-angle (product) vs large-angle (exp) combination
#ifndef CS_K3_SPARSE
#define CS_K3_SPARSE 32
#endif
// a super-round with at most this many rotating pairs (late sweeps) applies them
// one after the other to the panels in shared memory instead of forming D and
// running the tensor-core update (0: never)
constexpr int K3_SPARSE = CS_K3_SPARSE;
static_assert(K3_SPARSE <= 32, "the sparse list lives in the 64-word reduction scratch");
constexpr int GW = 4;  // Gram-issuing warps (one TMEM accumulator each)
constexpr int MAXC = 16;

#ifdef CS_TCB_CLOCKS
// experiment builds only (tools/ab_build.sh with CS_AB_FLAGS=-DCS_TCB_CLOCKS):
// CTA-0-thread-0 cycles per phase, summed over super-rounds
__device__ unsigned long long g_tcb_sweep[4][16];  // per sweep index: cycles, super-rounds, dense rotating, sparse rotating
__device__ unsigned long long g_tcb_cycles[32];  // [23..28] exchange sub-phases  // [9] super-round count, [10] load, [11] verdict, [12] epilogue, [13] matrices
 // -DCS_TCB_CLOCKS_SWEEPS=n: the phase counters cover only the first n sweeps of a matrix
#ifndef CS_TCB_CLOCKS_SWEEPS
#define CS_TCB_CLOCKS_SWEEPS 1000
#endif
#define TCB_MARK(i)                                                                  \
    do {                                                                             \
        if (tid == 0 && tcb_on) {                                                              \
            const long long _c = clock64();                                          \
            atomicAdd(&g_tcb_cycles[i], (unsigned long long)(_c - tcb_t));           \
            tcb_t = _c;                                                              \
        }                                                                            \
    } while (0)
#define TCB_ADD(i, t0)                                                               \
    do {                                                                             \
        if (tid == 0 && tcb_on) atomicAdd(&g_tcb_cycles[i], (unsigned long long)(clock64() - (t0))); \
    } while (0)
#else
#define TCB_MARK(i) do { } while (0)
#define TCB_ADD(i, t0) do { } while (0)
#endif

// the sweep's pairings and the exchange between consecutive ones (host-built)
struct Sched {
    signed char ida[2 * MAXC - 1][MAXC], idb[2 * MAXC - 1][MAXC];  // panels of CTA c at step t
    signed char src[2 * MAXC - 2][MAXC], dst[2 * MAXC - 2][MAXC];  // exchange t -> t+1
};

// global-memory coordination area of a launch (inside the SVD workspace)
struct Ws {
    unsigned char *ctrl;  // per CTA 256 B: flags (see CT_*)
    float *gsig;          // per group [2][NC] squared column norms (epilogue)
    unsigned char *mail;  // per CTA [NBOX] outgoing panels
    int ngroups;
};
constexpr int CT_VERD = 96, CT_EPI = 160, CT_WORK = 192, CT_META = 256, CT_BYTES = 512;
// VERD/EPI/WORK: [2] by parity; META: [16] 64-bit exchange flags by exchange number mod 16 -- low word the
// exchange number (the outgoing panel is in its mailbox), high word the panel's modified / tested stamps
// (16 bits each), so one release store publishes both and the receiver's acquire load returns both
// mailboxes per CTA: exchange e writes mailbox e % NBOX.  A sweep has 2C-2
// exchanges and ends with a group-wide verdict barrier, so a mailbox is
// rewritten (NBOX >= 2C-1 exchanges later) only after every CTA of the group
// passed a verdict that its receiver posted after consuming it: no
// acknowledgement flags are needed.  (Cfg::NBOX: the power of two >= 2C-1.)

// MR x NC working blocks; VEC: V rows (NC of them) ride along under the X
// rows (vectors requested), else the panels hold X only (sigma-only solves)
template <int MR, int NC, bool VEC>
struct Cfg {
    static constexpr int C = NC / N2;
    static constexpr int STEPS = 2 * C - 1;
    static constexpr int NBOX = STEPS <= 16 ? 16 : 32;
    static constexpr int ROWS = MR + (VEC ? NC : 0);
    static constexpr uint32_t SLOT = ROWS * 128;  // one panel: W complex = 32 real columns, SW128 K-major
    static constexpr uint32_t XBYTES = MR * 128;  // its X rows (the V rows follow)
    static constexpr int STAGES = MR / 64;        // Gram stages of 64 X rows
    static constexpr int MBLK = ROWS / 128;       // update M-blocks
    static constexpr int NBAR = 6 + STAGES;       // [0,1] update ring, [3] V in, [4,5] Gram ring, [6..] X in by stage
    static constexpr uint32_t SIG_OFF = 3 * SLOT;
    static constexpr uint32_t PERM_OFF = SIG_OFF + NC * 4;
    static constexpr uint32_t FLAG_OFF = PERM_OFF + 2 * NC * 4;
    static constexpr uint32_t RED_OFF = FLAG_OFF + 32 * 4;  // flags[16..31]: per-step cross-test stamps
    static constexpr uint32_t BAR_OFF = (RED_OFF + 64 * 4 + 15) & ~15u;
    static constexpr uint32_t TM_OFF = BAR_OFF + NBAR * 8;
    static constexpr uint32_t SMEM = TM_OFF + 16;
    static_assert(MR % 64 == 0 && ROWS % 128 == 0 && NC % N2 == 0, "tcb shape");
    static_assert(SLOT == 65536, "tcb panel slot = the 64 KB Gram/update scratch = one mailbox line per thread");
    static_assert(MBLK <= 4, "tcb TMEM budget (4 update accumulators of 128 columns)");
    static_assert(2 * NC >= 512, "the Gram norm partials reuse the permutation scratch");
    static_assert(C >= 2 && C <= MAXC, "tcb group size");
    static_assert(NBOX >= STEPS, "mailbox reuse must cross a sweep-verdict barrier");
    static_assert(STEPS <= 16, "per-step stamps: 16 shared-memory words (flags[16..31])");
    static_assert(SMEM <= 227 * 1024, "tcb shared memory");
};

// byte offset of (row r, real column k < 32) inside one panel slot, and of
// the 16-byte chunk k4 < 8 of row r (the pair layout of cs_tcb.cuh, one atom)
__device__ __forceinline__ uint32_t so(int r, int k) { return sw_off(r, k, 0); }
__device__ __forceinline__ uint32_t so4(int r, int k4) { return sw_chunk(r, k4, 0); }

// scratch offsets inside the scratch slot during the rotation phase (bytes)
// (HH, HL: real 64 x 65 partial Grams read from TMEM; dead once G is built)
constexpr uint32_t SC_D = 0, SC_PRM = 8448, SC_E = 16384, SC_T = 24832, SC_HH = 0, SC_HL = 16640, SC_G = 33792,
                   SC_BOP = 32768;
constexpr int LDR = 65;

// ---- global-memory flags and TMA bulk copies ------------------------------
__device__ __forceinline__ unsigned ld_acq(const void *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel(void *p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acq64(const void *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel64(void *p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void bulk_s2g(void *dst, uint32_t src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(mbar)
                 : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_but1() { asm volatile("cp.async.bulk.wait_group 1;" ::: "memory"); }

// a group peer that never arrives (it cannot: the launch is cooperative)
// must not hang the GPU: trap after ~10 s of polling
__device__ __noinline__ void spin_timeout(int what) {
    printf("jacobi_tcb_kernel: block %d timed out waiting on a group peer (%d)\n", (int)blockIdx.x, what);
    __trap();
}
__device__ __forceinline__ void spin_ge(const void *p, unsigned v, int what) {
    unsigned n = 0;
    while ((int)(ld_acq(p) - v) < 0) {
        if (++n > (1u << 25)) spin_timeout(what);
        __nanosleep(32);
    }
}
// exchange flag: low word = the exchange number, high word = the panel's stamps
__device__ __forceinline__ unsigned long long spin_ge64(const void *p, unsigned v, int what) {
    unsigned n = 0;
    unsigned long long x;
    while ((int)((unsigned)(x = ld_acq64(p)) - v) < 0) {
        if (++n > (1u << 25)) spin_timeout(what);
        __nanosleep(32);
    }
    return x;
}
__device__ __forceinline__ unsigned spin_tag(const void *p, unsigned tag, int what) {
    unsigned n = 0, v;
    while (((v = ld_acq(p)) >> 2) != tag) {
        if (++n > (1u << 25)) spin_timeout(what);
        __nanosleep(32);
    }
    return v;
}

// C = s * A B (+ I) on 32 x 32 complex matrices in shared memory (stride LDG).
// Register-blocked: each of the first 256 threads owns rows (i, i+16) x
// columns (j, j+16), so every shared-memory load feeds two complex MACs (the
// one-output-pair-per-thread form was shared-memory bound: 23.8k cycles per
// exp(E) with ~14 of these products).  C must not alias A or B.
__device__ __forceinline__ void cgemm32(const float2 *A, const float2 *B, float2 *Cm, float s, bool addI) {
    const int t = threadIdx.x;
    if (t >= 256) return;
    const int i = t >> 4, j = t & 15;
    float2 c[2][2];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) c[u][v] = make_float2(0.f, 0.f);
#pragma unroll 4
    for (int k = 0; k < N2; ++k) {
        float2 a[2], bb[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            a[u] = A[(i + 16 * u) * LDG + k];
            bb[u] = B[k * LDG + j + 16 * u];
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                c[u][v].x = fmaf(a[u].x, bb[v].x, fmaf(-a[u].y, bb[v].y, c[u][v].x));
                c[u][v].y = fmaf(a[u].x, bb[v].y, fmaf(a[u].y, bb[v].x, c[u][v].y));
            }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            float2 r = make_float2(c[u][v].x * s, c[u][v].y * s);
            if (addI && i + 16 * u == j + 16 * v) r.x += 1.f;
            Cm[(i + 16 * u) * LDG + j + 16 * v] = r;
        }
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

// Gram stage: rows [r0, r0+64) of the X rows of the pair (a: real columns
// 0..31, b: 32..63) -> the transposed hi|lo staging S (cs_tcb.cuh gram_stage)
// with MN rows ordered [hi_a | lo_a | hi_b | lo_b] (32 each), so the cross
// block needs only S x [hi_b | lo_b]^T (M = 128, N = 64).  Also accumulates
// this thread's share of the exact fp32 squared norm of real column
// tid & 63 (the Gram diagonal).
// The thread's addresses are stage-independent up to a constant: thread tid
// handles real column j = tid & 63 and the row quads q0 = tid >> 6 and q0 + 8
// of every stage, so the four swizzled load offsets and the store offset are
// computed once per Gram (GramThr) instead of per stage -- the staging loop is
// instruction-issue bound.
struct GramThr {
    const unsigned char *src;  // the column's panel + this thread's row-group offset
    uint32_t ld[4];            // byte offsets of rows 4 q0 + d of a stage (row quad q0 + 8: + 4096)
    uint32_t st;               // byte offset of the hi unit in the staging (lo: + 4096; row quad q0 + 8: + 16384)
};
__device__ __forceinline__ GramThr gram_thr(const unsigned char *Pa, const unsigned char *Pb) {
    static_assert(NT == 512, "gram staging: 64 columns x 8 row quads per pass");
    const int j = threadIdx.x & 63, q0 = threadIdx.x >> 6, k = j & 31;
    GramThr g;
    g.src = j < 32 ? Pa : Pb;
#pragma unroll
    for (int d = 0; d < 4; ++d) g.ld[d] = so(4 * q0 + d, k);
    const int hrow = j + (j & 32);  // hi_a 0..31, hi_b 64..95; lo 32 rows further
    g.st = sw_chunk(hrow, q0, 16384);
    return g;
}
__device__ __forceinline__ void gram_stage2(const GramThr &g, int st, unsigned char *stg, float &nsq) {
    const unsigned char *src = g.src + st * 8192;  // 64 rows = 8 row groups of 1 KB
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        float4 h;
        h.x = *reinterpret_cast<const float *>(src + i * 4096 + g.ld[0]);
        h.y = *reinterpret_cast<const float *>(src + i * 4096 + g.ld[1]);
        h.z = *reinterpret_cast<const float *>(src + i * 4096 + g.ld[2]);
        h.w = *reinterpret_cast<const float *>(src + i * 4096 + g.ld[3]);
        nsq = fmaf(h.x, h.x, fmaf(h.y, h.y, fmaf(h.z, h.z, fmaf(h.w, h.w, nsq))));
        // round-to-nearest split (hi symmetric around x): the dropped lo*lo
        // term is then unbiased
        const float4 hr = make_float4(rna_tf32(h.x), rna_tf32(h.y), rna_tf32(h.z), rna_tf32(h.w));
        const float4 lr = make_float4(rna_tf32(h.x - hr.x), rna_tf32(h.y - hr.y), rna_tf32(h.z - hr.z),
                                      rna_tf32(h.w - hr.w));
        *reinterpret_cast<float4 *>(stg + i * 16384 + g.st) = hr;
        *reinterpret_cast<float4 *>(stg + i * 16384 + g.st + 4096) = lr;
    }
}

template <int MR, int NC, bool VEC>
__global__ void __launch_bounds__(NT, 1) jacobi_tcb_kernel(const JacArgs<float> a, const Sched sc, const Ws ws) {
    using K = Cfg<MR, NC, VEC>;
    constexpr int C = K::C, STEPS = K::STEPS;
    constexpr uint32_t SLOT = K::SLOT, XBYTES = K::XBYTES;
    extern __shared__ __align__(1024) unsigned char sm[];
    float *sig2 = reinterpret_cast<float *>(sm + K::SIG_OFF);
    int *perm = reinterpret_cast<int *>(sm + K::PERM_OFF);
    int *flags = reinterpret_cast<int *>(sm + K::FLAG_OFF);
    float *red = reinterpret_cast<float *>(sm + K::RED_OFF);
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + K::BAR_OFF);  // [0,1] update ring, [3] V in, [4,5] Gram ring, [6..9] X in by stage
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sm + K::TM_OFF);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = blockIdx.x / C, rank = blockIdx.x % C;
    const float tol = a.tol;
    unsigned char *const myctl = ws.ctrl + (size_t)blockIdx.x * CT_BYTES;
    auto ctl = [&](int cta) { return ws.ctrl + ((size_t)g * C + cta) * CT_BYTES; };
    auto box = [&](int cta, int e) { return ws.mail + (((size_t)g * C + cta) * K::NBOX + (e % K::NBOX)) * SLOT; };
    float *const gsig = ws.gsig + (size_t)g * 2 * NC;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
        for (int i = 6; i < K::NBAR; ++i) mbar_init(&bar[i], 1);
        mbar_init(&bar[4], GW);  // one commit per Gram-issuing warp
        mbar_init(&bar[5], GW);
        fence_mbar_init();
    }
    __syncthreads();
    tc_after_sync();
    const uint32_t tmem = *tmem_slot;
    uint32_t ph1 = 0, ph2 = 0, phx = 0, phv = 0, pg0 = 0, pg1 = 0;  // mbarrier parities (CTA-uniform)
    auto ring_wait = [&](int slot) {
        if (slot == 0) { mbar_wait(&bar[0], ph1); ph1 ^= 1; }
        else { mbar_wait(&bar[1], ph2); ph2 ^= 1; }
    };
    auto gram_wait = [&](int slot) {
        if (slot == 0) { mbar_wait(&bar[4], pg0); pg0 ^= 1; }
        else { mbar_wait(&bar[5], pg1); pg1 ^= 1; }
    };
    unsigned epoch = 0, vseq = 0, mseq = 0;  // exchanges, sweeps, matrices of this launch (group-uniform)

    // dynamic schedule: the group's rank 0 takes the next matrix from a
    // launch-wide counter (sweep counts differ per matrix) and publishes it
    // to the group, tagged with the matrix sequence number
    unsigned *const next = reinterpret_cast<unsigned *>(ws.ctrl + (size_t)gridDim.x * CT_BYTES);
    for (;;) {
        if (tid == 0) {
            const unsigned slot = CT_WORK + 8 * ((mseq + 1) & 1);
            unsigned long long v;
            if (rank == 0) {
                const unsigned fi = atomicAdd(next, 1u);
                v = ((unsigned long long)(mseq + 1) << 32) | fi;
                asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(ctl(0) + slot), "l"(v) : "memory");
            } else {
                unsigned n = 0;
                for (;;) {
                    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctl(0) + slot) : "memory");
                    if ((unsigned)(v >> 32) == mseq + 1) break;
                    if (++n > (1u << 25)) spin_timeout(6);
                    __nanosleep(32);
                }
            }
            flags[2] = (int)(unsigned)v;
        }
        __syncthreads();
        const long long f = (unsigned)flags[2];
        __syncthreads();
        if (f >= a.count) break;
        const long long mid = a.index ? a.index[f] : f;
        ++mseq;
        // slots of panel a, panel b, scratch; stamps per role.  Scalars with selects, not arrays indexed by the
        // outgoing role: dynamically indexed arrays live in local memory (LDL / STL stalls at every super-round)
        int sl0 = 0, sl1 = 1, sl2 = 2;
        int ia = sc.ida[0][rank], ib = sc.idb[0][rank];
#ifdef CS_TCB_CLOCKS
        bool tcb_on = true;
        long long tcb_m = clock64();
        if (tid == 0) atomicAdd(&g_tcb_cycles[13], 1ull);
#else
        long long tcb_m = 0;
#endif
        // ---- load the two panels (panel x = working columns [x W, x W + W))
        {
            const float2 *X0 = a.initX ? a.initX + (size_t)f * MR * NC : nullptr;
            const float2 *V0 = a.initV ? a.initV + (size_t)a.initV_index[f] * NC * NC : nullptr;
            const float2 *A = a.blocks + (size_t)mid * a.co * a.ci;
            if (X0 && V0) {  // warm start: 16-byte loads (two complex columns), 16 in flight per thread
#pragma unroll 16
                for (int u = tid; u < 2 * K::ROWS * (W / 2); u += NT) {
                    const int half = u / (K::ROWS * (W / 2)), e = u % (K::ROWS * (W / 2));
                    const int r = e / (W / 2), j2 = e % (W / 2), j = (half == 0 ? ia : ib) * W + 2 * j2;
                    const float4 v = r < MR ? __ldg(reinterpret_cast<const float4 *>(X0 + (size_t)r * NC + j))
                                            : __ldg(reinterpret_cast<const float4 *>(V0 + (size_t)(r - MR) * NC + j));
                    *reinterpret_cast<float4 *>(sm + half * SLOT + so4(r, j2)) = v;
                }
            } else
            for (int half = 0; half < 2; ++half) {
                const int c0 = (half == 0 ? ia : ib) * W;
                unsigned char *P = sm + half * SLOT;
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
                    *reinterpret_cast<float2 *>(P + so(r, 2 * jj)) = v;
                }
            }
        }
        __syncthreads();

        TCB_ADD(10, tcb_m);
        int info = -1;
        bool wait_x = false, wait_v = false;  // incoming panel (in flight into slot a or b)
        // Skipping converged pair tests.  A pair block that passed its test at
        // super-round k and whose panels are unmodified since would pass the
        // identical (deterministic) test again, so its Gram, read-back and angles
        // are skipped -- results are bitwise those of testing.  Stamps (super-round
        // numbers of this matrix, group-uniform): per role the panel's last
        // modification and last within-panel test (they travel with the panel
        // through the exchange), per step this CTA's last cross test (CTA c meets
        // the same panel pair at step t in every sweep).
        unsigned sr = 0, mod0 = 0u, mod1 = 0u, wt0 = 0u, wt1 = 0u;
        // (CTA-uniform; in shared memory: every thread writes the same value, barriers separate it from the reads)
        volatile unsigned *const ctest = reinterpret_cast<volatile unsigned *>(flags) + 16;
        if (tid < K::STEPS) ctest[tid] = 0u;
        __syncthreads();
        int src_pending = 0;
        auto finish_v = [&]() {  // the incoming V rows have landed
            if (wait_v) {
                mbar_wait(&bar[3], phv);
                phv ^= 1;
                wait_v = false;
                // the mailbox is consumed: drop its dirty L2 lines instead of letting
                // them be written back to HBM (one 128-byte line per thread)
                static_assert(SLOT == NT * 128, "one mailbox line per thread");
                asm volatile("discard.global.L2 [%0], 128;" ::"l"(box(src_pending, epoch) + (size_t)tid * 128)
                             : "memory");
            }
        };
        // sweep verdicts (OR over the group, double-buffered by sweep parity) are
        // posted at the end of a sweep and collected after the first Gram and
        // angles of the next one: that super-round works on the pairing the
        // sweep ended on (odd sweeps run backwards) and changes no panel before
        // the collection, so the wait for the group's slowest CTA overlaps it
        bool vpend = false, stop = false;
        auto collect_verdict = [&]() {
#ifdef CS_TCB_CLOCKS
            const long long tv = clock64();
#endif
            if (warp == 0) {  // lane d polls CTA d: the C acquire loads overlap
                unsigned any = lane < C ? spin_tag(ctl(lane) + CT_VERD + 4 * (vseq & 1), vseq, 4) : 0u;
                any = __reduce_or_sync(0xffffffffu, any);
                if (lane == 0) flags[0] = (int)(any & 3u);
            }
            __syncthreads();
            const int v = flags[0];
            __syncthreads();
            TCB_ADD(11, tv);
            return v;  // bit 0: any rotation, bit 1: non-finite
        };
        for (int sweep = 0; sweep < a.max_sweeps && !stop; ++sweep) {
            const bool fwd = (sweep & 1) == 0;
            bool rot = false, bad = false;
#ifdef CS_TCB_CLOCKS
            tcb_on = sweep < CS_TCB_CLOCKS_SWEEPS;
#endif
#pragma unroll 1
            for (int i = 0; i < STEPS; ++i) {
                const int t = fwd ? i : STEPS - 1 - i;
                const bool full = (i == 0);
#ifdef CS_TCB_CLOCKS
                long long tcb_t = clock64();
                const long long tcb_t0 = tcb_t;
                if (tid == 0 && tcb_on) atomicAdd(&g_tcb_cycles[9], 1ull);
#endif
                unsigned char *const Pa = sm + sl0 * SLOT;
                unsigned char *const Pb = sm + sl1 * SLOT;
                unsigned char *const RG = sm + sl2 * SLOT;
                float2 *Dm = reinterpret_cast<float2 *>(RG + SC_D);
                float2 *Gm = reinterpret_cast<float2 *>(RG + SC_G);
                unsigned char *Bop = RG + SC_BOP;
                // the exchange after this super-round: outgoing role o, sender src
                const bool xchg = i < STEPS - 1;
                const int t2 = xchg ? (fwd ? t + 1 : t - 1) : t;
                const int o = (sc.ida[t2][rank] == ia) ? 1 : 0;
                unsigned char *const outbox = box(rank, epoch + 1);

                if (sr < 0xffffu) ++sr;  // stamps travel in 16 bits; saturated stamps never compare greater: no skips
                const unsigned mod_max = mod0 > mod1 ? mod0 : mod1;
                const bool skip = ctest[t] > mod_max && (!full || (wt0 > mod0 && wt1 > mod1));
                int any_rot = 0, any_big = 0, nact = 0;
                bool act_mine = false, mma_upd = false;  // this thread's pair rotates; the tensor-core update ran
                Prm<float> *prm = reinterpret_cast<Prm<float> *>(RG + SC_PRM);
                const int nround = full ? N2 - 1 : W;
                TCB_MARK(7);
                if (skip) {  // no test: only the incoming panel's X rows must land
                    if (wait_x) {
#pragma unroll 1
                        for (int st = 0; st < K::STAGES; ++st) mbar_wait(&bar[6 + st], phx);
                        phx ^= 1;
                        wait_x = false;
                        if constexpr (!VEC)
                            asm volatile("discard.global.L2 [%0], 128;" ::"l"(box(src_pending, epoch) + (size_t)tid * 128)
                                         : "memory");
                    }
                } else {
                // ---- (1) Gram: STAGES x 64 X rows, transposed hi|lo staging, 2-slot ring.
                // The 8 K-steps of a stage are issued by GW warps (2 each), warp w
                // accumulating its K-steps of every stage in accumulator w, so GW
                // MMA streams run side by side.
                float nsq = 0.f;
                const GramThr gthr = gram_thr(Pa, Pb);
#pragma unroll 1
                for (int st = 0; st < K::STAGES; ++st) {
                    const int slot = st & 1;
                    if (st >= 2) gram_wait(slot);
                    if (wait_x) mbar_wait(&bar[6 + st], phx);  // the incoming panel's rows of this stage
                    gram_stage2(gthr, st, RG + slot * 32768, nsq);
                    fence_proxy_async_smem();
                    __syncthreads();
                    if (warp < GW) {
                        if (lane == 0) {
                            tc_after_sync();
                            const uint32_t sa = smem_u32(RG + slot * 32768), d = tmem + 128 * warp;
#pragma unroll
                            for (int kk = 0; kk < 8 / GW; ++kk) {
                                const int ks = warp * (8 / GW) + kk;
                                const uint32_t o2 = (ks >> 2) * 16384 + (ks & 3) * 32;
                                const uint32_t acc = (st | kk) ? 1u : 0u;
                                if (full)  // S S^T: every block (within a, within b, cross)
                                    mma_tf32(d, desc_sw128(sa + o2), desc_sw128(sa + o2), IDESC_GRAM, acc);
                                else       // S [hi_b | lo_b]^T: the cross block
                                    mma_tf32(d, desc_sw128(sa + o2), desc_sw128(sa + 8192 + o2), IDESC_CROSS, acc);
                            }
                            mma_commit(&bar[4 + slot]);
                        }
                        __syncwarp();
                    }
                }
                reinterpret_cast<float *>(perm)[tid] = nsq;  // column tid & 63, row share tid >> 6
                if (wait_x) {
                    phx ^= 1;
                    wait_x = false;
                    if constexpr (!VEC)  // the whole mailbox has landed: drop its L2 lines
                        asm volatile("discard.global.L2 [%0], 128;" ::"l"(box(src_pending, epoch) + (size_t)tid * 128)
                                     : "memory");
                }
                if (K::STAGES >= 2) { gram_wait(K::STAGES & 1); gram_wait((K::STAGES + 1) & 1); }
                else gram_wait(0);
                tc_after_sync();
                TCB_MARK(0);
                // ---- (2) G (complex, 32 x 32) from the GW accumulators (summed in fp32).
                // TMEM lane = S row; S rows: hi(i) = i + (i & 32), lo(i) = hi(i) + 32
                // for real column i.  R = hi*hi + hi*lo + lo*hi.
                //   full:  T[i][k] = (S S^T)[hi(i)][k], k < 128   (lanes 0..31, 64..95)
                //          R[i][j] = T[i][hi(j)] + T[i][lo(j)] + T[j][lo(i)]
                //   cross: T0[i][k] = (S Sb^T)[i][k], k < 64  (hi_a rows, lanes 0..31)
                //          T1[i][k] = (S Sb^T)[32 + i][k], k < 32 (lo_a rows, lanes 32..63)
                //          R[i][32 + j] = T0[i][j] + T0[i][32 + j] + T1[i][j]
                // The diagonal is the exact fp32 column norms from the staging pass.
                {
                    float *T = reinterpret_cast<float *>(RG);
                    float *T0 = T, *T1 = T + 32 * 65;
                    const int q = warp & 3, cb = 32 * (warp >> 2);
                    const bool act_rd = full ? (q == 0 || q == 2) : ((q == 0 && cb < 64) || (q == 1 && cb == 0));
                    if (act_rd) {
                        float acc[32];
#pragma unroll
                        for (int i2 = 0; i2 < 32; ++i2) acc[i2] = 0.f;
#pragma unroll 1
                        for (int w = 0; w < GW; ++w) {
                            float v[16], w2[16];
                            tmem_ld16x2s(tmem + ((uint32_t)(32 * q) << 16) + 128 * w + cb, v, w2);
#pragma unroll
                            for (int i2 = 0; i2 < 16; ++i2) { acc[i2] += v[i2]; acc[16 + i2] += w2[i2]; }
                        }
                        float *dstp = full ? T + ((q == 0 ? 0 : 32) + lane) * 129 + cb
                                           : (q == 0 ? T0 + lane * 65 + cb : T1 + lane * 33);
#pragma unroll
                        for (int i2 = 0; i2 < 32; ++i2) dstp[i2] = acc[i2];
                    }
                    tc_before_sync();
                    __syncthreads();
                    const float *part = reinterpret_cast<const float *>(perm);
                    auto nrm = [&](int j) {
                        float sacc = 0.f;
#pragma unroll
                        for (int k = 0; k < NT / 64; ++k) sacc += part[j + 64 * k];
                        return sacc;
                    };
                    if (full) {
                        auto hi = [](int i) { return i + (i & 32); };
                        auto R = [&](int i2, int k) {
                            return T[i2 * 129 + hi(k)] + T[i2 * 129 + hi(k) + 32] + T[k * 129 + hi(i2) + 32];
                        };
                        for (int x = tid; x < N2 * N2; x += NT) {
                            const int c = x >> 5, j = x & 31;
                            // G_r = R[2c][2j] + R[2c+1][2j+1], G_i = R[2c][2j+1] - R[2c+1][2j]
                            Gm[c * LDG + j] = c == j ? make_float2(nrm(2 * c) + nrm(2 * c + 1), 0.f)
                                                     : make_float2(R(2 * c, 2 * j) + R(2 * c + 1, 2 * j + 1),
                                                                   R(2 * c, 2 * j + 1) - R(2 * c + 1, 2 * j));
                        }
                    } else {
                        auto R = [&](int i2, int k) { return T0[i2 * 65 + k] + T0[i2 * 65 + 32 + k] + T1[i2 * 33 + k]; };
                        if (tid < W * W) {
                            const int c = tid >> 4, d = tid & 15;
                            Gm[c * LDG + W + d] = make_float2(R(2 * c, 2 * d) + R(2 * c + 1, 2 * d + 1),
                                                              R(2 * c, 2 * d + 1) - R(2 * c + 1, 2 * d));
                        } else if (tid < W * W + N2) {
                            const int c = tid - W * W;
                            Gm[c * LDG + c] = make_float2(nrm(2 * c) + nrm(2 * c + 1), 0.f);
                        }
                    }
                    if (tid == 0) flags[6] = 0;  // the angles' block-wide tallies
                    __syncthreads();
                }
                // D starts from zero only where it is accumulated (the full rounds' product
                // form); the cross product form and exp(E) write every entry.  The tally
                // barrier below orders this before D is used.
                if (full)
                    for (int x = tid; x < N2 * LDG; x += NT) Dm[x] = make_float2(0.f, 0.f);
                TCB_MARK(1);
                // ---- (3) every pair's rotation from G at once (the reference's test
                // and root, rot_params), slot k of round r at prm[16 r + k]
                int act = 0;
                if (tid < nround * W) {
                    int p, qq;
                    inner_pair(full, tid % W, tid / W, p, qq);
                    const float2 gv = Gm[p * LDG + qq];
                    Rot<float> R;
                    const float al = Gm[p * LDG + p].x, be = Gm[qq * LDG + qq].x;
                    act = rot_params<float>(al, be, gv.x, gv.y, tol, R);
                    // "large": |gamma| / sqrt(alpha beta) > K3_TAU selects the exp combination
                    if (act > 0) act = (gv.x * gv.x + gv.y * gv.y > K3_TAU * K3_TAU * al * be) ? 2 : 1;
                    Prm<float> pm;
                    // a pair below the threshold is stored as the identity rotation, so the product form
                    // below needs no per-round selects (x + 0 = x exactly)
                    const bool on = act > 0;
                    pm.cm1 = on ? R.cm1 : 0.f; pm.wr = on ? R.wr : 0.f; pm.wi = on ? R.wi : 0.f; pm.act = act;
                    prm[tid] = pm;
                }
                {
                    // one barrier for the three block-wide tallies: rotating pairs (bits 0..15),
                    // warps with a large angle (16..23), warps with a non-finite pair (24..31)
                    const unsigned brot = __ballot_sync(0xffffffffu, act > 0);
                    const int wbig = __any_sync(0xffffffffu, act > 1), wbad = __any_sync(0xffffffffu, act < 0);
                    const int tally = __popc(brot) + (wbig << 16) + (wbad << 24);
                    if (lane == 0 && tally) atomicAdd(&flags[6], tally);
                    __syncthreads();
                    const int all = flags[6];
                    nact = all & 0xffff;
                    any_rot = nact > 0;
                    any_big = (all >> 16) & 0xff;
                    act_mine = act > 0;
                    if (all >> 24) bad = true;
                }
                ctest[t] = sr;
                if (full) wt0 = wt1 = sr;
                if (any_rot && !bad) mod0 = mod1 = sr;
                }  // !skip
                TCB_MARK(2);
                if (vpend) {  // the previous sweep's verdict, before this sweep changes anything
                    vpend = false;
                    const int v = collect_verdict();
                    if ((v & 2) || !(v & 1)) {
                        if (!(v & 2)) info = sweep;  // sweep `sweep - 1` (0-based) was rotation-free
                        stop = true;
                        break;
                    }
                }
                if (any_rot && !bad) {
                    rot = true;
#ifdef CS_TCB_CLOCKS
                    if (tid == 0 && tcb_on) atomicAdd(&g_tcb_cycles[any_big ? 15 : 14], 1ull);
#endif
#ifdef CS_TCB_CLOCKS
                    const long long tpf = clock64();
#endif
                    if (K3_SPARSE > 0 && !any_big && nact <= K3_SPARSE) {
                        // ---- (4s) a few rotating pairs (late sweeps): apply the rotations one
                        // after the other, in round order, to the panels themselves -- the same
                        // product Q of the rounds' rotations as (4a), without D and the
                        // tensor-core update.  A thread owns its rows through all rotations.
                        int *lst = reinterpret_cast<int *>(red);  // [0, 32) entries, [32, 48) per-warp counts
                        const unsigned bal = __ballot_sync(0xffffffffu, act_mine);
                        if (lane == 0) lst[32 + warp] = __popc(bal);
                        __syncthreads();
                        int base = 0;
                        for (int w2 = 0; w2 < warp; ++w2) base += lst[32 + w2];
                        if (act_mine) lst[base + __popc(bal & ((1u << lane) - 1u))] = tid;
                        finish_v();
                        __syncthreads();
#pragma unroll 1
                        for (int i2 = 0; i2 < nact; ++i2) {
                            const int e = lst[i2];
                            const Prm<float> pm = prm[e];
                            int p, qq;
                            inner_pair(full, e % W, e / W, p, qq);
                            unsigned char *const cp = (p < W ? Pa : Pb), *const cq = (qq < W ? Pa : Pb);
                            const int jp = 2 * (p & (W - 1)), jq = 2 * (qq & (W - 1));
                            Rot<float> R;
                            R.cm1 = pm.cm1; R.wr = pm.wr; R.wi = pm.wi;
                            for (int row = tid; row < K::ROWS; row += NT) {
                                float2 *xp = reinterpret_cast<float2 *>(cp + so(row, jp));
                                float2 *yp = reinterpret_cast<float2 *>(cq + so(row, jq));
                                float2 x = *xp, y = *yp;
                                rot_apply<float>(x, y, R);
                                *xp = x;
                                *yp = y;
                            }
                        }
                        __syncthreads();
#ifdef CS_TCB_CLOCKS
                        if (tid == 0 && tcb_on) atomicAdd(&g_tcb_cycles[29], 1ull);
                        TCB_ADD(30, tpf);
#endif
                        TCB_MARK(3);
                    } else {
                    mma_upd = true;
                    if (!any_big) {
                        // ---- (4a) small angles (every |gamma| / sqrt(alpha beta) <=
                        // GCHECK_TAU): D = Q - I for Q = the product of the rounds'
                        // rotations, D <- D J_r + (J_r - I).  Rows evolve independently,
                        // so the 16 threads of a row (half a warp) only sync warp-wide.
                        const int i2 = tid >> 4, k = tid & 15;
                        if (!full) {
                            // cross rounds: slot k pairs a-column k with b-column (k + r) mod W.
                            // Lane k of row i2's half-warp keeps D[i2][k] and the b-column of
                            // its current pair in registers; the b-columns move one lane down
                            // per round (after W rounds every lane holds its own again).
                            float2 x = make_float2(0.f, 0.f), y = x;
#pragma unroll 4
                            for (int r = 0; r < W; ++r) {
                                const Prm<float> pm = prm[r * W + k];
                                // branch-free (the lanes of a half-warp differ in act): inactive
                                // pairs are identity rotations (a warp-uniform skip of rounds
                                // without an active pair measured slower)
                                const int qq = W + ((k + r) & (W - 1));
                                Rot<float> R;
                                R.cm1 = pm.cm1; R.wr = pm.wr; R.wi = pm.wi;
                                rot_apply<float>(x, y, R);
                                if (i2 == k) { x.x += R.cm1; y.x += R.wr; y.y += R.wi; }
                                if (i2 == qq) { x.x -= R.wr; x.y += R.wi; y.x += R.cm1; }
                                y.x = __shfl_sync(0xffffffffu, y.x, (k + 1) & (W - 1), W);
                                y.y = __shfl_sync(0xffffffffu, y.y, (k + 1) & (W - 1), W);
                            }
                            Dm[i2 * LDG + k] = x;
                            Dm[i2 * LDG + W + k] = y;
                        } else {
#pragma unroll 1
                            for (int r = 0; r < nround; ++r) {
                                const Prm<float> pm = prm[r * W + k];
                                if (pm.act > 0) {
                                    int p, qq;
                                    inner_pair(full, k, r, p, qq);
                                    float2 x = Dm[i2 * LDG + p], y = Dm[i2 * LDG + qq];
                                    Rot<float> R;
                                    R.cm1 = pm.cm1; R.wr = pm.wr; R.wi = pm.wi;
                                    rot_apply<float>(x, y, R);
                                    if (i2 == p) { x.x += R.cm1; y.x += R.wr; y.y += R.wi; }
                                    if (i2 == qq) { x.x -= R.wr; x.y += R.wi; y.x += R.cm1; }
                                    Dm[i2 * LDG + p] = x;
                                    Dm[i2 * LDG + qq] = y;
                                }
                                __syncwarp();
                            }
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
                                const float fc = th / sn;
                                Em[p * LDG + qq] = make_float2(fc * pm.wr, fc * pm.wi);
                                Em[qq * LDG + p] = make_float2(-fc * pm.wr, fc * pm.wi);
                            }
                        }
                        __syncthreads();
#ifdef CS_TCB_CLOCKS
                        const long long te = clock64();
#endif
                        expm_minus_identity(Em, Tm, Dm, red);
                        TCB_ADD(16, te);
                    }
#ifdef CS_TCB_CLOCKS
                    if (!any_big) TCB_ADD(full ? 18 : 17, tpf);
#endif
                    TCB_MARK(3);
                    // ---- (5) B operand (D~, hi | lo) and (6) update P += P D
#ifdef CS_TCB_CLOCKS
                    long long tu = clock64();
#define TCB_UPD(i) do { TCB_ADD(i, tu); tu = clock64(); } while (0)
#else
#define TCB_UPD(i) do { } while (0)
#endif
                    build_bop<NT>(Dm, Bop);
                    finish_v();  // the V rows of an incoming panel are needed from here
                    fence_proxy_async_smem();  // the B operand is read by the tensor core
                    __syncthreads();
                    TCB_UPD(19);
                    // Warp-specialised pipeline over the 128-row M-blocks.  The A operands --
                    // the panel rows themselves (the tensor core truncates the fp32 word to
                    // tf32: "hi") and lo(P) -- go from registers into TENSOR MEMORY
                    // (tcgen05.st) and the MMAs read them from there: shared memory is the
                    // bound of the MMAs (K = 8 tf32, M = N = 128 with both operands in shared
                    // memory reads 8 KB per 64 cycles, the SM's whole 128 B/cycle), so a
                    // staged shared-memory copy of lo(P) (32 KB written and re-read per
                    // block) and the MMAs' own reads of the panel rows are what this saves;
                    // only the B operand (D~) still comes from shared memory.
                    //   warps 0-7 (stagers): block mb's operands -> TMEM, then one of them
                    //     issues its MMAs (each block's stream from its own warp,
                    //     tools/tc_rate_probe.cu);
                    //   warps 8-15 (epilogue): wait for block mb's MMAs, add its accumulator
                    //     (main + correction) to the panels -- the outgoing panel straight
                    //     to the mailbox.  TMEM reads run at 64 B/cycle (64 KB per block:
                    //     ~1k cycles), which the stagers' work now overlaps.
                    // TMEM: two accumulators [0, 256) and two operand blocks [256, 512)
                    // (hi | lo, 64 columns each), alternating by block.  A block's operands
                    // are restaged after its MMAs completed (mbarrier), an accumulator is
                    // overwritten after the epilogue warps read it (named barrier 2 + slot).
                    // bar[0/1] see two commits per update, so their phase parity at the
                    // start of an update is always 0: block mb completes phase (mb >> 1) & 1.
                    static_assert(K::MBLK == 4 && NT == 512, "update pipeline: 4 blocks, 8 + 8 warps");
                    constexpr uint32_t TM_OP = 256;
                    const int q = warp & 3, hsel = (warp >> 2) & 1;  // TMEM lane quarter; panel a / b (32 real columns)
                    unsigned char *const Ph = hsel ? Pb : Pa;
                    if (warp < 8) {
#pragma unroll 1
                        for (int mb = 0; mb < K::MBLK; ++mb) {
                            if (mb >= 2) mbar_wait(&bar[mb & 1], 0);  // block mb-2's MMAs done: its operand block is free
                            TCB_UPD(20);
                            const int row = mb * 128 + 32 * q + lane;
                            const uint32_t t0 = tmem + ((uint32_t)(32 * q) << 16) + TM_OP + 128 * (mb & 1) + 32 * hsel;
#pragma unroll
                            for (int hf = 0; hf < 2; ++hf) {
                                uint32_t hh[16], rr[16];
#pragma unroll
                                for (int u = 0; u < 4; ++u) {
                                    const float4 x = *reinterpret_cast<const float4 *>(Ph + so4(row, 4 * hf + u));
                                    const float4 l = lo4(x);
                                    hh[4 * u] = __float_as_uint(x.x);  // the raw word: the tensor core truncates it
                                    hh[4 * u + 1] = __float_as_uint(x.y);
                                    hh[4 * u + 2] = __float_as_uint(x.z);
                                    hh[4 * u + 3] = __float_as_uint(x.w);
                                    rr[4 * u] = __float_as_uint(l.x);
                                    rr[4 * u + 1] = __float_as_uint(l.y);
                                    rr[4 * u + 2] = __float_as_uint(l.z);
                                    rr[4 * u + 3] = __float_as_uint(l.w);
                                }
                                tmem_st16_nowait(t0 + 16 * hf, hh);
                                tmem_st16_nowait(t0 + 64 + 16 * hf, rr);
                            }
                            tmem_st_wait();
                            tc_before_sync();
                            named_sync(1, 256);  // the stagers
                            if (mb >= 2) named_sync(2 + (mb & 1), NT);  // the epilogue warps read accumulator mb & 1 (block mb-2)
                            TCB_UPD(21);
                            if (warp == mb) {
                                if (lane == 0) {
                                    tc_after_sync();
                                    const uint32_t d = tmem + 128 * (mb & 1), hi = tmem + TM_OP + 128 * (mb & 1), lo = hi + 64;
#pragma unroll
                                    for (int at = 0; at < 2; ++at) {
                                        const uint32_t bb = smem_u32(Bop) + at * 16384;
#pragma unroll
                                        for (int ks = 0; ks < 4; ++ks) {
                                            const uint64_t db = desc_sw128(bb + ks * 32);
                                            const uint32_t acc0 = (at | ks) ? 1u : 0u;
                                            mma_tf32_ts(d, hi + 32 * at + 8 * ks, db, IDESC_UPD, acc0);        // [hi*hi | hi*lo]
                                            mma_tf32_ts(d + 64, lo + 32 * at + 8 * ks, db, IDESC_UPD_LO, 1u);  // + lo*hi -> correction
                                        }
                                    }
                                    mma_commit(&bar[mb & 1]);
                                }
                                __syncwarp();
                            }
                            TCB_UPD(22);
                        }
                    } else {
#pragma unroll 1
                        for (int mb = 0; mb < K::MBLK; ++mb) {
                            mbar_wait(&bar[mb & 1], (uint32_t)(mb >> 1) & 1u);  // block mb's MMAs done
                            tc_after_sync();
                            const int row = mb * 128 + 32 * q + lane;
                            const bool out = xchg && hsel == o;  // the outgoing panel goes straight to the mailbox (same layout)
#pragma unroll
                            for (int hf = 0; hf < 2; ++hf) {
                                float v[16], vc[16];
                                tmem_ld16x2(tmem + ((uint32_t)(32 * q) << 16) + 128 * (mb & 1) + 32 * hsel + 16 * hf, v, vc);
#pragma unroll
                                for (int i2 = 0; i2 < 16; ++i2) v[i2] += vc[i2];
#pragma unroll
                                for (int u = 0; u < 4; ++u) {
                                    const uint32_t off = so4(row, 4 * hf + u);
                                    float4 *pp = reinterpret_cast<float4 *>(Ph + off);
                                    float4 x = *pp;
                                    x.x += v[4 * u]; x.y += v[4 * u + 1]; x.z += v[4 * u + 2]; x.w += v[4 * u + 3];
                                    if (out) __stcg(reinterpret_cast<float4 *>(outbox + off), x);
                                    else *pp = x;
                                }
                            }
                            if (mb < 2) {
                                tc_before_sync();
                                named_arrive(2 + (mb & 1), NT);  // accumulator mb & 1 may be overwritten (block mb+2)
                            }
                        }
                        tc_before_sync();
                    }
                    TCB_MARK(4);
                    }  // tensor-core update
                }
                finish_v();
                TCB_MARK(5);
                // ---- (8) exchange to the next pairing: keep one panel, send the other
                // to dst through this CTA's mailbox (written by the epilogue above
                // when the pair rotated, copied here otherwise), receive the new one
                // from src's mailbox into the scratch slot
                if (xchg) {
                    const int src = fwd ? sc.src[t][rank] : sc.dst[t2][rank];
                    if (!mma_upd) {
                        const float4 *sp = reinterpret_cast<const float4 *>(sm + (o ? sl1 : sl0) * SLOT);
                        float4 *dp = reinterpret_cast<float4 *>(outbox);
#pragma unroll 4
                        for (int u = tid; u < (int)(SLOT / 16); u += NT) __stcg(dp + u, sp[u]);
                    }
                    ++epoch;
                    __syncthreads();
#ifdef CS_TCB_CLOCKS
                    long long tx = clock64();
#define TCB_XCH(i) do { TCB_ADD(i, tx); tx = clock64(); } while (0)
                    if (tid == 0 && tcb_on) { atomicAdd(&g_tcb_cycles[23], (unsigned long long)(tx - tcb_t)); }
#else
#define TCB_XCH(i) do { } while (0)
#endif
                    if (tid == 32) {
                        // the release store after the CTA barrier publishes every thread's
                        // mailbox stores (release is cumulative over the barrier; one
                        // MEMBAR.ALL.GPU -- a separate __threadfence() first is a second,
                        // sequentially-consistent one: 2.6k cycles per exchange) together
                        // with the panel's stamps.  It waits ~1.6k cycles for the stores to
                        // drain, so a thread of another warp does it while thread 0 already
                        // waits for the sender.
                        fence_proxy_async_global();
                        st_rel64(myctl + CT_META + 8 * (epoch % 16),
                                 (unsigned long long)epoch | ((unsigned long long)((o ? mod1 : mod0) & 0xffffu) << 32) |
                                     ((unsigned long long)((o ? wt1 : wt0) & 0xffffu) << 48));
                    }
                    if (tid == 0) {
                        TCB_XCH(24);
                        const unsigned char *in = box(src, epoch);
                        const uint32_t is = smem_u32(sm + sl2 * SLOT);
#ifdef CS_TCB_CLOCKS
                        if ((int)((unsigned)ld_acq64(ctl(src) + CT_META + 8 * (epoch % 16)) - epoch) < 0)
                            if (tcb_on) atomicAdd(&g_tcb_cycles[28], 1ull);
#endif
                        const unsigned long long fx = spin_ge64(ctl(src) + CT_META + 8 * (epoch % 16), epoch, 2);
                        TCB_XCH(25);
                        flags[4] = (int)((fx >> 32) & 0xffffu);
                        flags[5] = (int)(fx >> 48);
                        fence_proxy_async_global();
                        TCB_XCH(26);
                        constexpr uint32_t XC = XBYTES / K::STAGES;  // the X rows of one Gram stage
#pragma unroll
                        for (int c = 0; c < K::STAGES; ++c) {
                            mbar_arrive_expect_tx(&bar[6 + c], XC);
                            bulk_g2s(is + c * XC, in + c * XC, XC, smem_u32(&bar[6 + c]));
                        }
                        if constexpr (VEC) {
                            mbar_arrive_expect_tx(&bar[3], SLOT - XBYTES);
                            bulk_g2s(is + XBYTES, in + XBYTES, SLOT - XBYTES, smem_u32(&bar[3]));
                        }
                    }
                    wait_x = true;
                    wait_v = VEC;
                    src_pending = src;
                    const int ns = sl2;
                    sl2 = o ? sl1 : sl0;
                    if (o) sl1 = ns;
                    else sl0 = ns;
                    ia = sc.ida[t2][rank];
                    ib = sc.idb[t2][rank];
                    __syncthreads();
                    if (o) { mod1 = (unsigned)flags[4]; wt1 = (unsigned)flags[5]; }  // the incoming panel's stamps
                    else { mod0 = (unsigned)flags[4]; wt0 = (unsigned)flags[5]; }
                } else {
                    __syncthreads();
                }
                TCB_MARK(6);
#ifdef CS_TCB_CLOCKS
                if (tid == 0) {
                    const int si = sweep < 15 ? sweep : 15;
                    atomicAdd(&g_tcb_sweep[0][si], (unsigned long long)(clock64() - tcb_t0));
                    atomicAdd(&g_tcb_sweep[1][si], 1ull);
                    if (any_rot && !bad) atomicAdd(&g_tcb_sweep[mma_upd ? 2 : 3][si], 1ull);
                }
#endif
            }
            if (stop) break;
            // ---- post this sweep's verdict; the last allowed sweep collects it here
            ++vseq;
            if (tid == 0)
                st_rel(myctl + CT_VERD + 4 * (vseq & 1), (vseq << 2) | (bad ? 2u : 0u) | (rot ? 1u : 0u));
            vpend = true;
            if (sweep + 1 == a.max_sweeps) {
                vpend = false;
                const int v = collect_verdict();
                if (!(v & 2) && !(v & 1)) info = sweep + 1;
            }
        }

#ifdef CS_TCB_CLOCKS
        tcb_m = clock64();
#endif
        // ---- epilogue: exact fp32 column norms of the local panels, gathered
        // over the group through global memory; stable descending order;
        // U = X / sigma, V
        float *gs = gsig + (mseq & 1) * NC;
        for (int c = warp; c < N2; c += NT / 32) {
            const int half = c / W, jj = c % W;
            const unsigned char *P = sm + (half == 0 ? sl0 : sl1) * SLOT;
            float acc = 0.f;
            for (int r = lane; r < MR; r += 32) {
                const float2 v = *reinterpret_cast<const float2 *>(P + so(r, 2 * jj));
                acc = fmaf(v.x, v.x, fmaf(v.y, v.y, acc));
            }
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            if (lane == 0) gs[(half == 0 ? ia : ib) * W + jj] = acc;
        }
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            st_rel(myctl + CT_EPI + 4 * (mseq & 1), mseq);
        }
        if (warp == 0) {
            __syncwarp();
            if (lane < C) spin_ge(ctl(lane) + CT_EPI + 4 * (mseq & 1), mseq, 5);
        }
        __syncthreads();
        for (int j = tid; j < NC; j += NT) sig2[j] = sqrtf(__ldcg(gs + j));
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
            const int c0 = (half == 0 ? ia : ib) * W;
            const unsigned char *P = sm + (half == 0 ? sl0 : sl1) * SLOT;
            if (a.Uw) {
                for (int idx = tid; idx < MR * W; idx += NT) {
                    const int r = idx / W, jj = idx % W, j = c0 + jj;
                    const float sj = sig2[j];
                    const float den = sj > 0.f ? sj : 1.f;
                    const float2 v = *reinterpret_cast<const float2 *>(P + so(r, 2 * jj));
                    a.Uw[((size_t)mid * MR + r) * NC + ipos[j]] = make_float2(__fdividef(v.x, den), __fdividef(v.y, den));
                }
            }
            if (a.Vw) {
                for (int idx = tid; idx < NC * W; idx += NT) {
                    const int r = idx / W, jj = idx % W, j = c0 + jj;
                    a.Vw[((size_t)mid * NC + r) * NC + ipos[j]] =
                        *reinterpret_cast<const float2 *>(P + so(MR + r, 2 * jj));
                }
            }
        }
        if (a.zero_sigma && rank == 0 && tid == 0) {
            int z = 0;
            for (int j = 0; j < NC; ++j) z |= !(sig2[j] > 0.f);
            a.zero_sigma[mid] = z;
        }
        __syncthreads();
        TCB_ADD(12, tcb_m);
    }
    tc_before_sync();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// circle-method round r, slot k -> panels (p, q) (cs_jacobi.cuh pair_cols)
static void pair_host(int k, int r, int np, int &p, int &q) {
    const int L = np - 1;
    int ca = 0;
    if (k != 0) {
        ca = k - 1 + r;
        if (ca >= L) ca -= L;
        ca += 1;
    }
    int cb = np - 2 - k + r;
    if (cb >= L) cb -= L;
    cb += 1;
    p = ca;
    q = cb;
}

// Pairings M_0..M_{2C-2} (circle method on panel labels) and, between
// consecutive ones, the exchange in which every CTA keeps one panel: walk
// each alternating cycle of M_t u M_{t+1}, the CTA keeping vertex v takes
// the M_{t+1} edge (v, w) and receives w from w's holder, which keeps its
// other panel.  Checked: every panel pair meets exactly once per sweep.
static bool build_sched(int C, Sched &s) {
    const int NP = 2 * C, S = NP - 1;
    if (C < 2 || C > MAXC) return false;
    s = Sched{};
    int hold[MAXC][2];
    for (int k = 0; k < C; ++k) {
        pair_host(k, 0, NP, hold[k][0], hold[k][1]);
        s.ida[0][k] = (signed char)hold[k][0];
        s.idb[0][k] = (signed char)hold[k][1];
    }
    for (int r = 0; r + 1 < S; ++r) {
        int partner[2 * MAXC], owner[2 * MAXC];
        for (int k = 0; k < C; ++k) {
            int p, q;
            pair_host(k, r + 1, NP, p, q);
            partner[p] = q;
            partner[q] = p;
            owner[hold[k][0]] = k;
            owner[hold[k][1]] = k;
        }
        bool done[MAXC] = {};
        int nh[MAXC][2];
        for (int c0 = 0; c0 < C; ++c0) {
            if (done[c0]) continue;
            int c = c0, kr = 1;  // CTA c keeps the panel in role kr
            for (int guard = 0;; ++guard) {
                if (guard > NP) return false;
                const int kv = hold[c][kr], w = partner[kv], c2 = owner[w];
                if (c2 == c || done[c]) return false;
                nh[c][kr] = kv;
                nh[c][1 - kr] = w;
                s.src[r][c] = (signed char)c2;
                s.dst[r][c2] = (signed char)c;
                done[c] = true;
                kr = hold[c2][0] == w ? 1 : 0;  // c2 sends w and keeps its other panel
                c = c2;
                if (c == c0) {
                    if (kr != 1) return false;
                    break;
                }
            }
        }
        for (int k = 0; k < C; ++k) {
            hold[k][0] = nh[k][0];
            hold[k][1] = nh[k][1];
            s.ida[r + 1][k] = (signed char)hold[k][0];
            s.idb[r + 1][k] = (signed char)hold[k][1];
        }
    }
    int seen[2 * MAXC][2 * MAXC] = {};
    for (int t = 0; t < S; ++t)
        for (int k = 0; k < C; ++k) {
            const int x = s.ida[t][k], y = s.idb[t][k];
            if (x == y) return false;
            ++seen[x < y ? x : y][x < y ? y : x];
        }
    for (int x = 0; x < NP; ++x)
        for (int y = x + 1; y < NP; ++y)
            if (seen[x][y] != 1) return false;
    return true;
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

template <int MR, int NC, bool VEC>
static size_t ws_bytes_for(int ngroups) {
    using K = Cfg<MR, NC, VEC>;
    return align256((size_t)ngroups * K::C * CT_BYTES + 256) + align256((size_t)ngroups * 2 * NC * sizeof(float)) +
           (size_t)ngroups * K::C * K::NBOX * K::SLOT;
}

static int max_groups(int C) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
    return sms / C;  // one CTA per SM (the three panel slots take ~200 KB)
}

template <int MR, int NC, bool VEC>
static int launch(const JacArgs<float> &a, void *wsp, size_t wsb, cudaStream_t st) {
    using K = Cfg<MR, NC, VEC>;
    static Sched sched;
    static int sched_ok = -1;
    if (sched_ok < 0) sched_ok = build_sched(K::C, sched) ? 1 : 0;
    if (!sched_ok) return fail(CS_EINVAL, "tcb SVD: exchange schedule construction failed");
    auto kern = jacobi_tcb_kernel<MR, NC, VEC>;
    CS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::SMEM));
    int per_sm = 0;
    CS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, K::SMEM));
    if (per_sm < 1) return fail(CS_ENOMEM, "tcb SVD: kernel does not fit on an SM");
    const long long ng = lmin(a.count, (long long)max_groups(K::C));
    if (ng < 1) return CS_OK;
    const size_t need = ws_bytes_for<MR, NC, VEC>(max_groups(K::C));
    if (!wsp || wsb < need) return fail(CS_ENOMEM, "tcb SVD: workspace too small (query cs_batched_svd_workspace)");
    unsigned char *base = (unsigned char *)wsp;
    Ws ws;
    ws.ctrl = base;
    ws.gsig = (float *)(base + align256((size_t)ng * K::C * CT_BYTES + 256));
    ws.mail = (unsigned char *)ws.gsig + align256((size_t)ng * 2 * NC * sizeof(float));
    ws.ngroups = (int)ng;
    CS_CUDA_TRY(cudaMemsetAsync(ws.ctrl, 0, (size_t)ng * K::C * CT_BYTES + 256, st));  // flags + work counter
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // the CTAs of a group must be co-resident
    attr[0].val.cooperative = 1;
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = K::SMEM;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3((unsigned)(ng * K::C));
    CS_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, a, sched, ws));
    return check_launch("jacobi_tcb_kernel");
}

}  // namespace tcb

// shapes the tensor-core blocked kernel is instantiated for (working
// orientation mr x nc, fp32): warm-started 256 x 256 + V (cfg5).  The
// kernel is written for sigma-only shapes too (VEC = false); 512 x 512
// sigma-only solves measured only 16% faster on cfg4 than the scalar kernel
// and drift further in energy over their ~12 cold sweeps (K3), so
// they stay on the scalar kernel.
bool tcb_supported(int mr, int nc, bool wantv) { return wantv && mr == 256 && nc == 256; }

size_t tcb_workspace(int mr, int nc, bool wantv) {
    if (!tcb_supported(mr, nc, wantv)) return 0;
    return tcb::ws_bytes_for<256, 256, true>(tcb::max_groups(tcb::Cfg<256, 256, true>::C));
}

#ifdef CS_TCB_CLOCKS
extern "C" int cs_debug_tcb_cycles(unsigned long long *out, int reset) {
    if (cudaDeviceSynchronize() != cudaSuccess) return 4;
    cudaMemcpyFromSymbol(out, tcb::g_tcb_cycles, sizeof(unsigned long long) * 32);
    if (reset) {
        unsigned long long z[32] = {};
        cudaMemcpyToSymbol(tcb::g_tcb_cycles, z, sizeof(z));
    }
    return 0;
}
extern "C" int cs_debug_tcb_sweeps(unsigned long long *out, int reset) {  // [4][16], see g_tcb_sweep
    if (cudaDeviceSynchronize() != cudaSuccess) return 4;
    cudaMemcpyFromSymbol(out, tcb::g_tcb_sweep, sizeof(unsigned long long) * 64);
    if (reset) {
        unsigned long long z[64] = {};
        cudaMemcpyToSymbol(tcb::g_tcb_sweep, z, sizeof(z));
    }
    return 0;
}
#endif

int tcb_dispatch(const JacArgs<float> &a, void *ws, size_t ws_bytes, cudaStream_t st) {
    if (a.s.mr == 256 && a.s.nc == 256 && a.Vw) return tcb::launch<256, 256, true>(a, ws, ws_bytes, st);
    return fail(CS_EINVAL, "tcb SVD: unsupported shape");
}

}  // namespace cs
