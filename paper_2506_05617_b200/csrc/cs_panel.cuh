// cs_panel.cuh -- K3: panel-blocked one-sided Jacobi for a cluster of C CTAs.
//
// Same rotation, tolerance and convergence rule as cs_jacobi.cuh (the
// reference's blocksvd.py:75-125 semantics); what changes is WHERE the data
// lives and hence which pair ordering is used.
//
// Data: the augmented working matrix [X; V] (mr + nc rows when vectors are
// requested, mr otherwise) has its ncp columns split into 2C panels of w
// columns.  CTA c of the cluster owns two whole panels ("a" and "b"), all
// rows -- so every (alpha, beta, gamma) reduction is local to one CTA
// (registers + warp shuffles), never across the cluster.  On B200 the
// cluster fabric moves only ~20 B/cycle/SM with ~300-cycle latency
// (tools/dsmem_bench.cu), so a per-round cross-CTA reduction cost more than
// the round itself; here the cluster exchanges whole panels only between
// super-rounds (once per w rounds), by per-thread DSMEM loads.
//
// Ordering (a block version of the circle method, every pair once per sweep):
//   sweep = [within-panel rounds: w-1 rounds, circle method inside each of
//            the CTA's two panels]
//         + 2C-1 super-rounds, each [w cross rounds a x b] followed (except
//           the last) by a panel rotation across the cluster (circle method
//           over 2C panel positions; position 0 never moves).
//   In cross round s, pair slot k rotates a_k (stationary: its rows live in
//   the slot's registers for the whole super-round) with b_{(k+s) mod w}
//   (read from and written back to shared memory).  w-1 + (2C-1) w = ncp-1
//   rounds of w pairs = all ncp(ncp-1)/2 pairs.
// Thread layout: slot k = tid / G (k < w), lane g = tid % G owns X rows
// g + G*i (i < RPLX) and V rows g + G*i (i < RPLV) of its two columns.
#pragma once

#include "cs_jacobi.cuh"

namespace cs {

#ifdef CS_PHASE_CLOCKS
// experiment builds only (tools/ab_build.sh with CS_AB_FLAGS=-DCS_PHASE_CLOCKS)
static __device__ unsigned long long g_phase_cycles[8];
#endif

// owner CTA of panel position p (CTA c holds positions c and 2C-1-c)
__device__ __forceinline__ int pos_owner(int p, int C) { return p < C ? p : 2 * C - 1 - p; }

// instantiations that carry the Gram convergence check (see gram_check)
template <typename T, int RPLX, int RPLV>
constexpr bool GCHECK_BUILT = RPLV > 0 && RPLX >= 8;

// 32-bit shared-memory accessors.  The hot loops walk a column with an
// opaque pointer bump (asm "+r") so the compiler keeps ONE live address per
// column instead of hoisting RPL runtime-strided addresses into registers.
template <typename T> struct SmemIO;
template <> struct SmemIO<float> {
    static __device__ __forceinline__ float2 ld(uint32_t a) {
        float2 v;
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a) : "memory");
        return v;
    }
    static __device__ __forceinline__ void st(uint32_t a, float2 v) {
        asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
    }
};
template <> struct SmemIO<double> {
    static __device__ __forceinline__ double2 ld(uint32_t a) {
        double2 v;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
        return v;
    }
    static __device__ __forceinline__ void st(uint32_t a, double2 v) {
        asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
    }
};

// call-free sqrt / quotient for the fp32 epilogue (IEEE slow paths are
// subroutine calls that cost spills in the whole kernel); fp64 stays IEEE
__device__ __forceinline__ float epi_sqrt(float x) { return x > 0.f ? x * nr_rsqrt(x) : 0.f; }
__device__ __forceinline__ double epi_sqrt(double x) { return sqrt(x); }
__device__ __forceinline__ float epi_div(float a, float b) { return __fdividef(a, b); }
__device__ __forceinline__ double epi_div(double a, double b) { return a / b; }

template <typename T, int N>
__device__ __forceinline__ void col_load(cplx_t<T> (&v)[N], uint32_t addr, uint32_t stride) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
        v[i] = SmemIO<T>::ld(addr);
        addr += stride;
        asm volatile("" : "+r"(addr));
    }
}
template <typename T, int N>
__device__ __forceinline__ void col_load_cluster(cplx_t<T> (&v)[N], uint32_t addr, uint32_t stride) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
        if constexpr (sizeof(T) == 4) {
            asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v[i].x), "=f"(v[i].y) : "r"(addr) : "memory");
        } else {
            asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v[i].x), "=d"(v[i].y) : "r"(addr) : "memory");
        }
        addr += stride;
        asm volatile("" : "+r"(addr));
    }
}
template <typename T, int N>
__device__ __forceinline__ void col_store(const cplx_t<T> (&v)[N], uint32_t addr, uint32_t stride) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
        SmemIO<T>::st(addr, v[i]);
        addr += stride;
        asm volatile("" : "+r"(addr));
    }
}

// within-panel rounds (w-1 rounds, circle method inside each of the CTA's two
// panels, both columns from shared memory); records the squared column norms
// of round 0 in sig2.  Returns bit0 = rotated, bit1 = non-finite.
// __noinline__: the two phases are register-allocated separately.
template <typename T, int C, int RPLX, int RPLV>
__device__ __noinline__ int panel_within(const JacShape &s, unsigned char *smem, cplx_t<T> *Abuf,
                                         cplx_t<T> *Bbuf, int start_a, int start_b, T tol) {
    using T2 = cplx_t<T>;
    constexpr bool WANTV = RPLV > 0;
    constexpr int RPLV1 = WANTV ? RPLV : 1;
    const int w = s.P, G = s.G, LD = s.ldx, VOFF = s.ldv;
    const int tid = threadIdx.x, k = tid / G, g = tid % G;
    const bool active = k < w;
    constexpr uint32_t T2SZ = sizeof(T2);
    const uint32_t rstride = (uint32_t)G * T2SZ;
    const uint32_t voff_b = (uint32_t)VOFF * T2SZ;
    const uint32_t colb = (uint32_t)LD * T2SZ;
    T *sig2 = reinterpret_cast<T *>(smem + s.off_sig);
    int *flags = reinterpret_cast<int *>(smem + s.off_mbar);
    bool rot = false, bad = false, big = false;
            {
                const int hw = w / 2;
                const int kk = k % hw;
                T2 *panel = (k < hw) ? Abuf : Bbuf;
                const int pid = (k < hw) ? start_a : start_b;
#pragma unroll 1
                for (int r = 0; r < w - 1; ++r) {
                    int p = 0, q = 0;
                    T2 x[RPLX], y[RPLX], xv[RPLV1], yv[RPLV1];
                    T al = 0, be = 0, gr = 0, gi = 0;
                    if (active) {
                        pair_cols(kk, r, w, p, q);
                        const uint32_t ap = smem_u32(panel) + p * colb + g * T2SZ;
                        const uint32_t aq = smem_u32(panel) + q * colb + g * T2SZ;
                        col_load<T, RPLX>(x, ap, rstride);
                        col_load<T, RPLX>(y, aq, rstride);
#pragma unroll
                        for (int i = 0; i < RPLX; ++i) {
                            al = fma(x[i].y, x[i].y, fma(x[i].x, x[i].x, al));
                            be = fma(y[i].y, y[i].y, fma(y[i].x, y[i].x, be));
                            gr = fma(x[i].y, y[i].y, fma(x[i].x, y[i].x, gr));
                            gi = fma(-x[i].y, y[i].x, fma(x[i].x, y[i].y, gi));
                        }
                    }
#pragma unroll
                    for (int off = 16; off >= 1; off >>= 1) {
                        if (off < G) {
                            al += __shfl_xor_sync(0xffffffffu, al, off);
                            be += __shfl_xor_sync(0xffffffffu, be, off);
                            gr += __shfl_xor_sync(0xffffffffu, gr, off);
                            gi += __shfl_xor_sync(0xffffffffu, gi, off);
                        }
                    }
                    if (active) {
                        if (r == 0 && g == 0) {
                            sig2[pid * w + p] = al;
                            sig2[pid * w + q] = be;
                        }
                        Rot<T> R;
                        const int act = rot_params<T>(al, be, gr, gi, tol, R);
                        if (act < 0) {
                            bad = true;
                        } else if (act > 0) {
                            rot = true;
                            if constexpr (GCHECK_BUILT<T, RPLX, RPLV>) big |= act > 1;
                            const uint32_t ap = smem_u32(panel) + p * colb + g * T2SZ;
                            const uint32_t aq = smem_u32(panel) + q * colb + g * T2SZ;
#pragma unroll
                            for (int i = 0; i < RPLX; ++i) rot_apply<T>(x[i], y[i], R);
                            col_store<T, RPLX>(x, ap, rstride);
                            col_store<T, RPLX>(y, aq, rstride);
                            if constexpr (WANTV) {  // V rows only after the decision
                                col_load<T, RPLV1>(xv, ap + voff_b, rstride);
                                col_load<T, RPLV1>(yv, aq + voff_b, rstride);
#pragma unroll
                                for (int i = 0; i < RPLV; ++i) rot_apply<T>(xv[i], yv[i], R);
                                col_store<T, RPLV1>(xv, ap + voff_b, rstride);
                                col_store<T, RPLV1>(yv, aq + voff_b, rstride);
                            }
                        }
                    }
                    __syncthreads();
                }
            }

    return (rot ? 1 : 0) | (bad ? 2 : 0) | (big ? 4 : 0);
}

// 2C-1 super-rounds of cross pairs a x b: the a panel lives in registers, b
// columns are read/written in shared memory; between super-rounds the panels
// rotate across the cluster (DSMEM pulls).  The current b buffer index is
// kept in flags[2].  Returns bit0 = rotated, bit1 = non-finite.
template <typename T, int C, int RPLX, int RPLV>
__device__ __noinline__ int panel_cross(const JacShape &s, unsigned char *smem, int rank,
                                        cplx_t<T> *Abuf, cplx_t<T> *Bbuf0, T tol) {
    using T2 = cplx_t<T>;
    constexpr bool WANTV = RPLV > 0;
    constexpr int RPLV1 = WANTV ? RPLV : 1;
    const int w = s.P, G = s.G, LD = s.ldx, VOFF = s.ldv;
    const int tid = threadIdx.x, k = tid / G, g = tid % G;
    const bool active = k < w;
    constexpr uint32_t T2SZ = sizeof(T2);
    const uint32_t rstride = (uint32_t)G * T2SZ;
    const uint32_t voff_b = (uint32_t)VOFF * T2SZ;
    const uint32_t colb = (uint32_t)LD * T2SZ;
    T *sig2 = reinterpret_cast<T *>(smem + s.off_sig);
    int *flags = reinterpret_cast<int *>(smem + s.off_mbar);
    bool rot = false, bad = false, big = false;
    int *pos = flags + 4;
    const size_t panel_elems = (size_t)w * LD;
    int bcur = flags[2];
    cplx_t<T> *Bbuf = Bbuf0 + (size_t)bcur * panel_elems;
            // ---- a panel -> registers -------------------------------------
            T2 ra[RPLX], rav[RPLV1];
            if (active) {
                const uint32_t aa = smem_u32(Abuf) + k * colb + g * T2SZ;
                col_load<T, RPLX>(ra, aa, rstride);
                if constexpr (WANTV) col_load<T, RPLV1>(rav, aa + voff_b, rstride);
            }

            // ---- 2C-1 super-rounds of cross pairs ---------------------------
#pragma unroll 1
            for (int t = 0; t < 2 * C - 1; ++t) {
#pragma unroll 1
                for (int sr = 0; sr < w; ++sr) {
                    int j = k + sr;
                    if (j >= w) j -= w;
                    T2 y[RPLX], yv[RPLV1];
                    T al = 0, be = 0, gr = 0, gi = 0;
                    const uint32_t ab = smem_u32(Bbuf) + j * colb + g * T2SZ;
                    if (active) {
                        col_load<T, RPLX>(y, ab, rstride);
#pragma unroll
                        for (int i = 0; i < RPLX; ++i) {
                            al = fma(ra[i].y, ra[i].y, fma(ra[i].x, ra[i].x, al));
                            be = fma(y[i].y, y[i].y, fma(y[i].x, y[i].x, be));
                            gr = fma(ra[i].y, y[i].y, fma(ra[i].x, y[i].x, gr));
                            gi = fma(-ra[i].y, y[i].x, fma(ra[i].x, y[i].y, gi));
                        }
                    }
#pragma unroll
                    for (int off = 16; off >= 1; off >>= 1) {
                        if (off < G) {
                            al += __shfl_xor_sync(0xffffffffu, al, off);
                            be += __shfl_xor_sync(0xffffffffu, be, off);
                            gr += __shfl_xor_sync(0xffffffffu, gr, off);
                            gi += __shfl_xor_sync(0xffffffffu, gi, off);
                        }
                    }
                    if (active) {
                        Rot<T> R;
                        const int act = rot_params<T>(al, be, gr, gi, tol, R);
                        if (act < 0) {
                            bad = true;
                        } else if (act > 0) {
                            rot = true;
                            if constexpr (GCHECK_BUILT<T, RPLX, RPLV>) big |= act > 1;
#pragma unroll
                            for (int i = 0; i < RPLX; ++i) rot_apply<T>(ra[i], y[i], R);
                            col_store<T, RPLX>(y, ab, rstride);
                            if constexpr (WANTV) {  // V rows only after the decision
                                col_load<T, RPLV1>(yv, ab + voff_b, rstride);
#pragma unroll
                                for (int i = 0; i < RPLV; ++i) rot_apply<T>(rav[i], yv[i], R);
                                col_store<T, RPLV1>(yv, ab + voff_b, rstride);
                            }
                        }
                    }
                    __syncthreads();
                }
                if constexpr (C > 1) {
                    if (t == 2 * C - 2) break;
                    // ---- panel rotation across the cluster --------------------
                    if (active) {  // a registers -> Abuf (peers may pull it)
                        const uint32_t aa = smem_u32(Abuf) + k * colb + g * T2SZ;
                        col_store<T, RPLX>(ra, aa, rstride);
                        if constexpr (WANTV) col_store<T, RPLV1>(rav, aa + voff_b, rstride);
                    }
                    cluster_sync_all();
                    cg::cluster_group cl = cg::this_cluster();
                    T2 *Bnext = Bbuf0 + (size_t)(bcur ^ 1) * panel_elems;
                    // new a: position rank <- rank+1 (CTA rank+1's a; CTA C-1 takes its own b)
                    if (rank != 0 && active) {
                        const uint32_t src = (rank == C - 1)
                                                 ? map_rank(smem_u32(Bbuf), rank)
                                                 : map_rank(smem_u32(Abuf), rank + 1);
                        const uint32_t aa = src + k * colb + g * T2SZ;
                        col_load_cluster<T, RPLX>(ra, aa, rstride);
                        if constexpr (WANTV) col_load_cluster<T, RPLV1>(rav, aa + voff_b, rstride);
                    }
                    // new b: position 2C-1-rank <- 2C-rank (CTA rank-1's b; CTA 0 takes CTA 1's a)
                    {
                        const T2 *src;
                        if (rank == 0) src = cl.map_shared_rank(Abuf, 1);
                        else src = cl.map_shared_rank(Bbuf0 + (size_t)bcur * panel_elems, rank - 1);
                        const float4 *s4 = reinterpret_cast<const float4 *>(src);
                        float4 *d4 = reinterpret_cast<float4 *>(Bnext);
                        const size_t n4 = panel_elems * sizeof(T2) / sizeof(float4);
                        for (size_t x = tid; x < n4; x += blockDim.x) d4[x] = s4[x];
                    }
                    int np = 0;
                    if (tid < 2 * C) np = (tid == 0) ? pos[0] : (tid == 2 * C - 1 ? pos[1] : pos[tid + 1]);
                    cluster_sync_all();
                    if (tid < 2 * C) pos[tid] = np;
                    bcur ^= 1;
                    Bbuf = Bnext;
                    if (tid == 0) flags[2] = bcur;
                    __syncthreads();
                }
            }
            // ---- a registers back to shared memory ---------------------------
            if (active) {
                const uint32_t aa = smem_u32(Abuf) + k * colb + g * T2SZ;
                col_store<T, RPLX>(ra, aa, rstride);
                if constexpr (WANTV) col_store<T, RPLV1>(rav, aa + voff_b, rstride);
            }
    return (rot ? 1 : 0) | (bad ? 2 : 0) | (big ? 4 : 0);
}


// ---------------------------------------------------------------------------
// Split-role variant (vectors requested): threads [0, wG) are X warps, threads
// [wG, 2wG) V warps.  X warps reduce and rotate the X rows and publish the
// rotation of every pair slot (prm, double-buffered by round parity); V warps
// apply the same rotation to the V rows ONE ROUND LATER.  V rows never enter
// a reduction, so this is exact reordering: twice the warps per SM with half
// the live registers each, and the V FMA work fills the X warps' shuffle /
// parameter latency.  Every phase runs one extra "drain" iteration.
// ---------------------------------------------------------------------------
template <typename T> struct __align__(16) Prm { T cm1, wr, wi; int act; };

template <typename T, int C, int RPLX, int RPLV>
__device__ __noinline__ int panel_within_split(const JacShape &s, unsigned char *smem,
                                               cplx_t<T> *Abuf, cplx_t<T> *Bbuf, int start_a,
                                               int start_b, T tol) {
    using T2 = cplx_t<T>;
    const int w = s.P, G = s.G, LD = s.ldx, VOFF = s.ldv;
    const bool xrole = (int)threadIdx.x < w * G;
    const int ltid = xrole ? threadIdx.x : threadIdx.x - w * G;
    const int k = ltid / G, g = ltid % G;
    const bool active = k < w;
    constexpr uint32_t T2SZ = sizeof(T2);
    const uint32_t rstride = (uint32_t)G * T2SZ;
    const uint32_t voff_b = (uint32_t)VOFF * T2SZ;
    const uint32_t colb = (uint32_t)LD * T2SZ;
    T *sig2 = reinterpret_cast<T *>(smem + s.off_sig);
    Prm<T> *prm = reinterpret_cast<Prm<T> *>(smem + s.off_recv);  // [2][w]
    bool rot = false, bad = false;
    const int hw = w / 2;
    const int kk = k % hw;
    T2 *panel = (k < hw) ? Abuf : Bbuf;
    const int pid = (k < hw) ? start_a : start_b;
#pragma unroll 1
    for (int r = 0; r < w; ++r) {  // w-1 rounds + 1 drain
        if (xrole) {
            T al = 0, be = 0, gr = 0, gi = 0;
            int p = 0, q = 0;
            T2 x[RPLX], y[RPLX];
            const bool live = active && r < w - 1;
            if (live) {
                pair_cols(kk, r, w, p, q);
                col_load<T, RPLX>(x, smem_u32(panel) + p * colb + g * T2SZ, rstride);
                col_load<T, RPLX>(y, smem_u32(panel) + q * colb + g * T2SZ, rstride);
#pragma unroll
                for (int i = 0; i < RPLX; ++i) {
                    al = fma(x[i].y, x[i].y, fma(x[i].x, x[i].x, al));
                    be = fma(y[i].y, y[i].y, fma(y[i].x, y[i].x, be));
                    gr = fma(x[i].y, y[i].y, fma(x[i].x, y[i].x, gr));
                    gi = fma(-x[i].y, y[i].x, fma(x[i].x, y[i].y, gi));
                }
            }
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) {
                if (off < G) {
                    al += __shfl_xor_sync(0xffffffffu, al, off);
                    be += __shfl_xor_sync(0xffffffffu, be, off);
                    gr += __shfl_xor_sync(0xffffffffu, gr, off);
                    gi += __shfl_xor_sync(0xffffffffu, gi, off);
                }
            }
            if (live) {
                if (r == 0 && g == 0) {
                    sig2[pid * w + p] = al;
                    sig2[pid * w + q] = be;
                }
                Rot<T> R;
                const int act = rot_params<T>(al, be, gr, gi, tol, R);
                if (g == 0) {
                    Prm<T> pm;
                    pm.cm1 = R.cm1; pm.wr = R.wr; pm.wi = R.wi; pm.act = act;
                    prm[(r & 1) * w + k] = pm;
                }
                if (act < 0) {
                    bad = true;
                } else if (act > 0) {
                    rot = true;
#pragma unroll
                    for (int i = 0; i < RPLX; ++i) rot_apply<T>(x[i], y[i], R);
                    col_store<T, RPLX>(x, smem_u32(panel) + p * colb + g * T2SZ, rstride);
                    col_store<T, RPLX>(y, smem_u32(panel) + q * colb + g * T2SZ, rstride);
                }
            }
        } else if (active && r >= 1) {  // V warps: round r-1
            const Prm<T> pm = prm[((r - 1) & 1) * w + k];
            if (pm.act > 0) {
                int p, q;
                pair_cols(kk, r - 1, w, p, q);
                Rot<T> R;
                R.cm1 = pm.cm1; R.wr = pm.wr; R.wi = pm.wi;
                T2 xv[RPLV], yv[RPLV];
                const uint32_t ap = smem_u32(panel) + p * colb + g * T2SZ + voff_b;
                const uint32_t aq = smem_u32(panel) + q * colb + g * T2SZ + voff_b;
                col_load<T, RPLV>(xv, ap, rstride);
                col_load<T, RPLV>(yv, aq, rstride);
#pragma unroll
                for (int i = 0; i < RPLV; ++i) rot_apply<T>(xv[i], yv[i], R);
                col_store<T, RPLV>(xv, ap, rstride);
                col_store<T, RPLV>(yv, aq, rstride);
            }
        }
        __syncthreads();
    }
    return (rot ? 1 : 0) | (bad ? 2 : 0);
}

template <typename T, int C, int RPLX, int RPLV>
__device__ __noinline__ int panel_cross_split(const JacShape &s, unsigned char *smem, int rank,
                                              cplx_t<T> *Abuf, cplx_t<T> *Bbuf0, T tol) {
    using T2 = cplx_t<T>;
    const int w = s.P, G = s.G, LD = s.ldx, VOFF = s.ldv;
    const int tid = threadIdx.x;
    const bool xrole = tid < w * G;
    const int ltid = xrole ? tid : tid - w * G;
    const int k = ltid / G, g = ltid % G;
    const bool active = k < w;
    constexpr uint32_t T2SZ = sizeof(T2);
    const uint32_t rstride = (uint32_t)G * T2SZ;
    const uint32_t voff_b = (uint32_t)VOFF * T2SZ;
    const uint32_t colb = (uint32_t)LD * T2SZ;
    const uint32_t roff = xrole ? 0u : voff_b;  // this role's rows inside a column
    int *flags = reinterpret_cast<int *>(smem + s.off_mbar);
    Prm<T> *prm = reinterpret_cast<Prm<T> *>(smem + s.off_recv);
    bool rot = false, bad = false;
    int *pos = flags + 4;
    const size_t panel_elems = (size_t)w * LD;
    int bcur = flags[2];
    T2 *Bbuf = Bbuf0 + (size_t)bcur * panel_elems;
    constexpr int RMAX = RPLX > RPLV ? RPLX : RPLV;
    // stationary a column rows of this role (X rows or V rows) in registers
    T2 ra[RMAX];
    if (active) {
        if (xrole) col_load<T, RPLX>(*reinterpret_cast<T2 (*)[RPLX]>(ra), smem_u32(Abuf) + k * colb + g * T2SZ, rstride);
        else col_load<T, RPLV>(*reinterpret_cast<T2 (*)[RPLV]>(ra), smem_u32(Abuf) + k * colb + g * T2SZ + voff_b, rstride);
    }
#pragma unroll 1
    for (int t = 0; t < 2 * C - 1; ++t) {
#pragma unroll 1
        for (int sr = 0; sr <= w; ++sr) {  // w rounds + 1 drain
            if (xrole) {
                T al = 0, be = 0, gr = 0, gi = 0;
                T2 y[RPLX];
                int j = k + sr;
                if (j >= w) j -= w;
                const bool live = active && sr < w;
                const uint32_t ab = smem_u32(Bbuf) + j * colb + g * T2SZ;
                if (live) {
                    col_load<T, RPLX>(y, ab, rstride);
#pragma unroll
                    for (int i = 0; i < RPLX; ++i) {
                        al = fma(ra[i].y, ra[i].y, fma(ra[i].x, ra[i].x, al));
                        be = fma(y[i].y, y[i].y, fma(y[i].x, y[i].x, be));
                        gr = fma(ra[i].y, y[i].y, fma(ra[i].x, y[i].x, gr));
                        gi = fma(-ra[i].y, y[i].x, fma(ra[i].x, y[i].y, gi));
                    }
                }
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) {
                    if (off < G) {
                        al += __shfl_xor_sync(0xffffffffu, al, off);
                        be += __shfl_xor_sync(0xffffffffu, be, off);
                        gr += __shfl_xor_sync(0xffffffffu, gr, off);
                        gi += __shfl_xor_sync(0xffffffffu, gi, off);
                    }
                }
                if (live) {
                    Rot<T> R;
                    const int act = rot_params<T>(al, be, gr, gi, tol, R);
                    if (g == 0) {
                        Prm<T> pm;
                        pm.cm1 = R.cm1; pm.wr = R.wr; pm.wi = R.wi; pm.act = act;
                        prm[(sr & 1) * w + k] = pm;
                    }
                    if (act < 0) {
                        bad = true;
                    } else if (act > 0) {
                        rot = true;
#pragma unroll
                        for (int i = 0; i < RPLX; ++i) rot_apply<T>(ra[i], y[i], R);
                        col_store<T, RPLX>(y, ab, rstride);
                    }
                }
            } else if (active && sr >= 1) {  // V warps: round sr-1
                const Prm<T> pm = prm[((sr - 1) & 1) * w + k];
                if (pm.act > 0) {
                    int j = k + sr - 1;
                    if (j >= w) j -= w;
                    Rot<T> R;
                    R.cm1 = pm.cm1; R.wr = pm.wr; R.wi = pm.wi;
                    T2 yv[RPLV];
                    const uint32_t ab = smem_u32(Bbuf) + j * colb + g * T2SZ + voff_b;
                    col_load<T, RPLV>(yv, ab, rstride);
#pragma unroll
                    for (int i = 0; i < RPLV; ++i) rot_apply<T>(ra[i], yv[i], R);
                    col_store<T, RPLV>(yv, ab, rstride);
                }
            }
            __syncthreads();
        }
        if constexpr (C > 1) {
            if (t == 2 * C - 2) break;
            // ---- panel rotation across the cluster (see panel_cross) ----------
            if (active) {
                if (xrole) col_store<T, RPLX>(*reinterpret_cast<T2 (*)[RPLX]>(ra), smem_u32(Abuf) + k * colb + g * T2SZ, rstride);
                else col_store<T, RPLV>(*reinterpret_cast<T2 (*)[RPLV]>(ra), smem_u32(Abuf) + k * colb + g * T2SZ + voff_b, rstride);
            }
            cluster_sync_all();
            cg::cluster_group cl = cg::this_cluster();
            T2 *Bnext = Bbuf0 + (size_t)(bcur ^ 1) * panel_elems;
            if (rank != 0 && active) {
                const uint32_t src = (rank == C - 1) ? map_rank(smem_u32(Bbuf), rank)
                                                     : map_rank(smem_u32(Abuf), rank + 1);
                const uint32_t aa = src + k * colb + g * T2SZ + roff;
                if (xrole) col_load_cluster<T, RPLX>(*reinterpret_cast<T2 (*)[RPLX]>(ra), aa, rstride);
                else col_load_cluster<T, RPLV>(*reinterpret_cast<T2 (*)[RPLV]>(ra), aa, rstride);
            }
            {
                const T2 *src;
                if (rank == 0) src = cl.map_shared_rank(Abuf, 1);
                else src = cl.map_shared_rank(Bbuf0 + (size_t)bcur * panel_elems, rank - 1);
                const float4 *s4 = reinterpret_cast<const float4 *>(src);
                float4 *d4 = reinterpret_cast<float4 *>(Bnext);
                const size_t n4 = panel_elems * sizeof(T2) / sizeof(float4);
                for (size_t x = tid; x < n4; x += blockDim.x) d4[x] = s4[x];
            }
            int np = 0;
            if (tid < 2 * C) np = (tid == 0) ? pos[0] : (tid == 2 * C - 1 ? pos[1] : pos[tid + 1]);
            cluster_sync_all();
            if (tid < 2 * C) pos[tid] = np;
            bcur ^= 1;
            Bbuf = Bnext;
            if (tid == 0) flags[2] = bcur;
            __syncthreads();
        }
    }
    if (active) {  // a rows back to shared memory
        if (xrole) col_store<T, RPLX>(*reinterpret_cast<T2 (*)[RPLX]>(ra), smem_u32(Abuf) + k * colb + g * T2SZ, rstride);
        else col_store<T, RPLV>(*reinterpret_cast<T2 (*)[RPLV]>(ra), smem_u32(Abuf) + k * colb + g * T2SZ + voff_b, rstride);
    }
    return (rot ? 1 : 0) | (bad ? 2 : 0);
}


// ---------------------------------------------------------------------------
// Gram-blocked cross phase ("blocked variant": the O(rows) work of a whole
// super-round becomes two GEMM-shaped passes).  Per super-round:
//   1. G = P^H P over the X rows of the CTA's two panels P = [a b] (2w x 2w,
//      Hermitian, 4x4 register tiles, row chunks reduced by warp shuffles);
//   2. the same w cross rounds of rotations run on G (two-sided: columns,
//      then rows) while D = Q - I accumulates the product Q of the rotations
//      (D <- D J + (J - I));
//   3. P <- P + P D for all X and V rows (register-streamed, in place).
// In exact arithmetic the rotations are those of the one-sided sweep; a
// rotation-free sweep makes no update, so convergence is still certified on
// freshly formed dot products.  The (Q - I) form keeps the rounding of the
// update relative to the (small) correction, as rot_apply does per rotation.
// Used when the 2w x 2w G and D fit next to the panels (w <= 16).
// ---------------------------------------------------------------------------
// phase 1: G = P^H P over the X rows (upper 4x4 tiles, 8 row chunks per tile
// reduced with warp shuffles); also clears D
template <typename T>
__device__ __noinline__ void gram_phase(unsigned char *smem, uint32_t abase, uint32_t bbase,
                                        int w, int LD, int mr, cplx_t<T> *Gm, cplx_t<T> *Dm) {
    using T2 = cplx_t<T>;
    const int n2 = 2 * w, ldg = n2 + 1, tid = threadIdx.x;
    const int ntile = n2 / 4, nup = ntile * (ntile + 1) / 2;
    // warp-uniform trip count: every lane runs the same iterations (shuffles)
    for (int base = 0; base < nup * 8; base += (int)blockDim.x) {
    const int item = base + tid;
    const int chunk = item & 7, tslot = item >> 3;
    int ti = 0, tj = 0;
    const bool tact = tslot < nup;
    if (tact) {
        int rem = tslot;
        while (rem >= ntile - ti) { rem -= ntile - ti; ++ti; }
        tj = ti + rem;
    }
    T gr[4][4], gi[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) gr[a][b] = gi[a][b] = (T)0;
    if (tact) {
        const int rows_per = (mr + 7) / 8;
        const int r0 = chunk * rows_per, r1 = min(mr, r0 + rows_per);
        const uint32_t colb = (uint32_t)LD * sizeof(T2);
        auto cbase = [&](int c) -> uint32_t { return c < w ? abase + c * colb : bbase + (c - w) * colb; };
        const uint32_t i0 = cbase(ti * 4), j0 = cbase(tj * 4);
        const bool icont = (ti * 4 + 3 < w) || (ti * 4 >= w);  // 4 columns in one panel
        const bool jcont = (tj * 4 + 3 < w) || (tj * 4 >= w);
        for (int r = r0; r < r1; ++r) {
            T2 xi[4], xj[4];
            const uint32_t ro = (uint32_t)r * sizeof(T2);
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                xi[a] = SmemIO<T>::ld((icont ? i0 + a * colb : cbase(ti * 4 + a)) + ro);
                xj[a] = SmemIO<T>::ld((jcont ? j0 + a * colb : cbase(tj * 4 + a)) + ro);
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) {  // conj(xi) * xj
                    gr[a][b] = fma(xi[a].y, xj[b].y, fma(xi[a].x, xj[b].x, gr[a][b]));
                    gi[a][b] = fma(-xi[a].y, xj[b].x, fma(xi[a].x, xj[b].y, gi[a][b]));
                }
        }
    }
#pragma unroll
    for (int off = 4; off >= 1; off >>= 1)
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                gr[a][b] += __shfl_xor_sync(0xffffffffu, gr[a][b], off);
                gi[a][b] += __shfl_xor_sync(0xffffffffu, gi[a][b], off);
            }
    if (tact && chunk == 0) {
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int i = ti * 4 + a, j = tj * 4 + b;
                Gm[(size_t)i * ldg + j] = mk<T>(gr[a][b], gi[a][b]);
                Gm[(size_t)j * ldg + i] = mk<T>(gr[a][b], -gi[a][b]);
            }
    }
    }
    for (int x = tid; x < n2 * n2; x += blockDim.x) Dm[(size_t)(x / n2) * ldg + (x % n2)] = mk<T>(0, 0);
}

// phase 2: the w cross rounds of rotations on G (two-sided), D <- D J + (J - I)
template <typename T>
__device__ __noinline__ int inner_phase(int w, cplx_t<T> *Gm, cplx_t<T> *Dm, Prm<T> *prm, T tol) {
    using T2 = cplx_t<T>;
    const int n2 = 2 * w, ldg = n2 + 1, tid = threadIdx.x, NT = blockDim.x;
    bool rot = false, bad = false;
#pragma unroll 1
    for (int sr = 0; sr < w; ++sr) {
        if (tid < w) {
            const int p = tid, q = w + ((tid + sr) % w);
            const T2 gpq = Gm[(size_t)p * ldg + q];
            Rot<T> R;
            const int act = rot_params<T>(Gm[(size_t)p * ldg + p].x, Gm[(size_t)q * ldg + q].x,
                                          gpq.x, gpq.y, tol, R);
            Prm<T> pm;
            pm.cm1 = R.cm1; pm.wr = R.wr; pm.wi = R.wi; pm.act = act;
            prm[tid] = pm;
            if (act < 0) bad = true;
            if (act > 0) rot = true;
        }
        __syncthreads();
        for (int x = tid; x < w * n2; x += NT) {  // columns p,q of G and D
            const int k = x / n2, i = x % n2;
            const Prm<T> pm = prm[k];
            if (pm.act <= 0) continue;
            const int p = k, q = w + ((k + sr) % w);
            Rot<T> R;
            R.cm1 = pm.cm1; R.wr = pm.wr; R.wi = pm.wi;
            T2 *gp = Gm + (size_t)i * ldg + p, *gq = Gm + (size_t)i * ldg + q;
            T2 u = *gp, v = *gq;
            rot_apply<T>(u, v, R);
            *gp = u; *gq = v;
            T2 *dp = Dm + (size_t)i * ldg + p, *dq = Dm + (size_t)i * ldg + q;
            u = *dp; v = *dq;
            rot_apply<T>(u, v, R);
            // + (J - I): J_pp = J_qq = 1 + cm1, J_qp = -conj(s ph), J_pq = s ph
            if (i == p) { u.x += R.cm1; v.x += R.wr; v.y += R.wi; }
            if (i == q) { u.x -= R.wr; u.y += R.wi; v.x += R.cm1; }
            *dp = u; *dq = v;
        }
        __syncthreads();
        for (int x = tid; x < w * n2; x += NT) {  // rows p,q of G: J^H G
            const int k = x / n2, j = x % n2;
            const Prm<T> pm = prm[k];
            if (pm.act <= 0) continue;
            const int p = k, q = w + ((k + sr) % w);
            Rot<T> R;
            R.cm1 = pm.cm1; R.wr = pm.wr; R.wi = pm.wi;
            T2 *gp = Gm + (size_t)p * ldg + j, *gq = Gm + (size_t)q * ldg + j;
            T2 u = *gp, v = *gq;
            u.y = -u.y; v.y = -v.y;
            rot_apply<T>(u, v, R);
            u.y = -u.y; v.y = -v.y;
            *gp = u; *gq = v;
        }
        __syncthreads();
    }
    return (rot ? 1 : 0) | (bad ? 2 : 0);
}

// phase 3: P <- P + P D for X rows and V rows, in place.  Two lanes per row
// (each producing half of the 2w outputs) read the whole row before writing.
template <typename T, int W>
__device__ __noinline__ void update_phase(uint32_t abase, uint32_t bbase, int LD, int mr,
                                          int nvr, int VOFF, const cplx_t<T> *Dm) {
    using T2 = cplx_t<T>;
    constexpr int w = W, n2 = 2 * W, ldg = n2 + 1;
    const int tid = threadIdx.x, NT = blockDim.x;
    const uint32_t colb = (uint32_t)LD * sizeof(T2);
    const int nrows = mr + nvr;
    for (int item = tid; item < 2 * ((nrows + 15) & ~15); item += NT) {
        const int rr = item >> 1, h = item & 1;
        const bool live = rr < nrows;
        const int row = rr < mr ? rr : VOFF + (rr - mr);
        const uint32_t ro = (uint32_t)row * sizeof(T2);
        T2 acc[W];
#pragma unroll
        for (int c = 0; c < W; ++c) acc[c] = mk<T>(0, 0);
        if (live) {
#pragma unroll 2
            for (int kk = 0; kk < n2; ++kk) {
                const uint32_t ca = kk < w ? abase + kk * colb : bbase + (kk - w) * colb;
                const T2 xv = SmemIO<T>::ld(ca + ro);
                const T2 *dk = Dm + (size_t)kk * ldg + h * w;
#pragma unroll
                for (int c = 0; c < W; ++c) {
                    const T2 d = dk[c];
                    acc[c].x = fma(xv.x, d.x, fma(-xv.y, d.y, acc[c].x));
                    acc[c].y = fma(xv.x, d.y, fma(xv.y, d.x, acc[c].y));
                }
            }
        }
        __syncwarp();  // the partner lane (other half of this row) has read the row
        if (live) {
            const uint32_t cb = h == 0 ? abase : bbase;
#pragma unroll
            for (int c = 0; c < W; ++c) {
                const uint32_t a = cb + c * colb + ro;
                T2 v = SmemIO<T>::ld(a);
                v.x += acc[c].x;
                v.y += acc[c].y;
                SmemIO<T>::st(a, v);
            }
        }
        __syncwarp();
    }
}

// the Gram-blocked cross phase (see the comment block above)
template <typename T, int C, int RPLX, int RPLV>
__device__ __noinline__ int panel_cross_gram(const JacShape &s, unsigned char *smem, int rank,
                                             cplx_t<T> *Abuf, cplx_t<T> *Bbuf0, T tol) {
    using T2 = cplx_t<T>;
    const int w = s.P, LD = s.ldx, VOFF = s.ldv;
    const int n2 = 2 * w, ldg = n2 + 1;
    const int mr = s.mr, nvr = s.Rv;
    const int tid = threadIdx.x, NT = blockDim.x;
    int *flags = reinterpret_cast<int *>(smem + s.off_mbar);
    int *pos = flags + 4;
    T2 *Gm = reinterpret_cast<T2 *>(smem + s.off_send);
    T2 *Dm = Gm + (size_t)n2 * ldg;
    Prm<T> *prm = reinterpret_cast<Prm<T> *>(smem + s.off_recv);
    int fl = 0;
    const size_t panel_elems = (size_t)w * LD;
    int bcur = flags[2];
    T2 *Bbuf = Bbuf0 + (size_t)bcur * panel_elems;
#pragma unroll 1
    for (int t = 0; t < 2 * C - 1; ++t) {
#ifdef CS_PHASE_CLOCKS
        long long c0 = clock64();
#endif
        gram_phase<T>(smem, smem_u32(Abuf), smem_u32(Bbuf), w, LD, mr, Gm, Dm);
        __syncthreads();
#ifdef CS_PHASE_CLOCKS
        long long c1 = clock64();
#endif
        const int f = inner_phase<T>(w, Gm, Dm, prm, tol);
        fl |= f;
#ifdef CS_PHASE_CLOCKS
        long long c2 = clock64();
#endif
        if (__syncthreads_or(f & 1)) {
            update_phase<T, 16>(smem_u32(Abuf), smem_u32(Bbuf), LD, mr, nvr, VOFF, Dm);
        }
        __syncthreads();
#ifdef CS_PHASE_CLOCKS
        if (threadIdx.x == 0) {  // per-phase cycle totals (tools/gram_split.py)
            long long c3 = clock64();
            atomicAdd(&g_phase_cycles[0], (unsigned long long)(c1 - c0));
            atomicAdd(&g_phase_cycles[1], (unsigned long long)(c2 - c1));
            atomicAdd(&g_phase_cycles[2], (unsigned long long)(c3 - c2));
        }
#endif
        if constexpr (C > 1) {
            if (t == 2 * C - 2) break;
            // panel rotation; the new a panel is staged through registers because
            // peers read this CTA's Abuf until the second cluster sync
            cluster_sync_all();
            cg::cluster_group cl = cg::this_cluster();
            T2 *Bnext = Bbuf0 + (size_t)(bcur ^ 1) * panel_elems;
            constexpr int STAGE = 16;
            T2 stage[STAGE];
            const int rows_real = mr + nvr;  // real rows per column (X then V)
            auto real_row = [&](int r) { return r < mr ? r : VOFF + (r - mr); };
            if (rank != 0) {
                const T2 *src = (rank == C - 1) ? Bbuf : cl.map_shared_rank(Abuf, rank + 1);
#pragma unroll
                for (int i = 0; i < STAGE; ++i) {
                    const int x = tid + i * NT;
                    if (x < w * rows_real) {
                        const int c = x / rows_real, r = real_row(x % rows_real);
                        stage[i] = src[(size_t)c * LD + r];
                    }
                }
            }
            {
                const T2 *src;
                if (rank == 0) src = cl.map_shared_rank(Abuf, 1);
                else src = cl.map_shared_rank(Bbuf0 + (size_t)bcur * panel_elems, rank - 1);
                const float4 *s4 = reinterpret_cast<const float4 *>(src);
                float4 *d4 = reinterpret_cast<float4 *>(Bnext);
                const size_t n4 = panel_elems * sizeof(T2) / sizeof(float4);
                for (size_t x = tid; x < n4; x += NT) d4[x] = s4[x];
            }
            int np = 0;
            if (tid < 2 * C) np = (tid == 0) ? pos[0] : (tid == 2 * C - 1 ? pos[1] : pos[tid + 1]);
            cluster_sync_all();
            if (rank != 0) {
#pragma unroll
                for (int i = 0; i < STAGE; ++i) {
                    const int x = tid + i * NT;
                    if (x < w * rows_real) {
                        const int c = x / rows_real, r = real_row(x % rows_real);
                        Abuf[(size_t)c * LD + r] = stage[i];
                    }
                }
            }
            if (tid < 2 * C) pos[tid] = np;
            bcur ^= 1;
            Bbuf = Bnext;
            if (tid == 0) flags[2] = bcur;
            __syncthreads();
        }
    }
    return fl;
}

// ---------------------------------------------------------------------------
// Gram convergence check.  A rotation-free sweep evaluates every pair (i, j)
// on the same, final columns: it is the test |x_i^H x_j|^2 <= tol^2 a_i a_j
// (rot_params) over the Gram matrix X^H X.  Computed blocked -- each warp a
// 4x4 sub-block of a w x w panel block, lanes splitting the rows, one
// transpose-reduce -- it costs a few percent of a sweep instead of the
// latency-bound rounds of a check sweep (~2/3 of a rotating one).  The CTAs
// of a cluster split the panel pairs: the three local blocks, all four blocks
// with the CTAs at cluster distance 1..(C-1)/2, and half of the four at
// distance C/2.  Remote panels are staged (X rows only) through the free
// exchange buffer.  Squared norms of the local columns land in sig2 where
// the epilogue gathers them.  Returns nonzero if some pair fails the test
// (or is non-finite): then the solve simply continues with the next sweep.
// ---------------------------------------------------------------------------
template <typename T, int NT>
__device__ __forceinline__ void gram_rows(const cplx_t<T> *const (&xp)[4],
                                          const cplx_t<T> *const (&yp)[4], int nt, T (&v)[32]) {
    // NT rows per lane: rows lane + 32 t, t < NT (NT == 0: none)
    using T2 = cplx_t<T>;
#pragma unroll
    for (int t = 0; t < (NT > 0 ? NT : 1); ++t) {
        if (NT == 0 && t >= nt) break;
        T2 xv[4], yv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            xv[u] = xp[u][t * 32];
            yv[u] = yp[u][t * 32];
        }
#pragma unroll
        for (int ii = 0; ii < 4; ++ii)
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                T &re = v[2 * (ii * 4 + jj)], &im = v[2 * (ii * 4 + jj) + 1];
                re = fma(xv[ii].y, yv[jj].y, fma(xv[ii].x, yv[jj].x, re));
                im = fma(-xv[ii].y, yv[jj].x, fma(xv[ii].x, yv[jj].y, im));
            }
    }
}

// rows % 64 == 0: every lane owns rows/32 rows, two per step (fast path)
template <typename T>
__device__ __forceinline__ void gram_block(const cplx_t<T> *X, int ldx, int px,
                                           const cplx_t<T> *Y, int ldy, int py, bool diag,
                                           int w, int rows, int nc, const T *nrm, T tol,
                                           bool &bad) {
    using T2 = cplx_t<T>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int nsub = (w + 3) / 4;
#pragma unroll 1
    for (int task = warp; task < nsub * nsub; task += nwarps) {
        const int i0 = (task / nsub) * 4, j0 = (task % nsub) * 4;
        if (diag && j0 + 3 <= i0) continue;  // strictly below the diagonal (warp-uniform)
        T v[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = 0;
        // columns past the panel edge are clamped (their entries are discarded)
        const T2 *xp[4], *yp[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            xp[u] = X + (size_t)min(i0 + u, w - 1) * ldx;
            yp[u] = Y + (size_t)min(j0 + u, w - 1) * ldy;
        }
        if ((rows & 63) == 0) {
            // one row per lane per step (rows % 64 == 0 keeps it branch-free).
            // Plain C++ loads: the same loop through the asm ld.shared accessors
            // (SmemIO) hung the <C=4, RPLX=8> instantiation (tools/_hang.py), and
            // two rows per step cost panel_cross 144 B of spills (ptxas splits
            // the kernel's 128 registers over its noinline phases).
            const T2 *xs[4], *ys[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                xs[u] = xp[u] + lane;
                ys[u] = yp[u] + lane;
            }
            const int nt = rows >> 5;
#pragma unroll 1
            for (int t = 0; t < nt; ++t) {
                T2 xv[4], yv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    xv[u] = xs[u][32 * t];
                    yv[u] = ys[u][32 * t];
                }
#pragma unroll
                for (int ii = 0; ii < 4; ++ii)
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) {
                        T &re = v[2 * (ii * 4 + jj)], &im = v[2 * (ii * 4 + jj) + 1];
                        re = fma(xv[ii].y, yv[jj].y, fma(xv[ii].x, yv[jj].x, re));
                        im = fma(-xv[ii].y, yv[jj].x, fma(xv[ii].x, yv[jj].y, im));
                    }
            }
        } else {
            // generic: rows r = lane + 32 t < rows; lanes past the end read row 0
            // (always in bounds) and add nothing
            const int nt = (rows + 31) / 32;
#pragma unroll 1
            for (int t = 0; t < nt; ++t) {
                const int r = lane + 32 * t;
                const bool ok = r < rows;
                const T2 *xq[4], *yq[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    xq[u] = xp[u] + (ok ? r : 0);
                    yq[u] = yp[u] + (ok ? r : 0);
                }
                T tmp[32];
#pragma unroll
                for (int e = 0; e < 32; ++e) tmp[e] = 0;
                gram_rows<T, 1>(xq, yq, 1, tmp);  // one row per lane
#pragma unroll
                for (int e = 0; e < 32; ++e) v[e] += ok ? tmp[e] : (T)0;
            }
        }
        // transpose-reduce: afterwards lane l holds the lane-sum of element l in v[0]
#pragma unroll
        for (int off = 16, n = 32; off >= 1; off >>= 1, n >>= 1) {
            const bool upper = lane & off;
#pragma unroll
            for (int e = 0; e < n / 2; ++e) {
                const T send = upper ? v[e] : v[e + n / 2];
                const T keep = upper ? v[e + n / 2] : v[e];
                v[e] = keep + __shfl_xor_sync(0xffffffffu, send, off);
            }
        }
        const T other = __shfl_xor_sync(0xffffffffu, v[0], 1);
        const int ent = lane >> 1, i = i0 + (ent >> 2), j = j0 + (ent & 3);
        if ((lane & 1) == 0 && i < w && j < w && (!diag || i < j)) {
            const int gi = px * w + i, gj = py * w + j;
            if (gi < nc && gj < nc) {
                const T q = v[0] * v[0] + other * other;
                const T ai = nrm[gi], aj = nrm[gj];
                if (!(isfinite(q) && isfinite(ai) && isfinite(aj))) bad = true;
                else if (ai != (T)0 && aj != (T)0 && !below_tol<T>(q, v[0], other, ai, aj, tol)) bad = true;
            }
        }
        // reconverge before the next task's shuffles: a warp left diverged here
        // can have lanes run ahead into a CTA barrier while the others wait in
        // a full-mask shuffle for them (observed as a hang on one instantiation)
        __syncwarp();
    }
}

template <typename T, int C>
__device__ __noinline__ int gram_check(const JacShape &s, unsigned char *smem, int rank,
                                       const cplx_t<T> *Abuf, const cplx_t<T> *Bbuf,
                                       cplx_t<T> *scratch, int rows, T tol) {
    using T2 = cplx_t<T>;
    const int w = s.P, LD = s.ldx, nc = s.nc, ncp = s.ncp;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    T *sig2 = reinterpret_cast<T *>(smem + s.off_sig);
    T *nrm = reinterpret_cast<T *>(smem + s.off_send);  // [ncp] squared norms, all columns
    int *flags = reinterpret_cast<int *>(smem + s.off_mbar);
    const int *pos = flags + 4;
    const int pa = pos[rank], pb = pos[2 * C - 1 - rank];

    // (1) squared norms of the local columns
#pragma unroll 1
    for (int c = warp; c < 2 * w; c += nwarps) {
        const T2 *col = (c < w ? Abuf : Bbuf) + (size_t)(c % w) * LD;
        T acc = 0;
        for (int r = lane; r < rows; r += 32) {
            const T2 v = col[r];
            acc = fma(v.y, v.y, fma(v.x, v.x, acc));
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) sig2[(c < w ? pa : pb) * w + c % w] = acc;
        __syncwarp();
    }
    if constexpr (C > 1) cluster_sync_all();
    else __syncthreads();
    // (2) every column's norm, from the CTA holding it
    for (int j = tid; j < ncp; j += blockDim.x) {
        const int panel = j / w;
        int p0 = 0;
        for (int p = 0; p < 2 * C; ++p)
            if (pos[p] == panel) p0 = p;
        const int owner = pos_owner(p0, C);
        if constexpr (C > 1)
            nrm[j] = (owner == rank) ? sig2[j] : cg::this_cluster().map_shared_rank(sig2, owner)[j];
        else
            nrm[j] = sig2[j];
    }
    __syncthreads();

    // (3) panel blocks
    bool bad = false;
    gram_block<T>(Abuf, LD, pa, Abuf, LD, pa, true, w, rows, nc, nrm, tol, bad);
    gram_block<T>(Bbuf, LD, pb, Bbuf, LD, pb, true, w, rows, nc, nrm, tol, bad);
    gram_block<T>(Abuf, LD, pa, Bbuf, LD, pb, false, w, rows, nc, nrm, tol, bad);
    if constexpr (C > 1) {
        cg::cluster_group cl = cg::this_cluster();
        // stage panel `which` (0 = a, 1 = b) of CTA d: rows [0, rows) into scratch
        auto stage = [&](int d, int which) -> int {
            __syncthreads();  // previous blocks done with scratch
            const T2 *src = cl.map_shared_rank(which == 0 ? Abuf : Bbuf, d);
            for (int idx = tid; idx < w * rows; idx += blockDim.x) {
                const int jj = idx / rows, r = idx - jj * rows;
                scratch[idx] = src[(size_t)jj * LD + r];
            }
            __syncthreads();
            return which == 0 ? pos[d] : pos[2 * C - 1 - d];
        };
#pragma unroll 1
        for (int dist = 1; 2 * dist < C; ++dist) {
            const int d = (rank + dist) % C;
#pragma unroll 1
            for (int which = 0; which < 2; ++which) {
                const int ps = stage(d, which);
                gram_block<T>(Abuf, LD, pa, scratch, rows, ps, false, w, rows, nc, nrm, tol, bad);
                gram_block<T>(Bbuf, LD, pb, scratch, rows, ps, false, w, rows, nc, nrm, tol, bad);
            }
        }
        if (C % 2 == 0) {  // distance C/2: the lower CTA takes its a panel x both,
            const int d = (rank + C / 2) % C;  // the upper one both panels x the lower's b
            if (rank < C / 2) {
#pragma unroll 1
                for (int which = 0; which < 2; ++which) {
                    const int ps = stage(d, which);
                    gram_block<T>(Abuf, LD, pa, scratch, rows, ps, false, w, rows, nc, nrm, tol, bad);
                }
            } else {
                const int ps = stage(d, 1);
                gram_block<T>(Abuf, LD, pa, scratch, rows, ps, false, w, rows, nc, nrm, tol, bad);
                gram_block<T>(Bbuf, LD, pb, scratch, rows, ps, false, w, rows, nc, nrm, tol, bad);
            }
        }
    }
    // (4) verdict, OR-ed over the cluster
    int any = __syncthreads_or(bad);
    if constexpr (C > 1) {
        if (tid == 0) flags[3] = any;
        cluster_sync_all();
        cg::cluster_group cl = cg::this_cluster();
        for (int d = 0; d < C; ++d) any |= cl.map_shared_rank(flags, d)[3];
        cluster_sync_all();
    }
    return any;
}

template <typename T, int C, int RPLX, int RPLV, bool SPLIT>
__global__ void __launch_bounds__(SPLIT ? 1024 : ((sizeof(T) == 8 && RPLX + RPLV > 8) ? 256 : JAC_MAX_THREADS))
jacobi_panel_kernel(const JacArgs<T> a) {
    using T2 = cplx_t<T>;
    constexpr bool WANTV = RPLV > 0;
    constexpr int RPLV1 = WANTV ? RPLV : 1;
    extern __shared__ __align__(16) unsigned char smem[];
    const JacShape &s = a.s;
    int rank = 0;
    if constexpr (C > 1) rank = (int)cg::this_cluster().block_rank();
    const long long cid = blockIdx.x / C;

    const int w = s.P;            // panel width (pairs per round)
    const int G = s.G;
    const int LD = s.ldx;         // column stride (complex) of [X rows | V rows]
    const int VOFF = s.ldv;       // row offset of the V rows inside a column
    const int ncp = s.ncp, nc = s.nc, mr = s.mr;
    const int tid = threadIdx.x, k = tid / G, g = tid % G;
    const bool active = k < w;
    const T tol = a.tol;

    T *sig2 = reinterpret_cast<T *>(smem + s.off_sig);            // [ncp] squared norms
    int *perm = reinterpret_cast<int *>(smem + s.off_perm);       // [2 ncp]
    int *flags = reinterpret_cast<int *>(smem + s.off_mbar);      // [4] rot, bad | [64] positions
    T2 *Abuf = reinterpret_cast<T2 *>(smem + s.off_x);            // [w][LD]
    T2 *Bbuf0 = reinterpret_cast<T2 *>(smem + s.off_v);           // [w][LD] (x2 when C>1)
    const size_t panel_elems = (size_t)w * LD;
    constexpr uint32_t T2SZ = sizeof(T2);
    const uint32_t rstride = (uint32_t)G * T2SZ;        // bytes between a lane's rows
    const uint32_t voff_b = (uint32_t)VOFF * T2SZ;       // byte offset of the V rows
    const uint32_t colb = (uint32_t)LD * T2SZ;           // bytes per column

    // panel ids by position (identical bookkeeping in every CTA) live in shared
    // memory: [0,32) current positions, [32,64) positions at sweep start
    int *pos = flags + 4;
    int *start_pos = flags + 4 + 32;
    for (long long f = cid; f < a.count; f += s.num_clusters) {
        if (tid < 32) pos[tid] = tid;
        if (tid == 0) flags[2] = 0;  // current b buffer
        __syncthreads();
        int bcur = 0;
        T2 *Bbuf = Bbuf0;

        // ---- load the two initial panels (a = panel rank, b = panel 2C-1-rank)
        const long long mid = a.index ? a.index[f] : f;  // matrix id (outputs too)
        {
            const T2 *A = a.blocks + (size_t)mid * a.co * a.ci;
            const T2 *X0 = a.initX ? a.initX + (size_t)f * mr * nc : nullptr;
            const T2 *V0 = a.initV ? a.initV + (size_t)a.initV_index[f] * nc * nc : nullptr;
            for (int half = 0; half < 2; ++half) {
                const int panel = half == 0 ? rank : 2 * C - 1 - rank;
                T2 *dst = half == 0 ? Abuf : Bbuf;
                const int c0 = panel * w;
                const int rows_x = G * RPLX;
                for (int idx = tid; idx < w * rows_x; idx += blockDim.x) {
                    int jj, r;
                    if (!s.wide || X0) { r = idx / w; jj = idx - r * w; }
                    else { jj = idx / rows_x; r = idx - jj * rows_x; }
                    const int j = c0 + jj;
                    T2 v = mk<T>(0, 0);
                    if (r < mr && j < nc) {
                        if (X0) v = X0[(size_t)r * nc + j];
                        else if (!s.wide) v = A[(size_t)r * a.ci + j];
                        else { v = A[(size_t)j * a.ci + r]; v.y = -v.y; }
                    }
                    dst[(size_t)jj * LD + r] = v;
                }
                if constexpr (WANTV) {
                    const int rows_v = G * RPLV;
                    for (int idx = tid; idx < w * rows_v; idx += blockDim.x) {
                        int jj, r;
                        if (V0) { r = idx / w; jj = idx - r * w; }
                        else { jj = idx / rows_v; r = idx - jj * rows_v; }
                        const int j = c0 + jj;
                        T2 v = mk<T>((r == j && r < nc) ? (T)1 : (T)0, 0);
                        if (V0) v = (r < nc && j < nc) ? V0[(size_t)r * nc + j] : mk<T>(0, 0);
                        dst[(size_t)jj * LD + VOFF + r] = v;
                    }
                }
            }
        }
        __syncthreads();

        int info = -1;
        for (int sweep = 0; sweep < a.max_sweeps; ++sweep) {
            if (a.dbg && tid == 0) *(volatile int *)&a.dbg[blockIdx.x] = 1000000 + 1000 * sweep;
            const int start_a = pos[rank];              // panel ids at the start of the sweep
            const int start_b = pos[2 * C - 1 - rank];
            __syncthreads();
            if (tid < 32) start_pos[tid] = pos[tid];

            int fl;
#ifdef CS_EXPERIMENTS  // slower opt-in variants: experiment builds only
            if constexpr (SPLIT) {
                fl = panel_within_split<T, C, RPLX, RPLV>(s, smem, Abuf, Bbuf, start_a, start_b, tol);
                fl |= panel_cross_split<T, C, RPLX, RPLV>(s, smem, rank, Abuf, Bbuf0, tol);
            } else if (s.gram) {
                fl = panel_within<T, C, RPLX, RPLV>(s, smem, Abuf, Bbuf, start_a, start_b, tol);
                fl |= panel_cross_gram<T, C, RPLX, RPLV>(s, smem, rank, Abuf, Bbuf0, tol);
            } else
#endif
            {
#ifdef CS_PHASE_CLOCKS
                long long c0 = clock64();
#endif
                fl = panel_within<T, C, RPLX, RPLV>(s, smem, Abuf, Bbuf, start_a, start_b, tol);
#ifdef CS_PHASE_CLOCKS
                long long c1 = clock64();
#endif
                fl |= panel_cross<T, C, RPLX, RPLV>(s, smem, rank, Abuf, Bbuf0, tol);
#ifdef CS_PHASE_CLOCKS
                if (tid == 0) {
                    atomicAdd(&g_phase_cycles[3], (unsigned long long)(c1 - c0));
                    atomicAdd(&g_phase_cycles[4], (unsigned long long)(clock64() - c1));
                }
#endif
            }
            bcur = flags[2];
            Bbuf = Bbuf0 + (size_t)bcur * panel_elems;
            const bool rot = fl & 1, bad = fl & 2, big = fl & 4;
            // ---- sweep verdict, OR-ed over the cluster ------------------------
            int any_bad = __syncthreads_or(bad);
            int any_rot = __syncthreads_or(rot);
            int any_big = __syncthreads_or(big);
            if constexpr (C > 1) {
                if (tid == 0) {
                    flags[0] = any_rot;
                    flags[1] = any_bad;
                    flags[3] = any_big;
                }
                cluster_sync_all();
                cg::cluster_group cl = cg::this_cluster();
                for (int d = 0; d < C; ++d) {
                    const int *pf = cl.map_shared_rank(flags, d);
                    any_rot |= pf[0];
                    any_bad |= pf[1];
                    any_big |= pf[3];
                }
                cluster_sync_all();
            }
            if (any_bad) break;
            if (!any_rot) {
                info = sweep + 1;
                break;
            }
            // no large rotation this sweep: the next one is likely rotation-free;
            // the Gram check decides that for a few percent of a sweep (counted
            // as one sweep, so max_sweeps keeps its meaning).  Compiled only
            // into the large vectors-requested instantiations: there it saves
            // ~6% (cfg5); elsewhere the check costs more than the sweep it
            // replaces, and its mere presence perturbs ptxas' register split of
            // the noinline phases (+3-5% on cfg2-4).
            if constexpr (GCHECK_BUILT<T, RPLX, RPLV> && !SPLIT) {
                if (s.gcheck && (!any_big || s.gcheck >= 2) && sweep + 2 <= a.max_sweeps) {
                    T2 *scratch = Bbuf0 + (size_t)((bcur ^ 1) & (C > 1 ? 1 : 0)) * panel_elems;
                    if (!gram_check<T, C>(s, smem, rank, Abuf, Bbuf, scratch, G * RPLX, tol) &&
                        s.gcheck == 1) {
                        if (tid < 32) start_pos[tid] = pos[tid];  // norms are where the columns are now
                        __syncthreads();
                        info = sweep + 2;
                        break;
                    }
                }
            }
        }

        // ---- epilogue ---------------------------------------------------------
        // squared norms were recorded per column at round 0 of the last sweep
        // by the CTA that held the column then; gather them from their owners
        if constexpr (C > 1) {
            T *stage = reinterpret_cast<T *>(smem + s.off_send);  // [ncp]
            cluster_sync_all();
            cg::cluster_group cl = cg::this_cluster();
            for (int j = tid; j < ncp; j += blockDim.x) {
                const int panel = j / w;
                int p0 = 0;
                for (int p = 0; p < 2 * C; ++p)
                    if (start_pos[p] == panel) p0 = p;
                const int owner = pos_owner(p0, C);
                stage[j] = (owner == rank) ? sig2[j] : cl.map_shared_rank(sig2, owner)[j];
            }
            cluster_sync_all();  // every CTA has read its peers' sig2
            for (int j = tid; j < ncp; j += blockDim.x) sig2[j] = stage[j];
            __syncthreads();
        }
        for (int j = tid; j < ncp; j += blockDim.x) {
            sig2[j] = epi_sqrt(sig2[j]);
            perm[j] = j;
        }
        __syncthreads();
        if (info >= 0) {
            int *rnk = perm + ncp;
            for (int j = tid; j < nc; j += blockDim.x) {
                const T sj = sig2[j];
                int pp = 0;
                for (int i = 0; i < nc; ++i) {
                    const T si = sig2[i];
                    pp += (si > sj) || (si == sj && i < j);
                }
                rnk[j] = pp;
            }
            __syncthreads();
            for (int j = tid; j < nc; j += blockDim.x) perm[rnk[j]] = j;
            __syncthreads();
        }
        if (rank == 0) {
            for (int p = tid; p < nc; p += blockDim.x) a.sigma[(size_t)mid * nc + p] = sig2[perm[p]];
            if (tid == 0) a.info[mid] = info;
        }
        if constexpr (WANTV) {
            // inverse permutation: column j -> output position
            int *ipos = perm + ncp;
            __syncthreads();
            for (int p = tid; p < nc; p += blockDim.x) ipos[perm[p]] = p;
            __syncthreads();
            const int pa = pos[rank], pb = pos[2 * C - 1 - rank];
            for (int half = 0; half < 2; ++half) {
                const T2 *src = half == 0 ? Abuf : Bbuf;
                const int c0 = (half == 0 ? pa : pb) * w;
                if (a.Uw) {
                    for (int idx = tid; idx < mr * w; idx += blockDim.x) {
                        const int r = idx / w, jj = idx - r * w, j = c0 + jj;
                        if (j >= nc) continue;
                        const T sj = sig2[j];
                        const T den = sj > (T)0 ? sj : (T)1;
                        const T2 v = src[(size_t)jj * LD + r];
                        a.Uw[((size_t)mid * mr + r) * nc + ipos[j]] = mk<T>(epi_div(v.x, den), epi_div(v.y, den));
                    }
                }
                if (a.Vw) {
                    for (int idx = tid; idx < nc * w; idx += blockDim.x) {
                        const int r = idx / w, jj = idx - r * w, j = c0 + jj;
                        if (j >= nc) continue;
                        a.Vw[((size_t)mid * nc + r) * nc + ipos[j]] = src[(size_t)jj * LD + VOFF + r];
                    }
                }
            }
            if (a.zero_sigma && rank == 0 && tid == 0) {
                int z = 0;
                for (int j = 0; j < nc; ++j) z |= !(sig2[j] > (T)0);
                a.zero_sigma[mid] = z;
            }
        }
        if constexpr (C > 1) cluster_sync_all();  // peers done reading this CTA's buffers
        __syncthreads();
    }
}

}  // namespace cs
