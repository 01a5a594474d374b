// cs_jacobi.cuh -- K2/K3 batched one-sided (Hestenes) complex Jacobi SVD kernels.
//
// Replaces the reference's numba batch drivers and solver
//   _svd_values_batch / _svd_full_batch -> _jacobi_sweeps -> _column_norms
//   (pkg/src/convspectra/blocksvd.py:75-173) and the per-block epilogue of
//   _finish_full (blocksvd.py:201-210: stable descending sort, U = B/sigma).
//
// Rotation (blocksvd.py:94-122): for columns a = x_p, b = x_q
//   alpha=|a|^2, beta=|b|^2, gamma=a^H b; skip if alpha*beta == 0 or
//   |gamma| <= tol*sqrt(alpha*beta); t = sign(tau)/(|tau|+sqrt(1+tau^2)) with
//   tau=(beta-alpha)/(2|gamma|), c=1/sqrt(1+t^2), s=t*c, ph=gamma/|gamma|;
//   a <- c a - s conj(ph) b,  b <- s ph a + c b  (V columns alike).
// Numerics: the update is applied as a <- a + ((c-1) a - s conj(ph) b) with
// c-1 = -t^2/(r(1+r)), r = sqrt(1+t^2), evaluated without cancellation.  In
// fp32 a plain c*a update makes every rotation non-unitary by ~1 ulp; summed
// over the ~nc*sweeps rotations a column sees, that drifts sigma by 3e-5 (256)
// .. 6e-5 (512) of sigma_max -- the (c-1) form keeps the drift at the storage
// rounding level (2e-7), matching an fp64-applied rotation (measured with a
// CPU simulation of this exact arithmetic).  t uses g/(|d|+hypot(d,g)) with
// d = beta-alpha, g = 2|gamma| (no tau^2 overflow).
//
// Ordering: parallel round-robin ("circle method") -- nc/2 disjoint pairs per
// round, nc-1 rounds per sweep, every pair once per sweep.  Norms are exact
// per round (not incremental); the round-0 norms of the final, rotation-free
// sweep are the column norms, so sigma needs no extra pass.
#pragma once

#include <cooperative_groups.h>

#include "cs_common.cuh"

namespace cg = cooperative_groups;

namespace cs {

constexpr int JAC_MAX_THREADS = 512;
constexpr size_t JAC_SMEM_LIMIT = 227 * 1024;

template <typename T> struct __align__(4 * sizeof(T)) Part { T a, b, gr, gi; };

struct JacShape {
    int kind;           // 0 = register-resident fast kernel, 1 = generic fallback
    int mr, nc, ncp, P, R, Rv, ldx, ldv, G, RPL, wide, C, threads, nbuf;
    size_t off_sig, off_perm, off_send, off_recv, off_mbar, off_x, off_v, smem;
    int smem_resident;
    int split;  // panel kernel: separate X and V warps (2x threads)
    int gram;   // panel kernel: Gram-blocked cross phase
    int gcheck; // panel kernel: Gram convergence check instead of the rotation-free sweep
    long long num_clusters;
    size_t scratch_per_cta;  // complex elements, generic global-memory mode
};

template <typename T> struct JacArgs {
    const cplx_t<T> *blocks;
    long long count;
    int co, ci;
    JacShape s;
    T tol;
    int max_sweeps;
    T *sigma;
    cplx_t<T> *Uw;  // factor with mr rows (A's U when tall, A's V when wide)
    cplx_t<T> *Vw;  // factor with nc rows
    int *info, *zero_sigma;
    cplx_t<T> *scratch;
    // warm start (panel kernel only): batch item i solves matrix index[i]
    // (outputs land there too), starting from X = initX[i] (mr x nc, working
    // orientation) and V = initV[initV_index[i]] (nc x nc) instead of (A, I)
    const long long *index;
    const cplx_t<T> *initX;
    const cplx_t<T> *initV;
    const long long *initV_index;
    int *dbg;  // debugging only: per-CTA progress codes in mapped host memory (null = off)
};

// ---------------------------------------------------------------------------
// PTX helpers: mbarrier + async bulk shared::cta -> shared::cluster copies
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "CS_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra CS_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint32_t map_rank(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void bulk_to_peer(uint32_t dst, uint32_t src, uint32_t bytes, uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "r"(src), "r"(bytes), "r"(mbar)
        : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// .aligned barriers need the whole warp converged at the instruction; inline
// asm is opaque to the compiler's reconvergence, so converge explicitly
// (without it the Gram check's <C=4, RPLX=8> instantiation hung).
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// ---------------------------------------------------------------------------
// shared math
// ---------------------------------------------------------------------------
// circle-method round-robin: round r, pair slot k -> columns (p, q).  Slot k
// holds positions k and ncp-1-k; position 0 is fixed, the others rotate by one
// per round, so consecutive slots hold consecutive p (and q) columns.
__device__ __forceinline__ void pair_cols(int k, int r, int ncp, int &p, int &q) {
    const int L = ncp - 1;
    int ca = 0;
    if (k != 0) {
        ca = k - 1 + r;
        if (ca >= L) ca -= L;
        ca += 1;
    }
    int cb = ncp - 2 - k + r;
    if (cb >= L) cb -= L;
    cb += 1;
    p = ca;
    q = cb;
}

template <typename T> struct Rot { T cm1, wr, wi; };

// 0: skip, 1: rotate (params in R), -1: non-finite input.
// The skip test compares squares (|gamma|^2 <= tol^2 alpha beta), so most
// late-sweep pairs cost no sqrt at all.
// Rotation parameters of the pair (alpha, beta, gamma = gr + i gi).  Returns
// -1 non-finite, 0 below the threshold (no rotation), 1 rotate, 2 rotate with
// |gamma|/sqrt(alpha beta) > GCHECK_TAU: the panel kernel runs its Gram
// convergence check only after sweeps without such a pair (quadratic
// convergence makes the next sweep likely rotation-free, tools/stopstudy.py).
#ifndef CS_GCHECK_TAU
#define CS_GCHECK_TAU 0.05
#endif
constexpr double GCHECK_TAU2 = CS_GCHECK_TAU * CS_GCHECK_TAU;

// Gram-check form of the skip test (the pair is not rotated there): the same
// rescaling when alpha*beta or |gamma|^2 leaves the normal range
template <typename T>
__device__ __forceinline__ bool below_tol(T q, T gr, T gi, T al, T be, T tol) {
    if (!(q <= (T)1e30 && al * be <= (T)1e30 && al * be >= (T)1e-30 && (q == (T)0 || q >= (T)1e-30 * tol * tol))) {
        const T inv = (T)1 / (al > be ? al : be);
        al *= inv; be *= inv; gr *= inv; gi *= inv;
        q = gr * gr + gi * gi;
    }
    return q <= tol * tol * (al * be);
}

// Column norms beyond ~1e9 / below ~1e-9 (fp32) put alpha*beta and |gamma|^2
// outside the normal range: the squared skip test would pass every pair
// (overflow) and the parameter math would turn inf/NaN.  Every
// quantity below depends only on ratios, so such pairs are rescaled by
// max(alpha, beta) first (|gamma|^2 <= alpha beta keeps them in range).
template <typename T>
__device__ __forceinline__ bool out_of_range(T q, T ab, T tol) {
    return !(q <= (T)1e30 && ab <= (T)1e30 && ab >= (T)1e-30 && (q == (T)0 || q >= (T)1e-30 * tol * tol));
}
template <typename T> __device__ __forceinline__ T recip(T s) { return (T)1 / s; }
template <> __device__ __forceinline__ float recip<float>(float s) { return __frcp_rn(s); }  // no div subroutine
template <typename T>
__device__ __forceinline__ void rescale_pair(T &al, T &be, T &gr, T &gi) {
    const T inv = recip<T>(al > be ? al : be);
    al *= inv; be *= inv; gr *= inv; gi *= inv;
}

template <typename T>
__device__ __forceinline__ int rot_params(T al, T be, T gr, T gi, T tol, Rot<T> &R) {
    if (!(dfinite(al) && dfinite(be) && dfinite(gr) && dfinite(gi))) return -1;
    if (al == (T)0 || be == (T)0) return 0;
    T q = gr * gr + gi * gi;
    if (out_of_range<T>(q, al * be, tol)) {
        rescale_pair<T>(al, be, gr, gi);
        q = gr * gr + gi * gi;
    }
    if (q <= tol * tol * (al * be)) return 0;
    const T ag = dsqrt(q);
    const T d = be - al, g = (T)2 * ag;
    T t = g / (fabs(d) + dhypot(d, g));
    if (d < (T)0) t = -t;
    const T r = dsqrt((T)1 + t * t);
    R.cm1 = -(t * t) / (r * ((T)1 + r));
    const T s = t / r;
    R.wr = s * (gr / ag);
    R.wi = s * (gi / ag);
    return q > (T)GCHECK_TAU2 * (al * be) ? 2 : 1;
}

// fp32: MUFU rsqrt + one Newton step and __fdividef -- no IEEE div/sqrt
// slow-path subroutine calls (whose calling convention forced register
// spills in the hot loop).  A relative error e in r = sqrt(1+t^2) makes the
// (c-1)-form rotation non-unitary by only ~e*t^2, so small late-sweep
// rotations stay unitary to storage precision.
__device__ __forceinline__ float nr_rsqrt(float x) {
    const float y = rsqrtf(x);
    return y * fmaf(-0.5f * x * y, y, 1.5f);
}
template <>
__device__ __forceinline__ int rot_params<float>(float al, float be, float gr, float gi, float tol,
                                                 Rot<float> &R) {
    if (!(isfinite(al) && isfinite(be) && isfinite(gr) && isfinite(gi))) return -1;
    if (al == 0.f || be == 0.f) return 0;
    float q = gr * gr + gi * gi;
    if (out_of_range<float>(q, al * be, tol)) {
        rescale_pair<float>(al, be, gr, gi);
        q = gr * gr + gi * gi;
    }
    if (q <= tol * tol * (al * be)) return 0;
    const float inv_ag = nr_rsqrt(q);
    const float ag = q * inv_ag;
    const float d = be - al, g = 2.f * ag;
    const float h2 = fmaf(d, d, g * g);
    const float hyp = h2 * nr_rsqrt(h2);
    float t = __fdividef(g, fabsf(d) + hyp);
    if (d < 0.f) t = -t;
    const float r2 = fmaf(t, t, 1.f);
    const float ir = nr_rsqrt(r2);
    const float r = r2 * ir;
    R.cm1 = -(t * t) * __fdividef(ir, 1.f + r);
    const float s = t * ir;
    R.wr = s * gr * inv_ag;
    R.wi = s * gi * inv_ag;
    return q > (float)GCHECK_TAU2 * (al * be) ? 2 : 1;
}

// x <- x + ((c-1) x - s conj(ph) y),  y <- y + (s ph x + (c-1) y)
template <typename T>
__device__ __forceinline__ void rot_apply(cplx_t<T> &x, cplx_t<T> &y, const Rot<T> &R) {
    const T dax = R.cm1 * x.x - (R.wr * y.x + R.wi * y.y);
    const T day = R.cm1 * x.y - (R.wr * y.y - R.wi * y.x);
    const T dbx = R.wr * x.x - R.wi * x.y + R.cm1 * y.x;
    const T dby = R.wr * x.y + R.wi * x.x + R.cm1 * y.y;
    x.x += dax;
    x.y += day;
    y.x += dbx;
    y.y += dby;
}

// ---------------------------------------------------------------------------
// load / epilogue shared by both kernels
// ---------------------------------------------------------------------------
template <typename T, bool WANTV>
__device__ __forceinline__ void load_slice(const JacArgs<T> &a, long long f, int rank,
                                           cplx_t<T> *Xs, cplx_t<T> *Vs, int rows_alloc_x,
                                           int rows_alloc_v) {
    using T2 = cplx_t<T>;
    const JacShape &s = a.s;
    const int tid = threadIdx.x, NT = blockDim.x;
    const int mr = s.mr, nc = s.nc, ncp = s.ncp, R = s.R, ldx = s.ldx;
    const int row0 = rank * R;
    const T2 *A = a.blocks + (size_t)f * a.co * a.ci;
    if (!s.wide) {  // X[r][j] = A[r][j]; rows beyond this CTA's slice are zero
        for (int idx = tid; idx < rows_alloc_x * ncp; idx += NT) {
            const int lr = idx / ncp, j = idx - lr * ncp, r = row0 + lr;
            T2 v = mk<T>(0, 0);
            if (lr < R && r < mr && j < nc) v = A[(size_t)r * a.ci + j];
            Xs[(size_t)j * ldx + lr] = v;
        }
    } else {  // X[r][j] = conj(A[j][r])
        for (int idx = tid; idx < rows_alloc_x * ncp; idx += NT) {
            const int j = idx / rows_alloc_x, lr = idx - j * rows_alloc_x, r = row0 + lr;
            T2 v = mk<T>(0, 0);
            if (lr < R && r < mr && j < nc) {
                v = A[(size_t)j * a.ci + r];
                v.y = -v.y;
            }
            Xs[(size_t)j * ldx + lr] = v;
        }
    }
    if constexpr (WANTV) {
        const int Rv = s.Rv, ldv = s.ldv, vrow0 = rank * Rv;
        for (int idx = tid; idx < rows_alloc_v * ncp; idx += NT) {
            const int j = idx / rows_alloc_v, lv = idx - j * rows_alloc_v, vr = vrow0 + lv;
            Vs[(size_t)j * ldv + lv] = mk<T>((lv < Rv && vr == j && vr < nc) ? (T)1 : (T)0, 0);
        }
    }
}

// sigma from squared norms, stable descending order, U = X/sigma, V, flags
template <typename T, bool WANTV>
__device__ __forceinline__ void epilogue(const JacArgs<T> &a, long long f, int rank, int info,
                                         const cplx_t<T> *Xs, const cplx_t<T> *Vs, T *sig,
                                         int *perm) {
    using T2 = cplx_t<T>;
    const JacShape &s = a.s;
    const int tid = threadIdx.x, NT = blockDim.x;
    const int nc = s.nc, ncp = s.ncp, mr = s.mr, R = s.R, ldx = s.ldx;
    for (int j = tid; j < ncp; j += NT) {
        sig[j] = dsqrt(sig[j]);
        perm[j] = j;
    }
    __syncthreads();
    if (info >= 0) {
        int *rnk = perm + ncp;
        for (int j = tid; j < nc; j += NT) {
            const T sj = sig[j];
            int pos = 0;
            for (int i = 0; i < nc; ++i) {
                const T si = sig[i];
                pos += (si > sj) || (si == sj && i < j);
            }
            rnk[j] = pos;
        }
        __syncthreads();
        for (int j = tid; j < nc; j += NT) perm[rnk[j]] = j;
        __syncthreads();
    }
    if (rank == 0) {
        for (int pos = tid; pos < nc; pos += NT) a.sigma[(size_t)f * nc + pos] = sig[perm[pos]];
        if (tid == 0) a.info[f] = info;
    }
    if constexpr (WANTV) {
        const int row0 = rank * R;
        if (a.Uw) {
            for (int idx = tid; idx < R * nc; idx += NT) {
                const int lr = idx / nc, pos = idx - lr * nc, row = row0 + lr;
                if (row >= mr) continue;
                const int j = perm[pos];
                const T sj = sig[j];
                const T den = sj > (T)0 ? sj : (T)1;
                const T2 v = Xs[(size_t)j * ldx + lr];
                a.Uw[((size_t)f * mr + row) * nc + pos] = mk<T>(v.x / den, v.y / den);
            }
        }
        const int Rv = s.Rv, ldv = s.ldv, vrow0 = rank * Rv;
        if (a.Vw) {
            for (int idx = tid; idx < Rv * nc; idx += NT) {
                const int lv = idx / nc, pos = idx - lv * nc, vrow = vrow0 + lv;
                if (vrow >= nc) continue;
                a.Vw[((size_t)f * nc + vrow) * nc + pos] = Vs[(size_t)perm[pos] * ldv + lv];
            }
        }
        if (a.zero_sigma && rank == 0 && tid == 0) {
            int z = 0;
            for (int j = 0; j < nc; ++j) z |= !(sig[j] > (T)0);
            a.zero_sigma[f] = z;
        }
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// fast kernel: rows in registers between the reduction and the rotation
// ---------------------------------------------------------------------------
// One cluster of C CTAs per matrix (persistent over matrices).  Thread layout:
// pair slot k = tid / G, lane_g = tid % G; lane owns rows lane_g + G*i,
// i < RPL, of columns p,q of its CTA's slice (and of V).  C == 1: the G-lane
// shuffle reduction already yields the full (alpha, beta, gamma) -- one
// __syncthreads per round.  C > 1: the leaders write partials to a send
// buffer, one thread ships it to the C-1 peers with async bulk copies
// (cp.async.bulk shared::cta -> shared::cluster) that complete_tx on the
// peers' mbarriers; everybody sums the C partials in rank order, so all CTAs
// take bit-identical decisions without any cluster barrier in the loop.
template <typename T, int C, int RPL, bool WANTV>
__global__ void __launch_bounds__(JAC_MAX_THREADS)
jacobi_fast_kernel(const JacArgs<T> a) {
    using T2 = cplx_t<T>;
    extern __shared__ __align__(16) unsigned char smem[];
    const JacShape &s = a.s;
    int rank = 0;
    if constexpr (C > 1) rank = (int)cg::this_cluster().block_rank();
    const long long cid = blockIdx.x / C;

    T *sig = reinterpret_cast<T *>(smem + s.off_sig);
    int *perm = reinterpret_cast<int *>(smem + s.off_perm);
    Part<T> *sendb = reinterpret_cast<Part<T> *>(smem + s.off_send);  // [2][P]
    Part<T> *recvb = reinterpret_cast<Part<T> *>(smem + s.off_recv);  // [2][C][P]
    uint64_t *mbar = reinterpret_cast<uint64_t *>(smem + s.off_mbar);  // [2]
    T2 *Xs = reinterpret_cast<T2 *>(smem + s.off_x);
    T2 *Vs = reinterpret_cast<T2 *>(smem + s.off_v);

    const int tid = threadIdx.x;
    const int G = s.G, lane_g = tid % G, k = tid / G;
    const int P = s.P, ncp = s.ncp, ldx = s.ldx, ldv = s.ldv;
    const bool active = k < P;
    const T tol = a.tol;
    const uint32_t part_bytes = (uint32_t)(P * sizeof(Part<T>));

    if constexpr (C > 1) {
        if (tid == 0) {
            mbar_init(&mbar[0], 1);
            mbar_init(&mbar[1], 1);
            fence_mbar_init();
        }
        cluster_sync_all();
    }

    unsigned rc = 0;  // running round counter (buffer parity / mbarrier phase)
    for (long long f = cid; f < a.count; f += s.num_clusters) {
        load_slice<T, WANTV>(a, f, rank, Xs, Vs, G * RPL, G * RPL);
        __syncthreads();
        int info = -1;
        for (int sweep = 0; sweep < a.max_sweeps; ++sweep) {
            bool rot = false, bad = false;
            for (int r = 0; r < ncp - 1; ++r, ++rc) {
                int p = 0, q = 0;
                T2 x[RPL], y[RPL];
                T2 vx[WANTV ? RPL : 1], vy[WANTV ? RPL : 1];
                T al = 0, be = 0, gr = 0, gi = 0;
                if (active) {
                    pair_cols(k, r, ncp, p, q);
                    const T2 *xp = Xs + (size_t)p * ldx + lane_g, *xq = Xs + (size_t)q * ldx + lane_g;
#pragma unroll
                    for (int i = 0; i < RPL; ++i) {
                        x[i] = xp[i * G];
                        y[i] = xq[i * G];
                    }
                    if constexpr (WANTV) {
                        const T2 *vp = Vs + (size_t)p * ldv + lane_g, *vq = Vs + (size_t)q * ldv + lane_g;
#pragma unroll
                        for (int i = 0; i < RPL; ++i) {
                            vx[i] = vp[i * G];
                            vy[i] = vq[i * G];
                        }
                    }
#pragma unroll
                    for (int i = 0; i < RPL; ++i) {
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
                if constexpr (C > 1) {
                    const int b = rc & 1;
                    if (active && lane_g == 0) {
                        Part<T> pt;
                        pt.a = al; pt.b = be; pt.gr = gr; pt.gi = gi;
                        sendb[b * P + k] = pt;
                        fence_proxy_async_smem();
                    }
                    __syncthreads();
                    if (tid == 0) {
                        mbar_arrive_expect_tx(&mbar[b], (uint32_t)(C - 1) * part_bytes);
                        const uint32_t src = smem_u32(sendb + b * P);
                        const uint32_t dst = smem_u32(recvb + ((size_t)b * C + rank) * P);
                        const uint32_t mb = smem_u32(&mbar[b]);
#pragma unroll
                        for (int d = 1; d < C; ++d) {
                            const uint32_t peer = (uint32_t)((rank + d) % C);
                            bulk_to_peer(map_rank(dst, peer), src, part_bytes, map_rank(mb, peer));
                        }
                        bulk_commit();
                        mbar_wait(&mbar[b], (rc >> 1) & 1);
                    }
                    __syncthreads();  // one spinner instead of the whole CTA
                    if (active) {
                        al = be = gr = gi = 0;
#pragma unroll
                        for (int d = 0; d < C; ++d) {
                            const Part<T> t = (d == rank) ? sendb[b * P + k] : recvb[((size_t)b * C + d) * P + k];
                            al += t.a; be += t.b; gr += t.gr; gi += t.gi;
                        }
                    }
                }
                if (active) {
                    if (r == 0 && lane_g == 0) {  // exact norms at sweep start -> sigma^2 at the end
                        sig[p] = al;
                        sig[q] = be;
                    }
                    Rot<T> R;
                    const int act = rot_params<T>(al, be, gr, gi, tol, R);
                    if (act < 0) {
                        bad = true;
                    } else if (act > 0) {
                        rot = true;
                        T2 *xp = Xs + (size_t)p * ldx + lane_g, *xq = Xs + (size_t)q * ldx + lane_g;
#pragma unroll
                        for (int i = 0; i < RPL; ++i) {
                            rot_apply<T>(x[i], y[i], R);
                            xp[i * G] = x[i];
                            xq[i * G] = y[i];
                        }
                        if constexpr (WANTV) {
                            T2 *vp = Vs + (size_t)p * ldv + lane_g, *vq = Vs + (size_t)q * ldv + lane_g;
#pragma unroll
                            for (int i = 0; i < RPL; ++i) {
                                rot_apply<T>(vx[i], vy[i], R);
                                vp[i * G] = vx[i];
                                vq[i * G] = vy[i];
                            }
                        }
                    }
                }
                if (r + 1 < ncp - 1) __syncthreads();
            }
            const int any_bad = __syncthreads_or(bad);
            const int any_rot = __syncthreads_or(rot);
            if (any_bad) break;
            if (!any_rot) {
                info = sweep + 1;
                break;
            }
        }
        epilogue<T, WANTV>(a, f, rank, info, Xs, Vs, sig, perm);
    }
    if constexpr (C > 1) {
        if (tid == 0) bulk_wait_read_all();
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// generic kernel: any size (rows re-read from shared or global memory)
// ---------------------------------------------------------------------------
template <int C> __device__ __forceinline__ void cluster_barrier() {
    if constexpr (C > 1) {
        cg::this_cluster().sync();
    } else {
        __syncthreads();
    }
}

template <typename T, int C, bool WANTV, bool SMEM>
__global__ void __launch_bounds__(JAC_MAX_THREADS)
jacobi_generic_kernel(const JacArgs<T> a) {
    using T2 = cplx_t<T>;
    extern __shared__ __align__(16) unsigned char smem[];
    const JacShape &s = a.s;
    int rank = 0;
    if constexpr (C > 1) rank = (int)cg::this_cluster().block_rank();
    const long long cid = blockIdx.x / C;

    Part<T> *xbuf = reinterpret_cast<Part<T> *>(smem + s.off_send);
    T *sig = reinterpret_cast<T *>(smem + s.off_sig);
    int *perm = reinterpret_cast<int *>(smem + s.off_perm);
    T2 *Xs, *Vs;
    if constexpr (SMEM) {
        Xs = reinterpret_cast<T2 *>(smem + s.off_x);
        Vs = reinterpret_cast<T2 *>(smem + s.off_v);
    } else {
        Xs = a.scratch + (size_t)blockIdx.x * s.scratch_per_cta;
        Vs = Xs + (size_t)s.ncp * s.ldx;
    }
    const int tid = threadIdx.x, NT = blockDim.x;
    const int G = s.G, lane_g = tid & (G - 1), grp = tid / G, ngrp = NT / G;
    const int P = s.P, ncp = s.ncp, R = s.R, Rv = s.Rv, ldx = s.ldx, ldv = s.ldv;
    const int iters = (P + ngrp - 1) / ngrp;
    const T tol = a.tol;

    for (long long f = cid; f < a.count; f += s.num_clusters) {
        cluster_barrier<C>();
        load_slice<T, WANTV>(a, f, rank, Xs, Vs, R, Rv);
        __syncthreads();
        int info = -1, rctr = 0;
        for (int sweep = 0; sweep < a.max_sweeps; ++sweep) {
            bool rot = false, bad = false;
            for (int r = 0; r < ncp - 1; ++r, ++rctr) {
                Part<T> *xb = xbuf + (size_t)((s.nbuf == 2) ? (rctr & 1) : 0) * C * P;
                for (int it = 0; it < iters; ++it) {
                    const int k = grp + it * ngrp;
                    const bool valid = k < P;
                    T al = 0, be = 0, gr = 0, gi = 0;
                    if (valid) {
                        int p, q;
                        pair_cols(k, r, ncp, p, q);
                        const T2 *xp = Xs + (size_t)p * ldx, *xq = Xs + (size_t)q * ldx;
                        for (int lr = lane_g; lr < R; lr += G) {
                            const T2 x = xp[lr], y = xq[lr];
                            al = fma(x.y, x.y, fma(x.x, x.x, al));
                            be = fma(y.y, y.y, fma(y.x, y.x, be));
                            gr = fma(x.y, y.y, fma(x.x, y.x, gr));
                            gi = fma(-x.y, y.x, fma(x.x, y.y, gi));
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
                    if (valid && lane_g == 0) {
                        Part<T> pt;
                        pt.a = al; pt.b = be; pt.gr = gr; pt.gi = gi;
                        Part<T> *slot = xb + (size_t)rank * P + k;
                        if constexpr (C > 1) {
                            cg::cluster_group cl = cg::this_cluster();
                            for (int d = 0; d < C; ++d) *cl.map_shared_rank(slot, d) = pt;
                        } else {
                            *slot = pt;
                        }
                    }
                }
                cluster_barrier<C>();
                for (int it = 0; it < iters; ++it) {
                    const int k = grp + it * ngrp;
                    if (k >= P) break;
                    T al = 0, be = 0, gr = 0, gi = 0;
                    for (int d = 0; d < C; ++d) {
                        const Part<T> td = xb[(size_t)d * P + k];
                        al += td.a; be += td.b; gr += td.gr; gi += td.gi;
                    }
                    int p, q;
                    pair_cols(k, r, ncp, p, q);
                    if (r == 0 && lane_g == 0) {
                        sig[p] = al;
                        sig[q] = be;
                    }
                    Rot<T> Rr;
                    const int act = rot_params<T>(al, be, gr, gi, tol, Rr);
                    if (act < 0) { bad = true; continue; }
                    if (act == 0) continue;
                    rot = true;
                    T2 *xp = Xs + (size_t)p * ldx, *xq = Xs + (size_t)q * ldx;
                    for (int lr = lane_g; lr < R; lr += G) {
                        T2 x = xp[lr], y = xq[lr];
                        rot_apply<T>(x, y, Rr);
                        xp[lr] = x;
                        xq[lr] = y;
                    }
                    if constexpr (WANTV) {
                        T2 *vp = Vs + (size_t)p * ldv, *vq = Vs + (size_t)q * ldv;
                        for (int lv = lane_g; lv < Rv; lv += G) {
                            T2 x = vp[lv], y = vq[lv];
                            rot_apply<T>(x, y, Rr);
                            vp[lv] = x;
                            vq[lv] = y;
                        }
                    }
                }
                if (s.nbuf == 2) {
                    __syncthreads();
                } else {
                    cluster_barrier<C>();
                }
            }
            const int any_bad = __syncthreads_or(bad);
            const int any_rot = __syncthreads_or(rot);
            if (any_bad) break;
            if (!any_rot) {
                info = sweep + 1;
                break;
            }
        }
        if (!SMEM) __threadfence_block();
        epilogue<T, WANTV>(a, f, rank, info, Xs, Vs, sig, perm);
    }
    cluster_barrier<C>();
}

// ---------------------------------------------------------------------------
// launch helper
// ---------------------------------------------------------------------------
template <typename T, int C, typename K>
static int launch_cluster_kernel(K kern, const JacArgs<T> &args0, cudaStream_t st, bool dry,
                                 long long *nclusters) {
    JacArgs<T> args = args0;
    CS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)args.s.smem));
    if (C > 8) CS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(args.s.threads);
    cfg.dynamicSmemBytes = args.s.smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(C);
    int maxc = 0;
    CS_CUDA_TRY(cudaOccupancyMaxActiveClusters(&maxc, (void *)kern, &cfg));
    if (maxc <= 0) return fail(CS_ENOMEM, "batched SVD: cluster configuration cannot be scheduled");
    const long long ncl = lmin(args.count, (long long)maxc);
    if (nclusters) *nclusters = ncl;
    if (dry) return CS_OK;
    args.s.num_clusters = ncl;
    cfg.gridDim = dim3((unsigned)(ncl * C));
    CS_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, args));
    return check_launch("jacobi kernel");
}

// per-dtype dispatchers (cs_jacobi_f32.cu / cs_jacobi_f64.cu)
int jacobi_dispatch_f32(const JacArgs<float> &a, bool wantv, cudaStream_t st, bool dry, long long *ncl);
int jacobi_dispatch_f64(const JacArgs<double> &a, bool wantv, cudaStream_t st, bool dry, long long *ncl);

}  // namespace cs
