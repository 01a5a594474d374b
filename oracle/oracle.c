/*
 * oracle.c -- CPU restatement of the reference's LFA hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path
 * (paper_2506_05617_b200/) links, loads or calls this file.  It is used by
 * tests/ (as the parity checker), by __graft_entry__.smoke() (checker) and by
 * bench.py's cpu_baseline / --impl reference leg (the reference's CPU path,
 * timed on the host cores).
 *
 * It restates, in plain C, the numba kernels of the reference package
 * conv-spectra 0.1.0 (/root/reference/pkg/src/convspectra):
 *
 *   orc_symbol_blocks      <- symbol.py:89-105   (_symbol_blocks, prange over F)
 *   orc_jacobi_sweeps      <- blocksvd.py:75-125 (_jacobi_sweeps, one-sided
 *                                                 cyclic-by-row complex Jacobi)
 *   orc_column_norms       <- blocksvd.py:128-136
 *   orc_svd_values_batch   <- blocksvd.py:139-152 (values, ascending per block)
 *   orc_svd_full_batch     <- blocksvd.py:155-173 (B=U*Sigma, V, raw sigma)
 *
 * All arithmetic is complex128 written out as explicit re/im doubles in the
 * same operation order as the reference; build with -ffp-contract=off so no
 * FMA contraction changes rounding.  Parity is pinned against vectors
 * produced by importing the reference itself (tests/golden/make_golden.py).
 *
 * The *_f32 variants keep the working matrix in float (complex64 storage) and
 * accumulate norms/dot products in double (*_f32acc: in float); they exist
 * only to study the fp32
 * convergence behaviour (tolerance / sweep counts) that the CUDA fp32 path
 * relies on.  They are not a parity reference.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static void set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* symbol.py:89-105.  freqs (F,2) f64, offs (T,2) f64 [col0 = height offset,
 * col1 = width offset], taps (T,co,ci) f64, out (F,co,ci) complex128 as
 * interleaved doubles; out must be zero-filled by the caller (symbol.py:134). */
void orc_symbol_blocks(const double *freqs, int64_t F, const double *offs, int T,
                       const double *taps, int co, int ci, double *out,
                       int nthreads) {
    set_threads(nthreads);
    const double two_pi = 2.0 * M_PI;
    const int64_t blk = (int64_t)co * ci;
#pragma omp parallel for schedule(static)
    for (int64_t f = 0; f < F; ++f) {
        const double k1 = freqs[2 * f], k2 = freqs[2 * f + 1];
        double *o = out + 2 * f * blk;
        for (int t = 0; t < T; ++t) {
            /* arg = 2pi (k1*y_w + k2*y_h); k[0] pairs with the width offset */
            const double arg = two_pi * (k1 * offs[2 * t + 1] + k2 * offs[2 * t]);
            const double pr = cos(arg), pi = sin(arg);
            const double *tp = taps + (int64_t)t * blk;
            for (int64_t e = 0; e < blk; ++e) {
                const double w = tp[e];
                /* complex(pr,pi) * complex(w,0), then += */
                o[2 * e] += pr * w - pi * 0.0;
                o[2 * e + 1] += pr * 0.0 + pi * w;
            }
        }
    }
}

/* ---------------------------------------------------------------------------
 * One-sided Jacobi.  B is (mr, nc) row-major complex, V is (nc, nc).
 * Restates blocksvd.py:75-125 line by line.
 * ------------------------------------------------------------------------- */
#define DEFINE_JACOBI(NAME, ST, AT)                                                  \
    int NAME(ST *B, int mr, int nc, ST *V, int accumulate_v, double tol,        \
             int max_sweeps, double *norms) {                                    \
        for (int sweep = 0; sweep < max_sweeps; ++sweep) {                       \
            for (int j = 0; j < nc; ++j) {                                       \
                AT acc = 0.0;                                                    \
                for (int r = 0; r < mr; ++r) {                                   \
                    const AT vr = B[2 * ((int64_t)r * nc + j)];                  \
                    const AT vi = B[2 * ((int64_t)r * nc + j) + 1];              \
                    acc += vr * vr + vi * vi;                                    \
                }                                                                \
                norms[j] = acc;                                                  \
            }                                                                    \
            int rotated = 0;                                                     \
            for (int p = 0; p < nc - 1; ++p) {                                   \
                for (int q = p + 1; q < nc; ++q) {                               \
                    const double alpha = norms[p], beta = norms[q];              \
                    if (alpha == 0.0 || beta == 0.0) continue;                   \
                    AT gr = 0.0, gi = 0.0;                                       \
                    for (int r = 0; r < mr; ++r) {                               \
                        const AT ar = B[2 * ((int64_t)r * nc + p)];              \
                        const AT ai = -B[2 * ((int64_t)r * nc + p) + 1];         \
                        const AT br = B[2 * ((int64_t)r * nc + q)];              \
                        const AT bi = B[2 * ((int64_t)r * nc + q) + 1];          \
                        gr += ar * br - ai * bi;                                 \
                        gi += ar * bi + ai * br;                                 \
                    }                                                            \
                    const double ag = hypot(gr, gi);                             \
                    if (ag <= tol * sqrt(alpha * beta)) continue;                \
                    rotated = 1;                                                 \
                    const double tau = (beta - alpha) / (2.0 * ag);              \
                    double t;                                                    \
                    if (tau >= 0.0) t = 1.0 / (tau + sqrt(1.0 + tau * tau));     \
                    else t = -1.0 / (-tau + sqrt(1.0 + tau * tau));              \
                    const double c = 1.0 / sqrt(1.0 + t * t);                    \
                    const double s = t * c;                                      \
                    const double phr = gr / ag, phi = gi / ag; /* ph=gamma/|g| */\
                    /* bp' = c*bp - s*(conj(ph)*bq); bq' = s*(ph*bp) + c*bq */   \
                    for (int r = 0; r < mr; ++r) {                               \
                        ST *xp = B + 2 * ((int64_t)r * nc + p);                  \
                        ST *xq = B + 2 * ((int64_t)r * nc + q);                  \
                        const double bpr = xp[0], bpi = xp[1];                   \
                        const double bqr = xq[0], bqi = xq[1];                   \
                        const double ur = phr * bqr + phi * bqi;                 \
                        const double ui = phr * bqi - phi * bqr;                 \
                        const double wr = phr * bpr - phi * bpi;                 \
                        const double wi = phr * bpi + phi * bpr;                 \
                        xp[0] = (ST)(c * bpr - s * ur);                          \
                        xp[1] = (ST)(c * bpi - s * ui);                          \
                        xq[0] = (ST)(s * wr + c * bqr);                          \
                        xq[1] = (ST)(s * wi + c * bqi);                          \
                    }                                                            \
                    if (accumulate_v) {                                          \
                        for (int r = 0; r < nc; ++r) {                           \
                            ST *vp = V + 2 * ((int64_t)r * nc + p);              \
                            ST *vq = V + 2 * ((int64_t)r * nc + q);              \
                            const double a_r = vp[0], a_i = vp[1];               \
                            const double b_r = vq[0], b_i = vq[1];               \
                            const double ur = phr * b_r + phi * b_i;             \
                            const double ui = phr * b_i - phi * b_r;             \
                            const double wr = phr * a_r - phi * a_i;             \
                            const double wi = phr * a_i + phi * a_r;             \
                            vp[0] = (ST)(c * a_r - s * ur);                      \
                            vp[1] = (ST)(c * a_i - s * ui);                      \
                            vq[0] = (ST)(s * wr + c * b_r);                      \
                            vq[1] = (ST)(s * wi + c * b_i);                      \
                        }                                                        \
                    }                                                            \
                    norms[p] = c * c * alpha + s * s * beta - 2.0 * c * s * ag;  \
                    norms[q] = s * s * alpha + c * c * beta + 2.0 * c * s * ag;  \
                }                                                                \
            }                                                                    \
            if (!rotated) return sweep + 1;                                      \
        }                                                                        \
        return -1;                                                               \
    }

DEFINE_JACOBI(orc_jacobi_sweeps, double, double)
DEFINE_JACOBI(orc_jacobi_sweeps_f32, float, double)
DEFINE_JACOBI(orc_jacobi_sweeps_f32acc, float, float)

/* blocksvd.py:128-136 */
#define DEFINE_NORMS(NAME, ST)                                                   \
    void NAME(const ST *B, int mr, int nc, double *out) {                        \
        for (int j = 0; j < nc; ++j) {                                           \
            double acc = 0.0;                                                    \
            for (int r = 0; r < mr; ++r) {                                       \
                const double vr = B[2 * ((int64_t)r * nc + j)];                  \
                const double vi = B[2 * ((int64_t)r * nc + j) + 1];              \
                acc += vr * vr + vi * vi;                                        \
            }                                                                    \
            out[j] = sqrt(acc);                                                  \
        }                                                                        \
    }
DEFINE_NORMS(orc_column_norms, double)
DEFINE_NORMS(orc_column_norms_f32, float)

static int cmp_double(const void *a, const void *b) {
    const double x = *(const double *)a, y = *(const double *)b;
    return (x > y) - (x < y);
}

/* blocksvd.py:139-152.  blocks (F,mr,nc) complex (the tall working view);
 * sig (F,nc) ascending; fail (F,) int8; sweeps (F,) int32 (extra: sweeps used
 * or -1, the reference discards this). */
#define DEFINE_VALUES_BATCH(NAME, ST, JAC, NORMS)                                \
    void NAME(const ST *blocks, int64_t F, int mr, int nc, double tol,           \
              int max_sweeps, double *sig, int8_t *fail, int32_t *sweeps,        \
              int nthreads) {                                                    \
        set_threads(nthreads);                                                   \
        const int64_t blk = 2 * (int64_t)mr * nc;                                \
        _Pragma("omp parallel")                                                  \
        {                                                                        \
            ST *B = (ST *)malloc(sizeof(ST) * blk);                              \
            double *norms = (double *)malloc(sizeof(double) * (nc + 1));         \
            _Pragma("omp for schedule(dynamic, 1)")                              \
            for (int64_t f = 0; f < F; ++f) {                                    \
                memcpy(B, blocks + f * blk, sizeof(ST) * blk);                   \
                const int sw = JAC(B, mr, nc, NULL, 0, tol, max_sweeps, norms);  \
                fail[f] = sw < 0 ? 1 : 0;                                        \
                if (sweeps) sweeps[f] = sw;                                      \
                NORMS(B, mr, nc, sig + f * nc);                                  \
                qsort(sig + f * nc, nc, sizeof(double), cmp_double);             \
            }                                                                    \
            free(B);                                                             \
            free(norms);                                                         \
        }                                                                        \
    }
DEFINE_VALUES_BATCH(orc_svd_values_batch, double, orc_jacobi_sweeps, orc_column_norms)
DEFINE_VALUES_BATCH(orc_svd_values_batch_f32, float, orc_jacobi_sweeps_f32,
                    orc_column_norms_f32)
DEFINE_VALUES_BATCH(orc_svd_values_batch_f32acc, float, orc_jacobi_sweeps_f32acc,
                    orc_column_norms_f32)

/* blocksvd.py:155-173.  Bout (F,mr,nc) = converged B, Vout (F,nc,nc),
 * sig (F,nc) raw (column order), fail (F,). */
void orc_svd_full_batch(const double *blocks, int64_t F, int mr, int nc, double tol,
                        int max_sweeps, double *Bout, double *Vout, double *sig,
                        int8_t *fail, int32_t *sweeps, int nthreads) {
    set_threads(nthreads);
    const int64_t blk = 2 * (int64_t)mr * nc, vblk = 2 * (int64_t)nc * nc;
#pragma omp parallel
    {
        double *norms = (double *)malloc(sizeof(double) * (nc + 1));
#pragma omp for schedule(dynamic, 1)
        for (int64_t f = 0; f < F; ++f) {
            double *B = Bout + f * blk;
            double *V = Vout + f * vblk;
            memcpy(B, blocks + f * blk, sizeof(double) * blk);
            memset(V, 0, sizeof(double) * vblk);
            for (int j = 0; j < nc; ++j) V[2 * ((int64_t)j * nc + j)] = 1.0;
            const int sw = orc_jacobi_sweeps(B, mr, nc, V, 1, tol, max_sweeps, norms);
            fail[f] = sw < 0 ? 1 : 0;
            if (sweeps) sweeps[f] = sw;
            orc_column_norms(B, mr, nc, sig + f * nc);
        }
        free(norms);
    }
}
