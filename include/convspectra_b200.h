/*
 * convspectra_b200.h -- C-ABI of the B200-native LFA SVD hot path.
 *
 * The reference (conv-spectra 0.1.0) is pure Python + numba and has no FFI;
 * its "plugin seam" is the method dispatch of compute_spectrum
 * (pkg/src/convspectra/pipeline.py:52-68).  Each entry point below replaces
 * one reference function on that path; the host-side mirror of the
 * reference API (paper_2506_05617_b200/*.py) binds them with ctypes, and
 * INTEGRATION.md shows the binding a reference maintainer would add.
 *
 * Conventions:
 *   - weights W: (c_out, c_in, k_h, k_w) row-major real, fp32 or fp64
 *   - frequencies k = (i/n, j/m), full-grid index f = i*m + j
 *     (kernels.py:119-140); tap offsets y = (p - k_h/2, q - k_w/2)
 *     (kernels.py:71-85); k[0] pairs with the WIDTH offset (symbol.py:68-71)
 *   - symbol A_f[o,c] = sum_{p,q} W[o,c,p,q] exp(+2 pi i (i y_w/n + j y_h/m))
 *   - half grid: conjugate-orbit representatives f <= f* in row-major order,
 *     F_u = (n*m + s)/2 (s = number of self-conjugate frequencies)
 *   - complex data is interleaved (re, im) of the real dtype
 *   - every pointer argument is a DEVICE pointer unless stated otherwise;
 *     `stream` is a cudaStream_t passed as void*; all calls are stream-ordered
 *     and asynchronous, the library owns no persistent device memory.
 *
 * Status codes: 0 ok; CS_EINVAL -> ValueError/ZeroDimension; CS_ENOMEM ->
 * AllocationFailure; CS_ENOCONV -> ConvergenceFailure; CS_ECUDA -> RuntimeError.
 * cs_last_error_string() describes the last non-zero status of this thread.
 */
#ifndef CONVSPECTRA_B200_H
#define CONVSPECTRA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CS_ABI_VERSION 1

enum cs_status { CS_OK = 0, CS_EINVAL = 1, CS_ENOMEM = 2, CS_ENOCONV = 3, CS_ECUDA = 4 };
enum cs_dtype { CS_F32 = 0, CS_F64 = 1 };
enum cs_layout { CS_BLOCK_CONTIGUOUS = 0, CS_FREQUENCY_STRIDED = 1 };

int cs_abi_version(void);
const char *cs_last_error_string(void);

/* Number of conjugate-orbit representatives of an n x m torus. */
long long cs_half_grid_count(int n, int m);

/* K1 -- symbol assembly.  Replaces symbol.py:108-137 (build_symbol_field ->
 * numba _symbol_blocks, symbol.py:89-105).
 * Evaluates A_f for the f_count frequencies starting at f_first, indexed in
 * the full grid (half_grid = 0) or in the representative list (half_grid = 1).
 * out: (f_count, c_out, c_in) complex for CS_BLOCK_CONTIGUOUS, or
 *      (c_out, c_in, f_count) for CS_FREQUENCY_STRIDED (symbol.py:146-161). */
int cs_symbol_field(const void *W, int dtype, int c_out, int c_in, int k_h, int k_w,
                    int n, int m, long long f_first, long long f_count, int half_grid,
                    void *out, int layout, void *stream);

/* K1 at explicit frequencies (k1,k2) (count,2) f64: replaces symbol.py:74-86
 * (symbol_at) and _symbol_blocks over FrequencyGrid(dims, frequencies=...). */
int cs_symbol_at(const void *W, int dtype, int c_out, int c_in, int k_h, int k_w,
                 const double *freqs, long long count, void *out, void *stream);

/* Expand a half-grid field (F_u, c_out, c_in) into the full grid (n*m, c_out, c_in)
 * with A_{f*} = conj(A_f). */
int cs_expand_half_grid(const void *half, int dtype, int c_out, int c_in, int n, int m,
                        void *full, void *stream);

/* *flag = 1 iff the full-grid field is exactly conjugate-symmetric
 * (A_{f*} == conj(A_f) bit for bit, all finite); used to decide whether a
 * caller-supplied field may be solved on the half grid. */
int cs_check_conj_symmetry(const void *full, int dtype, int c_out, int c_in, int n, int m,
                           int *flag, void *stream);

/* K2/K3 -- batched one-sided Jacobi SVD.  Replaces blocksvd.py:139-173
 * (_svd_values_batch / _svd_full_batch -> _jacobi_sweeps) plus the epilogue
 * of blocksvd.py:201-210 (_finish_full: per-block stable descending sort,
 * U = B/sigma).  Wide blocks (c_out < c_in) are solved on A^H with U/V
 * swapped (blocksvd.py:254-256, 268-270).
 *   blocks : (count, c_out, c_in) complex, read only
 *   sigma  : (count, r) real, descending,  r = min(c_out, c_in)
 *   U, V   : (count, c_out, r), (count, c_in, r) complex, or NULL (values only)
 *   info   : (count,) int32 -- sweeps used, or -1 when the block did not
 *            converge within max_sweeps or holds non-finite values
 *   zero_sigma : (count,) int32 or NULL -- set to 1 where a sigma is exactly 0
 *            and U needs the orthonormal completion (cs_complete_zero_columns)
 *   workspace : cs_batched_svd_workspace() bytes of device scratch (may be 0)
 * tol / max_sweeps have the meaning of blocksvd.py:75-125. */
size_t cs_batched_svd_workspace(int dtype, long long count, int c_out, int c_in,
                                int want_vectors);
int cs_batched_svd(const void *blocks, int dtype, long long count, int c_out, int c_in,
                   int want_vectors, double tol, int max_sweeps, void *sigma, void *U,
                   void *V, int *info, int *zero_sigma, void *workspace,
                   size_t workspace_bytes, void *stream);

/* Which kernel family the planner picks for a batch: 2 = panel (cluster,
 * register-resident), 0 = row-split fast kernel, 1 = generic; -1 = invalid. */
int cs_batched_svd_plan_kind(int dtype, long long count, int c_out, int c_in,
                             int want_vectors);

/* Indexed / warm-started variant (panel kernel only).  Batch item i solves
 * matrix index[i] of `blocks` (outputs are written at index[i] as well); with
 * init_X it starts from X = init_X[i] ((mr, nc) row-major, working
 * orientation X = A or A^H) instead of the block, and with init_V from
 * V = init_V[init_V_index[i]] ((nc, nc) row-major) instead of the identity.
 * Same algorithm, tolerance and outputs as cs_batched_svd.  index may be NULL
 * (item i solves matrix i).  plan_count > 0 makes the kernel configuration
 * (cluster size, panel width -- hence the rotation order and the result bits)
 * that of a batch of plan_count matrices, independent of `count`: a frequency
 * shard then reproduces the single-GPU solve bit for bit (the reference's
 * partition guarantee, blocksvd.py:4-8); <= 0 plans for `count`. */
int cs_batched_svd_indexed(const void *blocks, int dtype, long long count, int c_out,
                           int c_in, int want_vectors, double tol, int max_sweeps,
                           const long long *index, const void *init_X, const void *init_V,
                           const long long *init_V_index, long long plan_count, void *sigma,
                           void *U, void *V,
                           int *info, int *zero_sigma, void *workspace,
                           size_t workspace_bytes, void *stream);

/* Warm-start GEMM: out_X[i] = X_{warm_ids[i]} . Vw[seed_ids[i]] where X_f is
 * the working matrix of block f (A_f, or A_f^H when c_out < c_in) and Vw the
 * (nc, nc) working-orientation right factors of already solved blocks (the V
 * output for tall blocks, the U output for wide ones).  No reference
 * counterpart: the reference solves every frequency from scratch. */
int cs_warm_start_gemm(const void *blocks, int dtype, int c_out, int c_in, long long count,
                       const long long *warm_ids, const long long *seed_ids, const void *Vw,
                       void *out_X, void *stream);

/* Heterogeneous batch in one call (cfg4: 16 layers, 4 shapes).  `groups` is a
 * HOST array; each group is solved like cs_batched_svd (with its own tol when
 * group.tol > 0, else the call's); groups run concurrently on forked streams
 * joined back into `stream`. */
typedef struct cs_svd_group {
    const void *blocks;
    long long count;
    int c_out, c_in;
    void *sigma, *U, *V;
    int *info, *zero_sigma;
    double tol;
} cs_svd_group;
size_t cs_batched_svd_grouped_workspace(const cs_svd_group *groups, int num_groups,
                                        int dtype, int want_vectors);
int cs_batched_svd_grouped(const cs_svd_group *groups, int num_groups, int dtype,
                           int want_vectors, double tol, int max_sweeps, void *workspace,
                           size_t workspace_bytes, void *stream);

/* Orthonormal fill of U columns whose sigma is exactly zero, for blocks with
 * zero_sigma[f] != 0.  Replaces blocksvd.py:184-198 (_complete_zero_columns).
 * U here is the factor of the WORKING (tall) matrix: (count, mr, r). */
int cs_complete_zero_columns(void *U, int dtype, long long count, int mr, int r,
                             const void *sigma, const int *zero_sigma, void *stream);

/* First index f with info[f] < 0, written to *first (-1 if none).  Feeds the
 * ConvergenceFailure message of blocksvd.py:213-224. */
int cs_first_failure(const int *info, long long count, long long *first, void *stream);

/* Spectrum assembly: globally sorted descending singular values
 * (blocksvd.py:276 + sort_descending :69-72), as float64.
 *   sigma : (count, r) real per-block values of representatives [0, count)
 *   half_grid = 1: sigma covers the full half grid of an n x m torus and every
 *     non-self-conjugate representative is counted twice (its partner);
 *     half_grid = 0: values are taken as they are.
 *   values : (half_grid ? n*m*r : count*r) float64, descending */
size_t cs_spectrum_values_workspace(long long num_values, int dtype);
int cs_spectrum_values(const void *sigma, int dtype, long long count, int r, int n, int m,
                       int half_grid, double *values, void *workspace,
                       size_t workspace_bytes, void *stream);

/* Global singular vector of the unrolled periodic operator for one frequency
 * (grid indices fi, fj: k = (fi/n, fj/m)) and factor column `col` of `factor`
 * ((rows, r) row-major, the frequency's U or V): out[(x1*n + x2)*rows + ch] =
 * exp(2 pi i (k1 x2 + k2 x1))/sqrt(nm) factor[ch, col].  Replaces
 * blocksvd.py:292-311 (materialize_singular_vector). */
int cs_materialize_vector(const void *factor, int dtype, int rows, int r, int col, int fi,
                          int fj, int n, int m, void *out, void *stream);

/* Matrix-free periodic convolution y = A x on an n x m torus: x (m, n, c_in),
 * y (m, n, c_out) complex, W (c_out, c_in, k_h, k_w) real; fp64 accumulation.
 * Replaces explicit.py:149-178 (apply_conv_reference, periodic boundary). */
int cs_apply_conv(const void *W, int dtype, int c_out, int c_in, int k_h, int k_w, int n, int m,
                  const void *x, void *y, void *stream);

/* Spectrum post-processing (analysis.py:35-74), float64
 * device arrays, stream-ordered.
 *   cs_spectral_summary: stats[4] = max, min, sum, top (top = max if max > 0
 *     else 1); counts[64] = np.histogram(values, 64, range=(0, top)) exactly;
 *     edges[65] (optional) = np.linspace(0, top, 65).  n >= 1 (else CS_EINVAL:
 *     EmptySpectrum).  Replaces spectral_summary (analysis.py:35-53).
 *   cs_sort_descending_f64: out = values sorted descending (workspace from
 *     cs_analysis_workspace).
 *   cs_wasserstein1_sum: *out_sum = sum_i |a_i - b~_i| over the longer
 *     spectrum, both inputs sorted descending, the shorter resampled at its
 *     quantile positions as np.interp does; W1 = out_sum / max(La, Lb).
 *     Replaces wasserstein1 (analysis.py:56-74). */
size_t cs_analysis_workspace(long long n);
int cs_spectral_summary(const double *values, long long n, double *stats,
                        unsigned long long *counts, double *edges, void *workspace,
                        size_t workspace_bytes, void *stream);
int cs_sort_descending_f64(const double *in, double *out, long long n, void *workspace,
                           size_t workspace_bytes, void *stream);
int cs_wasserstein1_sum(const double *va, long long La, const double *vb, long long Lb,
                        double *out_sum, void *workspace, size_t workspace_bytes, void *stream);

/* FFT route to the symbol field (fft.py:103-151), the
 * paper's comparison baseline for K1:
 *   cs_fft_transform: emb (c_out*c_in, m, n) complex of dtype <- taps of each
 *     channel pair embedded at their wrapped torus offsets (collisions summed
 *     in tap order), then one forward 2D DFT per pair (cuFFT, exp(-2 pi i ..)).
 *     emb_bytes >= cs_fft_field_workspace(...).  Replaces fft.py:133-139.
 *   cs_fft_gather: out (F_u or n*m, c_out, c_in) <- coefficient
 *     (-j mod m, -i mod n) for block (i, j), representatives when half_grid=1
 *     (the layout of cs_symbol_field).  Replaces fft.py:141-146. */
size_t cs_fft_field_workspace(int dtype, int c_out, int c_in, int n, int m);
int cs_fft_transform(const void *W, int dtype, int c_out, int c_in, int k_h, int k_w, int n, int m,
                     void *emb, size_t emb_bytes, void *stream);
int cs_fft_gather(const void *emb, int dtype, int c_out, int c_in, int n, int m, int half_grid,
                  void *out, void *stream);

/* Device microbenchmarks for the roofline denominators: achieved FP32 / FP64
 * FMA rate in flop/s over `ms` milliseconds of a dependent-FMA kernel. */
double cs_measure_fma_peak(int dtype, int device);

#ifdef __cplusplus
}
#endif
#endif /* CONVSPECTRA_B200_H */
