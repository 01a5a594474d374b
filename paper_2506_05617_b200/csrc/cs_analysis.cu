// cs_analysis.cu -- spectrum post-processing on the device (SURVEY.md 8(f)
// row 2): the reference's spectral_summary and wasserstein1
// (pkg/src/convspectra/analysis.py:35-74), run on the already-sorted device
// spectrum (16.7M float64 values for cfg5) instead of a host numpy pass.
//
// Parity notes (numpy 2.x semantics the reference inherits):
//   * histogram: np.histogram(values, 64, range=(0, top)) -- bin edges are
//     np.linspace(0, top, 65) (edge_i = i * (top/64), last = top exactly),
//     bin index ((x - 0)/top)*64 truncated, then corrected by the edge
//     comparisons of numpy/lib/_histograms_impl.py; values outside [0, top]
//     are dropped.  Counts are exact integers.
//   * wasserstein1: both spectra sorted descending; the shorter is resampled
//     by np.interp at linspace(0, 1, L) positions (slope*(x - xp_j) + fp_j,
//     no FMA contraction, as numpy's compiled arr_interp); mean |a - b|.
//   * max / min / mean: exact max/min; sums are blocked fp64 reductions
//     (numpy sums pairwise: the means agree to a few ulp, not bitwise).
#include <cub/device/device_radix_sort.cuh>

#include "cs_common.cuh"

namespace cs {

constexpr int AN_THREADS = 256;
constexpr int AN_BLOCKS = 148 * 4;
constexpr int HIST_BINS = 64;

__device__ __forceinline__ void warp_minmaxsum(double &mx, double &mn, double &sm, int &nan) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, off));
        sm += __shfl_xor_sync(0xffffffffu, sm, off);
        nan |= __shfl_xor_sync(0xffffffffu, nan, off);
    }
}

// per-block partials: part[4*b + {0,1,2,3}] = max, min, sum, any-NaN
__global__ void __launch_bounds__(AN_THREADS) stats_partial_kernel(const double *__restrict__ v, long long n,
                                                                   double *__restrict__ part) {
    double mx = -INFINITY, mn = INFINITY, sm = 0.0;
    int nan = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double x = v[i];
        if (x != x) nan = 1;
        mx = fmax(mx, x);
        mn = fmin(mn, x);
        sm += x;
    }
    warp_minmaxsum(mx, mn, sm, nan);
    __shared__ double s[4][AN_THREADS / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        s[0][wid] = mx;
        s[1][wid] = mn;
        s[2][wid] = sm;
        s[3][wid] = nan;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < AN_THREADS / 32; ++w) {
            mx = fmax(mx, s[0][w]);
            mn = fmin(mn, s[1][w]);
            sm += s[2][w];
            nan |= s[3][w] != 0.0;
        }
        part[4 * blockIdx.x + 0] = mx;
        part[4 * blockIdx.x + 1] = mn;
        part[4 * blockIdx.x + 2] = sm;
        part[4 * blockIdx.x + 3] = nan;
    }
}

// one block: stats[0..3] = max, min, sum, top (np.max / np.min propagate NaN)
__global__ void stats_final_kernel(const double *__restrict__ part, int nblocks, double *__restrict__ stats) {
    if (threadIdx.x != 0) return;
    double mx = -INFINITY, mn = INFINITY, sm = 0.0;
    bool nan = false;
    for (int b = 0; b < nblocks; ++b) {
        mx = fmax(mx, part[4 * b]);
        mn = fmin(mn, part[4 * b + 1]);
        sm += part[4 * b + 2];
        nan |= part[4 * b + 3] != 0.0;
    }
    if (nan) mx = mn = NAN;
    stats[0] = mx;
    stats[1] = mn;
    stats[2] = sm;
    stats[3] = mx > 0.0 ? mx : 1.0;  // analysis.py:43 top = smax if smax > 0 else 1.0
}

// np.linspace(0, top, 65)[i]
__device__ __forceinline__ double hist_edge(int i, double top) {
    if (i == HIST_BINS) return top;
    return __dadd_rn(__dmul_rn((double)i, __ddiv_rn(top, (double)HIST_BINS)), 0.0);
}

__global__ void __launch_bounds__(AN_THREADS) histogram_kernel(const double *__restrict__ v, long long n,
                                                               const double *__restrict__ stats,
                                                               unsigned long long *__restrict__ counts,
                                                               double *__restrict__ edges) {
    __shared__ unsigned int h[HIST_BINS];
    __shared__ double e[HIST_BINS + 1];
    const double top = stats[3];
    for (int i = threadIdx.x; i < HIST_BINS; i += blockDim.x) h[i] = 0;
    for (int i = threadIdx.x; i <= HIST_BINS; i += blockDim.x) e[i] = hist_edge(i, top);
    __syncthreads();
    if (blockIdx.x == 0 && edges)
        for (int i = threadIdx.x; i <= HIST_BINS; i += blockDim.x) edges[i] = e[i];
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double x = v[i];
        if (!(x >= 0.0 && x <= top)) continue;  // keep = (a >= first) & (a <= last)
        const double f = __dmul_rn(__ddiv_rn(__dsub_rn(x, 0.0), top), (double)HIST_BINS);
        int idx = (int)f;
        if (idx == HIST_BINS) idx -= 1;
        if (x < e[idx]) idx -= 1;
        if (x >= e[idx + 1] && idx != HIST_BINS - 1) idx += 1;
        atomicAdd(&h[idx], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < HIST_BINS; i += blockDim.x)
        if (h[i]) atomicAdd(&counts[i], (unsigned long long)h[i]);
}

// np.linspace(0, 1, L)[q]
__device__ __forceinline__ double unit_linspace(long long q, long long L) {
    if (L == 1) return 0.0;
    if (q == L - 1) return 1.0;
    return __dadd_rn(__dmul_rn((double)q, __ddiv_rn(1.0, (double)(L - 1))), 0.0);
}

// |va[i] - vb_resampled[i]| partial sums: va descending (length L), vb
// descending (length Ls <= L).  vb_resampled = np.interp(t_L, t_Ls, vb[::-1])[::-1].
__global__ void __launch_bounds__(AN_THREADS) w1_partial_kernel(const double *__restrict__ va, long long L,
                                                                const double *__restrict__ vb, long long Ls,
                                                                double *__restrict__ part) {
    double sm = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < L;
         i += (long long)gridDim.x * blockDim.x) {
        double b;
        if (Ls == L) {
            b = vb[i];
        } else if (Ls == 1) {
            b = vb[0];
        } else {
            // ascending sample fp[j] = vb[Ls-1-j] at xp[j] = linspace(0,1,Ls)[j]
            const long long q = L - 1 - i;
            const double x = unit_linspace(q, L);
            long long j = (long long)(x * (double)(Ls - 1));
            if (j > Ls - 1) j = Ls - 1;
            if (j < 0) j = 0;
            while (j + 1 < Ls && unit_linspace(j + 1, Ls) <= x) ++j;
            while (j > 0 && unit_linspace(j, Ls) > x) --j;
            const double xj = unit_linspace(j, Ls);
            const double fj = vb[Ls - 1 - j];
            if (j == Ls - 1 || xj == x) {
                b = fj;
            } else {
                const double xj1 = unit_linspace(j + 1, Ls);
                const double fj1 = vb[Ls - 2 - j];
                const double slope = __ddiv_rn(__dsub_rn(fj1, fj), __dsub_rn(xj1, xj));
                b = __dadd_rn(__dmul_rn(slope, __dsub_rn(x, xj)), fj);
                if (b != b) {
                    b = __dadd_rn(__dmul_rn(slope, __dsub_rn(x, xj1)), fj1);
                    if (b != b && fj == fj1) b = fj;
                }
            }
        }
        sm += fabs(__dsub_rn(va[i], b));
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, off);
    __shared__ double s[AN_THREADS / 32];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = sm;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < AN_THREADS / 32; ++w) sm += s[w];
        part[blockIdx.x] = sm;
    }
}

__global__ void sum_final_kernel(const double *__restrict__ part, int nblocks, double *__restrict__ out) {
    if (threadIdx.x != 0) return;
    double sm = 0.0;
    for (int b = 0; b < nblocks; ++b) sm += part[b];
    *out = sm;
}

static unsigned an_blocks(long long n) {
    return (unsigned)lmax(1, lmin((n + AN_THREADS - 1) / AN_THREADS, (long long)AN_BLOCKS));
}

}  // namespace cs

using namespace cs;

extern "C" size_t cs_analysis_workspace(long long n) {
    size_t temp = 0;
    cub::DeviceRadixSort::SortKeysDescending((void *)nullptr, temp, (const double *)nullptr,
                                             (double *)nullptr, (int64_t)lmax(n, 1));
    return 4 * AN_BLOCKS * sizeof(double) + 256 + temp;
}

extern "C" int cs_spectral_summary(const double *values, long long n, double *stats,
                                   unsigned long long *counts, double *edges, void *workspace,
                                   size_t workspace_bytes, void *stream) {
    if (n <= 0) return fail(CS_EINVAL, "summary needs at least one singular value");
    if (!values || !stats || !counts || !workspace) return fail(CS_EINVAL, "cs_spectral_summary: null pointer");
    if (workspace_bytes < 4 * AN_BLOCKS * sizeof(double)) return fail(CS_ENOMEM, "cs_spectral_summary: workspace too small");
    cudaStream_t st = (cudaStream_t)stream;
    double *part = (double *)workspace;
    const unsigned nb = an_blocks(n);
    stats_partial_kernel<<<nb, AN_THREADS, 0, st>>>(values, n, part);
    stats_final_kernel<<<1, 32, 0, st>>>(part, (int)nb, stats);
    CS_CUDA_TRY(cudaMemsetAsync(counts, 0, HIST_BINS * sizeof(unsigned long long), st));
    histogram_kernel<<<nb, AN_THREADS, 0, st>>>(values, n, stats, counts, edges);
    return check_launch("histogram_kernel");
}

extern "C" int cs_sort_descending_f64(const double *in, double *out, long long n, void *workspace,
                                      size_t workspace_bytes, void *stream) {
    if (n <= 0) return CS_OK;
    if (!in || !out || !workspace) return fail(CS_EINVAL, "cs_sort_descending_f64: null pointer");
    size_t temp = 0;
    cub::DeviceRadixSort::SortKeysDescending((void *)nullptr, temp, in, out, (int64_t)n);
    if (workspace_bytes < temp) return fail(CS_ENOMEM, "cs_sort_descending_f64: workspace too small");
    CS_CUDA_TRY(cub::DeviceRadixSort::SortKeysDescending(workspace, temp, in, out, (int64_t)n, 0, 64,
                                                         (cudaStream_t)stream));
    return CS_OK;
}

extern "C" int cs_wasserstein1_sum(const double *va, long long La, const double *vb, long long Lb,
                                   double *out_sum, void *workspace, size_t workspace_bytes,
                                   void *stream) {
    if (La <= 0 || Lb <= 0) return fail(CS_EINVAL, "wasserstein1 needs nonempty spectra");
    if (!va || !vb || !out_sum || !workspace) return fail(CS_EINVAL, "cs_wasserstein1_sum: null pointer");
    if (workspace_bytes < AN_BLOCKS * sizeof(double)) return fail(CS_ENOMEM, "cs_wasserstein1_sum: workspace too small");
    if (La < Lb) {  // the longer one leads (analysis.py:65-66)
        const double *t = va; va = vb; vb = t;
        const long long l = La; La = Lb; Lb = l;
    }
    cudaStream_t st = (cudaStream_t)stream;
    double *part = (double *)workspace;
    const unsigned nb = an_blocks(La);
    w1_partial_kernel<<<nb, AN_THREADS, 0, st>>>(va, La, vb, Lb, part);
    sum_final_kernel<<<1, 32, 0, st>>>(part, (int)nb, out_sum);
    return check_launch("w1 kernels");
}
