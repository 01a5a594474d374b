// cs_common.cuh -- shared helpers of the B200 LFA-SVD library (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "../../include/convspectra_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "convspectra_b200 is built for sm_100a (B200) only"
#endif

namespace cs {

__host__ __device__ __forceinline__ long long lmin(long long a, long long b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ long long lmax(long long a, long long b) { return a > b ? a : b; }

// ---- error plumbing (thread-local last error, C-ABI status codes) ---------
void set_error(const std::string &msg);
int fail(int status, const std::string &msg);
int cuda_status(cudaError_t e, const char *what);

#define CS_CUDA_TRY(expr)                                   \
    do {                                                    \
        cudaError_t _e = (expr);                            \
        if (_e != cudaSuccess) return cs::cuda_status(_e, #expr); \
    } while (0)

inline int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_status(e, what);
    return CS_OK;
}

// ---- real/complex type traits --------------------------------------------
template <typename T> struct cplx;
template <> struct cplx<float> { using type = float2; };
template <> struct cplx<double> { using type = double2; };
template <typename T> using cplx_t = typename cplx<T>::type;

template <typename T> __host__ __device__ __forceinline__ cplx_t<T> mk(T r, T i) {
    cplx_t<T> z; z.x = r; z.y = i; return z;
}

__device__ __forceinline__ float dsqrt(float x) { return sqrtf(x); }
__device__ __forceinline__ double dsqrt(double x) { return sqrt(x); }
__device__ __forceinline__ float dhypot(float a, float b) { return hypotf(a, b); }
__device__ __forceinline__ double dhypot(double a, double b) { return hypot(a, b); }
__device__ __forceinline__ bool dfinite(float x) { return isfinite(x); }
__device__ __forceinline__ bool dfinite(double x) { return isfinite(x); }

// ---- half-grid (conjugate-orbit representative) index math ---
// Representatives f <= f* in row-major order:
//   row 0            : j in [0, h0)          h0 = m/2 + 1
//   rows 1..nmid     : all m columns         nmid = (n-1)/2
//   row n/2 (n even) : j in [0, h0)
struct HalfGrid {
    int n, m, h0, nmid;
    long long count;
    __host__ __device__ HalfGrid(int n_, int m_) : n(n_), m(m_) {
        h0 = m / 2 + 1;
        nmid = (n - 1) / 2;
        count = (long long)h0 + (long long)nmid * m + ((n % 2 == 0 && n > 1) ? h0 : 0);
        if (n == 1) count = h0;
    }
    // first representative index of grid row i (valid rows: 0..nmid, n/2)
    __host__ __device__ long long row_start(int i) const {
        if (i == 0) return 0;
        if (i <= nmid) return h0 + (long long)(i - 1) * m;
        return h0 + (long long)nmid * m;  // i == n/2, n even
    }
    __host__ __device__ int row_len(int i) const {
        if (i == 0) return h0;
        if (i <= nmid) return m;
        return h0;
    }
    // number of grid rows that hold representatives
    __host__ __device__ int rows() const { return (n == 1) ? 1 : (nmid + 1 + (n % 2 == 0 ? 1 : 0)); }
    // representative index -> (i, j)
    __host__ __device__ void ij(long long u, int &i, int &j) const {
        if (u < h0) { i = 0; j = (int)u; return; }
        long long v = u - h0;
        if (v < (long long)nmid * m) { i = 1 + (int)(v / m); j = (int)(v % m); return; }
        i = n / 2; j = (int)(v - (long long)nmid * m);
    }
};

__host__ __device__ inline long long half_grid_count(int n, int m) { return HalfGrid(n, m).count; }

}  // namespace cs
