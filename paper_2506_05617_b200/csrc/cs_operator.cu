// cs_operator.cu -- global singular vectors and the matrix-free operator.
//
// the per-frequency factors define global singular
// vectors of the unrolled periodic convolution (blocksvd.py:292-311,
// materialize_singular_vector):
//     vec[(x1*n + x2)*c + ch] = exp(2 pi i (k1 x2 + k2 x1)) / sqrt(n m) * W[ch, col]
// (x1 row in [0,m), x2 column in [0,n)), and the operator itself can be
// applied without materialising the (n m c_out) x (n m c_in) matrix
// (explicit.py:149-178, apply_conv_reference, periodic boundary):
//     y[x1, x2, o] = sum_{p,q,c} W[o, c, p, q] x[(x1 + p - k_h/2) mod m, (x2 + q - k_w/2) mod n, c]
// Together they give the acceptance check ||A v - sigma u|| at sizes where the
// dense matrix is impossible (cfg5: 16.7M x 16.7M).
#include "cs_common.cuh"

namespace cs {

template <typename T>
__global__ void materialize_kernel(const cplx_t<T> *__restrict__ fac, int rows, int r, int col,
                                   int fi, int fj, int n, int m, cplx_t<T> *__restrict__ out) {
    const long long total = (long long)n * m * rows;
    const double norm = 1.0 / sqrt((double)n * m);
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int ch = (int)(idx % rows);
        const long long pos = idx / rows;
        const int x1 = (int)(pos / n), x2 = (int)(pos % n);
        // k1 = fi/n pairs with x2 (period n), k2 = fj/m with x1 (period m): exact reduction
        const long long nm = (long long)n * m;
        long long e = ((long long)fi * x2 % n) * m + ((long long)fj * x1 % m) * n;
        e %= nm;
        double s, c;
        sincospi(2.0 * (double)e / (double)nm, &s, &c);
        const cplx_t<T> w = fac[(size_t)ch * r + col];
        const double wr = (double)w.x, wi = (double)w.y;
        out[idx] = mk<T>((T)((c * wr - s * wi) * norm), (T)((c * wi + s * wr) * norm));
    }
}

// one thread per (position, output channel); the input neighbourhood of a
// position is shared by all output channels, W stays in L2
template <typename T>
__global__ void apply_conv_kernel(const T *__restrict__ W, int co, int ci, int kh, int kw, int n,
                                  int m, const cplx_t<T> *__restrict__ x,
                                  cplx_t<T> *__restrict__ y) {
    const long long total = (long long)n * m * co;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int o = (int)(idx % co);
        const long long pos = idx / co;
        const int x1 = (int)(pos / n), x2 = (int)(pos % n);
        double ar = 0.0, ai = 0.0;
        for (int p = 0; p < kh; ++p) {
            int r1 = (x1 + p - kh / 2) % m;
            if (r1 < 0) r1 += m;
            for (int q = 0; q < kw; ++q) {
                int r2 = (x2 + q - kw / 2) % n;
                if (r2 < 0) r2 += n;
                const cplx_t<T> *xs = x + ((size_t)r1 * n + r2) * ci;
                const T *wp = W + ((size_t)o * ci) * kh * kw + p * kw + q;
                for (int c = 0; c < ci; ++c) {
                    const double wv = (double)wp[(size_t)c * kh * kw];
                    ar += wv * (double)xs[c].x;
                    ai += wv * (double)xs[c].y;
                }
            }
        }
        y[idx] = mk<T>((T)ar, (T)ai);
    }
}

}  // namespace cs

using namespace cs;

extern "C" int cs_materialize_vector(const void *factor, int dtype, int rows, int r, int col,
                                     int fi, int fj, int n, int m, void *out, void *stream) {
    if (!factor || !out) return fail(CS_EINVAL, "cs_materialize_vector: null pointer");
    if (rows < 1 || r < 1 || n < 1 || m < 1) return fail(CS_EINVAL, "cs_materialize_vector: dimensions must be >= 1");
    if (col < 0 || col >= r) return fail(CS_EINVAL, "cs_materialize_vector: column out of range");
    const long long total = (long long)n * m * rows;
    const unsigned blocks = (unsigned)lmin((total + 255) / 256, 148LL * 32);
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == CS_F32)
        materialize_kernel<float><<<blocks, 256, 0, st>>>((const float2 *)factor, rows, r, col, fi, fj, n, m, (float2 *)out);
    else if (dtype == CS_F64)
        materialize_kernel<double><<<blocks, 256, 0, st>>>((const double2 *)factor, rows, r, col, fi, fj, n, m, (double2 *)out);
    else
        return fail(CS_EINVAL, "cs_materialize_vector: unknown dtype");
    return check_launch("materialize_kernel");
}

extern "C" int cs_apply_conv(const void *W, int dtype, int c_out, int c_in, int k_h, int k_w,
                             int n, int m, const void *x, void *y, void *stream) {
    if (!W || !x || !y) return fail(CS_EINVAL, "cs_apply_conv: null pointer");
    if (c_out < 1 || c_in < 1 || k_h < 1 || k_w < 1 || n < 1 || m < 1)
        return fail(CS_EINVAL, "cs_apply_conv: dimensions must be >= 1");
    const long long total = (long long)n * m * c_out;
    const unsigned blocks = (unsigned)lmin((total + 255) / 256, 148LL * 32);
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == CS_F32)
        apply_conv_kernel<float><<<blocks, 256, 0, st>>>((const float *)W, c_out, c_in, k_h, k_w, n, m, (const float2 *)x, (float2 *)y);
    else if (dtype == CS_F64)
        apply_conv_kernel<double><<<blocks, 256, 0, st>>>((const double *)W, c_out, c_in, k_h, k_w, n, m, (const double2 *)x, (double2 *)y);
    else
        return fail(CS_EINVAL, "cs_apply_conv: unknown dtype");
    return check_launch("apply_conv_kernel");
}
