// cs_fft.cu -- the FFT comparison route to the symbol field (SURVEY.md 8(f)
// row 3), replacing the reference's fft_symbol_field
// (pkg/src/convspectra/fft.py:103-151):
//   1. embed: every (out,in) channel pair's taps placed on the m x n torus at
//      their wrapped offsets ((p - k_h/2) mod m, (q - k_w/2) mod n), summed in
//      tap order on collisions (fft.py:136-138);
//   2. transform: one batched 2D forward DFT per pair (negative exponent,
//      fft.py:82-91) -- cuFFT, 64-bit plan (cfg5 is 2^32 points);
//   3. gather: block (i, j) is coefficient (a, b) = (-j mod m, -i mod n)
//      (fft.py:142-145), written for the conjugate-orbit representatives (or
//      the full grid) in the (F, c_out, c_in) layout K1 produces.  A 32 x 32
//      tile transpose through shared memory keeps both the reads (along b)
//      and the writes (along the channel pairs) coalesced.
// The reference times 1+2 as s_transform and 3 as s_copy; the two calls
// below let the host put a device event between them.
#include <cufft.h>

#include "cs_common.cuh"

namespace cs {

template <typename T>
__global__ void fft_embed_kernel(const T *__restrict__ W, long long pairs, int kh, int kw, int n, int m,
                                 cplx_t<T> *__restrict__ emb) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= pairs) return;
    const long long mn = (long long)m * n;
    cplx_t<T> *g = emb + e * mn;
    const T *w = W + e * (long long)kh * kw;
    for (int p = 0; p < kh; ++p) {
        const int a = (int)(((long long)(p - kh / 2) % m + m) % m);
        for (int q = 0; q < kw; ++q) {
            const int b = (int)(((long long)(q - kw / 2) % n + n) % n);
            g[(long long)a * n + b].x += w[p * kw + q];
        }
    }
}

constexpr int FT = 32;  // gather tile: 32 torus cells x 32 channel pairs

template <typename T>
__global__ void __launch_bounds__(FT * 8) fft_gather_kernel(const cplx_t<T> *__restrict__ emb, long long pairs,
                                                            int n, int m, int half,
                                                            cplx_t<T> *__restrict__ out) {
    __shared__ cplx_t<T> tile[FT][FT + 1];
    const HalfGrid hg(n, m);
    const int btiles = (n + FT - 1) / FT;
    const int a = (int)(blockIdx.x / btiles);
    const int b0 = (int)(blockIdx.x % btiles) * FT;
    const long long e0 = (long long)blockIdx.y * FT;
    const long long mn = (long long)m * n;
    const int tx = threadIdx.x % FT, ty = threadIdx.x / FT;  // 32 x 8
    // read: pair e0+r, cells (a, b0 + tx)
    for (int r = ty; r < FT; r += 8) {
        const long long e = e0 + r;
        const int b = b0 + tx;
        if (e < pairs && b < n) tile[r][tx] = emb[e * mn + (long long)a * n + b];
    }
    __syncthreads();
    // write: frequency of cell (a, b0 + r), pairs e0 + tx
    const int j = (m - a) % m;
    for (int r = ty; r < FT; r += 8) {
        const int b = b0 + r;
        if (b >= n) continue;
        const int i = (n - b) % n;
        long long dst;
        if (half) {
            const long long f = (long long)i * m + j;
            const long long fs = (long long)((n - i) % n) * m + (m - j) % m;
            if (f > fs) continue;  // not a representative: its block is the partner's conj
            dst = hg.row_start(i) + j;
        } else {
            dst = (long long)i * m + j;
        }
        const long long e = e0 + tx;
        if (e < pairs) out[dst * pairs + e] = tile[tx][r];
    }
}

static int cufft_status(cufftResult r, const char *what) {
    if (r == CUFFT_SUCCESS) return CS_OK;
    if (r == CUFFT_ALLOC_FAILED) return fail(CS_ENOMEM, std::string(what) + ": cuFFT allocation failed");
    return fail(CS_ECUDA, std::string(what) + ": cuFFT error " + std::to_string((int)r));
}

}  // namespace cs

using namespace cs;

extern "C" size_t cs_fft_field_workspace(int dtype, int c_out, int c_in, int n, int m) {
    if (c_out < 1 || c_in < 1 || n < 1 || m < 1) return 0;
    const size_t esz = dtype == CS_F32 ? 8 : 16;
    return (size_t)c_out * c_in * (size_t)n * m * esz;
}

extern "C" int cs_fft_transform(const void *W, int dtype, int c_out, int c_in, int k_h, int k_w, int n,
                                int m, void *emb, size_t emb_bytes, void *stream) {
    if (!W || !emb) return fail(CS_EINVAL, "cs_fft_transform: null pointer");
    if (c_out < 1 || c_in < 1 || k_h < 1 || k_w < 1 || n < 1 || m < 1)
        return fail(CS_EINVAL, "cs_fft_transform: all dimensions must be >= 1");
    if (dtype != CS_F32 && dtype != CS_F64) return fail(CS_EINVAL, "cs_fft_transform: unknown dtype");
    if (emb_bytes < cs_fft_field_workspace(dtype, c_out, c_in, n, m))
        return fail(CS_ENOMEM, "cs_fft_transform: embedding buffer too small");
    cudaStream_t st = (cudaStream_t)stream;
    const long long pairs = (long long)c_out * c_in;
    CS_CUDA_TRY(cudaMemsetAsync(emb, 0, cs_fft_field_workspace(dtype, c_out, c_in, n, m), st));
    const unsigned nb = (unsigned)((pairs + 255) / 256);
    if (dtype == CS_F32)
        fft_embed_kernel<float><<<nb, 256, 0, st>>>((const float *)W, pairs, k_h, k_w, n, m, (float2 *)emb);
    else
        fft_embed_kernel<double><<<nb, 256, 0, st>>>((const double *)W, pairs, k_h, k_w, n, m, (double2 *)emb);
    int s = check_launch("fft_embed_kernel");
    if (s) return s;
    cufftHandle plan;
    if ((s = cufft_status(cufftCreate(&plan), "cufftCreate"))) return s;
    long long dims[2] = {m, n};  // row-major (m, n) grid per pair
    size_t work = 0;
    const cufftType ty = dtype == CS_F32 ? CUFFT_C2C : CUFFT_Z2Z;
    s = cufft_status(cufftMakePlanMany64(plan, 2, dims, nullptr, 1, 0, nullptr, 1, 0, ty, pairs, &work),
                     "cufftMakePlanMany64");
    if (!s) s = cufft_status(cufftSetStream(plan, st), "cufftSetStream");
    if (!s) {
        if (dtype == CS_F32)
            s = cufft_status(cufftExecC2C(plan, (cufftComplex *)emb, (cufftComplex *)emb, CUFFT_FORWARD),
                             "cufftExecC2C");
        else
            s = cufft_status(cufftExecZ2Z(plan, (cufftDoubleComplex *)emb, (cufftDoubleComplex *)emb,
                                          CUFFT_FORWARD), "cufftExecZ2Z");
    }
    cufftDestroy(plan);  // stream-ordered work already enqueued stays valid
    return s;
}

extern "C" int cs_fft_gather(const void *emb, int dtype, int c_out, int c_in, int n, int m, int half_grid,
                             void *out, void *stream) {
    if (!emb || !out) return fail(CS_EINVAL, "cs_fft_gather: null pointer");
    if (c_out < 1 || c_in < 1 || n < 1 || m < 1)
        return fail(CS_EINVAL, "cs_fft_gather: all dimensions must be >= 1");
    const long long pairs = (long long)c_out * c_in;
    const long long gx = (long long)m * ((n + FT - 1) / FT);
    const long long gy = (pairs + FT - 1) / FT;
    if (gy > 65535) return fail(CS_EINVAL, "cs_fft_gather: too many channel pairs");
    dim3 grid((unsigned)gx, (unsigned)gy);
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == CS_F32)
        fft_gather_kernel<float><<<grid, FT * 8, 0, st>>>((const float2 *)emb, pairs, n, m, half_grid, (float2 *)out);
    else if (dtype == CS_F64)
        fft_gather_kernel<double><<<grid, FT * 8, 0, st>>>((const double2 *)emb, pairs, n, m, half_grid, (double2 *)out);
    else
        return fail(CS_EINVAL, "cs_fft_gather: unknown dtype");
    return check_launch("fft_gather_kernel");
}
