// cs_warm.cu -- warm start across neighbouring frequencies.
//
// The symbol A_f varies smoothly with f, so the right singular basis of a
// neighbour f' is an excellent starting point: one-sided Jacobi on
// X' = X_f V_{f'} (working orientation, X = A or A^H) converges in 5-6
// sweeps instead of 12 on cfg5 blocks at the same accuracy (CPU study of the
// exact fp32 arithmetic), and V accumulates from V_{f'}
// so U/V come out directly.  This file forms X' for a batch with one tiled
// complex GEMM: out[i] = X_{wid[i]} . Vw[sid[i]].
#include "cs_common.cuh"

namespace cs {

constexpr int WG_TILE = 64, WG_K = 8, WG_THREADS = 256;

template <typename T>
__global__ void __launch_bounds__(WG_THREADS)
warm_gemm_kernel(const cplx_t<T> *__restrict__ blocks, int co, int ci, int wide,
                 const long long *__restrict__ wid, const long long *__restrict__ sid,
                 const cplx_t<T> *__restrict__ Vw, cplx_t<T> *__restrict__ out) {
    using T2 = cplx_t<T>;
    __shared__ T2 As[WG_K][WG_TILE + 1];  // As[k][row]
    __shared__ T2 Bs[WG_K][WG_TILE + 1];  // Bs[k][col]
    const int mr = wide ? ci : co, nc = wide ? co : ci;
    const long long item = blockIdx.z;
    const T2 *A = blocks + (size_t)wid[item] * co * ci;
    const T2 *V = Vw + (size_t)sid[item] * nc * nc;
    T2 *O = out + (size_t)item * mr * nc;
    const int row0 = blockIdx.y * WG_TILE, col0 = blockIdx.x * WG_TILE;
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    T accr[4][4], acci[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) accr[a][b] = acci[a][b] = (T)0;
    for (int k0 = 0; k0 < nc; k0 += WG_K) {
        for (int x = threadIdx.x; x < WG_K * WG_TILE; x += WG_THREADS) {
            // X tile: rows row0.., cols k0.. ; X[r][k] = A[r][k] or conj(A[k][r])
            int kk, rr;
            if (!wide) { rr = x / WG_K; kk = x % WG_K; }
            else { kk = x / WG_TILE; rr = x % WG_TILE; }
            const int r = row0 + rr, k = k0 + kk;
            T2 v = mk<T>(0, 0);
            if (r < mr && k < nc) {
                if (!wide) v = A[(size_t)r * ci + k];
                else { v = A[(size_t)k * ci + r]; v.y = -v.y; }
            }
            As[kk][rr] = v;
            const int kb = x / WG_TILE, cc = x % WG_TILE, c = col0 + cc, kv = k0 + kb;
            Bs[kb][cc] = (kv < nc && c < nc) ? V[(size_t)kv * nc + c] : mk<T>(0, 0);
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < WG_K; ++kk) {
            T2 av[4], bv[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) av[a] = As[kk][ty * 4 + a];
#pragma unroll
            for (int b = 0; b < 4; ++b) bv[b] = Bs[kk][tx * 4 + b];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    accr[a][b] += av[a].x * bv[b].x - av[a].y * bv[b].y;
                    acci[a][b] += av[a].x * bv[b].y + av[a].y * bv[b].x;
                }
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int r = row0 + ty * 4 + a;
        if (r >= mr) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int c = col0 + tx * 4 + b;
            if (c < nc) O[(size_t)r * nc + c] = mk<T>(accr[a][b], acci[a][b]);
        }
    }
}

}  // namespace cs

using namespace cs;

extern "C" int cs_warm_start_gemm(const void *blocks, int dtype, int c_out, int c_in,
                                  long long count, const long long *warm_ids,
                                  const long long *seed_ids, const void *Vw, void *out_X,
                                  void *stream) {
    if (count == 0) return CS_OK;
    if (!blocks || !warm_ids || !seed_ids || !Vw || !out_X)
        return fail(CS_EINVAL, "cs_warm_start_gemm: null pointer");
    if (c_out < 1 || c_in < 1 || count < 0 || count > 65535LL * 1024)
        return fail(CS_EINVAL, "cs_warm_start_gemm: bad dimensions");
    const int wide = c_out < c_in;
    const int mr = wide ? c_in : c_out, nc = wide ? c_out : c_in;
    cudaStream_t st = (cudaStream_t)stream;
    for (long long off = 0; off < count; off += 65535) {
        const long long cnt = lmin(65535, count - off);
        dim3 grid((nc + WG_TILE - 1) / WG_TILE, (mr + WG_TILE - 1) / WG_TILE, (unsigned)cnt);
        if (dtype == CS_F32)
            warm_gemm_kernel<float><<<grid, WG_THREADS, 0, st>>>(
                (const float2 *)blocks, c_out, c_in, wide, warm_ids + off, seed_ids + off,
                (const float2 *)Vw, (float2 *)out_X + (size_t)off * mr * nc);
        else if (dtype == CS_F64)
            warm_gemm_kernel<double><<<grid, WG_THREADS, 0, st>>>(
                (const double2 *)blocks, c_out, c_in, wide, warm_ids + off, seed_ids + off,
                (const double2 *)Vw, (double2 *)out_X + (size_t)off * mr * nc);
        else
            return fail(CS_EINVAL, "cs_warm_start_gemm: unknown dtype");
        int s = check_launch("warm_gemm_kernel");
        if (s) return s;
    }
    return CS_OK;
}
