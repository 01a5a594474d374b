// cs_spectrum.cu -- spectrum assembly and the small epilogue kernels.
//
//  * cs_spectrum_values: the reference's global merge
//      values = sort_descending(per_block.ravel())   (blocksvd.py:69-72, 276)
//    On the half grid every non-self-conjugate representative stands for
//    itself and its partner f* (sigma_{f*} = sigma_f), so its
//    values are emitted twice before one device radix sort (CUB, compiled
//    into this library) of all n*m*r values.  Equal values are
//    indistinguishable, so a descending key sort equals the reference's
//    stable sort.
//  * cs_first_failure: first f with info[f] < 0 (blocksvd.py:213-224).
//  * cs_complete_zero_columns: blocksvd.py:184-198 on the device.
//  * cs_measure_fma_peak: FFMA / DFMA throughput probe for the roofline.
#include <cub/device/device_radix_sort.cuh>

#include "cs_common.cuh"

namespace cs {

// self-conjugate representatives, ascending (at most 4)
static int self_conj_reps(int n, int m, long long out[4]) {
    const HalfGrid hg(n, m);
    int s = 0;
    const int is[2] = {0, n / 2};
    const int js[2] = {0, m / 2};
    for (int a = 0; a < ((n % 2 == 0) ? 2 : 1); ++a)
        for (int b = 0; b < ((m % 2 == 0) ? 2 : 1); ++b) {
            const int i = is[a], j = js[b];
            if (a == 1 && n == 1) continue;
            out[s++] = hg.row_start(i) + j;
        }
    // ascending insertion sort
    for (int x = 1; x < s; ++x)
        for (int y = x; y > 0 && out[y] < out[y - 1]; --y) {
            long long t = out[y]; out[y] = out[y - 1]; out[y - 1] = t;
        }
    return s;
}

struct SelfConj { long long v[4]; int s; };

template <typename T>
__global__ void gather_values_kernel(const T *__restrict__ sigma, long long count, int r,
                                     int half, SelfConj sc, T *__restrict__ flat) {
    const long long n1 = count * r;
    const long long n2 = half ? (count - sc.s) * r : 0;
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < n1 + n2;
         x += (long long)gridDim.x * blockDim.x) {
        if (x < n1) {
            flat[x] = sigma[x];
        } else {
            const long long d = (x - n1) / r, c = (x - n1) % r;
            long long u = d;
            for (int k = 0; k < sc.s; ++k)
                if (sc.v[k] <= u) ++u;  // skip self-conjugate representatives
            flat[x] = sigma[u * r + c];
        }
    }
}

template <typename T>
__global__ void widen_kernel(const T *__restrict__ src, long long nv, double *__restrict__ dst) {
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < nv;
         x += (long long)gridDim.x * blockDim.x)
        dst[x] = (double)src[x];
}

template <typename T>
static size_t values_ws(long long nv) {
    size_t temp = 0;
    cub::DeviceRadixSort::SortKeysDescending((void *)nullptr, temp, (const T *)nullptr,
                                             (T *)nullptr, (int64_t)nv);
    return 2 * ((nv * sizeof(T) + 255) & ~(size_t)255) + temp + 256;
}

template <typename T>
static int values_run(const void *sigma, long long count, int r, int n, int m, int half,
                      double *values, void *ws, size_t ws_bytes, cudaStream_t st) {
    SelfConj sc = {};
    long long nv = count * r;
    if (half) {
        if (count != half_grid_count(n, m))
            return fail(CS_EINVAL, "spectrum values: count does not match the half grid");
        sc.s = self_conj_reps(n, m, sc.v);
        nv = (long long)n * m * r;
    }
    if (nv == 0) return CS_OK;
    const size_t need = values_ws<T>(nv);
    if (!ws || ws_bytes < need) return fail(CS_ENOMEM, "spectrum values: workspace too small");
    char *p = (char *)ws;
    T *flat = (T *)p;
    p += (nv * sizeof(T) + 255) & ~(size_t)255;
    T *sorted = (T *)p;
    p += (nv * sizeof(T) + 255) & ~(size_t)255;
    size_t temp = need - 2 * ((nv * sizeof(T) + 255) & ~(size_t)255);
    const unsigned blocks = (unsigned)lmin((nv + 255) / 256, 148LL * 16);
    gather_values_kernel<T><<<blocks, 256, 0, st>>>((const T *)sigma, count, r, half, sc, flat);
    int s = check_launch("gather_values_kernel");
    if (s) return s;
    CS_CUDA_TRY(cub::DeviceRadixSort::SortKeysDescending((void *)p, temp, flat, sorted, (int64_t)nv,
                                                         0, (int)(sizeof(T) * 8), st));
    widen_kernel<T><<<blocks, 256, 0, st>>>(sorted, nv, values);
    return check_launch("widen_kernel");
}

__global__ void first_failure_kernel(const int *__restrict__ info, long long count,
                                     unsigned long long *best) {
    for (long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x; f < count;
         f += (long long)gridDim.x * blockDim.x)
        if (info[f] < 0) atomicMin(best, (unsigned long long)f);
}

__global__ void finish_failure_kernel(unsigned long long *best) {
    long long *out = reinterpret_cast<long long *>(best);
    if (*best == ~0ULL) *out = -1;
}

// blocksvd.py:184-198 for one block per CTA: for each column j with
// sigma_j == 0, try unit vectors e_t (t = 0..mr-1) orthogonalised against the
// current U; the first with norm > 0.5 becomes column j.
template <typename T>
__global__ void complete_zero_kernel(cplx_t<T> *U, long long count, int mr, int r,
                                     const T *__restrict__ sigma, const int *__restrict__ flag) {
    using T2 = cplx_t<T>;
    extern __shared__ __align__(16) unsigned char shm[];
    T2 *coef = reinterpret_cast<T2 *>(shm);  // r
    T2 *cand = coef + r;                     // mr
    __shared__ T red[32];
    __shared__ int done;
    for (long long f = blockIdx.x; f < count; f += gridDim.x) {
        if (!flag[f]) continue;
        T2 *M = U + (size_t)f * mr * r;
        for (int j = 0; j < r; ++j) {
            if (sigma[(size_t)f * r + j] > (T)0) continue;
            if (threadIdx.x == 0) done = 0;
            __syncthreads();
            for (int t = 0; t < mr && !done; ++t) {
                // coef_k = (U^H e_t)_k = conj(U[t,k])
                for (int k = threadIdx.x; k < r; k += blockDim.x) {
                    T2 v = M[(size_t)t * r + k];
                    coef[k] = mk<T>(v.x, -v.y);
                }
                __syncthreads();
                T part = 0;
                for (int row = threadIdx.x; row < mr; row += blockDim.x) {
                    T cr = (row == t) ? (T)1 : (T)0, cim = 0;
                    for (int k = 0; k < r; ++k) {
                        const T2 u = M[(size_t)row * r + k], c = coef[k];
                        cr -= u.x * c.x - u.y * c.y;
                        cim -= u.x * c.y + u.y * c.x;
                    }
                    cand[row] = mk<T>(cr, cim);
                    part += cr * cr + cim * cim;
                }
                for (int off = 16; off; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
                if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
                __syncthreads();
                if (threadIdx.x == 0) {
                    T tot = 0;
                    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
                    red[0] = dsqrt(tot);
                }
                __syncthreads();
                const T nrm = red[0];
                if (nrm > (T)0.5) {
                    for (int row = threadIdx.x; row < mr; row += blockDim.x) {
                        const T2 c = cand[row];
                        M[(size_t)row * r + j] = mk<T>(c.x / nrm, c.y / nrm);
                    }
                    if (threadIdx.x == 0) done = 1;
                }
                __syncthreads();
            }
        }
    }
}

template <typename T>
__global__ void fma_probe_kernel(T *out, int iters) {
    T a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
      a6 = a0 + 6, a7 = a0 + 7;
    const T b = (T)0.999999, c = (T)1e-7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            a0 = a0 * b + c; a1 = a1 * b + c; a2 = a2 * b + c; a3 = a3 * b + c;
            a4 = a4 * b + c; a5 = a5 * b + c; a6 = a6 * b + c; a7 = a7 * b + c;
        }
    }
    const T s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == (T)-1) out[0] = s;  // never true; keeps the chains live
}

template <typename T>
static double fma_peak(int device) {
    int sms = 0;
    cudaSetDevice(device);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    T *out = nullptr;
    if (cudaMalloc(&out, sizeof(T)) != cudaSuccess) return -1;
    const int threads = 512, blocks = sms * 4, iters = sizeof(T) == 4 ? 20000 : 5000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    fma_probe_kernel<T><<<blocks, threads>>>(out, 100);  // warm-up
    cudaEventRecord(e0);
    fma_probe_kernel<T><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (cudaGetLastError() != cudaSuccess || ms <= 0) return -1;
    const double flops = 2.0 * 8 * 4 * (double)iters * threads * blocks;
    return flops / (ms * 1e-3);
}

}  // namespace cs

using namespace cs;

extern "C" size_t cs_spectrum_values_workspace(long long num_values, int dtype) {
    if (num_values <= 0) return 0;
    return dtype == CS_F32 ? values_ws<float>(num_values) : values_ws<double>(num_values);
}

extern "C" int cs_spectrum_values(const void *sigma, int dtype, long long count, int r, int n,
                                  int m, int half_grid, double *values, void *workspace,
                                  size_t workspace_bytes, void *stream) {
    if (count < 0 || r < 0) return fail(CS_EINVAL, "spectrum values: bad sizes");
    if (count && (!sigma || !values)) return fail(CS_EINVAL, "spectrum values: null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == CS_F32)
        return values_run<float>(sigma, count, r, n, m, half_grid, values, workspace,
                                 workspace_bytes, st);
    if (dtype == CS_F64)
        return values_run<double>(sigma, count, r, n, m, half_grid, values, workspace,
                                  workspace_bytes, st);
    return fail(CS_EINVAL, "spectrum values: unknown dtype");
}

extern "C" int cs_first_failure(const int *info, long long count, long long *first,
                                void *stream) {
    if (!first || (count && !info)) return fail(CS_EINVAL, "cs_first_failure: null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    CS_CUDA_TRY(cudaMemsetAsync(first, 0xff, sizeof(long long), st));
    if (count > 0) {
        const unsigned blocks = (unsigned)lmin((count + 255) / 256, 1024);
        first_failure_kernel<<<blocks, 256, 0, st>>>(info, count, (unsigned long long *)first);
        int s = check_launch("first_failure_kernel");
        if (s) return s;
    }
    finish_failure_kernel<<<1, 1, 0, st>>>((unsigned long long *)first);
    return check_launch("finish_failure_kernel");
}

extern "C" int cs_complete_zero_columns(void *U, int dtype, long long count, int mr, int r,
                                        const void *sigma, const int *zero_sigma, void *stream) {
    if (count == 0) return CS_OK;
    if (!U || !sigma || !zero_sigma) return fail(CS_EINVAL, "cs_complete_zero_columns: null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned blocks = (unsigned)lmin(count, 1024);
    if (dtype == CS_F32) {
        const size_t shm = (size_t)(mr + r) * sizeof(float2);
        complete_zero_kernel<float><<<blocks, 256, shm, st>>>((float2 *)U, count, mr, r,
                                                             (const float *)sigma, zero_sigma);
    } else if (dtype == CS_F64) {
        const size_t shm = (size_t)(mr + r) * sizeof(double2);
        complete_zero_kernel<double><<<blocks, 256, shm, st>>>((double2 *)U, count, mr, r,
                                                              (const double *)sigma, zero_sigma);
    } else {
        return fail(CS_EINVAL, "cs_complete_zero_columns: unknown dtype");
    }
    return check_launch("complete_zero_kernel");
}

extern "C" double cs_measure_fma_peak(int dtype, int device) {
    return dtype == CS_F64 ? fma_peak<double>(device) : fma_peak<float>(device);
}
