// cs_symbol.cu -- K1: LFA symbol assembly on the (half) frequency grid.
//
// Replaces the reference's build_symbol_field -> numba _symbol_blocks
// (pkg/src/convspectra/symbol.py:89-105, 108-137):
//     A_f[o,c] = sum_{p,q} W[o,c,p,q] * exp(+2 pi i (i*y_w(q)/n + j*y_h(p)/m))
// with f = i*m + j, y_h = p - k_h/2, y_w = q - k_w/2 (kernels.py:71-85,
// symbol.py:68-71).
//
// B200 design: the work is HBM-store bound (8 B written per complex64 entry,
// W is read once and stays in L2).  The phase is separable, so per grid row i
// a thread forms G_p = sum_q W[o,c,p,q] w_n^{i y_w(q)} once (k_h complex
// values in registers) and then emits every column j of its chunk with
// k_h complex MACs: A = sum_p w_m^{j y_h(p)} G_p.  Phases are reduced exactly
// in integers ((i*y) mod n) and evaluated with sincospi in fp64, so the
// per-tap phase is correctly rounded regardless of dtype.  Each thread owns
// two consecutive (o,c) entries -> one 16-byte vector store per frequency
// (fp32), and a warp writes 512 contiguous bytes per frequency.  Only the
// conjugate-orbit representatives are produced (half_grid=1); the partner
// block is conj() and never touches HBM.
#include "cs_common.cuh"

namespace cs {

constexpr int K1_THREADS = 256;
constexpr int K1_JC = 256;      // grid columns j per CTA (W and G_p reused across them):
                                // 64 -> 256 took cfg5 from 4.97 to 6.43 TB/s (tools/k1_tune.cu)
constexpr int K1_KHMAX = 8;     // separable path handles k_h <= 8

__device__ __forceinline__ long long imod(long long a, long long n) {
    long long r = a % n;
    return r < 0 ? r + n : r;
}

// exp(2 pi i e / n) for integer e reduced mod n, evaluated in fp64
__device__ __forceinline__ double2 unit_phase(long long e, long long n) {
    double s, c;
    sincospi(2.0 * (double)imod(e, n) / (double)n, &s, &c);
    return make_double2(c, s);
}

template <typename T, int EPT, int KH>
__global__ void __launch_bounds__(K1_THREADS)
symbol_rows_kernel(const T *__restrict__ W, int co, int ci, int kw, int n, int m,
                   long long f_first, long long f_count, int half, int row0,
                   cplx_t<T> *__restrict__ out) {
    using T2 = cplx_t<T>;
    __shared__ double2 rowph[16];                 // w_n^{i*y_w(q)}, q < k_w (<= 16)
    __shared__ T2 colph[K1_JC][K1_KHMAX];         // w_m^{j*y_h(p)}, rounded to T
    const HalfGrid hg(n, m);
    const int i = row0 + blockIdx.y;
    const long long base = half ? hg.row_start(i) : (long long)i * m;
    const int rlen = half ? hg.row_len(i) : m;
    const int j0 = blockIdx.z * K1_JC;
    // clip the chunk to the requested [f_first, f_first + f_count) window
    const long long u_lo = base + j0;
    int jn = min(K1_JC, rlen - j0);
    int jskip = 0;
    if (u_lo < f_first) jskip = (int)lmin(f_first - u_lo, (long long)jn);
    const long long u_end = f_first + f_count;
    if (u_lo + jn > u_end) jn = (int)lmax(0, u_end - u_lo);
    if (jskip >= jn) return;

    const int t = threadIdx.x;
    if (t < kw) rowph[t] = unit_phase((long long)i * (t - kw / 2), n);
    for (int x = t; x < K1_JC * KH; x += K1_THREADS) {
        const int jj = x / KH, p = x % KH;
        const double2 z = unit_phase((long long)(j0 + jj) * (p - KH / 2), m);
        colph[jj][p] = mk<T>((T)z.x, (T)z.y);
    }
    __syncthreads();

    const long long nel = (long long)co * ci;
    const long long e0 = ((long long)blockIdx.x * K1_THREADS + t) * EPT;
    if (e0 >= nel) return;
    const int ne = (int)lmin(EPT, nel - e0);

    // G_p for each of this thread's entries (fp64 sums, rounded to T once)
    T2 G[EPT][KH];
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
#pragma unroll
        for (int p = 0; p < KH; ++p) {
            double gr = 0.0, gi = 0.0;
            if (e < ne) {
                const T *w = W + (e0 + e) * (long long)(KH * kw) + p * kw;
                for (int q = 0; q < kw; ++q) {
                    const double wv = (double)w[q];
                    gr += wv * rowph[q].x;
                    gi += wv * rowph[q].y;
                }
            }
            G[e][p] = mk<T>((T)gr, (T)gi);
        }
    }
    for (int jj = jskip; jj < jn; ++jj) {
        T2 v[EPT];
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
            T ar = 0, ai = 0;
#pragma unroll
            for (int p = 0; p < KH; ++p) {
                const T2 ph = colph[jj][p];
                ar += ph.x * G[e][p].x - ph.y * G[e][p].y;
                ai += ph.x * G[e][p].y + ph.y * G[e][p].x;
            }
            v[e] = mk<T>(ar, ai);
        }
        T2 *dst = out + (base + j0 + jj - f_first) * nel + e0;
        if (EPT == 2 && ne == 2) {
            if (sizeof(T) == 4) {
                // streaming store: the field is written once, read by the next kernel
                __stcs(reinterpret_cast<float4 *>(dst),
                       make_float4((float)v[0].x, (float)v[0].y, (float)v[1].x, (float)v[1].y));
            } else {
                dst[0] = v[0];
                dst[1] = v[1];
            }
        } else {
#pragma unroll
            for (int e = 0; e < EPT; ++e)
                if (e < ne) dst[e] = v[e];
        }
    }
}

// Direct form, one output entry per thread-iteration: explicit frequencies
// (symbol_at / sub-grids), the frequency_strided layout and k_h > 8.
// mode 0: grid frequencies (full or half indexing); mode 1: explicit (k1,k2).
template <typename T>
__global__ void __launch_bounds__(K1_THREADS)
symbol_direct_kernel(const T *__restrict__ W, int co, int ci, int kh, int kw, int n, int m,
                     long long f_first, long long f_count, int half,
                     const double *__restrict__ freqs, int strided,
                     cplx_t<T> *__restrict__ out) {
    extern __shared__ double2 ph[];  // k_h*k_w phases of this CTA's frequency
    const long long u = blockIdx.y + (long long)blockIdx.z * 65535;  // one frequency per CTA row
    if (u >= f_count) return;
    const int T_ = kh * kw;
    for (int tp = threadIdx.x; tp < T_; tp += blockDim.x) {
        const int p = tp / kw, q = tp % kw;
        const int yh = p - kh / 2, yw = q - kw / 2;
        if (freqs) {
            const double k1 = freqs[2 * u], k2 = freqs[2 * u + 1];
            double s, c;
            sincospi(2.0 * (k1 * yw + k2 * yh), &s, &c);
            ph[tp] = make_double2(c, s);
        } else {
            const long long g = f_first + u;
            int i, j;
            if (half) {
                HalfGrid(n, m).ij(g, i, j);
            } else {
                i = (int)(g / m);
                j = (int)(g % m);
            }
            // exp(2 pi i (i*yw/n + j*yh/m)) = exp(2 pi i ((i*yw*m + j*yh*n) mod nm)/(nm))
            const long long nm = (long long)n * m;
            const long long e = imod((long long)i * yw * m + (long long)j * yh * n, nm);
            double s, c;
            sincospi(2.0 * (double)e / (double)nm, &s, &c);
            ph[tp] = make_double2(c, s);
        }
    }
    __syncthreads();
    const long long nel = (long long)co * ci;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nel;
         e += (long long)gridDim.x * blockDim.x) {
        const T *w = W + e * T_;
        double ar = 0.0, ai = 0.0;
        for (int tp = 0; tp < T_; ++tp) {
            const double wv = (double)w[tp];
            ar += ph[tp].x * wv;
            ai += ph[tp].y * wv;
        }
        const long long idx = strided ? e * f_count + u : u * nel + e;
        out[idx] = mk<T>((T)ar, (T)ai);
    }
}

template <typename T>
static int launch_symbol(const void *W, int co, int ci, int kh, int kw, int n, int m,
                         long long f_first, long long f_count, int half, void *out,
                         int layout, const double *freqs, cudaStream_t st) {
    using T2 = cplx_t<T>;
    const long long nel = (long long)co * ci;
    if (f_count == 0 || nel == 0) return CS_OK;
    const bool separable = !freqs && layout == CS_BLOCK_CONTIGUOUS && kh <= K1_KHMAX && kw <= 16;
    if (separable) {
        const HalfGrid hg(n, m);
        // rows intersecting [f_first, f_first + f_count)
        int r_lo, r_hi, jtmp;
        if (half) {
            hg.ij(f_first, r_lo, jtmp);
            hg.ij(f_first + f_count - 1, r_hi, jtmp);
        } else {
            r_lo = (int)(f_first / m);
            r_hi = (int)((f_first + f_count - 1) / m);
        }
        const int maxlen = half ? max(hg.h0, (hg.nmid > 0 ? m : 0)) : m;
        const int ept = (nel % 2 == 0) ? 2 : 1;
        dim3 grid((unsigned)((nel + (long long)K1_THREADS * ept - 1) / ((long long)K1_THREADS * ept)),
                  (unsigned)(r_hi - r_lo + 1), (unsigned)((maxlen + K1_JC - 1) / K1_JC));
        if (grid.y > 65535u || grid.z > 65535u)
            return fail(CS_EINVAL, "symbol field: torus too large for the row launch");
        const T *Wt = (const T *)W;
        T2 *o = (T2 *)out;
#define CS_K1_ROWS(KH_)                                                                     \
    case KH_:                                                                               \
        if (ept == 2)                                                                       \
            symbol_rows_kernel<T, 2, KH_><<<grid, K1_THREADS, 0, st>>>(                     \
                Wt, co, ci, kw, n, m, f_first, f_count, half, r_lo, o);                     \
        else                                                                                \
            symbol_rows_kernel<T, 1, KH_><<<grid, K1_THREADS, 0, st>>>(                     \
                Wt, co, ci, kw, n, m, f_first, f_count, half, r_lo, o);                     \
        break;
        switch (kh) {
            CS_K1_ROWS(1) CS_K1_ROWS(2) CS_K1_ROWS(3) CS_K1_ROWS(4)
            CS_K1_ROWS(5) CS_K1_ROWS(6) CS_K1_ROWS(7) CS_K1_ROWS(8)
        }
#undef CS_K1_ROWS
        return check_launch("symbol_rows_kernel");
    }
    const size_t shm = sizeof(double2) * (size_t)kh * kw;
    if (shm > 48 * 1024) return fail(CS_EINVAL, "symbol field: kernel extent too large");
    const unsigned gx = (unsigned)lmin((nel + K1_THREADS - 1) / K1_THREADS, 64);
    const long long gz = (f_count + 65534) / 65535;
    if (gz > 65535) return fail(CS_EINVAL, "symbol field: too many frequencies");
    dim3 grid(gx, (unsigned)lmin(f_count, 65535), (unsigned)gz);
    symbol_direct_kernel<T><<<grid, K1_THREADS, shm, st>>>(
        (const T *)W, co, ci, kh, kw, n, m, f_first, f_count, half, freqs,
        layout == CS_FREQUENCY_STRIDED, (T2 *)out);
    return check_launch("symbol_direct_kernel");
}

// half -> full grid with A_{f*} = conj(A_f)
template <typename T>
__global__ void expand_half_kernel(const cplx_t<T> *__restrict__ half, int n, int m,
                                   long long nel, cplx_t<T> *__restrict__ full) {
    const HalfGrid hg(n, m);
    const long long f = blockIdx.y + (long long)blockIdx.z * 65535;
    if (f >= (long long)n * m) return;
    const int i = (int)(f / m), j = (int)(f % m);
    const int is = (n - i) % n, js = (m - j) % m;
    const long long fs = (long long)is * m + js;
    const bool rep = f <= fs;
    const int ri = rep ? i : is, rj = rep ? j : js;
    const long long u = hg.row_start(ri) + rj;
    const cplx_t<T> *src = half + u * nel;
    cplx_t<T> *dst = full + f * nel;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nel;
         e += (long long)gridDim.x * blockDim.x) {
        cplx_t<T> v = src[e];
        if (!rep) v.y = -v.y;
        dst[e] = v;
    }
}

template <typename T>
__global__ void check_sym_kernel(const cplx_t<T> *__restrict__ full, int n, int m,
                                 long long nel, int *__restrict__ flag) {
    const long long f = blockIdx.y + (long long)blockIdx.z * 65535;
    if (f >= (long long)n * m) return;
    const int i = (int)(f / m), j = (int)(f % m);
    const long long fs = (long long)((n - i) % n) * m + (m - j) % m;
    if (f > fs) return;
    const cplx_t<T> *a = full + f * nel;
    const cplx_t<T> *b = full + fs * nel;
    bool ok = true;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nel;
         e += (long long)gridDim.x * blockDim.x) {
        const cplx_t<T> x = a[e], y = b[e];
        if (!(x.x == y.x && x.y == -y.y)) ok = false;  // NaN never compares equal
    }
    if (!ok) atomicExch(flag, 0);
}

}  // namespace cs

using namespace cs;

extern "C" int cs_symbol_field(const void *W, int dtype, int c_out, int c_in, int k_h, int k_w,
                               int n, int m, long long f_first, long long f_count,
                               int half_grid, void *out, int layout, void *stream) {
    if (!W || !out) return fail(CS_EINVAL, "cs_symbol_field: null pointer");
    if (c_out < 1 || c_in < 1 || k_h < 1 || k_w < 1 || n < 1 || m < 1)
        return fail(CS_EINVAL, "cs_symbol_field: all dimensions must be >= 1");
    if (layout != CS_BLOCK_CONTIGUOUS && layout != CS_FREQUENCY_STRIDED)
        return fail(CS_EINVAL, "cs_symbol_field: unknown layout");
    const long long total = half_grid ? half_grid_count(n, m) : (long long)n * m;
    if (f_first < 0 || f_count < 0 || f_first + f_count > total)
        return fail(CS_EINVAL, "cs_symbol_field: frequency range out of bounds");
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == CS_F32)
        return launch_symbol<float>(W, c_out, c_in, k_h, k_w, n, m, f_first, f_count,
                                    half_grid, out, layout, nullptr, st);
    if (dtype == CS_F64)
        return launch_symbol<double>(W, c_out, c_in, k_h, k_w, n, m, f_first, f_count,
                                     half_grid, out, layout, nullptr, st);
    return fail(CS_EINVAL, "cs_symbol_field: unknown dtype");
}

extern "C" int cs_symbol_at(const void *W, int dtype, int c_out, int c_in, int k_h, int k_w,
                            const double *freqs, long long count, void *out, void *stream) {
    if (!W || !out || (!freqs && count)) return fail(CS_EINVAL, "cs_symbol_at: null pointer");
    if (c_out < 1 || c_in < 1 || k_h < 1 || k_w < 1)
        return fail(CS_EINVAL, "cs_symbol_at: all dimensions must be >= 1");
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == CS_F32)
        return launch_symbol<float>(W, c_out, c_in, k_h, k_w, 1, 1, 0, count, 0, out,
                                    CS_BLOCK_CONTIGUOUS, freqs, st);
    if (dtype == CS_F64)
        return launch_symbol<double>(W, c_out, c_in, k_h, k_w, 1, 1, 0, count, 0, out,
                                     CS_BLOCK_CONTIGUOUS, freqs, st);
    return fail(CS_EINVAL, "cs_symbol_at: unknown dtype");
}

static dim3 per_freq_grid(long long F, long long nel) {
    const unsigned gx = (unsigned)lmin((nel + 255) / 256, 16);
    const long long gy = lmin(F, 65535);
    const long long gz = (F + 65534) / 65535;
    return dim3(gx, (unsigned)gy, (unsigned)gz);
}

extern "C" int cs_expand_half_grid(const void *half, int dtype, int c_out, int c_in, int n,
                                   int m, void *full, void *stream) {
    if (!half || !full) return fail(CS_EINVAL, "cs_expand_half_grid: null pointer");
    if (c_out < 1 || c_in < 1 || n < 1 || m < 1)
        return fail(CS_EINVAL, "cs_expand_half_grid: dimensions must be >= 1");
    const long long nel = (long long)c_out * c_in;
    const dim3 grid = per_freq_grid((long long)n * m, nel);
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == CS_F32)
        expand_half_kernel<float><<<grid, 256, 0, st>>>((const float2 *)half, n, m, nel, (float2 *)full);
    else if (dtype == CS_F64)
        expand_half_kernel<double><<<grid, 256, 0, st>>>((const double2 *)half, n, m, nel, (double2 *)full);
    else
        return fail(CS_EINVAL, "cs_expand_half_grid: unknown dtype");
    return check_launch("expand_half_kernel");
}

extern "C" int cs_check_conj_symmetry(const void *full, int dtype, int c_out, int c_in, int n,
                                      int m, int *flag, void *stream) {
    if (!full || !flag) return fail(CS_EINVAL, "cs_check_conj_symmetry: null pointer");
    const long long nel = (long long)c_out * c_in;
    cudaStream_t st = (cudaStream_t)stream;
    const int one = 1;
    CS_CUDA_TRY(cudaMemcpyAsync(flag, &one, sizeof(int), cudaMemcpyHostToDevice, st));
    const dim3 grid = per_freq_grid((long long)n * m, nel);
    if (dtype == CS_F32)
        check_sym_kernel<float><<<grid, 256, 0, st>>>((const float2 *)full, n, m, nel, flag);
    else if (dtype == CS_F64)
        check_sym_kernel<double><<<grid, 256, 0, st>>>((const double2 *)full, n, m, nel, flag);
    else
        return fail(CS_EINVAL, "cs_check_conj_symmetry: unknown dtype");
    return check_launch("check_sym_kernel");
}

extern "C" long long cs_half_grid_count(int n, int m) {
    if (n < 1 || m < 1) return 0;
    return half_grid_count(n, m);
}
