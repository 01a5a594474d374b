// cs_warm.cu -- warm start across neighbouring frequencies.
//
// The symbol A_f varies smoothly with f, so the right singular basis of a
// neighbour f' is an excellent starting point: one-sided Jacobi on
// X' = X_f V_{f'} (working orientation, X = A or A^H) converges in 5-6
// sweeps instead of 12 on cfg5 blocks at the same accuracy (CPU study of the
// exact fp32 arithmetic), and V accumulates from V_{f'}
// so U/V come out directly.  This file forms X' for a batch with one tiled
// complex GEMM: out[i] = X_{wid[i]} . Vw[sid[i]].
#include <cstdlib>

#include <cuda.h>

#include "cs_tcb.cuh"

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

// ---------------------------------------------------------------------------
// Tensor-core path (fp32, tall blocks, mr % 128 == 0, nc % 64 == 0): the same
// out = X . V on the 5th-gen tensor cores, as a warp-specialised pipeline.
//
// Real form of the complex product with interleaved storage: a block row is
// the real vector [re0, im0, re1, im1, ...], so with k' = 2k + s and output
// real column n' = 2n + t
//   out_real[r][n'] = sum_k' A_real[r][k'] B[n'][k'],
//   B[2n][2k] = V_r[k][n], B[2n][2k+1] = -V_i[k][n],
//   B[2n+1][2k] = V_i[k][n], B[2n+1][2k+1] = V_r[k][n].
// A CTA owns 128 rows x 64 complex columns (a 128 x 128 real accumulator)
// and walks K in stages of 16 complex (32 real = one 128-byte swizzle atom):
//   * producer warp: TMA loads of the RAW fp32 tiles -- A (128 rows x 128 B,
//     SWIZZLE_128B: exactly the K-major layout tcgen05 reads) and V (16 rows
//     x 64 complex) -- into a 3-slot ring, one mbarrier (complete_tx) each;
//   * converter warps: lo(A) = rn_tf32(x - trunc(x)) elementwise in the same
//     swizzled layout (the raw word IS hi(A): the tensor core truncates fp32
//     operands to tf32), and B hi/lo (transposed, signs, round-to-nearest
//     split: the dropped lo(A) lo(B) term is unbiased) from the raw V tile;
//   * MMA warp: one elected thread issues hi.hi + hi.lo + lo.hi per K step
//     (3xTF32) into one of two TMEM accumulators (ping-pong), commits to the
//     accumulator's barrier and to the ring slot's "empty" barrier;
//   * read-back warps: tcgen05.ld of the finished accumulator, summed in fp32
//     registers (each stage's 96 real K terms in a fresh accumulator: keeping
//     all K in TMEM measured 5.5e-6 relative error, per stage ~3e-6), while
//     the tensor core already runs the next stage into the other one.
// ---------------------------------------------------------------------------
constexpr int TC_M = 128, TC_NC = 64, TC_KC = 16;   // rows, complex cols, complex K per stage
constexpr int TC_RING = 3;                          // raw/operand ring slots
constexpr int TC_RB_WARPS = 8, TC_CV_WARPS = 8;     // read-back, converter warps
#ifndef CS_WARM_MMAW
#define CS_WARM_MMAW 2
#endif
constexpr int TC_MMA_WARPS = CS_WARM_MMAW;  // MMA streams (N slices of the tile)
constexpr int TC_THREADS = 32 * (TC_RB_WARPS + TC_CV_WARPS + 1 + TC_MMA_WARPS);  // + producer
constexpr uint32_t TC_ARAW = 0, TC_ALO = 16384, TC_BHI = 32768, TC_BLO = 49152, TC_VRAW = 65536;
constexpr uint32_t TC_SLOT = 73728;                 // 72 KB, a multiple of 1 KB (SW128 alignment)
constexpr uint32_t TC_BAR_OFF = TC_RING * TC_SLOT;
constexpr size_t TC_SMEM = 1024 + TC_BAR_OFF + 256;  // + 1 KB alignment slack + barriers
constexpr uint32_t TC_TX = 16384 + 8192;            // A tile + V tile bytes per stage
constexpr uint32_t TC_IDESC = tcb::idesc_tf32(128, 128 / TC_MMA_WARPS);

// tf32 round-to-nearest (ties away, = cvt.rna.tf32.f32) for finite x in two
// integer ops; lo_rn(x) = rn(x - trunc(x)), the correction word of a raw
// fp32 operand that the tensor core truncates
__device__ __forceinline__ float rn_tf32(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
__device__ __forceinline__ float lo_rn(float x) {
    return rn_tf32(x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u));
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap *tm, int x, int y, uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(tm), "r"(x), "r"(y), "r"(mbar)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive1(uint64_t *bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}

template <int SPA>
__global__ void __launch_bounds__(TC_THREADS, 1)
warm_gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmV, int co,
                    int ci, long long count, const long long *__restrict__ wid,
                    const long long *__restrict__ sid, float2 *__restrict__ out) {
    extern __shared__ __align__(1024) unsigned char tsm_raw[];
    unsigned char *tsm = tsm_raw + ((1024u - (smem_u32(tsm_raw) & 1023u)) & 1023u);
    uint64_t *bar = reinterpret_cast<uint64_t *>(tsm + TC_BAR_OFF);
    // bar[0..2] full (TMA), [3..5] converted, [6..8] slot empty (MMA done),
    // [9,10] accumulator full, [11,12] accumulator drained
    uint64_t *full = bar, *conv = bar + 3, *empty = bar + 6, *accf = bar + 9, *acce = bar + 11;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar + 16);
    const int mr = co, nc = ci;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nstage = nc / TC_KC;              // K stages per tile
    const int mt = mr / TC_M, ntl = nc / TC_NC;  // tiles per item
    const long long ntiles = count * mt * ntl;
    constexpr int W_PROD = TC_RB_WARPS + TC_CV_WARPS, W_MMA = W_PROD + 1;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 32) {
        for (int i = 0; i < TC_RING; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&conv[i], 32 * TC_CV_WARPS);
            mbar_init(&empty[i], TC_MMA_WARPS);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&accf[i], TC_MMA_WARPS);
            mbar_init(&acce[i], TC_RB_WARPS);
        }
        fence_mbar_init();
    }
    if (tid == 32 * W_PROD) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmV) : "memory");
    }
    __syncthreads();
    tcb::tc_after_sync();
    const uint32_t tmem = *tmem_slot;
    const uint32_t base = smem_u32(tsm);
    // persistent: CTA b takes tiles b, b + grid, ...; tile -> (item, M tile, N tile)
    // with the item slowest, so the CTAs working at one time share items in L2.
    // Every role walks the same tiles and stages; g counts stages across tiles
    // (ring slot g % TC_RING, accumulator (g / SPA) & 1).
    auto decode = [&](long long t, long long &item, int &row0, int &col0) {
        item = t / (mt * ntl);
        const int sub = (int)(t % (mt * ntl));
        row0 = (sub / ntl) * TC_M;
        col0 = (sub % ntl) * TC_NC;
    };
    if (warp == W_PROD) {
        if (lane == 0) {
            unsigned g = 0;
            for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
                long long item; int row0, col0;
                decode(t, item, row0, col0);
                const int ya = (int)(wid[item] * (long long)mr) + row0;
                const int yv = (int)(sid[item] * (long long)nc);
                for (int s = 0; s < nstage; ++s, ++g) {
                    const int sl = g % TC_RING;
                    if (g >= TC_RING) mbar_wait(&empty[sl], ((g / TC_RING) - 1) & 1);
                    mbar_arrive_expect_tx(&full[sl], TC_TX);
                    const uint32_t sb = base + sl * TC_SLOT;
                    tma_2d(sb + TC_ARAW, &tmA, 2 * TC_KC * s, ya, smem_u32(&full[sl]));
                    tma_2d(sb + TC_VRAW, &tmV, 2 * col0, yv + TC_KC * s, smem_u32(&full[sl]));
                }
            }
        }
    } else if (warp >= W_MMA) {
        // MMA warps: stream h issues the N half h (B rows / accumulator columns
        // 64 h ..): one thread's tcgen05.mma stream completes ~285 cycles per
        // instruction at these shapes, streams of different warps overlap
        // (profiles/r02_tc_rate_probe.txt)
        const int h = warp - W_MMA;
        constexpr uint32_t NH = 128 / TC_MMA_WARPS;
        if (lane == 0) {
            unsigned g = 0;
            for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
                for (int s = 0; s < nstage; ++s, ++g) {
                    const int sl = g % TC_RING;
                    const unsigned grp = g / SPA, ab = grp & 1;
                    mbar_wait(&conv[sl], (g / TC_RING) & 1);
                    if (s % SPA == 0 && grp >= 2) mbar_wait(&acce[ab], ((grp >> 1) - 1) & 1);
                    tcb::tc_after_sync();
                    const uint32_t sb = base + sl * TC_SLOT, d = tmem + 128 * ab + NH * h;
                    const uint32_t bo = (NH / 8) * 1024 * h;  // B rows NH h.. (8-row groups of 1 KB)
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks) {
                        const uint64_t ah = tcb::desc_sw128(sb + TC_ARAW + ks * 32);
                        const uint64_t al = tcb::desc_sw128(sb + TC_ALO + ks * 32);
                        const uint64_t bh = tcb::desc_sw128(sb + TC_BHI + bo + ks * 32);
                        const uint64_t bl = tcb::desc_sw128(sb + TC_BLO + bo + ks * 32);
                        tcb::mma_tf32(d, ah, bh, TC_IDESC, (ks || s % SPA) ? 1u : 0u);
                        tcb::mma_tf32(d, ah, bl, TC_IDESC, 1u);
                        tcb::mma_tf32(d, al, bh, TC_IDESC, 1u);
                    }
                    if (s % SPA == SPA - 1) tcb::mma_commit(&accf[ab]);
                    tcb::mma_commit(&empty[sl]);
                }
            }
        }
    } else if (warp >= TC_RB_WARPS) {
        // converters (8 warps, two per scheduler: the conversion is a chain of
        // dependent integer/float ops per element)
        const int tc = tid - 32 * TC_RB_WARPS;
        const int n = tc & 63, kk = tc >> 6;  // output complex column n, complex K 4 kk .. 4 kk + 3
        unsigned g = 0;
        for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
            for (int s = 0; s < nstage; ++s, ++g) {
                const int sl = g % TC_RING;
                unsigned char *sp = tsm + sl * TC_SLOT;
                mbar_wait(&full[sl], (g / TC_RING) & 1);
                // lo(A): elementwise on the swizzled tile (layout-agnostic)
#pragma unroll
                for (int i = 0; i < 1024 / (32 * TC_CV_WARPS); ++i) {
                    const int u = tc + 32 * TC_CV_WARPS * i;
                    const float4 x = *reinterpret_cast<const float4 *>(sp + TC_ARAW + 16 * u);
                    *reinterpret_cast<float4 *>(sp + TC_ALO + 16 * u) =
                        make_float4(lo_rn(x.x), lo_rn(x.y), lo_rn(x.z), lo_rn(x.w));
                }
                // B hi/lo, rows 2n + p (p = 0: re out, 1: im out), real K chunk
                // c4 = 2 kk + j holds complex k = 4 kk + 2 j, +1.  Lanes alternate j
                // with bit 2 of n so a warp's 16-byte stores cover all 8 swizzle
                // positions (conflict-free)
                const float2 *vr = reinterpret_cast<const float2 *>(sp + TC_VRAW);  // [16 k][64 n]
                float2 v[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) v[j] = vr[(4 * kk + j) * TC_NC + n];
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const int j = ((n >> 2) ^ i) & 1;
                    const float2 v0 = j ? v[2] : v[0], v1 = j ? v[3] : v[1];
                    const int c4 = 2 * kk + j;
#pragma unroll
                    for (int p = 0; p < 2; ++p) {
                        const float4 x = p ? make_float4(v0.y, v0.x, v1.y, v1.x) : make_float4(v0.x, -v0.y, v1.x, -v1.y);
                        const float4 hh = make_float4(rn_tf32(x.x), rn_tf32(x.y), rn_tf32(x.z), rn_tf32(x.w));
                        const float4 ll = make_float4(rn_tf32(x.x - hh.x), rn_tf32(x.y - hh.y), rn_tf32(x.z - hh.z),
                                                      rn_tf32(x.w - hh.w));
                        const uint32_t off = tcb::sw_chunk(2 * n + p, c4, 0);
                        *reinterpret_cast<float4 *>(sp + TC_BHI + off) = hh;
                        *reinterpret_cast<float4 *>(sp + TC_BLO + off) = ll;
                    }
                }
                fence_proxy_async_smem();
                mbar_arrive1(&conv[sl]);
            }
        }
    } else {
        // read-back warps: TMEM lanes 32 (warp & 3).., real columns 64 (warp >> 2)..
        const int q = warp & 3, hcol = warp >> 2;
        const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16) + 64 * hcol;
        unsigned grp = 0;
        for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
            long long item; int row0, col0;
            decode(t, item, row0, col0);
            float acc[64];
#pragma unroll
            for (int i = 0; i < 64; ++i) acc[i] = 0.f;
            for (int s = 0; s < nstage / SPA; ++s, ++grp) {
                const unsigned ab = grp & 1;
                mbar_wait(&accf[ab], (grp >> 1) & 1);
                tcb::tc_after_sync();
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    float v[16];
                    tcb::tmem_ld16(tl + 128 * ab + 16 * h, v);
#pragma unroll
                    for (int i = 0; i < 16; ++i) acc[16 * h + i] += v[i];
                }
                tcb::tc_before_sync();
                __syncwarp();
                if (lane == 0) mbar_arrive1(&acce[ab]);
            }
            // interleaved accumulator columns: real col 2j = re, 2j+1 = im of complex col j
            float2 *orow = out + ((size_t)item * mr + row0 + 32 * q + lane) * nc + col0 + 32 * hcol;
#pragma unroll
            for (int i = 0; i < 64; i += 4)
                *reinterpret_cast<float4 *>(orow + i / 2) = make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]);
        }
    }
    tcb::tc_before_sync();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*TmapEncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                 const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static TmapEncodeFn tmap_encode() {
    static TmapEncodeFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<TmapEncodeFn>(p);
    }
    return fn;
}
// fp32 2D map over rows of `width` floats (row pitch = width * 4 B); the row
// count is an upper bound (only rows of valid block / seed ids are touched)
static bool make_tmap(CUtensorMap *tm, const void *ptr, uint64_t width, uint32_t box_w, uint32_t box_h,
                      CUtensorMapSwizzle sw) {
    TmapEncodeFn fn = tmap_encode();
    if (!fn) return false;
    const cuuint64_t dims[2] = {width, (cuuint64_t)1 << 31};
    const cuuint64_t strides[1] = {width * 4};
    const cuuint32_t box[2] = {box_w, box_h}, estr[2] = {1, 1};
    return fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(ptr), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
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
    const char *tcenv = std::getenv("CS_WARM_TC");  // "0": CUDA-core kernel
    if (dtype == CS_F32 && !wide && mr % TC_M == 0 && nc % TC_NC == 0 && !(tcenv && tcenv[0] == '0')) {
        CUtensorMap tmA, tmV;
        if (!make_tmap(&tmA, blocks, 2 * (uint64_t)c_in, 2 * TC_KC, TC_M, CU_TENSOR_MAP_SWIZZLE_128B) ||
            !make_tmap(&tmV, Vw, 2 * (uint64_t)nc, 2 * TC_NC, TC_KC, CU_TENSOR_MAP_SWIZZLE_NONE))
            return fail(CS_ECUDA, "cs_warm_start_gemm: cuTensorMapEncodeTiled failed");
#ifndef CS_WARM_SPA
#define CS_WARM_SPA 1
#endif
        auto kfn = warm_gemm_tc_kernel<CS_WARM_SPA>;
        CS_CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TC_SMEM));
        int dev = 0, nsm = 148;
        CS_CUDA_TRY(cudaGetDevice(&dev));
        CS_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        const long long ntiles = count * (mr / TC_M) * (nc / TC_NC);
        const int grid = (int)lmin(ntiles, (long long)nsm);
        kfn<<<grid, TC_THREADS, TC_SMEM, st>>>(tmA, tmV, c_out, c_in, count, warm_ids, seed_ids, (float2 *)out_X);
        int s = check_launch("warm_gemm_tc_kernel");
        if (s) return s;
        return CS_OK;
    }
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
