// cs_tcb.cuh -- building blocks of the tensor-core blocked one-sided Jacobi
// (K3 "tcb"): per super-round, the Gram of the CTA's panel pair on tcgen05,
// the rotations on that small Gram, and the rotation product applied to the
// panel pair [X; V] as a tcgen05 GEMM.  Replaces the per-rotation O(rows)
// updates of the reference's _jacobi_sweeps (blocksvd.py:110-120) with
//   G = P^H P            (64 x 64 real, K = X rows, 3xTF32)
//   w rounds on G, D = Q - I accumulated (D <- D J + (J - I))
//   P <- P + P D          (M = rows, N = K = 64 real, 3xTF32)
// The fixed point, tolerance test and rotation formula are the reference's
// (cs_jacobi.cuh rot_params / rot_apply); only where the O(rows) work runs
// changes.
//
// Shared-memory layouts (all tcgen05 K-major, 128-byte swizzle, measured in
// tools/tc_layout_probe.cu: the tf32 MN-major forms do not execute, K-major
// SW128 does, and the tensor core TRUNCATES fp32 operands to tf32, so the
// stored fp32 word itself is the "hi" operand and lo = x - trunc(x)):
//   panel pair: rows x 64 real columns as two 32-column atoms (a | b):
//     off(r, k) = (k>>5)*ATOM + (r>>3)*1024 + (r&7)*128 + ((((k&31)>>2) ^ (r&7))<<4) + (k&3)*4
//     (complex column c: real columns 2c (re), 2c+1 (im)); ATOM = rows*128.
//   Gram staging (transposed, K = rows): off(j, r) = (r>>5)*8K + (j>>3)*1024 + ...
//   update B operand D~ (N = 64 out, K = 64 in): same form as the staging.
#pragma once

#include "cs_panel.cuh"

namespace cs {
namespace tcb {

constexpr int W = 16;       // complex columns per panel
constexpr int N2 = 2 * W;   // complex columns of the panel pair
constexpr int KR = 2 * N2;  // real columns of the panel pair
constexpr int LDG = N2 + 1; // row stride of the complex G / D scratch

__device__ __forceinline__ uint32_t sw_off(int r, int k, uint32_t atom) {
    return (uint32_t)(k >> 5) * atom + (uint32_t)(r >> 3) * 1024u + (uint32_t)(r & 7) * 128u +
           ((uint32_t)(((k & 31) >> 2) ^ (r & 7)) << 4) + (uint32_t)(k & 3) * 4u;
}
// 16-byte chunk (4 real columns k4*4..k4*4+3) of row r
__device__ __forceinline__ uint32_t sw_chunk(int r, int k4, uint32_t atom) {
    return (uint32_t)(k4 >> 3) * atom + (uint32_t)(r >> 3) * 1024u + (uint32_t)(r & 7) * 128u +
           ((uint32_t)((k4 & 7) ^ (r & 7)) << 4);
}

// smem matrix descriptor: K-major, 128-byte swizzle, SBO = 1024 (8-row groups)
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           (1ull << 46) | (2ull << 61);
}
// kind::tf32, fp32 accumulate, K-major A and B
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
constexpr uint32_t IDESC_GRAM = idesc_tf32(128, 128);
constexpr uint32_t IDESC_CROSS = idesc_tf32(128, 64);  // S x [hi_b | lo_b]^T
constexpr uint32_t IDESC_UPD = idesc_tf32(128, 128);   // hi(P) x [hi(D); lo(D)]
constexpr uint32_t IDESC_UPD_LO = idesc_tf32(128, 64); // lo(P) x hi(D)

__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, q;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// A operand in tensor memory (lane = M row, one 32-bit column per K element), B in shared memory
__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, q;\n\t}" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
// 16 consecutive 32-bit columns of this thread's TMEM lane (warp w: lanes 32 (w & 3) + lane)
__device__ __forceinline__ void tmem_st16(uint32_t addr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(addr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// two such stores under one wait
__device__ __forceinline__ void tmem_st16x2(uint32_t a0, const uint32_t (&r)[16], uint32_t a1, const uint32_t (&q)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(a0),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(a1),
        "r"(q[0]), "r"(q[1]), "r"(q[2]), "r"(q[3]), "r"(q[4]), "r"(q[5]), "r"(q[6]), "r"(q[7]), "r"(q[8]), "r"(q[9]),
        "r"(q[10]), "r"(q[11]), "r"(q[12]), "r"(q[13]), "r"(q[14]), "r"(q[15])
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st16_nowait(uint32_t addr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(addr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// named barriers (id 1..15; 0 is __syncthreads) for the update's warp roles
__device__ __forceinline__ void named_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld16(uint32_t addr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
// two 32x32b.x16 loads (columns c and c + OFF of the same lanes) under one wait
template <int OFF>
__device__ __forceinline__ void tmem_ld16_pair(uint32_t addr, float (&v)[16], float (&w)[16]) {
    uint32_t r[16], q[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]),
          "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]), "=r"(q[15])
        : "r"(addr + OFF));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        v[i] = __uint_as_float(r[i]);
        w[i] = __uint_as_float(q[i]);
    }
}
__device__ __forceinline__ void tmem_ld16x2(uint32_t addr, float (&v)[16], float (&w)[16]) {
    tmem_ld16_pair<64>(addr, v, w);
}
__device__ __forceinline__ void tmem_ld16x2s(uint32_t addr, float (&v)[16], float (&w)[16]) {
    tmem_ld16_pair<16>(addr, v, w);
}
__device__ __forceinline__ float trunc_tf32(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }
// tf32 round-to-nearest (the residual of hi = trunc(x) has 13 significant
// bits; the tensor core would truncate it to 11 -- a bias that accumulates
// over super-rounds -- so it is rounded to tf32 here instead)
__device__ __forceinline__ float rna_tf32(float x) {
    // = cvt.rna.tf32.f32 (round to nearest, ties away from zero) for finite x, in two integer
    // instructions: ptxas expands the cvt into ~5 with an inf/nan pass-through, and the Gram staging
    // (16 of them per thread and stage) is instruction-issue bound.  Non-finite input is caught by the
    // exact fp32 column norms (rot_params), not here.
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
__device__ __forceinline__ float lo_tf32(float x) { return rna_tf32(x - trunc_tf32(x)); }
__device__ __forceinline__ float4 lo4(float4 x) {
    return make_float4(lo_tf32(x.x), lo_tf32(x.y), lo_tf32(x.z), lo_tf32(x.w));
}

// Gram stage: rows [r0, r0+64) of the X rows -> a transposed staging S whose
// MN "rows" 0..63 are the hi words (the raw fp32: the tensor core truncates)
// and rows 64..127 the lo parts of the 64 real columns.  S S^T then holds
// hi*hi (rows < 64, cols < 64) and hi*lo (rows < 64, cols >= 64) -- the
// 3xTF32 Gram in ONE M = N = 128 MMA per 8 rows, with the correction terms
// accumulated in their own TMEM columns (at their own scale); lo*hi is the
// transpose of hi*lo.  Layout: K-atom (32 rows) of 16 KB, row-group stride
// 1 KB, 128-byte swizzle.  Unit = 4 rows of one real column (conflict-free:
// a warp reads one row of 32 consecutive columns, a quarter-warp writes 8
// columns' 16-byte units).
template <int NT>
__device__ __forceinline__ void gram_stage(const unsigned char *P, uint32_t atom, int r0, unsigned char *stg) {
#pragma unroll
    for (int i = 0; i < 1024 / NT; ++i) {
        const int u = threadIdx.x + i * NT, j = u & 63, rq = u >> 6;
        float4 h;
        h.x = *reinterpret_cast<const float *>(P + sw_off(r0 + 4 * rq + 0, j, atom));
        h.y = *reinterpret_cast<const float *>(P + sw_off(r0 + 4 * rq + 1, j, atom));
        h.z = *reinterpret_cast<const float *>(P + sw_off(r0 + 4 * rq + 2, j, atom));
        h.w = *reinterpret_cast<const float *>(P + sw_off(r0 + 4 * rq + 3, j, atom));
        // round-to-nearest split (hi symmetric around x): the dropped lo*lo
        // term is then unbiased -- with the truncated hi it would be a
        // systematic positive term on the diagonal
        const float4 hr = make_float4(rna_tf32(h.x), rna_tf32(h.y), rna_tf32(h.z), rna_tf32(h.w));
        const float4 lr = make_float4(rna_tf32(h.x - hr.x), rna_tf32(h.y - hr.y), rna_tf32(h.z - hr.z),
                                      rna_tf32(h.w - hr.w));
        *reinterpret_cast<float4 *>(stg + sw_chunk(j, rq, 16384)) = hr;
        *reinterpret_cast<float4 *>(stg + sw_chunk(64 + j, rq, 16384)) = lr;
    }
}

// the 8 MMAs (K = 8 rows each) of one Gram stage into accumulator d (128 x 128)
__device__ __forceinline__ void gram_mma(uint32_t d, uint32_t stg_addr) {
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
        const uint64_t s = desc_sw128(stg_addr + (ks >> 2) * 16384 + (ks & 3) * 32);
        mma_tf32(d, s, s, IDESC_GRAM, ks ? 1u : 0u);
    }
}

// B operand of the update from D (complex N2 x N2, row = input column):
// Dt[n][k] with n = 2c'+part', k = 2c+part:  [re][re] = Dr, [re n][im k] = -Di,
// [im n][re k] = Di, [im][im] = Dr.  Stored as 128 "rows": hi(Dt) in rows
// 0..63, lo(Dt) in rows 64..127 (K-atoms of 16 KB), so hi(P) x [hi; lo]
// gives main | correction in one N = 128 MMA.
template <int NT>
__device__ __forceinline__ void build_bop(const float2 *Dm, unsigned char *B) {
#pragma unroll
    for (int e = 0; e < 4096 / NT; ++e) {
        const int x = threadIdx.x + e * NT, n = x >> 6, k = x & 63;
        const float2 dv = Dm[(k >> 1) * LDG + (n >> 1)];
        const float v = (n & 1) == 0 ? ((k & 1) == 0 ? dv.x : -dv.y) : ((k & 1) == 0 ? dv.y : dv.x);
        // round-to-nearest split of D: the panel's hi is the truncated word
        // (lo(P) >= 0 relative to P), so the dropped lo(P) lo(D) term is
        // unbiased only if lo(D) is symmetric -- a truncated split of D too
        // shrank column norms by ~2e-6 per solve (measured, cfg5)
        const float h = rna_tf32(v);
        *reinterpret_cast<float *>(B + sw_off(n, k, 16384)) = h;
        *reinterpret_cast<float *>(B + sw_off(64 + n, k, 16384)) = rna_tf32(v - h);
    }
}

// rotation pair of slot k in inner round r: cross rounds pair panel-a column
// k with panel-b column (k + r) mod W; full rounds are the circle method on
// all N2 columns (within a, within b and cross)
__device__ __forceinline__ void inner_pair(bool full, int k, int r, int &p, int &q) {
    if (full) {
        pair_cols(k, r, N2, p, q);
    } else {
        p = k;
        q = W + ((k + r) & (W - 1));
    }
}

}  // namespace tcb
}  // namespace cs
