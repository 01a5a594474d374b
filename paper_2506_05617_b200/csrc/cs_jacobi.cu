// cs_jacobi.cu -- planning + C-ABI entry points of the batched Jacobi SVD
// (kernels in cs_jacobi.cuh, instantiated per dtype in cs_jacobi_f{32,64}.cu).
//
// B200 mapping: one thread-block CLUSTER of C CTAs per matrix, persistent
// over the batch.  The tall working matrix X (mr x nc, X = A or A^H) and,
// with vectors, V (nc x nc) are split by ROWS across the C CTAs and stay in
// shared memory (column-major slices) for the whole solve; each thread keeps
// its RPL rows of the current column pair in registers from the reduction to
// the rotation.  C is the smallest cluster whose slices fit in 227 KB with at
// most 64 registers of row data per thread (fp32: 16x16 .. 128x128 on one
// CTA, 256x128 on 2, 256x256 + V on 8); a generic kernel that re-reads rows
// (shared or global memory) keeps every other size correct.
#include <algorithm>
#include <cstdlib>

#include "cs_jacobi.cuh"
#include "cs_panel.cuh"

// debugging only: per-CTA progress codes written by the panel kernel into
// mapped (pinned) host memory, readable while a kernel hangs
static int *g_debug_progress = nullptr;
extern "C" void cs_debug_progress(void *p) { g_debug_progress = (int *)p; }

namespace cs {

static int pow2ceil(int x) {
    int p = 1;
    while (p < x) p *= 2;
    return p;
}
static size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

static int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

// Run-time switches, all read here.  CS_GRAM_CHECK and
// CS_TCB select documented alternative paths that the tests compare with the
// default; the planner hooks (cluster size, generic kernel, the slower
// Gram-blocked / split-role variants) exist only in CS_EXPERIMENTS builds
// (tools/ab_build.sh).
struct Knobs {
    int gram_check = 1;  // CS_GRAM_CHECK: 0 = rotation-free final sweep, 2 = timing experiment
    bool tcb = true;     // CS_TCB=0: scalar panel kernel for warm-started 256 x 256 + V solves
    int panel_c = 0, generic_c = 0;  // experiments: force the panel cluster size / the generic kernel
    bool gram = false, split = false;  // experiments: opt-in panel variants
};
static Knobs knobs() {
    Knobs k;
    if (const char *e = std::getenv("CS_GRAM_CHECK")) k.gram_check = e[0] == '0' ? 0 : (e[0] == '2' ? 2 : 1);
    if (const char *e = std::getenv("CS_TCB")) k.tcb = e[0] != '0';
#ifdef CS_EXPERIMENTS
    if (const char *e = std::getenv("CS_PANEL_C")) k.panel_c = std::atoi(e);
    if (const char *e = std::getenv("CS_GENERIC_C")) k.generic_c = std::atoi(e);
    if (const char *e = std::getenv("CS_GRAM")) k.gram = e[0] == '1';
    k.split = std::getenv("CS_SPLIT") != nullptr;
#endif
    return k;
}

static void base_shape(int co, int ci, bool wantv, int C, JacShape &s) {
    s = JacShape{};
    const bool wide = co < ci;
    s.mr = wide ? ci : co;
    s.nc = wide ? co : ci;
    s.wide = wide;
    s.ncp = s.nc + (s.nc & 1);
    s.P = s.ncp / 2;
    s.C = C;
    s.R = (s.mr + C - 1) / C;
    s.Rv = wantv ? (s.nc + C - 1) / C : 0;
}

// Column stride of a slice (in complex elements).  In the circle ordering the
// pair slots of one warp hold consecutive columns (p0+g, q0-g), so with
// ld = G (mod W) -- W complex elements per 128-byte wavefront -- the lanes'
// addresses (p0+g)*ld + lane_g tile the 32 banks without conflicts.
static int pad_ld(int rows, int G, int elem_bytes) {
    const int W = 128 / elem_bytes;
    const int want = G % W;
    int ld = std::max(rows, 1);
    while (ld % W != want) ++ld;
    return ld;
}

template <typename T>
static bool plan_fast(int co, int ci, bool wantv, int C, JacShape &s) {
    base_shape(co, ci, wantv, C, s);
    s.kind = 0;
    const int rpl_target = sizeof(T) == 4 ? 8 : 4;
    const int rpl_max = sizeof(T) == 4 ? (wantv ? 8 : 16) : (wantv ? 4 : 8);
    int G = std::min(32, pow2ceil((s.R + rpl_target - 1) / rpl_target));
    while (s.P * G > JAC_MAX_THREADS && G > 1) G /= 2;
    int RPL = std::max(2, pow2ceil((s.R + G - 1) / G));
    while (s.P * G < 32 && G < 32 && RPL > 2) {  // fill at least one warp
        G *= 2;
        RPL = std::max(2, pow2ceil((s.R + G - 1) / G));
    }
    if (RPL > rpl_max || s.P * G > JAC_MAX_THREADS) return false;
    s.G = G;
    s.RPL = RPL;
    s.threads = ((s.P * G + 31) / 32) * 32;
    s.ldx = pad_ld(G * RPL, G, 2 * sizeof(T));
    s.ldv = wantv ? pad_ld(G * RPL, G, 2 * sizeof(T)) : 0;
    const size_t T2sz = 2 * sizeof(T), pb = sizeof(Part<T>);
    size_t off = 0;
    s.off_sig = off;
    off = align16(off + s.ncp * sizeof(T));
    s.off_perm = off;
    off = align16(off + 2 * s.ncp * sizeof(int));
    s.off_send = off;
    off = align16(off + (C > 1 ? 2 * (size_t)s.P * pb : 0));
    s.off_recv = off;
    off = align16(off + (C > 1 ? 2 * (size_t)C * s.P * pb : 0));
    s.off_mbar = off;
    off = align16(off + 2 * sizeof(uint64_t));
    s.off_x = off;
    off = align16(off + (size_t)s.ncp * s.ldx * T2sz);
    s.off_v = off;
    off = align16(off + (size_t)s.ncp * s.ldv * T2sz);
    s.smem = off;
    s.smem_resident = 1;
    s.nbuf = 2;
    return s.smem <= JAC_SMEM_LIMIT;
}

// Panel kernel (cs_panel.cuh): 2C column panels of w columns, whole columns
// of [X; V] per CTA; a-panel rows in registers, b panel (x2 when C > 1 for
// the cluster rotation) + a staging copy of the a panel in shared memory.
template <typename T>
static bool plan_panel(int co, int ci, bool wantv, int C, JacShape &s, const Knobs &kn) {
    base_shape(co, ci, wantv, C, s);
    s.kind = 2;
    s.ncp = ((s.nc + 4 * C - 1) / (4 * C)) * (4 * C);
    const int w = s.ncp / (2 * C);
    if (w > JAC_MAX_THREADS) return false;
    s.P = w;
    s.R = s.mr;
    s.Rv = wantv ? s.nc : 0;
    int G = 1;
    while (G * 2 <= 32 && w * G * 2 <= JAC_MAX_THREADS && G * 2 * 4 <= pow2ceil(s.mr)) G *= 2;
    const int rplx = std::max(2, pow2ceil((s.mr + G - 1) / G));
    // V rows per lane: nc rows (tall blocks: fewer than the mr X rows); fp32
    // panels carry rplx or rplx/2 (cs_jacobi_f32.cu instantiates both)
    const int rplv = !wantv ? 0
                     : (sizeof(T) == 4 ? std::max(rplx / 2, std::max(2, pow2ceil((s.nc + G - 1) / G))) : rplx);
    // complex rows per column held in registers; fp64 C = 16 panels run 256
    // threads (255 registers each) and take 16 (cfg5 in fp64, cs_jacobi_f64.cu)
    const int budget = sizeof(T) == 4 ? 16 : ((C == 16 && w * G <= 256 && wantv) ? 16 : 8);
    // with vectors, X and V rows go to separate warps when 2x the threads fit
    // (each thread then holds only one role's rows: budget/2 per role at 64 regs)
    s.split = (wantv && sizeof(T) == 4 && rplv == rplx && 2 * w * G <= 1024 && w * G % 32 == 0 &&
               rplx <= budget / 2 && kn.split) ? 1 : 0;  // opt-in: spills at 64 regs
    if (!s.split && rplx + rplv > budget) return false;
    s.G = G;
    s.RPL = rplx;
    s.threads = s.split ? 2 * w * G : ((w * G + 31) / 32) * 32;
    const int T2sz = 2 * sizeof(T);
    s.ldv = G * rplx;  // row offset of the V rows in a column
    s.ldx = pad_ld(G * (rplx + rplv), G, T2sz);
    size_t off = 0;
    s.off_sig = off;
    off = align16(off + s.ncp * sizeof(T));
    s.off_perm = off;
    off = align16(off + 2 * s.ncp * sizeof(int));
    s.off_send = off;  // staging for the cluster norm gather; Gram mode: G and D
    // Gram-blocked cross phase (opt-in CS_GRAM=1: correct, but 2.8x slower than the
    // scalar cross rounds on cfg5 in SIMT; kept as the skeleton for a tensor-core version)
    s.gram = (sizeof(T) == 4 && w == 16 && !s.split && kn.gram &&
              w * (s.mr + s.Rv) <= 16 * s.threads) ? 1 : 0;  // a-panel staging: 16 per thread
    const size_t gbytes = s.gram ? 2 * (size_t)(2 * w) * (2 * w + 1) * 2 * sizeof(T) : 0;
    off = align16(off + std::max(s.ncp * sizeof(T), gbytes));
    s.off_recv = off;  // split mode: rotation parameters [2][w]
    off = align16(off + 2 * (size_t)w * 4 * sizeof(T) + 64);
    s.off_mbar = off;  // sweep flags + panel position tables
    off = align16(off + (4 + 64) * sizeof(int));
    s.off_x = off;
    const size_t panel = (size_t)w * s.ldx * T2sz;
    off = align16(off + panel);
    s.off_v = off;
    off = align16(off + panel * (C > 1 ? 2 : 1));
    s.smem = off;
    s.smem_resident = 1;
    s.nbuf = 1;
    // "2" (timing experiment): check after every rotating sweep, ignore the verdict
    s.gcheck = (!s.split && !s.gram) ? kn.gram_check : 0;
    return s.smem <= JAC_SMEM_LIMIT;
}

template <typename T>
static bool plan_generic(int co, int ci, bool wantv, int C, bool smem_resident, JacShape &s) {
    base_shape(co, ci, wantv, C, s);
    s.kind = 1;
    const long long work = (long long)s.P * (s.R + s.Rv);
    s.threads = work >= 512LL * 8 ? 512 : (work >= 256LL * 4 ? 256 : 128);
    int G = 1;
    while (G * 2 <= std::max(1, s.threads / s.P) && G < 32) G *= 2;
    G = std::min(G, pow2ceil(std::max(s.R, 1)));
    s.G = std::max(G, 1);
    s.RPL = 0;
    s.ldx = pad_ld(((std::max(s.R, 1) + s.G - 1) / s.G) * s.G, s.G, 2 * sizeof(T));
    s.ldv = wantv ? pad_ld(((std::max(s.Rv, 1) + s.G - 1) / s.G) * s.G, s.G, 2 * sizeof(T)) : 0;
    const size_t T2sz = 2 * sizeof(T);
    const size_t part1 = (size_t)C * s.P * sizeof(Part<T>);
    for (int nbuf = 2; nbuf >= 1; --nbuf) {
        size_t off = 0;
        s.off_sig = off;
        off = align16(off + s.ncp * sizeof(T));
        s.off_perm = off;
        off = align16(off + 2 * s.ncp * sizeof(int));
        s.off_send = off;
        off = align16(off + part1 * nbuf);
        s.off_recv = s.off_mbar = off;
        s.off_x = off;
        if (smem_resident) {
            off = align16(off + (size_t)s.ncp * s.ldx * T2sz);
            s.off_v = off;
            off = align16(off + (size_t)s.ncp * s.ldv * T2sz);
        } else {
            s.off_v = off;
        }
        s.smem = off;
        s.nbuf = nbuf;
        s.smem_resident = smem_resident;
        s.scratch_per_cta = smem_resident ? 0 : (size_t)s.ncp * (s.ldx + s.ldv);
        if (s.smem <= JAC_SMEM_LIMIT) return true;
    }
    return false;
}

template <typename T>
static bool plan(int co, int ci, bool wantv, long long count, JacShape &s) {
    const int Cs[5] = {1, 2, 4, 8, 16};
    const Knobs kn = knobs();
    if (kn.panel_c) {  // experiment hook: force the cluster size
        if (plan_panel<T>(co, ci, wantv, kn.panel_c, s, kn)) return true;
    }
    if (kn.generic_c) {  // experiment hook: generic kernel, cluster C
        if (plan_generic<T>(co, ci, wantv, kn.generic_c, true, s)) return true;
        if (plan_generic<T>(co, ci, wantv, kn.generic_c, false, s)) return true;
    }
    for (int i = 0; i < 5; ++i) {
        if (!plan_panel<T>(co, ci, wantv, Cs[i], s, kn)) continue;
        // small batches: spread each matrix over more CTAs while fewer than
        // 4 CTAs per SM would be queued (cfg4's 394 128^2 blocks: C = 1 19.0 ms,
        // C = 2 12.0 ms, C = 4 13.4 ms; with a 2-per-SM cut they stayed at C = 1)
        int j = i;
        while (j < 4 && count * Cs[j] < 4LL * num_sms()) {
            JacShape t;  // panels narrower than 8 columns only add exchanges (cfg1 16^2)
            if (!plan_panel<T>(co, ci, wantv, Cs[j + 1], t, kn) || t.P < 8) break;
            ++j;
        }
        return plan_panel<T>(co, ci, wantv, Cs[j], s, kn);
    }
    for (int i = 0; i < 5; ++i) {
        if (!plan_fast<T>(co, ci, wantv, Cs[i], s)) continue;
        // few matrices: spread each over more SMs while rows per CTA stay >= 16
        int j = i;
        while (j < 4 && count * Cs[j] < 2LL * num_sms()) {
            JacShape t;
            if (!plan_fast<T>(co, ci, wantv, Cs[j + 1], t) || t.R < 16) break;
            ++j;
        }
        return plan_fast<T>(co, ci, wantv, Cs[j], s);
    }
    const int Cg[3] = {1, 8, 16};
    for (int i = 0; i < 3; ++i)
        if (plan_generic<T>(co, ci, wantv, Cg[i], true, s)) return true;
    return plan_generic<T>(co, ci, wantv, 8, false, s);
}

// tensor-core blocked kernel (cs_tcb.cu): fp32, vectors, instantiated shapes
bool tcb_supported(int mr, int nc, bool wantv);
size_t tcb_workspace(int mr, int nc, bool wantv);
int tcb_dispatch(const JacArgs<float> &a, void *ws, size_t ws_bytes, cudaStream_t st);
static bool tcb_enabled() { return knobs().tcb; }

template <typename T>
static int dispatch(const JacArgs<T> &a, bool wantv, cudaStream_t st, bool dry, long long *ncl) {
    if constexpr (sizeof(T) == 4) return jacobi_dispatch_f32(a, wantv, st, dry, ncl);
    else return jacobi_dispatch_f64(a, wantv, st, dry, ncl);
}

template <typename T>
static int svd_workspace(long long count, int co, int ci, bool wantv, size_t *bytes) {
    JacShape s;
    *bytes = 0;
    if (count <= 0) return CS_OK;
    if (!plan<T>(co, ci, wantv, count, s)) return fail(CS_EINVAL, "batched SVD: no plan");
    // warm-started solves of tcb shapes run the tensor-core kernel, whose
    // groups exchange panels through mailboxes in the workspace
    const size_t tcb_bytes = (sizeof(T) == 4 && tcb_enabled()) ? tcb_workspace(s.mr, s.nc, wantv) : 0;
    *bytes = tcb_bytes;
    if (s.smem_resident) return CS_OK;
    JacArgs<T> a = {};
    a.count = count;
    a.s = s;
    long long ncl = 0;
    int st = dispatch<T>(a, wantv, 0, true, &ncl);
    if (st) return st;
    *bytes = std::max(tcb_bytes, (size_t)ncl * s.C * s.scratch_per_cta * 2 * sizeof(T));
    return CS_OK;
}

template <typename T>
static int svd_run(const void *blocks, long long count, int co, int ci, bool wantv, double tol,
                   int max_sweeps, void *sigma, void *U, void *V, int *info, int *zero_sigma,
                   void *ws, size_t ws_bytes, cudaStream_t st, const long long *index = nullptr,
                   const void *initX = nullptr, const void *initV = nullptr,
                   const long long *initV_index = nullptr, long long plan_count = 0) {
    if (count == 0) return CS_OK;
    JacArgs<T> a = {};
    if (!plan<T>(co, ci, wantv, plan_count > 0 ? plan_count : count, a.s))
        return fail(CS_EINVAL, "batched SVD: no plan");
    if ((index || initX || initV) && a.s.kind != 2)
        return fail(CS_EINVAL, "batched SVD: indexed / warm-started solves need the panel kernel");
    if (initV && !(wantv && initV_index)) return fail(CS_EINVAL, "batched SVD: initV needs vectors and an index");
    a.index = index;
    a.initX = (const cplx_t<T> *)initX;
    a.initV = (const cplx_t<T> *)initV;
    a.initV_index = initV_index;
    a.blocks = (const cplx_t<T> *)blocks;
    a.count = count;
    a.co = co;
    a.ci = ci;
    a.tol = (T)tol;
    a.max_sweeps = max_sweeps;
    a.dbg = g_debug_progress;
    a.sigma = (T *)sigma;
    a.info = info;
    a.zero_sigma = zero_sigma;
    // working-orientation factors: for wide blocks X = A^H, so X's U is A's V
    a.Uw = (cplx_t<T> *)(a.s.wide ? V : U);
    a.Vw = (cplx_t<T> *)(a.s.wide ? U : V);
    if (!a.s.smem_resident) {
        size_t need = 0;
        int stt = svd_workspace<T>(plan_count > 0 ? std::max(count, plan_count) : count, co, ci, wantv, &need);
        if (stt) return stt;
        if (ws_bytes < need || (!ws && need))
            return fail(CS_ENOMEM, "batched SVD: workspace too small (query cs_batched_svd_workspace)");
        a.scratch = (cplx_t<T> *)ws;
    }
    if constexpr (sizeof(T) == 4) {
        // warm-started solves only: cold starts (large rotations in every early
        // sweep) are faster on the scalar panel kernel
        if (tcb_enabled() && a.initX && tcb_supported(a.s.mr, a.s.nc, wantv))
            return tcb_dispatch(a, ws, ws_bytes, st);
    }
    return dispatch<T>(a, wantv, st, false, nullptr);
}

}  // namespace cs

using namespace cs;

static int check_svd_args(int dtype, long long count, int c_out, int c_in, int max_sweeps) {
    if (dtype != CS_F32 && dtype != CS_F64) return fail(CS_EINVAL, "batched SVD: unknown dtype");
    if (count < 0 || c_out < 1 || c_in < 1)
        return fail(CS_EINVAL, "batched SVD: block dimensions must be >= 1");
    if (max_sweeps < 1) return fail(CS_EINVAL, "batched SVD: max_sweeps must be >= 1");
    if (std::min(c_out, c_in) > 4096) return fail(CS_EINVAL, "batched SVD: blocks larger than 4096");
    return CS_OK;
}

extern "C" size_t cs_batched_svd_workspace(int dtype, long long count, int c_out, int c_in,
                                           int want_vectors) {
    size_t b = 0;
    if (check_svd_args(dtype, count, c_out, c_in, 1)) return 0;
    if (dtype == CS_F32) svd_workspace<float>(count, c_out, c_in, want_vectors != 0, &b);
    else svd_workspace<double>(count, c_out, c_in, want_vectors != 0, &b);
    return b;
}

extern "C" int cs_batched_svd(const void *blocks, int dtype, long long count, int c_out,
                              int c_in, int want_vectors, double tol, int max_sweeps,
                              void *sigma, void *U, void *V, int *info, int *zero_sigma,
                              void *workspace, size_t workspace_bytes, void *stream) {
    int st = check_svd_args(dtype, count, c_out, c_in, max_sweeps);
    if (st) return st;
    if (count && (!blocks || !sigma || !info)) return fail(CS_EINVAL, "batched SVD: null pointer");
    if (want_vectors && count && (!U || !V))
        return fail(CS_EINVAL, "batched SVD: U and V required with want_vectors");
    const bool wv = want_vectors != 0;
    if (dtype == CS_F32)
        return svd_run<float>(blocks, count, c_out, c_in, wv, tol, max_sweeps, sigma, U, V, info,
                              zero_sigma, workspace, workspace_bytes, (cudaStream_t)stream);
    return svd_run<double>(blocks, count, c_out, c_in, wv, tol, max_sweeps, sigma, U, V, info,
                           zero_sigma, workspace, workspace_bytes, (cudaStream_t)stream);
}

extern "C" int cs_batched_svd_plan_kind(int dtype, long long count, int c_out, int c_in,
                                        int want_vectors) {
    if (check_svd_args(dtype, count, c_out, c_in, 1)) return -1;
    JacShape s;
    const bool ok = dtype == CS_F32 ? plan<float>(c_out, c_in, want_vectors != 0, std::max(count, 1LL), s)
                                    : plan<double>(c_out, c_in, want_vectors != 0, std::max(count, 1LL), s);
    return ok ? s.kind : -1;
}

extern "C" int cs_batched_svd_indexed(const void *blocks, int dtype, long long count, int c_out,
                                      int c_in, int want_vectors, double tol, int max_sweeps,
                                      const long long *index, const void *init_X,
                                      const void *init_V, const long long *init_V_index,
                                      long long plan_count, void *sigma, void *U, void *V,
                                      int *info, int *zero_sigma,
                                      void *workspace, size_t workspace_bytes, void *stream) {
    int st = check_svd_args(dtype, count, c_out, c_in, max_sweeps);
    if (st) return st;
    if (count && (!sigma || !info || (!blocks && !init_X)))
        return fail(CS_EINVAL, "batched SVD: null pointer");
    if (want_vectors && count && (!U || !V))
        return fail(CS_EINVAL, "batched SVD: U and V required with want_vectors");
    const bool wv = want_vectors != 0;
    if (dtype == CS_F32)
        return svd_run<float>(blocks, count, c_out, c_in, wv, tol, max_sweeps, sigma, U, V, info,
                              zero_sigma, workspace, workspace_bytes, (cudaStream_t)stream, index,
                              init_X, init_V, init_V_index, plan_count);
    return svd_run<double>(blocks, count, c_out, c_in, wv, tol, max_sweeps, sigma, U, V, info,
                           zero_sigma, workspace, workspace_bytes, (cudaStream_t)stream, index,
                           init_X, init_V, init_V_index, plan_count);
}

extern "C" size_t cs_batched_svd_grouped_workspace(const cs_svd_group *groups, int num_groups,
                                                   int dtype, int want_vectors) {
    size_t total = 0;
    for (int g = 0; g < num_groups; ++g) {
        total += (cs_batched_svd_workspace(dtype, groups[g].count, groups[g].c_out,
                                           groups[g].c_in, want_vectors) + 255) & ~(size_t)255;
    }
    return total;
}

extern "C" int cs_batched_svd_grouped(const cs_svd_group *groups, int num_groups, int dtype,
                                      int want_vectors, double tol, int max_sweeps,
                                      void *workspace, size_t workspace_bytes, void *stream) {
    if (num_groups < 0 || (num_groups && !groups)) return fail(CS_EINVAL, "grouped SVD: bad group table");
    cudaStream_t st = (cudaStream_t)stream;
    if (num_groups == 1)
        return cs_batched_svd(groups[0].blocks, dtype, groups[0].count, groups[0].c_out,
                              groups[0].c_in, want_vectors, groups[0].tol > 0 ? groups[0].tol : tol,
                              max_sweeps, groups[0].sigma,
                              groups[0].U, groups[0].V, groups[0].info, groups[0].zero_sigma,
                              workspace, workspace_bytes, stream);
    // fork: every group on its own stream so small and large shapes share the SMs.
    // The side streams are created per call: a pool of long-lived streams
    // reused across calls measured slower on cfg4 (380 vs 340 ms per step,
    // same box, two runs each) -- plausibly long-lived streams sharing a
    // hardware work queue with the caller's stream.
    cudaEvent_t fork_ev;
    CS_CUDA_TRY(cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming));
    CS_CUDA_TRY(cudaEventRecord(fork_ev, st));
    int status = CS_OK;
    size_t off = 0;
    const int NS = 8;
    cudaStream_t sides[NS];
    cudaEvent_t done[NS];
    int nside = std::min(num_groups, NS);
    for (int i = 0; i < nside; ++i) {
        CS_CUDA_TRY(cudaStreamCreateWithFlags(&sides[i], cudaStreamNonBlocking));
        CS_CUDA_TRY(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
        CS_CUDA_TRY(cudaStreamWaitEvent(sides[i], fork_ev, 0));
    }
    for (int g = 0; g < num_groups && status == CS_OK; ++g) {
        const cs_svd_group &G = groups[g];
        const size_t need = cs_batched_svd_workspace(dtype, G.count, G.c_out, G.c_in, want_vectors);
        if (off + need > workspace_bytes && need) {
            status = fail(CS_ENOMEM, "grouped SVD: workspace too small");
            break;
        }
        status = cs_batched_svd(G.blocks, dtype, G.count, G.c_out, G.c_in, want_vectors,
                                G.tol > 0 ? G.tol : tol, max_sweeps, G.sigma, G.U, G.V, G.info, G.zero_sigma,
                                need ? (char *)workspace + off : nullptr, need, sides[g % nside]);
        off += (need + 255) & ~(size_t)255;
    }
    for (int i = 0; i < nside; ++i) {
        cudaEventRecord(done[i], sides[i]);
        cudaStreamWaitEvent(st, done[i], 0);
        cudaEventDestroy(done[i]);
        cudaStreamDestroy(sides[i]);
    }
    cudaEventDestroy(fork_ev);
    return status;
}
