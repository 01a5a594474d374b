// cs_jacobi_f64.cu -- double instantiations of the batched Jacobi kernels (see cs_jacobi.cuh).
#include "cs_jacobi.cuh"
#include "cs_panel.cuh"

namespace cs {

// only the (rows-per-lane, vectors) combinations the planner can select:
// at most 64 registers of row data per thread
template <int C_, int RPL_>
static int fast_rpl(const JacArgs<double> &a, bool wantv, cudaStream_t st, bool dry, long long *ncl) {
    if constexpr (RPL_ <= 4)
        if (wantv) return launch_cluster_kernel<double, C_>(jacobi_fast_kernel<double, C_, RPL_, true>, a, st, dry, ncl);
    if constexpr (RPL_ <= 8)
        if (!wantv) return launch_cluster_kernel<double, C_>(jacobi_fast_kernel<double, C_, RPL_, false>, a, st, dry, ncl);
    return fail(CS_EINVAL, "batched SVD: rows per lane exceed the register budget");
}

template <int C_>
static int fast_c(const JacArgs<double> &a, bool wantv, cudaStream_t st, bool dry, long long *ncl) {
    switch (a.s.RPL) {
        case 2: return fast_rpl<C_, 2>(a, wantv, st, dry, ncl);
        case 4: return fast_rpl<C_, 4>(a, wantv, st, dry, ncl);
        case 8: return fast_rpl<C_, 8>(a, wantv, st, dry, ncl);
        case 16: return fast_rpl<C_, 16>(a, wantv, st, dry, ncl);
    }
    return fail(CS_EINVAL, "batched SVD: unsupported rows per lane");
}

template <int C_, int RPL_>
static int panel_rpl(const JacArgs<double> &a, bool wantv, cudaStream_t st, bool dry, long long *ncl) {
    // 256-thread fp64 panels with 8 X + 8 V rows per lane (cfg5 in fp64: C = 16)
    if constexpr (C_ == 16 && RPL_ == 8)
        if (wantv && !a.s.split)
            return launch_cluster_kernel<double, C_>(jacobi_panel_kernel<double, C_, 8, 8, false>, a, st, dry, ncl);
    if constexpr (2 * RPL_ <= 8 && false)
        if (wantv && a.s.split)
            return launch_cluster_kernel<double, C_>(jacobi_panel_kernel<double, C_, RPL_, RPL_, true>, a, st, dry, ncl);
    if constexpr (2 * RPL_ <= 8)
        if (wantv) return launch_cluster_kernel<double, C_>(jacobi_panel_kernel<double, C_, RPL_, RPL_, false>, a, st, dry, ncl);
    if constexpr (RPL_ <= 8)
        if (!wantv) return launch_cluster_kernel<double, C_>(jacobi_panel_kernel<double, C_, RPL_, 0, false>, a, st, dry, ncl);
    return fail(CS_EINVAL, "batched SVD: panel rows per lane exceed the register budget");
}

template <int C_>
static int panel_c(const JacArgs<double> &a, bool wantv, cudaStream_t st, bool dry, long long *ncl) {
    switch (a.s.RPL) {
        case 2: return panel_rpl<C_, 2>(a, wantv, st, dry, ncl);
        case 4: return panel_rpl<C_, 4>(a, wantv, st, dry, ncl);
        case 8: return panel_rpl<C_, 8>(a, wantv, st, dry, ncl);
        case 16: return panel_rpl<C_, 16>(a, wantv, st, dry, ncl);
    }
    return fail(CS_EINVAL, "batched SVD: unsupported panel rows per lane");
}

template <int C_>
static int generic_c(const JacArgs<double> &a, bool wantv, cudaStream_t st, bool dry, long long *ncl) {
    if (a.s.smem_resident) {
        if (wantv) return launch_cluster_kernel<double, C_>(jacobi_generic_kernel<double, C_, true, true>, a, st, dry, ncl);
        return launch_cluster_kernel<double, C_>(jacobi_generic_kernel<double, C_, false, true>, a, st, dry, ncl);
    }
    if (wantv) return launch_cluster_kernel<double, C_>(jacobi_generic_kernel<double, C_, true, false>, a, st, dry, ncl);
    return launch_cluster_kernel<double, C_>(jacobi_generic_kernel<double, C_, false, false>, a, st, dry, ncl);
}

int jacobi_dispatch_f64(const JacArgs<double> &a, bool wantv, cudaStream_t st, bool dry, long long *ncl) {
    if (a.s.kind == 2) {
        switch (a.s.C) {
            case 1: return panel_c<1>(a, wantv, st, dry, ncl);
            case 2: return panel_c<2>(a, wantv, st, dry, ncl);
            case 4: return panel_c<4>(a, wantv, st, dry, ncl);
            case 8: return panel_c<8>(a, wantv, st, dry, ncl);
            case 16: return panel_c<16>(a, wantv, st, dry, ncl);
        }
    } else if (a.s.kind == 0) {
        switch (a.s.C) {
            case 1: return fast_c<1>(a, wantv, st, dry, ncl);
            case 2: return fast_c<2>(a, wantv, st, dry, ncl);
            case 4: return fast_c<4>(a, wantv, st, dry, ncl);
            case 8: return fast_c<8>(a, wantv, st, dry, ncl);
            case 16: return fast_c<16>(a, wantv, st, dry, ncl);
        }
    } else {
        switch (a.s.C) {
            case 1: return generic_c<1>(a, wantv, st, dry, ncl);
            case 8: return generic_c<8>(a, wantv, st, dry, ncl);
            case 16: return generic_c<16>(a, wantv, st, dry, ncl);
        }
    }
    return fail(CS_EINVAL, "batched SVD: unsupported cluster size");
}

}  // namespace cs
