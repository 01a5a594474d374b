// cs_jacobi_f32.cu -- float instantiations of the batched Jacobi kernels (see cs_jacobi.cuh).
#include "cs_jacobi.cuh"
#include "cs_panel.cuh"

namespace cs {

// only the (rows-per-lane, vectors) combinations the planner can select:
// at most 64 registers of row data per thread
template <int C_, int RPL_>
static int fast_rpl(const JacArgs<float> &a, bool wantv, cudaStream_t st, bool dry, long long *ncl) {
    if constexpr (RPL_ <= 8)
        if (wantv) return launch_cluster_kernel<float, C_>(jacobi_fast_kernel<float, C_, RPL_, true>, a, st, dry, ncl);
    if constexpr (RPL_ <= 16)
        if (!wantv) return launch_cluster_kernel<float, C_>(jacobi_fast_kernel<float, C_, RPL_, false>, a, st, dry, ncl);
    return fail(CS_EINVAL, "batched SVD: rows per lane exceed the register budget");
}

template <int C_>
static int fast_c(const JacArgs<float> &a, bool wantv, cudaStream_t st, bool dry, long long *ncl) {
    switch (a.s.RPL) {
        case 2: return fast_rpl<C_, 2>(a, wantv, st, dry, ncl);
        case 4: return fast_rpl<C_, 4>(a, wantv, st, dry, ncl);
        case 8: return fast_rpl<C_, 8>(a, wantv, st, dry, ncl);
        case 16: return fast_rpl<C_, 16>(a, wantv, st, dry, ncl);
    }
    return fail(CS_EINVAL, "batched SVD: unsupported rows per lane");
}

template <int C_, int RPL_>
static int panel_rpl(const JacArgs<float> &a, bool wantv, cudaStream_t st, bool dry, long long *ncl) {
    // tall blocks: nc V rows need only half the lanes' X row count (planner)
    if constexpr (RPL_ >= 4 && RPL_ + RPL_ / 2 <= 16)
        if (wantv && !a.s.split && RPL_ / 2 >= 2 && (a.s.Rv + a.s.G - 1) / a.s.G <= RPL_ / 2)
            return launch_cluster_kernel<float, C_>(jacobi_panel_kernel<float, C_, RPL_, RPL_ / 2, false>, a, st, dry, ncl);
#ifdef CS_EXPERIMENTS
    if constexpr (2 * RPL_ <= 16 && true)
        if (wantv && a.s.split)
            return launch_cluster_kernel<float, C_>(jacobi_panel_kernel<float, C_, RPL_, RPL_, true>, a, st, dry, ncl);
#endif
    if constexpr (2 * RPL_ <= 16)
        if (wantv) return launch_cluster_kernel<float, C_>(jacobi_panel_kernel<float, C_, RPL_, RPL_, false>, a, st, dry, ncl);
    if constexpr (RPL_ <= 16)
        if (!wantv) return launch_cluster_kernel<float, C_>(jacobi_panel_kernel<float, C_, RPL_, 0, false>, a, st, dry, ncl);
    return fail(CS_EINVAL, "batched SVD: panel rows per lane exceed the register budget");
}

template <int C_>
static int panel_c(const JacArgs<float> &a, bool wantv, cudaStream_t st, bool dry, long long *ncl) {
    switch (a.s.RPL) {
        case 2: return panel_rpl<C_, 2>(a, wantv, st, dry, ncl);
        case 4: return panel_rpl<C_, 4>(a, wantv, st, dry, ncl);
        case 8: return panel_rpl<C_, 8>(a, wantv, st, dry, ncl);
        case 16: return panel_rpl<C_, 16>(a, wantv, st, dry, ncl);
    }
    return fail(CS_EINVAL, "batched SVD: unsupported panel rows per lane");
}

template <int C_>
static int generic_c(const JacArgs<float> &a, bool wantv, cudaStream_t st, bool dry, long long *ncl) {
    if (a.s.smem_resident) {
        if (wantv) return launch_cluster_kernel<float, C_>(jacobi_generic_kernel<float, C_, true, true>, a, st, dry, ncl);
        return launch_cluster_kernel<float, C_>(jacobi_generic_kernel<float, C_, false, true>, a, st, dry, ncl);
    }
    if (wantv) return launch_cluster_kernel<float, C_>(jacobi_generic_kernel<float, C_, true, false>, a, st, dry, ncl);
    return launch_cluster_kernel<float, C_>(jacobi_generic_kernel<float, C_, false, false>, a, st, dry, ncl);
}

int jacobi_dispatch_f32(const JacArgs<float> &a, bool wantv, cudaStream_t st, bool dry, long long *ncl) {
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

#ifdef CS_PHASE_CLOCKS
// experiment builds only: per-phase cycle totals of the f32 panel kernels
// [0] Gram G=P^H P, [1] rotations on G, [2] P += P D, [3] within rounds,
// [4] scalar cross phase (tools/gram_split.py)
extern "C" int cs_debug_phase_cycles(unsigned long long *out, int reset) {
    if (cudaDeviceSynchronize() != cudaSuccess) return 4;
    cudaMemcpyFromSymbol(out, cs::g_phase_cycles, sizeof(unsigned long long) * 8);
    if (reset) {
        unsigned long long z[8] = {};
        cudaMemcpyToSymbol(cs::g_phase_cycles, z, sizeof(z));
    }
    return 0;
}
#endif
