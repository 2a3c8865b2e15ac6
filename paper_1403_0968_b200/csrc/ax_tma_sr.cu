// ax_tma_sr.cu -- KA of the single-reduction (Chronopoulos-Gear) CG (NEXT-3,
// DESIGN.md reading R7): the TMA / high-order plain Ax kernels (ax_tma.cuh)
// with the DOT flag, w = A_L r plus per-CTA partials of (r, w).  Poisson
// operator.  Its own translation unit and __constant__ copy of D.
#include "ax_tma.cuh"
#include "ax_dmma.cuh"

namespace sem {

cudaError_t upload_const_D_sr(int N, const double *D_host) { return upload_D_this_tu(N, D_host); }

cudaError_t sr_prepare(const DevMesh &m) {
    if (m.use_dmma) return dmma_attr<false, false, false, true>();
    if (m.use_hi) return hi_prepare_dot(m.N);
    if (m.use_tma) return tma_prepare_dot(m.N);
    return cudaErrorInvalidValue;
}

// grid of KA = the number of its (r, w) partials (KB and the fold read exactly
// these; the CG kernel K1 has its own, larger or equal, grid)
int ka_blocks(const DevMesh &m) {
    int nb = 0;
    if (m.use_dmma) {
        nb = dmma_grid<false>(m.E, m.nsm);
    } else if (m.use_hi) {
        SEM_HI_DISPATCH(m.N, nb = hi_grid<NN, false>(m.E, m.nsm));
    } else if (m.use_tma) {
        SEM_TMA_DISPATCH(m.N, nb = tma_grid<NN, false>(m.E, m.nsm));
    }
    return nb;
}

// The operator half of the split CG K1 on the CUDA-core TMA / high-order
// kernels (use_k1ax without the tensor-core Ax): w = A_L p over the element
// range [eb, eb + ne) plus per-CTA (p, A p) partials into part1[pidx0 ..]
// at the iteration parity, a no-op after the stop (the DOT flag).
int k1dot_blocks(const DevMesh &m, int64_t ne) {
    int nb = 0;
    if (m.use_hi) {
        SEM_HI_DISPATCH(m.N, nb = hi_grid<NN, false>(ne, m.nsm));
    } else if (m.use_tma) {
        SEM_TMA_DISPATCH(m.N, nb = tma_grid<NN, false>(ne, m.nsm));
    }
    return nb;
}

cudaError_t launch_k1dot_range(const DevMesh &m, const CgVecs &v, int64_t eb, int64_t ne, int pidx0,
                               cudaStream_t s) {
    const int64_t o = eb * m.n3;
    TmaArgs a{};
    a.E = ne;
    a.G = m.G + 6 * o;
    a.u = v.p + o;
    a.w = v.w + o;
    a.red = make_red(m, v);
    a.part1 = v.part1 + pidx0;
    a.st = v.st;
    if (m.use_hi) {
        SEM_HI_DISPATCH(m.N, (ax_hi_kernel<NN, false, false, false, true>
                              <<<hi_grid<NN, false>(ne, m.nsm), HiCfg<NN, false>::NT,
                                 HiCfg<NN, false>::SMEM, s>>>(a)));
    } else if (m.use_tma) {
        SEM_TMA_DISPATCH(m.N, (ax_tma_kernel<NN, false, false, false, true>
                               <<<tma_grid<NN, false>(ne, m.nsm), TmaLayout<NN, false>::NT,
                                  TmaLayout<NN, false>::SMEM, s>>>(a)));
    } else {
        return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_ax_dot(const DevMesh &m, const CgVecs &v, cudaStream_t s) {
    if (m.use_dmma) return launch_dmma_plain<false, true>(sr_args(m, v), m.nsm, s);
    if (m.use_hi) return launch_ax_dot_hi_t(m, v, s);
    if (m.use_tma) return launch_ax_dot_tma_t(m, v, s);
    return cudaErrorInvalidValue;
}

}  // namespace sem
