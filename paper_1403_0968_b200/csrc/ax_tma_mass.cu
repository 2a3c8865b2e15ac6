// ax_tma_mass.cu -- the TMA Ax/K1 kernels (ax_tma.cuh) with the lumped
// screened-Coulomb mass term w += h u, h = alpha w_i w_j w_k J (NEXT-1,
// eq:semPDE / eq:semOperator).  A separate translation unit
// so the two variants compile in parallel.
#include "ax_tma.cuh"
#include "ax_dmma.cuh"

namespace sem {

cudaError_t upload_const_D_mass(int N, const double *D_host) { return upload_D_this_tu(N, D_host); }
cudaError_t tma_prepare_mass(int N) {
    cudaError_t e = tma_prepare_t<true>(N);
    if (e == cudaSuccess && N == 7) e = dmma_attr<false, true, false, false>();
    if (e == cudaSuccess && N == 7) e = dmma_attr<true, true, false, false>();
    return e;
}
cudaError_t hi_prepare_mass(int N) { return hi_prepare_t<true>(N); }

cudaError_t launch_ax_tma_mass(const DevMesh &m, const double *u, double *w, cudaStream_t s) {
    if (m.use_dmma) {
        TmaArgs a{};
        a.E = m.E;
        a.G = m.G;
        a.u = u;
        a.w = w;
        a.r = m.H;
        return launch_dmma_plain<true>(a, m.nsm, s);
    }
    return launch_ax_tma_t<true>(m, u, w, s);
}

cudaError_t launch_ax_hi_mass(const DevMesh &m, const double *u, double *w, cudaStream_t s) {
    return launch_ax_hi_t<true>(m, u, w, s);
}

cudaError_t launch_ax_cg_tma_mass(const DevMesh &m, const CgVecs &v, int64_t eb, int64_t ne,
                                  int pidx0, cudaStream_t s) {
    if (m.use_dmma) return launch_dmma_cg<true, false>(cg_args<true>(m, v, eb, ne, pidx0), m.nsm, s);
    return launch_ax_cg_tma_t<true>(m, v, eb, ne, pidx0, s);
}

cudaError_t launch_ax_cg_hi_mass(const DevMesh &m, const CgVecs &v, int64_t eb, int64_t ne,
                                 int pidx0, cudaStream_t s) {
    return launch_ax_cg_hi_t<true>(m, v, eb, ne, pidx0, s);
}

}  // namespace sem
