// ax_tma_pc.cu -- K1 of the Jacobi-preconditioned CG (NEXT-2, PCG of
// PAPER.md:672-673): the TMA / high-order K1 kernels (ax_tma.cuh) with the
// PCG scalar prologue (rho = (r,z) for alpha / beta, (r,r) for the stop) and
// z as the vector p is formed from; Poisson and screened operators.  Its own
// translation unit (and its own __constant__ copy of D) so the CG kernels keep
// their code and the variants compile in parallel.
#include "ax_tma.cuh"
#include "ax_dmma.cuh"

namespace sem {

cudaError_t upload_const_D_pc(int N, const double *D_host) { return upload_D_this_tu(N, D_host); }

// Jacobi PCG: does K1 form z = dinv r itself (so K2 need not store z)?  The
// N = 7 tensor-core K1 without a mass term does (ax_dmma.cuh PCZ).
bool pcg_z_in_k1(const DevMesh &m) { return m.use_dmma && !m.H; }

cudaError_t tma_prepare_pc(int N, bool mass) {
    cudaError_t e = mass ? tma_prepare_t<true, true>(N) : tma_prepare_t<false, true>(N);
    if (e == cudaSuccess && N == 7)
        e = mass ? dmma_attr<true, true, true, false>() : dmma_attr<true, false, true, false>();
    return e;
}

cudaError_t hi_prepare_pc(int N, bool mass) {
    if (N < 6) return cudaSuccess;
    return mass ? hi_prepare_t<true, true>(N) : hi_prepare_t<false, true>(N);
}

cudaError_t launch_ax_cg_tma_pc(const DevMesh &m, const CgVecs &v, int64_t eb, int64_t ne,
                                int pidx0, cudaStream_t s) {
    if (m.use_dmma) {
        if (m.H) return launch_dmma_cg<true, true>(cg_args<true>(m, v, eb, ne, pidx0), m.nsm, s);
        // Poisson PCG at N = 7: K1 forms z = dinv r from r and dinv itself
        // (pcg_z_in_k1), K2 does not store z
        TmaArgs a = cg_args<false>(m, v, eb, ne, pidx0);
        a.r = v.r + eb * m.n3;
        a.u = v.dinv + eb * m.n3;
        return launch_dmma_cg<false, true>(a, m.nsm, s);
    }
    return m.H ? launch_ax_cg_tma_t<true, true>(m, v, eb, ne, pidx0, s)
               : launch_ax_cg_tma_t<false, true>(m, v, eb, ne, pidx0, s);
}

cudaError_t launch_ax_cg_hi_pc(const DevMesh &m, const CgVecs &v, int64_t eb, int64_t ne,
                               int pidx0, cudaStream_t s) {
    return m.H ? launch_ax_cg_hi_t<true, true>(m, v, eb, ne, pidx0, s)
               : launch_ax_cg_hi_t<false, true>(m, v, eb, ne, pidx0, s);
}

}  // namespace sem
