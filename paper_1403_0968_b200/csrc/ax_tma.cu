// ax_tma.cu -- Poisson instantiations of the TMA Ax/K1 kernels (ax_tma.cuh)
// and the exported launchers; operators with a mass term (DevMesh::H) are
// forwarded to ax_tma_mass.cu.
#include "ax_tma.cuh"
#include "ax_dmma.cuh"
#include "ax_dmmag.cuh"

namespace sem {

// ax_tma_mass.cu
cudaError_t upload_const_D_mass(int N, const double *D_host);
cudaError_t tma_prepare_mass(int N);
cudaError_t hi_prepare_mass(int N);
cudaError_t launch_ax_tma_mass(const DevMesh &m, const double *u, double *w, cudaStream_t s);
cudaError_t launch_ax_hi_mass(const DevMesh &m, const double *u, double *w, cudaStream_t s);
cudaError_t launch_ax_cg_tma_mass(const DevMesh &m, const CgVecs &v, int64_t eb, int64_t ne,
                                  int pidx0, cudaStream_t s);
cudaError_t launch_ax_cg_hi_mass(const DevMesh &m, const CgVecs &v, int64_t eb, int64_t ne,
                                 int pidx0, cudaStream_t s);
// ax_tma_pc.cu (Jacobi PCG K1, both operators)
cudaError_t upload_const_D_pc(int N, const double *D_host);
cudaError_t tma_prepare_pc(int N, bool mass);
cudaError_t hi_prepare_pc(int N, bool mass);
cudaError_t launch_ax_cg_tma_pc(const DevMesh &m, const CgVecs &v, int64_t eb, int64_t ne,
                                int pidx0, cudaStream_t s);
cudaError_t launch_ax_cg_hi_pc(const DevMesh &m, const CgVecs &v, int64_t eb, int64_t ne,
                               int pidx0, cudaStream_t s);

cudaError_t upload_const_D(int N, const double *D_host) {
    cudaError_t e = upload_D_this_tu(N, D_host);
    if (e == cudaSuccess) e = upload_const_D_mass(N, D_host);
    if (e == cudaSuccess) e = upload_const_D_pc(N, D_host);
    if (e == cudaSuccess) e = upload_const_D_rcg(N, D_host);
    return e == cudaSuccess ? upload_const_D_sr(N, D_host) : e;
}

bool tma_supported(int N) { return N >= 1 && N <= kTmaMaxN; }
bool dmma_supported(int N) { return N == 7; }
bool hi_supported(int N) { return N >= 6 && N <= 15; }
bool dmmag_supported(int N) { return N >= 8 && N <= 15; }

#define SEM_DG_DISPATCH(N_, ...)                                             \
    switch (N_) {                                                            \
    case 8: { constexpr int NN = 8; __VA_ARGS__; } break;                    \
    case 9: { constexpr int NN = 9; __VA_ARGS__; } break;                    \
    case 10: { constexpr int NN = 10; __VA_ARGS__; } break;                  \
    case 11: { constexpr int NN = 11; __VA_ARGS__; } break;                  \
    case 12: { constexpr int NN = 12; __VA_ARGS__; } break;                  \
    case 13: { constexpr int NN = 13; __VA_ARGS__; } break;                  \
    case 14: { constexpr int NN = 14; __VA_ARGS__; } break;                  \
    case 15: { constexpr int NN = 15; __VA_ARGS__; } break;                  \
    default: break;                                                          \
    }

int dmmag_blocks(int N, int64_t E, int nsm) {
    int nb = 0;
    SEM_DG_DISPATCH(N, nb = dmmag_grid<NN>(E, nsm));
    return nb;
}

// The split CG K1 at N >= 10 (use_k1ax): the x / p update with the scalar
// prologue (k1u_kernel), then the tensor-core operator on the new p with the
// (p, A p) partials (ax_dmmag_kernel DOT) -- 8 B per node more than a fused
// K1 (p is read twice) but the operator runs on the tensor cores instead of
// the register-bound CUDA-core high-order kernels.
cudaError_t launch_ax_cg_dmmag(const DevMesh &m, const CgVecs &v, int64_t eb, int64_t ne, int pidx0,
                               cudaStream_t s) {
    cudaError_t e = launch_k1u(m, v, eb, ne, s);
    if (e != cudaSuccess) return e;
    if (!m.use_dmmag) return launch_k1dot_range(m, v, eb, ne, pidx0, s);   // CUDA-core operator
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
        SEM_DG_DISPATCH(m.N, e = launch_pdl(ax_dmmag_kernel<NN, true, true>, dmmag_grid<NN>(ne, m.nsm),
                                            DgCfg<NN>::NT, DgCfg<NN>::SMEM, s, a));
    } else {
        SEM_DG_DISPATCH(m.N, e = launch_pdl(ax_dmmag_kernel<NN, false, true>, dmmag_grid<NN>(ne, m.nsm),
                                            DgCfg<NN>::NT, DgCfg<NN>::SMEM, s, a));
    }
    return e;
}

cudaError_t dmmag_prepare(int N) {
    cudaError_t e = cudaSuccess;
    SEM_DG_DISPATCH(N, (e = cudaFuncSetAttribute(ax_dmmag_kernel<NN, false, true>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)DgCfg<NN>::SMEM),
                        e = (e == cudaSuccess ? cudaFuncSetAttribute(ax_dmmag_kernel<NN, true, true>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)DgCfg<NN>::SMEM) : e)));
    if (e != cudaSuccess) return e;
    SEM_DG_DISPATCH(N, (e = cudaFuncSetAttribute(ax_dmmag_kernel<NN, false>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)DgCfg<NN>::SMEM),
                        e = (e == cudaSuccess ? cudaFuncSetAttribute(ax_dmmag_kernel<NN, true>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)DgCfg<NN>::SMEM) : e)));
    return e;
}

// plain Ax at N = 8..11 on the tensor cores (G^ in either layout)
cudaError_t launch_ax_dmmag(const DevMesh &m, const double *u, double *w, cudaStream_t s) {
    TmaArgs a{};
    a.E = m.E;
    a.G = m.G;
    a.u = u;
    a.w = w;
    if (m.use_hi) {
        SEM_DG_DISPATCH(m.N, (ax_dmmag_kernel<NN, true><<<dmmag_grid<NN>(m.E, m.nsm), DgCfg<NN>::NT,
                                                           DgCfg<NN>::SMEM, s>>>(a)));
    } else {
        SEM_DG_DISPATCH(m.N, (ax_dmmag_kernel<NN, false><<<dmmag_grid<NN>(m.E, m.nsm), DgCfg<NN>::NT,
                                                            DgCfg<NN>::SMEM, s>>>(a)));
    }
    return cudaGetLastError();
}

static cudaError_t dmma_prepare() {
    cudaError_t e = dmma_attr<false, false, false, false>();
    return e == cudaSuccess ? dmma_attr<true, false, false, false>() : e;
}

int dmma_blocks(int64_t E, int nsm, bool cg) {
    return cg ? dmma_grid<true>(E, nsm) : dmma_grid<false>(E, nsm);
}

int tma_blocks(int N, int64_t E, int nsm, bool cg) {
    int nb = 0;
    if (cg) {
        SEM_TMA_DISPATCH(N, nb = tma_grid<NN, true>(E, nsm));
    } else {
        SEM_TMA_DISPATCH(N, nb = tma_grid<NN, false>(E, nsm));
    }
    return nb;
}

int hi_blocks(int N, int64_t E, int nsm, bool cg) {
    int nb = 0;
    if (cg) {
        SEM_HI_DISPATCH(N, nb = hi_grid<NN, true>(E, nsm));
    } else {
        SEM_HI_DISPATCH(N, nb = hi_grid<NN, false>(E, nsm));
    }
    return nb;
}

cudaError_t tma_prepare(int N, bool mass) {
    cudaError_t e = mass ? tma_prepare_mass(N) : tma_prepare_t<false>(N);
    if (e == cudaSuccess && dmma_supported(N)) e = dmma_prepare();
    return e == cudaSuccess ? tma_prepare_pc(N, mass) : e;
}

cudaError_t hi_prepare(int N, bool mass) {
    cudaError_t e = mass ? hi_prepare_mass(N) : hi_prepare_t<false>(N);
    return e == cudaSuccess ? hi_prepare_pc(N, mass) : e;
}

cudaError_t launch_ax_tma(const DevMesh &m, const double *u, double *w, cudaStream_t s) {
    if (m.use_dmma && !m.H) {
        TmaArgs a{};
        a.E = m.E;
        a.G = m.G;
        a.u = u;
        a.w = w;
        return launch_dmma_plain<false>(a, m.nsm, s);
    }
    return m.H ? launch_ax_tma_mass(m, u, w, s) : launch_ax_tma_t<false>(m, u, w, s);
}

cudaError_t launch_ax_hi(const DevMesh &m, const double *u, double *w, cudaStream_t s) {
    return m.H ? launch_ax_hi_mass(m, u, w, s) : launch_ax_hi_t<false>(m, u, w, s);
}

cudaError_t launch_ax_cg_tma(const DevMesh &m, const CgVecs &v, int64_t eb, int64_t ne, int pidx0,
                             cudaStream_t s) {
    if (v.dinv) return launch_ax_cg_tma_pc(m, v, eb, ne, pidx0, s);
    if (m.use_dmma && !m.H) {
        return launch_dmma_cg<false, false>(cg_args<false>(m, v, eb, ne, pidx0), m.nsm, s);
    }
    return m.H ? launch_ax_cg_tma_mass(m, v, eb, ne, pidx0, s)
               : launch_ax_cg_tma_t<false>(m, v, eb, ne, pidx0, s);
}

cudaError_t launch_ax_cg_hi(const DevMesh &m, const CgVecs &v, int64_t eb, int64_t ne, int pidx0,
                            cudaStream_t s) {
    if (v.dinv) return launch_ax_cg_hi_pc(m, v, eb, ne, pidx0, s);
    return m.H ? launch_ax_cg_hi_mass(m, v, eb, ne, pidx0, s)
               : launch_ax_cg_hi_t<false>(m, v, eb, ne, pidx0, s);
}

}  // namespace sem
