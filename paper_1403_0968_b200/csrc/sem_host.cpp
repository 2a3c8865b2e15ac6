// sem_host.cpp -- host orchestration behind the C ABI of include/sem.h.
//
// a0  GLL nodes/weights and the differentiation matrix (own implementation:
//     simultaneous Newton on all N+1 nodes with a Legendre Vandermonde, and the
//     barycentric form of D; it shares nothing with oracle/).
// a2  gather-scatter plan from the global-local numbering.
// a9  CG driver: device-resident scalars, no per-iteration host sync, exact
//     iteration count via a sticky device flag polled once per chunk.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>
#include <thread>
#include <chrono>

#include "../../include/sem.h"
#include "sem_internal.h"
#include "sem_comm.h"

using namespace sem;

// kernel classes for sem_profile_read (documented in include/sem.h)
enum { kProfAx = 0, kProfAxCg = 1, kProfK2 = 2, kProfGs = 3, kProfOther = 4, kProfRcg = 5, kProfClasses = 6 };

struct sem_ctx {
    int N = 0, n = 0, n3 = 0;
    int64_t E = 0, L = 0, nglobal = 0;
    int rank = 0, nranks = 1, device = 0;
    cudaStream_t stream = nullptr;
    DevMesh dm{};
    CgVecs cv{};
    int nb_ax = 0;
    CgState *host_state = nullptr;   // pinned, 2 slots for double-buffered polling
    cudaEvent_t ev[2] = {nullptr, nullptr};
    // chunk polling off the critical path: the state copy runs on its own
    // stream after an event, so the next chunk's graph does not queue behind it
    cudaStream_t poll_stream = nullptr;
    cudaEvent_t chunk_ev[2] = {nullptr, nullptr};
    int64_t launches = 0;
    bool broken = false;
    // optional per-kernel-class device timing (bench roofline), see sem_profile
    bool prof = false;
    struct Rec { cudaEvent_t a, b; int cls; int k; double bytes; };
    std::vector<Rec> recs;               // pending (not yet folded)
    std::vector<cudaEvent_t> evpool;
    double prof_ms[kProfClasses] = {0};
    double prof_bytes[kProfClasses] = {0};
    int64_t prof_n[kProfClasses] = {0};
    std::string err;
    Comm *comm = nullptr;            // nranks > 1 only
    // CUDA graph of kChunk CG iterations (captured on first use)
    bool use_graph = true;
    cudaStream_t cap_stream = nullptr;
    cudaGraphExec_t graph_exec[3] = {nullptr, nullptr, nullptr};   // CG, Jacobi PCG, single-reduction CG
    int64_t graph_kernels[3] = {0, 0, 0};
    int method = 0;                  // solver being run / captured: 0 CG, 1 Jacobi PCG, 2 single-reduction
    cudaGraphExec_t replay_exec = nullptr;   // sem_kernel_replay
    // boundary/interior K1 split (k1_split): the exchange runs on `side`
    // between fork (boundary K1 done) and join (before the pap all-gather)
    cudaStream_t side = nullptr;
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    // Jacobi preconditioner (NEXT-2): mask / Q Q^T diag(A_L), formed on first use
    double *dinv_buf = nullptr;
    bool dinv_ready = false;
    // L2 persistence of the CG work vectors r, p, w, xw (contiguous in the
    // workspace): access-policy window attached to the CG graph's kernel nodes
    bool l2_on = false;
    cudaAccessPolicyWindow l2win{};
    // resident CG (cg_resident.cu): eligible mesh / device, and its buffers
    bool rcg_ok = false;
    bool rcg_last = false;           // the last sem_cg ran resident (sem_cg_phases)
    int rcg_iters = 0;
    RcgBufs rcg{};
};

static constexpr int kChunk = 8;     // CG iterations per graph launch / poll (multiple of 4)

static thread_local std::string g_err;

static int fail(sem_ctx *c, int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    g_err = buf;
    return code;
}

struct sem_ctx;
static cudaEvent_t prof_event(sem_ctx *ctx);
static int build_cg_graph(sem_ctx *ctx);
static void prof_fold(sem_ctx *ctx, int iters);

#define CU(call)                                                                     \
    do {                                                                             \
        cudaError_t e_ = (call);                                                     \
        if (e_ != cudaSuccess) {                                                     \
            if (ctx) ctx->broken = true;                                             \
            return fail(ctx, SEM_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                         \
        }                                                                            \
    } while (0)

#define LAUNCH(call) LAUNCHP(kProfOther, 0.0, -1, call)

// Launch with optional device timing: class `cls`, algorithmic bytes `by`,
// CG iteration `kk` (-1 outside CG; CG launches at k >= iters are no-ops and
// are dropped when the solve is folded).
#define LAUNCHP(cls, by, kk, call)                                                   \
    do {                                                                             \
        ctx->launches++;                                                             \
        cudaEvent_t a_ = nullptr, b_ = nullptr;                                      \
        if (ctx->prof) {                                                             \
            a_ = prof_event(ctx);                                                    \
            b_ = prof_event(ctx);                                                    \
            CU(cudaEventRecord(a_, ctx->stream));                                    \
        }                                                                            \
        CU(call);                                                                    \
        if (ctx->prof) {                                                             \
            CU(cudaEventRecord(b_, ctx->stream));                                    \
            ctx->recs.push_back({a_, b_, (cls), (kk), (by)});                        \
        }                                                                            \
    } while (0)

static cudaEvent_t prof_event(sem_ctx *ctx) {
    cudaEvent_t e = nullptr;
    if (!ctx->evpool.empty()) {
        e = ctx->evpool.back();
        ctx->evpool.pop_back();
    } else if (cudaEventCreate(&e) != cudaSuccess) {
        e = nullptr;
    }
    return e;
}

// Fold completed records into the accumulators (stream must be synchronised).
// iters >= 0: records of a CG solve; launches with k >= iters were no-ops.
static void prof_fold(sem_ctx *ctx, int iters) {
    for (auto &r : ctx->recs) {
        float ms = 0.f;
        bool keep = (r.k < 0) || (iters >= 0 && r.k < iters);
        if (keep && cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
            ctx->prof_ms[r.cls] += ms;
            ctx->prof_bytes[r.cls] += r.bytes;
            ctx->prof_n[r.cls] += 1;
        }
        ctx->evpool.push_back(r.a);
        ctx->evpool.push_back(r.b);
    }
    ctx->recs.clear();
}

// ---------------------------------------------------------------------------
// a0: GLL nodes/weights and D
// ---------------------------------------------------------------------------
extern "C" int sem_gll(int N, double *xi, double *w) {
    if (N < 1 || N > 64 || !xi || !w) return fail(nullptr, SEM_EINVAL, "sem_gll: bad arguments");
    const int n = N + 1;
    std::vector<double> x(n), xold(n), P(n * (N + 1));
    // initial guess: Chebyshev-Gauss-Lobatto points, ascending
    for (int i = 0; i < n; ++i) x[i] = -std::cos(M_PI * i / N);
    // Newton on (1 - x^2) P'_N(x) for all nodes at once, using
    // (1 - x^2) P'_N = N (P_{N-1} - x P_N) and d/dx of that = -N (N+1) P_N:
    //   x <- x - (x P_N - P_{N-1}) / ((N+1) P_N)
    for (int it = 0; it < 200; ++it) {
        for (int i = 0; i < n; ++i) {
            double p0 = 1.0, p1 = x[i];
            for (int k = 2; k <= N; ++k) {
                double p2 = ((2 * k - 1) * x[i] * p1 - (k - 1) * p0) / k;
                p0 = p1;
                p1 = p2;
            }
            // p1 = P_N, p0 = P_{N-1}  (for N == 1: p1 = x, p0 = 1)
            P[i] = p1;
            xold[i] = x[i];
            x[i] = xold[i] - (xold[i] * p1 - p0) / ((N + 1) * p1);
        }
        double d = 0.0;
        for (int i = 0; i < n; ++i) d = std::max(d, std::fabs(x[i] - xold[i]));
        if (d < 4e-16) break;
    }
    // exact endpoints and mirror symmetry
    x[0] = -1.0;
    x[N] = 1.0;
    for (int i = 1; i < n / 2; ++i) {
        double a = 0.5 * (x[N - i] - x[i]);
        x[i] = -a;
        x[N - i] = a;
    }
    if (N % 2 == 0) x[N / 2] = 0.0;
    for (int i = 0; i < n; ++i) {
        double p0 = 1.0, p1 = x[i];
        for (int k = 2; k <= N; ++k) {
            double p2 = ((2 * k - 1) * x[i] * p1 - (k - 1) * p0) / k;
            p0 = p1;
            p1 = p2;
        }
        xi[i] = x[i];
        w[i] = 2.0 / (N * (N + 1.0) * p1 * p1);
    }
    return SEM_OK;
}

// Barycentric differentiation matrix: D_ij = (lam_j / lam_i) / (x_i - x_j),
// lam_j = 1 / prod_{k != j} (x_j - x_k); D_ii = -sum_{j != i} D_ij.
static void diff_matrix(int N, const double *x, double *D) {
    const int n = N + 1;
    std::vector<double> lam(n);
    for (int j = 0; j < n; ++j) {
        double p = 1.0;
        for (int k = 0; k < n; ++k)
            if (k != j) p *= (x[j] - x[k]);
        lam[j] = 1.0 / p;
    }
    for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int j = 0; j < n; ++j) {
            if (j == i) continue;
            double v = (lam[j] / lam[i]) / (x[i] - x[j]);
            D[i * n + j] = v;
            s += v;
        }
        D[i * n + i] = -s;
    }
}

// ---------------------------------------------------------------------------
// workspace layout
// ---------------------------------------------------------------------------
namespace {
struct Layout {
    size_t G, BM, H, r, p, w, xw, z, dinv, D, gs_idx, own, partials, rr_all, pap_all, st, total;
    size_t rcg_meta, rcg_sbq, rcg_push, rcg_X, rcg_part, rcg_bar;   // resident CG (N = 7, one rank, Poisson)
    int64_t nsurf_cap, partial_cap;
};

size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

Layout make_layout(int N, int64_t E, int nranks, bool mass) {
    Layout Lo{};
    const int64_t n = N + 1, n3 = n * n * n, L = E * n3;
    const int64_t ni = (n >= 2) ? (n - 2) : 0;
    Lo.nsurf_cap = E * (n3 - ni * ni * ni);
    // per-block partials of K1 / K2: both grids are <= 4 CTAs per SM
    Lo.partial_cap = kMaxPartials;
    size_t o = 0;
    auto take = [&](size_t bytes) {
        size_t at = o;
        o = align256(o + bytes);
        return at;
    };
    Lo.G = take(sizeof(double) * 6 * L);
    Lo.BM = take(sizeof(double) * L);
    Lo.H = mass ? take(sizeof(double) * L) : 0;
    Lo.r = take(sizeof(double) * L);
    Lo.p = take(sizeof(double) * L);
    Lo.w = take(sizeof(double) * L);
    Lo.xw = take(sizeof(double) * L);
    Lo.z = take(sizeof(double) * L);
    Lo.dinv = take(sizeof(double) * L);
    Lo.D = take(sizeof(double) * (n * n + n));
    Lo.gs_idx = take(sizeof(int32_t) * Lo.nsurf_cap);
    Lo.own = take(sizeof(uint32_t) * ((Lo.nsurf_cap + 31) / 32 + 1));
    Lo.partials = take(sizeof(double) * 6 * Lo.partial_cap);   // part1, part2, part3: [2][cap]
    Lo.rr_all = take(sizeof(double) * 2 * kRing * nranks);     // rr_all, then rz_all
    Lo.pap_all = take(sizeof(double) * kRing * nranks);
    Lo.st = take(sizeof(CgState));
    // the resident CG's tables (opt-in, SEM_CG_RESIDENT=1 when the workspace
    // is sized and the context set up: ~12 KB per element)
    const char *rcg_env = getenv("SEM_CG_RESIDENT");
    if (N == 7 && nranks == 1 && !mass && rcg_env && rcg_env[0] == '1') {
        // push-based DSSUM: meta per local node, slot bases per node position,
        // push destinations and receive slots (<= kRcgMaxSlots per element)
        Lo.rcg_meta = take(sizeof(uint8_t) * L);
        Lo.rcg_sbq = take(sizeof(int32_t) * n3);
        Lo.rcg_push = take(sizeof(int32_t) * E * kRcgMaxSlots);
        Lo.rcg_X = take(sizeof(double) * E * kRcgMaxSlots);
        Lo.rcg_part = take(sizeof(double) * 2 * Lo.partial_cap);
        Lo.rcg_bar = take(sizeof(uint32_t) * 64);
    }
    Lo.total = o;
    return Lo;
}
}  // namespace

static int check_mesh(const sem_mesh *m, int N) {
    if (!m) return fail(nullptr, SEM_EINVAL, "mesh is NULL");
    if (N < 1 || N > SEM_NMAX) return fail(nullptr, SEM_EINVAL, "N=%d outside [1,%d]", N, SEM_NMAX);
    if (m->nelem <= 0) return fail(nullptr, SEM_EINVAL, "nelem=%d must be > 0", m->nelem);
    if (m->nranks < 1 || m->nranks > kMaxRanks || m->rank < 0 || m->rank >= m->nranks)
        return fail(nullptr, SEM_EINVAL, "bad rank %d / nranks %d", m->rank, m->nranks);
    const int64_t n3 = int64_t(N + 1) * (N + 1) * (N + 1);
    if (int64_t(m->nelem) * n3 >= (int64_t(1) << 31))
        return fail(nullptr, SEM_EINVAL, "nlocal >= 2^31 not supported");
    return SEM_OK;
}

extern "C" int sem_workspace_bytes(const sem_mesh *m, int N, size_t *bytes) {
    int rc = check_mesh(m, N);
    if (rc) return rc;
    if (!bytes) return fail(nullptr, SEM_EINVAL, "bytes is NULL");
    *bytes = make_layout(N, m->nelem, m->nranks, m->alpha != nullptr).total;
    return SEM_OK;
}

// ---------------------------------------------------------------------------
// a2: gather-scatter plan (host)
// ---------------------------------------------------------------------------
namespace {
struct HostPlan {
    std::vector<int32_t> off, idx;      // CSR: copies of group q = idx[off[q]..off[q+1])
    std::vector<int32_t> cidx;          // the same copies, class-transposed (device layout)
    GsClasses cls{};
    int32_t ngroups = 0, ndir = 0;
    int64_t ndistinct = 0;
    // for multi-rank: distinct surface global ids (ascending) and their group
    std::vector<int64_t> surf_ids;
    std::vector<int32_t> surf_group;
};

// order[] = local indices sorted by (glo, local index) -- counting sort when the
// id range is compact, std::sort otherwise.
std::vector<int32_t> sort_by_glo(const int64_t *glo, int64_t L, int64_t gmin, int64_t gmax) {
    std::vector<int32_t> order(L);
    const int64_t range = gmax - gmin + 1;
    if (range <= 4 * L + 1024) {
        std::vector<int32_t> cnt(range + 1, 0);
        for (int64_t l = 0; l < L; ++l) cnt[glo[l] - gmin + 1]++;
        for (int64_t g = 0; g < range; ++g) cnt[g + 1] += cnt[g];
        for (int64_t l = 0; l < L; ++l) order[cnt[glo[l] - gmin]++] = (int32_t)l;
    } else {
        for (int64_t l = 0; l < L; ++l) order[l] = (int32_t)l;
        std::stable_sort(order.begin(), order.end(),
                         [&](int32_t a, int32_t b) { return glo[a] < glo[b]; });
    }
    return order;
}

int build_plan(const sem_mesh *m, int N, HostPlan &hp, std::string &err) {
    const int n = N + 1, n3 = n * n * n;
    const int64_t L = int64_t(m->nelem) * n3;
    const int64_t *glo = m->glo;
    const uint8_t *dir = m->dirichlet;
    int64_t gmin = glo[0], gmax = glo[0];
    for (int64_t l = 0; l < L; ++l) {
        if (glo[l] < 0) { err = "negative global id"; return SEM_EINVAL; }
        gmin = std::min(gmin, glo[l]);
        gmax = std::max(gmax, glo[l]);
    }
    std::vector<uint8_t> surf(n3);
    for (int q = 0; q < n3; ++q) {
        int i = q % n, j = (q / n) % n, k = q / (n * n);
        surf[q] = (i == 0 || i == N || j == 0 || j == N || k == 0 || k == N);
    }
    std::vector<int32_t> order = sort_by_glo(glo, L, gmin, gmax);
    struct G { int32_t a, b; uint8_t d; int32_t first; };
    std::vector<G> groups;
    int64_t a = 0;
    hp.ndistinct = 0;
    while (a < L) {
        int64_t b = a + 1;
        const int64_t g = glo[order[a]];
        while (b < L && glo[order[b]] == g) ++b;
        hp.ndistinct++;
        const uint8_t d0 = dir[order[a]] ? 1 : 0;
        bool any_interior = false;
        for (int64_t t = a; t < b; ++t) {
            if ((dir[order[t]] ? 1 : 0) != d0) {
                err = "inconsistent Dirichlet flags across copies of global id " + std::to_string(g);
                return SEM_EINVAL;
            }
            if (!surf[order[t] % n3]) any_interior = true;
        }
        if (any_interior) {
            if (b - a > 1) {
                err = "element-interior node shared (global id " + std::to_string(g) + ")";
                return SEM_EINVAL;
            }
            if (d0) {
                err = "element-interior node marked Dirichlet (global id " + std::to_string(g) + ")";
                return SEM_EINVAL;
            }
        } else {
            groups.push_back({(int32_t)a, (int32_t)b, d0, order[a]});
        }
        a = b;
    }
    // Dirichlet groups first, then by multiplicity, then by first local index
    std::stable_sort(groups.begin(), groups.end(), [](const G &x, const G &y) {
        if (x.d != y.d) return x.d > y.d;
        const int mx = x.b - x.a, my = y.b - y.a;
        if (mx != my) return mx < my;
        return x.first < y.first;
    });
    hp.ngroups = (int32_t)groups.size();
    hp.off.resize(groups.size() + 1);
    hp.idx.clear();
    hp.ndir = 0;
    hp.off[0] = 0;
    for (size_t q = 0; q < groups.size(); ++q) {
        for (int32_t t = groups[q].a; t < groups[q].b; ++t) hp.idx.push_back(order[t]);
        hp.off[q + 1] = (int32_t)hp.idx.size();
        if (groups[q].d) hp.ndir++;
    }
    // class layout: runs of equal (dirichlet, multiplicity)
    hp.cidx.assign(hp.idx.size(), 0);
    hp.cls.n = 0;
    {
        size_t q = 0;
        int32_t ioff = 0;
        while (q < groups.size()) {
            const int m = groups[q].b - groups[q].a;
            const uint8_t d = groups[q].d;
            size_t r = q;
            while (r < groups.size() && groups[r].d == d && groups[r].b - groups[r].a == m) ++r;
            if (hp.cls.n >= kMaxClasses) {
                err = "too many distinct (Dirichlet, multiplicity) classes in the mesh";
                return SEM_EINVAL;
            }
            const int c = hp.cls.n++;
            const int32_t cnt = (int32_t)(r - q);
            hp.cls.start[c] = (int32_t)q;
            hp.cls.m[c] = m;
            hp.cls.dir[c] = d;
            hp.cls.idxoff[c] = ioff;
            for (int32_t gq = 0; gq < cnt; ++gq)
                for (int t = 0; t < m; ++t)
                    hp.cidx[ioff + (int64_t)t * cnt + gq] = hp.idx[hp.off[q + gq] + t];
            ioff += cnt * m;
            q = r;
        }
        hp.cls.start[hp.cls.n] = (int32_t)groups.size();
    }
    // surface ids (for the inter-rank exchange)
    hp.surf_ids.resize(groups.size());
    hp.surf_group.resize(groups.size());
    {
        std::vector<std::pair<int64_t, int32_t>> sg(groups.size());
        for (size_t q = 0; q < groups.size(); ++q) sg[q] = {glo[hp.idx[hp.off[q]]], (int32_t)q};
        std::sort(sg.begin(), sg.end());
        for (size_t q = 0; q < sg.size(); ++q) {
            hp.surf_ids[q] = sg[q].first;
            hp.surf_group[q] = sg[q].second;
        }
    }
    return SEM_OK;
}
}  // namespace

// ---------------------------------------------------------------------------
// setup / teardown
// ---------------------------------------------------------------------------
// orders where the split K1 with the CUDA-core operator beats the fused K1
// (c4 CG, r02: N = 9 31.6 vs 28.0 GDOF/s; the fused K1 wins at 3..6 and 8 --
// 35.2 / 35.3 / 37.4 / 36.9 / 36.5 vs 31.8 / 31.4 / 32.2 / 32.1 / 31.4)
static bool k1dot_default(int N) { return N == 9; }

extern "C" int sem_setup(const sem_mesh *mesh, int N, void *workspace, size_t bytes,
                         void *cuda_stream, sem_ctx **out) {
    sem_ctx *ctx = nullptr;
    int rc = check_mesh(mesh, N);
    if (rc) return rc;
    if (!out || !workspace || !mesh->xyz || !mesh->glo || !mesh->dirichlet)
        return fail(nullptr, SEM_EINVAL, "NULL argument to sem_setup");
    if (reinterpret_cast<uintptr_t>(workspace) % 256)
        return fail(nullptr, SEM_EINVAL, "workspace must be 256-byte aligned");
    if (mesh->nranks > 1 && (!mesh->nccl_id || !mesh->allgather))
        return fail(nullptr, SEM_EINVAL, "nranks > 1 needs nccl_id and allgather");
    const Layout Lo = make_layout(N, mesh->nelem, mesh->nranks, mesh->alpha != nullptr);
    {
        const int64_t Lh = int64_t(mesh->nelem) * (N + 1) * (N + 1) * (N + 1);
        for (int64_t l = 0; mesh->kappa && l < Lh; ++l)
            if (!(mesh->kappa[l] > 0.0) || !std::isfinite(mesh->kappa[l]))
                return fail(nullptr, SEM_EINVAL, "kappa[%lld] must be > 0 and finite", (long long)l);
        for (int64_t l = 0; mesh->alpha && l < Lh; ++l)
            if (!(mesh->alpha[l] >= 0.0) || !std::isfinite(mesh->alpha[l]))
                return fail(nullptr, SEM_EINVAL, "alpha[%lld] must be >= 0 and finite", (long long)l);
    }
    if (bytes < Lo.total)
        return fail(nullptr, SEM_EINVAL, "workspace too small: %zu < %zu", bytes, Lo.total);
    *out = nullptr;

    HostPlan hp;
    std::string perr;
    rc = build_plan(mesh, N, hp, perr);
    if (rc) return fail(nullptr, rc, "%s", perr.c_str());

    ctx = new (std::nothrow) sem_ctx;
    if (!ctx) return fail(nullptr, SEM_EINVAL, "out of host memory");
    ctx->N = N;
    ctx->n = N + 1;
    ctx->n3 = ctx->n * ctx->n * ctx->n;
    ctx->E = mesh->nelem;
    ctx->L = ctx->E * ctx->n3;
    ctx->rank = mesh->rank;
    ctx->nranks = mesh->nranks;
    ctx->device = mesh->device;
    ctx->stream = (cudaStream_t)cuda_stream;
    ctx->nglobal = hp.ndistinct;
    auto bail = [&](int code) {
        sem_free(ctx);
        return code;
    };
    {
        cudaError_t e = cudaSetDevice(mesh->device);
        if (e != cudaSuccess) {
            fail(nullptr, SEM_ECUDA, "cudaSetDevice(%d): %s", mesh->device, cudaGetErrorString(e));
            return bail(SEM_ECUDA);
        }
    }
    char *ws = static_cast<char *>(workspace);
    DevMesh &dm = ctx->dm;
    dm.N = N;
    dm.n = ctx->n;
    dm.n3 = ctx->n3;
    dm.E = ctx->E;
    dm.L = ctx->L;
    dm.D = reinterpret_cast<double *>(ws + Lo.D);
    dm.G = reinterpret_cast<double *>(ws + Lo.G);
    dm.BM = reinterpret_cast<double *>(ws + Lo.BM);
    dm.H = mesh->alpha ? reinterpret_cast<double *>(ws + Lo.H) : nullptr;
    dm.cls = hp.cls;
    dm.gs_idx = reinterpret_cast<int32_t *>(ws + Lo.gs_idx);
    dm.ngroups = hp.ngroups;
    dm.ndir = hp.ndir;
    dm.nsurf = (int32_t)hp.idx.size();
    dm.rank = ctx->rank;
    dm.nranks = ctx->nranks;
    CgVecs &cv = ctx->cv;
    cv.r = reinterpret_cast<double *>(ws + Lo.r);
    cv.p = reinterpret_cast<double *>(ws + Lo.p);
    cv.w = reinterpret_cast<double *>(ws + Lo.w);
    cv.xw = reinterpret_cast<double *>(ws + Lo.xw);
    cv.part1 = reinterpret_cast<double *>(ws + Lo.partials);
    cv.part2 = cv.part1 + 2 * Lo.partial_cap;
    cv.part3 = cv.part2 + 2 * Lo.partial_cap;
    cv.z = reinterpret_cast<double *>(ws + Lo.z);
    cv.dinv = nullptr;
    ctx->dinv_buf = reinterpret_cast<double *>(ws + Lo.dinv);
    cv.s1 = cv.s2 = (int)Lo.partial_cap;
    cv.rr_all = reinterpret_cast<double *>(ws + Lo.rr_all);
    cv.rz_all = cv.rr_all + kRing * ctx->nranks;     // cg_device.cuh rho_src_t relies on it
    cv.pap_all = reinterpret_cast<double *>(ws + Lo.pap_all);
    cv.st = reinterpret_cast<CgState *>(ws + Lo.st);
    {
        int nsm = 148;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, mesh->device);
        dm.nsm = nsm;
        // Ax kernel family: element-staged TMA (low N), vector-staged TMA +
        // register-streamed G^ (high N), or the simple kernel (SEM_AX_KERNEL=
        // simple|tma|hi forces one; SEM_HI_MIN_N moves the automatic switch)
        const char *impl = getenv("SEM_AX_KERNEL");
        const char *himin = getenv("SEM_HI_MIN_N");
        // measured c4 sweep (profiles/order_sweep_r01*.json): element-staged
        // TMA wins up to N = 10, slice-streamed from N = 11
        const int hi_min = himin ? atoi(himin) : 11;
        // (the simple kernel has no mass term: not used for screened operators)
        const bool force_simple = impl && strcmp(impl, "simple") == 0 && !dm.H;
        const bool force_tma = impl && strcmp(impl, "tma") == 0;
        const bool force_hi = impl && strcmp(impl, "hi") == 0;
        dm.use_hi = !force_simple && !force_tma && hi_supported(N) && (force_hi || N >= hi_min);
        dm.use_tma = !force_simple && !dm.use_hi && tma_supported(N);
        // DMMA contractions for N = 7 (default; SEM_AX_KERNEL=tma|hi|simple
        // select the CUDA-core kernels); the TMA family serves every variant it
        // does not cover (mass term, preconditioner, single reduction)
        const bool force_dmma = impl && strcmp(impl, "dmma") == 0;
        dm.use_dmma = dmma_supported(N) && (force_dmma || (!impl || !*impl));
        if (dm.use_dmma) {
            dm.use_hi = false;
            dm.use_tma = true;
        }
        // the plain Ax at N = 8..14 on the tensor cores: default where it wins
        // (c4: N=10 0.47 vs 0.44, 11 0.58 vs 0.43, 12 0.44 vs 0.30, 13 0.39 vs
        // 0.36, 14 0.47 vs 0.29, 15 0.51 vs 0.38; N=8, 9 lose to the TMA kernel, the 2x2 tiles
        // of 8 waste 68% / 61% of the DMMA work there); SEM_DMMAG=1 forces it
        // for 8..14, SEM_DMMAG=0 disables it; K1 keeps the CUDA-core kernels
        const char *dg = getenv("SEM_DMMAG");
        const bool dg_on = dg ? dg[0] == '1' : (force_dmma || !impl || !*impl) && N >= 10;
        dm.use_dmmag = dmmag_supported(N) && (dm.use_tma || dm.use_hi) && dg_on;
        // the split K1 (x / p update + tensor-core operator with (p,Ap)) where
        // it beats the fused CUDA-core K1: N >= 11 (c4 CG per iteration, r02o:
        // N=11 544 vs 591 us, 12 679 vs 788, 13 569 vs 668, 14 594 vs 829,
        // 15 568 vs 671; N=10 586 vs 569).  SEM_K1_AX=fused|split forces.
        const char *k1ax = getenv("SEM_K1_AX");
        const bool ax_fused = k1ax && strcmp(k1ax, "fused") == 0;
        const bool ax_split = k1ax && strcmp(k1ax, "split") == 0;
        dm.use_k1ax = dm.use_dmmag && !ax_fused && (ax_split || N >= 11);
        // the split with the CUDA-core operator where no tensor-core Ax runs
        // (SEM_K1_AX=split forces it; default orders below, measured r02)
        if (!dm.use_dmmag && !dm.use_dmma && (dm.use_tma || dm.use_hi) && !ax_fused &&
            (ax_split || k1dot_default(N)))
            dm.use_k1ax = true;
        if (dm.H) dm.use_k1ax = false;             // (the tensor-core operator has no mass term)
        if (dm.H && !dm.use_tma && !dm.use_hi) {   // only TMA / hi carry the mass term
            dm.use_hi = hi_supported(N) && N >= hi_min;
            dm.use_tma = !dm.use_hi && tma_supported(N);
            if (!dm.use_tma && !dm.use_hi) dm.use_hi = hi_supported(N);
        }
        const char *gr = getenv("SEM_CG_GRAPH");
        ctx->use_graph = !(gr && strcmp(gr, "0") == 0);
        // L2 persistence of the CG work vectors (opt-in, SEM_L2_PERSIST=1):
        // r, p, w, xw are contiguous in the workspace; the persisting
        // set-aside is raised to cover them (device-wide limit, only raised).
        // Off by default: the vectors already stay L2-resident under the
        // kernels' evict-first G^ / evict-last vector hints (application-replay
        // ncu r02: K1 reads ~104 MB of DRAM per launch, G^ alone is 100.7) and
        // c3 measured the same with and without (bench r02f: 48.3-48.5 GDOF/s)
        const char *lp = getenv("SEM_L2_PERSIST");
        if (lp && lp[0] == '1') {
            int maxp = 0, maxw = 0;
            cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, mesh->device);
            cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, mesh->device);
            const size_t span = (size_t)((const char *)(cv.xw + ctx->L) - (const char *)cv.r);
            const size_t win = std::min(span, (size_t)maxw);
            size_t cur = 0;
            cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
            const size_t want = std::min(win, (size_t)maxp);
            if (want > cur) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
            cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
            if (win > 0 && cur > 0) {
                ctx->l2win.base_ptr = (void *)cv.r;
                ctx->l2win.num_bytes = win;
                ctx->l2win.hitRatio = (float)std::min(1.0, (double)cur / (double)win);
                ctx->l2win.hitProp = cudaAccessPropertyPersisting;
                ctx->l2win.missProp = cudaAccessPropertyStreaming;
                ctx->l2_on = true;
            }
            if (getenv("SEM_L2_VERBOSE"))
                fprintf(stderr, "libsem L2: max persisting %d B, max window %d B, span %zu B, limit %zu B, hitRatio %.3f\n",
                        maxp, maxw, span, cur, (double)ctx->l2win.hitRatio);
            cudaGetLastError();   // (attribute queries are best effort)
        }
    }
    // one rank: SEM_K1_SPLIT=<fraction of E> exercises the boundary/interior
    // K1 split without an exchange (testing only; multi-rank sets nbnd below)
    if (ctx->nranks == 1) {
        const char *sp = getenv("SEM_K1_SPLIT");
        dm.nbnd = sp ? (int64_t)(atof(sp) * (double)dm.E) : 0;
        if (dm.n3 & 1) dm.nbnd += dm.nbnd & 1;     // range launches need eb n^3 even
    }
    cv.nb1 = ax_cg_blocks(dm);
    cv.nb2 = k2_blocks(dm, false);
    if (cv.nb1 > cv.s1 || cv.nb2 > cv.s2) {
        fail(nullptr, SEM_EINVAL, "device has too many SMs for the partial buffers");
        return bail(SEM_EINVAL);
    }

    rc = [&]() -> int {
        const int n = ctx->n;
        std::vector<double> xw(n), wq(n), Dh(n * n + n);
        sem_gll(N, xw.data(), wq.data());
        diff_matrix(N, xw.data(), Dh.data());
        for (int i = 0; i < n; ++i) Dh[n * n + i] = wq[i];
        cudaStream_t s = ctx->stream;
        CU(cudaHostAlloc(&ctx->host_state, 2 * sizeof(CgState), cudaHostAllocDefault));
        CU(upload_const_D(N, Dh.data()));
        if (dm.use_tma) CU(tma_prepare(N, dm.H != nullptr));
        if (dm.use_hi) CU(hi_prepare(N, dm.H != nullptr));
        if ((dm.use_tma || dm.use_hi) && !dm.H) CU(sr_prepare(dm));
        if (dm.use_dmmag) CU(dmmag_prepare(N));
        {
            // one rank only: with several ranks the chunks' exchanges pair up
            // with the peers', and the harness transports (loopback, p2p on one
            // GPU) rely on the in-stream copy's pacing (timeouts without it)
            const char *ps = getenv("SEM_POLL_STREAM");
            if (ctx->nranks == 1 && !(ps && ps[0] == '0')) {
                CU(cudaStreamCreateWithFlags(&ctx->poll_stream, cudaStreamNonBlocking));
                CU(cudaEventCreateWithFlags(&ctx->chunk_ev[0], cudaEventDisableTiming));
                CU(cudaEventCreateWithFlags(&ctx->chunk_ev[1], cudaEventDisableTiming));
            }
        }
        CU(cudaEventCreateWithFlags(&ctx->ev[0], cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&ctx->ev[1], cudaEventDisableTiming));
        CU(cudaMemcpyAsync((void *)dm.D, Dh.data(), sizeof(double) * Dh.size(),
                           cudaMemcpyHostToDevice, s));
        if (!hp.cidx.empty())
            CU(cudaMemcpyAsync((void *)dm.gs_idx, hp.cidx.data(), sizeof(int32_t) * hp.cidx.size(),
                               cudaMemcpyHostToDevice, s));
        CU(cudaMemsetAsync(cv.st, 0, sizeof(CgState), s));
        // resident CG (cg_resident.cu): the push-based DSSUM tables.  Copy c of
        // element e at node position q with m copies (ascending c_0 < .. <
        // c_{m-1}, c = c_pos) receives the values of the m - 1 other copies in
        // ascending order into X[e S + sb(q) + t], t < m - 1 (S slots per
        // element, sb(q) = prefix of the per-position reservation R(q) = max
        // over elements of m - 1); push[e S + sb(q) + t] is where c writes its
        // own value for the t-th other copy (ascending).  meta = m | pos << 4
        // (m = 0: Dirichlet copy, never updated).
        if (Lo.rcg_meta && rcg_supported(dm)) {
            const int n3 = ctx->n3;
            const int64_t L = ctx->L;
            std::vector<uint8_t> meta(L, 1);      // interior / unshared: m = 1, pos = 0
            std::vector<int32_t> Rq(n3, 0);
            int mmax = 1;
            for (int32_t q = 0; q < hp.ngroups; ++q) {
                const int32_t a0 = hp.off[q], a1 = hp.off[q + 1], mq = a1 - a0;
                for (int32_t t = a0; t < a1; ++t) {
                    const int32_t c = hp.idx[t];
                    if (q < hp.ndir) {
                        meta[c] = 0;
                    } else {
                        meta[c] = (uint8_t)((mq & 15) | ((t - a0) << 4));
                        Rq[c % n3] = std::max(Rq[c % n3], mq - 1);
                    }
                }
                if (q >= hp.ndir) mmax = std::max(mmax, (int)mq);
            }
            std::vector<int32_t> sbq(n3 + 1, 0);
            for (int q = 0; q < n3; ++q) sbq[q + 1] = sbq[q] + Rq[q];
            const int64_t S = (sbq[n3] + 3) & ~int64_t(3);      // 16-byte bulk copies (X and push)
            if (mmax <= kRcgMaxM && S <= kRcgMaxSlots) {
                std::vector<int32_t> push((size_t)(ctx->E * S), -1);
                auto xslot = [&](int32_t c, int t) {
                    return (int64_t)(c / n3) * S + sbq[c % n3] + t;
                };
                for (int32_t q = hp.ndir; q < hp.ngroups; ++q) {
                    const int32_t a0 = hp.off[q], mq = hp.off[q + 1] - a0;
                    for (int j = 0; j < mq; ++j) {
                        int t = 0;
                        for (int i = 0; i < mq; ++i) {
                            if (i == j) continue;
                            // c_j's value is c_i's ((j < i) ? j : j - 1)-th other copy
                            push[xslot(hp.idx[a0 + j], t++)] = (int32_t)xslot(hp.idx[a0 + i], j < i ? j : j - 1);
                        }
                    }
                }
                std::vector<int32_t> sbh(sbq.begin(), sbq.begin() + n3);
                RcgBufs &rb = ctx->rcg;
                rb.S = (int32_t)S;
                rb.meta = reinterpret_cast<uint8_t *>(ws + Lo.rcg_meta);
                rb.sbq = reinterpret_cast<int32_t *>(ws + Lo.rcg_sbq);
                rb.push = reinterpret_cast<int32_t *>(ws + Lo.rcg_push);
                rb.X = reinterpret_cast<double *>(ws + Lo.rcg_X);
                rb.part = reinterpret_cast<double *>(ws + Lo.rcg_part);
                rb.bar = reinterpret_cast<uint32_t *>(ws + Lo.rcg_bar);
                CU(cudaMemcpyAsync(rb.meta, meta.data(), L, cudaMemcpyHostToDevice, s));
                CU(cudaMemcpyAsync(rb.sbq, sbh.data(), sizeof(int32_t) * n3, cudaMemcpyHostToDevice, s));
                CU(cudaMemcpyAsync(rb.push, push.data(), sizeof(int32_t) * push.size(),
                                   cudaMemcpyHostToDevice, s));
                CU(rcg_prepare());
                CU(cudaStreamSynchronize(s));   // (host vectors go out of scope)
                ctx->rcg_ok = true;
            }
        }
        CU(cudaMemsetAsync(cv.rr_all, 0, sizeof(double) * kRing * ctx->nranks, s));
        CU(cudaMemsetAsync(cv.rz_all, 0, sizeof(double) * kRing * ctx->nranks, s));
        CU(cudaMemsetAsync(cv.pap_all, 0, sizeof(double) * kRing * ctx->nranks, s));
        // xyz -> device (temporarily in r|p|w, exactly 3L doubles), then G^, B
        double *xyz_d = cv.r;
        int *bad_d = reinterpret_cast<int *>(cv.part1);
        CU(cudaMemcpyAsync(xyz_d, mesh->xyz, sizeof(double) * 3 * ctx->L, cudaMemcpyHostToDevice, s));
        CU(cudaMemsetAsync(bad_d, 0, sizeof(int), s));
        // kappa -> xw (scratch at setup); alpha -> H (scaled in place by w J)
        double *kappa_d = mesh->kappa ? cv.xw : nullptr;
        if (kappa_d)
            CU(cudaMemcpyAsync(kappa_d, mesh->kappa, sizeof(double) * ctx->L, cudaMemcpyHostToDevice, s));
        if (dm.H)
            CU(cudaMemcpyAsync(const_cast<double *>(dm.H), mesh->alpha, sizeof(double) * ctx->L,
                               cudaMemcpyHostToDevice, s));
        LAUNCH(launch_geom(dm, xyz_d, kappa_d, const_cast<double *>(dm.G), const_cast<double *>(dm.BM),
                           const_cast<double *>(dm.H), bad_d, s));
        int bad = 0;
        CU(cudaMemcpyAsync(&bad, bad_d, sizeof(int), cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        if (bad) return fail(ctx, SEM_EINVAL, "non-positive Jacobian in the mesh");
        if (ctx->nranks > 1) {
            std::string cerr;
            ExchangePlan ep;
            int crc = build_exchange_plan(mesh, hp.surf_ids, hp.surf_group, hp.ndistinct, ep, cerr);
            if (crc) return fail(ctx, crc, "%s", cerr.c_str());
            ctx->nglobal = ep.nglobal;
            crc = comm_setup(ctx->comm, mesh, ep, dm, s, cerr);
            if (crc) return fail(ctx, crc, "%s", cerr.c_str());
            if (!comm_capturable(ctx->comm)) ctx->use_graph = false;   // loopback transport
            // (r,r) ownership of interface groups: the lowest sharing rank counts them
            std::vector<uint32_t> own((hp.ngroups + 31) / 32 + 1, 0xffffffffu);
            for (int32_t g : ep.not_owned) own[g >> 5] &= ~(1u << (g & 31));
            uint32_t *own_d = reinterpret_cast<uint32_t *>(ws + Lo.own);
            CU(cudaMemcpyAsync(own_d, own.data(), sizeof(uint32_t) * own.size(),
                               cudaMemcpyHostToDevice, s));
            CU(cudaStreamSynchronize(s));
            dm.own = own_d;
            // boundary elements: every element holding a copy of a node the
            // exchange reads or writes lies in [0, nbnd) -- derived here from
            // the plan (mesh->nboundary is only an ordering hint)
            int64_t nbnd = 0;
            auto cover = [&](int32_t g) {
                for (int32_t t = hp.off[g]; t < hp.off[g + 1]; ++t)
                    nbnd = std::max<int64_t>(nbnd, hp.idx[t] / ctx->n3 + 1);
            };
            for (int32_t g : ep.send_group) cover(g);
            for (int32_t g : ep.if_group) cover(g);
            if (dm.n3 & 1) nbnd += nbnd & 1;            // range launches need eb n^3 even
            dm.nbnd = nbnd;
            cv.nb1 = ax_cg_blocks(dm);
            if (cv.nb1 > cv.s1) return fail(ctx, SEM_EINVAL, "too many K1 partials");
        }
        if (k1_split(dm)) {
            CU(cudaStreamCreateWithPriority(&ctx->side, cudaStreamNonBlocking, -1));
            CU(cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming));
            CU(cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming));
        }
        // peer-memory transport: capture, instantiate and upload the chunk
        // graphs of every method now, while no collective is in flight -- a
        // later instantiation could stall on a peer's spinning kernel when
        // several ranks share a device (include/sem.h)
        if (ctx->nranks > 1 && comm_device_only(ctx->comm) && ctx->use_graph) {
            const bool tma_like = dm.use_tma || dm.use_hi;
            for (int meth = 0; meth < 3; ++meth) {
                if (meth == 2 && (!tma_like || dm.H)) continue;     // (sem_cg_sr's limits)
                ctx->method = meth;
                cv.dinv = (meth == 1) ? ctx->dinv_buf : nullptr;
                int brc = build_cg_graph(ctx);
                if (brc) return brc;
                CU(cudaGraphUpload(ctx->graph_exec[meth], s));
            }
            cv.dinv = nullptr;
            ctx->method = 0;
            CU(cudaStreamSynchronize(s));
            // no rank leaves setup while another is still capturing (a
            // device-wide synchronisation elsewhere would invalidate it)
            int one = 1, all[kMaxRanks];
            if (mesh->allgather(mesh->allgather_user, &one, sizeof one, all) != 0)
                return fail(ctx, SEM_ENCCL, "setup all-gather (graph capture) failed");
        }
        return SEM_OK;
    }();
    if (rc) {
        g_err = ctx->err;
        return bail(rc);
    }
    *out = ctx;
    return SEM_OK;
}

extern "C" int sem_exchange_plan(const sem_mesh *mesh, int N, int64_t *counts, int64_t *ids,
                                 int64_t cap, int64_t *nslot, int64_t *nglobal) {
    int rc = check_mesh(mesh, N);
    if (rc) return rc;
    if (!mesh->glo || !mesh->dirichlet || !counts || !nslot || !nglobal)
        return fail(nullptr, SEM_EINVAL, "NULL argument to sem_exchange_plan");
    HostPlan hp;
    std::string err;
    rc = build_plan(mesh, N, hp, err);
    if (rc) return fail(nullptr, rc, "%s", err.c_str());
    ExchangePlan ep;
    rc = build_exchange_plan(mesh, hp.surf_ids, hp.surf_group, hp.ndistinct, ep, err);
    if (rc) return fail(nullptr, rc, "%s", err.c_str());
    *nslot = (int64_t)ep.shared_ids.size();
    *nglobal = ep.nglobal;
    for (int q = 0; q < mesh->nranks; ++q) counts[q] = 0;
    for (size_t p = 0; p < ep.peer.size(); ++p) counts[ep.peer[p]] = ep.peer_off[p + 1] - ep.peer_off[p];
    if (*nslot > cap || (*nslot > 0 && !ids))
        return fail(nullptr, SEM_EINVAL, "sem_exchange_plan: ids capacity %lld < %lld",
                    (long long)cap, (long long)*nslot);
    std::copy(ep.shared_ids.begin(), ep.shared_ids.end(), ids);
    return SEM_OK;
}

extern "C" void sem_free(sem_ctx *ctx) {
    if (!ctx) return;
    if (ctx->graph_exec[0] || ctx->graph_exec[1] || ctx->graph_exec[2] || ctx->replay_exec || ctx->l2_on)
        cudaStreamSynchronize(ctx->stream);
    if (ctx->l2_on) cudaCtxResetPersistingL2Cache();   // the work vectors' lines back to normal
    for (auto &g : ctx->graph_exec)
        if (g) cudaGraphExecDestroy(g);

    if (ctx->replay_exec) cudaGraphExecDestroy(ctx->replay_exec);
    if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
    if (ctx->side) cudaStreamDestroy(ctx->side);
    if (ctx->poll_stream) {
        cudaStreamSynchronize(ctx->poll_stream);
        cudaStreamDestroy(ctx->poll_stream);
    }
    for (auto &e : ctx->chunk_ev)
        if (e) cudaEventDestroy(e);
    if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
    if (ctx->join_ev) cudaEventDestroy(ctx->join_ev);
    if (ctx->comm) comm_free(ctx->comm);
    if (ctx->host_state) cudaFreeHost(ctx->host_state);
    for (auto &r : ctx->recs) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : ctx->evpool) cudaEventDestroy(e);
    for (auto &e : ctx->ev)
        if (e) cudaEventDestroy(e);
    delete ctx;
}

extern "C" int sem_sizes(const sem_ctx *ctx, int64_t *nlocal, int64_t *nglobal) {
    if (!ctx) return fail(nullptr, SEM_ESTATE, "NULL context");
    if (nlocal) *nlocal = ctx->L;
    if (nglobal) *nglobal = ctx->nglobal;
    return SEM_OK;
}

extern "C" int64_t sem_launch_count(const sem_ctx *ctx) { return ctx ? ctx->launches : -1; }

#define CHECK_CTX()                                                                  \
    do {                                                                             \
        if (!ctx) return fail(nullptr, SEM_ESTATE, "NULL context");                  \
        if (ctx->broken) return fail(ctx, SEM_ECUDA, "context unusable after a CUDA error"); \
    } while (0)

// vectors are staged by 16-byte bulk copies and read / written as double2
static bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

extern "C" int sem_ax(sem_ctx *ctx, const double *u, double *w) {
    CHECK_CTX();
    if (!u || !w || !aligned16(u) || !aligned16(w)) return fail(ctx, SEM_EINVAL, "sem_ax: bad pointer");
    if (u == w) return fail(ctx, SEM_EINVAL, "sem_ax: u and w must not alias");
    LAUNCHP(kProfAx, (ctx->dm.H ? 72.0 : 64.0) * ctx->L, -1, launch_ax(ctx->dm, u, w, ctx->stream));
    return SEM_OK;
}

// Cross-rank part of Q Q^T (no-op on one rank): after it, every interface
// node's first local copy holds the rank-ordered total and the others 0.
static int exchange_impl(sem_ctx *ctx, double *w, cudaStream_t s) {
    if (ctx->nranks == 1) return SEM_OK;
    std::string cerr;
    int64_t nl = 0;
    int rc = comm_exchange(ctx->comm, ctx->dm, w, s, nl, cerr);
    ctx->launches += nl;
    if (rc) {
        if (rc == SEM_ECUDA) ctx->broken = true;
        return fail(ctx, rc, "%s", cerr.c_str());
    }
    return SEM_OK;
}

static int dssum_impl(sem_ctx *ctx, double *w, int mode, int k, cudaStream_t s) {
    int rc = exchange_impl(ctx, w, s);
    if (rc) return rc;
    const double by = 16.0 * ctx->dm.nsurf;
    LAUNCHP(kProfGs, by, mode == 2 ? k : -1, launch_gs(ctx->dm, w, mode, &ctx->cv, s));
    return SEM_OK;
}

// A failed collective of the peer-memory transport (a spin that timed out)
// is sticky: every later collective of the context reports it.
static int transport_ok(sem_ctx *ctx) {
    if (ctx->nranks == 1 || !ctx->comm) return SEM_OK;
    std::string cerr;
    if (comm_poll(ctx->comm, cerr)) {
        ctx->broken = true;
        return fail(ctx, SEM_ENCCL, "%s", cerr.c_str());
    }
    return SEM_OK;
}

extern "C" int sem_status(sem_ctx *ctx) {
    if (!ctx) return fail(nullptr, SEM_ESTATE, "NULL context");
    int rc = transport_ok(ctx);
    if (rc) return rc;
    return ctx->broken ? SEM_ECUDA : SEM_OK;
}

extern "C" int sem_dssum(sem_ctx *ctx, double *w) {
    CHECK_CTX();
    if (int rc = transport_ok(ctx)) return rc;
    if (!w || !aligned16(w)) return fail(ctx, SEM_EINVAL, "sem_dssum: bad pointer");
    return dssum_impl(ctx, w, 0, -1, ctx->stream);
}

extern "C" int sem_mask(sem_ctx *ctx, double *w) {
    CHECK_CTX();
    if (!w || !aligned16(w)) return fail(ctx, SEM_EINVAL, "sem_mask: bad pointer");
    if (ctx->dm.ndir > 0) LAUNCH(launch_mask(ctx->dm, w, ctx->stream));
    return SEM_OK;
}

extern "C" int sem_mass(sem_ctx *ctx, const double *f, double *b) {
    CHECK_CTX();
    if (!f || !b || !aligned16(f) || !aligned16(b)) return fail(ctx, SEM_EINVAL, "sem_mass: bad pointer");
    LAUNCH(launch_mass(ctx->dm, f, b, ctx->stream));
    return SEM_OK;
}

// ---------------------------------------------------------------------------
// a9: CG driver
// ---------------------------------------------------------------------------
// site: which all-gather of the iteration (kSitePap / kSiteRr / kSiteRz; the
// peer-memory transport keeps one epoch counter and slot set per site)
static int allgather_scalar(sem_ctx *ctx, double *slot_base, int site, cudaStream_t s) {
    if (ctx->nranks == 1) return SEM_OK;
    std::string cerr;
    int rc = comm_allgather(ctx->comm, slot_base, 1, site, s, cerr);
    if (rc) return fail(ctx, rc, "%s", cerr.c_str());
    return SEM_OK;
}

// The rank fold of one CG scalar (which: 0 (p,Ap), 1 (r,r), 2 (r,z)) and its
// all-gather: one kernel with the peer-memory transport (the fold does the
// all-gather), else the fold, then the transport's all-gather.  wait_ev: an
// event the all-gather must also wait for (the side-stream exchange).
static int fold_allgather(sem_ctx *ctx, int which, double *slot_base, cudaStream_t s,
                          cudaEvent_t wait_ev = nullptr) {
    const P2PDev *p2p = comm_p2p_dev(ctx->comm);
    if (which == 0) LAUNCH(launch_cg_red_pap(ctx->dm, ctx->cv, p2p, s));
    else if (which == 1) LAUNCH(launch_cg_red_rr(ctx->dm, ctx->cv, p2p, s));
    else LAUNCH(launch_cg_red_rz(ctx->dm, ctx->cv, p2p, s));
    // (the join: everything after -- the NCCL all-gather, whose order on the
    // one communicator must follow the exchange's, and K2 -- waits for the
    // side-stream exchange; the fused p2p fold uses its own flags and runs
    // concurrently with the exchange)
    if (wait_ev) CU(cudaStreamWaitEvent(s, wait_ev, 0));
    if (p2p) return SEM_OK;
    static const int site[3] = {kSitePap, kSiteRr, kSiteRz};
    return allgather_scalar(ctx, slot_base, site[which], s);
}

// Algorithmic bytes of one K2 launch: w copies read + r copies written at
// surface nodes, r read once per non-Dirichlet group, and r read/write + w
// read at element-interior nodes.
// Jacobi PCG adds z written at every copy and dinv read once per group.
static double k2_bytes(const sem_ctx *ctx) {
    const int64_t ni = ctx->N - 1;
    const double nint = double(ctx->E) * ni * ni * ni;
    const double pc = ctx->cv.dinv ? 1.0 : 0.0;
    return (16.0 + 8.0 * pc) * ctx->dm.nsurf + (8.0 + 8.0 * pc) * (ctx->dm.ngroups - ctx->dm.ndir) +
           (24.0 + 16.0 * pc) * nint;
}

// One CG iteration: K1 (x/p update + Ax + (w,p) -> pap slot), [all-gather of
// pap], K2 (Q Q^T w + mask fused with r -= alpha w and (r,r) -> rr slot),
// [all-gather of rr].  k: host count (all-gather slot k & 3 and profiling
// only; the kernels read k from the device state).
static int enqueue_iteration(sem_ctx *ctx, int k, cudaStream_t s) {
    CgVecs &v = ctx->cv;
    const int P = ctx->nranks;
    int rc;
    // K1 algorithmic bytes per local node (+8: the mass diagonal, screened operator)
    // (split K1, use_k1ax: x / p update 40 B (16 at k = 0) + operator 64 B)
    const double k1_bpn = ctx->dm.use_k1ax ? (k == 0 ? 80.0 : 104.0)
                                           : (k == 0 ? 72.0 : 96.0) + (ctx->dm.H ? 8.0 : 0.0);
    if (k1_split(ctx->dm)) {
        // boundary elements first; the exchange of their w runs on the side
        // stream while the interior elements' K1 runs here
        const DevMesh &m = ctx->dm;
        const int64_t nb = m.nbnd, ni = m.E - m.nbnd;
        const int gA = ax_cg_range_blocks(m, nb);
        LAUNCHP(kProfAxCg, k1_bpn * m.n3 * nb, k, launch_ax_cg_range(m, v, 0, nb, 0, s));
        ctx->launches += m.use_k1ax ? 1 : 0;
        if (P > 1) CU(cudaEventRecord(ctx->fork_ev, s));
        // the interior launch is enqueued before the exchange: a transport
        // whose enqueue blocks the host (the loopback rendezvous) must not
        // hold it back (profiles/overlap_r02.md)
        LAUNCHP(kProfAxCg, k1_bpn * m.n3 * ni, k, launch_ax_cg_range(m, v, nb, ni, gA, s));
        ctx->launches += m.use_k1ax ? 1 : 0;
        if (P > 1) {
            CU(cudaStreamWaitEvent(ctx->side, ctx->fork_ev, 0));
            if ((rc = exchange_impl(ctx, v.w, ctx->side))) return rc;
            CU(cudaEventRecord(ctx->join_ev, ctx->side));
            if ((rc = fold_allgather(ctx, 0, v.pap_all + (k & 3) * P, s, ctx->join_ev))) return rc;
        }
    } else {
        LAUNCHP(kProfAxCg, k1_bpn * ctx->L, k, launch_ax_cg(ctx->dm, v, s));
        ctx->launches += ctx->dm.use_k1ax ? 1 : 0;
        if (P > 1) {
            if ((rc = exchange_impl(ctx, v.w, s))) return rc;
            if ((rc = fold_allgather(ctx, 0, v.pap_all + (k & 3) * P, s))) return rc;
        }
    }
    LAUNCHP(kProfK2, k2_bytes(ctx), k, launch_k2(ctx->dm, v, false, s));
    if (P > 1) {
        if ((rc = fold_allgather(ctx, 1, v.rr_all + ((k + 1) & 3) * P, s))) return rc;
        if (v.dinv && (rc = fold_allgather(ctx, 2, v.rz_all + ((k + 1) & 3) * P, s))) return rc;
    }
    return SEM_OK;
}

// Single-reduction CG (NEXT-3): KA (w = A_L r, (r,w) partials), [exchange of
// w, fold + ONE all-gather of the (gamma, delta) pair], KB (DSSUM + the
// recurrences + (r,r) partials; the only scalar reduction of the iteration).
static double kb_bytes(const sem_ctx *ctx) {
    const int64_t ni = ctx->N - 1;
    const double nint = double(ctx->E) * ni * ni * ni;
    return 16.0 * ctx->dm.nsurf + 56.0 * (ctx->dm.ngroups - ctx->dm.ndir) + 72.0 * nint;
}

static int enqueue_iteration_sr(sem_ctx *ctx, int k, cudaStream_t s) {
    CgVecs &v = ctx->cv;
    const int P = ctx->nranks;
    int rc;
    LAUNCHP(kProfAxCg, 64.0 * ctx->L, k, launch_ax_dot(ctx->dm, v, s));
    if (P > 1) {
        if ((rc = exchange_impl(ctx, v.w, s))) return rc;
        const P2PDev *p2p = comm_p2p_dev(ctx->comm);
        LAUNCH(launch_sr_fold(ctx->dm, v, p2p, s));     // (p2p: the all-gather inside)
        if (!p2p) {
            std::string cerr;
            rc = comm_allgather(ctx->comm, v.rr_all + (k & 3) * 2 * P, 2, kSiteSr, s, cerr);
            if (rc) return fail(ctx, rc, "%s", cerr.c_str());
        }
    }
    LAUNCHP(kProfK2, kb_bytes(ctx), k, launch_kb_sr(ctx->dm, v, s));
    return SEM_OK;
}

// Capture kChunk iterations once per context and method into a CUDA graph (on
// a private non-blocking stream; the graph is launched into the caller's stream).
static int build_cg_graph(sem_ctx *ctx) {
    if (!ctx->cap_stream) CU(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    const int64_t l0 = ctx->launches;
    CU(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
    int rc = SEM_OK;
    for (int q = 0; q < kChunk && rc == SEM_OK; ++q)
        rc = ctx->method == 2 ? enqueue_iteration_sr(ctx, q, ctx->cap_stream)
                              : enqueue_iteration(ctx, q, ctx->cap_stream);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(ctx->cap_stream, &g);
    ctx->graph_kernels[ctx->method] = ctx->launches - l0;
    ctx->launches = l0;
    if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
    }
    CU(e);
    if (ctx->l2_on) {
        // every kernel node of the chunk keeps the work vectors L2-resident
        size_t nn = 0;
        CU(cudaGraphGetNodes(g, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        CU(cudaGraphGetNodes(g, nodes.data(), &nn));
        cudaKernelNodeAttrValue av{};
        av.accessPolicyWindow = ctx->l2win;
        for (cudaGraphNode_t nd : nodes) {
            cudaGraphNodeType ty;
            CU(cudaGraphNodeGetType(nd, &ty));
            if (ty == cudaGraphNodeTypeKernel)
                CU(cudaGraphKernelNodeSetAttribute(nd, cudaKernelNodeAttributeAccessPolicyWindow, &av));
        }
    }
    e = cudaGraphInstantiate(&ctx->graph_exec[ctx->method], g, 0);
    cudaGraphDestroy(g);
    CU(e);
    return SEM_OK;
}

// The chunk graph of the current method (captured on first use); none while
// profiling (per-launch events) or with graphs off (SEM_CG_GRAPH=0, loopback).
static int chunk_graph(sem_ctx *ctx, cudaGraphExec_t &gexec) {
    gexec = nullptr;
    if (ctx->prof || !ctx->use_graph) return SEM_OK;
    int rc;
    if (!ctx->graph_exec[ctx->method] && (rc = build_cg_graph(ctx))) return rc;
    gexec = ctx->graph_exec[ctx->method];
    return SEM_OK;
}

// d = Q Q^T diag(A_L) (local storage, unmasked), the assembled diagonal.
static int diag_impl(sem_ctx *ctx, double *d, cudaStream_t s) {
    LAUNCH(launch_diag(ctx->dm, d, s));
    return dssum_impl(ctx, d, 0, -1, s);
}

extern "C" int sem_diag(sem_ctx *ctx, double *d) {
    CHECK_CTX();
    if (!d || !aligned16(d)) return fail(ctx, SEM_EINVAL, "sem_diag: bad pointer");
    return diag_impl(ctx, d, ctx->stream);
}

// Jacobi preconditioner dinv = mask / (Q Q^T diag A_L), once per context.
static int prepare_jacobi(sem_ctx *ctx, cudaStream_t s) {
    if (ctx->dinv_ready) return SEM_OK;
    double *d = ctx->cv.z;            // scratch: z is rewritten by the next K2 start
    int rc = diag_impl(ctx, d, s);
    if (rc) return rc;
    LAUNCH(launch_recip(ctx->dm, d, ctx->dinv_buf, s));
    if (ctx->dm.ndir > 0) LAUNCH(launch_mask(ctx->dm, ctx->dinv_buf, s));
    ctx->dinv_ready = true;
    return SEM_OK;
}

static int cg_impl(sem_ctx *ctx, int precond, const double *b, double *x, double tol, int maxit,
                   int *iters, double *rel_res);

extern "C" int sem_cg(sem_ctx *ctx, const double *b, double *x, double tol, int maxit,
                      int *iters, double *rel_res) {
    CHECK_CTX();
    return cg_impl(ctx, SEM_PC_NONE, b, x, tol, maxit, iters, rel_res);
}

extern "C" int sem_pcg(sem_ctx *ctx, int precond, const double *b, double *x, double tol,
                       int maxit, int *iters, double *rel_res) {
    CHECK_CTX();
    if (precond != SEM_PC_NONE && precond != SEM_PC_JACOBI)
        return fail(ctx, SEM_EINVAL, "sem_pcg: precond must be SEM_PC_NONE or SEM_PC_JACOBI");
    return cg_impl(ctx, precond, b, x, tol, maxit, iters, rel_res);
}

static int cg_sr_impl(sem_ctx *ctx, const double *b, double *x, double tol, int maxit,
                      int *iters, double *rel_res);

extern "C" int sem_cg_sr(sem_ctx *ctx, const double *b, double *x, double tol, int maxit,
                         int *iters, double *rel_res) {
    CHECK_CTX();
    return cg_sr_impl(ctx, b, x, tol, maxit, iters, rel_res);
}

// Wait for an event recorded on the context stream.  With several ranks the
// wait polls, so an asynchronous NCCL failure of a peer (ncclCommGetAsyncError)
// ends it with SEM_ENCCL -- the communicator is aborted and the context marked
// unusable -- instead of blocking forever (SURVEY.md §5 failure detection).
static int wait_event(sem_ctx *ctx, cudaEvent_t ev) {
    if (ctx->nranks == 1) {
        CU(cudaEventSynchronize(ev));
        return SEM_OK;
    }
    for (int spin = 0;; ++spin) {
        cudaError_t e = cudaEventQuery(ev);
        if (e == cudaSuccess) return SEM_OK;
        if (e != cudaErrorNotReady) CU(e);
        std::string cerr;
        if (comm_poll(ctx->comm, cerr)) {
            comm_abort(ctx->comm);
            ctx->broken = true;
            return fail(ctx, SEM_ENCCL, "%s", cerr.c_str());
        }
        if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
}

// Iterations in chunks of kChunk (a multiple of 4: the all-gather slot of
// position q in a chunk is q & 3 == k & 3).  The device decides when to stop;
// the host polls the sticky flag one chunk behind and launches no more chunks
// once it is set (later kernels of a chunk are no-ops).  Each chunk is one
// CUDA-graph launch unless profiling (per-launch events) or graphs are off.
// Returns with the stream's work for the last chunk enqueued.
static int run_chunks(sem_ctx *ctx, int maxit, cudaGraphExec_t gexec, cudaStream_t s) {
    CgVecs &v = ctx->cv;
    const bool graph = gexec != nullptr;
    int rc;
    int64_t k = 0;
    int c = 0;
    while (true) {
        if (graph) {
            CU(cudaGraphLaunch(gexec, s));
            ctx->launches += ctx->graph_kernels[ctx->method];
            k += kChunk;
        } else {
            for (int q = 0; q < kChunk; ++q, ++k) {
                // (the host k only selects all-gather slots (k & 3) and profiling records)
                const int kk = (int)(k & 0x3fffffff);
                rc = ctx->method == 2 ? enqueue_iteration_sr(ctx, kk, s) : enqueue_iteration(ctx, kk, s);
                if (rc) return rc;
            }
        }
        if (ctx->poll_stream) {
            // (the copy may see a later chunk's state words: done / iters are
            // sticky once set, which is all the poll reads)
            CU(cudaEventRecord(ctx->chunk_ev[c & 1], s));
            CU(cudaStreamWaitEvent(ctx->poll_stream, ctx->chunk_ev[c & 1], 0));
            CU(cudaMemcpyAsync(&ctx->host_state[c & 1], v.st, sizeof(CgState), cudaMemcpyDeviceToHost,
                               ctx->poll_stream));
            CU(cudaEventRecord(ctx->ev[c & 1], ctx->poll_stream));
        } else {
            CU(cudaMemcpyAsync(&ctx->host_state[c & 1], v.st, sizeof(CgState), cudaMemcpyDeviceToHost, s));
            CU(cudaEventRecord(ctx->ev[c & 1], s));
        }
        if (c > 0) {
            if ((rc = wait_event(ctx, ctx->ev[(c - 1) & 1]))) return rc;
            if (ctx->host_state[(c - 1) & 1].done) break;
        }
        if (k > (int64_t)maxit + 3 * kChunk) {  // the device must have stopped by now
            if ((rc = wait_event(ctx, ctx->ev[c & 1]))) return rc;
            break;
        }
        ++c;
    }
    // no poll copy may land after the caller's final state copy
    if (ctx->poll_stream) CU(cudaStreamSynchronize(ctx->poll_stream));
    return SEM_OK;
}

static int cg_sr_impl(sem_ctx *ctx, const double *b, double *x, double tol, int maxit,
                      int *iters, double *rel_res) {
    if (!b || !x || !aligned16(b) || !aligned16(x)) return fail(ctx, SEM_EINVAL, "sem_cg_sr: bad pointer");
    if (int rc = transport_ok(ctx)) return rc;
    if (!(tol >= 0.0) || maxit < 0) return fail(ctx, SEM_EINVAL, "sem_cg_sr: tol >= 0 and maxit >= 0 required");
    if (!ctx->dm.use_tma && !ctx->dm.use_hi)
        return fail(ctx, SEM_EINVAL, "sem_cg_sr: needs the TMA / high-order Ax kernels (not SEM_AX_KERNEL=simple)");
    if (ctx->dm.H) return fail(ctx, SEM_EINVAL, "sem_cg_sr: Poisson operator only (no alpha mass term)");
    cudaStream_t s = ctx->stream;
    CgVecs &v = ctx->cv;
    v.b = b;
    v.x = x;
    v.dinv = nullptr;
    ctx->method = 2;
    int rc;
    {
        CgState h{};
        h.tol = tol;
        h.maxit = maxit;
        CU(cudaMemcpyAsync(&v.st->tol, &h.tol, sizeof(double), cudaMemcpyHostToDevice, s));
        CU(cudaMemcpyAsync(&v.st->maxit, &h.maxit, sizeof(int32_t), cudaMemcpyHostToDevice, s));
    }
    // r = mask (b - Q Q^T A_L x0) and (r,r) partials (K2's start); p = s = x increment = 0
    LAUNCH(launch_ax(ctx->dm, x, v.w, s));
    if ((rc = exchange_impl(ctx, v.w, s))) return rc;
    LAUNCH(launch_sr_init(ctx->dm, v, s));
    LAUNCH(launch_k2(ctx->dm, v, true, s));
    cudaGraphExec_t gexec = nullptr;
    if ((rc = chunk_graph(ctx, gexec))) return rc;
    if ((rc = run_chunks(ctx, maxit, gexec, s))) return rc;
    LAUNCH(launch_sr_finish(ctx->dm, v, s));
    CU(cudaMemcpyAsync(&ctx->host_state[0], v.st, sizeof(CgState), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    const CgState &hs = ctx->host_state[0];
    if (int rc = transport_ok(ctx)) return rc;
    if (!hs.done) return fail(ctx, SEM_ECUDA, "sem_cg_sr: device did not reach a stopping decision");
    if (ctx->prof) prof_fold(ctx, hs.iters);
    if (iters) *iters = hs.iters;
    if (rel_res) *rel_res = hs.rel_res;
    if (!hs.converged && tol > 0.0) {
        fail(ctx, SEM_ENOCONV, "sem_cg_sr: maxit=%d reached, rel_res=%.3e > tol=%.3e", maxit, hs.rel_res, tol);
        return SEM_ENOCONV;
    }
    return SEM_OK;
}

// opt-in (SEM_CG_RESIDENT=1): measured slower than the two-kernel schedule at
// c3 (57.8 vs 44.0 us per iteration, DESIGN.md §6 "Resident CG")
static bool rcg_enabled() {
    const char *e = getenv("SEM_CG_RESIDENT");
    return e && e[0] == '1';
}

static int cg_impl(sem_ctx *ctx, int precond, const double *b, double *x, double tol, int maxit,
                   int *iters, double *rel_res) {
    if (!b || !x || !aligned16(b) || !aligned16(x)) return fail(ctx, SEM_EINVAL, "sem_cg: bad pointer");
    if (int rc = transport_ok(ctx)) return rc;
    if (!(tol >= 0.0) || maxit < 0) return fail(ctx, SEM_EINVAL, "sem_cg: tol >= 0 and maxit >= 0 required");
    cudaStream_t s = ctx->stream;
    CgVecs &v = ctx->cv;
    v.b = b;
    v.x = x;
    const int P = ctx->nranks;
    int rc;
    if (precond == SEM_PC_JACOBI && (rc = prepare_jacobi(ctx, s))) return rc;
    v.dinv = (precond == SEM_PC_JACOBI) ? ctx->dinv_buf : nullptr;
    ctx->method = (precond == SEM_PC_JACOBI) ? 1 : 0;
    // tol / maxit into the device state (the init kernel resets the rest)
    {
        CgState h{};
        h.tol = tol;
        h.maxit = maxit;
        CU(cudaMemcpyAsync(&v.st->tol, &h.tol, sizeof(double), cudaMemcpyHostToDevice, s));
        CU(cudaMemcpyAsync(&v.st->maxit, &h.maxit, sizeof(int32_t), cudaMemcpyHostToDevice, s));
    }
    // r = mask (b - Q Q^T A_L x0)
    LAUNCH(launch_ax(ctx->dm, x, v.w, s));
    if ((rc = exchange_impl(ctx, v.w, s))) return rc;
    LAUNCH(launch_cg_init(ctx->dm, v, s));
    LAUNCH(launch_k2(ctx->dm, v, true, s));
    if (P > 1) {
        if ((rc = fold_allgather(ctx, 1, v.rr_all + 0 * P, s))) return rc;
        if (v.dinv && (rc = fold_allgather(ctx, 2, v.rz_all + 0 * P, s))) return rc;
    }

    // one rank, N = 7, Poisson CG: the whole solve as one resident kernel
    // (cg_resident.cu) when SEM_CG_RESIDENT=1
    const bool resident = ctx->rcg_ok && !v.dinv && P == 1 && rcg_enabled();
    if (resident) {
        CU(cudaMemsetAsync(&v.st->rcg_err, 0, sizeof(int32_t), s));
        LAUNCHP(kProfRcg, 0.0, -1, launch_rcg(ctx->dm, v, ctx->rcg, s));
    } else {
        cudaGraphExec_t gexec = nullptr;
        if ((rc = chunk_graph(ctx, gexec))) return rc;
        if ((rc = run_chunks(ctx, maxit, gexec, s))) return rc;
        LAUNCH(launch_cg_finish(ctx->dm, v, s));
    }
    CU(cudaMemcpyAsync(&ctx->host_state[0], v.st, sizeof(CgState), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    const CgState &hs = ctx->host_state[0];
    if (int rc = transport_ok(ctx)) return rc;
    ctx->rcg_last = resident;
    ctx->rcg_iters = hs.iters;
    if (resident && hs.rcg_err)
        return fail(ctx, SEM_ECUDA, "sem_cg: resident CG grid barrier timed out");
    if (!hs.done) return fail(ctx, SEM_ECUDA, "sem_cg: device did not reach a stopping decision");
    if (ctx->prof) prof_fold(ctx, hs.iters);
    if (iters) *iters = hs.iters;
    if (rel_res) *rel_res = hs.rel_res;
    if (!hs.converged && tol > 0.0) {
        fail(ctx, SEM_ENOCONV, "sem_cg: maxit=%d reached, rel_res=%.3e > tol=%.3e", maxit, hs.rel_res, tol);
        return SEM_ENOCONV;
    }
    return SEM_OK;
}

// ---------------------------------------------------------------------------
// profiling (benchmark roofline)
// ---------------------------------------------------------------------------
extern "C" int sem_kernel_replay(sem_ctx *ctx, int which, int reps) {
    CHECK_CTX();
    if (reps < 1 || which < 0 || which > 3)
        return fail(ctx, SEM_EINVAL, "sem_kernel_replay: which in {0,1,2,3}, reps >= 1");
    if (which == 3 && ctx->nranks != 1) return fail(ctx, SEM_EINVAL, "sem_kernel_replay: single rank only");
    if (ctx->nranks != 1) return fail(ctx, SEM_EINVAL, "sem_kernel_replay: single rank only");
    cudaStream_t s = ctx->stream;
    CgVecs &v = ctx->cv;
    // a mid-solve state: not done, iteration 1 (both the x and the p update
    // are live); the partial buffers hold the scalars of the last solve
    {
        CgState h{};
        h.tol = 0.0;
        h.maxit = 1 << 30;
        h.k1 = 1;
        h.k2 = 1;
        CU(cudaMemcpyAsync(&v.st->tol, &h.tol, sizeof(double), cudaMemcpyHostToDevice, s));
        CU(cudaMemcpyAsync(&v.st->maxit, &h.maxit, sizeof(int32_t), cudaMemcpyHostToDevice, s));
        CU(cudaMemcpyAsync(&v.st->done, &h.done, sizeof(int32_t), cudaMemcpyHostToDevice, s));
        CU(cudaMemcpyAsync(&v.st->k1, &h.k1, 2 * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    }
    if (!ctx->cap_stream) CU(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    CU(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
    cudaError_t e = cudaSuccess;
    for (int q = 0; q < reps && e == cudaSuccess; ++q) {
        if (which == 1) e = launch_ax_cg(ctx->dm, v, ctx->cap_stream);
        else if (which == 2) e = launch_k2(ctx->dm, v, false, ctx->cap_stream);
        else if (which == 3) {     // sem_ax then sem_dssum (config c2)
            e = launch_ax(ctx->dm, v.r, v.w, ctx->cap_stream);
            if (e == cudaSuccess) e = launch_gs(ctx->dm, v.w, 0, nullptr, ctx->cap_stream);
        }
        else e = launch_ax(ctx->dm, v.r, v.w, ctx->cap_stream);
    }
    cudaGraph_t g = nullptr;
    cudaError_t e2 = cudaStreamEndCapture(ctx->cap_stream, &g);
    if (e != cudaSuccess || e2 != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        CU(e != cudaSuccess ? e : e2);
    }
    if (ctx->replay_exec) {     // the previous replay must be finished first
        CU(cudaStreamSynchronize(s));
        cudaGraphExecDestroy(ctx->replay_exec);
        ctx->replay_exec = nullptr;
    }
    e = cudaGraphInstantiate(&ctx->replay_exec, g, 0);
    cudaGraphDestroy(g);
    CU(e);
    CU(cudaGraphLaunch(ctx->replay_exec, s));
    ctx->launches += (which == 3 ? 2 : 1) * int64_t(reps);
    return SEM_OK;
}

extern "C" int sem_cg_phases(sem_ctx *ctx, double *us) {
    CHECK_CTX();
    if (!us) return fail(ctx, SEM_EINVAL, "sem_cg_phases: us is NULL");
    if (!ctx->rcg_last) return fail(ctx, SEM_EINVAL, "sem_cg_phases: the last sem_cg did not run resident");
    uint64_t ns[4];
    CU(cudaMemcpyAsync(ns, ctx->rcg.bar + 16, sizeof ns, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    const double it = ctx->rcg_iters > 0 ? ctx->rcg_iters : 1;
    for (int q = 0; q < 4; ++q) us[q] = 1e-3 * (double)ns[q] / it;
    return SEM_OK;
}

extern "C" int sem_profile(sem_ctx *ctx, int enable) {
    CHECK_CTX();
    if (!ctx->recs.empty()) {
        CU(cudaStreamSynchronize(ctx->stream));
        prof_fold(ctx, -1);
    }
    ctx->prof = enable != 0;
    for (int c = 0; c < kProfClasses; ++c) {
        ctx->prof_ms[c] = 0.0;
        ctx->prof_bytes[c] = 0.0;
        ctx->prof_n[c] = 0;
    }
    return SEM_OK;
}

extern "C" int sem_profile_read(sem_ctx *ctx, int which, double *ms, int64_t *launches,
                                double *bytes) {
    CHECK_CTX();
    if (which < 0 || which >= kProfClasses) return fail(ctx, SEM_EINVAL, "bad kernel class");
    if (!ctx->recs.empty()) {
        CU(cudaStreamSynchronize(ctx->stream));
        prof_fold(ctx, -1);
    }
    if (ms) *ms = ctx->prof_ms[which];
    if (launches) *launches = ctx->prof_n[which];
    if (bytes) *bytes = ctx->prof_bytes[which];
    return SEM_OK;
}

// ---------------------------------------------------------------------------
// errors / version
// ---------------------------------------------------------------------------
extern "C" const char *sem_strerror(int code) {
    switch (code) {
    case SEM_OK: return "SEM_OK";
    case SEM_EINVAL: return "SEM_EINVAL: invalid argument or mesh";
    case SEM_ECUDA: return "SEM_ECUDA: CUDA runtime failure";
    case SEM_ENCCL: return "SEM_ENCCL: NCCL failure";
    case SEM_ENOCONV: return "SEM_ENOCONV: maxit reached before tol";
    case SEM_ESTATE: return "SEM_ESTATE: bad context state";
    default: return "unknown status";
    }
}

extern "C" const char *sem_last_error(const sem_ctx *ctx) {
    if (ctx && !ctx->err.empty()) return ctx->err.c_str();
    return g_err.c_str();
}

extern "C" const char *sem_version(void) { return "libsem 0.1 (sm_100a, fp64)"; }
