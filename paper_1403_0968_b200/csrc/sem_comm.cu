// sem_comm.cu -- multi-rank DSSUM exchange and scalar all-gathers (NCCL over
// NVLink 5 / NVSwitch), SURVEY.md §8(e).  See sem_comm.h for the scheme.
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>

#include "cg_device.cuh"
#include "p2p_dev.cuh"
#include "sem_comm.h"

namespace sem {

// ---------------------------------------------------------------------------
// host: exchange plan
// ---------------------------------------------------------------------------
int build_exchange_plan(const sem_mesh *mesh, const std::vector<int64_t> &surf_ids,
                        const std::vector<int32_t> &surf_group, int64_t ndistinct,
                        ExchangePlan &ep, std::string &err) {
    const int P = mesh->nranks, me = mesh->rank;
    ep = ExchangePlan{};
    ep.rank = me;
    ep.nranks = P;
    if (P == 1) {
        ep.peer_off.push_back(0);
        ep.if_off.push_back(0);
        ep.nglobal = ndistinct;
        return SEM_OK;
    }
    if (!mesh->allgather) {
        err = "nranks > 1 needs an allgather callback";
        return SEM_EINVAL;
    }
    auto gather = [&](const void *send, size_t bytes, void *recv) -> bool {
        return mesh->allgather(mesh->allgather_user, send, bytes, recv) == 0;
    };
    // counts and distinct-id totals
    int64_t mine[2] = {(int64_t)surf_ids.size(), ndistinct};
    std::vector<int64_t> cnts(2 * P);
    if (!gather(mine, sizeof mine, cnts.data())) {
        err = "setup all-gather (counts) failed";
        return SEM_ENCCL;
    }
    int64_t maxc = 1;
    for (int q = 0; q < P; ++q) maxc = std::max(maxc, cnts[2 * q]);
    std::vector<int64_t> pad(maxc, -1);
    std::copy(surf_ids.begin(), surf_ids.end(), pad.begin());
    std::vector<int64_t> ids((size_t)P * maxc);
    if (!gather(pad.data(), sizeof(int64_t) * maxc, ids.data())) {
        err = "setup all-gather (surface ids) failed";
        return SEM_ENCCL;
    }
    // per peer: ids shared with it (both lists ascending -> same order on both)
    std::vector<std::vector<std::pair<int, int64_t>>> src_of(surf_ids.size());  // (rank, slot)
    ep.peer_off.push_back(0);
    for (int q = 0; q < P; ++q) {
        if (q == me) continue;
        const int64_t *o = ids.data() + (size_t)q * maxc;
        const int64_t no = cnts[2 * q];
        size_t a = 0;
        int64_t b = 0;
        const int64_t first_slot = (int64_t)ep.shared_ids.size();
        while (a < surf_ids.size() && b < no) {
            if (surf_ids[a] < o[b]) ++a;
            else if (surf_ids[a] > o[b]) ++b;
            else {
                const int64_t slot = (int64_t)ep.shared_ids.size();
                ep.shared_ids.push_back(surf_ids[a]);
                ep.send_group.push_back(surf_group[a]);
                src_of[a].push_back({q, slot});
                ++a;
                ++b;
            }
        }
        if ((int64_t)ep.shared_ids.size() > first_slot) {
            ep.peer.push_back(q);
            ep.peer_off.push_back((int64_t)ep.shared_ids.size());
        }
    }
    // interface groups with their sources in ascending rank order
    ep.if_off.push_back(0);
    for (size_t a = 0; a < surf_ids.size(); ++a) {
        if (src_of[a].empty()) continue;
        auto srcs = src_of[a];
        srcs.push_back({me, -1});
        std::sort(srcs.begin(), srcs.end());
        if (srcs.front().first != me) ep.not_owned.push_back(surf_group[a]);
        ep.if_group.push_back(surf_group[a]);
        for (auto &s : srcs) ep.if_src.push_back((int32_t)s.second);
        ep.if_off.push_back((int32_t)ep.if_src.size());
    }
    // distinct ids over all ranks: sum of per-rank counts minus the repeats of
    // shared surface ids
    int64_t tot = 0;
    for (int q = 0; q < P; ++q) tot += cnts[2 * q + 1];
    std::vector<int64_t> all;
    all.reserve((size_t)P * maxc);
    for (int q = 0; q < P; ++q)
        for (int64_t t = 0; t < cnts[2 * q]; ++t) all.push_back(ids[(size_t)q * maxc + t]);
    std::sort(all.begin(), all.end());
    for (size_t t = 1; t < all.size(); ++t)
        if (all[t] == all[t - 1]) --tot;
    ep.nglobal = tot;
    return SEM_OK;
}

// ---------------------------------------------------------------------------
// device
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// loopback transport (TEST ONLY): P ranks as P contexts in ONE process on ONE
// GPU, one host thread per rank.  Every rank's exchange and all-gather become
// device-to-device copies between the ranks' own buffers, ordered by CUDA
// events and two host rendezvous per collective:
//   1. each rank enqueues its producer (pack / reduction kernel), records
//      ev_ready[rank] on its stream and posts its buffer pointer;   barrier
//   2. each rank makes its stream wait for ev_ready of every peer, copies the
//      peers' values it needs into its own receive buffer / slots, records
//      ev_done[rank];                                                barrier
//   3. each rank's stream waits for ev_done of every peer (the peers have read
//      its send buffer / slot before it is overwritten).
// The pack / combine kernels, the plan, the rank-ordered sums and every
// multi-rank branch of the CG kernels run exactly as with NCCL; only the
// transfer differs.  Selected by an id from sem_loopback_unique_id() in
// sem_mesh.nccl_id.  CUDA-graph capture is off for loopback contexts (the
// host rendezvous cannot be captured).
// ---------------------------------------------------------------------------
static const char kLoopMagic[16] = {'S', 'E', 'M', '-', 'L', 'O', 'O', 'P', 'B', 'A', 'C', 'K', 0, 1, 2, 3};

struct LoopWorld {
    int P = 0;
    int refs = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    int64_t gen = 0;
    bool failed = false;
    std::vector<cudaEvent_t> ev_ready, ev_done;
    std::vector<double *> post;          // per rank: buffer posted for the current collective
    std::vector<double *> sendbuf;       // per rank: its exchange send buffer
    std::vector<std::vector<int>> peer;  // per rank: its peers (ascending)
    std::vector<std::vector<int64_t>> peer_off;
    std::vector<int> joined;
};

static std::mutex g_loop_mu;
static std::map<std::string, LoopWorld *> g_loop;

static int loop_timeout_ms() {
    const char *e = getenv("SEM_LOOPBACK_TIMEOUT_MS");
    return e ? atoi(e) : 120000;
}

// Host rendezvous of all P ranks (false: a peer failed or timed out).
static bool loop_barrier(LoopWorld &w) {
    std::unique_lock<std::mutex> lk(w.mu);
    if (w.failed) return false;
    const int64_t g = w.gen;
    if (++w.arrived == w.P) {
        w.arrived = 0;
        ++w.gen;
        w.cv.notify_all();
        return true;
    }
    const bool ok = w.cv.wait_for(lk, std::chrono::milliseconds(loop_timeout_ms()),
                                  [&] { return w.gen != g || w.failed; });
    if (!ok || w.failed) {
        w.failed = true;
        w.cv.notify_all();
        return false;
    }
    return true;
}

// ---------------------------------------------------------------------------
// peer-memory transport (SEM_COMM=p2p): every rank owns a window -- a header
// of per-site epoch counters, arrival flags and all-gather slots, then two
// receive areas for the interface exchange -- that its peers write into
// directly (device stores to peer memory: the same device for the one-GPU
// loopback world, CUDA IPC + NVLink peer access across processes).  A
// collective is device work only, so it is captured into the CUDA graphs:
//   exchange:   p2p_pack_kernel stores each partial sum straight into the
//               peer's receive area (parity of the next epoch), then
//               p2p_sync_kernel (one warp) bumps the epoch, releases a flag
//               at every neighbour and spins (acquire) until every
//               neighbour's flag for this epoch has arrived; combine_kernel
//               reads the local receive area of that parity;
//   all-gather: p2p_allgather_kernel (one warp) stores this rank's values
//               into every peer's slots, releases the flags, acquires the
//               peers' and copies their values out (the one-shot,
//               fixed-order reduction of SURVEY.md §8(e) step 3).
// Two parities suffice: a rank can only rewrite a peer's parity-p area at
// epoch e+2 after that peer signalled e+1, i.e. after it consumed epoch e.
// Spins time out (SEM_P2P_TIMEOUT_MS) and raise a host-mapped error flag,
// after which every later spin of the context fails at once.
// ---------------------------------------------------------------------------
struct Comm {
    ncclComm_t nccl = nullptr;
    // peer-memory transport (SEM_COMM=p2p)
    bool p2p = false;
    char *win = nullptr;                 // own window (cudaMalloc: IPC-exportable)
    P2PPeers peers{};
    std::vector<void *> ipc_opened;      // peers' windows opened through CUDA IPC
    int32_t *slot_rank = nullptr;        // per send slot: destination rank
    int64_t *slot_off = nullptr;         // ... and offset in its receive area
    int32_t *plist = nullptr;            // neighbour ranks (device)
    unsigned *err_h = nullptr, *err_d = nullptr;   // host-mapped timeout flag
    P2PDev *dev = nullptr;               // device copy of peers / rank / timeout (fused folds)
    unsigned long long timeout_ns = 0;
    LoopWorld *lw = nullptr;             // loopback transport (tests) instead of NCCL
    std::string lw_key;
    int rank = 0, nranks = 1;
    std::vector<int> peer;
    std::vector<int64_t> peer_off;
    std::vector<int64_t> peer_src_off;   // loopback: offset of my slots in each peer's send buffer
    int64_t nslot = 0;
    int nif = 0;
    double *sendbuf = nullptr, *recvbuf = nullptr;
    int32_t *send_group = nullptr, *if_group = nullptr, *if_off = nullptr, *if_src = nullptr;
};

// the host-rendezvous loopback transport cannot be captured; the peer-memory
// transport (device work only) and NCCL can
bool comm_capturable(const Comm *c) { return c && (!c->lw || c->p2p); }
bool comm_device_only(const Comm *c) { return c && c->p2p; }
const P2PDev *comm_p2p_dev(const Comm *c) { return (c && c->p2p) ? c->dev : nullptr; }

__device__ __forceinline__ void group_loc(const GsClasses &cls, int g, int &m, int &cnt, int &q,
                                          int &off) {
    int c = 0;
    while (c + 1 < cls.n && g >= cls.start[c + 1]) ++c;
    m = cls.m[c];
    cnt = cls.start[c + 1] - cls.start[c];
    q = g - cls.start[c];
    off = cls.idxoff[c];
}

// sum of the local copies of group g, ascending local order
__device__ __forceinline__ double group_local_sum(const GsClasses &cls, const int32_t *idx,
                                                  const double *w, int g) {
    int m, cnt, q, off;
    group_loc(cls, g, m, cnt, q, off);
    const int32_t *ix = idx + off;
    double s = w[__ldg(ix + q)];
    for (int t = 1; t < m; ++t) s += w[__ldg(ix + t * cnt + q)];
    return s;
}

__global__ void pack_kernel(const __grid_constant__ GsClasses cls, const int32_t *idx,
                            const double *w, const int32_t *send_group, int64_t nslot,
                            double *sendbuf) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < nslot) sendbuf[t] = group_local_sum(cls, idx, w, send_group[t]);
}

// total = partials of all sharing ranks in ascending rank order, into the
// group's first copy; the other copies zeroed
// (peer-memory transport: recvbuf1 != nullptr, the area of parity ctr & 1)
__global__ void combine_kernel(const __grid_constant__ GsClasses cls, const int32_t *idx,
                               double *w, const int32_t *if_group, const int32_t *if_off,
                               const int32_t *if_src, int nif, const double *recvbuf,
                               const double *recvbuf1, const unsigned long long *ctr) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nif) return;
    if (recvbuf1 && (*ctr & 1)) recvbuf = recvbuf1;
    const int g = if_group[i];
    const double local = group_local_sum(cls, idx, w, g);
    double tot = 0.0;
    for (int t = if_off[i]; t < if_off[i + 1]; ++t) {
        const int sslot = if_src[t];
        const double v = (sslot < 0) ? local : recvbuf[sslot];
        tot = (t == if_off[i]) ? v : tot + v;
    }
    int m, cnt, q, off;
    group_loc(cls, g, m, cnt, q, off);
    const int32_t *ix = idx + off;
    w[__ldg(ix + q)] = tot;
    for (int t = 1; t < m; ++t) w[__ldg(ix + t * cnt + q)] = 0.0;
}

// exchange, peer-memory transport: partial sums straight into the peers'
// receive areas (parity of the coming epoch)
__global__ void p2p_pack_kernel(const __grid_constant__ GsClasses cls, const int32_t *idx,
                                const double *w, const int32_t *send_group, int64_t nslot,
                                const int32_t *slot_rank, const int64_t *slot_off,
                                const __grid_constant__ P2PPeers peers, int me) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < nslot) {
        const int par = (int)((peers.head[me]->ctr[kSiteExchange] + 1) & 1);
        peers.recv[par][slot_rank[t]][slot_off[t]] = group_local_sum(cls, idx, w, send_group[t]);
    }
    __threadfence_system();     // the stores reach the peers before the flag does
}

// one warp: epoch of `site` += 1, flag at every rank of plist, wait for theirs
__global__ void p2p_sync_kernel(const __grid_constant__ P2PPeers peers, int me, int site,
                                const int32_t *plist, int np, unsigned long long timeout_ns,
                                unsigned *err) {
    P2PHead *mine = peers.head[me];
    const unsigned long long e = mine->ctr[site] + 1;
    __syncwarp();
    if (threadIdx.x == 0) mine->ctr[site] = e;
    __threadfence_system();
    for (int i = threadIdx.x; i < np; i += 32) st_release_sys(&peers.head[plist[i]]->flags[site][me], e);
    for (int i = threadIdx.x; i < np; i += 32) p2p_wait(&mine->flags[site][plist[i]], e, timeout_ns, err);
}

// one warp: the all-gather of `site` (p2p_dev.cuh)
__global__ void p2p_allgather_kernel(const P2PDev *d, int site, double *slot_base, int count) {
    p2p_allgather_warp(*d, site, slot_base, count);
}

#define NC(call)                                                                    \
    do {                                                                            \
        ncclResult_t r_ = (call);                                                   \
        if (r_ != ncclSuccess) {                                                    \
            err = std::string(#call) + ": " + ncclGetErrorString(r_);               \
            return SEM_ENCCL;                                                       \
        }                                                                           \
    } while (0)
#define CC(call)                                                                    \
    do {                                                                            \
        cudaError_t e_ = (call);                                                    \
        if (e_ != cudaSuccess) {                                                    \
            err = std::string(#call) + ": " + cudaGetErrorString(e_);               \
            return SEM_ECUDA;                                                       \
        }                                                                           \
    } while (0)

// Register this rank in the loopback world named by the id (created by the
// first rank to arrive), then learn where the peers keep the slots this rank
// receives.
static int loop_join(Comm &c, const sem_mesh *mesh, std::string &err) {
    c.lw_key.assign(static_cast<const char *>(mesh->nccl_id), 128);
    LoopWorld *w;
    {
        std::lock_guard<std::mutex> g(g_loop_mu);
        auto it = g_loop.find(c.lw_key);
        if (it == g_loop.end()) {
            w = new LoopWorld;
            w->P = c.nranks;
            w->ev_ready.assign(c.nranks, nullptr);
            w->ev_done.assign(c.nranks, nullptr);
            w->post.assign(c.nranks, nullptr);
            w->sendbuf.assign(c.nranks, nullptr);
            w->peer.assign(c.nranks, {});
            w->peer_off.assign(c.nranks, {});
            w->joined.assign(c.nranks, 0);
            g_loop[c.lw_key] = w;
        } else {
            w = it->second;
        }
        if (w->P != c.nranks || w->joined[c.rank]) {
            err = "loopback: nranks mismatch or rank joined twice";
            return SEM_EINVAL;
        }
        w->joined[c.rank] = 1;
        ++w->refs;
    }
    c.lw = w;
    CC(cudaEventCreateWithFlags(&w->ev_ready[c.rank], cudaEventDisableTiming));
    CC(cudaEventCreateWithFlags(&w->ev_done[c.rank], cudaEventDisableTiming));
    w->sendbuf[c.rank] = c.sendbuf;
    w->peer[c.rank] = c.peer;
    w->peer_off[c.rank] = c.peer_off;
    if (!loop_barrier(*w)) {
        err = "loopback: setup rendezvous failed (a peer failed or timed out)";
        return SEM_ENCCL;
    }
    c.peer_src_off.resize(c.peer.size());
    for (size_t p = 0; p < c.peer.size(); ++p) {
        const int q = c.peer[p];
        const auto &qp = w->peer[q];
        const auto at = std::find(qp.begin(), qp.end(), c.rank);
        if (at == qp.end()) {
            err = "loopback: asymmetric exchange plan";
            return SEM_EINVAL;
        }
        const size_t qi = size_t(at - qp.begin());
        if (w->peer_off[q][qi + 1] - w->peer_off[q][qi] != c.peer_off[p + 1] - c.peer_off[p]) {
            err = "loopback: shared-set sizes differ between peers";
            return SEM_EINVAL;
        }
        c.peer_src_off[p] = w->peer_off[q][qi];
    }
    if (!loop_barrier(*w)) {
        err = "loopback: setup rendezvous failed (a peer failed or timed out)";
        return SEM_ENCCL;
    }
    return SEM_OK;
}

// One loopback collective (steps 1-3 above).  copy(s) enqueues this rank's
// reads of the peers' posted buffers.
template <typename F>
static int loop_collective(Comm &c, double *mine, cudaStream_t s, std::string &err, F copy) {
    LoopWorld &w = *c.lw;
    CC(cudaEventRecord(w.ev_ready[c.rank], s));
    w.post[c.rank] = mine;
    if (!loop_barrier(w)) {
        err = "loopback: a peer failed or timed out";
        return SEM_ENCCL;
    }
    int rc = copy();
    if (rc) return rc;
    CC(cudaEventRecord(w.ev_done[c.rank], s));
    if (!loop_barrier(w)) {
        err = "loopback: a peer failed or timed out";
        return SEM_ENCCL;
    }
    for (int q = 0; q < c.nranks; ++q)
        if (q != c.rank) CC(cudaStreamWaitEvent(s, w.ev_done[q], 0));
    return SEM_OK;
}

// Peer-memory transport setup (collective over mesh->allgather): allocate and
// zero this rank's window, publish its address (the raw pointer inside one
// process -- the loopback world --, a CUDA IPC handle across processes), the
// size of its receive area and where in it each peer's slots start; open the
// peers' windows; per send slot, the destination rank and offset.
struct P2PInfo {
    unsigned long long ptr;
    long long nslot;
    cudaIpcMemHandle_t h;
    long long off_to[kMaxRanks];    // offset of the slots shared with rank q (-1: none)
    long long cnt_to[kMaxRanks];
};

static int p2p_join(Comm &c, const sem_mesh *mesh, bool same_process, std::string &err) {
    const int P = c.nranks, me = c.rank;
    const size_t ns = (size_t)std::max<int64_t>(c.nslot, 1);
    const size_t bytes = sizeof(P2PHead) + 2 * ns * sizeof(double);
    CC(cudaMalloc(&c.win, bytes));
    CC(cudaMemset(c.win, 0, bytes));
    CC(cudaDeviceSynchronize());
    P2PInfo mine{};
    mine.ptr = (unsigned long long)(uintptr_t)c.win;
    mine.nslot = (long long)ns;
    if (!same_process) CC(cudaIpcGetMemHandle(&mine.h, c.win));
    for (int q = 0; q < kMaxRanks; ++q) mine.off_to[q] = mine.cnt_to[q] = -1;
    for (size_t p = 0; p < c.peer.size(); ++p) {
        mine.off_to[c.peer[p]] = c.peer_off[p];
        mine.cnt_to[c.peer[p]] = c.peer_off[p + 1] - c.peer_off[p];
    }
    std::vector<P2PInfo> all(P);
    if (!mesh->allgather || mesh->allgather(mesh->allgather_user, &mine, sizeof mine, all.data()) != 0) {
        err = "p2p: setup all-gather failed";
        return SEM_ENCCL;
    }
    for (int q = 0; q < P; ++q) {
        char *base = nullptr;
        if (q == me) {
            base = c.win;
        } else if (same_process) {
            base = reinterpret_cast<char *>((uintptr_t)all[q].ptr);
        } else {
            void *ptr = nullptr;
            CC(cudaIpcOpenMemHandle(&ptr, all[q].h, cudaIpcMemLazyEnablePeerAccess));
            c.ipc_opened.push_back(ptr);
            base = static_cast<char *>(ptr);
        }
        c.peers.head[q] = reinterpret_cast<P2PHead *>(base);
        double *r0 = reinterpret_cast<double *>(base + sizeof(P2PHead));
        c.peers.recv[0][q] = r0;
        c.peers.recv[1][q] = r0 + all[q].nslot;
    }
    // destinations of my send slots
    std::vector<int32_t> srank((size_t)ns, 0);
    std::vector<int64_t> soff((size_t)ns, 0);
    for (size_t p = 0; p < c.peer.size(); ++p) {
        const int q = c.peer[p];
        const long long n = c.peer_off[p + 1] - c.peer_off[p];
        if (all[q].off_to[me] < 0 || all[q].cnt_to[me] != n) {
            err = "p2p: asymmetric exchange plan";
            return SEM_EINVAL;
        }
        for (long long t = 0; t < n; ++t) {
            srank[(size_t)(c.peer_off[p] + t)] = q;
            soff[(size_t)(c.peer_off[p] + t)] = all[q].off_to[me] + t;
        }
    }
    CC(cudaMalloc(&c.slot_rank, sizeof(int32_t) * ns));
    CC(cudaMalloc(&c.slot_off, sizeof(int64_t) * ns));
    CC(cudaMalloc(&c.plist, sizeof(int32_t) * std::max<size_t>(c.peer.size(), 1)));
    CC(cudaMemcpy(c.slot_rank, srank.data(), sizeof(int32_t) * ns, cudaMemcpyHostToDevice));
    CC(cudaMemcpy(c.slot_off, soff.data(), sizeof(int64_t) * ns, cudaMemcpyHostToDevice));
    if (!c.peer.empty())
        CC(cudaMemcpy(c.plist, c.peer.data(), sizeof(int32_t) * c.peer.size(), cudaMemcpyHostToDevice));
    CC(cudaHostAlloc(&c.err_h, sizeof(unsigned), cudaHostAllocMapped));
    *c.err_h = 0;
    CC(cudaHostGetDevicePointer(&c.err_d, c.err_h, 0));
    const char *to = getenv("SEM_P2P_TIMEOUT_MS");
    c.timeout_ns = (unsigned long long)(to ? atoll(to) : 20000) * 1000000ull;
    {
        P2PDev hd{};
        hd.peers = c.peers;
        hd.me = me;
        hd.P = P;
        hd.timeout_ns = c.timeout_ns;
        hd.err = c.err_d;
        CC(cudaMalloc(&c.dev, sizeof(P2PDev)));
        CC(cudaMemcpy(c.dev, &hd, sizeof hd, cudaMemcpyHostToDevice));
    }
    // every rank's window is zeroed before anyone can signal into it
    int ok = 1, oks[kMaxRanks];
    if (mesh->allgather(mesh->allgather_user, &ok, sizeof ok, oks) != 0) {
        err = "p2p: setup all-gather failed";
        return SEM_ENCCL;
    }
    return SEM_OK;
}

int comm_setup(Comm *&cp, const sem_mesh *mesh, const ExchangePlan &ep, const DevMesh &,
               cudaStream_t s, std::string &err) {
    cp = new Comm;
    Comm &c = *cp;
    c.rank = mesh->rank;
    c.nranks = mesh->nranks;
    c.peer = ep.peer;
    c.peer_off = ep.peer_off;
    c.nslot = (int64_t)ep.shared_ids.size();
    c.nif = (int)ep.if_group.size();
    const bool loop = std::memcmp(mesh->nccl_id, kLoopMagic, sizeof kLoopMagic) == 0;
    {
        const char *cm = getenv("SEM_COMM");
        c.p2p = cm && strcmp(cm, "p2p") == 0;
    }
    if (!loop && !c.p2p) {
        ncclUniqueId id;
        std::memcpy(&id, mesh->nccl_id, sizeof id);
        NC(ncclCommInitRank(&c.nccl, c.nranks, id, c.rank));
    }
    const size_t ns = std::max<int64_t>(c.nslot, 1);
    CC(cudaMalloc(&c.sendbuf, sizeof(double) * ns));
    CC(cudaMalloc(&c.recvbuf, sizeof(double) * ns));
    CC(cudaMalloc(&c.send_group, sizeof(int32_t) * ns));
    CC(cudaMalloc(&c.if_group, sizeof(int32_t) * std::max(c.nif, 1)));
    CC(cudaMalloc(&c.if_off, sizeof(int32_t) * (c.nif + 1)));
    CC(cudaMalloc(&c.if_src, sizeof(int32_t) * std::max<size_t>(ep.if_src.size(), 1)));
    if (c.nslot)
        CC(cudaMemcpyAsync(c.send_group, ep.send_group.data(), sizeof(int32_t) * c.nslot,
                           cudaMemcpyHostToDevice, s));
    if (c.nif) {
        CC(cudaMemcpyAsync(c.if_group, ep.if_group.data(), sizeof(int32_t) * c.nif,
                           cudaMemcpyHostToDevice, s));
        CC(cudaMemcpyAsync(c.if_src, ep.if_src.data(), sizeof(int32_t) * ep.if_src.size(),
                           cudaMemcpyHostToDevice, s));
    }
    CC(cudaMemcpyAsync(c.if_off, ep.if_off.data(), sizeof(int32_t) * (c.nif + 1),
                       cudaMemcpyHostToDevice, s));
    CC(cudaStreamSynchronize(s));
    if (c.p2p) return p2p_join(c, mesh, loop, err);
    if (loop) return loop_join(c, mesh, err);
    return SEM_OK;
}

int comm_exchange(Comm *cp, const DevMesh &m, double *w, cudaStream_t s, int64_t &nlaunch,
                  std::string &err) {
    nlaunch = 0;
    if (!cp) {
        err = "no communicator";
        return SEM_ESTATE;
    }
    Comm &c = *cp;
    if (c.p2p) {
        if (c.nslot) {
            p2p_pack_kernel<<<(int)((c.nslot + 255) / 256), 256, 0, s>>>(
                m.cls, m.gs_idx, w, c.send_group, c.nslot, c.slot_rank, c.slot_off, c.peers, c.rank);
            CC(cudaGetLastError());
            ++nlaunch;
        }
        p2p_sync_kernel<<<1, 32, 0, s>>>(c.peers, c.rank, kSiteExchange, c.plist, (int)c.peer.size(),
                                         c.timeout_ns, c.err_d);
        CC(cudaGetLastError());
        ++nlaunch;
        if (c.nif) {
            combine_kernel<<<(c.nif + 255) / 256, 256, 0, s>>>(
                m.cls, m.gs_idx, w, c.if_group, c.if_off, c.if_src, c.nif, c.peers.recv[0][c.rank],
                c.peers.recv[1][c.rank], &c.peers.head[c.rank]->ctr[kSiteExchange]);
            CC(cudaGetLastError());
            ++nlaunch;
        }
        return SEM_OK;
    }
    if (c.nslot) {
        pack_kernel<<<(int)((c.nslot + 255) / 256), 256, 0, s>>>(m.cls, m.gs_idx, w, c.send_group,
                                                                 c.nslot, c.sendbuf);
        CC(cudaGetLastError());
        ++nlaunch;
    }
    if (c.lw) {
        int rc = loop_collective(c, c.sendbuf, s, err, [&]() -> int {
            for (size_t p = 0; p < c.peer.size(); ++p) {
                const int q = c.peer[p];
                const size_t n = (size_t)(c.peer_off[p + 1] - c.peer_off[p]);
                CC(cudaStreamWaitEvent(s, c.lw->ev_ready[q], 0));
                CC(cudaMemcpyAsync(c.recvbuf + c.peer_off[p], c.lw->sendbuf[q] + c.peer_src_off[p],
                                   sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
            }
            return SEM_OK;
        });
        if (rc) return rc;
    } else {
        NC(ncclGroupStart());
        for (size_t p = 0; p < c.peer.size(); ++p) {
            const size_t o = (size_t)c.peer_off[p], n = (size_t)(c.peer_off[p + 1] - c.peer_off[p]);
            NC(ncclSend(c.sendbuf + o, n, ncclDouble, c.peer[p], c.nccl, s));
            NC(ncclRecv(c.recvbuf + o, n, ncclDouble, c.peer[p], c.nccl, s));
        }
        NC(ncclGroupEnd());
    }
    if (c.nif) {
        combine_kernel<<<(c.nif + 255) / 256, 256, 0, s>>>(m.cls, m.gs_idx, w, c.if_group, c.if_off,
                                                           c.if_src, c.nif, c.recvbuf, nullptr,
                                                           nullptr);
        CC(cudaGetLastError());
        ++nlaunch;
    }
    return SEM_OK;
}

int comm_allgather(Comm *cp, double *slot_base, int count, int site, cudaStream_t s,
                   std::string &err) {
    if (!cp) {
        err = "no communicator";
        return SEM_ESTATE;
    }
    Comm &c = *cp;
    if (count < 1 || count > 2 || site < 0 || site >= kSites) {
        err = "comm_allgather: bad count / site";
        return SEM_EINVAL;
    }
    if (c.p2p) {
        p2p_allgather_kernel<<<1, 32, 0, s>>>(c.dev, site, slot_base, count);
        CC(cudaGetLastError());
        return SEM_OK;
    }
    if (c.lw) {
        return loop_collective(c, slot_base, s, err, [&]() -> int {
            for (int q = 0; q < c.nranks; ++q) {
                if (q == c.rank) continue;
                CC(cudaStreamWaitEvent(s, c.lw->ev_ready[q], 0));
                CC(cudaMemcpyAsync(slot_base + size_t(q) * count, c.lw->post[q] + size_t(q) * count,
                                   sizeof(double) * count, cudaMemcpyDeviceToDevice, s));
            }
            return SEM_OK;
        });
    }
    NC(ncclAllGather(slot_base + size_t(c.rank) * count, slot_base, count, ncclDouble, c.nccl, s));
    return SEM_OK;
}

// Asynchronous NCCL failure of a peer / the network: polled by
// the CG drivers while they wait for the device.
int comm_poll(Comm *cp, std::string &err) {
    if (cp && cp->p2p) {
        if (cp->err_h && *reinterpret_cast<volatile unsigned *>(cp->err_h)) {
            err = "peer-memory transport: a peer did not arrive within SEM_P2P_TIMEOUT_MS";
            return SEM_ENCCL;
        }
        return SEM_OK;
    }
    if (!cp || cp->lw || !cp->nccl) return SEM_OK;
    ncclResult_t ar = ncclSuccess;
    ncclResult_t r = ncclCommGetAsyncError(cp->nccl, &ar);
    if (r != ncclSuccess || (ar != ncclSuccess && ar != ncclInProgress)) {
        err = std::string("NCCL asynchronous error: ") + ncclGetErrorString(r != ncclSuccess ? r : ar);
        return SEM_ENCCL;
    }
    return SEM_OK;
}

// Abort the communicator after a failure (pending NCCL work is cancelled so
// the stream can drain); the context is unusable afterwards.
void comm_abort(Comm *cp) {
    if (!cp) return;
    if (cp->nccl) {
        ncclCommAbort(cp->nccl);
        cp->nccl = nullptr;
    }
    if (cp->lw) {
        std::lock_guard<std::mutex> g(cp->lw->mu);
        cp->lw->failed = true;
        cp->lw->cv.notify_all();
    }
}

void comm_free(Comm *c) {
    if (!c) return;
    if (c->nccl) ncclCommDestroy(c->nccl);
    if (c->p2p) {
        cudaDeviceSynchronize();     // no peer kernel may still target a window being freed
        for (void *ptr : c->ipc_opened) cudaIpcCloseMemHandle(ptr);
        cudaFree(c->win);
        cudaFree(c->slot_rank);
        cudaFree(c->slot_off);
        cudaFree(c->plist);
        cudaFree(c->dev);
        if (c->err_h) cudaFreeHost(c->err_h);
    }
    if (c->lw) {
        // the events belong to the world: a peer still leaving its last
        // collective may wait on them after this rank is gone
        LoopWorld *w = c->lw;
        std::lock_guard<std::mutex> g(g_loop_mu);
        if (--w->refs == 0) {
            for (auto e : w->ev_ready)
                if (e) cudaEventDestroy(e);
            for (auto e : w->ev_done)
                if (e) cudaEventDestroy(e);
            g_loop.erase(c->lw_key);
            delete w;
        }
    }
    cudaFree(c->sendbuf);
    cudaFree(c->recvbuf);
    cudaFree(c->send_group);
    cudaFree(c->if_group);
    cudaFree(c->if_off);
    cudaFree(c->if_src);
    delete c;
}

}  // namespace sem

extern "C" int sem_loopback_unique_id(void *id_out) {
    if (!id_out) return SEM_EINVAL;
    static std::mutex mu;
    static uint64_t counter = 0;
    uint64_t serial;
    {
        std::lock_guard<std::mutex> g(mu);
        serial = ++counter;
    }
    unsigned char id[128] = {0};
    std::memcpy(id, sem::kLoopMagic, sizeof sem::kLoopMagic);
    const uint64_t t = (uint64_t)std::chrono::steady_clock::now().time_since_epoch().count();
    std::memcpy(id + 16, &serial, sizeof serial);
    std::memcpy(id + 24, &t, sizeof t);
    std::memcpy(id_out, id, sizeof id);
    return SEM_OK;
}

extern "C" int sem_nccl_id_bytes(void) { return (int)sizeof(ncclUniqueId); }
extern "C" int sem_nccl_get_unique_id(void *id_out) {
    if (!id_out) return SEM_EINVAL;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return SEM_ENCCL;
    memcpy(id_out, &id, sizeof id);
    return SEM_OK;
}
