// sem_comm.cu -- multi-rank DSSUM exchange and scalar all-gathers (NCCL over
// NVLink 5 / NVSwitch), SURVEY.md §8(e).  See sem_comm.h for the scheme.
#include <nccl.h>

#include <algorithm>
#include <cstring>

#include "cg_device.cuh"
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
struct Comm {
    ncclComm_t nccl = nullptr;
    int rank = 0, nranks = 1;
    std::vector<int> peer;
    std::vector<int64_t> peer_off;
    int64_t nslot = 0;
    int nif = 0;
    double *sendbuf = nullptr, *recvbuf = nullptr;
    int32_t *send_group = nullptr, *if_group = nullptr, *if_off = nullptr, *if_src = nullptr;
};

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
__global__ void combine_kernel(const __grid_constant__ GsClasses cls, const int32_t *idx,
                               double *w, const int32_t *if_group, const int32_t *if_off,
                               const int32_t *if_src, int nif, const double *recvbuf) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nif) return;
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
    ncclUniqueId id;
    std::memcpy(&id, mesh->nccl_id, sizeof id);
    NC(ncclCommInitRank(&c.nccl, c.nranks, id, c.rank));
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
    if (c.nslot) {
        pack_kernel<<<(int)((c.nslot + 255) / 256), 256, 0, s>>>(m.cls, m.gs_idx, w, c.send_group,
                                                                 c.nslot, c.sendbuf);
        CC(cudaGetLastError());
        ++nlaunch;
    }
    NC(ncclGroupStart());
    for (size_t p = 0; p < c.peer.size(); ++p) {
        const size_t o = (size_t)c.peer_off[p], n = (size_t)(c.peer_off[p + 1] - c.peer_off[p]);
        NC(ncclSend(c.sendbuf + o, n, ncclDouble, c.peer[p], c.nccl, s));
        NC(ncclRecv(c.recvbuf + o, n, ncclDouble, c.peer[p], c.nccl, s));
    }
    NC(ncclGroupEnd());
    if (c.nif) {
        combine_kernel<<<(c.nif + 255) / 256, 256, 0, s>>>(m.cls, m.gs_idx, w, c.if_group, c.if_off,
                                                           c.if_src, c.nif, c.recvbuf);
        CC(cudaGetLastError());
        ++nlaunch;
    }
    return SEM_OK;
}

int comm_allgather_scalar(Comm *cp, double *slot_base, cudaStream_t s, std::string &err) {
    if (!cp) {
        err = "no communicator";
        return SEM_ESTATE;
    }
    NC(ncclAllGather(slot_base + cp->rank, slot_base, 1, ncclDouble, cp->nccl, s));
    return SEM_OK;
}

int comm_allgather(Comm *cp, double *slot_base, int count, cudaStream_t s, std::string &err) {
    if (!cp) {
        err = "no communicator";
        return SEM_ESTATE;
    }
    NC(ncclAllGather(slot_base + size_t(cp->rank) * count, slot_base, count, ncclDouble, cp->nccl, s));
    return SEM_OK;
}

void comm_free(Comm *c) {
    if (!c) return;
    if (c->nccl) ncclCommDestroy(c->nccl);
    cudaFree(c->sendbuf);
    cudaFree(c->recvbuf);
    cudaFree(c->send_group);
    cudaFree(c->if_group);
    cudaFree(c->if_off);
    cudaFree(c->if_src);
    delete c;
}

}  // namespace sem

extern "C" int sem_nccl_id_bytes(void) { return (int)sizeof(ncclUniqueId); }
extern "C" int sem_nccl_get_unique_id(void *id_out) {
    if (!id_out) return SEM_EINVAL;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return SEM_ENCCL;
    memcpy(id_out, &id, sizeof id);
    return SEM_OK;
}
