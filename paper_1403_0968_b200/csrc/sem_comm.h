// sem_comm.h -- multi-rank plumbing for libsem.  Internal.
//
// Elements are partitioned across ranks; global ids are consistent.  A global
// node on a partition interface has local copies on several ranks.  Q Q^T
// over all ranks = (1) each rank sums its own copies (ascending local order),
// (2) the per-rank partial sums are exchanged with every peer sharing the node
// (grouped ncclSend/ncclRecv over NVLink), (3) every rank adds the partials in
// ASCENDING RANK ORDER, so all ranks hold bit-identical values, and writes the
// total into the node's first local copy (the others zeroed), after which the
// ordinary local gather-scatter (or K2) completes the operator.
#pragma once
#include <string>
#include <vector>

#include "../../include/sem.h"
#include "sem_internal.h"

namespace sem {

// Host-side exchange plan of one rank (pure host; uses mesh->allgather).
struct ExchangePlan {
    int rank = 0, nranks = 1;
    std::vector<int> peer;                // peers with a non-empty shared set, ascending
    std::vector<int64_t> peer_off;        // [npeer + 1] offsets into send/recv slots
    std::vector<int64_t> shared_ids;      // [nslot] global ids, ascending per peer
    std::vector<int32_t> send_group;      // [nslot] local group of each slot
    // interface groups: local group, and its sources in ascending rank order
    // (-1 = this rank's own partial, else a recv slot)
    std::vector<int32_t> if_group;
    std::vector<int32_t> if_off;          // [nif + 1]
    std::vector<int32_t> if_src;
    std::vector<int32_t> not_owned;       // interface groups a lower rank also holds:
                                          // counted there, not here, in (r,r)
    int64_t nglobal = 0;                  // distinct global ids over all ranks
};

// surf_ids: this rank's distinct element-surface global ids (ascending) with
// their local group (surf_group); ndistinct: distinct ids on this rank.
int build_exchange_plan(const sem_mesh *mesh, const std::vector<int64_t> &surf_ids,
                        const std::vector<int32_t> &surf_group, int64_t ndistinct,
                        ExchangePlan &ep, std::string &err);

struct Comm;

// NCCL communicator + device copies of the plan.  cudaMalloc's its buffers.
int comm_setup(Comm *&c, const sem_mesh *mesh, const ExchangePlan &ep, const DevMesh &dm,
               cudaStream_t s, std::string &err);
// Cross-rank part of Q Q^T on w (pack, exchange, ordered combine into the first
// copy).  nlaunch receives the kernel count.
int comm_exchange(Comm *c, const DevMesh &m, double *w, cudaStream_t s, int64_t &nlaunch,
                  std::string &err);
// All-gather sites (one epoch counter and slot set each in the peer-memory
// transport): the interface exchange and the CG scalars.
// all-gather sites (as p2p_dev.cuh)
#ifndef SEM_P2P_SITES
#define SEM_P2P_SITES
enum { kSiteExchange = 0, kSitePap = 1, kSiteRr = 2, kSiteRz = 3, kSiteSr = 4, kSites = 5 };
#endif
struct P2PDev;
// `count` (<= 2) doubles per rank, rank-major at slot_base (in place)
int comm_allgather(Comm *c, double *slot_base, int count, int site, cudaStream_t s, std::string &err);
void comm_free(Comm *c);
// false for the loopback transport (its host rendezvous cannot be graph-captured)
bool comm_capturable(const Comm *c);
// true for the peer-memory transport (its collectives spin on the device)
bool comm_device_only(const Comm *c);
// the peer-memory transport's device descriptor (nullptr for other transports):
// rank folds that take it do their all-gather themselves (one kernel)
const P2PDev *comm_p2p_dev(const Comm *c);
// SEM_ENCCL (with a message) if the communicator reported an asynchronous error
int comm_poll(Comm *c, std::string &err);
// abort after a failure (cancels pending NCCL work); wakes loopback peers
void comm_abort(Comm *c);

}  // namespace sem
