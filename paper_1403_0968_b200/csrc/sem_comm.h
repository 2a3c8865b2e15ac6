// sem_comm.h -- multi-rank plumbing (NCCL over NVLink) for libsem.  Internal.
#pragma once
#include <string>
#include <vector>

#include "../../include/sem.h"
#include "sem_internal.h"

namespace sem {

struct Comm;

// Build the NCCL communicator and the per-peer interface exchange lists.
int comm_setup(Comm *&c, const sem_mesh *mesh, const std::vector<int64_t> &surf_ids,
               const std::vector<int32_t> &surf_group, const std::vector<int32_t> &off,
               const std::vector<int32_t> &idx, int64_t &nglobal, cudaStream_t s,
               std::string &err);
// Q Q^T across ranks (mode as launch_gs).  nlaunch receives the kernel count.
int comm_dssum(Comm *c, const DevMesh &m, double *w, int mode, CgVecs *v,
               cudaStream_t s, int64_t &nlaunch, std::string &err);
// In-place all-gather of one double per rank at slot_base[0..nranks).
int comm_allgather_scalar(Comm *c, double *slot_base, cudaStream_t s, std::string &err);
void comm_free(Comm *c);

}  // namespace sem
