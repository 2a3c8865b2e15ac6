// sem_comm.cu -- multi-rank DSSUM exchange and scalar all-gathers (placeholder:
// single-rank build; the NCCL path lands with the multi-GPU milestone).
#include <cstring>

#include "sem_comm.h"

namespace sem {
struct Comm {};
int comm_setup(Comm *&c, const sem_mesh *, const std::vector<int64_t> &, const std::vector<int32_t> &,
               const std::vector<int32_t> &, const std::vector<int32_t> &, int64_t &, cudaStream_t,
               std::string &err) {
    c = nullptr;
    err = "nranks > 1 not built yet";
    return SEM_EINVAL;
}
int comm_dssum(Comm *, const DevMesh &, double *, int, CgVecs *, cudaStream_t, int64_t &,
               std::string &err) {
    err = "no communicator";
    return SEM_ESTATE;
}
int comm_allgather_scalar(Comm *, double *, cudaStream_t, std::string &err) {
    err = "no communicator";
    return SEM_ESTATE;
}
void comm_free(Comm *c) { delete c; }
}  // namespace sem

#include <nccl.h>
extern "C" int sem_nccl_id_bytes(void) { return (int)sizeof(ncclUniqueId); }
extern "C" int sem_nccl_get_unique_id(void *id_out) {
    if (!id_out) return SEM_EINVAL;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return SEM_ENCCL;
    memcpy(id_out, &id, sizeof id);
    return SEM_OK;
}
