// p2p_dev.cuh -- device side of the peer-memory transport (SEM_COMM=p2p,
// sem_comm.cu): window layout, system-scope release / acquire flags, the
// one-warp all-gather.  Shared by the transport's own kernels and by the
// rank folds that fuse their reduction with the all-gather (cg_red_kernel,
// sr_fold_kernel).  Internal.
#pragma once
#include "sem_internal.h"

namespace sem {

#ifndef SEM_P2P_SITES
#define SEM_P2P_SITES
enum { kSiteExchange = 0, kSitePap = 1, kSiteRr = 2, kSiteRz = 3, kSiteSr = 4, kSites = 5 };
#endif

struct P2PHead {
    unsigned long long flags[kSites][kMaxRanks];   // flags[site][q]: last epoch rank q signalled here
    unsigned long long ctr[kSites];                 // this rank's epoch per site
    double scal[kSites][2][2 * kMaxRanks];          // all-gather slots [site][parity][rank * count + c]
};
struct P2PPeers {
    P2PHead *head[kMaxRanks];                       // every rank's window header (own included)
    double *recv[2][kMaxRanks];                     // every rank's exchange receive areas
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// spin until *flag >= e (acquire); false on timeout (error flag raised)
__device__ __forceinline__ bool p2p_wait(const unsigned long long *flag, unsigned long long e,
                                         unsigned long long timeout_ns, unsigned *err) {
    const unsigned long long t0 = global_ns();
    while (ld_acquire_sys(flag) < e) {
        // after a first timeout every later collective fails fast
        if (*reinterpret_cast<volatile unsigned *>(err)) return false;
        if (global_ns() - t0 > timeout_ns) {
            atomicExch(err, 1u);
            return false;
        }
    }
    return true;
}


// everything a fused fold + all-gather kernel needs (device memory, one per
// context, written at setup)
struct P2PDev {
    P2PPeers peers;
    int me, P;
    unsigned long long timeout_ns;
    unsigned *err;
};

// one warp (all 32 lanes call it): epoch of `site` += 1; this rank's `count`
// values at slot_base[me * count ..] into every peer's slots, release a flag
// at every peer, acquire theirs, copy their values into slot_base
__device__ __forceinline__ void p2p_allgather_warp(const P2PDev &d, int site, double *slot_base,
                                                   int count) {
    const int me = d.me, P = d.P;
    P2PHead *mine = d.peers.head[me];
    const unsigned long long e = mine->ctr[site] + 1;
    const int par = (int)(e & 1);
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mine->ctr[site] = e;
    double v[2];
    for (int c = 0; c < count; ++c) v[c] = slot_base[me * count + c];
    for (int q = threadIdx.x & 31; q < P; q += 32) {
        if (q == me) continue;
        for (int c = 0; c < count; ++c) d.peers.head[q]->scal[site][par][me * count + c] = v[c];
    }
    __threadfence_system();
    for (int q = threadIdx.x & 31; q < P; q += 32)
        if (q != me) st_release_sys(&d.peers.head[q]->flags[site][me], e);
    for (int q = threadIdx.x & 31; q < P; q += 32) {
        if (q == me) continue;
        if (!p2p_wait(&mine->flags[site][q], e, d.timeout_ns, d.err)) continue;
        for (int c = 0; c < count; ++c) slot_base[q * count + c] = mine->scal[site][par][q * count + c];
    }
}

}  // namespace sem
