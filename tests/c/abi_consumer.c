/* A plain C99 consumer of the C ABI (include/sem.h, include/fd.h): compiled
 * with gcc -std=c99 -pedantic -Werror against the headers and linked against
 * libsem.so, so the headers are valid C (no C++ leaks) and every declared entry
 * point resolves.  Runs the host-only calls (no GPU needed); with argv[1] ==
 * "gpu" it also builds a context on device 0 and checks A_L 1 = 0.
 * Test infrastructure (tests/test_abi.py builds and runs it). */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "fd.h"
#include "sem.h"

/* every declared function, by address: a missing export fails the link */
typedef void (*fnp)(void);
static const fnp exported[] = {
    (fnp)sem_version, (fnp)sem_gll, (fnp)sem_workspace_bytes, (fnp)sem_setup,
    (fnp)sem_sizes, (fnp)sem_ax, (fnp)sem_dssum, (fnp)sem_mask, (fnp)sem_mass,
    (fnp)sem_cg, (fnp)sem_pcg, (fnp)sem_cg_sr, (fnp)sem_diag,
    (fnp)sem_nccl_id_bytes, (fnp)sem_nccl_get_unique_id, (fnp)sem_loopback_unique_id,
    (fnp)sem_profile, (fnp)sem_kernel_replay, (fnp)sem_profile_read,
    (fnp)sem_exchange_plan, (fnp)sem_status, (fnp)sem_launch_count, (fnp)sem_free, (fnp)sem_strerror,
    (fnp)sem_last_error, (fnp)fd_weights, (fnp)fd2d_step, (fnp)fd2d_run,
    (fnp)fd2d_run_ex};

#define CHECK(c)                                                   \
    do {                                                           \
        if (!(c)) {                                                \
            fprintf(stderr, "FAILED %s at line %d\n", #c, __LINE__); \
            return 1;                                              \
        }                                                          \
    } while (0)

int main(int argc, char **argv) {
    size_t i;
    double xi[SEM_NMAX + 1], w[SEM_NMAX + 1], sum = 0.0, om[2 * FD_RMAX + 1];
    unsigned char id[128];
    sem_mesh m;
    size_t bytes = 0;
    for (i = 0; i < sizeof exported / sizeof exported[0]; ++i) CHECK(exported[i] != 0);
    CHECK(sem_version() != NULL && strlen(sem_version()) > 0);
    /* GLL: N = 4 closed form, sum of weights 2 */
    CHECK(sem_gll(4, xi, w) == SEM_OK);
    CHECK(xi[0] == -1.0 && xi[4] == 1.0 && fabs(xi[2]) < 1e-15);
    CHECK(fabs(xi[3] - sqrt(3.0 / 7.0)) < 1e-14 && fabs(w[2] - 32.0 / 45.0) < 1e-14);
    for (i = 0; i < 5; ++i) sum += w[i];
    CHECK(fabs(sum - 2.0) < 1e-14);
    CHECK(sem_gll(0, xi, w) == SEM_EINVAL && sem_gll(4, NULL, w) == SEM_EINVAL);
    CHECK(strlen(sem_strerror(SEM_ENCCL)) > 0);
    /* workspace query is pure host */
    memset(&m, 0, sizeof m);
    m.nelem = 8;
    m.nranks = 1;
    CHECK(sem_workspace_bytes(&m, 4, &bytes) == SEM_OK && bytes > 8 * 125 * 8 * 10);
    m.nelem = 0;
    CHECK(sem_workspace_bytes(&m, 4, &bytes) == SEM_EINVAL);
    CHECK(sem_nccl_id_bytes() == 128);
    CHECK(sem_loopback_unique_id(id) == SEM_OK && sem_loopback_unique_id(NULL) == SEM_EINVAL);
    /* FD weights (reading R6): r = 1 central stencil (1, -2, 1) / dx^2 */
    CHECK(fd_weights(1, 0.5, om) == SEM_OK);
    CHECK(om[0] == 4.0 && om[1] == -8.0 && om[2] == 4.0);
    CHECK(fd_weights(0, 0.5, om) == SEM_EINVAL);
    CHECK(sem_ax(NULL, NULL, NULL) == SEM_ESTATE);
    if (argc > 1 && strcmp(argv[1], "gpu") == 0) {
        /* one 1x1x1 affine element, N = 2: A_L 1 = 0 (constants annihilated
         * before boundary conditions) */
        enum { N = 2, n = 3, n3 = 27 };
        double xyz[3 * n3], ones[n3];
        int64_t glo[n3];
        unsigned char dir[n3];
        void *ws = NULL, *du = NULL, *dw = NULL;
        sem_ctx *ctx = NULL;
        int a, b, c, rc;
        double out[n3];
        CHECK(sem_gll(N, xi, w) == SEM_OK);
        for (c = 0; c < n; ++c)
            for (b = 0; b < n; ++b)
                for (a = 0; a < n; ++a) {
                    const int q = a + n * (b + n * c);
                    xyz[q] = (1 + xi[a]) / 2;
                    xyz[n3 + q] = (1 + xi[b]) / 2;
                    xyz[2 * n3 + q] = (1 + xi[c]) / 2;
                    glo[q] = q;
                    dir[q] = 0;
                    ones[q] = 1.0;
                }
        memset(&m, 0, sizeof m);
        m.nelem = 1;
        m.xyz = xyz;
        m.glo = glo;
        m.dirichlet = dir;
        m.nranks = 1;
        CHECK(sem_workspace_bytes(&m, N, &bytes) == SEM_OK);
        CHECK(cudaMalloc(&ws, bytes) == 0 && cudaMalloc(&du, sizeof ones) == 0 &&
              cudaMalloc(&dw, sizeof ones) == 0);
        CHECK(sem_setup(&m, N, ws, bytes, NULL, &ctx) == SEM_OK);
        CHECK(cudaMemcpy(du, ones, sizeof ones, cudaMemcpyHostToDevice) == 0);
        rc = sem_ax(ctx, (const double *)du, (double *)dw);
        CHECK(rc == SEM_OK);
        CHECK(cudaDeviceSynchronize() == 0 && cudaMemcpy(out, dw, sizeof out, cudaMemcpyDeviceToHost) == 0);
        for (a = 0; a < n3; ++a) CHECK(fabs(out[a]) < 1e-13);
        sem_free(ctx);
    }
    printf("abi_consumer ok\n");
    return 0;
}
