/* A non-Python host on the C ABI alone (include/td_api.h + libtdb200.so +
 * the CUDA runtime): what a Go/cgo, JNI or N-API binding of the reference's
 * compare path would call.  rel_err of two device arrays (td_rel_err), the
 * perturbation of a bf16 tensor (td_perturb) and replica digests
 * (td_fingerprint), checked against host arithmetic.  Exit 0 = pass. */
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "td_api.h"

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_)); return 2; } } while (0)
#define TD(x) do { if ((x) != 0) { fprintf(stderr, "%s: %s\n", #x, td_last_error()); return 3; } } while (0)

static uint16_t f2bf(float f) {            /* RNE float -> bf16 bits (finite inputs) */
    uint32_t u;
    memcpy(&u, &f, 4);
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

static double bf2d(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

int main(void) {
    const int64_t n = (1 << 20) + 3;          /* vector body + scalar tail */
    uint16_t* ha = malloc(n * 2);
    uint16_t* hb = malloc(n * 2);
    double d2 = 0.0, a2 = 0.0;
    srand(7);
    for (int64_t i = 0; i < n; ++i) {
        const float x = (float)rand() / RAND_MAX - 0.5f;
        const float y = x * (1.0f + 0.01f * ((float)rand() / RAND_MAX - 0.5f));
        ha[i] = f2bf(x);
        hb[i] = f2bf(y);
        const double dx = bf2d(ha[i]), dy = bf2d(hb[i]);
        d2 += (dx - dy) * (dx - dy);
        a2 += dx * dx;
    }
    const double want = sqrt(d2) / sqrt(a2);
    void *da, *db, *work, *dy;
    double* dout;
    CK(cudaMalloc(&da, n * 2));
    CK(cudaMalloc(&db, n * 2));
    CK(cudaMalloc(&dy, n * 2));
    CK(cudaMalloc(&work, TD_REL_ERR_WORK_BYTES));
    CK(cudaMalloc((void**)&dout, 3 * sizeof(double)));
    CK(cudaMemset(work, 0, TD_REL_ERR_WORK_BYTES));
    CK(cudaMemcpy(da, ha, n * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db, hb, n * 2, cudaMemcpyHostToDevice));

    /* rel_err_arrays(a, b) */
    double out[3];
    TD(td_rel_err(da, db, TD_BF16, n, work, dout, NULL));
    CK(cudaMemcpy(out, dout, sizeof(out), cudaMemcpyDeviceToHost));
    const double got = out[2];
    if (!(fabs(got - want) <= 1e-9 * want)) {
        fprintf(stderr, "rel_err %.17g vs host %.17g\n", got, want);
        return 4;
    }

    /* perturbation with eps = 0 is the identity on bf16 values */
    unsigned long long* dnf;
    CK(cudaMalloc((void**)&dnf, 8));
    CK(cudaMemset(dnf, 0, 8));
    TD(td_perturb(da, dy, TD_BF16, TD_BF16, 1, n, n, 0, NULL, 0, 0x1234u, 0.0, TD_FMT_BF16,
                  TD_GEN_SPLITMIX64, dnf, NULL));
    TD(td_rel_err(da, dy, TD_BF16, n, work, dout, NULL));
    CK(cudaMemcpy(out, dout, sizeof(out), cudaMemcpyDeviceToHost));
    if (out[2] != 0.0) { fprintf(stderr, "eps=0 perturbation changed values: %g\n", out[2]); return 5; }

    /* digests: equal copies agree, a different copy does not */
    td_fp_item items[3] = {{da, n * 2}, {dy, n * 2}, {db, n * 2}};
    int64_t begin[4] = {0};
    for (int i = 0; i < 3; ++i) begin[i + 1] = begin[i] + (items[i].nbytes + TD_FP_CHUNK - 1) / TD_FP_CHUNK;
    void *ditems, *dbegin;
    unsigned long long* ddig;
    CK(cudaMalloc(&ditems, sizeof(items)));
    CK(cudaMalloc(&dbegin, sizeof(begin)));
    CK(cudaMalloc((void**)&ddig, 6 * 8));
    CK(cudaMemcpy(ditems, items, sizeof(items), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dbegin, begin, sizeof(begin), cudaMemcpyHostToDevice));
    CK(cudaMemset(ddig, 0, 6 * 8));
    TD(td_fingerprint((const td_fp_item*)ditems, (const int64_t*)dbegin, 3, begin[3], ddig, NULL));
    unsigned long long dig[6];
    CK(cudaMemcpy(dig, ddig, sizeof(dig), cudaMemcpyDeviceToHost));
    if (dig[0] != dig[2] || dig[1] != dig[3] || (dig[0] == dig[4] && dig[1] == dig[5])) {
        fprintf(stderr, "digests disagree\n");
        return 6;
    }
    /* the cross-GPU exchange on a one-rank NCCL communicator: the sums come
     * back unchanged (NCCL resolved by dlopen here as in the library) */
    void* nccl = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (nccl) {
        typedef struct { char internal[128]; } nccl_id;
        int (*get_id)(nccl_id*) = (int (*)(nccl_id*))dlsym(nccl, "ncclGetUniqueId");
        int (*init_rank)(void**, int, nccl_id, int) = (int (*)(void**, int, nccl_id, int))dlsym(nccl, "ncclCommInitRank");
        int (*destroy)(void*) = (int (*)(void*))dlsym(nccl, "ncclCommDestroy");
        nccl_id uid;
        void* comm = NULL;
        if (!get_id || !init_rank || get_id(&uid) != 0 || init_rank(&comm, 1, uid, 0) != 0) {
            fprintf(stderr, "cannot create a one-rank NCCL communicator\n");
            return 8;
        }
        double sl[3] = {1.5, -2.0, 3.25}, back[3];
        double* dsl;
        CK(cudaMalloc((void**)&dsl, sizeof(sl)));
        CK(cudaMemcpy(dsl, sl, sizeof(sl), cudaMemcpyHostToDevice));
        TD(td_allreduce_partials(comm, dsl, 3, NULL));
        TD(td_allreduce_digests(comm, (long long*)ddig, 6, NULL));
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(back, dsl, sizeof(back), cudaMemcpyDeviceToHost));
        unsigned long long dig2[6];
        CK(cudaMemcpy(dig2, ddig, sizeof(dig2), cudaMemcpyDeviceToHost));
        if (memcmp(back, sl, sizeof(sl)) != 0 || memcmp(dig, dig2, sizeof(dig)) != 0) {
            fprintf(stderr, "one-rank all-reduce changed the values\n");
            return 9;
        }
        destroy(comm);
    }
    /* errors come back as status codes with a message, not exceptions */
    if (td_rel_err(NULL, db, TD_BF16, n, work, dout, NULL) == 0 || !strstr(td_last_error(), "td_rel_err")) {
        fprintf(stderr, "invalid arguments not reported\n");
        return 7;
    }
    printf("c abi ok: td_version %d, rel_err %.17g (host %.17g), nccl exchange %s\n", td_version(), got, want,
           nccl ? "checked" : "skipped (no libnccl.so.2)");
    return 0;
}
