/*
 * INTEGRATION.md §4, compiled as plain C: a caller that owns its ZeRO rank partitions
 * in device memory drives the hot path through the C ABI with a tg_layout built from
 * checkpoint directories (tg_layout_from_checkpoints) — no synthetic family involved:
 *   load every snapshot's rank-shard and weights payloads into device buffers
 *   -> tg_scorer per rank -> FP64 partials [N][K-1][M][2] (rank order)
 *   -> tg_comm_allgather (the partials table through the library's NCCL communicator)
 *   -> tg_layout_select (a14: magnitude selection -> recipe over the directories)
 *   -> tg_mplan per output container (bind the device payloads, K2 gather)
 *   -> write the composite payload files (tg_mplan_prefix + gathered payload).
 * Usage: device_flow OUT_DIR RHO DIR_1 ... DIR_K. Prints the recipe YAML on stdout.
 * TEST INFRASTRUCTURE (tests/test_integration_build.py); built by tests/integration/Makefile.
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/stat.h>

#include "tailor_b200.h"

static void die(const char* what, int rc) {
    fprintf(stderr, "error: %s: %s (%d)\n", what, rc ? tg_last_error() : "", rc);
    exit(rc >= 1 && rc <= 9 ? 1 : 2);
}

static void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        fprintf(stderr, "cuda: %s: %s\n", what, cudaGetErrorString(e));
        exit(2);
    }
}

/* Payload of a container file (u64 LE header length, header, payload) into device memory. */
static uint8_t* load_payload(const char* path, uint64_t expect) {
    FILE* f = fopen(path, "rb");
    if (!f) {
        fprintf(stderr, "cannot open %s\n", path);
        exit(1);
    }
    unsigned char h8[8];
    if (fread(h8, 1, 8, f) != 8) exit(1);
    uint64_t hlen = 0;
    for (int i = 0; i < 8; ++i) hlen |= (uint64_t)h8[i] << (8 * i);
    fseek(f, (long)(8 + hlen), SEEK_SET);
    uint8_t* host = (uint8_t*)malloc(expect ? expect : 1);
    if (fread(host, 1, expect, f) != expect) {
        fprintf(stderr, "%s: short payload\n", path);
        exit(1);
    }
    fclose(f);
    uint8_t* dev = NULL;
    cuda(cudaMalloc((void**)&dev, expect ? expect : 16), "cudaMalloc");
    cuda(cudaMemcpy(dev, host, expect, cudaMemcpyHostToDevice), "H2D");
    free(host);
    return dev;
}

static char* text(int (*f)(const tg_layout*, const double*, int32_t, double, char*, size_t, size_t*, int32_t*, double*,
                           double*),
                  const tg_layout* l, const double* parts, int32_t n, double rho) {
    size_t need = 0;
    char* buf = (char*)malloc(1 << 16);
    int rc = f(l, parts, n, rho, buf, 1 << 16, &need, NULL, NULL, NULL);
    if (rc != TG_OK && need > (1 << 16)) {
        buf = (char*)realloc(buf, need);
        rc = f(l, parts, n, rho, buf, need, &need, NULL, NULL, NULL);
    }
    if (rc != TG_OK) die("tg_layout_select", rc);
    return buf;
}

/* One output container: plan, bind the loaded payloads of each window, gather, write. */
static void merge_container(const tg_layout* l, const char* yaml, int32_t container, uint8_t** shard_dev /* [K][N] */,
                            uint8_t** weights_dev /* [K] */, int32_t N, const char* path) {
    tg_mplan* p = tg_mplan_create(l, yaml, container, 0, 1);
    if (!p) die("tg_mplan_create", tg_last_error_kind());
    const int32_t nw = tg_mplan_num_windows(p);
    const uint8_t** ptrs = (const uint8_t**)calloc((size_t)nw + 1, sizeof(uint8_t*));
    for (int32_t w = 0; w < nw; ++w) {
        int32_t k = 0, c = 0;
        uint64_t lo = 0, hi = 0;
        int rc = tg_mplan_window(p, w, &k, &c, &lo, &hi);
        if (rc) die("tg_mplan_window", rc);
        ptrs[w] = (c < 0 ? weights_dev[k - 1] : shard_dev[(size_t)(k - 1) * N + c]) + lo;
    }
    int rc = tg_mplan_bind(p, ptrs);
    if (rc) die("tg_mplan_bind", rc);
    const uint64_t n = tg_mplan_bytes(p);
    uint8_t* d = NULL;
    cuda(cudaMalloc((void**)&d, n ? n : 16), "cudaMalloc");
    if ((rc = tg_mplan_run(p, d, 0, NULL))) die("tg_mplan_run", rc);
    cuda(cudaDeviceSynchronize(), "sync");
    uint8_t* h = (uint8_t*)malloc(n ? n : 1);
    cuda(cudaMemcpy(h, d, n, cudaMemcpyDeviceToHost), "D2H");
    size_t need = 0;
    tg_mplan_prefix(p, NULL, 0, &need);
    char* prefix = (char*)malloc(need);
    if ((rc = tg_mplan_prefix(p, prefix, need, &need))) die("tg_mplan_prefix", rc);
    FILE* f = fopen(path, "wb");
    if (!f || fwrite(prefix, 1, need, f) != need || fwrite(h, 1, n, f) != n) exit(2);
    fclose(f);
    free(prefix);
    free(h);
    free(ptrs);
    cudaFree(d);
    tg_mplan_destroy(p);
}

int main(int argc, char** argv) {
    if (argc < 5) {
        fprintf(stderr, "usage: device_flow OUT_DIR RHO DIR_1 ... DIR_K\n");
        return 1;
    }
    const char* out = argv[1];
    const double rho = atof(argv[2]);
    const int32_t K = argc - 3;
    const char* const* dirs = (const char* const*)(argv + 3);
    tg_layout* l = tg_layout_from_checkpoints(dirs, K);
    if (!l) die("tg_layout_from_checkpoints", tg_last_error_kind());
    const int32_t N = tg_layout_num_ranks(l), M = tg_layout_num_modules(l);

    uint8_t** shard_dev = (uint8_t**)calloc((size_t)K * N, sizeof(uint8_t*));
    uint8_t** weights_dev = (uint8_t**)calloc((size_t)K, sizeof(uint8_t*));
    char path[4096];
    for (int32_t k = 1; k <= K; ++k) {
        snprintf(path, sizeof path, "%s/model.weights", dirs[k - 1]);
        weights_dev[k - 1] = load_payload(path, tg_layout_weights_bytes(l, k));
        for (int32_t r = 0; r < N; ++r) {
            snprintf(path, sizeof path, "%s/optim/rank_%d.shard", dirs[k - 1], r);
            shard_dev[(size_t)(k - 1) * N + r] = load_payload(path, tg_layout_shard_bytes(l, k, r));
        }
    }

    /* score every rank partition; partials land in rank order */
    const size_t per_rank = (size_t)(K - 1) * M * 2;
    double* parts = (double*)calloc(per_rank * N, sizeof(double));
    double* d_out = NULL;
    cuda(cudaMalloc((void**)&d_out, per_rank * sizeof(double)), "cudaMalloc");
    for (int32_t r = 0; r < N; ++r) {
        tg_scorer* s = tg_scorer_create(l, r, 1, K, 0);
        if (!s) die("tg_scorer_create", tg_last_error_kind());
        const uint8_t** bases = (const uint8_t**)calloc((size_t)K, sizeof(uint8_t*));
        for (int32_t k = 0; k < K; ++k) bases[k] = shard_dev[(size_t)k * N + r];
        int rc = tg_scorer_run(s, bases, d_out, NULL);
        if (rc) die("tg_scorer_run", rc);
        cuda(cudaMemcpy(parts + per_rank * r, d_out, per_rank * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
        free(bases);
        tg_scorer_destroy(s);
    }
    /* the partials table through the library's NCCL all-gather: this process is the one
     * rank of its job here (a GPU per rank in a real job: rank 0 makes the id, the caller
     * ships it to the others, every rank contributes its own rows) */
    {
        uint8_t id[128];
        if (tg_comm_unique_id(id) != TG_OK) die("tg_comm_unique_id", tg_last_error_kind());
        tg_comm* c = tg_comm_create(id, 1, 0, 0);
        if (!c) die("tg_comm_create", tg_last_error_kind());
        double *d_rows = NULL, *d_table = NULL;
        const size_t n = per_rank * (size_t)N;
        cuda(cudaMalloc((void**)&d_rows, n * sizeof(double)), "cudaMalloc");
        cuda(cudaMalloc((void**)&d_table, n * sizeof(double)), "cudaMalloc");
        cuda(cudaMemcpy(d_rows, parts, n * sizeof(double), cudaMemcpyHostToDevice), "H2D");
        int rc = tg_comm_allgather(c, d_rows, d_table, n, NULL);
        if (rc) die("tg_comm_allgather", rc);
        cuda(cudaMemcpy(parts, d_table, n * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
        cudaFree(d_rows);
        cudaFree(d_table);
        tg_comm_destroy(c);
    }
    char* yaml = text(tg_layout_select, l, parts, N, rho);
    printf("%s", yaml);
    snprintf(path, sizeof path, "%s.recipe.yaml", out); /* stdout may also carry library banners */
    FILE* rf = fopen(path, "w");
    if (!rf) die("fopen recipe", 0);
    fputs(yaml, rf);
    fclose(rf);

    snprintf(path, sizeof path, "%s/optim", out);
    mkdir(out, 0755);
    mkdir(path, 0755);
    snprintf(path, sizeof path, "%s/model.weights", out);
    merge_container(l, yaml, -1, shard_dev, weights_dev, N, path);
    for (int32_t r = 0; r < N; ++r) {
        snprintf(path, sizeof path, "%s/optim/rank_%d.shard", out, r);
        merge_container(l, yaml, r, shard_dev, weights_dev, N, path);
    }
    tg_layout_destroy(l);
    return 0;
}
