/*
 * embed_c.c — using libigp from plain C through include/igp.h only (no Python, no torch).
 *
 * Builds a seeded random graph on the host, then:
 *   1. igp_embed_host: host edges in, host embeddings out (one call, one sync);
 *   2. the device path: cudaMalloc'd edges -> igp_build_graph -> igp_embed -> cudaMemcpy;
 * and checks that both agree bitwise, that every value is in (0, 1) (Eq. (4))
 * and that every column of the pre-sigmoid output is standardised (ZNorm).
 * Prints one line "ok N nnz max|host-device| ..." and exits 0, or exits 1 with a message.
 *
 *   usage: embed_c [num_nodes] [num_edges] [d] [steps]
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "igp.h"

#define CHECK(call)                                                                              \
    do {                                                                                         \
        igp_status st_ = (call);                                                                 \
        if (st_ != IGP_OK) {                                                                     \
            fprintf(stderr, "%s failed: %s (%s)\n", #call, igp_status_string(st_),               \
                    igp_last_error_message());                                                   \
            return 1;                                                                            \
        }                                                                                        \
    } while (0)

static uint64_t splitmix(uint64_t* x) {
    uint64_t z = (*x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

int main(int argc, char** argv) {
    const int32_t n = argc > 1 ? atoi(argv[1]) : 3000;
    const int64_t E = argc > 2 ? atoll(argv[2]) : 30000;
    const int32_t d = argc > 3 ? atoi(argv[3]) : 64;
    const int32_t L = argc > 4 ? atoi(argv[4]) : 10;
    int32_t* edges = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)E);
    float* h_host = (float*)malloc(sizeof(float) * (size_t)n * d);
    float* h_dev = (float*)malloc(sizeof(float) * (size_t)n * d);
    if (!edges || !h_host || !h_dev) return 1;
    uint64_t seed = 12345;
    for (int64_t e = 0; e < E; ++e) {
        edges[2 * e] = (int32_t)(splitmix(&seed) % (uint64_t)n);
        edges[2 * e + 1] = (int32_t)(splitmix(&seed) % (uint64_t)n);
    }
    igp_embed_opts o;
    igp_embed_opts_default(&o);
    o.tau = -1.0f;
    o.d = d;
    o.steps = L;
    o.seed = 7;

    /* 1. host buffers end to end */
    CHECK(igp_embed_host(edges, E, n, &o, h_host, NULL));

    /* 2. device path */
    int32_t* d_edges = NULL;
    float* d_out = NULL;
    if (cudaMalloc((void**)&d_edges, sizeof(int32_t) * 2 * (size_t)E) != cudaSuccess ||
        cudaMalloc((void**)&d_out, sizeof(float) * (size_t)n * d) != cudaSuccess) {
        fprintf(stderr, "cudaMalloc failed\n");
        return 1;
    }
    cudaMemcpy(d_edges, edges, sizeof(int32_t) * 2 * (size_t)E, cudaMemcpyHostToDevice);
    igp_graph_t g = NULL;
    CHECK(igp_build_graph(d_edges, E, n, NULL, &g));
    int32_t nn = 0;
    int64_t nnz = 0, m = 0;
    CHECK(igp_graph_info(g, &nn, &nnz, &m));
    CHECK(igp_embed_ex(g, &o, d_out, NULL));
    cudaMemcpy(h_dev, d_out, sizeof(float) * (size_t)n * d, cudaMemcpyDeviceToHost);

    double maxdiff = 0.0;
    for (size_t k = 0; k < (size_t)n * d; ++k) {
        const double x = h_dev[k];
        if (!(x > 0.0 && x < 1.0)) {
            fprintf(stderr, "value %g outside (0, 1) at %zu\n", x, k);
            return 1;
        }
        maxdiff = fmax(maxdiff, fabs(x - (double)h_host[k]));
    }
    if (maxdiff != 0.0) {
        fprintf(stderr, "host and device paths differ by %g\n", maxdiff);
        return 1;
    }

    /* pre-sigmoid columns are z-scores: mean 0, population std 1 */
    o.mode = IGP_MODE_PRE_SIGMOID;
    CHECK(igp_embed_ex(g, &o, d_out, NULL));
    cudaMemcpy(h_dev, d_out, sizeof(float) * (size_t)n * d, cudaMemcpyDeviceToHost);
    double worst = 0.0;
    for (int32_t c = 0; c < d; ++c) {
        double s1 = 0.0, s2 = 0.0;
        for (int32_t i = 0; i < n; ++i) {
            const double x = h_dev[(size_t)i * d + c];
            s1 += x;
            s2 += x * x;
        }
        const double mu = s1 / n, sd = sqrt(s2 / n - mu * mu);
        worst = fmax(worst, fmax(fabs(mu), fabs(sd - 1.0)));
    }
    if (worst > 1e-4) {
        fprintf(stderr, "pre-sigmoid column moments off by %g\n", worst);
        return 1;
    }
    CHECK(igp_destroy_graph(g));
    cudaFree(d_edges);
    cudaFree(d_out);
    printf("ok N=%d nnz=%lld M=%lld d=%d L=%d max|host-device|=%g column-moment error=%.2e launches=%llu\n", nn,
           (long long)nnz, (long long)m, d, L, maxdiff, worst, (unsigned long long)igp_kernel_launch_count());
    free(edges);
    free(h_host);
    free(h_dev);
    return 0;
}
