/* c_api_demo.c -- the libvpgpu C ABI (include/vpgpu.h) from plain C.
 *
 * A caller that owns its own device memory (here: cudaMalloc) plans a
 * permutation once, runs it on a stream, and checks the result on the host
 * against out[i] = in[f(i)] (core.py:173-178).  It then runs the fused
 * sharded exchange with G virtual ranks on the one device: each rank's
 * kernel reads its input shard and stores into all output shards.
 *
 *   gcc -O2 -I include examples/c_api_demo.c -o c_api_demo \
 *       -L paper_2506_03686_b200 -lvpgpu -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2506_03686_b200
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "vpgpu.h"

#define CHECK(call)                                                                    \
    do {                                                                               \
        vpg_status s_ = (call);                                                        \
        if (s_ != VPG_OK) {                                                            \
            fprintf(stderr, "%s failed (%d): %s\n", #call, (int)s_, vpg_last_error()); \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

/* destination offset i -> source offset, dims/sigma inner-first */
static int64_t src_of(int64_t i, int rank, const int64_t *dims, const int32_t *sigma) {
    int64_t stride[VPG_MAX_RANK], s = 0;
    stride[0] = 1;
    for (int k = 1; k < rank; ++k) stride[k] = stride[k - 1] * dims[k - 1];
    for (int j = 0; j < rank; ++j) {
        const int64_t d = dims[sigma[j]];
        s += (i % d) * stride[sigma[j]];
        i /= d;
    }
    return s;
}

int main(void) {
    /* numpy shape (64, 48, 40, 30), axes (2, 0, 3, 1) as inner-first dims/sigma */
    const int rank = 4;
    const int64_t dims[4] = {30, 40, 48, 64};
    const int32_t sigma[4] = {2, 0, 3, 1};
    int64_t n = 1;
    for (int k = 0; k < rank; ++k) n *= dims[k];
    const size_t bytes = (size_t)n * sizeof(uint32_t);
    uint32_t *h_in = malloc(bytes), *h_out = malloc(bytes);
    for (int64_t i = 0; i < n; ++i) h_in[i] = (uint32_t)(i * 2654435761u + 12345u);
    void *d_in = NULL, *d_out = NULL;
    cudaStream_t st;
    if (cudaMalloc(&d_in, bytes) != cudaSuccess || cudaMalloc(&d_out, bytes) != cudaSuccess ||
        cudaStreamCreate(&st) != cudaSuccess) {
        fprintf(stderr, "CUDA setup failed\n");
        return 1;
    }
    cudaMemcpy(d_in, h_in, bytes, cudaMemcpyHostToDevice);

    vpg_plan *plan = NULL;
    CHECK(vpg_plan_create(rank, dims, sigma, 4, 0, &plan));
    char text[4096];
    CHECK(vpg_plan_describe(plan, text, sizeof text));
    printf("%s", text);
    CHECK(vpg_permute(plan, d_in, d_out, st));
    cudaStreamSynchronize(st);
    cudaMemcpy(h_out, d_out, bytes, cudaMemcpyDeviceToHost);
    int64_t bad = 0;
    for (int64_t i = 0; i < n; ++i) bad += h_out[i] != h_in[src_of(i, rank, dims, sigma)];
    printf("permute: %lld mismatches of %lld\n", (long long)bad, (long long)n);
    vpg_plan_destroy(plan);
    if (bad) return 2;

    /* fused sharded exchange, G virtual ranks on this device */
    const int G = 4;
    void *shards[4];
    for (int q = 0; q < G; ++q) cudaMalloc(&shards[q], bytes / G);
    for (int r = 0; r < G; ++r) {
        vpg_plan *sp = NULL;
        CHECK(vpg_plan_create_sharded(rank, dims, sigma, 4, 0, G, r, &sp));
        CHECK(vpg_permute_sharded(sp, (const char *)d_in + (size_t)r * (bytes / G), shards, st));
        cudaStreamSynchronize(st);
        vpg_plan_destroy(sp);
    }
    for (int q = 0; q < G; ++q) cudaMemcpy((char *)h_out + (size_t)q * (bytes / G), shards[q], bytes / G,
                                          cudaMemcpyDeviceToHost);
    bad = 0;
    for (int64_t i = 0; i < n; ++i) bad += h_out[i] != h_in[src_of(i, rank, dims, sigma)];
    printf("sharded exchange (G=%d): %lld mismatches\n", G, (long long)bad);
    for (int q = 0; q < G; ++q) cudaFree(shards[q]);
    cudaFree(d_in);
    cudaFree(d_out);
    free(h_in);
    free(h_out);
    return bad ? 3 : 0;
}
