// copy_pattern_probe.cu -- SM copy kernels of 2 GiB: grid-stride vs per-warp contiguous chunks at
// several CTAs per SM, against cudaMemcpyAsync D2D (nvcc -O3 -gencode arch=compute_100a,code=sm_100a).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
// A: grid-stride, U=4
__global__ void copyA(const uint4* __restrict__ s, uint4* __restrict__ d, int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n; i += 4 * stride) {
        uint4 r0 = __ldg(s + i), r1 = __ldg(s + i + stride), r2 = __ldg(s + i + 2 * stride), r3 = __ldg(s + i + 3 * stride);
        d[i] = r0; d[i + stride] = r1; d[i + 2 * stride] = r2; d[i + 3 * stride] = r3;
    }
    for (; i < n; i += stride) d[i] = __ldg(s + i);
}
// B: each warp owns contiguous chunks of CH vectors (CH/32 per lane), chunks grid-strided
template <int CH>
__global__ void copyB(const uint4* __restrict__ s, uint4* __restrict__ d, int64_t n) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = warp * CH; c < n; c += nwarps * CH) {
        uint4 r[CH / 32];
#pragma unroll
        for (int j = 0; j < CH / 32; ++j) r[j] = __ldg(s + c + lane + 32 * j);
#pragma unroll
        for (int j = 0; j < CH / 32; ++j) d[c + lane + 32 * j] = r[j];
    }
}
int main() {
    const int64_t bytes = 1ll << 31, n = bytes / 16;
    uint4 *a, *b; cudaMalloc(&a, bytes); cudaMalloc(&b, bytes);
    char *fl; cudaMalloc(&fl, 512 << 20);
    cudaMemset(a, 1, bytes);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char *name, auto launch) {
        float best = 1e9, tot = 0;
        for (int it = 0; it < 8; ++it) {
            cudaMemsetAsync(fl, it, 512 << 20);
            cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (it >= 2) { tot += ms; best = ms < best ? ms : best; }
        }
        printf("%-28s mean %.1f us  %.0f GB/s (best %.0f)\n", name, tot / 6 * 1e3, 2.0 * bytes / (tot / 6 * 1e-3) / 1e9, 2.0 * bytes / (best * 1e-3) / 1e9);
    };
    int sms = 148;
    for (int bpsm : {4, 8, 16}) {
        char nm[64];
        snprintf(nm, 64, "A grid-stride %d/SM", bpsm);
        run(nm, [&] { copyA<<<sms * bpsm, 256>>>(a, b, n); });
        snprintf(nm, 64, "B warp 4KB %d/SM", bpsm);
        run(nm, [&] { copyB<256><<<sms * bpsm, 256>>>(a, b, n); });
        snprintf(nm, 64, "B warp 8KB %d/SM", bpsm);
        run(nm, [&] { copyB<512><<<sms * bpsm, 256>>>(a, b, n); });
        snprintf(nm, 64, "B warp 2KB %d/SM", bpsm);
        run(nm, [&] { copyB<128><<<sms * bpsm, 256>>>(a, b, n); });
    }
    run("cudaMemcpyAsync D2D", [&] { cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice); });
    return 0;
}
