// launch_probe.cu -- fixed cost of a flushed single launch vs the launch
// shape: 1 CTA vs 444 CTAs x 64 KiB dynamic smem vs 148 x 200 KiB, empty
// kernels, after the bench's L2 flush (write 2xL2, read 2xL2) and without.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/launch_probe tools/launch_probe.cu
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <vector>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)
__global__ void fill_k(float4 *p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_float4(1, 1, 1, 1);
}
__global__ void sum_k(const float4 *p, size_t n, float *out) {
    float s = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        float4 v = p[i];
        s += v.x + v.y + v.z + v.w;
    }
    if (s == 12345.f) *out = s;
}
__global__ void empty_k(int *p) {
    extern __shared__ int sm[];
    if (threadIdx.x == 0 && p[0] == 12345) sm[0] = 1;
}
__global__ void small_smem_k(int *p) {   // uses dynamic smem: touches it
    extern __shared__ int sm[];
    sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    if (sm[(threadIdx.x + 1) % blockDim.x] == 12345) p[0] = 1;
}
int main() {
    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    int l2 = 0;
    CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0));
    size_t fn = (size_t)2 * l2 / 16;
    float4 *w, *r;
    float *sumo;
    int *flag;
    CK(cudaMalloc(&w, fn * 16));
    CK(cudaMalloc(&r, fn * 16));
    CK(cudaMemset(r, 0, fn * 16));
    CK(cudaMalloc(&sumo, 4));
    CK(cudaMalloc(&flag, 4));
    CK(cudaMemset(flag, 0, 4));
    CK(cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CK(cudaFuncSetAttribute(small_smem_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    struct V { const char *name; void (*k)(int *); int grid, thr, smem; };
    V vs[] = {{"1 CTA x 32, no smem", empty_k, 1, 32, 0},
              {"444 CTAs x 256, no smem", empty_k, 444, 256, 0},
              {"444 CTAs x 256, 64 KiB smem", empty_k, 444, 256, 64 << 10},
              {"444 x 256, 64 KiB smem touched", small_smem_k, 444, 256, 64 << 10},
              {"148 CTAs x 256, 200 KiB smem", empty_k, 148, 256, 200 << 10},
              {"1568 CTAs x 256, 16 KiB smem", empty_k, 1568, 256, 16 << 10}};
    for (int flush = 0; flush < 2; ++flush)
        for (auto &v : vs) {
            const int R = 40;
            std::vector<cudaEvent_t> ev(2 * R);
            for (auto &e : ev) CK(cudaEventCreate(&e));
            for (int i = -3; i < R; ++i) {
                if (flush) {
                    fill_k<<<148 * 8, 512, 0, s>>>(w, fn);
                    sum_k<<<148 * 8, 512, 0, s>>>(r, fn, sumo);
                }
                if (i >= 0) CK(cudaEventRecord(ev[2 * i], s));
                v.k<<<v.grid, v.thr, v.smem, s>>>(flag);
                if (i >= 0) CK(cudaEventRecord(ev[2 * i + 1], s));
            }
            CK(cudaStreamSynchronize(s));
            std::vector<float> t(R);
            for (int i = 0; i < R; ++i) CK(cudaEventElapsedTime(&t[i], ev[2 * i], ev[2 * i + 1]));
            std::sort(t.begin(), t.end());
            printf("%s %-34s median %6.2f us  best %6.2f us\n", flush ? "flushed" : "plain  ", v.name, t[R / 2] * 1e3,
                   t[0] * 1e3);
            for (auto &e : ev) cudaEventDestroy(e);
        }
    return 0;
}
