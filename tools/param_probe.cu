// param_probe.cu -- launch cost vs kernel-parameter size on B200: an empty
// kernel taking a __grid_constant__ struct of N bytes, timed with the
// bench's flushed protocol (event pair around one launch, after a 2xL2
// write + read) and back to back.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/param_probe tools/param_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <algorithm>

template <int N>
struct P {
    unsigned char b[N];
};

template <int N>
__global__ void k_param(const __grid_constant__ P<N> p, int *out) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && p.b[N - 1] == 123) *out = p.b[0];
}

__global__ void fill(float *p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = 1.f;
}
__global__ void sum(const float *p, size_t n, float *o) {
    float s = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) s += p[i];
    if (s == 12345.f) *o = s;
}

template <int N>
void run(int *out, float *w, float *r, size_t fn, float *so, cudaStream_t st) {
    P<N> p{};
    std::vector<float> flushed, b2b;
    for (int rep = 0; rep < 43; ++rep) {
        fill<<<1184, 256, 0, st>>>(w, fn);
        sum<<<1184, 256, 0, st>>>(r, fn, so);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, st);
        k_param<N><<<296, 256, 0, st>>>(p, out);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep >= 3) flushed.push_back(ms * 1e3f);
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
    for (int i = 0; i < 200; ++i) k_param<N><<<296, 256, 0, st>>>(p, out);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    std::sort(flushed.begin(), flushed.end());
    double mean = 0;
    for (float v : flushed) mean += v;
    mean /= flushed.size();
    printf("param %5d B: flushed single launch mean %6.2f us median %6.2f us | back-to-back %6.2f us/launch\n", N, mean,
           flushed[flushed.size() / 2], ms * 1e3f / 200);
}

int main() {
    int *out;
    cudaMalloc(&out, 4);
    size_t fn = (size_t)2 * 126 * 1024 * 1024 / 4 * 2;
    float *w, *r, *so;
    cudaMalloc(&w, fn * 4);
    cudaMalloc(&r, fn * 4);
    cudaMalloc(&so, 4);
    cudaMemset(r, 0, fn * 4);
    cudaStream_t st;
    cudaStreamCreate(&st);
    run<64>(out, w, r, fn, so, st);
    run<1024>(out, w, r, fn, so, st);
    run<2048>(out, w, r, fn, so, st);
    run<4000>(out, w, r, fn, so, st);
    run<4096>(out, w, r, fn, so, st);
    run<5120>(out, w, r, fn, so, st);
    run<6144>(out, w, r, fn, so, st);
    run<8192>(out, w, r, fn, so, st);
    run<16384>(out, w, r, fn, so, st);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
