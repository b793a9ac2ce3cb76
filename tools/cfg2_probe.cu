// cfg2_probe.cu -- design probe for the small-problem transpose (cfg2:
// f32 (32,64,56,56) -> (0,2,3,1), i.e. 32 batched 64 x 3136 -> 3136 x 64).
// Times candidate kernel structures with the bench's flushed protocol
// (write 2xL2, read 2xL2, event, kernel, event) to find which one beats the
// current tile kernel's ~13.1 us (floor ~6.1 us) -- standalone, no library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/cfg2_probe tools/cfg2_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <string>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

// problem: NB batches of a C x HW -> HW x C transpose (cfg2: 32 x 64 x 3136;
// cfg1: 1 x 4096 x 4096 via argv "cfg1"); tiles of 64 c x 64 hw
__constant__ int d_NB, d_C, d_HW;
static int NB = 32, C = 64, HW = 3136;
static size_t N = (size_t)32 * 64 * 3136;

// ------------------------------------------------------------------ flush
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

// ------------------------------------------------------------------ V0 copy (bound)
__global__ void copy_k(const float4 *__restrict__ a, float4 *__restrict__ b, size_t n) {
    size_t i = blockIdx.x * (size_t)blockDim.x * 4 + threadIdx.x;
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) if (i + u * blockDim.x < n) v[u] = a[i + u * blockDim.x];
#pragma unroll
    for (int u = 0; u < 4; ++u) if (i + u * blockDim.x < n) b[i + u * blockDim.x] = v[u];
}

template <int U>
__global__ void copy_u(const float4 *__restrict__ a, float4 *__restrict__ b, size_t n) {
    size_t i = blockIdx.x * (size_t)blockDim.x * U + threadIdx.x;
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) if (i + u * blockDim.x < n) v[u] = a[i + u * blockDim.x];
#pragma unroll
    for (int u = 0; u < U; ++u) if (i + u * blockDim.x < n) b[i + u * blockDim.x] = v[u];
}

// ------------------------------------------------------------------ V1 LDG tile 64c x T hw per CTA
// smem tile [64 c][T hw] floats, 16B chunks XOR-swizzled by (c>>2)&7 ... (see below)
template <int T>
__global__ void __launch_bounds__(256) ldg_tile_k(const float *__restrict__ in, float *__restrict__ out) {
    constexpr int CH = T / 4;           // 16-byte chunks per c-row
    constexpr int CT = 64;              // c rows per tile
    __shared__ __align__(128) float4 s[CT * CH];
    const int C = d_C, HW = d_HW;
    const int tiles_per_n = HW / T, ctiles = C / CT;
    const int n = blockIdx.x / (tiles_per_n * ctiles), rem = blockIdx.x % (tiles_per_n * ctiles);
    const int c0 = (rem / tiles_per_n) * CT, h0 = (rem % tiles_per_n) * T;
    const float *src = in + ((size_t)n * C + c0) * HW + h0;
    float *dst = out + ((size_t)n * HW + h0) * C + c0;
    const int tid = threadIdx.x;
    constexpr int PER = CT * CH / 256;
    float4 v[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int q = tid + u * 256, c = q / CH, j = q % CH;
        v[u] = *reinterpret_cast<const float4 *>(src + (size_t)c * HW + j * 4);
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int q = tid + u * 256, c = q / CH, j = q % CH;
        s[c * CH + (j ^ ((c >> 2) & (CH - 1) & 7))] = v[u];
    }
    __syncthreads();
    // W: 4c x 4hw blocks; lanes: cb = lane%16 over c, hb across lanes/warps
    constexpr int NBLK = (CT / 4) * (T / 4);
    for (int b = tid; b < NBLK; b += 256) {
        const int cb = b % 16, hb = b / 16;
        float4 r[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int c = cb * 4 + i;
            r[i] = s[c * CH + (hb ^ ((c >> 2) & (CH - 1) & 7))];
        }
        const float *rr = reinterpret_cast<const float *>(r);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float4 o = make_float4(rr[0 * 4 + j], rr[1 * 4 + j], rr[2 * 4 + j], rr[3 * 4 + j]);
            *reinterpret_cast<float4 *>(dst + (size_t)(hb * 4 + j) * C + cb * 4) = o;
        }
    }
}

// ------------------------------------------------------------------ V3 TMA tile
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// one 64c x 64hw tile per CTA (or ITER tiles for a persistent grid), loaded as
// two TMA boxes {32 hw, 64 c} with SWIZZLE_128B: row c is 128 bytes, chunk j at
// ((j ^ (c & 7)) * 16)
template <int STAGES>
__global__ void __launch_bounds__(256) tma_tile_k(const __grid_constant__ CUtensorMap tm, float *__restrict__ out,
                                                  int ntiles) {
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char *sm = sm_raw + ((1024 - (su32(sm_raw) & 1023)) & 1023);
    __shared__ __align__(8) uint64_t bar[STAGES];
    const int tid = threadIdx.x;
    const int cnt = (ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    const int C = d_C, HW = d_HW;
    const int tiles_per_n = HW / 64, ctiles = C / 64;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tm) : "memory");
        for (int k = 0; k < STAGES && k < cnt; ++k) {
            const int t = blockIdx.x + k * gridDim.x;
            const int n = t / (tiles_per_n * ctiles), rem = t % (tiles_per_n * ctiles);
            const int c0 = (rem / tiles_per_n) * 64, h0 = (rem % tiles_per_n) * 64;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&bar[k])), "r"(16384)
                         : "memory");
            for (int h = 0; h < 2; ++h)
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
                        su32(sm + k * 16384 + h * 8192)),
                    "l"(&tm), "r"(h0 + 32 * h), "r"(c0), "r"(n), "r"(su32(&bar[k]))
                    : "memory");
        }
    }
    __syncthreads();
    const int lane = tid & 31, warp = tid >> 5;
    for (int k = 0; k < cnt; ++k) {
        const int st = k % STAGES;
        const int t = blockIdx.x + k * gridDim.x;
        const int n = t / (tiles_per_n * ctiles), rem = t % (tiles_per_n * ctiles);
        const int c0 = (rem / tiles_per_n) * 64, h0 = (rem % tiles_per_n) * 64;
        asm volatile(
            "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                su32(&bar[st])),
            "r"((k / STAGES) & 1)
            : "memory");
        const unsigned char *tile = sm + st * 16384;
        float *dst = out + ((size_t)n * HW + h0) * C + c0;
        // thread block: 4c x 4hw.  lane -> (j = lane & 7: hw chunk in half, cq = lane >> 3: c block 0..3)
        // warp -> (half = warp & 1, cgrp = warp >> 1: c blocks 4*cgrp .. +3)
        const int j = lane & 7, half = warp & 1, cb = (warp >> 1) * 4 + (lane >> 3);
        float4 r[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int c = cb * 4 + i;
            r[i] = *reinterpret_cast<const float4 *>(tile + half * 8192 + c * 128 + ((j ^ (c & 7)) * 16));
        }
        const float *rr = reinterpret_cast<const float *>(r);
        const int hw = half * 32 + j * 4;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float4 o = make_float4(rr[0 * 4 + q], rr[1 * 4 + q], rr[2 * 4 + q], rr[3 * 4 + q]);
            *reinterpret_cast<float4 *>(dst + (size_t)(hw + q) * C + cb * 4) = o;
        }
        __syncthreads();
        if (tid == 0 && k + STAGES < cnt) {
            const int t2 = blockIdx.x + (k + STAGES) * gridDim.x;
            const int n2 = t2 / (tiles_per_n * ctiles), rem2 = t2 % (tiles_per_n * ctiles);
            const int c2 = (rem2 / tiles_per_n) * 64, h2 = (rem2 % tiles_per_n) * 64;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&bar[st])), "r"(16384)
                         : "memory");
            for (int h = 0; h < 2; ++h)
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
                        su32(sm + st * 16384 + h * 8192)),
                    "l"(&tm), "r"(h2 + 32 * h), "r"(c2), "r"(n2), "r"(su32(&bar[st]))
                    : "memory");
        }
    }
}

// ------------------------------------------------------------------ host
static float *g_w, *g_r, *g_sum;
static size_t g_fn;
static void flush(cudaStream_t s) {
    fill_k<<<148 * 8, 512, 0, s>>>((float4 *)g_w, g_fn);
    sum_k<<<148 * 8, 512, 0, s>>>((const float4 *)g_r, g_fn, g_sum);
}

template <typename F>
static void timeit(const char *name, F launch, const float *dout, const std::vector<float> &ref, cudaStream_t s,
                   double bytes) {
    CK(cudaMemset((void *)dout, 0, N * 4));
    for (int i = 0; i < 3; ++i) { flush(s); launch(s); }
    CK(cudaStreamSynchronize(s));
    std::vector<float> h(N);
    CK(cudaMemcpy(h.data(), dout, N * 4, cudaMemcpyDeviceToHost));
    bool ok = ref.empty() || std::equal(h.begin(), h.end(), ref.begin());
    const int R = 40;
    std::vector<cudaEvent_t> ev(2 * R);
    for (auto &e : ev) CK(cudaEventCreate(&e));
    for (int i = 0; i < R; ++i) {
        flush(s);
        CK(cudaEventRecord(ev[2 * i], s));
        launch(s);
        CK(cudaEventRecord(ev[2 * i + 1], s));
    }
    CK(cudaStreamSynchronize(s));
    std::vector<float> t(R);
    for (int i = 0; i < R; ++i) CK(cudaEventElapsedTime(&t[i], ev[2 * i], ev[2 * i + 1]));
    std::sort(t.begin(), t.end());
    printf("%-28s median %7.2f us  best %7.2f us  (%5.1f%% of 6555)  parity %s\n", name, t[R / 2] * 1e3, t[0] * 1e3,
           bytes / (t[R / 2] * 1e-3) / 6555.2e9 * 100, ok ? "ok" : "FAIL");
    for (auto &e : ev) cudaEventDestroy(e);
}

int main(int argc, char **argv) {
    if (argc > 1 && std::string(argv[1]) == "cfg1") {
        NB = 1;
        C = 4096;
        HW = 4096;
    }
    N = (size_t)NB * C * HW;
    CK(cudaMemcpyToSymbol(d_NB, &NB, 4));
    CK(cudaMemcpyToSymbol(d_C, &C, 4));
    CK(cudaMemcpyToSymbol(d_HW, &HW, 4));
    printf("problem: %d x %d x %d f32 (C x HW -> HW x C per batch)\n", NB, C, HW);
    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    int l2 = 0;
    CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0));
    g_fn = (size_t)2 * l2 / 16;
    CK(cudaMalloc(&g_w, g_fn * 16));
    CK(cudaMalloc(&g_r, g_fn * 16));
    CK(cudaMemset(g_r, 0, g_fn * 16));
    CK(cudaMalloc(&g_sum, 4));
    float *din, *dout;
    CK(cudaMalloc(&din, N * 4));
    CK(cudaMalloc(&dout, N * 4));
    std::vector<float> hin(N), ref(N);
    for (size_t i = 0; i < N; ++i) hin[i] = (float)(i * 2654435761u % 1000003u);
    for (int n = 0; n < NB; ++n)
        for (int c = 0; c < C; ++c)
            for (int hw = 0; hw < HW; ++hw) ref[((size_t)n * HW + hw) * C + c] = hin[((size_t)n * C + c) * HW + hw];
    CK(cudaMemcpy(din, hin.data(), N * 4, cudaMemcpyHostToDevice));
    const double bytes = 2.0 * N * 4;
    std::vector<float> none;

    timeit("empty kernel (floor)", [&](cudaStream_t st) { fill_k<<<1, 32, 0, st>>>((float4 *)g_sum, 0); }, dout, none,
           s, bytes);
    timeit("copy 16B x4 (bound)", [&](cudaStream_t st) {
        size_t n4 = N / 4; copy_k<<<(unsigned)((n4 + 1023) / 1024), 256, 0, st>>>((const float4 *)din, (float4 *)dout, n4);
    }, dout, none, s, bytes);
    if (getenv("COPY_SWEEP")) {
        size_t n4 = N / 4;
        auto sweep = [&](auto kern, int U, int thr) {
            char nm[64]; snprintf(nm, 64, "copy U=%d thr=%d", U, thr);
            unsigned g = (unsigned)((n4 + (size_t)U * thr - 1) / ((size_t)U * thr));
            timeit(nm, [&](cudaStream_t st) { kern<<<g, thr, 0, st>>>((const float4 *)din, (float4 *)dout, n4); }, dout, none, s, bytes);
        };
        for (int thr : {128, 256, 512, 1024}) { sweep(copy_u<1>, 1, thr); sweep(copy_u<2>, 2, thr); sweep(copy_u<4>, 4, thr); sweep(copy_u<8>, 8, thr); sweep(copy_u<16>, 16, thr); }
        timeit("memcpy D2D", [&](cudaStream_t st) { cudaMemcpyAsync(dout, din, N * 4, cudaMemcpyDeviceToDevice, st); }, dout, none, s, bytes);
        return 0;
    }
    timeit("ldg tile 64x64", [&](cudaStream_t st) { ldg_tile_k<64><<<NB * (HW / 64) * (C / 64), 256, 0, st>>>(din, dout); },
           dout, ref, s, bytes);
    timeit("ldg tile 64x32", [&](cudaStream_t st) { ldg_tile_k<32><<<NB * (HW / 32) * (C / 64), 256, 0, st>>>(din, dout); },
           dout, ref, s, bytes);

    // TMA tensor map: 3-D {hw, c, n}, box {32, 64, 1}, SWIZZLE_128B
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q));
    CUtensorMap tm;
    cuuint64_t gdim[3] = {HW, C, NB};
    cuuint64_t gstr[2] = {(cuuint64_t)HW * 4, (cuuint64_t)HW * C * 4};
    cuuint32_t box[3] = {32, 64, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, din, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    const int ntiles = NB * (HW / 64) * (C / 64);
    auto tma = [&](auto kern, int stages, int grid, const char *name) {
        const int smem = stages * 16384 + 1024;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        timeit(name, [&](cudaStream_t st) { kern<<<grid, 256, smem, st>>>(tm, dout, ntiles); }, dout, ref, s, bytes);
    };
    tma(tma_tile_k<1>, 1, ntiles, "tma 1 tile/CTA");
    tma(tma_tile_k<2>, 2, (ntiles + 1) / 2, "tma 2 tiles/CTA (both up front)");
    tma(tma_tile_k<4>, 4, (ntiles + 3) / 4, "tma 4 tiles/CTA (all up front)");
    tma(tma_tile_k<2>, 2, 148 * 3, "tma persistent 444, S=2");
    tma(tma_tile_k<4>, 4, 148 * 3, "tma persistent 444, S=4");
    tma(tma_tile_k<4>, 4, 148 * 2, "tma persistent 296, S=4");
    tma(tma_tile_k<8>, 8, 148, "tma persistent 148, S=8");
    return 0;
}
