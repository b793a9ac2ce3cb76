// ldgsts_probe.cu -- how the R-phase load form affects L2 sector requests
// and time: a 1 GiB copy global -> smem -> global by 256-thread CTAs, 8 KiB
// per CTA step, four load forms:
//   0: cp.async.cg 16 B per lane, lanes on consecutive 16 B  (tile kernel today)
//   1: cp.async.cg 2 x 16 B per lane, each lane owns whole 32 B sectors
//   2: cp.async.ca 16 B per lane (L1-allocating)
//   3: ld.global.v4 + st.shared.v4 (registers)
//   4: cp.async.cg 16 B per lane in 64-row x 256-byte tiles of a matrix with
//      RW-byte rows (each warp instruction: 2 rows x 256 B, as the tile
//      kernel's R phase on cfg2); 5: the same with 16 rows x 1 KiB;
//      6: 64 rows x 256 B of 64 KiB rows; 7-9: 512-byte smem rows padded by
//      16 / 32 / 128 bytes; 10: 16-byte chunks XOR-swizzled by row within
//      each 128-byte block
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o ldgsts_probe tools/ldgsts_probe.cu
// Run under ncu --metrics lts__t_sectors_srcunit_tex_op_read.sum,gpu__time_duration.sum
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

// tiles of ROWS rows x (8192 / ROWS) bytes from a matrix with rw16 16-byte chunks per row
template <int ROWS>
__global__ void __launch_bounds__(256) probe_tile(const uint4 *__restrict__ src, uint4 *__restrict__ dst, size_t nvec,
                                                  size_t rw16) {
    __shared__ __align__(16) uint4 buf[512];
    constexpr int CPR = 512 / ROWS;           // chunks per tile row
    const int t = threadIdx.x;
    const size_t nrows = nvec / rw16, tiles_c = rw16 / CPR, tiles = (nrows / ROWS) * tiles_c;
    for (size_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const size_t r0 = (tile / tiles_c) * ROWS, c0 = (tile % tiles_c) * CPR;
        for (int k = 0; k < 2; ++k) {
            const int i = t + 256 * k, r = i / CPR, c = i % CPR;
            const uint32_t s = (uint32_t)__cvta_generic_to_shared(&buf[i]);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src + (r0 + r) * rw16 + c0 + c)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::: "memory");
        __syncthreads();
        dst[tile * 512 + t] = buf[t];
        dst[tile * 512 + t + 256] = buf[t + 256];
        __syncthreads();
    }
}

// 8 KiB steps staged in smem rows of 512 B plus PAD16 x 16 B of padding
// (the tile kernel pads its rows against W-phase bank conflicts)
template <int PAD16>
__global__ void __launch_bounds__(256) probe_pad(const uint4 *__restrict__ src, uint4 *__restrict__ dst, size_t nvec) {
    __shared__ __align__(16) uint4 buf[16 * (32 + PAD16)];
    const int t = threadIdx.x;
    for (size_t base = (size_t)blockIdx.x * 512; base < nvec; base += (size_t)gridDim.x * 512) {
        for (int k = 0; k < 2; ++k) {
            const int i = t + 256 * k, r = i / 32, c = i % 32;
            const uint32_t s = (uint32_t)__cvta_generic_to_shared(&buf[r * (32 + PAD16) + c]);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src + base + i) : "memory");
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::: "memory");
        __syncthreads();
        for (int k = 0; k < 2; ++k) {
            const int i = t + 256 * k, r = i / 32, c = i % 32;
            dst[base + i] = buf[r * (32 + PAD16) + c];
        }
        __syncthreads();
    }
}

// 512-byte smem rows, 16-byte chunks XOR-swizzled by row inside each 128-byte block
__global__ void __launch_bounds__(256) probe_xor(const uint4 *__restrict__ src, uint4 *__restrict__ dst, size_t nvec) {
    __shared__ __align__(128) uint4 buf[512];
    const int t = threadIdx.x;
    for (size_t base = (size_t)blockIdx.x * 512; base < nvec; base += (size_t)gridDim.x * 512) {
        for (int k = 0; k < 2; ++k) {
            const int i = t + 256 * k, r = i / 32, c = i % 32;
            const int pc = (c & ~7) | ((c ^ r) & 7);
            const uint32_t s = (uint32_t)__cvta_generic_to_shared(&buf[r * 32 + pc]);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src + base + i) : "memory");
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::: "memory");
        __syncthreads();
        for (int k = 0; k < 2; ++k) {
            const int i = t + 256 * k, r = i / 32, c = i % 32;
            dst[base + i] = buf[r * 32 + ((c & ~7) | ((c ^ r) & 7))];
        }
        __syncthreads();
    }
}

template <int MODE>
__global__ void __launch_bounds__(256) probe(const uint4 *__restrict__ src, uint4 *__restrict__ dst, size_t nvec) {
    __shared__ __align__(16) uint4 buf[512];   // 8 KiB
    const int t = threadIdx.x;
    for (size_t base = (size_t)blockIdx.x * 512; base < nvec; base += (size_t)gridDim.x * 512) {
        if (MODE == 0 || MODE == 2) {
            for (int k = 0; k < 2; ++k) {
                const int i = t + 256 * k;
                const uint32_t s = (uint32_t)__cvta_generic_to_shared(&buf[i]);
                if (MODE == 0)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src + base + i) : "memory");
                else
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src + base + i) : "memory");
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::: "memory");
        } else if (MODE == 1) {
            const int i = 2 * t;
            for (int k = 0; k < 2; ++k) {
                const uint32_t s = (uint32_t)__cvta_generic_to_shared(&buf[i + k]);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src + base + i + k) : "memory");
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::: "memory");
        } else {
            uint4 v0 = src[base + t], v1 = src[base + t + 256];
            buf[t] = v0;
            buf[t + 256] = v1;
        }
        __syncthreads();
        dst[base + t] = buf[t];
        dst[base + t + 256] = buf[t + 256];
        __syncthreads();
    }
}

int main() {
    const size_t bytes = (size_t)1 << 30, nvec = bytes / 16;
    uint4 *a, *b;
    cudaMalloc(&a, bytes);
    cudaMalloc(&b, bytes);
    cudaMemset(a, 1, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * 8;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 11; ++mode) {
        for (int rep = 0; rep < 4; ++rep) {
            cudaEventRecord(e0);
            switch (mode) {
                case 0: probe<0><<<grid, 256>>>(a, b, nvec); break;
                case 1: probe<1><<<grid, 256>>>(a, b, nvec); break;
                case 2: probe<2><<<grid, 256>>>(a, b, nvec); break;
                case 4: probe_tile<64><<<grid, 256>>>(a, b, nvec, 12544 / 16 * 4); break;
                case 5: probe_tile<16><<<grid, 256>>>(a, b, nvec, 12544 / 16 * 4); break;
                case 6: probe_tile<64><<<grid, 256>>>(a, b, nvec, 4096); break;
                case 7: probe_pad<1><<<grid, 256>>>(a, b, nvec); break;
                case 8: probe_pad<2><<<grid, 256>>>(a, b, nvec); break;
                case 9: probe_pad<8><<<grid, 256>>>(a, b, nvec); break;
                case 10: probe_xor<<<grid, 256>>>(a, b, nvec); break;
                default: probe<3><<<grid, 256>>>(a, b, nvec); break;
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep == 3) printf("mode %d: %.1f us  %.0f GB/s\n", mode, ms * 1e3, 2.0 * bytes / (ms * 1e-3) / 1e9);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
