// kernels.cu -- sm_100a kernels for general N-D tensor permutation.
//
// These replace the reference's CPU execution chain (butterfly shuffles,
// IR, emitted SIMD C: /root/reference/pkg/src/vecperm/shuffle.py:246-589,
// ir.py:171-456, emit.py:212-340).  Pure data movement: every kernel is
// bounded by HBM bandwidth, so the design goals are full 32-byte sectors on
// both sides, enough bytes in flight per SM, and few instructions per byte.
//
//   copy_kernel    merged rank 1 (identity): 16-byte vector grid-stride copy
//   rows_kernel    K1: stride-1 preserved, long rows: one thread group per
//                  destination row, 16-byte vectors, source row found by a
//                  mixed-radix decode of the row index (fast divmod)
//   tile_kernel    K2/K3: persistent CTAs walk tiles; each tile is read as
//                  contiguous source runs into padded shared memory and
//                  written as contiguous destination runs.  Run tables are
//                  built once per CTA; ragged boundary tiles are predicated
//                  (no read-modify-write, unlike the reference's "reserve"
//                  stores, shuffle.py:555-580, which would race across CTAs)
//   gather_kernel  K0: out[i] = in[f(i)] per element (core.py:173-178)
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "plan.h"

namespace vpg {

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv &f) {
    uint32_t t = __umulhi(n, f.m);
    return (uint32_t)(((uint64_t)t + n) >> f.s);
}

template <int E>
struct WordOf;
template <>
struct WordOf<1> {
    using T = unsigned char;
};
template <>
struct WordOf<2> {
    using T = unsigned short;
};
template <>
struct WordOf<4> {
    using T = unsigned int;
};
template <>
struct WordOf<8> {
    using T = unsigned long long;
};
template <>
struct WordOf<16> {
    using T = uint4;
};

template <typename W>
__device__ __forceinline__ W ld_stream(const W *p) {
    return __ldg(p);
}

// ------------------------------------------------------------------ COPY
template <typename V>
__global__ void __launch_bounds__(256) copy_kernel(const V *__restrict__ src, V *__restrict__ dst,
                                                   int64_t nvec) {
    constexpr int U = 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < nvec; i += U * stride) {
        V r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) r[u] = ld_stream(src + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) dst[i + u * stride] = r[u];
    }
    for (; i < nvec; i += stride) dst[i] = ld_stream(src + i);
}

// ------------------------------------------------------------------ ROWS (K1)
template <typename V>
__global__ void __launch_bounds__(256) rows_kernel(const __grid_constant__ RowsParams p,
                                                   const V *__restrict__ src, V *__restrict__ dst,
                                                   uint32_t vec_log2) {
    constexpr int U = 4;
    const uint32_t tpr = 1u << p.tpr_log2;
    const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t lane = gtid & (tpr - 1);
    const uint32_t ngroups = (gridDim.x * blockDim.x) >> p.tpr_log2;
    const uint32_t rv = p.row_vecs;
    for (uint32_t q = gtid >> p.tpr_log2; q < p.nrows; q += ngroups) {
        uint32_t rem = q;
        int64_t so = 0;
        for (int i = 0; i < p.ndig; ++i) {
            uint32_t qq = fdiv(rem, p.dig[i].ext);
            so += (int64_t)(rem - qq * p.dig[i].ext.d) * p.dig[i].src_stride;
            rem = qq;
        }
        const V *s = src + (so >> vec_log2);
        V *d = dst + (int64_t)q * rv;
        uint32_t i = lane;
        for (; i + (U - 1) * tpr < rv; i += U * tpr) {
            V r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) r[u] = ld_stream(s + i + u * tpr);
#pragma unroll
            for (int u = 0; u < U; ++u) d[i + u * tpr] = r[u];
        }
        for (; i < rv; i += tpr) d[i] = ld_stream(s + i);
    }
}

// ------------------------------------------------------------------ TILE (K2/K3)
template <typename W>
__global__ void __launch_bounds__(256) tile_kernel(const __grid_constant__ TileParams p,
                                                   const W *__restrict__ src, W *__restrict__ dst) {
    constexpr int U = 8;
    extern __shared__ __align__(16) unsigned char smem[];
    int64_t *S_off = reinterpret_cast<int64_t *>(smem + p.off_S_off);
    int64_t *W_off = reinterpret_cast<int64_t *>(smem + p.off_W_off);
    uint32_t *W_sm = reinterpret_cast<uint32_t *>(smem + p.off_W_sm);
    uint32_t *A_sm = reinterpret_cast<uint32_t *>(smem + p.off_A);
    uint32_t *S_c = reinterpret_cast<uint32_t *>(smem + p.off_S_c);
    uint32_t *W_a = reinterpret_cast<uint32_t *>(smem + p.off_W_a);
    W *tile = reinterpret_cast<W *>(smem + p.off_tile);
    __shared__ int64_t s_base[2];
    __shared__ uint32_t s_valid[2];

    const uint32_t tid = threadIdx.x, NT = blockDim.x;

    // ---- per-CTA run tables (identical for every tile)
    for (uint32_t r = tid; r < p.Ns; r += NT) {
        uint32_t idx = r, cc = 0;
        int64_t off = 0;
        for (int i = 0; i < p.nS; ++i) {
            uint32_t q = fdiv(idx, p.S[i].div);
            uint32_t c = idx - q * p.S[i].extent;
            idx = q;
            off += (int64_t)c * p.S[i].gstride;
            if (i == p.s_c_dim) cc = c;
        }
        S_off[r] = off;
        if (p.s_c_dim >= 0) S_c[r] = cc;
    }
    for (uint32_t r = tid; r < p.Nd; r += NT) {
        uint32_t idx = r, ca = 0, sm = 0;
        int64_t off = 0;
        for (int i = 0; i < p.nW; ++i) {
            uint32_t q = fdiv(idx, p.W[i].div);
            uint32_t c = idx - q * p.W[i].extent;
            idx = q;
            off += (int64_t)c * p.W[i].gstride;
            sm += c * p.W[i].sstride;
            if (i == p.w_a_dim) ca = c;
        }
        W_off[r] = off;
        W_sm[r] = sm;
        if (p.w_a_dim >= 0) W_a[r] = ca;
    }
    for (uint32_t c0 = tid; c0 < p.Ld; c0 += NT) {
        uint32_t idx = c0, sm = 0;
        for (int i = 0; i < p.nA; ++i) {
            uint32_t q = fdiv(idx, p.A[i].div);
            sm += (idx - q * p.A[i].extent) * p.A[i].sstride;
            idx = q;
        }
        A_sm[c0] = sm;
    }

    // ---- incremental (run, column) walkers: v advances by NT per step
    const uint32_t r0 = tid / p.Ls, c0 = tid - r0 * p.Ls;
    const uint32_t dR = NT / p.Ls, dC = NT - dR * p.Ls;
    const uint32_t q0 = tid / p.Ld, k0 = tid - q0 * p.Ld;
    const uint32_t dQ = NT / p.Ld, dK = NT - dQ * p.Ld;

    for (uint32_t t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        if (tid < 32) {
            int64_t sb = 0, db = 0;
            uint32_t va = p.e_a, vc = p.e_c;
            for (int i = (int)tid; i < p.ngrid; i += 32) {
                uint32_t q = fdiv(t, p.grid[i].cum);
                uint32_t c = q - fdiv(q, p.grid[i].ext) * p.grid[i].ext.d;
                sb += (int64_t)c * p.grid[i].src_stride;
                db += (int64_t)c * p.grid[i].dst_stride;
                if (i == p.grid_a) va = min(p.e_a, p.d_a - c * p.e_a);
                if (i == p.grid_c) vc = min(p.e_c, p.d_c - c * p.e_c);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                sb += __shfl_xor_sync(0xffffffffu, sb, o);
                db += __shfl_xor_sync(0xffffffffu, db, o);
                va = min(va, __shfl_xor_sync(0xffffffffu, va, o));
                vc = min(vc, __shfl_xor_sync(0xffffffffu, vc, o));
            }
            if (tid == 0) {
                s_base[0] = sb;
                s_base[1] = db;
                s_valid[0] = va;
                s_valid[1] = vc;
            }
        }
        __syncthreads();
        const int64_t sb = s_base[0], db = s_base[1];
        const uint32_t va = s_valid[0], vc = s_valid[1];
        const bool full = (va == p.e_a) && (vc == p.e_c);
        const uint32_t Ls_valid = (va == p.e_a) ? p.Ls : p.Ls_unit * va;
        const uint32_t Ld_valid = (vc == p.e_c) ? p.Ld : p.Ld_unit * vc;

        // ---- read phase: contiguous source runs -> smem (source order, padded pitch)
        {
            const W *sp = src + sb;
            uint32_t r = r0, c = c0;
            for (uint32_t v = tid; v < p.T; v += NT * U) {
                W reg[U];
                uint32_t sidx[U];
                bool ok[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t vv = v + u * NT;
                    bool valid = vv < p.T;
                    if (valid && !full)
                        valid = (c < Ls_valid) && (p.s_c_dim < 0 || S_c[r] < vc);
                    ok[u] = valid;
                    sidx[u] = r * p.pitch + c;
                    if (valid) reg[u] = ld_stream(sp + S_off[r] + c);
                    c += dC;
                    r += dR;
                    if (c >= p.Ls) {
                        c -= p.Ls;
                        ++r;
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (ok[u]) tile[sidx[u]] = reg[u];
            }
        }
        __syncthreads();
        // ---- write phase: smem -> contiguous destination runs
        {
            W *dp = dst + db;
            uint32_t q = q0, k = k0;
            for (uint32_t v = tid; v < p.T; v += NT * U) {
                W reg[U];
                int64_t didx[U];
                bool ok[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t vv = v + u * NT;
                    bool valid = vv < p.T;
                    if (valid && !full)
                        valid = (k < Ld_valid) && (p.w_a_dim < 0 || W_a[q] < va);
                    ok[u] = valid;
                    if (valid) {
                        reg[u] = tile[W_sm[q] + A_sm[k]];
                        didx[u] = W_off[q] + k;
                    }
                    k += dK;
                    q += dQ;
                    if (k >= p.Ld) {
                        k -= p.Ld;
                        ++q;
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (ok[u]) dp[didx[u]] = reg[u];
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ GATHER (K0)
template <typename W>
__global__ void __launch_bounds__(256) gather_kernel(const __grid_constant__ GatherParams p,
                                                     const W *__restrict__ src, W *__restrict__ dst) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < p.n; i += gridDim.x * blockDim.x) {
        uint32_t rem = i;
        int64_t s = 0;
        for (int j = 0; j < p.rank; ++j) {
            uint32_t q = fdiv(rem, p.ext[j]);
            s += (int64_t)(rem - q * p.ext[j].d) * p.src_stride[j];
            rem = q;
        }
        dst[i] = src[s];
    }
}

// ------------------------------------------------------------------ launch
namespace {

std::mutex g_mu;
std::map<int, int> g_sm_count;
std::map<std::tuple<const void *, int, int>, int> g_occ;
std::map<const void *, bool> g_attr_set;

int sm_count_for_current() {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_sm_count.find(dev);
    if (it != g_sm_count.end()) return it->second;
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    g_sm_count[dev] = n;
    return n;
}

template <typename K>
int occupancy(K kernel, int threads, int smem) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_mu);
    auto key = std::make_tuple((const void *)kernel, threads, smem + (dev << 24));
    auto it = g_occ.find(key);
    if (it != g_occ.end()) return it->second;
    if (!g_attr_set[(const void *)kernel]) {
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        g_attr_set[(const void *)kernel] = true;
    }
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, smem) != cudaSuccess || nb < 1)
        nb = 1;
    g_occ[key] = nb;
    return nb;
}

template <int E>
vpg_status launch_tile(const vpg_plan *p, const void *src, void *dst, cudaStream_t st) {
    using W = typename WordOf<E>::T;
    auto k = tile_kernel<W>;
    const int smem = (int)p->tile.smem_bytes;
    int nb = occupancy(k, p->threads, smem);
    int64_t grid = std::min<int64_t>(p->tile.num_tiles, (int64_t)nb * sm_count_for_current());
    if (grid < 1) grid = 1;
    k<<<(unsigned)grid, p->threads, smem, st>>>(p->tile, (const W *)src, (W *)dst);
    return VPG_OK;
}

template <int E>
vpg_status launch_gather(const vpg_plan *p, const void *src, void *dst, cudaStream_t st) {
    using W = typename WordOf<E>::T;
    int64_t grid = std::min<int64_t>((p->gather.n + 255) / 256, (int64_t)sm_count_for_current() * 8);
    if (grid < 1) grid = 1;
    gather_kernel<W><<<(unsigned)grid, 256, 0, st>>>(p->gather, (const W *)src, (W *)dst);
    return VPG_OK;
}

int ptr_align(const void *a, const void *b) {
    uintptr_t x = (uintptr_t)a | (uintptr_t)b;
    int al = 16;
    while (al > 1 && (x % al)) al >>= 1;
    return al;
}

vpg_status launch_rows(const vpg_plan *p, const void *src, void *dst, cudaStream_t st) {
    RowsParams rp = p->rows;
    const int E = p->elem_bytes;
    uint32_t V = rp.vec;
    int al = ptr_align(src, dst);
    while (V > 1 && (int)(V * E) > al) V >>= 1;
    if (V != rp.vec) {
        rp.row_vecs = (uint32_t)(rp.row_len / V);
        uint32_t tpr = 32;
        while (tpr > 1 && tpr / 2 >= rp.row_vecs) tpr >>= 1;
        rp.tpr_log2 = 0;
        while ((1u << rp.tpr_log2) < tpr) ++rp.tpr_log2;
        rp.vec = V;
    }
    uint32_t vlog = 0;
    while ((1u << vlog) < V) ++vlog;
    const int vb = (int)(V * E);
    int64_t need = ((int64_t)rp.nrows << rp.tpr_log2) + 255;
    need /= 256;
#define VPG_ROWS_CASE(BYTES, TYPE)                                                             \
    case BYTES: {                                                                              \
        auto k = rows_kernel<TYPE>;                                                            \
        int nb = occupancy(k, 256, 0);                                                         \
        int64_t grid = std::min<int64_t>(need, (int64_t)nb * sm_count_for_current());          \
        if (grid < 1) grid = 1;                                                                \
        k<<<(unsigned)grid, 256, 0, st>>>(rp, (const TYPE *)src, (TYPE *)dst, vlog);           \
        return VPG_OK;                                                                         \
    }
    switch (vb) {
        VPG_ROWS_CASE(1, unsigned char)
        VPG_ROWS_CASE(2, unsigned short)
        VPG_ROWS_CASE(4, unsigned int)
        VPG_ROWS_CASE(8, unsigned long long)
        VPG_ROWS_CASE(16, uint4)
        default:
            return VPG_EUNSUPPORTED;
    }
#undef VPG_ROWS_CASE
}

vpg_status launch_copy(const vpg_plan *p, const void *src, void *dst, cudaStream_t st) {
    int64_t nbytes = p->copy.n * p->elem_bytes;
    int al = ptr_align(src, dst);
    while (al > 1 && (nbytes % al)) al >>= 1;
    int64_t nvec = nbytes / al;
    int64_t grid = std::min<int64_t>((nvec + 255) / 256, (int64_t)sm_count_for_current() * 8);
    if (grid < 1) grid = 1;
    switch (al) {
        case 16: copy_kernel<uint4><<<(unsigned)grid, 256, 0, st>>>((const uint4 *)src, (uint4 *)dst, nvec); break;
        case 8: copy_kernel<unsigned long long><<<(unsigned)grid, 256, 0, st>>>((const unsigned long long *)src, (unsigned long long *)dst, nvec); break;
        case 4: copy_kernel<unsigned int><<<(unsigned)grid, 256, 0, st>>>((const unsigned int *)src, (unsigned int *)dst, nvec); break;
        case 2: copy_kernel<unsigned short><<<(unsigned)grid, 256, 0, st>>>((const unsigned short *)src, (unsigned short *)dst, nvec); break;
        default: copy_kernel<unsigned char><<<(unsigned)grid, 256, 0, st>>>((const unsigned char *)src, (unsigned char *)dst, nvec); break;
    }
    return VPG_OK;
}

}  // namespace

int device_sm_count() { return sm_count_for_current(); }

vpg_status launch_plan(const vpg_plan *p, const void *src, void *dst, void *stream, std::string *err) {
    cudaStream_t st = (cudaStream_t)stream;
    const int E = p->elem_bytes;
    if (((uintptr_t)src % E) || ((uintptr_t)dst % E)) {
        *err = "buffers must be aligned to the element width";
        return VPG_EINVAL;
    }
    if (p->n == 0) return VPG_OK;
    vpg_status s = VPG_OK;
    switch (p->kernel_class) {
        case VPG_KERNEL_COPY:
            s = launch_copy(p, src, dst, st);
            break;
        case VPG_KERNEL_ROWS:
            s = launch_rows(p, src, dst, st);
            break;
        case VPG_KERNEL_TILE:
            switch (E) {
                case 1: s = launch_tile<1>(p, src, dst, st); break;
                case 2: s = launch_tile<2>(p, src, dst, st); break;
                case 4: s = launch_tile<4>(p, src, dst, st); break;
                case 8: s = launch_tile<8>(p, src, dst, st); break;
                case 16: s = launch_tile<16>(p, src, dst, st); break;
                default: s = VPG_EUNSUPPORTED;
            }
            break;
        case VPG_KERNEL_GATHER:
            switch (E) {
                case 1: s = launch_gather<1>(p, src, dst, st); break;
                case 2: s = launch_gather<2>(p, src, dst, st); break;
                case 4: s = launch_gather<4>(p, src, dst, st); break;
                case 8: s = launch_gather<8>(p, src, dst, st); break;
                case 16: s = launch_gather<16>(p, src, dst, st); break;
                default: s = VPG_EUNSUPPORTED;
            }
            break;
        default:
            s = VPG_EUNSUPPORTED;
    }
    if (s != VPG_OK) {
        *err = "unsupported plan/element width";
        return s;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        *err = std::string("kernel launch failed: ") + cudaGetErrorString(e);
        return VPG_ECUDA;
    }
    return VPG_OK;
}

}  // namespace vpg
