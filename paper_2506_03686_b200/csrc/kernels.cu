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
struct OuterEntry {
    int64_t g;
    uint32_t s;
    uint16_t c0, c1;
};

struct ThreadPart {
    int64_t g;
    uint32_t s;
    uint32_t c0, c1, c2;
    uint32_t grp;
    bool active;
};

template <int E>
__device__ __forceinline__ void cp_async(void *sp, const void *gp) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(sp);
    if constexpr (E == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gp) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(s), "l"(gp), "n"(E) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

__device__ __forceinline__ ThreadPart decode_thread(const PhaseDesc &d, uint32_t tid) {
    ThreadPart t;
    t.grp = tid / d.nthr;
    uint32_t tr = tid - t.grp * d.nthr;
    t.active = t.grp < d.ngroups;
    t.g = 0;
    t.s = 0;
    t.c0 = t.c1 = t.c2 = 0;
    for (int i = 0; i < d.nthr_dims; ++i) {
        uint32_t q = fdiv(tr, d.thr[i].div);
        uint32_t c = tr - q * d.thr[i].div.d;
        tr = q;
        t.g += (int64_t)c * d.thr[i].gstride;
        t.s += c * d.thr[i].sstride;
        const uint32_t cv = c * d.thr[i].cmul;
        if (d.thr[i].slot == 0) t.c0 = cv;
        else if (d.thr[i].slot == 1) t.c1 = cv;
        else if (d.thr[i].slot == 2) t.c2 = cv;
    }
    return t;
}

struct Lim {
    uint32_t l0, l1, l2;
};

__device__ __forceinline__ bool slot_ok(uint32_t mask, uint32_t c0, uint32_t c1, uint32_t c2, const Lim &lim) {
    return (!(mask & 1u) || c0 < lim.l0) && (!(mask & 2u) || c1 < lim.l1) && (!(mask & 4u) || c2 < lim.l2);
}

// R phase: global (source order) -> smem.  ASYNC: cp.async (16-byte chunks
// when d.vec > 1), else LDG+STS.
template <typename W, bool ASYNC, bool VEC>
__device__ __forceinline__ void tile_read_impl(const PhaseDesc &d, const ThreadPart &t, const unsigned char *smem,
                                               const W *__restrict__ gsrc, W *buf, uint32_t mask,
                                               const Lim lim) {
    constexpr int U = 4;
    constexpr int CP = VEC ? 16 : (int)sizeof(W);
    const OuterEntry *tab = reinterpret_cast<const OuterEntry *>(smem + d.off_tab);
    const uint32_t n_in = d.n_in;
    const int64_t g_in = d.g_in;
    const uint32_t s_in = d.s_in;
    for (uint32_t o = t.grp; o < d.n_outer; o += d.ngroups) {
        const OuterEntry e = tab[o];
        const W *gp = gsrc + (t.g + e.g);
        W *sp = buf + (t.s + e.s);
        if (mask == 0) {
            uint32_t i = 0;
            for (; i + U <= n_in; i += U) {
                if constexpr (ASYNC) {
#pragma unroll
                    for (int u = 0; u < U; ++u) cp_async<CP>(sp + u * s_in, gp + u * g_in);
                } else {
                    W v[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) v[u] = __ldg(gp + u * g_in);
#pragma unroll
                    for (int u = 0; u < U; ++u) sp[u * s_in] = v[u];
                }
                gp += U * g_in;
                sp += U * s_in;
            }
            for (; i < n_in; ++i) {
                if constexpr (ASYNC) cp_async<CP>(sp, gp);
                else *sp = __ldg(gp);
                gp += g_in;
                sp += s_in;
            }
        } else {
            uint32_t c0 = t.c0 + e.c0, c1 = t.c1 + e.c1, c2 = t.c2;
            for (uint32_t i = 0; i < n_in; ++i) {
                if (slot_ok(mask, c0, c1, c2, lim)) {
                    if constexpr (ASYNC) cp_async<CP>(sp, gp);
                    else *sp = __ldg(gp);
                }
                gp += g_in;
                sp += s_in;
                c0 += d.c_in[0];
                c1 += d.c_in[1];
                c2 += d.c_in[2];
            }
        }
    }
}

template <typename W, bool ASYNC>
__device__ __forceinline__ void tile_read(const PhaseDesc &d, const ThreadPart &t, const unsigned char *smem,
                                          const W *__restrict__ gsrc, W *buf, uint32_t mask,
                                          const Lim lim) {
    if (!t.active) return;
    if constexpr (ASYNC && sizeof(W) < 16) {
        if (d.vec > 1) {
            tile_read_impl<W, true, true>(d, t, smem, gsrc, buf, mask, lim);
            return;
        }
    }
    tile_read_impl<W, ASYNC, false>(d, t, smem, gsrc, buf, mask, lim);
}

// W phase: smem -> global (destination order).  VEC: each position is a
// 16-byte smem vector of V consecutive dim-0 elements, stored to V
// destinations d.vstride apart (each store instruction stays coalesced
// across the warp's lanes).
template <typename W, bool VEC>
__device__ __forceinline__ void tile_write_impl(const PhaseDesc &d, const ThreadPart &t, const unsigned char *smem,
                                                W *__restrict__ gdst, const W *buf, uint32_t mask,
                                                const Lim lim) {
    constexpr int U = VEC ? 2 : 4;
    constexpr int V = VEC ? 16 / (int)sizeof(W) : 1;
    const OuterEntry *tab = reinterpret_cast<const OuterEntry *>(smem + d.off_tab);
    const uint32_t n_in = d.n_in;
    const int64_t g_in = d.g_in;
    const uint32_t s_in = d.s_in;
    const int64_t vs = d.vstride;
    for (uint32_t o = t.grp; o < d.n_outer; o += d.ngroups) {
        const OuterEntry e = tab[o];
        W *gp = gdst + (t.g + e.g);
        const W *sp = buf + (t.s + e.s);
        if (mask == 0) {
            uint32_t i = 0;
            for (; i + U <= n_in; i += U) {
                if constexpr (VEC) {
                    uint4 v[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) v[u] = *reinterpret_cast<const uint4 *>(sp + u * s_in);
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const W *w = reinterpret_cast<const W *>(&v[u]);
#pragma unroll
                        for (int j = 0; j < V; ++j) gp[u * g_in + j * vs] = w[j];
                    }
                } else {
                    W v[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) v[u] = sp[u * s_in];
#pragma unroll
                    for (int u = 0; u < U; ++u) gp[u * g_in] = v[u];
                }
                gp += U * g_in;
                sp += U * s_in;
            }
            for (; i < n_in; ++i) {
                if constexpr (VEC) {
                    uint4 v = *reinterpret_cast<const uint4 *>(sp);
                    const W *w = reinterpret_cast<const W *>(&v);
#pragma unroll
                    for (int j = 0; j < V; ++j) gp[j * vs] = w[j];
                } else {
                    *gp = *sp;
                }
                gp += g_in;
                sp += s_in;
            }
        } else {
            uint32_t c0 = t.c0 + e.c0, c1 = t.c1 + e.c1, c2 = t.c2;
            for (uint32_t i = 0; i < n_in; ++i) {
                if (slot_ok(mask, c0, c1, c2, lim)) {
                    if constexpr (VEC) {
                        uint4 v = *reinterpret_cast<const uint4 *>(sp);
                        const W *w = reinterpret_cast<const W *>(&v);
#pragma unroll
                        for (int j = 0; j < V; ++j) gp[j * vs] = w[j];
                    } else {
                        *gp = *sp;
                    }
                }
                gp += g_in;
                sp += s_in;
                c0 += d.c_in[0];
                c1 += d.c_in[1];
                c2 += d.c_in[2];
            }
        }
    }
}

template <typename W>
__device__ __forceinline__ void tile_write(const PhaseDesc &d, const ThreadPart &t, const unsigned char *smem,
                                           W *__restrict__ gdst, const W *buf, uint32_t mask,
                                           const Lim lim) {
    if (!t.active) return;
    if constexpr (sizeof(W) == 4 || sizeof(W) == 8) {
        if (d.vec > 1) {
            tile_write_impl<W, true>(d, t, smem, gdst, buf, mask, lim);
            return;
        }
    }
    tile_write_impl<W, false>(d, t, smem, gdst, buf, mask, lim);
}

// Warp 0 decodes tile `t` into slot `k`: source/destination base offsets and
// the valid extents of the ragged boundary dims a and c.
__device__ __forceinline__ void decode_tile(const TileParams &p, uint32_t t, int64_t (*s_base)[2],
                                            uint32_t (*s_valid)[2], int k) {
    const uint32_t lane = threadIdx.x & 31;
    int64_t sb = 0, db = 0;
    uint32_t va = p.e_a, vc = p.e_c;
    for (int i = (int)lane; i < p.ngrid; i += 32) {
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
    if (lane == 0) {
        s_base[k][0] = sb;
        s_base[k][1] = db;
        s_valid[k][0] = va;
        s_valid[k][1] = vc;
    }
}

template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
// wait until at most n committed cp.async groups are pending (n < 8)
__device__ __forceinline__ void cp_async_wait_pending(uint32_t n) {
    switch (n) {
        case 0: cp_async_wait_group<0>(); break;
        case 1: cp_async_wait_group<1>(); break;
        case 2: cp_async_wait_group<2>(); break;
        case 3: cp_async_wait_group<3>(); break;
        case 4: cp_async_wait_group<4>(); break;
        case 5: cp_async_wait_group<5>(); break;
        case 6: cp_async_wait_group<6>(); break;
        default: cp_async_wait_group<7>(); break;
    }
}

constexpr int kMaxStages = 8;
constexpr int kRing = kMaxStages + 2;

// Persistent CTAs walk tiles t_k = blockIdx.x + k*gridDim.x through an
// S-stage cp.async pipeline (S = p.nbuf smem tile buffers): the prologue
// streams the source runs of the first S tiles; each iteration writes tile
// k out of its buffer and refills that buffer with tile k+S.  Small
// problems are thereby staged in one wave; large ones keep S-1 tiles of
// loads in flight per CTA.  Without ASYNC (1- and 2-byte words) a single
// buffer is filled by LDG+STS.
template <typename W, bool ASYNC>
__global__ void __launch_bounds__(256) tile_kernel(const __grid_constant__ TileParams p,
                                                   const W *__restrict__ src, W *__restrict__ dst) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int64_t s_base[kRing][2];
    __shared__ uint32_t s_valid[kRing][2];
    const uint32_t tid = threadIdx.x, NT = blockDim.x;
    const uint32_t first = blockIdx.x, step = gridDim.x;
    if (first >= p.num_tiles) return;
    const uint32_t cnt = (p.num_tiles - first + step - 1) / step;   // tiles of this CTA
    const uint32_t S = ASYNC ? p.nbuf : 1u;
    const uint32_t R = S + 2;

    // per-CTA outer tables of both phases
    for (int ph = 0; ph < 2; ++ph) {
        const PhaseDesc &d = p.ph[ph];
        OuterEntry *tab = reinterpret_cast<OuterEntry *>(smem + d.off_tab);
        for (uint32_t o = tid; o < d.n_outer; o += NT) {
            uint32_t idx = o, s = 0, c0 = 0, c1 = 0;
            int64_t g = 0;
            for (int i = 0; i < d.nout_dims; ++i) {
                uint32_t q = fdiv(idx, d.out[i].div);
                uint32_t c = idx - q * d.out[i].div.d;
                idx = q;
                g += (int64_t)c * d.out[i].gstride;
                s += c * d.out[i].sstride;
                if (d.out[i].slot == 0) c0 = c * d.out[i].cmul;
                else if (d.out[i].slot == 1) c1 = c * d.out[i].cmul;
            }
            OuterEntry e;
            e.g = g;
            e.s = s;
            e.c0 = (uint16_t)c0;
            e.c1 = (uint16_t)c1;
            tab[o] = e;
        }
    }
    const ThreadPart tr = decode_thread(p.ph[0], tid);
    const ThreadPart tw = decode_thread(p.ph[1], tid);
    W *const buf0 = reinterpret_cast<W *>(smem + p.off_buf);
    const size_t bstride = ((size_t)p.tile_elems_alloc * sizeof(W) + 15) / 16 * 16 / sizeof(W);

    if (tid < 32)
        for (uint32_t j = 0; j < S && j < cnt; ++j) decode_tile(p, first + j * step, s_base, s_valid, (int)j);
    __syncthreads();
    auto limits = [&](uint32_t slot, int ph, Lim &lim) -> uint32_t {
        const uint32_t va = s_valid[slot][0], vc = s_valid[slot][1];
        lim.l0 = va;
        lim.l1 = vc;
        lim.l2 = p.lim_split[ph];
        const bool full = (va == p.e_a) && (vc == p.e_c);
        return full ? p.ph[ph].mask_full : p.ph[ph].mask_ragged;
    };
    auto load = [&](uint32_t k, W *b) {
        Lim lim;
        const uint32_t slot = k % R;
        const uint32_t m = limits(slot, 0, lim);
        tile_read<W, ASYNC>(p.ph[0], tr, smem, src + s_base[slot][0], b, m, lim);
    };
    // prologue: fill every stage
    for (uint32_t j = 0; j < S; ++j) {
        if (j < cnt) load(j, buf0 + j * bstride);
        if constexpr (ASYNC) cp_async_commit();
    }
    for (uint32_t k = 0; k < cnt; ++k) {
        if (tid < 32 && k + S < cnt) decode_tile(p, first + (k + S) * step, s_base, s_valid, (int)((k + S) % R));
        if constexpr (ASYNC) cp_async_wait_pending(S - 1);
        __syncthreads();
        W *b = buf0 + (k % S) * bstride;
        {
            Lim lim;
            const uint32_t slot = k % R;
            const uint32_t m = limits(slot, 1, lim);
            tile_write<W>(p.ph[1], tw, smem, dst + s_base[slot][1], b, m, lim);
        }
        __syncthreads();
        if (k + S < cnt) load(k + S, b);
        if constexpr (ASYNC) cp_async_commit();
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
        int optin = 0;
        if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || optin <= 0)
            optin = 227 * 1024;
        cudaFuncAttributes fa;
        size_t stat = cudaFuncGetAttributes(&fa, kernel) == cudaSuccess ? fa.sharedSizeBytes : 1024;
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)stat);
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
    const int smem = (int)p->tile.smem_bytes;
    auto launch = [&](auto k) {
        int nb = occupancy(k, p->threads, smem);
        int64_t grid = p->tile.num_tiles;
        if (p->tile.persistent) grid = std::min<int64_t>(grid, (int64_t)nb * sm_count_for_current());
        if (grid < 1) grid = 1;
        const TileParams &tp = (p->tile.ph[0].vec > 1 && ((uintptr_t)src % 16)) ? p->tile_unaligned : p->tile;
        k<<<(unsigned)grid, p->threads, smem, st>>>(tp, (const W *)src, (W *)dst);
    };
    if constexpr (E >= 4) {
        launch(tile_kernel<W, true>);
        return VPG_OK;
    }
    if constexpr (E < 4) launch(tile_kernel<W, false>);
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
