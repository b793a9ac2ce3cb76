// tile_body.cuh -- the K2/K3 tile transpose, shared by the ahead-of-time
// kernel (kernels.cu, parameters as a __grid_constant__ argument) and the
// run-time specialised kernels (jit.cpp: NVRTC, parameters baked in as
// constant bytes with VPG_JIT defined, so extents/strides/divisors fold to
// immediates and the per-thread walks unroll).  Device code only.
#pragma once

#include "plan_params.h"

#ifdef VPG_JIT
#define VPG_UNROLL _Pragma("unroll")
#else
#define VPG_UNROLL
#endif
#define VPG_PRAGMA(x) _Pragma(#x)
// scalar W walk: shared-memory loads issued ahead of their stores, per batch
#ifndef VPG_W_U
#define VPG_W_U 4
#endif
#define VPG_UNROLL_N(n) VPG_PRAGMA(unroll n)

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

// ------------------------------------------------------------------ TILE (K2/K3)
struct OuterEntry {
    int64_t g;
    uint32_t s;
    uint16_t c0, c1;
    uint32_t h;          // shifted-run mode: source-alignment shift contribution
    uint32_t pad_;
};
static_assert(sizeof(OuterEntry) == kOuterEntryBytes, "planner sizes the smem tables with kOuterEntryBytes");

struct ThreadPart {
    int64_t g;
    uint32_t s;
    uint32_t c0, c1, c2;
    uint32_t h;
    uint32_t grp;
    bool active;
};

// VPG_HINTS (specialised kernels, experiments): bit 1 = streaming (.cs)
// destination stores.  (Bit 0, L2 evict_first cp.async reads, was removed:
// it measured no gain in round 1 and its cache-hinted cp.async faulted with
// an illegal-instruction error on sm_100a in round 2.)
#ifndef VPG_HINTS
#define VPG_HINTS 0
#endif

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// cp.async of E bytes to the shared-window address s
template <int E>
__device__ __forceinline__ void cp_async(uint32_t s, const void *gp) {
    if constexpr (E == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gp) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(s), "l"(gp), "n"(E) : "memory");
}

template <typename W>
__device__ __forceinline__ void st_out(W *p, const W &v) {
#if VPG_HINTS & 2
    if constexpr (sizeof(W) >= 4) __stcs(p, v);
    else *p = v;
#else
    *p = v;
#endif
}
// Programmatic dependent launch (PDL): a launch with the programmatic
// stream-serialisation attribute may start while the previous kernel on
// the stream is still draining.  Every kernel here triggers its dependents
// at entry (the dependent grid can only start once every CTA of this grid
// has started, so a one-wave grid never loses SM slots to it) and waits for
// the previous grid's completion -- and the visibility of its memory --
// before its first global-memory access.  Without the attribute both are
// no-ops.
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

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
    t.h = 0;
    VPG_UNROLL
    for (int i = 0; i < kMaxPhaseDims; ++i) {
        if (i >= d.nthr_dims) break;
        uint32_t q = fdiv(tr, d.thr[i].div);
        uint32_t c = tr - q * d.thr[i].div.d;
        tr = q;
        t.g += (int64_t)c * d.thr[i].gstride;
        t.s += c * d.thr[i].sstride;
        t.h += c * d.thr[i].hmul;
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

// Physical smem element offset of logical offset s under the chunk swizzle
// (V elements per 16-byte chunk).
template <int V>
__device__ __forceinline__ uint32_t swizzle(const PhaseDesc &d, uint32_t s) {
    const uint32_t r = fdiv(s, d.spitch);
    const uint32_t c = s - r * d.spitch.d;
    const uint32_t f = (r >> (d.swz - 1)) & 7u;
    return r * d.spitch.d + ((((c / V) ^ f) * V) | (c % V));
}

// Address swizzle (PhaseDesc::swz == kSwzAddr): the 16-byte chunk index
// inside each 128-byte block of shared memory XOR the block index (mod 8),
// applied to the byte offset from the 128-byte aligned dynamic smem base,
// so it needs no row structure: the residue layouts use it.
__device__ __forceinline__ uint32_t swz_off(uint32_t a) { return a ^ (((a >> 7) & 7u) << 4); }

// Shared-memory accesses are addressed by 32-bit BYTE offsets from the
// 128-byte aligned dynamic smem base `smem`: pointers are formed as smem +
// offset, so the compiler keeps their address space and emits LDS/STS with
// 32-bit addresses and folded immediates (a swizzle applied to a generic
// 64-bit pointer made every access a generic LD/ST with 64-bit arithmetic).
//
// Byte offset of logical element s of the stage buffer at byte offset bb:
// plain, row-chunk-swizzled (d.swz: 16-byte chunks XOR-permuted by row inside
// each 128-byte block) or address-swizzled (kSwzAddr).
template <typename W>
__device__ __forceinline__ uint32_t soff(const PhaseDesc &d, uint32_t bb, uint32_t s) {
    if (d.swz == kSwzAddr) return swz_off(bb + s * (uint32_t)sizeof(W));
    return d.swz ? bb + swizzle<16 / (int)sizeof(W)>(d, s) * (uint32_t)sizeof(W) : bb + s * (uint32_t)sizeof(W);
}
template <typename W>
__device__ __forceinline__ W *sptr(unsigned char *smem, uint32_t off) {
    return reinterpret_cast<W *>(smem + off);
}
template <typename W>
__device__ __forceinline__ const W *sptr(const unsigned char *smem, uint32_t off) {
    return reinterpret_cast<const W *>(smem + off);
}

// Shared-memory load through an explicit 32-bit shared-window address (sb =
// smem_u32(smem) + byte offset).  In large unrolled (predicated) scalar W
// walks the compiler otherwise rebuilt the window address of the pointer in
// front of every load (VIADD + LEA with the CTA-in-cluster id + IADD3 per
// element); with the address in one register the per-element constants fold
// into the LDS immediate.
template <typename W>
struct RegOf {
    using T = W;
};
template <>
struct RegOf<unsigned char> {
    using T = uint32_t;
};
template <>
struct RegOf<unsigned short> {
    using T = uint32_t;
};
// (1- and 2-byte words travel in 32-bit registers between the load and the
// store: as unsigned char / short values every element cost a PRMT merge)
template <typename W>
__device__ __forceinline__ typename RegOf<W>::T lds(uint32_t a) {
    if constexpr (sizeof(W) == 1) {
        uint32_t v;
        asm volatile("ld.shared.u8 %0, [%1];\n" : "=r"(v) : "r"(a) : "memory");
        return v;
    } else if constexpr (sizeof(W) == 2) {
        uint32_t v;
        asm volatile("ld.shared.u16 %0, [%1];\n" : "=r"(v) : "r"(a) : "memory");
        return v;
    } else if constexpr (sizeof(W) == 4) {
        uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(v) : "r"(a) : "memory");
        return (W)v;
    } else if constexpr (sizeof(W) == 8) {
        unsigned long long v;
        asm volatile("ld.shared.u64 %0, [%1];\n" : "=l"(v) : "r"(a) : "memory");
        return (W)v;
    } else {
        uint4 v;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "r"(a)
                     : "memory");
        return v;
    }
}
template <typename W>
__device__ __forceinline__ void st_reg(W *p, const typename RegOf<W>::T &v) {
#ifdef VPG_JIT
    if constexpr (sizeof(W) == 1) asm volatile("st.global.u8 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
    else if constexpr (sizeof(W) == 2) asm volatile("st.global.u16 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
    else st_out(p, v);
#else
    st_out(p, (W)v);
#endif
}
// smem_u32(smem) pinned in a register (the compiler otherwise recomputes the
// window address -- cvta + the CTA-in-cluster id -- at its uses)
__device__ __forceinline__ uint32_t smem_base_reg(const void *smem) {
    uint32_t sb = smem_u32(smem);
    asm volatile("mov.u32 %0, %0;\n" : "+r"(sb));
    return sb;
}
// Scalar W load: explicit shared-window addressing in specialised kernels;
// the ahead-of-time kernels (rolled loops, run-time strides) keep the plain
// load -- the asm form cost them 10-17% on sub-MiB problems
// (profiles/w_lds_ab_r2.txt).
template <typename W>
__device__ __forceinline__ typename RegOf<W>::T lds_w(const unsigned char *smem, uint32_t sb, uint32_t off) {
#ifdef VPG_JIT
    return lds<W>(sb + off);
#else
    return *sptr<W>(smem, off);
#endif
}

__device__ __forceinline__ bool slot_ok(uint32_t mask, uint32_t c0, uint32_t c1, uint32_t c2, const Lim &lim) {
    return (!(mask & 1u) || c0 < lim.l0) && (!(mask & 2u) || c1 < lim.l1) && (!(mask & 4u) || c2 < lim.l2);
}

// Outer-dim entry o of a phase: from the per-CTA smem table (AOT), or
// decoded on the fly with constant divisors (JIT).
__device__ __forceinline__ OuterEntry outer_entry(const PhaseDesc &d, const unsigned char *smem, uint32_t o) {
#ifdef VPG_JIT
    OuterEntry e;
    e.g = 0;
    e.s = 0;
    e.h = 0;
    uint32_t c0 = 0, c1 = 0, idx = o;
    VPG_UNROLL
    for (int i = 0; i < kMaxPhaseDims; ++i) {
        if (i >= d.nout_dims) break;
        uint32_t q = fdiv(idx, d.out[i].div);
        uint32_t c = idx - q * d.out[i].div.d;
        idx = q;
        e.g += (int64_t)c * d.out[i].gstride;
        e.s += c * d.out[i].sstride;
        e.h += c * d.out[i].hmul;
        if (d.out[i].slot == 0) c0 = c * d.out[i].cmul;
        else if (d.out[i].slot == 1) c1 = c * d.out[i].cmul;
    }
    e.c0 = (uint16_t)c0;
    e.c1 = (uint16_t)c1;
    return e;
#else
    return reinterpret_cast<const OuterEntry *>(smem + d.off_tab)[o];
#endif
}

// R phase: global (source order) -> smem (stage buffer at byte offset bb).
// ASYNC: cp.async (16-byte chunks when d.vec > 1), else LDG+STS.
template <typename W, bool ASYNC, bool VEC>
__device__ __forceinline__ void tile_read_impl(const PhaseDesc &d, const ThreadPart &t, unsigned char *smem,
                                               const W *__restrict__ gsrc, uint32_t bb, uint32_t mask,
                                               const Lim lim) {
    constexpr int U = 4;
    constexpr int CP = VEC ? 16 : (int)sizeof(W);
    // cp.async moves 4, 8 or 16 bytes: scalar 1- and 2-byte words load
    // synchronously (their vectorised phases use 16-byte cp.async)
    constexpr bool CPA = ASYNC && CP >= 4;
    const uint32_t n_in = d.n_in;
    const int64_t g_in = d.g_in;
    const uint32_t s_in = d.s_in;
    const uint32_t sbase = smem_u32(smem);
    const uint32_t o0 = d.ngroups == 1 ? 0u : t.grp;   // constant in JIT builds
    VPG_UNROLL
    for (uint32_t o = o0; o < d.n_outer; o += d.ngroups) {
        const OuterEntry e = outer_entry(d, smem, o);
        const W *gp = (gsrc + t.g) + e.g;
        uint32_t so = t.s + e.s;
        if (mask == 0) {
            uint32_t i = 0;
            VPG_UNROLL
            for (; i + U <= n_in; i += U) {
                if constexpr (CPA) {
#pragma unroll
                    for (int u = 0; u < U; ++u) cp_async<CP>(sbase + soff<W>(d, bb, so + u * s_in), gp + u * g_in);
                } else {
                    W v[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) v[u] = __ldg(gp + u * g_in);
#pragma unroll
                    for (int u = 0; u < U; ++u) *sptr<W>(smem, soff<W>(d, bb, so + u * s_in)) = v[u];
                }
                gp += U * g_in;
                so += U * s_in;
            }
            for (; i < n_in; ++i) {
                if constexpr (CPA) cp_async<CP>(sbase + soff<W>(d, bb, so), gp);
                else *sptr<W>(smem, soff<W>(d, bb, so)) = __ldg(gp);
                gp += g_in;
                so += s_in;
            }
        } else {
            uint32_t c0 = t.c0 + e.c0, c1 = t.c1 + e.c1, c2 = t.c2;
            VPG_UNROLL
            for (uint32_t i = 0; i < n_in; ++i) {
                if (slot_ok(mask, c0, c1, c2, lim)) {
                    if constexpr (CPA) cp_async<CP>(sbase + soff<W>(d, bb, so), gp);
                    else *sptr<W>(smem, soff<W>(d, bb, so)) = __ldg(gp);
                }
                gp += g_in;
                so += s_in;
                c0 += d.c_in[0];
                c1 += d.c_in[1];
                c2 += d.c_in[2];
            }
        }
    }
}

// Byte offset of the 16-byte smem chunk that receives the aligned chunk of
// source run element s (misaligned runs).  Residue mode (rshift 2): s's own
// slot is congruent to its global address modulo 16 bytes, so the chunk goes
// to the aligned-down slot; chunk-aligned rows (rshift 1): s is the chunk's
// first slot.
template <typename W>
__device__ __forceinline__ uint32_t shift_chunk_off(const PhaseDesc &d, uint32_t bb, uint32_t s) {
    constexpr int V = 16 / (int)sizeof(W);
    if (d.rshift == 2) {
        const uint32_t a = (bb + s * (uint32_t)sizeof(W)) & ~15u;
        return d.swz == kSwzAddr ? swz_off(a) : a;
    }
    return d.swz ? bb + swizzle<V>(d, s) * (uint32_t)sizeof(W) : bb + s * (uint32_t)sizeof(W);
}

// R phase for misaligned source runs: each run is read as the 16-byte
// aligned superset that covers it (the address is rounded down per chunk),
// so the run lands at offset h = (run start mod V) inside its smem row; the
// W phase adds h back (or, with residue strides, reads it in place).
// Chunks reaching past the end of the source buffer fall back to element
// copies.
template <typename W, bool CHECK_END>
__device__ __forceinline__ void tile_read_shift(const PhaseDesc &d, const ThreadPart &t, unsigned char *smem,
                                                const W *__restrict__ gsrc, const W *gend, uint32_t bb,
                                                uint32_t mask, const Lim lim) {
    constexpr int V = 16 / (int)sizeof(W);
    const uint32_t n_in = d.n_in;
    const int64_t g_in = d.g_in;
    const uint32_t s_in = d.s_in;
    const uint32_t sbase = smem_u32(smem);
    const uint32_t o0 = d.ngroups == 1 ? 0u : t.grp;
    VPG_UNROLL
    for (uint32_t o = o0; o < d.n_outer; o += d.ngroups) {
        const OuterEntry e = outer_entry(d, smem, o);
        const W *gp = (gsrc + t.g) + e.g;
        uint32_t so = t.s + e.s;
        uint32_t c0 = t.c0 + e.c0, c1 = t.c1 + e.c1, c2 = t.c2;
        VPG_UNROLL
        for (uint32_t i = 0; i < n_in; ++i) {
            if (mask == 0 || slot_ok(mask, c0, c1, c2, lim)) {
                const W *ga = reinterpret_cast<const W *>((uintptr_t)gp & ~(uintptr_t)15);
                const uint32_t sd = sbase + shift_chunk_off<W>(d, bb, so);
                if (!CHECK_END || ga + V <= gend) {
                    cp_async<16>(sd, ga);
                } else {
#pragma unroll
                    for (int j = 0; j < V; ++j)
                        if (ga + j < gend) {
                            if constexpr (sizeof(W) >= 4) cp_async<sizeof(W)>(sd + j * (uint32_t)sizeof(W), ga + j);
                            else *sptr<W>(smem, sd - sbase + j * (uint32_t)sizeof(W)) = __ldg(ga + j);
                        }
                }
            }
            gp += g_in;
            so += s_in;
            c0 += d.c_in[0];
            c1 += d.c_in[1];
            c2 += d.c_in[2];
        }
    }
}

template <typename W, bool ASYNC>
__device__ __forceinline__ void tile_read(const PhaseDesc &d, const ThreadPart &t, unsigned char *smem,
                                          const W *__restrict__ gsrc, const W *gend, uint32_t bb, uint32_t mask,
                                          const Lim lim, bool near_end) {
    if (!t.active) return;
    if constexpr (ASYNC && sizeof(W) < 16) {
        if (d.rshift) {
            // tiles clear of the buffer end read every chunk unchecked
            // (straight-line cp.async sequences; the rare tile at the end checks)
            if (near_end) tile_read_shift<W, true>(d, t, smem, gsrc, gend, bb, mask, lim);
            else tile_read_shift<W, false>(d, t, smem, gsrc, gend, bb, mask, lim);
            return;
        }
    }
    if constexpr (ASYNC && sizeof(W) < 16) {
        if (d.vec > 1) {
            tile_read_impl<W, true, true>(d, t, smem, gsrc, bb, mask, lim);
            return;
        }
    }
    tile_read_impl<W, ASYNC, false>(d, t, smem, gsrc, bb, mask, lim);
}

// W phase: smem -> global (destination order).  VEC: each position is a
// 16-byte smem vector of V consecutive dim-0 elements, stored to V
// destinations d.vstride apart (each store instruction stays coalesced
// across the warp's lanes).
// W in V x V blocks (PhaseDesc::w2): V 16-byte smem vectors from V
// consecutive destination-innermost rows (one swizzle group, so one slot
// computation), transposed in registers into V 16-byte stores.
template <typename W>
__device__ __forceinline__ void w2_block(W *gp, const unsigned char *sp, uint32_t vrow_bytes, int64_t vs) {
    constexpr int V = 16 / (int)sizeof(W);
    uint4 v[V];
#pragma unroll
    for (int i = 0; i < V; ++i) v[i] = *reinterpret_cast<const uint4 *>(sp + i * vrow_bytes);
#pragma unroll
    for (int j = 0; j < V; ++j) {
        alignas(16) W o[V];
#pragma unroll
        for (int i = 0; i < V; ++i) o[i] = reinterpret_cast<const W *>(&v[i])[j];
        st_out(reinterpret_cast<uint4 *>(gp + j * vs), *reinterpret_cast<const uint4 *>(o));
    }
}

template <typename W>
__device__ __forceinline__ void tile_write_w2(const PhaseDesc &d, const ThreadPart &t, const unsigned char *smem,
                                              W *__restrict__ gdst, uint32_t bb, uint32_t mask, const Lim lim) {
    const uint32_t o0 = d.ngroups == 1 ? 0u : t.grp;
    VPG_UNROLL
    for (uint32_t o = o0; o < d.n_outer; o += d.ngroups) {
        const OuterEntry e = outer_entry(d, smem, o);
        W *gp = (gdst + t.g) + e.g;
        const uint32_t sb = t.s + e.s;
        uint32_t c0 = t.c0 + e.c0, c1 = t.c1 + e.c1, c2 = t.c2;
        VPG_UNROLL
        for (uint32_t i = 0; i < d.n_in; ++i) {
            if (mask == 0 || slot_ok(mask, c0, c1, c2, lim))
                w2_block<W>(gp + (int64_t)i * d.g_in, smem + soff<W>(d, bb, sb + i * d.s_in),
                            d.vrow * (uint32_t)sizeof(W), d.vstride);
            c0 += d.c_in[0];
            c1 += d.c_in[1];
            c2 += d.c_in[2];
        }
    }
}

// W in k x V interleave blocks (PhaseDesc::w2 = k >= 2): k 16-byte smem
// vectors (one per value of the destination-innermost dim c, V consecutive
// dim-0 elements each, rows vrow elements apart) are interleaved in
// registers into k*V consecutive destination elements -- destination
// element (w, c) is word w of vector c -- and stored as k 16-byte chunks.
template <typename W, int K>
__device__ __forceinline__ void wk_block(W *gp, const unsigned char *smem, const PhaseDesc &d, uint32_t bb,
                                         uint32_t s0) {
    constexpr int V = 16 / (int)sizeof(W);
    uint4 v[K];
#pragma unroll
    for (int c = 0; c < K; ++c) v[c] = *sptr<uint4>(smem, soff<W>(d, bb, s0 + (uint32_t)c * d.vrow));
#pragma unroll
    for (int j = 0; j < K; ++j) {
        alignas(16) W o[V];
#pragma unroll
        for (int i = 0; i < V; ++i) {
            const int e = j * V + i;
            o[i] = reinterpret_cast<const W *>(&v[e % K])[e / K];
        }
        st_out(reinterpret_cast<uint4 *>(gp + j * V), *reinterpret_cast<const uint4 *>(o));
    }
}

template <typename W, int K>
__device__ __forceinline__ void tile_write_wk_k(const PhaseDesc &d, const ThreadPart &t, const unsigned char *smem,
                                                W *__restrict__ gdst, uint32_t bb, uint32_t mask, const Lim lim) {
    const uint32_t o0 = d.ngroups == 1 ? 0u : t.grp;
    VPG_UNROLL
    for (uint32_t o = o0; o < d.n_outer; o += d.ngroups) {
        const OuterEntry e = outer_entry(d, smem, o);
        W *gp = (gdst + t.g) + e.g;
        const uint32_t sb = t.s + e.s;
        uint32_t c0 = t.c0 + e.c0, c1 = t.c1 + e.c1, c2 = t.c2;
        VPG_UNROLL
        for (uint32_t i = 0; i < d.n_in; ++i) {
            if (mask == 0 || slot_ok(mask, c0, c1, c2, lim))
                wk_block<W, K>(gp + (int64_t)i * d.g_in, smem, d, bb, sb + i * d.s_in);
            c0 += d.c_in[0];
            c1 += d.c_in[1];
            c2 += d.c_in[2];
        }
    }
}

// W in gather blocks (PhaseDesc::w2 >= kW2Gather): G destination-innermost
// elements from G smem rows vrow apart (scalar loads, any alignment: residue
// rows included) packed into one store of G words (16 bytes for G = V; 4 or
// 8 bytes for the narrow blocks of 1- and 2-byte words).
template <typename W, int G>
__device__ __forceinline__ void tile_write_wg_g(const PhaseDesc &d, const ThreadPart &t, const unsigned char *smem,
                                                W *__restrict__ gdst, uint32_t bb, uint32_t mask, const Lim lim) {
    constexpr int B = G * (int)sizeof(W);          // bytes per store: 4, 8 or 16
    using S = typename WordOf<B>::T;
    const uint32_t o0 = d.ngroups == 1 ? 0u : t.grp;
    VPG_UNROLL
    for (uint32_t o = o0; o < d.n_outer; o += d.ngroups) {
        const OuterEntry e = outer_entry(d, smem, o);
        W *gp = (gdst + t.g) + e.g;
        const uint32_t sb = t.s + e.s;
        uint32_t c0 = t.c0 + e.c0, c1 = t.c1 + e.c1, c2 = t.c2;
        VPG_UNROLL
        for (uint32_t i = 0; i < d.n_in; ++i) {
            if (mask == 0 || slot_ok(mask, c0, c1, c2, lim)) {
                alignas(16) W v[G];
                const uint32_t s0 = sb + i * d.s_in;
#pragma unroll
                for (int j = 0; j < G; ++j) v[j] = *sptr<W>(smem, soff<W>(d, bb, s0 + (uint32_t)j * d.vrow));
                st_out(reinterpret_cast<S *>(gp + (int64_t)i * d.g_in), *reinterpret_cast<const S *>(v));
            }
            c0 += d.c_in[0];
            c1 += d.c_in[1];
            c2 += d.c_in[2];
        }
    }
}

template <typename W>
__device__ __forceinline__ void tile_write_wg(const PhaseDesc &d, const ThreadPart &t, const unsigned char *smem,
                                              W *__restrict__ gdst, uint32_t bb, uint32_t mask, const Lim lim) {
    constexpr int V = 16 / (int)sizeof(W);
    if (d.w2 == kW2Gather) {
        tile_write_wg_g<W, V>(d, t, smem, gdst, bb, mask, lim);
        return;
    }
    if constexpr (V >= 4) {
        if (d.w2 == kW2Gather + 2) tile_write_wg_g<W, 2>(d, t, smem, gdst, bb, mask, lim);
    }
    if constexpr (V >= 8) {
        if (d.w2 == kW2Gather + 4) tile_write_wg_g<W, 4>(d, t, smem, gdst, bb, mask, lim);
    }
    if constexpr (V >= 16) {
        if (d.w2 == kW2Gather + 8) tile_write_wg_g<W, 8>(d, t, smem, gdst, bb, mask, lim);
    }
}

template <typename W>
__device__ __forceinline__ void tile_write_wk(const PhaseDesc &d, const ThreadPart &t, const unsigned char *smem,
                                              W *__restrict__ gdst, uint32_t bb, uint32_t mask, const Lim lim) {
    switch (d.w2) {
        case 2: tile_write_wk_k<W, 2>(d, t, smem, gdst, bb, mask, lim); break;
        case 3: tile_write_wk_k<W, 3>(d, t, smem, gdst, bb, mask, lim); break;
        case 4: tile_write_wk_k<W, 4>(d, t, smem, gdst, bb, mask, lim); break;
        case 5: tile_write_wk_k<W, 5>(d, t, smem, gdst, bb, mask, lim); break;
        case 6: tile_write_wk_k<W, 6>(d, t, smem, gdst, bb, mask, lim); break;
        case 7: tile_write_wk_k<W, 7>(d, t, smem, gdst, bb, mask, lim); break;
        default: tile_write_wk_k<W, 8>(d, t, smem, gdst, bb, mask, lim); break;
    }
}

// W with vec > 1: the V elements of one 16-byte smem vector go to V
// destinations vs apart -- one 16-byte store when they are consecutive
// (vs == 1: the stride-1 dim is preserved, the vector is a destination chunk)
template <typename W>
__device__ __forceinline__ void store_vec(W *gp, const uint4 &v, int64_t vs) {
    constexpr int V = 16 / (int)sizeof(W);
    if (vs == 1) {
        st_out(reinterpret_cast<uint4 *>(gp), v);
        return;
    }
    const W *w = reinterpret_cast<const W *>(&v);
#pragma unroll
    for (int j = 0; j < V; ++j) st_out(gp + j * vs, w[j]);
}

// Narrow W vectors (VB = 4 or 8 bytes: 2-8 elements of a 1- or 2-byte word
// along the source dim 0 in ONE shared-memory load, stored element by element
// vs apart).  For residue rows whose source runs are misaligned to 16 bytes
// but aligned to VB: a quarter to half of the scalar walk's LDS instructions.
template <typename W, int VB>
__device__ __forceinline__ void store_vec_n(W *gp, const typename WordOf<VB>::T &v, int64_t vs) {
    constexpr int V = VB / (int)sizeof(W);
#pragma unroll
    for (int j = 0; j < V; ++j) {
        // (st.global.u8/u16 store the low bits of the 32-bit register)
        st_reg(gp + j * vs, (uint32_t)(v >> (8 * (int)sizeof(W) * j)));
    }
}

template <typename W, bool VEC, int VB = 16>
__device__ __forceinline__ void tile_write_impl(const PhaseDesc &d, const ThreadPart &t, const unsigned char *smem,
                                                W *__restrict__ gdst, uint32_t bb, uint32_t mask,
                                                const Lim lim, uint32_t hb, uint32_t hmask) {
    constexpr int U = VEC ? (VB == 16 ? 2 : 4) : VPG_W_U;
    constexpr int V = VEC ? VB / (int)sizeof(W) : 1;
    using VT = typename WordOf<VB>::T;
    const uint32_t n_in = d.n_in;
    const int64_t g_in = d.g_in;
    const uint32_t s_in = d.s_in;
    const int64_t vs = d.vstride;
    const uint32_t sb = smem_base_reg(smem);
    const uint32_t o0 = d.ngroups == 1 ? 0u : t.grp;   // constant in JIT builds
    VPG_UNROLL
    for (uint32_t o = o0; o < d.n_outer; o += d.ngroups) {
        const OuterEntry e = outer_entry(d, smem, o);
        W *gp = (gdst + t.g) + e.g;
        uint32_t s = t.s + e.s;
        uint32_t hh = hb + t.h + e.h;          // shifted-run mode (hmask == 0 otherwise)
        const uint32_t h_in = d.h_in;
        if (mask == 0) {
            uint32_t i = 0;
            VPG_UNROLL
            for (; i + U <= n_in; i += U) {
                if constexpr (VEC) {
                    VT v[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) v[u] = *sptr<VT>(smem, soff<W>(d, bb, s + u * s_in));
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        if constexpr (VB == 16) store_vec<W>(gp + u * g_in, v[u], vs);
                        else store_vec_n<W, VB>(gp + u * g_in, v[u], vs);
                    }
                } else {
                    typename RegOf<W>::T v[U];
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        v[u] = lds_w<W>(smem, sb, soff<W>(d, bb, s + u * s_in + ((hh + u * h_in) & hmask)));
#pragma unroll
                    for (int u = 0; u < U; ++u) st_reg(gp + u * g_in, v[u]);
                }
                gp += U * g_in;
                s += U * s_in;
                hh += U * h_in;
            }
            for (; i < n_in; ++i) {
                if constexpr (VEC) {
                    if constexpr (VB == 16) store_vec<W>(gp, *sptr<uint4>(smem, soff<W>(d, bb, s)), vs);
                    else store_vec_n<W, VB>(gp, *sptr<VT>(smem, soff<W>(d, bb, s)), vs);
                } else {
                    st_reg(gp, lds_w<W>(smem, sb, soff<W>(d, bb, s + (hh & hmask))));
                }
                gp += g_in;
                s += s_in;
                hh += h_in;
            }
        } else {
            uint32_t c0 = t.c0 + e.c0, c1 = t.c1 + e.c1, c2 = t.c2;
            uint32_t i = 0;
            if constexpr (!VEC) {
                // checked walk, U elements at a time: all U (predicated) smem
                // loads issue before the first store, so the stores do not
                // each wait out a shared-memory latency
                VPG_UNROLL
                for (; i + U <= n_in; i += U) {
                    typename RegOf<W>::T v[U];
                    bool ok[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        ok[u] = slot_ok(mask, c0 + u * d.c_in[0], c1 + u * d.c_in[1], c2 + u * d.c_in[2], lim);
                        if (ok[u]) v[u] = lds_w<W>(smem, sb, soff<W>(d, bb, s + u * s_in + ((hh + u * h_in) & hmask)));
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (ok[u]) st_reg(gp + u * g_in, v[u]);
                    gp += U * g_in;
                    s += U * s_in;
                    hh += U * h_in;
                    c0 += U * d.c_in[0];
                    c1 += U * d.c_in[1];
                    c2 += U * d.c_in[2];
                }
            }
            VPG_UNROLL
            for (; i < n_in; ++i) {
                if (slot_ok(mask, c0, c1, c2, lim)) {
                    if constexpr (VEC) {
                        if constexpr (VB == 16) store_vec<W>(gp, *sptr<uint4>(smem, soff<W>(d, bb, s)), vs);
                        else store_vec_n<W, VB>(gp, *sptr<VT>(smem, soff<W>(d, bb, s)), vs);
                    } else {
                        st_reg(gp, lds_w<W>(smem, sb, soff<W>(d, bb, s + (hh & hmask))));
                    }
                }
                gp += g_in;
                s += s_in;
                hh += h_in;
                c0 += d.c_in[0];
                c1 += d.c_in[1];
                c2 += d.c_in[2];
            }
        }
    }
}

#ifdef VPG_JIT
// Scalar W walk of specialised kernels with a short inner dim (n_in < 4):
// the thread's (outer, inner) positions flattened and taken U at a time,
// all U smem loads ahead of the U stores (the nested walk issued each
// load-store pair back to back, one smem latency per element).
template <typename W>
__device__ __forceinline__ void tile_write_flat(const PhaseDesc &d, const ThreadPart &t, const unsigned char *smem,
                                                W *__restrict__ gdst, uint32_t bb, uint32_t mask, const Lim lim,
                                                uint32_t hb, uint32_t hmask) {
    constexpr int U = 8;
    const uint32_t sb = smem_base_reg(smem);
    const uint32_t o0 = d.ngroups == 1 ? 0u : t.grp;
    const uint32_t n_o = d.n_outer > o0 ? (d.n_outer - o0 + d.ngroups - 1) / d.ngroups : 0u;
    const uint32_t total = n_o * d.n_in;
#ifdef VPG_FLAT_UNROLL
    VPG_UNROLL_N(VPG_FLAT_UNROLL)
#else
    VPG_UNROLL
#endif
    for (uint32_t b0 = 0; b0 < total; b0 += U) {
        typename RegOf<W>::T v[U];
        W *gp[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t idx = b0 + u;
            ok[u] = idx < total;
            const uint32_t oi = idx / d.n_in, i = idx - oi * d.n_in;
            const OuterEntry e = outer_entry(d, smem, o0 + oi * d.ngroups);
            gp[u] = (gdst + t.g) + e.g + (int64_t)i * d.g_in;
            const uint32_t s = t.s + e.s + i * d.s_in;
            const uint32_t hh = hb + t.h + e.h + i * d.h_in;
            if (mask)
                ok[u] = ok[u] && slot_ok(mask, t.c0 + e.c0 + i * d.c_in[0], t.c1 + e.c1 + i * d.c_in[1],
                                         t.c2 + i * d.c_in[2], lim);
            if (ok[u]) v[u] = lds_w<W>(smem, sb, soff<W>(d, bb, s + (hh & hmask)));
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (ok[u]) st_reg(gp[u], v[u]);
    }
}
#endif

template <typename W>
__device__ __forceinline__ void tile_write(const PhaseDesc &d, const ThreadPart &t, const unsigned char *smem,
                                           W *__restrict__ gdst, uint32_t bb, uint32_t mask,
                                           const Lim lim, uint32_t hb, uint32_t hmask) {
    if (!t.active) return;
#if defined(VPG_JIT) && !defined(VPG_NO_FLAT)
    // The check mask of a tile is one of two plan constants (full or ragged
    // tile): the scalar walks are instantiated once per constant (their
    // shared-memory loads are volatile asm, which the compiler does not
    // unswitch by itself; with a run-time mask every element evaluated it).
    if (d.vec <= 1 && !d.w2 && d.n_in < 4) {
        if (mask == d.mask_full) tile_write_flat<W>(d, t, smem, gdst, bb, d.mask_full, lim, hb, hmask);
        else tile_write_flat<W>(d, t, smem, gdst, bb, d.mask_ragged, lim, hb, hmask);
        return;
    }
#endif
    if constexpr (sizeof(W) < 16) {
        if (d.w2 == 1) {
            tile_write_w2<W>(d, t, smem, gdst, bb, mask, lim);
            return;
        }
        if (d.w2 >= kW2Gather) {
            tile_write_wg<W>(d, t, smem, gdst, bb, mask, lim);
            return;
        }
        if (d.w2 >= 2) {
            tile_write_wk<W>(d, t, smem, gdst, bb, mask, lim);
            return;
        }
        if (d.vec > 1) {
            if constexpr (sizeof(W) <= 2) {
                // narrow vectors: 4 or 8 bytes of 1-2-byte words (residue rows)
                if (d.vec * (uint32_t)sizeof(W) == 4) {
                    tile_write_impl<W, true, 4>(d, t, smem, gdst, bb, mask, lim, 0, 0);
                    return;
                }
                if (d.vec * (uint32_t)sizeof(W) == 8) {
                    tile_write_impl<W, true, 8>(d, t, smem, gdst, bb, mask, lim, 0, 0);
                    return;
                }
            }
            tile_write_impl<W, true>(d, t, smem, gdst, bb, mask, lim, 0, 0);
            return;
        }
    }
#ifdef VPG_JIT
    if (mask == d.mask_full) tile_write_impl<W, false>(d, t, smem, gdst, bb, d.mask_full, lim, hb, hmask);
    else tile_write_impl<W, false>(d, t, smem, gdst, bb, d.mask_ragged, lim, hb, hmask);
#else
    tile_write_impl<W, false>(d, t, smem, gdst, bb, mask, lim, hb, hmask);
#endif
}

// W phase, lin mode (LinDesc in plan_params.h): the per-plan table of u16
// smem offsets, tab[m][c][e] = offset of destination-run position
// c*V - m + e (0 outside the run), built once per CTA.
template <int V>
__device__ __forceinline__ void lin_build_table(const LinDesc &L, unsigned char *smem, uint32_t tid, uint32_t NT) {
    uint16_t *tab = reinterpret_cast<uint16_t *>(smem + L.tab_off);
    const uint32_t per_m = L.cpr * V;
    for (uint32_t i = tid; i < V * per_m; i += NT) {
        const uint32_t m = i / per_m;
        const int32_t j = (int32_t)(i - m * per_m) - (int32_t)m;
        uint32_t off = 0;
        if (j >= 0 && (uint32_t)j < L.run_len) {
            uint32_t x = (uint32_t)j;
            VPG_UNROLL
            for (int k = 0; k < kMaxLinDims; ++k) {
                if (k >= L.nrd) break;
                const uint32_t q = fdiv(x, L.rd[k].div);
                off += (x - q * L.rd[k].div.d) * L.rd[k].sstride;
                x = q;
            }
        }
        tab[i] = (uint16_t)off;
    }
}

// a[k] <- a[(k + r) mod V] (selects, r lane-dependent): log2(V) stages,
// stage b rotating by 2^b when bit b of r is set
template <int V, typename T>
__device__ __forceinline__ void rot_left(T (&a)[V], uint32_t r) {
#pragma unroll
    for (int b = V / 2; b >= 1; b /= 2) {
        T t[V];
#pragma unroll
        for (int k = 0; k < V; ++k) t[k] = a[(k + b) % V];
        const bool on = (r & (uint32_t)b) != 0u;
#pragma unroll
        for (int k = 0; k < V; ++k) a[k] = on ? t[k] : a[k];
    }
}

// Chunk slots q = tid, tid + nt, ...: run r = q / cpr over the run-index
// dims, slot c = q % cpr.  The run starts at word m of its 16-byte chunk
// (from the address), so slot c covers run positions j0 = c*V - m ..
// j0 + V-1: V smem loads (offsets from one table load; positions outside
// the run read offset 0, harmlessly) and one aligned 16-byte store when all
// V positions are valid, element stores otherwise (run head and tail, and
// ragged tiles, whose valid positions are a prefix of Lv).
template <typename W>
__device__ __forceinline__ void tile_write_lin(const TileParams &p, const unsigned char *smem,
                                               W *__restrict__ gdst, uint32_t bb, bool ragged, const Lim lim,
                                               uint32_t tid) {
    constexpr int V = 16 / (int)sizeof(W);
    const LinDesc &L = p.lin;
    const PhaseDesc &d = p.ph[1];
    if (tid >= L.nt) return;
    uint32_t Lv = L.run_len;
    if (ragged && L.last_slot >= 0) Lv = L.last_unit * (L.last_slot == 0 ? lim.l0 : lim.l1);
    // bank spreading: load k of this lane fetches chunk element (k + rot) mod V
    const uint32_t rot = L.rot_shift < 32 ? ((tid & 31u) >> L.rot_shift) & (uint32_t)(V - 1) : 0u;
    // batches of B chunk slots per thread: every smem load of a batch issues
    // before its first store
    constexpr int B = sizeof(W) == 1 ? 2 : 4;
    VPG_UNROLL
    for (uint32_t q0 = tid; q0 < L.nchunks; q0 += B * L.nt) {
        alignas(16) W v[B][V];
        W *cp[B];
        int32_t j0[B];
        bool live[B];
#pragma unroll
        for (int b = 0; b < B; ++b) {
            const uint32_t q = q0 + b * L.nt;
            live[b] = q < L.nchunks;
            const uint32_t r = fdiv(q, L.cprd);
            const uint32_t c = q - r * L.cpr;
            int64_t go = 0;
            uint32_t so = 0;
            uint32_t x = r;
            VPG_UNROLL
            for (int i = 0; i < kMaxPhaseDims; ++i) {
                if (i >= L.nxd) break;
                const uint32_t qq = fdiv(x, L.xd[i].div);
                const uint32_t dg = x - qq * L.xd[i].div.d;
                x = qq;
                go += (int64_t)dg * L.xd[i].gstride;
                so += dg * L.xd[i].sstride;
                if (L.xd[i].slot >= 0 && ragged) live[b] = live[b] && dg < (L.xd[i].slot == 0 ? lim.l0 : lim.l1);
            }
            W *const rp = gdst + go;
            const uint32_t m = (uint32_t)(reinterpret_cast<uintptr_t>(rp) / sizeof(W)) & (uint32_t)(V - 1);
            j0[b] = (int32_t)(c * V) - (int32_t)m;
            cp[b] = rp + j0[b];      // 16-byte aligned
            if (!live[b]) continue;
            const unsigned char *tq = smem + L.tab_off + (m * L.cpr + c) * (uint32_t)(V * 2);
            uint32_t offs[V];
            if constexpr (V == 4) {
                const uint2 t = *reinterpret_cast<const uint2 *>(tq);
                offs[0] = t.x & 0xffffu;
                offs[1] = t.x >> 16;
                offs[2] = t.y & 0xffffu;
                offs[3] = t.y >> 16;
            } else if constexpr (V == 2) {
                const uint32_t t = *reinterpret_cast<const uint32_t *>(tq);
                offs[0] = t & 0xffffu;
                offs[1] = t >> 16;
            } else {
                // 1- and 2-byte words: V u16 entries in V/8 16-byte loads
#pragma unroll
                for (int h = 0; h < V / 8; ++h) {
                    const uint4 t = *reinterpret_cast<const uint4 *>(tq + 16 * h);
                    const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        offs[8 * h + 2 * k] = w[k] & 0xffffu;
                        offs[8 * h + 2 * k + 1] = w[k] >> 16;
                    }
                }
            }
            rot_left<V>(offs, rot);
#pragma unroll
            for (int e = 0; e < V; ++e) v[b][e] = *sptr<W>(smem, soff<W>(d, bb, so + offs[e]));
            rot_left<V>(v[b], (uint32_t)V - rot);
        }
#pragma unroll
        for (int b = 0; b < B; ++b) {
            if (!live[b]) continue;
            bool all = true;
#pragma unroll
            for (int e = 0; e < V; ++e) all = all && (uint32_t)(j0[b] + e) < Lv;
            if (all) {
                st_out(reinterpret_cast<uint4 *>(cp[b]), *reinterpret_cast<const uint4 *>(v[b]));
            } else {
#pragma unroll
                for (int e = 0; e < V; ++e)
                    if ((uint32_t)(j0[b] + e) < Lv) st_out(cp[b] + e, v[b][e]);
            }
        }
    }
}

// Warp 0 decodes tile `t` into slot `k`: source/destination base offsets and
// the valid extents of the ragged boundary dims a and c.  Sharded plans
// rebase the source offset onto the local input shard and the destination
// offset onto the owning output shard's buffer (sa.off, relative to dst).
// (A per-CTA shared-memory copy of the digits measured 6% slower on cfg5:
// 722 vs 683 us; the lane-indexed reads stay on the parameter block.)
__device__ __forceinline__ void decode_tile(const TileParams &p, const ShardArgs &sa, uint32_t t,
                                            int64_t (*s_base)[2], uint32_t (*s_valid)[2], int k) {
    const uint32_t lane = threadIdx.x & 31;
    t += p.tile_begin;
    int64_t sb = 0, db = 0;
    uint32_t va = p.e_a, vc = p.e_c;
#ifdef VPG_JIT
    // specialised kernels: every digit's divisors and strides are
    // compile-time constants (no parameter loads from global memory)
    VPG_UNROLL
    for (int i = 0; i < kMaxRank; ++i) {
        if (i >= p.ngrid) break;
        if ((i & 31) != (int)lane) continue;
#else
    for (int i = (int)lane; i < p.ngrid; i += 32) {
#endif
        const GridDigit &gd = p.grid[i];
        uint32_t q = fdiv(t, gd.cum);
        uint32_t c = q - fdiv(q, gd.ext) * gd.ext.d;
        sb += (int64_t)c * gd.src_stride;
        db += (int64_t)c * gd.dst_stride;
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
        if (p.nshards > 1 && p.pull) {
            db -= p.dst_bias;           // pull: local output shard; sources stay global
        } else if (p.nshards > 1) {
            const uint64_t q = (uint64_t)db / (uint64_t)p.shard_elems;
            sb -= p.src_bias;
            db += sa.off[q] - (int64_t)q * p.shard_elems;
        }
        s_base[k][0] = sb;
        s_base[k][1] = db;
        s_valid[k][0] = va;
        s_valid[k][1] = vc;
    }
}

#ifdef VPG_JIT
// Specialised kernels: ONE thread decodes tile t completely.  Every digit's
// divisors and strides are immediates and the digits are independent, so
// this is a short branch-free sequence; the prologue's S tiles are decoded
// by S threads in parallel and no shuffles (or warp-collective fallbacks)
// are needed.
__device__ __forceinline__ void decode_tile_thread(const TileParams &p, const ShardArgs &sa, uint32_t t,
                                                   int64_t (*s_base)[2], uint32_t (*s_valid)[2], int k) {
    t += p.tile_begin;
    int64_t sb = 0, db = 0;
    uint32_t va = p.e_a, vc = p.e_c;
    VPG_UNROLL
    for (int i = 0; i < kMaxRank; ++i) {
        if (i >= p.ngrid) break;
        const GridDigit &gd = p.grid[i];
        const uint32_t q = fdiv(t, gd.cum);
        const uint32_t c = q - fdiv(q, gd.ext) * gd.ext.d;
        sb += (int64_t)c * gd.src_stride;
        db += (int64_t)c * gd.dst_stride;
        if (i == p.grid_a) va = min(p.e_a, p.d_a - c * p.e_a);
        if (i == p.grid_c) vc = min(p.e_c, p.d_c - c * p.e_c);
    }
    if (p.nshards > 1 && p.pull) {
        db -= p.dst_bias;
    } else if (p.nshards > 1) {
        const uint64_t q = (uint64_t)db / (uint64_t)p.shard_elems;
        sb -= p.src_bias;
        db += sa.off[q] - (int64_t)q * p.shard_elems;
    }
    s_base[k][0] = sb;
    s_base[k][1] = db;
    s_valid[k][0] = va;
    s_valid[k][1] = vc;
}
#endif

// ------------------------------------------------------------------ pull exchange
// Source word at GLOBAL offset o of a pull exchange plan: input shard
// q = o / shard_elems, read through the per-launch shard table (peer memory
// for the other ranks' shards).
template <typename W>
__device__ __forceinline__ const W *pull_ptr(const TileParams &p, const ShardArgs &sa, const W *src, int64_t o) {
    // power-of-two shards: a shift; otherwise a 32-bit fast divide while every
    // global offset fits 32 bits, else a 64-bit divide (uniform branch; it
    // folds away in specialised kernels, where p is a constant)
    const uint32_t q = p.shard_shift               ? (uint32_t)((uint64_t)o >> p.shard_shift)
                       : p.n_elems <= 0xffffffffll ? fdiv((uint32_t)o, p.shard_div)
                                                   : (uint32_t)((uint64_t)o / (uint64_t)p.shard_elems);
    return src + (sa.off[q] + (o - (int64_t)q * p.shard_elems));
}

// R phase of a pull plan: the walk of tile_read_impl / tile_read_shift with
// every 16-byte chunk (or word) addressed through pull_ptr.  Chunks never
// straddle shards (launch_plan_pull requires shard_elems % V == 0 and
// 16-byte aligned shard buffers for the vectorised variants).
template <typename W, bool ASYNC>
__device__ __forceinline__ void tile_read_pull(const TileParams &p, const ShardArgs &sa, const PhaseDesc &d,
                                               const ThreadPart &t, unsigned char *smem, const W *src,
                                               int64_t sbase, uint32_t bb, uint32_t mask, const Lim lim) {
    if (!t.active) return;
    constexpr int V = 16 / (int)sizeof(W);
    const uint32_t sb32 = smem_u32(smem);
    const uint32_t o0 = d.ngroups == 1 ? 0u : t.grp;
    VPG_UNROLL
    for (uint32_t o = o0; o < d.n_outer; o += d.ngroups) {
        const OuterEntry e = outer_entry(d, smem, o);
        int64_t go = sbase + t.g + e.g;
        uint32_t so = t.s + e.s;
        uint32_t c0 = t.c0 + e.c0, c1 = t.c1 + e.c1, c2 = t.c2;
        VPG_UNROLL
        for (uint32_t i = 0; i < d.n_in; ++i) {
            if (mask == 0 || slot_ok(mask, c0, c1, c2, lim)) {
                const uint32_t sp = soff<W>(d, bb, so);
                if constexpr (ASYNC && sizeof(W) < 16) {
                    if (d.rshift) {
                        cp_async<16>(sb32 + shift_chunk_off<W>(d, bb, so), pull_ptr(p, sa, src, go & ~(int64_t)(V - 1)));
                    } else if (d.vec > 1) {
                        cp_async<16>(sb32 + sp, pull_ptr(p, sa, src, go));
                    } else if constexpr (sizeof(W) >= 4) {
                        cp_async<sizeof(W)>(sb32 + sp, pull_ptr(p, sa, src, go));
                    } else {
                        *sptr<W>(smem, sp) = __ldg(pull_ptr(p, sa, src, go));
                    }
                } else if constexpr (ASYNC) {
                    cp_async<16>(sb32 + sp, pull_ptr(p, sa, src, go));
                } else {
                    *sptr<W>(smem, sp) = __ldg(pull_ptr(p, sa, src, go));
                }
            }
            go += d.g_in;
            so += d.s_in;
            c0 += d.c_in[0];
            c1 += d.c_in[1];
            c2 += d.c_in[2];
        }
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

// ------------------------------------------------------------------ exchange barrier
// Device-side ordering of a fused exchange across the G ranks' kernels
// (ShardArgs::epoch != 0), instead of collectives around the launch:
//   start: CTA 0 of rank r stores epoch into slot r of every rank's flag
//          block (system-scope release, over NVLink for peers); every CTA
//          waits until its own block's G start slots reach epoch before
//          its first load -- every rank's kernel has started, so (stream
//          order) every input shard is complete and every output shard free.
//   end:   every CTA fences its stores system-wide and counts itself done;
//          the last CTA of rank r stores epoch into done-slot r of every
//          block and waits for its own G done-slots: the kernel (and hence
//          the stream) completes only when every rank's stores have landed
//          and every rank has finished reading.
// Spins are bounded (~4 s of globaltimer): a missing rank makes the kernel
// exit with an unfinished result instead of hanging the GPU.
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void wait_flags(const unsigned long long *f, uint32_t n, unsigned long long epoch) {
    unsigned long long t0 = 0;
    for (uint32_t q = 0; q < n; ++q) {
        while (ld_acquire_sys(f + q) < epoch) {
            const unsigned long long t = gtimer();
            if (t0 == 0) t0 = t;
            else if (t - t0 > 4000000000ull) return;   // bounded: never hang the device
            __nanosleep(64);
        }
    }
}
__device__ __forceinline__ void shard_barrier_start(const ShardArgs &sa, uint32_t G, uint32_t cta) {
    if (threadIdx.x == 0) {
        if (cta == 0)
            for (uint32_t q = 0; q < G; ++q) st_release_sys(sa.flags[q] + sa.rank, sa.epoch);
        wait_flags(sa.flags[sa.rank], G, sa.epoch);
    }
    __syncthreads();
}
__device__ __forceinline__ void shard_barrier_end(const ShardArgs &sa, uint32_t G, uint32_t ncta) {
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t prev;
        asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;\n" : "=r"(prev) : "l"(sa.done_ctr) : "memory");
        if (prev == ncta - 1) {
            atomicExch(sa.done_ctr, 0u);
            __threadfence_system();
            for (uint32_t q = 0; q < G; ++q) st_release_sys(sa.flags[q] + G + sa.rank, sa.epoch);
            wait_flags(sa.flags[sa.rank] + G, G, sa.epoch);
        }
    }
}

// Persistent CTAs walk tiles t_k = blockIdx.x + k*gridDim.x through an
// S-stage cp.async pipeline (S = p.nbuf smem tile buffers): the prologue
// streams the source runs of the first S tiles; each iteration writes tile
// k out of its buffer and refills that buffer with tile k+S.  Small
// problems are thereby staged in one wave; large ones keep S-1 tiles of
// loads in flight per CTA (every word size: 1- and 2-byte words move
// 16-byte cp.async vectors, their scalar phases load synchronously).
template <typename W, bool ASYNC>
__device__ __forceinline__ void tile_body(const TileParams &p, const W *__restrict__ src, W *__restrict__ dst,
                                          const ShardArgs &sa, uint32_t cta, uint32_t ncta) {
    // the planner's layout is relative to a 128-byte aligned base: staged
    // rows then sit at the same offset modulo 128 bytes as their source lines
    // (see PhaseDesc::swz).  Specialised kernels with a scalar W walk declare
    // the alignment (VPG_SMEM_DECL, jit.cpp) instead of computing it: the
    // run-time round-up of the base was rematerialised in front of every
    // predicated shared-memory load of large unrolled walks (7 of ~23
    // instructions per element in the slow 1-byte plans, tools/sass_per_store.sh).
    // Vector W walks keep the computed base: with the declared one the V x V
    // blocks spilled more at their 80-register cap (profiles/w_lds_ab_r2.txt).
#if VPG_SMEM_DECL
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *const smem = smem_raw;
#else
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned char *const smem = smem_raw + ((128u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 127u)) & 127u);
#endif
    __shared__ int64_t s_base[kRing][2];
    __shared__ uint32_t s_valid[kRing][2];
    const uint32_t tid = threadIdx.x, NT = blockDim.x;
    // CTA `cta` of the `ncta` CTAs running this plan (blockIdx.x / gridDim.x,
    // except in the cooperative multi-rank emulation of an exchange)
    const uint32_t first = cta, step = ncta;
    const bool xbar = p.nshards > 1 && sa.epoch != 0;      // device-side exchange barrier
    // (no static tile implies S * ncta >= num_tiles: no dynamic claims either)
    if (first >= p.num_tiles) {
        if (xbar) shard_barrier_end(sa, p.nshards, ncta);
        return;
    }
    const uint32_t S = ASYNC ? p.nbuf : 1u;
    const uint32_t R = S + 2;
    pdl_trigger();
    // development tracing: specialised kernels compiled with VPG_TRACE only
#ifdef VPG_TRACE_BUILD
    unsigned long long *const trc = sa.trace ? sa.trace + (size_t)blockIdx.x * kTraceWords : nullptr;
#else
    constexpr unsigned long long *trc = nullptr;
#endif
    if (trc && tid == 0) {
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        trc[0] = gtimer();
        trc[3] = smid;
    }

    // Tile schedule.  The first S tiles of a CTA are static (blockIdx.x +
    // j * gridDim.x, the prologue); later ones come from the dynamic
    // scheduler when the launch carries one (sa.sched): tile S * gridDim.x +
    // atomicAdd(next), so SMs that drain faster take more tiles (ncu on cfg5
    // with a static round-robin: SM active cycles 0.58-0.99 of the elapsed
    // ones).  Without it, tile first + j * gridDim.x.  One fetcher (thread
    // NT-1 in specialised kernels, warp 0 otherwise) claims and decodes the
    // tile of slot k+S during iteration k; the claim for the following one is
    // issued one iteration ahead, so its latency overlaps a W phase.
    __shared__ uint32_t s_ok[kRing];
    // (a grid whose prologue covers every tile claims nothing: no atomics)
    const bool dyn = sa.sched != nullptr && S * step < p.num_tiles;
    const uint32_t dyn_base = S * step;
    uint32_t pre = 0;        // fetcher: prefetched claim
    bool fetch_done = false; // fetcher: the counter ran past the last tile
    auto signal_done = [&]() {
        // the last CTA to finish claiming resets the pair for the ring's next use
        __threadfence();
        if (atomicAdd(sa.sched + 1, 1u) == ncta - 1) {
            atomicExch(sa.sched, 0u);
            atomicExch(sa.sched + 1, 0u);
        }
    };
#ifdef VPG_JIT
    const bool fetcher = tid == NT - 1;
#else
    const bool fetcher = tid == 0;
#endif
    // the first claim goes out at entry: its latency overlaps the prologue
    if (dyn && fetcher) pre = atomicAdd(sa.sched, 1u);

    // per-CTA outer tables of both phases (JIT builds decode entries inline)
#ifndef VPG_JIT
    for (int ph = 0; ph < 2; ++ph) {
        const PhaseDesc &d = p.ph[ph];
        OuterEntry *tab = reinterpret_cast<OuterEntry *>(smem + d.off_tab);
        for (uint32_t o = tid; o < d.n_outer; o += NT) {
            uint32_t idx = o, s = 0, c0 = 0, c1 = 0, h = 0;
            int64_t g = 0;
            for (int i = 0; i < d.nout_dims; ++i) {
                uint32_t q = fdiv(idx, d.out[i].div);
                uint32_t c = idx - q * d.out[i].div.d;
                idx = q;
                g += (int64_t)c * d.out[i].gstride;
                s += c * d.out[i].sstride;
                h += c * d.out[i].hmul;
                if (d.out[i].slot == 0) c0 = c * d.out[i].cmul;
                else if (d.out[i].slot == 1) c1 = c * d.out[i].cmul;
            }
            OuterEntry e;
            e.g = g;
            e.s = s;
            e.c0 = (uint16_t)c0;
            e.c1 = (uint16_t)c1;
            e.h = h;
            e.pad_ = 0;
            tab[o] = e;
        }
    }
#endif
    const ThreadPart tr = decode_thread(p.ph[0], tid);
    const ThreadPart tw = decode_thread(p.ph[1], tid);
    const W *const gend = src + p.n_elems;
    // stage buffer k at byte offset p.off_buf + k * bstride from smem
    const uint32_t bstride = ((uint32_t)p.tile_elems_alloc * (uint32_t)sizeof(W) + 15u) / 16u * 16u;

#ifdef VPG_JIT
    if (tid < S) {
        const uint32_t t = first + tid * step;
        const bool ok = t < p.num_tiles;
        if (ok) decode_tile_thread(p, sa, t, s_base, s_valid, (int)tid);
        s_ok[tid] = ok;
    }
#else
    if (tid < 32)
        for (uint32_t j = 0; j < S; ++j) {
            const uint32_t t = first + j * step;
            if (t < p.num_tiles) decode_tile(p, sa, t, s_base, s_valid, (int)j);
            if (tid == 0) s_ok[j] = t < p.num_tiles;
        }
#endif
    __syncthreads();
    auto limits = [&](uint32_t slot, int ph, Lim &lim) -> uint32_t {
        const uint32_t va = s_valid[slot][0], vc = s_valid[slot][1];
        lim.l0 = va;
        lim.l1 = vc;
        lim.l2 = p.lim_split[ph];
        const bool full = (va == p.e_a) && (vc == p.e_c);
        return full ? p.ph[ph].mask_full : p.ph[ph].mask_ragged;
    };
    // residue layouts: the tile sits at (source base mod rres) elements into its buffer
    auto shifted = [&](uint32_t b, uint32_t slot) {
        return b + (p.rres ? ((uint32_t)s_base[slot][0] & p.rres) * (uint32_t)sizeof(W) : 0u);
    };
    auto load = [&](uint32_t k, uint32_t b) {
        Lim lim;
        const uint32_t slot = k % R;
        const uint32_t m = limits(slot, 0, lim);
        const uint32_t bt = shifted(b, slot);
        if (p.pull) tile_read_pull<W, ASYNC>(p, sa, p.ph[0], tr, smem, src, s_base[slot][0], bt, m, lim);
        else
            tile_read<W, ASYNC>(p.ph[0], tr, smem, src + s_base[slot][0], gend, bt, m, lim,
                                s_base[slot][0] + p.src_span + 16 / (int64_t)sizeof(W) > p.n_elems);
    };
    pdl_wait();
    if (xbar) shard_barrier_start(sa, p.nshards, cta);
    if (trc && tid == 0) trc[kTraceWords - 2] = gtimer();      // first load about to issue
    // prologue: fill every stage
    for (uint32_t j = 0; j < S; ++j) {
        if (s_ok[j]) load(j, p.off_buf + j * bstride);
        if constexpr (ASYNC) cp_async_commit();
    }
    if (trc && tid == 0) trc[1] = gtimer();
    // lin W: the offset table (ordered before the first W by the loop's barrier)
    if constexpr (sizeof(W) < 16)
        if (p.lin.on) lin_build_table<16 / (int)sizeof(W)>(p.lin, smem, tid, NT);
    uint32_t tiles_done = 0;
    for (uint32_t k = 0;; ++k) {
        // claim + decode the tile of slot k+S
        {
            const uint32_t nslot = (k + S) % R;
#ifdef VPG_JIT
            if (fetcher) {
                uint32_t t = 0xffffffffu;
                if (dyn) {
                    if (!fetch_done) {
                        t = dyn_base + pre;
                        if (t < p.num_tiles) pre = atomicAdd(sa.sched, 1u);
                        else { fetch_done = true; signal_done(); }
                    }
                } else {
                    t = first + (k + S) * step;
                }
                const bool ok = t < p.num_tiles;
                if (ok) decode_tile_thread(p, sa, t, s_base, s_valid, (int)nslot);
                s_ok[nslot] = ok;
            }
#else
            if (tid < 32) {
                uint32_t t = 0xffffffffu;
                if (tid == 0) {
                    if (dyn) {
                        if (!fetch_done) {
                            t = dyn_base + pre;
                            if (t < p.num_tiles) pre = atomicAdd(sa.sched, 1u);
                            else { fetch_done = true; signal_done(); }
                        }
                    } else {
                        t = first + (k + S) * step;
                    }
                }
                t = __shfl_sync(0xffffffffu, t, 0);
                const bool ok = t < p.num_tiles;
                if (ok) decode_tile(p, sa, t, s_base, s_valid, (int)nslot);
                if (tid == 0) s_ok[nslot] = ok;
            }
#endif
        }
        if constexpr (ASYNC) cp_async_wait_pending(S - 1);
        __syncthreads();
        if (!s_ok[k % R]) break;           // uniform: this CTA has no tile k
        if (trc && tid == 0 && k < 19) trc[4 + 3 * k + 1] = gtimer();
        const uint32_t b = p.off_buf + (k % S) * bstride;
        {
            Lim lim;
            const uint32_t slot = k % R;
            const uint32_t m = limits(slot, 1, lim);
            bool lin_done = false;
            if constexpr (sizeof(W) < 16) {
                if (p.lin.on) {
                    tile_write_lin<W>(p, smem, dst + s_base[slot][1], shifted(b, slot),
                                      !(lim.l0 == p.e_a && lim.l1 == p.e_c), lim, tid);
                    lin_done = true;
                }
            }
            if (!lin_done)
                tile_write<W>(p.ph[1], tw, smem, dst + s_base[slot][1], shifted(b, slot), m, lim,
                              (uint32_t)s_base[slot][0], p.hmask);
        }
        __syncthreads();
        if (trc && tid == 0 && k < 19) {
            trc[4 + 3 * k] = (unsigned long long)(s_base[k % R][1]);
            trc[4 + 3 * k + 2] = gtimer();
        }
        ++tiles_done;
        if (s_ok[(k + S) % R]) load(k + S, b);
        if constexpr (ASYNC) cp_async_commit();
    }
    if (trc && tid == 0) {
        trc[2] = gtimer();
        trc[kTraceWords - 1] = tiles_done;
    }
    // peer stores of a sharded plan: performed system-wide before the grid
    // retires, so the exchange's completion barrier orders them
    if (xbar) shard_barrier_end(sa, p.nshards, ncta);
    else if (p.nshards > 1) __threadfence_system();
}

template <typename W, bool ASYNC>
__device__ __forceinline__ void tile_body(const TileParams &p, const W *__restrict__ src, W *__restrict__ dst,
                                          const ShardArgs &sa) {
    tile_body<W, ASYNC>(p, src, dst, sa, blockIdx.x, gridDim.x);
}


}  // namespace vpg

namespace vpg {

// ------------------------------------------------------------------ bulk mode
// The R phase as TMA bulk copies: a producer warp (the last warp of the
// CTA) issues one cp.async.bulk per source run into the stage buffer and
// arms the stage's `full` mbarrier with the expected byte count; the
// consumer warps wait on it, run the W phase, and release the stage through
// its `empty` mbarrier.  No CTA-wide barriers in the steady state.
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *sdst, const void *gsrc, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(sdst)),
                 "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

template <typename W>
__device__ __forceinline__ void tile_body_bulk(const TileParams &p, const W *__restrict__ src, W *__restrict__ dst,
                                               const ShardArgs &sa) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
    __shared__ int64_t s_base[kMaxStages][2];
    __shared__ uint32_t s_valid[kMaxStages][2];
    unsigned char *const smem = smem_raw + ((128u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 127u)) & 127u);
    const uint32_t tid = threadIdx.x;
    const uint32_t NC = blockDim.x - 32;              // consumer threads (the W phase was planned for NC)
    const uint32_t first = blockIdx.x, step = gridDim.x;
    if (first >= p.num_tiles) return;
    const uint32_t cnt = (p.num_tiles - first + step - 1) / step;
    const uint32_t S = p.nbuf;
    pdl_trigger();

#ifndef VPG_JIT
    {   // W-phase outer table (the producer needs no table)
        const PhaseDesc &d = p.ph[1];
        OuterEntry *tab = reinterpret_cast<OuterEntry *>(smem + d.off_tab);
        for (uint32_t o = tid; o < d.n_outer; o += blockDim.x) {
            uint32_t idx = o, s = 0, c0 = 0, c1 = 0, h = 0;
            int64_t g = 0;
            for (int i = 0; i < d.nout_dims; ++i) {
                uint32_t q = fdiv(idx, d.out[i].div);
                uint32_t c = idx - q * d.out[i].div.d;
                idx = q;
                g += (int64_t)c * d.out[i].gstride;
                s += c * d.out[i].sstride;
                h += c * d.out[i].hmul;
                if (d.out[i].slot == 0) c0 = c * d.out[i].cmul;
                else if (d.out[i].slot == 1) c1 = c * d.out[i].cmul;
            }
            OuterEntry e;
            e.g = g;
            e.s = s;
            e.c0 = (uint16_t)c0;
            e.c1 = (uint16_t)c1;
            e.h = h;
            e.pad_ = 0;
            tab[o] = e;
        }
    }
#endif
    if (tid == 0) {
        for (uint32_t s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NC / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    }
    pdl_wait();
    __syncthreads();
    const size_t bstride = ((size_t)p.tile_elems_alloc * sizeof(W) + 15) / 16 * 16 / sizeof(W);
    const uint32_t bstride_b = (uint32_t)(bstride * sizeof(W));

    if (tid >= NC) {
        // ---------------- producer warp
        const uint32_t lane = tid - NC;
        constexpr int V = 16 / (int)sizeof(W);
        // misaligned runs (residue rows, rshift 2): each run is fetched as its
        // 16-byte aligned superset; the part of a run in the last, partial
        // 16-byte chunk of the source buffer is copied by its lane instead
        const bool mis = p.ph[0].rshift == 2;
        for (uint32_t k = 0; k < cnt; ++k) {
            const uint32_t st = k % S;
            if (k >= S) mbar_wait(&empty[st], ((k / S) - 1) & 1);
#ifdef VPG_JIT
            if (lane == 0) decode_tile_thread(p, sa, first + k * step, s_base, s_valid, (int)st);
#else
            decode_tile(p, sa, first + k * step, s_base, s_valid, (int)st);
#endif
            __syncwarp();
            const int64_t sb = s_base[st][0];
            const uint32_t va = s_valid[st][0], vc = s_valid[st][1];
            const uint32_t rbytes = va == p.e_a ? p.run_bytes : p.run_unit_bytes * va;
            const uint32_t bb = p.off_buf + st * bstride_b + (mis ? ((uint32_t)sb & p.rres) * (uint32_t)sizeof(W) : 0u);
            // run r of this tile: global element offset, smem byte offset, valid
            auto run = [&](uint32_t r, int64_t &g0, uint32_t &so) -> bool {
                uint32_t idx = r, cc = 0, soff = 0;
                int64_t goff = 0;
                VPG_UNROLL
                for (int i = 0; i < kMaxPhaseDims; ++i) {
                    if (i >= p.nrdims) break;
                    const uint32_t q = fdiv(idx, p.rdims[i].div);
                    const uint32_t c = idx - q * p.rdims[i].div.d;
                    idx = q;
                    goff += (int64_t)c * p.rdims[i].gstride;
                    soff += c * p.rdims[i].sstride;
                    if (p.rdims[i].slot == 1) cc = c;
                }
                g0 = sb + goff;
                so = bb + soff * (uint32_t)sizeof(W);
                return p.grid_c < 0 || cc < vc;
            };
            // aligned superset [ga, ge) of a misaligned run (ge clipped to the
            // last whole chunk of the source buffer)
            auto span = [&](int64_t g0, int64_t &ga, int64_t &ge) {
                const int64_t len = rbytes / (uint32_t)sizeof(W);
                ga = g0 & ~(int64_t)(V - 1);
                ge = (g0 + len + V - 1) & ~(int64_t)(V - 1);
                if (ge > p.n_elems) ge = p.n_elems & ~(int64_t)(V - 1);
                if (ge < ga) ge = ga;
            };
            // valid runs of this lane and the total byte count of the stage
            uint32_t mine = 0;
            for (uint32_t r = lane; r < p.nruns; r += 32) {
                int64_t g0;
                uint32_t so;
                if (!run(r, g0, so)) continue;
                if (!mis) {
                    mine += rbytes;
                    continue;
                }
                int64_t ga, ge;
                span(g0, ga, ge);
                mine += (uint32_t)((ge - ga) * (int64_t)sizeof(W));
                // elements past the last whole chunk: plain copies (ordered
                // before the consumers by the warp barrier + the arrive below)
                const int64_t gend_run = g0 + rbytes / (uint32_t)sizeof(W);
                for (int64_t e = ge > g0 ? ge : g0; e < gend_run; ++e)
                    *sptr<W>(smem, so + (uint32_t)((e - g0) * (int64_t)sizeof(W))) = src[e];
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
            __syncwarp();
            if (lane == 0) mbar_arrive_expect_tx(&full[st], mine);
            __syncwarp();
            for (uint32_t r = lane; r < p.nruns; r += 32) {
                int64_t g0;
                uint32_t so;
                if (!run(r, g0, so)) continue;
                if (!mis) {
                    bulk_g2s(smem + so, src + g0, rbytes, &full[st]);
                    continue;
                }
                int64_t ga, ge;
                span(g0, ga, ge);
                if (ge > ga)
                    bulk_g2s(smem + (so & ~15u), src + ga, (uint32_t)((ge - ga) * (int64_t)sizeof(W)),
                             &full[st]);
            }
        }
        return;
    }
    // ---------------- consumer warps: the W phase
    const ThreadPart tw = decode_thread(p.ph[1], tid);
    for (uint32_t k = 0; k < cnt; ++k) {
        const uint32_t st = k % S;
        mbar_wait(&full[st], (k / S) & 1);
        const uint32_t va = s_valid[st][0], vc = s_valid[st][1];
        Lim lim;
        lim.l0 = va;
        lim.l1 = vc;
        lim.l2 = p.lim_split[1];
        const bool full_tile = (va == p.e_a) && (vc == p.e_c);
        const uint32_t m = full_tile ? p.ph[1].mask_full : p.ph[1].mask_ragged;
        const uint32_t bb = p.off_buf + st * bstride_b +
                            (p.ph[0].rshift == 2 ? ((uint32_t)s_base[st][0] & p.rres) * (uint32_t)sizeof(W) : 0u);
        tile_write<W>(p.ph[1], tw, smem, dst + s_base[st][1], bb, m, lim, (uint32_t)s_base[st][0], p.hmask);
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&empty[st]);
    }
    if (p.nshards > 1) __threadfence_system();
}

}  // namespace vpg
