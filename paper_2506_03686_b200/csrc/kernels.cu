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

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <atomic>
#include <mutex>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "plan.h"
#include "tile_body.cuh"

namespace vpg {

// ------------------------------------------------------------------ COPY
template <typename V>
__global__ void __launch_bounds__(256) copy_kernel(const V *__restrict__ src, V *__restrict__ dst,
                                                   int64_t nvec) {
    pdl_trigger();
    pdl_wait();
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

// 16-byte words: every warp streams contiguous 8 KiB chunks (16 loads in
// flight per lane before the stores) -- measured 6.41 TB/s on 2 GiB against
// 6.05 TB/s for the grid-stride form (tools/copy_pattern_probe.cu).
__global__ void __launch_bounds__(256) copy_kernel_chunked(const uint4 *__restrict__ src, uint4 *__restrict__ dst,
                                                           int64_t nvec) {
    constexpr int CH = 512;   // vectors per warp chunk (8 KiB)
    pdl_trigger();
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t full = nvec / CH * CH;
    for (int64_t c = warp * CH; c < full; c += nwarps * CH) {
        uint4 r[CH / 32];
#pragma unroll
        for (int j = 0; j < CH / 32; ++j) r[j] = ld_stream(src + c + lane + 32 * j);
#pragma unroll
        for (int j = 0; j < CH / 32; ++j) dst[c + lane + 32 * j] = r[j];
    }
    for (int64_t i = full + warp * 32 + lane; i < nvec; i += nwarps * 32) dst[i] = ld_stream(src + i);
}

// ------------------------------------------------------------------ ROWS (K1)
// One group of tpr lanes per destination row; each group iteration moves
// RPW consecutive destination rows with U vectors per lane per row in
// flight before the stores (U = 4, RPW = 2 measured best on cfg4: 346.8 vs
// 351.3 us for one row at a time, 353.2 for U = 8).
template <typename V, int U, int RPW, bool CHUNKED, bool EXACT>
__global__ void __launch_bounds__(256) rows_kernel(const __grid_constant__ RowsParams p,
                                                   const V *__restrict__ src, V *__restrict__ dst,
                                                   uint32_t vec_log2) {
    pdl_trigger();
    pdl_wait();
    const uint32_t tpr = 1u << p.tpr_log2;
    const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t lane = gtid & (tpr - 1);
    const uint32_t ngroups = (gridDim.x * blockDim.x) >> p.tpr_log2;
    const uint32_t rv = p.row_vecs, cv = CHUNKED ? p.chunk_vecs : p.row_vecs;
    for (uint32_t w0 = (gtid >> p.tpr_log2) * RPW; w0 < p.nitems; w0 += ngroups * RPW) {
        const V *s[RPW];
        V *d[RPW];
        uint32_t len[RPW];
        uint32_t maxlen = 0;
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
            const uint32_t w = w0 + r;
            const bool ok = w < p.nitems;
            uint32_t q = ok ? w : 0u, c0 = 0;
            if constexpr (CHUNKED) {
                q = ok ? fdiv(w, p.nchunks) : 0u;
                c0 = ok ? (w - q * p.nchunks.d) * cv : 0u;
            }
            uint32_t rem = q;
            int64_t so = 0;
            for (int i = 0; i < p.ndig; ++i) {
                uint32_t qq = fdiv(rem, p.dig[i].ext);
                so += (int64_t)(rem - qq * p.dig[i].ext.d) * p.dig[i].src_stride;
                rem = qq;
            }
            s[r] = src + (so >> vec_log2) + c0;
            d[r] = dst + (int64_t)q * rv + c0;
            len[r] = ok ? min(cv, rv - c0) : 0u;
            maxlen = max(maxlen, len[r]);
        }
        if constexpr (!CHUNKED) maxlen = rv;
        // every block of U x tpr vectors is loaded before it is stored,
        // predicated at the row end, so short rows keep U loads in flight
        for (uint32_t i = lane; i < maxlen; i += U * tpr) {
            V v[RPW][U];
#pragma unroll
            for (int r = 0; r < RPW; ++r)
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (EXACT ? len[r] != 0 : i + u * tpr < len[r]) v[r][u] = ld_stream(s[r] + i + u * tpr);
#pragma unroll
            for (int r = 0; r < RPW; ++r)
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (EXACT ? len[r] != 0 : i + u * tpr < len[r]) d[r][i + u * tpr] = v[r][u];
        }
    }
}

// ------------------------------------------------------------------ ROWS, TMA bulk
// K1 for long 16-byte-aligned rows as a DMA pipeline: one thread per CTA
// moves each work item (a row, or a chunk of a long row) global -> smem ->
// global with two cp.async.bulk operations (TMA), S slots deep: loads run
// S-1 items ahead, a slot is refilled once the bulk store that read it has
// finished reading (cp.async.bulk.wait_group.read).  No register round
// trip and no per-lane address math; several CTAs per SM keep enough bytes
// in flight.
constexpr int kRowsBulkSlots = 4;
constexpr int64_t kRowsBulkMinBytes = 2560;   // shorter rows: per-lane 16-byte rows_kernel (1.2-2 KiB rows: mixed, flushed -11..0%, steady -3..+7%)

__device__ __forceinline__ void bulk_s2g(void *gdst, const void *ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst),
                 "r"(smem_u32(ssrc)), "r"(bytes)
                 : "memory");
}

__global__ void __launch_bounds__(32) rows_bulk_kernel(const __grid_constant__ RowsParams p,
                                                       const unsigned char *__restrict__ src,
                                                       unsigned char *__restrict__ dst, uint32_t E,
                                                       uint32_t slot_bytes, uint32_t rpi, uint32_t *sched) {
    extern __shared__ __align__(128) unsigned char rb_smem[];
    __shared__ __align__(8) uint64_t bar[kRowsBulkSlots];
    constexpr uint32_t S = kRowsBulkSlots;
    pdl_trigger();
    if (threadIdx.x != 0) return;
    const uint32_t step = gridDim.x;
    // work items: the first S-1 of a CTA static (blockIdx.x + k * gridDim.x),
    // later ones claimed from the dynamic scheduler ((S-1) * gridDim.x +
    // atomicAdd(next), see tile_body) when the launch carries one, so CTAs on
    // SMs that drain faster move more rows; a claim is prefetched one item
    // ahead
    const bool dyn = sched != nullptr && (S - 1) * step < p.nitems;
    uint32_t pre = dyn ? atomicAdd(sched, 1u) : 0u;
    bool claimed_out = false;
    auto claim = [&](uint32_t k) -> uint32_t {
        if (k + 1 < S || !dyn) return blockIdx.x + k * step;
        if (claimed_out) return 0xffffffffu;
        const uint32_t w = (S - 1) * step + pre;
        if (w < p.nitems) {
            pre = atomicAdd(sched, 1u);
        } else {
            claimed_out = true;
            __threadfence();      // the last CTA to run out resets the pair
            if (atomicAdd(sched + 1, 1u) == gridDim.x - 1) {
                atomicExch(sched, 0u);
                atomicExch(sched + 1, 0u);
            }
        }
        return w;
    };
    for (uint32_t j = 0; j < S; ++j) mbar_init(&bar[j], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    pdl_wait();
    const uint32_t row_bytes = (uint32_t)(p.row_len * E), chunk_bytes = p.chunk_vecs * 16u;
    // work item w: rows [w*rpi, w*rpi + rpi) when rows are short (rpi > 1,
    // one load per row, one store of the contiguous destination block), else
    // chunk (w mod nchunks) of row (w / nchunks)
    auto src_row = [&](uint32_t q) {
        uint32_t rem = q;
        int64_t so = 0;
        for (int i = 0; i < p.ndig; ++i) {
            const uint32_t qq = fdiv(rem, p.dig[i].ext);
            so += (int64_t)(rem - qq * p.dig[i].ext.d) * p.dig[i].src_stride;
            rem = qq;
        }
        return src + so * E;
    };
    auto item = [&](uint32_t w, uint32_t &q0, uint32_t &nr, uint32_t &c0) -> uint32_t {
        if (rpi > 1) {
            q0 = w * rpi;
            nr = min(rpi, p.nrows - q0);
            c0 = 0;
            return nr * row_bytes;
        }
        q0 = fdiv(w, p.nchunks);
        nr = 1;
        c0 = (w - q0 * p.nchunks.d) * chunk_bytes;
        return min(chunk_bytes, row_bytes - c0);
    };
    auto load = [&](uint32_t k, uint32_t w) {
        uint32_t q0, nr, c0;
        const uint32_t n = item(w, q0, nr, c0);
        const uint32_t j = k % S;
        mbar_arrive_expect_tx(&bar[j], n);
        for (uint32_t r = 0; r < nr; ++r)
            bulk_g2s(rb_smem + j * slot_bytes + r * row_bytes, src_row(q0 + r) + c0, nr > 1 ? row_bytes : n, &bar[j]);
    };
    uint32_t ws[S];               // item of each slot (>= nitems: none)
    for (uint32_t k = 0; k + 1 < S; ++k) {
        ws[k] = claim(k);
        if (ws[k] < p.nitems) load(k, ws[k]);
    }
    for (uint32_t k = 0;; ++k) {
        const uint32_t j = k % S;
        const uint32_t w = ws[j];
        if (w >= p.nitems) break;
        mbar_wait(&bar[j], (k / S) & 1);
        uint32_t q0, nr, c0;
        const uint32_t n = item(w, q0, nr, c0);
        bulk_s2g(dst + (int64_t)q0 * row_bytes + c0, rb_smem + j * slot_bytes, n);
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        const uint32_t kn = k + S - 1;
        ws[kn % S] = claim(kn);
        if (ws[kn % S] < p.nitems) {
            // slot kn % S held item k - 1: its store must be done reading
            asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
            load(kn, ws[kn % S]);
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// ------------------------------------------------------------------ TILE (K2/K3)
// Ahead-of-time instantiation: the parameter block arrives as a
// __grid_constant__ kernel argument (run-time extents/strides).  jit.cpp
// compiles the same body with the block baked in as constants.
template <typename W, bool ASYNC>
__global__ void __launch_bounds__(1024) tile_kernel(const __grid_constant__ TileParams p,
                                                   const W *__restrict__ src, W *__restrict__ dst,
                                                   const __grid_constant__ ShardArgs sa) {
    tile_body<W, ASYNC>(p, src, dst, sa);
}

// Every rank of a fused exchange in ONE cooperative launch on one device
// (vpg_permute_sharded_emulated): CTAs [r*per, (r+1)*per) run rank r's plan
// with its own parameter block, buffers and ShardArgs (device memory), and
// the device-side exchange barrier between the ranks -- co-residency is
// guaranteed by the cooperative launch, so the flag waits cannot deadlock.
template <typename W>
__global__ void __launch_bounds__(1024) tile_kernel_ranks(const TileParams *ps, const W *const *srcs,
                                                          W *const *dsts, const ShardArgs *sas, uint32_t per) {
    const uint32_t r = blockIdx.x / per;
    tile_body<W, true>(ps[r], srcs[r], dsts[r], sas[r], blockIdx.x - r * per, per);
}

template <typename W>
__global__ void __launch_bounds__(1024) tile_kernel_bulk(const __grid_constant__ TileParams p,
                                                         const W *__restrict__ src, W *__restrict__ dst,
                                                         const __grid_constant__ ShardArgs sa) {
    tile_body_bulk<W>(p, src, dst, sa);
}

// ------------------------------------------------------------------ GATHER (K0)
template <typename W>
__global__ void __launch_bounds__(256) gather_kernel(const __grid_constant__ GatherParams p,
                                                     const W *__restrict__ src, W *__restrict__ dst) {
    pdl_trigger();
    pdl_wait();
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
// dynamic-smem opt-in is a per-device function attribute: keyed by (kernel, device)
std::map<std::pair<const void *, int>, bool> g_attr_set;

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

// Dynamic tile scheduler counters (tile_body.cuh): a ring of {next, done}
// pairs per device, zeroed once; each tile launch takes the next pair and
// its last CTA resets the pair, so a pair is reused only kSchedSlots launches
// later (launches in flight at once on other streams use other pairs).
// VPG_SCHED=0 keeps the static round-robin schedule.  Not during stream
// capture before the ring exists (allocation is not capturable); graph
// replays of one launch reuse its pair sequentially, which the reset allows.
constexpr uint32_t kSchedSlots = 4096;
std::map<int, uint32_t *> g_sched_ring;
std::atomic<uint32_t> g_sched_seq{0};

uint32_t *sched_slot(cudaStream_t st) {
    static const bool off = getenv("VPG_SCHED") && atoi(getenv("VPG_SCHED")) == 0;
    if (off) return nullptr;
    int dev = 0;
    cudaGetDevice(&dev);
    uint32_t *base = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = g_sched_ring.find(dev);
        if (it != g_sched_ring.end()) {
            base = it->second;
        } else {
            cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
            if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
                cudaGetLastError();
                return nullptr;
            }
            void *p = nullptr;
            if (cudaMalloc(&p, kSchedSlots * 2 * sizeof(uint32_t)) == cudaSuccess &&
                cudaMemset(p, 0, kSchedSlots * 2 * sizeof(uint32_t)) == cudaSuccess &&
                cudaDeviceSynchronize() == cudaSuccess) {
                base = (uint32_t *)p;
            } else {
                cudaGetLastError();
                if (p) cudaFree(p);
            }
            g_sched_ring[dev] = base;      // nullptr: static schedule on this device
        }
    }
    if (!base) return nullptr;
    return base + 2 * (g_sched_seq.fetch_add(1, std::memory_order_relaxed) % kSchedSlots);
}

// Development tracing (VPG_TRACE=<file>): tile launches record per-CTA
// globaltimer stamps (tile_body.cuh trc[]) into a device buffer; after each
// launch the stream is synchronised and the records are appended to the
// file (header: grid, num_tiles, kTraceWords; then grid x kTraceWords u64).
// tools/trace_view.py summarises them.  Off (nullptr) unless VPG_TRACE is set.
unsigned long long *g_trace_buf = nullptr;
constexpr int64_t kTraceMaxCtas = 4096;

unsigned long long *trace_begin(cudaStream_t st) {
    static const char *path = getenv("VPG_TRACE");
    if (!path || !*path) return nullptr;
    if (!g_trace_buf && cudaMalloc(&g_trace_buf, kTraceMaxCtas * kTraceWords * 8) != cudaSuccess) {
        g_trace_buf = nullptr;
        return nullptr;
    }
    cudaMemsetAsync(g_trace_buf, 0, kTraceMaxCtas * kTraceWords * 8, st);
    return g_trace_buf;
}

void trace_end(unsigned long long *buf, int64_t grid, uint32_t num_tiles, cudaStream_t st) {
    if (!buf) return;
    grid = std::min<int64_t>(grid, kTraceMaxCtas);
    std::vector<unsigned long long> h((size_t)grid * kTraceWords);
    cudaMemcpyAsync(h.data(), buf, h.size() * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (FILE *f = fopen(getenv("VPG_TRACE"), "ab")) {
        const unsigned long long hdr[3] = {(unsigned long long)grid, num_tiles, (unsigned long long)kTraceWords};
        fwrite(hdr, 8, 3, f);
        fwrite(h.data(), 8, h.size(), f);
        fclose(f);
    }
}

// Launches carry the programmatic stream-serialisation attribute (PDL, see
// pdl_wait in tile_body.cuh) unless VPG_PDL=0 or the plan is sharded (the
// exchange's barriers are collectives on the same stream).
bool pdl_enabled() {
    static const bool on = [] {
        const char *e = getenv("VPG_PDL");
        return !(e && atoi(e) == 0);
    }();
    return on;
}

struct LaunchCfg {
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute attr[1];
    LaunchCfg(int64_t grid, int threads, int smem, cudaStream_t st, bool pdl) {
        memset(&cfg, 0, sizeof(cfg));
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3((unsigned)threads);
        cfg.dynamicSmemBytes = (size_t)smem;
        cfg.stream = st;
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl && pdl_enabled() ? 1 : 0;
    }
};

template <typename... KArgs, typename... Args>
void launch_k(void (*k)(KArgs...), int64_t grid, int threads, int smem, cudaStream_t st, bool pdl,
              Args &&...args) {
    LaunchCfg lc(grid, threads, smem, st, pdl);
    cudaLaunchKernelEx(&lc.cfg, k, std::forward<Args>(args)...);
}

template <typename K>
int occupancy(K kernel, int threads, int smem) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_mu);
    auto key = std::make_tuple((const void *)kernel, threads, smem + (dev << 24));
    auto it = g_occ.find(key);
    if (it != g_occ.end()) return it->second;
    if (!g_attr_set[std::make_pair((const void *)kernel, dev)]) {
        int optin = 0;
        if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || optin <= 0)
            optin = 227 * 1024;
        cudaFuncAttributes fa;
        size_t stat = cudaFuncGetAttributes(&fa, kernel) == cudaSuccess ? fa.sharedSizeBytes : 1024;
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)stat);
        g_attr_set[std::make_pair((const void *)kernel, dev)] = true;
    }
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, smem) != cudaSuccess || nb < 1)
        nb = 1;
    g_occ[key] = nb;
    return nb;
}

int occupancy_ptr(const void *kernel, int threads, int smem) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_mu);
    auto key = std::make_tuple(kernel, threads, smem + (dev << 24));
    auto it = g_occ.find(key);
    if (it != g_occ.end()) return it->second;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, smem) != cudaSuccess || nb < 1) {
        cudaGetLastError();
        nb = 1;
    }
    g_occ[key] = nb;
    return nb;
}

template <int E>
vpg_status launch_tile(const vpg_plan *p, const void *src, void *dst, const ShardArgs &sa_in, cudaStream_t st) {
    using W = typename WordOf<E>::T;
    ShardArgs sa = sa_in;
    // dynamic tile schedule for persistent CTAs (not the bulk-read variant,
    // whose producer warp keeps the static order)
    sa.sched = p->tile.persistent && !p->tile.bulk ? sched_slot(st) : nullptr;
    sa.trace = trace_begin(st);
    const int smem = (int)p->tile.smem_bytes;
    bool aligned = !(p->tile.ph[0].vec > 1 && ((uintptr_t)src % 16));
    // 16-byte destination stores (V x V / interleave blocks, or vectors of a
    // preserved stride-1 dim): every destination buffer 16-byte aligned
    if (p->tile.ph[1].w2 || (p->tile.ph[1].vec > 1 && p->tile.ph[1].vstride == 1)) {
        if ((uintptr_t)dst % 16) aligned = false;
        for (int q = 1; q < (int)p->tile.nshards && !p->tile.pull; ++q)
            if ((sa.off[q] * E) % 16) aligned = false;
    }
    if (p->tile.pull && p->tile.ph[0].vec > 1) {
        // vectorised pull reads: 16-byte chunks of every shard, none straddling two
        if ((p->tile.shard_elems * E) % 16) aligned = false;
        for (int q = 0; q < (int)p->tile.nshards; ++q)
            if (((uintptr_t)src + sa.off[q] * E) % 16) aligned = false;
    }
    if (p->jit && aligned) {
        cudaKernel_t jk = jit_tile_kernel(p);
        if (jk) {
            const int jthreads = p->threads + (p->tile.bulk ? 32 : 0);
            int nb = occupancy_ptr((const void *)jk, jthreads, smem);
            int64_t grid = p->tile.num_tiles;
            if (p->tile.persistent) grid = std::min<int64_t>(grid, (int64_t)nb * sm_count_for_current());
            if (grid < 1) grid = 1;
            void *args[] = {(void *)&src, (void *)&dst, (void *)&sa};
            static const bool dbg = getenv("VPG_DEBUG_LAUNCH") != nullptr;
            if (dbg)
                fprintf(stderr, "[vpg] jit launch kernel %p grid %lld threads %d smem %d nb %d src %p dst %p\n",
                        (const void *)jk, (long long)grid, jthreads, smem, nb, src, dst);
            LaunchCfg lc(grid, jthreads, smem, st, p->shards <= 1);
            if (cudaLaunchKernelExC(&lc.cfg, (const void *)jk, args) == cudaSuccess) {
                trace_end(sa.trace, grid, p->tile.num_tiles, st);
                return VPG_OK;
            }
            cudaGetLastError();   // fall through to the ahead-of-time kernel
        }
    }
    auto launch = [&](auto k, int threads, const TileParams &tp) {
        const int smem = (int)tp.smem_bytes;     // the variants' tables differ in size
        int nb = occupancy(k, threads, smem);
        int64_t grid = p->tile.num_tiles;
        if (p->tile.persistent) grid = std::min<int64_t>(grid, (int64_t)nb * sm_count_for_current());
        if (grid < 1) grid = 1;
        launch_k(k, grid, threads, smem, st, p->shards <= 1, tp, (const W *)src, (W *)dst, sa);
    };
    if constexpr (E == 4 || E == 8) {
        if (aligned && p->tile.bulk) {
            launch(tile_kernel_bulk<W>, p->threads + 32, p->tile);
            return VPG_OK;
        }
    }
    const TileParams &tp = aligned ? p->tile : p->tile_unaligned;
    // (1- and 2-byte words: the cp.async pipeline moves their 16-byte
    // vectors; scalar phases of those words load synchronously)
    launch(tile_kernel<W, true>, p->threads, tp);
    return VPG_OK;
}

template <int E>
vpg_status launch_gather(const vpg_plan *p, const void *src, void *dst, cudaStream_t st) {
    using W = typename WordOf<E>::T;
    int64_t grid = std::min<int64_t>((p->gather.n + 255) / 256, (int64_t)sm_count_for_current() * 8);
    if (grid < 1) grid = 1;
    launch_k(gather_kernel<W>, grid, 256, 0, st, true, p->gather, (const W *)src, (W *)dst);
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
    // long 16-byte rows: the TMA bulk pipeline (rows_bulk_kernel)
    {
        static const int mode = getenv("VPG_ROWS_BULK") ? atoi(getenv("VPG_ROWS_BULK")) : -1;
        const int64_t row_bytes = rp.row_len * E;
        const bool ok = vb == 16 && row_bytes % 16 == 0 && rp.nrows < 0xffffffffull;
        if (ok && (mode == 1 || (mode < 0 && row_bytes >= kRowsBulkMinBytes))) {
            static const uint32_t kSlot = getenv("VPG_ROWS_SLOT") ? (uint32_t)atoi(getenv("VPG_ROWS_SLOT")) : 16384;
            RowsParams bp = rp;
            const uint64_t rv = (uint64_t)row_bytes / 16;                  // 16-byte units per row
            uint64_t cv = std::min<uint64_t>(rv, kSlot / 16);
            // short rows: several whole rows per item (one store per item)
            uint32_t rpi = row_bytes <= (int64_t)kSlot ? (uint32_t)(kSlot / row_bytes) : 1u;
            if (rpi > 1 && (int64_t)((rp.nrows + rpi - 1) / rpi) < (int64_t)sm_count_for_current() * 12)
                rpi = std::max<uint32_t>(1, (uint32_t)(rp.nrows / ((int64_t)sm_count_for_current() * 12)));
            // enough items for every CTA when rows are few
            const int64_t want = (int64_t)sm_count_for_current() * 6 * 4;
            if ((int64_t)rp.nrows * (int64_t)((rv + cv - 1) / cv) < want) {
                const uint64_t per = ((uint64_t)rp.nrows * rv + want - 1) / want;
                cv = std::max<uint64_t>(64, std::min<uint64_t>(cv, (per + 63) / 64 * 64));
            }
            const uint64_t nch = (rv + cv - 1) / cv;
            if ((uint64_t)rp.nrows * nch < 0xffffffffull) {
                bp.chunk_vecs = (uint32_t)cv;
                bp.nchunks = make_fastdiv((uint32_t)nch);
                bp.nitems = rpi > 1 ? (uint32_t)((rp.nrows + rpi - 1) / rpi) : (uint32_t)(rp.nrows * nch);
                const uint32_t slot = rpi > 1 ? (uint32_t)(rpi * row_bytes) : (uint32_t)(cv * 16);
                const int smem = (int)(slot * kRowsBulkSlots);
                int nb = occupancy(rows_bulk_kernel, 32, smem);
                nb = std::min(nb, 8);
                int64_t grid = std::min<int64_t>(bp.nitems, (int64_t)nb * sm_count_for_current());
                if (grid < 1) grid = 1;
                launch_k(rows_bulk_kernel, grid, 32, smem, st, true, bp, (const unsigned char *)src,
                         (unsigned char *)dst, (uint32_t)E, slot, rpi, sched_slot(st));
                return VPG_OK;
            }
        }
    }
    // cut long rows into chunks until there are enough work items to fill
    // every SM (few long rows would otherwise leave most warps idle)
    {
        const int64_t want = (int64_t)sm_count_for_current() * 64 * 2;   // two warps' worth per warp slot
        uint64_t cv = rp.row_vecs;
        if ((int64_t)rp.nrows < want) {
            const uint64_t per = ((uint64_t)rp.nrows * rp.row_vecs + want - 1) / want;
            const uint64_t unit = 32u * 4u;                                  // one warp x U vectors
            cv = std::max<uint64_t>(unit * 2, (per + unit - 1) / unit * unit);
            cv = std::min<uint64_t>(cv, rp.row_vecs);
        }
        const uint64_t nch = (rp.row_vecs + cv - 1) / cv;
        if ((uint64_t)rp.nrows * nch >= 0xffffffffull) {
            rp.chunk_vecs = rp.row_vecs;
            rp.nchunks = make_fastdiv(1);
            rp.nitems = rp.nrows;
        } else {
            rp.chunk_vecs = (uint32_t)cv;
            rp.nchunks = make_fastdiv((uint32_t)nch);
            rp.nitems = (uint32_t)(rp.nrows * nch);
        }
        // lanes per row (work item): enough that each lane moves at most
        // U = 4 vectors per pass; short rows share a warp
        uint32_t tpr = 1;
        while (tpr < 32 && tpr * 4 < rp.chunk_vecs) tpr <<= 1;
        rp.tpr_log2 = 0;
        while ((1u << rp.tpr_log2) < tpr) ++rp.tpr_log2;
    }
    int64_t need = ((int64_t)rp.nitems << rp.tpr_log2) + 255;
    need /= 256;
#define VPG_ROWS_LAUNCH(TYPE, U, R)                                                            \
    {                                                                                          \
        auto k = rp.nchunks.d > 1 ? rows_kernel<TYPE, U, R, true, false>                       \
                 : (rp.row_vecs % ((U) << rp.tpr_log2) == 0 ? rows_kernel<TYPE, U, R, false, true>  \
                                                             : rows_kernel<TYPE, U, R, false, false>); \
        int nb = occupancy(k, 256, 0);                                                         \
        int64_t grid = std::min<int64_t>(need, (int64_t)nb * sm_count_for_current());          \
        if (grid < 1) grid = 1;                                                                \
        launch_k(k, grid, 256, 0, st, true, rp, (const TYPE *)src, (TYPE *)dst, vlog);         \
        return VPG_OK;                                                                         \
    }
#define VPG_ROWS_CASE(BYTES, TYPE)                                                             \
    case BYTES: {                                                                              \
        VPG_ROWS_LAUNCH(TYPE, 4, 2)                                                            \
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
#undef VPG_ROWS_LAUNCH
}

vpg_status launch_copy(const vpg_plan *p, const void *src, void *dst, cudaStream_t st) {
    int64_t nbytes = p->copy.n * p->elem_bytes;
    int al = ptr_align(src, dst);
    while (al > 1 && (nbytes % al)) al >>= 1;
    int64_t nvec = nbytes / al;
    int64_t grid = std::min<int64_t>((nvec + 255) / 256, (int64_t)sm_count_for_current() * 8);
    if (grid < 1) grid = 1;
    switch (al) {
        case 16:
            if (nvec >= (1 << 16)) {   // >= 1 MiB: chunked form, 16 CTAs per SM
                const int64_t g16 = std::min<int64_t>((nvec + 511) / 512 / 8 + 1, (int64_t)sm_count_for_current() * 16);
                launch_k(copy_kernel_chunked, g16, 256, 0, st, true, (const uint4 *)src, (uint4 *)dst, nvec);
            } else {
                launch_k(copy_kernel<uint4>, grid, 256, 0, st, true, (const uint4 *)src, (uint4 *)dst, nvec);
            }
            break;
        case 8: launch_k(copy_kernel<unsigned long long>, grid, 256, 0, st, true, (const unsigned long long *)src, (unsigned long long *)dst, nvec); break;
        case 4: launch_k(copy_kernel<unsigned int>, grid, 256, 0, st, true, (const unsigned int *)src, (unsigned int *)dst, nvec); break;
        case 2: launch_k(copy_kernel<unsigned short>, grid, 256, 0, st, true, (const unsigned short *)src, (unsigned short *)dst, nvec); break;
        default: launch_k(copy_kernel<unsigned char>, grid, 256, 0, st, true, (const unsigned char *)src, (unsigned char *)dst, nvec); break;
    }
    return VPG_OK;
}

}  // namespace

int device_sm_count() { return sm_count_for_current(); }

static void apply_sync(ShardArgs &sa, const vpg_plan *p, const vpg_shard_sync *sync) {
    if (!sync || sync->epoch == 0 || p->shards < 2) return;
    for (int q = 0; q < p->shards; ++q) sa.flags[q] = sync->flags[q];
    sa.epoch = sync->epoch;
    sa.rank = (uint32_t)p->shard_index;
    sa.done_ctr = sync->done_counter;
}

vpg_status launch_plan_pull(const vpg_plan *p, const void *const *srcs, void *dst, void *stream, std::string *err,
                            const vpg_shard_sync *sync) {
    cudaStream_t st = (cudaStream_t)stream;
    const int E = p->elem_bytes;
    const int G = p->shards;
    if (p->kernel_class != VPG_KERNEL_TILE || !p->tile.pull || G < 1) {
        *err = "not a pull exchange plan";
        return VPG_EINVAL;
    }
    ShardArgs sa;
    memset(&sa, 0, sizeof(sa));
    apply_sync(sa, p, sync);
    const void *src = srcs[0];
    for (int q = 0; q < G; ++q) {
        if (!srcs[q] || ((uintptr_t)srcs[q] % E)) {
            *err = "source buffers must be non-null and aligned to the element width";
            return VPG_EINVAL;
        }
        const int64_t diff = (int64_t)((uintptr_t)srcs[q] - (uintptr_t)src);
        sa.off[q] = diff / E;
    }
    if (!dst || (uintptr_t)dst % E) {
        *err = "destination buffer must be non-null and aligned to the element width";
        return VPG_EINVAL;
    }
    if (p->n == 0) return VPG_OK;
    vpg_status s = VPG_OK;
    switch (E) {
        case 1: s = launch_tile<1>(p, src, dst, sa, st); break;
        case 2: s = launch_tile<2>(p, src, dst, sa, st); break;
        case 4: s = launch_tile<4>(p, src, dst, sa, st); break;
        case 8: s = launch_tile<8>(p, src, dst, sa, st); break;
        case 16: s = launch_tile<16>(p, src, dst, sa, st); break;
        default: s = VPG_EUNSUPPORTED;
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

vpg_status launch_plan(const vpg_plan *p, const void *src, void *const *dsts, int ndst, void *stream,
                       std::string *err, const vpg_shard_sync *sync) {
    cudaStream_t st = (cudaStream_t)stream;
    const int E = p->elem_bytes;
    const int G = p->shards > 0 ? p->shards : 1;
    if (ndst != G) {
        *err = "plan expects " + std::to_string(G) + " destination shard(s)";
        return VPG_EINVAL;
    }
    void *dst = dsts[0];
    ShardArgs sa;
    memset(&sa, 0, sizeof(sa));
    apply_sync(sa, p, sync);
    for (int q = 0; q < G; ++q) {
        if (!dsts[q] || ((uintptr_t)dsts[q] % E)) {
            *err = "destination buffers must be non-null and aligned to the element width";
            return VPG_EINVAL;
        }
        const int64_t diff = (int64_t)((uintptr_t)dsts[q] - (uintptr_t)dst);
        sa.off[q] = diff / E;
    }
    if ((uintptr_t)src % E) {
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
                case 1: s = launch_tile<1>(p, src, dst, sa, st); break;
                case 2: s = launch_tile<2>(p, src, dst, sa, st); break;
                case 4: s = launch_tile<4>(p, src, dst, sa, st); break;
                case 8: s = launch_tile<8>(p, src, dst, sa, st); break;
                case 16: s = launch_tile<16>(p, src, dst, sa, st); break;
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


// Every rank of a fused exchange in one cooperative launch (see
// tile_kernel_ranks): per-rank parameter blocks, buffer bases and
// ShardArgs in device memory, flag blocks + counters allocated here, epoch 1.
template <int E>
static vpg_status launch_ranks(const vpg_plan *const *plans, int G, const void *const *srcs, void *const *dsts,
                               cudaStream_t st, std::string *err) {
    using W = typename WordOf<E>::T;
    const bool pull = plans[0]->tile.pull != 0;
    std::vector<TileParams> ps(G);
    std::vector<const W *> sv(G);
    std::vector<W *> dv(G);
    std::vector<ShardArgs> sas(G);
    const size_t flag_words = (size_t)G * 2 * G;
    void *mem = nullptr;
    const size_t bytes = flag_words * 8 + (size_t)G * 4 + 64;
    if (cudaMalloc(&mem, bytes) != cudaSuccess || cudaMemsetAsync(mem, 0, bytes, st) != cudaSuccess) {
        cudaGetLastError();
        *err = "cannot allocate the exchange flag blocks";
        return VPG_ENOMEM;
    }
    unsigned long long *flags = (unsigned long long *)mem;
    uint32_t *ctrs = (uint32_t *)(flags + flag_words);
    bool aligned = true;
    for (int r = 0; r < G; ++r) {
        if (((uintptr_t)srcs[r] | (uintptr_t)dsts[r]) % 16) aligned = false;
        if ((plans[r]->tile.shard_elems * E) % 16) aligned = false;
    }
    for (int r = 0; r < G; ++r) {
        const vpg_plan *p = plans[r];
        ps[r] = aligned ? p->tile : p->tile_unaligned;
        ShardArgs &sa = sas[r];
        memset(&sa, 0, sizeof(sa));
        for (int q = 0; q < G; ++q) {
            sa.off[q] = pull ? (int64_t)((uintptr_t)srcs[q] - (uintptr_t)srcs[0]) / E
                             : (int64_t)((uintptr_t)dsts[q] - (uintptr_t)dsts[0]) / E;
            sa.flags[q] = flags + (size_t)q * 2 * G;
        }
        // VPG_EMU_NO_BARRIER=1: same launch without the barrier (its cost, A/B)
        static const bool nobar = getenv("VPG_EMU_NO_BARRIER") && atoi(getenv("VPG_EMU_NO_BARRIER")) != 0;
        sa.epoch = nobar ? 0 : 1;
        sa.rank = (uint32_t)r;
        sa.done_ctr = ctrs + r;
        sv[r] = (const W *)(pull ? srcs[0] : srcs[r]);
        dv[r] = (W *)(pull ? dsts[r] : dsts[0]);
    }
    // one device block: parameter blocks, pointer tables, ShardArgs
    const size_t o_ps = 0, o_s = o_ps + sizeof(TileParams) * G, o_d = o_s + sizeof(void *) * G,
                 o_sa = (o_d + sizeof(void *) * G + 15) / 16 * 16, tot = o_sa + sizeof(ShardArgs) * G;
    std::vector<unsigned char> host(tot);
    memcpy(host.data() + o_ps, ps.data(), sizeof(TileParams) * G);
    memcpy(host.data() + o_s, sv.data(), sizeof(void *) * G);
    memcpy(host.data() + o_d, dv.data(), sizeof(void *) * G);
    memcpy(host.data() + o_sa, sas.data(), sizeof(ShardArgs) * G);
    void *dblk = nullptr;
    if (cudaMalloc(&dblk, tot) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(mem);
        *err = "cannot allocate the emulation tables";
        return VPG_ENOMEM;
    }
    cudaMemcpyAsync(dblk, host.data(), tot, cudaMemcpyHostToDevice, st);
    auto k = tile_kernel_ranks<W>;
    const int threads = plans[0]->threads;
    const int smem = (int)ps[0].smem_bytes;
    int nb = occupancy(k, threads, smem);
    int dev = 0, coop = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    const uint32_t per = (uint32_t)std::max<int64_t>(1, (int64_t)nb * sm_count_for_current() / G);
    const TileParams *a0 = (const TileParams *)((unsigned char *)dblk + o_ps);
    const W *const *a1 = (const W *const *)((unsigned char *)dblk + o_s);
    W *const *a2 = (W *const *)((unsigned char *)dblk + o_d);
    const ShardArgs *a3 = (const ShardArgs *)((unsigned char *)dblk + o_sa);
    void *args[] = {(void *)&a0, (void *)&a1, (void *)&a2, (void *)&a3, (void *)&per};
    vpg_status s = VPG_OK;
    if (!coop) {
        *err = "device does not support cooperative launches";
        s = VPG_EUNSUPPORTED;
    } else if (cudaLaunchCooperativeKernel((const void *)k, dim3(per * G), dim3(threads), args, (size_t)smem, st) !=
               cudaSuccess) {
        *err = std::string("cooperative launch failed: ") + cudaGetErrorString(cudaGetLastError());
        s = VPG_ECUDA;
    }
    cudaError_t e = cudaStreamSynchronize(st);
    if (s == VPG_OK && e != cudaSuccess) {
        *err = std::string("exchange emulation failed: ") + cudaGetErrorString(e);
        s = VPG_ECUDA;
    }
    cudaFree(dblk);
    cudaFree(mem);
    return s;
}

vpg_status launch_sharded_emulated(const vpg_plan *const *plans, int G, const void *const *srcs, void *const *dsts,
                                   void *stream, std::string *err) {
    for (int r = 0; r < G; ++r) {
        const vpg_plan *p = plans[r];
        if (!p || p->kernel_class != VPG_KERNEL_TILE || p->shards != G || p->shard_index != r ||
            (p->tile.pull != 0) != (plans[0]->tile.pull != 0) || p->elem_bytes != plans[0]->elem_bytes ||
            p->tile.bulk) {
            *err = "plans[r] must be rank r's exchange plan of one push or pull exchange over nplans shards";
            return VPG_EINVAL;
        }
        if (!srcs[r] || !dsts[r] || (uintptr_t)srcs[r] % p->elem_bytes || (uintptr_t)dsts[r] % p->elem_bytes) {
            *err = "buffers must be non-null and aligned to the element width";
            return VPG_EINVAL;
        }
    }
    cudaStream_t st = (cudaStream_t)stream;
    switch (plans[0]->elem_bytes) {
        case 4: return launch_ranks<4>(plans, G, srcs, dsts, st, err);
        case 8: return launch_ranks<8>(plans, G, srcs, dsts, st, err);
        default: *err = "the exchange emulation supports 4- and 8-byte words"; return VPG_EUNSUPPORTED;
    }
}

}  // namespace vpg
