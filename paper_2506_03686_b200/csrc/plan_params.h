// plan_params.h -- POD parameter blocks of the permutation kernels.
//
// Device-safe (no STL): included by the AOT kernels (kernels.cu), by the
// host planner (through plan.h) and -- as text -- by the run-time
// specialised kernels compiled with NVRTC (jit.cpp), which embed a
// TileParams block as constant bytes so every extent, stride and divisor
// folds into immediates (GenTT's per-case code generation on the GPU).
#pragma once

#ifdef __CUDACC_RTC__
typedef unsigned char uint8_t;
typedef short int16_t;
typedef unsigned short uint16_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef long long int64_t;
typedef unsigned long long uint64_t;
typedef unsigned long long uintptr_t;
#else
#include <stdint.h>
#endif

namespace vpg {

// Merged ranks are bounded by log2(numel) since size-1 dims are dropped:
// 40 covers any tensor that fits in HBM (2^40 elements).
constexpr int kMaxRank = 40;
// Dims inside one tile (each >= 2 after merge, tile <= 2^14 elements).
constexpr int kMaxTileDims = 16;

// Division by a run-time invariant 32-bit divisor via multiply-high
// (round-up method): q = (umulhi(n, m) + n) >> s, exact for all n < 2^32.
struct FastDiv {
    uint32_t d;
    uint32_t m;
    uint32_t s;
};

#ifndef __CUDACC_RTC__
inline FastDiv make_fastdiv(uint32_t d) {
    uint32_t l = 0;
    while (l < 32 && (1ull << l) < d) ++l;
    uint64_t m = (((1ull << 32) * ((1ull << l) - d)) / d) + 1;
    FastDiv f;
    f.d = d;
    f.m = (uint32_t)m;
    f.s = l;
    return f;
}

inline uint32_t host_fastdiv(uint32_t n, FastDiv f) {
    uint64_t t = ((uint64_t)n * f.m) >> 32;
    return (uint32_t)((t + n) >> f.s);
}
#endif

// --------------------------------------------------------------------------
// TILE (K2/K3) parameters.
//
// The tile is a sub-box of the merged tensor made of
//   * the source run: dims 0..s-1 in source order, the last possibly
//     partial (extent e < d): one contiguous source range of Ls elements;
//   * the destination run: dims sigma[0..t-1], the last possibly partial:
//     one contiguous destination range of Ld elements;
//   * the union of both (the tile).  Tile elements are staged in shared
//     memory in source order with the run pitch padded to kill bank
//     conflicts on the transposed side.
// The remaining dims (and the tile positions along partial dims) form the
// grid digits, ordered by destination stride (fastest first) like the
// reference's counter digits (planner.py:324-342).
//
// Each of the two phases (R: global->smem in source order, W: smem->global
// in destination order) walks the tile as a separable 3-level nest so the
// per-element work is two adds, one predicate and the memory op:
//   thread part  -- the first phase dims (partial last one, factor f),
//                   decoded once per CTA: per-thread global/smem offsets;
//   inner dim    -- one dim with constant strides (stepped by f when it is
//                   the split dim), unrolled;
//   outer dims   -- the rest, through a per-CTA table in shared memory.
// Threads beyond one thread part form G groups that share the outer loop.
constexpr unsigned kSwzAddr = 16; // PhaseDesc::swz: chunk ^= 128-byte block index (row-layout independent)
constexpr int kNumSlots = 3;      // checked coordinates: 0 = dim a, 1 = dim c, 2 = split padding
constexpr int kMaxPhaseDims = 12; // thread-part / outer dims per phase
constexpr unsigned long long kOuterEntryBytes = 24;  // sizeof(OuterEntry) in tile_body.cuh

struct GridDigit {
    FastDiv cum;         // divides tile index by the product of faster digits
    FastDiv ext;         // divides by this digit's extent
    int64_t src_stride;  // elements, already multiplied by the tile extent
    int64_t dst_stride;
};

struct PhaseDim {
    int64_t gstride;     // global stride (elements; src for R, dst for W)
    FastDiv div;         // divides by extent
    uint32_t sstride;    // smem stride (elements)
    int16_t slot;        // coordinate slot fed by this dim (-1 none)
    uint16_t cmul;       // coordinate units per step (V for vector-grouped dims)
    uint16_t hmul;       // W in shifted-run mode: source-alignment shift per step (mod V)
    uint16_t pad_;
};

struct PhaseDesc {
    uint32_t nthr;                 // threads in one thread part (NTP)
    uint32_t ngroups;              // G
    int32_t nthr_dims;
    PhaseDim thr[kMaxPhaseDims];    // thread-part dims (fastest first)
    uint32_t n_in;                 // inner-dim steps
    int64_t g_in;                  // inner-dim global stride per step
    uint32_t s_in;                 // inner-dim smem stride per step
    uint32_t c_in[kNumSlots];      // inner-dim coordinate increment per slot
    uint32_t n_outer;
    int32_t nout_dims;
    PhaseDim out[kMaxPhaseDims];    // outer dims (fastest first)
    uint32_t vec;                  // elements per access: 1, or V = 16/E (16-byte accesses)
    uint32_t rshift;               // R: source runs read as 16-byte aligned supersets (misaligned runs);
                                   // 2 = residue row strides (TileParams::rres)
    uint32_t h_in;                 // W in shifted-run mode: shift increment per inner step
    int64_t vstride;               // W with vec > 1: global stride between the V elements
    uint32_t mask_full;            // slots checked in every tile (padding)
    uint32_t mask_ragged;          // slots checked in ragged tiles
    uint32_t off_tab;              // smem byte offset of this phase's outer table
    // 16-byte chunk swizzle of the smem rows.  Chunk j of row r = s / pitch
    // lives at chunk j ^ ((r >> (swz - 1)) & 7), so the W lanes, which read
    // one column across consecutive rows, spread over all banks (swz = 0:
    // off; pitch is a multiple of 8 chunks).  Shifted-run mode (opt-in), and
    // the 128-byte congruent layout of aligned runs: unpadded rows at the
    // same offset modulo 128 bytes as their source lines, so per-lane
    // cp.async requests each L2 sector once (a padded row makes the LDGSTS
    // split every line: ~2x L2 sector reads, tools/ldgsts_probe.cu)
    uint32_t swz;                  // (kSwzAddr: address swizzle, see swizzle() in tile_body.cuh)
    FastDiv spitch;                // divides an smem element offset by the pitch
    // W with vec > 1 and w2 = 1 (congruent swizzled layout only): each
    // position is a V x V block -- V smem vectors (V consecutive dim-0
    // elements each) from V consecutive destination-innermost rows vrow
    // elements apart, transposed in registers into V 16-byte stores of V
    // consecutive destination elements, vstride apart.  Lanes walk the
    // destination-innermost groups, so each store instruction writes 512
    // contiguous bytes; the swizzle keys on the row group (swz = 1 + log2 V),
    // so those lanes' smem vectors fall on distinct banks.
    uint32_t w2;                   // 1: V x V blocks; 2..8: k x V interleave blocks; kW2Gather: gather blocks
    uint32_t vrow;
};
// PhaseDesc::w2 values of the gather W mode: g destination-innermost elements
// (g smem rows vrow apart, scalar loads) packed into one store of g words.
// kW2Gather: g = V (16-byte stores); kW2Gather + g, g = 2, 4, 8 < V: narrower
// blocks (4- and 8-byte stores) for 1- and 2-byte words whose
// destination-innermost extent is a multiple of g but not of V.
constexpr uint32_t kW2Gather = 64;

// W phase as destination-linear 16-byte chunks ("lin" mode), for tiles whose
// destination runs are misaligned or not a multiple of V = 16/E elements
// long (cfg3: 270-element runs at arbitrary 4-byte offsets).  Each thread
// takes V-element chunk slots q = tid, tid + nt, ...: run r = q / cpr, slot
// c = q % cpr.  Slot c of a run whose first element sits at m = (address / E)
// mod V covers run positions j = c*V - m .. c*V - m + V-1, i.e. the 16-byte
// aligned destination chunk that contains them: V shared-memory loads and
// ONE 16-byte store when all V positions are inside the run (head and tail
// chunks store element by element).  Every store instruction of a warp then
// covers whole 32-byte sectors, where a scalar walk of a misaligned run
// splits every sector between two instructions.  The shared-memory offset
// of run position j comes from a per-plan table built once per CTA:
// u16 entries tab[m][c][e] = offset(c*V - m + e) (V shifted copies, so one
// aligned V*2-byte load fetches a chunk's V offsets).
constexpr int kMaxLinDims = 8;
struct LinDesc {
    uint32_t on;
    uint32_t nt;                  // CTA threads the walk is laid out for
    uint32_t run_len;             // elements of a full destination run
    uint32_t cpr;                 // chunk slots per run: ceil((run_len + V - 1) / V)
    FastDiv cprd;                 // divides by cpr
    uint32_t nchunks;             // nruns * cpr
    int32_t nrd;                  // destination-run dims (fastest first)
    int32_t nxd;                  // run-index dims (fastest first)
    int32_t last_slot;            // checked slot (0 = a, 1 = c) of the last run dim, -1 none
    uint32_t last_unit;           // run positions per step of the last run dim
    uint32_t tab_off;             // smem byte offset of the u16 offset tables (V * cpr * V entries)
    // bank spreading: shared-memory load k of lane l fetches chunk element
    // (k + (l >> rot_shift)) mod V (rotated back in registers before the
    // store); the planner picks the shift with the fewest wavefronts
    // (residue layouts fix every row stride modulo 32 banks, so the lanes'
    // positions are the only freedom).  32 = no rotation.
    uint32_t rot_shift;
    PhaseDim rd[kMaxLinDims];     // run dims: div = extent, sstride (gstride unused: contiguous)
    PhaseDim xd[kMaxPhaseDims];   // run-index dims: gstride = destination stride, sstride, slot
};

struct TileParams {
    int64_t n_elems;              // elements of the whole tensor (source bounds in shifted-run mode)
    uint32_t num_tiles;
    int32_t ngrid;
    uint32_t Ls, Ld;               // source / destination run lengths (elements)
    uint32_t T;                    // tile elements
    uint32_t pitch;                // smem pitch of one source run (elements, >= Ls)
    uint32_t tile_elems_alloc;     // elements of one smem tile buffer (Ns * pitch)
    // ragged boundary dims: a = source-run boundary, c = destination-run boundary
    int32_t grid_a, grid_c;        // grid digit carrying the tile position along a / c (-1: not partial)
    uint32_t e_a, d_a, e_c, d_c;
    uint32_t lim_split[2];         // static limit of slot 2 per phase (R, W)
    uint32_t hmask;                // shifted-run mode: V-1 (source runs sit at offset h in their smem row), else 0
    // bulk mode: the R phase is one cp.async.bulk (TMA bulk copy) per source
    // run, issued by a producer warp and tracked by mbarriers
    uint32_t bulk;
    uint32_t nruns;                // source runs per tile
    int32_t nrdims;
    uint32_t run_bytes;            // full run length in bytes
    uint32_t run_unit_bytes;       // bytes per step of the partial source-boundary dim a
    PhaseDim rdims[kMaxPhaseDims]; // run-index dims: gstride = src stride, sstride = smem row offset
    PhaseDesc ph[2];               // 0 = R (read), 1 = W (write)
    GridDigit grid[kMaxRank];
    uint32_t off_buf;              // smem byte offset of the tile buffers
    uint32_t nbuf;                 // 1 or 2 (double-buffered cp.async)
    uint32_t persistent;           // 1: grid = resident CTAs, 0: one CTA per tile
    uint32_t smem_bytes;
    // fused sharded exchange (nshards > 1): the tensor is split into nshards
    // contiguous input shards and nshards contiguous output shards.  This
    // plan walks the tiles [tile_begin, tile_begin + num_tiles) of the global
    // tile grid -- exactly the tiles whose source lies in input shard
    // (src_bias / shard_elems), because the input-shard digits are the
    // slowest grid digits -- reads them from the local shard (source offsets
    // minus src_bias) and stores each tile straight into output shard
    // q = dst / shard_elems through ShardArgs::off[q] (peer memory).
    uint32_t nshards;
    uint32_t tile_begin;
    int64_t src_bias;
    int64_t shard_elems;
    // shifted-run mode with residue row strides (rshift == 2): V-1, else 0.
    // Run-index dims have smem strides congruent to their source strides
    // modulo V and each tile buffer is used from offset (source tile base &
    // rres), so a misaligned run sits at the same offset modulo V in shared
    // and global memory: R copies 16-byte aligned chunks to 16-byte aligned
    // smem, W reads at affine offsets (no per-element shift, hmask == 0).
    uint32_t rres;
    // pull exchange (nshards > 1, pull = 1): this plan produces output shard
    // (dst_bias / shard_elems) and reads its source runs from every input
    // shard.  Source offsets stay global; each 16-byte chunk or element at
    // global offset o is read from input shard q = o / shard_elems (a shift
    // when shard_shift != 0, else shard_div) through ShardArgs::off[q]
    // (relative to src).  Destination offsets are rebased by dst_bias onto
    // the local output shard.
    uint32_t pull;
    uint32_t shard_shift;
    FastDiv shard_div;
    uint32_t pad_pull_;
    int64_t dst_bias;
    // largest source offset of any element of a full tile relative to the
    // tile's source base, + 1: a tile whose base + src_span + 16 bytes of
    // elements stays inside the source needs no end-of-buffer check on its
    // aligned-superset reads (shifted-run mode), so its R walk is branch-free
    int64_t src_span;
    LinDesc lin;
};
// (kernel parameters beyond 4 KB need CUDA >= 12.1; the ShardArgs block
// next to it already does)
static_assert(sizeof(TileParams) <= 8192, "kernel parameter block must stay under 8 KB");

// Per-launch destination table of a sharded tile plan: element offset of
// output shard q relative to the kernel's dst pointer (shard 0).  Passed by
// value next to the parameter block (CUDA >= 12.1 kernel parameter space).
constexpr int kMaxShards = 64;
struct ShardArgs {
    int64_t off[kMaxShards];
    // dynamic tile scheduler (tile kernels): a {next, done} counter pair from
    // the per-device ring (kernels.cu sched_slot), zero at launch and reset
    // by the last CTA; nullptr = static round-robin tiles
    uint32_t *sched;
    // development tracing (VPG_TRACE, kernels.cu): per-CTA globaltimer
    // records of the tile pipeline; nullptr in normal launches
    unsigned long long *trace;
    // device-side exchange barrier (sharded plans, epoch != 0; tile_body.cuh
    // shard_barrier_*): flags[q] = rank q's flag block as seen from this
    // device (2 x nshards u64: [0, G) "rank r started", [G, 2G) "rank r's
    // accesses done"), monotonically increasing epoch per exchange call,
    // this plan's rank, and a local CTA-completion counter (zero between calls)
    unsigned long long *flags[kMaxShards];
    unsigned long long epoch;
    uint32_t rank;
    uint32_t *done_ctr;
};
constexpr int kTraceWords = 64;     // per CTA: start, prologue issued, end, smid, (tile, data ready, written) x 19; [62] first load issue; [63] tiles

// --------------------------------------------------------------------------
// ROWS (K1): stride-1 preserved; each destination row of Lr elements is a
// contiguous source row.  Row q (destination order) starts at q*Lr in dst
// and at sum_j digit_j(q) * in_stride[sigma[j]] in src.
struct RowDigit {
    FastDiv ext;
    int64_t src_stride;
};

struct RowsParams {
    uint32_t nrows;
    uint32_t row_vecs;         // Lr / V
    uint32_t vec;              // V: elements per vector
    uint32_t tpr_log2;         // threads per row group (log2)
    int64_t row_len;           // Lr (elements)
    int32_t ndig;
    // work items: each row is cut into nchunks chunks of chunk_vecs vectors
    // (the last one shorter) so that few long rows still fill the GPU
    uint32_t chunk_vecs;
    FastDiv nchunks;
    uint32_t nitems;           // nrows * nchunks
    RowDigit dig[kMaxRank];    // destination dims 1..r-1, fastest first
};

// --------------------------------------------------------------------------
// COPY: merged to rank 1.
struct CopyParams {
    int64_t n;                 // elements
};

// --------------------------------------------------------------------------
// GATHER (K0): out[i] = in[f(i)], per element (core.py:173-178).
struct GatherParams {
    uint32_t n;
    int32_t rank;
    FastDiv ext[kMaxRank];     // destination dims, fastest first
    int64_t src_stride[kMaxRank];
};

}  // namespace vpg
