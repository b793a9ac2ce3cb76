/*
 * vpgpu.h -- C ABI of the B200 (sm_100a) N-D tensor permutation library
 * (libvpgpu.so).  Drop-in boundary for the permutation hot path of the
 * reference package `vecperm` (/root/reference/pkg).
 *
 * Conventions (identical to the reference, core.py:1-7):
 *   - dims are innermost-first: dims[0] is the stride-1 dimension;
 *   - sigma[j] is the SOURCE dim that lands at DESTINATION position j
 *     (inner-first), so the output's innermost dim is source dim sigma[0];
 *   - output layout: out.dims[j] = dims[sigma[j]], dense (core.py:128-132);
 *   - bijection: out[i] = in[f(i)] (core.py:173-178, 192-204);
 *   - elements are opaque words of elem_bytes bytes.  The reference accepts
 *     4 and 8 (core.py:29); this library accepts 1, 2, 4, 8 and 16.
 *
 * Buffers are DEVICE pointers owned by the caller (e.g. torch tensors).
 * The library never allocates tensor memory.  src and dst must not overlap
 * (out-of-place only, as the reference).  Unlike the reference's emitted
 * kernels (emit.py:5-8) there is NO slack requirement past either buffer.
 *
 * Threading: plans are immutable after creation and may be shared between
 * host threads; vpg_permute may be called concurrently on distinct streams.
 * vpg_last_error() is thread-local.
 */
#ifndef VPGPU_H
#define VPGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VPG_ABI_VERSION 6   /* 6: TileParams gains LinDesc (vpg_plan_tile_params block) */
#define VPG_MAX_RANK 64
#define VPG_MAX_SHARDS 64   /* shards of a fused exchange */

typedef enum {
    VPG_OK = 0,
    VPG_EINVAL = 1,        /* bad layout / map / buffer: maps to LayoutError (core.py:32-33) */
    VPG_EUNSUPPORTED = 2,  /* valid request the library cannot serve (e.g. > 2^32 tiles)     */
    VPG_ECUDA = 3,         /* CUDA runtime error: maps to RuntimeError                         */
    VPG_ENOMEM = 4
} vpg_status;

/* Kernel classes chosen by the planner. */
typedef enum {
    VPG_KERNEL_COPY = 0,     /* merged to rank 1: vectorised flat copy                      */
    VPG_KERNEL_ROWS = 1,     /* K1: stride-1 preserved, long rows: 128-bit copy-with-remap  */
    VPG_KERNEL_TILE = 2,     /* K2/K3: smem-staged tile transpose over merged/odd dims      */
    VPG_KERNEL_GATHER = 3    /* K0: per-element gather (tiny tensors / forced)              */
} vpg_kernel_class;

typedef struct vpg_plan vpg_plan;   /* opaque, immutable */

/* Summary of a plan (the format_plan / IRProgram.metadata analog,
 * planner.py:386-419, ir.py:96-108). */
typedef struct {
    int32_t kernel_class;           /* vpg_kernel_class */
    int32_t elem_bytes;
    int32_t rank;                   /* after merge_dimensions */
    int64_t dims[VPG_MAX_RANK];     /* merged dims, inner-first */
    int32_t sigma[VPG_MAX_RANK];    /* merged sigma, inner-first */
    int64_t num_elements;
    /* TILE: tile geometry */
    int64_t tile_elems;             /* elements in one full tile */
    int64_t src_run;                /* contiguous source run (elements) */
    int64_t dst_run;                /* contiguous destination run (elements) */
    int64_t num_tiles;
    int32_t smem_pitch;             /* padded source-run pitch in smem (elements) */
    int32_t smem_bytes;             /* dynamic shared memory per CTA */
    /* ROWS/COPY: vector width in elements; TILE: 1 */
    int32_t vec_elems;
    int32_t threads;                /* CTA size */
    int64_t grid_hint;              /* CTAs launched when the device has 148 SMs */
    double  predicted_efficiency;   /* planner's sector-efficiency estimate, 0..1 */
    int32_t host_chunks;            /* vpg_permute_host pipeline chunks (0 = single shot) */
    int32_t jit_state;              /* 0 no specialisation, 1 pending, 2 specialised kernel loaded, -1 failed */
    int32_t shards;                 /* sharded exchange plans: G (0 = ordinary plan) */
    int32_t shard_index;            /* sharded exchange plans: this plan's input shard */
} vpg_plan_info;

/* Library ABI version (VPG_ABI_VERSION). */
int vpg_version(void);

/* Thread-local message for the last non-OK status on this thread. */
const char *vpg_last_error(void);

/* Replaces vecperm.planner.merge_dimensions (planner.py:211-241): drops
 * size-1 dims and fuses adjacent dims whose adjacency and order survive the
 * map.  out_dims/out_sigma must hold `rank` entries. */
vpg_status vpg_merge_dimensions(int rank, const int64_t *dims, const int32_t *sigma,
                                int *out_rank, int64_t *out_dims, int32_t *out_sigma);

/* Replaces vecperm.ir.build_program (ir.py:441-456): merge + classify +
 * tile selection for (shape, map, element width).  Host-only; needs no GPU.
 * `flags`: 0 = planner's choice; VPG_FORCE_* to pin a kernel class (tests). */
#define VPG_FORCE_GATHER 0x1
#define VPG_FORCE_TILE   0x2
#define VPG_NO_MERGE     0x4
#define VPG_FORCE_JIT    0x8    /* TILE: always use the per-case NVRTC-specialised kernel  */
#define VPG_NO_JIT       0x10   /* TILE: always use the ahead-of-time kernel                */
#define VPG_SHARD_PULL   0x20   /* sharded plans: pull exchange (see vpg_permute_sharded_pull) */
/* TILE: use the n-th best tile candidate of the planner's cost model
 * (n >= 0); plan creation fails with VPG_EUNSUPPORTED past the last one.
 * Autotuners time a few candidates and keep the fastest. */
#define VPG_TILE_CANDIDATE(n) ((unsigned)(((n) + 1) & 0xff) << 8)
vpg_status vpg_plan_create(int rank, const int64_t *dims_inner_first,
                           const int32_t *sigma_inner_first, int elem_bytes,
                           unsigned flags, vpg_plan **out);

/* Replaces the emitted kernel `void permute_<hash>(const void *src, void *dst)`
 * (emit.py:118-128, 212-266) and the VM's execute (vm.py:105-110):
 * dst = permute(src) on device memory, asynchronously on `cuda_stream`
 * (a cudaStream_t; NULL = legacy default stream). */
vpg_status vpg_permute(const vpg_plan *plan, const void *src, void *dst, void *cuda_stream);

/* End-to-end variant over HOST buffers (the reference's execute() takes a host
 * buffer, vm.py:105-110): copies host_src -> dev_src, permutes into dev_dst,
 * copies dev_dst -> host_dst -- chunked and pipelined over the library's
 * copy/compute streams for large tensors -- ordered after earlier work on
 * `cuda_stream`, and synchronises that stream before returning.  Device
 * buffers are caller-provided scratch of num_elements*elem_bytes bytes
 * each; calls from several host threads may share them (the library orders
 * every writer of a scratch buffer after its earlier readers).  Pinned host
 * memory gives full-rate copies. */
vpg_status vpg_permute_host(const vpg_plan *plan, const void *host_src, void *host_dst,
                            void *dev_src, void *dev_dst, void *cuda_stream);

/* Asynchronous variant of vpg_permute_host: enqueues the chunked
 * H2D -> permute -> D2H pipeline on the library's copy/compute streams and
 * returns; completion is ordered on `cuda_stream` (synchronise it before
 * reading host_dst).  Consecutive calls overlap: the H2D of call k+1 runs
 * while the D2H of call k drains.  Reusing the same device scratch between
 * calls is safe (the library orders writers after earlier readers), and so
 * is feeding an earlier call's host_dst back as host_src (the H2D waits for
 * that D2H).  The call does not wait for other earlier work on cuda_stream:
 * host buffers must be ready and stay alive and unmodified until
 * completion, and the scratch must not be used by other in-flight work. */
vpg_status vpg_permute_host_async(const vpg_plan *plan, const void *host_src, void *host_dst,
                                  void *dev_src, void *dev_dst, void *cuda_stream);

/* Host buffers larger than the device: the permutation is cut into chunks
 * along dims that are outer on both sides and streamed through a ring of
 * slots in `dev_scratch` (scratch_bytes of device memory; each slot holds
 * one input and one output chunk, chunks are at most an eighth of the
 * scratch).  Synchronous.  VPG_EUNSUPPORTED when the tensor cannot be cut
 * finely enough for the scratch. */
vpg_status vpg_permute_host_bounded(const vpg_plan *plan, const void *host_src, void *host_dst,
                                    void *dev_scratch, size_t scratch_bytes, void *cuda_stream);

/* One-shot convenience with an internal plan cache keyed by
 * (dims, sigma, elem_bytes): the closest analog of the reference's
 * shape-specialised kernel call. */
vpg_status vpg_permute_nd(int rank, const int64_t *dims_inner_first,
                          const int32_t *sigma_inner_first, int elem_bytes,
                          const void *src, void *dst, void *cuda_stream);

/* Fused sharded exchange.  The tensor (dims, sigma as
 * in vpg_plan_create) is split into `shards` contiguous input shards and
 * `shards` contiguous output shards of num_elements/shards elements each:
 * input shard r is flat input [r*N/G, (r+1)*N/G), output shard q is flat
 * output [q*N/G, (q+1)*N/G) -- the leading-axis sharding of both sides.
 * A plan for input shard `shard_index` permutes that shard with ONE kernel
 * that stores every tile straight into the output shard that owns it:
 * dst_shards[q] is shard q's buffer as seen from this device (the local
 * buffer for q == shard_index, CUDA IPC / peer-mapped pointers over
 * NVLink/NVSwitch for the others).  No staging buffer, no collective.
 * Requires the leading dims on each side to split into factors whose
 * product is `shards` (VPG_EUNSUPPORTED otherwise, as when no tile avoids
 * the shard-indexing dims).  The caller orders the exchange: every shard's
 * buffer must be free before any rank launches, and no rank may read its
 * output before every rank's kernel has completed (e.g. a device-side
 * barrier such as a one-element NCCL all-reduce on each side).
 * shards <= 64. */
vpg_status vpg_plan_create_sharded(int rank, const int64_t *dims_inner_first,
                                   const int32_t *sigma_inner_first, int elem_bytes,
                                   unsigned flags, int shards, int shard_index, vpg_plan **out);
vpg_status vpg_permute_sharded(const vpg_plan *plan, const void *src_shard,
                               void *const *dst_shards, void *cuda_stream);

/* Pull variant of the fused exchange (plans created with VPG_SHARD_PULL;
 * shard_index then names the OUTPUT shard this plan produces).  ONE kernel
 * per rank reads the source runs of its output tiles straight from every
 * input shard -- src_shards[q] is input shard q's buffer as seen from this
 * device (peer-mapped pointers over NVLink/NVSwitch for q != own) -- and
 * writes its local output shard.  Destination runs are local, so the plan
 * keeps long runs on both sides even when an input-shard axis is the
 * output's second-innermost axis (where the push exchange would store
 * 16-byte runs across ranks).  Ordering as for vpg_permute_sharded: every
 * input shard must be complete before any rank launches, and no input shard
 * may be overwritten before every rank's kernel has completed. */
vpg_status vpg_permute_sharded_pull(const vpg_plan *plan, const void *const *src_shards,
                                    void *dst_shard, void *cuda_stream);

/* Device-side ordering of a fused exchange, instead of the caller's
 * barriers around the launch (replaces the two one-element all-reduces
 * the reference's SPEC.md:181 partitioned execution would need per step):
 *   flags[q]     rank q's flag block as seen from this device: 2 x shards
 *                uint64, zero-initialised once, CUDA IPC / peer-mapped for
 *                q != own (NVLink/NVSwitch);
 *   epoch        this call's value, greater than every earlier call's on
 *                the same flag blocks (e.g. a per-exchange call counter + 1);
 *   done_counter a zero uint32 in this device's memory (left zero).
 * The kernel starts reading/writing peer shards only after every rank's
 * kernel has started, and completes only after every rank's accesses have
 * finished, so stream order on each rank is the whole ordering.  All ranks
 * must launch with the same epoch.  Waits are bounded (~4 s). */
typedef struct vpg_shard_sync {
    unsigned long long *flags[VPG_MAX_SHARDS];
    unsigned long long epoch;
    unsigned int *done_counter;
} vpg_shard_sync;

/* Fused exchange step with optional device-side ordering (sync may be NULL:
 * then as vpg_permute_sharded / vpg_permute_sharded_pull).  Push plans:
 * src_shards[0] = this rank's input shard, dst_shards[q] = output shard q.
 * Pull plans: src_shards[q] = input shard q, dst_shards[0] = this rank's
 * output shard.  Replaces: the exchange step of the reference's
 * outer-counter-partitioned execution. */
vpg_status vpg_permute_sharded_sync(const vpg_plan *plan, const void *const *src_shards,
                                    void *const *dst_shards, const vpg_shard_sync *sync, void *cuda_stream);

/* Every rank of a fused exchange on ONE device in one cooperative launch,
 * with the device-side ordering above between the ranks (flag blocks and
 * counters allocated internally; returns after the step has finished).
 * plans[r] = rank r's plan (all push or all pull, same arguments),
 * src_shards[r] / dst_shards[r] = rank r's input / output shard.  Validates
 * the exchange protocol on single-GPU machines; a multi-GPU job runs one
 * vpg_permute_sharded_sync per rank instead. */
vpg_status vpg_permute_sharded_emulated(const vpg_plan *const *plans, int nplans, const void *const *src_shards,
                                        void *const *dst_shards, void *cuda_stream);

/* CUDA IPC for the exchange's peer table: export a device pointer (any
 * pointer inside a cudaMalloc allocation) as a VPG_IPC_HANDLE_BYTES handle
 * plus offset, import it in another process on this or a peer GPU (mapped
 * with lazy peer access), release the mapping. */
#define VPG_IPC_HANDLE_BYTES 64
vpg_status vpg_ipc_export(const void *dev_ptr, void *handle, uint64_t *offset);
vpg_status vpg_ipc_import(const void *handle, uint64_t offset, void **dev_ptr);
vpg_status vpg_ipc_release(void *dev_ptr);

/* Plan inspection (format_plan analog, planner.py:386-419). */
vpg_status vpg_plan_info_get(const vpg_plan *plan, vpg_plan_info *info);
vpg_status vpg_plan_describe(const vpg_plan *plan, char *buf, size_t len);

/* Generated CUDA source of the per-case specialised tile kernel (the
 * reference's emit_source, emit.py:343-363: shape, map and element width
 * baked in; kernel cubins are cached under an fnv1a64 name like
 * kernel_name, emit.py:118-128).  TILE plans only. */
vpg_status vpg_plan_emit_source(const vpg_plan *plan, char *buf, size_t len);

/* Compile the specialised source with NVRTC without loading it (needs no
 * GPU; the analog of verify_native's compile step, emit.py:444-483). */
vpg_status vpg_plan_jit_compile(const vpg_plan *plan);

/* Raw kernel parameter block of a TILE plan (inspection / host-side
 * validation of the tile walk, tests/sim_tile.py -- the analog of the
 * reference VM's role of checking a program before hardware runs it). */
vpg_status vpg_plan_tile_params(const vpg_plan *plan, void *buf, size_t len, size_t *needed);

void vpg_plan_destroy(vpg_plan *plan);

#ifdef __cplusplus
}
#endif

#endif /* VPGPU_H */
