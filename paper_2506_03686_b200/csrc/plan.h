// plan.h -- internal plan representation shared by the host planner
// (planner.cpp) and the sm_100a kernels (kernels.cu).
//
// A plan is the GPU analog of the reference's BlockPlan + IRProgram
// (/root/reference/pkg/src/vecperm/planner.py:86-201, ir.py:96-108): it
// carries the merged problem, the kernel class and a POD parameter block
// that is passed BY VALUE as the kernel argument (no device-side plan
// memory, so a plan is valid on every device and needs no GPU to build).
#pragma once

#include <stdint.h>
#include <string>
#include <vector>

#include "vpgpu.h"
#include <cuda_runtime.h>

#include "plan_params.h"


struct vpg_plan {
    int32_t kernel_class;      // vpg_kernel_class
    int32_t elem_bytes;
    int32_t rank;              // merged
    int64_t dims[VPG_MAX_RANK];
    int32_t sigma[VPG_MAX_RANK];
    int64_t n;
    int32_t threads;
    int64_t grid_hint;
    double predicted_eff;
    double tile_util;
    // TILE: the cost model's terms for the chosen tile (describe(); planner
    // calibration data, tools/cand_data.py)
    double geom_cost, walk_cost, eff_s, eff_d;
    int32_t jit;               // TILE: launch the NVRTC-specialised kernel (jit.cpp)
    int32_t shards;            // 0: ordinary plan; G >= 1: fused sharded exchange plan of rank shard_index
    int32_t shard_index;
    vpg::TileParams tile;
    vpg::TileParams tile_unaligned;   // same tile, scalar source reads
    vpg::RowsParams rows;
    vpg::CopyParams copy;
    vpg::GatherParams gather;
    std::string text;          // describe() output
};

namespace vpg {
// planner.cpp
int merge_dims(int rank, const int64_t *dims, const int32_t *sigma, int64_t *od, int32_t *os,
               const uint8_t *pin = nullptr, uint8_t *opin = nullptr);
// shards > 0: fused sharded exchange plan for input shard shard_index
bool squeeze_unit_dims(int &rank, const int64_t *&dims, const int32_t *&sigma, std::vector<int64_t> &sd,
                       std::vector<int32_t> &ss, std::string *err);
vpg_status make_plan(int rank, const int64_t *dims, const int32_t *sigma, int E, unsigned flags,
                     vpg_plan **out, std::string *err, int shards = 0, int shard_index = 0);
// ipc.cpp
vpg_status ipc_export(const void *ptr, void *handle, uint64_t *offset, std::string *err);
vpg_status ipc_import(const void *handle, uint64_t offset, void **ptr, std::string *err);
vpg_status ipc_release(void *ptr, std::string *err);
// kernels.cu
// dsts: one destination per output shard (1 for ordinary plans)
vpg_status launch_plan(const vpg_plan *p, const void *src, void *const *dsts, int ndst, void *stream,
                       std::string *err, const vpg_shard_sync *sync = nullptr);
// pull exchange plans: srcs = every input shard's buffer, dst = the local output shard
vpg_status launch_plan_pull(const vpg_plan *p, const void *const *srcs, void *dst, void *stream, std::string *err,
                            const vpg_shard_sync *sync = nullptr);
vpg_status launch_sharded_emulated(const vpg_plan *const *plans, int G, const void *const *srcs, void *const *dsts,
                                   void *stream, std::string *err);
inline vpg_status launch_plan(const vpg_plan *p, const void *src, void *dst, void *stream, std::string *err) {
    return launch_plan(p, src, &dst, 1, stream, err);
}
cudaKernel_t jit_tile_kernel(const vpg_plan *p);
void jit_forget(const vpg_plan *p);
int jit_state(const vpg_plan *p);
const char *jit_last_log();
std::string jit_source(const vpg_plan *p);
bool jit_compile_check(const vpg_plan *p, std::string *log);
int device_sm_count();
}  // namespace vpg
