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
    int32_t jit;               // TILE: launch the NVRTC-specialised kernel (jit.cpp)
    vpg::TileParams tile;
    vpg::TileParams tile_unaligned;   // same tile, scalar source reads
    vpg::RowsParams rows;
    vpg::CopyParams copy;
    vpg::GatherParams gather;
    std::string text;          // describe() output
};

namespace vpg {
// kernels.cu
vpg_status launch_plan(const vpg_plan *p, const void *src, void *dst, void *stream, std::string *err);
cudaKernel_t jit_tile_kernel(const vpg_plan *p);
void jit_forget(const vpg_plan *p);
int jit_state(const vpg_plan *p);
const char *jit_last_log();
std::string jit_source(const vpg_plan *p);
bool jit_compile_check(const vpg_plan *p, std::string *log);
int device_sm_count();
}  // namespace vpg
