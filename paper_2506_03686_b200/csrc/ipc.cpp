// ipc.cpp -- CUDA IPC helpers for the fused sharded exchange's peer table
// (include/vpgpu.h vpg_ipc_*).  One process per GPU: each rank exports its
// output shard, imports the others' and passes the mapped pointers to
// vpg_permute_sharded, whose kernel stores straight into them over
// NVLink/NVSwitch.  Allocation bases come from the driver (pointers handed
// out by caching allocators sit inside larger cudaMalloc segments).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "plan.h"

namespace {

typedef CUresult (*PfnGetAddressRange)(CUdeviceptr *, size_t *, CUdeviceptr);

std::mutex g_mu;
// A process maps each exported allocation once: buffers handed out by a
// caching allocator often share one cudaMalloc segment, so several imports
// can name the same handle.  Mappings are refcounted per handle.
struct Mapping {
    void *base;
    int refs;
};
std::map<std::string, Mapping> g_by_handle;          // handle bytes -> mapping
std::map<void *, std::pair<std::string, int>> g_imports;   // imported pointer -> (handle, count)

PfnGetAddressRange address_range_fn() {
    static PfnGetAddressRange fn = [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return (PfnGetAddressRange)f;
    }();
    return fn;
}

}  // namespace

namespace vpg {

vpg_status ipc_export(const void *ptr, void *handle, uint64_t *offset, std::string *err) {
    PfnGetAddressRange fn = address_range_fn();
    if (!fn) {
        *err = "cuMemGetAddressRange unavailable";
        return VPG_ECUDA;
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (fn(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS) {
        *err = "pointer is not a device allocation";
        return VPG_EINVAL;
    }
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, (void *)base);
    if (e != cudaSuccess) {
        *err = std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e);
        return VPG_ECUDA;
    }
    memcpy(handle, &h, sizeof(h));
    *offset = (uint64_t)((CUdeviceptr)ptr - base);
    return VPG_OK;
}

vpg_status ipc_import(const void *handle, uint64_t offset, void **ptr, std::string *err) {
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    const std::string key((const char *)&h, sizeof(h));
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_by_handle.find(key);
    void *base = nullptr;
    if (it != g_by_handle.end()) {
        base = it->second.base;
        ++it->second.refs;
    } else {
        cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            *err = std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e);
            return VPG_ECUDA;
        }
        g_by_handle[key] = Mapping{base, 1};
    }
    *ptr = (char *)base + offset;
    auto &imp = g_imports[*ptr];
    imp.first = key;
    ++imp.second;
    return VPG_OK;
}

vpg_status ipc_release(void *ptr, std::string *err) {
    void *base = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = g_imports.find(ptr);
        if (it == g_imports.end()) {
            *err = "pointer was not imported by vpg_ipc_import";
            return VPG_EINVAL;
        }
        const std::string key = it->second.first;
        if (--it->second.second == 0) g_imports.erase(it);
        auto m = g_by_handle.find(key);
        if (m == g_by_handle.end() || --m->second.refs > 0) return VPG_OK;
        base = m->second.base;
        g_by_handle.erase(m);
    }
    cudaError_t e = cudaIpcCloseMemHandle(base);
    if (e != cudaSuccess) {
        *err = std::string("cudaIpcCloseMemHandle: ") + cudaGetErrorString(e);
        return VPG_ECUDA;
    }
    return VPG_OK;
}

}  // namespace vpg
