// capi.cpp -- the extern "C" boundary of libvpgpu.so (declared in
// include/vpgpu.h).  Plain pointers and sizes only; no torch types.
#include <cuda_runtime.h>

#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "plan.h"

namespace vpg {
vpg_status permute_host_pipelined(const vpg_plan *p, const void *host_src, void *host_dst, void *dev_src,
                                  void *dev_dst, cudaStream_t user, bool async, std::string *err);
vpg_status permute_host_bounded(const vpg_plan *p, const void *host_src, void *host_dst, void *scratch,
                                size_t scratch_bytes, cudaStream_t user, std::string *err);
int host_pipeline_chunks(const vpg_plan *p);
void host_pipeline_forget(const vpg_plan *p);
}  // namespace vpg

namespace {
thread_local std::string t_err;

vpg_status fail(vpg_status s, const std::string &msg) {
    t_err = msg;
    return s;
}

std::mutex g_cache_mu;
std::map<std::vector<int64_t>, vpg_plan *> g_cache;  // never freed (process lifetime)
// [a, a+na) and [b, b+nb) intersect (out-of-place only: the kernels would race)
bool overlaps(const void *a, uint64_t na, const void *b, uint64_t nb) {
    const uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
    return na > 0 && nb > 0 && x < y + nb && y < x + na;
}
}  // namespace

extern "C" {

int vpg_version(void) { return VPG_ABI_VERSION; }

const char *vpg_last_error(void) { return t_err.c_str(); }

vpg_status vpg_merge_dimensions(int rank, const int64_t *dims, const int32_t *sigma, int *out_rank,
                                int64_t *out_dims, int32_t *out_sigma) {
    if (!dims || !sigma || !out_rank || !out_dims || !out_sigma)
        return fail(VPG_EINVAL, "null argument");
    std::vector<int64_t> sq_d;
    std::vector<int32_t> sq_s;
    std::string err;
    if (!vpg::squeeze_unit_dims(rank, dims, sigma, sq_d, sq_s, &err)) return fail(VPG_EINVAL, err);
    if (rank < 1 || rank > VPG_MAX_RANK) return fail(VPG_EINVAL, "rank out of range");
    std::vector<int> seen(rank, 0);
    for (int k = 0; k < rank; ++k) {
        if (dims[k] < 1) return fail(VPG_EINVAL, "dimension is not positive");
        if (sigma[k] < 0 || sigma[k] >= rank || seen[sigma[k]])
            return fail(VPG_EINVAL, "map is not a bijection");
        seen[sigma[k]] = 1;
    }
    *out_rank = vpg::merge_dims(rank, dims, sigma, out_dims, out_sigma);
    return VPG_OK;
}

vpg_status vpg_plan_create(int rank, const int64_t *dims, const int32_t *sigma, int elem_bytes,
                           unsigned flags, vpg_plan **out) {
    if (!dims || !sigma || !out) return fail(VPG_EINVAL, "null argument");
    std::string err;
    vpg_status s = vpg::make_plan(rank, dims, sigma, elem_bytes, flags, out, &err);
    if (s != VPG_OK) return fail(s, err);
    return VPG_OK;
}

vpg_status vpg_plan_create_sharded(int rank, const int64_t *dims, const int32_t *sigma, int elem_bytes,
                                   unsigned flags, int shards, int shard_index, vpg_plan **out) {
    if (!dims || !sigma || !out) return fail(VPG_EINVAL, "null argument");
    if (shards < 1) return fail(VPG_EINVAL, "shards must be >= 1");
    std::string err;
    vpg_status s = vpg::make_plan(rank, dims, sigma, elem_bytes, flags, out, &err, shards, shard_index);
    if (s != VPG_OK) return fail(s, err);
    return VPG_OK;
}

vpg_status vpg_permute_sharded(const vpg_plan *plan, const void *src_shard, void *const *dst_shards,
                               void *cuda_stream) {
    if (!plan || !dst_shards) return fail(VPG_EINVAL, "null argument");
    if (plan->shards < 1) return fail(VPG_EINVAL, "not a sharded plan (use vpg_permute)");
    if (plan->tile.pull) return fail(VPG_EINVAL, "pull exchange plan: use vpg_permute_sharded_pull");
    if (plan->n > 0 && !src_shard) return fail(VPG_EINVAL, "null buffer");
    const uint64_t sb = (uint64_t)(plan->n / plan->shards) * (uint64_t)plan->elem_bytes;
    for (int q = 0; q < plan->shards; ++q)
        if (overlaps(dst_shards[q], sb, src_shard, sb))
            return fail(VPG_EINVAL, "src and dst must not overlap (out-of-place only)");
    std::string err;
    vpg_status s = vpg::launch_plan(plan, src_shard, dst_shards, plan->shards, cuda_stream, &err);
    if (s != VPG_OK) return fail(s, err);
    return VPG_OK;
}

vpg_status vpg_permute_sharded_pull(const vpg_plan *plan, const void *const *src_shards, void *dst_shard,
                                    void *cuda_stream) {
    if (!plan || !src_shards) return fail(VPG_EINVAL, "null argument");
    if (plan->shards < 1 || !plan->tile.pull) return fail(VPG_EINVAL, "not a pull exchange plan (VPG_SHARD_PULL)");
    if (plan->n > 0 && !dst_shard) return fail(VPG_EINVAL, "null buffer");
    for (int q = 0; q < plan->shards; ++q) {
        if (plan->n > 0 && !src_shards[q]) return fail(VPG_EINVAL, "null buffer");
        const uint64_t sb = (uint64_t)(plan->n / plan->shards) * (uint64_t)plan->elem_bytes;
        if (overlaps(src_shards[q], sb, dst_shard, sb))
            return fail(VPG_EINVAL, "src and dst must not overlap (out-of-place only)");
    }
    std::string err;
    vpg_status s = vpg::launch_plan_pull(plan, src_shards, dst_shard, cuda_stream, &err);
    if (s != VPG_OK) return fail(s, err);
    return VPG_OK;
}

vpg_status vpg_permute_sharded_sync(const vpg_plan *plan, const void *const *src_shards, void *const *dst_shards,
                                    const vpg_shard_sync *sync, void *cuda_stream) {
    if (!plan || !src_shards || !dst_shards) return fail(VPG_EINVAL, "null argument");
    if (plan->shards < 1) return fail(VPG_EINVAL, "not a sharded plan (use vpg_permute)");
    const int G = plan->shards;
    if (sync && sync->epoch != 0) {
        if (!sync->done_counter) return fail(VPG_EINVAL, "sync: null done_counter");
        for (int q = 0; q < G; ++q)
            if (!sync->flags[q]) return fail(VPG_EINVAL, "sync: null flag block");
    }
    const uint64_t sb = (uint64_t)(plan->n / G) * (uint64_t)plan->elem_bytes;
    std::string err;
    vpg_status s;
    if (plan->tile.pull) {
        if (plan->n > 0 && !dst_shards[0]) return fail(VPG_EINVAL, "null buffer");
        for (int q = 0; q < G; ++q) {
            if (plan->n > 0 && !src_shards[q]) return fail(VPG_EINVAL, "null buffer");
            if (overlaps(src_shards[q], sb, dst_shards[0], sb))
                return fail(VPG_EINVAL, "src and dst must not overlap (out-of-place only)");
        }
        s = vpg::launch_plan_pull(plan, src_shards, dst_shards[0], cuda_stream, &err, sync);
    } else {
        if (plan->n > 0 && !src_shards[0]) return fail(VPG_EINVAL, "null buffer");
        for (int q = 0; q < G; ++q)
            if (overlaps(dst_shards[q], sb, src_shards[0], sb))
                return fail(VPG_EINVAL, "src and dst must not overlap (out-of-place only)");
        s = vpg::launch_plan(plan, src_shards[0], dst_shards, G, cuda_stream, &err, sync);
    }
    if (s != VPG_OK) return fail(s, err);
    return VPG_OK;
}

vpg_status vpg_permute_sharded_emulated(const vpg_plan *const *plans, int nplans, const void *const *src_shards,
                                        void *const *dst_shards, void *cuda_stream) {
    if (!plans || !src_shards || !dst_shards) return fail(VPG_EINVAL, "null argument");
    if (nplans < 2 || nplans > VPG_MAX_SHARDS) return fail(VPG_EINVAL, "nplans must be in 2..VPG_MAX_SHARDS");
    if (plans[0] && plans[0]->n == 0) return VPG_OK;
    std::string err;
    vpg_status s = vpg::launch_sharded_emulated(plans, nplans, src_shards, dst_shards, cuda_stream, &err);
    return s == VPG_OK ? s : fail(s, err);
}

vpg_status vpg_ipc_export(const void *dev_ptr, void *handle, uint64_t *offset) {
    if (!dev_ptr || !handle || !offset) return fail(VPG_EINVAL, "null argument");
    std::string err;
    vpg_status s = vpg::ipc_export(dev_ptr, handle, offset, &err);
    return s == VPG_OK ? s : fail(s, err);
}

vpg_status vpg_ipc_import(const void *handle, uint64_t offset, void **dev_ptr) {
    if (!handle || !dev_ptr) return fail(VPG_EINVAL, "null argument");
    std::string err;
    vpg_status s = vpg::ipc_import(handle, offset, dev_ptr, &err);
    return s == VPG_OK ? s : fail(s, err);
}

vpg_status vpg_ipc_release(void *dev_ptr) {
    if (!dev_ptr) return fail(VPG_EINVAL, "null argument");
    std::string err;
    vpg_status s = vpg::ipc_release(dev_ptr, &err);
    return s == VPG_OK ? s : fail(s, err);
}

vpg_status vpg_permute(const vpg_plan *plan, const void *src, void *dst, void *cuda_stream) {
    if (!plan) return fail(VPG_EINVAL, "null plan");
    if (plan->shards > 1) return fail(VPG_EINVAL, "sharded plan: use vpg_permute_sharded");
    if (plan->n > 0 && (!src || !dst)) return fail(VPG_EINVAL, "null buffer");
    const uint64_t nb = (uint64_t)plan->n * (uint64_t)plan->elem_bytes;
    if (overlaps(src, nb, dst, nb)) return fail(VPG_EINVAL, "src and dst must not overlap (out-of-place only)");
    std::string err;
    vpg_status s = vpg::launch_plan(plan, src, dst, cuda_stream, &err);
    if (s != VPG_OK) return fail(s, err);
    return VPG_OK;
}

vpg_status vpg_permute_host(const vpg_plan *plan, const void *host_src, void *host_dst, void *dev_src,
                            void *dev_dst, void *cuda_stream) {
    if (!plan || !host_src || !host_dst || !dev_src || !dev_dst) return fail(VPG_EINVAL, "null argument");
    if (plan->shards > 0) return fail(VPG_EINVAL, "sharded plans run through vpg_permute_sharded");
    {
        const uint64_t nb = (uint64_t)plan->n * (uint64_t)plan->elem_bytes;
        if (overlaps(host_src, nb, host_dst, nb))
            return fail(VPG_EINVAL, "host src and dst must not overlap (out-of-place only)");
    }
    if (plan->n == 0) return VPG_OK;
    std::string err;
    vpg_status s = vpg::permute_host_pipelined(plan, host_src, host_dst, dev_src, dev_dst, (cudaStream_t)cuda_stream,
                                               false, &err);
    return s == VPG_OK ? s : fail(s, err);
}

vpg_status vpg_permute_host_bounded(const vpg_plan *plan, const void *host_src, void *host_dst, void *dev_scratch,
                                    size_t scratch_bytes, void *cuda_stream) {
    if (!plan || !host_src || !host_dst || !dev_scratch) return fail(VPG_EINVAL, "null argument");
    if (plan->shards > 0) return fail(VPG_EINVAL, "sharded plans run through vpg_permute_sharded");
    {
        const uint64_t nb = (uint64_t)plan->n * (uint64_t)plan->elem_bytes;
        if (overlaps(host_src, nb, host_dst, nb))
            return fail(VPG_EINVAL, "host src and dst must not overlap (out-of-place only)");
    }
    if (plan->n == 0) return VPG_OK;
    std::string err;
    vpg_status s = vpg::permute_host_bounded(plan, host_src, host_dst, dev_scratch, scratch_bytes,
                                             (cudaStream_t)cuda_stream, &err);
    return s == VPG_OK ? s : fail(s, err);
}

vpg_status vpg_permute_host_async(const vpg_plan *plan, const void *host_src, void *host_dst, void *dev_src,
                                  void *dev_dst, void *cuda_stream) {
    if (!plan || !host_src || !host_dst || !dev_src || !dev_dst) return fail(VPG_EINVAL, "null argument");
    if (plan->shards > 0) return fail(VPG_EINVAL, "sharded plans run through vpg_permute_sharded");
    {
        const uint64_t nb = (uint64_t)plan->n * (uint64_t)plan->elem_bytes;
        if (overlaps(host_src, nb, host_dst, nb))
            return fail(VPG_EINVAL, "host src and dst must not overlap (out-of-place only)");
    }
    if (plan->n == 0) return VPG_OK;
    std::string err;
    vpg_status ps = vpg::permute_host_pipelined(plan, host_src, host_dst, dev_src, dev_dst,
                                                (cudaStream_t)cuda_stream, true, &err);
    if (ps != VPG_OK) return fail(ps, err);
    return VPG_OK;
}

vpg_status vpg_permute_nd(int rank, const int64_t *dims, const int32_t *sigma, int elem_bytes,
                          const void *src, void *dst, void *cuda_stream) {
    if (!dims || !sigma) return fail(VPG_EINVAL, "null argument");
    if (rank < 1) return fail(VPG_EINVAL, "rank out of range");
    std::vector<int64_t> key;
    key.reserve(2 * rank + 2);
    key.push_back(rank);
    key.push_back(elem_bytes);
    for (int k = 0; k < rank; ++k) key.push_back(dims[k]);
    for (int k = 0; k < rank; ++k) key.push_back(sigma[k]);
    vpg_plan *p = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        auto it = g_cache.find(key);
        if (it != g_cache.end()) p = it->second;
    }
    if (!p) {
        vpg_status s = vpg_plan_create(rank, dims, sigma, elem_bytes, 0, &p);
        if (s != VPG_OK) return s;
        std::lock_guard<std::mutex> lk(g_cache_mu);
        auto ins = g_cache.emplace(key, p);
        if (!ins.second) {
            vpg_plan_destroy(p);
            p = ins.first->second;
        }
    }
    return vpg_permute(p, src, dst, cuda_stream);
}

vpg_status vpg_plan_info_get(const vpg_plan *p, vpg_plan_info *info) {
    if (!p || !info) return fail(VPG_EINVAL, "null argument");
    memset(info, 0, sizeof(*info));
    info->kernel_class = p->kernel_class;
    info->elem_bytes = p->elem_bytes;
    info->rank = p->rank;
    for (int k = 0; k < p->rank; ++k) {
        info->dims[k] = p->dims[k];
        info->sigma[k] = p->sigma[k];
    }
    info->num_elements = p->n;
    info->threads = p->threads;
    info->grid_hint = p->grid_hint;
    info->predicted_efficiency = p->predicted_eff;
    info->host_chunks = vpg::host_pipeline_chunks(p);
    info->jit_state = vpg::jit_state(p);
    info->shards = p->shards;
    info->shard_index = p->shard_index;
    if (p->kernel_class == VPG_KERNEL_TILE) {
        info->tile_elems = p->tile.T;
        info->src_run = p->tile.Ls;
        info->dst_run = p->tile.Ld;
        info->num_tiles = p->tile.num_tiles;
        info->smem_pitch = (int32_t)p->tile.pitch;
        info->smem_bytes = (int32_t)p->tile.smem_bytes;
        info->vec_elems = 1;
    } else if (p->kernel_class == VPG_KERNEL_ROWS) {
        info->src_run = p->rows.row_len;
        info->dst_run = p->rows.row_len;
        info->vec_elems = (int32_t)p->rows.vec;
        info->num_tiles = p->rows.nrows;
    } else if (p->kernel_class == VPG_KERNEL_COPY) {
        info->src_run = info->dst_run = p->n;
        info->vec_elems = 16 / p->elem_bytes > 0 ? 16 / p->elem_bytes : 1;
    } else {
        info->src_run = info->dst_run = 1;
        info->vec_elems = 1;
    }
    return VPG_OK;
}

vpg_status vpg_plan_describe(const vpg_plan *p, char *buf, size_t len) {
    if (!p || !buf || len == 0) return fail(VPG_EINVAL, "null argument");
    size_t n = std::min(len - 1, p->text.size());
    memcpy(buf, p->text.data(), n);
    buf[n] = 0;
    return VPG_OK;
}

vpg_status vpg_plan_emit_source(const vpg_plan *p, char *buf, size_t len) {
    if (!p || !buf || len == 0) return fail(VPG_EINVAL, "null argument");
    if (p->kernel_class != VPG_KERNEL_TILE) return fail(VPG_EUNSUPPORTED, "only tile plans are specialised");
    const std::string src = vpg::jit_source(p);
    if (src.size() + 1 > len) return fail(VPG_EINVAL, "buffer too small: need " + std::to_string(src.size() + 1));
    memcpy(buf, src.c_str(), src.size() + 1);
    return VPG_OK;
}

vpg_status vpg_plan_tile_params(const vpg_plan *p, void *buf, size_t len, size_t *needed) {
    if (!p) return fail(VPG_EINVAL, "null argument");
    if (needed) *needed = sizeof(vpg::TileParams);
    if (p->kernel_class != VPG_KERNEL_TILE) return fail(VPG_EUNSUPPORTED, "not a tile plan");
    if (!buf || len < sizeof(vpg::TileParams)) return fail(VPG_EINVAL, "buffer too small");
    memcpy(buf, &p->tile, sizeof(vpg::TileParams));
    return VPG_OK;
}

vpg_status vpg_plan_jit_compile(const vpg_plan *p) {
    if (!p) return fail(VPG_EINVAL, "null argument");
    if (p->kernel_class != VPG_KERNEL_TILE) return fail(VPG_EUNSUPPORTED, "only tile plans are specialised");
    std::string log;
    if (!vpg::jit_compile_check(p, &log)) return fail(VPG_EUNSUPPORTED, "NVRTC: " + log);
    return VPG_OK;
}

void vpg_plan_destroy(vpg_plan *p) {
    if (!p) return;
    vpg::host_pipeline_forget(p);
    vpg::jit_forget(p);
    delete p;
}

}  // extern "C"
