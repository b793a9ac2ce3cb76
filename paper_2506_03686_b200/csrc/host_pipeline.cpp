// host_pipeline.cpp -- end-to-end permutation of HOST buffers (the
// reference's execute() takes a host buffer, vm.py:105-110).
//
// A permutation has no output that depends on only part of the input in
// general, but it does along dims that stay "outer" on both sides: fixing
// the coordinates of a set K of such dims selects an input sub-box and an
// output sub-box that map onto each other.  The host path cuts the tensor
// into C = prod_{k in K} d_k such chunks and pipelines them over three
// streams:
//     H2D (copy engine 0):  host input sub-box  -> dense device chunk
//     compute:              sub-permutation (one plan shared by all chunks)
//     D2H (copy engine 1):  dense device chunk  -> host output sub-box
// so the device->host traffic of chunk j overlaps the host->device traffic
// of chunk j+1 (PCIe is full duplex).  Each sub-box is moved as a few
// cudaMemcpy2DAsync calls (contiguous blocks x rows); K is chosen so blocks
// stay >= 256 KiB.  Small tensors (or no suitable K) use one H2D, one
// launch, one D2H.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "plan.h"

namespace {

using vpg::kMaxRank;

constexpr int64_t kMinPipelineBytes = 64ll << 20;   // below this: single shot
constexpr int64_t kMinBlockBytes = 256ll << 10;     // contiguous block per 2-D copy row
constexpr int kMaxChunks = 64;
constexpr int kMaxCopiesPerChunk = 256;

struct Copy2D {
    int64_t host_off, dev_off;   // bytes
    int64_t width, height, pitch;  // bytes, rows, host pitch (bytes)
};

// 2-D copies moving the sub-box of a dense tensor (dims inner-first,
// `fixed[k] >= 0` pins dim k at that coordinate) to/from a dense buffer
// holding only the varying dims.
bool region_copies(int r, const int64_t *dims, const int64_t *coord, int E, std::vector<Copy2D> &out,
                   int max_copies) {
    out.clear();
    int64_t stride[kMaxRank];
    stride[0] = 1;
    for (int k = 1; k < r; ++k) stride[k] = stride[k - 1] * dims[k - 1];
    int64_t base = 0;
    for (int k = 0; k < r; ++k)
        if (coord[k] >= 0) base += coord[k] * stride[k];
    int i = 0;
    int64_t B = 1;
    while (i < r && coord[i] < 0) B *= dims[i++];
    // row dim: next varying dim above the block
    int rowd = -1;
    for (int k = i; k < r; ++k)
        if (coord[k] < 0) {
            rowd = k;
            break;
        }
    std::vector<int> outer;
    if (rowd >= 0)
        for (int k = rowd + 1; k < r; ++k)
            if (coord[k] < 0) outer.push_back(k);
    int64_t ncopies = 1;
    for (int k : outer) ncopies *= dims[k];
    if (ncopies > max_copies) return false;
    const int64_t height = rowd >= 0 ? dims[rowd] : 1;
    const int64_t pitch = rowd >= 0 ? stride[rowd] * E : B * E;
    for (int64_t c = 0; c < ncopies; ++c) {
        int64_t rem = c, off = base;
        for (int k : outer) {
            off += (rem % dims[k]) * stride[k];
            rem /= dims[k];
        }
        out.push_back({off * E, c * height * B * E, B * E, height, pitch});
    }
    return true;
}

struct PipePlan {
    bool ok = false;
    std::vector<int64_t> dims;     // the dims the chunking works on (the plan's, or a refinement)
    std::vector<int32_t> sigma;
    std::vector<int> K;            // chunk dims (inner-first source numbering of `dims`)
    int64_t chunks = 1;
    int64_t chunk_elems = 0;
    vpg_plan *sub = nullptr;       // permutation of one chunk
};

std::mutex g_pipe_mu;
std::map<const vpg_plan *, PipePlan> g_pipe;   // keyed by parent plan (plans are immutable)

// min_chunks > 0 (bounded device scratch): at least that many chunks, up to
// kMaxBoundedChunks, whatever the tensor size.
constexpr int64_t kMaxBoundedChunks = 1 << 16;

PipePlan build_pipe_dims(int r, const int64_t *dims, const int32_t *sigma, int E, int64_t n,
                         int64_t min_chunks, bool relaxed) {
    PipePlan pp;
    struct PlanView {
        const int64_t *dims;
        const int32_t *sigma;
        int64_t n;
    } pv{dims, sigma, n}, *p = &pv;
    if (r > kMaxRank) return pp;
    int64_t max_chunks = min_chunks > 0 ? kMaxBoundedChunks : kMaxChunks;   // the cost model picks the count
    if (const char *e = getenv("VPG_HOST_CHUNKS"); e && min_chunks == 0)
        max_chunks = std::max(1, std::min(kMaxChunks, atoi(e)));
    if (min_chunks > max_chunks) return pp;
    if ((min_chunks == 0 && p->n * E < kMinPipelineBytes) || r < 2 || max_chunks < 2) return pp;
    int64_t in_stride[kMaxRank], out_stride[kMaxRank], odims[kMaxRank];
    in_stride[0] = 1;
    for (int k = 1; k < r; ++k) in_stride[k] = in_stride[k - 1] * p->dims[k - 1];
    int64_t acc = 1;
    int pos[kMaxRank];
    for (int j = 0; j < r; ++j) {
        out_stride[p->sigma[j]] = acc;
        pos[p->sigma[j]] = j;
        odims[j] = p->dims[p->sigma[j]];
        acc *= odims[j];
    }
    // bounded scratch: any block length that keeps copies reasonable
    const int64_t min_block = min_chunks > 0 ? (relaxed ? 512 : (16ll << 10)) : kMinBlockBytes;
    const int max_copies = min_chunks > 0 ? (relaxed ? (1 << 16) : 4096) : kMaxCopiesPerChunk;
    std::vector<int> cand;
    for (int k = 0; k < r; ++k)
        if (p->dims[k] >= 2 && std::min(in_stride[k], out_stride[k]) * E >= min_block) cand.push_back(k);
    std::sort(cand.begin(), cand.end(), [&](int a, int b) {
        return std::min(in_stride[a], out_stride[a]) > std::min(in_stride[b], out_stride[b]);
    });
    // Greedy over candidate dims; every accepted prefix is scored with a
    // model of the copy engines: both directions stream concurrently at
    // ~50 GB/s each (measured ~100 GB/s duplex on this pool's Gen5 x16),
    // the last chunk's D2H is exposed, and every cudaMemcpy2DAsync costs
    // ~8 us of setup.  The best-scoring prefix wins.
    const double bytes = (double)p->n * E;
    auto model = [&](int64_t C, int64_t copies) {
        return bytes / 50e9 + bytes / C / 57e9 + copies * 8e-6;
    };
    // Exhaustive search over subsets of the (at most 12 best) candidate dims.
    if (cand.size() > 12) cand.resize(12);
    std::vector<int> K, bestK;
    int64_t C = 1, bestC = 1;
    double best_t = min_chunks > 1 ? 1e300 : model(1, 2);
    const int nc = (int)cand.size();
    for (uint32_t mask = 1; mask < (1u << nc); ++mask) {
        std::vector<int> K2;
        int64_t C2 = 1;
        for (int b = 0; b < nc; ++b)
            if (mask & (1u << b)) {
                K2.push_back(cand[b]);
                C2 *= p->dims[cand[b]];
            }
        if (C2 > max_chunks || C2 < min_chunks) continue;
        int64_t ci[kMaxRank], co[kMaxRank];
        for (int q = 0; q < r; ++q) ci[q] = co[q] = -1;
        for (int q : K2) {
            ci[q] = 0;
            co[pos[q]] = 0;
        }
        std::vector<Copy2D> tin, tout;
        if (!region_copies(r, p->dims, ci, E, tin, max_copies)) continue;
        if (tin.empty() || tin[0].width < min_block) continue;
        if (!region_copies(r, odims, co, E, tout, max_copies)) continue;
        if (tout.empty() || tout[0].width < min_block) continue;
        double t = model(C2, C2 * (int64_t)(tin.size() + tout.size()));
        if (t < best_t - 1e-9) {
            best_t = t;
            bestK = K2;
            bestC = C2;
        }
    }
    K = bestK;
    C = bestC;
    if (C < 2) return pp;
    // sub-permutation: same dims with the K dims collapsed to 1
    int64_t sd[VPG_MAX_RANK];
    for (int k = 0; k < r; ++k) sd[k] = p->dims[k];
    for (int k : K) sd[k] = 1;
    std::string err;
    if (vpg::make_plan(r, sd, p->sigma, E, 0, &pp.sub, &err) != VPG_OK) return pp;
    pp.dims.assign(dims, dims + r);
    pp.sigma.assign(sigma, sigma + r);
    pp.K = K;
    pp.chunks = C;
    pp.chunk_elems = p->n / C;
    pp.ok = true;
    return pp;
}

PipePlan build_pipe(const vpg_plan *p, int64_t min_chunks = 0, bool relaxed = false) {
    return build_pipe_dims(p->rank, p->dims, p->sigma, p->elem_bytes, p->n, min_chunks, relaxed);
}

// Bounded scratch on a plan whose merged dims offer no dim outer on both
// sides (a 2-D transpose): split one dim into (inner, outer factor) pieces
// so the outer factor can be the chunk dim.  Largest dims first, smallest
// sufficient factor first.
PipePlan build_pipe_refined(const vpg_plan *p, int64_t min_chunks) {
    const int r = p->rank;
    if (r + 1 > VPG_MAX_RANK) return PipePlan{};
    std::vector<int> order(r);
    for (int k = 0; k < r; ++k) order[k] = k;
    std::sort(order.begin(), order.end(), [&](int a, int b) { return p->dims[a] > p->dims[b]; });
    for (int k : order) {
        const int64_t d = p->dims[k];
        for (int64_t f = 2; f <= std::min<int64_t>(d / 2, kMaxBoundedChunks); ++f) {
            if (d % f) continue;
            std::vector<int64_t> rd;
            std::vector<int32_t> rs;
            for (int q = 0; q < r; ++q) {
                if (q == k) {
                    rd.push_back(d / f);
                    rd.push_back(f);
                } else {
                    rd.push_back(p->dims[q]);
                }
            }
            for (int j = 0; j < r; ++j) {
                const int q = p->sigma[j];
                if (q == k) {
                    rs.push_back(k);
                    rs.push_back(k + 1);
                } else {
                    rs.push_back(q > k ? q + 1 : q);
                }
            }
            for (bool relaxed : {false, true}) {
                PipePlan pp = build_pipe_dims(r + 1, rd.data(), rs.data(), p->elem_bytes, p->n, min_chunks, relaxed);
                if (pp.ok) return pp;
                if (pp.sub) vpg_plan_destroy(pp.sub);
            }
        }
    }
    return PipePlan{};
}

struct DevStreams {
    cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
};
std::map<int, DevStreams> g_streams;

DevStreams streams_for_current(std::string *err) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_pipe_mu);
    auto it = g_streams.find(dev);
    if (it != g_streams.end()) return it->second;
    DevStreams s;
    if (cudaStreamCreateWithFlags(&s.h2d, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&s.comp, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&s.d2h, cudaStreamNonBlocking) != cudaSuccess) {
        *err = "stream creation failed";
        return DevStreams{};
    }
    g_streams[dev] = s;
    return s;
}

}  // namespace

namespace vpg {

// Scratch hazards across calls: a later call may reuse the same device
// scratch while an earlier call's chunk kernels / D2H copies are still in
// flight on the internal streams.  Per scratch pointer we remember the event
// after its last reader; the next writer waits on it.
std::map<const void *, cudaEvent_t> g_src_free;   // dev_src: last kernel reading it done
std::map<const void *, cudaEvent_t> g_dst_free;   // dev_dst: last D2H reading it done

// Host-output ranges of in-flight async calls: a later call whose host
// input overlaps one of them (chaining outputs into inputs) waits for that
// D2H.  Bounded ring; entries are events recorded after the call's D2H.
struct PendingOut {
    uintptr_t lo, hi;
    cudaEvent_t done;
};
std::vector<PendingOut> g_pending_out;

// One call enqueues at a time: the scratch hazard events above are read and
// re-recorded during the enqueue, so calls from several host threads that
// share scratch buffers must not interleave there (execution stays async).
std::mutex g_enqueue_mu;

void wait_host_input(const void *host_src, size_t nbytes, cudaStream_t waiter) {
    const uintptr_t lo = (uintptr_t)host_src, hi = lo + nbytes;
    std::lock_guard<std::mutex> lk(g_pipe_mu);
    for (const PendingOut &po : g_pending_out)
        if (lo < po.hi && po.lo < hi) cudaStreamWaitEvent(waiter, po.done, 0);
}

void remember_host_output(const void *host_dst, size_t nbytes, cudaStream_t d2h) {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaEventRecord(e, d2h);
    std::lock_guard<std::mutex> lk(g_pipe_mu);
    if (g_pending_out.size() >= 16) {
        cudaEventDestroy(g_pending_out.front().done);
        g_pending_out.erase(g_pending_out.begin());
    }
    g_pending_out.push_back({(uintptr_t)host_dst, (uintptr_t)host_dst + nbytes, e});
}

void wait_and_replace(std::map<const void *, cudaEvent_t> &m, const void *ptr, cudaStream_t waiter,
                      cudaEvent_t *slot_out) {
    std::lock_guard<std::mutex> lk(g_pipe_mu);
    auto it = m.find(ptr);
    if (it != m.end()) {
        cudaStreamWaitEvent(waiter, it->second, 0);
        *slot_out = it->second;
    } else {
        cudaEvent_t e;
        cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        m[ptr] = e;
        *slot_out = e;
    }
}

// Pipelined host->device->host permutation.  `async`: return after
// enqueueing (completion ordered on `user`), else synchronise `user`.
// Tensors without a chunked plan run as one H2D -> kernel -> D2H chunk on
// the same streams, so scratch reuse is ordered the same way.
vpg_status permute_host_pipelined(const vpg_plan *p, const void *host_src, void *host_dst, void *dev_src,
                                  void *dev_dst, cudaStream_t user, bool async, std::string *err) {
    PipePlan pp;
    bool found = false;
    {
        std::lock_guard<std::mutex> lk(g_pipe_mu);
        auto it = g_pipe.find(p);
        if (it != g_pipe.end()) {
            pp = it->second;
            found = true;
        }
    }
    if (!found) {
        PipePlan built = build_pipe(p);
        bool dup = false;
        {
            std::lock_guard<std::mutex> lk(g_pipe_mu);
            auto ins = g_pipe.emplace(p, built);
            dup = !ins.second;
            pp = ins.first->second;
        }
        if (dup && built.sub) vpg_plan_destroy(built.sub);   // lost the race; outside the lock
    }
    DevStreams s = streams_for_current(err);
    if (!s.h2d) return VPG_ECUDA;
    const int r = p->rank, E = p->elem_bytes;
    // single-chunk form (async calls of unchunkable tensors still overlap
    // with neighbouring calls through the three streams)
    const int64_t chunks = pp.ok ? pp.chunks : 1;
    const vpg_plan *kp = pp.ok ? pp.sub : p;
    const int64_t cbytes = (pp.ok ? pp.chunk_elems : p->n) * E;
    int64_t odims[kMaxRank];
    int pos[kMaxRank];
    for (int j = 0; j < r; ++j) {
        odims[j] = p->dims[p->sigma[j]];
        pos[p->sigma[j]] = j;
    }
    std::unique_lock<std::mutex> enqueue_lock(g_enqueue_mu);
    cudaEvent_t start, fin, src_free, dst_free;
    std::vector<cudaEvent_t> done_in(chunks), done_k(chunks);
    cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&fin, cudaEventDisableTiming);
    for (int64_t j = 0; j < chunks; ++j) {
        cudaEventCreateWithFlags(&done_in[j], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&done_k[j], cudaEventDisableTiming);
    }
    if (async) {
        // no dependency on the user stream's earlier work (that would chain
        // call k+1's H2D behind call k's D2H); only real hazards are ordered
        wait_host_input(host_src, (size_t)p->n * E, s.h2d);
    } else {
        cudaEventRecord(start, user);
        cudaStreamWaitEvent(s.h2d, start, 0);
        cudaStreamWaitEvent(s.comp, start, 0);
        cudaStreamWaitEvent(s.d2h, start, 0);
    }
    wait_and_replace(g_src_free, dev_src, s.h2d, &src_free);   // earlier kernels done reading dev_src
    wait_and_replace(g_dst_free, dev_dst, s.comp, &dst_free);  // earlier D2H done reading dev_dst
    std::vector<Copy2D> cps;
    vpg_status st = VPG_OK;
    for (int64_t j = 0; j < chunks && st == VPG_OK; ++j) {
        char *din = (char *)dev_src + j * cbytes;
        char *dout = (char *)dev_dst + j * cbytes;
        int64_t ci[kMaxRank], co[kMaxRank];
        for (int q = 0; q < r; ++q) ci[q] = co[q] = -1;
        if (pp.ok) {
            int64_t rem = j;
            for (int q : pp.K) {
                ci[q] = rem % p->dims[q];
                co[pos[q]] = ci[q];
                rem /= p->dims[q];
            }
            region_copies(r, p->dims, ci, E, cps, 1 << 30);
        } else {
            cps.assign(1, Copy2D{0, 0, cbytes, 1, cbytes});
        }
        for (const Copy2D &c : cps)
            if (cudaMemcpy2DAsync(din + c.dev_off, c.width, (const char *)host_src + c.host_off, c.pitch, c.width,
                                  c.height, cudaMemcpyHostToDevice, s.h2d) != cudaSuccess) {
                *err = "H2D copy failed";
                st = VPG_ECUDA;
            }
        cudaEventRecord(done_in[j], s.h2d);
        cudaStreamWaitEvent(s.comp, done_in[j], 0);
        vpg_status ks = launch_plan(kp, din, dout, s.comp, err);
        if (ks != VPG_OK) st = ks;
        cudaEventRecord(done_k[j], s.comp);
        cudaStreamWaitEvent(s.d2h, done_k[j], 0);
        if (pp.ok) region_copies(r, odims, co, E, cps, 1 << 30);
        for (const Copy2D &c : cps)
            if (cudaMemcpy2DAsync((char *)host_dst + c.host_off, c.pitch, dout + c.dev_off, c.width, c.width,
                                  c.height, cudaMemcpyDeviceToHost, s.d2h) != cudaSuccess) {
                *err = "D2H copy failed";
                st = VPG_ECUDA;
            }
    }
    cudaEventRecord(src_free, s.comp);   // all kernels of this call done reading dev_src
    cudaEventRecord(fin, s.d2h);
    cudaEventRecord(dst_free, s.d2h);    // all D2H of this call done reading dev_dst
    if (async) remember_host_output(host_dst, (size_t)p->n * E, s.d2h);
    cudaStreamWaitEvent(user, fin, 0);
    enqueue_lock.unlock();
    if (!async) {
        cudaError_t e = cudaStreamSynchronize(user);
        if (e != cudaSuccess && st == VPG_OK) {
            *err = std::string("stream sync: ") + cudaGetErrorString(e);
            st = VPG_ECUDA;
        }
    }
    // destroying recorded events is safe: resources are released once complete
    cudaEventDestroy(start);
    cudaEventDestroy(fin);
    for (int64_t j = 0; j < chunks; ++j) {
        cudaEventDestroy(done_in[j]);
        cudaEventDestroy(done_k[j]);
    }
    return st;
}

// Host buffers larger than the device can stage: the tensor is cut into
// chunks (dims outer on both sides, as above) and streamed through a ring of
// R = scratch / (2 x chunk) slots of caller-provided device scratch -- H2D
// of chunk j into slot j % R, its sub-permutation, its D2H -- so the device
// holds at most R chunks at once.  Synchronous.
vpg_status permute_host_bounded(const vpg_plan *p, const void *host_src, void *host_dst, void *scratch,
                                size_t scratch_bytes, cudaStream_t user, std::string *err) {
    const int E = p->elem_bytes;
    const int64_t total = p->n * E;
    // at least four slots in flight: chunks of at most an eighth of the scratch
    const int64_t min_chunks = std::max<int64_t>(2, (8 * total + (int64_t)scratch_bytes - 1) / (int64_t)scratch_bytes);
    PipePlan pp = build_pipe(p, min_chunks);
    if (!pp.ok) {                                        // finer copies before giving up
        if (pp.sub) vpg_plan_destroy(pp.sub);
        pp = build_pipe(p, min_chunks, true);
    }
    if (!pp.ok) {                                        // split a dim to get a chunk dim
        if (pp.sub) vpg_plan_destroy(pp.sub);
        pp = build_pipe_refined(p, min_chunks);
    }
    if (!pp.ok) {
        if (pp.sub) vpg_plan_destroy(pp.sub);
        *err = "cannot cut this permutation into chunks that fit " + std::to_string(scratch_bytes) +
               " bytes of device scratch";
        return VPG_EUNSUPPORTED;
    }
    struct SubGuard {
        vpg_plan *s;
        ~SubGuard() { if (s) vpg_plan_destroy(s); }
    } guard{pp.sub};
    DevStreams s = streams_for_current(err);
    if (!s.h2d) return VPG_ECUDA;
    const int64_t cbytes = pp.chunk_elems * E;
    const int64_t R = std::max<int64_t>(1, (int64_t)scratch_bytes / (2 * cbytes));
    const int r = (int)pp.dims.size();
    const int64_t *dims = pp.dims.data();
    int64_t odims[VPG_MAX_RANK];
    int pos[VPG_MAX_RANK];
    for (int j = 0; j < r; ++j) {
        odims[j] = dims[pp.sigma[j]];
        pos[pp.sigma[j]] = j;
    }
    std::unique_lock<std::mutex> enqueue_lock(g_enqueue_mu);
    cudaEvent_t start, fin;
    cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&fin, cudaEventDisableTiming);
    std::vector<cudaEvent_t> slot_free((size_t)R), done_in((size_t)R), done_k((size_t)R);
    for (int64_t i = 0; i < R; ++i) {
        cudaEventCreateWithFlags(&slot_free[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&done_in[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&done_k[i], cudaEventDisableTiming);
    }
    cudaEventRecord(start, user);
    cudaStreamWaitEvent(s.h2d, start, 0);
    cudaStreamWaitEvent(s.comp, start, 0);
    cudaStreamWaitEvent(s.d2h, start, 0);
    std::vector<Copy2D> cps;
    vpg_status st = VPG_OK;
    for (int64_t j = 0; j < pp.chunks && st == VPG_OK; ++j) {
        const int64_t slot = j % R;
        char *din = (char *)scratch + slot * 2 * cbytes;
        char *dout = din + cbytes;
        if (j >= R) cudaStreamWaitEvent(s.h2d, slot_free[slot], 0);   // chunk j - R has left the slot
        int64_t ci[VPG_MAX_RANK], co[VPG_MAX_RANK];
        for (int q = 0; q < r; ++q) ci[q] = co[q] = -1;
        int64_t rem = j;
        for (int q : pp.K) {
            ci[q] = rem % dims[q];
            co[pos[q]] = ci[q];
            rem /= dims[q];
        }
        region_copies(r, dims, ci, E, cps, 1 << 30);
        for (const Copy2D &c : cps)
            if (cudaMemcpy2DAsync(din + c.dev_off, c.width, (const char *)host_src + c.host_off, c.pitch, c.width,
                                  c.height, cudaMemcpyHostToDevice, s.h2d) != cudaSuccess) {
                *err = "H2D copy failed";
                st = VPG_ECUDA;
            }
        cudaEventRecord(done_in[slot], s.h2d);
        cudaStreamWaitEvent(s.comp, done_in[slot], 0);
        vpg_status ks = launch_plan(pp.sub, din, dout, s.comp, err);
        if (ks != VPG_OK) st = ks;
        cudaEventRecord(done_k[slot], s.comp);
        cudaStreamWaitEvent(s.d2h, done_k[slot], 0);
        region_copies(r, odims, co, E, cps, 1 << 30);
        for (const Copy2D &c : cps)
            if (cudaMemcpy2DAsync((char *)host_dst + c.host_off, c.pitch, dout + c.dev_off, c.width, c.width,
                                  c.height, cudaMemcpyDeviceToHost, s.d2h) != cudaSuccess) {
                *err = "D2H copy failed";
                st = VPG_ECUDA;
            }
        cudaEventRecord(slot_free[slot], s.d2h);
    }
    cudaEventRecord(fin, s.d2h);
    cudaStreamWaitEvent(user, fin, 0);
    enqueue_lock.unlock();
    cudaError_t e = cudaStreamSynchronize(user);
    if (e != cudaSuccess && st == VPG_OK) {
        *err = std::string("stream sync: ") + cudaGetErrorString(e);
        st = VPG_ECUDA;
    }
    cudaEventDestroy(start);
    cudaEventDestroy(fin);
    for (int64_t i = 0; i < R; ++i) {
        cudaEventDestroy(slot_free[i]);
        cudaEventDestroy(done_in[i]);
        cudaEventDestroy(done_k[i]);
    }
    return st;
}

// number of pipeline chunks the host path would use (0 = single shot)
int host_pipeline_chunks(const vpg_plan *p) {
    PipePlan pp = build_pipe(p);
    int c = pp.ok ? (int)pp.chunks : 0;
    if (pp.sub) vpg_plan_destroy(pp.sub);
    return c;
}

void host_pipeline_forget(const vpg_plan *p) {
    vpg_plan *sub = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_pipe_mu);
        auto it = g_pipe.find(p);
        if (it == g_pipe.end()) return;
        sub = it->second.sub;
        g_pipe.erase(it);
    }
    if (sub) vpg_plan_destroy(sub);   // its own forget takes the lock again
}

}  // namespace vpg
