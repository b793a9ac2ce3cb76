#!/usr/bin/env python
"""bench.py -- effective permutation bandwidth on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Metric: "permute effective GB/s (read+write bytes/s) and % of HBM peak at
1/2/4/8 B200" = algorithmic bytes (2 * N * elem) / kernel time.

Workload: cfg5 of BASELINE.json (rank-28 all-2 complex64, 2 GiB, seeded
random axes) -- the configuration the metric is quoted on at 1/2/4/8 GPUs.
At N=1 it is one kernel launch per step on one B200; at N>1 it is the
sharded permutation (local pack permute -> NCCL all-to-all -> local unpack
permute), total work fixed ("scaling": "strong").  The other BASELINE
configs (cfg1-cfg4) are timed in the same run with the same protocol and
reported under "configs".

Timing: W untimed warm-up steps; K timed steps, each preceded by an L2 flush
(write of a 2x-L2 buffer followed by a read of another 2x-L2 buffer, so the
timed kernel neither hits in L2 nor pays for write-backs of dirty flush
lines); CUDA events on the launching stream around the permutation only;
barrier + synchronize on both sides; max over ranks.  nvidia-smi-equivalent
clocks (NVML) are sampled during the timed region.

--impl reference: the reference's own CPU path (its emitted x86 AVX-512
kernel, oracle/_ref, built by oracle/build_ref.py) on the box's host cores,
all usable threads, each thread permuting the full workload (shared input,
private outputs); rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_CFG = "cfg5"


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------- clocks
NVML_REASONS = {
    0x1: "gpu_idle",
    0x2: "applications_clocks_setting",
    0x4: "sw_power_cap",
    0x8: "hw_slowdown",
    0x10: "sync_boost",
    0x20: "sw_thermal_slowdown",
    0x40: "hw_thermal_slowdown",
    0x80: "hw_power_brake_slowdown",
    0x100: "display_clock_setting",
}


class ClockSampler:
    """Samples SM clock and clock-event reasons every 20 ms via NVML."""

    def __init__(self, device_index=0):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._h = None
        try:
            import pynvml

            pynvml.nvmlInit()
            import torch

            uuid = str(torch.cuda.get_device_properties(device_index).uuid)
            uuid = uuid if uuid.startswith("GPU-") else "GPU-" + uuid
            try:
                self._h = pynvml.nvmlDeviceGetHandleByUUID(uuid)
            except Exception:
                self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._nv = pynvml
        except Exception as e:  # pragma: no cover - depends on the box
            self.error = str(e)

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in NVML_REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self._h is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._h is not None:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {
            "sm_mhz": statistics.median(self.samples),
            "sm_max_mhz": self.max_mhz,
            "reasons": sorted(self.reasons - {"gpu_idle"}),
            "samples": len(self.samples),
        }


# ---------------------------------------------------------------- device timing
class Flusher:
    """Evicts L2 between timed steps: write a 2xL2 buffer, then read another."""

    def __init__(self, torch, device):
        l2 = getattr(torch.cuda.get_device_properties(device), "L2_cache_size", 126 << 20)
        self.l2 = int(l2)
        nbytes = max(2 * self.l2, 256 << 20)
        self.w = torch.empty(nbytes // 4, dtype=torch.float32, device=device)
        self.r = torch.zeros(nbytes // 4, dtype=torch.float32, device=device)
        self.nbytes = nbytes

    def __call__(self):
        self.w.fill_(1.0)
        self.r.sum()


def time_device(torch, launch, steps, warmup, flush, stream):
    """Per-step CUDA-event times (ms) of `launch` on `stream`, L2 flushed."""
    for _ in range(warmup):
        flush()
        launch()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in evs:
        flush()
        a.record(stream)
        launch()
        b.record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def time_steady(torch, launch_i, nbuf, reps, stream):
    """Steady-state per-launch time (ms): `reps` rounds of back-to-back
    launches over `nbuf` rotating input/output pairs (together well over L2,
    so no launch finds its input cached), one CUDA event pair around all of
    them.  Consecutive kernels overlap launch and prologue (programmatic
    dependent launch); each still waits for its predecessor before its first
    global load."""
    for i in range(nbuf):
        launch_i(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        for i in range(nbuf):
            launch_i(i)
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / (reps * nbuf)


def steady_buffers(l2_bytes, nbytes, cap=8 << 30):
    """Rotating pairs so that the footprint is >= 3x L2 (at least 2 pairs)."""
    nb = max(2, -(-3 * l2_bytes // (2 * nbytes)))
    return int(max(2, min(nb, cap // (2 * nbytes))))


def event_floor_us(torch, flush, stream, reps=20):
    """Median event time of a trivial 1-element kernel after the same flush:
    the fixed event/launch overhead inside every flushed single-launch number
    (matters for the small configs, whose ideal times are 8-20 us)."""
    one = torch.zeros(1, dtype=torch.int32, device=flush.w.device)
    t = time_device(torch, lambda: one.fill_(1), reps, 3, flush, stream)
    return sorted(t)[len(t) // 2] * 1e3


def _traffic_from_profiles(cfg):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        e = d.get("kernels", {}).get(cfg)
        if e and e.get("dram_bytes") is not None:
            return int(e["dram_bytes"])
    except Exception:
        pass
    return None


# ---------------------------------------------------------------- reference CPU arm
def _mem_available():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 16 << 30


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference_cpu(cfg, steps, warmup, threads=None, x=None, private=None):
    """The reference's emitted CPU kernel, `threads` concurrent replicas.

    Each replica permutes its own copy of the input into its own output
    (`private`, the default when host memory allows): replicas that share
    one input in lockstep would serve each other's reads from the shared
    L3 and overstate the host's throughput.
    Returns (GB/s, per-step seconds list, threads, target, private)."""
    import numpy as np

    from oracle.refkernels import RefKernel
    from paper_2506_03686_b200.workloads import CONFIGS, make_input

    wl = CONFIGS[cfg]
    rk = RefKernel(cfg)
    ncpu = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    budget = int(_mem_available() * 0.5)
    if threads is None:
        threads = ncpu
    threads = max(1, min(threads, ncpu, 64))
    if private is None:
        private = 2 * threads * rk.nbytes <= budget
    cap_mem = max(1, budget // max(rk.nbytes, 1) // (2 if private else 1) - 1)
    threads = max(1, min(threads, cap_mem))
    if x is None:
        x = make_input(wl, threads=min(ncpu, 32))
    xb = x.reshape(-1).view(np.uint8)
    srcs = [rk.alloc() for _ in range(threads if private else 1)]
    for sb in srcs:
        sb.data[:] = xb
    src = srcs[0]
    outs = [rk.alloc() for _ in range(threads)]
    # parity of the baseline itself (cheap: numpy transpose comparison on a sample)
    rk.run_ptr(src.ptr, outs[0].ptr)
    want = np.ascontiguousarray(np.transpose(x, wl.axes)).reshape(-1).view(np.uint8)
    if not np.array_equal(outs[0].data, want):
        raise RuntimeError("reference kernel output differs from numpy transpose")
    del want
    barrier = threading.Barrier(threads + 1)
    stop = [False]

    def worker(i):
        while True:
            barrier.wait()
            if stop[0]:
                return
            rk.run_ptr(srcs[i % len(srcs)].ptr, outs[i].ptr)
            barrier.wait()

    ts = [threading.Thread(target=worker, args=(i,), daemon=True) for i in range(threads)]
    for t in ts:
        t.start()
    times = []
    for s in range(warmup + steps):
        t0 = time.perf_counter()
        barrier.wait()      # release
        barrier.wait()      # all done
        dt = time.perf_counter() - t0
        if s >= warmup:
            times.append(dt)
    stop[0] = True
    barrier.wait()
    for t in ts:
        t.join()
    gbs = threads * wl.algorithmic_bytes / (sum(times) / len(times)) / 1e9
    return gbs, times, threads, rk.target, private


def run_reference_cpu_1core(cfg, reps=3, x=None):
    """BASELINE.md §2 protocol: the reference's emitted kernel on ONE pinned
    core (the paper measures a single core; flags emit.py:433),
    best of `reps` full permutations.  The worker thread pins itself with
    sched_setaffinity (per-thread on Linux; the `taskset -c` equivalent).
    Returns (GB/s, best seconds, core id)."""
    import numpy as np

    from oracle.refkernels import RefKernel
    from paper_2506_03686_b200.workloads import CONFIGS, make_input

    wl = CONFIGS[cfg]
    rk = RefKernel(cfg)
    if x is None:
        x = make_input(wl, threads=16)
    src, dst = rk.alloc(), rk.alloc()
    src.data[:] = x.reshape(-1).view(np.uint8)
    cores = sorted(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else [0]
    core = cores[-1]
    res = {}

    def worker():
        if hasattr(os, "sched_setaffinity"):
            os.sched_setaffinity(0, {core})
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            rk.run_ptr(src.ptr, dst.ptr)
            ts.append(time.perf_counter() - t0)
        res["best"] = min(ts)

    t = threading.Thread(target=worker)
    t.start()
    t.join()
    want = np.ascontiguousarray(np.transpose(x, wl.axes)).reshape(-1).view(np.uint8)
    if not np.array_equal(dst.data, want):
        raise RuntimeError("reference kernel output differs from numpy transpose")
    return wl.algorithmic_bytes / res["best"] / 1e9, res["best"], core


def cpu_baseline_1core_only(cfg):
    """Sharded runs (N > 1): only the single-core line (bounded: 3 full
    permutations), run on rank 0 after every timed region."""
    try:
        g1, best, core = run_reference_cpu_1core(cfg)
        return {"value": round(g1, 3), "unit": "GB/s", "cores": 1, "kind": "reference",
                "sample": f"1 full {cfg} permutation, best of 3, worker pinned to core {core}; "
                          f"reference emitted kernel ({best * 1e3:.1f} ms); host {_cpu_model()}, "
                          f"nproc {os.cpu_count()}"}
    except Exception as e:
        return {"value": None, "unit": "GB/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}


def cpu_baseline_entry(cfg, cpu_threads=None):
    """cpu_baseline of the JSON line: the 1-core line of BASELINE.md §2
    (value, cores = 1) with the all-threads aggregate beside it."""
    try:
        g1, best, core = run_reference_cpu_1core(cfg)
        out = {"value": round(g1, 3), "unit": "GB/s", "cores": 1, "kind": "reference",
               "sample": f"1 full {cfg} permutation, best of 3, worker pinned to core {core} "
                         f"(sched_setaffinity); reference emitted kernel ({best * 1e3:.1f} ms); "
                         f"host {_cpu_model()}, nproc {os.cpu_count()}"}
    except Exception as e:  # reported, not fatal
        return {"value": None, "unit": "GB/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}
    try:
        gbs, times, threads, target, private = run_reference_cpu(cfg, 2, 1, threads=cpu_threads)
        out["all_threads"] = {"value": round(gbs, 2), "unit": "GB/s", "cores": threads,
                              "sample": f"{threads} concurrent full {cfg} permutations x 2 timed steps "
                                        f"(reference emitted {target} kernel, "
                                        f"{'private inputs' if private else 'shared input'})"}
    except Exception as e:
        out["all_threads"] = {"value": None, "sample": f"unavailable: {e}"}
    return out


def sample_parity(torch, x, y, shape, axes, nsamp=1 << 20, seed=0):
    """y[i] == x[f(i)] on random output offsets i (f per core.py:173-178)."""
    n = x.numel()
    g = torch.Generator(device=x.device).manual_seed(seed)
    idx = torch.randint(0, n, (nsamp,), device=x.device, generator=g, dtype=torch.int64)
    in_strides = [1] * len(shape)
    for k in range(len(shape) - 2, -1, -1):
        in_strides[k] = in_strides[k + 1] * shape[k + 1]
    rem = idx.clone()
    src = torch.zeros_like(idx)
    for a in reversed(axes):              # output dims, innermost first
        d = shape[a]
        src += (rem % d) * in_strides[a]
        rem //= d
    return bool(torch.equal(y[idx], x[src]))


def _numpy_baseline(cfg):
    """The paper's CPU comparator (SURVEY.md §8(d) secondary line): numpy
    transpose + contiguous copy of the full workload, one run, 1 thread."""
    import numpy as np

    from paper_2506_03686_b200.workloads import CONFIGS, make_input

    wl = CONFIGS[cfg]
    x = make_input(wl, threads=8)
    t0 = time.perf_counter()
    y = np.ascontiguousarray(np.transpose(x, wl.axes))
    dt = time.perf_counter() - t0
    del x, y
    return {"value": round(wl.algorithmic_bytes / dt / 1e9, 3), "unit": "GB/s", "cores": 1,
            "sample": f"np.ascontiguousarray(np.transpose(x, axes)) on the full {cfg} input, 1 run ({dt:.2f} s)"}


# ---------------------------------------------------------------- our arm
def bench_one_gpu(args, torch, cfg, with_e2e, peak):
    from paper_2506_03686_b200 import TensorLayout, build_program, execute, from_numpy_convention
    from paper_2506_03686_b200.api import execute_device
    from paper_2506_03686_b200.workloads import CONFIGS, make_input

    dev = torch.device("cuda", torch.cuda.current_device())
    wl = CONFIGS[cfg]
    lay, pm = TensorLayout.from_shape(wl.shape, wl.elem_bytes), from_numpy_convention(wl.axes)
    prog = build_program(lay, pm)
    nbytes = wl.numel * wl.elem_bytes
    host_in = None
    if with_e2e:
        x = make_input(wl, threads=16)
        host_in = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        host_in.numpy()[:] = x.reshape(-1).view("u1")
        xd = host_in.to(dev)
        del x
    else:
        xd = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        g = torch.Generator(device=dev).manual_seed(0)
        xd.view(torch.int32).copy_(torch.randint(-2**31, 2**31 - 1, (nbytes // 4,), device=dev,
                                                 dtype=torch.int32, generator=g))
    yd = torch.empty_like(xd)
    # --tune: measured planning (autotune, untimed) on the step's own
    # buffers -- the fastest of the cost model's best tile shapes on this
    # GPU.  Off by default: the model's choice is as fast on the BASELINE
    # configs, and a process that has timed many candidate kernels runs
    # the winner ~2% slower afterwards (run-to-run spread)
    if args.tune:
        from paper_2506_03686_b200 import autotune

        prog = autotune(lay, pm, src=xd, dst=yd)
    res = {"config": cfg, "kernel": prog.kernel,
           "tile": [prog.metadata["src_run"], prog.metadata["dst_run"]] if prog.kernel == "tile" else None,
           # the plan's layout choices (vpg_plan_describe lines)
           "plan": [ln for ln in prog.text.splitlines()
                    if ln.startswith(("vector elems", "smem chunk swizzle", "smem address swizzle", "smem pitch",
                                      "specialised", "rows"))]}
    stream = torch.cuda.current_stream(dev)
    flush = args._flusher
    launch = lambda: execute_device(prog, xd, out=yd, stream=stream)  # noqa: E731
    times = time_device(torch, launch, args.steps, args.warmup, flush, stream)
    # sampled parity (2^20 random output positions through the closed-form
    # bijection of core.py:173-178, in torch on device; tests/ hold the full
    # oracle checks -- torch.permute itself is limited to 25 dims)
    tdt = {"float32": torch.int32, "float64": torch.int64, "complex64": torch.int64}[wl.dtype]
    res["parity_sampled"] = sample_parity(torch, xd.view(tdt), yd.view(tdt), wl.shape, wl.axes)
    # same-run copy bandwidth of this box (torch copy_ of the same bytes, same
    # protocol): the achievable ceiling for any permutation of this size
    tc = time_device(torch, lambda: yd.copy_(xd), args.steps, args.warmup, flush, stream)
    res["copy_gbs"] = wl.algorithmic_bytes / (sum(tc) / len(tc) * 1e-3) / 1e9
    # the paper's comparator on the same GPU: torch's own permute+contiguous
    # copy (TensorIterator), same flush/event protocol
    if len(wl.shape) <= 25:
        xv = xd.view(tdt).reshape(wl.shape).permute(wl.axes)
        yv = yd.view(tdt).reshape(wl.out_shape)
        tt = time_device(torch, lambda: yv.copy_(xv), args.steps, args.warmup, flush, stream)
        res["torch_gbs"] = wl.algorithmic_bytes / (sum(tt) / len(tt) * 1e-3) / 1e9
    else:
        res["torch_gbs"] = None          # torch.permute supports at most 25 dims
    # steady state: back-to-back launches over rotating buffers (> 3x L2),
    # ours and torch copy_ of the same bytes; parity of the last outputs
    nb = steady_buffers(flush.l2, nbytes)
    xs = [xd] + [xd.clone() for _ in range(nb - 1)]
    ys = [yd] + [torch.empty_like(xd) for _ in range(nb - 1)]
    reps = max(3, min(50, int(4e9 // (nb * 2 * nbytes))))
    res["steady_ms"] = time_steady(torch, lambda i: execute_device(prog, xs[i], out=ys[i], stream=stream), nb,
                                   reps, stream)
    res["steady_parity"] = (sample_parity(torch, xd.view(tdt), ys[-1].view(tdt), wl.shape, wl.axes, nsamp=1 << 18)
                            and all(bool(torch.equal(ys[i], ys[-1])) for i in range(nb - 1)))
    res["steady_copy_ms"] = time_steady(torch, lambda i: ys[i].copy_(xs[i]), nb, reps, stream)
    res["steady_buffers"] = nb
    res["steady_launches"] = reps * nb
    del xs, ys
    ms = sum(times) / len(times)
    res["ms_per_launch"] = ms
    res["ms_best"] = min(times)
    res["gbs"] = wl.algorithmic_bytes / (ms * 1e-3) / 1e9
    res["frac_of_hbm"] = res["gbs"] / peak
    res["times_ms"] = times
    res["algorithmic_bytes"] = wl.algorithmic_bytes
    if with_e2e:
        launch()                          # yd held the copy/torch comparators' output
        host_out = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        # (1) one blocking call per step: latency of a single host permutation
        e2e_t = []
        for s in range(args.warmup + args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out, _ = execute(prog, host_in, out=host_out)
            t1 = time.perf_counter()
            if s >= args.warmup:
                e2e_t.append(t1 - t0)
        res["e2e_blocking_gbs"] = wl.algorithmic_bytes / (sum(e2e_t) / len(e2e_t)) / 1e9
        # (2) a stream of steps through the non-blocking API: every step still
        # copies its input in and its full result out, but step k+1's H2D
        # overlaps step k's D2H (PCIe is full duplex)
        host_outs = [host_out, torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)]
        for s in range(args.warmup):
            execute(prog, host_in, out=host_outs[s % 2], blocking=False)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for s in range(args.steps):
            execute(prog, host_in, out=host_outs[s % 2], blocking=False)
        torch.cuda.current_stream().synchronize()
        t1 = time.perf_counter()
        res["e2e_s"] = (t1 - t0) / args.steps
        res["e2e_gbs"] = wl.algorithmic_bytes / res["e2e_s"] / 1e9
        res["e2e_parity"] = bool(torch.equal(host_outs[(args.steps - 1) % 2], yd.cpu()))
        res["h2d_bytes"] = nbytes
        res["d2h_bytes"] = nbytes
    del xd, yd
    torch.cuda.empty_cache()
    return res


def _steady_entry(r, peak):
    b = r["algorithmic_bytes"]
    return {"us_per_launch": round(r["steady_ms"] * 1e3, 2), "gbs": round(b / (r["steady_ms"] * 1e-3) / 1e9, 1),
            "frac_of_hbm": round(b / (r["steady_ms"] * 1e-3) / 1e9 / peak, 4),
            "copy_gbs": round(b / (r["steady_copy_ms"] * 1e-3) / 1e9, 1),
            "buffers": r["steady_buffers"], "launches": r["steady_launches"], "parity": r["steady_parity"]}


# ---------------------------------------------------------------- sharded (N > 1)
NVLINK_GBS = 770.0   # fallback only: peer copy per direction per GPU (B200_PROFILING.md)


def torchrun_cmd(argv, n, port):
    """The command `bench.py --gpus N` re-executes itself with when it was not
    started under torchrun: one rank per GPU on this node, rendezvous on
    127.0.0.1 (the container hostname may not resolve)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + list(argv)


def _free_port():
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args, argv):
    """--gpus N > 1 without WORLD_SIZE: refuse loudly if this node has fewer
    than N GPUs (never print a 1-GPU line labelled N GPUs), else run N ranks
    under torch.distributed.run; rank 0 prints the one JSON line."""
    import subprocess

    if args.dist_backend == "nccl":
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs on this node, found {have}; "
                  f"refusing to report a {have}-GPU run as {args.gpus} GPUs", file=sys.stderr, flush=True)
            return 2
    cmd = torchrun_cmd(argv, args.gpus, _free_port())
    print("bench.py: launching " + " ".join(cmd), file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def measure_alltoall(torch, dist, dev, G, nbytes=256 << 20, iters=10, warm=3):
    """NCCL all_to_all_single on a 256 MiB per-rank buffer:
    device time of `iters` back-to-back collectives, max over ranks.
    Returns (algbw, busbw) in GB/s; busbw = algbw * (G-1)/G is the per-GPU
    NVLink traffic rate (the nccl-tests convention), the NVLink roofline
    denominator of the sharded line."""
    nbytes -= nbytes % G
    x = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
    for _ in range(warm):
        dist.all_to_all_single(y, x)
    torch.cuda.synchronize()
    dist.barrier()
    st = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(iters):
        dist.all_to_all_single(y, x)
    b.record(st)
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / iters], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    algbw = nbytes / (t.item() * 1e-3) / 1e9
    del x, y
    return algbw, algbw * (G - 1) / G


def bench_sharded(args, torch, base, config, peak, peak_kind):
    """cfg5 sharded over the torchrun ranks (strong scaling); device time max
    over ranks.  Per step either the fused exchange (one tile kernel per rank
    storing into the owning peers' output shards over NVLink, ShardExchange)
    or P1 permute -> NCCL all_to_all_single -> P2 permute; --shard-method
    auto picks the fused kernel when its destination runs are >= 128 B."""
    import numpy as np
    import torch.distributed as dist

    from paper_2506_03686_b200 import permute
    from paper_2506_03686_b200.sharded import (ShardExchange, fused_supported, permute_sharded,
                                               permute_sharded_pipelined, pipeline_chunks, plan_sharded,
                                               shard_bounds)
    from paper_2506_03686_b200.workloads import CONFIGS, make_input_slice

    # --sharded without torchrun: a one-rank process group on this node
    for k, v in (("MASTER_ADDR", "127.0.0.1"), ("RANK", "0"), ("WORLD_SIZE", "1"), ("LOCAL_RANK", "0")):
        os.environ.setdefault(k, v)
    os.environ.setdefault("MASTER_PORT", str(_free_port()))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    backend = args.dist_backend
    # gloo: code-path check only -- ranks may share a GPU, so its timings are
    # not multi-GPU results (the JSON line says so)
    dev_index = local_rank if backend == "nccl" else local_rank % torch.cuda.device_count()
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    # stdout carries the one JSON line: while the communicator comes up
    # (NCCL prints its version banner to stdout under NCCL_DEBUG=VERSION,
    # which the GPU boxes set) file descriptor 1 points at stderr
    sys.stdout.flush()
    saved_stdout = os.dup(1)
    os.dup2(2, 1)
    try:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
        G, r = dist.get_world_size(), dist.get_rank()
        red_dev = dev if backend == "nccl" else torch.device("cpu")
        warm = torch.zeros(1, device=red_dev)
        dist.all_reduce(warm)              # first collective: lazy communicator setup
        if backend == "nccl":
            torch.cuda.synchronize()
    finally:
        sys.stdout.flush()
        os.dup2(saved_stdout, 1)
        os.close(saved_stdout)
    a2a = None
    if backend == "nccl" and G > 1:
        a2a = measure_alltoall(torch, dist, dev, G)
    wl = CONFIGS[args.config]
    sp = plan_sharded(wl.shape, wl.axes, G)
    lo, hi = shard_bounds(wl.numel, G, r)
    host_in = torch.from_numpy(make_input_slice(wl, lo, hi).reshape(-1).view(np.uint8)).pin_memory()
    wdt = {4: torch.int32, 8: torch.int64}[wl.elem_bytes]     # opaque words of the element width
    x = host_in.to(dev).view(wdt)
    st = torch.cuda.current_stream()
    method = args.shard_method
    xmode = None
    if method == "auto":
        # the fused exchange where its remote runs are long enough, else the
        # chunk-pipelined all-to-all where the shard has a pipelining axis
        method = "fused" if fused_supported(wl.shape, wl.axes, wl.elem_bytes, G) else (
            "pipelined" if pipeline_chunks(sp) > 1 else "alltoall")
    if method in ("push", "pull"):
        method, xmode = "fused", method
    fused_fallback = None
    if method == "fused":
        # The fused exchange maps peer memory (CUDA IPC) and orders the ranks
        # with a device-side barrier.  Prove it on this box before timing it:
        # two calls, the second timed on the host, and a sampled parity check
        # of this rank's output shard.  If any rank fails (exception, a step
        # that ran into the barrier's bounded wait, wrong data), every rank
        # falls back to the NCCL all-to-all path and the JSON line says why.
        err, x_dev = None, x
        try:
            ex = ShardExchange(wl.shape, wl.axes, wdt, device=dev, mode=xmode or "auto")
            xmode = ex.mode
            if xmode == "pull":
                # the peers read this rank's input from the exchange's shared buffer
                ex.input.copy_(x)
                x = ex.input
            # (no collective inside this block: a rank that failed earlier
            # must not leave its peers waiting in one)
            ex(x)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            probe = ex(x)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            if os.environ.get("VPG_BENCH_FORCE_FUSED_FAIL"):
                err = "forced (VPG_BENCH_FORCE_FUSED_FAIL)"
            elif dt > 2.0:
                err = f"one exchange step took {dt:.1f} s (device-side barrier wait expired?)"
            elif not _sample_shard_parity(torch, host_in, probe, wl, sp, r, G, nsamp=1 << 14):
                err = "sampled parity mismatch"
            del probe
        except Exception as e:  # reported in the JSON line; the NCCL path takes over
            err = f"{type(e).__name__}: {e}"[:200]
        flag = torch.tensor([0 if err is None else 1], device=red_dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MAX)
        if flag.item():
            fused_fallback = err or "another rank failed"
            print(f"rank {r}: fused exchange ({xmode}) not used: {fused_fallback}", file=sys.stderr, flush=True)
            method, xmode, x, ex = ("pipelined" if pipeline_chunks(sp) > 1 else "alltoall"), None, x_dev, None
        else:
            run = ex
    if method == "fused":
        pass
    elif method == "pipelined":
        run = lambda xin: permute_sharded_pipelined(xin, wl.shape, wl.axes, local_permute=permute,  # noqa: E731
                                                    plan=sp)
    else:
        run = lambda xin: permute_sharded(xin, wl.shape, wl.axes, local_permute=permute, plan=sp)  # noqa: E731
    step = lambda: run(x)  # noqa: E731
    out = None
    for _ in range(args.warmup):
        out = step()          # same allocation pattern as the timed loop (two live outputs)
    torch.cuda.synchronize()
    dist.barrier()
    evs = []
    with ClockSampler(dev_index) as clk:
        for _ in range(args.steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            out = step()
            b.record(st)
            evs.append((a, b))
        torch.cuda.synchronize()
    dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    if os.environ.get("VPG_BENCH_DEBUG"):
        print(f"rank {r} step ms: {[round(v, 3) for v in step_ms]}", file=sys.stderr, flush=True)
    tot = torch.tensor([sum(step_ms)], device=red_dev, dtype=torch.float64)
    dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms = tot.item() / args.steps
    gbs = wl.algorithmic_bytes / (ms * 1e-3) / 1e9
    # parity on every rank: 2^18 sampled output positions of this rank's shard
    want_ok = _sample_shard_parity(torch, host_in, out, wl, sp, r, G)
    ok = torch.tensor([1 if want_ok else 0], device=red_dev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    # end to end: pinned host shard -> device -> sharded permute -> host
    # shard, as a stream of steps: the H2D of step k+1 (its own stream,
    # double-buffered) overlaps the D2H of step k; each step's permute
    # waits for its H2D and for the previous D2H (the exchange reuses its
    # output buffer).  Timed on the host around all steps, max over ranks.
    nb_out = out.numel() * out.element_size()
    host_outs = [torch.empty(nb_out, dtype=torch.uint8).pin_memory() for _ in range(2)]
    xins = [torch.empty_like(x) for _ in range(2)]
    s_h2d, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    consumed = [None, None]       # event: step using xins[i] has run
    d2h_done = None

    def e2e_step(k):
        nonlocal d2h_done
        i = k % 2
        with torch.cuda.stream(s_h2d):
            if consumed[i] is not None:
                s_h2d.wait_event(consumed[i])
            xins[i].view(torch.uint8).reshape(-1).copy_(host_in, non_blocking=True)
            h2d = torch.cuda.Event()
            h2d.record(s_h2d)
        st.wait_event(h2d)
        if d2h_done is not None:
            st.wait_event(d2h_done)
        y = run(xins[i])
        kd = torch.cuda.Event()
        kd.record(st)
        consumed[i] = kd
        with torch.cuda.stream(s_d2h):
            s_d2h.wait_event(kd)
            host_outs[i].copy_(y.reshape(-1).view(torch.uint8), non_blocking=True)
            d2h_done = torch.cuda.Event()
            d2h_done.record(s_d2h)

    for k in range(args.warmup):
        e2e_step(k)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for k in range(args.steps):
        e2e_step(args.warmup + k)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    e2e = [(t1 - t0) / args.steps]
    e2e_ok = bool(torch.equal(host_outs[(args.warmup + args.steps - 1) % 2],
                              out.reshape(-1).view(torch.uint8).cpu()))
    e2e_t = torch.tensor([sum(e2e) / len(e2e)], device=red_dev, dtype=torch.float64)
    dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    shard_bytes = wl.numel * wl.elem_bytes // G
    t_hbm = 2 * shard_bytes / (peak * 1e9)
    nvl_gbs = a2a[1] if a2a else NVLINK_GBS
    nvl_kind = ("measured all_to_all_single bus bandwidth, 256 MiB per rank, this run" if a2a else
                "fallback peer-copy figure (B200_PROFILING.md; no NCCL all-to-all measured at this N)")
    t_nvl = shard_bytes * (G - 1) / G / (nvl_gbs * 1e9)
    bound = "nvlink" if t_nvl > t_hbm else "hbm"
    roof_gbs = wl.algorithmic_bytes / max(t_hbm, t_nvl) / 1e9
    if r == 0:
        line = dict(base)
        line.update({
            "value": round(gbs, 2), "ms_per_step": ms, "config": config,
            "e2e": {"value": round(wl.algorithmic_bytes / e2e_t.item() / 1e9, 3), "unit": "GB/s",
                    "h2d_bytes_per_step": shard_bytes * G, "d2h_bytes_per_step": shard_bytes * G,
                    "api": ("paper_2506_03686_b200.sharded.ShardExchange" if method == "fused" else
                            "paper_2506_03686_b200.sharded.permute_sharded") +
                           " on pinned host shards, streamed (H2D of step k+1 overlaps D2H of step k)",
                    "parity": e2e_ok},
            "gpu_launches": (1 if method == "fused" or G == 1 else
                             pipeline_chunks(sp) + 1 if method == "pipelined" else 2) * args.steps,
            "shard_method": method if method != "fused" else f"fused ({xmode})",
            "fused_exchange_fallback": fused_fallback,
            "roofline": {"bound": bound, "achieved": round(gbs, 2), "peak": round(roof_gbs, 1),
                         "peak_kind": f"min over HBM ({peak_kind} {peak} GB/s per GPU) and NVLink "
                                      f"({nvl_gbs:.1f} GB/s per direction per GPU: {nvl_kind}) time bounds",
                         "nvlink_gbs": round(nvl_gbs, 1),
                         "frac_of_nvlink": round(gbs / (wl.algorithmic_bytes / t_nvl / 1e9), 4) if G > 1 else None,
                         "unit": "GB/s", "frac": round(gbs / roof_gbs, 4), "traffic": None,
                         "kernel": ("fused exchange tile kernel (peer stores over NVLink)" if xmode == "push" else
                                    "fused exchange tile kernel (peer reads over NVLink)") if method == "fused"
                         else ("tile (P1 per chunk, P2) + NCCL all_to_all_single per chunk, pipelined"
                               if method == "pipelined" else "tile (P1/P2) + NCCL all_to_all_single")},
            "parity_sampled": bool(ok.item()),
            "alltoall_256MiB": None if a2a is None else {"algbw_gbs": round(a2a[0], 1),
                                                          "busbw_gbs": round(a2a[1], 1)},
            "cpu_baseline": None if args.no_cpu else cpu_baseline_1core_only(args.config),
            "clocks": clk.summary(),
            "shard_plan": sp.describe()[:400],
            "dist_backend": backend if backend == "nccl" else
            "gloo (code-path check: ranks may share one GPU; not a multi-GPU timing)",
        })
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def _sample_shard_parity(torch, host_in, out, wl, sp, r, G, nsamp=1 << 18):
    """Rank-local check: sampled positions of this rank's output shard equal the
    closed-form bijection applied to the global input, using only the inputs
    this rank can regenerate (make_input_slice) -- no collective needed."""
    import numpy as np

    from paper_2506_03686_b200.sharded import shard_bounds
    from paper_2506_03686_b200.workloads import make_input_slice

    n = wl.numel
    lo, hi = shard_bounds(n, G, r)
    rng = np.random.default_rng(r)
    pos = rng.integers(lo, hi, size=nsamp)
    in_strides = [1] * len(wl.shape)
    for k in range(len(wl.shape) - 2, -1, -1):
        in_strides[k] = in_strides[k + 1] * wl.shape[k + 1]
    rem = pos.copy()
    src = np.zeros_like(pos)
    for a in reversed(wl.axes):
        d = wl.shape[a]
        src += (rem % d) * in_strides[a]
        rem //= d
    wnp = np.uint64 if wl.elem_bytes == 8 else np.uint32
    got = out.reshape(-1).cpu().numpy().view(wnp)[pos - lo]
    vals = np.empty(nsamp, dtype=wnp)
    # regenerate the needed global input words block by block
    blocks = np.unique(src // (1 << 22))
    for b in blocks:
        sel = (src // (1 << 22)) == b
        blk = make_input_slice(wl, int(b) << 22, min(n, (int(b) + 1) << 22)).view(wnp)
        vals[sel] = blk[src[sel] - (int(b) << 22)]
    return bool(np.array_equal(got, vals))


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CFG)
    ap.add_argument("--no-extra", action="store_true", help="skip cfg1-4 side measurements")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--tune", action="store_true", help="measured planning (autotune) before timing")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="N>1 process group; gloo only checks the code path (ranks may share a GPU)")
    ap.add_argument("--shard-method", default="auto",
                    choices=["auto", "fused", "push", "pull", "alltoall", "pipelined"],
                    help="N>1: fused exchange kernel (push: peer stores, pull: peer reads, fused: whichever "
                         "keeps long remote runs), P1 -> all-to-all -> P2, or that pipelined over chunks")
    ap.add_argument("--cpu-threads", type=int, default=None)
    ap.add_argument("--sharded", action="store_true",
                    help="use the sharded (torchrun/NCCL) code path even with one rank")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3   # contract: W >= 3

    if argv is None:
        argv = sys.argv[1:]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        return self_launch(args, argv)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1 and world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}; reporting n_gpus={world}", file=sys.stderr)
        args.gpus = world
    peak, peak_kind = _peaks()
    from paper_2506_03686_b200.workloads import CONFIGS

    wl = CONFIGS[args.config]
    base = {
        "metric": "permute effective GB/s (read+write bytes/s)",
        "unit": "GB/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "c64 words (u64)" if wl.dtype == "complex64" else wl.dtype,
        "data": "synthetic (seeded numpy PCG64, block-seeded; BASELINE.json cfg5 distribution)",
    }
    config = {
        "workload": f"{args.config}: {wl.title}",
        "shape": list(wl.shape),
        "axes": list(wl.axes),
        "elem_bytes": wl.elem_bytes,
        "algorithmic_bytes_per_step": wl.algorithmic_bytes,
        "parallelism": f"sharded{args.gpus}" if args.gpus > 1 else "single-gpu",
        "l2_flush": "write 2xL2 + read 2xL2 before every timed step (value); configs.*.steady: back-to-back "
                    "launches over rotating buffers totalling >= 3xL2, no flush (inputs larger than L2)",
        "planning": "autotune on the step's buffers: fastest of the cost model's best tile shapes (untimed)"
        if args.tune else "cost model (planner's first choice)",
    }

    if args.impl == "reference":
        if rank != 0:
            return 0
        gbs, times, threads, target, private = run_reference_cpu(args.config, args.steps, args.warmup,
                                                                 threads=args.cpu_threads)
        line = dict(base)
        line.update({
            "impl": "reference",
            "value": gbs,
            "ms_per_step": 1e3 * sum(times) / len(times),
            "config": config,
            "cpu_baseline": {
                "value": gbs, "unit": "GB/s", "cores": threads, "kind": "reference",
                "sample": f"{threads} concurrent full {args.config} permutations per step "
                          f"(reference emitted {target} kernel, "
                          f"{'private inputs and outputs' if private else 'shared input, private outputs'}); "
                          f"host {_cpu_model()}, {os.cpu_count()} logical CPUs",
            },
            "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        })
        print(json.dumps(line), flush=True)
        return 0

    import torch

    if world > 1 or args.sharded:
        return bench_sharded(args, torch, base, config, peak, peak_kind)

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    args._flusher = Flusher(torch, dev)
    with ClockSampler(0) as clk:
        main_res = bench_one_gpu(args, torch, args.config, True, peak)
    floor = event_floor_us(torch, args._flusher, torch.cuda.current_stream())
    extra = {}
    if not args.no_extra:
        for k in sorted(CONFIGS):
            if k == args.config:
                continue
            r = bench_one_gpu(args, torch, k, False, peak)
            extra[k] = {"gbs": round(r["gbs"], 1), "frac_of_hbm": round(r["frac_of_hbm"], 4),
                        "us_per_launch": round(r["ms_per_launch"] * 1e3, 2), "kernel": r["kernel"],
                        "tile_src_dst_run": r["tile"], "plan": r["plan"],
                        "parity_sampled": r["parity_sampled"],
                        "torch_permute_copy_gbs": None if r["torch_gbs"] is None else round(r["torch_gbs"], 1),
                        "same_run_copy_gbs": round(r["copy_gbs"], 1),
                        "frac_of_same_run_copy": round(r["gbs"] / r["copy_gbs"], 4),
                        "steady": _steady_entry(r, peak)}
    extra[args.config] = {"gbs": round(main_res["gbs"], 1), "frac_of_hbm": round(main_res["frac_of_hbm"], 4),
                          "us_per_launch": round(main_res["ms_per_launch"] * 1e3, 2),
                          "kernel": main_res["kernel"], "parity_sampled": main_res["parity_sampled"],
                          "tile_src_dst_run": main_res["tile"], "plan": main_res["plan"],
                          "torch_permute_copy_gbs": None if main_res["torch_gbs"] is None
                          else round(main_res["torch_gbs"], 1),
                          "same_run_copy_gbs": round(main_res["copy_gbs"], 1),
                          "frac_of_same_run_copy": round(main_res["gbs"] / main_res["copy_gbs"], 4),
                          "steady": _steady_entry(main_res, peak)}
    cpu = None
    if not args.no_cpu:
        cpu = cpu_baseline_entry(args.config, args.cpu_threads)
        cpu_numpy = _numpy_baseline(args.config)
    ms = main_res["ms_per_launch"]
    line = dict(base)
    line.update({
        "value": round(main_res["gbs"], 2),
        "ms_per_step": ms,
        "config": config,
        "e2e": {"value": round(main_res["e2e_gbs"], 3), "unit": "GB/s",
                "h2d_bytes_per_step": main_res["h2d_bytes"], "d2h_bytes_per_step": main_res["d2h_bytes"],
                "api": "paper_2506_03686_b200.execute(program, pinned CPU tensor, out=pinned, blocking=False) "
                       "per step -> vpg_permute_host_async; stream synchronised at the end",
                "blocking_value": round(main_res["e2e_blocking_gbs"], 3),
                "parity": main_res["e2e_parity"]},
        "gpu_launches": args.steps,
        "roofline": {"bound": "hbm", "achieved": round(main_res["gbs"], 2), "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": round(main_res["gbs"] / peak, 4),
                     "traffic": _traffic_from_profiles(args.config),
                     "kernel": f"{main_res['kernel']} ({args.config})"},
        "cpu_baseline": cpu,
        "cpu_numpy": None if args.no_cpu else cpu_numpy,
        "clocks": clk.summary(),
        "parity_sampled": main_res["parity_sampled"],
        "configs": extra,
        "event_floor_us": round(floor, 2),
        "l2_bytes": args._flusher.l2,
        "step_ms_stats": {"mean": round(ms, 5), "median": round(statistics.median(main_res["times_ms"]), 5),
                          "min": round(min(main_res["times_ms"]), 5), "max": round(max(main_res["times_ms"]), 5)},
    })
    print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
