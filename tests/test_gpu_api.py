"""GPU tests of the public API surface: guard bands, misaligned buffers,
streams, host-buffer execute(), dtypes, degenerate shapes, error mapping."""

from __future__ import annotations

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

SHAPES = [
    ((64, 48), (1, 0)),                       # 2-D transpose (vectorised tile)
    ((8, 24, 20, 12), (0, 2, 3, 1)),          # NCHW->NHWC
    ((7, 9, 13, 5, 11), (4, 1, 0, 3, 2)),     # misaligned dims
    ((6, 5, 7, 3), (1, 0, 2, 3)),             # merged preserved row
    ((16, 8, 64), (1, 0, 2)),                 # stride-1 preserved
    ((8, 4, 256), (1, 0, 2)),                 # stride-1 preserved, 1 KiB rows (rows kernel)
    ((6, 4, 2000), (0, 1, 2)),                # identity (copy kernel)
    ((2,) * 12, tuple(np.random.default_rng(3).permutation(12).tolist())),
]


def prog_kind(shape, axes):
    from paper_2506_03686_b200 import TensorLayout, build_program, from_numpy_convention

    return build_program(TensorLayout.from_shape(shape, 4), from_numpy_convention(axes)).kernel


def _want(x_np, axes):
    return np.ascontiguousarray(np.transpose(x_np, axes))


@pytest.mark.parametrize("shape,axes", SHAPES)
@pytest.mark.parametrize("dtype", ["int32", "int64", "int16", "uint8", "complex128"])
def test_permute_matches_numpy(cuda, shape, axes, dtype):
    import torch

    from paper_2506_03686_b200 import permute

    rng = np.random.default_rng(0)
    if dtype == "complex128":
        x = (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(np.complex128)
    else:
        x = rng.integers(np.iinfo(dtype).min, np.iinfo(dtype).max, size=shape, dtype=dtype)
    y = permute(torch.from_numpy(x).to(cuda), axes)
    assert np.array_equal(y.cpu().numpy(), _want(x, axes))


@pytest.mark.parametrize("shape,axes", SHAPES)
@pytest.mark.parametrize("offset", [1, 2, 3])
def test_misaligned_base_pointers(cuda, shape, axes, offset):
    """Buffers at element (not 16-byte) alignment take the scalar-read variant."""
    import torch

    from paper_2506_03686_b200 import TensorLayout, build_program, from_numpy_convention
    from paper_2506_03686_b200.api import execute_device

    n = int(np.prod(shape))
    rng = np.random.default_rng(offset)
    base = rng.integers(0, 2**31, size=n + 8, dtype=np.int64).astype(np.int32)
    xd = torch.from_numpy(base).to(cuda)
    x = xd[offset:offset + n]
    out_full = torch.zeros(n + 8, dtype=torch.int32, device=cuda)
    out = out_full[offset:offset + n]
    prog = build_program(TensorLayout.from_shape(shape, 4), from_numpy_convention(axes),
                         force=None if prog_kind(shape, axes) in ("rows", "copy") else "tile")
    execute_device(prog, x, out=out)
    want = _want(base[offset:offset + n].reshape(shape), axes).reshape(-1)
    assert np.array_equal(out.cpu().numpy(), want)
    # guard band around the destination untouched
    full = out_full.cpu().numpy()
    assert not full[:offset].any() and not full[offset + n:].any()


def test_guard_bands_and_sentinels(cuda):
    """Destination guard bands filled with sentinels stay intact (the VM's
    guard-band method, vm.py:28-33/220-224), for every kernel class."""
    import torch

    from paper_2506_03686_b200 import TensorLayout, build_program, from_numpy_convention
    from paper_2506_03686_b200.api import execute_device

    G = 4096
    rng = np.random.default_rng(11)
    for shape, axes in SHAPES + [((3, 5, 1024), (1, 0, 2)), ((1000,), (0,))]:
        for force in (None, "tile", "gather"):
            n = int(np.prod(shape))
            x = rng.integers(0, 2**63, size=n, dtype=np.int64)
            buf = torch.full((n + 2 * G,), -0x5A5A5A5A5A5A5A5B, dtype=torch.int64, device=cuda)
            prog = build_program(TensorLayout.from_shape(shape, 8), from_numpy_convention(axes), force=force)
            execute_device(prog, torch.from_numpy(x).to(cuda), out=buf[G:G + n])
            h = buf.cpu().numpy()
            assert (h[:G] == -0x5A5A5A5A5A5A5A5B).all() and (h[G + n:] == -0x5A5A5A5A5A5A5A5B).all()
            assert np.array_equal(h[G:G + n], _want(x.reshape(shape), axes).reshape(-1)), (shape, force)


def test_nondefault_stream(cuda):
    import torch

    from paper_2506_03686_b200 import permute

    s = torch.cuda.Stream()
    x = torch.randint(0, 1 << 30, (512, 768), dtype=torch.int32, device=cuda)
    with torch.cuda.stream(s):
        y = permute(x, (1, 0), stream=s)
    s.synchronize()
    assert torch.equal(y, x.t().contiguous())


def test_execute_host_buffers(cuda):
    """execute() on host numpy/bytes/pinned tensors mirrors vm.execute's
    (output, counters) contract (vm.py:105-110) through the GPU."""
    import torch

    from paper_2506_03686_b200 import PermutationMap, TensorLayout, build_program, execute

    lay = TensorLayout((3, 32, 32, 7))                 # README "library in five lines"
    pm = PermutationMap((2, 0, 1, 3))
    prog = build_program(lay, pm)
    data = np.arange(lay.num_elements, dtype=np.uint32)
    out, counters = execute(prog, data)
    assert out.dtype == np.dtype("<u4")
    assert np.array_equal(out, oracle.naive_permute_np(data, lay.dims, pm.sigma))
    assert counters["launches"] == 1 and counters["bytes_read"] == data.nbytes
    out2, _ = execute(prog, data.tobytes())
    assert np.array_equal(out2, out)
    pinned = torch.from_numpy(data.view(np.int32)).pin_memory()
    out3, _ = execute(prog, pinned)
    assert np.array_equal(out3.numpy().reshape(-1).view(np.uint32), out)


def test_degenerate_shapes(cuda):
    import torch

    from paper_2506_03686_b200 import permute

    x = torch.arange(7, dtype=torch.int32, device=cuda)
    assert torch.equal(permute(x, (0,)), x)
    s = torch.tensor(5, dtype=torch.int32, device=cuda)
    assert permute(s, ()).item() == 5
    e = torch.empty((0, 3), dtype=torch.float32, device=cuda)
    assert tuple(permute(e, (1, 0)).shape) == (3, 0)
    one = torch.ones((1, 1), dtype=torch.float64, device=cuda)
    assert torch.equal(permute(one, (1, 0)), one)


def test_errors_are_loud(cuda):
    import torch

    from paper_2506_03686_b200 import LayoutError, TensorLayout, PermutationMap, build_program, permute
    from paper_2506_03686_b200.api import execute_device

    x = torch.zeros((4, 5), dtype=torch.int32, device=cuda)
    with pytest.raises(LayoutError):
        permute(x, (0, 0))
    with pytest.raises(LayoutError):
        permute(x, (0,))
    with pytest.raises(LayoutError):
        permute(x.cpu(), (1, 0))                       # no CPU fallback
    prog = build_program(TensorLayout((5, 4)), PermutationMap((1, 0)))
    with pytest.raises(LayoutError):
        execute_device(prog, x, out=x)                 # in-place refused (out-of-place only)
    with pytest.raises(LayoutError):
        execute_device(prog, torch.zeros(21, dtype=torch.int32, device=cuda))


@pytest.mark.parametrize("G", [2, 4, 8])
def test_sharded_algorithm_on_one_gpu_cfg5(cuda, G):
    """The sharded P1 -> all-to-all -> P2 programs for cfg5 at G ranks, run
    rank after rank on one GPU, reproduce the single-GPU permutation."""
    import torch

    from paper_2506_03686_b200 import permute
    from paper_2506_03686_b200.sharded import emulate_sharded
    from paper_2506_03686_b200.workloads import CONFIGS

    wl = CONFIGS["cfg5"]
    x = torch.randint(-2**62, 2**62, (wl.numel,), dtype=torch.int64, device=cuda)
    want = permute(x.reshape(wl.shape), wl.axes).reshape(-1)
    outs = emulate_sharded(x, wl.shape, wl.axes, G)
    assert torch.equal(torch.cat([o.reshape(-1) for o in outs]), want)


def test_execute_host_pipelined_chunks(cuda):
    """Large host buffers go through the chunked H2D/kernel/D2H pipeline;
    the result equals the device-resident permutation."""
    import torch

    from paper_2506_03686_b200 import TensorLayout, build_program, execute, from_numpy_convention, permute

    rng = np.random.default_rng(5)
    for shape, axes in [((2,) * 24, tuple(rng.permutation(24).tolist())),
                        ((8, 16, 64, 2048), (3, 0, 2, 1)),
                        ((4, 4, 8, 8, 4096), (1, 0, 3, 2, 4)),
                        ((16, 8, 128, 1024), (0, 2, 1, 3))]:
        prog = build_program(TensorLayout.from_shape(shape, 8), from_numpy_convention(axes))
        n = prog.num_elements
        host = torch.randint(-2**62, 2**62, (n,), dtype=torch.int64).pin_memory()
        out = torch.empty(n, dtype=torch.int64).pin_memory()
        execute(prog, host, out=out)
        want = permute(host.to(cuda).reshape(shape), axes).reshape(-1).cpu()
        assert torch.equal(out, want), (shape, axes, prog.metadata["host_chunks"])


def test_execute_host_nonblocking_stream(cuda):
    """blocking=False calls overlap (shared staging buffers, library-ordered
    reuse); every result must still be exact."""
    import torch

    from paper_2506_03686_b200 import TensorLayout, build_program, execute, from_numpy_convention, permute

    for shape, axes in [((2,) * 23, tuple(np.random.default_rng(2).permutation(23).tolist())),
                        ((37, 41, 29), (2, 0, 1))]:
        prog = build_program(TensorLayout.from_shape(shape, 8), from_numpy_convention(axes))
        n = prog.num_elements
        ins = [torch.randint(-2**62, 2**62, (n,), dtype=torch.int64).pin_memory() for _ in range(4)]
        outs = [torch.empty(n, dtype=torch.int64).pin_memory() for _ in range(4)]
        for i in range(4):
            execute(prog, ins[i], out=outs[i], blocking=False)
        torch.cuda.current_stream().synchronize()
        for i in range(4):
            want = permute(ins[i].to(cuda).reshape(shape), axes).reshape(-1).cpu()
            assert torch.equal(outs[i], want), (shape, i)
    with pytest.raises(Exception):
        execute(prog, ins[0], blocking=False)          # needs a pinned `out`


def test_execute_host_nonblocking_chained(cuda):
    """Feeding a non-blocking call's output back as the next input is ordered
    by the library (H2D waits for the earlier D2H)."""
    import torch

    from paper_2506_03686_b200 import TensorLayout, build_program, execute, from_numpy_convention

    shape, axes = (2,) * 22, tuple(range(21, -1, -1))          # involution: applying twice = identity
    prog = build_program(TensorLayout.from_shape(shape, 4), from_numpy_convention(axes))
    a = torch.randint(-2**31, 2**31 - 1, (prog.num_elements,), dtype=torch.int32).pin_memory()
    b = torch.empty_like(a).pin_memory()
    c = torch.empty_like(a).pin_memory()
    execute(prog, a, out=b, blocking=False)
    execute(prog, b, out=c, blocking=False)
    torch.cuda.current_stream().synchronize()
    assert torch.equal(c, a)
    assert not torch.equal(b, a)


def test_autotune_candidates_are_exact(cuda):
    """Every tile candidate the autotuner may pick is a valid plan: bit-exact
    against the oracle; the tuned program replaces the cached default."""
    import torch

    import paper_2506_03686_b200 as vp
    from paper_2506_03686_b200.api import execute_device

    shape, axes = (96, 70, 130), (2, 0, 1)
    lay, pm = vp.TensorLayout.from_shape(shape, 4), vp.from_numpy_convention(axes)
    x = np.random.default_rng(3).integers(0, 2**31, size=shape, dtype=np.int32)
    want = oracle.naive_permute_np(x.reshape(-1), lay.dims, pm.sigma).reshape(np.transpose(x, axes).shape)
    assert np.array_equal(want, np.transpose(x, axes))
    xd = torch.from_numpy(x).cuda()
    n = 0
    for c in range(12):
        try:
            p = vp.build_program(lay, pm, force="tile", candidate=c)
        except vp.LayoutError:
            break
        y = execute_device(p, xd)
        assert np.array_equal(y.cpu().numpy(), want), (c, p.metadata["src_run"], p.metadata["dst_run"])
        n += 1
    assert n >= 3
    best = vp.autotune(lay, pm, force="tile", candidates=4)
    assert vp.build_program(lay, pm, force="tile") is best
    assert np.array_equal(execute_device(best, xd).cpu().numpy(), want)
    assert best.metadata["tuned_ms"] > 0


def test_permute_of_permuted_views(cuda):
    """Permuted views of dense memory are permuted from their base with the
    composed axes (one kernel); other strided views are rejected."""
    import torch

    import paper_2506_03686_b200 as vp
    from paper_2506_03686_b200 import permute

    base = torch.randint(-2**31, 2**31 - 1, (6, 1, 10, 12, 7), dtype=torch.int32, device="cuda")
    rng = np.random.default_rng(4)
    for _ in range(20):
        p1 = tuple(int(a) for a in rng.permutation(5))
        p2 = tuple(int(a) for a in rng.permutation(5))
        v = base.permute(p1)
        assert torch.equal(permute(v, p2), v.permute(p2).contiguous())
    m = base.reshape(60, 84)
    assert torch.equal(permute(m.mT, (1, 0)), m)
    with pytest.raises(vp.LayoutError):
        permute(base[:, :, ::2], (0, 1, 2, 3, 4))


def test_concurrent_host_threads(cuda):
    """Plans are shareable and vpg_permute is safe from several host threads
    on distinct streams (include/vpgpu.h threading contract), including the
    first launch of specialised kernels (NVRTC compile under contention) and
    the host-buffer pipeline."""
    import threading

    import torch

    import paper_2506_03686_b200 as vp
    from paper_2506_03686_b200.api import execute_device

    shapes = [((64, 96, 130), (2, 0, 1)), ((33, 65, 129), (1, 2, 0)), ((2,) * 22, tuple(range(21, -1, -1))),
              ((128, 40, 3, 64), (3, 1, 0, 2))]
    progs = [vp.build_program(vp.TensorLayout.from_shape(s, 4), vp.from_numpy_convention(a), jit=True)
             for s, a in shapes]
    vp.program_cache_clear()
    inputs = [torch.randint(-2**31, 2**31 - 1, s, dtype=torch.int32, device="cuda") for s, _ in shapes]
    wants = [x.permute(a).contiguous() for x, (_, a) in zip(inputs, shapes)]
    torch.cuda.synchronize()
    errors = []

    def worker(tid):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for it in range(6):
                    k = (tid + it) % len(shapes)
                    y = execute_device(progs[k], inputs[k], stream=st)
                    st.synchronize()
                    if not torch.equal(y, wants[k]):
                        errors.append((tid, k, "device"))
            if tid % 2 == 0:                               # host-buffer pipeline from threads too
                k = tid % len(shapes)
                out, _ = vp.execute(progs[k], inputs[k].cpu())
                if not torch.equal(torch.as_tensor(out).reshape(wants[k].shape), wants[k].cpu()):
                    errors.append((tid, k, "host"))
        except Exception as e:  # pragma: no cover - reported below
            errors.append((tid, repr(e)))

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    assert all(p.jit_state == 2 for p in progs)


def test_cuda_graph_capture_and_replay(cuda):
    """Launches are capturable in a CUDA graph (stream-ordered, no host
    synchronisation inside vpg_permute); replays stay bit-exact as the
    input buffer changes."""
    import torch

    import paper_2506_03686_b200 as vp
    from paper_2506_03686_b200.api import execute_device

    cases = [((64, 96, 130), (2, 0, 1)), ((2,) * 21, tuple(range(20, -1, -1))), ((128, 8, 1024), (1, 0, 2))]
    progs = [vp.build_program(vp.TensorLayout.from_shape(s, 4), vp.from_numpy_convention(a)) for s, a in cases]
    xs = [torch.empty(s, dtype=torch.int32, device="cuda") for s, _ in cases]
    ys = [torch.empty(p.out_shape, dtype=torch.int32, device="cuda") for p in progs]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for p, x, y in zip(progs, xs, ys):       # first launches (kernel loading) outside the capture
            execute_device(p, x, out=y, stream=st)
    st.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for p, x, y in zip(progs, xs, ys):
            execute_device(p, x, out=y, stream=st)
    for it in range(3):
        for x in xs:
            x.copy_(torch.randint(-2**31, 2**31 - 1, x.shape, dtype=torch.int32, device="cuda"))
        g.replay()
        torch.cuda.synchronize()
        for x, y, (_, a) in zip(xs, ys, cases):
            assert torch.equal(y, x.permute(a).contiguous()), it


def test_c_api_demo_program(cuda, tmp_path):
    """The C ABI from plain C (examples/c_api_demo.c): plan, permute and the
    fused sharded exchange on caller-owned cudaMalloc buffers, checked on the
    host against the closed-form bijection."""
    import os
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "c_api_demo")
    lib = os.path.join(root, "paper_2506_03686_b200")
    cmd = ["gcc", "-O2", "-I", os.path.join(root, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(root, "examples", "c_api_demo.c"), "-o", exe, "-L", lib, "-lvpgpu",
           "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{lib}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    res = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "permute: 0 mismatches" in res.stdout
    assert "sharded exchange (G=4): 0 mismatches" in res.stdout


@pytest.mark.parametrize("shape,axes,elem", [
    ((5, 3, 96, 29, 95), (1, 0, 2, 3, 4), 4),       # 15 rows of 264480 words: rows cut into chunks
    ((3, 2, 61, 1000), (1, 0, 2, 3), 8),            # 6 rows of 61000 8-byte words (odd lengths go to the tile kernel)
    ((7, 5, 1, 20016), (1, 0, 2, 3), 2),            # 2-byte words
    ((2, 3, 7, 4097), (1, 0, 2, 3), 16),            # 16-byte words
])
def test_rows_kernel_few_long_rows(cuda, shape, axes, elem):
    """Few long rows are cut into chunks (work items) so they fill the GPU;
    every chunk boundary and the short last chunk land bit-exact."""
    import torch

    import paper_2506_03686_b200 as vp
    from paper_2506_03686_b200.api import execute_device

    n = int(np.prod(shape))
    prog = vp.build_program(vp.TensorLayout.from_shape(shape, elem), vp.from_numpy_convention(axes))
    assert prog.kernel == "rows"
    words = np.random.default_rng(elem).integers(0, 256, size=n * elem, dtype=np.uint8)
    x = torch.from_numpy(words).cuda()
    y = execute_device(prog, x)
    want = np.ascontiguousarray(np.transpose(words.view(f"V{elem}").reshape(shape), axes)).reshape(-1).view(np.uint8)
    assert np.array_equal(y.cpu().numpy().reshape(-1), want)
    # misaligned base pointer: narrower vectors, same chunking
    xb = torch.empty(n * elem + 16, dtype=torch.uint8, device="cuda")
    xs = xb[elem:elem + n * elem]
    xs.copy_(x)
    y2 = execute_device(prog, xs)
    assert np.array_equal(y2.cpu().numpy().reshape(-1), want)


def test_env_measured_planning(cuda, monkeypatch):
    """VPG_TUNE=1: large tile plans are tuned on first build, bit-exact,
    and later builds return the tuned program."""
    import torch

    import paper_2506_03686_b200 as vp
    from paper_2506_03686_b200.api import execute_device

    monkeypatch.setenv("VPG_TUNE", "1")
    vp.program_cache_clear()
    shape, axes = (1031, 4099), (1, 0)
    lay, pm = vp.TensorLayout.from_shape(shape, 4), vp.from_numpy_convention(axes)
    p = vp.build_program(lay, pm)
    assert p.kernel == "tile" and p.metadata.get("tuned_ms", 0) > 0
    assert vp.build_program(lay, pm) is p
    x = torch.randint(-2**31, 2**31 - 1, shape, dtype=torch.int32, device="cuda")
    assert torch.equal(execute_device(p, x), x.permute(axes).contiguous())
    vp.program_cache_clear()


def test_rows_kernel_random_campaign(cuda):
    """Stride-1-preserving permutations of random shapes and word sizes (the
    ROWS kernel's row/chunk/lane-count choices, and the tile kernel where
    rows are narrow): bit-exact against numpy, aligned and offset bases."""
    import torch

    import paper_2506_03686_b200 as vp
    from paper_2506_03686_b200.api import execute_device

    rng = np.random.default_rng(77)
    kinds = set()
    for it in range(60):
        E = int(rng.choice([1, 2, 4, 8, 16]))
        r = int(rng.integers(2, 5))
        lead = [int(rng.integers(1, 12)) for _ in range(r - 1)]
        row = int(rng.choice([int(rng.integers(1, 3000)), int(rng.integers(3000, 200000))]))
        shape = tuple(lead + [row])
        n = int(np.prod(shape))
        if n * E > (64 << 20):
            continue
        axes = tuple(int(a) for a in rng.permutation(r - 1)) + (r - 1,)
        prog = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes))
        kinds.add(prog.kernel)
        words = rng.integers(0, 256, size=n * E, dtype=np.uint8)
        want = np.ascontiguousarray(np.transpose(words.view(f"V{E}").reshape(shape), axes)).reshape(-1).view(np.uint8)
        off = int(rng.choice([0, E, 16]))
        buf = torch.empty(n * E + 32, dtype=torch.uint8, device="cuda")
        x = buf[off:off + n * E]
        x.copy_(torch.from_numpy(words))
        y = execute_device(prog, x)
        assert np.array_equal(y.cpu().numpy().reshape(-1), want), (shape, axes, E, off, prog.kernel)
    assert "rows" in kinds


@pytest.mark.parametrize("shape,axes,elem,scratch_mib", [
    ((64, 48, 40, 512), (2, 0, 3, 1), 4, 64),       # 240 MiB through 64 MiB of scratch
    ((2,) * 26, tuple(range(25, -1, -1)), 8, 48),    # 512 MiB, rank 26
    ((96, 130, 4097), (1, 2, 0), 2, 40),             # odd extents, 2-byte words
])
def test_host_path_bounded_scratch(cuda, shape, axes, elem, scratch_mib):
    """Host tensors streamed through device scratch smaller than the tensor
    (chunk ring): bit-exact, and the device never holds the whole tensor."""
    import torch

    import paper_2506_03686_b200 as vp

    n = int(np.prod(shape))
    prog = vp.build_program(vp.TensorLayout.from_shape(shape, elem), vp.from_numpy_convention(axes))
    words = np.random.default_rng(elem).integers(0, 256, size=n * elem, dtype=np.uint8)
    x = torch.from_numpy(words).pin_memory()
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    out, _ = vp.execute(prog, x, max_device_bytes=scratch_mib << 20)
    peak = torch.cuda.max_memory_allocated() - base
    assert peak <= (scratch_mib << 20) + (1 << 20)
    want = np.ascontiguousarray(np.transpose(words.view(f"V{elem}").reshape(shape), axes)).reshape(-1).view(np.uint8)
    assert np.array_equal(out.view(torch.uint8).numpy().reshape(-1), want)


def test_host_path_bounded_scratch_unsplittable(cuda):
    """A 2-D transpose of prime extents cannot be cut into chunks: the
    bounded path reports it (LayoutError), it does not fall back."""
    import torch

    import paper_2506_03686_b200 as vp

    shape = (1009, 4093)
    prog = vp.build_program(vp.TensorLayout.from_shape(shape, 4), vp.from_numpy_convention((1, 0)))
    x = torch.zeros(shape, dtype=torch.int32)
    with pytest.raises(vp.LayoutError):
        vp.execute(prog, x, max_device_bytes=1 << 20)


@pytest.mark.parametrize("shape,axes,elem", [
    ((3, 2, 64, 1001), (1, 0, 2, 3), 8),        # rows cut into chunks
    ((20, 12, 66), (1, 0, 2), 8),               # short predicated rows
    ((7, 3, 4100), (1, 0, 2), 4),               # rows, exact-multiple fast path off
    ((3, 1000003), (0, 1), 4),                  # chunked copy with a tail
    ((2, 3, 7, 4097), (1, 0, 2, 3), 16),        # 16-byte words, rows
])
def test_guard_bands_new_paths(cuda, shape, axes, elem):
    """Guard bands around source AND destination for the chunked rows and
    copy kernels: no write outside the destination, no change to the
    source, bit-exact result (compute-sanitizer is unavailable here)."""
    import torch

    import paper_2506_03686_b200 as vp
    from paper_2506_03686_b200.api import execute_device

    n = int(np.prod(shape)) * elem
    G = 1 << 16
    words = np.random.default_rng(n).integers(0, 256, size=n, dtype=np.uint8)
    sbuf = torch.full((n + 2 * G,), 0xA5, dtype=torch.uint8, device="cuda")
    dbuf = torch.full((n + 2 * G,), 0x5A, dtype=torch.uint8, device="cuda")
    sbuf[G:G + n] = torch.from_numpy(words).cuda()
    prog = vp.build_program(vp.TensorLayout.from_shape(shape, elem), vp.from_numpy_convention(axes))
    execute_device(prog, sbuf[G:G + n], out=dbuf[G:G + n])
    d, s_ = dbuf.cpu().numpy(), sbuf.cpu().numpy()
    assert (d[:G] == 0x5A).all() and (d[G + n:] == 0x5A).all()
    assert (s_[:G] == 0xA5).all() and (s_[G + n:] == 0xA5).all() and np.array_equal(s_[G:G + n], words)
    want = np.ascontiguousarray(np.transpose(words.view(f"V{elem}").reshape(shape), axes)).reshape(-1).view(np.uint8)
    assert np.array_equal(d[G:G + n], want), prog.kernel


@pytest.mark.parametrize("shape,axes", [((4096, 4096), (1, 0)),                 # tile, specialised
                                        ((32, 64, 56, 56), (0, 2, 3, 1)),       # tile, multi-dim
                                        ((64, 32, 2048), (1, 0, 2)),            # rows
                                        ((1 << 24,), (0,)),                     # copy
                                        ((7, 9, 13, 5, 11), (4, 1, 0, 3, 2))])  # misaligned tile
def test_back_to_back_dependent_launches(cuda, shape, axes):
    """Launches carry the programmatic-dependent-launch attribute: a chain
    in which every launch reads the previous launch's output (x -> y -> x'
    -> y' ...) must still see complete inputs (the kernels' griddepcontrol
    wait precedes their first global load)."""
    import torch

    from paper_2506_03686_b200 import TensorLayout, build_program, from_numpy_convention
    from paper_2506_03686_b200.api import execute_device

    inv = tuple(int(i) for i in np.argsort(axes))
    out_shape = tuple(shape[a] for a in axes)
    fwd = build_program(TensorLayout.from_shape(shape, 4), from_numpy_convention(axes))
    bwd = build_program(TensorLayout.from_shape(out_shape, 4), from_numpy_convention(inv))
    g = torch.Generator(device=cuda).manual_seed(11)
    x0 = torch.randint(-2**31, 2**31 - 1, (int(np.prod(shape)),), dtype=torch.int32, device=cuda, generator=g)
    a, b = x0.clone(), torch.empty_like(x0)
    for _ in range(24):
        execute_device(fwd, a, out=b)
        execute_device(bwd, b, out=a)
    want_b = _want(x0.cpu().numpy().reshape(shape), axes).reshape(-1)
    torch.cuda.synchronize()
    assert torch.equal(a, x0)
    assert np.array_equal(b.cpu().numpy(), want_b)


def test_rank_above_64_unit_dims_permute(cuda):
    """A rank-70 tensor whose size-1 dims bring it within the limit permutes
    like its squeezed form (the reference has no rank cap, core.py:58-88)."""
    import numpy as np
    import torch

    from paper_2506_03686_b200 import permute

    rng = np.random.default_rng(11)
    shape = [1] * 70
    big = rng.choice(70, 5, replace=False)
    for k, e in zip(big, (33, 17, 9, 5, 12)):
        shape[k] = int(e)
    axes = tuple(int(v) for v in rng.permutation(70))
    n = int(np.prod(shape))
    x = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device=cuda)
    y = permute(x.view(shape), axes)
    torch.cuda.synchronize()
    keep = [a for a in range(70) if shape[a] > 1]
    sq_axes = [keep.index(a) for a in axes if shape[a] > 1]
    want = x.view([shape[a] for a in keep]).permute(sq_axes).contiguous()
    assert list(y.shape) == [shape[a] for a in axes]
    assert torch.equal(y.reshape(-1), want.reshape(-1))


def test_dynamic_tile_scheduler_reuse_and_streams(cuda):
    """The dynamic tile scheduler's counter pairs (kernels.cu sched_slot) are
    reset by each launch's last CTA and reused ring-wise: >4096 launches
    (the ring wraps) of multi-wave tile and rows plans, interleaved over two
    streams, all bit-exact."""
    import torch

    from paper_2506_03686_b200 import TensorLayout, build_program, from_numpy_convention
    from paper_2506_03686_b200.api import execute_device

    # (2048, 2048, 8) f32: 8192 tiles >> S x grid; (256, 64, 16, 1024): 4 KiB rows, TMA bulk rows kernel
    cases = [((2048, 2048, 8), (1, 0, 2)), ((256, 64, 16, 1024), (2, 0, 1, 3))]
    progs, xs, wants = [], [], []
    for shape, axes in cases:
        n = 1
        for d in shape:
            n *= d
        x = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device=cuda)
        p = build_program(TensorLayout.from_shape(shape, 4), from_numpy_convention(axes))
        progs.append(p)
        xs.append(x)
        wants.append(x.view(shape).permute(axes).contiguous().reshape(-1))
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [[torch.empty_like(x) for x in xs] for _ in streams]
    assert [p.kernel for p in progs] == ["tile", "rows"]
    for it in range(2100):
        for si, st in enumerate(streams):
            for ci in range(len(cases)):
                execute_device(progs[ci], xs[ci], out=outs[si][ci], stream=st)
        if it % 700 == 699:
            torch.cuda.synchronize()
            for si in range(len(streams)):
                for ci in range(len(cases)):
                    assert torch.equal(outs[si][ci], wants[ci]), (it, si, ci, progs[ci].kernel)
                    with torch.cuda.stream(streams[si]):
                        outs[si][ci].zero_()
    torch.cuda.synchronize()


@pytest.mark.parametrize("shape,axes", [((36, 106, 439), (1, 0, 2)), ((3, 2, 61, 1001), (1, 0, 2, 3)),
                                        ((7, 5, 257), (1, 0, 2))])
def test_odd_rows_take_tile_kernel(cuda, shape, axes):
    """Stride-1-preserving permutations of 8-byte words whose rows are not a
    multiple of 16 bytes run on the tile kernel (residue rows, 16-byte
    accesses), bit-exact, at aligned and offset bases."""
    import torch

    import paper_2506_03686_b200 as vp
    from paper_2506_03686_b200.api import execute_device

    prog = vp.build_program(vp.TensorLayout.from_shape(shape, 8), vp.from_numpy_convention(axes))
    assert prog.kernel == "tile", prog.text
    n = int(np.prod(shape))
    x = torch.randint(-2**62, 2**62, (n + 2,), dtype=torch.int64, device="cuda")
    for off in (0, 1):
        xv = x[off:off + n]
        y = execute_device(prog, xv.view(torch.uint8))
        assert torch.equal(y.view(torch.int64), xv.view(shape).permute(axes).reshape(-1)), off
