"""Sharded multi-GPU permutation: local pack permute -> all-to-all -> local
unpack permute (BASELINE.json cfg5 at 2/4/8 B200).

Input and output are each sharded along their own leading axis: rank r owns
the contiguous slice [r*N/G, (r+1)*N/G) of the flattened input and of the
flattened output.  When the leading axis is shorter than G (cfg5: extent 2,
G = 8) "leading axis" means the leading axes whose product is G; a dim that
straddles the boundary is split into (outer, inner) factors.  After that
refinement:

  I  = input axes that index the source rank (input-leading axes)
  O  = input axes that index the destination rank (output-leading axes)
  D  = O \\ I   (axes a rank sends along: one contiguous chunk per value)
  M  = axes in neither I nor O (they survive to the local output)

  P1 (local GPU permute):  local input [all axes but I, input order]
                           -> [D (output order)] + [M (output order)]
  all-to-all (NCCL over NVLink/NVSwitch): chunk d of P1 goes to rank s(d);
                           ranks whose I∩O coordinates differ exchange nothing
  P2 (local GPU permute):  received [I\\O (input order)] + [M (output order)]
                           -> local output [all axes but O, output order]

If I and O coincide (same set, same order) the step is purely local; if the
sets match in a different order it is a fixed pairwise exchange.  Both fall
out of the general formula (one chunk per rank).  There is no collective
other than the one all-to-all the permutation needs.

The local permutes default to the GPU kernels (``permute``); the CPU tests
inject the oracle to exercise the exchange logic with the gloo backend.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

from .core import LayoutError

__all__ = ["ShardPlan", "plan_sharded", "permute_sharded", "permute_sharded_pipelined", "pipeline_chunks", "pipeline_spec",
           "shard_bounds", "ShardExchange", "exchange_input", "emulate_fused", "emulate_sharded_pipelined", "fused_supported",
           "fused_method", "release_exchanges"]


def _lead_split(shape, G):
    """Walk `shape` from the outermost dim taking factors until their product
    is G.  Returns {dim: outer_factor} for every dim touched (outer_factor ==
    shape[dim] for whole dims).  Raises LayoutError if G does not divide the
    leading dims cleanly."""
    rem = G
    cuts = {}
    for i, d in enumerate(shape):
        if rem == 1:
            break
        if d <= rem and rem % d == 0:
            cuts[i] = d
            rem //= d
        elif d % rem == 0:
            cuts[i] = rem
            rem = 1
        else:
            g = math.gcd(d, rem)
            raise LayoutError(f"cannot shard: dim {i} of size {d} vs remaining factor {rem} (gcd {g})")
    if rem != 1:
        raise LayoutError(f"tensor of shape {tuple(shape)} has fewer than {G} leading elements")
    return cuts


@dataclass(frozen=True)
class ShardPlan:
    G: int
    shape: tuple            # global input shape (outer-first)
    axes: tuple             # global permutation (numpy convention)
    rshape: tuple           # refined input shape
    raxes: tuple            # refined permutation
    I: tuple                # refined input axes indexing the source rank (input order)
    O: tuple                # refined input axes indexing the destination rank (output order)
    D: tuple                # O \ I in output order
    M: tuple                # the rest, output order
    IO: tuple               # I \ O in input order

    @property
    def numel(self):
        n = 1
        for d in self.rshape:
            n *= d
        return n

    @property
    def local_numel(self):
        return self.numel // self.G

    def local_in_axes(self):
        return tuple(a for a in range(len(self.rshape)) if a not in self.I)

    def local_in_shape(self):
        return tuple(self.rshape[a] for a in self.local_in_axes())

    def out_shape(self):
        return tuple(self.shape[a] for a in self.axes)

    def local_out_axes(self):
        return tuple(a for a in self.raxes if a not in self.O)

    def local_out_shape(self):
        return tuple(self.rshape[a] for a in self.local_out_axes())

    def p1(self):
        """(local input shape, axes) of the pack permute."""
        L = self.local_in_axes()
        order = list(self.D) + list(self.M)
        return self.local_in_shape(), tuple(L.index(a) for a in order)

    def p2(self):
        """(received shape, axes) of the unpack permute."""
        recv = list(self.IO) + list(self.M)
        tgt = self.local_out_axes()
        return tuple(self.rshape[a] for a in recv), tuple(recv.index(a) for a in tgt)

    def _coords(self, index, axes_list):
        c = {}
        for a in reversed(axes_list):
            c[a] = index % self.rshape[a]
            index //= self.rshape[a]
        return c

    def _index(self, coords, axes_list):
        i = 0
        for a in axes_list:
            i = i * self.rshape[a] + coords[a]
        return i

    def send_counts(self, r):
        """Elements rank r sends to each destination rank."""
        cin = self._coords(r, self.I)
        chunk = 1
        for a in self.M:
            chunk *= self.rshape[a]
        counts = [0] * self.G
        nd = 1
        for a in self.D:
            nd *= self.rshape[a]
        for d in range(nd):
            c = dict(cin)
            c.update(self._coords(d, self.D))
            counts[self._index(c, self.O)] += chunk
        return counts

    def recv_counts(self, s):
        """Elements rank s receives from each source rank."""
        return [self.send_counts(r)[s] for r in range(self.G)]

    def describe(self):
        return (f"G={self.G} refined shape {self.rshape} axes {self.raxes}; I={self.I} O={self.O} "
                f"D={self.D} M={self.M}; P1 {self.p1()} P2 {self.p2()}")


def plan_sharded(shape, axes, G) -> ShardPlan:
    shape = tuple(int(d) for d in shape)
    axes = tuple(int(a) for a in axes)
    n = len(shape)
    if sorted(axes) != list(range(n)):
        raise LayoutError(f"axes {axes} are not a permutation of 0..{n - 1}")
    if G < 1:
        raise LayoutError("G must be >= 1")
    in_cuts = _lead_split(shape, G)
    out_cuts_pos = _lead_split([shape[a] for a in axes], G)
    out_cuts = {axes[j]: f for j, f in out_cuts_pos.items()}
    # refine every dim into nested (outer -> inner) factors
    pieces = []        # per original dim: list of (refined extent)
    for i, d in enumerate(shape):
        cuts = sorted({c for c in (in_cuts.get(i), out_cuts.get(i)) if c is not None and 1 < c < d})
        if len(cuts) == 2 and cuts[1] % cuts[0]:
            raise LayoutError(f"cannot shard: dim {i} needs incompatible splits {cuts}")
        fac = []
        prev = 1
        for c in cuts:
            fac.append(c // prev)
            prev = c
        fac.append(d // prev)
        pieces.append(fac)
    first = []
    acc = 0
    for fac in pieces:
        first.append(acc)
        acc += len(fac)
    rshape = tuple(x for fac in pieces for x in fac)
    raxes = tuple(first[a] + k for a in axes for k in range(len(pieces[a])))

    def lead(ax_order):
        got, prod = [], 1
        for a in ax_order:
            if prod == G:
                break
            got.append(a)
            prod *= rshape[a]
        if prod != G:
            raise LayoutError("internal: refined leading product mismatch")
        return tuple(got)

    I = lead(range(len(rshape))) if G > 1 else ()
    O = lead(raxes) if G > 1 else ()
    Iset, Oset = set(I), set(O)
    D = tuple(a for a in O if a not in Iset)
    M = tuple(a for a in raxes if a not in Iset and a not in Oset)
    IO = tuple(a for a in I if a not in Oset)
    return ShardPlan(G, shape, axes, rshape, raxes, I, O, D, M, IO)


def shard_bounds(numel, G, r):
    """Element range of rank r's contiguous shard."""
    per = numel // G
    return r * per, (r + 1) * per


def permute_sharded(local_in, global_shape, axes, group=None, local_permute=None, plan=None,
                    method: str = "alltoall"):
    """Permute a tensor sharded across the ranks of `group`.

    local_in: this rank's contiguous input shard (any shape, numel N/G).
    Returns this rank's contiguous output shard, shaped as the local output
    (output axes beyond the rank-indexing ones).  Collective: every rank of
    the group must call it with the same shape/axes.

    method: "alltoall" -- P1 permute -> all_to_all_single -> P2 permute;
    "pipelined" -- the same pipelined over chunks (permute_sharded_pipelined);
    "fused" -- one exchange kernel per rank over peer memory (ShardExchange:
    push = stores into the peers' output shards, whose result stays valid
    until the second-next fused call with the same arguments; pull = reads
    from the peers' input shards: produce the input in exchange_input(...)
    to avoid a staging copy); "auto" -- fused when one of the two keeps runs
    of at least 128 bytes on the remote side (fused_method), else pipelined
    when the shard has a pipelining axis, else the all-to-all.
    """
    import torch
    import torch.distributed as dist

    G = dist.get_world_size(group) if dist.is_initialized() else 1
    r = dist.get_rank(group) if dist.is_initialized() else 0
    if method not in ("alltoall", "fused", "auto", "pipelined"):
        raise ValueError(f"unknown method {method!r}")
    if method == "pipelined":
        return permute_sharded_pipelined(local_in, global_shape, axes, group=group, local_permute=local_permute,
                                         plan=plan)
    if method != "alltoall" and local_permute is None and local_in.is_cuda:
        if method == "fused" or fused_supported(global_shape, axes, local_in.element_size(), G):
            ex = _exchange_for(tuple(global_shape), tuple(axes), local_in.dtype, local_in.device, group)
            return ex(local_in)
    sp = plan or plan_sharded(global_shape, axes, G)
    if method == "auto" and pipeline_chunks(sp) > 1:
        return permute_sharded_pipelined(local_in, global_shape, axes, group=group, local_permute=local_permute,
                                         plan=sp)
    if local_permute is None:
        from .api import permute as local_permute  # GPU kernels; no CPU fallback
    if local_in.numel() != sp.local_numel:
        raise LayoutError(f"rank {r}: shard holds {local_in.numel()} elements, expected {sp.local_numel}")
    if G == 1:
        return local_permute(local_in.reshape(sp.shape), sp.axes)
    s1, a1 = sp.p1()
    packed = local_permute(local_in.reshape(s1), a1).reshape(-1)
    es = packed.element_size()
    send = [c * es for c in sp.send_counts(r)]
    recv_c = [c * es for c in sp.recv_counts(r)]
    # NCCL moves device buffers directly over NVLink/NVSwitch; the gloo
    # backend (CPU transport) needs host buffers, so device data is staged.
    staged = packed.is_cuda and dist.get_backend(group) == "gloo"
    payload = packed.view(torch.uint8)
    if staged:
        payload = payload.cpu()
    recv = torch.empty(sum(recv_c), dtype=torch.uint8, device=payload.device)
    dist.all_to_all_single(recv, payload, recv_c, send, group=group)
    if staged:
        recv = recv.to(packed.device)
    s2, a2 = sp.p2()
    got = recv.view(packed.dtype).reshape(s2)
    return local_permute(got, a2).reshape(sp.local_out_shape())


def pipeline_spec(sp: ShardPlan, chunks: int = 4):
    """Chunking of the pipelined all-to-all path: a list of (axis, factor)
    over the outermost axes of the local input, so every chunk is a
    contiguous slice of the shard.  Every listed axis must survive to the
    local output (an M axis: each destination then receives 1/C of its data
    per chunk); all but the last are enumerated whole, the last may be cut
    to a divisor of its extent.  C = product of the factors <= `chunks`
    (empty list: no pipelining)."""
    L = sp.local_in_axes()
    spec, C = [], 1
    for a in L:
        if sp.G == 1 or a not in sp.M or C >= chunks:
            break
        e = sp.rshape[a]
        f = next((c for c in range(min(chunks // C, e), 1, -1) if e % c == 0), 1)
        if f < 2:
            break
        spec.append((a, f))
        C *= f
        if f < e:
            break              # a cut axis ends the prefix
    return spec


def pipeline_chunks(sp: ShardPlan, chunks: int = 4) -> int:
    """Number of chunks of the pipelined path (1 = not pipelined)."""
    C = 1
    for _, f in pipeline_spec(sp, chunks):
        C *= f
    return C


def _pipelined_programs(sp: ShardPlan, spec):
    """(P1 chunk shape, axes) and (P2 shape, axes) of the pipelined path.
    P1 permutes one contiguous input chunk into [D][M_c] (M_c: M without the
    whole chunk axes, the cut axis at extent e/f); P2 permutes the
    chunk-major receive buffer [chunk digits][IO][M_c] into the local output,
    each chunk digit becoming (the outer factor of) its axis."""
    full = {a for a, f in spec if f == sp.rshape[a]}
    cut = {a: f for a, f in spec if f < sp.rshape[a]}

    def ext(a):
        return sp.rshape[a] // cut[a] if a in cut else sp.rshape[a]

    L = [a for a in sp.local_in_axes() if a not in full]
    T = [a for a in list(sp.D) + list(sp.M) if a not in full]
    p1 = (tuple(ext(a) for a in L), tuple(L.index(a) for a in T))
    recv = [a for a in list(sp.IO) + list(sp.M) if a not in full]
    k = len(spec)
    shape = tuple(f for _, f in spec) + tuple(ext(a) for a in recv)
    cidx = {a: i for i, (a, _) in enumerate(spec)}
    axes = []
    for a in sp.local_out_axes():
        if a in full:
            axes.append(cidx[a])
        elif a in cut:
            axes.extend([cidx[a], k + recv.index(a)])
        else:
            axes.append(k + recv.index(a))
    return p1, (shape, tuple(axes))


def permute_sharded_pipelined(local_in, global_shape, axes, group=None, local_permute=None, plan=None,
                              chunks: int = 4):
    """P1 -> all-to-all -> P2 with the pack permute and the exchange
    pipelined over C chunks: P1 of chunk c+1 runs on
    the current stream while the all-to-all of chunk c runs on NCCL's stream,
    and one P2 permutes the chunk-major receive buffer.  Shapes without a
    pipelining axis (pipeline_chunks == 1) take the serial path.  Same
    arguments and result as permute_sharded(method="alltoall")."""
    import torch
    import torch.distributed as dist

    G = dist.get_world_size(group) if dist.is_initialized() else 1
    r = dist.get_rank(group) if dist.is_initialized() else 0
    sp = plan or plan_sharded(global_shape, axes, G)
    spec = pipeline_spec(sp, chunks)
    C = pipeline_chunks(sp, chunks)
    if C == 1:
        return permute_sharded(local_in, global_shape, axes, group=group, local_permute=local_permute, plan=sp)
    if local_permute is None:
        from .api import permute as local_permute  # GPU kernels; no CPU fallback
    if local_in.numel() != sp.local_numel:
        raise LayoutError(f"rank {r}: shard holds {local_in.numel()} elements, expected {sp.local_numel}")
    (s1c, a1), (s2c, a2c) = _pipelined_programs(sp, spec)
    xin = local_in.reshape(C, -1)
    es = local_in.element_size()
    send = [c * es // C for c in sp.send_counts(r)]
    recv_c = [c * es // C for c in sp.recv_counts(r)]
    nrecv = sum(recv_c)
    staged = local_in.is_cuda and dist.get_backend(group) == "gloo"
    dev = local_in.device
    recv = torch.empty(C * nrecv, dtype=torch.uint8, device="cpu" if staged else dev)
    works, keep = [], []
    cuda = local_in.is_cuda and not staged
    comm = torch.cuda.Stream(dev) if cuda else None
    for c in range(C):
        packed = local_permute(xin[c].reshape(s1c), a1).reshape(-1).view(torch.uint8)
        if staged:
            packed = packed.cpu()
        if cuda:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(dev))
            comm.wait_event(ev)
            with torch.cuda.stream(comm):
                # NCCL orders the collective after `comm`, i.e. after P1 of
                # chunk c; P1 of chunk c+1 proceeds on the current stream
                works.append(dist.all_to_all_single(recv[c * nrecv:(c + 1) * nrecv], packed, recv_c, send,
                                                    group=group, async_op=True))
            packed.record_stream(comm)
        else:
            works.append(dist.all_to_all_single(recv[c * nrecv:(c + 1) * nrecv], packed, recv_c, send,
                                                group=group, async_op=True))
        keep.append(packed)
    for w in works:
        w.wait()                                    # current stream waits for every chunk's exchange
    if cuda:
        torch.cuda.current_stream(dev).wait_stream(comm)
        recv.record_stream(comm)
    if staged:
        recv = recv.to(dev)
    got = recv.view(local_in.dtype).reshape(s2c)
    return local_permute(got, a2c).reshape(sp.local_out_shape())


def emulate_sharded_pipelined(x_flat, global_shape, axes, G, local_permute=None, chunks: int = 4):
    """permute_sharded_pipelined for G virtual ranks on ONE device (rank after
    rank, the chunked all-to-all as buffer slicing): validates the chunked
    P1 programs, the chunk-major receive layout and the P2 program."""
    import torch

    if local_permute is None:
        from .api import permute as local_permute
    sp = plan_sharded(global_shape, axes, G)
    spec = pipeline_spec(sp, chunks)
    C = pipeline_chunks(sp, chunks)
    if C == 1:
        return emulate_sharded(x_flat, global_shape, axes, G, local_permute=local_permute)
    n = sp.numel
    (s1c, a1), (s2c, a2c) = _pipelined_programs(sp, spec)
    packed = []            # packed[r][c]
    for r in range(G):
        lo, hi = shard_bounds(n, G, r)
        xin = x_flat[lo:hi].reshape(C, -1)
        packed.append([local_permute(xin[c].reshape(s1c), a1).reshape(-1) for c in range(C)])
    outs = []
    for s in range(G):
        parts = []
        for c in range(C):
            for r in range(G):
                sc = [k // C for k in sp.send_counts(r)]
                off = sum(sc[:s])
                if sc[s]:
                    parts.append(packed[r][c][off:off + sc[s]])
        got = torch.cat(parts).reshape(s2c)
        outs.append(local_permute(got, a2c).reshape(sp.local_out_shape()))
    return outs


def emulate_sharded(x_flat, global_shape, axes, G, local_permute=None):
    """Run the G-rank algorithm on ONE device, rank after rank (P1 of every
    virtual rank, the all-to-all as buffer slicing, then P2 of every rank).
    Nothing waits on another rank's kernels; this validates the exact P1/P2
    programs and chunk bookkeeping the ranks execute.  Returns the list of
    per-rank output shards."""
    import torch

    if local_permute is None:
        from .api import permute as local_permute
    sp = plan_sharded(global_shape, axes, G)
    n = sp.numel
    s1, a1 = sp.p1()
    packed = []
    for r in range(G):
        lo, hi = shard_bounds(n, G, r)
        packed.append(local_permute(x_flat[lo:hi].reshape(s1), a1).reshape(-1))
    outs = []
    s2, a2 = sp.p2()
    for s in range(G):
        parts = []
        for r in range(G):
            sc = sp.send_counts(r)
            off = sum(sc[:s])
            if sc[s]:
                parts.append(packed[r][off:off + sc[s]])
        got = torch.cat(parts).reshape(s2)
        outs.append(local_permute(got, a2).reshape(sp.local_out_shape()))
    return outs


# ------------------------------------------------------------------ fused exchange (K5)
MIN_FUSED_RUN_BYTES = 128      # K5 when the remote-side runs are >= 128 B


def _programs(global_shape, axes, elem_bytes, G, ranks, jit=None, pull=False):
    from .api import build_sharded_program
    from .core import TensorLayout, from_numpy_convention

    lay = TensorLayout.from_shape(tuple(global_shape), elem_bytes)
    pm = from_numpy_convention(tuple(axes))
    return [build_sharded_program(lay, pm, G, r, jit=jit, pull=pull) for r in ranks]


def fused_method(global_shape, axes, elem_bytes, G):
    """Which fused exchange suits this permutation: "push" when the push
    plan's destination runs are at least MIN_FUSED_RUN_BYTES (remote stores
    in whole sectors), else "pull" when the pull plan's source runs are
    (remote reads of whole sectors; its stores are local), else None (the
    all-to-all path).  Same answer on every rank: the tile geometry does not
    depend on the shard index."""
    try:
        (p,) = _programs(global_shape, axes, elem_bytes, G, [0])
        if p.metadata["dst_run"] * elem_bytes >= MIN_FUSED_RUN_BYTES:
            return "push"
    except LayoutError:
        pass
    try:
        (p,) = _programs(global_shape, axes, elem_bytes, G, [0], pull=True)
        if (p.metadata["src_run"] * elem_bytes >= MIN_FUSED_RUN_BYTES
                and p.metadata["dst_run"] * elem_bytes >= MIN_FUSED_RUN_BYTES):
            return "pull"
    except LayoutError:
        pass
    return None


def fused_supported(global_shape, axes, elem_bytes, G) -> bool:
    """True when one of the fused exchanges suits this permutation (fused_method)."""
    return fused_method(global_shape, axes, elem_bytes, G) is not None


class ShardExchange:
    """Fused sharded permutation for one process per GPU.

    A call runs ONE kernel per rank over CUDA IPC mappings of the peers'
    buffers (NVLink/NVSwitch peer memory): one HBM read and one write per
    element, no staging buffers and no all-to-all.
      * push (vpg_permute_sharded): each rank reads its own input shard (any
        contiguous tensor) and stores every tile into the output shard that
        owns it.  The output shards are the exchange's registered buffers:
        two of them, used alternately, so a result stays valid until the
        call after next (``copy_out=True`` returns a private copy instead).
      * pull (vpg_permute_sharded_pull): each rank writes its own output
        shard (a fresh tensor, or ``out=``) and reads every tile's source runs
        from the input shard that holds them.  The input shards are the
        exchange's registered buffers: fill ``ex.input`` (``input_buffer()``)
        and the call moves nothing else; any other tensor is first copied
        into it.
    Two stream-ordered barriers order the exchange: before (every input
    complete, every output free) and after (every rank's accesses done).
    With NCCL they are one-element all-reduces on the current stream; with
    gloo (CPU transport, tests) the stream is synchronised and the group
    barrier runs on the host.  Collective: all ranks construct and call it
    with the same arguments."""

    def __init__(self, global_shape, axes, dtype, group=None, device=None, jit=None, mode="auto",
                 copy_out=False, device_barrier=None):
        import torch
        import torch.distributed as dist

        from . import _lib

        self.group = group
        self.G = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.dtype = dtype
        es = torch.empty((), dtype=dtype).element_size()
        if mode == "auto":
            mode = fused_method(global_shape, axes, es, self.G) or "push"
        if mode not in ("push", "pull"):
            raise ValueError(f"unknown exchange mode {mode!r}")
        self.mode = mode
        (self.program,) = _programs(global_shape, axes, es, self.G, [self.rank], jit=jit, pull=mode == "pull")
        self.splan = plan_sharded(global_shape, axes, self.G)
        self.local_numel = self.splan.local_numel
        self.copy_out = copy_out
        self.calls = 0
        # registered (peer-mapped) buffers: the input shard (pull) or two
        # alternating output shards (push)
        if mode == "pull":
            self.input = torch.empty(self.local_numel, dtype=dtype, device=self.device)
            shared = [self.input]
        else:
            self.input = None
            self._outs = [torch.empty(self.local_numel, dtype=dtype, device=self.device) for _ in range(2)]
            shared = self._outs
        self.backend = dist.get_backend(group) if dist.is_initialized() else None
        self._flag = torch.zeros(1, dtype=torch.float32, device=self.device)
        self._imported = []
        self.peer_tables = [self._map(t) for t in shared]     # per buffer: G peer pointers
        self.peers = self.peer_tables[0]
        # device-side ordering (vpg_permute_sharded_sync) instead of the two
        # collectives per call: NCCL jobs (one GPU per rank) by default;
        # never with gloo, whose test ranks share one GPU (a flag wait could
        # then hold SMs another rank's kernel needs)
        import os

        if device_barrier is None:
            device_barrier = self.backend == "nccl" and self.G > 1 and os.environ.get("VPG_DEVICE_BARRIER", "1") != "0"
        self.device_barrier = bool(device_barrier) and self.G > 1
        self._sync = None
        if self.device_barrier:
            from . import _lib

            self._flags = torch.zeros(2 * self.G, dtype=torch.int64, device=self.device)
            self._done = torch.zeros(1, dtype=torch.int32, device=self.device)
            fl = self._map(self._flags)
            self._sync = _lib.ShardSync()
            for q in range(self.G):
                self._sync.flags[q] = fl[q]
            self._sync.done_counter = self._done.data_ptr()

    def _map(self, shared):
        """Export `shared` and import every peer's counterpart (CUDA IPC);
        returns the G buffer pointers in rank order (own first-hand)."""
        import torch
        import torch.distributed as dist

        from . import _lib

        L = _lib.lib()
        mine = (self.rank, bytes(0), 0)
        if self.G > 1:
            h = ctypes.create_string_buffer(_lib.VPG_IPC_HANDLE_BYTES)
            off = ctypes.c_uint64(0)
            with torch.cuda.device(self.device):
                _check_ipc(L.vpg_ipc_export(ctypes.c_void_p(shared.data_ptr()), h, ctypes.byref(off)))
            mine = (self.rank, h.raw, off.value)
            allh = [None] * self.G
            dist.all_gather_object(allh, mine, group=self.group)
        else:
            allh = [mine]
        peers = []
        with torch.cuda.device(self.device):
            for q, hraw, off in sorted(allh):
                if q == self.rank:
                    peers.append(shared.data_ptr())
                    continue
                ptr = ctypes.c_void_p()
                buf = ctypes.create_string_buffer(hraw, _lib.VPG_IPC_HANDLE_BYTES)
                _check_ipc(L.vpg_ipc_import(buf, ctypes.c_uint64(off), ctypes.byref(ptr)))
                peers.append(ptr.value)
                self._imported.append(ptr.value)
        return peers

    def input_buffer(self):
        """Pull: the registered input shard -- write this rank's input here
        and pass it to the call (no copy).  Push: None (any tensor works)."""
        return self.input

    def _barrier(self):
        import torch
        import torch.distributed as dist

        if self.G == 1:
            return
        if self.backend == "nccl":
            dist.all_reduce(self._flag, group=self.group)        # device-side, stream-ordered
        else:
            torch.cuda.current_stream(self.device).synchronize()
            dist.barrier(group=self.group)

    def __call__(self, local_in, stream=None, out=None):
        import torch

        from .api import launch_sharded, launch_sharded_pull, launch_sharded_sync

        if local_in.numel() != self.local_numel or local_in.dtype != self.dtype:
            raise LayoutError(f"rank {self.rank}: expected {self.local_numel} elements of {self.dtype}")
        if local_in.device != self.device or not local_in.is_contiguous():
            raise LayoutError("input shard must be a contiguous tensor on the exchange's device")
        st = stream or torch.cuda.current_stream(self.device)
        with torch.cuda.stream(st):
            if self.mode == "pull":
                if out is None:
                    out = torch.empty(self.local_numel, dtype=self.dtype, device=self.device)
                elif out.numel() != self.local_numel or out.dtype != self.dtype or not out.is_contiguous():
                    raise LayoutError("out must be a contiguous tensor of the local output shard")
                if local_in.data_ptr() != self.input.data_ptr():
                    self.input.copy_(local_in.reshape(-1))     # not the registered buffer: stage it
                if self._sync is not None:
                    self._sync.epoch = self.calls + 1          # same on every rank
                    launch_sharded_sync(self.program, self.peers, [out.data_ptr()], self._sync,
                                        ctypes.c_void_p(st.cuda_stream))
                else:
                    self._barrier()           # every input shard complete
                    launch_sharded_pull(self.program, self.peers, out.data_ptr(), ctypes.c_void_p(st.cuda_stream))
                    self._barrier()           # every reader done before inputs change
                res = out
            else:
                i = self.calls % 2        # alternate registered outputs
                if self._sync is not None:
                    self._sync.epoch = self.calls + 1
                    launch_sharded_sync(self.program, [local_in.data_ptr()], self.peer_tables[i], self._sync,
                                        ctypes.c_void_p(st.cuda_stream))
                else:
                    self._barrier()
                    launch_sharded(self.program, local_in.data_ptr(), self.peer_tables[i],
                                   ctypes.c_void_p(st.cuda_stream))
                    self._barrier()
                res = self._outs[i]
                if self.copy_out or out is not None:
                    res = (out.reshape(-1) if out is not None else torch.empty_like(res)).copy_(res)
        self.calls += 1
        return res.view(self.splan.local_out_shape())

    def close(self):
        from . import _lib

        L = _lib.lib()
        for p in self._imported:
            L.vpg_ipc_release(ctypes.c_void_p(p))
        self._imported = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _check_ipc(status):
    from . import _lib

    if status != _lib.VPG_OK:
        raise RuntimeError(f"CUDA IPC: {_lib.last_error()}")


_exchanges: dict = {}


def release_exchanges():
    """Drop the cached ShardExchange objects of permute_sharded(method=
    "fused"/"auto") and their peer mappings and output buffers.  Collective
    in effect: call it on every rank."""
    for ex in list(_exchanges.values()):
        ex.close()
    _exchanges.clear()


def _exchange_for(shape, axes, dtype, device, group):
    key = (shape, axes, dtype, str(device), id(group))
    ex = _exchanges.get(key)
    if ex is None:
        ex = _exchanges[key] = ShardExchange(shape, axes, dtype, group=group, device=device)
    return ex


def exchange_input(global_shape, axes, dtype, group=None, device=None):
    """The tensor to produce this rank's input shard in for
    permute_sharded(method="fused"/"auto"): the cached pull exchange's
    registered input buffer (the call then launches one kernel and copies
    nothing), else a fresh tensor (push exchange and the all-to-all path
    take any input)."""
    import torch
    import torch.distributed as dist

    G = dist.get_world_size(group) if dist.is_initialized() else 1
    device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    es = torch.empty((), dtype=dtype).element_size()
    if fused_supported(global_shape, axes, es, G):
        ex = _exchange_for(tuple(global_shape), tuple(axes), dtype, device, group)
        if ex.input is not None:
            return ex.input
    return torch.empty(plan_sharded(global_shape, axes, G).local_numel, dtype=dtype, device=device)


def emulate_fused(x_flat, global_shape, axes, G, jit=None, mode="push", in_shards=None, device_barrier=False):
    """Run the G exchange kernels of the fused path on ONE device (virtual
    ranks, every shard a local buffer).  mode "push": rank r reads input
    shard r and stores into every output shard; "pull": rank r reads every
    input shard (``in_shards``, default the slices of x_flat) and writes
    output shard r.  ``device_barrier``: all ranks in ONE cooperative launch
    ordered by the device-side exchange barrier (flag blocks, epochs) that
    multi-GPU jobs use -- co-resident by construction, so no flag wait can
    starve another rank; otherwise G independent launches.  Returns the
    list of per-rank output shards (flat)."""
    import torch

    from .api import launch_sharded, launch_sharded_emulated, launch_sharded_pull

    n = x_flat.numel()
    progs = _programs(global_shape, axes, x_flat.element_size(), G, range(G), jit=jit, pull=mode == "pull")
    outs = [torch.empty(n // G, dtype=x_flat.dtype, device=x_flat.device) for _ in range(G)]
    ptrs = [o.data_ptr() for o in outs]
    st = torch.cuda.current_stream(x_flat.device)
    if in_shards is None:
        in_shards = [x_flat[slice(*shard_bounds(n, G, r))] for r in range(G)]
    srcs = [t.data_ptr() for t in in_shards]
    if device_barrier:
        launch_sharded_emulated(progs, srcs, ptrs, ctypes.c_void_p(st.cuda_stream))
        return outs
    for r in range(G):
        if mode == "pull":
            launch_sharded_pull(progs[r], srcs, ptrs[r], ctypes.c_void_p(st.cuda_stream))
        else:
            launch_sharded(progs[r], srcs[r], ptrs, ctypes.c_void_p(st.cuda_stream))
    return outs
