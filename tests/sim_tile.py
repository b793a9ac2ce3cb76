"""TEST INFRASTRUCTURE -- host simulation of the tile kernel's address walk.

The reference validates every generated program on a guard-banded VM
before hardware runs it (/root/reference/pkg/src/vecperm/vm.py:28-33,
113-226).  This is the same idea for the GPU plan: it decodes the kernel
parameter block of a TILE plan (``vpg_plan_tile_params``) and replays the
walk of csrc/tile_body.cuh -- tile decode, thread parts, inner/outer dims,
slot predicates, shifted-run reads, vector accesses -- in numpy, checking
that every shared-memory and global access is in bounds and aligned and
that the data lands where the permutation says.  It needs no GPU, so the
CPU suite can exercise the planner on thousands of shapes.

It is never used by the product (which has no CPU path).
"""

from __future__ import annotations

import ctypes

import numpy as np

from paper_2506_03686_b200 import _lib

MAXR, MAXPD = 40, 12


class FastDiv(ctypes.Structure):
    _fields_ = [("d", ctypes.c_uint32), ("m", ctypes.c_uint32), ("s", ctypes.c_uint32)]


class PhaseDim(ctypes.Structure):
    _fields_ = [("gstride", ctypes.c_int64), ("div", FastDiv), ("sstride", ctypes.c_uint32),
                ("slot", ctypes.c_int16), ("cmul", ctypes.c_uint16), ("hmul", ctypes.c_uint16),
                ("pad_", ctypes.c_uint16)]


class PhaseDesc(ctypes.Structure):
    _fields_ = [("nthr", ctypes.c_uint32), ("ngroups", ctypes.c_uint32), ("nthr_dims", ctypes.c_int32),
                ("thr", PhaseDim * MAXPD), ("n_in", ctypes.c_uint32), ("g_in", ctypes.c_int64),
                ("s_in", ctypes.c_uint32), ("c_in", ctypes.c_uint32 * 3), ("n_outer", ctypes.c_uint32),
                ("nout_dims", ctypes.c_int32), ("out", PhaseDim * MAXPD), ("vec", ctypes.c_uint32),
                ("rshift", ctypes.c_uint32), ("h_in", ctypes.c_uint32), ("vstride", ctypes.c_int64),
                ("mask_full", ctypes.c_uint32), ("mask_ragged", ctypes.c_uint32), ("off_tab", ctypes.c_uint32),
                ("swz", ctypes.c_uint32), ("spitch", FastDiv), ("w2", ctypes.c_uint32), ("vrow", ctypes.c_uint32)]


class GridDigit(ctypes.Structure):
    _fields_ = [("cum", FastDiv), ("ext", FastDiv), ("src_stride", ctypes.c_int64), ("dst_stride", ctypes.c_int64)]


MAXLIN = 8


class LinDesc(ctypes.Structure):
    _fields_ = [("on", ctypes.c_uint32), ("nt", ctypes.c_uint32), ("run_len", ctypes.c_uint32),
                ("cpr", ctypes.c_uint32), ("cprd", FastDiv), ("nchunks", ctypes.c_uint32),
                ("nrd", ctypes.c_int32), ("nxd", ctypes.c_int32), ("last_slot", ctypes.c_int32),
                ("last_unit", ctypes.c_uint32), ("tab_off", ctypes.c_uint32), ("rot_shift", ctypes.c_uint32),
                ("rd", PhaseDim * MAXLIN), ("xd", PhaseDim * MAXPD)]


class TileParams(ctypes.Structure):
    _fields_ = [("n_elems", ctypes.c_int64), ("num_tiles", ctypes.c_uint32), ("ngrid", ctypes.c_int32),
                ("Ls", ctypes.c_uint32), ("Ld", ctypes.c_uint32), ("T", ctypes.c_uint32),
                ("pitch", ctypes.c_uint32), ("tile_elems_alloc", ctypes.c_uint32),
                ("grid_a", ctypes.c_int32), ("grid_c", ctypes.c_int32),
                ("e_a", ctypes.c_uint32), ("d_a", ctypes.c_uint32), ("e_c", ctypes.c_uint32),
                ("d_c", ctypes.c_uint32), ("lim_split", ctypes.c_uint32 * 2), ("hmask", ctypes.c_uint32),
                ("bulk", ctypes.c_uint32), ("nruns", ctypes.c_uint32), ("nrdims", ctypes.c_int32),
                ("run_bytes", ctypes.c_uint32), ("run_unit_bytes", ctypes.c_uint32),
                ("rdims", PhaseDim * MAXPD),
                ("ph", PhaseDesc * 2), ("grid", GridDigit * MAXR), ("off_buf", ctypes.c_uint32),
                ("nbuf", ctypes.c_uint32), ("persistent", ctypes.c_uint32), ("smem_bytes", ctypes.c_uint32),
                ("nshards", ctypes.c_uint32), ("tile_begin", ctypes.c_uint32), ("src_bias", ctypes.c_int64),
                ("shard_elems", ctypes.c_int64), ("rres", ctypes.c_uint32), ("pull", ctypes.c_uint32),
                ("shard_shift", ctypes.c_uint32), ("shard_div", FastDiv), ("pad_pull_", ctypes.c_uint32),
                ("dst_bias", ctypes.c_int64), ("src_span", ctypes.c_int64), ("lin", LinDesc)]


def tile_params(program) -> TileParams:
    L = _lib.lib()
    need = ctypes.c_size_t(0)
    L.vpg_plan_tile_params(program.handle, None, 0, ctypes.byref(need))
    assert need.value == ctypes.sizeof(TileParams), (need.value, ctypes.sizeof(TileParams))
    tp = TileParams()
    st = L.vpg_plan_tile_params(program.handle, ctypes.byref(tp), ctypes.sizeof(tp), None)
    assert st == 0, _lib.last_error()
    return tp


class SimError(AssertionError):
    pass


def _decode(idx, dims, n):
    """Mixed-radix decode of an index array over `n` PhaseDims -> (g, s, c0, c1, c2, h)."""
    idx = np.asarray(idx, dtype=np.int64).copy()
    g = np.zeros_like(idx)
    s = np.zeros_like(idx)
    c = [np.zeros_like(idx) for _ in range(3)]
    h = np.zeros_like(idx)
    for i in range(n):
        d = dims[i]
        ext = d.div.d
        dig = idx % ext
        idx //= ext
        g += dig * d.gstride
        s += dig * d.sstride
        h += dig * d.hmul
        if d.slot >= 0:
            c[d.slot] = dig * d.cmul
    return g, s, c, h


def check_layout(tp: TileParams, E: int) -> None:
    """Shared-memory regions (two outer tables, pipeline buffers) are disjoint
    and inside the dynamic allocation."""
    ENTRY = 24
    t0 = (tp.ph[0].off_tab, tp.ph[0].off_tab + ENTRY * tp.ph[0].n_outer)
    t1 = (tp.ph[1].off_tab, tp.ph[1].off_tab + ENTRY * tp.ph[1].n_outer)
    buf = ((tp.tile_elems_alloc * E + 15) // 16) * 16
    b = (tp.off_buf, tp.off_buf + buf * tp.nbuf)
    regs = [t0, t1, b]
    if tp.lin.on:
        V = 16 // E
        regs.append((tp.lin.tab_off, tp.lin.tab_off + V * tp.lin.cpr * V * 2))
        if tp.lin.tab_off % 16:
            raise SimError("lin offset table misaligned")
    regs = sorted(regs)
    for (a0, a1), (b0, b1) in zip(regs, regs[1:]):
        if a1 > b0 and a1 > a0 and b1 > b0:
            raise SimError(f"smem regions overlap: {regs}")
    if max(r[1] for r in regs) > tp.smem_bytes or tp.off_buf % 16:
        raise SimError(f"buffers exceed smem_bytes or misaligned: {b} vs {tp.smem_bytes}")
    if tp.smem_bytes > 227 * 1024:
        raise SimError("more dynamic smem than a CTA can have")


def simulate(program, src_words: np.ndarray, threads: int | None = None, shard_out=None, tp=None):
    """Replay the tile kernel on host words; returns the destination words.

    Sharded exchange plans: ``src_words`` is the plan's input shard and
    ``shard_out = (dsts, counts)`` holds every output shard and its
    per-element write counters, updated in place (the caller checks the
    coverage after replaying every rank).  ``tp`` replaces the plan's
    parameter block (negative controls)."""
    tp = tp if tp is not None else tile_params(program)
    check_layout(tp, program.layout.elem_width)
    E = program.layout.elem_width
    NT = threads or program.metadata["threads"]
    n = tp.n_elems
    assert src_words.size == n
    sharded = shard_out is not None
    if sharded:
        dsts, counts = shard_out
        assert len(dsts) == tp.nshards and all(d.size == tp.shard_elems for d in dsts)
    else:
        dst = np.full(n, np.iinfo(np.uint64).max if src_words.dtype == np.uint64 else 0, dtype=src_words.dtype)
        written = np.zeros(n, dtype=np.int32)
    alloc = tp.tile_elems_alloc
    tid = np.arange(NT, dtype=np.int64)
    parts = []
    for ph in range(2):
        d = tp.ph[ph]
        grp = tid // d.nthr
        tr = tid - grp * d.nthr
        active = grp < d.ngroups
        g, s, c, h = _decode(tr, d.thr, d.nthr_dims)
        parts.append((d, grp, active, g, s, c, h))
    for t in range(tp.num_tiles):
        # tile decode (decode_tile)
        sb = db = 0
        va, vc = tp.e_a, tp.e_c
        tg_ = t + tp.tile_begin
        for i in range(tp.ngrid):
            gd = tp.grid[i]
            cdig = (tg_ // gd.cum.d) % gd.ext.d
            sb += cdig * gd.src_stride
            db += cdig * gd.dst_stride
            if i == tp.grid_a:
                va = min(tp.e_a, tp.d_a - cdig * tp.e_a)
            if i == tp.grid_c:
                vc = min(tp.e_c, tp.d_c - cdig * tp.e_c)
        if sharded and tp.pull:
            # pull exchange: global source offsets, local output shard
            q = tp.dst_bias // tp.shard_elems
            db -= tp.dst_bias
            if not 0 <= db < tp.shard_elems:
                raise SimError(f"pull tile {t} outside the plan's output shard")
            dst, written = dsts[q], counts[q]
            dbound = tp.shard_elems
        elif sharded:
            q = db // tp.shard_elems
            sb -= tp.src_bias
            db -= q * tp.shard_elems
            dst, written = dsts[q], counts[q]
            dbound = tp.shard_elems
        else:
            dbound = n
        full = va == tp.e_a and vc == tp.e_c
        lim = (va, vc)
        tbase = (sb & tp.rres) if tp.rres else 0     # residue mode: tile offset in its buffer
        smem = np.zeros(alloc + 64, dtype=src_words.dtype)
        smem_valid = np.zeros(alloc + 64, dtype=bool)
        if tp.bulk:
            # R as one bulk copy per source run (producer warp); misaligned
            # runs (rshift 2): the 16-byte aligned superset of each run into
            # residue rows, the part in the buffer's last partial chunk copied
            # element by element
            rbytes = tp.run_bytes if va == tp.e_a else tp.run_unit_bytes * va
            mis = tp.ph[0].rshift == 2
            if not mis and (rbytes % 16 or tp.run_bytes % 16):
                raise SimError("bulk copy size not a multiple of 16 bytes")
            nel = rbytes // E
            V = 16 // E
            claimed = np.zeros(alloc + 64, dtype=bool)      # superset rows of distinct runs must not overlap
            for r in range(tp.nruns):
                g_, s_, c_, _ = _decode([r], tp.rdims, tp.nrdims)
                if tp.grid_c >= 0 and c_[1][0] >= vc:
                    continue
                ga, sa = sb + g_[0], s_[0] + tbase
                if mis:
                    g0 = ga
                    ga = g0 - g0 % V
                    ge = min(-(-(g0 + nel) // V) * V, n - n % V)
                    ge = max(ge, ga)
                    if (sa - (g0 - ga)) % V or sa % V != g0 % V:
                        raise SimError("bulk residue: smem run start not congruent to its source mod 16 bytes")
                    s0 = sa - (g0 - ga)
                    hi = s0 + max(ge - ga, g0 + nel - ga)
                    if claimed[s0:hi].any():
                        raise SimError("bulk residue: aligned supersets of two runs overlap in smem")
                    claimed[s0:hi] = True
                    if ge > ga:
                        _chk(np.array([ga, ge - 1]), n, "bulk global")
                        _chk(np.array([s0, s0 + (ge - ga) - 1]), alloc, "bulk smem")
                        smem[s0:s0 + ge - ga] = src_words[ga:ge]
                        smem_valid[s0:s0 + ge - ga] = True
                    for e in range(max(ge, g0), g0 + nel):
                        _chk(np.array([e]), n, "bulk tail global")
                        smem[sa + e - g0] = src_words[e]
                        smem_valid[sa + e - g0] = True
                    continue
                if (ga * E) % 16 or (sa * E) % 16:
                    raise SimError("bulk copy address not 16-byte aligned")
                _chk(np.array([ga, ga + nel - 1]), n, "bulk global")
                _chk(np.array([sa, sa + nel - 1]), alloc, "bulk smem")
                smem[sa:sa + nel] = src_words[ga:ga + nel]
                smem_valid[sa:sa + nel] = True
        for ph in range(2):
            if ph == 0 and tp.bulk:
                continue
            if ph == 1 and tp.lin.on:
                _lin_write(tp, E, db, smem, smem_valid, tbase, dst, written, dbound, full, lim, t)
                continue
            d, grp, active, tg, ts, tc, th = parts[ph]
            mask = d.mask_full if full else d.mask_ragged
            V = d.vec
            for o_start in range(d.ngroups):
                sel = active & (grp == o_start)
                if not sel.any():
                    continue
                for o in range(o_start, d.n_outer, d.ngroups):
                    eg, es, ec, eh = _decode([o], d.out, d.nout_dims)
                    for i in range(d.n_in):
                        gp = tg[sel] + eg[0] + i * d.g_in
                        sp = ts[sel] + es[0] + i * d.s_in
                        c0 = tc[0][sel] + ec[0][0] + i * d.c_in[0]
                        c1 = tc[1][sel] + ec[1][0] + i * d.c_in[1]
                        c2 = tc[2][sel] + i * d.c_in[2]
                        ok = np.ones(gp.shape, dtype=bool)
                        if mask & 1:
                            ok &= c0 < lim[0]
                        if mask & 2:
                            ok &= c1 < lim[1]
                        if mask & 4:
                            ok &= c2 < tp.lim_split[ph]
                        gp, sp = gp[ok], sp[ok]
                        if ph == 0:
                            gabs = sb + gp
                            if tp.pull and V > 1:
                                S = tp.shard_elems
                                ga0 = gabs - (gabs % V)
                                if ((ga0 // S) != ((ga0 + V - 1) // S)).any():
                                    raise SimError("pull: 16-byte chunk straddles two input shards")
                            if d.rshift:
                                ga = gabs - (gabs % V)
                                if d.swz and d.rshift == 1 and (sp % V).any():
                                    raise SimError("swizzled R chunk not chunk-aligned")
                                if d.rshift == 2:
                                    spl = sp + tbase
                                    sd = spl - (spl % V)
                                    if ((spl - sd) != (gabs - ga)).any():
                                        raise SimError("residue mode: smem and global offsets differ mod V")
                                    M = tp.rres + 1          # residue modulus (elements)
                                    if ((spl - gabs) % M).any():
                                        raise SimError("residue mode: smem and global offsets differ mod the residue modulus")
                                    if d.swz == 16:          # address swizzle of the aligned chunk
                                        sd = _swizzle(d, sd, V)
                                else:
                                    sd = _swizzle(d, sp, V)
                                for j in range(V):
                                    inb = ga + j < n
                                    _chk(sd[inb] + j, alloc, "R shifted smem")
                                    smem[sd[inb] + j] = src_words[ga[inb] + j]
                                    smem_valid[sd[inb] + j] = True
                            else:
                                if V > 1 and ((gabs % V).any() or (sp % V).any()):
                                    raise SimError("R vector access misaligned")
                                # chunk swizzle (128-byte congruent layout): V-element
                                # vectors stay contiguous, scalar words move one by one
                                spx = _swizzle(d, sp, 16 // E if E <= 16 else 1)
                                # (the logical slot is congruent to the source mod 128 B;
                                # the swizzle only permutes chunks inside a 128-byte block)
                                if (d.swz and not tp.pull and V > 1 and _congruent(tp, E)
                                        and ((sp * E) % 128 != (gabs * E) % 128).any()):
                                    raise SimError("congruent layout: smem and global offsets differ mod 128 B")
                                if d.swz and ((spx * E) // 128 != (sp * E) // 128).any():
                                    raise SimError("chunk swizzle left its 128-byte block")
                                for j in range(V):
                                    _chk(gabs + j, n, "R global")
                                    _chk(spx + j, alloc, "R smem")
                                    smem[spx + j] = src_words[gabs + j]
                                    smem_valid[spx + j] = True
                        else:
                            if d.w2 >= 64:
                                # gather block: G destination-innermost elements from G smem
                                # rows vrow apart -> one store of G words (w2 == 64: G = V,
                                # 16 bytes; narrow blocks: G = w2 - 64 = 2, 4, 8)
                                Vg = 16 // E if d.w2 == 64 else d.w2 - 64
                                gabs = db + gp
                                if (gabs % Vg).any():
                                    raise SimError("W gather block store misaligned")
                                for j in range(Vg):
                                    spx = _swizzle(d, sp + tbase + j * d.vrow, 16 // E)
                                    _chk(spx, alloc, "Wg smem")
                                    dd = gabs + j
                                    _chk(dd, dbound, "Wg global")
                                    if not smem_valid[spx].all():
                                        raise SimError(f"W reads smem never written (tile {t})")
                                    dst[dd] = smem[spx]
                                    written[dd] += 1
                                continue
                            if d.w2 >= 2:
                                # k x V interleave block: k smem vectors (one per value of
                                # the destination-innermost dim, rows vrow apart) -> k*V
                                # consecutive destination elements, k 16-byte stores
                                K = d.w2
                                gabs = db + gp
                                if (gabs % V).any():
                                    raise SimError("W interleave block store misaligned")
                                for c in range(K):
                                    spx = _swizzle(d, sp + tbase + c * d.vrow, 16 // E)
                                    if (spx % V).any():
                                        raise SimError("W interleave smem vector misaligned")
                                    for w in range(V):
                                        so = spx + w
                                        _chk(so, alloc, "Wk smem")
                                        dd = gabs + w * K + c
                                        _chk(dd, dbound, "Wk global")
                                        if not smem_valid[so].all():
                                            raise SimError(f"W reads smem never written (tile {t})")
                                        dst[dd] = smem[so]
                                        written[dd] += 1
                                continue
                            if d.w2:
                                # V x V block: V smem vectors from rows vrow apart (same
                                # swizzle row group) -> V 16-byte stores of V consecutive
                                # destination elements
                                gabs = db + gp
                                spx = _swizzle(d, sp + tbase, 16 // E)
                                if (spx % V).any() or (d.vrow % V) or (gabs % V).any() or (d.vstride % V):
                                    raise SimError("W 2-D block access misaligned")
                                for ii in range(V):
                                    if (_swizzle(d, sp + tbase + ii * d.vrow, 16 // E) != spx + ii * d.vrow).any():
                                        raise SimError("W 2-D block rows do not share a swizzle group")
                                    for j in range(V):
                                        so = spx + ii * d.vrow + j
                                        _chk(so, alloc, "W2 smem")
                                        dd = gabs + j * d.vstride + ii
                                        _chk(dd, dbound, "W2 global")
                                        if not smem_valid[so].all():
                                            raise SimError(f"W reads smem never written (tile {t})")
                                        dst[dd] = smem[so]
                                        written[dd] += 1
                                continue
                            hh = (sb + th[sel][ok] + eh[0] + i * d.h_in) & tp.hmask if tp.hmask else 0
                            spx = _swizzle(d, sp + hh + tbase, 16 // E if E <= 16 else 1)
                            gabs = db + gp
                            if V > 1 and (spx % V).any():
                                raise SimError("W vector smem access misaligned")
                            if V > 1 and d.vstride == 1 and ((db + gp) % V).any():
                                raise SimError("W 16-byte destination chunk misaligned")
                            for j in range(V):
                                _chk(spx + j, alloc, "W smem")
                                dd = gabs + j * d.vstride
                                _chk(dd, dbound, "W global")
                                if not smem_valid[spx + j].all():
                                    raise SimError(f"W reads smem never written (tile {t})")
                                dst[dd] = smem[spx + j]
                                written[dd] += 1
    if sharded:
        return dsts
    if (written != 1).any():
        bad = np.nonzero(written != 1)[0][:5]
        raise SimError(f"destination elements written {written[bad]} times at {bad}")
    return dst


def simulate_exchange(programs, src_words: np.ndarray) -> np.ndarray:
    """Replay every rank's exchange kernel (push: rank r reads input shard r;
    pull: rank r reads the whole input through the shard table and writes
    output shard r); returns the concatenated output shards after checking
    that each output element was written exactly once."""
    tp0 = tile_params(programs[0])
    G, S = tp0.nshards, tp0.shard_elems
    fill = np.iinfo(np.uint64).max if src_words.dtype == np.uint64 else 0
    dsts = [np.full(S, fill, dtype=src_words.dtype) for _ in range(G)]
    counts = [np.zeros(S, dtype=np.int32) for _ in range(G)]
    for r, prog in enumerate(programs):
        words = src_words if tp0.pull else src_words[r * S:(r + 1) * S]
        simulate(prog, words, shard_out=(dsts, counts))
    c = np.concatenate(counts)
    if (c != 1).any():
        bad = np.nonzero(c != 1)[0][:5]
        raise SimError(f"destination elements written {c[bad]} times at {bad}")
    return np.concatenate(dsts)


def _lin_offsets(L, j):
    """smem offsets of destination-run positions j (the kernel's table entries)."""
    j = np.asarray(j, dtype=np.int64).copy()
    off = np.zeros_like(j)
    for k in range(L.nrd):
        e = L.rd[k].div.d
        off += (j % e) * L.rd[k].sstride
        j //= e
    return off


def _lin_write(tp, E, db, smem, smem_valid, tbase, dst, written, dbound, full, lim, t):
    """W phase in lin mode (tile_write_lin): chunk slots over runs, each the
    16-byte aligned destination chunk holding run positions c*V - m ..
    c*V - m + V-1 (m = the run start's word offset in its chunk; destination
    buffers are 16-byte aligned)."""
    L = tp.lin
    V = 16 // E
    d = tp.ph[1]
    if L.cpr != (L.run_len + V - 2) // V + 1 or L.nchunks % L.cpr:
        raise SimError("lin: chunk slot count does not cover every alignment")
    Lv = L.run_len
    if not full and L.last_slot >= 0:
        Lv = L.last_unit * lim[L.last_slot]
    q = np.arange(L.nchunks, dtype=np.int64)
    r, c = q // L.cpr, q % L.cpr
    go, so, cs, _ = _decode(r, L.xd, L.nxd)
    live = np.ones(q.shape, dtype=bool)
    if not full:
        for i in range(L.nxd):
            if L.xd[i].slot >= 0:
                live &= cs[L.xd[i].slot] < lim[L.xd[i].slot]
    rp = db + go
    m = rp % V
    j0 = c * V - m
    for e in range(V):
        j = j0 + e
        ok = live & (j >= 0) & (j < Lv)
        if not ok.any():
            continue
        if (j[ok] >= L.run_len).any():
            raise SimError("lin: position beyond the destination run")
        sp = so[ok] + _lin_offsets(L, j[ok]) + tbase
        if (_lin_offsets(L, j[ok]) >= 65536).any():
            raise SimError("lin: smem offset does not fit the u16 table")
        spx = _swizzle(d, sp, 16 // E)
        _chk(spx, smem.size - 64, "W lin smem")
        dd = rp[ok] + j[ok]
        _chk(dd, dbound, "W lin global")
        if ((rp[ok] + j0[ok]) % V).any():
            raise SimError("lin: chunk store not 16-byte aligned")
        if not smem_valid[spx].all():
            raise SimError(f"W lin reads smem never written (tile {t})")
        dst[dd] = smem[spx]
        written[dd] += 1


def _congruent(tp, E):
    """The swizzled unpadded layout keeps runs at their source lines' offset
    mod 128 B only when every stride that moves a run start (grid digits,
    R-phase dims at or above the run) is a multiple of 128 bytes; the planner
    also uses the layout without that congruence (planner.cpp
    sw128_layout_ok vs sw128_possible)."""
    q = 128 // E
    d = tp.ph[0]
    dims = [d.thr[i] for i in range(d.nthr_dims)] + [d.out[i] for i in range(d.nout_dims)]
    if any(tp.grid[i].src_stride % q for i in range(tp.ngrid)):
        return False
    if d.n_in > 1 and d.g_in >= tp.Ls and d.g_in % q:
        return False
    return not any(x.gstride >= tp.Ls and x.gstride % q for x in dims)


def _swizzle(d, s, V):
    """Chunk swizzle of smem element offsets (tile_body.cuh swizzle<V>)."""
    if not d.swz:
        return s
    if d.swz == 16:                       # kSwzAddr: chunk ^= 128-byte block index
        lv = {1: 0, 2: 1, 4: 2, 8: 3, 16: 4}[V]
        return s ^ (((s >> (lv + 3)) & 7) << lv)
    P = d.spitch.d
    r = s // P
    c = s - r * P
    f = (r >> (d.swz - 1)) & 7
    return r * P + (((c // V) ^ f) * V) + (c % V)


def _chk(idx, bound, what):
    if idx.size and (idx.min() < 0 or idx.max() >= bound):
        raise SimError(f"{what} out of bounds: [{idx.min()}, {idx.max()}] vs {bound}")
