"""TEST INFRASTRUCTURE ONLY -- build the reference's own CPU kernels into oracle/_ref/.

The reference (``vecperm``, pure Python) generates its CPU hot path as C
source at run time: ``build_program`` -> ``emit_source`` -> gcc
(/root/reference/pkg/src/vecperm/ir.py:441-456, emit.py:212-340,
emit.py:418-441).  This script runs that generator IN THIS CONTAINER (where
/root/reference exists, read-only) for every BASELINE configuration and
compiles the emitted kernels as shared objects with the reference's own
flags (``-O2 -mavx512f``, emit.py:433; ``-O2`` for the scalar target,
emit.py:424) plus ``-shared -fPIC``.

Outputs go to ``oracle/_ref/`` only (git-ignored, but shipped to the GPU box
by gpurun): ``<cfg>_<target>.c``, ``lib<cfg>_<target>.so`` and
``manifest.json``.  Nothing here copies reference sources into the repo; the
C text is the reference's *output* for these shapes.

Usage:  python oracle/build_ref.py [--configs cfg1,cfg2,...]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
REF_SRC = "/root/reference/pkg/src"
OUT = os.path.join(HERE, "_ref")
GCC = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"


def _import_reference():
    if not os.path.isdir(REF_SRC):
        raise RuntimeError(f"reference not present at {REF_SRC}")
    sys.dont_write_bytecode = True          # /root/reference is read-only
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import vecperm  # noqa: F401
    return vecperm


def build(configs=None, targets=("x86-avx", "scalar"), quiet=False) -> dict:
    vp = _import_reference()
    from vecperm.core import TensorLayout, from_numpy_convention
    from vecperm.emit import emit_source, kernel_name
    from vecperm.ir import build_program
    from vecperm.machine import MachineConfig

    sys.path.insert(0, REPO)
    from paper_2506_03686_b200.workloads import CONFIGS

    os.makedirs(OUT, exist_ok=True)
    manifest_path = os.path.join(OUT, "manifest.json")
    manifest = {}
    if os.path.exists(manifest_path):
        with open(manifest_path) as f:
            manifest = json.load(f)
    for key, wl in CONFIGS.items():
        if configs and key not in configs:
            continue
        elem = wl.elem_bytes                      # complex64 -> one 8-byte word
        layout = TensorLayout(tuple(reversed(wl.shape)), elem)
        pmap = from_numpy_convention(wl.axes)
        machine = MachineConfig("x86-avx", 512, elem, 32)
        ir = build_program(layout, pmap, machine)
        entry = {
            "shape": list(wl.shape),
            "axes": list(wl.axes),
            "dtype": wl.dtype,
            "elem_bytes": elem,
            "dims_inner_first": list(layout.dims),
            "sigma_inner_first": list(pmap.sigma),
            "slack_bytes": machine.lanes * elem,            # emit.py:470
            "plan": {k: str(v) for k, v in ir.metadata.items()},
            "reference_version": getattr(vp, "__version__", "?"),
            "targets": {},
        }
        for target in targets:
            src = emit_source(ir, target=target)
            sym = kernel_name(ir.layout, ir.pmap, machine)
            cpath = os.path.join(OUT, f"{key}_{target}.c")
            sopath = os.path.join(OUT, f"lib{key}_{target}.so")
            with open(cpath, "w") as f:
                f.write(src)
            flags = ["-O2", "-mavx512f"] if target == "x86-avx" else ["-O2"]
            cmd = [GCC, *flags, "-shared", "-fPIC", cpath, "-o", sopath]
            subprocess.run(cmd, check=True)
            entry["targets"][target] = {
                "so": os.path.basename(sopath),
                "symbol": sym,
                "cflags": flags,
            }
            if not quiet:
                print(f"[build_ref] {key} {target}: {sym} -> {os.path.relpath(sopath, REPO)}")
        manifest[key] = entry
    with open(manifest_path, "w") as f:
        json.dump(manifest, f, indent=1)
    return manifest


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="")
    args = ap.parse_args(argv)
    cfgs = [c for c in args.configs.split(",") if c]
    build(cfgs or None)


if __name__ == "__main__":
    main()
