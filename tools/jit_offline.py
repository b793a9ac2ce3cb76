"""Compile one plan's specialised kernel offline (NVRTC, no GPU):
    python tools/jit_offline.py CACHE_DIR "SHAPE" "AXES" ELEM_BYTES [candidate]
VPG_JIT_DUMP=<file> keeps the cubin (tools/sass_per_store.sh)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
cache = sys.argv[1]
os.environ["VPG_JIT_CACHE"] = cache
os.makedirs(cache, exist_ok=True)
import ast
import paper_2506_03686_b200 as vp
shape, axes, E = ast.literal_eval(sys.argv[2]), ast.literal_eval(sys.argv[3]), int(sys.argv[4])
k = int(sys.argv[5]) if len(sys.argv) > 5 else None
p = vp.build_program(vp.TensorLayout.from_shape(shape, E), vp.from_numpy_convention(axes), **({} if k is None else {"candidate": k}))
t=time.time(); vp.jit_compile(p); print("compile s", time.time()-t)
print([l for l in p.text.splitlines() if l.startswith(("phase","tile el","smem"))])
