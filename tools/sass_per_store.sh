#!/bin/bash
# Static SASS of a plan's specialised kernel, compiled offline with NVRTC (no
# GPU): instruction, STG, LDS, branch-region and spill counts, and the
# instructions per store in the middle of the W walk.
#   tools/sass_per_store.sh "SHAPE" "AXES" ELEM_BYTES [candidate]
# Environment knobs of the planner / jit.cpp apply (VPG_TILE_BUDGET, VPG_W_U,
# VPG_SMEM_DECL, VPG_LIB_PATH ...).
here=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
VPG_JIT_DUMP=$tmp/k.cubin PYTHONPATH=$here python "$here/tools/jit_offline.py" "$tmp/cache" "$1" "$2" "$3" $4 > "$tmp/plan.txt" 2>&1 || { tail -3 "$tmp/plan.txt"; exit 1; }
grep -o "phase W[^']*" "$tmp/plan.txt" | head -1
cuobjdump -sass "$tmp/k.cubin" > "$tmp/k.sass"
python - "$tmp/k.sass" <<'PY'
import collections, re, sys
ins = [l.split('*/')[1].strip() for l in open(sys.argv[1]) if re.search(r'/\*[0-9a-f]{4,5}\*/\s+\S', l)]
def op(l):
    t = l.split()
    return (t[1] if t[0].startswith('@') else t[0]).split('.')[0]
ops = [op(l) for l in ins]
idx = [i for i, o in enumerate(ops) if o == 'STG']
c = collections.Counter(ops)
print(f"instructions {len(ops)}  STG {c['STG']}  LDS {c['LDS']}  BSSY {c['BSSY']}  LDL {c['LDL']}  STL {c['STL']}")
if len(idx) > 20:
    a, b = idx[len(idx) // 4], idx[3 * len(idx) // 4]
    k = 3 * len(idx) // 4 - len(idx) // 4
    print(f"middle of the W walk: {(b - a) / k:.1f} instructions per STG", collections.Counter(ops[a:b]).most_common(8))
PY
cuobjdump -res-usage "$tmp/k.cubin" 2>/dev/null | grep -o "REG:[0-9]*\|STACK:[0-9]*" | tr '\n' ' '; echo
rm -rf "$tmp"
