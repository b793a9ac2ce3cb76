# usage: cnt2.sh libpath "shape" "axes" E
VPG_LIB_PATH=$1 VPG_JIT_DUMP=/tmp/ky.cubin PYTHONPATH=/root/repo python /root/repo/tools/jit_offline.py /tmp/jcy "$2" "$3" $4 > /tmp/ky.txt 2>&1 || { tail -3 /tmp/ky.txt; exit 1; }
grep -o "phase W.*" /tmp/ky.txt | head -1 | cut -c1-120
cuobjdump -sass /tmp/ky.cubin > /tmp/ky.sass
python - <<'PY'
import re,collections
ins=[l.split('*/')[1].strip() for l in open('/tmp/ky.sass') if re.search(r'/\*[0-9a-f]{4,5}\*/\s+\S', l)]
def op(l):
    t=l.split(); o=t[1] if t[0].startswith('@') else t[0]; return o.split('.')[0]
ops=[op(l) for l in ins]
idx=[i for i,o in enumerate(ops) if o=='STG']
c=collections.Counter(ops)
print(f"instrs {len(ops)} STG {c['STG']} LDS {c['LDS']} BSSY {c['BSSY']} LDL {c['LDL']} STL {c['STL']}")
if len(idx)>20:
    a,b=idx[len(idx)//4],idx[3*len(idx)//4]; n=b-a; k=3*len(idx)//4-len(idx)//4
    print(f"mid region {n/k:.1f} instr/STG", collections.Counter(ops[a:b]).most_common(8))
PY
cuobjdump -res-usage /tmp/ky.cubin 2>/dev/null | grep -o "REG:[0-9]*\|STACK:[0-9]*" | tr '\n' ' '; echo
