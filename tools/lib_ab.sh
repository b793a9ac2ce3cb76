#!/bin/bash
# tools/lib_ab.sh shapes.txt spec1 spec2 ...   spec = lib.so[:ENV=val[,ENV=val]]  -> joined table
shapes=$1; shift
# A base build for the comparison (kept out of git, *.so is ignored):
#   mkdir -p /tmp/base tools/ab && git archive <rev> paper_2506_03686_b200/csrc include | tar -x -C /tmp/base
#   make -C /tmp/base/paper_2506_03686_b200/csrc && cp /tmp/base/paper_2506_03686_b200/libvpgpu.so tools/ab/libvpgpu_base.so
i=0
for spec in "$@"; do
  lib=${spec%%:*}; envs=""
  if [[ "$spec" == *:* ]]; then envs=$(echo "${spec#*:}" | tr ',' ' '); fi
  env VPG_LIB_PATH=$PWD/$lib $envs timeout 900 python tools/lib_ab.py $shapes > gpurun_out/libab_$i.txt 2> gpurun_out/libab_$i.err || tail -3 gpurun_out/libab_$i.err
  i=$((i+1))
done
python - "$@" <<'PY'
import sys
libs=sys.argv[1:]
cols=[[l.strip().split('|') for l in open(f'gpurun_out/libab_{i}.txt')] for i in range(len(libs))]
print('variants:', libs)
for rows in zip(*cols):
    r0=rows[0]
    print(f"E={r0[2]} {r0[0]} {r0[1]}: " + "  ".join(f"{r[3]:>7s}us ({r[4]})" for r in rows))
PY
