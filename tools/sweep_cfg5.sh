# cfg5 / cfg4 knob sweep with the dynamic scheduler (tools/quick_cfgs.py)
for env in "X=1" "VPG_CTA_SMEM=150000" "VPG_CTA_SMEM=200000" "VPG_TILE_BUDGET=32768" "VPG_TILE_BUDGET=65536" "VPG_THREADS=512" "VPG_THREADS=128" "VPG_HINTS=1" "VPG_HINTS=2" "VPG_TILE_PICK=1" "VPG_TILE_PICK=2"; do
  echo "== $env"; env $env QC_STEPS=10 python tools/quick_cfgs.py cfg5 2>&1 | tail -1
done
for env in "X=1" "VPG_ROWS_SLOT=8192" "VPG_ROWS_SLOT=32768" "VPG_ROWS_BULK=0"; do
  echo "== $env"; env $env QC_STEPS=10 python tools/quick_cfgs.py cfg4 2>&1 | tail -1
done
