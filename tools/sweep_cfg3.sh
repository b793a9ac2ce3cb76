# cfg3 knob sweep (flushed/steady, tools/quick_cfgs.py); args: extra env for every line
for env in "X=1" "VPG_BULK=1" "VPG_BULK=1 VPG_NBUF=3" "VPG_BULK=1 VPG_NBUF=4" "VPG_BULK=1 VPG_CTA_SMEM=110000" "VPG_BULK=1 VPG_TILE_BUDGET=32768" "VPG_BULK=1 VPG_THREADS=128" "VPG_TILE_BUDGET=32768"; do
  echo "== $env"; env $env QC_STEPS=20 python tools/quick_cfgs.py ${CFGS:-cfg3} 2>&1 | tail -1
done
