# cfg3 knob sweep (flushed/steady, tools/quick_cfgs.py)
for env in "X=1" "VPG_THREADS=288" "VPG_THREADS=320" "VPG_THREADS=384" "VPG_THREADS=288 VPG_CTA_SMEM=110000" "X=2" "VPG_THREADS=288"; do
  echo "== $env"; env $env QC_STEPS=20 python tools/quick_cfgs.py ${CFGS:-cfg3} 2>&1 | tail -1
done
