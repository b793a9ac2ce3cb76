"""cfg3 tile-budget x CTA-smem x threads sweep (flushed mean / steady us),
one process per setting (plan knobs are read at plan creation)."""
import itertools
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
for b, c, t in itertools.product(["24576", "32768", "40960", "49152"], ["75000", "110000", "150000"], ["256", "128"]):
    env = dict(os.environ, VPG_TILE_BUDGET=b, VPG_CTA_SMEM=c, VPG_THREADS=t, QC_STEPS="20")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "quick_cfgs.py"), cfg], env=env,
                         capture_output=True, text=True).stdout.strip().splitlines()
    print(f"budget {b} cta_smem {c} threads {t}: {out[-1] if out else '?'}", flush=True)
