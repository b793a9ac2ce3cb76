"""Tile budget x CTA smem sweep over several configs (flushed mean / steady)."""
import itertools
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfgs = sys.argv[1] if len(sys.argv) > 1 else "cfg1,cfg2,cfg3"
budgets = (sys.argv[2] if len(sys.argv) > 2 else "24576,32768").split(",")
smems = (sys.argv[3] if len(sys.argv) > 3 else "75000,110000").split(",")
for b, c in itertools.product(budgets, smems):
    env = dict(os.environ, VPG_TILE_BUDGET=b, VPG_CTA_SMEM=c, QC_STEPS="20")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "quick_cfgs.py"), cfgs], env=env,
                         capture_output=True, text=True).stdout.strip().splitlines()
    for line in out:
        print(f"budget {b} cta_smem {c}: {line}", flush=True)
