"""Sweep the long-row threshold of the row-split plan (WalkOperator.LONG_ROW /
HUB_FACTOR) and time the DBLP bench step for each setting."""
import json
import subprocess
import sys

SETTINGS = [(64, 4), (32, 2), (48, 2), (24, 1.5), (128, 8)]
code = """
import sys, runpy
from paper_2408_05459_b200 import walk
walk.WalkOperator.LONG_ROW, walk.WalkOperator.HUB_FACTOR = {lr}, {hf}
sys.argv = ['bench.py', '--no-cpu-baseline', '--no-e2e']
runpy.run_path('bench.py', run_name='__main__')
"""
for lr, hf in SETTINGS:
    out = subprocess.run([sys.executable, "-c", code.format(lr=lr, hf=hf)], capture_output=True,
                         text=True, timeout=600).stdout.strip().splitlines()
    d = json.loads(out[-1])
    print(f"LONG_ROW={lr} HUB_FACTOR={hf}: step {d['ms_per_step']} ms, phases {d['phases_ms']}, "
          f"orth_fused {d['roofline']['duration_ms']} ms/launch", flush=True)
