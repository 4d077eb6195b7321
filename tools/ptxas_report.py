"""Registers / spills per kernel from `nvcc -Xptxas -v` (check before spending GPU time).

    python tools/ptxas_report.py [substring ...]
"""
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2403_13806_b200.build import NVCC_FLAGS, nvcc  # noqa: E402

import os  # noqa: E402
flags = [f for f in NVCC_FLAGS if f not in ("-shared", "-cudart", "static")]
flags += os.environ.get("RS_NVCC_EXTRA", "").split()  # the same experiment flags as build()
out = subprocess.run([nvcc(), *flags, "-Xptxas", "-v", "-c", str(ROOT / "paper_2403_13806_b200/csrc/api.cu"),
                      "-o", "/tmp/_ptxas_report.o"], capture_output=True, text=True).stderr
name, rows = None, []
for ln in out.splitlines():
    m = re.search(r"Compiling entry function '(\w+)'", ln)
    if m:
        name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        name = re.sub(r"\(.*", "", name).replace("rs::", "")
        spill = 0
    m = re.search(r"(\d+) bytes spill stores", ln)
    if m and name:
        spill = int(m.group(1))
    m = re.search(r"Used (\d+) registers", ln)
    if m and name:
        rows.append((name, int(m.group(1)), spill))
        name = None
pats = sys.argv[1:]
for n, r, sp in rows:
    if not pats or any(p in n for p in pats):
        print(f"{r:4d} regs  {sp:4d} B spill  {n}")
