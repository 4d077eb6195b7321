"""Instruction mix of a kernel's loops (backward-branch spans) from `cuobjdump -sass`.

    python tools/sass_loops.py LIB.so MANGLED_NAME_PREFIX
"""
import collections
import re
import subprocess
import sys

lib, fn = sys.argv[1], sys.argv[2]
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout.split("\n")
start = next(i for i, l in enumerate(txt) if "Function : " + fn in l)
end = next((i for i, l in enumerate(txt[start + 1:], start + 1) if "Function :" in l), len(txt))
ins = []
for l in txt[start:end]:
    m = re.match(r"\s+/\*([0-9a-f]{4})\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
for a, t in ins:
    m = re.search(r"BRA.*?(0x[0-9a-f]+)", t)
    if m and int(m.group(1), 16) < a:
        lo = int(m.group(1), 16)
        c = collections.Counter(re.sub(r"^@!?P\w+\s+", "", x).split()[0] for b, x in ins if lo <= b <= a)
        print(f"loop {lo:#x}-{a:#x}: {sum(c.values())} instructions  " +
              " ".join(f"{k}:{v}" for k, v in c.most_common(14)))
