"""Per CUDA-source-line warp-stall samples and executed instructions of one kernel.

    python tools/ncu_src.py REPORT.ncu-rep KERNEL_REGEX [launch_skip] [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda", "--kernel-name",
                      f"regex:{kern}", "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
out, fname = [], ""
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[2] == "-":
        d = dict(zip(hdr[:4], r[:4]))
        samp = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        ins = float(r[hdr.index("Instructions Executed")] or 0)
        out.append((samp, ins, f"{fname}:{r[0]}", r[1].strip()[:100]))
ts = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
print(f"samples {ts:.0f}  warp-instr {ti:.3e}")
for s, i, loc, src in sorted(out, key=lambda o: -o[0])[:top]:
    print(f"{100 * s / ts:5.1f}% stall  {100 * i / ti:5.1f}% instr  {loc:16s} {src}")
