"""Per-SASS-line executed instructions / thread utilisation for one kernel of an ncu report."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-skip", sys.argv[4] if len(sys.argv) > 4 else "0", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(r for r in rows if "Address" in r and "Source" in r)
data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


seen, uniq = set(), []
for d in data:
    if d["Address"] not in seen:
        seen.add(d["Address"])
        uniq.append(d)
tot_inst = sum(num(d["Instructions Executed"]) for d in uniq)
tot_thr = sum(num(d["Thread Instructions Executed"]) for d in uniq)
print(f"warp-instructions {tot_inst:.3e}  thread-instructions {tot_thr:.3e}  lanes/instr {tot_thr / max(tot_inst, 1):.1f}")
lo = float(sys.argv[3]) if len(sys.argv) > 3 else 0.002
for d in uniq:
    w = num(d["Instructions Executed"])
    if w / tot_inst >= lo:
        print(f"{d['Address'][-5:]} {w:10.3e} {100 * w / tot_inst:5.1f}% lanes {num(d['Avg. Threads Executed']):5.1f} "
              f"stall {d['Warp Stall Sampling (All Samples)']:>6}  {d['Source'][:70]}")
