"""Top SASS lines by executed warp-instructions: python tools/ncu_top.py REP REGEX SKIP [TOP]"""
import csv, io, subprocess, sys
rep, kern, skip = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(r for r in rows if "Address" in r and "Source" in r)
seen, data = set(), []
for r in rows[rows.index(hdr) + 1:]:
    if len(r) == len(hdr) and r[hdr.index("Address")] not in seen:
        seen.add(r[hdr.index("Address")]); data.append(dict(zip(hdr, r)))
f = lambda x: float(x) if x.replace('.', '', 1).isdigit() else 0.0  # noqa: E731
tot = sum(f(d["Instructions Executed"]) for d in data)
print(rows[0][1][:90], f"{tot:.3e} warp-instr")
for d in sorted(data, key=lambda d: -f(d["Instructions Executed"]))[:top]:
    w = f(d["Instructions Executed"])
    print(f"{d['Address'][-5:]} {w:9.3e} {100*w/tot:5.2f}% lanes {f(d['Avg. Threads Executed']):4.1f} {d['Source'][:80]}")
