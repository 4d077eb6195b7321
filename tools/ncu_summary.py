"""Summarise an ncu --set full report of one frame into profiles/.

    python tools/ncu_summary.py REPORT.ncu-rep OUT_PREFIX

Writes OUT_PREFIX.csv (per-launch duration, DRAM bytes, issue/occupancy, pipe use) and
OUT_PREFIX_traffic.json ({kernel: dram read+write bytes per launch}) that bench.py reads
for roofline.traffic.
"""
import csv
import io
import json
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
     "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
     "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
     "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
     "launch__grid_size", "launch__block_size"]
rep, out = sys.argv[1], sys.argv[2]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(M)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
         "ns": 1e-3, "us": 1, "ms": 1e3}
recs = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    name = d["Kernel Name"].split("(")[0].replace("void ", "")
    rec = {"kernel": name}
    for m in M:
        v = float(d[m].replace(",", "")) if d.get(m) not in (None, "", "n/a") else None
        if v is not None and m.startswith("dram__bytes"):
            v *= scale.get(u[m], 1)
        if v is not None and m == "gpu__time_duration.sum":
            v *= scale.get(u[m], 1)
        rec[m] = v
    recs.append(rec)
with open(out + ".csv", "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(["kernel", "us", "dram_read_MB", "dram_write_MB", "sm_throughput_pct", "warps_active_pct",
                "issue_active_pct", "warp_inst", "fma_pipe_pct", "xu_pipe_pct", "regs", "grid", "block"])
    for r in recs:
        w.writerow([r["kernel"], f"{r['gpu__time_duration.sum']:.2f}", f"{r['dram__bytes_read.sum'] / 1e6:.3f}",
                    f"{r['dram__bytes_write.sum'] / 1e6:.3f}"] +
                   [r[m] for m in M[3:]])
traffic = {}
for r in recs:
    traffic.setdefault(r["kernel"], []).append(r["dram__bytes_read.sum"] + r["dram__bytes_write.sum"])
# the LAST launch of each kernel: the warm-workspace frame (earlier launches of the capture are
# the workspace-sizing frames, whose blends return at once on the overflow flag)
json.dump({k: v[-1] for k, v in traffic.items()}, open(out + "_traffic.json", "w"), indent=1)
for r in recs:
    print(f"{r['kernel'][:40]:40s} {r['gpu__time_duration.sum']:8.1f} us  dram {(r['dram__bytes_read.sum'] + r['dram__bytes_write.sum']) / 1e6:8.2f} MB")
