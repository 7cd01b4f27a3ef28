"""Summarise an ncu launch list (csv) and a --set full capture (.ncu-rep) of
the fill kernels into profiles/<tag>_ncu_summary.{json,md} and a launch csv.

usage: python tools/ncu_summary.py <tag> gpurun_out/launches.csv gpurun_out/prof_x.ncu-rep
"""
import collections
import csv
import json
import subprocess
import sys

tag, launches, rep = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(launches)))
hdr, recs = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        recs.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for d in recs:
    if not any(k in d["Kernel Name"] for k in ("k_prep", "k_shells")):
        continue
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("gf::", "")
    agg[name][d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))
launch = {k: {m: sum(v) / len(v) for m, v in ms.items()} | {"launches": len(ms["gpu__time_duration.sum"])}
          for k, ms in agg.items()}
with open(f"profiles/{tag}_launches.csv", "w") as f:
    w = csv.writer(f)
    w.writerow(["kernel", "launches", "mean_time_ns", "mean_dram_read_bytes", "mean_dram_write_bytes"])
    for k, v in launch.items():
        w.writerow([k, v["launches"], v["gpu__time_duration.sum"], v["dram__bytes_read.sum"],
                    v["dram__bytes_write.sum"]])

out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
det = list(csv.reader(out.splitlines()))
h = det[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
want = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Executed Ipc Active", "Issue Slots Busy", "Executed Instructions", "DRAM Throughput",
        "Memory Throughput", "L2 Hit Rate", "Grid Size", "Block Size", "Waves Per SM",
        "Warp Cycles Per Issued Instruction", "Dynamic Shared Memory Per Block",
        "Static Shared Memory Per Block"]
full = collections.defaultdict(dict)
for r in det[1:]:
    if r[mi] in want:
        name = r[ki].split("(")[0].replace("void ", "").replace("gf::", "")
        full[name][r[mi]] = f"{r[vi]} {r[ui]}".strip()
traffic = sum(v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"] for v in launch.values())
head = subprocess.run(["git", "rev-parse", "--short=12", "HEAD"], capture_output=True,
                      text=True).stdout.strip()
summary = {"tag": tag, "head": head, "launch_list": launch, "full_capture": full,
           "fill_dram_bytes_per_launch": traffic, "algorithmic_bytes_per_frame": 53079040}
json.dump(summary, open(f"profiles/{tag}_ncu_summary.json", "w"), indent=1)
print(json.dumps(summary, indent=1))
