"""Per-instruction hot spots of an ncu --set full report (source page, SASS view):
instructions executed and stall samples per SASS line, grouped into address ranges.
Usage: python tools/ncu_sass_hot.py REPORT.ncu-rep [top_n]"""
import csv, io, subprocess, sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 60
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
# several kernels may be listed (device functions first); keep the largest block
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif cur is not None and r and r[0] != "Address":
        cur["rows"].append(r)
hdr = next(r for r in rows if r and r[0] == "Address")
ix = {h: i for i, h in enumerate(hdr)}
b = max(blocks, key=lambda b: sum(int(r[ix["Instructions Executed"]] or 0) for r in b["rows"]))
tot_i = sum(int(r[ix["Instructions Executed"]] or 0) for r in b["rows"])
tot_s = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in b["rows"])
print(b["name"], "instructions", tot_i, "samples", tot_s)
for k, r in enumerate(b["rows"]):
    ie = int(r[ix["Instructions Executed"]] or 0)
    ss = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    if ie > 0 or ss > 0:
        print(f"{k:5d} {ie:12d} {100*ss/max(tot_s,1):6.2f}% {r[ix['Source']][:90]}")
