"""Aggregate an ncu SASS source page (instructions executed, stall samples) by
CUDA source line, using nvdisasm -g line info of the same cubin.
Usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_SUBSTRING [N]"""
import csv, io, os, re, subprocess, sys, tempfile
from collections import defaultdict

rep, sub = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_1606_04473_b200", "libara.so")], cwd=tmp,
               capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
secs = re.split(r"\n\s*\.section\s+\.text\.", dis)
sec = [s for s in secs if sub in s.split("\n")[0]][0]
line_of = {}
cur = None
for ln in sec.split("\n"):
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = []
for r in rows[2:]:   # the first kernel's rows only (a report may hold several launches)
    if r and r[0] == "Address":
        break
    if len(r) == len(hdr):
        data.append(r)
ie, si = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
a0 = int(data[0][0], 16)
ins, stall = defaultdict(float), defaultdict(float)
for r in data:
    key = line_of.get(int(r[0], 16) - a0, ("?", 0))
    ins[key] += float(r[ie] or 0)
    stall[key] += float(r[si] or 0)
ti, ts = sum(ins.values()), sum(stall.values())
src = {}
for f in set(k[0] for k in ins):
    for base in (os.path.join(ROOT, "paper_1606_04473_b200", "csrc"), "/usr/local/cuda/include"):
        p = os.path.join(base, f)
        if os.path.exists(p):
            src[f] = open(p).read().split("\n")
print(f"total instructions executed {ti:.3e}")
for k in sorted(ins, key=lambda k: -ins[k])[:top]:
    text = src.get(k[0], [""] * (k[1] + 1))[k[1] - 1].strip() if k[1] else ""
    print(f"{100 * ins[k] / ti:5.1f}% ins {100 * stall[k] / ts:5.1f}% stall  {k[0]}:{k[1]}  {text[:80]}")
