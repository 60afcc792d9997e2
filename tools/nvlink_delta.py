"""Sum the NVLink data counters of `nvidia-smi nvlink -gt d` snapshots taken
before and after a run, per GPU, and relate them to the run's bench line.
Usage: python tools/nvlink_delta.py BEFORE AFTER BENCH_JSON"""
import json
import re
import sys


def parse(path):
    gpu, tot = None, {}
    for line in open(path):
        m = re.match(r"GPU (\d+):", line)
        if m:
            gpu = int(m.group(1))
            tot[gpu] = {"tx": 0, "rx": 0}
            continue
        m = re.search(r"Data (Tx|Rx):\s*([\d.]+)\s*(\w+)", line)
        if m and gpu is not None:
            scale = {"KiB": 1024, "MiB": 1024 ** 2, "GiB": 1024 ** 3, "B": 1}.get(m.group(3), 1024)
            tot[gpu][m.group(1).lower()] += float(m.group(2)) * scale
    return tot


b, a = parse(sys.argv[1]), parse(sys.argv[2])
try:
    d = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
    steps = d["steps"] + d["warmup"]
    info = {"ms_per_step": d["ms_per_step"], "value": d["value"], "breakdown_ms": d.get("breakdown_ms")}
except Exception as e:  # noqa: BLE001
    steps, info = None, {"error": str(e)}
out = {"run": sys.argv[3], "steps_incl_warmup": steps, "bench": info, "per_gpu": {}}
for g in sorted(a):
    tx = a[g]["tx"] - b.get(g, {}).get("tx", 0)
    rx = a[g]["rx"] - b.get(g, {}).get("rx", 0)
    out["per_gpu"][g] = {"tx_bytes": tx, "rx_bytes": rx,
                         "tx_bytes_per_step": tx / steps if steps else None}
print(json.dumps(out))
