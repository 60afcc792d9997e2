"""Summarise an ncu --set full report (one kernel) into the numbers DESIGN.md/bench use.
Usage: python tools/ncu_summary.py REPORT.ncu-rep [--json]"""
import csv, io, json, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_sectors_srcunit_tex_op_read.sum"]


def load(path, idx=0):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2 + idx]
    name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    d = {"kernel": name}
    for h, u, v in zip(hdr, units, vals):
        if h in KEYS or ("issue_stalled" in h and h.endswith("per_issue_active.ratio")):
            try:
                fv = float(v.replace(",", ""))
            except ValueError:
                continue
            if "issue_stalled" in h and fv < 0.05:
                continue
            d[h] = (fv, u)
    return d


def count(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    return len(list(csv.reader(io.StringIO(out)))) - 2


if __name__ == "__main__":
    if "--all" in sys.argv:
        for i in range(count(sys.argv[1])):
            d = load(sys.argv[1], i)
            print(f"[{i}] {d['kernel'][:80]}  time={d.get('gpu__time_duration.sum', ('?',))[0]} "
                  f"{d.get('gpu__time_duration.sum', ('', ''))[1]}  inst={d.get('smsp__inst_executed.sum', ('?',))[0]}  "
                  f"issue%={d.get('smsp__issue_active.avg.pct_of_peak_sustained_active', ('?',))[0]}  "
                  f"stalls={ {k.split('stalled_')[1].split('_per')[0]: round(v[0], 2) for k, v in d.items() if 'stalled' in k and v[0] > 0.5} }")
        sys.exit(0)
    d = load(sys.argv[1])
    if "--json" in sys.argv:
        print(json.dumps({k: (v[0] if isinstance(v, tuple) else v) for k, v in d.items()}, indent=1))
    else:
        for k, v in d.items():
            print(f"{k:90s} {v[1] if isinstance(v, tuple) else '':10s} {v[0] if isinstance(v, tuple) else v}")
