"""Record the DRAM traffic and L2->SM sectors of one ncu --set full capture of
the ARA trial kernel into profiles/ara_kernel_traffic.json, keyed by
workload/precision, with the kernel variant and the trials per launch it was
captured at (bench.py uses the record only for a launch of the same variant
and size).
Usage: python tools/ncu_traffic_record.py REPORT WORKLOAD PRECISION VARIANT N_TRIALS SUMMARY_PATH"""
import json, os, sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import load  # noqa: E402

rep, workload, precision, variant, n_trials, summary = sys.argv[1:7]
d = load(rep)
g = lambda k: d[k][0]
scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
dram = g("dram__bytes_read.sum") * scale[d["dram__bytes_read.sum"][1]] + \
    g("dram__bytes_write.sum") * scale[d["dram__bytes_write.sum"][1]]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path = os.path.join(root, "profiles", "ara_kernel_traffic.json")
rec = json.load(open(path)) if os.path.exists(path) else {}
old = rec.get(f"{workload}/{precision}")
if old:
    rec.setdefault("_history", {})[f"{workload}/{precision} variant {old.get('variant')}"] = old
rec[f"{workload}/{precision}"] = {
    "variant": int(variant), "n_trials_per_launch": int(n_trials), "kernel": d["kernel"],
    "dram_bytes_per_launch": int(dram),
    "l2_sectors_per_launch": int(g("lts__t_sectors_srcunit_tex_op_read.sum")),
    "l1_from_l2_bytes_per_launch": int(g("l1tex__m_xbar2l1tex_read_bytes.sum") *
                                       scale[d["l1tex__m_xbar2l1tex_read_bytes.sum"][1]]),
    "l2_hit_rate_pct": g("lts__t_sector_hit_rate.pct"),
    "warp_instructions_per_launch": int(g("smsp__inst_executed.sum")),
    "duration_ms_ncu": g("gpu__time_duration.sum") * (1e-3 if d["gpu__time_duration.sum"][1] == "usecond" else 1.0),
    "source": summary,
}
json.dump(rec, open(path, "w"), indent=1)
print(json.dumps(rec[f"{workload}/{precision}"], indent=1))
