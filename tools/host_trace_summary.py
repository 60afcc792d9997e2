"""Average the ARA_HOST_TRACE phase gaps of the last N steps (stderr of tools/step_host.py).
Usage: python tools/host_trace_summary.py TRACE [steps]"""
import collections
import sys

ev = [(float(l.split()[1]), " ".join(l.split()[2:])) for l in open(sys.argv[1]) if l.startswith("HT ")]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
# steps start at "ara_load_elts"
starts = [i for i, (_, w) in enumerate(ev) if w == "ara_load_elts"]
steps = [ev[a:b] for a, b in zip(starts, starts[1:] + [len(ev)])][-n - 1:-1]
acc = collections.defaultdict(list)
for st in steps:
    for (t0, w0), (t1, w1) in zip(st, st[1:]):
        acc[(w0, w1)].append(t1 - t0)
    acc[("step", "total")].append(st[-1][0] - st[0][0])
order = [(st[k][1], st[k + 1][1]) for k in range(len(steps[0]) - 1)] if steps else []
for k in order + [("step", "total")]:
    v = acc[k]
    print(f"{k[0]:>18s} -> {k[1]:<18s} {sum(v) / len(v):9.1f} us")
