"""Host vs device time of each C-ABI call in one bench step (paper config,
device-resident inputs): where the GPU idles between the calls.
Usage: python tools/step_host.py [--steps 30] [--config paper]"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="paper")
ap.add_argument("--steps", type=int, default=30)
a = ap.parse_args()
import torch  # noqa: E402
from paper_1606_04473_b200 import ara  # noqa: E402

w = synth.get_config(a.config)
off, ids = synth.gen_yet(w)
eo, ev, ls = synth.gen_elts(w)
d_off = torch.from_numpy(off.view(np.int64)).cuda()
d_ids = torch.from_numpy(ids.view(np.int32)).cuda()
d_eo, d_ev, d_ls = (torch.from_numpy(x).cuda() for x in (eo.view(np.int64), ev.view(np.int32), ls))
stream = torch.cuda.current_stream()
ctx = ara.Context(w.catalog, stream=stream)
terms = w.elt_terms()
R = list(w.return_periods)
names = ("load_elts", "load_yet", "run", "metrics")
host, dev, kern, met = [], [], [], []
evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
for i in range(a.steps + 3):
    h = [time.perf_counter()]
    evs[0].record(stream)
    ctx.load_elts(d_eo, d_ev, d_ls, terms, n_elts=w.n_elts)
    h.append(time.perf_counter())
    evs[1].record(stream)
    ctx.load_yet(w.n_trials, 0, d_off, d_ids)
    h.append(time.perf_counter())
    evs[2].record(stream)
    st = ctx.run(w.layers)
    h.append(time.perf_counter())
    evs[3].record(stream)
    _, _, _, mms = ctx.metrics(R)
    h.append(time.perf_counter())
    evs[4].record(stream)
    evs[4].synchronize()
    if i >= 3:
        host.append(np.diff(h) * 1e3)
        dev.append([evs[j].elapsed_time(evs[j + 1]) for j in range(4)])
        kern.append(st["kernel_ms"])
        met.append(mms)
host, dev = np.median(np.array(host), 0), np.median(np.array(dev), 0)
print(json.dumps({"host_ms": dict(zip(names, host.round(4).tolist())),
                  "event_ms": dict(zip(names, dev.round(4).tolist())),
                  "step_event_ms": round(float(dev.sum()), 4),
                  "kernel_ms": round(float(np.median(kern)), 4), "metrics_device_ms": round(float(np.median(met)), 4)}))
