"""Break the end-to-end (host-buffer) step into its C-ABI calls, wall-clock each.
Usage: python tools/e2e_probe.py [--mode chunked|all] [--chunk N] [--steps 3]"""
import argparse, json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth
ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="chunked")
ap.add_argument("--chunk", type=int, default=65536)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--config", default="paper")
a = ap.parse_args()
import torch
from paper_1606_04473_b200 import ara
w = synth.get_config(a.config)
off_pin = torch.empty(w.n_trials + 1, dtype=torch.int64, pin_memory=True)
synth.gen_offsets(w, 0, w.n_trials, out=off_pin.numpy().view(np.uint64))
n_ev = int(off_pin[-1])
ids_pin = torch.empty(n_ev, dtype=torch.int32, pin_memory=True)
synth.gen_events(w, 0, n_ev, out=ids_pin.numpy().view(np.uint32))
eo, ev, ls = synth.gen_elts(w)
eo_p, ev_p, ls_p = (torch.from_numpy(x).pin_memory() for x in (eo.view(np.int64), ev.view(np.int32), ls))
ylt = torch.empty((len(w.layers) + 1) * w.n_trials, dtype=torch.float64, pin_memory=True)
ctx = ara.Context(w.catalog, load_mode=a.mode, chunk_trials=a.chunk, stream=torch.cuda.current_stream())
res = []
for s in range(a.steps):
    t0 = time.perf_counter(); ctx.load_elts(eo_p, ev_p, ls_p, w.elt_terms())
    t1 = time.perf_counter(); ctx.load_yet(w.n_trials, 0, off_pin, ids_pin)
    t2 = time.perf_counter(); st = ctx.run(w.layers, ylt)
    t3 = time.perf_counter(); ctx.metrics(w.return_periods)
    t4 = time.perf_counter()
    res.append({"load_elts": t1 - t0, "load_yet": t2 - t1, "run": t3 - t2, "metrics": t4 - t3,
                "kernel_ms": st["kernel_ms"], "h2d_ms": st["h2d_ms"], "total_ms": st["total_ms"]})
print(json.dumps({"mode": a.mode, "chunk": a.chunk, "steps": res}))
