"""Minimal driver for ncu / A-B runs of the ARA hot path (device-resident inputs).
Usage: python tools/prof_ara.py [--config paper] [--precision f64] [--steps 2] [--l2-persist]"""
import argparse, json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="paper")
ap.add_argument("--precision", default="f64")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--l2-persist", action="store_true")
ap.add_argument("--rho", type=float, default=None)
ap.add_argument("--catalog", type=int, default=None)
ap.add_argument("--mode", default="direct")
a = ap.parse_args()
import torch
from paper_1606_04473_b200 import ara
w = synth.get_config(a.config)
if a.rho is not None:
    w = w.with_(rho=a.rho)
if a.catalog is not None:
    w = w.with_(catalog=a.catalog)
off, ids = synth.gen_yet(w)
eo, ev, ls = synth.gen_elts(w)
d_off = torch.from_numpy(off.view(np.int64)).cuda()
d_ids = torch.from_numpy(ids.view(np.int32)).cuda()
d_eo, d_ev, d_ls = (torch.from_numpy(x).cuda() for x in (eo.view(np.int64), ev.view(np.int32), ls))
ctx = ara.Context(w.catalog, precision=a.precision, stream=torch.cuda.current_stream(), l2_persist=a.l2_persist,
                  run_mode=a.mode)
res = []
for s in range(a.steps):
    ctx.load_elts(d_eo, d_ev, d_ls, w.elt_terms())
    ctx.load_yet(w.n_trials, 0, d_off, d_ids)
    st = ctx.run(w.layers)
    k, pml, tvar, mms = ctx.metrics(w.return_periods)
    res.append((st["kernel_ms"], mms))
torch.cuda.synchronize()
ctx.close()
print(json.dumps({"config": w.name, "catalog": w.catalog, "mode": a.mode, "precision": a.precision, "env": {k: v for k, v in os.environ.items() if k.startswith("ARA_")},
                  "l2_persist": a.l2_persist, "kernel_ms": [r[0] for r in res], "metrics_ms": [r[1] for r in res],
                  "events": len(ids), "pml0": pml[0].tolist()}))
