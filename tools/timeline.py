"""Copy/compute timeline of a chunked end-to-end run (host YET in pinned memory,
whole-trial chunks on the copy stream, each chunk's kernel waiting for its copy):
the B200 analogue of the paper's life-cycle grids.  Runs the
paper config through the C-ABI with ARA_TIMELINE set and summarises the JSON the
library writes.  Usage: python tools/timeline.py [--config paper] [--chunk 65536] [--out F]"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="paper")
ap.add_argument("--chunk", type=int, default=65536)
ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "timeline.json"))
a = ap.parse_args()
os.makedirs(os.path.dirname(a.out), exist_ok=True)
os.environ["ARA_TIMELINE"] = a.out          # read by the library at its first chunked run
import torch  # noqa: E402
import synth  # noqa: E402
from paper_1606_04473_b200 import ara  # noqa: E402

w = synth.get_config(a.config)
off, ids = synth.gen_yet(w)
eo, ev, ls = synth.gen_elts(w)
off_p = torch.from_numpy(off.view(np.int64)).pin_memory().numpy().view(np.uint64)
ids_p = torch.from_numpy(ids.view(np.int32)).pin_memory().numpy().view(np.uint32)
with ara.Context(w.catalog, load_mode="chunked", chunk_trials=a.chunk) as ctx:
    ctx.load_elts(eo, ev, ls, w.elt_terms())
    for _ in range(3):                       # the last run's timeline stays in the file
        ctx.load_yet(w.n_trials, 0, off_p, ids_p)
        st = ctx.run(w.layers)
tl = json.load(open(a.out))["chunks"]
c0, c1 = np.array([c["copy_ms"] for c in tl]).T
k0, k1 = np.array([c["kernel_ms"] for c in tl]).T
span = float(max(c1.max(), k1.max()))
copy_busy = float(np.sum(c1 - c0))
kern_busy = float(np.sum(k1 - k0))
# kernel time that ran while a later chunk's copy was in flight
hidden = float(sum(max(0.0, min(k1[i], c1[i + 1]) - max(k0[i], c0[i + 1])) for i in range(len(tl) - 1)))
print(json.dumps({"config": w.name, "chunks": len(tl), "chunk_trials": a.chunk, "span_ms": span,
                  "copy_busy_ms": copy_busy, "kernel_busy_ms": kern_busy,
                  "kernel_hidden_under_copies_ms": hidden, "overlap_fraction_of_kernel": hidden / kern_busy,
                  "exposed_after_last_copy_ms": float(k1.max() - c1.max()),
                  "h2d_gbs": 4.0 * len(ids) / (copy_busy * 1e6), "timeline": a.out}))
