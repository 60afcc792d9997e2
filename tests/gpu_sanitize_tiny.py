"""Small end-to-end exercise of every kernel path, for compute-sanitizer
(memcheck / racecheck / synccheck): all ARA_KERNEL variants on sparse and
dense tables, fold mode, packed + chunked YET, multi-layer edge windows,
metrics; each result checked against the CPU oracle.  No torch."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_1606_04473_b200 import ara  # noqa: E402


def run(w, layers, variant, **kw):
    os.environ["ARA_KERNEL"] = str(variant)
    off, ids = synth.gen_yet(w)
    elts = synth.gen_elts(w)
    packed = kw.pop("packed", False)
    with ara.Context(w.catalog, **kw) as ctx:
        ctx.load_elts(*elts, terms=w.elt_terms())
        if packed:
            b = ara.bits_for_catalog(w.catalog)
            ctx.load_yet_packed(w.n_trials, 0, off, ara.ara_pack_ids(ids, b), b)
        else:
            ctx.load_yet(w.n_trials, 0, off, ids)
        y, m, _ = ctx.run_host(layers)
        ctx.metrics([1, 2, 10, w.n_trials])
    return y


import oracle  # noqa: E402  (test infrastructure: the check below)


def check(y, w, layers, fp32=False):
    off, ids = synth.gen_yet(w)
    eo, ev, ls = synth.gen_elts(w)
    d, li = w.elt_terms()
    o = oracle.ara(off, ids, oracle.Elts(eo, ev, ls), w.catalog, d, li, oracle.layers_from_specs(layers),
                   fp32_storage=fp32)
    tol = 1e-9 * np.maximum(o["scale"], 1.0)
    assert (np.abs(y[:-1] - o["ylt"]) <= tol).all()


w = synth.get_config("tiny").with_(n_trials=300)
for rho in (0.02, 0.3):                       # sparse (packed rows) and dense tables
    wr = w.with_(rho=rho)
    for v in (-1, 0, 5, 12, 30):              # every trial kernel (ARA_KERNEL)
        check(run(wr, wr.layers, v), wr, wr.layers)
    check(run(wr, wr.layers, -1, run_mode="fold"), wr, wr.layers)
    check(run(wr, wr.layers, -1, load_mode="chunked", chunk_trials=37, packed=True), wr, wr.layers)
w2 = synth.get_config("tiny").with_(n_elts=40, catalog=500, rho=0.3, n_trials=100, nmin=0, nmax=70)
L = (synth.LayerSpec(0, 16, 1e4, 1e6, 1e5, 1e7), synth.LayerSpec(3, 19, 0, 1e6, 0, 1e7),
     synth.LayerSpec(5, 38, 0, 1e6, 0, 1e7), synth.LayerSpec(8, 24, 0, 1e6, 0, 1e7), synth.LayerSpec(8, 24, 1, 2e5, 3, 1e7))
for v in (-1, 0, 5, 12):
    check(run(w2, L, v), w2, L)
check(run(w2, L, 0, precision="f32"), w2, L, fp32=True)
check(run(w2, L[:2], -1, run_mode="fold", precision="f32"), w2, L[:2], fp32=True)
print("sanitize_tiny ok")
