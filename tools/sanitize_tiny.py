"""Small end-to-end exercise of every kernel path, for compute-sanitizer
(memcheck / racecheck / synccheck): all ARA_KERNEL variants, fold mode,
packed + chunked YET, multi-layer edge windows, metrics.  No torch."""
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


w = synth.get_config("tiny").with_(n_trials=300)
ref = run(w, w.layers, 0)
for v in (-1, 1, 5, 8, 9):
    assert np.array_equal(run(w, w.layers, v), ref), v
assert np.array_equal(run(w, w.layers, -1, run_mode="fold"), ref)
assert np.array_equal(run(w, w.layers, -1, load_mode="chunked", chunk_trials=37, packed=True), ref)
w2 = synth.get_config("tiny").with_(n_elts=40, catalog=500, rho=0.3, n_trials=100, nmin=0, nmax=70)
L = (synth.LayerSpec(0, 16, 1e4, 1e6, 1e5, 1e7), synth.LayerSpec(3, 19, 0, 1e6, 0, 1e7),
     synth.LayerSpec(5, 38, 0, 1e6, 0, 1e7), synth.LayerSpec(8, 24, 0, 1e6, 0, 1e7), synth.LayerSpec(8, 24, 1, 2e5, 3, 1e7))
a = run(w2, L, 0)
for v in (5, 8, 9):
    assert np.array_equal(run(w2, L, v), a)
a32 = run(w2, L, 0, precision="f32")
assert np.array_equal(run(w2, L[:2], -1, run_mode="fold", precision="f32")[:2], a32[:2])
print("sanitize_tiny ok")
