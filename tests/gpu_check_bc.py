"""Quick GPU check of one trial-kernel variant against the CPU oracle on the
sparse-table cases (tiny, edge trials, integer-valued, cross-trial patterns).
Usage: python tools/bc_check.py [variant]"""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import synth  # noqa: E402
from parity_util import assert_ylt_close, make_inputs, run_gpu, run_oracle  # noqa: E402

INF = math.inf
v = int(sys.argv[1]) if len(sys.argv) > 1 else 30
fails = 0


def check(name, off, ids, elts, w, layers, precision="f64", exact=False, terms=None):
    global fails
    orc = run_oracle(off, ids, elts, w, layers, fp32=precision == "f32", terms=terms)
    ylt, lossy, st, _ = run_gpu(off, ids, elts, w, layers, precision=precision, variant=v, terms=terms)
    try:
        if exact:
            assert np.array_equal(ylt[:-1], orc["ylt"]) and np.array_equal(ylt[-1], orc["portfolio"])
        else:
            assert_ylt_close(ylt, orc)
        assert np.array_equal(lossy, orc["lossy"])
        print(f"ok   {name} {precision} variant={st['kernel_variant']} ms={st['kernel_ms']:.3f}")
    except AssertionError as e:
        fails += 1
        print(f"FAIL {name} {precision} variant={st['kernel_variant']}: {str(e)[:300]}")


for rho in (0.02, 0.1, 0.3):
    for prec in ("f64", "f32"):
        w = synth.get_config("tiny").with_(rho=rho)
        off, ids, elts = make_inputs(w)
        check(f"tiny rho={rho}", off, ids, elts, w, w.layers, prec)
w = synth.get_config("tiny").with_(rho=0.02, int_cap=2.0 ** 31)
off, ids, elts = make_inputs(w)
check("tiny integer", off, ids, elts, w, w.layers, exact=True)

# edge trials
rng = np.random.default_rng(9)
w = synth.get_config("tiny").with_(n_elts=5, catalog=777, rho=0.04, n_trials=16)
_, _, elts = make_inputs(w)
lens = [0, 1, 2, 31, 32, 33, 0, 127, 128, 129, 255, 256, 257, 5000, 3, 0]
off = np.zeros(len(lens) + 1, dtype=np.uint64)
off[1:] = np.cumsum(lens)
ids = rng.integers(1, w.catalog + 1, size=int(off[-1])).astype(np.uint32)
layers = (synth.LayerSpec(0, 5, 2.5e4, 5e5, 6.5e5, 2.5e6), synth.LayerSpec(1, 4, 0.0, INF, 0.0, INF),
          synth.LayerSpec(3, 5, 1e5, 2e5, 1e6, 3e6), synth.LayerSpec(2, 3, 0.0, 1e4, 1e4, INF))
for prec in ("f64", "f32"):
    check("edge", off, ids, elts, w, layers, prec)

# short / empty / all-occupied trials back to back
rng = np.random.default_rng(21)
for rho in (0.01, 0.1, 0.3):
    w = synth.get_config("tiny").with_(catalog=4000, rho=rho, n_trials=8)
    _, _, elts = make_inputs(w)
    occupied = np.unique(elts[1])
    lens = rng.choice([0, 1, 2, 3, 5, 31, 32, 33, 127, 128, 129, 700], size=1500)
    trials = [rng.choice(occupied, n) if i % 7 == 3 else rng.integers(1, w.catalog + 1, n) for i, n in enumerate(lens)]
    off = np.zeros(len(trials) + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(t) for t in trials])
    ids = np.concatenate(trials).astype(np.uint32)
    w = w.with_(n_trials=len(trials))
    check(f"short/empty rho={rho}", off, ids, elts, w, w.layers)

# mini config, sparse
w = synth.get_config("mini").with_(n_trials=20000, rho=0.01)
off, ids, elts = make_inputs(w)
check("mini rho=0.01", off, ids, elts, w, w.layers)
# the paper's 2M-event catalogue (bitmap larger than shared memory: L1/L2 probes), 12k trials
for prec in ("f64", "f32"):
    w = synth.get_config("paper").with_(n_trials=12000)
    off, ids, elts = make_inputs(w)
    check("paper 12k trials", off, ids, elts, w, w.layers, prec)
w = synth.get_config("tower").with_(n_trials=6000)
off, ids, elts = make_inputs(w)
check("tower 6k trials", off, ids, elts, w, w.layers)
print("FAILS", fails)
sys.exit(1 if fails else 0)
