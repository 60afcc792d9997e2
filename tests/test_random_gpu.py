"""Randomised GPU cross-checks: many small random workloads (catalogue sizes,
trial lengths incl. empty and long trials, ELT densities from very sparse to
dense, layer windows aligned / unaligned / towers / disjoint) -- every kernel
family must match the oracle (A21 tolerance, exact lossy counts); the dense
kernels share the lane mapping and per-lane order, so they give the same YLT
bits; each fold-mode row equals the direct sparse kernel's (sparse fold pass)
or the dense kernels' (dense fold pass) bit for bit."""
import math

import numpy as np
import pytest

import synth
from parity_util import assert_ylt_close, run_gpu, run_oracle

pytestmark = pytest.mark.gpu
INF = math.inf


def _random_case(seed):
    rng = np.random.default_rng(seed)
    C = int(rng.choice([50, 700, 5000, 40_000]))
    n_elts = int(rng.integers(1, 40))
    rho = float(rng.choice([0.002, 0.01, 0.05, 0.3, 1.0]))
    T = int(rng.integers(1, 600))
    w = synth.get_config("tiny").with_(catalog=C, n_elts=n_elts, rho=rho, n_trials=T, nmin=0,
                                       nmax=int(rng.choice([5, 130, 700])), seed=1000 + seed)
    layers = []
    for _ in range(int(rng.integers(1, 5))):
        b = int(rng.integers(0, n_elts))
        e = int(rng.integers(b + 1, min(n_elts, b + 17) + 1))
        layers.append(synth.LayerSpec(b, e, float(rng.uniform(0, 8e4)),
                                      float(rng.choice([INF, rng.uniform(1e5, 2e6)])),
                                      float(rng.uniform(0, 1e6)), float(rng.choice([INF, rng.uniform(5e5, 5e6)]))))
    d = rng.uniform(0, 3e4, n_elts)
    li = np.where(rng.random(n_elts) < 0.3, INF, rng.uniform(5e4, 2e6, n_elts))
    return w, tuple(layers), (d, li)


@pytest.mark.parametrize("seed", range(24))
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_random_workloads(cuda, seed, precision):
    w, layers, terms = _random_case(seed)
    off, ids = synth.gen_yet(w)
    elts = synth.gen_elts(w)
    orc = run_oracle(off, ids, elts, w, layers, fp32=precision == "f32", terms=terms)
    ylt, lossy, _, _ = run_gpu(off, ids, elts, w, layers, precision=precision, terms=terms)
    assert_ylt_close(ylt, orc)
    assert np.array_equal(lossy, orc["lossy"])
    dense = {}
    for v in (30, 12, 5, 0):   # ballot-compacted rounds, cooperative ring, register pipeline (3 / 2 CTAs/SM)
        env = {"ARA_NO_SKIP": 1} if v != 30 else None
        other, olossy, _, _ = run_gpu(off, ids, elts, w, layers, precision=precision, terms=terms, variant=v, env=env)
        assert_ylt_close(other, orc)
        assert np.array_equal(olossy, orc["lossy"]), v
        if v != 30:
            dense[v] = other
    fold, flossy, _, _ = run_gpu(off, ids, elts, w, layers, precision=precision, terms=terms, run_mode="fold")
    # each fold chunk runs either the sparse fold pass (equal to the direct
    # sparse kernel, the default direct run on sparse blocks) or the dense one
    # (equal to the dense kernels): every row equals one of the two orders
    for r in range(fold.shape[0]):
        assert np.array_equal(fold[r], ylt[r]) or np.array_equal(fold[r], dense[12][r]), r
    assert np.array_equal(lossy, flossy)
    assert_ylt_close(fold, orc)
    assert np.array_equal(dense[12], dense[5]) and np.array_equal(dense[12], dense[0])
