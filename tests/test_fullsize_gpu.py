"""Full-size parity at BASELINE.json's sizes, in the launch configuration
bench.py times: the GPU computes every trial; the oracle recomputes a sample
of trials regenerated independently from the counter-based streams, plus the
properties that hold at any size (mass conservation on integer data, metrics
of the GPU YLT against the oracle's metrics routine)."""
import os

import numpy as np
import pytest

import oracle
import synth
from parity_util import RTOL

pytestmark = pytest.mark.gpu


def _sample(T, n, seed):
    rng = np.random.default_rng(seed)
    s = set(rng.choice(T, size=n, replace=False).tolist()) | {0, 1, T // 2, T - 2, T - 1}
    return sorted(s)


def _device_yet(w):
    import torch
    off, ids = synth.gen_yet(w)
    return (torch.from_numpy(off.view(np.int64)).cuda(), torch.from_numpy(ids.view(np.int32)).cuda(),
            off, ids)


@pytest.mark.parametrize("name,precision", [("paper", "f64"), ("paper", "f32"), ("multilayer", "f64")])
def test_fullsize_sampled(cuda, name, precision):
    import torch
    from paper_1606_04473_b200 import ara
    w = synth.get_config(name)
    eo, ev, ls = synth.gen_elts(w)
    d_off, d_ids, off, ids = _device_yet(w)
    L = len(w.layers)
    ylt = torch.empty((L + 1, w.n_trials), dtype=torch.float64, device="cuda")
    lossy = torch.empty((L, w.n_trials), dtype=torch.int32, device="cuda")
    with ara.Context(w.catalog, precision=precision, stream=torch.cuda.current_stream()) as ctx:
        ctx.load_elts(eo, ev, ls, w.elt_terms())
        ctx.load_yet(w.n_trials, 0, d_off, d_ids)
        st = ctx.run(w.layers, ylt, lossy)
        k, pml, tvar, _ = ctx.metrics(w.return_periods)
    torch.cuda.synchronize()
    Y = ylt.cpu().numpy()
    M = lossy.cpu().numpy().view(np.uint32)
    assert st["n_events_local"] == len(ids)

    pick = _sample(w.n_trials, 400, 7)
    so, si = synth.gen_trial_sample(w, pick)
    assert np.array_equal(si[:int(so[1])], ids[int(off[0]):int(off[1])])
    orc = oracle.ara(so, si, oracle.Elts(eo, ev, ls), w.catalog, *w.elt_terms(),
                     oracle.layers_from_specs(w.layers), lookup="map", fp32_storage=precision == "f32")
    tol = RTOL * np.maximum(orc["scale"], 1.0)
    assert (np.abs(Y[:L, pick] - orc["ylt"]) <= tol).all()
    assert np.array_equal(M[:, pick], orc["lossy"])
    assert (np.abs(Y[L, pick] - orc["portfolio"]) <= tol.sum(axis=0)).all()
    # every clamp binds somewhere in the sample (the calibrated terms of DESIGN.md)
    assert 0 < (Y[0] == 0).mean() < 1 and 0 < (Y[0] == w.layers[0].agg_limit).mean() < 1

    # metrics: the device radix select / tail sums against the oracle's metric
    # routine applied to the device YLT (PML bit-exact, TVaR to summation error)
    for r in range(L + 1):
        kk, p_o, t_o = oracle.metrics(Y[r], w.return_periods)
        assert np.array_equal(kk, k)
        assert np.array_equal(p_o, pml[r])
        assert np.allclose(t_o, tvar[r], rtol=1e-12, atol=0)


def test_mass_conservation_integer_identity(cuda):
    """P8 at 100k paper-shaped trials: identity terms on integer data ->
    sum_t Y_t == sum_e N_e rowsum(e) exactly (independent of trial order)."""
    import torch
    from paper_1606_04473_b200 import ara
    w = synth.get_config("paper").with_(n_trials=100_000, int_cap=2.0 ** 31)
    eo, ev, ls = synth.gen_elts(w)
    off, ids = synth.gen_yet(w)
    E = w.n_elts
    layer = (synth.LayerSpec(0, E, 0.0, float("inf"), 0.0, float("inf")),)
    with ara.Context(w.catalog) as ctx:
        ctx.load_elts(eo, ev, ls, (np.zeros(E), np.full(E, np.inf)))
        ctx.load_yet(w.n_trials, 0, off, ids)
        Y, _, _ = ctx.run_host(layer, with_lossy=False)
    rowsum = np.zeros(w.catalog + 1, dtype=np.int64)          # integer arithmetic: exact
    np.add.at(rowsum, ev, ls.astype(np.int64))
    N = np.bincount(ids, minlength=w.catalog + 1).astype(np.int64)
    assert (Y[0] == np.floor(Y[0])).all() and Y[0].max() < 2.0 ** 53
    assert int(Y[0].astype(np.int64).sum()) == int(np.dot(N, rowsum))
    assert np.array_equal(Y[0], Y[1])


def test_fullsize_full_oracle_ylt_and_metrics(cuda):
    """The whole paper-shaped YLT (1M trials, 1e9 events, 16 ELTs) computed by
    the CPU oracle on all host cores (threads over contiguous trial ranges; the
    oracle releases the GIL) and compared with the GPU's at every trial; then
    PML/TVaR of the oracle's YLT (the oracle's own metric routine) against the
    GPU's device select: order statistics and top-k means are 1-Lipschitz in the
    sup norm, so they may differ by at most the largest per-trial difference."""
    import threading
    import torch
    from paper_1606_04473_b200 import ara
    w = synth.get_config("paper")
    eo, ev, ls = synth.gen_elts(w)
    d_off, d_ids, off, ids = _device_yet(w)
    L = len(w.layers)
    ylt = torch.empty((L + 1, w.n_trials), dtype=torch.float64, device="cuda")
    lossy = torch.empty((L, w.n_trials), dtype=torch.int32, device="cuda")
    with ara.Context(w.catalog, stream=torch.cuda.current_stream()) as ctx:
        ctx.load_elts(eo, ev, ls, w.elt_terms())
        ctx.load_yet(w.n_trials, 0, d_off, d_ids)
        ctx.run(w.layers, ylt, lossy)
        k, pml, tvar, _ = ctx.metrics(w.return_periods)
    torch.cuda.synchronize()
    Y = ylt.cpu().numpy()
    M = lossy.cpu().numpy().view(np.uint32)
    del d_off, d_ids

    E = oracle.Elts(eo, ev, ls)
    dense = oracle.direct_access(E, w.catalog)
    d, li = w.elt_terms()
    lay = oracle.layers_from_specs(w.layers)
    T = w.n_trials
    nt = max(1, min(64, os.cpu_count() or 1))
    bounds = [T * i // nt for i in range(nt + 1)]
    oy = np.zeros((L, T))
    osc = np.zeros((L, T))
    olo = np.zeros((L, T), dtype=np.uint32)
    oport = np.zeros(T)

    def work(i):
        a, b = bounds[i], bounds[i + 1]
        so = off[a:b + 1] - off[a]
        r = oracle.ara(so, ids[int(off[a]):int(off[b])], E, w.catalog, d, li, lay, lookup="dense", dense=dense)
        oy[:, a:b], osc[:, a:b], olo[:, a:b], oport[a:b] = r["ylt"], r["scale"], r["lossy"], r["portfolio"]

    th = [threading.Thread(target=work, args=(i,)) for i in range(nt)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    tol = RTOL * np.maximum(osc, 1.0)
    assert (np.abs(Y[:L] - oy) <= tol).all()
    assert np.array_equal(M, olo)
    assert (np.abs(Y[L] - oport) <= tol.sum(axis=0)).all()
    rows = list(oy) + [oport]
    for r in range(L + 1):
        sup = np.abs(Y[r] - rows[r]).max()
        kk, p_o, t_o = oracle.metrics(rows[r], w.return_periods)
        assert np.array_equal(kk, k)
        assert (np.abs(pml[r] - p_o) <= sup).all()
        assert (np.abs(tvar[r] - t_o) <= sup + 1e-12 * np.abs(t_o)).all()
