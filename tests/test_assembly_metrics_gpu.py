"""GPU tests of the multi-rank code paths that a one-GPU box can run, each
against the CPU oracle:

* a9, the fused peer-store YLT assembly (Alg. 1 l.9 "Populate YLT from YLT_i",
  P:313, over the split of P:306): ARA_LOOPBACK="W,r" makes a one-rank
  context hold rank r's ara_partition shard of a W-rank job and run the same
  kernel epilogue (store_trial's peer stores at peer_t0 + t, row stride
  peer_ld = T_global) into a local global-YLT buffer;
* the distributed PML/TVaR select with an identity reduce
  (world 1: ARA_METRICS_DIST=1, and every loopback shard);
* ara_metrics at 11 and 64 return periods (two tail sweeps; > 48 KB of
  histogram shared memory), the reload-failure and metrics-after-reload state
  rules of include/ara.h."""
import math

import numpy as np
import pytest

import oracle
import synth
from parity_util import RTOL, assert_metrics_close, assert_ylt_close, make_inputs, oracle_rows, run_gpu, run_oracle

pytestmark = pytest.mark.gpu
INF = math.inf


def _ctx(w, env=None, **kw):
    import os
    from paper_1606_04473_b200 import ara
    env = dict(env or {})
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        return ara.Context(w.catalog, **kw)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _bumped(layers):
    return tuple(L.__class__(L.elt_begin, L.elt_end, L.occ_retention * 1.5 + 1.0, L.occ_limit, L.agg_retention,
                             L.agg_limit) for L in layers)


@pytest.mark.parametrize("W", [2, 3, 8])
@pytest.mark.parametrize("rho,tower", [(0.02, False), (0.3, False), (0.02, True)])
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_loopback_peer_store_assembly(cuda, W, rho, tower, precision):
    """Every shard r of a W-rank split run on its own: the global-YLT buffer
    holds the oracle's values at columns [first, first + count) -- the peer
    stores' global index -- and nothing anywhere else (NaN fill); three
    consecutive runs alternate the two buffers; the shard's metrics come from
    the distributed select with an identity reduce."""
    from paper_1606_04473_b200 import ara
    w = synth.get_config("tiny").with_(n_trials=1001, rho=rho)
    layers = w.layers
    if tower:   # 3 layers on one window: one launch, layers + portfolio rows all peer-stored
        L0 = w.layers[0]
        layers = (L0, L0.__class__(0, 3, 1e5, 4e5, 0.0, INF), L0.__class__(0, 3, 0.0, INF, 2e6, 3e6))
    off, ids, elts = make_inputs(w)
    orc = {False: run_oracle(off, ids, elts, w, layers, fp32=precision == "f32"),
           True: run_oracle(off, ids, elts, w, _bumped(layers), fp32=precision == "f32")}
    R = (2, 10, 100)
    got = np.full((len(layers) + 1, w.n_trials), np.nan)
    for r in range(W):
        f, c = ara.ara_partition(w.n_trials, W, r)
        so = off[f:f + c + 1].copy()
        si = ids[int(off[f]):int(off[f + c])].copy()
        with _ctx(w, {"ARA_LOOPBACK": f"{W},{r}"}, precision=precision) as ctx:
            ctx.load_elts(*elts, w.elt_terms())
            ctx.load_yet(w.n_trials, f, so, si)
            for i, bumped in enumerate((False, True, False)):
                ylt, lossy, st = ctx.run_host(_bumped(layers) if bumped else layers, n_local=c)
                o = orc[bumped]
                cols = slice(f, f + c)
                shard = {"ylt": o["ylt"][:, cols], "scale": o["scale"][:, cols], "portfolio": o["portfolio"][cols],
                         "lossy": o["lossy"][:, cols]}
                assert_ylt_close(ylt[:, cols], shard)
                if c:
                    assert np.array_equal(lossy, shard["lossy"])
                outside = np.ones(w.n_trials, bool)
                outside[cols] = False
                assert np.isnan(ylt[:, outside]).all(), "a peer store landed outside the shard"
                if c:
                    k, pml, tvar, _ = ctx.metrics(R)
                    rows = list(shard["ylt"]) + [shard["portfolio"]]
                    for q, y in enumerate(rows):
                        ko, po, to = oracle.metrics(y, R)
                        assert np.array_equal(ko, k)
                        tol = RTOL * max(float(shard["scale"].max()), 1.0) * len(layers)
                        assert np.all(np.abs(po - pml[q]) <= tol) and np.all(np.abs(to - tvar[q]) <= tol)
                if i == 0:
                    got[:, cols] = ylt[:, cols]
    # the shards tile the single-GPU YLT bit for bit (P11)
    ref, _, _, _ = run_gpu(off, ids, elts, w, layers, precision=precision)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("rows_rho", [(1, 0.3), (3, 0.02)])
def test_distributed_select_identity_reduce(cuda, rows_rho):
    """ARA_METRICS_DIST=1 on one rank: the histogram passes, digit picks and
    tail sums of the distributed select with the all-reduces replaced by the
    identity -- PML bit-identical to the oracle's order statistic on integer
    data, TVaR exact there too."""
    n_layers, rho = rows_rho
    R = (1, 2, 3.5, 10, 100, 1000, 5003)
    w = synth.get_config("tiny").with_(n_trials=5003, rho=rho, int_cap=2.0 ** 31)
    layers = tuple(synth.LayerSpec(0, 3, 2.5e4 * (i + 1), 5e5, 6.5e6 / (i + 1), 2.5e6) for i in range(n_layers))
    off, ids, elts = make_inputs(w)
    orc = run_oracle(off, ids, elts, w, layers)
    ylt, _, _, met = run_gpu(off, ids, elts, w, layers, return_periods=R, env={"ARA_METRICS_DIST": 1})
    assert np.array_equal(ylt[:-1], orc["ylt"])
    assert_metrics_close(met, oracle_rows(orc), orc["scale"], R, exact=True)
    _, _, _, met0 = run_gpu(off, ids, elts, w, layers, return_periods=R)
    assert np.array_equal(met[1], met0[1]) and np.array_equal(met[2], met0[2])


@pytest.mark.parametrize("n_rp", [11, 48, 49, 64])
@pytest.mark.parametrize("dist", [False, True])
def test_metrics_many_return_periods(cuda, n_rp, dist):
    """More return periods than one tail sweep holds (10), and more than 48 KB
    of per-block histograms (n_rp > 48): exact against oracle.metrics on
    integer-valued data, with repeated and fractional periods."""
    w = synth.get_config("tiny").with_(n_trials=3001, int_cap=2.0 ** 31)
    off, ids, elts = make_inputs(w)
    rng = np.random.default_rng(n_rp)
    R = np.concatenate([[1.0, 2.0, 2.0, 3001.0], rng.uniform(1.0, 3001.0, n_rp - 4)])
    orc = run_oracle(off, ids, elts, w, w.layers)
    _, _, _, met = run_gpu(off, ids, elts, w, w.layers, return_periods=R,
                           env={"ARA_METRICS_DIST": 1} if dist else None)
    assert_metrics_close(met, oracle_rows(orc), orc["scale"], R, exact=True)


def test_failed_reload_leaves_no_usable_table(cuda):
    """a reload rejected by the device (densify validation) after a
    successful load leaves the context without ELTs -- ara_run returns STATE
    instead of computing on a half-written table -- until a load succeeds."""
    from paper_1606_04473_b200 import ara
    w = synth.get_config("tiny")
    off, ids, elts = make_inputs(w)
    wb = w.with_(n_elts=5, seed=w.seed + 1)
    eb = synth.gen_elts(wb)
    bad_ev = np.where(np.arange(len(eb[1])) == 7, w.catalog + 3, eb[1]).astype(np.uint32)
    with ara.Context(w.catalog) as ctx:
        ctx.load_elts(*elts, w.elt_terms())
        ctx.load_yet(w.n_trials, 0, off, ids)
        ctx.run_host(w.layers)
        ctx.metrics((2, 10))
        with pytest.raises(ara.AraError) as e:
            ctx.load_elts(eb[0], bad_ev, eb[2])
        assert e.value.status == ara.ARA_ERR_OUT_OF_RANGE
        for call in (lambda: ctx.run(w.layers), lambda: ctx.metrics((2, 10))):
            with pytest.raises(ara.AraError) as e:
                call()
            assert e.value.status == ara.ARA_ERR_STATE
        ctx.load_elts(*elts, w.elt_terms())
        ylt, lossy, _ = ctx.run_host(w.layers)
    orc = run_oracle(off, ids, elts, w, w.layers)
    assert_ylt_close(ylt, orc)
    assert np.array_equal(lossy, orc["lossy"])


def test_metrics_read_the_last_run_after_a_new_yet(cuda):
    """ara_metrics reads the last run's YLT with that run's trial
    count and row stride, even after ara_load_yet loaded a larger (or smaller)
    YET -- no out-of-bounds read, no stride mix-up."""
    from paper_1606_04473_b200 import ara
    w = synth.get_config("tiny").with_(n_trials=2000)
    off, ids, elts = make_inputs(w)
    w2 = w.with_(n_trials=3500, seed=w.seed + 5)
    off2, ids2 = synth.gen_yet(w2)
    w3 = w.with_(n_trials=700, seed=w.seed + 6)
    off3, ids3 = synth.gen_yet(w3)
    orc = run_oracle(off, ids, elts, w, w.layers)
    R = (2, 10, 100, 1000)
    with ara.Context(w.catalog) as ctx:
        ctx.load_elts(*elts, w.elt_terms())
        ctx.load_yet(w.n_trials, 0, off, ids)
        ctx.run_host(w.layers)
        ref = ctx.metrics(R)
        for o, i, n in ((off2, ids2, w2.n_trials), (off3, ids3, w3.n_trials)):
            ctx.load_yet(n, 0, o, i)
            got = ctx.metrics(R)
            assert all(np.array_equal(a, b) for a, b in zip(got[:3], ref[:3]))
    assert_metrics_close(ref, oracle_rows(orc), orc["scale"], R)


@pytest.mark.parametrize("int_cap", [None, 2.0 ** 31])
def test_ep_curve_matches_oracle(cuda, int_cap):
    """SURVEY 8f F4 EP curve (A23): counts[row][i] = #{t : Y_t > x_i}, exact
    against the oracle's brute-force count over the same YLT (the GPU's, and
    on integer-valued data the oracle's own), for thresholds at -inf, below,
    at and between the losses (ties), at the maximum and +inf; consistent
    with the device PML: #{Y > PML(R)} < k <= #{Y >= PML(R)}."""
    from paper_1606_04473_b200 import ara
    kw = {"int_cap": int_cap} if int_cap else {}
    w = synth.get_config("tiny").with_(n_trials=5003, rho=0.02, **kw)
    layers = (w.layers[0], w.layers[0].__class__(0, 3, 1e5, 4e5, 0.0, INF))
    off, ids, elts = make_inputs(w)
    orc = run_oracle(off, ids, elts, w, layers)
    R = (1, 2, 5, 10, 100, 1000, 5003)
    with ara.Context(w.catalog) as ctx:
        ctx.load_elts(*elts, w.elt_terms())
        ctx.load_yet(w.n_trials, 0, off, ids)
        ylt, _, _ = ctx.run_host(layers)
        k, pml, _, _ = ctx.metrics(R)
        vals = np.unique(ylt)
        x = np.sort(np.concatenate([[-INF, -1.0, 0.0], vals[:: max(1, len(vals) // 500)],
                                    np.quantile(ylt, np.linspace(0, 1, 300)), [ylt.max(), ylt.max() * 2, INF]]))
        counts = ctx.ep_curve(x)
        assert counts.shape == (len(layers) + 1, len(x))
        for r in range(len(layers) + 1):
            assert np.array_equal(counts[r], oracle.ep_counts(ylt[r], x))
            if int_cap:
                rows = list(orc["ylt"]) + [orc["portfolio"]]
                assert np.array_equal(counts[r], oracle.ep_counts(rows[r], x))
            above = ctx.ep_curve(pml[r])[r]
            at_or_above = ctx.ep_curve(np.nextafter(pml[r], -INF))[r]
            assert (above < k).all() and (k <= at_or_above).all()
        assert counts[:, 0].tolist() == [w.n_trials] * (len(layers) + 1) and (counts[:, -1] == 0).all()
        for bad, status in (([2.0, 1.0], ara.ARA_ERR_DOMAIN), ([0.0, np.nan], ara.ARA_ERR_DOMAIN)):
            with pytest.raises(ara.AraError) as e:
                ctx.ep_curve(bad)
            assert e.value.status == status
        with pytest.raises(ara.AraError) as e:
            ctx.ep_curve([])
        assert e.value.status == ara.ARA_ERR_INVALID_ARG
