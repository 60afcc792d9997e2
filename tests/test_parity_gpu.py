"""GPU parity: the CUDA path (through the C-ABI binding) vs the CPU oracle,
element by element on the same seeded inputs (tolerances: parity_util)."""
import math

import numpy as np
import pytest

import oracle
import synth
from parity_util import (KERNEL_VARIANTS, RTOL, assert_metrics_close, assert_ylt_close, make_inputs,
                         oracle_rows, run_gpu, run_oracle)

pytestmark = pytest.mark.gpu
INF = math.inf


def _ara():
    from paper_1606_04473_b200 import ara
    return ara


# ------------------------------------------------------------------ tiny configs
@pytest.mark.parametrize("variant", KERNEL_VARIANTS)
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_tiny(cuda, precision, variant):
    w = synth.get_config("tiny").with_(return_periods=(1, 2, 3.5, 10, 100, 1000))
    off, ids, elts = make_inputs(w)
    orc = run_oracle(off, ids, elts, w, w.layers, fp32=precision == "f32")
    ylt, lossy, st, met = run_gpu(off, ids, elts, w, w.layers, precision=precision,
                                  return_periods=w.return_periods, variant=variant)
    assert_ylt_close(ylt, orc)
    assert np.array_equal(lossy, orc["lossy"])
    assert_metrics_close(met, oracle_rows(orc), orc["scale"], w.return_periods)
    assert st["n_events_local"] == len(ids) and st["n_lookups_local"] == len(ids) * w.n_elts


@pytest.mark.parametrize("variant", KERNEL_VARIANTS)
@pytest.mark.parametrize("precision,cap", [("f64", 2.0 ** 31), ("f32", 2.0 ** 24)])
def test_tiny_integer_valued_is_bitwise(cuda, precision, cap, variant):
    """P10: integer-valued losses and terms make every sum exact, so the GPU
    must match the oracle bit for bit in any summation order (YLT, portfolio,
    lossy counts, PML, TVaR)."""
    w = synth.get_config("tiny").with_(int_cap=cap, return_periods=(1, 2, 5, 10, 50, 1000))
    off, ids, elts = make_inputs(w)
    orc = run_oracle(off, ids, elts, w, w.layers, fp32=precision == "f32")
    ylt, lossy, _, met = run_gpu(off, ids, elts, w, w.layers, precision=precision,
                                 return_periods=w.return_periods, variant=variant)
    assert np.array_equal(ylt[:-1], orc["ylt"]) and np.array_equal(ylt[-1], orc["portfolio"])
    assert np.array_equal(lossy, orc["lossy"])
    assert_metrics_close(met, oracle_rows(orc), orc["scale"], w.return_periods, exact=True)


@pytest.mark.parametrize("variant", KERNEL_VARIANTS)
@pytest.mark.parametrize("rho", [0.02, 0.3])
def test_sparse_elts_row_skipping_is_exact(cuda, variant, rho):
    """ELTs as sparse as the paper's (10k-30k losses over a large catalogue,
    P:237): most rows of the direct-access table are all zero and the kernel
    skips their lookups via the row-occupancy bitmap.  A zero row adds an
    exact +0 (deductibles and retentions are >= 0): the YLT must match the
    oracle with and without skipping (ARA_NO_SKIP), lossy counts exactly."""
    w = synth.get_config("tiny").with_(rho=rho, return_periods=(2, 10, 100))
    off, ids, elts = make_inputs(w)
    orc = run_oracle(off, ids, elts, w, w.layers)
    ylt, lossy, _, met = run_gpu(off, ids, elts, w, w.layers, return_periods=w.return_periods, variant=variant)
    assert_ylt_close(ylt, orc)
    assert np.array_equal(lossy, orc["lossy"])
    assert_metrics_close(met, oracle_rows(orc), orc["scale"], w.return_periods)
    ylt2, lossy2, _, _ = run_gpu(off, ids, elts, w, w.layers, variant=variant, env={"ARA_NO_SKIP": 1})
    assert_ylt_close(ylt2, orc)
    assert np.array_equal(lossy2, orc["lossy"])


def test_device_pointer_inputs_match_host_inputs(cuda):
    w = synth.get_config("tiny")
    off, ids, elts = make_inputs(w)
    a = run_gpu(off, ids, elts, w, w.layers)
    b = run_gpu(off, ids, elts, w, w.layers, device_inputs=True)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


# ------------------------------------------------------------------ edge cases
def _edge_yet(C, rng):
    lens = [0, 1, 2, 31, 32, 33, 0, 127, 128, 129, 255, 256, 257, 5000, 3, 0]
    off = np.zeros(len(lens) + 1, dtype=np.uint64)
    off[1:] = np.cumsum(lens)
    ids = rng.integers(1, C + 1, size=int(off[-1])).astype(np.uint32)
    ids[:3] = [1, C, 1]
    ids[-3:] = [C, C, 1]
    return off, ids


@pytest.mark.parametrize("variant", KERNEL_VARIANTS)
@pytest.mark.parametrize("rho", [0.5, 0.04])
def test_edge_trials_and_unaligned_layers(cuda, variant, rho):
    rng = np.random.default_rng(9)
    w = synth.get_config("tiny").with_(n_elts=5, catalog=777, rho=rho, n_trials=16)
    _, _, elts = make_inputs(w)
    off, ids = _edge_yet(w.catalog, rng)
    layers = (synth.LayerSpec(0, 5, 2.5e4, 5e5, 6.5e5, 2.5e6), synth.LayerSpec(1, 4, 0.0, INF, 0.0, INF),
              synth.LayerSpec(3, 5, 1e5, 2e5, 1e6, 3e6), synth.LayerSpec(2, 3, 0.0, 1e4, 1e4, INF))
    for precision in ("f64", "f32"):
        orc = run_oracle(off, ids, elts, w, layers, fp32=precision == "f32")
        ylt, lossy, _, _ = run_gpu(off, ids, elts, w, layers, precision=precision, variant=variant)
        assert_ylt_close(ylt, orc)
        assert np.array_equal(lossy, orc["lossy"])
        assert (ylt[:, [0, 6, 15]] == 0).all()


@pytest.mark.parametrize("variant", KERNEL_VARIANTS)
def test_compacted_rounds_fifo_pressure(cuda, variant):
    """Sparse table, adversarial occupancy patterns for the compacted-rounds
    kernel: every event occupied (four rounds per 128-event batch), occupied
    events on one lane only, alternating, none, and random."""
    rng = np.random.default_rng(11)
    w = synth.get_config("tiny").with_(catalog=5000, rho=0.03, n_trials=8)
    _, _, elts = make_inputs(w)
    occupied = np.unique(elts[1])
    empty = np.setdiff1d(np.arange(1, w.catalog + 1), occupied)
    hot, cold = int(occupied[0]), int(empty[0])
    trials = [
        np.full(3000, hot),                                          # all occupied
        np.where(np.arange(2000) % 32 == 5, hot, cold),             # one lane only
        np.where(np.arange(1500) % 2 == 0, hot, cold),              # alternating
        np.full(700, cold),                                          # none
        rng.choice(occupied, 1000),                                  # random occupied ids
        rng.integers(1, w.catalog + 1, 4097),                        # random
        np.array([hot]),
        np.array([], dtype=np.int64),
    ]
    off = np.zeros(len(trials) + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(t) for t in trials])
    ids = np.concatenate(trials).astype(np.uint32)
    orc = run_oracle(off, ids, elts, w, w.layers)
    ylt, lossy, _, _ = run_gpu(off, ids, elts, w, w.layers, variant=variant)
    assert_ylt_close(ylt, orc)
    assert np.array_equal(lossy, orc["lossy"])


@pytest.mark.parametrize("variant", KERNEL_VARIANTS)
@pytest.mark.parametrize("rho", [0.2, 0.01])
def test_wide_windows_tower_and_many_layers(cuda, variant, rho):
    """40 ELTs: aligned, unaligned, 8-sector, >8-sector (generic kernel) and
    single-ELT layers; 4 identical windows (shared-load path); 9 layers ->
    three launches with the portfolio accumulated across them.  rho = 0.01
    makes every column block sparse (zero rows skipped, compacted rounds)."""
    w = synth.get_config("tiny").with_(n_elts=40, catalog=3000, rho=rho, n_trials=700, nmin=1, nmax=300)
    off, ids, elts = make_inputs(w)
    rng = np.random.default_rng(4)
    d = rng.uniform(0, 2e4, w.n_elts)
    li = np.where(rng.random(w.n_elts) < 0.3, INF, rng.uniform(1e5, 2e6, w.n_elts))
    layers = (synth.LayerSpec(0, 16, 2.5e4, 7.5e5, 1.2e6, 8e6), synth.LayerSpec(3, 19, 1e5, 4e5, 6.5e5, 4e6),
              synth.LayerSpec(0, 32, 0.0, INF, 1e6, INF), synth.LayerSpec(5, 38, 2.5e5, 5e5, 4e5, 3.5e6),
              synth.LayerSpec(39, 40, 0.0, INF, 0.0, INF),
              synth.LayerSpec(8, 24, 1e4, 1e6, 0.0, 2e6), synth.LayerSpec(8, 24, 5e4, 2e5, 1e5, 1e6),
              synth.LayerSpec(8, 24, 1e5, 1e5, 3e5, INF), synth.LayerSpec(8, 24, 0.0, 7e4, 0.0, 9e5))
    for precision in ("f64", "f32"):
        orc = run_oracle(off, ids, elts, w, layers, fp32=precision == "f32", terms=(d, li))
        ylt, lossy, st, _ = run_gpu(off, ids, elts, w, layers, precision=precision, terms=(d, li), variant=variant)
        assert_ylt_close(ylt, orc)
        assert np.array_equal(lossy, orc["lossy"])
        assert st["n_kernel_launches"] >= 3


def test_single_elt_single_event_lookup(cuda):
    """P12 on the GPU: one ELT, one event per trial, identity terms -> Y_t = L[e_t] exactly."""
    w = synth.get_config("tiny").with_(n_elts=1, n_trials=4000, nmin=1, nmax=1)
    off, ids, elts = make_inputs(w)
    dense = oracle.direct_access(oracle.Elts(*elts), w.catalog)
    ylt, _, _, _ = run_gpu(off, ids, elts, w, (synth.LayerSpec(0, 1, 0.0, INF, 0.0, INF),),
                           terms=(np.zeros(1), np.full(1, INF)))
    assert np.array_equal(ylt[0], dense[0, ids])


# ------------------------------------------------------------------ invariants
@pytest.mark.parametrize("variant", KERNEL_VARIANTS)
@pytest.mark.parametrize("rho", [0.3, 0.03])
def test_partition_and_alignment_invariance(cuda, variant, rho):
    """P11 on the GPU: shards loaded as independent YETs (different base
    alignment of every trial, different warp streams of the persistent sparse
    kernel) reproduce the unsharded YLT bit for bit: every kernel's summation
    order depends only on the trial's own events."""
    w = synth.get_config("tiny").with_(n_trials=1001, rho=rho)
    off, ids, elts = make_inputs(w)
    full, _, _, _ = run_gpu(off, ids, elts, w, w.layers, variant=variant)
    assert_ylt_close(full, run_oracle(off, ids, elts, w, w.layers))
    ara = _ara()
    for N in (2, 3, 8, 16):
        parts = []
        for r in range(N):
            f, c = ara.ara_partition(w.n_trials, N, r)
            so = off[f:f + c + 1].copy()
            si = ids[int(off[f]):int(off[f + c])]
            if r % 2:                      # misalign the shard by one element
                si = np.concatenate([np.zeros(1, np.uint32), si])[1:]
            y, _, _, _ = run_gpu(so, si, elts, w, w.layers, variant=variant)
            parts.append(y[:, :c])
        assert np.array_equal(np.concatenate(parts, axis=1), full)


def test_monotone_in_retentions_and_bounded(cuda):
    """P9 on the GPU, exact comparisons: raising a retention never raises any Y_t."""
    w = synth.get_config("tiny")
    off, ids, elts = make_inputs(w)
    base, _, _, _ = run_gpu(off, ids, elts, w, w.layers)
    L0 = w.layers[0]
    assert (base[0] >= 0).all() and (base[0] <= L0.agg_limit).all()
    for bumped in (L0.__class__(0, 3, L0.occ_retention * 2, L0.occ_limit, L0.agg_retention, L0.agg_limit),
                   L0.__class__(0, 3, L0.occ_retention, L0.occ_limit, L0.agg_retention * 1.3, L0.agg_limit)):
        y, _, _, _ = run_gpu(off, ids, elts, w, (bumped,))
        assert (y[0] <= base[0]).all() and (y[0] < base[0]).any()
    d, li = w.elt_terms()
    d2 = d.copy()
    d2[1] *= 4
    y, _, _, _ = run_gpu(off, ids, elts, w, w.layers, terms=(d2, li))
    assert (y[0] <= base[0]).all() and (y[0] < base[0]).any()


@pytest.mark.parametrize("pinned", [True, False])
@pytest.mark.parametrize("rho", [0.3, 0.03])
def test_chunked_h2d_equals_all_at_once(cuda, pinned, rho):
    import torch
    w = synth.get_config("tiny").with_(n_trials=3000, rho=rho)
    off, ids, elts = make_inputs(w)
    ref, ref_lossy, _, _ = run_gpu(off, ids, elts, w, w.layers)
    if pinned:
        po = torch.from_numpy(off.view(np.int64)).pin_memory()
        pi = torch.from_numpy(ids.view(np.int32)).pin_memory()
        off_h, ids_h = po.numpy().view(np.uint64), pi.numpy().view(np.uint32)
    else:
        off_h, ids_h = off.copy(), ids.copy()
    orc = run_oracle(off, ids, elts, w, w.layers)
    assert_ylt_close(ref, orc)
    assert np.array_equal(ref_lossy, orc["lossy"])
    for chunk in (1, 7, 333, 10 ** 7):
        ylt, lossy, st, met = run_gpu(off_h, ids_h, elts, w, w.layers, load_mode="chunked", chunk_trials=chunk,
                                      return_periods=(2, 10, 100))
        assert_ylt_close(ylt, orc)                                   # the oracle decides
        assert np.array_equal(lossy, orc["lossy"])
        assert_metrics_close(met, oracle_rows(orc), orc["scale"], (2, 10, 100))
        assert np.array_equal(ylt, ref) and np.array_equal(lossy, ref_lossy)   # P11: chunking changes no bit
        assert st["h2d_bytes"] == ids.nbytes + off.nbytes


@pytest.mark.parametrize("rho_a,rho_b", [(0.3, 0.02), (0.02, 0.3), (0.02, 0.02)])
def test_reload_elts_equals_fresh_context(cuda, rho_a, rho_b):
    """Reloading ELTs into a used context (the table is cleared row by row via
    the previous load's occupancy bitmap, not re-zeroed in full) gives exactly
    the YLT of a fresh context."""
    from paper_1606_04473_b200 import ara
    wa = synth.get_config("tiny").with_(rho=rho_a)
    wb = synth.get_config("tiny").with_(rho=rho_b, seed=wa.seed + 7)
    off, ids = synth.gen_yet(wb)
    ea, eb = synth.gen_elts(wa), synth.gen_elts(wb)
    with ara.Context(wb.catalog) as ctx:
        ctx.load_elts(*ea, wa.elt_terms())
        ctx.load_yet(wb.n_trials, 0, off, ids)
        ctx.run_host(wb.layers)
        ctx.load_elts(*eb, wb.elt_terms())
        ylt, lossy, _ = ctx.run_host(wb.layers)
    fresh, flossy, _, _ = run_gpu(off, ids, eb, wb, wb.layers)
    assert np.array_equal(ylt, fresh) and np.array_equal(lossy, flossy)
    orc = run_oracle(off, ids, eb, wb, wb.layers)
    assert_ylt_close(ylt, orc)


def test_set_elt_terms_equals_fresh_load(cuda):
    ara = _ara()
    w = synth.get_config("tiny")
    off, ids, elts = make_inputs(w)
    d, li = w.elt_terms()
    d2, li2 = d * 0.5, li * 2
    fresh, _, _, _ = run_gpu(off, ids, elts, w, w.layers, terms=(d2, li2))
    with ara.Context(w.catalog) as ctx:
        ctx.load_elts(*elts, terms=(d, li))
        ctx.load_yet(w.n_trials, 0, off, ids)
        a, _, _ = ctx.run_host(w.layers)
        ctx.set_elt_terms((d2, li2))
        b, _, _ = ctx.run_host(w.layers)
    assert np.array_equal(b, fresh) and not np.array_equal(a, b)


@pytest.mark.parametrize("rows_rho", [(1, 0.3), (3, 0.02)])
@pytest.mark.parametrize("graph", [0, 1])
def test_metrics_general_path_matches_oracle(cuda, rows_rho, graph):
    """The two launch sequences of the radix select — the fast path (n_rp <= 11:
    three full sweeps, then the 16-bit-prefix candidates; default) and the
    general one (ARA_METRICS_M3=1: eight full sweeps) — each give the oracle's PML
    (bit for bit) and TVaR, with and without the CUDA graph of the fast path."""
    n_layers, rho = rows_rho
    w = synth.get_config("tiny").with_(n_trials=5003, rho=rho, return_periods=(1, 2, 3.5, 10, 100, 1000, 5003))
    layers = tuple(synth.LayerSpec(0, 3, 2.5e4 * (i + 1), 5e5, 6.5e6 / (i + 1), 2.5e6) for i in range(n_layers))
    off, ids, elts = make_inputs(w)
    orc = run_oracle(off, ids, elts, w, layers)
    _, _, _, met = run_gpu(off, ids, elts, w, layers, return_periods=w.return_periods, env={"ARA_METRICS_M3": 1})
    _, _, _, met0 = run_gpu(off, ids, elts, w, layers, return_periods=w.return_periods, env={"ARA_METRICS_GRAPH": graph})
    assert_metrics_close(met, oracle_rows(orc), orc["scale"], w.return_periods)
    assert_metrics_close(met0, oracle_rows(orc), orc["scale"], w.return_periods)
    assert np.array_equal(met[1], met0[1]) and np.allclose(met[2], met0[2], rtol=1e-12, atol=0)


def test_metrics_many_return_periods(cuda):
    """n_rp = 40 (> 11: the general path) and 11 (the fast path's limit) on the
    same YLT: PML bit for bit, TVaR within tolerance of the oracle."""
    rps = tuple(float(x) for x in np.unique(np.geomspace(1, 5003, 40).round(2)))
    w = synth.get_config("tiny").with_(n_trials=5003, rho=0.2, return_periods=rps)
    off, ids, elts = make_inputs(w)
    orc = run_oracle(off, ids, elts, w, w.layers)
    _, _, _, met = run_gpu(off, ids, elts, w, w.layers, return_periods=rps)
    assert_metrics_close(met, oracle_rows(orc), orc["scale"], rps)
    _, _, _, met11 = run_gpu(off, ids, elts, w, w.layers, return_periods=rps[::4][:11])
    assert_metrics_close(met11, oracle_rows(orc), orc["scale"], rps[::4][:11])


def test_metrics_ties_extremes(cuda):
    """Many ties (capped and zero years) plus R = 1 (k = T, min / mean) and R = T (max)."""
    w = synth.get_config("tiny").with_(int_cap=2.0 ** 31)
    off, ids, elts = make_inputs(w)
    layers = (synth.LayerSpec(0, 3, 2.5e4, 5e5, 6.5e6, 2.5e5), synth.LayerSpec(0, 3, 0, INF, 0, INF))
    orc = run_oracle(off, ids, elts, w, layers)
    R = (1, 1.5, 2, 7.25, 999.9, 1000)
    _, _, _, met = run_gpu(off, ids, elts, w, layers, return_periods=R)
    assert (orc["ylt"][0] == 2.5e5).mean() > 0.2
    assert_metrics_close(met, oracle_rows(orc), orc["scale"], R, exact=True)


# ------------------------------------------------------------------ errors
@pytest.mark.parametrize("rho", [0.3, 0.02])   # 0.02: sparse table, the compacted-rounds kernel validates
def test_errors_are_reported_and_context_survives(cuda, rho):
    ara = _ara()
    w = synth.get_config("tiny").with_(rho=rho)
    off, ids, elts = make_inputs(w)
    eo, ev, ls = elts
    C = w.catalog
    with ara.Context(C) as ctx:
        with pytest.raises(ara.AraError) as e:
            ctx.run(w.layers)
        assert e.value.status == ara.ARA_ERR_STATE
        for bad_ev, bad_ls, status in ((np.where(np.arange(len(ev)) == 5, C + 1, ev).astype(np.uint32), ls,
                                        ara.ARA_ERR_OUT_OF_RANGE),
                                       (ev[::-1].copy(), ls, ara.ARA_ERR_INVALID_ARG),
                                       (ev, np.where(np.arange(len(ls)) == 3, -1.0, ls), ara.ARA_ERR_DOMAIN),
                                       (ev, np.where(np.arange(len(ls)) == 3, np.nan, ls), ara.ARA_ERR_DOMAIN)):
            with pytest.raises(ara.AraError) as e:
                ctx.load_elts(eo, bad_ev, bad_ls)
            assert e.value.status == status
        ctx.load_elts(eo, ev, ls, w.elt_terms())
        for bad in (0, C + 1):
            bi = ids.copy()
            bi[1234] = bad
            ctx.load_yet(w.n_trials, 0, off, bi)
            with pytest.raises(ara.AraError) as e:
                ctx.run(w.layers)
            assert e.value.status == ara.ARA_ERR_OUT_OF_RANGE
        bo = off.copy()
        bo[10], bo[11] = bo[11], bo[10]
        ctx.load_yet(w.n_trials, 0, bo, ids)
        with pytest.raises(ara.AraError) as e:
            ctx.run(w.layers)
        assert e.value.status == ara.ARA_ERR_OUT_OF_RANGE
        with pytest.raises(ara.AraError) as e:
            ctx.metrics([2.0])
        assert e.value.status == ara.ARA_ERR_STATE
        ctx.load_yet(w.n_trials, 0, off, ids)
        for L, status in (((0, 4, 0, 1, 0, 1),), ara.ARA_ERR_INVALID_ARG), (((1, 1, 0, 1, 0, 1),), ara.ARA_ERR_INVALID_ARG), \
                         (((0, 3, -1, 1, 0, 1),), ara.ARA_ERR_DOMAIN), (((0, 3, 0, 0.0, 0, 1),), ara.ARA_ERR_DOMAIN):
            with pytest.raises(ara.AraError) as e:
                ctx.run(L)
            assert e.value.status == status
        ylt, lossy, _ = ctx.run_host(w.layers)          # still usable
        orc = run_oracle(off, ids, elts, w, w.layers)
        assert_ylt_close(ylt, orc)
        with pytest.raises(ara.AraError) as e:
            ctx.metrics([w.n_trials + 1.0])
        assert e.value.status == ara.ARA_ERR_DOMAIN


@pytest.mark.parametrize("load_mode,chunk", [("all", 0), ("chunked", 1), ("chunked", 37), ("chunked", 10 ** 6)])
def test_packed_yet_transfer_equals_u32(cuda, load_mode, chunk):
    """F3: bit-packed ids (14/21/32 bits) through host or device memory give the
    same YLT bits as u32 ids; chunk boundaries split words."""
    import torch
    from paper_1606_04473_b200 import ara
    w = synth.get_config("tiny").with_(n_trials=1500)
    off, ids, elts = make_inputs(w)
    ref, ref_lossy, _, _ = run_gpu(off, ids, elts, w, w.layers)
    orc = run_oracle(off, ids, elts, w, w.layers)
    for bits in (ara.bits_for_catalog(w.catalog), 21, 32):
        packed = ara.ara_pack_ids(ids, bits)
        for device in (False, True):
            src = torch.from_numpy(packed.view(np.int32)).cuda() if device else packed
            with ara.Context(w.catalog, load_mode=load_mode, chunk_trials=chunk) as ctx:
                ctx.load_elts(*elts, terms=w.elt_terms())
                ctx.load_yet_packed(w.n_trials, 0, off, src, bits)
                ylt, lossy, st = ctx.run_host(w.layers)
                met = ctx.metrics((2, 10, 100))
            assert_ylt_close(ylt, orc)                               # the oracle decides
            assert np.array_equal(lossy, orc["lossy"]), (bits, device)
            assert_metrics_close(met, oracle_rows(orc), orc["scale"], (2, 10, 100))
            assert np.array_equal(ylt, ref) and np.array_equal(lossy, ref_lossy), (bits, device)
            if load_mode == "chunked" and not device:
                assert st["h2d_bytes"] < ids.nbytes + off.nbytes or bits == 32


def test_packed_out_of_range_id_reported(cuda):
    from paper_1606_04473_b200 import ara
    w = synth.get_config("tiny")
    off, ids, elts = make_inputs(w)
    bad = ids.copy()
    bad[777] = w.catalog + 5
    with ara.Context(w.catalog, load_mode="chunked", chunk_trials=100) as ctx:
        ctx.load_elts(*elts)
        ctx.load_yet_packed(w.n_trials, 0, off, ara.ara_pack_ids(bad, 14), 14)
        with pytest.raises(ara.AraError) as e:
            ctx.run(w.layers)
        assert e.value.status == ara.ARA_ERR_OUT_OF_RANGE


@pytest.mark.parametrize("run_mode", ["direct", "fold"])
def test_portfolio_programs_and_explicit_elt_lists(cuda, run_mode):
    """F4: programs of layers with explicit (non-contiguous, ascending) ELT
    lists, including a >8-sector list (generic kernel); YLT rows = layers,
    programs, portfolio; metrics over every row."""
    w = synth.get_config("tiny").with_(n_elts=48, catalog=4000, rho=0.2, n_trials=800, nmin=0, nmax=200)
    off, ids, elts = make_inputs(w)
    d, li = w.elt_terms()
    progs = [
        [([0, 2, 5, 9, 14], 2.5e4, 5e5, 6.5e5, 2.5e6), ([1, 3], 0.0, INF, 0.0, INF)],
        [([20, 21, 22, 23, 24, 25, 26, 27, 28, 29, 30, 31, 32, 33, 34, 35], 1e4, 1e6, 1e5, 8e6)],
        [([4, 40, 47], 5e4, 2e5, 2e5, INF), ([6, 7, 8], 0.0, 3e5, 0.0, 5e6), (list(range(0, 48, 2)), 1e5, 1e6, 3e5, INF)],
    ]
    flat = [L for p in progs for L in p]
    orc = oracle.ara(off, ids, oracle.Elts(*elts), w.catalog, d, li, flat, lookup="dense")
    pl = np.cumsum([0] + [len(p) for p in progs])
    orc_prog = oracle.programs(orc["ylt"], pl)
    from paper_1606_04473_b200 import ara
    with ara.Context(w.catalog, run_mode=run_mode) as ctx:
        ctx.load_elts(*elts, terms=(d, li))
        ctx.load_yet(w.n_trials, 0, off, ids)
        ylt, lossy, st = ctx.run_portfolio_host(progs)
        k, pml, tvar, _ = ctx.metrics((2, 10, 100))
    L, P = len(flat), len(progs)
    assert ylt.shape == (L + P + 1, w.n_trials) and pml.shape == (L + P + 1, 3)
    tol = RTOL * np.maximum(orc["scale"], 1.0)
    assert (np.abs(ylt[:L] - orc["ylt"]) <= tol).all()
    assert np.array_equal(lossy, orc["lossy"])
    for q in range(P):
        assert (np.abs(ylt[L + q] - orc_prog[q]) <= tol[pl[q]:pl[q + 1]].sum(axis=0)).all()
    assert (np.abs(ylt[L + P] - orc["portfolio"]) <= tol.sum(axis=0)).all()
    for r in range(L + P + 1):
        kk, p_o, _ = oracle.metrics(ylt[r], (2, 10, 100))
        assert np.array_equal(p_o, pml[r]) and np.array_equal(kk, k)


@pytest.mark.parametrize("variant", (-1, 30))
@pytest.mark.parametrize("precision", ("f64", "f32"))
def test_packed_rows_overflow_and_offset_windows(cuda, variant, precision):
    """Packed rows (trial_kernel_bc): a sparse block whose first 400 rows are
    non-zero in EVERY ELT, so those rows hold more non-zeros than a packed slot
    (3 fp64 / 6 fp32 values) and the rest are read from the dense table; layers
    whose window starts inside the block (the slot mask is shifted), a window
    over the block's tail, and one spanning two fp64 blocks (no bitmap).  Must
    match the oracle, with and without skipping."""
    rng = np.random.default_rng(17)
    w = synth.get_config("tiny").with_(catalog=20000, n_elts=20, n_trials=600, nmin=1, nmax=250)
    off, ids = synth.gen_yet(w)
    eo, ev, ls = [0], [], []
    for j in range(w.n_elts):
        tail = rng.choice(np.arange(401, w.catalog + 1), 200, replace=False)
        e = np.unique(np.concatenate([np.arange(1, 401), tail])).astype(np.uint32)
        ev.append(e)
        ls.append(np.floor(rng.lognormal(np.log(5e4), 1.5, len(e))))
        eo.append(eo[-1] + len(e))
    elts = (np.array(eo, dtype=np.uint64), np.concatenate(ev), np.concatenate(ls))
    d = rng.uniform(0, 2e4, w.n_elts)
    li = np.where(rng.random(w.n_elts) < 0.3, INF, rng.uniform(1e5, 2e6, w.n_elts))
    layers = (synth.LayerSpec(0, 16, 2.5e4, 7.5e5, 1.2e6, 8e6), synth.LayerSpec(4, 12, 1e4, 4e5, 6.5e5, 4e6),
              synth.LayerSpec(16, 20, 0.0, INF, 1e5, INF), synth.LayerSpec(0, 20, 2.5e5, 5e5, 4e5, 3.5e6))
    orc = run_oracle(off, ids, elts, w, layers, fp32=precision == "f32", terms=(d, li))
    ylt, lossy, st, _ = run_gpu(off, ids, elts, w, layers, precision=precision, terms=(d, li), variant=variant)
    assert_ylt_close(ylt, orc)
    assert np.array_equal(lossy, orc["lossy"])
    ylt2, lossy2, _, _ = run_gpu(off, ids, elts, w, layers, precision=precision, terms=(d, li), variant=variant,
                                 env={"ARA_NO_SKIP": 1})
    assert_ylt_close(ylt2, orc)
    assert np.array_equal(lossy2, orc["lossy"])


@pytest.mark.parametrize("variant", (30,))
@pytest.mark.parametrize("rho", (0.01, 0.1, 0.3))
def test_cross_trial_rounds_short_and_empty_trials(cuda, variant, rho):
    """Deferred trial finalisation (trial_kernel_bc): many short, empty and
    long trials back to back, so a trial's last round is finished while the
    next trials scan, trials without occupied events are finalised between
    rounds, and several trials share one 128-event batch.  Within tolerance of
    the oracle, with and without skipping; integer-valued data bit for bit."""
    rng = np.random.default_rng(21)
    w = synth.get_config("tiny").with_(catalog=4000, rho=rho, n_trials=8)
    _, _, elts = make_inputs(w)
    occupied = np.unique(elts[1])
    lens = rng.choice([0, 1, 2, 3, 5, 31, 32, 33, 127, 128, 129, 700], size=1500)
    trials = []
    for i, n in enumerate(lens):
        if i % 7 == 3:
            trials.append(rng.choice(occupied, n))             # every event occupied
        else:
            trials.append(rng.integers(1, w.catalog + 1, n))   # random
    off = np.zeros(len(trials) + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(t) for t in trials])
    ids = np.concatenate(trials).astype(np.uint32)
    w = w.with_(n_trials=len(trials))
    orc = run_oracle(off, ids, elts, w, w.layers)
    ylt, lossy, st, _ = run_gpu(off, ids, elts, w, w.layers, variant=variant)
    assert_ylt_close(ylt, orc)
    assert np.array_equal(lossy, orc["lossy"])
    ylt0, lossy0, _, _ = run_gpu(off, ids, elts, w, w.layers, variant=variant, env={"ARA_NO_SKIP": 1})
    assert_ylt_close(ylt0, orc)
    assert np.array_equal(lossy0, orc["lossy"])
    wi = w.with_(int_cap=2.0 ** 31)
    elts_i = synth.gen_elts(wi)
    orc_i = run_oracle(off, ids, elts_i, wi, wi.layers)
    ylt_i, lossy_i, _, _ = run_gpu(off, ids, elts_i, wi, wi.layers, variant=variant)
    assert np.array_equal(ylt_i[:-1], orc_i["ylt"]) and np.array_equal(ylt_i[-1], orc_i["portfolio"])
    assert np.array_equal(lossy_i, orc_i["lossy"])


@pytest.mark.parametrize("rho", [0.02, 1.0])
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_l2_persisting_window(cuda, rho, precision):
    """cfg.l2_persist: an L2 access-policy window over the packed rows (sparse
    kernel) or the layer's column block (dense kernels) during ara_run --
    a cache hint only: the oracle's YLT and counts, and the same bits as
    without the window."""
    w = synth.get_config("tiny").with_(rho=rho, n_trials=2000, catalog=50_000, n_elts=6)
    off, ids, elts = make_inputs(w)
    orc = run_oracle(off, ids, elts, w, w.layers, fp32=precision == "f32")
    ylt, lossy, _, met = run_gpu(off, ids, elts, w, w.layers, precision=precision, return_periods=(2, 10),
                                 l2_persist=True)
    assert_ylt_close(ylt, orc)
    assert np.array_equal(lossy, orc["lossy"])
    ref, ref_lossy, _, _ = run_gpu(off, ids, elts, w, w.layers, precision=precision)
    assert np.array_equal(ylt, ref) and np.array_equal(lossy, ref_lossy)


@pytest.mark.parametrize("rho", [0.02, 0.3])
@pytest.mark.parametrize("catalog", [10_014, 10_000])
def test_out_of_range_ids_everywhere(cuda, rho, catalog):
    """A14: an id outside [1, C] -- 0, C + 1 (the sparse kernel's clamp target,
    a never-set padding bit of the bitmap), C + 2 and 2^32 - 1 -- is reported
    wherever it sits: a trial's first or last event (partially covered
    batches) or the middle of a trial (fully covered batches), with C + 2 a
    multiple of 32 (the padding bit is the first bit of a word) or not.  The
    context stays usable and matches the oracle afterwards."""
    ara = _ara()
    w = synth.get_config("tiny").with_(rho=rho, catalog=catalog)
    off, ids, elts = make_inputs(w)
    C = w.catalog
    t = 37
    positions = (int(off[t]), int(off[t + 1]) - 1, int(off[t]) + (int(off[t + 1]) - int(off[t])) // 2)
    with ara.Context(C) as ctx:
        ctx.load_elts(*elts, terms=w.elt_terms())
        for bad in (0, C + 1, C + 2, 0xFFFFFFFF):
            for pos in positions:
                bi = ids.copy()
                bi[pos] = bad
                ctx.load_yet(w.n_trials, 0, off, bi)
                with pytest.raises(ara.AraError) as e:
                    ctx.run(w.layers)
                assert e.value.status == ara.ARA_ERR_OUT_OF_RANGE, (bad, pos)
        ctx.load_yet(w.n_trials, 0, off, ids)
        ylt, lossy, _ = ctx.run_host(w.layers)
    orc = run_oracle(off, ids, elts, w, w.layers)
    assert_ylt_close(ylt, orc)
    assert np.array_equal(lossy, orc["lossy"])
