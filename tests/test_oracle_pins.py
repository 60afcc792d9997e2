"""Pins for the CPU oracle, all CPU-only.

Each test checks the oracle against something other than itself: values
worked by hand from the paper's formulas (tests/golden/), closed forms,
invariants that are exact in fp64, or brute force on tiny inputs.  The
comment on each test names the plausible oracle mistake it would catch.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")
INF = math.inf


def _lim(x):
    return INF if x is None else float(x)


# ---------------------------------------------------------------- term formula
def test_term_examples():
    """P4. Catches swapped retention/limit, min/max, missing floor."""
    rows = []
    for line in open(os.path.join(GOLD, "term_examples.txt")):
        line = line.split("#")[0].strip()
        if line:
            rows.append([float(v) for v in line.split()])
    assert len(rows) == 6
    for loss, r, lim, want in rows:
        assert oracle.apply_terms(loss, r, lim) == want


def test_term_identity_and_properties():
    """identity at (0, inf); monotone, bounded in [0, limit] on 10k inputs."""
    rng = np.random.default_rng(1)
    xs = rng.lognormal(10, 2, 10_000)
    for x in xs[:200]:
        assert oracle.apply_terms(x, 0.0, INF) == x
    for _ in range(10_000 // 50):
        r, lim = rng.uniform(0, 1e5), rng.uniform(1, 1e5)
        v = sorted(rng.lognormal(10, 2, 50))
        out = [oracle.apply_terms(x, r, lim) for x in v]
        assert all(0.0 <= o <= lim for o in out)
        assert all(a <= b for a, b in zip(out, out[1:]))


# ---------------------------------------------------------- worked examples
def _run_case(elts_maps, catalog, case):
    elts = oracle.Elts.from_maps([{int(k): v for k, v in m.items()} for m in elts_maps])
    ded = [float(t[0]) for t in case["elt_terms"]]
    lim = [_lim(t[1]) for t in case["elt_terms"]]
    layers = [(L["elts"], float(L["occ"][0]), _lim(L["occ"][1]),
               float(L["agg"][0]), _lim(L["agg"][1])) for L in case["layers"]]
    off = [0, len(case["trial"])]
    return oracle.ara(off, case["trial"], elts, catalog, ded, lim, layers)


@pytest.mark.parametrize("lookup", ["map", "dense"])
def test_worked_trials(lookup):
    """P1, P2, P3.  Catches: occurrence terms applied to the
    trial sum instead of per event (A2), per-ELT terms dropped, repeated events
    de-duplicated (A7), portfolio not summed over layers (A8)."""
    g = json.load(open(os.path.join(GOLD, "worked_trials.json")))
    for case in g["cases"]:
        r = _run_case(g["elts"], g["catalog"], case)
        assert list(r["ylt"][:, 0]) == case["ylt"], case["pin"]
        assert list(r["scale"][:, 0]) == case["scale"], case["pin"]
        assert list(r["lossy"][:, 0]) == case["lossy"], case["pin"]
        assert r["portfolio"][0] == case["portfolio"], case["pin"]


def test_direct_access_examples():
    """P5.  Catches off-by-one event indexing in the dense table."""
    e = oracle.Elts.from_maps([{2: 5.0}])
    assert list(oracle.direct_access(e, 3)[0, 1:]) == [0.0, 5.0, 0.0]
    e = oracle.Elts.from_maps([{}])
    assert list(oracle.direct_access(e, 2)[0, 1:]) == [0.0, 0.0]
    e = oracle.Elts.from_maps([{1: 1.0, 3: 2.0}])
    assert oracle.lookup_map(e, 0, 2) == 0.0
    assert oracle.direct_access(e, 3)[0, 2] == 0.0
    with pytest.raises(ValueError):
        oracle.direct_access(oracle.Elts.from_maps([{4: 1.0}]), 3)


def test_dense_equals_map_exhaustive():
    """S:99 dense-table lookup == map lookup for every id, and whole-run
    equality of the two lookup modes (bitwise)."""
    rng = np.random.default_rng(7)
    C = 300
    maps = []
    for j in range(5):
        ks = rng.choice(np.arange(1, C + 1), size=int(rng.integers(0, 120)), replace=False)
        maps.append({int(k): float(rng.lognormal(8, 1)) for k in ks})
    e = oracle.Elts.from_maps(maps)
    dense = oracle.direct_access(e, C)
    for j, m in enumerate(maps):
        for ev in range(1, C + 1):
            assert oracle.lookup_map(e, j, ev) == m.get(ev, 0.0) == dense[j, ev]
    off = np.array([0, 5, 5, 40, 41, 200], dtype=np.uint64)
    ids = rng.integers(1, C + 1, size=200).astype(np.uint32)
    lay = [([0, 2, 4], 10.0, 5e3, 100.0, 2e4), ([1, 3], 0.0, INF, 0.0, INF)]
    d = np.full(5, 50.0)
    li = np.full(5, 3e3)
    a = oracle.ara(off, ids, e, C, d, li, lay, lookup="map")
    b = oracle.ara(off, ids, e, C, d, li, lay, lookup="dense", dense=dense)
    for k in a:
        assert np.array_equal(a[k], b[k])


def test_out_of_range_event_rejected():
    """A14: ids are 1-based within [1, C]; 0 and C+1 are errors."""
    e = oracle.Elts.from_maps([{1: 1.0}])
    for bad in (0, 4):
        with pytest.raises(ValueError):
            oracle.ara([0, 1], [bad], e, 3, [0.0], [INF], [([0], 0.0, INF, 0.0, INF)])


# ------------------------------------------------------------------ metrics
def test_metrics_examples():
    """P6 (S:209-216 + tie cases).  Catches 0- vs 1-based rank, floor vs ceil,
    ascending sort, TVaR over k-1 or k+1 values."""
    g = json.load(open(os.path.join(GOLD, "metrics_examples.json")))
    for c in g["cases"]:
        k, pml, tvar = oracle.metrics(c["ylt"], [c["R"]])
        assert int(k[0]) == c["k"], c
        assert pml[0] == c["pml"], c
        want = c["tvar"] if "tvar" in c else c["tvar_num"] / c["tvar_den"]
        assert tvar[0] == want, c


def _brute(y, R):
    """Order statistics by counting (P7): PML is the unique v with
    #{Y > v} < k <= #{Y >= v}; TVaR = (sum_{Y>v} Y + (k - #{Y>v}) v) / k."""
    T = len(y)
    k = math.ceil(Fraction(T) / Fraction(R))
    cands = sorted(set(y))
    v = [c for c in cands if sum(1 for x in y if x > c) < k <= sum(1 for x in y if x >= c)]
    assert len(v) == 1
    v = v[0]
    gt = [x for x in y if x > v]
    tv = Fraction(sum(Fraction(x) for x in gt) + (k - len(gt)) * Fraction(v), k)
    return k, v, tv


def test_metrics_bruteforce_2000():
    """P7: 2,000 random tiny integer YLTs (many ties), integer and non-integer R."""
    rng = np.random.default_rng(11)
    for it in range(2000):
        T = int(rng.integers(1, 40))
        y = [float(v) for v in rng.integers(0, 8, size=T) * int(rng.integers(1, 1000))]
        R = float(rng.integers(1, T + 1)) if it % 2 == 0 else float(rng.uniform(1.0, T))
        k, pml, tvar = oracle.metrics(y, [R])
        bk, bv, btv = _brute(y, R)
        assert int(k[0]) == bk and pml[0] == bv
        assert tvar[0] == float(btv)        # exact: integer sums < 2^53, one rounding


def test_rank_domain_and_extremes():
    """P12: R = T -> k = 1 -> max; R = 1 -> k = T -> min, TVaR = mean; R outside [1,T] -> error."""
    y = [3.0, 9.0, 1.0, 4.0, 4.0]
    k, pml, tvar = oracle.metrics(y, [5, 1])
    assert list(k) == [1, 5] and pml[0] == 9.0 and pml[1] == 1.0 and tvar[1] == 21.0 / 5
    assert oracle.rank(10, 3) == 4 and oracle.rank(10, 2.5) == 4 and oracle.rank(10, 3.3) == 4
    assert oracle.rank(1_000_000, 3) == 333_334
    for bad in (0.5, 11, -1):
        assert oracle.rank(10, bad) == 0
        with pytest.raises(ValueError):
            oracle.metrics(np.zeros(10), [bad])


# ------------------------------------------------- closed forms on synthetic data
def _small(name="tiny", **kw):
    w = synth.get_config(name).with_(**kw)
    off, ids = synth.gen_yet(w)
    eo, ev, ls = synth.gen_elts(w)
    return w, off, ids, oracle.Elts(eo, ev, ls)


def _dense_rows(w, elts):
    return oracle.direct_access(elts, w.catalog)            # [E][C+1]


def test_identity_terms_mass_conservation():
    """P8: zero retentions, infinite limits -> Y_t = sum of raw ELT losses of the
    trial's events; globally sum_t Y_t = sum_e N_e rowsum(e) (exact on
    integer-valued data).  Catches a dropped ELT, a dropped event, or a wrong
    lookup index."""
    w, off, ids, e = _small(int_cap=2.0**31)
    E = w.n_elts
    r = oracle.ara(off, ids, e, w.catalog, np.zeros(E), np.full(E, INF),
                   [(list(range(E)), 0.0, INF, 0.0, INF)])
    rowsum = _dense_rows(w, e).sum(axis=0)                  # exact: integers < 2^53
    per_trial = np.add.reduceat(rowsum[ids], off[:-1].astype(np.int64)) if len(ids) else []
    empty = off[1:] == off[:-1]
    per_trial = np.where(empty, 0.0, per_trial)
    assert np.array_equal(r["ylt"][0], per_trial)
    N = np.bincount(ids, minlength=w.catalog + 1)
    assert r["ylt"][0].sum() == float((N * rowsum).sum())
    assert np.array_equal(r["scale"][0], r["ylt"][0])


def test_occurrence_limit_counts_lossy_events():
    """OccR = 0, OccL = 0.5 below every positive integer loss: Y_t = 0.5 m_t and
    m_t = #{events with a positive combined loss}.  Catches m counting the
    wrong condition and OccL not applied per event."""
    w, off, ids, e = _small(int_cap=2.0**31)
    E = w.n_elts
    r = oracle.ara(off, ids, e, w.catalog, np.zeros(E), np.full(E, INF),
                   [(list(range(E)), 0.0, 0.5, 0.0, INF)])
    pos = (_dense_rows(w, e).sum(axis=0) > 0).astype(np.int64)
    m = np.array([pos[ids[a:b]].sum() for a, b in zip(off[:-1], off[1:])])
    assert np.array_equal(r["lossy"][0], m)
    assert np.array_equal(r["ylt"][0], 0.5 * m)


def test_elt_limit_counts_records():
    """Per-ELT D = 0, Lim = 0.5: Y_t = 0.5 * sum_e #{j : L_j[e] > 0}.  Catches
    per-ELT terms applied to the combined loss instead of each lookup (A5)."""
    w, off, ids, e = _small(int_cap=2.0**31)
    E = w.n_elts
    r = oracle.ara(off, ids, e, w.catalog, np.zeros(E), np.full(E, 0.5),
                   [(list(range(E)), 0.0, INF, 0.0, INF)])
    cnt = (_dense_rows(w, e) > 0).sum(axis=0)
    want = np.array([0.5 * cnt[ids[a:b]].sum() for a, b in zip(off[:-1], off[1:])])
    assert np.array_equal(r["ylt"][0], want)


def test_deductible_above_every_loss_gives_zero():
    w, off, ids, e = _small()
    E = w.n_elts
    r = oracle.ara(off, ids, e, w.catalog, np.full(E, 1e300), np.full(E, INF),
                   [(list(range(E)), 0.0, INF, 0.0, INF)])
    assert not r["ylt"].any() and not r["scale"].any() and not r["lossy"].any()


def test_single_event_single_elt_is_lookup():
    """P12: one ELT, one event per trial, identity terms -> Y_t = L[e_t]."""
    w, _, _, e = _small()
    rng = np.random.default_rng(5)
    ids = rng.integers(1, w.catalog + 1, size=500).astype(np.uint32)
    off = np.arange(501, dtype=np.uint64)
    dense = _dense_rows(w, e)
    for j in range(w.n_elts):
        r = oracle.ara(off, ids, e, w.catalog, np.zeros(w.n_elts), np.full(w.n_elts, INF),
                       [([j], 0.0, INF, 0.0, INF)])
        assert np.array_equal(r["ylt"][0], dense[j, ids])


def test_bounds_and_monotone_in_every_retention():
    """P9: 0 <= Y <= AggL exactly; raising D_j, OccR or AggR never raises any
    Y_t (exact in fp64 for a fixed order).  Catches a sign error on a retention."""
    w, off, ids, e = _small()
    lay = [s for s in oracle.layers_from_specs(w.layers)]
    d, li = w.elt_terms()
    base = oracle.ara(off, ids, e, w.catalog, d, li, lay)["ylt"][0]
    aggl = lay[0][4]
    assert (base >= 0).all() and (base <= aggl).all()
    assert 0 < (base == aggl).mean() < 1 and 0 < (base == 0).mean() < 1
    for j in range(w.n_elts):
        d2 = d.copy()
        d2[j] *= 3
        y = oracle.ara(off, ids, e, w.catalog, d2, li, lay)["ylt"][0]
        assert (y <= base).all() and (y < base).any()
    (el, occr, occl, aggr, aggl) = lay[0]
    for bumped in ([(el, occr * 2, occl, aggr, aggl)], [(el, occr, occl, aggr * 1.5, aggl)]):
        y = oracle.ara(off, ids, e, w.catalog, d, li, bumped)["ylt"][0]
        assert (y <= base).all() and (y < base).any()


def test_partition_invariance():
    """P11 (S:223, S:523 #7): shards over N in {1,2,4,8,16} concatenated by
    trial index == unsharded, bitwise."""
    w, off, ids, e = _small()
    lay = oracle.layers_from_specs(w.layers)
    d, li = w.elt_terms()
    full = oracle.ara(off, ids, e, w.catalog, d, li, lay)
    T = w.n_trials
    for N in (1, 2, 4, 8, 16):
        parts = []
        for r in range(N):
            q, rem = divmod(T, N)
            a = r * q + min(r, rem)
            b = a + q + (1 if r < rem else 0)
            sub_off = off[a:b + 1]
            sub_ids = ids[int(off[a]):int(off[b])]
            parts.append(oracle.ara(sub_off, sub_ids, e, w.catalog, d, li, lay)["ylt"])
        assert np.array_equal(np.concatenate(parts, axis=1), full["ylt"])


def test_identity_terms_permutation_invariant():
    """identity terms -> invariant under event permutation (exact on integers)."""
    w, off, ids, e = _small(int_cap=2.0**31)
    E = w.n_elts
    lay = [(list(range(E)), 0.0, INF, 0.0, INF)]
    a = oracle.ara(off, ids, e, w.catalog, np.zeros(E), np.full(E, INF), lay)["ylt"]
    rng = np.random.default_rng(3)
    ids2 = ids.copy()
    for s, t in zip(off[:-1], off[1:]):
        rng.shuffle(ids2[int(s):int(t)])
    b = oracle.ara(off, ids2, e, w.catalog, np.zeros(E), np.full(E, INF), lay)["ylt"]
    assert np.array_equal(a, b)


def test_fp32_storage_reads_rounded_losses():
    """A13: the fp32-storage oracle == the fp64 oracle on losses pre-rounded to fp32."""
    w, off, ids, e = _small()
    lay = oracle.layers_from_specs(w.layers)
    d, li = w.elt_terms()
    a = oracle.ara(off, ids, e, w.catalog, d, li, lay, fp32_storage=True)
    e32 = oracle.Elts(e.offsets, e.event_ids, e.losses.astype(np.float32).astype(np.float64))
    b = oracle.ara(off, ids, e32, w.catalog, d, li, lay)
    assert not np.array_equal(e.losses, e32.losses)
    for k in a:
        assert np.array_equal(a[k], b[k])


def test_aggregate_terms_special_case():
    """Identity per-ELT and occurrence terms reduce the year loss to the
    aggregate term formula of the raw trial sum."""
    w, off, ids, e = _small(int_cap=2.0**31)
    E = w.n_elts
    raw = oracle.ara(off, ids, e, w.catalog, np.zeros(E), np.full(E, INF),
                     [(list(range(E)), 0.0, INF, 0.0, INF)])["ylt"][0]
    aggr, aggl = float(np.median(raw)), float(np.percentile(raw, 90) - np.median(raw))
    y = oracle.ara(off, ids, e, w.catalog, np.zeros(E), np.full(E, INF),
                   [(list(range(E)), 0.0, INF, aggr, aggl)])["ylt"][0]
    assert np.array_equal(y, np.minimum(np.maximum(raw - aggr, 0.0), aggl))


def test_programs_closed_forms():
    """Programs: a program of one layer is that layer's row; on
    integer-valued data the program rows sum (exactly) to the portfolio of all
    layers; malformed program lists are rejected.  Catches an off-by-one layer
    range or a program summing the wrong rows."""
    w, off, ids, e = _small(int_cap=2.0 ** 31)
    d, li = w.elt_terms()
    lay = [([0, 1, 2], 2.5e4, 5e5, 6.5e5, 2.5e6), ([1], 0.0, INF, 0.0, INF), ([0, 2], 1e4, 1e5, 0.0, 1e6),
           ([2], 5e3, INF, 1e5, INF)]
    r = oracle.ara(off, ids, e, w.catalog, d, li, lay)
    single = oracle.programs(r["ylt"], [0, 1, 2, 3, 4])
    assert np.array_equal(single, r["ylt"])
    two = oracle.programs(r["ylt"], [0, 1, 4])
    assert np.array_equal(two[0], r["ylt"][0])
    assert np.array_equal(two[0] + two[1], r["portfolio"])
    assert np.array_equal(two[1], r["ylt"][1] + r["ylt"][2] + r["ylt"][3])
    for bad in ([0, 2, 2, 4], [1, 4], [0, 3]):
        with pytest.raises(ValueError):
            oracle.programs(r["ylt"], bad)


# ------------------------------------------------- EP curve
def test_ep_counts_against_sorted_search_and_pml():
    """A23: counts[i] = #{t : y[t] > x_i}.  Pinned against an independent
    method (binary search in the sorted YLT), closed forms (a threshold below
    every loss counts all T years, one at or above the maximum counts none,
    thresholds at each distinct loss count the strictly larger ones), the
    curve's monotonicity, and its relation to the oracle's PML: with
    k = ceil(T/R), #{Y > PML(R)} < k <= #{Y >= PML(R)}.  Catches >= for >,
    an off-by-one count, a reversed threshold order."""
    rng = np.random.default_rng(23)
    for it in range(300):
        T = int(rng.integers(1, 60))
        y = rng.integers(0, 9, size=T).astype(np.float64) * float(rng.choice([1.0, 0.5, 1e6]))
        x = np.sort(np.concatenate([rng.uniform(-1, y.max() + 1, 5), y[: min(T, 4)], [-1.0, y.max()]]))
        got = oracle.ep_counts(y, x)
        s = np.sort(y)
        want = T - np.searchsorted(s, x, side="right")      # #{y > x}
        assert np.array_equal(got, want)
        assert got[0] == T and got[-1] == 0                  # x = -1 and x = max
        assert (np.diff(got.astype(np.int64)) <= 0).all()     # non-increasing in x
        R = float(rng.integers(1, T + 1))
        k, pml, _ = oracle.metrics(y, [R])
        above = int(oracle.ep_counts(y, [pml[0]])[0])
        at_or_above = T - int(np.searchsorted(s, pml[0], side="left"))
        assert above < int(k[0]) <= at_or_above
