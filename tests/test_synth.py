"""Generator checks: determinism, shapes and ranges of the paper's inputs."""
import numpy as np

import synth


def test_yet_deterministic_and_in_range():
    w = synth.get_config("tiny")
    a = synth.gen_yet(w)
    b = synth.gen_yet(w)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    off, ids = a
    n = np.diff(off)
    assert off[0] == 0 and len(off) == w.n_trials + 1
    assert n.min() >= w.nmin and n.max() <= w.nmax
    assert ids.min() >= 1 and ids.max() <= w.catalog
    assert abs(n.mean() - w.mean_events) < 2


def test_sub_range_and_sample_regenerate_independently():
    w = synth.get_config("tiny").with_(n_trials=500)
    off, ids = synth.gen_yet(w)
    so, si = synth.gen_yet(w, first=123, n=77)
    assert np.array_equal(si, ids[int(off[123]):int(off[200])])
    assert np.array_equal(so, off[123:201] - off[123])
    pick = [499, 0, 17, 17, 250]
    po, pi = synth.gen_trial_sample(w, pick)
    for i, t in enumerate(pick):
        assert np.array_equal(pi[int(po[i]):int(po[i + 1])], ids[int(off[t]):int(off[t + 1])])


def test_multithreaded_events_equal_single_threaded():
    w = synth.get_config("paper")
    a = synth.gen_events(w, 10_000, 3_000_000, nthreads=1)
    b = synth.gen_events(w, 10_000, 3_000_000, nthreads=8)
    assert np.array_equal(a, b)


def test_elts_sorted_unique_and_lognormal():
    w = synth.get_config("tiny")
    off, ev, ls = synth.gen_elts(w)
    assert len(off) == w.n_elts + 1
    for j in range(w.n_elts):
        e = ev[int(off[j]):int(off[j + 1])]
        assert (np.diff(e.astype(np.int64)) > 0).all() and e.min() >= 1 and e.max() <= w.catalog
        assert abs(len(e) / w.catalog - w.rho) < 0.02
    lg = np.log(ls)
    assert abs(lg.mean() - w.mu) < 0.05 and abs(lg.std() - w.sigma) < 0.05
    wi = w.with_(int_cap=2.0 ** 24)
    _, _, li = synth.gen_elts(wi)
    assert (li == np.floor(li)).all() and li.max() < 2 ** 24


def test_timestamps_sorted_unit_interval():
    w = synth.get_config("tiny")
    ts = synth.gen_timestamps(w, 5, 1000)
    assert (np.diff(ts) > 0).all() and ts[0] >= 0 and ts[-1] < 1
