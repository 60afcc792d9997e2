"""Seeded synthetic inputs for the ARA hot path (YET + ELTs).

This package is the ONLY code shared by the oracle side and the CUDA side, and
it holds none of the method's arithmetic: it draws event ids, events-per-trial
counts and ELT (event, loss) records, nothing else.  See ``synth.h`` for the
stream definitions and DESIGN.md "Input recipe" for the distributions
(§IV-A).
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field, replace
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libsynth.so")
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run `make` (or __graft_entry__.build())")
        L = ctypes.CDLL(path)
        u64, u32, i32, dbl, vp = (ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int,
                                  ctypes.c_double, ctypes.c_void_p)
        L.synth_u64.restype = u64
        L.synth_u64.argtypes = [u64, u64, u64]
        L.synth_trial_counts.argtypes = [u64, u64, u64, u32, u32, vp]
        L.synth_event_base.restype = u64
        L.synth_event_base.argtypes = [u64, u64, u32, u32]
        L.synth_yet_offsets.restype = u64
        L.synth_yet_offsets.argtypes = [u64, u64, u64, u32, u32, vp]
        L.synth_yet_events.argtypes = [u64, u32, u64, u64, vp, i32]
        L.synth_trial_timestamps.argtypes = [u64, u64, u32, vp]
        L.synth_elt_count.restype = u64
        L.synth_elt_count.argtypes = [u64, u32, u32, dbl]
        L.synth_elt_fill.argtypes = [u64, u32, u32, dbl, dbl, dbl, dbl, vp, vp]
        _LIB = L
    return _LIB


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


@dataclass(frozen=True)
class LayerSpec:
    """One layer L = (E, T) (Eq. 3): a contiguous ELT range plus the
    occurrence/aggregate terms."""
    elt_begin: int
    elt_end: int
    occ_retention: float
    occ_limit: float
    agg_retention: float
    agg_limit: float


@dataclass(frozen=True)
class Workload:
    name: str
    seed: int
    n_trials: int
    nmin: int
    nmax: int
    catalog: int
    n_elts: int
    rho: float
    layers: Tuple[LayerSpec, ...]
    elt_deductible: float = 1e4          # per-ELT terms I = (D, Lim) (reading A3)
    elt_limit: float = 1e6
    mu: float = math.log(5e4)            # LogNormal(ln 5e4, 1.5) losses
    sigma: float = 1.5
    int_cap: float = 0.0                 # >0: integer-valued losses < int_cap (P10)
    return_periods: Tuple[float, ...] = (2, 5, 10, 25, 50, 100, 200, 250, 500, 1000)

    def with_(self, **kw) -> "Workload":
        return replace(self, **kw)

    def elt_terms(self) -> Tuple[np.ndarray, np.ndarray]:
        d = np.full(self.n_elts, self.elt_deductible, dtype=np.float64)
        l = np.full(self.n_elts, self.elt_limit, dtype=np.float64)
        return d, l

    @property
    def mean_events(self) -> float:
        return 0.5 * (self.nmin + self.nmax)


def gen_counts(w: Workload, first: int = 0, n: Optional[int] = None) -> np.ndarray:
    n = w.n_trials - first if n is None else n
    c = np.empty(n, dtype=np.uint32)
    lib().synth_trial_counts(w.seed, first, n, w.nmin, w.nmax, _ptr(c))
    return c


def gen_offsets(w: Workload, first: int = 0, n: Optional[int] = None,
                out: Optional[np.ndarray] = None) -> np.ndarray:
    n = w.n_trials - first if n is None else n
    off = np.empty(n + 1, dtype=np.uint64) if out is None else out
    assert off.dtype == np.uint64 and off.size >= n + 1 and off.flags.c_contiguous
    lib().synth_yet_offsets(w.seed, first, n, w.nmin, w.nmax, _ptr(off))
    return off


def event_base(w: Workload, first: int) -> int:
    return int(lib().synth_event_base(w.seed, first, w.nmin, w.nmax))


def gen_events(w: Workload, begin: int, n: int, out: Optional[np.ndarray] = None,
               nthreads: Optional[int] = None) -> np.ndarray:
    ids = np.empty(n, dtype=np.uint32) if out is None else out
    assert ids.dtype == np.uint32 and ids.size >= n and ids.flags.c_contiguous
    nt = nthreads or min(64, os.cpu_count() or 1)
    lib().synth_yet_events(w.seed, w.catalog, begin, n, _ptr(ids), nt)
    return ids


def gen_yet(w: Workload, first: int = 0, n: Optional[int] = None,
            out_offsets: Optional[np.ndarray] = None, out_ids: Optional[np.ndarray] = None,
            nthreads: Optional[int] = None) -> Tuple[np.ndarray, np.ndarray]:
    """YET (Eq. 1) for trials [first, first+n) as CSR: (offsets[n+1] from 0, ids)."""
    n = w.n_trials - first if n is None else n
    off = gen_offsets(w, first, n, out_offsets)
    base = event_base(w, first)
    ne = int(off[n])
    ids = gen_events(w, base, ne, out_ids, nthreads)
    return off, ids


def gen_trial_sample(w: Workload, trials: Sequence[int]) -> Tuple[np.ndarray, np.ndarray]:
    """Mini-CSR holding only the listed trials (any order), regenerated from
    the counter-based streams independently of every other trial."""
    trials = np.asarray(trials, dtype=np.int64)
    order = np.argsort(trials, kind="stable")
    counts_all = None
    # global event base per trial: prefix sum over all trial counts up to max
    tmax = int(trials.max()) + 1 if trials.size else 0
    counts_all = gen_counts(w, 0, tmax).astype(np.uint64)
    bases = np.zeros(tmax + 1, dtype=np.uint64)
    np.cumsum(counts_all, out=bases[1:])
    off = np.zeros(trials.size + 1, dtype=np.uint64)
    off[1:] = np.cumsum(counts_all[trials]) if trials.size else []
    ids = np.empty(int(off[-1]), dtype=np.uint32)
    for i, t in enumerate(trials):
        n = int(counts_all[t])
        if n:
            gen_events(w, int(bases[t]), n, ids[int(off[i]):int(off[i]) + n], nthreads=1)
    del order
    return off, ids


def gen_elts(w: Workload) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """ELTs (Eq. 2) as concatenated sparse lists: (offsets[E+1], event_ids, losses),
    each ELT ascending by event id."""
    L = lib()
    counts = [int(L.synth_elt_count(w.seed, j, w.catalog, w.rho)) for j in range(w.n_elts)]
    off = np.zeros(w.n_elts + 1, dtype=np.uint64)
    off[1:] = np.cumsum(counts)
    ev = np.empty(int(off[-1]), dtype=np.uint32)
    ls = np.empty(int(off[-1]), dtype=np.float64)
    for j in range(w.n_elts):
        a, b = int(off[j]), int(off[j + 1])
        if b > a:
            L.synth_elt_fill(w.seed, j, w.catalog, w.rho, w.mu, w.sigma, w.int_cap,
                             _ptr(ev[a:b]), _ptr(ls[a:b]))
    return off, ev, ls


def gen_timestamps(w: Workload, trial: int, n: int) -> np.ndarray:
    ts = np.empty(n, dtype=np.float64)
    lib().synth_trial_timestamps(w.seed, trial, n, _ptr(ts))
    return ts


from .configs import CONFIGS, get_config  # noqa: E402,F401
