"""CPU oracle for Aggregate Risk Analysis — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_1606_04473_b200``) never imports it; the two share no code.

Thin ctypes marshalling over ``liboracle.so`` (oracle.c, plain C, fp64,
-ffp-contract=off).  Every function cites the passage it follows in oracle.h.
"""
from __future__ import annotations

import ctypes
import os
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

LOOKUP_MAP = 0
LOOKUP_DENSE = 1


class _Elts(ctypes.Structure):
    _fields_ = [("n_elts", ctypes.c_uint32), ("offsets", ctypes.c_void_p),
                ("event_ids", ctypes.c_void_p), ("losses", ctypes.c_void_p)]


class _Layer(ctypes.Structure):
    _fields_ = [("n_elts", ctypes.c_uint32), ("elts", ctypes.c_void_p),
                ("occ_retention", ctypes.c_double), ("occ_limit", ctypes.c_double),
                ("agg_retention", ctypes.c_double), ("agg_limit", ctypes.c_double)]


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run `make` (or __graft_entry__.build())")
        L = ctypes.CDLL(path)
        d, u32, u64, vp, i32 = (ctypes.c_double, ctypes.c_uint32, ctypes.c_uint64,
                                ctypes.c_void_p, ctypes.c_int)
        L.oracle_apply_terms.restype = d
        L.oracle_apply_terms.argtypes = [d, d, d]
        L.oracle_lookup_map.restype = d
        L.oracle_lookup_map.argtypes = [ctypes.POINTER(_Elts), u32, u32]
        L.oracle_direct_access.restype = i32
        L.oracle_direct_access.argtypes = [ctypes.POINTER(_Elts), u32, vp]
        L.oracle_ara.restype = i32
        L.oracle_ara.argtypes = [vp, vp, u64, ctypes.POINTER(_Elts), u32, vp, vp, u32,
                                 ctypes.POINTER(_Layer), i32, vp, i32, vp, vp, vp, vp]
        L.oracle_programs.restype = i32
        L.oracle_programs.argtypes = [vp, u64, u32, u32, vp, vp]
        L.oracle_rank.restype = u64
        L.oracle_rank.argtypes = [u64, d]
        L.oracle_metrics.restype = i32
        L.oracle_metrics.argtypes = [vp, u64, u32, vp, vp, vp, vp]
        L.oracle_ep_counts.restype = None
        L.oracle_ep_counts.argtypes = [vp, u64, u32, vp, vp]
        _LIB = L
    return _LIB


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


class Elts:
    """ELT set (Eq. 2): concatenated ascending sparse lists."""

    def __init__(self, offsets, event_ids, losses):
        self.offsets = _c(offsets, np.uint64)
        self.event_ids = _c(event_ids, np.uint32)
        self.losses = _c(losses, np.float64)
        self._s = _Elts(len(self.offsets) - 1, self.offsets.ctypes.data,
                        self.event_ids.ctypes.data, self.losses.ctypes.data)

    @classmethod
    def from_maps(cls, maps: Sequence[Dict[int, float]]) -> "Elts":
        off, ev, ls = [0], [], []
        for m in maps:
            for e in sorted(m):
                ev.append(e)
                ls.append(float(m[e]))
            off.append(len(ev))
        return cls(off, ev, ls)

    @property
    def n_elts(self) -> int:
        return len(self.offsets) - 1


def apply_terms(loss: float, retention: float, limit: float) -> float:
    return lib().oracle_apply_terms(loss, retention, limit)


def lookup_map(elts: Elts, j: int, e: int) -> float:
    return lib().oracle_lookup_map(ctypes.byref(elts._s), j, e)


def direct_access(elts: Elts, catalog: int) -> np.ndarray:
    dense = np.empty((elts.n_elts, catalog + 1), dtype=np.float64)
    rc = lib().oracle_direct_access(ctypes.byref(elts._s), catalog, dense.ctypes.data)
    if rc != 0:
        raise ValueError("ELT event id outside [1, catalog]")
    return dense


def ara(trial_off, event_ids, elts: Elts, catalog: int, elt_deductible, elt_limit,
        layers: Sequence[Tuple[Sequence[int], float, float, float, float]],
        lookup: str = "map", dense: Optional[np.ndarray] = None, fp32_storage: bool = False):
    """Alg. 1 + Alg. 3.  layers = [(elt list, OccR, OccL, AggR, AggL), ...].
    Returns dict(ylt[L][T], scale[L][T], lossy[L][T], portfolio[T])."""
    off = _c(trial_off, np.uint64)
    ev = _c(event_ids, np.uint32)
    T = len(off) - 1
    Lc = len(layers)
    ded = _c(elt_deductible, np.float64)
    lim = _c(elt_limit, np.float64)
    keep = []
    arr = (_Layer * max(Lc, 1))()
    for i, (el, occr, occl, aggr, aggl) in enumerate(layers):
        e = _c(el, np.uint32)
        keep.append(e)
        arr[i] = _Layer(len(e), e.ctypes.data, occr, occl, aggr, aggl)
    mode = LOOKUP_DENSE if lookup == "dense" else LOOKUP_MAP
    if mode == LOOKUP_DENSE and dense is None:
        dense = direct_access(elts, catalog)
    dptr = dense.ctypes.data if dense is not None else None
    ylt = np.zeros((Lc, T), dtype=np.float64)
    scale = np.zeros((Lc, T), dtype=np.float64)
    lossy = np.zeros((Lc, T), dtype=np.uint32)
    port = np.zeros(T, dtype=np.float64)
    rc = lib().oracle_ara(off.ctypes.data, ev.ctypes.data, T, ctypes.byref(elts._s), catalog,
                          ded.ctypes.data, lim.ctypes.data, Lc, arr, mode, dptr,
                          1 if fp32_storage else 0, ylt.ctypes.data, scale.ctypes.data,
                          lossy.ctypes.data, port.ctypes.data)
    if rc != 0:
        raise ValueError("oracle_ara: event id outside [1, catalog] or unresolved ELT")
    return {"ylt": ylt, "scale": scale, "lossy": lossy, "portfolio": port}


def programs(ylt, program_layers):
    """Program year losses: sums of each program's layer rows in layer order."""
    y = _c(ylt, np.float64)
    pl = _c(program_layers, np.uint32)
    P = len(pl) - 1
    out = np.zeros((P, y.shape[1]), dtype=np.float64)
    if lib().oracle_programs(y.ctypes.data, y.shape[1], y.shape[0], P, pl.ctypes.data, out.ctypes.data) != 0:
        raise ValueError("malformed program_layers")
    return out


def rank(n_trials: int, return_period: float) -> int:
    return int(lib().oracle_rank(n_trials, float(return_period)))


def metrics(y, return_periods):
    """(k[n_rp], pml[n_rp], tvar[n_rp]) of S:206/S:215 (A9, A10)."""
    y = _c(y, np.float64)
    R = _c(return_periods, np.float64)
    k = np.zeros(len(R), dtype=np.uint64)
    pml = np.zeros(len(R), dtype=np.float64)
    tvar = np.zeros(len(R), dtype=np.float64)
    rc = lib().oracle_metrics(y.ctypes.data, len(y), len(R), R.ctypes.data, k.ctypes.data,
                              pml.ctypes.data, tvar.ctypes.data)
    if rc != 0:
        raise ValueError("return period outside [1, T]")
    return k, pml, tvar


def ep_counts(y, thresholds):
    """counts[i] = #{t : y[t] > thresholds[i]} (A23, SURVEY 8f F4 EP curve)."""
    y = _c(y, np.float64)
    x = _c(thresholds, np.float64)
    out = np.zeros(len(x), dtype=np.uint64)
    lib().oracle_ep_counts(y.ctypes.data, len(y), len(x), x.ctypes.data, out.ctypes.data)
    return out


def layers_from_specs(specs) -> List[Tuple[List[int], float, float, float, float]]:
    """Contiguous-range LayerSpecs (synth) -> oracle layer lists."""
    return [(list(range(s.elt_begin, s.elt_end)), s.occ_retention, s.occ_limit,
             s.agg_retention, s.agg_limit) for s in specs]
