"""ctypes binding of ``libara.so`` (include/ara.h) — argument marshalling only.

Every step of the ARA path runs in the library's CUDA kernels; this module
only converts numpy arrays / torch tensors to pointers and status codes to
exceptions.  There is no CPU fallback: if ``libara.so`` is missing the import
fails loudly.

Functions carry the C names (``ara_create``, ``ara_load_elts``, ...); the
``Context`` class wraps them for convenience.
"""
from __future__ import annotations

import ctypes
import math
import os
from typing import Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# ARA_LIB_PATH: another build of the same library (A/B timing of two builds on one box)
LIB_PATH = os.environ.get("ARA_LIB_PATH") or os.path.join(_HERE, "libara.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
                      "there is no CPU fallback")
_lib = ctypes.CDLL(LIB_PATH)

ARA_OK, ARA_ERR_INVALID_ARG, ARA_ERR_OUT_OF_RANGE, ARA_ERR_DOMAIN = 0, 1, 2, 3
ARA_ERR_STATE, ARA_ERR_OOM, ARA_ERR_CUDA, ARA_ERR_NCCL = 4, 5, 6, 7
ARA_F64, ARA_F32_STORAGE = 0, 1
ARA_LOAD_ALL_AT_ONCE, ARA_LOAD_CHUNKED = 0, 1
ARA_RUN_DIRECT, ARA_RUN_FOLD = 0, 1
ARA_NCCL_ID_BYTES = 128
ARA_MAX_LAYERS = 64
ARA_MAX_RP = 64
ARA_MAX_EP_POINTS = 4096


class ara_config(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("precision", ctypes.c_int), ("stream", ctypes.c_void_p),
                ("rank", ctypes.c_int), ("world", ctypes.c_int), ("nccl_unique_id", ctypes.c_void_p),
                ("load_mode", ctypes.c_int), ("chunk_trials", ctypes.c_uint64),
                ("l2_persist", ctypes.c_int), ("run_mode", ctypes.c_int)]


class ara_elt_terms(ctypes.Structure):
    _fields_ = [("deductible", ctypes.c_double), ("limit", ctypes.c_double)]


class ara_layer(ctypes.Structure):
    _fields_ = [("elt_begin", ctypes.c_uint32), ("elt_end", ctypes.c_uint32),
                ("occ_retention", ctypes.c_double), ("occ_limit", ctypes.c_double),
                ("agg_retention", ctypes.c_double), ("agg_limit", ctypes.c_double)]


class ara_layer_list(ctypes.Structure):
    _fields_ = [("elts", ctypes.c_void_p), ("n_elts", ctypes.c_uint32),
                ("occ_retention", ctypes.c_double), ("occ_limit", ctypes.c_double),
                ("agg_retention", ctypes.c_double), ("agg_limit", ctypes.c_double)]


class ara_run_stats(ctypes.Structure):
    _fields_ = [("n_trials_local", ctypes.c_uint64), ("n_events_local", ctypes.c_uint64),
                ("n_lookups_local", ctypes.c_uint64), ("kernel_ms", ctypes.c_double),
                ("h2d_ms", ctypes.c_double), ("allgather_ms", ctypes.c_double),
                ("total_ms", ctypes.c_double), ("h2d_bytes", ctypes.c_uint64),
                ("n_kernel_launches", ctypes.c_uint32), ("kernel_variant", ctypes.c_int32),
                ("occupancy", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_vp, _u32, _u64, _i, _d = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_double
_sig = {
    "ara_version": (ctypes.c_char_p, []),
    "ara_status_string": (ctypes.c_char_p, [_i]),
    "ara_partition": (_i, [_u64, _i, _i, ctypes.POINTER(_u64), ctypes.POINTER(_u64)]),
    "ara_return_period_rank": (_i, [_u64, _d, ctypes.POINTER(_u64)]),
    "ara_nccl_unique_id": (_i, [_vp]),
    "ara_create": (_i, [_u32, ctypes.POINTER(ara_config), ctypes.POINTER(_vp)]),
    "ara_destroy": (None, [_vp]),
    "ara_last_error": (ctypes.c_char_p, [_vp]),
    "ara_load_elts": (_i, [_vp, _u32, _vp, _vp, _vp, _vp]),
    "ara_set_elt_terms": (_i, [_vp, _u32, _vp]),
    "ara_load_yet": (_i, [_vp, _u64, _u64, _u64, _vp, _vp]),
    "ara_load_yet_packed": (_i, [_vp, _u64, _u64, _u64, _vp, _vp, _u32]),
    "ara_packed_words": (_u64, [_u64, _u32]),
    "ara_pack_ids": (_i, [_vp, _u64, _u32, _vp]),
    "ara_run": (_i, [_vp, _u32, _vp, _vp, _vp, ctypes.POINTER(ara_run_stats)]),
    "ara_run_portfolio": (_i, [_vp, _u32, _vp, _u32, _vp, _vp, _vp, ctypes.POINTER(ara_run_stats)]),
    "ara_metrics": (_i, [_vp, _u32, _vp, _vp, _vp, _vp, ctypes.POINTER(_d)]),
    "ara_ep_curve": (_i, [_vp, _u32, _vp, _vp]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args
EXPORTED = tuple(_sig)


class AraError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{status_string(status)}: {message}")
        self.status = status


def status_string(s: int) -> str:
    return _lib.ara_status_string(s).decode()


def version() -> str:
    return _lib.ara_version().decode()


def _ptr(a) -> Optional[int]:
    """numpy array / torch tensor / int / None -> raw address."""
    if a is None:
        return None
    if isinstance(a, int):
        return a
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr()
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    raise TypeError(f"cannot take the address of {type(a)}")


def _check(st: int, ctx=None, what: str = ""):
    if st != ARA_OK:
        msg = _lib.ara_last_error(ctx).decode() if ctx else what
        raise AraError(st, msg or what)


# ---------------------------------------------------------- C-named wrappers
def ara_partition(n_trials: int, world: int, rank: int) -> Tuple[int, int]:
    f, c = _u64(), _u64()
    _check(_lib.ara_partition(n_trials, world, rank, ctypes.byref(f), ctypes.byref(c)), what="ara_partition")
    return f.value, c.value


def ara_return_period_rank(n_trials: int, return_period: float) -> int:
    k = _u64()
    _check(_lib.ara_return_period_rank(n_trials, float(return_period), ctypes.byref(k)),
           what=f"return period {return_period} outside [1, {n_trials}]")
    return k.value


def ara_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(ARA_NCCL_ID_BYTES)
    _check(_lib.ara_nccl_unique_id(buf), what="ncclGetUniqueId")
    return buf.raw


def ara_create(catalog_size: int, device: int = 0, precision: int = ARA_F64, stream=None, rank: int = 0,
               world: int = 1, nccl_id: Optional[bytes] = None, load_mode: int = ARA_LOAD_ALL_AT_ONCE,
               chunk_trials: int = 0, l2_persist: bool = False, run_mode: int = ARA_RUN_DIRECT):
    idbuf = ctypes.create_string_buffer(nccl_id, ARA_NCCL_ID_BYTES) if nccl_id else None
    cfg = ara_config(device, precision, _stream_ptr(stream), rank, world,
                     ctypes.cast(idbuf, _vp) if idbuf is not None else None, load_mode, chunk_trials,
                     1 if l2_persist else 0, run_mode)
    h = _vp()
    st = _lib.ara_create(catalog_size, ctypes.byref(cfg), ctypes.byref(h))
    _check(st, what="ara_create (no CUDA device, bad config, or NCCL init failure)")
    return h


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)   # torch.cuda.Stream


def ara_destroy(h) -> None:
    _lib.ara_destroy(h)


def ara_load_elts(h, elt_offsets, event_ids, losses, terms=None, n_elts=None) -> None:
    n = (len(elt_offsets) - 1) if elt_offsets is not None else int(n_elts or 0)
    t = _terms_array(terms)
    _check(_lib.ara_load_elts(h, n, _ptr(elt_offsets), _ptr(event_ids), _ptr(losses), t), h)


def _terms_array(terms):
    if terms is None:
        return None
    if isinstance(terms, tuple) and len(terms) == 2:
        d, l = (np.asarray(x, dtype=np.float64) for x in terms)
        terms = list(zip(d, l))
    arr = (ara_elt_terms * len(terms))(*[ara_elt_terms(float(a), float(b)) for a, b in terms])
    return ctypes.cast(arr, _vp) if len(terms) else None


def ara_set_elt_terms(h, terms) -> None:
    n = len(terms[0]) if isinstance(terms, tuple) else len(terms)
    _check(_lib.ara_set_elt_terms(h, n, _terms_array(terms)), h)


def ara_load_yet(h, n_trials_global: int, first_trial: int, trial_offsets, event_ids) -> None:
    n_local = len(trial_offsets) - 1
    _check(_lib.ara_load_yet(h, n_trials_global, first_trial, n_local, _ptr(trial_offsets), _ptr(event_ids)), h)


def ara_load_yet_packed(h, n_trials_global: int, first_trial: int, trial_offsets, packed_ids, bits: int) -> None:
    n_local = len(trial_offsets) - 1
    _check(_lib.ara_load_yet_packed(h, n_trials_global, first_trial, n_local, _ptr(trial_offsets),
                                    _ptr(packed_ids), bits), h)


def ara_packed_words(n_ids: int, bits: int) -> int:
    return int(_lib.ara_packed_words(n_ids, bits))


def ara_pack_ids(ids, bits: int, out=None):
    """Bit-pack u32 ids (host) into the ara_load_yet_packed word stream."""
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    words = ara_packed_words(len(ids), bits)
    if out is None:
        out = np.empty(words, dtype=np.uint32)
    _check(_lib.ara_pack_ids(ids.ctypes.data, len(ids), bits, _ptr(out)), what="id does not fit in bits")
    return out


def bits_for_catalog(catalog_size: int) -> int:
    return max(1, int(catalog_size).bit_length())


def _layers_array(layers):
    arr = (ara_layer * len(layers))()
    for i, L in enumerate(layers):
        if isinstance(L, ara_layer):
            arr[i] = L
        else:   # synth.LayerSpec or tuple (begin, end, occR, occL, aggR, aggL)
            v = (L.elt_begin, L.elt_end, L.occ_retention, L.occ_limit, L.agg_retention, L.agg_limit) \
                if hasattr(L, "elt_begin") else tuple(L)
            arr[i] = ara_layer(int(v[0]), int(v[1]), float(v[2]), float(v[3]), float(v[4]), float(v[5]))
    return arr


def ara_run(h, layers, ylt=None, lossy=None) -> dict:
    arr = _layers_array(layers)
    stats = ara_run_stats()
    _check(_lib.ara_run(h, len(layers), ctypes.cast(arr, _vp), _ptr(ylt), _ptr(lossy), ctypes.byref(stats)), h)
    return stats.as_dict()


def ara_run_portfolio(h, programs, ylt=None, lossy=None) -> dict:
    """programs: list of programs, each a list of layers (elts, OccR, OccL, AggR, AggL)
    with `elts` strictly ascending ELT indices."""
    flat = [L for prog in programs for L in prog]
    pl = np.zeros(len(programs) + 1, dtype=np.uint32)
    pl[1:] = np.cumsum([len(p) for p in programs])
    keep = []
    arr = (ara_layer_list * len(flat))()
    for i, L in enumerate(flat):
        e = np.ascontiguousarray(L[0], dtype=np.uint32)
        keep.append(e)
        arr[i] = ara_layer_list(e.ctypes.data, len(e), float(L[1]), float(L[2]), float(L[3]), float(L[4]))
    stats = ara_run_stats()
    _check(_lib.ara_run_portfolio(h, len(programs), pl.ctypes.data, len(flat), ctypes.cast(arr, _vp), _ptr(ylt),
                                  _ptr(lossy), ctypes.byref(stats)), h)
    return stats.as_dict()


def ara_metrics(h, n_rows: int, return_periods: Sequence[float]):
    """n_rows: YLT rows of the last run (n_layers + 1, or n_layers + n_programs + 1)."""
    R = np.ascontiguousarray(return_periods, dtype=np.float64)
    k = np.zeros(len(R), dtype=np.uint64)
    pml = np.zeros((n_rows, len(R)), dtype=np.float64)
    tvar = np.zeros((n_rows, len(R)), dtype=np.float64)
    ms = _d()
    _check(_lib.ara_metrics(h, len(R), R.ctypes.data, k.ctypes.data, pml.ctypes.data, tvar.ctypes.data,
                            ctypes.byref(ms)), h)
    return k, pml, tvar, ms.value


def ara_ep_curve(h, n_rows: int, thresholds):
    """counts [n_rows][n] u64: #{t : Y[row][t] > thresholds[i]} (thresholds non-decreasing)."""
    x = np.ascontiguousarray(thresholds, dtype=np.float64)
    counts = np.zeros((n_rows, len(x)), dtype=np.uint64)
    _check(_lib.ara_ep_curve(h, len(x), x.ctypes.data, counts.ctypes.data), h)
    return counts


class Context:
    """One ARA context on one GPU (one per rank).  See include/ara.h."""

    def __init__(self, catalog_size: int, device: int = 0, precision: str = "f64", stream=None,
                 rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None, load_mode: str = "all",
                 chunk_trials: int = 0, l2_persist: bool = False, run_mode: str = "direct"):
        prec = {"f64": ARA_F64, "f32": ARA_F32_STORAGE}[precision]
        mode = {"all": ARA_LOAD_ALL_AT_ONCE, "chunked": ARA_LOAD_CHUNKED}[load_mode]
        rmode = {"direct": ARA_RUN_DIRECT, "fold": ARA_RUN_FOLD}[run_mode]
        self.h = ara_create(catalog_size, device, prec, stream, rank, world, nccl_id, mode, chunk_trials,
                            l2_persist, rmode)
        self.n_layers = 0
        self.n_rows = 0
        self.n_trials = 0

    def close(self):
        if self.h:
            ara_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load_elts(self, elt_offsets, event_ids, losses, terms=None, n_elts=None):
        """n_elts is only needed by non-root ranks passing None arrays (world > 1)."""
        ara_load_elts(self.h, elt_offsets, event_ids, losses, terms, n_elts)

    def set_elt_terms(self, terms):
        ara_set_elt_terms(self.h, terms)

    def load_yet(self, n_trials_global: int, first_trial: int, trial_offsets, event_ids):
        ara_load_yet(self.h, n_trials_global, first_trial, trial_offsets, event_ids)
        self.n_trials = n_trials_global
        self._yet_refs = (trial_offsets, event_ids)   # CHUNKED mode reads them during ara_run

    def load_yet_packed(self, n_trials_global: int, first_trial: int, trial_offsets, packed_ids, bits: int):
        ara_load_yet_packed(self.h, n_trials_global, first_trial, trial_offsets, packed_ids, bits)
        self.n_trials = n_trials_global
        self._yet_refs = (trial_offsets, packed_ids)   # CHUNKED mode reads them during ara_run

    def run(self, layers, ylt=None, lossy=None) -> dict:
        st = ara_run(self.h, layers, ylt, lossy)
        self.n_layers = len(layers)
        self.n_rows = len(layers) + 1
        return st

    def run_portfolio(self, programs, ylt=None, lossy=None) -> dict:
        st = ara_run_portfolio(self.h, programs, ylt, lossy)
        self.n_layers = sum(len(p) for p in programs)
        self.n_rows = self.n_layers + len(programs) + 1
        return st

    def run_portfolio_host(self, programs, with_lossy: bool = True):
        L = sum(len(p) for p in programs)
        ylt = np.empty((L + len(programs) + 1, self.n_trials), dtype=np.float64)
        lossy = np.empty((L, self.n_trials), dtype=np.uint32) if with_lossy else None
        st = self.run_portfolio(programs, ylt, lossy)
        return ylt, lossy, st

    def run_host(self, layers, with_lossy: bool = True, n_local: Optional[int] = None):
        """Convenience: YLT [(L+1)][T] and lossy [L][T_local] into new host arrays."""
        L = len(layers)
        ylt = np.empty((L + 1, self.n_trials), dtype=np.float64)
        nl = self.n_trials if n_local is None else n_local
        lossy = np.empty((L, max(nl, 0)), dtype=np.uint32) if with_lossy else None
        st = self.run(layers, ylt, lossy if (with_lossy and nl > 0) else None)
        return ylt, lossy, st

    def metrics(self, return_periods):
        return ara_metrics(self.h, self.n_rows, return_periods)

    def ep_curve(self, thresholds):
        return ara_ep_curve(self.h, self.n_rows, thresholds)


__all__ = ["Context", "AraError", "ara_create", "ara_destroy", "ara_load_elts", "ara_set_elt_terms",
           "ara_load_yet", "ara_run", "ara_metrics", "ara_partition", "ara_return_period_rank",
           "ara_nccl_unique_id", "ara_load_yet_packed", "ara_ep_curve", "ara_run_portfolio", "ara_pack_ids", "ara_packed_words", "bits_for_catalog",
           "status_string", "version", "EXPORTED"]
