"""Helpers shared by the GPU parity tests: run the CUDA path through the C-ABI
binding and the CPU oracle on the same seeded inputs, compare element-wise.

Tolerance (reading A21): |Y_gpu - Y_oracle| <= rtol * max(S_t, 1)
with S_t the trial's sum of per-event losses (the oracle's `scale`), rtol =
1e-9 in fp64 and in the fp32-storage variant (whose arithmetic is fp64 on
identically rounded inputs).  Trials with S_t == 0 must be exactly 0.  Counts
(lossy occurrences), ranks k and, on integer-valued data, every float are
compared bit for bit.
"""
import math

import numpy as np

import oracle
import synth

RTOL = 1e-9


def make_inputs(w: synth.Workload):
    off, ids = synth.gen_yet(w)
    eo, ev, ls = synth.gen_elts(w)
    return off, ids, (eo, ev, ls)


def run_oracle(off, ids, elts, w, layers, fp32=False, terms=None):
    d, li = (w.elt_terms() if terms is None else terms)
    return oracle.ara(off, ids, oracle.Elts(*elts), w.catalog, d, li,
                      oracle.layers_from_specs(layers), lookup="dense", fp32_storage=fp32)


KERNEL_VARIANTS = (-1, 0, 5, 12, 30)   # ARA_KERNEL: auto, register pipeline (2 / 3 CTAs/SM), cooperative cp.async ring, ballot-compacted rounds (sparse blocks; elsewhere the auto choice)


def run_gpu(off, ids, elts, w, layers, precision="f64", terms=None, load_mode="all", chunk_trials=0,
            device_inputs=False, return_periods=None, variant=None, run_mode="direct", env=None, l2_persist=False):
    """env: extra ARA_* tuning variables read at ara_create (e.g. ARA_NO_SKIP)."""
    import os
    import torch
    from paper_1606_04473_b200 import ara
    d, li = (w.elt_terms() if terms is None else terms)
    env = dict(env or {})
    if variant is not None:
        env["ARA_KERNEL"] = str(variant)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        ctx = ara.Context(w.catalog, precision=precision, load_mode=load_mode, chunk_trials=chunk_trials,
                          run_mode=run_mode, l2_persist=l2_persist)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    with ctx:
        eo, ev, ls = elts
        if device_inputs:
            t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
            eo_, ev_, ls_ = t(eo.astype(np.int64)), t(ev.astype(np.int32)), t(ls)
            off_, ids_ = t(off.astype(np.int64)), t(ids.astype(np.int32))
            ctx.load_elts(eo_, ev_, ls_, (d, li))
            ctx.load_yet(len(off) - 1, 0, off_, ids_)
        else:
            ctx.load_elts(eo, ev, ls, (d, li))
            ctx.load_yet(len(off) - 1, 0, off, ids)
        ylt, lossy, stats = ctx.run_host(layers)
        met = ctx.metrics(return_periods) if return_periods is not None else None
        if device_inputs:
            torch.cuda.synchronize()
    return ylt, lossy, stats, met


def assert_ylt_close(gpu_ylt, orc, rtol=RTOL):
    """gpu_ylt [(L+1)][T] vs oracle dict; lossy compared separately."""
    L = orc["ylt"].shape[0]
    scale = orc["scale"]
    tol = rtol * np.maximum(scale, 1.0)
    diff = np.abs(gpu_ylt[:L] - orc["ylt"])
    bad = diff > tol
    assert not bad.any(), (f"{bad.sum()} trials out of tolerance; worst diff {diff.max()} "
                           f"at {np.unravel_index(diff.argmax(), diff.shape)}")
    z = scale == 0
    assert (gpu_ylt[:L][z] == 0).all()
    ptol = tol.sum(axis=0)
    assert (np.abs(gpu_ylt[L] - orc["portfolio"]) <= ptol).all()


def assert_metrics_close(gpu_met, ylt_rows_oracle, scale, return_periods, rtol=RTOL, exact=False):
    k_g, pml_g, tvar_g, _ = gpu_met
    for r, y in enumerate(ylt_rows_oracle):
        k, pml, tvar = oracle.metrics(y, return_periods)
        assert np.array_equal(k, k_g), (k, k_g)
        if exact:
            assert np.array_equal(pml, pml_g[r]) and np.array_equal(tvar, tvar_g[r]), (r, pml, pml_g[r], tvar, tvar_g[r])
        else:
            tol = rtol * max(float(np.max(scale)) if np.size(scale) else 1.0, 1.0) * (1 if r < len(ylt_rows_oracle) - 1 else len(ylt_rows_oracle))
            assert np.all(np.abs(pml - pml_g[r]) <= tol), (r, pml, pml_g[r])
            assert np.all(np.abs(tvar - tvar_g[r]) <= tol), (r, tvar, tvar_g[r])


def oracle_rows(orc):
    return list(orc["ylt"]) + [orc["portfolio"]]
