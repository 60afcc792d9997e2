"""Workload presets: BASELINE.json ``configs`` as concrete synthetic inputs.

Shapes follow the paper (800-1500 events/trial P:221-224; 10k-30k losses per
ELT P:237; 3-30 ELTs per layer P:263; YET 4 GB P:433).  Term values are the
calibrated ones of SURVEY.md §8d, chosen so every clamp binds at a
non-trivial rate.  Terms are inputs, not method arithmetic.
"""
import math

from . import LayerSpec, Workload

INF = math.inf

_PAPER_LAYER = LayerSpec(0, 16, 2.5e4, 7.5e5, 1.2e7, 8e6)

CONFIGS = {
    # BASELINE configs[0]: oracle finishes in ms
    "tiny": Workload(
        name="tiny", seed=1606044731, n_trials=1000, nmin=80, nmax=120,
        catalog=10_000, n_elts=3, rho=0.30,
        layers=(LayerSpec(0, 3, 2.5e4, 5e5, 6.5e6, 2.5e6),)),
    # BASELINE configs[1]: the bench workload (1 B200)
    "paper": Workload(
        name="paper", seed=1606044732, n_trials=1_000_000, nmin=800, nmax=1200,
        catalog=2_000_000, n_elts=16, rho=0.01, layers=(_PAPER_LAYER,)),
    # BASELINE configs[3]: 4 disjoint layers x 16 ELTs, PML/TVaR at 10 return periods
    "multilayer": Workload(
        name="multilayer", seed=1606044734, n_trials=1_000_000, nmin=800, nmax=1200,
        catalog=2_000_000, n_elts=64, rho=0.01,
        layers=(LayerSpec(0, 16, 2.5e4, 7.5e5, 1.2e7, 8e6),
                LayerSpec(16, 32, 1e5, 4e5, 6.5e6, 4e6),
                LayerSpec(32, 48, 2.5e5, 5e5, 4e6, 3.5e6),
                LayerSpec(48, 64, 5e5, 5e5, 0.0, INF))),
    # SURVEY §8d config 4 "tower" variant: 4 layers over the same 16 ELTs
    # (one row window serves every layer), multilayer terms
    "tower": Workload(
        name="tower", seed=1606044734, n_trials=1_000_000, nmin=800, nmax=1200,
        catalog=2_000_000, n_elts=16, rho=0.01,
        layers=(LayerSpec(0, 16, 2.5e4, 7.5e5, 1.2e7, 8e6),
                LayerSpec(0, 16, 1e5, 4e5, 6.5e6, 4e6),
                LayerSpec(0, 16, 2.5e5, 5e5, 4e6, 3.5e6),
                LayerSpec(0, 16, 5e5, 5e5, 0.0, INF))),
    # BASELINE configs[4]: streamed 10M-trial YET (40 GB of ids)
    "stream10m": Workload(
        name="stream10m", seed=1606044735, n_trials=10_000_000, nmin=800, nmax=1200,
        catalog=2_000_000, n_elts=16, rho=0.01, layers=(_PAPER_LAYER,)),
    # SPEC S:164 desk-scale preset (partition-invariance tests)
    "mini": Workload(
        name="mini", seed=1606044730, n_trials=100_000, nmin=800, nmax=1500,
        catalog=50_000, n_elts=10, rho=0.2,
        layers=(LayerSpec(0, 10, 2.5e4, 7.5e5, 1.2e7, 8e6),)),
}


def get_config(name: str) -> Workload:
    try:
        return CONFIGS[name]
    except KeyError:
        raise KeyError(f"unknown workload {name!r}; have {sorted(CONFIGS)}") from None
