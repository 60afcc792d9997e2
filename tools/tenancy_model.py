"""The paper's performance model for (multi-tenant) GPU execution, §V-F
(PAPER.md P:651-698), used as a *predictor* for B200.

  T_computation(#GPUs)   = ComputationTime_1pGPU / #GPUs                 (eq:t_computation)
  T_transfer(#GPUs)      = #GPUs (T_cudaMalloc + T_small + T_4MB + T_120MB)
                           + T_4GB                                        (eq:t_transfer)
  fully_overlapped       = T_transfer(V) / v + v T_computation(V)         (eq:multitenancy1)
  not_fully_overlapped   = T_transfer(V) + T_computation(V)               (eq:multitenancy2)
  ExecTime_Multitenancy  = MAX(fully, not_fully)                          (eq:multitenancy)
with V = P v (P physical GPUs, v tenants per GPU).  Table II
gives the K20/rCUDA constants; `fit_b200` builds the same parameter set from
B200 measurements (per-GPU setup, replicated ELT bytes, the YET over PCIe).
"""
from dataclasses import dataclass, replace


@dataclass(frozen=True)
class ModelParams:
    computation_time_1pgpu: float     # s, the ARA kernel on one GPU
    t_cudamalloc: float               # s per (v)GPU
    t_small_transfers: float          # s per (v)GPU
    t_transfer_4mb: float             # s per (v)GPU (portfolio / terms)
    t_transfer_120mb: float           # s per (v)GPU (replicated ELT data)
    t_transfer_4gb: float             # s, the split YET (all GPUs)


# Table II
QDR = ModelParams(9.55, 0.00267, 0.0048, 0.00133, 0.036, 1.171)
FDR = ModelParams(9.55, 0.0027, 0.0028, 0.00079, 0.0205, 0.67)


def t_computation(n_gpus: int, p: ModelParams) -> float:
    if n_gpus < 1:
        raise ValueError("n_gpus >= 1")
    return p.computation_time_1pgpu / n_gpus


def t_transfer(n_gpus: int, p: ModelParams) -> float:
    if n_gpus < 1:
        raise ValueError("n_gpus >= 1")
    return n_gpus * (p.t_cudamalloc + p.t_small_transfers + p.t_transfer_4mb + p.t_transfer_120mb) + p.t_transfer_4gb


def exec_time_multitenancy(P: int, v: int, p: ModelParams):
    """(total, regime, fully, not_fully) for P physical GPUs x v tenants each."""
    V = P * v
    fully = t_transfer(V, p) / v + v * t_computation(V, p)
    not_fully = t_transfer(V, p) + t_computation(V, p)
    if fully >= not_fully:
        return fully, "fully_overlapped", fully, not_fully
    return not_fully, "not_fully_overlapped", fully, not_fully


def fit_b200(kernel_1gpu_s: float, setup_s: float, small_s: float, elts_s: float, yet_bytes: float,
             h2d_gbs_per_link: float, P: int = 1) -> ModelParams:
    """B200 parameter set from measurements.  Every B200 has its own PCIe link,
    so the split YET's transfer time shrinks with the number of physical GPUs
    (the paper's single 4 GB term assumed one shared link)."""
    return ModelParams(kernel_1gpu_s, setup_s, small_s, 0.0, elts_s, yet_bytes / (h2d_gbs_per_link * 1e9) / P)
