"""Pins for the paper's §V-F performance model (tools/tenancy_model.py): Table
II constants, the published measurements it is checked against, and the
worked values in SPEC.md S:360-378."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import tenancy_model as tm  # noqa: E402


def test_computation_scaling():
    assert tm.t_computation(1, tm.FDR) == 9.55                       # Table II
    assert tm.t_computation(16, tm.FDR) == pytest.approx(0.596875)   # S:365; P:490 measured 0.62 s
    assert abs(tm.t_computation(16, tm.FDR) - 0.62) / 0.62 < 0.04


def test_transfer_model():
    assert tm.t_transfer(1, tm.FDR) == pytest.approx(0.69679)         # S:372; "0.68 s with FDR"
    assert tm.t_transfer(16, tm.FDR) == pytest.approx(1.09864)
    assert 16 * tm.FDR.t_cudamalloc == pytest.approx(0.0432)         # P:513 "43.2 milliseconds for 16 remote GPUs"
    assert tm.t_transfer(14, tm.QDR) == pytest.approx(1.7982, abs=1e-4)


def test_multitenancy_worked_values():
    total, regime, fully, not_fully = tm.exec_time_multitenancy(4, 2, tm.FDR)
    assert fully == pytest.approx(2.8297, abs=1e-4) and not_fully == pytest.approx(2.078, abs=1e-3)
    assert regime == "fully_overlapped" and total == fully
    assert tm.exec_time_multitenancy(4, 4, tm.FDR)[0] == pytest.approx(2.6622, abs=1e-4)   # P:614 ~ 76 cells = 2.66 s
    t16 = tm.exec_time_multitenancy(16, 1, tm.FDR)[0]
    assert t16 == pytest.approx(1.6956, abs=1e-4) and abs(t16 - 1.66) / 1.66 < 0.03    # P:515 measured 1.66 s


def test_v1_reduces_to_non_tenant_total():
    for P in (1, 2, 4, 16):
        assert tm.exec_time_multitenancy(P, 1, tm.QDR)[0] == pytest.approx(
            tm.t_transfer(P, tm.QDR) + tm.t_computation(P, tm.QDR))
