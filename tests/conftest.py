import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C-ABI)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs")
    # The CPU suite needs the oracle + generator libraries; build them if absent
    # (nvcc cross-compiles libara.so here too, so build everything).
    subprocess.run(["make", "-C", ROOT, "oracle/liboracle.so", "synth/libsynth.so"], check=True,
                   stdout=subprocess.DEVNULL, stderr=subprocess.STDOUT)
    # libara.so (nvcc cross-compiles here); a build failure surfaces in test_abi.
    subprocess.run(["make", "-j8", "-C", ROOT], stdout=subprocess.DEVNULL, stderr=subprocess.STDOUT)


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def cuda():
    if not gpu_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    import torch
    return torch.device("cuda:0")
