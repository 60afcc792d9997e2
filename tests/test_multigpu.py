"""Multi-GPU path on real GPUs (gpurun --gpus 2/4): the sharded, all-gathered
YLT is bit-identical to the 1-GPU YLT (P11) and every rank derives the same
PML/TVaR.  Skipped when fewer than 2 GPUs are visible."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import synth
from parity_util import make_inputs, run_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)


def _ngpu():
    import torch
    return torch.cuda.device_count()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name,n_trials,rho,p2p,mdist", [("tiny", 1000, None, True, False),
                                                         ("tiny", 997, None, True, False),
                                                         ("mini", 20_000, None, True, False),
                                                         ("mini", 20_001, 0.01, True, False),
                                                         ("tiny", 997, None, False, False),
                                                         ("mini", 20_001, 0.01, False, False),
                                                         ("multilayer", 4001, None, True, False),
                                                         ("tiny", 997, None, True, True),
                                                         ("mini", 20_001, 0.01, False, True)])
def test_sharded_run_matches_single_gpu(cuda, tmp_path, name, n_trials, rho, p2p, mdist):
    """p2p: the kernels store the YLT straight into every rank's global buffer
    over NVLink (fused assembly, the default); otherwise ncclAllGather
    (ARA_NO_P2P=1).  Both must equal the 1-GPU run bit for bit.  mdist: the
    metrics by distributed select (ARA_METRICS_DIST=1: each rank histograms
    its shard, histograms and tail sums all-reduced) -- same PML bits, TVaR
    within rounding of the summation order."""
    n = _ngpu()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(n, 4)
    out = str(tmp_path / "r0.npz")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(HERE, "mgpu_worker.py"),
           name, str(n_trials), out] + ([str(rho)] if rho is not None else [])
    env = dict(os.environ)
    if not p2p:
        env["ARA_NO_P2P"] = "1"
    env["ARA_METRICS_DIST"] = "1" if mdist else "0"
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    got = np.load(out)
    assert bool(got["same"])
    w = synth.get_config(name).with_(n_trials=n_trials)
    if rho is not None:        # sparse ELTs: zero rows skipped, compacted rounds on every rank
        w = w.with_(rho=rho)
    off, ids, elts = make_inputs(w)
    R = [x for x in w.return_periods if x <= w.n_trials]
    ylt, _, _, met = run_gpu(off, ids, elts, w, w.layers, return_periods=R)
    assert np.array_equal(got["ylt"], ylt)
    import oracle
    from mgpu_worker import EP_X
    for r in range(ylt.shape[0]):   # EP curve: the all-reduced shard counts == a count over the global YLT
        assert np.array_equal(got["ep"][r], oracle.ep_counts(ylt[r], EP_X))
    assert np.array_equal(got["pml"], met[1]) and np.array_equal(got["k"], met[0])
    assert np.allclose(got["tvar"], met[2], rtol=1e-12, atol=0)
    # the second and third consecutive runs (other terms, then the first again)
    from mgpu_worker import bumped_layers
    ylt_b, _, _, met_b = run_gpu(off, ids, elts, w, bumped_layers(w.layers), return_periods=R)
    assert np.array_equal(got["ylt_b"], ylt_b) and np.array_equal(got["pml_b"], met_b[1])
    assert np.array_equal(got["ylt_c"], ylt)
