"""SURVEY 8f F1 on the GPU: v tenants on one B200 -- independent ARA contexts
with their own streams, driven from their own host threads at the same time
(the vGPU-per-pGPU setting of P:583-618, "each vGPU ... processes a subset of
the trials") -- each loading and running its own sub-shard of the
YET.  Trials are independent, so the tenants' YLTs, concatenated,
must be the one-tenant YLT bit for bit (P11), and within the A21 bound of
the oracle; lossy counts exact."""
import threading

import numpy as np
import pytest

import synth
from parity_util import assert_ylt_close, make_inputs, run_gpu, run_oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("v", [2, 4])
@pytest.mark.parametrize("rho,load_mode", [(0.02, "all"), (0.3, "all"), (0.02, "chunked")])
def test_concurrent_tenants_reproduce_one_tenant(cuda, v, rho, load_mode):
    import torch
    from paper_1606_04473_b200 import ara
    w = synth.get_config("tiny").with_(n_trials=4001, rho=rho, nmin=50, nmax=400)
    off, ids, elts = make_inputs(w)
    one, one_lossy, _, _ = run_gpu(off, ids, elts, w, w.layers)
    orc = run_oracle(off, ids, elts, w, w.layers)
    assert_ylt_close(one, orc)
    out = [None] * v
    errors = []
    start = threading.Barrier(v)

    def tenant(r):
        try:
            f, c = ara.ara_partition(w.n_trials, v, r)
            so = off[f:f + c + 1].copy()
            si = ids[int(off[f]):int(off[f + c])].copy()
            stream = torch.cuda.Stream()
            with ara.Context(w.catalog, stream=stream, load_mode=load_mode, chunk_trials=97) as ctx:
                ctx.load_elts(*elts, w.elt_terms())
                start.wait()                       # all tenants load and run at the same time
                for _ in range(3):
                    ctx.load_yet(c, 0, so, si)     # each tenant: its sub-shard as a whole YET
                    ylt, lossy, st = ctx.run_host(w.layers)
                out[r] = (f, c, ylt, lossy)
        except Exception as e:   # surfaced in the main thread
            errors.append(e)
            start.abort()

    th = [threading.Thread(target=tenant, args=(r,)) for r in range(v)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    got = np.full_like(one, np.nan)
    got_lossy = np.zeros_like(one_lossy)
    for f, c, ylt, lossy in out:
        got[:, f:f + c] = ylt
        got_lossy[:, f:f + c] = lossy
    assert np.array_equal(got, one) and np.array_equal(got_lossy, one_lossy)
