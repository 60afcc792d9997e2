"""N>1 host logic on CPU (world_size 2 and 4, gloo): each rank takes its
ara_partition() shard, computes its YLT slice (the oracle stands in for the
device here), and the slices are all-gathered and merged by trial index
(Alg. 1 l.9).  The merged YLT must equal the unsharded one
bit for bit (P11), and the metrics every rank derives must agree."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _body(rank, world, q)
    except BaseException as e:  # report instead of hanging the parent
        q.put((rank, repr(e), False))
        raise
    finally:
        dist.destroy_process_group()


def _body(rank, world, q):
    if True:
        import oracle
        import synth
        from paper_1606_04473_b200 import ara
        w = synth.get_config("tiny").with_(n_trials=999, return_periods=(2, 5, 10, 999))  # ragged: 999 % 2, 4 != 0
        first, count = ara.ara_partition(w.n_trials, world, rank)
        off, ids = synth.gen_yet(w, first=first, n=count)         # this rank's shard only
        eo, ev, ls = synth.gen_elts(w)
        d, li = w.elt_terms()
        part = oracle.ara(off, ids, oracle.Elts(eo, ev, ls), w.catalog, d, li,
                          oracle.layers_from_specs(w.layers))["ylt"]
        got = [None] * world
        dist.all_gather_object(got, (first, count, part))
        merged = np.zeros((part.shape[0], w.n_trials))
        for f, c, p in got:                                       # keyed scatter by trial index
            merged[:, f:f + c] = p
        k, pml, tvar = oracle.metrics(merged[0], w.return_periods)
        allm = [None] * world
        dist.all_gather_object(allm, (pml.tobytes(), tvar.tobytes()))
        q.put((rank, merged, len(set(allm)) == 1))


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_ylt_equals_unsharded(world):
    import oracle
    import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = synth.get_config("tiny").with_(n_trials=999)
    off, ids = synth.gen_yet(w)
    eo, ev, ls = synth.gen_elts(w)
    d, li = w.elt_terms()
    full = oracle.ara(off, ids, oracle.Elts(eo, ev, ls), w.catalog, d, li,
                      oracle.layers_from_specs(w.layers))["ylt"]
    for rank, merged, agree in res:
        assert agree, merged
        assert np.array_equal(merged, full)
