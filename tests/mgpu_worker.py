"""torchrun worker for tests/test_multigpu.py: the collective C-ABI path on N GPUs.

Each rank: NCCL bootstrap through torch.distributed, ELTs from rank 0 only
(NVLink broadcast inside ara_load_elts), its ara_partition() shard of the YET,
ara_run (all-gather of the YLT) and ara_metrics.  Rank 0 writes the global YLT
and metrics to OUT (npz) for the parent test to compare with a 1-GPU run."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


EP_X = np.concatenate([[-1.0, 0.0], np.linspace(1.0, 1.2e7, 255), [np.inf]])   # EP-curve thresholds


def bumped_layers(layers):
    return tuple(L.__class__(L.elt_begin, L.elt_end, L.occ_retention * 1.5 + 1.0, L.occ_limit, L.agg_retention,
                             L.agg_limit) for L in layers)


def main():
    import torch
    import torch.distributed as dist
    import synth
    from paper_1606_04473_b200 import ara
    name, n_trials, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    rho = float(sys.argv[4]) if len(sys.argv) > 4 else None
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    obj = [ara.ara_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    w = synth.get_config(name).with_(n_trials=n_trials)
    if rho is not None:
        w = w.with_(rho=rho)
    first, count = ara.ara_partition(w.n_trials, world, rank)
    off, ids = synth.gen_yet(w, first=first, n=count)
    with ara.Context(w.catalog, device=local, rank=rank, world=world, nccl_id=obj[0]) as ctx:
        if rank == 0:
            eo, ev, ls = synth.gen_elts(w)
            ctx.load_elts(eo, ev, ls, w.elt_terms())
        else:
            ctx.load_elts(None, None, None, w.elt_terms(), n_elts=w.n_elts)
        ctx.load_yet(w.n_trials, first, off, ids)
        R = [r for r in w.return_periods if r <= w.n_trials]
        res = []
        # three consecutive runs (base, bumped occurrence retention, base): the
        # fused assembly alternates its two global buffers between runs
        for layers in (w.layers, bumped_layers(w.layers), w.layers):
            ylt, lossy, st = ctx.run_host(layers, n_local=count)
            k, pml, tvar, _ = ctx.metrics(R)
            ep = ctx.ep_curve(EP_X)           # collective: shard counts all-reduced
            res.append((ylt, pml, tvar, k, st, ep))
        # every rank holds the same global YLT and metrics
        g = [None] * world
        dist.all_gather_object(g, [(y.tobytes(), p.tobytes(), t.tobytes(), e.tobytes()) for y, p, t, _, _, e in res])
        same = all(x == g[0] for x in g)
        if rank == 0:
            np.savez(out, ylt=res[0][0], pml=res[0][1], tvar=res[0][2], k=res[0][3], same=same, ep=res[0][5],
                     allgather_ms=res[0][4]["allgather_ms"], ylt_b=res[1][0], pml_b=res[1][1], ylt_c=res[2][0])
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
