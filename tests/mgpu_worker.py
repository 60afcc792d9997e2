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
        ylt, lossy, st = ctx.run_host(w.layers, n_local=count)
        R = [r for r in w.return_periods if r <= w.n_trials]
        k, pml, tvar, _ = ctx.metrics(R)
        # every rank holds the same global YLT and metrics
        g = [None] * world
        dist.all_gather_object(g, (ylt.tobytes(), pml.tobytes(), tvar.tobytes()))
        same = all(x == g[0] for x in g)
        if rank == 0:
            np.savez(out, ylt=ylt, pml=pml, tvar=tvar, k=k, same=same, allgather_ms=st["allgather_ms"])
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
