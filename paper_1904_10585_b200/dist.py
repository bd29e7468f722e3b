"""Process-group plumbing for the row-block split (one process per GPU).

torch.distributed is used only to ship the 128-byte NCCL unique id from rank 0 to the other
ranks and for the bench's barriers / max-over-ranks timing; every collective of the hot path
runs on the NCCL communicator that libpf.so owns (pf_create_dist)."""
from __future__ import annotations

from typing import Callable

import torch.distributed as dist

from .solver import rows_of  # noqa: F401  (re-exported: the C library's row split)


def broadcast_nccl_id(make_id: Callable[[], bytes] | None = None, group=None) -> bytes:
    """Rank 0 creates the NCCL unique id (pf_nccl_unique_id) and broadcasts it to all ranks."""
    if make_id is None:
        from ._lib import nccl_unique_id as make_id
    obj = [make_id() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def max_over_ranks(value: float, device=None) -> float:
    """Max of a host float over all ranks (bench timing: the slowest rank defines the step)."""
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_loopback(cfg, world: int, iters: int | None = None, problem=None) -> list[dict]:
    """Run the row-block split with `world` ranks on ONE GPU (pf_create_loop): one host thread
    and one stream per rank, every exchange through the in-process loopback communicator.
    Returns each rank's run() result (records hold that rank's local rows of V)."""
    import threading

    import torch

    from ._lib import Loopback
    from .solver import run

    hub = Loopback(world)
    out: list = [None] * world
    errs: list = [None] * world

    def worker(r: int):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                out[r] = run(cfg, iters=iters, problem=problem, rank=r, world=world, loop=hub)
        except BaseException as e:  # noqa: BLE001  (re-raised in the caller)
            errs[r] = e

    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in errs:
        if e is not None:
            raise e
    return out
