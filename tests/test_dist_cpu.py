"""Host logic of the row-block split, exercised with world_size 2 over gloo on CPU:
partition arithmetic, per-rank slicing of the seeded problems, NCCL-id broadcast plumbing and
the max-over-ranks timing helper.  (The NCCL data path itself is covered on the GPU by
tests/test_gpu_dist.py with a single-rank communicator.)"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from pfinputs import CONFIGS, reduced, initial_block, pfpg_problem, pfam_problem


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1904_10585_b200.solver import rows_of
    from paper_1904_10585_b200.dist import broadcast_nccl_id, max_over_ranks
    res = {}
    ident = broadcast_nccl_id(make_id=lambda: bytes(range(128)))
    res["id_ok"] = ident == bytes(range(128))
    cfg = reduced(CONFIGS[2], n=203)
    r0, r1 = rows_of(cfg.n, rank, world)
    prob = pfpg_problem(cfg)
    parts = [None] * world
    dist.all_gather_object(parts, (r0, r1, initial_block(cfg)[r0:r1], prob["omega_bits"][r0:r1]))
    res["parts"] = parts
    res["tmax"] = max_over_ranks(float(rank + 1))
    out[rank] = res
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_partition_and_plumbing():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    cfg = reduced(CONFIGS[2], n=203)
    full_U = initial_block(cfg)
    full_bits = pfpg_problem(cfg)["omega_bits"]
    for rank in range(world):
        res = out[rank]
        assert res["id_ok"]
        assert res["tmax"] == 2.0
        parts = res["parts"]
        # contiguous, disjoint, covering [0, n)
        assert parts[0][0] == 0 and parts[-1][1] == cfg.n
        assert all(parts[g][1] == parts[g + 1][0] for g in range(world - 1))
        np.testing.assert_array_equal(np.concatenate([q[2] for q in parts]), full_U)
        np.testing.assert_array_equal(np.concatenate([q[3] for q in parts]), full_bits)


def test_rows_of_matches_c_split():
    from paper_1904_10585_b200.solver import rows_of
    for n in (1, 7, 16384, 32768, 65537):
        for world in (1, 2, 3, 4, 8):
            cuts = [rows_of(n, g, world) for g in range(world)]
            assert cuts[0][0] == 0 and cuts[-1][1] == n
            for g in range(world):
                assert cuts[g][0] == g * n // world          # pf_api.cu: row0 = rank * n / world
                assert cuts[g][1] - cuts[g][0] in (n // world, n // world + 1)


def _worker_tf32(rank, world, port, out):
    """TF32 row-block layout: each rank holds the p-major slab Y^T[:, r0:r1] (p x n_local); the
    NCCL all-gather concatenates slabs rank-major ([world][p][n_local]) and the filter GEMM
    addresses column k of Y^T as slab k // n_local, offset k % n_local (3-D TMA coordinates
    (k % n_local, c, k // n_local), pf_gemm_tf32.cu)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    from paper_1904_10585_b200.solver import rows_of
    cfg = reduced(CONFIGS[5], n=16 * world * 7, p=64)
    r0, r1 = rows_of(cfg.n, rank, world)
    slab = torch.from_numpy(np.ascontiguousarray(initial_block(cfg)[r0:r1].T)).float()
    gathered = [torch.empty_like(slab) for _ in range(world)]
    dist.all_gather(gathered, slab)                  # rank-major, as ncclAllGather lays it out
    out[rank] = (r1 - r0, torch.stack(gathered).numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_tf32_gathered_layout_addressing():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_tf32, args=(world, _free_port(), out), nprocs=world, join=True)
    cfg = reduced(CONFIGS[5], n=16 * world * 7, p=64)
    Yt = initial_block(cfg).T.astype(np.float32)     # p x n
    for rank in range(world):
        nl, g = out[rank]
        assert nl % 16 == 0 and g.shape == (world, cfg.p, nl)
        k = np.arange(cfg.n)
        # the kernel's 3-D coordinates: (k % n_local, c, k // n_local)
        np.testing.assert_array_equal(g[k // nl, :, k % nl].T, Yt)
