"""The NCCL (distributed) code path of libpf.so on one GPU: a single-rank communicator runs the
same gathers / all-reduces as the multi-rank split; results must match the plain context."""
import numpy as np
import pytest
import torch

import oracle as O
from pfinputs import CONFIGS, reduced

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a B200")]


@pytest.mark.parametrize("cfg", [reduced(CONFIGS[3], n=1500, iters=6, edge_prob=82 / 1500),
                                 reduced(CONFIGS[2], n=1000, iters=6),
                                 reduced(CONFIGS[1], iters=4),
                                 reduced(CONFIGS[5], n=2048, p=128, nbig=40, nrefl=16, iters=3),
                                 reduced(CONFIGS[3], n=1500, iters=4, edge_prob=82 / 1500,
                                         dtype="f64i8")],
                         ids=["pfam", "pfpg", "sweep", "tf32_sweep", "pfam_i8"])
def test_single_rank_nccl_path_matches(cfg, monkeypatch):
    from paper_1904_10585_b200 import run
    from paper_1904_10585_b200._lib import nccl_unique_id
    # one-GPU-only shortcuts off (upper-triangle Lanczos GEMV, digits written by the PFAM
    # update): both runs then do the same arithmetic
    monkeypatch.setenv("PF_LZ_SYM", "0")
    monkeypatch.setenv("PF_FUSE_DIGITS", "0")
    monkeypatch.setenv("PF_K7TMA", "0")
    a = run(cfg)["records"]
    b = run(cfg, nccl_id=nccl_unique_id(), rank=0, world=1)["records"]
    for x, y in zip(a, b):
        den = max(O.lowrank_fro(x["V"], x["f"]), 1e-300)
        # fp64: same arithmetic; TF32: the B operand comes through the 3-D map of the gathered
        # block (same data, same schedule -> same bits)
        assert O.lowrank_diff_fro(x["V"], x["f"], y["V"], y["f"]) <= 1e-13 * den
        if "objective" in x:
            assert y["objective"] == pytest.approx(x["objective"], rel=1e-13)
            assert y["aux"] == pytest.approx(x["aux"], rel=1e-12)
