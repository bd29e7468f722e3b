"""CUDA-graph replay of the iteration body (Solver(graphs=True)): the same kernels in the same
order on the same buffers, so the trajectory must be bit-identical to the eager one."""
import numpy as np
import pytest
import torch

from pfinputs import CONFIGS, NEXT_CONFIGS, reduced

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a B200")]


@pytest.mark.parametrize("cfg", [CONFIGS[1],
                                 reduced(CONFIGS[2], n=1000, iters=12),
                                 reduced(CONFIGS[3], n=1500, iters=12, edge_prob=82 / 1500),
                                 reduced(CONFIGS[5], n=2048, p=128, nbig=40, nrefl=16, iters=4),
                                 reduced(NEXT_CONFIGS["nce7"], n=600, iters=8)],
                         ids=["sweep", "pfpg", "pfam", "tf32", "nce"])
def test_graph_replay_is_bit_identical(cfg):
    from paper_1904_10585_b200 import run
    a = run(cfg)
    b = run(cfg, graphs=True)
    sb = b["solver"]
    assert sb.graphs and len(sb._graph) == 2 and all(v > 0 for v in sb.graph_launches.values())
    for x, y in zip(a["records"], b["records"]):
        assert np.array_equal(x["theta"], y["theta"])
        assert np.array_equal(x["f"], y["f"]) and np.array_equal(x["V"], y["V"])
        if "objective" in x:
            assert x["objective"] == y["objective"] and x["aux"] == y["aux"]
    assert a["status"]["names"] == b["status"]["names"]
