"""The row-block split (include/pf.h pf_create_dist) with W ranks on ONE GPU through
the in-process loopback communicator (pf_create_loop, csrc/pf_comm.cu): W contexts, one host thread
and one stream each, every exchange a host rendezvous plus stream-ordered copies / a fixed-order sum.
This executes every row0 > 0 path of the library (row-local diagonals and mask offsets in the
rebuild / prox / admm / nce / rna / perturb kernels, ragged row blocks, the gathered B operand,
replicated Cholesky / Jacobi / f) and compares:

  * the assembled trajectory (V rows concatenated in rank order) against the oracle at the fp64
    bar (1e-10) / the TF32 bar (1e-4) on X_k and the objective (north_star);
  * theta, f, rank and the objective BIT-identical across ranks -- the all-reduce delivers the
    same bits to every rank, so the replicated p x p work agrees exactly (asserted).
"""
import numpy as np
import pytest
import torch

import oracle as O
from pfinputs import CONFIGS, NEXT_CONFIGS, reduced, pfpg_problem, pfam_problem, nce_problem

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a B200")]


def _problem(cfg):
    if cfg.mode == "pfpg":
        return pfpg_problem(cfg)
    if cfg.mode == "pfam":
        return pfam_problem(cfg)
    if cfg.mode == "nce":
        return nce_problem(cfg)
    return None


def _check(cfg, world, tol):
    from paper_1904_10585_b200.dist import run_loopback
    prob = _problem(cfg)
    ref = O.run(cfg, problem=prob)["records"]
    outs = run_loopback(cfg, world, problem=prob)
    recs = [o["records"] for o in outs]
    n_rows = [o["solver"].n_local for o in outs]
    assert sum(n_rows) == cfg.n
    for k, r in enumerate(ref):
        per = [rr[k] for rr in recs]
        g0 = per[0]
        for g in per[1:]:                                  # replicated objects: same bits
            assert np.array_equal(g["theta"], g0["theta"]), ("theta", k)
            assert np.array_equal(g["f"], g0["f"]) and g["rank"] == g0["rank"], ("f", k)
            if "objective" in g0:
                assert g["objective"] == g0["objective"] and g["aux"] == g0["aux"], ("obj", k)
            if "x" in g0:
                pass                                        # x is row-distributed
        V = np.concatenate([g["V"] for g in per], axis=0)  # rank order = row order
        den = max(O.lowrank_fro(r["V"], r["f"]), 1e-300)
        err = O.lowrank_diff_fro(V, g0["f"], r["V"], r["f"]) / den
        assert err <= tol, (k, err)
        if "objective" in r:
            assert abs(g0["objective"] - r["objective"]) <= tol * max(1.0, abs(r["objective"])), k
        if "x" in r:
            x = np.concatenate([g["x"] for g in per])
            assert np.abs(x - r["x"]).max() <= tol * max(1.0, np.abs(r["x"]).max()), k


CASES = [
    (reduced(CONFIGS[2], n=1001, iters=6), 2, 1e-10),
    (reduced(CONFIGS[2], n=1001, iters=6, dtype="f64i8"), 3, 1e-10),
    (reduced(CONFIGS[3], n=1501, iters=6, edge_prob=82 / 1501), 3, 1e-10),
    (reduced(CONFIGS[3], n=1501, iters=6, edge_prob=82 / 1501, dtype="f64i8"), 2, 1e-10),
    (reduced(CONFIGS[4], n=1203, p=128, iters=4), 4, 1e-10),
    (reduced(CONFIGS[4], n=1203, p=128, iters=4, dtype="f64i8"), 2, 1e-10),
    (reduced(CONFIGS[1], iters=5), 3, 1e-10),
    (reduced(CONFIGS[5], n=2048, p=128, nbig=40, nrefl=16, iters=3), 2, 1e-4),
    (reduced(CONFIGS[5], n=2048, p=64, nbig=24, nrefl=16, iters=3), 4, 1e-4),
    (reduced(NEXT_CONFIGS["nce7a"], n=401, p=32, iters=8), 3, 1e-10),
]
IDS = ["pfpg_w2", "pfpg_i8_w3", "pfam_w3", "pfam_i8_w2", "pfpg_p128_w4", "pfpg_p128_i8_w2",
       "sweep_w3", "tf32_w2", "tf32_p64_w4", "nce_rna_w3"]


@pytest.mark.parametrize("cfg,world,tol", CASES, ids=IDS)
def test_loopback_split_matches_oracle(cfg, world, tol):
    _check(cfg, world, tol)


def test_loopback_world1_matches_plain_context(monkeypatch):
    """world = 1: the loopback context runs the distributed code path (gathers through the
    communicator, no one-GPU shortcuts) -- same arithmetic as the plain context with the
    shortcuts off."""
    from paper_1904_10585_b200 import run
    from paper_1904_10585_b200.dist import run_loopback
    monkeypatch.setenv("PF_LZ_SYM", "0")
    monkeypatch.setenv("PF_FUSE_DIGITS", "0")
    monkeypatch.setenv("PF_K7TMA", "0")
    cfg = reduced(CONFIGS[3], n=900, iters=4, edge_prob=0.09)
    a = run(cfg)["records"]
    b = run_loopback(cfg, 1)[0]["records"]
    for x, y in zip(a, b):
        assert np.array_equal(x["theta"], y["theta"])
        assert x["objective"] == y["objective"]


def test_loopback_missing_peer_times_out(monkeypatch):
    """A rank whose peer never reaches the collective fails with PF_ERR_NCCL after the hub's
    rendezvous timeout (PF_LOOP_TIMEOUT_S, read at pf_loop_create) instead of hanging, and the
    aborted hub fails every later collective at once."""
    import time
    from paper_1904_10585_b200._lib import Context, Loopback, PFError
    monkeypatch.setenv("PF_LOOP_TIMEOUT_S", "2")
    hub = Loopback(2)
    n, p = 512, 32
    c = Context(n, p, 4, rank=0, world=2, loop=hub)
    U = torch.randn(c.n_local, p, dtype=torch.float64, device="cuda")
    t0 = time.time()
    with pytest.raises(PFError, match="PF_ERR_NCCL"):
        c.orth(U)                                   # rank 1 never arrives
    assert 1.5 <= time.time() - t0 < 30
    t0 = time.time()
    with pytest.raises(PFError, match="PF_ERR_NCCL"):
        c.orth(U)
    assert time.time() - t0 < 1.0


@pytest.mark.parametrize("world", [2, 4])
def test_overlapped_gather_matches_single_gather(world, monkeypatch):
    """TF32 row-block split, the config-5 path: the slab-by-slab GEMM overlapped with the
    slab-by-slab gather (PF_OVERLAP=1, the default) against one all-gather then one GEMM
    (PF_OVERLAP=0).  The slab sums regroup the fp32 accumulation, so the two agree to fp32
    rounding (not bit for bit); both match the oracle at the TF32 bar."""
    from paper_1904_10585_b200.dist import run_loopback
    cfg = reduced(CONFIGS[5], n=2048, p=128, nbig=40, nrefl=16, iters=3)
    ref = O.run(cfg)["records"]
    outs = {}
    for ov in ("1", "0"):
        monkeypatch.setenv("PF_OVERLAP", ov)
        outs[ov] = run_loopback(cfg, world)
    for k, r in enumerate(ref):
        Vs = {}
        for ov, out in outs.items():
            per = [o["records"][k] for o in out]
            V = np.concatenate([g["V"] for g in per], axis=0)
            Vs[ov] = (V, per[0]["f"])
            den = O.lowrank_fro(r["V"], r["f"])
            assert O.lowrank_diff_fro(V, per[0]["f"], r["V"], r["f"]) <= 1e-4 * den, (ov, k)
        d = O.lowrank_diff_fro(*Vs["1"], *Vs["0"]) / O.lowrank_fro(*Vs["0"])
        assert d <= 1e-5, (k, d)
