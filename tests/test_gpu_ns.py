"""Rayleigh-Ritz + spectral operator by Newton-Schulz sign iterations (pf_rr_ns, NEXT-4, reading
R26): F = f(U^T A U) against numpy's eigendecomposition, for both spectral operators and both
storage paths; sweep trajectories against the oracle; the breakdown fallback."""
import numpy as np
import pytest
import torch

import oracle as O
from pfinputs import CONFIGS, reduced

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a B200")]


def _f(H, op, thr):
    lam, W = np.linalg.eigh(0.5 * (H + H.T))
    f = np.maximum(lam, 0.0) if op == 0 else np.sign(lam) * np.maximum(np.abs(lam) - thr, 0.0)
    return (W * f) @ W.T, int((f != 0).sum())


@pytest.mark.parametrize("op", [0, 1])
def test_rr_ns_fp64(op):
    from paper_1904_10585_b200._lib import Context
    n, p = 600, 64
    rs = np.random.default_rng(op)
    q, _ = np.linalg.qr(rs.standard_normal((n, n)))
    lam = np.concatenate([rs.uniform(2, 9, 20), rs.uniform(-1.5, 1.5, n - 20)])
    A = (q * lam) @ q.T
    A = 0.5 * (A + A.T)
    U, _ = np.linalg.qr(rs.standard_normal((n, p)))
    ctx = Context(n, p, 4)
    F = torch.empty((p, p), dtype=torch.float64, device="cuda")
    rank = torch.zeros(1, dtype=torch.int32, device="cuda")
    thr = 1.0
    it = ctx.rr_ns(torch.from_numpy(A).cuda(), torch.from_numpy(U).cuda(), op, thr, F, rank)
    want, r = _f(U.T @ A @ U, op, thr)
    assert it > 0
    np.testing.assert_allclose(F.cpu().numpy(), want, rtol=0, atol=1e-11 * np.abs(want).max())
    assert int(rank.item()) == r


def test_rr_ns_tf32_matches_eigh():
    from paper_1904_10585_b200._lib import Context, PF_TF32
    n, p = 2048, 128
    rs = np.random.default_rng(7)
    q, _ = np.linalg.qr(rs.standard_normal((n, n)))
    lam = np.concatenate([rs.uniform(5, 50, 40), rs.uniform(-1, 1, n - 40)])
    A = ((q * lam) @ q.T).astype(np.float32)
    A = np.triu(A) + np.triu(A, 1).T
    U, _ = np.linalg.qr(rs.standard_normal((n, p)))
    U32 = np.ascontiguousarray(U.T.astype(np.float32))           # p-major blocks
    ctx = Context(n, p, 4, dtype=PF_TF32)
    F = torch.empty((p, p), dtype=torch.float64, device="cuda")
    rank = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.rr_ns(torch.from_numpy(A).cuda(), torch.from_numpy(U32).cuda(), 1, 3.0, F, rank)
    Uf = U32.T.astype(np.float64)
    want, r = _f(Uf.T @ A.astype(np.float64) @ Uf, 1, 3.0)
    np.testing.assert_allclose(F.cpu().numpy(), want, rtol=0, atol=1e-5 * np.abs(want).max())
    assert int(rank.item()) == r


@pytest.mark.parametrize("cfg,tol", [
    (reduced(CONFIGS[1], rr_ns=True), 1e-10),
    (reduced(CONFIGS[5], n=2048, p=128, nbig=40, nrefl=16, iters=4, rr_ns=True), 1e-4)],
    ids=["sweep_psd_fp64", "sweep_soft_tf32"])
def test_ns_trajectory_matches_oracle(cfg, tol):
    from paper_1904_10585_b200 import run
    ref = O.run(reduced(cfg, rr_ns=False))["records"]
    got = run(cfg)["records"]
    for x, y in zip(ref, got):
        den = O.lowrank_fro(x["V"], x["f"])
        if "QF" in y:
            one = np.ones(y["Q"].shape[1])
            err = O.lowrank_rect_diff_fro(x["V"] * x["f"], np.ones(x["f"].size), x["V"],
                                          y["QF"], one, y["Q"])
        else:   # a Jacobi fallback iteration
            err = O.lowrank_diff_fro(x["V"], x["f"], y["V"], y["f"])
        assert err <= tol * den, (x["k"], err / den)
        assert y["rank"] == x["rank"]


def test_ns_breakdown_falls_back_to_jacobi(monkeypatch):
    """When the sign iterations do not converge (forced here by capping them at 3 with the
    PF_NS_MAXIT knob) pf_rr_ns returns PF_ERR_BREAKDOWN and the solver runs Jacobi for that
    iteration: the trajectory still matches the oracle."""
    from paper_1904_10585_b200 import run
    from paper_1904_10585_b200._lib import Context, PFError
    monkeypatch.setenv("PF_NS_MAXIT", "3")
    n, p = 200, 16
    rs = np.random.default_rng(3)
    A = rs.standard_normal((n, n))
    A = A + A.T
    U, _ = np.linalg.qr(rs.standard_normal((n, p)))
    ctx = Context(n, p, 4)
    F = torch.empty((p, p), dtype=torch.float64, device="cuda")
    rank = torch.zeros(1, dtype=torch.int32, device="cuda")
    with pytest.raises(PFError, match="BREAKDOWN"):
        ctx.rr_ns(torch.from_numpy(A).cuda(), torch.from_numpy(U).cuda(), 0, 0.0, F, rank)
    cfg = reduced(CONFIGS[1], iters=4, rr_ns=True)
    out = run(cfg)
    assert out["solver"].ns_fallbacks == 4
    ref = O.run(reduced(cfg, rr_ns=False))["records"]
    for x, y in zip(ref, out["records"]):
        assert O.lowrank_diff_fro(x["V"], x["f"], y["V"], y["f"]) <= 1e-10 * O.lowrank_fro(x["V"], x["f"])
