"""PFSVT (NEXT-3) on the GPU against numpy / the oracle (oracle/pf_svt.py): the sparse kernels
(pf_spmm CSR and CSC-with-perm, pf_svt_ritz, pf_svt_update) element by element, then PFSVT
trajectories (X^k = U diag(s) V^T, svp, residual) at the fp64 bar, and the full m = n = 1000
tab:SVT-MKL case to convergence."""
import numpy as np
import pytest
import scipy.sparse as sp
import torch

import oracle as O
from pfinputs import NEXT_CONFIGS, reduced, svt_problem

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a B200")]


def _dev(a, dt=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dt).cuda()


def _ctx(n, p):
    from paper_1904_10585_b200._lib import Context
    return Context(n, p, 4)


def _problem(n=700, r=5, sr=0.07):
    cfg = reduced(NEXT_CONFIGS["svt1k"], n=n, r=r, sr=sr)
    prob = svt_problem(cfg)
    # ragged rows: empty the first three rows of Omega
    return cfg, prob


@pytest.mark.parametrize("p", [16, 32, 64, 128])
def test_spmm_csr_and_transpose(p):
    n = 700
    rs = np.random.default_rng(p)
    S = sp.random(n, n, density=0.03, random_state=p, format="csr")
    S[:3] = 0.0
    S.eliminate_zeros()
    S.sort_indices()
    val = rs.standard_normal(S.nnz)
    S.data[:] = val
    X = rs.standard_normal((n, p))
    Yc, Yp = rs.standard_normal((n, p)), rs.standard_normal((n, p))
    ctx = _ctx(n, p)
    out = torch.empty((n, p), dtype=torch.float64, device="cuda")
    i32 = lambda a: _dev(a.astype(np.int32), torch.int32)
    ctx.spmm(i32(S.indptr), i32(S.indices), _dev(val), _dev(X), out, (0.7, -0.3, 2.0),
             ycur=_dev(Yc), yprev=_dev(Yp))
    want = 0.7 * (S @ X) - 0.3 * Yc + 2.0 * Yp
    np.testing.assert_allclose(out.cpu().numpy(), want, rtol=1e-13, atol=1e-13)
    # S^T through the CSC view of the same values: perm maps CSC positions to CSR positions
    rows, cols = np.repeat(np.arange(n), np.diff(S.indptr)), S.indices
    perm = np.lexsort((rows, cols)).astype(np.int32)
    col_ptr = np.zeros(n + 1, np.int32)
    np.cumsum(np.bincount(cols, minlength=n), out=col_ptr[1:])
    ctx.spmm(i32(col_ptr), i32(rows[perm]), _dev(val), _dev(X), out, vperm=i32(perm))
    np.testing.assert_allclose(out.cpu().numpy(), S.T @ X, rtol=1e-13, atol=1e-13)


def test_svt_ritz_and_update():
    cfg, prob = _problem()
    n, p = cfg.n, 32
    rs = np.random.default_rng(1)
    x = rs.standard_normal(prob["b"].size)
    S = O.svt_matrix(prob, x, n)
    Q, _ = np.linalg.qr(rs.standard_normal((n, p)))
    ctx = _ctx(n, p)
    i32 = lambda a: _dev(a, torch.int32)
    U = torch.empty((n, p), dtype=torch.float64, device="cuda")
    V = torch.empty_like(U)
    sig = torch.empty(p, dtype=torch.float64, device="cuda")
    s = torch.empty_like(sig)
    svp = torch.zeros(1, dtype=torch.int32, device="cuda")
    mu = 0.5 * np.linalg.norm(S @ Q, 2)
    ctx.svt_ritz(i32(prob["row_ptr"]), i32(prob["J"]), _dev(x), _dev(Q), mu, U, V, sig, s, svp)
    Ur, sr_, Vr = O.svt_ritz(S, Q)
    np.testing.assert_allclose(sig.cpu().numpy(), sr_, rtol=1e-12, atol=1e-12 * sr_[0])
    # basis-invariant: U diag(sigma) V^T = (Y Q) Q^T
    Ug, Vg, sg = U.cpu().numpy(), V.cpu().numpy(), sig.cpu().numpy()
    assert O.lowrank_rect_diff_fro(Ug, sg, Vg, Ur, sr_, Vr) <= 1e-12 * O.lowrank_rect_fro(Ur, sr_, Vr)
    sh = np.maximum(sr_ - mu, 0.0)
    np.testing.assert_allclose(s.cpu().numpy(), sh, rtol=1e-12, atol=1e-12 * sr_[0])
    assert int(svp.item()) == int((sh > 0).sum())
    # the dual step on Omega
    xd = _dev(x)
    rss = torch.zeros(1, dtype=torch.float64, device="cuda")
    ctx.svt_update(i32(prob["row_ptr"]), i32(prob["J"]), _dev(prob["b"]), xd, U, V, s, 1.7, rss)
    w = O.svt_sample(Ug, s.cpu().numpy(), Vg, prob["I"], prob["J"])
    np.testing.assert_allclose(xd.cpu().numpy(), x + 1.7 * (prob["b"] - w), rtol=1e-12, atol=1e-12)
    assert float(rss.item()) == pytest.approx(float(np.sum((prob["b"] - w) ** 2)), rel=1e-12)


@pytest.mark.parametrize("d,p", [(1, 16), (3, 16), (1, 64)])
def test_pfsvt_trajectory_matches_oracle(d, p):
    from paper_1904_10585_b200 import run_svt
    cfg = reduced(NEXT_CONFIGS["svt1k"], n=600, r=5, sr=0.25, p=p, d=d, iters=15)
    prob = svt_problem(cfg)
    ref = O.pfsvt_run(cfg, prob)["records"]
    got = run_svt(cfg, problem=prob)["records"]
    for x, y in zip(ref, got):
        assert x["svp"] == y["svp"]
        den = max(O.lowrank_rect_fro(x["U"], x["s"], x["V"]), 1e-300)
        assert O.lowrank_rect_diff_fro(x["U"], x["s"], x["V"], y["U"], y["s"], y["V"]) <= 1e-10 * den
        assert y["res"] == pytest.approx(x["res"], rel=1e-9)


def test_pfsvt_converges_like_tab_svt_mkl():
    """m = n = 1000, SR 20%, r = 10: the GPU run stops at the oracle's iteration (paper: 78),
    recovers rank 10 and mse ~ 1.4e-4."""
    from paper_1904_10585_b200 import run_svt
    cfg = NEXT_CONFIGS["svt1k"]
    prob = svt_problem(cfg)
    ref = O.pfsvt_run(cfg, prob, stop=True, record_factors=False)["records"]
    got = run_svt(cfg, problem=prob, stop=True)["records"]
    assert abs(len(got) - len(ref)) <= 1
    last = got[-1]
    assert last["svp"] == cfg.r and last["res"] <= cfg.svt_tol
    M = prob["ML"] @ prob["MR"].T
    mse = np.linalg.norm((last["U"] * last["s"]) @ last["V"].T - M) / np.linalg.norm(M)
    assert 0.5e-4 <= mse <= 2.5e-4


def test_adaptive_block_size_matches_oracle():
    """NEXT-2 (reading R27): p_k = the smallest of 16/32/64 >= svp_{k-1} + 5, grown blocks
    completed with the seeded guard columns; the GPU follows the oracle's block sizes and
    iterates (r = 20, so the block grows 16 -> 32 during the run)."""
    from paper_1904_10585_b200 import run_svt
    cfg = reduced(NEXT_CONFIGS["svt5k"], n=800, r=20, sr=0.3, p=64, iters=14, svt_adapt=True)
    prob = svt_problem(cfg)
    ref = O.pfsvt_run(cfg, prob)["records"]
    got = run_svt(cfg, problem=prob)["records"]
    assert len({r["p"] for r in ref}) > 1, [r["p"] for r in ref]
    for x, y in zip(ref, got):
        assert x["p"] == y["p"] and x["svp"] == y["svp"]
        den = max(O.lowrank_rect_fro(x["U"], x["s"], x["V"]), 1e-300)
        assert O.lowrank_rect_diff_fro(x["U"], x["s"], x["V"], y["U"], y["s"], y["V"]) <= 1e-10 * den
