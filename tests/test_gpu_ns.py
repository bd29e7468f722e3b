"""Rayleigh-Ritz + spectral operator by Newton-Schulz sign iterations (pf_rr_ns, NEXT-4, reading
R26): F = f(U^T A U) against numpy's eigendecomposition, for both spectral operators and both
storage paths; sweep trajectories against the oracle (also replayed as CUDA graphs: the iteration
runs on the device, no host synchronisation); the device-side Jacobi fallback."""
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
    it = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.rr_ns(torch.from_numpy(A).cuda(), torch.from_numpy(U).cuda(), op, thr, F, rank, it)
    want, r = _f(U.T @ A @ U, op, thr)
    assert it.item() > 0
    assert "NS_FALLBACK" not in ctx.status()["names"]
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


@pytest.mark.parametrize("p,tf32", [(16, False), (32, False), (128, False), (256, True),
                                    (512, True)])
def test_rr_ns_sizes_and_symmetry(p, tf32):
    """Tile edges (p < 32 is padded inside the kernel), the two-sign soft threshold at every
    block width, and the exact symmetry of F (every product is formed on upper tiles and
    mirrored)."""
    from paper_1904_10585_b200._lib import Context, PF_TF32
    n = max(3 * p, 600)
    rs = np.random.default_rng(p)
    q, _ = np.linalg.qr(rs.standard_normal((n, n)))
    lam = np.concatenate([rs.uniform(2, 9, p // 3), rs.uniform(-1.5, 1.5, n - p // 3)])
    A = (q * lam) @ q.T
    A = 0.5 * (A + A.T)
    U, _ = np.linalg.qr(rs.standard_normal((n, p)))
    if tf32:
        ctx = Context(n, p, 4, dtype=PF_TF32)
        A32 = A.astype(np.float32)
        A32 = np.triu(A32) + np.triu(A32, 1).T
        U32 = np.ascontiguousarray(U.T.astype(np.float32))
        Ad, Ud = torch.from_numpy(A32).cuda(), torch.from_numpy(U32).cuda()
        Uf = U32.T.astype(np.float64)
        H, tol = Uf.T @ A32.astype(np.float64) @ Uf, 1e-5
    else:
        ctx = Context(n, p, 4)
        Ad, Ud = torch.from_numpy(A).cuda(), torch.from_numpy(U).cuda()
        H, tol = U.T @ A @ U, 1e-11
    F = torch.empty((p, p), dtype=torch.float64, device="cuda")
    rank = torch.zeros(1, dtype=torch.int32, device="cuda")
    ctx.rr_ns(Ad, Ud, 1, 1.0, F, rank)
    Fh = F.cpu().numpy()
    assert np.array_equal(Fh, Fh.T)
    want, r = _f(H, 1, 1.0)
    np.testing.assert_allclose(Fh, want, rtol=0, atol=tol * np.abs(H).max())
    assert int(rank.item()) == r


@pytest.mark.parametrize("cfg,tol,graphs", [
    (reduced(CONFIGS[1], rr_ns=True), 1e-10, False),
    (reduced(CONFIGS[1], rr_ns=True), 1e-10, True),
    (reduced(CONFIGS[5], n=2048, p=128, nbig=40, nrefl=16, iters=4, rr_ns=True), 1e-4, False),
    (reduced(CONFIGS[5], n=2048, p=512, nbig=40, nrefl=16, iters=3, rr_ns=True), 1e-4, True)],
    ids=["sweep_psd_fp64", "sweep_psd_fp64_graphs", "sweep_soft_tf32", "sweep_soft_tf32_p512_graphs"])
def test_ns_trajectory_matches_oracle(cfg, tol, graphs):
    from paper_1904_10585_b200 import run
    ref = O.run(reduced(cfg, rr_ns=False))["records"]
    got = run(cfg, graphs=graphs)["records"]
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
    PF_NS_MAXIT knob, read once per process -- so this test runs in a subprocess) the same
    pf_rr_ns call runs the cooperative Jacobi solver on the device and forms F = Y f(theta) Y^T;
    PF_FLAG_NS_FALLBACK is set and the trajectory still matches the oracle."""
    import subprocess
    import sys
    import textwrap
    code = textwrap.dedent("""
        import numpy as np, torch, oracle as O
        from pfinputs import CONFIGS, reduced
        from paper_1904_10585_b200 import run
        from paper_1904_10585_b200._lib import Context
        n, p = 200, 16
        rs = np.random.default_rng(3)
        A = rs.standard_normal((n, n)); A = A + A.T
        U, _ = np.linalg.qr(rs.standard_normal((n, p)))
        ctx = Context(n, p, 4)
        F = torch.empty((p, p), dtype=torch.float64, device="cuda")
        rank = torch.zeros(1, dtype=torch.int32, device="cuda")
        it = torch.zeros(1, dtype=torch.int32, device="cuda")
        ctx.rr_ns(torch.from_numpy(A).cuda(), torch.from_numpy(U).cuda(), 0, 0.0, F, rank, it)
        assert it.item() == -1 and "NS_FALLBACK" in ctx.status()["names"]
        lam, W = np.linalg.eigh(U.T @ A @ U)
        want = (W * np.maximum(lam, 0)) @ W.T
        assert np.abs(F.cpu().numpy() - want).max() <= 1e-11 * np.abs(want).max()
        assert rank.item() == int((lam > 0).sum())
        # p = 256 (TF32 context): the cooperative Jacobi fallback
        from paper_1904_10585_b200._lib import PF_TF32
        n, p = 1024, 256
        q, _ = np.linalg.qr(rs.standard_normal((n, n)))
        lam0 = np.concatenate([rs.uniform(5, 50, 40), rs.uniform(-1, 1, n - 40)])
        A32 = ((q * lam0) @ q.T).astype(np.float32)
        A32 = np.triu(A32) + np.triu(A32, 1).T
        U32 = np.ascontiguousarray(np.linalg.qr(rs.standard_normal((n, p)))[0].T.astype(np.float32))
        c32 = Context(n, p, 4, dtype=PF_TF32)
        F = torch.empty((p, p), dtype=torch.float64, device="cuda")
        c32.rr_ns(torch.from_numpy(A32).cuda(), torch.from_numpy(U32).cuda(), 1, 3.0, F, rank, it)
        assert it.item() == -1 and "NS_FALLBACK" in c32.status()["names"]
        Uf = U32.T.astype(np.float64)
        lam, W = np.linalg.eigh(Uf.T @ A32.astype(np.float64) @ Uf)
        fl = np.sign(lam) * np.maximum(np.abs(lam) - 3.0, 0.0)
        want = (W * fl) @ W.T
        assert np.abs(F.cpu().numpy() - want).max() <= 1e-5 * np.abs(want).max()
        assert rank.item() == int((fl != 0).sum())
        cfg = reduced(CONFIGS[1], iters=4, rr_ns=True)
        out = run(cfg, graphs=True)
        ref = O.run(reduced(cfg, rr_ns=False))["records"]
        for x, y in zip(ref, out["records"]):
            one = np.ones(y["Q"].shape[1])
            err = O.lowrank_rect_diff_fro(x["V"] * x["f"], np.ones(x["f"].size), x["V"],
                                          y["QF"], one, y["Q"])
            assert err <= 1e-10 * O.lowrank_fro(x["V"], x["f"]), (x["k"], err)
            assert y["ns_iters"] == -1
        print("fallback ok")
    """)
    import os
    env = dict(os.environ, PF_NS_MAXIT="3")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "fallback ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("cfg,graphs", [
    (reduced(CONFIGS[3], n=1100, iters=6, edge_prob=0.07, rr_ns=True), False),
    (reduced(CONFIGS[3], n=1100, iters=6, edge_prob=0.07, rr_ns=True, dtype="f64i8"), True),
    (reduced(CONFIGS[3], n=1500, iters=4, edge_prob=82 / 1500, p=32, rr_ns=True), False)],
    ids=["pfam_f64", "pfam_i8_graphs", "pfam_p32"])
def test_pfam_matrix_form_matches_oracle(cfg, graphs):
    """PFAM with the Rayleigh-Ritz spectral operator in matrix form (reading R30): H positive
    definite -> F = H (no eigensolver), else Newton-Schulz; the update W = Q F Q^T
    (pf_admm_step_f, fused digits on the int8 path).  X_k and <C, W> vs the oracle's
    eigendecomposition route at the fp64 bar."""
    from paper_1904_10585_b200 import run
    ref = O.run(reduced(cfg, rr_ns=False))["records"]
    got = run(cfg, graphs=graphs)["records"]
    for x, y in zip(ref, got):
        one = np.ones(y["Q"].shape[1])
        den = O.lowrank_fro(x["V"], x["f"])
        err = O.lowrank_rect_diff_fro(x["V"] * x["f"], np.ones(x["f"].size), x["V"],
                                      y["QF"], one, y["Q"])
        assert err <= 1e-10 * den, (x["k"], err / den)
        assert y["rank"] == x["rank"]
        assert y["objective"] == pytest.approx(x["objective"], rel=1e-10)
        assert y["aux"] == pytest.approx(x["residual"], rel=1e-9)


def test_admm_step_f_matches_oracle():
    """pf_admm_step_f on random data: Z_new = offdiag(Q F Q^T - tC) + Diag(1 - W_ii + Z_ii)
    element by element, <C, W> and ||Z_new - Z||_F, against the oracle's pfam_next on the
    eigen-factors of F."""
    from paper_1904_10585_b200._lib import Context
    from pfinputs import pfam_problem, unpack_bitmask
    from paper_1904_10585_b200.solver import _bits
    cfg = reduced(CONFIGS[3], n=777, edge_prob=0.1)
    prob = pfam_problem(cfg)
    n, p = cfg.n, 64
    rs = np.random.default_rng(4)
    Q = np.linalg.qr(rs.standard_normal((n, p)))[0]
    B = rs.standard_normal((p, p))
    F = B @ B.T / p
    Z = rs.standard_normal((n, n)) * 0.1
    Z = Z + Z.T
    lam, Y = np.linalg.eigh(F)
    C = O.maxcut_C(unpack_bitmask(prob["adj_bits"], n), prob["deg"])
    Zr, cw, res = O.pfam_next(Q @ Y, lam, Z, C, 1.0)
    c = Context(n, p, 4)
    Zd = torch.from_numpy(Z.copy()).cuda()
    obj = torch.zeros(2, dtype=torch.float64, device="cuda")
    c.admm_step_f(torch.from_numpy(Q).cuda(), torch.from_numpy(F).cuda(), 1.0,
                  _bits(prob["adj_bits"]), torch.from_numpy(prob["deg"]).cuda(), Zd, obj)
    np.testing.assert_allclose(Zd.cpu().numpy(), Zr, rtol=0, atol=1e-13 * np.abs(Zr).max())
    o = obj.cpu().numpy()
    assert o[0] == pytest.approx(cw, rel=1e-12) and o[1] == pytest.approx(res, rel=1e-11)
