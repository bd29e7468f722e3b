"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

* config 2 (n = 4096): the first iterations of the trajectory against the oracle, element-wise
  on X_k (via factors) and the objective.
* config 3 (n = 16384, the bench workload): one-step parity -- the oracle is fed the GPU's own
  state (Z_k, U_{k-1}) after a few GPU iterations and runs the same iteration (filter, orth, RR,
  P_+, DRS update) in fp64 on the host; the GPU step from the same state must agree on X_k,
  <C, W>, ||Z+ - Z|| and on sampled entries of Z+ computed one by one.
* config 4 shape (n = 32768, p = 128, d = 10): one GPU step checked through properties that
  hold at any size (orthonormality, Ritz residuals of sampled Ritz pairs computed on the host,
  the update formula on sampled entries).
"""
import numpy as np
import pytest
import torch

import oracle as O
from pfinputs import CONFIGS, reduced, lanczos_start, pfam_problem, unpack_bitmask

pytestmark = [pytest.mark.gpu, pytest.mark.slow,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a B200")]


def _err(g, r):
    den = max(O.lowrank_fro(r["V"], r["f"]), 1e-300)
    return O.lowrank_diff_fro(g["V"], g["f"], r["V"], r["f"]) / den


@pytest.mark.parametrize("dtype", ["f64", "f64i8"])
def test_config2_fullsize_trajectory_prefix(dtype):
    from paper_1904_10585_b200 import run
    cfg = reduced(CONFIGS[2], dtype=dtype)
    K = 12
    ref = O.run(cfg, iters=K)["records"]
    got = run(cfg, iters=K, graphs=True)["records"]
    for r, g in zip(ref, got):
        assert _err(g, r) <= 1e-10, (r["k"], _err(g, r))
        assert abs(g["objective"] - r["objective"]) <= 1e-10 * abs(r["objective"])


@pytest.mark.parametrize("dtype", ["f64", "f64i8"])   # f64i8 + graphs: the bench's path
def test_config3_fullsize_one_step(dtype):
    from paper_1904_10585_b200 import Solver
    cfg = reduced(CONFIGS[3], dtype=dtype)
    prob = pfam_problem(cfg)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    s = Solver(cfg, problem=prob, stream=st, graphs=True)
    for _ in range(3):
        s.step()                                   # k = 0, 1, 2 on the GPU
    k = s.k                                        # next iteration index (3)
    Z = s.A.cpu().numpy()                          # Z_k (GPU state)
    U = s.U.cpu().numpy()                          # warm-start block (Ritz vectors of k-1)
    th_prev = s.theta.cpu().numpy()
    # ---- GPU step k from that state
    s.step()
    torch.cuda.synchronize()
    f_g = s.f.cpu().numpy()
    keep = f_g != 0
    V_g = s.ritz.cpu().numpy()[:, keep]
    cw_g, res_g = s.objective()
    Zg = s.A
    # ---- oracle step k from the same state and the interval the GPU used (one-step parity,
    # SURVEY §8(c) "shared interval" mode); re-basing is span-exact, so the oracle's plan is its own
    a, b = s.interval.cpu().numpy()
    C = O.maxcut_C(unpack_bitmask(prob["adj_bits"], cfg.n), prob["deg"])
    plan = O.rebase_plan(a, b, float(np.max(np.abs(th_prev))), cfg.d, cfg.rho_max)
    Uk = O.filter_update(Z, O.orth(U), a, b, cfg.d, 1, plan)
    th, V = O.rayleigh_ritz(Z, Uk)
    f = O.spectral_psd(th)
    Zn, cw, res = O.pfam_next(V[:, f != 0], f[f != 0], Z, C, cfg.t)
    err = O.lowrank_diff_fro(V_g, f_g[keep], V[:, f != 0], f[f != 0]) / O.lowrank_fro(V[:, f != 0], f[f != 0])
    assert err <= 1e-10, err
    assert abs(cw_g - cw) <= 1e-10 * abs(cw)
    assert abs(res_g - res) <= 1e-10 * abs(res)
    rng = np.random.default_rng(7)
    idx = rng.integers(0, cfg.n, size=(2000, 2))
    zs = Zg[torch.as_tensor(idx[:, 0]), torch.as_tensor(idx[:, 1])].cpu().numpy()
    np.testing.assert_allclose(zs, Zn[idx[:, 0], idx[:, 1]], rtol=0, atol=1e-10 * np.abs(Zn).max())
    torch.cuda.set_stream(torch.cuda.default_stream())


def test_config4_shape_fullsize_properties():
    """n = 32768, p = 128, d = 10 on one GPU: properties of one filtered PFPG step."""
    from paper_1904_10585_b200 import Context
    n, p, d = 32768, 128, 10
    rng = np.random.default_rng(11)
    # A = G + G^T / 2 scaled, built on the device from a seeded host factor (low rank + noise)
    torch.manual_seed(0)
    Wt = torch.randn(n, 50, dtype=torch.float64, device="cuda")
    A = (Wt @ Wt.T) / 50.0
    A += 0.01 * torch.randn(n, n, dtype=torch.float64, device="cuda")
    A = 0.5 * (A + A.T)
    U = torch.randn(n, p, dtype=torch.float64, device="cuda")
    ctx = Context(n, p, d)
    ctx.orth(U)
    lohi = torch.zeros(2, dtype=torch.float64, device="cuda")
    ctx.lanczos(A, torch.ones(n, dtype=torch.float64, device="cuda"), 20, lohi)  # re-base plan
    iv = torch.tensor([-3.0, 3.0], dtype=torch.float64, device="cuda")
    ctx.filter(A, U, iv, 1, 1e6)
    V = torch.empty_like(U)
    th = torch.empty(p, dtype=torch.float64, device="cuda")
    ctx.rayleigh_ritz(A, U, V, th)
    torch.cuda.synchronize()
    G = (U.T @ U).cpu().numpy()
    assert np.abs(G - np.eye(p)).max() < 1e-12
    Vh = V.cpu().numpy()
    thh = th.cpu().numpy()
    assert np.all(np.diff(thh) <= 0)
    # Ritz residuals of the 8 leading pairs on the host (one GEMV each, fp64)
    Ah = A.cpu().numpy()
    for i in range(8):
        r = Ah @ Vh[:, i] - thh[i] * Vh[:, i]
        # the top eigenvalues (~n) are well separated: after one degree-10 sweep the leading
        # Ritz pairs are converged to a small residual relative to ||A||
        assert np.linalg.norm(r) <= 1e-6 * abs(thh[0])
        # Rayleigh quotient consistency (exact in any basis)
        assert abs(Vh[:, i] @ (Ah @ Vh[:, i]) - thh[i]) <= 1e-11 * abs(thh[0])
