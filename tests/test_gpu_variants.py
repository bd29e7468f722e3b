"""Driver variants of the method on the CUDA path vs the oracle:
q applications of the polynomial per filter, the degree schedule of thm:conv1
 and the top-r interval."""
import numpy as np
import pytest
import torch

import oracle as O
from pfinputs import CONFIGS, reduced

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a B200")]


def _traj(cfg, tol):
    from paper_1904_10585_b200 import run
    ref = O.run(cfg)["records"]
    got = run(cfg)["records"]
    for r, g in zip(ref, got):
        assert g["rank"] == r["rank"]
        den = O.lowrank_fro(r["V"], r["f"])
        assert O.lowrank_diff_fro(g["V"], g["f"], r["V"], r["f"]) <= tol * den, r["k"]
        if "objective" in r:
            assert g["objective"] == pytest.approx(r["objective"], rel=tol)


@pytest.mark.parametrize("cfg,tol", [
    (reduced(CONFIGS[1], iters=6, q=2), 1e-10),
    (reduced(CONFIGS[3], n=900, iters=6, edge_prob=82 / 900, q=2), 1e-10),
    (reduced(CONFIGS[5], n=1536, p=64, nbig=24, nrefl=16, iters=3, q=2), 1e-4),
], ids=["cfg1_q2", "cfg3_q2", "cfg5_tf32_q2"])
def test_q_repeats(cfg, tol):
    _traj(cfg, tol)


@pytest.mark.parametrize("cfg,tol", [
    (reduced(CONFIGS[3], n=900, iters=8, d=2, deg_c=3.0, edge_prob=82 / 900), 1e-10),
    (reduced(CONFIGS[2], n=800, iters=8, d=3, deg_c=2.5), 1e-10),
], ids=["cfg3_sched", "cfg2_sched"])
def test_degree_schedule(cfg, tol):
    _traj(cfg, tol)


def test_interval_top_r_matches_oracle():
    from paper_1904_10585_b200 import Context
    n, p = 700, 32
    rng = np.random.default_rng(3)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.concatenate([np.linspace(5, 1, 20), rng.uniform(-2, 0.5, n - 20)])
    A = (q * lam) @ q.T
    A = 0.5 * (A + A.T)
    ctx = Context(n, p, 4)
    dA = torch.as_tensor(A).cuda()
    U = torch.as_tensor(O.orth(rng.standard_normal((n, p)))).cuda()
    V = torch.empty_like(U)
    th = torch.empty(p, dtype=torch.float64, device="cuda")
    lohi = torch.tensor([-2.5, 6.0], dtype=torch.float64, device="cuda")
    iv = torch.zeros(2, dtype=torch.float64, device="cuda")
    ctx.interval_top_r(lohi, 10, 0.1, iv)       # before any RR: b = eta a
    np.testing.assert_allclose(iv.cpu().numpy(), O.interval_psd(-2.5, 0.1), rtol=0, atol=0)
    ctx.rayleigh_ritz(dA, U, V, th)
    ctx.interval_top_r(lohi, 10, 0.1, iv)
    theta = th.cpu().numpy()
    np.testing.assert_allclose(iv.cpu().numpy(), O.interval_top_r(-2.5, theta[9], 0.1),
                               rtol=1e-15, atol=1e-15)


@pytest.mark.parametrize("q", [1, 2])
def test_relative_gap_and_eta_diagnostics_match_oracle(q):
    """pf_diagnostics' relative gap (NEXT-2, eqn:relative-gap) and eta_k estimate (eqn:etak,
    reading R28) from the device Ritz values and the damped interval equal the oracle's on every
    iteration of a sweep (q = 2: the polynomial applied twice per filter)."""
    from paper_1904_10585_b200 import Solver
    import oracle as O
    cfg = reduced(CONFIGS[1], iters=6, q=q)
    ref = O.run(cfg)["records"]
    s = Solver(cfg)
    from pfinputs import cfg1_noise
    from paper_1904_10585_b200.solver import _dev
    for k in range(cfg.iters):
        s.step()
        dg = s.ctx.diagnostics()
        g = dg["relative_gap"]
        # q = 2: the gap is set by a guard Ritz value just beyond the interval edge, fixed only
        # to ~1e-6 by the (twice damped) unconverged direction -- looser bar
        rel = 1e-9 if q == 1 else 1e-5
        assert g == pytest.approx(ref[k]["gap"], rel=rel), (k, g, ref[k]["gap"])
        assert np.isnan(ref[k]["eta"]) == np.isnan(dg["eta"])
        if not np.isnan(ref[k]["eta"]):
            assert dg["eta"] == pytest.approx(ref[k]["eta"], rel=100 * rel, abs=1e-300), k
            assert 0.0 <= dg["eta"] < 1.0
            # the device value is the bound of its own gap: (1 / T_d(1 + G))^q
            assert dg["eta"] == pytest.approx((1.0 / O.cheb_T(cfg.d, 1.0 + g)) ** q, rel=1e-12)
        if k + 1 < cfg.iters:
            s.perturb(_dev(cfg1_noise(cfg, k)))


@pytest.mark.parametrize("cfg,tol", [
    (reduced(CONFIGS[1], iters=12, lanczos_every=3, lanczos_warm=8), 1e-10),
    (reduced(CONFIGS[3], n=900, iters=12, edge_prob=82 / 900, lanczos_every=3, lanczos_warm=8),
     1e-10),
    (reduced(CONFIGS[3], n=1100, iters=12, edge_prob=0.07, lanczos_every=3, lanczos_warm=8,
             dtype="f64i8"), 1e-10),
], ids=["cfg1_warm", "cfg3_warm", "cfg3_i8_warm"])
def test_lanczos_warm_start_trajectory(cfg, tol):
    """NEXT-2 lambda_min tracking (reading R29): refreshes after the first restart a short
    Lanczos from the previous bottom Ritz vector (pf_lanczos with v0 = NULL) on both sides."""
    _traj(cfg, tol)


def test_schedule_degree_matches_oracle_and_rejects_bad_arguments():
    """pf_schedule_degree (thm:conv1 schedule in the library) against the oracle's own
    degree_schedule for a range of k, and its synchronous argument errors."""
    from paper_1904_10585_b200._lib import Context, PFError
    c = Context(256, 16, 3)
    for cc in (0.0, 1.5, 3.0):
        for k in (0, 1, 5, 40, 1000, 10**6):
            assert c.schedule_degree(cc, k) == O.degree_schedule(3, cc, k), (cc, k)
    with pytest.raises(PFError, match="PF_ERR_ARG"):
        c.schedule_degree(-1.0, 3)
    with pytest.raises(PFError, match="PF_ERR_ARG"):
        c.schedule_degree(30.0, 10**9)          # d_k > 64
