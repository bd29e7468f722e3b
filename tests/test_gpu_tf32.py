"""fp32-storage / TF32 tensor-core path (config 5, BASELINE configs[4]) vs the CPU oracle,
through the C ABI.

The oracle runs in fp64 on the same fp32-rounded iterate.  Tolerance (BASELINE.json
north_star): relative Frobenius <= 1e-4 per iteration on X_k = V diag(f) V^T for TF32/fp32
configurations.  Unit kernels are held to bounds derived from fp32 storage (u32 = 2^-24).
"""
import numpy as np
import pytest
import torch

import oracle as O
from pfinputs import (CONFIGS, reduced, cfg5_problem, cfg5_noise_rows, cfg5_spectrum,
                      cfg5_reflectors, cfg5_basis_columns)

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a B200")]

TOL_X = 1e-4


def _ctx(n, p, d=8):
    from paper_1904_10585_b200 import Context, PF_TF32
    return Context(n, p, d, dtype=PF_TF32)


def _f32(x):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float32).cuda()


def _f32_pitched(A):
    """Row-major fp32 matrix with a 16-byte row pitch (TMA), e.g. for ragged n."""
    n, m = A.shape
    buf = torch.zeros((n, (m + 3) // 4 * 4), dtype=torch.float32, device="cuda")
    buf[:, :m] = torch.from_numpy(np.ascontiguousarray(A))
    return buf[:, :m]


def _sym32(n, seed, spec):
    rng = np.random.default_rng(seed)
    q, r = np.linalg.qr(rng.standard_normal((n, n)))
    q = q * np.sign(np.diag(r))
    A = (q * np.asarray(spec, float)) @ q.T
    A = (0.5 * (A + A.T)).astype(np.float32)
    A = np.triu(A) + np.triu(A, 1).T
    return A


# ------------------------------------------------------------------ workload generator
def test_perturb_hash_matches_host_generator():
    """pf_perturb_hash implements pfinputs.hash_gauss: identical fp32 noise (up to rare
    last-ulp libm differences in log/cos before the fp32 rounding)."""
    cfg = reduced(CONFIGS[5], n=777, p=64)
    A = np.zeros((777, 780), dtype=np.float32)
    dA = _f32(A)
    ctx = _ctx(777, 64)
    ctx.perturb_hash(dA[:, :777], cfg.seed, 5, cfg.noise)
    got = dA.cpu().numpy()[:, :777]
    ref = cfg5_noise_rows(cfg, 5, 0, 777)
    diff = got != ref
    assert diff.mean() < 1e-4, diff.sum()
    np.testing.assert_allclose(got, ref, rtol=2 ** -22, atol=0)
    assert (got == got.T).all()
    # additive on a non-zero iterate, every entry updated exactly once (both triangles of the
    # symmetric tile-pair kernel), fp32 add rounded to nearest
    A1 = np.random.default_rng(1).standard_normal((777, 780)).astype(np.float32)
    dA1 = _f32(A1)
    ctx.perturb_hash(dA1[:, :777], cfg.seed, 5, cfg.noise)
    want = (A1[:, :777] + ref).astype(np.float32)
    assert (dA1.cpu().numpy()[:, :777] != want).mean() < 1e-4


# ------------------------------------------------------------------ orthonormalisation
@pytest.mark.parametrize("p", [64, 128, 256, 512])
def test_orth32(p):
    n = 1500 if p < 512 else 2100
    rng = np.random.default_rng(p)
    Y = rng.standard_normal((n, p)) * np.logspace(0, 3, p)[None, :]
    Y32 = Y.astype(np.float32)
    ctx = _ctx(n, p)
    U = _f32(Y32.T)                       # p-major
    ctx.orth(U)
    Q = U.cpu().numpy().T.astype(np.float64)
    assert np.linalg.norm(Q.T @ Q - np.eye(p)) < 1e-5 * np.sqrt(p)
    # same span as the fp64 Householder Q of the fp32 block (fp32 storage: ~u32 * kappa)
    assert np.max(O.sin_theta(O.orth(Y32.astype(np.float64)), Q)) < 1e-4


# ------------------------------------------------------------------ filter + RR units
@pytest.mark.parametrize("p,n", [(64, 1000), (128, 1333), (256, 1800), (512, 2600)])
def test_filter_span_vs_oracle(p, n):
    """One pf_filter call (degree 8, soft interval) against the oracle's filter_update on the
    same fp32 A: the spans agree to the fp32-storage level (well-separated wanted space)."""
    k = p // 2
    rng = np.random.default_rng(n)
    spec = np.concatenate([rng.uniform(5, 50, k), rng.uniform(-1, 1, n - k)])
    A = _sym32(n, n, spec)
    U0 = O.orth(rng.standard_normal((n, p)))
    a, b = O.interval_soft(3.0, 0.1)
    ref = O.filter_update(A.astype(np.float64), U0, a, b, 8, 1, [3, 5, 7])
    ctx = _ctx(n, p, 8)
    dA = _f32_pitched(A)
    U = _f32(U0.T)
    iv = torch.tensor([a, b], dtype=torch.float64, device="cuda")
    # the re-base schedule needs a spread estimate (reading R7): Lanczos first, as the solver does
    lohi = torch.zeros(2, dtype=torch.float64, device="cuda")
    ctx.lanczos(dA, torch.as_tensor(rng.standard_normal(n)).cuda(), 20, lohi)
    assert 45.0 < lohi[1].item() < 60.0     # theta_max + |r| around the top eigenvalue (<= 50)
    ctx.filter(dA, U, iv, 1, 1e3)
    assert ctx.status()["rebases"] == 3
    Q = U.cpu().numpy().T.astype(np.float64)
    assert np.linalg.norm(Q.T @ Q - np.eye(p)) < 1e-5 * np.sqrt(p)
    # Only the wanted k directions (|lambda| >= 5, amplified by >= T_8(5/2.7) over the bulk) are
    # determined by the filter; the other p - k columns are arbitrary mixtures of bulk
    # eigenvectors, so spans are compared on the wanted space: both sides must contain it to
    # the same accuracy.
    ev, evec = np.linalg.eigh(A.astype(np.float64))
    want = evec[:, np.argsort(-np.abs(ev))[:k]]
    s_ref = np.max(O.sin_theta(ref, want))
    s_gpu = np.max(O.sin_theta(Q, want))
    assert s_gpu < max(2e-5, 10 * s_ref), (s_gpu, s_ref)


@pytest.mark.parametrize("p,n", [(64, 900), (512, 2100)])
def test_rayleigh_ritz32(p, n):
    rng = np.random.default_rng(7 * p)
    A = _sym32(n, p, rng.standard_normal(n) * 3)
    Q0 = O.orth(rng.standard_normal((n, p))).astype(np.float32)
    ctx = _ctx(n, p)
    dA, U = _f32(A), _f32(Q0.T)
    V = torch.empty((p, n), dtype=torch.float32, device="cuda")
    th = torch.empty(p, dtype=torch.float64, device="cuda")
    ctx.rayleigh_ritz(dA, U, V, th)
    theta_ref, V_ref = O.rayleigh_ritz(A.astype(np.float64), Q0.astype(np.float64))
    theta = th.cpu().numpy()
    nrm = np.abs(theta_ref).max()
    assert np.all(np.diff(theta) <= 0)
    np.testing.assert_allclose(theta, theta_ref, atol=1e-5 * nrm)
    Vg = V.cpu().numpy().T.astype(np.float64)
    assert np.linalg.norm(Vg.T @ Vg - np.eye(p)) < 1e-4
    # basis-invariant: V diag(theta) V^T against the oracle's
    den = O.lowrank_fro(V_ref, theta_ref)
    assert O.lowrank_diff_fro(Vg, theta, V_ref, theta_ref) / den < 1e-5


# ------------------------------------------------------------------ trajectories
def _trajectory(cfg):
    from paper_1904_10585_b200 import run
    ref = O.run(cfg)["records"]
    got = run(cfg)["records"]
    errs = []
    for r, g in zip(ref, got):
        assert g["rank"] == r["rank"]
        den = O.lowrank_fro(r["V"], r["f"])
        errs.append(O.lowrank_diff_fro(g["V"], g["f"], r["V"], r["f"]) / den)
    return errs


def test_config5_reduced_trajectory():
    """Config 5 recipe at n = 1536 (p = 64, d = 8, 24 large eigenvalues), 5 iterations with the
    device-generated noise: X_k within 1e-4 of the oracle every iteration."""
    cfg = reduced(CONFIGS[5], n=1536, p=64, nbig=24, nrefl=16, iters=5)
    errs = _trajectory(cfg)
    assert max(errs) < TOL_X, errs


@pytest.mark.parametrize("d", [4, 16])
def test_config5_degrees(d):
    """The other degrees of config 5 (d in {4, 8, 16}) at reduced size, p = 128."""
    cfg = reduced(CONFIGS[5], n=2048, p=128, d=d, nbig=48, nrefl=16, iters=3)
    errs = _trajectory(cfg)
    assert max(errs) < TOL_X, errs


def test_config5_p512_trajectory():
    """p = 512 (config 5's block width) at n = 4096, 2 iterations: exercises the 512-wide
    tcgen05 tiles, the 512 x 512 Cholesky and the cooperative Jacobi."""
    cfg = reduced(CONFIGS[5], n=4096, p=512, nbig=200, nrefl=32, iters=2)
    errs = _trajectory(cfg)
    assert max(errs) < TOL_X, errs


@pytest.mark.slow
def test_config5_full_size_k0_closed_form():
    """Full config 5 (n = 65536, p = 512, d = 8) at k = 0 against the closed form the oracle
    is pinned to (tests/test_oracle_pins.py::test_config5_k0_closed_form): A_0 = Q Lambda Q^T
    with Q, Lambda from the generator, so the exact soft threshold is
    Q[:, big] diag(sign(l)(|l| - 3)) Q[:, big]^T.  Also the 256 Ritz values above the threshold
    against the known eigenvalues."""
    from paper_1904_10585_b200 import Solver
    cfg = reduced(CONFIGS[5], iters=1)
    s = Solver(cfg)
    s.step()
    torch.cuda.synchronize()
    f = s.f.cpu().numpy()
    keep = f != 0
    V = s.ritz_factors()[:, keep]
    lam = cfg5_spectrum(cfg)
    Vh, T = cfg5_reflectors(cfg)
    big = np.where(np.abs(lam) > cfg.theta)[0]
    fex = np.sign(lam[big]) * (np.abs(lam[big]) - cfg.theta)
    assert keep.sum() == len(big) == 256
    np.testing.assert_allclose(np.sort(f[keep]), np.sort(fex), rtol=0, atol=1e-4 * fex.max())
    Qb = cfg5_basis_columns(Vh, T, big)
    err = O.lowrank_diff_fro(V, f[keep], Qb, fex) / O.lowrank_fro(Qb, fex)
    assert err < TOL_X, err
