"""Seeded input generators (pfinputs): determinism and the structure BASELINE.json states."""
import numpy as np

from pfinputs import (CONFIGS, reduced, initial_block, cfg1_problem, pfpg_problem, pfam_problem,
                      sym_bernoulli_bitmask, unpack_bitmask)


def test_bitmask_roundtrip_symmetric():
    rng = np.random.default_rng(0)
    for n in (1, 31, 32, 33, 100):
        bits = sym_bernoulli_bitmask(n, 0.3, np.random.default_rng([1, n]), diagonal=True)
        m = unpack_bitmask(bits, n)
        assert m.shape == (n, n) and (m == m.T).all()
        assert bits.shape == (n, (n + 31) // 32) and bits.dtype == np.uint32
        # padding bits beyond column n are zero
        if n % 32:
            assert (bits[:, -1] >> (n % 32) == 0).all()
    bits = sym_bernoulli_bitmask(200, 0.2, np.random.default_rng(3), diagonal=False)
    assert not unpack_bitmask(bits, 200).diagonal().any()


def test_determinism_and_structure():
    cfg = reduced(CONFIGS[2], n=300)
    a, b = pfpg_problem(cfg), pfpg_problem(cfg)
    assert (a["omega_bits"] == b["omega_bits"]).all() and (a["W"] == b["W"]).all()
    assert a["mu"] == b["mu"] and a["mu"] > 0
    dens = unpack_bitmask(a["omega_bits"], 300).mean()
    assert 0.07 < dens < 0.13
    cfg3 = reduced(CONFIGS[3], n=400, edge_prob=0.05)
    g = pfam_problem(cfg3)
    adj = unpack_bitmask(g["adj_bits"], 400)
    np.testing.assert_array_equal(adj.sum(1), g["deg"])
    assert (initial_block(cfg) == initial_block(cfg)).all()


def test_config1_spectrum():
    A = cfg1_problem(CONFIGS[1])
    lam = np.linalg.eigvalsh(A)
    assert (lam > 0).sum() == 8
    assert lam.max() <= 10 + 1e-10 and lam.min() >= -1 - 1e-10
    assert np.allclose(A, A.T)


def test_config5_generator():
    """Config 5 (BASELINE configs[4]): Q = product of Householder reflectors (compact WY equals
    the explicit product), A_0 = Q diag(lambda) Q^T stored exactly symmetric in fp32 with the
    spectrum lambda (up to the fp32 rounding), semicircle bulk in [-1, 1]."""
    from pfinputs import cfg5_problem, cfg5_spectrum, cfg5_reflectors, cfg5_basis_columns
    cfg = reduced(CONFIGS[5], n=200, nbig=10, nrefl=7)
    V, T = cfg5_reflectors(cfg)
    Q = np.eye(200)
    for j in range(7):
        Q = Q @ (np.eye(200) - 2.0 * np.outer(V[:, j], V[:, j]))
    np.testing.assert_allclose(np.eye(200) - V @ T @ V.T, Q, atol=1e-13)
    np.testing.assert_allclose(cfg5_basis_columns(V, T, np.array([0, 5, 199])), Q[:, [0, 5, 199]],
                               atol=1e-13)
    lam = cfg5_spectrum(cfg)
    assert ((lam >= 5) & (lam <= 50)).sum() == 10 and (np.abs(lam) <= 1).sum() == 190
    A = cfg5_problem(cfg, chunk=48)
    assert A.dtype == np.float32 and (A == A.T).all()
    ev = np.linalg.eigvalsh(A.astype(np.float64))
    # fp32 rounding perturbs each entry by <= 2^-24 |a_ij|: Weyl bound via the Frobenius norm
    bound = 2.0 ** -24 * np.linalg.norm(A.astype(np.float64))
    assert np.abs(np.sort(ev) - np.sort(lam)).max() <= bound
    assert (cfg5_problem(cfg) == A).all()


def test_config5_noise_hash():
    """E_k: symmetric, deterministic, depends on (seed, k) only, law noise * (G + G^T)/2."""
    from pfinputs import cfg5_noise_rows, hash_gauss
    cfg = reduced(CONFIGS[5], n=700)
    E = cfg5_noise_rows(cfg, 3, 0, 700)
    assert E.dtype == np.float32 and (E == E.T).all()
    np.testing.assert_array_equal(cfg5_noise_rows(cfg, 3, 100, 200), E[100:200])
    assert not (cfg5_noise_rows(cfg, 4, 0, 700) == E).all()
    off = E[np.triu_indices(700, 1)] / cfg.noise
    assert abs(off.std() - 2 ** -0.5) < 0.01 and abs(off.mean()) < 0.01
    assert abs(np.diag(E).std() / cfg.noise - 1.0) < 0.1
    g = hash_gauss(0, 0, np.arange(200000), np.arange(200000) + 1)
    # standard normal moments
    assert abs(g.mean()) < 0.01 and abs(g.var() - 1) < 0.01 and abs((g ** 4).mean() - 3) < 0.06
