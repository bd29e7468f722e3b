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
