"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

* config 2 (n = 4096): the first iterations of the trajectory against the oracle, element-wise
  on X_k (via factors) and the objective.
* config 3 (n = 16384, the bench workload and method options, pfinputs.BENCH_METHOD): an
  independent 12-iteration trajectory (a warm-started Lanczos refresh at k = 10) -- each side runs
  its own Lanczos interval, filter, orthonormalisation, Rayleigh-Ritz, P_+ and DRS update -- on
  X_k, <C, W> and ||Z+ - Z||, plus sampled entries of the final Z+ computed one by one.
* config 4 (n = 32768, p = 128, d = 10): an independent 4-iteration trajectory on X_k and the
  PFPG objective (the int8-digit products run past the exact-int32 fold bound, K = 32768).
* config 5 (n = 65536, p = 512, fp32 / TF32): iterations k = 0..2 (d = 4, two perturbations)
  against the oracle computing in fp64 on the same fp32 iterates, at the TF32 bar 1e-4.
Both dtypes of configs 3 and 4 run the bench's launch configuration (CUDA graphs) against one
oracle run per config (module-scoped fixtures; the oracle takes ~5 s / ~20 s per iteration).
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


def _compare(ref, got, tol, aux_tol=None, aux_key=None):
    for r, g in zip(ref, got):
        assert _err(g, r) <= tol, (r["k"], _err(g, r))
        if "objective" in r:
            assert abs(g["objective"] - r["objective"]) <= tol * abs(r["objective"]), r["k"]
        if aux_key:
            assert abs(g["aux"] - r[aux_key]) <= aux_tol * abs(r[aux_key]), (r["k"], g["aux"], r[aux_key])


@pytest.fixture(scope="module")
def cfg3_ref():
    from pfinputs import bench_config
    cfg = bench_config(3)
    prob = pfam_problem(cfg)
    out = O.run(reduced(cfg, rr_ns=False), iters=12, problem=prob)   # the oracle diagonalises H
    return cfg, prob, out["records"], out["final_A"]


def _compare_qf(ref, got, tol, aux_tol):
    """X_k from the matrix-form records (Q F, Q) vs the oracle's eigen-factors."""
    for r, g in zip(ref, got):
        one = np.ones(g["Q"].shape[1])
        den = O.lowrank_fro(r["V"], r["f"])
        err = O.lowrank_rect_diff_fro(r["V"] * r["f"], np.ones(r["f"].size), r["V"],
                                      g["QF"], one, g["Q"])
        assert err <= tol * den, (r["k"], err / den)
        assert abs(g["objective"] - r["objective"]) <= tol * abs(r["objective"]), r["k"]
        assert abs(g["aux"] - r["residual"]) <= aux_tol * abs(r["residual"]), r["k"]


@pytest.mark.parametrize("dtype", ["f64i8", "f64"])   # f64i8 + graphs: the bench's path
def test_config3_fullsize_trajectory(cfg3_ref, dtype):
    from paper_1904_10585_b200 import run
    cfg, prob, ref, Zref = cfg3_ref
    out = run(reduced(cfg, dtype=dtype), iters=12, problem=prob, graphs=True)
    _compare_qf(ref, out["records"], 1e-10, 1e-9)
    solver = out["solver"]
    assert solver.z_upper == (dtype == "f64i8")   # the bench's storage (pf_set_z_upper)
    rng = np.random.default_rng(7)
    idx = rng.integers(0, cfg.n, size=(4000, 2))
    zs = solver.iterate_entries(idx[:, 0], idx[:, 1]).cpu().numpy()
    np.testing.assert_allclose(zs, Zref[idx[:, 0], idx[:, 1]], rtol=0,
                               atol=1e-10 * np.abs(Zref).max())


@pytest.fixture(scope="module")
def cfg4_ref():
    from pfinputs import pfpg_problem
    cfg = reduced(CONFIGS[4])
    prob = pfpg_problem(cfg)
    return cfg, prob, O.run(cfg, iters=4, problem=prob)["records"]


@pytest.mark.parametrize("dtype", ["f64i8", "f64"])
def test_config4_fullsize_trajectory(cfg4_ref, dtype):
    from paper_1904_10585_b200 import run
    cfg, prob, ref = cfg4_ref
    got = run(reduced(cfg, dtype=dtype), iters=4, problem=prob, graphs=True)["records"]
    _compare(ref, got, 1e-10, 1e-10, "fit")


def test_config5_fullsize_k0_to_2():
    """n = 65536, p = 512, d = 4: k = 0 (4 warm-up sweeps), 1, 2 after two perturbations of the
    fp32 iterate (the GPU draws E_k with pf_perturb_hash, the oracle with pfinputs' host copy of
    the same counter-based generator); the oracle computes in fp64 on the fp32 iterates."""
    from paper_1904_10585_b200 import run
    from pfinputs import cfg5_problem
    cfg = reduced(CONFIGS[5], d=4, iters=3)
    A0 = cfg5_problem(cfg)
    got = run(cfg, problem={"A0": A0})["records"]
    torch.cuda.empty_cache()
    ref = O.run(cfg, problem={"A0": A0})["records"]
    for r, g in zip(ref, got):
        assert g["rank"] == r["rank"], r["k"]
        assert _err(g, r) <= 1e-4, (r["k"], _err(g, r))
