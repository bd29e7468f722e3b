"""Degenerate-interval semantics (reading R23): when the PSD interval collapses
(a = lambda_min estimate >= 0: the iterate is already PSD) pf_filter skips the filter, returns
orth(U) and raises PF_FLAG_DEGENERATE_INT -- on both storage paths -- and the GPU trajectory
matches the oracle, which skips the filter on the same iterations."""
import numpy as np
import pytest
import torch

import oracle as O
from pfinputs import CONFIGS, reduced

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a B200")]


def _psd(n, seed=11, lo=1.0, hi=10.0):
    rs = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rs.standard_normal((n, n)))
    A = (q * rs.uniform(lo, hi, n)) @ q.T
    return 0.5 * (A + A.T)


@pytest.mark.parametrize("dtype", ["f64", "tf32"])
def test_psd_iterate_skips_filter(dtype):
    from paper_1904_10585_b200 import run
    n, p = 512, (32 if dtype == "f64" else 64)
    if dtype == "f64":
        cfg = reduced(CONFIGS[1], n=n, p=p, iters=3, noise=0.0)
        A = _psd(n)
        tol = 1e-10
    else:
        cfg = reduced(CONFIGS[5], n=n, p=p, iters=3, noise=0.0, mode="sweep_psd", nbig=8,
                      nrefl=4)
        A = _psd(n).astype(np.float32)
        tol = 1e-4
    ref = O.run(cfg, problem={"A0": A})["records"]
    out = run(cfg, problem={"A0": A})
    assert "DEGENERATE_INTERVAL" in out["status"]["names"]
    for x, y in zip(ref, out["records"]):
        assert x["degenerate"]
        den = O.lowrank_fro(x["V"], x["f"])
        assert O.lowrank_diff_fro(x["V"], x["f"], y["V"], y["f"]) <= tol * den


def test_mixed_trajectory_recovers_after_degenerate_step():
    """Noise pushes a PSD start (lambda_min ~ 0.05) indefinite after a few steps: the first
    iterations skip the filter, later ones filter again; GPU and oracle agree throughout."""
    from paper_1904_10585_b200 import run
    n, p = 384, 16
    cfg = reduced(CONFIGS[1], n=n, p=p, iters=6, noise=0.05, lanczos_every=1)
    A = _psd(n, seed=5, lo=0.02, hi=4.0)
    ref = O.run(cfg, problem={"A0": A})["records"]
    flags = [r["degenerate"] for r in ref]
    assert flags[0] and not flags[-1], flags
    out = run(cfg, problem={"A0": A})
    for x, y in zip(ref, out["records"]):
        den = O.lowrank_fro(x["V"], x["f"])
        assert O.lowrank_diff_fro(x["V"], x["f"], y["V"], y["f"]) <= 1e-10 * den
