"""Lanczos on one GPU in fp64 reads only the upper triangle of A (`lz_symv_tiles_kernel` +
`lz_symv_reduce_kernel`): the extremes agree with the oracle (paper's `eigs`
reading R5) at the fp64 bar and with the full-matrix GEMV (`PF_LZ_SYM=0`) to rounding, on sizes
with ragged 64-tiles (odd n inside an even pitch), a single tile, and a run that breaks down."""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a B200")]


def _sym(n, seed):
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.concatenate([[-7.0], np.linspace(-3, 2, n - 2), [4.0]])
    A = (q * lam) @ q.T
    return 0.5 * (A + A.T)


def _pitched(A):
    n = A.shape[1]
    buf = torch.full((A.shape[0], (n + 1) // 2 * 2), float("nan"), dtype=torch.float64,
                     device="cuda")                    # NaN padding: must never be multiplied
    buf[:, :n].copy_(torch.from_numpy(A))
    return buf[:, :n]


def _run(A, v0, m, monkeypatch=None, sym=True):
    from paper_1904_10585_b200 import Context
    if monkeypatch is not None:
        monkeypatch.setenv("PF_LZ_SYM", "1" if sym else "0")
    n = A.shape[0]
    ctx = Context(n, 16, 4)
    lohi = torch.zeros(2, dtype=torch.float64, device="cuda")
    ctx.lanczos(_pitched(A), torch.from_numpy(v0).cuda(), m, lohi)
    return lohi.cpu().numpy()


@pytest.mark.parametrize("n", [64, 333, 700, 1333, 4099])
def test_upper_triangle_gemv_matches_oracle_and_full(n, monkeypatch):
    A = _sym(n, n)
    v0 = np.random.default_rng(1).standard_normal(n)
    lo_ref, hi_ref = O.lanczos_extremes(A, v0, 20)
    lo, hi = _run(A, v0, 20, monkeypatch, sym=True)
    lo_f, hi_f = _run(A, v0, 20, monkeypatch, sym=False)
    assert lo == pytest.approx(lo_ref, rel=1e-10) and hi == pytest.approx(hi_ref, rel=1e-10)
    assert lo == pytest.approx(lo_f, rel=1e-12) and hi == pytest.approx(hi_f, rel=1e-12)


def test_upper_triangle_ignores_lower(monkeypatch):
    """Only the 64 x 64 tiles on and above the diagonal are read: garbage in the tiles below
    does not change the result."""
    n = 700
    A = _sym(n, 5)
    v0 = np.random.default_rng(2).standard_normal(n)
    ref = _run(A, v0, 20, monkeypatch, sym=True)
    B = A.copy()
    r, c = np.indices((n, n))
    B[(r // 64) > (c // 64)] = 1e300
    got = _run(B, v0, 20, monkeypatch, sym=True)
    assert np.array_equal(ref, got)


def test_breakdown_on_symmetric_path(monkeypatch):
    A = np.diag(np.arange(1.0, 17.0))
    lo, hi = _run(A, np.ones(16), 20, monkeypatch, sym=True)
    lo_ref, hi_ref = O.lanczos_extremes(A, np.ones(16), 20)
    assert lo == pytest.approx(lo_ref, abs=1e-10) and hi == pytest.approx(hi_ref, abs=1e-10)
