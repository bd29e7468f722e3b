"""PF_FP64_I8: the fp64 filter GEMM formed from exact int8 tensor-core products of 7-bit digit
slices (pf_gemm_i8.cu, DESIGN.md §4 K1-i8).

  * integer operands with few digits: every product is exact on both sides -> bit-equal to numpy;
  * random fp64 operands with wide per-row / per-column scales, ragged n, zero rows / columns:
    within the splitting bound K 2^(E_i + F_c) (S + 2) 2^-7S of the exact product;
  * trajectories of configs 1-3 (reduced) and NCE against the oracle at the fp64 bar (1e-10),
    and bit-identical CUDA-graph replay."""
import numpy as np
import pytest
import torch

import oracle as O
from pfinputs import CONFIGS, NEXT_CONFIGS, reduced

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a B200")]


def _ctx(n, p, slices=7):
    from paper_1904_10585_b200._lib import Context, PF_FP64_I8
    c = Context(n, p, 4, dtype=PF_FP64_I8)
    c.set_i8_slices(slices)
    return c


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _pitched(A):
    n = A.shape[1]
    buf = torch.zeros((A.shape[0], (n + 1) // 2 * 2), dtype=torch.float64, device="cuda")
    buf[:, :n].copy_(torch.from_numpy(A))
    return buf[:, :n]


@pytest.mark.parametrize("n,p", [(64, 16), (1000, 32), (1333, 64), (700, 128), (16384, 64)])
def test_integer_operands_exact(n, p):
    """|a|, |y| < 2^k with few digits: the digit expansion is exact and so is every level sum."""
    rs = np.random.default_rng(n + p)
    A = rs.integers(-100, 101, (n, n)).astype(np.float64)
    A[3] = 0.0                                        # zero row (scale exponent 0)
    Y = rs.integers(-50, 51, (n, p)).astype(np.float64)
    Y[:, 1] = 0.0                                     # zero column
    ref = A @ Y                                       # exact (integers < 2^53)
    c = _ctx(n, p)
    out = torch.empty((n, p), dtype=torch.float64, device="cuda")
    c.matmul(_pitched(A), _dev(Y), out)
    assert np.array_equal(out.cpu().numpy(), ref)


@pytest.mark.parametrize("pair", ["0", "1"])
@pytest.mark.parametrize("n,p", [(64, 64), (129, 64), (1333, 64), (2049, 128), (4160, 64)])
def test_pair_and_single_cta_kernels_exact(monkeypatch, n, p, pair):
    """K1-i8p (CTA pairs, cta_group::2, the default at S = 7, p % 64 == 0) and the one-CTA
    K1-i8 (PF_I8PAIR=0) on integer operands: bit-equal to numpy.  Odd tile counts (n = 64, 1333,
    4160: a pair whose second tile lies past n, zero-filled by TMA), two column groups (p = 128)
    and stream-K splits across pair items."""
    monkeypatch.setenv("PF_I8PAIR", pair)
    rs = np.random.default_rng(3 * n + p)
    A = rs.integers(-127, 128, (n, n)).astype(np.float64)
    Y = rs.integers(-90, 91, (n, p)).astype(np.float64)
    Y[:, -1] = 0.0
    ref = A @ Y
    c = _ctx(n, p)
    out = torch.empty((n, p), dtype=torch.float64, device="cuda")
    c.matmul(_pitched(A), _dev(Y), out)
    assert np.array_equal(out.cpu().numpy(), ref)


@pytest.mark.parametrize("n,p", [(1333, 64), (6000, 128)])
def test_pair_kernel_matches_single_cta_kernel(monkeypatch, n, p):
    """Gaussian operands: the two kernels form the same exact level sums; only the stream-K
    split points (fp64 partial sums) differ, so they agree to the fp64 rounding of the sum."""
    rs = np.random.default_rng(n + 5)
    A = rs.standard_normal((n, n))
    A = A + A.T
    Y = rs.standard_normal((n, p))
    outs = []
    for pair in ("1", "0"):
        monkeypatch.setenv("PF_I8PAIR", pair)
        c = _ctx(n, p)
        out = torch.empty((n, p), dtype=torch.float64, device="cuda")
        c.matmul(_pitched(A), _dev(Y), out)
        outs.append(out.cpu().numpy())
    scale = np.abs(A).max() * np.abs(Y).max() * n
    assert np.abs(outs[0] - outs[1]).max() <= 2.0 ** -50 * scale
    assert np.abs(outs[0] - A @ Y).max() <= 2.0 ** -47 * scale


@pytest.mark.parametrize("slices", [6, 7])
@pytest.mark.parametrize("n,p", [(1000, 32), (1333, 64), (2049, 128), (300, 16)])
def test_random_operands_within_split_bound(n, p, slices):
    rs = np.random.default_rng(7 * n + p)
    A = rs.standard_normal((n, n)) * np.exp2(rs.integers(-30, 30, n))[:, None]
    A[:, rs.integers(0, n, 5)] *= 1e6                 # a few large columns (row scales move)
    Y = rs.standard_normal((n, p)) * np.exp2(rs.integers(-20, 20, p))[None, :]
    Y[rs.integers(0, n, 3)] *= 1e-9
    c = _ctx(n, p, slices)
    out = torch.empty((n, p), dtype=torch.float64, device="cuda")
    c.matmul(_pitched(A), _dev(Y), out)
    got = out.cpu().numpy()
    ref = A @ Y
    _, ea = np.frexp(np.abs(A).max(axis=1))
    _, ey = np.frexp(np.abs(Y).max(axis=0))
    bound = n * np.exp2(ea[:, None] + ey[None, :]) * (slices + 2) * 2.0 ** (-7 * slices)
    bound += 4 * n * np.finfo(float).eps * (np.abs(A) @ np.abs(Y))   # numpy's own rounding
    err = np.abs(got - ref)
    assert (err <= bound).all(), float((err / bound).max())


@pytest.mark.parametrize("n,p", [(1333, 64), (4096, 32)])
def test_gaussian_operands_fp64_grade(n, p):
    """Operands without wide in-row dynamic range (the iterates of configs 1-4): the S = 7 product
    is as accurate as the fp64 DMMA GEMM's (same context, pf_set_i8_slices(0))."""
    rs = np.random.default_rng(n)
    A = rs.standard_normal((n, n))
    A = A + A.T
    Y = rs.standard_normal((n, p))
    ref = A @ Y
    c = _ctx(n, p)
    out = torch.empty((n, p), dtype=torch.float64, device="cuda")
    c.matmul(_pitched(A), _dev(Y), out)
    err = np.abs(out.cpu().numpy() - ref).max()
    c.set_i8_slices(0)
    c.matmul(_pitched(A), _dev(Y), out)
    dm = np.abs(out.cpu().numpy() - ref).max()
    scale = np.abs(A).max() * np.abs(Y).max() * n
    assert err <= 2.0 ** -47 * scale and err <= 16 * max(dm, 1e-16 * scale), (err, dm)


def test_slices_reused_only_while_valid():
    """pf_rayleigh_ritz / pf_matmul reuse the slices of the same A; pf_invalidate forces a split."""
    n, p = 512, 32
    rs = np.random.default_rng(3)
    A = rs.standard_normal((n, n))
    Y = rs.standard_normal((n, p))
    c = _ctx(n, p)
    Ad = _pitched(A)
    out = torch.empty((n, p), dtype=torch.float64, device="cuda")
    c.matmul(Ad, _dev(Y), out)
    Ad.mul_(2.0)                                        # written outside libpf
    c.invalidate()
    c.matmul(Ad, _dev(Y), out)
    np.testing.assert_allclose(out.cpu().numpy(), 2 * A @ Y, rtol=0, atol=1e-10)


CFGS = [reduced(CONFIGS[1], dtype="f64i8"),
        reduced(CONFIGS[2], n=1000, iters=8, dtype="f64i8"),
        reduced(CONFIGS[3], n=1500, iters=8, edge_prob=82 / 1500, dtype="f64i8"),
        reduced(CONFIGS[4], n=1200, p=128, iters=4, dtype="f64i8"),
        reduced(NEXT_CONFIGS["nce7"], n=600, iters=10, dtype="f64i8")]
IDS = ["sweep", "pfpg", "pfam", "pfpg_p128", "nce"]


@pytest.mark.parametrize("cfg", CFGS, ids=IDS)
def test_trajectory_matches_oracle(cfg):
    from paper_1904_10585_b200 import run
    ref = O.run(cfg)["records"]
    out = run(cfg)["records"]
    for x, y in zip(ref, out):
        den = max(O.lowrank_fro(x["V"], x["f"]), 1e-300)
        assert O.lowrank_diff_fro(x["V"], x["f"], y["V"], y["f"]) <= 1e-10 * den
        if "objective" in x:
            assert y["objective"] == pytest.approx(x["objective"], rel=1e-10)


@pytest.mark.parametrize("graphs", [False, True])
def test_pfam_trajectory_half_storage_filter(monkeypatch, graphs):
    """PF_I8SYM=1: the PFAM iterate's fused digits are written for the upper tiles only and every
    product runs the half-storage symmetric kernel (lower tiles = stored upper tiles read
    transposed, K1-i8s); the trajectory matches the oracle at the fp64 bar."""
    from paper_1904_10585_b200 import run
    monkeypatch.setenv("PF_I8SYM", "1")
    cfg = CFGS[2]
    ref = O.run(cfg)["records"]
    out = run(cfg, graphs=graphs)["records"]
    for x, y in zip(ref, out):
        den = max(O.lowrank_fro(x["V"], x["f"]), 1e-300)
        assert O.lowrank_diff_fro(x["V"], x["f"], y["V"], y["f"]) <= 1e-10 * den
        if "objective" in x:
            assert y["objective"] == pytest.approx(x["objective"], rel=1e-10)


@pytest.mark.parametrize("cfg", CFGS[1:3], ids=IDS[1:3])
def test_graph_replay_bit_identical(cfg):
    from paper_1904_10585_b200 import run
    a = run(cfg)["records"]
    b = run(cfg, graphs=True)["records"]
    for x, y in zip(a, b):
        assert np.array_equal(x["V"], y["V"]) and np.array_equal(x["f"], y["f"])


@pytest.mark.parametrize("slices", [7, 6])
def test_pfam_update_digits_match_fresh_split(monkeypatch, slices):
    """PFAM on one GPU: pf_admm_step writes Z_new's digit slices under its row bounds
    (pf_rebuild.cu, K4 'fused digits'); the next product reuses them.  The product from
    the fused digits is within the split bound of the exact Z_new Y, and agrees with a fresh split
    (pf_invalidate) to the same bar; PF_FUSE_DIGITS=0 gives the same trajectory."""
    from paper_1904_10585_b200 import run
    from paper_1904_10585_b200._lib import Context, PF_FP64_I8
    from pfinputs import pfam_problem
    cfg = reduced(CONFIGS[3], n=1500, iters=3, edge_prob=82 / 1500, dtype="f64i8")
    n, p = cfg.n, 64
    prob = pfam_problem(cfg)
    rs = np.random.default_rng(11)
    V = np.linalg.qr(rs.standard_normal((n, p)))[0]
    f = np.abs(rs.standard_normal(p)) * 3.0
    f[5:9] = 0.0
    Z0 = rs.standard_normal((n, n)) * 1e-2
    Z0 = Z0 + Z0.T
    from paper_1904_10585_b200.solver import _bits
    c = Context(n, p, 4, dtype=PF_FP64_I8)
    c.set_i8_slices(slices)
    Z = _pitched(Z0)
    obj = torch.zeros(2, dtype=torch.float64, device="cuda")
    c.admm_step(_dev(V), _dev(f), cfg.t, _bits(prob["adj_bits"]), _dev(prob["deg"]), Z, obj)
    Zn = Z.cpu().numpy()
    Y = rs.standard_normal((n, p))
    out = torch.empty((n, p), dtype=torch.float64, device="cuda")
    c.matmul(Z, _dev(Y), out)                           # reuses the fused digits
    fused = out.cpu().numpy()
    c.invalidate()
    c.matmul(Z, _dev(Y), out)                           # fresh split of Z_new
    fresh = out.cpu().numpy()
    ref = Zn @ Y
    scale = np.abs(Zn).max() * np.abs(Y).max() * n
    ef, es = np.abs(fused - ref).max(), np.abs(fresh - ref).max()
    assert ef <= 2.0 ** (5 - 7 * slices) * scale, (ef, es)
    assert ef <= 16 * max(es, 1e-16 * scale), (ef, es)
    if slices != 7:
        return
    a = run(cfg)["records"]
    monkeypatch.setenv("PF_FUSE_DIGITS", "0")
    b = run(cfg)["records"]
    for x, y in zip(a, b):
        den = max(O.lowrank_fro(x["V"], x["f"]), 1e-300)
        assert O.lowrank_diff_fro(x["V"], x["f"], y["V"], y["f"]) <= 1e-10 * den


@pytest.mark.parametrize("n,p", [(1333, 64), (700, 128), (300, 16)])
def test_schedule_uses_leading_slices_of_the_tiled_layout(n, p):
    """pf_set_i8_schedule(6, 0) on a 7-slice context multiplies the 6 leading digit slices of
    each (tile, k-block) group of the tiled A layout: the truncating 7-digit expansion starts
    with the 6-digit one, so the filter equals a 6-slice context's bit for bit."""
    rs = np.random.default_rng(n + p)
    A = rs.standard_normal((n, n))
    A = A + A.T
    U = np.linalg.qr(rs.standard_normal((n, p)))[0]
    interval = torch.tensor([-5.0, 5.0], dtype=torch.float64, device="cuda")
    outs = []
    for slices, sched in ((7, (6, 0)), (6, None)):
        c = _ctx(n, p, slices)
        if sched:
            c.set_i8_schedule(*sched)
        Ud = _dev(U)
        c.filter(_pitched(A), Ud, interval, 1, 1e6)
        outs.append(Ud.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])


# ---------------------------------------------------------------- past the exact-int32 K bound
# i8_plan bounds one exact int32 accumulation to chunk_kb = 292 k-blocks (K = 18688 at S = 7);
# longer K ranges fold each chunk into the fp64 accumulator in the epilogue (pf_gemm_i8.cu), and
# at n = 32768 (config 4) the stream-K split cuts items at arbitrary k-blocks, so CTA segments
# straddle a fold boundary.  Operands are built on the host in int8 (1 GB at n = 32768) and the
# exact reference is formed in fp64 row blocks (integer sums < 2^53: exact in any order).
def _int_problem(n, p, seed):
    rs = np.random.default_rng(seed)
    A8 = rs.integers(-100, 101, (n, n), dtype=np.int8)
    A8[5] = 0                                         # zero row (scale exponent 0)
    Y = rs.integers(-50, 51, (n, p)).astype(np.float64)
    Y[:, 2] = 0.0                                     # zero column
    ref = np.empty((n, p))
    for r0 in range(0, n, 2048):
        ref[r0:r0 + 2048] = A8[r0:r0 + 2048].astype(np.float64) @ Y
    A = torch.empty((n, n), dtype=torch.float64, device="cuda")
    for r0 in range(0, n, 4096):
        A[r0:r0 + 4096].copy_(torch.from_numpy(A8[r0:r0 + 4096]).cuda().to(torch.float64))
    return A, Y, ref


@pytest.mark.slow
@pytest.mark.parametrize("n,p", [(18752, 16), (20000, 64), (32768, 128)])
def test_integer_operands_exact_past_fold(n, p):
    A, Y, ref = _int_problem(n, p, n + p)
    c = _ctx(n, p)
    out = torch.empty((n, p), dtype=torch.float64, device="cuda")
    c.matmul(A, _dev(Y), out)
    got = out.cpu().numpy()
    bad = np.argwhere(got != ref)
    assert bad.size == 0, (bad[:5], got[tuple(bad[0])], ref[tuple(bad[0])])


@pytest.mark.slow
@pytest.mark.parametrize("n,p", [(18752, 64), (32768, 128)])
def test_gaussian_operands_fp64_grade_past_fold(n, p):
    """Symmetric Gaussian A (the iterates' profile), K past the fold: within 2^-47 of the scale
    and within 16x the fp64 DMMA GEMM's own error on the same context."""
    g = torch.Generator(device="cuda").manual_seed(n)
    A = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
    A = A + A.T
    rs = np.random.default_rng(n)
    Y = rs.standard_normal((n, p))
    Ah = A.cpu().numpy()
    ref = Ah @ Y
    scale = np.abs(Ah).max() * np.abs(Y).max() * n
    del Ah
    c = _ctx(n, p)
    out = torch.empty((n, p), dtype=torch.float64, device="cuda")
    c.matmul(A, _dev(Y), out)
    err = np.abs(out.cpu().numpy() - ref).max()
    c.set_i8_slices(0)
    c.matmul(A, _dev(Y), out)
    dm = np.abs(out.cpu().numpy() - ref).max()
    assert err <= 2.0 ** -47 * scale and err <= 16 * max(dm, 1e-16 * scale), (err, dm)


def _digit_bound(X, p):
    """Elementwise bound on |W - V'V^T| for the int8-digit product (pf_rebuild_i8.cu): rows of V'
    and V split under their own scales 2^E_i, 2^F_j (|x| < 2^E), 7 digits (truncation residual
    < 2^(E-49) per entry), levels s + t <= 6 kept (dropped levels < 7 * 127^2 * 128^-9 2^(E+F) per
    product); summed over p products: < 4 p 2^(E_i + F_j - 49)."""
    m = np.abs(X).max(axis=1)
    e = np.where(m > 0, np.floor(np.log2(np.where(m > 0, m, 1.0))) + 1, 0)
    return 2.0 ** e


@pytest.mark.parametrize("n", [64, 100, 300, 1333, 2050, 5000])
@pytest.mark.parametrize("form", ["diag", "matrix"])
@pytest.mark.parametrize("sym", ["1", "0"])
def test_pfam_update_int8_matches_oracle(monkeypatch, n, form, sym):
    """PFAM update with W = V' V^T from int8 tcgen05 digit products (pf_rebuild_i8.cu, one GPU,
    p = 64, fused digits): Z_new = offdiag(W - tC) + Diag(1 - W_ii + Z_ii) element by element
    within the digit-split bound of the exact W (eq:PFAM1 P:389), <C, W> and ||Z_new - Z||_F;
    ragged n (tiles of 128 x 32), the 128 x 128 diagonal blocks, n < 128.  PF_K7I8=0 (the DMMA
    update) agrees within the same bound.  The next product from the fused digits: the
    half-storage symmetric kernel (upper tiles only, the lower ones read transposed; K1-i8s) or,
    PF_I8SYM=0, the full stream-K kernel -- within the split bound of Z_new Y."""
    monkeypatch.setenv("PF_I8SYM", sym)
    from paper_1904_10585_b200._lib import Context, PF_FP64_I8
    from paper_1904_10585_b200.solver import _bits
    from pfinputs import sym_bernoulli_bitmask, unpack_bitmask
    p = 64
    rs = np.random.default_rng(n + (form == "matrix"))
    V = np.linalg.qr(rs.standard_normal((n, p)))[0]
    V[3] *= 1e-3                                        # rows on other scales
    V[min(7, n - 1)] = 0.0                              # a zero row
    bits = sym_bernoulli_bitmask(n, 0.08, np.random.default_rng(5), diagonal=False)
    adj = unpack_bitmask(bits, n)
    deg = adj.sum(1).astype(float)
    C = O.maxcut_C(adj, deg)
    Z = rs.standard_normal((n, n)) * 0.05
    Z = Z + Z.T
    if form == "diag":
        f = np.abs(rs.standard_normal(p)) * 20.0
        f[:4] = 0.0
        Vp, Vr, fr = V * f, V, f
    else:
        B = rs.standard_normal((p, p))
        F = B @ B.T / p
        lam, Y = np.linalg.eigh(F)
        Vp, Vr, fr = V @ F, V @ Y, lam
    Zr, cw, res = O.pfam_next(Vr, fr, Z, C, 0.7)
    bound = 4 * p * 2.0 ** -49 * np.outer(_digit_bound(Vp, p), _digit_bound(V, p))
    bound = np.maximum(bound, bound.T) + 1e-15 * np.abs(Zr).max()
    outs = []
    for k7 in ("1", "0"):
        monkeypatch.setenv("PF_K7I8", k7)
        c = Context(n, p, 4, dtype=PF_FP64_I8)
        Zd = _pitched(Z)
        obj = torch.zeros(2, dtype=torch.float64, device="cuda")
        if form == "diag":
            c.admm_step(_dev(V), _dev(f), 0.7, _bits(bits), _dev(deg), Zd, obj)
        else:
            c.admm_step_f(_dev(V), _dev(F), 0.7, _bits(bits), _dev(deg), Zd, obj)
        Zg = Zd.cpu().numpy()
        err = np.abs(Zg - Zr)
        assert np.all(err <= bound), (k7, float((err / bound).max()))
        if k7 == "1":  # off the 128 x 128 diagonal blocks the mirror store is the tile's
            blk = np.arange(n) // 128
            off = blk[:, None] != blk[None, :]
            assert np.array_equal(Zg[off], Zg.T[off])
        o = obj.cpu().numpy()
        assert o[0] == pytest.approx(cw, rel=1e-11, abs=1e-12)
        assert o[1] == pytest.approx(res, rel=1e-11)
        outs.append(Zg)
        # the fused digits of Z_new drive the next product within the split bound
        Y = rs.standard_normal((n, p))
        out = torch.empty((n, p), dtype=torch.float64, device="cuda")
        c.matmul(Zd, _dev(Y), out)
        ref = Zg @ Y
        scale = np.abs(Zg).max() * np.abs(Y).max() * n
        assert np.abs(out.cpu().numpy() - ref).max() <= 2.0 ** (5 - 49) * scale


@pytest.mark.parametrize("n", [1100, 2300])
def test_z_upper_storage_same_trajectory(n):
    """pf_set_z_upper (the bench's storage): the PFAM update skips the fp64 mirror below the
    128 x 128 diagonal blocks.  Every reader of the iterate on this path reads the stored part
    only, so the trajectory (factors, <C, W>, ||Z+ - Z||) and the stored part of Z are
    bit-identical to full storage; the blocks below keep their stale values."""
    from pfinputs import bench_config, pfam_problem
    from paper_1904_10585_b200 import run
    cfg = reduced(bench_config(3), n=n, p=64, iters=5, edge_prob=0.07, dtype="f64i8",
                  lanczos_every=2)
    prob = pfam_problem(cfg)
    outs = [run(reduced(cfg, z_upper=zu), iters=5, problem=prob, graphs=True) for zu in (True, False)]
    assert outs[0]["solver"].z_upper and not outs[1]["solver"].z_upper
    for a, b in zip(outs[0]["records"], outs[1]["records"]):
        assert a["objective"] == b["objective"] and a["aux"] == b["aux"]
        assert np.array_equal(a["Q"], b["Q"]) and np.array_equal(a["QF"], b["QF"])
    Zu, Zf = outs[0]["solver"].A.cpu().numpy(), outs[1]["solver"].A.cpu().numpy()
    rows = np.arange(n)[:, None]
    stored = np.arange(n)[None, :] >= (rows // 128) * 128
    assert np.array_equal(Zu[stored], Zf[stored])
    i, j = np.nonzero(~stored)
    if i.size:
        got = outs[0]["solver"].iterate_entries(i, j).cpu().numpy()
        assert np.array_equal(got, Zf[i, j])           # read through the mirror
        assert not np.array_equal(Zu[i, j], Zf[i, j])  # the stale part really is not written


def test_z_upper_storage_argument_errors():
    from paper_1904_10585_b200._lib import Context, PF_FP64, PF_FP64_I8, load
    lib = load()
    c = Context(2000, 64, 4, dtype=PF_FP64_I8)
    assert lib.pf_set_z_upper(c.h, 2) == 1                 # not 0 / 1 -> ARG
    assert lib.pf_set_z_upper(c.h, 1) == 0 and lib.pf_set_z_upper(c.h, 0) == 0
    assert lib.pf_set_z_upper(Context(2000, 64, 4, dtype=PF_FP64).h, 1) == 7   # DMMA update
    assert lib.pf_set_z_upper(Context(2000, 32, 4, dtype=PF_FP64_I8).h, 1) == 7  # p != 64
    assert lib.pf_set_z_upper(Context(20000, 64, 4, dtype=PF_FP64_I8).h, 1) == 7  # full GEMV


def test_z_upper_storage_refuses_a_fresh_split():
    """After an upper-only update, a digit split of that iterate (it would read the stale lower
    blocks) fails loudly until pf_invalidate declares the matrix written in full."""
    from pfinputs import bench_config, pfam_problem
    from paper_1904_10585_b200 import run
    from paper_1904_10585_b200._lib import PFError
    cfg = reduced(bench_config(3), n=700, p=64, iters=2, edge_prob=0.1, dtype="f64i8")
    out = run(cfg, iters=2, problem=pfam_problem(cfg))
    s = out["solver"]
    Z = s.A
    Y = torch.randn((cfg.n, 64), dtype=torch.float64, device="cuda")
    o = torch.empty_like(Y)
    s.ctx.matmul(Z, Y, o)                    # the update's own digits: fine
    s.ctx.set_i8_slices(7)                   # drops the digits: the next product re-splits Z
    with pytest.raises(PFError):
        s.ctx.matmul(Z, Y, o)
    s.ctx.invalidate()                       # the caller declares Z written in full
    s.ctx.matmul(Z, Y, o)


@pytest.mark.parametrize("n", [1100, 1333, 2600])
def test_lower_transposed_filter_same_trajectory(monkeypatch, n):
    """K1-i8p in lower-transposed mode (the default, PF_I8T): the update writes the digit slices
    of the upper tiles and of the 256 x 256 diagonal super-blocks only, and the filter reads every
    tile left of a pair's super-block as the stored upper tile transposed (MN-major A).  The
    digits and every exact level sum are the same, so the trajectory is bit-identical to the one
    with all mirror digits written (PF_I8T=0); odd tile counts and graphs included."""
    from pfinputs import bench_config, pfam_problem
    from paper_1904_10585_b200 import run
    cfg = reduced(bench_config(3), n=n, p=64, iters=4, edge_prob=0.07, dtype="f64i8",
                  lanczos_every=2)
    prob = pfam_problem(cfg)
    outs = []
    for flag in ("1", "0"):
        monkeypatch.setenv("PF_I8T", flag)
        outs.append(run(cfg, iters=4, problem=prob, graphs=True))
    for a, b in zip(outs[0]["records"], outs[1]["records"]):
        assert a["objective"] == b["objective"] and a["aux"] == b["aux"]
        assert np.array_equal(a["Q"], b["Q"]) and np.array_equal(a["QF"], b["QF"])
