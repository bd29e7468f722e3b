"""Problem generators for the five BASELINE.json configs.

Every random quantity comes from numpy's PCG64 seeded with ``[seed, stream]`` so the
oracle and the GPU path see bit-identical inputs.  Stream ids:

    1  initial block G0 (n x p, N(0,1))                    -- SURVEY §8(c) step 1
    2  Lanczos start vector for refresh k (stream [seed,2,k])
    3  Haar basis Q for config 1
    4  spectrum lambda for config 1
    5  per-iteration symmetric noise E_k for config 1 ([seed,5,k])
    6  ground-truth factor W (M = W W^T) for configs 2/4
    7  sampling mask Omega for configs 2/4
    8  Erdos-Renyi edges for config 3
    9  config-5 spectrum (large eigenvalues, semicircle bulk, positions)
   10  config-5 Householder vectors
   11  NCE data matrix G (Examples 5.2 / 5.3 of the paper)

Config-5 noise is NOT drawn from a numpy stream: at n = 65536 it is 2^31 Gaussians per
iteration, generated on the device by the library's workload helper.  Both sides implement the
same counter-based generator (`hash_gauss` below, pf_perturb_hash in libpf): entry (i, j) of
E_k depends only on (seed, k, min(i,j), max(i,j)).

Masks (Omega, graph adjacency) are delivered as a packed row-major bitmask of uint32
words: bit (j & 31) of word [i, j >> 5] is entry (i, j); row stride = ceil(n/32) words.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    """One BASELINE.json config (or a reduced parity-test variant of it)."""
    name: str
    n: int
    p: int
    d: int
    iters: int
    mode: str                 # "sweep_psd" | "pfpg" | "pfam" | "sweep_soft"
    dtype: str = "f64"        # "f64" | "f64i8" (fp64 via exact int8 products) | "tf32"
    seed: int = 0
    # interval / filter knobs (readings R4-R7)
    eta: float = 0.1
    warmup: int = 4
    lanczos_steps: int = 20
    lanczos_every: int = 10
    # NEXT-2 lambda_min tracking (reading R29): > 0 -> every refresh after the first runs this
    # many Lanczos steps from the bottom Ritz vector of the previous refresh (0 = seeded restarts)
    lanczos_warm: int = 0
    rho_max: float = 1e6      # re-base threshold on the predicted amplification
    # config-1/5 sweep
    noise: float = 1e-3
    # PFPG (configs 2/4): 0.5||P_Omega(X-M)||^2 + mu ||X||_*
    r: int = 0
    omega_prob: float = 0.0
    tau: float = 1.0
    mu_factor: float = 1e-2
    # PFAM (config 3): max-cut SDP on G(n, edge_prob)
    edge_prob: float = 0.0
    t: float = 1.0
    # config 5 soft threshold (reading R11) and workload shape
    theta: float = 3.0
    gen: str = "cfg1"         # sweep workload: "cfg1" (Haar basis) | "cfg5" (Householder basis)
    # TF32 precision schedule of the GPU filter (reading R18; the fp64 oracle ignores it):
    # the first d - tf32_tail Chebyshev steps at tf32_early MMA passes, the rest in 3xTF32
    tf32_early: int = 3
    tf32_tail: int = 0
    # int8-digit fp64 path (dtype "f64i8", reading R25; the oracle ignores it): Chebyshev steps
    # before the last i8_tail multiply i8_early digit slices, the tail and RR all 7
    i8_early: int = 7
    i8_tail: int = 2
    # sweep modes: Rayleigh-Ritz + spectral operator as F = f(H) by Newton-Schulz sign
    # iterations instead of a Jacobi EVD (NEXT-4 / reading R26; the oracle ignores it)
    rr_ns: bool = False
    # PFAM on the one-GPU int8-digit path: the iterate in upper-block storage (pf_set_z_upper,
    # the update skips the fp64 mirror; storage only, the oracle ignores it)
    z_upper: bool = False
    # nearest correlation estimation (mode "nce"): paper Example eg:5.6 (6) or eg:5.7 (7)
    nce_example: int = 7
    # regularized extrapolation of the iterates (§4.3; NEXT-4): window l (0 = off)
    # and lambda = accel_lam * ||U^T U||_2 (SPEC defaults l = 5, 1e-8; reading R21)
    accel_l: int = 0
    accel_lam: float = 1e-8
    # driver variants (NEXT-4): q applications of the polynomial per iteration, and the
    # degree schedule d_k = max(d, ceil(deg_c log(k + 2))) of thm:conv1 (0 = constant)
    q: int = 1
    deg_c: float = 0.0
    nbig: int = 256           # config 5: eigenvalues drawn from U[5, 50]
    nrefl: int = 64           # config 5: Householder reflectors in the basis
    # PFSVT matrix completion (mode "svt", NEXT-3, paper §5.2 Example eg:MC, tab:SVT-MKL):
    # m = n, rank r, sampling ratio sr; SVT parameters (reading R24): threshold
    # svt_tau * sqrt(m n), step svt_delta / sr, stop at ||P_Omega(X - M)|| <= svt_tol ||P_Omega(M)||
    sr: float = 0.0
    svt_tau: float = 5.0
    svt_delta: float = 1.2
    svt_tol: float = 1e-4
    # NEXT-2 adaptive block size (paper §4.2, reading R27): p_k = the smallest supported size
    # >= svp_{k-1} + p_guard (capped at p), starting from p0; grown blocks are completed with
    # seeded Gaussian guard columns (svt_guard_block)
    svt_adapt: bool = False
    p_guard: int = 5
    p0: int = 16


CONFIGS = {
    1: Config("cfg1_psd_sweep_n256", n=256, p=16, d=4, iters=20, mode="sweep_psd"),
    2: Config("cfg2_pfpg_n4096", n=4096, p=32, d=6, iters=200, mode="pfpg",
              r=10, omega_prob=0.1),
    3: Config("cfg3_pfam_maxcut_n16384", n=16384, p=64, d=8, iters=100, mode="pfam",
              edge_prob=0.005),
    4: Config("cfg4_pfpg_n32768", n=32768, p=128, d=10, iters=100, mode="pfpg",
              r=50, omega_prob=0.05),
    5: Config("cfg5_soft_sweep_n65536", n=65536, p=512, d=8, iters=30, mode="sweep_soft",
              dtype="tf32", rho_max=1e3, gen="cfg5", tf32_early=1, tf32_tail=2),
}


# Beyond BASELINE.json: the dual gradient method for nearest correlation
# estimation, paper §5.1 (eqn:NCE-dual, Examples eg:5.6 / eg:5.7, Table tab:ncm).
NEXT_CONFIGS = {
    "nce7": Config("nce_ex57_n4000", n=4000, p=64, d=8, iters=300, mode="nce", nce_example=7),
    "nce6": Config("nce_ex56_n2000", n=2000, p=128, d=8, iters=200, mode="nce", nce_example=6),
    # with the paper's acceleration (§4.3): the configuration tab:ncm's PFPG column is run with
    "nce7a": Config("nce_ex57_n4000_accel", n=4000, p=64, d=8, iters=300, mode="nce",
                    nce_example=7, accel_l=5),
    "nce6a": Config("nce_ex56_n2000_accel", n=2000, p=128, d=8, iters=200, mode="nce",
                    nce_example=6, accel_l=5),
}


# NEXT-3: polynomial-filtered SVT on the matrix completion problems of tab:SVT-MKL;
# d = 1 as in the paper, p = r + guard columns
NEXT_CONFIGS.update({
    "svt1k": Config("svt_mc_n1000_sr20_r10", n=1000, p=16, d=1, iters=300, mode="svt", r=10,
                    sr=0.20),
    "svt5k": Config("svt_mc_n5000_sr10_r50", n=5000, p=64, d=1, iters=300, mode="svt", r=50,
                    sr=0.10),
    "svt10k": Config("svt_mc_n10000_sr15_r50", n=10000, p=64, d=1, iters=300, mode="svt", r=50,
                     sr=0.15),
})


def config(i: int) -> Config:
    return CONFIGS[i]


def reduced(cfg: Config, **kw) -> Config:
    """A smaller variant of a config for oracle-speed parity tests."""
    return dataclasses.replace(cfg, **kw)


# The method options bench.py times on config 3 (both are the method, DESIGN.md readings):
# R30 -- the Rayleigh-Ritz spectral operator in matrix form (P_+(H) = H when H is positive
# definite, else Newton-Schulz with a Jacobi fallback; update W = Q F Q^T), and R29 -- lambda_min
# tracked by warm-started 8-step Lanczos refreshes.  The full-size parity test runs the same.
BENCH_METHOD = {"rr_ns": True, "lanczos_warm": 8, "z_upper": True}


def bench_config(cfg_id: int = 3) -> Config:
    return dataclasses.replace(CONFIGS[cfg_id], **(BENCH_METHOD if cfg_id == 3 else {}))


def _rng(seed: int, *stream: int) -> np.random.Generator:
    return np.random.default_rng([seed, *stream])


def bitmask_words(n: int) -> int:
    return (n + 31) // 32


def initial_block(cfg: Config) -> np.ndarray:
    """G0: n x p iid N(0,1), the un-orthonormalised warm-start block (row-major)."""
    return _rng(cfg.seed, 1).standard_normal((cfg.n, cfg.p))


def lanczos_start(cfg: Config, k: int) -> np.ndarray:
    """Start vector (un-normalised, N(0,1)) for the Lanczos refresh at iteration k."""
    return _rng(cfg.seed, 2, k).standard_normal(cfg.n)


# ----------------------------------------------------------------------------- config 1
def cfg1_problem(cfg: Config) -> np.ndarray:
    """A_0 = Q diag(lambda) Q^T, Q Haar (sign-fixed QR of a Gaussian), lambda = 8 x U[1,10]
    and n-8 x U[-1,-0.01] (BASELINE.json configs[0])."""
    n = cfg.n
    g = _rng(cfg.seed, 3).standard_normal((n, n))
    q, r = np.linalg.qr(g)
    q = q * np.sign(np.diag(r))[None, :]
    rs = _rng(cfg.seed, 4)
    npos = min(8, n)
    lam = np.concatenate([rs.uniform(1.0, 10.0, npos), rs.uniform(-1.0, -0.01, n - npos)])
    a0 = (q * lam[None, :]) @ q.T
    return 0.5 * (a0 + a0.T)


def cfg1_noise(cfg: Config, k: int) -> np.ndarray:
    """E_k = noise * (G_k + G_k^T)/2, G_k iid N(0,1): A_{k+1} = A_k + E_k."""
    g = _rng(cfg.seed, 5, k).standard_normal((cfg.n, cfg.n))
    return cfg.noise * 0.5 * (g + g.T)


# ----------------------------------------------------------------------------- masks
def sym_bernoulli_bitmask(n: int, prob: float, rng: np.random.Generator,
                          diagonal: bool) -> np.ndarray:
    """Symmetric Bernoulli(prob) pattern: entry (i, j), i <= j, drawn iid (row by row, the
    full row of n uniforms is drawn so the stream does not depend on chunking), then
    mirrored.  Returns the packed uint32 bitmask [n, ceil(n/32)]."""
    w = bitmask_words(n)
    upper = np.zeros((n, 32 * w), dtype=bool)
    chunk = max(1, (1 << 24) // max(n, 1))
    for i0 in range(0, n, chunk):
        i1 = min(n, i0 + chunk)
        u = rng.random((i1 - i0, n))
        m = u < prob
        rows = np.arange(i0, i1)[:, None]
        cols = np.arange(n)[None, :]
        m &= (cols > rows) | ((cols == rows) & diagonal)
        upper[i0:i1, :n] = m
    full = upper[:, :n] | upper[:, :n].T
    upper[:, :n] = full
    del full
    packed = np.packbits(upper, axis=1, bitorder="little")
    return np.ascontiguousarray(packed).view(np.uint32).reshape(n, w)


def unpack_bitmask(bits: np.ndarray, n: int) -> np.ndarray:
    """Inverse of the packing above: bool [rows, n] (rows = bits.shape[0])."""
    b8 = np.ascontiguousarray(bits).view(np.uint8).reshape(bits.shape[0], -1)
    return np.unpackbits(b8, axis=1, bitorder="little")[:, :n].astype(bool)


# ----------------------------------------------------------------------------- configs 2/4
def _spectral_norm_masked(W: np.ndarray, mask_bits: np.ndarray, n: int) -> float:
    """||P_Omega(W W^T)||_2 via ARPACK on the sparse masked matrix (problem-data setup for
    mu = mu_factor * ||P_Omega(M)||_2, BASELINE.json configs[1]); not the method."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as sla
    rows, cols = [], []
    chunk = max(1, (1 << 24) // max(n, 1))
    for i0 in range(0, n, chunk):
        m = unpack_bitmask(mask_bits[i0:i0 + chunk], n)
        r_, c_ = np.nonzero(m)
        rows.append(r_ + i0)
        cols.append(c_)
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    vals = np.empty(rows.shape[0])
    step = 1 << 22
    for s in range(0, rows.shape[0], step):
        vals[s:s + step] = np.einsum("ij,ij->i", W[rows[s:s + step]], W[cols[s:s + step]])
    A = sp.csr_matrix((vals, (rows, cols)), shape=(n, n))
    v0 = _rng(0, 99).standard_normal(n)
    ev = sla.eigsh(A, k=1, which="LM", v0=v0, tol=1e-13, return_eigenvectors=False)
    return float(abs(ev[0]))


def pfpg_problem(cfg: Config) -> dict:
    """Configs 2/4: min 0.5||P_Omega(X - M)||_F^2 + mu ||X||_*, M = W W^T, W iid N(0,1)
    n x r, Omega symmetric Bernoulli(omega_prob) with the diagonal drawn too,
    mu = mu_factor * ||P_Omega(M)||_2, tau = 1 (BASELINE.json configs[1], configs[3])."""
    n = cfg.n
    W = _rng(cfg.seed, 6).standard_normal((n, cfg.r))
    omega = sym_bernoulli_bitmask(n, cfg.omega_prob, _rng(cfg.seed, 7), diagonal=True)
    mu = cfg.mu_factor * _spectral_norm_masked(W, omega, n)
    return {"W": W, "omega_bits": omega, "mu": mu, "tau": cfg.tau}


# ----------------------------------------------------------------------------- config 3
def pfam_problem(cfg: Config) -> dict:
    """Config 3: min <C, X> s.t. diag(X) = 1, X PSD, C = -L/4, L the Laplacian of an
    Erdos-Renyi G(n, edge_prob) graph with unit weights (BASELINE.json configs[2]).
    Delivered as the adjacency bitmask plus the degree vector; C_ij = 1/4 on edges,
    C_ii = -deg_i/4, 0 elsewhere."""
    n = cfg.n
    adj = sym_bernoulli_bitmask(n, cfg.edge_prob, _rng(cfg.seed, 8), diagonal=False)
    deg = np.zeros(n)
    chunk = max(1, (1 << 24) // max(n, 1))
    for i0 in range(0, n, chunk):
        deg[i0:i0 + chunk] = unpack_bitmask(adj[i0:i0 + chunk], n).sum(axis=1)
    return {"adj_bits": adj, "deg": deg, "t": cfg.t}


# ----------------------------------------------------------------------------- config 5
def cfg5_spectrum(cfg: Config) -> np.ndarray:
    """lambda: nbig entries U[5, 50] and n - nbig from the Wigner semicircle on [-1, 1]
    (x = sqrt(u1) cos(2 pi u2): the abscissa of a uniform point of the unit disk), placed at
    seeded random positions (BASELINE.json configs[4]; reading R16)."""
    n, nb = cfg.n, min(cfg.nbig, cfg.n)
    rs = _rng(cfg.seed, 9)
    big = rs.uniform(5.0, 50.0, nb)
    u1 = rs.random(n - nb)
    u2 = rs.random(n - nb)
    bulk = np.sqrt(u1) * np.cos(2.0 * np.pi * u2)
    lam = np.concatenate([big, bulk])
    return lam[rs.permutation(n)]


def cfg5_reflectors(cfg: Config) -> tuple[np.ndarray, np.ndarray]:
    """Q = H_1 H_2 ... H_m, H_i = I - 2 v_i v_i^T, v_i = w_i / |w_i|, w_i iid N(0, I_n), in the
    compact WY form Q = I - V T V^T (T upper triangular): appending H_j to Q_{j-1} =
    I - V T V^T gives T' = [[T, -2 T V^T v_j], [0, 2]].  Returns (V, T)."""
    n, m = cfg.n, cfg.nrefl
    W = _rng(cfg.seed, 10).standard_normal((n, m))
    V = W / np.linalg.norm(W, axis=0)[None, :]
    T = np.zeros((m, m))
    for j in range(m):
        T[j, j] = 2.0
        if j:
            T[:j, j] = -2.0 * T[:j, :j] @ (V[:, :j].T @ V[:, j])
    return V, T


def cfg5_basis_columns(V: np.ndarray, T: np.ndarray, idx: np.ndarray) -> np.ndarray:
    """Columns idx of Q = I - V T V^T (n x len(idx))."""
    n = V.shape[0]
    cols = -(V @ (T @ V[idx].T))
    cols[idx, np.arange(len(idx))] += 1.0
    return cols


class Cfg5Matrix:
    """A_0 = Q diag(lambda) Q^T for config 5, formed row block by row block in fp64 from the
    compact WY factors: A_0 = Lam - V T P^T - P T^T V^T + V (T V^T P T^T) V^T with P = Lam V."""

    def __init__(self, cfg: Config):
        self.n = cfg.n
        self.lam = cfg5_spectrum(cfg)
        self.V, self.T = cfg5_reflectors(cfg)
        self.P = self.lam[:, None] * self.V
        self.K = self.T @ (self.V.T @ self.P) @ self.T.T
        self.VT_T = self.V @ self.T            # n x m
        self.P_Tt = self.P @ self.T.T          # n x m

    def rows(self, i0: int, i1: int, j0: int = 0) -> np.ndarray:
        """fp64 entries [i0, i1) x [j0, n) of A_0."""
        V, P = self.V[j0:], self.P[j0:]
        out = -(self.VT_T[i0:i1] @ P.T) - (self.P_Tt[i0:i1] @ V.T) + (self.V[i0:i1] @ self.K) @ V.T
        r = np.arange(i0, i1)
        on = (r >= j0)
        out[np.arange(i1 - i0)[on], r[on] - j0] += self.lam[i0:i1][on]
        return out


def cfg5_problem(cfg: Config, chunk: int = 2048) -> np.ndarray:
    """A_0 rounded once to fp32 (the stored iterate of config 5), n x n float32.  The upper
    triangle (fp64 rows rounded to fp32) defines the matrix; the lower triangle is its exact
    mirror, so the stored matrix is exactly symmetric."""
    M = Cfg5Matrix(cfg)
    n = cfg.n
    A = np.empty((n, n), dtype=np.float32)
    for i0 in range(0, n, chunk):
        i1 = min(n, i0 + chunk)
        A[i0:i1, i0:] = M.rows(i0, i1, i0)
        blk = A[i0:i1, i0:i1]
        lower = np.tril_indices(i1 - i0, -1)
        blk[lower] = blk.T[lower]
        if i0:
            A[i0:i1, :i0] = A[:i0, i0:i1].T
    return A


_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _mix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 step on uint64 arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def hash_gauss(seed: int, k: int, i: np.ndarray, j: np.ndarray) -> np.ndarray:
    """Counter-based N(0,1) for the symmetric pair {i, j} of noise draw k:
    c = min(i,j) * 2^32 + max(i,j); z1 = mix(c ^ mix(seed * 2^32 + k)); z2 = mix(z1);
    u1 = ((z1 >> 11) + 1) 2^-53 in (0, 1], u2 = (z2 >> 11) 2^-53; g = sqrt(-2 ln u1) cos(2 pi u2)
    (Box-Muller), all in fp64.  pf_perturb_hash implements the same function."""
    lo = np.minimum(i, j).astype(np.uint64)
    hi = np.maximum(i, j).astype(np.uint64)
    key = _mix64(np.uint64(seed) * np.uint64(1 << 32) + np.uint64(k))
    z1 = _mix64(((lo << np.uint64(32)) | hi) ^ key)
    z2 = _mix64(z1)
    u1 = ((z1 >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * (2.0 ** -53)
    u2 = (z2 >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos((2.0 * np.pi) * u2)


def cfg5_noise_rows(cfg: Config, k: int, i0: int, i1: int) -> np.ndarray:
    """Rows [i0, i1) of E_k in fp32: E_ij = fl32(noise * g_ij * s_ij), s = 1 on the diagonal and
    1/sqrt(2) off it -- the law of noise * (G + G^T)/2 with G iid N(0,1) ("1e-3 Gaussian
    symmetric noise", BASELINE.json configs[4]).  The product is evaluated as
    (noise * g) * s in fp64, then rounded once to fp32."""
    rows = np.arange(i0, i1)[:, None]
    cols = np.arange(cfg.n)[None, :]
    g = hash_gauss(cfg.seed, k, rows, cols)
    e = cfg.noise * g
    e = np.where(rows == cols, e, e * 0.7071067811865476)
    return e.astype(np.float32)


def cfg5_perturb(cfg: Config, A32: np.ndarray, k: int, chunk: int = 256,
                 threads: int | None = None) -> None:
    """In place: A_{k+1} = fl32(A_k + E_k) (fp32 add, round to nearest) on an fp32 array.

    E_k is symmetric entry by entry (the hash keys on the unordered pair), so each row chunk
    [i0, i1) draws only its upper part E[i0:i1, i0:] and adds it to both A[i0:i1, i0:] and the
    mirrored A[i1:, i0:i1] -- the same values cfg5_noise_rows gives row by row.  Chunks touch
    disjoint entries, so they run on a thread pool (numpy releases the GIL in the element-wise
    kernels); the result does not depend on the thread count."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    n = cfg.n

    def one(i0):
        i1 = min(n, i0 + chunk)
        rows = np.arange(i0, i1)[:, None]
        cols = np.arange(i0, n)[None, :]
        e = cfg.noise * hash_gauss(cfg.seed, k, rows, cols)
        e = np.where(rows == cols, e, e * 0.7071067811865476).astype(np.float32)
        A32[i0:i1, i0:] += e
        if i1 < n:
            A32[i1:, i0:i1] += e[:, i1 - i0:].T

    starts = range(0, n, chunk)
    nt = threads or len(os.sched_getaffinity(0))
    if nt <= 1 or n <= chunk:
        for i0 in starts:
            one(i0)
        return
    with ThreadPoolExecutor(max_workers=nt) as ex:
        list(ex.map(one, starts))


# ----------------------------------------------------------------------------- NCE (NEXT-1)
def nce_problem(cfg: Config) -> dict:
    """G of Examples eg:5.6 / eg:5.7: G_ij iid uniform in [-1, 1] (5.6) or [0, 2]
    (5.7) for i < j, mirrored, G_ii = 1.  Upper triangle drawn row by row from stream 11."""
    n = cfg.n
    lo, hi = (-1.0, 1.0) if cfg.nce_example == 6 else (0.0, 2.0)
    rs = _rng(cfg.seed, 11)
    G = np.empty((n, n))
    for i in range(n):
        G[i, i:] = rs.uniform(lo, hi, n - i)
    iu = np.triu_indices(n, 1)
    G[(iu[1], iu[0])] = G[iu]
    np.fill_diagonal(G, 1.0)
    return {"G": G}


def svt_guard_block(cfg: Config, k: int, m: int) -> np.ndarray:
    """m new N(0, 1) columns (n x m) for a block grown after iteration k (NEXT-2, reading R27)."""
    return _rng(cfg.seed, 14, k).standard_normal((cfg.n, m))


def svt_problem(cfg: Config) -> dict:
    """Example eg:MC: M = M_L M_R^T with M_L, M_R iid N(0, 1) (n x r), Omega = a
    uniformly sampled set of round(sr n^2) index pairs (without replacement), b = P_Omega(M).
    Omega is delivered sorted row-major (CSR order: rows I, columns J, row pointer) plus its
    column-major view (CSC pointer, rows, and perm: CSC position -> CSR position).  norm2 =
    ||P_Omega(M)||_2 (ARPACK, setup for the SVT kick k0 = ceil(tau / (delta norm2)), reading R24)."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as sla
    n, r = cfg.n, cfg.r
    rs = _rng(cfg.seed, 11)
    ML = rs.standard_normal((n, r))
    MR = rs.standard_normal((n, r))
    nnz = int(round(cfg.sr * n * n))
    lin = np.sort(_rng(cfg.seed, 12).choice(n * n, nnz, replace=False))
    I = (lin // n).astype(np.int32)
    J = (lin % n).astype(np.int32)
    b = np.einsum("ij,ij->i", ML[I], MR[J])
    row_ptr = np.zeros(n + 1, dtype=np.int32)
    np.cumsum(np.bincount(I, minlength=n), out=row_ptr[1:])
    perm = np.lexsort((I, J)).astype(np.int32)        # CSC order: by column, then row
    col_ptr = np.zeros(n + 1, dtype=np.int32)
    np.cumsum(np.bincount(J, minlength=n), out=col_ptr[1:])
    S = sp.csr_matrix((b, J, row_ptr), shape=(n, n))
    norm2 = float(sla.svds(S, k=1, v0=_rng(cfg.seed, 13).standard_normal(n), tol=1e-12,
                           return_singular_vectors=False)[0])
    return {"ML": ML, "MR": MR, "I": I, "J": J, "b": b, "row_ptr": row_ptr, "col_ptr": col_ptr,
            "perm": perm, "rows_csc": I[perm], "norm2": norm2,
            "tau": cfg.svt_tau * n, "delta": cfg.svt_delta / cfg.sr}
