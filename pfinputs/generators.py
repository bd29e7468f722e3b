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
    dtype: str = "f64"
    seed: int = 0
    # interval / filter knobs (readings R4-R7)
    eta: float = 0.1
    warmup: int = 4
    lanczos_steps: int = 20
    lanczos_every: int = 10
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
    # config 5 soft threshold (reading R11)
    theta: float = 3.0


CONFIGS = {
    1: Config("cfg1_psd_sweep_n256", n=256, p=16, d=4, iters=20, mode="sweep_psd"),
    2: Config("cfg2_pfpg_n4096", n=4096, p=32, d=6, iters=200, mode="pfpg",
              r=10, omega_prob=0.1),
    3: Config("cfg3_pfam_maxcut_n16384", n=16384, p=64, d=8, iters=100, mode="pfam",
              edge_prob=0.005),
    4: Config("cfg4_pfpg_n32768", n=32768, p=128, d=10, iters=100, mode="pfpg",
              r=50, omega_prob=0.05),
    5: Config("cfg5_soft_sweep_n65536", n=65536, p=512, d=8, iters=30, mode="sweep_soft",
              dtype="tf32", rho_max=1e3),
}


def config(i: int) -> Config:
    return CONFIGS[i]


def reduced(cfg: Config, **kw) -> Config:
    """A smaller variant of a config for oracle-speed parity tests."""
    return dataclasses.replace(cfg, **kw)


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
