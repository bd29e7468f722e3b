"""TEST INFRASTRUCTURE ONLY -- plain fp64 CPU oracle of polynomial-filtered SVT (PFSVT, NEXT-3).

Paper §5.2: the SVT iteration (eqn:svt)

    W^k = shrink_mu(A*(x^{k-1})),      x^k = x^{k-1} + tau_k (b - A(W^k)),

is gradient descent on the dual (eqn:ANM-dual) of min ||X||_* + ||X||_F^2 / (2 mu)
s.t. A(X) = b; here A = P_Omega (matrix completion, Example eg:MC), so A*(x) is the
sparse matrix Y with the values x on Omega.  PFSVT replaces the SVD inside shrink_mu by a
polynomial-filtered subspace of Y^T Y ("subspace extraction from A^T A"), degree
d = 1 in the paper's runs.  Readings (R24): SVT's own parameters
(Cai-Candes-Shen): threshold mu = 5 sqrt(m n) (cfg.svt_tau), step tau_k = 1.2 / SR, the kick
x^0 = ceil(mu / (tau ||b||_2-as-matrix)) tau b, stop at ||P_Omega(X^k) - b|| <= 1e-4 ||b||; the
filter damps the eigenvalues of Y^T Y in [a, b] = [0, (1 - eta) mu^2] (singular values below
the threshold), c = (a + b)/2, e = (b - a)/2 (eqn:cheb-linear-map); orthonormalisation
by Householder QR; Rayleigh-Ritz for singular triplets: B = Y Q, B^T B = W Lambda W^T,
sigma = sqrt(lambda), V = Q W, U = B W Sigma^-1 (P:269-286 applied to Y^T Y).

Only `tests/`, `__graft_entry__.smoke()` and `bench` CPU legs may import this module; the product
shares no code with it (inputs come from `pfinputs`).
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp

from pfinputs import Config, initial_block, svt_guard_block, svt_problem

__all__ = ["svt_kick", "svt_matrix", "shrink_exact", "svt_exact_run", "svt_filter", "svt_ritz",
           "svt_sample", "pfsvt_run", "lowrank_rect_diff_fro", "lowrank_rect_fro",
           "svt_dual_objective"]


def svt_kick(prob: dict) -> np.ndarray:
    """x^0 = k0 tau b, k0 = ceil(mu / (tau ||P_Omega(M)||_2)) (SVT's kicking; reading R24)."""
    k0 = math.ceil(prob["tau"] / (prob["delta"] * prob["norm2"]))
    return k0 * prob["delta"] * prob["b"]


def svt_matrix(prob: dict, x: np.ndarray, n: int) -> sp.csr_matrix:
    """A*(x): the n x n sparse matrix with values x on Omega (CSR order)."""
    return sp.csr_matrix((x, prob["J"], prob["row_ptr"]), shape=(n, n))


def svt_sample(U: np.ndarray, s: np.ndarray, V: np.ndarray, I: np.ndarray,
               J: np.ndarray) -> np.ndarray:
    """A(W) for W = U diag(s) V^T: the entries W_ij on Omega, written out as the sum over l."""
    return np.einsum("el,l,el->e", U[I], s, V[J])


def shrink_exact(Y: np.ndarray, mu: float):
    """shrink_mu(Y) = U diag((sigma - mu)_+) V^T by a full SVD (pins only)."""
    U, sig, Vt = np.linalg.svd(Y, full_matrices=False)
    keep = sig > mu
    return U[:, keep], sig[keep] - mu, Vt[keep].T


def svt_dual_objective(prob: dict, x: np.ndarray, n: int) -> float:
    """eqn:ANM-dual: 0.5 ||shrink_mu(A*(x))||_F^2 - b^T x (exact SVD; pins only)."""
    U, s, V = shrink_exact(svt_matrix(prob, x, n).toarray(), prob["tau"])
    return 0.5 * float(np.sum(s * s)) - float(prob["b"] @ x)


def svt_exact_run(cfg: Config, prob: dict | None = None, iters: int | None = None) -> dict:
    """Plain SVT (eqn:svt) with an exact SVD shrink: the p = n limit of PFSVT (pins only)."""
    prob = svt_problem(cfg) if prob is None else prob
    n = cfg.n
    x = svt_kick(prob)
    recs = []
    nb = float(np.linalg.norm(prob["b"]))
    for k in range(cfg.iters if iters is None else iters):
        U, s, V = shrink_exact(svt_matrix(prob, x, n).toarray(), prob["tau"])
        w = svt_sample(U, s, V, prob["I"], prob["J"])
        res = float(np.linalg.norm(w - prob["b"])) / nb
        recs.append({"k": k, "U": U, "s": s, "V": V, "res": res, "svp": int(s.size)})
        x = x + prob["delta"] * (prob["b"] - w)
    return {"records": recs, "x": x}


def _orth(Y: np.ndarray) -> np.ndarray:
    """Householder QR, sign-fixed."""
    q, r = np.linalg.qr(Y)
    d = np.sign(np.diag(r))
    d[d == 0] = 1.0
    return q * d[None, :]


def svt_filter(S: sp.csr_matrix, Q: np.ndarray, a: float, b: float, d: int) -> np.ndarray:
    """orth(T_d(L(Y^T Y)) Q): the three-term recurrence (eq:cheb) with the operator
    C = Y^T Y applied as two sparse products, L(t) = (t - c)/e."""
    c, e = 0.5 * (a + b), 0.5 * (b - a)
    ST = S.T.tocsr()

    def C(Z):
        return ST @ (S @ Z)

    y_prev, y = Q, (C(Q) - c * Q) / e
    for _ in range(1, d):
        y_prev, y = y, (2.0 / e) * (C(y) - c * y) - y_prev
    return _orth(y)


def svt_ritz(S: sp.csr_matrix, Q: np.ndarray):
    """Singular triplets of Y restricted to span(Q): B = Y Q, B^T B = W diag(lambda) W^T
    (descending), sigma = sqrt(max(lambda, 0)), V = Q W, U = B W diag(1/sigma) (0 where sigma = 0)."""
    B = S @ Q
    lam, W = np.linalg.eigh(B.T @ B)
    order = np.argsort(-lam, kind="stable")
    lam, W = lam[order], W[:, order]
    sig = np.sqrt(np.maximum(lam, 0.0))
    V = Q @ W
    inv = np.where(sig > 0.0, 1.0 / np.where(sig > 0.0, sig, 1.0), 0.0)
    U = (B @ W) * inv[None, :]
    return U, sig, V


def pfsvt_run(cfg: Config, prob: dict | None = None, iters: int | None = None,
              stop: bool = False, record_factors: bool = True) -> dict:
    """PFSVT, step by step: per iteration k
      1. interval [a, b] = [0, (1 - eta) mu^2] on the spectrum of Y^T Y (reading R24);
      2. Q <- orth(T_d(L(Y^T Y)) Q)  (`warmup` sweeps at k = 0, reading R8);
      3. (U, sigma, V) = Rayleigh-Ritz of Y on span(Q);  s = (sigma - mu)_+ (shrink);
      4. w = A(U diag(s) V^T) on Omega;  x <- x + tau (b - w)  (eqn:svt);
      5. warm start Q <- V.
    Records the factors of W^k = U diag(s) V^T (kept columns), svp and the relative residual
    ||w - b|| / ||b|| (the SVT stopping quantity; `stop` ends the run below cfg.svt_tol).
    cfg.svt_adapt (NEXT-2, paper §4.2 "the number of [wanted] eigenvalues in the previous
    iteration is used as an estimation ... guard vectors are also added", reading R27): the next
    block has p_{k+1} = min(p, the smallest of 16/32/64/128 >= svp_k + p_guard) columns -- the
    leading Ritz vectors, or all of them plus svt_guard_block(cfg, k, .) columns."""
    prob = svt_problem(cfg) if prob is None else prob
    n = cfg.n
    mu, tau = prob["tau"], prob["delta"]
    x = svt_kick(prob)

    def bucket(m):
        m = min(m, cfg.p)
        return next(q for q in (16, 32, 64, 128) if q >= m)

    p_cur = bucket(cfg.p0) if cfg.svt_adapt else cfg.p
    Q = _orth(initial_block(cfg)[:, :p_cur])
    a, b = 0.0, (1.0 - cfg.eta) * mu * mu
    nb = float(np.linalg.norm(prob["b"]))
    recs = []
    for k in range(cfg.iters if iters is None else iters):
        S = svt_matrix(prob, x, n)
        for _ in range(cfg.warmup if k == 0 else 1):
            Q = svt_filter(S, Q, a, b, cfg.d)
        U, sig, V = svt_ritz(S, Q)
        s = np.maximum(sig - mu, 0.0)
        keep = s > 0.0
        w = svt_sample(U[:, keep], s[keep], V[:, keep], prob["I"], prob["J"])
        res = float(np.linalg.norm(w - prob["b"])) / nb
        rec = {"k": k, "sigma": sig, "svp": int(keep.sum()), "res": res,
               "saturated": bool(keep.all()), "p": p_cur}
        if record_factors:
            rec.update(U=U[:, keep], s=s[keep], V=V[:, keep])
        recs.append(rec)
        x = x + tau * (prob["b"] - w)
        Q = V
        if cfg.svt_adapt:
            p_next = bucket(int(keep.sum()) + cfg.p_guard)
            if p_next < p_cur:
                Q = V[:, :p_next]
            elif p_next > p_cur:
                Q = np.hstack([V, svt_guard_block(cfg, k, p_next - p_cur)])
            p_cur = p_next
        if stop and res <= cfg.svt_tol:
            break
    return {"records": recs, "x": x, "prob": prob}


def lowrank_rect_fro(U: np.ndarray, s: np.ndarray, V: np.ndarray) -> float:
    """||U diag(s) V^T||_F via thin QRs (no n x n buffer)."""
    if s.size == 0:
        return 0.0
    _, ru = np.linalg.qr(U * s[None, :])
    _, rv = np.linalg.qr(V)
    return float(np.linalg.norm(ru @ rv.T))


def lowrank_rect_diff_fro(U1, s1, V1, U2, s2, V2) -> float:
    """||U1 S1 V1^T - U2 S2 V2^T||_F = ||R_a R_b^T||_F with [U1 S1, -U2 S2] = Q_a R_a and
    [V1, V2] = Q_b R_b (stacked thin QRs: no n x n buffer, no cancellation of squares)."""
    L = np.hstack([U1 * s1[None, :], -U2 * s2[None, :]])
    R = np.hstack([V1, V2])
    if L.shape[1] == 0:
        return 0.0
    _, ra = np.linalg.qr(L)
    _, rb = np.linalg.qr(R)
    return float(np.linalg.norm(ra @ rb.T))
