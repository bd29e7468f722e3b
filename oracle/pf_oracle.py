"""Plain fp64 CPU oracle of the polynomial-filtered PFPG / PFAM iteration (arXiv 1904.10585).

TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module.  It shares no code with the CUDA path.

Citations: ``P:n`` = line n of the paper's LaTeX source, with the section /
equation label.  Readings where the paper is silent, ambiguous or wrong are numbered
R1..R27 and listed in DESIGN.md §2 (R23: a PSD iterate skips the filter).

Each function is the paper's definition or algorithm written out step by step in numpy
fp64; library primitives used as single steps: ``@`` (matmul), ``numpy.linalg.qr``
(Householder QR), ``numpy.linalg.eigh`` (symmetric EVD), ``numpy.linalg.solve``-style
triangular solves.  No blocking, fusion or reordering.

Pins (tests/test_oracle_pins.py) -- what fixes each function independently of itself:
  cheb_T ............ closed values, T_2d(x)=T_d(2x^2-1), Lemma lem:cheb-est grid
  chebyshev_filter .. diagonal A: exact T_d(L(lambda_i)) scaling; known-EVD commutation
  orth .............. Q^T Q = I, span preserved (QR residual)
  rayleigh_ritz ..... invariant-subspace exactness; interlacing; 2x2 closed form; own Jacobi
  spectral ops ...... p = n special case == exact P_+ / soft-threshold from brute-force Jacobi
                      EVD; Moreau invariants; soft-threshold optimality conditions
  lanczos ........... diagonal / known spectrum: extremes within residual bound
  pfam_next ......... 2-node max-cut optimum; 5-cycle SDP value -(25+5 sqrt 5)/8 (closed form);
                      diag(prox) == 1; fixed point maps to itself
  pfpg_next ......... p = n, tau = 1: objective non-increasing; exact-subspace equivalence
  nce_next .......... 2x2 closed form; constant off-diagonal -> 11^T; p = n exact; objective
                      values of tab:ncm
  rna_extrapolate ... trivial windows, the l = 1 closed form, exact recovery of a linear fixed point
  relative_gap ...... hand example of eqn:relative-gap
  eta_k / eta_bound . hand example (T_3(2) = 26); the bound equals the definition when
                      lambda_{s_{p+1}} sits at the interval edge, dominates it otherwise
  degree_schedule ... Theta(log k) growth (thm:conv1's requirement), floor, c = 0 constant; on a
                      static config-1 matrix it reaches exact P_+ where the fixed d = 1 lags
  run ............... config 1 k = 0 == exact P_+; degenerate (PSD) interval == compression P A P;
                      q repeats on a diagonal A (closed form);
                      trajectories of configs 2-5 at full size -- parity unpinned beyond the
                      invariants above and the p = n special case (no published values exist
                      for these inputs).
  PFSVT (pf_svt.py) . dual-gradient identity, p = n == exact-SVD SVT, tab:SVT-MKL row 1.
"""
from __future__ import annotations

import math

import numpy as np

from pfinputs import (Config, initial_block, lanczos_start, cfg1_problem, cfg1_noise,
                      pfpg_problem, pfam_problem, unpack_bitmask, cfg5_problem, cfg5_perturb,
                      nce_problem)

__all__ = [
    "cheb_T", "growth_lower_bound", "interval_map", "interval_psd", "interval_top_r",
    "relative_gap",
    "interval_soft", "lanczos_extremes", "rebase_plan", "spread_estimate", "chebyshev_filter",
    "orth", "filter_update", "rayleigh_ritz", "spectral_psd", "spectral_soft", "jacobi_eig",
    "exact_spectral", "maxcut_C", "prox_tG_diag", "pfam_next", "pfpg_next", "nce_next",
    "rna_extrapolate", "run", "degree_schedule", "eta_k", "eta_bound",
    "lowrank_diff_fro", "lowrank_fro", "sin_theta",
]


# ============================================================================ Chebyshev
def cheb_T(d: int, t: float) -> float:
    """T_d(t), the closed form eq:cheb:
    cos(d arccos t) for |t| <= 1, 1/2((t - sqrt(t^2-1))^d + (t + sqrt(t^2-1))^d) otherwise."""
    t = float(t)
    if abs(t) <= 1.0:
        return math.cos(d * math.acos(t))
    s = math.sqrt(t * t - 1.0)
    return 0.5 * ((t - s) ** d + (t + s) ** d)


def growth_lower_bound(d: int, eps: float) -> float:
    """Lemma lem:cheb-est: T_d(+-(1+eps)) >= 2^(d min(sqrt eps, 1) - 1)."""
    return 2.0 ** (d * min(math.sqrt(eps), 1.0) - 1.0)


def interval_map(a: float, b: float) -> tuple[float, float]:
    """eqn:cheb-linear-map: L(t) = (t - c)/e, c = (b+a)/2, e = (b-a)/2."""
    if not b > a:
        raise ValueError("degenerate interval: b <= a (S:225-226)")
    return 0.5 * (b + a), 0.5 * (b - a)


def interval_psd(lam_min_est: float, eta: float) -> tuple[float, float]:
    """All-positive case: a = lambda_min estimate, b = eta * a (requires a < 0)."""
    a = lam_min_est
    if not a < 0:
        raise ValueError("PSD interval needs a < 0 (S:230)")
    return a, eta * a


def interval_top_r(lam_min_est: float, lam_r_est: float, eta: float) -> tuple[float, float]:
    """Top-r case: b = (1 - eta) lambda_r + eta a."""
    a = lam_min_est
    return a, (1.0 - eta) * lam_r_est + eta * a


def interval_soft(thr: float, eta: float) -> tuple[float, float]:
    """Two-sided soft threshold |lambda| > thr: [-beta, beta], beta = (1-eta) thr
    (reading R6 in DESIGN.md; equals the paper's A^T A route P:1113-1115 since
    T_2d(x) = T_d(2x^2 - 1))."""
    beta = (1.0 - eta) * thr
    return -beta, beta


# ============================================================================ Lanczos
def lanczos_extremes(A: np.ndarray, v0: np.ndarray, m: int, ritz_vector: bool = False):
    """m-step Lanczos with full re-orthogonalisation (the paper's `eigs` for lambda_n,
    P:855-859; reading R5).  Returns (theta_min - |r_min|, theta_max + |r_max|), where
    theta are the Ritz values of the tridiagonal T_m and r the Ritz residual norms
    |beta_m s_{m,i}|.  Stops early on breakdown (beta_j <= 1e-12 * max|alpha|).
    ritz_vector: also return Q_m s_min, the Ritz vector of theta_min (the warm start of the next
    refresh when lambda_min is tracked, reading R29)."""
    n = A.shape[0]
    m = min(m, n)
    Q = np.zeros((n, m))
    alpha = np.zeros(m)
    beta = np.zeros(m)
    q = v0 / np.linalg.norm(v0)
    steps = 0
    for j in range(m):
        Q[:, j] = q
        w = A @ q
        alpha[j] = q @ w
        for _ in range(2):                       # classical Gram-Schmidt, twice
            w = w - Q[:, :j + 1] @ (Q[:, :j + 1].T @ w)
        beta[j] = np.linalg.norm(w)
        steps = j + 1
        if beta[j] <= 1e-12 * max(1.0, np.max(np.abs(alpha[:j + 1]))):
            beta[j] = 0.0
            break
        q = w / beta[j]
    T = np.diag(alpha[:steps]) + np.diag(beta[:steps - 1], 1) + np.diag(beta[:steps - 1], -1)
    theta, S = np.linalg.eigh(T)
    r_min = abs(beta[steps - 1] * S[steps - 1, 0])
    r_max = abs(beta[steps - 1] * S[steps - 1, -1])
    if ritz_vector:
        return float(theta[0] - r_min), float(theta[-1] + r_max), Q[:, :steps] @ S[:, 0]
    return float(theta[0] - r_min), float(theta[-1] + r_max)


# ============================================================================ filter
def spread_estimate(theta_prev, lanczos_lo: float, lanczos_hi: float) -> float:
    """s = max |lambda| estimate used only to schedule re-basing (reading R7):
    the largest previous Ritz magnitude, else the Lanczos extremes."""
    if theta_prev is not None and len(theta_prev):
        return float(np.max(np.abs(theta_prev)))
    return float(max(abs(lanczos_lo), abs(lanczos_hi)))


def rebase_plan(a: float, b: float, spread: float, d: int, rho_max: float) -> list[int]:
    """Steps j (1 <= j < d) after which the pair (Y_j, Y_{j-1}) is re-based (reading R7):
    t_hat = max |L(+-1.1 spread)|; re-base after j when T_j(t_hat)/T_base(t_hat) > rho_max."""
    c, e = interval_map(a, b)
    t_hat = max(1.0, abs((1.1 * spread - c) / e), abs((-1.1 * spread - c) / e))
    plan, base = [], 0
    for j in range(1, d):
        if cheb_T(j, t_hat) / cheb_T(base, t_hat) > rho_max:
            plan.append(j)
            base = j
    return plan


def chebyshev_filter(A: np.ndarray, U: np.ndarray, a: float, b: float, d: int,
                     rebase_after=()) -> np.ndarray:
    """Y_d = T_d(L(A)) U by the three-term recurrence of eq:cheb under the map
    eqn:cheb-linear-map: Y_0 = U, Y_1 = (A Y_0 - c Y_0)/e,
    Y_{j+1} = (2/e)(A Y_j - c Y_j) - Y_{j-1}.
    Re-basing (reading R7): after step j in `rebase_after`, Y_j = Q R (Householder) and
    (Y_j, Y_{j-1}) <- (Y_j R^-1, Y_{j-1} R^-1); the recurrence is right-linear, so Range(Y_d)
    is unchanged in exact arithmetic."""
    if d < 1:
        raise ValueError("degree must be >= 1 (S:112)")
    c, e = interval_map(a, b)
    y_prev = U
    y = (A @ U - c * U) / e
    for j in range(1, d + 1):
        if j in rebase_after and j < d:
            qf, rf = np.linalg.qr(y)
            y = qf
            y_prev = np.linalg.solve(rf.T, y_prev.T).T         # y_prev R^-1
        if j == d:
            break
        y_next = (2.0 / e) * (A @ y - c * y) - y_prev
        y_prev, y = y, y_next
    return y


def orth(Y: np.ndarray) -> np.ndarray:
    """The orthogonalisation of eqn:subspace-update, 'a single QR decomposition'
    (P:220-222): Householder QR (LAPACK geqrf/orgqr), Q factor."""
    q, _ = np.linalg.qr(Y)
    return q


def filter_update(A, U, a, b, d, q=1, rebase_after=()):
    """eqn:subspace-update / eq:pfpg2 / eq:PFAM2:
    U+ = orth(rho^q(A) U), rho applied q times before the orthogonalisation."""
    Y = U
    for _ in range(q):
        Y = chebyshev_filter(A, Y, a, b, d, rebase_after)
    return orth(Y)


# ============================================================================ Rayleigh-Ritz
def rayleigh_ritz(A: np.ndarray, U: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """eqn:RR: H = U^T A U (symmetrised), H = Y Lambda Y^T (LAPACK),
    Ritz values descending, Ritz vectors V = U Y."""
    H = U.T @ (A @ U)
    H = 0.5 * (H + H.T)
    lam, Y = np.linalg.eigh(H)
    order = np.argsort(-lam, kind="stable")
    return lam[order], U @ Y[:, order]


def spectral_psd(theta: np.ndarray) -> np.ndarray:
    """P_+ on the Ritz values: f(lambda) = max(lambda, 0)."""
    return np.maximum(theta, 0.0)


def spectral_soft(theta: np.ndarray, thr: float) -> np.ndarray:
    """Eigenvalue soft threshold sign(lambda) max(|lambda| - thr, 0): the prox of thr*||.||_*
    on S^n (shrink_mu, applied to eigenvalues of a symmetric matrix)."""
    return np.sign(theta) * np.maximum(np.abs(theta) - thr, 0.0)


def jacobi_eig(H: np.ndarray, tol: float = 1e-15, max_sweeps: int = 60):
    """Brute-force cyclic Jacobi EVD (Golub & Van Loan, Alg. 8.5.2/8.5.3), written out; used
    as an EVD independent of LAPACK for the p = n pins.  Returns (values desc, vectors)."""
    A = np.array(H, dtype=np.float64, copy=True)
    n = A.shape[0]
    V = np.eye(n)
    for _ in range(max_sweeps):
        off = float(np.linalg.norm(A - np.diag(np.diag(A))))
        if off <= tol * max(1e-300, np.linalg.norm(A)):
            break
        for p_ in range(n - 1):
            for q_ in range(p_ + 1, n):
                apq = A[p_, q_]
                if apq == 0.0:
                    continue
                tau = (A[q_, q_] - A[p_, p_]) / (2.0 * apq)
                t = (1.0 if tau >= 0 else -1.0) / (abs(tau) + math.sqrt(1.0 + tau * tau))
                c = 1.0 / math.sqrt(1.0 + t * t)
                s = t * c
                ap, aq = A[:, p_].copy(), A[:, q_].copy()
                A[:, p_], A[:, q_] = c * ap - s * aq, s * ap + c * aq
                ap, aq = A[p_, :].copy(), A[q_, :].copy()
                A[p_, :], A[q_, :] = c * ap - s * aq, s * ap + c * aq
                vp, vq = V[:, p_].copy(), V[:, q_].copy()
                V[:, p_], V[:, q_] = c * vp - s * vq, s * vp + c * vq
    lam = np.diag(A).copy()
    order = np.argsort(-lam, kind="stable")
    return lam[order], V[:, order]


def exact_spectral(A: np.ndarray, op: str, thr: float = 0.0) -> np.ndarray:
    """Dense Phi(A) from a brute-force Jacobi EVD (for the p = n pins, n <= 64)."""
    lam, V = jacobi_eig(A)
    f = spectral_psd(lam) if op == "psd" else spectral_soft(lam, thr)
    return (V * f) @ V.T


# ============================================================================ updates
def maxcut_C(adj: np.ndarray, deg: np.ndarray) -> np.ndarray:
    """C = -L/4, L = Diag(deg) - Adj (BASELINE.json configs[2])."""
    return 0.25 * adj.astype(np.float64) - np.diag(0.25 * deg)


def prox_tG_diag(Y: np.ndarray, C: np.ndarray, t: float) -> np.ndarray:
    """prox_tG for G(X) = 1{A X = b} + <C, X> WITH THE SIGN CORRECTED
    (reading R1): (Y - tC) - A^*(A A^*)^{-1}(A(Y - tC) - b), instantiated for
    A = diag, A^* = Diag, A A^* = I, b = 1 (the max-cut SDP constraint diag(X) = 1)."""
    Yc = Y - t * C
    resid = np.diag(Yc) - 1.0                    # A(Y - tC) - b
    return Yc - np.diag(resid)                   # minus A^*(A A^*)^{-1} resid


def pfam_next(V, f, Z, C, t):
    """eq:PFAM1: W = P_+(P_U(Z)) = V diag(f) V^T (f = max(theta, 0)),
    Z+ = prox_tG(2W - Z) - W + Z.  Returns (Z+, <C, W>, ||Z+ - Z||_F)."""
    W = (V * f) @ V.T
    Zn = prox_tG_diag(2.0 * W - Z, C, t) - W + Z
    return Zn, float(np.sum(C * W)), float(np.linalg.norm(Zn - Z))


def pfpg_next(V, f, omega: np.ndarray, M: np.ndarray, tau: float):
    """eq:pfpg1 for F(X) = 1/2||P_Omega(X - M)||^2, R = mu ||X||_*:
    X+ = V diag(f) V^T (the filtered prox of the previous gradient point), the next
    gradient point is A+ = X+ - tau * grad F(X+) = X+ - tau * Omega o (X+ - M).
    Returns (A+, 1/2 ||P_Omega(X+ - M)||_F^2)."""
    X = (V * f) @ V.T
    R = omega * (X - M)
    return X - tau * R, float(0.5 * np.sum(R * R))


def nce_next(V, f, x, G, tau):
    """Dual gradient step of nearest correlation estimation (eqn:NCE-dual, eqn:NCE-gradient,
    P:910-923): with B = G + Diag(x), Pi_+(B) ~ V diag(f) V^T (f = max(theta, 0)),
    F(x) = 1/2 sum f_i^2 - 1^T x, grad F(x) = diag(Pi_+(B)) - 1, x+ = x - tau grad F(x).
    Returns (x+, B+ = G + Diag(x+), F(x), ||grad F(x)||)."""
    d = np.sum((V * V) * f[None, :], axis=1)          # diag(V diag(f) V^T)
    g = d - 1.0
    F = 0.5 * float(np.sum(f * f)) - float(np.sum(x))
    xn = x - tau * g
    B = G + np.diag(xn)
    return xn, B, F, float(np.linalg.norm(g))


def rna_extrapolate(X: np.ndarray, lam_rel: float) -> tuple[np.ndarray, np.ndarray]:
    """Regularized extrapolation (§4.3, Scieur et al.): X = [x^{k-l}, ..., x^{k+1}]
    (n x (l+2), oldest first); U = [x^{k-l+1} - x^{k-l}, ..., x^{k+1} - x^k];
    c = argmin_{1^T c = 1} c^T (U^T U + lambda I) c = (U^T U + lambda I)^{-1} 1 / (1^T (.)^{-1} 1),
    lambda = lam_rel ||U^T U||_F (reading R21); returns (x~ = sum_i c_i x^{k-l+i}, c)."""
    U = X[:, 1:] - X[:, :-1]
    M = U.T @ U
    lam = lam_rel * np.linalg.norm(M)
    if lam == 0.0:
        lam = lam_rel
    z = np.linalg.solve(M + lam * np.eye(M.shape[0]), np.ones(M.shape[0]))
    c = z / z.sum()
    return X[:, :-1] @ c, c


# ============================================================================ metrics
def lowrank_fro(V, f) -> float:
    """||V diag(f) V^T||_F = ||R diag(f) R^T||_F with V = Q R (thin QR; no n x n buffer)."""
    _, R = np.linalg.qr(V)
    return float(np.linalg.norm((R * f[None, :]) @ R.T))


def lowrank_diff_fro(V1, f1, V2, f2) -> float:
    """||V1 F1 V1^T - V2 F2 V2^T||_F = ||R D R^T||_F, [V1 V2] = Q R, D = diag(f1, -f2).
    (Stacking avoids the sqrt(u) cancellation of the Gram-trace expansion.)"""
    B = np.concatenate([V1, V2], axis=1)
    D = np.concatenate([f1, -f2])
    if B.shape[1] == 0:
        return 0.0
    _, R = np.linalg.qr(B)
    return float(np.linalg.norm((R * D[None, :]) @ R.T))


def sin_theta(X: np.ndarray, Y: np.ndarray) -> np.ndarray:
    """Principal-angle sines (Definition) for orthonormal X, Y (n x p), ascending
    angle order reversed (largest first).  Computed as the singular values of
    (I - X X^T) Y, which equal sin(arccos sigma_i(X^T Y)) and stay accurate for tiny angles."""
    R = Y - X @ (X.T @ Y)
    s = np.linalg.svd(R, compute_uv=False)
    return np.clip(s, 0.0, 1.0)


# ============================================================================ driver
def degree_schedule(d0: int, c: float, k: int) -> int:
    """Chebyshev degree of iteration k (thm:conv1): PFPG converges if
    d_k = Omega(log k / min{l, 1}); the schedule d_k = max(d0, ceil(c ln(k + 2))) (c = 0: the
    fixed degree d0) grows like c ln k."""
    if c <= 0.0:
        return d0
    return max(d0, int(math.ceil(c * math.log(k + 2))))



def _threshold(cfg: Config, prob) -> float:
    if cfg.mode == "pfpg":
        return prob["tau"] * prob["mu"]
    return cfg.theta


def relative_gap(theta: np.ndarray, a: float, b: float) -> float:
    """eqn:relative-gap: G_k = min over i in I_k of |lambda_i - (a+b)/2| / ((b-a)/2) - 1,
    I_k the eigenvalues beyond [a, b]; the Ritz values stand in for the eigenvalues (NEXT-2
    diagnostic; the printed denominator (a_k - b_k)/2 is negative -- read as (b - a)/2, SURVEY
    §8(c)).  +inf when no Ritz value lies outside, or the interval is degenerate."""
    if not b > a:
        return float("inf")
    c, e = 0.5 * (a + b), 0.5 * (b - a)
    out = theta[(theta < a) | (theta > b)]
    return float(np.min(np.abs(out - c) / e - 1.0)) if out.size else float("inf")


def eta_k(eigs: np.ndarray, a: float, b: float, d: int, p: int, q: int = 1) -> float:
    """eqn:etak, the definition: with rho = T_d(L(.))^q and the eigenvalues ordered by
    |rho| decreasing (lambda_{s_1}, lambda_{s_2}, ...), eta_k = |rho(lambda_{s_{p+1}})| /
    |rho(lambda_{s_p})| (needs the whole spectrum: pins only)."""
    c, e = interval_map(a, b)
    r = np.sort(np.array([abs(cheb_T(d, (x - c) / e)) ** q for x in eigs]))[::-1]
    return float(r[p] / r[p - 1])


def eta_bound(theta: np.ndarray, a: float, b: float, d: int, q: int = 1) -> float:
    """NEXT-2 diagnostic (reading R28): eta_k of the wanted values, estimated from the
    Rayleigh-Ritz values of the block.  With r Ritz values beyond the damped interval [a, b] and
    at least one inside (a guard direction, so the block holds every eigenvalue beyond [a, b]),
    lambda_{s_{r+1}} lies in [a, b] where |rho| <= 1 and |rho(lambda_{s_r})| >= T_d(1 + G)^q with
    G the relative gap (eqn:relative-gap), so eta_k <= (1 / T_d(1 + G))^q -- the bound behind
    the paper's "eta_k < 1 since G_k >= l > 0".  The Ritz values stand in for the
    eigenvalues (as for G); nan when every Ritz value lies beyond [a, b] (the block may be
    saturated: nothing bounds lambda_{s_{p+1}}), 0 when none does (G = +inf)."""
    if not b > a:
        return float("nan")
    outside = (theta < a) | (theta > b)
    if outside.all():
        return float("nan")
    g = relative_gap(theta, a, b)
    if math.isinf(g):
        return 0.0
    return float((1.0 / cheb_T(d, 1.0 + g)) ** q)


def run(cfg: Config, iters: int | None = None, record_factors: bool = True,
        problem: dict | None = None, progress=None) -> dict:
    """The PFPG / PFAM / sweep iteration of SURVEY.md §8(c), step by step.

    Iteration k (k = 0..K-1), state (A_k, U_{k-1}):
      a1  interval: PSD  -> a from Lanczos (refresh at k = 0 and every `lanczos_every`),
                            b = eta a;
                    soft -> [-beta, beta], beta = (1-eta) thr (reading R6)
      a2/a3  U_k = orth(rho(A_k) U_{k-1}) (eqn:subspace-update); `warmup` sweeps at k = 0 (R8)
      a4  Rayleigh-Ritz of A_k on U_k (eqn:RR)
      a5  f = Phi(theta) (PSD projection or soft threshold)
      a6  update: sweep  A_{k+1} = A_k + E_k (BASELINE configs[0]);
                  PFPG   A_{k+1} = X_{k+1} - tau Omega o (X_{k+1} - M) (eq:pfpg1);
                  PFAM   Z_{k+1} = prox_tG(2W - Z_k) - W + Z_k (eq:PFAM1, corrected sign R1).
    PFAM starts from Z_0 = 0, whose exact iteration (P_+(0) = 0) gives
    Z_1 = prox_tG(0) = offdiag(-tC) + I (reading R9); the filtered iterations then act on Z_1.
    Returns a dict with per-iteration records (factors V_k[:, f != 0], f_k, objective, a, b).
    """
    K = cfg.iters if iters is None else iters
    U = orth(initial_block(cfg))
    M = omega = C = A32 = None
    if cfg.mode in ("sweep_psd", "sweep_soft") and cfg.gen == "cfg5":
        # config 5 stores the iterate in fp32 (BASELINE configs[4]); the oracle computes in fp64
        # on exactly those fp32 values, and the workload's noise update is the fp32 add
        A32 = cfg5_problem(cfg) if problem is None else np.array(problem["A0"], dtype=np.float32)
        A = A32.astype(np.float64)
    elif cfg.mode in ("sweep_psd", "sweep_soft"):
        A = cfg1_problem(cfg) if problem is None else problem["A0"]
    elif cfg.mode == "pfpg":
        prob = pfpg_problem(cfg) if problem is None else problem
        omega = unpack_bitmask(prob["omega_bits"], cfg.n).astype(np.float64)
        M = prob["W"] @ prob["W"].T
        A = cfg.tau * omega * M                                   # X_0 = 0
    elif cfg.mode == "pfam":
        prob = pfam_problem(cfg) if problem is None else problem
        C = maxcut_C(unpack_bitmask(prob["adj_bits"], cfg.n), prob["deg"])
        A = prox_tG_diag(np.zeros((cfg.n, cfg.n)), C, cfg.t)      # Z_1 (reading R9)
    elif cfg.mode == "nce":
        prob = nce_problem(cfg) if problem is None else problem
        Gn = prob["G"]
        xn = 1.0 - np.diag(Gn)                                    # x^0 = 1 - diag(G)
        A = Gn + np.diag(xn)
        hist = [xn.copy()]                                        # extrapolation window (R21)
    else:
        raise ValueError(cfg.mode)
    psd = cfg.mode in ("sweep_psd", "pfam", "nce")
    thr = None if psd else _threshold(cfg, prob if cfg.mode == "pfpg" else None)

    recs = []
    theta_prev = None
    lo = hi = None
    for k in range(K):
        # a1: interval
        if k == 0 or (psd and k % cfg.lanczos_every == 0):
            if cfg.lanczos_warm > 0 and k > 0:     # lambda_min tracking (NEXT-2, reading R29)
                lo, hi, v_bot = lanczos_extremes(A, v_bot, cfg.lanczos_warm, ritz_vector=True)
            else:
                lo, hi, v_bot = lanczos_extremes(A, lanczos_start(cfg, k), cfg.lanczos_steps,
                                                 ritz_vector=True)
        # PSD iterate (a >= 0: nothing to damp): degenerate interval, the filter is
        # skipped this iteration and U_{k-1} is reused (SURVEY §8(c) reading)
        degenerate = psd and not lo < 0
        if degenerate:
            a = b = lo
        elif psd:
            a, b = interval_psd(lo, cfg.eta)
        else:
            a, b = interval_soft(thr, cfg.eta)
        dk = degree_schedule(cfg.d, cfg.deg_c, k)                # NEXT-4 degree schedule
        if not degenerate:
            plan = rebase_plan(a, b, spread_estimate(theta_prev, lo, hi), dk, cfg.rho_max)
            # a2/a3 (q applications of the polynomial per filter)
            for _ in range(cfg.warmup if k == 0 else 1):
                U = filter_update(A, U, a, b, dk, cfg.q, plan)
        else:
            plan = []
        # a4/a5
        theta, V = rayleigh_ritz(A, U)
        f = spectral_psd(theta) if psd else spectral_soft(theta, thr)
        keep = f != 0.0
        rec = {"k": k, "a": a, "b": b, "theta": theta, "rank": int(keep.sum()),
               "saturated": bool(keep.all()), "rebase": plan, "degenerate": degenerate,
               "gap": relative_gap(theta, a, b),
               "eta": eta_bound(theta, a, b, dk, cfg.q) if not degenerate else float("nan")}
        if record_factors:
            rec["V"], rec["f"] = V[:, keep], f[keep]
        # a6
        if cfg.mode in ("sweep_psd", "sweep_soft"):
            if k + 1 < K and A32 is not None:
                cfg5_perturb(cfg, A32, k)                         # A_{k+1} = fl32(A_k + E_k)
                A = A32.astype(np.float64)
            elif k + 1 < K:
                A = A + cfg1_noise(cfg, k)
        elif cfg.mode == "pfpg":
            A, fit = pfpg_next(V[:, keep], f[keep], omega, M, cfg.tau)
            rec["objective"] = fit + prob["mu"] * float(np.sum(np.abs(f)))
            rec["fit"] = fit
        elif cfg.mode == "nce":
            xn, A, F, gn = nce_next(V[:, keep], f[keep], xn, Gn, cfg.tau)
            rec["objective"] = F
            rec["grad_norm"] = gn
            if cfg.accel_l > 0:
                # every l+2 iterates: x <- sum c_i x^{k-l+i} (§4.3), window restarts at x~ (R21)
                hist.append(xn.copy())
                if len(hist) == cfg.accel_l + 2:
                    xn, rec["accel_c"] = rna_extrapolate(np.stack(hist, axis=1), cfg.accel_lam)
                    A = Gn + np.diag(xn)
                    hist = [xn.copy()]
            rec["x"] = xn
        else:
            A, cw, res = pfam_next(V[:, keep], f[keep], A, C, cfg.t)
            rec["objective"] = cw
            rec["residual"] = res
        recs.append(rec)
        theta_prev = theta
        if progress:
            progress(rec)
    return {"cfg": cfg, "records": recs, "final_A": A, "final_U": U}
