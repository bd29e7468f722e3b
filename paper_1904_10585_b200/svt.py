"""GPU driver of polynomial-filtered SVT (PFSVT, NEXT-3; paper §5.2, eqn:svt P:1098-1104) over
the C ABI: sequences pf_svt_kick, pf_svt_filter (the filter on Y^T Y), pf_svt_ritz and
pf_svt_update.
Python only moves the problem data to the device and sequences the calls: the kick, the filter
(interval, recurrence coefficients, sparse products, orthonormalisation; reading R24), the
singular-triplet Rayleigh-Ritz and the dual step all run behind the C ABI."""
from __future__ import annotations

import math

import numpy as np
import torch

from pfinputs import Config, initial_block, svt_guard_block, svt_problem

from ._lib import Context, PF_FP64, PF_FP64_I8


def _i32(a) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).cuda()


def _f64(a) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


class SVTSolver:
    """Device state of one PFSVT run: Omega in CSR + CSC views, b, the dual values x, the block Q
    (n x p) and the factors U, s, V of W^k = shrink_mu(A*(x^{k-1}))."""

    def __init__(self, cfg: Config, problem: dict | None = None, stream=None):
        assert cfg.mode == "svt"
        self.cfg, self.stream = cfg, stream
        prob = svt_problem(cfg) if problem is None else problem
        self.prob = prob
        n = cfg.n
        # NEXT-2 adaptive block size (reading R27): a context and block buffers per supported p,
        # created on first use; the sparse data, b and x are shared
        p = self._bucket(cfg.p0) if cfg.svt_adapt else cfg.p
        self._per_p = {}
        self.mu, self.delta = float(prob["tau"]), float(prob["delta"])
        self.row_ptr, self.col = _i32(prob["row_ptr"]), _i32(prob["J"])
        self.col_ptr, self.row_csc, self.perm = (_i32(prob["col_ptr"]), _i32(prob["rows_csc"]),
                                                 _i32(prob["perm"]))
        self.b = _f64(prob["b"])
        self.nb = float(np.linalg.norm(prob["b"]))
        self.x = torch.empty_like(self.b)
        self.svp = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.rss = torch.zeros(1, dtype=torch.float64, device="cuda")
        self._use(p)
        # SVT's kick x^0 = k0 delta b (reading R24), on the device
        self.ctx.svt_kick(self.b, self.mu, self.delta, prob["norm2"], self.x, stream)
        self.Q = self.blocks[0]
        self.Q.copy_(torch.from_numpy(np.ascontiguousarray(initial_block(cfg)[:, :p])))
        self.ctx.orth(self.Q, stream)
        self.k = 0

    @staticmethod
    def _bucket_sizes():
        return (16, 32, 64, 128)

    def _bucket(self, m: int) -> int:
        m = min(m, self.cfg.p)
        return next(q for q in self._bucket_sizes() if q >= m)

    def _use(self, p: int):
        """Switch the context / block buffers to block size p (allocated on first use)."""
        if p not in self._per_p:
            n, cfg = self.cfg.n, self.cfg
            buf = lambda: torch.empty((n, p), dtype=torch.float64, device="cuda")
            self._per_p[p] = {
                "ctx": Context(n, p, max(cfg.d, 1),
                               dtype=PF_FP64_I8 if cfg.dtype == "f64i8" else PF_FP64),
                "blocks": [buf() for _ in range(2)], "T": None, "U": buf(),
                "sigma": torch.zeros(p, dtype=torch.float64, device="cuda"),
                "s": torch.zeros(p, dtype=torch.float64, device="cuda")}
        d = self._per_p[p]
        self.p = p
        self.ctx, self.blocks, self.T, self.U = d["ctx"], d["blocks"], d["T"], d["U"]
        self.sigma, self.s = d["sigma"], d["s"]

    def _filter(self):
        """Q <- orth(T_d(L(Y^T Y)) Q) on [0, (1 - eta) mu^2] (pf_svt_filter)."""
        self.ctx.svt_filter(self.row_ptr, self.col, self.col_ptr, self.row_csc, self.perm, self.x,
                            self.Q, self.mu, self.cfg.eta, self.stream)

    def step(self):
        cfg, ctx, st = self.cfg, self.ctx, self.stream
        for _ in range(cfg.warmup if self.k == 0 else 1):
            self._filter()
        V = next(y for y in self.blocks if y is not self.Q)
        ctx.svt_ritz(self.row_ptr, self.col, self.x, self.Q, self.mu, self.U, V, self.sigma,
                     self.s, self.svp, st)
        ctx.svt_update(self.row_ptr, self.col, self.b, self.x, self.U, V, self.s, self.delta,
                       self.rss, st)
        self.Q = V            # warm start: span(V) = span(Q)
        self.last = {"U": self.U, "s": self.s, "V": V, "sigma": self.sigma}  # W^k's factors
        if self.cfg.svt_adapt:
            # next block size from this iteration's recovered rank (host read of svp)
            p_next = self._bucket(int(self.svp.item()) + self.cfg.p_guard)
            if p_next != self.p:
                V, p_old, st = self.Q, self.p, self.stream
                self._use(p_next)
                Qn = self.blocks[0]
                if p_next < p_old:
                    Qn.copy_(V[:, :p_next])                    # leading Ritz vectors
                else:
                    Qn[:, :p_old].copy_(V)                     # + seeded guard columns
                    Qn[:, p_old:].copy_(torch.from_numpy(
                        svt_guard_block(self.cfg, self.k, p_next - p_old)))
                self.Q = Qn
        self.k += 1

    def residual(self) -> float:
        """||P_Omega(W^k) - b|| / ||b|| of the last step (host read)."""
        return math.sqrt(float(self.rss.item())) / self.nb

    def factors(self):
        """(U, s, V) of W^k on the host, kept columns only (s > 0)."""
        L = self.last
        s = L["s"].cpu().numpy()
        keep = s > 0.0
        return (L["U"].cpu().numpy()[:, keep], s[keep], L["V"].cpu().numpy()[:, keep])


def run_svt(cfg: Config, iters: int | None = None, problem=None, stop: bool = False,
            record: bool = True) -> dict:
    """K PFSVT iterations on the GPU (or until the relative residual <= cfg.svt_tol)."""
    s = SVTSolver(cfg, problem)
    recs = []
    for k in range(cfg.iters if iters is None else iters):
        s.step()
        rec = {"k": k, "res": s.residual(), "svp": int(s.svp.item())}
        if record:
            rec["U"], rec["s"], rec["V"] = s.factors()
            rec["sigma"] = s.last["sigma"].cpu().numpy()
            rec["p"] = int(s.last["s"].numel())
        recs.append(rec)
        if stop and rec["res"] <= cfg.svt_tol:
            break
    torch.cuda.synchronize()
    return {"records": recs, "solver": s}
