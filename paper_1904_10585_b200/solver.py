"""GPU driver of the PFPG / PFAM / sweep iteration (SURVEY §8(c) order) over the C ABI.

Python only sequences C-ABI calls and moves inputs to device memory; the interval, filter,
orthonormalisation, Rayleigh-Ritz, spectral operator and update all run in libpf.so kernels.
The per-iteration order matches the paper: eq:pfpg1/eq:pfpg2 and
eq:PFAM1/eq:PFAM2, shifted so each iteration is filter -> orth -> RR -> f -> update.
"""
from __future__ import annotations

import numpy as np
import torch

from pfinputs import (Config, initial_block, lanczos_start, cfg1_problem, cfg1_noise, pfpg_problem,
                      pfam_problem, cfg5_problem, nce_problem)

from ._lib import Context, PF_FP64, PF_FP64_I8, PF_TF32, PF_OP_PSD, PF_OP_SOFT_THRESHOLD


def _dev(x, dtype=torch.float64):
    return torch.as_tensor(x, dtype=dtype).cuda()


def _bits(b: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(b).view(np.int32)).cuda()


def _iterate64(nl: int, n: int, init=None) -> torch.Tensor:
    """An (nl x n) fp64 iterate with an even row pitch (16-byte TMA rows, include/pf.h) for any n
    (zeros, or a copy of the host array `init`)."""
    buf = torch.zeros((nl, (n + 1) // 2 * 2), dtype=torch.float64, device="cuda")
    if init is not None:
        buf[:, :n].copy_(torch.from_numpy(np.ascontiguousarray(init)))
    return buf[:, :n]


def rows_of(n: int, rank: int, world: int) -> tuple[int, int]:
    """Row block [r0, r1) owned by `rank` (the C library's split: floor(g n / world))."""
    return rank * n // world, (rank + 1) * n // world


class Solver:
    """Holds the device state of one run: iterate A/Z (local rows x n), block U, factors V, f.

    Distributed (nccl_id given): this process owns rows [r0, r1) = rows_of(n, rank, world) of
    A/Z, U, V and of the row-wise masks; small objects are replicated (include/pf.h)."""

    def __init__(self, cfg: Config, problem: dict | None = None, stream=None,
                 nccl_id: bytes | None = None, rank: int = 0, world: int = 1,
                 graphs: bool = False, ctx: Context | None = None, loop=None):
        self.cfg = cfg
        # CUDA graphs: iterations k >= 1 replay one captured graph of the iteration body
        # (interval -> filter -> RR -> f -> update); the Lanczos refresh stays an eager launch
        # in front of it.  Iterations with a host-side change (degree schedule, extrapolation
        # window) are not graphed.
        self.graphs = (graphs and cfg.deg_c <= 0.0 and not (cfg.mode == "nce" and cfg.accel_l > 0))
        if cfg.rr_ns and cfg.mode not in ("sweep_psd", "sweep_soft", "pfam"):
            raise ValueError("rr_ns: sweep modes and PFAM (pf_admm_step_f) only")
        self.F = None            # f(H) of the last Newton-Schulz Rayleigh-Ritz (p x p)
        self.ns_it = None        # device int: sign iterations of the last pf_rr_ns (-1: fallback)
        self.last_ns = False     # the last iteration's RR ran as Newton-Schulz
        self._graph = {}
        self.graph_launches = {}
        self.replayed_launches = 0   # kernels launched by graph replays (not seen by the counter)
        n, p, d = cfg.n, cfg.p, cfg.d
        self.stream = stream
        if self.graphs and (stream is None or stream.cuda_stream == 0):
            raise ValueError("graphs=True needs a non-default stream (stream capture)")
        self.f32 = cfg.dtype == "tf32"   # fp32 storage, TF32 tensor-core filter (config 5)
        dtype = PF_TF32 if self.f32 else PF_FP64_I8 if cfg.dtype == "f64i8" else PF_FP64
        if ctx is not None:  # a context created beforehand for this shape (scratch reused)
            assert (ctx.n, ctx.p, ctx.d, ctx.dtype) == (n, p, d, dtype), "context shape mismatch"
            self.ctx = ctx
        else:
            self.ctx = Context(n, p, d, nccl_id=nccl_id, rank=rank, world=world, dtype=dtype,
                               loop=loop)
        if self.f32:
            self.ctx.set_tf32_schedule(cfg.tf32_early, cfg.tf32_tail)
        if cfg.dtype == "f64i8":
            self.ctx.set_i8_schedule(cfg.i8_early, cfg.i8_tail)
        dist = nccl_id is not None or loop is not None
        # upper-block storage of the PFAM iterate where the library supports it (one GPU, int8
        # digits, p = 64, n <= 18944); elsewhere the iterate stays in full storage
        self.z_upper = (cfg.z_upper and cfg.mode == "pfam" and cfg.dtype == "f64i8" and not dist
                        and p == 64 and n <= 18944)
        if self.z_upper:
            self.ctx.set_z_upper(True)
        r0, r1 = rows_of(n, rank, world) if dist else (0, n)
        self.r0, self.r1, self.n_local = r0, r1, r1 - r0
        assert self.n_local == self.ctx.n_local
        nl = self.n_local
        self.psd = cfg.mode in ("sweep_psd", "pfam", "nce")
        self.op = PF_OP_PSD if self.psd else PF_OP_SOFT_THRESHOLD
        # problem["_dev"]: inputs already on the device (the e2e path uploads them itself)
        devp = (problem or {}).get("_dev") or {}
        if self.f32:  # p-major fp32 blocks: tensors of shape (p, n_local)
            self.U = devp["U0"] if "U0" in devp else \
                _dev(np.ascontiguousarray(initial_block(cfg)[r0:r1].T), torch.float32)
            self.V = torch.empty((p, nl), dtype=torch.float32, device="cuda")
        else:
            self.U = devp["U0"] if "U0" in devp else _dev(initial_block(cfg)[r0:r1])
            self.V = torch.empty((nl, p), dtype=torch.float64, device="cuda")
        self.theta = torch.empty(p, dtype=torch.float64, device="cuda")
        self.f = torch.zeros(p, dtype=torch.float64, device="cuda")
        self.rank = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.obj = torch.zeros(2, dtype=torch.float64, device="cuda")
        self.lohi = torch.zeros(2, dtype=torch.float64, device="cuda")
        self.interval = torch.zeros(2, dtype=torch.float64, device="cuda")
        self.k = 0
        self.thr = 0.0
        if cfg.mode in ("sweep_psd", "sweep_soft") and cfg.gen == "cfg5":
            if "A0" in devp:
                self.A = devp["A0"]
            else:
                A0 = cfg5_problem(cfg) if problem is None else problem["A0"]
                # 16-byte row pitch for the TMA descriptors (include/pf.h: lda % 4 == 0)
                buf = torch.empty((nl, (n + 3) // 4 * 4), dtype=torch.float32, device="cuda")
                buf[:, :n].copy_(torch.from_numpy(np.ascontiguousarray(A0[r0:r1])))
                self.A = buf[:, :n]
            self.thr = cfg.theta
        elif cfg.mode in ("sweep_psd", "sweep_soft"):
            A0 = cfg1_problem(cfg) if problem is None else problem["A0"]
            self.A = _iterate64(nl, n, A0[r0:r1])
            self.thr = cfg.theta
        elif cfg.mode == "pfpg":
            prob = pfpg_problem(cfg) if problem is None else problem
            self.prob = prob
            self.omega = _bits(prob["omega_bits"][r0:r1])
            self.W = _dev(prob["W"])
            self.mu = prob["mu"]
            self.thr = cfg.tau * prob["mu"]
            self.A = _iterate64(nl, n)
            # X_0 = 0: A_0 = 0 - tau Omega o (0 - M)  (the update kernel with zero factors)
            self.ctx.prox_step(self.V.zero_(), self.f, cfg.tau, self.mu, self.omega, self.W,
                               self.A, self.obj, stream)
        elif cfg.mode == "pfam":
            if "adj_bits" in devp:
                self.adj, self.deg = devp["adj_bits"], devp["deg"]
            else:
                prob = pfam_problem(cfg) if problem is None else problem
                self.prob = prob
                self.adj = _bits(prob["adj_bits"][r0:r1])
                self.deg = _dev(prob["deg"])
            self.A = _iterate64(nl, n)
            # Z_0 = 0 -> Z_1 = prox_tG(0) = offdiag(-tC) + I  (reading R9)
            self.ctx.admm_step(self.V.zero_(), self.f, cfg.t, self.adj, self.deg, self.A,
                               self.obj, stream)
        elif cfg.mode == "nce":
            # nearest correlation estimation (NEXT-1): B = G + Diag(x), x^0 = 1 - diag(G)
            prob = nce_problem(cfg) if problem is None else problem
            self.prob = prob
            G = prob["G"]
            self.gdiag = _dev(np.ascontiguousarray(np.diag(G)))
            self.x = _dev((1.0 - np.diag(G))[r0:r1])
            # extrapolation window (paper §4.3, reading R21): a ring of l + 2 x-buffers IS the
            # history; pf_nce_step writes the next iterate into the next buffer
            self.xbuf = [self.x] + [torch.empty_like(self.x) for _ in range(cfg.accel_l + 1)] \
                if cfg.accel_l > 0 else [self.x]
            self.win = 1                                             # points in the window
            B0 = G[r0:r1].copy()
            B0[np.arange(nl), r0 + np.arange(nl)] = 1.0           # G_ii + x^0_i = 1
            self.A = _iterate64(nl, n, B0)
        else:
            raise ValueError(cfg.mode)
        self.ctx.orth(self.U, stream)
        self._v0 = {}

    def lanczos_vector(self, k: int) -> torch.Tensor:
        if k not in self._v0:
            self._v0[k] = _dev(lanczos_start(self.cfg, k)[self.r0:self.r1])
        return self._v0[k]

    def step(self):
        """One iteration k: interval -> filter (+warm-up at k = 0) -> RR -> f -> update."""
        cfg, ctx, st, k = self.cfg, self.ctx, self.stream, self.k
        if k == 0 or (self.psd and k % cfg.lanczos_every == 0):
            if cfg.lanczos_warm > 0 and k > 0:   # lambda_min tracking (NEXT-2, reading R29)
                ctx.lanczos(self.A, None, cfg.lanczos_warm, self.lohi, st)
            else:
                ctx.lanczos(self.A, self.lanczos_vector(k), cfg.lanczos_steps, self.lohi, st)
        if self.graphs and k >= 1:
            self._replay()
        else:
            self._body(k)
        # Warm start the next filter from the Ritz vectors: Range(V) = Range(U), so the method
        # is unchanged (eqn:subspace-update depends on Range(U) only), but the next H = Q^T A Q
        # is then nearly diagonal and the Jacobi solve converges in one or two sweeps.
        if self.last_ns:
            self.ritz = self.U       # X = U F U^T: the filtered basis itself is the warm start
        else:
            self.ritz = self.V
            self.U, self.V = self.V, self.U
        self.k += 1

    def _replay(self):
        """Replay the captured body for the current (U, V) buffer pair (two graphs: the pair
        swaps every iteration); the first use captures it and then replays it."""
        from ._lib import kernel_launches
        key = self.U.data_ptr()
        g = self._graph.get(key)
        if g is None:
            # capture without a device synchronisation (torch.cuda.graph() would drain the GPU
            # first): the body allocates nothing, so capturing while earlier work still runs
            # is safe, and the GPU stays busy during the host-side capture
            g = torch.cuda.CUDAGraph()
            l0 = kernel_launches()
            with torch.cuda.stream(self.stream):
                g.capture_begin()
                try:
                    self._body(1)
                finally:
                    g.capture_end()
            self.graph_launches[key] = kernel_launches() - l0
            self._graph[key] = g
        with torch.cuda.stream(self.stream):
            g.replay()
        self.replayed_launches += self.graph_launches[key]

    def _body(self, k: int):
        cfg, ctx, st = self.cfg, self.ctx, self.stream
        if self.psd:
            ctx.interval_psd(self.lohi, cfg.eta, self.interval, st)
        else:
            ctx.interval_soft(self.thr, cfg.eta, self.interval, st)
        if cfg.deg_c > 0.0:                                   # thm:conv1 degree schedule (NEXT-4)
            ctx.schedule_degree(cfg.deg_c, k)
        for _ in range(cfg.warmup if k == 0 else 1):
            ctx.filter(self.A, self.U, self.interval, cfg.q, cfg.rho_max, st)
        if cfg.rr_ns:
            # Newton-Schulz f(H) on the device; an eigenvalue at the threshold (no convergence)
            # falls back to Jacobi inside the same call (PF_FLAG_NS_FALLBACK)
            if self.F is None:
                self.F = torch.empty((cfg.p, cfg.p), dtype=torch.float64, device="cuda")
                self.ns_it = torch.zeros(1, dtype=torch.int32, device="cuda")
            ctx.rr_ns(self.A, self.U, self.op, self.thr, self.F, self.rank, self.ns_it, st)
            self.last_ns = True
            if cfg.mode == "pfam":   # W = Q F Q^T (F = H when H is positive definite, R30)
                ctx.admm_step_f(self.U, self.F, cfg.t, self.adj, self.deg, self.A, self.obj, st)
            return
        ctx.rayleigh_ritz(self.A, self.U, self.V, self.theta, st)
        ctx.spectral_op(self.op, self.thr, self.theta, self.f, self.rank, st)
        self.last_ns = False
        if cfg.mode == "pfpg":
            ctx.prox_step(self.V, self.f, cfg.tau, self.mu, self.omega, self.W, self.A, self.obj,
                          st)
        elif cfg.mode == "pfam":
            ctx.admm_step(self.V, self.f, cfg.t, self.adj, self.deg, self.A, self.obj, st)
        elif cfg.mode == "nce":
            if cfg.accel_l > 0:
                nxt = self.xbuf[self.win]
                ctx.nce_step(self.V, self.f, cfg.tau, self.gdiag, self.x, nxt, self.A, self.obj, st)
                self.x = nxt
                self.win += 1
                if self.win == cfg.accel_l + 2:                    # every l + 2 iterates
                    ctx.extrapolate(self.xbuf, cfg.accel_lam, self.gdiag, self.xbuf[0], self.A,
                                    stream=st)
                    self.x = self.xbuf[0]
                    self.win = 1                                     # window restarts at x~
            else:
                ctx.nce_step(self.V, self.f, cfg.tau, self.gdiag, self.x, self.x, self.A, self.obj,
                             st)

    def iterate_entries(self, i, j) -> torch.Tensor:
        """Entries Z[i, j] of the symmetric iterate, read where they are stored: in upper-block
        storage (pf_set_z_upper) an entry left of row i's 128 x 128 diagonal block is read at
        (j, i)."""
        i = torch.as_tensor(i, device=self.A.device)
        j = torch.as_tensor(j, device=self.A.device)
        if self.z_upper:
            low = j < torch.div(i, 128, rounding_mode="floor") * 128
            i, j = torch.where(low, j, i), torch.where(low, i, j)
        return self.A[i, j]

    def perturb(self, E: torch.Tensor):
        self.ctx.perturb(self.A, E, self.stream)

    def perturb_hash(self, k: int):
        """Config-5 workload noise E_k generated on the device (pfinputs.hash_gauss)."""
        self.ctx.perturb_hash(self.A, self.cfg.seed, k, self.cfg.noise, self.stream)

    def ritz_factors(self) -> np.ndarray:
        """Ritz vectors of the last iteration as an (n_local x p) fp64 host array."""
        v = self.ritz.cpu().numpy()
        return (v.T if self.f32 else v).astype(np.float64)

    def objective(self) -> tuple[float, float]:
        """(objective, aux) on the host, as the library wrote them: PFPG (h = fit + mu sum|f|,
        fit); PFAM (<C,W>, ||dZ||_F); NCE (F(x), ||grad F||)."""
        o = self.obj.cpu().numpy()
        if self.cfg.mode == "nce":
            return float(o[0]), float(o[1])            # F(x_k), ||grad F(x_k)||
        return float(o[0]), float(o[1])


def run(cfg: Config, iters: int | None = None, record: bool = True, problem=None,
        nccl_id: bytes | None = None, rank: int = 0, world: int = 1, graphs: bool = False,
        loop=None) -> dict:
    """Run K iterations on the GPU, recording per-iteration factors (local rows) / objectives.
    Distributed: nccl_id (one process per GPU) or loop (a Loopback hub; one thread per rank)."""
    K = cfg.iters if iters is None else iters
    if graphs:                      # capture needs a non-default stream; make it the current one
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            return _run(cfg, K, record, problem, nccl_id, rank, world, st, True, loop)
    return _run(cfg, K, record, problem, nccl_id, rank, world, None, False, loop)


def _run(cfg, K, record, problem, nccl_id, rank, world, stream, graphs, loop=None):
    s = Solver(cfg, problem, stream=stream, nccl_id=nccl_id, rank=rank, world=world,
               graphs=graphs, loop=loop)
    recs = []
    for k in range(K):
        s.step()
        rec = {"k": k}
        if record and s.last_ns:
            # X = Q F Q^T: recorded as the factor pair (Q F, Q) with unit weights
            Q = s.ritz_factors()
            F = s.F.cpu().numpy()
            rec.update(rank=int(s.rank.item()), QF=Q @ F, Q=Q, ns_iters=int(s.ns_it.item()))
            if cfg.mode == "pfam":
                rec["objective"], rec["aux"] = s.objective()
        elif record:
            f = s.f.cpu().numpy()
            keep = f != 0.0
            rec.update(theta=s.theta.cpu().numpy(), rank=int(s.rank.item()),
                       V=s.ritz_factors()[:, keep], f=f[keep])
            if cfg.mode in ("pfpg", "pfam", "nce"):
                rec["objective"], rec["aux"] = s.objective()
            if cfg.mode == "nce":
                rec["x"] = s.x.cpu().numpy()
        if cfg.mode in ("sweep_psd", "sweep_soft") and k + 1 < K:
            if cfg.gen == "cfg5":
                s.perturb_hash(k)
            else:
                s.perturb(_dev(cfg1_noise(cfg, k)[s.r0:s.r1]))
        recs.append(rec)
    torch.cuda.synchronize()
    return {"records": recs, "status": s.ctx.status(), "solver": s}
