"""ctypes binding of libpf.so (include/pf.h).  Argument marshalling only: every step of the
hot path runs in the CUDA kernels behind the C ABI.  There is no CPU fallback -- if the shared
library is missing or fails to load, importing the binding raises."""
from __future__ import annotations

import ctypes
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpf.so")

PF_FP64 = 0
PF_TF32 = 2
PF_FP64_I8 = 3   # fp64, filter products from exact int8 tensor-core digit products
PF_OP_PSD = 0
PF_OP_SOFT_THRESHOLD = 1
STATUS = {0: "PF_OK", 1: "PF_ERR_ARG", 2: "PF_ERR_DIM", 3: "PF_ERR_INTERVAL", 4: "PF_ERR_CUDA",
          5: "PF_ERR_NOMEM", 6: "PF_ERR_NCCL", 7: "PF_ERR_UNSUPPORTED", 8: "PF_ERR_BREAKDOWN"}
FLAGS = {0x1: "CHOL_SHIFT", 0x2: "NONFINITE", 0x4: "DEGENERATE_INTERVAL", 0x8: "SATURATED",
         0x10: "JACOBI_MAXSWEEP", 0x20: "LANCZOS_BREAK", 0x40: "NS_FALLBACK"}

_lib = None


def load() -> ctypes.CDLL:
    """Load libpf.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I64, I32, D, U32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_uint32
    sig = {
        "pf_create": [I64, I32, I32, I32, ctypes.POINTER(P)],
        "pf_create_dist": [I64, I32, I32, I32, P, I32, I32, ctypes.POINTER(P)],
        "pf_destroy": [P],
        "pf_status_string": [I32],
        "pf_last_error": [P],
        "pf_local_rows": [P],
        "pf_row0": [P],
        "pf_get_device_status": [P, P, ctypes.POINTER(U32), ctypes.POINTER(I32), P],
        "pf_lanczos": [P, P, I64, P, I32, P, P],
        "pf_interval_psd": [P, P, D, P, P],
        "pf_interval_soft": [P, D, D, P, P],
        "pf_interval_top_r": [P, P, I32, D, P, P],
        "pf_set_degree": [P, I32],
        "pf_filter": [P, P, I64, P, I64, P, I32, D, P],
        "pf_orth": [P, P, I64, P],
        "pf_rayleigh_ritz": [P, P, I64, P, I64, P, I64, P, P],
        "pf_spectral_op": [P, I32, D, P, P, P, P],
        "pf_prox_step": [P, P, I64, P, D, D, P, I64, P, I64, I32, P, I64, P, P],
        "pf_schedule_degree": [P, D, I32, ctypes.POINTER(I32)],
        "pf_svt_kick": [P, P, I64, D, D, D, P, P],
        "pf_svt_filter": [P, P, P, P, P, P, P, P, I64, D, D, P],
        "pf_admm_step": [P, P, I64, P, D, P, I64, P, P, I64, P, P],
        "pf_admm_step_f": [P, P, I64, P, D, P, I64, P, P, I64, P, P],
        "pf_rebuild": [P, P, I64, P, P, I64, P],
        "pf_perturb": [P, P, I64, P, I64, P],
        "pf_perturb_hash": [P, P, I64, ctypes.c_uint64, I32, D, P],
        "pf_nce_step": [P, P, I64, P, D, P, P, P, P, I64, P, P],
        "pf_extrapolate": [P, P, I32, D, P, P, P, I64, P, P],
        "pf_set_tf32_passes": [P, I32],
        "pf_set_tf32_schedule": [P, I32, I32],
        "pf_set_i8_slices": [P, I32],
        "pf_set_i8_schedule": [P, I32, I32],
        "pf_invalidate": [P],
        "pf_set_z_upper": [P, I32],
        "pf_matmul": [P, P, I64, P, I64, P, I64, P],
        "pf_spmm": [P, P, P, P, P, P, I64, D, D, D, P, I64, P, I64, P, I64, P],
        "pf_rr_ns": [P, P, I64, P, I64, I32, D, P, P, P, P],
        "pf_svt_ritz": [P, P, P, P, P, I64, D, P, I64, P, I64, P, P, P, P],
        "pf_svt_update": [P, P, P, P, P, P, I64, P, I64, P, D, P, P],
        "pf_profile": [P, I32],
        "pf_profile_read": [P, P, ctypes.POINTER(D), ctypes.POINTER(I64)],
        "pf_profile_read_update": [P, P, ctypes.POINTER(D), ctypes.POINTER(I64)],
        "pf_kernel_launches": [],
        "pf_diagnostics": [P, P, ctypes.POINTER(D)],
        "pf_nccl_unique_id": [P, I32],
        "pf_loop_create": [I32, ctypes.POINTER(P)],
        "pf_overlap_timeline": [P, P, P, I32, ctypes.POINTER(I32)],
        "pf_loop_destroy": [P],
        "pf_create_loop": [I64, I32, I32, I32, P, I32, ctypes.POINTER(P)],
    }
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int32
    lib.pf_status_string.restype = ctypes.c_char_p
    lib.pf_last_error.restype = ctypes.c_char_p
    lib.pf_local_rows.restype = ctypes.c_int64
    lib.pf_row0.restype = ctypes.c_int64
    lib.pf_kernel_launches.restype = ctypes.c_longlong
    _lib = lib
    return lib


def kernel_launches() -> int:
    """Process-wide number of CUDA kernels launched by libpf."""
    return int(load().pf_kernel_launches())


class PFError(RuntimeError):
    pass


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (128 bytes) for pf_create_dist; broadcast it to every rank."""
    buf = ctypes.create_string_buffer(128)
    st = load().pf_nccl_unique_id(buf, 128)
    if st != 0:
        raise PFError(f"pf_nccl_unique_id: {STATUS.get(st, st)}")
    return buf.raw


def _ptr(t) -> int | None:
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        if not t.is_cuda:
            raise PFError("pf: tensors must live on the GPU (no CPU fallback)")
        return t.data_ptr()
    return int(t)


def _ld(t: torch.Tensor) -> int:
    if t.dim() != 2 or t.stride(1) != 1:
        raise PFError("pf: matrices must be 2-D row-major with unit column stride")
    return t.stride(0)


def _stream(stream) -> int | None:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


class Loopback:
    """In-process loopback communicator for `world` ranks on one GPU (pf_loop_create): the
    test harness of the row-block split.  Each rank's Context(loop=hub, rank=r) must be driven by
    its own host thread on its own stream (every collective is a rendezvous of the W calls)."""

    def __init__(self, world: int):
        self.lib = load()
        self.world = world
        h = ctypes.c_void_p()
        st = self.lib.pf_loop_create(world, ctypes.byref(h))
        if st != 0:
            raise PFError(f"pf_loop_create: {STATUS.get(st, st)}")
        self.h = h

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.pf_loop_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Context:
    """One pf_ctx: scratch for order-n problems with block width p and degree d.

    dtype PF_FP64: A and the n x p blocks are fp64 row-major tensors.
    dtype PF_TF32: A is fp32 row-major, blocks are fp32 p-major tensors of shape (p, n_local)."""

    def __init__(self, n: int, p: int, d: int, nccl_id: bytes | None = None, rank: int = 0,
                 world: int = 1, dtype: int = PF_FP64, loop: "Loopback | None" = None):
        self.lib = load()
        self.n, self.p, self.d, self.dtype = n, p, d, dtype
        self.loop = loop                     # keeps the hub alive as long as the context
        h = ctypes.c_void_p()
        if loop is not None:
            assert loop.world == world, "loopback hub world mismatch"
            st = self.lib.pf_create_loop(n, p, d, dtype, loop.h, rank, ctypes.byref(h))
        elif nccl_id is None:
            st = self.lib.pf_create(n, p, d, dtype, ctypes.byref(h))
        else:
            buf = ctypes.create_string_buffer(nccl_id, 128)
            st = self.lib.pf_create_dist(n, p, d, dtype, buf, rank, world, ctypes.byref(h))
        if st != 0:
            raise PFError(f"pf_create failed: {STATUS.get(st, st)}")
        self.h = h
        self.n_local = self.lib.pf_local_rows(h)
        self.row0 = self.lib.pf_row0(h)

    def _check(self, st: int, what: str):
        if st != 0:
            msg = self.lib.pf_last_error(self.h).decode()
            raise PFError(f"{what}: {STATUS.get(st, st)} {msg}")

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.pf_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ ABI wrappers
    def status(self, stream=None):
        fl, rb = ctypes.c_uint32(), ctypes.c_int32()
        lohi = (ctypes.c_double * 2)()
        self._check(self.lib.pf_get_device_status(self.h, _stream(stream), ctypes.byref(fl),
                                                  ctypes.byref(rb), lohi), "pf_get_device_status")
        names = [v for k, v in FLAGS.items() if fl.value & k]
        return {"flags": fl.value, "names": names, "rebases": rb.value, "lanczos": (lohi[0], lohi[1])}

    def diagnostics(self, stream=None) -> dict:
        d = (ctypes.c_double * 4)()
        self._check(self.lib.pf_diagnostics(self.h, _stream(stream), d), "pf_diagnostics")
        return {"jacobi_sweeps": int(d[0]), "lanczos_steps": int(d[1]), "relative_gap": d[2],
                "eta": d[3]}

    def profile(self, enable: bool):
        self._check(self.lib.pf_profile(self.h, 1 if enable else 0), "pf_profile")

    def profile_read(self, stream=None):
        """(summed ms, launches) of the Chebyshev-step GEMM since profile(True)."""
        ms, n = ctypes.c_double(), ctypes.c_int64()
        self._check(self.lib.pf_profile_read(self.h, _stream(stream), ctypes.byref(ms),
                                             ctypes.byref(n)), "pf_profile_read")
        return ms.value, n.value

    def profile_read_update(self, stream=None):
        """(summed ms, count) of the PFAM updates (pf_admm_step*) since profile(True)."""
        ms, n = ctypes.c_double(), ctypes.c_int64()
        self._check(self.lib.pf_profile_read_update(self.h, _stream(stream), ctypes.byref(ms),
                                                    ctypes.byref(n)), "pf_profile_read_update")
        return ms.value, n.value

    def overlap_timeline(self, stream=None) -> list[float]:
        """Last overlapped step (pf_profile on): [arrival x W, gemm begin x W, gemm end x W] ms."""
        buf = (ctypes.c_double * 192)()
        cnt = ctypes.c_int32(0)
        self._check(self.lib.pf_overlap_timeline(self.h, _stream(stream), buf, 192,
                                                 ctypes.byref(cnt)), "pf_overlap_timeline")
        return [buf[i] for i in range(cnt.value)]

    def lanczos(self, A, v0, m, lo_hi, stream=None):
        self._check(self.lib.pf_lanczos(self.h, _ptr(A), _ld(A), _ptr(v0), m, _ptr(lo_hi),
                                        _stream(stream)), "pf_lanczos")

    def interval_psd(self, lo_hi, eta, interval, stream=None):
        self._check(self.lib.pf_interval_psd(self.h, _ptr(lo_hi), eta, _ptr(interval),
                                             _stream(stream)), "pf_interval_psd")

    def interval_soft(self, thr, eta, interval, stream=None):
        self._check(self.lib.pf_interval_soft(self.h, thr, eta, _ptr(interval), _stream(stream)),
                    "pf_interval_soft")

    def interval_top_r(self, lo_hi, r, eta, interval, stream=None):
        self._check(self.lib.pf_interval_top_r(self.h, _ptr(lo_hi), r, eta, _ptr(interval),
                                               _stream(stream)), "pf_interval_top_r")

    def set_degree(self, d: int):
        self._check(self.lib.pf_set_degree(self.h, d), "pf_set_degree")

    def schedule_degree(self, c: float, k: int) -> int:
        """thm:conv1 degree schedule for iteration k (pf_schedule_degree); returns d_k."""
        d = ctypes.c_int32(0)
        self._check(self.lib.pf_schedule_degree(self.h, float(c), int(k), ctypes.byref(d)),
                    "pf_schedule_degree")
        return int(d.value)

    def filter(self, A, U, interval, q=1, rho_max=1e6, stream=None):
        self._check(self.lib.pf_filter(self.h, _ptr(A), _ld(A), _ptr(U), _ld(U), _ptr(interval),
                                       q, rho_max, _stream(stream)), "pf_filter")

    def orth(self, U, stream=None):
        self._check(self.lib.pf_orth(self.h, _ptr(U), _ld(U), _stream(stream)), "pf_orth")

    def rayleigh_ritz(self, A, U, V, theta, stream=None):
        self._check(self.lib.pf_rayleigh_ritz(self.h, _ptr(A), _ld(A), _ptr(U), _ld(U), _ptr(V),
                                              _ld(V), _ptr(theta), _stream(stream)),
                    "pf_rayleigh_ritz")

    def spectral_op(self, op, thr, theta, f, rank, stream=None):
        self._check(self.lib.pf_spectral_op(self.h, op, thr, _ptr(theta), _ptr(f), _ptr(rank),
                                            _stream(stream)), "pf_spectral_op")

    def prox_step(self, V, f, tau, mu, omega, W, A_out, obj, stream=None):
        """obj <- {h = fit + mu sum|f|, fit} (device)."""
        r = 0 if W is None else W.shape[1]
        ldw = 0 if W is None else _ld(W)
        self._check(self.lib.pf_prox_step(self.h, _ptr(V), _ld(V), _ptr(f), tau, mu, _ptr(omega),
                                          _ld(omega), _ptr(W), ldw, r, _ptr(A_out), _ld(A_out),
                                          _ptr(obj), _stream(stream)), "pf_prox_step")

    def admm_step(self, V, f, t, adj, deg, Z, obj, stream=None):
        self._check(self.lib.pf_admm_step(self.h, _ptr(V), _ld(V), _ptr(f), t, _ptr(adj),
                                          _ld(adj), _ptr(deg), _ptr(Z), _ld(Z), _ptr(obj),
                                          _stream(stream)), "pf_admm_step")

    def rebuild(self, V, f, X, stream=None):
        """X = V diag(f) V^T (dense, local rows; pf_rebuild)."""
        self._check(self.lib.pf_rebuild(self.h, _ptr(V), _ld(V), _ptr(f), _ptr(X), _ld(X),
                                        _stream(stream)), "pf_rebuild")

    def admm_step_f(self, Q, F, t, adj, deg, Z, obj, stream=None):
        """PFAM update with W = Q F Q^T (pf_admm_step_f)."""
        self._check(self.lib.pf_admm_step_f(self.h, _ptr(Q), _ld(Q), _ptr(F), t, _ptr(adj),
                                            _ld(adj), _ptr(deg), _ptr(Z), _ld(Z), _ptr(obj),
                                            _stream(stream)), "pf_admm_step_f")

    def perturb(self, A, E, stream=None):
        self._check(self.lib.pf_perturb(self.h, _ptr(A), _ld(A), _ptr(E), _ld(E),
                                        _stream(stream)), "pf_perturb")

    def nce_step(self, V, f, tau, gdiag, x_in, x_out, B, obj, stream=None):
        self._check(self.lib.pf_nce_step(self.h, _ptr(V), _ld(V), _ptr(f), tau, _ptr(gdiag),
                                         _ptr(x_in), _ptr(x_out), _ptr(B), _ld(B), _ptr(obj),
                                         _stream(stream)), "pf_nce_step")

    def extrapolate(self, hist, lam_rel, gdiag, x_out, B, coef=None, stream=None):
        """hist: list of l+2 device vectors, oldest first."""
        arr = (ctypes.c_void_p * len(hist))(*[_ptr(h) for h in hist])
        self._check(self.lib.pf_extrapolate(self.h, arr, len(hist) - 2, lam_rel, _ptr(gdiag),
                                            _ptr(x_out), _ptr(B), _ld(B), _ptr(coef),
                                            _stream(stream)), "pf_extrapolate")

    def perturb_hash(self, A, seed: int, k: int, noise: float, stream=None):
        self._check(self.lib.pf_perturb_hash(self.h, _ptr(A), _ld(A), seed, k, noise,
                                             _stream(stream)), "pf_perturb_hash")

    def set_tf32_passes(self, passes: int):
        self._check(self.lib.pf_set_tf32_passes(self.h, passes), "pf_set_tf32_passes")

    def set_i8_slices(self, slices: int):
        """PF_FP64_I8: digit slices per operand (6 or 7), 0 = the fp64 DMMA GEMM."""
        self._check(self.lib.pf_set_i8_slices(self.h, slices), "pf_set_i8_slices")

    def set_i8_schedule(self, early_slices: int, exact_tail: int):
        """PF_FP64_I8: early Chebyshev steps on early_slices digits, the last exact_tail on S."""
        self._check(self.lib.pf_set_i8_schedule(self.h, early_slices, exact_tail),
                    "pf_set_i8_schedule")

    def set_z_upper(self, upper: bool):
        """PFAM iterate in upper-block storage (pf_set_z_upper): the update skips the fp64 mirror."""
        self._check(self.lib.pf_set_z_upper(self.h, 1 if upper else 0), "pf_set_z_upper")

    def invalidate(self):
        """A was written outside libpf: the next product re-splits it (PF_FP64_I8)."""
        self._check(self.lib.pf_invalidate(self.h), "pf_invalidate")

    def matmul(self, A, Y, out, stream=None):
        """out = A Y with the context's filter GEMM (fp64 dtypes; local rows)."""
        self._check(self.lib.pf_matmul(self.h, _ptr(A), _ld(A), _ptr(Y), _ld(Y), _ptr(out),
                                       _ld(out), _stream(stream)), "pf_matmul")

    def rr_ns(self, A, U, op, thr, F, rank, iters=None, stream=None):
        """F = f(U^T A U) by Newton-Schulz in one device-side kernel (pf_rr_ns); iters: optional
        device int32 tensor <- sign iterations used (-1 after the device-side Jacobi fallback)."""
        self._check(self.lib.pf_rr_ns(self.h, _ptr(A), _ld(A), _ptr(U), _ld(U), int(op),
                                      float(thr), _ptr(F), _ptr(rank), _ptr(iters),
                                      _stream(stream)), "pf_rr_ns")

    # ---- PFSVT (NEXT-3): sparse operators in compressed-row form (torch int32 / fp64 tensors)
    def spmm(self, ptr, idx, val, X, out, coef=(1.0, 0.0, 0.0), ycur=None, yprev=None,
             vperm=None, stream=None):
        """out = s1 (S X) + s2 ycur + s3 yprev, S = (ptr, idx, val[vperm])."""
        self._check(self.lib.pf_spmm(
            self.h, _ptr(ptr), _ptr(idx), _ptr(val), _ptr(vperm), _ptr(X), _ld(X),
            float(coef[0]), float(coef[1]), float(coef[2]), _ptr(ycur),
            _ld(ycur) if ycur is not None else 0, _ptr(yprev),
            _ld(yprev) if yprev is not None else 0, _ptr(out), _ld(out), _stream(stream)),
            "pf_spmm")

    def svt_kick(self, b, mu, delta, norm2, x, stream=None):
        self._check(self.lib.pf_svt_kick(self.h, _ptr(b), b.numel(), float(mu), float(delta),
                                         float(norm2), _ptr(x), _stream(stream)), "pf_svt_kick")

    def svt_filter(self, ptr, idx, cptr, cidx, perm, x, Q, mu, eta, stream=None):
        self._check(self.lib.pf_svt_filter(self.h, _ptr(ptr), _ptr(idx), _ptr(cptr), _ptr(cidx),
                                           _ptr(perm), _ptr(x), _ptr(Q), _ld(Q), float(mu),
                                           float(eta), _stream(stream)), "pf_svt_filter")

    def svt_ritz(self, ptr, idx, val, Q, mu, U, V, sigma, s, svp, stream=None):
        self._check(self.lib.pf_svt_ritz(self.h, _ptr(ptr), _ptr(idx), _ptr(val), _ptr(Q), _ld(Q),
                                         float(mu), _ptr(U), _ld(U), _ptr(V), _ld(V), _ptr(sigma),
                                         _ptr(s), _ptr(svp), _stream(stream)), "pf_svt_ritz")

    def svt_update(self, ptr, idx, b, x, U, V, s, delta, rss, stream=None):
        self._check(self.lib.pf_svt_update(self.h, _ptr(ptr), _ptr(idx), _ptr(b), _ptr(x), _ptr(U),
                                           _ld(U), _ptr(V), _ld(V), _ptr(s), float(delta),
                                           _ptr(rss), _stream(stream)), "pf_svt_update")

    def set_tf32_schedule(self, early_passes: int, exact_tail: int):
        self._check(self.lib.pf_set_tf32_schedule(self.h, early_passes, exact_tail),
                    "pf_set_tf32_schedule")
