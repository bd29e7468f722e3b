/*
 * pf.h -- C ABI of the B200 hot path of the polynomial-filtered first-order methods PFPG / PFAM
 * (Liu, Wen, Zhang et al., arXiv 1904.10585).  Citations "P:n" are lines of the paper's LaTeX
 * source with the equation label; DESIGN.md lists the readings R1..R14.
 *
 * Conventions (all entry points)
 *  - The context's dtype fixes the storage of the n-row objects:
 *      PF_FP64: A/Z and the blocks U, V are fp64 ROW-MAJOR (block element (i, c) at U[i*ldu + c]);
 *               ld even (16-byte TMA row pitch), base 16-byte aligned; p in {16, 32, 64, 128}.
 *      PF_TF32: A is fp32 ROW-MAJOR (lda % 4 == 0, base 16-byte aligned) and the blocks U, V are
 *               fp32 P-MAJOR: block element (i, c) at U[c*ldu + i], ldu >= n_local (the block's
 *               transpose, row-major); p in {64, 128, 256, 512}.  The filter GEMM runs on the
 *               tcgen05 TF32 tensor cores in 3xTF32 (hi/lo split, fp32 accumulation); Gram, H and
 *               every p x p object are fp64.  BASELINE configs[4] ("fp32/TF32").
 *    Every matrix argument is a DEVICE pointer with its leading dimension (elements between
 *    consecutive rows of the stored array) given next to it.
 *  - n is the matrix order, p the block width (p <= n).
 *  - With world > 1 (pf_create_dist) rank g owns rows [row0, row0 + n_local) of every n-row
 *    object (A, Z, U, V) where row0 = g*n/world (integer division); those row blocks are what
 *    the caller passes.  Small objects (theta, f, rank, obj, interval) are replicated.
 *  - Scalar outputs are device pointers so a whole iteration can be captured in a CUDA graph.
 *  - The caller allocates all arguments; the context owns only scratch allocated in pf_create.
 *    No call allocates device memory.  One context is used by one host thread at a time; calls
 *    are stream-ordered on the stream argument and never synchronise the host (except
 *    pf_get_device_status, which synchronises `stream`).
 *  - Argument errors are returned synchronously (nothing is enqueued).  Numerical events
 *    (Cholesky shift used, non-finite values, degenerate interval, saturation) set bits in a
 *    device status word read by pf_get_device_status.
 */
#ifndef PF_H_
#define PF_H_
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pf_ctx_s* pf_ctx;
typedef void* pf_stream; /* a cudaStream_t; NULL = legacy default stream */

typedef enum {
  PF_FP64 = 0, /* fp64 storage + fp64 DMMA tensor cores (mma.sync .f64)                    */
  PF_FP32 = 1, /* reserved (plain fp32 SIMT filter): not built, PF_ERR_UNSUPPORTED          */
  PF_TF32 = 2, /* fp32 storage, tcgen05 kind::tf32 filter GEMM (3xTF32), fp64 small objects */
  PF_FP64_I8 = 3 /* fp64 storage and arithmetic; the filter / Rayleigh-Ritz products A Y are
                    formed from EXACT int8 tensor-core products (tcgen05 kind::i8) of S = 7
                    signed 7-bit digit slices of A (per-row power-of-two scale) and of Y (per
                    column), levels combined in fp64 (pf_set_i8_slices; DESIGN.md §4 K1-i8).
                    Everything else is the PF_FP64 path.  Scratch: 7 n_local n + 7 p n bytes. */
} pf_dtype;

typedef enum { PF_OP_PSD = 0, PF_OP_SOFT_THRESHOLD = 1 } pf_op;

typedef enum {
  PF_OK = 0,
  PF_ERR_ARG = 1,       /* invalid argument (null pointer, q or degree out of range, bad op) */
  PF_ERR_DIM = 2,       /* dimension / leading-dimension / alignment mismatch */
  PF_ERR_INTERVAL = 3,  /* b <= a */
  PF_ERR_CUDA = 4,      /* a CUDA runtime call failed (message in pf_last_error) */
  PF_ERR_NOMEM = 5,     /* scratch allocation failed in pf_create */
  PF_ERR_NCCL = 6,      /* NCCL initialisation / collective failed */
  PF_ERR_UNSUPPORTED = 7,
  PF_ERR_BREAKDOWN = 8   /* an iterative step did not converge (pf_rr_ns); nothing was written */
} pf_status;

/* device status word bits (pf_get_device_status) */
#define PF_FLAG_CHOL_SHIFT 0x1u      /* CholeskyQR fell back to the shifted variant (3 passes) */
#define PF_FLAG_NONFINITE 0x2u       /* a non-finite value reached the Gram / H matrix */
#define PF_FLAG_DEGENERATE_INT 0x4u  /* b <= a (e.g. PSD iterate: a >= 0): filter skipped */
#define PF_FLAG_SATURATED 0x8u       /* rank == p after the spectral operator */
#define PF_FLAG_JACOBI_MAXSWEEP 0x10u /* Jacobi hit its sweep limit before the tolerance */
#define PF_FLAG_LANCZOS_BREAK 0x20u  /* Lanczos stopped early (invariant subspace found) */
#define PF_FLAG_NS_FALLBACK 0x40u    /* pf_rr_ns: Newton-Schulz did not converge; Jacobi used */

/* ---------------------------------------------------------------------------- lifetime */
/* Create a single-GPU context for order-n problems with block width p and Chebyshev degree
 * `degree` (1 <= degree <= 64) on the current CUDA device.  Allocates all scratch. */
pf_status pf_create(int64_t n, int32_t p, int32_t degree, pf_dtype dtype, pf_ctx* out);

/* Same, for rank `rank` of `world` processes (one per GPU, current device) sharing the NCCL
 * unique id `nccl_id` (128 bytes from pf_nccl_unique_id on one rank, broadcast by the caller).
 * Row block of this rank: rows [rank*n/world, (rank+1)*n/world).  Collective: every rank must
 * call it.  Per Chebyshev step the context all-gathers Y_j over NCCL; Gram / H matrices and
 * scalar objectives are all-reduced; Jacobi and the spectral operator run replicated.
 * world = 1 is allowed (single-rank communicator, same code path). */
pf_status pf_create_dist(int64_t n, int32_t p, int32_t degree, pf_dtype dtype,
                         const void* nccl_id, int32_t rank, int32_t world, pf_ctx* out);
/* In-process loopback communicator (a test harness for the row-block split on ONE GPU; the
 * exchange semantics of pf_create_dist without NCCL): pf_loop_create makes a hub for `world`
 * ranks (1 <= world <= 16); each rank's context is created with pf_create_loop(..., hub, rank)
 * and driven by its own host thread on its own stream.  Every collective is a host rendezvous
 * of the `world` calls followed by stream-ordered device work: an all-gather waits on each
 * peer's block-ready event and copies the peer slab (cudaMemcpyAsync); an all-reduce sums the
 * peers' buffers in rank order in one kernel (identical bits on every rank).  A rendezvous that
 * waits longer than 300 s (environment PF_LOOP_TIMEOUT_S at pf_loop_create), or a failed peer, fails the call with PF_ERR_NCCL (and every later
 * collective on the hub).  The hub must outlive its contexts; it owns no device memory. */
typedef struct pf_loop_s* pf_loop;
pf_status pf_loop_create(int32_t world, pf_loop* out);
pf_status pf_loop_destroy(pf_loop hub);
pf_status pf_create_loop(int64_t n, int32_t p, int32_t degree, pf_dtype dtype, pf_loop hub,
                         int32_t rank, pf_ctx* out);

/* Writes a fresh NCCL unique id (ncclGetUniqueId) into out[0 .. bytes); bytes >= 128. */
pf_status pf_nccl_unique_id(void* out, int32_t bytes);

pf_status pf_destroy(pf_ctx ctx);
const char* pf_status_string(pf_status s);
const char* pf_last_error(pf_ctx ctx);      /* last CUDA/NCCL error text of this context */
int64_t pf_local_rows(pf_ctx ctx);          /* n_local of this rank */
int64_t pf_row0(pf_ctx ctx);                /* first global row of this rank */

/* Synchronises `stream`, then returns (and clears) the device status word, the number of
 * re-basing steps executed since the last call and the last Lanczos extremes estimate. */
pf_status pf_get_device_status(pf_ctx ctx, pf_stream stream, uint32_t* flags, int32_t* rebases,
                               double* lanczos_lo_hi /* [2], may be NULL */);

/* ---------------------------------------------------------------------------- interval
 * The suppression interval [a, b] lives in device memory (double[2]) so it can be computed
 * on the device.  Every pf_filter call reads it from `interval`.                         */

/* m-step Lanczos with full re-orthogonalisation on the symmetric A (reading R5):
 * writes lo_hi[0] = theta_min - |r_min|, lo_hi[1] = theta_max + |r_max| (device double[2]),
 * and remembers them in the context.  v0: device start vector (n_local entries, any norm), or
 * NULL to start from the Ritz vector of the smallest Ritz value of this context's previous
 * pf_lanczos (lambda_min tracking across refreshes, NEXT-2, reading R29; PF_ERR_ARG if there was
 * none).  1 <= m <= 64.  fp64 dtypes on one GPU (n <= 18944): only the 64 x 64 tiles on and above the
 * diagonal of A are read (A must be symmetric, as the method's iterates are; half the HBM
 * bytes); the environment variable PF_LZ_SYM=0 at pf_create reads all of A. */
pf_status pf_lanczos(pf_ctx ctx, const void* A, int64_t lda, const double* v0, int32_t m,
                     double* lo_hi, pf_stream stream);

/* PSD / all-positive interval: a = lo_hi[0], b = eta * a.  Writes interval[2].
 * If a >= 0 (the iterate is PSD) the interval is the degenerate [a, a]: a pf_filter call
 * on a degenerate interval skips the filter (returns orth(U)) and sets PF_FLAG_DEGENERATE_INT. */
pf_status pf_interval_psd(pf_ctx ctx, const double* lo_hi, double eta, double* interval,
                          pf_stream stream);

/* Two-sided soft-threshold interval [-beta, beta], beta = (1 - eta) * thr (reading R6). */
pf_status pf_interval_soft(pf_ctx ctx, double thr, double eta, double* interval,
                           pf_stream stream);

/* Top-r interval: a = lo_hi[0], b = (1 - eta) theta_r + eta a, theta_r the r-th
 * largest Ritz value of the previous pf_rayleigh_ritz on this context (1 <= r <= p); before any
 * Rayleigh-Ritz the all-positive rule b = eta a is used (R22).  Writes interval[2]. */
pf_status pf_interval_top_r(pf_ctx ctx, const double* lo_hi, int32_t r, double eta,
                            double* interval, pf_stream stream);

/* Chebyshev degree of subsequent pf_filter calls (1 <= degree <= 64).  Scratch does not depend
 * on the degree. */
pf_status pf_set_degree(pf_ctx ctx, int32_t degree);

/* Degree schedule of thm:conv1 (PFPG converges when d_k = Omega(log k / min{l, 1})):
 * sets the degree of subsequent pf_filter calls for iteration k >= 0 to
 * d_k = max(d_0, ceil(c ln(k + 2))), d_0 = the degree given at create (c = 0: d_0), and writes it
 * to *degree (host, may be NULL).  PF_ERR_ARG if c < 0 or d_k > 64. */
pf_status pf_schedule_degree(pf_ctx ctx, double c, int32_t k, int32_t* degree);

/* ---------------------------------------------------------------------------- hot path */
/* U <- orth(rho^q(A) U) with rho(t) = T_d(L(t)), L(t) = (t - (a+b)/2)/((b-a)/2)
 * (eq:cheb P:185-191, eqn:cheb-linear-map P:216-218, eqn:subspace-update P:225-227).
 * Three-term recurrence Y_1 = (A Y_0 - c Y_0)/e, Y_{j+1} = (2/e)(A Y_j - c Y_j) - Y_{j-1};
 * span-exact re-basing when the predicted amplification exceeds rho_max (reading R7);
 * orth = CholeskyQR2 with a shifted CholeskyQR3 fallback ("a single QR" -> any
 * span-exact orthonormalisation).  A: n_local x n (lda), U: n_local x p (ldu), in place.
 * interval: device double[2] {a, b}.  1 <= q <= 10. */
pf_status pf_filter(pf_ctx ctx, const void* A, int64_t lda, void* U, int64_t ldu,
                    const double* interval, int32_t q, double rho_max, pf_stream stream);

/* U <- orth(U) (CholeskyQR2 + shifted fallback).  U: n_local x p. */
pf_status pf_orth(pf_ctx ctx, void* U, int64_t ldu, pf_stream stream);

/* Rayleigh-Ritz (eqn:RR P:269-286): H = U^T A U (symmetrised), H = Y Lambda Y^T by an on-device
 * parallel cyclic Jacobi, theta = Ritz values DESCENDING (device double[p]), V = U Y
 * (n_local x p, ldv).  U must be orthonormal (output of pf_filter / pf_orth). */
pf_status pf_rayleigh_ritz(pf_ctx ctx, const void* A, int64_t lda, const void* U,
                           int64_t ldu, void* V, int64_t ldv, double* theta, pf_stream stream);

/* Spectral operator on the Ritz values: PSD f = max(theta, 0) or soft threshold
 * f = sign(theta) max(|theta| - thr, 0) (shrink).  f: device double[p];
 * rank: device int32 = #{f != 0}. */
pf_status pf_spectral_op(pf_ctx ctx, pf_op op, double thr, const double* theta, double* f,
                         int32_t* rank, pf_stream stream);

/* The rank-p rebuild alone (§8(b)'s optional dense output of the spectral operator): X = V diag(f)
 * V^T, written to X (n_local x n, ldx >= n; every entry).  V: local rows (n_local x p, ldv even,
 * 16-byte aligned), f: device double[p] (e.g. from pf_spectral_op).  fp64 dtypes; DMMA on
 * symmetric tile pairs (the PFPG update kernel with no mask and tau = 0). */
pf_status pf_rebuild(pf_ctx ctx, const double* V, int64_t ldv, const double* f, double* X,
                     int64_t ldx, pf_stream stream);

/* PFPG update for F = 1/2 ||P_Omega(X - M)||_F^2, M = W W^T, R = mu ||.||_* (eq:pfpg1 P:338-341):
 * X = V diag(f) V^T, A_out = X - tau * Omega o (X - M)  (n_local x n, lda_out).
 * omega: packed row-major symmetric bitmask, uint32 words, bit (j & 31) of word [i][j >> 5],
 * row pitch ldo words (>= ceil(n/32)), local rows.  W: n x r FULL (all rows), ldw >= r,
 * 0 <= r <= 64 (the low-rank factor of M is staged in shared memory next to the V panels; the
 * BASELINE configs use r = 10 / 50).  mu >= 0.  obj: device double[2] = {h(X), 1/2 ||P_Omega(X - M)||_F^2} with the
 * PFPG objective h(X) = 1/2 ||P_Omega(X - M)||_F^2 + mu sum_i |f_i| (= mu ||X||_* for
 * orthonormal V), summed over all ranks. */
pf_status pf_prox_step(pf_ctx ctx, const double* V, int64_t ldv, const double* f, double tau,
                       double mu, const uint32_t* omega, int64_t ldo, const double* W,
                       int64_t ldw, int32_t r, double* A_out, int64_t lda_out, double* obj,
                       pf_stream stream);

/* PFAM update for the max-cut SDP min <C,X> s.t. diag(X) = 1, X PSD, C = -L/4 (eq:PFAM1 P:389
 * with the prox sign corrected, reading R1): W = V diag(f) V^T,
 * Z <- prox_tG(2W - Z) - W + Z = offdiag(W - tC) + Diag(1 - W_ii + Z_ii), in place.
 * adj: packed adjacency bitmask (as omega above, local rows, no self loops); deg: device
 * double[n] FULL degree vector.  obj: device double[2] = {<C, W>, ||Z_new - Z_old||_F}.
 * Z must be symmetric (it is the DRS iterate on S^n): with world = 1 only its upper triangle
 * is read and the lower triangle is written as the exact mirror of the upper one. */
pf_status pf_admm_step(pf_ctx ctx, const double* V, int64_t ldv, const double* f, double t,
                       const uint32_t* adj, int64_t ldadj, const double* deg, double* Z,
                       int64_t ldz, double* obj, pf_stream stream);

/* PFAM update in matrix form (with pf_rr_ns, reading R30): W = Q F Q^T, F p x p row-major fp64
 * (device, symmetric), Q the local rows of the orthonormal block (n_local x p, ldq); otherwise as
 * pf_admm_step (same Z contract, obj, fused digit output on one GPU).  With the PSD projection
 * of a positive definite H = Q^T A Q, F = H (pf_rr_ns's PD test), so no eigendecomposition is
 * needed at all. */
pf_status pf_admm_step_f(pf_ctx ctx, const double* Q, int64_t ldq, const double* F, double t,
                         const uint32_t* adj, int64_t ldadj, const double* deg, double* Z,
                         int64_t ldz, double* obj, pf_stream stream);

/* Nearest correlation estimation, dual gradient step (eqn:NCE-dual and
 * eqn:NCE-gradient), PF_FP64 contexts: with Pi_+(B) ~ V diag(f) V^T for the iterate
 * B = G + Diag(x) (f = max(theta, 0) from pf_spectral_op PF_OP_PSD):
 *   grad_i = diag(V diag(f) V^T)_i - 1,  x <- x - tau grad,  B_ii <- G_ii + x_i.
 * V: local rows (n_local x p, ldv); gdiag: device double[n] (full diag(G)); x_in / x_out:
 * device double[n_local] (this rank's slice; may alias); B: local rows (n_local x n, ldb) -- only its
 * diagonal entries (i, row0 + i) are written.  obj: device double[2] = {F(x_old),
 * ||grad F(x_old)||}, F(x) = 1/2 sum f_i^2 - 1^T x.  tau > 0 (the paper uses tau = 1). */
pf_status pf_nce_step(pf_ctx ctx, const double* V, int64_t ldv, const double* f, double tau,
                      const double* gdiag, const double* x_in, double* x_out, double* B,
                      int64_t ldb, double* obj, pf_stream stream);

/* Regularized extrapolation of the iterates (paper §4.3),
 * PF_FP64 contexts, for the NCE dual variable: hist[0..l+1] are l+2 device vectors (this rank's
 * n_local entries, OLDEST FIRST; host array of device pointers), U = [h_1 - h_0, ..., h_{l+1} - h_l],
 * c = (U^T U + lam I)^{-1} 1 / (1^T (U^T U + lam I)^{-1} 1), lam = lam_rel ||U^T U||_F (U^T U summed
 * over all ranks), x_out = sum_{i<=l} c_i h_i (may alias any h_i), B_ii <- G_ii + x_out_i.
 * coef: device double[l+1] or NULL.  0 <= l <= 7, lam_rel > 0 (the SPEC default is l = 5,
 * lam_rel = 1e-8; reading R21). */
pf_status pf_extrapolate(pf_ctx ctx, const double* const* hist, int32_t l, double lam_rel,
                         const double* gdiag, double* x_out, double* B, int64_t ldb, double* coef,
                         pf_stream stream);

/* ---------------------------------------------------------------------------- measurement */
/* Enable (1) / disable (0) per-launch CUDA-event timing of the Chebyshev-step GEMM (the
 * dominant kernel): each launch inside pf_filter / pf_rayleigh_ritz is bracketed by events on
 * its own stream.  Resets the accumulated record.  Up to 4096 launches are recorded. */
pf_status pf_profile(pf_ctx ctx, int32_t enable);
/* Synchronises `stream`; returns the summed GEMM time (ms) and the number of timed launches
 * since pf_profile, then clears the record.  PF_ERR_ARG if launches were dropped. */
pf_status pf_profile_read(pf_ctx ctx, pf_stream stream, double* gemm_ms, int64_t* gemm_launches);
/* Synchronises `stream`; returns the summed time (ms) and count of the PFAM updates
 * (pf_admm_step / pf_admm_step_f: row bounds, splits and the update kernel, bracketed by events
 * on their stream) timed since pf_profile, then clears that record (up to 512 updates). */
pf_status pf_profile_read_update(pf_ctx ctx, pf_stream stream, double* ms, int64_t* launches);
/* Overlapped all-gather (PF_TF32, world > 1; environment PF_OVERLAP=0 at create turns it off):
 * the timeline of the last overlapped GEMM step recorded while pf_profile is on.  Synchronises
 * `stream`; writes 3 world values (ms from the step start): ms[s] = arrival of the s-th slab in
 * consumption order (rank, rank - 1, ...), ms[world + s] / ms[2 world + s] = begin / end of its
 * slab GEMM.  *count = 0 when no overlapped step was recorded.  cap >= 3 world. */
pf_status pf_overlap_timeline(pf_ctx ctx, pf_stream stream, double* ms, int32_t cap,
                              int32_t* count);
/* Process-wide number of CUDA kernels launched by this library so far. */
long long pf_kernel_launches(void);
/* Synchronises `stream`; diag[0] = Jacobi sweeps of the last Rayleigh-Ritz solve,
 * diag[1] = Lanczos steps of the last refresh, diag[2] = the relative gap of eqn:relative-gap
 * (NEXT-2 diagnostic) G = min over the Ritz values theta_i outside the damped
 * interval [a, b] of the last pf_filter of |theta_i - (a + b)/2| / ((b - a)/2) - 1, with the
 * Ritz values standing in for the eigenvalues (+inf when none lies outside), diag[3] = the
 * eta_k estimate of eqn:etak (reading R28) for the wanted values of the last filter:
 * (1 / T_d(1 + G))^q, the bound that holds when a guard Ritz value lies inside [a, b]; NaN when
 * every Ritz value lies beyond [a, b] (saturated block) or no pf_filter preceded, 0 when none
 * does. */
pf_status pf_diagnostics(pf_ctx ctx, pf_stream stream, double* diag /* [4] */);

/* Workload helper (not the method): A <- A + E (config 1 noise, BASELINE configs[0]).
 * PF_FP64 contexts only. */
pf_status pf_perturb(pf_ctx ctx, double* A, int64_t lda, const double* E, int64_t lde,
                     pf_stream stream);

/* Workload helper (not the method), PF_TF32 contexts: config-5 noise (BASELINE configs[4])
 * A_ij <- fl32(A_ij + fl32((noise * g) * s)), s = 1 on the diagonal, 1/sqrt(2) off it, and
 * g = Box-Muller N(0,1) from the counter-based hash of (seed, k, min(i,j), max(i,j)) --
 * the same function as pfinputs.generators.hash_gauss.  Local rows of A (n_local x n, fp32). */
pf_status pf_perturb_hash(pf_ctx ctx, float* A, int64_t lda, uint64_t seed, int32_t k,
                          double noise, pf_stream stream);

/* TF32 MMA passes of every filter / Rayleigh-Ritz GEMM (PF_TF32 contexts): 3 = 3xTF32
 * (A_hi B_hi + A_lo B_hi + A_hi B_lo, error ~ fp32; the default), 2 = A_hi B_hi + A_lo B_hi (exact
 * operator, iterate rounded to tf32), 1 = plain TF32 (operator rounded to 10 mantissa bits).
 * PF_ERR_ARG outside 1..3. */
pf_status pf_set_tf32_passes(pf_ctx ctx, int32_t passes);

/* Precision schedule of pf_filter (PF_TF32 contexts): the first degree - exact_tail Chebyshev
 * steps run at early_passes (1..3), the last exact_tail steps and the Rayleigh-Ritz product in
 * 3xTF32.  Errors injected by the cheaper early steps are damped by the exact tail steps
 * (reading R18). */
pf_status pf_set_tf32_schedule(pf_ctx ctx, int32_t early_passes, int32_t exact_tail);

/* PF_FP64_I8 contexts: digit slices per operand, S in {6, 7} (default 7: operator error
 * < 2^-48 of the row / column scales), or 0 to run the fp64 DMMA GEMM of PF_FP64 instead (same
 * context, for comparisons).  PF_ERR_ARG otherwise, PF_ERR_UNSUPPORTED for other dtypes. */
pf_status pf_set_i8_slices(pf_ctx ctx, int32_t slices);

/* PF_FP64_I8 precision schedule of pf_filter (reading R25): the first degree -
 * exact_tail Chebyshev steps multiply only the early_slices (4..S) most significant digit slices
 * (early_slices (early_slices + 1) / 2 products instead of S (S + 1) / 2), the last exact_tail
 * steps and the Rayleigh-Ritz product use all S.  The early steps' error off the wanted span is
 * damped by the later steps.  Default: early_slices = S (no schedule). */
pf_status pf_set_i8_schedule(pf_ctx ctx, int32_t early_slices, int32_t exact_tail);

/* PF_FP64_I8: pf_filter splits A into digit slices, except right after pf_admm_step on one GPU,
 * whose update writes the slices of Z_new itself (row scales from a bound on |Z_new|, DESIGN.md
 * §4 "fused digits"; disabled by the environment variable PF_FUSE_DIGITS=0 at pf_create);
 * pf_rayleigh_ritz and pf_matmul reuse the slices of the last split of the same A (pointer, lda)
 * unless a libpf call wrote an iterate since (pf_prox_step, pf_nce_step, pf_extrapolate,
 * pf_perturb; pf_admm_step leaves its own Z_new's slices valid).  A caller that writes A by other
 * means between libpf calls calls pf_invalidate first.  No-op for other dtypes. */
pf_status pf_invalidate(pf_ctx ctx);

/* Upper-block storage of the PFAM iterate (DESIGN.md §4 "K7-i8, upper-block storage"): with
 * upper = 1, pf_admm_step / pf_admm_step_f on this context write Z_new only in the rows' 128 x 128
 * diagonal blocks and to their right (entries (i, j) with j >= 128 floor(i / 128)), not the exact
 * mirror below them -- Z is symmetric, and every libpf reader of the iterate on this path reads
 * only that region: pf_filter / pf_rayleigh_ritz / pf_rr_ns take the update's digit slices
 * (mirror slices included), pf_lanczos reads the upper 64 x 64 tiles, the next update the upper
 * tiles.  A fresh digit split of such an iterate (it would read the stale lower part) fails with
 * PF_ERR_UNSUPPORTED until pf_invalidate (the caller declares the full matrix written) or upper
 * = 0.  Applies when the int8-digit update runs (one GPU, PF_FP64_I8, p = 64, S = 7, fused digits,
 * PF_K7I8 not 0) and pf_lanczos uses the symmetric tile GEMV (one GPU, n <= 18944); otherwise
 * PF_ERR_UNSUPPORTED.  upper = 0 (the default) restores full storage. */
pf_status pf_set_z_upper(pf_ctx ctx, int32_t upper);

/* out = A Y with the context's filter GEMM (fp64 dtypes): A local rows (n_local x n, lda as for
 * pf_filter), Y the local rows of an n x p block (n_local x p, ldy >= p; gathered internally when
 * distributed), out n_local x p (ldo >= p).  The kernel of every Chebyshev step, exposed for
 * measurement and tests.  PF_ERR_UNSUPPORTED for PF_TF32. */
pf_status pf_matmul(pf_ctx ctx, const double* A, int64_t lda, const double* Y, int64_t ldy,
                    double* out, int64_t ldo, pf_stream stream);

/* Rayleigh-Ritz and the spectral operator without an eigendecomposition (SURVEY NEXT-4,
 * DESIGN.md reading R26): H = U^T A U as in pf_rayleigh_ritz (same layouts and dtypes), then
 * F = f(H) (p x p row-major fp64, device) through Newton-Schulz matrix sign iterations
 * (PSD: f(H) = (H + H sign(H)) / 2; soft threshold thr: f(H) = H + ((H - thr I) sign(H - thr I)
 * - (H + thr I) sign(H + thr I)) / 2) and *rank = #{f != 0} (device int) from traces, so
 * X = U F U^T.  PSD with p <= 128: a Cholesky test first -- if H is positive definite,
 * P_+(H) = H exactly, so F = H and rank = p without sign iterations (reading R30).  The whole
 * iteration runs in one cooperative kernel (hand-written fp64 DMMA
 * products, device-side convergence test ||X^2 - I||_F <= 1e-12 sqrt(p), at most 100 steps): no
 * host synchronisation, capturable in a CUDA graph.  If a sign does not converge (an eigenvalue
 * at the threshold) the same call falls back on the device to the Jacobi eigensolver
 * (F = Y diag(f(theta)) Y^T) and sets PF_FLAG_NS_FALLBACK.  iters: DEVICE int (may be NULL) =
 * sign iterations used, -1 after a fallback.  Scratch (7 p^2 doubles) is allocated on the first
 * call of a context. */
pf_status pf_rr_ns(pf_ctx ctx, const void* A, int64_t lda, const void* U, int64_t ldu, pf_op op,
                   double thr, double* F, int32_t* rank, int32_t* iters, pf_stream stream);

/* ---------------------------------------------------------------- PFSVT (NEXT-3, paper §5.2)
 * Polynomial-filtered SVT for matrix completion (eqn:svt P:1098-1104, Example eg:MC): the dual
 * iterate Y = A*(x) is an n x n sparse matrix with the values x on the sampled set Omega
 * (|Omega| = nnz), given in compressed-row form: ptr[n + 1], idx[nnz] (int32, device), values
 * val[nnz] in the same order.  The CSC view of Omega (column pointer, row indices, and
 * perm: CSC position -> CSR position) addresses the SAME values for Y^T.  fp64 contexts only
 * (PF_FP64 / PF_FP64_I8), one GPU (PF_ERR_UNSUPPORTED when distributed); blocks are n x p
 * row-major; p in {16, 32, 64, 128}. */

/* out = s1 * (S X) + s2 * Ycur + s3 * Yprev with S = (ptr, idx, val[vperm[e] or e]) -- one
 * Chebyshev step of the filter on Y^T Y is pf_spmm(CSR, X = Y_j) into a temporary T followed by
 * pf_spmm(CSC with perm, X = T, coefficients of eq:cheb).  Deterministic (each row's nonzeros
 * in storage order).  Ycur / Yprev may be NULL when their coefficient is 0. */
pf_status pf_spmm(pf_ctx ctx, const int32_t* ptr, const int32_t* idx, const double* val,
                  const int32_t* vperm, const double* X, int64_t ldx, double s1, double s2,
                  double s3, const double* Ycur, int64_t ldc, const double* Yprev, int64_t ldp,
                  double* out, int64_t ldo, pf_stream stream);

/* SVT's kick (reading R24): x = k0 delta b on the nnz sampled entries, k0 = ceil(mu / (delta
 * norm2)) with norm2 = ||P_Omega(M)||_2 (host scalar, computed by the problem's generator).
 * b, x: device double[nnz]. */
pf_status pf_svt_kick(pf_ctx ctx, const double* b, int64_t nnz, double mu, double delta,
                      double norm2, double* x, pf_stream stream);

/* The PFSVT filter ("subspace extraction from A^T A"; reading R24): Q <- orth(
 * T_d(L(Y^T Y)) Q) with the context's degree d, Y = A*(x) the sparse dual iterate (CSR ptr / idx
 * and its CSC view cptr / cidx / perm addressing the same values val = x, as for pf_spmm),
 * damped interval [0, (1 - eta) mu^2] of Y^T Y, L(t) = (t - c)/e (eqn:cheb-linear-map), the
 * three-term recurrence eq:cheb with each product Y^T (Y Y_j) as two sparse products, then
 * CholeskyQR2.  Q: n x p row-major (ldq >= p), in place.  mu > 0, 0 <= eta < 1. */
pf_status pf_svt_filter(pf_ctx ctx, const int32_t* ptr, const int32_t* idx, const int32_t* cptr,
                        const int32_t* cidx, const int32_t* perm, const double* val, double* Q,
                        int64_t ldq, double mu, double eta, pf_stream stream);

/* Singular triplets of Y on span(Q) (Q orthonormal, n x p): B = Y Q, B^T B = W diag(lambda) W^T
 * by Jacobi (descending), sigma = sqrt(max(lambda, 0)) (device, p), V = Q W, U = B W / sigma
 * (columns with sigma = 0 are zero), the shrink s = (sigma - mu)_+ (device, p) and
 * *svp = #{s > 0} (device int). */
pf_status pf_svt_ritz(pf_ctx ctx, const int32_t* ptr, const int32_t* idx, const double* val,
                      const double* Q, int64_t ldq, double mu, double* U, int64_t ldu, double* V,
                      int64_t ldv, double* sigma, double* s, int32_t* svp, pf_stream stream);

/* SVT dual step on Omega (CSR order): w_e = sum_l U_{i_e l} s_l V_{j_e l} (the sampled entries of
 * W = U diag(s) V^T), x_e <- x_e + delta (b_e - w_e), *rss = sum_e (b_e - w_e)^2 (device double,
 * fixed-order reduction). */
pf_status pf_svt_update(pf_ctx ctx, const int32_t* ptr, const int32_t* idx, const double* b,
                        double* x, const double* U, int64_t ldu, const double* V, int64_t ldv,
                        const double* s, double delta, double* rss, pf_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* PF_H_ */
