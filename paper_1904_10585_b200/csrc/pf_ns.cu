// pf_ns.cu -- the spectral operator of Rayleigh-Ritz without an eigendecomposition (SURVEY §8(f)
// NEXT-4 "Newton-Schulz f(H) for p = 512"; reading R26):
//
//     X = V f(Lambda) V^T = Q f(H) Q^T,   H = Q^T A Q  (eqn:RR P:269-286 with V = Q Y_eig)
//
// so the update only needs F = f(H) (p x p).  Both spectral operators are polynomials in matrix
// sign functions:
//     PSD projection:          f(H) = (H + H sign(H)) / 2
//     soft threshold theta:  f(H) = H + ((H - theta I) S+ - (H + theta I) S-) / 2,
//                                          S+ = sign(H - theta I), S- = sign(H + theta I)
// and rank = #{f != 0} = tr(I + S+)/2 + tr(I - S-)/2 (PSD: tr(I + S)/2).  sign(M) by the
// Newton-Schulz iteration X <- X (3 I - X^2) / 2 from X_0 = M / ||M||_inf (all eigenvalues in
// [-1, 1]), stopped when ||X^2 - I||_F <= tol.
//
// B200 design: ONE cooperative kernel runs the whole iteration on the device (no host sync, so
// a Rayleigh-Ritz step can be captured in a CUDA graph).  Every iterate is a polynomial in the
// symmetric M, so it is kept EXACTLY symmetric: each product is formed on the upper 32 x 32 tiles
// only (fp64 DMMA, both operands row panels: C = A B^T) and mirrored, which also halves the work.
// For the soft threshold the two signs iterate side by side (two halves of the grid).  Per step:
// T = X X^T with the residual ||T - I||_F^2 as per-CTA partials, grid barrier, every CTA sums the
// partials in the same order (a uniform convergence decision), X <- X (3 I - T) / 2, barrier.
// A sign that has not converged after max_it steps sets the fail flag; the caller then runs the
// cooperative Jacobi eigensolver on the same H (a conditional launch: no host decision).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "../../include/pf.h"
#include "pf_kernels.cuh"

namespace pf {
namespace cg = cooperative_groups;

constexpr int kNsT = 32;         // tile edge
constexpr int kNsK = 32;         // K chunk (doubles)
constexpr int kNsLd = kNsK + 4;  // smem row pitch
constexpr int kNsThreads = 128;  // 4 warps, warp tile 16 x 16

struct NsWork {
  int p = 0, tt = 0, nup = 0;  // tiles per dimension, upper tiles (I <= J)
  double* buf = nullptr;       // per sign: 3 rotating p x p buffers; shared: Hs (p x p)
  double* part = nullptr;      // per CTA residual partials
  int* ctrl = nullptr;         // [0] fail, [1] iterations, [2] PD shortcut taken
  unsigned long long* nrm = nullptr;  // per sign ||M||_inf bits
};

struct NsArgs {
  const double* H;
  int p, tt, nup, nsign, max_it;
  double shift[2];  // M_s = Hs - shift[s] I
  double tol;
  int soft;
  double* Hs;
  double* X[2][3];  // per sign: three rotating p x p buffers
  double* F;
  int* rank;
  double* part;
  int* ctrl;
  unsigned long long* nrm;
  int* iters_out;  // device, may be NULL
  DevState* state;
  const int* skip;  // device: the PD test already wrote F (PSD of a positive definite H)
};

__device__ __forceinline__ void ns_cp16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}

// upper tile e (0 <= e < tt (tt + 1) / 2) -> (I, J), I <= J, row-major over the upper triangle
__device__ __forceinline__ void ns_tile(int e, int tt, int& I, int& J) {
  int i = 0;
  while ((i + 1) * tt - (i + 1) * i / 2 <= e) ++i;
  I = i;
  J = i + (e - (i * tt - i * (i - 1) / 2));
}

// acc (warp tile 16 x 16 at (wr, wc) inside the 32 x 32 tile) = A[rows I] B[rows J]^T over K = p
// (row-major p x p operands, rows / columns >= p read as 0)
__device__ __forceinline__ void ns_tile_mma(const double* __restrict__ A, const double* __restrict__ B,
                                            int p, int I, int J, double* sm, double (&acc)[2][4]) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int wr = (warp & 1) * 16, wc = (warp >> 1) * 16;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[nt][k] = 0.0;
  const int nchunk = (p + kNsK - 1) / kNsK;
  auto stage = [&](int c, int buf) {
    double* sa = sm + buf * 2 * kNsT * kNsLd;
    double* sb = sa + kNsT * kNsLd;
    const int k0 = c * kNsK;
    // 32 rows x 32 doubles per operand = 512 16-byte pieces, 4 per thread and operand
    for (int e = tid; e < kNsT * (kNsK / 2); e += kNsThreads) {
      const int r = e / (kNsK / 2), k = (e % (kNsK / 2)) * 2;
      const int ra = I * kNsT + r, rb = J * kNsT + r, kk = k0 + k;
      if (ra < p && kk < p) ns_cp16(sa + r * kNsLd + k, A + (size_t)ra * p + kk);
      else *reinterpret_cast<double2*>(sa + r * kNsLd + k) = make_double2(0.0, 0.0);
      if (rb < p && kk < p) ns_cp16(sb + r * kNsLd + k, B + (size_t)rb * p + kk);
      else *reinterpret_cast<double2*>(sb + r * kNsLd + k) = make_double2(0.0, 0.0);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  stage(0, 0);
  for (int c = 0; c < nchunk; ++c) {
    if (c + 1 < nchunk) {
      stage(c + 1, (c + 1) & 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const double* sa = sm + (c & 1) * 2 * kNsT * kNsLd + (wr + g) * kNsLd + t;
    const double* sb = sm + (c & 1) * 2 * kNsT * kNsLd + kNsT * kNsLd + (wc + g) * kNsLd + t;
#pragma unroll
    for (int ks = 0; ks < kNsK / 4; ++ks) {
      const double a0 = sa[ks * 4], a1 = sa[8 * kNsLd + ks * 4];
      const double b0 = sb[ks * 4], b1 = sb[8 * kNsLd + ks * 4];
      dmma16884(acc[0], a0, a1, b0);
      dmma16884(acc[1], a0, a1, b1);
    }
    __syncthreads();  // the buffer is refilled two chunks later
  }
}

// store the warp tile of C (tile (I, J), upper) and its mirror; value(i, j, acc) transforms
template <typename Fn>
__device__ __forceinline__ void ns_store(double* __restrict__ C, int p, int I, int J,
                                         const double (&acc)[2][4], Fn value) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int wr = (warp & 1) * 16, wc = (warp >> 1) * 16;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int i = I * kNsT + wr + g + 8 * h, j = J * kNsT + wc + nt * 8 + 2 * t + c;
        if (i < p && j < p && (I < J || i <= j)) {
          const double v = value(i, j, acc[nt][2 * h + c]);
          C[(size_t)i * p + j] = v;
          C[(size_t)j * p + i] = v;
        }
      }
}

__global__ void __launch_bounds__(kNsThreads) ns_kernel(const NsArgs a) {
  if (a.skip && *a.skip) return;  // uniform over the grid
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[32];
  const int p = a.p, tid = threadIdx.x;
  const int sg = blockIdx.x / a.nup, e = blockIdx.x % a.nup;
  int I, J;
  ns_tile(e, a.tt, I, J);
  const int gtid = blockIdx.x * kNsThreads + tid, gthreads = gridDim.x * kNsThreads;
  const int sthreads = a.nup * kNsThreads, stid = e * kNsThreads + tid;  // within the sign group
  // ---- Hs = (H + H^T) / 2 and ||M_s||_inf per sign
  if (gtid == 0) a.ctrl[0] = 0;
  for (int x = gtid; x < p * p; x += gthreads) {
    const int i = x / p, j = x - i * p;
    a.Hs[x] = 0.5 * (a.H[(size_t)i * p + j] + a.H[(size_t)j * p + i]);
  }
  grid.sync();
  for (int r = stid >> 5; r < p; r += sthreads >> 5) {  // a warp per row
    double s = 0.0;
    for (int c = tid & 31; c < p; c += 32) s += fabs(a.Hs[(size_t)r * p + c] - (r == c ? a.shift[sg] : 0.0));
    s = warp_sum(s);
    if ((tid & 31) == 0) atomicMax(a.nrm + sg, (unsigned long long)__double_as_longlong(s));
  }
  grid.sync();
  {
    const double nrm = __longlong_as_double((long long)a.nrm[sg]);
    const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
    for (int x = stid; x < p * p; x += sthreads) {
      const int i = x / p, j = x - i * p;
      a.X[sg][0][x] = (a.Hs[x] - (i == j ? a.shift[sg] : 0.0)) * inv;
    }
  }
  grid.sync();
  // ---- Newton-Schulz iterations.  Three buffers per sign rotate: X (current), T' = 3 I - X^2,
  // the next X; every buffer is rewritten only after two grid barriers since its last reader.
  int cur[2] = {0, 0};
  bool conv[2] = {a.nsign < 1, a.nsign < 2};
  int its[2] = {0, 0};
  double acc[2][4];
  for (int it = 0; it < a.max_it; ++it) {
    if (!conv[sg]) {  // T = X X^T (= X^2: X is symmetric); T' = 3 I - T
      const double* X = a.X[sg][cur[sg]];
      double* T = a.X[sg][(cur[sg] + 1) % 3];
      ns_tile_mma(X, X, p, I, J, sm, acc);
      double r = 0.0;
      ns_store(T, p, I, J, acc, [&](int i, int j, double v) {
        const double d = v - (i == j ? 1.0 : 0.0);
        r += (i == j ? 1.0 : 2.0) * d * d;
        return (i == j ? 3.0 : 0.0) - v;
      });
      r = block_sum(r, red);
      if (tid == 0) a.part[blockIdx.x] = r;
    }
    grid.sync();
    // uniform convergence decision: every CTA sums each group's partials in the same order
    bool all = true;
    for (int s = 0; s < a.nsign; ++s) {
      if (!conv[s]) {
        double res = 0.0;
        for (int q = 0; q < a.nup; ++q) res += __ldcg(a.part + s * a.nup + q);
        if (sqrt(res) <= a.tol) {
          conv[s] = true;  // the current X is the sign
          its[s] = it;
        }
      }
      all = all && conv[s];
    }
    if (all) break;
    if (!conv[sg])  // X <- X T' / 2 (T' symmetric: row panels of both)
      ns_tile_mma(a.X[sg][cur[sg]], a.X[sg][(cur[sg] + 1) % 3], p, I, J, sm, acc),
          ns_store(a.X[sg][(cur[sg] + 2) % 3], p, I, J, acc, [](int, int, double v) { return 0.5 * v; });
    grid.sync();
    for (int s = 0; s < a.nsign; ++s)
      if (!conv[s]) cur[s] = (cur[s] + 2) % 3;
  }
  bool ok = true;
  for (int s = 0; s < a.nsign; ++s) ok = ok && conv[s];
  if (!ok) {
    if (gtid == 0) {
      a.ctrl[0] = 1;  // fall back to the Jacobi eigensolver (conditional launches follow)
      a.ctrl[1] = a.max_it * a.nsign;
      if (a.iters_out) *a.iters_out = -1;
      atomicOr(&a.state->flags, PF_FLAG_NS_FALLBACK);
    }
    return;
  }
  // ---- F: G_s = M_s S_s = Hs S_s - shift_s S_s (upper tiles + mirror; symmetric in exact
  // arithmetic), into the free T' buffer; then F elementwise (exactly symmetric)
  double* G[2] = {a.X[0][(cur[0] + 1) % 3], a.X[1][(cur[1] + 1) % 3]};
  {
    const double* S = a.X[sg][cur[sg]];
    ns_tile_mma(a.Hs, S, p, I, J, sm, acc);
    const double sh = a.shift[sg];
    ns_store(G[sg], p, I, J, acc,
             [&](int i, int j, double v) { return v - sh * S[(size_t)i * p + j]; });
  }
  grid.sync();
  for (int x = gtid; x < p * p; x += gthreads) {
    const double h = a.Hs[x];
    a.F[x] = a.soft ? h + 0.5 * (G[0][x] - G[1][x]) : 0.5 * (h + G[0][x]);
  }
  if (blockIdx.x == 0) {
    double tr = 0.0;
    for (int i = tid; i < p; i += kNsThreads) {
      const double sp = a.X[0][cur[0]][(size_t)i * p + i];
      tr += a.soft ? 0.5 * (1.0 + sp) + 0.5 * (1.0 - a.X[1][cur[1]][(size_t)i * p + i])
                   : 0.5 * (1.0 + sp);
    }
    tr = block_sum(tr, red);
    if (tid == 0) {
      *a.rank = (int)llrint(tr);
      a.ctrl[1] = its[0] + its[1];
      if (a.iters_out) *a.iters_out = its[0] + its[1];
    }
  }
}

NsWork* ns_create(int p) {
  NsWork* w = new NsWork();
  w->p = p;
  w->tt = (p + kNsT - 1) / kNsT;
  w->nup = w->tt * (w->tt + 1) / 2;
  const size_t mb = (size_t)p * p * 8;
  bool ok = cudaMalloc(&w->buf, 7 * mb) == cudaSuccess &&
            cudaMalloc(&w->part, (size_t)2 * w->nup * 8) == cudaSuccess &&
            cudaMalloc(&w->ctrl, 16) == cudaSuccess && cudaMalloc(&w->nrm, 16) == cudaSuccess &&
            cudaMemset(w->ctrl, 0, 16) == cudaSuccess;
  // (ctrl[2] is written by pd_test_kernel before every PSD call; 0 otherwise)
  if (!ok) {
    ns_destroy(w);
    return nullptr;
  }
  return w;
}

void ns_destroy(NsWork* w) {
  if (!w) return;
  for (void* q : {(void*)w->buf, (void*)w->part, (void*)w->ctrl, (void*)w->nrm})
    if (q) cudaFree(q);
  delete w;
}

const int* ns_fail_flag(const NsWork* w) { return w->ctrl; }

// PD test for the PSD projection (reading R30): H (symmetrised) positive definite <=> its Cholesky
// factorisation runs through with positive pivots; then P_+(H) = H exactly (every eigenvalue is
// kept), F = H, rank = p and the sign iterations are skipped.  Right-looking, one CTA, one barrier
// per column (p <= 128); pivots must exceed 1e-13 of their original diagonal (an H indefinite
// only by rounding takes the Newton-Schulz path).
__global__ void __launch_bounds__(512) pd_test_kernel(const double* __restrict__ H, int p,
                                                    double* __restrict__ F, int* rank, int* ctrl,
                                                    int* iters_out, DevState* state) {
  extern __shared__ double M[];  // p x (p + 1)
  __shared__ int s_fail;
  __shared__ double s_inf, s_fro;
  const int P1 = p + 1, tid = threadIdx.x, nt = blockDim.x, tx = tid & 31, ty = tid >> 5;
  const int nty = nt >> 5;
  for (int e = tid; e < p * p; e += nt) {
    const int i = e / p, j = e - i * p;
    const double v = 0.5 * (H[(size_t)i * p + j] + H[(size_t)j * p + i]);
    F[e] = v;
    if (j <= i) M[i * P1 + j] = v;
    if (i == j) M[i * P1 + p] = v;  // original diagonal
  }
  if (tid == 0) {
    s_fail = 0;
    s_inf = 0.0;
    s_fro = 0.0;
  }
  __syncthreads();
  // ||H||_inf and ||H||_F: a bound on the spread max |theta| of the Ritz values for the next
  // re-base plan (the PD path computes no Ritz values)
  for (int i = tid; i < p; i += nt) {  // row i of the symmetric H from the lower triangle in M
    double r = 0.0, f = 0.0;
    for (int k = 0; k < p; ++k) {
      const double v = k <= i ? M[i * P1 + k] : M[k * P1 + i];
      r += fabs(v);
      f += v * v;
    }
    atomicMax(reinterpret_cast<unsigned long long*>(&s_inf), (unsigned long long)__double_as_longlong(r));
    atomicAdd(&s_fro, f);
  }
  __syncthreads();
  for (int j = 0; j < p; ++j) {
    const double d = M[j * P1 + j];
    if (!(d > 1e-13 * M[j * P1 + p])) {  // uniform
      if (tid == 0) s_fail = 1;
      break;
    }
    const double inv_d = 1.0 / d;
    for (int i = j + 1 + ty; i < p; i += nty) {
      const double lij = M[i * P1 + j] * inv_d;
      for (int k = j + 1 + tx; k <= i; k += 32) M[i * P1 + k] -= lij * M[k * P1 + j];
    }
    __syncthreads();
  }
  __syncthreads();
  if (tid == 0) {
    const int pd = !s_fail;
    ctrl[2] = pd;
    ctrl[0] = 0;
    if (pd) {
      *rank = p;
      ctrl[1] = 0;
      if (iters_out) *iters_out = 0;
      // theta_max <= min(||H||_inf, ||H||_F) (all Ritz values are positive): the plan's spread
      state->theta[0] = fmin(s_inf, sqrt(s_fro));
      for (int k = 1; k < p; ++k) state->theta[k] = 0.0;
      state->have_theta = 1;
    }
  }
}

static cudaError_t pd_shortcut(NsWork* w, const double* H, double* F, int* rank, int* iters,
                               DevState* state, cudaStream_t st) {
  const int p = w->p;
  if (p > 128) return cudaMemsetAsync(w->ctrl + 2, 0, sizeof(int), st);
  const size_t smem = (size_t)p * (p + 1) * 8;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(pd_test_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  count_launch();
  pd_test_kernel<<<1, 512, smem, st>>>(H, p, F, rank, w->ctrl, iters, state);
  return cudaGetLastError();
}

cudaError_t ns_spectral(NsWork* w, const double* H, int op_soft, double thr, double* F, int* rank,
                        int* iters_dev, DevState* state, cudaStream_t st) {
  const int p = w->p;
  static int max_it = -1;
  if (max_it < 0) {
    const char* e = getenv("PF_NS_MAXIT");  // development / test knob
    max_it = e ? atoi(e) : 100;
  }
  NsArgs a{};
  a.H = H;
  a.p = p;
  a.tt = w->tt;
  a.nup = w->nup;
  a.nsign = op_soft ? 2 : 1;
  a.max_it = max_it;
  a.shift[0] = op_soft ? thr : 0.0;
  a.shift[1] = -thr;
  a.tol = 1e-12 * sqrt((double)p);
  a.soft = op_soft;
  const size_t pp = (size_t)p * p;
  a.Hs = w->buf + 6 * pp;
  for (int s = 0; s < 2; ++s)
    for (int b = 0; b < 3; ++b) a.X[s][b] = w->buf + (3 * s + b) * pp;
  a.F = F;
  a.rank = rank;
  a.part = w->part;
  a.ctrl = w->ctrl;
  a.nrm = w->nrm;
  a.iters_out = iters_dev;
  a.state = state;
  a.skip = w->ctrl + 2;
  cudaError_t e = cudaMemsetAsync(w->nrm, 0, 16, st);
  if (e != cudaSuccess) return e;
  if (!op_soft) {  // PSD: if H is positive definite, P_+(H) = H (no sign iterations)
    e = pd_shortcut(w, H, F, rank, iters_dev, state, st);
    if (e != cudaSuccess) return e;
  } else {
    e = cudaMemsetAsync(w->ctrl + 2, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
  }
  const size_t smem = (size_t)2 * 2 * kNsT * kNsLd * 8;
  static bool attr = false;
  if (!attr) {
    e = cudaFuncSetAttribute(ns_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  void* args[] = {(void*)&a};
  count_launch();
  return cudaLaunchCooperativeKernel((const void*)ns_kernel, dim3(a.nup * a.nsign),
                                     dim3(kNsThreads), args, smem, st);
}

// ---- Jacobi fallback (the NS iteration did not converge): f(theta), F = Y diag(f) Y^T, rank
__global__ void ns_fallback_kernel(const int* fail, int op_soft, double thr,
                                   const double* __restrict__ theta, const double* __restrict__ Y,
                                   int p, double* __restrict__ F, int* rank) {
  if (*fail == 0) return;
  extern __shared__ double fv[];
  for (int k = threadIdx.x; k < p; k += blockDim.x) {
    const double t = theta[k];
    fv[k] = op_soft ? (t > thr ? t - thr : (t < -thr ? t + thr : 0.0)) : (t > 0.0 ? t : 0.0);
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int r = 0;
    for (int k = 0; k < p; ++k) r += fv[k] != 0.0;
    *rank = r;
  }
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < p * p; x += gridDim.x * blockDim.x) {
    const int i = x / p, j = x - i * p;
    if (j < i) continue;
    double s = 0.0;
    for (int k = 0; k < p; ++k) s += Y[(size_t)i * p + k] * fv[k] * Y[(size_t)j * p + k];
    F[(size_t)i * p + j] = s;
    F[(size_t)j * p + i] = s;
  }
}

cudaError_t ns_fallback_launch(const int* fail, int op_soft, double thr, const double* theta,
                               const double* Y, int p, double* F, int* rank, cudaStream_t st) {
  count_launch();
  ns_fallback_kernel<<<std::max(1, (p * p + 255) / 256), 256, p * sizeof(double), st>>>(
      fail, op_soft, thr, theta, Y, p, F, rank);
  return cudaGetLastError();
}

}  // namespace pf
