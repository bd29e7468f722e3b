// pf_small.cu -- the p x p side of the hot path and the tall-skinny n x p kernels:
//   Gram / cross-Gram (fp64 DMMA) for CholeskyQR2 and H = Q^T (A Q)
//   Cholesky + triangular inverse, shifted on breakdown                       (reading R10)
//   right multiplication Y <- Y R (fp64 DMMA): Q = Y R^-1, V = Q Y_eig, re-basing
//   two-sided parallel cyclic Jacobi eigensolver (single CTA)                  (eqn:RR)
//   spectral operator, interval / re-base plan, Lanczos, perturbation helper.
#include <cooperative_groups.h>

#include <algorithm>

#include <cstdlib>

#include "pf_kernels.cuh"
#include "../../include/pf.h"

namespace pf {

// =============================================================================== Gram
// partials[blk] = X[rows of blk]^T Y[rows of blk]; then gram_reduce sums blocks in order.
constexpr int kGramRows = 32;       // rows per block are a multiple of this
constexpr int kGramMaxBlocks = 148;

template <int P>
struct GramCfg {
  static constexpr int WTN = P < 32 ? P : 32;        // warp tile 16 x WTN
  static constexpr int NT = WTN / 8;
  static constexpr int NWT = (P / 16) * (P / WTN);   // warp tiles
  static constexpr int PER_WARP = (NWT + 7) / 8;
  static constexpr int LD = P + 4;                   // padded smem row (conflict-free frags)
  static constexpr int R = P >= 128 ? 16 : 32;       // rows per smem sub-chunk (static smem)
};

// One cooperative launch: per-CTA partial products, a grid barrier, then every CTA sums a slice
// of the p x p entries over the partials in CTA order (deterministic; the same order as a
// separate reduction kernel, one launch fewer per Gram).
template <int P>
__global__ void __launch_bounds__(256) gram_partial_kernel(const double* __restrict__ X,
                                                          const double* __restrict__ Y,
                                                          int n_rows, int rows_per_block,
                                                          double* __restrict__ partials,
                                                          const int* cond, double* G) {
  using C = GramCfg<P>;
  if (cond && *cond == 0) return;  // uniform over the grid
  __shared__ __align__(16) double Xs[C::R * C::LD];
  __shared__ __align__(16) double Ys[C::R * C::LD];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g8 = lane >> 2, t4 = lane & 3;
  const int r0 = blockIdx.x * rows_per_block;
  const int r1 = min(n_rows, r0 + rows_per_block);
  double acc[C::PER_WARP][C::NT][4];
#pragma unroll
  for (int w = 0; w < C::PER_WARP; ++w)
#pragma unroll
    for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[w][nt][i] = 0.0;

  // sub-chunk loads staged in registers one chunk ahead: every load of a chunk is in flight at
  // once, and the next chunk's loads overlap this chunk's DMMAs
  constexpr int NE = C::R * P / 2 / 256;  // double2 per thread per matrix per chunk
  static_assert(NE >= 1 && (C::R * P / 2) % 256 == 0, "chunk split");
  double2 xr[NE], yr[NE];
  auto load = [&](int rb) {
#pragma unroll
    for (int i = 0; i < NE; ++i) {
      const int e = threadIdx.x + 256 * i;
      const int rr = e / (P / 2), cc = (e % (P / 2)) * 2;
      const int row = rb + rr;
      xr[i] = yr[i] = make_double2(0.0, 0.0);
      if (row < r1) {
        xr[i] = __ldcg(reinterpret_cast<const double2*>(X + (size_t)row * P + cc));
        yr[i] = __ldcg(reinterpret_cast<const double2*>(Y + (size_t)row * P + cc));
      }
    }
  };
  if (r0 < r1) load(r0);
  for (int rb = r0; rb < r1; rb += C::R) {
#pragma unroll
    for (int i = 0; i < NE; ++i) {
      const int e = threadIdx.x + 256 * i;
      const int rr = e / (P / 2), cc = (e % (P / 2)) * 2;
      *reinterpret_cast<double2*>(Xs + rr * C::LD + cc) = xr[i];
      *reinterpret_cast<double2*>(Ys + rr * C::LD + cc) = yr[i];
    }
    __syncthreads();
    if (rb + C::R < r1) load(rb + C::R);
#pragma unroll
    for (int w = 0; w < C::PER_WARP; ++w) {
      const int wt = warp + 8 * w;
      if (wt < C::NWT) {
        const int m0 = (wt % (P / 16)) * 16, n0 = (wt / (P / 16)) * C::WTN;
#pragma unroll
        for (int ks = 0; ks < C::R / 4; ++ks) {
          const int k = ks * 4 + t4;
          const double a0 = Xs[k * C::LD + m0 + g8];
          const double a1 = Xs[k * C::LD + m0 + g8 + 8];
#pragma unroll
          for (int nt = 0; nt < C::NT; ++nt)
            dmma16884(acc[w][nt], a0, a1, Ys[k * C::LD + n0 + nt * 8 + g8]);
        }
      }
    }
    __syncthreads();
  }
  double* out = partials + (size_t)blockIdx.x * P * P;
#pragma unroll
  for (int w = 0; w < C::PER_WARP; ++w) {
    const int wt = warp + 8 * w;
    if (wt < C::NWT) {
      const int m0 = (wt % (P / 16)) * 16, n0 = (wt / (P / 16)) * C::WTN;
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int m = m0 + g8 + 8 * h, n = n0 + nt * 8 + 2 * t4;
          *reinterpret_cast<double2*>(out + m * P + n) =
              make_double2(acc[w][nt][2 * h], acc[w][nt][2 * h + 1]);
        }
    }
  }
  cooperative_groups::this_grid().sync();
  // G[e] = sum over the CTA partials: TPE lanes per entry (a power of two up to 32, as many as the
  // grid has threads for), each summing every TPE-th partial in order, then a fixed xor tree
  // (deterministic; 8 lanes per entry at p = 64 instead of one lane walking 128 partials)
  const int nb = gridDim.x;
  const int nthr = gridDim.x * blockDim.x;
  int tpe = 1;
  while (tpe < 32 && tpe * 2 * P * P <= nthr) tpe *= 2;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int sub = gt & (tpe - 1);
  // warp-uniform trip count (the shuffles need every lane): entries e0 = base + lane / tpe
  for (int base = (gt >> 5) * (32 / tpe); base < P * P; base += nthr / tpe) {
    const int e0 = base + (threadIdx.x & 31) / tpe;
    double s = 0.0;
    if (e0 < P * P)
      for (int b = sub; b < nb; b += tpe) s += __ldcg(partials + (size_t)b * P * P + e0);
    for (int o = 1; o < tpe; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (sub == 0 && e0 < P * P) G[e0] = s;
  }
}

static int gram_rows_per_block(int n_rows) {
  int nb = std::min(kGramMaxBlocks, std::max(1, (n_rows + 63) / 64));
  int rpb = (n_rows + nb - 1) / nb;
  rpb = ((rpb + kGramRows - 1) / kGramRows) * kGramRows;
  return std::max(rpb, kGramRows);
}

int gram_blocks(int n_rows, int p) {
  (void)p;
  const int rpb = gram_rows_per_block(n_rows);
  return std::max(1, (n_rows + rpb - 1) / rpb);
}

template <int P>
static cudaError_t gram_coop(const double* X, const double* Y, int n_rows, int rpb, int nb,
                             double* partials, const int* cond, double* G, cudaStream_t st) {
  void* args[] = {(void*)&X, (void*)&Y, (void*)&n_rows, (void*)&rpb, (void*)&partials,
                  (void*)&cond, (void*)&G};
  return cudaLaunchCooperativeKernel((const void*)gram_partial_kernel<P>, dim3(nb), dim3(256),
                                     args, 0, st);
}

cudaError_t gram_launch(const double* X, const double* Y, int n_rows, int p, double* G,
                        double* partials, int* counter, const int* cond, cudaStream_t st) {
  (void)counter;
  const int rpb = gram_rows_per_block(n_rows);
  const int nb = std::max(1, (n_rows + rpb - 1) / rpb);  // <= 148: one CTA per SM fits
  count_launch();
  switch (p) {
    case 16: return gram_coop<16>(X, Y, n_rows, rpb, nb, partials, cond, G, st);
    case 32: return gram_coop<32>(X, Y, n_rows, rpb, nb, partials, cond, G, st);
    case 64: return gram_coop<64>(X, Y, n_rows, rpb, nb, partials, cond, G, st);
    case 128: return gram_coop<128>(X, Y, n_rows, rpb, nb, partials, cond, G, st);
    default: return cudaErrorInvalidValue;
  }
}

// =============================================================================== Cholesky
// One CTA.  M (p x (p+1), smem): lower triangle incl. diagonal = L, X = L^{-1} stored
// transposed in the strict upper part: X[i][c] (i >= c) at M[c][i+1].  Output Rinv = L^{-T}.
__global__ void __launch_bounds__(512) chol_inv_kernel(const double* __restrict__ G, int p,
                                                     double shift_scale, double* __restrict__ Rinv,
                                                     DevState* state, int* shift_flag_out,
                                                     const int* cond) {
  if (cond && *cond == 0) return;
  extern __shared__ double M[];
  __shared__ double red[32];
  const int P1 = p + 1;
  const int tid = threadIdx.x, nt = blockDim.x;

  // finiteness + trace
  double tr = 0.0;
  int bad = 0;
  for (int e = tid; e < p * p; e += nt) {
    const double v = G[e];
    if (!isfinite(v)) bad = 1;
    if (e / p == e % p) tr += v;
  }
  bad = __syncthreads_or(bad);
  tr = block_sum(tr, red);
  if (bad && tid == 0) atomicOr(&state->flags, PF_FLAG_NONFINITE);

  // 2-D thread layout for the triangular updates (no integer division in the inner loops)
  const int tx = tid & 31, ty = tid >> 5, nty = nt >> 5;
  double* gdiag = M + p * P1;  // p doubles after M
  for (int i = tid; i < p; i += nt) gdiag[i] = G[i * p + i];

  double shift = 0.0;
  int attempt = 0;
  for (;;) {
    for (int i = ty; i < p; i += nty)
      for (int j = tx; j <= i; j += 32) M[i * P1 + j] = G[i * p + j] + ((i == j) ? shift : 0.0);
    __syncthreads();
    // right-looking Cholesky, one barrier per column: the trailing update uses the unscaled
    // column j divided by the pivot, and column j is scaled afterwards (disjoint elements)
    bool fail = false;
    for (int j = 0; j < p; ++j) {
      const double d = M[j * P1 + j];
      if (!(d > 1e-12 * gdiag[j]) || !(d > 0.0)) {  // uniform: every thread reads the same d
        fail = true;
        break;
      }
      const double rsd = rsqrt(d);      // 1 / sqrt(d): one MUFU + refinement, no division
      const double inv_d = rsd * rsd;
      for (int i = j + 1 + ty; i < p; i += nty) {
        const double lij = M[i * P1 + j] * inv_d;
        for (int k = j + 1 + tx; k <= i; k += 32) M[i * P1 + k] -= lij * M[k * P1 + j];
      }
      __syncthreads();
      for (int i = j + 1 + tid; i < p; i += nt) M[i * P1 + j] *= rsd;
      if (tid == 0) M[j * P1 + j] = d * rsd;
    }
    __syncthreads();
    if (!fail) break;
    if (attempt == 1) {
      if (tid == 0) atomicOr(&state->flags, PF_FLAG_NONFINITE);
      break;
    }
    attempt = 1;
    shift = shift_scale * (tr > 0.0 ? tr : 1.0);
  }
  if (tid == 0) {
    if (attempt) atomicOr(&state->flags, PF_FLAG_CHOL_SHIFT);
    if (shift_flag_out && attempt) *shift_flag_out = 1;
  }
  // X = L^{-1}, right-looking with one barrier per column: X[i][c] -= L[i][j] X[j][c] / L[j][j]
  // for i > j, c <= j (row j unscaled), then row j is scaled by 1/L[j][j] (disjoint elements).
  for (int i = ty; i < p; i += nty)
    for (int c = tx; c <= i; c += 32) M[c * P1 + i + 1] = (i == c) ? 1.0 : 0.0;
  for (int i = tid; i < p; i += nt) gdiag[i] = 1.0 / M[i * P1 + i];  // reciprocals of diag(L)
  __syncthreads();
  for (int j = 0; j < p; ++j) {
    const double inv = gdiag[j];
    for (int i = j + 1 + ty; i < p; i += nty) {
      const double lij = M[i * P1 + j] * inv;
      for (int c = tx; c <= j; c += 32) M[c * P1 + i + 1] -= lij * M[c * P1 + j + 1];
    }
    __syncthreads();
    for (int c = tid; c <= j; c += nt) M[c * P1 + j + 1] *= inv;
  }
  __syncthreads();
  // Rinv = L^{-T}: Rinv[c][i] = X[i][c] (upper triangular)
  for (int e = tid; e < p * p; e += nt) {
    const int c = e / p, i = e % p;
    Rinv[e] = (i >= c) ? M[c * P1 + i + 1] : 0.0;
  }
}

cudaError_t chol_inv_launch(const double* G, int p, int64_t n_global, double* Rinv,
                            DevState* state, int* shift_flag_out, const int* cond,
                            cudaStream_t st) {
  const double u = 1.1102230246251565e-16;
  const double scale = 11.0 * ((double)n_global * p + (double)p * (p + 1)) * u;
  const size_t smem = (size_t)p * (p + 2) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(128 * 130 * sizeof(double)));
    attr = true;
  }
  count_launch();
  chol_inv_kernel<<<1, 512, smem, st>>>(G, p, scale, Rinv, state, shift_flag_out, cond);
  return cudaGetLastError();
}

// Same factorisation and inverse as chol_inv_kernel for p <= 64, with the matrix held in
// registers: 256 threads, thread t owns the 4 x 4 block (rows 4 (t / 16).., cols 4 (t % 16)..)
// of the 64 x 64 matrix padded with the identity.  Each column step publishes the current
// column through a double-buffered 64-vector and needs ONE barrier; every thread then updates
// its 16 entries in registers (chol_inv_kernel keeps M in shared memory and walks rows and
// columns in loops: ~75 us per active call at p = 64 vs 56 us here, measured).  Arithmetic per entry is the
// same: M_ik -= (M_ij / d) M_kj, L_ij = M_ij / sqrt(d); X_ic -= (L_ij / L_jj) X_jc with row j
// unscaled, then row j scaled by 1 / L_jj.
__global__ void __launch_bounds__(256) chol_inv_reg_kernel(const double* __restrict__ G, int p,
                                                         double shift_scale,
                                                         double* __restrict__ Rinv,
                                                         DevState* state, int* shift_flag_out,
                                                         const int* cond) {
  if (cond && *cond == 0) return;
  constexpr int PC = 64;
  __shared__ double Ls[PC * (PC + 1)];  // L (lower), then read by the inverse
  __shared__ double buf[2][PC];
  __shared__ double red[32];
  __shared__ double gdiag[PC];
  const int tid = threadIdx.x, bi = tid >> 4, bj = tid & 15;
  const int r0 = 4 * bi, c0 = 4 * bj;
  const bool act = bj <= bi;  // lower-triangle blocks (incl. diagonal)

  double tr = 0.0;
  int bad = 0;
  for (int e = tid; e < p * p; e += 256) {
    const double v = G[e];
    if (!isfinite(v)) bad = 1;
    if (e / p == e % p) tr += v;
  }
  bad = __syncthreads_or(bad);
  tr = block_sum(tr, red);
  if (bad && tid == 0) atomicOr(&state->flags, PF_FLAG_NONFINITE);
  for (int i = tid; i < PC; i += 256) gdiag[i] = i < p ? G[(size_t)i * p + i] : 1.0;

  double a[4][4];
  double shift = 0.0;
  int attempt = 0;
  for (;;) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int r = r0 + u, c = c0 + v;
        a[u][v] = (r < p && c < p) ? G[(size_t)r * p + c] + (r == c ? shift : 0.0)
                                   : (r == c ? 1.0 : 0.0);
      }
    __syncthreads();
    bool fail = false;
    for (int j = 0; j < p; ++j) {  // the identity padding past p needs no steps
      double* cb = buf[j & 1];
      if (bj == (j >> 2) && act) {  // owners of column j publish it (rows >= 4 (j / 4))
        const int jj = j & 3;  // static register indices only (no local-memory arrays)
#pragma unroll
        for (int u = 0; u < 4; ++u)
          cb[r0 + u] = jj == 0 ? a[u][0] : jj == 1 ? a[u][1] : jj == 2 ? a[u][2] : a[u][3];
      }
      __syncthreads();
      const double d = cb[j];
      if (!(d > 1e-12 * gdiag[j]) || !(d > 0.0)) {  // uniform
        fail = true;
        break;
      }
      const double rsd = rsqrt(d);
      const double inv_d = rsd * rsd;
      if (tid < PC) Ls[tid * (PC + 1) + j] = tid > j ? cb[tid] * rsd : (tid == j ? d * rsd : 0.0);
      if (act && r0 + 3 > j) {
        double li[4], lk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) li[u] = cb[r0 + u] * inv_d;
#pragma unroll
        for (int v = 0; v < 4; ++v) lk[v] = cb[c0 + v];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v)
            if (r0 + u > j && c0 + v > j && c0 + v <= r0 + u) a[u][v] -= li[u] * lk[v];
      }
    }
    __syncthreads();
    if (!fail) break;
    if (attempt == 1) {
      if (tid == 0) atomicOr(&state->flags, PF_FLAG_NONFINITE);
      break;
    }
    attempt = 1;
    shift = shift_scale * (tr > 0.0 ? tr : 1.0);
  }
  if (tid == 0) {
    if (attempt) atomicOr(&state->flags, PF_FLAG_CHOL_SHIFT);
    if (shift_flag_out && attempt) *shift_flag_out = 1;
  }
  // X = L^{-1}: x holds rows r0.., cols c0.. of X (identity to start)
  double x[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) x[u][v] = (r0 + u == c0 + v) ? 1.0 : 0.0;
  if (tid < p) gdiag[tid] = 1.0 / Ls[tid * (PC + 1) + tid];
  __syncthreads();
  for (int j = 0; j < p; ++j) {
    double* rb = buf[j & 1];
    if (bi == (j >> 2) && act) {  // owners of row j publish it (unscaled), columns <= j
      const int jj = j & 3;
#pragma unroll
      for (int v = 0; v < 4; ++v)
        rb[c0 + v] = jj == 0 ? x[0][v] : jj == 1 ? x[1][v] : jj == 2 ? x[2][v] : x[3][v];
    }
    __syncthreads();
    const double inv = gdiag[j];
    if (act && r0 + 3 > j && c0 <= j) {
      double lij[4], xj[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) lij[u] = Ls[(r0 + u) * (PC + 1) + j] * inv;
#pragma unroll
      for (int v = 0; v < 4; ++v) xj[v] = rb[c0 + v];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v)
          if (r0 + u > j && c0 + v <= j) x[u][v] -= lij[u] * xj[v];
    }
    if (bi == (j >> 2) && act) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v)
          if (r0 + u == j && c0 + v <= j) x[u][v] *= inv;
    }
  }
  // Rinv = L^{-T}: Rinv[c][i] = X[i][c] (upper triangular), p x p
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int i = r0 + u, c = c0 + v;
      if (i < p && c < p) Rinv[(size_t)c * p + i] = act ? x[u][v] : 0.0;
    }
  // blocks above the diagonal (inactive threads) write the zero lower part of Rinv
}

cudaError_t chol_inv_reg_launch(const double* G, int p, int64_t n_global, double* Rinv,
                                DevState* state, int* shift_flag_out, const int* cond,
                                cudaStream_t st) {
  if (p > 64) return cudaErrorInvalidValue;
  const double u = 1.1102230246251565e-16;
  const double scale = 11.0 * ((double)n_global * p + (double)p * (p + 1)) * u;
  count_launch();
  chol_inv_reg_kernel<<<1, 256, 0, st>>>(G, p, scale, Rinv, state, shift_flag_out, cond);
  return cudaGetLastError();
}

// =============================================================================== Y R
template <int P>
struct RmulCfg {
  static constexpr int BM = 64;
  static constexpr int LD = P + 4;
  static constexpr int WN = P / 2;                  // warps 4 (M) x 2 (N), warp tile 16 x WN
  static constexpr int NT = WN / 8;
  static constexpr int SMEM = (P * LD + BM * LD) * 8;
};

template <int P>
__global__ void __launch_bounds__(256) rmul_kernel(const double* in, int64_t ldi,
                                                  const double* __restrict__ R, double* out,
                                                  int64_t ldo, int n_rows, const int* cond) {
  using C = RmulCfg<P>;
  if (cond && *cond == 0) return;
  extern __shared__ __align__(16) double sm[];
  double* Rs = sm;
  double* Ys = sm + P * C::LD;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g8 = lane >> 2, t4 = lane & 3;
  const int row0 = blockIdx.x * C::BM;
  // all loads into registers first (in / out may alias, so the compiler will not hoist loads
  // above the shared-memory stores by itself): one memory latency instead of one per element
  constexpr int NR = (P * P / 2 + 255) / 256, NY = (C::BM * P / 2 + 255) / 256;
  double2 rv[NR], yv[NY];
#pragma unroll
  for (int i = 0; i < NR; ++i) {
    const int e = threadIdx.x + 256 * i;
    const int r = e / (P / 2), c = (e % (P / 2)) * 2;
    rv[i] = e < P * P / 2 ? __ldg(reinterpret_cast<const double2*>(R + r * P + c))
                          : make_double2(0.0, 0.0);
  }
#pragma unroll
  for (int i = 0; i < NY; ++i) {
    const int e = threadIdx.x + 256 * i;
    const int r = e / (P / 2), c = (e % (P / 2)) * 2;
    yv[i] = make_double2(0.0, 0.0);
    if (e < C::BM * P / 2 && row0 + r < n_rows)
      yv[i] = *reinterpret_cast<const double2*>(in + (size_t)(row0 + r) * ldi + c);
  }
#pragma unroll
  for (int i = 0; i < NR; ++i) {
    const int e = threadIdx.x + 256 * i;
    const int r = e / (P / 2), c = (e % (P / 2)) * 2;
    if (e < P * P / 2) *reinterpret_cast<double2*>(Rs + r * C::LD + c) = rv[i];
  }
#pragma unroll
  for (int i = 0; i < NY; ++i) {
    const int e = threadIdx.x + 256 * i;
    const int r = e / (P / 2), c = (e % (P / 2)) * 2;
    if (e < C::BM * P / 2) *reinterpret_cast<double2*>(Ys + r * C::LD + c) = yv[i];
  }
  __syncthreads();
  const int wm = warp & 3, wn = warp >> 2;
  double acc[C::NT][4];
#pragma unroll
  for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[nt][i] = 0.0;
#pragma unroll 4
  for (int ks = 0; ks < P / 4; ++ks) {
    const int k = ks * 4 + t4;
    const double a0 = Ys[(wm * 16 + g8) * C::LD + k];
    const double a1 = Ys[(wm * 16 + g8 + 8) * C::LD + k];
#pragma unroll
    for (int nt = 0; nt < C::NT; ++nt)
      dmma16884(acc[nt], a0, a1, Rs[k * C::LD + wn * C::WN + nt * 8 + g8]);
  }
#pragma unroll
  for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int row = row0 + wm * 16 + g8 + 8 * h;
      if (row < n_rows) {
        const int col = wn * C::WN + nt * 8 + 2 * t4;
        *reinterpret_cast<double2*>(out + (size_t)row * ldo + col) =
            make_double2(acc[nt][2 * h], acc[nt][2 * h + 1]);
      }
    }
}

template <int P>
static cudaError_t rmul_p(const double* in, int64_t ldi, const double* R, double* out,
                          int64_t ldo, int n_rows, const int* cond, cudaStream_t st) {
  using C = RmulCfg<P>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(rmul_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  const int grid = std::max(1, (n_rows + C::BM - 1) / C::BM);
  count_launch();
  rmul_kernel<P><<<grid, 256, C::SMEM, st>>>(in, ldi, R, out, ldo, n_rows, cond);
  return cudaGetLastError();
}

cudaError_t rmul_launch(const double* in, int64_t ldi, const double* R, double* out, int64_t ldo,
                        int n_rows, int p, const int* cond, cudaStream_t st) {
  switch (p) {
    case 16: return rmul_p<16>(in, ldi, R, out, ldo, n_rows, cond, st);
    case 32: return rmul_p<32>(in, ldi, R, out, ldo, n_rows, cond, st);
    case 64: return rmul_p<64>(in, ldi, R, out, ldo, n_rows, cond, st);
    case 128: return rmul_p<128>(in, ldi, R, out, ldo, n_rows, cond, st);
    default: return cudaErrorInvalidValue;
  }
}

// =============================================================================== Jacobi
// Two-sided cyclic Jacobi with the round-robin (tournament) parallel ordering: in each round the
// PE/2 disjoint pairs are rotated simultaneously; every 2x2 block (pair a, pair b) of H is
// updated by exactly one thread as B' = J_a^T B J_b (J = [[c, s], [-s, c]], Golub & Van Loan
// sym.schur2), so no row/column phasing is needed.  PE (compile time) >= p is the padded even
// order; indices >= p are inert dummies (identity rotations, zero rows).  H is stored full for
// PE <= 64 and as a packed upper triangle for PE = 128 (so H + V fit in 227 KB of smem).
template <int PE>
struct JacCfg {
  static constexpr bool PACKED = PE > 64;
  static constexpr int HALF = PE / 2;
  static constexpr int NBLK = HALF * (HALF + 1) / 2;
  static constexpr int HSIZE = PACKED ? PE * (PE + 1) / 2 : PE * PE;
  static constexpr int THREADS = PE <= 32 ? 256 : 1024;
  static constexpr size_t SMEM =
      (size_t)(HSIZE + PE * PE + 6 * HALF) * 8 + 4 * HALF * 4 + NBLK * 2;
};

template <int PE>
__device__ __forceinline__ int hix(int i, int j) {
  if (JacCfg<PE>::PACKED) {
    if (i > j) {
      const int t = i;
      i = j;
      j = t;
    }
    return i * PE - (i * (i - 1)) / 2 + (j - i);
  }
  return i * PE + j;
}

template <int PE>
__global__ void __launch_bounds__(JacCfg<PE>::THREADS) jacobi_kernel(
    const double* __restrict__ H, int p_static, const int* p_dev, double* __restrict__ theta,
    double* __restrict__ Yout, DevState* state, double tol, int max_sweeps, const int* cond) {
  if (cond && *cond == 0) return;  // conditional launch
  using C = JacCfg<PE>;
  extern __shared__ double js[];
  __shared__ double red[32];
  __shared__ int s_cnt;
  __shared__ double s_norm;
  const int p = p_dev ? *p_dev : p_static;
  if (p <= 0) return;
  double* Hs = js;                                       // HSIZE
  double* V = Hs + C::HSIZE;                             // PE x PE
  double* cs2 = V + PE * PE;                             // [2][HALF][3] = c, s, t
  int* pi2 = reinterpret_cast<int*>(cs2 + 6 * C::HALF);  // [2][HALF]
  int* pj2 = pi2 + 2 * C::HALF;                          // [2][HALF]
  unsigned short* blk = reinterpret_cast<unsigned short*>(pj2 + 2 * C::HALF);  // (a << 8) | b
  const int tid = threadIdx.x;
  constexpr int NT = C::THREADS;

  for (int e = tid; e < C::NBLK; e += NT) {
    int a = 0, rem = e;
    while (rem >= C::HALF - a) {
      rem -= C::HALF - a;
      ++a;
    }
    blk[e] = (unsigned short)((a << 8) | (a + rem));
  }
  for (int e = tid; e < PE * PE; e += NT) {
    const int i = e / PE, j = e % PE;
    V[e] = (i == j) ? 1.0 : 0.0;
    if (!C::PACKED || i <= j)
      Hs[hix<PE>(i, j)] = (i < p && j < p) ? 0.5 * (H[i * p + j] + H[j * p + i]) : 0.0;
  }
  __syncthreads();

  int sweep = 0;
  bool converged = false;
  for (; sweep < max_sweeps; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int e = tid; e < PE * PE; e += NT) {
      const int i = e / PE, j = e % PE;
      const double v = Hs[hix<PE>(i, j)];
      tot += v * v;
      if (i != j) off += v * v;
    }
    off = block_sum(off, red);
    tot = block_sum(tot, red);
    if (off <= tol * tol * tot || off == 0.0) {
      converged = true;
      break;
    }
    if (tid == 0) {
      s_cnt = 0;
      s_norm = sqrt(tot);
    }
    __syncthreads();
    for (int r = 0; r <= PE - 1; ++r) {
      // phase 1: the first warp computes the rotations of round r (double-buffered) while the
      // other warps apply the V update of round r - 1 (V is not read inside a sweep)
      double* cs = cs2 + (r & 1) * 3 * C::HALF;
      int* pi = pi2 + (r & 1) * C::HALF;
      int* pj = pj2 + (r & 1) * C::HALF;
      if (r > 0 && tid >= 32) {
        // V is stored transposed (row i of the buffer = column i of V): the rotation of columns
        // i, j is two contiguous rows, one warp per pair, c / s broadcast, no bank conflicts
        const double* csp = cs2 + ((r - 1) & 1) * 3 * C::HALF;
        const int* pip = pi2 + ((r - 1) & 1) * C::HALF;
        const int* pjp = pj2 + ((r - 1) & 1) * C::HALF;
        const int lane = tid & 31;
        for (int m = (tid >> 5) - 1; m < C::HALF; m += NT / 32 - 1) {
          const double c = csp[3 * m], s = csp[3 * m + 1];
          if (s != 0.0) {
            double* vi = V + pip[m] * PE;
            double* vj = V + pjp[m] * PE;
            for (int k = lane; k < PE; k += 32) {
              const double a = vi[k], b = vj[k];
              vi[k] = c * a - s * b;
              vj[k] = s * a + c * b;
            }
          }
        }
      }
      if (r == PE - 1) {  // flush of the last round's V update done above
        __syncthreads();
        break;
      }
      if (tid < C::HALF) {
        const int m = tid;
        int a, b;
        if (m == 0) {
          a = PE - 1;
          b = r;
        } else {
          a = (r + m) % (PE - 1);
          b = (r - m + (PE - 1)) % (PE - 1);
        }
        const int i = a < b ? a : b, j = a < b ? b : a;
        pi[m] = i;
        pj[m] = j;
        double c = 1.0, s = 0.0, t = 0.0;
        if (j < p) {
          const double hij = Hs[hix<PE>(i, j)];
          // threshold Jacobi: skip rotations below the rounding floor of H; the error this
          // leaves in V diag(f) V^T is <= |h_ij| (a rotation mixes pairs within their gap)
          if (fabs(hij) > 1e-16 * s_norm) {
            const double hii = Hs[hix<PE>(i, i)], hjj = Hs[hix<PE>(j, j)];
            // sym.schur2 via cot(2 phi) = (h_jj - h_ii) / (2 h_ij), |phi| <= pi/4, written with
            // two reciprocal square roots instead of the div/sqrt/div chain:
            // cos 2phi = |d|/r, c = sqrt((1 + cos 2phi)/2), s = sign(d) e / (2 r c), t = s / c
            const double dd = hjj - hii, ee = 2.0 * hij;
            const double ir = rsqrt(dd * dd + ee * ee);
            const double hh = 0.5 + 0.5 * fabs(dd) * ir;
            const double rc = rsqrt(hh);
            c = hh * rc;
            s = (dd >= 0.0 ? 0.5 : -0.5) * ee * ir * rc;
            t = s * rc;
          }
        }
        cs[3 * m] = c;
        cs[3 * m + 1] = s;
        cs[3 * m + 2] = t;
        // count rotations with a ballot (a shared atomic per rotating pair serialises the round)
        const unsigned wmask = C::HALF >= 32 ? 0xffffffffu : ((1u << C::HALF) - 1u);
        const unsigned rot = __ballot_sync(wmask, s != 0.0);
        if ((m & 31) == 0) atomicAdd(&s_cnt, __popc(rot));
      }
      __syncthreads();
      for (int e = tid; e < C::NBLK; e += NT) {
        const int a = blk[e] >> 8, b = blk[e] & 0xff;
        const int ia = pi[a], ja = pj[a];
        const double ca = cs[3 * a], sa = cs[3 * a + 1];
        if (a == b) {
          if (sa != 0.0) {
            const double ta = cs[3 * a + 2];
            const double hij = Hs[hix<PE>(ia, ja)];
            Hs[hix<PE>(ia, ia)] -= ta * hij;
            Hs[hix<PE>(ja, ja)] += ta * hij;
            Hs[hix<PE>(ia, ja)] = 0.0;
            if (!C::PACKED) Hs[hix<PE>(ja, ia)] = 0.0;
          }
        } else {
          const int ib = pi[b], jb = pj[b];
          const double cb = cs[3 * b], sb = cs[3 * b + 1];
          if (sa != 0.0 || sb != 0.0) {
            const int k11 = hix<PE>(ia, ib), k12 = hix<PE>(ia, jb), k21 = hix<PE>(ja, ib),
                      k22 = hix<PE>(ja, jb);
            const double b11 = Hs[k11], b12 = Hs[k12], b21 = Hs[k21], b22 = Hs[k22];
            const double t11 = ca * b11 - sa * b21, t12 = ca * b12 - sa * b22;
            const double t21 = sa * b11 + ca * b21, t22 = sa * b12 + ca * b22;
            const double n11 = t11 * cb - t12 * sb, n12 = t11 * sb + t12 * cb;
            const double n21 = t21 * cb - t22 * sb, n22 = t21 * sb + t22 * cb;
            Hs[k11] = n11;
            Hs[k12] = n12;
            Hs[k21] = n21;
            Hs[k22] = n22;
            if (!C::PACKED) {  // mirror into the lower triangle
              Hs[hix<PE>(ib, ia)] = n11;
              Hs[hix<PE>(jb, ia)] = n12;
              Hs[hix<PE>(ib, ja)] = n21;
              Hs[hix<PE>(jb, ja)] = n22;
            }
          }
        }
      }
      __syncthreads();
    }
    if (s_cnt == 0) {
      converged = true;
      ++sweep;
      break;
    }
  }
  if (tid == 0) {
    state->scratch[1] = (double)sweep;
    if (!converged) atomicOr(&state->flags, PF_FLAG_JACOBI_MAXSWEEP);
  }
  // sort descending (stable by index) and emit
  for (int i = tid; i < p; i += NT) {
    const double li = Hs[hix<PE>(i, i)];
    int rank = 0;
    for (int k = 0; k < p; ++k) {
      const double lk = Hs[hix<PE>(k, k)];
      if (lk > li || (lk == li && k < i)) ++rank;
    }
    theta[rank] = li;
    for (int row = 0; row < p; ++row) Yout[row * p + rank] = V[i * PE + row];  // V transposed
  }
}

// Row-owner variant for PE <= 64 (the same two-sided cyclic Jacobi, same rotations and ordering):
// full H and V^T in shared memory, warp a owns the rows i_a, j_a of its pair in round r.  Phase 1:
// lane 0 of warp a computes rotation a from its own rows.  Phase 2: lane b of warp a forms block
// (a, b) of J^T H J -- rows i_a, j_a only, so every warp writes only rows it owns (in place, no
// mirror stores, conflict-light row accesses) -- and warp a rotates its two rows of V^T.  Each
// block entry is summed as (P11 b11 + P22 b22) + (P12 b12 + P21 b21) with P = products of the
// rotation entries and no contraction, which is exactly symmetric under (a, b) -> (b, a), so H
// stays bit-symmetric.  Two barriers per round.
template <int PE>
__global__ void __launch_bounds__(PE * 16) jacobi_rows_kernel(
    const double* __restrict__ H, int p_static, const int* p_dev, double* __restrict__ theta,
    double* __restrict__ Yout, DevState* state, double tol, int max_sweeps, const int* cond) {
  if (cond && *cond == 0) return;  // conditional launch
  constexpr int HALF = PE / 2, NT = PE * 16;  // HALF warps
  extern __shared__ double js[];
  __shared__ double red[32];
  __shared__ int s_any;
  __shared__ double s_norm;
  const int p = p_dev ? *p_dev : p_static;
  if (p <= 0) return;
  double* Hs = js;                   // PE x PE, both triangles
  double* Vt = Hs + PE * PE;         // V transposed
  double* rc = Vt + PE * PE;         // [HALF] c
  double* rs = rc + HALF;            // [HALF] s
  double* rt = rs + HALF;            // [HALF] t
  int* ri = reinterpret_cast<int*>(rt + HALF);
  int* rj = ri + HALF;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < PE * PE; e += NT) {
    const int i = e / PE, j = e % PE;
    Vt[e] = (i == j) ? 1.0 : 0.0;
    Hs[e] = (i < p && j < p) ? 0.5 * (H[i * p + j] + H[j * p + i]) : 0.0;
  }
  __syncthreads();
  int sweep = 0;
  bool converged = false;
  for (; sweep < max_sweeps; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int e = tid; e < PE * PE; e += NT) {
      const double v = Hs[e];
      tot += v * v;
      if (e / PE != e % PE) off += v * v;
    }
    off = block_sum(off, red);
    tot = block_sum(tot, red);
    if (off <= tol * tol * tot || off == 0.0) {
      converged = true;
      break;
    }
    if (tid == 0) {
      s_any = 0;
      s_norm = sqrt(tot);
    }
    __syncthreads();
    for (int r = 0; r < PE - 1; ++r) {
      const int m = warp;  // this warp's pair
      int a0, b0;
      if (m == 0) {
        a0 = PE - 1;
        b0 = r;
      } else {
        a0 = (r + m) % (PE - 1);
        b0 = (r - m + (PE - 1)) % (PE - 1);
      }
      const int ia = a0 < b0 ? a0 : b0, ja = a0 < b0 ? b0 : a0;
      if (lane == 0) {
        double c = 1.0, s = 0.0, t = 0.0;
        if (ja < p) {
          const double hij = Hs[ia * PE + ja];
          if (fabs(hij) > 1e-16 * s_norm) {  // same threshold and schur2 as jacobi_kernel
            const double hii = Hs[ia * PE + ia], hjj = Hs[ja * PE + ja];
            const double dd = hjj - hii, ee = 2.0 * hij;
            const double ir = rsqrt(dd * dd + ee * ee);
            const double hh = 0.5 + 0.5 * fabs(dd) * ir;
            const double rcp = rsqrt(hh);
            c = hh * rcp;
            s = (dd >= 0.0 ? 0.5 : -0.5) * ee * ir * rcp;
            t = s * rcp;
            s_any = 1;
          }
        }
        rc[m] = c;
        rs[m] = s;
        rt[m] = t;
        ri[m] = ia;
        rj[m] = ja;
      }
      __syncthreads();
      const double ca = rc[m], sa = rs[m];
      for (int bb = lane; bb < HALF; bb += 32) {
        const double cb = rc[bb], sb = rs[bb];
        if (sa == 0.0 && sb == 0.0) continue;
        const int ib = ri[bb], jb = rj[bb];
        if (bb == m) {
          const double ta = rt[m];
          const double hij = Hs[ia * PE + ja];
          Hs[ia * PE + ia] -= ta * hij;
          Hs[ja * PE + ja] += ta * hij;
          Hs[ia * PE + ja] = 0.0;
          Hs[ja * PE + ia] = 0.0;
        } else {
          const double b11 = Hs[ia * PE + ib], b12 = Hs[ia * PE + jb];
          const double b21 = Hs[ja * PE + ib], b22 = Hs[ja * PE + jb];
          // J_a = [[ca, sa], [-sa, ca]] on (ia, ja), J_b likewise; n = J_a^T B J_b
          const double pcc = __dmul_rn(ca, cb), pcs = __dmul_rn(ca, sb);
          const double psc = __dmul_rn(sa, cb), pss = __dmul_rn(sa, sb);
          // n11 = cc b11 - cs b12 - sc b21 + ss b22; n12 = cs b11 + cc b12 - ss b21 - sc b22
          // n21 = sc b11 - ss b12 + cc b21 - cs b22; n22 = ss b11 + sc b12 + cs b21 + cc b22
          const double n11 = __dadd_rn(__dadd_rn(__dmul_rn(pcc, b11), __dmul_rn(pss, b22)),
                                       -__dadd_rn(__dmul_rn(pcs, b12), __dmul_rn(psc, b21)));
          const double n22 = __dadd_rn(__dadd_rn(__dmul_rn(pss, b11), __dmul_rn(pcc, b22)),
                                       __dadd_rn(__dmul_rn(psc, b12), __dmul_rn(pcs, b21)));
          const double n12 = __dadd_rn(__dadd_rn(__dmul_rn(pcs, b11), -__dmul_rn(psc, b22)),
                                       __dadd_rn(__dmul_rn(pcc, b12), -__dmul_rn(pss, b21)));
          const double n21 = __dadd_rn(__dadd_rn(__dmul_rn(psc, b11), -__dmul_rn(pcs, b22)),
                                       __dadd_rn(__dmul_rn(pcc, b21), -__dmul_rn(pss, b12)));
          Hs[ia * PE + ib] = n11;
          Hs[ia * PE + jb] = n12;
          Hs[ja * PE + ib] = n21;
          Hs[ja * PE + jb] = n22;
        }
      }
      if (sa != 0.0) {  // columns ia, ja of V = rows of V^T
        double* vi = Vt + ia * PE;
        double* vj = Vt + ja * PE;
        for (int k = lane; k < PE; k += 32) {
          const double x = vi[k], y = vj[k];
          vi[k] = ca * x - sa * y;
          vj[k] = sa * x + ca * y;
        }
      }
      __syncthreads();
    }
    if (s_any == 0) {
      converged = true;
      ++sweep;
      break;
    }
  }
  if (tid == 0) {
    state->scratch[1] = (double)sweep;
    if (!converged) atomicOr(&state->flags, PF_FLAG_JACOBI_MAXSWEEP);
  }
  for (int i = tid; i < p; i += NT) {  // sort descending (stable by index) and emit
    const double li = Hs[i * PE + i];
    int rank = 0;
    for (int k = 0; k < p; ++k) {
      const double lk = Hs[k * PE + k];
      if (lk > li || (lk == li && k < i)) ++rank;
    }
    theta[rank] = li;
    for (int row = 0; row < p; ++row) Yout[row * p + rank] = Vt[i * PE + row];
  }
}

template <int PE>
static cudaError_t jacobi_rows_pe(const double* H, int p, const int* p_dev, double* theta,
                                  double* Y, DevState* state, double tol, int max_sweeps,
                                  cudaStream_t st, const int* cond) {
  constexpr size_t SMEM = (size_t)(2 * PE * PE + 3 * (PE / 2)) * 8 + (PE / 2) * 8;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(jacobi_rows_kernel<PE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)SMEM);
    attr = true;
  }
  count_launch();
  jacobi_rows_kernel<PE><<<1, PE * 16, SMEM, st>>>(H, p, p_dev, theta, Y, state, tol, max_sweeps,
                                                   cond);
  return cudaGetLastError();
}

template <int PE>
static cudaError_t jacobi_pe(const double* H, int p, const int* p_dev, double* theta, double* Y,
                             DevState* state, double tol, int max_sweeps, cudaStream_t st,
                             const int* cond) {
  using C = JacCfg<PE>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(jacobi_kernel<PE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)C::SMEM);
    attr = true;
  }
  count_launch();
  jacobi_kernel<PE><<<1, C::THREADS, C::SMEM, st>>>(H, p, p_dev, theta, Y, state, tol, max_sweeps,
                                                    cond);
  return cudaGetLastError();
}

// p: order (runtime bound when p_dev != NULL: the kernel reads *p_dev <= p)
cudaError_t jacobi_launch(const double* H, int p, const int* p_dev, double* theta, double* Y,
                          DevState* state, double tol, int max_sweeps, cudaStream_t st,
                          const int* cond) {
  static int rows = -1;  // development knob PF_JACOBI_ROWS=0 selects the block-thread kernel
  if (rows < 0) {
    const char* e = getenv("PF_JACOBI_ROWS");
    rows = e ? atoi(e) : 1;
  }
  // measured (tools/bench_jacobi.py): 1.74 vs 2.03 us per round at p = 64, no gain at p <= 32
  if (rows && p > 32 && p <= 64)
    return jacobi_rows_pe<64>(H, p, p_dev, theta, Y, state, tol, max_sweeps, st, cond);
  if (p <= 16) return jacobi_pe<16>(H, p, p_dev, theta, Y, state, tol, max_sweeps, st, cond);
  if (p <= 32) return jacobi_pe<32>(H, p, p_dev, theta, Y, state, tol, max_sweeps, st, cond);
  if (p <= 64) return jacobi_pe<64>(H, p, p_dev, theta, Y, state, tol, max_sweeps, st, cond);
  if (p <= 128) return jacobi_pe<128>(H, p, p_dev, theta, Y, state, tol, max_sweeps, st, cond);
  return cudaErrorInvalidValue;
}


// =============================================================================== spectral op
__global__ void spectral_kernel(int op, double thr, const double* __restrict__ theta, int p,
                                double* __restrict__ f, int* rank, DevState* state) {
  const int i = threadIdx.x;
  int nz = 0;
  if (i < p) {
    const double t = theta[i];
    double v;
    if (op == PF_OP_PSD)
      v = t > 0.0 ? t : 0.0;  // P_+ 
    else
      v = (t > thr) ? (t - thr) : ((t < -thr) ? (t + thr) : 0.0);  // shrink
    f[i] = v;
    nz = (v != 0.0);
  }
  const int cnt = __syncthreads_count(nz);
  if (i == 0) {
    *rank = cnt;
    if (cnt == p) atomicOr(&state->flags, PF_FLAG_SATURATED);
  }
}

cudaError_t spectral_launch(int op, double thr, const double* theta, int p, double* f, int* rank,
                            DevState* state, cudaStream_t st) {
  count_launch();
  spectral_kernel<<<1, kMaxP, 0, st>>>(op, thr, theta, p, f, rank, state);
  return cudaGetLastError();
}

// =============================================================================== plan
// Per pf_filter call: coefficients of the recurrence and the re-base schedule (reading R7).
__global__ void plan_kernel(const double* __restrict__ interval, int d, double rho_max, int p,
                            DevState* state) {
  // the spread max |theta_prev| by one warp (a serial loop of dependent global loads took ~15 us)
  double sp = 0.0;
  if (state->have_theta)
    for (int i = threadIdx.x; i < p; i += 32) sp = fmax(sp, fabs(state->theta[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sp = fmax(sp, __shfl_xor_sync(0xffffffffu, sp, o));
  if (threadIdx.x != 0) return;
  const double a = interval[0], b = interval[1];
  state->interval[0] = a;
  state->interval[1] = b;
  if (!(b > a)) {
    // degenerate interval (e.g. a PSD iterate: no eigenvalue to damp), SURVEY §8(c) reading:
    // the filter is skipped for this call -- identity recurrence Y_{j+1} = Y_j, no re-base --
    // so pf_filter returns orth(U), i.e. the previous subspace
    atomicOr(&state->flags, PF_FLAG_DEGENERATE_INT);
    for (int j = 0; j < d; ++j) {
      state->coef[j][0] = 0.0;
      state->coef[j][1] = 1.0;
      state->coef[j][2] = 0.0;
      state->rebase[j] = 0;
    }
    return;
  }
  const double c = 0.5 * (b + a), e = 0.5 * (b - a);
  double spread;
  if (state->have_theta) {
    spread = sp;
  } else if (state->have_lanczos) {
    spread = fmax(fabs(state->lanczos[0]), fabs(state->lanczos[1]));
  } else {
    spread = fmax(fabs(a), fabs(b));
  }
  const double that = fmax(1.0, fmax(fabs((1.1 * spread - c) / e), fabs((-1.1 * spread - c) / e)));
  for (int j = 0; j < d; ++j) {
    if (j == 0) {
      state->coef[0][0] = 1.0 / e;
      state->coef[0][1] = -c / e;
      state->coef[0][2] = 0.0;
    } else {
      state->coef[j][0] = 2.0 / e;
      state->coef[j][1] = -2.0 * c / e;
      state->coef[j][2] = -1.0;
    }
  }
  // T_0 .. T_d at t_hat by the three-term recurrence (t_hat >= 1: all positive, increasing);
  // the closed form's two fp64 pow() per value cost ~15 us on one thread
  double Tj[kMaxDeg + 1];
  Tj[0] = 1.0;
  Tj[1] = that;
  for (int j = 2; j <= d; ++j) Tj[j] = 2.0 * that * Tj[j - 1] - Tj[j - 2];
  int base = 0;
  for (int j = 1; j <= d; ++j) {
    int rb = 0;
    if (j < d && Tj[j] / Tj[base] > rho_max) {
      rb = 1;
      base = j;
    }
    state->rebase[j - 1] = rb;
    state->rebases += rb;
  }
}

cudaError_t plan_launch(const double* interval, int d, double rho_max, int p, DevState* state,
                        cudaStream_t st) {
  count_launch();
  plan_kernel<<<1, 32, 0, st>>>(interval, d, rho_max, p, state);
  return cudaGetLastError();
}

__global__ void interval_psd_kernel(const double* lo_hi, double eta, double* interval,
                                    DevState* state) {
  const double a = lo_hi[0];
  interval[0] = a;
  // b = eta a; a >= 0 (nothing to damp: the iterate is PSD) leaves the
  // degenerate interval [a, a], on which pf_filter skips the filter (plan_kernel)
  interval[1] = (a < 0.0) ? eta * a : a;
}

cudaError_t interval_psd_launch(const double* lo_hi, double eta, double* interval,
                                DevState* state, cudaStream_t st) {
  count_launch();
  interval_psd_kernel<<<1, 1, 0, st>>>(lo_hi, eta, interval, state);
  return cudaGetLastError();
}

// top-r interval: a = lo_hi[0], b = (1 - eta) theta_r + eta a with theta_r the r-th
// largest Ritz value of the previous Rayleigh-Ritz (state->theta, descending); without previous
// Ritz values the all-positive rule b = eta a is used (reading R22)
__global__ void interval_top_r_kernel(const double* lo_hi, int r, double eta, double* interval,
                                      DevState* state) {
  double a = lo_hi[0];
  double b = eta * a;
  if (state->have_theta) b = (1.0 - eta) * state->theta[r - 1] + eta * a;
  interval[0] = a;
  interval[1] = (b > a) ? b : a;  // degenerate -> the filter is skipped (plan_kernel)
}

cudaError_t interval_top_r_launch(const double* lo_hi, int r, double eta, double* interval,
                                  DevState* state, cudaStream_t st) {
  count_launch();
  interval_top_r_kernel<<<1, 1, 0, st>>>(lo_hi, r, eta, interval, state);
  return cudaGetLastError();
}

__global__ void interval_soft_kernel(double thr, double eta, double* interval) {
  const double beta = (1.0 - eta) * thr;
  interval[0] = -beta;
  interval[1] = beta;
}

cudaError_t interval_soft_launch(double thr, double eta, double* interval, DevState* state,
                                 cudaStream_t st) {
  (void)state;
  count_launch();
  interval_soft_kernel<<<1, 1, 0, st>>>(thr, eta, interval);
  return cudaGetLastError();
}

__global__ void copy_theta_kernel(const double* theta, int p, DevState* state, int d, int q) {
  __shared__ double red[32];
  __shared__ int n_out;
  const int i = threadIdx.x;
  if (i == 0) n_out = 0;
  __syncthreads();
  // relative gap (eqn:relative-gap) of the Ritz values beyond the damped interval
  const double a = state->interval[0], b = state->interval[1];
  const double c = 0.5 * (a + b), e = 0.5 * (b - a);
  double g = INFINITY;
  if (i < p) {
    const double t = theta[i];
    state->theta[i] = t;
    if (e > 0.0 && (t < a || t > b)) {
      g = fabs(t - c) / e - 1.0;
      atomicAdd(&n_out, 1);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) g = fmin(g, __shfl_xor_sync(0xffffffffu, g, o));
  if ((i & 31) == 0) red[i >> 5] = g;
  __syncthreads();
  if (i == 0) {
    double m = INFINITY;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmin(m, red[w]);
    state->scratch[2] = m;
    // eta_k of the wanted values (eqn:etak P:613-616, reading R28): (1 / T_d(1 + G))^q when a
    // guard Ritz value lies inside [a, b]; T_d(x) = cosh(d acosh x) for x >= 1
    double eta = NAN;
    if (d > 0 && e > 0.0 && n_out < p) eta = isinf(m) ? 0.0 : exp(-(double)q * d * acosh(1.0 + m));
    state->scratch[4] = eta;
    state->have_theta = 1;
  }
}

cudaError_t copy_theta_launch(const double* theta, int p, DevState* state, cudaStream_t st,
                              int d, int q) {
  count_launch();
  copy_theta_kernel<<<1, kMaxP, 0, st>>>(theta, p, state, d, q);
  return cudaGetLastError();
}

// =============================================================================== perturb
__global__ void perturb_kernel(double* A, int64_t lda, const double* E, int64_t lde, int rows,
                               int cols) {
  const int c = blockIdx.y * blockDim.x + threadIdx.x;  // rows on x: gridDim.y <= 65535
  const int r = blockIdx.x;
  if (c < cols && r < rows) A[(size_t)r * lda + c] += E[(size_t)r * lde + c];
}

cudaError_t perturb_launch(double* A, int64_t lda, const double* E, int64_t lde, int rows,
                           int cols, cudaStream_t st) {
  dim3 grid(rows, (cols + 255) / 256);
  count_launch();
  perturb_kernel<<<grid, 256, 0, st>>>(A, lda, E, lde, rows, cols);
  return cudaGetLastError();
}

}  // namespace pf
