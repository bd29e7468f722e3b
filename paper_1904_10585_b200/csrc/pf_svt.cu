// pf_svt.cu -- sparse kernels of polynomial-filtered SVT (PFSVT, NEXT-3; paper §5.2, eqn:svt
// P:1098-1104, Example eg:MC P:1120-1126): the iterate Y = A*(x) is the n x n sparse matrix with
// the dual values x on the sampled set Omega, so the filter on Y^T Y is two sparse
// x dense products per Chebyshev step, and the SVT update needs the sampled entries of the
// low-rank W = U diag(s) V^T.  All of it is HBM / L2-gather bound:
//   * spmm_kernel: out = s1 * (S X) + s2 * Ycur + s3 * Yprev, S in compressed-row form (CSR, or
//     the CSC view of the same Omega for S^T with values addressed through perm), X n x p
//     row-major; a group of min(p, 32) lanes per row, each lane owning p / 32 columns, the row's
//     nonzeros walked in storage order (deterministic), X rows gathered as contiguous p-vectors.
//   * svt_sample_kernel: w_e = sum_l U_{i_e l} s_l V_{j_e l} for every e in Omega (SDDMM), the
//     dual update x_e += delta (b_e - w_e) and the residual sum of squares, one warp per sampled
//     row with (U s)_i in registers, V rows gathered coalesced, warp-shuffle dots; residual
//     partials per block, summed in block order by the last block (deterministic).
//   * svt_sigma_kernel: sigma = sqrt(max(lambda, 0)) of the Rayleigh-Ritz eigenvalues, shrink
//     s = (sigma - mu)_+, svp = #{s > 0}, 1 / sigma for the left vectors.
#include <algorithm>

#include "pf_kernels.cuh"

namespace pf {

template <int P>
__global__ void __launch_bounds__(256) spmm_kernel(int rows, const int* __restrict__ ptr,
                                                   const int* __restrict__ idx,
                                                   const double* __restrict__ val,
                                                   const int* __restrict__ vperm,
                                                   const double* __restrict__ X, int64_t ldx,
                                                   double s1, double s2, double s3,
                                                   const double* __restrict__ ycur, int64_t ldc,
                                                   const double* __restrict__ yprev, int64_t ldp,
                                                   double* __restrict__ out, int64_t ldo) {
  constexpr int TPR = P < 32 ? P : 32;  // lanes per row
  constexpr int CPL = P / TPR;          // columns per lane
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int row = gt / TPR, l = gt % TPR;
  if (row >= rows) return;
  double acc[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) acc[c] = 0.0;
  const int e0 = ptr[row], e1 = ptr[row + 1];
  int e = e0;
  for (; e + 2 <= e1; e += 2) {  // two nonzeros in flight
    const int j0 = __ldg(idx + e), j1 = __ldg(idx + e + 1);
    const double v0 = __ldg(val + (vperm ? __ldg(vperm + e) : e));
    const double v1 = __ldg(val + (vperm ? __ldg(vperm + e + 1) : e + 1));
    const double* x0 = X + (int64_t)j0 * ldx + l;
    const double* x1 = X + (int64_t)j1 * ldx + l;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      acc[c] = fma(v0, __ldg(x0 + c * TPR), acc[c]);
      acc[c] = fma(v1, __ldg(x1 + c * TPR), acc[c]);
    }
  }
  if (e < e1) {
    const int j0 = __ldg(idx + e);
    const double v0 = __ldg(val + (vperm ? __ldg(vperm + e) : e));
    const double* x0 = X + (int64_t)j0 * ldx + l;
#pragma unroll
    for (int c = 0; c < CPL; ++c) acc[c] = fma(v0, __ldg(x0 + c * TPR), acc[c]);
  }
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int col = l + c * TPR;
    double y = s1 * acc[c];
    if (s2 != 0.0) y = fma(s2, ycur[(int64_t)row * ldc + col], y);
    if (s3 != 0.0) y = fma(s3, yprev[(int64_t)row * ldp + col], y);
    out[(int64_t)row * ldo + col] = y;
  }
}

// one warp per sampled row i; lanes hold (U s)_{i, lane + 32 c}
template <int P>
__global__ void __launch_bounds__(256) svt_sample_kernel(
    int rows, const int* __restrict__ ptr, const int* __restrict__ idx,
    const double* __restrict__ b, double* __restrict__ x, const double* __restrict__ U,
    int64_t ldu, const double* __restrict__ V, int64_t ldv, const double* __restrict__ s,
    double delta, double* __restrict__ partials, int* __restrict__ counter, double* obj) {
  constexpr int CPL = (P + 31) / 32;
  __shared__ double red[8];
  __shared__ bool last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + warp;
  double rss = 0.0;
  if (row < rows) {
    double us[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int col = lane + 32 * c;
      us[c] = (col < P) ? U[(int64_t)row * ldu + col] * s[col] : 0.0;
    }
    const int e0 = ptr[row], e1 = ptr[row + 1];
    for (int e = e0; e < e1; ++e) {
      const int j = __ldg(idx + e);
      const double* v = V + (int64_t)j * ldv;
      double d = 0.0;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int col = lane + 32 * c;
        if (col < P) d = fma(us[c], __ldg(v + col), d);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      if (lane == 0) {
        const double r = b[e] - d;
        x[e] = fma(delta, r, x[e]);
        rss = fma(r, r, rss);
      }
    }
  }
  if (lane == 0) red[warp] = rss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    partials[blockIdx.x] = t;
    __threadfence();
    last = (atomicAdd(counter, 1) == (int)gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {  // fixed-order sum of the block partials
    __threadfence();
    double t = 0.0;
    for (int k = 0; k < (int)gridDim.x; ++k) t += __ldcg(partials + k);
    obj[0] = t;
    *counter = 0;
  }
}

__global__ void svt_sigma_kernel(const double* lam, int p, double mu, double* sigma, double* s,
                                 double* inv, int* svp) {
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < p; i += blockDim.x) {
    const double sg = sqrt(fmax(lam[i], 0.0));
    sigma[i] = sg;
    const double sh = fmax(sg - mu, 0.0);
    s[i] = sh;
    inv[i] = sg > 0.0 ? 1.0 / sg : 0.0;
    if (sh > 0.0) atomicAdd(&cnt, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) *svp = cnt;
}

__global__ void scale_cols_inplace_kernel(double* X, int64_t ldx, int rows, int p,
                                          const double* d) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)rows * p) return;
  const int r = (int)(i / p), c = (int)(i % p);
  X[(int64_t)r * ldx + c] *= d[c];
}

// ------------------------------------------------------------------------------ host side
template <int P>
static cudaError_t spmm_p(int rows, const int* ptr, const int* idx, const double* val,
                          const int* vperm, const double* X, int64_t ldx, const double* coef,
                          const double* ycur, int64_t ldc, const double* yprev, int64_t ldp,
                          double* out, int64_t ldo, cudaStream_t st) {
  constexpr int TPR = P < 32 ? P : 32;
  const long long threads = (long long)rows * TPR;
  count_launch();
  spmm_kernel<P><<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(
      rows, ptr, idx, val, vperm, X, ldx, coef[0], coef[1], coef[2], ycur, ldc, yprev, ldp, out,
      ldo);
  return cudaGetLastError();
}

cudaError_t spmm_launch(int rows, int p, const int* ptr, const int* idx, const double* val,
                        const int* vperm, const double* X, int64_t ldx, const double* coef,
                        const double* ycur, int64_t ldc, const double* yprev, int64_t ldp,
                        double* out, int64_t ldo, cudaStream_t st) {
  switch (p) {
    case 16: return spmm_p<16>(rows, ptr, idx, val, vperm, X, ldx, coef, ycur, ldc, yprev, ldp, out, ldo, st);
    case 32: return spmm_p<32>(rows, ptr, idx, val, vperm, X, ldx, coef, ycur, ldc, yprev, ldp, out, ldo, st);
    case 64: return spmm_p<64>(rows, ptr, idx, val, vperm, X, ldx, coef, ycur, ldc, yprev, ldp, out, ldo, st);
    case 128: return spmm_p<128>(rows, ptr, idx, val, vperm, X, ldx, coef, ycur, ldc, yprev, ldp, out, ldo, st);
    default: return cudaErrorInvalidValue;
  }
}

int svt_sample_blocks(int rows) { return (rows + 7) / 8; }

cudaError_t svt_sample_launch(int rows, int p, const int* ptr, const int* idx, const double* b,
                              double* x, const double* U, int64_t ldu, const double* V,
                              int64_t ldv, const double* s, double delta, double* partials,
                              int* counter, double* obj, cudaStream_t st) {
  const int g = svt_sample_blocks(rows);
  count_launch();
  switch (p) {
    case 16: svt_sample_kernel<16><<<g, 256, 0, st>>>(rows, ptr, idx, b, x, U, ldu, V, ldv, s, delta, partials, counter, obj); break;
    case 32: svt_sample_kernel<32><<<g, 256, 0, st>>>(rows, ptr, idx, b, x, U, ldu, V, ldv, s, delta, partials, counter, obj); break;
    case 64: svt_sample_kernel<64><<<g, 256, 0, st>>>(rows, ptr, idx, b, x, U, ldu, V, ldv, s, delta, partials, counter, obj); break;
    case 128: svt_sample_kernel<128><<<g, 256, 0, st>>>(rows, ptr, idx, b, x, U, ldu, V, ldv, s, delta, partials, counter, obj); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t svt_sigma_launch(const double* lam, int p, double mu, double* sigma, double* s,
                             double* inv, int* svp, cudaStream_t st) {
  count_launch();
  svt_sigma_kernel<<<1, 128, 0, st>>>(lam, p, mu, sigma, s, inv, svp);
  return cudaGetLastError();
}

cudaError_t scale_cols_inplace_launch(double* X, int64_t ldx, int rows, int p, const double* d,
                                      cudaStream_t st) {
  const long long t = (long long)rows * p;
  count_launch();
  scale_cols_inplace_kernel<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(X, ldx, rows, p, d);
  return cudaGetLastError();
}

// x = alpha b (SVT's kick, pf_svt_kick)
__global__ void svt_kick_kernel(double* __restrict__ x, const double* __restrict__ b, double alpha,
                                int64_t nnz) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    x[e] = alpha * b[e];
}

cudaError_t svt_kick_launch(double* x, const double* b, double alpha, int64_t nnz,
                            cudaStream_t st) {
  if (nnz == 0) return cudaSuccess;
  count_launch();
  const int grid = (int)std::min<int64_t>((nnz + 255) / 256, 4096);
  svt_kick_kernel<<<grid, 256, 0, st>>>(x, b, alpha, nnz);
  return cudaGetLastError();
}

}  // namespace pf
