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
// [-1, 1]), stopped when ||X^2 - I||_F <= tol; each step is two p x p fp64 GEMMs (cuBLAS DGEMM:
// plain library GEMMs) and one elementwise kernel.  The iteration count grows like
// log(||M|| / min |lambda(M)|): eigenvalues close to the threshold are slow, so the host loop
// caps it and the caller falls back to Jacobi (PF_ERR_BREAKDOWN) when it does not converge.
#include <cublas_v2.h>

#include <cmath>
#include <cstdlib>

#include "pf_kernels.cuh"

namespace pf {

// X = (H - shift I), and the max absolute row sum of it into *nrm (one block per 32 rows)
__global__ void ns_shift_kernel(const double* __restrict__ H, int p, double shift,
                                double* __restrict__ X, unsigned long long* nrm_bits) {
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= p) return;
  double s = 0.0;
  for (int c = lane; c < p; c += 32) {
    const double v = H[(size_t)r * p + c] - (r == c ? shift : 0.0);
    X[(size_t)r * p + c] = v;
    s += fabs(v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) atomicMax(nrm_bits, (unsigned long long)__double_as_longlong(s));
}

__global__ void ns_scale_kernel(double* __restrict__ X, int n, const unsigned long long* nrm_bits) {
  const double nrm = __longlong_as_double((long long)*nrm_bits);
  const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    X[i] *= inv;
}

// T <- 3 I - T (T = X^2), and res = ||X^2 - I||_F^2 (fixed-order: per-block partials, last block)
__global__ void ns_prep_kernel(double* __restrict__ T, int p, double* __restrict__ part,
                               int* counter, double* res) {
  __shared__ double red[32];
  __shared__ bool last;
  double s = 0.0;
  const int n = p * p;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const bool diag = (i / p) == (i % p);
    const double t = T[i];
    const double d = t - (diag ? 1.0 : 0.0);
    s += d * d;
    T[i] = (diag ? 3.0 : 0.0) - t;
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s;
    __threadfence();
    last = (atomicAdd(counter, 1) == (int)gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double t = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) t += __ldcg(part + b);
    *res = t;
    *counter = 0;
  }
}

// rank = #{f != 0} from the traces of the sign matrices
__global__ void ns_rank_kernel(int p, const double* __restrict__ Sp, const double* __restrict__ Sm,
                               int soft, int* rank) {
  __shared__ double red[32];
  double tr = 0.0;
  for (int i = threadIdx.x; i < p; i += blockDim.x)
    tr += soft ? 0.5 * (1.0 + Sp[(size_t)i * p + i]) + 0.5 * (1.0 - Sm[(size_t)i * p + i])
               : 0.5 * (1.0 + Sp[(size_t)i * p + i]);
  tr = block_sum(tr, red);
  if (threadIdx.x == 0) *rank = (int)llrint(tr);
}

// F <- (F + F^T) / 2: one thread per element pair i < j (grid-wide)
__global__ void ns_symmetrize_kernel(double* __restrict__ F, int p) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= p * p) return;
  const int i = e / p, j = e - i * p;
  if (i < j) {
    const double v = 0.5 * (F[(size_t)i * p + j] + F[(size_t)j * p + i]);
    F[(size_t)i * p + j] = v;
    F[(size_t)j * p + i] = v;
  }
}

struct NsWork {
  cublasHandle_t h = nullptr;
  double *X = nullptr, *T = nullptr, *Y = nullptr, *Sp = nullptr, *Sm = nullptr, *M = nullptr;
  double* part = nullptr;
  int* cnt = nullptr;
  double* res = nullptr;                 // device
  unsigned long long* nrm = nullptr;     // device
  double* res_host = nullptr;            // pinned
  int p = 0;
  int last_it[2] = {0, 0};               // iterations the previous call's signs needed
};

NsWork* ns_create(int p) {
  NsWork* w = new NsWork();
  w->p = p;
  const size_t mb = (size_t)p * p * 8;
  bool ok = cublasCreate(&w->h) == CUBLAS_STATUS_SUCCESS;
  ok = ok && cudaMalloc(&w->X, mb) == cudaSuccess && cudaMalloc(&w->T, mb) == cudaSuccess &&
       cudaMalloc(&w->Y, mb) == cudaSuccess && cudaMalloc(&w->Sp, mb) == cudaSuccess &&
       cudaMalloc(&w->Sm, mb) == cudaSuccess && cudaMalloc(&w->M, mb) == cudaSuccess &&
       cudaMalloc(&w->part, 64 * 8) == cudaSuccess && cudaMalloc(&w->cnt, 16) == cudaSuccess &&
       cudaMalloc(&w->res, 8) == cudaSuccess && cudaMalloc(&w->nrm, 8) == cudaSuccess &&
       cudaMallocHost(&w->res_host, 8) == cudaSuccess &&
       cudaMemset(w->cnt, 0, 16) == cudaSuccess;
  if (!ok) {
    ns_destroy(w);
    return nullptr;
  }
  return w;
}

void ns_destroy(NsWork* w) {
  if (!w) return;
  if (w->h) cublasDestroy(w->h);
  for (void* q : {(void*)w->X, (void*)w->T, (void*)w->Y, (void*)w->Sp, (void*)w->Sm, (void*)w->M,
                  (void*)w->part, (void*)w->cnt, (void*)w->res, (void*)w->nrm})
    if (q) cudaFree(q);
  if (w->res_host) cudaFreeHost(w->res_host);
  delete w;
}

// row-major C = alpha A B + beta C (p x p) with column-major cuBLAS: C^T = alpha B^T A^T + beta C^T
static bool dgemm(NsWork* w, const double* A, const double* B, double* C, double alpha,
                  double beta) {
  const int p = w->p;
  return cublasDgemm(w->h, CUBLAS_OP_N, CUBLAS_OP_N, p, p, p, &alpha, B, p, A, p, &beta, C, p) ==
         CUBLAS_STATUS_SUCCESS;
}

// S = sign(H - shift I); returns the iterations used, -1 if not converged within max_it
static int ns_sign(NsWork* w, const double* H, double shift, double* S, int max_it, double tol,
                   int slot, cudaStream_t st) {
  const int p = w->p, n = p * p;
  cudaMemsetAsync(w->nrm, 0, 8, st);
  count_launch();
  ns_shift_kernel<<<(p + 7) / 8, 256, 0, st>>>(H, p, shift, w->X, w->nrm);
  count_launch();
  ns_scale_kernel<<<64, 256, 0, st>>>(w->X, n, w->nrm);
  double* X = w->X;
  double* Xn = S;
  for (int it = 1; it <= max_it; ++it) {
    if (!dgemm(w, X, X, w->T, 1.0, 0.0)) return -2;  // T = X^2
    count_launch();
    ns_prep_kernel<<<64, 256, 0, st>>>(w->T, p, w->part, w->cnt, w->res);  // T = 3I - X^2
    if (!dgemm(w, X, w->T, Xn, 0.5, 0.0)) return -2;  // X <- X (3I - X^2) / 2
    double* t = X;
    X = Xn;
    Xn = t;
    // ||X_prev^2 - I|| measured before this step.  Each check is a host sync: the first one
    // comes where the previous call (a nearby H in a sweep) converged, then every 2 steps
    const int first = w->last_it[slot] > 2 ? w->last_it[slot] - 1 : 8;
    if ((it >= first && ((it - first) & 1) == 0) || it == max_it) {
      cudaMemcpyAsync(w->res_host, w->res, 8, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      if (sqrt(*w->res_host) <= tol) {
        if (X != S) cudaMemcpyAsync(S, X, (size_t)n * 8, cudaMemcpyDeviceToDevice, st);
        w->last_it[slot] = it;
        return it;
      }
    }
  }
  w->last_it[slot] = 0;
  return -1;
}

// F = f(H) (row-major p x p, ld p), rank (device int); iterations (host) for diagnostics.
// Returns 0, -1 (not converged: use Jacobi), -2 (cuBLAS failure)
int ns_spectral(NsWork* w, const double* H, int op_soft, double thr, double* F, int* rank,
                int* iters, cudaStream_t st) {
  const int p = w->p;
  int max_it = 100;
  if (const char* e = getenv("PF_NS_MAXIT")) max_it = atoi(e);  // development / test knob
  const double tol = 1e-12 * sqrt((double)p);
  if (cublasSetStream(w->h, st) != CUBLAS_STATUS_SUCCESS) return -2;
  cublasSetMathMode(w->h, CUBLAS_DEFAULT_MATH);  // fp64 arithmetic, no emulation
  int it1, it2 = 0;
  if (op_soft) {
    it1 = ns_sign(w, H, thr, w->Sp, max_it, tol, 0, st);
    if (it1 < 0) return it1;
    it2 = ns_sign(w, H, -thr, w->Sm, max_it, tol, 1, st);
    if (it2 < 0) return it2;
    // F = H + ((H - thr I) S+ - (H + thr I) S-) / 2
    cudaMemcpyAsync(F, H, (size_t)p * p * 8, cudaMemcpyDeviceToDevice, st);
    cudaMemsetAsync(w->nrm, 0, 8, st);
    count_launch();
    ns_shift_kernel<<<(p + 7) / 8, 256, 0, st>>>(H, p, thr, w->M, w->nrm);    // H - thr I
    if (!dgemm(w, w->M, w->Sp, F, 0.5, 1.0)) return -2;
    count_launch();
    ns_shift_kernel<<<(p + 7) / 8, 256, 0, st>>>(H, p, -thr, w->M, w->nrm);   // H + thr I
    if (!dgemm(w, w->M, w->Sm, F, -0.5, 1.0)) return -2;
  } else {
    it1 = ns_sign(w, H, 0.0, w->Sp, max_it, tol, 0, st);
    if (it1 < 0) return it1;
    // F = (H + H S) / 2
    cudaMemcpyAsync(F, H, (size_t)p * p * 8, cudaMemcpyDeviceToDevice, st);
    if (!dgemm(w, H, w->Sp, F, 0.5, 0.5)) return -2;
  }
  count_launch();
  ns_rank_kernel<<<1, 512, 0, st>>>(p, w->Sp, w->Sm, op_soft, rank);
  count_launch();
  ns_symmetrize_kernel<<<(p * p + 255) / 256, 256, 0, st>>>(F, p);
  if (iters) *iters = it1 + it2;
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

}  // namespace pf
