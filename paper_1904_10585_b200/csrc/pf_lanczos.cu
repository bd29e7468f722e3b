// pf_lanczos.cu -- m-step Lanczos with full re-orthogonalisation (CGS2) for the interval end a
// (the paper's `eigs` for lambda_n; reading R5).  Vectors are row blocks of n_local
// rows (pitch ldq); the matrix-vector product reads the local rows of A against the full
// (all-gathered) Lanczos vector, so every step is one HBM pass over the local block of A.
// Each phase produces LOCAL partial sums (dots, norms) reduced deterministically inside the
// kernel; the host all-reduces them between phases when the context is distributed.
#include <algorithm>

#include "pf_kernels.cuh"
#include "../../include/pf.h"

namespace pf {

constexpr int kLzThreads = 256;

int lanczos_blocks(int n_rows) { return std::max(1, std::min(4 * 148, (n_rows + 7) / 8)); }

__device__ bool last_block_done(int* counter, int* s_last) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int prev = atomicAdd(counter, 1);
    *s_last = (prev == (int)gridDim.x - 1);
  }
  __syncthreads();
  return *s_last != 0;
}

// deterministic warp reduction of partials[b * kMaxLanczos + i] over b (fixed lane stride + tree)
__device__ __forceinline__ double warp_reduce_partials(const double* partials, int nb, int i) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int b = lane; b < nb; b += 32) s += __ldcg(partials + (size_t)b * kMaxLanczos + i);
  return warp_sum(s);
}

// s[0] = sum of squares of the local rows of v
__global__ void lz_norm2_kernel(const double* __restrict__ v, int n_local, double* s) {
  __shared__ double red[32];
  double a = 0.0;
  for (int i = threadIdx.x; i < n_local; i += blockDim.x) a += v[i] * v[i];
  a = block_sum(a, red);
  if (threadIdx.x == 0) s[0] = a;
}

// q0 = v0 / sqrt(s[0]) (s = global sum of squares); marks the Lanczos run as active
__global__ void lz_start_kernel(const double* __restrict__ v0, int n_local, const double* s,
                                double* q, DevState* state) {
  const double inv = 1.0 / sqrt(s[0]);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_local; i += gridDim.x * blockDim.x)
    q[i] = v0[i] * inv;
  if (blockIdx.x == 0 && threadIdx.x == 0) state->lanczos_steps = -1;  // running
}

cudaError_t lz_start_launch(const double* v0, int n_local, double* s, double* q0,
                            DevState* state, cudaStream_t st, bool norm_only) {
  if (norm_only) {
    count_launch();
    lz_norm2_kernel<<<1, 1024, 0, st>>>(v0, n_local, s);
  } else {
    count_launch();
    lz_start_kernel<<<std::max(1, std::min(148, (n_local + 255) / 256)), 256, 0, st>>>(
        v0, n_local, s, q0, state);
  }
  return cudaGetLastError();
}

// w = A_local q_full (one HBM pass over the local rows of A), then local partial dots
// h_i = Q_i . w (i <= j) reduced in block order by the last block.
// two consecutive entries of a row of A as doubles (streaming load: A is read once per step)
__device__ __forceinline__ double2 lz_ld2(const double* p) {
  return __ldcs(reinterpret_cast<const double2*>(p));
}
__device__ __forceinline__ double2 lz_ld2(const float* p) {
  const float2 f = __ldcs(reinterpret_cast<const float2*>(p));
  return make_double2((double)f.x, (double)f.y);
}

template <typename TA>
__global__ void __launch_bounds__(kLzThreads, 4) lz_gemv_kernel(
    const TA* __restrict__ A, int64_t lda, int n_local, int n, const double* __restrict__ q,
    const double* __restrict__ Q, int64_t ldq, int j, double* __restrict__ w,
    double* __restrict__ h, double* __restrict__ partials, int* counter, DevState* state) {
  if (state->lanczos_steps >= 0) return;  // stopped (breakdown)
  __shared__ double ws[64];
  __shared__ int s_last;
  __shared__ double red2[2][kLzThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = kLzThreads / 32;
  const int rows_per = (n_local + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * rows_per, r1 = min(n_local, r0 + rows_per);
  // All 8 warps cooperate on each pair of rows (warp w owns the column segment w): every warp
  // has the same work, 8 independent 16-byte streaming loads of A per lane are in flight, and
  // the warp's segment of q stays in L1 (A is read once with .cs).
  const int seg = (((n + nw - 1) / nw) + 1) & ~1;
  const int c0 = min(n, warp * seg), c1 = min(n, c0 + seg);
  for (int r = r0; r < r1; r += 2) {
    const bool two = (r + 1 < r1);
    const TA* a0 = A + (size_t)r * lda;
    const TA* a1 = A + (size_t)(two ? r + 1 : r) * lda;
    double s0 = 0.0, s1 = 0.0;
    int c = c0 + lane * 2;
    for (; c + 64 * 3 + 1 < c1; c += 64 * 4) {
      double2 x0[4], x1[4], y[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        x0[u] = lz_ld2(a0 + c + 64 * u);
        x1[u] = lz_ld2(a1 + c + 64 * u);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) y[u] = __ldg(reinterpret_cast<const double2*>(q + c + 64 * u));
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        s0 += x0[u].x * y[u].x + x0[u].y * y[u].y;
        s1 += x1[u].x * y[u].x + x1[u].y * y[u].y;
      }
    }
    for (; c < c1; c += 64) {
      s0 += (double)a0[c] * q[c];
      s1 += (double)a1[c] * q[c];
      if (c + 1 < c1) {
        s0 += (double)a0[c + 1] * q[c + 1];
        s1 += (double)a1[c + 1] * q[c + 1];
      }
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    if (lane == 0) {
      red2[0][warp] = s0;
      red2[1][warp] = s1;
    }
    __syncthreads();
    if (threadIdx.x < 2 && (threadIdx.x == 0 || two)) {
      double s = 0.0;
      for (int u = 0; u < nw; ++u) s += red2[threadIdx.x][u];  // fixed order: deterministic
      const int rr = r + threadIdx.x;
      w[rr] = s;
      if (rr - r0 < 64) ws[rr - r0] = s;
    }
    __syncthreads();
  }
  // partial dots with Q_0..Q_j over this block's rows (one warp per vector)
  for (int i = warp; i <= j; i += nw) {
    const double* qi = Q + (size_t)i * ldq;
    double s = 0.0;
    for (int r = r0 + lane; r < r1; r += 32) s += qi[r] * ((r - r0 < 64) ? ws[r - r0] : w[r]);
    s = warp_sum(s);
    if (lane == 0) partials[(size_t)blockIdx.x * kMaxLanczos + i] = s;
  }
  if (last_block_done(counter, &s_last)) {
    __threadfence();
    for (int i = warp; i <= j; i += nw) {
      const double s = warp_reduce_partials(partials, (int)gridDim.x, i);
      if (lane == 0) h[i] = s;
    }
    if (threadIdx.x == 0) *counter = 0;
  }
}

// ---- symmetric GEMV (fp64, one GPU): w = A q from the upper triangle only -- half the HBM
// bytes of lz_gemv_kernel (A is symmetric: the PFPG / PFAM iterates are written with exact
// mirrors).  Pass 1: persistent CTAs walk contiguous ranges of the 64 x 64 tiles (I <= J) of
// the upper triangle; tile (I, J) yields A_IJ q_J (rows of I) and, for I < J, A_IJ^T q_I (rows of
// J), written as 64-vectors to ws (no atomics).  Pass 2 sums, for every row block R, the T
// contributions in a fixed order, then the partial dots with Q_0..Q_j as lz_gemv_kernel.
constexpr int kSyT = 64;

__device__ __forceinline__ long long sym_tile_index(int I, int J, int T) {
  return (long long)I * T - (long long)I * (I - 1) / 2 + (J - I);
}

__device__ __forceinline__ void sym_pair_of(long long e, int T, int& I, int& J) {
  const double b = 2.0 * T + 1.0;
  int i = (int)floor((b - sqrt(b * b - 8.0 * (double)e)) * 0.5);
  if (i < 0) i = 0;
  while (i > 0 && sym_tile_index(i, i, T) > e) --i;
  while (i + 1 < T && sym_tile_index(i + 1, i + 1, T) <= e) ++i;
  I = i;
  J = i + (int)(e - sym_tile_index(i, i, T));
}

// 16-byte cp.async with zero fill past src_bytes (0, 8 or 16)
__device__ __forceinline__ void lz_cp16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes)
               : "memory");
}

// tile (I, J) of A -> smem stage (64 x 64, row-major): 2048 16-byte chunks, 8 per thread,
// coalesced (a warp copies one 512-byte row); entries past n are zero-filled
__device__ __forceinline__ void sym_issue(const double* __restrict__ A, int64_t lda, int n, int I,
                                          int J, double* stage, int tid) {
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int ch = tid + 256 * u, r = ch >> 5, c = (ch & 31) * 2;
    const int row = I * kSyT + r, col = J * kSyT + c;
    const int bytes = (row < n) ? max(0, min(2, n - col)) * 8 : 0;
    const double* src = bytes ? A + (size_t)row * lda + col : A;
    lz_cp16(stage + r * kSyT + c, src, bytes);
  }
}

constexpr int kSyStages = 2;  // tiles in flight per CTA (3 CTAs / SM: 6 x 32 KB per SM)

// thread t: rows 4 (t / 16) .. +3 and columns {2c, 2c + 1, 32 + 2c, 33 + 2c}, c = t % 16
__global__ void __launch_bounds__(256, 3) lz_symv_tiles_kernel(
    const double* __restrict__ A, int64_t lda, int n, const double* __restrict__ q,
    double* __restrict__ ws, DevState* state) {
  if (state->lanczos_steps >= 0) return;
  extern __shared__ __align__(16) double sy_smem[];
  __shared__ double red[8][kSyT];
  const int T = (n + kSyT - 1) / kSyT;
  const long long nt = (long long)T * (T + 1) / 2;
  const long long t0 = nt * blockIdx.x / gridDim.x, t1 = nt * (blockIdx.x + 1) / gridDim.x;
  const int tid = threadIdx.x, rg = tid >> 4, cc = tid & 15, warp = tid >> 5, lane = tid & 31;
  if (t0 >= t1) return;
  // prologue: the first kSyStages - 1 tiles in flight
  int In, Jn;  // next tile to issue
  sym_pair_of(t0, T, In, Jn);
  auto advance = [&](int& I, int& J) {
    if (++J == T) {
      ++I;
      J = I;
    }
  };
  long long issued = t0;
#pragma unroll
  for (int s = 0; s < kSyStages - 1; ++s) {
    if (issued < t1) {
      sym_issue(A, lda, n, In, Jn, sy_smem + (size_t)(s) * kSyT * kSyT, tid);
      advance(In, Jn);
      ++issued;
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  int I, J;
  sym_pair_of(t0, T, I, J);
  for (long long t = t0; t < t1; ++t) {
    const int k = (int)((t - t0) % kSyStages);
    __syncthreads();  // the stage about to be refilled was read by every thread (tile t - 1)
    if (issued < t1) {
      sym_issue(A, lda, n, In, Jn,
                sy_smem + (size_t)((k + kSyStages - 1) % kSyStages) * kSyT * kSyT, tid);
      advance(In, Jn);
      ++issued;
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group %0;\n" ::"n"(kSyStages - 1) : "memory");
    __syncthreads();
    const double* tl = sy_smem + (size_t)k * kSyT * kSyT;
    const int i0 = I * kSyT, j0 = J * kSyT;
    double qc[4], qr[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = j0 + 2 * cc + (u & 1) + 32 * (u >> 1), r = i0 + 4 * rg + u;
      qc[u] = c < n ? __ldg(q + c) : 0.0;
      qr[u] = r < n ? __ldg(q + r) : 0.0;
    }
    double rs[4], cs[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const double* rowp = tl + (4 * rg + rr) * kSyT + 2 * cc;
      const double2 v0 = *reinterpret_cast<const double2*>(rowp);
      const double2 v1 = *reinterpret_cast<const double2*>(rowp + 32);
      rs[rr] = ((v0.x * qc[0] + v0.y * qc[1]) + v1.x * qc[2]) + v1.y * qc[3];
      cs[0] += v0.x * qr[rr];
      cs[1] += v0.y * qr[rr];
      cs[2] += v1.x * qr[rr];
      cs[3] += v1.y * qr[rr];
    }
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) rs[rr] += __shfl_xor_sync(0xffffffffu, rs[rr], o);
    }
    double* wrow = ws + (size_t)t * (2 * kSyT);
    if (cc == 0) {
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) __stcg(wrow + 4 * rg + rr, rs[rr]);
    }
    if (I < J) {  // column sums: the two row groups of a warp, then the 8 warps in order
#pragma unroll
      for (int u = 0; u < 4; ++u) cs[u] += __shfl_xor_sync(0xffffffffu, cs[u], 16);
      if (lane < 16) {
#pragma unroll
        for (int u = 0; u < 4; ++u) red[warp][2 * cc + (u & 1) + 32 * (u >> 1)] = cs[u];
      }
      __syncthreads();
      if (tid < kSyT) {
        double v = 0.0;
#pragma unroll
        for (int w8 = 0; w8 < 8; ++w8) v += red[w8][tid];
        __stcg(wrow + kSyT + tid, v);
      }
      // red is rewritten only after the next tile's two barriers
    }
    advance(I, J);
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// w_i = sum_{J >= R} ws_row[(R, J)]_i + sum_{I < R} ws_col[(I, R)]_i (R = i / 64, fixed order),
// then the partial dots h_i = Q_i . w as lz_gemv_kernel
__global__ void __launch_bounds__(kLzThreads) lz_symv_reduce_kernel(
    int n, const double* __restrict__ ws, const double* __restrict__ Q, int64_t ldq, int j,
    double* __restrict__ w, double* __restrict__ h, double* __restrict__ partials, int* counter,
    DevState* state) {
  if (state->lanczos_steps >= 0) return;
  __shared__ double part[8][32];
  __shared__ double wsm[32];
  __shared__ int s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = kLzThreads / 32;
  const int T = (n + kSyT - 1) / kSyT;
  const int rows_per = (n + gridDim.x - 1) / gridDim.x;  // <= 32 (lanczos_blocks)
  const int r0 = blockIdx.x * rows_per, r1 = min(n, r0 + rows_per);
  const int i = r0 + lane;
  double s = 0.0;
  if (lane < rows_per && i < r1) {
    const int R = i / kSyT, ii = i - R * kSyT;
#pragma unroll 8
    for (int K = warp; K < T; K += nw) {  // independent loads, summed in K order
      const long long t = K >= R ? sym_tile_index(R, K, T) : sym_tile_index(K, R, T);
      s += __ldcg(ws + (size_t)t * (2 * kSyT) + (K >= R ? 0 : kSyT) + ii);
    }
  }
  part[warp][lane] = s;
  __syncthreads();
  if (warp == 0) {
    double v = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) v += part[u][lane];
    wsm[lane] = v;
    if (lane < rows_per && i < r1) w[i] = v;
  }
  __syncthreads();
  for (int k = warp; k <= j; k += nw) {
    const double* qk = Q + (size_t)k * ldq;
    double d = (lane < rows_per && i < r1) ? qk[i] * wsm[lane] : 0.0;
    d = warp_sum(d);
    if (lane == 0) partials[(size_t)blockIdx.x * kMaxLanczos + k] = d;
  }
  if (last_block_done(counter, &s_last)) {
    __threadfence();
    for (int k = warp; k <= j; k += nw) {
      const double v = warp_reduce_partials(partials, (int)gridDim.x, k);
      if (lane == 0) h[k] = v;
    }
    if (threadIdx.x == 0) *counter = 0;
  }
}

size_t lz_symv_ws_doubles(int n) {
  const long long T = (n + kSyT - 1) / kSyT;
  return (size_t)(T * (T + 1) / 2) * 2 * kSyT;
}

cudaError_t lz_symv_launch(const double* A, int64_t lda, int n, const double* q, const double* Q,
                           int64_t ldq, int j, double* w, double* h, double* ws,
                           double* partials, int* counter, DevState* state, int num_sms,
                           cudaStream_t st) {
  const long long T = (n + kSyT - 1) / kSyT, nt = T * (T + 1) / 2;
  const int grid = (int)std::max(1LL, std::min(nt, 3LL * num_sms));
  const size_t smem = (size_t)kSyStages * kSyT * kSyT * 8;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(lz_symv_tiles_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = true;
  }
  count_launch();
  lz_symv_tiles_kernel<<<grid, 256, smem, st>>>(A, lda, n, q, ws, state);
  count_launch();
  lz_symv_reduce_kernel<<<lanczos_blocks(n), kLzThreads, 0, st>>>(n, ws, Q, ldq, j, w, h,
                                                                   partials, counter, state);
  return cudaGetLastError();
}

// w -= Q h (local rows); phase 1: local partial dots -> out[0..j]; phase 2: local |w|^2 -> out[0]
__global__ void __launch_bounds__(kLzThreads) lz_orth_kernel(
    int n_local, const double* __restrict__ Q, int64_t ldq, int j, double* __restrict__ w,
    const double* __restrict__ h, double* __restrict__ out, double* __restrict__ partials,
    int* counter, DevState* state, int phase) {
  if (state->lanczos_steps >= 0) return;
  __shared__ double hs[kMaxLanczos];
  __shared__ int s_last;
  __shared__ double red[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = kLzThreads / 32;
  for (int i = threadIdx.x; i <= j; i += blockDim.x) hs[i] = h[i];
  if (phase == 1 && blockIdx.x == 0 && threadIdx.x == 0)
    state->lanczos_alpha[j] = h[j];  // alpha_j = q_j . A q_j (global after the all-reduce)
  __syncthreads();
  const int rows_per = (n_local + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * rows_per, r1 = min(n_local, r0 + rows_per);
  if (rows_per <= 32) {
    // lane = row, warp = vectors i = warp (mod 8): the j + 1 loads per row run in parallel; the
    // 8 warp partials are combined in a fixed order
    __shared__ double pq[kLzThreads / 32][32];
    const int r = r0 + lane;
    double v = 0.0;
    if (r < r1)
      for (int i = warp; i <= j; i += nw) v += Q[(size_t)i * ldq + r] * hs[i];
    pq[warp][lane] = v;
    __syncthreads();
    if (warp == 0 && r < r1) {
      double sum = 0.0;
#pragma unroll
      for (int u = 0; u < kLzThreads / 32; ++u) sum += pq[u][lane];
      w[r] -= sum;
    }
  } else {
    for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
      double v = w[r];
      for (int i = 0; i <= j; ++i) v -= Q[(size_t)i * ldq + r] * hs[i];
      w[r] = v;
    }
  }
  __syncthreads();
  if (phase == 1) {
    for (int i = warp; i <= j; i += nw) {
      const double* qi = Q + (size_t)i * ldq;
      double s = 0.0;
      for (int r = r0 + lane; r < r1; r += 32) s += qi[r] * w[r];
      s = warp_sum(s);
      if (lane == 0) partials[(size_t)blockIdx.x * kMaxLanczos + i] = s;
    }
  } else {
    double s = 0.0;
    for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) s += w[r] * w[r];
    s = block_sum(s, red);
    if (threadIdx.x == 0) partials[(size_t)blockIdx.x * kMaxLanczos] = s;
  }
  if (last_block_done(counter, &s_last)) {
    __threadfence();
    if (phase == 1) {
      for (int i = warp; i <= j; i += nw) {
        const double s = warp_reduce_partials(partials, (int)gridDim.x, i);
        if (lane == 0) out[i] = s;
      }
    } else if (warp == 0) {
      const double s = warp_reduce_partials(partials, (int)gridDim.x, 0);
      if (lane == 0) out[0] = s;
    }
    if (threadIdx.x == 0) *counter = 0;
  }
}

// beta_j = sqrt(s) with the breakdown test of reading R5, then q_{j+1} = w / beta_j
__global__ void lz_next_kernel(int n_local, double* Q, int64_t ldq, int j, const double* w,
                               const double* s, DevState* state) {
  __shared__ int s_stop;
  if (state->lanczos_steps >= 0) return;
  const double beta = sqrt(s[0]);
  if (threadIdx.x == 0) {
    double amax = 1.0;
    for (int i = 0; i <= j; ++i) amax = fmax(amax, fabs(state->lanczos_alpha[i]));
    s_stop = (beta <= 1e-12 * amax);
  }
  __syncthreads();
  if (s_stop) {
    // every block reaches the same decision from the same (all-reduced) s; block 0 records it
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      state->lanczos_beta[j] = 0.0;
      atomicOr(&state->flags, PF_FLAG_LANCZOS_BREAK);
    }
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) state->lanczos_beta[j] = beta;
  const double inv = 1.0 / beta;
  double* q = Q + (size_t)(j + 1) * ldq;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_local; r += gridDim.x * blockDim.x)
    q[r] = w[r] * inv;
}

// the stop flag is applied after the step in a separate single-thread kernel so no block of
// lz_next reads a half-updated lanczos_steps
__global__ void lz_commit_kernel(int j, DevState* state) {
  if (state->lanczos_steps >= 0) return;
  if (state->lanczos_beta[j] == 0.0) state->lanczos_steps = j + 1;
}

cudaError_t lz_gemv_launch(const double* A, int64_t lda, int n_local, int n, const double* q,
                           const double* Q, int64_t ldq, int j, double* w, double* h,
                           double* partials, int* counter, DevState* state, cudaStream_t st) {
  count_launch();
  lz_gemv_kernel<double><<<lanczos_blocks(n_local), kLzThreads, 0, st>>>(
      A, lda, n_local, n, q, Q, ldq, j, w, h, partials, counter, state);
  return cudaGetLastError();
}

cudaError_t lz_gemv_f32_launch(const float* A, int64_t lda, int n_local, int n, const double* q,
                               const double* Q, int64_t ldq, int j, double* w, double* h,
                               double* partials, int* counter, DevState* state, cudaStream_t st) {
  count_launch();
  lz_gemv_kernel<float><<<lanczos_blocks(n_local), kLzThreads, 0, st>>>(
      A, lda, n_local, n, q, Q, ldq, j, w, h, partials, counter, state);
  return cudaGetLastError();
}

cudaError_t lz_orth_launch(int n_local, const double* Q, int64_t ldq, int j, double* w,
                           const double* h, double* out, double* partials, int* counter,
                           DevState* state, int phase, cudaStream_t st) {
  count_launch();
  lz_orth_kernel<<<lanczos_blocks(n_local), kLzThreads, 0, st>>>(n_local, Q, ldq, j, w, h, out,
                                                                 partials, counter, state, phase);
  return cudaGetLastError();
}

cudaError_t lz_next_launch(int n_local, double* Q, int64_t ldq, int j, const double* w,
                           const double* s, DevState* state, cudaStream_t st) {
  count_launch();
  lz_next_kernel<<<std::max(1, std::min(148, (n_local + 255) / 256)), 256, 0, st>>>(n_local, Q, ldq,
                                                                                   j, w, s, state);
  count_launch();
  lz_commit_kernel<<<1, 1, 0, st>>>(j, state);
  return cudaGetLastError();
}

// build T (m_eff x m_eff) from alpha/beta; m_eff is written to a device int for the Jacobi
__global__ void lanczos_T_kernel(int m, double* T, DevState* state, int* m_out) {
  int me = state->lanczos_steps;
  if (me < 0) me = m;  // ran all m steps
  if (threadIdx.x == 0) *m_out = me;
  for (int e = threadIdx.x; e < me * me; e += blockDim.x) {
    const int i = e / me, k = e % me;
    double v = 0.0;
    if (i == k) v = state->lanczos_alpha[i];
    else if (k == i + 1) v = state->lanczos_beta[i];
    else if (i == k + 1) v = state->lanczos_beta[k];
    T[e] = v;
  }
}

// lo = theta_min - |beta_last s_{last,min}|, hi = theta_max + |beta_last s_{last,max}|
__global__ void lanczos_extremes_kernel(const double* theta, const double* S, const int* m_dev,
                                        double* lo_hi, DevState* state) {
  const int me = *m_dev;
  const double bl = state->lanczos_beta[me - 1];
  const double rmin = fabs(bl * S[(me - 1) * me + (me - 1)]);
  const double rmax = fabs(bl * S[(me - 1) * me + 0]);
  const double lo = theta[me - 1] - rmin, hi = theta[0] + rmax;
  lo_hi[0] = lo;
  lo_hi[1] = hi;
  state->lanczos[0] = lo;
  state->lanczos[1] = hi;
  state->have_lanczos = 1;
  state->lanczos_steps = me;
}

// v = Q_me s_min: the Ritz vector of the smallest Ritz value (the warm start of the next refresh,
// NEXT-2 lambda_min tracking); S row-major me x me, columns by descending theta
__global__ void lz_ritz_vector_kernel(const double* __restrict__ Q, int64_t ldq, int n_local,
                                      const double* __restrict__ S, const int* m_dev,
                                      double* __restrict__ v) {
  const int me = *m_dev;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_local; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < me; ++j) s += Q[(size_t)j * ldq + i] * S[j * me + me - 1];
    v[i] = s;
  }
}

cudaError_t lz_ritz_vector_launch(const double* Q, int64_t ldq, int n_local, const double* S,
                                  const DevState* state, double* v, cudaStream_t st) {
  const int* m_dev = reinterpret_cast<const int*>(&state->scratch[0]);
  count_launch();
  lz_ritz_vector_kernel<<<std::max(1, std::min(296, (n_local + 255) / 256)), 256, 0, st>>>(
      Q, ldq, n_local, S, m_dev, v);
  return cudaGetLastError();
}

cudaError_t lanczos_finish_launch(int m, double* T, double* theta, double* S, double* lo_hi,
                                  DevState* state, cudaStream_t st) {
  int* m_dev = reinterpret_cast<int*>(&state->scratch[0]);
  count_launch();
  lanczos_T_kernel<<<1, 256, 0, st>>>(m, T, state, m_dev);
  cudaError_t e = jacobi_launch(T, m, m_dev, theta, S, state, 1e-15, 40, st);
  if (e != cudaSuccess) return e;
  count_launch();
  lanczos_extremes_kernel<<<1, 1, 0, st>>>(theta, S, m_dev, lo_hi, state);
  return cudaGetLastError();
}

}  // namespace pf
