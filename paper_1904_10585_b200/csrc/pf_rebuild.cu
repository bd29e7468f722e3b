// pf_rebuild.cu -- fused rank-p rebuild + elementwise update (step a6 of SURVEY §8(a)):
//   PFPG (eq:pfpg1):  X = V diag(f) V^T,  A+ = X - tau * Omega o (X - M),  M = W W^T,
//                                obj = {1/2 ||P_Omega(X - M)||_F^2, sum |f|}
//   PFAM (eq:PFAM1, prox sign corrected -- reading R1), max-cut SDP (A = diag, b = 1):
//                                W = V diag(f) V^T,
//                                Z+ = offdiag(W - tC) + Diag(1 - W_ii + Z_ii),  C = -L/4,
//                                obj = {<C, W>, ||Z+ - Z||_F}
// The low-rank products run on fp64 DMMA with the f scaling folded into the smem load; the
// masks (Omega / adjacency) are read as packed bits, so C and Omega cost n^2/8 bytes.
// Reductions are deterministic: per-CTA partials, summed in CTA order by the last CTA.
#include <algorithm>

#include "pf_kernels.cuh"

namespace pf {

constexpr int kRbTile = 64;  // 64 x 64 output tile, 4 warps (2 x 2), warp tile 32 x 32

template <int P, bool PFPG>
struct RbCfg {
  static constexpr int LD = P + 4;
  static constexpr int SMEM_V = 2 * kRbTile * LD * 8;
};

__device__ __forceinline__ bool mask_bit(const uint32_t* bits, int64_t ld, int i, int j) {
  return (__ldg(bits + (size_t)i * ld + (j >> 5)) >> (j & 31)) & 1u;
}

template <int P, bool PFPG>
__global__ void __launch_bounds__(128) rebuild_kernel(
    const double* __restrict__ V, int64_t ldv, const double* __restrict__ f, double tau_or_t,
    const uint32_t* __restrict__ bits, int64_t ldb, const double* __restrict__ W, int64_t ldw,
    int r, int ldw_s, const double* __restrict__ deg, double* Out, int64_t ldo, int n_rows, int n,
    int row0, double* __restrict__ partials, int* counter, double* __restrict__ obj) {
  using C = RbCfg<P, PFPG>;
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[32];
  __shared__ int s_last;
  double* VFi = sm;                       // 64 x LD   f-scaled rows I (local rows -> global row0+i)
  double* Vj = sm + kRbTile * C::LD;      // 64 x LD   rows J
  double* Wi = Vj + kRbTile * C::LD;      // 64 x ldw_s (PFPG)
  double* Wj = Wi + kRbTile * ldw_s;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g8 = lane >> 2, t4 = lane & 3;
  const int i0 = blockIdx.y * kRbTile;  // local row tile
  const int j0 = blockIdx.x * kRbTile;  // global column tile

  for (int e = tid; e < kRbTile * P; e += 128) {
    const int rr = e / P, c = e % P;
    const int gi = row0 + i0 + rr, gj = j0 + rr;
    VFi[rr * C::LD + c] = (i0 + rr < n_rows) ? V[(size_t)gi * ldv + c] * f[c] : 0.0;
    Vj[rr * C::LD + c] = (gj < n) ? V[(size_t)gj * ldv + c] : 0.0;
  }
  if (PFPG) {
    for (int e = tid; e < kRbTile * ldw_s; e += 128) {
      const int rr = e / ldw_s, c = e % ldw_s;
      const int gi = row0 + i0 + rr, gj = j0 + rr;
      Wi[e] = (c < r && i0 + rr < n_rows) ? W[(size_t)gi * ldw + c] : 0.0;
      Wj[e] = (c < r && gj < n) ? W[(size_t)gj * ldw + c] : 0.0;
    }
  }
  __syncthreads();

  const int wm = warp & 1, wn = warp >> 1;
  double acc[2][4][4];
  double accm[PFPG ? 2 : 1][PFPG ? 4 : 1][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[a][b][k] = 0.0;
#pragma unroll 2
  for (int ks = 0; ks < P / 4; ++ks) {
    const int k = ks * 4 + t4;
    double a0[2], a1[2], b0[4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      a0[mt] = VFi[(wm * 32 + mt * 16 + g8) * C::LD + k];
      a1[mt] = VFi[(wm * 32 + mt * 16 + g8 + 8) * C::LD + k];
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) b0[nt] = Vj[(wn * 32 + nt * 8 + g8) * C::LD + k];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) dmma16884(acc[mt][nt], a0[mt], a1[mt], b0[nt]);
  }
  if (PFPG) {
#pragma unroll
    for (int a = 0; a < (PFPG ? 2 : 1); ++a)
#pragma unroll
      for (int b = 0; b < (PFPG ? 4 : 1); ++b)
#pragma unroll
        for (int k = 0; k < 4; ++k) accm[a][b][k] = 0.0;
    for (int ks = 0; ks < (ldw_s - 4) / 4; ++ks) {
      const int k = ks * 4 + t4;
      double a0[2], a1[2], b0[4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        a0[mt] = Wi[(wm * 32 + mt * 16 + g8) * ldw_s + k];
        a1[mt] = Wi[(wm * 32 + mt * 16 + g8 + 8) * ldw_s + k];
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) b0[nt] = Wj[(wn * 32 + nt * 8 + g8) * ldw_s + k];
#pragma unroll
      for (int mt = 0; mt < (PFPG ? 2 : 1); ++mt)
#pragma unroll
        for (int nt = 0; nt < (PFPG ? 4 : 1); ++nt)
          dmma16884(accm[mt][nt], a0[mt], a1[mt], b0[nt]);
    }
  }

  // ------------------------------------------------------------------ elementwise update
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int li = i0 + wm * 32 + mt * 16 + g8 + 8 * h;  // local row
      if (li >= n_rows) continue;
      const int gi = row0 + li;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int j = j0 + wn * 32 + nt * 8 + 2 * t4;
        if (j >= n) continue;
        const bool two = (j + 1 < n);
        double* op = Out + (size_t)li * ldo + j;
        double o[2];
        if (PFPG) {
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const double x = acc[mt][nt][2 * h + c];
            const double m = accm[PFPG ? mt : 0][PFPG ? nt : 0][2 * h + c];
            const bool om = (c == 0 || two) ? mask_bit(bits, ldb, li, j + c) : false;
            const double dxm = x - m;
            o[c] = om ? x - tau_or_t * dxm : x;
            if (om) s0 += dxm * dxm;
          }
        } else {
          double zold[2];
          if (two && ((reinterpret_cast<uintptr_t>(op) & 15) == 0)) {
            const double2 z2 = *reinterpret_cast<const double2*>(op);
            zold[0] = z2.x;
            zold[1] = z2.y;
          } else {
            zold[0] = op[0];
            zold[1] = two ? op[1] : 0.0;
          }
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            if (c == 1 && !two) break;
            const int jj = j + c;
            const double w = acc[mt][nt][2 * h + c];
            double znew;
            if (jj == gi) {
              znew = 1.0 - w + zold[c];            // Diag(1 - W_ii + Z_ii)
              s0 += -0.25 * deg[gi] * w;           // C_ii = -deg_i / 4
            } else {
              const bool a = mask_bit(bits, ldb, li, jj);
              znew = a ? w - 0.25 * tau_or_t : w;  // W_ij - t C_ij, C_ij = adj_ij / 4
              if (a) s0 += 0.25 * w;
            }
            const double dz = znew - zold[c];
            s1 += dz * dz;
            o[c] = znew;
          }
        }
        if (two && ((reinterpret_cast<uintptr_t>(op) & 15) == 0)) {
          *reinterpret_cast<double2*>(op) = make_double2(o[0], o[1]);
        } else {
          op[0] = o[0];
          if (two) op[1] = o[1];
        }
      }
    }
  s0 = block_sum(s0, red);
  s1 = block_sum(s1, red);
  const int bid = blockIdx.y * gridDim.x + blockIdx.x;
  const int nb = gridDim.x * gridDim.y;
  if (tid == 0) {
    partials[2 * (size_t)bid] = s0;
    partials[2 * (size_t)bid + 1] = s1;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(counter, 1) == nb - 1);
  __syncthreads();
  if (s_last) {
    __threadfence();
    double t0 = 0.0, t1 = 0.0;
    // fixed assignment of blocks to threads + fixed tree -> deterministic
    for (int b = tid; b < nb; b += 128) {
      t0 += __ldcg(partials + 2 * (size_t)b);
      t1 += __ldcg(partials + 2 * (size_t)b + 1);
    }
    t0 = block_sum(t0, red);
    t1 = block_sum(t1, red);
    if (tid == 0) {
      if (PFPG) {
        double sf = 0.0;
        for (int c = 0; c < P; ++c) sf += fabs(f[c]);
        obj[0] = 0.5 * t0;
        obj[1] = sf;
      } else {
        obj[0] = t0;
        obj[1] = sqrt(t1);
      }
      *counter = 0;
    }
  }
}

int rebuild_blocks(int n_rows, int n) {
  return ((n + kRbTile - 1) / kRbTile) * ((n_rows + kRbTile - 1) / kRbTile);
}

template <int P, bool PFPG>
static cudaError_t rb_launch(const double* V, int64_t ldv, const double* f, double tt,
                             const uint32_t* bits, int64_t ldb, const double* W, int64_t ldw,
                             int r, const double* deg, double* Out, int64_t ldo, int n_rows,
                             int n, int row0, double* obj, double* partials, int* counter,
                             cudaStream_t st) {
  using C = RbCfg<P, PFPG>;
  const int rpad = PFPG ? ((r + 3) / 4) * 4 : 0;
  const int ldw_s = PFPG ? (rpad + 4) : 0;
  const size_t smem = C::SMEM_V + (PFPG ? (size_t)2 * kRbTile * ldw_s * 8 : 0);
  static bool attr = false;
  if (!attr) {
    const int mx = C::SMEM_V + (PFPG ? 2 * kRbTile * (64 + 4) * 8 : 0);
    cudaFuncSetAttribute(rebuild_kernel<P, PFPG>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    attr = true;
  }
  dim3 grid((n + kRbTile - 1) / kRbTile, (n_rows + kRbTile - 1) / kRbTile);
  count_launch();
  rebuild_kernel<P, PFPG><<<grid, 128, smem, st>>>(V, ldv, f, tt, bits, ldb, W, ldw, r, ldw_s, deg,
                                                   Out, ldo, n_rows, n, row0, partials, counter,
                                                   obj);
  return cudaGetLastError();
}

#define PF_RB_DISPATCH(PFPG_, ...)                                        \
  switch (p) {                                                            \
    case 16: return rb_launch<16, PFPG_>(__VA_ARGS__);                    \
    case 32: return rb_launch<32, PFPG_>(__VA_ARGS__);                    \
    case 64: return rb_launch<64, PFPG_>(__VA_ARGS__);                    \
    case 128: return rb_launch<128, PFPG_>(__VA_ARGS__);                  \
    default: return cudaErrorInvalidValue;                                \
  }

cudaError_t prox_launch(const double* V, int64_t ldv, const double* f, double tau,
                        const uint32_t* omega, int64_t ldo, const double* W, int64_t ldw, int r,
                        double* Aout, int64_t lda, int n_rows, int n, int row0, int p,
                        double* obj, double* partials, int* counter, cudaStream_t st) {
  PF_RB_DISPATCH(true, V, ldv, f, tau, omega, ldo, W, ldw, r, nullptr, Aout, lda, n_rows, n, row0,
                 obj, partials, counter, st)
}

cudaError_t admm_launch(const double* V, int64_t ldv, const double* f, double t,
                        const uint32_t* adj, int64_t ldadj, const double* deg, double* Z,
                        int64_t ldz, int n_rows, int n, int row0, int p, double* obj,
                        double* partials, int* counter, cudaStream_t st) {
  PF_RB_DISPATCH(false, V, ldv, f, t, adj, ldadj, nullptr, 0, 0, deg, Z, ldz, n_rows, n, row0,
                 obj, partials, counter, st)
}

}  // namespace pf
