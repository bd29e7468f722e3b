// pf_common.cuh -- sm_100a device primitives shared by the PF kernels:
// fp64 DMMA (mma.sync m16n8k4 .f64 -> SASS DMMA.8x8x4), mbarrier, TMA (cp.async.bulk.tensor),
// named barriers and warp reductions.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define PF_DEV __device__ __forceinline__

namespace pf {

constexpr int kMaxP = 512;
constexpr int kMaxDeg = 64;
constexpr int kMaxLanczos = 64;

// Device-resident state of one context (written by the plan / RR / Lanczos kernels).
struct DevState {
  double interval[2];          // a, b in use by the last pf_filter
  double lanczos[2];           // lo, hi of the last Lanczos
  double coef[kMaxDeg][3];     // per Chebyshev step: out = s1*(A Y) + s2*Ycur + s3*Yprev
  int rebase[kMaxDeg];         // 1: re-base (Y_j, Y_{j-1}) after step j (index j-1)
  double theta[kMaxP];         // Ritz values of the last Rayleigh-Ritz (descending)
  int have_theta;              // theta valid
  int have_lanczos;            // lanczos valid
  unsigned int flags;          // PF_FLAG_* bits
  int rebases;                 // re-base count since last status read
  int chol_shift;              // current CholeskyQR pass used a shift -> extra pass needed
  int lanczos_steps;           // Lanczos steps actually taken (breakdown)
  double lanczos_alpha[kMaxLanczos];
  double lanczos_beta[kMaxLanczos];
  double coef_rr[3];          // {1, 0, 0}: plain A Q for Rayleigh-Ritz
  double scratch[8];
};

// ------------------------------------------------------------------------------ DMMA
// D(16x8) += A(16x4, row) * B(4x8, col), fp64.  Fragment ownership (lane = 4*g + t):
//   a0 = A[g][t], a1 = A[g+8][t]; b0 = B[t][g];
//   c0 = C[g][2t], c1 = C[g][2t+1], c2 = C[g+8][2t], c3 = C[g+8][2t+1].
PF_DEV void dmma16884(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// ------------------------------------------------------------------------------ mbarrier
PF_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

PF_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
PF_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::); }
PF_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::); }

PF_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
PF_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
PF_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// ------------------------------------------------------------------------------ TMA
PF_DEV void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
// 2-D tile load: coordinates (c0 = innermost element index, c1 = row index).
PF_DEV void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];\n" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// ------------------------------------------------------------------------------ barriers
PF_DEV void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

PF_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide deterministic sum (fixed tree); all threads get the result. blockDim multiple of 32.
PF_DEV double block_sum(double v, double* red /* >= 32 doubles smem */) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = lane < nw ? red[lane] : 0.0;
    r = warp_sum(r);
    if (lane == 0) red[0] = r;
  }
  __syncthreads();
  r = red[0];
  __syncthreads();
  return r;
}

// Chebyshev T_d(t) closed form (eq:cheb) for the re-base plan (device copy of the scalar rule).
PF_DEV double cheb_T(int d, double t) {
  if (fabs(t) <= 1.0) return cos(d * acos(t));
  double s = sqrt(t * t - 1.0);
  return 0.5 * (pow(t - s, (double)d) + pow(t + s, (double)d));
}

}  // namespace pf
