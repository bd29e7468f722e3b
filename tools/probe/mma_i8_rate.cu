// mma_i8_rate.cu -- tcgen05.mma kind::i8 issue rate on B200 vs N (M = 128 single CTA, M = 256
// CTA pair), SWIZZLE_64B K-major operands (the layout of pf_gemm_i8.cu).  The leader issues
// ITERS MMAs back to back, commits and waits.  Reports cycles / MMA and int8 ops / clk / SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/probe/mma_i8_rate tools/probe/mma_i8_rate.cu
#include <cstdio>

#include "../../paper_1904_10585_b200/csrc/pf_tc.cuh"

using namespace pf;

__device__ __forceinline__ uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int CG>
__global__ void mma_rate(int iters, int N, int nmix, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* buf = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(buf + 64 * 1024);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<int*>(buf)[i] = 0x01010101;
  const int warp = threadIdx.x >> 5;
  uint32_t rank = CG == 2 ? tc::cluster_ctarank() : 0;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  fence_proxy_async();
  if (warp == 0) {
    if (CG == 2) tc::tmem_alloc_pair<512>(slot);
    else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
  }
  tc::fence_before_sync();
  if (CG == 2) tc::cluster_sync(); else __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *slot;
  if (rank == 0 && threadIdx.x == 32) {
    const uint32_t a = smem_u32(buf), b = smem_u32(buf + 32 * 1024);
    const uint32_t M = CG == 2 ? 256 : 128;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t ko = (i & 1) * 32;
      // nmix > 0: cycle through N = 64 * (1 + i % nmix) (the stacked-B mix of the GEMM)
      const int n = nmix ? 64 * (1 + i % nmix) : N;
      const uint64_t da = tc::sdesc_k_sw64(a + ko), db = tc::sdesc_k_sw64(b + ko);
      const uint32_t idesc = idesc_i8(M, n);
      if (CG == 2)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                     "l"(da), "l"(db), "r"(idesc), "r"(1));
      else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                     "l"(da), "l"(db), "r"(idesc), "r"(1));
    }
    if (CG == 2) tc::mma_commit_pair(bar);
    else asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar)));
    mbar_wait(bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  if (CG == 2 && rank == 1 && threadIdx.x == 32) mbar_wait(bar, 0);
  __syncwarp();
  tc::fence_before_sync();
  if (CG == 2) tc::cluster_sync(); else __syncthreads();
  if (warp == 0) {
    tc::fence_after_sync();
    if (CG == 2) tc::tmem_dealloc_pair<512>(tmem);
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
}

template <int CG>
void run(int N, int nmix, int grid) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 512);
  auto k = mma_rate<CG>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  const int iters = 4096;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(grid * CG);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 80 * 1024;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, iters, N, nmix, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[512];
  cudaMemcpy(h, d, sizeof(long long) * grid * CG, cudaMemcpyDeviceToHost);
  const int M = CG == 2 ? 256 : 128, K = 32;
  double cyc = (double)h[0] / iters;
  double avgN = nmix ? 64.0 * (nmix + 1) / 2 : N;
  printf("i8 cg%d M=%d N=%s%3d grid %3d: %7.1f cyc/MMA  -> %6.0f int8 ops/cyc/SM (%s)\n", CG, M,
         nmix ? "mix<=" : "", nmix ? 64 * nmix : N, grid, cyc, 2.0 * M * avgN * K / cyc / CG,
         cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int grid : {1, 148}) {
    for (int N : {64, 128, 192, 256}) run<1>(N, 0, grid);
    run<1>(0, 4, grid);
  }
  for (int grid : {1, 74})
    for (int N : {64, 128, 256}) run<2>(N, 0, grid);
  return 0;
}
