// i8_seq.cu -- cycles per K = 32 step of the K1-i8 MMA sequence issued the way pf_gemm_i8.cu
// issues it (the whole warp runs the loop, one elected lane issues; operands at the kernel's
// smem offsets, no TMA), single CTA vs CTA pair:
//   mode 0  cta_group::1, M = 128: A_s x stacked [B_0 .. B_{6-s}], N = 64 (7 - s) split at 256
//           (10 MMAs per step, 1792 columns)
//   mode 1  cta_group::2, M = 256: the same 10 MMAs, each CTA supplying its 128 rows of A and
//           HALF of the N rows of B (per-MMA B regions laid out so both halves share an offset)
//   mode 2  cta_group::1, 7 MMAs of N = 256 with a new A slice each (same column count)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/probe/i8_seq tools/probe/i8_seq.cu
#include <cstdio>

#include "../../paper_1904_10585_b200/csrc/pf_tc.cuh"

using namespace pf;

__device__ __forceinline__ uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
template <int CG>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id) {
  if (CG == 2)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(id), "r"(1));
  else
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(id), "r"(1));
}

// B-row offsets (in 64-byte rows) and N of the 10 MMAs per K step; mode 1: region offsets of
// this CTA's half (both CTAs use the same offset)
struct Seq {
  int s[10], brow[10], n[10], col[10];
};

template <int CG>
__global__ void seq(int steps, int mode, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* buf = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  unsigned char* A = buf;                // 7 x 8 KB
  unsigned char* B = buf + 7 * 8192;     // up to 512 rows x 64 B = 32 KB
  uint64_t* bar = reinterpret_cast<uint64_t*>(buf + 7 * 8192 + 32768);
  uint64_t* done = bar + 1;   // completed phase 0: waits on it return at once
  uint64_t* sink = bar + 2;   // commits land here (never completes)
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 3);
  for (int i = threadIdx.x; i < (7 * 8192 + 32768) / 4; i += blockDim.x)
    reinterpret_cast<int*>(buf)[i] = 0x01010101;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = CG == 2 ? tc::cluster_ctarank() : 0;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(done, 1);
    mbar_init(sink, (1u << 20) - 1);
    fence_mbar_init();
    mbar_arrive(done);
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
  // the sequences
  Seq q;
  int nm = 0;
  if (mode == 0) {
    for (int s = 0; s < 7; ++s)
      for (int t0 = 0; t0 < 7 - s; t0 += 4) {
        const int c = min(4, 7 - s - t0);
        q.s[nm] = s; q.brow[nm] = 64 * t0; q.n[nm] = 64 * c; q.col[nm] = 64 * (s + t0); ++nm;
      }
  } else if (mode == 1) {
    // regions (rows per CTA): Ra 128 [B0B1|B2B3], Rb 96 [B4 B5a|B5b B6], Rc 64 [B4|B5],
    // Rd 32 [B4a|B4b], Re 96 [B0 B1a|B1b B2], Rf 64 [B0|B1], Rg 32 [B0a|B0b]
    const int Ra = 0, Rb = 128, Rc = 224, Rd = 288, Re = 320, Rf = 416, Rg = 480;
    const int reg1[7] = {Rb, Rc, Rd, -1, -1, -1, -1};
    const int n1[7] = {192, 128, 64, 0, 0, 0, 0};
    const int reg0[7] = {Ra, Ra, Ra, Ra, Re, Rf, Rg};
    const int n0[7] = {256, 256, 256, 256, 192, 128, 64};
    for (int s = 0; s < 7; ++s) {
      q.s[nm] = s; q.brow[nm] = reg0[s]; q.n[nm] = n0[s]; q.col[nm] = 64 * s; ++nm;
      if (reg1[s] >= 0) { q.s[nm] = s; q.brow[nm] = reg1[s]; q.n[nm] = n1[s]; q.col[nm] = 64 * (s + 4); ++nm; }
    }
  } else if (mode == 2) {
    for (int s = 0; s < 7; ++s) { q.s[nm] = s; q.brow[nm] = 0; q.n[nm] = 256; q.col[nm] = 0; ++nm; }
  } else {  // mode 3: mode 0 with an MN-major A (transpose bit, LBO 4096, SBO 512)
    for (int s = 0; s < 7; ++s)
      for (int t0 = 0; t0 < 7 - s; t0 += 4) {
        const int c = min(4, 7 - s - t0);
        q.s[nm] = s; q.brow[nm] = 64 * t0; q.n[nm] = 64 * c; q.col[nm] = 64 * (s + t0); ++nm;
      }
  }
  const bool tr = mode == 3;
  if (mode >= 4 && mode < 10) {  // mode 0's sequence with the kernel's per-slice (4) / per-k-block (5) sync
    for (int s = 0; s < 7; ++s)
      for (int t0 = 0; t0 < 7 - s; t0 += 4) {
        const int c = min(4, 7 - s - t0);
        q.s[nm] = s; q.brow[nm] = 64 * t0; q.n[nm] = 64 * c; q.col[nm] = 64 * (s + t0); ++nm;
      }
  }
  const uint32_t M = CG == 2 ? 256 : 128;
  if (rank == 0 && warp == 1) {
    const uint32_t a0 = smem_u32(A), b0 = smem_u32(B);
    long long t0 = clock64();
    if (mode >= 4 && mode < 10) {
      // per k-block (2 K steps): for each slice s: [wait + fence], MMAs of ks = 0, 1, [commit]
      for (int kb = 0; kb < steps / 2; ++kb) {
        if (mode == 5 || mode == 9) {
          mbar_wait(done, 0);
          if (mode == 5) tc::fence_after_sync();
        }
#pragma unroll
        for (int s = 0; s < 7; ++s) {
          // 4: wait + fence + commit per slice (the kernel); 6: wait + commit per slice, no
          // fence; 7: wait per slice (no fence), commit per k-block; 8: wait + commit per
          // slice pair {0,1},{2,3},{4,5},{6}; 9: wait + commit per k-block, no fence
          if (mode == 4 || mode == 6 || mode == 7 || (mode == 8 && (s & 1) == 0)) {
            mbar_wait(done, 0);
            if (mode == 4) tc::fence_after_sync();
          }
          if (tc::elect_one()) {
#pragma unroll
            for (int ks = 0; ks < 2; ++ks)
#pragma unroll
              for (int t0 = 0; t0 < 7 - s; t0 += 4) {
                const int c = min(4, 7 - s - t0);
                mma<CG>(tmem + (uint32_t)((64 * (s + t0)) % 256),
                        tc::sdesc_k_sw64(a0 + s * 8192 + ks * 32),
                        tc::sdesc_k_sw64(b0 + 64 * t0 * 64 + ks * 32), idesc_i8(M, 64 * c));
              }
            if (mode == 4 || mode == 6 || (mode == 8 && ((s & 1) == 1 || s == 6)))
              asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(sink)));
          }
          __syncwarp();
        }
        if ((mode == 5 || mode == 7 || mode == 9) && tc::elect_one())
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(sink)));
        __syncwarp();
      }
    }
    if (mode >= 10) {
      // 10: one wait per k-block, every MMA of the k-block inside ONE elected block (s, ks, t0)
      // 11: as 10 in the K-step-outer order (ks, s, t0)
      // 12: per-slice wait + commit by the elected lane alone (no warp sync between slices)
      for (int kb = 0; kb < steps / 2; ++kb) {
        if (mode != 12) mbar_wait(done, 0);
        if (tc::elect_one()) {
          if (mode == 11) {
#pragma unroll
            for (int ks = 0; ks < 2; ++ks)
#pragma unroll
              for (int s = 0; s < 7; ++s)
#pragma unroll
                for (int t0 = 0; t0 < 7 - s; t0 += 4) {
                  const int c = min(4, 7 - s - t0);
                  mma<CG>(tmem + (uint32_t)((64 * (s + t0)) % 256),
                          tc::sdesc_k_sw64(a0 + s * 8192 + ks * 32),
                          tc::sdesc_k_sw64(b0 + 64 * t0 * 64 + ks * 32), idesc_i8(M, 64 * c));
                }
          } else {
#pragma unroll
            for (int s = 0; s < 7; ++s) {
              if (mode == 12) mbar_wait(done, 0);
#pragma unroll
              for (int ks = 0; ks < 2; ++ks)
#pragma unroll
                for (int t0 = 0; t0 < 7 - s; t0 += 4) {
                  const int c = min(4, 7 - s - t0);
                  mma<CG>(tmem + (uint32_t)((64 * (s + t0)) % 256),
                          tc::sdesc_k_sw64(a0 + s * 8192 + ks * 32),
                          tc::sdesc_k_sw64(b0 + 64 * t0 * 64 + ks * 32), idesc_i8(M, 64 * c));
                }
              if (mode == 12)
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(sink)));
            }
          }
          if (mode != 12)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(sink)));
        }
        __syncwarp();
      }
    }
    for (int k = 0; k < (mode >= 4 ? 0 : steps); ++k) {
      const uint32_t ko = (k & 1) * 32;
      if (tc::elect_one()) {
#pragma unroll
        for (int i = 0; i < 10; ++i) {
          if (i < nm) {
            const uint32_t ncols = (uint32_t)q.n[i];
            const uint64_t ad = tr ? ((tc::sdesc_k_sw64(a0 + q.s[i] * 8192 + ko * 64) &
                                       ~(0x3FFFull << 16)) | ((uint64_t)(4096 >> 4) << 16))
                                   : tc::sdesc_k_sw64(a0 + q.s[i] * 8192 + ko);
            mma<CG>(tmem + (uint32_t)(q.col[i] % 256), ad,
                    tc::sdesc_k_sw64(b0 + q.brow[i] * 64 + ko),
                    idesc_i8(M, ncols) | (tr ? (1u << 15) : 0u));
          }
        }
      }
      __syncwarp();
    }
    if (tc::elect_one()) {
      if (CG == 2) tc::mma_commit_pair(bar);
      else asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar)));
    }
    __syncwarp();
    mbar_wait(bar, 0);
    long long t1 = clock64();
    if (tc::elect_one()) {
      out[2 * blockIdx.x] = t1 - t0;
      out[2 * blockIdx.x + 1] = mode >= 4 ? 10 : nm;
    }
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
void run(int mode, int clusters) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 1024);
  auto k = seq<CG>;
  const int smem = 7 * 8192 + 32768 + 2048;  // + barriers
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int steps = 4096;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(clusters * CG);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, steps, mode, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[2];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double cyc = (double)h[0] / steps;
  // int8 ops per SM per step: 28 slice products x 128 rows x 64 cols x 32 K x 2 (per 128 rows)
  const double ops = (mode == 2 ? 7.0 * 256 : 1792.0) * 128 * 32 * 2;
  printf("mode %d cg%d %3d clusters: %7.1f cyc per K=32 step (per 128 rows), %4.1f MMAs, "
         "%6.0f int8 ops/cyc/SM (%s)\n", mode, CG, clusters, cyc, (double)h[1], ops / cyc,
         cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<1>(0, 148);
  for (int m = 4; m <= 12; ++m) run<1>(m, 148);
  run<2>(1, 74);
  return 0;
}
