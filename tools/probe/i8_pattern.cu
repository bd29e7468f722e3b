// i8_pattern.cu -- cycles per k-step of the MMA sequences pf_gemm_i8.cu can issue (no TMA, static
// shared-memory operands at the real offsets): S = 7 A slices (distinct 8 KB tiles), B = stacked
// 64-column slices.  mode 0: one MMA per A slice over all its B slices (N = 64 (7 - s), split at
// 256 -- mixed N); mode 1: uniform N = 128 windows; mode 2: uniform N = 256 windows (TMEM
// overflow ignored: timing only); mode 3: one N = 64 MMA per (s, t) pair.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/probe/i8_pattern tools/probe/i8_pattern.cu
#include <cstdio>

#include "../../paper_1904_10585_b200/csrc/pf_tc.cuh"

using namespace pf;

__device__ __forceinline__ uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(1));
}

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, int sw) {
  if (sw == 64) return tc::sdesc_k_sw64(saddr);
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | (1ull << 16) | ((uint64_t)(1024u >> 4) << 32) |
         (1ull << 46) | (2ull << 61);   // SWIZZLE_128B, 8-row groups 1 KB apart
}

__global__ void pattern(int ksteps, int mode, int sw, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* buf = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  const int S = 7;
  const int at = sw == 64 ? 8192 : 16384, bt = sw == 64 ? 4096 : 8192;   // tile strides
  unsigned char* A = buf;                 // 7 A tiles
  unsigned char* B = buf + 7 * 16384;     // 10 B slice tiles
  uint64_t* bar = reinterpret_cast<uint64_t*>(buf + 7 * 16384 + 10 * 8192);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < (7 * 16384 + 10 * 8192) / 4; i += blockDim.x)
    reinterpret_cast<int*>(buf)[i] = 0x01010101;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  fence_proxy_async();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *slot;
  if (threadIdx.x == 32) {
    const uint32_t a0 = smem_u32(A), b0 = smem_u32(B);
    long long nmma = 0;
    long long t0 = clock64();
    for (int k = 0; k < ksteps; ++k) {
      const uint32_t ko = (k & (sw == 64 ? 1 : 3)) * 32;
      for (int s = 0; s < S; ++s) {
        const uint64_t ad = sdesc(a0 + s * at + ko, sw);
        if (mode == 0) {
          for (int t0 = 0; t0 < S - s; t0 += 4) {
            const int c = min(4, S - s - t0);
            mma(tmem + (s + t0) * 64, ad, sdesc(b0 + t0 * bt + ko, sw), idesc_i8(128, 64 * c));
            ++nmma;
          }
        } else if (mode == 1) {
          for (int t0 = 0; t0 < S - s; t0 += 2) {
            mma(tmem + (s + t0) * 64, ad, sdesc(b0 + t0 * bt + ko, sw), idesc_i8(128, 128));
            ++nmma;
          }
        } else if (mode == 2) {
          for (int t0 = 0; t0 < S - s; t0 += 4) {
            mma(tmem + ((s + t0) % 4) * 64, ad, sdesc(b0 + t0 * bt + ko, sw), idesc_i8(128, 256));
            ++nmma;
          }
        } else if (mode == 4) {        // A changes per MMA, B fixed: N = 256
          mma(tmem + (s % 2) * 256, ad, sdesc(b0 + ko, sw), idesc_i8(128, 256));
          ++nmma;
        } else if (mode == 5) {        // A fixed, B window changes: N = 256
          mma(tmem + (s % 2) * 256, sdesc(a0 + ko, sw), sdesc(b0 + (s % 4) * bt + ko, sw),
              idesc_i8(128, 256));
          ++nmma;
        } else if (mode == 6) {        // both fixed: N = 256
          mma(tmem + (s % 2) * 256, sdesc(a0 + ko, sw), sdesc(b0 + ko, sw), idesc_i8(128, 256));
          ++nmma;
        } else if (mode == 7) {        // A changes, B fixed, same TMEM region
          mma(tmem, ad, sdesc(b0 + ko, sw), idesc_i8(128, 256));
          ++nmma;
        } else {
          for (int t = 0; t < S - s; ++t) {
            mma(tmem + (s + t) * 64, ad, sdesc(b0 + t * bt + ko, sw), idesc_i8(128, 64));
            ++nmma;
          }
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar)));
    mbar_wait(bar, 0);
    long long t1 = clock64();
    out[2 * blockIdx.x] = t1 - t0;
    out[2 * blockIdx.x + 1] = nmma;
  }
  __syncwarp();
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 512);
  const int smem = 7 * 16384 + 10 * 8192 + 2048;
  cudaFuncSetAttribute(pattern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[8] = {"mixed N (stacked, <=256)", "uniform N=128", "uniform N=256", "N=64 per pair",
                          "A changes, B fixed N=256", "A fixed, B changes N=256", "both fixed N=256",
                          "A changes, 1 TMEM region"};
  for (int sw : {64})
    for (int mode = 0; mode < 8; ++mode) {
      const int grid = 148;
      const int ksteps = 512;
      pattern<<<grid, 128, smem>>>(ksteps, mode, sw, d);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[2];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("sw%d grid %3d %-26s: %7.1f cyc/k-step, %5.1f MMAs/k-step, %6.1f cyc/MMA (%s)\n", sw, grid,
             names[mode], (double)h[0] / ksteps, (double)h[1] / ksteps, (double)h[0] / h[1],
             cudaGetErrorString(e));
    }
  return 0;
}
