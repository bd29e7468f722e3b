// i8_mn.cu -- does tcgen05.mma kind::i8 accept an MN-major A operand, and with which descriptor
// strides?  (Needed by the half-storage symmetric filter: the lower-triangle tiles are the
// stored upper tiles read transposed.)  One CTA, one MMA M = 128, N = 64, K = 32:
//   A MN-major, SWIZZLE_64B: two 64-row chunks (m = 0..63, 64..127), each [k row][64 bytes of m],
//     chunk stride CH bytes; the swizzle XORs 16-byte chunk bits 4-5 with bits 7-8 of the offset
//   B K-major, SWIZZLE_64B: [n row][64 bytes of k] (the layout of pf_gemm_i8.cu)
// D (s32) read back from TMEM and compared with the host product, for several (LBO, SBO).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/probe/i8_mn tools/probe/i8_mn.cu
#include <cstdio>
#include <cstdlib>

#include "../../paper_1904_10585_b200/csrc/pf_tc.cuh"

using namespace pf;

__device__ __forceinline__ uint32_t swz64(uint32_t off) { return off ^ (((off >> 7) & 3u) << 4); }

__global__ void probe(const int8_t* Ah /* [128][32] m-major host copy: A[m][k] */,
                      const int8_t* Bh /* [64][32] B[n][k] */, int lbo, int sbo, int tA, int CH,
                      int* D /* [128][64] */) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* buf = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  unsigned char* A = buf;            // 2 chunks
  unsigned char* B = buf + 16384;    // 64 rows x 64 B
  uint64_t* bar = reinterpret_cast<uint64_t*>(buf + 16384 + 4096);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < (16384 + 4096) / 4; i += blockDim.x) reinterpret_cast<int*>(buf)[i] = 0;
  __syncthreads();
  for (int e = threadIdx.x; e < 128 * 32; e += blockDim.x) {
    const int m = e / 32, k = e % 32;
    uint32_t off;
    if (tA) off = swz64((uint32_t)((m >> 6) * CH + k * 64 + (m & 63)));   // MN-major
    else off = swz64((uint32_t)(m * 64 + k));                              // K-major
    A[off] = (unsigned char)Ah[e];
  }
  for (int e = threadIdx.x; e < 64 * 32; e += blockDim.x) {
    const int n = e / 32, k = e % 32;
    B[swz64((uint32_t)(n * 64 + k))] = (unsigned char)Bh[e];
  }
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  fence_proxy_async();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;\n" ::"r"(smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *slot;
  if (warp == 1) {
    if (tc::elect_one()) {
      uint64_t ad = 0;
      const uint32_t sa = smem_u32(A);
      ad |= (uint64_t)((sa >> 4) & 0x3FFFu);
      ad |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
      ad |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
      ad |= (uint64_t)1u << 46;
      ad |= (uint64_t)4u << 61;  // SWIZZLE_64B
      const uint64_t bd = tc::sdesc_k_sw64(smem_u32(B));
      const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)tA << 15) |
                             ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                   "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                   "l"(ad), "l"(bd), "r"(idesc), "r"(0));
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar)));
    }
    __syncwarp();
  }
  mbar_wait(bar, 0);
  tc::fence_after_sync();
  {
    const int lane = threadIdx.x & 31, row = 32 * warp + lane;
    for (int c = 0; c < 64; c += 32) {
      float v[32];
      tc::tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + c, v);
      for (int j = 0; j < 32; ++j) D[row * 64 + c + j] = __float_as_int(v[j]);
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;\n" ::"r"(tmem));
  }
}

int main() {
  int8_t hA[128 * 32], hB[64 * 32];
  srand(1);
  for (auto& x : hA) x = (int8_t)(rand() % 255 - 127);
  for (auto& x : hB) x = (int8_t)(rand() % 255 - 127);
  int ref[128 * 64];
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 64; ++n) {
      int s = 0;
      for (int k = 0; k < 32; ++k) s += hA[m * 32 + k] * hB[n * 32 + k];
      ref[m * 64 + n] = s;
    }
  int8_t *dA, *dB;
  int* dD;
  cudaMalloc(&dA, sizeof(hA));
  cudaMalloc(&dB, sizeof(hB));
  cudaMalloc(&dD, sizeof(ref));
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 24 * 1024);
  struct V { int tA, CH, lbo, sbo; } vs[] = {
      {0, 0, 16, 512},                                   // K-major control
      {1, 4096, 4096, 512}, {1, 4096, 512, 4096},        // MN-major, chunks 4 KB apart
      {1, 2048, 2048, 512}, {1, 2048, 512, 2048},        // chunks 2 KB apart (K = 32 rows)
      {1, 8192, 8192, 512}, {1, 8192, 512, 8192}};
  for (auto v : vs) {
    cudaMemset(dD, 0xff, sizeof(ref));
    probe<<<1, 128, 24 * 1024>>>(dA, dB, v.lbo, v.sbo, v.tA, v.CH, dD);
    cudaError_t e = cudaDeviceSynchronize();
    int h[128 * 64];
    cudaMemcpy(h, dD, sizeof(h), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < 128 * 64; ++i) bad += h[i] != ref[i];
    printf("tA=%d chunk=%5d LBO=%5d SBO=%5d: %5d / 8192 wrong (%s)\n", v.tA, v.CH, v.lbo, v.sbo,
           bad, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
