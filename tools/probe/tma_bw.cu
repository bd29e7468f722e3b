// tma_bw.cu -- TMA load throughput vs box shape on B200 (design probe for the TF32 filter GEMM).
// One CTA per SM streams a disjoint row band of a large fp32 matrix through a ring of smem
// stages (1 producer lane issues cp.async.bulk.tensor.2d, 1 consumer warp waits and frees).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/probe/tma_bw \
//   tools/probe/tma_bw.cu paper_1904_10585_b200/csrc/pf_gemm.cu -lcuda
#include <cstdio>
#include <cstdlib>

#include "../../paper_1904_10585_b200/csrc/pf_kernels.cuh"

namespace pf {
void count_launch() {}
bool encode_map_f32(CUtensorMap* map, const float* base, int64_t pitch, int rows, int cols,
                    int box_rows, int box_cols, bool swizzle);
}  // namespace pf
using namespace pf;

__global__ void __launch_bounds__(64, 1)
    tma_stream(const __grid_constant__ CUtensorMap map, int rows_per_cta, int box_rows,
               int box_cols, int cols, int stages, int stage_bytes) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* buf = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(buf + stages * stage_bytes);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int r0 = blockIdx.x * rows_per_cta;
  const int nrb = rows_per_cta / box_rows, ncb = cols / box_cols;
  const int total = nrb * ncb;
  int s = 0;
  uint32_t ph = 0;
  if (warp == 0) {
    if (lane == 0)
      for (int i = 0; i < total; ++i) {
        mbar_wait(&empty[s], ph ^ 1u);
        mbar_arrive_expect_tx(&full[s], stage_bytes);
        // walk K (columns) fastest inside a row band, like the GEMM's A tiles
        const int rb = i / ncb, cb = i % ncb;
        tma_load_2d(buf + s * stage_bytes, &map, &full[s], cb * box_cols, r0 + rb * box_rows);
        if (++s == stages) { s = 0; ph ^= 1u; }
      }
  } else {
    for (int i = 0; i < total; ++i) {
      mbar_wait(&full[s], ph);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == stages) { s = 0; ph ^= 1u; }
    }
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int cols = 16384, rows = 148 * 256;  // 2.3 GiB fp32
  float* A;
  cudaMalloc(&A, sizeof(float) * (size_t)rows * cols);
  cudaMemset(A, 0, sizeof(float) * (size_t)rows * cols);
  struct Case { int bc, br; bool sw; } cases[] = {
      {16, 128, true}, {16, 256, true}, {32, 128, false}, {32, 256, false}, {64, 128, false},
      {16, 128, false}, {8, 256, false}};
  cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  for (auto c : cases) {
    for (int ring_kb : {48, 96, 192}) {
      CUtensorMap map;
      if (!encode_map_f32(&map, A, cols, rows, cols, c.br, c.bc, c.sw)) {
        printf("encode fail %d %d\n", c.bc, c.br);
        continue;
      }
      const int sb = c.bc * c.br * 4;
      const int stages = ring_kb * 1024 / sb;
      if (stages < 2) continue;
      const int smem = stages * sb + 1024 + 16 * stages + 64;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      tma_stream<<<sms, 64, smem>>>(map, 256, c.br, c.bc, cols, stages, sb);
      cudaEventRecord(e0);
      for (int r = 0; r < 3; ++r) tma_stream<<<sms, 64, smem>>>(map, 256, c.br, c.bc, cols, stages, sb);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 3;
      double bytes = (double)sms * 256 * cols * 4;
      printf("box %3d x %3d %s ring %3d KB (%2d stages of %5d B): %7.1f GB/s  (%5.1f B/cyc/SM @1.965GHz) %s\n",
             c.bc * 4, c.br, c.sw ? "sw64" : "none", ring_kb, stages, sb, bytes / ms * 1e-6,
             bytes / ms * 1e-6 / sms / 1.965, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
