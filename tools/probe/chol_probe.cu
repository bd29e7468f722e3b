// chol_probe.cu -- phase timing of chol_inv_big (pf_f32.cu) at p = 512 on a random SPD Gram.
// nvcc -DPF_CHOL_PHASES -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//   -o tools/probe/chol_probe tools/probe/chol_probe.cu paper_1904_10585_b200/csrc/pf_f32.cu
#include <cstdio>
#include <vector>
#include <random>

#include "../../paper_1904_10585_b200/csrc/pf_kernels.cuh"

namespace pf {
void count_launch() {}
extern __device__ long long g_chol_t[8];
}  // namespace pf

int main() {
  const int p = 512, n = 4096;
  std::mt19937_64 rng(1);
  std::normal_distribution<double> N(0, 1);
  std::vector<double> Y((size_t)n * p), G((size_t)p * p, 0.0);
  for (auto& v : Y) v = N(rng);
  for (int a = 0; a < p; ++a)
    for (int b = 0; b <= a; ++b) {
      double s = 0;
      for (int i = 0; i < n; ++i) s += Y[(size_t)i * p + a] * Y[(size_t)i * p + b];
      G[(size_t)a * p + b] = G[(size_t)b * p + a] = s;
    }
  double *dG, *W, *D, *R;
  pf::DevState* st;
  cudaMalloc(&dG, 8 * p * p); cudaMalloc(&W, 8 * p * p); cudaMalloc(&D, 8 * p * 32);
  cudaMalloc(&R, 8 * p * p); cudaMalloc(&st, sizeof(pf::DevState));
  cudaMemset(st, 0, sizeof(pf::DevState));
  cudaMemcpy(dG, G.data(), 8 * p * p, cudaMemcpyHostToDevice);
  for (int it = 0; it < 3; ++it) pf::chol_inv_big_launch(dG, p, n, W, D, R, st, nullptr, nullptr, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int it = 0; it < 10; ++it) pf::chol_inv_big_launch(dG, p, n, W, D, R, st, nullptr, nullptr, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long t[8];
  cudaMemcpyFromSymbol(t, pf::g_chol_t, sizeof(t));
  printf("chol_inv_big + linv_big p=%d: %.3f ms/call (%s)\n", p, ms / 10, cudaGetErrorString(cudaGetLastError()));
  printf("kernel-1 phases (cycles): setup %lld  cholesky %lld  diag-inverses %lld\n", t[1] - t[0],
         t[2] - t[1], t[3] - t[2]);
  // check R^T G R = I
  std::vector<double> Rh((size_t)p * p);
  cudaMemcpy(Rh.data(), R, 8 * p * p, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int a = 0; a < p; a += 37)
    for (int b = 0; b < p; b += 41) {
      double s = 0;
      for (int i = 0; i < p; ++i) {
        double gi = 0;
        for (int j = 0; j < p; ++j) gi += G[(size_t)i * p + j] * Rh[(size_t)j * p + b];
        s += Rh[(size_t)i * p + a] * gi;
      }
      err = std::max(err, std::abs(s - (a == b)));
    }
  printf("panel 0 (cycles): load->(a) %lld  (a) top block %lld  (b) rows %lld  writeback+(c) update %lld\n",
         t[4] - t[1], t[5] - t[4], t[6] - t[5], t[7] - t[6]);
  printf("max |R^T G R - I| (sampled) = %.3e\n", err);
  return 0;
}
