// coop_launch.cu -- replay cost of a CUDA graph of N kernels that return at once (a device flag
// is clear): normal vs cooperative launches, 128 CTAs x 256 threads; and of N kernels that do a
// little work in between (the launch gaps of the filter's inactive re-base slots).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/probe/coop_launch tools/probe/coop_launch.cu
#include <cooperative_groups.h>
#include <cstdio>

__global__ void empty_kernel(const int* flag, double* out) {
  if (*flag == 0) return;
  out[blockIdx.x] = 1.0;
}
__global__ void coop_kernel(const int* flag, double* out) {
  if (*flag == 0) return;
  cooperative_groups::this_grid().sync();
  out[blockIdx.x] = 1.0;
}

int main() {
  int* flag;
  double* out;
  cudaMalloc(&flag, 4);
  cudaMemset(flag, 0, 4);
  cudaMalloc(&out, 8 * 1024);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int mode = 0; mode < 2; ++mode) {
    for (int N : {1, 28}) {
      cudaGraph_t g;
      cudaGraphExec_t ge;
      cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
      for (int i = 0; i < N; ++i) {
        if (mode == 0) {
          empty_kernel<<<128, 256, 0, st>>>(flag, out);
        } else {
          void* args[] = {(void*)&flag, (void*)&out};
          cudaLaunchCooperativeKernel((const void*)coop_kernel, dim3(128), dim3(256), args, 0, st);
        }
      }
      cudaStreamEndCapture(st, &g);
      cudaGraphInstantiate(&ge, g, 0);
      for (int w = 0; w < 5; ++w) cudaGraphLaunch(ge, st);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, st);
      const int R = 200;
      for (int r = 0; r < R; ++r) cudaGraphLaunch(ge, st);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("%s N=%2d: %.2f us per graph, %.2f us per kernel (%s)\n",
             mode ? "cooperative" : "normal     ", N, ms * 1e3 / R, ms * 1e3 / R / N,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
