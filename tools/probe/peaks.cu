// Microbenchmark: fp64 DMMA (mma.sync m8n8k4 / m16n8k4 f64) vs DFMA issue throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_loop(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1e-4, b0 = 1.0 + threadIdx.x * 1e-6;
  double c[8][4];
  for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) c[i][j] = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b0));
    }
  }
  double s = 0;
  for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) s += c[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void dfma_loop(double* out, int iters) {
  double x[16];
  for (int i = 0; i < 16; i++) x[i] = threadIdx.x * 1e-3 + i;
  double m = 0.999999, a = 1e-9;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) x[i] = fma(x[i], m, a);
  }
  double s = 0;
  for (int i = 0; i < 16; i++) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * 148 * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps = 4; warps <= 16; warps *= 2) {
    int iters = 20000;
    dmma_loop<<<sms * 2, 32 * warps>>>(out, 100);
    cudaEventRecord(e0);
    dmma_loop<<<sms * 2, 32 * warps>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * 8 * 4 * 8.0 * iters * (double)(sms * 2) * warps;
    printf("DMMA m16n8k4 warps/CTA=%d x2 CTA/SM: %.2f TFLOP/s (%.3f ms)\n", warps, flops / ms / 1e9, ms);
  }
  for (int warps = 8; warps <= 32; warps *= 2) {
    int iters = 20000;
    dfma_loop<<<sms * 2, 32 * warps>>>(out, 100);
    cudaEventRecord(e0);
    dfma_loop<<<sms * 2, 32 * warps>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * iters * 32.0 * warps * (double)(sms * 2);
    printf("DFMA warps/CTA=%d x2: %.2f TFLOP/s (%.3f ms)\n", warps, flops / ms / 1e9, ms);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
