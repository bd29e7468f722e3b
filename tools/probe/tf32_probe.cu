// tf32_probe.cu -- bring-up check of the tcgen05 TF32 filter GEMM (pf_gemm_tf32.cu) outside
// libpf: out = s1 A Y + s2 Ycur + s3 Yprev against an fp64-accumulating reference kernel,
// plus CUDA-event timing.  Not part of the product; build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/probe/tf32_probe \
//     tools/probe/tf32_probe.cu paper_1904_10585_b200/csrc/pf_gemm.cu \
//     paper_1904_10585_b200/csrc/pf_gemm_tf32.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_1904_10585_b200/csrc/pf_kernels.cuh"

namespace pf {
void count_launch() {}
#ifdef PF_TRACE
void tf32_trace_read(unsigned long long* host);
#endif
}  // namespace pf

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

__global__ void fill(float* x, size_t n, unsigned long long seed, int positive) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long z = seed + i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    const double u = (double)(z >> 11) * (1.0 / 9007199254740992.0);
    x[i] = (float)(positive ? u : u * 2.0 - 1.0);
  }
}

// ref[c][i] (pitch ldy) = s1 sum_k A[i][k] Yt[c][k] + s2 ycur + s3 yprev, fp64; also bound
__global__ void ref_kernel(const float* A, int64_t lda, const float* Yt, int64_t ldy, int rows,
                           int nk, int p, const float* ycur, const float* yprev, double s1,
                           double s2, double s3, double* ref, double* bound, int row_stride) {
  int c = blockIdx.y;
  int i = (blockIdx.x * blockDim.x + threadIdx.x) * row_stride;
  if (i >= rows || c >= p) return;
  double s = 0, b = 0;
  for (int k = 0; k < nk; ++k) {
    double a = A[(size_t)i * lda + k], y = Yt[(size_t)c * ldy + k];
    s += a * y;
    b += fabs(a * y);
  }
  size_t o = (size_t)c * ldy + i;
  ref[o] = s1 * s + s2 * ycur[o] + s3 * yprev[o];
  bound[o] = fabs(s1) * b + fabs(s2 * ycur[o]) + fabs(s3 * yprev[o]);
}

int main(int argc, char** argv) {
  int rows = atoi(argv[1]), nk = atoi(argv[2]), p = atoi(argv[3]), npass = atoi(argv[4]);
  int reps = argc > 5 ? atoi(argv[5]) : 0;
  int row_stride = argc > 6 ? atoi(argv[6]) : 1;
  int dbg = argc > 7 ? atoi(argv[7]) : 0;
  int positive = argc > 8 ? atoi(argv[8]) : 0;
  int64_t lda = (nk + 3) / 4 * 4, ldy = (std::max(rows, nk) + 3) / 4 * 4;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float *A, *Y, *yc, *yp, *out, *ws;
  double *ref, *bound, *coef;
  int* cnt;
  CK(cudaMalloc(&A, sizeof(float) * rows * lda));
  CK(cudaMalloc(&Y, sizeof(float) * p * ldy));
  CK(cudaMalloc(&yc, sizeof(float) * p * ldy));
  CK(cudaMalloc(&yp, sizeof(float) * p * ldy));
  CK(cudaMalloc(&out, sizeof(float) * p * ldy));
  CK(cudaMalloc(&ref, sizeof(double) * p * ldy));
  CK(cudaMalloc(&bound, sizeof(double) * p * ldy));
  fill<<<1024, 256>>>(A, (size_t)rows * lda, 1, positive);
  fill<<<1024, 256>>>(Y, (size_t)p * ldy, 2, positive);
  fill<<<1024, 256>>>(yc, (size_t)p * ldy, 3, positive);
  fill<<<1024, 256>>>(yp, (size_t)p * ldy, 4, positive);
  CK(cudaMemset(out, 0, sizeof(float) * p * ldy));
  double hc[3] = {0.75, -0.5, -1.0};
  CK(cudaMalloc(&coef, sizeof(hc)));
  CK(cudaMemcpy(coef, hc, sizeof(hc), cudaMemcpyHostToDevice));
  pf::Tf32Plan pl = pf::tf32_plan(p, rows, nk, sms);
  CK(cudaMalloc(&ws, sizeof(float) * pl.ws_floats));
  float* accb;
  CK(cudaMalloc(&accb, sizeof(float) * pl.acc_floats));
  if (getenv("CHUNK_KB")) pl.chunk_kb = atoi(getenv("CHUNK_KB"));
  CK(cudaMalloc(&cnt, sizeof(int) * pl.counters));
  CK(cudaMemset(cnt, 0, sizeof(int) * pl.counters));
  CUtensorMap mA, mB, mApf;
  if (!pf::tf32_encode_A(&mA, &mApf, A, lda, rows, nk) || !pf::tf32_encode_B(&mB, Y, ldy, p, nk)) {
    printf("encode failed\n");
    return 1;
  }
  // VWORLD=W: read B through the 3-D map of a rank-major "all-gather" [W][p][nk/W] assembled
  // here from Y (exercises the distributed addressing on one GPU)
  int vworld = getenv("VWORLD") ? atoi(getenv("VWORLD")) : 0, bdist_kb = 0;
  if (vworld > 0) {
    const int nl = nk / vworld;
    float* Yg;
    CK(cudaMalloc(&Yg, sizeof(float) * (size_t)p * nk));
    for (int r = 0; r < vworld; ++r)
      CK(cudaMemcpy2D(Yg + (size_t)r * p * nl, nl * 4, Y + (size_t)r * nl, ldy * 4, nl * 4, p,
                      cudaMemcpyDeviceToDevice));
    if (!pf::tf32_encode_B_dist(&mB, Yg, p, nl, vworld)) {
      printf("encode 3-D failed\n");
      return 1;
    }
    bdist_kb = nl / 16;
    printf("virtual world %d, n_local %d (3-D B map)\n", vworld, nl);
  }
  printf("rows %d nk %d p %d npass %d: pairs %d split %d mtiles %d kblocks %d\n", rows, nk, p, npass, pl.pairs,
         pl.split, pl.mtiles, pl.kblocks);
  CK(pf::tf32_gemm_launch(pl, mA, mB, mApf, yc, yp, out, ldy, coef, ws, accb, cnt, npass, 0, bdist_kb));
  CK(cudaDeviceSynchronize());
  dim3 rg((rows / row_stride + 127) / 128, p);
  ref_kernel<<<rg, 128>>>(A, lda, Y, ldy, rows, nk, p, yc, yp, hc[0], hc[1], hc[2], ref, bound,
                          row_stride);
  CK(cudaDeviceSynchronize());
  std::vector<float> ho((size_t)p * ldy);
  std::vector<double> hr((size_t)p * ldy), hb((size_t)p * ldy);
  CK(cudaMemcpy(ho.data(), out, sizeof(float) * p * ldy, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hr.data(), ref, sizeof(double) * p * ldy, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hb.data(), bound, sizeof(double) * p * ldy, cudaMemcpyDeviceToHost));
  double maxrel = 0, maxabs = 0;
  long bad = 0;
  for (int c = 0; c < p; ++c)
    for (int i = 0; i < rows; i += row_stride) {
      size_t o = (size_t)c * ldy + i;
      double e = fabs((double)ho[o] - hr[o]);
      double r = e / (hb[o] > 0 ? hb[o] : 1.0);
      if (r > maxrel) maxrel = r;
      if (e > maxabs) maxabs = e;
      if (!(r < 1e-2)) {
        if (bad < 5) printf("  bad c=%d i=%d got %g ref %g\n", c, i, ho[o], hr[o]);
        ++bad;
      }
    }
  double bias = 0, nb = 0;
  for (int c = 0; c < p; ++c)
    for (int i = 0; i < rows; i += row_stride) {
      size_t o = (size_t)c * ldy + i;
      bias += ((double)ho[o] - hr[o]) / (hb[o] > 0 ? hb[o] : 1.0);
      nb += 1;
    }
  printf("max |err|/bound = %.3e  max |err| = %.3e  mean signed err/bound = %.3e  bad = %ld\n",
         maxrel, maxabs, bias / nb, bad);
  if (reps > 0) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int w = 0; w < 2; ++w)
      CK(pf::tf32_gemm_launch(pl, mA, mB, mApf, yc, yp, out, ldy, coef, ws, accb, cnt, npass, 0, bdist_kb));
    CK(cudaEventRecord(e0));
    for (int r = 0; r < reps; ++r)
      CK(pf::tf32_gemm_launch(pl, mA, mB, mApf, yc, yp, out, ldy, coef, ws, accb, cnt, npass, 0, bdist_kb));
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= reps;
    double fl = 2.0 * rows * (double)nk * p;
    printf("avg %.3f ms  algorithmic %.1f TF/s  tensor (x%d) %.1f TF/s  A-read %.0f GB/s\n", ms,
           fl / ms * 1e-9, npass, npass * fl / ms * 1e-9, 4.0 * rows * (double)nk / ms * 1e-6);
  }
#ifdef PF_TRACE
  {
    CK(pf::tf32_gemm_launch(pl, mA, mB, mApf, yc, yp, out, ldy, coef, ws, accb, cnt, npass, 0, bdist_kb));
    CK(cudaDeviceSynchronize());
    static unsigned long long tr[12][512];
    pf::tf32_trace_read(&tr[0][0]);
    printf("kb: L:issue lofree full done(w2) done(w7) | P:issue lofree full done(w2) done(w7) | mma_wait mma_ready\n");
    for (int i = 0; i < 512; i += (i < 24 ? 1 : 61))
    {
      long long z = (long long)tr[0][0];
      printf("%3d %6lld %6lld %6lld %6lld %6lld | %6lld %6lld %6lld %6lld %6lld | %6lld %6lld\n", i,
             (long long)tr[0][i] - z, (long long)tr[1][i] - z, (long long)tr[2][i] - z,
             (long long)tr[5][i] - z, (long long)tr[9][i] - z, (long long)tr[6][i] - z,
             (long long)tr[7][i] - z, (long long)tr[8][i] - z, (long long)tr[11][i] - z,
             (long long)tr[10][i] - z, (long long)tr[3][i] - z, (long long)tr[4][i] - z);
    }
  }
#endif
  return bad ? 2 : 0;
}
