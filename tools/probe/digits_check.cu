// digits_check.cu -- the two digit extractions of pf_digits.cuh agree bit for bit: the integer
// form (exponent decode + 64-bit shift, digit_words) and the fp64 form (|x| 2^(7S-E) + 2^52 with
// round-toward-zero, digit_words_sc) on random values of every magnitude below 2^E, zeros,
// subnormals, values just below 2^E, both signs, S = 6 and 7, E over its whole range.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1904_10585_b200/csrc \
//      digits_check.cu -o digits_check && ./digits_check
#include <cstdio>

#include "pf_digits.cuh"

using namespace pf;

__device__ unsigned long long mix(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <int S>
__global__ void check(long long n, unsigned long long* bad, unsigned long long* first) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long r = mix(i * 2 + S), r2 = mix(r);
    const int E = (int)(r2 % 2001) - 1000;       // scale_exp's clamp range
    if (E < 7 * S - 1022) continue;               // slices4 takes the integer form there
    double x;
    const int kind = (int)(r % 8);
    if (kind == 0) {
      x = 0.0;
    } else if (kind == 1) {                       // just below 2^E
      x = __longlong_as_double(__double_as_longlong(i8::pow2(E)) - 1 - (long long)(r2 >> 60));
    } else if (kind == 2) {                       // subnormal / tiny
      x = __longlong_as_double((long long)(r2 >> 13));
    } else {                                      // m 2^(E - k), m in [0.5, 1), k in [1, 80]
      const double m = 0.5 + 0.5 * (double)(r2 >> 11) * 0x1.0p-53;
      const int k = 1 + (int)((r >> 8) % 80);
      x = ldexp(m, E - k);
    }
    if (r & (1ull << 40)) x = -x;
    uint32_t a0, a1, b0, b1;
    i8::digit_words<S>(x, E, a0, a1);
    i8::digit_words_sc<S>(x, i8::pow2(7 * S - E), b0, b1);
    if (a0 != b0 || a1 != b1) {
      if (atomicAdd(bad, 1ull) == 0) *first = (unsigned long long)i;
    }
  }
}

int main() {
  unsigned long long *bad, *first;
  cudaMallocManaged(&bad, 16);
  cudaMallocManaged(&first, 8);
  int fails = 0;
  for (int S = 6; S <= 7; ++S) {
    *bad = 0;
    *first = 0;
    const long long n = 1ll << 28;
    if (S == 6) check<6><<<148 * 8, 256>>>(n, bad, first);
    else check<7><<<148 * 8, 256>>>(n, bad, first);
    cudaDeviceSynchronize();
    printf("S = %d: %lld values, %llu mismatches (first index %llu)\n", S, n, *bad, *first);
    fails += *bad != 0;
  }
  return fails;
}
