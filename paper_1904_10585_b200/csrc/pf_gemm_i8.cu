// pf_gemm_i8.cu -- the fp64 Chebyshev-step filter GEMM computed from EXACT int8 tensor-core
// products (dtype PF_FP64_I8; DESIGN.md §4 K1-i8):
//
//     out = s1 * (A B) + s2 * Ycur + s3 * Yprev        (eq:cheb, eqn:cheb-linear-map)
//
// B200's fp64 tensor pipe (DMMA) peaks at ~37 TF/s while its int8 tensor cores (tcgen05.mma
// kind::i8, s32 accumulation) run ~4.8 POPS dense (tools/probe/mma_i8_rate.cu: 16.4k int8
// ops/clk/SM).  An fp64 operand is split into S base-128 digits relative to a power-of-two scale
// (one per row of A, one per column of B): with V = trunc(x 2^(7S-E)) (exact, |V| < 2^7S),
//
//     x = 2^E * sum_{s=1..S} d_s 128^-s  +  r,   |r| < 2^(E - 7S),
//     V = d_1 128^(S-1) + ... + d_S,  d_s in [-127, 127], every digit carrying the sign of x
//
// (sign-symmetric truncating digits of |V| with the sign applied to each, pf_digits.cuh; the
// int32 bound below assumes |d| <= 128 and is therefore conservative).  Then
// (A B)_ic = 2^(E_i + F_c) sum_l 128^-l D_l[i, c] with the level sums D_l = sum_{s+t=l} A_s B_t
// (l = 2..S+1; products below level S+1 are dropped, < 2^-7S relative), each an integer matrix
// product computed EXACTLY by the tensor core in int32 (the K range per accumulation is bounded so
// that (l-1) K 128^2 < 2^31).  The levels are combined in
// fp64 in the epilogue, smallest first.  With S = 7 the operator error is ~2^-48 of the row / column
// scales -- the same order as an fp64 GEMM's own rounding bound (n u |A| |B|).
//
// Kernel structure (one CTA per SM, persistent over (128-row tile, column group) items):
//  * warp 0: TMA producer.  A slices live tiled, [128-row tile][k-block][S][128][64] int8
//    (pf_digits.cuh a8_offset): each A stage is ONE slice's contiguous 8 KB
//    128 x 64-byte box (8 KB) -- small stages so the ring is deep (TMA latency), A tagged L2
//    evict_first.  B = the digit slices of Y stored K-major [S][p][kpad]: one 3-D box
//    {64 B, NC columns, S slices} per k-block, L2 evict_last (re-read by every tile).
//  * warp 1 (one lane): MMA issuer, tcgen05.mma.cta_group::1.kind::i8, M = 128.  The S slices of
//    B sit stacked in shared memory, so A_s times [B_1 .. B_{S+1-s}] is ONE MMA of N = NC (S+1-s)
//    (split at 256) whose output columns land exactly on the TMEM regions of levels s+1 .. S+1:
//    TMEM holds S level accumulators of NC int32 columns side by side (S NC <= 512).
//  * warps 4..7: epilogue, tcgen05.ld of every level, fp64 combination, row / column scales,
//    the Chebyshev scale-shift-subtract, fp64 stores.  K ranges longer than the int32 bound are
//    folded into an fp64 workspace (deterministic order).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "pf_digits.cuh"
#include "pf_kernels.cuh"
#include "pf_tc.cuh"
#include "pf_i8mma.cuh"

namespace pf {


// ------------------------------------------------------------------------------ A splitting
// A (n_rows x n_k fp64, lda) -> tiled int8 digit slices A8 (a8_offset), rscale[row] = 2^E_row.
// One CTA per row at a time: pass 1 the row max (HBM), pass 2 re-reads the row (L2) and writes
// the S slices, 8 digits (8 bytes) per thread per slice.
template <int S>
__global__ void __launch_bounds__(512) a_split_kernel(const double* __restrict__ A, int64_t lda,
                                                      int n_rows, int n_k, int8_t* __restrict__ A8,
                                                      int KB, double* __restrict__ rscale) {
  __shared__ double red[32];
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int row = blockIdx.x; row < n_rows; row += gridDim.x) {
    const double* a = A + (int64_t)row * lda;
    double m = 0.0;
    const int n2 = n_k >> 1;
#pragma unroll 4
    for (int j = tid; j < n2; j += nt) {
      const double2 v = reinterpret_cast<const double2*>(a)[j];  // stays in L2 for pass 2
      m = fmax(m, fmax(fabs(v.x), fabs(v.y)));
    }
    if ((n_k & 1) && tid == 0) m = fmax(m, fabs(a[n_k - 1]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    __syncthreads();
    if ((tid & 31) == 0) red[tid >> 5] = m;
    __syncthreads();
    if (tid < 32) {
      double v = tid < (nt >> 5) ? red[tid] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (tid == 0) red[0] = v;
    }
    __syncthreads();
    const int E = i8::scale_exp(red[0]);
    if (tid == 0) rscale[row] = i8::pow2(E);
    int8_t* o = A8 + i8::a8_offset(row, 0, 0, KB, S);  // (row, k-block 0, slice 0)
    for (int j0 = tid * 8; j0 < n_k; j0 += nt * 8) {
      if (j0 + 8 <= n_k) {
        const double2 v0 = __ldcs(reinterpret_cast<const double2*>(a + j0));
        const double2 v1 = __ldcs(reinterpret_cast<const double2*>(a + j0) + 1);
        const double2 v2 = __ldcs(reinterpret_cast<const double2*>(a + j0) + 2);
        const double2 v3 = __ldcs(reinterpret_cast<const double2*>(a + j0) + 3);
        uint32_t lo[S], hi[S];
        i8::slices4<S>(v0.x, v0.y, v1.x, v1.y, E, lo);
        i8::slices4<S>(v2.x, v2.y, v3.x, v3.y, E, hi);
#pragma unroll
        for (int s = 0; s < S; ++s)
          __stcs(reinterpret_cast<uint2*>(o + ((size_t)(j0 >> 6) * S + s) * 8192 + (j0 & 63)),
                 make_uint2(lo[s], hi[s]));
      } else {
        for (int j = j0; j < n_k; ++j)
#pragma unroll
          for (int s = 0; s < S; ++s)
            o[((size_t)(j >> 6) * S + s) * 8192 + (j & 63)] = i8::digit<S>(a[j], E, s);
      }
    }
    __syncthreads();  // red[] reuse
  }
}

// ------------------------------------------------------------------------------ Y splitting
// One cooperative launch for the B operand split: the column maxima of Y (n_k x p row-major, ldy;
// grid-stride, atomicMax of the fp64 bit patterns of |y| >= 0, whose integer order is the fp64
// order; the accumulator zeroed by CTA 0 before a first grid barrier), a second grid barrier,
// then the digit split of each CTA's 32-row chunks (rows re-read from L2): Y -> Y8[s][c][kpad]
// (K-major digit slices), cscale[c] = 2^F_c.
template <int S>
__global__ void __launch_bounds__(256) y_colmax_split_kernel(const double* __restrict__ Y,
                                                            int64_t ldy, int n_k, int p,
                                                            unsigned long long* cmax,
                                                            int8_t* __restrict__ Y8, int64_t kpad,
                                                            double* __restrict__ cscale) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  constexpr int R = 32;
  __shared__ double tile[R * 65];
  if (blockIdx.x == 0)
    for (int c = threadIdx.x; c < p; c += blockDim.x) cmax[c] = 0ull;
  grid.sync();
  {
    double* smx = tile;  // 256 doubles
    const int c = threadIdx.x % p, r0 = threadIdx.x / p, rstep = blockDim.x / p;
    double m = 0.0;
    for (int r = blockIdx.x * rstep + r0; r < n_k; r += gridDim.x * rstep)
      m = fmax(m, fabs(__ldg(Y + (int64_t)r * ldy + c)));
    smx[threadIdx.x] = m;
    __syncthreads();
    if (threadIdx.x < p) {
      for (int k = 1; k < rstep; ++k) m = fmax(m, smx[k * p + threadIdx.x]);
      if (m > 0.0) atomicMax(cmax + c, (unsigned long long)__double_as_longlong(m));
    }
  }
  grid.sync();
  for (int chunk = blockIdx.x; chunk * R < n_k; chunk += gridDim.x) {
    const int k0 = chunk * R;
    for (int cb = 0; cb < p; cb += 64) {
      const int pc = min(64, p - cb);
      __syncthreads();
      for (int i = threadIdx.x; i < R * pc; i += blockDim.x) {
        const int r = i / pc, c = i % pc;
        tile[r * 65 + c] = (k0 + r < n_k) ? Y[(int64_t)(k0 + r) * ldy + cb + c] : 0.0;
      }
      __syncthreads();
      for (int i = threadIdx.x; i < pc * (R / 8); i += blockDim.x) {
        const int c = i / (R / 8), g = i % (R / 8);  // column, 8-row group
        const int E = i8::scale_exp(__longlong_as_double((long long)__ldcg(cmax + cb + c)));
        if (chunk == 0 && g == 0) cscale[cb + c] = i8::pow2(E);
        uint32_t lo[S], hi[S];
        const double* tc0 = tile + (g * 8) * 65 + c;
        i8::slices4<S>(tc0[0], tc0[65], tc0[130], tc0[195], E, lo);
        i8::slices4<S>(tc0[260], tc0[325], tc0[390], tc0[455], E, hi);
        const int k = k0 + g * 8;
        if (k < n_k) {
#pragma unroll
          for (int s = 0; s < S; ++s)
            *reinterpret_cast<uint2*>(Y8 + ((int64_t)s * p + cb + c) * kpad + k) =
                make_uint2(lo[s], hi[s]);
        }
      }
    }
  }
}

// The same split in ONE grid barrier when every 32-row chunk has its own CTA (p <= 64): each CTA
// loads its chunk once into shared memory, publishes the chunk's column maxima (atomicMax), waits
// at the barrier, and splits the chunk from shared memory -- no second read of Y and no barrier
// for zeroing the accumulator, which alternates between two halves of cmax (cmax[2p] selects the
// half; the other half is zeroed for the next call).
template <int S>
__global__ void __launch_bounds__(256) y_split_tile_kernel(const double* __restrict__ Y,
                                                          int64_t ldy, int n_k, int p,
                                                          unsigned long long* cmax,
                                                          int8_t* __restrict__ Y8, int64_t kpad,
                                                          double* __restrict__ cscale) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  constexpr int R = 32;
  __shared__ double tile[R * 65];
  __shared__ double smx[256];
  const int sel = (int)__ldcg(cmax + 2 * p);
  unsigned long long* cm = cmax + (size_t)sel * p;
  const int k0 = blockIdx.x * R;
  const int half = p >> 1;
  for (int i = threadIdx.x; i < R * half; i += blockDim.x) {
    const int r = i / half, c = (i - r * half) * 2;
    double2 v = make_double2(0.0, 0.0);
    if (k0 + r < n_k) v = __ldcg(reinterpret_cast<const double2*>(Y + (int64_t)(k0 + r) * ldy + c));
    tile[r * 65 + c] = v.x;
    tile[r * 65 + c + 1] = v.y;
  }
  __syncthreads();
  {
    const int c = threadIdx.x % p, r0 = threadIdx.x / p, rstep = blockDim.x / p;
    double m = 0.0;
    for (int r = r0; r < R; r += rstep) m = fmax(m, fabs(tile[r * 65 + c]));
    smx[threadIdx.x] = m;
    __syncthreads();
    if (threadIdx.x < p) {
      for (int k = 1; k < rstep; ++k) m = fmax(m, smx[k * p + threadIdx.x]);
      if (m > 0.0) atomicMax(cm + c, (unsigned long long)__double_as_longlong(m));
    }
  }
  grid.sync();
  if (blockIdx.x == 0) {
    for (int c = threadIdx.x; c < p; c += blockDim.x) cmax[(size_t)(1 - sel) * p + c] = 0ull;
    if (threadIdx.x == 0) cmax[2 * p] = (unsigned long long)(1 - sel);  // every CTA read sel
  }
  for (int i = threadIdx.x; i < p * (R / 8); i += blockDim.x) {
    const int c = i / (R / 8), g = i % (R / 8);  // column, 8-row group
    const int E = i8::scale_exp(__longlong_as_double((long long)__ldcg(cm + c)));
    if (blockIdx.x == 0 && g == 0) cscale[c] = i8::pow2(E);
    uint32_t lo[S], hi[S];
    const double* tc0 = tile + (g * 8) * 65 + c;
    i8::slices4<S>(tc0[0], tc0[65], tc0[130], tc0[195], E, lo);
    i8::slices4<S>(tc0[260], tc0[325], tc0[390], tc0[455], E, hi);
    const int k = k0 + g * 8;
    if (k < n_k) {
#pragma unroll
      for (int s = 0; s < S; ++s)
        *reinterpret_cast<uint2*>(Y8 + ((int64_t)s * p + c) * kpad + k) = make_uint2(lo[s], hi[s]);
    }
  }
}

// ------------------------------------------------------------------------------ GEMM
template <int S, int NC>
struct I8Cfg {
  static constexpr int BK = 64;                  // K bytes per k-block (SWIZZLE_64B rows)
  static constexpr int BM = 128;                 // rows per tile (M of the MMA)
  static constexpr int A_TILE = BM * BK;         // one slice of one k-block: 8 KB
  // A_s x [B_0 .. B_{S-1-s}] as few MMAs as possible (N up to 256): with operands that change
  // from one MMA to the next, an MMA costs ~100 cycles of M-side (A) operand fetch plus ~0.33
  // cycle per N column (tools/probe/i8_pattern.cu: 1524 cycles per K = 32 step for this
  // sequence vs 1951 for uniform N = 128 windows and 2866 for one N = 64 MMA per slice pair),
  // so the fewest A fetches win.
  static constexpr int CMAX = 256 / NC;          // B slices per MMA
  static constexpr int B_LOAD = S * NC * BK;     // TMA bytes per B k-block
  static constexpr int B_STAGE = B_LOAD;
  static constexpr int NB = B_STAGE <= 8192 ? 4 : 2;  // B comes from L2 (short latency)
  static constexpr int BUDGET = 216 * 1024;
  static constexpr int NA0 = (BUDGET - NB * B_STAGE) / A_TILE;
  static constexpr int NA = NA0 > 24 ? 24 : NA0;
  static constexpr int COLS = S * NC;            // TMEM columns used (level-major)
  static constexpr int TMEM_COLS = COLS <= 32 ? 32 : COLS <= 64 ? 64 : COLS <= 128 ? 128
                                   : COLS <= 256 ? 256 : 512;
  static constexpr int CW = NC < 32 ? NC : 32;   // epilogue column chunk
  static constexpr int THREADS = 256;            // w0 TMA, w1 MMA, w2 TMEM alloc, w4..7 epilogue
  static constexpr int BAR_BYTES = 8 * (2 * NA + 2 * NB + 2) + 16;
  static constexpr int SMEM = NA * A_TILE + NB * B_STAGE + 1024 + BAR_BYTES;
  static_assert(COLS <= 512, "TMEM");
  static_assert(NC % 16 == 0 && NC <= 64, "NC");
  static_assert(NA >= 6, "A ring");
  static_assert(SMEM <= 227 * 1024, "smem");
};

struct I8Args {
  int pf_dist;           // L2 prefetch distance of the A k-blocks (0: off)
  int lower_t;           // K1-i8p: A holds the upper tiles (+ diagonal super-blocks) only; the
                         // units left of the pair's super-block read the stored upper tile transposed
  int lS;                // slices per (tile, k-block) in the A8 layout (the split's S >= S used)
  const double* ycur;
  const double* yprev;
  double* out;
  int64_t ldy;
  const double* coef;    // {s1, s2, s3} (device)
  const double* rscale;  // [n_rows]
  const double* cscale;  // [p]
  double* acc;           // fold workspace [grid][NC][128]
  double* part;          // stream-K partial tiles [items][maxp][NC][128]
  int* counters;         // [items], zero between launches
  int maxp;
  int n_rows, kblocks, mtiles, ngroups, chunk_kb;
};

// Stream-K work split: the items x kblocks (tile, k-block) units are cut into gridDim.x equal
// contiguous ranges, so every SM gets the same share of the tensor work; an item cut between
// CTAs is finished by the last contributor, which sums the fp64 partials in k order.  Items are
// column-group major (item = cg * mtiles + tile): with p = 128 (two 64-column groups) CTAs b and
// b + G/2 walk the same A tile over the same k-blocks at the same time, so A's digit slices are
// read from HBM once and hit in L2 by the other group.
struct SegIter {
  long long u, u1;
  int KB;
  __device__ SegIter(long long U, int G, int b, int KB_) : KB(KB_) {
    u = U * b / G;
    u1 = U * (b + 1) / G;
  }
  __device__ bool next(int& item, int& kb0, int& kb1) {
    if (u >= u1) return false;
    item = (int)(u / KB);
    kb0 = (int)(u - (long long)item * KB);
    kb1 = (int)min((long long)KB, kb0 + (u1 - u));
    u += kb1 - kb0;
    return true;
  }
};
// CTA owning unit u
__device__ __forceinline__ int seg_owner(long long u, long long U, int G) {
  int b = (int)(u * G / U);
  while (b + 1 < G && U * (b + 1) / G <= u) ++b;
  while (b > 0 && U * b / G > u) --b;
  return b;
}

// v[j] += sum_L 128^-(L+2) D_L[c0 + j], L = S-1 .. 0 in that order (smallest weight first),
// one TMEM wait per level (all CW columns of the level in flight)
template <int S, int NC, int CW>
__device__ __forceinline__ void i8_combine_levels(uint32_t taddr, int c0, double (&v)[CW]) {
  static_assert(CW % 16 == 0, "CW");
  struct R16 {
    uint32_t x[16];
  };
#pragma unroll 1
  for (int L = S - 1; L >= 0; --L) {
    R16 a[CW / 16];
#pragma unroll
    for (int h = 0; h < CW / 16; ++h)
      i8::tmem_ld16_nw(taddr + (uint32_t)(L * NC + c0 + 16 * h), a[h].x);
    i8::tmem_wait_ld();
    const double w = i8::pow2(-7 * (L + 2));
#pragma unroll
    for (int h = 0; h < CW / 16; ++h)
#pragma unroll
      for (int j = 0; j < 16; ++j) v[16 * h + j] = fma((double)(int)a[h].x[j], w, v[16 * h + j]);
  }
}

struct RingI {
  int n, s;
  uint32_t ph;
  __device__ RingI(int n_) : n(n_), s(0), ph(0) {}
  __device__ void next() {
    if (++s == n) {
      s = 0;
      ph ^= 1u;
    }
  }
};

template <int S, int NC>
__global__ void __launch_bounds__(I8Cfg<S, NC>::THREADS, 1)
    cheb_gemm_i8_kernel(const __grid_constant__ CUtensorMap mapA8,
                        const __grid_constant__ CUtensorMap mapY8,
                        const __grid_constant__ CUtensorMap mapA8pf, I8Args args) {
  using C = I8Cfg<S, NC>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* ring_a = smem;                              // NA x [128][64] int8
  unsigned char* ring_b = smem + C::NA * C::A_TILE;          // NB x [S][NC][64] int8
  uint64_t* afull = reinterpret_cast<uint64_t*>(ring_b + C::NB * C::B_STAGE);
  uint64_t* aempty = afull + C::NA;
  uint64_t* bfull = aempty + C::NA;
  uint64_t* bempty = bfull + C::NB;
  uint64_t* tfull = bempty + C::NB;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  volatile int* sflag = reinterpret_cast<volatile int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NA; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], 1);
    }
    for (int s = 0; s < C::NB; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&bempty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mapA8);
    tma_prefetch_desc(&mapY8);
    tma_prefetch_desc(&mapA8pf);
  }
  if (warp == 2) i8::tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  const int KB = args.kblocks;
  const int nitems = args.mtiles * args.ngroups;
  const int kch = args.chunk_kb;
  const long long U = (long long)nitems * KB;
  const int G = gridDim.x;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (one warp)
    // warp-uniform loop, one elected lane issues (as the MMA issuer); one B box per k-block
    // (a separate B producer warp, as in K1-i8p, measured 0.383 vs 0.381 ms: no gain here)
    RingI ra(C::NA), rb(C::NB);
    const uint64_t pol_a = tc::policy_evict_first(), pol_b = tc::policy_evict_last();
    SegIter si(U, G, blockIdx.x, KB);
    int it, kbs, kbe;
    while (si.next(it, kbs, kbe)) {
      const int cg = it / args.mtiles, tile = it - cg * args.mtiles;  // column-group major
      if (args.pf_dist > 0 && i8::elect_one())  // warm the first k-blocks of the segment
        for (int kb = kbs; kb < min(kbe, kbs + args.pf_dist); ++kb)
          tc::tma_prefetch_3d(&mapA8pf, 0, 0, (tile * KB + kb) * args.lS, pol_a);
      __syncwarp();
      for (int kb = kbs; kb < kbe; ++kb) {
        // A streams from HBM once: every slice of k-block kb + pf_dist into L2 ahead of its load
        if (args.pf_dist > 0 && kb + args.pf_dist < kbe && i8::elect_one())
          tc::tma_prefetch_3d(&mapA8pf, 0, 0, (tile * KB + kb + args.pf_dist) * args.lS, pol_a);
        __syncwarp();
        mbar_wait(&bempty[rb.s], rb.ph ^ 1u);
        if (i8::elect_one()) {
          mbar_arrive_expect_tx(&bfull[rb.s], C::B_LOAD);
          tc::tma_load_3d_hint(ring_b + rb.s * C::B_STAGE, &mapY8, &bfull[rb.s], kb * C::BK,
                               cg * NC, 0, pol_b);
        }
        __syncwarp();
        rb.next();
#pragma unroll
        for (int s = 0; s < S; ++s) {
          mbar_wait(&aempty[ra.s], ra.ph ^ 1u);
          if (i8::elect_one()) {
            mbar_arrive_expect_tx(&afull[ra.s], C::A_TILE);
            tc::tma_load_3d_hint(ring_a + ra.s * C::A_TILE, &mapA8, &afull[ra.s], 0, 0,
                                 (tile * KB + kb) * args.lS + s, pol_a);
          }
          __syncwarp();
          ra.next();
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (one warp)
    // The whole warp runs the loop (its values are warp-uniform, so descriptors and TMEM
    // addresses live in uniform registers) and one elected lane issues: issuing from a lone
    // thread made every MMA wait for a scalar-to-uniform broadcast of its seven operands
    // (~100 cycles each, more than the N = 64..256 MMA itself).
    RingI ra(C::NA), rb(C::NB);
    uint32_t tph = 0;
    SegIter si(U, G, blockIdx.x, KB);
    int it, kbs, kbe;
    const uint64_t adesc_ring = tc::sdesc_k_sw64(smem_u32(ring_a));
    const uint64_t bdesc_ring = tc::sdesc_k_sw64(smem_u32(ring_b));
    while (si.next(it, kbs, kbe)) {
      for (int k0 = kbs; k0 < kbe; k0 += kch) {
        const int k1 = min(kbe, k0 + kch);
        mbar_wait(tempty, tph ^ 1u);  // the epilogue drained the accumulators
        tc::fence_after_sync();
        for (int kb = k0; kb < k1; ++kb) {
          mbar_wait(&bfull[rb.s], rb.ph);
          // descriptors by addition: the start-address field is (addr >> 4) in the low 14 bits
          // (smem < 256 KB, no carry out), so desc(addr + off) = desc(addr) + off / 16 -- a few
          // integer adds per MMA instead of rebuilding every descriptor
          const uint64_t bd0 = bdesc_ring + (uint64_t)(rb.s * (C::B_STAGE >> 4));
#pragma unroll
          for (int s = 0; s < S; ++s) {
            mbar_wait(&afull[ra.s], ra.ph);
            tc::fence_after_sync();
            const uint64_t ad0 = adesc_ring + (uint64_t)(ra.s * (C::A_TILE >> 4));
            if (i8::elect_one()) {
#pragma unroll
              for (int ks = 0; ks < 2; ++ks) {
                const uint32_t acc = (kb == k0 && s == 0 && ks == 0) ? 0u : 1u;
                const uint64_t ad = ad0 + (uint64_t)(ks * 2);
                // A_s x [B_0 .. B_{S-1-s}] -> levels s .. S-1 (0-based), chunks of <= CMAX
                // slices; s = 0 initialises every level
#pragma unroll
                for (int t0 = 0; t0 < S - s; t0 += C::CMAX) {
                  const int c = (S - s - t0) < C::CMAX ? (S - s - t0) : C::CMAX;
                  i8::mma_i8(tmem + (uint32_t)((s + t0) * NC), ad,
                             bd0 + (uint64_t)((t0 * NC * C::BK + ks * 32) >> 4),
                             i8::idesc_i8(C::BM, c * NC), acc);
                }
              }
              i8::mma_commit(&aempty[ra.s]);  // A slice stage free once these MMAs complete
            }
            __syncwarp();
            ra.next();
          }
          if (i8::elect_one()) i8::mma_commit(&bempty[rb.s]);
          __syncwarp();
          rb.next();
        }
        if (i8::elect_one()) i8::mma_commit(tfull);
        __syncwarp();
        tph ^= 1u;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue (4 warps)
    const int q = warp & 3;
    const int et = 32 * q + lane;  // row within the tile = TMEM lane
    const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16);
    const double s1 = args.coef[0], s2 = args.coef[1], s3 = args.coef[2];
    double* accp = args.acc + (size_t)blockIdx.x * (NC * 128) + et;
    uint32_t tph = 0;
    SegIter si(U, G, blockIdx.x, KB);
    int it, kbs, kbe;
    while (si.next(it, kbs, kbe)) {
      const int cg = it / args.mtiles, tile = it - cg * args.mtiles;  // column-group major
      const int row = tile * C::BM + et;
      const bool row_ok = row < args.n_rows;
      const double rs = row_ok ? args.rscale[row] : 0.0;
      const bool whole = (kbs == 0 && kbe == KB);
      int part = 0, nparts = 1;
      if (!whole) {
        const int f = seg_owner((long long)it * KB, U, G);
        part = blockIdx.x - f;
        nparts = seg_owner((long long)it * KB + KB - 1, U, G) - f + 1;
      }
      double* mypart = args.part + ((size_t)it * args.maxp + part) * (NC * 128) + et;
      if (!whole && kbe - kbs <= kch) {
        // ------------------------------------------------ split item, one accumulation
        // If every other contributor has already published its partial (the usual case: this
        // CTA runs the item's long part), the item is finished straight from TMEM without
        // writing and re-reading this CTA's partial.  Sum order is the general fixup's (parts
        // in index order, this one in its slot): bit-identical either way.
        mbar_wait(tfull, tph);
        tph ^= 1u;
        tc::fence_after_sync();
        named_bar_sync(1, 128);
        if (et == 0) *sflag = (atomicAdd(&args.counters[it], 0) + 1 == nparts) ? 1 : 0;
        named_bar_sync(1, 128);
        const bool early = (*sflag != 0);
        named_bar_sync(1, 128);
        bool lastc = early;
        if (!early) {
#pragma unroll 1
          for (int c0 = 0; c0 < NC; c0 += C::CW) {
            double v[C::CW];
#pragma unroll
            for (int j = 0; j < C::CW; ++j) v[j] = 0.0;
            i8_combine_levels<S, NC, C::CW>(taddr, c0, v);
#pragma unroll
            for (int j = 0; j < C::CW; ++j) __stcg(mypart + (size_t)(c0 + j) * 128, v[j]);
          }
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) mbar_arrive(tempty);
          __threadfence();
          named_bar_sync(1, 128);
          if (et == 0) *sflag = (atomicAdd(&args.counters[it], 1) + 1 == nparts) ? 1 : 0;
          named_bar_sync(1, 128);
          lastc = (*sflag != 0);
          named_bar_sync(1, 128);
        } else {
          __threadfence();
        }
        if (lastc) {
          const double* p0 = args.part + (size_t)it * args.maxp * (NC * 128) + et;
#pragma unroll 1
          for (int c0 = 0; c0 < NC; c0 += C::CW) {
            double m[C::CW];  // this CTA's part: from TMEM (early) or its own published partial
#pragma unroll
            for (int j = 0; j < C::CW; ++j) m[j] = 0.0;
            if (early) i8_combine_levels<S, NC, C::CW>(taddr, c0, m);
            double v[C::CW];
#pragma unroll
            for (int j = 0; j < C::CW; ++j) v[j] = 0.0;
#pragma unroll 1
            for (int q2 = 0; q2 < nparts; ++q2) {
              if (q2 == part && early) {
#pragma unroll
                for (int j = 0; j < C::CW; ++j) v[j] += m[j];
              } else {
#pragma unroll
                for (int j = 0; j < C::CW; ++j)
                  v[j] += __ldcg(p0 + (size_t)q2 * (NC * 128) + (size_t)(c0 + j) * 128);
              }
            }
            if (row_ok) {
              const int cbase = cg * NC + c0;
              const size_t o = (size_t)row * args.ldy + cbase;
#pragma unroll
              for (int j = 0; j < C::CW; ++j) {
                double y = s1 * (v[j] * rs * __ldg(args.cscale + cbase + j));
                if (s2 != 0.0) y = fma(s2, args.ycur[o + j], y);
                if (s3 != 0.0) y = fma(s3, args.yprev[o + j], y);
                args.out[o + j] = y;
              }
            }
          }
          if (et == 0) args.counters[it] = 0;  // ready for the next launch
        }
        if (early) {
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) mbar_arrive(tempty);
        }
        continue;
      }
      for (int k0 = kbs; k0 < kbe; k0 += kch) {
        const bool first = (k0 == kbs), last = (k0 + kch >= kbe);
        mbar_wait(tfull, tph);
        tph ^= 1u;
        tc::fence_after_sync();
#pragma unroll 1
        for (int c0 = 0; c0 < NC; c0 += C::CW) {
          double v[C::CW];
#pragma unroll
          for (int j = 0; j < C::CW; ++j) v[j] = 0.0;
          // smallest level first: level L (0-based) carries weight 128^-(L+2)
          i8_combine_levels<S, NC, C::CW>(taddr, c0, v);
          if (!first) {
#pragma unroll
            for (int j = 0; j < C::CW; ++j) v[j] += __ldcg(accp + (size_t)(c0 + j) * 128);
          }
          if (!last) {
#pragma unroll
            for (int j = 0; j < C::CW; ++j) __stcg(accp + (size_t)(c0 + j) * 128, v[j]);
          } else if (!whole) {  // partial of a split item
#pragma unroll
            for (int j = 0; j < C::CW; ++j) __stcg(mypart + (size_t)(c0 + j) * 128, v[j]);
          } else if (row_ok) {
            const int cbase = cg * NC + c0;
            const size_t o = (size_t)row * args.ldy + cbase;
#pragma unroll
            for (int j = 0; j < C::CW; ++j) {
              double y = s1 * (v[j] * rs * __ldg(args.cscale + cbase + j));
              if (s2 != 0.0) y = fma(s2, args.ycur[o + j], y);
              if (s3 != 0.0) y = fma(s3, args.yprev[o + j], y);
              args.out[o + j] = y;
            }
          }
        }
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty);
      }
      if (!whole) {
        // ------------------------------------------------ stream-K fixup (last contributor)
        __threadfence();
        named_bar_sync(1, 128);
        if (et == 0) {
          const int prev = atomicAdd(&args.counters[it], 1);
          *sflag = (prev + 1 == nparts) ? 1 : 0;
        }
        named_bar_sync(1, 128);
        const bool lastc = (*sflag != 0);
        named_bar_sync(1, 128);
        if (lastc) {
          __threadfence();
            const double* p0 = args.part + (size_t)it * args.maxp * (NC * 128) + et;
#pragma unroll 1
          for (int c0 = 0; c0 < NC; c0 += C::CW) {
            double v[C::CW];
#pragma unroll
            for (int j = 0; j < C::CW; ++j) v[j] = 0.0;
#pragma unroll 1
            for (int q2 = 0; q2 < nparts; ++q2) {
#pragma unroll
              for (int j = 0; j < C::CW; ++j)
                v[j] += __ldcg(p0 + (size_t)q2 * (NC * 128) + (size_t)(c0 + j) * 128);
            }
            if (row_ok) {
              const int cbase = cg * NC + c0;
              const size_t o = (size_t)row * args.ldy + cbase;
#pragma unroll
              for (int j = 0; j < C::CW; ++j) {
                double y = s1 * (v[j] * rs * __ldg(args.cscale + cbase + j));
                if (s2 != 0.0) y = fma(s2, args.ycur[o + j], y);
                if (s3 != 0.0) y = fma(s3, args.yprev[o + j], y);
                args.out[o + j] = y;
              }
            }
          }
          if (et == 0) args.counters[it] = 0;  // ready for the next launch
        }
      }
    }
  }

  __syncwarp();
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 2) {
    tc::fence_after_sync();
    i8::tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// ------------------------------------------------------------------------------ CTA pairs
// K1-i8p: the same product on CTA pairs -- cluster 2 x 1,
// tcgen05.mma.cta_group::2.kind::i8, M = 256 (the pair's two 128-row tiles).  Each CTA holds its
// own tile's A slices and supplies HALF of every MMA's N rows of B, so the tensor core's B reads
// per SM halve: the K1-i8 MMA sequence reads ~96 KB of operands per 32-byte K step per SM from
// shared memory (40 KB of A, 56 KB of stacked B) against the ~1792-cycle budget of a k-block
// at the int8 peak, next to the TMA writes of the ring -- the per-SM operand bandwidth, not the
// MMA rate, was the limit.  The pair reads 40 + 28 KB per K step per SM.
//
// An MMA's N rows are split in halves between the CTAs at ONE shared-memory offset, and its
// D columns are [first half | second half]; to land every slice product on its level's TMEM
// columns (level l at 64 l, as in K1-i8) the B block is staged per k-block as 7 regions whose
// halves differ by rank (512 rows of 64 bytes per CTA, 32 KB):
//   rows   0..127  Ra  [B0 B1 | B2 B3]      A_0..A_3 x Ra, N = 256, TMEM column 64 s
//   rows 128..223  Rb  [B4 B5a | B5b B6]    A_0 x Rb, N = 192, column 256
//   rows 224..287  Rc  [B4 | B5]            A_1 x Rc, N = 128, column 320
//   rows 288..319  Rd  [B4a | B4b]          A_2 x Rd, N =  64, column 384
//   rows 320..415  Re  [B0 B1a | B1b B2]    A_4 x Re, N = 192, column 256
//   rows 416..479  Rf  [B0 | B1]            A_5 x Rf, N = 128, column 320
//   rows 480..511  Rg  [B0a | B0b]          A_6 x Rg, N =  64, column 384
// (a / b = columns 0..31 / 32..63 of a slice; "|" separates rank 0's rows from rank 1's).
// The same 10 MMAs per K step as K1-i8, each twice as tall.  Both CTAs' TMA loads complete on
// the LEADER's full barriers (cta_group::2 TMA), the leader's MMA commits free the stages of both
// (multicast), both epilogues drain their own TMEM lanes and arrive on the leader's tempty.
// Stream-K runs over (pair tile, k-block) units per cluster; each CTA finishes its own rows
// (partials and counters per CTA).  S = 7, NC = 64 (p a multiple of 64).
struct I8PCfg {
  static constexpr int S = 7, NC = 64, BK = 64, BM = 128;
  static constexpr int A_TILE = BM * BK;               // 8 KB: one slice of one k-block
  static constexpr int B_ROWS = 512;                   // staged B rows per CTA per k-block
  static constexpr int B_STAGE = B_ROWS * BK;          // 32 KB
  static constexpr int NB = 2;
  static constexpr int NA = 20;  // the A ring takes what the B ring and the barriers leave
  static constexpr int TMEM_COLS = 512;                // 448 used
  static constexpr int CW = 32;
  static constexpr int THREADS = 256;
  static constexpr int BAR_BYTES = 8 * (2 * NA + 2 * NB + 2) + 16;
  static constexpr int SMEM = NA * A_TILE + NB * B_STAGE + 1024 + BAR_BYTES;
  static_assert(SMEM <= 227 * 1024, "smem");
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(I8PCfg::THREADS, 1)
    cheb_gemm_i8p_kernel(const __grid_constant__ CUtensorMap mapA8,
                         const __grid_constant__ CUtensorMap mapB64,
                         const __grid_constant__ CUtensorMap mapB32,
                         const __grid_constant__ CUtensorMap mapA8t, I8Args args) {
  using C = I8PCfg;
  constexpr int S = C::S, NC = C::NC;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* ring_a = smem;                              // NA x [128][64] int8
  unsigned char* ring_b = smem + C::NA * C::A_TILE;          // NB x [512][64] int8
  uint64_t* afull = reinterpret_cast<uint64_t*>(ring_b + C::NB * C::B_STAGE);
  uint64_t* aempty = afull + C::NA;
  uint64_t* bfull = aempty + C::NA;
  uint64_t* bempty = bfull + C::NB;
  uint64_t* tfull = bempty + C::NB;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  volatile int* sflag = reinterpret_cast<volatile int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = tc::cluster_ctarank();
  const int G = (int)tc::nclusters_x(), g = (int)tc::cluster_id_x();
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NA; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], 1);
    }
    for (int s = 0; s < C::NB; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&bempty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 8);  // 4 epilogue warps x 2 CTAs (the leader's copy is used)
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mapA8);
    tma_prefetch_desc(&mapB64);
    tma_prefetch_desc(&mapB32);
    if (args.lower_t) tma_prefetch_desc(&mapA8t);
  }
  if (warp == 2) tc::tmem_alloc_pair<C::TMEM_COLS>(tmem_slot);
  tc::fence_before_sync();
  tc::cluster_sync();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  const int KB = args.kblocks;
  const int mpairs = (args.mtiles + 1) >> 1;
  const int nitems = mpairs * args.ngroups;
  const int kch = args.chunk_kb;
  const long long U = (long long)nitems * KB;

  if (warp == 0 || warp == 3) {
    // ------------------------------------------------------------ TMA producers (both CTAs)
    // warp 0 streams the A slices, warp 3 the B regions: two loops, so the A ring runs up to
    // NA slices ahead whatever the depth of the B ring
    const bool is_a = (warp == 0);
    RingI ra(C::NA), rb(C::NB);
    const uint64_t pol_a = tc::policy_evict_first(), pol_b = tc::policy_evict_last();
    const uint32_t afull_l = tc::mapa(smem_u32(afull), 0), bfull_l = tc::mapa(smem_u32(bfull), 0);
    // this rank's B boxes per k-block: {smem row, slice, row in slice, 64-row box?}
    constexpr int T0[10][4] = {{0, 0, 0, 1},   {64, 1, 0, 1},   {128, 4, 0, 1}, {192, 5, 0, 0},
                               {224, 4, 0, 1}, {288, 4, 0, 0},  {320, 0, 0, 1}, {384, 1, 0, 0},
                               {416, 0, 0, 1}, {480, 0, 0, 0}};
    constexpr int T1[10][4] = {{0, 2, 0, 1},    {64, 3, 0, 1},  {128, 5, 32, 0}, {160, 6, 0, 1},
                               {224, 5, 0, 1},  {288, 4, 32, 0}, {320, 1, 32, 0}, {352, 2, 0, 1},
                               {416, 1, 0, 1},  {480, 0, 32, 0}};
    SegIter si(U, G, g, KB);
    int it, kbs, kbe;
    while (si.next(it, kbs, kbe)) {
      const int cg = it / mpairs, pt = it - cg * mpairs;  // column-group major
      const int tile = 2 * pt + (int)crank;               // past mtiles: zero-filled by TMA
      for (int kb = kbs; kb < kbe; ++kb) {
        if (!is_a) {
          mbar_wait(&bempty[rb.s], rb.ph ^ 1u);
          if (i8::elect_one()) {
            if (crank == 0) mbar_arrive_expect_tx(&bfull[rb.s], 2 * C::B_STAGE);
            unsigned char* dst = ring_b + rb.s * C::B_STAGE;
#pragma unroll
            for (int i = 0; i < 10; ++i) {
              const int srow = crank ? T1[i][0] : T0[i][0];
              const int sl = crank ? T1[i][1] : T0[i][1];
              const int ro = crank ? T1[i][2] : T0[i][2];
              const bool big = crank ? T1[i][3] : T0[i][3];
              tc::tma_load_3d_pair(dst + srow * C::BK, big ? &mapB64 : &mapB32,
                                   bfull_l + 8u * (uint32_t)rb.s, kb * C::BK, cg * NC + ro, sl,
                                   pol_b);
            }
          }
          __syncwarp();
          rb.next();
          continue;
        }
        // lower-transposed mode: column tile J = kb / 2 left of the pair's 256 x 256 diagonal
        // super-block -> rows 64 (kb & 1) .. +63 of the stored tile (J, tile)'s k-blocks 2 tile,
        // 2 tile + 1 (an MN-major operand, two 64-row boxes; K1-i8s reads them the same way)
        const bool tr = args.lower_t && (kb >> 1) < 2 * pt;
#pragma unroll
        for (int s = 0; s < S; ++s) {
          mbar_wait(&aempty[ra.s], ra.ph ^ 1u);
          if (i8::elect_one()) {
            if (crank == 0) mbar_arrive_expect_tx(&afull[ra.s], 2 * C::A_TILE);
            unsigned char* dst = ring_a + ra.s * C::A_TILE;
            const uint32_t bar = afull_l + 8u * (uint32_t)ra.s;
            if (!tr) {
              tc::tma_load_3d_pair(dst, &mapA8, bar, 0, 0, (tile * KB + kb) * args.lS + s, pol_a);
            } else {
              const int blk = (kb >> 1) * KB + 2 * tile;  // past the tensor: zero-filled
              tc::tma_load_3d_pair(dst, &mapA8t, bar, 0, 64 * (kb & 1), blk * args.lS + s, pol_a);
              tc::tma_load_3d_pair(dst + C::A_TILE / 2, &mapA8t, bar, 0, 64 * (kb & 1),
                                   (blk + 1) * args.lS + s, pol_a);
            }
          }
          __syncwarp();
          ra.next();
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (pair leader)
    if (crank == 0) {
      RingI ra(C::NA), rb(C::NB);
      uint32_t tph = 0;
      SegIter si(U, G, g, KB);
      int it, kbs, kbe;
      const uint64_t adesc_ring = tc::sdesc_k_sw64(smem_u32(ring_a));
      // MN-major A (lower-transposed units): the two 64-byte M chunks 4 KB apart (LBO), a K step
      // of 32 rows = 2 KB; instruction-descriptor bit 15 = transpose A (tools/probe/i8_mn.cu)
      const uint64_t adesc_ring_t = (adesc_ring & ~(0x3FFFull << 16)) | ((uint64_t)(4096 >> 4) << 16);
      const uint64_t bdesc_ring = tc::sdesc_k_sw64(smem_u32(ring_b));
      // per A slice: up to two MMAs {B region row, N, TMEM column}
      constexpr int MM[7][2][3] = {{{0, 256, 0}, {128, 192, 256}},  {{0, 256, 64}, {224, 128, 320}},
                                   {{0, 256, 128}, {288, 64, 384}}, {{0, 256, 192}, {0, 0, 0}},
                                   {{320, 192, 256}, {0, 0, 0}},    {{416, 128, 320}, {0, 0, 0}},
                                   {{480, 64, 384}, {0, 0, 0}}};
      while (si.next(it, kbs, kbe)) {
        const int pt = it % mpairs;
        for (int k0 = kbs; k0 < kbe; k0 += kch) {
          const int k1 = min(kbe, k0 + kch);
          tc::mbar_wait_cluster(tempty, tph ^ 1u);  // both epilogues drained the accumulators
          tc::fence_after_sync();
          for (int kb = k0; kb < k1; ++kb) {
            tc::mbar_wait_cluster(&bfull[rb.s], rb.ph);
            const uint64_t bd0 = bdesc_ring + (uint64_t)(rb.s * (C::B_STAGE >> 4));
            const bool tr = args.lower_t && (kb >> 1) < 2 * pt;
            const uint32_t tbit = tr ? (1u << 15) : 0u;
#pragma unroll
            for (int s = 0; s < S; ++s) {
              tc::mbar_wait_cluster(&afull[ra.s], ra.ph);
              tc::fence_after_sync();
              const uint64_t ad0 = (tr ? adesc_ring_t : adesc_ring) +
                                   (uint64_t)(ra.s * (C::A_TILE >> 4));
              if (i8::elect_one()) {
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                  const uint32_t acc = (kb == k0 && s == 0 && ks == 0) ? 0u : 1u;
                  const uint64_t ad = ad0 + (uint64_t)(tr ? ks * (2048 >> 4) : ks * 2);
#pragma unroll
                  for (int m = 0; m < 2; ++m) {
                    if (MM[s][m][1] == 0) continue;
                    i8::mma_i8_pair(tmem + (uint32_t)MM[s][m][2], ad,
                                    bd0 + (uint64_t)((MM[s][m][0] * C::BK + ks * 32) >> 4),
                                    i8::idesc_i8(256, MM[s][m][1]) | tbit, acc);
                  }
                }
                tc::mma_commit_pair(&aempty[ra.s]);  // the slice stage is free in both CTAs
              }
              __syncwarp();
              ra.next();
            }
            if (i8::elect_one()) tc::mma_commit_pair(&bempty[rb.s]);
            __syncwarp();
            rb.next();
          }
          if (i8::elect_one()) tc::mma_commit_pair(tfull);
          __syncwarp();
          tph ^= 1u;
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue (4 warps, both CTAs)
    const int q = warp & 3;
    const int et = 32 * q + lane;  // row within this CTA's tile = TMEM lane
    const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t tempty_l = tc::mapa(smem_u32(tempty), 0);
    const double s1 = args.coef[0], s2 = args.coef[1], s3 = args.coef[2];
    double* accp = args.acc + (size_t)blockIdx.x * (NC * 128) + et;
    uint32_t tph = 0;
    SegIter si(U, G, g, KB);
    int it, kbs, kbe;
    auto drained = [&]() {  // this warp's TMEM reads are done: tell the leader's MMA warp
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_cluster(tempty_l);
    };
    // The CTA's last segment ends with every MMA complete and every ring stage consumed, so its
    // output tile is staged in the A ring (128 x 64 fp64, pitch 65) and written by rows:
    // coalesced Y_j / Y_{j-1} reads and out stores instead of one 512-byte row per lane
    // (the kernel's exposed tail, DESIGN.md §4 K1-i8p)
    double* stg = reinterpret_cast<double*>(ring_a);
    bool stage = false;
    int cg = 0, pt = 0;
    auto emit = [&](const double (&v)[C::CW], int c0) {
      const int row = (2 * pt + (int)crank) * C::BM + et;
      if (stage) {
        fence_proxy_async();  // after the tensor core's reads of the ring (tfull observed)
#pragma unroll
        for (int j = 0; j < C::CW; ++j) stg[et * 65 + c0 + j] = v[j];
        return;
      }
      if (row < args.n_rows) {
        const double rs = args.rscale[row];
        const int cbase = cg * NC + c0;
        const size_t o = (size_t)row * args.ldy + cbase;
#pragma unroll
        for (int j = 0; j < C::CW; ++j) {
          double y = s1 * (v[j] * rs * __ldg(args.cscale + cbase + j));
          if (s2 != 0.0) y = fma(s2, args.ycur[o + j], y);
          if (s3 != 0.0) y = fma(s3, args.yprev[o + j], y);
          args.out[o + j] = y;
        }
      }
    };
    double* srs = stg + C::BM * 65;  // the tile's row scales
    auto flush = [&]() {  // the staged tile -> out, 64 consecutive columns of a row per 2 warps
      const int r0 = (2 * pt + (int)crank) * C::BM;
      srs[et] = (r0 + et < args.n_rows) ? args.rscale[r0 + et] : 0.0;
      named_bar_sync(1, 128);
      const int c = et & 63;
      const double cs = __ldg(args.cscale + cg * NC + c);
      const int nr = min(C::BM, args.n_rows - r0);
      if (nr <= 0) return;  // the pair's second tile past n (uniform over the CTA)
      // 8 rows per batch: the batch's Y_j / Y_{j-1} loads are all in flight together
#pragma unroll 1
      for (int rb = 0; rb < C::BM; rb += 16) {
        double y[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = rb + 2 * i + (et >> 6);
          y[i] = s1 * (stg[r * 65 + c] * srs[r] * cs);
        }
        if (s2 != 0.0 || s3 != 0.0) {
          double a[8], b[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = rb + 2 * i + (et >> 6);
            const size_t o = (size_t)(r0 + min(r, nr - 1)) * args.ldy + cg * NC + c;
            a[i] = s2 != 0.0 ? args.ycur[o] : 0.0;
            b[i] = s3 != 0.0 ? args.yprev[o] : 0.0;
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (s2 != 0.0) y[i] = fma(s2, a[i], y[i]);
            if (s3 != 0.0) y[i] = fma(s3, b[i], y[i]);
          }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = rb + 2 * i + (et >> 6);
          if (r < nr) args.out[(size_t)(r0 + r) * args.ldy + cg * NC + c] = y[i];
        }
      }
    };
    while (si.next(it, kbs, kbe)) {
      cg = it / mpairs;
      pt = it - cg * mpairs;
      stage = si.u >= si.u1;  // last segment: the ring is idle once its accumulation completes
      const bool whole = (kbs == 0 && kbe == KB);
      int part = 0, nparts = 1;
      if (!whole) {
        const int f = seg_owner((long long)it * KB, U, G);
        part = g - f;
        nparts = seg_owner((long long)it * KB + KB - 1, U, G) - f + 1;
      }
      const int cit = 2 * it + (int)crank;  // this CTA's counter / partial slot
      double* mypart = args.part + ((size_t)cit * args.maxp + part) * (NC * 128) + et;
      if (!whole && kbe - kbs <= kch) {
        // ------------------------------------------------ split item, one accumulation
        mbar_wait(tfull, tph);
        tph ^= 1u;
        tc::fence_after_sync();
        named_bar_sync(1, 128);
        if (et == 0) *sflag = (atomicAdd(&args.counters[cit], 0) + 1 == nparts) ? 1 : 0;
        named_bar_sync(1, 128);
        const bool early = (*sflag != 0);
        named_bar_sync(1, 128);
        bool lastc = early;
        if (!early) {
#pragma unroll 1
          for (int c0 = 0; c0 < NC; c0 += C::CW) {
            double v[C::CW];
#pragma unroll
            for (int j = 0; j < C::CW; ++j) v[j] = 0.0;
            i8_combine_levels<S, NC, C::CW>(taddr, c0, v);
#pragma unroll
            for (int j = 0; j < C::CW; ++j) __stcg(mypart + (size_t)(c0 + j) * 128, v[j]);
          }
          drained();
          __threadfence();
          named_bar_sync(1, 128);
          if (et == 0) *sflag = (atomicAdd(&args.counters[cit], 1) + 1 == nparts) ? 1 : 0;
          named_bar_sync(1, 128);
          lastc = (*sflag != 0);
          named_bar_sync(1, 128);
        } else {
          __threadfence();
        }
        if (lastc) {
          const double* p0 = args.part + (size_t)cit * args.maxp * (NC * 128) + et;
#pragma unroll 1
          for (int c0 = 0; c0 < NC; c0 += C::CW) {
            double m[C::CW];
#pragma unroll
            for (int j = 0; j < C::CW; ++j) m[j] = 0.0;
            if (early) i8_combine_levels<S, NC, C::CW>(taddr, c0, m);
            double v[C::CW];
#pragma unroll
            for (int j = 0; j < C::CW; ++j) v[j] = 0.0;
#pragma unroll 1
            for (int q2 = 0; q2 < nparts; ++q2) {
              if (q2 == part && early) {
#pragma unroll
                for (int j = 0; j < C::CW; ++j) v[j] += m[j];
              } else {
#pragma unroll
                for (int j = 0; j < C::CW; ++j)
                  v[j] += __ldcg(p0 + (size_t)q2 * (NC * 128) + (size_t)(c0 + j) * 128);
              }
            }
            emit(v, c0);
          }
          if (stage) flush();
          if (et == 0) args.counters[cit] = 0;  // ready for the next launch
        }
        if (early) drained();
        continue;
      }
      for (int k0 = kbs; k0 < kbe; k0 += kch) {
        const bool first = (k0 == kbs), last = (k0 + kch >= kbe);
        mbar_wait(tfull, tph);
        tph ^= 1u;
        tc::fence_after_sync();
#pragma unroll 1
        for (int c0 = 0; c0 < NC; c0 += C::CW) {
          double v[C::CW];
#pragma unroll
          for (int j = 0; j < C::CW; ++j) v[j] = 0.0;
          i8_combine_levels<S, NC, C::CW>(taddr, c0, v);
          if (!first) {
#pragma unroll
            for (int j = 0; j < C::CW; ++j) v[j] += __ldcg(accp + (size_t)(c0 + j) * 128);
          }
          if (!last) {
#pragma unroll
            for (int j = 0; j < C::CW; ++j) __stcg(accp + (size_t)(c0 + j) * 128, v[j]);
          } else if (!whole) {
#pragma unroll
            for (int j = 0; j < C::CW; ++j) __stcg(mypart + (size_t)(c0 + j) * 128, v[j]);
          } else {
            emit(v, c0);
          }
        }
        drained();
        if (stage && last && whole) flush();
      }
      if (!whole) {
        // ------------------------------------------------ stream-K fixup (last contributor)
        __threadfence();
        named_bar_sync(1, 128);
        if (et == 0) *sflag = (atomicAdd(&args.counters[cit], 1) + 1 == nparts) ? 1 : 0;
        named_bar_sync(1, 128);
        const bool lastc = (*sflag != 0);
        named_bar_sync(1, 128);
        if (lastc) {
          __threadfence();
          const double* p0 = args.part + (size_t)cit * args.maxp * (NC * 128) + et;
#pragma unroll 1
          for (int c0 = 0; c0 < NC; c0 += C::CW) {
            double v[C::CW];
#pragma unroll
            for (int j = 0; j < C::CW; ++j) v[j] = 0.0;
#pragma unroll 1
            for (int q2 = 0; q2 < nparts; ++q2) {
#pragma unroll
              for (int j = 0; j < C::CW; ++j)
                v[j] += __ldcg(p0 + (size_t)q2 * (NC * 128) + (size_t)(c0 + j) * 128);
            }
            emit(v, c0);
          }
          if (stage) flush();
          if (et == 0) args.counters[cit] = 0;
        }
      }
    }
  }

  __syncwarp();
  tc::fence_before_sync();
  tc::cluster_sync();  // the peer's MMAs / TMEM reads are done before the pair's dealloc
  if (warp == 2) {
    tc::fence_after_sync();
    tc::tmem_dealloc_pair<C::TMEM_COLS>(tmem);
  }
}

// ------------------------------------------------------------------------------ symmetric A
// Half-storage filter product for a SYMMETRIC A whose digit slices share one scale (the fused
// PFAM digits, scale 2^Eg for every row; DESIGN.md §4 "K1-i8s"): only the 128 x 128 tiles
// (I, J >= I) of the tiled layout are read.  CTA I owns row tile I and walks the column tiles in
// the order J = (t - I) mod T, t = 0 .. T-1: the lower tiles (J < I) are the stored tiles (J, I)
// read transposed -- an MN-major A operand (two 64-row boxes of tile J's k-blocks 2I, 2I+1;
// descriptor LBO = 4096 between the two 64-byte M chunks, SBO = 512 between 8-row K groups,
// instruction-descriptor transpose-A bit; tools/probe/i8_mn.cu checks it bit-exactly).  Stored
// tile (a, b) is needed by CTA a and CTA b at the same step t = a + b (mod T), so the second read
// of every off-diagonal tile is an L2 hit while the CTAs advance together: HBM reads 7n²/2
// bytes instead of 7n².  One CTA per row tile (T <= SMs), no K split: the whole K range is one
// exact int32 accumulation (K <= chunk_kb k-blocks), the epilogue runs once.  S = 7, NC = p = 64.
constexpr int kSymS = 7, kSymNC = 64;
using SymCfg = I8Cfg<kSymS, kSymNC>;

__global__ void __launch_bounds__(SymCfg::THREADS, 1)
    cheb_gemm_i8s_kernel(const __grid_constant__ CUtensorMap mapA8,
                         const __grid_constant__ CUtensorMap mapA8t,
                         const __grid_constant__ CUtensorMap mapY8, I8Args args) {
  using C = SymCfg;
  constexpr int S = kSymS, NC = kSymNC;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* ring_a = smem;                              // NA x 8 KB
  unsigned char* ring_b = smem + C::NA * C::A_TILE;          // NB x [S][NC][64] int8
  uint64_t* afull = reinterpret_cast<uint64_t*>(ring_b + C::NB * C::B_STAGE);
  uint64_t* aempty = afull + C::NA;
  uint64_t* bfull = aempty + C::NA;
  uint64_t* bempty = bfull + C::NB;
  uint64_t* tfull = bempty + C::NB;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NA; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], 1);
    }
    for (int s = 0; s < C::NB; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&bempty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mapA8);
    tma_prefetch_desc(&mapA8t);
    tma_prefetch_desc(&mapY8);
  }
  if (warp == 2) i8::tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  const int KB = args.kblocks, T = args.mtiles, I = blockIdx.x;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    RingI ra(C::NA), rb(C::NB);
    const uint64_t pol_b = tc::policy_evict_last();
    const uint64_t pol_d = tc::policy_evict_first();  // diagonal tiles: read once
    for (int t = 0; t < T; ++t) {
      const int J = (t - I + T) % T;
      for (int kk = 0; kk < 2; ++kk) {
        const int kb = 2 * J + kk;
        if (kb >= KB) break;
        mbar_wait(&bempty[rb.s], rb.ph ^ 1u);
        if (i8::elect_one()) {
          mbar_arrive_expect_tx(&bfull[rb.s], C::B_LOAD);
          tc::tma_load_3d_hint(ring_b + rb.s * C::B_STAGE, &mapY8, &bfull[rb.s], kb * C::BK, 0,
                               0, pol_b);
        }
        __syncwarp();
        rb.next();
#pragma unroll 1
        for (int s = 0; s < S; ++s) {
          mbar_wait(&aempty[ra.s], ra.ph ^ 1u);
          if (i8::elect_one()) {
            unsigned char* dst = ring_a + ra.s * C::A_TILE;
            if (J >= I) {  // stored tile (I, J): K-major box of k-block kb
              mbar_arrive_expect_tx(&afull[ra.s], C::A_TILE);
              if (J == I)
                tc::tma_load_3d_hint(dst, &mapA8, &afull[ra.s], 0, 0, (I * KB + kb) * args.lS + s,
                                     pol_d);
              else
                tc::tma_load_3d(dst, &mapA8, &afull[ra.s], 0, 0, (I * KB + kb) * args.lS + s);
            } else {  // stored tile (J, I) transposed: rows 64 kk.. of its k-blocks 2I, 2I+1
              const bool two = 2 * I + 1 < KB;
              mbar_arrive_expect_tx(&afull[ra.s], two ? C::A_TILE : C::A_TILE / 2);
              tc::tma_load_3d(dst, &mapA8t, &afull[ra.s], 0, 64 * kk,
                              (J * KB + 2 * I) * args.lS + s);
              if (two)
                tc::tma_load_3d(dst + C::A_TILE / 2, &mapA8t, &afull[ra.s], 0, 64 * kk,
                                (J * KB + 2 * I + 1) * args.lS + s);
            }
          }
          __syncwarp();
          ra.next();
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    RingI ra(C::NA), rb(C::NB);
    const uint32_t ring_a0 = smem_u32(ring_a), ring_b0 = smem_u32(ring_b);
    bool first = true;
    for (int t = 0; t < T; ++t) {
      const int J = (t - I + T) % T;
      const bool tr = J < I;
      for (int kk = 0; kk < 2; ++kk) {
        const int kb = 2 * J + kk;
        if (kb >= KB) break;
        mbar_wait(&bfull[rb.s], rb.ph);
        const uint32_t b0 = ring_b0 + rb.s * C::B_STAGE;
#pragma unroll
        for (int s = 0; s < S; ++s) {
          mbar_wait(&afull[ra.s], ra.ph);
          tc::fence_after_sync();
          const uint32_t a0 = ring_a0 + ra.s * C::A_TILE;
          if (i8::elect_one()) {
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
              const uint32_t acc = (first && s == 0 && ks == 0) ? 0u : 1u;
              // K-major: 32-byte K step inside the 64-byte rows; MN-major: 32 rows of K (2 KB),
              // the two 64-byte M chunks 4 KB apart
              const uint64_t ad = tr ? (tc::sdesc_k_sw64(a0 + ks * 2048) & ~(0x3FFFull << 16)) |
                                           ((uint64_t)(4096 >> 4) << 16)
                                     : tc::sdesc_k_sw64(a0 + ks * 32);
              const uint32_t tbit = tr ? (1u << 15) : 0u;
#pragma unroll
              for (int t0 = 0; t0 < S - s; t0 += C::CMAX) {
                const int c = (S - s - t0) < C::CMAX ? (S - s - t0) : C::CMAX;
                i8::mma_i8(tmem + (uint32_t)((s + t0) * NC), ad,
                           tc::sdesc_k_sw64(b0 + t0 * NC * C::BK + ks * 32),
                           i8::idesc_i8(C::BM, c * NC) | tbit, acc);
              }
            }
            i8::mma_commit(&aempty[ra.s]);
          }
          __syncwarp();
          ra.next();
        }
        first = false;
        if (i8::elect_one()) i8::mma_commit(&bempty[rb.s]);
        __syncwarp();
        rb.next();
      }
    }
    if (i8::elect_one()) i8::mma_commit(tfull);
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue (4 warps)
    const int q = warp & 3;
    const int et = 32 * q + lane;
    const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16);
    const double s1 = args.coef[0], s2 = args.coef[1], s3 = args.coef[2];
    const int row = I * C::BM + et;
    const bool row_ok = row < args.n_rows;
    const double rs = row_ok ? args.rscale[row] : 0.0;
    mbar_wait(tfull, 0);
    tc::fence_after_sync();
#pragma unroll 1
    for (int c0 = 0; c0 < NC; c0 += C::CW) {
      double v[C::CW];
#pragma unroll
      for (int j = 0; j < C::CW; ++j) v[j] = 0.0;
      i8_combine_levels<S, NC, C::CW>(taddr, c0, v);
      if (row_ok) {
        const size_t o = (size_t)row * args.ldy + c0;
#pragma unroll
        for (int j = 0; j < C::CW; ++j) {
          double y = s1 * (v[j] * rs * __ldg(args.cscale + c0 + j));
          if (s2 != 0.0) y = fma(s2, args.ycur[o + j], y);
          if (s3 != 0.0) y = fma(s3, args.yprev[o + j], y);
          args.out[o + j] = y;
        }
      }
    }
  }

  __syncwarp();
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 2) {
    tc::fence_after_sync();
    i8::tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// ------------------------------------------------------------------------------ host side
bool encode_map_i8_3d(CUtensorMap* map, const int8_t* base, int64_t pitch, int64_t slice_pitch,
                      int cols, int rows, int slices, int box_rows, int box_slices,
                      bool swizzle = true);

I8Plan i8_plan(int p, int n_rows, int n_k, int slices, int num_sms) {
  I8Plan pl;
  pl.p = p;
  pl.S = slices;
  pl.n_rows = n_rows;
  pl.n_k = n_k;
  pl.NC = std::min(p, 64);
  pl.ngroups = p / pl.NC;
  pl.mtiles = (n_rows + 127) / 128;
  pl.kblocks = (n_k + 63) / 64;
  pl.kpad = ((int64_t)n_k + 15) / 16 * 16;
  // exact int32 level sums: S K 128^2 < 2^31 for the deepest level (S products)
  const long long kmax = 2147483647LL / ((long long)slices * 128 * 128);  // |d| <= 128
  pl.chunk_kb = (int)std::max(1LL, kmax / 64);
  const long long items = (long long)pl.mtiles * pl.ngroups;
  const long long U = items * pl.kblocks;
  // stream-K: every SM gets an equal share of the (tile, k-block) units, at least 8 k-blocks
  pl.grid = (int)std::max(1LL, std::min<long long>(num_sms, U / 8));
  if (const char* e = getenv("PF_I8_GRID")) pl.grid = std::max(1, std::min(pl.grid, atoi(e)));  // dev
  const long long per = U / pl.grid;  // fewest units a CTA owns
  pl.maxp = (int)std::min<long long>(pl.grid, (pl.kblocks + per - 1) / per + 1);
  pl.items = (int)items;
  pl.acc_doubles = (size_t)pl.grid * pl.NC * 128;
  pl.part_doubles = (size_t)items * pl.maxp * pl.NC * 128;
  pl.pf_dist = 0;
  if (const char* e = getenv("PF_I8_PFDIST")) pl.pf_dist = atoi(e);  // development knob
  // K1-i8p: CTA pairs (PF_I8PAIR=0 keeps the one-CTA kernel); workspaces sized for both
  pl.pair = 0;
  pl.pgrid = pl.grid;
  pl.pmaxp = pl.maxp;
  const char* ep = getenv("PF_I8PAIR");
  if (slices == 7 && pl.NC == 64 && num_sms >= 2 && !(ep && ep[0] == '0')) {
    const long long pit = (long long)((pl.mtiles + 1) / 2) * pl.ngroups;
    const long long PU = pit * pl.kblocks;
    const long long G2 = std::max(1LL, std::min<long long>(pl.grid / 2, PU / 8));
    const long long pper = PU / G2;
    pl.pair = 1;
    pl.pgrid = (int)(2 * G2);
    pl.pmaxp = (int)std::min<long long>(G2, (pl.kblocks + pper - 1) / pper + 1);
    pl.part_doubles = std::max(pl.part_doubles, (size_t)(pit * pl.pmaxp * 2) * pl.NC * 128);
    pl.items = std::max<int>(pl.items, (int)(2 * pit));
    pl.acc_doubles = std::max(pl.acc_doubles, (size_t)pl.pgrid * pl.NC * 128);
  }
  return pl;
}

bool i8_encode_A(CUtensorMap* map, CUtensorMap* map_pf, const int8_t* A8, const I8Plan& pl) {
  // tiled layout: 8 KB blocks (64 bytes x 128 rows), one per (tile, k-block, slice)
  const int blocks = pl.mtiles * pl.kblocks * pl.S;
  return encode_map_i8_3d(map, A8, 64, 8192, 64, 128, blocks, 128, 1) &&
         encode_map_i8_3d(map_pf, A8, 64, 8192, 64, 128, blocks, 128,
                          pl.S, false);
}
bool i8_encode_B(CUtensorMap* map, const int8_t* Y8, const I8Plan& pl, int su) {
  return encode_map_i8_3d(map, Y8, pl.kpad, pl.kpad * pl.p, pl.n_k, pl.p, pl.S, pl.NC, su);
}
// K1-i8p B boxes: 64 or 32 rows of one slice
bool i8_encode_B_pair(CUtensorMap* map64, CUtensorMap* map32, const int8_t* Y8, const I8Plan& pl) {
  return encode_map_i8_3d(map64, Y8, pl.kpad, pl.kpad * pl.p, pl.n_k, pl.p, pl.S, 64, 1) &&
         encode_map_i8_3d(map32, Y8, pl.kpad, pl.kpad * pl.p, pl.n_k, pl.p, pl.S, 32, 1);
}

template <int S>
static cudaError_t a_split_s(const double* A, int64_t lda, const I8Plan& pl, int8_t* A8,
                             double* rscale, int num_sms, cudaStream_t st) {
  count_launch();
  a_split_kernel<S><<<std::min(pl.n_rows, 2 * num_sms), 512, 0, st>>>(A, lda, pl.n_rows, pl.n_k,
                                                                      A8, pl.kblocks, rscale);
  return cudaGetLastError();
}
cudaError_t i8_split_A_launch(const double* A, int64_t lda, const I8Plan& pl, int8_t* A8,
                              double* rscale, int num_sms, cudaStream_t st) {
  switch (pl.S) {
    case 6: return a_split_s<6>(A, lda, pl, A8, rscale, num_sms, st);
    case 7: return a_split_s<7>(A, lda, pl, A8, rscale, num_sms, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int S>
static cudaError_t y_split_s(const double* Y, int64_t ldy, const I8Plan& pl,
                             unsigned long long* cmax, int8_t* Y8, double* cscale,
                             int num_sms, cudaStream_t st) {
  static int per_sm = 0;
  if (!per_sm) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, y_colmax_split_kernel<S>, 256, 0);
    per_sm = std::max(1, std::min(per_sm, 4));
  }
  const int chunks = (pl.n_k + 31) / 32;
  int n_k = pl.n_k, p = pl.p;
  int64_t kpad = pl.kpad;
  void* args[] = {(void*)&Y, (void*)&ldy, (void*)&n_k, (void*)&p, (void*)&cmax, (void*)&Y8,
                  (void*)&kpad, (void*)&cscale};
  static int per_sm_t = 0;
  if (!per_sm_t) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_t, y_split_tile_kernel<S>, 256, 0);
    per_sm_t = std::max(1, per_sm_t);
  }
  if (p <= 64 && (ldy % 2) == 0 && chunks <= per_sm_t * num_sms) {
    count_launch();
    return cudaLaunchCooperativeKernel((const void*)y_split_tile_kernel<S>, dim3(chunks),
                                       dim3(256), args, 0, st);
  }
  const int grid = std::max(1, std::min(chunks, per_sm * num_sms));
  count_launch();
  return cudaLaunchCooperativeKernel((const void*)y_colmax_split_kernel<S>, dim3(grid), dim3(256),
                                     args, 0, st);
}
cudaError_t i8_split_Y_launch(const double* Y, int64_t ldy, const I8Plan& pl,
                              unsigned long long* cmax, int8_t* Y8, double* cscale, int num_sms,
                              cudaStream_t st) {
  switch (pl.S) {
    case 6: return y_split_s<6>(Y, ldy, pl, cmax, Y8, cscale, num_sms, st);
    case 7: return y_split_s<7>(Y, ldy, pl, cmax, Y8, cscale, num_sms, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int S, int NC>
static cudaError_t i8_launch_t(const I8Plan& pl, const CUtensorMap& mapA8,
                               const CUtensorMap& mapY8, const CUtensorMap& mapA8pf,
                               const I8Args& a, cudaStream_t st) {
  using C = I8Cfg<S, NC>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(cheb_gemm_i8_kernel<S, NC>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  count_launch();
  cheb_gemm_i8_kernel<S, NC><<<pl.grid, C::THREADS, C::SMEM, st>>>(mapA8, mapY8, mapA8pf, a);
  return cudaGetLastError();
}

template <int S>
static cudaError_t i8_launch_s(const I8Plan& pl, const CUtensorMap& mapA8,
                               const CUtensorMap& mapY8, const CUtensorMap& mapA8pf,
                               const I8Args& a, cudaStream_t st) {
  switch (pl.NC) {
    case 16: return i8_launch_t<S, 16>(pl, mapA8, mapY8, mapA8pf, a, st);
    case 32: return i8_launch_t<S, 32>(pl, mapA8, mapY8, mapA8pf, a, st);
    case 64: return i8_launch_t<S, 64>(pl, mapA8, mapY8, mapA8pf, a, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t i8_gemm_launch(const I8Plan& pl, const CUtensorMap& mapA8, const CUtensorMap& mapY8,
                           const CUtensorMap& mapA8pf, const double* rscale, const double* cscale, const double* ycur,
                           const double* yprev, double* out, int64_t ldy, const double* coef,
                           double* acc, double* part, int* counters, int su, cudaStream_t st,
                           const CUtensorMap* mapB64, const CUtensorMap* mapB32,
                           const CUtensorMap* mapA8t) {
  // su <= pl.S: only the su most significant digit slices of both operands are multiplied --
  // exactly the su-digit expansion (the digits of a longer truncating expansion start with
  // those of a shorter one), levels 2..su+1; the B map must have a box of su slices
  I8Args a = {};
  a.part = part;
  a.counters = counters;
  a.maxp = pl.maxp;
  a.ycur = ycur;
  a.yprev = yprev;
  a.out = out;
  a.ldy = ldy;
  a.coef = coef;
  a.rscale = rscale;
  a.cscale = cscale;
  a.acc = acc;
  a.n_rows = pl.n_rows;
  a.kblocks = pl.kblocks;
  a.mtiles = pl.mtiles;
  a.ngroups = pl.ngroups;
  a.chunk_kb = pl.chunk_kb;
  a.pf_dist = pl.pf_dist;
  a.lS = pl.S;
  if (su < 4 || su > pl.S) return cudaErrorInvalidValue;
  if (pl.pair && su == 7 && pl.S == 7 && mapB64 && mapB32) {
    static bool attr_p = false;
    if (!attr_p) {
      cudaError_t e = cudaFuncSetAttribute(cheb_gemm_i8p_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           I8PCfg::SMEM);
      if (e != cudaSuccess) return e;
      attr_p = true;
    }
    a.maxp = pl.pmaxp;
    a.lower_t = mapA8t ? 1 : 0;
    count_launch();
    cheb_gemm_i8p_kernel<<<pl.pgrid, I8PCfg::THREADS, I8PCfg::SMEM, st>>>(
        mapA8, *mapB64, *mapB32, mapA8t ? *mapA8t : mapA8, a);
    return cudaGetLastError();
  }
  switch (su) {
    case 4: return i8_launch_s<4>(pl, mapA8, mapY8, mapA8pf, a, st);
    case 5: return i8_launch_s<5>(pl, mapA8, mapY8, mapA8pf, a, st);
    case 6: return i8_launch_s<6>(pl, mapA8, mapY8, mapA8pf, a, st);
    case 7: return i8_launch_s<7>(pl, mapA8, mapY8, mapA8pf, a, st);
    default: return cudaErrorInvalidValue;
  }
}

// the symmetric kernel applies: one GPU's whole matrix, p = 64, S = 7 slices used, one CTA per row
// tile, one exact accumulation over K
bool i8s_supported(const I8Plan& pl, int num_sms) {
  return pl.p == 64 && pl.S == 7 && pl.n_rows == pl.n_k && pl.mtiles <= num_sms &&
         pl.kblocks <= pl.chunk_kb;
}
bool i8s_encode_At(CUtensorMap* map, const int8_t* A8, const I8Plan& pl) {
  const int blocks = pl.mtiles * pl.kblocks * pl.S;
  return encode_map_i8_3d(map, A8, 64, 8192, 64, 128, blocks, 64, 1);
}
cudaError_t i8s_gemm_launch(const I8Plan& pl, const CUtensorMap& mapA8, const CUtensorMap& mapA8t,
                            const CUtensorMap& mapY8, const double* rscale, const double* cscale,
                            const double* ycur, const double* yprev, double* out, int64_t ldy,
                            const double* coef, cudaStream_t st) {
  I8Args a = {};
  a.ycur = ycur;
  a.yprev = yprev;
  a.out = out;
  a.ldy = ldy;
  a.coef = coef;
  a.rscale = rscale;
  a.cscale = cscale;
  a.n_rows = pl.n_rows;
  a.kblocks = pl.kblocks;
  a.mtiles = pl.mtiles;
  a.lS = pl.S;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(cheb_gemm_i8s_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, SymCfg::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  count_launch();
  cheb_gemm_i8s_kernel<<<pl.mtiles, SymCfg::THREADS, SymCfg::SMEM, st>>>(mapA8, mapA8t, mapY8, a);
  return cudaGetLastError();
}

}  // namespace pf
