// pf_rebuild_i8.cu -- the PFAM update (step a6, eq:PFAM1 P:389 with the corrected prox, reading
// R1) on one GPU for PF_FP64_I8 contexts, with the rank-p product W = V' V^T formed from EXACT
// int8 tensor-core products (tcgen05 kind::i8) of 7-bit digit slices -- the same Ozaki-style
// splitting as the filter GEMM K1-i8 (pf_gemm_i8.cu):
//
//     V' = V diag(f) (or Q F, pf_admm_step_f),  V'_i = 2^{E_i} sum_s d_s 128^-(s+1) + r,
//     V_j = 2^{F_j} sum_t e_t 128^-(t+1) + r',   W_ij = 2^{E_i + F_j} sum_l 128^-(l+2) D_l[i][j],
//     D_l = sum_{s+t=l} A_s B_t^T  (exact int32, K = p = 64 digits: one 64-byte k-block)
//
// then Z_new = offdiag(W - tC) + Diag(1 - W_ii + Z_ii), written with its mirror and (fused
// digits) the digit slices of Z_new for the next filter.  Why: the fp64 DMMA formulation
// (rebuild_kernel) spends ~0.46 ms of DMMA pipe time on W at config 3 and cannot overlap it with
// the 5.1 GB HBM stream inside its CTAs (1.64 ms, DRAM ~37%); here W costs ~0.18 ms of tensor
// time issued by one thread, accumulates in TMEM (two buffers), and 8 update warps do nothing
// but the memory-bound update while the tensor core fills the other buffer.
//
// Tiles: 128 rows (a block I of V') x 32 columns (a block J of V), J * 32 >= I * 128 (upper part;
// the 4 tiles J = 4I .. 4I+3 cover the 128 x 128 diagonal block, both triangles, no mirror).
// Warp 0: TMA (A = the 7 slices of V' block I, 56 KB, reloaded when I changes; B = the 7 slices
// of V block J, 14 KB, 4-stage ring).  Warp 1: 14 MMAs per tile (A_s x [B_0 .. B_{6-s}], N =
// 32 (7 - s), levels s .. 6 at TMEM columns 32 s ..).  Warps 4-11: TMEM lane = tile row,
// 16 columns each: levels combined in fp64, the update, fp64 stores (tile rows, and mirror rows
// coalesced across the warp), digit slices (tile words directly, mirror words by 4 x 4 byte
// transposes across 4 lanes).  Deterministic sums (fixed per-thread order, CTA partials summed
// in CTA order by the last CTA).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "pf_digits.cuh"
#include "pf_i8mma.cuh"
#include "pf_kernels.cuh"
#include "pf_tc.cuh"

namespace pf {

constexpr int kR8S = 7;                       // digit slices of V' and V
constexpr int kR8M = 128, kR8N = 32;          // tile
constexpr int kR8BS = 4;                      // B ring stages
constexpr int kR8Threads = 384;               // w0 TMA, w1 MMA, w2 TMEM, w3 idle, w4..11 update
constexpr int kR8A = kR8S * 8192;             // A bytes (7 slices x 128 rows x 64 B)
constexpr int kR8B = kR8S * 2048;             // B bytes per stage (7 slices x 32 rows x 64 B)
constexpr int kR8Smem = 1024 + kR8A + kR8BS * kR8B + 256;

struct R8Args {
  const double* rsA;  // [n] 2^E_i of V' rows
  const double* rsB;  // [n] 2^F_j of V rows
  const uint32_t* bits;
  int64_t ldb;
  const double* deg;
  double tt;
  double* Z;
  int64_t ldz;
  int n, TC, MT;
  int8_t* A8;         // fused digit output (nullptr: none)
  int KB, S;
  const int* E;       // global digit exponent of Z_new
  double* rscale;
  double* partials;
  int* counter;
  double* obj;
};

// tile e -> (I, J): rows I of 128 (I < MT), columns J of 32 from 4I to TC - 1; cnt(I) = tiles
// before row block I = I TC - 2 I (I - 1)
__device__ __forceinline__ void r8_tile(long long e, int TC, int MT, int& I, int& J) {
  const double b = (double)TC + 2.0;
  double disc = b * b - 8.0 * (double)e;
  int i = (int)floor((b - sqrt(fmax(disc, 0.0))) * 0.25);
  i = max(0, min(MT - 1, i));
  auto cnt = [&](long long x) { return x * TC - 2 * x * (x - 1); };
  while (i > 0 && cnt(i) > e) --i;
  while (i + 1 < MT && cnt(i + 1) <= e) ++i;
  I = i;
  J = 4 * i + (int)(e - cnt(i));
}

__global__ void __launch_bounds__(kR8Threads, 1)
    rebuild_i8_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                      const R8Args a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* sA = smem;
  unsigned char* sB = smem + kR8A;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + kR8BS * kR8B);
  uint64_t* afull = bars;           // A landed
  uint64_t* aempty = bars + 1;      // MMAs that read A (this row block) complete
  uint64_t* bfull = bars + 2;       // [4]
  uint64_t* bempty = bars + 6;      // [4]
  uint64_t* tfull = bars + 10;      // [2] accumulator buffer complete
  uint64_t* tempty = bars + 12;     // [2] accumulator buffer drained (8 update warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);
  __shared__ double red[32];
  __shared__ int s_last;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(afull, 1);
    mbar_init(aempty, 1);
    for (int q = 0; q < kR8BS; ++q) {
      mbar_init(&bfull[q], 1);
      mbar_init(&bempty[q], 1);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&tfull[q], 1);
      mbar_init(&tempty[q], 8);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mapA);
    tma_prefetch_desc(&mapB);
  }
  if (warp == 2) i8::tmem_alloc(tmem_slot, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  const long long ntiles = (long long)a.MT * a.TC - 2LL * a.MT * (a.MT - 1);
  const long long t_begin = ntiles * blockIdx.x / gridDim.x;
  const long long t_end = ntiles * (blockIdx.x + 1) / gridDim.x;
  double s0 = 0.0, s1 = 0.0;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    int curI = -1;
    uint32_t aeph = 0;
    int bs = 0;
    uint32_t bph = 0;
    const uint64_t pol = tc::policy_evict_last();  // V' and V digits are re-read (L2)
    for (long long t = t_begin; t < t_end; ++t) {
      int I, J;
      r8_tile(t, a.TC, a.MT, I, J);
      if (I != curI) {
        if (curI >= 0) {
          mbar_wait(aempty, aeph);
          aeph ^= 1u;
        }
        if (i8::elect_one()) {
          mbar_arrive_expect_tx(afull, kR8A);
          tc::tma_load_3d_hint(sA, &mapA, afull, 0, 0, I * kR8S, pol);
        }
        __syncwarp();
        curI = I;
      }
      mbar_wait(&bempty[bs], bph ^ 1u);
      if (i8::elect_one()) {
        mbar_arrive_expect_tx(&bfull[bs], kR8B);
        const int j0 = J * kR8N;
        tc::tma_load_3d_hint(sB + bs * kR8B, &mapB, &bfull[bs], 0, j0 & 127, (j0 >> 7) * kR8S, pol);
      }
      __syncwarp();
      if (++bs == kR8BS) {
        bs = 0;
        bph ^= 1u;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    int curI = -1;
    uint32_t aph = 0;
    int bs = 0;
    uint32_t bph = 0;
    uint32_t tph[2] = {0u, 0u};
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    int it = 0;
    for (long long t = t_begin; t < t_end; ++t, ++it) {
      int I, J;
      r8_tile(t, a.TC, a.MT, I, J);
      if (I != curI) {
        mbar_wait(afull, aph);
        aph ^= 1u;
        curI = I;
      }
      const int buf = it & 1;
      mbar_wait(&tempty[buf], tph[buf] ^ 1u);  // the update warps drained this buffer
      tph[buf] ^= 1u;
      mbar_wait(&bfull[bs], bph);
      tc::fence_after_sync();
      int In = -1, Jn;
      if (t + 1 < t_end) r8_tile(t + 1, a.TC, a.MT, In, Jn);
      if (i8::elect_one()) {
        const uint32_t bst = b0 + bs * kR8B;
#pragma unroll
        for (int s = 0; s < kR8S; ++s)
#pragma unroll
          for (int ks = 0; ks < 2; ++ks)
            i8::mma_i8(tmem + (uint32_t)(buf * 256 + s * kR8N),
                       tc::sdesc_k_sw64(a0 + s * 8192 + ks * 32),
                       tc::sdesc_k_sw64(bst + ks * 32), i8::idesc_i8(kR8M, kR8N * (kR8S - s)),
                       (s | ks) ? 1u : 0u);
        i8::mma_commit(&bempty[bs]);
        i8::mma_commit(&tfull[buf]);
        if (In != I) i8::mma_commit(aempty);  // the next tile loads another row block of V'
      }
      __syncwarp();
      if (++bs == kR8BS) {
        bs = 0;
        bph ^= 1u;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ update warps
    const int q = warp & 3, h = (warp - 4) >> 2;
    const int r = 32 * q + lane;  // tile row = TMEM lane
    const bool dig = a.A8 != nullptr;
    const int Eg = dig ? *a.E : 0;
    if (dig) {
      const double sc = i8::pow2(Eg);
      for (int i = blockIdx.x * 256 + (threadIdx.x - 128); i < a.n; i += gridDim.x * 256)
        a.rscale[i] = sc;
    }
    const double qt = 0.25 * a.tt;
    uint32_t tph[2] = {0u, 0u};
    double zo[16];
    auto load_zo = [&](long long t) {
      int I, J;
      r8_tile(t, a.TC, a.MT, I, J);
      const int i = I * kR8M + r, jb = J * kR8N + 16 * h;
      const double* zr = a.Z + (size_t)i * a.ldz + jb;
      if (i < a.n && jb + 16 <= a.n) {
#pragma unroll
        for (int c = 0; c < 16; c += 2) {
          const double2 v = __ldcs(reinterpret_cast<const double2*>(zr + c));
          zo[c] = v.x;
          zo[c + 1] = v.y;
        }
      } else {
#pragma unroll
        for (int c = 0; c < 16; ++c) zo[c] = (i < a.n && jb + c < a.n) ? zr[c] : 0.0;
      }
    };
    if (t_begin < t_end) load_zo(t_begin);
    int it = 0;
    for (long long t = t_begin; t < t_end; ++t, ++it) {
      int I, J;
      r8_tile(t, a.TC, a.MT, I, J);
      const int i0 = I * kR8M, j0 = J * kR8N;
      const int i = i0 + r, jb = j0 + 16 * h;
      const bool diagblk = J < 4 * I + 4;            // inside the 128 x 128 diagonal block
      const bool interior = (i0 + kR8M <= a.n) && (j0 + kR8N <= a.n);
      const bool fast = interior && !diagblk;
      const uint32_t word = (i < a.n) ? (__ldg(a.bits + (size_t)i * a.ldb + (jb >> 5)) >> (jb & 31)) : 0u;
      const double rs = (i < a.n) ? a.rsA[i] : 0.0;
      double cs[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) cs[c] = (jb + c < a.n) ? __ldg(a.rsB + jb + c) : 0.0;
      // ---- W from the TMEM levels (smallest weight first)
      const int buf = it & 1;
      mbar_wait(&tfull[buf], tph[buf]);
      tph[buf] ^= 1u;
      tc::fence_after_sync();
      double w[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) w[c] = 0.0;
      const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * 256 + 16 * h);
#pragma unroll 1
      for (int L = kR8S - 1; L >= 0; --L) {
        uint32_t rr[16];
        i8::tmem_ld16(taddr + (uint32_t)(L * kR8N), rr);
        const double wl = i8::pow2(-7 * (L + 2));
#pragma unroll
        for (int c = 0; c < 16; ++c) w[c] = fma((double)(int)rr[c], wl, w[c]);
      }
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);  // the MMA may refill this buffer
#pragma unroll
      for (int c = 0; c < 16; ++c) w[c] *= rs * cs[c];  // exact: powers of two
      // ---- Z_new
      double z[16];
      if (fast) {
        double ts0 = 0.0, ts1 = 0.0;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const bool b = (word >> c) & 1u;
          const double x = w[c];
          const double o = b ? x - qt : x;          // W_ij - t C_ij, C_ij = adj_ij / 4
          ts0 += b ? x : 0.0;
          const double e = o - zo[c];
          ts1 = fma(e, e, ts1);
          z[c] = o;
        }
        s0 += 2.0 * 0.25 * ts0;
        s1 += 2.0 * ts1;
      } else {
        const double wgt = diagblk ? 1.0 : 2.0;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const int j = jb + c;
          z[c] = 0.0;
          if (i >= a.n || j >= a.n) continue;
          const bool b = (word >> c) & 1u;
          const double x = w[c], zold = zo[c];
          double o;
          if (j == i) {
            o = 1.0 - x + zold;                    // Diag(1 - W_ii + Z_ii)
            s0 += -0.25 * a.deg[i] * x;            // C_ii = -deg_i / 4
            s1 += (o - zold) * (o - zold);
          } else {
            o = b ? x - qt : x;
            if (b) s0 += wgt * 0.25 * x;
            s1 += wgt * (o - zold) * (o - zold);
          }
          z[c] = o;
        }
      }
      // the next tile's Z_old (its HBM latency overlaps the stores and digits below)
      if (t + 1 < t_end) load_zo(t + 1);
      // ---- fp64 stores: the tile row piece (128 B) and, off the diagonal block, the mirror
      if (i < a.n) {
        double* zr = a.Z + (size_t)i * a.ldz + jb;
        if (jb + 16 <= a.n && ((reinterpret_cast<uintptr_t>(zr) & 15) == 0)) {
#pragma unroll
          for (int c = 0; c < 16; c += 2)
            __stcs(reinterpret_cast<double2*>(zr + c), make_double2(z[c], z[c + 1]));
        } else {
#pragma unroll
          for (int c = 0; c < 16; ++c)
            if (jb + c < a.n) zr[c] = z[c];
        }
        if (!diagblk) {
#pragma unroll
          for (int c = 0; c < 16; ++c)  // warp: 32 consecutive rows of mirror row jb + c
            if (jb + c < a.n) __stcs(a.Z + (size_t)(jb + c) * a.ldz + i, z[c]);
        }
      }
      if (!dig) continue;
      // ---- digit slices of Z_new (one scale 2^Eg, DESIGN.md §4 "fused digits")
      uint32_t dw[4][kR8S];
#pragma unroll
      for (int g = 0; g < 4; ++g)
        i8::slices4<kR8S>(z[4 * g], z[4 * g + 1], z[4 * g + 2], z[4 * g + 3], Eg, dw[g]);
      if (i < a.n && jb < a.n) {  // tile row: 16 digits per slice
        int8_t* base = a.A8 + i8::a8_offset(i, jb, 0, a.KB, kR8S);
#pragma unroll
        for (int sl = 0; sl < kR8S; ++sl)
          __stcs(reinterpret_cast<uint4*>(base + sl * 8192),
                 make_uint4(dw[0][sl], dw[1][sl], dw[2][sl], dw[3][sl]));
      }
      if (!diagblk) {
        // mirror rows: a 4 x 4 byte transpose across lanes 4k .. 4k+3 (rows i .. i+3); lane
        // 4k + u gets column 4g + u of those 4 rows
        const int u = lane & 3;
        const int rbase = i0 + 32 * q + (lane & ~3);
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const int c = jb + 4 * g + u;
#pragma unroll
          for (int sl = 0; sl < kR8S; ++sl) {
            const uint32_t x0 = __shfl_sync(0xffffffffu, dw[g][sl], 0, 4);
            const uint32_t x1 = __shfl_sync(0xffffffffu, dw[g][sl], 1, 4);
            const uint32_t x2 = __shfl_sync(0xffffffffu, dw[g][sl], 2, 4);
            const uint32_t x3 = __shfl_sync(0xffffffffu, dw[g][sl], 3, 4);
            uint32_t tt[4];
            i8::transpose4(x0, x1, x2, x3, tt);
            const uint32_t v = u == 0 ? tt[0] : u == 1 ? tt[1] : u == 2 ? tt[2] : tt[3];
            if (c < a.n && rbase < a.n)
              __stcs(reinterpret_cast<uint32_t*>(a.A8 + i8::a8_offset(c, rbase, sl, a.KB, kR8S)), v);
          }
        }
      }
    }
  }
  __syncwarp();
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 2) {
    tc::fence_after_sync();
    i8::tmem_dealloc(tmem, 512);
  }
  // ---- deterministic reduction: block tree, then the last CTA sums CTA partials in order
  s0 = block_sum(s0, red);
  s1 = block_sum(s1, red);
  if (threadIdx.x == 0) {
    a.partials[2 * (size_t)blockIdx.x] = s0;
    a.partials[2 * (size_t)blockIdx.x + 1] = s1;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(a.counter, 1) == (int)gridDim.x - 1);
  __syncthreads();
  if (s_last) {
    __threadfence();
    double t0 = 0.0, t1 = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += kR8Threads) {
      t0 += __ldcg(a.partials + 2 * (size_t)b);
      t1 += __ldcg(a.partials + 2 * (size_t)b + 1);
    }
    t0 = block_sum(t0, red);
    t1 = block_sum(t1, red);
    if (threadIdx.x == 0) {
      a.obj[0] = t0;
      a.obj[1] = sqrt(t1);
      *a.counter = 0;
    }
  }
}

// rows of X (n x 64 fp64, ldx) -> 7 digit slices in the tiled layout [128-row tile][slice][128][64]
// (a8_offset with KB = 1), scale[row] = 2^E_row; rows n .. up to the tile end are zeros.
// 16 threads per row, 4 values each.
__global__ void __launch_bounds__(256) r8_split_kernel(const double* __restrict__ X, int64_t ldx,
                                                      int n, int rows_pad, int8_t* __restrict__ X8,
                                                      double* __restrict__ scale) {
  const int row = blockIdx.x * 16 + (threadIdx.x >> 4), t = threadIdx.x & 15;
  if (row >= rows_pad) return;
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  if (row < n) {
    const double2 x = *reinterpret_cast<const double2*>(X + (size_t)row * ldx + 4 * t);
    const double2 y = *reinterpret_cast<const double2*>(X + (size_t)row * ldx + 4 * t + 2);
    v[0] = x.x;
    v[1] = x.y;
    v[2] = y.x;
    v[3] = y.y;
  }
  double m = fmax(fmax(fabs(v[0]), fabs(v[1])), fmax(fabs(v[2]), fabs(v[3])));
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o, 16));
  const int E = i8::scale_exp(m);
  uint32_t w[kR8S];
  i8::slices4<kR8S>(v[0], v[1], v[2], v[3], E, w);
#pragma unroll
  for (int s = 0; s < kR8S; ++s)
    *reinterpret_cast<uint32_t*>(X8 + i8::a8_offset(row, 4 * t, s, 1, kR8S)) = w[s];
  if (t == 0 && row < n) scale[row] = i8::pow2(E);
}

bool encode_map_i8_3d(CUtensorMap* map, const int8_t* base, int64_t pitch, int64_t slice_pitch,
                      int cols, int rows, int slices, int box_rows, int box_slices,
                      bool swizzle = true);

bool r8_encode(CUtensorMap* mapA, CUtensorMap* mapB, const int8_t* VF8, const int8_t* V8, int n) {
  const int mtiles = (n + 127) / 128;
  return encode_map_i8_3d(mapA, VF8, 64, 8192, 64, 128, mtiles * kR8S, 128, kR8S) &&
         encode_map_i8_3d(mapB, V8, 64, 8192, 64, 128, mtiles * kR8S, kR8N, kR8S);
}

size_t r8_bytes(int n) { return (size_t)((n + 127) / 128) * kR8S * 8192; }

cudaError_t admm_i8_launch(const CUtensorMap& mapA, const CUtensorMap& mapB, const double* VF,
                           const double* V, int64_t ldv, int8_t* VF8, int8_t* V8, double* rsA,
                           double* rsB, const uint32_t* adj, int64_t ldadj, const double* deg,
                           double t, double* Z, int64_t ldz, int n, double* obj, double* partials,
                           int* counter, const RbDigits* dig, int num_sms, cudaStream_t st) {
  const int mtiles = (n + 127) / 128, rows_pad = mtiles * 128;
  count_launch();
  r8_split_kernel<<<(rows_pad + 15) / 16, 256, 0, st>>>(VF, 64, n, rows_pad, VF8, rsA);
  count_launch();
  r8_split_kernel<<<(rows_pad + 15) / 16, 256, 0, st>>>(V, ldv, n, rows_pad, V8, rsB);
  R8Args a;
  a.rsA = rsA;
  a.rsB = rsB;
  a.bits = adj;
  a.ldb = ldadj;
  a.deg = deg;
  a.tt = t;
  a.Z = Z;
  a.ldz = ldz;
  a.n = n;
  a.TC = (n + kR8N - 1) / kR8N;
  a.MT = mtiles;
  a.A8 = dig ? dig->A8 : nullptr;
  a.KB = dig ? dig->KB : 0;
  a.S = kR8S;
  a.E = dig ? dig->E : nullptr;
  a.rscale = dig ? dig->rscale : nullptr;
  a.partials = partials;
  a.counter = counter;
  a.obj = obj;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(rebuild_i8_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kR8Smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const long long ntiles = (long long)a.MT * a.TC - 2LL * a.MT * (a.MT - 1);
  const int grid = (int)std::max<long long>(1, std::min<long long>(ntiles, num_sms));
  count_launch();
  rebuild_i8_kernel<<<grid, kR8Threads, kR8Smem, st>>>(mapA, mapB, a);
  return cudaGetLastError();
}

}  // namespace pf
