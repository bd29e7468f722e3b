// pf_rebuild_i8.cu -- the PFAM update (step a6, eq:PFAM1 P:389 with the corrected prox, reading
// R1) on one GPU for PF_FP64_I8 contexts, with the rank-p product W = V' V^T formed from EXACT
// int8 tensor-core products (tcgen05 kind::i8) of 7-bit digit slices -- the same splitting as the
// filter GEMM K1-i8 (pf_gemm_i8.cu):
//
//     V' = V diag(f) (or Q F, pf_admm_step_f),  V'_i = 2^{E_i} sum_s d_s 128^-(s+1) + r,
//     V_j = 2^{F_j} sum_t e_t 128^-(t+1) + r',   W_ij = 2^{E_i + F_j} sum_l 128^-(l+2) D_l[i][j],
//     D_l = sum_{s+t=l} A_s B_t^T  (exact int32, K = p = 64 digits: one 64-byte k-block)
//
// then Z_new = offdiag(W - tC) + Diag(1 - W_ii + Z_ii), written with its mirror and the digit
// slices of Z_new for the next filter (one scale 2^Eg, DESIGN.md §4 "fused digits").  Why: the
// fp64 DMMA formulation (rebuild_kernel) spends ~0.46 ms of DMMA pipe time on W at config 3 and
// its CTAs cannot overlap it with the 5.1 GB HBM stream; here W costs ~0.18 ms of tensor time
// issued by one thread into TMEM, and every byte of the stream moves by TMA: Z_old tiles are
// loaded into shared memory ahead of use, Z_new (tile and mirror) and its digit slices are
// staged in shared memory and written by TMA stores, so the update warps only compute.
//
// Tiles: 128 rows (a block I of V') x 32 columns (a block J of V), J >= 4 I (upper part; the 4
// tiles J = 4I .. 4I+3 cover the 128 x 128 diagonal block, both triangles, no mirror).
//   warp 0   TMA loads: A = the 7 slices of V' block I (56 KB, reloaded when I changes), B = the
//            7 slices of V block J (14 KB), Z_old tile (2 x 16 KB boxes, SWIZZLE_128B, 2 buffers)
//   warp 1   14 MMAs per tile (A_s x [B_0 .. B_{6-s}], N = 32 (7 - s)): level l at TMEM column
//            32 l of one of two 256-column accumulators
//   warp 2   TMEM allocation
//   warp 3   TMA stores: Z_new tile (from the Z_old buffer, updated in place), mirror tile, digit
//            slices of both; releases the buffers when the stores have read them
//   warps 4-19  (kR8UW = 16 update warps) TMEM lane = tile row r, kR8C = 8 columns (h = 0..3):
//            levels combined in fp64, the update, Z_new in place, the mirror (transposed) and
//            the digit slices into staging
// Deterministic sums: fixed per-thread order, CTA partials summed in CTA order by the last CTA.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "pf_digits.cuh"
#include "pf_i8mma.cuh"
#include "pf_kernels.cuh"
#include "pf_tc.cuh"

namespace pf {

bool encode_map_gen(CUtensorMap* map, bool f64, int rank, const void* base, const uint64_t* dims,
                    const uint64_t* strides, const uint32_t* box, int swizzle);

constexpr int kR8S = 7;                        // digit slices of V', V and Z_new
constexpr int kR8M = 128, kR8N = 32;           // tile
constexpr int kR8UW = 16;                      // update warps (4 per TMEM lane quarter)
constexpr int kR8C = kR8N / (kR8UW / 4);       // tile columns per update thread
constexpr int kR8Threads = 128 + 32 * kR8UW;
constexpr int kOffA = 0;                       // 7 x 128 x 64 B
constexpr int kOffB = kOffA + kR8S * 8192;     // 7 x 32 x 64 B
constexpr int kOffZ = kOffB + kR8S * 2048;     // 2 buffers x 2 boxes {16 fp64, 128 rows}
constexpr int kOffM = kOffZ + 2 * 32768;       // mirror: 8 boxes {16 fp64, 32 rows}
constexpr int kOffDt = kOffM + 32768;          // tile digits: box {32 B, 128 rows, 7 slices}
constexpr int kOffDm = kOffDt + kR8S * 4096;   // mirror digits: 2 boxes {64 B, 32 rows, 7}
constexpr int kOffBar = kOffDm + 2 * kR8S * 2048;
constexpr int kR8Smem = kOffBar + 256 + 1024;
static_assert(kR8Smem <= 232448, "shared memory");
static_assert(kOffZ % 1024 == 0 && kOffM % 1024 == 0 && kOffDt % 1024 == 0 && kOffDm % 1024 == 0,
              "swizzled boxes need 1024-byte alignment");

struct R8Args {
  const double* rsA;  // [n] 2^E_i of V' rows
  const double* rsB;  // [n] 2^F_j of V rows
  const uint32_t* bits;
  int64_t ldb;
  const double* deg;
  double tt;
  int n, TC, MT, KB;
  int mirror_dig;     // 0: the digit slices of the upper tiles (and of the lower tiles inside the
                      // 256 x 256 diagonal super-blocks) only: K1-i8s and K1-i8p in lower-
                      // transposed mode read no others
  int mirror_z;       // 0: Z_new on and above the diagonal blocks only (pf_set_z_upper)
  const int* E;       // global digit exponent Eg of Z_new
  double* rscale;
  double* partials;
  int* counter;
  double* obj;
};

struct R8Maps {
  CUtensorMap a, b;   // V', V digit slices
  CUtensorMap z, zm;  // Z: boxes {16, 128} (tile, Z_old) and {16, 32} (mirror)
  CUtensorMap dt, dm; // Z_new digit slices: {32 B, 128, 7} (tile), {64 B, 32, 7} (mirror)
};

// tile e -> (I, J): rows I of 128 (I < MT), columns J of 32 from 4I to TC - 1; cnt(I) = tiles
// before row block I = I TC - 2 I (I - 1)
__device__ __forceinline__ void r8_tile(long long e, int TC, int MT, int& I, int& J) {
  const double b = (double)TC + 2.0;
  const double disc = b * b - 8.0 * (double)e;
  int i = (int)floor((b - sqrt(fmax(disc, 0.0))) * 0.25);
  i = max(0, min(MT - 1, i));
  auto cnt = [&](long long x) { return x * TC - 2 * x * (x - 1); };
  while (i > 0 && cnt(i) > e) --i;
  while (i + 1 < MT && cnt(i + 1) <= e) ++i;
  I = i;
  J = 4 * i + (int)(e - cnt(i));
}

__device__ __forceinline__ void r8_next(int TC, int& I, int& J) {
  if (++J == TC) {
    ++I;
    J = 4 * I;
  }
}

// mbarrier wait for the producer / MMA / store warps: back off between polls so the spinning
// warp leaves its scheduler's issue slots to the update warps
__device__ __forceinline__ void mbar_wait_idle(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done;
  for (;;) {
    asm volatile(
        "{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(64);
  }
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1,
                                             int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];\n" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

// 32 lanes x kR8C consecutive 32-bit TMEM columns (then a wait)
template <int N>
__device__ __forceinline__ void tmem_ld_c(uint32_t taddr, uint32_t (&r)[N]) {
  if constexpr (N == 16) {
    i8::tmem_ld16(taddr, r);
  } else {
    static_assert(N == 8, "kR8C");
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                   "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  }
}

__global__ void __launch_bounds__(kR8Threads, 1)
    rebuild_i8_kernel(const __grid_constant__ R8Maps m, const R8Args a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* afull = bars;       // A landed
  uint64_t* aempty = bars + 1;  // the MMAs that read A (this row block) completed
  uint64_t* bfull = bars + 2;
  uint64_t* bempty = bars + 3;
  uint64_t* tfull = bars + 4;   // [2] accumulator complete
  uint64_t* tempty = bars + 6;  // [2] accumulator drained (8 update warps)
  uint64_t* zfull = bars + 8;   // [nz] Z_old tile landed
  uint64_t* zempty = bars + 11; // [nz] the Z_new stores have read the buffer
  uint64_t* sfull = bars + 14;  // staging + Z_new written (8 update warps)
  uint64_t* sempty = bars + 15; // the stores have read the staging
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);
  // Z_old / Z_new buffers: 2, or 3 when no fp64 mirror is written (its staging area is free)
  const int nz = a.mirror_z ? 2 : 3;
  auto zbuf = [&](int zb) { return smem + (zb < 2 ? kOffZ + zb * 32768 : kOffM); };
  __shared__ double red[32];
  __shared__ int s_last;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(afull, 1);
    mbar_init(aempty, 1);
    mbar_init(bfull, 1);
    mbar_init(bempty, 1);
    for (int q = 0; q < 2; ++q) {
      mbar_init(&tfull[q], 1);
      mbar_init(&tempty[q], kR8UW);
    }
    for (int q = 0; q < 3; ++q) {
      mbar_init(&zfull[q], 1);
      mbar_init(&zempty[q], 1);
    }
    mbar_init(sfull, kR8UW);
    mbar_init(sempty, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&m.a);
    tma_prefetch_desc(&m.b);
    tma_prefetch_desc(&m.z);
  }
  if (warp == 3 && lane == 0) {
    tma_prefetch_desc(&m.zm);
    tma_prefetch_desc(&m.dt);
    tma_prefetch_desc(&m.dm);
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
    // ------------------------------------------------------------------ TMA loads
    int curI = -1;
    uint32_t aeph = 0;
    const uint64_t keep = tc::policy_evict_last();   // V', V digits: re-read across tiles
    const uint64_t stream = tc::policy_evict_first(); // Z_old: read once
    int it = 0, I = 0, J = 0;
    if (t_begin < t_end) r8_tile(t_begin, a.TC, a.MT, I, J);
    for (long long t = t_begin; t < t_end; ++t, ++it, r8_next(a.TC, I, J)) {
      const int i0 = I * kR8M, j0 = J * kR8N, zb = it % nz;
      const uint32_t zph = (uint32_t)((it / nz) & 1);
      // Z_old first: the update warps wait for it; the MMA has slack
      mbar_wait_idle(&zempty[zb], zph ^ 1u);
      if (i8::elect_one()) {
        mbar_arrive_expect_tx(&zfull[zb], 32768);
        unsigned char* zs = zbuf(zb);
        tc::tma_load_2d_hint(zs, &m.z, &zfull[zb], j0, i0, stream);
        tc::tma_load_2d_hint(zs + 16384, &m.z, &zfull[zb], j0 + 16, i0, stream);
      }
      __syncwarp();
      if (I != curI) {
        if (curI >= 0) {
          mbar_wait_idle(aempty, aeph);
          aeph ^= 1u;
        }
        if (i8::elect_one()) {
          mbar_arrive_expect_tx(afull, kR8S * 8192);
          tc::tma_load_3d_hint(smem + kOffA, &m.a, afull, 0, 0, I * kR8S, keep);
        }
        __syncwarp();
        curI = I;
      }
      mbar_wait_idle(bempty, (it & 1) ^ 1u);
      if (i8::elect_one()) {
        mbar_arrive_expect_tx(bfull, kR8S * 2048);
        tc::tma_load_3d_hint(smem + kOffB, &m.b, bfull, 0, j0 & 127, (j0 >> 7) * kR8S, keep);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    int curI = -1;
    uint32_t aph = 0;
    const uint32_t a0 = smem_u32(smem + kOffA), b0 = smem_u32(smem + kOffB);
    int it = 0, I = 0, J = 0;
    if (t_begin < t_end) r8_tile(t_begin, a.TC, a.MT, I, J);
    for (long long t = t_begin; t < t_end; ++t, ++it, r8_next(a.TC, I, J)) {
      if (I != curI) {
        mbar_wait_idle(afull, aph);
        aph ^= 1u;
        curI = I;
      }
      const int tb = it & 1;
      mbar_wait_idle(&tempty[tb], ((it >> 1) & 1) ^ 1u);  // the update warps drained this buffer
      mbar_wait_idle(bfull, it & 1);
      tc::fence_after_sync();
      int In = I, Jn = J;
      r8_next(a.TC, In, Jn);
      if (t + 1 >= t_end) In = -1;
      if (i8::elect_one()) {
#pragma unroll
        for (int s = 0; s < kR8S; ++s)
#pragma unroll
          for (int ks = 0; ks < 2; ++ks)
            i8::mma_i8(tmem + (uint32_t)(tb * 256 + s * kR8N),
                       tc::sdesc_k_sw64(a0 + s * 8192 + ks * 32), tc::sdesc_k_sw64(b0 + ks * 32),
                       i8::idesc_i8(kR8M, kR8N * (kR8S - s)), (s | ks) ? 1u : 0u);
        i8::mma_commit(bempty);
        i8::mma_commit(&tfull[tb]);
        if (In != I) i8::mma_commit(aempty);  // the next tile loads another row block of V'
      }
      __syncwarp();
    }
  } else if (warp == 3) {
    // ------------------------------------------------------------------ TMA stores
    int it = 0, I = 0, J = 0;
    if (t_begin < t_end) r8_tile(t_begin, a.TC, a.MT, I, J);
    for (long long t = t_begin; t < t_end; ++t, ++it, r8_next(a.TC, I, J)) {
      const int i0 = I * kR8M, j0 = J * kR8N, zb = it % nz;
      const bool diagblk = J < 4 * I + 4;
      const bool sblk = (I & 1) == 0 && (J >> 2) == I + 1;
      mbar_wait_idle(sfull, it & 1);
      if (i8::elect_one()) {
        const unsigned char* zs = zbuf(zb);
        // two bulk groups: the staging (digits, mirrors) first, released as soon as its stores
        // have read it (the update warps write the next tile's digits there), then Z_new
        tma_store_3d(&m.dt, smem + kOffDt, j0 & 63, 0, (I * a.KB + (j0 >> 6)) * kR8S);
        if (!diagblk) {
          if (a.mirror_z)
#pragma unroll
            for (int k = 0; k < 8; ++k)
              tma_store_2d(&m.zm, smem + kOffM + k * 4096, i0 + 16 * k, j0);
          const int kb0 = i0 >> 6, jt = (j0 >> 7) * a.KB;
          if (a.mirror_dig || sblk) {
            tma_store_3d(&m.dm, smem + kOffDm, 0, j0 & 127, (jt + kb0) * kR8S);
            if (kb0 + 1 < a.KB)
              tma_store_3d(&m.dm, smem + kOffDm + kR8S * 2048, 0, j0 & 127,
                           (jt + kb0 + 1) * kR8S);
          }
        }
        bulk_commit();
        tma_store_2d(&m.z, zs, j0, i0);
        tma_store_2d(&m.z, zs + 16384, j0 + 16, i0);
        bulk_commit();
        bulk_wait_read1();
        mbar_arrive(sempty);
        bulk_wait_read0();
        mbar_arrive(&zempty[zb]);
      }
      __syncwarp();
    }
    if (i8::elect_one()) bulk_wait0();
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ update warps
    const int q = warp & 3, h = (warp - 4) >> 2;
    const int r = 32 * q + lane;  // tile row = TMEM lane
    const int Eg = *a.E;
    {
      const double sc = i8::pow2(Eg);
      for (int i = blockIdx.x * (32 * kR8UW) + (threadIdx.x - 128); i < a.n;
           i += gridDim.x * (32 * kR8UW))
        a.rscale[i] = sc;
    }
    const double qt = 0.25 * a.tt;
    const int sw = r & 7;
    // transposes of 4 x 4 byte blocks across lanes 4k .. 4k+3 (two exchange rounds)
    const int u = lane & 3;
    const uint32_t sel1 = (u & 2) ? 0x3276u : 0x5410u, sel2 = (u & 1) ? 0x3715u : 0x6240u;
    int it = 0, I = 0, J = 0;
    if (t_begin < t_end) r8_tile(t_begin, a.TC, a.MT, I, J);
    // this tile's adjacency word and row scale, loaded one tile ahead
    uint32_t wraw = 0u;
    double rs = 0.0;
    if (t_begin < t_end) {
      const int i = I * kR8M + r;
      wraw = (i < a.n) ? __ldg(a.bits + (size_t)i * a.ldb + ((J * kR8N + kR8C * h) >> 5)) : 0u;
      rs = __ldg(a.rsA + i);
    }
    for (long long t = t_begin; t < t_end; ++t, ++it) {
      const int i0 = I * kR8M, j0 = J * kR8N;
      const int i = i0 + r, jb = j0 + kR8C * h;
      const bool diagblk = J < 4 * I + 4;             // inside the 128 x 128 diagonal block
      // mirror inside a 256 x 256 diagonal super-block (written even without mirror_dig)
      const bool sblk = (I & 1) == 0 && (J >> 2) == I + 1;
      const bool fast = !diagblk && (i0 + kR8M <= a.n) && (j0 + kR8N <= a.n);
      const uint32_t word = wraw >> (jb & 31);
      const double rsi = rs;
      {
        int In = I, Jn = J;
        r8_next(a.TC, In, Jn);
        if (t + 1 < t_end) {
          const int inx = In * kR8M + r;
          wraw = (inx < a.n) ? __ldg(a.bits + (size_t)inx * a.ldb + ((Jn * kR8N + kR8C * h) >> 5)) : 0u;
          rs = __ldg(a.rsA + inx);
        }
        I = In;
        J = Jn;
      }
      double cs[kR8C];
#pragma unroll
      for (int c = 0; c < kR8C; c += 2) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(a.rsB + jb + c));
        cs[c] = v.x;
        cs[c + 1] = v.y;
      }
      // ---- W from the TMEM levels (smallest weight first)
      const int tb = it & 1, zb = it % nz;
      mbar_wait(&tfull[tb], (it >> 1) & 1);
      tc::fence_after_sync();
      // levels in pairs: 128 D_l + D_{l+1} is exact in int32 (|D_l| <= (l+1) 64 127^2 < 2^23),
      // then 4 exact conversions; summed smallest weight first
      double w[kR8C];
      const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(tb * 256 + kR8C * h);
      {
        uint32_t r6[kR8C];
        tmem_ld_c(taddr + (uint32_t)(6 * kR8N), r6);
#pragma unroll
        for (int c = 0; c < kR8C; ++c) w[c] = (double)(int)r6[c] * i8::pow2(-56);
      }
#pragma unroll 1
      for (int L = 4; L >= 0; L -= 2) {
        uint32_t ra[kR8C], rb2[kR8C];
        tmem_ld_c(taddr + (uint32_t)(L * kR8N), ra);
        tmem_ld_c(taddr + (uint32_t)((L + 1) * kR8N), rb2);
        const double wl = i8::pow2(-7 * (L + 3));
#pragma unroll
        for (int c = 0; c < kR8C; ++c) w[c] = fma((double)((int)ra[c] * 128 + (int)rb2[c]), wl, w[c]);
      }
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[tb]);  // the MMA may refill this accumulator
#pragma unroll
      for (int c = 0; c < kR8C; ++c) w[c] *= rsi * cs[c];  // exact: powers of two
      // ---- Z_old (swizzled 128-byte rows: chunk k of row r at k ^ (r % 8))
      mbar_wait(&zfull[zb], (uint32_t)((it / nz) & 1));
      // the thread's columns: 16-column box (kR8C h) / 16, its 16-byte chunks k0 .. k0 + kR8C / 2 - 1
      double* zrow = reinterpret_cast<double*>(zbuf(zb) + ((kR8C * h) >> 4) * 16384 + r * 128);
      const int k0 = ((kR8C * h) & 15) >> 1;
      double z[kR8C];
#pragma unroll
      for (int k = 0; k < kR8C / 2; ++k) {
        const double2 v = *reinterpret_cast<const double2*>(zrow + 2 * ((k0 + k) ^ sw));
        z[2 * k] = v.x;
        z[2 * k + 1] = v.y;
      }
      // ---- Z_new
      if (fast) {
        double ts0 = 0.0, ts1 = 0.0;
#pragma unroll
        for (int c = 0; c < kR8C; ++c) {
          const bool b = (word >> c) & 1u;
          const double x = w[c];
          const double o = b ? x - qt : x;          // W_ij - t C_ij, C_ij = adj_ij / 4
          ts0 += b ? x : 0.0;
          const double e = o - z[c];
          ts1 = fma(e, e, ts1);
          z[c] = o;
        }
        s0 += 2.0 * 0.25 * ts0;
        s1 += 2.0 * ts1;
      } else {
        const double wgt = diagblk ? 1.0 : 2.0;
#pragma unroll
        for (int c = 0; c < kR8C; ++c) {
          const int j = jb + c;
          const double x = w[c], zold = z[c];
          double o = 0.0;                           // outside the matrix: 0 (digits too)
          if (i < a.n && j < a.n) {
            const bool b = (word >> c) & 1u;
            if (j == i) {
              o = 1.0 - x + zold;                    // Diag(1 - W_ii + Z_ii)
              s0 += -0.25 * a.deg[i] * x;            // C_ii = -deg_i / 4
              s1 += (o - zold) * (o - zold);
            } else {
              o = b ? x - qt : x;
              if (b) s0 += wgt * 0.25 * x;
              s1 += wgt * (o - zold) * (o - zold);
            }
          }
          z[c] = o;
        }
      }
#pragma unroll
      for (int k = 0; k < kR8C / 2; ++k)
        *reinterpret_cast<double2*>(zrow + 2 * ((k0 + k) ^ sw)) = make_double2(z[2 * k], z[2 * k + 1]);
      // ---- digit slices of Z_new (scale 2^Eg): word g of slice s = columns 4g .. 4g+3
      uint32_t dw[kR8C / 4][kR8S];
#pragma unroll
      for (int g = 0; g < kR8C / 4; ++g)
        i8::slices4<kR8S>(z[4 * g], z[4 * g + 1], z[4 * g + 2], z[4 * g + 3], Eg, dw[g]);
      mbar_wait(sempty, (it & 1) ^ 1u);             // the previous tile's stores read the staging
      // tile digits: [slice][row][32 B], SWIZZLE_32B (16-byte chunk ^= bit 7 of the offset)
#pragma unroll
      for (int s = 0; s < kR8S; ++s) {
        int off = s * 4096 + r * 32 + kR8C * h;
        off ^= ((off >> 7) & 1) << 4;
        if constexpr (kR8C == 16)
          *reinterpret_cast<uint4*>(smem + kOffDt + off) =
              make_uint4(dw[0][s], dw[1][s], dw[kR8C / 4 - 2][s], dw[kR8C / 4 - 1][s]);
        else
          *reinterpret_cast<uint2*>(smem + kOffDt + off) = make_uint2(dw[0][s], dw[1][s]);
      }
      if (!diagblk) {
        // mirror fp64: box k = r / 16 holds mirror rows jj = 0..31 (tile columns), columns
        // r % 16, SWIZZLE_128B
        if (a.mirror_z) {
          unsigned char* mb = smem + kOffM + (r >> 4) * 4096;
          const int mc = r & 15;
#pragma unroll
          for (int c = 0; c < kR8C; ++c) {
            const int jj = kR8C * h + c;
            *reinterpret_cast<double*>(mb + jj * 128 + ((((mc >> 1) ^ (jj & 7))) << 4) +
                                       (mc & 1) * 8) = z[c];
          }
        }
        // mirror digits: 4 x 4 byte transposes across lanes 4k .. 4k+3 (rows rb .. rb+3); lane
        // 4k + u gets mirror row 16h + 4g + u, bytes = rows rb .. rb+3: exchange 16-bit halves
        // with lane u ^ 2, then bytes with lane u ^ 1.  [kb][slice][32 rows][64 B], SWIZZLE_64B
        // (16-byte chunk ^= bits 7-8 of the offset)
        const int rb = 32 * q + (lane & ~3);
        // (sblk: the mirror lies in a 256 x 256 diagonal super-block, which K1-i8p reads
        // directly even in lower-transposed mode)
        if (a.mirror_dig || sblk)
#pragma unroll
        for (int g = 0; g < kR8C / 4; ++g) {
          const int jj = kR8C * h + 4 * g + u;
#pragma unroll
          for (int s = 0; s < kR8S; ++s) {
            const uint32_t x = dw[g][s];
            const uint32_t y = __byte_perm(x, __shfl_xor_sync(0xffffffffu, x, 2), sel1);
            const uint32_t v = __byte_perm(y, __shfl_xor_sync(0xffffffffu, y, 1), sel2);
            int off = ((rb >> 6) * kR8S + s) * 2048 + jj * 64 + (rb & 63);
            off ^= ((off >> 7) & 3) << 4;
            *reinterpret_cast<uint32_t*>(smem + kOffDm + off) = v;
          }
        }
      }
      fence_proxy_async();  // generic-proxy smem writes -> visible to the TMA stores
      __syncwarp();
      if (lane == 0) mbar_arrive(sfull);
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

// ============================================================================== fp64 variant
// The same TMA-staged PFAM update for PF_FP64 contexts (no digit output, one GPU, p = 64), with
// W = V' V^T formed in fp64 on DMMA (mma.sync m16n8k4) by the 8 compute warps from shared-memory
// panels instead of int8 digit products: V' row block (128 x 64, four SWIZZLE_128B boxes,
// reloaded when I changes), V column block (32 x 64, two stages), Z_old tiles (two buffers), Z_new
// written in place and by TMA stores with its mirror.  The DMMA rebuild_kernel (K7) interleaves
// the product with LSU loads / stores inside each CTA and runs at 0.46 of HBM at config 3.
//   warp 0   TMA loads          warp 1   TMA stores
//   warps 2-9  compute: warp w owns rows 16w .. 16w+15 of the tile (all 32 columns, 4 n8 blocks)
constexpr int kTdThreads = 320;
constexpr int kTdOffVi = 0;                    // 4 boxes {16 fp64, 128 rows} = 64 KB
constexpr int kTdOffVj = kTdOffVi + 65536;     // 2 stages x 4 boxes {16, 32} = 2 x 16 KB
constexpr int kTdOffZ = kTdOffVj + 32768;      // 2 buffers x 2 boxes {16, 128}
constexpr int kTdOffM = kTdOffZ + 65536;       // mirror: 8 boxes {16, 32}
constexpr int kTdOffBar = kTdOffM + 32768;
constexpr int kTdSmem = kTdOffBar + 256 + 1024;
static_assert(kTdSmem <= 232448, "shared memory");

struct TdMaps {
  CUtensorMap vi, vj;  // V' rows (box {16, 128}), V rows (box {16, 32})
  CUtensorMap z, zm;   // Z: {16, 128} (tile, Z_old), {16, 32} (mirror)
};

// element (r, c) of a SWIZZLE_128B box of 16 fp64 columns (128-byte rows): byte offset
__device__ __forceinline__ int sw128(int r, int c) {
  return r * 128 + ((((c >> 1) ^ (r & 7))) << 4) + (c & 1) * 8;
}

__global__ void __launch_bounds__(kTdThreads, 1)
    rebuild_tma_kernel(const __grid_constant__ TdMaps m, const R8Args a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kTdOffBar);
  uint64_t* vifull = bars;
  uint64_t* viempty = bars + 1;   // compute warps done with this row block's V' panel
  uint64_t* vjfull = bars + 2;    // [2]
  uint64_t* vjempty = bars + 4;   // [2]
  uint64_t* zfull = bars + 6;     // [2]
  uint64_t* zempty = bars + 8;    // [2]
  uint64_t* sfull = bars + 10;
  uint64_t* sempty = bars + 11;
  __shared__ double red[32];
  __shared__ int s_last;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(vifull, 1);
    mbar_init(viempty, 8);
    for (int q = 0; q < 2; ++q) {
      mbar_init(&vjfull[q], 1);
      mbar_init(&vjempty[q], 8);
      mbar_init(&zfull[q], 1);
      mbar_init(&zempty[q], 1);
    }
    mbar_init(sfull, 8);
    mbar_init(sempty, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&m.vi);
    tma_prefetch_desc(&m.vj);
    tma_prefetch_desc(&m.z);
  }
  if (warp == 1 && lane == 0) tma_prefetch_desc(&m.zm);
  __syncthreads();

  const long long ntiles = (long long)a.MT * a.TC - 2LL * a.MT * (a.MT - 1);
  const long long t_begin = ntiles * blockIdx.x / gridDim.x;
  const long long t_end = ntiles * (blockIdx.x + 1) / gridDim.x;
  double s0 = 0.0, s1 = 0.0;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA loads
    int curI = -1;
    uint32_t viph = 0;
    const uint64_t keep = tc::policy_evict_last();    // V', V panels: re-read across tiles
    const uint64_t stream = tc::policy_evict_first(); // Z_old: read once
    int it = 0, I = 0, J = 0;
    if (t_begin < t_end) r8_tile(t_begin, a.TC, a.MT, I, J);
    for (long long t = t_begin; t < t_end; ++t, ++it, r8_next(a.TC, I, J)) {
      const int i0 = I * kR8M, j0 = J * kR8N, b = it & 1;
      mbar_wait_idle(&zempty[b], ((it >> 1) & 1) ^ 1u);
      if (i8::elect_one()) {
        mbar_arrive_expect_tx(&zfull[b], 32768);
        unsigned char* zs = smem + kTdOffZ + b * 32768;
        tc::tma_load_2d_hint(zs, &m.z, &zfull[b], j0, i0, stream);
        tc::tma_load_2d_hint(zs + 16384, &m.z, &zfull[b], j0 + 16, i0, stream);
      }
      __syncwarp();
      if (I != curI) {
        if (curI >= 0) {
          mbar_wait_idle(viempty, viph);
          viph ^= 1u;
        }
        if (i8::elect_one()) {
          mbar_arrive_expect_tx(vifull, 65536);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            tc::tma_load_2d_hint(smem + kTdOffVi + q * 16384, &m.vi, vifull, 16 * q, i0, keep);
        }
        __syncwarp();
        curI = I;
      }
      mbar_wait_idle(&vjempty[b], ((it >> 1) & 1) ^ 1u);
      if (i8::elect_one()) {
        mbar_arrive_expect_tx(&vjfull[b], 16384);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          tc::tma_load_2d_hint(smem + kTdOffVj + b * 16384 + q * 4096, &m.vj, &vjfull[b], 16 * q,
                               j0, keep);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ TMA stores
    int it = 0, I = 0, J = 0;
    if (t_begin < t_end) r8_tile(t_begin, a.TC, a.MT, I, J);
    for (long long t = t_begin; t < t_end; ++t, ++it, r8_next(a.TC, I, J)) {
      const int i0 = I * kR8M, j0 = J * kR8N, b = it & 1;
      const bool diagblk = J < 4 * I + 4;
      const bool sblk = (I & 1) == 0 && (J >> 2) == I + 1;
      mbar_wait_idle(sfull, it & 1);
      if (i8::elect_one()) {
        const unsigned char* zs = smem + kTdOffZ + b * 32768;
        tma_store_2d(&m.z, zs, j0, i0);
        tma_store_2d(&m.z, zs + 16384, j0 + 16, i0);
        if (!diagblk) {
#pragma unroll
          for (int k = 0; k < 8; ++k) tma_store_2d(&m.zm, smem + kTdOffM + k * 4096, i0 + 16 * k, j0);
        }
        bulk_commit();
        bulk_wait_read0();
        mbar_arrive(&zempty[b]);
        mbar_arrive(sempty);
      }
      __syncwarp();
    }
    if (i8::elect_one()) bulk_wait0();
    __syncwarp();
  } else {
    // ------------------------------------------------------------------ compute warps
    const int w = warp - 2, g8 = lane >> 2, t4 = lane & 3;
    const double qt = 0.25 * a.tt;
    int curI = -1;
    uint32_t viph = 0;
    int it = 0, I = 0, J = 0;
    if (t_begin < t_end) r8_tile(t_begin, a.TC, a.MT, I, J);
    const unsigned char* vi = smem + kTdOffVi;
    for (long long t = t_begin; t < t_end; ++t, ++it) {
      const int i0 = I * kR8M, j0 = J * kR8N, b = it & 1;
      const bool diagblk = J < 4 * I + 4;
      const bool fast = !diagblk && (i0 + kR8M <= a.n) && (j0 + kR8N <= a.n);
      if (I != curI) {
        if (curI >= 0) {  // release the previous row block's panel
          __syncwarp();
          if (lane == 0) mbar_arrive(viempty);
        }
        mbar_wait(vifull, viph);
        viph ^= 1u;
        curI = I;
      }
      // adjacency words of this thread's two rows (columns j0 .. j0+31: one 32-bit word)
      const int ra = i0 + 16 * w + g8, rb = ra + 8;
      const uint32_t wa = ra < a.n ? __ldg(a.bits + (size_t)ra * a.ldb + (j0 >> 5)) : 0u;
      const uint32_t wb = rb < a.n ? __ldg(a.bits + (size_t)rb * a.ldb + (j0 >> 5)) : 0u;
      // ---- W = V'_I V_J^T on DMMA: rows 16w + (g8, g8 + 8), columns 8 nt + 2 t4 + (0, 1)
      mbar_wait(&vjfull[b], (it >> 1) & 1);
      const unsigned char* vj = smem + kTdOffVj + b * 16384;
      double acc[4][4];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[nt][q] = 0.0;
#pragma unroll
      for (int ks = 0; ks < 16; ++ks) {
        const int k = 4 * ks + t4, kb = k >> 4, kc = k & 15;
        const double a0 = *reinterpret_cast<const double*>(vi + kb * 16384 + sw128(16 * w + g8, kc));
        const double a1 =
            *reinterpret_cast<const double*>(vi + kb * 16384 + sw128(16 * w + g8 + 8, kc));
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
          dmma16884(acc[nt], a0, a1,
                    *reinterpret_cast<const double*>(vj + kb * 4096 + sw128(8 * nt + g8, kc)));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&vjempty[b]);
      // ---- the update against Z_old (swizzled buffer), Z_new in place
      mbar_wait(&zfull[b], (it >> 1) & 1);
      unsigned char* zs = smem + kTdOffZ + b * 32768;
      double z[4][2][2];  // [nt][row h][c]
      double wgt = diagblk ? 1.0 : 2.0;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = 16 * w + g8 + 8 * h, cc = 8 * nt + 2 * t4;  // tile coordinates
          double2* zp = reinterpret_cast<double2*>(zs + (cc >> 4) * 16384 + sw128(r, cc & 15));
          const double2 zo = *zp;
          const uint32_t word = h ? wb : wa;
          const int i = i0 + r;
          double o[2];
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int j = j0 + cc + c;
            const double x = acc[nt][2 * h + c], zold = c ? zo.y : zo.x;
            const bool bit = (word >> (cc + c)) & 1u;
            if (fast) {
              o[c] = bit ? x - qt : x;
              if (bit) s0 += wgt * 0.25 * x;
              s1 = fma(wgt * (o[c] - zold), o[c] - zold, s1);
            } else if (i < a.n && j < a.n) {
              if (j == i) {
                o[c] = 1.0 - x + zold;                // Diag(1 - W_ii + Z_ii)
                s0 += -0.25 * a.deg[i] * x;           // C_ii = -deg_i / 4
                s1 += (o[c] - zold) * (o[c] - zold);
              } else {
                o[c] = bit ? x - qt : x;
                if (bit) s0 += wgt * 0.25 * x;
                s1 += wgt * (o[c] - zold) * (o[c] - zold);
              }
            } else {
              o[c] = 0.0;
            }
            z[nt][h][c] = o[c];
          }
          *zp = make_double2(o[0], o[1]);
        }
      // ---- mirror staging (after the previous tile's stores read it)
      mbar_wait(sempty, (it & 1) ^ 1u);
      if (!diagblk) {
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              const int r = 16 * w + g8 + 8 * h, jj = 8 * nt + 2 * t4 + c;
              *reinterpret_cast<double*>(smem + kTdOffM + (r >> 4) * 4096 + sw128(jj, r & 15)) =
                  z[nt][h][c];
            }
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(sfull);
      // next tile
      r8_next(a.TC, I, J);
    }
    if (curI >= 0) {
      __syncwarp();
      if (lane == 0) mbar_arrive(viempty);
    }
  }
  __syncthreads();
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
    for (int bb = threadIdx.x; bb < (int)gridDim.x; bb += kTdThreads) {
      t0 += __ldcg(a.partials + 2 * (size_t)bb);
      t1 += __ldcg(a.partials + 2 * (size_t)bb + 1);
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

bool td_usable(const double* VF, const double* V, int64_t ldv, const double* Z, int64_t ldz) {
  return (ldv % 2) == 0 && (ldz % 2) == 0 && (reinterpret_cast<uintptr_t>(VF) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(V) & 15) == 0 && (reinterpret_cast<uintptr_t>(Z) & 15) == 0;
}

cudaError_t admm_tma_launch(const double* VF, const double* V, int64_t ldv, const uint32_t* adj,
                            int64_t ldadj, const double* deg, double t, double* Z, int64_t ldz,
                            int n, double* obj, double* partials, int* counter, int num_sms,
                            cudaStream_t st) {
  TdMaps m;
  {
    const uint64_t dv[2] = {64, (uint64_t)n};
    const uint64_t svf[1] = {64 * 8}, sv[1] = {(uint64_t)ldv * 8};
    const uint32_t bi[2] = {16, 128}, bj[2] = {16, 32};
    const uint64_t dz[2] = {(uint64_t)n, (uint64_t)n}, sz[1] = {(uint64_t)ldz * 8};
    if (!encode_map_gen(&m.vi, true, 2, VF, dv, svf, bi, 128) ||
        !encode_map_gen(&m.vj, true, 2, V, dv, sv, bj, 128) ||
        !encode_map_gen(&m.z, true, 2, Z, dz, sz, bi, 128) ||
        !encode_map_gen(&m.zm, true, 2, Z, dz, sz, bj, 128))
      return cudaErrorInvalidValue;
  }
  R8Args a = {};
  a.bits = adj;
  a.ldb = ldadj;
  a.deg = deg;
  a.tt = t;
  a.n = n;
  a.TC = (n + kR8N - 1) / kR8N;
  a.MT = (n + 127) / 128;
  a.partials = partials;
  a.counter = counter;
  a.obj = obj;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(rebuild_tma_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kTdSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const long long ntiles = (long long)a.MT * a.TC - 2LL * a.MT * (a.MT - 1);
  const int grid = (int)std::max<long long>(1, std::min<long long>(ntiles, num_sms));
  count_launch();
  rebuild_tma_kernel<<<grid, kTdThreads, kTdSmem, st>>>(m, a);
  return cudaGetLastError();
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
  double mx = fmax(fmax(fabs(v[0]), fabs(v[1])), fmax(fabs(v[2]), fabs(v[3])));
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o, 16));
  const int E = i8::scale_exp(mx);
  uint32_t w[kR8S];
  i8::slices4<kR8S>(v[0], v[1], v[2], v[3], E, w);
#pragma unroll
  for (int s = 0; s < kR8S; ++s)
    *reinterpret_cast<uint32_t*>(X8 + i8::a8_offset(row, 4 * t, s, 1, kR8S)) = w[s];
  if (t == 0) scale[row] = i8::pow2(E);  // padded rows: 1 (their digits are 0)
}


size_t r8_bytes(int n) { return (size_t)((n + 127) / 128) * kR8S * 8192; }

// the maps that do not depend on Z: V', V digit buffers and the A8 layout of Z_new's digits
bool r8_encode(CUtensorMap* maps, const int8_t* VF8, const int8_t* V8, const int8_t* A8, int n,
               int KB) {
  const uint64_t mt = (uint64_t)(n + 127) / 128;
  const uint64_t dv[3] = {64, 128, mt * kR8S}, sv[2] = {64, 8192};
  const uint32_t ba[3] = {64, 128, kR8S}, bb[3] = {64, kR8N, kR8S};
  const uint64_t dd[3] = {64, 128, mt * (uint64_t)KB * kR8S};
  const uint32_t bt[3] = {32, 128, kR8S}, bm[3] = {64, 32, kR8S};
  return encode_map_gen(&maps[0], false, 3, VF8, dv, sv, ba, 64) &&
         encode_map_gen(&maps[1], false, 3, V8, dv, sv, bb, 64) &&
         encode_map_gen(&maps[2], false, 3, A8, dd, sv, bt, 32) &&
         encode_map_gen(&maps[3], false, 3, A8, dd, sv, bm, 64);
}

bool r8_usable(const double* Z, int64_t ldz) {
  return (ldz % 2) == 0 && (reinterpret_cast<uintptr_t>(Z) & 15) == 0;
}

cudaError_t admm_i8_launch(const CUtensorMap* maps, const double* VF, const double* V,
                           int64_t ldv, int8_t* VF8, int8_t* V8, double* rsA, double* rsB,
                           const uint32_t* adj, int64_t ldadj, const double* deg, double t,
                           double* Z, int64_t ldz, int n, double* obj, double* partials,
                           int* counter, const RbDigits* dig, int mirror_dig, int mirror_z,
                           int num_sms, cudaStream_t st) {
  const int mtiles = (n + 127) / 128, rows_pad = mtiles * 128;
  R8Maps m;
  m.a = maps[0];
  m.b = maps[1];
  m.dt = maps[2];
  m.dm = maps[3];
  {
    const uint64_t dz[2] = {(uint64_t)n, (uint64_t)n}, sz[1] = {(uint64_t)ldz * 8};
    const uint32_t bz[2] = {16, 128}, bzm[2] = {16, 32};
    if (!encode_map_gen(&m.z, true, 2, Z, dz, sz, bz, 128) ||
        !encode_map_gen(&m.zm, true, 2, Z, dz, sz, bzm, 128))
      return cudaErrorInvalidValue;
  }
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
  a.n = n;
  a.TC = (n + kR8N - 1) / kR8N;
  a.MT = mtiles;
  a.KB = dig->KB;
  a.mirror_dig = mirror_dig;
  a.mirror_z = mirror_z;
  a.E = dig->E;
  a.rscale = dig->rscale;
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
  rebuild_i8_kernel<<<grid, kR8Threads, kR8Smem, st>>>(m, a);
  return cudaGetLastError();
}

}  // namespace pf
