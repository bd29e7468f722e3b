// pf_gemm_tf32.cu -- the Chebyshev-step filter GEMM for fp32-storage problems (config 5,
// BASELINE configs[4]) on the 5th-generation tensor cores (tcgen05.mma kind::tf32):
//
//     out = s1 * (A B) + s2 * Ycur + s3 * Yprev        (eq:cheb, eqn:cheb-linear-map)
//
// A: n_rows x n_k fp32 row-major (the local row block of the symmetric iterate).
// Blocks B = Y_j, Ycur, Yprev, out are stored TRANSPOSED ("p-major"): element (row i, col c)
// of the n x p block lives at Y[c * ldy + i].  That makes the B operand K-major for the MMA and
// lets each epilogue warp store 32 consecutive rows of one column as one 128-byte line.
//
// Precision: 3xTF32 (npass = 3).  TF32 keeps 10 mantissa bits, which perturbs the operator by
// ~1e-3 relative -- too much for the 1e-4 parity bar.  Each fp32 operand is split
// x = hi + lo with hi = trunc13(x) (tf32) and lo = x - hi (exact in fp32), and the product is
// A_hi B_hi + A_hi B_lo + A_lo B_hi (dropped A_lo B_lo ~ 2^-22 relative), fp32 accumulation
// in TMEM.  npass = 2 drops A_hi B_lo (exact operator, iterate rounded to tf32), npass = 1 runs
// the single A_hi B_hi product (plain TF32).
//
// B200 design (DESIGN.md §4 K1-tf32):
//  * CTA pair (cluster 2x1, tcgen05 cta_group::2): the pair owns a 256-row tile of A; each CTA
//    stages its 128 rows of A and HALF of every 256-column slice of B, so per-SM B traffic is
//    halved; the leader CTA issues M=256 x N=min(p,256) x K=8 MMAs into both CTAs' TMEM
//    (128 lanes x p fp32 columns each).
//  * TMA (cp.async.bulk.tensor.2d, SWIZZLE_64B, 16-wide K boxes) into a STAGES-deep ring, A loads
//    tagged L2 evict_first (streamed once), Y loads evict_last (re-read by every pair).
//  * kind::tf32 reads an fp32 operand as tf32 by dropping the low 13 mantissa bits (checked on
//    the device: tools/probe/tf32_probe.cu), so the raw TMA tile IS the hi operand; converter
//    warps write lo = x - trunc13(x) (exact in fp32) into a separate, shallower ring and release
//    it to the leader's MMA issuer through a cluster-scope mbarrier.  The raw ring alone covers
//    the TMA latency (profiles/r01_tf32_trace.txt: ~3.5 us issue-to-land under load).
//  * schedule: full waves of whole 256-row tiles with every pair walking K in the same order
//    (Y is re-read once per wave from HBM and hit in L2 by the other pairs), then the leftover
//    tiles split along K; split tiles go through a workspace and the last contributor sums
//    them in fixed order (deterministic) before the Chebyshev scale-shift-subtract epilogue.
//  * epilogue warps drain TMEM with tcgen05.ld (32 lanes x 32 columns per instruction).
#include <algorithm>
#include <cstdlib>

#include "pf_kernels.cuh"
#include "pf_tc.cuh"

namespace pf {

template <int P>
struct Tf32Cfg {
  static constexpr int BK = 16;                   // K per stage: 64-byte rows (SWIZZLE_64B)
  static constexpr int BM = 128;                  // A rows per CTA (M = 256 per pair)
  static constexpr int NMMA = P < 256 ? P : 256;  // N per MMA instruction
  static constexpr int NH = P / NMMA;             // N slices
  static constexpr int BROWS = P / 2;             // B rows staged per CTA (half of each slice)
  static constexpr int A_BYTES = BM * BK * 4;
  static constexpr int B_BYTES = BROWS * BK * 4;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;  // one raw (TMA) or one lo stage
  // raw ring (TMA destination, read by the MMA as the hi operand: kind::tf32 drops the low 13
  // mantissa bits of an fp32 operand) and a shallower lo ring (x - trunc13(x), converter
  // output).  Only the raw ring has to cover the TMA latency.
  static constexpr int RING = (200 * 1024) / STAGE_BYTES;
  static constexpr int NL = RING >= 12 ? 4 : 3;
  static constexpr int NT = (RING - NL) > 12 ? 12 : (RING - NL);
  static constexpr int TMEM_COLS = P < 32 ? 32 : P;
  static constexpr int NCONV_WARPS = 6;           // warps 2..7
  static constexpr int NEPI_WARPS = 8;            // warps 8..15: lane quarter x column half
  static constexpr int THREADS = 16 * 32;
  static constexpr int BAR_BYTES = 8 * (2 * NT + 2 * NL + 2) + 16;
  static constexpr int SMEM = (NT + NL) * STAGE_BYTES + 1024 + BAR_BYTES;
  static_assert(P % 32 == 0 && P >= 64 && P <= 512, "p");
  static_assert(B_BYTES % 1024 == 0 && A_BYTES % 1024 == 0, "1 KiB aligned sub-tiles");
  static_assert(NT >= 4 && NL >= 2, "stages");
};

struct Tf32Args {
  const float* ycur;
  const float* yprev;
  float* out;
  const double* coef;  // {s1, s2, s3} (device)
  float* ws;           // split-K partials: [pair][2 ctas][P][128]
  int* counters;       // [tiles][2], zero between launches
  int64_t ldy;         // pitch (elements) of ycur / yprev / out
  int n_rows;
  int kblocks;
  int mtiles;
  int split;           // K-split of the tail wave
  int npass;
  int chunk_kb;        // k-blocks accumulated in TMEM before folding into `acc` (0: no limit)
  int bdist_kb;        // > 0: B is the rank-major all-gather [world][p][n_local] read through a
                       // 3-D map; k-blocks per rank (n_local / 16)
  float* acc;          // fp32 chunk accumulators: [pair][2 ctas][P][128]
  int pf_dist;         // L2 prefetch distance of A in k-blocks (0: off)
};

// Work schedule of pair g among G pairs: F = M / G full waves in which every pair runs a whole
// 256-row tile over K in the same order (so the Y k-block that all pairs read at about the same
// time is fetched from HBM once and then hit in L2 -- Y can exceed L2 at p = 512), then the
// R = M % G leftover tiles split S ways along K (pair g < R S takes K-chunk g % S of tile
// F G + g / S).  Split tiles are reduced by the last contributor in chunk order.
struct Sched {
  int F, R, S, G, g, KB;
  __device__ Sched(int M, int KB_, int S_, int G_, int g_) : S(S_), G(G_), g(g_), KB(KB_) {
    F = M / G;
    R = M - F * G;
  }
  __device__ int count() const { return F + ((R > 0 && g < R * S) ? 1 : 0); }
  __device__ void item(int w, int& tile, int& kb0, int& kb1) const {
    if (w < F) {
      tile = w * G + g;
      kb0 = 0;
      kb1 = KB;
    } else {
      tile = F * G + g / S;
      const int c = g % S;
      kb0 = (int)((long long)c * KB / S);
      kb1 = (int)((long long)(c + 1) * KB / S);
    }
  }
};

#ifdef PF_TRACE
__device__ unsigned long long g_trace[12][512];
__device__ __forceinline__ void trace(int what, int w, int i, int g) {
  if (g == 0 && w == 0 && i < 512) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_trace[what][i] = t;
  }
}
void tf32_trace_read(unsigned long long* host) {
  cudaMemcpyFromSymbol(host, g_trace, sizeof(g_trace));
}
#define TRACE(what, w, i) trace(what, w, i, g)
#else
#define TRACE(what, w, i)
#endif

// ring position of the i-th k-block of this pair
struct Ring {
  int n, s;
  uint32_t ph;
  __device__ Ring(int n_) : n(n_), s(0), ph(0) {}
  __device__ void next() {
    if (++s == n) {
      s = 0;
      ph ^= 1u;
    }
  }
};

template <int P>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Tf32Cfg<P>::THREADS, 1)
    cheb_gemm_tf32_kernel(const __grid_constant__ CUtensorMap mapA,
                          const __grid_constant__ CUtensorMap mapB,
                          const __grid_constant__ CUtensorMap mapApf, Tf32Args args) {
  using C = Tf32Cfg<P>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* raw = smem;                             // NT stages: [A | B] fp32 (TMA)
  unsigned char* low = smem + C::NT * C::STAGE_BYTES;    // NL stages: [A_lo | B_lo]
  uint64_t* full = reinterpret_cast<uint64_t*>(low + C::NL * C::STAGE_BYTES);  // TMA landed
  uint64_t* empty = full + C::NT;      // raw stage consumed (MMA commit, multicast)
  uint64_t* ready = empty + C::NT;     // lo stage written (leader's copy; both CTAs arrive)
  uint64_t* lfree = ready + C::NL;     // lo stage consumed (MMA commit, multicast)
  uint64_t* tfull = lfree + C::NL;     // accumulator complete (MMA commit, multicast)
  uint64_t* tempty = tfull + 1;        // accumulator drained (leader's copy; both CTAs arrive)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  volatile int* sflag = reinterpret_cast<volatile int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = tc::cluster_ctarank();
  const int G = (int)tc::nclusters_x(), g = (int)tc::cluster_id_x();

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NT; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < C::NL; ++s) {
      mbar_init(&ready[s], 2 * C::NCONV_WARPS);
      mbar_init(&lfree[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 2 * C::NEPI_WARPS);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mapA);
    tma_prefetch_desc(&mapB);
    tma_prefetch_desc(&mapApf);
  }
  if (warp == 1) tc::tmem_alloc_pair<C::TMEM_COLS>(tmem_slot);
  tc::fence_before_sync();
  tc::cluster_sync();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  const int KB = args.kblocks;
  const Sched sch(args.mtiles, KB, args.split, G, g);
  const int nitems = sch.count();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (one lane)
    if (lane == 0) {
      Ring rt(C::NT);
      const uint64_t pol_a = tc::policy_evict_first(), pol_b = tc::policy_evict_last();
      for (int w = 0; w < nitems; ++w) {
        int tile, kb0, kb1;
        sch.item(w, tile, kb0, kb1);
        const int arow = tile * 256 + (int)crank * C::BM;
        for (int kb = kb0; kb < kb1; ++kb, rt.next()) {
          // A streams from HBM exactly once: pull it into L2 PF_DIST k-blocks ahead in
          // 128-byte row segments (every other k-block)
          if (args.pf_dist > 0 && ((kb - kb0) & 1) == 0 && kb + args.pf_dist < kb1)
            tc::tma_prefetch_2d(&mapApf, (kb + args.pf_dist) * C::BK, arow, pol_a);
          mbar_wait(&empty[rt.s], rt.ph ^ 1u);
          TRACE(0 + 6 * crank, w, kb - kb0);
          unsigned char* st = raw + rt.s * C::STAGE_BYTES;
          mbar_arrive_expect_tx(&full[rt.s], C::STAGE_BYTES);
          tc::tma_load_2d_hint(st, &mapA, &full[rt.s], kb * C::BK, arow, pol_a);
          if (args.bdist_kb > 0) {
            // global k-block kb lives in rank kb / bdist_kb's slab at local k-block kb % bdist_kb
            const int rk = kb / args.bdist_kb, lk = kb - rk * args.bdist_kb;
#pragma unroll
            for (int h = 0; h < C::NH; ++h)
              tc::tma_load_3d_hint(st + C::A_BYTES + h * (C::NMMA / 2) * 64, &mapB, &full[rt.s],
                                   lk * C::BK, h * C::NMMA + (int)crank * (C::NMMA / 2), rk,
                                   pol_b);
          } else {
#pragma unroll
            for (int h = 0; h < C::NH; ++h)
              tc::tma_load_2d_hint(st + C::A_BYTES + h * (C::NMMA / 2) * 64, &mapB, &full[rt.s],
                                   kb * C::BK, h * C::NMMA + (int)crank * (C::NMMA / 2), pol_b);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (pair leader)
    // the whole warp runs the loop (warp-uniform operands in uniform registers), one elected
    // lane issues (see pf_gemm_i8.cu)
    if (crank == 0) {
      const uint32_t idesc = tc::idesc_tf32(256, C::NMMA);
      Ring rt(C::NT), rl(C::NL);
      uint32_t tphase = 0;
      const int kch = args.chunk_kb > 0 ? args.chunk_kb : (1 << 30);
      for (int w = 0; w < nitems; ++w) {
        int tile, kb0, kb1;
        sch.item(w, tile, kb0, kb1);
        for (int s0 = kb0; s0 < kb1; s0 += kch) {
        const int s1 = min(kb1, s0 + kch);
        tc::mbar_wait_cluster(tempty, tphase ^ 1u);  // both epilogues drained the accumulator
        tc::fence_after_sync();
        for (int kb = s0; kb < s1; ++kb, rt.next(), rl.next()) {
          // the converters of BOTH CTAs saw this raw stage land and wrote its lo copy
          if (lane == 0) TRACE(3, w, kb - kb0);
          tc::mbar_wait_cluster(&ready[rl.s], rl.ph);
          tc::fence_after_sync();
          if (lane == 0) TRACE(4, w, kb - kb0);
          const uint32_t a_hi = smem_u32(raw + rt.s * C::STAGE_BYTES);
          const uint32_t a_lo = smem_u32(low + rl.s * C::STAGE_BYTES);
          const uint32_t b_hi = a_hi + C::A_BYTES, b_lo = a_lo + C::A_BYTES;
          if (tc::elect_one()) {
#pragma unroll
          for (int ks = 0; ks < C::BK / 8; ++ks) {
#pragma unroll
            for (int h = 0; h < C::NH; ++h) {
              const uint32_t d = tmem + h * C::NMMA;
              const uint32_t boff = h * (C::NMMA / 2) * 64 + ks * 32;
              const uint32_t acc = (kb == s0 && ks == 0) ? 0u : 1u;
              tc::mma_tf32_pair(d, tc::sdesc_k_sw64(a_hi + ks * 32),
                                tc::sdesc_k_sw64(b_hi + boff), idesc, acc);
              if (args.npass >= 2)  // exact operator: + A_lo B_hi
                tc::mma_tf32_pair(d, tc::sdesc_k_sw64(a_lo + ks * 32),
                                  tc::sdesc_k_sw64(b_hi + boff), idesc, 1u);
              if (args.npass == 3)  // exact iterate: + A_hi B_lo
                tc::mma_tf32_pair(d, tc::sdesc_k_sw64(a_hi + ks * 32),
                                  tc::sdesc_k_sw64(b_lo + boff), idesc, 1u);
            }
          }
          tc::mma_commit_pair(&empty[rt.s]);  // raw stage free in both CTAs
          tc::mma_commit_pair(&lfree[rl.s]);  // lo stage free in both CTAs
          }
          __syncwarp();
        }
        if (tc::elect_one()) tc::mma_commit_pair(tfull);  // accumulator complete -> epilogues
        __syncwarp();
        tphase ^= 1u;
        }
      }
    }
  } else if (warp < 2 + C::NCONV_WARPS) {
    // ------------------------------------------------------------ converters: lo = x - trunc13(x)
    const int ct = threadIdx.x - 64;  // 0 .. 32*NCONV_WARPS-1
    const uint32_t ready_leader0 = tc::mapa(smem_u32(&ready[0]), 0);
    Ring rt(C::NT), rl(C::NL);
    for (int w = 0; w < nitems; ++w) {
      int tile, kb0, kb1;
      sch.item(w, tile, kb0, kb1);
      for (int kb = kb0; kb < kb1; ++kb, rt.next(), rl.next()) {
        mbar_wait(&lfree[rl.s], rl.ph ^ 1u);
        if (ct == 0) TRACE(1 + 6 * crank, w, kb - kb0);
        mbar_wait(&full[rt.s], rt.ph);
        if (ct == 0) TRACE(2 + 6 * crank, w, kb - kb0);
        if (args.npass >= 2) {  // npass 2: lo of A only; npass 3: lo of A and B
          const float4* src = reinterpret_cast<const float4*>(raw + rt.s * C::STAGE_BYTES);
          float4* dst = reinterpret_cast<float4*>(low + rl.s * C::STAGE_BYTES);
          const int nvec = (args.npass == 3 ? C::STAGE_BYTES : C::A_BYTES) / 16;
#pragma unroll 4
          for (int i = ct; i < nvec; i += 32 * C::NCONV_WARPS) {
            const float4 x = src[i];
            float4 l;
            l.x = x.x - __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
            l.y = x.y - __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
            l.z = x.z - __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
            l.w = x.w - __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
            dst[i] = l;
          }
          fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor core
        }
        __syncwarp();
        if (ct == 0) TRACE(5 + 6 * crank, w, kb - kb0);
        if (ct == 160) TRACE(9 + crank, w, kb - kb0);
        if (lane == 0) tc::mbar_arrive_cluster(ready_leader0 + rl.s * 8);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (8 warps)
    // warp 8 + 4h + q drains TMEM lanes 32q..32q+31 (rows) and columns [h P/2, (h+1) P/2).
    // The tensor core's fp32 accumulation truncates (tools/probe: one-signed data drifts by
    // -3e-4 relative over K = 65536), so at most chunk_kb k-blocks are accumulated in TMEM;
    // chunk results are folded into `acc` with round-to-nearest fp32 adds (same thread, same
    // order every launch: deterministic).
    const int q = warp & 3, hc = (warp - 8) >> 2;
    const int et = 32 * q + lane;  // row within this CTA's 128 rows
    const int cb = hc * (P / 2), ce = cb + P / 2;
    const uint32_t tempty_leader = tc::mapa(smem_u32(tempty), 0);
    const float s1 = (float)args.coef[0], s2 = (float)args.coef[1], s3 = (float)args.coef[2];
    const int kch = args.chunk_kb > 0 ? args.chunk_kb : (1 << 30);
    float* accp = args.acc + ((size_t)g * 2 + crank) * (size_t)(P * 128) + et;
    uint32_t tphase = 0;
    for (int w = 0; w < nitems; ++w) {
      int tile, kb0, kb1;
      sch.item(w, tile, kb0, kb1);
      const int row = tile * 256 + (int)crank * C::BM + et;
      const bool row_ok = row < args.n_rows;
      const bool whole = (kb0 == 0 && kb1 == KB);
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16);
      float* mine = args.ws + ((size_t)g * 2 + crank) * (size_t)(P * 128) + et;
      for (int s0 = kb0; s0 < kb1; s0 += kch) {
        const bool first = (s0 == kb0), last = (s0 + kch >= kb1);
        mbar_wait(tfull, tphase);
        tphase ^= 1u;
        tc::fence_after_sync();
#pragma unroll 1
        for (int c0 = cb; c0 < ce; c0 += 32) {
          float v[32];
          tc::tmem_ld32(taddr + c0, v);
          if (!first) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += __ldcg(accp + (size_t)(c0 + j) * 128);
          }
          if (!last) {
#pragma unroll
            for (int j = 0; j < 32; ++j) __stcg(accp + (size_t)(c0 + j) * 128, v[j]);
          } else if (whole) {
            if (row_ok) {
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const size_t o = (size_t)(c0 + j) * args.ldy + row;
                float y = s1 * v[j];
                if (s2 != 0.f) y = fmaf(s2, args.ycur[o], y);
                if (s3 != 0.f) y = fmaf(s3, args.yprev[o], y);
                args.out[o] = y;
              }
            }
          } else {  // split-K partial of a tail tile
#pragma unroll
            for (int j = 0; j < 32; ++j) __stcg(mine + (size_t)(c0 + j) * 128, v[j]);
          }
        }
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_cluster(tempty_leader);  // TMEM free: MMA may go on
      }
      if (!whole) {
        // -------------------------------------------------- split-K fixup (last contributor)
        __threadfence();
        named_bar_sync(1, 256);
        if (threadIdx.x == 256) {
          const int add = kb1 - kb0;
          const int prev = atomicAdd(&args.counters[tile * 2 + crank], add);
          *sflag = (prev + add == KB) ? 1 : 0;
        }
        named_bar_sync(1, 256);
        const bool lastc = (*sflag != 0);
        named_bar_sync(1, 256);
        if (lastc) {
          __threadfence();
          const int u0 = (tile - sch.F * G) * sch.S;  // first contributing pair
#pragma unroll 1
          for (int c0 = cb; c0 < ce; c0 += 32) {
            float acc[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[j] = 0.f;
#pragma unroll 1
            for (int c = 0; c < sch.S; ++c) {
              const float* src = args.ws + ((size_t)(u0 + c) * 2 + crank) * (size_t)(P * 128) +
                                 (size_t)c0 * 128 + et;
#pragma unroll
              for (int j = 0; j < 32; ++j) acc[j] += __ldcg(src + (size_t)j * 128);
            }
            if (row_ok) {
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const size_t o = (size_t)(c0 + j) * args.ldy + row;
                float y = s1 * acc[j];
                if (s2 != 0.f) y = fmaf(s2, args.ycur[o], y);
                if (s3 != 0.f) y = fmaf(s3, args.yprev[o], y);
                args.out[o] = y;
              }
            }
          }
          named_bar_sync(1, 256);
          if (threadIdx.x == 256) args.counters[tile * 2 + crank] = 0;  // ready for next launch
        }
      }
    }
  }

  __syncwarp();
  tc::fence_before_sync();
  tc::cluster_sync();
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc_pair<C::TMEM_COLS>(tmem);
  }
}

// ------------------------------------------------------------------------------ host side
bool encode_map_f32(CUtensorMap* map, const float* base, int64_t pitch, int rows, int cols,
                    int box_rows, int box_cols = 16, bool swizzle = true);

Tf32Plan tf32_plan(int p, int n_rows, int n_k, int num_sms) {
  Tf32Plan pl;
  pl.p = p;
  pl.n_rows = n_rows;
  pl.n_k = n_k;
  pl.mtiles = (n_rows + 255) / 256;
  pl.kblocks = (n_k + 15) / 16;
  const int smax = std::max(1, std::min(16, pl.kblocks / 8));  // >= 8 k-blocks per chunk
  int G = std::max(1, num_sms / 2);
  G = std::min<long long>(G, (long long)pl.mtiles * smax);
  const int R = pl.mtiles % G;
  pl.pairs = G;
  pl.split = R ? std::max(1, std::min(smax, G / R)) : 1;
  pl.ws_floats = (size_t)G * 2 * (size_t)p * 128;
  pl.acc_floats = pl.ws_floats;
  // K_c = 4096 per TMEM accumulation (truncating accumulator, see kernel): error floor 1.9e-5 on
  // config 5 vs 9.2e-6 at K_c = 2048, half the fold traffic (profiles/r01_tf32_schedule.txt)
  pl.chunk_kb = 256;
  if (const char* e = getenv("PF_TF32_CHUNK_KB")) pl.chunk_kb = atoi(e);  // development knob
  // L2 prefetch of A off by default: measured to evict Y and the fold accumulators (DRAM reads
  // 28.2 -> 20.5 GB per pass at n = 65536, p = 512, and slower; profiles/r01_tf32_dram.txt)
  pl.pf_dist = 0;
  if (const char* e = getenv("PF_TF32_PFDIST")) pl.pf_dist = atoi(e);     // development knob
  pl.counters = (size_t)pl.mtiles * 2;
  return pl;
}

bool tf32_encode_A(CUtensorMap* map, CUtensorMap* map_pf, const float* A, int64_t lda,
                   int n_rows, int n_k) {
  return encode_map_f32(map, A, lda, n_rows, n_k, 128) &&
         encode_map_f32(map_pf, A, lda, n_rows, n_k, 128, 32, false);
}
bool tf32_encode_B(CUtensorMap* map, const float* Yt, int64_t ldy, int p, int n_k) {
  return encode_map_f32(map, Yt, ldy, p, n_k, std::min(p, 256) / 2);
}


template <int P>
static cudaError_t tf32_launch_p(const Tf32Plan& pl, const CUtensorMap& mapA,
                                 const CUtensorMap& mapB, const CUtensorMap& mapApf,
                                 const Tf32Args& a, cudaStream_t st) {
  using C = Tf32Cfg<P>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(cheb_gemm_tf32_kernel<P>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  count_launch();
  cheb_gemm_tf32_kernel<P><<<2 * pl.pairs, C::THREADS, C::SMEM, st>>>(mapA, mapB, mapApf, a);
  return cudaGetLastError();
}

cudaError_t tf32_gemm_launch(const Tf32Plan& pl, const CUtensorMap& mapA, const CUtensorMap& mapB,
                             const CUtensorMap& mapApf,
                             const float* ycur, const float* yprev, float* out, int64_t ldy,
                             const double* coef, float* ws, float* acc, int* counters,
                             int npass, cudaStream_t st, int bdist_kb) {
  Tf32Args a;
  a.ycur = ycur;
  a.yprev = yprev;
  a.out = out;
  a.coef = coef;
  a.ws = ws;
  a.counters = counters;
  a.ldy = ldy;
  a.n_rows = pl.n_rows;
  a.kblocks = pl.kblocks;
  a.mtiles = pl.mtiles;
  a.split = pl.split;
  a.npass = npass;
  a.chunk_kb = pl.chunk_kb;
  a.pf_dist = pl.pf_dist;
  a.bdist_kb = bdist_kb;
  a.acc = acc;
  switch (pl.p) {
    case 64: return tf32_launch_p<64>(pl, mapA, mapB, mapApf, a, st);
    case 128: return tf32_launch_p<128>(pl, mapA, mapB, mapApf, a, st);
    case 256: return tf32_launch_p<256>(pl, mapA, mapB, mapApf, a, st);
    case 512: return tf32_launch_p<512>(pl, mapA, mapB, mapApf, a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace pf
