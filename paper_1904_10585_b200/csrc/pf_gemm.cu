// pf_gemm.cu -- the Chebyshev-step filter GEMM (hot loop of eq:cheb / eqn:subspace-update,
// P:185-227): out = s1 * (A B) + s2 * Ycur + s3 * Yprev, with A the n_rows x n_k row block of the
// dense symmetric iterate and B = Y_j (n_k x p).  One launch per Chebyshev step; the same
// kernel computes W = A Q for Rayleigh-Ritz (s1 = 1, s2 = s3 = 0).
//
// B200 design (DESIGN.md §4 K1):
//  * fp64 tensor cores: mma.sync.m16n8k4.f64 (SASS DMMA.8x8x4) -- tcgen05 has no f64 kind.
//  * A and B tiles staged by TMA (cp.async.bulk.tensor.2d) into a STAGES-deep smem ring guarded
//    by mbarriers; A uses the 128-byte swizzle so the m16n8k4 fragment loads are conflict-free.
//  * one producer warp (TMA) + 8 consumer warps; 1 CTA per SM.
//  * stream-K: the (m-tile, k-block) iteration space is split evenly over `grid` = #SMs CTAs, so
//    the 128-256 m-tiles of the filter shapes do not leave SMs idle.  Partial tiles are written
//    to a workspace and the LAST contributor (atomic tile counter) sums all partials in fixed
//    CTA order -> deterministic results, no co-residency assumption.
//  * the Chebyshev recurrence's scale-shift-subtract is applied in the epilogue of the owner.
#include <algorithm>

#include "pf_kernels.cuh"

namespace pf {

template <int P>
struct GemmCfg {
  // 9 warps per CTA -> one SMSP hosts 3 warps -> <= 168 registers per thread (16K regs/SMSP),
  // so every warp tile is kept at <= 32 x 32 doubles of accumulator: BM = 64 for P = 128.
  // BK = 32: two 16-column SWIZZLE_128B A sub-tiles per stage (8 k4-steps between barriers)
  static constexpr int BM = (P >= 128) ? 64 : 128, BK = 32;
  static constexpr int NCW = 8;  // consumer warps
  static constexpr int NCT = NCW * 32;
  static constexpr int THREADS = NCT + 32;
  static constexpr int WARPS_M = (P >= 128) ? 2 : ((P >= 64) ? 4 : 8);
  static constexpr int WARPS_N = NCW / WARPS_M;
  static constexpr int WM = BM / WARPS_M;
  static constexpr int WN = P / WARPS_N;
  static constexpr int MT = WM / 16;
  static constexpr int NT = WN / 8;
  static constexpr int NACC = MT * NT * 4;
  static constexpr int A_BYTES = BM * BK * 8;
  static constexpr int B_BYTES = BK * P * 8;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES_RAW = (200 * 1024) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 10 ? 10 : STAGES_RAW;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align slack*/ + 2 * STAGES * 8 + 64;
  static_assert(WN % 8 == 0 && WM % 16 == 0, "warp tile");
  static_assert(A_BYTES % 1024 == 0, "A tiles must stay 1024-byte aligned for SWIZZLE_128B");
};

struct ChebArgs {
  const double* ycur;
  const double* yprev;
  double* out;
  const double* coef;
  double* ws;
  int* counters;
  int n_rows;
  int kblocks;
  long long total;
};

// owner of iteration i: largest q with floor(T q / G) <= i
__device__ __forceinline__ int cta_of(long long i, long long T, int G) {
  return (int)(((i + 1) * (long long)G + T - 1) / T) - 1;
}

template <int P>
__global__ void __launch_bounds__(GemmCfg<P>::THREADS, 1)
    cheb_gemm_kernel(const __grid_constant__ CUtensorMap mapA,
                     const __grid_constant__ CUtensorMap mapB, ChebArgs args) {
  using C = GemmCfg<P>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // align to 1024 B (SWIZZLE_128B atom) by pointer offset so the compiler keeps the shared
  // address space (a uintptr_t round trip would turn every fragment load into a generic LD)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  double* sA = reinterpret_cast<double*>(smem);
  double* sB = reinterpret_cast<double*>(smem + C::STAGES * C::A_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  volatile int* sflag = reinterpret_cast<volatile int*>(empty + C::STAGES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NCW);
    }
    fence_mbar_init();
  }
  if (warp == C::NCW && lane == 0) {
    tma_prefetch_desc(&mapA);
    tma_prefetch_desc(&mapB);
  }
  __syncthreads();

  const long long T = args.total;
  const int G = gridDim.x, g = blockIdx.x;
  const int KB = args.kblocks;
  const long long it_begin = T * g / G, it_end = T * (g + 1) / G;

  if (warp == C::NCW) {
    // ------------------------------------------------------------ TMA producer (one lane)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (long long it = it_begin; it < it_end; ++it) {
        const int tile = (int)(it / KB), kb = (int)(it % KB);
        mbar_wait(&empty[stage], phase ^ 1u);
        mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
#pragma unroll
        for (int sub = 0; sub < C::BK / 16; ++sub)
          tma_load_2d(sA + stage * (C::BM * C::BK) + sub * (C::BM * 16), &mapA, &full[stage],
                      kb * C::BK + 16 * sub, tile * C::BM);
        // B = Y_j rows [kb*BK, (kb+1)*BK): P/8 boxes of BK x 8 doubles, SWIZZLE_64B each
#pragma unroll
        for (int j = 0; j < P / 8; ++j)
          tma_load_2d(sB + stage * (C::BK * P) + j * (C::BK * 8), &mapB, &full[stage], 8 * j,
                      kb * C::BK);
        if (++stage == C::STAGES) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers (8 warps)
  const int ctid = threadIdx.x;  // 0 .. NCT-1
  const int wm = warp % C::WARPS_M, wn = warp / C::WARPS_M;
  const int g8 = lane >> 2, t4 = lane & 3;
  int stage = 0;
  uint32_t phase = 0;

  // per-thread constant parts of the swizzled A fragment address (in doubles)
  // element (r, k) of a BM x 16 tile with SWIZZLE_128B: r*16 + (((k>>1) ^ (r&7)) << 1) + (k&1)
  int a_off[C::MT][4];
#pragma unroll
  for (int mt = 0; mt < C::MT; ++mt) {
    const int r = wm * C::WM + mt * 16 + g8;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int k = ks * 4 + t4;
      a_off[mt][ks] = r * 16 + ((((k >> 1) ^ (r & 7))) << 1) + (k & 1);
    }
  }
  // B stage = P/8 boxes [BK k][8 n] with SWIZZLE_64B (16-byte chunk ^= (k >> 1) & 3):
  // element (k, n): (n >> 3) * 8 BK + k * 8 + ((((n & 7) >> 1) ^ ((k >> 1) & 3)) << 1) + (n & 1)
  int b_off[C::BK / 4];
#pragma unroll
  for (int ks = 0; ks < C::BK / 4; ++ks) {
    const int k = ks * 4 + t4;
    b_off[ks] = ((wn * C::WN) >> 3) * (C::BK * 8) + k * 8 +
                ((((g8 >> 1) ^ ((k >> 1) & 3))) << 1) + (g8 & 1);
  }

  long long it = it_begin;
  while (it < it_end) {
    const int tile = (int)(it / KB);
    const int kb0 = (int)(it % KB);
    const long long seg_end = min(it_end, (long long)(tile + 1) * KB);
    const int kb1 = kb0 + (int)(seg_end - it);

    double acc[C::MT][C::NT][4];
#pragma unroll
    for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[mt][nt][i] = 0.0;

    for (int kb = kb0; kb < kb1; ++kb) {
      mbar_wait(&full[stage], phase);
      const double* a = sA + stage * (C::BM * C::BK);
      const double* b = sB + stage * (C::BK * P);
#pragma unroll
      for (int ks = 0; ks < C::BK / 4; ++ks) {
        double af[C::MT][2], bf[C::NT];
        const int sub = (ks >> 2) * (C::BM * 16);  // A sub-tile of this k-step
#pragma unroll
        for (int mt = 0; mt < C::MT; ++mt) {
          af[mt][0] = a[sub + a_off[mt][ks & 3]];
          af[mt][1] = a[sub + a_off[mt][ks & 3] + 8 * 16];
        }
#pragma unroll
        for (int nt = 0; nt < C::NT; ++nt) bf[nt] = b[b_off[ks] + nt * (C::BK * 8)];
#pragma unroll
        for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < C::NT; ++nt) dmma16884(acc[mt][nt], af[mt][0], af[mt][1], bf[nt]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == C::STAGES) {
        stage = 0;
        phase ^= 1u;
      }
    }

    bool do_epilogue = true;
    if (!(kb0 == 0 && kb1 == KB)) {
      // ---------------------------------------------------- stream-K partial tile
      const int slot = (it == it_begin) ? 0 : 1;
      double* mine = args.ws + (size_t)(g * 2 + slot) * (C::NCT * C::NACC);
#pragma unroll
      for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
          for (int i = 0; i < 4; ++i)
            __stcg(mine + ((mt * C::NT + nt) * 4 + i) * C::NCT + ctid, acc[mt][nt][i]);
      __threadfence();
      named_bar_sync(1, C::NCT);
      if (ctid == 0) {
        const int add = kb1 - kb0;
        const int prev = atomicAdd(&args.counters[tile], add);
        *sflag = (prev + add == KB) ? 1 : 0;
      }
      named_bar_sync(1, C::NCT);
      do_epilogue = (*sflag != 0);
      named_bar_sync(1, C::NCT);  // sflag reused by the next segment
      if (do_epilogue) {
        __threadfence();
        const long long t0 = (long long)tile * KB;
        const int gf = cta_of(t0, T, G), gl = cta_of(t0 + KB - 1, T, G);
#pragma unroll
        for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[mt][nt][i] = 0.0;
        for (int q = gf; q <= gl; ++q) {
          const long long qb = T * q / G;
          const int qslot = (qb >= t0) ? 0 : 1;
          const double* src = args.ws + (size_t)(q * 2 + qslot) * (C::NCT * C::NACC);
#pragma unroll
          for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
              for (int i = 0; i < 4; ++i)
                acc[mt][nt][i] += __ldcg(src + ((mt * C::NT + nt) * 4 + i) * C::NCT + ctid);
        }
        if (ctid == 0) args.counters[tile] = 0;  // ready for the next launch
      }
    }

    if (do_epilogue) {
      // ------------------------------------------------------ fused Chebyshev epilogue
      const double s1 = args.coef[0], s2 = args.coef[1], s3 = args.coef[2];
#pragma unroll
      for (int mt = 0; mt < C::MT; ++mt) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = tile * C::BM + wm * C::WM + mt * 16 + g8 + h * 8;
          if (row >= args.n_rows) continue;
#pragma unroll
          for (int nt = 0; nt < C::NT; ++nt) {
            const int col = wn * C::WN + nt * 8 + 2 * t4;
            const size_t o = (size_t)row * P + col;
            double2 v;
            v.x = s1 * acc[mt][nt][2 * h];
            v.y = s1 * acc[mt][nt][2 * h + 1];
            if (s2 != 0.0) {
              const double2 y = *reinterpret_cast<const double2*>(args.ycur + o);
              v.x += s2 * y.x;
              v.y += s2 * y.y;
            }
            if (s3 != 0.0) {
              const double2 y = *reinterpret_cast<const double2*>(args.yprev + o);
              v.x += s3 * y.x;
              v.y += s3 * y.y;
            }
            *reinterpret_cast<double2*>(args.out + o) = v;
          }
        }
      }
    }
    it = seg_end;
  }
}

// ------------------------------------------------------------------------------ host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

bool encode_map_A(CUtensorMap* map, const double* A, int64_t lda, int n_rows, int n_k, int p) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)n_k, (cuuint64_t)n_rows};
  cuuint64_t strides[1] = {(cuuint64_t)lda * 8};
  cuuint32_t box[2] = {16, (cuuint32_t)((p >= 128) ? 64 : 128)};
  cuuint32_t es[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(A), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// generic tiled map (pf_rebuild_i8.cu): element type fp64 (f64) or bytes, rank 2 or 3, strides
// in bytes for dims 1.., swizzle span 0 / 32 / 64 / 128 bytes
bool encode_map_gen(CUtensorMap* map, bool f64, int rank, const void* base, const uint64_t* dims,
                    const uint64_t* strides, const uint32_t* box, int swizzle) {
  PFN_encodeTiled enc = get_encode();
  if (!enc || rank < 2 || rank > 3) return false;
  cuuint64_t d[3], s[2];
  cuuint32_t b[3], es[3] = {1, 1, 1};
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    if (i) s[i - 1] = strides[i - 1];
  }
  const CUtensorMapSwizzle sw = swizzle == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                : swizzle == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                : CU_TENSOR_MAP_SWIZZLE_NONE;
  return enc(map, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_UINT8,
             (cuuint32_t)rank, const_cast<void*>(base), d, s, b, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool encode_map_B(CUtensorMap* map, const double* B, int p, int n_k) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)p, (cuuint64_t)n_k};
  cuuint64_t strides[1] = {(cuuint64_t)p * 8};
  cuuint32_t box[2] = {8, (cuuint32_t)GemmCfg<64>::BK};
  cuuint32_t es[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(B), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// fp32 2-D map for the TF32 filter GEMM: rows x cols (cols contiguous, pitch in elements),
// box = box_cols (16 -> 64 bytes, SWIZZLE_64B) x box_rows; unswizzled boxes are L2 prefetches.
bool encode_map_f32(CUtensorMap* map, const float* base, int64_t pitch, int rows, int cols,
                    int box_rows, int box_cols, bool swizzle) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)pitch * 4};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
             box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             swizzle ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// int8 digit slices [slices][rows][cols] (pitch bytes per row, slice_pitch bytes per slice),
// SWIZZLE_64B boxes {64 bytes, box_rows, box_slices}; out-of-range K reads as zero digits.
bool encode_map_i8_3d(CUtensorMap* map, const int8_t* base, int64_t pitch, int64_t slice_pitch,
                      int cols, int rows, int slices, int box_rows, int box_slices, bool swizzle) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)slices};
  cuuint64_t strides[2] = {(cuuint64_t)pitch, (cuuint64_t)slice_pitch};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, (cuuint32_t)box_slices};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             swizzle ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Rank-major all-gather of p-major blocks: [world][p][n_local] contiguous (n_local % 16 == 0).
bool tf32_encode_B_dist(CUtensorMap* map, const float* Yg, int p, int n_local, int world) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)n_local, (cuuint64_t)p, (cuuint64_t)world};
  cuuint64_t strides[2] = {(cuuint64_t)n_local * 4, (cuuint64_t)n_local * 4 * p};
  cuuint32_t box[3] = {16, (cuuint32_t)(std::min(p, 256) / 2), 1};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(Yg), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int P>
static size_t ws_per_cta() {
  return (size_t)2 * GemmCfg<P>::NCT * GemmCfg<P>::NACC;
}

ChebGemmPlan cheb_gemm_plan(int p, int n_rows, int n_k, int num_sms) {
  ChebGemmPlan pl;
  pl.p = p;
  pl.n_rows = n_rows;
  pl.n_k = n_k;
  const int bm = (p >= 128) ? 64 : 128;
  pl.mtiles = (n_rows + bm - 1) / bm;
  pl.kblocks = (n_k + GemmCfg<64>::BK - 1) / GemmCfg<64>::BK;  // BK is the same for every P
  const long long T = (long long)pl.mtiles * pl.kblocks;
  // at least 8 k-blocks per CTA so the fixup stays amortised
  long long g = std::min<long long>(num_sms, std::max<long long>(1, T / 8));
  pl.grid = (int)g;
  size_t per = 0;
  switch (p) {
    case 16: per = ws_per_cta<16>(); break;
    case 32: per = ws_per_cta<32>(); break;
    case 64: per = ws_per_cta<64>(); break;
    case 128: per = ws_per_cta<128>(); break;
    default: per = ws_per_cta<128>(); break;
  }
  pl.ws_doubles = per * (size_t)num_sms;
  return pl;
}

template <int P>
static cudaError_t launch_p(const ChebGemmPlan& pl, const CUtensorMap& mapA,
                            const CUtensorMap& mapB, const ChebArgs& a, cudaStream_t st) {
  using C = GemmCfg<P>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(cheb_gemm_kernel<P>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  count_launch();
  cheb_gemm_kernel<P><<<pl.grid, C::THREADS, C::SMEM, st>>>(mapA, mapB, a);
  return cudaGetLastError();
}

cudaError_t cheb_gemm_launch(const ChebGemmPlan& pl, const CUtensorMap& mapA,
                             const CUtensorMap& mapB, const double* ycur, const double* yprev,
                             double* out, const double* coef, double* ws, int* counters,
                             cudaStream_t st) {
  ChebArgs a;
  a.ycur = ycur;
  a.yprev = yprev;
  a.out = out;
  a.coef = coef;
  a.ws = ws;
  a.counters = counters;
  a.n_rows = pl.n_rows;
  a.kblocks = pl.kblocks;
  a.total = (long long)pl.mtiles * pl.kblocks;
  switch (pl.p) {
    case 16: return launch_p<16>(pl, mapA, mapB, a, st);
    case 32: return launch_p<32>(pl, mapA, mapB, a, st);
    case 64: return launch_p<64>(pl, mapA, mapB, a, st);
    case 128: return launch_p<128>(pl, mapA, mapB, a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace pf
