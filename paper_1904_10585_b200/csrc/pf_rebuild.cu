// pf_rebuild.cu -- fused rank-p rebuild + elementwise update (step a6 of SURVEY §8(a)):
//   PFPG (eq:pfpg1):  X = V diag(f) V^T,  A+ = X - tau * Omega o (X - M),  M = W W^T,
//                                obj = {1/2 ||P_Omega(X - M)||_F^2, sum |f|}
//   PFAM (eq:PFAM1, prox sign corrected -- reading R1), max-cut SDP (A = diag, b = 1):
//                                W = V diag(f) V^T,
//                                Z+ = offdiag(W - tC) + Diag(1 - W_ii + Z_ii),  C = -L/4,
//                                obj = {<C, W>, ||Z+ - Z||_F}
// B200 design (DESIGN.md §4 K7):
//  * 64 x 64 output tiles on fp64 DMMA (K = p); the I panel is V diag(f) (scaled once per
//    call by scale_cols_kernel), the J panel V;
//  * single GPU (whole rows): only tiles I <= J are computed; the (J, I) tile is written as the
//    transpose straight from the accumulator fragments -> n^2 p flops instead of 2 n^2 p, and the
//    old iterate is read only on the upper half (PFAM; Z is symmetric by contract), none at all
//    for PFPG;
//  * each persistent CTA owns a contiguous range of tile pairs, so consecutive tiles share the
//    row block I and its staged V diag(f) panel is reused;
//  * V panels staged with cp.async, the old-iterate tile prefetched into registers before the
//    MMA loop so its HBM latency overlaps the math; masks (Omega / adjacency) are packed bits.
//  * reductions are deterministic: per-CTA partials summed in CTA order by the last CTA.
#include <algorithm>
#include <climits>
#include <cmath>

#include "pf_digits.cuh"
#include "pf_kernels.cuh"

namespace pf {

constexpr int kRb = 64;          // tile edge
constexpr int kRbThreads = 256;  // 8 warps (2 x 4), warp tile 32 x 16: ~half the accumulator and
                                 // prefetch registers of a 32 x 32 warp tile -> 16 warps / SM
constexpr int kWn = 16, kNt = kWn / 8;

struct RbArgs {
  const double* V;   // all n rows (J panels)
  int64_t ldv;
  const double* VF;  // local rows of V diag(f) (I panels), pitch p

  const double* f;
  double tt;  // tau (PFPG) or t (PFAM)
  const uint32_t* bits;
  int64_t ldb;
  const double* W;
  int64_t ldw;
  int r, rpad;
  int w_async;  // W rows 16-byte aligned (even ldw, aligned base): stage W panels with cp.async
  const double* deg;
  double* Out;
  int64_t ldo;
  int n_rows, n, row0;
  int sym, T;
  int raw;  // 1: obj[1] (PFAM) is left as the raw sum of squares for a cross-rank all-reduce
  double* partials;
  int* counter;
  double* obj;
  // PF_FP64_I8 (PFAM, one GPU): the update also writes the S-digit slices of Z_new for the next
  // filter (A8 != nullptr): row exponents E (row bounds computed before the update), slices
  // in the tiled layout of pf_digits.cuh a8_offset (KB k-blocks) -- the separate split pass over
  // Z disappears
  int8_t* A8;
  int KB;
  const int* E;     // the digit scale exponent Eg (one int, pfam_bound2_kernel)
  int S;
  double* rscale;   // row scales of the digit slices (all 2^Eg), written by the update
};

template <int P, bool PFPG>
struct RbCfg {
  static constexpr int LD = P + 4;
  static constexpr int LDS = kRb + 1;  // transpose staging row pitch
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// decode pair index e (0 <= e < T(T+1)/2) into (I, J), I <= J, row-major over the upper triangle
__device__ __forceinline__ void pair_of(int e, int T, int& I, int& J) {
  // number of pairs before row I: I*T - I*(I-1)/2
  double b = 2.0 * T + 1.0;
  int i = (int)floor((b - sqrt(b * b - 8.0 * e)) * 0.5);
  if (i < 0) i = 0;
  while (i > 0 && (long long)i * T - (long long)i * (i - 1) / 2 > e) --i;
  while ((long long)(i + 1) * T - (long long)(i + 1) * i / 2 <= e) ++i;
  I = i;
  J = i + (e - (int)((long long)i * T - (long long)i * (i - 1) / 2));
}

// Z_new staging for the digit output: 4 x 4 blocks stored column-block-major, 16 doubles + 2 pad
// per block (lanes reading 16-byte chunks of consecutive blocks hit distinct bank groups)
constexpr int kTzBlk = 18;
__device__ __forceinline__ int tz4(int r, int c) {
  return ((c >> 2) * (kRb / 4) + (r >> 2)) * kTzBlk + (r & 3) * 4 + (c & 3);
}
constexpr int kDgPitch = 80;  // bytes per staged digit row (64 + 16: 16-byte rows, few conflicts)
static_assert(7 * kRb * kDgPitch <= (kRb / 4) * (kRb / 4) * kTzBlk * 8, "digit staging fits");

// Z_new tile (64 x 64, staged in Tz4) -> digit slices of the tile AND of its mirror.  The fused
// digits use ONE scale 2^E for the whole matrix (E = the max of the row-bound exponents), so the
// mirror tile's digits are the byte transpose of the tile's: thread t owns the 4 x 4 block
// (rows 4 (t % 16).., cols 4 (t / 16)..) and forms its digit words once (4 rows x S slices, a
// word = 4 consecutive columns).  Mirror rows: the 4 x 4 byte transpose of each slice's words,
// stored directly (16 consecutive lanes = one 64-byte mirror row).  Tile rows: staged through
// shared memory (the same buffer, after every thread has read its values) and stored as 16-byte
// row pieces.  Entries outside the matrix are written as 0.
template <int S, bool FULL>
__device__ __forceinline__ void rb_digits(const RbArgs& a, double* Tz, int i0, int j0,
                                          bool mirror, int tid, int E) {
  // FULL: the tile and its mirror lie inside the matrix (no bounds checks; constant offsets)
  const int rb = (tid & 15) * 4, cb = (tid >> 4) * 4;
  uint32_t w[4][S];
  const double* blk = Tz + ((cb >> 2) * (kRb / 4) + (rb >> 2)) * kTzBlk;
  const int c = j0 + cb;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double2 v01 = *reinterpret_cast<const double2*>(blk + i * 4);
    const double2 v23 = *reinterpret_cast<const double2*>(blk + i * 4 + 2);
    if (FULL) {
      i8::slices4<S>(v01.x, v01.y, v23.x, v23.y, E, w[i]);
    } else {
      const bool rok = i0 + rb + i < a.n_rows;
      i8::slices4<S>(rok && c < a.n ? v01.x : 0.0, rok && c + 1 < a.n ? v01.y : 0.0,
                     rok && c + 2 < a.n ? v23.x : 0.0, rok && c + 3 < a.n ? v23.y : 0.0, E,
                     w[i]);
    }
  }
  if (mirror && (FULL || i0 + rb < a.n)) {
    // rows c .. c+3 of the mirror share one 128-row tile: slice s, row c + j at + s 8 KB + 64 j
    int8_t* base = a.A8 + i8::a8_offset(c, i0 + rb, 0, a.KB, S);
#pragma unroll
    for (int sl = 0; sl < S; ++sl) {
      uint32_t t[4];
      i8::transpose4(w[0][sl], w[1][sl], w[2][sl], w[3][sl], t);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (FULL || c + j < a.n)
          __stcs(reinterpret_cast<uint32_t*>(base + sl * 8192 + j * 64), t[j]);
    }
  }
  __syncthreads();  // every thread has read its values: the staging becomes the digit buffer
  uint8_t* dg = reinterpret_cast<uint8_t*>(Tz);  // [S][64 rows][kDgPitch]
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int sl = 0; sl < S; ++sl)
      *reinterpret_cast<uint32_t*>(dg + (sl * kRb + rb + i) * kDgPitch + cb) = w[i][sl];
  __syncthreads();
  // tile rows: thread t stores the 16-byte piece q = t % 4 of row t / 4 of every slice
  const int row = tid >> 2, q = tid & 3;
  if (FULL || (j0 < a.n && i0 + row < a.n_rows)) {
    int8_t* base = a.A8 + i8::a8_offset(i0 + row, j0 + 16 * q, 0, a.KB, S);
#pragma unroll
    for (int sl = 0; sl < S; ++sl)
      __stcs(reinterpret_cast<uint4*>(base + sl * 8192),
             *reinterpret_cast<const uint4*>(dg + (sl * kRb + row) * kDgPitch + 16 * q));
  }
}

template <int S>
__device__ __forceinline__ void rb_digits_any(const RbArgs& a, double* Tz, int i0, int j0,
                                              bool mirror, int tid, int E, bool full) {
  if (full) rb_digits<S, true>(a, Tz, i0, j0, mirror, tid, E);
  else rb_digits<S, false>(a, Tz, i0, j0, mirror, tid, E);
}

template <int P, bool PFPG>
__global__ void __launch_bounds__(kRbThreads, 2) rebuild_kernel(const RbArgs a) {
  using C = RbCfg<P, PFPG>;
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[32];
  __shared__ int s_last;
  const int ldw_s = a.rpad + 4;
  double* Vi = sm;                  // 64 x LD  rows I (local row block)
  double* Vj = sm + kRb * C::LD;    // 64 x LD  rows J
  double* Wi = Vj + kRb * C::LD;    // 64 x ldw_s (PFPG)
  double* Wj = Wi + kRb * ldw_s;
  double* Tz = Vj + kRb * C::LD;    // block-major staging of Z_new (PFAM digit output, tz4)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g8 = lane >> 2, t4 = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;  // 2 (rows) x 4 (cols) warps, 32 x 16 each
  const int tc = (a.n + kRb - 1) / kRb, tr = (a.n_rows + kRb - 1) / kRb;
  const int ntiles = a.sym ? (tc * (tc + 1)) / 2 : tr * tc;
  // 16-byte stores of row pairs need an aligned base and an even pitch
  const bool al = ((reinterpret_cast<uintptr_t>(a.Out) & 15) == 0) && ((a.ldo & 1) == 0);
  if (PFPG && a.w_async)  // zero padding columns of both W panels (never written by cp.async)
    for (int e = tid; e < kRb * ldw_s; e += kRbThreads)
      if (e % ldw_s >= a.r - (a.r & 1)) Wi[e] = Wj[e] = 0.0;
  double s0 = 0.0, s1 = 0.0;
  // persistent CTAs: each owns a CONTIGUOUS range of tiles (deterministic sums; in the row-major
  // upper-triangle order consecutive tiles share the row block I, so the staged I panel is
  // reused), one reduction at the end
  const long long nt_all = ntiles;
  const int t_begin = (int)(nt_all * blockIdx.x / gridDim.x);
  const int t_end = (int)(nt_all * (blockIdx.x + 1) / gridDim.x);
  int curI = -1;
  // digits of the previous tile's Z_new (staged in Tz) are written during this tile's panel loads
  int pv_i0 = -1, pv_j0 = 0;
  bool pv_mirror = false, pv_full = false;
  // one digit scale 2^Eg for the whole matrix (pfam_bound2_kernel); the row scales the next
  // product reads are all 2^Eg
  int Eg = 0;
  if (!PFPG && a.A8) {
    Eg = *a.E;
    const double sc = i8::pow2(Eg);
    for (int i = blockIdx.x * kRbThreads + tid; i < a.n_rows; i += gridDim.x * kRbThreads)
      a.rscale[i] = sc;
  }
  for (int tile = t_begin; tile < t_end; ++tile) {
  int I, J;
  if (a.sym) {
    pair_of(tile, a.T, I, J);
  } else {
    I = tile / tc;
    J = tile % tc;
  }
  const int i0 = I * kRb, j0 = J * kRb;  // local row tile start, global column tile start
  const bool mirror = a.sym && I < J;
  const double wgt = mirror ? 2.0 : 1.0;
  const bool newI = (I != curI);
  curI = I;
  // fast tile: inside the matrix, off the global diagonal, aligned rows -- the epilogue runs
  // without bounds, diagonal or alignment checks
  const int gi0 = a.row0 + i0;
  const bool full = i0 + kRb <= a.n_rows && j0 + kRb <= a.n;
  const bool fast = full && al && !(gi0 < j0 + kRb && j0 < gi0 + kRb);
  __syncthreads();  // the previous tile's readers of the panels are done

  // ---- stage V panels (cp.async 16 B), f, W panels; the I panel only when I changed
  for (int e = tid; e < kRb * (P / 2); e += kRbThreads) {
    const int rr = e / (P / 2), c = (e % (P / 2)) * 2;
    double* di = Vi + rr * C::LD + c;
    double* dj = Vj + rr * C::LD + c;
    if (newI) {
      if (i0 + rr < a.n_rows) cp_async16(di, a.VF + (size_t)(i0 + rr) * P + c);
      else *reinterpret_cast<double2*>(di) = make_double2(0.0, 0.0);
    }
    if (j0 + rr < a.n) cp_async16(dj, a.V + (size_t)(j0 + rr) * a.ldv + c);
    else *reinterpret_cast<double2*>(dj) = make_double2(0.0, 0.0);
  }
  if (PFPG && a.w_async) {
    // W panels by cp.async (plain loads + stores stalled every thread on its own loads); the
    // padding columns r .. ldw_s-1 were zeroed once and are never written
    const int r2 = a.r >> 1;
    for (int e = tid; e < kRb * r2; e += kRbThreads) {
      const int rr = e / r2, c = (e - rr * r2) * 2;
      if (newI) {
        double* d = Wi + rr * ldw_s + c;
        if (i0 + rr < a.n_rows) cp_async16(d, a.W + (size_t)(a.row0 + i0 + rr) * a.ldw + c);
        else *reinterpret_cast<double2*>(d) = make_double2(0.0, 0.0);
      }
      double* d = Wj + rr * ldw_s + c;
      if (j0 + rr < a.n) cp_async16(d, a.W + (size_t)(j0 + rr) * a.ldw + c);
      else *reinterpret_cast<double2*>(d) = make_double2(0.0, 0.0);
    }
    if (a.r & 1) {  // odd rank: the last column by plain loads
      const int c = a.r - 1;
      for (int rr = tid; rr < kRb; rr += kRbThreads) {
        if (newI) Wi[rr * ldw_s + c] = i0 + rr < a.n_rows ? a.W[(size_t)(a.row0 + i0 + rr) * a.ldw + c] : 0.0;
        Wj[rr * ldw_s + c] = j0 + rr < a.n ? a.W[(size_t)(j0 + rr) * a.ldw + c] : 0.0;
      }
    }
  } else if (PFPG) {
    for (int e = tid; e < kRb * ldw_s; e += kRbThreads) {
      const int rr = e / ldw_s, c = e % ldw_s;
      if (newI)
        Wi[e] = (c < a.r && i0 + rr < a.n_rows) ? a.W[(size_t)(a.row0 + i0 + rr) * a.ldw + c] : 0.0;
      Wj[e] = (c < a.r && j0 + rr < a.n) ? a.W[(size_t)(j0 + rr) * a.ldw + c] : 0.0;
    }
  }

  if (!PFPG && a.A8 && pv_i0 >= 0) {  // overlaps the cp.async panel loads in flight
    if (a.S == 7) rb_digits_any<7>(a, Tz, pv_i0, pv_j0, pv_mirror, tid, Eg, pv_full);
    else rb_digits_any<6>(a, Tz, pv_i0, pv_j0, pv_mirror, tid, Eg, pv_full);
  }
  // ---- PFAM: prefetch the old iterate at this thread's fragment positions (overlaps the MMA)
  double zo[2][2][kNt][2];
  if (!PFPG) {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int li = i0 + wm * 32 + mt * 16 + g8 + 8 * h;
        const double* zrow = a.Out + (size_t)li * a.ldo + j0 + wn * kWn + 2 * t4;
#pragma unroll
        for (int nt = 0; nt < kNt; ++nt) {
          const int j = j0 + wn * kWn + nt * 8 + 2 * t4;
          if (fast) {
            const double2 z2 = __ldcs(reinterpret_cast<const double2*>(zrow + nt * 8));
            zo[mt][h][nt][0] = z2.x;
            zo[mt][h][nt][1] = z2.y;
            continue;
          }
          zo[mt][h][nt][0] = zo[mt][h][nt][1] = 0.0;
          if (li < a.n_rows && j < a.n) {
            const double* zp = zrow + nt * 8;
            if (j + 1 < a.n && ((reinterpret_cast<uintptr_t>(zp) & 15) == 0)) {
              const double2 z2 = __ldcs(reinterpret_cast<const double2*>(zp));
              zo[mt][h][nt][0] = z2.x;
              zo[mt][h][nt][1] = z2.y;
            } else {
              zo[mt][h][nt][0] = zp[0];
              if (j + 1 < a.n) zo[mt][h][nt][1] = zp[1];
            }
          }
        }
      }
  }
  // mask words of this thread's 4 rows (one 32-column word covers the warp's 16 columns),
  // loaded before the MMA so their latency overlaps it
  uint32_t wbits[2][2];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int li = i0 + wm * 32 + mt * 16 + g8 + 8 * h;
      wbits[mt][h] = (li < a.n_rows && a.bits)  // no mask (pf_rebuild): every bit 0
                         ? __ldg(a.bits + (size_t)li * a.ldb + ((j0 + wn * kWn) >> 5))
                                   : 0u;
    }
  cp_async_wait_all();
  __syncthreads();

  // ---- X tile = (V_I diag(f)) V_J^T on DMMA (fragment loads at constant offsets)
  double acc[2][kNt][4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < kNt; ++nt)
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[mt][nt][k] = 0.0;
  {
    const double* pa = Vi + (wm * 32 + g8) * C::LD + t4;
    const double* pb = Vj + (wn * kWn + g8) * C::LD + t4;
#pragma unroll
    for (int ks = 0; ks < P / 4; ++ks) {
      double a0[2], a1[2], b0[kNt];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        a0[mt] = pa[(mt * 16) * C::LD + ks * 4];
        a1[mt] = pa[(mt * 16 + 8) * C::LD + ks * 4];
      }
#pragma unroll
      for (int nt = 0; nt < kNt; ++nt) b0[nt] = pb[(nt * 8) * C::LD + ks * 4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < kNt; ++nt) dmma16884(acc[mt][nt], a0[mt], a1[mt], b0[nt]);
    }
  }
  double accm[PFPG ? 2 : 1][PFPG ? kNt : 1][4];
  if (PFPG) {
#pragma unroll
    for (int mt = 0; mt < (PFPG ? 2 : 1); ++mt)
#pragma unroll
      for (int nt = 0; nt < (PFPG ? kNt : 1); ++nt)
#pragma unroll
        for (int k = 0; k < 4; ++k) accm[mt][nt][k] = 0.0;
    for (int ks = 0; ks < a.rpad / 4; ++ks) {
      const int k = ks * 4 + t4;
      double a0[2], a1[2], b0[kNt];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        a0[mt] = Wi[(wm * 32 + mt * 16 + g8) * ldw_s + k];
        a1[mt] = Wi[(wm * 32 + mt * 16 + g8 + 8) * ldw_s + k];
      }
#pragma unroll
      for (int nt = 0; nt < kNt; ++nt) b0[nt] = Wj[(wn * kWn + nt * 8 + g8) * ldw_s + k];
#pragma unroll
      for (int mt = 0; mt < (PFPG ? 2 : 1); ++mt)
#pragma unroll
        for (int nt = 0; nt < (PFPG ? kNt : 1); ++nt)
          dmma16884(accm[mt][nt], a0[mt], a1[mt], b0[nt]);
    }
  }

  // ---- elementwise update + reductions
  if (fast) {
    // interior off-diagonal tile: no bounds / diagonal / alignment branches; the tile's sums are
    // accumulated unweighted and folded in once
    double ts0 = 0.0, ts1 = 0.0;
    const double qt = 0.25 * a.tt;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rt = wm * 32 + mt * 16 + g8 + 8 * h;
        const int li = i0 + rt;
        const uint32_t word = wbits[mt][h];
        double* rowp = a.Out + (size_t)li * a.ldo + j0;
#pragma unroll
        for (int nt = 0; nt < kNt; ++nt) {
          const int ct = wn * kWn + nt * 8 + 2 * t4;
          const bool b0 = (word >> (ct & 31)) & 1u, b1 = (word >> ((ct + 1) & 31)) & 1u;
          const double x0 = acc[mt][nt][2 * h], x1 = acc[mt][nt][2 * h + 1];
          double o0, o1;
          if (PFPG) {
            const double d0 = x0 - accm[PFPG ? mt : 0][PFPG ? nt : 0][2 * h];
            const double d1 = x1 - accm[PFPG ? mt : 0][PFPG ? nt : 0][2 * h + 1];
            o0 = b0 ? x0 - a.tt * d0 : x0;
            o1 = b1 ? x1 - a.tt * d1 : x1;
            ts0 += (b0 ? d0 * d0 : 0.0) + (b1 ? d1 * d1 : 0.0);
          } else {
            o0 = b0 ? x0 - qt : x0;                 // W_ij - t C_ij, C_ij = adj_ij / 4
            o1 = b1 ? x1 - qt : x1;
            ts0 += (b0 ? x0 : 0.0) + (b1 ? x1 : 0.0);
            const double e0 = o0 - zo[mt][h][nt][0], e1 = o1 - zo[mt][h][nt][1];
            ts1 = fma(e0, e0, fma(e1, e1, ts1));
            if (a.A8) *reinterpret_cast<double2*>(Tz + tz4(rt, ct)) = make_double2(o0, o1);
          }
          __stcs(reinterpret_cast<double2*>(rowp + ct), make_double2(o0, o1));
          if (mirror) {
            __stcs(a.Out + (size_t)(j0 + ct) * a.ldo + li, o0);
            __stcs(a.Out + (size_t)(j0 + ct + 1) * a.ldo + li, o1);
          }
        }
      }
    if (PFPG) {
      s0 += wgt * ts0;
    } else {
      s0 += wgt * 0.25 * ts0;
      s1 += wgt * ts1;
    }
  } else {
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int rt = wm * 32 + mt * 16 + g8 + 8 * h;  // row within tile
      const int li = i0 + rt;
      if (li >= a.n_rows) continue;
      const int gi = a.row0 + li;
      const uint32_t word = wbits[mt][h];
#pragma unroll
      for (int nt = 0; nt < kNt; ++nt) {
        const int ct = wn * kWn + nt * 8 + 2 * t4;  // column within tile
        const int j = j0 + ct;
        if (j >= a.n) continue;
        const bool two = (j + 1 < a.n);
        double o[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int jj = j + c;
          const bool bit = (c == 0 || two) ? ((word >> (jj & 31)) & 1u) : false;
          const double x = acc[mt][nt][2 * h + c];
          if (PFPG) {
            const double m = accm[PFPG ? mt : 0][PFPG ? nt : 0][2 * h + c];
            const double dxm = x - m;
            o[c] = bit ? x - a.tt * dxm : x;
            if (bit) s0 += wgt * dxm * dxm;
          } else {
            const double zold = zo[mt][h][nt][c];
            double znew;
            if (jj == gi) {
              znew = 1.0 - x + zold;               // Diag(1 - W_ii + Z_ii)
              s0 += -0.25 * a.deg[gi] * x;         // C_ii = -deg_i / 4
            } else {
              znew = bit ? x - 0.25 * a.tt : x;    // W_ij - t C_ij, C_ij = adj_ij / 4
              if (bit) s0 += wgt * 0.25 * x;
            }
            if (c == 0 || two) {
              const double dz = znew - zold;
              s1 += wgt * dz * dz;
            }
            o[c] = znew;
          }
        }
        if (!PFPG && a.A8)
          *reinterpret_cast<double2*>(Tz + tz4(rt, ct)) = make_double2(o[0], two ? o[1] : 0.0);
        double* op = a.Out + (size_t)li * a.ldo + j;
        if (two && ((reinterpret_cast<uintptr_t>(op) & 15) == 0)) {
          __stcs(reinterpret_cast<double2*>(op), make_double2(o[0], o[1]));
        } else {
          op[0] = o[0];
          if (two) op[1] = o[1];
        }
        if (mirror) {
          // (J, I) tile = transpose, stored straight from the fragment: for a fixed (nt, c)
          // the warp writes 4 rows x 8 consecutive doubles (full 32-byte sectors), no smem pass
          __stcs(a.Out + (size_t)j * a.ldo + li, o[0]);
          if (two) __stcs(a.Out + (size_t)(j + 1) * a.ldo + li, o[1]);
        }
      }
    }
  }

    pv_i0 = i0;  // digit slices of this tile: written after the next tile's barrier
    pv_j0 = j0;
    pv_mirror = mirror;
    pv_full = full;
  }  // tile loop
  if (!PFPG && a.A8 && pv_i0 >= 0) {
    __syncthreads();
    if (a.S == 7) rb_digits_any<7>(a, Tz, pv_i0, pv_j0, pv_mirror, tid, Eg, pv_full);
    else rb_digits_any<6>(a, Tz, pv_i0, pv_j0, pv_mirror, tid, Eg, pv_full);
  }

  // ---- deterministic reduction: block tree, then the last CTA sums CTA partials in order
  s0 = block_sum(s0, red);
  s1 = block_sum(s1, red);
  const int bid = blockIdx.y * gridDim.x + blockIdx.x;
  const int nb = gridDim.x * gridDim.y;
  if (tid == 0) {
    a.partials[2 * (size_t)bid] = s0;
    a.partials[2 * (size_t)bid + 1] = s1;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(a.counter, 1) == nb - 1);
  __syncthreads();
  if (s_last) {
    __threadfence();
    double t0 = 0.0, t1 = 0.0;
    for (int b = tid; b < nb; b += kRbThreads) {
      t0 += __ldcg(a.partials + 2 * (size_t)b);
      t1 += __ldcg(a.partials + 2 * (size_t)b + 1);
    }
    t0 = block_sum(t0, red);
    t1 = block_sum(t1, red);
    if (tid == 0) {
      if (PFPG) {
        double sf = 0.0;
        for (int c = 0; c < P; ++c) sf += fabs(a.f[c]);
        a.obj[0] = 0.5 * t0;
        a.obj[1] = sf;
      } else {
        a.obj[0] = t0;
        a.obj[1] = a.raw ? t1 : sqrt(t1);
      }
      *a.counter = 0;
    }
  }
}

int rebuild_blocks(int n_rows, int n) {
  return ((n + kRb - 1) / kRb) * ((n_rows + kRb - 1) / kRb);
}

template <int P, bool PFPG>
static cudaError_t rb_launch(RbArgs a, cudaStream_t st) {
  using C = RbCfg<P, PFPG>;
  a.rpad = PFPG ? ((a.r + 3) / 4) * 4 : 0;
  const int ldw_s = a.rpad + 4;
  const size_t panels = (size_t)2 * kRb * C::LD * 8 + (PFPG ? (size_t)2 * kRb * ldw_s * 8 : 0) +
                        ((!PFPG && a.A8) ? (size_t)(kRb / 4) * (kRb / 4) * kTzBlk * 8 : 0);
  const size_t stage = (size_t)kRb * C::LDS * 8;
  const size_t smem = std::max(panels, stage);
  static bool attr = false;
  if (!attr) {
    const size_t mx = std::max((size_t)2 * kRb * C::LD * 8 +
                                   (PFPG ? (size_t)2 * kRb * 68 * 8
                                         : (size_t)(kRb / 4) * (kRb / 4) * kTzBlk * 8), stage);
    cudaFuncSetAttribute(rebuild_kernel<P, PFPG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)mx);
    attr = true;
  }
  const int tr = (a.n_rows + kRb - 1) / kRb, tc = (a.n + kRb - 1) / kRb;
  a.sym = (a.row0 == 0 && a.n_rows == a.n) ? 1 : 0;
  a.T = tc;
  const long long ntiles = a.sym ? (long long)tc * (tc + 1) / 2 : (long long)tr * tc;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rebuild_kernel<P, PFPG>, kRbThreads,
                                                smem);
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  dim3 grid((unsigned)std::max<long long>(1, std::min<long long>(ntiles, (long long)std::max(per_sm, 1) * sms)));
  count_launch();
  rebuild_kernel<P, PFPG><<<grid, kRbThreads, smem, st>>>(a);
  return cudaGetLastError();
}

template <bool PFPG>
static cudaError_t rb_dispatch(int p, const RbArgs& a, cudaStream_t st) {
  switch (p) {
    case 16: return rb_launch<16, PFPG>(a, st);
    case 32: return rb_launch<32, PFPG>(a, st);
    case 64: return rb_launch<64, PFPG>(a, st);
    case 128: return rb_launch<128, PFPG>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

__global__ void scale_cols_kernel(const double* __restrict__ V, int64_t ldv,
                                  const double* __restrict__ f, int n_rows, int p,
                                  double* __restrict__ out) {
  // p is a multiple of 16: each thread scales 2 adjacent columns of one row (no 64-bit division)
  const int half = p >> 1;
  for (int i = blockIdx.x; i < n_rows; i += gridDim.x)
    for (int c2 = threadIdx.x; c2 < half; c2 += blockDim.x) {
      const int c = 2 * c2;
      const double2 v = *reinterpret_cast<const double2*>(V + (size_t)i * ldv + c);
      *reinterpret_cast<double2*>(out + (size_t)i * p + c) = make_double2(v.x * f[c], v.y * f[c + 1]);
    }
}

static cudaError_t scale_cols(const double* V, int64_t ldv, const double* f, int n_rows, int p,
                              double* out, cudaStream_t st) {
  count_launch();
  scale_cols_kernel<<<std::max(1, std::min(n_rows, 16 * 148)), std::max(32, p / 2), 0, st>>>(
      V, ldv, f, n_rows, p, out);
  return cudaGetLastError();
}

cudaError_t prox_launch(const double* V, int64_t ldv, const double* Vloc, int64_t ldvl,
                        const double* f, double tau, const uint32_t* omega, int64_t ldo,
                        const double* W, int64_t ldw, int r, double* Aout, int64_t lda,
                        int n_rows, int n, int row0, int p, double* obj, double* partials,
                        int* counter, double* vf, cudaStream_t st) {
  cudaError_t e = scale_cols(Vloc, ldvl, f, n_rows, p, vf, st);
  if (e != cudaSuccess) return e;
  RbArgs a{V, ldv, vf, f, tau, omega, ldo, W, ldw, r, 0,
           (r > 0 && (ldw & 1) == 0 && (reinterpret_cast<uintptr_t>(W) & 15) == 0) ? 1 : 0,
           nullptr, Aout, lda, n_rows, n, row0,
           0, 0, 0, partials, counter, obj, nullptr, 0, nullptr, 0, nullptr};
  return rb_dispatch<true>(p, a, st);
}

// Row bounds of Z_new = offdiag(W - tC) + Diag(1 - W_ii + Z_ii), W = V diag(f) V^T: with
// a_i = sum_k |f_k| V_ik^2, Cauchy-Schwarz gives |W_ij| <= sqrt(a_i a_j) <= sqrt(a_i) w_max
// (w_max = max_j sqrt(a_j)); |t C_ij| <= |t| / 4 off the diagonal, so
// max_j |Z_new_ij| <= B_i = max(sqrt(a_i) w_max + |t|/4, |1 - W_ii + Z_ii|).  Margins: the update's
// own W_ij is a DMMA sum, within p u a_i of these (p <= 512: relative 1e-12 on the off-diagonal
// term, absolute 1e-13 (a_i + 1 + |Z_ii|) on the diagonal one).  E_i = the digit-scale exponent
// of B_i: every |Z_new_ij| < 2^E_i, as the digit expansion requires.  The fused digits use the
// single exponent Eg = max_i E_i (one scale for the matrix: the mirror tile's digits are then the
// byte transpose of the tile's, DESIGN.md §4 "fused digits"); a row whose own bound is below
// 2^Eg loses Eg - E_i bits of the 49-bit expansion (measured spread on the config-3 iterates:
// <= 3 bits).
__global__ void pfam_bound1_kernel(const double* __restrict__ VF, const double* __restrict__ V,
                                   int64_t ldv, int n, int p, double2* __restrict__ wa,
                                   unsigned long long* wmax) {
  __shared__ unsigned long long bmax;
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (threadIdx.x == 0) bmax = 0ull;
  __syncthreads();
  if (i < n) {
    double s = 0.0, sa = 0.0;
    for (int k = lane; k < p; k += 32) {
      const double x = VF[(size_t)i * p + k] * V[(size_t)i * ldv + k];
      s += x;
      sa += fabs(x);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, o);
      sa += __shfl_xor_sync(0xffffffffu, sa, o);
    }
    if (lane == 0) {
      wa[i] = make_double2(s, sa);
      atomicMax(&bmax, (unsigned long long)__double_as_longlong(sqrt(sa)));
    }
  }
  __syncthreads();  // one global atomic per block instead of one per row
  if (threadIdx.x == 0 && bmax) atomicMax(wmax, bmax);
}

// matrix form W = Q F Q^T (pf_admm_step_f): |W_ij| <= ||F||_2 ||q_i|| ||q_j||, with ||F||_2 bounded
// by min(||F||_F, max row sum) (pfam_fnorm_kernel, stored as bits in wmax[1]); W_ii exactly
__global__ void pfam_fnorm_kernel(const double* __restrict__ F, int p, unsigned long long* out) {
  __shared__ double red[32];
  double f2 = 0.0, rmax = 0.0;
  for (int i = threadIdx.x; i < p; i += blockDim.x) {
    double r = 0.0;
    for (int k = 0; k < p; ++k) {
      const double v = F[(size_t)i * p + k];
      f2 += v * v;
      r += fabs(v);
    }
    rmax = fmax(rmax, r);
  }
  f2 = block_sum(f2, red);
  __syncthreads();
  for (int o = 16; o > 0; o >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = rmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    *out = (unsigned long long)__double_as_longlong(fmin(sqrt(f2), m) * (1.0 + 1e-12));
  }
}

__global__ void pfam_bound1f_kernel(const double* __restrict__ VF, const double* __restrict__ V,
                                    int64_t ldv, int n, int p, const unsigned long long* fn,
                                    double2* __restrict__ wa, unsigned long long* wmax) {
  __shared__ unsigned long long bmax;
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (threadIdx.x == 0) bmax = 0ull;
  __syncthreads();
  if (i < n) {
    const double nf = __longlong_as_double((long long)*fn);
    double s = 0.0, q2 = 0.0;
    for (int k = lane; k < p; k += 32) {
      const double v = V[(size_t)i * ldv + k];
      s += VF[(size_t)i * p + k] * v;
      q2 += v * v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, o);
      q2 += __shfl_xor_sync(0xffffffffu, q2, o);
    }
    if (lane == 0) {
      const double sa = nf * q2 * (1.0 + 1e-12);
      wa[i] = make_double2(s, sa);
      atomicMax(&bmax, (unsigned long long)__double_as_longlong(sqrt(sa)));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && bmax) atomicMax(wmax, bmax);
}

__global__ void pfam_bound2_kernel(const double2* __restrict__ wa,
                                   const unsigned long long* __restrict__ wmax,
                                   const double* __restrict__ Z, int64_t ldz, int n, double t,
                                   int* __restrict__ Eg) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  int e = INT_MIN;
  if (i < n) {
    const double wm = __longlong_as_double((long long)*wmax);
    const double2 w = wa[i];
    const double zii = Z[(size_t)i * ldz + i];
    const double off = (sqrt(w.y) * wm + 0.25 * fabs(t)) * (1.0 + 1e-12);
    const double dg = fabs(1.0 - w.x + zii) + 1e-13 * (w.y + 1.0 + fabs(zii));
    e = i8::scale_exp(fmax(off, dg));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) e = max(e, __shfl_xor_sync(0xffffffffu, e, o));
  if ((threadIdx.x & 31) == 0 && e != INT_MIN) atomicMax(Eg, e);
}

cudaError_t admm_launch(const double* V, int64_t ldv, const double* Vloc, int64_t ldvl,
                        const double* f, double t, const uint32_t* adj, int64_t ldadj,
                        const double* deg, double* Z, int64_t ldz, int n_rows, int n, int row0,
                        int p, double* obj, double* partials, int* counter, int raw, double* vf,
                        cudaStream_t st, const RbDigits* dig, const double* Fmat,
                        const R8Bufs* r8, int tma_sms) {
  cudaError_t e = cudaSuccess;
  if (!Fmat) {
    e = scale_cols(Vloc, ldvl, f, n_rows, p, vf, st);
    if (e != cudaSuccess) return e;
  }
  RbArgs a{V, ldv, vf, f, t, adj, ldadj, nullptr, 0, 0, 0, 0, deg, Z, ldz, n_rows, n, row0,
           0, 0, raw, partials, counter, obj, nullptr, 0, nullptr, 0, nullptr};
  if (dig && dig->A8 && row0 == 0 && n_rows == n) {
    e = cudaMemsetAsync(dig->wmax, 0, 8, st);
    if (e != cudaSuccess) return e;
    if (Fmat) {
      count_launch();
      pfam_fnorm_kernel<<<1, 128, 0, st>>>(Fmat, p, dig->wmax + 1);
      count_launch();
      pfam_bound1f_kernel<<<(n + 7) / 8, 256, 0, st>>>(vf, Vloc, ldvl, n, p, dig->wmax + 1,
                                                        dig->wa, dig->wmax);
    } else {
      count_launch();
      pfam_bound1_kernel<<<(n + 7) / 8, 256, 0, st>>>(vf, Vloc, ldvl, n, p, dig->wa, dig->wmax);
    }
    e = cudaMemsetAsync(dig->E, 0x80, sizeof(int), st);  // INT_MIN-ish start for atomicMax
    if (e != cudaSuccess) return e;
    count_launch();
    pfam_bound2_kernel<<<(n + 255) / 256, 256, 0, st>>>(dig->wa, dig->wmax, Z, ldz, n, t, dig->E);
    a.A8 = dig->A8;
    a.KB = dig->KB;
    a.E = dig->E;
    a.S = dig->S;
    a.rscale = dig->rscale;
    if (r8 && p == 64 && dig->S == 7 && r8_usable(Z, ldz))
      return admm_i8_launch(r8->maps, vf, V, ldv, r8->VF8, r8->V8, r8->rsA, r8->rsB, adj, ldadj,
                            deg, t, Z, ldz, n, obj, partials, counter, dig, r8->mirror_dig,
                            r8->mirror_z, r8->num_sms, st);
  } else if (tma_sms > 0 && p == 64 && row0 == 0 && n_rows == n && !raw &&
             td_usable(vf, V, ldv, Z, ldz)) {
    // one GPU, no digit output: the TMA-staged update with W on DMMA
    return admm_tma_launch(vf, V, ldv, adj, ldadj, deg, t, Z, ldz, n, obj, partials, counter,
                           tma_sms, st);
  }
  return rb_dispatch<false>(p, a, st);
}

__global__ void sqrt_inplace_kernel(double* x) { x[0] = sqrt(x[0]); }

__global__ void coef_acc_kernel(const double* c, double* d) {
  d[0] = c[0];
  d[1] = 1.0;
  d[2] = 0.0;
}

cudaError_t coef_acc_launch(const double* c, double* d, cudaStream_t st) {
  count_launch();
  coef_acc_kernel<<<1, 1, 0, st>>>(c, d);
  return cudaGetLastError();
}

cudaError_t sqrt_inplace_launch(double* x, cudaStream_t st) {
  count_launch();
  sqrt_inplace_kernel<<<1, 1, 0, st>>>(x);
  return cudaGetLastError();
}

}  // namespace pf

namespace pf {

// ============================================================================== NCE update
// Dual gradient step of nearest correlation estimation (eqn:NCE-dual,
// eqn:NCE-gradient): with Pi_+(G + Diag x) ~ V diag(f) V^T on the local rows,
//   d_i = sum_c f_c V_ic^2,  g_i = d_i - 1,  x_i <- x_i - tau g_i,  B_{i, row0 + i} = G_ii + x_i.
// Only the diagonal of the iterate changes, so the update is O(n p) -- the filter dominates even
// more than in PFPG / PFAM.  One warp per row (coalesced row of V); raw sums {sum x_old,
// sum g^2} reduced deterministically (per-CTA partials, last CTA sums in CTA order); the
// objective is finished by nce_finish_kernel after the (optional) cross-rank all-reduce.
constexpr int kNceThreads = 256;

__global__ void __launch_bounds__(kNceThreads) nce_kernel(
    const double* __restrict__ V, int64_t ldv, const double* __restrict__ f, int p, double tau,
    const double* __restrict__ gdiag, const double* x_in, double* x_out, double* __restrict__ B,
    int64_t ldb, int n_rows, int row0, double* partials, int* counter, double* obj) {
  __shared__ double red[32];
  __shared__ int s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpb = kNceThreads / 32;
  double sx = 0.0, sg = 0.0;
  for (int i = blockIdx.x * wpb + warp; i < n_rows; i += gridDim.x * wpb) {
    double d = 0.0;
    for (int c = lane; c < p; c += 32) {
      const double v = V[(size_t)i * ldv + c];
      d += f[c] * v * v;
    }
    d = warp_sum(d);
    if (lane == 0) {
      const double g = d - 1.0, xo = x_in[i], xn = xo - tau * g;
      x_out[i] = xn;
      B[(size_t)i * ldb + row0 + i] = gdiag[row0 + i] + xn;
      sx += xo;
      sg += g * g;
    }
  }
  sx = block_sum(sx, red);
  sg = block_sum(sg, red);
  if (threadIdx.x == 0) {
    partials[2 * (size_t)blockIdx.x] = sx;
    partials[2 * (size_t)blockIdx.x + 1] = sg;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(counter, 1) == (int)gridDim.x - 1);
  __syncthreads();
  if (s_last) {
    __threadfence();
    if (threadIdx.x == 0) {
      double tx = 0.0, tg = 0.0;
      for (int b = 0; b < (int)gridDim.x; ++b) {
        tx += __ldcg(partials + 2 * (size_t)b);
        tg += __ldcg(partials + 2 * (size_t)b + 1);
      }
      obj[0] = tx;  // raw: sum x_old (local rows)
      obj[1] = tg;  // raw: sum g^2
      *counter = 0;
    }
  }
}

// obj <- {1/2 sum f^2 - sum x_old, sqrt(sum g^2)}  (F(x_old), ||grad F(x_old)||)
__global__ void nce_finish_kernel(const double* f, int p, double* obj) {
  if (threadIdx.x != 0) return;
  double s = 0.0;
  for (int c = 0; c < p; ++c) s += f[c] * f[c];
  obj[0] = 0.5 * s - obj[0];
  obj[1] = sqrt(obj[1]);
}

cudaError_t nce_launch(const double* V, int64_t ldv, const double* f, int p, double tau,
                       const double* gdiag, const double* x_in, double* x_out, double* B,
                       int64_t ldb, int n_rows, int row0, double* partials, int* counter,
                       double* obj, cudaStream_t st) {
  const int blocks = std::max(1, std::min(256, (n_rows + 7) / 8));
  count_launch();
  nce_kernel<<<blocks, kNceThreads, 0, st>>>(V, ldv, f, p, tau, gdiag, x_in, x_out, B, ldb, n_rows,
                                             row0, partials, counter, obj);
  return cudaGetLastError();
}

// PFPG objective h = 1/2 ||P_Omega(X - M)||_F^2 + mu sum |f| (eq:pfpg1 P:338-341 with
// R = mu ||.||_*, whose value at X = V diag(f) V^T, V orthonormal, is mu sum_i |f_i|):
// obj {fit, sum |f|} -> {fit + mu sum |f|, fit}
__global__ void pfpg_obj_finish_kernel(double* obj, double mu) {
  if (threadIdx.x != 0) return;
  const double fit = obj[0];
  obj[0] = fit + mu * obj[1];
  obj[1] = fit;
}

cudaError_t pfpg_obj_finish_launch(double* obj, double mu, cudaStream_t st) {
  count_launch();
  pfpg_obj_finish_kernel<<<1, 32, 0, st>>>(obj, mu);
  return cudaGetLastError();
}

cudaError_t nce_finish_launch(const double* f, int p, double* obj, cudaStream_t st) {
  count_launch();
  nce_finish_kernel<<<1, 32, 0, st>>>(f, p, obj);
  return cudaGetLastError();
}

}  // namespace pf

namespace pf {

// ============================================================================== extrapolation
// Regularized extrapolation of the iterates (paper §4.3; NEXT-4): history
// h_0..h_L (L = l + 1 <= kRnaMax, oldest first), U = [h_1 - h_0, ..., h_L - h_{L-1}],
// M = U^T U (all-reduced over row blocks), c = (M + lam I)^{-1} 1 / (1^T (M + lam I)^{-1} 1) with
// lam = lam_rel ||M||_F (reading R21), x~ = sum_{i<L} c_i h_i.
constexpr int kRnaMax = 8;
struct RnaHist {
  const double* h[kRnaMax + 1];
};

__global__ void __launch_bounds__(256) rna_gram_kernel(RnaHist hs, int L, int n_rows,
                                                       double* partials, int* counter,
                                                       double* M) {
  __shared__ double red[32];
  __shared__ int s_last;
  double acc[kRnaMax * (kRnaMax + 1) / 2];
#pragma unroll
  for (int e = 0; e < kRnaMax * (kRnaMax + 1) / 2; ++e) acc[e] = 0.0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += gridDim.x * blockDim.x) {
    double u[kRnaMax];
#pragma unroll
    for (int i = 0; i < kRnaMax; ++i) u[i] = (i < L) ? hs.h[i + 1][r] - hs.h[i][r] : 0.0;
    int e = 0;
#pragma unroll
    for (int i = 0; i < kRnaMax; ++i)
#pragma unroll
      for (int j = i; j < kRnaMax; ++j) acc[e++] += u[i] * u[j];
  }
  const int ne = L * (L + 1) / 2;
  int e = 0;
  for (int i = 0; i < L; ++i)
    for (int j = i; j < L; ++j) {
      // packed index over kRnaMax for the accumulator, over L for the partials
      const int ek = i * kRnaMax - i * (i - 1) / 2 + (j - i);
      const double v = block_sum(acc[ek], red);
      if (threadIdx.x == 0) partials[(size_t)blockIdx.x * ne + e] = v;
      ++e;
    }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(counter, 1) == (int)gridDim.x - 1);
  __syncthreads();
  if (s_last) {
    __threadfence();
    if (threadIdx.x < ne) {
      double t = 0.0;
      for (int b = 0; b < (int)gridDim.x; ++b) t += __ldcg(partials + (size_t)b * ne + threadIdx.x);
      int i = 0, rem = threadIdx.x;
      while (rem >= L - i) {
        rem -= L - i;
        ++i;
      }
      const int j = i + rem;
      M[i * L + j] = t;
      M[j * L + i] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) *counter = 0;
  }
}

// every block solves the L x L system redundantly (L <= 8), then combines its rows
__global__ void __launch_bounds__(256) rna_combine_kernel(RnaHist hs, int L, int n_rows,
                                                          const double* M, double lam_rel,
                                                          const double* gdiag, double* x_out,
                                                          double* B, int64_t ldb, int row0,
                                                          double* coef) {
  __shared__ double c[kRnaMax];
  if (threadIdx.x == 0) {
    double a[kRnaMax][kRnaMax], z[kRnaMax];
    double fro = 0.0;
    for (int i = 0; i < L; ++i)
      for (int j = 0; j < L; ++j) fro += M[i * L + j] * M[i * L + j];
    double lam = lam_rel * sqrt(fro);
    if (lam == 0.0) lam = lam_rel;
    for (int i = 0; i < L; ++i) {
      for (int j = 0; j < L; ++j) a[i][j] = M[i * L + j] + (i == j ? lam : 0.0);
      z[i] = 1.0;
    }
    // Cholesky of the SPD regularised matrix, then two triangular solves
    for (int j = 0; j < L; ++j) {
      double d = a[j][j];
      for (int k = 0; k < j; ++k) d -= a[j][k] * a[j][k];
      d = sqrt(d);
      a[j][j] = d;
      for (int i = j + 1; i < L; ++i) {
        double v = a[i][j];
        for (int k = 0; k < j; ++k) v -= a[i][k] * a[j][k];
        a[i][j] = v / d;
      }
    }
    for (int i = 0; i < L; ++i) {
      double v = z[i];
      for (int k = 0; k < i; ++k) v -= a[i][k] * z[k];
      z[i] = v / a[i][i];
    }
    for (int i = L - 1; i >= 0; --i) {
      double v = z[i];
      for (int k = i + 1; k < L; ++k) v -= a[k][i] * z[k];
      z[i] = v / a[i][i];
    }
    double sz = 0.0;
    for (int i = 0; i < L; ++i) sz += z[i];
    for (int i = 0; i < L; ++i) c[i] = z[i] / sz;
    if (blockIdx.x == 0 && coef)
      for (int i = 0; i < L; ++i) coef[i] = c[i];
  }
  __syncthreads();
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += gridDim.x * blockDim.x) {
    double x = 0.0;
    for (int i = 0; i < L; ++i) x += c[i] * hs.h[i][r];
    x_out[r] = x;
    B[(size_t)r * ldb + row0 + r] = gdiag[row0 + r] + x;
  }
}

int rna_blocks(int n_rows) { return std::max(1, std::min(128, (n_rows + 255) / 256)); }

cudaError_t rna_gram_launch(const double* const* hist, int L, int n_rows, double* partials,
                            int* counter, double* M, cudaStream_t st) {
  if (L < 1 || L > kRnaMax) return cudaErrorInvalidValue;
  RnaHist hs{};
  for (int i = 0; i <= L; ++i) hs.h[i] = hist[i];
  count_launch();
  rna_gram_kernel<<<rna_blocks(n_rows), 256, 0, st>>>(hs, L, n_rows, partials, counter, M);
  return cudaGetLastError();
}

cudaError_t rna_combine_launch(const double* const* hist, int L, int n_rows, const double* M,
                               double lam_rel, const double* gdiag, double* x_out, double* B,
                               int64_t ldb, int row0, double* coef, cudaStream_t st) {
  RnaHist hs{};
  for (int i = 0; i <= L; ++i) hs.h[i] = hist[i];
  count_launch();
  rna_combine_kernel<<<rna_blocks(n_rows), 256, 0, st>>>(hs, L, n_rows, M, lam_rel, gdiag, x_out,
                                                         B, ldb, row0, coef);
  return cudaGetLastError();
}

}  // namespace pf
