// pf_kernels.cuh -- host-side launchers of the PF kernels (internal to libpf.so).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "pf_common.cuh"

namespace pf {

// process-wide count of kernels launched by libpf (defined in pf_api.cu)
void count_launch();

// ---- Chebyshev-step GEMM (pf_gemm.cu): out = s1*(A B) + s2*Ycur + s3*Yprev (rows of A local)
struct ChebGemmPlan {
  int p;
  int n_rows;         // rows of A (local block)
  int n_k;            // columns of A == rows of B
  int grid;           // stream-K CTAs
  int mtiles, kblocks;
  size_t ws_doubles;  // partial workspace size needed
};
ChebGemmPlan cheb_gemm_plan(int p, int n_rows, int n_k, int num_sms);
// Encode the TMA descriptors (host only, no device work).
bool encode_map_A(CUtensorMap* map, const double* A, int64_t lda, int n_rows, int n_k, int p);
bool encode_map_B(CUtensorMap* map, const double* B, int p, int n_k);
cudaError_t cheb_gemm_launch(const ChebGemmPlan& pl, const CUtensorMap& mapA,
                             const CUtensorMap& mapB, const double* ycur, const double* yprev,
                             double* out, const double* coef, double* ws, int* counters,
                             cudaStream_t st);

// ---- fp32-storage filter GEMM on tcgen05 TF32 tensor cores (pf_gemm_tf32.cu).  Blocks are
// p-major (transposed): element (i, c) of an n x p block at Y[c * ldy + i].
struct Tf32Plan {
  int p;
  int n_rows, n_k;
  int mtiles, kblocks;  // 256-row pair tiles, 16-wide k-blocks
  int pairs;            // launched CTA pairs
  int split;            // K-split of the leftover (tail) tiles
  size_t ws_floats;     // partial workspace
  size_t acc_floats;    // chunk accumulators
  int chunk_kb;         // k-blocks per TMEM accumulation chunk
  int pf_dist;          // L2 prefetch distance of A (k-blocks)
  size_t counters;      // tile counters (ints)
};
Tf32Plan tf32_plan(int p, int n_rows, int n_k, int num_sms);
// map: 16 x 128 SWIZZLE_64B load boxes; map_pf: 32 x 128 L2-prefetch boxes
bool tf32_encode_A(CUtensorMap* map, CUtensorMap* map_pf, const float* A, int64_t lda,
                   int n_rows, int n_k);
bool tf32_encode_B(CUtensorMap* map, const float* Yt, int64_t ldy, int p, int n_k);
// B as the rank-major all-gather [world][p][n_local] of p-major blocks (3-D map)
bool tf32_encode_B_dist(CUtensorMap* map, const float* Yg, int p, int n_local, int world);
cudaError_t tf32_gemm_launch(const Tf32Plan& pl, const CUtensorMap& mapA, const CUtensorMap& mapB,
                             const CUtensorMap& mapApf,
                             const float* ycur, const float* yprev, float* out, int64_t ldy,
                             const double* coef, float* ws, float* acc, int* counters,
                             int npass, cudaStream_t st, int bdist_kb = 0);

// ---- fp64 filter GEMM from exact int8 tensor-core products of S-digit splits (pf_gemm_i8.cu).
// A8: tiled int8 digit slices of A (pf_digits.cuh a8_offset; mtiles x kblocks x S blocks of
// 8 KB; row scales rscale), Y8: [S][p][kpad] K-major
// slices of the B block (column scales cscale).
struct I8Plan {
  int p, S, NC, ngroups;  // NC = columns per work item (<= 64), ngroups = p / NC
  int n_rows, n_k;
  int mtiles, kblocks;    // 128-row tiles, 64-byte k-blocks
  int64_t kpad;           // slice pitch (bytes), n_k rounded up to 16
  int chunk_kb;           // k-blocks per exact int32 accumulation
  int grid;               // persistent CTAs
  size_t acc_doubles;     // fold workspace
  int pf_dist;            // L2 prefetch distance of A (k-blocks, 0 = off)
  int pair;               // K1-i8p (CTA pairs, cta_group::2) for full-precision S = 7, NC = 64
  int pgrid, pmaxp;       // its CTAs (2 per cluster) and most clusters sharing a pair item
  int items;              // mtiles * ngroups
  int maxp;               // most CTAs sharing one item (stream-K)
  size_t part_doubles;    // stream-K partial workspace
};
I8Plan i8_plan(int p, int n_rows, int n_k, int slices, int num_sms);
bool i8_encode_A(CUtensorMap* map, CUtensorMap* map_pf, const int8_t* A8, const I8Plan& pl);
bool i8_encode_B(CUtensorMap* map, const int8_t* Y8, const I8Plan& pl, int su);  // box: su slices
bool i8_encode_B_pair(CUtensorMap* map64, CUtensorMap* map32, const int8_t* Y8, const I8Plan& pl);
cudaError_t i8_split_A_launch(const double* A, int64_t lda, const I8Plan& pl, int8_t* A8,
                              double* rscale, int num_sms, cudaStream_t st);
cudaError_t i8_split_Y_launch(const double* Y, int64_t ldy, const I8Plan& pl,
                              unsigned long long* cmax, int8_t* Y8, double* cscale, int num_sms,
                              cudaStream_t st);
bool i8s_supported(const I8Plan& pl, int num_sms);
bool i8s_encode_At(CUtensorMap* map, const int8_t* A8, const I8Plan& pl);
cudaError_t i8s_gemm_launch(const I8Plan& pl, const CUtensorMap& mapA8, const CUtensorMap& mapA8t,
                            const CUtensorMap& mapY8, const double* rscale, const double* cscale,
                            const double* ycur, const double* yprev, double* out, int64_t ldy,
                            const double* coef, cudaStream_t st);
cudaError_t i8_gemm_launch(const I8Plan& pl, const CUtensorMap& mapA8, const CUtensorMap& mapY8,
                           const CUtensorMap& mapA8pf, const double* rscale, const double* cscale, const double* ycur,
                           const double* yprev, double* out, int64_t ldy, const double* coef,
                           double* acc, double* part, int* counters, int su, cudaStream_t st,
                           const CUtensorMap* mapB64 = nullptr, const CUtensorMap* mapB32 = nullptr,
                           const CUtensorMap* mapA8t = nullptr);  // K1-i8p lower-transposed mode

// ---- Newton-Schulz spectral operator (pf_ns.cu): F = f(H) of a p x p symmetric fp64 matrix
struct NsWork;
NsWork* ns_create(int p);
void ns_destroy(NsWork* w);
// F = f(H) by Newton-Schulz sign iterations in one cooperative kernel (pf_ns.cu); on
// non-convergence the fail flag (ns_fail_flag) is set and F is left for the Jacobi fallback
cudaError_t ns_spectral(NsWork* w, const double* H, int op_soft, double thr, double* F, int* rank,
                        int* iters_dev, DevState* state, cudaStream_t st);
const int* ns_fail_flag(const NsWork* w);
// if *fail: f(theta), F = Y diag(f) Y^T, rank (Y, theta from a Jacobi solve)
cudaError_t ns_fallback_launch(const int* fail, int op_soft, double thr, const double* theta,
                               const double* Y, int p, double* F, int* rank, cudaStream_t st);

// ---- PFSVT sparse kernels (pf_svt.cu): S n x n in compressed-row form (CSR, or the CSC view)
cudaError_t svt_kick_launch(double* x, const double* b, double alpha, int64_t nnz,
                            cudaStream_t st);
cudaError_t spmm_launch(int rows, int p, const int* ptr, const int* idx, const double* val,
                        const int* vperm, const double* X, int64_t ldx, const double* coef,
                        const double* ycur, int64_t ldc, const double* yprev, int64_t ldp,
                        double* out, int64_t ldo, cudaStream_t st);
int svt_sample_blocks(int rows);
cudaError_t svt_sample_launch(int rows, int p, const int* ptr, const int* idx, const double* b,
                              double* x, const double* U, int64_t ldu, const double* V,
                              int64_t ldv, const double* s, double delta, double* partials,
                              int* counter, double* obj, cudaStream_t st);
cudaError_t svt_sigma_launch(const double* lam, int p, double mu, double* sigma, double* s,
                             double* inv, int* svp, cudaStream_t st);
cudaError_t scale_cols_inplace_launch(double* X, int64_t ldx, int rows, int p, const double* d,
                                      cudaStream_t st);

// ---- fp32-path kernels (pf_f32.cu); blocks fp32 p-major, p x p objects fp64 row-major
int gram32_slices(int n_rows, int p, int num_sms);
// G = X Y^T over the n_rows columns of the p-major blocks; partials: nslices * p * p doubles
cudaError_t gram32_launch(const float* X, int64_t ldx, const float* Y, int64_t ldy, int n_rows,
                          int p, double* G, double* partials, int nslices, const int* cond,
                          cudaStream_t st);
// out = in R (block view), in place allowed
cudaError_t rmul32_launch(const float* in, int64_t ldi, const double* R, float* out, int64_t ldo,
                          int n_rows, int p, const int* cond, cudaStream_t st);
// W: p*p doubles scratch, Dinv: p*32 doubles scratch
cudaError_t chol_inv_big_launch(const double* G, int p, int64_t n_global, double* W, double* Dinv,
                                double* Rinv, DevState* state, int* shift_flag_out,
                                const int* cond, cudaStream_t st);
int jacobi_big_grid();
// damped: device double[2] {a, b} (may be NULL): pairs whose two diagonal entries both lie in
// (a, b) are not rotated (their eigenpairs have f = 0)
cudaError_t jacobi_big_launch(const double* H, int p, double* theta, double* Y, double* Hw,
                              double* Vw, double* red_ws, int* cnt_ws, DevState* state, double tol,
                              int max_sweeps, const double* damped, cudaStream_t st,
                              const int* cond = nullptr);
cudaError_t perturb_hash32_launch(float* A, int64_t lda, int rows, int cols, int row0,
                                  unsigned long long seed, int k, double noise, cudaStream_t st);
// Lanczos GEMV on an fp32 iterate (fp64 accumulation), same contract as lz_gemv_launch
cudaError_t lz_gemv_f32_launch(const float* A, int64_t lda, int n_local, int n, const double* q,
                               const double* Q, int64_t ldq, int j, double* w, double* h,
                               double* partials, int* counter, DevState* state, cudaStream_t st);

// ---- small dense kernels (pf_small.cu); all p x p objects are row-major, ld = p
// G = X^T Y over rows [0, n_rows) (X, Y: n_rows x p, ld p).  Deterministic two-level sum:
// per-CTA partials then the last CTA reduces in CTA order.  If `cond` != NULL the kernel is a
// no-op unless *cond != 0.  Returns the grid used (<= max_blocks).
int gram_blocks(int n_rows, int p);
cudaError_t gram_launch(const double* X, const double* Y, int n_rows, int p, double* G,
                        double* partials, int* counter, const int* cond, cudaStream_t st);
// Cholesky G = L L^T (shifted on breakdown) and Rinv = L^{-T}; n_global for the shift.
// p <= 64: the same factorisation with the matrix in registers (one barrier per column)
cudaError_t chol_inv_reg_launch(const double* G, int p, int64_t n_global, double* Rinv,
                                DevState* state, int* shift_flag_out, const int* cond,
                                cudaStream_t st);
cudaError_t chol_inv_launch(const double* G, int p, int64_t n_global, double* Rinv,
                            DevState* state, int* shift_flag_out, const int* cond,
                            cudaStream_t st);
// out(n_rows x p, ldo) = in(n_rows x p, ldi) * R (p x p); in place allowed (in == out, ldi == ldo)
cudaError_t rmul_launch(const double* in, int64_t ldi, const double* R, double* out, int64_t ldo,
                        int n_rows, int p, const int* cond, cudaStream_t st);
// two-sided parallel cyclic Jacobi: H (p x p symmetric, only read) -> theta desc, Y (p x p)
cudaError_t jacobi_launch(const double* H, int p, const int* p_dev, double* theta, double* Y,
                          DevState* state, double tol, int max_sweeps, cudaStream_t st,
                          const int* cond = nullptr);
cudaError_t spectral_launch(int op, double thr, const double* theta, int p, double* f,
                            int* rank, DevState* state, cudaStream_t st);
// plan kernel: interval -> per-step coefficients + re-base flags
cudaError_t plan_launch(const double* interval, int d, double rho_max, int p, DevState* state,
                        cudaStream_t st);
cudaError_t interval_psd_launch(const double* lo_hi, double eta, double* interval,
                                DevState* state, cudaStream_t st);
cudaError_t interval_soft_launch(double thr, double eta, double* interval, DevState* state,
                                 cudaStream_t st);
cudaError_t interval_top_r_launch(const double* lo_hi, int r, double eta, double* interval,
                                  DevState* state, cudaStream_t st);
// theta -> state (re-base plan), relative gap and the eta_k estimate of the last filter (degree d,
// q repeats; d = 0: no filter since -> nan)
cudaError_t copy_theta_launch(const double* theta, int p, DevState* state, cudaStream_t st,
                              int d = 0, int q = 1);
// Lanczos (pf_lanczos.cu): vectors are local row blocks with pitch ldq; every phase leaves
// LOCAL sums that the host all-reduces between phases when the context is distributed.
int lanczos_blocks(int n_rows);
// norm_only: s[0] = |v0|^2 (local); else q0 = v0 / sqrt(s[0]) and the run is marked active
cudaError_t lz_start_launch(const double* v0, int n_local, double* s, double* q0,
                            DevState* state, cudaStream_t st, bool norm_only);
cudaError_t lz_gemv_launch(const double* A, int64_t lda, int n_local, int n, const double* q,
                           const double* Q, int64_t ldq, int j, double* w, double* h,
                           double* partials, int* counter, DevState* state, cudaStream_t st);
// symmetric Lanczos GEMV (fp64, one GPU, n <= 32 lanczos_blocks(n)): reads only the upper
// triangle of A; ws = lz_symv_ws_doubles(n) doubles of scratch
size_t lz_symv_ws_doubles(int n);
cudaError_t lz_symv_launch(const double* A, int64_t lda, int n, const double* q, const double* Q,
                           int64_t ldq, int j, double* w, double* h, double* ws,
                           double* partials, int* counter, DevState* state, int num_sms,
                           cudaStream_t st);
cudaError_t lz_orth_launch(int n_local, const double* Q, int64_t ldq, int j, double* w,
                           const double* h, double* out, double* partials, int* counter,
                           DevState* state, int phase, cudaStream_t st);
cudaError_t lz_next_launch(int n_local, double* Q, int64_t ldq, int j, const double* w,
                           const double* s, DevState* state, cudaStream_t st);
cudaError_t lz_ritz_vector_launch(const double* Q, int64_t ldq, int n_local, const double* S,
                                  const DevState* state, double* v, cudaStream_t st);
cudaError_t lanczos_finish_launch(int m, double* T, double* theta, double* S, double* lo_hi,
                                  DevState* state, cudaStream_t st);
cudaError_t perturb_launch(double* A, int64_t lda, const double* E, int64_t lde, int rows,
                           int cols, cudaStream_t st);

// ---- rebuild + update (pf_rebuild.cu)
int rebuild_blocks(int n_rows, int n);
// V: all n rows (ldv); Vloc: this rank's rows (ldvl); vf: scratch n_local x p for V diag(f)
cudaError_t prox_launch(const double* V, int64_t ldv, const double* Vloc, int64_t ldvl,
                        const double* f, double tau, const uint32_t* omega, int64_t ldo,
                        const double* W, int64_t ldw, int r, double* Aout, int64_t lda,
                        int n_rows, int n, int row0, int p, double* obj, double* partials,
                        int* counter, double* vf, cudaStream_t st);
cudaError_t pfpg_obj_finish_launch(double* obj, double mu, cudaStream_t st);
// PF_FP64_I8 on one GPU: the PFAM update also writes the digit slices of Z_new (pf_gemm_i8.cu
// tiled layout, a8_offset) and their row scales, so the next filter skips its split pass
struct RbDigits {
  int8_t* A8;
  int KB;                   // k-blocks of the tiled layout
  int S;
  int* E;                   // [n] row exponents
  double* rscale;           // [n] 2^E
  double2* wa;              // [n] scratch (W_ii, sum_k |f_k| V_ik^2)
  unsigned long long* wmax; // scratch (wmax[1]: ||F|| bound of the matrix form)
};
// PF_FP64_I8, one GPU, p = 64, fused digits: W = V' V^T from int8 digit products on tcgen05
// (pf_rebuild_i8.cu) -- digit buffers of V' and V (r8_bytes each), their row scales, TMA maps
struct R8Bufs {
  const CUtensorMap* maps;  // [4]: V' digits, V digits, Z_new digit tile / mirror boxes (r8_encode)
  int8_t* VF8;
  int8_t* V8;
  double* rsA;
  double* rsB;
  int num_sms;
  int mirror_dig;           // 0: upper-tile digits only (the half-storage product reads no others)
  int mirror_z;             // 0: Z_new on and above the 128 x 128 diagonal blocks only
};
size_t r8_bytes(int n);
bool r8_encode(CUtensorMap* maps, const int8_t* VF8, const int8_t* V8, const int8_t* A8, int n,
               int KB);
bool r8_usable(const double* Z, int64_t ldz);  // TMA on Z: even pitch, 16-byte aligned base
// PF_FP64, one GPU, p = 64: the TMA-staged PFAM update with W on DMMA (pf_rebuild_i8.cu)
bool td_usable(const double* VF, const double* V, int64_t ldv, const double* Z, int64_t ldz);
cudaError_t admm_tma_launch(const double* VF, const double* V, int64_t ldv, const uint32_t* adj,
                            int64_t ldadj, const double* deg, double t, double* Z, int64_t ldz,
                            int n, double* obj, double* partials, int* counter, int num_sms,
                            cudaStream_t st);
cudaError_t admm_i8_launch(const CUtensorMap* maps, const double* VF, const double* V,
                           int64_t ldv, int8_t* VF8, int8_t* V8, double* rsA, double* rsB,
                           const uint32_t* adj, int64_t ldadj, const double* deg, double t,
                           double* Z, int64_t ldz, int n, double* obj, double* partials,
                           int* counter, const RbDigits* dig, int mirror_dig, int mirror_z,
                           int num_sms, cudaStream_t st);
cudaError_t admm_launch(const double* V, int64_t ldv, const double* Vloc, int64_t ldvl,
                        const double* f, double t, const uint32_t* adj, int64_t ldadj,
                        const double* deg, double* Z, int64_t ldz, int n_rows, int n, int row0,
                        int p, double* obj, double* partials, int* counter, int raw, double* vf,
                        cudaStream_t st, const RbDigits* dig = nullptr,
                        const double* Fmat = nullptr, const R8Bufs* r8 = nullptr,
                        int tma_sms = 0);
// (tma_sms > 0: a one-GPU update without digit output may use the TMA-staged kernel with W on
//  DMMA on that many SMs, pf_rebuild_i8.cu)
// (Fmat != NULL: W = V F V^T with F p x p row-major; vf must already hold the local rows of V F
//  and f is unused)
cudaError_t sqrt_inplace_launch(double* x, cudaStream_t st);
// d = {c[0], 1, 0}: the coefficients that ADD s1 (A_g Y_g) to an output in place (slab GEMMs)
cudaError_t coef_acc_launch(const double* c, double* d, cudaStream_t st);
// NCE dual gradient update (NEXT-1): partials >= 2 * 256 doubles; obj gets raw sums
cudaError_t nce_launch(const double* V, int64_t ldv, const double* f, int p, double tau,
                       const double* gdiag, const double* x_in, double* x_out, double* B,
                       int64_t ldb, int n_rows, int row0, double* partials, int* counter,
                       double* obj, cudaStream_t st);
// regularized extrapolation (NEXT-4): L = l + 1 <= 8 differences; partials >= 128 * 36 doubles
int rna_blocks(int n_rows);
cudaError_t rna_gram_launch(const double* const* hist, int L, int n_rows, double* partials,
                            int* counter, double* M, cudaStream_t st);
cudaError_t rna_combine_launch(const double* const* hist, int L, int n_rows, const double* M,
                               double lam_rel, const double* gdiag, double* x_out, double* B,
                               int64_t ldb, int row0, double* coef, cudaStream_t st);
cudaError_t nce_finish_launch(const double* f, int p, double* obj, cudaStream_t st);

}  // namespace pf
