// pf_api.cu -- the C ABI (include/pf.h): context / scratch management and the orchestration of
// the hot-path kernels for one PFPG / PFAM iteration.  All work is stream-ordered; nothing here
// synchronises the host except pf_get_device_status / pf_profile_read / pf_diagnostics.
//
// Distributed contexts (pf_create_dist: NCCL; pf_create_loop: in-process loopback on one GPU,
// pf_comm.cuh) own a communicator: rank g holds the row block
// [g n / world, (g + 1) n / world) of A and of every n x p block.  Each Chebyshev step
// all-gathers Y_j (the B operand), every Gram / H matrix is all-reduced (p x p), the Lanczos
// vector is all-gathered per step and its dots / norms all-reduced, and the rebuild gathers V.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/pf.h"
#include "pf_comm.cuh"
#include "pf_kernels.cuh"

using namespace pf;

static std::atomic<long long> g_launches{0};
void pf::count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

struct pf_ctx_s {
  int64_t n = 0, n_local = 0, row0 = 0;
  int p = 0, d = 0, d0 = 0, rank = 0, world = 1, num_sms = 148;  // d0: degree at create
  pf_dtype dtype = PF_FP64;
  bool dist = false;                           // communicator present (NCCL or loopback)
  DevState* state = nullptr;
  double* Y[3] = {nullptr, nullptr, nullptr};  // n_local x p, ld p
  double* Yfull = nullptr;                     // n x p gathered block (dist)
  double* Wbuf = nullptr;                      // n_local x p (A Q)
  double* VFbuf = nullptr;                     // n_local x p (V diag(f) for the rebuild)
  double* Vfull = nullptr;                     // n x p (dist)
  double* G = nullptr;                         // p x p
  double* Rinv = nullptr;
  double* Yeig = nullptr;
  double* gram_part = nullptr;
  double* cheb_ws = nullptr;
  int* cheb_cnt = nullptr;
  double* lz_Q = nullptr;                      // (kMaxLanczos + 1) local vectors, pitch lz_ldq
  int64_t lz_ldq = 0;
  double* lz_qfull = nullptr;                  // n (dist)
  double* lz_w = nullptr;
  double* lz_h = nullptr;                      // h1[kMaxLanczos], h2[kMaxLanczos], s[8]
  double* lz_part = nullptr;
  int* lz_cnt = nullptr;
  double* lz_sym_ws = nullptr;                 // symmetric-GEMV tile partials (fp64, one GPU)
  double* lz_T = nullptr;
  double* lz_theta = nullptr;
  double* lz_S = nullptr;
  double* lz_v0 = nullptr;                     // bottom Ritz vector of the last refresh (n_local)
  bool lz_have_v0 = false;
  double* rb_part = nullptr;
  double* rb_obj = nullptr;                    // [2] objective scratch of pf_rebuild
  int* rb_cnt = nullptr;
  int* shift_flag = nullptr;
  ChebGemmPlan plan;
  CUtensorMap mapB[3];
  CUtensorMap mapBfull;
  const double* mapA_ptr = nullptr;
  int64_t mapA_lda = 0;
  CUtensorMap mapA;
  Comm* comm = nullptr;
  // profiling of the dominant kernel: event pairs around every Chebyshev-step GEMM launch
  bool prof = false;
  std::vector<cudaEvent_t> ev;
  size_t ev_used = 0;
  std::vector<cudaEvent_t> evu;               // ... and around every PFAM update (pf_admm_step*)
  size_t evu_used = 0;
  long long prof_dropped = 0;
  // ---- fp32 storage / TF32 tensor-core path (dtype PF_TF32): p-major fp32 blocks
  int64_t ldy32 = 0;                           // pitch of the internal blocks (>= n_local, %4)
  float* Yf[3] = {nullptr, nullptr, nullptr};  // p x ldy32
  float* Wf = nullptr;                         // A Q
  float* Yfull32 = nullptr;                    // dist: rank-major all-gather [world][p][n_local]
  CUtensorMap mapBfull32;
  double* g32_part = nullptr;
  int g32_slices = 1;
  double* chol_W = nullptr;                    // p x p
  double* chol_D = nullptr;                    // p x 32
  double* jac_H = nullptr;                     // 2 p x p
  double* jac_V = nullptr;                     // p x p
  double* jac_red = nullptr;
  int* jac_cnt = nullptr;
  double* jac_theta = nullptr;                 // p (Newton-Schulz fallback)
  float* tf_ws = nullptr;
  float* tf_acc = nullptr;
  int* tf_cnt = nullptr;
  int tf_early = 3;  // TF32 passes of the Chebyshev steps before the exact tail
  int tf_tail = 0;   // number of final Chebyshev steps run in 3xTF32
  int tf_rr = 3;     // passes of the Rayleigh-Ritz product A Q
  bool filtered = false;  // a pf_filter ran: state->interval holds its damped interval
  int last_d = 0, last_q = 1;  // degree and repeats of the last pf_filter (eta_k diagnostic)
  Tf32Plan tplan;
  CUtensorMap mapBf[3];
  CUtensorMap mapAf, mapApf;
  // overlapped all-gather (TF32, world > 1): the GEMM runs slab by slab
  // (K range of rank g's rows) as each peer slab lands, on SMs left free for the transfers
  bool overlap = false;
  int comm_sms = 16;                           // SMs not used by the slab GEMMs (NCCL kernels)
  cudaStream_t comm_st = nullptr;
  cudaEvent_t ev_start = nullptr, ev_comm_done = nullptr;
  std::vector<cudaEvent_t> ev_slab;
  Tf32Plan tplan_s;                            // one slab: n_local x n_local
  std::vector<CUtensorMap> mapA_s, mapApf_s, mapB_s;
  double* coef_acc = nullptr;                  // {s1, 1, 0} of the current step
  std::vector<cudaEvent_t> ev_tl;              // timeline of the last overlapped step (pf_profile)
  bool tl_valid = false;
  const float* mapAf_ptr = nullptr;
  int64_t mapAf_lda = 0;
  // ---- fp64 via exact int8 tensor-core products (dtype PF_FP64_I8, pf_gemm_i8.cu)
  bool i8 = false;
  I8Plan i8plan;                               // S = 0: this context runs the DMMA GEMM
  int8_t* A8 = nullptr;                        // tiled digit slices (pf_digits.cuh a8_offset)
  double* a8_rscale = nullptr;                 // [n_local]
  int8_t* Y8 = nullptr;                        // [kI8MaxSlices][p][kpad]
  double* y8_cscale = nullptr;                 // [p]
  unsigned long long* y8_cmax = nullptr;       // [p]
  double* i8_acc = nullptr;
  double* i8_part = nullptr;                   // stream-K partials
  int* i8_cnt = nullptr;                       // [items], self-resetting
  CUtensorMap mapA8, mapA8pf;
  // half-storage symmetric product (K1-i8s, pf_gemm_i8.cu) on fused digits: the stored tiles
  // (I, J >= I) only; PF_I8SYM=1 at create turns it on
  bool i8s_ok = false;
  bool i8t_ok = false;                         // K1-i8p reads upper-tile digits (lower transposed)
  CUtensorMap mapA8t;                          // 64-row boxes read transposed
  bool a8_half = false;                        // A8 holds the upper tiles only (no mirror digits)
  CUtensorMap mapY8[4];                        // B boxes of 4..7 digit slices
  CUtensorMap mapY8p[2];                       // K1-i8p B boxes (64 / 32 rows of one slice)
  int i8_early = 7;                            // slices of the Chebyshev steps before the tail
  int i8_tail = 0;                             // final steps (and RR) at the full slice count
  // PF_FUSE_DIGITS=0: the PFAM update does not write digits (pf_filter splits Z itself)
  bool fuse_digits = [] {
    const char* e = getenv("PF_FUSE_DIGITS");
    return !(e && e[0] == '0');
  }();
  const double* a8_src = nullptr;              // A whose digit slices A8 holds (pf_filter)
  int64_t a8_lda = 0;
  bool a8_valid = false;                       // cleared by every libpf call that writes A
  bool a8_fused = false;                       // A8 written by pf_admm_step's update (no split)
  int* a8_E = nullptr;                         // [n_local] row exponents of the fused digits
  double2* a8_wa = nullptr;                    // [n_local] row-bound scratch
  unsigned long long* a8_wmax = nullptr;
  // PFAM update on int8 tensor cores (pf_rebuild_i8.cu; one GPU, p = 64, fused digits)
  bool r8_on = false;
  bool z_upper = false;                        // pf_set_z_upper: the update skips the fp64 mirror
  const void* z_upper_src = nullptr;           // the iterate last written upper-only
  bool k7tma = true;                           // PF_K7TMA=0 at create: rebuild_kernel on PF_FP64
  int8_t* r8_VF8 = nullptr;                    // digit slices of V' (r8_bytes)
  int8_t* r8_V8 = nullptr;                     // digit slices of V
  double* r8_rs = nullptr;                     // [2 x n padded to 128] row scales of V', V
  CUtensorMap r8_maps[4];
  NsWork* ns = nullptr;                        // pf_rr_ns workspace (created on first use)
  // ---- PFSVT (pf_svt.cu)
  double* svt_part = nullptr;                  // residual partials (one per 8 rows)
  int* svt_cnt = nullptr;
  char err[512] = {0};
};

static constexpr int kI8MaxSlices = 7;
static constexpr int kMaxWorld = 64;  // row-block ranks (the loopback hub allows 16)

static pf_status cuda_fail(pf_ctx c, cudaError_t e, const char* where) {
  if (c) snprintf(c->err, sizeof(c->err), "%s: %s", where, cudaGetErrorString(e));
  return PF_ERR_CUDA;
}
#define PF_CU(call)                                          \
  do {                                                       \
    cudaError_t e_ = (call);                                 \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call); \
  } while (0)
#define PF_TRY(call)                 \
  do {                               \
    pf_status s_ = (call);           \
    if (s_ != PF_OK) return s_;      \
  } while (0)

static bool p_supported(int p, pf_dtype dt) {
  if (dt == PF_TF32) return p == 64 || p == 128 || p == 256 || p == 512;
  // PF_FP64 and PF_FP64_I8
  return p == 16 || p == 32 || p == 64 || p == 128;
}
static bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; }

extern "C" {

const char* pf_status_string(pf_status s) {
  switch (s) {
    case PF_OK: return "PF_OK";
    case PF_ERR_ARG: return "PF_ERR_ARG";
    case PF_ERR_DIM: return "PF_ERR_DIM";
    case PF_ERR_INTERVAL: return "PF_ERR_INTERVAL";
    case PF_ERR_CUDA: return "PF_ERR_CUDA";
    case PF_ERR_NOMEM: return "PF_ERR_NOMEM";
    case PF_ERR_NCCL: return "PF_ERR_NCCL";
    case PF_ERR_UNSUPPORTED: return "PF_ERR_UNSUPPORTED";
    case PF_ERR_BREAKDOWN: return "PF_ERR_BREAKDOWN";
  }
  return "PF_ERR_UNKNOWN";
}

const char* pf_last_error(pf_ctx c) { return c ? c->err : "null context"; }
int64_t pf_local_rows(pf_ctx c) { return c ? c->n_local : -1; }
int64_t pf_row0(pf_ctx c) { return c ? c->row0 : -1; }

pf_status pf_nccl_unique_id(void* out, int32_t bytes) {
  if (!out || bytes < (int32_t)sizeof(ncclUniqueId)) return PF_ERR_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return PF_ERR_NCCL;
  memcpy(out, &id, sizeof(id));
  return PF_OK;
}

static bool encode_i8_maps(pf_ctx ctx) {
  if (!i8_encode_A(&ctx->mapA8, &ctx->mapA8pf, ctx->A8, ctx->i8plan)) return false;
  if ((ctx->i8s_ok || ctx->i8t_ok) && !i8s_encode_At(&ctx->mapA8t, ctx->A8, ctx->i8plan))
    return false;
  for (int su = 4; su <= ctx->i8plan.S; ++su)
    if (!i8_encode_B(&ctx->mapY8[su - 4], ctx->Y8, ctx->i8plan, su)) return false;
  if (ctx->i8plan.pair && !i8_encode_B_pair(&ctx->mapY8p[0], &ctx->mapY8p[1], ctx->Y8, ctx->i8plan))
    return false;
  return true;
}

static pf_status alloc_all(pf_ctx ctx) {
  const int64_t n = ctx->n, nl = ctx->n_local;
  const int p = ctx->p;
  auto A = [&](void** ptr, size_t bytes) -> bool {
    return cudaMalloc(ptr, std::max<size_t>(bytes, 16)) == cudaSuccess;
  };
  bool ok = true;
  const bool f32 = ctx->dtype == PF_TF32;
  ok &= A((void**)&ctx->state, sizeof(DevState));
  if (f32) {
    // distributed: n_local % 16 == 0, so the blocks are contiguous p x n_local slabs that
    // ncclAllGather concatenates rank-major; the B operand is then read through a 3-D map
    ctx->ldy32 = ctx->dist ? nl : (nl + 3) / 4 * 4;
    if (ctx->dist) ok &= A((void**)&ctx->Yfull32, (size_t)p * n * 4);
    for (int i = 0; i < 3; ++i) ok &= A((void**)&ctx->Yf[i], (size_t)p * ctx->ldy32 * 4);
    ok &= A((void**)&ctx->Wf, (size_t)p * ctx->ldy32 * 4);
    ctx->g32_slices = gram32_slices((int)nl, p, ctx->num_sms);
    ok &= A((void**)&ctx->g32_part, (size_t)ctx->g32_slices * p * p * 8);
    ok &= A((void**)&ctx->chol_W, (size_t)p * p * 8);
    ok &= A((void**)&ctx->chol_D, (size_t)p * 32 * 8);
    ok &= A((void**)&ctx->tf_ws, ctx->tplan.ws_floats * 4);
    ok &= A((void**)&ctx->tf_acc, ctx->tplan.acc_floats * 4);
    ok &= A((void**)&ctx->tf_cnt, ctx->tplan.counters * 4);
  } else {
    // panel Cholesky scratch (chol_inv_big, used for p >= 64 on the fp64 path too)
    ok &= A((void**)&ctx->chol_W, (size_t)p * p * 8);
    ok &= A((void**)&ctx->chol_D, (size_t)p * 32 * 8);
    for (int i = 0; i < 3; ++i) ok &= A((void**)&ctx->Y[i], (size_t)nl * p * 8);
    ok &= A((void**)&ctx->Wbuf, (size_t)nl * p * 8);
    ok &= A((void**)&ctx->VFbuf, (size_t)nl * p * 8);
  }
  if (ctx->i8) {
    const I8Plan& ip = ctx->i8plan;
    // tiled digit slices: (128-row tiles) x (64-byte k-blocks) x S blocks of 8 KB
    ok &= A((void**)&ctx->A8, (size_t)ip.mtiles * ip.kblocks * kI8MaxSlices * 8192);
    ok &= A((void**)&ctx->a8_rscale, (size_t)nl * 8);
    ok &= A((void**)&ctx->a8_E, (size_t)nl * 4);
    ok &= A((void**)&ctx->a8_wa, (size_t)nl * 16);
    ok &= A((void**)&ctx->a8_wmax, 16);
    if (!ctx->dist && p == 64 && ip.S == 7) {
      const char* e = getenv("PF_K7I8");  // 0: the DMMA update kernel (measurement)
      ctx->r8_on = !(e && e[0] == '0');
    }
    if (ctx->r8_on) {
      ok &= A((void**)&ctx->r8_VF8, r8_bytes((int)n));
      ok &= A((void**)&ctx->r8_V8, r8_bytes((int)n));
      ok &= A((void**)&ctx->r8_rs, (size_t)2 * ip.mtiles * 128 * 8);
      ok = ok && r8_encode(ctx->r8_maps, ctx->r8_VF8, ctx->r8_V8, ctx->A8, (int)n, ip.kblocks);
    }
    ok &= A((void**)&ctx->Y8, (size_t)kI8MaxSlices * p * ip.kpad);
    ok &= A((void**)&ctx->y8_cscale, (size_t)p * 8);
    ok &= A((void**)&ctx->y8_cmax, (size_t)(2 * p + 1) * 8);  // two halves + selector
    ok &= A((void**)&ctx->i8_acc, ip.acc_doubles * 8);
    // sized for the largest plan of any slice count (the split does not depend on S)
    ok &= A((void**)&ctx->i8_part, ip.part_doubles * 8);
    ok &= A((void**)&ctx->i8_cnt, (size_t)ip.items * 4);
  }
  if (ctx->dist) {
    ok &= A((void**)&ctx->Yfull, (size_t)n * p * 8);
    ok &= A((void**)&ctx->Vfull, (size_t)n * p * 8);
    ok &= A((void**)&ctx->lz_qfull, (size_t)n * 8);
  }
  ok &= A((void**)&ctx->G, (size_t)p * p * 8);
  // cooperative Jacobi scratch (TF32 Rayleigh-Ritz; the Newton-Schulz fallback on every dtype)
  ok &= A((void**)&ctx->jac_H, (size_t)2 * p * p * 8);
  ok &= A((void**)&ctx->jac_V, (size_t)p * p * 8);
  ok &= A((void**)&ctx->jac_red, (size_t)2 * jacobi_big_grid() * 8);
  ok &= A((void**)&ctx->jac_cnt, 16);
  ok &= A((void**)&ctx->jac_theta, (size_t)p * 8);
  ok &= A((void**)&ctx->Rinv, (size_t)p * p * 8);
  ok &= A((void**)&ctx->Yeig, (size_t)p * p * 8);
  if (!f32) {
    ok &= A((void**)&ctx->gram_part, (size_t)gram_blocks((int)nl, p) * p * p * 8);
    ok &= A((void**)&ctx->cheb_ws, ctx->plan.ws_doubles * 8);
    ok &= A((void**)&ctx->cheb_cnt, (size_t)(ctx->plan.mtiles + 1) * 4);
  }
  ctx->lz_ldq = ((nl + 31) / 32) * 32;
  ok &= A((void**)&ctx->lz_Q, (size_t)ctx->lz_ldq * (kMaxLanczos + 1) * 8);
  ok &= A((void**)&ctx->lz_w, (size_t)nl * 8);
  ok &= A((void**)&ctx->lz_h, (size_t)(2 * kMaxLanczos + 8) * 8);
  ok &= A((void**)&ctx->lz_part, (size_t)lanczos_blocks((int)nl) * kMaxLanczos * 8);
  ok &= A((void**)&ctx->lz_cnt, 16);
  // PF_LZ_SYM=0: the Lanczos GEMV reads all of A (else only its upper triangle, fp64 one GPU)
  {
    const char* e = getenv("PF_LZ_SYM");
    const bool sym_ok = !(e && e[0] == '0') && !ctx->dist && !f32 &&
                        n <= 32LL * lanczos_blocks((int)n);
    if (sym_ok) ok &= A((void**)&ctx->lz_sym_ws, lz_symv_ws_doubles((int)n) * 8);
  }
  ok &= A((void**)&ctx->lz_T, (size_t)kMaxLanczos * kMaxLanczos * 8);
  ok &= A((void**)&ctx->lz_theta, (size_t)kMaxLanczos * 8);
  ok &= A((void**)&ctx->lz_S, (size_t)kMaxLanczos * kMaxLanczos * 8);
  ok &= A((void**)&ctx->lz_v0, (size_t)nl * 8);
  // shared by the rebuild (2 per tile CTA), NCE (2 x 256) and extrapolation (128 x 36) reductions
  ok &= A((void**)&ctx->rb_part,
          std::max<size_t>((size_t)rebuild_blocks((int)nl, (int)n) * 2, 128 * 36) * 8);
  ok &= A((void**)&ctx->rb_cnt, 16);
  ok &= A((void**)&ctx->rb_obj, 16);
  if (!f32) {
    ok &= A((void**)&ctx->svt_part, (size_t)svt_sample_blocks((int)nl) * 8);
    ok &= A((void**)&ctx->svt_cnt, 16);
  }
  ok &= A((void**)&ctx->shift_flag, 16);
  if (!ok) {
    snprintf(ctx->err, sizeof(ctx->err), "cudaMalloc of scratch failed");
    return PF_ERR_NOMEM;
  }
  PF_CU(cudaMemset(ctx->state, 0, sizeof(DevState)));
  if (f32) PF_CU(cudaMemset(ctx->tf_cnt, 0, ctx->tplan.counters * 4));
  else PF_CU(cudaMemset(ctx->cheb_cnt, 0, (size_t)(ctx->plan.mtiles + 1) * 4));
  PF_CU(cudaMemset(ctx->lz_cnt, 0, 16));
  PF_CU(cudaMemset(ctx->rb_cnt, 0, 16));
  if (!f32) PF_CU(cudaMemset(ctx->svt_cnt, 0, 16));
  PF_CU(cudaMemset(ctx->shift_flag, 0, 16));
  const double rr[3] = {1.0, 0.0, 0.0};
  PF_CU(cudaMemcpy(&ctx->state->coef_rr[0], rr, sizeof(rr), cudaMemcpyHostToDevice));
  // TMA descriptors of the internal B operands
  if (f32 && ctx->dist) {
    if (!tf32_encode_B_dist(&ctx->mapBfull32, ctx->Yfull32, p, (int)nl, ctx->world)) {
      snprintf(ctx->err, sizeof(ctx->err), "cuTensorMapEncodeTiled(B, fp32, 3-D) failed");
      return PF_ERR_CUDA;
    }
  } else if (f32) {
    for (int i = 0; i < 3; ++i)
      if (!tf32_encode_B(&ctx->mapBf[i], ctx->Yf[i], ctx->ldy32, p, (int)n)) {
        snprintf(ctx->err, sizeof(ctx->err), "cuTensorMapEncodeTiled(B, fp32) failed");
        return PF_ERR_CUDA;
      }
  } else if (!ctx->dist) {
    for (int i = 0; i < 3; ++i)
      if (!encode_map_B(&ctx->mapB[i], ctx->Y[i], p, (int)n)) {
        snprintf(ctx->err, sizeof(ctx->err), "cuTensorMapEncodeTiled(B) failed");
        return PF_ERR_CUDA;
      }
  } else if (!encode_map_B(&ctx->mapBfull, ctx->Yfull, p, (int)n)) {
    snprintf(ctx->err, sizeof(ctx->err), "cuTensorMapEncodeTiled(B) failed");
    return PF_ERR_CUDA;
  }
  if (ctx->i8) PF_CU(cudaMemset(ctx->i8_cnt, 0, (size_t)ctx->i8plan.items * 4));
  if (ctx->i8) PF_CU(cudaMemset(ctx->y8_cmax, 0, (size_t)(2 * ctx->p + 1) * 8));
  if (ctx->i8 && !encode_i8_maps(ctx)) {
    snprintf(ctx->err, sizeof(ctx->err), "cuTensorMapEncodeTiled(int8 slices) failed");
    return PF_ERR_CUDA;
  }
  PF_CU(cudaDeviceSynchronize());
  return PF_OK;
}

static pf_status setup_overlap(pf_ctx ctx) {
  const int W = ctx->world, nl = (int)ctx->n_local, p = ctx->p;
  PF_CU(cudaStreamCreateWithFlags(&ctx->comm_st, cudaStreamNonBlocking));
  PF_CU(cudaEventCreateWithFlags(&ctx->ev_start, cudaEventDisableTiming));
  PF_CU(cudaEventCreateWithFlags(&ctx->ev_comm_done, cudaEventDisableTiming));
  ctx->ev_slab.assign(W, nullptr);
  for (auto& e : ctx->ev_slab) PF_CU(cudaEventCreate(&e));  // timed: pf_overlap_timeline
  PF_CU(cudaMalloc(&ctx->coef_acc, 4 * sizeof(double)));
  ctx->tplan_s = tf32_plan(p, nl, nl, std::max(2, ctx->num_sms - ctx->comm_sms));
  ctx->mapA_s.resize(W);
  ctx->mapApf_s.resize(W);
  ctx->mapB_s.resize(W);
  for (int g = 0; g < W; ++g)
    if (!tf32_encode_B(&ctx->mapB_s[g], ctx->Yfull32 + (size_t)g * p * nl, nl, p, nl)) {
      snprintf(ctx->err, sizeof(ctx->err), "cuTensorMapEncodeTiled(B slab, fp32) failed");
      return PF_ERR_CUDA;
    }
  return PF_OK;
}

static pf_status create_common(int64_t n, int32_t p, int32_t degree, pf_dtype dtype, int rank,
                               int world, const void* nccl_id, LoopHub* hub, pf_ctx* out) {
  if (!out) return PF_ERR_ARG;
  *out = nullptr;
  if (world > kMaxWorld) return PF_ERR_ARG;
  if (dtype != PF_FP64 && dtype != PF_TF32 && dtype != PF_FP64_I8) return PF_ERR_UNSUPPORTED;
  // fp32 path, distributed: equal row blocks with n_local % 16 == 0 (a 16-wide TMA K box never
  // straddles two ranks' slabs of the gathered block)
  const bool dist = nccl_id != nullptr || hub != nullptr;
  if (dtype == PF_TF32 && dist && (n % (16 * (int64_t)world)) != 0)
    return PF_ERR_DIM;
  if (degree < 1 || degree > kMaxDeg) return PF_ERR_ARG;
  if (world < 1 || rank < 0 || rank >= world) return PF_ERR_ARG;
  if (!p_supported(p, dtype) || n < p || n > (int64_t)1 << 30 || n < world * (int64_t)p)
    return PF_ERR_DIM;
  pf_ctx ctx = new (std::nothrow) pf_ctx_s();
  if (!ctx) return PF_ERR_NOMEM;
  ctx->n = n;
  ctx->p = p;
  ctx->d = ctx->d0 = degree;
  ctx->dtype = dtype;
  ctx->rank = rank;
  ctx->world = world;
  ctx->dist = dist;
  ctx->row0 = (int64_t)rank * n / world;
  ctx->n_local = (int64_t)(rank + 1) * n / world - ctx->row0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess)
    e = cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) {
    pf_status s = cuda_fail(ctx, e, "cudaGetDevice");
    delete ctx;
    return s;
  }
  if (dtype == PF_TF32) ctx->tplan = tf32_plan(p, (int)ctx->n_local, (int)n, ctx->num_sms);
  else ctx->plan = cheb_gemm_plan(p, (int)ctx->n_local, (int)n, ctx->num_sms);
  if (dtype == PF_FP64_I8) {
    ctx->i8 = true;
    ctx->i8plan = i8_plan(p, (int)ctx->n_local, (int)n, 7, ctx->num_sms);  // S = 7
    // the half-storage product is opt-in (PF_I8SYM=1): it halves the A-digit reads but runs on
    // one CTA per 128-row tile (128 of 148 SMs at n = 16384) and measured slower
    const char* e8 = getenv("PF_I8SYM");
    ctx->i8s_ok = !dist && (e8 && e8[0] == '1') && i8s_supported(ctx->i8plan, ctx->num_sms);
    // K1-i8p on upper-tile digits (PF_I8T=0: the update writes every mirror digit tile)
    const char* et = getenv("PF_I8T");
    ctx->i8t_ok = !dist && !ctx->i8s_ok && !(et && et[0] == '0') && ctx->i8plan.pair;
  }
  {
    const char* e = getenv("PF_K7TMA");
    ctx->k7tma = !(e && e[0] == '0');
  }
  pf_status s = alloc_all(ctx);
  if (s == PF_OK && ctx->dist) {
    int cs = PF_OK;
    // largest all-reduce: a p x p Gram / H, the Lanczos coefficients, the extrapolation Gram
    const size_t max_reduce = std::max<size_t>((size_t)p * p, 2 * kMaxLanczos + 8);
    ctx->comm = hub ? comm_loop_create(hub, rank, max_reduce, ctx->err, &cs)
                    : comm_nccl_create(nccl_id, rank, world, ctx->err, &cs);
    s = (pf_status)cs;
  }
  if (s == PF_OK && ctx->dist && dtype == PF_TF32 && world > 1) {
    const char* e = getenv("PF_OVERLAP");  // 0: one all-gather, then one GEMM (measurement)
    ctx->overlap = !(e && e[0] == '0');
    if (const char* c = getenv("PF_COMM_SMS")) ctx->comm_sms = std::max(0, atoi(c));
  }
  if (s == PF_OK && ctx->overlap) s = setup_overlap(ctx);
  if (s != PF_OK) {
    fprintf(stderr, "pf_create: %s\n", ctx->err);
    pf_destroy(ctx);
    return s;
  }
  *out = ctx;
  return PF_OK;
}

pf_status pf_create(int64_t n, int32_t p, int32_t degree, pf_dtype dtype, pf_ctx* out) {
  return create_common(n, p, degree, dtype, 0, 1, nullptr, nullptr, out);
}

pf_status pf_create_dist(int64_t n, int32_t p, int32_t degree, pf_dtype dtype,
                         const void* nccl_id, int32_t rank, int32_t world, pf_ctx* out) {
  if (!nccl_id) return PF_ERR_ARG;
  return create_common(n, p, degree, dtype, rank, world, nccl_id, nullptr, out);
}

pf_status pf_loop_create(int32_t world, pf_loop* out) {
  if (!out) return PF_ERR_ARG;
  *out = reinterpret_cast<pf_loop>(loop_hub_create(world));
  return *out ? PF_OK : PF_ERR_ARG;
}

pf_status pf_loop_destroy(pf_loop hub) {
  if (!hub) return PF_ERR_ARG;
  loop_hub_destroy(reinterpret_cast<LoopHub*>(hub));
  return PF_OK;
}

pf_status pf_create_loop(int64_t n, int32_t p, int32_t degree, pf_dtype dtype, pf_loop hub,
                         int32_t rank, pf_ctx* out) {
  if (!hub) return PF_ERR_ARG;
  LoopHub* h = reinterpret_cast<LoopHub*>(hub);
  return create_common(n, p, degree, dtype, rank, loop_hub_world(h), nullptr, h, out);
}

long long pf_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

pf_status pf_diagnostics(pf_ctx ctx, pf_stream stream, double* diag) {
  if (!ctx || !diag) return PF_ERR_ARG;
  PF_CU(cudaStreamSynchronize((cudaStream_t)stream));
  DevState h;
  PF_CU(cudaMemcpy(&h, ctx->state, sizeof(DevState), cudaMemcpyDeviceToHost));
  diag[0] = h.scratch[1];
  diag[1] = (double)h.lanczos_steps;
  diag[2] = h.scratch[2];
  diag[3] = h.scratch[4];
  return PF_OK;
}

pf_status pf_profile(pf_ctx ctx, int32_t enable) {
  if (!ctx) return PF_ERR_ARG;
  if (enable && ctx->ev.empty()) {
    ctx->ev.resize(8192);
    for (auto& e : ctx->ev) PF_CU(cudaEventCreate(&e));
    ctx->evu.resize(1024);
    for (auto& e : ctx->evu) PF_CU(cudaEventCreate(&e));
  }
  ctx->prof = enable != 0;
  ctx->ev_used = 0;
  ctx->evu_used = 0;
  ctx->prof_dropped = 0;
  return PF_OK;
}

pf_status pf_profile_read_update(pf_ctx ctx, pf_stream stream, double* ms_out, int64_t* launches) {
  if (!ctx || !ms_out || !launches) return PF_ERR_ARG;
  PF_CU(cudaStreamSynchronize((cudaStream_t)stream));
  double tot = 0.0;
  for (size_t i = 0; i + 1 < ctx->evu_used; i += 2) {
    float ms = 0.f;
    PF_CU(cudaEventElapsedTime(&ms, ctx->evu[i], ctx->evu[i + 1]));
    tot += ms;
  }
  *ms_out = tot;
  *launches = (int64_t)(ctx->evu_used / 2);
  ctx->evu_used = 0;
  return PF_OK;
}

pf_status pf_profile_read(pf_ctx ctx, pf_stream stream, double* gemm_ms, int64_t* gemm_launches) {
  if (!ctx || !gemm_ms || !gemm_launches) return PF_ERR_ARG;
  PF_CU(cudaStreamSynchronize((cudaStream_t)stream));
  double tot = 0.0;
  for (size_t i = 0; i + 1 < ctx->ev_used; i += 2) {
    float ms = 0.f;
    PF_CU(cudaEventElapsedTime(&ms, ctx->ev[i], ctx->ev[i + 1]));
    tot += ms;
  }
  *gemm_ms = tot;
  *gemm_launches = (int64_t)(ctx->ev_used / 2);
  ctx->ev_used = 0;
  return ctx->prof_dropped ? PF_ERR_ARG : PF_OK;
}

pf_status pf_overlap_timeline(pf_ctx ctx, pf_stream stream, double* ms, int32_t cap,
                              int32_t* count) {
  if (!ctx || !ms || !count) return PF_ERR_ARG;
  *count = 0;
  if (!ctx->overlap || !ctx->tl_valid) return PF_OK;
  const int W = ctx->world;
  if (cap < 3 * W) return PF_ERR_DIM;
  PF_CU(cudaStreamSynchronize((cudaStream_t)stream));
  PF_CU(cudaStreamSynchronize(ctx->comm_st));
  // ms[s]: arrival of the s-th slab in consumption order (g = rank - s); ms[W + s] / ms[2W + s]:
  // begin / end of its GEMM; all relative to the step start
  for (int i = 0; i < 3 * W; ++i) {
    float t = 0.f;
    cudaEvent_t e = i < W ? ctx->ev_slab[(ctx->rank - i + W) % W] : ctx->ev_tl[1 + i];
    PF_CU(cudaEventElapsedTime(&t, ctx->ev_tl[0], e));
    ms[i] = t;
  }
  *count = 3 * W;
  return PF_OK;
}

pf_status pf_destroy(pf_ctx ctx) {
  if (!ctx) return PF_ERR_ARG;
  ns_destroy(ctx->ns);
  for (auto e : ctx->ev) cudaEventDestroy(e);
  for (auto e : ctx->evu) cudaEventDestroy(e);
  delete ctx->comm;
  if (ctx->comm_st) cudaStreamDestroy(ctx->comm_st);
  if (ctx->ev_start) cudaEventDestroy(ctx->ev_start);
  if (ctx->ev_comm_done) cudaEventDestroy(ctx->ev_comm_done);
  for (auto e : ctx->ev_slab)
    if (e) cudaEventDestroy(e);
  if (ctx->coef_acc) cudaFree(ctx->coef_acc);
  for (auto e : ctx->ev_tl)
    if (e) cudaEventDestroy(e);
  void* ptrs[] = {ctx->state,  ctx->Y[0],     ctx->Y[1],      ctx->Y[2],    ctx->Yfull,
                  ctx->Wbuf,   ctx->VFbuf,    ctx->Vfull,    ctx->G,         ctx->Rinv,    ctx->Yeig,
                  ctx->gram_part, ctx->cheb_ws, ctx->cheb_cnt, ctx->lz_Q,   ctx->lz_qfull,
                  ctx->lz_w,   ctx->lz_h,     ctx->lz_part,   ctx->lz_cnt,  ctx->lz_T,
                  ctx->lz_theta, ctx->lz_S,   ctx->rb_part,   ctx->rb_cnt,  ctx->shift_flag,
                  ctx->Yf[0],  ctx->Yf[1],    ctx->Yf[2],     ctx->Wf,      ctx->g32_part,
                  ctx->chol_W, ctx->chol_D,   ctx->jac_H,     ctx->jac_V,   ctx->jac_red,
                  ctx->jac_cnt, ctx->tf_ws,   ctx->tf_cnt,    ctx->tf_acc,  ctx->Yfull32,
                  ctx->A8,     ctx->a8_rscale, ctx->Y8,       ctx->y8_cscale, ctx->y8_cmax,
                  ctx->i8_acc, ctx->i8_part, ctx->i8_cnt, ctx->svt_part, ctx->svt_cnt,
                  ctx->lz_sym_ws, ctx->a8_E, ctx->a8_wa, ctx->a8_wmax, ctx->jac_theta,
                  ctx->lz_v0, ctx->rb_obj, ctx->r8_VF8, ctx->r8_V8, ctx->r8_rs};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  delete ctx;
  return PF_OK;
}

pf_status pf_get_device_status(pf_ctx ctx, pf_stream stream, uint32_t* flags, int32_t* rebases,
                               double* lanczos_lo_hi) {
  if (!ctx) return PF_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  PF_CU(cudaStreamSynchronize(st));
  DevState h;
  PF_CU(cudaMemcpy(&h, ctx->state, sizeof(DevState), cudaMemcpyDeviceToHost));
  if (flags) *flags = h.flags;
  if (rebases) *rebases = h.rebases;
  if (lanczos_lo_hi) {
    lanczos_lo_hi[0] = h.lanczos[0];
    lanczos_lo_hi[1] = h.lanczos[1];
  }
  // cleared on the caller's stream (ordered before the next libpf kernel on it)
  PF_CU(cudaMemsetAsync(&ctx->state->flags, 0, sizeof(unsigned int), st));
  PF_CU(cudaMemsetAsync(&ctx->state->rebases, 0, sizeof(int), st));
  return PF_OK;
}

// ------------------------------------------------------------------------------ internals
static pf_status check_A(pf_ctx ctx, const double* A, int64_t lda) {
  if (!A) return PF_ERR_ARG;
  if (lda < ctx->n || (lda & 1) || !aligned16(A)) return PF_ERR_DIM;
  return PF_OK;
}

static pf_status map_A(pf_ctx ctx, const double* A, int64_t lda) {
  if (A != ctx->mapA_ptr || lda != ctx->mapA_lda) {
    if (!encode_map_A(&ctx->mapA, A, lda, (int)ctx->n_local, (int)ctx->n, ctx->p)) {
      snprintf(ctx->err, sizeof(ctx->err), "cuTensorMapEncodeTiled(A) failed");
      return PF_ERR_CUDA;
    }
    ctx->mapA_ptr = A;
    ctx->mapA_lda = lda;
  }
  return PF_OK;
}

// Gather the local row block `loc` (n_local x cols doubles, contiguous) into `full` (n x cols).
static pf_status gather(pf_ctx ctx, const double* loc, double* full, int cols, cudaStream_t st) {
  size_t off[kMaxWorld + 1];
  for (int g = 0; g <= ctx->world; ++g)
    off[g] = (size_t)((int64_t)g * ctx->n / ctx->world) * cols * sizeof(double);
  return (pf_status)ctx->comm->allgatherv(loc, full, off, st);
}

static pf_status allreduce(pf_ctx ctx, double* buf, size_t count, cudaStream_t st) {
  if (!ctx->dist) return PF_OK;
  return (pf_status)ctx->comm->allreduce_sum(buf, count, st);
}

// One Chebyshev step / plain product: out = coef * (A B) + ..., B = Y[bidx] (all rows).
static bool use_i8(pf_ctx ctx) { return ctx->i8 && ctx->i8plan.S > 0; }

// PF_FP64_I8: digit slices of A for the products that follow (pf_gemm_i8.cu).  pf_filter always
// re-splits (A may have changed since the last iteration); pf_rayleigh_ritz / pf_matmul reuse
// the slices when they were made from the same A and no libpf call wrote an iterate since.
static pf_status split_A(pf_ctx ctx, const double* A, int64_t lda, bool reuse, cudaStream_t st) {
  if (!use_i8(ctx)) return PF_OK;
  if (reuse && ctx->a8_valid && ctx->a8_src == A && ctx->a8_lda == lda) return PF_OK;
  if (ctx->z_upper_src == A) {  // its blocks below the diagonal were not written (pf_set_z_upper)
    snprintf(ctx->err, sizeof(ctx->err),
             "iterate stored upper-only by pf_admm_step: a fresh digit split needs the full matrix");
    return PF_ERR_UNSUPPORTED;
  }
  PF_CU(i8_split_A_launch(A, lda, ctx->i8plan, ctx->A8, ctx->a8_rscale, ctx->num_sms, st));
  ctx->a8_fused = ctx->a8_half = false;
  ctx->a8_src = A;
  ctx->a8_lda = lda;
  ctx->a8_valid = true;
  return PF_OK;
}
static void iterate_written(pf_ctx ctx) { ctx->a8_valid = ctx->a8_fused = ctx->a8_half = false; }

static bool is_fp64(pf_ctx ctx) { return ctx->dtype == PF_FP64 || ctx->dtype == PF_FP64_I8; }

static pf_status gemm_step(pf_ctx ctx, int bidx, const double* ycur, const double* yprev,
                           double* out, const double* coef, cudaStream_t st, int su = 0) {
  const CUtensorMap* mb;
  const double* bsrc;
  if (!ctx->dist) {
    mb = &ctx->mapB[bidx];
    bsrc = ctx->Y[bidx];
  } else {
    PF_TRY(gather(ctx, ctx->Y[bidx], ctx->Yfull, ctx->p, st));
    mb = &ctx->mapBfull;
    bsrc = ctx->Yfull;
  }
  if (use_i8(ctx))
    PF_CU(i8_split_Y_launch(bsrc, ctx->p, ctx->i8plan, ctx->y8_cmax, ctx->Y8, ctx->y8_cscale,
                            ctx->num_sms, st));
  const bool rec = ctx->prof && ctx->ev_used + 2 <= ctx->ev.size();
  if (ctx->prof && !rec) ++ctx->prof_dropped;
  if (rec) PF_CU(cudaEventRecord(ctx->ev[ctx->ev_used], st));
  if (use_i8(ctx)) {
    const int S = ctx->i8plan.S;
    su = (su <= 0 || su > S) ? S : su;
    // fused digits of a symmetric iterate (one scale): the half-storage product
    const bool sym = ctx->i8s_ok && ctx->a8_fused && su == S && S == 7;
    // upper-tile digits (the update skipped the mirror tiles): K1-i8p reads the lower part
    // transposed
    const bool lowt = ctx->i8t_ok && ctx->a8_half && su == S && S == 7 && ctx->i8plan.pair;
    if (ctx->a8_half && !sym && !lowt) {
      snprintf(ctx->err, sizeof(ctx->err), "upper-tile digits need the full slice count");
      return PF_ERR_UNSUPPORTED;
    }
    if (sym)
      PF_CU(i8s_gemm_launch(ctx->i8plan, ctx->mapA8, ctx->mapA8t, ctx->mapY8[su - 4],
                            ctx->a8_rscale, ctx->y8_cscale, ycur, yprev, out, ctx->p, coef, st));
    else
      PF_CU(i8_gemm_launch(ctx->i8plan, ctx->mapA8, ctx->mapY8[su - 4], ctx->mapA8pf,
                           ctx->a8_rscale, ctx->y8_cscale, ycur, yprev, out, ctx->p, coef,
                           ctx->i8_acc, ctx->i8_part, ctx->i8_cnt, su, st, &ctx->mapY8p[0],
                           &ctx->mapY8p[1], lowt ? &ctx->mapA8t : nullptr));
  }
  else
    PF_CU(cheb_gemm_launch(ctx->plan, ctx->mapA, *mb, ycur, yprev, out, coef, ctx->cheb_ws,
                           ctx->cheb_cnt, st));
  if (rec) {
    PF_CU(cudaEventRecord(ctx->ev[ctx->ev_used + 1], st));
    ctx->ev_used += 2;
  }
  return PF_OK;
}

// G = X^T Y summed over all ranks
static pf_status gram_all(pf_ctx ctx, const double* X, const double* Y, double* G, const int* cond,
                          cudaStream_t st) {
  PF_CU(gram_launch(X, Y, (int)ctx->n_local, ctx->p, G, ctx->gram_part, nullptr, cond, st));
  return allreduce(ctx, G, (size_t)ctx->p * ctx->p, st);
}

// G = R^T R and Rinv = R^{-1} of the p x p Gram: p = 64 the register-blocked kernel (56 vs ~75 us
// per factorisation, PF_CHOL_REG=0 to disable); p >= 128 the 32-column panel kernel of the fp32
// path (tools/bench_orth.py: CholeskyQR2 626 vs 853 us at p = 128); p <= 32 (or PF_CHOL_BIG=0)
// the single-CTA column kernel
static cudaError_t chol64(pf_ctx ctx, int* shift_out, const int* cond, cudaStream_t st) {
  static int big = -1, reg = -1;
  if (big < 0) {
    const char* e = getenv("PF_CHOL_BIG");
    big = e ? atoi(e) : 1;
    const char* r = getenv("PF_CHOL_REG");  // p = 64: register-blocked kernel (default)
    reg = r ? atoi(r) : 1;
  }
  // p <= 32 stays on chol_inv (no gain measured: configs 1 / 2 within noise or slower)
  if (reg && ctx->p > 32 && ctx->p <= 64)
    return chol_inv_reg_launch(ctx->G, ctx->p, ctx->n, ctx->Rinv, ctx->state, shift_out, cond,
                               st);
  if (big && ctx->p >= 64)
    return chol_inv_big_launch(ctx->G, ctx->p, ctx->n, ctx->chol_W, ctx->chol_D, ctx->Rinv,
                               ctx->state, shift_out, cond, st);
  return chol_inv_launch(ctx->G, ctx->p, ctx->n, ctx->Rinv, ctx->state, shift_out, cond, st);
}

// One CholeskyQR pass on Y (in place); cond: only if *cond != 0.
static pf_status chol_pass(pf_ctx ctx, double* Y, int* shift_out, const int* cond,
                           cudaStream_t st) {
  PF_TRY(gram_all(ctx, Y, Y, ctx->G, cond, st));
  PF_CU(chol64(ctx, shift_out, cond, st));
  PF_CU(rmul_launch(Y, ctx->p, ctx->Rinv, Y, ctx->p, (int)ctx->n_local, ctx->p, cond, st));
  return PF_OK;
}

// CholeskyQR2, plus a third pass when either pass had to shift (shifted CholeskyQR3).
static pf_status orth_internal(pf_ctx ctx, double* Y, cudaStream_t st) {
  PF_CU(cudaMemsetAsync(ctx->shift_flag, 0, sizeof(int), st));
  PF_TRY(chol_pass(ctx, Y, ctx->shift_flag, nullptr, st));
  PF_TRY(chol_pass(ctx, Y, ctx->shift_flag, nullptr, st));
  return chol_pass(ctx, Y, nullptr, ctx->shift_flag, st);
}


// ------------------------------------------------------------------------------ fp32 internals
static pf_status check_A32(pf_ctx ctx, const float* A, int64_t lda) {
  if (!A) return PF_ERR_ARG;
  if (lda < ctx->n || (lda & 3) || !aligned16(A)) return PF_ERR_DIM;
  return PF_OK;
}

static pf_status map_A32(pf_ctx ctx, const float* A, int64_t lda) {
  if (A != ctx->mapAf_ptr || lda != ctx->mapAf_lda) {
    if (!tf32_encode_A(&ctx->mapAf, &ctx->mapApf, A, lda, (int)ctx->n_local, (int)ctx->n)) {
      snprintf(ctx->err, sizeof(ctx->err), "cuTensorMapEncodeTiled(A, fp32) failed");
      return PF_ERR_CUDA;
    }
    const int nl = (int)ctx->n_local;
    for (int g = 0; ctx->overlap && g < ctx->world; ++g)  // columns of rank g's rows
      if (!tf32_encode_A(&ctx->mapA_s[g], &ctx->mapApf_s[g], A + (size_t)g * nl, lda, nl, nl)) {
        snprintf(ctx->err, sizeof(ctx->err), "cuTensorMapEncodeTiled(A slab, fp32) failed");
        return PF_ERR_CUDA;
      }
    ctx->mapAf_ptr = A;
    ctx->mapAf_lda = lda;
  }
  return PF_OK;
}

// user p-major block (pitch ld) <-> internal block (pitch ldy32)
static pf_status copy_block32(pf_ctx ctx, float* dst, int64_t ldd, const float* src, int64_t lds,
                              cudaStream_t st) {
  PF_CU(cudaMemcpy2DAsync(dst, ldd * 4, src, lds * 4, (size_t)ctx->n_local * 4, ctx->p,
                          cudaMemcpyDeviceToDevice, st));
  return PF_OK;
}

// Overlapped step (the gather of Y_j "must overlap" the GEMM): the communication
// stream gathers the slabs one by one (Comm::allgather_slabs: own slab, then rank - 1, rank - 2,
// ...), and the compute stream runs the product slab by slab in that order, each launch waiting
// only for its own slab: the first writes s1 (A_g Y_g) + s2 Ycur + s3 Yprev, the others add
// s1 (A_g Y_g) in place.  The slab GEMMs use num_sms - comm_sms SMs, so the NCCL kernels of the
// next slabs run beside them.
static pf_status gemm_step32_overlap(pf_ctx ctx, int bidx, const float* ycur, const float* yprev,
                                     float* out, const double* coef, int npass, cudaStream_t st) {
  const int W = ctx->world, nl = (int)ctx->n_local;
  PF_CU(cudaEventRecord(ctx->ev_start, st));  // Y_j is ready
  PF_CU(cudaStreamWaitEvent(ctx->comm_st, ctx->ev_start, 0));
  const bool tl = ctx->prof;  // timeline: step start, slab arrivals, slab GEMM begin / end
  if (tl && ctx->ev_tl.empty()) {
    ctx->ev_tl.assign(1 + 3 * W, nullptr);
    for (auto& e : ctx->ev_tl) PF_CU(cudaEventCreate(&e));
  }
  if (tl) PF_CU(cudaEventRecord(ctx->ev_tl[0], st));
  PF_TRY((pf_status)ctx->comm->allgather_slabs(ctx->Yf[bidx], ctx->Yfull32,
                                                (size_t)ctx->p * nl * 4, ctx->comm_st,
                                                ctx->ev_slab.data()));

  PF_CU(cudaEventRecord(ctx->ev_comm_done, ctx->comm_st));
  PF_CU(coef_acc_launch(coef, ctx->coef_acc, st));
  const bool rec = ctx->prof && ctx->ev_used + 2 <= ctx->ev.size();
  if (ctx->prof && !rec) ++ctx->prof_dropped;
  if (rec) PF_CU(cudaEventRecord(ctx->ev[ctx->ev_used], st));
  for (int s = 0; s < W; ++s) {
    const int g = (ctx->rank - s + W) % W;
    PF_CU(cudaStreamWaitEvent(st, ctx->ev_slab[g], 0));
    if (tl) PF_CU(cudaEventRecord(ctx->ev_tl[1 + W + s], st));
    PF_CU(tf32_gemm_launch(ctx->tplan_s, ctx->mapA_s[g], ctx->mapB_s[g], ctx->mapApf_s[g],
                           s == 0 ? ycur : out, s == 0 ? yprev : nullptr, out, ctx->ldy32,
                           s == 0 ? coef : ctx->coef_acc, ctx->tf_ws, ctx->tf_acc, ctx->tf_cnt,
                           npass, st, 0));
    if (tl) PF_CU(cudaEventRecord(ctx->ev_tl[1 + 2 * W + s], st));
  }
  ctx->tl_valid = tl;
  if (rec) {
    PF_CU(cudaEventRecord(ctx->ev[ctx->ev_used + 1], st));
    ctx->ev_used += 2;
  }
  PF_CU(cudaStreamWaitEvent(st, ctx->ev_comm_done, 0));  // Yf[bidx] / Yfull32 reusable after
  return PF_OK;
}

static pf_status gemm_step32(pf_ctx ctx, int bidx, const float* ycur, const float* yprev,
                             float* out, const double* coef, int npass, cudaStream_t st) {
  if (ctx->overlap) return gemm_step32_overlap(ctx, bidx, ycur, yprev, out, coef, npass, st);
  const CUtensorMap* mb = &ctx->mapBf[bidx];
  int bdist_kb = 0;
  if (ctx->dist) {
    // all-gather the p-major blocks rank-major: [world][p][n_local] (equal slabs)
    size_t off[kMaxWorld + 1];
    for (int g = 0; g <= ctx->world; ++g) off[g] = (size_t)g * ctx->p * ctx->n_local * 4;
    PF_TRY((pf_status)ctx->comm->allgatherv(ctx->Yf[bidx], ctx->Yfull32, off, st));
    mb = &ctx->mapBfull32;
    bdist_kb = (int)(ctx->n_local / 16);
  }
  const bool rec = ctx->prof && ctx->ev_used + 2 <= ctx->ev.size();
  if (ctx->prof && !rec) ++ctx->prof_dropped;
  if (rec) PF_CU(cudaEventRecord(ctx->ev[ctx->ev_used], st));
  PF_CU(tf32_gemm_launch(ctx->tplan, ctx->mapAf, *mb, ctx->mapApf, ycur, yprev, out, ctx->ldy32,
                         coef, ctx->tf_ws, ctx->tf_acc, ctx->tf_cnt, npass, st, bdist_kb));
  if (rec) {
    PF_CU(cudaEventRecord(ctx->ev[ctx->ev_used + 1], st));
    ctx->ev_used += 2;
  }
  return PF_OK;
}

static pf_status gram32_all(pf_ctx ctx, const float* X, const float* Y, double* G, const int* cond,
                            cudaStream_t st) {
  PF_CU(gram32_launch(X, ctx->ldy32, Y, ctx->ldy32, (int)ctx->n_local, ctx->p, G, ctx->g32_part,
                      ctx->g32_slices, cond, st));
  // p x p sum over the row blocks.  Under a re-base condition the all-reduce runs regardless
  // (collectives cannot be skipped per rank); every rank evaluates the same plan, so either all
  // ranks consume the sum or none does.
  return allreduce(ctx, G, (size_t)ctx->p * ctx->p, st);
}

static pf_status chol32(pf_ctx ctx, int* shift_out, const int* cond, cudaStream_t st) {
  PF_CU(chol_inv_big_launch(ctx->G, ctx->p, ctx->n, ctx->chol_W, ctx->chol_D, ctx->Rinv,
                            ctx->state, shift_out, cond, st));
  return PF_OK;
}

static pf_status chol_pass32(pf_ctx ctx, float* Y, int* shift_out, const int* cond,
                             cudaStream_t st) {
  PF_TRY(gram32_all(ctx, Y, Y, ctx->G, cond, st));
  PF_TRY(chol32(ctx, shift_out, cond, st));
  PF_CU(rmul32_launch(Y, ctx->ldy32, ctx->Rinv, Y, ctx->ldy32, (int)ctx->n_local, ctx->p, cond, st));
  return PF_OK;
}

static pf_status orth_internal32(pf_ctx ctx, float* Y, cudaStream_t st) {
  PF_CU(cudaMemsetAsync(ctx->shift_flag, 0, sizeof(int), st));
  PF_TRY(chol_pass32(ctx, Y, ctx->shift_flag, nullptr, st));
  PF_TRY(chol_pass32(ctx, Y, ctx->shift_flag, nullptr, st));
  return chol_pass32(ctx, Y, nullptr, ctx->shift_flag, st);
}

static pf_status filter32(pf_ctx ctx, const float* A, int64_t lda, float* U, int64_t ldu,
                          const double* interval, int32_t q, double rho_max, cudaStream_t st) {
  if (ldu < ctx->n_local) return PF_ERR_DIM;
  PF_TRY(check_A32(ctx, A, lda));
  PF_TRY(map_A32(ctx, A, lda));
  const int p = ctx->p, d = ctx->d, nl = (int)ctx->n_local;
  PF_CU(plan_launch(interval, d, rho_max, p, ctx->state, st));
  ctx->filtered = true;
  ctx->last_d = d;
  ctx->last_q = q;
  PF_TRY(copy_block32(ctx, ctx->Yf[0], ctx->ldy32, U, ldu, st));
  int cur = 0, prev = -1;
  for (int rep = 0; rep < q; ++rep) {
    prev = -1;
    for (int j = 0; j < d; ++j) {
      const int out = (prev < 0) ? (cur + 1) % 3 : 3 - cur - prev;
      const double* coef = &ctx->state->coef[j][0];
      // precision schedule: early steps at tf_early passes, the last tf_tail steps in 3xTF32
      // (errors injected by the early steps are damped by the exact tail, reading R18)
      const int npass = (j >= d - ctx->tf_tail) ? 3 : ctx->tf_early;
      PF_TRY(gemm_step32(ctx, cur, ctx->Yf[cur], prev < 0 ? ctx->Yf[cur] : ctx->Yf[prev],
                         ctx->Yf[out], coef, npass, st));
      prev = cur;
      cur = out;
      if (j + 1 < d) {
        const int* cond = &ctx->state->rebase[j];
        PF_TRY(gram32_all(ctx, ctx->Yf[cur], ctx->Yf[cur], ctx->G, cond, st));
        PF_TRY(chol32(ctx, nullptr, cond, st));
        PF_CU(rmul32_launch(ctx->Yf[cur], ctx->ldy32, ctx->Rinv, ctx->Yf[cur], ctx->ldy32, nl, p,
                            cond, st));
        PF_CU(rmul32_launch(ctx->Yf[prev], ctx->ldy32, ctx->Rinv, ctx->Yf[prev], ctx->ldy32, nl, p,
                            cond, st));
      }
    }
  }
  PF_TRY(orth_internal32(ctx, ctx->Yf[cur], st));
  return copy_block32(ctx, U, ldu, ctx->Yf[cur], ctx->ldy32, st);
}

static pf_status rayleigh_ritz32(pf_ctx ctx, const float* A, int64_t lda, const float* U,
                                 int64_t ldu, float* V, int64_t ldv, double* theta,
                                 cudaStream_t st) {
  if (ldu < ctx->n_local || ldv < ctx->n_local) return PF_ERR_DIM;
  PF_TRY(check_A32(ctx, A, lda));
  PF_TRY(map_A32(ctx, A, lda));
  const int p = ctx->p, nl = (int)ctx->n_local;
  PF_TRY(copy_block32(ctx, ctx->Yf[0], ctx->ldy32, U, ldu, st));
  PF_TRY(gemm_step32(ctx, 0, ctx->Yf[0], ctx->Yf[0], ctx->Wf, &ctx->state->coef_rr[0], ctx->tf_rr,
                     st));
  PF_TRY(gram32_all(ctx, ctx->Yf[0], ctx->Wf, ctx->G, nullptr, st));  // H = Q^T (A Q)
  // H is formed from fp32 blocks (relative accuracy ~1e-7): diagonalise to off(H) <= 1e-12 ||H||
  // (fp64 storage of H; eigenvector error ~1e-12 / gap, far below the fp32 data error)
  // partial diagonalisation (reading R19): the damped interval of the last pf_filter call
  // (state->interval, set by its plan) bounds the Ritz values whose f is 0
  PF_CU(jacobi_big_launch(ctx->G, p, theta, ctx->Yeig, ctx->jac_H, ctx->jac_V, ctx->jac_red,
                          ctx->jac_cnt, ctx->state, 1e-12, 40,
                          ctx->filtered ? &ctx->state->interval[0] : nullptr, st));
  PF_CU(copy_theta_launch(theta, p, ctx->state, st, ctx->last_d, ctx->last_q));
  PF_CU(rmul32_launch(ctx->Yf[0], ctx->ldy32, ctx->Yeig, V, ldv, nl, p, nullptr, st));
  return PF_OK;
}

// ------------------------------------------------------------------------------ ABI
pf_status pf_lanczos(pf_ctx ctx, const void* Av, int64_t lda, const double* v0, int32_t m,
                     double* lo_hi, pf_stream stream) {
  if (!ctx || !lo_hi) return PF_ERR_ARG;
  if (!v0 && !ctx->lz_have_v0) return PF_ERR_ARG;  // warm start needs a previous refresh
  if (m < 1 || m > kMaxLanczos) return PF_ERR_ARG;
  if (!v0) v0 = ctx->lz_v0;  // lambda_min tracking: start from the last bottom Ritz vector
  const bool f32 = ctx->dtype == PF_TF32;
  const double* A = static_cast<const double*>(Av);
  const float* A32 = static_cast<const float*>(Av);
  if (f32) PF_TRY(check_A32(ctx, A32, lda));
  else PF_TRY(check_A(ctx, A, lda));
  cudaStream_t st = (cudaStream_t)stream;
  const int nl = (int)ctx->n_local, n = (int)ctx->n;
  m = (int32_t)std::min<int64_t>(m, ctx->n);
  double* h1 = ctx->lz_h;
  double* h2 = ctx->lz_h + kMaxLanczos;
  double* s = ctx->lz_h + 2 * kMaxLanczos;
  PF_CU(lz_start_launch(v0, nl, s, nullptr, ctx->state, st, /*norm_only=*/true));
  PF_TRY(allreduce(ctx, s, 1, st));
  PF_CU(lz_start_launch(v0, nl, s, ctx->lz_Q, ctx->state, st, /*norm_only=*/false));
  for (int j = 0; j < m; ++j) {
    double* qj = ctx->lz_Q + (size_t)j * ctx->lz_ldq;
    const double* qfull = qj;
    if (ctx->dist) {
      PF_TRY(gather(ctx, qj, ctx->lz_qfull, 1, st));
      qfull = ctx->lz_qfull;
    }
    if (f32)
      PF_CU(lz_gemv_f32_launch(A32, lda, nl, n, qfull, ctx->lz_Q, ctx->lz_ldq, j, ctx->lz_w, h1,
                               ctx->lz_part, ctx->lz_cnt, ctx->state, st));
    else if (ctx->lz_sym_ws)  // A symmetric: upper triangle only (half the HBM bytes)
      PF_CU(lz_symv_launch(A, lda, n, qfull, ctx->lz_Q, ctx->lz_ldq, j, ctx->lz_w, h1,
                           ctx->lz_sym_ws, ctx->lz_part, ctx->lz_cnt, ctx->state, ctx->num_sms,
                           st));
    else
      PF_CU(lz_gemv_launch(A, lda, nl, n, qfull, ctx->lz_Q, ctx->lz_ldq, j, ctx->lz_w, h1,
                           ctx->lz_part, ctx->lz_cnt, ctx->state, st));
    PF_TRY(allreduce(ctx, h1, (size_t)j + 1, st));
    PF_CU(lz_orth_launch(nl, ctx->lz_Q, ctx->lz_ldq, j, ctx->lz_w, h1, h2, ctx->lz_part,
                         ctx->lz_cnt, ctx->state, 1, st));
    PF_TRY(allreduce(ctx, h2, (size_t)j + 1, st));
    PF_CU(lz_orth_launch(nl, ctx->lz_Q, ctx->lz_ldq, j, ctx->lz_w, h2, s, ctx->lz_part,
                         ctx->lz_cnt, ctx->state, 2, st));
    PF_TRY(allreduce(ctx, s, 1, st));
    PF_CU(lz_next_launch(nl, ctx->lz_Q, ctx->lz_ldq, j, ctx->lz_w, s, ctx->state, st));
  }
  PF_CU(lanczos_finish_launch(m, ctx->lz_T, ctx->lz_theta, ctx->lz_S, lo_hi, ctx->state, st));
  PF_CU(lz_ritz_vector_launch(ctx->lz_Q, ctx->lz_ldq, nl, ctx->lz_S, ctx->state, ctx->lz_v0, st));
  ctx->lz_have_v0 = true;
  return PF_OK;
}

pf_status pf_interval_psd(pf_ctx ctx, const double* lo_hi, double eta, double* interval,
                          pf_stream stream) {
  if (!ctx || !lo_hi || !interval) return PF_ERR_ARG;
  if (!(eta > 0.0 && eta < 1.0)) return PF_ERR_ARG;
  PF_CU(interval_psd_launch(lo_hi, eta, interval, ctx->state, (cudaStream_t)stream));
  return PF_OK;
}

pf_status pf_interval_soft(pf_ctx ctx, double thr, double eta, double* interval,
                           pf_stream stream) {
  if (!ctx || !interval) return PF_ERR_ARG;
  if (!(eta >= 0.0 && eta < 1.0)) return PF_ERR_ARG;
  if (!(thr > 0.0)) return PF_ERR_INTERVAL;
  PF_CU(interval_soft_launch(thr, eta, interval, ctx->state, (cudaStream_t)stream));
  return PF_OK;
}

pf_status pf_interval_top_r(pf_ctx ctx, const double* lo_hi, int32_t r, double eta,
                            double* interval, pf_stream stream) {
  if (!ctx || !lo_hi || !interval) return PF_ERR_ARG;
  if (r < 1 || r > ctx->p || !(eta >= 0.0 && eta < 1.0)) return PF_ERR_ARG;
  PF_CU(interval_top_r_launch(lo_hi, r, eta, interval, ctx->state, (cudaStream_t)stream));
  return PF_OK;
}

pf_status pf_set_degree(pf_ctx ctx, int32_t degree) {
  if (!ctx || degree < 1 || degree > kMaxDeg) return PF_ERR_ARG;
  ctx->d = degree;
  return PF_OK;
}

pf_status pf_schedule_degree(pf_ctx ctx, double c, int32_t k, int32_t* degree) {
  if (!ctx || k < 0 || !(c >= 0.0)) return PF_ERR_ARG;
  // thm:conv1: convergence of PFPG needs d_k = Omega(log k / min{l, 1}); the
  // schedule d_k = max(d_0, ceil(c ln(k + 2))) grows like c ln k (c = 0: the fixed degree d_0)
  int dk = ctx->d0;
  if (c > 0.0) dk = std::max(dk, (int)std::ceil(c * std::log((double)k + 2.0)));
  if (dk > kMaxDeg) return PF_ERR_ARG;
  ctx->d = dk;
  if (degree) *degree = dk;
  return PF_OK;
}

pf_status pf_orth(pf_ctx ctx, void* Uv, int64_t ldu, pf_stream stream) {
  if (!ctx || !Uv) return PF_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (ctx->dtype == PF_TF32) {
    float* U = static_cast<float*>(Uv);
    if (ldu < ctx->n_local) return PF_ERR_DIM;
    PF_TRY(copy_block32(ctx, ctx->Yf[0], ctx->ldy32, U, ldu, st));
    PF_TRY(orth_internal32(ctx, ctx->Yf[0], st));
    return copy_block32(ctx, U, ldu, ctx->Yf[0], ctx->ldy32, st);
  }
  double* U = static_cast<double*>(Uv);
  if (ldu < ctx->p) return PF_ERR_DIM;
  const size_t row = (size_t)ctx->p * 8;
  PF_CU(cudaMemcpy2DAsync(ctx->Y[0], row, U, ldu * 8, row, ctx->n_local, cudaMemcpyDeviceToDevice, st));
  PF_TRY(orth_internal(ctx, ctx->Y[0], st));
  PF_CU(cudaMemcpy2DAsync(U, ldu * 8, ctx->Y[0], row, row, ctx->n_local, cudaMemcpyDeviceToDevice, st));
  return PF_OK;
}

pf_status pf_filter(pf_ctx ctx, const void* Av, int64_t lda, void* Uv, int64_t ldu,
                    const double* interval, int32_t q, double rho_max, pf_stream stream) {
  if (!ctx || !Uv || !interval) return PF_ERR_ARG;
  if (q < 1 || q > 10 || !(rho_max > 1.0)) return PF_ERR_ARG;
  if (ctx->dtype == PF_TF32)
    return filter32(ctx, static_cast<const float*>(Av), lda, static_cast<float*>(Uv), ldu,
                    interval, q, rho_max, (cudaStream_t)stream);
  const double* A = static_cast<const double*>(Av);
  double* U = static_cast<double*>(Uv);
  if (ldu < ctx->p) return PF_ERR_DIM;
  PF_TRY(check_A(ctx, A, lda));
  PF_TRY(map_A(ctx, A, lda));
  cudaStream_t st = (cudaStream_t)stream;
  // the digits pf_admm_step wrote with Z_new are reused; any other A is split afresh
  PF_TRY(split_A(ctx, A, lda, ctx->a8_fused, st));
  const int p = ctx->p, d = ctx->d;
  const int nl = (int)ctx->n_local;
  const size_t row = (size_t)p * 8;
  PF_CU(plan_launch(interval, d, rho_max, p, ctx->state, st));
  ctx->last_d = d;
  ctx->last_q = q;
  PF_CU(cudaMemcpy2DAsync(ctx->Y[0], row, U, ldu * 8, row, nl, cudaMemcpyDeviceToDevice, st));
  int cur = 0, prev = -1;
  for (int rep = 0; rep < q; ++rep) {
    prev = -1;
    for (int j = 0; j < d; ++j) {
      const int out = (prev < 0) ? (cur + 1) % 3 : 3 - cur - prev;
      const double* coef = &ctx->state->coef[j][0];
      // PF_FP64_I8 precision schedule (reading R25): the steps before the last i8_tail use
      // i8_early digit slices; their error off the wanted span is damped by the steps after
      const int su = (j < d - ctx->i8_tail) ? ctx->i8_early : 0;
      PF_TRY(gemm_step(ctx, cur, ctx->Y[cur], prev < 0 ? ctx->Y[cur] : ctx->Y[prev], ctx->Y[out],
                       coef, st, su));
      prev = cur;
      cur = out;
      if (j + 1 < d) {
        // span-exact re-base of (Y_j, Y_{j-1}) when the plan asks for it (device flag)
        const int* cond = &ctx->state->rebase[j];
        PF_TRY(gram_all(ctx, ctx->Y[cur], ctx->Y[cur], ctx->G, cond, st));
        PF_CU(chol64(ctx, nullptr, cond, st));
        PF_CU(rmul_launch(ctx->Y[cur], p, ctx->Rinv, ctx->Y[cur], p, nl, p, cond, st));
        PF_CU(rmul_launch(ctx->Y[prev], p, ctx->Rinv, ctx->Y[prev], p, nl, p, cond, st));
      }
    }
  }
  PF_TRY(orth_internal(ctx, ctx->Y[cur], st));
  PF_CU(cudaMemcpy2DAsync(U, ldu * 8, ctx->Y[cur], row, row, nl, cudaMemcpyDeviceToDevice, st));
  return PF_OK;
}

pf_status pf_rayleigh_ritz(pf_ctx ctx, const void* Av, int64_t lda, const void* Uv,
                           int64_t ldu, void* Vv, int64_t ldv, double* theta, pf_stream stream) {
  if (!ctx || !Uv || !Vv || !theta) return PF_ERR_ARG;
  if (ctx->dtype == PF_TF32)
    return rayleigh_ritz32(ctx, static_cast<const float*>(Av), lda, static_cast<const float*>(Uv),
                           ldu, static_cast<float*>(Vv), ldv, theta, (cudaStream_t)stream);
  const double* A = static_cast<const double*>(Av);
  const double* U = static_cast<const double*>(Uv);
  double* V = static_cast<double*>(Vv);
  if (ldu < ctx->p || ldv < ctx->p || (ldv & 1) || !aligned16(V)) return PF_ERR_DIM;
  PF_TRY(check_A(ctx, A, lda));
  PF_TRY(map_A(ctx, A, lda));
  cudaStream_t st = (cudaStream_t)stream;
  PF_TRY(split_A(ctx, A, lda, true, st));
  const int p = ctx->p, nl = (int)ctx->n_local;
  const size_t row = (size_t)p * 8;
  PF_CU(cudaMemcpy2DAsync(ctx->Y[0], row, U, ldu * 8, row, nl, cudaMemcpyDeviceToDevice, st));
  PF_TRY(gemm_step(ctx, 0, ctx->Y[0], ctx->Y[0], ctx->Wbuf, &ctx->state->coef_rr[0], st));
  PF_TRY(gram_all(ctx, ctx->Y[0], ctx->Wbuf, ctx->G, nullptr, st));  // H = Q^T (A Q)
  // stop once off(H) <= tol ||H||_F.  X = V f(Lambda) V^T is a 1-Lipschitz spectral function of
  // H, so the residual off-diagonal moves X by O(tol ||H||); PF_JACOBI_TOL (development knob)
  // defaults to p * 1e-16 (the rounding floor of H)
  static double jtol = -1.0;
  if (jtol < 0.0) {
    const char* e = getenv("PF_JACOBI_TOL");
    jtol = e ? atof(e) : 0.0;
  }
  PF_CU(jacobi_launch(ctx->G, p, nullptr, theta, ctx->Yeig, ctx->state,
                      jtol > 0.0 ? jtol : std::max(1e-15, 1e-16 * p), 40, st));
  PF_CU(copy_theta_launch(theta, p, ctx->state, st, ctx->last_d, ctx->last_q));
  PF_CU(rmul_launch(ctx->Y[0], p, ctx->Yeig, V, ldv, nl, p, nullptr, st));
  return PF_OK;
}

pf_status pf_spectral_op(pf_ctx ctx, pf_op op, double thr, const double* theta, double* f,
                         int32_t* rank, pf_stream stream) {
  if (!ctx || !theta || !f || !rank) return PF_ERR_ARG;
  if (op != PF_OP_PSD && op != PF_OP_SOFT_THRESHOLD) return PF_ERR_ARG;
  if (op == PF_OP_SOFT_THRESHOLD && !(thr >= 0.0)) return PF_ERR_ARG;
  PF_CU(spectral_launch((int)op, thr, theta, ctx->p, f, rank, ctx->state, (cudaStream_t)stream));
  return PF_OK;
}

static pf_status full_V(pf_ctx ctx, const double* V, int64_t ldv, const double** Vf,
                        int64_t* ldf, cudaStream_t st) {
  if (!ctx->dist) {
    *Vf = V;
    *ldf = ldv;
    return PF_OK;
  }
  const size_t row = (size_t)ctx->p * 8;
  PF_CU(cudaMemcpy2DAsync(ctx->Wbuf, row, V, ldv * 8, row, ctx->n_local, cudaMemcpyDeviceToDevice, st));
  *Vf = ctx->Vfull;
  *ldf = ctx->p;
  return gather(ctx, ctx->Wbuf, ctx->Vfull, ctx->p, st);
}

pf_status pf_prox_step(pf_ctx ctx, const double* V, int64_t ldv, const double* f, double tau,
                       double mu, const uint32_t* omega, int64_t ldo, const double* W,
                       int64_t ldw, int32_t r, double* A_out, int64_t lda_out, double* obj,
                       pf_stream stream) {
  if (!ctx || !V || !f || !omega || !A_out || !obj) return PF_ERR_ARG;
  if (!(mu >= 0.0)) return PF_ERR_ARG;
  if (!is_fp64(ctx)) return PF_ERR_UNSUPPORTED;
  if (r < 0 || r > 64 || (r > 0 && !W)) return PF_ERR_ARG;
  if (ldv < ctx->p || (ldv & 1) || !aligned16(V) || ldo < (ctx->n + 31) / 32 ||
      lda_out < ctx->n || (r > 0 && ldw < r))
    return PF_ERR_DIM;
  cudaStream_t st = (cudaStream_t)stream;
  iterate_written(ctx);
  const double* Vf;
  int64_t ldf;
  PF_TRY(full_V(ctx, V, ldv, &Vf, &ldf, st));
  PF_CU(prox_launch(Vf, ldf, V, ldv, f, tau, omega, ldo, W, ldw, r, A_out, lda_out,
                    (int)ctx->n_local, (int)ctx->n, (int)ctx->row0, ctx->p, obj, ctx->rb_part,
                    ctx->rb_cnt, ctx->VFbuf, st));
  // obj[0] (the fit) is a sum over row blocks; obj[1] = sum |f| is replicated
  PF_TRY(allreduce(ctx, obj, 1, st));
  PF_CU(pfpg_obj_finish_launch(obj, mu, st));
  return PF_OK;
}

pf_status pf_rebuild(pf_ctx ctx, const double* V, int64_t ldv, const double* f, double* X,
                     int64_t ldx, pf_stream stream) {
  if (!ctx || !V || !f || !X) return PF_ERR_ARG;
  if (!is_fp64(ctx)) return PF_ERR_UNSUPPORTED;
  if (ldv < ctx->p || (ldv & 1) || !aligned16(V) || ldx < ctx->n) return PF_ERR_DIM;
  cudaStream_t st = (cudaStream_t)stream;
  const double* Vf;
  int64_t ldf;
  PF_TRY(full_V(ctx, V, ldv, &Vf, &ldf, st));
  // the PFPG update kernel with no mask and tau = 0: X - 0 * Omega o (X - M) = X (its objective
  // partials land in scratch)
  PF_CU(prox_launch(Vf, ldf, V, ldv, f, 0.0, nullptr, 0, nullptr, 0, 0, X, ldx, (int)ctx->n_local,
                    (int)ctx->n, (int)ctx->row0, ctx->p, ctx->rb_obj, ctx->rb_part, ctx->rb_cnt,
                    ctx->VFbuf, st));
  if (X == ctx->a8_src) iterate_written(ctx);
  return PF_OK;
}

pf_status pf_admm_step(pf_ctx ctx, const double* V, int64_t ldv, const double* f, double t,
                       const uint32_t* adj, int64_t ldadj, const double* deg, double* Z,
                       int64_t ldz, double* obj, pf_stream stream) {
  if (!ctx || !V || !f || !adj || !deg || !Z || !obj) return PF_ERR_ARG;
  if (!is_fp64(ctx)) return PF_ERR_UNSUPPORTED;
  if (ldv < ctx->p || (ldv & 1) || !aligned16(V) || ldadj < (ctx->n + 31) / 32 || ldz < ctx->n)
    return PF_ERR_DIM;
  cudaStream_t st = (cudaStream_t)stream;
  iterate_written(ctx);
  const double* Vf;
  int64_t ldf;
  PF_TRY(full_V(ctx, V, ldv, &Vf, &ldf, st));
  // one GPU, int8-digit filter: the update writes Z_new's digit slices for the next pf_filter
  const bool fuse = use_i8(ctx) && !ctx->dist && ctx->fuse_digits &&
                    (ctx->i8plan.S == 6 || ctx->i8plan.S == 7);
  RbDigits dig{ctx->A8, ctx->i8plan.kblocks, ctx->i8plan.S, ctx->a8_E, ctx->a8_rscale, ctx->a8_wa, ctx->a8_wmax};
  // the half-storage product reads the upper tiles only: no mirror digits (unless a precision
  // schedule will run products on fewer slices, which the half-storage kernel does not do)
  const bool half = (ctx->i8s_ok || ctx->i8t_ok) && ctx->i8_early >= ctx->i8plan.S;
  R8Bufs r8{ctx->r8_maps, ctx->r8_VF8, ctx->r8_V8, ctx->r8_rs,
            ctx->r8_rs + (size_t)ctx->i8plan.mtiles * 128, ctx->num_sms, half ? 0 : 1,
            ctx->z_upper ? 0 : 1};
  const bool urec = ctx->prof && ctx->evu_used + 2 <= ctx->evu.size();
  if (urec) PF_CU(cudaEventRecord(ctx->evu[ctx->evu_used], st));
  PF_CU(admm_launch(Vf, ldf, V, ldv, f, t, adj, ldadj, deg, Z, ldz, (int)ctx->n_local,
                    (int)ctx->n, (int)ctx->row0, ctx->p, obj, ctx->rb_part, ctx->rb_cnt,
                    ctx->dist ? 1 : 0, ctx->VFbuf, st, fuse ? &dig : nullptr, nullptr,
                    fuse && ctx->r8_on ? &r8 : nullptr, ctx->k7tma ? ctx->num_sms : 0));
  if (urec) {
    PF_CU(cudaEventRecord(ctx->evu[ctx->evu_used + 1], st));
    ctx->evu_used += 2;
  }
  if (fuse) {
    ctx->a8_src = Z;
    ctx->a8_lda = ldz;
    ctx->a8_valid = ctx->a8_fused = true;
    ctx->a8_half = half && ctx->r8_on && ctx->i8plan.S == 7 && r8_usable(Z, ldz);
    if (ctx->z_upper && ctx->r8_on && ctx->p == 64 && ctx->i8plan.S == 7 && r8_usable(Z, ldz))
      ctx->z_upper_src = Z;
  }
  if (ctx->dist) {
    // <C, W> and the squared residual are sums over row blocks; sqrt after the reduction
    PF_TRY(allreduce(ctx, obj, 2, st));
    PF_CU(sqrt_inplace_launch(obj + 1, st));
  }
  return PF_OK;
}

pf_status pf_admm_step_f(pf_ctx ctx, const double* Q, int64_t ldq, const double* F, double t,
                         const uint32_t* adj, int64_t ldadj, const double* deg, double* Z,
                         int64_t ldz, double* obj, pf_stream stream) {
  if (!ctx || !Q || !F || !adj || !deg || !Z || !obj) return PF_ERR_ARG;
  if (!is_fp64(ctx)) return PF_ERR_UNSUPPORTED;
  if (ldq < ctx->p || (ldq & 1) || !aligned16(Q) || ldadj < (ctx->n + 31) / 32 || ldz < ctx->n)
    return PF_ERR_DIM;
  cudaStream_t st = (cudaStream_t)stream;
  iterate_written(ctx);
  const double* Qf;
  int64_t ldf;
  PF_TRY(full_V(ctx, Q, ldq, &Qf, &ldf, st));
  // local rows of Q F (the I panels of the rebuild); full_V used Wbuf only when distributed
  PF_CU(rmul_launch(Q, ldq, F, ctx->VFbuf, ctx->p, (int)ctx->n_local, ctx->p, nullptr, st));
  const bool fuse = use_i8(ctx) && !ctx->dist && ctx->fuse_digits &&
                    (ctx->i8plan.S == 6 || ctx->i8plan.S == 7);
  RbDigits dig{ctx->A8, ctx->i8plan.kblocks, ctx->i8plan.S, ctx->a8_E, ctx->a8_rscale, ctx->a8_wa, ctx->a8_wmax};
  // the half-storage product reads the upper tiles only: no mirror digits (unless a precision
  // schedule will run products on fewer slices, which the half-storage kernel does not do)
  const bool half = (ctx->i8s_ok || ctx->i8t_ok) && ctx->i8_early >= ctx->i8plan.S;
  R8Bufs r8{ctx->r8_maps, ctx->r8_VF8, ctx->r8_V8, ctx->r8_rs,
            ctx->r8_rs + (size_t)ctx->i8plan.mtiles * 128, ctx->num_sms, half ? 0 : 1,
            ctx->z_upper ? 0 : 1};
  const bool urec = ctx->prof && ctx->evu_used + 2 <= ctx->evu.size();
  if (urec) PF_CU(cudaEventRecord(ctx->evu[ctx->evu_used], st));
  PF_CU(admm_launch(Qf, ldf, Q, ldq, nullptr, t, adj, ldadj, deg, Z, ldz, (int)ctx->n_local,
                    (int)ctx->n, (int)ctx->row0, ctx->p, obj, ctx->rb_part, ctx->rb_cnt,
                    ctx->dist ? 1 : 0, ctx->VFbuf, st, fuse ? &dig : nullptr, F,
                    fuse && ctx->r8_on ? &r8 : nullptr, ctx->k7tma ? ctx->num_sms : 0));
  if (urec) {
    PF_CU(cudaEventRecord(ctx->evu[ctx->evu_used + 1], st));
    ctx->evu_used += 2;
  }
  if (fuse) {
    ctx->a8_src = Z;
    ctx->a8_lda = ldz;
    ctx->a8_valid = ctx->a8_fused = true;
    ctx->a8_half = half && ctx->r8_on && ctx->i8plan.S == 7 && r8_usable(Z, ldz);
    if (ctx->z_upper && ctx->r8_on && ctx->p == 64 && ctx->i8plan.S == 7 && r8_usable(Z, ldz))
      ctx->z_upper_src = Z;
  }
  if (ctx->dist) {
    PF_TRY(allreduce(ctx, obj, 2, st));
    PF_CU(sqrt_inplace_launch(obj + 1, st));
  }
  return PF_OK;
}

pf_status pf_nce_step(pf_ctx ctx, const double* V, int64_t ldv, const double* f, double tau,
                      const double* gdiag, const double* x_in, double* x_out, double* B,
                      int64_t ldb, double* obj, pf_stream stream) {
  if (!ctx || !V || !f || !gdiag || !x_in || !x_out || !B || !obj) return PF_ERR_ARG;
  if (!is_fp64(ctx)) return PF_ERR_UNSUPPORTED;
  if (ldv < ctx->p || ldb < ctx->n) return PF_ERR_DIM;
  if (!(tau > 0.0)) return PF_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  iterate_written(ctx);
  PF_CU(nce_launch(V, ldv, f, ctx->p, tau, gdiag, x_in, x_out, B, ldb, (int)ctx->n_local,
                   (int)ctx->row0, ctx->rb_part, ctx->rb_cnt, obj, st));
  PF_TRY(allreduce(ctx, obj, 2, st));  // raw sums over the row blocks
  PF_CU(nce_finish_launch(f, ctx->p, obj, st));
  return PF_OK;
}

pf_status pf_extrapolate(pf_ctx ctx, const double* const* hist, int32_t l, double lam_rel,
                         const double* gdiag, double* x_out, double* B, int64_t ldb, double* coef,
                         pf_stream stream) {
  if (!ctx || !hist || !gdiag || !x_out || !B) return PF_ERR_ARG;
  if (!is_fp64(ctx)) return PF_ERR_UNSUPPORTED;
  if (l < 0 || l + 1 > 8 || !(lam_rel > 0.0)) return PF_ERR_ARG;
  if (ldb < ctx->n) return PF_ERR_DIM;
  for (int i = 0; i <= l + 1; ++i)
    if (!hist[i]) return PF_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  iterate_written(ctx);
  const int L = l + 1;
  // partials: rna_blocks * L(L+1)/2 <= 128 * 36 doubles fit the rebuild partials buffer
  PF_CU(rna_gram_launch(hist, L, (int)ctx->n_local, ctx->rb_part, ctx->rb_cnt, ctx->G, st));
  PF_TRY(allreduce(ctx, ctx->G, (size_t)L * L, st));
  PF_CU(rna_combine_launch(hist, L, (int)ctx->n_local, ctx->G, lam_rel, gdiag, x_out, B, ldb,
                           (int)ctx->row0, coef, st));
  return PF_OK;
}

pf_status pf_perturb(pf_ctx ctx, double* A, int64_t lda, const double* E, int64_t lde,
                     pf_stream stream) {
  if (!ctx || !A || !E) return PF_ERR_ARG;
  if (!is_fp64(ctx)) return PF_ERR_UNSUPPORTED;
  if (lda < ctx->n || lde < ctx->n) return PF_ERR_DIM;
  iterate_written(ctx);
  PF_CU(perturb_launch(A, lda, E, lde, (int)ctx->n_local, (int)ctx->n, (cudaStream_t)stream));
  return PF_OK;
}

pf_status pf_perturb_hash(pf_ctx ctx, float* A, int64_t lda, uint64_t seed, int32_t k,
                          double noise, pf_stream stream) {
  if (!ctx || !A) return PF_ERR_ARG;
  if (ctx->dtype != PF_TF32) return PF_ERR_UNSUPPORTED;
  if (lda < ctx->n) return PF_ERR_DIM;
  PF_CU(perturb_hash32_launch(A, lda, (int)ctx->n_local, (int)ctx->n, (int)ctx->row0,
                              (unsigned long long)seed, k, noise, (cudaStream_t)stream));
  return PF_OK;
}

pf_status pf_set_tf32_passes(pf_ctx ctx, int32_t passes) {
  if (!ctx || passes < 1 || passes > 3) return PF_ERR_ARG;
  if (ctx->dtype != PF_TF32) return PF_ERR_UNSUPPORTED;
  ctx->tf_early = passes;
  ctx->tf_tail = 0;
  ctx->tf_rr = passes;
  return PF_OK;
}

pf_status pf_set_i8_slices(pf_ctx ctx, int32_t slices) {
  if (!ctx) return PF_ERR_ARG;
  if (ctx->dtype != PF_FP64_I8) return PF_ERR_UNSUPPORTED;
  if (slices != 0 && (slices < 6 || slices > kI8MaxSlices)) return PF_ERR_ARG;
  if (slices > 0) {
    ctx->i8plan = i8_plan(ctx->p, (int)ctx->n_local, (int)ctx->n, slices, ctx->num_sms);
    ctx->i8_early = std::min(ctx->i8_early, slices);
    if (!encode_i8_maps(ctx)) {
      snprintf(ctx->err, sizeof(ctx->err), "cuTensorMapEncodeTiled(int8 slices) failed");
      return PF_ERR_CUDA;
    }
  } else {
    ctx->i8plan.S = 0;
  }
  ctx->a8_valid = false;
  return PF_OK;
}

pf_status pf_set_i8_schedule(pf_ctx ctx, int32_t early_slices, int32_t exact_tail) {
  if (!ctx) return PF_ERR_ARG;
  if (ctx->dtype != PF_FP64_I8) return PF_ERR_UNSUPPORTED;
  if (early_slices < 4 || early_slices > kI8MaxSlices || exact_tail < 0) return PF_ERR_ARG;
  ctx->i8_early = std::min<int>(early_slices, ctx->i8plan.S > 0 ? ctx->i8plan.S : kI8MaxSlices);
  ctx->i8_tail = exact_tail;
  return PF_OK;
}

pf_status pf_invalidate(pf_ctx ctx) {
  if (!ctx) return PF_ERR_ARG;
  iterate_written(ctx);
  ctx->z_upper_src = nullptr;  // the caller wrote the iterate (in full)
  return PF_OK;
}

pf_status pf_set_z_upper(pf_ctx ctx, int32_t upper) {
  if (!ctx || (upper != 0 && upper != 1)) return PF_ERR_ARG;
  if (!upper) {
    ctx->z_upper = false;
    ctx->z_upper_src = nullptr;
    return PF_OK;
  }
  if (!use_i8(ctx) || ctx->dist || !ctx->fuse_digits || !ctx->r8_on || ctx->p != 64 ||
      ctx->i8plan.S != 7 || !ctx->lz_sym_ws) {
    snprintf(ctx->err, sizeof(ctx->err),
             "upper-block storage needs the one-GPU int8-digit update (p = 64, S = 7) and the "
             "symmetric Lanczos GEMV");
    return PF_ERR_UNSUPPORTED;
  }
  ctx->z_upper = true;
  return PF_OK;
}

pf_status pf_matmul(pf_ctx ctx, const double* A, int64_t lda, const double* Y, int64_t ldy,
                    double* out, int64_t ldo, pf_stream stream) {
  if (!ctx || !A || !Y || !out) return PF_ERR_ARG;
  if (!is_fp64(ctx)) return PF_ERR_UNSUPPORTED;
  if (ldy < ctx->p || ldo < ctx->p) return PF_ERR_DIM;
  PF_TRY(check_A(ctx, A, lda));
  PF_TRY(map_A(ctx, A, lda));
  cudaStream_t st = (cudaStream_t)stream;
  PF_TRY(split_A(ctx, A, lda, true, st));
  const int p = ctx->p, nl = (int)ctx->n_local;
  const size_t row = (size_t)p * 8;
  PF_CU(cudaMemcpy2DAsync(ctx->Y[0], row, Y, ldy * 8, row, nl, cudaMemcpyDeviceToDevice, st));
  PF_TRY(gemm_step(ctx, 0, ctx->Y[0], ctx->Y[0], ctx->Wbuf, &ctx->state->coef_rr[0], st));
  PF_CU(cudaMemcpy2DAsync(out, ldo * 8, ctx->Wbuf, row, row, nl, cudaMemcpyDeviceToDevice, st));
  return PF_OK;
}

// ------------------------------------------------------------------------------ Newton-Schulz RR
pf_status pf_rr_ns(pf_ctx ctx, const void* Av, int64_t lda, const void* Uv, int64_t ldu,
                   pf_op op, double thr, double* F, int32_t* rank, int32_t* iters,
                   pf_stream stream) {
  if (!ctx || !Uv || !F || !rank) return PF_ERR_ARG;
  if (op != PF_OP_PSD && op != PF_OP_SOFT_THRESHOLD) return PF_ERR_ARG;
  if (op == PF_OP_SOFT_THRESHOLD && !(thr > 0.0)) return PF_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const int p = ctx->p;
  if (ctx->dtype == PF_TF32) {
    const float* A = static_cast<const float*>(Av);
    if (ldu < ctx->n_local) return PF_ERR_DIM;
    PF_TRY(check_A32(ctx, A, lda));
    PF_TRY(map_A32(ctx, A, lda));
    PF_TRY(copy_block32(ctx, ctx->Yf[0], ctx->ldy32, static_cast<const float*>(Uv), ldu, st));
    PF_TRY(gemm_step32(ctx, 0, ctx->Yf[0], ctx->Yf[0], ctx->Wf, &ctx->state->coef_rr[0],
                       ctx->tf_rr, st));
    PF_TRY(gram32_all(ctx, ctx->Yf[0], ctx->Wf, ctx->G, nullptr, st));  // H = Q^T (A Q)
  } else {
    const double* A = static_cast<const double*>(Av);
    if (ldu < p) return PF_ERR_DIM;
    PF_TRY(check_A(ctx, A, lda));
    PF_TRY(map_A(ctx, A, lda));
    PF_TRY(split_A(ctx, A, lda, true, st));
    const size_t row = (size_t)p * 8;
    PF_CU(cudaMemcpy2DAsync(ctx->Y[0], row, Uv, ldu * 8, row, ctx->n_local,
                            cudaMemcpyDeviceToDevice, st));
    PF_TRY(gemm_step(ctx, 0, ctx->Y[0], ctx->Y[0], ctx->Wbuf, &ctx->state->coef_rr[0], st));
    PF_TRY(gram_all(ctx, ctx->Y[0], ctx->Wbuf, ctx->G, nullptr, st));
  }
  if (!ctx->ns) {
    ctx->ns = ns_create(p);
    if (!ctx->ns) {
      snprintf(ctx->err, sizeof(ctx->err), "pf_rr_ns: workspace allocation failed");
      return PF_ERR_NOMEM;
    }
  }
  const int soft = op == PF_OP_SOFT_THRESHOLD ? 1 : 0;
  // no Ritz values: the next re-base plan falls back to the Lanczos spread estimate, unless the
  // PD test below records its norm bound of H
  PF_CU(cudaMemsetAsync(&ctx->state->have_theta, 0, sizeof(int), st));
  PF_CU(ns_spectral(ctx->ns, ctx->G, soft, thr, F, rank, iters, ctx->state, st));
  // device-side fallback (no host decision): Jacobi on the same H, then F = Y f(theta) Y^T;
  // both launches return at once unless the Newton-Schulz kernel raised its fail flag
  const int* fail = ns_fail_flag(ctx->ns);
  if (p <= 128)  // single-CTA Jacobi (the cooperative one needs p >= 64 pairs of lanes)
    PF_CU(jacobi_launch(ctx->G, p, nullptr, ctx->jac_theta, ctx->Yeig, ctx->state,
                        std::max(1e-15, 1e-16 * p), 40, st, fail));
  else
    PF_CU(jacobi_big_launch(ctx->G, p, ctx->jac_theta, ctx->Yeig, ctx->jac_H, ctx->jac_V,
                            ctx->jac_red, ctx->jac_cnt, ctx->state, 1e-13, 40, nullptr, st, fail));
  PF_CU(ns_fallback_launch(fail, soft, thr, ctx->jac_theta, ctx->Yeig, p, F, rank, st));
  ctx->filtered = false;
  return PF_OK;
}

// ------------------------------------------------------------------------------ PFSVT (NEXT-3)
static pf_status svt_check(pf_ctx ctx) {
  if (!is_fp64(ctx)) return PF_ERR_UNSUPPORTED;
  if (ctx->dist) return PF_ERR_UNSUPPORTED;  // one GPU: the sampled set is not row-split
  return PF_OK;
}

pf_status pf_spmm(pf_ctx ctx, const int32_t* ptr, const int32_t* idx, const double* val,
                  const int32_t* vperm, const double* X, int64_t ldx, double s1, double s2,
                  double s3, const double* Ycur, int64_t ldc, const double* Yprev, int64_t ldp,
                  double* out, int64_t ldo, pf_stream stream) {
  if (!ctx || !ptr || !idx || !val || !X || !out) return PF_ERR_ARG;
  PF_TRY(svt_check(ctx));
  if ((s2 != 0.0 && !Ycur) || (s3 != 0.0 && !Yprev)) return PF_ERR_ARG;
  const int p = ctx->p;
  if (ldx < p || ldo < p || (s2 != 0.0 && ldc < p) || (s3 != 0.0 && ldp < p)) return PF_ERR_DIM;
  const double coef[3] = {s1, s2, s3};
  PF_CU(spmm_launch((int)ctx->n, p, ptr, idx, val, vperm, X, ldx, coef, Ycur, ldc, Yprev, ldp,
                    out, ldo, (cudaStream_t)stream));
  return PF_OK;
}

pf_status pf_svt_kick(pf_ctx ctx, const double* b, int64_t nnz, double mu, double delta,
                      double norm2, double* x, pf_stream stream) {
  if (!ctx || !b || !x || nnz < 0) return PF_ERR_ARG;
  PF_TRY(svt_check(ctx));
  if (!(mu > 0.0) || !(delta > 0.0) || !(norm2 > 0.0)) return PF_ERR_ARG;
  // SVT's kicking (reading R24): x^0 = k0 delta b, k0 = ceil(mu / (delta ||P_Omega(M)||_2))
  const double k0 = std::ceil(mu / (delta * norm2));
  PF_CU(svt_kick_launch(x, b, k0 * delta, nnz, (cudaStream_t)stream));
  return PF_OK;
}

pf_status pf_svt_filter(pf_ctx ctx, const int32_t* ptr, const int32_t* idx, const int32_t* cptr,
                        const int32_t* cidx, const int32_t* perm, const double* val, double* Q,
                        int64_t ldq, double mu, double eta, pf_stream stream) {
  if (!ctx || !ptr || !idx || !cptr || !cidx || !perm || !val || !Q) return PF_ERR_ARG;
  PF_TRY(svt_check(ctx));
  const int p = ctx->p, n = (int)ctx->n, d = ctx->d;
  if (ldq < p) return PF_ERR_DIM;
  if (!(mu > 0.0) || !(eta >= 0.0 && eta < 1.0)) return PF_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  // damped interval of Y^T Y: [a, b] = [0, (1 - eta) mu^2] (singular values below the threshold,
  // reading R24); L(t) = (t - c) / e (eqn:cheb-linear-map P:216-218)
  const double a = 0.0, bb = (1.0 - eta) * mu * mu;
  const double c = 0.5 * (a + bb), e = 0.5 * (bb - a);
  const size_t row = (size_t)p * 8;
  PF_CU(cudaMemcpy2DAsync(ctx->Y[0], row, Q, ldq * 8, row, n, cudaMemcpyDeviceToDevice, st));
  int cur = 0, prev = -1;
  for (int j = 0; j < d; ++j) {
    // T = Y Y_j (CSR), then Y_{j+1} = s1 Y^T T + s2 Y_j + s3 Y_{j-1} (CSC view, eq:cheb)
    const double one[3] = {1.0, 0.0, 0.0};
    PF_CU(spmm_launch(n, p, ptr, idx, val, nullptr, ctx->Y[cur], p, one, nullptr, 0, nullptr, 0,
                      ctx->Wbuf, p, st));
    const int out = (prev < 0) ? (cur + 1) % 3 : 3 - cur - prev;
    const double first[3] = {1.0 / e, -c / e, 0.0};
    const double next[3] = {2.0 / e, -2.0 * c / e, -1.0};
    PF_CU(spmm_launch(n, p, cptr, cidx, val, perm, ctx->Wbuf, p, j == 0 ? first : next,
                      ctx->Y[cur], p, prev < 0 ? nullptr : ctx->Y[prev], p, ctx->Y[out], p, st));
    prev = cur;
    cur = out;
  }
  PF_TRY(orth_internal(ctx, ctx->Y[cur], st));
  PF_CU(cudaMemcpy2DAsync(Q, ldq * 8, ctx->Y[cur], row, row, n, cudaMemcpyDeviceToDevice, st));
  return PF_OK;
}

pf_status pf_svt_ritz(pf_ctx ctx, const int32_t* ptr, const int32_t* idx, const double* val,
                      const double* Q, int64_t ldq, double mu, double* U, int64_t ldu, double* V,
                      int64_t ldv, double* sigma, double* s, int32_t* svp, pf_stream stream) {
  if (!ctx || !ptr || !idx || !val || !Q || !U || !V || !sigma || !s || !svp) return PF_ERR_ARG;
  PF_TRY(svt_check(ctx));
  const int p = ctx->p, n = (int)ctx->n;
  if (ldq < p || ldu < p || ldv < p) return PF_ERR_DIM;
  if (!(mu >= 0.0)) return PF_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const double one[3] = {1.0, 0.0, 0.0};
  PF_CU(spmm_launch(n, p, ptr, idx, val, nullptr, Q, ldq, one, nullptr, 0, nullptr, 0,
                    ctx->Wbuf, p, st));                                  // B = Y Q
  PF_CU(gram_launch(ctx->Wbuf, ctx->Wbuf, n, p, ctx->G, ctx->gram_part, nullptr, nullptr, st));
  PF_CU(jacobi_launch(ctx->G, p, nullptr, sigma, ctx->Yeig, ctx->state,
                      std::max(1e-15, 1e-16 * p), 40, st));              // B^T B = W L W^T
  PF_CU(svt_sigma_launch(sigma, p, mu, sigma, s, ctx->Rinv, svp, st));  // sigma, shrink, 1/sigma
  PF_CU(rmul_launch(Q, ldq, ctx->Yeig, V, ldv, n, p, nullptr, st));      // V = Q W
  PF_CU(rmul_launch(ctx->Wbuf, p, ctx->Yeig, U, ldu, n, p, nullptr, st));  // U = B W / sigma
  PF_CU(scale_cols_inplace_launch(U, ldu, n, p, ctx->Rinv, st));
  return PF_OK;
}

pf_status pf_svt_update(pf_ctx ctx, const int32_t* ptr, const int32_t* idx, const double* b,
                        double* x, const double* U, int64_t ldu, const double* V, int64_t ldv,
                        const double* s, double delta, double* rss, pf_stream stream) {
  if (!ctx || !ptr || !idx || !b || !x || !U || !V || !s || !rss) return PF_ERR_ARG;
  PF_TRY(svt_check(ctx));
  const int p = ctx->p;
  if (ldu < p || ldv < p) return PF_ERR_DIM;
  PF_CU(svt_sample_launch((int)ctx->n, p, ptr, idx, b, x, U, ldu, V, ldv, s, delta, ctx->svt_part,
                          ctx->svt_cnt, rss, (cudaStream_t)stream));
  return PF_OK;
}

pf_status pf_set_tf32_schedule(pf_ctx ctx, int32_t early_passes, int32_t exact_tail) {
  if (!ctx || early_passes < 1 || early_passes > 3 || exact_tail < 0) return PF_ERR_ARG;
  if (ctx->dtype != PF_TF32) return PF_ERR_UNSUPPORTED;
  ctx->tf_early = early_passes;
  ctx->tf_tail = exact_tail;
  ctx->tf_rr = 3;
  return PF_OK;
}

}  // extern "C"
