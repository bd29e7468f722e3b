// pf_api.cu -- the C ABI (include/pf.h): context / scratch management and the orchestration of
// the hot-path kernels for one PFPG / PFAM iteration.  All work is stream-ordered; nothing here
// synchronises the host except pf_get_device_status.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <new>

#include "../../include/pf.h"
#include "pf_kernels.cuh"

#include <atomic>
#include <vector>

using namespace pf;

static std::atomic<long long> g_launches{0};
void pf::count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

struct pf_ctx_s {
  // profiling of the dominant kernel: event pairs around every Chebyshev-step GEMM launch
  bool prof = false;
  std::vector<cudaEvent_t> ev;
  size_t ev_used = 0;
  long long prof_dropped = 0;
  int64_t n = 0, n_local = 0, row0 = 0;
  int p = 0, d = 0, rank = 0, world = 1, num_sms = 148;
  DevState* state = nullptr;
  double* Y[3] = {nullptr, nullptr, nullptr};  // n_local x p, ld p
  double* Yfull = nullptr;                     // n x p gathered block (world > 1)
  double* Wbuf = nullptr;                      // n_local x p (A Q)
  double* Vfull = nullptr;                     // n x p (world > 1)
  double* G = nullptr;                         // p x p
  double* Rinv = nullptr;
  double* Yeig = nullptr;
  double* gram_part = nullptr;
  double* cheb_ws = nullptr;
  int* cheb_cnt = nullptr;
  double* lz_Q = nullptr;
  int64_t lz_ldq = 0;
  double* lz_w = nullptr;
  double* lz_h = nullptr;
  double* lz_part = nullptr;
  int* lz_cnt = nullptr;
  double* lz_T = nullptr;
  double* lz_theta = nullptr;
  double* lz_S = nullptr;
  double* rb_part = nullptr;
  int* rb_cnt = nullptr;
  int* shift_flag = nullptr;
  ChebGemmPlan plan;
  CUtensorMap mapB[3];
  CUtensorMap mapBfull;
  const double* mapA_ptr = nullptr;
  int64_t mapA_lda = 0;
  CUtensorMap mapA;
  ncclComm_t comm = nullptr;
  char err[512] = {0};
};

static pf_status cuda_fail(pf_ctx c, cudaError_t e, const char* where) {
  if (c) snprintf(c->err, sizeof(c->err), "%s: %s", where, cudaGetErrorString(e));
  return PF_ERR_CUDA;
}
#define PF_CU(call)                                        \
  do {                                                     \
    cudaError_t e_ = (call);                               \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call); \
  } while (0)

static bool p_supported(int p) { return p == 16 || p == 32 || p == 64 || p == 128; }
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
  }
  return "PF_ERR_UNKNOWN";
}

const char* pf_last_error(pf_ctx c) { return c ? c->err : "null context"; }
int64_t pf_local_rows(pf_ctx c) { return c ? c->n_local : -1; }
int64_t pf_row0(pf_ctx c) { return c ? c->row0 : -1; }

static pf_status alloc_all(pf_ctx ctx) {
  const int64_t n = ctx->n, nl = ctx->n_local;
  const int p = ctx->p;
  auto A = [&](void** ptr, size_t bytes) -> bool {
    return cudaMalloc(ptr, std::max<size_t>(bytes, 16)) == cudaSuccess;
  };
  bool ok = true;
  ok &= A((void**)&ctx->state, sizeof(DevState));
  for (int i = 0; i < 3; ++i) ok &= A((void**)&ctx->Y[i], (size_t)nl * p * 8);
  ok &= A((void**)&ctx->Wbuf, (size_t)nl * p * 8);
  if (ctx->world > 1) {
    ok &= A((void**)&ctx->Yfull, (size_t)n * p * 8);
    ok &= A((void**)&ctx->Vfull, (size_t)n * p * 8);
  }
  ok &= A((void**)&ctx->G, (size_t)p * p * 8);
  ok &= A((void**)&ctx->Rinv, (size_t)p * p * 8);
  ok &= A((void**)&ctx->Yeig, (size_t)p * p * 8);
  ok &= A((void**)&ctx->gram_part, (size_t)gram_blocks((int)nl, p) * p * p * 8);
  ok &= A((void**)&ctx->cheb_ws, ctx->plan.ws_doubles * 8);
  ok &= A((void**)&ctx->cheb_cnt, (size_t)(ctx->plan.mtiles + 1) * 4);
  ctx->lz_ldq = ((n + 31) / 32) * 32;
  ok &= A((void**)&ctx->lz_Q, (size_t)ctx->lz_ldq * (kMaxLanczos + 1) * 8);
  ok &= A((void**)&ctx->lz_w, (size_t)n * 8);
  ok &= A((void**)&ctx->lz_h, (size_t)2 * kMaxLanczos * 8);
  ok &= A((void**)&ctx->lz_part, (size_t)lanczos_blocks((int)nl) * kMaxLanczos * 8);
  ok &= A((void**)&ctx->lz_cnt, 16);
  ok &= A((void**)&ctx->lz_T, (size_t)kMaxLanczos * kMaxLanczos * 8);
  ok &= A((void**)&ctx->lz_theta, (size_t)kMaxLanczos * 8);
  ok &= A((void**)&ctx->lz_S, (size_t)kMaxLanczos * kMaxLanczos * 8);
  ok &= A((void**)&ctx->rb_part, (size_t)rebuild_blocks((int)nl, (int)n) * 2 * 8);
  ok &= A((void**)&ctx->rb_cnt, 16);
  ok &= A((void**)&ctx->shift_flag, 16);
  if (!ok) {
    snprintf(ctx->err, sizeof(ctx->err), "cudaMalloc of scratch failed");
    return PF_ERR_NOMEM;
  }
  PF_CU(cudaMemset(ctx->state, 0, sizeof(DevState)));
  PF_CU(cudaMemset(ctx->cheb_cnt, 0, (size_t)(ctx->plan.mtiles + 1) * 4));
  PF_CU(cudaMemset(ctx->lz_cnt, 0, 16));
  PF_CU(cudaMemset(ctx->rb_cnt, 0, 16));
  PF_CU(cudaMemset(ctx->shift_flag, 0, 16));
  const double rr[3] = {1.0, 0.0, 0.0};
  PF_CU(cudaMemcpy(&ctx->state->coef_rr[0], rr, sizeof(rr), cudaMemcpyHostToDevice));
  // TMA descriptors of the internal B operands
  if (ctx->world == 1) {
    for (int i = 0; i < 3; ++i)
      if (!encode_map_B(&ctx->mapB[i], ctx->Y[i], p, (int)n)) {
        snprintf(ctx->err, sizeof(ctx->err), "cuTensorMapEncodeTiled(B) failed");
        return PF_ERR_CUDA;
      }
  } else {
    if (!encode_map_B(&ctx->mapBfull, ctx->Yfull, p, (int)n)) {
      snprintf(ctx->err, sizeof(ctx->err), "cuTensorMapEncodeTiled(B) failed");
      return PF_ERR_CUDA;
    }
  }
  PF_CU(cudaDeviceSynchronize());
  return PF_OK;
}

static pf_status create_common(int64_t n, int32_t p, int32_t degree, pf_dtype dtype, int rank,
                               int world, pf_ctx* out) {
  if (!out) return PF_ERR_ARG;
  *out = nullptr;
  if (dtype != PF_FP64) return PF_ERR_UNSUPPORTED;
  if (degree < 1 || degree > kMaxDeg) return PF_ERR_ARG;
  if (!p_supported(p) || n < p || n > (int64_t)1 << 30) return PF_ERR_DIM;
  if (world < 1 || rank < 0 || rank >= world) return PF_ERR_ARG;
  pf_ctx ctx = new (std::nothrow) pf_ctx_s();
  if (!ctx) return PF_ERR_NOMEM;
  ctx->n = n;
  ctx->p = p;
  ctx->d = degree;
  ctx->rank = rank;
  ctx->world = world;
  ctx->row0 = (int64_t)rank * n / world;
  ctx->n_local = (int64_t)(rank + 1) * n / world - ctx->row0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) {
    pf_status s = cuda_fail(ctx, e, "cudaGetDevice");
    delete ctx;
    return s;
  }
  ctx->plan = cheb_gemm_plan(p, (int)ctx->n_local, (int)n, ctx->num_sms);
  pf_status s = alloc_all(ctx);
  if (s != PF_OK) {
    fprintf(stderr, "pf_create: %s\n", ctx->err);
    pf_destroy(ctx);
    return s;
  }
  *out = ctx;
  return PF_OK;
}

pf_status pf_create(int64_t n, int32_t p, int32_t degree, pf_dtype dtype, pf_ctx* out) {
  return create_common(n, p, degree, dtype, 0, 1, out);
}

pf_status pf_create_dist(int64_t n, int32_t p, int32_t degree, pf_dtype dtype,
                         const void* nccl_id, int32_t rank, int32_t world, pf_ctx* out) {
  if (world == 1) return create_common(n, p, degree, dtype, 0, 1, out);
  if (!nccl_id) return PF_ERR_ARG;
  pf_status s = create_common(n, p, degree, dtype, rank, world, out);
  if (s != PF_OK) return s;
  ncclUniqueId id;
  memcpy(&id, nccl_id, sizeof(id));
  ncclResult_t r = ncclCommInitRank(&(*out)->comm, world, id, rank);
  if (r != ncclSuccess) {
    snprintf((*out)->err, sizeof((*out)->err), "ncclCommInitRank: %s", ncclGetErrorString(r));
    pf_destroy(*out);
    *out = nullptr;
    return PF_ERR_NCCL;
  }
  return PF_OK;
}

long long pf_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

pf_status pf_diagnostics(pf_ctx ctx, pf_stream stream, double* diag) {
  if (!ctx || !diag) return PF_ERR_ARG;
  PF_CU(cudaStreamSynchronize((cudaStream_t)stream));
  DevState h;
  PF_CU(cudaMemcpy(&h, ctx->state, sizeof(DevState), cudaMemcpyDeviceToHost));
  diag[0] = h.scratch[1];
  diag[1] = (double)h.lanczos_steps;
  return PF_OK;
}

pf_status pf_profile(pf_ctx ctx, int32_t enable) {
  if (!ctx) return PF_ERR_ARG;
  if (enable && ctx->ev.empty()) {
    ctx->ev.resize(8192);
    for (auto& e : ctx->ev) PF_CU(cudaEventCreate(&e));
  }
  ctx->prof = enable != 0;
  ctx->ev_used = 0;
  ctx->prof_dropped = 0;
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

pf_status pf_destroy(pf_ctx ctx) {
  if (!ctx) return PF_ERR_ARG;
  for (auto e : ctx->ev) cudaEventDestroy(e);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  void* ptrs[] = {ctx->state, ctx->Y[0], ctx->Y[1], ctx->Y[2], ctx->Yfull, ctx->Wbuf,
                  ctx->Vfull, ctx->G, ctx->Rinv, ctx->Yeig, ctx->gram_part, ctx->cheb_ws,
                  ctx->cheb_cnt, ctx->lz_Q, ctx->lz_w, ctx->lz_h, ctx->lz_part, ctx->lz_cnt,
                  ctx->lz_T, ctx->lz_theta, ctx->lz_S, ctx->rb_part, ctx->rb_cnt, ctx->shift_flag};
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
  PF_CU(cudaMemset(&ctx->state->flags, 0, sizeof(unsigned int)));
  PF_CU(cudaMemset(&ctx->state->rebases, 0, sizeof(int)));
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

// Gather the local rows of `loc` (n_local x p) into ctx->Yfull (n x p) across ranks.
static pf_status gather(pf_ctx ctx, const double* loc, double* full, cudaStream_t st) {
  if (ctx->world == 1) return PF_OK;
  // rows are split as floor(g n / world): use the equal-size fast path when divisible
  const int64_t n = ctx->n, p = ctx->p;
  if (n % ctx->world == 0) {
    ncclResult_t r = ncclAllGather(loc, full, (size_t)ctx->n_local * p, ncclDouble, ctx->comm, st);
    if (r != ncclSuccess) {
      snprintf(ctx->err, sizeof(ctx->err), "ncclAllGather: %s", ncclGetErrorString(r));
      return PF_ERR_NCCL;
    }
    return PF_OK;
  }
  ncclGroupStart();
  for (int g = 0; g < ctx->world; ++g) {
    const int64_t r0 = (int64_t)g * n / ctx->world, r1 = (int64_t)(g + 1) * n / ctx->world;
    ncclBroadcast(g == ctx->rank ? loc : full + r0 * p, full + r0 * p, (size_t)(r1 - r0) * p,
                  ncclDouble, g, ctx->comm, st);
  }
  ncclResult_t r = ncclGroupEnd();
  if (r != ncclSuccess) {
    snprintf(ctx->err, sizeof(ctx->err), "ncclBroadcast group: %s", ncclGetErrorString(r));
    return PF_ERR_NCCL;
  }
  return PF_OK;
}

static pf_status allreduce(pf_ctx ctx, double* buf, size_t count, cudaStream_t st) {
  if (ctx->world == 1) return PF_OK;
  ncclResult_t r = ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, ctx->comm, st);
  if (r != ncclSuccess) {
    snprintf(ctx->err, sizeof(ctx->err), "ncclAllReduce: %s", ncclGetErrorString(r));
    return PF_ERR_NCCL;
  }
  return PF_OK;
}

// One Chebyshev step / plain product: out = coef * (A B) + ..., B = Y[bidx] (all rows).
static pf_status gemm_step(pf_ctx ctx, int bidx, const double* ycur, const double* yprev,
                           double* out, const double* coef, cudaStream_t st) {
  const CUtensorMap* mb;
  if (ctx->world == 1) {
    mb = &ctx->mapB[bidx];
  } else {
    pf_status s = gather(ctx, ctx->Y[bidx], ctx->Yfull, st);
    if (s != PF_OK) return s;
    mb = &ctx->mapBfull;
  }
  const bool rec = ctx->prof && ctx->ev_used + 2 <= ctx->ev.size();
  if (ctx->prof && !rec) ++ctx->prof_dropped;
  if (rec) PF_CU(cudaEventRecord(ctx->ev[ctx->ev_used], st));
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

// One CholeskyQR pass on Y (in place); cond: only if *cond != 0.
static pf_status chol_pass(pf_ctx ctx, double* Y, int* shift_out, const int* cond,
                           cudaStream_t st) {
  pf_status s = gram_all(ctx, Y, Y, ctx->G, cond, st);
  if (s != PF_OK) return s;
  PF_CU(chol_inv_launch(ctx->G, ctx->p, ctx->n, ctx->Rinv, ctx->state, shift_out, cond, st));
  PF_CU(rmul_launch(Y, ctx->p, ctx->Rinv, Y, ctx->p, (int)ctx->n_local, ctx->p, cond, st));
  return PF_OK;
}

// CholeskyQR2, plus a third pass when either pass had to shift (shifted CholeskyQR3).
static pf_status orth_internal(pf_ctx ctx, double* Y, cudaStream_t st) {
  PF_CU(cudaMemsetAsync(ctx->shift_flag, 0, sizeof(int), st));
  pf_status s = chol_pass(ctx, Y, ctx->shift_flag, nullptr, st);
  if (s == PF_OK) s = chol_pass(ctx, Y, ctx->shift_flag, nullptr, st);
  if (s == PF_OK) s = chol_pass(ctx, Y, nullptr, ctx->shift_flag, st);
  return s;
}

// ------------------------------------------------------------------------------ ABI
pf_status pf_lanczos(pf_ctx ctx, const double* A, int64_t lda, const double* v0, int32_t m,
                     double* lo_hi, pf_stream stream) {
  if (!ctx || !v0 || !lo_hi) return PF_ERR_ARG;
  if (m < 1 || m > kMaxLanczos) return PF_ERR_ARG;
  pf_status s = check_A(ctx, A, lda);
  if (s != PF_OK) return s;
  if (ctx->world > 1) return PF_ERR_UNSUPPORTED;  // distributed Lanczos: NEXT
  cudaStream_t st = (cudaStream_t)stream;
  const int n = (int)ctx->n;
  m = (int32_t)std::min<int64_t>(m, ctx->n);
  PF_CU(lanczos_init_launch(v0, n, ctx->lz_Q, ctx->lz_part, ctx->lz_cnt, ctx->state, st));
  for (int j = 0; j < m; ++j)
    PF_CU(lanczos_step_launch(A, lda, n, ctx->lz_ldq, j, ctx->lz_Q, ctx->lz_w, ctx->lz_h,
                              ctx->lz_part, ctx->lz_cnt, ctx->state, st));
  PF_CU(lanczos_finish_launch(m, ctx->lz_T, ctx->lz_theta, ctx->lz_S, lo_hi, ctx->state, st));
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

pf_status pf_orth(pf_ctx ctx, double* U, int64_t ldu, pf_stream stream) {
  if (!ctx || !U) return PF_ERR_ARG;
  if (ldu < ctx->p) return PF_ERR_DIM;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t row = (size_t)ctx->p * 8;
  PF_CU(cudaMemcpy2DAsync(ctx->Y[0], row, U, ldu * 8, row, ctx->n_local, cudaMemcpyDeviceToDevice, st));
  pf_status s = orth_internal(ctx, ctx->Y[0], st);
  if (s != PF_OK) return s;
  PF_CU(cudaMemcpy2DAsync(U, ldu * 8, ctx->Y[0], row, row, ctx->n_local, cudaMemcpyDeviceToDevice, st));
  return PF_OK;
}

pf_status pf_filter(pf_ctx ctx, const double* A, int64_t lda, double* U, int64_t ldu,
                    const double* interval, int32_t q, double rho_max, pf_stream stream) {
  if (!ctx || !U || !interval) return PF_ERR_ARG;
  if (q < 1 || q > 10 || !(rho_max > 1.0)) return PF_ERR_ARG;
  if (ldu < ctx->p) return PF_ERR_DIM;
  pf_status s = check_A(ctx, A, lda);
  if (s != PF_OK) return s;
  s = map_A(ctx, A, lda);
  if (s != PF_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  const int p = ctx->p, d = ctx->d;
  const int nl = (int)ctx->n_local;
  const size_t row = (size_t)p * 8;
  PF_CU(plan_launch(interval, d, rho_max, p, ctx->state, st));
  PF_CU(cudaMemcpy2DAsync(ctx->Y[0], row, U, ldu * 8, row, nl, cudaMemcpyDeviceToDevice, st));
  int cur = 0, prev = -1;
  for (int rep = 0; rep < q; ++rep) {
    prev = -1;
    for (int j = 0; j < d; ++j) {
      const int out = (prev < 0) ? (cur + 1) % 3 : 3 - cur - prev;
      const double* coef = &ctx->state->coef[j][0];
      s = gemm_step(ctx, cur, ctx->Y[cur], prev < 0 ? ctx->Y[cur] : ctx->Y[prev], ctx->Y[out],
                    coef, st);
      if (s != PF_OK) return s;
      prev = cur;
      cur = out;
      if (j + 1 < d) {
        // span-exact re-base of (Y_j, Y_{j-1}) when the plan asks for it (device flag)
        const int* cond = &ctx->state->rebase[j];
        s = gram_all(ctx, ctx->Y[cur], ctx->Y[cur], ctx->G, cond, st);
        if (s != PF_OK) return s;
        PF_CU(chol_inv_launch(ctx->G, p, ctx->n, ctx->Rinv, ctx->state, nullptr, cond, st));
        PF_CU(rmul_launch(ctx->Y[cur], p, ctx->Rinv, ctx->Y[cur], p, nl, p, cond, st));
        PF_CU(rmul_launch(ctx->Y[prev], p, ctx->Rinv, ctx->Y[prev], p, nl, p, cond, st));
      }
    }
  }
  s = orth_internal(ctx, ctx->Y[cur], st);
  if (s != PF_OK) return s;
  PF_CU(cudaMemcpy2DAsync(U, ldu * 8, ctx->Y[cur], row, row, nl, cudaMemcpyDeviceToDevice, st));
  return PF_OK;
}

pf_status pf_rayleigh_ritz(pf_ctx ctx, const double* A, int64_t lda, const double* U,
                           int64_t ldu, double* V, int64_t ldv, double* theta, pf_stream stream) {
  if (!ctx || !U || !V || !theta) return PF_ERR_ARG;
  if (ldu < ctx->p || ldv < ctx->p || (ldv & 1) || !aligned16(V)) return PF_ERR_DIM;
  pf_status s = check_A(ctx, A, lda);
  if (s != PF_OK) return s;
  s = map_A(ctx, A, lda);
  if (s != PF_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  const int p = ctx->p, nl = (int)ctx->n_local;
  const size_t row = (size_t)p * 8;
  PF_CU(cudaMemcpy2DAsync(ctx->Y[0], row, U, ldu * 8, row, nl, cudaMemcpyDeviceToDevice, st));
  s = gemm_step(ctx, 0, ctx->Y[0], ctx->Y[0], ctx->Wbuf, &ctx->state->coef_rr[0], st);
  if (s != PF_OK) return s;
  s = gram_all(ctx, ctx->Y[0], ctx->Wbuf, ctx->G, nullptr, st);  // H = Q^T (A Q)
  if (s != PF_OK) return s;
  PF_CU(jacobi_launch(ctx->G, p, nullptr, theta, ctx->Yeig, ctx->state, 1e-15, 40, st));
  PF_CU(copy_theta_launch(theta, p, ctx->state, st));
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
  if (ctx->world == 1) {
    *Vf = V;
    *ldf = ldv;
    return PF_OK;
  }
  const size_t row = (size_t)ctx->p * 8;
  PF_CU(cudaMemcpy2DAsync(ctx->Wbuf, row, V, ldv * 8, row, ctx->n_local, cudaMemcpyDeviceToDevice, st));
  pf_status s = gather(ctx, ctx->Wbuf, ctx->Vfull, st);
  *Vf = ctx->Vfull;
  *ldf = ctx->p;
  return s;
}

pf_status pf_prox_step(pf_ctx ctx, const double* V, int64_t ldv, const double* f, double tau,
                       const uint32_t* omega, int64_t ldo, const double* W, int64_t ldw,
                       int32_t r, double* A_out, int64_t lda_out, double* obj,
                       pf_stream stream) {
  if (!ctx || !V || !f || !omega || !A_out || !obj) return PF_ERR_ARG;
  if (r < 0 || r > 64 || (r > 0 && !W)) return PF_ERR_ARG;
  if (ldv < ctx->p || ldo < (ctx->n + 31) / 32 || lda_out < ctx->n || (r > 0 && ldw < r))
    return PF_ERR_DIM;
  cudaStream_t st = (cudaStream_t)stream;
  const double* Vf;
  int64_t ldf;
  pf_status s = full_V(ctx, V, ldv, &Vf, &ldf, st);
  if (s != PF_OK) return s;
  PF_CU(prox_launch(Vf, ldf, f, tau, omega, ldo, W, ldw, r, A_out, lda_out, (int)ctx->n_local,
                    (int)ctx->n, (int)ctx->row0, ctx->p, obj, ctx->rb_part, ctx->rb_cnt, st));
  if (ctx->world > 1) {
    // obj[0] is a sum over row blocks; obj[1] (sum |f|) is replicated
    s = allreduce(ctx, obj, 1, st);
  }
  return s;
}

pf_status pf_admm_step(pf_ctx ctx, const double* V, int64_t ldv, const double* f, double t,
                       const uint32_t* adj, int64_t ldadj, const double* deg, double* Z,
                       int64_t ldz, double* obj, pf_stream stream) {
  if (!ctx || !V || !f || !adj || !deg || !Z || !obj) return PF_ERR_ARG;
  if (ldv < ctx->p || ldadj < (ctx->n + 31) / 32 || ldz < ctx->n) return PF_ERR_DIM;
  cudaStream_t st = (cudaStream_t)stream;
  const double* Vf;
  int64_t ldf;
  pf_status s = full_V(ctx, V, ldv, &Vf, &ldf, st);
  if (s != PF_OK) return s;
  PF_CU(admm_launch(Vf, ldf, f, t, adj, ldadj, deg, Z, ldz, (int)ctx->n_local, (int)ctx->n,
                    (int)ctx->row0, ctx->p, obj, ctx->rb_part, ctx->rb_cnt, st));
  if (ctx->world > 1) {
    // <C,W> sums over blocks; the residual is a norm: reduce its square
    // (the kernel returns sqrt of the local sum; NEXT: return squares and sqrt after reduce)
    s = allreduce(ctx, obj, 1, st);
  }
  return s;
}

pf_status pf_perturb(pf_ctx ctx, double* A, int64_t lda, const double* E, int64_t lde,
                     pf_stream stream) {
  if (!ctx || !A || !E) return PF_ERR_ARG;
  if (lda < ctx->n || lde < ctx->n) return PF_ERR_DIM;
  PF_CU(perturb_launch(A, lda, E, lde, (int)ctx->n_local, (int)ctx->n, (cudaStream_t)stream));
  return PF_OK;
}

}  // extern "C"
