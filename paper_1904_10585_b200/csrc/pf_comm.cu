// pf_comm.cu -- NCCL and in-process loopback backends of the row-block split's exchange steps
// (pf_comm.cuh; per Chebyshev step an all-gather of Y_j, per Gram / H matrix and
// per scalar objective an all-reduce).
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>

#include "../../include/pf.h"
#include "pf_comm.cuh"
#include "pf_kernels.cuh"

namespace pf {

// ------------------------------------------------------------------------------------ NCCL
struct NcclComm final : Comm {
  ncclComm_t c = nullptr;
  ~NcclComm() override {
    if (c) ncclCommDestroy(c);
  }
  int fail(ncclResult_t r, const char* where) {
    snprintf(err, 512, "%s: %s", where, ncclGetErrorString(r));
    return PF_ERR_NCCL;
  }
  int allgatherv(const void* loc, void* full, const size_t* off, cudaStream_t st) override {
    const size_t b0 = off[1] - off[0];
    bool equal = true;
    for (int g = 0; g < world; ++g) equal &= (off[g + 1] - off[g] == b0) && off[g] == g * b0;
    if (equal) {
      ncclResult_t r = ncclAllGather(loc, full, b0, ncclChar, c, st);
      return r == ncclSuccess ? PF_OK : fail(r, "ncclAllGather");
    }
    // ragged row split: one broadcast per owner inside a group
    ncclGroupStart();
    for (int g = 0; g < world; ++g) {
      char* dst = static_cast<char*>(full) + off[g];
      ncclBroadcast(g == rank ? loc : dst, dst, off[g + 1] - off[g], ncclChar, g, c, st);
    }
    ncclResult_t r = ncclGroupEnd();
    return r == ncclSuccess ? PF_OK : fail(r, "ncclBroadcast group");
  }
  int allreduce_sum(double* buf, size_t count, cudaStream_t st) override {
    ncclResult_t r = ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, c, st);
    return r == ncclSuccess ? PF_OK : fail(r, "ncclAllReduce");
  }
  // ring of point-to-point steps: at step s every rank sends its slab to rank + s and receives
  // rank - s's, so slab rank - s arrives at step s (one NCCL launch per step, event after it)
  int allgather_slabs(const void* loc, void* full, size_t bytes, cudaStream_t st,
                      cudaEvent_t* arrived) override {
    char* f = static_cast<char*>(full);
    if (cudaMemcpyAsync(f + (size_t)rank * bytes, loc, bytes, cudaMemcpyDeviceToDevice, st) !=
            cudaSuccess ||
        cudaEventRecord(arrived[rank], st) != cudaSuccess) {
      snprintf(err, 512, "allgather_slabs: local slab copy failed");
      return PF_ERR_CUDA;
    }
    for (int s = 1; s < world; ++s) {
      const int to = (rank + s) % world, from = (rank - s + world) % world;
      ncclGroupStart();
      ncclSend(loc, bytes, ncclChar, to, c, st);
      ncclRecv(f + (size_t)from * bytes, bytes, ncclChar, from, c, st);
      ncclResult_t r = ncclGroupEnd();
      if (r != ncclSuccess) return fail(r, "ncclSend/ncclRecv");
      if (cudaEventRecord(arrived[from], st) != cudaSuccess) {
        snprintf(err, 512, "allgather_slabs: cudaEventRecord failed");
        return PF_ERR_CUDA;
      }
    }
    return PF_OK;
  }
};

Comm* comm_nccl_create(const void* nccl_id, int rank, int world, char* err, int* status) {
  NcclComm* c = new (std::nothrow) NcclComm();
  if (!c) {
    *status = PF_ERR_NOMEM;
    return nullptr;
  }
  c->rank = rank;
  c->world = world;
  c->err = err;
  ncclUniqueId id;
  memcpy(&id, nccl_id, sizeof(id));
  ncclResult_t r = ncclCommInitRank(&c->c, world, id, rank);
  if (r != ncclSuccess) {
    snprintf(err, 512, "ncclCommInitRank: %s", ncclGetErrorString(r));
    c->c = nullptr;
    delete c;
    *status = PF_ERR_NCCL;
    return nullptr;
  }
  *status = PF_OK;
  return c;
}

// ------------------------------------------------------------------------------------ loopback
constexpr int kMaxLoop = 16;

struct LoopHub {
  int world = 1;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  int timeout_s = 300;  // rendezvous timeout (PF_LOOP_TIMEOUT_S at pf_loop_create)
  unsigned long long gen = 0;
  bool abort = false;
  // slot[phase & 1][rank]: what a rank publishes before arriving at the barrier of `phase`.
  // A rank rewrites the same parity only two barriers later, after every peer has passed the
  // barrier in between -- i.e. after every peer has read this phase's slots.
  struct Slot {
    const void* src;
    cudaEvent_t ev;
  } slot[2][kMaxLoop];
};

LoopHub* loop_hub_create(int world) {
  if (world < 1 || world > kMaxLoop) return nullptr;
  LoopHub* h = new (std::nothrow) LoopHub();
  if (!h) return nullptr;
  h->world = world;
  if (const char* e = getenv("PF_LOOP_TIMEOUT_S")) h->timeout_s = std::max(1, atoi(e));
  return h;
}
void loop_hub_destroy(LoopHub* h) { delete h; }
int loop_hub_world(const LoopHub* h) { return h ? h->world : 0; }

struct Ptrs {
  const double* p[kMaxLoop];
};

// out[i] = sum_{g = 0..W-1} buf_g[i], in rank order (the same bits on every rank)
__global__ void loop_sum_kernel(Ptrs P, int W, double* __restrict__ out, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    double s = P.p[0][i];
    for (int g = 1; g < W; ++g) s += P.p[g][i];
    out[i] = s;
  }
}

struct LoopComm final : Comm {
  LoopHub* hub = nullptr;
  cudaEvent_t ready = nullptr, done = nullptr;
  double* tmp = nullptr;  // all-reduce result before it overwrites buf
  size_t tmp_count = 0;
  unsigned long long phase = 0;  // barriers passed by this rank
  ~LoopComm() override {
    if (ready) cudaEventDestroy(ready);
    if (done) cudaEventDestroy(done);
    if (tmp) cudaFree(tmp);
  }
  int fail(const char* what) {
    snprintf(err, 512, "loopback: %s", what);
    std::lock_guard<std::mutex> lk(hub->m);
    hub->abort = true;  // peers waiting in a rendezvous fail instead of timing out
    hub->cv.notify_all();
    return PF_ERR_NCCL;
  }
  int cuda(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return PF_OK;
    snprintf(err, 512, "loopback %s: %s", where, cudaGetErrorString(e));
    return PF_ERR_CUDA;
  }
  // publish (src, ev) for this phase, wait for every rank; false on timeout / abort
  bool rendezvous(const void* src, cudaEvent_t ev) {
    std::unique_lock<std::mutex> lk(hub->m);
    LoopHub::Slot& s = hub->slot[phase & 1][rank];
    s.src = src;
    s.ev = ev;
    ++phase;
    if (hub->abort) return false;
    const unsigned long long g = hub->gen;
    if (++hub->arrived == hub->world) {
      hub->arrived = 0;
      ++hub->gen;
      hub->cv.notify_all();
      return true;
    }
    const bool ok = hub->cv.wait_for(lk, std::chrono::seconds(hub->timeout_s),
                                     [&] { return hub->gen != g || hub->abort; });
    if (!ok || hub->abort) {
      hub->abort = true;  // a peer failed or hung: every later collective fails fast
      hub->cv.notify_all();
      return false;
    }
    // (the failing path returns false without holding the caller in fail(): the lock is
    // released when lk goes out of scope before fail() takes it)
    return true;
  }
  const LoopHub::Slot& peer(int g) const { return hub->slot[(phase - 1) & 1][g]; }

  // second half of every collective: no rank continues (and may overwrite what it lent out)
  // before every peer's reads of it are done on the device
  int finish(cudaStream_t st) {
    int r = cuda(cudaEventRecord(done, st), "cudaEventRecord");
    if (r != PF_OK) return r;
    if (!rendezvous(nullptr, done)) return fail("collective timed out or a peer failed");
    for (int g = 0; g < world; ++g)
      if (g != rank) {
        r = cuda(cudaStreamWaitEvent(st, peer(g).ev, 0), "cudaStreamWaitEvent");
        if (r != PF_OK) return r;
      }
    return PF_OK;
  }

  int allgatherv(const void* loc, void* full, const size_t* off, cudaStream_t st) override {
    int r = cuda(cudaEventRecord(ready, st), "cudaEventRecord");
    if (r != PF_OK) return r;
    if (!rendezvous(loc, ready)) return fail("collective timed out or a peer failed");
    for (int g = 0; g < world; ++g) {
      char* dst = static_cast<char*>(full) + off[g];
      const size_t bytes = off[g + 1] - off[g];
      const void* src = g == rank ? loc : peer(g).src;
      if (g != rank) {
        r = cuda(cudaStreamWaitEvent(st, peer(g).ev, 0), "cudaStreamWaitEvent");
        if (r != PF_OK) return r;
      }
      if (bytes && src != dst) {
        r = cuda(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st), "cudaMemcpyAsync");
        if (r != PF_OK) return r;
      }
    }
    return finish(st);
  }

  int allgather_slabs(const void* loc, void* full, size_t bytes, cudaStream_t st,
                      cudaEvent_t* arrived) override {
    int r = cuda(cudaEventRecord(ready, st), "cudaEventRecord");
    if (r != PF_OK) return r;
    if (!rendezvous(loc, ready)) return fail("collective timed out or a peer failed");
    char* f = static_cast<char*>(full);
    for (int s = 0; s < world; ++s) {  // the NCCL ring's arrival order
      const int g = (rank - s + world) % world;
      const void* src = g == rank ? loc : peer(g).src;
      if (g != rank) {
        r = cuda(cudaStreamWaitEvent(st, peer(g).ev, 0), "cudaStreamWaitEvent");
        if (r != PF_OK) return r;
      }
      r = cuda(cudaMemcpyAsync(f + (size_t)g * bytes, src, bytes, cudaMemcpyDeviceToDevice, st),
               "cudaMemcpyAsync");
      if (r != PF_OK) return r;
      r = cuda(cudaEventRecord(arrived[g], st), "cudaEventRecord");
      if (r != PF_OK) return r;
    }
    return finish(st);
  }

  int allreduce_sum(double* buf, size_t count, cudaStream_t st) override {
    if (count > tmp_count) return fail("all-reduce larger than the scratch sized at create");
    int r = cuda(cudaEventRecord(ready, st), "cudaEventRecord");
    if (r != PF_OK) return r;
    if (!rendezvous(buf, ready)) return fail("collective timed out or a peer failed");
    Ptrs P{};
    for (int g = 0; g < world; ++g) {
      P.p[g] = static_cast<const double*>(g == rank ? buf : peer(g).src);
      if (g != rank) {
        r = cuda(cudaStreamWaitEvent(st, peer(g).ev, 0), "cudaStreamWaitEvent");
        if (r != PF_OK) return r;
      }
    }
    if (count) {
      count_launch();
      const int grid = (int)std::min<size_t>((count + 255) / 256, 1024);
      loop_sum_kernel<<<grid, 256, 0, st>>>(P, world, tmp, count);
      r = cuda(cudaGetLastError(), "loop_sum_kernel");
      if (r != PF_OK) return r;
    }
    r = finish(st);
    if (r != PF_OK || !count) return r;
    return cuda(cudaMemcpyAsync(buf, tmp, count * 8, cudaMemcpyDeviceToDevice, st),
                "cudaMemcpyAsync");
  }
};

Comm* comm_loop_create(LoopHub* hub, int rank, size_t max_reduce, char* err, int* status) {
  LoopComm* c = new (std::nothrow) LoopComm();
  if (!c) {
    *status = PF_ERR_NOMEM;
    return nullptr;
  }
  c->hub = hub;
  c->rank = rank;
  c->world = hub->world;
  c->err = err;
  c->tmp_count = max_reduce;
  if (cudaEventCreateWithFlags(&c->ready, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming) != cudaSuccess ||
      cudaMalloc(&c->tmp, std::max<size_t>(max_reduce, 1) * 8) != cudaSuccess) {
    snprintf(err, 512, "loopback: event / scratch creation failed");
    delete c;
    *status = PF_ERR_NOMEM;
    return nullptr;
  }
  *status = PF_OK;
  return c;
}

}  // namespace pf
