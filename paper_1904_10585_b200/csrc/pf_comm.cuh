// pf_comm.cuh -- the exchange steps of the row-block split (include/pf.h
// pf_create_dist / pf_create_loop) behind one interface with two backends:
//
//  * NCCL (one process per GPU, NVLink / NVSwitch): ncclAllGather / grouped ncclBroadcast for
//    ragged row blocks, ncclAllReduce(sum).
//  * loopback (W contexts in one process, one host thread and one stream each, on ONE GPU --
//    the test harness for the multi-rank paths when only one GPU is available): a collective is
//    a host rendezvous of the W calls, then stream-ordered device work only --
//    all-gather = cudaStreamWaitEvent on every peer's "block ready" event + one cudaMemcpyAsync
//    per peer slab; all-reduce = one fixed-order (rank 0, 1, ..., W-1) sum kernel over the W
//    peer buffers, so every rank receives identical bits; a second rendezvous exchanges "done
//    reading" events so no rank overwrites a buffer a peer still reads.  No kernel ever waits
//    on another kernel (device-side waits are stream/event waits only).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace pf {

struct LoopHub;  // shared by the W loopback contexts (pf_loop_create)

struct Comm {
  int rank = 0, world = 1;
  char* err = nullptr;  // the owning context's error buffer (512 bytes)
  virtual ~Comm() = default;
  // rank g's `loc` (off[g+1] - off[g] bytes) lands at full + off[g] on every rank
  virtual int allgatherv(const void* loc, void* full, const size_t* off, cudaStream_t st) = 0;
  // buf <- sum over ranks (fp64); identical bits on every rank
  virtual int allreduce_sum(double* buf, size_t count, cudaStream_t st) = 0;
  // Equal slabs, one at a time, for a consumer that overlaps them: rank
  // g's `loc` (bytes) lands at full + g bytes; enqueued on `st` (the communication stream) in the
  // fixed order g = rank, rank - 1, ..., rank - W + 1 (mod W), and arrived[g] is recorded on `st`
  // right after slab g landed.  The caller orders its reuse of `loc` and `full` after `st`.
  virtual int allgather_slabs(const void* loc, void* full, size_t bytes, cudaStream_t st,
                              cudaEvent_t* arrived) = 0;
};

// the return value of the methods is a pf_status (PF_OK = 0)
Comm* comm_nccl_create(const void* nccl_id, int rank, int world, char* err, int* status);
// max_reduce: the largest all-reduce (doubles) this context issues (scratch allocated here)
Comm* comm_loop_create(LoopHub* hub, int rank, size_t max_reduce, char* err, int* status);

LoopHub* loop_hub_create(int world);
void loop_hub_destroy(LoopHub* hub);
int loop_hub_world(const LoopHub* hub);

}  // namespace pf
