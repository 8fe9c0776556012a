// dist.cuh — communicator interface of the distributed power iteration
// (SURVEY.md §8(a) a8, §8(e)). Two implementations live in dist.cu:
//   * NcclComm  — one process per GPU, NCCL (dlopen'd) over NVLink/NVSwitch;
//   * LocalComm — W ranks driven by W host threads of ONE process (one or
//     several devices), collectives done with stream-ordered copies between
//     the ranks' buffers and a host barrier. It runs the exact same loop and
//     stream/event schedule as the NCCL path, so the multi-rank logic
//     (interior/halo overlap, halo exchange) is exercised on a single GPU.
// Every collective is stream-ordered on the stream passed in; buffers are
// device pointers.
#pragma once
#include <vector>

#include "handle.cuh"

namespace spmv {

struct P2P {
  int peer;
  void* ptr;
  size_t bytes;
};

struct CommBase {
  int rank = 0, world = 1, device = 0;
  virtual ~CommBase() = default;
  virtual const char* kind() const = 0;
  // true when collectives run as kernels on the SMs (NCCL): the overlapped
  // interior SpMV then leaves a few SMs free for them.
  virtual bool uses_sms() const = 0;
  // buf[0..n) <- Σ over ranks (rank order for LocalComm).
  virtual void allreduce_f64(double* buf, size_t n, cudaStream_t s) = 0;
  // In place: rank r's chunk is buf[r·chunk_bytes, (r+1)·chunk_bytes); on
  // return every chunk holds its owner's bytes.
  virtual void allgather_inplace(void* buf, size_t chunk_bytes, cudaStream_t s) = 0;
  // Grouped point-to-point: every send (peer, ptr, bytes) is matched with the
  // peer's recv from this rank (in list order per peer pair).
  virtual void exchange(const std::vector<P2P>& sends, const std::vector<P2P>& recvs, cudaStream_t s) = 0;
  // Mark the group failed so peers blocked in a collective give up (LocalComm).
  virtual void abort() {}
};

inline CommBase* as_comm(void* c) { return static_cast<CommBase*>(c); }

// dist.cu: W in-process communicators sharing one group (devices[r] per rank).
std::vector<CommBase*> local_group(int world, const int* devices);

}  // namespace spmv
