// dist.cu — native power-iteration driver and the NCCL exchange
// (SURVEY.md §8(a) a8, §8(e)). The whole E-step loop runs in C++ on the
// handle's stream: per step one SpMV kernel with the fused norm epilogue,
// then (multi-GPU) ncclAllReduce of the two partial sums and ncclAllGather of
// the row slab into the replicated x — no per-iteration Python.
// NCCL is loaded lazily with dlopen("libnccl.so.2") so the library has no
// link-time NCCL dependency (single-GPU users and CPU-side tests never need it).
#include <dlfcn.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "dist.cuh"
#include "spmv_common.cuh"

namespace spmv {
namespace {

// Minimal NCCL ABI (stable across NCCL 2.x; values from nccl.h).
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
constexpr int ncclInt8 = 0, ncclFloat64 = 8, ncclSumOp = 0;

struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* l = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!l) l = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!l) return;
    api.lib = l;
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(l, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(l, "ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(l, "ncclCommDestroy");
    api.AllReduce = (decltype(api.AllReduce))dlsym(l, "ncclAllReduce");
    api.AllGather = (decltype(api.AllGather))dlsym(l, "ncclAllGather");
    api.Send = (decltype(api.Send))dlsym(l, "ncclSend");
    api.Recv = (decltype(api.Recv))dlsym(l, "ncclRecv");
    api.GroupStart = (decltype(api.GroupStart))dlsym(l, "ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))dlsym(l, "ncclGroupEnd");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(l, "ncclGetErrorString");
  });
  if (!api.lib || !api.GetUniqueId || !api.CommInitRank || !api.AllReduce || !api.AllGather || !api.Send ||
      !api.Recv || !api.GroupStart || !api.GroupEnd)
    fail(SPMV_ERR_NCCL, "libnccl.so.2 not loadable or incomplete");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != 0) {
    const char* m = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
    fail(SPMV_ERR_NCCL, std::string(what) + ": " + m);
  }
}

// ------------------------------------------------------------------ NCCL
struct NcclComm : CommBase {
  ncclComm_t c = nullptr;
  const char* kind() const override { return "nccl"; }
  bool uses_sms() const override { return world > 1; }
  void allreduce_f64(double* buf, size_t n, cudaStream_t s) override {
    nccl_check(nccl().AllReduce(buf, buf, n, ncclFloat64, ncclSumOp, c, s), "ncclAllReduce");
  }
  void allgather_inplace(void* buf, size_t chunk_bytes, cudaStream_t s) override {
    char* b = static_cast<char*>(buf);
    nccl_check(nccl().AllGather(b + (size_t)rank * chunk_bytes, b, chunk_bytes, ncclInt8, c, s), "ncclAllGather");
  }
  void exchange(const std::vector<P2P>& sends, const std::vector<P2P>& recvs, cudaStream_t s) override {
    nccl_check(nccl().GroupStart(), "ncclGroupStart");
    ncclResult_t r = 0;
    for (const P2P& p : sends)
      if (r == 0 && p.bytes) r = nccl().Send(p.ptr, p.bytes, ncclInt8, p.peer, c, s);
    for (const P2P& p : recvs)
      if (r == 0 && p.bytes) r = nccl().Recv(p.ptr, p.bytes, ncclInt8, p.peer, c, s);
    ncclResult_t e = nccl().GroupEnd();
    nccl_check(r, "ncclSend/ncclRecv");
    nccl_check(e, "ncclGroupEnd");
  }
  ~NcclComm() override {
    if (c && nccl().CommDestroy) nccl().CommDestroy(c);
  }
};

// ------------------------------------------------------------------ in-process group
constexpr size_t kLocalStage = 64;  // max doubles per local all-reduce

__global__ void k_sum_slots(const double* __restrict__ all, int world, int n, double* __restrict__ out) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double a = all[i];
    for (int q = 1; q < world; ++q) a += all[(size_t)q * n + i];  // rank order
    out[i] = a;
  }
}

struct LocalShared {
  int world = 1;
  std::vector<int> devices;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool broken = false;
  std::vector<cudaEvent_t> ev_in, ev_out;
  std::vector<void*> posted;
  std::vector<std::vector<P2P>> posted_sends;
  std::vector<double*> staging;  // per rank, on its device
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) fail(SPMV_ERR_NCCL, "local group: a peer rank failed");
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g || broken; })) {
      broken = true;
      cv.notify_all();
      fail(SPMV_ERR_NCCL, "local group: barrier timed out (a rank did not enter the collective)");
    }
    if (gen == g) fail(SPMV_ERR_NCCL, "local group: a peer rank failed");
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    broken = true;
    cv.notify_all();
  }
  ~LocalShared() {
    for (int r = 0; r < world; ++r) {
      cudaSetDevice(devices[r]);
      if (ev_in[r]) cudaEventDestroy(ev_in[r]);
      if (ev_out[r]) cudaEventDestroy(ev_out[r]);
      if (staging[r]) cudaFree(staging[r]);
    }
  }
};

struct LocalComm : CommBase {
  std::shared_ptr<LocalShared> g;
  double* gather = nullptr;  // [world][kLocalStage] on this rank's device
  const char* kind() const override { return "local"; }
  bool uses_sms() const override { return false; }
  void abort() override { g->abort(); }
  // Collective entry/exit: every rank's stream waits for every rank's entry
  // (inputs ready) and, at the end, for every rank's exit (outputs consumed),
  // like a collective that completes everywhere at once.
  void enter(cudaStream_t s) {
    CK(cudaEventRecord(g->ev_in[rank], s));
    g->barrier();
    for (int q = 0; q < world; ++q) CK(cudaStreamWaitEvent(s, g->ev_in[q], 0));
  }
  void leave(cudaStream_t s) {
    CK(cudaEventRecord(g->ev_out[rank], s));
    g->barrier();
    for (int q = 0; q < world; ++q) CK(cudaStreamWaitEvent(s, g->ev_out[q], 0));
  }
  void allreduce_f64(double* buf, size_t n, cudaStream_t s) override {
    if (n > kLocalStage) fail(SPMV_ERR_INVALID_ARG, "local group: all-reduce of more than 64 doubles");
    CK(cudaMemcpyAsync(g->staging[rank], buf, n * 8, cudaMemcpyDefault, s));
    enter(s);
    for (int q = 0; q < world; ++q)
      CK(cudaMemcpyAsync(gather + (size_t)q * n, g->staging[q], n * 8, cudaMemcpyDefault, s));
    LAUNCH(k_sum_slots, 1, 64, 0, s, (const double*)gather, world, (int)n, buf);
    leave(s);
  }
  void allgather_inplace(void* buf, size_t chunk_bytes, cudaStream_t s) override {
    g->posted[rank] = buf;
    enter(s);
    for (int q = 0; q < world; ++q)
      if (q != rank && chunk_bytes)
        CK(cudaMemcpyAsync(static_cast<char*>(buf) + (size_t)q * chunk_bytes,
                           static_cast<const char*>(g->posted[q]) + (size_t)q * chunk_bytes, chunk_bytes,
                           cudaMemcpyDefault, s));
    leave(s);
  }
  void exchange(const std::vector<P2P>& sends, const std::vector<P2P>& recvs, cudaStream_t s) override {
    g->posted_sends[rank] = sends;
    enter(s);
    std::vector<size_t> used(world, 0);
    for (const P2P& r : recvs) {
      const std::vector<P2P>& ps = g->posted_sends[r.peer];
      size_t k = used[r.peer];
      while (k < ps.size() && ps[k].peer != rank) ++k;
      if (k == ps.size()) fail(SPMV_ERR_NCCL, "local group: receive without a matching send");
      used[r.peer] = k + 1;
      if (ps[k].bytes != r.bytes) fail(SPMV_ERR_NCCL, "local group: send/receive size mismatch");
      if (r.bytes) CK(cudaMemcpyAsync(r.ptr, ps[k].ptr, r.bytes, cudaMemcpyDefault, s));
    }
    leave(s);
  }
  ~LocalComm() override {
    if (gather) {
      cudaSetDevice(device);
      cudaFree(gather);
    }
  }
};

}  // namespace

// Power iteration loop (declared in handle.cuh). z_k is written straight
// into this rank's chunk of the next replicated buffer; the all-gather is in
// place (chunk_buf is not needed).
// Device-to-device copy as a kernel: a cudaMemcpyAsync would go to a copy
// engine, where it can queue behind another stream's host upload.
__global__ void k_copy16(uint4* __restrict__ dst, const uint4* __restrict__ src, int64_t n16) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) dst[i] = src[i];
}
__global__ void k_copy1(unsigned char* __restrict__ dst, const unsigned char* __restrict__ src, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = src[i];
}
static void device_copy(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  if ((((uintptr_t)dst | (uintptr_t)src | bytes) & 15) == 0) {
    const int64_t n16 = (int64_t)(bytes / 16);
    LAUNCH(k_copy16, grid_for(n16, 256), 256, 0, s, static_cast<uint4*>(dst), static_cast<const uint4*>(src), n16);
  } else {
    LAUNCH(k_copy1, grid_for((int64_t)bytes, 256), 256, 0, s, static_cast<unsigned char*>(dst),
           static_cast<const unsigned char*>(src), (int64_t)bytes);
  }
}

void power_iterate(spmv_matrix* h, const void* x0, void* buf0, void* buf1, int64_t n_full, int64_t steps,
                   double* sums, void* comm_v, int64_t chunk, void* /*chunk_buf*/, float* kernel_ms, float* loop_ms,
                   int* final_buf) {
  cudaStream_t s = h->stream;
  CommBase* comm = as_comm(comm_v);
  const int vb = h->vbytes;
  if (x0 != buf0) device_copy(buf0, x0, (size_t)n_full * vb, s);
  const int64_t row_offset = comm ? (int64_t)comm->rank * chunk : 0;
  if (comm && (comm->rank + 1) * chunk > n_full) fail(SPMV_ERR_INVALID_ARG, "power_iterate: world·chunk > n_full");
  // S_0 = ||z_0||² over this rank's rows, then summed over ranks
  spmv_norm2_internal(h, static_cast<char*>(buf0) + row_offset * vb, h->rows, sums);
  if (comm) comm->allreduce_f64(sums, 2, s);
  std::vector<cudaEvent_t> ev;
  if (kernel_ms) {
    ev.resize(2 * (size_t)steps);
    for (auto& e : ev) CK(cudaEventCreate(&e));
  }
  cudaEvent_t l0 = nullptr, l1 = nullptr;
  if (loop_ms) {
    CK(cudaEventCreate(&l0));
    CK(cudaEventCreate(&l1));
    CK(cudaEventRecord(l0, s));
  }
  void* cur = buf0;
  void* nxt = buf1;
  for (int64_t k = 0; k < steps; ++k) {
    void* y = static_cast<char*>(nxt) + row_offset * vb;
    if (kernel_ms) CK(cudaEventRecord(ev[2 * k], s));
    power_step_internal(h, cur, y, sums + 2 * k, sums + 2 * (k + 1), row_offset);
    if (kernel_ms) CK(cudaEventRecord(ev[2 * k + 1], s));
    if (comm) {  // also at world = 1, so the collective path is testable on one GPU
      comm->allreduce_f64(sums + 2 * (k + 1), 2, s);
      comm->allgather_inplace(nxt, (size_t)chunk * vb, s);
    }
    std::swap(cur, nxt);
  }
  if (loop_ms) {
    CK(cudaEventRecord(l1, s));
    CK(cudaEventSynchronize(l1));
    CK(cudaEventElapsedTime(loop_ms, l0, l1));
    cudaEventDestroy(l0);
    cudaEventDestroy(l1);
  }
  if (final_buf) *final_buf = (cur == buf0) ? 0 : 1;
  if (kernel_ms) {
    CK(cudaEventSynchronize(ev.back()));
    for (int64_t k = 0; k < steps; ++k) CK(cudaEventElapsedTime(&kernel_ms[k], ev[2 * k], ev[2 * k + 1]));
    for (auto& e : ev) cudaEventDestroy(e);
  }
}

void* dist_init(const uint8_t id[128], int rank, int world, int device) {
  ncclUniqueId u;
  std::memcpy(u.internal, id, 128);
  NcclComm* c = new NcclComm();
  c->rank = rank;
  c->world = world;
  c->device = device;
  CK(cudaSetDevice(device));
  try {
    nccl_check(nccl().CommInitRank(&c->c, world, u, rank), "ncclCommInitRank");
  } catch (...) {
    delete c;
    throw;
  }
  return static_cast<CommBase*>(c);
}

void dist_unique_id(uint8_t out[128]) {
  ncclUniqueId u;
  nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
  std::memcpy(out, u.internal, 128);
}

void dist_destroy(void* comm) { delete as_comm(comm); }

std::vector<CommBase*> local_group(int world, const int* devices) {
  auto g = std::make_shared<LocalShared>();
  g->world = world;
  g->devices.assign(devices, devices + world);
  g->ev_in.assign(world, nullptr);
  g->ev_out.assign(world, nullptr);
  g->posted.assign(world, nullptr);
  g->posted_sends.assign(world, {});
  g->staging.assign(world, nullptr);
  std::vector<CommBase*> out;
  try {
    for (int r = 0; r < world; ++r) {
      CK(cudaSetDevice(devices[r]));
      CK(cudaEventCreateWithFlags(&g->ev_in[r], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&g->ev_out[r], cudaEventDisableTiming));
      CK(cudaMalloc(&g->staging[r], kLocalStage * sizeof(double)));
    }
    for (int r = 0; r < world; ++r) {
      LocalComm* c = new LocalComm();
      out.push_back(c);
      c->g = g;
      c->rank = r;
      c->world = world;
      c->device = devices[r];
      CK(cudaSetDevice(devices[r]));
      CK(cudaMalloc(&c->gather, (size_t)world * kLocalStage * sizeof(double)));
    }
  } catch (...) {
    for (CommBase* c : out) delete c;
    throw;
  }
  return out;
}

}  // namespace spmv
