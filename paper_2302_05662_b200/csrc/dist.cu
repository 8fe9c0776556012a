// dist.cu — native power-iteration driver and the NCCL exchange
// (SURVEY.md §8(a) a8, §8(e)). The whole E-step loop runs in C++ on the
// handle's stream: per step one SpMV kernel with the fused norm epilogue,
// then (multi-GPU) ncclAllReduce of the two partial sums and ncclAllGather of
// the row slab into the replicated x — no per-iteration Python.
// NCCL is loaded lazily with dlopen("libnccl.so.2") so the library has no
// link-time NCCL dependency (single-GPU users and CPU-side tests never need it).
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <vector>

#include "spmv_common.cuh"

namespace spmv {
namespace {

// Minimal NCCL ABI (stable across NCCL 2.x; values from nccl.h).
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
constexpr int ncclFloat32 = 7, ncclFloat64 = 8, ncclSumOp = 0;

struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
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
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(l, "ncclGetErrorString");
  });
  if (!api.lib || !api.GetUniqueId || !api.CommInitRank || !api.AllReduce || !api.AllGather)
    fail(SPMV_ERR_NCCL, "libnccl.so.2 not loadable or incomplete");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != 0) {
    const char* m = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
    fail(SPMV_ERR_NCCL, std::string(what) + ": " + m);
  }
}

struct Comm {
  ncclComm_t c = nullptr;
  int rank = 0, world = 1, device = 0;
};

}  // namespace

// Power iteration loop (declared in handle.cuh).
void power_iterate(spmv_matrix* h, const void* x0, void* buf0, void* buf1, int64_t n_full, int64_t steps,
                   double* sums, void* comm_v, int64_t chunk, void* chunk_buf, float* kernel_ms, float* loop_ms,
                   int* final_buf) {
  cudaStream_t s = h->stream;
  Comm* comm = static_cast<Comm*>(comm_v);
  const int vb = h->vbytes;
  const int dtype = h->dtype == SPMV_R64F ? ncclFloat64 : ncclFloat32;
  if (x0 != buf0) CK(cudaMemcpyAsync(buf0, x0, (size_t)n_full * vb, cudaMemcpyDeviceToDevice, s));
  const int64_t row_offset = comm ? (int64_t)comm->rank * chunk : 0;
  // S_0 = ||z_0||² over this rank's rows, then summed over ranks
  spmv_norm2_internal(h, static_cast<char*>(buf0) + row_offset * vb, h->rows, sums);
  if (comm) nccl_check(nccl().AllReduce(sums, sums, 2, ncclFloat64, ncclSumOp, comm->c, s), "ncclAllReduce");
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
    void* y = comm ? chunk_buf : nxt;
    if (kernel_ms) CK(cudaEventRecord(ev[2 * k], s));
    power_step_internal(h, cur, y, sums + 2 * k, sums + 2 * (k + 1), row_offset);
    if (kernel_ms) CK(cudaEventRecord(ev[2 * k + 1], s));
    if (comm) {  // also at world = 1, so the NCCL path is testable on one GPU
      nccl_check(nccl().AllReduce(sums + 2 * (k + 1), sums + 2 * (k + 1), 2, ncclFloat64, ncclSumOp, comm->c, s),
                 "ncclAllReduce");
      nccl_check(nccl().AllGather(chunk_buf, nxt, (size_t)chunk, dtype, comm->c, s), "ncclAllGather");
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
  Comm* c = new Comm();
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
  return c;
}

void dist_unique_id(uint8_t out[128]) {
  ncclUniqueId u;
  nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
  std::memcpy(out, u.internal, 128);
}

void dist_destroy(void* comm) {
  Comm* c = static_cast<Comm*>(comm);
  if (!c) return;
  if (c->c && nccl().CommDestroy) nccl().CommDestroy(c->c);
  delete c;
}

}  // namespace spmv
