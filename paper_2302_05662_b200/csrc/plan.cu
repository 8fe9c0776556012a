// plan.cu — the distributed power-iteration plan.
//
//  (i)  Each rank's row slab is split into an INTERIOR row block, whose
//       columns all lie in the rank's own chunk of the padded vector layout,
//       and two HALO blocks (the leading rows that reference columns below
//       the chunk, the trailing rows that reference columns above it). The
//       split is exact for any matrix: h0 = 1 + the last row with a column
//       below the chunk, h1 = the first row with a column above it.
//  (ii) Per step the interior SpMV runs as soon as the previous step's
//       all-reduce has landed, concurrently with the exchange of the previous
//       iterate on a second stream; the halo SpMVs wait for the exchange.
//  (iii) Normalisation is folded into the next step's alpha, read on the
//       device from the all-reduced partial sums (Σ over the three parts in
//       a fixed order, identical on every rank).
//  f4   With SPMV_PLAN_HALO the all-gather of the whole iterate is replaced
//       by a point-to-point exchange of exactly the remote entries the halo
//       rows reference (lists built once with the same communicator).
// Every kernel is the handle's own power-step kernel; the plan adds only the
// split, the list builders, the pack/unpack gathers and the stream schedule.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "dist.cuh"
#include "primitives.cuh"
#include "spmv_common.cuh"

struct spmv_dist_plan {
  spmv::CommBase* comm = nullptr;
  int rank = 0, world = 1, device = 0;
  cudaStream_t s = nullptr;   // compute stream (the parent handle's)
  cudaStream_t cs = nullptr;  // communication stream (owned)
  cudaEvent_t ev_done = nullptr, ev_reduced = nullptr, ev_gathered = nullptr;
  spmv_dtype_t dtype = SPMV_R64F;
  int vb = 8;
  int64_t chunk = 0, own_lo = 0, n_local = 0, n_full = 0;
  int64_t h0 = 0, h1 = 0;
  spmv_matrix* part[3] = {nullptr, nullptr, nullptr};  // interior [h0,h1), lo halo [0,h0), hi halo [h1,n)
  int64_t part_r0[3] = {0, 0, 0};
  uint32_t flags = 0;
  int sm_reserve = 0;
  // halo exchange (f4)
  bool halo = false;
  std::vector<int64_t> need_cnt, need_off;  // per owner q: entries received from q (segments of U)
  std::vector<int64_t> give_cnt, give_off;  // per requester r: entries sent to r (segments of send_idx)
  std::vector<int64_t> recv_first, send_first;
  bool recv_direct = false, send_direct = false;
  int32_t* U = nullptr;  // sorted padded positions received
  int64_t nU = 0;
  int32_t* send_idx = nullptr;  // padded positions (own chunk) sent, grouped by requester
  int64_t n_send = 0;
  void* recv_buf = nullptr;
  void* send_buf = nullptr;
  double* psums = nullptr;  // [(steps+1)][3 parts][2]
  int64_t psums_cap = 0;
  std::string last_error;
};

namespace spmv {
namespace {

constexpr int kParts = 3;
constexpr int kTile = 4096;  // compaction tile: 256 threads × 16 entries

template <class RP>
__global__ void k_split(const RP* __restrict__ rp, const int32_t* __restrict__ col, int64_t n, int64_t lo,
                        int64_t hi, unsigned long long* maxlo_p1, unsigned long long* minhi) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t a = rp[i], b = rp[i + 1];
    if (a == b) continue;
    if (col[a] < lo) atomicMax(maxlo_p1, (unsigned long long)(i + 1));
    if (col[b - 1] >= hi) atomicMin(minhi, (unsigned long long)i);
  }
}

__global__ void k_mark_remote(const int32_t* __restrict__ col, int64_t nnz, int64_t lo, int64_t hi,
                              uint8_t* __restrict__ mark) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride) {
    const int64_t c = col[k];
    if (c < lo || c >= hi) mark[c] = 1;
  }
}

__global__ void __launch_bounds__(256) k_count_marks(const uint8_t* __restrict__ m, int64_t n, int64_t* cnt) {
  const int64_t base = (int64_t)blockIdx.x * kTile;
  int c = 0;
  for (int i = 0; i < kTile / 256; ++i) {
    const int64_t j = base + (int64_t)i * 256 + threadIdx.x;
    c += __syncthreads_count(j < n && m[j]);
  }
  if (threadIdx.x == 0) cnt[blockIdx.x] = c;
}

// Positions of the marked entries, ascending: thread t of block b owns the 16
// consecutive entries [b·4096 + 16t, +16); a block scan of the per-thread
// counts gives each thread its output offset.
__global__ void __launch_bounds__(256) k_emit_marks(const uint8_t* __restrict__ m, int64_t n,
                                                    const int64_t* __restrict__ off, int32_t* __restrict__ out) {
  __shared__ int warp_tot[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t first = (int64_t)blockIdx.x * kTile + (int64_t)threadIdx.x * 16;
  int c = 0;
  for (int i = 0; i < 16; ++i) c += (first + i < n && m[first + i]) ? 1 : 0;
  int inc = c;
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  int before = 0;
  for (int w = 0; w < warp; ++w) before += warp_tot[w];
  int64_t pos = off[blockIdx.x] + before + inc - c;
  for (int i = 0; i < 16; ++i)
    if (first + i < n && m[first + i]) out[pos++] = (int32_t)(first + i);
}

template <class T>
__global__ void k_pack(const T* __restrict__ x, const int32_t* __restrict__ idx, int64_t n, T* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) out[j] = x[idx[j]];
}

template <class T>
__global__ void k_unpack(const T* __restrict__ in, const int32_t* __restrict__ idx, int64_t n, T* __restrict__ x) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) x[idx[j]] = in[j];
}

// sums[k] = Σ_p psums[k][p] (part order) for k = 0..n-1.
__global__ void k_fold_sums(const double* __restrict__ ps, int64_t n, double* __restrict__ sums) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
    double a = 0, b = 0;
    for (int p = 0; p < kParts; ++p) {
      a += ps[(k * kParts + p) * 2];
      b += ps[(k * kParts + p) * 2 + 1];
    }
    sums[2 * k] = a;
    sums[2 * k + 1] = b;
  }
}

struct SmReserve {
  int old;
  explicit SmReserve(int r) : old(g_sm_reserve) { g_sm_reserve = r; }
  ~SmReserve() { g_sm_reserve = old; }
};

void convert_like(spmv_matrix* d, const spmv_matrix* p) {
  const int fmt = p->active;
  switch (fmt) {
    case SPMV_FMT_CSR:
      d->csr_alg = p->csr_alg;
      d->csr_T = p->csr_T;
      break;
    case SPMV_FMT_COO: build_coo(d); break;
    // ELL/SELL: 16-bit column offsets from the part's own diagonal whenever they fit
    case SPMV_FMT_ELL: build_ell(d, -1); break;
    case SPMV_FMT_SELL: build_sell(d, p->sell_C, p->sell_sigma, -1); break;
    case SPMV_FMT_HYB: build_hyb(d, p->hyb_K); break;
    case SPMV_FMT_BELL: build_bell(d, p->bell_b); break;
    default: fail(SPMV_ERR_INVALID_ARG, "plan: bad parent format");
  }
  d->active = fmt;
  d->launch[fmt] = p->launch[fmt];
}

template <class T>
T host_copy1(const T* d, cudaStream_t s) {
  T v;
  CK(cudaMemcpyAsync(&v, d, sizeof(T), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return v;
}

// Interior/halo bounds of the slab (device pass + 2 values back).
void find_split(spmv_dist_plan* P, spmv_matrix* h) {
  cudaStream_t s = P->s;
  const int64_t n = h->rows;
  Scratch sc(s);
  unsigned long long* d = sc.get<unsigned long long>(2);
  unsigned long long init[2] = {0ull, (unsigned long long)n};
  CK(cudaMemcpyAsync(d, init, sizeof(init), cudaMemcpyHostToDevice, s));
  if (n > 0) {
    const unsigned g = grid_for(n, 256);
    const int64_t lo = P->own_lo, hi = P->own_lo + P->n_local;
    if (h->rp64)
      LAUNCH(k_split<int64_t>, g, 256, 0, s, static_cast<const int64_t*>(h->row_ptr), h->col, n, lo, hi, d, d + 1);
    else
      LAUNCH(k_split<int32_t>, g, 256, 0, s, static_cast<const int32_t*>(h->row_ptr), h->col, n, lo, hi, d, d + 1);
  }
  unsigned long long r[2];
  CK(cudaMemcpyAsync(r, d, sizeof(r), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  P->h0 = (int64_t)r[0];
  P->h1 = std::max<int64_t>((int64_t)r[1], P->h0);
}

// f4: lists of the remote entries each rank's halo rows reference, exchanged
// once so the owner knows what to send every step. Returns false (on every
// rank alike) when the lists would move at least half of what the all-gather
// moves — the plan then keeps the all-gather.
bool build_halo_lists(spmv_dist_plan* P) {
  CommBase* comm = P->comm;
  cudaStream_t s = P->s;
  const int W = P->world;
  const int64_t lo = P->own_lo, hi = P->own_lo + P->n_local;
  Scratch sc(s);
  uint8_t* mark = sc.get<uint8_t>(P->n_full);
  CK(cudaMemsetAsync(mark, 0, (size_t)P->n_full, s));
  for (int p = 1; p < kParts; ++p) {
    spmv_matrix* h = P->part[p];
    if (h && h->nnz > 0) LAUNCH(k_mark_remote, grid_for(h->nnz, 256), 256, 0, s, h->col, h->nnz, lo, hi, mark);
  }
  const int64_t nb = (P->n_full + kTile - 1) / kTile;
  int64_t* cnt = sc.get<int64_t>(nb);
  int64_t* off = sc.get<int64_t>(nb + 1);
  if (nb > 0) {
    LAUNCH(k_count_marks, (unsigned)nb, 256, 0, s, (const uint8_t*)mark, P->n_full, cnt);
    exclusive_scan_i64(cnt, off, nb, s);
  } else {
    CK(cudaMemsetAsync(off, 0, sizeof(int64_t), s));
  }
  P->nU = host_copy1(off + nb, s);
  P->U = dalloc_n<int32_t>(P->nU, s);
  if (nb > 0 && P->nU > 0)
    LAUNCH(k_emit_marks, (unsigned)nb, 256, 0, s, (const uint8_t*)mark, P->n_full, (const int64_t*)off, P->U);
  std::vector<int32_t> Uh((size_t)P->nU);
  if (P->nU) CK(cudaMemcpyAsync(Uh.data(), P->U, (size_t)P->nU * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));

  // collective decision: halo lists only if every rank receives < half of the all-gather
  double* vote = sc.get<double>(1);
  const double mine = (2 * P->nU > (W - 1) * P->chunk) ? 1.0 : 0.0;
  CK(cudaMemcpyAsync(vote, &mine, sizeof(double), cudaMemcpyHostToDevice, s));
  comm->allreduce_f64(vote, 1, s);
  const double votes = host_copy1(vote, s);
  if (votes != 0.0) {
    dfree(P->U, s);
    P->U = nullptr;
    P->nU = 0;
    return false;
  }
  // segments of U per owner q (U is sorted, owner = position / chunk)
  P->need_cnt.assign(W, 0);
  for (int32_t u : Uh) P->need_cnt[u / P->chunk]++;
  P->need_off.assign(W + 1, 0);
  for (int q = 0; q < W; ++q) P->need_off[q + 1] = P->need_off[q] + P->need_cnt[q];
  // counts matrix: row r = what r needs from each owner
  int64_t* cm = sc.get<int64_t>((int64_t)W * W);
  CK(cudaMemcpyAsync(cm + (size_t)P->rank * W, P->need_cnt.data(), W * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  comm->allgather_inplace(cm, W * sizeof(int64_t), s);
  std::vector<int64_t> cmh((size_t)W * W);
  CK(cudaMemcpyAsync(cmh.data(), cm, cmh.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  P->give_cnt.assign(W, 0);
  for (int r = 0; r < W; ++r) P->give_cnt[r] = cmh[(size_t)r * W + P->rank];
  P->give_off.assign(W + 1, 0);
  for (int r = 0; r < W; ++r) P->give_off[r + 1] = P->give_off[r] + P->give_cnt[r];
  P->n_send = P->give_off[W];
  P->send_idx = dalloc_n<int32_t>(P->n_send, s);
  // each rank sends its request list to the owner
  std::vector<P2P> sends, recvs;
  for (int q = 0; q < W; ++q)
    if (P->need_cnt[q]) sends.push_back({q, P->U + P->need_off[q], (size_t)P->need_cnt[q] * 4});
  for (int r = 0; r < W; ++r)
    if (P->give_cnt[r]) recvs.push_back({r, P->send_idx + P->give_off[r], (size_t)P->give_cnt[r] * 4});
  comm->exchange(sends, recvs, s);
  std::vector<int32_t> Sh((size_t)P->n_send);
  if (P->n_send) CK(cudaMemcpyAsync(Sh.data(), P->send_idx, (size_t)P->n_send * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  // contiguous segments travel straight from/into the vector (no pack/unpack)
  auto contiguous = [](const std::vector<int32_t>& v, int64_t a, int64_t n) {
    return n == 0 || (int64_t)v[(size_t)(a + n - 1)] - v[(size_t)a] + 1 == n;
  };
  P->recv_first.assign(W, 0);
  P->send_first.assign(W, 0);
  P->recv_direct = true;
  for (int q = 0; q < W; ++q) {
    P->recv_direct = P->recv_direct && contiguous(Uh, P->need_off[q], P->need_cnt[q]);
    if (P->need_cnt[q]) P->recv_first[q] = Uh[(size_t)P->need_off[q]];
  }
  P->send_direct = true;
  for (int r = 0; r < W; ++r) {
    P->send_direct = P->send_direct && contiguous(Sh, P->give_off[r], P->give_cnt[r]);
    if (P->give_cnt[r]) P->send_first[r] = Sh[(size_t)P->give_off[r]];
  }
  const char* env = getenv("SPMV_PLAN_FORCE_STAGED");  // testing: always pack/unpack
  if (env && env[0] == '1') P->recv_direct = P->send_direct = false;
  if (!P->recv_direct) P->recv_buf = dalloc((size_t)std::max<int64_t>(P->nU, 1) * P->vb, s);
  if (!P->send_direct) P->send_buf = dalloc((size_t)std::max<int64_t>(P->n_send, 1) * P->vb, s);
  return true;
}

void exchange_step(spmv_dist_plan* P, void* x) {
  const NvtxRange nvtx_range("plan_exchange");
  cudaStream_t cs = P->cs;
  char* xb = static_cast<char*>(x);
  const int vb = P->vb;
  if (!P->halo) {
    P->comm->allgather_inplace(x, (size_t)P->chunk * vb, cs);
    return;
  }
  const int W = P->world;
  if (!P->send_direct && P->n_send > 0) {
    const unsigned g = grid_for(P->n_send, 256, 148 * 8);
    if (P->dtype == SPMV_R64F)
      LAUNCH(k_pack<double>, g, 256, 0, cs, (const double*)x, (const int32_t*)P->send_idx, P->n_send,
             (double*)P->send_buf);
    else
      LAUNCH(k_pack<float>, g, 256, 0, cs, (const float*)x, (const int32_t*)P->send_idx, P->n_send,
             (float*)P->send_buf);
  }
  std::vector<P2P> sends, recvs;
  for (int r = 0; r < W; ++r)
    if (P->give_cnt[r])
      sends.push_back({r,
                       P->send_direct ? (void*)(xb + P->send_first[r] * vb)
                                      : (void*)(static_cast<char*>(P->send_buf) + P->give_off[r] * vb),
                       (size_t)P->give_cnt[r] * vb});
  for (int q = 0; q < W; ++q)
    if (P->need_cnt[q])
      recvs.push_back({q,
                       P->recv_direct ? (void*)(xb + P->recv_first[q] * vb)
                                      : (void*)(static_cast<char*>(P->recv_buf) + P->need_off[q] * vb),
                       (size_t)P->need_cnt[q] * vb});
  P->comm->exchange(sends, recvs, cs);
  if (!P->recv_direct && P->nU > 0) {
    const unsigned g = grid_for(P->nU, 256, 148 * 8);
    if (P->dtype == SPMV_R64F)
      LAUNCH(k_unpack<double>, g, 256, 0, cs, (const double*)P->recv_buf, (const int32_t*)P->U, P->nU, (double*)x);
    else
      LAUNCH(k_unpack<float>, g, 256, 0, cs, (const float*)P->recv_buf, (const int32_t*)P->U, P->nU, (float*)x);
  }
}

}  // namespace

void plan_destroy(spmv_dist_plan* P);

spmv_dist_plan* plan_create(spmv_matrix* h, void* comm_v, int64_t chunk, uint32_t flags) {
  CommBase* comm = as_comm(comm_v);
  spmv_dist_plan* P = new spmv_dist_plan();
  try {
    P->comm = comm;
    P->rank = comm ? comm->rank : 0;
    P->world = comm ? comm->world : 1;
    P->device = h->device;
    P->s = h->stream;
    P->dtype = h->dtype;
    P->vb = h->vbytes;
    P->flags = flags;
    P->chunk = comm ? chunk : h->rows;
    P->n_local = h->rows;
    P->own_lo = (int64_t)P->rank * P->chunk;
    P->n_full = comm ? (int64_t)P->world * P->chunk : h->cols;
    if (comm && (chunk < h->rows || h->cols > P->n_full))
      fail(SPMV_ERR_INVALID_ARG, "plan: chunk < local rows or matrix columns beyond world·chunk");
    const char* env = getenv("SPMV_PLAN_SM_RESERVE");
    P->sm_reserve = env ? std::atoi(env) : 16;
    if (comm && P->world > 1) {
      find_split(P, h);
    } else {
      P->h0 = 0;
      P->h1 = h->rows;
    }
    const int64_t r0[kParts] = {P->h0, 0, P->h1}, r1[kParts] = {P->h1, P->h0, h->rows};
    for (int p = 0; p < kParts; ++p) {
      P->part_r0[p] = r0[p];
      if (r1[p] > r0[p]) {
        P->part[p] = make_row_slice(h, r0[p], r1[p]);
        P->part[p]->col_origin = P->own_lo + r0[p];  // row i of the part sits at column position origin + i
        convert_like(P->part[p], h);
      }
    }
    if (comm && P->world > 1 && (flags & SPMV_PLAN_HALO)) P->halo = build_halo_lists(P);
    CK(cudaStreamCreateWithFlags(&P->cs, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&P->ev_done, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&P->ev_reduced, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&P->ev_gathered, cudaEventDisableTiming));
    CK(cudaStreamSynchronize(P->s));
  } catch (...) {
    plan_destroy(P);
    throw;
  }
  return P;
}

void plan_destroy(spmv_dist_plan* P) {
  if (!P) return;
  cudaSetDevice(P->device);
  cudaStream_t s = P->s;
  if (P->cs) cudaStreamSynchronize(P->cs);
  for (auto*& p : P->part)
    if (p) {
      spmv_destroy(p);
      p = nullptr;
    }
  dfree(P->U, s);
  dfree(P->send_idx, s);
  dfree(P->recv_buf, s);
  dfree(P->send_buf, s);
  dfree(P->psums, s);
  if (P->ev_done) cudaEventDestroy(P->ev_done);
  if (P->ev_reduced) cudaEventDestroy(P->ev_reduced);
  if (P->ev_gathered) cudaEventDestroy(P->ev_gathered);
  if (P->cs) cudaStreamDestroy(P->cs);
  delete P;
}

void plan_iterate(spmv_dist_plan* P, const void* x0, void* buf0, void* buf1, int64_t steps, double* sums,
                  float* loop_ms, float* interior_ms, int* final_buf) {
  cudaStream_t s = P->s;
  CommBase* comm = (P->comm && P->world >= 1) ? P->comm : nullptr;
  const int vb = P->vb;
  const bool overlap = (P->flags & SPMV_PLAN_OVERLAP) != 0;
  try {
    if (x0 != buf0) CK(cudaMemcpyAsync(buf0, x0, (size_t)P->n_full * vb, cudaMemcpyDeviceToDevice, s));
    const int64_t need = (steps + 1) * kParts * 2;
    if (P->psums_cap < need) {
      dfree(P->psums, s);
      P->psums = dalloc_n<double>(need, s);
      P->psums_cap = need;
    }
    CK(cudaMemsetAsync(P->psums, 0, (size_t)need * sizeof(double), s));
    spmv_matrix* any = P->part[0] ? P->part[0] : (P->part[1] ? P->part[1] : P->part[2]);
    if (any) spmv_norm2_internal(any, static_cast<char*>(buf0) + P->own_lo * vb, P->n_local, P->psums);
    if (comm) comm->allreduce_f64(P->psums, kParts * 2, s);
    std::vector<cudaEvent_t> iev;
    if (interior_ms) {
      iev.resize(2 * (size_t)steps);
      for (auto& e : iev) CK(cudaEventCreate(&e));
    }
    cudaEvent_t l0 = nullptr, l1 = nullptr;
    if (loop_ms) {
      CK(cudaEventCreate(&l0));
      CK(cudaEventCreate(&l1));
      CK(cudaEventRecord(l0, s));
    }
    void* cur = buf0;
    void* nxt = buf1;
    const int reserve = (comm && comm->uses_sms() && overlap) ? P->sm_reserve : 0;
    for (int64_t k = 0; k < steps; ++k) {
      const double* sp = P->psums + k * kParts * 2;
      double* so = P->psums + (k + 1) * kParts * 2;
      char* ybase = static_cast<char*>(nxt) + P->own_lo * vb;
      if (comm && k > 0) {
        CK(cudaStreamWaitEvent(s, P->ev_reduced, 0));             // alpha_k needs S_{k-1} (iii)
        if (!overlap) CK(cudaStreamWaitEvent(s, P->ev_gathered, 0));
      }
      if (interior_ms) CK(cudaEventRecord(iev[2 * k], s));
      if (P->part[0]) {
        SmReserve r(reserve);
        power_step_internal(P->part[0], cur, ybase + P->h0 * vb, sp, so, P->own_lo + P->h0, kParts, false);
      }
      if (interior_ms) CK(cudaEventRecord(iev[2 * k + 1], s));
      if (comm && k > 0 && overlap) CK(cudaStreamWaitEvent(s, P->ev_gathered, 0));  // halo rows need the exchange
      if (P->part[1]) power_step_internal(P->part[1], cur, ybase, sp, so + 2, P->own_lo, kParts, false);
      if (P->part[2])
        power_step_internal(P->part[2], cur, ybase + P->h1 * vb, sp, so + 4, P->own_lo + P->h1, kParts, false);
      if (comm) {
        CK(cudaEventRecord(P->ev_done, s));
        CK(cudaStreamWaitEvent(P->cs, P->ev_done, 0));
        comm->allreduce_f64(so, kParts * 2, P->cs);
        CK(cudaEventRecord(P->ev_reduced, P->cs));
        exchange_step(P, nxt);
        CK(cudaEventRecord(P->ev_gathered, P->cs));
      }
      std::swap(cur, nxt);
    }
    if (comm && steps > 0) CK(cudaStreamWaitEvent(s, P->ev_gathered, 0));
    if (loop_ms) CK(cudaEventRecord(l1, s));
    LAUNCH(k_fold_sums, grid_for(steps + 1, 256), 256, 0, s, (const double*)P->psums, steps + 1, sums);
    if (loop_ms) {
      CK(cudaEventSynchronize(l1));
      CK(cudaEventElapsedTime(loop_ms, l0, l1));
      cudaEventDestroy(l0);
      cudaEventDestroy(l1);
    }
    if (interior_ms) {
      CK(cudaEventSynchronize(iev.back()));
      for (int64_t k = 0; k < steps; ++k) CK(cudaEventElapsedTime(&interior_ms[k], iev[2 * k], iev[2 * k + 1]));
      for (auto& e : iev) cudaEventDestroy(e);
    }
    if (final_buf) *final_buf = (cur == buf0) ? 0 : 1;
  } catch (...) {
    if (comm) comm->abort();  // peers blocked in a collective fail instead of waiting
    throw;
  }
}

void plan_info(const spmv_dist_plan* P, spmv_dist_plan_info_t* o) {
  std::memset(o, 0, sizeof(*o));
  o->rank = P->rank;
  o->world = P->world;
  o->rows = P->n_local;
  o->chunk = P->chunk;
  o->h0 = P->h0;
  o->h1 = P->h1;
  for (int p = 0; p < kParts; ++p) {
    o->part_rows[p] = P->part[p] ? P->part[p]->rows : 0;
    o->part_nnz[p] = P->part[p] ? P->part[p]->nnz : 0;
  }
  o->overlap = (P->flags & SPMV_PLAN_OVERLAP) ? 1 : 0;
  o->halo = P->halo ? 1 : 0;
  o->recv_elems = P->world > 1 ? (P->halo ? P->nU : (int64_t)(P->world - 1) * P->chunk) : 0;
  o->send_elems = P->world > 1 ? (P->halo ? P->n_send : P->chunk) : 0;
  o->recv_bytes_per_step = o->recv_elems * P->vb;
  o->direct_recv = P->recv_direct ? 1 : 0;
  o->direct_send = P->send_direct ? 1 : 0;
}

int plan_device(const spmv_dist_plan* P) { return P->device; }

spmv_matrix* plan_part(spmv_dist_plan* P, int p) { return (p >= 0 && p < kParts) ? P->part[p] : nullptr; }

}  // namespace spmv
