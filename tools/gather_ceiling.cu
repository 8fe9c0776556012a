// tools/gather_ceiling.cu — MEASUREMENT TOOL (not product code): the ceiling
// of the x gathers of a matrix's own column stream, with no FMA and no y.
//
// SpMV on scattered columns (c3 RMAT, c4 uniform random) is bound by the
// gathers x[col[k]], not by HBM ("random access to X"; VERDICT r1 item
// 5). This library times, over the column array exactly as a format stores
// it, only the work every kernel must do for x:
//   mode 0 LSU, warp order   : lane l of a warp gathers entry base + 32·q + l
//                              (32 consecutive stored entries per instruction)
//   mode 1 LSU, lane order   : lane l gathers entries base + 8·l + q (the COO
//                              kernel's order: 8 consecutive entries per lane)
//   mode 2 TMA gather4       : cp.async.bulk.tensor.2d ... tile::gather4 —
//                              x viewed as 16-byte rows; one instruction brings
//                              4 rows (4 gathers) into shared memory through
//                              the TMA unit instead of the LSU/L1TEX path
//   mode 3 TMA bulk 16 B     : cp.async.bulk of one 16-byte row per gather
// Every mode reads the column array with coalesced 128-bit loads and folds
// the gathered values into one checksum per thread (so nothing is dead code).
// Built by tools/build_tools.py; called from bench.py and tools/gather_sweep.py.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ int4 ld_idx4(const int* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
template <class T>
__device__ __forceinline__ double ldx(const T* p) {
  return (double)__ldg(p);
}

// mode 0/1: LSU gathers. U entries per lane per iteration (U/4 index loads).
template <class T, int U, bool LANE_ORDER>
__global__ void __launch_bounds__(256) k_gather_lsu(const int* __restrict__ col, int64_t nnz, const T* __restrict__ x,
                                                    double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  const int64_t per = 32LL * U;
  for (int64_t base = warp * per; base < nnz; base += nwarps * per) {
    int c[U];
    if (base + per <= nnz) {
#pragma unroll
      for (int q = 0; q < U / 4; ++q) {
        // warp order: index vector q of lane l covers entries base + 128q + 4l .. +3;
        // the gather of item j of that vector is at base + 128q + 4l + j.
        // lane order: lane l owns entries base + U·l .. base + U·l + U − 1.
        const int64_t k = LANE_ORDER ? base + (int64_t)U * lane + 4 * q : base + 128LL * q + 4 * lane;
        int4 v = ld_idx4(col + k);
        c[4 * q] = v.x; c[4 * q + 1] = v.y; c[4 * q + 2] = v.z; c[4 * q + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < U / 4; ++q)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int64_t k = LANE_ORDER ? base + (int64_t)U * lane + 4 * q + j : base + 128LL * q + 4 * lane + j;
          c[4 * q + j] = k < nnz ? col[k] : -1;
        }
    }
    double v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) v[j] = c[j] >= 0 ? ldx(x + c[j]) : 0.0;
#pragma unroll
    for (int j = 0; j < U; ++j) acc += v[j];
  }
  out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// mode 2/3: TMA gathers. A warp owns a ring of S stages; in a stage each lane
// brings 4 gathers (one gather4, or four 16-byte bulk copies) into its own
// 128-byte slot; lane 0 arrives on the stage barrier with the transaction
// count. The stage issued S−1 chunks ago is consumed (wait, read, fold).
constexpr int kS = 4;          // stages per warp
constexpr int kWarps = 8;      // warps per block
constexpr int kSlot = 128;     // bytes per lane slot (tensor copies want 128-byte aligned destinations)

template <class T, bool G4>
__global__ void __launch_bounds__(kWarps * 32) k_gather_tma(const __grid_constant__ CUtensorMap tm,
                                                            const int* __restrict__ col, int64_t nnz,
                                                            const T* __restrict__ x, double* __restrict__ out) {
  constexpr int EPR = 16 / sizeof(T);  // elements per 16-byte row
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[kWarps][kS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned char* ring = smem + (size_t)w * kS * 32 * kSlot;
  if (lane == 0)
    for (int s = 0; s < kS; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar[w][s])) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int64_t gw = ((int64_t)blockIdx.x * kWarps + w);
  const int64_t nw = (int64_t)gridDim.x * kWarps;
  const int64_t nchunks = (nnz + 127) / 128;
  (void)x;
  double acc = 0.0;
  int cl[kS][4];
  // stage s of round r holds chunk gw + (r·kS + s)·nw; the stage loop is
  // unrolled so cl[][] stays in registers
  auto consume = [&](int s, uint32_t phase) {  // phase = parity of the round that issued stage s
    asm volatile(
        "{\n\t.reg .pred P1;\nW%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra W%=;\n\t}" ::"r"(saddr(&bar[w][s])),
        "r"(phase)
        : "memory");
    const T* slot = reinterpret_cast<const T*>(ring + ((size_t)s * 32 + lane) * kSlot);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (cl[s][j] >= 0) acc += (double)slot[j * EPR + (cl[s][j] % EPR)];
    // the next async-proxy write into this slot must follow these reads
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  };
  bool live[kS] = {};
  int64_t r = 0;
  for (;; ++r) {
    const int64_t first = gw + r * kS * nw;
    if (first >= nchunks) break;
#pragma unroll
    for (int s = 0; s < kS; ++s) {
      const int64_t ch = first + (int64_t)s * nw;
      if (live[s]) {
        consume(s, (uint32_t)((r - 1) & 1));
        live[s] = false;
      }
      if (ch >= nchunks) continue;
      const int64_t k = ch * 128 + 4 * lane;
      int c4[4];
      if (k + 4 <= nnz) {
        int4 v = ld_idx4(col + k);
        c4[0] = v.x; c4[1] = v.y; c4[2] = v.z; c4[3] = v.w;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) c4[j] = k + j < nnz ? col[k + j] : -1;
      }
      unsigned char* dst = ring + ((size_t)s * 32 + lane) * kSlot;
      if (G4) {
        const int r0 = c4[0] >= 0 ? c4[0] / EPR : 0, r1 = c4[1] >= 0 ? c4[1] / EPR : 0;
        const int r2 = c4[2] >= 0 ? c4[2] / EPR : 0, r3 = c4[3] >= 0 ? c4[3] / EPR : 0;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(saddr(dst)),
            "l"(&tm), "r"(saddr(&bar[w][s])), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
            : "memory");
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int rr = c4[j] >= 0 ? c4[j] / EPR : 0;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(
                  saddr(dst + 16 * j)),
              "l"(x + (int64_t)rr * EPR), "r"(saddr(&bar[w][s]))
              : "memory");
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) cl[s][j] = c4[j];
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(&bar[w][s])),
                     "r"(64 * 32)
                     : "memory");
      live[s] = true;
    }
  }
  // drain: the live stages were issued in round r − 1
#pragma unroll
  for (int s = 0; s < kS; ++s)
    if (live[s]) consume(s, (uint32_t)((r - 1) & 1));
  out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

template <class T>
int run(int mode, const int* col, int64_t nnz, const void* xv, int64_t n, int reps, double* out_ms,
        cudaStream_t st) {
  const T* x = static_cast<const T*>(xv);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out = nullptr;
  const int64_t maxthreads = (int64_t)sms * 2048;
  if (cudaMallocAsync(&out, maxthreads * sizeof(double), st) != cudaSuccess) return 1;
  CUtensorMap tm{};
  const void* fn = nullptr;
  int block = 256, grid = 0;
  size_t smem = 0;
  if (mode == 0) fn = (const void*)k_gather_lsu<T, 16, false>;
  else if (mode == 1) fn = (const void*)k_gather_lsu<T, 16, true>;
  else if (mode == 2 || mode == 3) {
    fn = mode == 2 ? (const void*)k_gather_tma<T, true> : (const void*)k_gather_tma<T, false>;
    block = kWarps * 32;
    smem = (size_t)kWarps * kS * 32 * kSlot;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 2;
    auto enc = get_encode();
    if (!enc) return 3;
    constexpr int EPR = 16 / sizeof(T);
    cuuint64_t dims[2] = {(cuuint64_t)EPR, (cuuint64_t)((n + EPR - 1) / EPR)};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {(cuuint32_t)EPR, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                     const_cast<T*>(x), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return 100 + (int)r;
  } else {
    return 4;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, block, smem) != cudaSuccess || per_sm < 1) return 5;
  grid = sms * per_sm;
  void* args_lsu[] = {&col, &nnz, &x, &out};
  void* args_tma[] = {&tm, &col, &nnz, &x, &out};
  void** args = mode >= 2 ? args_tma : args_lsu;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 2; ++w)
    if (cudaLaunchKernel(fn, grid, block, args, smem, st) != cudaSuccess) return 6;
  cudaEventRecord(a, st);
  for (int r = 0; r < reps; ++r) cudaLaunchKernel(fn, grid, block, args, smem, st);
  cudaEventRecord(b, st);
  if (cudaEventSynchronize(b) != cudaSuccess) return 7;
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  *out_ms = ms / reps;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFreeAsync(out, st);
  return cudaGetLastError() == cudaSuccess ? 0 : 8;
}

}  // namespace

// mode 0..3 (above); dtype 0 = fp64 x, 1 = fp32 x. Returns 0 on success and
// the average milliseconds of one pass over the nnz column entries in *out_ms.
extern "C" int gather_ceiling(int mode, int dtype, const int* col, int64_t nnz, const void* x, int64_t n, int reps,
                              double* out_ms, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return dtype == 0 ? run<double>(mode, col, nnz, x, n, reps, out_ms, st)
                    : run<float>(mode, col, nnz, x, n, reps, out_ms, st);
}
