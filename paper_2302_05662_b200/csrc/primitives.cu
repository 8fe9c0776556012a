// primitives.cu — device-wide exclusive scan (reduce-then-scan, 4096-item
// tiles) and a stable LSD radix sort (8-bit digits, per-tile histograms,
// warp match-based stable ranking). Both deterministic.
#include "primitives.cuh"

namespace spmv {

namespace {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

// Exclusive block scan for 1024 threads; returns this thread's exclusive
// prefix and writes the block total to *total.
__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t* total) {
  __shared__ int64_t s_warp[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < nwarps ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    s_warp[lane] = w;
  }
  __syncthreads();
  int64_t pre = warp > 0 ? s_warp[warp - 1] : 0;
  *total = s_warp[nwarps - 1];
  __syncthreads();
  return pre + x - v;
}

__global__ void k_tile_sums(const int64_t* __restrict__ in, int64_t n, int64_t* __restrict__ sums) {
  int64_t base = (int64_t)blockIdx.x * kScanTile;
  int64_t v = 0;
#pragma unroll
  for (int q = 0; q < kScanItems; ++q) {
    int64_t i = base + (int64_t)q * kScanThreads + threadIdx.x;
    if (i < n) v += in[i];
  }
  int64_t total;
  block_exclusive_scan(v, &total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void k_tile_scan(const int64_t* __restrict__ in, int64_t* __restrict__ out, int64_t n,
                            const int64_t* __restrict__ offs) {
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int64_t v[kScanItems];
  int64_t t = 0;
#pragma unroll
  for (int q = 0; q < kScanItems; ++q) {
    v[q] = (base + q < n) ? in[base + q] : 0;
    t += v[q];
  }
  int64_t total;
  int64_t pre = block_exclusive_scan(t, &total);
  if (offs) pre += offs[blockIdx.x];
#pragma unroll
  for (int q = 0; q < kScanItems; ++q) {
    if (base + q < n) out[base + q] = pre;
    pre += v[q];
    if (base + q == n - 1) out[n] = pre;
  }
}

__global__ void k_set_zero(int64_t* p) { *p = 0; }

// ------------------------------------------------------------------- radix sort
constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortItems = 8;
constexpr int kSortTile = kSortThreads * kSortItems;

__global__ void k_radix_hist(const uint64_t* __restrict__ keys, int64_t n, int shift,
                             int64_t ntiles, int64_t* __restrict__ hist) {
  __shared__ unsigned s_cnt[256];
  s_cnt[threadIdx.x] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * kSortTile;
#pragma unroll
  for (int q = 0; q < kSortItems; ++q) {
    int64_t i = base + (int64_t)q * kSortThreads + threadIdx.x;
    if (i < n) atomicAdd(&s_cnt[(keys[i] >> shift) & 0xFF], 1u);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = s_cnt[threadIdx.x];
}

__global__ void k_radix_scatter(const uint64_t* __restrict__ keys_in,
                                const uint32_t* __restrict__ pay_in, uint64_t* __restrict__ keys_out,
                                uint32_t* __restrict__ pay_out, int64_t n, int shift,
                                int64_t ntiles, const int64_t* __restrict__ offs) {
  __shared__ unsigned s_w[kSortWarps][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int d = threadIdx.x; d < kSortWarps * 256; d += kSortThreads) (&s_w[0][0])[d] = 0;
  __syncthreads();
  const int64_t wbase = (int64_t)blockIdx.x * kSortTile + (int64_t)warp * (32 * kSortItems);
  uint64_t key[kSortItems];
  uint32_t pay[kSortItems];
  unsigned rank[kSortItems];
  int dig[kSortItems];
  const unsigned lt_mask = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    int64_t i = wbase + j * 32 + lane;
    bool valid = i < n;
    key[j] = valid ? keys_in[i] : 0;
    pay[j] = valid ? (pay_in ? pay_in[i] : (uint32_t)i) : 0;
    int d = valid ? (int)((key[j] >> shift) & 0xFF) : 256;
    dig[j] = d;
    unsigned peers = __match_any_sync(0xffffffffu, d);
    unsigned before = (d < 256) ? s_w[warp][d] : 0u;
    __syncwarp();
    int leader = __ffs(peers) - 1;
    if (d < 256 && lane == leader) s_w[warp][d] = before + __popc(peers);
    __syncwarp();
    rank[j] = before + __popc(peers & lt_mask);
  }
  __syncthreads();
  {  // exclusive scan over warps per digit (thread d owns digit d)
    int d = threadIdx.x;
    unsigned run = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
      unsigned c = s_w[w][d];
      s_w[w][d] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    if (dig[j] < 256) {
      int64_t pos = offs[(int64_t)dig[j] * ntiles + blockIdx.x] + s_w[warp][dig[j]] + rank[j];
      keys_out[pos] = key[j];
      pay_out[pos] = pay[j];
    }
  }
}

__global__ void k_iota_u32(uint32_t* p, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) p[i] = (uint32_t)i;
}

}  // namespace

void exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s) {
  if (n <= 0) {
    LAUNCH(k_set_zero, 1, 1, 0, s, out);
    return;
  }
  int64_t ntiles = (n + kScanTile - 1) / kScanTile;
  if (ntiles == 1) {
    LAUNCH(k_tile_scan, 1, kScanThreads, 0, s, in, out, n, (const int64_t*)nullptr);
    return;
  }
  int64_t* sums = dalloc_n<int64_t>(ntiles, s);
  int64_t* offs = dalloc_n<int64_t>(ntiles + 1, s);
  LAUNCH(k_tile_sums, (unsigned)ntiles, kScanThreads, 0, s, in, n, sums);
  exclusive_scan_i64(sums, offs, ntiles, s);
  LAUNCH(k_tile_scan, (unsigned)ntiles, kScanThreads, 0, s, in, out, n, (const int64_t*)offs);
  dfree(sums, s);
  dfree(offs, s);
}

void radix_sort_pairs(const uint64_t* keys_in, const uint32_t* payload_in, uint64_t* keys_out,
                      uint32_t* payload_out, int64_t n, int bits, cudaStream_t s) {
  if (n <= 0) return;
  int passes = (bits + 7) / 8;
  if (passes == 0) {
    CK(cudaMemcpyAsync(keys_out, keys_in, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
    if (payload_in)
      CK(cudaMemcpyAsync(payload_out, payload_in, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
    else
      LAUNCH(k_iota_u32, grid_for(n, 256), 256, 0, s, payload_out, n);
    return;
  }
  int64_t ntiles = (n + kSortTile - 1) / kSortTile;
  int64_t* hist = dalloc_n<int64_t>(256 * ntiles, s);
  int64_t* offs = dalloc_n<int64_t>(256 * ntiles + 1, s);
  uint64_t* ktmp = dalloc_n<uint64_t>(n, s);
  uint32_t* ptmp = dalloc_n<uint32_t>(n, s);
  const uint64_t* ksrc = keys_in;
  const uint32_t* psrc = payload_in;
  for (int p = 0; p < passes; ++p) {
    bool to_out = ((passes - p) & 1) == 1;
    uint64_t* kdst = to_out ? keys_out : ktmp;
    uint32_t* pdst = to_out ? payload_out : ptmp;
    LAUNCH(k_radix_hist, (unsigned)ntiles, kSortThreads, 0, s, ksrc, n, 8 * p, ntiles, hist);
    exclusive_scan_i64(hist, offs, 256 * ntiles, s);
    LAUNCH(k_radix_scatter, (unsigned)ntiles, kSortThreads, 0, s, ksrc, psrc, kdst, pdst, n, 8 * p,
           ntiles, (const int64_t*)offs);
    ksrc = kdst;
    psrc = pdst;
  }
  dfree(hist, s);
  dfree(offs, s);
  dfree(ktmp, s);
  dfree(ptmp, s);
}

}  // namespace spmv
