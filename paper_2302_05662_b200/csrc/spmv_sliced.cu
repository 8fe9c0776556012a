// spmv_sliced.cu — ELL/SELL launchers (kernels: kern_sliced.cuh).
#include "kern_sliced_decl.cuh"

namespace spmv {
namespace {

template <class T>
void launch_sliced(spmv_matrix* h, kern::SlicedParams& p, int C, const spmv_launch_t& L) {
  const int bi = block_index(L.block), ri = reg_index(L.maxreg);
  const void* fn;
  const int enc = p.col8 ? 2 : (p.col16 ? 1 : 0);
  const bool carry = (L.knob & kern::kSlicedCarry) != 0;
#define SL_ENC(CC, E) (carry ? (const void*)kern::sliced_fn<T, CC, E, true>(bi, ri) \
                             : (const void*)kern::sliced_fn<T, CC, E, false>(bi, ri))
#define SL_PICK(CC) fn = enc == 2 ? SL_ENC(CC, 2) : (enc == 1 ? SL_ENC(CC, 1) : SL_ENC(CC, 0))
  switch (C) {
    case 32: SL_PICK(32); break;
    case 64: SL_PICK(64); break;
    case 128: SL_PICK(128); break;
    case 256: SL_PICK(256); break;
    default: fail(SPMV_ERR_UNSUPPORTED, "slice height C must be 32, 64, 128 or 256");
  }
#undef SL_PICK
#undef SL_ENC
  const LaunchAttrs attrs(fn, L.carveout_pct);
  const int64_t warps_per_block = L.block / 32;
  const int64_t grid = persistent_grid(fn, L.block, (p.nslices + warps_per_block - 1) / warps_per_block);
  if (grid <= 0) return;
  if (p.e.mode == 1) {
    ensure_pi_scratch(h, (size_t)grid);
    p.e.partials = h->pi_partials;
    p.e.counter = h->pi_counter;
  }
  void* args[] = {&p};
  if (p.e.mode == 1 && p.e.pdl) {
    // power step: programmatic dependent launch (see k_sliced)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(L.block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = h->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
    if (e != cudaSuccess) cudaGetLastError();
    cuda_check(e, "cudaLaunchKernelExC");
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return;
  }
  launch_checked(fn, dim3((unsigned)grid), dim3(L.block), args, 0, h->stream);
}

}  // namespace

void run_ell_arrays(spmv_matrix* h, const int32_t* col, const void* val, int64_t K, int64_t n_pad,
                    const Epilogue& e, const void* x, void* y, const spmv_launch_t& L, const int16_t* col16,
                    const uint8_t* col8, const int32_t* tab8) {
  kern::SlicedParams p{};
  const int C = L.knob & 0xffff;
  if (C == 0 || n_pad % C != 0) fail(SPMV_ERR_UNSUPPORTED, "ELL rows-per-warp must divide n_pad (a multiple of 128)");
  if (n_pad > INT32_MAX) fail(SPMV_ERR_UNSUPPORTED, "ELL: n_pad must fit 31 bits (the kernel's k-step stride)");
  p.col = col;
  p.col16 = col16;
  p.col8 = col8;
  p.tab8 = tab8;
  p.col_origin = h->col_origin;
  p.val = val;
  p.sp = nullptr;
  p.perm = nullptr;
  p.rows = h->rows;
  p.nslices = n_pad / C;
  p.ell_K = K;
  p.ell_stride = n_pad;
  p.x = x;
  p.y = y;
  p.e = e;
  if (h->dtype == SPMV_R64F) launch_sliced<double>(h, p, C, L);
  else launch_sliced<float>(h, p, C, L);
}

void run_ell(spmv_matrix* h, const Epilogue& e, const void* x, void* y, const spmv_launch_t& L) {
  run_ell_arrays(h, h->ell_col, h->ell_val, h->ell_K, h->ell_npad, e, x, y, L, h->ell_col16, h->ell_col8,
                 h->dict8_tab);
}

void run_sell(spmv_matrix* h, const Epilogue& e, const void* x, void* y, const spmv_launch_t& L) {
  kern::SlicedParams p{};
  p.col = h->sell_col;
  p.col16 = h->sell_col16;
  p.col8 = h->sell_col8;
  p.tab8 = h->dict8_tab;
  p.col_origin = h->col_origin;
  p.val = h->sell_val;
  p.sp = h->sell_sp;
  p.perm = h->sell_perm;
  p.rows = h->rows;
  p.nslices = h->sell_ns;
  p.x = x;
  p.y = y;
  p.e = e;
  if (h->dtype == SPMV_R64F) launch_sliced<double>(h, p, (int)h->sell_C, L);
  else launch_sliced<float>(h, p, (int)h->sell_C, L);
}

}  // namespace spmv
