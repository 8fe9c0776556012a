// spmv_bell.cu — BELL launcher (kernel: kern_bell.cuh).
#include "kern_bell_decl.cuh"

namespace spmv {
namespace {

template <class T>
void launch_bell(spmv_matrix* h, kern::BellParams& p, const spmv_launch_t& L) {
  const int bi = block_index(L.block), ri = reg_index(L.maxreg);
  const void* fn;
  switch (h->bell_b) {
    case 2: fn = (const void*)kern::bell_fn<T, 2>(bi, ri); break;
    case 3: fn = (const void*)kern::bell_fn<T, 3>(bi, ri); break;
    case 4: fn = (const void*)kern::bell_fn<T, 4>(bi, ri); break;
    default: fail(SPMV_ERR_UNSUPPORTED, "BELL block dimension must be 2, 3 or 4");
  }
  const LaunchAttrs attrs(fn, L.carveout_pct);
  const int64_t grid = persistent_grid(fn, L.block, (p.nbr + L.block - 1) / L.block);
  if (grid <= 0) return;
  if (p.e.mode == 1) {
    ensure_pi_scratch(h, (size_t)grid);
    p.e.partials = h->pi_partials;
    p.e.counter = h->pi_counter;
  }
  void* args[] = {&p};
  launch_checked(fn, dim3((unsigned)grid), dim3(L.block), args, 0, h->stream);
}

}  // namespace

void run_bell(spmv_matrix* h, const Epilogue& e, const void* x, void* y, const spmv_launch_t& L) {
  kern::BellParams p{};
  p.bcol = h->bell_col;
  p.bval = h->bell_val;
  p.rows = h->rows;
  p.cols = h->cols;
  p.nbr = h->bell_nbr;
  p.nbr_pad = h->bell_nbr_pad;
  p.kb = h->bell_kb;
  p.x = x;
  p.y = y;
  p.e = e;
  if (h->dtype == SPMV_R64F) launch_bell<double>(h, p, L);
  else launch_bell<float>(h, p, L);
}

}  // namespace spmv
