// spmv_csr.cu — CSR launchers (kernels: kern_csr.cuh).
#include "kern_csr_decl.cuh"

namespace spmv {
template <class T, class RP>
void csr_typed(spmv_matrix* h, const Epilogue& e, const void* x, void* y, const spmv_launch_t& L) {
  kern::CsrParams p{};
  p.rp = h->row_ptr;
  p.col = h->col;
  p.val = h->val;
  p.rows = h->rows;
  p.nnz = h->nnz;
  p.x = x;
  p.y = y;
  p.e = e;
  const int bi = block_index(L.block), ri = reg_index(L.maxreg);
  const bool merge = h->csr_alg == SPMV_CSR_MERGE;
  if (h->csr_alg == SPMV_CSR_STREAM) {
    const int ept = L.knob;
    const void* fn;
    switch (ept) {
      case 16: fn = (const void*)kern::csr_stream_fn<T, RP, 16>(bi, ri); break;
      case 32: fn = (const void*)kern::csr_stream_fn<T, RP, 32>(bi, ri); break;
      case 64: fn = (const void*)kern::csr_stream_fn<T, RP, 64>(bi, ri); break;
      default: fail(SPMV_ERR_INVALID_ARG, "CSR-stream entries per row slot must be 16, 32 or 64");
    }
    if (!fn) fail(SPMV_ERR_UNSUPPORTED, "CSR-stream: block + producer warp exceeds 1024 threads");
    const size_t smem = kern::stream_smem_bytes<T>(L.block, ept);
    if (smem > 227 * 1024 - 1024) fail(SPMV_ERR_UNSUPPORTED, "CSR-stream block × entries exceeds shared memory");
    if (((uintptr_t)h->col | (uintptr_t)h->val) & 15)
      fail(SPMV_ERR_UNSUPPORTED, "CSR-stream: col/val must be 16-byte aligned for the bulk copies");
    const LaunchAttrs attrs(fn, L.carveout_pct, smem);
    const int threads = L.block + 32;  // B consumer threads + one TMA producer warp
    const int64_t grid = persistent_grid(fn, threads, (h->rows + L.block - 1) / L.block, smem);
    if (grid <= 0) return;
    if (e.mode == 1) {
      ensure_pi_scratch(h, (size_t)grid);
      p.e.partials = h->pi_partials;
      p.e.counter = h->pi_counter;
    }
    void* args[] = {&p};
    launch_checked(fn, dim3((unsigned)grid), dim3(threads), args, smem, h->stream);
    return;
  }
  if (!merge && (L.knob & kern::kCsrQuad)) {
    const int lanes = L.knob & 0xff;
    const void* fn;
    switch (lanes) {
      case 4: fn = (const void*)kern::csr_vector4_fn<T, RP, 4>(bi, ri); break;
      case 8: fn = (const void*)kern::csr_vector4_fn<T, RP, 8>(bi, ri); break;
      case 16: fn = (const void*)kern::csr_vector4_fn<T, RP, 16>(bi, ri); break;
      case 32: fn = (const void*)kern::csr_vector4_fn<T, RP, 32>(bi, ri); break;
      default: fail(SPMV_ERR_INVALID_ARG, "CSR-vector quad loads take 4, 8, 16 or 32 lanes per row");
    }
    if (((uintptr_t)h->col | (uintptr_t)h->val) & 15)
      fail(SPMV_ERR_UNSUPPORTED, "CSR-vector quad loads: col/val must be 16-byte aligned");
    const LaunchAttrs attrs(fn, L.carveout_pct);
    const int ur = lanes >= 16 ? 2 : 1;
    const int64_t groups = (h->rows + ur - 1) / ur;
    const int64_t grid = persistent_grid(fn, L.block, (groups * lanes + L.block - 1) / L.block);
    if (grid <= 0) return;
    if (e.mode == 1) {
      ensure_pi_scratch(h, (size_t)grid);
      p.e.partials = h->pi_partials;
      p.e.counter = h->pi_counter;
    }
    void* args[] = {&p};
    launch_checked(fn, dim3((unsigned)grid), dim3(L.block), args, 0, h->stream);
    return;
  }
  if (!merge) {
    const int lanes = L.knob;
    const void* fn;
    switch (lanes) {
      case 1: fn = (const void*)kern::csr_vector_fn<T, RP, 1>(bi, ri); break;
      case 2: fn = (const void*)kern::csr_vector_fn<T, RP, 2>(bi, ri); break;
      case 4: fn = (const void*)kern::csr_vector_fn<T, RP, 4>(bi, ri); break;
      case 8: fn = (const void*)kern::csr_vector_fn<T, RP, 8>(bi, ri); break;
      case 16: fn = (const void*)kern::csr_vector_fn<T, RP, 16>(bi, ri); break;
      case 32: fn = (const void*)kern::csr_vector_fn<T, RP, 32>(bi, ri); break;
      default: fail(SPMV_ERR_INVALID_ARG, "CSR-vector lanes per row must be 1,2,4,8,16 or 32");
    }
    const LaunchAttrs attrs(fn, L.carveout_pct);
    const int ur = lanes >= 16 ? 4 : (lanes >= 4 ? 2 : 1);
    const int64_t groups = (h->rows + ur - 1) / ur;
    const int64_t grid = persistent_grid(fn, L.block, (groups * lanes + L.block - 1) / L.block);
    if (grid <= 0) return;
    if (e.mode == 1) {
      ensure_pi_scratch(h, (size_t)grid);
      p.e.partials = h->pi_partials;
      p.e.counter = h->pi_counter;
    }
    void* args[] = {&p};
    launch_checked(fn, dim3((unsigned)grid), dim3(L.block), args, 0, h->stream);
    return;
  }
  if (L.knob & kern::kMergeRowmap) {
    // nnz-split chunks of 256 entries with the cached row map; empty rows from the handle's list
    if ((L.knob & 0xff) != 8) fail(SPMV_ERR_INVALID_ARG, "row-map CSR takes 8 entries per lane");
    const void* fn = (const void*)kern::csr_nnz_map_fn<T, RP>(bi, ri);
    if (((uintptr_t)h->col | (uintptr_t)h->val) & 15)
      fail(SPMV_ERR_UNSUPPORTED, "row-map CSR: col/val must be 16-byte aligned for the vector loads");
    build_csr_empty(h);
    run_rows_scale(h, h->csr_empty, h->csr_n_empty, e, y);  // disjoint from every row the chunks write
    if (h->nnz <= 0) return;
    build_csr_rowmap(h);
    const int64_t nchunks = h->rm_nchunks;
    const LaunchAttrs attrs(fn, L.carveout_pct);
    p.recs = static_cast<ChunkRec*>(ensure_seg_scratch(h, (size_t)nchunks * sizeof(ChunkRec)));
    p.nchunks = nchunks;
    p.rm_bits = h->rm_bits;
    p.rm_rows = h->rm_rows;
    p.rm_ord0 = h->rm_ord0;
    p.rm_identity = h->csr_n_empty == 0;
    void* args[] = {&p};
    launch_checked(fn, dim3((unsigned)((nchunks * 32 + L.block - 1) / L.block)), dim3(L.block), args, 0, h->stream);
    run_seg_fixup(h, p.recs, nchunks, e, y);
    return;
  }
  if (L.knob & kern::kMergeNnz) {
    // nnz-split chunks: 32·W entries per warp; empty rows from the handle's list
    const int W = L.knob & 0xff;
    const void* fn;
    switch (W) {
      case 4: fn = (const void*)kern::csr_nnz_fn<T, RP, 4>(bi, ri); break;
      case 8: fn = (const void*)kern::csr_nnz_fn<T, RP, 8>(bi, ri); break;
      default: fail(SPMV_ERR_INVALID_ARG, "nnz-split CSR entries per lane must be 4 or 8");
    }
    if (((uintptr_t)h->col | (uintptr_t)h->val) & 15)
      fail(SPMV_ERR_UNSUPPORTED, "nnz-split CSR: col/val must be 16-byte aligned for the vector loads");
    build_csr_empty(h);
    run_rows_scale(h, h->csr_empty, h->csr_n_empty, e, y);  // disjoint from every row the chunks write
    if (h->nnz <= 0) return;
    const int64_t per = 32LL * W;
    const int64_t nchunks = (h->nnz + per - 1) / per;
    const LaunchAttrs attrs(fn, L.carveout_pct);
    p.recs = static_cast<ChunkRec*>(ensure_seg_scratch(h, (size_t)nchunks * sizeof(ChunkRec)));
    if (!h->merge_coords || h->merge_coords_ipt != -per || h->merge_coords_n != nchunks) {
      dfree(h->merge_coords, h->stream);
      h->merge_coords = nullptr;
      h->merge_coords = static_cast<int64_t*>(dalloc((size_t)(nchunks + 1) * sizeof(int64_t), h->stream));
      kern::nnz_partition(h->row_ptr, h->rp64, h->rows, h->nnz, per, nchunks, h->merge_coords, h->stream);
      h->merge_coords_ipt = (int)-per;
      h->merge_coords_n = nchunks;
    }
    p.coords = h->merge_coords;
    p.nchunks = nchunks;
    void* args[] = {&p};
    launch_checked(fn, dim3((unsigned)((nchunks * 32 + L.block - 1) / L.block)), dim3(L.block), args, 0, h->stream);
    run_seg_fixup(h, p.recs, nchunks, e, y);
    return;
  }
  const bool tile = (L.knob & kern::kMergeTile) != 0, pipe = (L.knob & kern::kMergeStream) != 0;
  const int ipt = L.knob & 0xff;
  if (tile && pipe) fail(SPMV_ERR_INVALID_ARG, "merge-path knob: kMergeTile and kMergeStream are exclusive");
  const void* fn;
#define MERGE_PICK(I)                                                              \
  fn = pipe ? (const void*)kern::csr_merge_stream_fn<T, RP, I>(bi, ri)            \
            : (tile ? (const void*)kern::csr_merge_tile_fn<T, RP, I>(bi, ri)      \
                    : (const void*)kern::csr_merge_fn<T, RP, I>(bi, ri))
  switch (ipt) {
    case 4: MERGE_PICK(4); break;
    case 8: MERGE_PICK(8); break;
    case 16: MERGE_PICK(16); break;
    case 32:  // tiles only: a tile of block·32 items keeps every thread on a row of a ~30-entry stencil
      if (!tile && !pipe) fail(SPMV_ERR_INVALID_ARG, "merge-path per-warp walk takes 4, 8 or 16 items per thread");
      fn = pipe ? (const void*)kern::csr_merge_stream_fn<T, RP, 32>(bi, ri)
                : (const void*)kern::csr_merge_tile_fn<T, RP, 32>(bi, ri);
      break;
    default: fail(SPMV_ERR_INVALID_ARG, "merge-path items per thread must be 4, 8 or 16 (| kMergeTile or kMergeStream)");
  }
#undef MERGE_PICK
  if (!fn) fail(SPMV_ERR_UNSUPPORTED, "merge-path tile: block (+ producer warp) × items exceeds the block or shared memory");
  if (pipe && (((uintptr_t)h->col | (uintptr_t)h->val | (uintptr_t)h->row_ptr) & 15))
    fail(SPMV_ERR_UNSUPPORTED, "merge-path stream: row_ptr/col/val must be 16-byte aligned for the bulk copies");
  const size_t smem = pipe ? kern::merge_stream_smem<T, RP>(L.block, ipt)
                           : (tile ? kern::merge_tile_smem<T>(L.block, ipt) : kern::merge_smem_bytes<T>(L.block, ipt));
  const LaunchAttrs attrs(fn, L.carveout_pct, smem);
  const int64_t total = h->rows + h->nnz;
  const int64_t items = (tile || pipe) ? (int64_t)L.block * ipt : 32LL * ipt;
  const int64_t nchunks = (total + items - 1) / items;
  if (nchunks <= 0) return;
  p.recs = static_cast<ChunkRec*>(ensure_seg_scratch(h, (size_t)nchunks * sizeof(ChunkRec)));
  // chunk coordinates depend only on the CSR arrays and the items per chunk
  if (!h->merge_coords || h->merge_coords_ipt != items || h->merge_coords_n != nchunks) {
    dfree(h->merge_coords, h->stream);
    h->merge_coords = nullptr;
    h->merge_coords = static_cast<int64_t*>(dalloc((size_t)(nchunks + 1) * 2 * sizeof(int64_t), h->stream));
    kern::merge_partition(h->row_ptr, h->rp64, h->rows, h->nnz, items, nchunks, h->merge_coords, h->stream);
    h->merge_coords_ipt = items;
    h->merge_coords_n = nchunks;
  }
  p.coords = h->merge_coords;
  p.nchunks = nchunks;
  // mode 1 (power step): alpha from device, beta = 0; the norms are computed
  // afterwards by run_norms because boundary rows finish in the fixup.
  const int64_t grid = pipe ? persistent_grid(fn, L.block + 32, nchunks, smem)
                            : (tile ? nchunks : (nchunks * 32 + L.block - 1) / L.block);
  const int threads = pipe ? L.block + 32 : L.block;
  void* args[] = {&p};
  launch_checked(fn, dim3((unsigned)grid), dim3(threads), args, smem, h->stream);
  run_seg_fixup(h, p.recs, nchunks, e, y);
}

void run_csr(spmv_matrix* h, const Epilogue& e, const void* x, void* y, const spmv_launch_t& L) {
  if (h->dtype == SPMV_R64F) {
    if (h->rp64) csr_typed<double, int64_t>(h, e, x, y, L);
    else csr_typed<double, int32_t>(h, e, x, y, L);
  } else {
    if (h->rp64) csr_typed<float, int64_t>(h, e, x, y, L);
    else csr_typed<float, int32_t>(h, e, x, y, L);
  }
}

}  // namespace spmv
