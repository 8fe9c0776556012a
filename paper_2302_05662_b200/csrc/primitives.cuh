// primitives.cuh — device-wide scan and LSD radix sort used by the format
// converters. Deterministic: no order-dependent
// atomics feed any output.
#pragma once
#include "common.cuh"

namespace spmv {

// out[0..n] = exclusive prefix sums of in[0..n), out[n] = total. in/out may
// not alias. int64 throughout.
void exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s);

// Stable LSD radix sort of (key, payload) pairs on the low `bits` bits of the
// keys (8-bit digits). payload_in == nullptr means the identity permutation.
// On return keys_out/payload_out hold the sorted sequence. Scratch is
// allocated internally (stream-ordered). n < 2^32.
void radix_sort_pairs(const uint64_t* keys_in, const uint32_t* payload_in, uint64_t* keys_out,
                      uint32_t* payload_out, int64_t n, int bits, cudaStream_t s);

// Number of bits needed to represent values in [0, v] (0 for v == 0).
inline int bits_for(uint64_t v) {
  int b = 0;
  while (b < 64 && (v >> b) != 0) ++b;
  return b;
}

}  // namespace spmv
