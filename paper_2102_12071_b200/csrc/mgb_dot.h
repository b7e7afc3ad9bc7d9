// The 3x3 stencil dot product shared by the fused V-cycle passes (mgb_stream.cu,
// mgb_tile.cu): init +/- sum_o w[o] x[o] over the window rows r0 (di = -1), r1, r2.
// Both passes evaluate it through this one function, so they round identically.
#pragma once

#ifndef MGB_DOT_CHAINS
#define MGB_DOT_CHAINS 1
#endif

namespace mgb {

// MGB_DOT_CHAINS == 1: one fused-multiply-add chain seeded with init (9 dependent
// FP64 instructions).  3: one chain per window row, summed at the end — a 5-deep
// dependency instead of 9 (the passes are FP64-latency-bound at low occupancy).
template <bool NEG>
__device__ __forceinline__ double stencil_dot(const double* w, const double* r0, const double* r1,
                                              const double* r2, double init) {
#if MGB_DOT_CHAINS == 1
  double a = init;
#pragma unroll
  for (int c = 0; c < 3; ++c) a = fma(NEG ? -w[c] : w[c], r0[c], a);
#pragma unroll
  for (int c = 0; c < 3; ++c) a = fma(NEG ? -w[3 + c] : w[3 + c], r1[c], a);
#pragma unroll
  for (int c = 0; c < 3; ++c) a = fma(NEG ? -w[6 + c] : w[6 + c], r2[c], a);
  return a;
#else
  double a0 = init;
#pragma unroll
  for (int c = 0; c < 3; ++c) a0 = fma(NEG ? -w[c] : w[c], r0[c], a0);
  double a1 = (NEG ? -w[3] : w[3]) * r1[0];
  a1 = fma(NEG ? -w[4] : w[4], r1[1], a1);
  a1 = fma(NEG ? -w[5] : w[5], r1[2], a1);
  double a2 = (NEG ? -w[6] : w[6]) * r2[0];
  a2 = fma(NEG ? -w[7] : w[7], r2[1], a2);
  a2 = fma(NEG ? -w[8] : w[8], r2[2], a2);
  return a0 + (a1 + a2);
#endif
}

}  // namespace mgb
