// Shared-kernel convolutional smoother (mgb_conv.cu).
#pragma once

#include "mgb_internal.h"

namespace mgb {

struct ConvW {
  double w[9];  // [di + 1][dj + 1]
};

constexpr int CONV_MAX_LAYERS = 8;

// ConvSmoother (smoothers.py:105-145): nl chained 3x3 layers, optional skip,
// leaky activation between chained layers, output gain
struct ConvSm {
  int nl = 0;
  ConvW layer[CONV_MAX_LAYERS];
  bool has_skip = false;
  ConvW skip;
  bool leaky = false;
  double slope = 0.01;
  double gain = 1.0;
};

// dst = mask ? sum_{w != 0} w * act(src(p + o)) : 0 (convolve, grid.py:229-239)
cudaError_t launch_convolve(const Grid& g, const ConvW& w, const uint8_t* mask, const double* src, double* dst,
                            bool act, double slope, cudaStream_t s);
// u_out = u_in + gain * (v + skip * r)
cudaError_t launch_conv_finish(const Grid& g, const ConvW* skip, const uint8_t* mask, const double* v,
                               const double* r, const double* u_in, double* u_out, double gain, cudaStream_t s);
// out = u_in + M(r)  (u_in == null: out = M(r)); t1, t2 scratch distinct from r, u_in
cudaError_t conv_smoother_apply(const Grid& g, const ConvSm& cs, const uint8_t* mask, const double* r,
                                const double* u_in, double* out, double* t1, double* t2, cudaStream_t s);

}  // namespace mgb
