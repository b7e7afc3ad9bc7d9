// Hot-loop kernels (mgb_cycle.cu): storage descriptor and launchers.
#pragma once

#include "mgb_internal.h"

namespace mgb {

// A table of ks stages of 3x3 weights per grid point, either as per-point planes
// ([b][s][o][p], plane length n) or, when `cls` is non-null, as 25 band-class
// tables ([b][class][s][o]) that represent it exactly.
struct Op {
  const double* planes;
  const double* cls;
  int64_t n;
  int ks;
};

bool classed(const Op& t);
int host_band(int i, int n);
int sweep_blocks(const Grid& g);
int resnorm_blocks(const Grid& g);

// uo = u + M (f - A u); u == null: u = 0.  partials != null: per-block sum of
// squares of the residual of the input u over the block's own points.
cudaError_t launch_sweep2(const Grid& g, const Op& A, const Op& K, const uint8_t* mask, const double* f,
                          const double* u, double* uo, double* partials, cudaStream_t s);
// rc = R (f - A u); u == null: rc = R f
cudaError_t launch_resid_restrict2(const Grid& g, const Op& A, const uint8_t* mask_f, const uint8_t* mask_c,
                                   const double* f, const double* u, double* rc, cudaStream_t s);
// per-block sums of (f - A u)^2 ; u == null: of f^2
cudaError_t launch_resnorm(const Grid& g, const Op& A, const uint8_t* mask, const double* f, const double* u,
                           double* partials, cudaStream_t s);
// band-class detection and gather (rep: 25 representative flat indices or -1)
cudaError_t launch_classify(const Grid& g, const Op& T, const int64_t* rep, int* flag, cudaStream_t s);
cudaError_t launch_corner_check(int64_t n, int batch, const double* planes, int* flag, cudaStream_t s);
cudaError_t launch_gather_cls(const Grid& g, const Op& T, const int64_t* rep, double* out, cudaStream_t s);

}  // namespace mgb
