// Single-launch coarse V-cycle (mgb_coarse.cu).
#pragma once

#include <algorithm>

#include "mgb_cycle.h"


namespace mgb {

constexpr int COARSE_MAX_LEVELS = 16;

struct CLevel {
  int rows, cols;
  Op A, K;               // ks == 1
  const uint8_t* mask;   // null = all active
  double* u;             // level solution (correction), batch-strided
  double* f;             // level right-hand side
  double* r;             // residual scratch
};

struct CoarseArgs {
  int nlev;              // levels handled: lv[0] (finest of the block) .. lv[nlev-1] (coarsest)
  int nu1, nu2;
  int zero_top;          // lv[0].u starts at zero (not read)
  int nc;                // coarsest active unknowns
  const double* lu;      // coarsest LU (batch x nc x nc)
  const int32_t* perm;
  const int32_t* actp;
  CLevel lv[COARSE_MAX_LEVELS];
};

// shared-memory bytes the block kernel needs for these levels (<= 227 KB to run)
size_t coarse_block_smem(const CoarseArgs& a);
cudaError_t launch_coarse_block(const CoarseArgs& a, int batch, cudaStream_t s);

}  // namespace mgb
