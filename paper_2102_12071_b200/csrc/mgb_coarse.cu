// The coarse end of the V-cycle in ONE launch: a thread-block cluster per problem
// runs every level below a size threshold (sweeps, residual, restriction, the
// coarsest LU solve, prolongation) with cluster barriers between dependent
// phases instead of kernel boundaries.  Coarse levels are latency-bound (a few
// thousand points each); as separate kernels each pass costs a launch and a
// memory round trip, here a phase costs a cluster barrier.
//
// Reference: v_cycle hierarchy.py:96-111 (V(nu1, nu2) as RepeatedSmoother,
// cli.py:365-377), coarse_solve hierarchy.py:91-93 / lu_solve dense.py:50-63,
// restrict transfer.py:108-121, prolong transfer.py:124-147.
#include <cooperative_groups.h>

#include "mgb_coarse.h"

namespace cg = cooperative_groups;

namespace mgb {
namespace {

constexpr int CT = 1024;  // threads per CTA
constexpr int NCLS = 25;

__device__ __forceinline__ int bandk(int i, int n) { return i < 2 ? i : (i >= n - 2 ? 4 - (n - 1 - i) : 2); }

// weight o of a table at point p = (i, j): band class table or per-point plane
__device__ __forceinline__ double wgt(const Op& t, int b, int o, int64_t p, int i, int j, int rows, int cols) {
  if (t.cls) return __ldg(t.cls + ((int64_t)b * NCLS + bandk(i, rows) * 5 + bandk(j, cols)) * 9 + o);
  return __ldg(t.planes + (int64_t)b * 9 * t.n + (int64_t)o * t.n + p);
}

// sum_o T(p)[o] v(p + o), zero outside the grid (plain loads: v is written in-kernel)
__device__ __forceinline__ double apply9(const Op& t, int b, const double* v, int i, int j, int rows, int cols) {
  const int64_t p = (int64_t)i * cols + j;
  double s = 0.0;
#pragma unroll
  for (int di = -1; di <= 1; ++di) {
    const int ii = i + di;
    if (ii < 0 || ii >= rows) continue;
#pragma unroll
    for (int dj = -1; dj <= 1; ++dj) {
      const int jj = j + dj;
      if (jj < 0 || jj >= cols) continue;
      s = fma(wgt(t, b, (di + 1) * 3 + dj + 1, p, i, j, rows, cols), v[(int64_t)ii * cols + jj], s);
    }
  }
  return s;
}

__global__ void __cluster_dims__(COARSE_CLUSTER, 1, 1) __launch_bounds__(CT)
    k_coarse_cluster(CoarseArgs a) {
  extern __shared__ double xs[];
  cg::cluster_group cl = cg::this_cluster();
  const int b = blockIdx.y;
  const int rank = (int)cl.block_rank();
  const int gt = rank * CT + threadIdx.x;
  constexpr int GT = COARSE_CLUSTER * CT;

  // one smoothing sweep on level l: r = f - A u (u = 0 if zero), then u = u + M r
  auto sweep = [&](const CLevel& L, bool zero) {
    const int64_t n = (int64_t)L.rows * L.cols;
    double* u = L.u + b * n;
    const double* f = L.f + b * n;
    double* r = L.r + b * n;
    for (int64_t p = gt; p < n; p += GT) {
      const int i = (int)(p / L.cols), j = (int)(p % L.cols);
      double v = 0.0;
      if (!L.mask || L.mask[p]) v = zero ? f[p] : f[p] - apply9(L.A, b, u, i, j, L.rows, L.cols);
      r[p] = v;
    }
    cl.sync();
    for (int64_t p = gt; p < n; p += GT) {
      const int i = (int)(p / L.cols), j = (int)(p % L.cols);
      double v = 0.0;
      if (!L.mask || L.mask[p]) v = (zero ? 0.0 : u[p]) + apply9(L.K, b, r, i, j, L.rows, L.cols);
      u[p] = v;
    }
    cl.sync();
  };

  // descend
  for (int l = 0; l + 1 < a.nlev; ++l) {
    const CLevel& L = a.lv[l];
    const CLevel& Cc = a.lv[l + 1];
    const bool zero0 = l > 0 || a.zero_top;
    for (int q = 0; q < a.nu1; ++q) sweep(L, zero0 && q == 0);
    const int64_t n = (int64_t)L.rows * L.cols;
    double* u = L.u + b * n;
    const double* f = L.f + b * n;
    double* r = L.r + b * n;
    if (a.nu1 == 0 && zero0) {
      for (int64_t p = gt; p < n; p += GT) u[p] = 0.0;
      cl.sync();
    }
    for (int64_t p = gt; p < n; p += GT) {
      const int i = (int)(p / L.cols), j = (int)(p % L.cols);
      double v = 0.0;
      if (!L.mask || L.mask[p]) v = f[p] - apply9(L.A, b, u, i, j, L.rows, L.cols);
      r[p] = v;
    }
    cl.sync();
    const int64_t nc = (int64_t)Cc.rows * Cc.cols;
    double* fc = Cc.f + b * nc;
    for (int64_t pc = gt; pc < nc; pc += GT) {
      const int ci = (int)(pc / Cc.cols), cj = (int)(pc % Cc.cols);
      double s = 0.0;
#pragma unroll
      for (int di = 0; di < 3; ++di)
#pragma unroll
        for (int dj = 0; dj < 3; ++dj) {
          const int fi = 2 * ci + di, fj = 2 * cj + dj;
          const double wv = (di == 1 ? 2.0 : 1.0) * (dj == 1 ? 2.0 : 1.0) * 0.0625;
          if (fi < L.rows && fj < L.cols) s = fma(wv, r[(int64_t)fi * L.cols + fj], s);
        }
      fc[pc] = (!Cc.mask || Cc.mask[pc]) ? s : 0.0;
    }
    cl.sync();
  }
  // coarsest: dense LU solve (dense.py:50-63) in CTA 0
  {
    const CLevel& L = a.lv[a.nlev - 1];
    const int64_t n = (int64_t)L.rows * L.cols;
    if (rank == 0) {
      const int nn = a.nc;
      const double* lu = a.lu + (int64_t)b * nn * nn;
      const int32_t* pm = a.perm + (int64_t)b * nn;
      const double* f = L.f + b * n;
      double* x = L.u + b * n;
      for (int q = threadIdx.x; q < nn; q += CT) xs[q] = f[a.actp[pm[q]]];
      for (int64_t q = threadIdx.x; q < n; q += CT) x[q] = 0.0;
      __syncthreads();
      for (int k = 0; k < nn; ++k) {
        const double xk = xs[k];
        for (int i = k + 1 + threadIdx.x; i < nn; i += CT) xs[i] = xs[i] - lu[(int64_t)i * nn + k] * xk;
        __syncthreads();
      }
      for (int k = nn - 1; k >= 0; --k) {
        if (threadIdx.x == 0) xs[k] = xs[k] / lu[(int64_t)k * nn + k];
        __syncthreads();
        const double xk = xs[k];
        for (int i = threadIdx.x; i < k; i += CT) xs[i] = xs[i] - lu[(int64_t)i * nn + k] * xk;
        __syncthreads();
      }
      for (int q = threadIdx.x; q < nn; q += CT) x[a.actp[q]] = xs[q];
    }
    cl.sync();
  }
  // ascend: u_l += P u_{l+1}, then nu2 sweeps
  for (int l = a.nlev - 2; l >= 0; --l) {
    const CLevel& L = a.lv[l];
    const CLevel& Cc = a.lv[l + 1];
    const int64_t n = (int64_t)L.rows * L.cols;
    const int64_t ncc = (int64_t)Cc.rows * Cc.cols;
    double* u = L.u + b * n;
    const double* ec = Cc.u + b * ncc;
    for (int64_t p = gt; p < n; p += GT) {
      const int i = (int)(p / L.cols), j = (int)(p % L.cols);
      double s = 0.0;
#pragma unroll
      for (int di = -1; di <= 1; ++di) {
        const int t = i - 1 - di;
        if (t < 0 || (t & 1) || (t >> 1) >= Cc.rows) continue;
#pragma unroll
        for (int dj = -1; dj <= 1; ++dj) {
          const int tt = j - 1 - dj;
          if (tt < 0 || (tt & 1) || (tt >> 1) >= Cc.cols) continue;
          const double wv = (di == 0 ? 2.0 : 1.0) * (dj == 0 ? 2.0 : 1.0) * 0.125;
          s = fma(wv, ec[(int64_t)(t >> 1) * Cc.cols + (tt >> 1)], s);
        }
      }
      u[p] = (!L.mask || L.mask[p]) ? u[p] + s : 0.0;
    }
    cl.sync();
    for (int q = 0; q < a.nu2; ++q) sweep(L, false);
  }
}

}  // namespace

cudaError_t launch_coarse_cluster(const CoarseArgs& a, int batch, cudaStream_t s) {
  static bool attr = false;
  const size_t smem = sizeof(double) * (size_t)std::max(a.nc, 1);
  if (!attr || smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_coarse_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)std::max<size_t>(smem, 48 * 1024));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  ++g_launches;
  k_coarse_cluster<<<dim3(COARSE_CLUSTER, batch), CT, smem, s>>>(a);
  return MGB_DBG(__func__);
}

}  // namespace mgb
