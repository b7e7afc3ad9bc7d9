// Hot-loop kernels of the V-cycle: fused residual+smoother sweep (with the
// previous cycle's history norm folded in), fused residual+full-weighting
// restriction, residual norm.  fp64, HBM-bound.
//
// Two storage modes for the operator A and the smoother kernels M:
//  * per-point planes: 9 fp64 planes per table (the reference data model,
//    grid.py:163 StencilField / smoothers.py:291 InferredSmoother);
//  * stencil classes: when a level's table is constant away from the boundary
//    (every constant-coefficient problem and its Galerkin chain), the table is
//    exactly represented by 25 "band classes" — 5 row bands x 5 column bands,
//    band(i) = 0, 1 for the first two rows, 3, 4 for the last two, 2 inside.
//    The class tables (25 x 9 doubles) live in shared memory, so a sweep streams
//    only u and f.  The classification is verified point-by-point on the device
//    (mgb_api.cu classify), so both modes compute bit-identical values.
//
// Reference map: residual grid.py:216-226 + hierarchy.py:107-111; smoother
// smoothers.py:325-343; restriction transfer.py:108-121; history norm
// hierarchy.py:129-141.
#include "mgb_cycle.h"

namespace mgb {
namespace {

constexpr int BX = 32, BY = 8, NT = BX * BY;
constexpr int NCLS = 25;

__device__ __forceinline__ int band(int i, int n) { return i < 2 ? i : (i >= n - 2 ? 4 - (n - 1 - i) : 2); }
__device__ __forceinline__ bool act(const uint8_t* m, int64_t p) { return m == nullptr || m[p] != 0; }

__constant__ double c_fw2[9] = {1.0 / 16, 2.0 / 16, 1.0 / 16, 2.0 / 16, 4.0 / 16,
                                2.0 / 16, 1.0 / 16, 2.0 / 16, 1.0 / 16};

__device__ __forceinline__ double block_sum2(double v, double* sh) {
  const int lane = threadIdx.x & 31, wid = (threadIdx.y * blockDim.x + threadIdx.x) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  const int nw = (blockDim.x * blockDim.y) >> 5;
  if (wid == 0) {
    t = lane < nw ? sh[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
  }
  return t;
}

// table value: classed (shared-memory copy) or per-point plane
template <bool CLS>
__device__ __forceinline__ double tv(const Op& t, const double* sh, int b, int s, int o, int64_t p, int cls) {
  if (CLS) return sh[(cls * t.ks + s) * 9 + o];
  return __ldg(t.planes + (int64_t)b * t.ks * 9 * t.n + ((int64_t)s * 9 + o) * t.n + p);
}

template <bool CLS>
__device__ __forceinline__ void load_cls(const Op& t, double* sh, int b, int tid) {
  if (CLS)
    for (int q = tid; q < NCLS * 9 * t.ks; q += NT) sh[q] = t.cls[(int64_t)b * NCLS * 9 * t.ks + q];
}

// ---------------------------------------------------------------------------
// fused sweep: uo = u + M (f - A u) on a TY x TX tile.  u (halo 2) is staged in
// shared memory, the residual over the tile + halo 1 is computed once into
// shared memory, then the 3x3 smoother reads it.  NORM: per-block sum of r^2
// over the tile's own points (r is the residual of the INPUT u, i.e. the
// previous cycle's history residual when this is the first pre-sweep).

constexpr int TX = 32, TY = 32;

template <bool ZU, bool CA, bool CK, bool NORM>
__global__ void __launch_bounds__(NT) k_sweep_t(Grid g, Op A, Op K, const uint8_t* __restrict__ mask,
                                                const double* __restrict__ f, const double* __restrict__ u,
                                                double* __restrict__ uo, double* __restrict__ partials) {
  constexpr int UW = TX + 4, UH = TY + 4, RW = TX + 2, RH = TY + 2;
  __shared__ double us[ZU ? 1 : UH * UW];
  __shared__ double rs[RH * RW];
  __shared__ double tA[CA ? NCLS * 9 : 1];
  __shared__ double tK[CK ? NCLS * 9 : 1];
  __shared__ double red[32];
  const int b = blockIdx.z;
  const int64_t n = g.n();
  const int i0 = blockIdx.y * TY, j0 = blockIdx.x * TX;
  const int tid = threadIdx.y * BX + threadIdx.x;
  const double* fb = f + b * n;
  load_cls<CA>(A, tA, b, tid);
  load_cls<CK>(K, tK, b, tid);
  if (!ZU) {
    const double* ub = u + b * n;
    for (int q = tid; q < UH * UW; q += NT) {
      const int qi = q / UW, qj = q - qi * UW;
      const int i = i0 - 2 + qi, j = j0 - 2 + qj;
      us[q] = (i >= 0 && i < g.rows && j >= 0 && j < g.cols) ? __ldg(ub + (int64_t)i * g.cols + j) : 0.0;
    }
  }
  __syncthreads();
  double acc = 0.0;
  for (int q = tid; q < RH * RW; q += NT) {
    const int ri = q / RW, rj = q - ri * RW;
    const int i = i0 - 1 + ri, j = j0 - 1 + rj;
    double r = 0.0;
    if (i >= 0 && i < g.rows && j >= 0 && j < g.cols) {
      const int64_t p = (int64_t)i * g.cols + j;
      if (act(mask, p)) {
        if (ZU) {
          r = __ldg(fb + p) - 0.0;
        } else {
          const int cls = CA ? band(i, g.rows) * 5 + band(j, g.cols) : 0;
          double s = 0.0;
#pragma unroll
          for (int di = 0; di < 3; ++di)
#pragma unroll
            for (int dj = 0; dj < 3; ++dj)
              s = s + tv<CA>(A, tA, b, 0, di * 3 + dj, p, cls) * us[(ri + di) * UW + rj + dj];
          r = __ldg(fb + p) - s;
        }
      }
      if (NORM && ri >= 1 && ri <= TY && rj >= 1 && rj <= TX) acc += r * r;
    }
    rs[q] = r;
  }
  __syncthreads();
  for (int ti = threadIdx.y; ti < TY; ti += BY) {
    const int i = i0 + ti;
    if (i >= g.rows) break;
    const int tj = threadIdx.x;
    const int j = j0 + tj;
    if (j >= g.cols) continue;
    const int64_t p = (int64_t)i * g.cols + j;
    const int cls = CK ? band(i, g.rows) * 5 + band(j, g.cols) : 0;
    double c = 0.0;
#pragma unroll
    for (int di = 0; di < 3; ++di)
#pragma unroll
      for (int dj = 0; dj < 3; ++dj)
        c = c + tv<CK>(K, tK, b, 0, di * 3 + dj, p, cls) * rs[(ti + di) * RW + tj + dj];
    double v;
    if (!act(mask, p)) v = 0.0;
    else v = ZU ? 0.0 + c : us[(ti + 2) * UW + tj + 2] + c;
    uo[b * n + p] = v;
  }
  if (NORM) {
    const double t = block_sum2(acc, red);
    if (tid == 0) partials[(int64_t)b * gridDim.x * gridDim.y + blockIdx.y * gridDim.x + blockIdx.x] = t;
  }
}

// ---------------------------------------------------------------------------
// rc = R (f - A u): coarse tile CTY x CTX, fine residual region (2CTY+1) x (2CTX+1)
// in shared memory, u region with halo 1 staged too.

constexpr int CTX = 32, CTY = 16;

template <bool ZU, bool CA>
__global__ void __launch_bounds__(NT) k_resid_restrict_t(Grid g, Op A, const uint8_t* __restrict__ mask_f,
                                                         const uint8_t* __restrict__ mask_c,
                                                         const double* __restrict__ f,
                                                         const double* __restrict__ u,
                                                         double* __restrict__ rc) {
  constexpr int FW = 2 * CTX + 1, FH = 2 * CTY + 1, UW = FW + 2, UH = FH + 2;
  __shared__ double us[ZU ? 1 : UH * UW];
  __shared__ double rs[FH * FW];
  __shared__ double tA[CA ? NCLS * 9 : 1];
  const int b = blockIdx.z;
  const int64_t n = g.n();
  const int rows_c = g.rows / 2, cols_c = g.cols / 2;
  const int ci0 = blockIdx.y * CTY, cj0 = blockIdx.x * CTX;
  const int fi0 = 2 * ci0, fj0 = 2 * cj0;
  const int tid = threadIdx.y * BX + threadIdx.x;
  const double* fb = f + b * n;
  load_cls<CA>(A, tA, b, tid);
  if (!ZU) {
    const double* ub = u + b * n;
    for (int q = tid; q < UH * UW; q += NT) {
      const int qi = q / UW, qj = q - qi * UW;
      const int i = fi0 - 1 + qi, j = fj0 - 1 + qj;
      us[q] = (i >= 0 && i < g.rows && j >= 0 && j < g.cols) ? __ldg(ub + (int64_t)i * g.cols + j) : 0.0;
    }
  }
  __syncthreads();
  for (int q = tid; q < FH * FW; q += NT) {
    const int ri = q / FW, rj = q - ri * FW;
    const int i = fi0 + ri, j = fj0 + rj;
    double r = 0.0;
    if (i < g.rows && j < g.cols) {
      const int64_t p = (int64_t)i * g.cols + j;
      if (act(mask_f, p)) {
        if (ZU) {
          r = __ldg(fb + p) - 0.0;
        } else {
          const int cls = CA ? band(i, g.rows) * 5 + band(j, g.cols) : 0;
          double s = 0.0;
#pragma unroll
          for (int di = 0; di < 3; ++di)
#pragma unroll
            for (int dj = 0; dj < 3; ++dj)
              s = s + tv<CA>(A, tA, b, 0, di * 3 + dj, p, cls) * us[(ri + di) * UW + rj + dj];
          r = __ldg(fb + p) - s;
        }
      }
    }
    rs[q] = r;
  }
  __syncthreads();
  for (int ti = threadIdx.y; ti < CTY; ti += BY) {
    const int ci = ci0 + ti;
    if (ci >= rows_c) break;
    const int tj = threadIdx.x;
    const int cj = cj0 + tj;
    if (cj >= cols_c) continue;
    double s = 0.0;
#pragma unroll
    for (int di = 0; di < 3; ++di)
#pragma unroll
      for (int dj = 0; dj < 3; ++dj) s = s + c_fw2[di * 3 + dj] * rs[(2 * ti + di) * FW + 2 * tj + dj];
    const int64_t pc = (int64_t)ci * cols_c + cj;
    rc[b * (int64_t)rows_c * cols_c + pc] = act(mask_c, pc) ? s : 0.0;
  }
}

// ---------------------------------------------------------------------------
// residual norm (history / ||f||): per-block sum of r^2, 32 x 64 points per block

constexpr int NRPT = 8;

template <bool ZU, bool CA>
__global__ void __launch_bounds__(NT) k_resnorm_t(Grid g, Op A, const uint8_t* __restrict__ mask,
                                                  const double* __restrict__ f, const double* __restrict__ u,
                                                  double* __restrict__ partials) {
  __shared__ double tA[CA ? NCLS * 9 : 1];
  __shared__ double red[32];
  const int b = blockIdx.z;
  const int tid = threadIdx.y * BX + threadIdx.x;
  const int64_t n = g.n();
  load_cls<CA>(A, tA, b, tid);
  if (CA) __syncthreads();
  const int j = blockIdx.x * BX + threadIdx.x;
  const double* ub = ZU ? nullptr : u + b * n;
  double acc = 0.0;
  for (int q = 0; q < NRPT; ++q) {
    const int i = (blockIdx.y * NRPT + q) * BY + threadIdx.y;
    if (i < g.rows && j < g.cols) {
      const int64_t p = (int64_t)i * g.cols + j;
      double v = 0.0;
      if (act(mask, p)) {
        if (ZU) {
          v = __ldg(f + b * n + p) - 0.0;
        } else {
          const int cls = CA ? band(i, g.rows) * 5 + band(j, g.cols) : 0;
          double s = 0.0;
#pragma unroll
          for (int di = -1; di <= 1; ++di) {
            const int ii = i + di;
#pragma unroll
            for (int dj = -1; dj <= 1; ++dj) {
              const int jj = j + dj;
              const double w = tv<CA>(A, tA, b, 0, (di + 1) * 3 + dj + 1, p, cls);
              const double x = (ii >= 0 && ii < g.rows && jj >= 0 && jj < g.cols)
                                   ? __ldg(ub + (int64_t)ii * g.cols + jj) : 0.0;
              s = s + w * x;
            }
          }
          v = __ldg(f + b * n + p) - s;
        }
      }
      acc += v * v;
    }
  }
  const double t = block_sum2(acc, red);
  if (tid == 0) partials[(int64_t)b * gridDim.x * gridDim.y + blockIdx.y * gridDim.x + blockIdx.x] = t;
}

// ---------------------------------------------------------------------------
// stencil-class detection: flag |= 1 if a point's table differs from its class
// representative; then gather the 25 class tables.

__global__ void k_classify(Grid g, Op T, const int64_t* __restrict__ rep, int* __restrict__ flag) {
  const int j = blockIdx.x * BX + threadIdx.x, i = blockIdx.y * BY + threadIdx.y, b = blockIdx.z;
  if (i >= g.rows || j >= g.cols) return;
  const int64_t p = (int64_t)i * g.cols + j;
  const int64_t rp = rep[band(i, g.rows) * 5 + band(j, g.cols)];
  bool diff = false;
  for (int s = 0; s < T.ks; ++s)
    for (int o = 0; o < 9; ++o)
      diff |= tv<false>(T, nullptr, b, s, o, p, 0) != tv<false>(T, nullptr, b, s, o, rp, 0);
  if (diff) atomicOr(flag, 1);
}

// flag |= 1 if a corner entry (planes 0, 2, 6, 8) of a k = 3 table is nonzero anywhere:
// a 5-point operator, whose corner planes the per-point streaming passes skip
__global__ void k_corner_check(int64_t n, int batch, const double* __restrict__ planes, int* __restrict__ flag) {
  const int64_t total = n * batch;
  bool nz = false;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = q / n, p = q - b * n;
    const double* t = planes + b * 9 * n + p;
    nz |= t[0] != 0.0 || t[2 * n] != 0.0 || t[6 * n] != 0.0 || t[8 * n] != 0.0;
  }
  if (__syncthreads_or(nz) && threadIdx.x == 0) atomicOr(flag, 1);
}

__global__ void k_gather_cls(Grid g, Op T, const int64_t* __restrict__ rep, double* __restrict__ out) {
  const int b = blockIdx.x;
  for (int q = threadIdx.x; q < NCLS * T.ks * 9; q += blockDim.x) {
    const int c = q / (T.ks * 9), s = (q / 9) % T.ks, o = q % 9;
    out[(int64_t)b * NCLS * T.ks * 9 + q] = rep[c] >= 0 ? tv<false>(T, nullptr, b, s, o, rep[c], 0) : 0.0;
  }
}

}  // namespace

bool classed(const Op& t) { return t.cls != nullptr; }

int sweep_blocks(const Grid& g) { return ((g.cols + TX - 1) / TX) * ((g.rows + TY - 1) / TY); }

cudaError_t launch_sweep2(const Grid& g, const Op& A, const Op& K, const uint8_t* mask, const double* f,
                          const double* u, double* uo, double* partials, cudaStream_t s) {
  ++g_launches;
  dim3 grid((g.cols + TX - 1) / TX, (g.rows + TY - 1) / TY, g.batch);
  dim3 blk(BX, BY);
  const bool ca = classed(A), ck = classed(K), zu = u == nullptr, nm = partials != nullptr;
#define MGB_SW(ZU_, CA_, CK_, NM_) \
  if (zu == ZU_ && ca == CA_ && ck == CK_ && nm == NM_) { \
    k_sweep_t<ZU_, CA_, CK_, NM_><<<grid, blk, 0, s>>>(g, A, K, mask, f, u, uo, partials); \
    return MGB_DBG(__func__); }
  MGB_SW(false, false, false, false) MGB_SW(false, false, false, true)
  MGB_SW(false, false, true, false)  MGB_SW(false, false, true, true)
  MGB_SW(false, true, false, false)  MGB_SW(false, true, false, true)
  MGB_SW(false, true, true, false)   MGB_SW(false, true, true, true)
  MGB_SW(true, false, false, false)  MGB_SW(true, false, false, true)
  MGB_SW(true, false, true, false)   MGB_SW(true, false, true, true)
  MGB_SW(true, true, false, false)   MGB_SW(true, true, false, true)
  MGB_SW(true, true, true, false)    MGB_SW(true, true, true, true)
#undef MGB_SW
  return cudaErrorInvalidValue;
}

cudaError_t launch_resid_restrict2(const Grid& g, const Op& A, const uint8_t* mask_f, const uint8_t* mask_c,
                                   const double* f, const double* u, double* rc, cudaStream_t s) {
  ++g_launches;
  const int rows_c = g.rows / 2, cols_c = g.cols / 2;
  dim3 grid((cols_c + CTX - 1) / CTX, (rows_c + CTY - 1) / CTY, g.batch);
  dim3 blk(BX, BY);
  const bool ca = classed(A), zu = u == nullptr;
  if (zu && ca) k_resid_restrict_t<true, true><<<grid, blk, 0, s>>>(g, A, mask_f, mask_c, f, u, rc);
  else if (zu) k_resid_restrict_t<true, false><<<grid, blk, 0, s>>>(g, A, mask_f, mask_c, f, u, rc);
  else if (ca) k_resid_restrict_t<false, true><<<grid, blk, 0, s>>>(g, A, mask_f, mask_c, f, u, rc);
  else k_resid_restrict_t<false, false><<<grid, blk, 0, s>>>(g, A, mask_f, mask_c, f, u, rc);
  return MGB_DBG(__func__);
}

int resnorm_blocks(const Grid& g) {
  return ((g.cols + BX - 1) / BX) * ((g.rows + BY * NRPT - 1) / (BY * NRPT));
}

cudaError_t launch_resnorm(const Grid& g, const Op& A, const uint8_t* mask, const double* f, const double* u,
                           double* partials, cudaStream_t s) {
  ++g_launches;
  dim3 grid((g.cols + BX - 1) / BX, (g.rows + BY * NRPT - 1) / (BY * NRPT), g.batch);
  dim3 blk(BX, BY);
  const bool ca = classed(A), zu = u == nullptr;
  if (zu) k_resnorm_t<true, false><<<grid, blk, 0, s>>>(g, A, mask, f, u, partials);
  else if (ca) k_resnorm_t<false, true><<<grid, blk, 0, s>>>(g, A, mask, f, u, partials);
  else k_resnorm_t<false, false><<<grid, blk, 0, s>>>(g, A, mask, f, u, partials);
  return MGB_DBG(__func__);
}

cudaError_t launch_classify(const Grid& g, const Op& T, const int64_t* rep, int* flag, cudaStream_t s) {
  ++g_launches;
  dim3 grid((g.cols + BX - 1) / BX, (g.rows + BY - 1) / BY, g.batch);
  k_classify<<<grid, dim3(BX, BY), 0, s>>>(g, T, rep, flag);
  return MGB_DBG(__func__);
}

cudaError_t launch_corner_check(int64_t n, int batch, const double* planes, int* flag, cudaStream_t s) {
  ++g_launches;
  k_corner_check<<<4 * 148, 256, 0, s>>>(n, batch, planes, flag);
  return MGB_DBG(__func__);
}

cudaError_t launch_gather_cls(const Grid& g, const Op& T, const int64_t* rep, double* out, cudaStream_t s) {
  ++g_launches;
  k_gather_cls<<<g.batch, 256, 0, s>>>(g, T, rep, out);
  return MGB_DBG(__func__);
}

int host_band(int i, int n) { return i < 2 ? i : (i >= n - 2 ? 4 - (n - 1 - i) : 2); }

}  // namespace mgb
