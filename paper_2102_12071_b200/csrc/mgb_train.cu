// Device kernels of the training path: the backward passes of the
// grid operations the solver loss is built from, the small dense / batched-convolution
// operations of the kernel-inference nets with their backward passes, and Adam.  The
// Python tape (paper_2102_12071_b200/autodiff.py) strings them together exactly as the
// reference's reverse-mode tape does (autodiff.py:139-325, training.py:73-93); forward
// stencil / transfer / LU operations reuse the stateless kernels of mgb_kernels.cu.
//
// Everything is fp64.  Reductions over points (kernel gradients of shared kernels, weight
// gradients of the nets, norms) are deterministic: a fixed grid, per-block tree sums in
// shared memory, then one block sums the partials in index order.
//
//   stencil adjoint        autodiff.py:171-192 (stencil_apply back), :257-280 (pointwise_conv back, du)
//   per-point kernel grad  autodiff.py:268-273
//   shared-kernel grad     autodiff.py:152-159 (conv2d back, dk)
//   conv_batch fwd / bwd   autodiff.py:283-325
//   matmul                 autodiff.py:128-137
//   leaky, sum_axis        autodiff.py:86-96, :109-115
//   lu_solve_t             dense.py:66-80 (coarse_solve_const back, autodiff.py:328-344)
//   Adam                   training.py:73-93
#include <algorithm>
#include <cmath>
#include <cstdint>

#include "mgb_internal.h"

namespace mgb {
namespace {

constexpr int TB = 256;

static cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
static int blocks_for(int64_t n) { return (int)std::min<int64_t>((n + TB - 1) / TB, 65535); }

// ---- elementwise ------------------------------------------------------------------
__global__ void k_axpby(int64_t n, double a, const double* __restrict__ x, double b, const double* __restrict__ y,
                        double* __restrict__ z) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    // a = 1 / b = +-1 reproduce x + y and x - y exactly (no contraction: -fmad=false)
    const double ax = a == 1.0 ? x[i] : a * x[i];
    z[i] = y ? (b == 1.0 ? ax + y[i] : (b == -1.0 ? ax - y[i] : ax + b * y[i])) : ax;
  }
}

__global__ void k_mul(int64_t n, const double* __restrict__ x, const double* __restrict__ c, int64_t cmod,
                      double* __restrict__ z) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    z[i] = x[i] * c[cmod > 0 ? i / cmod : i];
}

// mode 0: z = x * f(x);  mode 1: z = g * f(x)   with f = 1 where x > 0, slope elsewhere
__global__ void k_leaky(int64_t n, const double* __restrict__ x, double slope, const double* __restrict__ g, int mode,
                        double* __restrict__ z) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double f = x[i] > 0.0 ? 1.0 : slope;
    z[i] = (mode == 0 ? x[i] : g[i]) * f;
  }
}

// x (n, c, inner) -> z (n, inner): sum over c in index order
__global__ void k_sum_axis1(int64_t n, int c, int inner, const double* __restrict__ x, double* __restrict__ z) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * inner; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i / inner, q = i - p * inner;
    double s = 0.0;
    for (int k = 0; k < c; ++k) s += x[(p * c + k) * inner + q];
    z[i] = s;
  }
}
// gx (n, c, inner) += g (n, inner) broadcast over c
__global__ void k_bcast_axis1(int64_t n, int c, int inner, const double* __restrict__ g, double* __restrict__ gx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * c * inner;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i / ((int64_t)c * inner), q = i % inner;
    gx[i] += g[p * inner + q];
  }
}

// ---- deterministic reductions -------------------------------------------------------
// sums of term(i) over i < n for `nout` independent outputs: block (o, b) reduces a slice
__device__ __forceinline__ double block_sum(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int s = TB / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  return sh[0];
}

__global__ void k_sum_partials(int nout, int nparts, const double* __restrict__ part, double* __restrict__ out,
                               int accumulate) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= nout) return;
  double s = 0.0;
  for (int b = 0; b < nparts; ++b) s += part[(int64_t)o * nparts + b];
  out[o] = accumulate ? out[o] + s : s;
}

__global__ void k_dot_part(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
                           double* __restrict__ part) {
  __shared__ double sh[TB];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += x[i] * y[i];
  const double t = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// ---- stencil adjoint: du(q) = sum_d T(q - d)[d] gm(q - d), gm = g on the mask --------
// T: (rows, cols, 3, 3) AoS.  mask_in masks g (null: none), mask_out zeroes du off it.
// order 0: offsets o = -d ascending (the transposed-table form of stencil_apply's
// backward); order 1: d ascending (pointwise_conv's backward).
__global__ void k_stencil_adjoint(int rows, int cols, const double* __restrict__ T, const uint8_t* __restrict__ mask_in,
                                  const uint8_t* __restrict__ mask_out, const double* __restrict__ g, int order,
                                  double* __restrict__ du) {
  const int64_t n = (int64_t)rows * cols;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(q / cols), j = (int)(q - (int64_t)i * cols);
    double s = 0.0;
    for (int e = 0; e < 9; ++e) {
      const int dd = order == 0 ? 8 - e : e;          // d index (di + 1) * 3 + (dj + 1)
      const int di = dd / 3 - 1, dj = dd % 3 - 1;
      const int si = i - di, sj = j - dj;             // source point q - d
      if (si < 0 || si >= rows || sj < 0 || sj >= cols) continue;
      const int64_t sp = (int64_t)si * cols + sj;
      const double gv = (mask_in == nullptr || mask_in[sp]) ? g[sp] : 0.0;
      s += T[sp * 9 + dd] * gv;
    }
    du[q] = (mask_out == nullptr || mask_out[q]) ? s : 0.0;
  }
}

// dK(p)[d] (+)= gm(p) u(p + d), zero outside the grid
__global__ void k_pconv_kgrad(int rows, int cols, const uint8_t* __restrict__ mask, const double* __restrict__ g,
                              const double* __restrict__ u, int accumulate, double* __restrict__ dK) {
  const int64_t n = (int64_t)rows * cols;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(p / cols), j = (int)(p - (int64_t)i * cols);
    const double gv = (mask == nullptr || mask[p]) ? g[p] : 0.0;
    for (int d = 0; d < 9; ++d) {
      const int ii = i + d / 3 - 1, jj = j + d % 3 - 1;
      const double uv = (ii < 0 || ii >= rows || jj < 0 || jj >= cols) ? 0.0 : u[(int64_t)ii * cols + jj];
      const double v = gv * uv;
      dK[p * 9 + d] = accumulate ? dK[p * 9 + d] + v : v;
    }
  }
}

// shared-kernel gradient: part[d][block] = sum over the block's points of gm(p) u(p + d)
__global__ void k_conv_kgrad_part(int rows, int cols, int ksize, const uint8_t* __restrict__ mask,
                                  const double* __restrict__ g, const double* __restrict__ u, int nparts,
                                  double* __restrict__ part) {
  __shared__ double sh[TB];
  const int d = blockIdx.y, r = ksize / 2;
  const int di = d / ksize - r, dj = d % ksize - r;
  const int64_t n = (int64_t)rows * cols;
  double s = 0.0;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(p / cols), j = (int)(p - (int64_t)i * cols);
    const int ii = i + di, jj = j + dj;
    if (ii < 0 || ii >= rows || jj < 0 || jj >= cols) continue;
    const double gv = (mask == nullptr || mask[p]) ? g[p] : 0.0;
    s += gv * u[(int64_t)ii * cols + jj];
  }
  const double t = block_sum(s, sh);
  if (threadIdx.x == 0) part[(int64_t)d * nparts + blockIdx.x] = t;
}

// ---- conv_batch: kern (c, 3, 3), img (n, 3, 3) -> out (n, c, 3, 3), zero padding -------
__global__ void k_conv_batch(int64_t n, int c, const double* __restrict__ kern, const double* __restrict__ img,
                             double* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * c * 9; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = t / (c * 9);
    const int ch = (int)((t / 9) % c), i = (int)(t % 9) / 3, j = (int)(t % 3);
    double s = 0.0;
    for (int di = -1; di <= 1; ++di)
      for (int dj = -1; dj <= 1; ++dj) {
        const int ii = i + di, jj = j + dj;
        if (ii < 0 || ii > 2 || jj < 0 || jj > 2) continue;
        s += kern[ch * 9 + (di + 1) * 3 + dj + 1] * img[p * 9 + ii * 3 + jj];
      }
    out[t] = s;
  }
}
// dimg (n, 3, 3) (+)= sum_c sum_d kern[c][d] g[n][c][pos - d]
__global__ void k_conv_batch_dimg(int64_t n, int c, const double* __restrict__ kern, const double* __restrict__ g,
                                  int accumulate, double* __restrict__ dimg) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * 9; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = t / 9;
    const int i = (int)(t % 9) / 3, j = (int)(t % 3);
    double s = 0.0;
    for (int di = -1; di <= 1; ++di)
      for (int dj = -1; dj <= 1; ++dj) {
        const int oi = i - di, oj = j - dj;           // output position that read img(i, j) through offset d
        if (oi < 0 || oi > 2 || oj < 0 || oj > 2) continue;
        for (int ch = 0; ch < c; ++ch) s += kern[ch * 9 + (di + 1) * 3 + dj + 1] * g[(p * c + ch) * 9 + oi * 3 + oj];
      }
    dimg[t] = accumulate ? dimg[t] + s : s;
  }
}
// part[(c, d)][block] = sum over the block's samples of sum_pos g[n][c][pos] img[n][pos + d]
__global__ void k_conv_batch_dk_part(int64_t n, int c, const double* __restrict__ g, const double* __restrict__ img,
                                     int nparts, double* __restrict__ part) {
  __shared__ double sh[TB];
  const int o = blockIdx.y, ch = o / 9, d = o % 9, di = d / 3 - 1, dj = d % 3 - 1;
  double s = 0.0;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        const int ii = i + di, jj = j + dj;
        if (ii < 0 || ii > 2 || jj < 0 || jj > 2) continue;
        s += g[(p * c + ch) * 9 + i * 3 + j] * img[p * 9 + ii * 3 + jj];
      }
  const double t = block_sum(s, sh);
  if (threadIdx.x == 0) part[(int64_t)o * nparts + blockIdx.x] = t;
}

// ---- small dense products: C (M, N) (+)= op(A) op(B), row-major, k summed in order ------
__global__ void k_matmul(int M, int K, int N, const double* __restrict__ A, int ta, const double* __restrict__ B, int tb,
                         int accumulate, double* __restrict__ C) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)M * N; t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t / N), j = (int)(t % N);
    double s = 0.0;
    for (int k = 0; k < K; ++k) {
      const double a = ta ? A[(int64_t)k * M + i] : A[(int64_t)i * K + k];
      const double b = tb ? B[(int64_t)j * K + k] : B[(int64_t)k * N + j];
      s += a * b;
    }
    C[t] = accumulate ? C[t] + s : s;
  }
}
// reductions over many rows (weight gradients: C = A^T B with K = number of points):
// part[(i, j)][block] over a slice of k, then k_sum_partials
__global__ void k_matmul_tn_part(int M, int K, int N, const double* __restrict__ A, const double* __restrict__ B,
                                 int nparts, double* __restrict__ part) {
  __shared__ double sh[TB];
  const int o = blockIdx.y, i = o / N, j = o % N;
  double s = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < K; k += (int64_t)gridDim.x * blockDim.x)
    s += A[k * M + i] * B[k * N + j];
  const double t = block_sum(s, sh);
  if (threadIdx.x == 0) part[(int64_t)o * nparts + blockIdx.x] = t;
}

// ---- transposed LU solve (dense.py:66-80), one block ----------------------------------
__global__ void k_lu_solve_t(int n, const double* __restrict__ lu, const int32_t* __restrict__ perm,
                             const double* __restrict__ b, double* __restrict__ x, double* __restrict__ y) {
  // y lives in global scratch (n <= 4096); one block, barriers between pivots
  for (int i = threadIdx.x; i < n; i += blockDim.x) y[i] = b[i];
  __syncthreads();
  for (int k = 0; k < n; ++k) {           // U^T y = b
    if (threadIdx.x == 0) y[k] = y[k] / lu[(int64_t)k * n + k];
    __syncthreads();
    const double yk = y[k];
    for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) y[i] = y[i] - lu[(int64_t)k * n + i] * yk;
    __syncthreads();
  }
  for (int k = n - 1; k >= 0; --k) {      // L^T w = y (unit diagonal): y[k] -= lu[k+1:, k] . y[k+1:]
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int i = k + 1; i < n; ++i) s += lu[(int64_t)i * n + k] * y[i];
      y[k] = y[k] - s;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) x[perm[i]] = y[i];
}

// ---- Adam (training.py:73-93) -----------------------------------------------------------
__global__ void k_adam(int64_t n, double* __restrict__ p, const double* __restrict__ g, double* __restrict__ m,
                       double* __restrict__ v, double lr, double b1, double b2, double eps, double bc1, double bc2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double gi = g ? g[i] : 0.0;
    const double mi = m[i] * b1 + (1.0 - b1) * gi;
    const double vi = v[i] * b2 + (1.0 - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    p[i] = p[i] - lr * (mi / bc1) / (sqrt(vi / bc2) + eps);
  }
}

constexpr int RED_PARTS = 64;   // blocks per reduced output

}  // namespace
}  // namespace mgb

using namespace mgb;

#define MGB_LAUNCH_OK()                                     \
  do {                                                      \
    ++g_launches;                                           \
    cudaError_t _e = MGB_DBG(__func__);                     \
    if (_e != cudaSuccess) return cuda_fail(_e, __func__);  \
  } while (0)

extern "C" int mgb_ad_axpby(int64_t n, double a, const double* x_dev, double b, const double* y_dev, double* z_dev,
                            void* stream) {
  if (n < 0 || (n > 0 && (!x_dev || !z_dev))) return fail(MGB_CONTRACT, "bad vector arguments");
  if (n == 0) return MGB_OK;
  k_axpby<<<blocks_for(n), TB, 0, S(stream)>>>(n, a, x_dev, b, y_dev, z_dev);
  MGB_LAUNCH_OK();
  return MGB_OK;
}

extern "C" int mgb_ad_mul(int64_t n, const double* x_dev, const double* c_dev, int64_t c_repeat, double* z_dev,
                          void* stream) {
  if (n < 0 || (n > 0 && (!x_dev || !c_dev || !z_dev))) return fail(MGB_CONTRACT, "bad vector arguments");
  if (n == 0) return MGB_OK;
  k_mul<<<blocks_for(n), TB, 0, S(stream)>>>(n, x_dev, c_dev, c_repeat, z_dev);
  MGB_LAUNCH_OK();
  return MGB_OK;
}

extern "C" int mgb_ad_leaky(int64_t n, const double* x_dev, double slope, const double* g_dev, double* z_dev,
                            void* stream) {
  if (n < 0 || (n > 0 && (!x_dev || !z_dev))) return fail(MGB_CONTRACT, "bad vector arguments");
  if (n == 0) return MGB_OK;
  k_leaky<<<blocks_for(n), TB, 0, S(stream)>>>(n, x_dev, slope, g_dev, g_dev ? 1 : 0, z_dev);
  MGB_LAUNCH_OK();
  return MGB_OK;
}

extern "C" int mgb_ad_sum_axis1(int64_t n, int c, int inner, const double* x_dev, double* z_dev, void* stream) {
  if (n <= 0 || c <= 0 || inner <= 0 || !x_dev || !z_dev) return fail(MGB_CONTRACT, "bad sum_axis arguments");
  k_sum_axis1<<<blocks_for(n * inner), TB, 0, S(stream)>>>(n, c, inner, x_dev, z_dev);
  MGB_LAUNCH_OK();
  return MGB_OK;
}

extern "C" int mgb_ad_bcast_axis1(int64_t n, int c, int inner, const double* g_dev, double* gx_dev, void* stream) {
  if (n <= 0 || c <= 0 || inner <= 0 || !g_dev || !gx_dev) return fail(MGB_CONTRACT, "bad broadcast arguments");
  k_bcast_axis1<<<blocks_for(n * c * inner), TB, 0, S(stream)>>>(n, c, inner, g_dev, gx_dev);
  MGB_LAUNCH_OK();
  return MGB_OK;
}

// out_dev[0] = sum x y (y == NULL: sum x x); scratch_dev: RED_PARTS doubles
extern "C" int mgb_ad_dot(int64_t n, const double* x_dev, const double* y_dev, double* scratch_dev, double* out_dev,
                          void* stream) {
  if (n < 0 || !x_dev || !scratch_dev || !out_dev) return fail(MGB_CONTRACT, "bad dot arguments");
  k_dot_part<<<RED_PARTS, TB, 0, S(stream)>>>(n, x_dev, y_dev ? y_dev : x_dev, scratch_dev);
  MGB_LAUNCH_OK();
  k_sum_partials<<<1, 32, 0, S(stream)>>>(1, RED_PARTS, scratch_dev, out_dev, 0);
  MGB_LAUNCH_OK();
  return MGB_OK;
}

extern "C" int mgb_ad_scratch_doubles(int outputs) { return outputs * RED_PARTS; }

extern "C" int mgb_ad_stencil_adjoint(int rows, int cols, const double* T_dev, const uint8_t* mask_in_dev,
                                      const uint8_t* mask_out_dev, const double* g_dev, int order, double* du_dev,
                                      void* stream) {
  if (rows <= 0 || cols <= 0 || !T_dev || !g_dev || !du_dev) return fail(MGB_CONTRACT, "bad adjoint arguments");
  k_stencil_adjoint<<<blocks_for((int64_t)rows * cols), TB, 0, S(stream)>>>(rows, cols, T_dev, mask_in_dev, mask_out_dev,
                                                                            g_dev, order, du_dev);
  MGB_LAUNCH_OK();
  return MGB_OK;
}

extern "C" int mgb_ad_pconv_kgrad(int rows, int cols, const uint8_t* mask_dev, const double* g_dev, const double* u_dev,
                                  int accumulate, double* dK_dev, void* stream) {
  if (rows <= 0 || cols <= 0 || !g_dev || !u_dev || !dK_dev) return fail(MGB_CONTRACT, "bad kernel-gradient arguments");
  k_pconv_kgrad<<<blocks_for((int64_t)rows * cols), TB, 0, S(stream)>>>(rows, cols, mask_dev, g_dev, u_dev, accumulate,
                                                                        dK_dev);
  MGB_LAUNCH_OK();
  return MGB_OK;
}

extern "C" int mgb_ad_conv_kgrad(int rows, int cols, int ksize, const uint8_t* mask_dev, const double* g_dev,
                                 const double* u_dev, double* scratch_dev, int accumulate, double* dk_dev, void* stream) {
  if (rows <= 0 || cols <= 0 || ksize < 1 || !(ksize & 1) || !g_dev || !u_dev || !scratch_dev || !dk_dev)
    return fail(MGB_CONTRACT, "bad shared-kernel gradient arguments");
  const int nout = ksize * ksize;
  k_conv_kgrad_part<<<dim3(RED_PARTS, nout), TB, 0, S(stream)>>>(rows, cols, ksize, mask_dev, g_dev, u_dev, RED_PARTS,
                                                                 scratch_dev);
  MGB_LAUNCH_OK();
  k_sum_partials<<<(nout + 31) / 32, 32, 0, S(stream)>>>(nout, RED_PARTS, scratch_dev, dk_dev, accumulate);
  MGB_LAUNCH_OK();
  return MGB_OK;
}

extern "C" int mgb_ad_conv_batch(int64_t n, int c, const double* kern_dev, const double* img_dev, double* out_dev,
                                 void* stream) {
  if (n <= 0 || c <= 0 || !kern_dev || !img_dev || !out_dev) return fail(MGB_CONTRACT, "bad conv_batch arguments");
  k_conv_batch<<<blocks_for(n * c * 9), TB, 0, S(stream)>>>(n, c, kern_dev, img_dev, out_dev);
  MGB_LAUNCH_OK();
  return MGB_OK;
}

extern "C" int mgb_ad_conv_batch_bwd(int64_t n, int c, const double* kern_dev, const double* img_dev,
                                     const double* g_dev, double* scratch_dev, int acc_k, double* dk_dev, int acc_img,
                                     double* dimg_dev, void* stream) {
  if (n <= 0 || c <= 0 || !kern_dev || !img_dev || !g_dev) return fail(MGB_CONTRACT, "bad conv_batch arguments");
  if (dk_dev) {
    if (!scratch_dev) return fail(MGB_CONTRACT, "conv_batch kernel gradient needs scratch");
    k_conv_batch_dk_part<<<dim3(RED_PARTS, c * 9), TB, 0, S(stream)>>>(n, c, g_dev, img_dev, RED_PARTS, scratch_dev);
    MGB_LAUNCH_OK();
    k_sum_partials<<<(c * 9 + 31) / 32, 32, 0, S(stream)>>>(c * 9, RED_PARTS, scratch_dev, dk_dev, acc_k);
    MGB_LAUNCH_OK();
  }
  if (dimg_dev) {
    k_conv_batch_dimg<<<blocks_for(n * 9), TB, 0, S(stream)>>>(n, c, kern_dev, g_dev, acc_img, dimg_dev);
    MGB_LAUNCH_OK();
  }
  return MGB_OK;
}

// C (M, N) (+)= op(A) op(B); trans_a: A is stored (K, M); trans_b: B is stored (N, K).
// reduce != 0 (with trans_a, !trans_b): the k sum is split over RED_PARTS blocks
// (weight gradients, K = number of points); scratch_dev: M * N * RED_PARTS doubles.
extern "C" int mgb_ad_matmul(int M, int K, int N, const double* A_dev, int trans_a, const double* B_dev, int trans_b,
                             int accumulate, double* C_dev, double* scratch_dev, void* stream) {
  if (M <= 0 || K <= 0 || N <= 0 || !A_dev || !B_dev || !C_dev) return fail(MGB_CONTRACT, "bad matmul arguments");
  if (scratch_dev && trans_a && !trans_b && K >= 4 * TB) {
    k_matmul_tn_part<<<dim3(RED_PARTS, M * N), TB, 0, S(stream)>>>(M, K, N, A_dev, B_dev, RED_PARTS, scratch_dev);
    MGB_LAUNCH_OK();
    k_sum_partials<<<(M * N + 31) / 32, 32, 0, S(stream)>>>(M * N, RED_PARTS, scratch_dev, C_dev, accumulate);
    MGB_LAUNCH_OK();
    return MGB_OK;
  }
  k_matmul<<<blocks_for((int64_t)M * N), TB, 0, S(stream)>>>(M, K, N, A_dev, trans_a, B_dev, trans_b, accumulate, C_dev);
  MGB_LAUNCH_OK();
  return MGB_OK;
}

extern "C" int mgb_lu_solve_t(int n, const double* lu_dev, const int32_t* perm_dev, const double* b_dev, double* x_dev,
                              double* scratch_dev, void* stream) {
  if (n <= 0 || n > 4096 || !lu_dev || !perm_dev || !b_dev || !x_dev || !scratch_dev)
    return fail(MGB_CONTRACT, "bad transposed-solve arguments");
  k_lu_solve_t<<<1, 256, 0, S(stream)>>>(n, lu_dev, perm_dev, b_dev, x_dev, scratch_dev);
  MGB_LAUNCH_OK();
  return MGB_OK;
}

extern "C" int mgb_ad_adam(int64_t n, double* p_dev, const double* g_dev, double* m_dev, double* v_dev, double lr,
                           double beta1, double beta2, double eps, int step, void* stream) {
  if (n <= 0 || !p_dev || !m_dev || !v_dev || step < 1) return fail(MGB_CONTRACT, "bad Adam arguments");
  const double bc1 = 1.0 - pow(beta1, (double)step), bc2 = 1.0 - pow(beta2, (double)step);
  k_adam<<<blocks_for(n), TB, 0, S(stream)>>>(n, p_dev, g_dev, m_dev, v_dev, lr, beta1, beta2, eps, bc1, bc2);
  MGB_LAUNCH_OK();
  return MGB_OK;
}
