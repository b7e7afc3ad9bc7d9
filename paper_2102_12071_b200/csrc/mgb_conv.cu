// Shared-kernel convolutional smoother (ConvSmoother, smoothers.py:105-145) and
// the masked cross-correlation it is built from (convolve, grid.py:229-239).
//
//   M(r) = gain * ( L_{n-1} * act( ... act(L_1 * act?(L_0 * r)) ) + S * r )
//
// with 3x3 layer kernels L_i shared by every grid point (five plus a skip kernel
// S for the "full" form, two and no skip for "rb"), zero padding outside the grid,
// every convolution re-masked, and an optional leaky activation between chained
// layers.  One launch per layer (each reads the previous layer's whole output
// with a one-point halo); the skip convolution, the gain and the update
// u_out = u_in + M(r) are fused into the last launch.
//
// Arithmetic follows the reference exactly (built with -fmad=false): a layer
// accumulates out = out + w * x over the non-zero weights in di-major, dj-minor
// order starting from 0.0, as convolve() does with NumPy arrays; the combination
// is (v + s), then gain * (.), then u + (.) — bit-identical to the reference.
#include "mgb_conv.h"

namespace mgb {
namespace {

constexpr int CX = 32, CY = 8;

__device__ __forceinline__ double leaky_in(double x, double slope) { return x > 0.0 ? x : slope * x; }

// acc = sum over non-zero w[o] of w[o] * act(src(i + di, j + dj)), zero outside the grid
template <bool ACT>
__device__ __forceinline__ double conv_at(const Grid& g, const ConvW& w, const double* __restrict__ src, int i,
                                          int j, double slope) {
  double acc = 0.0;
#pragma unroll
  for (int di = -1; di <= 1; ++di)
#pragma unroll
    for (int dj = -1; dj <= 1; ++dj) {
      const double wo = w.w[(di + 1) * 3 + dj + 1];
      if (wo != 0.0) {
        const int ii = i + di, jj = j + dj;
        double x = 0.0;
        if ((unsigned)ii < (unsigned)g.rows && (unsigned)jj < (unsigned)g.cols) x = src[(int64_t)ii * g.cols + jj];
        if (ACT) x = leaky_in(x, slope);
        acc = acc + wo * x;
      }
    }
  return acc;
}

template <bool ACT>
__global__ void __launch_bounds__(CX* CY) k_convolve(Grid g, ConvW w, const uint8_t* __restrict__ mask,
                                                     const double* __restrict__ src, double* __restrict__ dst,
                                                     double slope) {
  const int j = blockIdx.x * CX + threadIdx.x, i = blockIdx.y * CY + threadIdx.y, b = blockIdx.z;
  if (i >= g.rows || j >= g.cols) return;
  const int64_t n = g.n(), p = (int64_t)i * g.cols + j;
  const double v = conv_at<ACT>(g, w, src + b * n, i, j, slope);
  dst[b * n + p] = (mask == nullptr || mask[p]) ? v : 0.0;
}

// u_out = u_in + gain * (v + S * r)   (u_in == null: u_out = gain * (v + S * r);
// skip == false: no S term).  v may alias u_out (read before write, same point).
template <bool SKIP, bool UIN>
__global__ void __launch_bounds__(CX* CY) k_conv_finish(Grid g, ConvW s, const uint8_t* __restrict__ mask,
                                                        const double* v, const double* __restrict__ r,
                                                        const double* u_in, double* u_out, double gain) {
  const int j = blockIdx.x * CX + threadIdx.x, i = blockIdx.y * CY + threadIdx.y, b = blockIdx.z;
  if (i >= g.rows || j >= g.cols) return;
  const int64_t n = g.n(), p = (int64_t)i * g.cols + j;
  const bool act = mask == nullptr || mask[p];
  double out = v[b * n + p];
  if (SKIP) out = out + (act ? conv_at<false>(g, s, r + b * n, i, j, 0.0) : 0.0);
  out = gain * out;
  u_out[b * n + p] = UIN ? u_in[b * n + p] + out : out;
}

}  // namespace

cudaError_t launch_convolve(const Grid& g, const ConvW& w, const uint8_t* mask, const double* src, double* dst,
                            bool act, double slope, cudaStream_t s) {
  ++g_launches;
  dim3 grid((g.cols + CX - 1) / CX, (g.rows + CY - 1) / CY, g.batch);
  if (act) k_convolve<true><<<grid, dim3(CX, CY), 0, s>>>(g, w, mask, src, dst, slope);
  else k_convolve<false><<<grid, dim3(CX, CY), 0, s>>>(g, w, mask, src, dst, slope);
  return MGB_DBG(__func__);
}

cudaError_t launch_conv_finish(const Grid& g, const ConvW* skip, const uint8_t* mask, const double* v,
                               const double* r, const double* u_in, double* u_out, double gain, cudaStream_t s) {
  ++g_launches;
  dim3 grid((g.cols + CX - 1) / CX, (g.rows + CY - 1) / CY, g.batch);
  const ConvW sw = skip ? *skip : ConvW{};
  if (skip && u_in) k_conv_finish<true, true><<<grid, dim3(CX, CY), 0, s>>>(g, sw, mask, v, r, u_in, u_out, gain);
  else if (skip) k_conv_finish<true, false><<<grid, dim3(CX, CY), 0, s>>>(g, sw, mask, v, r, u_in, u_out, gain);
  else if (u_in) k_conv_finish<false, true><<<grid, dim3(CX, CY), 0, s>>>(g, sw, mask, v, r, u_in, u_out, gain);
  else k_conv_finish<false, false><<<grid, dim3(CX, CY), 0, s>>>(g, sw, mask, v, r, u_in, u_out, gain);
  return MGB_DBG(__func__);
}

// out = u_in + M(r) with the chain through t1 / t2 (t1, t2 distinct from r; out may
// equal t2 but not r or u_in)
cudaError_t conv_smoother_apply(const Grid& g, const ConvSm& cs, const uint8_t* mask, const double* r,
                                const double* u_in, double* out, double* t1, double* t2, cudaStream_t s) {
  const double* cur = r;
  for (int l = 0; l < cs.nl; ++l) {
    double* dst = (l & 1) ? t2 : t1;
    cudaError_t e = launch_convolve(g, cs.layer[l], mask, cur, dst, l > 0 && cs.leaky, cs.slope, s);
    if (e != cudaSuccess) return e;
    cur = dst;
  }
  return launch_conv_finish(g, cs.has_skip ? &cs.skip : nullptr, mask, cur, r, u_in, out, cs.gain, s);
}

}  // namespace mgb
