// Stencil -> smoother-kernel CNN inference (setup path), one thread per grid point.
//
// Reference: smoothers.py build_feature_map :184-210, KernelInferenceNet :217-235,
// _conv3x3_same :256-270, net_forward :273-288, infer_kernels :302-322.
//
// The nets are tiny (conv: 7/5/3 single-channel 3x3 filters on a 3x3 image with
// channel *summation*, then a 27 x 9k head; fc: 81-40-40-40-9k), so they are not
// dense contractions worth a tensor-core tile: every point evaluates the whole
// net in registers with the weights broadcast from shared memory.  T = double is
// the parity mode; T = float is the fast mode (diagonal normalisation stays fp64).
#include "mgb_internal.h"

namespace mgb {
namespace {

constexpr int MAXK = 4;  // smoother stages supported by the inference kernels

template <typename T>
__device__ __forceinline__ T lk(T x, T s) { return x > T(0) ? x : s * x; }

__device__ __forceinline__ double tabv(const Tab& t, int b, int s, int o, int64_t p) { return tab_get(t, b, s, o, p); }
__device__ __forceinline__ void tabwv(const TabW& t, int b, int s, int o, int64_t p, double v) { tab_put(t, b, s, o, p, v); }

// one 3x3 "same" correlation of a single-channel 3x3 image, reference order
template <typename T>
__device__ __forceinline__ void conv_same(const T* w, const T* x, T* out) {
#pragma unroll
  for (int q = 0; q < 9; ++q) out[q] = T(0);
#pragma unroll
  for (int di = -1; di <= 1; ++di)
#pragma unroll
    for (int dj = -1; dj <= 1; ++dj) {
      const T wv = w[(di + 1) * 3 + (dj + 1)];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        if (i + di < 0 || i + di > 2) continue;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          if (j + dj < 0 || j + dj > 2) continue;
          out[i * 3 + j] = out[i * 3 + j] + wv * x[(i + di) * 3 + (j + dj)];
        }
      }
    }
}

template <typename T>
__global__ void __launch_bounds__(128) k_infer_conv(const int64_t* __restrict__ pts, int npts, Grid g, Tab A,
                                                    const uint8_t* __restrict__ mask,
                                                    int kst, const double* __restrict__ Wd,
                                                    double slope_d, TabW K) {
  // weights: W0 (7,3,3) W1 (5,3,3) W2 (3,3,3) W3 (27, 9k)
  extern __shared__ unsigned char smraw[];
  T* W = reinterpret_cast<T*>(smraw);
  const int nw = 63 + 45 + 27 + 27 * 9 * kst;
  for (int q = threadIdx.x; q < nw; q += blockDim.x) W[q] = T(Wd[q]);
  __syncthreads();
  const T* W0 = W;
  const T* W1 = W + 63;
  const T* W2 = W + 108;
  const T* W3 = W + 135;
  const T slope = T(slope_d);
  const int64_t n = g.n();
  const int b = blockIdx.y;
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pts) {
    if (p >= npts || pts[p] < 0) return;
    p = pts[p];
  }
  if (p >= n) return;
  const int nout = 9 * kst;
  if (mask && !mask[p]) {
    for (int m = 0; m < nout; ++m) tabwv(K, b, m / 9, m % 9, p, 0.0);
    return;
  }
  const double d = tabv(A, b, 0, 4, p);
  T x[9], h[9], y[9];
#pragma unroll
  for (int o = 0; o < 9; ++o) x[o] = T(tabv(A, b, 0, o, p) / d);
  // layers 0 and 1: leaky(conv) per channel, summed over channels
#pragma unroll
  for (int layer = 0; layer < 2; ++layer) {
    const T* Wl = layer == 0 ? W0 : W1;
    const int nc = layer == 0 ? 7 : 5;
#pragma unroll
    for (int q = 0; q < 9; ++q) h[q] = T(0);
    for (int c = 0; c < nc; ++c) {
      conv_same<T>(Wl + 9 * c, x, y);
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        const T v = lk(y[q], slope);
        h[q] = c == 0 ? v : h[q] + v;
      }
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) x[q] = h[q];
  }
  // layer 2: 3 channels kept, flattened c*9 + i*3 + j, then the head
  T acts[27];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    conv_same<T>(W2 + 9 * c, x, y);
#pragma unroll
    for (int q = 0; q < 9; ++q) acts[c * 9 + q] = lk(y[q], slope);
  }
  for (int m = 0; m < nout; ++m) {
    T s = T(0);
#pragma unroll
    for (int q = 0; q < 27; ++q) s = s + acts[q] * W3[q * nout + m];
    tabwv(K, b, m / 9, m % 9, p, double(s) / d);
  }
}

template <typename T>
__global__ void __launch_bounds__(128) k_infer_fc(const int64_t* __restrict__ pts, int npts, Grid g, Tab A,
                                                    const uint8_t* __restrict__ mask,
                                                  int kst, const double* __restrict__ Wd,
                                                  double slope_d, TabW K) {
  // weights: W0 (81,40) W1 (40,40) W2 (40,40) W3 (40, 9k)
  extern __shared__ unsigned char smraw[];
  T* W = reinterpret_cast<T*>(smraw);
  const int nout = 9 * kst;
  const int nw = 3240 + 1600 + 1600 + 40 * nout;
  for (int q = threadIdx.x; q < nw; q += blockDim.x) W[q] = T(Wd[q]);
  __syncthreads();
  const T* W0 = W;
  const T* W1 = W + 3240;
  const T* W2 = W + 4840;
  const T* W3 = W + 6440;
  const T slope = T(slope_d);
  const int64_t n = g.n();
  const int b = blockIdx.y;
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pts) {
    if (p >= npts || pts[p] < 0) return;
    p = pts[p];
  }
  if (p >= n) return;
  if (mask && !mask[p]) {
    for (int m = 0; m < nout; ++m) tabwv(K, b, m / 9, m % 9, p, 0.0);
    return;
  }
  const int i = (int)(p / g.cols), j = (int)(p % g.cols);
  const double d = tabv(A, b, 0, 4, p);
  T h1[40];
#pragma unroll
  for (int m = 0; m < 40; ++m) h1[m] = T(0);
  // features: block (oi+1)*3+(oj+1) = neighbour's table, zero off-grid / inactive
  for (int blk = 0; blk < 9; ++blk) {
    const int ii = i + blk / 3 - 1, jj = j + blk % 3 - 1;
    const bool in = ii >= 0 && ii < g.rows && jj >= 0 && jj < g.cols &&
                    (mask == nullptr || mask[(int64_t)ii * g.cols + jj]);
    const int64_t q = (int64_t)ii * g.cols + jj;
    for (int e = 0; e < 9; ++e) {
      const T xv = in ? T(tabv(A, b, 0, e, q) / d) : T(0);
      const T* wr = W0 + (blk * 9 + e) * 40;
#pragma unroll
      for (int m = 0; m < 40; ++m) h1[m] = h1[m] + xv * wr[m];
    }
  }
#pragma unroll
  for (int m = 0; m < 40; ++m) h1[m] = lk(h1[m], slope);
  T h2[40];
#pragma unroll
  for (int m = 0; m < 40; ++m) h2[m] = T(0);
  for (int q = 0; q < 40; ++q) {
    const T xv = h1[q];
#pragma unroll
    for (int m = 0; m < 40; ++m) h2[m] = h2[m] + xv * W1[q * 40 + m];
  }
#pragma unroll
  for (int m = 0; m < 40; ++m) { h2[m] = lk(h2[m], slope); h1[m] = T(0); }
  for (int q = 0; q < 40; ++q) {
    const T xv = h2[q];
#pragma unroll
    for (int m = 0; m < 40; ++m) h1[m] = h1[m] + xv * W2[q * 40 + m];
  }
#pragma unroll
  for (int m = 0; m < 40; ++m) h1[m] = lk(h1[m], slope);
  for (int m = 0; m < nout; ++m) {
    T s = T(0);
#pragma unroll
    for (int q = 0; q < 40; ++q) s = s + h1[q] * W3[q * nout + m];
    tabwv(K, b, m / 9, m % 9, p, double(s) / d);
  }
}

template <typename KF>
cudaError_t launch_k(KF kern, const Grid& g, size_t smem, Tab A, const uint8_t* mask, int kst,
                     const double* W, double slope, TabW K, cudaStream_t s, const int64_t* pts, int npts) {
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  ++g_launches;
  dim3 grid((unsigned)(((pts ? npts : g.n()) + 127) / 128), g.batch);
  kern<<<grid, 128, smem, s>>>(pts, npts, g, A, mask, kst, W, slope, K);
  return MGB_DBG(__func__);
}

}  // namespace

int64_t net_weight_count(int variant, int kst) {
  if (variant == MGB_NET_CONV) return 63 + 45 + 27 + 27 * 9 * (int64_t)kst;
  return 3240 + 1600 + 1600 + 40 * 9 * (int64_t)kst;
}

cudaError_t launch_infer(const Grid& g, Tab A, const uint8_t* mask, int variant, int kst,
                         const double* W_dev, double slope, int precision, TabW K,
                         cudaStream_t s, const int64_t* pts, int npts) {
  if (kst < 1 || kst > MAXK) return cudaErrorInvalidValue;
  const size_t nw = (size_t)net_weight_count(variant, kst);
  if (variant == MGB_NET_CONV) {
    if (precision == 32)
      return launch_k(k_infer_conv<float>, g, nw * sizeof(float), A, mask, kst, W_dev, slope, K, s, pts, npts);
    return launch_k(k_infer_conv<double>, g, nw * sizeof(double), A, mask, kst, W_dev, slope, K, s, pts, npts);
  }
  if (precision == 32)
    return launch_k(k_infer_fc<float>, g, nw * sizeof(float), A, mask, kst, W_dev, slope, K, s, pts, npts);
  return launch_k(k_infer_fc<double>, g, nw * sizeof(double), A, mask, kst, W_dev, slope, K, s, pts, npts);
}

}  // namespace mgb
