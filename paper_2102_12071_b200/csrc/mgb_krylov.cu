// Flexible GMRES with the V-cycle as right preconditioner, and plain GMRES, on
// the flat grid vector.
//
// The Arnoldi loop is the reference's, step for step (krylov.py:60-236):
// modified Gram-Schmidt with one conditional re-orthogonalisation sweep, Givens
// rotations of the Hessenberg column, the breakdown test, back substitution and
// u = u0 + sum y_i z_i.  The scalar recurrences (Hessenberg, rotations, y) run on
// the host in double precision in the reference's order; every vector operation
// runs on the GPU:
//   * the operator action w = A z is the stateless apply_stencil kernel on the
//     per-point table (grid.py:216, the reference's grid_action, krylov.py:249);
//   * the preconditioner is one V(nu1, nu2)-cycle from zero of a device
//     hierarchy (cycle_preconditioner, krylov.py:261-270), run by the same
//     streaming / tile passes as the solve;
//   * MGS steps fuse w <- w - h v_i with the next inner product v_{i+1} . w (or
//     w . w) in one pass over the vectors; the re-orthogonalisation test's j + 1
//     inner products share one pass over w.  Inner products are deterministic
//     (fixed grid, fixed-order two-stage reduction).
// AXPYs round like NumPy's elementwise w - h * v (the library is built with
// -fmad=false); inner products differ from BLAS ddot in summation order only.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "mgb_cycle.h"
#include "mgb_dd.h"

namespace mgb {
namespace {

constexpr int KT = 256;        // threads per block
constexpr int KMAXB = 1184;    // reduction blocks (8 per SM on 148 SMs)
constexpr int KCH = 8;         // inner products per multi-dot pass

int dot_blocks(int64_t n) {
  const int64_t b = (n + KT * 4 - 1) / (KT * 4);
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, KMAXB));
}

__device__ __forceinline__ double block_reduce(double v, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < KT / 32 ? sh[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
  }
  return t;
}

// partials[q * G + block] = sum over the block's elements of V[q] . w, q < m
struct VecList {
  const double* v[KCH];
};

__global__ void __launch_bounds__(KT) k_multidot(int64_t n, const double* __restrict__ w, VecList vl, int m,
                                                 double* __restrict__ partials) {
  __shared__ double sh[32];
  double acc[KCH];
#pragma unroll
  for (int q = 0; q < KCH; ++q) acc[q] = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * KT + threadIdx.x; i < n; i += (int64_t)gridDim.x * KT) {
    const double x = w[i];
#pragma unroll
    for (int q = 0; q < KCH; ++q)
      if (q < m) acc[q] += vl.v[q][i] * x;
  }
  for (int q = 0; q < m; ++q) {
    const double t = block_reduce(acc[q], sh);
    if (threadIdx.x == 0) partials[(int64_t)q * gridDim.x + blockIdx.x] = t;
  }
}

// w <- w - h v, then partials of nxt . w (nxt == nullptr: w . w)
__global__ void __launch_bounds__(KT) k_axpy_dot(int64_t n, double* __restrict__ w, const double* __restrict__ v,
                                                 double h, const double* __restrict__ nxt,
                                                 double* __restrict__ partials) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * KT + threadIdx.x; i < n; i += (int64_t)gridDim.x * KT) {
    const double x = w[i] - h * v[i];
    w[i] = x;
    acc += (nxt ? nxt[i] : x) * x;
  }
  const double t = block_reduce(acc, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = t;
}

// out[q] = sum of partials[q * G .. q * G + G - 1] (fixed order)
__global__ void __launch_bounds__(KT) k_finalize_dots(int G, const double* __restrict__ partials,
                                                      double* __restrict__ out) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < G; i += KT) acc += partials[(int64_t)blockIdx.x * G + i];
  const double t = block_reduce(acc, sh);
  if (threadIdx.x == 0) out[blockIdx.x] = t;
}

// out = x / s   (krylov.py:73, :123: r / beta, w / hsub)
__global__ void k_scale_div(int64_t n, const double* __restrict__ x, double s, double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = x[i] / s;
}

// r = f - a   (krylov.py:62)
__global__ void k_sub(int64_t n, const double* __restrict__ f, const double* __restrict__ a,
                      double* __restrict__ r) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    r[i] = f[i] - a[i];
}

// out = x * mask   (krylov.py:268: r * spec.mask)
__global__ void k_mask_mul(int64_t n, const double* __restrict__ x, const uint8_t* __restrict__ mask,
                           double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = x[i] * (mask[i] ? 1.0 : 0.0);
}

// u = (((u + y0 z0) + y1 z1) + ...)   (krylov.py:133-134, the reference's sequence)
struct LinComb {
  const double* z[KCH];
  double y[KCH];
};
__global__ void k_lincomb(int64_t n, double* __restrict__ u, LinComb lc, int m) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double x = u[i];
#pragma unroll
    for (int q = 0; q < KCH; ++q)
      if (q < m) x = x + lc.y[q] * lc.z[q][i];
    u[i] = x;
  }
}

int elem_blocks(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

constexpr double REORTH_TOL = 1e-8;     // krylov.py:19
constexpr double BREAKDOWN_TOL = 1e-14; // krylov.py:20

// Device vector workspace and primitives of one Krylov solve.
struct Kry {
  Grid g;
  int64_t n;
  Tab A;
  const uint8_t* mask;
  mgb_work* pc;
  int nu1, nu2;
  cudaStream_t s;
  int G;
  double* partials = nullptr;  // KCH x G
  double* dres = nullptr;      // KCH
  double* hres = nullptr;      // host pinned KCH
  double* tmp = nullptr;       // n: A u / masked preconditioner input
  std::vector<double*> pool;   // vectors owned by this solve

  ~Kry() {
    for (double* p : pool) cudaFreeAsync(p, s);
    if (partials) cudaFreeAsync(partials, s);
    if (dres) cudaFreeAsync(dres, s);
    if (tmp) cudaFreeAsync(tmp, s);
    cudaStreamSynchronize(s);
    if (hres) cudaFreeHost(hres);
  }
  cudaError_t init() {
    G = dot_blocks(n);
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&partials), sizeof(double) * KCH * G, s);
    if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&dres), sizeof(double) * KCH, s);
    if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&tmp), sizeof(double) * n, s);
    if (e == cudaSuccess) e = cudaMallocHost(reinterpret_cast<void**>(&hres), sizeof(double) * KCH);
    return e;
  }
  cudaError_t vec(double** out) {
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(out), sizeof(double) * n, s);
    if (e == cudaSuccess) pool.push_back(*out);
    return e;
  }
  cudaError_t fetch(int m, double* out) {
    ++g_launches;
    k_finalize_dots<<<m, KT, 0, s>>>(G, partials, dres);
    cudaError_t e = cudaMemcpyAsync(hres, dres, sizeof(double) * m, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    for (int q = 0; q < m; ++q) out[q] = hres[q];
    return e;
  }
  // out[q] = vs[q] . w
  cudaError_t dots(const double* w, const double* const* vs, int m, double* out) {
    for (int c0 = 0; c0 < m; c0 += KCH) {
      VecList vl{};
      const int mc = std::min(KCH, m - c0);
      for (int q = 0; q < mc; ++q) vl.v[q] = vs[c0 + q];
      ++g_launches;
      k_multidot<<<G, KT, 0, s>>>(n, w, vl, mc, partials);
      if (cudaError_t e = fetch(mc, out + c0)) return e;
    }
    return cudaSuccess;
  }
  // w <- w - h v; returns nxt . w (nxt == null: w . w)
  cudaError_t axpy_dot(double* w, const double* v, double h, const double* nxt, double* out) {
    ++g_launches;
    k_axpy_dot<<<G, KT, 0, s>>>(n, w, v, h, nxt, partials);
    return fetch(1, out);
  }
  // out = A x (reference apply_stencil, masked)
  cudaError_t apply(const double* x, double* out) { return launch_apply(g, 3, A, mask, x, out, s); }
  // z = one V(nu1, nu2)-cycle from zero on the masked v (MGB status)
  int precond(const double* v, double* z) {
    const double* fin = v;
    if (mask) {
      ++g_launches;
      k_mask_mul<<<elem_blocks(n), 256, 0, s>>>(n, v, mask, tmp);
      fin = tmp;
    }
    double* res = nullptr;
    if (int st = work_vcycle_level(pc, 0, fin, z, true, nu1, nu2, s, &res)) return st;
    if (res != z) MGB_CUDA_TRY(cudaMemcpyAsync(z, res, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    return MGB_OK;
  }
};

// One Arnoldi cycle from u (in place), krylov.py:60-135 (fgmres) / :189-230
// (gmres: precond off, same arithmetic).  Returns MGB status; *done, *took.
// early_exit: fgmres returns at once when the restart residual already meets the
// tolerance (krylov.py:66-67); gmres has no such test (krylov.py:189-197).
int arnoldi_cycle(Kry& K, const double* f, double* u, int steps, double tol_abs, std::vector<double>& history,
                  bool record_beta, bool use_pc, bool early_exit, bool* done, int* took) {
  const int64_t n = K.n;
  double* r = nullptr;
  MGB_CUDA_TRY(K.vec(&r));
  MGB_CUDA_TRY(K.apply(u, K.tmp));
  ++g_launches;
  k_sub<<<elem_blocks(n), 256, 0, K.s>>>(n, f, K.tmp, r);
  double rr = 0.0;
  const double* rv[1] = {r};
  MGB_CUDA_TRY(K.dots(r, rv, 1, &rr));
  const double beta = std::sqrt(rr);
  if (record_beta) history.push_back(beta);
  *done = false;
  *took = 0;
  if (early_exit && beta <= tol_abs) {
    *done = true;
    return MGB_OK;
  }
  steps = (int)std::min<int64_t>(steps, n);
  std::vector<double*> V, Z;
  V.push_back(r);
  ++g_launches;
  k_scale_div<<<elem_blocks(n), 256, 0, K.s>>>(n, r, beta, r);
  std::vector<double> H((size_t)(steps + 1) * steps, 0.0), cs(steps, 0.0), sn(steps, 0.0), gv(steps + 1, 0.0);
  auto Hm = [&](int i, int j) -> double& { return H[(size_t)i * steps + j]; };
  gv[0] = beta;
  int j = 0;
  std::vector<double> d(steps + 2);
  while (j < steps) {
    double* z = V[j];
    if (use_pc) {
      MGB_CUDA_TRY(K.vec(&z));
      if (int st = K.precond(V[j], z)) return st;
    }
    Z.push_back(z);
    double* w = nullptr;
    MGB_CUDA_TRY(K.vec(&w));
    MGB_CUDA_TRY(K.apply(z, w));
    // ||w|| and v_0 . w in one pass
    const double* first[2] = {w, V[0]};
    double d2[2];
    MGB_CUDA_TRY(K.dots(w, first, 2, d2));
    const double wnorm0 = std::sqrt(d2[0]);
    double hij = d2[1];
    double ww = 0.0;
    for (int i = 0; i <= j; ++i) {
      Hm(i, j) = hij;
      const double* nxt = i < j ? V[i + 1] : nullptr;
      double nv = 0.0;
      MGB_CUDA_TRY(K.axpy_dot(w, V[i], hij, nxt, &nv));
      if (i < j) hij = nv;
      else ww = nv;
    }
    double wnorm = std::sqrt(ww);
    // one extra Gram-Schmidt sweep when cancellation ate the orthogonality
    MGB_CUDA_TRY(K.dots(w, V.data(), j + 1, d.data()));
    bool reorth = wnorm < REORTH_TOL * wnorm0;
    for (int i = 0; i <= j && !reorth; ++i)
      if (std::fabs(d[i]) > REORTH_TOL * std::max(wnorm, 1e-300)) reorth = true;
    double hsub = wnorm;
    if (reorth) {
      double c = d[0];
      for (int i = 0; i <= j; ++i) {
        Hm(i, j) += c;
        const double* nxt = i < j ? V[i + 1] : nullptr;
        double nv = 0.0;
        MGB_CUDA_TRY(K.axpy_dot(w, V[i], c, nxt, &nv));
        if (i < j) c = nv;
        else hsub = std::sqrt(nv);
      }
    }
    Hm(j + 1, j) = hsub;
    for (int i = 0; i < j; ++i) {
      const double t = cs[i] * Hm(i, j) + sn[i] * Hm(i + 1, j);
      Hm(i + 1, j) = -sn[i] * Hm(i, j) + cs[i] * Hm(i + 1, j);
      Hm(i, j) = t;
    }
    {
      const double a = Hm(j, j), b = Hm(j + 1, j);
      const double rr2 = std::hypot(a, b);
      cs[j] = rr2 == 0.0 ? 1.0 : a / rr2;
      sn[j] = rr2 == 0.0 ? 0.0 : b / rr2;
    }
    Hm(j, j) = cs[j] * Hm(j, j) + sn[j] * Hm(j + 1, j);
    Hm(j + 1, j) = 0.0;
    gv[j + 1] = -sn[j] * gv[j];
    gv[j] = cs[j] * gv[j];
    const double res = std::fabs(gv[j + 1]);
    history.push_back(res);
    ++j;
    if (res <= tol_abs) break;
    if (hsub <= BREAKDOWN_TOL * std::max(wnorm0, 1.0)) {
      char buf[160];
      snprintf(buf, sizeof buf, "Arnoldi breakdown at step %d with residual %.3e above tolerance", j, res);
      return fail(MGB_NUMERIC, buf);
    }
    ++g_launches;
    k_scale_div<<<elem_blocks(n), 256, 0, K.s>>>(n, w, hsub, w);
    V.push_back(w);
  }
  // back substitution on the rotated Hessenberg (krylov.py:129-132)
  std::vector<double> y(j, 0.0);
  for (int i = j - 1; i >= 0; --i) {
    double dotv = 0.0;
    for (int q = i + 1; q < j; ++q) dotv += Hm(i, q) * y[q];
    y[i] = (gv[i] - dotv) / Hm(i, i);
  }
  for (int c0 = 0; c0 < j; c0 += KCH) {
    LinComb lc{};
    const int mc = std::min(KCH, j - c0);
    for (int q = 0; q < mc; ++q) {
      lc.z[q] = Z[c0 + q];
      lc.y[q] = y[c0 + q];
    }
    ++g_launches;
    k_lincomb<<<elem_blocks(n), 256, 0, K.s>>>(n, u, lc, mc);
  }
  MGB_CUDA_TRY(cudaGetLastError());
  *done = std::fabs(gv[j]) <= tol_abs;
  *took = j;
  // vectors of this cycle are released before the next one
  for (double* p : K.pool) cudaFreeAsync(p, K.s);
  K.pool.clear();
  return MGB_OK;
}

}  // namespace
}  // namespace mgb

using namespace mgb;

extern "C" int mgb_krylov(int method, int rows, int cols, const double* A_dev, const uint8_t* mask_dev,
                          mgb_work* pc, int nu1, int nu2, const double* f_dev, double* u_dev, double tol,
                          int max_iter, int restart, double* history_host, int* n_hist, int* iterations,
                          int* converged, void* stream) {
  if (!A_dev || !f_dev || !u_dev || !history_host) return fail(MGB_CONTRACT, "null argument");
  if (rows < 1 || cols < 1) return fail(MGB_CONTRACT, "empty grid");
  if (method != 0 && method != 1) return fail(MGB_CONFIG, "method must be 0 (fgmres) or 1 (gmres)");
  if (method == 1 && pc) return fail(MGB_CONFIG, "gmres takes no preconditioner");
  if (!(tol > 0)) return fail(MGB_CONFIG, "tol must be positive");
  if (max_iter < 1) return fail(MGB_CONFIG, "max_iter must be >= 1");
  if (pc) {
    const mgb_hier* h = work_hier(pc);
    if (hier_batch(h) != 1 || hier_rows(h, 0) != rows || hier_cols(h, 0) != cols)
      return fail(MGB_CONTRACT, "preconditioner hierarchy does not match the operator's grid");
    if (nu1 < 0 || nu2 < 0) return fail(MGB_CONFIG, "sweep counts must be non-negative");
    if (int st = work_prepare(pc)) return st;
  }
  Kry K;
  K.g = Grid{1, rows, cols};
  K.n = (int64_t)rows * cols;
  K.A = tab_aos(A_dev, K.n, 1);
  K.mask = mask_dev;
  K.pc = pc;
  K.nu1 = nu1;
  K.nu2 = nu2;
  K.s = reinterpret_cast<cudaStream_t>(stream);
  MGB_CUDA_TRY(K.init());
  const int64_t n = K.n;
  std::vector<double> history;
  // ||f|| (krylov.py:156 / :186)
  double ff = 0.0;
  const double* fv[1] = {f_dev};
  MGB_CUDA_TRY(K.dots(f_dev, fv, 1, &ff));
  const double beta0 = std::sqrt(ff);
  MGB_CUDA_TRY(cudaMemsetAsync(u_dev, 0, sizeof(double) * n, K.s));
  int total = 0;
  bool done = false;
  if (beta0 == 0.0) {
    history.push_back(0.0);
    done = true;
  } else if (method == 0) {
    const double tol_abs = tol * beta0;
    while (total < max_iter && !done) {
      int steps = max_iter - total;
      if (restart > 0) steps = std::min(steps, restart);
      int took = 0;
      if (int st = arnoldi_cycle(K, f_dev, u_dev, steps, tol_abs, history, history.empty(), pc != nullptr, true, &done,
                                 &took))
        return st;
      total += took;
      if (took == 0) break;
    }
  } else {
    const double tol_abs = tol * beta0;
    history.push_back(beta0);
    if (beta0 <= tol_abs) {
      done = true;
    } else {
      int budget = max_iter;
      total = max_iter;
      while (budget > 0) {
        int steps = budget;
        if (restart > 0) steps = std::min(steps, restart);
        int took = 0;
        if (int st = arnoldi_cycle(K, f_dev, u_dev, steps, tol_abs, history, false, false, false, &done, &took)) return st;
        budget -= took;
        if (done || took == 0) {
          total = max_iter - budget;
          break;
        }
      }
    }
  }
  MGB_CUDA_TRY(cudaStreamSynchronize(K.s));
  const int nh = (int)std::min<size_t>(history.size(), (size_t)max_iter + 1);
  for (int i = 0; i < nh; ++i) history_host[i] = history[i];
  if (n_hist) *n_hist = nh;
  if (iterations) *iterations = total;
  if (converged) *converged = done ? 1 : 0;
  return MGB_OK;
}
