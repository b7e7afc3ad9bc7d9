// sm_100a kernels for the learned-smoother V-cycle (fp64, HBM-bound).
//
// Arithmetic follows the reference's elementwise order exactly (the library is
// compiled with -fmad=false, so a + b*c is a rounded multiply then a rounded
// add, as NumPy evaluates `out += w * shifted(u)`); standalone stencil,
// transfer and Galerkin results are therefore bit-identical to the reference.
//
// Reference map (bare file:line = /root/reference/pkg/src/mgsmooth/<file>):
//   apply / residual      grid.py:216-226 (shifted :27-35), hierarchy.py:107-111
//   fused sweep           smoothers.py:325-343 on the residual of hierarchy.py:107,111
//   residual+restriction  transfer.py:108-121 on f - A u (hierarchy.py:108)
//   prolong(+correct)     transfer.py:124-147 (hierarchy.py:110)
//   Galerkin RAP          transfer.py:150-209, _trim :212-222
//   LU factor / solve     dense.py:21-63, coarse_solve hierarchy.py:91-93
//   materialize           grid.py:269-292
//   jacobi                smoothers.py:29-50
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>

#include "mgb_internal.h"

namespace mgb {

thread_local int64_t g_launches = 0;

bool pdl_enabled() {
  static const bool off = getenv("MGB_NO_PDL") && atoi(getenv("MGB_NO_PDL")) != 0;
  return !off;
}

// ---- guard mode -----------------------------------------------------------------
namespace {
constexpr size_t GUARD_BYTES = 4096;
constexpr unsigned char GUARD_PATTERN = 0xA5;
std::mutex g_guard_mu;
std::map<void*, size_t> g_guarded;   // user pointer -> user bytes
bool guard_on() {
  static const bool on = getenv("MGB_GUARD") && atoi(getenv("MGB_GUARD")) != 0;
  return on;
}
}  // namespace

cudaError_t guarded_malloc(void** p, size_t bytes) {
  if (!guard_on()) return cudaMalloc(p, bytes);
  const size_t user = (bytes + 255) / 256 * 256;
  unsigned char* base = nullptr;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&base), user + 2 * GUARD_BYTES);
  if (e != cudaSuccess) return e;
  e = cudaMemset(base, GUARD_PATTERN, user + 2 * GUARD_BYTES);
  if (e != cudaSuccess) return e;
  *p = base + GUARD_BYTES;
  std::lock_guard<std::mutex> lk(g_guard_mu);
  g_guarded[*p] = bytes;
  return cudaSuccess;
}

void guarded_free(void* p) {
  if (!guard_on()) {
    cudaFree(p);
    return;
  }
  std::lock_guard<std::mutex> lk(g_guard_mu);
  g_guarded.erase(p);
  cudaFree(static_cast<unsigned char*>(p) - GUARD_BYTES);
}

}  // namespace mgb

extern "C" int mgb_guard_check(int* allocations, int* corrupted) {
  using namespace mgb;
  if (!allocations || !corrupted) return fail(MGB_CONTRACT, "null argument");
  *allocations = *corrupted = 0;
  if (!guard_on()) return fail(MGB_CONFIG, "guard mode is off (set MGB_GUARD=1 before loading the library)");
  MGB_CUDA_TRY(cudaDeviceSynchronize());
  std::lock_guard<std::mutex> lk(g_guard_mu);
  std::vector<unsigned char> buf(GUARD_BYTES);
  std::string report;
  for (auto& kv : g_guarded) {
    ++*allocations;
    unsigned char* user = static_cast<unsigned char*>(kv.first);
    // the bytes right after the user region up to the rounded size belong to the back canary
    const size_t back_off = kv.second;
    const size_t back_len = GUARD_BYTES;
    bool bad = false;
    MGB_CUDA_TRY(cudaMemcpy(buf.data(), user - GUARD_BYTES, GUARD_BYTES, cudaMemcpyDeviceToHost));
    for (size_t q = 0; q < GUARD_BYTES; ++q) bad |= buf[q] != GUARD_PATTERN;
    MGB_CUDA_TRY(cudaMemcpy(buf.data(), user + (back_off + 255) / 256 * 256, back_len, cudaMemcpyDeviceToHost));
    for (size_t q = 0; q < back_len; ++q) bad |= buf[q] != GUARD_PATTERN;
    if (bad) {
      ++*corrupted;
      report += " [" + std::to_string(kv.second) + " B]";
    }
  }
  if (*corrupted) set_error(MGB_OK, "guard canaries overwritten around allocations of" + report);
  return MGB_OK;
}

namespace mgb {

cudaError_t debug_sync(const char* what) {
  static const bool on = getenv("MGB_DEBUG_SYNC") && getenv("MGB_DEBUG_SYNC")[0] == '1';
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || !on) return e;
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) fprintf(stderr, "[mgb debug] %s failed: %s\n", what, cudaGetErrorString(e));
  return e;
}

namespace {

constexpr int BX = 32, BY = 8, NT = BX * BY;

__device__ __forceinline__ double tab(const Tab& t, int b, int s, int o, int64_t p) { return tab_get(t, b, s, o, p); }
__device__ __forceinline__ void tabw(const TabW& t, int b, int s, int o, int64_t p, double v) { tab_put(t, b, s, o, p, v); }
__device__ __forceinline__ bool act(const uint8_t* m, int64_t p) { return m == nullptr || m[p] != 0; }

// out(p) = sum over (di, dj) in row-major order of A(p)[o] * u(p + o), 0 outside.
__device__ __forceinline__ double stencil3(const Tab& A, int b, const double* __restrict__ u,
                                           int i, int j, int rows, int cols) {
  const int64_t p = (int64_t)i * cols + j;
  double s = 0.0;
#pragma unroll
  for (int di = -1; di <= 1; ++di) {
    const int ii = i + di;
    const bool rin = ii >= 0 && ii < rows;
#pragma unroll
    for (int dj = -1; dj <= 1; ++dj) {
      const int jj = j + dj;
      const double w = tab(A, b, 0, (di + 1) * 3 + (dj + 1), p);
      const double uv = (rin && jj >= 0 && jj < cols) ? __ldg(u + (int64_t)ii * cols + jj) : 0.0;
      s = s + w * uv;
    }
  }
  return s;
}

__device__ __forceinline__ double leaky(double x, double slope) { return x > 0.0 ? x : slope * x; }

// ---------------------------------------------------------------------------
// apply (k = 1 or 3), reference layout or planes

template <int K>
__global__ void __launch_bounds__(NT) k_apply(Grid g, Tab A, const uint8_t* __restrict__ mask,
                                              const double* __restrict__ u, double* __restrict__ out) {
  const int j = blockIdx.x * BX + threadIdx.x, i = blockIdx.y * BY + threadIdx.y, b = blockIdx.z;
  if (i >= g.rows || j >= g.cols) return;
  const int64_t n = g.n(), p = (int64_t)i * g.cols + j;
  const double* ub = u + b * n;
  double s;
  if (K == 3) {
    s = stencil3(A, b, ub, i, j, g.rows, g.cols);
  } else {
    s = 0.0 + tab(A, b, 0, 0, p) * __ldg(ub + p);
  }
  out[b * n + p] = act(mask, p) ? s : 0.0;
}

// ---------------------------------------------------------------------------
// deterministic block reduction of one double per thread (fixed shuffle tree)

__device__ __forceinline__ double block_sum(double v, double* sh) {
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
  return t;  // valid in thread 0
}

// r = f - A u, masked.  Optional r output and per-block sum of squares.  Each
// block covers 32 columns x (8 * RES_RPT) rows so the partials stay few.
constexpr int RES_RPT = 8;
__global__ void __launch_bounds__(NT) k_residual(Grid g, Tab A, const uint8_t* __restrict__ mask,
                                                 const double* __restrict__ f,
                                                 const double* __restrict__ u,
                                                 double* __restrict__ r,
                                                 double* __restrict__ partials) {
  __shared__ double sh[32];
  const int j = blockIdx.x * BX + threadIdx.x, b = blockIdx.z;
  const int64_t n = g.n();
  double acc = 0.0;
#pragma unroll 2
  for (int q = 0; q < RES_RPT; ++q) {
    const int i = (blockIdx.y * RES_RPT + q) * BY + threadIdx.y;
    if (i < g.rows && j < g.cols) {
      const int64_t p = (int64_t)i * g.cols + j;
      double v = 0.0;
      if (act(mask, p))
        v = u ? __ldg(f + b * n + p) - stencil3(A, b, u + b * n, i, j, g.rows, g.cols)
              : __ldg(f + b * n + p) - 0.0;
      if (r) r[b * n + p] = v;
      acc += v * v;
    }
  }
  if (partials) {
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0 && threadIdx.y == 0)
      partials[(int64_t)b * gridDim.x * gridDim.y + blockIdx.y * gridDim.x + blockIdx.x] = t;
  }
}

// one block per problem: out2[b] = fixed-order sum of partials; optional history entry
__global__ void __launch_bounds__(1024) k_finalize(int nblk, const double* __restrict__ partials,
                                                  double* __restrict__ out2,
                                                  const double* __restrict__ fnorm2,
                                                  double* __restrict__ hist, int64_t hstride) {
  __shared__ double sh[32];
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.x;
  double v = 0.0;
  for (int q = threadIdx.x; q < nblk; q += blockDim.x) v += partials[(int64_t)b * nblk + q];
  const double t = block_sum(v, sh);
  if (threadIdx.x == 0) {
    if (out2) out2[b] = t;
    if (hist) {
      const double nr = sqrt(t);
      // out2 without fnorm2: the sum is ||f||^2 itself (zero-start residual), stored as
      // the denominator of this and later entries
      const double fn = fnorm2 ? sqrt(fnorm2[b]) : (out2 ? nr : 1.0);
      const double den = fn > 0.0 ? fn : 1.0;          // hierarchy.py:126-127
      hist[b * hstride] = nr == 0.0 ? 0.0 : nr / den;    // hierarchy.py:129-131
    }
  }
}

// ---------------------------------------------------------------------------
// fused sweep (k = 1): uo = u + M(f - A u).  The residual over the tile plus a
// one-point halo is computed once into shared memory; the smoother then reads
// its 3x3 neighbourhood from there.

template <int TX, int TY, bool ZU>
__global__ void __launch_bounds__(NT) k_sweep(Grid g, Tab A, Tab K, const uint8_t* __restrict__ mask,
                                              const double* __restrict__ f,
                                              const double* __restrict__ u,
                                              double* __restrict__ uo) {
  constexpr int RW = TX + 2, RH = TY + 2;
  __shared__ double rs[RH * RW];
  const int b = blockIdx.z;
  const int64_t n = g.n();
  const int i0 = blockIdx.y * TY, j0 = blockIdx.x * TX;
  const int tid = threadIdx.y * BX + threadIdx.x;
  const double* fb = f + b * n;
  const double* ub = ZU ? nullptr : u + b * n;
  for (int q = tid; q < RH * RW; q += NT) {
    const int ri = q / RW, rj = q - ri * RW;
    const int i = i0 - 1 + ri, j = j0 - 1 + rj;
    double r = 0.0;
    if (i >= 0 && i < g.rows && j >= 0 && j < g.cols) {
      const int64_t p = (int64_t)i * g.cols + j;
      if (act(mask, p)) {
        if (ZU) r = __ldg(fb + p) - 0.0;
        else r = __ldg(fb + p) - stencil3(A, b, ub, i, j, g.rows, g.cols);
      }
    }
    rs[q] = r;
  }
  __syncthreads();
  for (int ti = threadIdx.y; ti < TY; ti += BY) {
    const int i = i0 + ti;
    if (i >= g.rows) break;
    for (int tj = threadIdx.x; tj < TX; tj += BX) {
      const int j = j0 + tj;
      if (j >= g.cols) break;
      const int64_t p = (int64_t)i * g.cols + j;
      double c = 0.0;
#pragma unroll
      for (int di = -1; di <= 1; ++di)
#pragma unroll
        for (int dj = -1; dj <= 1; ++dj)
          c = c + tab(K, b, 0, (di + 1) * 3 + (dj + 1), p) * rs[(ti + 1 + di) * RW + (tj + 1 + dj)];
      double v;
      if (!act(mask, p)) v = 0.0;
      else v = ZU ? 0.0 + c : __ldg(ub + p) + c;
      uo[b * n + p] = v;
    }
  }
}

// one stage of a (possibly multi-stage) per-point smoother
__global__ void __launch_bounds__(NT) k_pointwise(Grid g, Tab K, int stage, const uint8_t* __restrict__ mask,
                                                  const double* __restrict__ in, int lk, double slope,
                                                  const double* __restrict__ base,
                                                  double* __restrict__ out) {
  const int j = blockIdx.x * BX + threadIdx.x, i = blockIdx.y * BY + threadIdx.y, b = blockIdx.z;
  if (i >= g.rows || j >= g.cols) return;
  const int64_t n = g.n(), p = (int64_t)i * g.cols + j;
  const double* ib = in + b * n;
  double c = 0.0;
#pragma unroll
  for (int di = -1; di <= 1; ++di) {
    const int ii = i + di;
#pragma unroll
    for (int dj = -1; dj <= 1; ++dj) {
      const int jj = j + dj;
      double x = 0.0;
      if (ii >= 0 && ii < g.rows && jj >= 0 && jj < g.cols) {
        x = __ldg(ib + (int64_t)ii * g.cols + jj);
        if (lk) x = leaky(x, slope);
      }
      c = c + tab(K, b, stage, (di + 1) * 3 + (dj + 1), p) * x;
    }
  }
  double v = c;
  if (!act(mask, p)) v = 0.0;
  if (base) v = act(mask, p) ? __ldg(base + b * n + p) + v : 0.0;
  out[b * n + p] = v;
}

// ---------------------------------------------------------------------------
// full-weighting restriction (R = FW/16), fused with the fine residual.
// Coarse tile CTX x CTY; fine residual region (2CTY+1) x (2CTX+1) in smem.

__constant__ double c_fw[9] = {1.0 / 16, 2.0 / 16, 1.0 / 16, 2.0 / 16, 4.0 / 16,
                               2.0 / 16, 1.0 / 16, 2.0 / 16, 1.0 / 16};
__constant__ double c_pw[9] = {2.0 / 16, 4.0 / 16, 2.0 / 16, 4.0 / 16, 8.0 / 16,
                               4.0 / 16, 2.0 / 16, 4.0 / 16, 2.0 / 16};

template <int CTX, int CTY, int MODE>  // MODE 0: residual f - A u, 1: residual with u = 0, 2: plain fine values
__global__ void __launch_bounds__(NT) k_restrict(Grid g, Tab A, const uint8_t* __restrict__ mask_f,
                                                 const uint8_t* __restrict__ mask_c,
                                                 const double* __restrict__ f,
                                                 const double* __restrict__ u,
                                                 double* __restrict__ rc) {
  constexpr int FW_ = 2 * CTX + 1, FH = 2 * CTY + 1;
  __shared__ double rs[FH * FW_];
  const int b = blockIdx.z;
  const int64_t n = g.n();
  const int rows_c = g.rows / 2, cols_c = g.cols / 2;
  const int ci0 = blockIdx.y * CTY, cj0 = blockIdx.x * CTX;
  const int fi0 = 2 * ci0, fj0 = 2 * cj0;
  const int tid = threadIdx.y * BX + threadIdx.x;
  const double* fb = f + b * n;
  for (int q = tid; q < FH * FW_; q += NT) {
    const int ri = q / FW_, rj = q - ri * FW_;
    const int i = fi0 + ri, j = fj0 + rj;
    double r = 0.0;
    if (i < g.rows && j < g.cols) {
      const int64_t p = (int64_t)i * g.cols + j;
      if (MODE == 2) {
        r = __ldg(fb + p);
      } else if (act(mask_f, p)) {
        if (MODE == 1) r = __ldg(fb + p) - 0.0;
        else r = __ldg(fb + p) - stencil3(A, b, u + b * n, i, j, g.rows, g.cols);
      }
    }
    rs[q] = r;
  }
  __syncthreads();
  for (int ti = threadIdx.y; ti < CTY; ti += BY) {
    const int ci = ci0 + ti;
    if (ci >= rows_c) break;
    for (int tj = threadIdx.x; tj < CTX; tj += BX) {
      const int cj = cj0 + tj;
      if (cj >= cols_c) break;
      double s = 0.0;
#pragma unroll
      for (int di = 0; di < 3; ++di)
#pragma unroll
        for (int dj = 0; dj < 3; ++dj) s = s + c_fw[di * 3 + dj] * rs[(2 * ti + di) * FW_ + 2 * tj + dj];
      const int64_t pc = (int64_t)ci * cols_c + cj;
      rc[b * (int64_t)rows_c * cols_c + pc] = act(mask_c, pc) ? s : 0.0;
    }
  }
}

// prolongation (P = 2 FW/16) in gather form, contributions in the reference's
// (di, dj) order; optional coarse-grid correction u += P e.
template <bool ADD>
__global__ void __launch_bounds__(NT) k_prolong(Grid g, const uint8_t* __restrict__ mask_f,
                                                const double* __restrict__ ec,
                                                double* __restrict__ u) {
  const int j = blockIdx.x * BX + threadIdx.x, i = blockIdx.y * BY + threadIdx.y, b = blockIdx.z;
  if (i >= g.rows || j >= g.cols) return;
  const int rows_c = g.rows / 2, cols_c = g.cols / 2;
  const int64_t n = g.n(), p = (int64_t)i * g.cols + j;
  const double* eb = ec + b * (int64_t)rows_c * cols_c;
  double s = 0.0;
#pragma unroll
  for (int di = -1; di <= 1; ++di) {
    const int t = i - 1 - di;
    if (t < 0 || (t & 1)) continue;
    const int ci = t >> 1;
    if (ci >= rows_c) continue;
#pragma unroll
    for (int dj = -1; dj <= 1; ++dj) {
      const int tt = j - 1 - dj;
      if (tt < 0 || (tt & 1)) continue;
      const int cj = tt >> 1;
      if (cj >= cols_c) continue;
      s = s + c_pw[(di + 1) * 3 + (dj + 1)] * __ldg(eb + (int64_t)ci * cols_c + cj);
    }
  }
  const bool a = act(mask_f, p);
  if (!a) s = 0.0;
  if (ADD) u[b * n + p] = a ? u[b * n + p] + s : 0.0;
  else u[b * n + p] = s;
}

// ---------------------------------------------------------------------------
// Galerkin coarse operator, one thread per coarse point, chain order u, v, w
// exactly as transfer.py:166-198.
__global__ void __launch_bounds__(NT) k_galerkin(Grid g, Tab A, const uint8_t* __restrict__ mf,
                                                 const uint8_t* __restrict__ mc, TabW Ac,
                                                 int* __restrict__ ring, const int64_t* __restrict__ pts,
                                                 int npts) {
  const int rows_c = g.rows / 2, cols_c = g.cols / 2;
  int cj = blockIdx.x * BX + threadIdx.x, ci = blockIdx.y * BY + threadIdx.y;
  const int b = blockIdx.z;
  if (pts) {
    const int q = blockIdx.x * NT + threadIdx.y * BX + threadIdx.x;
    if (q >= npts || pts[q] < 0) return;
    ci = (int)(pts[q] / cols_c);
    cj = (int)(pts[q] % cols_c);
  }
  if (ci >= rows_c || cj >= cols_c) return;
  auto fmask = [&](int i, int j) -> double {
    if (i < 0 || i >= g.rows || j < 0 || j >= g.cols) return 0.0;
    return act(mf, (int64_t)i * g.cols + j) ? 1.0 : 0.0;
  };
  auto cmask = [&](int i, int j) -> double {
    if (i < 0 || i >= rows_c || j < 0 || j >= cols_c) return 0.0;
    return act(mc, (int64_t)i * cols_c + j) ? 1.0 : 0.0;
  };
  double acc[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) acc[q] = 0.0;
  for (int ui = -1; ui <= 1; ++ui)
    for (int uj = -1; uj <= 1; ++uj) {
      const double rw = c_fw[(ui + 1) * 3 + (uj + 1)];
      const int fi = 2 * ci + 1 + ui, fj = 2 * cj + 1 + uj;
      const double src = fmask(fi, fj);
      const bool fin = fi >= 0 && fi < g.rows && fj >= 0 && fj < g.cols;
      const int64_t fp = (int64_t)fi * g.cols + fj;
      for (int vi = -1; vi <= 1; ++vi)
        for (int vj = -1; vj <= 1; ++vj) {
          const double a = fin ? tab(A, b, 0, (vi + 1) * 3 + (vj + 1), fp) : 0.0;
          double e = a * src;
          e = e * fmask(fi + vi, fj + vj);
          for (int wi = -1; wi <= 1; ++wi) {
            const int xi = ui + vi - wi;
            if (xi & 1) continue;
            const int di = xi >> 1;  // exact: xi even, arithmetic shift = floor
            for (int wj = -1; wj <= 1; ++wj) {
              const int xj = uj + vj - wj;
              if (xj & 1) continue;
              const int dj = xj >> 1;
              const double pw = c_pw[(wi + 1) * 3 + (wj + 1)];
              const double tg = cmask(ci + di, cj + dj);
              const int q = (di + 1) * 3 + (dj + 1);
              acc[q] = acc[q] + ((rw * pw) * e) * tg;
            }
          }
        }
    }
  const int64_t pc = (int64_t)ci * cols_c + cj;
  if (!act(mc, pc)) {
#pragma unroll
    for (int q = 0; q < 9; ++q) acc[q] = (q == 4) ? 1.0 : 0.0;
  }
  bool nz = false;
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    if (q != 4 && acc[q] != 0.0) nz = true;
    tabw(Ac, b, 0, q, pc, acc[q]);
  }
  if (nz && ring) atomicOr(ring, 1);
}

// dense operator over active points: M[a][index[p_a + o]] = A(p_a)[o]
__global__ void k_materialize(Grid g, Tab A, const int32_t* __restrict__ index_map, int nact,
                              const int32_t* __restrict__ actp, double* __restrict__ M) {
  const int b = blockIdx.y;
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= nact) return;
  const int64_t p = actp[a];
  const int i = (int)(p / g.cols), j = (int)(p % g.cols);
  double* Mb = M + (int64_t)b * nact * nact;
  for (int di = -1; di <= 1; ++di)
    for (int dj = -1; dj <= 1; ++dj) {
      const int ii = i + di, jj = j + dj;
      if (ii < 0 || ii >= g.rows || jj < 0 || jj >= g.cols) continue;
      const int q = index_map[(int64_t)ii * g.cols + jj];
      if (q < 0) continue;
      Mb[(int64_t)a * nact + q] = tab(A, b, 0, (di + 1) * 3 + (dj + 1), p);
    }
}

// ---------------------------------------------------------------------------
// LU with partial pivoting, one block per problem (dense.py:21-47)

__global__ void __launch_bounds__(256) k_lu_factor(int n, double* __restrict__ LU,
                                                   int32_t* __restrict__ perm, int* __restrict__ status) {
  __shared__ double sv[256];
  __shared__ int si[256];
  __shared__ double s_scale;
  __shared__ int s_piv;
  const int b = blockIdx.x, t = threadIdx.x, nt = blockDim.x;
  double* a = LU + (int64_t)b * n * n;
  int32_t* pm = perm + (int64_t)b * n;
  for (int q = t; q < n; q += nt) pm[q] = q;
  // scale = max |A|
  double m = 0.0;
  for (int64_t q = t; q < (int64_t)n * n; q += nt) m = fmax(m, fabs(a[q]));
  sv[t] = m;
  __syncthreads();
  for (int o = nt / 2; o > 0; o >>= 1) {
    if (t < o) sv[t] = fmax(sv[t], sv[t + o]);
    __syncthreads();
  }
  if (t == 0) s_scale = sv[0];
  __syncthreads();
  const double scale = s_scale;
  if (scale == 0.0) {
    if (t == 0) status[b] = 0;
    return;
  }
  for (int k = 0; k < n; ++k) {
    // argmax |a[i][k]|, i >= k, first occurrence on ties (np.argmax)
    double bv = -1.0;
    int bi = n;
    for (int i = k + t; i < n; i += nt) {
      const double v = fabs(a[(int64_t)i * n + k]);
      if (v > bv) { bv = v; bi = i; }
    }
    sv[t] = bv;
    si[t] = bi;
    __syncthreads();
    for (int o = nt / 2; o > 0; o >>= 1) {
      if (t < o) {
        const double v2 = sv[t + o];
        const int i2 = si[t + o];
        if (v2 > sv[t] || (v2 == sv[t] && i2 < si[t])) { sv[t] = v2; si[t] = i2; }
      }
      __syncthreads();
    }
    if (t == 0) s_piv = si[0];
    __syncthreads();
    const int p = s_piv;
    if (fabs(a[(int64_t)p * n + k]) <= 1e-12 * scale) {
      if (t == 0) status[b] = k;
      return;
    }
    if (p != k) {
      for (int j = t; j < n; j += nt) {
        const double x = a[(int64_t)k * n + j];
        a[(int64_t)k * n + j] = a[(int64_t)p * n + j];
        a[(int64_t)p * n + j] = x;
      }
      if (t == 0) { const int32_t x = pm[k]; pm[k] = pm[p]; pm[p] = x; }
    }
    __syncthreads();
    const double piv = a[(int64_t)k * n + k];
    for (int i = k + 1 + t; i < n; i += nt) a[(int64_t)i * n + k] = a[(int64_t)i * n + k] / piv;
    __syncthreads();
    const int m2 = n - k - 1;
    for (int64_t q = t; q < (int64_t)m2 * m2; q += nt) {
      const int i = k + 1 + (int)(q / m2), j = k + 1 + (int)(q % m2);
      a[(int64_t)i * n + j] = a[(int64_t)i * n + j] - a[(int64_t)i * n + k] * a[(int64_t)k * n + j];
    }
    __syncthreads();
  }
  if (t == 0) status[b] = -1;
}

// forward (unit L) and backward (U) substitution, dense.py:50-63.
// x_full (grid mode): gathers f at active points, scatters the solution into the grid.
__global__ void __launch_bounds__(256) k_lu_solve(int n, const double* __restrict__ LU,
                                                  const int32_t* __restrict__ perm,
                                                  const int32_t* __restrict__ actp,
                                                  const double* __restrict__ f, int64_t fstride,
                                                  double* __restrict__ x, int64_t xstride) {
  extern __shared__ double xs[];
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.x, t = threadIdx.x, nt = blockDim.x;
  const double* a = LU + (int64_t)b * n * n;
  const int32_t* pm = perm + (int64_t)b * n;
  const double* fb = f + b * fstride;
  double* xb = x + b * xstride;
  if (n <= 32) {
    // the factors are staged in shared memory by the whole block (one round of L2
    // loads instead of 2n dependent ones), then one warp, unknowns over the lanes,
    // substitutes with shuffles: no block barriers on the latency path
    for (int q = t; q < n * n; q += nt) xs[q] = a[q];
    __syncthreads();
    if (t < 32) {
      double v = t < n ? (actp ? fb[actp[pm[t]]] : fb[pm[t]]) : 0.0;
      for (int k = 0; k < n; ++k) {
        const double xk = __shfl_sync(0xffffffffu, v, k);
        if (t > k && t < n) v = v - xs[t * n + k] * xk;
      }
      for (int k = n - 1; k >= 0; --k) {
        if (t == k) v = v / xs[k * n + k];
        const double xk = __shfl_sync(0xffffffffu, v, k);
        if (t < k) v = v - xs[t * n + k] * xk;
      }
      if (t < n) {
        if (actp) xb[actp[t]] = v;
        else xb[t] = v;
      }
    }
    return;
  }
  for (int q = t; q < n; q += nt) {
    const int src = pm[q];
    xs[q] = actp ? fb[actp[src]] : fb[src];
  }
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    const double xk = xs[k];
    for (int i = k + 1 + t; i < n; i += nt) xs[i] = xs[i] - a[(int64_t)i * n + k] * xk;
    __syncthreads();
  }
  for (int k = n - 1; k >= 0; --k) {
    if (t == 0) xs[k] = xs[k] / a[(int64_t)k * n + k];
    __syncthreads();
    const double xk = xs[k];
    for (int i = t; i < k; i += nt) xs[i] = xs[i] - a[(int64_t)i * n + k] * xk;
    __syncthreads();
  }
  if (actp) {
    for (int q = t; q < n; q += nt) xb[actp[q]] = xs[q];
  } else {
    for (int q = t; q < n; q += nt) xb[q] = xs[q];
  }
}

__global__ void __launch_bounds__(NT) k_jacobi(Grid g, Tab A, const uint8_t* __restrict__ mask,
                                               double omega, TabW K, int* __restrict__ flag,
                                               const int64_t* __restrict__ pts, int npts) {
  int j = blockIdx.x * BX + threadIdx.x, i = blockIdx.y * BY + threadIdx.y;
  const int b = blockIdx.z;
  if (pts) {
    const int q = blockIdx.x * NT + threadIdx.y * BX + threadIdx.x;
    if (q >= npts || pts[q] < 0) return;
    i = (int)(pts[q] / g.cols);
    j = (int)(pts[q] % g.cols);
  }
  if (i >= g.rows || j >= g.cols) return;
  const int64_t p = (int64_t)i * g.cols + j;
  const double d = tab(A, b, 0, 4, p);
  const bool a = act(mask, p);
  if (a && d == 0.0) atomicOr(flag, 1);
  for (int o = 0; o < 9; ++o) tabw(K, b, 0, o, p, (o == 4 && a && d != 0.0) ? omega / d : 0.0);
}

__global__ void __launch_bounds__(NT) k_convert(Grid g, int kst, Tab src, TabW dst) {
  const int j = blockIdx.x * BX + threadIdx.x, i = blockIdx.y * BY + threadIdx.y, b = blockIdx.z;
  if (i >= g.rows || j >= g.cols) return;
  const int64_t p = (int64_t)i * g.cols + j;
  for (int s = 0; s < kst; ++s)
    for (int o = 0; o < 9; ++o) tabw(dst, b, s, o, p, tab(src, b, s, o, p));
}

inline dim3 pgrid(const Grid& g) {
  return dim3((g.cols + BX - 1) / BX, (g.rows + BY - 1) / BY, g.batch);
}

}  // namespace

// ---------------------------------------------------------------------------
// launch wrappers

cudaError_t launch_apply(const Grid& g, int k, Tab A, const uint8_t* mask, const double* u,
                         double* out, cudaStream_t s) {
  ++g_launches;
  if (k == 3) k_apply<3><<<pgrid(g), dim3(BX, BY), 0, s>>>(g, A, mask, u, out);
  else k_apply<1><<<pgrid(g), dim3(BX, BY), 0, s>>>(g, A, mask, u, out);
  return MGB_DBG(__func__);
}

static dim3 resgrid(const Grid& g) {
  return dim3((g.cols + BX - 1) / BX, (g.rows + BY * RES_RPT - 1) / (BY * RES_RPT), g.batch);
}

int residual_blocks(const Grid& g) {
  const dim3 d = resgrid(g);
  return (int)(d.x * d.y);
}

cudaError_t launch_residual(const Grid& g, Tab A, const uint8_t* mask, const double* f,
                            const double* u, double* r, double* partials, int* nblk,
                            cudaStream_t s) {
  ++g_launches;
  if (nblk) *nblk = residual_blocks(g);
  k_residual<<<resgrid(g), dim3(BX, BY), 0, s>>>(g, A, mask, f, u, r, partials);
  return MGB_DBG(__func__);
}

cudaError_t launch_finalize(int batch, int nblk, const double* partials, double* out2,
                            const double* fnorm2, double* hist, int64_t hstride, cudaStream_t s) {
  ++g_launches;
  cudaError_t e = launch_pdl(k_finalize, dim3(batch), dim3(1024), 0, s, nblk, partials, out2, fnorm2, hist, hstride);
  if (e != cudaSuccess) return e;
  return MGB_DBG(__func__);
}

constexpr int SW_TX = 32, SW_TY = 32;

cudaError_t launch_sweep(const Grid& g, Tab A, Tab K, const uint8_t* mask, const double* f,
                         const double* u, double* uo, cudaStream_t s) {
  ++g_launches;
  dim3 grid((g.cols + SW_TX - 1) / SW_TX, (g.rows + SW_TY - 1) / SW_TY, g.batch);
  if (u) k_sweep<SW_TX, SW_TY, false><<<grid, dim3(BX, BY), 0, s>>>(g, A, K, mask, f, u, uo);
  else k_sweep<SW_TX, SW_TY, true><<<grid, dim3(BX, BY), 0, s>>>(g, A, K, mask, f, u, uo);
  return MGB_DBG(__func__);
}

cudaError_t launch_pointwise(const Grid& g, Tab K, int stage, const uint8_t* mask,
                             const double* in, bool lk, double slope, const double* base,
                             double* out, cudaStream_t s) {
  ++g_launches;
  k_pointwise<<<pgrid(g), dim3(BX, BY), 0, s>>>(g, K, stage, mask, in, lk ? 1 : 0, slope, base, out);
  return MGB_DBG(__func__);
}

constexpr int RS_CTX = 32, RS_CTY = 16;

static dim3 rgrid(const Grid& g) {
  const int rows_c = g.rows / 2, cols_c = g.cols / 2;
  return dim3((cols_c + RS_CTX - 1) / RS_CTX, (rows_c + RS_CTY - 1) / RS_CTY, g.batch);
}

cudaError_t launch_resid_restrict(const Grid& g, Tab A, const uint8_t* mask_f,
                                  const uint8_t* mask_c, const double* f, const double* u,
                                  double* rc, cudaStream_t s) {
  ++g_launches;
  if (u) k_restrict<RS_CTX, RS_CTY, 0><<<rgrid(g), dim3(BX, BY), 0, s>>>(g, A, mask_f, mask_c, f, u, rc);
  else k_restrict<RS_CTX, RS_CTY, 1><<<rgrid(g), dim3(BX, BY), 0, s>>>(g, A, mask_f, mask_c, f, u, rc);
  return MGB_DBG(__func__);
}

cudaError_t launch_restrict(const Grid& g, const uint8_t* mask_c, const double* fine,
                            double* coarse, cudaStream_t s) {
  ++g_launches;
  Tab none{nullptr, 0, 0, 0, 0};
  k_restrict<RS_CTX, RS_CTY, 2><<<rgrid(g), dim3(BX, BY), 0, s>>>(g, none, nullptr, mask_c, fine, nullptr, coarse);
  return MGB_DBG(__func__);
}

cudaError_t launch_prolong(const Grid& g, const uint8_t* mask_f, const double* coarse,
                           double* fine, bool add, cudaStream_t s) {
  ++g_launches;
  if (add) k_prolong<true><<<pgrid(g), dim3(BX, BY), 0, s>>>(g, mask_f, coarse, fine);
  else k_prolong<false><<<pgrid(g), dim3(BX, BY), 0, s>>>(g, mask_f, coarse, fine);
  return MGB_DBG(__func__);
}

cudaError_t launch_galerkin(const Grid& g, Tab A, const uint8_t* mask_f, const uint8_t* mask_c,
                            TabW Ac, int* ring_flag, cudaStream_t s, const int64_t* pts, int npts) {
  ++g_launches;
  const int rows_c = g.rows / 2, cols_c = g.cols / 2;
  dim3 grid = pts ? dim3((npts + NT - 1) / NT, 1, g.batch)
                  : dim3((cols_c + BX - 1) / BX, (rows_c + BY - 1) / BY, g.batch);
  k_galerkin<<<grid, dim3(BX, BY), 0, s>>>(g, A, mask_f, mask_c, Ac, ring_flag, pts, npts);
  return MGB_DBG(__func__);
}

cudaError_t launch_materialize(const Grid& g, Tab A, const int32_t* index_map, int nact,
                               const int32_t* actp, double* M, cudaStream_t s) {
  ++g_launches;
  dim3 grid((nact + 127) / 128, g.batch);
  k_materialize<<<grid, 128, 0, s>>>(g, A, index_map, nact, actp, M);
  return MGB_DBG(__func__);
}

cudaError_t launch_lu_factor(int batch, int n, double* lu, int32_t* perm, int* status,
                             cudaStream_t s) {
  ++g_launches;
  k_lu_factor<<<batch, 256, 0, s>>>(n, lu, perm, status);
  return MGB_DBG(__func__);
}

static cudaError_t lu_solve_smem(int n) {
  const size_t bytes = (size_t)n * sizeof(double);
  if (bytes > 48 * 1024)
    return cudaFuncSetAttribute(k_lu_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  return cudaSuccess;
}

cudaError_t launch_lu_solve_grid(const Grid& g, int n, const double* lu, const int32_t* perm,
                                 const int32_t* actp, const double* f, double* x,
                                 cudaStream_t s) {
  cudaError_t e = lu_solve_smem(n);
  if (e != cudaSuccess) return e;
  ++g_launches;
  // the coarse grid is zero outside the active set
  if (g.n() != n) {
    e = cudaMemsetAsync(x, 0, sizeof(double) * g.n() * g.batch, s);
    if (e != cudaSuccess) return e;
  }
  e = launch_pdl(k_lu_solve, dim3(g.batch), dim3(256), sizeof(double) * (n <= 32 ? n * n : n), s, n, lu, perm, actp, f,
                 g.n(), x, g.n());
  if (e != cudaSuccess) return e;
  return MGB_DBG(__func__);
}

cudaError_t launch_lu_solve_vec(int n, const double* lu, const int32_t* perm, const double* b,
                                double* x, cudaStream_t s) {
  cudaError_t e = lu_solve_smem(n);
  if (e != cudaSuccess) return e;
  ++g_launches;
  k_lu_solve<<<1, 256, sizeof(double) * (n <= 32 ? n * n : n), s>>>(n, lu, perm, nullptr, b, n, x, n);
  return MGB_DBG(__func__);
}

cudaError_t launch_jacobi(const Grid& g, Tab A, const uint8_t* mask, double omega, TabW K,
                          int* zero_diag_flag, cudaStream_t s, const int64_t* pts, int npts) {
  ++g_launches;
  const dim3 grid = pts ? dim3((npts + NT - 1) / NT, 1, g.batch) : pgrid(g);
  k_jacobi<<<grid, dim3(BX, BY), 0, s>>>(g, A, mask, omega, K, zero_diag_flag, pts, npts);
  return MGB_DBG(__func__);
}

cudaError_t launch_convert(const Grid& g, int kst, Tab src, TabW dst, cudaStream_t s) {
  ++g_launches;
  k_convert<<<pgrid(g), dim3(BX, BY), 0, s>>>(g, kst, src, dst);
  return MGB_DBG(__func__);
}

}  // namespace mgb
