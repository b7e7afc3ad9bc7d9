// The coarse end of the V-cycle in ONE launch: one CTA per problem runs every
// level below a size threshold (sweeps, residual, restriction, the coarsest LU
// solve, prolongation) with all of those levels' u, f, r and class tables
// resident in shared memory and __syncthreads between dependent phases.
// Coarse levels are latency-bound (a few thousand points each): as separate
// kernels each pass costs a launch and an HBM/L2 round trip, here a phase costs
// a block barrier and shared-memory accesses.
//
// Reference: v_cycle hierarchy.py:96-111 (V(nu1, nu2) as RepeatedSmoother,
// cli.py:365-377), coarse_solve hierarchy.py:91-93 / lu_solve dense.py:50-63,
// restrict transfer.py:108-121, prolong transfer.py:124-147.
#include <cstdlib>

#include "mgb_coarse.h"
#include "mgb_dot.h"

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

// smem-resident variant of apply9: v in shared memory, weights from the level's
// class table (shared) or per-point planes (global)
struct SLevel {
  int rows, cols;
  const double* tA;      // shared class tables (null: planes)
  const double* tK;
};

__device__ __forceinline__ double apply9s(const Op& t, const double* tab, int b, const double* v, int i, int j,
                                          int rows, int cols) {
  const int64_t p = (int64_t)i * cols + j;
  const double* w = tab ? tab + (bandk(i, rows) * 5 + bandk(j, cols)) * 9 : nullptr;
  double s = 0.0;
#pragma unroll
  for (int di = -1; di <= 1; ++di) {
    const int ii = i + di;
    if (ii < 0 || ii >= rows) continue;
#pragma unroll
    for (int dj = -1; dj <= 1; ++dj) {
      const int jj = j + dj;
      if (jj < 0 || jj >= cols) continue;
      const int o = (di + 1) * 3 + dj + 1;
      const double wo = w ? w[o] : __ldg(t.planes + (int64_t)b * 9 * t.n + (int64_t)o * t.n + p);
      s = fma(wo, v[ii * cols + jj], s);
    }
  }
  return s;
}

// One CTA per problem runs levels lv[0..nlev-1] with every level's u, f, r (and
// the class tables) resident in shared memory; phases are separated by
// __syncthreads only.
__global__ void __launch_bounds__(CT) k_coarse_block(CoarseArgs a) {
  extern __shared__ double sm[];
  const int b = blockIdx.x;
  const int tid = threadIdx.x;
  // carve shared memory: per level u, f, r (rows*cols each), then class tables
  double* su[COARSE_MAX_LEVELS];
  double* sf[COARSE_MAX_LEVELS];
  double* sr[COARSE_MAX_LEVELS];
  const double* stA[COARSE_MAX_LEVELS];
  const double* stK[COARSE_MAX_LEVELS];
  double* cur = sm;
  for (int l = 0; l < a.nlev; ++l) {
    const int n = a.lv[l].rows * a.lv[l].cols;
    su[l] = cur; cur += n;
    sf[l] = cur; cur += n;
    sr[l] = cur; cur += n;
  }
  for (int l = 0; l < a.nlev; ++l) {
    stA[l] = nullptr;
    stK[l] = nullptr;
    if (a.lv[l].A.cls) {
      for (int q = tid; q < NCLS * 9; q += CT) cur[q] = a.lv[l].A.cls[(int64_t)b * NCLS * 9 + q];
      stA[l] = cur;
      cur += NCLS * 9;
    }
    if (l + 1 < a.nlev && a.lv[l].K.cls) {
      for (int q = tid; q < NCLS * 9; q += CT) cur[q] = a.lv[l].K.cls[(int64_t)b * NCLS * 9 + q];
      stK[l] = cur;
      cur += NCLS * 9;
    }
  }
  double* xs = cur;  // coarsest LU work vector
  {
    const CLevel& L = a.lv[0];
    const int n = L.rows * L.cols;
    for (int p = tid; p < n; p += CT) sf[0][p] = L.f[(int64_t)b * n + p];
    if (!a.zero_top)
      for (int p = tid; p < n; p += CT) su[0][p] = L.u[(int64_t)b * n + p];
  }
  __syncthreads();

  auto act = [&](int l, int p) { return !a.lv[l].mask || a.lv[l].mask[p]; };
  auto sweep = [&](int l, bool zero) {
    const CLevel& L = a.lv[l];
    const int n = L.rows * L.cols;
    for (int p = tid; p < n; p += CT) {
      const int i = p / L.cols, j = p - (p / L.cols) * L.cols;
      double v = 0.0;
      if (act(l, p)) v = zero ? sf[l][p] : sf[l][p] - apply9s(L.A, stA[l], b, su[l], i, j, L.rows, L.cols);
      sr[l][p] = v;
    }
    __syncthreads();
    for (int p = tid; p < n; p += CT) {
      const int i = p / L.cols, j = p - (p / L.cols) * L.cols;
      double v = 0.0;
      if (act(l, p)) v = (zero ? 0.0 : su[l][p]) + apply9s(L.K, stK[l], b, sr[l], i, j, L.rows, L.cols);
      su[l][p] = v;
    }
    __syncthreads();
  };

  for (int l = 0; l + 1 < a.nlev; ++l) {
    const CLevel& L = a.lv[l];
    const CLevel& Cc = a.lv[l + 1];
    const bool zero0 = l > 0 || a.zero_top;
    const int n = L.rows * L.cols;
    for (int q = 0; q < a.nu1; ++q) sweep(l, zero0 && q == 0);
    if (a.nu1 == 0 && zero0) {
      for (int p = tid; p < n; p += CT) su[l][p] = 0.0;
      __syncthreads();
    }
    for (int p = tid; p < n; p += CT) {
      const int i = p / L.cols, j = p - (p / L.cols) * L.cols;
      sr[l][p] = act(l, p) ? sf[l][p] - apply9s(L.A, stA[l], b, su[l], i, j, L.rows, L.cols) : 0.0;
    }
    __syncthreads();
    const int nc = Cc.rows * Cc.cols;
    for (int pc = tid; pc < nc; pc += CT) {
      const int ci = pc / Cc.cols, cj = pc - (pc / Cc.cols) * Cc.cols;
      double s = 0.0;
#pragma unroll
      for (int di = 0; di < 3; ++di)
#pragma unroll
        for (int dj = 0; dj < 3; ++dj) {
          const int fi = 2 * ci + di, fj = 2 * cj + dj;
          const double wv = (di == 1 ? 2.0 : 1.0) * (dj == 1 ? 2.0 : 1.0) * 0.0625;
          if (fi < L.rows && fj < L.cols) s = fma(wv, sr[l][fi * L.cols + fj], s);
        }
      sf[l + 1][pc] = act(l + 1, pc) ? s : 0.0;
    }
    __syncthreads();
  }
  {
    const int lc = a.nlev - 1;
    const CLevel& L = a.lv[lc];
    const int n = L.rows * L.cols;
    const int nn = a.nc;
    const double* lu = a.lu + (int64_t)b * nn * nn;
    const int32_t* pm = a.perm + (int64_t)b * nn;
    for (int q = tid; q < n; q += CT) su[lc][q] = 0.0;
    if (nn <= 32) {
      // one warp: forward (unit lower) and back substitution with the unknowns
      // distributed over the lanes (dense.py:50-63 order of operations)
      if (tid < 32) {
        const int i = tid;
        double x = i < nn ? sf[lc][a.actp[pm[i]]] : 0.0;
        for (int k = 0; k < nn; ++k) {
          const double xk = __shfl_sync(0xffffffffu, x, k);
          if (i > k && i < nn) x = x - __ldg(lu + (int64_t)i * nn + k) * xk;
        }
        for (int k = nn - 1; k >= 0; --k) {
          if (i == k) x = x / __ldg(lu + (int64_t)k * nn + k);
          const double xk = __shfl_sync(0xffffffffu, x, k);
          if (i < k) x = x - __ldg(lu + (int64_t)i * nn + k) * xk;
        }
        xs[i] = x;
      }
    } else {
      for (int q = tid; q < nn; q += CT) xs[q] = sf[lc][a.actp[pm[q]]];
      __syncthreads();
      for (int k = 0; k < nn; ++k) {
        const double xk = xs[k];
        for (int i = k + 1 + tid; i < nn; i += CT) xs[i] = xs[i] - lu[(int64_t)i * nn + k] * xk;
        __syncthreads();
      }
      for (int k = nn - 1; k >= 0; --k) {
        if (tid == 0) xs[k] = xs[k] / lu[(int64_t)k * nn + k];
        __syncthreads();
        const double xk = xs[k];
        for (int i = tid; i < k; i += CT) xs[i] = xs[i] - lu[(int64_t)i * nn + k] * xk;
        __syncthreads();
      }
    }
    __syncthreads();
    for (int q = tid; q < nn; q += CT) su[lc][a.actp[q]] = xs[q];
    __syncthreads();
  }
  for (int l = a.nlev - 2; l >= 0; --l) {
    const CLevel& L = a.lv[l];
    const CLevel& Cc = a.lv[l + 1];
    const int n = L.rows * L.cols;
    for (int p = tid; p < n; p += CT) {
      const int i = p / L.cols, j = p - (p / L.cols) * L.cols;
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
          s = fma(wv, su[l + 1][(t >> 1) * Cc.cols + (tt >> 1)], s);
        }
      }
      su[l][p] = act(l, p) ? su[l][p] + s : 0.0;
    }
    __syncthreads();
    for (int q = 0; q < a.nu2; ++q) sweep(l, false);
  }
  {
    const CLevel& L = a.lv[0];
    const int n = L.rows * L.cols;
    for (int p = tid; p < n; p += CT) L.u[(int64_t)b * n + p] = su[0][p];
  }
}


// ---- fast path: band-class levels of at most 1024 points, no masks, zero start ---------
// One point per thread on every level; every level's u, f, r sit in shared memory with a
// zero ring around them (no bounds tests: the ring is the zero closure of grid.py:27-35),
// a thread's class-table rows are looked up once per level visit, and every stage is the
// stencil_dot chain of the tile / streaming passes (mgb_dot.h) in their stage order, so the
// result is bitwise the per-level passes' (tested).  Replaces 2 launches per level plus the
// LU launch by one launch: the levels up to 31^2 of a V(2,2) cycle cost ~19 us as separate
// launches (launch latency) and run here in a few microseconds.
struct TailLevel {
  int rows, cols, P;     // P: padded pitch (cols + 2)
  double *U, *F, *R;     // (rows + 2) x P each, interior at (+1, +1)
  const double *tA, *tK; // 25 x 9 class tables in shared memory
};

__global__ void __launch_bounds__(CT) k_coarse_tail(CoarseArgs a) {
  extern __shared__ double sm[];
  pdl_trigger();
  const int b = blockIdx.x, tid = threadIdx.x;
  __shared__ TailLevel lv[COARSE_MAX_LEVELS];   // level descriptors (dynamic level index: not registers)
  double* cur = sm;
  size_t grid_doubles = 0;
  for (int l = 0; l < a.nlev; ++l) {
    const int P = a.lv[l].cols + 2, cnt = (a.lv[l].rows + 2) * P;
    if (tid == 0) {
      TailLevel& t = lv[l];
      t.rows = a.lv[l].rows;
      t.cols = a.lv[l].cols;
      t.P = P;
      t.U = cur;
      t.F = cur + cnt;
      t.R = cur + 2 * cnt;
    }
    cur += 3 * cnt;
    grid_doubles += 3 * (size_t)cnt;
  }
  for (size_t q = tid; q < grid_doubles; q += CT) sm[q] = 0.0;   // fields and their zero rings
  for (int l = 0; l < a.nlev; ++l) {
    for (int q = tid; q < NCLS * 9; q += CT) {
      cur[q] = a.lv[l].A.cls[(int64_t)b * NCLS * 9 + q];
      if (l + 1 < a.nlev) cur[NCLS * 9 + q] = a.lv[l].K.cls[(int64_t)b * NCLS * 9 + q];
    }
    if (tid == 0) {
      lv[l].tA = cur;
      lv[l].tK = cur + NCLS * 9;
    }
    cur += 2 * NCLS * 9;
  }
  const int nn = a.nc;
  double* slu = cur;            // coarsest factors
  for (int q = tid; q < nn * nn; q += CT) slu[q] = a.lu[(int64_t)b * nn * nn + q];
  pdl_wait();                   // f of the top level comes from the preceding pass
  __syncthreads();
  {
    const TailLevel t = lv[0];
    const int n = t.rows * t.cols;
    if (tid < n) {
      const int i = tid / t.cols, j = tid - i * t.cols;
      t.F[(i + 1) * t.P + j + 1] = a.lv[0].f[(int64_t)b * n + tid];
    }
  }
  __syncthreads();

  // the thread's point on level l: padded index q and its class-table rows
  struct Pt {
    bool on;
    int i, j, q;
    const double *wA, *wK;
  };
  auto point = [&](int l) {
    const TailLevel t = lv[l];
    Pt p;
    p.on = tid < t.rows * t.cols;
    p.i = p.on ? tid / t.cols : 0;
    p.j = p.on ? tid - p.i * t.cols : 0;
    p.q = (p.i + 1) * t.P + p.j + 1;
    const int cls = bandk(p.i, t.rows) * 5 + bandk(p.j, t.cols);
    p.wA = t.tA + cls * 9;
    p.wK = t.tK + cls * 9;
    return p;
  };
  auto resid = [&](const TailLevel& t, const Pt& p) {   // R = F - A U
    if (p.on) {
      const double* s = t.U + p.q - t.P - 1;
      t.R[p.q] = stencil_dot<true>(p.wA, s, s + t.P, s + 2 * t.P, t.F[p.q]);
    }
    __syncthreads();
  };
  auto update = [&](const TailLevel& t, const Pt& p, const double* src, bool from_zero) {   // U = U + K src
    if (p.on) {
      const double* s = src + p.q - t.P - 1;
      t.U[p.q] = stencil_dot<false>(p.wK, s, s + t.P, s + 2 * t.P, from_zero ? 0.0 : t.U[p.q]);
    }
    __syncthreads();
  };

  // ---- down: nu1 sweeps from zero, residual, full weighting
  for (int l = 0; l + 1 < a.nlev; ++l) {
    const TailLevel t = lv[l];
    const TailLevel c = lv[l + 1];
    const Pt p = point(l);
    update(t, p, t.F, true);           // r = f - A 0 = f: the first sweep reads f itself
    for (int q = 1; q < a.nu1; ++q) {
      resid(t, p);
      update(t, p, t.R, false);
    }
    resid(t, p);
    if (tid < c.rows * c.cols) {
      const int ci = tid / c.cols, cj = tid - ci * c.cols;
      const double* r0 = t.R + (2 * ci + 1) * t.P + 2 * cj + 1;
      const double* r1 = r0 + t.P;
      const double* r2 = r1 + t.P;
      double s = 0.0625 * r0[0];
      s = fma(0.125, r0[1], s);
      s = fma(0.0625, r0[2], s);
      s = fma(0.125, r1[0], s);
      s = fma(0.25, r1[1], s);
      s = fma(0.125, r1[2], s);
      s = fma(0.0625, r2[0], s);
      s = fma(0.125, r2[1], s);
      s = fma(0.0625, r2[2], s);
      c.F[(ci + 1) * c.P + cj + 1] = s;
    }
    __syncthreads();
  }
  // ---- coarsest: one warp, forward (unit lower) and back substitution (dense.py:50-63)
  {
    const TailLevel t = lv[a.nlev - 1];
    const int32_t* pm = a.perm + (int64_t)b * nn;
    auto padded = [&](int flat) { return (flat / t.cols + 1) * t.P + flat % t.cols + 1; };
    if (tid < 32) {
      const int i = tid;
      double x = i < nn ? t.F[padded(a.actp[pm[i]])] : 0.0;
      for (int k = 0; k < nn; ++k) {
        const double xk = __shfl_sync(0xffffffffu, x, k);
        if (i > k && i < nn) x = x - slu[i * nn + k] * xk;
      }
      for (int k = nn - 1; k >= 0; --k) {
        if (i == k) x = x / slu[k * nn + k];
        const double xk = __shfl_sync(0xffffffffu, x, k);
        if (i < k) x = x - slu[i * nn + k] * xk;
      }
      if (i < nn) t.U[padded(a.actp[i])] = x;
    }
    __syncthreads();
  }
  // ---- up: u += P e (the tile pass's gather order), nu2 sweeps
  for (int l = a.nlev - 2; l >= 0; --l) {
    const TailLevel t = lv[l];
    const TailLevel c = lv[l + 1];
    const Pt p = point(l);
    if (p.on) {
      double s = 0.0;
#pragma unroll
      for (int di = -1; di <= 1; ++di) {
        const int tt = p.i - 1 - di;
        if (tt & 1) continue;
#pragma unroll
        for (int dj = -1; dj <= 1; ++dj) {
          const int uu = p.j - 1 - dj;
          if (uu & 1) continue;
          const double wgt = (di == 0 ? 2.0 : 1.0) * (dj == 0 ? 2.0 : 1.0) * 0.125;
          s = fma(wgt, c.U[((tt >> 1) + 1) * c.P + (uu >> 1) + 1], s);
        }
      }
      t.U[p.q] = t.U[p.q] + s;
    }
    __syncthreads();
    for (int q = 0; q < a.nu2; ++q) {
      resid(t, p);
      update(t, p, t.R, false);
    }
  }
  {
    const TailLevel t = lv[0];
    const int n = t.rows * t.cols;
    if (tid < n) {
      const int i = tid / t.cols, j = tid - i * t.cols;
      a.lv[0].u[(int64_t)b * n + tid] = t.U[(i + 1) * t.P + j + 1];
    }
  }
}

static bool tail_ok(const CoarseArgs& a) {
  if (!a.zero_top || a.nc > 32 || a.nu1 < 1 || a.nu1 > 2 || a.nu2 < 1 || a.nu2 > 2) return false;
  for (int l = 0; l < a.nlev; ++l) {
    const CLevel& c = a.lv[l];
    if (c.rows * c.cols > CT || c.mask || !c.A.cls || (l + 1 < a.nlev && !c.K.cls)) return false;
  }
  return true;
}

static size_t tail_smem(const CoarseArgs& a) {
  size_t d = 0;
  for (int l = 0; l < a.nlev; ++l) d += 3 * (size_t)(a.lv[l].rows + 2) * (a.lv[l].cols + 2) + 2 * NCLS * 9;
  return (d + (size_t)a.nc * a.nc) * sizeof(double);
}

}  // namespace

size_t coarse_block_smem(const CoarseArgs& a) {
  size_t d = 0;
  for (int l = 0; l < a.nlev; ++l) {
    d += 3 * (size_t)a.lv[l].rows * a.lv[l].cols;
    if (a.lv[l].A.cls) d += NCLS * 9;
    if (l + 1 < a.nlev && a.lv[l].K.cls) d += NCLS * 9;
  }
  d += std::max(a.nc, 32);
  return d * sizeof(double);
}

cudaError_t launch_coarse_block(const CoarseArgs& a, int batch, cudaStream_t s) {
  static const bool no_tail = getenv("MGB_COARSE_TAIL") && atoi(getenv("MGB_COARSE_TAIL")) == 0;   // A/B experiments
  if (!no_tail && tail_ok(a)) {
    const size_t tsm = tail_smem(a);
    cudaError_t e = cudaFuncSetAttribute(k_coarse_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm);
    if (e != cudaSuccess) return e;
    ++g_launches;
    e = launch_pdl(k_coarse_tail, dim3(batch), dim3(CT), tsm, s, a);
    if (e != cudaSuccess) return e;
    return MGB_DBG("k_coarse_tail");
  }
  const size_t smem = coarse_block_smem(a);
  cudaError_t e = cudaFuncSetAttribute(k_coarse_block, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  ++g_launches;
  k_coarse_block<<<batch, CT, smem, s>>>(a);
  return MGB_DBG(__func__);
}

}  // namespace mgb
