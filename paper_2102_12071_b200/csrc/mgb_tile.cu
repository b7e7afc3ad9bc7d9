// Tile-local, temporally blocked V-cycle passes for the mid-size levels.
//
// The same PRE / sweep / POST passes as the row-streaming kernel (mgb_stream.cu),
// for levels too small to fill the GPU with row streams (below ~1.5 M points per
// launch).  There the cycle is launch- and latency-bound: as separate kernels a
// V(2,2) level costs 6 launches (sweep, sweep, residual+restriction; prolongation,
// sweep, sweep), each an L2 round trip.  Here each pass is ONE launch: a CTA owns
// a T x T tile of fine points, stages u and f over the tile plus a halo of S = the
// pass's stencil depth into shared memory, and runs every stage (residual, update,
// ..., residual, restriction) over a region that shrinks by one point per stage,
// with a __syncthreads between stages.  The halo work is redundant (the overlapped
// tile scheme); at these sizes latency, not arithmetic, is the bound.
//
// Arithmetic is the streaming kernel's, operation for operation (the same fused
// multiply-add chains in the same order), so both passes produce bit-identical u
// and restricted residuals (tested); the history partial sums differ only in the
// order of the per-CTA reduction.
//
// Reference: v_cycle hierarchy.py:96-111 with RepeatedSmoother cli.py:365-377,
// apply_stencil grid.py:216-226, inferred_apply smoothers.py:325-343, restrict
// transfer.py:108-121, prolong transfer.py:124-147, history hierarchy.py:129-141.
#include <atomic>
#include <algorithm>
#include <cstdlib>

#include "mgb_tile.h"
#include "mgb_dot.h"

#ifndef MGB_TILE_NTMAX
#define MGB_TILE_NTMAX 1024
#endif


namespace mgb {
namespace {

constexpr int NCLS = 25;

__device__ __forceinline__ int bandt(int i, int n) { return i < 2 ? i : (i >= n - 2 ? 4 - (n - 1 - i) : 2); }

template <int NSW, bool RES, bool PRO, int T>
struct TP {
  static constexpr int S = 2 * NSW + (RES ? 1 : 0);   // stencil stages after the input field
  static constexpr int C = T + (RES ? 1 : 0);         // core: the last stage's region
  static constexpr int W = C + 2 * S;                 // staged region side
  // threads: about one per staged point (small levels are latency-bound: a stage's
  // critical path is the points a thread evaluates in sequence), at most MGB_TILE_NTMAX
  static constexpr int NT = (W * W + 31) / 32 * 32 > MGB_TILE_NTMAX ? MGB_TILE_NTMAX : (W * W + 31) / 32 * 32;
  static constexpr int EH = W / 2 + 3;                // coarse correction rows/cols staged (POST)
};

template <int NSW, bool RES, bool PRO, bool NORM, bool ZU, bool CLS, bool MSK, int T>
__global__ void __launch_bounds__(TP<NSW, RES, PRO, T>::NT) k_tile(StreamArgs a) {
  using P = TP<NSW, RES, PRO, T>;
  constexpr int S = P::S, W = P::W, NT = P::NT, EH = P::EH;
  extern __shared__ double sm[];
  double* U = sm;                       // W x W: current u iterate
  double* R = U + W * W;                // W x W: current residual
  double* F = R + W * W;                // W x W: right-hand side
  double* E = F + W * W;                // EH x EH coarse correction (POST)
  double* tA = E + (PRO ? EH * EH : 0); // 25 x 9 band-class tables
  double* tK = tA + NCLS * 9;
  double* red = tK + NCLS * 9;          // NT / 32
  pdl_trigger();
  const Grid g = a.g;
  const int tid = threadIdx.x, b = blockIdx.z;
  const int64_t n = g.n();
  const int i0 = blockIdx.y * T, j0 = blockIdx.x * T;
  const int gi0 = i0 - S, gj0 = j0 - S;  // global coordinates of region point (0, 0)
  const double* fb = a.f + b * n;
  const double* ub = ZU ? nullptr : a.u + b * n;
  double* uob = a.uo + b * n;
  const uint8_t* mk = MSK ? a.mask : nullptr;

  if (CLS) {
    for (int q = tid; q < NCLS * 9; q += NT) {
      tA[q] = a.A.cls[(int64_t)b * NCLS * 9 + q];
      tK[q] = a.K.cls[(int64_t)b * NCLS * 9 + q];
    }
  }
  pdl_wait();  // u, f, ec come from the preceding kernels
  // ---- stage 0: f and the input u over the whole region (zero outside the grid)
  for (int q = tid; q < W * W; q += NT) {
    const int li = q / W, lj = q - (q / W) * W;
    const int i = gi0 + li, j = gj0 + lj;
    const bool in = (unsigned)i < (unsigned)g.rows && (unsigned)j < (unsigned)g.cols;
    const int64_t p = (int64_t)i * g.cols + j;
    F[q] = in ? __ldg(fb + p) : 0.0;
    if (!ZU) U[q] = in ? __ldg(ub + p) : 0.0;
  }
  if (PRO) {
    // coarse rows/cols ci0 .. ci0 + EH - 1 (anchors 2c + 1 within one point of the region)
    const int rows_c = g.rows / 2, cols_c = g.cols / 2;
    const int ci0 = (gi0 - 2) >> 1, cj0 = (gj0 - 2) >> 1;
    const double* ecb = a.ec + b * (int64_t)rows_c * cols_c;
    for (int q = tid; q < EH * EH; q += NT) {
      const int ei = q / EH, ej = q - (q / EH) * EH;
      const int ci = ci0 + ei, cj = cj0 + ej;
      E[q] = ((unsigned)ci < (unsigned)rows_c && (unsigned)cj < (unsigned)cols_c)
                 ? __ldg(ecb + (int64_t)ci * cols_c + cj) : 0.0;
    }
    __syncthreads();
    // u += P ec (gather form of the scatter-add prolongation, the streaming kernel's order)
    for (int q = tid; q < W * W; q += NT) {
      const int li = q / W, lj = q - (q / W) * W;
      const int i = gi0 + li, j = gj0 + lj;
      const bool in = (unsigned)i < (unsigned)g.rows && (unsigned)j < (unsigned)g.cols;
      double s = 0.0;
#pragma unroll
      for (int di = -1; di <= 1; ++di) {
        const int tt = i - 1 - di;
        if (tt & 1) continue;
#pragma unroll
        for (int dj = -1; dj <= 1; ++dj) {
          const int uu = j - 1 - dj;
          if (uu & 1) continue;
          const double wgt = (di == 0 ? 2.0 : 1.0) * (dj == 0 ? 2.0 : 1.0) * 0.125;
          s = fma(wgt, E[((tt >> 1) - ci0) * EH + (uu >> 1) - cj0], s);
        }
      }
      double v = U[q] + s;
      if (MSK && in && !mk[(int64_t)i * g.cols + j]) v = 0.0;
      U[q] = in ? v : 0.0;
    }
  }
  __syncthreads();

  double acc = 0.0;
  // ---- stages k = 1..S: odd = residual into R, even = smoother update of U; the
  // region of stage k is [k, W - k)^2
#pragma unroll
  for (int k = 1; k <= S; ++k) {
    const int lo = k, wk = W - 2 * k;
    const bool res_stage = k & 1;
    // zero start without a mask: r = f - A 0 = f is F itself (zero outside the grid),
    // so stage 1 only accumulates the history norm and stage 2 reads F
    constexpr bool ZF = ZU && !MSK;
    if (ZF && k == 1) {
      if (NORM) {
        for (int q = tid; q < wk * wk; q += NT) {
          const int li = lo + q / wk, lj = lo + q - (q / wk) * wk;
          const int i = gi0 + li, j = gj0 + lj;
          const bool in = (unsigned)i < (unsigned)g.rows && (unsigned)j < (unsigned)g.cols;
          const bool own = in && li >= S && li < S + T && lj >= S && lj < S + T;
          if (own) acc = fma(F[li * W + lj], F[li * W + lj], acc);
        }
      }
      continue;
    }
    const double* src = res_stage ? U : ((ZF && k == 2) ? F : R);  // the stage's input field
    const Op& op = res_stage ? a.A : a.K;
    for (int q = tid; q < wk * wk; q += NT) {
      const int li = lo + q / wk, lj = lo + q - (q / wk) * wk;
      const int i = gi0 + li, j = gj0 + lj;
      const bool in = (unsigned)i < (unsigned)g.rows && (unsigned)j < (unsigned)g.cols;
      const int64_t p = (int64_t)i * g.cols + j;
      const int lq = li * W + lj;
      double val = 0.0;
      if (in) {
        double wt[9];
        if (CLS) {
          const double* tab = (res_stage ? tA : tK) + (bandt(i, g.rows) * 5 + bandt(j, g.cols)) * 9;
#pragma unroll
          for (int o = 0; o < 9; ++o) wt[o] = tab[o];
        } else {
          const double* base = op.planes + (int64_t)b * 9 * op.n + p;
#pragma unroll
          for (int o = 0; o < 9; ++o) wt[o] = __ldg(base + (int64_t)o * op.n);
        }
        const double* sp = src + lq - W - 1;
        const double x0[3] = {sp[0], sp[1], sp[2]};
        const double x1[3] = {sp[W], sp[W + 1], sp[W + 2]};
        const double x2[3] = {sp[2 * W], sp[2 * W + 1], sp[2 * W + 2]};
        if (res_stage) {
          val = (ZU && k == 1) ? F[lq] : stencil_dot<true>(wt, x0, x1, x2, F[lq]);  // zero start: r = f
        } else {
          val = stencil_dot<false>(wt, x0, x1, x2, (ZU && k == 2) ? 0.0 : U[lq]);
        }
        if (MSK && !mk[p]) val = 0.0;
      }
      const bool own = in && li >= S && li < S + T && lj >= S && lj < S + T;
      if (res_stage) {
        R[lq] = val;
        if (NORM && k == 1 && own) acc = fma(val, val, acc);
      } else {
        U[lq] = val;
        if (k == 2 * NSW && own) uob[p] = val;
      }
    }
    __syncthreads();
  }
  if (RES) {
    // full-weighting restriction of the last residual at the tile's coarse points
    const int rows_c = g.rows / 2, cols_c = g.cols / 2;
    constexpr int TC = T / 2;
    for (int q = tid; q < TC * TC; q += NT) {
      const int ci = (i0 >> 1) + q / TC, cj = (j0 >> 1) + q % TC;
      if (ci >= rows_c || cj >= cols_c) continue;
      const int li = 2 * ci - gi0, lj = 2 * cj - gj0;  // region index of fine (2ci, 2cj)
      const double* r0p = R + li * W + lj;
      const double* r1p = r0p + W;
      const double* r2p = r1p + W;
      double s = 0.0625 * r0p[0];
      s = fma(0.125, r0p[1], s);
      s = fma(0.0625, r0p[2], s);
      s = fma(0.125, r1p[0], s);
      s = fma(0.25, r1p[1], s);
      s = fma(0.125, r1p[2], s);
      s = fma(0.0625, r2p[0], s);
      s = fma(0.125, r2p[1], s);
      s = fma(0.0625, r2p[2], s);
      const int64_t pc = (int64_t)ci * cols_c + cj;
      const bool actc = a.mask_c == nullptr || a.mask_c[pc];
      a.rc[b * (int64_t)rows_c * cols_c + pc] = actc ? s : 0.0;
    }
  }
  if (NORM) {
    double v = acc;
    const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[wid] = v;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int q = 0; q < NT / 32; ++q) s += red[q];
      a.partials[(int64_t)b * gridDim.x * gridDim.y + blockIdx.y * gridDim.x + blockIdx.x] = s;
    }
  }
}

template <int NSW, bool RES, bool PRO, int T>
constexpr size_t tile_smem() {
  using P = TP<NSW, RES, PRO, T>;
  return sizeof(double) * (3 * P::W * P::W + (PRO ? P::EH * P::EH : 0) + 2 * NCLS * 9 + P::NT / 32);
}

template <int NSW, bool RES, bool PRO, bool NORM, bool ZU, bool CLS, bool MSK, int T>
cudaError_t run_tile(const StreamArgs& a, int* nblocks) {
  auto kern = k_tile<NSW, RES, PRO, NORM, ZU, CLS, MSK, T>;
  constexpr size_t smem = tile_smem<NSW, RES, PRO, T>();
  static std::atomic<uint64_t> attr{0};  // per instantiation: one bit per device set up
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr.load(std::memory_order_acquire) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr.fetch_or(bit, std::memory_order_acq_rel);
  }
  const dim3 grid((a.g.cols + T - 1) / T, (a.g.rows + T - 1) / T, a.g.batch);
  if (nblocks) *nblocks = (int)(grid.x * grid.y);
  const cudaError_t e = launch_pdl(kern, grid, dim3(TP<NSW, RES, PRO, T>::NT), smem, a.stream, a);
  if (e != cudaSuccess) return e;
  return MGB_DBG("k_tile");
}

template <int NSW, bool RES, bool PRO, bool NORM, bool ZU, bool CLS, bool MSK>
cudaError_t run_tile_t(const StreamArgs& a, int T, int* nblocks) {
  if (T == 32) return run_tile<NSW, RES, PRO, NORM, ZU, CLS, MSK, 32>(a, nblocks);
  if (T == 16) return run_tile<NSW, RES, PRO, NORM, ZU, CLS, MSK, 16>(a, nblocks);
  return run_tile<NSW, RES, PRO, NORM, ZU, CLS, MSK, 8>(a, nblocks);
}

}  // namespace

// Tile side: the largest of 32, 16, 8 that still gives every SM a CTA
int tile_side(const Grid& g) {
  static const int force = getenv("MGB_TILE_T") ? atoi(getenv("MGB_TILE_T")) : 0;  // experiments only
  if (force == 8 || force == 16 || force == 32) return force;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  // one CTA per SM is enough: fewer, larger tiles re-stage fewer halo points (measured:
  // 255^2 on 16-tiles 12.4 us per V(2,2) level vs 15.9 on 8-tiles, 511^2 and 256 x 31^2
  // on 32-tiles), but no tile wider than the grid needs (256 x 15^2: 16-tiles 6.3 us,
  // 32-tiles 10.4)
  for (int T = 32; T > 8; T /= 2) {
    if (T / 2 >= std::max(g.rows, g.cols)) continue;
    const int64_t ctas = (int64_t)((g.rows + T - 1) / T) * ((g.cols + T - 1) / T) * g.batch;
    if (ctas >= sms) return T;
  }
  return 8;
}

int tile_max_blocks(const Grid& g) { return ((g.rows + 7) / 8) * ((g.cols + 7) / 8); }

cudaError_t launch_tile(const StreamArgs& a, int nsw, bool res, bool pro, bool norm, int* nblocks) {
  const bool zu = a.u == nullptr;
  const bool msk = a.mask != nullptr;
  const bool cls = a.A.cls != nullptr && a.K.cls != nullptr;
  if (a.A.ks != 1 || a.K.ks != 1 || (!cls && (!a.A.planes || !a.K.planes))) return cudaErrorInvalidValue;
  const int T = tile_side(a.g);
  ++g_launches;
#define MGB_TL(NSW_, RES_, PRO_, NORM_, ZU_)                                                              \
  if (nsw == NSW_ && res == RES_ && pro == PRO_ && norm == NORM_ && zu == ZU_) {                        \
    if (cls && msk) return run_tile_t<NSW_, RES_, PRO_, NORM_, ZU_, true, true>(a, T, nblocks);         \
    if (cls) return run_tile_t<NSW_, RES_, PRO_, NORM_, ZU_, true, false>(a, T, nblocks);               \
    if (msk) return run_tile_t<NSW_, RES_, PRO_, NORM_, ZU_, false, true>(a, T, nblocks);               \
    return run_tile_t<NSW_, RES_, PRO_, NORM_, ZU_, false, false>(a, T, nblocks);                        \
  }
  MGB_TL(1, true, false, false, false) MGB_TL(1, true, false, true, false)
  MGB_TL(1, true, false, false, true)  MGB_TL(1, true, false, true, true)
  MGB_TL(2, true, false, false, false) MGB_TL(2, true, false, true, false)
  MGB_TL(2, true, false, false, true)  MGB_TL(2, true, false, true, true)
  MGB_TL(1, false, false, false, false) MGB_TL(1, false, false, true, false)
  MGB_TL(1, false, false, false, true)  MGB_TL(1, false, false, true, true)
  MGB_TL(1, false, true, false, false) MGB_TL(2, false, true, false, false)
#undef MGB_TL
  return cudaErrorInvalidValue;
}

}  // namespace mgb
