// Row-streaming, temporally blocked V-cycle passes (the level-l hot kernels).
//
//   PRE(l)  = [history norm of the input u] + NSW sweeps u <- u + M (f - A u)
//             + residual + full-weighting restriction   -> u_out, rc
//   POST(l) = prolongation/coarse-grid correction u <- u + P ec + NSW sweeps -> u_out
//
// One CTA owns a strip of SWOUT columns (plus a halo of H columns on each side,
// one column per thread) and a segment of rows, and marches down the rows: at
// step t it brings in row t of u and f (cp.async prefetch ring, D rows ahead)
// and advances every pipeline stage by one row.  Stage k (k = 1..S, odd =
// residual, even = smoother update) produces row t - 2k, so every stage reads
// only rows that earlier steps published and one __syncthreads per step is
// enough.  Each stage keeps the 3x3 window of its input field in registers
// (own column + left/right neighbours, exchanged through a double-buffered
// shared-memory row); the own-column residual and update values never leave
// registers.  u and f are read from HBM once per pass and u is written once,
// so a V(2,2) cycle level costs ~2 x (16 + 8) B per point instead of
// 4 x 24 + 18 + 18 + 16 for separate passes.
//
// A, M: band-class tables (constant-coefficient levels; 25 x 9 in shared
// memory, the interior class in registers) or per-point planes (read through
// L1/L2).  Arithmetic uses fused multiply-add; results agree with the separate
// passes and with the reference to rounding (SURVEY §8(c) gate: 1e-10).
//
// Reference: v_cycle hierarchy.py:96-111 (with RepeatedSmoother cli.py:365-377),
// apply_stencil grid.py:216-226, inferred_apply smoothers.py:325-343, restrict
// transfer.py:108-121, prolong transfer.py:124-147, history hierarchy.py:129-141.
#include <cstdlib>
#include <utility>
#include <vector>
#include <algorithm>

#include "mgb_stream.h"
#include "mgb_dot.h"

namespace mgb {
namespace {

#ifndef MGB_SWT
#define MGB_SWT 128
#endif
constexpr int SWT = MGB_SWT;  // threads (= columns incl. halo) per CTA
constexpr int PD = 8;      // prefetch ring depth (rows) for u (power of two)
constexpr int PDF = 16;    // ring depth for f (also read by the later residual stages): rows t-10 .. t+DIST
constexpr int DIST = 5;    // prefetch distance (rows ahead)
#ifndef MGB_MINB
#define MGB_MINB 3
#endif
constexpr int MINB = MGB_MINB;  // CTAs per SM the register budget is sized for
constexpr int PE = 8;      // ring of coarse rows (POST prolongation), power of two
constexpr int EW = SWT / 2 + 4;  // coarse columns staged per CTA
constexpr int NCLS = 25;
constexpr int CINT = 12;   // interior band class (2 * 5 + 2)

__device__ __forceinline__ int bandc(int i, int n) { return i < 2 ? i : (i >= n - 2 ? 4 - (n - 1 - i) : 2); }

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Per-point planes (CM 0): the rows of A are read by stages 1, 3, 5 (8 steps apart)
// and those of M by stages 2, 4, so the reuse lives in L2.  A plane row's last read is
// marked evict-first so the rows still to be reused are the ones that stay.  (The same
// hint on the cp.async ring copies makes ptxas emit an LDGSTS that faults: not used.)
#ifndef MGB_EVH
#define MGB_EVH 1
#endif
// 1: each step's plane weights are loaded into registers at the end of the previous
// step (before its barrier), so their L2 latency overlaps the barrier and the
// neighbour exchange instead of stalling the stage chains (2 CTAs/SM: 255 registers)
#ifndef MGB_WPRE
#define MGB_WPRE 1
#endif
// the L2 cache-policy word of createpolicy.fractional.L2::evict_first 1.0 (the value
// CUTLASS uses for its TMA hints); an immediate, so it lands in a uniform register
constexpr uint64_t POL_EVICT_FIRST = 0x12F0000000000000ull;
__device__ __forceinline__ double ldg_hint(const double* ptr, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;\n" : "=d"(v) : "l"(ptr), "l"(pol));
  return v;
}

// CM 0: the first-use plane rows (A for stage 1, M for stage 2) are prefetched into L2
// by the ring issue, MGB_L2PF_AHEAD steps beyond the ring's DIST rows, so the register
// loads of every stage hit L2 (the passes were load-latency bound at 8 warps/SM)
#ifndef MGB_L2PF
#define MGB_L2PF 1
#endif
#ifndef MGB_L2PF_AHEAD
#define MGB_L2PF_AHEAD 0
#endif
__device__ __forceinline__ void prefetch_l2(const double* p) {
  asm volatile("prefetch.global.L2::evict_last [%0];\n" ::"l"(p));
}
// One warp-wide pass: the warp's 32 columns of a plane row span at most three 128-byte
// lines, touched by columns wc0, wc0 + 16 and wc0 + 31, so lane q prefetches line
// (q mod 3) of plane item q / 3 (A's nonzero planes at rowA, then M's nine at rowM):
// two prefetch instructions per warp and step instead of one per plane.
__device__ __forceinline__ void prefetch_planes(const StreamArgs& a, int b, const Grid& g, int wc0, int rowA, int rowM,
                                                int lane) {
  const int nA = a.a5 ? 5 : 9;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int q = lane + 32 * r, item = q / 3, part = q - 3 * item;
    if (item >= nA + 9) break;
    const bool isA = item < nA;
    const int row = isA ? rowA : rowM;
    if ((unsigned)row >= (unsigned)g.rows) continue;
    const int plane = !isA ? item - nA : (!a.a5 ? item : (item < 2 ? 2 * item + 1 : (item == 4 ? 7 : item + 2)));
    const int col = min(max(wc0 + (part == 0 ? 0 : (part == 1 ? 16 : 31)), 0), g.cols - 1);
    const Op& op = isA ? a.A : a.K;
    prefetch_l2(op.planes + (int64_t)b * 9 * op.n + (int64_t)plane * op.n + ((int64_t)row * g.cols + col));
  }
}

template <int NSW, bool RES, bool PRO>
struct SP {
  static constexpr int S = 2 * NSW + (RES ? 1 : 0);  // stencil stages after the input field
  static constexpr int H = 2 * NSW + 2;              // column halo per side
  static constexpr int WOUT = SWT - 2 * H;           // owned columns per strip (even)
  static constexpr int NF = S;                       // fields with a window (F_0 .. F_{S-1})
};

// compile-time positive modulo 3
__host__ __device__ constexpr int m3(int x) { return ((x % 3) + 3) % 3; }

// 3x3 dot product over the register window (slots s0, s1, s2 = rows di = -1, 0, 1);
// the same function as the tile passes (mgb_tile.cu), so both round identically
template <bool NEG>
__device__ __forceinline__ double dot9(const double* wt, const double (&x)[3][3], int s0, int s1, int s2,
                                       double init) {
  return stencil_dot<NEG>(wt, x[s0], x[s1], x[s2], init);
}

// Per-CTA constants of a streaming pass.
struct Ctx {
  Grid g;
  int b, tid, j0, col, colL, colR, R0, R1;
  bool cin, owned_c;
  int ccls;
  const double* fb;
  const double* ub;
  double* uob;
  double* ring_u;
  double* ring_f;
  double* ring_e;   // PE x EW coarse correction rows (POST)
  int cjb;          // coarse column of ring_e entry 0
  double* xch;
  double* rlast;
  const double* tA;
  const double* tK;
  const uint8_t* mk;
};

// The nine per-point weights of stage k (odd: A, even: M) at (row, column); a plane
// row's last read (A at stage S (PRE) / S - 1 (POST), M at stage 2 NSW) is evict-first.
template <int NSW, bool RES>
__device__ __forceinline__ void load_planes(const StreamArgs& a, const Ctx& c, int k, int row, double (&wt)[9]) {
  constexpr int S = 2 * NSW + (RES ? 1 : 0);
  const Op& op = (k & 1) ? a.A : a.K;
  const double* base = op.planes + (int64_t)c.b * 9 * op.n + ((int64_t)row * c.g.cols + (c.cin ? c.col : 0));
  const bool last = MGB_EVH && (k == (RES ? S : S - 1) || k == 2 * NSW);
  // 5-point A: the corner weights are exact zeros (checked at build), so the chains are
  // unchanged and 4 of the 9 plane reads are saved
  const bool skipc = (k & 1) && a.a5;
#pragma unroll
  for (int o = 0; o < 9; ++o) {
    if ((o == 0 || o == 2 || o == 6 || o == 8) && skipc) {
      wt[o] = 0.0;
    } else {
      wt[o] = last ? ldg_hint(base + (int64_t)o * op.n, POL_EVICT_FIRST) : __ldg(base + (int64_t)o * op.n);
    }
  }
}

// One pipeline step (row t).  FAST: every row the step touches is an interior
// row, every column of the CTA is an interior in-grid column, so no bounds,
// band-class or column tests are needed.  PH = t mod 3 (window slots).
template <int NSW, bool RES, bool PRO, bool NORM, bool ZU, int CM, bool MSK, bool FAST, int PH>
__device__ __forceinline__ void stream_step(const StreamArgs& a, const Ctx& c, const int t,
                                            double (&w)[SP<NSW, RES, PRO>::NF][3][3], double (&hold)[NSW],
                                            double& acc, double (&wp)[SP<NSW, RES, PRO>::S][9]) {
  using P = SP<NSW, RES, PRO>;
  constexpr int S = P::S, H = P::H, WOUT = P::WOUT, NF = P::NF;
  constexpr bool CL = CM != 0;
  const Grid& g = c.g;
  double nv[NF + 1];
  // ---- F_0 = u (+ P ec) at row t
  {
    double u0 = 0.0;
    const bool rv = FAST || ((unsigned)t < (unsigned)g.rows && c.cin);
    if (!ZU) u0 = c.ring_u[(t & (PD - 1)) * SWT + c.tid];
    if (PRO && rv) {
      // u += P ec with the coarse rows staged in shared memory (ring_e)
      double s = 0.0;
#pragma unroll
      for (int di = -1; di <= 1; ++di) {
        const int tt = t - 1 - di;
        if (tt & 1) continue;
        const double* er = c.ring_e + ((tt >> 1) & (PE - 1)) * EW;  // out-of-range rows were zero-filled
#pragma unroll
        for (int dj = -1; dj <= 1; ++dj) {
          const int uu = c.col - 1 - dj;
          if (uu & 1) continue;
          const double wgt = (di == 0 ? 2.0 : 1.0) * (dj == 0 ? 2.0 : 1.0) * 0.125;
          s = fma(wgt, er[(uu >> 1) - c.cjb], s);
        }
      }
      u0 += s;
    }
    if (MSK && rv && !c.mk[(int64_t)t * g.cols + c.col]) u0 = 0.0;
    nv[0] = (FAST || rv) ? u0 : 0.0;
  }
  // ---- stages k = 1..S at row t - 2k (rows are CTA-uniform)
#pragma unroll
  for (int k = 1; k <= S; ++k) {
    const int row = t - 2 * k;
    constexpr int dummy = 0;
    (void)dummy;
    const int s0 = m3(PH - 2 * k - 1), s1 = m3(PH - 2 * k), s2 = m3(PH - 2 * k + 1);
    double val = 0.0;
    if (FAST || (unsigned)row < (unsigned)g.rows) {
      const Op& op = (k & 1) ? a.A : a.K;
      const bool res_stage = k & 1;
      const double init = res_stage ? c.ring_f[(row & (PDF - 1)) * SWT + c.tid] : hold[k / 2 - 1];
      if (ZU && k == 1) {
        val = init;  // zero start: r = f - A 0 = f (as the tile passes)
      } else if (!CL) {
        double wt[9];
        if (MGB_WPRE) {
#pragma unroll
          for (int o = 0; o < 9; ++o) wt[o] = wp[k - 1][o];
        } else {
          load_planes<NSW, RES>(a, c, k, row, wt);
        }
        val = res_stage ? dot9<true>(wt, w[k - 1], s0, s1, s2, init) : dot9<false>(wt, w[k - 1], s0, s1, s2, init);
      } else if (FAST) {
        const double* reg = CM == 2 ? ((k & 1) ? a.ci : a.ci + 9) : (((k & 1) ? c.tA : c.tK) + CINT * 9);
        val = res_stage ? dot9<true>(reg, w[k - 1], s0, s1, s2, init) : dot9<false>(reg, w[k - 1], s0, s1, s2, init);
      } else {
        const double* tab = (k & 1) ? c.tA : c.tK;
        const double* wt = tab + (bandc(row, g.rows) * 5 + c.ccls) * 9;
        val = res_stage ? dot9<true>(wt, w[k - 1], s0, s1, s2, init) : dot9<false>(wt, w[k - 1], s0, s1, s2, init);
      }
      if (MSK && c.cin && !c.mk[(int64_t)row * g.cols + c.col]) val = 0.0;
      if (!FAST) val = c.cin ? val : 0.0;
      if (NORM && k == 1 && c.owned_c && row >= c.R0 && row < c.R1) acc = fma(val, val, acc);
      if (k == 2 * NSW && a.uo && c.owned_c && row >= c.R0 && row < c.R1) c.uob[(int64_t)row * g.cols + c.col] = val;
    }
    nv[k] = val;
  }
  // ---- publish, then slide the windows (slot of the evicted row)
  const int sl = t & 1;
#pragma unroll
  for (int k = 0; k < NF; ++k) c.xch[(k * 2 + sl) * SWT + c.tid] = nv[k];
  if (RES) c.rlast[((t - 2 * S) & 3) * SWT + c.tid] = nv[S];
  if (!CL && MGB_WPRE) {
    // plane weights of step t + 1 (its stage rows are CTA-uniform)
#pragma unroll
    for (int k = ZU ? 2 : 1; k <= S; ++k) {
      const int row = t + 1 - 2 * k;
      if ((unsigned)row < (unsigned)g.rows) load_planes<NSW, RES>(a, c, k, row, wp[k - 1]);
    }
  }
  __syncthreads();
  if (RES) {
    const int top = t - 2 * S;
    if (top >= 2 && !(top & 1)) {
      const int ci = (top - 2) >> 1;
      const int rows_c = g.rows / 2, cols_c = g.cols / 2;
      const int cj = (c.j0 >> 1) + c.tid;
      if (c.tid < WOUT / 2 && ci >= (c.R0 >> 1) && 2 * ci + 1 < c.R1 && ci < rows_c && cj < cols_c) {
        const int base = H + 2 * c.tid;
        const double* r0p = &c.rlast[((top - 2) & 3) * SWT + base];
        const double* r1p = &c.rlast[((top - 1) & 3) * SWT + base];
        const double* r2p = &c.rlast[(top & 3) * SWT + base];
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
        a.rc[c.b * (int64_t)rows_c * cols_c + pc] = actc ? s : 0.0;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NF; ++k) {
    const int sn = m3(PH - 2 * k);  // slot of the new row t - 2k (evicts row t - 2k - 3)
    if (!(k & 1) && k / 2 < NSW) hold[k / 2] = w[k][sn][1];
    w[k][sn][0] = c.xch[(k * 2 + sl) * SWT + c.colL];
    w[k][sn][1] = nv[k];
    w[k][sn][2] = c.xch[(k * 2 + sl) * SWT + c.colR];
  }
}

// CM: 0 = per-point planes for A and M; 1 = band-class tables in shared memory;
// 2 = band-class tables with the interior class read from the kernel parameters
// (constant-bank operands: no registers, no shared-memory traffic).
template <int NSW, bool RES, bool PRO, bool NORM, bool ZU, int CM, bool MSK>
__global__ void __launch_bounds__(SWT, (CM == 0 && MGB_WPRE) ? 2 : MINB) k_stream(StreamArgs a) {
  pdl_trigger();
  using P = SP<NSW, RES, PRO>;
  constexpr int S = P::S, H = P::H, WOUT = P::WOUT, NF = P::NF;
  extern __shared__ double smem[];
  Ctx c;
  c.g = a.g;
  const Grid& g = c.g;
  c.ring_u = smem;                               // PD x SWT (unused when ZU)
  c.ring_f = c.ring_u + PD * SWT;                // PDF x SWT
  c.ring_e = c.ring_f + PDF * SWT;               // PE x EW (POST only; allocated always)
  c.xch = c.ring_e + PE * EW;                    // NF x 2 x SWT neighbour exchange rows
  c.rlast = c.xch + NF * 2 * SWT;                // 4 x SWT last-residual ring (RES)
  double* tA = c.rlast + 4 * SWT;                // 25 x 9
  double* tK = tA + NCLS * 9;                    // 25 x 9
  double* red = tK + NCLS * 9;                   // 32
  c.tA = tA;
  c.tK = tK;
  c.tid = threadIdx.x;
  c.b = blockIdx.z;
  const int64_t n = g.n();
  c.j0 = blockIdx.x * WOUT;                      // first owned column (even)
  c.col = c.j0 - H + c.tid;
  c.cin = c.col >= 0 && c.col < g.cols;
  c.owned_c = c.tid >= H && c.tid < H + WOUT && c.cin;
  c.ccls = c.cin ? bandc(c.col, g.cols) : 2;     // out-of-grid columns are zeroed anyway
  c.cjb = ((c.j0 - H) >> 1) - 1;
  c.R0 = a.own0 + blockIdx.y * a.seg;
  c.R1 = min(a.own1 > 0 ? a.own1 : g.rows, c.R0 + a.seg);
  c.fb = a.f + c.b * n;
  c.ub = ZU ? nullptr : a.u + c.b * n;
  c.uob = a.uo + c.b * n;
  c.colL = max(c.tid - 1, 0);
  c.colR = min(c.tid + 1, SWT - 1);
  c.mk = MSK ? a.mask : nullptr;
  // fast steps need every CTA column interior (band class 2) and in the grid
  const bool cta_fast = c.j0 - H >= 2 && c.j0 - H + SWT - 1 <= g.cols - 3;

  if (CM != 0) {
    for (int q = c.tid; q < NCLS * 9; q += SWT) {
      tA[q] = a.A.cls[(int64_t)c.b * NCLS * 9 + q];
      tK[q] = a.K.cls[(int64_t)c.b * NCLS * 9 + q];
    }
  }
  __syncthreads();
  pdl_wait();  // u, f, ec come from the preceding kernels

  double w[NF][3][3];
#pragma unroll
  for (int k = 0; k < NF; ++k)
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int q = 0; q < 3; ++q) w[k][r][q] = 0.0;
  double hold[NSW];
#pragma unroll
  for (int m = 0; m < NSW; ++m) hold[m] = 0.0;
  double acc = 0.0;
  double wp[S][9];  // CM 0: plane weights of the next step
  if (CM == 0 && MGB_WPRE) {
#pragma unroll
    for (int k = 1; k <= S; ++k)
#pragma unroll
      for (int o = 0; o < 9; ++o) wp[k - 1][o] = 0.0;
  }

  // steps t in [t0, t1], t0 aligned to a multiple of 3 (extra leading steps only
  // compute rows nobody needs)
  int t0 = c.R0 - S - 1;
  t0 -= m3(t0);
  const int t1 = c.R1 + 2 * S;
  int prow = t0;
  const int64_t cstride = g.cols;
  const double* pu = ZU ? nullptr : c.ub + (int64_t)prow * cstride + c.col;
  const double* pf = c.fb + (int64_t)prow * cstride + c.col;
  const int rows_c = g.rows / 2, cols_c = g.cols / 2;
  const double* ecb = PRO ? a.ec + c.b * (int64_t)rows_c * cols_c : nullptr;
  // rows the owned outputs depend on (a ghost band of S + 1 rows each side); rows
  // outside are never read, so domain-decomposed blocks need only S + 1 ghost rows
  const int lo_row = max(0, c.R0 - S - 1), hi_row = min(g.rows - 1, c.R1 + S);
  const int lo_c = (lo_row - 2) >> 1, hi_c = (hi_row >> 1) + 1;
  auto issue = [&]() {
    const bool rv = prow >= lo_row && prow <= hi_row && c.cin;
    // (a zero-size copy reads nothing: the row pointer is passed unselected)
    if (!ZU) cp_async8(&c.ring_u[(prow & (PD - 1)) * SWT + c.tid], pu, rv);
    cp_async8(&c.ring_f[(prow & (PDF - 1)) * SWT + c.tid], pf, rv);
    if (PRO && !(prow & 1) && c.tid < EW) {
      // coarse row ci is first needed by fine row 2ci (as di = -1); stage it with the
      // group of fine row 2ci - 2 so every thread's copy is complete and published by
      // the barrier of step 2ci - 2.  Out-of-range coarse points read as zero.
      const int ci = (prow >> 1) + 1, cj = c.cjb + c.tid;
      const bool ev = ci >= 0 && ci < rows_c && ci >= lo_c && ci <= hi_c && cj >= 0 && cj < cols_c;
      cp_async8(&c.ring_e[(ci & (PE - 1)) * EW + c.tid], ev ? ecb + (int64_t)ci * cols_c + cj : ecb, ev);
    }
    if (CM == 0 && MGB_L2PF)
      prefetch_planes(a, c.b, g, c.col - (c.tid & 31), prow + MGB_L2PF_AHEAD - (ZU ? 6 : 2),
                      prow + MGB_L2PF_AHEAD - 4, c.tid & 31);  // zero start: A first read by stage 3
    cp_commit();
    ++prow;
    if (!ZU) pu += cstride;
    pf += cstride;
  };
  if (PRO) {
    // coarse rows needed before the first regular issue can stage them
    for (int ci = (t0 >> 1) - 1; ci <= (t0 >> 1) + 1; ++ci) {
      const int cj = c.cjb + c.tid;
      if (c.tid < EW) {
        const bool ev = ci >= 0 && ci < rows_c && ci >= lo_c && ci <= hi_c && cj >= 0 && cj < cols_c;
        cp_async8(&c.ring_e[(ci & (PE - 1)) * EW + c.tid], ev ? ecb + (int64_t)ci * cols_c + cj : ecb, ev);
      }
    }
    cp_commit();
    cp_wait<0>();
    __syncthreads();
  }
  for (int q = 0; q < DIST; ++q) issue();
  if (CM == 0 && MGB_WPRE) {
#pragma unroll
    for (int k = ZU ? 2 : 1; k <= S; ++k) {
      const int row = t0 - 2 * k;
      if ((unsigned)row < (unsigned)g.rows) load_planes<NSW, RES>(a, c, k, row, wp[k - 1]);
    }
  }

#define MGB_STEP(PH_)                                                                                  \
  {                                                                                                    \
    const int t = tb + PH_;                                                                            \
    issue();                                                                                           \
    cp_wait<DIST>();                                                                                   \
    if (cta_fast && t - 2 * S >= 2 && t <= g.rows - 3)                                                 \
      stream_step<NSW, RES, PRO, NORM, ZU, CM, MSK, true, PH_>(a, c, t, w, hold, acc, wp);                 \
    else                                                                                               \
      stream_step<NSW, RES, PRO, NORM, ZU, CM, MSK, false, PH_>(a, c, t, w, hold, acc, wp);                \
  }
  for (int tb = t0; tb <= t1; tb += 3) {
    MGB_STEP(0)
    MGB_STEP(1)
    MGB_STEP(2)
  }
#undef MGB_STEP
  cp_wait<0>();
  if (NORM) {
    double v = acc;
    const int lane = c.tid & 31, wid = c.tid >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[wid] = v;
    __syncthreads();
    if (c.tid == 0) {
      double s = 0.0;
      for (int q = 0; q < SWT / 32; ++q) s += red[q];
      a.partials[(int64_t)c.b * gridDim.x * gridDim.y + blockIdx.y * gridDim.x + blockIdx.x] = s;
    }
  }
}

}  // namespace

static size_t stream_smem(int nsw, bool res) {
  const int nf = 2 * nsw + (res ? 1 : 0);
  return sizeof(double) * ((size_t)(PD + PDF + 2 * nf + 4) * SWT + PE * EW + 2 * NCLS * 9 + 32);
}

// Rows per CTA segment: minimise waves x (segment + pipeline fill) for the
// kernel's measured occupancy (the whole grid runs ~one row step per CTA at a time).
// Any segment length is allowed, so the grid can be sized to fill whole waves
// (e.g. 4095 rows x 36 strips: 12 segments of 342 rows = 432 CTAs, one wave on
// 148 SMs x 3, instead of 2.6 waves of 128-row segments).
static int choose_seg(const Grid& g, int nsw, bool res, int occ) {
  const int H = 2 * nsw + 2, wout = SWT - 2 * H, S = 2 * nsw + (res ? 1 : 0);
  const int64_t strips = (g.cols + wout - 1) / wout;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int64_t slots = (int64_t)sms * std::max(occ, 1);
  int best = g.rows;
  double best_t = 1e300;
  // measured: per-step cost rises with the segment length beyond ~128 rows (4095^2:
  // 64 -> 481 us, 128 -> 485, 171 -> 544, 256 -> 660 per V(2,2) level), so segments
  // are capped and the count is chosen to fill whole waves below the cap
  // (very large grids, many waves even at 512-row segments, keep long segments:
  // 32767^2 measured 6% faster at 512 than at 96)
  static const int seg_max_env = getenv("MGB_SEG_MAX") ? atoi(getenv("MGB_SEG_MAX")) : 0;
  const int64_t ctas512 = strips * (int64_t)((g.rows + 511) / 512) * g.batch;
  const int seg_max = seg_max_env > 0 ? seg_max_env : (ctas512 >= 8 * slots ? 512 : 96);
  for (int nseg = 1; nseg <= std::max(1, g.rows / 16); ++nseg) {
    const int seg = (g.rows + nseg - 1) / nseg;
    if (seg > seg_max && nseg < g.rows / 16) continue;
    const int64_t ctas = strips * (int64_t)((g.rows + seg - 1) / seg) * g.batch;
    const int64_t waves = (ctas + slots - 1) / slots;
    // a partial last wave still costs a full CTA time; fill = 3S + 3 steps
    const double t = (double)waves * (seg + 3 * S + 3);
    if (t < best_t) { best_t = t; best = seg; }
  }
  return best;
}

template <typename KF>
static cudaError_t run_k(KF kern, int nsw, bool res, StreamArgs a, int* nblocks) {
  // the >48 KB shared-memory attribute and the occupancy are per device
  struct Occ {
    const void* k;
    int dev, occ;
  };
  static thread_local std::vector<Occ> occ_cache;
  const size_t smem = stream_smem(nsw, res);
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  int occ = -1;
  for (auto& e : occ_cache)
    if (e.k == (const void*)kern && e.dev == dev) occ = e.occ;
  if (occ < 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, SWT, smem);
    if (e != cudaSuccess) return e;
    occ_cache.push_back({(const void*)kern, dev, occ});
  }
  static const int force_seg = getenv("MGB_SEG") ? atoi(getenv("MGB_SEG")) : 0;  // experiments only
  if (a.own1 <= 0) {
    a.own0 = 0;
    a.own1 = a.g.rows;
  }
  Grid go = a.g;
  go.rows = a.own1 - a.own0;
  a.seg = force_seg > 0 ? force_seg : choose_seg(go, nsw, res, occ);
  const int H = 2 * nsw + 2, wout = SWT - 2 * H;
  const dim3 grid((a.g.cols + wout - 1) / wout, (go.rows + a.seg - 1) / a.seg, a.g.batch);
  if (nblocks) *nblocks = (int)(grid.x * grid.y);
  const cudaError_t e = launch_pdl(kern, grid, dim3(SWT), smem, a.stream, a);
  if (e != cudaSuccess) return e;
  return MGB_DBG(__func__);
}

// The warp-strip kernel (mgb_stream3.cu) runs where it is forced (kernel 3) and, by
// default, on single-problem uniform band-class levels of at least 1M points (config
// 2 / 5 level 0); MGB_STREAM3=0 / 1 turns the default off / extends it to every
// single-problem band-class level of that size (A/B experiments).
bool warp_strip_selected(int kernel, int64_t n, int batch, bool uniform, int nsw) {
  static const int env = getenv("MGB_STREAM3") ? atoi(getenv("MGB_STREAM3")) : -1;
  static const bool no_batch = getenv("MGB_STREAM3_BATCH") && atoi(getenv("MGB_STREAM3_BATCH")) == 0;   // A/B experiments
  if (batch > 1 && (nsw != 1 || !uniform || no_batch)) return false;   // batched flavour: uniform levels, one sweep per pass
  if (kernel == 3) return true;
  static const int64_t min_n = getenv("MGB_STREAM3_MIN") ? atoll(getenv("MGB_STREAM3_MIN")) : 1000000;
  if (kernel != 0 || n * batch < min_n || env == 0) return false;
  return uniform || env == 1;
}

cudaError_t launch_stream(const StreamArgs& a, int nsw, bool res, bool pro, bool norm, int* nblocks) {
  const bool zu = a.u == nullptr;
  const bool msk = a.mask != nullptr;
  const int cm = (a.A.cls != nullptr && a.K.cls != nullptr && !msk) ? (a.ci_valid ? 2 : 1) : 0;
  static const bool one_col = getenv("MGB_STREAM1") && atoi(getenv("MGB_STREAM1")) != 0;
  ++g_launches;
  // column-pair kernel: band-class levels of >= 1M points (batch included; interior
  // weights from the constant bank or, batched, from registers)
  const bool pairs = a.kernel == 2 || (a.kernel == 0 && !one_col && a.g.n() * a.g.batch >= 1000000);
  if ((cm == 2 || (cm == 1 && a.g.batch > 1)) && warp_strip_selected(a.kernel, a.g.n(), a.g.batch, a.uniform != 0, nsw) &&
      stream3_ok(a, nsw))
    return launch_stream3(a, nsw, res, pro, norm, nblocks);
  if (cm != 0 && (pairs || a.kernel == 3)) return launch_stream2(a, nsw, res, pro, norm, nblocks);
#define MGB_ST(NSW_, RES_, PRO_, NORM_, ZU_)                                                           \
  if (nsw == NSW_ && res == RES_ && pro == PRO_ && norm == NORM_ && zu == ZU_) {                     \
    if (msk) return run_k(k_stream<NSW_, RES_, PRO_, NORM_, ZU_, 0, true>, nsw, res, a, nblocks);     \
    if (cm == 2) return run_k(k_stream<NSW_, RES_, PRO_, NORM_, ZU_, 2, false>, nsw, res, a, nblocks); \
    if (cm == 1) return run_k(k_stream<NSW_, RES_, PRO_, NORM_, ZU_, 1, false>, nsw, res, a, nblocks); \
    return run_k(k_stream<NSW_, RES_, PRO_, NORM_, ZU_, 0, false>, nsw, res, a, nblocks);             \
  }
  // PRE (restriction, optional history norm, optional zero start), plain sweeps,
  // POST (prolongation)
  MGB_ST(1, true, false, false, false) MGB_ST(1, true, false, true, false)
  MGB_ST(1, true, false, false, true)  MGB_ST(1, true, false, true, true)
  MGB_ST(2, true, false, false, false) MGB_ST(2, true, false, true, false)
  MGB_ST(2, true, false, false, true)  MGB_ST(2, true, false, true, true)
  MGB_ST(1, false, false, false, false) MGB_ST(1, false, false, true, false)
  MGB_ST(1, false, false, false, true)  MGB_ST(1, false, false, true, true)
  MGB_ST(1, false, true, false, false) MGB_ST(2, false, true, false, false)
#undef MGB_ST
  return cudaErrorInvalidValue;
}

int stream_kernel_kind(const StreamArgs& a, int nsw) {
  const int cm = (a.A.cls != nullptr && a.K.cls != nullptr && a.mask == nullptr) ? (a.ci_valid ? 2 : 1) : 0;
  static const bool one_col = getenv("MGB_STREAM1") && atoi(getenv("MGB_STREAM1")) != 0;
  const bool pairs = a.kernel == 2 || (a.kernel == 0 && !one_col && a.g.n() * a.g.batch >= 1000000);
  if ((cm == 2 || (cm == 1 && a.g.batch > 1)) && warp_strip_selected(a.kernel, a.g.n(), a.g.batch, a.uniform != 0, nsw) &&
      stream3_ok(a, nsw))
    return 3;
  if (cm != 0 && (pairs || a.kernel == 3)) return 2;
  return 1;
}

int stream_max_blocks(const Grid& g) {
  // upper bound on the CTAs of any streaming pass over g (segments of at least 16 rows; the
  // warp-strip kernel's edge strips down to 8: counted with 8 for every strip)
  const int wout = SWT - 2 * 4 - 4;
  return (int)(((g.cols + wout - 1) / wout) * ((g.rows + 7) / 8));
}

}  // namespace mgb
