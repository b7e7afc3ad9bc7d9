// Row-streaming V-cycle passes, two columns per thread (band-class levels).
//
// The same PRE / sweep / POST passes and the same pipeline as k_stream
// (mgb_stream.cu): a CTA owns a strip of columns and a segment of rows, marches
// down the rows, and stage k (odd = residual, even = smoother update) produces
// row t - 2k at step t, each stage keeping the 3x3 window of its input field in
// registers.  The difference is the work per thread: every thread owns a column
// PAIR (2c, 2c+1), so the per-row fixed cost of a step (prefetch issue, the
// barrier, loop control, neighbour exchange, row tests) is paid once per two
// points and the two columns' fused-multiply-add chains interleave (ILP 2 x S).
// The strip is 256 columns (128 threads), so the column halo costs 12/256 instead
// of 12/128.  With one column per thread the level-0 pass issued ~240
// instructions per fine point for ~50 FP64 FMAs (issue-bound, ncu r01); the pair
// form halves the non-FMA part.
//
// Only band-class levels run here (A and M constant per band class: every
// constant-coefficient operator, its Galerkin chain and its CNN kernels), without
// masks; per-point planes and masked levels stay on k_stream.  The FMA chains are
// the shared stencil_dot (mgb_dot.h) in the same order, so results are
// bit-identical to k_stream and to the tile passes (tested).
//
// Reference: v_cycle hierarchy.py:96-111 (with RepeatedSmoother cli.py:365-377),
// apply_stencil grid.py:216-226, inferred_apply smoothers.py:325-343, restrict
// transfer.py:108-121, prolong transfer.py:124-147, history hierarchy.py:129-141.
#include <cstdlib>
#include <utility>
#include <vector>
#include <algorithm>
#include <cstdint>
#include <cmath>

#include "mgb_stream.h"
#include "mgb_dot.h"

#ifdef MGB_CTA_PROF
// experiment builds only: per-CTA (smid, start, end) of the last streaming launch
__device__ unsigned long long g_cta_prof[3 * 8192];
#endif

namespace mgb {
namespace {

#ifndef MGB_S2T
#define MGB_S2T 128
#endif
constexpr int T2 = MGB_S2T;       // widest strip: threads per CTA (column pairs)
#ifndef MGB_S2DIST
#define MGB_S2DIST 5
#endif
#ifndef MGB_S2PDF
#define MGB_S2PDF 16
#endif
constexpr int PD = 8;             // prefetch ring depth (rows) for u (power of two)
constexpr int PDF = MGB_S2PDF;    // ring depth for f: rows t-10 .. t+DIST
constexpr int DIST = MGB_S2DIST;  // prefetch distance (rows ahead)
static_assert(PDF >= 11 + DIST && PD >= DIST + 1, "ring depths");
#ifndef MGB_S2MINB
#define MGB_S2MINB 2
#endif
#ifndef MGB_S2MINB_PRE
#define MGB_S2MINB_PRE 2
#endif
// CTAs per SM the register budget is sized for (3 PRE CTAs fit in shared memory with
// the compact exchange layout, but measured 40 % slower at 168 registers)
constexpr int MINB = MGB_S2MINB, MINB_PRE = MGB_S2MINB_PRE;
// Step loop: per-step variant dispatch, or three phases (boundary steps with dispatch,
// the interior run with one variant, boundary steps) -- measured faster only for the
// V(2,2) POST pass (c2 level 0: 118 -> 114 us; PRE 124 -> 130 us, c4 V(1,1) slower)
#ifndef MGB_S2_PHASED
#define MGB_S2_PHASED 0   // 1: phased V(2,2) POST, 2: three phases everywhere (experiments)
#endif
constexpr int PE = 8;             // ring of coarse rows (POST prolongation), power of two
constexpr int NCLS = 25;
constexpr int CINT = 12;          // interior band class (2 * 5 + 2)

__device__ __forceinline__ int bandc(int i, int n) { return i < 2 ? i : (i >= n - 2 ? 4 - (n - 1 - i) : 2); }

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int NSW, bool RES>
struct SP2 {
  static constexpr int S = 2 * NSW + (RES ? 1 : 0);  // stencil stages after the input field
  static constexpr int H = 2 * NSW + 2;              // column halo per side (even)
};

__host__ __device__ constexpr int m3(int x) { return ((x % 3) + 3) % 3; }

struct Ctx2 {
  Grid g;
  int b, tid, j0, c0, R0, R1;
  int tw, sw, ew, xb;  // threads (column pairs), strip columns, staged coarse columns, and one
                       // exchange buffer: NX fields x (even, odd) column planes, the restriction
                       // field F_S (last) with its even plane only (right neighbours)
  double wI[18];       // CM 1: the problem's interior-class A and M weights (registers)
  bool cin0, cin1, own;
  int cc0, cc1;     // band classes of columns c0, c0 + 1
  double* ring_u;
  double* ring_f;
  double* ring_e;
  double* xch;
  double* rlast;
  const double* tA;
  const double* tK;
  double* uob;
};

// Per-thread pipeline state (push form).  Stage k's output rows are accumulated
// as their input rows arrive: input row x of field k-1 adds the top weights to
// output row x+1 (a fresh chain seeded with f or the old u), the middle weights
// to row x and the bottom weights to row x-1, which completes.  So each output
// chain sees its nine terms in stencil_dot's order (bit-identical results) while a
// step carries 6 S independent three-term chains instead of 2 S nine-term ones,
// and only two open rows per stage (acc, ring of 3 by row mod 3) plus the newest
// own values of each field (cur) stay in registers instead of 3 x 4 windows.
template <int NSW, bool RES>
struct St3 {
  static constexpr int S = 2 * NSW + (RES ? 1 : 0);
  static constexpr int NX = RES ? S + 1 : S;   // exchanged fields (F_S feeds the restriction)
  double acc[S][3][2];    // open output rows of stage k (slot = row mod 3), two columns
  double cur[NX][2];      // own values of field j published at the previous step
  double prev[NSW][2];    // own values of fields 0, 2, .. published two steps back
  double racc;            // open restriction sum (coarse row being accumulated)
  double eA0, eA1;        // POST: coarse correction row t >> 1 at columns m - 1, m (registers:
  double eB0, eB1;        // each coarse row is read from ring_e once), and row (t >> 1) - 1
  double norm;            // history: sum of squares of the input residual
};


// One pipeline step (row t) for the thread's column pair.  PH = t mod 3.
// MODE 0: interior strip, interior rows (constant-bank weights, no tests);
//      1: uniform level, edge strip, interior rows (constant weights, out-of-grid columns zeroed);
//      2: edge strip, interior rows (each column's row-band-2 class weights, columns zeroed);
//      3: anything else (per output row band and column class, rows and columns tested).
template <int NSW, bool RES, bool PRO, bool NORM, bool ZU, int CM, int MODE, int PH>
__device__ __forceinline__ void step3(const StreamArgs& a, const Ctx2& c, const int t, St3<NSW, RES>& st) {
  constexpr bool FAST = MODE < 3;                  // every row the step touches is interior
  constexpr bool CMASK = MODE == 1 || MODE == 2;   // zero out-of-grid columns
  using P = SP2<NSW, RES>;
  constexpr int S = P::S, NX = St3<NSW, RES>::NX;
  const Grid& g = c.g;
  const int slp = (t - 1) & 1;  // exchange slot published by step t - 1
  // ---- neighbours of the rows published by step t - 1 (even / odd column planes)
  double L[NX], R[NX];
  {
    const int iL = max(c.tid - 1, 0), iR = min(c.tid + 1, c.tw - 1);
#pragma unroll
    for (int j = 0; j < NX; ++j) {
      if (ZU && j <= 1) continue;
      const double* xr = &c.xch[slp * c.xb + j * c.sw];
      L[j] = (RES && j == S) ? 0.0 : xr[c.tw + iL];
      R[j] = xr[iR];
    }
    if (ZU) {
      // zero start: field 1 (the first residual f - A 0) is f itself, so stage 2 takes
      // the neighbours of its input row t - 3 straight from the f ring (out-of-grid
      // columns and rows outside the pass's range are zero-filled there, as the
      // computed field would be); fields 0 and 1 are never exchanged
      const double* fr = &c.ring_f[((t - 3) & (PDF - 1)) * c.sw];
      L[0] = R[0] = 0.0;
      L[1] = fr[max(2 * c.tid - 1, 0)];
      R[1] = fr[min(2 * c.tid + 2, c.sw - 1)];
    }
  }
  double out[S + 1][2];
  // ---- stages k = 1..S: push field k-1 row x = t - 2k + 1; completes row t - 2k
#pragma unroll
  for (int k = 1; k <= S; ++k) {
    const bool resid = k & 1;
    const int x = t - 2 * k + 1;
    double v0, v1;
    if (ZU && k == 1) {
      // zero start: f - A 0 = f (the chain fma(-w, 0, f) returns f), row t - 2
      const double2 fv = *reinterpret_cast<const double2*>(&c.ring_f[((t - 2) & (PDF - 1)) * c.sw + 2 * c.tid]);
      v0 = fv.x;
      v1 = fv.y;
    } else {
    const int sN = m3(PH - 2 * k + 2), sM = m3(PH - 2 * k + 1), sB = m3(PH - 2 * k);  // rows x+1, x, x-1
    const double in0 = L[k - 1], in1 = st.cur[k - 1][0], in2 = st.cur[k - 1][1], in3 = R[k - 1];
    // seed of the new chain (row x + 1): f, or the u the update adds to
    double s0, s1;
    if (resid) {
      const double2 fv = *reinterpret_cast<const double2*>(&c.ring_f[((x + 1) & (PDF - 1)) * c.sw + 2 * c.tid]);
      s0 = fv.x;
      s1 = fv.y;
    } else {
      s0 = st.prev[k / 2 - 1][0];
      s1 = st.prev[k / 2 - 1][1];
    }
    const double* wN0;  // weights of rows x+1, x, x-1 for the two columns
    const double* wN1;
    const double* wM0;
    const double* wM1;
    const double* wB0;
    const double* wB1;
    if (MODE <= 1) {
      const double* wi = CM == 2 ? (resid ? a.ci : a.ci + 9) : (resid ? c.wI : c.wI + 9);
      wN0 = wN1 = wM0 = wM1 = wB0 = wB1 = wi;
    } else if (MODE == 2) {
      const double* tab = resid ? c.tA : c.tK;
      wN0 = wM0 = wB0 = tab + (10 + c.cc0) * 9;   // row band 2: nine weights per column
      wN1 = wM1 = wB1 = tab + (10 + c.cc1) * 9;
    } else {
      const double* tab = resid ? c.tA : c.tK;
      const int bN = ((unsigned)(x + 1) < (unsigned)g.rows ? bandc(x + 1, g.rows) : 2) * 5;
      const int bM = ((unsigned)x < (unsigned)g.rows ? bandc(x, g.rows) : 2) * 5;
      const int bB = ((unsigned)(x - 1) < (unsigned)g.rows ? bandc(x - 1, g.rows) : 2) * 5;
      wN0 = tab + (bN + c.cc0) * 9; wN1 = tab + (bN + c.cc1) * 9;
      wM0 = tab + (bM + c.cc0) * 9; wM1 = tab + (bM + c.cc1) * 9;
      wB0 = tab + (bB + c.cc0) * 9; wB1 = tab + (bB + c.cc1) * 9;
    }
    double (&A)[3][2] = st.acc[k - 1];
#define FMS(w_, x_, a_) fma(resid ? -(w_) : (w_), (x_), (a_))
    // bottom terms complete row x - 1
    A[sB][0] = FMS(wB0[6], in0, A[sB][0]);
    A[sB][1] = FMS(wB1[6], in1, A[sB][1]);
    A[sM][0] = FMS(wM0[3], in0, A[sM][0]);
    A[sM][1] = FMS(wM1[3], in1, A[sM][1]);
    s0 = FMS(wN0[0], in0, s0);
    s1 = FMS(wN1[0], in1, s1);
    A[sB][0] = FMS(wB0[7], in1, A[sB][0]);
    A[sB][1] = FMS(wB1[7], in2, A[sB][1]);
    A[sM][0] = FMS(wM0[4], in1, A[sM][0]);
    A[sM][1] = FMS(wM1[4], in2, A[sM][1]);
    s0 = FMS(wN0[1], in1, s0);
    s1 = FMS(wN1[1], in2, s1);
    A[sB][0] = FMS(wB0[8], in2, A[sB][0]);
    A[sB][1] = FMS(wB1[8], in3, A[sB][1]);
    A[sM][0] = FMS(wM0[5], in2, A[sM][0]);
    A[sM][1] = FMS(wM1[5], in3, A[sM][1]);
    s0 = FMS(wN0[2], in2, s0);
    s1 = FMS(wN1[2], in3, s1);
#undef FMS
    v0 = A[sB][0];
    v1 = A[sB][1];
    A[sN][0] = s0;   // slot of row x + 1 (was row x - 2, long complete)
    A[sN][1] = s1;
    }
    const int row = x - 1;  // = t - 2k
    if (!FAST) {
      const bool rv = (unsigned)row < (unsigned)g.rows;
      v0 = rv && c.cin0 ? v0 : 0.0;
      v1 = rv && c.cin1 ? v1 : 0.0;
    } else if (CMASK) {
      v0 = c.cin0 ? v0 : 0.0;
      v1 = c.cin1 ? v1 : 0.0;
    }
    const bool orow = c.own && row >= c.R0 && row < c.R1;
    if (NORM && k == 1 && orow) {
      st.norm = fma(v0, v0, st.norm);   // out-of-grid columns hold 0
      st.norm = fma(v1, v1, st.norm);
    }
    if (k == 2 * NSW && orow && a.uo) {
      double* dst = c.uob + (int64_t)row * g.cols + c.c0;
      dst[0] = v0;                                   // owned pairs start in the grid
      if ((FAST && !CMASK) || c.cin1) dst[1] = v1;
    }
    out[k][0] = v0;
    out[k][1] = v1;
  }
  // ---- restriction: push field S row y = t - 1 - 2S (columns c0, c0+1, c0+2)
  if (RES) {
    const int y = t - 1 - 2 * S;
    const double x0 = st.cur[S][0], x1 = st.cur[S][1], x2 = R[S];
    if (y & 1) {
      st.racc = fma(0.125, x0, st.racc);
      st.racc = fma(0.25, x1, st.racc);
      st.racc = fma(0.125, x2, st.racc);
    } else {
      // bottom row of coarse row ci = y/2 - 1 (completes), top row of coarse row y/2
      double s = fma(0.0625, x0, st.racc);
      s = fma(0.125, x1, s);
      s = fma(0.0625, x2, s);
      const int ci = (y - 2) >> 1;
      const int rows_c = g.rows / 2, cols_c = g.cols / 2;
      const int cj = c.c0 >> 1;
      if (c.own && y >= 2 && ci >= (c.R0 >> 1) && 2 * ci + 1 < c.R1 && ci < rows_c && cj < cols_c) {
        const int64_t pc = (int64_t)ci * cols_c + cj;
        const bool actc = a.mask_c == nullptr || a.mask_c[pc];
        a.rc[c.b * (int64_t)rows_c * cols_c + pc] = actc ? s : 0.0;
      }
      double r = 0.0625 * x0;
      r = fma(0.125, x1, r);
      st.racc = fma(0.0625, x2, r);
    }
  }
  // ---- F_0 = u (+ P ec) at row t
  {
    double u0 = 0.0, u1 = 0.0;
    const bool rvr = FAST || (unsigned)t < (unsigned)g.rows;
    if (!ZU) {
      const double2 v = *reinterpret_cast<const double2*>(&c.ring_u[(t & (PD - 1)) * c.sw + 2 * c.tid]);
      u0 = v.x;
      u1 = v.y;
    }
    if (PRO && !(t & 1)) {
      // coarse row t/2 enters (staged in ring_e, entry q = coarse column cjb + q; read
      // once, kept in registers for fine rows t, t + 1, t + 2); row t/2 - 1 moves down
      st.eB0 = st.eA0;
      st.eB1 = st.eA1;
      const double* ea = c.ring_e + ((t >> 1) & (PE - 1)) * c.ew;
      st.eA0 = ea[c.tid];
      st.eA1 = ea[c.tid + 1];
    }
    if (PRO && rvr) {
      // u += P ec; the k_stream loop order: di = -1, 0, 1 (row parity), dj = -1, 0, 1
      // (column parity)
      double p0 = 0.0, p1 = 0.0;
      if (t & 1) {
        p0 = fma(0.25, st.eA1, p0);   // (di 0, dj -1): coarse row (t - 1)/2, column m
        p0 = fma(0.25, st.eA0, p0);   // (di 0, dj +1): column m - 1
        p1 = fma(0.5, st.eA1, p1);    // (di 0, dj 0)
      } else {
        p0 = fma(0.125, st.eA1, p0);  // di = -1: coarse row t/2
        p0 = fma(0.125, st.eA0, p0);
        p1 = fma(0.25, st.eA1, p1);
        p0 = fma(0.125, st.eB1, p0);  // di = +1: coarse row t/2 - 1
        p0 = fma(0.125, st.eB0, p0);
        p1 = fma(0.25, st.eB1, p1);
      }
      u0 += p0;
      u1 += p1;
    }
    // (the prolongation can reach one column past the grid: zero it there too)
    const bool m0 = FAST ? (!CMASK || c.cin0) : (rvr && c.cin0);
    const bool m1 = FAST ? (!CMASK || c.cin1) : (rvr && c.cin1);
    out[0][0] = m0 ? u0 : 0.0;
    out[0][1] = m1 ? u1 : 0.0;
  }
  // ---- publish this step's rows (field j: row t - 2j), shift the own-value history
  const int sl = t & 1;
#pragma unroll
  for (int j = 0; j < NX; ++j) {
    if (ZU && j <= 1) continue;
    c.xch[sl * c.xb + j * c.sw + c.tid] = out[j][0];
    if (!(RES && j == S)) c.xch[sl * c.xb + j * c.sw + c.tw + c.tid] = out[j][1];
  }
#pragma unroll
  for (int m = 0; m < NSW; ++m) {
    st.prev[m][0] = st.cur[2 * m][0];
    st.prev[m][1] = st.cur[2 * m][1];
  }
#pragma unroll
  for (int j = 0; j < NX; ++j) {
    st.cur[j][0] = out[j][0];
    st.cur[j][1] = out[j][1];
  }
  __syncthreads();
}

// CM: 1 = band-class tables in shared memory, the interior class copied to registers
// (batched levels: one problem per CTA); 2 = the interior class read from the kernel
// parameters (constant-bank operands; single problem).
template <int NSW, bool RES, bool PRO, bool NORM, bool ZU, int CM>
__global__ void __launch_bounds__(T2, RES ? MINB_PRE : MINB) k_stream2(StreamArgs a) {
  pdl_trigger();
  using P = SP2<NSW, RES>;
  constexpr int S = P::S, H = P::H;
  extern __shared__ __align__(16) double smem2[];
  Ctx2 c;
  c.g = a.g;
  const Grid& g = c.g;
  // strip width: 128 column pairs for single problems (compile-time strides), batched
  // levels blockDim.x (the launcher picks 64, 96 or 128 for the problems' width)
  c.tw = CM == 2 ? T2 : (int)blockDim.x;
  c.sw = 2 * c.tw;
  c.ew = c.tw + 2;
  c.xb = St3<NSW, RES>::NX * c.sw - (RES ? c.tw : 0);
  const int WOUT = c.sw - 2 * H;                  // owned columns per strip (even)
  c.ring_u = smem2;                               // PD x sw (unused when ZU)
  c.ring_f = c.ring_u + PD * c.sw;                // PDF x sw
  c.xch = c.ring_f + PDF * c.sw;                  // 2 buffers x NX fields x (even, odd) planes
  c.ring_e = c.xch + 2 * c.xb;                    // PE x ew (POST)
  double* tA = c.ring_e + (PRO ? PE * c.ew : 0);  // 25 x 9
  double* tK = tA + NCLS * 9;                     // 25 x 9
  double* red = tK + NCLS * 9;                    // 32
  c.tA = tA;
  c.tK = tK;
  c.tid = threadIdx.x;
  c.b = blockIdx.z;
  const int64_t n = g.n();
  // CTA -> (strip, row segment): the edge strips' CTAs first, then the interior ones
  int strip, seg, seg1, srem, sy, nsegs;
  {
    const int id = blockIdx.x;
    const int ne = a.nedge;
    if (id < ne * a.nseg_edge) {
      strip = (id % ne == 0) ? 0 : a.nstrips - 1;
      sy = id / ne;
      seg = a.seg_edge;
      seg1 = a.seg_edge_first;
      srem = a.seg_edge_rem;
      nsegs = a.nseg_edge;
    } else {
      const int q = id - ne * a.nseg_edge, ni = a.nstrips - ne;
      strip = 1 + q % ni;
      sy = q / ni;
      seg = a.seg;
      seg1 = a.seg_first;
      srem = a.seg_rem;
      nsegs = a.nseg;
    }
  }
  c.j0 = strip * WOUT;                            // first owned column (even)
  c.c0 = c.j0 - H + 2 * c.tid;                    // the thread's pair (even column)
  c.cin0 = c.c0 >= 0 && c.c0 < g.cols;
  c.cin1 = c.c0 + 1 >= 0 && c.c0 + 1 < g.cols;
  c.own = 2 * c.tid >= H && 2 * c.tid < H + WOUT && c.cin0;
  c.cc0 = c.cin0 ? bandc(c.c0, g.cols) : 2;       // out-of-grid columns are zeroed anyway
  c.cc1 = c.cin1 ? bandc(c.c0 + 1, g.cols) : 2;
  c.R0 = a.own0 + (sy == 0 ? 0 : seg1 + (sy - 1) * seg + min(sy - 1, srem));
  const int rend = a.own1 > 0 ? a.own1 : g.rows;  // the last segment takes the rest
  c.R1 = sy == nsegs - 1 ? rend : min(rend, c.R0 + (sy == 0 ? seg1 : seg + (sy - 1 < srem ? 1 : 0)));
  const double* fb = a.f + c.b * n;
  const double* ub = ZU ? nullptr : a.u + c.b * n;
  c.uob = a.uo + c.b * n;
  // fast steps: every CTA column interior (band class 2) and in the grid, or a level
  // whose band classes are all equal (then only out-of-grid columns need zeroing)
  const bool cta_int = c.j0 - H >= 2 && c.j0 - H + c.sw - 1 <= g.cols - 3;
  const bool cta_fast = cta_int || a.uniform == 1;
#ifdef MGB_CTA_PROF
  unsigned long long prof_t0 = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prof_t0));
#endif

  for (int q = c.tid; q < NCLS * 9; q += c.tw) {
    tA[q] = a.A.cls[(int64_t)c.b * NCLS * 9 + q];
    tK[q] = a.K.cls[(int64_t)c.b * NCLS * 9 + q];
  }
  __syncthreads();
  if (CM == 1) {
    // batched levels: this problem's interior weights live in registers for the pass
#pragma unroll
    for (int o = 0; o < 9; ++o) {
      c.wI[o] = tA[CINT * 9 + o];
      c.wI[9 + o] = tK[CINT * 9 + o];
    }
  }

  St3<NSW, RES> st;
#pragma unroll
  for (int k = 0; k < S; ++k)
#pragma unroll
    for (int r = 0; r < 3; ++r) st.acc[k][r][0] = st.acc[k][r][1] = 0.0;
#pragma unroll
  for (int j = 0; j < St3<NSW, RES>::NX; ++j) st.cur[j][0] = st.cur[j][1] = 0.0;
#pragma unroll
  for (int m = 0; m < NSW; ++m) st.prev[m][0] = st.prev[m][1] = 0.0;
  st.racc = 0.0;
  st.norm = 0.0;
  st.eA0 = st.eA1 = st.eB0 = st.eB1 = 0.0;
  // the first step reads the exchange slot of step t0 - 1: start it at zero
  for (int q = c.tid; q < 2 * c.xb; q += c.tw) c.xch[q] = 0.0;
  pdl_wait();  // u, f, ec come from the preceding kernels; uo / rc may still be read there

  int t0 = c.R0 - S - 1;
  t0 -= m3(t0);
  // the restriction pushes field S row t - 1 - 2S: its last row R1 at step R1 + 2S + 1
  const int t1 = c.R1 + 2 * S + (RES ? 1 : 0);
  int prow = t0;
  const int64_t cstride = g.cols;
  // prefetch: thread copies strip columns tid and tid + tw (coalesced rows)
  const int ca = c.j0 - H + c.tid, cb = ca + c.tw;
  const bool ina = ca >= 0 && ca < g.cols, inb = cb >= 0 && cb < g.cols;
  const double* pu = ZU ? nullptr : ub + (int64_t)prow * cstride + ca;
  const double* pf = fb + (int64_t)prow * cstride + ca;
  const int rows_c = g.rows / 2, cols_c = g.cols / 2;
  const double* ecb = PRO ? a.ec + c.b * (int64_t)rows_c * cols_c : nullptr;
  const int cjb = ((c.j0 - H) >> 1) - 1;          // coarse column of ring_e entry 0
  const int lo_row = max(0, c.R0 - S - 1), hi_row = min(g.rows - 1, c.R1 + S);
  const int lo_c = (lo_row - 2) >> 1, hi_c = (hi_row >> 1) + 1;
  auto stage_e = [&](int ci) {
    for (int q = c.tid; q < c.ew; q += c.tw) {
      const int cj = cjb + q;
      const bool ev = ci >= 0 && ci < rows_c && ci >= lo_c && ci <= hi_c && cj >= 0 && cj < cols_c;
      cp_async8(&c.ring_e[(ci & (PE - 1)) * c.ew + q], ev ? ecb + (int64_t)ci * cols_c + cj : ecb, ev);
    }
  };
  auto issue = [&]() {
    const bool rv = prow >= lo_row && prow <= hi_row;
    double* du = &c.ring_u[(prow & (PD - 1)) * c.sw + c.tid];
    double* df = &c.ring_f[(prow & (PDF - 1)) * c.sw + c.tid];
    // (a zero-size copy reads nothing: the row pointer is passed unselected)
    if (!ZU) {
      cp_async8(du, pu, rv && ina);
      cp_async8(du + c.tw, pu + c.tw, rv && inb);
    }
    cp_async8(df, pf, rv && ina);
    cp_async8(df + c.tw, pf + c.tw, rv && inb);
    // coarse row ci is first needed by fine row 2ci (as di = -1); staged with the
    // group of fine row 2ci - 2 so it is complete and published by that step's barrier
    if (PRO && !(prow & 1)) stage_e((prow >> 1) + 1);
    cp_commit();
    ++prow;
    if (!ZU) pu += cstride;
    pf += cstride;
  };
  if (PRO) {
    for (int ci = (t0 >> 1) - 1; ci <= (t0 >> 1) + 1; ++ci) stage_e(ci);
    cp_commit();
    cp_wait<0>();
    __syncthreads();
    // the register copy of coarse row (t0 - 1) >> 1, as if step t0 - 1 had run
    const double* ea = c.ring_e + (((t0 - 1) >> 1) & (PE - 1)) * c.ew;
    st.eA0 = ea[c.tid];
    st.eA1 = ea[c.tid + 1];
  }
  for (int q = 0; q < DIST; ++q) issue();
  // ring rows are copied by other threads than the ones reading the pair: row t
  // must be complete before the barrier of step t - 1 (row t0: this one)
  cp_wait<DIST - 1>();
  __syncthreads();

#define MGB_STEP2(PH_)                                                                     \
  {                                                                                        \
    const int t = tb + PH_;                                                                \
    issue();                                                                               \
    cp_wait<DIST - 1>(); /* row t + 1 lands before this step's barrier publishes it */     \
    const bool rows_int = t - 2 * S >= 2 && t <= g.rows - 3;                               \
    if (rows_int && cta_int)                                                               \
      step3<NSW, RES, PRO, NORM, ZU, CM, 0, PH_>(a, c, t, st);                             \
    else if (rows_int && cta_fast)                                                         \
      step3<NSW, RES, PRO, NORM, ZU, CM, 1, PH_>(a, c, t, st);                             \
    else if (rows_int)                                                                     \
      step3<NSW, RES, PRO, NORM, ZU, CM, 2, PH_>(a, c, t, st);                             \
    else                                                                                   \
      step3<NSW, RES, PRO, NORM, ZU, CM, 3, PH_>(a, c, t, st);                             \
  }
#define MGB_STEP2F(MODE_, PH_)                                                             \
  {                                                                                        \
    const int t = tb + PH_;                                                                \
    issue();                                                                               \
    cp_wait<DIST - 1>();                                                                   \
    step3<NSW, RES, PRO, NORM, ZU, CM, MODE_, PH_>(a, c, t, st);                           \
  }
  // three phases: the leading boundary steps (general dispatch), the run of interior
  // steps (one step variant, no per-step dispatch), the trailing ones
  int tb = t0;
  const int fa = 2 * S + 2, fz = min(t1, g.rows - 3);  // interior steps: rows_int
  constexpr bool phased = MGB_S2_PHASED == 2 || (MGB_S2_PHASED == 1 && PRO && NSW == 2);
  if (phased && cta_fast) {
    for (; tb <= t1 && tb < fa; tb += 3) {
      MGB_STEP2(0)
      MGB_STEP2(1)
      MGB_STEP2(2)
    }
    if (cta_int) {
      for (; tb + 2 <= fz; tb += 3) {
        MGB_STEP2F(0, 0)
        MGB_STEP2F(0, 1)
        MGB_STEP2F(0, 2)
      }
    } else {
      for (; tb + 2 <= fz; tb += 3) {
        MGB_STEP2F(1, 0)
        MGB_STEP2F(1, 1)
        MGB_STEP2F(1, 2)
      }
    }
  }
  for (; tb <= t1; tb += 3) {
    MGB_STEP2(0)
    MGB_STEP2(1)
    MGB_STEP2(2)
  }
#undef MGB_STEP2F
#undef MGB_STEP2
  cp_wait<0>();
#ifdef MGB_CTA_PROF
  if (c.tid == 0 && blockIdx.x < 8192) {
    unsigned long long t1, sm;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    sm = smid;
    g_cta_prof[3 * blockIdx.x] = sm;
    g_cta_prof[3 * blockIdx.x + 1] = prof_t0;
    g_cta_prof[3 * blockIdx.x + 2] = t1;
  }
#endif
  if (NORM) {
    double v = st.norm;
    const int lane = c.tid & 31, wid = c.tid >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[wid] = v;
    __syncthreads();
    if (c.tid == 0) {
      double s = 0.0;
      for (int q = 0; q < (c.tw + 31) / 32; ++q) s += red[q];
      a.partials[(int64_t)c.b * gridDim.x + blockIdx.x] = s;
    }
  }
}

}  // namespace

static size_t stream2_smem(int nsw, bool res, bool pro, int tw) {
  const int nx = 2 * nsw + (res ? 2 : 0);
  const int sw = 2 * tw, xb = nx * sw - (res ? tw : 0);
  return sizeof(double) * ((size_t)(PD + PDF) * sw + 2 * xb + (pro ? PE * (tw + 2) : 0) + 2 * NCLS * 9 + 32);
}

// Strip width (threads = column pairs per CTA, a multiple of 32 up to 128) for
// batched levels: 64 pairs (more CTAs per SM: measured 21 % faster than 96 on
// config 4's 511-wide problems) unless that pads the width 15 % more than the
// tightest choice.
static int choose_tw(int cols, int nsw) {
  static const int tw_env = getenv("MGB_S2TW") ? atoi(getenv("MGB_S2TW")) : 0;  // experiments only
  if (tw_env > 0) return tw_env;
  const int H = 2 * nsw + 2;
  int best = T2;
  int64_t best_w = INT64_MAX;
  for (int tw = T2; tw >= 64; tw -= 32) {
    const int wout = 2 * tw - 2 * H;
    const int64_t padded = (int64_t)((cols + wout - 1) / wout) * 2 * tw;
    if (padded < best_w) {
      best_w = padded;
      best = tw;
    }
  }
  const int w64 = 2 * 64 - 2 * H;
  const int64_t pad64 = (int64_t)((cols + w64 - 1) / w64) * 128;
  return pad64 * 100 <= best_w * 115 ? 64 : best;
}

static int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// Rows per CTA segment.  Interior strips get segments of seg rows, the edge strips
// (boundary columns: every step takes a class-lookup variant, r times the cost of
// an interior step) segments of about seg / r rows, and the first / last segment on
// the grid's top / bottom edge is shorter by the extra cost of its boundary-row
// steps, so that all CTAs finish together (per-CTA %globaltimer probes); the
// segment counts fill whole waves of the measured occupancy with the fewest
// pipeline fills (3S + 3 steps per segment).
struct SegPlan {
  int seg, first, rem, n;
};
// n segments over R rows: first = seg - dt, middle seg (the first rem of them seg + 1),
// last = the rest (~ seg - db)
static SegPlan seg_plan(int R, int n, int dt, int db) {
  SegPlan p;
  p.n = std::max(1, std::min(n, R));
  if (p.n == 1) {
    p.seg = p.first = R;
    p.rem = 0;
    return p;
  }
  p.seg = std::max(1, (R + dt + db) / p.n);
  p.first = std::max(1, std::min(R - (p.n - 1), p.seg - dt));
  const int64_t mid = (int64_t)(p.n - 2) * p.seg;
  const int64_t last = R - p.first - mid;       // before spreading the remainder
  const int64_t want = std::max(1, p.seg - db);
  p.rem = (int)std::max<int64_t>(0, std::min<int64_t>(p.n - 2, last - want));
  if (R - p.first - mid - p.rem < 1) {           // degenerate: fall back to equal segments
    p.seg = (R + p.n - 1) / p.n;
    p.first = p.seg;
    p.rem = 0;
    while (p.n > 1 && (int64_t)(p.n - 1) * p.seg >= R) --p.n;
  }
  return p;
}

static void choose_seg2(const Grid& g, int nsw, bool res, int occ, int tw, bool uniform, bool top, bool bot,
                        StreamArgs& a) {
  const int H = 2 * nsw + 2, wout = 2 * tw - 2 * H, S = 2 * nsw + (res ? 1 : 0);
  const int strips = (g.cols + wout - 1) / wout;
  const int ne = std::min(strips, 2), ni = strips - ne;
  const int64_t slots = (int64_t)sm_count() * std::max(occ, 1);
  static const double r_env = getenv("MGB_EDGE_RATIO") ? atof(getenv("MGB_EDGE_RATIO")) : 0.0;
  // measured (k_stream2, 4095^2 / 2047^2, per-CTA timers): uniform edge strips ~1.05x,
  // class-weight edge steps ~1.3x, boundary-row steps ~2.2x an interior step
  const double r = ni == 0 ? 1.0 : (r_env > 0.0 ? r_env : (uniform ? 1.05 : 1.3));
  const int F = 3 * S + 3;
  const int dtrim = (int)(1.2 * (2 * S + 2));
  const int dt = top ? dtrim : 0, db = bot ? dtrim : 0;
  double best_t = 1e300;
  a.nstrips = strips;
  a.nedge = ne;
  for (int nseg = 1; nseg <= std::max(1, g.rows / 16); ++nseg) {
    const SegPlan pi = seg_plan(g.rows, nseg, dt, db);
    const int seg_e_target = std::max(8, (int)((pi.seg + F) / r) - F);
    const SegPlan pe = seg_plan(g.rows, (g.rows + dt + db + seg_e_target - 1) / seg_e_target, dt, db);
    const int64_t ctas = ((int64_t)(ni > 0 ? ni : 0) * pi.n + (int64_t)ne * pe.n) * g.batch;
    // one or two waves: a partial wave costs a full CTA time; beyond, CTAs start as
    // others finish and the tail is half a CTA time on average
    const double w = (double)ctas / slots;
    const double waves = w <= 2.0 ? std::ceil(w) : w + 0.5;
    const double t = waves * std::max((double)(pi.seg + F), r * (pe.seg + F));
    if (t < best_t) {
      best_t = t;
      a.seg = pi.seg;
      a.seg_first = pi.first;
      a.seg_rem = pi.rem;
      a.nseg = pi.n;
      a.seg_edge = pe.seg;
      a.seg_edge_first = pe.first;
      a.seg_edge_rem = pe.rem;
      a.nseg_edge = pe.n;
    }
  }
  static const int force_seg = getenv("MGB_SEG") ? atoi(getenv("MGB_SEG")) : 0;  // experiments only
  if (force_seg > 0) {
    const SegPlan p = seg_plan(g.rows, (g.rows + force_seg - 1) / force_seg, 0, 0);
    a.seg = a.seg_edge = p.seg;
    a.seg_first = a.seg_edge_first = p.first;
    a.seg_rem = a.seg_edge_rem = p.rem;
    a.nseg = a.nseg_edge = p.n;
  }
}

template <typename KF>
static cudaError_t run_k2(KF kern, int nsw, bool res, bool pro, StreamArgs a, int* nblocks) {
  struct Occ {
    const void* k;
    int dev, tw, occ;
  };
  // the >48 KB shared-memory attribute and the occupancy are per device
  static thread_local std::vector<Occ> occ_cache;
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  const int tw = a.ci_valid ? T2 : choose_tw(a.g.cols, nsw);  // CM 2 kernels assume T2
  const size_t smem = stream2_smem(nsw, res, pro, tw);
  int occ = -1;
  for (auto& e : occ_cache)
    if (e.k == (const void*)kern && e.dev == dev && e.tw == tw) occ = e.occ;
  if (occ < 0) {
    // the attribute is sized for the widest strip once per kernel
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)stream2_smem(nsw, res, pro, T2));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, tw, smem);
    if (e != cudaSuccess) return e;
    occ_cache.push_back({(const void*)kern, dev, tw, occ});
  }
  if (a.own1 <= 0) {
    a.own0 = 0;
    a.own1 = a.g.rows;
  }
  Grid go = a.g;
  go.rows = a.own1 - a.own0;
  choose_seg2(go, nsw, res, occ, tw, a.uniform == 1, a.own0 == 0, a.own1 == a.g.rows, a);
  const int ni = a.nstrips - a.nedge;
  const int nctas = a.nedge * a.nseg_edge + ni * a.nseg;
  const dim3 grid(nctas, 1, a.g.batch);
  if (nblocks) *nblocks = nctas;
  const cudaError_t e = launch_pdl(kern, grid, dim3(tw), smem, a.stream, a);
  if (e != cudaSuccess) return e;
  return MGB_DBG(__func__);
}

cudaError_t launch_stream2(const StreamArgs& a, int nsw, bool res, bool pro, bool norm, int* nblocks) {
  const bool zu = a.u == nullptr;
  const int cm = a.ci_valid ? 2 : 1;
#define MGB_ST2(NSW_, RES_, PRO_, NORM_, ZU_)                                                     \
  if (nsw == NSW_ && res == RES_ && pro == PRO_ && norm == NORM_ && zu == ZU_) {                \
    if (cm == 2) return run_k2(k_stream2<NSW_, RES_, PRO_, NORM_, ZU_, 2>, nsw, res, pro, a, nblocks); \
    return run_k2(k_stream2<NSW_, RES_, PRO_, NORM_, ZU_, 1>, nsw, res, pro, a, nblocks);             \
  }
  MGB_ST2(1, true, false, false, false) MGB_ST2(1, true, false, true, false)
  MGB_ST2(1, true, false, false, true)  MGB_ST2(1, true, false, true, true)
  MGB_ST2(2, true, false, false, false) MGB_ST2(2, true, false, true, false)
  MGB_ST2(2, true, false, false, true)  MGB_ST2(2, true, false, true, true)
  MGB_ST2(1, false, false, false, false) MGB_ST2(1, false, false, true, false)
  MGB_ST2(1, false, false, false, true)  MGB_ST2(1, false, false, true, true)
  MGB_ST2(1, false, true, false, false) MGB_ST2(2, false, true, false, false)
#undef MGB_ST2
  return cudaErrorInvalidValue;
}

}  // namespace mgb

#ifdef MGB_CTA_PROF
extern "C" __attribute__((visibility("default"))) int mgb_debug_cta_prof(unsigned long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, g_cta_prof, sizeof(unsigned long long) * 3 * n);
}
#endif
