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
#include "mgb_stream.h"

namespace mgb {
namespace {

constexpr int SWC = 128;   // columns (incl. halo) per CTA
constexpr int CPT = 2;     // columns per thread
constexpr int SWT = SWC / CPT;  // threads per CTA
constexpr int PD = 8;      // prefetch ring depth (rows) for u (power of two)
constexpr int PDF = 16;    // ring depth for f (rows t-10 .. t+DIST; power of two)
constexpr int DIST = 5;    // prefetch distance (rows ahead)
constexpr int MINB = 5;    // CTAs per SM the register budget is sized for
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

template <int NSW, bool RES, bool PRO>
struct SP {
  static constexpr int S = 2 * NSW + (RES ? 1 : 0);  // stencil stages after the input field
  static constexpr int H = 2 * NSW + 2;              // column halo per side (even)
  static constexpr int WOUT = SWC - 2 * H;           // owned columns per strip (even)
  static constexpr int NF = S;                       // fields with a window (F_0 .. F_{S-1})
};

// compile-time positive modulo 3
__host__ __device__ constexpr int m3(int x) { return ((x % 3) + 3) % 3; }

// 3x3 dot product of weights with window columns c0..c0+2 of rows s0, s1, s2,
// three independent accumulation chains, the first seeded with `init`:
//   returns init + sgn * sum(w * x)
template <bool NEG>
__device__ __forceinline__ double dot9(const double* wt, const double (&x)[3][4], int s0, int s1, int s2, int c0,
                                       double init) {
  double a0 = NEG ? fma(-wt[0], x[s0][c0], init) : fma(wt[0], x[s0][c0], init);
  double a1 = wt[3] * x[s1][c0];
  double a2 = wt[6] * x[s2][c0];
  a0 = fma(wt[1], x[s0][c0 + 1], NEG ? -a0 : a0);
  a1 = fma(wt[4], x[s1][c0 + 1], a1);
  a2 = fma(wt[7], x[s2][c0 + 1], a2);
  a0 = fma(wt[2], x[s0][c0 + 2], a0);
  a1 = fma(wt[5], x[s1][c0 + 2], a1);
  a2 = fma(wt[8], x[s2][c0 + 2], a2);
  const double t = (a0 + a1) + a2;
  return NEG ? -t : t;
}

// Per-CTA constants of a streaming pass.
struct Ctx {
  Grid g;
  int b, tid, j0, R0, R1;
  int col[CPT];
  bool cin[CPT], owned_c[CPT];
  int ccls[CPT];
  int lL, lR;   // exchange-row indices of the left / right neighbour columns
  const double* fb;
  const double* ub;
  double* uob;
  double* ring_u;
  double* ring_f;
  double* xch;
  double* rlast;
  const double* tA;
  const double* tK;
  const uint8_t* mk;
};

// One pipeline step (row t).  FAST: every row the step touches is an interior
// row and every column of the CTA an interior in-grid column, so no bounds,
// band-class or column tests are needed.  PH = t mod 3 (window slots).
template <int NSW, bool RES, bool PRO, bool NORM, bool ZU, int CM, bool MSK, bool FAST, int PH>
__device__ __forceinline__ void stream_step(const StreamArgs& a, const Ctx& c, const int t,
                                            double (&w)[SP<NSW, RES, PRO>::NF][3][4],
                                            double (&hold)[NSW][CPT], double& acc) {
  using P = SP<NSW, RES, PRO>;
  constexpr int S = P::S, H = P::H, WOUT = P::WOUT, NF = P::NF;
  constexpr bool CL = CM != 0;
  const Grid& g = c.g;
  double nv[NF + 1][CPT];
  const int tc = CPT * c.tid;  // first exchange column of this thread
  // ---- F_0 = u (+ P ec) at row t
#pragma unroll
  for (int q = 0; q < CPT; ++q) {
    double u0 = 0.0;
    const bool rv = FAST || ((unsigned)t < (unsigned)g.rows && c.cin[q]);
    if (!ZU) u0 = c.ring_u[(t & (PD - 1)) * SWC + tc + q];
    if (PRO && rv) {
      const int rc_ = g.rows / 2, cc_ = g.cols / 2;
      const double* eb = a.ec + c.b * (int64_t)rc_ * cc_;
      double s = 0.0;
#pragma unroll
      for (int di = -1; di <= 1; ++di) {
        const int tt = t - 1 - di;
        if ((tt & 1) || (!FAST && (tt < 0 || (tt >> 1) >= rc_))) continue;
        const double* er = eb + (int64_t)(tt >> 1) * cc_;
#pragma unroll
        for (int dj = -1; dj <= 1; ++dj) {
          const int uu = c.col[q] - 1 - dj;
          if ((uu & 1) || (!FAST && (uu < 0 || (uu >> 1) >= cc_))) continue;
          const double wgt = (di == 0 ? 2.0 : 1.0) * (dj == 0 ? 2.0 : 1.0) * 0.125;
          s = fma(wgt, __ldg(er + (uu >> 1)), s);
        }
      }
      u0 += s;
    }
    if (MSK && rv && !c.mk[(int64_t)t * g.cols + c.col[q]]) u0 = 0.0;
    nv[0][q] = (FAST || rv) ? u0 : 0.0;
  }
  // ---- stages k = 1..S at row t - 2k (rows are CTA-uniform)
#pragma unroll
  for (int k = 1; k <= S; ++k) {
    const int row = t - 2 * k;
    const int s0 = m3(PH - 2 * k - 1), s1 = m3(PH - 2 * k), s2 = m3(PH - 2 * k + 1);
    const bool rowv = FAST || (unsigned)row < (unsigned)g.rows;
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      double val = 0.0;
      if (rowv) {
        const Op& op = (k & 1) ? a.A : a.K;
        const double init = (k & 1) ? c.ring_f[(row & (PDF - 1)) * SWC + tc + q] : hold[k / 2 - 1][q];
        if (!CL) {
          const double* base = op.planes + (int64_t)c.b * 9 * op.n +
                               ((int64_t)row * g.cols + (c.cin[q] ? c.col[q] : 0));
          double wt[9];
#pragma unroll
          for (int o = 0; o < 9; ++o) wt[o] = __ldg(base + (int64_t)o * op.n);
          val = (k & 1) ? dot9<true>(wt, w[k - 1], s0, s1, s2, q, init) : dot9<false>(wt, w[k - 1], s0, s1, s2, q, init);
        } else {
          const double* wt = FAST ? (CM == 2 ? ((k & 1) ? a.ci : a.ci + 9) : (((k & 1) ? c.tA : c.tK) + CINT * 9))
                                  : (((k & 1) ? c.tA : c.tK) + (bandc(row, g.rows) * 5 + c.ccls[q]) * 9);
          val = (k & 1) ? dot9<true>(wt, w[k - 1], s0, s1, s2, q, init) : dot9<false>(wt, w[k - 1], s0, s1, s2, q, init);
        }
        if (MSK && c.cin[q] && !c.mk[(int64_t)row * g.cols + c.col[q]]) val = 0.0;
        if (!FAST) val = c.cin[q] ? val : 0.0;
        if (NORM && k == 1 && c.owned_c[q] && row >= c.R0 && row < c.R1) acc = fma(val, val, acc);
        if (k == 2 * NSW && c.owned_c[q] && row >= c.R0 && row < c.R1)
          c.uob[(int64_t)row * g.cols + c.col[q]] = val;
      }
      nv[k][q] = val;
    }
  }
  // ---- publish (one 16-byte store per field), then slide the windows
  const int sl = t & 1;
#pragma unroll
  for (int k = 0; k < NF; ++k)
    *reinterpret_cast<double2*>(&c.xch[(k * 2 + sl) * SWC + tc]) = make_double2(nv[k][0], nv[k][1]);
  if (RES) *reinterpret_cast<double2*>(&c.rlast[((t - 2 * S) & 3) * SWC + tc]) = make_double2(nv[S][0], nv[S][1]);
  __syncthreads();
  if (RES) {
    const int top = t - 2 * S;
    if (top >= 2 && !(top & 1)) {
      const int ci = (top - 2) >> 1;
      const int rows_c = g.rows / 2, cols_c = g.cols / 2;
      const int cj = (c.j0 >> 1) + c.tid;
      if (c.tid < WOUT / 2 && ci >= (c.R0 >> 1) && 2 * ci + 1 < c.R1 && ci < rows_c && cj < cols_c) {
        const int base = H + 2 * c.tid;
        const double* r0p = &c.rlast[((top - 2) & 3) * SWC + base];
        const double* r1p = &c.rlast[((top - 1) & 3) * SWC + base];
        const double* r2p = &c.rlast[(top & 3) * SWC + base];
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
    if (!(k & 1) && k / 2 < NSW) {
      hold[k / 2][0] = w[k][sn][1];
      hold[k / 2][1] = w[k][sn][2];
    }
    w[k][sn][0] = c.xch[(k * 2 + sl) * SWC + c.lL];
    w[k][sn][1] = nv[k][0];
    w[k][sn][2] = nv[k][1];
    w[k][sn][3] = c.xch[(k * 2 + sl) * SWC + c.lR];
  }
}

// CM: 0 = per-point planes for A and M; 1 = band-class tables in shared memory;
// 2 = band-class tables with the interior class read from the kernel parameters
// (constant-bank operands: no registers, no shared-memory traffic).
template <int NSW, bool RES, bool PRO, bool NORM, bool ZU, int CM, bool MSK>
__global__ void __launch_bounds__(SWT, MINB) k_stream(StreamArgs a) {
  using P = SP<NSW, RES, PRO>;
  constexpr int S = P::S, H = P::H, WOUT = P::WOUT, NF = P::NF;
  extern __shared__ double smem[];
  Ctx c;
  c.g = a.g;
  const Grid& g = c.g;
  c.ring_u = smem;                               // PD x SWC (unused when ZU)
  c.ring_f = c.ring_u + PD * SWC;                // PDF x SWC
  c.xch = c.ring_f + PDF * SWC;                  // NF x 2 x SWC neighbour exchange rows
  c.rlast = c.xch + NF * 2 * SWC;                // 4 x SWC last-residual ring (RES)
  double* tA = c.rlast + 4 * SWC;                // 25 x 9
  double* tK = tA + NCLS * 9;                    // 25 x 9
  double* red = tK + NCLS * 9;                   // 32
  c.tA = tA;
  c.tK = tK;
  c.tid = threadIdx.x;
  c.b = blockIdx.z;
  const int64_t n = g.n();
  c.j0 = blockIdx.x * WOUT;                      // first owned column (even)
#pragma unroll
  for (int q = 0; q < CPT; ++q) {
    const int lc = CPT * c.tid + q;
    c.col[q] = c.j0 - H + lc;
    c.cin[q] = c.col[q] >= 0 && c.col[q] < g.cols;
    c.owned_c[q] = lc >= H && lc < H + WOUT && c.cin[q];
    c.ccls[q] = c.cin[q] ? bandc(c.col[q], g.cols) : 2;  // out-of-grid columns are zeroed anyway
  }
  c.lL = max(CPT * c.tid - 1, 0);
  c.lR = min(CPT * c.tid + CPT, SWC - 1);
  c.R0 = blockIdx.y * a.seg;
  c.R1 = min(g.rows, c.R0 + a.seg);
  c.fb = a.f + c.b * n;
  c.ub = ZU ? nullptr : a.u + c.b * n;
  c.uob = a.uo + c.b * n;
  c.mk = MSK ? a.mask : nullptr;
  // fast steps need every CTA column interior (band class 2) and in the grid
  const bool cta_fast = c.j0 - H >= 2 && c.j0 - H + SWC - 1 <= g.cols - 3;

  if (CM != 0) {
    for (int q = c.tid; q < NCLS * 9; q += SWT) {
      tA[q] = a.A.cls[(int64_t)c.b * NCLS * 9 + q];
      tK[q] = a.K.cls[(int64_t)c.b * NCLS * 9 + q];
    }
  }
  __syncthreads();

  double w[NF][3][4];
#pragma unroll
  for (int k = 0; k < NF; ++k)
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q) w[k][r][q] = 0.0;
  double hold[NSW][CPT];
#pragma unroll
  for (int m = 0; m < NSW; ++m) hold[m][0] = hold[m][1] = 0.0;
  double acc = 0.0;

  // steps t in [t0, t1], t0 aligned to a multiple of 3 (extra leading steps only
  // compute rows nobody needs)
  int t0 = c.R0 - S - 1;
  t0 -= m3(t0);
  const int t1 = c.R1 + 2 * S;
  int prow = t0;
  const int64_t cstride = g.cols;
  const int tc = CPT * c.tid;
  const double* pu = ZU ? nullptr : c.ub + (int64_t)prow * cstride + c.col[0];
  const double* pf = c.fb + (int64_t)prow * cstride + c.col[0];
  auto issue = [&]() {
    const bool rok = (unsigned)prow < (unsigned)g.rows;
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      const bool rv = rok && c.cin[q];
      if (!ZU) cp_async8(&c.ring_u[(prow & (PD - 1)) * SWC + tc + q], rv ? pu + q : c.ub, rv);
      cp_async8(&c.ring_f[(prow & (PDF - 1)) * SWC + tc + q], rv ? pf + q : c.fb, rv);
    }
    cp_commit();
    ++prow;
    if (!ZU) pu += cstride;
    pf += cstride;
  };
  for (int q = 0; q < DIST; ++q) issue();

#define MGB_STEP(PH_)                                                                                  \
  {                                                                                                    \
    const int t = tb + PH_;                                                                            \
    issue();                                                                                           \
    cp_wait<DIST>();                                                                                   \
    if (cta_fast && t - 2 * S >= 2 && t <= g.rows - 3)                                                 \
      stream_step<NSW, RES, PRO, NORM, ZU, CM, MSK, true, PH_>(a, c, t, w, hold, acc);                 \
    else                                                                                               \
      stream_step<NSW, RES, PRO, NORM, ZU, CM, MSK, false, PH_>(a, c, t, w, hold, acc);                \
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

int stream_seg(const Grid& g) {
  // rows per CTA segment (even): long segments amortise the pipeline fill,
  // enough segments keep ~2 CTAs per SM busy
  const int strips = (g.cols + (SWC - 12) - 1) / (SWC - 12);
  int seg = 256;
  while (seg > 32 && (int64_t)strips * ((g.rows + seg - 1) / seg) * g.batch < 2 * 148) seg /= 2;
  return seg;
}

dim3 stream_grid(const Grid& g, int nsw, bool res) {
  const int H = 2 * nsw + 2;
  const int wout = SWC - 2 * H;
  const int seg = stream_seg(g);
  return dim3((g.cols + wout - 1) / wout, (g.rows + seg - 1) / seg, g.batch);
}

int stream_blocks(const Grid& g, int nsw, bool res) {
  const dim3 d = stream_grid(g, nsw, res);
  return (int)(d.x * d.y);
}

static size_t stream_smem(int nsw, bool res) {
  const int nf = 2 * nsw + (res ? 1 : 0);
  return sizeof(double) * ((size_t)(PD + PDF + 2 * nf + 4) * SWC + 2 * NCLS * 9 + 32);
}

template <typename KF>
static cudaError_t run_k(KF kern, dim3 grid, size_t smem, cudaStream_t s, const StreamArgs& a) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, SWT, smem, s>>>(a);
  return MGB_DBG(__func__);
}

cudaError_t launch_stream(const StreamArgs& a0, int nsw, bool res, bool pro, bool norm) {
  StreamArgs a = a0;
  a.seg = stream_seg(a.g);
  const dim3 grid = stream_grid(a.g, nsw, res);
  const bool zu = a.u == nullptr;
  const bool msk = a.mask != nullptr;
  const int cm = (a.A.cls != nullptr && a.K.cls != nullptr && !msk) ? (a.ci_valid ? 2 : 1) : 0;
  cudaStream_t s = a.stream;
  const size_t sm = stream_smem(nsw, res);
  ++g_launches;
#define MGB_ST(NSW_, RES_, PRO_, NORM_, ZU_)                                                           \
  if (nsw == NSW_ && res == RES_ && pro == PRO_ && norm == NORM_ && zu == ZU_) {                     \
    if (msk) return run_k(k_stream<NSW_, RES_, PRO_, NORM_, ZU_, 0, true>, grid, sm, s, a);           \
    if (cm == 2) return run_k(k_stream<NSW_, RES_, PRO_, NORM_, ZU_, 2, false>, grid, sm, s, a);      \
    if (cm == 1) return run_k(k_stream<NSW_, RES_, PRO_, NORM_, ZU_, 1, false>, grid, sm, s, a);      \
    return run_k(k_stream<NSW_, RES_, PRO_, NORM_, ZU_, 0, false>, grid, sm, s, a);                   \
  }
  // PRE: restriction, optional norm, optional zero start; POST: prolongation, no norm
  MGB_ST(1, true, false, false, false) MGB_ST(1, true, false, true, false)
  MGB_ST(1, true, false, false, true)  MGB_ST(1, true, false, true, true)
  MGB_ST(2, true, false, false, false) MGB_ST(2, true, false, true, false)
  MGB_ST(2, true, false, false, true)  MGB_ST(2, true, false, true, true)
  MGB_ST(1, false, true, false, false) MGB_ST(2, false, true, false, false)
#undef MGB_ST
  return cudaErrorInvalidValue;
}

}  // namespace mgb
