// Row-streaming V-cycle passes, one warp per CTA, four columns per lane
// (single-problem band-class levels: config 2 / 5 levels 0-2).
//
// Same passes as k_stream / k_stream2 (PRE: [history norm] + nu sweeps + residual +
// full-weighting restriction; POST: prolongation + nu sweeps; plain sweeps; the
// residual-norm pass), same push-form FMA chains, hence bit-identical results.  One pass
// more: POST with the norm of the residual of its own output (res && pro), which folds the
// per-iteration residual of solve() and the last history entry of run_cycles into the
// last pass instead of a separate pass over u and f.  The
// design differs in three ways that remove what bounded k_stream2 (a CTA-wide
// barrier and a shared-memory neighbour exchange per row step at 8 warps/SM):
//
// * one warp owns a 128-column strip (4 columns per lane) and a row segment; the
//   column neighbours of a lane's run come from its neighbour lanes by warp
//   shuffles, so there is no barrier and no exchange buffer at all;
// * no lag between stages: at step t stage k pushes the row of field k-1 that stage
//   k-1 completed in the SAME step (field 0 row t, field k row t - k), so the state
//   carried from step to step is only the two open output rows per stage (an update
//   stage's seed, field k-2, was completed earlier in the same step).  About 130
//   registers instead of 200+, and the pipeline fill is 2S + 2 rows per segment
//   instead of 3S + 3;
// * the per-lane step overhead (ring fill, shuffles, stores, control) is paid once
//   per four points.
//
// u and f rows arrive through per-warp cp.async rings (row t + 3 issued at step t,
// fully coalesced: lane q copies strip columns q + 32 m), read back as two 16-byte
// halves per lane from a swizzled layout (conflict-free).  Coarse correction rows
// (POST) are loaded into registers one coarse row ahead.
//
// Reference: v_cycle hierarchy.py:96-111 (with RepeatedSmoother cli.py:365-377),
// apply_stencil grid.py:216-226, inferred_apply smoothers.py:325-343, restrict
// transfer.py:108-121, prolong transfer.py:124-147, history hierarchy.py:129-141.
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cstdint>
#include <cmath>

#include "mgb_stream.h"

// This file is compiled twice to halve the build's critical path: as itself (the NSW = 1
// passes, stream3_ok and the launch_stream3 dispatcher) and through mgb_stream3b.cu with
// MGB_S3_PART 2 (the NSW = 2 passes behind launch_stream3_nsw2).
#ifndef MGB_S3_PART
#define MGB_S3_PART 1
#endif
#if defined(MGB_CTA_PROF) && MGB_S3_PART != 2
#undef MGB_CTA_PROF   // the per-warp timeline probe lives with the NSW = 2 passes
#endif

#ifdef MGB_CTA_PROF
// experiment builds only: per-CTA (smid, entry, loop start, end) of the last warp-strip launch
__device__ unsigned long long g_cta_prof3[4 * 8192];
#endif

namespace mgb {
namespace {

constexpr int CPT = 4;             // columns per lane
constexpr int SW3 = 32 * CPT;      // strip width
#ifndef MGB_S3NR
#define MGB_S3NR 1
#endif
#ifndef MGB_S3DG
#define MGB_S3DG 2
#endif
#ifndef MGB_S3MINB
#define MGB_S3MINB 12
#endif
#ifndef MGB_S3WPC
#define MGB_S3WPC 1
#endif
#ifndef MGB_S3SYNC
#define MGB_S3SYNC 0
#endif
// Experiment knobs (defaults: one warp per CTA, no pacing).  The warp schedulers serve the
// lowest warp slot first: on config 2's level-0 PRE pass (per-warp %globaltimer,
// scripts/cta_prof3.py) the three warps of a scheduler finish after 64 / 75 / 85 us.  Putting
// WPC3 warps (each still owning its own strip and row segment) into one CTA per SM with a CTA
// barrier every SYNC3 rows keeps them in step (a warp that has finished exits, the barrier
// goes on with the rest) - and measured SLOWER (PRE 95 - 101 us for periods 16 - 2 against
// 92.7 us unpaced): the schedulers lose nothing when the favoured warp finishes early, the
// others speed up.
constexpr int WPC3 = MGB_S3WPC;
constexpr int SYNC3 = WPC3 > 1 ? MGB_S3SYNC : 0;   // rows between pacing barriers (a power of two; 0: none)
static_assert((SYNC3 & (SYNC3 - 1)) == 0, "pacing period");
static_assert(MGB_S3MINB % WPC3 == 0, "warps per SM must be a multiple of the warps per CTA");
constexpr int NR3 = MGB_S3NR;      // rows entering per step
constexpr int DG3 = MGB_S3DG;      // ring groups (of NR3 rows) in flight beyond the next one
constexpr int pow2_at_least(int v) { return v <= 1 ? 1 : 2 * pow2_at_least((v + 1) / 2); }
constexpr int RU3 = pow2_at_least(NR3 * (DG3 + 2));       // u ring rows (t .. t + NR (DG + 2) - 1)
constexpr int RF3 = pow2_at_least(NR3 * (DG3 + 2) + 4);   // f ring rows (t - 4 .. t + NR (DG + 2) - 1)
static_assert(NR3 * (DG3 + 2) <= RU3 && NR3 * (DG3 + 2) + 4 <= RF3, "ring depths");
constexpr int NCLS3 = 25;
// One stage lag (experiment knob, default off: measured no faster, see DESIGN): stages 3.. consume the field-2 row that stage 2 completed in
// the PREVIOUS step (kept in four registers), so a step holds two independent stage chains
// (1-2 and 3-5) instead of one chain through all five.  A warp issues in order, and a
// dependent stage costs a shuffle plus three dependent DFMAs (~100 cycles): the single chain
// kept a lone warp at ~1,000 cycles per step for ~470 cycles of issue.
#ifndef MGB_S3LAG
#define MGB_S3LAG 0
#endif
constexpr bool LAG3 = MGB_S3LAG != 0;
// quasi-uniform flavour: whether steps inside the segment get their own (test-free) body
#ifndef MGB_S3Q_MODE0
#define MGB_S3Q_MODE0 0
#endif
static_assert(!LAG3 || NR3 == 1, "the stage lag is written for one row per step");
__host__ __device__ constexpr int lag3(int k) { return LAG3 && k >= 3 ? 1 : 0; }

template <int NSW, bool RES, bool NOUT>
struct P3 {
  static constexpr int S = NOUT ? 1 : 2 * NSW + (RES ? 1 : 0);   // stages after field 0
  static constexpr int H = ((RES ? S + 1 : S) + 1) & ~1;          // halo columns per side (even)
  static constexpr int WOUT = SW3 - 2 * H;                         // owned columns per strip
};

__device__ __forceinline__ int band3(int i, int n) { return i < 2 ? i : (i >= n - 2 ? 4 - (n - 1 - i) : 2); }

// ring slot position of strip column s: lane i's columns 4i .. 4i+3 as two 16-byte
// halves, the halves swapped on every other group of four lanes (conflict-free reads)
__device__ __forceinline__ int swz(int s) {
  const int i = s >> 2, h = (s >> 1) & 1;
  return 4 * i + 2 * (h ^ ((i >> 2) & 1)) + (s & 1);
}

__device__ __forceinline__ void cpa8s(unsigned sa, const double* gmem, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cpa8f(unsigned sa, const double* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cpa16(unsigned sa, const double* gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cpa16f(unsigned sa, const double* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// the lane's four values of a ring row
__device__ __forceinline__ void ld_own(const double* row, int lane, double v[4]) {
  const int x = (lane >> 2) & 1;
  const double2 p = *reinterpret_cast<const double2*>(row + 4 * lane + 2 * x);
  const double2 q = *reinterpret_cast<const double2*>(row + 4 * lane + 2 * (x ^ 1));
  v[0] = p.x;
  v[1] = p.y;
  v[2] = q.x;
  v[3] = q.y;
}

struct Lane3 {
  int lane, c0, R0, R1;
  int64_t ld;          // row pitch of f, u, uo
  int64_t ldo;         // row pitch of uo when it is a dense array beside padded inputs (0: ld)
  int64_t ldc;         // row pitch of the coarse arrays rc / ec (cols / 2, or the next level's padded pitch)
  int64_t boffc;       // batched levels: the problem's offset into the coarse arrays rc / ec (0: one problem)
  const double* kq;    // quasi-uniform levels: the nine M class tables (a.kq in the constant bank; a batch: the
                       // problem's own, in shared memory)
  const double* wci;   // interior-class A (9) and M (9) weights: a.ci (constant bank), or the problem's own in
                       // registers (batched uniform levels)
  unsigned cin, own;   // bit c: column c0 + c in the grid / owned
  int cb[4];           // band of column c0 + c (2 when outside the grid)
  int ecol, eside;     // quasi-uniform levels: the lane's boundary column (0 or 2; -1 none: c0 is even, the
                       // grid's first and last columns are even); the strip's boundary column band
                       // (0 first strip, 2 last strip, -1 interior strip; warp-uniform)
  const double* tab;   // shared-memory class tables: A [25][9], then K [25][9]
  int lo_c, hi_c, mcol;  // POST: coarse rows that may be read, first coarse column of the lane
  double* uo_t;          // uo at (row t - 2 NSW, column c0) of the current step (advanced per step)
};

// POST: the lane's coarse correction values (columns m - 1 .. m + 1) of coarse row ci
__device__ __forceinline__ void load_e3(const StreamArgs& a, const Lane3& L, int ci, double (&dst)[3]) {
  const int rows_c = a.g.rows / 2, cols_c = a.g.cols / 2;
  const bool rv = ci >= 0 && ci < rows_c && ci >= L.lo_c && ci <= L.hi_c;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const int cj = L.mcol + q;
    dst[q] = (rv && (unsigned)cj < (unsigned)cols_c) ? __ldg(a.ec + L.boffc + (int64_t)ci * L.ldc + cj) : 0.0;
  }
}

// One pipeline step: field-0 rows t .. t + NR - 1 enter; stage k completes rows
// t - k .. t - k + NR - 1.  P0 = t mod 2 (static).
// MODE 0: interior rows, interior strip, inside the segment (constant-bank weights, no
//         row or column tests: only the lane-constant column ownership of outputs)
//      1: interior rows, uniform level or interior strip (constant weights; out-of-grid
//         columns zeroed, output rows tested against the segment)
//      2: interior rows, edge strip of a non-uniform level (per-column class weights)
//      3: anything else (per row band and column class; rows and columns tested)
// Quasi-uniform levels (UNI == 2, StreamArgs::uniform == 2) use modes 0 and 1 and
//      4: interior rows, edge strip: constant weights as in mode 1 (the residual stages'
//         interior A weights are exact everywhere: the class tables differ only in entries
//         that multiply the zero closure); the update stages' three chains of the grid's
//         boundary column are redone with its class weights (a.kq, constant bank) in the one
//         lane that holds it, in stencil_dot's term order, and replace the constant-weight ones
//      5: rows at the grid's top / bottom: mode 4's scheme with the row-band class of each of
//         the three rows an update stage pushes into (one warp-uniform table per row role),
//         rows tested against the grid
// instead of modes 2 and 3: no per-column class tables, no shared-memory table.
template <int NSW, bool RES, bool PRO, bool NORM, bool ZU, bool NOUT, int UNI, bool ZA, bool ALN, int NR, int MODE, int P0>
__device__ __forceinline__ void step3(const StreamArgs& a, const Lane3& L, const int t, const int tq,
                                      double (&acc)[P3<NSW, RES, NOUT>::S][2][4], double (&racc)[2], double& norm,
                                      const double* ringF, const double* ringU, double (&e0)[3], double (&e1)[3],
                                      double (&eN)[3], double (&prev)[4]) {
  using P = P3<NSW, RES, NOUT>;
  constexpr int S = P::S;
  const Grid& g = a.g;
  constexpr bool CMASK = MODE >= 1;            // zero out-of-grid columns
  constexpr bool EFIX = MODE >= 4;             // boundary-column chains of the update stages
  constexpr bool RTEST = MODE == 3 || MODE == 5;   // rows may leave the grid / the interior band
  const int lane = L.lane;
  double fld[S + 1][NR][4];
  // ---- field 0: u (+ P ec) at rows t + j
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    const int row = t + j;
    const bool podd = (P0 + j) & 1;
    if (ZU) {
#pragma unroll
      for (int c = 0; c < 4; ++c) fld[0][j][c] = 0.0;
      continue;
    }
    ld_own(ringU + (row & (RU3 - 1)) * SW3, lane, fld[0][j]);
    if (PRO) {
      if (!podd) {   // coarse row row / 2 enters: rows row/2 - 1, row/2 in e0, e1; the next in flight
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          e0[q] = e1[q];
          e1[q] = eN[q];
        }
        load_e3(a, L, (row >> 1) + 1, eN);
      }
      if (!RTEST || (unsigned)row < (unsigned)g.rows) {
        double p[4];
        if (podd) {   // odd fine row: coarse row row >> 1 only (di = 0)
          p[0] = fma(0.25, e1[1], 0.0);
          p[0] = fma(0.25, e1[0], p[0]);
          p[1] = fma(0.5, e1[1], 0.0);
          p[2] = fma(0.25, e1[2], 0.0);
          p[2] = fma(0.25, e1[1], p[2]);
          p[3] = fma(0.5, e1[2], 0.0);
        } else {      // even fine row: coarse rows row / 2 (di = -1) and row / 2 - 1 (di = +1)
          p[0] = fma(0.125, e1[1], 0.0);
          p[0] = fma(0.125, e1[0], p[0]);
          p[1] = fma(0.25, e1[1], 0.0);
          p[0] = fma(0.125, e0[1], p[0]);
          p[0] = fma(0.125, e0[0], p[0]);
          p[1] = fma(0.25, e0[1], p[1]);
          p[2] = fma(0.125, e1[2], 0.0);
          p[2] = fma(0.125, e1[1], p[2]);
          p[3] = fma(0.25, e1[2], 0.0);
          p[2] = fma(0.125, e0[2], p[2]);
          p[2] = fma(0.125, e0[1], p[2]);
          p[3] = fma(0.25, e0[2], p[3]);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) fld[0][j][c] += p[c];
      }
      if (CMASK) {
        const bool rv = !RTEST || (unsigned)row < (unsigned)g.rows;
#pragma unroll
        for (int c = 0; c < 4; ++c) fld[0][j][c] = (rv && ((L.cin >> c) & 1)) ? fld[0][j][c] : 0.0;
      }
    }
  }
  // ---- stages k = 1..S: push field k-1 rows t - k - lag + 1 + j, complete rows t - k - lag + j
#pragma unroll
  for (int k = 1; k <= S; ++k) {
    const bool resid = k & 1;
    const double* tabk = L.tab + (resid ? 0 : NCLS3 * 9);
    const int dk = lag3(k);
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const int row = t - k - dk + j;
      double* out = fld[k][j];
#ifndef MGB_S3_NOGUARD
      // (not on uniform levels: their segments are long, and the test costs config 2's level-0
      // PRE pass 3 us; it saves 8 / 5 us on the PRE passes of levels 1 / 2)
      // pipeline fill: stage k's first needed row (R0 - 1 - (S - k), or R0 - (S - k) without a
      // restriction) starts its chain 2k - 2 steps after the segment's first step; before
      // that the stage would only compute rows nothing reads (warp-uniform test; steps inside
      // the segment, MODE 0, are past it)
      if (UNI != 1 && MODE != 0 && k > 1 && tq + j < 2 * k - 2 + dk) {
#pragma unroll
        for (int c = 0; c < 4; ++c) out[c] = 0.0;
        continue;
      }
#endif
      if (ZU && k == 1) {
        // zero start: f - A 0 = f (the chain fma(-w, 0, f) returns f)
        ld_own(ringF + (row & (RF3 - 1)) * SW3, lane, out);
      } else {
        // the lagged stage's input is last step's field-2 row
        const double* v = (LAG3 && k == 3) ? prev : fld[k - 1][j];
        double in[6];
        in[0] = __shfl_up_sync(0xffffffffu, v[3], 1);     // column c0 - 1 (lane 0: strip halo)
        in[1] = v[0];
        in[2] = v[1];
        in[3] = v[2];
        in[4] = v[3];
        in[5] = __shfl_down_sync(0xffffffffu, v[0], 1);   // column c0 + 4 (lane 31: strip halo)
        double seed[4];
        if (resid) {
          ld_own(ringF + ((row + 2) & (RF3 - 1)) * SW3, lane, seed);
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c) seed[c] = (LAG3 && k == 4) ? prev[c] : fld[k - 2][j][c];
        }
        const int s_old = (P0 + j + k + dk) & 1;   // slot of row t - k - lag + j (completes now); static
        int bN = 2, bM = 2, bB = 2;
        if (MODE == 3 || MODE == 5) {
          const int x = row + 1;              // the input row
          bN = (unsigned)(x + 1) < (unsigned)g.rows ? band3(x + 1, g.rows) : 2;
          bM = (unsigned)x < (unsigned)g.rows ? band3(x, g.rows) : 2;
          bB = (unsigned)(x - 1) < (unsigned)g.rows ? band3(x - 1, g.rows) : 2;
        }
        const double* wN[4];
        const double* wM[4];
        const double* wB[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (MODE <= 1 || MODE == 4 || UNI == 1 || (MODE == 5 && resid)) {
            wN[c] = wM[c] = wB[c] = resid ? L.wci : L.wci + 9;
          } else if (MODE == 5) {
            // the row band's table of the interior column band (bands 1 and 3 equal band 2)
            wN[c] = L.kq + ((bN == 0 ? 0 : bN == 4 ? 2 : 1) * 3 + 1) * 9;
            wM[c] = L.kq + ((bM == 0 ? 0 : bM == 4 ? 2 : 1) * 3 + 1) * 9;
            wB[c] = L.kq + ((bB == 0 ? 0 : bB == 4 ? 2 : 1) * 3 + 1) * 9;
          } else if (MODE == 2) {
            wN[c] = wM[c] = wB[c] = tabk + (10 + L.cb[c]) * 9;
          } else {
            wN[c] = tabk + (bN * 5 + L.cb[c]) * 9;
            wM[c] = tabk + (bM * 5 + L.cb[c]) * 9;
            wB[c] = tabk + (bB * 5 + L.cb[c]) * 9;
          }
        }
        double (&Ao)[4] = acc[k - 1][s_old];        // row t - k + j: its bottom terms complete it
        double (&Am)[4] = acc[k - 1][s_old ^ 1];    // row t - k + j + 1: middle terms
        // mode 4: the boundary column's three chains (completing row, middle row, new row)
        // with its own class weights, from the accumulators as they are before this stage
        double eo = 0.0, em = 0.0, es = 0.0;
        if (EFIX && !resid && (MODE == 4 || L.eside >= 0)) {
          const bool e2 = L.ecol == 2;
          // the boundary column's class per row role (interior rows: one table)
          const double* weN = L.kq + ((MODE == 4 ? 1 : (bN == 0 ? 0 : bN == 4 ? 2 : 1)) * 3 + L.eside) * 9;
          const double* weM = MODE == 4 ? weN : L.kq + ((bM == 0 ? 0 : bM == 4 ? 2 : 1) * 3 + L.eside) * 9;
          const double* weB = MODE == 4 ? weN : L.kq + ((bB == 0 ? 0 : bB == 4 ? 2 : 1) * 3 + L.eside) * 9;
          double xe[3];
#pragma unroll
          for (int q = 0; q < 3; ++q) xe[q] = e2 ? in[2 + q] : in[q];
          eo = e2 ? Ao[2] : Ao[0];
          em = e2 ? Am[2] : Am[0];
          es = e2 ? seed[2] : seed[0];
#pragma unroll
          for (int q = 0; q < 3; ++q) eo = fma(weB[6 + q], xe[q], eo);
#pragma unroll
          for (int q = 0; q < 3; ++q) em = fma(weM[3 + q], xe[q], em);
#pragma unroll
          for (int q = 0; q < 3; ++q) es = fma(weN[q], xe[q], es);
        }
#define FMS(w_, x_, a_) fma(resid ? -(w_) : (w_), (x_), (a_))
        // critical path first (the completed row feeds the next stage through shuffles),
        // one wave of four independent chains per weight; every chain keeps
        // stencil_dot's term order
#pragma unroll
        for (int o = 6; o < 9; ++o)
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (!(ZA && resid && o == 6)) Ao[c] = FMS(wB[c][o], in[c + o - 6], Ao[c]);
#pragma unroll
        for (int c = 0; c < 4; ++c) out[c] = Ao[c];
#pragma unroll
        for (int o = 3; o < 6; ++o)
#pragma unroll
          for (int c = 0; c < 4; ++c) Am[c] = FMS(wM[c][o], in[c + o - 3], Am[c]);
#pragma unroll
        for (int o = 0; o < 3; ++o)
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (!(ZA && resid && o == 2)) seed[c] = FMS(wN[c][o], in[c + o], seed[c]);
#undef FMS
        // row t - k + j + 2 reuses the completed row's slot
#pragma unroll
        for (int c = 0; c < 4; ++c) Ao[c] = seed[c];
        if (EFIX && !resid && (MODE == 4 || L.eside >= 0)) {
#pragma unroll
          for (int c = 0; c < 4; c += 2) {
            const bool fix = L.ecol == c;
            out[c] = fix ? eo : out[c];
            Am[c] = fix ? em : Am[c];
            Ao[c] = fix ? es : Ao[c];
          }
        }
      }
      // zero the completed row outside the grid
      if (RTEST) {
        const bool rv = (unsigned)row < (unsigned)g.rows;
#pragma unroll
        for (int c = 0; c < 4; ++c) out[c] = (rv && ((L.cin >> c) & 1)) ? out[c] : 0.0;
      } else if (CMASK) {
#pragma unroll
        for (int c = 0; c < 4; ++c) out[c] = ((L.cin >> c) & 1) ? out[c] : 0.0;
      }
      // MODE 0 steps lie inside the segment (every output row owned): no row tests
      const bool orow = MODE == 0 || (row >= L.R0 && row < L.R1);
      if (NORM && k == 1) {
        // excluded points are skipped (adding their exact +0 would leave the same bits)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (orow && ((L.own >> c) & 1)) norm = fma(out[c], out[c], norm);
      }
      if (!NOUT && k == 2 * NSW && orow && (MODE == 0 || a.uo)) {
        double* dst = L.uo_t + (int64_t)j * (L.ldo ? L.ldo : L.ld);   // row t - 2 NSW - lag + j
#ifdef MGB_S3_NOSTORE
        if (out[0] == 1.2345e300)   // experiment builds only: (practically) no HBM writes
#endif
        if (ALN && L.ldo == 0) {
          // padded layout: 16-byte aligned pairs (c0 even), owned pairs whole (even bounds)
          if (L.own & 1) *reinterpret_cast<double2*>(dst) = make_double2(out[0], out[1]);
          if (L.own & 4) *reinterpret_cast<double2*>(dst + 2) = make_double2(out[2], out[3]);
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if ((L.own >> c) & 1) dst[c] = out[c];
        }
      }
    }
  }
  if (LAG3 && S >= 3) {
#pragma unroll
    for (int c = 0; c < 4; ++c) prev[c] = fld[2][NR - 1][c];
  }
  // ---- POST with RES: the norm of the last residual (field S) instead of a restriction: the
  // relative residual of the pass's OUTPUT u, folded into the pass (hierarchy.py:135-141)
  if (RES && PRO) {
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const int y = t - S - lag3(S) + j;
      const bool orow = MODE == 0 || (y >= L.R0 && y < L.R1);
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (orow && ((L.own >> c) & 1)) norm = fma(fld[S][j][c], fld[S][j][c], norm);
    }
  }
  // ---- restriction: push field S rows y = t - S + j (coarse anchors c0 + 1, c0 + 3)
  if (RES && !PRO) {
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const int y = t - S - lag3(S) + j;
      const double* xs = fld[S][j];
      const double xr = __shfl_down_sync(0xffffffffu, xs[0], 1);
      if ((P0 + j + S + lag3(S)) & 1) {   // y odd: middle row of coarse row (y - 1) / 2
        racc[0] = fma(0.125, xs[0], racc[0]);
        racc[0] = fma(0.25, xs[1], racc[0]);
        racc[0] = fma(0.125, xs[2], racc[0]);
        racc[1] = fma(0.125, xs[2], racc[1]);
        racc[1] = fma(0.25, xs[3], racc[1]);
        racc[1] = fma(0.125, xr, racc[1]);
      } else {
        // bottom row of coarse row (y - 2) / 2 (completes), top row of coarse row y / 2
        double sA = fma(0.0625, xs[0], racc[0]);
        sA = fma(0.125, xs[1], sA);
        sA = fma(0.0625, xs[2], sA);
        double sB = fma(0.0625, xs[2], racc[1]);
        sB = fma(0.125, xs[3], sB);
        sB = fma(0.0625, xr, sB);
        const int ci = (y - 2) >> 1;
        const int rows_c = g.rows / 2, cols_c = g.cols / 2;
        if (MODE == 0 || (y >= 2 && ci >= (L.R0 >> 1) && 2 * ci + 1 < L.R1 && ci < rows_c)) {
          const int cj = L.c0 >> 1;
          double* dst = a.rc + L.boffc + (int64_t)ci * L.ldc + cj;
          if ((L.own & 1) && cj < cols_c) {
            const bool act = a.mask_c == nullptr || a.mask_c[(int64_t)ci * cols_c + cj];
            dst[0] = act ? sA : 0.0;
          }
          if ((L.own & 4) && cj + 1 < cols_c) {
            const bool act = a.mask_c == nullptr || a.mask_c[(int64_t)ci * cols_c + cj + 1];
            dst[1] = act ? sB : 0.0;
          }
        }
        double r = 0.0625 * xs[0];
        r = fma(0.125, xs[1], r);
        racc[0] = fma(0.0625, xs[2], r);
        r = 0.0625 * xs[2];
        r = fma(0.125, xs[3], r);
        racc[1] = fma(0.0625, xr, r);
      }
    }
  }
}

// UNI: every band class equals the interior one (config 2 / 5 level 0): constant
// weights everywhere.  NR rows enter per step (one ring group, one wait per step);
// the register file holds 8 warps/SM at MINB 8.
// ZA (uniform levels only): the operator's anti-diagonal corners A[-1][+1], A[+1][-1]
// are exact zeros (the rotated finite-difference stencil, problems.py:45-52): their
// FMAs are skipped (adding an exact zero product leaves every chain's value unchanged).
// ALN: f, u, uo use the padded layout (16-byte copies bypassing L1, 128-bit stores, no
// column predicates: the margins read as zeros).
// BAT: a batch of problems on a uniform level (config 4's level 0, V(1,1)): a work item is
// (problem, strip, segment), and the problem's own interior weights live in registers instead
// of the constant bank (36 registers: the NSW = 1 passes have room for them).
template <int NSW, bool RES, bool PRO, bool NORM, bool ZU, bool NOUT, int UNI, bool ZA, bool ALN, bool BAT = false>
__global__ void __launch_bounds__(32 * WPC3, MGB_S3MINB / WPC3) k_stream3(StreamArgs a) {
#ifdef MGB_CTA_PROF
  unsigned long long prof_t0 = 0, prof_t1 = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prof_t0));
#endif
  pdl_trigger();
  using P = P3<NSW, RES, NOUT>;
  constexpr int S = P::S, H = P::H, WOUT = P::WOUT;
  constexpr int NR = NR3;
  extern __shared__ __align__(16) double sm3[];
  // work item of this warp; warps beyond the last item leave before any barrier
  // (the lane-0 broadcast tells the compiler that the warp index, and with it the strip, the
  // segment and every row bound derived from it, is warp-uniform: uniform registers and
  // uniform branches, as in a one-warp CTA)
  const int wib = WPC3 > 1 ? __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0) : 0;
  const int item = blockIdx.x * WPC3 + wib;
  const int nitems1 = a.nedge * a.nseg_edge + (a.nstrips - a.nedge) * a.nseg;   // per problem
  const int nitems = BAT ? nitems1 * a.g.batch : nitems1;
  if (WPC3 > 1 && item >= nitems) return;
  const int bprob = BAT ? item / nitems1 : 0;
  double* ringF = sm3 + (size_t)wib * (RF3 * SW3 + (ZU ? 0 : RU3 * SW3) + (UNI != 0 ? 0 : 2 * NCLS3 * 9) +
                                       (BAT && UNI == 2 ? 82 : 0));  // RF3 x SW3
  double* ringU = ringF + RF3 * SW3;         // RU3 x SW3 (unused when ZU)
  double* tab = ringU + (ZU ? 0 : RU3 * SW3);  // 2 x 25 x 9 class tables (non-uniform levels)
  const Grid& g = a.g;
  Lane3 L;
  L.lane = threadIdx.x & 31;
  // CTA -> (strip, row segment): the two edge strips' CTAs first (shorter segments on
  // non-uniform levels, whose edge steps read class weights), then the interior ones
  int strip, sy, seg, nseg;
  {
    const int id = BAT ? item - bprob * nitems1 : item, ne = a.nedge;
    if (id < ne * a.nseg_edge) {
      strip = (id % ne == 0) ? 0 : a.nstrips - 1;
      sy = id / ne;
      seg = a.seg_edge;
      nseg = a.nseg_edge;
    } else {
      const int q = id - ne * a.nseg_edge, ni = a.nstrips - ne;
      strip = (ne > 0 ? 1 : 0) + q % ni;
      sy = q / ni;
      seg = a.seg;
      nseg = a.nseg;
    }
  }
  const int j0 = strip * WOUT;
  L.c0 = j0 - H + CPT * L.lane;
  L.cin = L.own = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int gc = L.c0 + c;
    const bool in = (unsigned)gc < (unsigned)g.cols;
    L.cin |= (in ? 1u : 0u) << c;
    L.own |= ((in && gc >= j0 && gc < j0 + WOUT) ? 1u : 0u) << c;
    L.cb[c] = in ? band3(gc, g.cols) : 2;
  }
  L.ecol = -1;
  L.eside = strip == 0 ? 0 : (strip == a.nstrips - 1 ? 2 : -1);
#pragma unroll
  for (int c = 0; c < 4; c += 2)
    if (L.c0 + c == 0 || L.c0 + c == g.cols - 1) L.ecol = c;
  const int own0 = a.own1 > 0 ? a.own0 : 0, rend = a.own1 > 0 ? a.own1 : g.rows;
  L.R0 = own0 + sy * seg;
  L.R1 = sy == nseg - 1 ? rend : min(rend, L.R0 + seg);
  L.tab = tab;
  L.ld = a.ld > 0 ? a.ld : g.cols;
  L.ldo = ALN && a.ld_out > 0 ? a.ld_out : 0;
  L.boffc = BAT ? (int64_t)bprob * (g.rows / 2) * (g.cols / 2) : 0;
  L.ldc = a.ldc > 0 ? a.ldc : g.cols / 2;
  double wreg[18];
  if (BAT) {
#pragma unroll
    for (int o = 0; o < 9; ++o) {
      wreg[o] = __ldg(a.A.cls + (int64_t)bprob * NCLS3 * 9 + 12 * 9 + o);
      wreg[9 + o] = __ldg(a.K.cls + (int64_t)bprob * NCLS3 * 9 + 12 * 9 + o);
    }
  }
  L.wci = BAT ? wreg : a.ci;
  L.kq = a.kq;
  if (BAT && UNI == 2) {
    // the problem's class tables of the row / column bands {first, interior, last} (StreamArgs::kq's layout)
    double* kqs = ringU + (ZU ? 0 : RU3 * SW3);
    for (int q = L.lane; q < 81; q += 32) {
      const int cls = q / 9, o = q - 9 * cls, r = cls / 3, c = cls - 3 * r;
      kqs[q] = __ldg(a.K.cls + (int64_t)bprob * NCLS3 * 9 + ((2 * r) * 5 + 2 * c) * 9 + o);
    }
    __syncwarp();
    L.kq = kqs;
  }
  const bool strip_int = j0 - H >= 2 && j0 - H + SW3 - 1 <= g.cols - 3;
  if (UNI == 0) {
    for (int q = L.lane; q < 2 * NCLS3 * 9; q += 32)
      tab[q] = q < NCLS3 * 9 ? a.A.cls[q] : a.K.cls[q - NCLS3 * 9];
    __syncwarp();
  }
  // rows: field S rows [ylo, yhi] are needed (restriction: one row beyond the owned
  // range on each side), field 0 rows [ylo - S, yhi + S]; steps start at a multiple of NR
  const int ylo = RES ? L.R0 - 1 : L.R0, yhi = RES ? L.R1 : L.R1 - 1;
  const int tfirst = ylo - S;   // the first step that matters (stage k: 2k - 2 steps later)
  int t0 = tfirst;
  t0 -= (t0 & 1);   // even: static row parities (NR = 2 steps, or the two-step unroll)
  const int t1 = yhi + S + lag3(S);   // the lagged stages finish one step later
  const int lo_row = max(0, ylo - S), hi_row = min(g.rows - 1, yhi + S);
  L.lo_c = (lo_row - 2) >> 1;
  L.hi_c = (hi_row >> 1) + 1;
  L.mcol = (L.c0 >> 1) - 1;
  // ring fill: lane q copies strip columns q + 32 m (coalesced rows) to the ring
  // positions swz(q + 32 m) = swz(q) + 32 m; rows outside [lo_row, hi_row] and columns
  // outside the grid are zero-filled (size-0 copies).  Padded layout: lane q copies the
  // 16-byte column pairs q and q + 32 (positions swz(2q), swz(2q + 64) = swz(2q) + 64),
  // the margins supplying the zeros outside the grid.
  const int colq = j0 - H + (ALN ? 2 : 1) * L.lane;
  const unsigned sF = (unsigned)__cvta_generic_to_shared(ringF + swz((ALN ? 2 : 1) * L.lane));
  const unsigned sU = (unsigned)__cvta_generic_to_shared(ringU + swz((ALN ? 2 : 1) * L.lane));
  const bool cols_all = j0 - H >= 0 && j0 - H + SW3 <= g.cols;   // every strip column in the grid
  unsigned cq = 0;
#pragma unroll
  for (int m = 0; m < 4; ++m) cq |= (((unsigned)(colq + 32 * m) < (unsigned)g.cols) ? 1u : 0u) << m;
  const int64_t boff = BAT ? (int64_t)bprob * g.n() : 0;
  const double* fb = a.f + boff;
  const double* ub = a.u ? a.u + boff : nullptr;
  // padded layout: every row a segment touches ([-11, rows + 8], inside the PAD_ROWS margins)
  // and every strip column is addressable and the margins hold zeros, so the copies need no
  // predicate; rows are issued in sequence, so the source pointers just advance by the pitch
  const double* fnx = nullptr;
  const double* unx = nullptr;
  auto issue_row = [&](int r, bool wu) {
#ifdef MGB_S3_NOLOAD
    return;   // experiment builds only: no HBM reads (compute-only timing)
#endif
    const unsigned of = sF + (unsigned)((r & (RF3 - 1)) * SW3 * 8);
    const unsigned ou = sU + (unsigned)((r & (RU3 - 1)) * SW3 * 8);
    if (ALN) {
      cpa16f(of, fnx);
      cpa16f(of + 512, fnx + 64);
      fnx += L.ld;
      if (!ZU && wu) {
        cpa16f(ou, unx);
        cpa16f(ou + 512, unx + 64);
        unx += L.ld;
      }
      return;
    }
    const bool rv = r >= lo_row && r <= hi_row;
    const int64_t ro = (int64_t)r * L.ld + colq;
    if (rv && cols_all) {
#pragma unroll
      for (int m = 0; m < 4; ++m) cpa8f(of + 256 * m, fb + ro + 32 * m);
      if (!ZU && wu) {
#pragma unroll
        for (int m = 0; m < 4; ++m) cpa8f(ou + 256 * m, ub + ro + 32 * m);
      }
    } else {
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const bool v = rv && ((cq >> m) & 1);
        cpa8s(of + 256 * m, v ? fb + ro + 32 * m : fb, v);
        if (!ZU && wu) cpa8s(ou + 256 * m, v ? ub + ro + 32 * m : ub, v);
      }
    }
  };
  // ring group s: rows s NR .. s NR + NR - 1
  // wu: with the u rows (the groups before t0 carry f rows only: u rows before t0 are
  // never read, and copying them would race with rows t0 .. for the same ring slots)
  auto issue = [&](int s, bool wu) {
#pragma unroll
    for (int j = 0; j < NR; ++j) issue_row(s * NR + j, wu);
    cpa_commit();
  };
  double acc[S][2][4];
#pragma unroll
  for (int k = 0; k < S; ++k)
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[k][r][c] = 0.0;
  double racc[2] = {0.0, 0.0};
  double norm = 0.0;
  // POST: coarse rows (t >> 1) - 1, t >> 1 (e0, e1) and the next one in flight (eN)
  double e0[3] = {0.0, 0.0, 0.0}, e1[3] = {0.0, 0.0, 0.0}, eN[3] = {0.0, 0.0, 0.0};
  double prev[4] = {0.0, 0.0, 0.0, 0.0};   // field 2's newest row (the stage lag)
  pdl_wait();  // u, f, ec come from the preceding kernels; uo / rc may still be read there
  if (PRO) {
    load_e3(a, L, (t0 >> 1) - 1, e1);
    load_e3(a, L, t0 >> 1, eN);
  }
  // groups of rows t0 - 4 .. : the residual seeds reach back to row t - 3
  const int s0 = t0 / NR - (4 + NR - 1) / NR;
  const int sstart = t0 / NR;
  if (ALN) {
    fnx = fb + (int64_t)(s0 * NR) * L.ld + colq;
    if (!ZU) unx = ub + (int64_t)t0 * L.ld + colq;
  }
  for (int s = s0; s <= sstart + DG3; ++s) issue(s, s >= sstart);
  L.uo_t = NOUT || !a.uo ? nullptr : a.uo + boff + (int64_t)(t0 - 2 * NSW - lag3(2 * NSW)) * (L.ldo ? L.ldo : L.ld) + L.c0;
#ifdef MGB_CTA_PROF
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prof_t1));
#endif

#define MGB_STEP3(P0_)                                                                                       \
  {                                                                                                          \
    const int t = tb + (P0_) * NR, tq = t - tfirst;                                                          \
    __syncwarp();                                                                                            \
    issue(t / NR + 1 + DG3, true);                                                                           \
    cpa_wait<DG3>(); /* f rows up to t + NR and u rows t .. t + NR - 1 have landed */                       \
    __syncwarp();                                                                                            \
    const bool rows_int = t - S - lag3(S) >= 2 && t + NR <= g.rows - 3;                                      \
    /* core: every row an output of this step touches is owned (norm, u, coarse rows) */                    \
    const bool core = t - S - lag3(S) - 2 >= L.R0 && t + NR <= L.R1 - 1;                                     \
    if (UNI == 2) {                                                                                                                                   \
      if (!rows_int)                                                                                                                                  \
        step3<NSW, RES, PRO, NORM, ZU, NOUT, UNI, ZA, ALN, NR, 5, (P0_) * NR & 1>(a, L, t, tq, acc, racc, norm, ringF, ringU, e0, e1, eN, prev);            \
      else if (!strip_int)                                                                                                                            \
        step3<NSW, RES, PRO, NORM, ZU, NOUT, UNI, ZA, ALN, NR, 4, (P0_) * NR & 1>(a, L, t, tq, acc, racc, norm, ringF, ringU, e0, e1, eN, prev);            \
      else if (MGB_S3Q_MODE0 && core && (NOUT || a.uo))                                                                                                                \
        step3<NSW, RES, PRO, NORM, ZU, NOUT, UNI, ZA, ALN, NR, 0, (P0_) * NR & 1>(a, L, t, tq, acc, racc, norm, ringF, ringU, e0, e1, eN, prev);            \
      else                                                                                                                                            \
        step3<NSW, RES, PRO, NORM, ZU, NOUT, UNI, ZA, ALN, NR, 1, (P0_) * NR & 1>(a, L, t, tq, acc, racc, norm, ringF, ringU, e0, e1, eN, prev);            \
    } else if (rows_int && strip_int && core && (NOUT || a.uo))                                                                                       \
      step3<NSW, RES, PRO, NORM, ZU, NOUT, UNI, ZA, ALN, NR, 0, (P0_) * NR & 1>(a, L, t, tq, acc, racc, norm, ringF, ringU, e0, e1, eN, prev);              \
    else if (rows_int && (UNI != 0 || strip_int))                                                                                                     \
      step3<NSW, RES, PRO, NORM, ZU, NOUT, UNI, ZA, ALN, NR, 1, (P0_) * NR & 1>(a, L, t, tq, acc, racc, norm, ringF, ringU, e0, e1, eN, prev);              \
    else if (rows_int)                                                                                                                                \
      step3<NSW, RES, PRO, NORM, ZU, NOUT, UNI, ZA, ALN, NR, 2, (P0_) * NR & 1>(a, L, t, tq, acc, racc, norm, ringF, ringU, e0, e1, eN, prev);              \
    else                                                                                                                                              \
      step3<NSW, RES, PRO, NORM, ZU, NOUT, UNI, ZA, ALN, NR, 3, (P0_) * NR & 1>(a, L, t, tq, acc, racc, norm, ringF, ringU, e0, e1, eN, prev);              \
    L.uo_t += NR * (L.ldo ? L.ldo : L.ld);                                                                                     \
  }
  // t0 is even: with one row per step, unroll two steps so each step's parity is static
  constexpr int ADV = NR == 2 ? NR : 2 * NR;
#pragma unroll 1
  for (int tb = t0; tb <= t1; tb += ADV) {
    if (SYNC3 > 0 && (tb & ((SYNC3 > ADV ? SYNC3 : ADV) - 1)) == 0) __syncthreads();   // pacing only
    MGB_STEP3(0)
    if (NR != 2) MGB_STEP3(1)
  }
#undef MGB_STEP3
  cpa_wait<0>();
#ifdef MGB_CTA_PROF
  if (L.lane == 0 && item < 8192) {
    unsigned long long t2;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    unsigned wid;
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
    smid |= wid << 16;
    g_cta_prof3[4 * item] = smid;
    g_cta_prof3[4 * item + 1] = prof_t0;
    g_cta_prof3[4 * item + 2] = prof_t1;
    g_cta_prof3[4 * item + 3] = t2;
  }
#endif
  if (NORM || (RES && PRO)) {
    double v = norm;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (L.lane == 0) a.partials[item] = v;
  }
}

}  // namespace

static size_t stream3_smem(bool zu, int uni, bool bat) {
  return sizeof(double) * ((size_t)(RF3 + (zu ? 0 : RU3)) * SW3 + (uni != 0 ? 0 : 2 * NCLS3 * 9) + (bat && uni == 2 ? 82 : 0));
}

static int sm_count3() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

// Row segments: whole waves of the measured occupancy with the fewest pipeline fills
// (2S + 3 steps per segment); the two edge strips of a non-uniform level get
// segments shorter by the measured cost ratio of their class-weight steps.
static void choose_seg3(int rows, int cols, int S, int wout, int occ, int uniform, StreamArgs& a, int batch = 1) {
  const int strips = (cols + wout - 1) / wout;
  const int ne = uniform == 1 ? 0 : std::min(strips, 2), ni = strips - ne;
  const int64_t slots = (int64_t)sm_count3() * std::max(occ, 1);
  static const double r_env = getenv("MGB_EDGE3") ? atof(getenv("MGB_EDGE3")) : 0.0;
  // edge-strip step cost relative to an interior strip's: class lookups for every column
  // 1.8 (measured); the boundary-column fix-up of a quasi-uniform level ~1.25
  const double r = ni == 0 ? 1.0 : (r_env > 0.0 ? r_env : (uniform == 2 ? 1.25 : 1.8));
  const int F = 2 * S + 2 + NR3 + lag3(S);
  double best_t = 1e300;
  a.nstrips = strips;
  a.nedge = ne;
  static const int min_rows = getenv("MGB_SEG3_MINROWS") ? std::max(1, atoi(getenv("MGB_SEG3_MINROWS"))) : 12;
  const int maxseg = std::max(1, (rows + min_rows - 1) / min_rows);
  for (int nseg = 1; nseg <= maxseg; ++nseg) {
    const int seg = (rows + nseg - 1) / nseg;
    int nse = ne ? std::max(1, (int)std::ceil(rows / std::max(1.0, (seg + F) / r - F))) : 0;
    static const int edge_min_rows = getenv("MGB_EDGE3_MINROWS") ? atoi(getenv("MGB_EDGE3_MINROWS")) : 8;   // measured: 8 beats 16 on c2 levels 1-2
    nse = std::min(nse, std::max(1, (rows + edge_min_rows - 1) / edge_min_rows));
    const int sege = ne ? (rows + nse - 1) / nse : 0;
    const int64_t ctas = ((int64_t)ni * nseg + (int64_t)ne * nse) * batch;
    const double w = (double)ctas / slots;
    const double waves = w <= 2.0 ? std::ceil(w) : w + 0.5;
    const double t = waves * std::max((double)(seg + F), ne ? r * (sege + F) : 0.0);
    if (t < best_t) {
      best_t = t;
      a.seg = seg;
      a.nseg = nseg;
      a.seg_edge = sege;
      a.nseg_edge = nse;
    }
  }
  static const int force_seg = getenv("MGB_SEG3") ? atoi(getenv("MGB_SEG3")) : 0;  // experiments only
  if (force_seg > 0) {
    a.nseg = std::max(1, std::min(maxseg, (rows + force_seg - 1) / force_seg));
    a.seg = (rows + a.nseg - 1) / a.nseg;
    a.nseg_edge = a.nseg;
    a.seg_edge = a.seg;
  }
}

template <int NSW, bool RES, bool PRO, bool NORM, bool ZU, bool NOUT, int UNI, bool ZA, bool ALN, bool BAT = false>
static cudaError_t run_k3(StreamArgs a, int* nblocks) {
  using P = P3<NSW, RES, NOUT>;
  auto kern = k_stream3<NSW, RES, PRO, NORM, ZU, NOUT, UNI, ZA, ALN, BAT>;
  struct Occ {
    int dev, occ;
  };
  static thread_local std::vector<Occ> occ_cache;   // per instantiation, per device
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  const size_t smem = WPC3 * stream3_smem(ZU, UNI, BAT);
  int occ = -1;
  for (auto& e : occ_cache)
    if (e.dev == dev) occ = e.occ;
  if (occ < 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * WPC3, smem);
    if (e != cudaSuccess) return e;
    occ *= WPC3;   // warps (work items) per SM
    occ_cache.push_back({dev, occ});
  }
  if (a.own1 <= 0) {
    a.own0 = 0;
    a.own1 = a.g.rows;
  }
  static const int occ_env = getenv("MGB_S3_OCC") ? atoi(getenv("MGB_S3_OCC")) : 0;   // experiments: warps per SM the segments are sized for
  static const int occ_env_q = getenv("MGB_S3_OCC_Q") ? atoi(getenv("MGB_S3_OCC_Q")) : 0;   // the same, quasi-uniform flavour only
  if (occ_env > 0) occ = std::min(occ, occ_env);
  if (UNI == 2 && occ_env_q > 0) occ = std::min(occ, occ_env_q);
  choose_seg3(a.own1 - a.own0, a.g.cols, P::S, P::WOUT, occ, UNI == 2 ? 2 : (a.uniform == 1 ? 1 : 0), a,
              BAT ? a.g.batch : 1);
  const int ni = a.nstrips - a.nedge;
  const int nctas = a.nedge * a.nseg_edge + ni * a.nseg;
  if (nblocks) *nblocks = nctas;   // per problem (the history partials are [problem][item])
  const int64_t total = (int64_t)nctas * (BAT ? a.g.batch : 1);
  const cudaError_t e = launch_pdl(kern, dim3((unsigned)((total + WPC3 - 1) / WPC3), 1, 1), dim3(32 * WPC3), smem, a.stream, a);
  if (e != cudaSuccess) return e;
  return MGB_DBG("k_stream3");
}

cudaError_t launch_stream3_nsw2(const StreamArgs& a, bool res, bool pro, bool norm, int* nblocks);

#if MGB_S3_PART == 1
bool stream3_ok(const StreamArgs& a, int nsw) {
  const bool tabs = a.mask == nullptr && a.A.cls != nullptr && a.K.cls != nullptr && a.A.ks == 1 && a.K.ks == 1;
  if (a.g.batch > 1)   // the batched flavours: uniform, or quasi-uniform with the first and last strip distinct
    return tabs && (a.uniform == 1 || (a.uniform == 2 && quasi_cols_ok(a.g.cols))) && nsw == 1 && !a.padded && a.own1 <= 0;
  return tabs && a.ci_valid;
}
#endif

#if MGB_S3_PART == 1
cudaError_t launch_stream3(const StreamArgs& a, int nsw, bool res, bool pro, bool norm, int* nblocks) {
  if (nsw == 2) return launch_stream3_nsw2(a, res, pro, norm, nblocks);
#else
cudaError_t launch_stream3_nsw2(const StreamArgs& a, bool res, bool pro, bool norm, int* nblocks) {
  const int nsw = 2;
#endif
  const bool zu = a.u == nullptr;
  const bool nout = a.uo == nullptr && !res && !pro;
  static const bool no_za = getenv("MGB_NO_ZA") && atoi(getenv("MGB_NO_ZA")) != 0;   // A/B experiments
  const bool za = !no_za && a.ci[2] == 0.0 && a.ci[6] == 0.0;   // uniform: every class is the interior one
  // quasi-uniform flavour: the first and the last strip must be different strips
  const bool quasi = a.uniform == 2 && quasi_cols_ok(a.g.cols);
#if MGB_S3_PART == 1
#define MGB_ST3B(NSW_, RES_, PRO_, NORM_, ZU_, NOUT_)                                              \
  if (a.g.batch > 1 && nsw == NSW_ && res == RES_ && pro == PRO_ && norm == NORM_ && zu == ZU_ && nout == NOUT_) \
    return a.uniform == 2 ? run_k3<NSW_, RES_, PRO_, NORM_, ZU_, NOUT_, 2, false, false, true>(a, nblocks) \
                          : run_k3<NSW_, RES_, PRO_, NORM_, ZU_, NOUT_, 1, false, false, true>(a, nblocks);
#else
#define MGB_ST3B(NSW_, RES_, PRO_, NORM_, ZU_, NOUT_)
#endif
#define MGB_ST3(NSW_, RES_, PRO_, NORM_, ZU_, NOUT_)                                                \
  MGB_ST3B(NSW_, RES_, PRO_, NORM_, ZU_, NOUT_)                                                     \
  if (nsw == NSW_ && res == RES_ && pro == PRO_ && norm == NORM_ && zu == ZU_ && nout == NOUT_)    \
    return quasi           ? (a.padded ? run_k3<NSW_, RES_, PRO_, NORM_, ZU_, NOUT_, 2, false, true>(a, nblocks)   \
                                       : run_k3<NSW_, RES_, PRO_, NORM_, ZU_, NOUT_, 2, false, false>(a, nblocks)) \
           : a.uniform != 1 ? run_k3<NSW_, RES_, PRO_, NORM_, ZU_, NOUT_, 0, false, false>(a, nblocks) \
           : !a.padded ? (za ? run_k3<NSW_, RES_, PRO_, NORM_, ZU_, NOUT_, 1, true, false>(a, nblocks)  \
                             : run_k3<NSW_, RES_, PRO_, NORM_, ZU_, NOUT_, 1, false, false>(a, nblocks)) \
           : za        ? run_k3<NSW_, RES_, PRO_, NORM_, ZU_, NOUT_, 1, true, true>(a, nblocks)       \
                       : run_k3<NSW_, RES_, PRO_, NORM_, ZU_, NOUT_, 1, false, true>(a, nblocks);
#if MGB_S3_PART == 2
  MGB_ST3(2, true, false, false, false, false) MGB_ST3(2, true, false, true, false, false)
  MGB_ST3(2, true, false, false, true, false)  MGB_ST3(2, true, false, true, true, false)
  MGB_ST3(2, false, true, false, false, false)
  MGB_ST3(2, true, true, false, false, false)   // POST + output residual norm
#elif !defined(MGB_S3_FEW)   // MGB_S3_FEW (experiment builds): the NSW = 2 passes only (fast compile)
  MGB_ST3(1, true, false, false, false, false) MGB_ST3(1, true, false, true, false, false)
  MGB_ST3(1, true, false, false, true, false)  MGB_ST3(1, true, false, true, true, false)
  MGB_ST3(1, false, false, false, false, false) MGB_ST3(1, false, false, true, false, false)
  MGB_ST3(1, false, false, false, true, false)  MGB_ST3(1, false, false, true, true, false)
  MGB_ST3(1, false, false, true, false, true)
  MGB_ST3(1, false, true, false, false, false)
  MGB_ST3(1, true, true, false, false, false)   // POST + output residual norm
#endif
#undef MGB_ST3
#undef MGB_ST3B
  return cudaErrorInvalidValue;
}

}  // namespace mgb

#ifdef MGB_CTA_PROF
extern "C" __attribute__((visibility("default"))) int mgb_debug_cta_prof3(unsigned long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, g_cta_prof3, sizeof(unsigned long long) * 4 * n);
}
#endif
