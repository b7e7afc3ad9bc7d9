// Row-streaming fused V-cycle passes (mgb_stream.cu).
#pragma once

#include "mgb_cycle.h"

namespace mgb {

struct StreamArgs {
  Grid g;
  Op A, K;                 // operator / smoother tables (planes or band classes), ks == 1
  const uint8_t* mask;     // fine mask (null = all active)
  const uint8_t* mask_c;   // coarse mask (restriction output)
  const double* f;         // right-hand side
  const double* u;         // input u (null = zero)
  double* uo;              // output u (must not alias u)
  const double* ec;        // coarse correction (POST)
  double* rc;              // restricted residual (PRE)
  double* partials;        // per-CTA sums of the input residual squared (history)
  int seg;                 // rows per CTA segment (set by the launcher)
  int own0, own1;          // owned global rows [own0, own1) (own1 == 0: the whole grid).  Rows
                           // own0 - 6 .. own1 + 5 of u, f (and the matching coarse rows of ec)
                           // must be addressable: with domain decomposition the arrays are
                           // ghosted row blocks passed as pointers pre-offset to global rows.
  int ci_valid;            // 1: ci holds the interior-class weights (batch == 1, classed A and M)
  int uniform;             // 1: every band class equals the interior one (ci valid everywhere);
                           // 2: quasi-uniform (LevelD::quasi_uniform: the classes differ only on the boundary
                           // rows / columns, A only in entries that point out of the grid)
  int kernel;              // streaming kernel: 0 auto, 1 one column per thread, 2 column pairs, 3 one warp per strip
  int a5;                  // per-point A with zero corner planes: their loads are skipped
  // two-column kernel CTA map (set by its launcher): edge strips (first / last) get
  // shorter segments (their steps take the boundary-class path), listed first
  // segments of a strip: the first has seg_first rows, the others seg (the last: the
  // rest); first / last segments on the grid's top / bottom are trimmed because their
  // boundary rows take the slow step variant
  // (the first seg_rem middle segments have one row more)
  int nstrips, nedge, seg_first, nseg, seg_rem, seg_edge, seg_edge_first, nseg_edge, seg_edge_rem;
  // warp-strip kernel only: row pitch (elements) of f, u and uo (0: cols), and whether
  // they use the padded level layout (pad_layout(): 16-byte aligned rows, zero margins of
  // PAD_ROWS rows and PAD_LCOLS / >= 122 columns around the grid, margins never written)
  int64_t ld;
  int padded;
  int64_t ldc;             // > 0: row pitch of the coarse arrays rc (PRE) and ec (POST): the next level's padded
                           // buffers (warp-strip kernel only; 0: cols / 2)
  int64_t ld_out;          // > 0: uo is a dense array of this pitch (the caller's own u) although f and u use
                           // the padded layout: the last POST pass of a solve writes its result there directly
  double ci[18];           // interior-class A (9) and M (9) weights, read from the constant bank
  double kq[81];           // quasi-uniform levels: M class tables [row band first / interior / last][column band
                           // first / interior / last][9], read from the constant bank
  cudaStream_t stream;
};

// Padded level layout of the warp-strip kernel: rows [-PAD_ROWS, rows + PAD_ROWS) x
// columns [-PAD_LCOLS, pitch - PAD_LCOLS); the base pointer addresses (0, 0).
constexpr int PAD_ROWS = 16, PAD_LCOLS = 8;
inline int64_t pad_pitch(int cols) { return ((int64_t)PAD_LCOLS + cols + 122 + 15) / 16 * 16; }
inline int64_t pad_elems(int rows, int cols) { return ((int64_t)rows + 2 * PAD_ROWS) * pad_pitch(cols); }
inline int64_t pad_offset(int cols) { return (int64_t)PAD_ROWS * pad_pitch(cols) + PAD_LCOLS; }

// PRE: res = true, pro = false (norm optional, u null = zero start);
// plain sweeps: res = pro = false, nsw = 1 (norm optional);
// POST: res = false, pro = true; res = pro = true (warp-strip kernel only, see
// stream_post_norm_ok): POST that also writes the partial sums of its output's residual.
// nsw in {1, 2}.  *nblocks receives the CTA count
// (the number of history partials written when norm is set).
cudaError_t launch_stream(const StreamArgs& a, int nsw, bool res, bool pro, bool norm, int* nblocks);
int stream_max_blocks(const Grid& g);
// which streaming kernel launch_stream picks for these arguments: 1, 2 or 3
int stream_kernel_kind(const StreamArgs& a, int nsw = 0);
// whether launch_stream(a, nsw, true, true, false, ..) — POST + output residual norm — is available
inline bool stream_post_norm_ok(const StreamArgs& a, int nsw = 0) { return stream_kernel_kind(a, nsw) == 3; }
// Two-columns-per-thread variant for band-class levels without masks (mgb_stream2.cu);
// launch_stream dispatches to it (MGB_STREAM1=1 keeps the one-column kernel).
cudaError_t launch_stream2(const StreamArgs& a, int nsw, bool res, bool pro, bool norm, int* nblocks);
// One warp per strip, four columns per lane (mgb_stream3.cu): single-problem band-class
// levels without masks (stream3_ok); launch_stream dispatches to it for kernel == 3
// (and for kernel == 0 on large levels, see launch_stream).
// (nsw: sweeps per pass; a batch of problems runs there only on a uniform level with nsw == 1)
bool stream3_ok(const StreamArgs& a, int nsw = 0);
// quasi-uniform flavour: the grid's first and last column must lie in different strips of
// every pass (a strip owns at most 124 columns)
inline bool quasi_cols_ok(int cols) { return cols > 124; }
bool warp_strip_selected(int kernel, int64_t n, int batch, bool uniform, int nsw = 0);
cudaError_t launch_stream3(const StreamArgs& a, int nsw, bool res, bool pro, bool norm, int* nblocks);

}  // namespace mgb
