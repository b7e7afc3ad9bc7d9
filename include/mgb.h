/*
 * mgb.h — C-ABI of the B200-native learned-smoother multigrid hot path.
 *
 * Drop-in boundary for the reference's Python solver API (mgsmooth 0.1.0,
 * /root/reference/pkg/src/mgsmooth).  The reference has no FFI; its "plugin"
 * surface is the Python module API re-exported by __init__.py:9-35 plus the
 * duck-typed smoother protocol obj.apply(r) (hierarchy.py:107,111).  Each
 * entry point below names the reference function it replaces.  The Python
 * facade paper_2102_12071_b200/ binds these through ctypes.
 *
 * Conventions
 *  - All fp64.  Grid arrays are dense row-major (rows, cols) with i = row = y,
 *    j = col = x (grid.py:3-13).  Batched calls stack `batch` problems of the
 *    same shape contiguously: (batch, rows, cols).
 *  - Stencil tables in the reference layout ("AoS"): (rows, cols, 3, 3), entry
 *    [di+1][dj+1] multiplies u(i+di, j+dj) (cross-correlation, zero outside).
 *    Smoother kernels: (rows, cols, k, 3, 3) (smoothers.py:291-300).
 *  - Masks are uint8 (rows, cols), 1 = active; NULL means every point active.
 *  - Pointers documented "dev" are CUDA device pointers; "host" are host
 *    pointers.  `stream` is a cudaStream_t passed as void* (NULL = legacy).
 *  - Every function returns an mgb_status.  Non-zero statuses map onto the
 *    reference's exception classes (errors.py:8-42); the message is available
 *    from mgb_last_error() (thread-local), and for MGB_SINGULAR the failing
 *    elimination step from mgb_last_pivot() (dense.py:38-40).
 *  - Compute functions never fall back to the CPU.  Without a usable sm_100
 *    device they return MGB_CUDA.
 */
#ifndef MGB_H
#define MGB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef enum {
  MGB_OK = 0,
  MGB_CONFIG = 1,       /* ConfigError            errors.py:16 */
  MGB_NUMERIC = 2,      /* NumericError           errors.py:20 */
  MGB_NONCONVERGED = 3, /* NonConvergedError      errors.py:40 */
  MGB_CONTRACT = 4,     /* ContractError          errors.py:12 */
  MGB_SINGULAR = 5,     /* SingularMatrixError    errors.py:24 */
  MGB_CUDA = 6,         /* RuntimeError (CUDA failure / no device) */
  MGB_NCCL = 7          /* RuntimeError (collective failure) */
} mgb_status;

enum { MGB_NET_CONV = 0, MGB_NET_FC = 1 };          /* smoothers.py:213-214 */

typedef struct mgb_hier mgb_hier;   /* device MultigridHierarchy (hierarchy.py:38) */
typedef struct mgb_work mgb_work;   /* per-solve workspace: concurrent solves on one hierarchy are safe */

/* ---- library / errors ---------------------------------------------------- */
int         mgb_version(void);
const char* mgb_last_error(void);
int         mgb_last_pivot(void);
int         mgb_device_info(int device, int* sm_count, int* cc_major, int* cc_minor);

/* ---- stateless grid ops on reference layouts (device pointers) ----------- */

/* grid.apply_stencil (grid.py:216-226): out = A u, zero outside, masked. k odd (1 or 3). */
int mgb_apply_stencil(int batch, int rows, int cols, int k, const double* A_dev,
                      const uint8_t* mask_dev, const double* u_dev, double* out_dev, void* stream);

/* transfer.restrict for full coarsening (transfer.py:108-121, coarsen_full :50-61):
   coarse = FW/16 gather about fine anchor 2c+1; coarse shape (rows/2, cols/2);
   mask_c_dev is the COARSE mask (= fine mask[1::2,1::2]). */
int mgb_restrict(int batch, int rows, int cols, const uint8_t* mask_c_dev,
                 const double* fine_dev, double* coarse_dev, void* stream);

/* transfer.prolong (transfer.py:124-147): fine = (2 FW/16) scatter of coarse; masked by the fine mask. */
int mgb_prolong(int batch, int rows, int cols, const uint8_t* mask_f_dev,
                const double* coarse_dev, double* fine_dev, void* stream);

/* transfer.galerkin_product (transfer.py:150-209) for full coarsening and k = 3 or 1 fine
   stencils: Ac (rows/2, cols/2, 3, 3) = R A P per coarse point; masks may be NULL.
   *k_out receives the trimmed stencil size (_trim, transfer.py:212-222): 3, or 1 when
   the outer ring is zero everywhere. */
int mgb_galerkin_product(int batch, int rows, int cols, int k, const double* A_dev,
                         const uint8_t* mask_f_dev, const uint8_t* mask_c_dev,
                         double* Ac_dev, int* k_out, void* stream);

/* smoothers.inferred_apply (smoothers.py:325-343): out = M(r), kernels (rows, cols, kst, 3, 3),
   leaky(slope) between stages. */
int mgb_smoother_apply(int batch, int rows, int cols, int kst, const double* K_dev,
                       const uint8_t* mask_dev, double slope, const double* r_dev,
                       double* out_dev, void* stream);

/* smoothers.infer_kernels (smoothers.py:302-322, net_forward :273-288, features :184-210):
   K_dev (rows, cols, kst, 3, 3) from A_dev (rows, cols, 3, 3).  weights_host is the
   concatenation of the net's weight arrays in row-major order (conv: (7,3,3),(5,3,3),
   (3,3,3),(27,9k); fc: (81,40),(40,40),(40,40),(40,9k)).  precision 64 = fp64 network
   (parity), 32 = fp32 network with fp64 diagonal normalisation. */
int mgb_infer_kernels(int batch, int rows, int cols, const double* A_dev, const uint8_t* mask_dev,
                      int variant, int kst, const double* weights_host, int64_t n_weights,
                      double slope, int precision, double* K_dev, void* stream);

/* dense.lu_factor / lu_solve (dense.py:21-63) on the device, n <= 4096.
   lu_dev (n, n) row-major is overwritten in place; perm_dev (n) int32. */
int mgb_lu_factor(int n, double* lu_dev, int32_t* perm_dev, void* stream);
int mgb_lu_solve(int n, const double* lu_dev, const int32_t* perm_dev, const double* b_dev,
                 double* x_dev, void* stream);

/* ---- hierarchy (hierarchy.py:70-214) -------------------------------------- */

/* build_hierarchy (hierarchy.py:70-88): Galerkin chain on the device, materialise and
   LU-factor the coarsest operator.  A0 is (batch, rows, cols, 3, 3) in the reference
   layout, on the host (a0_on_device = 0) or the device (1).  mask_host may be NULL
   (all active); it is shared by the batch.  The hierarchy lives on `device`. */
int mgb_hier_build(int device, int batch, int rows, int cols, double spacing,
                   const double* A0, int a0_on_device, const uint8_t* mask_host,
                   int levels, void* stream, mgb_hier** out);
/* Constant-coefficient hierarchy from band-class tables, with no per-point planes
   anywhere (memory = grid functions only; config 5's 32767^2 fits one GPU).
   cls_host: (batch, 25, 3, 3) tables of A0 for the band classes band(i)*5 + band(j),
   band = 0, 1 (first two rows/cols), 2 (interior), 3, 4 (last two).  A constant
   stencil (grid.py:209 constant_stencil) is 25 copies of its table.  All points
   active.  Galerkin products, the coarsest LU, CNN inference and Jacobi run on one
   representative point per class; results equal the per-point build. */
int mgb_hier_build_classed(int device, int batch, int rows, int cols, double spacing, const double* cls_host,
                           int levels, void* stream, mgb_hier** out);
void mgb_hier_destroy(mgb_hier* h);
int mgb_hier_depth(const mgb_hier* h, int* depth, int* batch);
/* level geometry; k = trimmed operator size; ks = installed smoother stages (0 = none) */
int mgb_hier_level_info(const mgb_hier* h, int level, int* rows, int* cols, int* k, int* ks,
                        double* spacing);
/* copy level operator / smoother kernels / mask out (host pointers, reference layouts;
   the operator is written as (batch, rows, cols, k, k) with the trimmed k). */
int mgb_hier_get_operator(const mgb_hier* h, int level, double* out_host);
int mgb_hier_get_kernels(const mgb_hier* h, int level, double* out_host);
int mgb_hier_get_mask(const mgb_hier* h, int level, uint8_t* out_host);
/* device pointer to the level operator in the internal layout (9 planes of
   batch*rows*cols each, plane o = (di+1)*3 + (dj+1)). */
int mgb_hier_operator_planes(const mgb_hier* h, int level, const double** planes_dev);

/* Storage of operator / smoother tables in the hot loop: mode 0 (default) keeps, per
   level and table, an exact 25-entry band-class representation when the table is
   constant away from the boundary (constant-coefficient problems); mode 1 forces
   per-point planes everywhere.  Results are bit-identical in both modes.
   mgb_hier_storage_info reports whether level `level`'s A / M tables are class-compact. */
int mgb_hier_set_storage(mgb_hier* h, int mode, void* stream);
int mgb_hier_storage_info(const mgb_hier* h, int level, int* a_classed, int* k_classed);
/* Number of operator entries per point the streaming passes read for level `level`'s
   per-point A: 5 when its corner planes are zero everywhere (a 5-point operator,
   checked on the device at build), else 9 (0 for class-compact A). */
int mgb_hier_stencil_points(const mgb_hier* h, int level, int* a_points);
/* How far level `level`'s band-class tables are from constant: 1 uniform (every class equals
   the interior one: the level-0 operator of a constant-coefficient problem, grid.py:163-206),
   2 quasi-uniform (the classes differ only on the first / last row and column, A only in
   entries that point out of the grid: the Galerkin chain of such a problem,
   transfer.py:150-222, with kernels inferred from each point's own table,
   smoothers.py:302-322), 0 neither (or per-point planes / masked).  The warp-strip passes
   use constant-bank weights everywhere on 1, and everywhere but the boundary column / rows on 2. */
int mgb_hier_level_uniformity(const mgb_hier* h, int level, int* uniformity);
/* Which kernel runs level `level`'s fused V(nu, nu) passes (measurement labels):
   0 separate sweep / restriction / prolongation kernels, 1 k_stream (one column per
   thread), 2 k_stream2 (column pairs), 3 k_stream3 (one warp per 128-column strip),
   4 k_tile (tile-local passes). */
int mgb_hier_pass_kernel(const mgb_hier* h, int level, int nu, int* kind);
/* Cycle pass structure for V(1|2, 1|2) with 1-stage smoothers: 2 (default) one
   row-streaming pass per smoothing phase (sweeps + restriction, prolongation +
   sweeps); 1: one streaming pass per sweep; 0: separate sweep / restriction /
   prolongation kernels. */
int mgb_hier_set_fused(mgb_hier* h, int enable);
/* Which fused pass runs where: levels with batch*rows*cols >= stream_min use the
   row-streaming passes (large, HBM-bound levels), smaller ones the tile-local passes
   when tile = 1 (latency-bound levels: one launch per phase) or separate kernels when
   tile = 0 (streaming and tile passes are bit-identical).  coarse_max > 0 runs every
   level with at most that many points in one single-CTA shared-memory kernel (default
   0: off, the tile passes measured faster).  Negative arguments keep a setting. */
int mgb_hier_set_passes(mgb_hier* h, int64_t stream_min, int tile, int64_t coarse_max);
/* Row-streaming kernel for single-problem band-class levels: 0 auto (column pairs
   per thread on levels of >= 2M points, one column per thread below), 1 always one
   column, 2 always column pairs.  Both produce bit-identical results (tests, tuning). */
int mgb_hier_set_stream_kernel(mgb_hier* h, int kind);

/* equip_inferred (hierarchy.py:207-214): per-level CNN inference on levels 0..L-2. */
int mgb_hier_equip_inferred(mgb_hier* h, int variant, int kst, const double* weights_host,
                            int64_t n_weights, double slope, int precision, void* stream);
/* equip_classical(kind="jacobi") (hierarchy.py:152-161, smoothers.py:29-50). */
int mgb_hier_equip_jacobi(mgb_hier* h, double omega, void* stream);
/* Shared-kernel convolutional smoother on level `level` (ConvSmoother,
   smoothers.py:105-145; equip_conv_init / retarget / equip_trained,
   hierarchy.py:164-204): M(r) = gain * (L_{nl-1} * act(... act(L_0 * r)) + S * r)
   with nl 3x3 layer kernels (layers_host: nl x 9, [di+1][dj+1]), skip kernel S
   (skip_host: 9, NULL = none), leaky(slope) between chained layers when leaky != 0.
   Replaces any per-point smoother on that level. */
int mgb_hier_set_conv_smoother(mgb_hier* h, int level, int nl, const double* layers_host,
                               const double* skip_host, int leaky, double slope, double gain);
/* convolve (grid.py:229-239): out = mask ? sum over non-zero w of w * u(p + o) : 0,
   zero padding; w_host: 9 weights.  Bit-identical to the reference. */
int mgb_convolve(int batch, int rows, int cols, const double* w_host, const uint8_t* mask_dev,
                 const double* u_dev, double* out_dev, void* stream);
/* ConvSmoother.apply (smoothers.py:133-145): out = M(r).  Bit-identical. */
int mgb_conv_smoother_apply(int batch, int rows, int cols, int nl, const double* layers_host,
                            const double* skip_host, int leaky, double slope, double gain,
                            const uint8_t* mask_dev, const double* r_dev, double* out_dev, void* stream);
/* install explicit kernels on one level: (batch, rows, cols, kst, 3, 3) host or device. */
int mgb_hier_set_kernels(mgb_hier* h, int level, int kst, const double* K, int on_device,
                         double slope, void* stream);

/* coarse_solve (hierarchy.py:91-93): x = A_L^{-1} f on the coarsest level (device). */
int mgb_coarse_solve(const mgb_hier* h, const double* f_dev, double* x_dev, void* stream);

/* ---- per-level fused passes on a hierarchy (device pointers, dense layout) ---- */
/* r = f - A_l u (masked); optionally (norm2_dev != NULL) per-problem sum of squares. */
int mgb_residual(const mgb_hier* h, int level, const double* f_dev, const double* u_dev,
                 double* r_dev, double* norm2_dev, void* stream);
/* u <- u + M(f - A u), `sweeps` times (u in/out; uses the workspace). */
int mgb_smooth(const mgb_hier* h, mgb_work* w, int level, const double* f_dev, double* u_dev,
               int sweeps, void* stream);
/* rc = R (f - A_l u) on level l -> l+1 (fused residual + full weighting). */
int mgb_restrict_residual(const mgb_hier* h, int level, const double* f_dev, const double* u_dev,
                          double* rc_dev, void* stream);
/* u <- u + P ec on level l (fused prolongation + coarse-grid correction). */
int mgb_prolong_correct(const mgb_hier* h, int level, const double* ec_dev, double* u_dev,
                        void* stream);

/* ---- cycles and solve ------------------------------------------------------ */
int  mgb_work_create(const mgb_hier* h, mgb_work** out);
void mgb_work_destroy(mgb_work* w);

/* v_cycle (hierarchy.py:96-111) from level `level`, V(nu1, nu2) (RepeatedSmoother,
   cli.py:365-377); u_dev in/out. */
int mgb_vcycle(const mgb_hier* h, mgb_work* w, int level, const double* f_dev, double* u_dev,
               int nu1, int nu2, void* stream);

/* Fixed-count cycle loop with the per-cycle residual history kept on the device:
   history_dev (batch, cycles + 1) receives ||f - A u_i|| / ||f|| (0 if ||f|| = 0 uses
   denominator 1, hierarchy.py:125-133).  No host synchronisation; the launch sequence
   is replayed from a CUDA graph after the first call with the same arguments.
   u_zero != 0 starts from u = 0 without reading u_dev. */
int mgb_run_cycles(const mgb_hier* h, mgb_work* w, const double* f_dev, double* u_dev,
                   int nu1, int nu2, int cycles, int u_zero, double* history_dev, void* stream);

/* Host-buffer variant of mgb_run_cycles (the drop-in call for callers holding host
   arrays): copies f (and u unless u_zero) host->device, runs the graph-replayed cycle
   loop, copies u and the history device->host and synchronises `stream`.  Pinned host
   memory gives asynchronous full-bandwidth copies; pageable memory also works. */
int mgb_run_cycles_host(const mgb_hier* h, mgb_work* w, const double* f_host, double* u_host,
                        int nu1, int nu2, int cycles, int u_zero, double* history_host,
                        void* stream);
/* A stream of `count` independent host-buffer solves (each as mgb_run_cycles_host),
   pipelined: the host->device copy of solve k+1 and the device->host copy of solve
   k overlap the cycles of solve k (two staging sets, two copy streams).  Returns
   after every copy has landed. */
int mgb_run_cycles_host_many(const mgb_hier* h, mgb_work* w, int count, const double* const* f_hosts,
                             double* const* u_hosts, int nu1, int nu2, int cycles, int u_zero,
                             double* const* history_hosts, void* stream);

/* solve (hierarchy.py:119-146) for batch == 1: loop until history < tol or max_iter,
   NonConvergedError (MGB_NONCONVERGED) when rr is non-finite or > 1e6 max(r0, tol).
   history_host has room for max_iter + 1 entries; *n_history receives its length. */
int mgb_solve(const mgb_hier* h, mgb_work* w, const double* f_dev, double* u_dev,
              int nu1, int nu2, double tol, int max_iter, double* history_host,
              int* n_history, int* iterations, int* converged, double* loop_seconds,
              void* stream);

/* Average device time (ms, CUDA events on `stream`) of one smoothing phase of the
   cycle on `level` over `reps` back-to-back repetitions: pass 0 = PRE (nu sweeps +
   residual + restriction), pass 1 = POST (prolongation + nu sweeps), in whatever
   pass structure the hierarchy uses (mgb_hier_set_fused).  f_dev / u_dev are
   level-sized device arrays; u_dev is overwritten. */
int mgb_time_pass(const mgb_hier* h, mgb_work* w, int level, int pass, int nu, const double* f_dev,
                  double* u_dev, int reps, double* ms, void* stream);

/* ---- domain decomposition ------------------------------------------
   The fine levels of a band-class hierarchy (mgb_hier_build_classed) split into
   `nparts` row blocks; every streaming pass runs on a block with 6 ghost rows per
   edge, refreshed by a halo exchange before each pass; levels with at most
   `agglomerate_rows` rows are solved redundantly on every part after an
   all-gather of the restricted residual.  Two layouts:
     virtual: nlocal == nparts, first_part = 0 — all parts on this GPU, halos by
              device copies (single-GPU test of the decomposition);
     NCCL:    nlocal == 1, first_part = rank — one part per process, halos by grouped
              ncclSend/ncclRecv, agglomeration by ncclAllGather, history norms by an
              8-byte ncclAllReduce; nccl_id from mgb_dd_nccl_unique_id on rank 0.
   The hierarchy must be built identically on every rank. */
typedef struct mgb_dd mgb_dd;
int  mgb_dd_nccl_unique_id(void* id_out /* 128 bytes */);
int  mgb_dd_create(const mgb_hier* h, int nparts, int first_part, int nlocal, const void* nccl_id,
                   int agglomerate_rows, mgb_dd** out);
void mgb_dd_destroy(mgb_dd* d);
/* level-0 rows [r0, r1) owned by `part`; number of distributed levels */
int  mgb_dd_info(const mgb_dd* d, int part, int* r0, int* r1, int* dist_levels);
int  mgb_dd_set_rhs(mgb_dd* d, int part, const double* f_owned_dev, void* stream);
int  mgb_dd_get_solution(const mgb_dd* d, int part, double* u_owned_dev, void* stream);
/* fixed-count V(nu1, nu2) cycles of the decomposed solve (graph-replayed); history_dev
   (cycles + 1) as mgb_run_cycles, identical on every rank. */
int  mgb_dd_run_cycles(mgb_dd* d, int nu1, int nu2, int cycles, int u_zero, double* history_dev, void* stream);
/* Callback exchange backend (one part per process, created with nccl_id == NULL): every
   exchange of the rank-local schedule is handed to `fn` after the stream has been
   synchronised (the cycles then run eagerly, without a graph).  op 0: send `count`
   doubles at send_dev to rank `peer` and receive `count` doubles from it into recv_dev;
   op 1: all-gather, `count` doubles at send_dev from every rank into recv_dev in rank
   order (send_dev is this rank's slot of recv_dev); op 2: all-reduce (sum) of `count`
   doubles in place at recv_dev.  All pointers are device pointers; return 0 on success. */
typedef int (*mgb_dd_exchange_fn)(void* ctx, int op, int peer, const double* send_dev, double* recv_dev, int64_t count);
int  mgb_dd_set_exchange(mgb_dd* d, mgb_dd_exchange_fn fn, void* ctx);
/* "overlap" (default 1): split every pass into an interior launch that overlaps the halo
   exchange (side stream) and an edge launch after it; "exchange" (default 1): 0 skips
   every exchange — wrong results, for timing the exposed exchange cost only. */
int  mgb_dd_set_option(mgb_dd* d, const char* key, int value);
/* bytes this process sent (halos + its all-gather slot) and the number of exchange steps
   in the last enqueued run (all cycles of it) */
int  mgb_dd_stats(const mgb_dd* d, int64_t* sent_bytes, int* exchanges);

/* ---- training path: device kernels behind the Python tape ----------
   The backward passes of the grid operations (autodiff.py:139-325), the small dense and
   batched-convolution operations of the kernel-inference nets, the transposed coarsest
   solve (dense.py:66-80) and Adam (training.py:73-93).  All pointers are device pointers,
   fp64; reductions over points are deterministic.  `scratch_dev` buffers hold
   mgb_ad_scratch_doubles(outputs) doubles. */
int mgb_ad_scratch_doubles(int outputs);
/* z = a x + b y (y == NULL: z = a x); a = 1, b = +-1 give x + y and x - y exactly */
int mgb_ad_axpby(int64_t n, double a, const double* x_dev, double b, const double* y_dev, double* z_dev, void* stream);
/* z[i] = x[i] * c[i / c_repeat] (c_repeat <= 1: c[i]) */
int mgb_ad_mul(int64_t n, const double* x_dev, const double* c_dev, int64_t c_repeat, double* z_dev, void* stream);
/* g_dev == NULL: z = leaky(x); else z = g * leaky'(x)  (autodiff.py:86-96) */
int mgb_ad_leaky(int64_t n, const double* x_dev, double slope, const double* g_dev, double* z_dev, void* stream);
/* x (n, c, inner) -> z (n, inner) summed over c; and its backward gx += broadcast(g)  (autodiff.py:109-115) */
int mgb_ad_sum_axis1(int64_t n, int c, int inner, const double* x_dev, double* z_dev, void* stream);
int mgb_ad_bcast_axis1(int64_t n, int c, int inner, const double* g_dev, double* gx_dev, void* stream);
/* out_dev[0] = sum x y (y == NULL: sum x^2) */
int mgb_ad_dot(int64_t n, const double* x_dev, const double* y_dev, double* scratch_dev, double* out_dev, void* stream);
/* du(q) = sum_d T(q - d)[d] gm(q - d) with gm = g on mask_in, du zeroed off mask_out (either
   mask may be NULL); T (rows, cols, 3, 3).  order 0: the backward of stencil_apply
   (autodiff.py:183-190, T = the operator table), 1: the du of pointwise_conv (:274-279). */
int mgb_ad_stencil_adjoint(int rows, int cols, const double* T_dev, const uint8_t* mask_in_dev,
                           const uint8_t* mask_out_dev, const double* g_dev, int order, double* du_dev, void* stream);
/* dK(p)[d] (+)= gm(p) u(p + d): the kernel gradient of pointwise_conv (autodiff.py:268-273) */
int mgb_ad_pconv_kgrad(int rows, int cols, const uint8_t* mask_dev, const double* g_dev, const double* u_dev,
                       int accumulate, double* dK_dev, void* stream);
/* dk[d] (+)= sum_p gm(p) u(p + d): the kernel gradient of conv2d (autodiff.py:152-159) */
int mgb_ad_conv_kgrad(int rows, int cols, int ksize, const uint8_t* mask_dev, const double* g_dev, const double* u_dev,
                      double* scratch_dev, int accumulate, double* dk_dev, void* stream);
/* conv_batch (autodiff.py:283-325): kern (c, 3, 3), img (n, 3, 3) -> out (n, c, 3, 3); backward
   into dk_dev (c, 3, 3) and / or dimg_dev (n, 3, 3) (either may be NULL) */
int mgb_ad_conv_batch(int64_t n, int c, const double* kern_dev, const double* img_dev, double* out_dev, void* stream);
int mgb_ad_conv_batch_bwd(int64_t n, int c, const double* kern_dev, const double* img_dev, const double* g_dev,
                          double* scratch_dev, int acc_k, double* dk_dev, int acc_img, double* dimg_dev, void* stream);
/* C (M, N) (+)= op(A) op(B), row-major; trans_a: A stored (K, M); trans_b: B stored (N, K)
   (autodiff.py:128-137 forward and both backward products) */
int mgb_ad_matmul(int M, int K, int N, const double* A_dev, int trans_a, const double* B_dev, int trans_b,
                  int accumulate, double* C_dev, double* scratch_dev, void* stream);
/* dense.lu_solve_t (dense.py:66-80): A^T x = b from the factorisation of A; scratch_dev: n doubles */
int mgb_lu_solve_t(int n, const double* lu_dev, const int32_t* perm_dev, const double* b_dev, double* x_dev,
                   double* scratch_dev, void* stream);
/* one Adam step of training.py:73-93 on a parameter array (g_dev == NULL: zero gradient) */
int mgb_ad_adam(int64_t n, double* p_dev, const double* g_dev, double* m_dev, double* v_dev, double lr, double beta1,
                double beta2, double eps, int step, void* stream);

/* Guard mode (environment MGB_GUARD=1 when the library is loaded; tests only): every
   device allocation of the library carries a 4 KiB canary region on each side.  Reports
   the number of live allocations and of those whose canaries were overwritten (their
   sizes are listed in mgb_last_error).  MGB_CONFIG when guard mode is off. */
int mgb_guard_check(int* allocations, int* corrupted);

/* instrumentation for bench.py: number of kernel launches issued by the last
   mgb_run_cycles / mgb_vcycle call (graph replays count their nodes). */
int64_t mgb_last_launch_count(const mgb_work* w);

/* Flexible GMRES (method 0; krylov.py:60-164 fgmres/_fgmres_cycle) and plain GMRES
   (method 1; krylov.py:167-236) on the flat grid vector.  Operator: apply_stencil
   with the per-point table A_dev (rows*cols*9, reference AoS layout; grid_action,
   krylov.py:249-258) and mask_dev (NULL = all active).  Right preconditioner: one
   V(nu1, nu2)-cycle from zero of the hierarchy behind workspace `pc` on the masked
   vector (cycle_preconditioner, krylov.py:261-270), or none (pc == NULL; required
   for gmres).  restart <= 0: no restart.  u_dev receives the solution (initial
   guess 0); history_host (max_iter + 1 entries) the absolute residual estimates,
   *n_hist their count, *iterations the Arnoldi steps, *converged the stopping
   test.  MGB_NUMERIC on an Arnoldi breakdown (krylov.py:119-122). */
int mgb_krylov(int method, int rows, int cols, const double* A_dev, const uint8_t* mask_dev, mgb_work* pc,
               int nu1, int nu2, const double* f_dev, double* u_dev, double tol, int max_iter, int restart,
               double* history_host, int* n_hist, int* iterations, int* converged, void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* MGB_H */
