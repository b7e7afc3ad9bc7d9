// C-ABI (include/mgb.h): hierarchy objects, workspaces, cycle driver, CUDA graphs.
//
// Reference map: hierarchy.py build_hierarchy :70-88, coarse_solve :91-93,
// v_cycle :96-111, solve :119-146, equip_classical :152-161, equip_inferred
// :207-214; cli.py RepeatedSmoother :365-377 (V(nu1, nu2)); errors.py.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "mgb_cycle.h"
#include "mgb_stream.h"
#include "mgb_tile.h"
#include "mgb_coarse.h"
#include "mgb_conv.h"
#include "mgb_dd.h"
#include "mgb_internal.h"

namespace mgb {

static thread_local std::string g_err;
static thread_local int g_pivot = -1;

void set_error(int status, const std::string& msg, int pivot) {
  (void)status;
  g_err = msg;
  g_pivot = pivot;
}
int fail(int status, const std::string& msg) {
  set_error(status, msg);
  return status;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ") in " + what;
  return MGB_CUDA;
}

}  // namespace mgb

using namespace mgb;

// ---------------------------------------------------------------------------
// objects

struct LevelD {
  int rows = 0, cols = 0, k = 3, ks = 0;
  double h = 0.0;
  int64_t n = 0;
  double* A = nullptr;     // batch x 9 planes of n
  double* K = nullptr;     // batch x ks x 9 planes of n
  uint8_t* mask = nullptr; // null = all active
  double* Acls = nullptr;  // band-class tables (batch x 25 x 9) when A is class-constant
  double* Kcls = nullptr;  // band-class tables (batch x 25 x ks x 9) when M is class-constant
  // band-class tables, host copies (batch x 225; class 12 = interior)
  std::vector<double> hAcls = std::vector<double>(225, 0.0), hKcls = std::vector<double>(225, 0.0);
  const double* hAint() const { return hAcls.data() + 12 * 9; }
  const double* hKint() const { return hKcls.data() + 12 * 9; }
  // every class equals its problem's interior one (A and M): boundary strips need no
  // class lookups
  bool uniform() const {
    if (hAcls.size() != hKcls.size()) return false;
    for (size_t q = 0; q < hAcls.size(); ++q) {
      const size_t i = q - q % 225 + 108 + q % 9;
      if (hAcls[q] != hAcls[i] || hKcls[q] != hKcls[i]) return false;
    }
    return true;
  }
  // Quasi-uniform (single problem): the classes differ from the interior one only on the
  // boundary rows / columns themselves (bands 1 and 3 equal band 2), and A differs there
  // only in the entries that point out of the grid - which multiply the exact zeros of the
  // zero closure (grid.py:27-35), so the interior A weights give the same values everywhere.
  // What a constant-coefficient operator's Galerkin chain with kernels inferred from each
  // point's own table looks like (config 2 / 5 levels >= 1): the warp-strip passes then need
  // class weights only for the update stages of the boundary column of the two edge strips
  // and for the steps that touch the first / last row.
  bool quasi_uniform() const {
    static const bool off = getenv("MGB_NO_QUASI") && atoi(getenv("MGB_NO_QUASI")) != 0;   // A/B experiments
    if (off || hAcls.size() != hKcls.size() || hAcls.size() % 225 != 0 || hAcls.empty() || cols % 2 == 0 || cols < 8 ||
        rows < 8)
      return false;
    for (size_t pb = 0; pb < hAcls.size(); pb += 225)   // every problem of a batch
      for (int bi = 0; bi < 5; ++bi)
        for (int bj = 0; bj < 5; ++bj) {
          const int qi = bi == 1 || bi == 3 ? 2 : bi, qj = bj == 1 || bj == 3 ? 2 : bj;
          for (int o = 0; o < 9; ++o) {
            const int di = o / 3 - 1, dj = o % 3 - 1;
            const bool outside = (bi == 0 && di < 0) || (bi == 4 && di > 0) || (bj == 0 && dj < 0) || (bj == 4 && dj > 0);
            const double av = hAcls[pb + (bi * 5 + bj) * 9 + o];
            if (!std::isfinite(av) || (!outside && av != hAcls[pb + 12 * 9 + o])) return false;
            if (hKcls[pb + (bi * 5 + bj) * 9 + o] != hKcls[pb + (qi * 5 + qj) * 9 + o]) return false;
          }
        }
    return true;
  }
  // StreamArgs::kq: the smoother's class tables of the row / column bands {first, interior, last}
  void fill_kq(double* kq) const {
    if (hKcls.size() < 225) return;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c)
        for (int o = 0; o < 9; ++o) kq[(r * 3 + c) * 9 + o] = hKcls[((2 * r) * 5 + 2 * c) * 9 + o];
  }
  // StreamArgs::uniform: 1 uniform, 2 quasi-uniform, 0 neither
  int uniformity() const {
    if (!Acls || !Kcls || mask) return 0;
    return uniform() ? 1 : (quasi_uniform() ? 2 : 0);
  }
  std::vector<uint8_t> hmask;
  int64_t nact = 0;
  bool a5 = false;         // per-point A with all-zero corner planes (5-point operator)
  ConvSm conv;             // shared-kernel convolutional smoother (conv.nl > 0 replaces K)
  bool has_smoother() const { return K != nullptr || conv.nl > 0; }
  Op opA() const { return Op{A, Acls, n, 1}; }
  Op opK() const { return Op{K == Kcls ? nullptr : K, Kcls, n, ks}; }
};

struct mgb_hier {
  int device = 0, batch = 1;
  std::vector<LevelD> lv;
  int nc = 0;               // active unknowns on the coarsest level
  double* lu = nullptr;     // batch x nc x nc
  int32_t* perm = nullptr;  // batch x nc
  int32_t* actp = nullptr;  // nc flat indices of active coarsest points
  double slope = 0.01;
  int version = 0;          // bumped whenever smoother kernels are (re)installed
  int compact = 1;          // use band-class tables where they represent a table exactly
  int classed_only = 0;     // built from band-class tables: no per-point planes exist
  int64_t stream_min = 1000000;   // row-streaming passes on levels with at least this many points
                                  // (batch x rows x cols); smaller levels use tile passes
  int tile = 1;                   // 1: tile-local fused passes below stream_min; 0: separate kernels
  int stream_kernel = 0;          // 0 auto, 1 one-column streaming kernel, 2 column-pair kernel, 3 warp-strip kernel
  int64_t coarse_max = 0;         // levels up to this many points run in the single-launch
                                  // shared-memory coarse cycle (0 disables it)
  int fused = 2;            // 2: one fused pass per smoothing phase; 1: one fused pass per sweep;
                            // 0: separate sweep / restriction / prolongation kernels
  ~mgb_hier() {
    DeviceGuard dg(device);
    for (auto& l : lv) {
      dfree(l.A);
      if (l.K == l.Kcls) l.K = nullptr;
      dfree(l.K);
      dfree(l.mask);
      dfree(l.Acls);
      dfree(l.Kcls);
    }
    dfree(lu);
    dfree(perm);
    dfree(actp);
  }
  Grid grid(int l) const { return Grid{batch, lv[l].rows, lv[l].cols}; }
  int depth() const { return (int)lv.size(); }
};

struct GraphKey {
  const double* f;
  double* u;
  int nu1, nu2, cycles, u_zero, mode;
  double* hist;
  bool operator==(const GraphKey& o) const {
    return f == o.f && u == o.u && nu1 == o.nu1 && nu2 == o.nu2 && cycles == o.cycles &&
           u_zero == o.u_zero && mode == o.mode && hist == o.hist;
  }
};
struct GraphEntry {
  GraphKey key;
  cudaGraphExec_t exec = nullptr;
  int64_t launches = 0;
};

struct mgb_work {
  const mgb_hier* h = nullptr;
  cudaStream_t cap = nullptr;
  std::vector<double*> u, t, f, r, v;
  double* partials = nullptr;
  int max_nblk = 0;
  double* fnorm2 = nullptr;   // batch
  double* scratch = nullptr;  // batch x 4 (solve history slots)
  double *hf = nullptr, *hu = nullptr, *hh = nullptr;  // host-call staging (level 0 f, u, history)
  int64_t hh_cap = 0;
  // second staging set + copy streams / events of the pipelined host call
  double *hf2 = nullptr, *hu2 = nullptr, *hh2 = nullptr;
  double* hist_pinned = nullptr;  // pinned host staging of the histories (pageable copies would block)
  int64_t hist_pinned_cap = 0;
  cudaStream_t cin = nullptr, cout = nullptr;
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
  // padded copies of level 0 (pad_layout, mgb_stream.h) for the warp-strip passes of a
  // run_cycles solve: f, u and the ping-pong partner; pad0 is set while such a solve is
  // enqueued (stream_args / vcycle_rec then address level 0 through them)
  double *pf0 = nullptr, *pu0 = nullptr, *pt0 = nullptr;
  bool pad0 = false;
  // padded buffers of the levels >= 1 that a warp-strip parent feeds (level_padded): f, u and the
  // ping-pong partner; vcycle_rec / stream_args recognise them by address
  std::vector<double*> pf, pu, pt;
  double* plain_out = nullptr;   // while enqueuing the last cycle of a padded run_cycles solve: the caller's u
  std::vector<GraphEntry> graphs;
  int graph_version = -1;   // hierarchy version the cached graphs were captured against
  int64_t last_launches = 0;
  ~mgb_work() {
    DeviceGuard dg(h ? h->device : -1);
    for (auto& g : graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    for (auto* vec : {&u, &t, &f, &r, &v})
      for (auto*& p : *vec) dfree(p);
    dfree(partials);
    dfree(fnorm2);
    dfree(scratch);
    dfree(hf);
    dfree(hu);
    dfree(hh);
    dfree(hf2);
    dfree(hu2);
    dfree(hh2);
    for (double** p : {&pf0, &pu0, &pt0})
      if (*p) {
        double* base = *p - pad_offset(h->lv[0].cols);
        dfree(base);
        *p = nullptr;
      }
    for (auto* vec : {&pf, &pu, &pt})
      for (size_t l = 0; l < vec->size(); ++l)
        if ((*vec)[l]) {
          double* base = (*vec)[l] - pad_offset(h->lv[l].cols);
          dfree(base);
          (*vec)[l] = nullptr;
        }
    if (hist_pinned) cudaFreeHost(hist_pinned);
    for (int b = 0; b < 2; ++b)
      for (cudaEvent_t e : {ev_in[b], ev_done[b], ev_out[b]})
        if (e) cudaEventDestroy(e);
    if (cin) cudaStreamDestroy(cin);
    if (cout) cudaStreamDestroy(cout);
    if (cap) cudaStreamDestroy(cap);
  }
};

static cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
int prepare_work(mgb_work* w);  // sizes per-solve scratch before any capture

static Tab tabA(const mgb_hier* h, const LevelD& l) {
  return h->classed_only ? tab_cls(l.Acls, l.rows, l.cols, 1) : tab_soa(l.A, l.n, 1);
}
static Tab tabK(const mgb_hier* h, const LevelD& l) {
  return h->classed_only ? tab_cls(l.Kcls, l.rows, l.cols, l.ks) : tab_soa(l.K, l.n, l.ks);
}



// ---------------------------------------------------------------------------
// library / errors

extern "C" int mgb_version(void) { return 1; }
extern "C" const char* mgb_last_error(void) { return g_err.c_str(); }
extern "C" int mgb_last_pivot(void) { return g_pivot; }

extern "C" int mgb_device_info(int device, int* sm_count, int* cc_major, int* cc_minor) {
  int cnt = 0;
  cudaError_t e = cudaGetDeviceCount(&cnt);
  if (e != cudaSuccess || cnt == 0) return fail(MGB_CUDA, "no CUDA device available");
  if (device < 0 || device >= cnt) return fail(MGB_CONFIG, "device index out of range");
  cudaDeviceProp pr;
  MGB_CUDA_TRY(cudaGetDeviceProperties(&pr, device));
  if (sm_count) *sm_count = pr.multiProcessorCount;
  if (cc_major) *cc_major = pr.major;
  if (cc_minor) *cc_minor = pr.minor;
  return MGB_OK;
}

static int check_dims(int batch, int rows, int cols) {
  if (batch < 1) return fail(MGB_CONTRACT, "batch must be positive");
  if (rows < 1 || cols < 1) return fail(MGB_CONTRACT, "grid dimensions must be positive");
  if ((int64_t)rows * cols > (int64_t)1 << 34) return fail(MGB_CONTRACT, "grid too large");
  return MGB_OK;
}

// ---------------------------------------------------------------------------
// stateless ops (reference layouts)

extern "C" int mgb_apply_stencil(int batch, int rows, int cols, int k, const double* A_dev,
                                 const uint8_t* mask_dev, const double* u_dev, double* out_dev,
                                 void* stream) {
  if (int st = check_dims(batch, rows, cols)) return st;
  if (k != 1 && k != 3) return fail(MGB_CONTRACT, "apply_stencil supports k = 1 or 3");
  Grid g{batch, rows, cols};
  Tab A = k == 3 ? tab_aos(A_dev, g.n(), 1) : Tab{A_dev, g.n(), 1, 0, 1};
  MGB_CUDA_TRY(launch_apply(g, k, A, mask_dev, u_dev, out_dev, S(stream)));
  return MGB_OK;
}

extern "C" int mgb_restrict(int batch, int rows, int cols, const uint8_t* mask_c_dev,
                            const double* fine_dev, double* coarse_dev, void* stream) {
  if (int st = check_dims(batch, rows, cols)) return st;
  if (rows / 2 < 1 || cols / 2 < 1) return fail(MGB_CONFIG, "grid cannot be coarsened further");
  Grid g{batch, rows, cols};
  MGB_CUDA_TRY(launch_restrict(g, mask_c_dev, fine_dev, coarse_dev, S(stream)));
  return MGB_OK;
}

extern "C" int mgb_prolong(int batch, int rows, int cols, const uint8_t* mask_f_dev,
                           const double* coarse_dev, double* fine_dev, void* stream) {
  if (int st = check_dims(batch, rows, cols)) return st;
  if (rows / 2 < 1 || cols / 2 < 1) return fail(MGB_CONFIG, "grid cannot be coarsened further");
  Grid g{batch, rows, cols};
  MGB_CUDA_TRY(launch_prolong(g, mask_f_dev, coarse_dev, fine_dev, false, S(stream)));
  return MGB_OK;
}

extern "C" int mgb_galerkin_product(int batch, int rows, int cols, int k, const double* A_dev,
                                    const uint8_t* mask_f_dev, const uint8_t* mask_c_dev,
                                    double* Ac_dev, int* k_out, void* stream) {
  if (int st = check_dims(batch, rows, cols)) return st;
  if (k != 3) return fail(MGB_CONTRACT, "galerkin_product supports 3x3 fine stencils");
  if (rows / 2 < 1 || cols / 2 < 1) return fail(MGB_CONFIG, "grid cannot be coarsened further");
  Grid g{batch, rows, cols};
  const int64_t nc = (int64_t)(rows / 2) * (cols / 2);
  int* ring = nullptr;
  MGB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&ring), sizeof(int), S(stream)));
  MGB_CUDA_TRY(cudaMemsetAsync(ring, 0, sizeof(int), S(stream)));
  MGB_CUDA_TRY(launch_galerkin(g, tab_aos(A_dev, g.n(), 1), mask_f_dev, mask_c_dev,
                               tabw_aos(Ac_dev, nc, 1), ring, S(stream)));
  int hr = 0;
  MGB_CUDA_TRY(cudaMemcpyAsync(&hr, ring, sizeof(int), cudaMemcpyDeviceToHost, S(stream)));
  MGB_CUDA_TRY(cudaFreeAsync(ring, S(stream)));
  MGB_CUDA_TRY(cudaStreamSynchronize(S(stream)));
  if (k_out) *k_out = hr ? 3 : 1;
  return MGB_OK;
}

// out = M(r) for a kst-stage smoother whose kernels are in table K
static int smoother_apply_tab(const Grid& g, int kst, Tab K, const uint8_t* mask, double slope,
                              const double* r, double* out, double* tmp1, double* tmp2,
                              const double* base, cudaStream_t s) {
  const double* in = r;
  for (int st = 0; st < kst; ++st) {
    const bool last = st == kst - 1;
    double* dst = last ? out : ((st & 1) ? tmp2 : tmp1);
    MGB_CUDA_TRY(launch_pointwise(g, K, st, mask, in, st > 0, slope, last ? base : nullptr, dst, s));
    in = dst;
  }
  return MGB_OK;
}

extern "C" int mgb_smoother_apply(int batch, int rows, int cols, int kst, const double* K_dev,
                                  const uint8_t* mask_dev, double slope, const double* r_dev,
                                  double* out_dev, void* stream) {
  if (int st = check_dims(batch, rows, cols)) return st;
  if (kst < 1) return fail(MGB_CONTRACT, "smoother needs at least one stage");
  Grid g{batch, rows, cols};
  double *t1 = nullptr, *t2 = nullptr;
  const size_t bytes = sizeof(double) * g.n() * batch;
  if (kst > 1) {
    MGB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&t1), bytes, S(stream)));
    MGB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&t2), bytes, S(stream)));
  }
  int st = smoother_apply_tab(g, kst, tab_aos(K_dev, g.n(), kst), mask_dev, slope, r_dev, out_dev,
                              t1, t2, nullptr, S(stream));
  if (t1) cudaFreeAsync(t1, S(stream));
  if (t2) cudaFreeAsync(t2, S(stream));
  return st;
}

static int upload_weights(int variant, int kst, const double* w_host, int64_t nw, double** w_dev,
                          cudaStream_t s) {
  if (variant != MGB_NET_CONV && variant != MGB_NET_FC)
    return fail(MGB_CONFIG, "unknown net variant");
  if (kst < 1 || kst > 4) return fail(MGB_CONFIG, "inference supports 1 <= k <= 4 stages");
  if (nw != net_weight_count(variant, kst))
    return fail(MGB_CONFIG, "weight count does not match the net architecture");
  for (int64_t q = 0; q < nw; ++q)
    if (!std::isfinite(w_host[q])) return fail(MGB_NUMERIC, "non-finite net weights");
  MGB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(w_dev), sizeof(double) * nw, s));
  MGB_CUDA_TRY(cudaMemcpyAsync(*w_dev, w_host, sizeof(double) * nw, cudaMemcpyHostToDevice, s));
  return MGB_OK;
}

extern "C" int mgb_infer_kernels(int batch, int rows, int cols, const double* A_dev,
                                 const uint8_t* mask_dev, int variant, int kst,
                                 const double* weights_host, int64_t n_weights, double slope,
                                 int precision, double* K_dev, void* stream) {
  if (int st = check_dims(batch, rows, cols)) return st;
  if (precision != 32 && precision != 64) return fail(MGB_CONFIG, "precision must be 32 or 64");
  double* w = nullptr;
  if (int st = upload_weights(variant, kst, weights_host, n_weights, &w, S(stream))) return st;
  Grid g{batch, rows, cols};
  cudaError_t e = launch_infer(g, tab_aos(A_dev, g.n(), 1), mask_dev, variant, kst, w, slope,
                               precision, tabw_aos(K_dev, g.n(), kst), S(stream));
  cudaFreeAsync(w, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "launch_infer");
  return MGB_OK;
}

extern "C" int mgb_lu_factor(int n, double* lu_dev, int32_t* perm_dev, void* stream) {
  if (n < 1 || n > 4096) return fail(MGB_CONFIG, "dense LU supports 1 <= n <= 4096");
  int* st = nullptr;
  MGB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&st), sizeof(int), S(stream)));
  MGB_CUDA_TRY(launch_lu_factor(1, n, lu_dev, perm_dev, st, S(stream)));
  int hs = -1;
  MGB_CUDA_TRY(cudaMemcpyAsync(&hs, st, sizeof(int), cudaMemcpyDeviceToHost, S(stream)));
  MGB_CUDA_TRY(cudaFreeAsync(st, S(stream)));
  MGB_CUDA_TRY(cudaStreamSynchronize(S(stream)));
  if (hs >= 0) {
    set_error(MGB_SINGULAR, "singular to working precision at pivot " + std::to_string(hs), hs);
    return MGB_SINGULAR;
  }
  return MGB_OK;
}

extern "C" int mgb_lu_solve(int n, const double* lu_dev, const int32_t* perm_dev,
                            const double* b_dev, double* x_dev, void* stream) {
  if (n < 1 || n > 4096) return fail(MGB_CONFIG, "dense LU supports 1 <= n <= 4096");
  MGB_CUDA_TRY(launch_lu_solve_vec(n, lu_dev, perm_dev, b_dev, x_dev, S(stream)));
  return MGB_OK;
}

// ---------------------------------------------------------------------------
// hierarchy

static int64_t count_active(const std::vector<uint8_t>& m) {
  int64_t c = 0;
  for (uint8_t x : m) c += x != 0;
  return c;
}

// flat index of the first point of each band class (-1 if the class is empty)
static void class_reps(int rows, int cols, int64_t rep[25]) {
  for (int c = 0; c < 25; ++c) rep[c] = -1;
  int ri[5], rj[5];
  for (int c = 0; c < 5; ++c) ri[c] = rj[c] = -1;
  for (int i = rows - 1; i >= 0; --i) ri[host_band(i, rows)] = i;
  for (int j = cols - 1; j >= 0; --j) rj[host_band(j, cols)] = j;
  for (int a = 0; a < 5; ++a)
    for (int b = 0; b < 5; ++b)
      if (ri[a] >= 0 && rj[b] >= 0) rep[a * 5 + b] = (int64_t)ri[a] * cols + rj[b];
}

// Band-class compaction (mgb_cycle.cu): if every point of the table equals its
// class representative, keep the 25 class tables (exact) for the hot loop.
static int classify_table(mgb_hier* h, int l, const double* planes, int ks, double** cls_out, cudaStream_t s,
                          std::vector<double>* host_copy = nullptr) {
  if (h->classed_only) return MGB_OK;
  dfree(*cls_out);
  LevelD& lv = h->lv[l];
  if (!h->compact || lv.mask || !planes) return MGB_OK;
  int64_t rep[25];
  for (int c = 0; c < 25; ++c) rep[c] = -1;
  for (int i = 0; i < lv.rows; ++i)
    for (int j = 0; j < lv.cols; ++j) {
      const int c = host_band(i, lv.rows) * 5 + host_band(j, lv.cols);
      if (rep[c] < 0) rep[c] = (int64_t)i * lv.cols + j;
      if (i > 2 && i < lv.rows - 3 && j > 2) j = std::max(j, lv.cols - 4);  // skip the interior
    }
  int64_t* drep = nullptr;
  int* flag = nullptr;
  MGB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&drep), sizeof(rep), s));
  MGB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&flag), sizeof(int), s));
  MGB_CUDA_TRY(cudaMemcpyAsync(drep, rep, sizeof(rep), cudaMemcpyHostToDevice, s));
  MGB_CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int), s));
  const Op T{planes, nullptr, lv.n, ks};
  MGB_CUDA_TRY(launch_classify(h->grid(l), T, drep, flag, s));
  int hf = 1;
  MGB_CUDA_TRY(cudaMemcpyAsync(&hf, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  MGB_CUDA_TRY(cudaStreamSynchronize(s));
  if (!hf) {
    MGB_CUDA_TRY(dalloc(cls_out, (size_t)h->batch * 25 * ks * 9));
    MGB_CUDA_TRY(launch_gather_cls(h->grid(l), T, drep, *cls_out, s));
    if (host_copy && ks == 1) {
      host_copy->assign((size_t)h->batch * 225, 0.0);
      MGB_CUDA_TRY(cudaMemcpyAsync(host_copy->data(), *cls_out, host_copy->size() * sizeof(double),
                                   cudaMemcpyDeviceToHost, s));
    }
  }
  MGB_CUDA_TRY(cudaFreeAsync(drep, s));
  MGB_CUDA_TRY(cudaFreeAsync(flag, s));
  MGB_CUDA_TRY(cudaStreamSynchronize(s));
  return MGB_OK;
}

// Per-point A whose corner planes are zero everywhere (a 5-point operator such as
// config 3's cell-centred diffusion): the streaming passes skip those loads.
static int check_corners(mgb_hier* h, int l, cudaStream_t s) {
  LevelD& lv = h->lv[l];
  lv.a5 = false;
  if (!lv.A || lv.Acls) return MGB_OK;
  int* flag = nullptr;
  MGB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&flag), sizeof(int), s));
  MGB_CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int), s));
  MGB_CUDA_TRY(launch_corner_check(lv.n, h->batch, lv.A, flag, s));
  int hf = 1;
  MGB_CUDA_TRY(cudaMemcpyAsync(&hf, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  MGB_CUDA_TRY(cudaFreeAsync(flag, s));
  MGB_CUDA_TRY(cudaStreamSynchronize(s));
  lv.a5 = hf == 0;
  return MGB_OK;
}

static int classify_all(mgb_hier* h, cudaStream_t s) {
  for (int l = 0; l < h->depth(); ++l) {
    LevelD& lv = h->lv[l];
    if (int st = classify_table(h, l, lv.A, 1, &lv.Acls, s, &lv.hAcls)) return st;
    if (int st = check_corners(h, l, s)) return st;
    if (lv.K) {
      if (int st = classify_table(h, l, lv.K, lv.ks, &lv.Kcls, s, &lv.hKcls)) return st;
    } else {
      dfree(lv.Kcls);
    }
  }
  ++h->version;
  return MGB_OK;
}

extern "C" int mgb_hier_build(int device, int batch, int rows, int cols, double spacing,
                              const double* A0, int a0_on_device, const uint8_t* mask_host,
                              int levels, void* stream, mgb_hier** out) {
  if (!out) return fail(MGB_CONTRACT, "null output handle");
  *out = nullptr;
  if (int st = check_dims(batch, rows, cols)) return st;
  if (!(spacing > 0.0)) return fail(MGB_CONTRACT, "grid spacing must be positive");
  if (levels < 2) return fail(MGB_CONFIG, "a hierarchy needs at least two levels");
  int cnt = 0;
  if (cudaGetDeviceCount(&cnt) != cudaSuccess || cnt == 0)
    return fail(MGB_CUDA, "no CUDA device available");
  if (device < 0 || device >= cnt) return fail(MGB_CONFIG, "device index out of range");
  DeviceGuard dg(device);
  cudaStream_t s = S(stream);

  std::unique_ptr<mgb_hier> h(new mgb_hier());
  h->device = device;
  h->batch = batch;
  // level geometry + masks on the host (coarsen_full, transfer.py:50-61)
  const bool has_mask = mask_host != nullptr;
  {
    LevelD l0;
    l0.rows = rows;
    l0.cols = cols;
    l0.h = spacing;
    l0.n = (int64_t)rows * cols;
    l0.k = 3;
    l0.hmask.assign(mask_host ? mask_host : nullptr, mask_host ? mask_host + l0.n : nullptr);
    if (!has_mask) l0.hmask.assign(l0.n, 1);
    l0.nact = count_active(l0.hmask);
    if (l0.nact == 0) return fail(MGB_CONTRACT, "grid has no active points");
    h->lv.push_back(std::move(l0));
  }
  for (int step = 0; step < levels - 1; ++step) {
    const LevelD& f = h->lv.back();
    LevelD c;
    c.rows = f.rows / 2;
    c.cols = f.cols / 2;
    if (c.rows < 1 || c.cols < 1)
      return fail(MGB_CONFIG, "level " + std::to_string(step) + ": " + std::to_string(f.rows) + "x" +
                                  std::to_string(f.cols) + " grid cannot be coarsened further");
    c.h = 2.0 * f.h;
    c.n = (int64_t)c.rows * c.cols;
    c.hmask.resize(c.n);
    for (int i = 0; i < c.rows; ++i)
      for (int j = 0; j < c.cols; ++j)
        c.hmask[(int64_t)i * c.cols + j] = f.hmask[(int64_t)(2 * i + 1) * f.cols + (2 * j + 1)];
    c.nact = count_active(c.hmask);
    if (c.nact == 0)
      return fail(MGB_CONFIG, "level " + std::to_string(step) + ": coarsening left no active points");
    if (c.nact >= f.nact)
      return fail(MGB_CONFIG, "level " + std::to_string(step) + ": coarsening does not shrink the active set");
    h->lv.push_back(std::move(c));
  }
  const int L = h->depth();
  const LevelD& lc = h->lv[L - 1];
  if (lc.nact > 4096)
    return fail(MGB_CONFIG, "coarsest level has " + std::to_string(lc.nact) +
                                " unknowns; the dense direct solve supports at most 4096 (add levels)");
  // non-finite input check (StencilField, grid.py:182-183)
  if (!a0_on_device) {
    const int64_t tot = (int64_t)batch * h->lv[0].n * 9;
    for (int64_t q = 0; q < tot; ++q)
      if (!std::isfinite(A0[q])) return fail(MGB_NUMERIC, "non-finite stencil weights");
  }
  // device allocations
  for (auto& l : h->lv) {
    MGB_CUDA_TRY(dalloc(&l.A, (size_t)batch * 9 * l.n));
    if (has_mask) {
      MGB_CUDA_TRY(dalloc(&l.mask, (size_t)l.n));
      MGB_CUDA_TRY(cudaMemcpyAsync(l.mask, l.hmask.data(), l.n, cudaMemcpyHostToDevice, s));
    }
  }
  // level 0: reference AoS -> planes
  {
    LevelD& l0 = h->lv[0];
    const double* src = A0;
    double* tmp = nullptr;
    if (!a0_on_device) {
      MGB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&tmp), sizeof(double) * batch * 9 * l0.n, s));
      MGB_CUDA_TRY(cudaMemcpyAsync(tmp, A0, sizeof(double) * batch * 9 * l0.n, cudaMemcpyHostToDevice, s));
      src = tmp;
    }
    MGB_CUDA_TRY(launch_convert(h->grid(0), 1, tab_aos(src, l0.n, 1), tabw_soa(l0.A, l0.n, 1), s));
    if (tmp) MGB_CUDA_TRY(cudaFreeAsync(tmp, s));
  }
  // Galerkin chain (transfer.py:150-209) with the _trim ring test
  int* ring = nullptr;
  MGB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&ring), sizeof(int) * L, s));
  MGB_CUDA_TRY(cudaMemsetAsync(ring, 0, sizeof(int) * L, s));
  for (int l = 0; l + 1 < L; ++l) {
    LevelD& f = h->lv[l];
    LevelD& c = h->lv[l + 1];
    MGB_CUDA_TRY(launch_galerkin(h->grid(l), tab_soa(f.A, f.n, 1), f.mask, c.mask,
                                 tabw_soa(c.A, c.n, 1), ring + l + 1, s));
  }
  std::vector<int> hring(L, 1);
  MGB_CUDA_TRY(cudaMemcpyAsync(hring.data(), ring, sizeof(int) * L, cudaMemcpyDeviceToHost, s));
  MGB_CUDA_TRY(cudaFreeAsync(ring, s));
  MGB_CUDA_TRY(cudaStreamSynchronize(s));
  for (int l = 1; l < L; ++l) h->lv[l].k = hring[l] ? 3 : 1;
  // coarsest: materialise over active points and LU-factor (hierarchy.py:87)
  {
    LevelD& c = h->lv[L - 1];
    const int nc = (int)c.nact;
    h->nc = nc;
    std::vector<int32_t> idx(c.n, -1), actp(nc);
    int a = 0;
    for (int64_t p = 0; p < c.n; ++p)
      if (c.hmask[p]) { idx[p] = a; actp[a] = (int32_t)p; ++a; }
    int32_t* didx = nullptr;
    int* dst = nullptr;
    MGB_CUDA_TRY(dalloc(&h->actp, nc));
    MGB_CUDA_TRY(dalloc(&h->lu, (size_t)batch * nc * nc));
    MGB_CUDA_TRY(dalloc(&h->perm, (size_t)batch * nc));
    MGB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&didx), sizeof(int32_t) * c.n, s));
    MGB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&dst), sizeof(int) * batch, s));
    MGB_CUDA_TRY(cudaMemcpyAsync(didx, idx.data(), sizeof(int32_t) * c.n, cudaMemcpyHostToDevice, s));
    MGB_CUDA_TRY(cudaMemcpyAsync(h->actp, actp.data(), sizeof(int32_t) * nc, cudaMemcpyHostToDevice, s));
    MGB_CUDA_TRY(cudaMemsetAsync(h->lu, 0, sizeof(double) * batch * nc * nc, s));
    MGB_CUDA_TRY(launch_materialize(h->grid(L - 1), tab_soa(c.A, c.n, 1), didx, nc, h->actp, h->lu, s));
    MGB_CUDA_TRY(launch_lu_factor(batch, nc, h->lu, h->perm, dst, s));
    std::vector<int> hs(batch);
    MGB_CUDA_TRY(cudaMemcpyAsync(hs.data(), dst, sizeof(int) * batch, cudaMemcpyDeviceToHost, s));
    MGB_CUDA_TRY(cudaFreeAsync(didx, s));
    MGB_CUDA_TRY(cudaFreeAsync(dst, s));
    MGB_CUDA_TRY(cudaStreamSynchronize(s));
    for (int b = 0; b < batch; ++b)
      if (hs[b] >= 0) {
        set_error(MGB_SINGULAR, "coarsest operator singular to working precision at pivot " +
                                    std::to_string(hs[b]) + " (problem " + std::to_string(b) + ")",
                  hs[b]);
        return MGB_SINGULAR;
      }
  }
  if (const char* e = getenv("MGB_STORAGE")) h->compact = std::string(e) != "planes";
  if (const char* e = getenv("MGB_FUSED")) h->fused = atoi(e);
  if (const char* e = getenv("MGB_STREAM_MIN")) h->stream_min = atoll(e);
  if (const char* e = getenv("MGB_TILE")) h->tile = atoi(e);
  if (const char* e = getenv("MGB_COARSE_MAX")) h->coarse_max = atoll(e);
  if (int st = classify_all(h.get(), s)) return st;
  *out = h.release();
  return MGB_OK;
}

extern "C" int mgb_hier_set_storage(mgb_hier* h, int mode, void* stream) {
  if (!h) return fail(MGB_CONTRACT, "null hierarchy");
  if (mode != 0 && mode != 1) return fail(MGB_CONFIG, "storage mode must be 0 (auto) or 1 (per-point planes)");
  if (h->classed_only) {
    if (mode == 1) return fail(MGB_CONFIG, "a band-class hierarchy has no per-point planes");
    return MGB_OK;
  }
  DeviceGuard dg(h->device);
  h->compact = mode == 0;
  return classify_all(h, S(stream));
}

extern "C" int mgb_hier_set_fused(mgb_hier* h, int enable) {
  if (!h) return fail(MGB_CONTRACT, "null hierarchy");
  h->fused = enable < 0 ? 0 : (enable > 2 ? 2 : enable);
  ++h->version;
  return MGB_OK;
}

extern "C" int mgb_hier_set_stream_kernel(mgb_hier* h, int kind) {
  if (!h) return fail(MGB_CONTRACT, "null hierarchy");
  if (kind < 0 || kind > 3) return fail(MGB_CONFIG, "stream kernel must be 0 (auto), 1, 2 or 3");
  h->stream_kernel = kind;
  ++h->version;
  return MGB_OK;
}

extern "C" int mgb_hier_set_passes(mgb_hier* h, int64_t stream_min, int tile, int64_t coarse_max) {
  if (!h) return fail(MGB_CONTRACT, "null hierarchy");
  if (stream_min >= 0) h->stream_min = stream_min;
  if (tile >= 0) h->tile = tile ? 1 : 0;
  if (coarse_max >= 0) h->coarse_max = coarse_max;
  ++h->version;
  return MGB_OK;
}

extern "C" int mgb_hier_set_conv_smoother(mgb_hier* h, int level, int nl, const double* layers_host,
                                          const double* skip_host, int leaky, double slope, double gain) {
  if (!h) return fail(MGB_CONTRACT, "null hierarchy");
  if (level < 0 || level + 1 >= h->depth()) return fail(MGB_CONFIG, "level has no smoother slot");
  if (nl < 1 || nl > CONV_MAX_LAYERS) return fail(MGB_CONFIG, "conv smoother needs 1..8 layers");
  if (!layers_host) return fail(MGB_CONTRACT, "null layer weights");
  DeviceGuard dg(h->device);
  LevelD& l = h->lv[level];
  ConvSm cs;
  cs.nl = nl;
  for (int q = 0; q < nl; ++q)
    for (int o = 0; o < 9; ++o) cs.layer[q].w[o] = layers_host[q * 9 + o];
  cs.has_skip = skip_host != nullptr;
  if (skip_host)
    for (int o = 0; o < 9; ++o) cs.skip.w[o] = skip_host[o];
  cs.leaky = leaky != 0;
  cs.slope = slope;
  cs.gain = gain;
  for (int q = 0; q < nl * 9; ++q)
    if (!std::isfinite(layers_host[q])) return fail(MGB_NUMERIC, "non-finite kernel weights");
  if (!std::isfinite(gain)) return fail(MGB_NUMERIC, "non-finite gain");
  if (l.K == l.Kcls) l.K = nullptr;
  dfree(l.K);
  dfree(l.Kcls);
  l.ks = 0;
  l.conv = cs;
  ++h->version;
  return MGB_OK;
}

extern "C" int mgb_convolve(int batch, int rows, int cols, const double* w_host, const uint8_t* mask_dev,
                            const double* u_dev, double* out_dev, void* stream) {
  if (int st = check_dims(batch, rows, cols)) return st;
  if (!w_host) return fail(MGB_CONTRACT, "null kernel");
  ConvW w;
  for (int o = 0; o < 9; ++o) w.w[o] = w_host[o];
  MGB_CUDA_TRY(launch_convolve(Grid{batch, rows, cols}, w, mask_dev, u_dev, out_dev, false, 0.0, S(stream)));
  return MGB_OK;
}

extern "C" int mgb_conv_smoother_apply(int batch, int rows, int cols, int nl, const double* layers_host,
                                       const double* skip_host, int leaky, double slope, double gain,
                                       const uint8_t* mask_dev, const double* r_dev, double* out_dev, void* stream) {
  if (int st = check_dims(batch, rows, cols)) return st;
  if (nl < 1 || nl > CONV_MAX_LAYERS || !layers_host) return fail(MGB_CONFIG, "conv smoother needs 1..8 layers");
  ConvSm cs;
  cs.nl = nl;
  for (int q = 0; q < nl; ++q)
    for (int o = 0; o < 9; ++o) cs.layer[q].w[o] = layers_host[q * 9 + o];
  cs.has_skip = skip_host != nullptr;
  if (skip_host)
    for (int o = 0; o < 9; ++o) cs.skip.w[o] = skip_host[o];
  cs.leaky = leaky != 0;
  cs.slope = slope;
  cs.gain = gain;
  const Grid g{batch, rows, cols};
  double *t1 = nullptr, *t2 = nullptr;
  const size_t bytes = sizeof(double) * g.n() * batch;
  MGB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&t1), bytes, S(stream)));
  MGB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&t2), bytes, S(stream)));
  cudaError_t e = conv_smoother_apply(g, cs, mask_dev, r_dev, nullptr, out_dev, t1, t2, S(stream));
  cudaFreeAsync(t1, S(stream));
  cudaFreeAsync(t2, S(stream));
  MGB_CUDA_TRY(e);
  return MGB_OK;
}

extern "C" int mgb_hier_storage_info(const mgb_hier* h, int level, int* a_classed, int* k_classed) {
  if (!h) return fail(MGB_CONTRACT, "null hierarchy");
  if (level < 0 || level >= h->depth()) return fail(MGB_CONFIG, "level out of range");
  if (a_classed) *a_classed = h->lv[level].Acls != nullptr;
  if (k_classed) *k_classed = h->lv[level].Kcls != nullptr;
  return MGB_OK;
}

extern "C" int mgb_hier_stencil_points(const mgb_hier* h, int level, int* a_points) {
  if (!h || !a_points) return fail(MGB_CONTRACT, "null argument");
  if (level < 0 || level >= h->depth()) return fail(MGB_CONFIG, "level out of range");
  const LevelD& lv = h->lv[level];
  *a_points = lv.Acls || !lv.A ? 0 : (lv.a5 ? 5 : 9);
  return MGB_OK;
}

extern "C" int mgb_hier_level_uniformity(const mgb_hier* h, int level, int* uniformity) {
  if (!h || !uniformity) return fail(MGB_CONTRACT, "null argument");
  if (level < 0 || level >= h->depth()) return fail(MGB_CONFIG, "level out of range");
  *uniformity = h->lv[level].uniformity();
  return MGB_OK;
}

// forward declarations (defined with the cycle code below)
static int pass_kind(const mgb_hier* h, int l, int nu1, int nu2);

extern "C" int mgb_hier_pass_kernel(const mgb_hier* h, int level, int nu, int* kind) {
  if (!h || !kind) return fail(MGB_CONTRACT, "null argument");
  if (level < 0 || level + 1 >= h->depth()) return fail(MGB_CONFIG, "level out of range");
  const int pk = pass_kind(h, level, nu, nu);
  if (pk == 0) {
    *kind = 0;
  } else if (pk == 2) {
    *kind = 4;
  } else {
    const LevelD& lv = h->lv[level];
    StreamArgs a{};
    a.g = h->grid(level);
    a.A = lv.opA();
    a.K = lv.opK();
    a.mask = lv.mask;
    a.ci_valid = h->batch == 1 && lv.Acls && lv.Kcls;
    a.uniform = lv.uniformity();
    a.kernel = h->stream_kernel;
    *kind = stream_kernel_kind(a, nu);
  }
  return MGB_OK;
}

// Constant-coefficient hierarchy held entirely as band-class tables (no per-point
// planes): the Galerkin product and the coarsest materialisation read the fine
// tables through the class accessor and evaluate one representative point per
// coarse class.  Memory is O(grid functions) only, so 32767^2 (config 5) fits one GPU.
extern "C" int mgb_hier_build_classed(int device, int batch, int rows, int cols, double spacing,
                                      const double* cls_host, int levels, void* stream, mgb_hier** out) {
  if (!out) return fail(MGB_CONTRACT, "null output handle");
  *out = nullptr;
  if (int st = check_dims(batch, rows, cols)) return st;
  if (!(spacing > 0.0)) return fail(MGB_CONTRACT, "grid spacing must be positive");
  if (levels < 2) return fail(MGB_CONFIG, "a hierarchy needs at least two levels");
  int cnt = 0;
  if (cudaGetDeviceCount(&cnt) != cudaSuccess || cnt == 0) return fail(MGB_CUDA, "no CUDA device available");
  if (device < 0 || device >= cnt) return fail(MGB_CONFIG, "device index out of range");
  for (int64_t q = 0; q < (int64_t)batch * 225; ++q)
    if (!std::isfinite(cls_host[q])) return fail(MGB_NUMERIC, "non-finite stencil weights");
  DeviceGuard dg(device);
  cudaStream_t s = S(stream);
  std::unique_ptr<mgb_hier> h(new mgb_hier());
  h->device = device;
  h->batch = batch;
  h->classed_only = 1;
  int r = rows, c = cols;
  double sp = spacing;
  for (int l = 0; l < levels; ++l) {
    if (r < 1 || c < 1)
      return fail(MGB_CONFIG, "level " + std::to_string(l - 1) + ": grid cannot be coarsened further");
    LevelD lv;
    lv.rows = r;
    lv.cols = c;
    lv.h = sp;
    lv.n = (int64_t)r * c;
    lv.k = 3;
    lv.nact = lv.n;
    h->lv.push_back(std::move(lv));
    r /= 2;
    c /= 2;
    sp *= 2.0;
  }
  const int L = h->depth();
  if (h->lv[L - 1].n > 4096) return fail(MGB_CONFIG, "coarsest level too large for the dense direct solve (add levels)");
  for (auto& lv : h->lv) MGB_CUDA_TRY(dalloc(&lv.Acls, (size_t)batch * 225));
  MGB_CUDA_TRY(cudaMemcpyAsync(h->lv[0].Acls, cls_host, sizeof(double) * batch * 225, cudaMemcpyHostToDevice, s));
  int* ring = nullptr;
  int64_t* drep = nullptr;
  MGB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&ring), sizeof(int) * L, s));
  MGB_CUDA_TRY(cudaMemsetAsync(ring, 0, sizeof(int) * L, s));
  MGB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&drep), sizeof(int64_t) * 25 * L, s));
  for (int l = 0; l + 1 < L; ++l) {
    LevelD& f = h->lv[l];
    LevelD& cl = h->lv[l + 1];
    int64_t rep[25];
    class_reps(cl.rows, cl.cols, rep);
    MGB_CUDA_TRY(cudaMemcpyAsync(drep + 25 * l, rep, sizeof(rep), cudaMemcpyHostToDevice, s));
    MGB_CUDA_TRY(cudaMemsetAsync(cl.Acls, 0, sizeof(double) * batch * 225, s));
    MGB_CUDA_TRY(launch_galerkin(h->grid(l), tab_cls(f.Acls, f.rows, f.cols, 1), nullptr, nullptr,
                                 tabw_cls(cl.Acls, cl.rows, cl.cols, 1), ring + l + 1, s, drep + 25 * l, 25));
  }
  std::vector<int> hring(L, 1);
  MGB_CUDA_TRY(cudaMemcpyAsync(hring.data(), ring, sizeof(int) * L, cudaMemcpyDeviceToHost, s));
  for (auto& lv : h->lv) {
    lv.hAcls.assign((size_t)batch * 225, 0.0);
    MGB_CUDA_TRY(cudaMemcpyAsync(lv.hAcls.data(), lv.Acls, lv.hAcls.size() * sizeof(double),
                                 cudaMemcpyDeviceToHost, s));
  }
  MGB_CUDA_TRY(cudaFreeAsync(ring, s));
  MGB_CUDA_TRY(cudaFreeAsync(drep, s));
  MGB_CUDA_TRY(cudaStreamSynchronize(s));
  for (int l = 1; l < L; ++l) h->lv[l].k = hring[l] ? 3 : 1;
  // coarsest LU (all points active)
  {
    LevelD& cl = h->lv[L - 1];
    const int nc = (int)cl.n;
    h->nc = nc;
    std::vector<int32_t> idx(cl.n), actp(nc);
    for (int q = 0; q < nc; ++q) idx[q] = actp[q] = q;
    int32_t* didx = nullptr;
    int* dst = nullptr;
    MGB_CUDA_TRY(dalloc(&h->actp, nc));
    MGB_CUDA_TRY(dalloc(&h->lu, (size_t)batch * nc * nc));
    MGB_CUDA_TRY(dalloc(&h->perm, (size_t)batch * nc));
    MGB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&didx), sizeof(int32_t) * cl.n, s));
    MGB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&dst), sizeof(int) * batch, s));
    MGB_CUDA_TRY(cudaMemcpyAsync(didx, idx.data(), sizeof(int32_t) * cl.n, cudaMemcpyHostToDevice, s));
    MGB_CUDA_TRY(cudaMemcpyAsync(h->actp, actp.data(), sizeof(int32_t) * nc, cudaMemcpyHostToDevice, s));
    MGB_CUDA_TRY(cudaMemsetAsync(h->lu, 0, sizeof(double) * batch * nc * nc, s));
    MGB_CUDA_TRY(launch_materialize(h->grid(L - 1), tab_cls(cl.Acls, cl.rows, cl.cols, 1), didx, nc, h->actp,
                                    h->lu, s));
    MGB_CUDA_TRY(launch_lu_factor(batch, nc, h->lu, h->perm, dst, s));
    std::vector<int> hs(batch);
    MGB_CUDA_TRY(cudaMemcpyAsync(hs.data(), dst, sizeof(int) * batch, cudaMemcpyDeviceToHost, s));
    MGB_CUDA_TRY(cudaFreeAsync(didx, s));
    MGB_CUDA_TRY(cudaFreeAsync(dst, s));
    MGB_CUDA_TRY(cudaStreamSynchronize(s));
    for (int b = 0; b < batch; ++b)
      if (hs[b] >= 0) {
        set_error(MGB_SINGULAR, "coarsest operator singular to working precision at pivot " + std::to_string(hs[b]),
                  hs[b]);
        return MGB_SINGULAR;
      }
  }
  if (const char* e = getenv("MGB_FUSED")) h->fused = atoi(e);
  if (const char* e = getenv("MGB_STREAM_MIN")) h->stream_min = atoll(e);
  if (const char* e = getenv("MGB_TILE")) h->tile = atoi(e);
  if (const char* e = getenv("MGB_COARSE_MAX")) h->coarse_max = atoll(e);
  *out = h.release();
  return MGB_OK;
}

extern "C" void mgb_hier_destroy(mgb_hier* h) { delete h; }

extern "C" int mgb_hier_depth(const mgb_hier* h, int* depth, int* batch) {
  if (!h) return fail(MGB_CONTRACT, "null hierarchy");
  if (depth) *depth = h->depth();
  if (batch) *batch = h->batch;
  return MGB_OK;
}

extern "C" int mgb_hier_level_info(const mgb_hier* h, int level, int* rows, int* cols, int* k,
                                   int* ks, double* spacing) {
  if (!h) return fail(MGB_CONTRACT, "null hierarchy");
  if (level < 0 || level >= h->depth()) return fail(MGB_CONFIG, "level out of range");
  const LevelD& l = h->lv[level];
  if (rows) *rows = l.rows;
  if (cols) *cols = l.cols;
  if (k) *k = l.k;
  if (ks) *ks = l.ks;
  if (spacing) *spacing = l.h;
  return MGB_OK;
}

static int download_table(const mgb_hier* h, const LevelD& l, const double* planes, int kst,
                          double* out_host) {
  DeviceGuard dg(h->device);
  double* tmp = nullptr;
  const size_t cnt = (size_t)h->batch * kst * 9 * l.n;
  MGB_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&tmp), cnt * sizeof(double)));
  Grid g{h->batch, l.rows, l.cols};
  const Tab src = h->classed_only ? tab_cls(planes, l.rows, l.cols, kst) : tab_soa(planes, l.n, kst);
  cudaError_t e = launch_convert(g, kst, src, tabw_aos(tmp, l.n, kst), nullptr);
  if (e == cudaSuccess) e = cudaMemcpy(out_host, tmp, cnt * sizeof(double), cudaMemcpyDeviceToHost);
  cudaFree(tmp);
  if (e != cudaSuccess) return cuda_fail(e, "download_table");
  return MGB_OK;
}

extern "C" int mgb_hier_get_operator(const mgb_hier* h, int level, double* out_host) {
  if (!h) return fail(MGB_CONTRACT, "null hierarchy");
  if (level < 0 || level >= h->depth()) return fail(MGB_CONFIG, "level out of range");
  const LevelD& l = h->lv[level];
  const double* tabp = h->classed_only ? l.Acls : l.A;
  if (l.k == 3) return download_table(h, l, tabp, 1, out_host);
  std::vector<double> full((size_t)h->batch * 9 * l.n);
  if (int st = download_table(h, l, tabp, 1, full.data())) return st;
  for (size_t q = 0; q < (size_t)h->batch * l.n; ++q) out_host[q] = full[q * 9 + 4];
  return MGB_OK;
}

extern "C" int mgb_hier_get_kernels(const mgb_hier* h, int level, double* out_host) {
  if (!h) return fail(MGB_CONTRACT, "null hierarchy");
  if (level < 0 || level >= h->depth()) return fail(MGB_CONFIG, "level out of range");
  const LevelD& l = h->lv[level];
  if (l.conv.nl > 0) return fail(MGB_CONFIG, "level " + std::to_string(level) + " has a convolutional smoother (no per-point kernels)");
  if (!l.K) return fail(MGB_CONFIG, "level " + std::to_string(level) + " has no smoother installed");
  return download_table(h, l, h->classed_only ? l.Kcls : l.K, l.ks, out_host);
}

extern "C" int mgb_hier_get_mask(const mgb_hier* h, int level, uint8_t* out_host) {
  if (!h) return fail(MGB_CONTRACT, "null hierarchy");
  if (level < 0 || level >= h->depth()) return fail(MGB_CONFIG, "level out of range");
  std::memcpy(out_host, h->lv[level].hmask.data(), h->lv[level].n);
  return MGB_OK;
}

extern "C" int mgb_hier_operator_planes(const mgb_hier* h, int level, const double** planes_dev) {
  if (!h) return fail(MGB_CONTRACT, "null hierarchy");
  if (level < 0 || level >= h->depth()) return fail(MGB_CONFIG, "level out of range");
  *planes_dev = h->lv[level].A;
  return MGB_OK;
}

static int alloc_kernels(mgb_hier* h, LevelD& l, int kst) {
  ++h->version;
  l.conv.nl = 0;
  if (h->classed_only) {
    if (l.Kcls && l.ks == kst) return MGB_OK;
    dfree(l.Kcls);
    l.ks = 0;
    MGB_CUDA_TRY(dalloc(&l.Kcls, (size_t)h->batch * 25 * kst * 9));
    MGB_CUDA_TRY(cudaMemset(l.Kcls, 0, sizeof(double) * h->batch * 25 * kst * 9));
    l.K = l.Kcls;  // marks the level as equipped; the hot path reads Kcls
    l.ks = kst;
    return MGB_OK;
  }
  if (l.K && l.ks == kst) return MGB_OK;
  dfree(l.K);
  l.ks = 0;
  MGB_CUDA_TRY(dalloc(&l.K, (size_t)h->batch * kst * 9 * l.n));
  l.ks = kst;
  return MGB_OK;
}

extern "C" int mgb_hier_equip_inferred(mgb_hier* h, int variant, int kst, const double* weights_host,
                                       int64_t n_weights, double slope, int precision, void* stream) {
  if (!h) return fail(MGB_CONTRACT, "null hierarchy");
  if (precision != 32 && precision != 64) return fail(MGB_CONFIG, "precision must be 32 or 64");
  for (int l = 0; l + 1 < h->depth(); ++l)
    if (h->lv[l].k != 3) return fail(MGB_CONFIG, "kernel inference needs 3x3 stencils on every level");
  DeviceGuard dg(h->device);
  cudaStream_t s = S(stream);
  double* w = nullptr;
  if (int st = upload_weights(variant, kst, weights_host, n_weights, &w, s)) return st;
  for (int l = 0; l + 1 < h->depth(); ++l) {
    LevelD& lv = h->lv[l];
    if (int st = alloc_kernels(h, lv, kst)) return st;
    cudaError_t e;
    if (h->classed_only) {
      // one evaluation per band class at its representative point
      int64_t rep[25];
      class_reps(lv.rows, lv.cols, rep);
      int64_t* drep = nullptr;
      MGB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&drep), sizeof(rep), s));
      MGB_CUDA_TRY(cudaMemcpyAsync(drep, rep, sizeof(rep), cudaMemcpyHostToDevice, s));
      e = launch_infer(h->grid(l), tabA(h, lv), nullptr, variant, kst, w, slope, precision,
                       tabw_cls(lv.Kcls, lv.rows, lv.cols, kst), s, drep, 25);
      cudaFreeAsync(drep, s);
      if (e == cudaSuccess && kst == 1) {
        lv.hKcls.assign((size_t)h->batch * 225, 0.0);
        e = cudaMemcpyAsync(lv.hKcls.data(), lv.Kcls, lv.hKcls.size() * sizeof(double), cudaMemcpyDeviceToHost, s);
      }
    } else {
      e = launch_infer(h->grid(l), tab_soa(lv.A, lv.n, 1), lv.mask, variant, kst, w, slope,
                       precision, tabw_soa(lv.K, lv.n, kst), s);
    }
    if (e != cudaSuccess) {
      cudaFreeAsync(w, s);
      return cuda_fail(e, "launch_infer");
    }
  }
  h->slope = slope;
  MGB_CUDA_TRY(cudaFreeAsync(w, s));
  MGB_CUDA_TRY(cudaStreamSynchronize(s));
  return classify_all(h, s);
}

extern "C" int mgb_hier_equip_jacobi(mgb_hier* h, double omega, void* stream) {
  if (!h) return fail(MGB_CONTRACT, "null hierarchy");
  if (!(omega > 0.0 && omega < 2.0)) return fail(MGB_CONFIG, "jacobi weight out of range");
  DeviceGuard dg(h->device);
  cudaStream_t s = S(stream);
  int* flag = nullptr;
  const int L = h->depth();
  MGB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&flag), sizeof(int) * L, s));
  MGB_CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int) * L, s));
  for (int l = 0; l + 1 < L; ++l) {
    LevelD& lv = h->lv[l];
    if (int st = alloc_kernels(h, lv, 1)) return st;
    if (h->classed_only) {
      int64_t rep[25];
      class_reps(lv.rows, lv.cols, rep);
      int64_t* drep = nullptr;
      MGB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&drep), sizeof(rep), s));
      MGB_CUDA_TRY(cudaMemcpyAsync(drep, rep, sizeof(rep), cudaMemcpyHostToDevice, s));
      MGB_CUDA_TRY(launch_jacobi(h->grid(l), tabA(h, lv), nullptr, omega, tabw_cls(lv.Kcls, lv.rows, lv.cols, 1),
                                 flag + l, s, drep, 25));
      MGB_CUDA_TRY(cudaFreeAsync(drep, s));
      lv.hKcls.assign((size_t)h->batch * 225, 0.0);
      MGB_CUDA_TRY(cudaMemcpyAsync(lv.hKcls.data(), lv.Kcls, lv.hKcls.size() * sizeof(double),
                                   cudaMemcpyDeviceToHost, s));
    } else {
      MGB_CUDA_TRY(launch_jacobi(h->grid(l), tab_soa(lv.A, lv.n, 1), lv.mask, omega,
                                 tabw_soa(lv.K, lv.n, 1), flag + l, s));
    }
  }
  std::vector<int> hf(L);
  MGB_CUDA_TRY(cudaMemcpyAsync(hf.data(), flag, sizeof(int) * L, cudaMemcpyDeviceToHost, s));
  MGB_CUDA_TRY(cudaFreeAsync(flag, s));
  MGB_CUDA_TRY(cudaStreamSynchronize(s));
  for (int l = 0; l + 1 < L; ++l)
    if (hf[l]) return fail(MGB_CONFIG, "jacobi: operator has zero diagonal entries");
  return classify_all(h, s);
}

extern "C" int mgb_hier_set_kernels(mgb_hier* h, int level, int kst, const double* K, int on_device,
                                    double slope, void* stream) {
  if (!h) return fail(MGB_CONTRACT, "null hierarchy");
  if (level < 0 || level + 1 >= h->depth()) return fail(MGB_CONFIG, "no smoother on this level");
  if (kst < 1) return fail(MGB_CONTRACT, "smoother needs at least one stage");
  if (h->classed_only) return fail(MGB_CONFIG, "per-point kernels cannot be installed in a band-class hierarchy");
  DeviceGuard dg(h->device);
  cudaStream_t s = S(stream);
  LevelD& lv = h->lv[level];
  if (int st = alloc_kernels(h, lv, kst)) return st;
  const size_t cnt = (size_t)h->batch * kst * 9 * lv.n;
  const double* src = K;
  double* tmp = nullptr;
  if (!on_device) {
    for (size_t q = 0; q < cnt; ++q)
      if (!std::isfinite(K[q])) return fail(MGB_NUMERIC, "non-finite smoother kernels");
    MGB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&tmp), cnt * sizeof(double), s));
    MGB_CUDA_TRY(cudaMemcpyAsync(tmp, K, cnt * sizeof(double), cudaMemcpyHostToDevice, s));
    src = tmp;
  }
  MGB_CUDA_TRY(launch_convert(h->grid(level), kst, tab_aos(src, lv.n, kst), tabw_soa(lv.K, lv.n, kst), s));
  if (tmp) MGB_CUDA_TRY(cudaFreeAsync(tmp, s));
  h->slope = slope;
  MGB_CUDA_TRY(cudaStreamSynchronize(s));
  return classify_all(h, s);
}

extern "C" int mgb_coarse_solve(const mgb_hier* h, const double* f_dev, double* x_dev, void* stream) {
  if (!h) return fail(MGB_CONTRACT, "null hierarchy");
  DeviceGuard dg(h->device);
  const int L = h->depth();
  MGB_CUDA_TRY(launch_lu_solve_grid(h->grid(L - 1), h->nc, h->lu, h->perm, h->actp, f_dev, x_dev, S(stream)));
  return MGB_OK;
}

// ---------------------------------------------------------------------------
// per-level passes

static int check_level(const mgb_hier* h, int level, bool smoothed) {
  if (!h) return fail(MGB_CONTRACT, "null hierarchy");
  if (level < 0 || level >= h->depth()) return fail(MGB_CONFIG, "level out of range");
  if (smoothed && level == h->depth() - 1) return fail(MGB_CONFIG, "the coarsest level has no smoother");
  return MGB_OK;
}

extern "C" int mgb_residual(const mgb_hier* h, int level, const double* f_dev, const double* u_dev,
                            double* r_dev, double* norm2_dev, void* stream) {
  if (int st = check_level(h, level, false)) return st;
  DeviceGuard dg(h->device);
  const LevelD& l = h->lv[level];
  const Grid g = h->grid(level);
  cudaStream_t s = S(stream);
  double* part = nullptr;
  int nblk = residual_blocks(g);
  if (norm2_dev) MGB_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&part), sizeof(double) * nblk * g.batch, s));
  MGB_CUDA_TRY(launch_residual(g, tabA(h, l), l.mask, f_dev, u_dev, r_dev, part, &nblk, s));
  if (norm2_dev) {
    MGB_CUDA_TRY(launch_finalize(g.batch, nblk, part, norm2_dev, nullptr, nullptr, 0, s));
    MGB_CUDA_TRY(cudaFreeAsync(part, s));
  }
  return MGB_OK;
}

extern "C" int mgb_restrict_residual(const mgb_hier* h, int level, const double* f_dev,
                                     const double* u_dev, double* rc_dev, void* stream) {
  if (int st = check_level(h, level, true)) return st;
  DeviceGuard dg(h->device);
  const LevelD& l = h->lv[level];
  MGB_CUDA_TRY(launch_resid_restrict2(h->grid(level), l.opA(), l.mask, h->lv[level + 1].mask,
                                      f_dev, u_dev, rc_dev, S(stream)));
  return MGB_OK;
}

extern "C" int mgb_prolong_correct(const mgb_hier* h, int level, const double* ec_dev, double* u_dev,
                                   void* stream) {
  if (int st = check_level(h, level, true)) return st;
  DeviceGuard dg(h->device);
  MGB_CUDA_TRY(launch_prolong(h->grid(level), h->lv[level].mask, ec_dev, u_dev, true, S(stream)));
  return MGB_OK;
}

// ---------------------------------------------------------------------------
// workspace + cycle driver

// workspace for cycles starting at level `first` (levels below it get no buffers)
int mgb::work_create_from(const mgb_hier* h, int first, mgb_work** out) {
  if (!h || !out) return fail(MGB_CONTRACT, "null argument");
  *out = nullptr;
  DeviceGuard dg(h->device);
  std::unique_ptr<mgb_work> w(new mgb_work());
  w->h = h;
  const int L = h->depth();
  w->u.assign(L, nullptr);
  w->t.assign(L, nullptr);
  w->f.assign(L, nullptr);
  w->r.assign(L, nullptr);
  w->v.assign(L, nullptr);
  for (int l = first; l < L; ++l) {
    const size_t cnt = (size_t)h->batch * h->lv[l].n;
    if (l > 0) {
      MGB_CUDA_TRY(dalloc(&w->u[l], cnt));
      MGB_CUDA_TRY(dalloc(&w->f[l], cnt));
    }
    if (l + 1 < L) MGB_CUDA_TRY(dalloc(&w->t[l], cnt));
  }
  const Grid g0 = h->grid(first);
  w->max_nblk = std::max(std::max(residual_blocks(g0), resnorm_blocks(g0)),
                         std::max(std::max(sweep_blocks(g0), stream_max_blocks(g0)), tile_max_blocks(g0)));
  MGB_CUDA_TRY(dalloc(&w->partials, (size_t)w->max_nblk * h->batch));
  MGB_CUDA_TRY(dalloc(&w->fnorm2, (size_t)h->batch));
  MGB_CUDA_TRY(dalloc(&w->scratch, (size_t)h->batch * 4));
  MGB_CUDA_TRY(cudaStreamCreateWithFlags(&w->cap, cudaStreamNonBlocking));
  *out = w.release();
  return MGB_OK;
}

extern "C" int mgb_work_create(const mgb_hier* h, mgb_work** out) { return work_create_from(h, 0, out); }

extern "C" void mgb_work_destroy(mgb_work* w) { delete w; }

extern "C" int64_t mgb_last_launch_count(const mgb_work* w) { return w ? w->last_launches : 0; }

static int ensure_generic(mgb_work* w, int l) {
  const mgb_hier* h = w->h;
  const size_t cnt = (size_t)h->batch * h->lv[l].n;
  if (!w->r[l]) MGB_CUDA_TRY(dalloc(&w->r[l], cnt));
  if (!w->v[l]) MGB_CUDA_TRY(dalloc(&w->v[l], cnt));
  return MGB_OK;
}

// one smoothing sweep on level l: out = in + M(f - A in); in == null means in = 0
static int sweep(mgb_work* w, int l, const double* f, const double* in, double* out, cudaStream_t s) {
  const mgb_hier* h = w->h;
  const LevelD& lv = h->lv[l];
  const Grid g = h->grid(l);
  if (lv.conv.nl > 0) {
    // u_out = u_in + M(f - A u_in) with the layer chain in v[l] / out
    if (int st = ensure_generic(w, l)) return st;
    const double* r = f;
    if (in) {
      MGB_CUDA_TRY(launch_residual(g, tabA(h, lv), lv.mask, f, in, w->r[l], nullptr, nullptr, s));
      r = w->r[l];
    }
    MGB_CUDA_TRY(conv_smoother_apply(g, lv.conv, lv.mask, r, in, out, w->v[l], out, s));
    return MGB_OK;
  }
  if (lv.ks == 1) {
    MGB_CUDA_TRY(launch_sweep2(g, lv.opA(), lv.opK(), lv.mask, f, in, out, nullptr, s));
    return MGB_OK;
  }
  // multi-stage (nonlinear) smoother: residual, then k stages with leaky between
  if (int st = ensure_generic(w, l)) return st;
  const double* r = f;
  if (in) {
    MGB_CUDA_TRY(launch_residual(g, tabA(h, lv), lv.mask, f, in, w->r[l], nullptr, nullptr, s));
    r = w->r[l];
  }
  return smoother_apply_tab(g, lv.ks, tabK(h, lv), lv.mask, h->slope, r, out, w->v[l],
                            w->r[l], in, s);
}

// hist[b * hstride] = sqrt(partials sum) / ||f|| (fnorm2 must be current)
static int enqueue_finalize(mgb_work* w, int nblk, double* hist, int64_t hstride, cudaStream_t s) {
  MGB_CUDA_TRY(launch_finalize(w->h->batch, nblk, w->partials, nullptr, w->fnorm2, hist, hstride, s));
  return MGB_OK;
}

static StreamArgs stream_args(const mgb_work* w, int l, const double* f, cudaStream_t s);

// hist[b * hstride] = ||f - A u|| / ||f|| on level 0
static int enqueue_resnorm(mgb_work* w, const double* f, const double* u, double* hist, int64_t hstride,
                           cudaStream_t s) {
  const mgb_hier* h = w->h;
  const LevelD& l0 = h->lv[0];
  if (u && h->fused && l0.ks == 1 && l0.K && (int64_t)l0.n * h->batch >= h->stream_min) {
    // row-streaming residual pass (the plain-sweep pass with its norm and no output):
    // HBM-bound, where the per-point residual kernel is load-latency-bound at this size
    StreamArgs a = stream_args(w, 0, f, s);
    a.u = u;
    a.uo = nullptr;
    a.partials = w->partials;
    int nb = 0;
    MGB_CUDA_TRY(launch_stream(a, 1, false, false, true, &nb));
    return enqueue_finalize(w, nb, hist, hstride, s);
  }
  MGB_CUDA_TRY(launch_resnorm(h->grid(0), l0.opA(), l0.mask, f, u, w->partials, s));
  return enqueue_finalize(w, resnorm_blocks(h->grid(0)), hist, hstride, s);
}

static int enqueue_fnorm(mgb_work* w, const double* f, cudaStream_t s) {
  const mgb_hier* h = w->h;
  const LevelD& l0 = h->lv[0];
  MGB_CUDA_TRY(launch_resnorm(h->grid(0), l0.opA(), l0.mask, f, nullptr, w->partials, s));
  MGB_CUDA_TRY(launch_finalize(h->batch, resnorm_blocks(h->grid(0)), w->partials, w->fnorm2, nullptr, nullptr, 0, s));
  return MGB_OK;
}

// ---- single-launch coarse cycle (mgb_coarse.cu) ------------------------------

// first level handled by the cluster kernel (levels lc..L-1), or -1
static int coarse_first_level(const mgb_hier* h) {
  if (h->coarse_max <= 0) return -1;
  const int L = h->depth();
  if (L - 1 > COARSE_MAX_LEVELS - 1) return -1;
  int lc = L - 1;
  while (lc > 0 && h->lv[lc - 1].n <= h->coarse_max) --lc;
  if (lc >= L - 1) return -1;  // only the coarsest: nothing to gain
  for (int l = lc; l + 1 < L; ++l)
    if (h->lv[l].ks != 1 || !h->lv[l].K) return -1;
  if (h->nc > 4096) return -1;
  // shared-memory budget of the block kernel: drop the finest levels until it fits
  while (lc < L - 1) {
    size_t d = 0;
    for (int l = lc; l < L; ++l) d += 3 * (size_t)h->lv[l].n + 2 * 25 * 9;
    d += std::max(h->nc, 32);
    if (d * sizeof(double) <= 200 * 1024) break;
    ++lc;
  }
  if (lc >= L - 1) return -1;
  return lc;
}

static int enqueue_coarse(mgb_work* w, int lc, bool zero, int nu1, int nu2, cudaStream_t s) {
  const mgb_hier* h = w->h;
  CoarseArgs a{};
  a.nlev = h->depth() - lc;
  a.nu1 = nu1;
  a.nu2 = nu2;
  a.zero_top = zero ? 1 : 0;
  a.nc = h->nc;
  a.lu = h->lu;
  a.perm = h->perm;
  a.actp = h->actp;
  for (int q = 0; q < a.nlev; ++q) {
    const LevelD& lv = h->lv[lc + q];
    CLevel& c = a.lv[q];
    c.rows = lv.rows;
    c.cols = lv.cols;
    c.A = lv.opA();
    c.K = q + 1 < a.nlev ? lv.opK() : Op{nullptr, nullptr, lv.n, 1};
    c.mask = lv.mask;
    c.u = w->u[lc + q];
    c.f = w->f[lc + q];
    c.r = w->r[lc + q];
  }
  MGB_CUDA_TRY(launch_coarse_block(a, h->batch, s));
  return MGB_OK;
}

// ---- row-streaming passes (mgb_stream.cu) -----------------------------------

// Row streaming for levels of at least stream_min points, except batches of narrow
// problems (< 96 columns: a strip is mostly halo and a segment mostly pipeline fill;
// config 4's 63^2 level: tile passes 55 us vs 72 us per cycle) unless stream_min = 0
// forces streaming everywhere.
static bool streamed(const mgb_hier* h, int l) {
  const LevelD& lv = h->lv[l];
  if ((int64_t)lv.n * h->batch < h->stream_min) return false;
  return !(h->stream_min > 0 && h->batch > 1 && lv.cols < 96);
}

// fused pass kind for level l: 0 separate kernels, 1 row streaming, 2 tile-local
static int pass_kind(const mgb_hier* h, int l, int nu1, int nu2) {
  const LevelD& lv = h->lv[l];
  if (!h->fused || lv.ks != 1 || !(nu1 == 1 || nu1 == 2) || !(nu2 == 1 || nu2 == 2)) return 0;
  if (streamed(h, l)) return 1;
  return h->tile ? 2 : 0;
}
static bool use_stream(const mgb_hier* h, int l, int nu1, int nu2) { return pass_kind(h, l, nu1, nu2) != 0; }

static cudaError_t launch_pass(const mgb_hier* h, int l, const StreamArgs& a, int nsw, bool res, bool pro,
                               bool norm, int* nb) {
  if (streamed(h, l)) return launch_stream(a, nsw, res, pro, norm, nb);
  return launch_tile(a, nsw, res, pro, norm, nb);
}

static StreamArgs stream_args(const mgb_work* w, int l, const double* f, cudaStream_t s) {
  const mgb_hier* h = w->h;
  const LevelD& lv = h->lv[l];
  StreamArgs a{};
  a.g = h->grid(l);
  a.A = lv.opA();
  a.K = lv.opK();
  a.mask = lv.mask;
  a.mask_c = h->lv[l + 1].mask;
  a.f = f;
  a.stream = s;
  a.ci_valid = h->batch == 1 && lv.Acls && lv.Kcls;
  a.uniform = lv.uniformity();
  a.kernel = h->stream_kernel;
  a.a5 = lv.a5 && !lv.Acls;
  if ((l == 0 && w->pad0) || (l > 0 && f && l < (int)w->pf.size() && w->pf[l] && f == w->pf[l])) {
    a.ld = pad_pitch(lv.cols);
    a.padded = 1;
  }
  for (int o = 0; o < 9; ++o) {
    a.ci[o] = lv.hAint()[o];
    a.ci[9 + o] = lv.hKint()[o];
  }
  lv.fill_kq(a.kq);
  return a;
}

// history entry from a fused pass's partial sums.  Zero start: the input residual is
// f itself (f - A 0 = f exactly), so the same sums give ||f||^2: stored as the
// denominator (history[0] = 1 exactly; no separate ||f|| pass, see get_graph).
static cudaError_t finalize_pre(mgb_work* w, int nb, bool zero_start, double* hist, int64_t hstride,
                                cudaStream_t s) {
  if (zero_start) return launch_finalize(w->h->batch, nb, w->partials, w->fnorm2, nullptr, hist, hstride, s);
  return launch_finalize(w->h->batch, nb, w->partials, nullptr, w->fnorm2, hist, hstride, s);
}

// the first fused PRE of a zero-start solve yields ||f|| (finalize_pre)
static bool pre_gives_fnorm(const mgb_hier* h, int nu1, int nu2) {
  return use_stream(h, 0, nu1, nu2) && nu1 > 0 && h->lv[0].ks == 1;
}

// PRE on level l: [history norm of the input] + nu1 sweeps + residual + restriction
// into w->f[l+1].  in == null: zero initial guess.  *cur / *oth: ping-pong buffers
// (the result ends in *cur).  hist != null: relative residual of the input.
static int enqueue_pre(mgb_work* w, int l, const double* f, const double* in, double** cur, double** oth, int nu1,
                       double* hist, int64_t hstride, cudaStream_t s, bool child_padded = false) {
  const mgb_hier* h = w->h;
  StreamArgs a = stream_args(w, l, f, s);
  const bool split = h->fused == 1;
  int nb = 0;
  if (split && nu1 == 2) {
    a.u = in;
    a.uo = *oth;
    a.partials = hist ? w->partials : nullptr;
    MGB_CUDA_TRY(launch_pass(h, l, a, 1, false, false, hist != nullptr, &nb));
    if (hist) MGB_CUDA_TRY(finalize_pre(w, nb, in == nullptr, hist, hstride, s));
    std::swap(*cur, *oth);
    in = *cur;
    hist = nullptr;
  }
  a.u = in;
  a.uo = *oth;
  a.rc = w->f[l + 1];
  if (child_padded) {   // the next level runs on its padded buffers (level_padded)
    a.rc = w->pf[l + 1];
    a.ldc = pad_pitch(h->lv[l + 1].cols);
  }
  a.partials = hist ? w->partials : nullptr;
  MGB_CUDA_TRY(launch_pass(h, l, a, split ? 1 : nu1, true, false, hist != nullptr, &nb));
  if (hist) MGB_CUDA_TRY(finalize_pre(w, nb, in == nullptr, hist, hstride, s));
  std::swap(*cur, *oth);
  return MGB_OK;
}

// POST on level l: u <- u + P ec, then nu2 sweeps (result ends in *cur)
static int enqueue_post(mgb_work* w, int l, const double* f, const double* ec, double** cur, double** oth, int nu2,
                        cudaStream_t s, double* out_hist = nullptr, int64_t out_stride = 0, bool child_padded = false) {
  const mgb_hier* h = w->h;
  StreamArgs a = stream_args(w, l, f, s);
  if (child_padded) a.ldc = pad_pitch(h->lv[l + 1].cols);
  const bool split = h->fused == 1;
  int nb = 0;
  a.u = *cur;
  a.uo = *oth;
  a.ec = ec;
  if (l == 0 && w->pad0 && w->plain_out && !split) {
    // the last POST pass of a run_cycles solve: straight into the caller's dense u instead of
    // the padded copy plus a 2-D copy back (nothing reads the padded u afterwards)
    a.uo = w->plain_out;
    a.ld_out = h->lv[0].cols;
  }
  if (out_hist) {
    // the relative residual of the pass's output folded into the pass (post_norm_ok checked by the caller)
    a.partials = w->partials;
    MGB_CUDA_TRY(launch_pass(h, l, a, nu2, true, true, false, &nb));
    std::swap(*cur, *oth);
    return finalize_pre(w, nb, false, out_hist, out_stride, s);
  }
  MGB_CUDA_TRY(launch_pass(h, l, a, split ? 1 : nu2, false, true, false, &nb));
  std::swap(*cur, *oth);
  if (split && nu2 == 2) {
    a.u = *cur;
    a.uo = *oth;
    a.ec = nullptr;
    MGB_CUDA_TRY(launch_pass(h, l, a, 1, false, false, false, &nb));
    std::swap(*cur, *oth);
  }
  return MGB_OK;
}

// V(nu1, nu2) from level l; zero means a zero initial guess (u not read).  Returns
// the buffer holding the result (u_l or the level's ping-pong partner).  With
// hist != null (level 0 only) the relative residual of the INPUT u is written to
// hist[b * hstride], folded into the first pre-sweep when it is a fused sweep.
// out_hist != null (level 0, post_norm_ok): the relative residual of the cycle's OUTPUT is
// written there by the level's POST pass.
static bool post_norm_ok(const mgb_work* w, int nu1, int nu2);
static bool level_padded(const mgb_hier* h, int l, int nu1, int nu2);

static int vcycle_rec(mgb_work* w, int l, const double* f, double* u, bool zero, int nu1, int nu2,
                      cudaStream_t s, double** result, double* hist = nullptr, int64_t hstride = 0,
                      double* out_hist = nullptr, int64_t out_stride = 0) {
  const mgb_hier* h = w->h;
  const int L = h->depth();
  if (l == L - 1) {
    MGB_CUDA_TRY(launch_lu_solve_grid(h->grid(l), h->nc, h->lu, h->perm, h->actp, f, u, s));
    *result = u;
    return MGB_OK;
  }
  const LevelD& lv = h->lv[l];
  if (!lv.has_smoother()) return fail(MGB_CONFIG, "level " + std::to_string(l) + " has no smoother installed");
  if (!hist && l > 0 && l == coarse_first_level(h) && u == w->u[l] && f == w->f[l] && w->r[l]) {
    if (int st = enqueue_coarse(w, l, zero, nu1, nu2, s)) return st;
    *result = u;
    return MGB_OK;
  }
  double* cur = u;
  const bool padl = l > 0 && l < (int)w->pf.size() && w->pf[l] && f == w->pf[l];   // this level on its padded buffers
  double* oth = (l == 0 && w->pad0) ? w->pt0 : (padl ? w->pt[l] : w->t[l]);
  const Grid g = h->grid(l);
  const bool fuse_norm = hist && nu1 > 0 && lv.ks == 1;
  if (use_stream(h, l, nu1, nu2)) {
    // the next level's buffers: padded when both levels run warp-strip passes
    const bool cp = level_padded(h, l + 1, nu1, nu2) && l + 1 < (int)w->pf.size() && w->pf[l + 1];
    if (int st = enqueue_pre(w, l, f, zero ? nullptr : cur, &cur, &oth, nu1, fuse_norm ? hist : nullptr, hstride, s, cp))
      return st;
    double* ec = nullptr;
    if (int st = vcycle_rec(w, l + 1, cp ? w->pf[l + 1] : w->f[l + 1], cp ? w->pu[l + 1] : w->u[l + 1], true, nu1,
                            nu2, s, &ec))
      return st;
    if (int st = enqueue_post(w, l, f, ec, &cur, &oth, nu2, s, l == 0 ? out_hist : nullptr, out_stride, cp)) return st;
    *result = cur;
    return MGB_OK;
  }
  if (hist && !fuse_norm) {
    if (int st = enqueue_resnorm(w, f, zero ? nullptr : u, hist, hstride, s)) return st;
  }
  if (zero && nu1 == 0) MGB_CUDA_TRY(cudaMemsetAsync(cur, 0, sizeof(double) * h->batch * lv.n, s));
  for (int q = 0; q < nu1; ++q) {
    const double* in = (zero && q == 0) ? nullptr : cur;
    if (q == 0 && fuse_norm) {
      MGB_CUDA_TRY(launch_sweep2(g, lv.opA(), lv.opK(), lv.mask, f, in, oth, w->partials, s));
      if (int st = enqueue_finalize(w, sweep_blocks(g), hist, hstride, s)) return st;
    } else {
      if (int st = sweep(w, l, f, in, oth, s)) return st;
    }
    std::swap(cur, oth);
  }
  MGB_CUDA_TRY(launch_resid_restrict2(g, lv.opA(), lv.mask, h->lv[l + 1].mask, f, cur, w->f[l + 1], s));
  double* ec = nullptr;
  if (int st = vcycle_rec(w, l + 1, w->f[l + 1], w->u[l + 1], true, nu1, nu2, s, &ec)) return st;
  MGB_CUDA_TRY(launch_prolong(g, lv.mask, ec, cur, true, s));
  for (int q = 0; q < nu2; ++q) {
    if (int st = sweep(w, l, f, cur, oth, s)) return st;
    std::swap(cur, oth);
  }
  *result = cur;
  return MGB_OK;
}

static int enqueue_vcycle(mgb_work* w, int l, const double* f, double* u, int nu1, int nu2, cudaStream_t s,
                          bool zero = false, double* hist = nullptr, int64_t hstride = 0, double* out_hist = nullptr,
                          int64_t out_stride = 0) {
  double* res = nullptr;
  if (int st = vcycle_rec(w, l, f, u, zero, nu1, nu2, s, &res, hist, hstride, out_hist, out_stride)) return st;
  if (res != u) {
    if (l == 0 && w->pad0) {   // both padded level-0 buffers: copy whole allocations (margins are zero)
      const int cols = w->h->lv[0].cols;
      MGB_CUDA_TRY(cudaMemcpyAsync(u - pad_offset(cols), res - pad_offset(cols),
                                   sizeof(double) * pad_elems(w->h->lv[0].rows, cols), cudaMemcpyDeviceToDevice, s));
    } else {
      MGB_CUDA_TRY(cudaMemcpyAsync(u, res, sizeof(double) * w->h->batch * w->h->lv[l].n,
                                   cudaMemcpyDeviceToDevice, s));
    }
  }
  return MGB_OK;
}

// Level 0 of a run_cycles solve runs on padded copies when its passes are the
// warp-strip kernel's (single problem, uniform band classes, streamed, fused).
static bool level0_padded(const mgb_hier* h, int nu1, int nu2) {
  static const bool off = getenv("MGB_NO_PAD0") && atoi(getenv("MGB_NO_PAD0")) != 0;   // A/B experiments
  if (off) return false;
  const LevelD& l0 = h->lv[0];
  return h->batch == 1 && h->depth() > 1 && pass_kind(h, 0, nu1, nu2) == 1 && l0.ks == 1 && l0.Acls && l0.Kcls &&
         !l0.mask && l0.conv.nl == 0 && l0.uniform() &&
         warp_strip_selected(h->stream_kernel, l0.n, h->batch, true);
}

// Level l >= 1 runs on padded buffers (16-byte aligned pitch, zero margins: the warp-strip
// kernel's aligned path, as level 0 of a run_cycles solve) when it and its parent level both
// run fused warp-strip passes: the parent's PRE pass restricts straight into the padded f and
// its POST pass prolongs from the padded u (StreamArgs::ldc), so no staging copy exists.
static bool level_padded(const mgb_hier* h, int l, int nu1, int nu2) {
  static const bool off = getenv("MGB_NO_PADL") && atoi(getenv("MGB_NO_PADL")) != 0;   // A/B experiments
  if (off || l < 1 || l + 1 >= h->depth() || h->batch != 1 || h->fused != 2 || l == coarse_first_level(h)) return false;
  for (int q = l - 1; q <= l; ++q) {
    const LevelD& lv = h->lv[q];
    if (pass_kind(h, q, nu1, nu2) != 1 || lv.ks != 1 || !lv.Acls || !lv.Kcls || lv.mask || lv.conv.nl != 0) return false;
    const int uni = lv.uniformity();
    if (uni == 0 || (uni == 2 && !quasi_cols_ok(lv.cols))) return false;   // generic flavour: no aligned path
    if (!warp_strip_selected(h->stream_kernel, lv.n, h->batch, true)) return false;
  }
  return true;
}

static int ensure_padl(mgb_work* w) {
  const mgb_hier* h = w->h;
  const int L = h->depth();
  if ((int)w->pf.size() != L) {
    w->pf.assign(L, nullptr);
    w->pu.assign(L, nullptr);
    w->pt.assign(L, nullptr);
  }
  for (int l = 1; l + 1 < L; ++l) {
    if (!w->t[l] || !w->t[l - 1]) continue;   // a workspace that starts below this level's parent (work_create_from)
    if (!(level_padded(h, l, 2, 2) || level_padded(h, l, 1, 1))) continue;
    for (std::vector<double*>* vec : {&w->pf, &w->pu, &w->pt}) {
      if ((*vec)[l]) continue;
      double* base = nullptr;
      const size_t cnt = (size_t)pad_elems(h->lv[l].rows, h->lv[l].cols);
      MGB_CUDA_TRY(dalloc(&base, cnt));
      MGB_CUDA_TRY(cudaMemset(base, 0, sizeof(double) * cnt));
      (*vec)[l] = base + pad_offset(h->lv[l].cols);
    }
  }
  return MGB_OK;
}

// The level-0 POST pass can carry the residual norm of its output: fused passes (not one
// pass per sweep) in the warp-strip kernel.
static bool post_norm_ok(const mgb_work* w, int nu1, int nu2) {
  const mgb_hier* h = w->h;
  static const bool off = getenv("MGB_NO_POST_NORM") && atoi(getenv("MGB_NO_POST_NORM")) != 0;   // A/B experiments
  if (off || h->depth() < 2 || h->fused != 2 || pass_kind(h, 0, nu1, nu2) != 1) return false;
  return stream_post_norm_ok(stream_args(w, 0, nullptr, nullptr), nu2);
}

static int ensure_pad0(mgb_work* w) {
  const LevelD& l0 = w->h->lv[0];
  for (double** p : {&w->pf0, &w->pu0, &w->pt0}) {
    if (*p) continue;
    double* base = nullptr;
    MGB_CUDA_TRY(dalloc(&base, (size_t)pad_elems(l0.rows, l0.cols)));
    MGB_CUDA_TRY(cudaMemset(base, 0, sizeof(double) * pad_elems(l0.rows, l0.cols)));
    *p = base + pad_offset(l0.cols);
  }
  return MGB_OK;
}

// dense <-> padded level-0 copies (the margins are never touched).  A copy kernel of our own:
// the dense rows of an odd-width grid are only 8-byte aligned, and cudaMemcpy2DAsync moved
// config 2's 134 MB in 136 us (2 TB/s) where 256-column x 8-row tiles of coalesced 8-byte
// accesses run at the HBM rate.
__global__ void __launch_bounds__(256) k_pitch_copy(double* __restrict__ dst, int64_t dp, const double* __restrict__ src,
                                                    int64_t sp, int rows, int cols) {
  const int c = blockIdx.x * 256 + threadIdx.x;
  const int r0 = blockIdx.y * 8;
  if (c >= cols) return;
  double v[8];
#pragma unroll
  for (int q = 0; q < 8; ++q)
    if (r0 + q < rows) v[q] = src[(int64_t)(r0 + q) * sp + c];
#pragma unroll
  for (int q = 0; q < 8; ++q)
    if (r0 + q < rows) dst[(int64_t)(r0 + q) * dp + c] = v[q];
}

static cudaError_t pad0_copy(const mgb_hier* h, double* dst, bool dst_padded, const double* src, bool src_padded,
                             cudaStream_t s) {
  const LevelD& l0 = h->lv[0];
  const int64_t P = pad_pitch(l0.cols), D = l0.cols;
  static const bool memcpy2d = getenv("MGB_PAD_MEMCPY2D") && atoi(getenv("MGB_PAD_MEMCPY2D")) != 0;   // A/B experiments
  if (memcpy2d)
    return cudaMemcpy2DAsync(dst, sizeof(double) * (dst_padded ? P : D), src, sizeof(double) * (src_padded ? P : D),
                             sizeof(double) * D, l0.rows, cudaMemcpyDeviceToDevice, s);
  k_pitch_copy<<<dim3((l0.cols + 255) / 256, (l0.rows + 7) / 8), 256, 0, s>>>(dst, dst_padded ? P : D, src,
                                                                            src_padded ? P : D, l0.rows, l0.cols);
  return cudaGetLastError();
}

static int check_equipped(const mgb_hier* h) {
  for (int l = 0; l + 1 < h->depth(); ++l)
    if (!h->lv[l].has_smoother()) return fail(MGB_CONFIG, "level " + std::to_string(l) + " has no smoother installed");
  return MGB_OK;
}

extern "C" int mgb_vcycle(const mgb_hier* h, mgb_work* w, int level, const double* f_dev, double* u_dev,
                          int nu1, int nu2, void* stream) {
  if (!h || !w || w->h != h) return fail(MGB_CONTRACT, "workspace does not belong to this hierarchy");
  if (level < 0 || level >= h->depth()) return fail(MGB_CONFIG, "level out of range");
  if (nu1 < 0 || nu2 < 0) return fail(MGB_CONFIG, "sweep counts must be non-negative");
  DeviceGuard dg(h->device);
  for (int l = level; l + 1 < h->depth(); ++l)
    if (!h->lv[l].has_smoother()) return fail(MGB_CONFIG, "level " + std::to_string(l) + " has no smoother installed");
  if (int st = prepare_work(w)) return st;
  const int64_t l0 = g_launches;
  int st = enqueue_vcycle(w, level, f_dev, u_dev, nu1, nu2, S(stream));
  w->last_launches = g_launches - l0;
  return st;
}

extern "C" int mgb_smooth(const mgb_hier* h, mgb_work* w, int level, const double* f_dev, double* u_dev,
                          int sweeps, void* stream) {
  if (int st = check_level(h, level, true)) return st;
  if (!w || w->h != h) return fail(MGB_CONTRACT, "workspace does not belong to this hierarchy");
  if (!h->lv[level].has_smoother()) return fail(MGB_CONFIG, "level " + std::to_string(level) + " has no smoother installed");
  DeviceGuard dg(h->device);
  cudaStream_t s = S(stream);
  double* cur = u_dev;
  double* oth = w->t[level];
  for (int q = 0; q < sweeps; ++q) {
    if (int st = sweep(w, level, f_dev, cur, oth, s)) return st;
    std::swap(cur, oth);
  }
  if (cur != u_dev)
    MGB_CUDA_TRY(cudaMemcpyAsync(u_dev, cur, sizeof(double) * h->batch * h->lv[level].n,
                                 cudaMemcpyDeviceToDevice, s));
  return MGB_OK;
}

// Capture (once per key) and launch a graph.  mode 0: run_cycles; mode 1: one
// solve iteration (cycle + residual norm into scratch).
// allocations are not allowed while capturing: size the workspace first
static int coarse_first_level(const mgb_hier* h);

int prepare_work(mgb_work* w) {
  if (level0_padded(w->h, 2, 2) || level0_padded(w->h, 1, 1))
    if (int st = ensure_pad0(w)) return st;
  if (int st = ensure_padl(w)) return st;
  for (int l = 0; l + 1 < w->h->depth(); ++l)
    if (w->h->lv[l].ks > 1 || w->h->lv[l].conv.nl > 0)
      if (int st = ensure_generic(w, l)) return st;
  const int lc = coarse_first_level(w->h);
  if (lc >= 0)
    for (int l = lc; l < w->h->depth(); ++l)
      if (!w->r[l]) MGB_CUDA_TRY(dalloc(&w->r[l], (size_t)w->h->batch * w->h->lv[l].n));
  return MGB_OK;
}

// run_cycles (mode 0): history entry c (residual of the input of cycle c) is folded
// into cycle c's first pre-sweep; the last entry needs its own residual pass.  When
// level 0 runs warp-strip passes, the cycles work on padded copies of f and u (staged
// in / out once per solve, 2 x 2 x 8 B per point: ~2 % of a 10-cycle solve).
static int enqueue_run(mgb_work* w, const GraphKey& key, cudaStream_t cs) {
  const mgb_hier* h = w->h;
  const int64_t nb = h->batch * (int64_t)h->lv[0].n;
  int st = MGB_OK;
  if (key.u_zero && key.cycles == 0) {
    cudaError_t e = cudaMemsetAsync(key.u, 0, sizeof(double) * nb, cs);
    if (e != cudaSuccess) return cuda_fail(e, "memset");
  }
  if (!(key.u_zero && key.cycles > 0 && pre_gives_fnorm(h, key.nu1, key.nu2)))
    if ((st = enqueue_fnorm(w, key.f, cs))) return st;
  const bool pad = key.cycles > 0 && level0_padded(h, key.nu1, key.nu2) && w->pf0;
  const double* f = key.f;
  double* u = key.u;
  if (pad) {
    MGB_CUDA_TRY(pad0_copy(h, w->pf0, true, key.f, false, cs));
    if (!key.u_zero) MGB_CUDA_TRY(pad0_copy(h, w->pu0, true, key.u, false, cs));
    f = w->pf0;
    u = w->pu0;
  }
  w->pad0 = pad;
  // the last history entry (residual of the final u): folded into the last cycle's level-0
  // POST pass where that pass supports it, else a residual pass of its own
  const bool fold = key.cycles > 0 && post_norm_ok(w, key.nu1, key.nu2);
  // padded solve whose last history entry rides on the last POST pass: that pass writes the
  // caller's u itself (the separate residual pass of the other case reads the padded u)
  static const bool no_direct = getenv("MGB_NO_DIRECT_OUT") && atoi(getenv("MGB_NO_DIRECT_OUT")) != 0;   // A/B experiments
  const bool direct = pad && fold && h->fused == 2 && key.nu2 > 0 && !no_direct;
  for (int c = 0; c < key.cycles && !st; ++c) {
    w->plain_out = direct && c + 1 == key.cycles ? key.u : nullptr;
    st = enqueue_vcycle(w, 0, f, u, key.nu1, key.nu2, cs, key.u_zero && c == 0, key.hist + c, key.cycles + 1,
                        fold && c + 1 == key.cycles ? key.hist + key.cycles : nullptr, key.cycles + 1);
  }
  w->plain_out = nullptr;
  if (!st && !fold) st = enqueue_resnorm(w, f, u, key.hist + key.cycles, key.cycles + 1, cs);
  w->pad0 = false;
  if (!st && pad && !direct) MGB_CUDA_TRY(pad0_copy(h, key.u, false, w->pu0, true, cs));
  return st;
}

// One solve() iteration (modes 1 / 2): a V-cycle and the relative residual of its result
// into w->scratch.  Mode 2: key.f / key.u are the padded level-0 copies.
static int enqueue_iteration(mgb_work* w, const GraphKey& key, cudaStream_t cs) {
  w->pad0 = key.mode == 2;
  const bool fold = post_norm_ok(w, key.nu1, key.nu2);
  int st = enqueue_vcycle(w, 0, key.f, key.u, key.nu1, key.nu2, cs, false, nullptr, 0, fold ? w->scratch : nullptr, 4);
  if (!st && !fold) st = enqueue_resnorm(w, key.f, key.u, w->scratch, 4, cs);
  w->pad0 = false;
  return st;
}

static int get_graph(mgb_work* w, const GraphKey& key, GraphEntry** out) {
  if (w->graph_version != w->h->version) {
    for (auto& g : w->graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    w->graphs.clear();
    w->graph_version = w->h->version;
  }
  GraphEntry* ent = nullptr;
  for (auto& g : w->graphs)
    if (g.key == key) ent = &g;
  if (!ent) {
    if (int st = prepare_work(w)) return st;
    const int64_t l0 = g_launches;
    cudaGraph_t graph = nullptr;
    MGB_CUDA_TRY(cudaStreamBeginCapture(w->cap, cudaStreamCaptureModeThreadLocal));
    int st = MGB_OK;
    const int64_t nb = w->h->batch * (int64_t)w->h->lv[0].n;
    if (key.mode == 0) {
      (void)nb;
      st = enqueue_run(w, key, w->cap);
    } else {
      st = enqueue_iteration(w, key, w->cap);
    }
    cudaError_t e = cudaStreamEndCapture(w->cap, &graph);
    if (st) {
      if (graph) cudaGraphDestroy(graph);
      return st;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
    GraphEntry ge;
    ge.key = key;
    ge.launches = g_launches - l0;
    e = cudaGraphInstantiate(&ge.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
    if (w->graphs.size() >= 8) {
      cudaGraphExecDestroy(w->graphs.front().exec);
      w->graphs.erase(w->graphs.begin());
    }
    w->graphs.push_back(ge);
    ent = &w->graphs.back();
  }
  *out = ent;
  return MGB_OK;
}

static int enqueue_key(mgb_work* w, const GraphKey& key, cudaStream_t cs) {
  int st = MGB_OK;
  const int64_t nb = w->h->batch * (int64_t)w->h->lv[0].n;
  if (key.mode == 0) {
    (void)nb;
    st = enqueue_run(w, key, cs);
  } else {
    st = enqueue_iteration(w, key, cs);
  }
  return st;
}

static int launch_graph(mgb_work* w, const GraphKey& key, cudaStream_t s) {
  static const bool no_graph = getenv("MGB_NO_GRAPH") && std::string(getenv("MGB_NO_GRAPH")) == "1";
  if (no_graph) {
    if (int st = prepare_work(w)) return st;
    const int64_t l0 = g_launches;
    int st = enqueue_key(w, key, s);
    w->last_launches = g_launches - l0;
    return st;
  }
  GraphEntry* ent = nullptr;
  if (int st = get_graph(w, key, &ent)) return st;
  MGB_CUDA_TRY(cudaGraphLaunch(ent->exec, s));
  w->last_launches = ent->launches;
  return MGB_OK;
}

extern "C" int mgb_run_cycles(const mgb_hier* h, mgb_work* w, const double* f_dev, double* u_dev, int nu1,
                              int nu2, int cycles, int u_zero, double* history_dev, void* stream) {
  if (!h || !w || w->h != h) return fail(MGB_CONTRACT, "workspace does not belong to this hierarchy");
  if (cycles < 0 || nu1 < 0 || nu2 < 0) return fail(MGB_CONFIG, "counts must be non-negative");
  if (!history_dev) return fail(MGB_CONTRACT, "history buffer required");
  if (int st = check_equipped(h)) return st;
  DeviceGuard dg(h->device);
  GraphKey key{f_dev, u_dev, nu1, nu2, cycles, u_zero ? 1 : 0, 0, history_dev};
  return launch_graph(w, key, S(stream));
}

// History staging of the host-buffer calls: hh (and hh2, the second staging set
// of the pipelined call) always share one capacity hh_cap >= nh; growing it
// reallocates both, so neither call can launch a graph whose history writes
// exceed the buffer (graphs are keyed on the buffer pointer).
static int ensure_hist(mgb_work* w, int64_t nh, bool second) {
  if (nh > w->hh_cap) {
    dfree(w->hh);
    dfree(w->hh2);
    w->hh_cap = 0;
    MGB_CUDA_TRY(dalloc(&w->hh, (size_t)nh));
    w->hh_cap = nh;
  }
  if (second && !w->hh2) MGB_CUDA_TRY(dalloc(&w->hh2, (size_t)w->hh_cap));
  return MGB_OK;
}

extern "C" int mgb_run_cycles_host(const mgb_hier* h, mgb_work* w, const double* f_host, double* u_host,
                                   int nu1, int nu2, int cycles, int u_zero, double* history_host,
                                   void* stream) {
  if (!h || !w || w->h != h) return fail(MGB_CONTRACT, "workspace does not belong to this hierarchy");
  if (!f_host || !u_host || !history_host) return fail(MGB_CONTRACT, "null host buffer");
  if (cycles < 0 || nu1 < 0 || nu2 < 0) return fail(MGB_CONFIG, "counts must be non-negative");
  if (int st = check_equipped(h)) return st;
  DeviceGuard dg(h->device);
  cudaStream_t s = S(stream);
  const size_t cnt = (size_t)h->batch * h->lv[0].n;
  if (!w->hf) MGB_CUDA_TRY(dalloc(&w->hf, cnt));
  if (!w->hu) MGB_CUDA_TRY(dalloc(&w->hu, cnt));
  const int64_t nh = (int64_t)h->batch * (cycles + 1);
  if (int st = ensure_hist(w, nh, false)) return st;
  MGB_CUDA_TRY(cudaMemcpyAsync(w->hf, f_host, cnt * sizeof(double), cudaMemcpyHostToDevice, s));
  if (!u_zero) MGB_CUDA_TRY(cudaMemcpyAsync(w->hu, u_host, cnt * sizeof(double), cudaMemcpyHostToDevice, s));
  GraphKey key{w->hf, w->hu, nu1, nu2, cycles, u_zero ? 1 : 0, 0, w->hh};
  if (int st = launch_graph(w, key, s)) return st;
  MGB_CUDA_TRY(cudaMemcpyAsync(u_host, w->hu, cnt * sizeof(double), cudaMemcpyDeviceToHost, s));
  MGB_CUDA_TRY(cudaMemcpyAsync(history_host, w->hh, nh * sizeof(double), cudaMemcpyDeviceToHost, s));
  MGB_CUDA_TRY(cudaStreamSynchronize(s));
  return MGB_OK;
}

// A stream of `count` independent solves with host buffers, pipelined: the
// host->device copy of solve k+1 (copy stream cin) and the device->host copy of
// solve k (copy stream cout) overlap the cycles of solve k (stream `stream`);
// two staging sets alternate.  Same per-solve semantics as mgb_run_cycles_host.
extern "C" int mgb_run_cycles_host_many(const mgb_hier* h, mgb_work* w, int count, const double* const* f_hosts,
                                        double* const* u_hosts, int nu1, int nu2, int cycles, int u_zero,
                                        double* const* history_hosts, void* stream) {
  if (!h || !w || w->h != h) return fail(MGB_CONTRACT, "workspace does not belong to this hierarchy");
  if (count < 0 || !f_hosts || !u_hosts || !history_hosts) return fail(MGB_CONTRACT, "null host buffer list");
  if (cycles < 0 || nu1 < 0 || nu2 < 0) return fail(MGB_CONFIG, "counts must be non-negative");
  for (int k = 0; k < count; ++k)
    if (!f_hosts[k] || !u_hosts[k] || !history_hosts[k]) return fail(MGB_CONTRACT, "null host buffer");
  if (int st = check_equipped(h)) return st;
  DeviceGuard dg(h->device);
  cudaStream_t s = S(stream);
  const size_t cnt = (size_t)h->batch * h->lv[0].n;
  const int64_t nh = (int64_t)h->batch * (cycles + 1);
  if (!w->hf) MGB_CUDA_TRY(dalloc(&w->hf, cnt));
  if (!w->hu) MGB_CUDA_TRY(dalloc(&w->hu, cnt));
  if (!w->hf2) MGB_CUDA_TRY(dalloc(&w->hf2, cnt));
  if (!w->hu2) MGB_CUDA_TRY(dalloc(&w->hu2, cnt));
  if (int st = ensure_hist(w, nh, true)) return st;
  if (!w->cin) MGB_CUDA_TRY(cudaStreamCreateWithFlags(&w->cin, cudaStreamNonBlocking));
  if (!w->cout) MGB_CUDA_TRY(cudaStreamCreateWithFlags(&w->cout, cudaStreamNonBlocking));
  for (int b = 0; b < 2; ++b)
    for (cudaEvent_t* e : {&w->ev_in[b], &w->ev_done[b], &w->ev_out[b]})
      if (!*e) MGB_CUDA_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  if ((int64_t)count * nh > w->hist_pinned_cap) {
    if (w->hist_pinned) cudaFreeHost(w->hist_pinned);
    w->hist_pinned = nullptr;
    MGB_CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&w->hist_pinned), sizeof(double) * count * nh));
    w->hist_pinned_cap = (int64_t)count * nh;
  }
  double* hf[2] = {w->hf, w->hf2};
  double* hu[2] = {w->hu, w->hu2};
  double* hh[2] = {w->hh, w->hh2};
  // the copy streams start after everything already queued on `stream`
  MGB_CUDA_TRY(cudaEventRecord(w->ev_done[0], s));
  MGB_CUDA_TRY(cudaEventRecord(w->ev_done[1], s));
  MGB_CUDA_TRY(cudaEventRecord(w->ev_out[0], s));
  MGB_CUDA_TRY(cudaEventRecord(w->ev_out[1], s));
  for (int k = 0; k < count; ++k) {
    const int b = k & 1;
    // inputs of solve k once solve k-2 no longer reads this staging set
    MGB_CUDA_TRY(cudaStreamWaitEvent(w->cin, w->ev_done[b], 0));
    MGB_CUDA_TRY(cudaMemcpyAsync(hf[b], f_hosts[k], cnt * sizeof(double), cudaMemcpyHostToDevice, w->cin));
    if (!u_zero) {
      MGB_CUDA_TRY(cudaStreamWaitEvent(w->cin, w->ev_out[b], 0));
      MGB_CUDA_TRY(cudaMemcpyAsync(hu[b], u_hosts[k], cnt * sizeof(double), cudaMemcpyHostToDevice, w->cin));
    }
    MGB_CUDA_TRY(cudaEventRecord(w->ev_in[b], w->cin));
    // cycles of solve k after its inputs arrived and solve k-2's results left
    MGB_CUDA_TRY(cudaStreamWaitEvent(s, w->ev_in[b], 0));
    MGB_CUDA_TRY(cudaStreamWaitEvent(s, w->ev_out[b], 0));
    GraphKey key{hf[b], hu[b], nu1, nu2, cycles, u_zero ? 1 : 0, 0, hh[b]};
    if (int st = launch_graph(w, key, s)) return st;
    MGB_CUDA_TRY(cudaEventRecord(w->ev_done[b], s));
    // results of solve k
    MGB_CUDA_TRY(cudaStreamWaitEvent(w->cout, w->ev_done[b], 0));
    MGB_CUDA_TRY(cudaMemcpyAsync(u_hosts[k], hu[b], cnt * sizeof(double), cudaMemcpyDeviceToHost, w->cout));
    MGB_CUDA_TRY(cudaMemcpyAsync(w->hist_pinned + (int64_t)k * nh, hh[b], nh * sizeof(double),
                                 cudaMemcpyDeviceToHost, w->cout));
    MGB_CUDA_TRY(cudaEventRecord(w->ev_out[b], w->cout));
  }
  MGB_CUDA_TRY(cudaStreamSynchronize(w->cin));
  MGB_CUDA_TRY(cudaStreamSynchronize(w->cout));
  MGB_CUDA_TRY(cudaStreamSynchronize(s));
  for (int k = 0; k < count; ++k)
    std::memcpy(history_hosts[k], w->hist_pinned + (int64_t)k * nh, sizeof(double) * nh);
  return MGB_OK;
}

extern "C" int mgb_solve(const mgb_hier* h, mgb_work* w, const double* f_dev, double* u_dev, int nu1, int nu2,
                         double tol, int max_iter, double* history_host, int* n_history, int* iterations,
                         int* converged, double* loop_seconds, void* stream) {
  if (!h || !w || w->h != h) return fail(MGB_CONTRACT, "workspace does not belong to this hierarchy");
  if (!(tol > 0.0)) return fail(MGB_CONFIG, "tolerance must be positive");
  if (h->batch != 1) return fail(MGB_CONTRACT, "mgb_solve handles one problem; use mgb_run_cycles for batches");
  if (max_iter < 0) return fail(MGB_CONFIG, "max_iter must be non-negative");
  if (int st = check_equipped(h)) return st;
  DeviceGuard dg(h->device);
  cudaStream_t s = S(stream);
  // r0 (hierarchy.py:125-133)
  if (int st = enqueue_fnorm(w, f_dev, s)) return st;
  if (int st = enqueue_resnorm(w, f_dev, u_dev, w->scratch, 4, s)) return st;
  double rr = 0.0;
  MGB_CUDA_TRY(cudaMemcpyAsync(&rr, w->scratch, sizeof(double), cudaMemcpyDeviceToHost, s));
  MGB_CUDA_TRY(cudaStreamSynchronize(s));
  const double r0 = rr;
  int nh = 0;
  history_host[nh++] = r0;
  int it = 0;
  // where level 0 runs the warp-strip passes, the loop iterates on the padded copies of f and
  // u (staged once, as mgb_run_cycles does) and u is copied back when the loop ends
  if (int st = prepare_work(w)) return st;
  const bool pad = level0_padded(h, nu1, nu2) && w->pf0;
  if (pad) {
    MGB_CUDA_TRY(pad0_copy(h, w->pf0, true, f_dev, false, s));
    MGB_CUDA_TRY(pad0_copy(h, w->pu0, true, u_dev, false, s));
  }
  GraphKey key{pad ? w->pf0 : f_dev, pad ? w->pu0 : u_dev, nu1, nu2, 1, 0, pad ? 2 : 1, nullptr};
  GraphEntry* pre = nullptr;
  if (int st = get_graph(w, key, &pre)) return st;  // capture outside the timed loop
  const auto t0 = std::chrono::steady_clock::now();
  while (history_host[nh - 1] >= tol && it < max_iter) {
    if (int st = launch_graph(w, key, s)) return st;
    MGB_CUDA_TRY(cudaMemcpyAsync(&rr, w->scratch, sizeof(double), cudaMemcpyDeviceToHost, s));
    MGB_CUDA_TRY(cudaStreamSynchronize(s));
    ++it;
    history_host[nh++] = rr;
    if (!std::isfinite(rr) || rr > 1e6 * std::max(r0, tol)) {
      char buf[160];
      snprintf(buf, sizeof buf, "diverged at iteration %d: relative residual %.3e", it, rr);
      if (n_history) *n_history = nh;
      if (iterations) *iterations = it;
      if (pad) pad0_copy(h, u_dev, false, w->pu0, true, s);
      return fail(MGB_NONCONVERGED, buf);
    }
  }
  if (pad) {
    MGB_CUDA_TRY(pad0_copy(h, u_dev, false, w->pu0, true, s));
    MGB_CUDA_TRY(cudaStreamSynchronize(s));
  }
  const auto t1 = std::chrono::steady_clock::now();
  if (n_history) *n_history = nh;
  if (iterations) *iterations = it;
  if (converged) *converged = history_host[nh - 1] < tol ? 1 : 0;
  if (loop_seconds) *loop_seconds = std::chrono::duration<double>(t1 - t0).count();
  return MGB_OK;
}

// Average device time of one PRE (pass 0) or POST (pass 1) phase on `level`,
// measured with CUDA events on `stream` around `reps` back-to-back launches
// (bench.py's roofline of the dominant kernel).  f_dev / u_dev: level arrays.
extern "C" int mgb_time_pass(const mgb_hier* h, mgb_work* w, int level, int pass, int nu, const double* f_dev,
                             double* u_dev, int reps, double* ms, void* stream) {
  if (!h || !w || w->h != h) return fail(MGB_CONTRACT, "workspace does not belong to this hierarchy");
  if (level < 0 || level + 1 >= h->depth()) return fail(MGB_CONFIG, "level has no smoothing phase");
  if (pass != 0 && pass != 1) return fail(MGB_CONFIG, "pass must be 0 (PRE) or 1 (POST)");
  if (reps < 1) return fail(MGB_CONFIG, "reps must be positive");
  if (int st = check_equipped(h)) return st;
  DeviceGuard dg(h->device);
  cudaStream_t s = S(stream);
  if (int st = prepare_work(w)) return st;
  cudaEvent_t e0, e1;
  MGB_CUDA_TRY(cudaEventCreate(&e0));
  MGB_CUDA_TRY(cudaEventCreate(&e1));
  const bool stream_pass = use_stream(h, level, nu, nu);
  double* bufs[2] = {u_dev, w->t[level]};
  // level 0 of run_cycles solves: the warp-strip passes on the padded copies
  const bool pad = level == 0 && stream_pass && level0_padded(h, nu, nu) && w->pf0;
  if (pad) {
    MGB_CUDA_TRY(pad0_copy(h, w->pf0, true, f_dev, false, s));
    MGB_CUDA_TRY(pad0_copy(h, w->pu0, true, u_dev, false, s));
    f_dev = w->pf0;
    bufs[0] = w->pu0;
    bufs[1] = w->pt0;
  }
  struct Pad0Scope {   // level 0 addressed through the padded copies for this call only
    mgb_work* w;
    ~Pad0Scope() { w->pad0 = false; }
  } pad_scope{w};
  w->pad0 = pad;
  int st = MGB_OK;
  auto one = [&](int r) -> int {
    double* cur = bufs[r & 1];
    double* oth = bufs[(r + 1) & 1];
    if (stream_pass) {
      if (pass == 0) return enqueue_pre(w, level, f_dev, cur, &cur, &oth, nu, nullptr, 0, s);
      return enqueue_post(w, level, f_dev, w->u[level + 1], &cur, &oth, nu, s);
    }
    // separate passes: the same work as the fused phase
    const LevelD& lv = h->lv[level];
    const Grid g = h->grid(level);
    if (pass == 0) {
      for (int q = 0; q < nu; ++q) {
        if (int e = sweep(w, level, f_dev, cur, oth, s)) return e;
        std::swap(cur, oth);
      }
      MGB_CUDA_TRY(launch_resid_restrict2(g, lv.opA(), lv.mask, h->lv[level + 1].mask, f_dev, cur, w->f[level + 1], s));
    } else {
      MGB_CUDA_TRY(launch_prolong(g, lv.mask, w->u[level + 1], cur, true, s));
      for (int q = 0; q < nu; ++q) {
        if (int e = sweep(w, level, f_dev, cur, oth, s)) return e;
        std::swap(cur, oth);
      }
    }
    return MGB_OK;
  };
  MGB_CUDA_TRY(cudaMemsetAsync(w->u[level + 1], 0, sizeof(double) * h->batch * h->lv[level + 1].n, s));
  st = one(0);  // warm
  if (!st) MGB_CUDA_TRY(cudaEventRecord(e0, s));
  for (int r = 0; r < reps && !st; ++r) st = one(r);
  if (!st) MGB_CUDA_TRY(cudaEventRecord(e1, s));
  if (!st) MGB_CUDA_TRY(cudaEventSynchronize(e1));
  float t = 0.f;
  if (!st) MGB_CUDA_TRY(cudaEventElapsedTime(&t, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (ms) *ms = (double)t / reps;
  return st;
}

// ---- accessors used by the domain-decomposition driver (mgb_dd.cu) ------------
namespace mgb {
int hier_rows(const mgb_hier* h, int l) { return h->lv[l].rows; }
int hier_cols(const mgb_hier* h, int l) { return h->lv[l].cols; }
int hier_batch(const mgb_hier* h) { return h->batch; }
int hier_depth(const mgb_hier* h) { return h->depth(); }
int hier_device(const mgb_hier* h) { return h->device; }
int hier_level_ks(const mgb_hier* h, int l) { return h->lv[l].ks; }
bool hier_level_classed(const mgb_hier* h, int l) { return h->lv[l].Acls && h->lv[l].Kcls && !h->lv[l].mask; }
bool hier_level_conv(const mgb_hier* h, int l) { return h->lv[l].conv.nl > 0; }
const uint8_t* hier_mask(const mgb_hier* h, int l) { return h->lv[l].mask; }
int hier_a5(const mgb_hier* h, int l) { return h->lv[l].a5 && !h->lv[l].Acls; }
Grid hier_grid(const mgb_hier* h, int l) { return h->grid(l); }
Op hier_opA(const mgb_hier* h, int l) { return h->lv[l].opA(); }
Op hier_opK(const mgb_hier* h, int l) { return h->lv[l].opK(); }
void hier_interior(const mgb_hier* h, int l, int* valid, double* ci, int* uniform, int* kernel, double* kq) {
  const LevelD& lv = h->lv[l];
  *valid = h->batch == 1 && lv.Acls && lv.Kcls;
  if (uniform) *uniform = lv.uniformity();
  if (kernel) *kernel = h->stream_kernel;
  for (int o = 0; o < 9; ++o) {
    ci[o] = lv.hAint()[o];
    ci[9 + o] = lv.hKint()[o];
  }
  if (kq) lv.fill_kq(kq);
}
double* work_level_u(mgb_work* w, int l) { return w->u[l]; }
double* work_level_f(mgb_work* w, int l) { return w->f[l]; }
int work_prepare(mgb_work* w) { return prepare_work(w); }
const mgb_hier* work_hier(const mgb_work* w) { return w->h; }
int work_vcycle_level(mgb_work* w, int l, const double* f, double* u, bool zero, int nu1, int nu2, cudaStream_t s,
                      double** result) {
  return vcycle_rec(w, l, f, u, zero, nu1, nu2, s, result);
}
}  // namespace mgb
