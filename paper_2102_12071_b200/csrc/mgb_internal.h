// Internal declarations shared by the kernel translation units and the C-ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

#include <string>

#include "../../include/mgb.h"

namespace mgb {

// ---- error plumbing ---------------------------------------------------------
void set_error(int status, const std::string& msg, int pivot = -1);
int fail(int status, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define MGB_CUDA_TRY(expr)                                   \
  do {                                                       \
    cudaError_t _e = (expr);                                 \
    if (_e != cudaSuccess) return ::mgb::cuda_fail(_e, #expr); \
  } while (0)

// Counts kernel launches issued by the wrappers below (bench instrumentation).
extern thread_local int64_t g_launches;

// MGB_DEBUG_SYNC=1: synchronise after every launch and report the failing kernel
// (debug aid; never set in measurements).
cudaError_t debug_sync(const char* what);
#define MGB_DBG(name) ::mgb::debug_sync(name)

// ---- programmatic dependent launch (PDL) for the V-cycle kernels -------------
// Every cycle kernel triggers its dependents at entry and waits (griddepcontrol.wait:
// the predecessor grid complete, its writes visible) only after loading what no
// predecessor writes (band-class tables), so the next kernel's launch and prologue
// overlap the current kernel's tail (measured ~0.6 us per small launch inside a
// CUDA graph).  MGB_NO_PDL=1 launches them plainly (A/B experiments).
bool pdl_enabled();
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
#endif

// ---- small RAII / allocation helpers ----------------------------------------
struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (dev >= 0 && dev != prev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Guard mode (MGB_GUARD=1, tests only; compute-sanitizer is not available on every GPU
// pool): every device allocation of the library gets a 4 KiB canary region on each side,
// and mgb_guard_check() reports the allocations whose canaries were overwritten.
cudaError_t guarded_malloc(void** p, size_t bytes);
void guarded_free(void* p);
template <typename T>
inline cudaError_t dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) return cudaSuccess;
  return guarded_malloc(reinterpret_cast<void**>(p), count * sizeof(T));
}
template <typename T>
inline void dfree(T*& p) {
  if (p) guarded_free(p);
  p = nullptr;
}


// ---- stencil storage descriptors --------------------------------------------
// Operators and smoother kernels are addressed per problem b of a batch as
//   value(p, s, o) = base[b * bstride + s * sstride + o * ostride + p * pstride]
// which covers both the reference "AoS" layout (rows, cols, k, 3, 3):
//   pstride = kst*9, sstride = 9, ostride = 1, bstride = n*kst*9
// and the internal "SoA" plane layout used by the hierarchy:
//   pstride = 1, ostride = n, sstride = 9n, bstride = kst*9n.
struct Tab {
  const double* base;
  int64_t bstride, sstride, ostride, pstride;
  // band-class mode (base unused): table [b][class][s][o], class of p = (i, j) from
  // band(i, crow) * 5 + band(j, ccol), band = 0, 1 first rows, 3, 4 last rows, 2 inside
  const double* cls = nullptr;
  int crow = 0, ccol = 0, cks = 1;
};
struct TabW {
  double* base;
  int64_t bstride, sstride, ostride, pstride;
  double* cls = nullptr;
  int crow = 0, ccol = 0, cks = 1;
};

inline Tab tab_cls(const double* cls, int rows, int cols, int kst) {
  Tab t{nullptr, 0, 0, 0, 0};
  t.cls = cls; t.crow = rows; t.ccol = cols; t.cks = kst;
  return t;
}
inline TabW tabw_cls(double* cls, int rows, int cols, int kst) {
  TabW t{nullptr, 0, 0, 0, 0};
  t.cls = cls; t.crow = rows; t.ccol = cols; t.cks = kst;
  return t;
}

#ifdef __CUDACC__
__device__ __forceinline__ int band_of(int i, int n) { return i < 2 ? i : (i >= n - 2 ? 4 - (n - 1 - i) : 2); }
__device__ __forceinline__ int64_t tab_index(int64_t bstride, int64_t sstride, int64_t ostride, int64_t pstride,
                                             int b, int s, int o, int64_t p) {
  return b * bstride + s * sstride + o * ostride + p * pstride;
}
__device__ __forceinline__ int64_t cls_index(int crow, int ccol, int cks, int b, int s, int o, int64_t p) {
  const int i = (int)(p / ccol), j = (int)(p - (int64_t)(p / ccol) * ccol);
  return ((int64_t)(b * 25 + band_of(i, crow) * 5 + band_of(j, ccol)) * cks + s) * 9 + o;
}
__device__ __forceinline__ double tab_get(const Tab& t, int b, int s, int o, int64_t p) {
  if (t.cls) return __ldg(t.cls + cls_index(t.crow, t.ccol, t.cks, b, s, o, p));
  return __ldg(t.base + tab_index(t.bstride, t.sstride, t.ostride, t.pstride, b, s, o, p));
}
__device__ __forceinline__ void tab_put(const TabW& t, int b, int s, int o, int64_t p, double v) {
  if (t.cls) t.cls[cls_index(t.crow, t.ccol, t.cks, b, s, o, p)] = v;
  else t.base[tab_index(t.bstride, t.sstride, t.ostride, t.pstride, b, s, o, p)] = v;
}
#endif

inline Tab tab_aos(const double* p, int64_t n, int kst) {
  return Tab{p, n * kst * 9, 9, 1, (int64_t)kst * 9};
}
inline Tab tab_soa(const double* p, int64_t n, int kst) {
  return Tab{p, n * kst * 9, 9 * n, n, 1};
}
inline TabW tabw_aos(double* p, int64_t n, int kst) {
  return TabW{p, n * kst * 9, 9, 1, (int64_t)kst * 9};
}
inline TabW tabw_soa(double* p, int64_t n, int kst) {
  return TabW{p, n * kst * 9, 9 * n, n, 1};
}

struct Grid {
  int batch, rows, cols;
  __host__ __device__ int64_t n() const { return (int64_t)rows * cols; }
};

// ---- launch wrappers (mgb_kernels.cu) ----------------------------------------
// out = A u (masked); k in {1, 3}
cudaError_t launch_apply(const Grid& g, int k, Tab A, const uint8_t* mask, const double* u,
                         double* out, cudaStream_t s);
// r = f - A u (masked); r may be null (norm only); partials (batch, nblk) may be null
cudaError_t launch_residual(const Grid& g, Tab A, const uint8_t* mask, const double* f,
                            const double* u, double* r, double* partials, int* nblk,
                            cudaStream_t s);
int residual_blocks(const Grid& g);
// fixed-order sum of partials -> out[b] (sum of squares); if hist != null, also
// hist[b*hstride] = sqrt(out)/denom rule against fnorm2[b] (null -> denominator is
// the value itself: used to compute ||f||)
cudaError_t launch_finalize(int batch, int nblk, const double* partials, double* out2,
                            const double* fnorm2, double* hist, int64_t hstride, cudaStream_t s);
// fused sweep, k = 1 kernels: uo = u + M(f - A u); u == null means u = 0
cudaError_t launch_sweep(const Grid& g, Tab A, Tab K, const uint8_t* mask, const double* f,
                         const double* u, double* uo, cudaStream_t s);
// pointwise stage: out = (base ? base + c : c), c = sum_o K_s[o] g(in(p+o)), g = leaky if lk
cudaError_t launch_pointwise(const Grid& g, Tab K, int stage, const uint8_t* mask,
                             const double* in, bool lk, double slope, const double* base,
                             double* out, cudaStream_t s);
// rc = R (f - A u) ; u == null means u = 0 (rc = R f)
cudaError_t launch_resid_restrict(const Grid& g, Tab A, const uint8_t* mask_f,
                                  const uint8_t* mask_c, const double* f, const double* u,
                                  double* rc, cudaStream_t s);
// coarse = R fine
cudaError_t launch_restrict(const Grid& g, const uint8_t* mask_c, const double* fine,
                            double* coarse, cudaStream_t s);
// fine = P coarse (add == false) or fine += P coarse (add == true); masked by mask_f
cudaError_t launch_prolong(const Grid& g, const uint8_t* mask_f, const double* coarse,
                           double* fine, bool add, cudaStream_t s);
// Ac = R A P; ring_flag (int, device) |= 1 where the outer ring is non-zero.
// pts (optional, npts entries, -1 = skip): evaluate only these coarse points
// (band-class representatives when Ac is a class table).
cudaError_t launch_galerkin(const Grid& g, Tab A, const uint8_t* mask_f, const uint8_t* mask_c,
                            TabW Ac, int* ring_flag, cudaStream_t s, const int64_t* pts = nullptr,
                            int npts = 0);
// dense materialisation of the (coarsest) operator over active points
cudaError_t launch_materialize(const Grid& g, Tab A, const int32_t* index_map, int nact,
                               const int32_t* act, double* M, cudaStream_t s);
// batched LU (one block per problem); status (batch) receives -1 or the failing pivot
cudaError_t launch_lu_factor(int batch, int n, double* lu, int32_t* perm, int* status,
                             cudaStream_t s);
cudaError_t launch_lu_solve_grid(const Grid& g, int n, const double* lu, const int32_t* perm,
                                 const int32_t* act, const double* f, double* x,
                                 cudaStream_t s);
cudaError_t launch_lu_solve_vec(int n, const double* lu, const int32_t* perm, const double* b,
                                double* x, cudaStream_t s);
// jacobi kernels: K (SoA, kst = 1) = omega / diag at the centre, 0 elsewhere / inactive
cudaError_t launch_jacobi(const Grid& g, Tab A, const uint8_t* mask, double omega, TabW K,
                          int* zero_diag_flag, cudaStream_t s, const int64_t* pts = nullptr, int npts = 0);
// layout conversion between reference AoS and internal SoA tables
cudaError_t launch_convert(const Grid& g, int kst, Tab src, TabW dst, cudaStream_t s);

// ---- CNN inference (mgb_cnn.cu) -------------------------------------------------
cudaError_t launch_infer(const Grid& g, Tab A, const uint8_t* mask, int variant, int kst,
                         const double* W_dev, double slope, int precision, TabW K,
                         cudaStream_t s, const int64_t* pts = nullptr, int npts = 0);
int64_t net_weight_count(int variant, int kst);

}  // namespace mgb
