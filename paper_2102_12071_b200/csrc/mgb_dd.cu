// Domain-decomposed V-cycle: the fine levels are split into row
// blocks ("parts"), one per GPU; every pass is the same row-streaming kernel run
// on a ghosted block (pointers pre-offset to global rows, owned range
// [R0, R1)), preceded by a halo exchange of the S + 1 = 6 rows it reads across
// each block edge.  Below the agglomeration level the restricted residual is
// all-gathered and every rank runs the coarse cycle redundantly (no idle ranks,
// no scatter), then prolongs from its rows of the replicated correction.
//
// Exchange backends:
//  * NCCL (one part per process): grouped ncclSend/ncclRecv of contiguous ghost
//    row blocks on the solve stream, ncclAllGather for agglomeration,
//    ncclAllReduce of the 8-byte history partial sums — all graph-capturable;
//  * virtual (all parts in one process on one GPU): the same schedule with
//    device-to-device copies; used to test the decomposition on a single B200;
//  * callback (one part per process, mgb_dd_set_exchange): every exchange is handed
//    to a host function after a stream synchronisation (no graph), e.g. a
//    host-staged gloo exchange between processes that share one GPU — the test of
//    the rank-local schedule itself where only one GPU exists.
// Overlap: a pass over a block is split into an interior launch (rows that read no
// ghost row) and an edge launch; the exchanges run on a side stream while the
// interior launch runs, the edge launch waits for them (fork / join by events,
// captured with the rest).  Per-point results do not depend on the split.
// Levels may hold band-class tables or per-point planes and masks (the tables are
// replicated on every rank and addressed by global row).
// Per-point results are independent of the partition (every point runs the
// same operation sequence), so u matches the single-domain solve bitwise; only
// the history norms are summed in a different order.
//
// NCCL is loaded at run time (dlopen of the libnccl.so.2 the process already has,
// e.g. PyTorch's), so the library has no link-time NCCL dependency.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "mgb_dd.h"

namespace mgb {

// ---- minimal NCCL binding (types from the public ABI of nccl.h) -------------
namespace nccl {
typedef struct ncclComm* Comm;
struct UniqueId { char internal[128]; };
enum Result { Success = 0 };
enum DataType { Float64 = 8 };
enum RedOp { Sum = 0 };
typedef Result (*CommInitRank_t)(Comm*, int, UniqueId, int);
typedef Result (*CommDestroy_t)(Comm);
typedef Result (*Send_t)(const void*, size_t, DataType, int, Comm, cudaStream_t);
typedef Result (*Recv_t)(void*, size_t, DataType, int, Comm, cudaStream_t);
typedef Result (*AllReduce_t)(const void*, void*, size_t, DataType, RedOp, Comm, cudaStream_t);
typedef Result (*AllGather_t)(const void*, void*, size_t, DataType, Comm, cudaStream_t);
typedef Result (*Group_t)();
typedef Result (*GetUniqueId_t)(UniqueId*);
typedef const char* (*GetErrorString_t)(Result);
struct Api {
  CommInitRank_t CommInitRank = nullptr;
  CommDestroy_t CommDestroy = nullptr;
  Send_t Send = nullptr;
  Recv_t Recv = nullptr;
  AllReduce_t AllReduce = nullptr;
  AllGather_t AllGather = nullptr;
  Group_t GroupStart = nullptr, GroupEnd = nullptr;
  GetUniqueId_t GetUniqueId = nullptr;
  GetErrorString_t GetErrorString = nullptr;
  bool ok = false;
};
static Api& api() {
  static Api a;
  static bool tried = false;
  if (tried) return a;
  tried = true;
  void* hdl = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!hdl) hdl = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!hdl) hdl = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!hdl) return a;
  a.CommInitRank = (CommInitRank_t)dlsym(hdl, "ncclCommInitRank");
  a.CommDestroy = (CommDestroy_t)dlsym(hdl, "ncclCommDestroy");
  a.Send = (Send_t)dlsym(hdl, "ncclSend");
  a.Recv = (Recv_t)dlsym(hdl, "ncclRecv");
  a.AllReduce = (AllReduce_t)dlsym(hdl, "ncclAllReduce");
  a.AllGather = (AllGather_t)dlsym(hdl, "ncclAllGather");
  a.GroupStart = (Group_t)dlsym(hdl, "ncclGroupStart");
  a.GroupEnd = (Group_t)dlsym(hdl, "ncclGroupEnd");
  a.GetUniqueId = (GetUniqueId_t)dlsym(hdl, "ncclGetUniqueId");
  a.GetErrorString = (GetErrorString_t)dlsym(hdl, "ncclGetErrorString");
  a.ok = a.CommInitRank && a.CommDestroy && a.Send && a.Recv && a.AllReduce && a.AllGather && a.GroupStart &&
         a.GroupEnd && a.GetUniqueId;
  return a;
}
}  // namespace nccl

#define MGB_NCCL_TRY(expr)                                                                   \
  do {                                                                                      \
    nccl::Result _r = (expr);                                                               \
    if (_r != nccl::Success) {                                                              \
      const char* m = nccl::api().GetErrorString ? nccl::api().GetErrorString(_r) : "?";   \
      return fail(MGB_NCCL, std::string("NCCL error in " #expr ": ") + m);                 \
    }                                                                                       \
  } while (0)

namespace {

__global__ void k_sum_norm(const double* __restrict__ parts, int n, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < n; ++q) s += parts[q];
    *out = s;
  }
}

__global__ void k_hist_entry(const double* __restrict__ r2, const double* __restrict__ f2,
                             double* __restrict__ hist) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const double nr = sqrt(*r2), fn = sqrt(*f2);
    const double den = fn > 0.0 ? fn : 1.0;      // hierarchy.py:126-127
    *hist = nr == 0.0 ? 0.0 : nr / den;           // hierarchy.py:129-131
  }
}

}  // namespace
}  // namespace mgb

using namespace mgb;

struct DDPart {
  int part = 0;
  std::vector<int> R0, R1;       // owned rows per distributed level
  std::vector<double*> u, t, f;  // ghosted blocks: rows [R0 - ga, R1 + ga) x pitch (mgb_dd::view)
  double* partials = nullptr;
  double* norm2 = nullptr;       // per-part sum of squares (device scalar)
};

struct mgb_dd {
  const mgb_hier* h = nullptr;
  int device = 0, nparts = 1, first = 0, nlocal = 1, Ld = 0, La = 0, cols0 = 0;
  std::vector<DDPart> parts;
  mgb_work* cw = nullptr;        // replicated coarse levels (>= La)
  double* gather = nullptr;      // padded all-gather target for the agglomerated residual
  int Bc = 0;                    // coarse rows per part in the gather layout
  double* norm_parts = nullptr;  // nlocal doubles
  double* r2 = nullptr;          // total residual^2 (device scalar)
  double* f2 = nullptr;          // total ||f||^2
  double* hist_scratch = nullptr;
  nccl::Comm comm = nullptr;
  mgb_dd_exchange_fn xfn = nullptr;   // callback backend
  void* xctx = nullptr;
  bool overlap = true, do_exchange = true;
  cudaStream_t side = nullptr;        // exchanges of the overlapped schedule
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int64_t halo_bytes = 0;             // bytes this rank sent in the last enqueued run (all cycles)
  int exchanges = 0;
  cudaStream_t cap = nullptr;
  cudaGraphExec_t graph = nullptr;
  int gkey[4] = {-1, -1, -1, -1};
  double* ghist = nullptr;
  int max_blocks = 0;
  ~mgb_dd() {
    DeviceGuard dg(device);
    if (graph) cudaGraphExecDestroy(graph);
    for (auto& p : parts) {
      for (auto* v : {&p.u, &p.t, &p.f})
        for (auto*& q : *v) dfree(q);
      dfree(p.partials);
      dfree(p.norm2);
    }
    dfree(gather);
    dfree(norm_parts);
    dfree(r2);
    dfree(f2);
    dfree(hist_scratch);
    if (cw) mgb_work_destroy(cw);
    if (comm && nccl::api().ok) nccl::api().CommDestroy(comm);
    if (cap) cudaStreamDestroy(cap);
    if (side) cudaStreamDestroy(side);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
  }
  int rows(int l) const { return hier_rows(h, l); }
  int cols(int l) const { return hier_cols(h, l); }
  // Block layout of a distributed level: stored rows [R0 - ga, R1 + ga), row pitch `pitch`,
  // `lc` margin columns left of column 0.  Dense levels: ga = 6 (the ghost rows), pitch =
  // cols, lc = 0.  Level 0 of a uniform band-class hierarchy (the warp-strip kernel) uses
  // that kernel's padded layout: 16-byte aligned pitch, zero column margins, 16 allocated
  // rows per edge (its unpredicated ring copies touch up to 11 rows beyond a block; only
  // the 6 ghost rows next to the block carry data, the rest stay zero).
  std::vector<int64_t> pitch;
  std::vector<int> ga, lc;
  std::vector<char> padded;
  // pointer to global (row 0, column 0) of a block whose owned rows start at R0
  double* view(double* blk, int R0, int l) const { return blk + lc[l] - (int64_t)(R0 - ga[l]) * pitch[l]; }
  // start of stored row `row` (its left margin included) given the (0, 0) pointer
  double* rowp(double* v0, int row, int l) const { return v0 + (int64_t)row * pitch[l] - lc[l]; }
  size_t block_doubles(int r0, int r1, int l) const { return (size_t)(r1 - r0 + 2 * ga[l]) * pitch[l]; }
};

static constexpr int G = DD_GHOST;
static cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" int mgb_dd_nccl_unique_id(void* id_out) {
  if (!nccl::api().ok) return fail(MGB_NCCL, "libnccl.so.2 not available");
  nccl::UniqueId id;
  MGB_NCCL_TRY(nccl::api().GetUniqueId(&id));
  std::memcpy(id_out, &id, sizeof(id));
  return MGB_OK;
}

extern "C" int mgb_dd_create(const mgb_hier* h, int nparts, int first_part, int nlocal, const void* nccl_id,
                             int agglomerate_rows, mgb_dd** out) {
  if (!h || !out) return fail(MGB_CONTRACT, "null argument");
  *out = nullptr;
  if (nparts < 1 || nlocal < 1 || first_part < 0 || first_part + nlocal > nparts)
    return fail(MGB_CONFIG, "invalid part layout");
  if (nlocal != nparts && nlocal != 1) return fail(MGB_CONFIG, "either all parts local (virtual) or one per rank");
  // nlocal == 1, nparts > 1 without an NCCL id: the callback backend (mgb_dd_set_exchange)
  if (hier_batch(h) != 1) return fail(MGB_CONFIG, "domain decomposition takes a single problem");
  const int L = hier_depth(h);
  for (int l = 0; l + 1 < L; ++l)
    if (hier_level_ks(h, l) != 1 || hier_level_conv(h, l))
      return fail(MGB_CONFIG, "domain decomposition needs per-point (or band-class) 1-stage smoothers on every level");
  DeviceGuard dg(hier_device(h));
  std::unique_ptr<mgb_dd> d(new mgb_dd());
  d->h = h;
  d->device = hier_device(h);
  d->nparts = nparts;
  d->first = first_part;
  d->nlocal = nlocal;
  d->cols0 = d->cols(0);
  // distributed levels: rows > agglomerate_rows, at least one, coarse cycle needs >= 2 levels below
  int Ld = 0;
  while (Ld + 2 < L && d->rows(Ld) > agglomerate_rows) ++Ld;
  if (Ld == 0) Ld = 1;
  d->Ld = Ld;
  d->La = Ld;
  // level-0 blocks: multiples of 2^Ld so every distributed level's block start is even
  const int align = 1 << Ld;
  const int rows0 = d->rows(0);
  int blk = (rows0 + nparts - 1) / nparts;
  blk = (blk + align - 1) / align * align;
  for (int p = 0; p < nparts; ++p) {
    const int r0 = std::min(p * blk, rows0), r1 = std::min((p + 1) * blk, rows0);
    if (r1 - r0 < 2 * G * align) return fail(MGB_CONFIG, "too many parts for this grid (blocks smaller than the halo)");
  }
  d->Bc = blk >> Ld;
  for (int l = 0; l < Ld; ++l) {
    StreamArgs a{};
    a.g = hier_grid(h, l);
    a.A = hier_opA(h, l);
    a.K = hier_opK(h, l);
    a.mask = hier_mask(h, l);
    hier_interior(h, l, &a.ci_valid, a.ci, &a.uniform, &a.kernel, a.kq);
    static const bool no_pad = getenv("MGB_DD_PAD") && atoi(getenv("MGB_DD_PAD")) == 0;   // A/B experiments
    const bool pad = !no_pad && a.uniform == 1 && stream_kernel_kind(a) == 3;
    d->padded.push_back(pad ? 1 : 0);
    d->pitch.push_back(pad ? pad_pitch(d->cols(l)) : d->cols(l));
    d->ga.push_back(pad ? PAD_ROWS : G);
    d->lc.push_back(pad ? PAD_LCOLS : 0);
  }
  for (int q = 0; q < nlocal; ++q) {
    DDPart P;
    P.part = first_part + q;
    for (int l = 0; l < Ld; ++l) {
      const int r0 = std::min(P.part * blk, rows0) >> l;
      const int r1 = P.part == nparts - 1 ? d->rows(l) : (std::min((P.part + 1) * blk, rows0) >> l);
      P.R0.push_back(r0);
      P.R1.push_back(r1);
      const size_t cnt = d->block_doubles(r0, r1, l);
      double *a = nullptr, *b = nullptr, *c = nullptr;
      MGB_CUDA_TRY(dalloc(&a, cnt));
      MGB_CUDA_TRY(dalloc(&b, cnt));
      MGB_CUDA_TRY(dalloc(&c, cnt));
      MGB_CUDA_TRY(cudaMemset(a, 0, cnt * sizeof(double)));
      MGB_CUDA_TRY(cudaMemset(b, 0, cnt * sizeof(double)));
      MGB_CUDA_TRY(cudaMemset(c, 0, cnt * sizeof(double)));
      P.u.push_back(a);
      P.t.push_back(b);
      P.f.push_back(c);
    }
    d->parts.push_back(std::move(P));
  }
  d->max_blocks = stream_max_blocks(hier_grid(h, 0));
  for (auto& P : d->parts) {
    MGB_CUDA_TRY(dalloc(&P.partials, (size_t)3 * d->max_blocks + 64));   // interior + edge launches
    MGB_CUDA_TRY(dalloc(&P.norm2, 1));
  }
  MGB_CUDA_TRY(dalloc(&d->norm_parts, (size_t)nlocal));
  MGB_CUDA_TRY(dalloc(&d->r2, 1));
  MGB_CUDA_TRY(dalloc(&d->f2, 1));
  MGB_CUDA_TRY(dalloc(&d->hist_scratch, 1));
  // replicated coarse workspace from the agglomeration level + padded gather buffer
  if (int st = work_create_from(h, d->La, &d->cw)) return st;
  MGB_CUDA_TRY(dalloc(&d->gather, (size_t)nparts * d->Bc * d->cols(d->La)));
  MGB_CUDA_TRY(cudaMemset(d->gather, 0, sizeof(double) * nparts * d->Bc * d->cols(d->La)));
  MGB_CUDA_TRY(cudaStreamCreateWithFlags(&d->cap, cudaStreamNonBlocking));
  MGB_CUDA_TRY(cudaStreamCreateWithFlags(&d->side, cudaStreamNonBlocking));
  MGB_CUDA_TRY(cudaEventCreateWithFlags(&d->ev_fork, cudaEventDisableTiming));
  MGB_CUDA_TRY(cudaEventCreateWithFlags(&d->ev_join, cudaEventDisableTiming));
  {
    static const char* e = getenv("MGB_DD_OVERLAP");
    if (e) d->overlap = atoi(e) != 0;
  }
  if (nlocal == 1 && nccl_id) {  // (a 1-rank communicator also takes the NCCL path: tested on one GPU)
    if (!nccl::api().ok) return fail(MGB_NCCL, "libnccl.so.2 not available");
    nccl::UniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    MGB_NCCL_TRY(nccl::api().CommInitRank(&d->comm, nparts, id, first_part));
  }
  *out = d.release();
  return MGB_OK;
}

extern "C" void mgb_dd_destroy(mgb_dd* d) { delete d; }

extern "C" int mgb_dd_info(const mgb_dd* d, int part, int* r0, int* r1, int* dist_levels) {
  if (!d) return fail(MGB_CONTRACT, "null decomposition");
  const int q = part - d->first;
  if (q < 0 || q >= d->nlocal) return fail(MGB_CONFIG, "part not held by this process");
  if (r0) *r0 = d->parts[q].R0[0];
  if (r1) *r1 = d->parts[q].R1[0];
  if (dist_levels) *dist_levels = d->Ld;
  return MGB_OK;
}

// ---- halo exchange of one level's field (ghost rows [R0-G, R0) and [R1, R1+G)) ----
// which: 0 = u, 1 = t, 2 = f
static int exchange(mgb_dd* d, int l, int which, cudaStream_t s) {
  if (!d->do_exchange) return MGB_OK;   // timing runs only (results are wrong without the halos)
  const int rows = d->rows(l);
  const int64_t pitch = d->pitch[l];    // whole stored rows travel (margins included: they are zero)
  auto buf = [&](DDPart& P) -> double* { return which == 0 ? P.u[l] : which == 1 ? P.t[l] : P.f[l]; };
  const size_t gcount = (size_t)G * pitch;
  if (d->comm == nullptr && d->xfn == nullptr) {
    // virtual: all parts local
    for (int q = 0; q < d->nlocal; ++q) {
      DDPart& P = d->parts[q];
      double* v = d->view(buf(P), P.R0[l], l);
      if (q > 0) {
        DDPart& A = d->parts[q - 1];
        double* va = d->view(buf(A), A.R0[l], l);
        MGB_CUDA_TRY(cudaMemcpyAsync(d->rowp(v, P.R0[l] - G, l), d->rowp(va, P.R0[l] - G, l), gcount * sizeof(double),
                                     cudaMemcpyDeviceToDevice, s));
        d->halo_bytes += gcount * sizeof(double);
      }
      if (q + 1 < d->nlocal) {
        DDPart& B = d->parts[q + 1];
        double* vb = d->view(buf(B), B.R0[l], l);
        const int n = std::min(G, rows - P.R1[l]);
        MGB_CUDA_TRY(cudaMemcpyAsync(d->rowp(v, P.R1[l], l), d->rowp(vb, P.R1[l], l), (size_t)n * pitch * sizeof(double),
                                     cudaMemcpyDeviceToDevice, s));
        d->halo_bytes += (size_t)n * pitch * sizeof(double);
      }
    }
    ++d->exchanges;
    return MGB_OK;
  }
  DDPart& P = d->parts[0];
  double* v = d->view(buf(P), P.R0[l], l);
  const int me = P.part;
  const int nb = me + 1 < d->nparts ? std::min(G, rows - P.R1[l]) : 0;
  ++d->exchanges;
  d->halo_bytes += ((me > 0 ? gcount : 0) + (size_t)nb * pitch) * sizeof(double);
  double* up_send = d->rowp(v, P.R0[l], l);
  double* up_recv = d->rowp(v, P.R0[l] - G, l);
  double* dn_send = d->rowp(v, P.R1[l] - nb, l);
  double* dn_recv = d->rowp(v, P.R1[l], l);
  if (d->xfn) {
    // callback backend: the neighbour above first, then the one below (rank 0 starts the chain)
    MGB_CUDA_TRY(cudaStreamSynchronize(s));
    if (me > 0)
      if (d->xfn(d->xctx, 0, me - 1, up_send, up_recv, (int64_t)gcount))
        return fail(MGB_NCCL, "exchange callback failed (halo, upper neighbour)");
    if (nb > 0)
      if (d->xfn(d->xctx, 0, me + 1, dn_send, dn_recv, (int64_t)nb * pitch))
        return fail(MGB_NCCL, "exchange callback failed (halo, lower neighbour)");
    return MGB_OK;
  }
  auto& A = nccl::api();
  MGB_NCCL_TRY(A.GroupStart());
  if (me > 0) {
    MGB_NCCL_TRY(A.Send(up_send, gcount, nccl::Float64, me - 1, d->comm, s));
    MGB_NCCL_TRY(A.Recv(up_recv, gcount, nccl::Float64, me - 1, d->comm, s));
  }
  if (nb > 0) {
    MGB_NCCL_TRY(A.Send(dn_send, (size_t)nb * pitch, nccl::Float64, me + 1, d->comm, s));
    MGB_NCCL_TRY(A.Recv(dn_recv, (size_t)nb * pitch, nccl::Float64, me + 1, d->comm, s));
  }
  MGB_NCCL_TRY(A.GroupEnd());
  return MGB_OK;
}

// sum the per-part sums of squares into *dst (all ranks)
static int reduce_norm(mgb_dd* d, double* dst, cudaStream_t s) {
  for (int q = 0; q < d->nlocal; ++q)
    MGB_CUDA_TRY(cudaMemcpyAsync(d->norm_parts + q, d->parts[q].norm2, sizeof(double), cudaMemcpyDeviceToDevice, s));
  k_sum_norm<<<1, 32, 0, s>>>(d->norm_parts, d->nlocal, dst);
  MGB_CUDA_TRY(cudaGetLastError());
  if (d->comm) MGB_NCCL_TRY(nccl::api().AllReduce(dst, dst, 1, nccl::Float64, nccl::Sum, d->comm, s));
  if (d->xfn) {
    MGB_CUDA_TRY(cudaStreamSynchronize(s));
    if (d->xfn(d->xctx, 2, -1, nullptr, dst, 1)) return fail(MGB_NCCL, "exchange callback failed (all-reduce)");
  }
  return MGB_OK;
}

static StreamArgs dd_args(const mgb_dd* d, int l, cudaStream_t s) {
  StreamArgs a{};
  a.g = hier_grid(d->h, l);
  a.A = hier_opA(d->h, l);
  a.K = hier_opK(d->h, l);
  a.mask = hier_mask(d->h, l);
  a.mask_c = hier_mask(d->h, l + 1);
  a.a5 = hier_a5(d->h, l);
  a.stream = s;
  hier_interior(d->h, l, &a.ci_valid, a.ci, &a.uniform, &a.kernel, a.kq);
  if (l < (int)d->padded.size() && d->padded[l]) {
    a.ld = d->pitch[l];
    a.padded = 1;
  }
  return a;
}

// Rows of a block's edge launches: a pass over rows [x, y) reads rows [x - 6, y + 5], so
// the interior launch over [R0 + EDGE, R1 - EDGE) touches owned rows only.  Even, so the
// sub-ranges start at even rows like the blocks themselves (coarse anchors 2c + 1 never
// straddle a boundary).
#ifndef MGB_DD_EDGE
#define MGB_DD_EDGE 8
#endif
static constexpr int EDGE = MGB_DD_EDGE;   // >= 6 and even; 8: the shortest edge launch (8 rows + pipeline fill)

// One pass (PRE: res; POST: pro; or the plain norm sweep) over part P's rows of level l.
// phase 0: the interior rows, 1: the edge rows, 2: the whole block in one launch.  With
// norm, the launches' partial sums are appended at P.partials + *npart.
static int launch_rows(mgb_dd* d, int l, DDPart& P, StreamArgs a, int nsw, bool res, bool pro, bool norm, int phase,
                       int* npart) {
  const int R0 = P.R0[l], R1 = P.R1[l];
  // a block edge on the physical boundary needs no ghost rows: it belongs to the interior launch
  const int lo = P.part == 0 ? R0 : R0 + EDGE, hi = P.part == d->nparts - 1 ? R1 : R1 - EDGE;
  int ranges[2][2], nr = 0;
  if (phase == 2) {
    ranges[nr][0] = R0, ranges[nr++][1] = R1;
  } else if (phase == 0) {
    ranges[nr][0] = lo, ranges[nr++][1] = hi;
  } else {
    if (lo > R0) ranges[nr][0] = R0, ranges[nr++][1] = lo;
    if (hi < R1) ranges[nr][0] = hi, ranges[nr++][1] = R1;
  }
  for (int q = 0; q < nr; ++q) {
    a.own0 = ranges[q][0];
    a.own1 = ranges[q][1];
    if (a.own1 <= a.own0) continue;
    a.partials = norm ? P.partials + *npart : nullptr;
    int nb = 0;
    MGB_CUDA_TRY(launch_stream(a, nsw, res, pro, norm, &nb));
    if (norm) *npart += nb;
  }
  return MGB_OK;
}

static bool split_ok(const mgb_dd* d, int l) {
  if (!d->overlap || d->nparts == 1) return false;
  for (auto& P : d->parts)
    if (P.R1[l] - P.R0[l] < 128) return false;
  return true;
}

// Run `exchanges` (the halo exchanges a pass needs) and the pass `rows(phase)`.  Overlapped:
// the exchanges go to the side stream while the interior rows run on s; the edge rows wait
// for them.  Otherwise: exchanges, then the whole block.
template <typename FX, typename FR>
static int exchange_and_pass(mgb_dd* d, int l, cudaStream_t s, bool any_exchange, FX exchanges, FR rows) {
  if (!any_exchange || !split_ok(d, l)) {
    if (int st = exchanges(s)) return st;
    return rows(2);
  }
  if (d->xfn) {   // callback backend: eager and synchronous, same launches
    if (int st = exchanges(s)) return st;
    if (int st = rows(0)) return st;
    return rows(1);
  }
  MGB_CUDA_TRY(cudaEventRecord(d->ev_fork, s));
  MGB_CUDA_TRY(cudaStreamWaitEvent(d->side, d->ev_fork, 0));
  if (int st = exchanges(d->side)) return st;
  MGB_CUDA_TRY(cudaEventRecord(d->ev_join, d->side));
  if (int st = rows(0)) return st;
  MGB_CUDA_TRY(cudaStreamWaitEvent(s, d->ev_join, 0));
  return rows(1);
}

// residual norm^2 of the current level-0 u (or of f when u == null) per part, via a
// streaming plain-sweep pass whose output goes to scratch
static int norm_pass(mgb_dd* d, bool of_f, double* dst, cudaStream_t s) {
  std::vector<int> np(d->parts.size(), 0);
  auto rows = [&](int phase) -> int {
    for (size_t q = 0; q < d->parts.size(); ++q) {
      DDPart& P = d->parts[q];
      StreamArgs a = dd_args(d, 0, s);
      a.f = d->view(P.f[0], P.R0[0], 0);
      a.u = of_f ? nullptr : d->view(P.u[0], P.R0[0], 0);
      a.uo = d->view(P.t[0], P.R0[0], 0);
      if (int st = launch_rows(d, 0, P, a, 1, false, false, true, phase, &np[q])) return st;
    }
    return MGB_OK;
  };
  if (int st = exchange_and_pass(d, 0, s, !of_f, [&](cudaStream_t x) { return of_f ? MGB_OK : exchange(d, 0, 0, x); },
                                 rows))
    return st;
  for (size_t q = 0; q < d->parts.size(); ++q)
    MGB_CUDA_TRY(launch_finalize(1, np[q], d->parts[q].partials, d->parts[q].norm2, nullptr, nullptr, 0, s));
  return reduce_norm(d, dst, s);
}

// one V(nu1, nu2) cycle; hist != null: the relative residual of the input u
static int dd_cycle(mgb_dd* d, int nu1, int nu2, bool zero, double* hist, cudaStream_t s) {
  const int Ld = d->Ld, La = d->La;
  // descend over the distributed levels
  for (int l = 0; l < Ld; ++l) {
    const bool z = zero || l > 0;
    const bool last = l + 1 == Ld;
    const bool nrm = hist && l == 0;
    std::vector<int> np(d->parts.size(), 0);
    auto rows = [&](int phase) -> int {
      for (size_t q = 0; q < d->parts.size(); ++q) {
        DDPart& P = d->parts[q];
        StreamArgs a = dd_args(d, l, s);
        a.f = d->view(P.f[l], P.R0[l], l);
        a.u = z ? nullptr : d->view(P.u[l], P.R0[l], l);
        a.uo = d->view(P.t[l], P.R0[l], l);
        if (last) {
          // restricted residual straight into this part's slot of the gather layout
          const int cc = d->cols(La);
          a.rc = d->gather + (int64_t)P.part * d->Bc * cc - (int64_t)(P.R0[l] / 2) * cc;
        } else {
          a.rc = d->view(P.f[l + 1], P.R0[l + 1], l + 1);   // (dense: levels >= 1 are never padded)
        }
        if (int st = launch_rows(d, l, P, a, nu1, true, false, nrm, phase, &np[q])) return st;
      }
      return MGB_OK;
    };
    auto xch = [&](cudaStream_t x) -> int {
      if (!z)
        if (int st = exchange(d, l, 0, x)) return st;
      if (l > 0)
        if (int st = exchange(d, l, 2, x)) return st;
      return MGB_OK;
    };
    if (int st = exchange_and_pass(d, l, s, !z || l > 0, xch, rows)) return st;
    for (size_t q = 0; q < d->parts.size(); ++q) {
      DDPart& P = d->parts[q];
      if (nrm) MGB_CUDA_TRY(launch_finalize(1, np[q], P.partials, P.norm2, nullptr, nullptr, 0, s));
      std::swap(P.u[l], P.t[l]);
    }
    if (nrm) {
      if (int st = reduce_norm(d, d->r2, s)) return st;
      k_hist_entry<<<1, 32, 0, s>>>(d->r2, d->f2, hist);
      MGB_CUDA_TRY(cudaGetLastError());
    }
  }
  // agglomerate: every rank gets the whole restricted residual, solves the coarse part
  const int cc = d->cols(La);
  const size_t blkc = (size_t)d->Bc * cc;
  if (d->comm && d->do_exchange) {
    MGB_NCCL_TRY(nccl::api().AllGather(d->gather + (int64_t)d->first * blkc, d->gather, blkc, nccl::Float64,
                                       d->comm, s));
  }
  if (d->xfn && d->do_exchange) {
    MGB_CUDA_TRY(cudaStreamSynchronize(s));
    if (d->xfn(d->xctx, 1, -1, d->gather + (int64_t)d->first * blkc, d->gather, (int64_t)blkc))
      return fail(MGB_NCCL, "exchange callback failed (all-gather)");
  }
  if (d->nparts > 1 && d->do_exchange) d->halo_bytes += blkc * sizeof(double) * (d->comm || d->xfn ? 1 : d->nparts);
  double* cf = work_level_f(d->cw, La);
  double* cu = work_level_u(d->cw, La);
  MGB_CUDA_TRY(cudaMemcpyAsync(cf, d->gather, sizeof(double) * d->rows(La) * cc, cudaMemcpyDeviceToDevice, s));
  double* ec_full = nullptr;
  if (int st = work_vcycle_level(d->cw, La, cf, cu, true, nu1, nu2, s, &ec_full)) return st;
  // ascend
  for (int l = Ld - 1; l >= 0; --l) {
    int unused = 0;
    auto rows = [&](int phase) -> int {
      for (auto& P : d->parts) {
        StreamArgs a = dd_args(d, l, s);
        a.f = d->view(P.f[l], P.R0[l], l);
        a.u = d->view(P.u[l], P.R0[l], l);
        a.uo = d->view(P.t[l], P.R0[l], l);
        if (l + 1 < Ld) a.ec = d->view(P.u[l + 1], P.R0[l + 1], l + 1);
        else a.ec = ec_full;
        if (int st = launch_rows(d, l, P, a, nu2, false, true, false, phase, &unused)) return st;
      }
      return MGB_OK;
    };
    auto xch = [&](cudaStream_t x) -> int {
      if (int st = exchange(d, l, 0, x)) return st;
      if (l + 1 < Ld)
        if (int st = exchange(d, l + 1, 0, x)) return st;
      return MGB_OK;
    };
    if (int st = exchange_and_pass(d, l, s, true, xch, rows)) return st;
    for (auto& P : d->parts) std::swap(P.u[l], P.t[l]);
  }
  return MGB_OK;
}

extern "C" int mgb_dd_set_exchange(mgb_dd* d, mgb_dd_exchange_fn fn, void* ctx) {
  if (!d) return fail(MGB_CONTRACT, "null decomposition");
  if (d->comm) return fail(MGB_CONFIG, "this decomposition already exchanges through NCCL");
  if (d->nlocal != 1) return fail(MGB_CONFIG, "the callback backend holds one part per process");
  d->xfn = fn;
  d->xctx = ctx;
  return MGB_OK;
}

extern "C" int mgb_dd_set_option(mgb_dd* d, const char* key, int value) {
  if (!d || !key) return fail(MGB_CONTRACT, "null argument");
  const std::string k(key);
  if (k == "overlap") d->overlap = value != 0;
  else if (k == "exchange") d->do_exchange = value != 0;
  else return fail(MGB_CONFIG, "unknown decomposition option " + k);
  if (d->graph) cudaGraphExecDestroy(d->graph);   // the captured schedule depends on both
  d->graph = nullptr;
  return MGB_OK;
}

extern "C" int mgb_dd_stats(const mgb_dd* d, int64_t* sent_bytes, int* exchanges) {
  if (!d) return fail(MGB_CONTRACT, "null decomposition");
  if (sent_bytes) *sent_bytes = d->halo_bytes;
  if (exchanges) *exchanges = d->exchanges;
  return MGB_OK;
}

extern "C" int mgb_dd_set_rhs(mgb_dd* d, int part, const double* f_owned_dev, void* stream) {
  if (!d) return fail(MGB_CONTRACT, "null decomposition");
  const int q = part - d->first;
  if (q < 0 || q >= d->nlocal) return fail(MGB_CONFIG, "part not held by this process");
  DeviceGuard dg(d->device);
  DDPart& P = d->parts[q];
  const int cols = d->cols(0);
  MGB_CUDA_TRY(cudaMemcpy2DAsync(d->view(P.f[0], P.R0[0], 0) + (int64_t)P.R0[0] * d->pitch[0], sizeof(double) * d->pitch[0],
                                 f_owned_dev, sizeof(double) * cols, sizeof(double) * cols, (size_t)(P.R1[0] - P.R0[0]),
                                 cudaMemcpyDeviceToDevice, S(stream)));
  return MGB_OK;
}

extern "C" int mgb_dd_get_solution(const mgb_dd* d, int part, double* u_owned_dev, void* stream) {
  if (!d) return fail(MGB_CONTRACT, "null decomposition");
  const int q = part - d->first;
  if (q < 0 || q >= d->nlocal) return fail(MGB_CONFIG, "part not held by this process");
  DeviceGuard dg(d->device);
  const DDPart& P = d->parts[q];
  const int cols = d->cols(0);
  MGB_CUDA_TRY(cudaMemcpy2DAsync(u_owned_dev, sizeof(double) * cols,
                                 d->view(P.u[0], P.R0[0], 0) + (int64_t)P.R0[0] * d->pitch[0], sizeof(double) * d->pitch[0],
                                 sizeof(double) * cols, (size_t)(P.R1[0] - P.R0[0]), cudaMemcpyDeviceToDevice, S(stream)));
  return MGB_OK;
}

static int dd_enqueue(mgb_dd* d, int nu1, int nu2, int cycles, int u_zero, double* hist, cudaStream_t s) {
  d->halo_bytes = 0;
  d->exchanges = 0;
  if (int st = exchange(d, 0, 2, s)) return st;  // f ghosts of level 0
  if (int st = norm_pass(d, true, d->f2, s)) return st;
  for (int c = 0; c < cycles; ++c)
    if (int st = dd_cycle(d, nu1, nu2, u_zero && c == 0, hist + c, s)) return st;
  if (int st = norm_pass(d, false, d->r2, s)) return st;
  k_hist_entry<<<1, 32, 0, s>>>(d->r2, d->f2, hist + cycles);
  MGB_CUDA_TRY(cudaGetLastError());
  return MGB_OK;
}

extern "C" int mgb_dd_run_cycles(mgb_dd* d, int nu1, int nu2, int cycles, int u_zero, double* history_dev,
                                 void* stream) {
  if (!d) return fail(MGB_CONTRACT, "null decomposition");
  if ((nu1 != 1 && nu1 != 2) || (nu2 != 1 && nu2 != 2)) return fail(MGB_CONFIG, "decomposed cycles support V(1|2, 1|2)");
  if (cycles < 0 || !history_dev) return fail(MGB_CONFIG, "bad cycle count or history buffer");
  DeviceGuard dg(d->device);
  cudaStream_t s = S(stream);
  if (int st = work_prepare(d->cw)) return st;
  if (d->nlocal == 1 && d->nparts > 1 && !d->comm && !d->xfn)
    return fail(MGB_CONFIG, "this decomposition has neither an NCCL communicator nor an exchange callback");
  if (d->xfn) return dd_enqueue(d, nu1, nu2, cycles, u_zero, history_dev, s);   // eager: host exchanges
  // one CUDA graph per (nu1, nu2, cycles, u_zero, history) (halo copies / NCCL ops are captured too)
  const int key[4] = {nu1, nu2, cycles, u_zero};
  if (!d->graph || std::memcmp(key, d->gkey, sizeof(key)) != 0 || d->ghist != history_dev) {
    if (d->graph) cudaGraphExecDestroy(d->graph);
    d->graph = nullptr;
    cudaGraph_t g = nullptr;
    MGB_CUDA_TRY(cudaStreamBeginCapture(d->cap, cudaStreamCaptureModeThreadLocal));
    int st = dd_enqueue(d, nu1, nu2, cycles, u_zero, history_dev, d->cap);
    cudaError_t e = cudaStreamEndCapture(d->cap, &g);
    if (st) {
      if (g) cudaGraphDestroy(g);
      return st;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(&d->graph, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
    std::memcpy(d->gkey, key, sizeof(key));
    d->ghist = history_dev;
  }
  MGB_CUDA_TRY(cudaGraphLaunch(d->graph, s));
  return MGB_OK;
}
