// Domain decomposition driver (mgb_dd.cu) and the hierarchy accessors it uses.
#pragma once

#include "mgb_stream.h"

#define DD_GHOST 6  // ghost rows per block edge: the streaming passes read S + 1 <= 6 rows across

struct mgb_work;
struct mgb_dd;

namespace mgb {
int hier_rows(const mgb_hier* h, int l);
int hier_cols(const mgb_hier* h, int l);
int hier_batch(const mgb_hier* h);
int hier_depth(const mgb_hier* h);
int hier_device(const mgb_hier* h);
int hier_level_ks(const mgb_hier* h, int l);
bool hier_level_classed(const mgb_hier* h, int l);
bool hier_level_conv(const mgb_hier* h, int l);
const uint8_t* hier_mask(const mgb_hier* h, int l);
int hier_a5(const mgb_hier* h, int l);
Grid hier_grid(const mgb_hier* h, int l);
Op hier_opA(const mgb_hier* h, int l);
Op hier_opK(const mgb_hier* h, int l);
void hier_interior(const mgb_hier* h, int l, int* valid, double* ci, int* uniform = nullptr, int* kernel = nullptr,
                   double* kq = nullptr);
int work_create_from(const mgb_hier* h, int first, mgb_work** out);
double* work_level_u(mgb_work* w, int l);
double* work_level_f(mgb_work* w, int l);
int work_prepare(mgb_work* w);
const mgb_hier* work_hier(const mgb_work* w);
int work_vcycle_level(mgb_work* w, int l, const double* f, double* u, bool zero, int nu1, int nu2, cudaStream_t s,
                      double** result);
}  // namespace mgb
