// extern "C" boundary (include/mhdg.h; A/B knobs in mhdg_tuning.h): dispatch on the
// dimension and launch.
#include "mhdg_tuning.h"
#include "common.cuh"
#include "packed_lu.cuh"
#include "tiled_inv.cuh"

namespace mhdg {
long long g_launches = 0;

template <int D> int apply_local(const mhdg_disc&, const mhdg_blocks&, const mhdg_factors&, const double*, double*, cudaStream_t);
template <int D> int rhs_local(const mhdg_disc&, const mhdg_blocks&, const mhdg_factors&, const double*, const double*, double*, cudaStream_t);
template <int D> int recover(const mhdg_disc&, const mhdg_blocks&, const mhdg_factors&, const double*, const double*, const double*, double*, double*, cudaStream_t);
template <int D> int grad_refresh(const mhdg_disc&, const double*, const double*, double*, cudaStream_t);
template <int D> int schur_matrix(const mhdg_disc&, const mhdg_blocks&, double*, cudaStream_t);
template <int D> int assemble(const mhdg_disc&, const mhdg_flow&, const mhdg_stage&, const double*, const double*,
                              const double*, double*, double*, double*, double*, int, const mhdg_blocks*,
                              const mhdg_frozen*, const mhdg_frozen*, int*, cudaStream_t);
template <int D> int precond_build(const mhdg_disc&, const mhdg_blocks&, const double*, double*, int*, cudaStream_t);
template <int D> int face_sum_window(const mhdg_disc&, const mhdg_blocks&, int, int, double*, cudaStream_t);
template <int D> int side_blocks(const mhdg_disc&, const mhdg_blocks&, const int*, const int*, int, double*, cudaStream_t);
int precond_apply(const mhdg_disc&, const double*, const double*, double*, cudaStream_t);
int face_reduce(const mhdg_disc&, const double*, const double*, double, double*, cudaStream_t);
int lu_solve(const mhdg_disc&, const mhdg_factors&, const double*, double*, cudaStream_t);
int inv_factor(int n, int n_mac, double* scratch, double* tiled, int* status, cudaStream_t st);
int inv_factor3(int n, int n_mac, double* scratch, int* piv, double* tiled, int* status, cudaStream_t st);
int lu_factor4(int n, int n_mac, double* scratch, int* piv, double* packed, int* status, cudaStream_t st);
int lu_max_n();
extern int g_schur_variant;
int icgs(int n, int j, const double* V, long long ldv, double* w, double* out, double* scratch, cudaStream_t st);
int vec_pass_api(long long n, int rows, const double* V, long long ldv, double* w, const double* coef, int mode,
                 double* out, double* scratch, cudaStream_t st);
long long icgs_scratch_size(int n);
size_t gj_smem_bytes(int n);
int apply_stream(const mhdg_disc&, const mhdg_blocks&, const mhdg_factors&, const double*, double*, cudaStream_t);
int cond_stream(const mhdg_disc& g, const mhdg_blocks& b, const mhdg_factors& f, bool rhs, const double* Rg,
                const double* Ru, const double* dtrace, double* y_loc, double* du, double* dq, cudaStream_t st);
int halo_gather(long long n, const int* idx, const double* src, double* buf, cudaStream_t st);
int halo_scatter(long long n, const int* idx, const double* buf, double* dst, int accumulate, cudaStream_t st);
int face_reduce_remote(const mhdg_disc& g, const double* y_loc, const int* remote_src, const double* remote,
                       int n_out, double* y, cudaStream_t st);
}  // namespace mhdg

using namespace mhdg;

#define DISPATCH(g, call2, call3) \
  ((g)->dim == 2 ? (call2) : (g)->dim == 3 ? (call3) : MHDG_ERR_CONFIG)

static inline cudaStream_t S(void* s) { return (cudaStream_t)s; }

// ---- per-kernel timeline ----
namespace mhdg {
static bool g_tl_on = false;
static int g_tl_cap = 0, g_tl_used = 0;
static cudaEvent_t* g_tl_ev = nullptr;  // 2 per record
static int* g_tl_slot = nullptr;
static int g_tl_open[TL_NSLOTS];

void tl_begin(int slot, cudaStream_t st) {
  if (!g_tl_on || g_tl_used >= g_tl_cap) return;
  g_tl_open[slot] = g_tl_used;
  g_tl_slot[g_tl_used] = slot;
  cudaEventRecord(g_tl_ev[2 * g_tl_used], st);
  ++g_tl_used;
}

void tl_end(int slot, cudaStream_t st) {
  if (!g_tl_on || g_tl_open[slot] < 0) return;
  cudaEventRecord(g_tl_ev[2 * g_tl_open[slot] + 1], st);
  g_tl_open[slot] = -1;
}
}  // namespace mhdg

extern "C" {

int mhdg_icgs(int n, int j, const double* V, long long ldv, double* w, double* out, double* scratch, void* st) {
  return icgs(n, j, V, ldv, w, out, scratch, S(st));
}

long long mhdg_icgs_scratch_size(int n) { return icgs_scratch_size(n); }

int mhdg_vec_pass(long long n, int rows, const double* V, long long ldv, double* w, const double* coef, int mode,
                  double* out, double* scratch, void* st) {
  return vec_pass_api(n, rows, V, ldv, w, coef, mode, out, scratch, S(st));
}

int mhdg_timeline_begin(int capacity) {
  if (capacity > g_tl_cap) {
    for (int i = 0; i < 2 * g_tl_cap; ++i) cudaEventDestroy(g_tl_ev[i]);
    delete[] g_tl_ev;
    delete[] g_tl_slot;
    g_tl_ev = new cudaEvent_t[2 * capacity];
    g_tl_slot = new int[capacity];
    for (int i = 0; i < 2 * capacity; ++i)
      if (cudaEventCreate(&g_tl_ev[i]) != cudaSuccess) return MHDG_ERR_CUDA;
    g_tl_cap = capacity;
  }
  g_tl_used = 0;
  for (int i = 0; i < TL_NSLOTS; ++i) g_tl_open[i] = -1;
  g_tl_on = true;
  return MHDG_OK;
}

int mhdg_timeline_end(double* ms, int* counts) {
  g_tl_on = false;
  for (int i = 0; i < TL_NSLOTS; ++i) {
    ms[i] = 0.0;
    counts[i] = 0;
  }
  if (g_tl_used && cudaEventSynchronize(g_tl_ev[2 * g_tl_used - 1]) != cudaSuccess) return MHDG_ERR_CUDA;
  for (int r = 0; r < g_tl_used; ++r) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, g_tl_ev[2 * r], g_tl_ev[2 * r + 1]) != cudaSuccess) return MHDG_ERR_CUDA;
    ms[g_tl_slot[r]] += t;
    counts[g_tl_slot[r]] += 1;
  }
  return MHDG_OK;
}


long long mhdg_launch_count(void) { return g_launches; }

long long mhdg_packed_lu_size(int n) { return ti_size(n) > plu_size(n) ? ti_size(n) : plu_size(n); }

long long mhdg_apply_work_size(const mhdg_disc* g) {
  const long long n = (long long)g->L * g->ns, np = n + (n & 1), ltr = (long long)g->nf * g->Lf * g->ns;
  return (long long)g->n_mac * (2 * np + 2 * ltr);
}

static int g_stream_enabled = 1;
void mhdg_set_stream_enabled(int on) { g_stream_enabled = on; }

int mhdg_apply_trace_local(const mhdg_disc* g, const mhdg_blocks* b, const mhdg_factors* f, const double* x,
                           double* y_loc, void* st) {
  // compile-time specialised, TMA-streamed kernel when one matches (dim, m, p)
  if (g_stream_enabled) {
    const int rc = apply_stream(*g, *b, *f, x, y_loc, S(st));
    if (rc >= 0) return rc;
  }
  tl_begin(TL_APPLY_GENERIC, S(st));
  const int rc2 =
      DISPATCH(g, apply_local<2>(*g, *b, *f, x, y_loc, S(st)), apply_local<3>(*g, *b, *f, x, y_loc, S(st)));
  tl_end(TL_APPLY_GENERIC, S(st));
  return rc2;
}

// views of the macro range [mac0, mac0 + count): every per-macro array offset by mac0
// (mhdg.h layouts); the factors' scratch is offset only when it holds every macro
// blocks_resident = false: `b` already holds the window only (the coupling-recompute
// representation's chunk buffers), so it is not offset
static void macro_view(const mhdg_disc* g, const mhdg_blocks* b, const mhdg_factors* f, int mac0, int count,
                       mhdg_disc* gv, mhdg_blocks* bv, mhdg_factors* fv, bool blocks_resident = true) {
  const size_t m0 = (size_t)mac0, d = g->dim, nf = g->nf, ns = g->ns, n = (size_t)g->L * ns;
  const size_t bs = (size_t)g->Lf * ns, ltr = nf * bs, nqf_f = (size_t)g->n_tri * g->nqf;
  *gv = *g;
  gv->n_mac = count;
  gv->det += m0;
  gv->inv_jac += m0 * d * d;
  gv->normals += m0 * nf * d;
  gv->areas += m0 * nf;
  gv->h_sub += m0 * g->n_sub;
  gv->gather += m0 * ltr;
  if (gv->bc_kind) gv->bc_kind += m0 * nf;
  if (gv->wall_e) gv->wall_e += m0 * nf;
  if (gv->wall_u) gv->wall_u += m0 * nf * d;
  if (gv->u_dir) gv->u_dir += m0 * nf * nqf_f * ns;
  if (gv->source) gv->source += m0 * g->n_sub * g->nq * ns;
  *bv = *b;
  if (blocks_resident) {
  bv->state_state += m0 * n * n;
  bv->face_state_trace += m0 * nf * bs * bs;
  bv->face_trace_state += m0 * nf * bs * bs;
  bv->face_trace_trace += m0 * nf * bs * bs;
  bv->wdgdq_vol += m0 * g->n_sub * g->nq * d * d * ns * ns;
  bv->wdgdq_face += m0 * nf * nqf_f * d * ns * ns;
  bv->trace_face_scale += m0 * nf;
  }
  *fv = *f;
  if (fv->lu) fv->lu += m0 * (size_t)mhdg_packed_lu_size((int)n);
  if (fv->perm) fv->perm += m0 * n;
  if (fv->scratch && (f->scratch_macros <= 0 || f->scratch_macros >= g->n_mac)) fv->scratch += m0 * n * n;
  if (fv->work) fv->work += m0 * (size_t)(mhdg_apply_work_size(g) / g->n_mac);
}

int mhdg_apply_trace_local_range(const mhdg_disc* g, const mhdg_blocks* b, const mhdg_factors* f, const double* x,
                                 double* y_loc, int mac0, int count, void* st) {
  if (mac0 < 0 || count < 0 || mac0 + count > g->n_mac) return MHDG_ERR_CONFIG;
  if (count == 0) return MHDG_OK;
  mhdg_disc gv;
  mhdg_blocks bv;
  mhdg_factors fv;
  macro_view(g, b, f, mac0, count, &gv, &bv, &fv);
  return mhdg_apply_trace_local(&gv, &bv, &fv, x, y_loc + (size_t)mac0 * g->nf * g->Lf * g->ns, st);
}

// ---- coupling-recompute representation (B_min): window entry points ----
// `bw` holds the blocks of macros [mac0, mac0 + count) only; factors and vectors are whole-mesh.
static bool window_ok(const mhdg_disc* g, int mac0, int count) {
  return mac0 >= 0 && count >= 0 && mac0 + count <= g->n_mac;
}

int mhdg_assemble_window(const mhdg_disc* g, const mhdg_flow* fl, const mhdg_stage* sg, const double* u, const double* q,
                         const double* uhat, double* Rg_w, double* Ru_w, double* Rtl_w, int want_jac,
                         const mhdg_blocks* bw, const mhdg_frozen* fo_w, int mac0, int count, int* status, void* st) {
  if (!window_ok(g, mac0, count)) return MHDG_ERR_CONFIG;
  if (count == 0) return MHDG_OK;
  mhdg_disc gv;
  mhdg_blocks bv;
  mhdg_factors fv{}, f0{};
  const mhdg_blocks b0{};
  macro_view(g, bw ? bw : &b0, &f0, mac0, count, &gv, &bv, &fv, false);
  const size_t n = (size_t)g->L * g->ns;
  mhdg_stage sv = *sg;
  if (sv.hist) sv.hist += (size_t)mac0 * n;
  tl_begin(TL_ASSEMBLE, S(st));
  const double *uw = u + (size_t)mac0 * n, *qw = q + (size_t)mac0 * g->dim * n;
  const int rc = DISPATCH(g, assemble<2>(gv, *fl, sv, uw, qw, uhat, Rg_w, Ru_w, Rtl_w, nullptr, want_jac, bw ? &bv : nullptr,
                                         fo_w, nullptr, status, S(st)),
                          assemble<3>(gv, *fl, sv, uw, qw, uhat, Rg_w, Ru_w, Rtl_w, nullptr, want_jac, bw ? &bv : nullptr,
                                      fo_w, nullptr, status, S(st)));
  tl_end(TL_ASSEMBLE, S(st));
  return rc;
}

int mhdg_condense_window(const mhdg_disc* g, const mhdg_blocks* bw, const mhdg_factors* f, int mac0, int count,
                         int* status, void* st) {
  if (!window_ok(g, mac0, count)) return MHDG_ERR_CONFIG;
  if (count == 0) return MHDG_OK;
  if (f->scratch_macros > 0 && f->scratch_macros < count) return MHDG_ERR_CONFIG;
  mhdg_disc gv;
  mhdg_blocks bv;
  mhdg_factors fv;
  macro_view(g, bw, f, mac0, count, &gv, &bv, &fv, false);
  fv.scratch_macros = 0;  // the view's scratch holds the whole window
  int rc = mhdg_schur_matrix(&gv, &bv, &fv, st);
  if (!rc) rc = mhdg_lu_factor(&gv, &fv, status, st);
  return rc;
}

int mhdg_apply_trace_local_window(const mhdg_disc* g, const mhdg_blocks* bw, const mhdg_factors* f, const double* x,
                                  double* y_loc, int mac0, int count, void* st) {
  if (!window_ok(g, mac0, count)) return MHDG_ERR_CONFIG;
  if (count == 0) return MHDG_OK;
  mhdg_disc gv;
  mhdg_blocks bv;
  mhdg_factors fv;
  macro_view(g, bw, f, mac0, count, &gv, &bv, &fv, false);
  return mhdg_apply_trace_local(&gv, &bv, &fv, x, y_loc + (size_t)mac0 * g->nf * g->Lf * g->ns, st);
}

int mhdg_condensed_rhs_local_window(const mhdg_disc* g, const mhdg_blocks* bw, const mhdg_factors* f, const double* Rg,
                                    const double* Ru, double* b_loc, int mac0, int count, void* st) {
  if (!window_ok(g, mac0, count)) return MHDG_ERR_CONFIG;
  if (count == 0) return MHDG_OK;
  mhdg_disc gv;
  mhdg_blocks bv;
  mhdg_factors fv;
  macro_view(g, bw, f, mac0, count, &gv, &bv, &fv, false);
  fv.scratch_macros = 0;
  const size_t n = (size_t)g->L * g->ns, ltr = (size_t)g->nf * g->Lf * g->ns;
  const double *rg = Rg + (size_t)mac0 * g->dim * n, *ru = Ru + (size_t)mac0 * n;
  double* bl = b_loc + (size_t)mac0 * ltr;
  if (g_stream_enabled) {
    const int rs = cond_stream(gv, bv, fv, true, rg, ru, nullptr, bl, nullptr, nullptr, S(st));
    if (rs >= 0) return rs;
  }
  return DISPATCH(g, rhs_local<2>(gv, bv, fv, rg, ru, bl, S(st)), rhs_local<3>(gv, bv, fv, rg, ru, bl, S(st)));
}

int mhdg_recover_window(const mhdg_disc* g, const mhdg_blocks* bw, const mhdg_factors* f, const double* Rg,
                        const double* Ru, const double* dtr, double* du, double* dq, int mac0, int count, void* st) {
  if (!window_ok(g, mac0, count)) return MHDG_ERR_CONFIG;
  if (count == 0) return MHDG_OK;
  mhdg_disc gv;
  mhdg_blocks bv;
  mhdg_factors fv;
  macro_view(g, bw, f, mac0, count, &gv, &bv, &fv, false);
  fv.scratch_macros = 0;
  const size_t n = (size_t)g->L * g->ns;
  const double *rg = Rg + (size_t)mac0 * g->dim * n, *ru = Ru + (size_t)mac0 * n;
  double *duw = du + (size_t)mac0 * n, *dqw = dq + (size_t)mac0 * g->dim * n;
  if (g_stream_enabled) {
    const int rs = cond_stream(gv, bv, fv, false, rg, ru, dtr, nullptr, duw, dqw, S(st));
    if (rs >= 0) return rs;
  }
  return DISPATCH(g, recover<2>(gv, bv, fv, rg, ru, dtr, duw, dqw, S(st)),
                  recover<3>(gv, bv, fv, rg, ru, dtr, duw, dqw, S(st)));
}

int mhdg_face_sum_window(const mhdg_disc* g, const mhdg_blocks* bw, double* sums, int mac0, int count, void* st) {
  if (!window_ok(g, mac0, count)) return MHDG_ERR_CONFIG;
  if (count == 0) return MHDG_OK;
  return DISPATCH(g, face_sum_window<2>(*g, *bw, mac0, count, sums, S(st)),
                  face_sum_window<3>(*g, *bw, mac0, count, sums, S(st)));
}

int mhdg_precond_build_sums(const mhdg_disc* g, const double* sums, double* inv, int* status, void* st) {
  const mhdg_blocks none{};
  return DISPATCH(g, precond_build<2>(*g, none, sums, inv, status, S(st)),
                  precond_build<3>(*g, none, sums, inv, status, S(st)));
}

int mhdg_face_reduce_axpy(const mhdg_disc* g, const double* y_loc, const double* add, double alpha, double* y,
                          void* st) {
  return face_reduce(*g, y_loc, add, alpha, y, S(st));
}

int mhdg_halo_gather(long long n, const int* idx, const double* src, double* buf, void* st) {
  return halo_gather(n, idx, src, buf, S(st));
}

int mhdg_halo_scatter(long long n, const int* idx, const double* buf, double* dst, int accumulate, void* st) {
  return halo_scatter(n, idx, buf, dst, accumulate, S(st));
}

int mhdg_face_reduce_remote(const mhdg_disc* g, const double* y_loc, const int* remote_src, const double* remote,
                            int n_out, double* y, void* st) {
  return face_reduce_remote(*g, y_loc, remote_src, remote, n_out, y, S(st));
}

int mhdg_face_reduce(const mhdg_disc* g, const double* y_loc, double* y, void* st) {
  tl_begin(TL_FACE_REDUCE, S(st));
  const int rc = face_reduce(*g, y_loc, nullptr, 0.0, y, S(st));
  tl_end(TL_FACE_REDUCE, S(st));
  return rc;
}

int mhdg_apply_trace(const mhdg_disc* g, const mhdg_blocks* b, const mhdg_factors* f, const double* x, double* y,
                     double* y_loc, void* st) {
  int rc = mhdg_apply_trace_local(g, b, f, x, y_loc, st);
  if (rc) return rc;
  return mhdg_face_reduce(g, y_loc, y, st);
}

int mhdg_condensed_rhs(const mhdg_disc* g, const mhdg_blocks* b, const mhdg_factors* f, const double* Rg,
                       const double* Ru, const double* Rt, double* bvec, double* b_loc, void* st) {
  // the split apply's streamed kernels when an instantiation matches, else the generic kernel
  if (g_stream_enabled) {
    const int rs = cond_stream(*g, *b, *f, true, Rg, Ru, nullptr, b_loc, nullptr, nullptr, S(st));
    if (rs > 0) return rs;
    if (rs == 0) return face_reduce(*g, b_loc, Rt, -1.0, bvec, S(st));
  }
  int rc = DISPATCH(g, rhs_local<2>(*g, *b, *f, Rg, Ru, b_loc, S(st)), rhs_local<3>(*g, *b, *f, Rg, Ru, b_loc, S(st)));
  if (rc) return rc;
  return face_reduce(*g, b_loc, Rt, -1.0, bvec, S(st));
}

int mhdg_recover(const mhdg_disc* g, const mhdg_blocks* b, const mhdg_factors* f, const double* Rg,
                 const double* Ru, const double* dtr, double* du, double* dq, void* st) {
  if (g_stream_enabled) {
    // the streamed pre part writes its face terms into the work buffer only; y_loc is unused
    const int rs = cond_stream(*g, *b, *f, false, Rg, Ru, dtr, nullptr, du, dq, S(st));
    if (rs >= 0) return rs;
  }
  return DISPATCH(g, recover<2>(*g, *b, *f, Rg, Ru, dtr, du, dq, S(st)),
                  recover<3>(*g, *b, *f, Rg, Ru, dtr, du, dq, S(st)));
}

int mhdg_gradient_refresh(const mhdg_disc* g, const double* u, const double* uhat, double* q, void* st) {
  return DISPATCH(g, grad_refresh<2>(*g, u, uhat, q, S(st)), grad_refresh<3>(*g, u, uhat, q, S(st)));
}

int mhdg_schur_matrix(const mhdg_disc* g, const mhdg_blocks* b, const mhdg_factors* f, void* st) {
  tl_begin(TL_SCHUR, S(st));
  const int rc =
      DISPATCH(g, schur_matrix<2>(*g, *b, f->scratch, S(st)), schur_matrix<3>(*g, *b, f->scratch, S(st)));
  tl_end(TL_SCHUR, S(st));
  return rc;
}

void mhdg_set_schur_variant(int v) { mhdg::g_schur_variant = v; }

int mhdg_factor_max_n(int kind) {
  if (kind == 1) return lu_max_n();
  int n = 384;  // k_gj3; beyond it k_gj while its 32-column panel fits shared memory
  while (gj_smem_bytes(n + 1) <= 227 * 1024) ++n;
  return n;
}

int mhdg_lu_factor(const mhdg_disc* g, const mhdg_factors* f, int* status, void* st) {
  const int n = g->L * g->ns;
  if (f->kind == 1) {  // packed LU (lu.cu)
    const int rc1 = lu_factor4(n, g->n_mac, f->scratch, f->perm, f->lu, status, S(st));
    return rc1 < 0 ? MHDG_ERR_CONFIG : rc1;
  }
  // explicit inverse: DMMA panel-64 Gauss-Jordan when its panel fits shared memory, else
  // the 32-column FFMA one
  const int rc = inv_factor3(n, g->n_mac, f->scratch, f->perm, f->lu, status, S(st));
  if (rc >= 0) return rc;
  if (gj_smem_bytes(n) > 227 * 1024) return MHDG_ERR_CONFIG;
  return inv_factor(n, g->n_mac, f->scratch, f->lu, status, S(st));
}

int mhdg_condense(const mhdg_disc* g, const mhdg_blocks* b, const mhdg_factors* f, int* status, void* st) {
  const int chunk = f->scratch_macros;
  if (chunk <= 0 || chunk >= g->n_mac) {
    int rc = mhdg_schur_matrix(g, b, f, st);
    if (rc) return rc;
    return mhdg_lu_factor(g, f, status, st);
  }
  // scratch for `chunk` macros: Schur + factor + pack chunk by chunk
  for (int c0 = 0; c0 < g->n_mac; c0 += chunk) {
    const int cnt = g->n_mac - c0 < chunk ? g->n_mac - c0 : chunk;
    mhdg_disc gv;
    mhdg_blocks bv;
    mhdg_factors fv;
    macro_view(g, b, f, c0, cnt, &gv, &bv, &fv);
    int rc = mhdg_schur_matrix(&gv, &bv, &fv, st);
    if (!rc) rc = mhdg_lu_factor(&gv, &fv, status, st);
    if (rc) return rc;
  }
  return MHDG_OK;
}

int mhdg_lu_solve(const mhdg_disc* g, const mhdg_factors* f, const double* bvec, double* y, void* st) {
  return lu_solve(*g, *f, bvec, y, S(st));
}

int mhdg_assemble(const mhdg_disc* g, const mhdg_flow* fl, const mhdg_stage* sg, const double* u, const double* q,
                  const double* uhat, double* Rg, double* Ru, double* Rtl, double* Rt, int want_jac,
                  const mhdg_blocks* b, const mhdg_frozen* fo, const mhdg_frozen* fi, int* status, void* st) {
  tl_begin(TL_ASSEMBLE, S(st));
  const int rc = DISPATCH(g, assemble<2>(*g, *fl, *sg, u, q, uhat, Rg, Ru, Rtl, Rt, want_jac, b, fo, fi, status, S(st)),
                          assemble<3>(*g, *fl, *sg, u, q, uhat, Rg, Ru, Rtl, Rt, want_jac, b, fo, fi, status, S(st)));
  tl_end(TL_ASSEMBLE, S(st));
  return rc;
}

int mhdg_precond_build(const mhdg_disc* g, const mhdg_blocks* b, double* inv, int* status, void* st) {
  return DISPATCH(g, precond_build<2>(*g, *b, nullptr, inv, status, S(st)),
                  precond_build<3>(*g, *b, nullptr, inv, status, S(st)));
}

int mhdg_precond_build_ext(const mhdg_disc* g, const mhdg_blocks* b, const double* extra, double* inv, int* status,
                           void* st) {
  return DISPATCH(g, precond_build<2>(*g, *b, extra, inv, status, S(st)),
                  precond_build<3>(*g, *b, extra, inv, status, S(st)));
}

int mhdg_side_blocks(const mhdg_disc* g, const mhdg_blocks* b, const int* macs, const int* lfs, int count, double* out,
                     void* st) {
  return DISPATCH(g, side_blocks<2>(*g, *b, macs, lfs, count, out, S(st)),
                  side_blocks<3>(*g, *b, macs, lfs, count, out, S(st)));
}

int mhdg_precond_apply(const mhdg_disc* g, const double* inv, const double* v, double* y, void* st) {
  return precond_apply(*g, inv, v, y, S(st));
}

}  // extern "C"
