// Matrix-free condensed trace operator and the per-macro solves around it.
//
// k_apply_local   CondensedSchur.apply_trace  (condense.py:91-103), local part,
//                 Algorithm 2 steps 1-4, one CTA per macro
// k_face_reduce   _scatter_add (condense.py:48-51), deterministic two-sided sum
// k_rhs_local     CondensedSchur.rhs          (condense.py:105-110)
// k_recover       CondensedSchur.recover      (condense.py:112-127)
// k_grad_refresh  Discretization.gradient_refresh (assembly.py:247-252)
// k_lu_solve      CondensedSchur._schur_solve (condense.py:80-83) with LU factors
#include "local_ops.cuh"
#include "tiled_inv.cuh"

namespace mhdg {

constexpr int APPLY_THREADS = 256;

struct ApplySmem {
  int xl, z, y, cfgz, acc, tmp, big, vv, wv, cv, wf, z2, cfg2, total;
};

template <int D>
__host__ __device__ inline ApplySmem apply_smem(const Sz& s) {
  constexpr int NS = D + 2, NF = D + 1;
  ApplySmem m;
  int o = 0;
  m.xl = o; o += s.ltr;
  m.z = o; o += D * s.L * NS;
  m.y = o; o += s.n;
  m.cfgz = o; o += s.ltr;
  m.acc = o; o += s.ltr;
  m.tmp = o; o += (s.n > s.ltr ? s.n : s.ltr);
  m.big = o;
  const int nwf = NF * s.n_tri * s.nqf * NS;
  // phase C: vv | wv | cv | wf     phase E: z2 | wf | cfg2
  m.vv = o;
  m.wv = m.vv + s.pc * D * NS;
  m.cv = m.wv + s.pc * D * NS;
  m.wf = m.cv + s.n_sub * s.nloc * NS;
  int endC = m.wf + nwf;
  m.z2 = o;
  int wf2 = m.z2 + D * s.L * NS;
  if (wf2 > m.wf) m.wf = wf2;  // wf must not overlap z2
  endC = m.wf + nwf;
  m.cfg2 = endC;
  m.total = endC + s.ltr;
  return m;
}

template <int D>
__global__ void __launch_bounds__(APPLY_THREADS) k_apply_local(mhdg_disc g, mhdg_blocks b, mhdg_factors fac,
                                                               const double* __restrict__ x,
                                                               double* __restrict__ y_loc) {
  extern __shared__ double sm[];
  const Sz sz = make_sz<D>(g);
  const ApplySmem o = apply_smem<D>(sz);
  const int mac = blockIdx.x;
  double *xl = sm + o.xl, *z = sm + o.z, *y = sm + o.y, *cfgz = sm + o.cfgz, *acc = sm + o.acc,
         *tmp = sm + o.tmp;

  const int* gat = g.gather + (size_t)mac * sz.ltr;
  for (int i = threadIdx.x; i < sz.ltr; i += blockDim.x) xl[i] = __ldg(x + __ldg(gat + i));
  __syncthreads();
  // step 1: z = A_qq^-1 A_qh x ;  y1 = -A_uh x + A_uq z
  grad_trace_solve<D>(g, sz, mac, xl, z, false, 1.0);
  state_trace<D>(g, b, sz, mac, xl, tmp, y, false, -1.0);
  __syncthreads();
  state_grad<D>(g, b, sz, mac, z, sm + o.vv, sm + o.wv, sm + o.cv, sm + o.wf, cfgz, y, true, 1.0);
  // step 2: y2 = S^-1 y1
  factor_solve_cta(fac, mac, sz.n, y, tmp);
  for (int i = threadIdx.x; i < sz.n; i += blockDim.x) y[i] = tmp[i];
  __syncthreads();
  // steps 3-4: y4 = A_hu y2 - A_hq A_qq^-1 A_qu y2 + A_hh x - A_hq z
  double* z2 = sm + o.z2;
  grad_state_solve<D>(g, sz, mac, y, z2, false, 1.0);
  __syncthreads();
  face_stash_nodes<D>(g, b, sz, mac, z2, sm + o.wf, sm + o.cfg2);
  trace_state<D>(g, b, sz, mac, y, tmp, acc, false, 1.0);
  trace_grad_from_cfg<D>(b, sz, mac, sm + o.cfg2, acc, -1.0);
  __syncthreads();
  trace_trace<D>(b, sz, mac, xl, acc, true, 1.0);
  trace_grad_from_cfg<D>(b, sz, mac, cfgz, acc, -1.0);
  __syncthreads();
  double* out = y_loc + (size_t)mac * sz.ltr;
  for (int i = threadIdx.x; i < sz.ltr; i += blockDim.x) out[i] = acc[i];
}

// y[dof] = add[dof]*add_sign + (y_loc[src0] + y_loc[src1]); the pair is summed
// lower flat index first, as np.add.at does.
__global__ void k_face_reduce(int n_trace, const int* __restrict__ src, const double* __restrict__ y_loc,
                              const double* __restrict__ add, double add_sign, double* __restrict__ y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_trace; i += gridDim.x * blockDim.x) {
    const int a = __ldg(src + 2 * i), c = __ldg(src + 2 * i + 1);
    double v = __ldg(y_loc + a);
    if (c >= 0) v += __ldg(y_loc + c);
    y[i] = add ? add_sign * __ldg(add + i) + v : v;
  }
}

template <int D>
__global__ void __launch_bounds__(APPLY_THREADS) k_rhs_local(mhdg_disc g, mhdg_blocks b, mhdg_factors fac,
                                                             const double* __restrict__ R_grad,
                                                             const double* __restrict__ R_state,
                                                             double* __restrict__ b_loc) {
  extern __shared__ double sm[];
  constexpr int NS = D + 2;
  const Sz sz = make_sz<D>(g);
  const ApplySmem o = apply_smem<D>(sz);
  const int mac = blockIdx.x;
  double *zr = sm + o.z, *y = sm + o.y, *cfgz = sm + o.cfgz, *acc = sm + o.acc, *tmp = sm + o.tmp;
  mass_solve<D>(g, sz, mac, R_grad + (size_t)mac * D * sz.L * NS, zr);
  for (int i = threadIdx.x; i < sz.n; i += blockDim.x) y[i] = __ldg(R_state + (size_t)mac * sz.n + i);
  __syncthreads();
  // t2 = S^-1 (R_U - A_uq zr)
  state_grad<D>(g, b, sz, mac, zr, sm + o.vv, sm + o.wv, sm + o.cv, sm + o.wf, cfgz, y, true, -1.0);
  factor_solve_cta(fac, mac, sz.n, y, tmp);
  for (int i = threadIdx.x; i < sz.n; i += blockDim.x) y[i] = tmp[i];
  __syncthreads();
  // b_loc = (A_hu t2 - A_hq A_qq^-1 A_qu t2) + A_hq zr
  double* z2 = sm + o.z2;
  grad_state_solve<D>(g, sz, mac, y, z2, false, 1.0);
  __syncthreads();
  face_stash_nodes<D>(g, b, sz, mac, z2, sm + o.wf, sm + o.cfg2);
  trace_state<D>(g, b, sz, mac, y, tmp, acc, false, 1.0);
  trace_grad_from_cfg<D>(b, sz, mac, sm + o.cfg2, acc, -1.0);
  __syncthreads();
  trace_grad_from_cfg<D>(b, sz, mac, cfgz, acc, 1.0);
  __syncthreads();
  for (int i = threadIdx.x; i < sz.ltr; i += blockDim.x) b_loc[(size_t)mac * sz.ltr + i] = acc[i];
}

struct RecSmem {
  int xl, z, zr, y, w, tmp, dblk, big, total;
};

template <int D>
__global__ void __launch_bounds__(APPLY_THREADS) k_recover(mhdg_disc g, mhdg_blocks b, mhdg_factors fac,
                                                           const double* __restrict__ R_grad,
                                                           const double* __restrict__ R_state,
                                                           const double* __restrict__ dtrace,
                                                           double* __restrict__ du, double* __restrict__ dq) {
  extern __shared__ double sm[];
  constexpr int NS = D + 2;
  const Sz sz = make_sz<D>(g);
  const ApplySmem o = apply_smem<D>(sz);
  const int mac = blockIdx.x;
  // reuse the apply layout: z -> z, cfgz -> (face sums), extra vectors after o.total
  double *xl = sm + o.xl, *z = sm + o.z, *y = sm + o.y, *cfg = sm + o.cfgz, *tmp = sm + o.tmp;
  double *zr = sm + o.total, *w = zr + D * sz.L * NS;
  const int* gat = g.gather + (size_t)mac * sz.ltr;
  for (int i = threadIdx.x; i < sz.ltr; i += blockDim.x) xl[i] = __ldg(dtrace + __ldg(gat + i));
  mass_solve<D>(g, sz, mac, R_grad + (size_t)mac * D * sz.L * NS, zr);
  __syncthreads();
  grad_trace_solve<D>(g, sz, mac, xl, z, false, 1.0);
  state_trace<D>(g, b, sz, mac, xl, tmp, y, false, -1.0);
  __syncthreads();
  state_grad<D>(g, b, sz, mac, z, sm + o.vv, sm + o.wv, sm + o.cv, sm + o.wf, cfg, y, true, 1.0);
  state_grad<D>(g, b, sz, mac, zr, sm + o.vv, sm + o.wv, sm + o.cv, sm + o.wf, cfg, w, false, 1.0);
  for (int i = threadIdx.x; i < sz.n; i += blockDim.x)
    y[i] = (w[i] - __ldg(R_state + (size_t)mac * sz.n + i)) + y[i];
  __syncthreads();
  factor_solve_cta(fac, mac, sz.n, y, tmp);
  for (int i = threadIdx.x; i < sz.n; i += blockDim.x) y[i] = tmp[i];
  __syncthreads();
  for (int i = threadIdx.x; i < sz.n; i += blockDim.x) du[(size_t)mac * sz.n + i] = y[i];
  double* z2 = sm + o.z2;
  grad_state_solve<D>(g, sz, mac, y, z2, false, 1.0);
  __syncthreads();
  for (int i = threadIdx.x; i < D * sz.L * NS; i += blockDim.x)
    dq[(size_t)mac * D * sz.L * NS + i] = (-zr[i] - z2[i]) - z[i];
}

template <int D>
__global__ void __launch_bounds__(APPLY_THREADS) k_grad_refresh(mhdg_disc g, const double* __restrict__ u,
                                                                const double* __restrict__ uhat,
                                                                double* __restrict__ q) {
  extern __shared__ double sm[];
  constexpr int NS = D + 2;
  const Sz sz = make_sz<D>(g);
  const int mac = blockIdx.x;
  double *xl = sm, *y = xl + sz.ltr, *z = y + sz.n;
  const int* gat = g.gather + (size_t)mac * sz.ltr;
  for (int i = threadIdx.x; i < sz.ltr; i += blockDim.x) xl[i] = __ldg(uhat + __ldg(gat + i));
  for (int i = threadIdx.x; i < sz.n; i += blockDim.x) y[i] = __ldg(u + (size_t)mac * sz.n + i);
  __syncthreads();
  grad_state_solve<D>(g, sz, mac, y, z, false, -1.0);
  __syncthreads();
  grad_trace_solve<D>(g, sz, mac, xl, z, true, -1.0);
  __syncthreads();
  for (int i = threadIdx.x; i < D * sz.L * NS; i += blockDim.x) q[(size_t)mac * D * sz.L * NS + i] = z[i];
}

__global__ void __launch_bounds__(APPLY_THREADS) k_lu_solve(int n, mhdg_factors fac, const double* __restrict__ b,
                                                            double* __restrict__ yout) {
  extern __shared__ double sm[];
  const int mac = blockIdx.x;
  double *y = sm, *tmp = y + n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) y[i] = b[(size_t)mac * n + i];
  __syncthreads();
  factor_solve_cta(fac, mac, n, y, tmp);
  for (int i = threadIdx.x; i < n; i += blockDim.x) y[i] = tmp[i];
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) yout[(size_t)mac * n + i] = y[i];
}

// zr = A_qq^-1 R_Q for every macro (the first step of rhs / recover, condense.py:105-127),
// into global memory for the streamed rhs / recovery (apply_stream.cu: cond_stream)
template <int D>
__global__ void __launch_bounds__(APPLY_THREADS) k_mass_solve(mhdg_disc g, const double* __restrict__ R_grad,
                                                              double* __restrict__ zr) {
  constexpr int NS = D + 2;
  const Sz sz = make_sz<D>(g);
  const size_t off = (size_t)blockIdx.x * D * sz.L * NS;
  mass_solve<D>(g, sz, blockIdx.x, R_grad + off, zr + off);
}

// The tail of the streamed recovery: du = y2 (the factor solve's output in the split
// apply's work buffer), dq = -zr - A_qq^-1 A_qu du - A_qq^-1 A_qh dtrace (condense.py:112-127)
template <int D>
__global__ void __launch_bounds__(APPLY_THREADS) k_recover_dq(mhdg_disc g, const double* __restrict__ dtrace,
                                                              const double* __restrict__ zr,
                                                              const double* __restrict__ y2, long long y2_stride,
                                                              double* __restrict__ du, double* __restrict__ dq) {
  extern __shared__ double sm[];
  constexpr int NS = D + 2;
  const Sz sz = make_sz<D>(g);
  const int mac = blockIdx.x;
  double *xl = sm, *y = xl + sz.ltr, *z = y + sz.n, *z2 = z + D * sz.L * NS;
  const int* gat = g.gather + (size_t)mac * sz.ltr;
  const double* y2m = y2 + (size_t)mac * y2_stride;
  for (int i = threadIdx.x; i < sz.ltr; i += blockDim.x) xl[i] = __ldg(dtrace + __ldg(gat + i));
  for (int i = threadIdx.x; i < sz.n; i += blockDim.x) {
    const double v = y2m[i];
    y[i] = v;
    du[(size_t)mac * sz.n + i] = v;
  }
  __syncthreads();
  grad_trace_solve<D>(g, sz, mac, xl, z, false, 1.0);
  grad_state_solve<D>(g, sz, mac, y, z2, false, 1.0);
  __syncthreads();
  const double* zrm = zr + (size_t)mac * D * sz.L * NS;
  for (int i = threadIdx.x; i < D * sz.L * NS; i += blockDim.x)
    dq[(size_t)mac * D * sz.L * NS + i] = (-zrm[i] - z2[i]) - z[i];
}

template <int D>
int mass_solve_all(const mhdg_disc& g, const double* R_grad, double* zr, cudaStream_t st) {
  k_mass_solve<D><<<g.n_mac, APPLY_THREADS, 0, st>>>(g, R_grad, zr);
  return launch_ok();
}

template <int D>
int recover_dq(const mhdg_disc& g, const double* dtrace, const double* zr, const double* y2, long long y2_stride,
               double* du, double* dq, cudaStream_t st) {
  const Sz sz = make_sz<D>(g);
  const size_t bytes = sizeof(double) * ((size_t)sz.ltr + sz.n + 2 * (size_t)D * sz.L * (D + 2));
  if (bytes > 48 * 1024) cudaFuncSetAttribute(k_recover_dq<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  k_recover_dq<D><<<g.n_mac, APPLY_THREADS, bytes, st>>>(g, dtrace, zr, y2, y2_stride, du, dq);
  return launch_ok();
}

template int mass_solve_all<2>(const mhdg_disc&, const double*, double*, cudaStream_t);
template int mass_solve_all<3>(const mhdg_disc&, const double*, double*, cudaStream_t);
template int recover_dq<2>(const mhdg_disc&, const double*, const double*, const double*, long long, double*, double*,
                           cudaStream_t);
template int recover_dq<3>(const mhdg_disc&, const double*, const double*, const double*, long long, double*, double*,
                           cudaStream_t);

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------

template <typename K>
static void set_smem(K kern, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int D>
int apply_local(const mhdg_disc& g, const mhdg_blocks& b, const mhdg_factors& f, const double* x, double* y_loc,
                cudaStream_t st) {
  const Sz sz = make_sz<D>(g);
  const size_t bytes = sizeof(double) * apply_smem<D>(sz).total;
  set_smem(k_apply_local<D>, bytes);
  k_apply_local<D><<<g.n_mac, APPLY_THREADS, bytes, st>>>(g, b, f, x, y_loc);
  return launch_ok();
}

int face_reduce(const mhdg_disc& g, const double* y_loc, const double* add, double add_sign, double* y,
                cudaStream_t st) {
  const int threads = 256;
  int blocks = (g.n_trace + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_face_reduce<<<blocks, threads, 0, st>>>(g.n_trace, g.scatter_src, y_loc, add, add_sign, y);
  return launch_ok();
}

template <int D>
int rhs_local(const mhdg_disc& g, const mhdg_blocks& b, const mhdg_factors& f, const double* Rg, const double* Ru,
              double* b_loc, cudaStream_t st) {
  const Sz sz = make_sz<D>(g);
  const size_t bytes = sizeof(double) * apply_smem<D>(sz).total;
  set_smem(k_rhs_local<D>, bytes);
  k_rhs_local<D><<<g.n_mac, APPLY_THREADS, bytes, st>>>(g, b, f, Rg, Ru, b_loc);
  return launch_ok();
}

template <int D>
int recover(const mhdg_disc& g, const mhdg_blocks& b, const mhdg_factors& f, const double* Rg, const double* Ru,
            const double* dtr, double* du, double* dq, cudaStream_t st) {
  const Sz sz = make_sz<D>(g);
  const size_t bytes = sizeof(double) * (apply_smem<D>(sz).total + D * sz.L * (D + 2) + sz.n);
  set_smem(k_recover<D>, bytes);
  k_recover<D><<<g.n_mac, APPLY_THREADS, bytes, st>>>(g, b, f, Rg, Ru, dtr, du, dq);
  return launch_ok();
}

template <int D>
int grad_refresh(const mhdg_disc& g, const double* u, const double* uhat, double* q, cudaStream_t st) {
  const Sz sz = make_sz<D>(g);
  const size_t bytes = sizeof(double) * (sz.ltr + sz.n + D * sz.L * (D + 2));
  set_smem(k_grad_refresh<D>, bytes);
  k_grad_refresh<D><<<g.n_mac, APPLY_THREADS, bytes, st>>>(g, u, uhat, q);
  return launch_ok();
}

int lu_solve(const mhdg_disc& g, const mhdg_factors& f, const double* bvec, double* y, cudaStream_t st) {
  const int n = g.L * g.ns;
  const size_t bytes = sizeof(double) * 2 * n;
  set_smem(k_lu_solve, bytes);
  k_lu_solve<<<g.n_mac, APPLY_THREADS, bytes, st>>>(n, f, bvec, y);
  return launch_ok();
}

template int apply_local<2>(const mhdg_disc&, const mhdg_blocks&, const mhdg_factors&, const double*, double*, cudaStream_t);
template int apply_local<3>(const mhdg_disc&, const mhdg_blocks&, const mhdg_factors&, const double*, double*, cudaStream_t);
template int rhs_local<2>(const mhdg_disc&, const mhdg_blocks&, const mhdg_factors&, const double*, const double*, double*, cudaStream_t);
template int rhs_local<3>(const mhdg_disc&, const mhdg_blocks&, const mhdg_factors&, const double*, const double*, double*, cudaStream_t);
template int recover<2>(const mhdg_disc&, const mhdg_blocks&, const mhdg_factors&, const double*, const double*, const double*, double*, double*, cudaStream_t);
template int recover<3>(const mhdg_disc&, const mhdg_blocks&, const mhdg_factors&, const double*, const double*, const double*, double*, double*, cudaStream_t);
template int grad_refresh<2>(const mhdg_disc&, const double*, const double*, double*, cudaStream_t);
template int grad_refresh<3>(const mhdg_disc&, const double*, const double*, double*, cudaStream_t);

}  // namespace mhdg
