// Per-macro block actions of the condensed HDG operator, executed by one CTA
// per macro-element with every intermediate in shared memory.
//
// These are the factored block applications of the reference
// (assembly.py:255-283 structural gradient blocks, assembly.py:643-718
// stash-based A_uq / A_hq and dense face blocks) restated for a CTA:
//   grad_trace_solve   z  = A_qq^-1 A_qh x       (grad_mass_solve o grad_trace_apply)
//   grad_state_solve   z  = A_qq^-1 A_qu y       (grad_mass_solve o _grad_state_apply)
//   mass_solve         z  = A_qq^-1 r            (grad_mass_solve)
//   state_trace        y  = A_uh x               (state_trace_apply)
//   state_grad         y  = A_uq z + face part   (state_grad_apply), also returns
//                      the per-face-node sums reused by trace_grad_apply
//   trace_state        t  = A_hu y               (trace_state_apply)
//   trace_trace        t  = A_hh x               (trace_trace_apply)
// Deterministic: every accumulation runs in a fixed order through the
// inverse-incidence tables (no atomics).
#pragma once
#include "common.cuh"

namespace mhdg {

template <int D>
struct Dims {
  static constexpr int NS = D + 2;
  static constexpr int NF = D + 1;
};

// Sizes derived once per launch.
struct Sz {
  int L, Lf, n, bs, ltr, n_sub, nloc, nq, n_tri, nlocf, nqf, kc, pc;
};

template <int D>
__host__ __device__ inline Sz make_sz(const mhdg_disc& g) {
  Sz s;
  s.L = g.L;
  s.Lf = g.Lf;
  s.n = g.L * (D + 2);
  s.bs = g.Lf * (D + 2);
  s.ltr = (D + 1) * s.bs;
  s.n_sub = g.n_sub;
  s.nloc = g.nloc;
  s.nq = g.nq;
  s.n_tri = g.n_tri;
  s.nlocf = g.nlocf;
  s.nqf = g.nqf;
  // sub-elements per chunk of the volume-stash pass (<= 64 points per chunk)
  s.kc = g.nq >= 64 ? 1 : 64 / g.nq;
  if (s.kc > g.n_sub) s.kc = g.n_sub;
  s.pc = s.kc * g.nq;
  return s;
}

// z[l][I][s] = (A_qq^-1 A_qh xl), with Gf = M^-1[:, fvn[f]] Mf precomputed:
// z = -(fac/det) sum_f area_f n_f,l Gf xl_f.
template <int D>
__device__ void grad_trace_solve(const mhdg_disc& g, const Sz& sz, int mac, const double* xl,
                                 double* z, bool accumulate, double sign) {
  constexpr int NS = D + 2, NF = D + 1;
  const double idet = 1.0 / __ldg(g.det + mac);
  for (int idx = threadIdx.x; idx < sz.L * NS; idx += blockDim.x) {
    const int I = idx / NS, s = idx - I * NS;
    double acc[D];
#pragma unroll
    for (int l = 0; l < D; ++l) acc[l] = 0.0;
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      const double* gr = g.gf + ((size_t)f * sz.L + I) * sz.Lf;
      const double* xf = xl + f * sz.bs + s;
      double t = 0.0;
      for (int h = 0; h < sz.Lf; ++h) t += __ldg(gr + h) * xf[h * NS];
      const double c = -g.face_fac * __ldg(g.areas + mac * NF + f) * idet * t;
#pragma unroll
      for (int l = 0; l < D; ++l) acc[l] += c * __ldg(g.normals + (mac * NF + f) * D + l);
    }
#pragma unroll
    for (int l = 0; l < D; ++l) {
      double* o = z + (l * sz.L + I) * NS + s;
      *o = accumulate ? *o + sign * acc[l] : sign * acc[l];
    }
  }
}

// z[l][I][s] (+)= sign * sum_r inv_jac[r][l] (M^-1 D_r y)[I][s]
template <int D>
__device__ void grad_state_solve(const mhdg_disc& g, const Sz& sz, int mac, const double* y,
                                 double* z, bool accumulate, double sign) {
  constexpr int NS = D + 2;
  const double* ij = g.inv_jac + (size_t)mac * D * D;
  for (int idx = threadIdx.x; idx < sz.L * NS; idx += blockDim.x) {
    const int I = idx / NS, s = idx - I * NS;
    double t[D];
#pragma unroll
    for (int r = 0; r < D; ++r) {
      const double* row = g.minv_d + ((size_t)r * sz.L + I) * sz.L;
      double a = 0.0;
      for (int J = 0; J < sz.L; ++J) a += __ldg(row + J) * y[J * NS + s];
      t[r] = a;
    }
#pragma unroll
    for (int l = 0; l < D; ++l) {
      double v = 0.0;
#pragma unroll
      for (int r = 0; r < D; ++r) v += __ldg(ij + r * D + l) * t[r];
      double* o = z + (l * sz.L + I) * NS + s;
      *o = accumulate ? *o + sign * v : sign * v;
    }
  }
}

// z[l][I][s] = (1/det) sum_J M^-1[I][J] r[l][J][s]   (r from global memory)
template <int D>
__device__ void mass_solve(const mhdg_disc& g, const Sz& sz, int mac, const double* __restrict__ r,
                           double* z) {
  constexpr int NS = D + 2;
  const double idet = 1.0 / __ldg(g.det + mac);
  for (int idx = threadIdx.x; idx < D * sz.L * NS; idx += blockDim.x) {
    const int s = idx % NS, I = (idx / NS) % sz.L, l = idx / (NS * sz.L);
    const double* row = g.mass_inv + (size_t)I * sz.L;
    const double* rl = r + (size_t)l * sz.L * NS + s;
    double a = 0.0;
    for (int J = 0; J < sz.L; ++J) a += __ldg(row + J) * __ldg(rl + J * NS);
    z[idx] = idet * a;
  }
}

// out[I][s] = sum over faces f with fvn[f][g] = I of t[(f Lf + g) NS + s], in face order.
template <int D>
__device__ void gather_face_to_nodes(const mhdg_disc& g, const Sz& sz, const double* t, double* out,
                                     bool accumulate, double sign) {
  constexpr int NS = D + 2;
  for (int idx = threadIdx.x; idx < sz.L * NS; idx += blockDim.x) {
    const int I = idx / NS, s = idx - I * NS;
    double acc = 0.0;
    for (int e = __ldg(g.vf_ptr + I); e < __ldg(g.vf_ptr + I + 1); ++e)
      acc += t[__ldg(g.vf_ent + e) * NS + s];
    out[idx] = accumulate ? out[idx] + sign * acc : sign * acc;
  }
}

// tmp[f][row] = (face_state_trace[f] xl_f)[row]; then out (+)= sign * node gather.
template <int D>
__device__ void state_trace(const mhdg_disc& g, const mhdg_blocks& b, const Sz& sz, int mac,
                            const double* xl, double* tmp, double* out, bool accumulate, double sign) {
  constexpr int NF = D + 1;
  for (int f = 0; f < NF; ++f)
    warp_gemv<false>(b.face_state_trace + ((size_t)mac * NF + f) * sz.bs * sz.bs, sz.bs, sz.bs,
                     xl + f * sz.bs, tmp + f * sz.bs, 1.0);
  __syncthreads();
  gather_face_to_nodes<D>(g, sz, tmp, out, accumulate, sign);
}

// Face-stash contraction at every face quadrature point, then summed onto face
// nodes: cfg[f][g][s] = sum_{(T,a): tc[T,a]=g} sum_q phi_f[q,a] wf[(f,T,q)][s],
// wf[s] = sum_{l,t} wdgdq_face[mac,f,T nqf+q][l][s][t] v[l][t], v = z at the point.
template <int D>
__device__ void face_stash_nodes(const mhdg_disc& g, const mhdg_blocks& b, const Sz& sz, int mac,
                                 const double* z, double* wf, double* cfg) {
  constexpr int NS = D + 2, NF = D + 1;
  const int npf = NF * sz.n_tri * sz.nqf;
  for (int idx = threadIdx.x; idx < npf * NS; idx += blockDim.x) {
    const int s = idx % NS, pf = idx / NS;
    const int q = pf % sz.nqf, T = (pf / sz.nqf) % sz.n_tri, f = pf / (sz.nqf * sz.n_tri);
    double v[D][NS];
#pragma unroll
    for (int l = 0; l < D; ++l)
#pragma unroll
      for (int t = 0; t < NS; ++t) v[l][t] = 0.0;
    for (int a = 0; a < sz.nlocf; ++a) {
      const double ph = __ldg(g.phi_face + q * sz.nlocf + a);
      const int node = __ldg(g.face_vol_nodes + f * sz.Lf + __ldg(g.tri_conn + T * sz.nlocf + a));
#pragma unroll
      for (int l = 0; l < D; ++l)
#pragma unroll
        for (int t = 0; t < NS; ++t) v[l][t] += ph * z[(l * sz.L + node) * NS + t];
    }
    const double* W = b.wdgdq_face + (((size_t)mac * NF + f) * sz.n_tri * sz.nqf + T * sz.nqf + q) * D * NS * NS;
    double acc = 0.0;
#pragma unroll
    for (int l = 0; l < D; ++l)
#pragma unroll
      for (int t = 0; t < NS; ++t) acc += __ldg(W + (l * NS + s) * NS + t) * v[l][t];
    wf[idx] = acc;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < NF * sz.Lf * NS; idx += blockDim.x) {
    const int s = idx % NS, gg = (idx / NS) % sz.Lf, f = idx / (NS * sz.Lf);
    double acc = 0.0;
    for (int e = __ldg(g.fn_ptr + gg); e < __ldg(g.fn_ptr + gg + 1); ++e) {
      const int ent = __ldg(g.fn_ent + e), T = ent / sz.nlocf, a = ent - T * sz.nlocf;
      const double* w = wf + ((f * sz.n_tri + T) * sz.nqf) * NS + s;
      for (int q = 0; q < sz.nqf; ++q) acc += __ldg(g.phi_face + q * sz.nlocf + a) * w[q * NS];
    }
    cfg[idx] = acc;
  }
  __syncthreads();
}

// y[I][s] (+)= sign * (A_uq z)[I][s].  Volume part streamed in chunks of kc
// sub-elements (vv/wv hold pc*D*NS values each), face part through
// face_stash_nodes (cfg is left holding the per-face-node sums).
template <int D>
__device__ void state_grad(const mhdg_disc& g, const mhdg_blocks& b, const Sz& sz, int mac,
                           const double* z, double* vv, double* wv, double* cv, double* wf,
                           double* cfg, double* y, bool accumulate, double sign) {
  constexpr int NS = D + 2;
  const double* ij = g.inv_jac + (size_t)mac * D * D;
  const size_t wbase = (size_t)mac * sz.n_sub * sz.nq;
  for (int K0 = 0; K0 < sz.n_sub; K0 += sz.kc) {
    const int kc = min(sz.kc, sz.n_sub - K0), np = kc * sz.nq;
    // (a) z at the chunk's quadrature points
    for (int idx = threadIdx.x; idx < np * D * NS; idx += blockDim.x) {
      const int t = idx % NS, l = (idx / NS) % D, p = idx / (NS * D);
      const int K = K0 + p / sz.nq, q = p % sz.nq;
      double a = 0.0;
      for (int bb = 0; bb < sz.nloc; ++bb)
        a += __ldg(g.phi_vol + q * sz.nloc + bb) * z[(l * sz.L + __ldg(g.sub_conn + K * sz.nloc + bb)) * NS + t];
      vv[idx] = a;
    }
    __syncthreads();
    // (b) w[k][s] = sum_{l,t} wdgdq_vol[k][l][s][t] v[l][t]
    for (int idx = threadIdx.x; idx < np * D * NS; idx += blockDim.x) {
      const int s = idx % NS, k = (idx / NS) % D, p = idx / (NS * D);
      const double* W = b.wdgdq_vol + (wbase + K0 * sz.nq + p) * D * D * NS * NS + k * D * NS * NS + s * NS;
      const double* v = vv + p * D * NS;
      double a = 0.0;
#pragma unroll
      for (int l = 0; l < D; ++l)
#pragma unroll
        for (int t = 0; t < NS; ++t) a += __ldg(W + l * NS * NS + t) * v[l * NS + t];
      wv[idx] = a;
    }
    __syncthreads();
    // (c) c[K][a][s] = sum_q sum_k gphys[K,q,a,k] w[K,q][k][s]
    for (int idx = threadIdx.x; idx < kc * sz.nloc * NS; idx += blockDim.x) {
      const int s = idx % NS, a = (idx / NS) % sz.nloc, kk = idx / (NS * sz.nloc), K = K0 + kk;
      double acc = 0.0;
      for (int q = 0; q < sz.nq; ++q) {
        const double* gr = g.grad_ref + (((size_t)K * sz.nq + q) * sz.nloc + a) * D;
        const double* w = wv + ((kk * sz.nq + q) * D) * NS + s;
#pragma unroll
        for (int k = 0; k < D; ++k) {
          double gp = 0.0;
#pragma unroll
          for (int r = 0; r < D; ++r) gp += __ldg(gr + r) * __ldg(ij + r * D + k);
          acc += gp * w[k * NS];
        }
      }
      cv[(K * sz.nloc + a) * NS + s] = acc;
    }
    __syncthreads();
  }
  face_stash_nodes<D>(g, b, sz, mac, z, wf, cfg);
  // out[I][s] = -(sum of volume contributions) + (sum of face contributions)
  for (int idx = threadIdx.x; idx < sz.L * NS; idx += blockDim.x) {
    const int I = idx / NS, s = idx - I * NS;
    double acc = 0.0;
    for (int e = __ldg(g.vn_ptr + I); e < __ldg(g.vn_ptr + I + 1); ++e) acc -= cv[__ldg(g.vn_sub + e) * NS + s];
    for (int e = __ldg(g.vf_ptr + I); e < __ldg(g.vf_ptr + I + 1); ++e) acc += cfg[__ldg(g.vf_ent + e) * NS + s];
    y[idx] = accumulate ? y[idx] + sign * acc : sign * acc;
  }
  __syncthreads();
}

// out[f][row] (+)= sign * (face_trace_state[f] y|_{fvn[f]})[row]; yf is scratch (ltr).
template <int D>
__device__ void trace_state(const mhdg_disc& g, const mhdg_blocks& b, const Sz& sz, int mac,
                            const double* y, double* yf, double* out, bool accumulate, double sign) {
  constexpr int NS = D + 2, NF = D + 1;
  for (int idx = threadIdx.x; idx < sz.ltr; idx += blockDim.x) {
    const int t = idx % NS, h = (idx / NS) % sz.Lf, f = idx / sz.bs;
    yf[idx] = y[__ldg(g.face_vol_nodes + f * sz.Lf + h) * NS + t];
  }
  __syncthreads();
  for (int f = 0; f < NF; ++f) {
    const double* A = b.face_trace_state + ((size_t)mac * NF + f) * sz.bs * sz.bs;
    if (accumulate)
      warp_gemv<true>(A, sz.bs, sz.bs, yf + f * sz.bs, out + f * sz.bs, sign);
    else
      warp_gemv<false>(A, sz.bs, sz.bs, yf + f * sz.bs, out + f * sz.bs, sign);
  }
  __syncthreads();
}

template <int D>
__device__ void trace_trace(const mhdg_blocks& b, const Sz& sz, int mac, const double* xl, double* out,
                            bool accumulate, double sign) {
  constexpr int NF = D + 1;
  for (int f = 0; f < NF; ++f) {
    const double* A = b.face_trace_trace + ((size_t)mac * NF + f) * sz.bs * sz.bs;
    if (accumulate)
      warp_gemv<true>(A, sz.bs, sz.bs, xl + f * sz.bs, out + f * sz.bs, sign);
    else
      warp_gemv<false>(A, sz.bs, sz.bs, xl + f * sz.bs, out + f * sz.bs, sign);
  }
  __syncthreads();
}

// out[f][g][s] (+)= sign * trace_grad_apply(z)[f][g][s] = -sign * scale_f * cfg[f][g][s]
template <int D>
__device__ void trace_grad_from_cfg(const mhdg_blocks& b, const Sz& sz, int mac, const double* cfg,
                                    double* out, double sign) {
  constexpr int NS = D + 2, NF = D + 1;
  for (int idx = threadIdx.x; idx < sz.ltr; idx += blockDim.x) {
    const int f = idx / sz.bs;
    out[idx] += -sign * __ldg(b.trace_face_scale + mac * NF + f) * cfg[idx];
  }
  (void)NS;
}

}  // namespace mhdg
