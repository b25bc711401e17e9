// Pointwise compressible Navier-Stokes quantities, entry by entry.
//
// Device restatement of the reference's pointwise kernels
// (kernels/numba_backend.py:20-326, numpy twin kernels/numpy_backend.py:18-212)
// for d = 2, 3 (ns = d+2, lambda = -2/d).  Every Jacobian entry is a pure
// function of the point state, so a CTA can generate the (k,l,s,t) arrays
// with one thread per entry and fully coalesced stores, instead of one
// thread per point holding 225-entry register arrays.
#pragma once
#include "common.cuh"

namespace mhdg {

struct FlowC {
  double gamma, g1, mu_e, kg, lam, re_flow, svis_e, nu_supg;
};

template <int D>
__host__ __device__ inline FlowC make_flow(const mhdg_flow& f) {
  FlowC c;
  c.gamma = f.gamma;
  c.g1 = f.gamma - 1.0;
  c.mu_e = f.mu / f.re_acoustic;
  // k_t * gamma (gamma - 1), k_t = gamma mu / ((gamma-1) Re Pr)
  c.kg = f.gamma * f.mu / ((f.gamma - 1.0) * f.re_acoustic * f.prandtl) * f.gamma * (f.gamma - 1.0);
  c.lam = -2.0 / D;
  c.re_flow = f.re_flow;
  c.svis_e = 1.0 / ((f.gamma - 1.0) * f.mach_ref * f.mach_ref * f.prandtl);
  const double gp = f.gamma / f.prandtl;
  c.nu_supg = (f.mu / f.re_acoustic) * (4.0 / 3.0 > gp ? 4.0 / 3.0 : gp);
  return c;
}

template <int D>
struct Prim {
  double rho, irho, v[D], kin, P, H, c, et;  // irho = 1/rho: the Jacobian entries multiply by it
};

template <int D>
__device__ __forceinline__ Prim<D> prim(const double* u, const FlowC& f) {
  Prim<D> p;
  p.rho = u[0];
  p.irho = 1.0 / p.rho;
  p.kin = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    p.v[i] = u[1 + i] / p.rho;
    p.kin += 0.5 * p.v[i] * p.v[i];
  }
  p.et = u[D + 1];
  p.P = f.g1 * (p.et - p.rho * p.kin);
  p.H = (p.et + p.P) / p.rho;
  const double c2 = f.gamma * p.P / p.rho;
  p.c = sqrt(c2 > 1e-300 ? c2 : 1e-300);
  return p;
}

// admissibility (physics.py:85-94): 0 ok, 1 rho, 2 pressure
template <int D>
__device__ __forceinline__ int admissible_code(const double* u, double gamma) {
  const double rho = u[0];
  if (!(rho > 0.0) || !isfinite(rho)) return 1;
  double m2 = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) m2 += u[1 + i] * u[1 + i];
  const double pres = (gamma - 1.0) * (u[D + 1] - 0.5 * m2 / rho);
  if (!(pres > 0.0) || !isfinite(pres)) return 2;
  return 0;
}

// F[s][k]
template <int D>
__device__ __forceinline__ double euler_flux(const Prim<D>& p, const double* u, int s, int k) {
  if (s == 0) return u[1 + k];
  if (s <= D) return u[s] * p.v[k] + (s - 1 == k ? p.P : 0.0);
  return p.rho * p.H * p.v[k];
}

// A[k][s][t] = dF[s][k] / du_t
template <int D>
__device__ __forceinline__ double euler_jac(const Prim<D>& p, const FlowC& f, int k, int s, int t) {
  constexpr int E = D + 1;
  if (s == 0) return t == 1 + k ? 1.0 : 0.0;
  if (s <= D) {
    const int i = s - 1;
    if (t == 0) return -p.v[i] * p.v[k] + (i == k ? f.g1 * p.kin : 0.0);
    if (t <= D) {
      const int j = t - 1;
      return (j == k ? p.v[i] : 0.0) + (i == j ? p.v[k] : 0.0) - (i == k ? f.g1 * p.v[j] : 0.0);
    }
    return i == k ? f.g1 : 0.0;
  }
  // explicit FMA: left to the compiler, g1 kin - H is contracted in some inlining contexts and
  // not in others (k_assemble vs k_couplings differed by 1 ulp in this entry)
  if (t == 0) return p.v[k] * __fma_rn(f.g1, p.kin, -p.H);
  if (t <= D) {
    const int j = t - 1;
    return (j == k ? p.H : 0.0) - f.g1 * p.v[j] * p.v[k];
  }
  (void)E;
  return f.gamma * p.v[k];
}

// velocity gradient gvel[a][b] = d v_b / d x_a from conserved gradients q[a][s]
template <int D>
__device__ __forceinline__ double gvel(const Prim<D>& p, const double* q, int a, int b) {
  constexpr int NS = D + 2;
  return (q[a * NS + 1 + b] - p.v[b] * q[a * NS]) * p.irho;
}

template <int D>
__device__ __forceinline__ double tau_entry(const Prim<D>& p, const FlowC& f, const double* q, int i, int k) {
  double div = 0.0;
#pragma unroll
  for (int c = 0; c < D; ++c) div += gvel<D>(p, q, c, c);
  return f.mu_e * (gvel<D>(p, q, k, i) + gvel<D>(p, q, i, k) + (i == k ? f.lam * div : 0.0));
}

// d(internal energy)/dx_k
template <int D>
__device__ __forceinline__ double egrad(const Prim<D>& p, const double* q, int k) {
  constexpr int NS = D + 2;
  const double* qk = q + k * NS;
  double vq = 0.0, v2 = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    vq += p.v[j] * qk[1 + j];
    v2 += p.v[j] * p.v[j];
  }
  const double ir = p.irho;
  return qk[D + 1] * ir - p.et * qk[0] * (ir * ir) - vq * ir + v2 * qk[0] * ir;
}

// G[s][k]
template <int D>
__device__ __forceinline__ double visc_flux(const Prim<D>& p, const FlowC& f, const double* q, int s, int k) {
  if (s == 0) return 0.0;
  if (s <= D) return -tau_entry<D>(p, f, q, s - 1, k);
  double tv = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) tv += tau_entry<D>(p, f, q, k, j) * p.v[j];
  return -tv - f.kg * egrad<D>(p, q, k);
}

// g(b, t) = d gvel[a][b] / d q[a][t]
template <int D>
__device__ __forceinline__ double gq(const Prim<D>& p, int b, int t) {
  if (t == 1 + b) return p.irho;
  if (t == 0) return -p.v[b] * p.irho;
  return 0.0;
}

// d tau[i][k] / d q[l][t]
template <int D>
__device__ __forceinline__ double dtau_dq(const Prim<D>& p, const FlowC& f, int i, int k, int l, int t) {
  return f.mu_e * ((k == l ? gq<D>(p, i, t) : 0.0) + (i == l ? gq<D>(p, k, t) : 0.0) +
                   (i == k ? f.lam * gq<D>(p, l, t) : 0.0));
}

// dG[s][k] / dq[l][t] (independent of q)
template <int D>
__device__ __forceinline__ double visc_dgdq(const Prim<D>& p, const FlowC& f, int k, int l, int s, int t) {
  constexpr int E = D + 1;
  if (s == 0) return 0.0;
  if (s <= D) return -dtau_dq<D>(p, f, s - 1, k, l, t);
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) acc += p.v[j] * dtau_dq<D>(p, f, k, j, l, t);
  double out = -acc;
  if (k == l) {
    double h;
    if (t == 0) {
      double v2 = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) v2 += p.v[j] * p.v[j];
      h = -p.et * (p.irho * p.irho) + v2 * p.irho;
    } else if (t <= D) {
      h = -p.v[t - 1] * p.irho;
    } else {
      h = p.irho;
    }
    out -= f.kg * h;
  }
  (void)E;
  return out;
}

// d gvel[a][b] / d u_t
template <int D>
__device__ __forceinline__ double dgv_du(const Prim<D>& p, const double* q, int a, int b, int t) {
  constexpr int NS = D + 2;
  const double q0 = q[a * NS];
  if (t == 0) return (p.v[b] * p.irho * q0 - gvel<D>(p, q, a, b)) * p.irho;
  if (t == 1 + b) return -q0 * (p.irho * p.irho);
  return 0.0;
}

template <int D>
__device__ __forceinline__ double dtau_du(const Prim<D>& p, const FlowC& f, const double* q, int i, int k, int t) {
  double dd = 0.0;
  if (i == k) {
#pragma unroll
    for (int c = 0; c < D; ++c) dd += dgv_du<D>(p, q, c, c, t);
  }
  return f.mu_e * (dgv_du<D>(p, q, k, i, t) + dgv_du<D>(p, q, i, k, t) + (i == k ? f.lam * dd : 0.0));
}

// dG[s][k] / du_t
template <int D>
__device__ __forceinline__ double visc_dgdu(const Prim<D>& p, const FlowC& f, const double* q, int k, int s, int t) {
  constexpr int NS = D + 2, E = D + 1;
  if (s == 0) return 0.0;
  if (s <= D) return -dtau_du<D>(p, f, q, s - 1, k, t);
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    acc += dtau_du<D>(p, f, q, k, j, t) * p.v[j];
    double dv = 0.0;
    if (t == 0) dv = -p.v[j] * p.irho;
    else if (t == 1 + j) dv = p.irho;
    if (dv != 0.0) acc += tau_entry<D>(p, f, q, k, j) * dv;
  }
  const double* qk = q + k * NS;
  const double ir2 = p.irho * p.irho;
  double dge;
  if (t == 0) {
    double vq = 0.0, v2 = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      vq += p.v[j] * qk[1 + j];
      v2 += p.v[j] * p.v[j];
    }
    dge = -qk[E] * ir2 + 2.0 * p.et * qk[0] * (ir2 * p.irho) + 2.0 * vq * ir2 - 3.0 * v2 * qk[0] * ir2;
  } else if (t <= D) {
    dge = -qk[t] * ir2 + 2.0 * p.v[t - 1] * qk[0] * ir2;
  } else {
    dge = -qk[0] * ir2;
  }
  return -acc - f.kg * dge;
}

// interface stabilisation, diagonal: S[s][s] = |v.n| + c + svis[s]/Re_flow
template <int D>
__device__ __forceinline__ double stab_diag(const Prim<D>& p, const FlowC& f, const double* n, int s) {
  double vn = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) vn += p.v[i] * n[i];
  const double lam = fabs(vn) + p.c;
  double sv = 0.0;
  if (s >= 1 && s <= D) sv = 1.0;
  if (s == D + 1) sv = f.svis_e;
  return lam + sv / f.re_flow;
}

template <int D>
__device__ __forceinline__ double supg_tau(const Prim<D>& p, const FlowC& f, double h, double inv_dt) {
  double v2 = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) v2 += p.v[i] * p.v[i];
  const double lam = sqrt(v2) + p.c;
  const double t1 = 2.0 * inv_dt, t2 = 2.0 * lam / h, t3 = 12.0 * f.nu_supg / (h * h);
  return 1.0 / sqrt(t1 * t1 + t2 * t2 + t3 * t3);
}

}  // namespace mhdg
