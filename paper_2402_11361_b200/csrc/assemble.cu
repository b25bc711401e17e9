// Residual and Jacobian assembly, one CTA per macro-element.
//
// Restates assemble_system (assembly.py:339-618) of the reference:
//   R_Q   = J M Q + weak-derivative(U) - face term(Uhat)      (assembly.py:360-365)
//   R_U   = temporal mass + volume flux/source/SUPG terms      (assembly.py:367-457)
//           + face numerical fluxes                           (assembly.py:477-533)
//   R_hat = interior: -int phi [(F+G)(uhat).n + S(u-uhat)]; boundary: the
//           boundary-operator rows (Dirichlet / isothermal wall, optionally
//           moving)                                           (assembly.py:533-554)
//   Jacobian: state_state (flux, SUPG W1^T tau W1, SUPG temporal, mass/PTC,
//   face S), face_state_trace / face_trace_state / face_trace_trace with the
//   boundary rows, the w*dG/dq stashes and the frozen coefficients
//   (assembly.py:397-405, 459-475, 556-612).
// Per sub-element (and chunk of its quadrature points) the phases between CTA
// barriers are laid out so that all warps have work: interpolation one component
// per thread, pointwise Jacobians as (case, point) items whose entry indices are
// compile-time inside a case (pointwise.cuh folds to straight-line code), the
// sub-element's state_state contraction as two FP64 tensor-core GEMMs summed in a
// shared-memory tile (3D), the faces of a group through their per-point phases
// together with the face blocks formed entry by entry and written once.  Every
// accumulation runs in a fixed order (sub-element loop, sub-faces ascending,
// inverse-incidence gathers): results are bitwise reproducible run to run.
//
// k_couplings (end of this file) re-forms only the coupling blocks the trace apply streams
// (face blocks, dG/dq stashes) for the coupling-recompute representation (want_jac = 2).
#include <type_traits>

#include "dmma.cuh"
#include "local_ops.cuh"
#include "pointwise.cuh"
#include "tma.cuh"

namespace mhdg {

// threads per CTA (one macro per CTA; the work arrays fill shared memory, so one CTA per
// SM in 3D): measured 2D 256 (512: 18.3 -> 32.2 ms at C2), 3D 768 (256: 224 ms, 384: 188,
// 512: 170, 768: 159, 1024: 158 with 128 bytes of spills, at C3)
#ifndef MHDG_ASM_THREADS_3D
#define MHDG_ASM_THREADS_3D 384
#endif
#ifndef MHDG_ASM_CTAS_3D
#define MHDG_ASM_CTAS_3D 2
#endif
#ifndef MHDG_ASM_RES_THREADS_3D
#define MHDG_ASM_RES_THREADS_3D 320
#endif
#ifndef MHDG_ASM_RES_CTAS_3D
#define MHDG_ASM_RES_CTAS_3D 2
#endif
template <int D>
__host__ __device__ constexpr int asm_threads() { return D == 2 ? 256 : MHDG_ASM_THREADS_3D; }
// 3D: CTAs per SM the shared-memory budget is cut for (the volume points go in chunks that
// fit): the serial phases of one macro run under the parallel phases of another
template <int D>
__host__ __device__ constexpr int asm_ctas() { return D == 2 ? 1 : MHDG_ASM_CTAS_3D; }
// register budget (CTAs per SM in __launch_bounds__): the 2D work arrays are small enough
// for three CTAs per SM (C2: 64 KB each)
template <int D>
__host__ __device__ constexpr int asm_min_ctas() { return D == 2 ? 3 : MHDG_ASM_CTAS_3D; }

// The state_state contraction of a sub-element runs on the FP64 tensor cores: W1 is stored as
// the K x N matrix W1T[(q, u)][(a, s)] with row stride w1t_ld (= 4 mod 16: conflict-free DMMA
// fragments) and the sub-element's (nloc NS)^2 block is summed in the shared-memory tile Csm.
__host__ __device__ inline int w1t_ld(int nr) {
  int ld = (nr + 3) & ~3;
  while (ld % 16 != 4) ld += 4;
  return ld;
}
__host__ __device__ inline int csm_ld(int nr) { return (nr + 3) & ~1; }

// f(integral_constant<int, c>) for the runtime c in [0, N)
template <int I, int N>
struct StaticSwitch {
  template <class F>
  static __device__ __forceinline__ void run(int c, F& f) {
    if (c == I) f(std::integral_constant<int, I>{});
    else StaticSwitch<I + 1, N>::run(c, f);
  }
};
template <int N>
struct StaticSwitch<N, N> {
  template <class F>
  static __device__ __forceinline__ void run(int, F&) {}
};
template <int N, class F>
__device__ __forceinline__ void static_switch(int c, F f) {
  StaticSwitch<0, N>::run(c, f);
}

constexpr int ASM_MAXFLOC = 1024;  // n_tri x Lf entries of the sub-face node table

template <int D>
struct AsmSmem {
  int us, qs, uh, td, tf, gph, upt, qpt, wq, tq, prv, As, Adu, FG, Pp, sw, gus, tdps, rs, wts, W1, csm, cvol;
  int fuh, fu, fq, fuv, fw, fpr, fpv, fS, fK1, ffn, fbh, cf, ctr, total;
};

template <int D>
__host__ __device__ inline AsmSmem<D> asm_smem(const Sz& s0, int nqc, int nfg, bool jac = true) {
  Sz s = s0;
  s.nq = nqc;  // the volume per-point work arrays hold one chunk of points
  constexpr int NS = D + 2, NF = D + 1;
  constexpr int PRIM = (int)((sizeof(Prim<D>) + 7) / 8);
  AsmSmem<D> m;
  int o = 0;
#define TAKE(field, cnt) \
  m.field = o;           \
  o += (cnt);
  // kept for the whole macro
  TAKE(us, s.n)
  TAKE(qs, D * s.n)
  TAKE(uh, s.ltr)
  TAKE(td, s.n)
  TAKE(tf, s.ltr)
  TAKE(cvol, s.n_sub * s.nloc * NS)
  TAKE(cf, NF * s.n_tri * s.nlocf * NS)
  TAKE(ctr, NF * s.n_tri * s.nlocf * NS)
  // volume work arrays (one chunk of points of one sub-element) ...
  const int work = o;
  TAKE(gph, s.nq * s.nloc * D)
  TAKE(upt, s.nq * NS)
  TAKE(qpt, s.nq * D * NS)
  TAKE(wq, s.nq)
  TAKE(tq, s.nq)
  TAKE(prv, s.nq * PRIM)
  TAKE(As, s.nq * D * NS * NS)
  TAKE(Adu, jac ? s.nq * D * NS * NS : 0)  // residual-only launches: no Jacobian work arrays
  TAKE(FG, s.nq * NS * D)
  TAKE(Pp, s.nq * D * NS)
  TAKE(sw, s.nq * NS)
  TAKE(gus, s.nq * D * NS)
  TAKE(tdps, s.nq * NS)
  TAKE(rs, s.nq * NS)
  TAKE(wts, s.nq)
  TAKE(W1, jac ? s.nq * NS * w1t_ld(s.nloc * NS) : 0)
  TAKE(csm, jac ? s.nloc * NS * csm_ld(s.nloc * NS) : 0)
  const int vol_end = o;
  // ... share their memory with the face work arrays (all sub-faces of nfg faces)
  o = work;
  const int nqf_one = s.nqf;
  s.nqf = nfg * s.n_tri * nqf_one;
  TAKE(fuh, s.nqf * NS)
  TAKE(fu, s.nqf * NS)
  TAKE(fq, s.nqf * D * NS)
  TAKE(fuv, s.nqf * NS)
  TAKE(fw, s.nqf)
  TAKE(fpr, s.nqf * PRIM)
  TAKE(fpv, s.nqf * PRIM)
  TAKE(fS, s.nqf * NS * NS)
  TAKE(fK1, s.nqf * NS * NS)
  TAKE(ffn, s.nqf * NS)
  TAKE(fbh, s.nqf * NS)
  if (o < vol_end) o = vol_end;
  s.nqf = nqf_one;
#undef TAKE
  m.total = o;
  return m;
}

// Interpolate nodal state (and gradient) to one quadrature point.
template <int D>
__device__ __forceinline__ void interp_point(const double* ph, int nb, const int* nodes, const int* nmap,
                                             const double* src, int src_stride_l, const double* qs, int L,
                                             double* uu, double* qv) {
  constexpr int NS = D + 2;
#pragma unroll
  for (int s = 0; s < NS; ++s) uu[s] = 0.0;
  if (qv) {
#pragma unroll
    for (int s = 0; s < D * NS; ++s) qv[s] = 0.0;
  }
  for (int a = 0; a < nb; ++a) {
    const int node = nmap ? nmap[nodes[a]] : nodes[a];
    const double p = ph[a];
#pragma unroll
    for (int s = 0; s < NS; ++s) uu[s] += p * src[node * NS + s];
    if (qv) {
#pragma unroll
      for (int l = 0; l < D; ++l)
#pragma unroll
        for (int s = 0; s < NS; ++s) qv[l * NS + s] += p * qs[(l * L + node) * NS + s];
    }
  }
  (void)src_stride_l;
}

template <int D>
__global__ void __launch_bounds__(asm_threads<D>(), asm_min_ctas<D>())
    k_assemble(mhdg_disc g, mhdg_flow flow, mhdg_stage stage, const double* __restrict__ u,
               const double* __restrict__ q, const double* __restrict__ uhat, double* __restrict__ R_grad,
               double* __restrict__ R_state, double* __restrict__ R_tl, int want_jac, mhdg_blocks bk,
               mhdg_frozen fo, mhdg_frozen fi, int use_frozen, int* status, int nqc, int nfg) {
  extern __shared__ double sm[];
  constexpr int NS = D + 2, NF = D + 1, E = D + 1;
  const Sz sz = make_sz<D>(g);
  const AsmSmem<D> o = asm_smem<D>(sz, nqc, nfg, want_jac != 0);
  const FlowC fl = make_flow<D>(flow);
  const int mac = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const int n = sz.n, L = sz.L, Lf = sz.Lf, nq = sz.nq, nloc = sz.nloc, nqf = sz.nqf, nlocf = sz.nlocf;
  const double det = g.det[mac];
  const double* ij = g.inv_jac + (size_t)mac * D * D;
  const bool temporal = stage.dt_coeff != 0.0 || stage.hist != nullptr;
  // want_jac == 2: couplings only (face blocks and dG/dq stashes, what the trace apply streams);
  // no state_state, no frozen coefficients, no residual vectors (the coupling-recompute
  // representation re-forms them per apply from (u, q, uhat), condense.py RecomputeBlocks)
  const bool want_ss = want_jac == 1, want_res = want_jac != 2;
  const double inv_sdt = isinf(stage.supg_dt) ? 0.0 : 1.0 / stage.supg_dt;

  double *us = sm + o.us, *qs = sm + o.qs, *uh = sm + o.uh, *td = sm + o.td, *tf = sm + o.tf;
  double *gph = sm + o.gph, *upt = sm + o.upt, *qpt = sm + o.qpt, *wq = sm + o.wq, *tq = sm + o.tq;
  Prim<D>* prv = (Prim<D>*)(sm + o.prv);
  double *As = sm + o.As, *Adu = sm + o.Adu, *FG = sm + o.FG, *Pp = sm + o.Pp, *sw = sm + o.sw;
  double *W1 = sm + o.W1, *cvol = sm + o.cvol, *gus = sm + o.gus, *tdps = sm + o.tdps, *rs = sm + o.rs, *wts = sm + o.wts;

  // face lattice node -> local node of sub-face T (or -1)
  __shared__ short floc[ASM_MAXFLOC];
  for (int i = tid; i < sz.n_tri * Lf; i += nt) {
    const int T = i / Lf, gg = i - T * Lf;
    short a = -1;
    for (int k = 0; k < nlocf; ++k)
      if (g.tri_conn[T * nlocf + k] == gg) a = (short)k;
    floc[i] = a;
  }
  // ---- load state ---------------------------------------------------------
  for (int i = tid; i < n; i += nt) us[i] = u[(size_t)mac * n + i];
  for (int i = tid; i < D * n; i += nt) qs[i] = q[(size_t)mac * D * n + i];
  for (int i = tid; i < sz.ltr; i += nt) uh[i] = uhat[g.gather[(size_t)mac * sz.ltr + i]];
  __syncthreads();
  if (temporal)
    for (int i = tid; i < n; i += nt)
      td[i] = stage.hist ? stage.dt_coeff * us[i] + stage.hist[(size_t)mac * n + i] : stage.dt_coeff * us[i];

  // ---- gradient equation residual (linear, assembly.py:360-365) -----------
  if (want_res) {
  for (int idx = tid; idx < sz.ltr; idx += nt) {
    const int s = idx % NS, gg = (idx / NS) % Lf, f = idx / sz.bs;
    double a = 0.0;
    for (int h = 0; h < Lf; ++h) a += g.face_mass[gg * Lf + h] * uh[(f * Lf + h) * NS + s];
    tf[idx] = a * (g.face_fac * g.areas[mac * NF + f]);
  }
  __syncthreads();
  if ((1 + D) * L * L + 2 * D * n <= o.total - o.gph) {
    // the mass and weak-derivative tables staged through the (still unused) work area: one
    // round of coalesced loads instead of 4 L dependent L2 reads per entry; the derivative
    // sums T[r][I][s] are formed once, not once per gradient direction l
    double *tm = sm + o.gph, *tw = tm + L * L, *sT = tw + D * L * L, *sA = sT + D * n;
    for (int i = tid; i < L * L; i += nt) tm[i] = g.mass[i];
    for (int i = tid; i < D * L * L; i += nt) tw[i] = g.weak_deriv[i];
    __syncthreads();
    for (int idx = tid; idx < 2 * D * n; idx += nt) {
      const bool isT = idx < D * n;
      const int e = isT ? idx : idx - D * n, s = e % NS, I = (e / NS) % L, rl = e / n;
      const double* row = isT ? tw + ((size_t)rl * L + I) * L : tm + I * L;
      const double* src = isT ? us + s : qs + rl * n + s;
      double acc = 0.0;
      for (int J = 0; J < L; ++J) acc += row[J] * src[J * NS];
      (isT ? sT : sA)[e] = acc;
    }
    __syncthreads();
    for (int idx = tid; idx < D * n; idx += nt) {
      const int s = idx % NS, I = (idx / NS) % L, l = idx / n;
      double b = 0.0;
#pragma unroll
      for (int r = 0; r < D; ++r) b += ij[r * D + l] * sT[(r * L + I) * NS + s];
      double c = 0.0;
      for (int e = g.vf_ptr[I]; e < g.vf_ptr[I + 1]; ++e) {
        const int ent = g.vf_ent[e], f = ent / Lf;
        c -= g.normals[(mac * NF + f) * D + l] * tf[ent * NS + s];
      }
      R_grad[(size_t)mac * D * n + idx] = (det * sA[idx] + det * b) + c;
    }
  } else {
  for (int idx = tid; idx < D * n; idx += nt) {
    const int s = idx % NS, I = (idx / NS) % L, l = idx / n;
    double a = 0.0;
    for (int J = 0; J < L; ++J) a += g.mass[I * L + J] * qs[(l * L + J) * NS + s];
    double b = 0.0;
#pragma unroll
    for (int r = 0; r < D; ++r) {
      const double* Dr = g.weak_deriv + ((size_t)r * L + I) * L;
      double t = 0.0;
      for (int J = 0; J < L; ++J) t += Dr[J] * us[J * NS + s];
      b += ij[r * D + l] * t;
    }
    double c = 0.0;
    for (int e = g.vf_ptr[I]; e < g.vf_ptr[I + 1]; ++e) {
      const int ent = g.vf_ent[e], f = ent / Lf;
      c -= g.normals[(mac * NF + f) * D + l] * tf[ent * NS + s];
    }
    R_grad[(size_t)mac * D * n + idx] = (det * a + det * b) + c;
  }

  }
  }  // want_res
  // ---- Jacobian initialisation (mass / PTC term, assembly.py:397-405) -----
  if (want_jac == 2 && tid < NF) bk.trace_face_scale[mac * NF + tid] = g.bc_kind[mac * NF + tid] > 0 ? 0.0 : 1.0;
  if (want_ss) {
    const double coeff = stage.dt_coeff + (isinf(stage.pseudo_dt) ? 0.0 : 1.0 / stage.pseudo_dt);
    double* SSm = bk.state_state + (size_t)mac * n * n;
    const int lane = tid & 31, nwarp = nt >> 5;
    for (int r = tid >> 5; r < n; r += nwarp) {  // a warp per row: no runtime divisions per entry
      const int I = r / NS, s = r % NS;
      double* row = SSm + (size_t)r * n;
      if ((n & 1) == 0) {  // 16-byte stores
        for (int c = 2 * lane; c < n; c += 64) {
          double v[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int J = (c + e) / NS, t = c + e - J * NS;
            v[e] = (s == t && coeff != 0.0) ? coeff * det * g.mass[I * L + J] : 0.0;
          }
          *reinterpret_cast<double2*>(row + c) = make_double2(v[0], v[1]);
        }
      } else {
        for (int c = lane; c < n; c += 32) {
          const int J = c / NS, t = c - J * NS;
          row[c] = (s == t && coeff != 0.0) ? coeff * det * g.mass[I * L + J] : 0.0;
        }
      }
    }
    if (tid < NF) bk.trace_face_scale[mac * NF + tid] = g.bc_kind[mac * NF + tid] > 0 ? 0.0 : 1.0;
  }
  __syncthreads();

  // ---- volume terms, one sub-element at a time (assembly.py:409-475) ------
  // quadrature points in chunks of nqc (= nq unless the per-point work arrays would
  // exceed shared memory, e.g. 3D p = 3); sums over points accumulate chunk by chunk
  const int nA = D * NS * NS;
  for (int K = 0; K < sz.n_sub; ++K) {
    const int* conn = g.sub_conn + K * nloc;
    for (int q0 = 0; q0 < nq; q0 += nqc) {
    const int nc = min(nqc, nq - q0);
    {
      if (want_ss && q0 == 0) {
        // the sub-element's block of state_state copied asynchronously into the shared-memory
        // tile the GEMMs accumulate into (no read-modify-write latency at the end)
        const int nr = nloc * NS, cld = csm_ld(nr);
        double* Csm = sm + o.csm;
        const double* SSm = bk.state_state + (size_t)mac * n * n;
        for (int idx = tid; idx < nr * nr; idx += nt) {
          const int cb = idx % nr, rb = idx / nr, t = cb % NS, b = cb / NS, s = rb % NS, a = rb / NS;
          cp_async8(Csm + rb * cld + cb, SSm + (size_t)(conn[a] * NS + s) * n + conn[b] * NS + t, 8);
        }
      }
    }
    for (int idx = tid; idx < nc * nloc * D; idx += nt) {
      const int k = idx % D, a = (idx / D) % nloc, qq = idx / (D * nloc);
      const double* gr = g.grad_ref + (((size_t)K * nq + q0 + qq) * nloc + a) * D;
      double v = 0.0;
#pragma unroll
      for (int r = 0; r < D; ++r) v += gr[r] * ij[r * D + k];
      gph[idx] = v;  // gphys[q][a][k]
    }
    // state and gradient at the points, one component per thread (nodes in order, as interp_point)
    for (int idx = tid; idx < nc * (1 + D) * NS; idx += nt) {
      const int c = idx % ((1 + D) * NS), qq = idx / ((1 + D) * NS);
      const double* ph = g.phi_vol + (q0 + qq) * nloc;
      const double* src = c < NS ? us + c : qs + (size_t)((c - NS) / NS) * n + (c - NS) % NS;
      double acc = 0.0;
      for (int a = 0; a < nloc; ++a) acc += ph[a] * src[conn[a] * NS];
      if (c < NS) upt[qq * NS + c] = acc;
      else qpt[qq * D * NS + (c - NS)] = acc;
    }
    __syncthreads();
    for (int qq = tid; qq < nc; qq += nt) {
      double uu[NS];
#pragma unroll
      for (int s = 0; s < NS; ++s) uu[s] = upt[qq * NS + s];
      const int bad = admissible_code<D>(uu, fl.gamma);
      if (bad) set_status(status, MHDG_ERR_ADMISSIBILITY, mac, bad - 1, uu[0]);
      const Prim<D> p = prim<D>(uu, fl);
      prv[qq] = p;
      wq[qq] = g.w_ref[K * nq + q0 + qq] * det;
      const size_t fidx = ((size_t)mac * sz.n_sub + K) * nq + q0 + qq;
      tq[qq] = use_frozen ? fi.supg_tau[fidx] : supg_tau<D>(p, fl, g.h_sub[mac * sz.n_sub + K], inv_sdt);
      if (want_ss) fo.supg_tau[fidx] = tq[qq];
      wts[qq] = sqrt(wq[qq] * tq[qq]);  // W1 rows carry sqrt(w tau): GEMM 2 is then W1s^T W1s
    }
    // physical gradient of u (and the temporal term) at the points, for the strong residual
    for (int idx = tid; idx < nc * (D + 1) * NS; idx += nt) {
      const int c = idx % ((D + 1) * NS), qq = idx / ((D + 1) * NS), t = c % NS, k = c / NS;
      double acc = 0.0;
      if (k < D) {
        for (int a = 0; a < nloc; ++a) acc += gph[(qq * nloc + a) * D + k] * us[conn[a] * NS + t];
        gus[(qq * D + k) * NS + t] = acc;
      } else {
        if (temporal)
          for (int a = 0; a < nloc; ++a) acc += g.phi_vol[(q0 + qq) * nloc + a] * td[conn[a] * NS + t];
        tdps[qq * NS + t] = acc;
      }
    }
    __syncthreads();
    // pointwise Jacobians and fluxes.  An item is (case, point) with the case -- a (k, l) block
    // of the stash or a (k, s) row of the Euler / viscous state Jacobians -- uniform over
    // (most of) a warp and the lanes over points, so the entry indices are compile-time inside
    // a case (the pointwise functions fold to straight-line code).
    {
      const int ncase = (want_jac ? D * D : 0) + (want_res ? D * NS : 0);
      constexpr int nW = D * D * NS * NS;
      for (int idx = tid; idx < ncase * nc; idx += nt) {
        const int cs = idx / nc, qq = idx - cs * nc;
        const Prim<D> pr = prv[qq];
        const size_t pidx = ((size_t)mac * sz.n_sub + K) * nq + q0 + qq;
        const int c0 = want_jac ? cs : cs + D * D;
        if (c0 < D * D) {
          double* Wd = bk.wdgdq_vol + pidx * nW + c0 * NS * NS;
          const double w = wq[qq];
          static_switch<D * D>(c0, [&](auto kl) {
            constexpr int k = decltype(kl)::value / D, l = decltype(kl)::value % D;
#pragma unroll
            for (int s = 0; s < NS; ++s)
#pragma unroll
              for (int t = 0; t < NS; ++t) Wd[s * NS + t] = w * visc_dgdq<D>(pr, fl, k, l, s, t);
          });
        } else {
          const int c1 = c0 - D * D;  // k * NS + s
          const double* qp = qpt + qq * D * NS;
          const double* up = upt + qq * NS;
          double* Ar = As + qq * nA + c1 * NS;
          double* Adr = Adu + qq * nA + c1 * NS;
          const size_t fidx = pidx * nA + c1 * NS;
          static_switch<D * NS>(c1, [&](auto ks) {
            constexpr int k = decltype(ks)::value / NS, sr = decltype(ks)::value % NS;
#pragma unroll
            for (int t = 0; t < NS; ++t) {
              const double a = euler_jac<D>(pr, fl, k, sr, t);
              Ar[t] = use_frozen ? fi.supg_jac[fidx + t] : a;
              if (want_ss) {
                Adr[t] = a + visc_dgdu<D>(pr, fl, qp, k, sr, t);
                fo.supg_jac[fidx + t] = a;
              }
            }
            FG[(qq * NS + sr) * D + k] = euler_flux<D>(pr, up, sr, k) + visc_flux<D>(pr, fl, qp, sr, k);
          });
        }
      }
    }
    __syncthreads();
    if (!want_res) continue;  // couplings only: the stash rows of this chunk are written
    // strong SUPG residual r[q][u] = sum_{k,t} A[k][u][t] gu[k][t] + td, then the per-point
    // residual vector Pp[q][k][s]
    for (int idx = tid; idx < nc * NS; idx += nt) {
      const int uu = idx % NS, qq = idx / NS;
      const double* A = As + qq * nA;
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k)
#pragma unroll
        for (int t = 0; t < NS; ++t) acc += A[(k * NS + uu) * NS + t] * gus[(qq * D + k) * NS + t];
      rs[idx] = acc + tdps[idx];
    }
    __syncthreads();
    for (int idx = tid; idx < nc * D * NS; idx += nt) {
      const int s = idx % NS, k = (idx / NS) % D, qq = idx / (D * NS);
      const double* A = As + qq * nA;
      const double w = wq[qq], wt = w * tq[qq];
      double acc = 0.0;
#pragma unroll
      for (int uu = 0; uu < NS; ++uu) acc += A[(k * NS + uu) * NS + s] * rs[qq * NS + uu];
      Pp[(qq * D + k) * NS + s] = -w * FG[(qq * NS + s) * D + k] + wt * acc;
    }
    if (g.source)
      for (int idx = tid; idx < nc * NS; idx += nt) {
        const int qq = idx / NS;
        sw[idx] = -wq[qq] * g.source[(((size_t)mac * sz.n_sub + K) * nq + q0) * NS + idx];
      }
    __syncthreads();
    for (int idx = tid; idx < nloc * NS; idx += nt) {
      const int s = idx % NS, a = idx / NS;
      double acc = 0.0;
      for (int qq = 0; qq < nc; ++qq) {
#pragma unroll
        for (int k = 0; k < D; ++k) acc += gph[(qq * nloc + a) * D + k] * Pp[(qq * D + k) * NS + s];
        if (g.source) acc += g.phi_vol[(q0 + qq) * nloc + a] * sw[qq * NS + s];
      }
      cvol[(K * nloc + a) * NS + s] = q0 == 0 ? acc : cvol[(K * nloc + a) * NS + s] + acc;
    }
    if (want_ss) {
      const int nw = nloc * NS * NS;
      double* SSm = bk.state_state + (size_t)mac * n * n;
      const int nr = nloc * NS;
      {
        const int wld = w1t_ld(nr), cld = csm_ld(nr);
        double* Csm = sm + o.csm;
        const int warp = tid >> 5, lane = tid & 31, g8 = lane >> 2, t4 = lane & 3, nwarp = nt >> 5;
        for (int row = warp; row < nc * NS; row += nwarp) {  // a warp per row (q, u) of W1T: no runtime divisions
          const int qq = row / NS, uu = row - qq * NS;
          const double* Aq = As + (qq * D * NS + uu) * NS;
          const double* gq_ = gph + qq * nloc * D;
          const double swt = wts[qq];
          for (int col = lane; col < nr; col += 32) {
            const int a = col / NS, s = col - a * NS;
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) acc += Aq[k * NS * NS + s] * gq_[a * D + k];
            W1[row * wld + col] = acc * swt;  // sqrt(w tau) W1T[(q, u)][(a, s)]
          }
        }
        cp_async_wait_all();  // Csm holds this sub-element's state_state entries (copied since the chunk began)
        __syncthreads();
        // contrib[(a,s),(b,t)] = sum_{(q,u)} (w tau W1T[(q,u)][(a,s)]) W1T[(q,u)][(b,t)]        (GEMM 2)
        //                      + sum_q Y[q][(a,s,t)] phi[q][b],                                 (GEMM 1)
        //   Y = -w sum_k Adu[q,k,s,t] gphys[q,a,k] + dt_coeff w tau W1T[(q,t)][(a,s)]   (assembly.py:465-470)
        // GEMM 2 is symmetric: one 8 x 8 tile (mt <= nt) per unit, mirrored into Csm
        const int mtl = (nr + 7) / 8;
        const int nun = mtl * (mtl + 1) / 2, K2 = nc * NS, ks2 = (K2 + 3) / 4;
        for (int un = warp; un < nun; un += nwarp) {
          int mt = 0, rem = un;
          while (rem >= mtl - mt) {
            rem -= mtl - mt;
            ++mt;
          }
          const int ntile = mt + rem;
          const int m = mt * 8 + g8, nn = ntile * 8 + g8;
          const bool mok = m < nr, nok = nn < nr;
          const int mc = mok ? m : 0, ncol = nok ? nn : 0;
          double c0 = 0.0, c1 = 0.0;
          for (int ks = 0; ks < ks2; ++ks) {
            const int kk = 4 * ks + t4;
            const bool kok = kk < K2;
            const int kc = kok ? kk : 0;
            const double* wr = W1 + kc * wld;
            const double af = (mok && kok) ? wr[mc] : 0.0;
            const double bf = (kok && nok) ? wr[ncol] : 0.0;
            dmma_8x8x4(c0, c1, af, bf);
          }
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = ntile * 8 + 2 * t4 + e;
            const double cv = e ? c1 : c0;
            if (mok && col < nr) {
              Csm[m * cld + col] += cv;
              if (ntile != mt) Csm[col * cld + m] += cv;
            }
          }
        }
        __syncthreads();
        const int mt1 = (nw + 7) / 8, ks1 = (nc + 3) / 4;
        constexpr int NB1 = 3;  // b-tiles: nloc <= 24
        const int nb1 = (nloc + 7) / 8;
        for (int un = warp; un < mt1; un += nwarp) {
          const int m = un * 8 + g8;
          const bool mok = m < nw;
          const int a = mok ? m / (NS * NS) : 0, s = (m / NS) % NS, t = m % NS;
          double c[NB1][2];
#pragma unroll
          for (int h = 0; h < NB1; ++h) c[h][0] = c[h][1] = 0.0;
          for (int ks = 0; ks < ks1; ++ks) {
            const int qq = 4 * ks + t4;
            const bool kok = qq < nc;
            double af = 0.0;
            if (mok && kok) {
              double y = 0.0;
#pragma unroll
              for (int k = 0; k < D; ++k) y += Adu[((qq * D + k) * NS + s) * NS + t] * gph[(qq * nloc + a) * D + k];
              const double w = wq[qq];
              y = -w * y;
              if (stage.dt_coeff != 0.0) y += stage.dt_coeff * wts[qq] * W1[(qq * NS + t) * wld + a * NS + s];
              af = y;
            }
#pragma unroll
            for (int h = 0; h < NB1; ++h)
              if (h < nb1) {
                const int bb = h * 8 + g8;
                const double bf = (kok && bb < nloc) ? __ldg(g.phi_vol + (q0 + qq) * nloc + bb) : 0.0;
                dmma_8x8x4(c[h][0], c[h][1], af, bf);
              }
          }
#pragma unroll
          for (int h = 0; h < NB1; ++h)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int bb = h * 8 + 2 * t4 + e;
              if (mok && h < nb1 && bb < nloc) Csm[(a * NS + s) * cld + bb * NS + t] += c[h][e];
            }
        }
        if (q0 + nqc >= nq) {  // the sub-element's block is complete (summed over the point chunks in Csm)
          __syncthreads();
          for (int idx = tid; idx < nr * nr; idx += nt) {
            const int cb = idx % nr, rb = idx / nr, t = cb % NS, b = cb / NS, s = rb % NS, a = rb / NS;
            SSm[(size_t)(conn[a] * NS + s) * n + conn[b] * NS + t] = Csm[rb * cld + cb];
          }
        }
      }
    }
    __syncthreads();
    }  // point chunks
  }

  // ---- face terms (assembly.py:477-612) -----------------------------------
  // All sub-faces of a group of nfg faces go through the per-point phases together (point
  // p = ((f - f0) n_tri + T) nqf + qq); the face blocks are then formed entry by entry, each
  // entry summing its sub-faces in order (T ascending, as the reference accumulates) and
  // written once -- no zero fill and no read-modify-write of the three face blocks.
  double *fuh = sm + o.fuh, *fu = sm + o.fu, *fq = sm + o.fq, *fuv = sm + o.fuv, *fw = sm + o.fw;
  Prim<D>* fpr = (Prim<D>*)(sm + o.fpr);
  Prim<D>* fpv = (Prim<D>*)(sm + o.fpv);
  double *fS = sm + o.fS, *fK1 = sm + o.fK1, *ffn = sm + o.ffn, *fbh = sm + o.fbh, *cf = sm + o.cf,
         *ctr = sm + o.ctr;
  const int nqt = sz.n_tri * nqf;
  constexpr int NC = (2 + D) * NS;  // interpolated components per face point: uhat, u, q
  for (int f0 = 0; f0 < NF; f0 += nfg) {
    const int nfa = min(nfg, NF - f0), npt = nfa * nqt;
    // interpolation to the face points, one component per thread
    for (int idx = tid; idx < npt * NC; idx += nt) {
      const int comp = idx % NC, pp = idx / NC, qq = pp % nqf, T = (pp / nqf) % sz.n_tri, f = f0 + pp / nqt;
      const double* ph = g.phi_face + qq * nlocf;
      const int* tc = g.tri_conn + T * nlocf;
      double acc = 0.0;
      if (comp < NS) {
        const double* src = uh + f * Lf * NS + comp;
        for (int a = 0; a < nlocf; ++a) acc += ph[a] * src[tc[a] * NS];
        fuh[pp * NS + comp] = acc;
      } else {
        const int* fvn = g.face_vol_nodes + f * Lf;
        const int c2 = comp - NS;
        const double* src = c2 < NS ? us + c2 : qs + (size_t)((c2 - NS) / NS) * n + (c2 - NS) % NS;
        for (int a = 0; a < nlocf; ++a) acc += ph[a] * src[fvn[tc[a]] * NS];
        if (c2 < NS) fu[pp * NS + c2] = acc;
        else fq[pp * D * NS + (c2 - NS)] = acc;
      }
    }
    __syncthreads();
    for (int pp = tid; pp < npt; pp += nt) {
      const int qq = pp % nqf, T = (pp / nqf) % sz.n_tri, f = f0 + pp / nqt;
      const size_t pg = ((size_t)mac * NF + f) * nqt + T * nqf + qq;  // face point index (frozen / stash)
      double a_uh[NS];
#pragma unroll
      for (int s = 0; s < NS; ++s) a_uh[s] = fuh[pp * NS + s];
      const int bad = admissible_code<D>(a_uh, fl.gamma);
      if (bad) set_status(status, MHDG_ERR_ADMISSIBILITY, mac, bad - 1, a_uh[0]);
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        fuv[pp * NS + s] = use_frozen ? fi.face_visc_state[pg * NS + s] : a_uh[s];
        if (want_ss) fo.face_visc_state[pg * NS + s] = a_uh[s];
      }
      fpr[pp] = prim<D>(a_uh, fl);
      fpv[pp] = use_frozen ? prim<D>(fuv + pp * NS, fl) : fpr[pp];
      fw[pp] = g.w_face_ref[T * nqf + qq] * (g.face_fac * g.areas[mac * NF + f]);
    }
    __syncthreads();
    // stabilisation / flux Jacobian rows and stash rows as (case, point) items: the case (a row
    // s of S and K1, or a row (l, s) of the stash) is uniform over (most of) a warp, the lanes
    // run over points, and the entry indices are compile-time inside a case
    {
      const int ncase = NS + (want_jac ? D * NS : 0);
      for (int idx = tid; idx < ncase * npt; idx += nt) {
        const int cs = idx / npt, pp = idx - cs * npt, f = f0 + pp / nqt;
        const size_t pg = ((size_t)mac * NF + f) * nqt + pp % nqt;
        double nv[D];
#pragma unroll
        for (int k = 0; k < D; ++k) nv[k] = g.normals[(mac * NF + f) * D + k];
        if (cs < NS) {
          const Prim<D> pr = fpr[pp];
          static_switch<NS>(cs, [&](auto sc) {
            constexpr int sr = decltype(sc)::value;
#pragma unroll
            for (int t = 0; t < NS; ++t) {
              const double S = use_frozen ? fi.face_stab[pg * NS * NS + sr * NS + t]
                                          : ((sr == t) ? stab_diag<D>(pr, fl, nv, sr) : 0.0);
              fS[(pp * NS + sr) * NS + t] = S;
              if (want_jac) {
                if (want_ss) fo.face_stab[pg * NS * NS + sr * NS + t] = S;
                double an = 0.0;
#pragma unroll
                for (int k = 0; k < D; ++k) an += euler_jac<D>(pr, fl, k, sr, t) * nv[k];
                fK1[(pp * NS + sr) * NS + t] = an - S;  // d(flux.n)/d uhat, viscous uhat-dependence dropped
              }
            }
          });
        } else {
          const Prim<D> pr = fpv[pp];
          const double w = fw[pp];
          double* Wf = bk.wdgdq_face + pg * (D * NS * NS) + (cs - NS) * NS;
          static_switch<D * NS>(cs - NS, [&](auto lsc) {
            constexpr int l = decltype(lsc)::value / NS, sr = decltype(lsc)::value % NS;
#pragma unroll
            for (int t = 0; t < NS; ++t) {
              double acc = 0.0;
#pragma unroll
              for (int k = 0; k < D; ++k) acc += visc_dgdq<D>(pr, fl, k, l, sr, t) * nv[k];
              Wf[t] = w * acc;
            }
          });
        }
      }
    }
    __syncthreads();
    for (int idx0 = want_res ? tid : npt * NS; idx0 < npt * NS; idx0 += nt) {
      const int s = idx0 / npt, pp = idx0 - s * npt, f = f0 + pp / nqt, idx = pp * NS + s;  // lanes over points
      const int kind = g.bc_kind[mac * NF + f];
      const double* nv = g.normals + (mac * NF + f) * D;
      double fn = 0.0;
      {
        const Prim<D> pr = fpr[pp], pv = fpv[pp];
        static_switch<NS>(s, [&](auto sc) {
          constexpr int sr = decltype(sc)::value;
#pragma unroll
          for (int k = 0; k < D; ++k)
            fn += (euler_flux<D>(pr, fuh + pp * NS, sr, k) + visc_flux<D>(pv, fl, fq + pp * D * NS, sr, k)) * nv[k];
        });
      }
      double sa = 0.0;
#pragma unroll
      for (int t = 0; t < NS; ++t) sa += fS[(pp * NS + s) * NS + t] * (fu[pp * NS + t] - fuh[pp * NS + t]);
      ffn[idx] = fn + sa;
      if (kind == 1) {  // Dirichlet: uhat - u_D
        const size_t pg = ((size_t)mac * NF + f) * nqt + pp % nqt;
        fbh[idx] = fuh[idx] - g.u_dir[pg * NS + s];
      } else if (kind == 2) {  // isothermal wall (moving with u_w)
        const double* u_w = g.wall_u + (mac * NF + f) * D;
        double uw2 = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) uw2 += u_w[i] * u_w[i];
        const double e_tot = g.wall_e[mac * NF + f] + 0.5 * uw2;
        const double rh = fuh[pp * NS];
        double v;
        if (s == 0) v = rh - fu[pp * NS];
        else if (s <= D) v = fuh[idx] - rh * u_w[s - 1];
        else v = fuh[pp * NS + E] - rh * e_tot;
        fbh[idx] = v;
      } else if (kind == 3) {  // adiabatic no-slip wall: rho_hat - rho, m_hat, E_hat - E
        fbh[idx] = (s == 0 || s == E) ? fuh[idx] - fu[idx] : fuh[idx];
      }
    }
    __syncthreads();
    // projections onto the face sub-elements' nodes
    for (int idx = want_res ? tid : nfa * sz.n_tri * nlocf * NS; idx < nfa * sz.n_tri * nlocf * NS; idx += nt) {
      const int s = idx % NS, a = (idx / NS) % nlocf, T = (idx / (NS * nlocf)) % sz.n_tri,
                fl_ = idx / (NS * nlocf * sz.n_tri), f = f0 + fl_;
      const int kind = g.bc_kind[mac * NF + f];
      const int p0 = (fl_ * sz.n_tri + T) * nqf;
      double acc = 0.0, accb = 0.0;
      for (int qq = 0; qq < nqf; ++qq) {
        const double wp = fw[p0 + qq] * g.phi_face[qq * nlocf + a];
        acc += wp * ffn[(p0 + qq) * NS + s];
        if (kind > 0) accb += wp * fbh[(p0 + qq) * NS + s];
      }
      const int slot = ((f * sz.n_tri + T) * nlocf + a) * NS + s;
      cf[slot] = acc;
      ctr[slot] = kind > 0 ? accb : -acc;
    }
    if (want_jac) {
      double* SSm = bk.state_state + (size_t)mac * n * n;
      for (int fl_ = 0; fl_ < nfa; ++fl_) {  // faces in turn: they share state_state entries on their common edges
        const int f = f0 + fl_;
        const int kind = g.bc_kind[mac * NF + f];
        const int* fvn = g.face_vol_nodes + f * Lf;
        const double* u_w = g.wall_u + (mac * NF + f) * D;
        double uw2 = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) uw2 += u_w[i] * u_w[i];
        const double e_tot = g.wall_e[mac * NF + f] + 0.5 * uw2;
        const size_t fboff = ((size_t)mac * NF + f) * sz.bs * sz.bs;
        for (int idx = tid; idx < sz.bs * sz.bs; idx += nt) {
          const int cl = idx % sz.bs, rl = idx / sz.bs, t = cl % NS, gc = cl / NS, s = rl % NS, gr = rl / NS;
          double ust = 0.0, uss = 0.0, pr = 0.0;
          bool any = false;
          for (int T = 0; T < sz.n_tri; ++T) any |= want_ss && floc[T * Lf + gr] >= 0 && floc[T * Lf + gc] >= 0;
          double* pss = SSm + (size_t)(fvn[gr] * NS + s) * n + fvn[gc] * NS + t;
          const double ss_old = any ? *pss : 0.0;  // issued before the sums: its latency runs under them
          for (int T = 0; T < sz.n_tri; ++T) {
            const int a = floc[T * Lf + gr], b = floc[T * Lf + gc];
            if (a < 0 || b < 0) continue;
            const int p0 = (fl_ * sz.n_tri + T) * nqf;
            double ust_T = 0.0, uss_T = 0.0, pr_T = 0.0;
            for (int qq = 0; qq < nqf; ++qq) {
              const double pq = fw[p0 + qq] * g.phi_face[qq * nlocf + a] * g.phi_face[qq * nlocf + b];
              ust_T += pq * fK1[((p0 + qq) * NS + s) * NS + t];
              uss_T += pq * fS[((p0 + qq) * NS + s) * NS + t];
              pr_T += pq;
            }
            ust += ust_T;
            uss += uss_T;
            pr += pr_T;
          }
          double tst, ttt;
          if (kind == 0) {
            tst = -uss;
            ttt = -ust;
          } else {
            // boundary rows: Khh (identity; wall: [1+i,0] = -u_w, [E,0] = -(e_w+|u_w|^2/2)), Kuu
            double khh = (s == t) ? 1.0 : 0.0, kuu = 0.0;
            if (kind == 2) {
              if (t == 0 && s >= 1 && s <= D) khh = -u_w[s - 1];
              if (t == 0 && s == E) khh = -e_tot;
              if (s == 0 && t == 0) kuu = -1.0;
            } else if (kind == 3) {
              if (s == t && (s == 0 || s == E)) kuu = -1.0;
            }
            tst = pr * kuu;
            ttt = pr * khh;
          }
          bk.face_state_trace[fboff + idx] = ust;
          bk.face_trace_state[fboff + idx] = tst;
          bk.face_trace_trace[fboff + idx] = ttt;
          if (any) *pss = ss_old + uss;
        }
        __syncthreads();
      }
    }
    __syncthreads();
  }

  // ---- R_U and the local trace residual ------------------------------------
  if (!want_res) return;
  for (int idx = tid; idx < n; idx += nt) {
    const int I = idx / NS, s = idx % NS;
    double acc = 0.0;
    if (temporal) {
      double t = 0.0;
      for (int J = 0; J < L; ++J) t += g.mass[I * L + J] * td[J * NS + s];
      acc = det * t;
    }
    for (int e = g.vn_ptr[I]; e < g.vn_ptr[I + 1]; ++e) acc += cvol[g.vn_sub[e] * NS + s];
    for (int e = g.vf_ptr[I]; e < g.vf_ptr[I + 1]; ++e) {
      const int ent = g.vf_ent[e], f = ent / Lf, gg = ent % Lf;
      for (int e2 = g.fn_ptr[gg]; e2 < g.fn_ptr[gg + 1]; ++e2)
        acc += cf[(f * sz.n_tri * nlocf + g.fn_ent[e2]) * NS + s];
    }
    R_state[(size_t)mac * n + idx] = acc;
  }
  for (int idx = tid; idx < sz.ltr; idx += nt) {
    const int s = idx % NS, gg = (idx / NS) % Lf, f = idx / sz.bs;
    double acc = 0.0;
    for (int e2 = g.fn_ptr[gg]; e2 < g.fn_ptr[gg + 1]; ++e2) acc += ctr[(f * sz.n_tri * nlocf + g.fn_ent[e2]) * NS + s];
    R_tl[(size_t)mac * sz.ltr + idx] = acc;
  }
}

// ---- couplings only (want_jac == 2): the data the trace apply streams ------------------
// The coupling-recompute representation (B_min) re-forms, per apply and
// per window of macros, exactly the blocks the apply reads: the w dG/dq stashes (volume and
// face) and the three face blocks, from (u, uhat) alone -- none of them depends on q.  A
// dedicated kernel instead of k_assemble's Jacobian path: no residual phases, no
// state_state, small shared memory (several CTAs per SM).  Every value is formed by the
// same expressions in the same order as in k_assemble, so the blocks are bitwise equal.
//   volume: prims at all points, then (case, point) items write tiles of CPL_TP points to
//     shared memory that leave as one bulk copy (cp.async.bulk shared -> global) each;
//   faces, all of them per phase: prims, (case, point) items for S, d(flux.n)/d uhat (rows
//     padded for 16-byte loads, the diagonal of S in the pad) and the stash, then the face
//     blocks as (face, node pair, row s) items: the quadrature weight products are formed
//     once per NS entries and each thread writes NS consecutive doubles of the three blocks.
constexpr int CPL_THREADS = 256, CPL_TP = 16;
static int g_couplings_kernel = 1;  // A/B: 0 = k_assemble's couplings-only path
extern "C" void mhdg_set_couplings_kernel(int on) { g_couplings_kernel = on; }

template <int D>
struct CplSmem {
  int us, uh, phf, stage, prv, wq, tile, fpr, fw, wphi, fK1, total;
};

// rows of d(flux.n)/d uhat padded to K1P doubles with the diagonal of S in the last slot:
// a row is K1P / 2 16-byte loads
template <int D>
__host__ __device__ constexpr int cpl_k1p() { return (D + 2 + 2) & ~1; }

template <int D>
__host__ __device__ inline CplSmem<D> cpl_smem(const Sz& s) {
  constexpr int NS = D + 2, NF = D + 1;
  constexpr int PRIM = (int)((sizeof(Prim<D>) + 7) / 8);
  CplSmem<D> m;
  int o = 0;
  m.us = o, o += s.n;
  m.uh = o, o += s.ltr;
  m.phf = o, o += s.nqf * s.nlocf;
  m.stage = o, o += (CPL_THREADS / 32) * 32 * NS;  // per-warp transpose buffers of the face-block stores
  o = (o + 1) & ~1;
  const int work = o, npv = s.n_sub * s.nq, npf = NF * s.n_tri * s.nqf;
  m.tile = o, o += CPL_TP * D * D * NS * NS;  // first: 16-byte aligned for the bulk stores
  o = (o + 1) & ~1;
  m.prv = o, o += npv * PRIM;
  m.wq = o, o += npv;
  const int vol_end = o;
  o = work;  // the face arrays (all faces) share the volume arrays' memory
  m.fK1 = o, o += npf * NS * cpl_k1p<D>();
  m.fpr = o, o += npf * PRIM;
  m.fw = o, o += npf;
  m.wphi = o, o += npf * s.nlocf;
  m.total = o > vol_end ? o : vol_end;
  return m;
}

template <int D>
__global__ void __launch_bounds__(CPL_THREADS, 3) k_couplings(mhdg_disc g, mhdg_flow flow, const double* __restrict__ u,
                                                           const double* __restrict__ uhat, mhdg_blocks bk) {
  extern __shared__ __align__(16) double sm[];
  constexpr int NS = D + 2, NF = D + 1, E = D + 1, NW = D * D * NS * NS, NWF = D * NS * NS, K1P = cpl_k1p<D>();
  const Sz sz = make_sz<D>(g);
  const CplSmem<D> o = cpl_smem<D>(sz);
  const FlowC fl = make_flow<D>(flow);
  const int mac = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const int n = sz.n, Lf = sz.Lf, nq = sz.nq, nloc = sz.nloc, nqf = sz.nqf, nlocf = sz.nlocf, bs = sz.bs;
  const double det = g.det[mac];
  double *us = sm + o.us, *uh = sm + o.uh, *phf = sm + o.phf, *wq = sm + o.wq, *tile = sm + o.tile;
  Prim<D>* prv = (Prim<D>*)(sm + o.prv);
  __shared__ short floc[ASM_MAXFLOC];
  for (int i = tid; i < sz.n_tri * Lf; i += nt) {
    const int T = i / Lf, gg = i - T * Lf;
    short a = -1;
    for (int k = 0; k < nlocf; ++k)
      if (g.tri_conn[T * nlocf + k] == gg) a = (short)k;
    floc[i] = a;
  }
  for (int i = tid; i < n; i += nt) us[i] = u[(size_t)mac * n + i];
  for (int i = tid; i < sz.ltr; i += nt) uh[i] = uhat[g.gather[(size_t)mac * sz.ltr + i]];
  for (int i = tid; i < nqf * nlocf; i += nt) phf[i] = g.phi_face[i];
  if (tid < NF) bk.trace_face_scale[mac * NF + tid] = g.bc_kind[mac * NF + tid] > 0 ? 0.0 : 1.0;
  __syncthreads();
  // ---- volume stash (assembly.py:459-463) ------------------------------------------------
  const int npv = sz.n_sub * nq;
  for (int P = tid; P < npv; P += nt) {
    const int K = P / nq, qq = P - K * nq;
    const int* conn = g.sub_conn + K * nloc;
    const double* ph = g.phi_vol + qq * nloc;
    double uu[NS];
#pragma unroll
    for (int c = 0; c < NS; ++c) {
      double acc = 0.0;
      for (int a = 0; a < nloc; ++a) acc += ph[a] * us[conn[a] * NS + c];
      uu[c] = acc;
    }
    prv[P] = prim<D>(uu, fl);
    wq[P] = g.w_ref[P] * det;
  }
  __syncthreads();
  double* Wv = bk.wdgdq_vol + (size_t)mac * npv * NW;
  // a tile leaves as one bulk copy (TMA) issued by thread 0 when its global range is 16-byte
  // aligned (NW odd in 3D: every tile of CPL_TP points is, if the macro's base is)
#ifndef MHDG_CPL_BULK
#define MHDG_CPL_BULK 1
#endif
  const bool bulk = MHDG_CPL_BULK && (((size_t)mac * npv * NW) & 1) == 0 && ((CPL_TP * NW) & 1) == 0;
  for (int p0 = 0; p0 < npv; p0 += CPL_TP) {
    const int tp = min(CPL_TP, npv - p0);
    for (int idx = tid; idx < D * D * tp; idx += nt) {
      const int cs = idx / tp, pp = idx - cs * tp;
      const Prim<D> pr = prv[p0 + pp];
      const double w = wq[p0 + pp];
      double* Wd = tile + pp * NW + cs * NS * NS;
      static_switch<D * D>(cs, [&](auto kl) {
        constexpr int k = decltype(kl)::value / D, l = decltype(kl)::value % D;
#pragma unroll
        for (int s = 0; s < NS; ++s)
#pragma unroll
          for (int t = 0; t < NS; ++t) Wd[s * NS + t] = w * visc_dgdq<D>(pr, fl, k, l, s, t);
      });
    }
    double* dst = Wv + (size_t)p0 * NW;
    if (bulk && ((tp * NW) & 1) == 0) {
      fence_proxy_async();  // this thread's tile writes -> visible to the async proxy
      __syncthreads();
      if (tid == 0) {
        bulk_s2g(dst, tile, (uint32_t)(tp * NW * sizeof(double)));
        bulk_commit();
        bulk_wait_read0();  // the tile has been read: the next pass may overwrite it
      }
      __syncthreads();
    } else {
      __syncthreads();
      for (int i = tid; i < tp * NW; i += nt) dst[i] = tile[i];
      __syncthreads();
    }
  }
  // ---- faces (assembly.py:556-612), all of them per phase ---------------------------------
  Prim<D>* fpr = (Prim<D>*)(sm + o.fpr);
  double *fw = sm + o.fw, *wphi = sm + o.wphi, *fK1 = sm + o.fK1;
  const int nqt = sz.n_tri * nqf, npf = NF * nqt;
  for (int pp = tid; pp < npf; pp += nt) {
    const int f = pp / nqt, r = pp - f * nqt, T = r / nqf, qq = r - T * nqf;
    const double* ph = phf + qq * nlocf;
    const int* tc = g.tri_conn + T * nlocf;
    double a_uh[NS];
#pragma unroll
    for (int c = 0; c < NS; ++c) {
      const double* src = uh + f * Lf * NS + c;
      double acc = 0.0;
      for (int a = 0; a < nlocf; ++a) acc += ph[a] * src[tc[a] * NS];
      a_uh[c] = acc;
    }
    fpr[pp] = prim<D>(a_uh, fl);
    const double w = g.w_face_ref[T * nqf + qq] * (g.face_fac * g.areas[mac * NF + f]);
    fw[pp] = w;
    for (int a = 0; a < nlocf; ++a) wphi[pp * nlocf + a] = w * ph[a];
  }
  __syncthreads();
  for (int idx = tid; idx < (NS + D * NS) * npf; idx += nt) {
    const int cs = idx / npf, pp = idx - cs * npf, f = pp / nqt;
    const Prim<D> pr = fpr[pp];
    double nv[D];
#pragma unroll
    for (int k = 0; k < D; ++k) nv[k] = g.normals[(mac * NF + f) * D + k];
    if (cs < NS) {
      static_switch<NS>(cs, [&](auto sc) {
        constexpr int sr = decltype(sc)::value;
        double* row = fK1 + (pp * NS + sr) * K1P;
#pragma unroll
        for (int t = 0; t < NS; ++t) {
          const double S = (sr == t) ? stab_diag<D>(pr, fl, nv, sr) : 0.0;
          if (sr == t) row[NS] = S;
          double an = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) an += euler_jac<D>(pr, fl, k, sr, t) * nv[k];
          row[t] = an - S;
        }
      });
    } else {
      const double w = fw[pp];
      // the point's stash rows straight to global memory (NS consecutive doubles per item;
      // 5% of the macro's bytes)
      double* Wf = bk.wdgdq_face + ((size_t)mac * npf + pp) * NWF + (cs - NS) * NS;
      static_switch<D * NS>(cs - NS, [&](auto lsc) {
        constexpr int l = decltype(lsc)::value / NS, sr = decltype(lsc)::value % NS;
#pragma unroll
        for (int t = 0; t < NS; ++t) {
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) acc += visc_dgdq<D>(pr, fl, k, l, sr, t) * nv[k];
          Wf[t] = w * acc;
        }
      });
    }
  }
  __syncthreads();
  // face blocks: item r = ((gr NS + s) Lf + gc) of a face -> entries (gr NS + s, gc NS + t), t < NS,
  // i.e. doubles [NS r, NS r + NS) of each of the three blocks: a warp's 32 consecutive items
  // cover 32 NS contiguous doubles, handed through a per-warp shared-memory buffer so that every
  // store instruction writes 256 contiguous bytes (five times fewer L2 write transactions than
  // NS-double runs per lane)
  const int per_face = Lf * Lf * NS, warp = tid >> 5, lane = tid & 31;
  double* stg = sm + o.stage + warp * 32 * NS;
#pragma unroll 1
  for (int f = 0; f < NF; ++f) {
    const int kind = g.bc_kind[mac * NF + f];
    const double* u_w = g.wall_u + (mac * NF + f) * D;
    double uw2 = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) uw2 += u_w[i] * u_w[i];
    const double e_tot = g.wall_e[mac * NF + f] + 0.5 * uw2;
    const size_t fboff = ((size_t)mac * NF + f) * bs * bs;
    for (int r0 = warp * 32; r0 < per_face; r0 += nt) {
      const int r = r0 + lane;
      const bool active = r < per_face;
      const int cnt = min(32, per_face - r0) * NS;  // doubles this warp pass writes per block
      const int row = r / Lf, gc = r - row * Lf, gr = row / NS, s = row - gr * NS;
      double ust[NS], tst[NS], ttt[NS];
      if (active) {
        double uss = 0.0, pr = 0.0;
#pragma unroll
        for (int t = 0; t < NS; ++t) ust[t] = 0.0;
        for (int T = 0; T < sz.n_tri; ++T) {
          const int a = floc[T * Lf + gr], b = floc[T * Lf + gc];
          if (a < 0 || b < 0) continue;
          const int p0 = f * nqt + T * nqf;
          double ust_T[NS], uss_T = 0.0, pr_T = 0.0;
#pragma unroll
          for (int t = 0; t < NS; ++t) ust_T[t] = 0.0;
#pragma unroll 3
          for (int qq = 0; qq < nqf; ++qq) {
            const double pq = wphi[(p0 + qq) * nlocf + a] * phf[qq * nlocf + b];
            const double2* k2 = reinterpret_cast<const double2*>(fK1 + ((p0 + qq) * NS + s) * K1P);
            double k1[K1P];
#pragma unroll
            for (int h = 0; h < K1P / 2; ++h) {
              const double2 v = k2[h];
              k1[2 * h] = v.x;
              k1[2 * h + 1] = v.y;
            }
#pragma unroll
            for (int t = 0; t < NS; ++t) ust_T[t] += pq * k1[t];
            uss_T += pq * k1[NS];
            pr_T += pq;
          }
#pragma unroll
          for (int t = 0; t < NS; ++t) ust[t] += ust_T[t];
          uss += uss_T;
          pr += pr_T;
        }
#pragma unroll
        for (int t = 0; t < NS; ++t) {
          // S is diagonal here (no frozen coefficients): the off-diagonal sums of k_assemble are
          // sums of pq * 0.0, i.e. +0.0
          const double uss_t = (s == t) ? uss : 0.0;
          if (kind == 0) {
            tst[t] = -uss_t;
            ttt[t] = -ust[t];
          } else {
            double khh = (s == t) ? 1.0 : 0.0, kuu = 0.0;
            if (kind == 2) {
              if (t == 0 && s >= 1 && s <= D) khh = -u_w[s - 1];
              if (t == 0 && s == E) khh = -e_tot;
              if (s == 0 && t == 0) kuu = -1.0;
            } else if (kind == 3) {
              if (s == t && (s == 0 || s == E)) kuu = -1.0;
            }
            tst[t] = pr * kuu;
            ttt[t] = pr * khh;
          }
        }
      }
      const size_t off = fboff + (size_t)NS * r0;
#pragma unroll
      for (int blk = 0; blk < 3; ++blk) {
        double* dst = (blk == 0 ? bk.face_state_trace : blk == 1 ? bk.face_trace_state : bk.face_trace_trace) + off;
        __syncwarp();
        if (active) {
#pragma unroll
          for (int t = 0; t < NS; ++t) stg[lane * NS + t] = blk == 0 ? ust[t] : blk == 1 ? tst[t] : ttt[t];
        }
        __syncwarp();
        for (int k = lane; k < cnt; k += 32) dst[k] = stg[k];
      }
    }
  }
}

template <int D>
static int launch_couplings(const mhdg_disc& g, const mhdg_flow& fl, const double* u, const double* uhat,
                            const mhdg_blocks& b, cudaStream_t st) {
  const Sz sz = make_sz<D>(g);
  const size_t bytes = sizeof(double) * cpl_smem<D>(sz).total;
  if (bytes > 227 * 1024 || sz.n_tri * sz.Lf > ASM_MAXFLOC) return -1;
  static size_t set_bytes = 0;  // once per size: launches inside a CUDA-graph capture stay pure launches
  if (bytes > 48 * 1024 && bytes != set_bytes) {
    cudaFuncSetAttribute(k_couplings<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    set_bytes = bytes;
  }
  k_couplings<D><<<g.n_mac, CPL_THREADS, bytes, st>>>(g, fl, u, uhat, b);
  return launch_ok();
}

int face_reduce(const mhdg_disc&, const double*, const double*, double, double*, cudaStream_t);

template <int D>
int assemble(const mhdg_disc& g, const mhdg_flow& fl, const mhdg_stage& sg, const double* u, const double* q,
             const double* uhat, double* Rg, double* Ru, double* Rtl, double* Rt, int want_jac, const mhdg_blocks* b,
             const mhdg_frozen* fo, const mhdg_frozen* fi, int* status, cudaStream_t st) {
  const Sz sz = make_sz<D>(g);
  if (want_jac == 2 && b && !fi && g_couplings_kernel) {  // couplings only: the dedicated kernel when it fits
    const int rc2 = launch_couplings<D>(g, fl, u, uhat, *b, st);
    if (rc2 >= 0) return rc2;
  }
  // budget per CTA: 227 KB, or the SM's 228 KB (1 KB reserved per CTA) over asm_ctas CTAs
  // 3D residual-only launches: 320 threads (measured at C3: 384 x 2: 13.6 ms, 320 x 2: 11.6, 256 x 2: 12.6, 256 x 3: 14.2)
  const int ctas = (D == 3 && !want_jac) ? MHDG_ASM_RES_CTAS_3D : asm_ctas<D>();
  const int threads = (D == 3 && !want_jac) ? MHDG_ASM_RES_THREADS_3D : asm_threads<D>();
  size_t budget = ctas > 1 ? (228 * 1024) / ctas - 1024 : 227 * 1024;
  int nqc = sz.nq;  // largest point chunk whose work arrays fit shared memory
  while (nqc > 1 && sizeof(double) * asm_smem<D>(sz, nqc, 1, want_jac != 0).total > budget) nqc = (nqc + 1) / 2;
  if (sizeof(double) * asm_smem<D>(sz, nqc, 1, want_jac != 0).total > budget) {  // no chunk fits the shared budget: one CTA per SM
    budget = 227 * 1024;
    nqc = sz.nq;
    while (nqc > 1 && sizeof(double) * asm_smem<D>(sz, nqc, 1, want_jac != 0).total > budget) nqc = (nqc + 1) / 2;
  }
  if (sizeof(double) * asm_smem<D>(sz, nqc, 1, want_jac != 0).total > budget || sz.n_tri * sz.Lf > ASM_MAXFLOC) return MHDG_ERR_CONFIG;
  int nfg = D + 1;  // faces per group of the face phases: as many as fit beside the kept arrays
  while (nfg > 1 && sizeof(double) * asm_smem<D>(sz, nqc, nfg, want_jac != 0).total > budget) --nfg;
  const size_t bytes = sizeof(double) * asm_smem<D>(sz, nqc, nfg, want_jac != 0).total;
  if (bytes > 48 * 1024) cudaFuncSetAttribute(k_assemble<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  mhdg_blocks bb{};
  mhdg_frozen fzo{}, fzi{};
  if (want_jac) {
    if (!b || (want_jac == 1 && !fo)) return MHDG_ERR_CONFIG;
    bb = *b;
    if (fo) fzo = *fo;
  }
  if (fi) fzi = *fi;
  k_assemble<D><<<g.n_mac, threads, bytes, st>>>(g, fl, sg, u, q, uhat, Rg, Ru, Rtl, want_jac, bb, fzo, fzi,
                                                     fi ? 1 : 0, status, nqc, nfg);
  int rc = launch_ok();
  if (rc) return rc;
  return Rt ? face_reduce(g, Rtl, nullptr, 0.0, Rt, st) : MHDG_OK;
}

template int assemble<2>(const mhdg_disc&, const mhdg_flow&, const mhdg_stage&, const double*, const double*,
                         const double*, double*, double*, double*, double*, int, const mhdg_blocks*, const mhdg_frozen*,
                         const mhdg_frozen*, int*, cudaStream_t);
template int assemble<3>(const mhdg_disc&, const mhdg_flow&, const mhdg_stage&, const double*, const double*,
                         const double*, double*, double*, double*, double*, int, const mhdg_blocks*, const mhdg_frozen*,
                         const mhdg_frozen*, int*, cudaStream_t);

}  // namespace mhdg
