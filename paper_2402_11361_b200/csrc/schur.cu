// Second-layer Schur complement S = A_uu - A_uq A_qq^-1 A_qu on the FP64 tensor
// cores (_schur_correction, condense.py:130-158 of the reference).
//
// k_schur2: one CTA per macro.  With the inverse Jacobian folded into the
// stashed viscous Jacobians, each volume (face) sub-element K contributes
//   X[(a,s,r), j] = sum_{(q,r')} T1[(a,s,r),(q,r')] PM_K[(q,r'), j],
//   T1[(a,s,r),(q,r')] = sum_k gphys[q,a,k] W'[q][(k,r')][s][r]
//   (faces: T1 = -W'[q][r'][s][r] phi_face[q,a]),
// added to S rows (conn[a], s), columns (j, r), in the reference's sub-element
// order (so S is deterministic).  Sub-elements are a pipeline of shared-memory
// stages: while the warps run stage i, stage i+1's stash W (per macro, HBM)
// and table PM (macro-independent, L2) stream in with cp.async.  Inside a
// stage every warp owns 8-row tiles of X and needs no barrier: its DMMA
// A fragments are formed in registers straight from W' and the gradient
// table, B fragments come from PM (row stride = 4 mod 16: conflict-free), and
// the accumulators are seeded from the S rows they update (from state_state
// on a row's first touch), so the read-modify-write of S is the MMA
// accumulate.
#include "common.cuh"
#include "dmma.cuh"

namespace mhdg {

template <int D>
struct Sch2 {
  static constexpr int NS = D + 2, NW = D * D * NS * NS, NWF = D * NS * NS;
  static constexpr int NT = D == 2 ? 12 : 5;   // n-tiles: L <= 8 NT
  static constexpr int KS = D == 2 ? 8 : 21;   // k-steps: nq D <= 4 KS
#ifndef MHDG_SCHUR3_NBUF
#define MHDG_SCHUR3_NBUF 1
#endif
  // 2D: two stage buffers (stage i+1 streams in during stage i), 8 warps, 2 CTAs per SM;
  // 3D: one stage buffer (a 3D stash is 48 KB) so two CTAs share an SM and cover each
  // other's loads
  static constexpr int NBUF = D == 2 ? 2 : MHDG_SCHUR3_NBUF;
  static constexpr int NWARP = (D == 2 || NBUF == 1) ? 8 : 16;
  static constexpr int MINB = (D == 2 || NBUF == 1) ? 2 : 1;  // CTAs per SM the registers are budgeted for
};

struct Sch2Dims {
  int kv, kf, ksv, ksf, LP, wmax, stage, ngph;
  template <int D>
  static Sch2Dims make(const mhdg_disc& g) {
    using C = Sch2<D>;
    Sch2Dims d{};
    d.kv = g.nq * D;
    d.kf = g.nqf * D;
    d.ksv = (d.kv + 3) / 4;
    d.ksf = (d.kf + 3) / 4;
    d.LP = (g.L + 3) / 4 * 4;
    while (d.LP % 16 != 4) d.LP += 4;
    const int wv = g.nq * C::NW, wf = g.nqf * C::NWF;
    d.wmax = ((wv > wf ? wv : wf) + 1) & ~1;
    // + padding: the last B fragments of a row read up to 8 NT - LP columns past it
    // (columns >= L are never stored; the padding is zero)
    d.stage = d.wmax + 4 * C::KS * d.LP + 8 * C::NT;
    d.ngph = (g.n_grad_cls * g.nq * g.nloc * D + 1) & ~1;
    return d;
  }
  template <int D>
  size_t smem_bytes() const { return sizeof(double) * ((size_t)ngph + Sch2<D>::NBUF * (size_t)stage); }
};

template <int D>
__global__ void __launch_bounds__(Sch2<D>::NWARP * 32, Sch2<D>::MINB) k_schur2(mhdg_disc g, mhdg_blocks b, Sch2Dims dm,
                                                                   double* __restrict__ S) {
  using C = Sch2<D>;
  constexpr int NS = D + 2, NF = D + 1, NW = C::NW, NWF = C::NWF, NT = C::NT, KS = C::KS, NWP = C::NWARP;
  constexpr int NT_THREADS = NWP * 32;
  extern __shared__ __align__(16) double sm[];
  const int mac = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g8 = lane >> 2, t4 = lane & 3;
  const int L = g.L, n = L * NS, nq = g.nq, nloc = g.nloc, nqf = g.nqf, nlocf = g.nlocf;
  double* gph = sm;                      // n_grad_cls x nq x nloc x D: physical basis gradients
  double* stg = sm + dm.ngph;            // 2 stages: [W' (wmax) | PM (4 KS x LP)]
  double* Sm = S + (size_t)mac * n * n;
  const double* SSm = b.state_state + (size_t)mac * n * n;
  double ij[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int c = 0; c < D; ++c) ij[a][c] = __ldg(g.inv_jac + (size_t)mac * D * D + a * D + c);
  const int nvol = g.n_sub, nstage = g.n_sub + NF * g.n_tri;

  auto prefetch = [&](int i) {
    if (i >= nstage) return;
    double* W = stg + (size_t)(i % C::NBUF) * dm.stage;
    double* PM = W + dm.wmax;
    const double* wsrc;
    const double* psrc;
    int wcnt, kk;
    if (i < nvol) {
      wsrc = b.wdgdq_vol + ((size_t)mac * nvol + i) * nq * NW;
      wcnt = nq * NW;
      psrc = g.pm_vol + (size_t)i * dm.kv * L;
      kk = dm.kv;
    } else {
      const int fT = i - nvol;
      wsrc = b.wdgdq_face + ((size_t)mac * NF * g.n_tri + fT) * nqf * NWF;
      wcnt = nqf * NWF;
      psrc = g.pm_face + (size_t)fT * dm.kf * L;
      kk = dm.kf;
    }
    for (int e = tid; e < wcnt; e += NT_THREADS) cp_async8(W + e, wsrc + e, 8);
    for (int e = tid; e < kk * L; e += NT_THREADS) {
      const int row = e / L, j = e - row * L;
      cp_async8(PM + row * dm.LP + j, psrc + e, 8);
    }
  };

  // PM padding (rows >= kv, columns >= L) must be finite: zero both stages once
  for (int e = tid; e < C::NBUF * dm.stage; e += NT_THREADS) stg[e] = 0.0;
  __syncthreads();
  prefetch(0);
  // physical gradients per class (geometry folded in once per macro)
  for (int idx = tid; idx < g.n_grad_cls * nq * nloc * D; idx += NT_THREADS) {
    const int k = idx % D, base = idx - k;
    double v = 0.0;
#pragma unroll
    for (int r = 0; r < D; ++r) v += __ldg(g.grad_cls + base + r) * ij[r][k];
    gph[idx] = v;
  }

  for (int i = 0; i < nstage; ++i) {
    if (C::NBUF == 1 && i > 0) {
      __syncthreads();  // stage i-1 consumed: its buffer takes stage i
      prefetch(i);
    }
    cp_async_wait_all();
    __syncthreads();  // stage i landed; stage i-1 consumed (its buffer is free)
    if (C::NBUF > 1) prefetch(i + 1);
    const bool vol = i < nvol;
    double* W = stg + (size_t)(i % C::NBUF) * dm.stage;
    const double* PM = W + dm.wmax;
    {  // fold inv_jac into the stash in place: W'[..(k, r')..] = sum_l ij[r'][l] W[..(k, l)..]
      const int ngrp = (vol ? nq * D : nqf) * NS * NS;
      for (int e = tid; e < ngrp; e += NT_THREADS) {
        const int sr = e % (NS * NS), qk = e / (NS * NS);
        double* w = W + (size_t)qk * D * NS * NS + sr;
        double v[D];
#pragma unroll
        for (int l = 0; l < D; ++l) v[l] = w[l * NS * NS];
#pragma unroll
        for (int rp = 0; rp < D; ++rp) {
          double t = 0.0;
#pragma unroll
          for (int l = 0; l < D; ++l) t += ij[rp][l] * v[l];
          w[rp * NS * NS] = t;
        }
      }
    }
    __syncthreads();
    const int rows = (vol ? nloc : nlocf) * NS * NS;
    const int kdim = vol ? dm.kv : dm.kf, nks = vol ? dm.ksv : dm.ksf;
    const int K = i, fT = i - nvol, f = fT / (g.n_tri > 0 ? g.n_tri : 1), T = fT - f * g.n_tri;
    const int cls = vol ? __ldg(g.grad_cls_of + K) : 0;
    // S row of an 8-row tile's output row, and where its accumulators start from
    struct Row {
      double* srow;
      const double* crow;
      int a, s, r;
      bool ok;
    };
    auto row_of = [&](int mt) {
      Row q;
      const int m = mt * 8 + g8;
      q.ok = m < rows;
      q.a = q.ok ? m / (NS * NS) : 0;
      q.s = (m / NS) % NS;
      q.r = m % NS;
      int node;
      bool first = false;
      if (vol) {
        node = __ldg(g.sub_conn + K * nloc + q.a);
        first = __ldg(g.vn_sub + __ldg(g.vn_ptr + node)) / nloc == K;
      } else {
        node = __ldg(g.face_vol_nodes + f * g.Lf + __ldg(g.tri_conn + T * nlocf + q.a));
      }
      q.srow = Sm + (size_t)(node * NS + q.s) * n + q.r;
      q.crow = first ? SSm + (size_t)(node * NS + q.s) * n + q.r : q.srow;
      return q;
    };
    auto load_c = [&](const Row& q, double (&c)[NT][2]) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int j0 = nt * 8 + 2 * t4;
        c[nt][0] = (q.ok && j0 < L) ? q.crow[j0 * NS] : 0.0;
        c[nt][1] = (q.ok && j0 + 1 < L) ? q.crow[(j0 + 1) * NS] : 0.0;
      }
    };
    for (int mt = warp; mt * 8 < rows; mt += NWP) {
      const Row q = row_of(mt);
      double c[NT][2];
      load_c(q, c);
      // A fragments of this row: T1[m][(q, r') = 4 ks + t4]
      double af[KS];
      if (vol) {
        const double* gp = gph + (size_t)(cls * nq) * nloc * D + q.a * D;
        const double* w = W + (q.s * NS + q.r);
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const int kq = 4 * ks + t4;
          double v = 0.0;
          if (q.ok && ks < nks && kq < kdim) {
            const int qq = kq / D, rp = kq - qq * D;
            const double* gq = gp + (size_t)qq * nloc * D;
            const double* wq = w + (size_t)qq * NW + rp * NS * NS;
#pragma unroll
            for (int k = 0; k < D; ++k) v += gq[k] * wq[k * D * NS * NS];
          }
          af[ks] = v;
        }
      } else {
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const int kq = 4 * ks + t4;
          double v = 0.0;
          if (q.ok && ks < nks && kq < kdim) {
            const int qq = kq / D, rp = kq - qq * D;
            v = -W[((qq * D + rp) * NS + q.s) * NS + q.r] * __ldg(g.phi_face + qq * nlocf + q.a);
          }
          af[ks] = v;
        }
      }
#pragma unroll
      for (int ks = 0; ks < KS; ++ks)
        if (ks < nks) {
          const double* pb = PM + (4 * ks + t4) * dm.LP + g8;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(c[nt][0], c[nt][1], af[ks], pb[nt * 8]);
        }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int j0 = nt * 8 + 2 * t4;
        if (q.ok && j0 < L) q.srow[j0 * NS] = c[nt][0];
        if (q.ok && j0 + 1 < L) q.srow[(j0 + 1) * NS] = c[nt][1];
      }
    }
  }
}

// -1 when the shapes exceed the compile-time tiles or shared memory
template <int D>
int schur2(const mhdg_disc& g, const mhdg_blocks& b, double* S, cudaStream_t st) {
  using C = Sch2<D>;
  const Sch2Dims dm = Sch2Dims::make<D>(g);
  const size_t bytes = dm.smem_bytes<D>();
  if (!g.grad_cls || g.L > 8 * C::NT || dm.ksv > C::KS || dm.ksf > C::KS || bytes > 227 * 1024) return -1;
  cudaFuncSetAttribute(k_schur2<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  k_schur2<D><<<g.n_mac, C::NWARP * 32, bytes, st>>>(g, b, dm, S);
  return launch_ok();
}

template int schur2<2>(const mhdg_disc&, const mhdg_blocks&, double*, cudaStream_t);
template int schur2<3>(const mhdg_disc&, const mhdg_blocks&, double*, cudaStream_t);

}  // namespace mhdg
