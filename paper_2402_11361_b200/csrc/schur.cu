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

constexpr int SCH2_MAXT = 256;
constexpr int SCH2_MAXPHF = 256;  // nqf x nlocf entries of the face basis table
  // n_sub x nloc entries of the per-CTA node table

template <int D>
struct Sch2 {
  static constexpr int NS = D + 2, NW = D * D * NS * NS, NWF = D * NS * NS;
  // shared-memory strides of the stash (doubles): the (s, r) block of gradient direction l at
  // SR (= 4 mod 16), flux direction k at SK, point q at SQ (= 4 D mod 16), so the A-fragment
  // reads of a half-warp -- 4 consecutive (s, r) x 4 consecutive (q, r') -- fall in 16
  // different banks (the dense strides ns^2, D ns^2, D^2 ns^2 gave 2-way (3D) and 4-way (2D)
  // conflicts); faces: SR per direction, SQF per point
  static constexpr int SR = D == 2 ? 20 : 28, SK = D * SR, SQ = D == 2 ? 88 : 252, SQF = D == 2 ? 40 : 92;
  static constexpr int NT = D == 2 ? 12 : 5;   // n-tiles: L <= 8 NT
  static constexpr int KS = D == 2 ? 8 : 21;   // k-steps: nq D <= 4 KS
  static constexpr int KSF = D == 2 ? 8 : 12;  // face k-steps per sub-face: nqf D <= 4 KSF (3D p <= 3)
#ifndef MHDG_SCHUR_KB3
#define MHDG_SCHUR_KB3 7
#endif
#ifndef MHDG_SCHUR_KB2
#define MHDG_SCHUR_KB2 8
#endif
  static constexpr int KB = D == 2 ? MHDG_SCHUR_KB2 : MHDG_SCHUR_KB3;  // A-fragment k-steps formed at once (divides KS)
#ifndef MHDG_SCHUR3_NBUF
#define MHDG_SCHUR3_NBUF 1
#endif
  // 2D: two stage buffers (stage i+1 streams in during stage i), 8 warps, 2 CTAs per SM;
  // 3D: one stage buffer (a 3D stash is 48 KB) so two CTAs share an SM and cover each
  // other's loads
  static constexpr int NBUF = D == 2 ? 2 : MHDG_SCHUR3_NBUF;
#ifndef MHDG_SCHUR2_NW2D
#define MHDG_SCHUR2_NW2D 8
#endif
  static constexpr int NWARP = D == 2 ? MHDG_SCHUR2_NW2D : (NBUF == 1 ? 8 : 16);
#ifndef MHDG_SCHUR2_MINB2D
#define MHDG_SCHUR2_MINB2D 2
#endif
  static constexpr int MINB = D == 2 ? MHDG_SCHUR2_MINB2D : (NBUF == 1 ? 2 : 1);  // CTAs per SM (register budget)
};

struct Sch2Dims {
  int kv, kf, ksv, ksf, LP, wmax, pmrows, stage, ngph, kfp, rpn, qs, nsl;
  template <int D>
  static Sch2Dims make(const mhdg_disc& g) {
    using C = Sch2<D>;
    Sch2Dims d{};
    // a volume stage holds qs points of one sub-element (its k extent fits the KS
    // compile-time k-steps); nsl stages per sub-element (1 unless nq D > 4 KS, e.g. 3D p = 3)
    d.qs = g.nq * D <= 4 * C::KS ? g.nq : 4 * C::KS / D;
    d.nsl = (g.nq + d.qs - 1) / d.qs;
    d.kv = d.qs * D;
    d.kf = g.nqf * D;
    d.ksv = (d.kv + 3) / 4;
    d.ksf = (d.kf + 3) / 4;
    d.LP = (g.L + 3) / 4 * 4;
    while (d.LP % 16 != 4) d.LP += 4;
    // a face stage holds all n_tri sub-faces of one face: stashes back to back, tables at
    // rows T kfp + k (kfp = 4 ksf: each sub-face starts on a k-step)
    d.kfp = 4 * d.ksf;
    d.rpn = (C::NS * C::NS + 7) / 8 * 8;  // face-stage rows per face node (8-row tiles stay on one node)
    const int wv = d.qs * C::SQ, wf = g.n_tri * g.nqf * C::SQF;
    d.wmax = ((wv > wf ? wv : wf) + 1) & ~1;
    d.pmrows = 4 * C::KS > g.n_tri * d.kfp ? 4 * C::KS : g.n_tri * d.kfp;
    // + padding: the last B fragments of a row read up to 8 NT - LP columns past it
    // (columns >= L are never stored; the padding is zero)
    d.stage = d.wmax + d.pmrows * d.LP + 8 * C::NT;
    d.ngph = (g.nq * g.nloc * D + 1) & ~1;  // one gradient class at a time (the stage's sub-element)
    return d;
  }
  template <int D>
  size_t smem_bytes() const { return sizeof(double) * ((size_t)ngph + Sch2<D>::NBUF * (size_t)stage); }
};

// SLICED: volume stages hold point slices (nsl > 1); the unsliced instantiation keeps the
// k extent per stage uniform (it measured 4% faster in 3D)
template <int D, bool SLICED>
__global__ void __launch_bounds__(Sch2<D>::NWARP * 32, Sch2<D>::MINB) k_schur2(mhdg_disc g, mhdg_blocks b, Sch2Dims dm,
                                                                   double* __restrict__ S) {
  using C = Sch2<D>;
  constexpr int NS = D + 2, NF = D + 1, NW = C::NW, NWF = C::NWF, NT = C::NT, KS = C::KS, NWP = C::NWARP;
  constexpr int NT_THREADS = NWP * 32;
  extern __shared__ __align__(16) double sm[];
  const int mac = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g8 = lane >> 2, t4 = lane & 3;
  const int L = g.L, n = L * NS, nq = g.nq, nloc = g.nloc, nqf = g.nqf, nlocf = g.nlocf;
  double* gph = sm;                      // nq x nloc x D: physical basis gradients of the stage's class
  double* stg = sm + dm.ngph;            // 2 stages: [W' (wmax) | PM (4 KS x LP)]
  double* Sm = S + (size_t)mac * n * n;
  const double* SSm = b.state_state + (size_t)mac * n * n;
  double ij[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int c = 0; c < D; ++c) ij[a][c] = __ldg(g.inv_jac + (size_t)mac * D * D + a * D + c);
  // volume stages (sub-element K = i / nsl, point slice i % nsl), then one stage per face
  const int nvol = g.n_sub * dm.nsl, nstage = nvol + NF;
  // per (sub-element K, local node a): the macro node and whether K is its first toucher
  // (the tile's S rows start from state_state) -- once per CTA, off the tiles' load chains
  // (measured 8.84 -> 8.56 ms at C2)
  __shared__ int tnode[SCH2_MAXT];
  for (int e = tid; e < g.n_sub * nloc; e += NWP * 32) {
    const int node = __ldg(g.sub_conn + e);
    const bool first = __ldg(g.vn_sub + __ldg(g.vn_ptr + node)) / nloc == e / nloc;
    tnode[e] = first ? -1 - node : node;
  }
  // face-lattice incidence: node g lies in sub-faces finc_T[g][k] as local node finc_a[g][k]
  constexpr int MAXINC = 8;
  __shared__ unsigned char finc_T[64][MAXINC], finc_a[64][MAXINC], finc_n[64];
  __shared__ double phf[SCH2_MAXPHF];  // phi_face (nqf x nlocf)
  for (int e = tid; e < nqf * nlocf; e += NT_THREADS) phf[e] = __ldg(g.phi_face + e);
  if (tid == 0) {
    for (int gg = 0; gg < g.Lf && gg < 64; ++gg) finc_n[gg] = 0;
    for (int T = 0; T < g.n_tri; ++T)
      for (int a = 0; a < nlocf; ++a) {
        const int gg = __ldg(g.tri_conn + T * nlocf + a);
        if (gg < 64 && finc_n[gg] < MAXINC) {
          finc_T[gg][finc_n[gg]] = (unsigned char)T;
          finc_a[gg][finc_n[gg]] = (unsigned char)a;
          ++finc_n[gg];
        }
      }
  }

  auto prefetch = [&](int i) {
    if (i >= nstage) return;
    double* W = stg + (size_t)(i % C::NBUF) * dm.stage;
    double* PM = W + dm.wmax;
    const double* wsrc;
    const double* psrc;
    int wcnt, kk;
    if (i < nvol) {
      const int K = SLICED ? i / dm.nsl : i, q0 = SLICED ? (i % dm.nsl) * dm.qs : 0;
      const int nqs = SLICED ? min(dm.qs, nq - q0) : nq;
      wsrc = b.wdgdq_vol + (((size_t)mac * g.n_sub + K) * nq + q0) * NW;
      wcnt = nqs * NW;
      psrc = g.pm_vol + ((size_t)K * nq + q0) * D * L;
      kk = nqs * D;
    } else {
      const int f = i - nvol;
      wsrc = b.wdgdq_face + ((size_t)mac * NF + f) * g.n_tri * nqf * NWF;
      wcnt = g.n_tri * nqf * NWF;
      psrc = g.pm_face + (size_t)f * g.n_tri * dm.kf * L;
      kk = g.n_tri * dm.kf;
    }
    if (i < nvol) {
      for (int e = tid; e < wcnt; e += NT_THREADS) {
        const int pt = e / NW, rem = e - pt * NW, k = rem / (D * NS * NS), l = (rem / (NS * NS)) % D,
                  sr = rem % (NS * NS);
        cp_async8(W + pt * C::SQ + k * C::SK + l * C::SR + sr, wsrc + e, 8);
      }
    } else {
      for (int e = tid; e < wcnt; e += NT_THREADS) {
        const int pt = e / NWF, rem = e - pt * NWF, l = rem / (NS * NS), sr = rem % (NS * NS);
        cp_async8(W + pt * C::SQF + l * C::SR + sr, wsrc + e, 8);
      }
    }
    for (int e = tid; e < kk * L; e += NT_THREADS) {
      const int row = e / L, j = e - row * L;
      const int prow = i < nvol ? row : (row / dm.kf) * dm.kfp + row % dm.kf;
      cp_async8(PM + prow * dm.LP + j, psrc + e, 8);
    }
  };

  // PM padding (rows >= kv, columns >= L) must be finite: zero both stages once
  for (int e = tid; e < C::NBUF * dm.stage; e += NT_THREADS) stg[e] = 0.0;
  __syncthreads();
  prefetch(0);

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
    if (vol && (!SLICED || i % dm.nsl == 0)) {  // physical gradients of this sub-element's class (geometry folded in)
      const double* gc = g.grad_cls + (size_t)__ldg(g.grad_cls_of + (SLICED ? i / dm.nsl : i)) * nq * nloc * D;
      for (int idx = tid; idx < nq * nloc * D; idx += NT_THREADS) {
        const int k = idx % D, base = idx - k;
        double v = 0.0;
#pragma unroll
        for (int r = 0; r < D; ++r) v += __ldg(gc + base + r) * ij[r][k];
        gph[idx] = v;
      }
    }
    {  // fold inv_jac into the stash in place: W'[..(k, r')..] = sum_l ij[r'][l] W[..(k, l)..]
      const int ngrp = (vol ? (SLICED ? min(dm.qs, nq - (i % dm.nsl) * dm.qs) : nq) * D : g.n_tri * nqf) * NS * NS;
      for (int e = tid; e < ngrp; e += NT_THREADS) {
        const int sr = e % (NS * NS), qk = e / (NS * NS);  // volume: qk = q D + k; faces: the point
        double* w = W + (vol ? (qk / D) * C::SQ + (qk % D) * C::SK : qk * C::SQF) + sr;
        double v[D];
#pragma unroll
        for (int l = 0; l < D; ++l) v[l] = w[l * C::SR];
#pragma unroll
        for (int rp = 0; rp < D; ++rp) {
          double t = 0.0;
#pragma unroll
          for (int l = 0; l < D; ++l) t += ij[rp][l] * v[l];
          w[rp * C::SR] = t;
        }
      }
    }
    __syncthreads();
    if (vol) {
      const int rows = nloc * NS * NS;
      const int K = SLICED ? i / dm.nsl : i, sl = SLICED ? i % dm.nsl : 0, q0 = sl * dm.qs;
      const int kvs = SLICED ? min(dm.qs, nq - q0) * D : dm.kv;  // this slice's k extent
      const int ksv = SLICED ? (kvs + 3) / 4 : dm.ksv;
      const int cls = __ldg(g.grad_cls_of + K);
      for (int mt = warp; mt * 8 < rows; mt += NWP) {
        const int m = mt * 8 + g8;
        const bool mok = m < rows;
        const int a = mok ? m / (NS * NS) : 0, s = (m / NS) % NS, r = m % NS;
        // S row of this thread's output row, and where its accumulators start from
        int node;
        bool first;
        {
          const int tn = tnode[K * nloc + a];
          first = tn < 0;
          node = first ? -1 - tn : tn;
        }
        first = first && sl == 0;
        double* srow = Sm + (size_t)(node * NS + s) * n + r;
        const double* crow = first ? SSm + (size_t)(node * NS + s) * n + r : srow;
        double c[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int j0 = nt * 8 + 2 * t4;
          c[nt][0] = (mok && j0 < L) ? crow[j0 * NS] : 0.0;
          c[nt][1] = (mok && j0 + 1 < L) ? crow[(j0 + 1) * NS] : 0.0;
        }
        const double* gp = gph + a * D;
        const double* w = W + (s * NS + r);
        if constexpr (D == 3) {
          // 3D: the k index runs over blocks of 4 points, r' inside a block: lane t4 owns point
          // 4 b + t4 of block b, so every offset is a per-lane base plus a compile-time constant
          // (no index divisions), a point's gradient entries are loaded once for its D k-steps,
          // and the lanes' stash / PM rows fall in different banks (SQ = 12, D LP = 12 mod 16)
          constexpr int NBK = KS / D;
          const int nqs = SLICED ? min(dm.qs, nq - q0) : nq, nblk = (nqs + 3) / 4;
          const double* gq0 = gp + (size_t)(q0 + t4) * nloc * D;
          const double* wq0 = w + t4 * C::SQ;
          const double* pb0 = PM + (t4 * D) * dm.LP + g8;
#pragma unroll
          for (int b = 0; b < NBK; b += 2) {
            double af[2 * D];
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const int bb = b + hh;
              const bool ok = mok && bb < NBK && 4 * bb + t4 < nqs;
              double gk[D];
#pragma unroll
              for (int k = 0; k < D; ++k) gk[k] = ok ? gq0[4 * bb * nloc * D + k] : 0.0;
#pragma unroll
              for (int rp = 0; rp < D; ++rp) {
                double v = 0.0;
                if (ok) {
                  const double* wq = wq0 + 4 * bb * C::SQ + rp * C::SR;
#pragma unroll
                  for (int k = 0; k < D; ++k) v += gk[k] * wq[k * C::SK];
                }
                af[hh * D + rp] = v;
              }
            }
#pragma unroll
            for (int hh = 0; hh < 2; ++hh)
              if (b + hh < NBK && b + hh < nblk) {
#pragma unroll
                for (int rp = 0; rp < D; ++rp) {
                  const double* pb = pb0 + (4 * (b + hh) * D + rp) * dm.LP;
#pragma unroll
                  for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(c[nt][0], c[nt][1], af[hh * D + rp], pb[nt * 8]);
                }
              }
          }
        } else {
        // A fragments of this row, T1[m][(q, r') = 4 ks + t4], formed KB k-steps at a time (3D:
        // the 21 k-steps at once spilled registers inside this loop)
        constexpr int KB = C::KB;
#pragma unroll
        for (int kb = 0; kb < KS; kb += KB) {
          double af[KB];
#pragma unroll
          for (int kk = 0; kk < KB; ++kk) {
            const int ks = kb + kk, kq = 4 * ks + t4;
            double v = 0.0;
            if (mok && ks < ksv && kq < kvs) {
              const int q = kq / D, rp = kq - q * D;  // slice-local point; q0 + q in the tables
              const double* gq = gp + (size_t)(q0 + q) * nloc * D;
              const double* wq = w + q * C::SQ + rp * C::SR;
#pragma unroll
              for (int k = 0; k < D; ++k) v += gq[k] * wq[k * C::SK];
            }
            af[kk] = v;
          }
#pragma unroll
          for (int kk = 0; kk < KB; ++kk)
            if (kb + kk < ksv) {
              const double* pb = PM + (4 * (kb + kk) + t4) * dm.LP + g8;
#pragma unroll
              for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(c[nt][0], c[nt][1], af[kk], pb[nt * 8]);
            }
        }
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int j0 = nt * 8 + 2 * t4;
          if (mok && j0 < L) srow[j0 * NS] = c[nt][0];
          if (mok && j0 + 1 < L) srow[(j0 + 1) * NS] = c[nt][1];
        }
      }
    } else {
      // face f, all sub-faces at once: rows (face node gg, s, r), rpn rows per node, so an
      // 8-row tile stays on one node and sums its sub-faces in order (T ascending: the
      // reference's accumulation order), -W'_T[q][r'][s][r] phi_face[q][a] against PM_T
      const int f = i - nvol;
      constexpr int KSF = C::KSF;
      for (int mt = warp; mt * 8 < g.Lf * dm.rpn; mt += NWP) {
        const int gg = (mt * 8) / dm.rpn, sr = mt * 8 - gg * dm.rpn + g8;
        const bool mok = sr < NS * NS;
        const int s = mok ? sr / NS : 0, r = mok ? sr % NS : 0;
        const int node = __ldg(g.face_vol_nodes + f * g.Lf + gg);
        double* srow = Sm + (size_t)(node * NS + s) * n + r;
        double c[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int j0 = nt * 8 + 2 * t4;
          c[nt][0] = (mok && j0 < L) ? srow[j0 * NS] : 0.0;
          c[nt][1] = (mok && j0 + 1 < L) ? srow[(j0 + 1) * NS] : 0.0;
        }
        const int ninc = finc_n[gg];
        for (int e = 0; e < ninc; ++e) {
          const int T = finc_T[gg][e], a = finc_a[gg][e];
          const double* WT = W + T * nqf * C::SQF;
          double af[KSF];
          if constexpr (D == 3) {
            // k index by blocks of 4 points, r' inside a block (as the volume stages): lane t4
            // owns point 4 b + t4, one basis value per point, compile-time offsets, no divisions
            constexpr int NBF = KSF / D;
            const int nblk = (nqf + 3) / 4;
            const double* wq0 = WT + s * NS + r;
            const double* pb0 = PM + (T * dm.kfp) * dm.LP + g8;
#pragma unroll
            for (int bq = 0; bq < NBF; ++bq) {
              const int q = 4 * bq + t4;
              const bool ok = mok && bq < nblk && q < nqf;
              const double ph = ok ? -phf[q * nlocf + a] : 0.0;
#pragma unroll
              for (int rp = 0; rp < D; ++rp) af[bq * D + rp] = ok ? wq0[q * C::SQF + rp * C::SR] * ph : 0.0;
            }
#pragma unroll
            for (int bq = 0; bq < NBF; ++bq)
              if (bq < nblk) {
                const int qc = min(4 * bq + t4, nqf - 1);  // rows of padded points: any finite row (af = 0)
#pragma unroll
                for (int rp = 0; rp < D; ++rp) {
                  const double* pb = pb0 + (qc * D + rp) * dm.LP;
#pragma unroll
                  for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(c[nt][0], c[nt][1], af[bq * D + rp], pb[nt * 8]);
                }
              }
            continue;
          }
#pragma unroll
          for (int ks = 0; ks < KSF; ++ks) {
            const int kq = 4 * ks + t4;
            double v = 0.0;
            if (mok && ks < dm.ksf && kq < dm.kf) {
              const int q = kq / D, rp = kq - q * D;
              v = -WT[q * C::SQF + rp * C::SR + s * NS + r] * phf[q * nlocf + a];
            }
            af[ks] = v;
          }
#pragma unroll
          for (int ks = 0; ks < KSF; ++ks)
            if (ks < dm.ksf) {
              const double* pb = PM + (T * dm.kfp + 4 * ks + t4) * dm.LP + g8;
#pragma unroll
              for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(c[nt][0], c[nt][1], af[ks], pb[nt * 8]);
            }
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int j0 = nt * 8 + 2 * t4;
          if (mok && j0 < L) srow[j0 * NS] = c[nt][0];
          if (mok && j0 + 1 < L) srow[(j0 + 1) * NS] = c[nt][1];
        }
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
  if (!g.grad_cls || g.L > 8 * C::NT || dm.ksv > C::KS || dm.ksf > C::KSF || g.Lf > 64 || bytes > 227 * 1024 ||
      g.n_sub * g.nloc > SCH2_MAXT || g.nqf * g.nlocf > SCH2_MAXPHF)
    return -1;
  auto kern = dm.nsl > 1 ? k_schur2<D, true> : k_schur2<D, false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  kern<<<g.n_mac, C::NWARP * 32, bytes, st>>>(g, b, dm, S);
  return launch_ok();
}

template int schur2<2>(const mhdg_disc&, const mhdg_blocks&, double*, cudaStream_t);
template int schur2<3>(const mhdg_disc&, const mhdg_blocks&, double*, cudaStream_t);

}  // namespace mhdg
