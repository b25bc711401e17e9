// Streaming matrix-free trace apply: warp-specialised, TMA-fed, persistent.
//
// Same operator as k_apply_local (CondensedSchur.apply_trace,
// condense.py:91-103; Algorithm 2 steps 1-4), restructured
// for the B200 memory system:
//   * sizes are compile-time (template <D, M, P>): every index is a constant
//     multiply/shift and every small loop unrolls;
//   * one producer warp streams each macro's operator data -- face blocks,
//     dG/dq stashes and the packed LU factor (packed_lu.cuh) -- in exactly
//     the order the math consumes it, as 1D bulk copies (cp.async.bulk, TMA)
//     into a ring of shared-memory stages guarded by mbarriers;
//   * eight consumer warps do all arithmetic out of shared memory, so the
//     bytes in flight are set by the ring depth, not by thread count;
//   * CTAs are persistent (grid = SMs x CTAs/SM) and walk the macros.
// Results match k_apply_local to rounding; all reductions are in a fixed order.
#include "local_ops.cuh"
#include "packed_lu.cuh"
#include "tiled_inv.cuh"
#include "tma.cuh"

namespace mhdg {

__host__ __device__ constexpr int cbinom(int n, int k) {
  int r = 1;
  for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return r;
}
__host__ __device__ constexpr int cpow(int b, int e) {
  int r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}
__host__ __device__ constexpr int ceven(int x) { return x + (x & 1); }

constexpr int ST_DBL = 2112;  // doubles per ring stage (16.5 KB: one 64x32 LU tile or a 64-row inverted triangle)
constexpr int NCONS = 256;    // consumer threads (8 warps)

template <int D_, int M_, int P_>
struct Cfg {
  static constexpr int D = D_, M = M_, P = P_;
  static constexpr int NS = D + 2, NF = D + 1, N = M * P;
  static constexpr int L = cbinom(N + D, D), LF = cbinom(N + D - 1, D - 1);
  static constexpr int n = L * NS, BS = LF * NS, LTR = NF * BS;
  static constexpr int NSUB = cpow(M, D), NLOC = cbinom(P + D, D), NQ = cpow(P + 1, D);
  static constexpr int NTRI = cpow(M, D - 1), NLOCF = cbinom(P + D - 1, D - 1), NQF = cpow(P + 1, D - 1);
  static constexpr int NW = D * D * NS * NS, NWF = D * NS * NS;
  static constexpr int NPV = NSUB * NQ, NPF = NF * NTRI * NQF;
  // rows / points per ring stage (even counts where the unit has odd size)
  static constexpr int RPP = (BS & 1) ? ((ST_DBL / BS) & ~1) : ST_DBL / BS;
  static constexpr int PPV = (NW & 1) ? ((ST_DBL / NW) & ~1) : ST_DBL / NW;
  static constexpr int PPF = (NWF & 1) ? ((ST_DBL / NWF) & ~1) : ST_DBL / NWF;
  static constexpr int NBLK = (n + TI_RB - 1) / TI_RB;
  static constexpr int NFN = L - (N - 1 >= D ? cbinom(N - 1, D) : 0);  // boundary lattice nodes
};

enum : int { K_FST = 0, K_FTT, K_WV, K_WFZ, K_SI, K_LFD, K_UB, K_UBD, K_WF2, K_FTS, K_GF, K_MD };

struct Piece {
  unsigned char kind, blk;
  unsigned short u0, nu, cnt;  // cnt: doubles (even)
  unsigned off;                // doubles from the segment's per-macro (or table) base
};

__host__ __device__ __forceinline__ int units_per_piece(int unit) {
  int r = ST_DBL / unit;
  if (unit & 1) r &= ~1;
  return r < 1 ? 1 : r;
}

// Walks one macro's pieces in consumption order; the producer and the
// consumers run identical copies.  Segment order:
//   Gf table | FST | FTT | W_vol | W_face(z) | LU fwd | LU bwd | M^-1 D table | W_face(z2) | FTS
template <class C>
struct Sched {
  int seg = 0, i = 0, b = 0, r = 0;
  __host__ __device__ bool rows(Piece& p, int kind, int nrows, int unit) {
    const int per = units_per_piece(unit);
    if (i * per >= nrows) return false;
    p.kind = (unsigned char)kind;
    p.u0 = (unsigned short)(i * per);
    p.nu = (unsigned short)(per < nrows - i * per ? per : nrows - i * per);
    p.off = (unsigned)((long long)p.u0 * unit);
    p.cnt = (unsigned short)ceven(p.nu * unit);
    p.blk = 0;
    ++i;
    return true;
  }
  __host__ __device__ bool next(Piece& p) {
    while (seg < 10) {
      switch (seg) {
        case 0: if (rows(p, K_GF, C::NF * C::L, C::LF)) return true; break;
        case 1: if (rows(p, K_FST, C::NF * C::BS, C::BS)) return true; break;
        case 2: if (rows(p, K_FTT, C::NF * C::BS, C::BS)) return true; break;
        case 3: if (rows(p, K_WV, C::NPV, C::NW)) return true; break;
        case 4: if (rows(p, K_WFZ, C::NPF, C::NWF)) return true; break;
        case 5:  // S^-1: row blocks of TI_RB rows, each as TI_CW-column tiles
          if (b < C::NBLK) {
            const int nb = ti_rows(C::n, b);
            const int w = (C::n - r) < TI_CW ? C::n - r : TI_CW;
            p.kind = K_SI;
            p.u0 = (unsigned short)r;
            p.nu = (unsigned short)w;
            p.off = (unsigned)(ti_block_off(C::n, b) + (long long)(r / TI_CW) * nb * TI_CW);
            p.cnt = (unsigned short)ti_even((long long)nb * w);
            p.blk = (unsigned char)b;
            r += w;
            if (r >= C::n) { r = 0; ++b; }
            return true;
          }
          break;
        case 6:
          break;
        case 7: if (rows(p, K_MD, C::D * C::NFN, C::L)) return true; break;
        case 8: if (rows(p, K_WF2, C::NPF, C::NWF)) return true; break;
        case 9: if (rows(p, K_FTS, C::NF * C::BS, C::BS)) return true; break;
      }
      ++seg;
      i = 0;
      r = 0;
      b = 0;
    }
    return false;
  }
};

template <class C>
struct SSm {  // consumer work layout (doubles), after the ring
  static constexpr int PPV = ST_DBL / C::NW > 0 ? ((C::NW & 1) ? ((ST_DBL / C::NW) & ~1) : ST_DBL / C::NW) : 1;
  static constexpr int PPF = (C::NWF & 1) ? ((ST_DBL / C::NWF) & ~1) : ST_DBL / C::NWF;
  static constexpr int xl = 0;
  static constexpr int z = xl + C::LTR;  // z, later z2
  static constexpr int y = z + C::D * C::n;
  static constexpr int t = y + C::n;
  static constexpr int rfst = t + C::n;
  static constexpr int ftt = rfst + C::LTR;
  static constexpr int fts = ftt + C::LTR;
  static constexpr int cfgz = fts + C::LTR;
  static constexpr int yf = cfgz + C::LTR;
  static constexpr int wfz = yf + C::LTR;
  static constexpr int wf2 = wfz + C::NPF * C::NS;
  static constexpr int vv = wf2 + C::NPF * C::NS;  // 8 warps x 32 doubles
  static constexpr int cv = vv + 8 * 32;
  static constexpr int tg = cv + C::NSUB * C::NLOC * C::NS;  // Gf x | W_vol results | M^-1 D y
  static constexpr int TGN0 = C::NF * C::n;
  static constexpr int TGN = TGN0 > C::NPV * C::D * C::NS ? TGN0 : C::NPV * C::D * C::NS;
  static constexpr int tp = tg + TGN;
  static constexpr int total = tp + PLU_NB;
};

__device__ __forceinline__ void cbar() { named_bar(1, NCONS); }

constexpr int NWARP_C = NCONS / 32;

// optional cycle accounting (build with -DMHDG_STREAM_PROFILE): per piece kind,
// [wait-for-data, compute, transition] cycles summed over CTAs (warp 0 lane 0)
#ifdef MHDG_STREAM_PROFILE
__device__ unsigned long long g_prof[16][3];
#define PROF_T(v) long long v = clock64()
#define PROF_ADD(k, j, v) atomicAdd(&g_prof[k][j], (unsigned long long)(clock64() - (v)))
#else
#define PROF_T(v)
#define PROF_ADD(k, j, v)
#endif
constexpr int MAXP = 256;  // pieces per macro (checked on the host)

// acc_r = sum_c A[r][c] vec_r[c] for the nu rows of a staged piece, LPR lanes
// per row; out(r, acc) on one lane per row.  Warps take rows independently.
template <int LPR, class VecF, class OutF>
__device__ __forceinline__ void rows_dot(const double* A, int nu, int ncol, VecF vec, OutF out) {
  constexpr int RPW = 32 / LPR;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / LPR, l = lane % LPR;
  for (int r0 = warp * RPW; r0 < nu; r0 += NWARP_C * RPW) {
    const int rl = r0 + sub;
    double acc = 0.0;
    if (rl < nu) {
      const double* a = A + rl * ncol;
      const double* v = vec(rl);
      for (int c = l; c < ncol; c += LPR) acc += a[c] * v[c];
    }
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(MHDG_FULL, acc, o);
    if (l == 0 && rl < nu) out(rl, acc);
  }
}

template <class C, int STAGES>
__global__ void __launch_bounds__(NCONS + 32) k_apply_stream(mhdg_disc g, mhdg_blocks bk, mhdg_factors fac,
                                                             const double* __restrict__ x,
                                                             double* __restrict__ y_loc, int pref_ahead) {
  constexpr int D = C::D, NS = C::NS, NF = C::NF, L = C::L, LF = C::LF, BS = C::BS, LTR = C::LTR, n = C::n;
  constexpr int NLOC = C::NLOC, NQ = C::NQ, NLOCF = C::NLOCF, NQF = C::NQF, NTRI = C::NTRI;
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES];
  __shared__ Piece pieces[MAXP];
  __shared__ int npieces;
  double* ring = smem;
  double* W = smem + STAGES * ST_DBL;
  using S = SSm<C>;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long PK = ti_size(n);

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], NWARP_C);  // one arrival per consumer warp
    }
    fence_mbar_init();
    // the piece schedule is identical for every macro: build it once
    Sched<C> sc;
    int np = 0;
    while (np < MAXP && sc.next(pieces[np])) ++np;
    npieces = np;
  }
  __syncthreads();
  const int np = npieces;

  // ----------------------------- producer ---------------------------------
  // One thread walks the (macro, piece) sequence twice: a prefetch cursor
  // pulls pieces from HBM into L2 up to PREF_AHEAD pieces ahead, and the copy
  // cursor moves them L2 -> shared ring stage once the consumers free it.
  if (warp == NWARP_C) {
    if (lane == 0) {
      auto src_of = [&](int mac, const Piece& p) -> const double* {
        switch (p.kind) {
          case K_GF: return g.gf + p.off;
          case K_MD: return g.minv_d_face + p.off;
          case K_FST: return bk.face_state_trace + (size_t)mac * NF * BS * BS + p.off;
          case K_FTT: return bk.face_trace_trace + (size_t)mac * NF * BS * BS + p.off;
          case K_FTS: return bk.face_trace_state + (size_t)mac * NF * BS * BS + p.off;
          case K_WV: return bk.wdgdq_vol + (size_t)mac * C::NPV * C::NW + p.off;
          case K_WFZ:
          case K_WF2: return bk.wdgdq_face + (size_t)mac * C::NPF * C::NWF + p.off;
          default: return fac.lu + (size_t)mac * PK + p.off;  // S^-1 tiles
        }
      };
      int pm = blockIdx.x, pp = 0, pref = 0;  // prefetch cursor (macro, piece), pieces issued
      int it = 0;
      for (int mac = blockIdx.x; mac < g.n_mac; mac += gridDim.x) {
        for (int pi = 0; pi < np; ++pi) {
          const Piece& p = pieces[pi];
          const int s = it % STAGES;
          // keep the prefetch cursor PREF_AHEAD pieces ahead of the copy cursor
          while (pref < it + pref_ahead && pm < g.n_mac) {
            const Piece& q = pieces[pp];
            if (q.kind != K_GF && q.kind != K_MD && q.cnt) bulk_prefetch_l2(src_of(pm, q), (uint32_t)q.cnt * 8u);
            ++pref;
            if (++pp == np) { pp = 0; pm += gridDim.x; }
          }
          if (it >= STAGES) mbar_wait(&empty_bar[s], ((it / STAGES) + 1) & 1);
          const uint32_t bytes = (uint32_t)p.cnt * 8u;
          mbar_arrive_expect_tx(&full_bar[s], bytes);
          if (bytes) bulk_g2s(ring + s * ST_DBL, src_of(mac, p), bytes, &full_bar[s]);
          ++it;
        }
      }
    }
    return;
  }

  // ----------------------------- consumers --------------------------------
  double *xl = W + S::xl, *z = W + S::z, *y = W + S::y, *t = W + S::t, *rfst = W + S::rfst, *ftt = W + S::ftt,
         *fts = W + S::fts, *cfgz = W + S::cfgz, *yf = W + S::yf, *wfz = W + S::wfz, *wf2 = W + S::wf2,
         *vv = W + S::vv, *cv = W + S::cv, *tg = W + S::tg, *tp = W + S::tp;
  double* wv = tg;   // W_vol contraction results, lifetime: W_vol pieces .. LU start
  double* z2 = z;    // z is dead once the W_face(z) pieces are consumed
  double* vw = vv + warp * 32;  // warp-private scratch
  int it = 0;
  for (int mac = blockIdx.x; mac < g.n_mac; mac += gridDim.x) {
    double ij[D][D];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) ij[a][b] = __ldg(g.inv_jac + (size_t)mac * D * D + a * D + b);
    double siacc = 0.0;  // per-lane partial of S^-1 y1 for the rows this lane owns
    for (int i = tid; i < LTR; i += NCONS) xl[i] = __ldg(x + __ldg(g.gather + (size_t)mac * LTR + i));
    cbar();

    int prev = -1;
    for (int pi = 0; pi < np; ++pi) {
      const Piece p = pieces[pi];
      // ---------------- phase transitions (no stage held) ----------------
      PROF_T(t_tr);
      if (p.kind != prev) {
        cbar();  // every warp has finished the previous kind
        if (p.kind == K_FST) {
          // z = A_qq^-1 A_qh x = -(fac/det) sum_f area_f n_f (Gf x_f); then cv <- 0 (aliases tg)
          const double idet = 1.0 / __ldg(g.det + mac);
          double cfl[NF][D];
#pragma unroll
          for (int f = 0; f < NF; ++f)
#pragma unroll
            for (int l = 0; l < D; ++l)
              cfl[f][l] =
                  -g.face_fac * __ldg(g.areas + mac * NF + f) * idet * __ldg(g.normals + (mac * NF + f) * D + l);
          for (int idx = tid; idx < n; idx += NCONS) {
            double acc[D] = {};
#pragma unroll
            for (int f = 0; f < NF; ++f) {
              const double tv = tg[f * n + idx];
#pragma unroll
              for (int l = 0; l < D; ++l) acc[l] += cfl[f][l] * tv;
            }
#pragma unroll
            for (int l = 0; l < D; ++l) z[l * n + idx] = acc[l];
          }
          cbar();
        } else if (p.kind == K_SI) {
          // y1 = -A_uh x + A_uq z
          // cv[K][a][s] = sum_q sum_k gphys[K,q,a,k] w[K,q][k][s]
          for (int idx = tid; idx < C::NSUB * NLOC * NS; idx += NCONS) {
            const int s = idx % NS, a = (idx / NS) % NLOC, K = idx / (NS * NLOC);
            double acc = 0.0;
#pragma unroll 4
            for (int q = 0; q < NQ; ++q) {
              const double* gr = g.grad_ref + ((K * NQ + q) * NLOC + a) * D;
              const double* w = wv + (K * NQ + q) * D * NS + s;
              double grv[D];
#pragma unroll
              for (int r2 = 0; r2 < D; ++r2) grv[r2] = __ldg(gr + r2);
#pragma unroll
              for (int k = 0; k < D; ++k) {
                double gp = 0.0;
#pragma unroll
                for (int r2 = 0; r2 < D; ++r2) gp += grv[r2] * ij[r2][k];
                acc += gp * w[k * NS];
              }
            }
            cv[idx] = acc;
          }
          for (int idx = tid; idx < LTR; idx += NCONS) {
            const int s = idx % NS, gg = (idx / NS) % LF, f = idx / BS;
            double acc = 0.0;
            for (int e = __ldg(g.fn_ptr + gg); e < __ldg(g.fn_ptr + gg + 1); ++e) {
              const int ent = __ldg(g.fn_ent + e), T = ent / NLOCF, a = ent % NLOCF;
              const double* w = wfz + ((f * NTRI + T) * NQF) * NS + s;
#pragma unroll
              for (int q = 0; q < NQF; ++q) acc += __ldg(g.phi_face + q * NLOCF + a) * w[q * NS];
            }
            cfgz[idx] = acc;
          }
          cbar();
          for (int idx = tid; idx < n; idx += NCONS) {
            const int I = idx / NS, s = idx % NS;
            double st = 0.0, sg = 0.0;
            for (int e = __ldg(g.vf_ptr + I); e < __ldg(g.vf_ptr + I + 1); ++e) st += rfst[__ldg(g.vf_ent + e) * NS + s];
            for (int e = __ldg(g.vn_ptr + I); e < __ldg(g.vn_ptr + I + 1); ++e) sg -= cv[__ldg(g.vn_sub + e) * NS + s];
            for (int e = __ldg(g.vf_ptr + I); e < __ldg(g.vf_ptr + I + 1); ++e) sg += cfgz[__ldg(g.vf_ent + e) * NS + s];
            y[idx] = -st + sg;
          }
          cbar();
        } else if (p.kind == K_MD) {
          // y <- y2 = S^-1 y1 (held in t); y2 restricted to the face nodes, for A_hu
          for (int i = tid; i < n; i += NCONS) y[i] = t[i];
          cbar();
          for (int idx = tid; idx < LTR; idx += NCONS) {
            const int s = idx % NS, h = (idx / NS) % LF, f = idx / BS;
            yf[idx] = y[__ldg(g.face_vol_nodes + f * LF + h) * NS + s];
          }
        } else if (p.kind == K_WF2) {
          // z2 = A_qq^-1 A_qu y2 = sum_r inv_jac[r][l] (M^-1 D_r y2), at the face nodes only
          constexpr int FNS = C::NFN * NS;
          for (int idx = tid; idx < FNS; idx += NCONS) {
            double tr[D];
#pragma unroll
            for (int r = 0; r < D; ++r) tr[r] = tg[r * FNS + idx];
#pragma unroll
            for (int l = 0; l < D; ++l) {
              double v = 0.0;
#pragma unroll
              for (int r = 0; r < D; ++r) v += ij[r][l] * tr[r];
              z2[l * FNS + idx] = v;
            }
          }
          cbar();
        }
      }

      if (tid == 0) { PROF_ADD(p.kind, 2, t_tr); }
      // ---------------- wait for the stage ----------------
      const int stg = it % STAGES;
      PROF_T(t_w);
      mbar_wait(&full_bar[stg], (it / STAGES) & 1);
      if (tid == 0) { PROF_ADD(p.kind, 0, t_w); }
      PROF_T(t_c);
      const double* A = ring + stg * ST_DBL;

      // ---------------- consume ----------------
      switch (p.kind) {
        case K_GF: {  // tg[f][I][s] = sum_h Gf[f][I][h] x[f][h][s]
          for (int idx = tid; idx < p.nu * NS; idx += NCONS) {
            const int s = idx % NS, rl = idx / NS, row = p.u0 + rl, f = row / L;
            const double* a = A + rl * LF;
            const double* xf = xl + f * BS + s;
            double acc = 0.0;
#pragma unroll
            for (int h = 0; h < LF; ++h) acc += a[h] * xf[h * NS];
            tg[row * NS + s] = acc;
          }
          break;
        }
        case K_MD: {  // tg[r][i][s] = sum_J (M^-1 D_r)[fnode_i][J] y2[J][s], face nodes only
          constexpr int LPR = 8, RPW = 32 / LPR;
          const int sub = lane / LPR, l = lane % LPR;
          for (int r0 = warp * RPW; r0 < p.nu; r0 += NWARP_C * RPW) {
            const int rl = r0 + sub;
            double acc[NS] = {};
            if (rl < p.nu) {
              const double* a = A + rl * L;
              for (int J = l; J < L; J += LPR) {
                const double m = a[J];
#pragma unroll
                for (int s = 0; s < NS; ++s) acc[s] += m * y[J * NS + s];
              }
            }
#pragma unroll
            for (int s = 0; s < NS; ++s)
#pragma unroll
              for (int o = LPR / 2; o > 0; o >>= 1) acc[s] += __shfl_xor_sync(MHDG_FULL, acc[s], o);
            if (l == 0 && rl < p.nu) {
#pragma unroll
              for (int s = 0; s < NS; ++s) tg[(p.u0 + rl) * NS + s] = acc[s];
            }
          }
          break;
        }
        case K_FST:
        case K_FTT:
        case K_FTS: {
          const double* vec = p.kind == K_FTS ? yf : xl;
          double* out = p.kind == K_FST ? rfst : p.kind == K_FTT ? ftt : fts;
          const int u0 = p.u0;
          rows_dot<4>(A, p.nu, BS, [&](int rl) { return vec + ((u0 + rl) / BS) * BS; },
                      [&](int rl, double acc) { out[u0 + rl] = acc; });
          break;
        }
        case K_WV: {  // warp-local: each warp its own points, PPI points per pass
          constexpr int DN = D * NS, PPI = 32 / DN;
          const int per = (p.nu + NWARP_C - 1) / NWARP_C;
          const int pbeg = warp * per, pend = min(p.nu, pbeg + per);
          const int pi = lane / DN, j = lane % DN;
          for (int pl0 = pbeg; pl0 < pend; pl0 += PPI) {
            const int pl = pl0 + pi;
            const bool on = pi < PPI && pl < pend;
            if (on) {
              const int tt = j % NS, l = j / NS, pt = p.u0 + pl, K = pt / NQ, q = pt % NQ;
              double a = 0.0;
#pragma unroll
              for (int b = 0; b < NLOC; ++b)
                a += __ldg(g.phi_vol + q * NLOC + b) * z[(l * L + __ldg(g.sub_conn + K * NLOC + b)) * NS + tt];
              vw[pi * DN + j] = a;
            }
            __syncwarp();
            if (on) {
              const int s = j % NS, k = j / NS;
              const double* w = A + pl * C::NW + k * D * NS * NS + s * NS;
              const double* v = vw + pi * DN;
              double a = 0.0;
#pragma unroll
              for (int l = 0; l < D; ++l)
#pragma unroll
                for (int tt = 0; tt < NS; ++tt) a += w[l * NS * NS + tt] * v[l * NS + tt];
              wv[(p.u0 + pl) * DN + j] = a;
            }
            __syncwarp();
          }
          break;
        }
        case K_WFZ:
        case K_WF2: {  // warp-local, as K_WV
          constexpr int DN = D * NS, PPI = 32 / DN;
          const bool second = p.kind == K_WF2;
          const double* zs = second ? z2 : z;
          const int lstride = second ? C::NFN : L;
          double* wf = p.kind == K_WFZ ? wfz : wf2;
          const int per = (p.nu + NWARP_C - 1) / NWARP_C;
          const int pbeg = warp * per, pend = min(p.nu, pbeg + per);
          const int pi = lane / DN, j = lane % DN;
          for (int pl0 = pbeg; pl0 < pend; pl0 += PPI) {
            const int pl = pl0 + pi;
            const bool on = pi < PPI && pl < pend;
            if (on) {
              const int tt = j % NS, l = j / NS;
              const int pf = p.u0 + pl, q = pf % NQF, T = (pf / NQF) % NTRI, f = pf / (NQF * NTRI);
              double a = 0.0;
#pragma unroll
              for (int b = 0; b < NLOCF; ++b) {
                int node = __ldg(g.face_vol_nodes + f * LF + __ldg(g.tri_conn + T * NLOCF + b));
                if (second) node = __ldg(g.node_to_face + node);
                a += __ldg(g.phi_face + q * NLOCF + b) * zs[(l * lstride + node) * NS + tt];
              }
              vw[pi * DN + j] = a;
            }
            __syncwarp();
            if (on && j < NS) {
              const int s = j;
              const double* w = A + pl * C::NWF + s * NS;
              const double* v = vw + pi * DN;
              double a = 0.0;
#pragma unroll
              for (int l = 0; l < D; ++l)
#pragma unroll
                for (int tt = 0; tt < NS; ++tt) a += w[l * NS * NS + tt] * v[l * NS + tt];
              wf[(p.u0 + pl) * NS + s] = a;
            }
            __syncwarp();
          }
          break;
        }
        case K_SI: {  // one column tile of a row block; warp w owns rows 8w..8w+7 of every block
          const int nb = ti_rows(n, p.blk), w = p.nu, c0 = p.u0;
          const int r = 8 * warp + (lane >> 2), l = lane & 3;
          if (c0 == 0) siacc = 0.0;
          if (r < nb) {
            const double* a = A + r * w;
            const double* yv = y + c0;
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int k = 0; k < TI_CW / 4; k += 2) {
              const int c = l + 4 * k;
              if (c < w) a0 += a[c] * yv[c];
              if (c + 4 < w) a1 += a[c + 4] * yv[c + 4];
            }
            siacc += a0 + a1;
          }
          if (c0 + w == n) {  // last tile of the block: reduce over the row's 4 lanes
            double acc = siacc;
            acc += __shfl_xor_sync(MHDG_FULL, acc, 2);
            acc += __shfl_xor_sync(MHDG_FULL, acc, 1);
            if (l == 0 && r < nb) t[p.blk * TI_RB + r] = acc;
          }
          break;
        }
      }
      __syncwarp();
      if (tid == 0) { PROF_ADD(p.kind, 1, t_c); }
      if (lane == 0) mbar_arrive(&empty_bar[stg]);
      ++it;
      prev = p.kind;
    }
    PROF_T(t_end);
    cbar();

    // y4 = ((A_hu y2 - A_hq z2) + A_hh x) - A_hq z, with -A_hq z = scale * cfg
    for (int idx = tid; idx < LTR; idx += NCONS) {
      const int s = idx % NS, gg = (idx / NS) % LF, f = idx / BS;
      double acc = 0.0;
      for (int e = __ldg(g.fn_ptr + gg); e < __ldg(g.fn_ptr + gg + 1); ++e) {
        const int ent = __ldg(g.fn_ent + e), T = ent / NLOCF, a = ent % NLOCF;
        const double* w = wf2 + ((f * NTRI + T) * NQF) * NS + s;
#pragma unroll
        for (int q = 0; q < NQF; ++q) acc += __ldg(g.phi_face + q * NLOCF + a) * w[q * NS];
      }
      const double sc = __ldg(bk.trace_face_scale + mac * NF + f);
      y_loc[(size_t)mac * LTR + idx] = ((fts[idx] + sc * acc) + ftt[idx]) + sc * cfgz[idx];
    }
    cbar();
    if (tid == 0) { PROF_ADD(12, 2, t_end); }
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

static int g_stream_grid = 0;
static int g_pref_ahead = 0;  // L2 prefetch lookahead in pieces (0: ring only)
extern "C" void mhdg_set_stream_prefetch(int pieces) { g_pref_ahead = pieces < 0 ? 0 : pieces; }
extern "C" int mhdg_stream_grid(void) { return g_stream_grid; }

template <class C>
static int count_pieces() {
  Sched<C> sc;
  Piece p;
  int k = 0;
  while (sc.next(p)) ++k;
  return k;
}

template <class C>
static bool stream_ok(const mhdg_disc& g, const mhdg_blocks& b, const mhdg_factors& f) {
  static const int npieces = count_pieces<C>();
  if (npieces > MAXP) return false;
  if (g.dim != C::D || g.L != C::L || g.Lf != C::LF || g.nloc != C::NLOC || g.nq != C::NQ || g.n_sub != C::NSUB ||
      g.n_tri != C::NTRI || g.nlocf != C::NLOCF || g.nqf != C::NQF)
    return false;
  // 16-byte alignment of every per-macro segment base
  auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  const bool sizes = ((C::NF * C::BS * C::BS) % 2 == 0) && ((C::NPV * C::NW) % 2 == 0) &&
                     ((C::NPF * C::NWF) % 2 == 0);
  return sizes && al(b.face_state_trace) && al(b.face_trace_trace) && al(b.face_trace_state) && al(b.wdgdq_vol) &&
         al(b.wdgdq_face) && al(f.lu);
}

template <class C, int STAGES>
static int launch_stream(const mhdg_disc& g, const mhdg_blocks& b, const mhdg_factors& f, const double* x,
                         double* y_loc, cudaStream_t st) {
  const size_t bytes = sizeof(double) * ((size_t)STAGES * ST_DBL + SSm<C>::total);
  auto kern = k_apply_stream<C, STAGES>;
  static int ctas = 0;
  if (!ctas) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, NCONS + 32, bytes);
    ctas = sms * (per > 0 ? per : 1);
  }
  const int grid = g.n_mac < ctas ? g.n_mac : ctas;
  g_stream_grid = grid;
  kern<<<grid, NCONS + 32, bytes, st>>>(g, b, f, x, y_loc, g_pref_ahead);
  return launch_ok();
}

#ifdef MHDG_STREAM_PROFILE
extern "C" int mhdg_stream_profile(unsigned long long* out, int reset) {
  if (out) cudaMemcpyFromSymbol(out, g_prof, sizeof(g_prof));
  if (reset) {
    unsigned long long z[16][3] = {};
    cudaMemcpyToSymbol(g_prof, z, sizeof(z));
  }
  return 0;
}
#endif

// returns -1 when no streamed instantiation matches (caller uses k_apply_local)
int apply_stream(const mhdg_disc& g, const mhdg_blocks& b, const mhdg_factors& f, const double* x, double* y_loc,
                 cudaStream_t st) {
  if (stream_ok<Cfg<2, 4, 3>>(g, b, f)) return launch_stream<Cfg<2, 4, 3>, 3>(g, b, f, x, y_loc, st);
  if (stream_ok<Cfg<2, 2, 2>>(g, b, f)) return launch_stream<Cfg<2, 2, 2>, 3>(g, b, f, x, y_loc, st);
  if (stream_ok<Cfg<3, 2, 2>>(g, b, f)) return launch_stream<Cfg<3, 2, 2>, 3>(g, b, f, x, y_loc, st);
  if (stream_ok<Cfg<3, 1, 2>>(g, b, f)) return launch_stream<Cfg<3, 1, 2>, 3>(g, b, f, x, y_loc, st);
  if (stream_ok<Cfg<3, 2, 1>>(g, b, f)) return launch_stream<Cfg<3, 2, 1>, 3>(g, b, f, x, y_loc, st);
  return -1;
}

}  // namespace mhdg
